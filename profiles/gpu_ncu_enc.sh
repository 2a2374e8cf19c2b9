# ncu --set full of the step kernels (join+encode, tail, adam) as the bench launches them.
TAG="${1:-enc}"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_encode -s 2 -c 1 -o gpurun_out/enc_$TAG -f python profiles/kernel_driver.py --config c3 --what chain --reps 4 > gpurun_out/ncu_enc_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:tail_tc|adam" -s 2 -c 2 -o gpurun_out/tail_$TAG -f python profiles/kernel_driver.py --config c3 --what chain --reps 4 > gpurun_out/ncu_tail_$TAG.log 2>&1
tail -3 gpurun_out/ncu_enc_$TAG.log
