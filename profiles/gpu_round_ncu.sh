# Round-end evidence, part B: ncu --set full of the step kernels, the scorer and
# the preprocess kernels, summarised ON the box (text + JSON); only the
# join+encode report is kept (gpurun copies back <= 64 MiB).
TAG="${1:-round}"
mkdir -p gpurun_out
summ() {  # rep name
  ncu -i gpurun_out/$1.ncu-rep --page details > gpurun_out/ncu_$1_details.txt 2>&1
  python profiles/ncu_source_top.py gpurun_out/$1.ncu-rep 30 > gpurun_out/ncu_$1_top.txt 2>&1
}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_encode -s 2 -c 1 -o gpurun_out/enc_$TAG -f python profiles/kernel_driver.py --config c3 --what chain --reps 4 > /dev/null 2>&1
summ enc_$TAG; python profiles/ncu_summary.py gpurun_out/enc_$TAG.ncu-rep c3 wj_join_encode > /dev/null; cp profiles/c3_wj_join_encode_ncu.json gpurun_out/
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:tail_tc|adam" -s 2 -c 2 -o gpurun_out/tail_$TAG -f python profiles/kernel_driver.py --config c3 --what chain --reps 4 > /dev/null 2>&1
summ tail_$TAG; rm -f gpurun_out/tail_$TAG.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:infer_shared -s 2 -c 1 -o gpurun_out/score_$TAG -f python profiles/kernel_driver.py --config c3 --what score --reps 4 > /dev/null 2>&1
summ score_$TAG; python profiles/ncu_summary.py gpurun_out/score_$TAG.ncu-rep c3 wj_score_shared > /dev/null; cp profiles/c3_wj_score_shared_ncu.json gpurun_out/; rm -f gpurun_out/score_$TAG.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:rpe_kernel|sample_walks|intern|vindex|rpe_count" -o gpurun_out/pre_$TAG -f python profiles/kernel_driver.py --config c3 --what preprocess > /dev/null 2>&1
summ pre_$TAG; rm -f gpurun_out/pre_$TAG.ncu-rep
du -sh gpurun_out; ls gpurun_out
