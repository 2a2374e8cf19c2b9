# Round-end evidence on one B200: full GPU suite, smoke, bench (with the CPU
# baseline), warm launch list of a short bench run, ncu --set full of every
# step kernel and of the preprocess kernels.  Outputs under gpurun_out/.
TAG="${1:-round}"
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt
python -m paper_2202_13538_b200.build > gpurun_out/build_$TAG.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; head -c 300 gpurun_out/bench_$TAG.json; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; head -c 300 gpurun_out/bench_ref_$TAG.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_encode -s 2 -c 1 -o gpurun_out/enc_$TAG -f python profiles/kernel_driver.py --config c3 --what chain --reps 4 > gpurun_out/ncu_enc_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:tail_tc|adam" -s 2 -c 2 -o gpurun_out/tail_$TAG -f python profiles/kernel_driver.py --config c3 --what chain --reps 4 > gpurun_out/ncu_tail_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:rpe_kernel|sample_walks|intern|vindex" -o gpurun_out/pre_$TAG -f python profiles/kernel_driver.py --config c3 --what preprocess > gpurun_out/ncu_pre_$TAG.log 2>&1
ls -la gpurun_out | tail -30
