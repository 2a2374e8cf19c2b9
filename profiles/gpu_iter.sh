# quick GPU iteration: parity subset, bench without the CPU leg, ncu of the hot kernel
# usage (under gpurun): bash profiles/gpu_iter.sh "<pytest -k expr>" <tag>
K="${1:-fused}"; TAG="${2:-iter}"
mkdir -p gpurun_out
python -m paper_2202_13538_b200.build > /dev/null
timeout 900 python -m pytest tests -x -q -m gpu -k "$K" > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json | head -c 600; echo
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_encode -s 1 -c 1 -o gpurun_out/enc_$TAG -f python profiles/kernel_driver.py --config c3 --what enc --reps 3 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
