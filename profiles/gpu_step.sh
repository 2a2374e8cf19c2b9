# train-step iteration: fused tests, bench (no CPU leg), launch times of the step kernels
TAG="${1:-step}"
mkdir -p gpurun_out
python -m paper_2202_13538_b200.build > gpurun_out/build_$TAG.log 2>&1 || { tail -20 gpurun_out/build_$TAG.log; exit 1; }
timeout 600 python -m pytest tests -x -q -m gpu -k "fused or dropout or encoder or train or dist" > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('value', d['value'], 'ms/step', d['ms_per_step'], 'kernel_ms', d['roofline']['kernel_ms'], 'ns_frac', d['roofline']['north_star']['frac'], 'e2e', d['e2e']['value'], 'pre', d['config']['t_pre_phase_ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:join_encode|adam|tail|grad" --csv --log-file gpurun_out/launch_$TAG.csv python profiles/kernel_driver.py --config c3 --what step --reps 6 > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/launch_$TAG.csv x 10
