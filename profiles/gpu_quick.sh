# quick GPU check: a pytest subset, bench without the CPU leg, warm launch list of a short bench
K="${1:-fused}"; TAG="${2:-quick}"
mkdir -p gpurun_out
python -m paper_2202_13538_b200.build > /dev/null
timeout 900 python -m pytest tests -x -q -m gpu -k "$K" > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; head -c 300 gpurun_out/bench_$TAG.json; echo
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('kernel_ms', d['roofline']['kernel_ms'], 'ns_frac', d['roofline']['north_star']['frac'], 'e2e', d['e2e'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k "regex:tail|adam|join_encode|sum_rows" -c 300 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/launches_$TAG.csv x 14
