# full GPU check: every -m gpu test, smoke, bench (with CPU leg), launch list of a short bench
TAG="${1:-full}"
mkdir -p gpurun_out
python -m paper_2202_13538_b200.build > /dev/null
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; head -c 400 gpurun_out/bench_$TAG.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/launches_$TAG.csv x 12
