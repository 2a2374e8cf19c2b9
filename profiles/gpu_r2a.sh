mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_r2a.txt
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 600 > gpurun_out/pytest_r2a.log 2>&1; tail -5 gpurun_out/pytest_r2a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2a.log 2>&1; tail -1 gpurun_out/smoke_r2a.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; head -c 600 gpurun_out/bench_r2a.json; echo
