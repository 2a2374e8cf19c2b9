# tcgen05 kernel check: fused-kernel GPU tests, then the bench (no CPU leg)
TAG="${1:-tc}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests -x -q -m gpu --timeout 60 -k "fused or dropout or chain or no_dropout" > gpurun_out/pytest_$TAG.log 2>&1; tail -15 gpurun_out/pytest_$TAG.log
timeout 240 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; head -c 400 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('kernel_ms', d['roofline']['kernel_ms'], 'e2e', d['e2e']['value'])"
