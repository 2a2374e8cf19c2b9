# end-game splitting sweep at c3: step and kernel time per WJ_SPLIT_UNITS
timeout 300 python -m pytest tests/test_gpu_chain.py -x -q --timeout 200 2>&1 | tail -1
for k in ${KS:-0 75 100 150 200 300}; do
  WJ_SPLIT_UNITS=$k timeout 300 python bench.py --no-cpu-baseline --steps 200 --no-epoch > gpurun_out/split_$k.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/split_$k.json')); print('split', $k, 'step_ms', d['ms_per_step'], 'kernel_ms', d['roofline']['kernel_ms'], 'value', d['value'])"
done
