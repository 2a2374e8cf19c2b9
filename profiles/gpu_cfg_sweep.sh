# join+encode launch-shape sweep at c3 (kernel time alone + step time)
for cfg in ${CFGS:-4x3 8x2 4x2 4x4}; do
  WJ_ENC_CFG=$cfg timeout 300 python bench.py --no-cpu-baseline --steps 100 --no-epoch > gpurun_out/sweep_$cfg.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sweep_$cfg.json')); print('$cfg', 'step_ms', d['ms_per_step'], 'kernel_ms', d['roofline']['kernel_ms'])"
done
