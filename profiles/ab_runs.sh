# A/B bench runs (measurement aid): env variants of one build, interleaved, two reps
mkdir -p gpurun_out
for rep in 1 2; do for v in 3 1 0 2 F1; do
  if [ "$v" = F1 ]; then f=1; vv=1; else f=0; vv=$v; fi
  WJ_FUSED_ADAM=$f WJ_TAIL_VARIANT=$vv timeout 300 python bench.py --no-cpu-baseline --no-epoch --no-clocks > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('v=$v',d['value'],d['ms_per_step'],d['roofline']['kernel_ms'])" >> gpurun_out/$OUT
done; done
