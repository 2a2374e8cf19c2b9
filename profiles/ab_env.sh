# A/B bench runs (measurement aid): env settings of one build, interleaved;
# usage: OUT=file ENVS="WJ_X=0 WJ_X=1" REPS=2 bash profiles/ab_env.sh
mkdir -p gpurun_out
for rep in $(seq ${REPS:-2}); do for e in $ENVS; do
  env $e timeout 300 python bench.py --no-cpu-baseline --no-epoch --no-clocks $BENCH_ARGS > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$e',d['value'],d['ms_per_step'],d['roofline']['kernel_ms'])" >> gpurun_out/$OUT || echo "$e FAILED" >> gpurun_out/$OUT
done; done
