# A/B of the end-to-end t_pre (measurement aid): env settings, default bench
# with the full-epoch e2e; usage: OUT=file ENVS="A=1 A=2" REPS=2 bash profiles/ab_e2e.sh
mkdir -p gpurun_out
for rep in $(seq ${REPS:-2}); do for e in $ENVS; do
  env $e WJ_PLANNER_TIMING=1 timeout 400 python bench.py --no-cpu-baseline --no-clocks --steps 20 > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);e=d['e2e'];p=e['t_pre_parts_ms'];print('$e',e['value'],e['t_pre_ms'],p['preprocess_device'],p['planner_ready'],p['preprocess_phases']['before_first_phase'])" >> gpurun_out/$OUT
  grep "wj_planner_create" gpurun_out/ab.err | tail -2 >> gpurun_out/$OUT
done; done
