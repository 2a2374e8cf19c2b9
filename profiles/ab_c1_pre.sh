# C1 preprocess phases for alternative builds (measurement aid)
mkdir -p gpurun_out
for rep in $(seq ${REPS:-3}); do for lib in $LIBS; do
  if [ "$lib" = default ]; then unset WJ_LIB; else export WJ_LIB=$lib; fi
  timeout 300 python bench.py --config c1 --no-cpu-baseline --no-epoch --no-clocks --steps 20 > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);c=d['config'];print('$lib',d['value'],c['t_pre_ms'],c['t_pre_phase_ms'])" >> gpurun_out/$OUT
done; done
unset WJ_LIB
