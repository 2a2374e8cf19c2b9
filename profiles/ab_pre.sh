# A/B of the preprocess phases (measurement aid): t_pre and its phases of the
# default bench for alternative builds (WJ_LIB=ab/<name>.so) vs the in-tree one
mkdir -p gpurun_out
for rep in $(seq ${REPS:-2}); do for lib in $LIBS; do
  if [ "$lib" = default ]; then unset WJ_LIB; else export WJ_LIB=$lib; fi
  timeout 300 python bench.py --no-cpu-baseline --no-epoch --no-clocks --steps 20 > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);c=d['config'];print('$lib',c['t_pre_ms'],c['t_pre_phase_ms'])" >> gpurun_out/$OUT
done; done
unset WJ_LIB
