# A/B bench runs (measurement aid): alternative builds of the library
# (WJ_LIB=ab/<name>.so, profiles/ab_variant.py) vs the in-tree build,
# interleaved, REPS reps; usage: OUT=file LIBS="ab/x.so default" bash profiles/ab_libs.sh
mkdir -p gpurun_out
for rep in $(seq ${REPS:-2}); do for lib in $LIBS; do
  if [ "$lib" = default ]; then unset WJ_LIB; else export WJ_LIB=$lib; fi
  timeout 300 python bench.py --no-cpu-baseline --no-epoch --no-clocks $BENCH_ARGS > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$lib',d['value'],d['ms_per_step'],d['roofline']['kernel_ms'])" >> gpurun_out/$OUT
done; done
unset WJ_LIB
