# Round-end evidence on one B200, part A: full GPU suite, smoke, default bench
# (with the CPU baseline), reference arm, every named workload, the inference
# bench and the warm launch list of a short bench run.  Outputs in gpurun_out/.
TAG="${1:-round}"
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt
WJ_TRAIN_DROPOUT_REPORT=gpurun_out/train_dropout_$TAG.json timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; head -c 300 gpurun_out/bench_$TAG.json; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; head -c 300 gpurun_out/bench_ref_$TAG.json; echo
for c in c2 c1 c5b c5a c4; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "$c $(head -c 120 gpurun_out/bench_${c}_$TAG.json)"
done
timeout 600 python bench.py --what infer > gpurun_out/bench_infer_$TAG.json 2> gpurun_out/bench_infer_$TAG.err; head -c 300 gpurun_out/bench_infer_$TAG.json; echo
timeout 600 python bench.py --what infer --impl reference --steps 2 --warmup 1 > gpurun_out/bench_infer_ref_$TAG.json 2> gpurun_out/bench_infer_ref_$TAG.err; head -c 300 gpurun_out/bench_infer_ref_$TAG.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-epoch > /dev/null 2>&1
ls -la gpurun_out | tail -40
