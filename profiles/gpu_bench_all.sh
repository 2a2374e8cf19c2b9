# Every named workload at N=1 (train), the c3 inference bench, and the ncu
# summaries (issue roof, DRAM traffic) the bench lines read.  Outputs in gpurun_out/.
TAG="${1:-r02}"
mkdir -p gpurun_out
for c in c3 c2 c1 c5b c5a c4; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
  echo "$c rc=$? $(head -c 200 gpurun_out/bench_${c}_$TAG.json)"; tail -2 gpurun_out/bench_${c}_$TAG.err
done
timeout 300 python bench.py --what infer --no-cpu-baseline > gpurun_out/bench_infer_c3_$TAG.json 2> gpurun_out/bench_infer_c3_$TAG.err
echo "infer rc=$? $(head -c 300 gpurun_out/bench_infer_c3_$TAG.json)"; tail -2 gpurun_out/bench_infer_c3_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_encode -s 2 -c 1 -o gpurun_out/enc_$TAG -f python profiles/kernel_driver.py --config c3 --what chain --reps 4 > gpurun_out/ncu_enc_$TAG.log 2>&1
python profiles/ncu_summary.py gpurun_out/enc_$TAG.ncu-rep c3 wj_join_encode | cut -c1-300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_encode -s 2 -c 1 -o gpurun_out/score_$TAG -f python profiles/kernel_driver.py --config c3 --what score --reps 4 > gpurun_out/ncu_score_$TAG.log 2>&1
python profiles/ncu_summary.py gpurun_out/score_$TAG.ncu-rep c3 wj_join_encode_infer | cut -c1-300
