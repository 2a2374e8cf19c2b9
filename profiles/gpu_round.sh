set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_encode -s 1 -c 1 -o gpurun_out/enc_full -f python profiles/kernel_driver.py --config c3 --what enc --reps 3 > gpurun_out/ncu_enc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rpe_kernel -c 2 -o gpurun_out/rpe_full -f python profiles/kernel_driver.py --config c3 --what preprocess > gpurun_out/ncu_rpe.log 2>&1
ls -la gpurun_out
