import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2202_13538_b200.pipeline import BatchPlanner, TrainConfig
wl = bench.build_workload(bench.CONFIGS["c3"], torch.device("cuda", 0))
for r in range(4):
    t = time.perf_counter()
    pl = BatchPlanner(wl.train_pos, wl.filter_rows, wl.n, TrainConfig(batch_size=32, k_neg=50), np.random.default_rng(7), depth=8, background=True)
    pl.wait()
    print("build", r, (time.perf_counter() - t) * 1e3, "ms", flush=True)
    pl.close()
print(os.cpu_count(), open("/sys/kernel/mm/transparent_hugepage/enabled").read(), open("/sys/kernel/mm/transparent_hugepage/defrag").read())
