"""Host cost of the native planner per C3 batch (synchronous next(), which
also groups the batch's identical queries), vs the device step time."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
import bench  # noqa: E402
from paper_2202_13538_b200 import _lib  # noqa: E402
from paper_2202_13538_b200.pipeline import GROUP_MAX, BatchPlanner, TrainConfig  # noqa: E402

cfg = bench.CONFIGS["c3"]
split, index, filt = bench.build_inputs(cfg, torch.device("cuda", 0))
n = cfg["n"]
filt_rows = np.stack([split.all_edges // n, split.all_edges % n], 1)
t0 = time.perf_counter()
bp = BatchPlanner(split.train_pos, filt_rows, n, TrainConfig(), np.random.default_rng(1), depth=8)
print(f"planner build {1e3 * (time.perf_counter() - t0):.1f} ms")
lib = _lib.load()
o = bp._out
q0, y0 = bp._q[0].data_ptr(), bp._y[0].data_ptr()
for k in range(20):
    lib.wj_planner_next(bp._h, q0, y0, bp.cap, ctypes.byref(o, 0), ctypes.byref(o, 8), ctypes.byref(o, 16))
N = 500
t0 = time.perf_counter()
for k in range(N):
    lib.wj_planner_next(bp._h, q0, y0, bp.cap, ctypes.byref(o, 0), ctypes.byref(o, 8), ctypes.byref(o, 16))
t1 = time.perf_counter()
g0 = bp._g[0].data_ptr()
for k in range(N):
    lib.wj_group_queries(q0, int(o[0]), 2, GROUP_MAX, g0, None)
t2 = time.perf_counter()
print(f"plan {1e6 * (t1 - t0) / N:.1f} us/batch, group {1e6 * (t2 - t1) / N:.1f} us/batch")
