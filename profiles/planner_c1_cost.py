"""Host cost of the native batch planner at the C1 shape (measurement aid):
synchronous wj_planner_next + wj_group_queries per batch, and the epoch
producer thread's throughput (acquire / release loop, no device work).

    python profiles/planner_c1_cost.py
"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_13538_b200 import _lib  # noqa: E402
from paper_2202_13538_b200.pipeline import GROUP_MAX, BatchPlanner, TrainConfig  # noqa: E402

rng = np.random.default_rng(0)
n, m = 10_000, 100_000
e = rng.integers(0, n, size=(m, 2))
e = e[e[:, 0] != e[:, 1]]
key = np.unique(np.minimum(e[:, 0], e[:, 1]) * n + np.maximum(e[:, 0], e[:, 1]))
allr = np.stack([key // n, key % n], 1)
tr = allr[rng.permutation(len(allr))[: int(0.05 * len(allr))]]
lib = _lib.load()
cfg = TrainConfig(batch_size=32, k_neg=50)
bp = BatchPlanner(tr, allr, n, cfg, np.random.default_rng(1), depth=8, pinned=False)
o = bp._out
q, y, g = bp._q[0], bp._y[0], bp._g[0]
tp = tg = 0.0
K = 150
for _ in range(K):
    t0 = time.perf_counter()
    lib.wj_planner_next(bp._h, q.data_ptr(), y.data_ptr(), bp.cap, ctypes.byref(o, 0), ctypes.byref(o, 8),
                        ctypes.byref(o, 16))
    t1 = time.perf_counter()
    lib.wj_group_queries(q.data_ptr(), int(o[0]), 2, GROUP_MAX, g.data_ptr(), None)
    tp += t1 - t0
    tg += time.perf_counter() - t1
print(f"sync: plan {tp / K * 1e6:.1f} us, group (hashed) {tg / K * 1e6:.1f} us per batch")
for rep in range(3):
    bp = BatchPlanner(tr, allr, n, cfg, np.random.default_rng(1), depth=8, pinned=False)
    s, nq, npos = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
    t0 = time.perf_counter()
    lib.wj_planner_start_epoch(bp._h, ctypes.c_void_p(bp._q.data_ptr()), ctypes.c_void_p(bp._y.data_ptr()),
                               ctypes.c_void_p(bp._g.data_ptr()), 8, ctypes.c_int64(bp.cap))
    k = 0
    while True:
        lib.wj_planner_acquire(bp._h, ctypes.byref(s), ctypes.byref(nq), ctypes.byref(npos))
        if nq.value == 0:
            break
        lib.wj_planner_release(bp._h, s)
        k += 1
    print(f"producer: {k} batches, {(time.perf_counter() - t0) / k * 1e6:.1f} us per batch")
