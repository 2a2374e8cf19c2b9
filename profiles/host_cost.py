"""Host-side cost per training step of the e2e loop at C3 (native planner ->
DeviceFeeder -> chain executor): time in the feeder hand-off, the step call
and consumed(), against the device time per step (CUDA events).  When the
host is faster it blocks in the hand-off (ring backpressure).

    python profiles/host_cost.py
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
import bench  # noqa: E402
import paper_2202_13538_b200 as wj  # noqa: E402
from paper_2202_13538_b200.pipeline import BatchPlanner, DeviceFeeder, TrainConfig  # noqa: E402

cfg = bench.CONFIGS["c3"]
dev = torch.device("cuda", 0)
split, index, filt = bench.build_inputs(cfg, dev)
store = wj.preprocess(split.walk_graph, cfg["M"], cfg["L"], bench.STORE_SEED)
n = cfg["n"]
filt_rows = np.stack([split.all_edges // n, split.all_edges % n], 1)
planner = BatchPlanner(split.train_pos, filt_rows, n, TrainConfig(), np.random.default_rng(1), depth=8)
feeder = DeviceFeeder(planner, dev)
p = wj.init_params(2, cfg["L"], dropout=0.1, seed=11, device=dev)
st = wj.AdamState.for_params(p)
step = wj.TrainStep(store, p, st, use_graph=True, seed=3, launch="chain", overlap_inputs=True)
loss_h = torch.zeros(400, dtype=torch.float32).pin_memory()
N = 300
it = feeder.epoch()
for k in range(6):
    q, y, _ = next(it)
    step(q, y, loss_out=loss_h[k:k + 1])
    feeder.consumed()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
w0 = time.perf_counter()
ta = tb = tc = 0.0
for k in range(N):
    t0 = time.perf_counter()
    q, y, _ = next(it)
    t1 = time.perf_counter()
    step(q, y, loss_out=loss_h[k % 400:k % 400 + 1])
    t2 = time.perf_counter()
    feeder.consumed()
    t3 = time.perf_counter()
    ta, tb, tc = ta + t1 - t0, tb + t2 - t1, tc + t3 - t2
e1.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - w0) / N * 1e6
it.close()
print(f"host us per step: hand-off {ta / N * 1e6:.1f}, step call {tb / N * 1e6:.1f}, consumed {tc / N * 1e6:.1f}; "
      f"wall {wall:.1f}, device {e0.elapsed_time(e1) / N * 1e3:.1f}")
# the same with the GPU held by a sleep kernel: pure host enqueue cost (the
# ring backpressure blocks after a few steps, so only 3 steps are timed)
torch.cuda._sleep(500_000_000)
it = feeder.epoch()
t0 = time.perf_counter()
for k in range(3):
    q, y, _ = next(it)
    step(q, y, loss_out=loss_h[k:k + 1])
    feeder.consumed()
print(f"host us per step with the GPU busy (3 steps): {(time.perf_counter() - t0) / 3 * 1e6:.1f}")
torch.cuda.synchronize()
it.close()
