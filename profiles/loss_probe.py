"""Chain step with the loss written by the Adam kernel into pinned host
memory vs into device memory (device time per step, C3)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
import bench  # noqa: E402
import paper_2202_13538_b200 as wj  # noqa: E402
from paper_2202_13538_b200 import _lib  # noqa: E402
from paper_2202_13538_b200.pipeline import GROUP_MAX  # noqa: E402

cfg = bench.CONFIGS["c3"]
dev = torch.device("cuda", 0)
split, index, filt = bench.build_inputs(cfg, dev)
store = wj.preprocess(split.walk_graph, cfg["M"], cfg["L"], bench.STORE_SEED)
plan = bench.make_plan(split, index, filt, 16, bench.BATCH_SEED)
qs = [torch.from_numpy(q).to(dev) for q, _ in plan]
ys = [torch.from_numpy(y).to(dev) for _, y in plan]
gs = []
for q, _ in plan:
    gb = np.empty((2 + q.shape[1]) * q.shape[0] + 2, dtype=np.int32)
    _lib.call("wj_group_queries", q.ctypes.data, q.shape[0], q.shape[1], GROUP_MAX, gb.ctypes.data, None)
    gs.append((torch.from_numpy(gb).to(dev), int(gb[0])))
K = 100
loss_h = torch.zeros(K, dtype=torch.float32).pin_memory()
loss_d = torch.zeros(K, dtype=torch.float32, device=dev)
for where in ("device", "pinned", "device", "pinned"):
    p = wj.init_params(2, cfg["L"], dropout=0.1, seed=11, device=dev)
    st = wj.AdamState.for_params(p)
    step = wj.TrainStep(store, p, st, use_graph=True, seed=3, launch="chain", overlap_inputs=True)
    for k in range(8):
        step(qs[k % 16], ys[k % 16], groups=gs[k % 16])
    torch.cuda.synchronize()
    torch.cuda._sleep(2_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(K):
        out = loss_d[k:k + 1] if where == "device" else loss_h[k:k + 1]
        step(qs[k % 16], ys[k % 16], loss_out=out, groups=gs[k % 16])
    e1.record()
    torch.cuda.synchronize()
    print(f"loss in {where}: {e0.elapsed_time(e1) / K * 1e3:.1f} us/step")
