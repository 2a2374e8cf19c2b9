"""Per-CTA timeline of the join+encode kernel in the chain step (debug
builds with wj_enc_ts stamps): wait release, exit, units per CTA."""
import sys, ctypes, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
import paper_2202_13538_b200 as wj
from paper_2202_13538_b200 import _lib
from paper_2202_13538_b200.pipeline import GROUP_MAX
dev = torch.device("cuda", 0)
wl = bench.build_workload(bench.CONFIGS["c3"], dev)
store = wl.prep(wl.walk_graph)
plan = bench.make_plan(wl, 30, bench.BATCH_SEED)
p = wj.init_params(2, 4, dropout=0.1, seed=11, device=dev)
st = wj.AdamState.for_params(p)
step = wj.TrainStep(store, p, st, seed=3, launch="chain", overlap_inputs=True)
qs = []
for q, y in plan:
    gb = np.empty((2 + q.shape[1]) * q.shape[0] + 2, dtype=np.int32)
    _lib.call("wj_group_queries", q.ctypes.data, q.shape[0], q.shape[1], GROUP_MAX, gb.ctypes.data, None)
    qs.append((torch.from_numpy(q).to(dev), torch.from_numpy(y).to(dev), (torch.from_numpy(gb).to(dev), int(gb[0]))))
for k in range(30):
    q, y, g = qs[k]
    step(q, y, groups=g)
torch.cuda.synchronize()
L = _lib.load()
buf = (ctypes.c_ulonglong * (512 * 4))()
L.wj_debug_enc_ts(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(512, 4).astype(np.int64)[:444]
base = a[:, 1].min()
w = (a[:, 1] - base) / 1e3
e = (a[:, 2] - base) / 1e3
print("wait release  min/med/max us", w.min(), np.median(w), w.max())
print("CTA exit      min/med/max us", e.min(), np.median(e), e.max())
print("exit percentiles 10/50/90/99", np.percentile(e, [10, 50, 90, 99]))
print("units per CTA hist", np.bincount(a[:, 3]))
