import sys, ctypes, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
import paper_2202_13538_b200 as wj
from paper_2202_13538_b200 import _lib
from paper_2202_13538_b200.pipeline import GROUP_MAX
dev = torch.device("cuda", 0)
cfg = bench.CONFIGS["c3"]
wl = bench.build_workload(cfg, dev)
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
buf = (ctypes.c_ulonglong * (128 * 12))()
L.wj_debug_tail_ts(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(128, 12).astype(np.int64)
rows = 102
t = a[:rows, :10]
base = t[:, 1].min()
print("tail phases (us rel. to first pdl_wait return): min / median / max over CTAs")
names = ["launch", "wait_ret", "pooled_rdy", "prod1", "prod2", "dW", "S_rdy", "loop_end", "stage_done", "row_written"]
for k in range(10):
    v = (t[:, k] - base) / 1e3
    print(f"{names[k]:12s} {v.min():8.2f} {np.median(v):8.2f} {v.max():8.2f}")
ad = a[:128, 10:12]
print("adam launch min/max", (ad[:, 0].min() - base) / 1e3, (ad[:, 0].max() - base) / 1e3, " wait_ret min/max", (ad[:, 1].min() - base) / 1e3, (ad[:, 1].max() - base) / 1e3)
