"""Per-unit phase durations of the join+encode kernel (debug builds with
wj_unit_ts stamps): staging, merge, rows, tiles (first member), rest."""
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
for q, y in plan:
    gb = np.empty((2 + q.shape[1]) * q.shape[0] + 2, dtype=np.int32)
    _lib.call("wj_group_queries", q.ctypes.data, q.shape[0], q.shape[1], GROUP_MAX, gb.ctypes.data, None)
    step(torch.from_numpy(q).to(dev), torch.from_numpy(y).to(dev), groups=(torch.from_numpy(gb).to(dev), int(gb[0])))
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (448 * 4 * 6))()
_lib.load().wj_debug_unit_ts(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(448, 4, 6).astype(np.int64)[:444]
names = ["stage", "merge", "rows", "(wait)+tiles m0", "red + members"]
for slot in range(3):
    x = a[:, slot]
    ok = (x > 0).all(axis=1)
    d = np.diff(x[ok], axis=1) / 1e3
    print(f"unit slot {slot}: {ok.sum()} units, total median {np.median(x[ok][:,5]-x[ok][:,0])/1e3:.2f} us")
    for k, nm in enumerate(names):
        print(f"   {nm:18s} median {np.median(d[:, k]):7.2f}  p90 {np.percentile(d[:, k], 90):7.2f} us")
