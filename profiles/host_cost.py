"""Host-side cost of one TrainStep call (pinned host inputs, C2 store): the
GPU is held busy by a sleep kernel so only the Python/driver enqueue time
is measured.

    python profiles/host_cost.py
"""
import time, torch, sys
sys.path.insert(0, '/root/repo')
import bench, paper_2202_13538_b200 as wj
cfg = bench.CONFIGS["c2"]
dev = torch.device("cuda", 0)
split, index, filt = bench.build_inputs(cfg, dev)
store = wj.preprocess(split.walk_graph, cfg["M"], cfg["L"], bench.STORE_SEED)
plan = bench.make_plan(split, index, filt, 8, 1)
qh = [torch.from_numpy(q).pin_memory() for q, _ in plan]
yh = [torch.from_numpy(y).pin_memory() for _, y in plan]
p = wj.init_params(2, cfg["L"], dropout=0.1, seed=11, device=dev)
st = wj.AdamState.for_params(p)
step = wj.TrainStep(store, p, st, use_graph=True, seed=3)
for k in range(4): step(qh[k % 8], yh[k % 8])
torch.cuda.synchronize()
torch.cuda._sleep(200_000_000)
t0 = time.perf_counter()
for k in range(200): step(qh[k % 8], yh[k % 8])
t1 = time.perf_counter()
torch.cuda.synchronize()
print("host us per step call:", (t1 - t0) / 200 * 1e6)
