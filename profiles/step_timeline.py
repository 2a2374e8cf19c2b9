"""Kernel timeline of the C3 training step (torch.profiler / CUPTI): start,
duration and gap of every kernel / memcpy in a few steady-state steps.

    python profiles/step_timeline.py [graph|chain]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2202_13538_b200 as wj  # noqa: E402


def main():
    cfg = bench.CONFIGS["c3"]
    dev = torch.device("cuda", 0)
    split, index, filt = bench.build_inputs(cfg, dev)
    store = wj.preprocess(split.walk_graph, cfg["M"], cfg["L"], bench.STORE_SEED)
    plan = bench.make_plan(split, index, filt, 10, bench.BATCH_SEED)
    qd = [torch.from_numpy(q).to(dev) for q, _ in plan]
    yd = [torch.from_numpy(y).to(dev) for _, y in plan]
    p = wj.init_params(2, cfg["L"], dropout=0.1, seed=11, device=dev)
    st = wj.AdamState.for_params(p)
    launch = sys.argv[1] if len(sys.argv) > 1 else "graph"
    step = wj.TrainStep(store, p, st, use_graph=True, seed=3, overlap_inputs=True, launch=launch)
    for k in range(5):
        step(qd[k], yd[k])
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for k in range(5, 10):
            step(qd[k], yd[k])
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    prev_end = None
    for e in evs:
        s, d = e.time_range.start, e.time_range.end - e.time_range.start
        gap = (s - prev_end) if prev_end is not None else 0
        print(f"{(s - t0):9.1f} us  dur {d:7.1f}  gap {gap:6.1f}  {e.name[:70]}")
        prev_end = e.time_range.end


if __name__ == "__main__":
    main()
