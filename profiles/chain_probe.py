"""Chain-executor variants at C3 (device time per step, CUDA events):
device-resident inputs with / without a per-step event record, pinned host
inputs read in place with / without it.

    python profiles/chain_probe.py
"""
import sys

import torch

sys.path.insert(0, '/root/repo')
import bench  # noqa: E402
import paper_2202_13538_b200 as wj  # noqa: E402

cfg = bench.CONFIGS["c3"]
dev = torch.device("cuda", 0)
split, index, filt = bench.build_inputs(cfg, dev)
store = wj.preprocess(split.walk_graph, cfg["M"], cfg["L"], bench.STORE_SEED)
plan = bench.make_plan(split, index, filt, 16, bench.BATCH_SEED)
K = 60
for where in ("device", "pinned"):
    for ev in (False, True):
        p = wj.init_params(2, cfg["L"], dropout=0.1, seed=11, device=dev)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(store, p, st, use_graph=True, seed=3, launch="chain", overlap_inputs=True)
        step.record_input_events = False
        qs = [torch.from_numpy(q) for q, _ in plan]
        ys = [torch.from_numpy(y) for _, y in plan]
        qs = [q.to(dev) if where == "device" else q.pin_memory() for q in qs]
        ys = [y.to(dev) if where == "device" else y.pin_memory() for y in ys]
        events = [torch.cuda.Event() for _ in range(8)]
        for k in range(8):
            step(qs[k % 16], ys[k % 16])
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(K):
            step(qs[k % 16], ys[k % 16])
            if ev:
                events[k % 8].record()
        e1.record()
        torch.cuda.synchronize()
        print(f"{where:7s} event_per_step={ev}: {e0.elapsed_time(e1) / K * 1e3:.1f} us/step")
