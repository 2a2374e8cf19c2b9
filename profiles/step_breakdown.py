"""Where the training step's time goes (C3): full step() vs graph replay alone
vs the per-step input copies, CUDA events on the current stream.

    python profiles/step_breakdown.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2202_13538_b200 as wj  # noqa: E402


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main():
    cfg = bench.CONFIGS["c3"]
    dev = torch.device("cuda", 0)
    split, index, filt = bench.build_inputs(cfg, dev)
    store = wj.preprocess(split.walk_graph, cfg["M"], cfg["L"], bench.STORE_SEED)
    plan = bench.make_plan(split, index, filt, 8, bench.BATCH_SEED)
    qd = [torch.from_numpy(q).to(dev) for q, _ in plan]
    yd = [torch.from_numpy(y).to(dev) for _, y in plan]
    p = wj.init_params(2, cfg["L"], dropout=0.1, seed=11, device=dev)
    st = wj.AdamState.for_params(p)
    step = wj.TrainStep(store, p, st, use_graph=True, seed=3, overlap_inputs=True)
    for k in range(4):
        step(qd[k], yd[k])
    g = step._graphs[(qd[0].shape[0], 2)][0]
    out = {
        "step_us": timed(lambda: step(qd[0], yd[0]), 50),
        "replay_us": timed(lambda: g["graph"].replay(), 50),
        "copies_us": timed(lambda: (g["q"].copy_(qd[0], non_blocking=True), g["y"].copy_(yd[0], non_blocking=True)), 50),
    }
    print(json.dumps({k: round(v, 2) for k, v in out.items()}))


if __name__ == "__main__":
    main()
