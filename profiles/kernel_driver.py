"""Small driver for ncu captures of the hot-path kernels (run under gpurun).

    ncu ... python profiles/kernel_driver.py --config c2 --what preprocess
    ncu ... python profiles/kernel_driver.py --config c3 --what join --reps 3
    ncu ... python profiles/kernel_driver.py --config c3 --what step --reps 3
    ncu ... python profiles/kernel_driver.py --config c3 --what chain --reps 4   (the bench's step
        executor: dynamic scheduling over query groups)
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2202_13538_b200 as wj  # noqa: E402
from paper_2202_13538_b200.joiner import dense_batch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--what", default="join", choices=["preprocess", "join", "step", "enc", "chain", "score"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dense", default="float32")
    ap.add_argument("--mode", default="fused")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    wl = bench.build_workload(cfg, dev)
    store = wl.prep(wl.walk_graph)
    if a.what == "preprocess":
        torch.cuda.synchronize()
        return
    if a.what == "score":  # the inference scorer (keep = 1 join+encode + logits tail)
        p = wj.init_params(cfg["A"], cfg["L"], dropout=0.1, seed=11, device=dev)
        sc = wj.encoder.FusedScorer(p, store)
        for c in bench.infer_queries(wl, a.reps, bench.BATCH_SEED + 100):
            sc.logits(torch.from_numpy(c).to(dev))
        torch.cuda.synchronize()
        return
    split, index, filt = wl, None, None
    plan = bench.make_plan(split, index, filt, a.reps, bench.BATCH_SEED)
    qd = [torch.from_numpy(q).to(dev) for q, _ in plan]
    yd = [torch.from_numpy(y).to(dev) for _, y in plan]
    if a.what == "join":
        dt = getattr(torch, a.dense)
        for q in qd:
            dense_batch(store, q, dtype=dt, validate=False)
    elif a.what == "enc":
        p = wj.init_params(cfg["A"], cfg["L"], dropout=0.1, seed=11, device=dev)
        step_t = torch.zeros(1, dtype=torch.int64, device=dev)
        for q in qd:
            wj.encoder.forward_fused(p, store, q, training=True, seed=3, step=step_t)
    elif a.what == "chain":
        from paper_2202_13538_b200 import _lib
        from paper_2202_13538_b200.pipeline import GROUP_MAX

        p = wj.init_params(cfg["A"], cfg["L"], dropout=0.1, seed=11, device=dev)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(store, p, st, use_graph=True, launch="chain", seed=3)
        for (q, _), qq, y in zip(plan, qd, yd):
            gb = np.empty((2 + q.shape[1]) * q.shape[0] + 2, dtype=np.int32)
            _lib.call("wj_group_queries", q.ctypes.data, q.shape[0], q.shape[1], GROUP_MAX, gb.ctypes.data, None)
            step(qq, y, groups=(torch.from_numpy(gb).to(dev), int(gb[0])))
    else:
        p = wj.init_params(cfg["A"], cfg["L"], dropout=0.1, seed=11, device=dev)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(store, p, st, use_graph=False, mode=a.mode)
        for q, y in zip(qd, yd):
            step(q, y)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
