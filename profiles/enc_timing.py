"""Time wj_join_encode alone on the C3 store (CUDA events, K batches).

    python profiles/enc_timing.py [--config c3] [--reps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2202_13538_b200 as wj  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--repeat", type=int, default=5)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    split, index, filt = bench.build_inputs(cfg, dev)
    store = wj.preprocess(split.walk_graph, cfg["M"], cfg["L"], bench.STORE_SEED)
    plan = bench.make_plan(split, index, filt, a.reps, bench.BATCH_SEED)
    qd = [torch.from_numpy(q).to(dev) for q, _ in plan]
    p = wj.init_params(cfg["A"], cfg["L"], dropout=0.1, seed=11, device=dev)
    step_t = torch.zeros(1, dtype=torch.int64, device=dev)
    B = max(q.shape[0] for q in qd)
    AW = cfg["A"] * (cfg["L"] + 1)
    pooled = torch.empty((B, 64), device=dev)
    S = torch.empty((B, AW, 64), device=dev)
    ms = torch.empty((B, 64), device=dev)
    t = p.tensors

    cross = torch.empty((B, 2, 1, store.max_unique), dtype=torch.int32, device=dev)
    use_cross = os.environ.get("WJ_CROSS") is not None  # precomputed cross ids (else in-kernel merge)

    def run():
        for q in qd:
            c = wj.encoder.join_cross(store, q, cross[: q.shape[0]]) if use_cross else None
            wj.encoder.join_encode(store, q, t["w1"], t["b1"], 0.9, 5, step_t, pooled, S, ms, cross=c)

    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(a.repeat):
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / len(qd))
    ms_k = min(times)
    # the cross-id kernel alone
    tc = []
    for _ in range(a.repeat):
        e0.record()
        for q in qd:
            wj.encoder.join_cross(store, q, cross[: q.shape[0]])
        e1.record()
        torch.cuda.synchronize()
        tc.append(e0.elapsed_time(e1) / len(qd))
    print(json.dumps({"config": a.config, "cfg": os.environ.get("WJ_ENC_CFG", "default"), "cross": use_cross,
                      "kernel_ms": round(ms_k, 4), "cross_ms": round(min(tc), 4), "mu": store.max_unique,
                      "q_per_batch": sum(q.shape[0] for q in qd) / len(qd)}))


if __name__ == "__main__":
    main()
