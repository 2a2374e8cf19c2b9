"""Small invocation of every hot-path kernel, for compute-sanitizer
(memcheck / racecheck / synccheck): sampler (+ dead-end fix-up), RPE count /
fill, interning, vindex, join (dense + ids), join+encode (mma.sync and
tcgen05 kernels, dynamic scheduling over query groups, keep < 1 and keep = 1),
encoder tail + Adam through the step executor, the native epoch loop, the
typed sampler and the SURL pack.

    compute-sanitizer --tool memcheck python profiles/sanitize_driver.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_13538_b200 as wj  # noqa: E402
from paper_2202_13538_b200.pipeline import BatchPlanner, TrainConfig  # noqa: E402


def main():
    rng = np.random.default_rng(1)
    n = 600
    edges = rng.integers(0, n, size=(3000, 2))
    g = wj.Graph.from_edges(edges, n)
    s = wj.preprocess(g, 24, 4, 5)                    # sampler, rpe count/fill, intern, vindex
    # a non-symmetric CSR with dead ends (fix-up launch)
    ip = np.array([0, 1, 2, 2], dtype=np.int64)
    ix = np.array([1, 2], dtype=np.int32)
    wj.preprocess(wj.Graph(3, ip, ix), 8, 3, 2)
    q = np.stack([rng.choice(n, 2, replace=False) for _ in range(40)]).astype(np.int64)
    q[5] = q[4]                                       # identical queries -> query groups
    wj.join_batch_arrays(s, q)
    wj.dense_batch(s, torch.from_numpy(q).cuda(), dtype=torch.float32)
    for tc in ("0", "8"):
        os.environ["WJ_ENC_TC"] = tc
        p = wj.init_params(2, 4, dropout=0.1, seed=3)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(s, p, st, seed=7, launch="chain")
        y = torch.from_numpy((np.arange(40) % 5 == 0).astype(np.float32)).cuda()
        for _ in range(2):
            step(torch.from_numpy(q).cuda(), y)
        wj.score_array(s, p, q)                       # keep = 1 variant + logits tail
        pos = np.stack([rng.choice(n, 2, replace=False) for _ in range(120)]).astype(np.int64)
        planner = BatchPlanner(pos, pos, n, TrainConfig(batch_size=8, k_neg=3), np.random.default_rng(2), depth=4)
        step.run_epoch(planner, max_steps=6)          # native epoch loop
        planner.close()
    os.environ["WJ_ENC_TC"] = "0"
    # the shared-first-anchor scorer, dense enough for several co-reached rounds
    g2 = wj.Graph.from_edges(rng.integers(0, 300, size=(6000, 2)), 300)
    s2 = wj.preprocess(g2, 64, 4, 8)
    p2 = wj.init_params(2, 4, dropout=0.1, seed=4)
    qs = np.concatenate([np.stack([np.full(40, u), rng.integers(0, 300, 40)], 1)
                         for u in rng.choice(300, 3, replace=False)]).astype(np.int64)
    os.environ["WJ_SCORE_SHARED"] = "1"
    wj.score_array(s2, p2, qs)
    del os.environ["WJ_SCORE_SHARED"]
    et = wj.edge_types_from_node_types(g, (np.arange(n) % 2), 2)
    wj.preprocess_typed(g, et, [1, 2], 10, 3, 4)      # typed sampler
    torch.cuda.synchronize()
    print("sanitize driver done")


if __name__ == "__main__":
    main()
