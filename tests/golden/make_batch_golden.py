"""Golden training-batch sequences from the REAL reference (build container only).

    python tests/golden/make_batch_golden.py

Drives the reference's own ``sample_minibatch`` + ``sample_negatives`` (or the
fixed-pool draw) exactly as ``train`` does per batch (pipeline.py:287-305,
pos_filter built as at pipeline.py:278-280) for a few epochs, and records the
inputs (positives, filter tuples, pool, config, seed), every batch's queries
and labels, and the generator's final PCG64 state.  The native planner
(csrc/planner.cpp) must reproduce each sequence exactly
(tests/test_planner.py).  Cases: the reference's SBM link split (arity 2),
random hyperedges (arity 3), the fixed negative pool, and a small
batch_capacity that makes the BFS stop on the seed-node limit.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import walkjoin  # noqa: E402,F401  (sets NUMBA_NUM_THREADS before numba loads)
import numpy as np  # noqa: E402
from walkjoin import graph as G  # noqa: E402
from walkjoin import pipeline as P  # noqa: E402
from walkjoin._seeds import derive_seed  # noqa: E402
from walkjoin.graph import Query  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "batches")


def run(name, positives, extra_filter, num_nodes, cfg, epochs, pool=None):
    pos_q = [Query(tuple(int(v) for v in r), 1) for r in positives]
    index = P.QueryOverlapIndex(pos_q)
    pos_filter = {P.canonical_nodes(q.nodes) for q in pos_q}
    pos_filter.update(P.canonical_nodes(r) for r in extra_filter)
    rng = np.random.default_rng(derive_seed(cfg.seed, "minibatch"))
    pool_q = None if pool is None else [Query(tuple(int(v) for v in r), 0) for r in pool]
    qs, ys, sizes, epoch_of = [], [], [], []
    for ep in range(epochs):
        consumed = 0
        while consumed < len(pos_q):  # pipeline.py:292-305
            seed_list, batch_ids = P.sample_minibatch(index, pos_q, cfg, rng)
            if not batch_ids:
                break
            pos_batch = [pos_q[i] for i in batch_ids]
            n_neg = cfg.k_neg * len(pos_batch)
            if pool_q:
                picks = rng.integers(0, len(pool_q), size=n_neg)
                negs = [pool_q[int(i)] for i in picks]
            else:
                negs = P.sample_negatives(seed_list, len(positives[0]), n_neg, pos_filter, rng)
            q = np.array([x.nodes for x in pos_batch + negs], dtype=np.int64)
            qs.append(q)
            ys.append(np.concatenate([np.ones(len(pos_batch)), np.zeros(len(negs))]).astype(np.float32))
            sizes.append(len(q))
            epoch_of.append(ep)
            consumed += len(pos_batch)
    st = rng.bit_generator.state
    m64 = (1 << 64) - 1
    words = np.array([st["state"]["state"] >> 64, st["state"]["state"] & m64, st["state"]["inc"] >> 64,
                      st["state"]["inc"] & m64, st["has_uint32"], st["uinteger"]], dtype=np.uint64)
    np.savez_compressed(
        os.path.join(OUT, name + ".npz"), positives=np.asarray(positives, np.int64),
        filter_extra=np.asarray(extra_filter, np.int64).reshape(-1, len(positives[0])),
        pool=np.zeros((0, len(positives[0])), np.int64) if pool is None else np.asarray(pool, np.int64),
        num_nodes=num_nodes, batch_capacity=cfg.batch_capacity, batch_size=cfg.batch_size, k_neg=cfg.k_neg,
        seed=cfg.seed, epochs=epochs, queries=np.concatenate(qs), labels=np.concatenate(ys),
        sizes=np.asarray(sizes, np.int64), epoch_of=np.asarray(epoch_of, np.int64), final_rng=words)
    print(name, "batches", len(sizes), "queries", int(np.sum(sizes)))


def main():
    os.makedirs(OUT, exist_ok=True)
    # reference SBM link split (graph.py:239-354)
    g = G.generate_sbm(2, 150, 0.08, 0.01, seed=1)
    split = G.split_link_queries(g, train_frac=0.7, k_neg=5, seed=1)
    qa = lambda qs: np.asarray([q.nodes for q in qs], dtype=np.int64).reshape(-1, 2)  # noqa: E731
    run("sbm2x150", qa(split.train_pos), np.concatenate([qa(split.valid_pos), qa(split.test_pos)]),
        g.num_nodes, P.TrainConfig(seed=4, k_neg=50), epochs=2)
    run("sbm2x150_k3_bs8", qa(split.train_pos), np.concatenate([qa(split.valid_pos), qa(split.test_pos)]),
        g.num_nodes, P.TrainConfig(seed=9, k_neg=3, batch_size=8), epochs=2)
    # capacity-bound BFS: the seed set stops growing at 6 nodes
    run("sbm2x150_cap6", qa(split.train_pos), qa(split.valid_pos), g.num_nodes,
        P.TrainConfig(seed=2, k_neg=2, batch_capacity=6, batch_size=32), epochs=1)
    # fixed negative pool (pipeline.py:298-300)
    rng = np.random.default_rng(11)
    pool = np.array([rng.choice(g.num_nodes, 2, replace=False) for _ in range(400)], dtype=np.int64)
    run("sbm2x150_pool", qa(split.train_pos), qa(split.valid_pos), g.num_nodes,
        P.TrainConfig(seed=5, k_neg=10), epochs=1, pool=pool)
    # arity-3 hyperedges over 60 nodes (dense: many rejected negatives)
    rng = np.random.default_rng(3)
    tri = np.array([rng.choice(60, 3, replace=False) for _ in range(200)], dtype=np.int64)
    extra = np.array([rng.choice(60, 3, replace=False) for _ in range(300)], dtype=np.int64)
    run("hyper60_a3", tri, extra, 60, P.TrainConfig(seed=6, k_neg=20, batch_size=16), epochs=2)


if __name__ == "__main__":
    main()
