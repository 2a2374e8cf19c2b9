"""Golden training trajectories from the REAL reference (build container only).

    python tests/golden/make_train_golden.py

Runs the reference ``pipeline.train`` (pipeline.py:241-326) end to end on
small SBM link-prediction splits made by the reference's own generators
(graph.py:239-354) and records, per case: the split, the per-epoch history
(train loss, validation AUC / MRR), the best parameters and the test scores
(``infer``).  Dropout is off so the trajectory is a deterministic function of
the batch draws, which the device ``train(..., exact_batches=True)``
reproduces; the GPU test then checks the validation metric of every epoch and
the final test metric within 0.5 points.  Uses the SURVEY Appendix A shim
(numba 0.65 TypingError in sample_all_walks).
"""

from __future__ import annotations

import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import walkjoin as wj  # noqa: E402
import numpy as np  # noqa: E402
from numba import njit, prange  # noqa: E402
from walkjoin import _kernels as K  # noqa: E402
from walkjoin import graph as G  # noqa: E402
from walkjoin import metrics as MX  # noqa: E402
from walkjoin import pipeline as P  # noqa: E402


@njit(parallel=True)
def _sample_all_walks(idxptr, indices, num_walks, num_steps, seed, walks):  # K:69-74, int64 index
    n = idxptr.shape[0] - 1
    for u in prange(n):
        uu = np.int64(u)
        K.sample_node_walks(idxptr, indices, uu, num_walks, num_steps, K.node_stream_state(seed, uu), walks[u])


K.sample_all_walks = _sample_all_walks
HERE = os.path.dirname(os.path.abspath(__file__))


def qarr(qs):
    return np.asarray([q.nodes for q in qs], dtype=np.int64)


def case(name, blocks, npb, p_in, p_out, M, L, metric, epochs, k_neg_split, k_neg, seed, pool=0):
    g = G.generate_sbm(blocks, npb, p_in, p_out, seed=1)
    split = G.split_link_queries(g, train_frac=0.7, k_neg=k_neg_split, seed=1)
    store = wj.preprocess(split.train_graph, M, L, seed=3, threads=8)
    cfg = P.TrainConfig(k_neg=k_neg, max_epochs=epochs, seed=seed, threads=8, metric=metric, patience=epochs,
                        dropout=0.0, batch_size=32, batch_capacity=1500)
    t = time.time()
    train_negatives = None
    if pool:
        # a fixed pool of uniform non-edges of the full graph (the reference's
        # ``train_negatives`` option, pipeline.py:262,299-301)
        rng = np.random.default_rng(5)
        cand = rng.integers(0, g.num_nodes, size=(4 * pool, 2))
        keep = [(int(u), int(v)) for u, v in cand if u != v and not g.has_edge(int(u), int(v))][:pool]
        train_negatives = [G.Query(q, 0) for q in keep]
    params, hist = P.train(store, split, cfg, train_negatives=train_negatives)
    pos = P.infer(store, params, split.test_pos, threads=8)
    neg_groups = split.test_neg
    neg = P.infer(store, params, [q for grp in neg_groups for q in grp], threads=8)
    test_auc = MX.roc_auc(pos, neg)
    res = [MX.RankedQueryResult(float(pos[i]), neg[i * k_neg_split:(i + 1) * k_neg_split]) for i in range(len(pos))]
    d = dict(
        n=np.int64(g.num_nodes), M=np.int64(M), L=np.int64(L), k_neg=np.int64(k_neg), epochs=np.int64(epochs),
        seed=np.int64(seed), metric=np.array(metric),
        idxptr=split.train_graph.idxptr, indices=split.train_graph.indices,
        train_pos=qarr(split.train_pos), valid_pos=qarr(split.valid_pos), test_pos=qarr(split.test_pos),
        valid_neg=np.stack([qarr(gp) for gp in split.valid_neg]),
        test_neg=np.stack([qarr(gp) for gp in split.test_neg]),
        hist_loss=np.array([h["train_loss"] for h in hist]),
        hist_valid=np.array([h["valid_metric"] for h in hist]),
        test_pos_scores=pos, test_neg_scores=neg, test_auc=np.float64(test_auc),
        test_mrr=np.float64(MX.mrr(res)), test_hits10=np.float64(MX.hits_at_k(res, 10)),
    )
    if train_negatives is not None:
        d["train_negatives"] = qarr(train_negatives)
    for k, v in params.tensors().items():
        d["p_" + k] = v
    np.savez_compressed(os.path.join(HERE, "train", f"{name}.npz"), **d)
    print(name, "epochs", len(hist), "valid", d["hist_valid"].round(4), "test auc %.4f mrr %.4f" %
          (test_auc, d["test_mrr"]), "%.1fs" % (time.time() - t), flush=True)


def main():
    os.makedirs(os.path.join(HERE, "train"), exist_ok=True)
    case("sbm2x150_auc", 2, 150, 0.06, 0.004, M=20, L=2, metric="auc", epochs=4, k_neg_split=10, k_neg=5,
         seed=0)
    case("sbm2x150_mrr", 2, 150, 0.06, 0.004, M=20, L=3, metric="mrr", epochs=3, k_neg_split=10, k_neg=5,
         seed=1)
    case("sbm2x150_pool", 2, 150, 0.06, 0.004, M=20, L=2, metric="auc", epochs=4, k_neg_split=10, k_neg=5,
         seed=2, pool=3000)


if __name__ == "__main__":
    main()
