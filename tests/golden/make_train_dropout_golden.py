"""Training-quality fixtures WITH dropout, from the REAL reference (build container only).

    python tests/golden/make_train_dropout_golden.py [seed ...]

BASELINE.json configs[0] (C1): the reference's own ER generator
(``generate_sbm(1, 10000, p, 0, seed=1)``, graph.py:298-354) with 100K
expected edges, the 5 % link split (``split_link_queries(g, 0.05, 10,
seed=1)``, graph.py:239-280), store ``preprocess(M=50, L=3, seed=3)``, then
ONE epoch of the reference ``train`` (pipeline.py:241-326) with the default
``dropout=0.1`` for each training seed.  Dropout masks come from numpy PCG64
(encoder.py:154-158), which the device kernel does not reproduce (its
dropout is equal in distribution, not in stream), so the device test
compares the MEAN over the seeds of the final metrics (north_star: "final
MRR/AUC must agree within 0.5 points").

Validation and test use the first 2,000 / 4,000 positives of the split (each
with its 10 negatives) so the float64 reference scores them in minutes; the
subset is part of the fixture.  Uses the SURVEY Appendix A shim (numba 0.65
TypingError in sample_all_walks).  Output: tests/golden/train_dropout/c1.npz
(split + graph, written once) and c1_seed<k>.npz per seed.
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
OUT = os.path.join(HERE, "train_dropout")
N, E, M, L, K_SPLIT, N_VALID, N_TEST = 10_000, 100_000, 50, 3, 10, 2_000, 4_000
THREADS = int(os.environ.get("WJ_THREADS", "6"))


def qarr(qs):
    return np.asarray([q.nodes for q in qs], dtype=np.int64)


def make_split():
    g = G.generate_sbm(1, N, E / (N * (N - 1) / 2), 0.0, seed=1)
    full = G.split_link_queries(g, train_frac=0.05, k_neg=K_SPLIT, seed=1)
    split = G.QuerySplit(train_pos=full.train_pos, valid_pos=full.valid_pos[:N_VALID],
                         test_pos=full.test_pos[:N_TEST], valid_neg=full.valid_neg[:N_VALID],
                         test_neg=full.test_neg[:N_TEST], train_graph=full.train_graph)
    return g, split


def main(seeds):
    os.makedirs(OUT, exist_ok=True)
    t = time.time()
    g, split = make_split()
    tg = split.train_graph
    np.savez_compressed(os.path.join(OUT, "c1.npz"), n=np.int64(g.num_nodes), M=np.int64(M), L=np.int64(L),
                        idxptr=tg.idxptr, indices=tg.indices, train_pos=qarr(split.train_pos),
                        valid_pos=qarr(split.valid_pos), test_pos=qarr(split.test_pos),
                        valid_neg=np.stack([qarr(gp) for gp in split.valid_neg]),
                        test_neg=np.stack([qarr(gp) for gp in split.test_neg]))
    print("split", len(split.train_pos), "train pos; %.1fs" % (time.time() - t), flush=True)
    store = wj.preprocess(tg, M, L, seed=3, threads=THREADS)
    for seed in seeds:
        t = time.time()
        cfg = P.TrainConfig(k_neg=50, max_epochs=1, seed=seed, threads=THREADS, metric="auc", patience=1,
                            dropout=0.1)
        params, hist = P.train(store, split, cfg)
        pos = P.infer(store, params, split.test_pos, threads=THREADS)
        neg = P.infer(store, params, [q for grp in split.test_neg for q in grp], threads=THREADS)
        res = [MX.RankedQueryResult(float(pos[i]), neg[i * K_SPLIT:(i + 1) * K_SPLIT]) for i in range(len(pos))]
        d = dict(seed=np.int64(seed), train_loss=np.float64(hist[0]["train_loss"]),
                 valid_auc=np.float64(hist[0]["valid_metric"]), test_auc=np.float64(MX.roc_auc(pos, neg)),
                 test_mrr=np.float64(MX.mrr(res)), test_hits10=np.float64(MX.hits_at_k(res, 10)),
                 test_pos_scores=pos, test_neg_scores=neg)
        np.savez_compressed(os.path.join(OUT, f"c1_seed{seed}.npz"), **d)
        print("seed", seed, "loss %.5f valid_auc %.4f test auc %.4f mrr %.4f hits10 %.4f  %.0fs" % (
            d["train_loss"], d["valid_auc"], d["test_auc"], d["test_mrr"], d["test_hits10"], time.time() - t),
            flush=True)


if __name__ == "__main__":
    main([int(s) for s in sys.argv[1:]] or [0, 1, 2, 3, 4])
