"""Generate the golden fixtures by running the REAL reference (build container only).

    python tests/golden/make_golden.py

Imports /root/reference/pkg/src/walkjoin (numba) with the SURVEY Appendix A
shim (sample_all_walks re-jitted with an int64 prange index, because the
reference kernel fails to type under numba 0.65 at _kernels.py:57-74) and
writes small .npz fixtures next to this file.  The fixtures travel to the GPU
box; /root/reference does not.  Nothing else in the repo imports the
reference.
"""

from __future__ import annotations

import json
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import walkjoin as wj  # noqa: E402  (must precede numba, walkjoin/__init__.py:14)
import numpy as np  # noqa: E402
from numba import njit, prange  # noqa: E402
from walkjoin import _kernels as K  # noqa: E402
from walkjoin import encoder as E  # noqa: E402
from walkjoin import pipeline as P  # noqa: E402


@njit(parallel=True)
def _sample_all_walks(idxptr, indices, num_walks, num_steps, seed, walks):  # K:69-74, int64 index
    n = idxptr.shape[0] - 1
    for u in prange(n):
        uu = np.int64(u)
        K.sample_node_walks(idxptr, indices, uu, num_walks, num_steps, K.node_stream_state(seed, uu), walks[u])


K.sample_all_walks = _sample_all_walks

HERE = os.path.dirname(os.path.abspath(__file__))


def graph_from_csr(n, idxptr, indices):
    return wj.Graph(n, np.asarray(idxptr, np.int64), np.asarray(indices, np.int32))


def random_queries(rng, n, B, A):
    out = np.empty((B, A), np.int64)
    for b in range(B):
        out[b] = rng.choice(n, size=A, replace=False)
    return out


def store_case(name, g, M, L, seed, queries=None, encoder=True, threads=4):
    store = wj.preprocess(g, M, L, seed, threads=threads)
    d = dict(
        n=np.int64(g.num_nodes), M=np.int64(M), L=np.int64(L), seed=np.uint64(int(seed) & (2**64 - 1)),
        idxptr=g.idxptr, indices=g.indices, walks=store.walks, table=store.table.vectors,
        dict_offsets=store.dict_offsets, dict_keys=store.dict_keys, dict_vals=store.dict_vals,
    )
    if queries is not None:
        wn, ri = wj.joiner.join_batch_arrays(store, queries, threads=threads)
        dense = P._dense_batch(store, queries, threads, None)
        d.update(queries=queries, walk_nodes=wn, rpe_ids=ri, dense=dense)
        if encoder:
            A = queries.shape[1]
            params = E.init_params(A, L, hidden=64, dropout=0.0, seed=123)
            logits, cache = E.forward(params, dense, training=False)
            labels = (np.arange(queries.shape[0]) % 2 == 0).astype(np.float64)
            loss = E.bce_loss(logits, labels)
            grads = E.backward(params, cache, labels)
            state = E.AdamState.for_params(params, lr=1e-3)
            p2 = params.copy()
            E.adam_step(p2, grads, state)
            d.update(labels=labels, logits=logits, loss=np.float64(loss))
            for k, v in params.tensors().items():
                d["p_" + k] = v
            for k, v in grads.items():
                d["g_" + k] = v
            for k, v in p2.tensors().items():
                d["p2_" + k] = v
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    return store


def main():
    meta = {}
    # --- SPEC examples -------------------------------
    path = wj.load_edge_list(["0 1"])
    store_case("path", path, 2, 2, 5, queries=np.array([[0, 1], [1, 0]], np.int64), encoder=False)
    iso = wj.Graph.from_edges(np.empty((0, 2), np.int64), 1)
    store_case("isolated", iso, 1, 1, 9)
    tri = wj.load_edge_list(["0 1", "1 2", "0 2"])
    store_case("triangle", tri, 4, 3, 42, queries=np.array([[0, 1], [2, 0]], np.int64), encoder=False)
    rng_tri = wj.WalkRng.for_node(42, 0)
    meta["triangle_state_42_0"] = int(rng_tri.state)
    ws = wj.sample_walks(tri, 0, 4, 3, rng_tri)
    meta["triangle_walks_u0"] = ws.walks.tolist()
    meta["triangle_end_state"] = int(rng_tri.state)
    raw = wj.compute_rpe(ws)
    meta["triangle_rpe_u0"] = {str(k): v.tolist() for k, v in raw.entries.items()}
    table, dicts = wj.dedup_and_reindex([{0: np.array([2, 0, 2]), 1: np.array([0, 2, 0])},
                                         {1: np.array([2, 0, 2]), 0: np.array([0, 2, 0])}])
    meta["dedup_path_table"] = table.vectors.tolist()
    meta["dedup_path_dicts"] = [{str(k): v for k, v in dd.items()} for dd in dicts]

    # --- random graphs ------------------------------------------------------------------
    rng = np.random.default_rng(2024)
    g = wj.generate_sbm(1, 300, 0.03, 0.0, seed=1)
    store_case("er300", g, 20, 3, 7, queries=random_queries(rng, g.num_nodes, 6, 2))
    g = wj.generate_sbm(1, 400, 0.004, 0.0, seed=2)  # sparse: isolated nodes + dead ends
    store_case("sparse400", g, 16, 4, 11, queries=random_queries(rng, g.num_nodes, 5, 2))
    g = wj.generate_sbm(2, 100, 0.1, 0.005, seed=1)  # SPEC.md:176 determinism case
    store_case("sbm2x100", g, 10, 3, 3, queries=random_queries(rng, g.num_nodes, 4, 2))
    g = wj.generate_sbm(1, 1000, 0.02, 0.0, seed=5)  # C1-like degree, M=50 L=3
    store_case("er1000_m50", g, 50, 3, 3, queries=random_queries(rng, g.num_nodes, 3, 2))
    # hyperedges -> arity-3 joins (tags-math shape, A=3)
    hl = []
    for _ in range(120):
        hl.append(" ".join(str(v) for v in rng.choice(60, size=3, replace=False)))
    g = wj.project_hyperedges(hl)
    store_case("hyper60_a3", g, 12, 2, 13, queries=random_queries(rng, g.num_nodes, 4, 3))
    # directed CSR built directly (not symmetric): mid-walk dead ends consume no draw
    # node 3 has out-degree 0 but is reachable from 0 and 2
    idxptr = np.array([0, 2, 3, 5, 5, 6], np.int64)
    indices = np.array([1, 3, 2, 0, 3, 4], np.int32)
    store_case("directed5", graph_from_csr(5, idxptr, indices), 6, 3, 21,
               queries=np.array([[0, 2], [1, 4]], np.int64), encoder=False)
    # large-M (uint16 counts path): M=300 > 255
    g = wj.generate_sbm(1, 150, 0.04, 0.0, seed=8)
    store_case("er150_m300", g, 300, 2, 17, queries=random_queries(rng, g.num_nodes, 2, 2))

    # --- BFS mini-batcher + negatives (pipeline.py:77-166) -------------------------------
    g = wj.generate_sbm(1, 500, 0.02, 0.0, seed=4)
    split = wj.split_link_queries(g, 0.3, 5, seed=1)
    cfg = P.TrainConfig(batch_capacity=60, batch_size=8, k_neg=5)
    index = P.QueryOverlapIndex(split.train_pos)
    pos_filter = {P.canonical_nodes(q.nodes) for q in split.train_pos}
    for grp in (split.valid_pos, split.test_pos):
        pos_filter.update(P.canonical_nodes(q.nodes) for q in grp)
    brng = np.random.default_rng(77)
    batches = []
    for _ in range(3):
        seeds, ids = P.sample_minibatch(index, split.train_pos, cfg, brng)
        negs = P.sample_negatives(seeds, 2, cfg.k_neg * len(ids), pos_filter, brng)
        batches.append({"seeds": [int(s) for s in seeds], "ids": [int(i) for i in ids],
                        "negs": [list(q.nodes) for q in negs]})
    meta["minibatch"] = {
        "train_pos": [list(q.nodes) for q in split.train_pos],
        "pos_filter_extra": [list(q.nodes) for grp in (split.valid_pos, split.test_pos) for q in grp],
        "batch_capacity": 60, "batch_size": 8, "k_neg": 5, "rng_seed": 77, "batches": batches,
    }
    meta["derive_seed"] = {f"{s}:{lab}": int(wj._seeds.derive_seed(s, lab))
                           for s in (0, 1, 42) for lab in ("preprocess", "train", "init", "sbm")}
    with open(os.path.join(HERE, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("fixtures written to", HERE)


if __name__ == "__main__":
    main()
