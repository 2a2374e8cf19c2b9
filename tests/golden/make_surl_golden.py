"""Generate SURL store-file fixtures by running the REAL reference save_store
(build container only; /root/reference does not travel to the GPU box).

    python tests/golden/make_surl_golden.py

Writes, next to this file, ``surl_<case>.surl`` (the exact bytes
walkjoin.store.save_store produces, store.py:167-201) and
``surl_<case>.npz`` (the graph it was built from and the preprocess
arguments).  Uses the same numba shim as make_golden.py.
"""

from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

import make_golden as MG  # noqa: E402  (imports the reference with the shim)

wj = MG.wj


def case(name, g, M, L, seed):
    store = wj.preprocess(g, M, L, seed, threads=4)
    path = os.path.join(HERE, f"surl_{name}.surl")
    wj.save_store(store, path)
    id_keys = np.array(sorted(g.id_map), np.int64) if g.id_map else np.empty(0, np.int64)
    id_vals = np.array([g.id_map[k] for k in id_keys], np.int64) if g.id_map else np.empty(0, np.int64)
    np.savez_compressed(os.path.join(HERE, f"surl_{name}.npz"), n=np.int64(g.num_nodes), idxptr=g.idxptr,
                        indices=g.indices, M=np.int64(M), L=np.int64(L),
                        seed=np.uint64(int(seed) & (2**64 - 1)), id_keys=id_keys, id_vals=id_vals)
    print(name, os.path.getsize(path), "bytes")


def main():
    rng = np.random.default_rng(21)
    n = 200
    pairs = rng.integers(0, n, size=(900, 2))
    case("er200", wj.Graph.from_edges(pairs, n), 12, 3, 5)
    # sparse original ids -> a graph with an id_map (written after the records)
    orig = rng.choice(10_000_000, size=120, replace=False).astype(np.int64)
    e = rng.integers(0, 120, size=(400, 2))
    id_map = {}
    dense = []
    for u, v in e:
        for x in (orig[u], orig[v]):
            if int(x) not in id_map:
                id_map[int(x)] = len(id_map)
        dense.append((id_map[int(orig[u])], id_map[int(orig[v])]))
    g2 = wj.Graph.from_edges(np.array(dense, np.int64), len(id_map), id_map=id_map)
    case("idmap120", g2, 8, 2, 9)


if __name__ == "__main__":
    main()
