"""Typed / metapath walks.

The reference has no typed sampler (SPEC.md:121-124 leaves typed walks
open), so the typed semantics are ours (include/walkjoin_b200.h,
wj_sample_walks_typed) and their parity is against the oracle restatement
only ("parity unpinned").  The homogeneous special case IS pinned: with
metapath [-1], or one edge type on every edge, the walks must equal the
reference's own walks (tests/golden fixtures written by the reference) on
every symmetric-CSR fixture.
"""

import numpy as np
import pytest

from conftest import golden_cases, load_golden
from oracle import core


def _symmetric(idxptr, indices):
    n = idxptr.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(idxptr))
    a = np.sort(rows * n + indices)
    b = np.sort(indices.astype(np.int64) * n + rows)
    return np.array_equal(a, b)


SYM_CASES = [c for c in golden_cases() if _symmetric(load_golden(c)["idxptr"], load_golden(c)["indices"])]


def _typed_graph(n=400, m=3000, T=3, seed=0, isolated=10):
    """Random symmetric graph with per-edge types (same type both directions)."""
    rng = np.random.default_rng(seed)
    a = rng.integers(isolated, n, size=m)
    b = rng.integers(isolated, n, size=m)
    keep = a != b
    a, b = a[keep], b[keep]
    t = rng.integers(0, T, size=a.shape[0])
    src = np.concatenate([a, b])
    dst = np.concatenate([b, a])
    ty = np.concatenate([t, t])
    order = np.lexsort((dst, src))
    src, dst, ty = src[order], dst[order], ty[order]
    idxptr = np.zeros(n + 1, np.int64)
    np.add.at(idxptr, src + 1, 1)
    idxptr = np.cumsum(idxptr)
    return idxptr, dst.astype(np.int32), ty.astype(np.uint8)


@pytest.mark.parametrize("name", SYM_CASES)
def test_oracle_homogeneous_case_is_reference(name):
    g = load_golden(name)
    M, L, seed = int(g["M"]), int(g["L"]), int(g["seed"])
    et = np.zeros(g["indices"].shape[0], np.uint8)
    for mp in ([-1], [0], [0, -1]):
        w = core.sample_typed_walks(g["idxptr"], g["indices"], et, mp, M, L, seed, threads=2)
        np.testing.assert_array_equal(w, g["walks"])


def test_oracle_typed_walks_follow_the_metapath():
    idxptr, indices, et = _typed_graph()
    n = idxptr.shape[0] - 1
    mp = [0, 2, -1, 1]
    w = core.sample_typed_walks(idxptr, indices, et, mp, 12, 6, 7, threads=2)
    edge_type = {}
    for u in range(n):
        for e in range(idxptr[u], idxptr[u + 1]):
            edge_type.setdefault((u, int(indices[e])), set()).add(int(et[e]))
    for u in range(n):
        for j in range(12):
            for i in range(1, 7):
                a, b = int(w[u, j, i - 1]), int(w[u, j, i])
                t = mp[(i - 1) % len(mp)]
                has = any(t < 0 or et[e] == t for e in range(idxptr[a], idxptr[a + 1]))
                if not has:
                    assert a == b  # no edge of the required type: stay
                else:
                    assert (a, b) in edge_type and (t < 0 or t in edge_type[(a, b)])
    assert np.all(w[:10] == np.arange(10)[:, None, None])  # isolated anchors repeat


@pytest.mark.gpu
@pytest.mark.parametrize("mp", [[-1], [0], [1, 2], [0, 2, -1, 1], [2] * 5])
@pytest.mark.parametrize("seed", [1, 99])
def test_device_typed_walks_match_oracle(mp, seed):
    import torch

    import paper_2202_13538_b200 as wj

    idxptr, indices, et = _typed_graph(seed=seed)
    g = wj.Graph(idxptr.shape[0] - 1, idxptr, indices)
    tc = wj.typed_csr(g, et, 3)
    w = wj.sample_walks_typed(g, tc, mp, 16, 5, seed).cpu().numpy()
    ref = core.sample_typed_walks(idxptr, indices, et, mp, 16, 5, seed, threads=4)
    np.testing.assert_array_equal(w, ref)
    # shard: anchors [lo, hi) only
    w2 = wj.sample_walks_typed(g, tc, mp, 16, 5, seed, lo=37, hi=211).cpu().numpy()
    np.testing.assert_array_equal(w2, ref[37:211])
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_typed_csr_groups_stably():
    import paper_2202_13538_b200 as wj

    idxptr, indices, et = _typed_graph(n=200, m=1500, T=4, seed=3)
    g = wj.Graph(idxptr.shape[0] - 1, idxptr, indices)
    tc = wj.typed_csr(g, et, 4)
    off = tc.type_off.cpu().numpy()
    ti = tc.typed_indices.cpu().numpy()
    n = idxptr.shape[0] - 1
    assert off[-1] == indices.shape[0]
    for u in range(n):
        for t in range(4):
            seg = ti[off[u * 4 + t]: off[u * 4 + t + 1]]
            want = [indices[e] for e in range(idxptr[u], idxptr[u + 1]) if et[e] == t]
            assert list(seg) == want


@pytest.mark.gpu
@pytest.mark.parametrize("name", SYM_CASES)
def test_device_homogeneous_case_is_reference(name):
    import paper_2202_13538_b200 as wj

    g = load_golden(name)
    M, L, seed = int(g["M"]), int(g["L"]), int(g["seed"])
    gr = wj.Graph(int(g["n"]), g["idxptr"], g["indices"])
    et = np.zeros(g["indices"].shape[0], np.uint8)
    for mp in ([-1], [0]):
        s = wj.preprocess_typed(gr, et, mp, M, L, seed, num_types=1)
        np.testing.assert_array_equal(s.walks, g["walks"])
        np.testing.assert_array_equal(s.table.vectors, g["table"])
        np.testing.assert_array_equal(s.dict_keys, g["dict_keys"])
        np.testing.assert_array_equal(s.dict_vals, g["dict_vals"])


@pytest.mark.gpu
def test_preprocess_typed_store_matches_oracle_store():
    """The typed store (RPE, interning, dicts, join) equals the oracle's
    reference-algorithm store built from the oracle's typed walks."""
    import paper_2202_13538_b200 as wj

    idxptr, indices, et = _typed_graph(n=500, m=5000, T=3, seed=5)
    g = wj.Graph(idxptr.shape[0] - 1, idxptr, indices)
    mp = [0, 1, 2]
    s = wj.preprocess_typed(g, et, mp, 24, 4, 11, num_types=3)
    walks = core.sample_typed_walks(idxptr, indices, et, mp, 24, 4, 11, threads=4)
    ref = core.store_from_walks(walks, seed=11, threads=4)
    np.testing.assert_array_equal(s.walks, walks)
    np.testing.assert_array_equal(s.table.vectors, ref.table)
    np.testing.assert_array_equal(s.dict_keys, ref.dict_keys)
    np.testing.assert_array_equal(s.dict_vals, ref.dict_vals)
    rng = np.random.default_rng(0)
    q = np.stack([rng.choice(500, 2, replace=False) for _ in range(32)]).astype(np.int64)
    wn, ri = wj.join_batch_arrays(s, q)
    wn_r, ri_r = core.join_batch_arrays(ref, q)
    np.testing.assert_array_equal(wn, wn_r)
    np.testing.assert_array_equal(ri, ri_r)


def test_edge_types_from_node_types():
    from paper_2202_13538_b200.sampler import edge_types_from_node_types

    class G:
        num_nodes = 4
        idxptr = np.array([0, 2, 3, 4, 5])
        indices = np.array([1, 2, 0, 0, 0])

    et = edge_types_from_node_types(G, [0, 1, 1, 0], 2)
    assert et.tolist() == [0 * 2 + 1, 0 * 2 + 1, 1 * 2 + 0, 1 * 2 + 0, 0 * 2 + 0]
    with pytest.raises(ValueError):
        edge_types_from_node_types(G, [0, 1, 2, 0], 2)
