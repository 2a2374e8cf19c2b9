"""wj_score_shared (scoring of queries in runs of equal first anchors: a
positive and its negatives) against the keep = 1 join+encode kernel: pooled,
S and msum bit for bit -- including queries whose second anchor's walks reach
many of the first anchor's landings (several co-reached rounds) and runs that
change anchor inside a CTA's range."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wj():
    import paper_2202_13538_b200 as m

    m._lib.load()
    return m


def _batch(rng, n, anchors, per, neighbours=None):
    rows = []
    for u in anchors:
        if neighbours is not None and len(neighbours[u]):
            rows.append((u, int(rng.choice(neighbours[u]))))
        vs = rng.integers(0, n, per)
        vs[vs == u] = (u + 1) % n
        rows += [(u, int(v)) for v in vs]
    return torch.from_numpy(np.asarray(rows, dtype=np.int64)).cuda()


@pytest.mark.parametrize("n,m,M,L", [(3000, 30000, 40, 4), (200, 9000, 100, 3), (400, 4000, 60, 2)])
def test_score_shared_equals_join_encode(wj, n, m, M, L):
    rng = np.random.default_rng(n)
    g = wj.Graph.from_edges(rng.integers(0, n, size=(m, 2)), n)
    s = wj.preprocess(g, M, L, 5)
    nb = [g.indices[g.idxptr[u]:g.idxptr[u + 1]] for u in range(n)]
    q = _batch(rng, n, rng.choice(n, 9, replace=False), 230, nb)
    p = wj.init_params(2, L, dropout=0.0, seed=3)
    B, AW = q.shape[0], 2 * (L + 1)
    outs = []
    for shared in (False, True):
        pooled = torch.empty((B, 64), device="cuda")
        S = torch.empty((B, AW, 64), device="cuda")
        ms = torch.empty((B, 64), device="cuda")
        if shared:
            wj.encoder.score_shared(s, q, p.w1, p.b1, pooled, S, ms)
        else:
            wj.encoder.join_encode(s, q, p.w1, p.b1, 1.0, 0, None, pooled, S, ms)
        outs.append((pooled, S, ms))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_score_array_uses_shared_path_bit_exact(wj, monkeypatch):
    rng = np.random.default_rng(7)
    n = 2000
    g = wj.Graph.from_edges(rng.integers(0, n, size=(20000, 2)), n)
    s = wj.preprocess(g, 50, 4, 9)
    q = _batch(rng, n, rng.choice(n, 4, replace=False), 1000).cpu().numpy()
    p = wj.init_params(2, 4, dropout=0.1, seed=5)
    monkeypatch.setenv("WJ_SCORE_SHARED", "0")
    a = wj.score_array(s, p, q)
    monkeypatch.setenv("WJ_SCORE_SHARED", "1")
    b = wj.score_array(s, p, q)
    monkeypatch.delenv("WJ_SCORE_SHARED")
    c = wj.score_array(s, p, q)  # auto: 4 runs in 4,004 queries -> shared
    assert torch.equal(a, b) and torch.equal(a, c)


def test_score_array_host_input_decides_on_host(wj):
    """Host (pinned or not) query arrays: the id range check and the shared-
    path choice are made on the host before the copy; same scores as the
    device-resident input, the same ValueError for out-of-range ids."""
    rng = np.random.default_rng(11)
    n = 1500
    g = wj.Graph.from_edges(rng.integers(0, n, size=(15000, 2)), n)
    s = wj.preprocess(g, 40, 3, 2)
    q = _batch(rng, n, rng.choice(n, 3, replace=False), 700)
    p = wj.init_params(2, 3, dropout=0.1, seed=1)
    scorer = wj.encoder.FusedScorer(p, s)
    runs = 1 + int((q[1:, 0] != q[:-1, 0]).sum())
    assert scorer._use_shared(q) == scorer.use_shared_runs(q.shape[0], runs)
    dev = wj.score_array(s, p, q)
    host = wj.score_array(s, p, q.cpu())
    pinned = wj.score_array(s, p, q.cpu().pin_memory())
    mixed = wj.score_array(s, p, q.cpu()[torch.randperm(q.shape[0])])  # short runs: the keep = 1 kernel
    torch.cuda.synchronize()
    assert torch.equal(dev, host) and torch.equal(dev, pinned)
    assert mixed.shape == dev.shape
    for bad in (-1, n):
        qb = q.cpu().clone()
        qb[5, 1] = bad
        with pytest.raises(ValueError):
            wj.score_array(s, p, qb)
        with pytest.raises(ValueError):
            wj.score_array(s, p, qb.cuda())
