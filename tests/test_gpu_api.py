"""The rest of the drop-in surface on the device: interning / dedup
(store.py:107-121,134-157), the no-dropout join+encode variant and the fused
scorer (pipeline.py:185-198,329-355), and the routing of shapes outside the
fused kernels' envelope (train / score / infer still run, as the reference
does for any shape)."""

import numpy as np
import pytest

from oracle import core

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wj():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2202_13538_b200 as m

    m._lib.load()
    return m


def _er(n, m, seed):
    import paper_2202_13538_b200 as wjm

    rng = np.random.default_rng(seed)
    return wjm.Graph.from_edges(rng.integers(0, n, size=(m, 2)), n)


def test_dedup_and_reindex_matches_reference(wj, golden_meta):
    table, dicts = wj.dedup_and_reindex([{0: [2, 0, 2], 1: [0, 2, 0]}, {1: [2, 0, 2], 0: [0, 2, 0]}])
    assert table.vectors.tolist() == golden_meta["dedup_path_table"]
    assert [{str(k): v for k, v in d.items()} for d in dicts] == golden_meta["dedup_path_dicts"]
    with pytest.raises(ValueError):
        wj.dedup_and_reindex([])


@pytest.mark.parametrize("kind", ["counts", "zeros", "negative", "wide"])
def test_intern_vectors_matches_oracle(wj, kind):
    rng = np.random.default_rng(7)
    if kind == "counts":      # store-like count vectors: the interning kernels
        v = rng.integers(0, 4, size=(5000, 5))
    elif kind == "zeros":     # all-zero rows get their own id, like the reference
        v = rng.integers(0, 2, size=(3000, 3))
        v[::7] = 0
    elif kind == "negative":  # not packable: device unique path
        v = rng.integers(-3, 3, size=(4000, 4))
    else:                     # 6 x 16-bit fields do not fit 63 bits
        v = rng.integers(0, 60000, size=(2000, 6)) * (rng.random((2000, 6)) < 0.01)
    v = v.astype(np.int32)
    ids, table = wj.intern_vectors(v)
    ids_r, table_r = core.intern_vectors(v)
    np.testing.assert_array_equal(ids, ids_r)
    np.testing.assert_array_equal(table, table_r)
    # random raw maps, node lists in first-appearance order
    maps = []
    for _ in range(40):
        xs = rng.permutation(200)[: rng.integers(1, 30)]
        maps.append({int(x): rng.integers(0, 3, size=4).tolist() for x in xs})
    t, d = wj.dedup_and_reindex(maps)
    t_r, d_r = core.dedup_and_reindex(maps)
    np.testing.assert_array_equal(t.vectors, t_r)
    assert d == d_r


@pytest.mark.parametrize("arity,L,M", [(2, 4, 40), (3, 3, 30), (2, 2, 200)])
def test_no_dropout_variant_equals_every_row_kept(wj, arity, L, M):
    """keep = 1 runs the distinct-landing variant (G = 2 n_l, no random
    stream); keep just below 1 runs the virtual-landing kernel with every
    threshold at 1: pooled, S and msum must agree bit for bit."""
    g = _er(900, 7_000, 5)
    s = wj.preprocess(g, M, L, 11)
    rng = np.random.default_rng(4)
    B = 77
    q = torch.from_numpy(np.stack([rng.choice(900, arity, replace=False) for _ in range(B)])).cuda()
    p = wj.init_params(arity, L, seed=3)
    outs = []
    for keep in (1.0, float(np.nextafter(np.float32(1.0), np.float32(0.0)))):
        pooled = torch.empty((B, 64), device="cuda")
        S = torch.empty((B, arity * (L + 1), 64), device="cuda")
        msum = torch.empty((B, 64), device="cuda")
        step = torch.zeros(1, dtype=torch.int64, device="cuda")
        wj.encoder.join_encode(s, q, p.w1, p.b1, keep, 5, step, pooled, S, msum)
        outs.append((pooled, S, msum))
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)


def test_fused_scorer_matches_pytorch_tail(wj):
    g = _er(2_000, 16_000, 8)
    s = wj.preprocess(g, 50, 3, 2)
    rng = np.random.default_rng(5)
    q = np.stack([rng.choice(2000, 2, replace=False) for _ in range(3000)]).astype(np.int64)
    p = wj.init_params(2, 3, seed=6)
    fast = wj.score_array(s, p, q, chunk=1024)
    logits, _ = wj.encoder.forward_fused(p, s, torch.from_numpy(q).cuda(), training=False, need_grad=False)
    torch.testing.assert_close(fast, torch.sigmoid(logits.double()), rtol=1e-5, atol=1e-6)
    # infer() == score_array on the host, and the reference's input checks
    np.testing.assert_allclose(wj.infer(s, p, [wj.Query(tuple(r)) for r in q[:50]]), fast[:50].cpu().numpy())
    with pytest.raises(ValueError):
        wj.infer(s, p, [(0, 2000)])
    with pytest.raises(ValueError):
        wj.infer(s, p, [(0, 1, 2)])
    # features are ignored for an RPE-only model (reference pipeline.py:351-352)
    np.testing.assert_allclose(wj.infer(s, p, q[:5], features=np.ones((3, 7))), fast[:5].cpu().numpy())


def test_shapes_outside_the_fused_envelope_still_train_and_score(wj):
    """hidden 48 (no fused kernel), arity 4 (no tensor-core kernel: the chain
    executor falls back to the graph step): train / score / infer run."""
    g = _er(600, 5_000, 9)
    s = wj.preprocess(g, 20, 2, 4)
    rng = np.random.default_rng(2)
    p48 = wj.init_params(2, 2, hidden=48, seed=1)
    assert not wj.encoder.fused_supported(p48, s)
    q = np.stack([rng.choice(600, 2, replace=False) for _ in range(40)]).astype(np.int64)
    sc = wj.score_array(s, p48, q)
    dense = wj.dense_batch(s, torch.from_numpy(q).cuda(), dtype=torch.float32)
    lg, _ = wj.forward(p48, dense, training=False)
    torch.testing.assert_close(sc, torch.sigmoid(lg.double()))
    st = wj.AdamState.for_params(p48)
    step = wj.TrainStep(s, p48, st, launch="chain")
    assert step.mode == "pooled" and step.launch == "graph"
    y = torch.from_numpy((np.arange(40) < 5).astype(np.float32)).cuda()
    assert np.isfinite(float(step(torch.from_numpy(q).cuda(), y)))
    # arity 4 through train()
    pos = np.stack([rng.choice(600, 4, replace=False) for _ in range(200)]).astype(np.int64)
    val = np.stack([rng.choice(600, 4, replace=False) for _ in range(20)]).astype(np.int64)
    neg = [np.stack([rng.choice(600, 4, replace=False) for _ in range(3)]).astype(np.int64) for _ in range(20)]
    split = wj.QuerySplit(train_pos=pos, valid_pos=val, test_pos=val, valid_neg=neg, test_neg=neg)
    cfg = wj.TrainConfig(k_neg=3, max_epochs=1, seed=0, batch_size=16, hidden_dim=64)
    params, hist = wj.train(s, split, cfg)
    assert len(hist) == 1 and np.isfinite(hist[0]["train_loss"])
    assert np.isfinite(wj.infer(s, params, val)).all()


def test_eager_adam_bias_corrections_from_device_counter(wj):
    """Non-fused steps (PyTorch tail): Adam's bias corrections come from the
    device step counter; eager and graph steps equal the host-scheduled
    reference update (encoder.adam_step) step after step."""
    g = _er(800, 6_000, 3)
    s = wj.preprocess(g, 20, 2, 1)
    rng = np.random.default_rng(0)
    q = torch.from_numpy(np.stack([rng.choice(800, 2, replace=False) for _ in range(64)])).cuda()
    y = torch.from_numpy((np.arange(64) < 9).astype(np.float32)).cuda()
    res = []
    for use_graph in (False, True, None):
        p = wj.init_params(2, 2, dropout=0.0, seed=4)
        st = wj.AdamState.for_params(p)
        if use_graph is None:  # the reference schedule on the host
            for _ in range(6):
                dense = wj.dense_batch(s, q, dtype=torch.float32)
                lg, cache = wj.forward(p, dense, training=False)
                wj.adam_step(p, wj.backward(p, cache, y), st)
        else:
            step = wj.TrainStep(s, p, st, mode="pooled", use_graph=use_graph)
            for _ in range(6):
                step(q, y)
        torch.cuda.synchronize()
        res.append({k: v.clone() for k, v in p.tensors.items()})
    for k in res[0]:
        torch.testing.assert_close(res[0][k], res[2][k], rtol=1e-5, atol=1e-6)
        torch.testing.assert_close(res[1][k], res[2][k], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("nbytes", [3, 17 << 20, (40 << 20) + 12, (130 << 20) + 4])
def test_upload_is_an_exact_copy(wj, nbytes):
    """wj_upload (multi-threaded pinned staging of the host CSR) == the host
    bytes, for sizes below, at and across its chunking."""
    from paper_2202_13538_b200.graph import upload

    rng = np.random.default_rng(nbytes)
    host = rng.integers(0, 256, size=nbytes, dtype=np.uint8)
    dev = upload(host, "cuda:0")
    assert dev.device.type == "cuda" and dev.dtype == torch.uint8
    assert np.array_equal(dev.cpu().numpy(), host)
    # through the C-ABI directly, into an int32 view with an odd element count
    h32 = rng.integers(-2**31, 2**31 - 1, size=(nbytes // 4) or 1, dtype=np.int32)
    d32 = torch.empty(h32.shape, dtype=torch.int32, device="cuda:0")
    torch.cuda.synchronize()
    wj._lib.call("wj_upload", d32.data_ptr(), h32.ctypes.data, h32.nbytes, 5)
    assert np.array_equal(d32.cpu().numpy(), h32)
