"""Parity of the CUDA path (through the C ABI) with the reference fixtures and
the CPU oracle.  Bit-exact for walks / RPE index / table / dicts / join /
dense; encoder logits within 1e-5 relative (north_star tolerance)."""

import os

import numpy as np
import pytest

from conftest import golden_cases, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wj():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2202_13538_b200 as m

    m._lib.load()
    return m


def _graph(wj, g):
    return wj.Graph(int(g["n"]), g["idxptr"].astype(np.int64), g["indices"].astype(np.int32))


@pytest.mark.parametrize("name", golden_cases())
def test_store_bit_exact_vs_reference(wj, name):
    g = load_golden(name)
    store = wj.preprocess(_graph(wj, g), int(g["M"]), int(g["L"]), int(g["seed"]))
    np.testing.assert_array_equal(store.walks, g["walks"])
    np.testing.assert_array_equal(store.table.vectors, g["table"])
    np.testing.assert_array_equal(store.dict_offsets, g["dict_offsets"])
    np.testing.assert_array_equal(store.dict_keys, g["dict_keys"])
    np.testing.assert_array_equal(store.dict_vals, g["dict_vals"])
    assert store.walk_slot_count == int(g["n"]) * int(g["M"]) * (int(g["L"]) + 1)


@pytest.mark.parametrize("name", [c for c in golden_cases() if "queries" in load_golden(c)])
def test_join_dense_bit_exact_vs_reference(wj, name):
    g = load_golden(name)
    store = wj.preprocess(_graph(wj, g), int(g["M"]), int(g["L"]), int(g["seed"]))
    wn, ri = wj.join_batch_arrays(store, g["queries"])
    np.testing.assert_array_equal(wn, g["walk_nodes"])
    np.testing.assert_array_equal(ri, g["rpe_ids"])
    dense = wj.dense_batch(store, g["queries"])
    assert dense.dtype == np.float64
    np.testing.assert_array_equal(dense, g["dense"])
    # device path, every dense dtype (counts are exact in all of them for M <= 256)
    qd = torch.from_numpy(g["queries"]).cuda()
    for dt in (torch.float32, torch.float64, torch.bfloat16, torch.float16):
        if dt in (torch.bfloat16,) and int(g["M"]) > 256:
            continue
        dd = wj.dense_batch(store, qd, dtype=dt)
        np.testing.assert_array_equal(dd.double().cpu().numpy(), g["dense"])
    for b in range(g["queries"].shape[0]):
        jq = wj.join_query(store, tuple(int(v) for v in g["queries"][b]))
        np.testing.assert_array_equal(wj.gather_rpe(store.table, jq), g["dense"][b])


@pytest.mark.parametrize("name", [c for c in golden_cases() if "logits" in load_golden(c)])
@pytest.mark.parametrize("mode", ["pooled", "reference"])
def test_encoder_logits_and_grads(wj, name, mode):
    g = load_golden(name)
    A, L = g["queries"].shape[1], int(g["L"])
    p = wj.encoder.params_from_numpy({k: g["p_" + k] for k in wj.encoder.TENSOR_ORDER}, A, L)
    dense = torch.from_numpy(g["dense"]).cuda()
    logits, cache = wj.forward(p, dense, training=False, mode=mode)
    ref = g["logits"]
    tol = 1e-5 * max(np.abs(ref).max(), 1e-3)
    np.testing.assert_allclose(logits.double().cpu().numpy(), ref, rtol=1e-5, atol=tol)
    labels = torch.from_numpy(g["labels"]).cuda()
    assert abs(float(wj.bce_loss(logits.double(), labels)) - float(g["loss"])) < 1e-5 * abs(float(g["loss"]))
    grads = wj.backward(p, cache, labels)
    for k in wj.encoder.TENSOR_ORDER:
        r = g["g_" + k]
        np.testing.assert_allclose(grads[k].double().cpu().numpy(), r, rtol=1e-4,
                                   atol=1e-4 * max(np.abs(r).max(), 1e-12))
    state = wj.AdamState.for_params(p)
    wj.adam_step(p, grads, state)
    for k in wj.encoder.TENSOR_ORDER:
        np.testing.assert_allclose(p.tensors[k].double().cpu().numpy(), g["p2_" + k], rtol=1e-5, atol=1e-6)


def test_spec_examples(wj, golden_meta):
    tri = wj.load_edge_list(["0 1", "1 2", "0 2"])
    rng = wj.WalkRng.for_node(42, 0)
    assert rng.state == 0xBDD732262FEB6E95
    ws = wj.sample_walks(tri, 0, 4, 3, rng)
    assert ws.walks.tolist() == golden_meta["triangle_walks_u0"]
    assert rng.state == golden_meta["triangle_end_state"]
    raw = wj.compute_rpe(ws)
    assert list(raw.entries) == [int(k) for k in golden_meta["triangle_rpe_u0"]]
    assert {str(k): v.tolist() for k, v in raw.entries.items()} == golden_meta["triangle_rpe_u0"]
    path = wj.load_edge_list(["0 1"])
    s = wj.preprocess(path, 2, 2, seed=5)
    assert wj.get_rpe_id(s, 0, 1) == 2 and wj.get_rpe_id(s, 0, 99) == 0
    with pytest.raises(ValueError):
        wj.get_rpe_id(s, 2, 0)
    assert s.entry(0).dict == {0: 1, 1: 2} and s.entry(1).dict == {0: 2, 1: 1}
    jq = wj.join_query(s, (0, 1))
    assert jq.walk_nodes.tolist() == [[0, 1, 0], [0, 1, 0], [1, 0, 1], [1, 0, 1]]
    assert wj.gather_rpe(s.table, jq)[0].tolist() == [2, 0, 2, 0, 2, 0]
    assert wj.join_batch(s, []) == []
    with pytest.raises(ValueError):
        wj.join_batch(s, [(0, 1), (0,)])
    with pytest.raises(ValueError):
        wj.join_query(s, (0, 7))
    # isolated node, M=1, m=1 -> T = [[0,0],[1,1]]
    iso = wj.Graph.from_edges(np.empty((0, 2), np.int64), 1)
    s1 = wj.preprocess(iso, 1, 1, seed=9)
    assert s1.table.vectors.tolist() == [[0, 0], [1, 1]] and s1.walks.tolist() == [[[0, 0]]]
    with pytest.raises(ValueError):
        wj.preprocess(path, 0, 2, seed=1)


def _er(n, m, seed, isolated_frac=0.0):
    rng = np.random.default_rng(seed)
    import paper_2202_13538_b200 as wjm

    hi = int(n * (1 - isolated_frac))
    pairs = rng.integers(0, hi, size=(m, 2))
    return wjm.Graph.from_edges(pairs, n)


@pytest.mark.parametrize("n,m,M,L,seed", [
    (10_000, 100_000, 50, 3, 3),     # C1 shape
    (3_000, 6_000, 200, 4, 1),       # sparse, M=200 L=4 (citation2 M/L)
    (2_000, 40_000, 100, 3, 7),      # dense, tags-math M/L
    (1_500, 3_000, 400, 2, 2),       # M=400 L=2 (paper's vessel / collab setting, uint16-class counts)
])
def test_store_and_join_vs_oracle(wj, n, m, M, L, seed):
    from oracle import core

    g = _er(n, m, seed, isolated_frac=0.05)
    s = wj.preprocess(g, M, L, seed)
    r = core.preprocess(g.idxptr, g.indices, M, L, seed)
    np.testing.assert_array_equal(s.walks, r.walks)
    np.testing.assert_array_equal(s.table.vectors, r.table)
    np.testing.assert_array_equal(s.dict_keys, r.dict_keys)
    np.testing.assert_array_equal(s.dict_vals, r.dict_vals)
    rng = np.random.default_rng(seed)
    for A in (2, 3):
        q = np.stack([rng.choice(n, A, replace=False) for _ in range(64)]).astype(np.int64)
        wn, ri = wj.join_batch_arrays(s, q)
        wr, rr = core.join_batch_arrays(r, q)
        np.testing.assert_array_equal(wn, wr)
        np.testing.assert_array_equal(ri, rr)
    qd = torch.from_numpy(q).cuda()
    dd = wj.dense_batch(s, qd, dtype=torch.float32).double().cpu().numpy()
    np.testing.assert_array_equal(dd, core.dense_batch(r, q))


def test_directed_dead_end_fixup(wj):
    """Non-symmetric CSR: a mid-walk dead end consumes no draw, so later walks
    shift; the device re-samples such anchors sequentially (bit-exact)."""
    from oracle import core

    rng = np.random.default_rng(5)
    n = 400
    deg = rng.integers(0, 4, size=n)
    idxptr = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=idxptr[1:])
    indices = np.concatenate([np.sort(rng.choice(n, d, replace=False)) for d in deg]).astype(np.int32)
    g = wj.Graph(n, idxptr, indices)
    s = wj.preprocess(g, 30, 4, 99)
    r = core.preprocess(idxptr, indices, 30, 4, 99)
    np.testing.assert_array_equal(s.walks, r.walks)
    np.testing.assert_array_equal(s.table.vectors, r.table)
    np.testing.assert_array_equal(s.dict_vals, r.dict_vals)
    for u in range(0, n, 37):
        st = core.node_stream_state(7, u) ^ 0x1234
        ws = wj.sample_walks(g, u, 9, 3, wj.WalkRng(st))
        w_r, _ = core.sample_walks(idxptr, indices, u, 9, 3, st)
        np.testing.assert_array_equal(ws.walks, w_r)


def test_properties_at_collab_scale(wj):
    """Size-independent properties at C2 scale (235K nodes, M=200, L=4)."""
    dev = torch.device("cuda")
    split = wj.graph.synthetic_link_graph(235_868, 1_285_465, 0.05, seed=1, device=dev)
    g = split.walk_graph
    s = wj.preprocess(g, 200, 4, 3)
    n, M, W = g.num_nodes, 200, 5
    walks = s.walks_d
    # column 0 is the anchor
    assert torch.equal(walks[:, :, 0], torch.arange(n, device=dev, dtype=torch.int32)[:, None].expand(n, M))
    # every step is an edge (or a repeat at an isolated anchor)
    ip = g.idxptr.long()
    deg = ip[1:] - ip[:-1]
    a = walks[:, :, :-1].reshape(-1).long()
    b = walks[:, :, 1:].reshape(-1).long()
    iso = deg[a] == 0
    assert torch.all(a[iso] == b[iso])
    ka = a[~iso][:5_000_000]
    kb = b[~iso][:5_000_000]
    key_e = ip.new_tensor(0)
    lo = ip[ka]
    hi = ip[ka + 1]
    # binary search kb in the sorted neighbour row of ka
    idx = g.indices.long()
    left, right = lo.clone(), hi.clone()
    for _ in range(32):
        mid = (left + right) // 2
        go = (left < right) & (idx[mid.clamp(max=idx.numel() - 1)] < kb)
        left = torch.where(go, mid + 1, left)
        right = torch.where(go | (left >= right), right, mid)
    assert torch.all(idx[left.clamp(max=idx.numel() - 1)] == kb)
    # RPE mass: every anchor's count vectors sum to M in every column
    tab = s.table_d.long()
    sums = torch.zeros((n, W), dtype=torch.int64, device=dev)
    owner = torch.repeat_interleave(torch.arange(n, device=dev), s.anchor_counts())
    sums.index_add_(0, owner, tab[s.uniq_id_d.long()])
    assert torch.all(sums == M)
    # the table has no duplicates and row 0 is the zero sentinel
    assert torch.all(tab[0] == 0)
    assert torch.unique(s.table_keys_d).numel() == s.table_keys_d.numel()
    # uniq lists are strictly increasing within each anchor
    ux = s.uniq_x_d.long()
    inner = torch.ones_like(ux, dtype=torch.bool)
    inner[s.offsets_d[:-1][s.anchor_counts() > 0]] = False
    assert torch.all((ux[1:] > ux[:-1])[inner[1:]])


def test_chi_square_transitions(wj):
    """Each step is uniform over the current node's neighbours."""
    from scipy.stats import chisquare

    g = _er(2_000, 8_000, 11)
    s = wj.preprocess(g, 200, 4, 17)
    w = s.walks
    for c in (5, 17, 123):
        deg = g.degree(c)
        if deg < 3:
            continue
        prev, nxt = w[:, :, :-1].reshape(-1), w[:, :, 1:].reshape(-1)
        sel = nxt[prev == c]
        counts = np.array([(sel == v).sum() for v in g.neighbors(c)])
        assert counts.sum() == sel.size
        assert chisquare(counts).pvalue > 1e-4


def test_train_step_graph_matches_eager(wj):
    """The captured training step equals the eager step (same RNG stream)."""
    g = _er(3_000, 30_000, 2)
    s = wj.preprocess(g, 50, 3, 5)
    rng = np.random.default_rng(0)
    q = torch.from_numpy(np.stack([rng.choice(3000, 2, replace=False) for _ in range(96)])).cuda()
    y = torch.from_numpy((np.arange(96) < 8).astype(np.float32)).cuda()
    outs = []
    for use_graph in (False, True):
        p = wj.init_params(2, 3, dropout=0.0, seed=1)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(s, p, st, use_graph=use_graph, mode="pooled")
        losses = [float(step(q, y)) for _ in range(3)]
        outs.append((losses, {k: v.clone() for k, v in p.tensors.items()}))
    np.testing.assert_allclose(outs[0][0], outs[1][0], rtol=1e-6)
    for k in outs[0][1]:
        torch.testing.assert_close(outs[0][1][k], outs[1][1][k], rtol=1e-5, atol=1e-7)


# ------------------------------------------------------------ fused encoder --

_M64 = (1 << 64) - 1


def _mix64(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _fused_model(store, q, w1, b1, keep, seed, step, warps=8):
    """Host model of wj_join_encode: pooled / S / msum per query, including
    the kernel's dropout stream (same counters, same row segmentation)."""
    G = 0x9E3779B97F4A7C15
    off = store.offsets_d.cpu().numpy()
    ux = store.uniq_x_d.cpu().numpy()
    uid = store.uniq_id_d.cpu().numpy()
    T = store.table.vectors.astype(np.int64)
    B, A = q.shape
    W = store.width
    P = store.landings
    H = w1.shape[1]
    thr = 65536 if keep >= 1 else int(keep * 65536.0 + 0.5)
    skey = _mix64((seed + G * (step + 1)) & _M64)
    pooled = np.zeros((B, H))
    S = np.zeros((B, A * W, H))
    msum = np.zeros((B, H))
    for b in range(B):
        lists = [(ux[off[q[b, j]]:off[q[b, j] + 1]], uid[off[q[b, j]]:off[q[b, j] + 1]]) for j in range(A)]
        for a in range(A):
            xa, ida = lists[a]
            ids = np.zeros((len(xa), A), np.int64)
            for j in range(A):
                if j == a:
                    ids[:, j] = ida
                else:
                    xj, idj = lists[j]
                    pos = np.searchsorted(xj, xa)
                    pos_c = np.minimum(pos, len(xj) - 1)
                    ids[:, j] = np.where((pos < len(xj)) & (xj[pos_c] == xa), idj[pos_c], 0)
            X = T[ids].reshape(len(xa), A * W).astype(np.float64)
            n_l = T[ida].sum(1)
            rowoff = np.concatenate([[0], np.cumsum(n_l)])
            z = (b1[None, :].astype(np.float64) + X @ w1.astype(np.float64)).astype(np.float32)
            kept = np.zeros((len(xa), H))
            if thr >= 65536:
                kept[:] = n_l[:, None]
            else:
                # draw of (row, unit u, lane): word (row // RPW, lane), field (row % RPW) * HU + u
                qkey = _mix64(skey ^ _mix64((b << 3) | a))
                HU = H // 32
                rpw = max(4 // HU, 1)
                owner = np.repeat(np.arange(len(xa)), n_l)  # local of each virtual row
                for wi in range((P + rpw - 1) // rpw):
                    for lane in range(32):
                        rnd = _mix64((qkey + ((wi << 5) | lane) * G) & _M64)
                        for rr in range(rpw):
                            row = wi * rpw + rr
                            if row >= P:
                                break
                            for u in range(HU):
                                if ((rnd >> (16 * (rr * HU + u))) & 0xFFFF) < thr:
                                    kept[owner[row], u * 32 + lane] += 1
            posm = z > 0
            pooled[b] += (np.where(posm, z, 0) * kept).sum(0)
            gk = posm * kept
            msum[b] += gk.sum(0)
            S[b] += X.T @ gk
    return pooled, S, msum


_M32 = (1 << 32) - 1


def _hash32(x):
    x = np.asarray(x, dtype=np.uint64)
    x ^= x >> np.uint64(16)
    x = (x * np.uint64(0x7FEB352D)) & np.uint64(_M32)
    x ^= x >> np.uint64(15)
    x = (x * np.uint64(0x846CA68B)) & np.uint64(_M32)
    x ^= x >> np.uint64(16)
    return x


def _lcg_jump_tables():
    a, c, A, C = 747796405, 2891336453, 1, 0
    ta, tc = [], []
    for _ in range(16):
        A, C = (A * a) & _M32, (C * a + c) & _M32
        ta.append(A)
        tc.append(C)
    return np.array(ta, dtype=np.uint64), np.array(tc, dtype=np.uint64)


_LCG_A, _LCG_C = _lcg_jump_tables()


def _thresholds14(keep):
    """14-bit inverse-CDF thresholds of the tensor-core kernel:
    (1-row P(K>=1), 2-row P(K>=1), 2-row P(K>=2))."""
    k = float(np.float32(keep))
    if k >= 1.0:
        return 16384, 16384, 16384
    t = lambda p: int(p * 16384.0 + 0.5)  # noqa: E731
    return t(k), t(1.0 - (1.0 - k) * (1.0 - k)), t(k * k)


def _fused_model_mma(store, q, w1, b1, keep, seed, step):
    """Host model of the tensor-core wj_join_encode: the query's virtual
    landings in the store's vindex order (section 2: landing l repeated
    floor(n_l/2) times per anchor, padded to 16; section 1: odd-n_l landings,
    padded), Binomial(2, keep) / Bernoulli(keep) kept rows from the kernel's
    14-bit hash stream; pooled / S / msum per query (float64)."""
    G = 0x9E3779B97F4A7C15
    off = store.offsets_d.cpu().numpy()
    ux = store.uniq_x_d.cpu().numpy()
    uid = store.uniq_id_d.cpu().numpy()
    T = store.table.vectors.astype(np.int64)
    B, A = q.shape
    W = store.width
    H = w1.shape[1]
    t11, t21, t22 = _thresholds14(keep)
    skey = _mix64((seed + G * (step + 1)) & _M64)
    h = np.arange(H, dtype=np.uint64)
    gq, hb, mt = h % 8, (h // 8) % 2, h // 16
    pooled = np.zeros((B, H))
    S = np.zeros((B, A * W, H))
    msum = np.zeros((B, H))
    for b in range(B):
        qq = _mix64(skey ^ _mix64(b)) & _M32
        qq ^= qq >> 16
        lists = [(ux[off[q[b, j]]:off[q[b, j] + 1]], uid[off[q[b, j]]:off[q[b, j] + 1]]) for j in range(A)]
        sec2, sec1 = [], []
        for a in range(A):
            xa, ida = lists[a]
            ids = np.zeros((len(xa), A), np.int64)
            for j in range(A):
                if j == a:
                    ids[:, j] = ida
                else:
                    xj, idj = lists[j]
                    pos = np.searchsorted(xj, xa)
                    pos_c = np.minimum(pos, len(xj) - 1)
                    ids[:, j] = np.where((pos < len(xj)) & (xj[pos_c] == xa), idj[pos_c], 0)
            X = T[ids].reshape(len(xa), A * W)
            n_l = T[ida].sum(1)
            for l in range(len(xa)):
                sec2 += [X[l]] * int(n_l[l] // 2)
            for l in range(len(xa)):
                if n_l[l] % 2:
                    sec1.append(X[l])
        zero = np.zeros(A * W, np.int64)
        pad = lambda r: r + [zero] * ((-len(r)) % 16)  # noqa: E731
        rows2, rows1 = pad(sec2), pad(sec1)
        X = np.asarray(rows2 + rows1, np.float64).reshape(-1, A * W)
        two = np.arange(X.shape[0]) < len(rows2)
        V = X.shape[0]
        z = (b1[None, :].astype(np.float64) + X @ w1.astype(np.float64)).astype(np.float32)
        z[np.all(X == 0, axis=1)] = 0.0  # padding rows: contribute nothing
        v = np.arange(V, dtype=np.uint64)[:, None]
        # per-tile part cq (landing tile v0, pair tq, unit row gq), plus the
        # per-pair counter k (block t, unit tile mt, unit half hb)
        tq = (v >> np.uint64(1)) & np.uint64(3)
        v0 = v & ~np.uint64(15)
        tt = (v >> np.uint64(3)) & np.uint64(1)
        cq = (np.uint64(qq) ^ (v0 << np.uint64(5)) ^ (tq << np.uint64(6)) ^ gq) & np.uint64(_M32)
        # per (lane, tile) seed = one full hash of cq; draw k = 8t + 2mt + hb is
        # the LCG (a = 747796405, c = 2891336453) jumped k + 1 steps ahead
        sd = (cq * np.uint64(0x7FEB352D)) & np.uint64(_M32)
        sd ^= sd >> np.uint64(15)
        sd = (sd * np.uint64(0x846CA68B)) & np.uint64(_M32)
        sd ^= sd >> np.uint64(16)
        k = (np.uint64(8) * tt + np.uint64(2) * mt + hb).astype(np.int64)
        x = (sd * _LCG_A[k] + _LCG_C[k]) & np.uint64(_M32)
        y = ~(x ^ (x >> np.uint64(16))) & np.uint64(0x3FFF3FFF)
        lane = np.where((v & np.uint64(1)) == 1, y >> np.uint64(16), y & np.uint64(0xFFFF)).astype(np.int64)
        u = 0x3FFF - lane
        ta = np.where(two, t21, t11)[:, None]
        tb = np.where(two, t22, 0)[:, None]
        kept = (u < ta).astype(np.float64) + (u < tb)
        posm = z >= 0
        pooled[b] = (np.where(posm, z, 0) * kept).sum(0)
        gk = posm * kept
        msum[b] = (gk * X.any(axis=1)[:, None]).sum(0)  # the bias column is 0 on padding rows
        S[b] = X.T @ gk
    return pooled, S, msum


def _tc_kernel_active(arity, L):
    """WJ_ENC_TC=4|8 selects the tcgen05 kernel (encode_tc.cu) for arity <= 2
    with A(L+1)+1 <= 16; otherwise the mma.sync kernel serves the shape."""
    return os.environ.get("WJ_ENC_TC", "0") in ("4", "8") and arity <= 2 and arity * (L + 1) + 1 <= 16


def _fused_model_tc(store, q, w1, b1, keep, seed, step):
    """Host model of the tcgen05 wj_join_encode (encode_tc.cu): the query's
    virtual landings in vindex order (section 2 padded to 32, section 1, the
    total padded to 128), counter (landing v, unit pair k): x = (qq + (v << 5)
    + k) * C1, one xorshift-multiply-xorshift round, the low 14-bit lane for
    unit 2k and the high one for unit 2k + 1."""
    G = 0x9E3779B97F4A7C15
    off = store.offsets_d.cpu().numpy()
    ux = store.uniq_x_d.cpu().numpy()
    uid = store.uniq_id_d.cpu().numpy()
    T = store.table.vectors.astype(np.int64)
    B, A = q.shape
    W = store.width
    H = w1.shape[1]
    t11, t21, t22 = _thresholds14(keep)
    skey = _mix64((seed + G * (step + 1)) & _M64)
    pooled = np.zeros((B, H))
    S = np.zeros((B, A * W, H))
    msum = np.zeros((B, H))
    kk = np.arange(H // 2, dtype=np.uint64)[None, :]
    for b in range(B):
        qq = _mix64(skey ^ _mix64(b)) & _M32
        qq ^= qq >> 16
        lists = [(ux[off[q[b, j]]:off[q[b, j] + 1]], uid[off[q[b, j]]:off[q[b, j] + 1]]) for j in range(A)]
        sec2, sec1 = [], []
        for a in range(A):
            xa, ida = lists[a]
            ids = np.zeros((len(xa), A), np.int64)
            for j in range(A):
                if j == a:
                    ids[:, j] = ida
                else:
                    xj, idj = lists[j]
                    pos = np.searchsorted(xj, xa)
                    pos_c = np.minimum(pos, len(xj) - 1)
                    ids[:, j] = np.where((pos < len(xj)) & (xj[pos_c] == xa), idj[pos_c], 0)
            X = T[ids].reshape(len(xa), A * W)
            n_l = T[ida].sum(1)
            for l in range(len(xa)):
                sec2 += [X[l]] * int(n_l[l] // 2)
            for l in range(len(xa)):
                if n_l[l] % 2:
                    sec1.append(X[l])
        zero = np.zeros(A * W, np.int64)
        rows2 = sec2 + [zero] * ((-len(sec2)) % 32)
        rows = rows2 + sec1
        rows = rows + [zero] * ((-len(rows)) % 128)
        X = np.asarray(rows, np.float64).reshape(-1, A * W)
        two = np.arange(X.shape[0]) < len(rows2)
        V = X.shape[0]
        z = (b1[None, :].astype(np.float64) + X @ w1.astype(np.float64)).astype(np.float32)
        z[np.all(X == 0, axis=1)] = 0.0  # padding rows: contribute nothing
        v = np.arange(V, dtype=np.uint64)[:, None]
        x = ((np.uint64(qq) + (v << np.uint64(5)) + kk) * np.uint64(0x7FEB352D)) & np.uint64(_M32)
        x ^= x >> np.uint64(15)
        x = (x * np.uint64(0x846CA68B)) & np.uint64(_M32)
        y = ~(x ^ (x >> np.uint64(16))) & np.uint64(0x3FFF3FFF)
        lanes = np.empty((V, H), np.int64)
        lanes[:, 0::2] = (y & np.uint64(0xFFFF)).astype(np.int64)
        lanes[:, 1::2] = (y >> np.uint64(16)).astype(np.int64)
        u = 0x3FFF - lanes
        ta = np.where(two, t21, t11)[:, None]
        tb = np.where(two, t22, 0)[:, None]
        kept = (u < ta).astype(np.float64) + (u < tb)
        posm = z >= 0
        pooled[b] = (np.where(posm, z, 0) * kept).sum(0)
        gk = posm * kept
        msum[b] = (gk * X.any(axis=1)[:, None]).sum(0)
        S[b] = X.T @ gk
    return pooled, S, msum


@pytest.mark.parametrize("keep", [1.0, 0.9])
@pytest.mark.parametrize("kernel", ["mma", "simt"])
@pytest.mark.parametrize("arity,L", [(2, 4), (3, 3)])
def test_fused_join_encode_matches_host_model(wj, keep, kernel, arity, L):
    g = _er(800, 6_000, 4)
    s = wj.preprocess(g, 40, L, 21)
    rng = np.random.default_rng(3)
    q = np.stack([rng.choice(800, arity, replace=False) for _ in range(12)]).astype(np.int64)
    p = wj.init_params(arity, L, dropout=1 - keep, seed=2)
    step = torch.tensor([6], dtype=torch.int64, device="cuda")
    pooled = torch.empty((12, 64), device="cuda")
    S = torch.empty((12, arity * (L + 1), 64), device="cuda")
    msum = torch.empty((12, 64), device="cuda")
    qd = torch.from_numpy(q).cuda()
    wj.encoder.join_encode(s, qd, p.w1, p.b1, float(keep), 99, step, pooled, S, msum, simt=(kernel == "simt"))
    w1 = p.w1.cpu().numpy()
    b1 = p.b1.cpu().numpy()
    model = _fused_model if kernel == "simt" else (_fused_model_tc if _tc_kernel_active(arity, L) else _fused_model_mma)
    mp, mS, mm = model(s, q, w1, b1, keep, 99, 6)
    np.testing.assert_allclose(pooled.cpu().numpy(), mp, rtol=2e-5, atol=1e-3)
    # S and msum are integer-weighted sums: exact unless a z sits within rounding of 0
    assert np.mean(np.abs(S.cpu().numpy() - mS) < 0.5) > 0.999
    assert np.mean(np.abs(msum.cpu().numpy() - mm) < 0.5) > 0.999
    if keep < 1:  # kept fraction ~ keep
        nod = model(s, q, w1, b1, 1.0, 99, 6)[2]
        frac = mm.sum() / nod.sum()
        assert abs(frac - keep) < 0.01


@pytest.mark.parametrize("nw", ["8", "4"])
@pytest.mark.parametrize("keep", [1.0, 0.9])
@pytest.mark.parametrize("arity,L", [(2, 4), (1, 3), (2, 6)])
def test_tcgen05_join_encode_matches_host_model(wj, monkeypatch, nw, keep, arity, L):
    """The tcgen05 + TMEM kernel (encode_tc.cu, WJ_ENC_TC=4|8) against the
    host model of its dropout stream: pooled within 2e-5, S / msum exact."""
    monkeypatch.setenv("WJ_ENC_TC", nw)
    g = _er(800, 6_000, 4)
    s = wj.preprocess(g, 40, L, 21)
    rng = np.random.default_rng(5)
    q = np.stack([rng.choice(800, arity, replace=False) for _ in range(20)]).astype(np.int64)
    p = wj.init_params(arity, L, dropout=1 - keep, seed=2)
    step = torch.tensor([6], dtype=torch.int64, device="cuda")
    pooled = torch.empty((20, 64), device="cuda")
    S = torch.empty((20, arity * (L + 1), 64), device="cuda")
    msum = torch.empty((20, 64), device="cuda")
    wj.encoder.join_encode(s, torch.from_numpy(q).cuda(), p.w1, p.b1, float(keep), 99, step, pooled, S, msum)
    mp, mS, mm = _fused_model_tc(s, q, p.w1.cpu().numpy(), p.b1.cpu().numpy(), keep, 99, 6)
    np.testing.assert_allclose(pooled.cpu().numpy(), mp, rtol=2e-5, atol=1e-3)
    assert np.mean(np.abs(S.cpu().numpy() - mS) < 0.5) > 0.999
    assert np.mean(np.abs(msum.cpu().numpy() - mm) < 0.5) > 0.999


def test_dropout_stream_statistics(wj):
    """Kept-row counts of the tensor-core kernel: mean keep * rows, binomial
    variance, and no correlation between neighbouring units / landings."""
    from paper_2202_13538_b200 import _lib

    g = _er(3_000, 40_000, 5)
    s = wj.preprocess(g, 100, 4, 13)
    rng = np.random.default_rng(8)
    q = torch.from_numpy(np.stack([rng.choice(3000, 2, replace=False) for _ in range(256)])).cuda()
    keep = 0.9
    p = wj.init_params(2, 4, dropout=0.0, seed=4)
    with torch.no_grad():  # z > 0 everywhere: msum counts kept rows
        p.tensors["w1"].abs_()
        p.tensors["b1"].fill_(0.5)
    outs = []
    for st in range(6):
        step = torch.tensor([st], dtype=torch.int64, device="cuda")
        ms = torch.empty((256, 64), device="cuda")
        pooled = torch.empty((256, 64), device="cuda")
        S = torch.empty((256, 10, 64), device="cuda")
        wj.encoder.join_encode(s, q, p.w1, p.b1, keep, 7, step, pooled, S, ms)
        outs.append(ms.double().cpu().numpy())
    rows = 2 * s.landings
    k = np.stack(outs)  # [steps, B, 64] kept rows out of `rows`
    frac = k / rows
    assert abs(frac.mean() - keep) < 2e-3
    # each entry is a sum of `rows` Bernoulli(keep): var = rows * keep * (1 - keep)
    var = k.var(axis=0).mean()
    assert 0.8 < var / (rows * keep * (1 - keep)) < 1.25
    # steps decorrelated, units decorrelated
    c_steps = np.corrcoef(k[0].ravel(), k[1].ravel())[0, 1]
    c_units = np.corrcoef(k[:, :, :-1].ravel(), k[:, :, 1:].ravel())[0, 1]
    assert abs(c_steps) < 0.05 and abs(c_units) < 0.05


@pytest.mark.parametrize("name", [c for c in golden_cases() if "logits" in load_golden(c)])
def test_fused_logits_and_grads_vs_reference(wj, name):
    """Fused path (no dropout) reproduces the reference logits and gradients."""
    g = load_golden(name)
    A, L = g["queries"].shape[1], int(g["L"])
    store = wj.preprocess(_graph(wj, g), int(g["M"]), L, int(g["seed"]))
    p = wj.encoder.params_from_numpy({k: g["p_" + k] for k in wj.encoder.TENSOR_ORDER}, A, L)
    qd = torch.from_numpy(g["queries"]).cuda()
    logits, cache = wj.encoder.forward_fused(p, store, qd, training=False)
    ref = g["logits"]
    np.testing.assert_allclose(logits.double().cpu().numpy(), ref, rtol=1e-5,
                               atol=1e-5 * max(np.abs(ref).max(), 1e-3))
    grads = wj.backward(p, cache, torch.from_numpy(g["labels"]).cuda())
    for k in wj.encoder.TENSOR_ORDER:
        r = g["g_" + k]
        np.testing.assert_allclose(grads[k].double().cpu().numpy(), r, rtol=1e-4,
                                   atol=1e-4 * max(np.abs(r).max(), 1e-12))


def test_fused_train_step_graph(wj):
    """Captured fused step == eager fused step; dropout masks change per step."""
    g = _er(3_000, 30_000, 2)
    s = wj.preprocess(g, 50, 3, 5)
    rng = np.random.default_rng(0)
    q = torch.from_numpy(np.stack([rng.choice(3000, 2, replace=False) for _ in range(96)])).cuda()
    y = torch.from_numpy((np.arange(96) < 8).astype(np.float32)).cuda()
    runs = []
    for use_graph in (False, True):
        p = wj.init_params(2, 3, dropout=0.1, seed=1)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(s, p, st, use_graph=use_graph, mode="fused", seed=4)
        losses = [float(step(q, y)) for _ in range(4)]
        runs.append((losses, {k: v.clone() for k, v in p.tensors.items()}))
    np.testing.assert_allclose(runs[0][0], runs[1][0], rtol=1e-5)
    for k in runs[0][1]:
        torch.testing.assert_close(runs[0][1][k], runs[1][1][k], rtol=1e-4, atol=1e-6)


def test_fast_tail_matches_torch_tail(wj):
    """wj_encoder_tail + wj_adam (flat buffers, deterministic partial sums)
    == the PyTorch tail of the same fused step, dropout included."""
    g = _er(2_000, 20_000, 6)
    s = wj.preprocess(g, 60, 4, 8)
    rng = np.random.default_rng(1)
    q = torch.from_numpy(np.stack([rng.choice(2000, 2, replace=False) for _ in range(203)])).cuda()
    y = torch.from_numpy((np.arange(203) % 7 == 0).astype(np.float32)).cuda()
    out = []
    for fast in (False, True):
        p = wj.init_params(2, 4, dropout=0.1, seed=3)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(s, p, st, mode="fused", seed=9, use_graph=fast, fast_tail=fast)
        assert step.fast_tail == fast
        losses = [float(step(q, y)) for _ in range(3)]
        out.append((losses, {k: v.clone() for k, v in p.tensors.items()}, {k: v.clone() for k, v in st.m.items()}))
    np.testing.assert_allclose(out[0][0], out[1][0], rtol=2e-5)
    for k in out[0][1]:
        torch.testing.assert_close(out[0][1][k], out[1][1][k], rtol=1e-4, atol=2e-6)
        torch.testing.assert_close(out[0][2][k], out[1][2][k], rtol=2e-3, atol=1e-7)


@pytest.mark.parametrize("arity", [2, 3])
def test_join_cross_matches_sorted_lookup(wj, arity):
    """wj_join_cross (merge path) == the RPE id of every landing of every
    anchor relative to every other anchor, by host binary search."""
    g = _er(1_500, 12_000, 7)
    s = wj.preprocess(g, 40, 3, 17)
    rng = np.random.default_rng(5)
    q = np.stack([rng.choice(1_500, arity, replace=False) for _ in range(64)]).astype(np.int64)
    q[0, 1] = q[0, 0]  # repeated anchor: every landing matches itself
    cross = wj.encoder.join_cross(s, torch.from_numpy(q).cuda()).cpu().numpy()
    off = s.offsets_d.cpu().numpy()
    ux = s.uniq_x_d.cpu().numpy()
    uid = s.uniq_id_d.cpu().numpy()
    for b in range(q.shape[0]):
        for a in range(arity):
            xa = ux[off[q[b, a]]:off[q[b, a] + 1]]
            others = [j for j in range(arity) if j != a]
            for jj, j in enumerate(others):
                xj = ux[off[q[b, j]]:off[q[b, j] + 1]]
                ij = uid[off[q[b, j]]:off[q[b, j] + 1]]
                pos = np.searchsorted(xj, xa)
                pc = np.minimum(pos, len(xj) - 1)
                want = np.where((pos < len(xj)) & (xj[pc] == xa), ij[pc], 0)
                np.testing.assert_array_equal(cross[b, a, jj, :len(xa)], want)


@pytest.mark.parametrize("name", ["er200", "idmap120"])
def test_save_store_is_byte_identical_to_reference(wj, name, tmp_path):
    """save_store of the device store == the file the reference save_store
    wrote for the same graph and arguments (tests/golden/make_surl_golden.py);
    load_store of that file gives back the same walks, table and dicts."""
    import os

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    d = np.load(os.path.join(here, f"surl_{name}.npz"))
    ref = open(os.path.join(here, f"surl_{name}.surl"), "rb").read()
    id_map = {int(k): int(v) for k, v in zip(d["id_keys"], d["id_vals"])} if len(d["id_keys"]) else None
    g = wj.Graph(int(d["n"]), d["idxptr"], d["indices"], id_map=id_map)
    s = wj.preprocess(g, int(d["M"]), int(d["L"]), int(d["seed"]))
    out = tmp_path / "store.surl"
    wj.save_store(s, out, chunk_bytes=4096)  # several device chunks
    assert out.read_bytes() == ref
    t = wj.load_store(out)
    assert np.array_equal(t.walks, s.walks) and np.array_equal(t.table.vectors, s.table.vectors)
    assert np.array_equal(t.dict_keys, s.dict_keys) and np.array_equal(t.dict_vals, s.dict_vals)
    assert t.seed == s.seed and t.id_map == s.id_map


def test_load_store_rejects_bad_files(wj, tmp_path):
    import os

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    ref = open(os.path.join(here, "surl_er200.surl"), "rb").read()
    cases = {"magic": b"XURL" + ref[4:], "truncated": ref[:-7], "trailing": ref + b"\0\0\0\0",
             "version": ref[:4] + b"\x02" + ref[5:]}
    for k, blob in cases.items():
        p = tmp_path / f"{k}.surl"
        p.write_bytes(blob)
        with pytest.raises(wj.StoreFormatError):
            wj.load_store(p)
