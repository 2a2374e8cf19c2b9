"""Parity at the BASELINE configs' shapes.

* C2 (ogbl-collab shape, 235,868 nodes / 1,285,465 edges, 5 % link split,
  M=200, L=4): the FULL device store against the oracle's full preprocess --
  walks, table and every dict slot bit for bit -- and a 4,096-query join
  (walk_nodes, rpe_ids) plus the fp64 dense tensor.
* C5a (tags-math shape: 1,629 nodes / 91,685 projected edges, triplet
  queries A=3, M=100, L=3): full store, arity-3 join + dense, the fused
  tensor-core encoder against the dense fp32 reference (logits 1e-5, grads
  1e-4, dropout off) and the production step executor against the graph step.
* C5b (ogbl-vessel shape: 3,538,495 nodes / 5,345,897 edges, degree ~3, so
  ~5 % isolated anchors that exercise the dead-end rule): the full store's
  properties over every anchor and the interning order, sampled anchors bit
  for bit against the oracle, and the full store of a 1/10-scale graph of the
  same degree bit for bit.
"""

import numpy as np
import pytest
import torch

from oracle import core

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wj():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2202_13538_b200 as m

    m._lib.load()
    return m


def _host_csr(g):
    return g.idxptr.long().cpu().numpy(), g.indices.cpu().numpy()


def assert_store_equals_oracle(store, ref):
    np.testing.assert_array_equal(store.walks, ref.walks)
    np.testing.assert_array_equal(store.table.vectors, ref.table)
    np.testing.assert_array_equal(store.dict_offsets, ref.dict_offsets)
    np.testing.assert_array_equal(store.dict_keys, ref.dict_keys)
    np.testing.assert_array_equal(store.dict_vals, ref.dict_vals)


def assert_join_equals_oracle(wj, store, ref, q, chunk=512):
    for lo in range(0, q.shape[0], chunk):
        qq = q[lo:lo + chunk]
        wn, ri = wj.join_batch_arrays(store, qq)
        wn_r, ri_r = core.join_batch_arrays(ref, qq)
        np.testing.assert_array_equal(wn, wn_r)
        np.testing.assert_array_equal(ri, ri_r)
        np.testing.assert_array_equal(wj.dense_batch(store, qq), core.dense_batch(ref, qq))


def interning_order_check(s, walks_of=None):
    """SURVEY Appendix B item 2 on the device, for every id k >= 1: the
    minimum scan position (anchor << 16 | first appearance) over the id's
    entries is strictly increasing in k (ids are first-occurrence ranks), and
    table row k is the count vector of that first entry recomputed from the
    walks (and the entry is the landing's first appearance)."""
    dev = s.device
    T = int(s.table_keys_d.numel())
    n = s.num_nodes
    big = torch.iinfo(torch.int64).max
    minord = torch.full((T,), big, dtype=torch.int64, device=dev)
    counts = s.anchor_counts()
    step = 1 << 18
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        e0, e1 = int(s.offsets_d[lo]), int(s.offsets_d[hi])
        owner = torch.repeat_interleave(torch.arange(lo, hi, device=dev), counts[lo:hi])
        first = s.uniq_first_d[e0:e1].to(torch.int64) & 0xFFFF
        minord.scatter_reduce_(0, s.uniq_id_d[e0:e1].long(), (owner << 16) | first, reduce="amin")
    assert int(minord[0]) == big, "id 0 (the zero sentinel) was assigned to an entry"
    mo = minord[1:]
    assert torch.all(mo < big), "an id of the table has no entry"
    assert torch.all(mo[1:] > mo[:-1]), "ids are not in first-occurrence order"
    anchors, first = mo >> 16, mo & 0xFFFF
    w = s.walks_d[anchors].reshape(T - 1, -1).long()  # [T-1, M*(L+1)]
    x = w.gather(1, first[:, None])
    hit = w == x
    pos = torch.arange(w.shape[1], device=dev)[None, :]
    assert not torch.any(hit & (pos < first[:, None])), "first is not the landing's first appearance"
    W = s.width
    cnt = hit.reshape(T - 1, s.num_walks, W).sum(1)
    assert torch.equal(cnt, s.table_d[1:].long())


def properties_every_anchor(g, s):
    """Column 0 is the anchor, every step is an edge (a repeat at an isolated
    node), every anchor's count vectors sum to M per column, sorted lists,
    no duplicate table rows."""
    dev = s.walks_d.device
    n, M, W = g.num_nodes, s.num_walks, s.width
    ip = g.idxptr.long()
    idx = g.indices.long()
    tab = s.table_d.long()
    counts = s.anchor_counts()
    assert torch.unique(s.table_keys_d).numel() == s.table_keys_d.numel()
    assert torch.all(tab[0] == 0)
    step = 262_144
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        w = s.walks_d[lo:hi].long()
        assert torch.equal(w[:, :, 0], torch.arange(lo, hi, device=dev)[:, None].expand(hi - lo, M))
        a = w[:, :, :-1].reshape(-1)
        b = w[:, :, 1:].reshape(-1)
        deg = ip[a + 1] - ip[a]
        iso = deg == 0
        assert torch.all(a[iso] == b[iso])
        a, b = a[~iso], b[~iso]
        left, right = ip[a].clone(), ip[a + 1].clone()
        for _ in range(32):
            mid = (left + right) // 2
            go = (left < right) & (idx[mid.clamp(max=idx.numel() - 1)] < b)
            left = torch.where(go, mid + 1, left)
            right = torch.where(go | (left >= right), right, mid)
        assert torch.all(idx[left.clamp(max=idx.numel() - 1)] == b)
        e0, e1 = int(s.offsets_d[lo]), int(s.offsets_d[hi])
        owner = torch.repeat_interleave(torch.arange(hi - lo, device=dev), counts[lo:hi])
        sums = torch.zeros((hi - lo, W), dtype=torch.int64, device=dev)
        sums.index_add_(0, owner, tab[s.uniq_id_d[e0:e1].long()])
        assert torch.all(sums == M)
        ux = s.uniq_x_d[e0:e1].long()
        first = torch.zeros(e1 - e0, dtype=torch.bool, device=dev)
        first[(s.offsets_d[lo:hi] - e0)[counts[lo:hi] > 0]] = True
        assert torch.all((ux[1:] > ux[:-1]) | first[1:])


def sampled_anchors_vs_oracle(g, s, nodes, seed):
    """Walks, sorted landings with count vectors and first-appearance slots
    of the sampled anchors against the oracle's sampler + compute_rpe."""
    ip, ix = _host_csr(g)
    M, L = s.num_walks, s.walk_steps
    ref_walks = core.sample_nodes(ip, ix, nodes, M, L, seed)
    np.testing.assert_array_equal(s.walks_d[torch.from_numpy(nodes).cuda()].cpu().numpy(), ref_walks)
    off = s.offsets_d.cpu()
    tab = s.table_d.cpu().numpy()
    for k, u in enumerate(nodes):
        e0, e1 = int(off[u]), int(off[u + 1])
        ux = s.uniq_x_d[e0:e1].cpu().numpy()
        vec = tab[s.uniq_id_d[e0:e1].long().cpu().numpy()]
        ref = core.compute_rpe(ref_walks[k])
        keys = np.array(sorted(ref), dtype=np.int64)
        np.testing.assert_array_equal(ux, keys)
        np.testing.assert_array_equal(vec, np.stack([ref[int(x)] for x in keys]))
        flat = ref_walks[k].reshape(-1)
        want_first = np.array([int(np.argmax(flat == x)) for x in keys])
        np.testing.assert_array_equal(s.uniq_first_d[e0:e1].cpu().numpy().view(np.uint16), want_first)
    return ref_walks


# ---------------------------------------------------------------- C2 --

def test_c2_full_store_and_join_bit_exact_vs_oracle(wj):
    split = wj.graph.synthetic_link_graph(235_868, 1_285_465, 0.05, seed=1, device="cuda")
    g = split.walk_graph
    s = wj.preprocess(g, 200, 4, 3)
    ip, ix = _host_csr(g)
    ref = core.preprocess(ip, ix, 200, 4, 3)
    assert_store_equals_oracle(s, ref)
    rng = np.random.default_rng(11)
    # training-batch-like queries (pairs inside small seed sets) and uniform pairs
    seeds = rng.integers(0, g.num_nodes, 64)
    q = np.concatenate([np.stack([rng.choice(seeds, 2, replace=False) for _ in range(2048)]),
                        np.stack([rng.choice(g.num_nodes, 2, replace=False) for _ in range(2048)])])
    assert_join_equals_oracle(wj, s, ref, q.astype(np.int64))
    interning_order_check(s)


# --------------------------------------------------------------- C5a --

@pytest.fixture(scope="module")
def c5a(wj):
    split = wj.graph.synthetic_link_graph(1_629, 91_685, 0.05, seed=2, device="cuda")
    g = split.walk_graph
    s = wj.preprocess(g, 100, 3, 3)
    ip, ix = _host_csr(g)
    return g, s, core.preprocess(ip, ix, 100, 3, 3)


def _triplets(rng, n, count):
    return np.stack([rng.choice(n, 3, replace=False) for _ in range(count)]).astype(np.int64)


def test_c5a_store_and_triplet_join_bit_exact(wj, c5a):
    g, s, ref = c5a
    assert_store_equals_oracle(s, ref)
    assert_join_equals_oracle(wj, s, ref, _triplets(np.random.default_rng(1), g.num_nodes, 1024), chunk=256)
    interning_order_check(s)


def test_c5a_fused_encoder_vs_dense_reference(wj, c5a):
    g, s, _ = c5a
    rng = np.random.default_rng(5)
    q = torch.from_numpy(_triplets(rng, g.num_nodes, 120)).cuda()
    y = torch.from_numpy((np.arange(120) < 11).astype(np.float32)).cuda()
    p = wj.init_params(3, 3, dropout=0.0, seed=8)
    logits, cache = wj.encoder.forward_fused(p, s, q, training=False)
    grads = wj.backward(p, cache, y)
    dense = wj.dense_batch(s, q, dtype=torch.float32)
    logits_r, cache_r = wj.forward(p, dense, training=False, mode="reference")
    grads_r = wj.backward(p, cache_r, y)
    lr = logits_r.double()
    torch.testing.assert_close(logits.double(), lr, rtol=1e-5, atol=1e-5 * float(lr.abs().max()))
    for k in wj.encoder.TENSOR_ORDER:
        r = grads_r[k].double()
        torch.testing.assert_close(grads[k].double(), r, rtol=1e-4, atol=1e-4 * max(float(r.abs().max()), 1e-12))
    # scoring (keep = 1 variant + tail kernel) == the dense reference's sigmoid
    torch.testing.assert_close(wj.score_array(s, p, q), torch.sigmoid(lr), rtol=1e-5, atol=1e-6)


def test_c5a_step_executor_equals_graph_step(wj, c5a):
    g, s, _ = c5a
    rng = np.random.default_rng(6)
    q = torch.from_numpy(_triplets(rng, g.num_nodes, 330)).cuda()
    y = torch.from_numpy((np.arange(330) < 30).astype(np.float32)).cuda()
    outs = []
    for launch in ("graph", "chain"):
        p = wj.init_params(3, 3, dropout=0.1, seed=4)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(s, p, st, seed=3, launch=launch)
        assert step.launch == launch
        losses = [float(step(q, y)) for _ in range(3)]
        outs.append((losses, {k: v.clone() for k, v in p.tensors.items()}))
    assert outs[0][0] == outs[1][0]
    assert all(torch.equal(outs[0][1][k], outs[1][1][k]) for k in outs[0][1])


# --------------------------------------------------------------- C5b --

def test_c5b_vessel_shape_full_size(wj):
    n, m = 3_538_495, 5_345_897
    split = wj.graph.synthetic_link_graph(n, m, 0.05, seed=1, device="cuda")
    g = split.walk_graph
    deg = g.idxptr[1:].long() - g.idxptr[:-1].long()
    iso = torch.nonzero(deg == 0).squeeze(1)
    assert iso.numel() > 0.04 * n  # the dead-end path is exercised at scale
    s = wj.preprocess(g, 200, 4, 3)
    properties_every_anchor(g, s)
    interning_order_check(s)
    rng = np.random.default_rng(9)
    nodes = np.unique(np.concatenate([rng.integers(0, n, 300), iso[:40].cpu().numpy(), [0, n - 1]]))
    ref_walks = sampled_anchors_vs_oracle(g, s, nodes, 3)
    # isolated anchors: every walk repeats the anchor (_kernels.py:61-64)
    isoset = set(iso[:40].tolist())
    for k, u in enumerate(nodes):
        if int(u) in isoset:
            assert np.all(ref_walks[k] == u)
    # joined queries over sampled anchors (incl. isolated ones)
    q = np.stack([rng.choice(nodes, 2, replace=False) for _ in range(64)]).astype(np.int64)
    wn, ri = wj.join_batch_arrays(s, q)
    tab = s.table_d.cpu().numpy()
    for b in range(q.shape[0]):
        blocks = [ref_walks[np.searchsorted(nodes, q[b, a])] for a in range(2)]
        np.testing.assert_array_equal(wn[b], np.concatenate(blocks))
        rpes = [core.compute_rpe(blk) for blk in blocks]
        cells = np.concatenate(blocks).reshape(-1)
        for a in range(2):
            want = np.stack([rpes[a].get(int(x), np.zeros(5, np.int32)) for x in cells])
            np.testing.assert_array_equal(tab[ri[b][:, a]], want)


def test_c5b_vessel_shape_tenth_scale_full_store(wj):
    split = wj.graph.synthetic_link_graph(353_850, 534_590, 0.05, seed=1, device="cuda")
    g = split.walk_graph
    s = wj.preprocess(g, 200, 4, 3)
    ip, ix = _host_csr(g)
    ref = core.preprocess(ip, ix, 200, 4, 3)
    assert_store_equals_oracle(s, ref)
    rng = np.random.default_rng(2)
    iso = np.nonzero(np.diff(ip) == 0)[0]
    q = np.concatenate([np.stack([rng.choice(g.num_nodes, 2, replace=False) for _ in range(1000)]),
                        np.stack([iso[:24], rng.choice(g.num_nodes, 24)], 1)]).astype(np.int64)
    q = q[q[:, 0] != q[:, 1]]
    assert_join_equals_oracle(wj, s, ref, q)
    interning_order_check(s)
