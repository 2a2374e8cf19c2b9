"""Parity at the headline size (BASELINE configs[2]: citation2 shape,
2,927,963 nodes / 30,561,187 edges, M=200, L=4; store ~35 GB on the device).

The full store cannot be checked against the oracle (its interning is a
sequential scan over ~1.5 G entries), so this checks (1) size-independent
properties over EVERY anchor -- column 0 is the anchor, every step is an
edge, each anchor's count vectors sum to M in every column, uniq lists are
strictly increasing, the table has no duplicates -- and (2) bit-exactness
against the oracle on a random sample of anchors spread over the whole node
range: their walks, their sorted distinct landings with count vectors (the
table row of every RPE id), and the join of sampled queries.
"""

import numpy as np
import pytest
import torch

from oracle import core

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    import paper_2202_13538_b200 as wj

    dev = torch.device("cuda")
    split = wj.graph.synthetic_link_graph(2_927_963, 30_561_187, 0.05, seed=1, device=dev)
    g = split.walk_graph
    s = wj.preprocess(g, 200, 4, 3)
    yield g, s
    del s
    torch.cuda.empty_cache()


def test_c3_properties_every_anchor(c3):
    g, s = c3
    dev = s.walks_d.device
    n, M, W = g.num_nodes, 200, 5
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
        for _ in range(32):  # binary search b in a's sorted neighbour row
            mid = (left + right) // 2
            go = (left < right) & (idx[mid.clamp(max=idx.numel() - 1)] < b)
            left = torch.where(go, mid + 1, left)
            right = torch.where(go | (left >= right), right, mid)
        assert torch.all(idx[left.clamp(max=idx.numel() - 1)] == b)
        # RPE mass and sortedness of this anchor range's entries
        e0, e1 = int(s.offsets_d[lo]), int(s.offsets_d[hi])
        owner = torch.repeat_interleave(torch.arange(hi - lo, device=dev), counts[lo:hi])
        sums = torch.zeros((hi - lo, W), dtype=torch.int64, device=dev)
        sums.index_add_(0, owner, tab[s.uniq_id_d[e0:e1].long()])
        assert torch.all(sums == M)
        ux = s.uniq_x_d[e0:e1].long()
        first = torch.zeros(e1 - e0, dtype=torch.bool, device=dev)
        first[(s.offsets_d[lo:hi] - e0)[counts[lo:hi] > 0]] = True
        assert torch.all((ux[1:] > ux[:-1]) | first[1:])


def test_c3_sampled_anchors_bit_exact_vs_oracle(c3):
    import paper_2202_13538_b200 as wj

    g, s = c3
    rng = np.random.default_rng(7)
    n = g.num_nodes
    nodes = np.unique(np.concatenate([rng.integers(0, n, 400), [0, n - 1]]))
    ip = g.idxptr.long().cpu().numpy()
    ix = g.indices.cpu().numpy()
    ref_walks = core.sample_nodes(ip, ix, nodes, 200, 4, 3)
    walks = s.walks_d[torch.from_numpy(nodes).cuda()].cpu().numpy()
    np.testing.assert_array_equal(walks, ref_walks)
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
    # the join of sampled queries: walk nodes and per-cell RPE vectors
    q = np.stack([rng.choice(nodes, 2, replace=False) for _ in range(16)]).astype(np.int64)
    wn, ri = wj.join_batch_arrays(s, q)
    for b in range(q.shape[0]):
        A = q.shape[1]
        blocks = [ref_walks[np.searchsorted(nodes, q[b, a])] for a in range(A)]
        np.testing.assert_array_equal(wn[b], np.concatenate(blocks))
        rpes = [core.compute_rpe(blk) for blk in blocks]
        cells = np.concatenate(blocks).reshape(-1)
        for a in range(A):  # every cell's RPE id maps to its count vector w.r.t. anchor a
            want = np.stack([rpes[a].get(int(x), np.zeros(5, np.int32)) for x in cells])
            np.testing.assert_array_equal(tab[ri[b][:, a]], want)


def test_c3_interning_order_every_id(c3):
    """At the headline size: every global RPE id is the first-occurrence
    rank of its vector in (anchor, first appearance) order, and each table
    row is the count vector of that first entry recomputed from the walks
    (the sequential definition _kernels.py:137-171)."""
    from test_gpu_configs import interning_order_check

    g, s = c3
    interning_order_check(s)


def test_c3_sampled_first_appearance_slots(c3):
    from test_gpu_configs import sampled_anchors_vs_oracle

    g, s = c3
    rng = np.random.default_rng(17)
    nodes = np.unique(rng.integers(0, g.num_nodes, 64))
    sampled_anchors_vs_oracle(g, s, nodes, 3)


def test_c3_fused_encoder_vs_dense_reference(c3):
    """The fused join+encode kernel at the headline size (lists of ~530
    distinct landings per anchor, the training batch's query mix) against the
    dense path (wj_join -> fp32 PyTorch encoder, mode="reference" order),
    dropout off: logits within 1e-5, gradients within 1e-4 (relative)."""
    import paper_2202_13538_b200 as wj

    g, s = c3
    rng = np.random.default_rng(3)
    n = g.num_nodes
    seeds = rng.integers(0, n, 48)
    q = np.stack([rng.choice(seeds, 2, replace=False) for _ in range(96)]).astype(np.int64)
    y = torch.from_numpy((np.arange(96) < 6).astype(np.float32)).cuda()
    qd = torch.from_numpy(q).cuda()
    p = wj.init_params(2, 4, dropout=0.0, seed=21)
    logits, cache = wj.encoder.forward_fused(p, s, qd, training=False)
    grads = wj.backward(p, cache, y)
    dense = wj.dense_batch(s, qd, dtype=torch.float32)
    logits_r, cache_r = wj.forward(p, dense, training=False, mode="reference")
    grads_r = wj.backward(p, cache_r, y)
    lr = logits_r.double()
    torch.testing.assert_close(logits.double(), lr, rtol=1e-5, atol=1e-5 * float(lr.abs().max()))
    for k in wj.encoder.TENSOR_ORDER:
        r = grads_r[k].double()
        torch.testing.assert_close(grads[k].double(), r, rtol=1e-4, atol=1e-4 * max(float(r.abs().max()), 1e-12))
