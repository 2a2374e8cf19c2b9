"""Multi-GPU sharding of the hot path (one process per GPU, NCCL over NVLink).

Sampling and RPE are independent per anchor (the walk stream of u depends
only on (seed, u), reference _kernels.py:47-50,72-74), so rank r builds the
index of the contiguous node range [r*n/P, (r+1)*n/P) of the replicated CSR.
The path has exactly two exchange steps:

1. global RPE-id numbering -- each rank folds its entries into a local table
   of distinct vectors with their first scan order; the (key, order) sets
   (thousands of entries) are all-gathered and merged identically on every
   rank, so every rank derives the same ids as the single-GPU store;
2. the store itself -- walks / slot_idx (fixed size per anchor) and the
   variable-size per-anchor lists are all-gathered so that any rank can join
   any query (queries touch anchors of every shard).

Training is data parallel: each rank steps its own batches and the encoder
gradients (~9K floats) are all-reduced inside the captured step
(``TrainStep(process_group=...)``).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib
from .graph import DeviceGraph
from .sampler import _Phases, _u64
from .store import SubgraphStore


def shard_range(n: int, world: int, rank: int):
    return rank * n // world, (rank + 1) * n // world


_NCCL_DTYPES = (torch.uint8, torch.int8, torch.int32, torch.int64, torch.float16, torch.bfloat16,
                torch.float32, torch.float64)


def all_gather_variable(t: torch.Tensor, group=None) -> list:
    """All-gather tensors whose first dimension differs per rank (pad to the
    max, one all_gather, slice).  Works on gloo (CPU) and NCCL; dtypes NCCL
    lacks (int16 slot indices, uint16 first-appearance slots) travel as bytes."""
    if t.dtype not in _NCCL_DTYPES:
        dt = t.dtype
        rows = t.shape[0]
        per_row = t.element_size() * (t[0].numel() if rows else int(torch.tensor(t.shape[1:]).prod()))
        as_bytes = t.contiguous().view(torch.uint8).reshape(rows, per_row)
        return [p.reshape(-1).view(dt).reshape((p.shape[0],) + tuple(t.shape[1:]))
                for p in all_gather_variable(as_bytes, group)]
    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return [b[:s] for b, s in zip(bufs, sizes)]


def _bytes_view(t: torch.Tensor) -> torch.Tensor:
    return t if t.dtype in _NCCL_DTYPES else t.view(torch.uint8)


def gather_into(out: torch.Tensor, local: torch.Tensor, rows: list, group=None) -> torch.Tensor:
    """Concatenate every rank's ``local`` (rows[j] rows on rank j) into the
    preallocated ``out`` in rank order: one broadcast per rank straight into
    its slice of ``out`` -- no padding, no per-rank temporaries, no second copy
    of the store (the padded all_gather + cat this replaces held ~2x the
    store at the citation2 shape)."""
    rank = dist.get_rank(group)
    off = 0
    for j, n in enumerate(rows):
        dst = out[off: off + n]
        if j == rank:
            dst.copy_(local[:n])
        if n:
            dist.broadcast(_bytes_view(dst), src=dist.get_global_rank(group, j) if group is not None else j,
                           group=group)
        off += n
    return out


def all_gather_sizes(n: int, device, group=None) -> list:
    world = dist.get_world_size(group)
    t = torch.tensor([int(n)], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(sizes, t, group=group)
    return [int(x.item()) for x in sizes]


def merge_distinct(keys: torch.Tensor, orders: torch.Tensor):
    """Merge per-rank (packed vector, first scan order) pairs: min order per
    distinct vector, then ids = 1 + rank by that order.  Returns
    (sorted_keys, id_of_sorted_key int32, table_keys [T] with row 0 = 0)."""
    uk, inv = torch.unique(keys, sorted=True, return_inverse=True)
    big = torch.iinfo(torch.int64).max
    mins = torch.full((uk.numel(),), big, dtype=torch.int64, device=keys.device)
    mins.scatter_reduce_(0, inv, orders, reduce="amin")
    perm = torch.argsort(mins)
    ids = torch.empty(uk.numel(), dtype=torch.int32, device=keys.device)
    ids[perm] = torch.arange(1, uk.numel() + 1, dtype=torch.int32, device=keys.device)
    table_keys = torch.cat([torch.zeros(1, dtype=torch.int64, device=keys.device), uk[perm]])
    return uk, ids, table_keys


def preprocess_sharded(g, num_walks: int, num_steps: int, seed: int, threads: int = 1,
                       phases: list = None, group=None) -> SubgraphStore:
    """Sharded Alg. 1: every rank returns the full, identical store."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    dg = DeviceGraph.from_graph(g, dev)
    n, M, L = dg.num_nodes, int(num_walks), int(num_steps)
    W, P = L + 1, int(num_walks) * (int(num_steps) + 1)
    lo, hi = shard_range(n, world, rank)
    nl = hi - lo
    s = _lib.stream_handle(dev)
    ph = _Phases(phases)
    ph.mark("sample")
    walks_l = torch.empty((nl, M, W), dtype=torch.int32, device=dev)
    flags = torch.zeros(max(nl, 1), dtype=torch.uint8, device=dev)
    _lib.call("wj_sample_walks", _lib.ptr(dg.idxptr), dg.idxptr_bytes, _lib.ptr(dg.indices), n, lo, hi,
              M, L, _u64(seed), _lib.ptr(walks_l), _lib.ptr(flags), s)
    ph.mark("rpe_count")
    counts_l = torch.empty(nl, dtype=torch.int32, device=dev)
    _lib.call("wj_rpe_count", _lib.ptr(walks_l), nl, M, L, n, _lib.ptr(counts_l), s)
    off_l = torch.zeros(nl + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts_l, 0, out=off_l[1:])
    total_l = int(off_l[-1].item())
    ph.mark("rpe_fill")
    ux_l = torch.empty(total_l, dtype=torch.int32, device=dev)
    ukey_l = torch.empty(total_l, dtype=torch.int64, device=dev)
    uf_l = torch.empty(total_l, dtype=torch.int16, device=dev)
    slot_l = torch.empty((nl, P), dtype=torch.int16, device=dev)
    _lib.call("wj_rpe_fill", _lib.ptr(walks_l), nl, M, L, n, _lib.ptr(off_l), _lib.ptr(ux_l),
              _lib.ptr(ukey_l), _lib.ptr(uf_l), _lib.ptr(slot_l), s)
    ph.mark("intern")
    cap = 1 << max(12, (2 * min(max(total_l, 1), 1 << 20) - 1).bit_length())
    keys = torch.zeros(cap, dtype=torch.int64, device=dev)
    order = torch.full((cap,), -1, dtype=torch.int64, device=dev)
    overflow = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("wj_intern_insert", _lib.ptr(ukey_l), _lib.ptr(uf_l), _lib.ptr(off_l), nl, lo,
              _lib.ptr(keys), _lib.ptr(order), cap, _lib.ptr(overflow), s)
    if int(overflow.item()):
        raise RuntimeError("sharded intern table overflow")
    occ = keys != 0
    gk = torch.cat(all_gather_variable(keys[occ], group))
    go = torch.cat(all_gather_variable(order[occ], group))
    uk, ids, table_keys = merge_distinct(gk, go)
    uid_l = ids[torch.searchsorted(uk, ukey_l)]
    ph.mark("gather")
    # exchange the store: every array gathered straight into its full-size
    # buffer (fixed-size per anchor: walks / slot_idx; variable: the lists)
    world_rows = [shard_range(n, world, j)[1] - shard_range(n, world, j)[0] for j in range(world)]
    counts = gather_into(torch.empty(n, dtype=torch.int32, device=dev), counts_l, world_rows, group)
    offsets = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=offsets[1:])
    walks = gather_into(torch.empty((n, M, W), dtype=torch.int32, device=dev), walks_l, world_rows, group)
    del walks_l
    slot = gather_into(torch.empty((n, P), dtype=torch.int16, device=dev), slot_l, world_rows, group)
    del slot_l
    ent_rows = all_gather_sizes(total_l, dev, group)
    total = sum(ent_rows)
    ux = gather_into(torch.empty(total, dtype=torch.int32, device=dev), ux_l, ent_rows, group)
    uid = gather_into(torch.empty(total, dtype=torch.int32, device=dev), uid_l, ent_rows, group)
    uf = gather_into(torch.empty(total, dtype=torch.int16, device=dev), uf_l, ent_rows, group)
    del ux_l, uid_l, uf_l
    store = SubgraphStore(n, M, L, _u64(seed), walks, offsets, ux, uid, uf, slot, table_keys,
                          int(counts.max().item()) if n else 0, id_map=getattr(g, "id_map", None))
    ph.mark("vindex")
    store.build_vindex()  # every rank holds the full store: no exchange needed
    ph.mark("end")
    return store


def all_reduce_mean(t: torch.Tensor, group=None) -> None:
    """In-place mean over ranks: one ncclAllReduce(avg) on NCCL (capturable
    in a CUDA graph), sum + divide on gloo."""
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.AVG, group=group)
    else:
        dist.all_reduce(t, group=group)
        t.div_(dist.get_world_size(group))


def all_reduce_grads(grads: dict, order, group=None) -> None:
    """Average the encoder gradients over ranks with one flat all-reduce."""
    flat = torch.cat([grads[k].reshape(-1) for k in order])
    all_reduce_mean(flat, group)
    off = 0
    for k in order:
        n = grads[k].numel()
        grads[k] = flat[off: off + n].view_as(grads[k])
        off += n
