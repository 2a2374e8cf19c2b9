"""Walk sampling + RPE construction on the B200 (reference sampler.py).

``preprocess`` is Alg. 1 (reference sampler.py:94-151) with every phase on
the device: wj_sample_walks -> wj_rpe_count -> cumsum -> wj_rpe_fill ->
wj_intern_insert -> (rank distinct vectors by first occurrence) ->
wj_intern_assign.  The result is bit-identical to the reference store for
the same (graph, M, L, seed): walks, table and every per-node RPE id.
``threads`` is accepted for signature compatibility and ignored (the grid
covers the whole GPU).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph
from .store import SubgraphStore, unpack_table

_MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def _mix64(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


@dataclass
class WalkSet:
    """M walks of m steps from one anchor; column 0 is the anchor (sampler.py:26-31)."""

    anchor: int
    walks: np.ndarray


@dataclass
class RawRpeMap:
    """Positional counts per reached node, first-appearance order (sampler.py:34-39)."""

    entries: dict = field(default_factory=dict)


class WalkRng:
    """Counter stream of one node (sampler.py:42-51)."""

    def __init__(self, state: int):
        self.state = int(state) & _MASK64

    @classmethod
    def for_node(cls, seed: int, node: int) -> "WalkRng":
        return cls(_mix64((int(seed) + _GOLDEN * (int(node) + 1)) & _MASK64))


def _u64(x: int) -> int:
    return int(x) & _MASK64


def sample_walks(g, u: int, num_walks: int, num_steps: int, rng: WalkRng, device=None) -> WalkSet:
    """M uniform walks from u on the device; advances ``rng`` (sampler.py:61-76)."""
    if not 0 <= u < g.num_nodes:
        raise ValueError(f"node id {u} out of range [0, {g.num_nodes})")
    if num_walks < 1 or num_steps < 1:
        raise ValueError("num_walks and num_steps must be >= 1")
    dev = _lib.require_cuda(device if device is not None else getattr(g, "device", None))
    dg = DeviceGraph.from_graph(g, dev)
    out = torch.empty((num_walks, num_steps + 1), dtype=torch.int32, device=dev)
    end = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.call("wj_sample_node_walks", _lib.ptr(dg.idxptr), dg.idxptr_bytes, _lib.ptr(dg.indices),
              int(u), num_walks, num_steps, _u64(rng.state), _lib.ptr(out), _lib.ptr(end),
              _lib.stream_handle(dev))
    rng.state = int(end.item()) & _MASK64
    return WalkSet(anchor=int(u), walks=out.cpu().numpy())


def compute_rpe(ws: WalkSet, device=None) -> RawRpeMap:
    """Exact positional counts of one walk set, first-appearance order
    (sampler.py:79-91), computed by the RPE kernels on one anchor."""
    walks = np.ascontiguousarray(ws.walks, dtype=np.int32)
    M, W = walks.shape
    dev = _lib.require_cuda(device)
    wd = torch.from_numpy(walks).to(dev)
    n_nodes = int(walks.max()) + 1 if walks.size else 1
    counts = torch.empty(1, dtype=torch.int32, device=dev)
    s = _lib.stream_handle(dev)
    _lib.call("wj_rpe_count", _lib.ptr(wd), 1, M, W - 1, n_nodes, _lib.ptr(counts), s)
    total = int(counts.item())
    offsets = torch.tensor([0, total], dtype=torch.int64, device=dev)
    ux = torch.empty(total, dtype=torch.int32, device=dev)
    ukey = torch.empty(total, dtype=torch.int64, device=dev)
    ufirst = torch.empty(total, dtype=torch.int16, device=dev)
    slot = torch.empty(M * W, dtype=torch.int16, device=dev)
    _lib.call("wj_rpe_fill", _lib.ptr(wd), 1, M, W - 1, n_nodes, _lib.ptr(offsets), _lib.ptr(ux),
              _lib.ptr(ukey), _lib.ptr(ufirst), _lib.ptr(slot), s)
    vecs = unpack_table(ukey, M, W).cpu().numpy()
    first = ufirst.cpu().numpy().view(np.uint16)
    xs = ux.cpu().numpy()
    order = np.argsort(first, kind="stable")
    return RawRpeMap({int(xs[i]): vecs[i].copy() for i in order})


def _next_pow2(v: int) -> int:
    return 1 << max(1, (int(v) - 1).bit_length())


def intern_device(uniq_key, uniq_first, offsets, n_anchors, anchor_base, num_walks, width, return_order=False):
    """Global RPE ids for every entry: phase 1/3 on device, phase 2 (order the
    distinct vectors by first occurrence) with torch.  Returns
    (uniq_id int32 [E], table_keys int64 [T] with row 0 = 0) [+ the scan
    order (anchor << 16 | first) of each id's first occurrence, int64 [T-1],
    with ``return_order``]."""
    dev = uniq_key.device
    total = int(uniq_key.numel())
    s = _lib.stream_handle(dev)
    cap = _next_pow2(max(4096, 2 * min(total, 1 << 20)))
    while True:
        keys = torch.zeros(cap, dtype=torch.int64, device=dev)
        order = torch.full((cap,), -1, dtype=torch.int64, device=dev)
        overflow = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("wj_intern_insert", _lib.ptr(uniq_key), _lib.ptr(uniq_first), _lib.ptr(offsets),
                  n_anchors, anchor_base, _lib.ptr(keys), _lib.ptr(order), cap, _lib.ptr(overflow), s)
        if int(overflow.item()) == 0:
            break
        if cap >= 2 * total + 2:
            raise RuntimeError("intern table overflow at full capacity")
        cap = min(cap * 8, _next_pow2(2 * total + 2))
    occ = torch.nonzero(keys != 0).squeeze(1)
    perm = torch.argsort(order[occ])
    ids = torch.zeros(cap, dtype=torch.int32, device=dev)
    ids[occ[perm]] = torch.arange(1, occ.numel() + 1, dtype=torch.int32, device=dev)
    table_keys = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), keys[occ[perm]]])
    uniq_id = torch.empty(total, dtype=torch.int32, device=dev)
    _lib.call("wj_intern_assign", _lib.ptr(uniq_key), total, _lib.ptr(keys), _lib.ptr(ids), cap,
              _lib.ptr(uniq_id), s)
    if return_order:
        return uniq_id, table_keys, order[occ[perm]]
    return uniq_id, table_keys


class _Phases:
    """Optional CUDA-event bracketing of preprocess phases (for bench.py)."""

    def __init__(self, sink):
        self.sink = sink
        self.last = None

    def mark(self, name):
        if self.sink is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        if self.last is not None:
            self.sink.append((self.last[0], self.last[1], ev))
        self.last = (name, ev)


def preprocess(g, num_walks: int, num_steps: int, seed: int, threads: int = 1,
               device=None, keep_keys: bool = False, phases: list = None) -> SubgraphStore:
    """Build the device store (Alg. 1, reference sampler.py:94-151).

    ``phases`` (optional list) receives (name, start_event, end_event) per
    phase: sample, rpe_count, rpe_fill, intern, vindex."""
    if num_walks < 1 or num_steps < 1:
        raise ValueError("num_walks and num_steps must be >= 1")
    if threads < 1:
        raise ValueError("threads must be >= 1")
    if g.num_nodes >= 2 ** 31:
        raise ValueError("graphs with >= 2^31 nodes are not supported")
    dev = _lib.require_cuda(device if device is not None else getattr(g, "device", None))
    dg = DeviceGraph.from_graph(g, dev)
    n, M, L = dg.num_nodes, int(num_walks), int(num_steps)
    W = L + 1
    seed64 = _u64(seed)
    s = _lib.stream_handle(dev)
    walks = torch.empty((n, M, W), dtype=torch.int32, device=dev)
    flags = torch.zeros(n, dtype=torch.uint8, device=dev)
    ph = _Phases(phases)
    ph.mark("sample")
    _lib.call("wj_sample_walks", _lib.ptr(dg.idxptr), dg.idxptr_bytes, _lib.ptr(dg.indices), n, 0, n,
              M, L, seed64, _lib.ptr(walks), _lib.ptr(flags), s)
    del flags
    return store_from_walks(walks, n, M, L, seed64, id_map=getattr(g, "id_map", None), keep_keys=keep_keys,
                            ph=ph)


def store_from_walks(walks: torch.Tensor, n: int, M: int, L: int, seed64: int, id_map=None,
                     keep_keys: bool = False, ph=None) -> SubgraphStore:
    """Distinct landings + counts, global interning, virtual-landing index of
    a device walk table [n, M, L+1] int32 (sampler.py:117-151 after
    sampling); also the path of load_store."""
    dev = walks.device
    W = L + 1
    s = _lib.stream_handle(dev)
    ph = ph if ph is not None else _Phases(None)
    counts = torch.empty(n, dtype=torch.int32, device=dev)
    ph.mark("rpe_count")
    _lib.call("wj_rpe_count", _lib.ptr(walks), n, M, L, n, _lib.ptr(counts), s)
    offsets = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=offsets[1:])
    # one device -> host read for both sizes (the fill's allocation needs them)
    if n:
        total, max_unique = (int(v) for v in torch.stack([offsets[-1], counts.max().to(torch.int64)]).cpu())
    else:
        total, max_unique = 0, 0
    ux = torch.empty(total, dtype=torch.int32, device=dev)
    ukey = torch.empty(total, dtype=torch.int64, device=dev)
    ufirst = torch.empty(total, dtype=torch.int16, device=dev)
    slot = torch.empty((n, M * W), dtype=torch.int16, device=dev)
    ph.mark("rpe_fill")
    _lib.call("wj_rpe_fill", _lib.ptr(walks), n, M, L, n, _lib.ptr(offsets), _lib.ptr(ux),
              _lib.ptr(ukey), _lib.ptr(ufirst), _lib.ptr(slot), s)
    ph.mark("intern")
    uid, table_keys = intern_device(ukey, ufirst, offsets, n, 0, M, W)
    store = SubgraphStore(n, M, L, seed64, walks, offsets, ux, uid, ufirst, slot, table_keys,
                          max_unique, id_map=id_map)
    ph.mark("vindex")
    store.build_vindex()
    ph.mark("end")
    if keep_keys:
        store.uniq_key_d = ukey
    return store


# ------------------------------------------------------ typed / metapath walks
# SURVEY C4.  The reference has no typed sampler (SPEC.md:121-124 leaves it
# open); the semantics are defined in include/walkjoin_b200.h
# (wj_sample_walks_typed) so that metapath [-1] -- or a single edge type -- is
# exactly the reference sampler.

@dataclass
class TypedCSR:
    """Edge-type grouping of a device CSR (wj_typed_csr)."""

    num_types: int
    type_off: torch.Tensor       # [n*T + 1] int64
    typed_indices: torch.Tensor  # [2E] int32


def edge_types_from_node_types(g, node_types, num_node_types: int) -> np.ndarray:
    """Per-CSR-entry relation type of a heterogeneous graph: the edge from a
    type-a node to a type-b node gets type a*K + b (K = num_node_types), so a
    metapath is a sequence of (from, to) node-type pairs."""
    nt = np.asarray(node_types, dtype=np.int64)
    K = int(num_node_types)
    if nt.shape[0] != g.num_nodes or (nt.size and (nt.min() < 0 or nt.max() >= K)):
        raise ValueError("node_types must give a type in [0, num_node_types) for every node")
    if K * K > 64:
        raise ValueError("at most 8 node types (64 relation types)")
    idxptr = np.asarray(g.idxptr if not isinstance(g.idxptr, torch.Tensor) else g.idxptr.cpu().numpy(), np.int64)
    indices = np.asarray(g.indices if not isinstance(g.indices, torch.Tensor) else g.indices.cpu().numpy(), np.int64)
    rows = np.repeat(np.arange(g.num_nodes, dtype=np.int64), np.diff(idxptr))
    return (nt[rows] * K + nt[indices]).astype(np.uint8)


def typed_csr(g, edge_types, num_types: int = None, device=None) -> TypedCSR:
    """Group every node's neighbours by edge type on the device (stable)."""
    dev = _lib.require_cuda(device if device is not None else getattr(g, "device", None))
    dg = DeviceGraph.from_graph(g, dev)
    et = torch.as_tensor(np.asarray(edge_types, dtype=np.uint8) if not isinstance(edge_types, torch.Tensor)
                         else edge_types).to(dev, torch.uint8)
    if et.numel() != dg.indices.numel():
        raise ValueError(f"edge_types has {et.numel()} entries for {dg.indices.numel()} CSR entries")
    T = int(num_types) if num_types is not None else (int(et.max().item()) + 1 if et.numel() else 1)
    type_off = torch.empty(dg.num_nodes * T + 1, dtype=torch.int64, device=dev)
    if dg.num_nodes == 0:
        type_off.zero_()
    typed = torch.empty_like(dg.indices)
    _lib.call("wj_typed_csr", _lib.ptr(dg.idxptr), dg.idxptr_bytes, _lib.ptr(dg.indices), _lib.ptr(et),
              dg.num_nodes, T, _lib.ptr(type_off), _lib.ptr(typed), _lib.stream_handle(dev))
    return TypedCSR(T, type_off, typed)


def sample_walks_typed(g, tcsr: TypedCSR, metapath, num_walks: int, num_steps: int, seed: int,
                       lo: int = 0, hi: int = None, device=None) -> torch.Tensor:
    """Metapath walks of anchors [lo, hi) -> device int32 [hi-lo, M, L+1]."""
    if num_walks < 1 or num_steps < 1:
        raise ValueError("num_walks and num_steps must be >= 1")
    mp = np.ascontiguousarray(metapath, dtype=np.int8)
    if mp.ndim != 1 or not 1 <= mp.shape[0] <= 32:
        raise ValueError("metapath must be a sequence of 1..32 edge types (negative = any edge)")
    dev = _lib.require_cuda(device if device is not None else getattr(g, "device", None))
    dg = DeviceGraph.from_graph(g, dev)
    hi = dg.num_nodes if hi is None else int(hi)
    walks = torch.empty((hi - lo, num_walks, num_steps + 1), dtype=torch.int32, device=dev)
    T = 0 if tcsr is None else tcsr.num_types
    _lib.call("wj_sample_walks_typed", _lib.ptr(dg.idxptr), dg.idxptr_bytes, _lib.ptr(dg.indices),
              None if tcsr is None else _lib.ptr(tcsr.type_off),
              None if tcsr is None else _lib.ptr(tcsr.typed_indices), T, mp.ctypes.data, mp.shape[0],
              dg.num_nodes, int(lo), hi, int(num_walks), int(num_steps), _u64(seed), _lib.ptr(walks),
              _lib.stream_handle(dev))
    return walks


def preprocess_typed(g, edge_types, metapath, num_walks: int, num_steps: int, seed: int, num_types: int = None,
                     device=None, keep_keys: bool = False) -> SubgraphStore:
    """Alg. 1 with metapath walks: typed sampling, then the same RPE /
    interning / index phases as ``preprocess``; the store joins, encodes and
    exports like any other."""
    if g.num_nodes >= 2 ** 31:
        raise ValueError("graphs with >= 2^31 nodes are not supported")
    dev = _lib.require_cuda(device if device is not None else getattr(g, "device", None))
    mp = np.ascontiguousarray(metapath, dtype=np.int8)
    tcsr = typed_csr(g, edge_types, num_types, dev) if (mp >= 0).any() else None
    walks = sample_walks_typed(g, tcsr, mp, num_walks, num_steps, seed, device=dev)
    del tcsr
    return store_from_walks(walks, int(g.num_nodes), int(num_walks), int(num_steps), _u64(seed),
                            id_map=getattr(g, "id_map", None), keep_keys=keep_keys)
