"""Graph types: the host CSR the reference API takes, and its HBM twin.

``Graph`` mirrors the reference type (/root/reference/pkg/src/walkjoin/
graph.py:49-119): immutable, undirected, simple, CSR with int64 ``idxptr``
and int32 per-node-sorted ``indices``.  ``preprocess`` also accepts the
reference's own Graph (anything with num_nodes / idxptr / indices / id_map).

``DeviceGraph`` is the CSR resident in HBM that the sampler kernel reads:
int32 ``idxptr`` whenever 2E < 2^31 (every configured shape; halves the
L2-resident offset array) and int32 ``indices``.

``synthetic_link_graph`` builds the benchmark inputs on the device: an
Erdos-Renyi graph of a named shape (the reference builds the same family as
``generate_sbm(1, n, p, 0)``, graph.py:298-354) and the 5% link split of
``split_link_queries`` (graph.py:239-280), with the training positives
removed from the walk graph.
"""

from __future__ import annotations

import itertools
import logging
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

import warnings

import numpy as np
import torch

logger = logging.getLogger(__name__)


class GraphFormatError(ValueError):
    """Malformed edge-list / hyperedge / query input (graph.py:24-25)."""


@dataclass(frozen=True)
class Query:
    """An ordered node set to score (graph.py:28-46)."""

    nodes: tuple
    label: Optional[int] = None

    def __post_init__(self):
        nodes = tuple(int(v) for v in self.nodes)
        object.__setattr__(self, "nodes", nodes)
        if len(nodes) < 1:
            raise ValueError("query needs at least one node")
        if len(set(nodes)) != len(nodes):
            raise ValueError(f"duplicate nodes in query {nodes}")
        if self.label is not None and self.label not in (0, 1):
            raise ValueError(f"query label must be 0 or 1, got {self.label}")

    def __len__(self) -> int:
        return len(self.nodes)


@dataclass(frozen=True)
class Graph:
    """Immutable undirected CSR graph (graph.py:49-119)."""

    num_nodes: int
    idxptr: np.ndarray
    indices: np.ndarray
    node_features: Optional[np.ndarray] = None
    id_map: Optional[dict] = None

    def __post_init__(self):
        self.idxptr.setflags(write=False)
        self.indices.setflags(write=False)

    @classmethod
    def from_edges(cls, pairs, num_nodes: int, node_features=None, id_map=None) -> "Graph":
        """Drop self-loops and duplicates, symmetrise, sort (graph.py:65-98)."""
        pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
        if pairs.size and (pairs.min() < 0 or pairs.max() >= num_nodes):
            raise ValueError("edge endpoint out of range")
        n = int(num_nodes)
        pairs = pairs[pairs[:, 0] != pairs[:, 1]]
        lo = np.minimum(pairs[:, 0], pairs[:, 1])
        hi = np.maximum(pairs[:, 0], pairs[:, 1])
        canon = np.unique(lo * n + hi)
        lo, hi = canon // n, canon % n
        key = np.concatenate([lo * n + hi, hi * n + lo])
        key.sort()
        idxptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(key // n, minlength=n), out=idxptr[1:])
        return cls(n, idxptr, (key % n).astype(np.int32), node_features, id_map)

    @property
    def num_edges(self) -> int:
        return self.indices.shape[0] // 2

    def degree(self, u: int) -> int:
        return int(self.idxptr[u + 1] - self.idxptr[u])

    def neighbors(self, u: int) -> np.ndarray:
        return self.indices[self.idxptr[u]: self.idxptr[u + 1]]

    def has_edge(self, u: int, v: int) -> bool:
        row = self.neighbors(u)
        i = np.searchsorted(row, v)
        return bool(i < row.shape[0] and row[i] == v)

    def edge_array(self) -> np.ndarray:
        src = np.repeat(np.arange(self.num_nodes, dtype=np.int64), np.diff(self.idxptr))
        keep = src < self.indices
        return np.column_stack([src[keep], self.indices[keep].astype(np.int64)])


def _strip(line: str) -> str:
    return line.split("#", 1)[0].strip()


def _parse_int(tok: str, lineno: int) -> int:
    try:
        v = int(tok)
    except ValueError:
        raise GraphFormatError(f"line {lineno}: expected integer, got {tok!r}") from None
    if v < 0:
        raise GraphFormatError(f"line {lineno}: node ids must be non-negative, got {v}")
    return v


def load_edge_list(lines: Iterable[str], undirected: bool = True) -> Graph:
    """``u v`` per line, '#' comments, dense remap by first appearance
    (graph.py:149-179).  ``undirected=False``: the input must already list
    both directions of every edge (validated, GraphFormatError otherwise)."""
    id_map: dict = {}
    pairs = []
    for lineno, raw in enumerate(lines, 1):
        line = _strip(raw)
        if not line:
            continue
        toks = line.split()
        if len(toks) != 2:
            raise GraphFormatError(f"line {lineno}: expected 'u v', got {raw.strip()!r}")
        u, v = (_parse_int(t, lineno) for t in toks)
        for o in (u, v):
            if o not in id_map:
                id_map[o] = len(id_map)
        pairs.append((id_map[u], id_map[v]))
    if not id_map:
        raise GraphFormatError("empty edge list")
    arr = np.array(pairs, np.int64)
    if not undirected:
        fwd = set(map(tuple, arr.tolist()))
        missing = [e for e in fwd if (e[1], e[0]) not in fwd and e[0] != e[1]]
        if missing:
            raise GraphFormatError(f"directed input is not symmetric, e.g. edge {missing[0]}")
    return Graph.from_edges(arr, len(id_map), id_map=id_map)


def project_hyperedges(lines: Iterable[str]) -> Graph:
    """Clique projection of hyperedges (graph.py:182-206)."""
    id_map: dict = {}
    pairs = []
    for lineno, raw in enumerate(lines, 1):
        line = _strip(raw)
        if not line:
            continue
        members = []
        for tok in line.split():
            o = _parse_int(tok, lineno)
            if o not in id_map:
                id_map[o] = len(id_map)
            if id_map[o] not in members:
                members.append(id_map[o])
        if len(members) < 2:
            raise GraphFormatError(f"line {lineno}: hyperedge needs at least 2 distinct nodes")
        pairs.extend(itertools.combinations(members, 2))
    if not pairs:
        raise GraphFormatError("empty hyperedge list")
    return Graph.from_edges(np.array(pairs, np.int64), len(id_map), id_map=id_map)


# ----------------------------------------------------------------- device --

_UPLOAD_MIN = 16 << 20  # below this a plain copy is as fast


def upload(arr: np.ndarray, device) -> torch.Tensor:
    """Contiguous host array -> new device tensor.  Large arrays go through
    wj_upload (several host threads staging through pinned buffers, ~4x the
    driver's single-threaded pageable copy); the call returns with the data
    on the device."""
    import os

    from . import _lib

    arr = np.ascontiguousarray(arr)
    device = torch.device(device)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)  # non-writable numpy view: only read
        src = torch.from_numpy(arr)
    if device.type != "cuda" or arr.nbytes < _UPLOAD_MIN:
        return src.to(device)
    out = torch.empty(arr.shape, dtype=src.dtype, device=device)
    with torch.cuda.device(device):
        # the new block may have been freed by work still queued on this
        # stream; wj_upload writes from its own streams
        torch.cuda.current_stream(device).synchronize()
        # 8 staging threads, or 2 while a background batch-planner build runs
        # (it is host-core / DRAM bound: at C3, t_pre 145-152 ms with 8 upload
        # threads vs 119-126 ms with 2); WJ_UPLOAD_THREADS overrides
        from .pipeline import planner_builds_in_flight

        env = os.environ.get("WJ_UPLOAD_THREADS")
        threads = int(env) if env else (2 if planner_builds_in_flight() else max(1, min(8, (os.cpu_count() or 2) // 2)))
        _lib.call("wj_upload", out.data_ptr(), arr.ctypes.data, arr.nbytes, threads)
    return out


class DeviceGraph:
    """CSR resident in HBM: int32 idxptr when 2E < 2^31, int32 indices."""

    def __init__(self, num_nodes: int, idxptr: torch.Tensor, indices: torch.Tensor, id_map=None):
        self.num_nodes = int(num_nodes)
        self.idxptr = idxptr
        self.indices = indices
        self.id_map = id_map
        self.device = idxptr.device

    @property
    def idxptr_bytes(self) -> int:
        return self.idxptr.element_size()

    @classmethod
    def from_graph(cls, g, device) -> "DeviceGraph":
        if isinstance(g, DeviceGraph):
            return g
        n = int(g.num_nodes)
        if n >= 2 ** 31:
            raise ValueError("graphs with >= 2^31 nodes are not supported")
        idxptr = np.asarray(g.idxptr)
        small = idxptr.shape[0] == 0 or int(idxptr[-1]) < 2 ** 31
        ip = np.ascontiguousarray(idxptr, dtype=np.int32 if small else np.int64)
        # no host-side copy of the (large) indices array when it is already
        # contiguous int32; read-only arrays are fine for the H2D copy
        ix = np.ascontiguousarray(np.asarray(g.indices), dtype=np.int32)
        return cls(n, upload(ip, device), upload(ix, device), getattr(g, "id_map", None))

    def to_host(self) -> Graph:
        return Graph(self.num_nodes, self.idxptr.cpu().numpy().astype(np.int64),
                     self.indices.cpu().numpy(), None, self.id_map)


def _csr_from_canonical(lo: torch.Tensor, hi: torch.Tensor, n: int):
    """Symmetrised CSR from canonical lo < hi edge keys (device sort)."""
    key = torch.cat([lo * n + hi, hi * n + lo])
    key, _ = torch.sort(key)
    src = torch.div(key, n, rounding_mode="floor")
    counts = torch.bincount(src, minlength=n)
    idxptr = torch.zeros(n + 1, dtype=torch.int64, device=key.device)
    torch.cumsum(counts, 0, out=idxptr[1:])
    indices = (key - src * n).to(torch.int32)
    if key.numel() < 2 ** 31:
        idxptr = idxptr.to(torch.int32)
    return idxptr, indices


@dataclass
class LinkSplit:
    """Benchmark split: walk graph without the training edges + positives."""

    walk_graph: DeviceGraph
    train_pos: np.ndarray   # [P, 2] int64 (host; the mini-batcher runs on host)
    all_edges: np.ndarray   # sorted canonical keys lo*n+hi of every edge (negative filter)
    num_nodes: int


def synthetic_link_graph(n: int, m: int, train_frac: float, seed: int, device) -> LinkSplit:
    """ER graph with n nodes / m undirected edges and a ``train_frac`` link
    split, built on the device (deterministic for a given seed and device
    type).  Mirrors the inputs of SURVEY §8(d): generate_sbm(1, n, p, 0) +
    split_link_queries(g, 0.05, ...)."""
    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed))
    pairs = int(m * 1.02) + 1024
    keys = torch.empty(0, dtype=torch.int64, device=dev)
    while keys.numel() < m:
        a = torch.randint(0, n, (pairs,), device=dev, generator=gen)
        b = torch.randint(0, n, (pairs,), device=dev, generator=gen)
        ok = a != b
        lo = torch.minimum(a[ok], b[ok])
        hi = torch.maximum(a[ok], b[ok])
        keys = torch.unique(torch.cat([keys, lo * n + hi]))
    keys = keys[torch.randperm(keys.numel(), device=dev, generator=gen)[:m]]
    perm = torch.randperm(m, device=dev, generator=gen)
    n_train = min(max(int(round(train_frac * m)), 1), m - 1)
    train = keys[perm[:n_train]]
    rest = keys[perm[n_train:]]
    all_sorted, _ = torch.sort(keys)
    lo = torch.div(rest, n, rounding_mode="floor")
    idxptr, indices = _csr_from_canonical(lo, rest - lo * n, n)
    tlo = torch.div(train, n, rounding_mode="floor")
    train_pos = torch.stack([tlo, train - tlo * n], 1).cpu().numpy()
    return LinkSplit(DeviceGraph(n, idxptr, indices), train_pos, all_sorted.cpu().numpy(), n)
