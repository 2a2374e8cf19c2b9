"""Query-level join of per-node walk sets on the B200 (reference joiner.py).

Host in -> host out, device in -> device out: numpy query arrays get numpy
results exactly like the reference (``join_batch_arrays`` returns int32
``walk_nodes`` [B, A*M, L+1] and ``rpe_ids`` [B, A*M*(L+1), A]); CUDA tensors
stay on the device.  ``dense_batch`` is the reference ``pipeline._dense_batch``
(pipeline.py:169-182): the join kernel writes ``table[rpe_id]`` straight into
the encoder's input buffer (float64 for host callers, any of fp32 / bf16 /
fp16 / fp64 on the device).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence, Union

import numpy as np
import torch

from . import _lib
from .graph import Query
from .store import RpeTable, SubgraphStore

QueryLike = Union[Query, Sequence[int]]


@dataclass
class JoinedQuery:
    """Per-query tensor pair fed to the encoder (joiner.py:24-30)."""

    query: tuple
    walk_nodes: np.ndarray
    rpe_ids: np.ndarray


def _query_nodes(q: QueryLike) -> tuple:
    nodes = q.nodes if hasattr(q, "nodes") else tuple(int(v) for v in q)
    if len(nodes) < 1:
        raise ValueError("query needs at least one node")
    return nodes


def _as_query_array(store: SubgraphStore, queries) -> np.ndarray:
    """Uniform arity + id range check (joiner.py:40-50)."""
    rows = [_query_nodes(q) for q in queries]
    arity = len(rows[0])
    for i, r in enumerate(rows):
        if len(r) != arity:
            raise ValueError(f"mixed query arity in batch: query 0 has {arity} nodes, query {i} has {len(r)}")
    arr = np.asarray(rows, dtype=np.int64)
    _check_range(store, arr)
    return arr


def _check_range(store: SubgraphStore, arr: np.ndarray):
    if arr.size and (arr.min() < 0 or arr.max() >= store.num_nodes):
        bad = arr[(arr < 0) | (arr >= store.num_nodes)][0]
        raise ValueError(f"query node id {bad} out of range [0, {store.num_nodes})")


def _to_device_queries(store: SubgraphStore, query_array, validate: bool):
    if isinstance(query_array, torch.Tensor):
        q = query_array.to(store.device, torch.int64).contiguous()
        if validate and q.numel():
            lo, hi = int(q.min().item()), int(q.max().item())
            if lo < 0 or hi >= store.num_nodes:
                raise ValueError(f"query node id out of range [0, {store.num_nodes})")
        return q, False
    arr = np.ascontiguousarray(np.asarray(query_array, dtype=np.int64))
    if arr.ndim != 2:
        raise ValueError("query_array must be [B, arity]")
    _check_range(store, arr)  # host arrays are always checked (an OOB id would fault)
    return torch.from_numpy(arr).to(store.device), True


def join_device(store: SubgraphStore, q: torch.Tensor, walk_nodes: Optional[torch.Tensor] = None,
                rpe_ids: Optional[torch.Tensor] = None, dense: Optional[torch.Tensor] = None,
                row_stride: Optional[int] = None):
    """Launch wj_join on preallocated device buffers (any may be None)."""
    B, A = q.shape
    if dense is not None:
        if dense.dtype not in _lib.DTYPE_CODES:
            raise ValueError(f"unsupported dense dtype {dense.dtype}")
        code = _lib.DTYPE_CODES[dense.dtype]
        stride = row_stride if row_stride is not None else dense.shape[-1]
    else:
        code, stride = 0, A * store.width
    _lib.call("wj_join", _lib.ptr(q), B, A, _lib.ptr(store.walks_d), _lib.ptr(store.offsets_d),
              _lib.ptr(store.uniq_x_d), _lib.ptr(store.uniq_id_d), _lib.ptr(store.slot_idx_d),
              store.num_walks, store.walk_steps, store.max_unique, _lib.ptr(store.table_keys_d),
              int(store.table_keys_d.numel()), _lib.ptr(walk_nodes), _lib.ptr(rpe_ids),
              _lib.ptr(dense), code, stride, _lib.stream_handle(store.device))


def join_batch_arrays(store: SubgraphStore, query_array, threads: int = 1, validate: bool = True):
    """Join a [B, arity] id array into walk_nodes / rpe_ids (joiner.py:53-71)."""
    q, host = _to_device_queries(store, query_array, validate)
    B, A = q.shape
    M, W = store.num_walks, store.width
    wn = torch.empty((B, A * M, W), dtype=torch.int32, device=store.device)
    ri = torch.empty((B, A * M * W, A), dtype=torch.int32, device=store.device)
    join_device(store, q, walk_nodes=wn, rpe_ids=ri)
    if host:
        return wn.cpu().numpy(), ri.cpu().numpy()
    return wn, ri


def join_query(store: SubgraphStore, q: QueryLike) -> JoinedQuery:
    """joiner.py:74-79."""
    nodes = _query_nodes(q)
    arr = _as_query_array(store, [nodes])
    wn, ri = join_batch_arrays(store, arr)
    return JoinedQuery(query=nodes, walk_nodes=wn[0], rpe_ids=ri[0])


def join_batch(store: SubgraphStore, queries, threads: int = 1) -> list:
    """joiner.py:82-93."""
    if not queries:
        return []
    arr = _as_query_array(store, queries)
    wn, ri = join_batch_arrays(store, arr, threads=threads)
    return [JoinedQuery(query=tuple(int(v) for v in arr[b]), walk_nodes=wn[b], rpe_ids=ri[b])
            for b in range(arr.shape[0])]


def gather_rpe(table, jq, device=None):
    """Densify a joined query with the wj_gather_rpe kernel (joiner.py:96-104).

    ``table`` is an RpeTable (or [T, L+1] array / tensor); ``jq`` a
    JoinedQuery or an rpe_ids array.  Returns float64 numpy for host inputs."""
    ids = jq.rpe_ids if hasattr(jq, "rpe_ids") else jq
    vec = table.vectors if hasattr(table, "vectors") else table
    host = not isinstance(ids, torch.Tensor)
    dev = _lib.require_cuda(device if device is not None else (None if host else ids.device))
    ids_d = torch.as_tensor(np.asarray(ids, dtype=np.int32) if host else ids).to(dev, torch.int32).contiguous()
    tab_d = torch.as_tensor(vec).to(dev, torch.int32).contiguous()
    n_rows, arity = ids_d.shape
    width = tab_d.shape[1]
    out = torch.empty((n_rows, arity * width), dtype=torch.float64, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("wj_gather_rpe", _lib.ptr(ids_d), ids_d.numel(), _lib.ptr(tab_d), tab_d.shape[0], width,
              _lib.ptr(out), _lib.DTYPE_CODES[torch.float64], _lib.ptr(bad), _lib.stream_handle(dev))
    if int(bad.item()):
        raise ValueError(f"rpe id out of range for table of size {tab_d.shape[0]} (corrupt store?)")
    return out.cpu().numpy() if host else out


def dense_batch(store: SubgraphStore, query_array, threads: int = 1, features=None,
                dtype=None, out: Optional[torch.Tensor] = None, validate: bool = True):
    """Reference ``pipeline._dense_batch`` (pipeline.py:169-182): join and
    densify in one kernel -> [B, A*M*(L+1), A*(L+1) (+ d)].

    Host query arrays return float64 numpy (reference dtype); device tensors
    return a device tensor of ``dtype`` (default float32), written into
    ``out`` when given (so a captured training step reuses one buffer)."""
    q, host = _to_device_queries(store, query_array, validate)
    B, A = q.shape
    rows, w = A * store.landings, A * store.width
    d = 0 if features is None else int(features.shape[1])
    dt = torch.float64 if host else (dtype or torch.float32)
    if out is None:
        out = torch.empty((B, rows, w + d), dtype=dt, device=store.device)
    wn = None
    if features is not None:
        wn = torch.empty((B, A * store.num_walks, store.width), dtype=torch.int32, device=store.device)
    join_device(store, q, walk_nodes=wn, dense=out, row_stride=w + d)
    if features is not None:
        feats = torch.as_tensor(features).to(store.device, out.dtype)
        out[:, :, w:] = feats[wn.reshape(B, rows).long()]
    return out.cpu().numpy() if host else out
