"""numpy + ctypes glue of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Restates the host-side drivers of the reference around the C kernels in
``walkjoin_oracle.c``.  Citations are to ``/root/reference/pkg/src/walkjoin``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

_lib = None


def build_oracle() -> str:
    """Compile liboracle.so with the committed Makefile (gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build_oracle()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        U64 = ctypes.c_uint64
        I = ctypes.c_int
        L.wjo_node_stream_state.argtypes = [U64, I64]
        L.wjo_node_stream_state.restype = U64
        L.wjo_sample_node_walks.argtypes = [P, P, I64, I64, I64, U64, P]
        L.wjo_sample_node_walks.restype = U64
        L.wjo_sample_all_walks.argtypes = [P, P, I64, I64, I64, U64, P, I]
        L.wjo_sample_nodes.argtypes = [P, P, P, I64, I64, I64, U64, P, I]
        L.wjo_count_distinct_all.argtypes = [P, I64, I64, I64, P, I]
        L.wjo_fill_distinct_all.argtypes = [P, I64, I64, I64, P, I64, P, P, I]
        L.wjo_intern_rows.argtypes = [P, I64, I64, P, P]
        L.wjo_intern_rows.restype = I64
        L.wjo_build_dicts.argtypes = [P, P, P, P, I64, P, P, I]
        L.wjo_dict_get_one.argtypes = [P, P, P, I64, I64]
        L.wjo_dict_get_one.restype = ctypes.c_int32
        L.wjo_join_fill.argtypes = [P, I64, I64, P, P, P, P, I64, I64, P, P, I]
        L.wjo_densify.argtypes = [P, I64, P, I64, P, I]
        L.wjo_sample_typed.argtypes = [P, P, P, P, I64, I64, I64, I64, U64, P, I]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ---------------------------------------------------------------- sampler --

def node_stream_state(seed: int, u: int) -> int:
    """_kernels.py:47-50."""
    return int(lib().wjo_node_stream_state(int(seed) & _MASK64, int(u)))


def sample_walks(idxptr, indices, u, num_walks, num_steps, state):
    """sampler.py:61-76 (rng state in, (walks, end state) out)."""
    idxptr = np.ascontiguousarray(idxptr, np.int64)
    indices = np.ascontiguousarray(indices, np.int32)
    out = np.empty((num_walks, num_steps + 1), np.int32)
    end = lib().wjo_sample_node_walks(_p(idxptr), _p(indices), int(u), num_walks, num_steps,
                                      int(state) & _MASK64, _p(out))
    return out, int(end)


def sample_all_walks(idxptr, indices, num_walks, num_steps, seed, threads=None):
    """_kernels.py:69-74 over all nodes."""
    idxptr = np.ascontiguousarray(idxptr, np.int64)
    indices = np.ascontiguousarray(indices, np.int32)
    n = idxptr.shape[0] - 1
    walks = np.empty((n, num_walks, num_steps + 1), np.int32)
    lib().wjo_sample_all_walks(_p(idxptr), _p(indices), n, num_walks, num_steps,
                               int(seed) & _MASK64, _p(walks), threads or default_threads())
    return walks


def sample_nodes(idxptr, indices, nodes, num_walks, num_steps, seed, threads=None):
    """_kernels.py:69-74 for an explicit anchor list (rows in list order)."""
    idxptr = np.ascontiguousarray(idxptr, np.int64)
    indices = np.ascontiguousarray(indices, np.int32)
    nodes = np.ascontiguousarray(nodes, np.int64)
    walks = np.empty((nodes.shape[0], num_walks, num_steps + 1), np.int32)
    lib().wjo_sample_nodes(_p(idxptr), _p(indices), _p(nodes), nodes.shape[0], num_walks,
                           num_steps, int(seed) & _MASK64, _p(walks), threads or default_threads())
    return walks


def sample_typed_walks(idxptr, indices, edge_types, metapath, num_walks, num_steps, seed, threads=None):
    """Typed / metapath walks (our definition, no reference
    implementation -- see walkjoin_oracle.c wjo_sample_typed)."""
    idxptr = np.ascontiguousarray(idxptr, np.int64)
    indices = np.ascontiguousarray(indices, np.int32)
    et = np.ascontiguousarray(edge_types, np.uint8)
    mp = np.ascontiguousarray(metapath, np.int8)
    n = idxptr.shape[0] - 1
    walks = np.empty((n, num_walks, num_steps + 1), np.int32)
    lib().wjo_sample_typed(_p(idxptr), _p(indices), _p(et), _p(mp), mp.shape[0], n, num_walks, num_steps,
                           int(seed) & _MASK64, _p(walks), threads or default_threads())
    return walks


def store_from_walks(walks, seed=0, threads=None, timed=False):
    """sampler.py:117-151 on a given walk table (rows = anchors in order):
    distinct lists, interning, dicts.  Used to time preprocess on a shard and
    to build a batch's sub-store for the CPU baseline."""
    import time

    threads = threads or default_threads()
    L = lib()
    walks = np.ascontiguousarray(walks, np.int32)
    n, num_walks, width = walks.shape
    t = {}
    local_cap = 1
    while local_cap < 2 * num_walks * width:
        local_cap <<= 1
    t0 = time.perf_counter()
    counts = np.empty(n, np.int64)
    L.wjo_count_distinct_all(_p(walks), n, num_walks * width, local_cap, _p(counts), threads)
    item_offsets = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=item_offsets[1:])
    total = int(item_offsets[-1])
    t["count"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    nodes_flat = np.empty(total, np.int32)
    vecs = np.empty((total, width), np.int32)
    L.wjo_fill_distinct_all(_p(walks), n, num_walks, width, _p(item_offsets), local_cap,
                            _p(nodes_flat), _p(vecs), threads)
    t["fill"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    rpe_ids, table = intern_vectors(vecs)
    del vecs
    t["intern"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    caps = dict_capacities(counts)
    cap_offsets = np.zeros(n + 1, np.int64)
    np.cumsum(caps, out=cap_offsets[1:])
    dict_keys = np.full(int(cap_offsets[-1]), -1, np.int32)
    dict_vals = np.zeros(int(cap_offsets[-1]), np.int32)
    L.wjo_build_dicts(_p(nodes_flat), _p(rpe_ids), _p(item_offsets), _p(cap_offsets), n,
                      _p(dict_keys), _p(dict_vals), threads)
    t["dicts"] = time.perf_counter() - t0
    return OracleStore(n, num_walks, width - 1, int(seed) & _MASK64, walks, table, cap_offsets,
                       dict_keys, dict_vals, item_offsets, nodes_flat, rpe_ids,
                       phase_seconds=t if timed else None)


def compute_rpe(walks: np.ndarray) -> dict:
    """sampler.py:79-91: {x: int32[L+1]} in first-appearance order."""
    width = walks.shape[1]
    entries: dict[int, np.ndarray] = {}
    for row in walks:
        for i in range(width):
            x = int(row[i])
            vec = entries.get(x)
            if vec is None:
                vec = np.zeros(width, np.int32)
                entries[x] = vec
            vec[i] += 1
    return entries


# ------------------------------------------------------------------ store --

def intern_vectors(vecs: np.ndarray):
    """store.py:107-121 -> (ids 1-based, table with zero row)."""
    vecs = np.ascontiguousarray(vecs, np.int32)
    total, width = vecs.shape
    ids = np.empty(total, np.int32)
    reps = np.empty(max(total, 1), np.int64)
    n_unique = lib().wjo_intern_rows(_p(vecs), total, width, _p(ids), _p(reps)) if total else 0
    table = np.zeros((n_unique + 1, width), np.int32)
    if n_unique:
        table[1:] = vecs[reps[:n_unique]]
    return ids + 1, table


def dict_capacities(counts: np.ndarray) -> np.ndarray:
    """store.py:124-131: smallest power of two >= max(2, 2*count)."""
    need = np.maximum(2 * np.asarray(counts, np.int64), 2)
    caps = np.int64(1) << np.ceil(np.log2(need)).astype(np.int64)
    caps[caps < need] <<= 1
    shrink = (caps >> 1) >= need
    caps[shrink] >>= 1
    return caps


def dedup_and_reindex(raw_maps):
    """store.py:134-157."""
    vec_rows, node_lists = [], []
    for entries in raw_maps:
        nodes = list(entries.keys())
        node_lists.append(nodes)
        vec_rows.extend(np.asarray(entries[x], np.int32) for x in nodes)
    ids, table = intern_vectors(np.array(vec_rows, np.int32))
    dicts, pos = [], 0
    for nodes in node_lists:
        dicts.append({int(x): int(ids[pos + i]) for i, x in enumerate(nodes)})
        pos += len(nodes)
    return table, dicts


@dataclass
class OracleStore:
    """Flat arrays of the reference SubgraphStore (store.py:58-71) plus the
    intermediate per-anchor distinct lists the GPU store is checked against."""

    num_nodes: int
    num_walks: int
    walk_steps: int
    seed: int
    walks: np.ndarray         # [n, M, L+1] int32
    table: np.ndarray         # [T, L+1] int32, row 0 zero
    dict_offsets: np.ndarray  # [n+1] int64
    dict_keys: np.ndarray     # int32, -1 empty
    dict_vals: np.ndarray     # int32
    item_offsets: np.ndarray  # [n+1] int64 (first-appearance lists)
    nodes_flat: np.ndarray    # [sum U] int32, first-appearance order
    rpe_ids_flat: np.ndarray  # [sum U] int32, 1-based ids aligned with nodes_flat
    phase_seconds: Optional[dict] = None

    def entry_dict(self, u: int) -> dict:
        lo, hi = self.dict_offsets[u], self.dict_offsets[u + 1]
        k, v = self.dict_keys[lo:hi], self.dict_vals[lo:hi]
        f = k != -1
        return {int(a): int(b) for a, b in zip(k[f], v[f])}


def preprocess(idxptr, indices, num_walks, num_steps, seed, threads=None, timed=False):
    """sampler.py:94-151 (Alg. 1): walks -> distinct lists -> intern -> dicts."""
    import time

    if num_walks < 1 or num_steps < 1:
        raise ValueError("num_walks and num_steps must be >= 1")
    threads = threads or default_threads()
    L = lib()
    idxptr = np.ascontiguousarray(idxptr, np.int64)
    indices = np.ascontiguousarray(indices, np.int32)
    n = idxptr.shape[0] - 1
    width = num_steps + 1
    seed64 = int(seed) & _MASK64
    t = {}
    t0 = time.perf_counter()
    walks = np.empty((n, num_walks, width), np.int32)
    L.wjo_sample_all_walks(_p(idxptr), _p(indices), n, num_walks, num_steps, seed64, _p(walks), threads)
    t["sample"] = time.perf_counter() - t0
    local_cap = 1
    while local_cap < 2 * num_walks * width:
        local_cap <<= 1
    t0 = time.perf_counter()
    counts = np.empty(n, np.int64)
    L.wjo_count_distinct_all(_p(walks), n, num_walks * width, local_cap, _p(counts), threads)
    item_offsets = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=item_offsets[1:])
    total = int(item_offsets[-1])
    t["count"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    nodes_flat = np.empty(total, np.int32)
    vecs = np.empty((total, width), np.int32)
    L.wjo_fill_distinct_all(_p(walks), n, num_walks, width, _p(item_offsets), local_cap,
                            _p(nodes_flat), _p(vecs), threads)
    t["fill"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    rpe_ids, table = intern_vectors(vecs)
    del vecs
    t["intern"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    caps = dict_capacities(counts)
    cap_offsets = np.zeros(n + 1, np.int64)
    np.cumsum(caps, out=cap_offsets[1:])
    dict_keys = np.full(int(cap_offsets[-1]), -1, np.int32)
    dict_vals = np.zeros(int(cap_offsets[-1]), np.int32)
    L.wjo_build_dicts(_p(nodes_flat), _p(rpe_ids), _p(item_offsets), _p(cap_offsets), n,
                      _p(dict_keys), _p(dict_vals), threads)
    t["dicts"] = time.perf_counter() - t0
    return OracleStore(n, num_walks, num_steps, seed64, walks, table, cap_offsets, dict_keys,
                       dict_vals, item_offsets, nodes_flat, rpe_ids,
                       phase_seconds=t if timed else None)


def get_rpe_id(store: OracleStore, u: int, x: int) -> int:
    """store.py:160-164."""
    if not 0 <= u < store.num_nodes:
        raise ValueError(f"node id {u} out of range [0, {store.num_nodes})")
    return int(lib().wjo_dict_get_one(_p(store.dict_keys), _p(store.dict_vals),
                                      _p(store.dict_offsets), int(u), int(x)))


# ----------------------------------------------------------------- joiner --

def join_batch_arrays(store: OracleStore, query_array, threads=None):
    """joiner.py:53-71 -> (walk_nodes [B,A*M,L+1], rpe_ids [B,A*M*(L+1),A])."""
    q = np.ascontiguousarray(query_array, np.int64)
    B, A = q.shape
    M, W = store.num_walks, store.walk_steps + 1
    walk_nodes = np.empty((B, A * M, W), np.int32)
    rpe_ids = np.empty((B, A * M * W, A), np.int32)
    if B:
        lib().wjo_join_fill(_p(store.walks), M, W, _p(store.dict_keys), _p(store.dict_vals),
                            _p(store.dict_offsets), _p(q), B, A, _p(walk_nodes), _p(rpe_ids),
                            threads or default_threads())
    return walk_nodes, rpe_ids


def gather_rpe(table: np.ndarray, rpe_ids: np.ndarray) -> np.ndarray:
    """joiner.py:96-104 for one joined query."""
    if rpe_ids.size and (rpe_ids.min() < 0 or rpe_ids.max() >= len(table)):
        raise ValueError(f"rpe id out of range for table of size {len(table)} (corrupt store?)")
    n_rows, arity = rpe_ids.shape
    return table[rpe_ids].reshape(n_rows, arity * table.shape[1]).astype(np.float64)


def dense_batch(store: OracleStore, query_array, threads=None, features=None):
    """pipeline.py:169-182 (_dense_batch): join, then table[rpe_ids] as float64."""
    walk_nodes, rpe_ids = join_batch_arrays(store, query_array, threads)
    B, rows, A = rpe_ids.shape
    W = store.walk_steps + 1
    dense = np.empty((B, rows, A * W), np.float64)
    ids = np.ascontiguousarray(rpe_ids.reshape(-1))
    if ids.size:
        lib().wjo_densify(_p(np.ascontiguousarray(store.table, np.int32)), W, _p(ids), ids.size,
                          _p(dense), threads or default_threads())
    if features is not None:
        flat = walk_nodes.reshape(B, rows)
        dense = np.concatenate([dense, features[flat]], axis=2)
    return dense


SURL_MAGIC, SURL_VERSION = b"SURL", 1


def write_surl(store: OracleStore, id_map=None) -> bytes:
    """Restatement of store._write_store (store.py:167-193): magic, the
    little-endian header <IIIQQQQ (version, M, L, seed, n, |table|, |id_map|),
    the table, then per node: capacity (u32), walks[u], dict_keys, dict_vals,
    and finally the original ids (int64, dense order) when there is an id_map."""
    import struct

    n = store.num_nodes
    id_len = n if id_map is not None else 0
    parts = [SURL_MAGIC, struct.pack("<IIIQQQQ", SURL_VERSION, store.num_walks, store.walk_steps,
                                     store.seed & _MASK64, n, store.table.shape[0], id_len),
             np.ascontiguousarray(store.table, np.int32).tobytes()]
    caps = np.diff(store.dict_offsets)
    for u in range(n):
        lo, hi = store.dict_offsets[u], store.dict_offsets[u + 1]
        parts += [struct.pack("<I", int(caps[u])), store.walks[u].tobytes(),
                  store.dict_keys[lo:hi].tobytes(), store.dict_vals[lo:hi].tobytes()]
    if id_len:
        origs = np.empty(n, np.int64)
        for orig, dense in id_map.items():
            origs[dense] = orig
        parts.append(origs.tobytes())
    return b"".join(parts)
