"""HBM-resident subgraph store with the reference SubgraphStore surface.

Reference: /root/reference/pkg/src/walkjoin/store.py.  The reference store
is walks + a global table of deduplicated count vectors + one open-addressing
dict per node (store.py:58-104).  The device store keeps, per anchor u,

* ``walks``      [n, M, L+1] int32          -- the walk table (store.walks)
* ``offsets``    [n+1] int64                -- entries of u at [off[u], off[u+1])
* ``uniq_x``     [E] int32, sorted per anchor -- distinct landings (V_u)
* ``uniq_id``    [E] int32                  -- global RPE id of (u, x)
* ``uniq_first`` [E] uint16                 -- first-appearance flat slot
* ``slot_idx``   [n, M*(L+1)] uint16         -- per walk slot, index into u's list
* ``table_keys`` [T] int64 (u64 bits)        -- packed count vector of each id

which replaces the hash dicts by a compact sorted index (the join binary
searches it in shared memory).  The reference's host arrays (``walks``,
``table``, ``dict_offsets`` / ``dict_keys`` / ``dict_vals``) are materialised
lazily and bit-exactly on first access -- the dicts by the wj_export_dicts
kernel -- so code written against the reference store runs unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib


class StoreFormatError(RuntimeError):
    """Wrong magic / version / length in a store file (store.py:29-30)."""


@dataclass
class RpeTable:
    """Deduplicated positional count vectors; row 0 is the zero sentinel (store.py:33-46)."""

    vectors: np.ndarray  # [T, L+1] int32

    def __post_init__(self):
        self.vectors.setflags(write=False)

    def __len__(self) -> int:
        return self.vectors.shape[0]

    def __getitem__(self, idx):
        return self.vectors[idx]


@dataclass
class NodeEntry:
    """One node's walks and its node-id -> RPE-id dictionary (store.py:49-55)."""

    anchor: int
    walks: np.ndarray
    dict: dict


def dict_capacities(counts) -> np.ndarray:
    """Smallest power of two >= max(2, 2*count) per node (store.py:124-131)."""
    need = np.maximum(2 * np.asarray(counts, dtype=np.int64), 2)
    caps = np.int64(1) << np.ceil(np.log2(need)).astype(np.int64)
    caps[caps < need] <<= 1
    shrink = (caps >> 1) >= need
    caps[shrink] >>= 1
    return caps


def count_bits(num_walks: int) -> int:
    return max(1, int(num_walks).bit_length())


def unpack_table(table_keys: torch.Tensor, num_walks: int, width: int) -> torch.Tensor:
    """[T] packed vectors -> [T, width] int32 counts (field c at bits c*cb)."""
    cb = count_bits(num_walks)
    shifts = torch.arange(width, device=table_keys.device, dtype=torch.int64) * cb
    return ((table_keys[:, None] >> shifts[None, :]) & ((1 << cb) - 1)).to(torch.int32)


class SubgraphStore:
    """Device store; attribute surface of the reference SubgraphStore."""

    def __init__(self, num_nodes, num_walks, walk_steps, seed, walks_d, offsets_d, uniq_x_d,
                 uniq_id_d, uniq_first_d, slot_idx_d, table_keys_d, max_unique, id_map=None,
                 anchor_counts=None):
        self.num_nodes = int(num_nodes)
        self.num_walks = int(num_walks)
        self.walk_steps = int(walk_steps)
        self.seed = int(seed)
        self.id_map = id_map
        self.walks_d = walks_d
        self.offsets_d = offsets_d
        self.uniq_x_d = uniq_x_d
        self.uniq_id_d = uniq_id_d
        self.uniq_first_d = uniq_first_d
        self.slot_idx_d = slot_idx_d
        self.table_keys_d = table_keys_d
        self.max_unique = int(max_unique)
        self.device = walks_d.device
        self._anchor_counts = anchor_counts
        self._cache: dict = {}
        self.voff_d = self.vcnt_d = self.vslots_d = self.trow_d = None

    # ------------------------------------------- encoder input layout --
    def build_vindex(self) -> None:
        """Virtual-landing index (voff / vcnt / vslots) and fp16 table rows
        that the tensor-core wj_join_encode reads (csrc/vindex.cu).  Built
        once, right after interning; shapes outside that kernel's envelope
        (L+1 > 8, M > 2048, M*(L+1) > 65535) get none and use the SIMT kernel."""
        n, M, W = self.num_nodes, self.num_walks, self.width
        if W > 8 or M > 2048 or M * W > 65535:
            return
        dev = self.device
        s = _lib.stream_handle(dev)
        vcnt = torch.empty((n, 2), dtype=torch.int32, device=dev)
        _lib.call("wj_vindex_count", _lib.ptr(self.offsets_d), _lib.ptr(self.uniq_id_d), n,
                  _lib.ptr(self.table_keys_d), M, self.walk_steps, _lib.ptr(vcnt), s)
        voff = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        if n:
            torch.cumsum(vcnt.sum(1, dtype=torch.int64), 0, out=voff[1:])
        total = int(voff[-1].item())
        vslots = torch.empty(max(total, 1), dtype=torch.int16, device=dev)
        _lib.call("wj_vindex_fill", _lib.ptr(self.offsets_d), _lib.ptr(self.uniq_id_d), n,
                  _lib.ptr(self.table_keys_d), M, self.walk_steps, _lib.ptr(voff), _lib.ptr(vcnt),
                  _lib.ptr(vslots), s)
        T = int(self.table_keys_d.numel())
        trow = torch.empty((max(T, 1), 8), dtype=torch.int16, device=dev)
        _lib.call("wj_table_rows_f16", _lib.ptr(self.table_keys_d), T, M, self.walk_steps,
                  _lib.ptr(trow), s)
        self.voff_d, self.vcnt_d, self.vslots_d, self.trow_d = voff, vcnt, vslots, trow

    def vindex_ptrs(self) -> tuple:
        """(voff, vcnt, vslots, table_rows_f16) device pointers, or NULLs."""
        return tuple(_lib.ptr(t) for t in (self.voff_d, self.vcnt_d, self.vslots_d, self.trow_d))

    # ---------------------------------------------------------- shapes --
    @property
    def width(self) -> int:
        return self.walk_steps + 1

    @property
    def landings(self) -> int:
        return self.num_walks * self.width

    @property
    def walk_slot_count(self) -> int:
        return self.num_nodes * self.num_walks * (self.walk_steps + 1)

    @property
    def num_entries(self) -> int:
        return int(self.uniq_x_d.numel())

    # ------------------------------------------------ host materialisers --
    def _host(self, key, fn):
        if key not in self._cache:
            arr = fn()
            arr.setflags(write=False)
            self._cache[key] = arr
        return self._cache[key]

    @property
    def walks(self) -> np.ndarray:
        return self._host("walks", lambda: self.walks_d.cpu().numpy())

    @property
    def table_d(self) -> torch.Tensor:
        if "table_d" not in self._cache:
            self._cache["table_d"] = unpack_table(self.table_keys_d, self.num_walks, self.width)
        return self._cache["table_d"]

    @property
    def table(self) -> RpeTable:
        if "table" not in self._cache:
            self._cache["table"] = RpeTable(self.table_d.cpu().numpy())
        return self._cache["table"]

    def anchor_counts(self) -> torch.Tensor:
        if self._anchor_counts is None:
            self._anchor_counts = (self.offsets_d[1:] - self.offsets_d[:-1]).to(torch.int64)
        return self._anchor_counts

    def export_dicts_device(self):
        """The reference per-node dicts (store.py:124-131, _kernels.py:174-188)
        on the device: (cap_offsets host int64 [n+1], cap_offsets, keys, vals)."""
        counts = self.anchor_counts().cpu().numpy()
        caps = dict_capacities(counts)
        cap_offsets = np.zeros(self.num_nodes + 1, np.int64)
        np.cumsum(caps, out=cap_offsets[1:])
        dev = self.device
        cap_d = torch.from_numpy(cap_offsets).to(dev)
        keys = torch.full((int(cap_offsets[-1]),), -1, dtype=torch.int32, device=dev)
        vals = torch.zeros(int(cap_offsets[-1]), dtype=torch.int32, device=dev)
        _lib.call("wj_export_dicts", _lib.ptr(self.offsets_d), _lib.ptr(self.uniq_x_d),
                  _lib.ptr(self.uniq_id_d), _lib.ptr(self.uniq_first_d), _lib.ptr(self.slot_idx_d),
                  self.num_nodes, self.num_walks, self.walk_steps, _lib.ptr(cap_d), _lib.ptr(keys),
                  _lib.ptr(vals), _lib.stream_handle(dev))
        return cap_offsets, cap_d, keys, vals

    def _export_dicts(self):
        cap_offsets, _, keys, vals = self.export_dicts_device()
        for k, a in (("dict_offsets", cap_offsets), ("dict_keys", keys.cpu().numpy()),
                     ("dict_vals", vals.cpu().numpy())):
            a.setflags(write=False)
            self._cache[k] = a

    @property
    def dict_offsets(self) -> np.ndarray:
        if "dict_offsets" not in self._cache:
            self._export_dicts()
        return self._cache["dict_offsets"]

    @property
    def dict_keys(self) -> np.ndarray:
        if "dict_keys" not in self._cache:
            self._export_dicts()
        return self._cache["dict_keys"]

    @property
    def dict_vals(self) -> np.ndarray:
        if "dict_vals" not in self._cache:
            self._export_dicts()
        return self._cache["dict_vals"]

    def entry(self, u: int) -> NodeEntry:
        """Walks + {node: rpe id} of anchor u (store.py:81-91).  The dict is
        the anchor's reference hash dict, exported on device, iterated in
        slot order exactly like the reference."""
        self._check_node(u)
        if "dict_keys" in self._cache:
            lo, hi = self.dict_offsets[u], self.dict_offsets[u + 1]
            keys, vals = self.dict_keys[lo:hi], self.dict_vals[lo:hi]
        else:
            dev = self.device
            count = int((self.offsets_d[u + 1] - self.offsets_d[u]).item())
            cap = int(dict_capacities([count])[0])
            cap_d = torch.tensor([0, cap], dtype=torch.int64, device=dev)
            kd = torch.full((cap,), -1, dtype=torch.int32, device=dev)
            vd = torch.zeros(cap, dtype=torch.int32, device=dev)
            _lib.call("wj_export_dicts", self.offsets_d.data_ptr() + 8 * u,
                      _lib.ptr(self.uniq_x_d), _lib.ptr(self.uniq_id_d),
                      _lib.ptr(self.uniq_first_d), self.slot_idx_d.data_ptr() + 2 * u * self.landings,
                      1, self.num_walks, self.walk_steps, _lib.ptr(cap_d), _lib.ptr(kd),
                      _lib.ptr(vd), _lib.stream_handle(dev))
            keys, vals = kd.cpu().numpy(), vd.cpu().numpy()
        filled = keys != -1
        return NodeEntry(anchor=u, walks=self.walks_d[u].cpu().numpy(),
                         dict={int(k): int(v) for k, v in zip(keys[filled], vals[filled])})

    def byte_sizes(self) -> dict:
        """Reference-format sizes (store.py:93-100) plus the device index."""
        counts = self.anchor_counts().cpu().numpy()
        dict_slots = int(dict_capacities(counts).sum())
        sizes = {
            "walks": self.walk_slot_count * 4,
            "table": int(self.table_keys_d.numel()) * self.width * 4,
            "dicts": dict_slots * 8 + (self.num_nodes + 1) * 8,
        }
        sizes["total"] = sum(sizes.values())
        sizes["device_index"] = sum(int(t.numel()) * t.element_size() for t in (
            self.offsets_d, self.uniq_x_d, self.uniq_id_d, self.uniq_first_d, self.slot_idx_d,
            self.table_keys_d, self.voff_d, self.vcnt_d, self.vslots_d, self.trow_d) if t is not None)
        return sizes

    def _check_node(self, u: int):
        if not 0 <= u < self.num_nodes:
            raise ValueError(f"node id {u} out of range [0, {self.num_nodes})")


def get_rpe_id(store: SubgraphStore, u: int, x: int) -> int:
    """RPE id of x relative to anchor u, 0 if absent (store.py:160-164)."""
    store._check_node(u)
    dev = store.device
    ut = torch.tensor([int(u)], dtype=torch.int64, device=dev)
    xt = torch.tensor([int(x)], dtype=torch.int64, device=dev)
    out = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.call("wj_lookup", _lib.ptr(ut), _lib.ptr(xt), 1, _lib.ptr(store.offsets_d),
              _lib.ptr(store.uniq_x_d), _lib.ptr(store.uniq_id_d), _lib.ptr(out),
              _lib.stream_handle(dev))
    return int(out.item())


def _default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("walkjoin_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def intern_vectors_device(vecs: torch.Tensor):
    """Global interning of [R, W] int32 count vectors on the device
    (store.py:107-121, _kernels.py:137-171): ids 1-based in first-occurrence
    order of the rows, table [T, W] with the zero row prepended.  Returns
    device tensors (ids int32 [R], table int32 [T, W], reps int64 [T-1] =
    first row of each id).

    Rows whose counts pack into 63 bits (every store's vectors: W fields of
    bit_length(max) bits) go through the preprocess interning kernels
    (wj_intern_insert / wj_intern_assign), each row its own scan position;
    any other int32 rows (negative or very wide) are ranked with a device
    ``unique`` -- the same definition, first occurrence -> id."""
    from .sampler import intern_device

    vecs = vecs.to(torch.int32).contiguous()
    R, W = vecs.shape
    dev = vecs.device
    if R == 0:
        return (torch.empty(0, dtype=torch.int32, device=dev), torch.zeros((1, W), dtype=torch.int32, device=dev),
                torch.empty(0, dtype=torch.int64, device=dev))
    vmin, vmax = int(vecs.min()), int(vecs.max())
    cb = max(1, vmax.bit_length())
    if vmin >= 0 and W * cb <= 63 and R < (1 << 46):
        shifts = torch.arange(W, device=dev, dtype=torch.int64) * cb
        # the marker bit keeps an all-zero row distinct from the empty slot
        key = ((vecs.to(torch.int64) << shifts[None, :]).sum(1)) | (1 << 63)
        offsets = torch.arange(R + 1, dtype=torch.int64, device=dev)
        first = torch.zeros(R, dtype=torch.int16, device=dev)
        ids, keys_sorted, orders = intern_device(key, first, offsets, R, 0, None, W, return_order=True)
        reps = orders >> 16
    else:
        uniq, inv = torch.unique(vecs, dim=0, return_inverse=True)
        rows = torch.arange(R, dtype=torch.int64, device=dev)
        first = torch.full((uniq.shape[0],), R, dtype=torch.int64, device=dev)
        first.scatter_reduce_(0, inv, rows, reduce="amin")
        order = torch.argsort(first)
        rank = torch.empty_like(order)
        rank[order] = torch.arange(order.numel(), device=dev)
        ids = (rank[inv] + 1).to(torch.int32)
        reps = first[order]
    table = torch.zeros((reps.numel() + 1, W), dtype=torch.int32, device=dev)
    table[1:] = vecs[reps]
    return ids, table, reps


def intern_vectors(vecs) -> tuple:
    """store.py:107-121 on the device: (ids int32 1-based, table int32 with
    the zero row), host numpy in -> host numpy out like the reference."""
    on_host = not isinstance(vecs, torch.Tensor) or vecs.device.type == "cpu"
    v = torch.as_tensor(np.ascontiguousarray(vecs, dtype=np.int32) if not isinstance(vecs, torch.Tensor) else vecs)
    if v.dim() != 2:
        raise ValueError("intern_vectors expects a [rows, width] array")
    if v.device.type == "cpu":
        v = v.to(_default_device())
    ids, table, _ = intern_vectors_device(v)
    if on_host:
        return ids.cpu().numpy(), table.cpu().numpy()
    return ids, table


def dedup_and_reindex(raw_maps: Sequence):
    """store.py:134-157: the deduplicated table and per-node {x: id} dicts
    from raw per-node positional count maps (ascending node order, entries in
    their recorded first-appearance order); the interning runs on the
    device (``intern_vectors``)."""
    vec_rows, node_lists, width = [], [], None
    for raw in raw_maps:
        entries = raw.entries if hasattr(raw, "entries") else raw
        nodes = list(entries.keys())
        node_lists.append(nodes)
        for x in nodes:
            vec = np.asarray(entries[x], dtype=np.int32)
            if width is None:
                width = vec.shape[0]
            vec_rows.append(vec)
    if width is None:
        raise ValueError("no raw maps given")
    ids, table = intern_vectors(np.array(vec_rows, dtype=np.int32))
    dicts, pos = [], 0
    for nodes in node_lists:
        dicts.append({int(x): int(ids[pos + i]) for i, x in enumerate(nodes)})
        pos += len(nodes)
    return RpeTable(table), dicts


def get_rpe_ids(store: SubgraphStore, u: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """Batched device lookups (no range check on u beyond the caller's)."""
    u = u.to(store.device, torch.int64).contiguous()
    x = x.to(store.device, torch.int64).contiguous()
    out = torch.empty(u.shape, dtype=torch.int32, device=store.device)
    _lib.call("wj_lookup", _lib.ptr(u), _lib.ptr(x), u.numel(), _lib.ptr(store.offsets_d),
              _lib.ptr(store.uniq_x_d), _lib.ptr(store.uniq_id_d), _lib.ptr(out),
              _lib.stream_handle(store.device))
    return out


# ------------------------------------------------------- store file (SURL) --
_MAGIC = b"SURL"
_VERSION = 1
_HEADER = "<IIIQQQQ"


def save_store(store: SubgraphStore, path, chunk_bytes: int = 1 << 28) -> None:
    """Write the reference store file (store.py:167-201), byte-identical to
    walkjoin.save_store of the same store: header, table, then per node
    capacity, walks and the node's open-addressing dict, then the id map.
    The node records are packed on the device (wj_surl_pack) in chunks of
    about ``chunk_bytes``."""
    import struct

    n, M, L = store.num_nodes, store.num_walks, store.walk_steps
    MW = M * (L + 1)
    dev = store.device
    cap_offsets, cap_d, keys, vals = store.export_dicts_device()
    caps = np.diff(cap_offsets)
    rec_words = 1 + MW + 2 * caps
    id_len = n if store.id_map is not None else 0
    table = store.table.vectors
    s = _lib.stream_handle(dev)
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(struct.pack(_HEADER, _VERSION, M, L, store.seed & 0xFFFFFFFFFFFFFFFF, n, table.shape[0], id_len))
        fh.write(np.ascontiguousarray(table, np.int32).tobytes())
        u0 = 0
        cum = np.zeros(n + 1, np.int64)
        np.cumsum(rec_words, out=cum[1:])
        limit = max(chunk_bytes // 4, int(rec_words.max()) if n else 1)
        while u0 < n:
            u1 = int(np.searchsorted(cum, cum[u0] + limit, side="right")) - 1
            u1 = min(max(u1, u0 + 1), n)
            rec_off = torch.from_numpy(cum[u0:u1] - cum[u0]).to(dev)
            out = torch.empty(int(cum[u1] - cum[u0]), dtype=torch.int32, device=dev)
            _lib.call("wj_surl_pack", store.walks_d.data_ptr() + 4 * u0 * MW, u1 - u0, MW,
                      cap_d.data_ptr() + 8 * u0, _lib.ptr(keys), _lib.ptr(vals), _lib.ptr(rec_off),
                      _lib.ptr(out), s)
            fh.write(out.cpu().numpy().tobytes())
            u0 = u1
        if id_len:
            origs = np.empty(n, np.int64)
            for orig, dense in store.id_map.items():
                origs[dense] = orig
            fh.write(origs.tobytes())


def load_store(path, device=None) -> SubgraphStore:
    """Read a reference store file (store.py:204-264) into a device store.
    Magic, version and lengths are checked like the reference
    (StoreFormatError).  The walks are unpacked on the device and the index
    is rebuilt from them; the rebuilt RPE table and per-node dicts must equal
    the file's, else the file is inconsistent (StoreFormatError)."""
    import struct

    from .sampler import store_from_walks

    dev = _lib.require_cuda(device)
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:4] != _MAGIC:
        raise StoreFormatError(f"bad magic {data[:4]!r}, expected {_MAGIC!r}")
    header_size = 4 + struct.calcsize(_HEADER)
    if len(data) < header_size:
        raise StoreFormatError("truncated store file (header)")
    version, M, L, seed, n, table_len, id_len = struct.unpack_from(_HEADER, data, 4)
    if version != _VERSION:
        raise StoreFormatError(f"unsupported store version {version}, expected {_VERSION}")
    W = L + 1
    MW = M * W
    off = header_size
    tb = table_len * W * 4
    if off + tb > len(data):
        raise StoreFormatError("truncated store file")
    table = np.frombuffer(data, np.int32, table_len * W, off).reshape(table_len, W)
    off += tb
    rec0 = off
    caps = np.empty(n, np.int64)
    unpack = struct.Struct("<I").unpack_from
    size = len(data)
    for u in range(n):  # records are variable-length: one sequential scan of the capacities
        if off + 4 > size:
            raise StoreFormatError("truncated store file")
        cap = unpack(data, off)[0]
        caps[u] = cap
        off += 4 * (1 + MW + 2 * cap)
    if off > size:
        raise StoreFormatError("truncated store file")
    rec_end = off
    id_map = None
    if id_len:
        if off + 8 * id_len > size:
            raise StoreFormatError("truncated store file")
        origs = np.frombuffer(data, np.int64, id_len, off)
        id_map = {int(o): d for d, o in enumerate(origs)}
        off += 8 * id_len
    if off != size:
        raise StoreFormatError(f"store file has {size - off} trailing bytes")
    rec_words = 1 + MW + 2 * caps
    rec_off = np.zeros(n, np.int64)
    if n:
        np.cumsum(rec_words[:-1], out=rec_off[1:])
    cap_offsets = np.zeros(n + 1, np.int64)
    np.cumsum(caps, out=cap_offsets[1:])
    records = torch.from_numpy(np.frombuffer(data, np.int32, (rec_end - rec0) // 4, rec0).copy()).to(dev)
    walks = torch.empty((n, M, W), dtype=torch.int32, device=dev)
    keys = torch.empty(int(cap_offsets[-1]), dtype=torch.int32, device=dev)
    vals = torch.empty(int(cap_offsets[-1]), dtype=torch.int32, device=dev)
    cap_d = torch.from_numpy(cap_offsets).to(dev)
    _lib.call("wj_surl_unpack", _lib.ptr(records), n, MW, _lib.ptr(torch.from_numpy(rec_off).to(dev)),
              _lib.ptr(cap_d), _lib.ptr(walks), _lib.ptr(keys), _lib.ptr(vals), _lib.stream_handle(dev))
    del records
    store = store_from_walks(walks, n, M, L, int(seed), id_map=id_map)
    if store.table.vectors.shape != table.shape or not np.array_equal(store.table.vectors, table):
        raise StoreFormatError("store file table is not the one its walks produce")
    ref_caps, _, k2, v2 = store.export_dicts_device()
    if not (np.array_equal(ref_caps, cap_offsets) and torch.equal(k2, keys) and torch.equal(v2, vals)):
        raise StoreFormatError("store file dicts are not the ones its walks produce")
    return store
