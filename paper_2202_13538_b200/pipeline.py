"""Training orchestration around the device hot path (reference pipeline.py).

The batch plan (BFS mini-batches over query overlap + in-seed negatives,
pipeline.py:54-166) stays on the host: it is sequential and tiny.  Each
training step -- join+densify kernel, encoder forward, BCE, backward, Adam --
runs on the device and is captured once per batch shape as a CUDA graph, so a
step is one graph launch plus the H2D copy of the batch's query ids.
"""

from __future__ import annotations

import ctypes
import logging
import os
import threading
import time
from collections import deque
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from . import encoder as E
from .graph import Query
from .joiner import dense_batch
from .store import SubgraphStore

logger = logging.getLogger(__name__)

# largest unit of identical queries the join+encode kernel runs in one CTA
# (wj_group_queries; the planner's producer thread uses the same)
GROUP_MAX = 4


@dataclass
class TrainConfig:
    """pipeline.py:30-51 (same defaults)."""

    batch_capacity: int = 1500
    batch_size: int = 32
    k_neg: int = 50
    lr: float = 1e-3
    max_epochs: int = 50
    patience: int = 5
    seed: int = 0
    threads: int = 1
    hidden_dim: int = 64
    dropout: float = 0.1
    metric: str = "auc"
    use_features: bool = False

    def __post_init__(self):
        if self.batch_capacity < 1 or self.batch_size < 1 or self.k_neg < 1:
            raise ValueError("batch_capacity, batch_size, and k_neg must be >= 1")
        if self.metric not in ("auc", "mrr"):
            raise ValueError(f"unknown validation metric {self.metric!r}")


class QueryOverlapIndex:
    """node id -> training queries containing it (pipeline.py:54-69), CSR form."""

    def __init__(self, queries):
        q = np.asarray([getattr(x, "nodes", x) for x in queries], dtype=np.int64)
        if q.ndim != 2:
            raise ValueError("queries must share one arity")
        self.queries = q
        flat = q.reshape(-1)
        qid = np.repeat(np.arange(q.shape[0], dtype=np.int64), q.shape[1])
        order = np.argsort(flat, kind="stable")  # per node, query ids ascending
        self._qids = qid[order]
        self.nodes, starts, counts = np.unique(flat[order], return_index=True, return_counts=True)
        self._start = dict(zip(self.nodes.tolist(), starts.tolist()))
        self._count = dict(zip(self.nodes.tolist(), counts.tolist()))

    def queries_of(self, u: int):
        s = self._start.get(u)
        if s is None:
            return []
        return self._qids[s: s + self._count[u]].tolist()

    def __len__(self) -> int:
        return int(self.nodes.shape[0])


def canonical_nodes(nodes) -> tuple:
    return tuple(sorted(int(v) for v in nodes))


def sample_minibatch(index: QueryOverlapIndex, queries, cfg: TrainConfig, rng: np.random.Generator,
                     n_seeds: Optional[int] = None, exact: bool = True):
    """BFS over query-sharing neighbours (pipeline.py:77-129).

    ``exact=True`` (the default, the reference's draw) takes the seed nodes
    with ``rng.choice(..., replace=False)`` exactly like the reference (a
    full permutation of the node list per batch); ``exact=False`` draws the
    same uniform distinct subset by rejection, which is O(n_seeds)."""
    if len(index) == 0:
        raise ValueError("empty training query set")
    if n_seeds is None:
        n_seeds = min(16, cfg.batch_capacity)
    n_seeds = min(n_seeds, len(index.nodes))
    if exact:
        seeds = rng.choice(index.nodes, size=n_seeds, replace=False)
    else:
        picked: list = []
        seen: set = set()
        while len(picked) < n_seeds:
            for i in rng.integers(0, len(index.nodes), size=2 * (n_seeds - len(picked))).tolist():
                if i not in seen and len(picked) < n_seeds:
                    seen.add(i)
                    picked.append(i)
        seeds = index.nodes[np.asarray(picked, dtype=np.int64)]
    qarr = index.queries
    seed_list, in_seed, batch, in_batch, queue = [], set(), [], set(), deque()
    for s in seeds.tolist():
        if s not in in_seed:
            in_seed.add(s)
            seed_list.append(s)
            queue.append(s)
    full = False
    while queue and not full:
        u = queue.popleft()
        for qid in index.queries_of(u):
            if qid in in_batch:
                continue
            if len(batch) >= cfg.batch_size:
                full = True
                break
            in_batch.add(qid)
            batch.append(qid)
            for w in qarr[qid].tolist():
                if w not in in_seed:
                    if len(seed_list) >= cfg.batch_capacity:
                        full = True
                        break
                    in_seed.add(w)
                    seed_list.append(w)
                    queue.append(w)
            if full:
                break
    return seed_list, batch


class PositiveFilter:
    """Membership test of canonical node tuples against the positive set,
    vectorised over sorted packed keys (pipeline.py:278-280)."""

    def __init__(self, tuples: np.ndarray, num_nodes: int):
        t = np.sort(np.asarray(tuples, dtype=np.int64), axis=1)
        self.n = int(num_nodes)
        self.keys = np.unique(self._pack(t))

    def _pack(self, t: np.ndarray) -> np.ndarray:
        k = np.zeros(t.shape[0], dtype=np.int64)
        for c in range(t.shape[1]):
            k = k * self.n + t[:, c]
        return k

    def contains(self, rows: np.ndarray) -> np.ndarray:
        k = self._pack(np.sort(rows, axis=1))
        pos = np.searchsorted(self.keys, k)
        pos = np.minimum(pos, len(self.keys) - 1)
        return self.keys[pos] == k if len(self.keys) else np.zeros(len(k), bool)


def sample_negatives_array(seed_set: Sequence[int], arity: int, count: int, positive_filter,
                           rng: np.random.Generator) -> np.ndarray:
    """Uniform distinct-node tuples inside the seed set, rejected against the
    positives (pipeline.py:132-166), as an int64 [count, arity] array.
    Vectorised per chunk with the same rng draws and acceptance order as the
    reference loop, so for the same generator state it returns the same
    queries.  ``positive_filter`` is a PositiveFilter or a set of canonical
    tuples."""
    nodes = np.asarray(list(seed_set), dtype=np.int64)
    if nodes.shape[0] < arity:
        raise ValueError(f"seed set of {nodes.shape[0]} nodes cannot host arity-{arity} negatives")
    out = []
    have = 0
    budget = 1000 * count
    while have < count:
        chunk = min(max(2 * (count - have), 64), budget)
        if chunk <= 0:
            break
        draws = rng.integers(0, nodes.shape[0], size=(chunk, arity))
        budget -= chunk
        picked = nodes[draws]
        s = np.sort(picked, axis=1)
        ok = np.all(s[:, 1:] != s[:, :-1], axis=1) if arity > 1 else np.ones(chunk, bool)
        if isinstance(positive_filter, PositiveFilter):
            ok &= ~positive_filter.contains(picked)
        else:
            ok &= np.array([tuple(r) not in positive_filter for r in s.tolist()], bool)
        acc = picked[ok][: count - have]
        out.append(acc)
        have += acc.shape[0]
        if budget <= 0 and have < count:
            raise ValueError(f"negative sampling budget exhausted after producing {have}/{count} queries")
    return np.concatenate(out) if out else np.empty((0, arity), np.int64)


def sample_negatives(seed_set: Sequence[int], arity: int, count: int, positive_filter,
                     rng: np.random.Generator) -> list:
    """The reference signature and return type (pipeline.py:132-166): a list
    of label-0 ``Query`` objects, same draws as ``sample_negatives_array``."""
    arr = sample_negatives_array(seed_set, arity, count, positive_filter, rng)
    return [Query(tuple(int(v) for v in row), 0) for row in arr.tolist()]


def make_batch(index, positives: np.ndarray, pos_filter, cfg: TrainConfig, rng, exact=False):
    """One batch of query ids + labels (pipeline.py:293-304)."""
    seeds, ids = sample_minibatch(index, positives, cfg, rng, exact=exact)
    pos = positives[np.asarray(ids, dtype=np.int64)]
    negs = sample_negatives_array(seeds, positives.shape[1], cfg.k_neg * len(ids), pos_filter, rng)
    q = np.concatenate([pos, negs]).astype(np.int64)
    labels = np.concatenate([np.ones(len(ids)), np.zeros(len(negs))]).astype(np.float32)
    return q, labels


def _rng_words(rng: np.random.Generator) -> np.ndarray:
    s = rng.bit_generator.state
    if s.get("bit_generator") != "PCG64":
        raise NotImplementedError(f"the native planner restates numpy's PCG64, not {s.get('bit_generator')}")
    m64 = (1 << 64) - 1
    st, inc = int(s["state"]["state"]), int(s["state"]["inc"])
    return np.array([st >> 64, st & m64, inc >> 64, inc & m64, int(s["has_uint32"]), int(s["uinteger"])],
                    dtype=np.uint64)


# background planner builds in flight: the build is DRAM / core bound on the
# host, so a concurrent host -> device upload (graph.upload) uses fewer threads
_builds_lock = threading.Lock()
_builds_in_flight = 0


def planner_builds_in_flight() -> int:
    return _builds_in_flight


def _build_count(delta: int) -> None:
    global _builds_in_flight
    with _builds_lock:
        _builds_in_flight += delta


class BatchPlanner:
    """Training batches from the native planner (csrc/planner.cpp,
    ``wj_planner_*``): the reference's ``sample_minibatch`` +
    ``sample_negatives`` (or the fixed negative pool) per batch
    (pipeline.py:292-304) restated in C++ on the caller's numpy PCG64
    generator, so the batches are the reference's own for the same seed and
    ``rng`` ends in the state the reference would leave it in (after
    ``sync()``).  Batches are written into a ring of pinned host buffers
    (``depth`` deep; a buffer is reused only after the event recorded by the
    consumer's copy of it has completed), ready for a non-blocking H2D.

    ``next()`` -> (q [B, A] int64, y [B] float32, n_pos), views into the ring
    (B = 0: empty batch)."""

    def __init__(self, positives, filter_rows, num_nodes: int, cfg: TrainConfig, rng: np.random.Generator,
                 pool=None, depth: int = 4, pinned: bool = True, background: bool = False):
        from . import _lib

        pos = np.ascontiguousarray(positives, dtype=np.int64)
        if pos.ndim != 2 or pos.shape[0] == 0:
            raise ValueError("empty training query set")
        filt = np.ascontiguousarray(filter_rows, dtype=np.int64).reshape(-1, pos.shape[1])
        pl = None if pool is None or len(pool) == 0 else np.ascontiguousarray(pool, dtype=np.int64)
        self._lib = _lib.load()
        self.rng, self.arity = rng, int(pos.shape[1])
        self.n_pos = int(pos.shape[0])
        self.cap = int(cfg.batch_size) * (1 + int(cfg.k_neg))
        self._h = ctypes.c_void_p()
        cargs = (pos.ctypes.data, pos.shape[0], self.arity, filt.ctypes.data, filt.shape[0], int(num_nodes),
                 int(cfg.batch_capacity), int(cfg.batch_size), int(cfg.k_neg),
                 None if pl is None else pl.ctypes.data, 0 if pl is None else pl.shape[0], ctypes.byref(self._h))
        self._words = _rng_words(rng)
        self._builder, self._build_err = None, None
        self.depth = int(depth)
        if background:
            # the build (query index + positive-tuple set, ~0.15 s at C3) runs on
            # a host thread -- ctypes releases the GIL -- e.g. while the device
            # preprocess runs; the first use waits for it
            self._keep = (pos, filt, pl)

            def build():
                try:
                    _lib.call("wj_planner_create", *cargs)
                    # the pinned ring too (a cudaHostAlloc per buffer: ~7 ms
                    # that would otherwise sit before the preprocess)
                    self._alloc_ring(pinned)
                except BaseException as e:  # re-raised by wait()
                    self._build_err = e
                finally:
                    _build_count(-1)

            self._builder = threading.Thread(target=build, name="wj-planner-build", daemon=True)
            _build_count(1)
            self._builder.start()
        else:
            _lib.call("wj_planner_create", *cargs)
            _lib.call("wj_planner_set_rng", self._h, self._words.ctypes.data)
            self._alloc_ring(pinned)
        self.groups_view = None
        self._ev = [None] * self.depth
        self._i = 0
        self._cur = 0
        self._running = False
        self._out = (ctypes.c_int64 * 3)()

    def _alloc_ring(self, pinned: bool) -> None:
        """The planner's ring of batch slots (pinned: the H2D copies and the
        native epoch loop read them in place)."""
        mk = (lambda t: t.pin_memory()) if pinned and torch.cuda.is_available() else (lambda t: t)
        self._q = mk(torch.empty((self.depth, self.cap, self.arity), dtype=torch.int64))
        self._y = mk(torch.empty((self.depth, self.cap), dtype=torch.float32))
        # per slot: units of identical queries [G | start[0..G] | order | tuple] (wj_group_queries)
        self._g = mk(torch.empty((self.depth, (2 + self.arity) * self.cap + 2), dtype=torch.int32))

    def wait(self) -> None:
        """Block until a background build has finished (no-op otherwise)."""
        from . import _lib

        if self._builder is not None:
            self._builder.join()
            self._builder = None
            self._keep = None
            if self._build_err is not None:
                raise self._build_err
            _lib.call("wj_planner_set_rng", self._h, self._words.ctypes.data)

    def next(self):
        """One batch, planned on the calling thread."""
        from . import _lib

        self.wait()
        i = self._i
        self._i = (i + 1) % self.depth
        if self._ev[i] is not None:  # the copy that last read this buffer
            self._ev[i].synchronize()
            self._ev[i] = None
        o = self._out
        _lib.call("wj_planner_next", self._h, self._q[i].data_ptr(), self._y[i].data_ptr(), self.cap,
                  ctypes.byref(o, 0), ctypes.byref(o, 8), ctypes.byref(o, 16))
        B = int(o[0])
        _lib.call("wj_group_queries", self._q[i].data_ptr(), B, self.arity, GROUP_MAX, self._g[i].data_ptr(), None)
        self.groups_view = self._g[i]
        self._cur = i
        return self._q[i][:B], self._y[i][:B], int(o[1])

    def release(self, event) -> None:
        """The last batch's buffers are read by work ``event`` completes
        (e.g. the step's H2D copy); the slot is reused only after it."""
        self._ev[self._cur] = event

    def epoch(self):
        """One epoch of train()'s batch loop (pipeline.py:287-305), planned
        ahead on the native producer thread (``wj_planner_start_epoch``).
        Yields (q, y, n_pos) views into the pinned ring; call ``release`` with
        the event of the batch's copy before asking for the next one (no
        event: the batch was consumed synchronously).  After a completed
        epoch the rng is in the reference's end-of-epoch state."""
        from . import _lib

        self.wait()
        _lib.call("wj_planner_start_epoch", self._h, self._q.data_ptr(), self._y.data_ptr(), self._g.data_ptr(),
                  self.depth, self.cap)
        self._running = True
        pending = deque()
        slot = ctypes.c_int32()
        o = self._out
        try:
            while True:
                # hand back the slots whose copies have completed; keep at
                # most depth-1 outstanding so the producer can always advance
                while pending and (pending[0][1] is None or pending[0][1].query()):
                    _lib.call("wj_planner_release", self._h, pending.popleft()[0])
                while len(pending) >= self.depth - 1:
                    s, ev = pending.popleft()
                    if ev is not None:
                        ev.synchronize()
                    _lib.call("wj_planner_release", self._h, s)
                _lib.call("wj_planner_acquire", self._h, ctypes.byref(slot), ctypes.byref(o, 0), ctypes.byref(o, 8))
                s = int(slot.value)
                if s < 0:
                    self._running = False
                    return
                B = int(o[0])
                self._cur = s
                self._ev[s] = None
                self.groups_view = self._g[s]
                yield self._q[s][:B], self._y[s][:B], int(o[1])
                pending.append((s, self._ev[s]))
                self._ev[s] = None
        finally:
            if self._running:
                self._lib.wj_planner_stop(self._h)
                self._running = False

    def start_native(self) -> None:
        """Start an epoch's producer thread for a native consumer
        (``TrainStep.run_epoch`` / wj_train_epoch) instead of ``epoch()``."""
        from . import _lib

        self.wait()
        _lib.call("wj_planner_start_epoch", self._h, self._q.data_ptr(), self._y.data_ptr(), self._g.data_ptr(),
                  self.depth, self.cap)
        self._running = True

    def end_native(self, stopped: bool) -> None:
        """After a native epoch: the producer returned (epoch complete) or is
        stopped here (the consumer ended early)."""
        if stopped:
            self._lib.wj_planner_stop(self._h)
        self._running = False

    def sync(self) -> None:
        """Write the planner's PCG64 state back into the numpy generator."""
        from . import _lib

        self.wait()
        _lib.call("wj_planner_get_rng", self._h, self._words.ctypes.data)
        w = [int(x) for x in self._words]
        st = self.rng.bit_generator.state
        st["state"] = {"state": (w[0] << 64) | w[1], "inc": (w[2] << 64) | w[3]}
        st["has_uint32"], st["uinteger"] = w[4], w[5]
        self.rng.bit_generator.state = st

    def close(self) -> None:
        self.wait()
        if getattr(self, "_h", None) is not None and self._h.value:
            if not self._running:
                self.sync()
            self._lib.wj_planner_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None and self._h.value:
                self._lib.wj_planner_destroy(self._h)
                self._h = None
        except Exception:
            pass


class DeviceFeeder:
    """Planner batches (pinned host slots) -> a device ring, for the chain
    executor: each batch's H2D copy is issued on a side stream one batch
    ahead and its completion is checked on the HOST before the batch is
    handed out, so the training stream carries no copy or wait between steps
    and its programmatic-dependent chain stays unbroken (the kernels then
    read device memory, not mapped host memory: ~5 us per step less at C3).
    A device slot is overwritten only after the step that read it (the
    consumer calls ``consumed()`` after each step)."""

    def __init__(self, planner: "BatchPlanner", device, depth: int = 4):
        self.planner, self.dev, self.depth = planner, torch.device(device), int(depth)
        self.q = torch.empty((self.depth, planner.cap, planner.arity), dtype=torch.int64, device=self.dev)
        self.g = torch.empty((self.depth, (2 + planner.arity) * planner.cap + 2), dtype=torch.int32, device=self.dev)
        self._ng = [0] * self.depth
        self.groups, self.n_groups = None, 0  # the current batch's query groups (device) and their count
        self._ycache = {}
        self.stream = torch.cuda.Stream(self.dev)
        self.copied = [torch.cuda.Event() for _ in range(self.depth)]
        self.done = [torch.cuda.Event() for _ in range(self.depth)]
        self._used = [False] * self.depth
        self._cur = None
        self._k = 0

    def _labels(self, B: int, n_pos: int) -> torch.Tensor:
        # the planner's labels are 1 for the first n_pos queries, 0 after:
        # one resident device vector per (B, n_pos) instead of a copy per step
        y = self._ycache.get((B, n_pos))
        if y is None:
            y = torch.zeros(B, dtype=torch.float32, device=self.dev)
            y[:n_pos] = 1.0
            self._ycache[(B, n_pos)] = y
        return y

    def _issue(self, batch):
        q, y, n_pos = batch
        s = self._k % self.depth
        self._k += 1
        B = int(q.shape[0])
        if self._used[s]:  # the step that last read this slot
            self.stream.wait_event(self.done[s])
        gv = self.planner.groups_view
        G = int(gv[0])
        self._ng[s] = G
        with torch.cuda.stream(self.stream):
            self.q[s, :B].copy_(q, non_blocking=True)
            self.g[s, :G + 2 + B + G * self.planner.arity].copy_(gv[:G + 2 + B + G * self.planner.arity],
                                                                non_blocking=True)
            self.copied[s].record(self.stream)
        self.planner.release(self.copied[s])  # the pinned slot is free once copied
        return s, B, n_pos

    def epoch(self):
        """Yields (q, y, n_pos) device views, one epoch of the planner."""
        it = self.planner.epoch()
        try:
            b = next(it, None)
            nxt = self._issue(b) if b is not None else None
            first = True
            while nxt is not None:
                s, B, n_pos = nxt
                if not first:  # the next batch's copy goes out before this one is handed over
                    b = next(it, None)
                    nxt = self._issue(b) if b is not None else None
                self.copied[s].synchronize()  # long complete: issued a step ago
                self._cur = s
                self.groups, self.n_groups = self.g[s], self._ng[s]
                yield self.q[s, :B], self._labels(B, n_pos), n_pos
                if first:  # the first batch is handed over as soon as it is copied
                    first = False
                    b = next(it, None)
                    nxt = self._issue(b) if b is not None else None
        finally:
            it.close()

    def consumed(self) -> None:
        """Call after enqueueing the step that reads the last batch."""
        s = self._cur
        self.done[s].record(torch.cuda.current_stream(self.dev))
        self._used[s] = True


class TrainStep:
    """One training step on the device, captured as CUDA graphs per batch
    shape (``use_graph``; two graphs with their own input buffers, so the
    next batch's copy overlaps the current step on a side stream).

    mode="fused" (default): wj_join_encode (join + densify + layer 1 + ReLU +
    dropout + row mean + backward statistics, one kernel) -> wj_encoder_tail
    (tensor-core tail + partial gradients) -> wj_adam, PDL-chained (the
    PyTorch tail is used for hidden != 64).  mode="pooled" / "reference": the
    wj_join dense kernel feeds the PyTorch encoder (``E.forward``).

    overlap_inputs: device-resident q / y are complete when passed (their
    producers finished), so their copy need not wait for the current stream;
    host (pinned) inputs always overlap."""

    def __init__(self, store: SubgraphStore, params: E.ModelParams, state: E.AdamState,
                 dense_dtype=torch.float32, mode: str = "fused", use_graph: bool = True,
                 process_group=None, seed: int = 0, fast_tail: Optional[bool] = None,
                 features: Optional[torch.Tensor] = None, overlap_inputs: bool = False, launch: str = "graph",
                 dp_mode: str = "replicate"):
        if dp_mode not in ("replicate", "shard"):
            raise ValueError(f"dp_mode must be 'replicate' or 'shard', got {dp_mode!r}")
        self.dp_mode = dp_mode
        if features is not None and mode == "fused":
            raise ValueError("node features need mode='pooled' or 'reference' (the fused kernel is RPE-only)")
        if mode == "fused" and not E.fused_supported(params, store):
            # outside every fused kernel's envelope: the dense join + PyTorch encoder
            mode = "pooled"
        self.store, self.params, self.state = store, params, state
        self.features = features
        self.dense_dtype, self.mode, self.use_graph = dense_dtype, mode, use_graph
        self.group = process_group
        self.seed = int(seed)
        self.dev = store.device
        self.inv_bc = None
        self.step_t = torch.full((1,), int(state.step), dtype=torch.int64, device=self.dev)
        self._graphs: dict = {}
        self._slot: dict = {}
        self._copy_stream = torch.cuda.Stream(self.dev) if use_graph else None
        self.overlap_inputs = bool(overlap_inputs)
        # fused + hidden 64: tail and Adam as two CUDA kernels on flat buffers
        self.fast_tail = (mode == "fused" and params.hidden == 64 and params.feature_dim == 0
                          and params.w1.dtype == torch.float32
                          and store.width * params.arity in (2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 14, 15, 16))
        if fast_tail is not None:
            self.fast_tail = self.fast_tail and fast_tail
        if self.fast_tail:
            self.flat, self.offs = E.flatten_params(params)
            self.m_flat = torch.cat([state.m[k].reshape(-1) for k in E.TENSOR_ORDER])
            self.v_flat = torch.cat([state.v[k].reshape(-1) for k in E.TENSOR_ORDER])
            for k, o, o2 in zip(E.TENSOR_ORDER, self.offs[:-1], self.offs[1:]):
                state.m[k] = self.m_flat[o:o2].view(params.tensors[k].shape)
                state.v[k] = self.v_flat[o:o2].view(params.tensors[k].shape)
            self.offs_c = (ctypes.c_int32 * 9)(*[int(x) for x in self.offs])
            from ._lib import sm_count_of

            self.tail_rows = 2 * sm_count_of(self.dev)
            self.loss_buf = torch.zeros(1, dtype=torch.float32, device=self.dev)
            if process_group is not None:  # data parallel: [grads | loss] all-reduced
                self.grad_flat = torch.zeros(int(self.offs[-1]) + 1, dtype=torch.float32, device=self.dev)
        if launch not in ("graph", "chain"):
            raise ValueError(f"launch must be 'graph' or 'chain', got {launch!r}")
        # "chain": the native step executor (wj_stepper_*): three programmatic-
        # dependent launches per step, consecutive steps chained on the stream
        self.launch = launch if self.fast_tail else "graph"
        self._stepper = None
        self._stepper_cap = 0
        # chain mode: the join+encode kernel grabs queries from a device counter
        self.dynamic_queries = os.environ.get("WJ_DYNAMIC_QUERIES", "1") != "0"
        self._sched = torch.zeros(2, dtype=torch.int32, device=self.dev)
        self.record_input_events = True
        self._loss_hist = None
        self._n_calls = 0
        self.input_event = None
        if self.launch == "chain":
            # the step executor needs the tensor-core kernel and the store's
            # virtual-landing index; other shapes step through the graph path
            try:
                self._make_stepper(16)
            except (NotImplementedError, ValueError):
                self._stepper, self._stepper_cap = None, 0
                self.launch = "graph"
        if process_group is not None and dp_mode == "shard" and self.launch != "chain":
            raise NotImplementedError("dp_mode='shard' needs the chain step executor (launch='chain', fused, "
                                      "hidden 64)")

    def _buffers(self, B, A):
        if self.mode == "fused":
            H, AW = self.params.hidden, A * self.store.width
            bufs = {"pooled": torch.empty((B, H), device=self.dev),
                    "S": torch.empty((B, AW, H), device=self.dev),
                    "msum": torch.empty((B, H), device=self.dev)}
            if self.fast_tail:
                # tail CTAs of 16 queries each (fixed-order partial rows)
                rows = max(1, min((B + 15) // 16, self.tail_rows))
                bufs["partial"] = torch.empty((rows, int(self.offs[-1]) + 1), device=self.dev)
            return bufs
        d = 0 if self.features is None else int(self.features.shape[1])
        return {"dense": torch.empty((B, A * self.store.landings, A * self.store.width + d),
                                     dtype=self.dense_dtype, device=self.dev)}

    def _fast_body(self, q, y, bufs):
        """fused kernel -> encoder tail kernels -> Adam (4 launches)."""
        from . import _lib

        p, st, store = self.params, self.state, self.store
        B, A = q.shape
        keep = (1.0 - p.dropout) if p.dropout > 0.0 else 1.0
        scale = 1.0 / (keep * A * store.landings)
        dev = _lib.stream_handle(self.dev)
        rows = bufs["partial"].shape[0]
        E.forward_fused(p, store, q, training=True, seed=self.seed, step=self.step_t, out=bufs, tail=False)
        _lib.call("wj_encoder_tail", _lib.ptr(bufs["pooled"]), _lib.ptr(bufs["S"]), _lib.ptr(bufs["msum"]),
                  _lib.ptr(y), B, A * store.width, p.hidden, _lib.ptr(self.flat), self.offs_c, scale,
                  None, _lib.ptr(bufs["partial"]), rows, None, _lib.ptr(self.step_t), dev)
        partial, prow = bufs["partial"], rows
        if self.group is not None:
            from .distributed import all_reduce_mean

            _lib.call("wj_sum_partials", _lib.ptr(partial), rows, int(self.offs[-1]) + 1,
                      _lib.ptr(self.grad_flat), dev)
            all_reduce_mean(self.grad_flat, self.group)
            partial, prow = self.grad_flat, 1
        _lib.call("wj_adam", _lib.ptr(self.flat), _lib.ptr(self.m_flat), _lib.ptr(self.v_flat),
                  _lib.ptr(partial), prow, int(self.offs[-1]), st.lr, st.beta1, st.beta2,
                  st.eps, _lib.ptr(self.step_t), None, _lib.ptr(self.loss_buf), dev)
        return self.loss_buf[0]

    def _body(self, q, y, bufs, inv_bc):
        if self.fast_tail:
            return self._fast_body(q, y, bufs)
        if self.mode == "fused":
            # the dropout stream is keyed by the step counter BEFORE this step's
            # increment (the fast path's tail kernel increments it)
            logits, cache = E.forward_fused(self.params, self.store, q, training=True, seed=self.seed,
                                            step=self.step_t, out=bufs)
            self.step_t.add_(1)
        else:
            self.step_t.add_(1)
            dense_batch(self.store, q, dtype=self.dense_dtype, out=bufs["dense"], validate=False,
                        features=self.features)
            logits, cache = E.forward(self.params, bufs["dense"], training=True, mode=self.mode)
        loss = E.bce_loss(logits, y)
        grads = E.backward(self.params, cache, y)
        if self.group is not None:
            from .distributed import all_reduce_grads

            all_reduce_grads(grads, E.TENSOR_ORDER, self.group)
        # Adam bias corrections from the device step counter (already advanced
        # for this step), so they stay in stream order with the step itself
        t = self.step_t.to(self.params.w1.dtype)
        st = self.state
        inv_bc = 1.0 / (1.0 - torch.cat([torch.pow(st.beta1, t), torch.pow(st.beta2, t)]))
        E.adam_step_graphable(self.params, grads, self.state, inv_bc)
        return loss

    def _prepare_bc(self):
        # host bookkeeping only: every path derives Adam's bias corrections
        # on the device from the step counter
        self.state.step += 1

    # ------------------------------------------------------------ chain mode
    _LOSS_HIST = 4096

    def _make_stepper(self, B: int):
        from . import _lib

        st, p, store = self.state, self.params, self.store
        A, W = p.arity, store.width
        if self._stepper is not None:
            _lib.load().wj_stepper_destroy(self._stepper)
            self._stepper = None
        cap = max(B, 16)
        rows_max = max(1, min((cap + 15) // 16, self.tail_rows))
        self._chain_bufs = {"pooled": torch.empty((cap, 64), device=self.dev),
                            "S": torch.empty((cap, A * W, 64), device=self.dev),
                            "msum": torch.empty((cap, 64), device=self.dev),
                            "partial": torch.empty((rows_max, int(self.offs[-1]) + 1), device=self.dev)}
        b = self._chain_bufs
        keep = (1.0 - p.dropout) if p.dropout > 0.0 else 1.0
        h = ctypes.c_void_p()
        if store.voff_d is None:
            store.build_vindex()
        _lib.call("wj_stepper_create", _lib.ptr(store.offsets_d), _lib.ptr(store.uniq_x_d),
                  _lib.ptr(store.uniq_id_d), *store.vindex_ptrs(),
                  A, store.num_walks, store.walk_steps, store.max_unique, _lib.ptr(self.flat),
                  _lib.ptr(self.m_flat), _lib.ptr(self.v_flat), self.offs_c, keep,
                  1.0 / (keep * A * store.landings), self.seed & ((1 << 64) - 1),
                  st.lr, st.beta1, st.beta2, st.eps, _lib.ptr(self.step_t), _lib.ptr(b["pooled"]),
                  _lib.ptr(b["S"]), _lib.ptr(b["msum"]), _lib.ptr(b["partial"]), rows_max,
                  _lib.ptr(self._sched) if self.dynamic_queries else None, ctypes.byref(h))
        self._stepper, self._stepper_cap = h, cap
        self._rows_max = rows_max
        if self.group is not None and self.dp_mode == "shard":
            n1 = int(self.offs[-1]) + 1
            self._shard_partial = torch.empty((rows_max, n1), device=self.dev)
            self._full_partial = torch.empty((rows_max, n1), device=self.dev)
        if self._loss_hist is None:
            self._loss_hist = torch.zeros(self._LOSS_HIST, dtype=torch.float32, device=self.dev)

    def _chain_call(self, q: torch.Tensor, y: torch.Tensor, loss_out=None, groups=None) -> torch.Tensor:
        from . import _lib

        B = q.shape[0]
        if q.device.type == "cpu" and not q.is_pinned():
            q = q.to(self.dev)
        if y.device.type == "cpu" and not y.is_pinned():
            y = y.to(self.dev, torch.float32)
        if y.dtype != torch.float32:
            y = y.to(torch.float32)
        q = q.contiguous()
        if self._stepper is None or B > self._stepper_cap:
            self._make_stepper(B)
        i = self._n_calls % self._LOSS_HIST
        self._n_calls += 1
        out = self._loss_hist[i] if loss_out is None else loss_out
        gptr, ng = (None, 0)
        if groups is not None and self.dynamic_queries:
            gt, ng = groups
            gptr = gt.data_ptr()
        sh = _lib.stream_handle(self.dev)
        if self.group is None:
            _lib.call("wj_stepper_run", self._stepper, q.data_ptr(), y.data_ptr(), B, gptr, int(ng), out.data_ptr(),
                      sh)
        elif self.dp_mode == "shard":  # one global batch sharded over the ranks
            self._shard_step(q, y, out, sh)
        else:  # data parallel: grads + loss -> NCCL average -> Adam
            from .distributed import all_reduce_mean

            _lib.call("wj_stepper_grads", self._stepper, q.data_ptr(), y.data_ptr(), B, gptr, int(ng),
                      _lib.ptr(self.grad_flat), sh)
            all_reduce_mean(self.grad_flat, self.group)
            _lib.call("wj_stepper_apply", self._stepper, _lib.ptr(self.grad_flat), out.data_ptr(), sh)
        if (q.device.type == "cpu" or y.device.type == "cpu") and self.record_input_events:
            # host inputs are read in place: their buffers are free once this completes
            if not hasattr(self, "_events"):
                self._events = [torch.cuda.Event() for _ in range(16)]
            ev = self._events[i % 16]
            ev.record()
            self.input_event = ev
        else:
            self.input_event = None
        self.params.version += 1
        return out

    def _shard_step(self, q: torch.Tensor, y: torch.Tensor, out: torch.Tensor, sh) -> None:
        """Batch-sharded data parallel: every rank holds the
        same global batch and runs the queries of its share of the
        single-GPU step's tail rows (wj_stepper_grads_shard); the ranks'
        partial rows are gathered in row order (one broadcast per rank) and
        every rank applies the same fixed-order Adam reduction to them, so the
        step is bit-identical to one GPU stepping the whole batch."""
        import torch.distributed as dist

        from . import _lib

        B = q.shape[0]
        world, rank = dist.get_world_size(self.group), dist.get_rank(self.group)
        R = max(1, min((B + 15) // 16, self._rows_max))
        if R < world:
            raise ValueError(f"a batch of {B} queries has {R} tail rows, fewer than the {world} ranks")
        pc = -(-B // R)
        bounds = [(j * R // world, (j + 1) * R // world) for j in range(world)]
        r0, r1 = bounds[rank]
        b0, b1 = min(B, r0 * pc), min(B, r1 * pc)
        _lib.call("wj_stepper_grads_shard", self._stepper, q[b0:].data_ptr(), y[b0:].data_ptr(), b1 - b0, None, 0,
                  b0, B, pc, r1 - r0, _lib.ptr(self._shard_partial), sh)
        full = self._full_partial
        for j, (j0, j1) in enumerate(bounds):
            if j == rank:
                full[j0:j1].copy_(self._shard_partial[: j1 - j0])
            dist.broadcast(full[j0:j1], src=j, group=self.group)
        _lib.call("wj_stepper_apply_rows", self._stepper, _lib.ptr(full), R, out.data_ptr(), sh)

    def run_epoch(self, planner: "BatchPlanner", loss_out: Optional[torch.Tensor] = None,
                  max_steps: int = -1, device_depth: int = 4) -> int:
        """One epoch (or ``max_steps`` batches) of the native planner through
        the step executor with no Python between steps (wj_train_epoch):
        pinned planner slot -> H2D one batch ahead on a copy stream -> step ->
        loss into ``loss_out[k]`` (device or pinned host, float32; default: a
        device buffer, see ``epoch_losses``).  Same batches, kernels and
        results as iterating ``DeviceFeeder.epoch()`` with ``__call__``.
        Single process, chain launch only.  Returns the number of steps."""
        from . import _lib

        if self.launch != "chain" or self.group is not None:
            raise ValueError("run_epoch needs launch='chain' and no process group")
        cap, A = planner.cap, planner.arity
        if self._stepper is None or cap > self._stepper_cap:
            self._make_stepper(cap)
        ring = getattr(self, "_ering", None)
        if ring is None or ring[0].shape[1] != cap or ring[0].shape[2] != A or ring[0].shape[0] != device_depth:
            lab = torch.zeros(2 * cap, dtype=torch.float32, device=self.dev)
            lab[:cap] = 1.0
            ring = (torch.empty((device_depth, cap, A), dtype=torch.int64, device=self.dev),
                    torch.empty((device_depth, (2 + A) * cap + 2), dtype=torch.int32, device=self.dev), lab,
                    torch.cuda.Stream(self.dev))
            self._ering = ring
        dq, dg, lab, cstream = ring
        if loss_out is None:
            n = max_steps if max_steps >= 0 else planner.n_pos + 1
            if getattr(self, "epoch_losses", None) is None or self.epoch_losses.numel() < n:
                self.epoch_losses = torch.empty(n, dtype=torch.float32, device=self.dev)
            loss_out = self.epoch_losses
        done, nbytes = ctypes.c_int64(0), ctypes.c_int64(0)
        planner.start_native()
        try:
            _lib.call("wj_train_epoch", self._stepper, planner._h, planner._q.data_ptr(), planner._g.data_ptr(),
                      planner.depth, cap, A, dq.data_ptr(), dg.data_ptr(), device_depth, lab.data_ptr(),
                      loss_out.data_ptr(), int(max_steps), _lib.stream_handle(self.dev), cstream.cuda_stream,
                      ctypes.byref(done), ctypes.byref(nbytes))
        except BaseException:
            planner.end_native(stopped=True)
            raise
        k = int(done.value)
        self.last_epoch_h2d_bytes = int(nbytes.value)  # batches issued (incl. one look-ahead copy)
        planner.end_native(stopped=max_steps >= 0 and k >= max_steps)
        self.state.step += k
        self._n_calls += k
        self.params.version += k
        return k

    def encode_only(self, q: torch.Tensor, groups=None) -> None:
        """Chain mode: launch just this step's join+encode kernel (same
        plan, scheduling and buffers; the step counter is not advanced)."""
        from . import _lib

        if self.launch != "chain":
            raise ValueError("encode_only needs launch='chain'")
        if self._stepper is None or q.shape[0] > self._stepper_cap:
            self._make_stepper(q.shape[0])
        gptr, ng = (None, 0)
        if groups is not None and self.dynamic_queries:
            gptr, ng = groups[0].data_ptr(), int(groups[1])
        _lib.call("wj_stepper_encode", self._stepper, q.data_ptr(), q.shape[0], gptr, ng,
                  _lib.stream_handle(self.dev))

    def __del__(self):
        try:
            if getattr(self, "_stepper", None) is not None:
                from . import _lib

                _lib.load().wj_stepper_destroy(self._stepper)
                self._stepper = None
        except Exception:
            pass

    def __call__(self, q: torch.Tensor, y: torch.Tensor, loss_out: Optional[torch.Tensor] = None,
                 groups=None) -> torch.Tensor:
        """q: [B, A] int64 ids, y: [B] labels (device, or pinned host for the
        end-to-end path).  Returns the loss (device scalar, valid in stream
        order).  ``launch="chain"``: the inputs are read by the kernels in
        place (pinned host memory stays untouched until the step completes)
        and ``loss_out`` (a one-element device or pinned host tensor)
        optionally receives the loss instead; ``groups`` = (device int32
        tensor [G | start | order | tuple] from wj_group_queries, G) lets the
        join+encode kernel share the staging of identical queries."""
        B, A = q.shape
        self._prepare_bc()
        if self.launch == "chain":
            return self._chain_call(q, y, loss_out, groups)
        if not self.use_graph:
            qd, yd = q.to(self.dev, non_blocking=True), y.to(self.dev, self.params.w1.dtype, non_blocking=True)
            self.input_event = torch.cuda.Event()
            self.input_event.record()
            out = self._body(qd, yd, self._buffers(B, A), self.inv_bc)
            self.params.version += 1
            return out
        key = (B, A)
        slots = self._graphs.get(key)
        if slots is None:  # two captured graphs with their own input buffers
            slots = [self._capture(B, A) for _ in range(2)]
            self._graphs[key] = slots
        i = self._slot.get(key, 0)
        self._slot[key] = i ^ 1
        g = slots[i]
        cur = torch.cuda.current_stream(self.dev)
        cs = self._copy_stream
        # the batch is copied into this slot on a side stream, overlapping the
        # previous step's kernels; the copy waits only for the replay that last
        # read this slot (and, for device inputs not declared ready, for the
        # current stream)
        if q.device.type == "cuda" and not self.overlap_inputs:
            cs.wait_stream(cur)
        cs.wait_event(g["done"])
        with torch.cuda.stream(cs):
            g["q"].copy_(q, non_blocking=True)
            g["y"].copy_(y, non_blocking=True)
            g["ready"].record(cs)
        for t in (q, y):
            if t.device.type == "cuda":
                t.record_stream(cs)
        cur.wait_event(g["ready"])
        self.input_event = g["ready"]  # completes once q / y have been read
        g["graph"].replay()
        g["done"].record(cur)
        self.params.version += 1
        return g["loss"]

    def _capture(self, B, A):
        dev = self.dev
        q = torch.zeros((B, A), dtype=torch.int64, device=dev)
        q[:, :] = torch.arange(A, device=dev)[None, :] % max(self.store.num_nodes, 1)
        y = torch.zeros(B, dtype=self.params.w1.dtype, device=dev)
        bufs = self._buffers(B, A)
        # warm up on a side stream (allocator + cuBLAS handles), then capture;
        # params / Adam state / step counter are snapshotted so warm-up leaves no trace
        snap_p = {k: v.clone() for k, v in self.params.tensors.items()}
        snap_m = {k: v.clone() for k, v in self.state.m.items()}
        snap_v = {k: v.clone() for k, v in self.state.v.items()}
        snap_step = self.step_t.clone()
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            for _ in range(2):
                self._body(q, y, bufs, self.inv_bc)
        torch.cuda.current_stream(dev).wait_stream(s)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            loss = self._body(q, y, bufs, self.inv_bc)
        for k in snap_p:
            self.params.tensors[k].copy_(snap_p[k])
            self.state.m[k].copy_(snap_m[k])
            self.state.v[k].copy_(snap_v[k])
        self.step_t.copy_(snap_step)
        return {"graph": graph, "q": q, "y": y, "bufs": bufs, "loss": loss, "ready": torch.cuda.Event(),
                "done": torch.cuda.Event()}


@dataclass
class QuerySplit:
    """Inductive link-query split (graph.py:123-132): positives per phase,
    per-positive negative groups for evaluation, and the walk graph with the
    training edges removed.  Any object with these attributes (e.g. the
    reference's own QuerySplit) is accepted by ``train``."""

    train_pos: list
    valid_pos: list
    test_pos: list
    valid_neg: list = field(default_factory=list)
    test_neg: list = field(default_factory=list)
    train_graph: object = None


def _rows(queries) -> np.ndarray:
    if isinstance(queries, np.ndarray):
        return queries.astype(np.int64, copy=False)
    if len(queries) == 0:
        return np.empty((0, 0), np.int64)
    return np.asarray([getattr(q, "nodes", q) for q in queries], dtype=np.int64)


def _check_ids(store: SubgraphStore, q: torch.Tensor) -> None:
    """One range check of a device query batch (joiner.py:40-50): min and max
    in one reduction and one device-to-host read."""
    if q.numel():
        mn, mx = (int(v) for v in torch.stack(torch.aminmax(q)).cpu())
        if mn < 0 or mx >= store.num_nodes:
            raise ValueError(f"query node ids must lie in [0, {store.num_nodes})")


def score_array(store: SubgraphStore, params: E.ModelParams, query_array, features=None,
                chunk: int = 1 << 16, validate: bool = True) -> torch.Tensor:
    """Sigmoid scores of a query array as a float64 DEVICE tensor
    (pipeline.py:185-198 without the host round trip).  RPE-only fp32 models
    inside the fused kernels' envelope score through wj_join_encode (keep = 1:
    no dropout stream, no backward statistics); feature models and other
    shapes through the dense join kernel + PyTorch encoder."""
    q_all = torch.as_tensor(query_array, dtype=torch.int64)
    if q_all.shape[0] == 0:
        return torch.empty(0, dtype=torch.float64, device=store.device)
    if q_all.dim() != 2 or q_all.shape[1] != params.arity:
        raise ValueError(f"queries must be [B, {params.arity}] for this model")
    host_runs = None
    if q_all.device.type == "cpu":
        # host input: the range check and the first-anchor run count on the
        # host, before the copy, so the device stream never waits on the host
        if validate:
            qn = q_all.numpy()
            if int(qn.min()) < 0 or int(qn.max()) >= store.num_nodes:
                raise ValueError(f"query node ids must lie in [0, {store.num_nodes})")
        host_runs = q_all[:, 0].numpy()
        q_all = q_all.to(store.device, non_blocking=q_all.is_pinned())
    elif validate:
        _check_ids(store, q_all)
    fused = features is None and E.fused_supported(params, store)
    scorer = None
    if fused and params.hidden == 64 and params.arity * store.width in E.TAIL_AW:
        # join+encode (keep = 1) -> tail kernel; the scorer (buffers) is cached
        # on the parameters, its flat copy of them refreshed on every call
        scorer = getattr(params, "_scorer", None)
        if scorer is None or scorer.store is not store:
            scorer = E.FusedScorer(params, store)
            params._scorer = scorer
        else:
            scorer.refresh()
    out = []
    for lo in range(0, q_all.shape[0], chunk):
        q = q_all[lo: lo + chunk]
        if scorer is not None:
            shared = None
            if host_runs is not None:
                f = host_runs[lo: lo + chunk]
                shared = scorer.use_shared_runs(q.shape[0], 1 + int(np.count_nonzero(f[1:] != f[:-1])))
            logits = scorer.logits(q, shared=shared)  # .double() below copies it out of the scorer
        elif fused:
            logits, _ = E.forward_fused(params, store, q, training=False, need_grad=False)
        else:
            dense = dense_batch(store, q, features=features, dtype=params.w1.dtype, validate=False)
            logits, _ = E.forward(params, dense, training=False)
        out.append(torch.sigmoid(logits.double()))
    return out[0] if len(out) == 1 else torch.cat(out)


def validation_metric(store: SubgraphStore, params: E.ModelParams, split, cfg: TrainConfig,
                      features=None, phase: str = "valid") -> float:
    """pipeline.py:214-238 on the device: AUC over all positive / negative
    scores, or MRR of each positive among its own negative group."""
    from . import metrics as Mx

    pos_q = _rows(getattr(split, f"{phase}_pos"))
    groups = getattr(split, f"{phase}_neg")
    flat = [getattr(q, "nodes", q) for grp in groups for q in grp]
    if not flat:
        raise ValueError(f"validation requires negative queries (split.{phase}_neg is empty)")
    pos = score_array(store, params, pos_q, features)
    neg = score_array(store, params, np.asarray(flat, dtype=np.int64), features)
    if cfg.metric == "auc":
        return Mx.roc_auc_device(pos, neg)
    return Mx.mrr_device(pos, neg, [len(g) for g in groups[: pos_q.shape[0]]])


def train(store: SubgraphStore, split, cfg: TrainConfig, features=None, train_negatives=None,
          use_graph: bool = True, exact_batches: bool = False, native_planner: bool = True):
    """Mini-batched training with early stopping (pipeline.py:241-326), same
    seeds, batch contract and history; every step runs on the device
    (``TrainStep``).  Returns (best params, history).

    Batches come from the native planner (``BatchPlanner``, arity <= 4): a
    producer thread that restates the reference's batch draws on the same
    numpy PCG64 stream, so with the same seed every batch -- positives,
    negatives, labels -- is the reference's own, and with dropout off the
    trajectory differs from the reference only by fp32 vs fp64 rounding.
    ``native_planner=False`` plans in Python: ``exact_batches=True`` then
    draws the BFS seeds with the reference's ``rng.choice`` (exact), the
    default by rejection (same distribution, different draws)."""
    from .seeds import derive_seed

    positives = _rows(split.train_pos)
    if positives.shape[0] == 0:
        raise ValueError("empty training set")
    arity = positives.shape[1]
    if not len(split.valid_pos):
        raise ValueError("training requires validation positives for early stopping")
    if cfg.use_features and features is None and getattr(split, "train_graph", None) is not None:
        features = getattr(split.train_graph, "node_features", None)
    features = features if cfg.use_features else None
    if features is not None:
        features = np.asarray(features, dtype=np.float64)
        if features.shape[0] != store.num_nodes:
            raise ValueError(f"feature matrix has {features.shape[0]} rows for {store.num_nodes} nodes")
    feature_dim = 0 if features is None else int(features.shape[1])
    dev = store.device
    filt_rows = [positives] + [_rows(g) for g in (split.valid_pos, split.test_pos) if len(g)]
    batch_rng = np.random.default_rng(derive_seed(cfg.seed, "minibatch"))
    pool = _rows(train_negatives) if train_negatives is not None and len(train_negatives) else None
    planner = feeder = index = pos_filter = None
    if native_planner and arity <= 4:
        # built on a host thread while the model and the step executor are set up
        planner = BatchPlanner(positives, np.concatenate(filt_rows), store.num_nodes, cfg, batch_rng, pool=pool,
                               background=True)
        feeder = DeviceFeeder(planner, dev)
    else:  # Python planning: the reference's structures
        index = QueryOverlapIndex(positives)
        pos_filter = PositiveFilter(np.concatenate(filt_rows), store.num_nodes)
    params = E.init_params(arity, store.walk_steps, hidden=cfg.hidden_dim, feature_dim=feature_dim,
                           dropout=cfg.dropout, seed=derive_seed(cfg.seed, "init"), device=dev)
    state = E.AdamState.for_params(params, lr=cfg.lr)
    feats_d = None if features is None else torch.as_tensor(features, dtype=torch.float32, device=dev)
    step = TrainStep(store, params, state, mode="fused" if feats_d is None else "pooled",
                     use_graph=use_graph, seed=derive_seed(cfg.seed, "dropout"), features=feats_d,
                     launch="chain" if use_graph else "graph")
    history = []
    best_params, best_metric, best_epoch = params.copy(), -np.inf, 0
    for epoch in range(1, cfg.max_epochs + 1):
        t0 = time.perf_counter()
        consumed, n_steps = 0, 0
        loss_sum = torch.zeros((), dtype=torch.float64, device=dev)
        if planner is not None and step.launch == "chain" and step.group is None:
            # the native epoch loop: planner -> H2D -> chain executor with no
            # Python between steps; per-step losses in a device buffer
            n_steps = step.run_epoch(planner)
            loss_sum += step.epoch_losses[:n_steps].double().sum()
        elif planner is not None and step.launch == "chain":
            # native planner -> device ring -> chain executor; per-step losses
            # stay in the executor's ring and are summed in blocks
            pending = []
            for q, y, _ in feeder.epoch():
                pending.append(step(q, y, groups=(feeder.groups, feeder.n_groups)))
                feeder.consumed()
                n_steps += 1
                if len(pending) == TrainStep._LOSS_HIST // 2:
                    loss_sum += torch.stack(pending).double().sum()
                    pending = []
            if pending:
                loss_sum += torch.stack(pending).double().sum()
        elif planner is not None:  # native planner, graph steps on pinned batches
            for q, y, _ in planner.epoch():
                loss_sum += step(q, y).double()
                planner.release(step.input_event)
                n_steps += 1
        while planner is None and consumed < positives.shape[0]:
            seeds, ids = sample_minibatch(index, positives, cfg, batch_rng, exact=exact_batches)
            if not ids:
                break
            pos = positives[np.asarray(ids, dtype=np.int64)]
            n_neg = cfg.k_neg * len(ids)
            if pool is not None:
                negs = pool[batch_rng.integers(0, pool.shape[0], size=n_neg)]
            else:
                negs = sample_negatives_array(seeds, arity, n_neg, pos_filter, batch_rng)
            q = torch.from_numpy(np.concatenate([pos, negs]).astype(np.int64))
            y = torch.from_numpy(np.concatenate([np.ones(len(ids)), np.zeros(negs.shape[0])]).astype(np.float32))
            loss_sum += step(q, y).double()
            consumed += len(ids)
            n_steps += 1
        valid = validation_metric(store, params, split, cfg, features=feats_d)
        train_loss = float(loss_sum) / max(n_steps, 1)
        history.append({"epoch": epoch, "train_loss": train_loss, "valid_metric": valid})
        logger.info("epoch %d train_loss %.6f valid_%s %.6f wall %.2fs", epoch, train_loss, cfg.metric,
                    valid, time.perf_counter() - t0)
        if valid > best_metric:
            best_metric, best_params, best_epoch = valid, params.copy(), epoch
        if epoch - best_epoch >= cfg.patience:
            break
    if planner is not None:
        planner.close()  # the generator ends in the reference's state
    return best_params, history


def infer(store: SubgraphStore, params: E.ModelParams, queries, threads: int = 1, features=None,
          chunk: int = 8192) -> np.ndarray:
    """Sigmoid scores, input order (pipeline.py:329-355): the reference's
    checks (arity, feature_dim / feature matrix), one range check of every
    query id, then ``score_array``."""
    if len(queries) == 0:
        return np.empty(0, dtype=np.float64)
    if isinstance(queries, np.ndarray):
        rows = queries.astype(np.int64, copy=False)
        if rows.ndim != 2:
            raise ValueError("queries must share one arity")
    else:
        lists = [tuple(getattr(q, "nodes", q)) for q in queries]
        if len(lists[0]) != params.arity:
            raise ValueError(f"queries have arity {len(lists[0])} but model was trained with arity {params.arity}")
        if any(len(r) != params.arity for r in lists):
            raise ValueError("queries must share one arity")
        rows = np.asarray(lists, dtype=np.int64)
    if rows.shape[1] != params.arity:
        raise ValueError(f"queries have arity {rows.shape[1]} but model was trained with arity {params.arity}")
    if params.feature_dim > 0:
        if features is None:
            raise ValueError("model expects node features but none were given")
        f = features if isinstance(features, torch.Tensor) else np.asarray(features, dtype=np.float64)
        if f.shape[0] != store.num_nodes:
            raise ValueError(f"feature matrix has {f.shape[0]} rows for {store.num_nodes} nodes")
        if f.shape[1] != params.feature_dim:
            raise ValueError(f"feature matrix width {f.shape[1]} != model feature_dim {params.feature_dim}")
        features = torch.as_tensor(f, dtype=params.w1.dtype, device=store.device)
    else:
        features = None  # the reference ignores features for an RPE-only model
    if rows.size and (rows.min() < 0 or rows.max() >= store.num_nodes):
        raise ValueError(f"query node ids must lie in [0, {store.num_nodes})")
    return score_array(store, params, rows, features=features, chunk=chunk, validate=False).cpu().numpy()
