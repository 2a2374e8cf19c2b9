"""Host-side logic of the multi-GPU path on CPU with gloo, world_size 2:
variable-size all-gather, the global RPE-id merge of per-rank distinct sets
(must reproduce the single-process reference table and ids), and the data-
parallel gradient average."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _pack_keys(vecs, cb):
    keys = np.zeros(vecs.shape[0], np.int64)
    for c in range(vecs.shape[1]):
        keys |= vecs[:, c].astype(np.int64) << (cb * c)
    return keys


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import core
        from paper_2202_13538_b200.distributed import (all_gather_sizes, all_gather_variable, all_reduce_grads,
                                                       all_reduce_mean, gather_into, merge_distinct, shard_range)

        # 0. gather straight into a preallocated buffer (rank order, no padding;
        # int16 as bytes; an empty shard)
        rows = [3 + 4 * r for r in range(world)]
        assert all_gather_sizes(rows[rank], "cpu") == rows
        loc = torch.arange(rows[rank] * 2, dtype=torch.int16).reshape(-1, 2) - 7 * rank
        out = gather_into(torch.empty((sum(rows), 2), dtype=torch.int16), loc, rows)
        want = torch.cat([torch.arange(rows[r] * 2, dtype=torch.int16).reshape(-1, 2) - 7 * r for r in range(world)])
        assert torch.equal(out, want)
        rows0 = [0 if r == 0 else 5 for r in range(world)]
        loc0 = torch.full((rows0[rank],), float(rank))
        out0 = gather_into(torch.empty(sum(rows0)), loc0, rows0)
        assert torch.equal(out0, torch.cat([torch.full((rows0[r],), float(r)) for r in range(world)]))

        # 1. variable-size all-gather
        t = torch.arange(3 + 4 * rank, dtype=torch.int64).reshape(-1, 1).repeat(1, 2) + 100 * rank
        parts = all_gather_variable(t)
        assert [p.shape[0] for p in parts] == [3 + 4 * r for r in range(world)]
        assert all(torch.equal(p, torch.arange(3 + 4 * r).reshape(-1, 1).repeat(1, 2) + 100 * r)
                   for r, p in enumerate(parts))

        # int16 / uint16 store arrays travel as bytes (NCCL has no 16-bit integer type)
        t16 = (torch.arange(2 + rank, dtype=torch.int16).reshape(-1, 1) * torch.tensor([1, -3], dtype=torch.int16))
        parts16 = all_gather_variable(t16)
        assert all(p.dtype == torch.int16 and torch.equal(p, torch.arange(2 + r, dtype=torch.int16).reshape(-1, 1)
                                                          * torch.tensor([1, -3], dtype=torch.int16))
                   for r, p in enumerate(parts16))

        # 2. sharded interning reproduces the reference table and ids
        g = load_golden("er1000_m50")
        M, L = int(g["M"]), int(g["L"])
        ref = core.preprocess(g["idxptr"], g["indices"], M, L, int(g["seed"]))
        n = int(g["n"])
        cb = max(1, M.bit_length())
        lo, hi = shard_range(n, world, rank)
        keys_all, ords_all = [], []
        for u in range(lo, hi):
            a, b = ref.item_offsets[u], ref.item_offsets[u + 1]
            vec = ref.table[ref.rpe_ids_flat[a:b]]          # count vectors of u's entries
            keys_all.append(_pack_keys(vec, cb))
            ords_all.append((np.int64(u) << 16) + np.arange(b - a))  # first-appearance rank order
        keys = np.concatenate(keys_all)
        ords = np.concatenate(ords_all)
        # local distinct (key, min order) -- what wj_intern_insert leaves in its table
        uk, inv = np.unique(keys, return_inverse=True)
        mins = np.full(uk.shape[0], np.iinfo(np.int64).max)
        np.minimum.at(mins, inv, ords)
        gk = torch.cat(all_gather_variable(torch.from_numpy(uk)))
        go = torch.cat(all_gather_variable(torch.from_numpy(mins)))
        suk, ids, table_keys = merge_distinct(gk, go)
        want = torch.from_numpy(_pack_keys(ref.table, cb))
        assert torch.equal(table_keys, want)
        mine = ids[torch.searchsorted(suk, torch.from_numpy(keys))]
        ref_ids = np.concatenate([ref.rpe_ids_flat[ref.item_offsets[u]:ref.item_offsets[u + 1]]
                                  for u in range(lo, hi)])
        assert np.array_equal(mine.numpy(), ref_ids)

        # 3. DP gradient average
        grads = {"a": torch.full((2, 3), float(rank + 1)), "b": torch.tensor([2.0 * rank])}
        all_reduce_grads(grads, ["a", "b"])
        assert torch.allclose(grads["a"], torch.full((2, 3), 1.5))
        assert torch.allclose(grads["b"], torch.tensor([1.0]))
        # 4. the fused step's flat [grads | loss] vector: mean over ranks in place
        flat = torch.arange(5, dtype=torch.float32) * (rank + 1)
        all_reduce_mean(flat)
        assert torch.allclose(flat, torch.arange(5, dtype=torch.float32) * 1.5)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_host_logic():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_shard_ranges_cover_nodes():
    from paper_2202_13538_b200.distributed import shard_range

    for n in (1, 7, 1000, 2_927_963):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
