"""Native mini-batch planner (csrc/planner.cpp) -- host code, runs on CPU.

Pinned to batch sequences written by the REAL reference
(tests/golden/make_batch_golden.py: the reference's sample_minibatch +
sample_negatives / fixed pool driven as train() drives them,
pipeline.py:287-305): every batch and the generator's final PCG64 state must
match exactly, both through the synchronous ``next()`` and through the
producer-thread ``epoch()``.  Also checked against numpy itself (the
package's vectorised ``make_batch(exact=True)``) and for the reference's
error behaviour."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

BATCH_DIR = os.path.join(GOLDEN, "batches")
CASES = sorted(f[:-4] for f in os.listdir(BATCH_DIR) if f.endswith(".npz"))


def _load(name):
    with np.load(os.path.join(BATCH_DIR, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def _planner(d, rng, depth=4):
    from paper_2202_13538_b200.pipeline import BatchPlanner, TrainConfig

    cfg = TrainConfig(batch_capacity=int(d["batch_capacity"]), batch_size=int(d["batch_size"]),
                      k_neg=int(d["k_neg"]), seed=int(d["seed"]))
    filt = np.concatenate([d["positives"], d["filter_extra"]])
    pool = d["pool"] if d["pool"].shape[0] else None
    return BatchPlanner(d["positives"], filt, int(d["num_nodes"]), cfg, rng, pool=pool, depth=depth,
                        pinned=False)


def _rng(d):
    from paper_2202_13538_b200.seeds import derive_seed

    return np.random.default_rng(derive_seed(int(d["seed"]), "minibatch"))


def _words(rng):
    from paper_2202_13538_b200.pipeline import _rng_words

    return _rng_words(rng)


def _split(d):
    offs = np.concatenate([[0], np.cumsum(d["sizes"])])
    return [(d["queries"][a:b], d["labels"][a:b]) for a, b in zip(offs[:-1], offs[1:])]


@pytest.mark.parametrize("name", CASES)
def test_epochs_match_reference(name):
    """Producer thread: every batch of every epoch + the end rng state."""
    d = _load(name)
    ref = _split(d)
    rng = _rng(d)
    bp = _planner(d, rng)
    got = []
    for _ in range(int(d["epochs"])):
        got += [(q.numpy().copy(), y.numpy().copy()) for q, y, _ in bp.epoch()]
    bp.close()
    assert len(got) == len(ref)
    for k, ((q, y), (qr, yr)) in enumerate(zip(got, ref)):
        assert np.array_equal(q, qr), f"batch {k} queries"
        assert np.array_equal(y, yr), f"batch {k} labels"
    assert np.array_equal(_words(rng), d["final_rng"])


@pytest.mark.parametrize("name", CASES)
def test_next_matches_reference(name):
    """Synchronous planning: the first epoch's batches in order."""
    d = _load(name)
    ref = [r for r, e in zip(_split(d), d["epoch_of"]) if e == 0]
    bp = _planner(d, _rng(d), depth=2)
    for k, (qr, yr) in enumerate(ref):
        q, y, n_pos = bp.next()
        assert np.array_equal(q.numpy(), qr), f"batch {k}"
        assert np.array_equal(y.numpy(), yr) and n_pos == int(yr.sum())


def test_matches_numpy_make_batch_and_state():
    """Against numpy directly (make_batch(exact=True) consumes the generator
    through rng.choice / rng.integers), 300 batches, and the state after."""
    from paper_2202_13538_b200.pipeline import (BatchPlanner, PositiveFilter, QueryOverlapIndex, TrainConfig,
                                                make_batch)

    g = np.random.default_rng(5)
    n = 4000
    pos = g.integers(0, n, size=(6000, 2))
    pos = pos[pos[:, 0] != pos[:, 1]]
    filt = np.concatenate([pos, g.integers(0, n, size=(9000, 2))])
    cfg = TrainConfig(batch_size=32, k_neg=50)
    idx, pf = QueryOverlapIndex(pos), PositiveFilter(filt, n)
    r1, r2 = np.random.default_rng(7), np.random.default_rng(7)
    bp = BatchPlanner(pos, filt, n, cfg, r2, pinned=False)
    for k in range(300):
        q, y = make_batch(idx, pos, pf, cfg, r1, exact=True)
        q2, y2, _ = bp.next()
        assert np.array_equal(q, q2.numpy()) and np.array_equal(y, y2.numpy()), k
    bp.sync()
    assert r1.bit_generator.state == r2.bit_generator.state
    bp.close()


def test_abandoned_epoch_and_restart():
    d = _load(CASES[0])
    bp = _planner(d, _rng(d))
    it = bp.epoch()
    next(it)
    next(it)
    it.close()  # stops the producer thread
    q, y, n = bp.next()  # the handle is usable again
    assert q.shape[0] == y.shape[0] > 0
    bp.close()


def test_reference_errors():
    from paper_2202_13538_b200.pipeline import BatchPlanner, TrainConfig

    rng = np.random.default_rng(0)
    # only (0, 1) exists and it is positive: every draw is rejected
    bp = BatchPlanner(np.array([[0, 1]]), np.array([[0, 1]]), 2, TrainConfig(k_neg=1), rng, pinned=False)
    with pytest.raises(ValueError, match="budget exhausted"):
        bp.next()
    # seed set capped at 2 nodes cannot host arity-3 negatives
    bp = BatchPlanner(np.array([[0, 1, 2]]), np.zeros((0, 3)), 3, TrainConfig(batch_capacity=2), rng,
                      pinned=False)
    with pytest.raises(ValueError, match="cannot host arity-3"):
        bp.next()
    with pytest.raises(ValueError, match="out of range"):
        BatchPlanner(np.array([[0, 5]]), np.zeros((0, 2)), 3, TrainConfig(), rng, pinned=False)
    with pytest.raises(NotImplementedError):
        BatchPlanner(np.array([[0, 1, 2, 3, 4]]), np.zeros((0, 5)), 6, TrainConfig(), rng, pinned=False)


def _check_groups(q, gb, cap=0):
    """Units: identical ordered tuples, members in batch order, <= cap
    members (0: a unit is a whole tuple), larger units first, then first
    occurrence; every query exactly once."""
    G = int(gb[0])
    start, order = gb[1:G + 2], gb[G + 2:G + 2 + q.shape[0]]
    tup = gb[G + 2 + q.shape[0]:G + 2 + q.shape[0] + G * q.shape[1]].reshape(G, q.shape[1])
    assert np.array_equal(tup, q[order[start[:-1]]])  # each unit's anchor tuple
    sizes = np.diff(start)
    assert start[0] == 0 and start[-1] == q.shape[0] and np.all(sizes > 0)
    assert sorted(order.tolist()) == list(range(q.shape[0]))
    assert np.all(np.diff(sizes) <= 0)
    if cap:
        assert sizes.max() <= cap
    seen = {}
    for g in range(G):
        mem = order[start[g]:start[g + 1]]
        assert np.all(np.diff(mem) > 0)  # batch order inside a unit
        t = tuple(q[mem[0]])
        assert all(tuple(q[i]) == t for i in mem)
        if not cap:
            assert t not in seen
        seen.setdefault(t, []).append(g)
    for s in np.unique(sizes):  # equal-size units: by their tuple's first occurrence, then chunk
        firsts = [min(order[start[h]] for h in seen[tuple(q[order[start[g]]])]) for g in range(G) if sizes[g] == s]
        assert firsts == sorted(firsts)
    if not cap:
        assert G == len({tuple(r) for r in q.tolist()})
    else:
        counts = {}
        for r in q.tolist():
            counts[tuple(r)] = counts.get(tuple(r), 0) + 1
        assert G == sum(-(-c // cap) for c in counts.values())


def test_group_queries():
    """wj_group_queries: identical ordered tuples grouped, first-occurrence
    order, members in batch order; (a, b) and (b, a) are different."""
    import ctypes

    from paper_2202_13538_b200 import _lib

    rng = np.random.default_rng(0)
    for A in (1, 2, 3, 4):
        for n in (1, 7, 500):
            q = rng.integers(0, 6, size=(n, A)).astype(np.int64)
            for cap in (0, 1, 2, 3):
                gb = np.empty((2 + A) * n + 2, np.int32)
                ng = ctypes.c_int64()
                _lib.call("wj_group_queries", q.ctypes.data, n, A, cap, gb.ctypes.data, ctypes.byref(ng))
                assert ng.value == gb[0]
                _check_groups(q, gb, cap)


@pytest.mark.parametrize("name", CASES[:2])
def test_planner_emits_groups(name):
    d = _load(name)
    bp = _planner(d, _rng(d))
    from paper_2202_13538_b200.pipeline import GROUP_MAX

    for q, y, _ in bp.epoch():
        _check_groups(q.numpy(), bp.groups_view.numpy(), GROUP_MAX)
    bp.close()
    bp = _planner(d, _rng(d))
    q, y, _ = bp.next()
    _check_groups(q.numpy(), bp.groups_view.numpy(), GROUP_MAX)


def test_background_build_same_batches():
    """BatchPlanner(background=True) builds on a host thread; the first use
    waits for it and the batches are the same."""
    d = _load(CASES[0])
    from paper_2202_13538_b200.pipeline import BatchPlanner, TrainConfig

    cfg = TrainConfig(batch_capacity=int(d["batch_capacity"]), batch_size=int(d["batch_size"]),
                      k_neg=int(d["k_neg"]), seed=int(d["seed"]))
    filt = np.concatenate([d["positives"], d["filter_extra"]])
    a = BatchPlanner(d["positives"], filt, int(d["num_nodes"]), cfg, _rng(d), pinned=False)
    b = BatchPlanner(d["positives"], filt, int(d["num_nodes"]), cfg, _rng(d), pinned=False, background=True)
    for _ in range(5):
        qa, ya, _ = a.next()
        qb, yb, _ = b.next()
        assert np.array_equal(qa.numpy(), qb.numpy()) and np.array_equal(ya.numpy(), yb.numpy())
    a.close()
    b.close()
