"""The native step executor (``TrainStep(launch="chain")``, wj_stepper_*):
three programmatic-dependent launches per step, consecutive steps chained on
one stream, inputs read in place (device or pinned host memory).  It must
give exactly the graph-mode step's results -- same kernels, same dropout
stream, same fixed-order reductions -- step after step, for varying batch
sizes, and with the loss written straight into pinned host memory."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def store_and_batches():
    import paper_2202_13538_b200 as wj

    rng = np.random.default_rng(5)
    g = wj.Graph.from_edges(rng.integers(0, 3000, size=(30000, 2)), 3000)
    s = wj.preprocess(g, 50, 4, 9)
    batches = []
    for B in (330, 330, 200, 330, 17, 400, 330, 1):
        q = torch.from_numpy(np.stack([rng.choice(3000, 2, replace=False) for _ in range(B)]).astype(np.int64))
        y = torch.from_numpy((rng.random(B) < 0.2).astype(np.float32))
        batches.append((q, y))
    return s, batches


def _run(store, batches, launch, where):
    import paper_2202_13538_b200 as wj

    p = wj.init_params(2, 4, dropout=0.1, seed=3)
    st = wj.AdamState.for_params(p, lr=1e-3)
    step = wj.TrainStep(store, p, st, use_graph=True, seed=77, launch=launch, overlap_inputs=True)
    assert step.launch == launch
    losses = []
    for q, y in batches:
        if where == "device":
            q, y = q.cuda(), y.cuda()
        else:
            q, y = q.pin_memory(), y.pin_memory()
        if launch == "chain" and where == "pinned":
            out = torch.zeros(1, dtype=torch.float32).pin_memory()
            step(q, y, loss_out=out)
            torch.cuda.synchronize()
            losses.append(float(out[0]))
        else:
            losses.append(float(step(q, y)))
    torch.cuda.synchronize()
    return {k: v.detach().clone() for k, v in p.tensors.items()}, losses, int(step.step_t.item())


@pytest.mark.parametrize("kernel", ["mma", "tc"])
@pytest.mark.parametrize("where", ["device", "pinned"])
def test_chain_equals_graph(store_and_batches, where, kernel, monkeypatch):
    if kernel == "tc":  # the tcgen05 join+encode kernel (encode_tc.cu)
        monkeypatch.setenv("WJ_ENC_TC", "8")
    store, batches = store_and_batches
    pg, lg, tg = _run(store, batches, "graph", where)
    pc, lc, tc = _run(store, batches, "chain", where)
    assert tg == tc == len(batches)
    assert lg == lc
    for k in pg:
        assert torch.equal(pg[k], pc[k]), k


@pytest.mark.parametrize("dynamic", [True, False])
def test_chain_back_to_back_without_syncs(store_and_batches, dynamic):
    """Many chained steps enqueued with no host sync in between (the PDL
    chain proper) end in the same parameters as the graph path."""
    import paper_2202_13538_b200 as wj

    store, batches = store_and_batches
    seq = [batches[k % 4] for k in range(40)]
    outs = []
    for launch in ("graph", "chain"):
        p = wj.init_params(2, 4, dropout=0.1, seed=3)
        st = wj.AdamState.for_params(p, lr=1e-3)
        step = wj.TrainStep(store, p, st, use_graph=True, seed=5, launch=launch, overlap_inputs=True)
        step.dynamic_queries = dynamic  # join+encode grabs queries from a counter (chain mode)
        qd = [(q.cuda(), y.cuda()) for q, y in seq]
        torch.cuda.synchronize()
        for q, y in qd:
            step(q, y)
        torch.cuda.synchronize()
        outs.append({k: v.clone() for k, v in p.tensors.items()})
    for k in outs[0]:
        assert torch.equal(outs[0][k], outs[1][k]), k


def test_chain_with_query_groups_is_bit_identical(store_and_batches):
    """Scheduling groups of identical queries (shared staging / merge / rows,
    tiles + reduction per member) gives exactly the ungrouped results; the
    batches repeat tuples as the reference's in-seed negatives do."""
    import ctypes

    import paper_2202_13538_b200 as wj
    from paper_2202_13538_b200 import _lib
    from paper_2202_13538_b200.pipeline import GROUP_MAX

    store, batches = store_and_batches
    rng = np.random.default_rng(9)
    seq = []
    for q, y in batches[:5]:
        qq = q.numpy().copy()
        dup = rng.integers(0, qq.shape[0], size=qq.shape[0] // 2)
        qq[rng.integers(0, qq.shape[0], size=dup.shape[0])] = qq[dup]  # many repeated tuples
        gb = np.empty(4 * qq.shape[0] + 2, np.int32)
        _lib.call("wj_group_queries", qq.ctypes.data, qq.shape[0], 2, GROUP_MAX, gb.ctypes.data, None)
        assert gb[0] < qq.shape[0]
        seq.append((torch.from_numpy(qq).cuda(), y.cuda(), (torch.from_numpy(gb).cuda(), int(gb[0]))))
    outs = []
    for grouped in (False, True):
        p = wj.init_params(2, 4, dropout=0.1, seed=3)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(store, p, st, use_graph=True, seed=5, launch="chain", overlap_inputs=True)
        losses = [float(step(q, y, groups=g if grouped else None)) for q, y, g in seq]
        torch.cuda.synchronize()
        outs.append((losses, {k: v.clone() for k, v in p.tensors.items()}))
    assert outs[0][0] == outs[1][0]
    for k in outs[0][1]:
        assert torch.equal(outs[0][1][k], outs[1][1][k]), k


def test_device_feeder_delivers_the_planner_batches():
    """DeviceFeeder (side-stream H2D one batch ahead, host-checked): the device
    batches equal the planner's, labels are positives-first, the copied unit
    block is the planner's grouping; consumed() gates slot reuse."""
    from paper_2202_13538_b200.pipeline import BatchPlanner, DeviceFeeder, TrainConfig

    rng = np.random.default_rng(2)
    n = 3000
    pos = rng.integers(0, n, size=(4000, 2))
    pos = pos[pos[:, 0] != pos[:, 1]]
    cfg = TrainConfig(batch_size=16, k_neg=10)
    ref = BatchPlanner(pos, pos, n, cfg, np.random.default_rng(4), pinned=False)
    want = []
    for _ in range(12):  # next() returns views into its ring: copy at once
        q, _, p = ref.next()
        want.append((q.numpy().copy(), int(p)))
    bp = BatchPlanner(pos, pos, n, cfg, np.random.default_rng(4), depth=3)
    fd = DeviceFeeder(bp, torch.device("cuda"), depth=2)
    got = []
    for k, (q, y, n_pos) in enumerate(fd.epoch()):
        G = fd.n_groups
        gb = fd.groups[:G + 2 + q.shape[0]].cpu().numpy()
        qq = q.cpu().numpy()
        start, order = gb[1:G + 2], gb[G + 2:]
        for g in range(G):
            mem = order[start[g]:start[g + 1]]
            assert all(tuple(qq[i]) == tuple(qq[mem[0]]) for i in mem)
        yy = y.cpu().numpy()
        assert yy[:n_pos].sum() == n_pos and yy[n_pos:].sum() == 0
        got.append((qq, n_pos))
        fd.consumed()
        if k == 11:
            break
    for (a, pa), (b, pb) in zip(want, got):
        assert np.array_equal(a, b) and pa == pb
    bp.close()


def test_chain_equals_graph_hyperedges():
    """Arity-3 queries (hyperedges, L=3): the step executor with query units
    equals the graph step exactly."""
    import paper_2202_13538_b200 as wj
    from paper_2202_13538_b200 import _lib
    from paper_2202_13538_b200.pipeline import GROUP_MAX

    rng = np.random.default_rng(8)
    g = wj.Graph.from_edges(rng.integers(0, 800, size=(9000, 2)), 800)
    s = wj.preprocess(g, 40, 3, 4)
    seeds = rng.choice(800, 30, replace=False)
    batches = []
    for B in (96, 96, 50):
        q = np.stack([rng.choice(seeds, 3, replace=False) for _ in range(B)]).astype(np.int64)
        gb = np.empty(5 * B + 2, np.int32)
        _lib.call("wj_group_queries", q.ctypes.data, B, 3, GROUP_MAX, gb.ctypes.data, None)
        y = (rng.random(B) < 0.3).astype(np.float32)
        batches.append((torch.from_numpy(q).cuda(), torch.from_numpy(y).cuda(),
                        (torch.from_numpy(gb).cuda(), int(gb[0]))))
    outs = []
    for launch in ("graph", "chain"):
        p = wj.init_params(3, 3, dropout=0.1, seed=2)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(s, p, st, use_graph=True, seed=6, launch=launch, overlap_inputs=True)
        assert step.launch == launch
        losses = [float(step(q, y, groups=gr)) for q, y, gr in batches]
        torch.cuda.synchronize()
        outs.append((losses, {k: v.clone() for k, v in p.tensors.items()}))
    assert outs[0][0] == outs[1][0]
    for k in outs[0][1]:
        assert torch.equal(outs[0][1][k], outs[1][1][k]), k


@pytest.mark.parametrize("max_steps", [-1, 5])
def test_native_epoch_equals_python_loop(max_steps):
    """TrainStep.run_epoch (wj_train_epoch: planner -> H2D -> step executor,
    no Python between steps) == the DeviceFeeder + per-step chain loop: same
    batches, losses and parameters bit for bit, and the planner's generator
    ends in the same state."""
    import paper_2202_13538_b200 as wj
    from paper_2202_13538_b200.pipeline import BatchPlanner, DeviceFeeder, TrainConfig

    rng = np.random.default_rng(11)
    n = 2000
    g = wj.Graph.from_edges(rng.integers(0, n, size=(16000, 2)), n)
    s = wj.preprocess(g, 40, 4, 5)
    pos = np.stack([rng.choice(n, 2, replace=False) for _ in range(700)]).astype(np.int64)
    cfg = TrainConfig(batch_size=16, k_neg=7)
    outs = []
    for native in (False, True):
        planner = BatchPlanner(pos, pos, n, cfg, np.random.default_rng(3), depth=4)
        p = wj.init_params(2, 4, dropout=0.1, seed=9)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(s, p, st, seed=21, launch="chain")
        if native:
            k = step.run_epoch(planner, max_steps=max_steps)
            losses = step.epoch_losses[:k].cpu().tolist()
        else:
            feeder = DeviceFeeder(planner, torch.device("cuda", 0))
            losses = []
            it = feeder.epoch()
            for q, y, _ in it:
                losses.append(float(step(q, y, groups=(feeder.groups, feeder.n_groups))))
                feeder.consumed()
                if max_steps >= 0 and len(losses) == max_steps:
                    break
            it.close()
        torch.cuda.synchronize()
        planner.close()
        outs.append((losses, {k_: v.clone() for k_, v in p.tensors.items()}, int(step.step_t.item()),
                     planner.rng.bit_generator.state["state"]["state"] if max_steps < 0 else None))
    (l0, p0, t0, r0), (l1, p1, t1, r1) = outs
    assert len(l0) == len(l1) > 3 and l0 == l1
    assert t0 == t1 == len(l0)
    assert all(torch.equal(p0[k], p1[k]) for k in p0)
    assert r0 == r1
