"""The data-parallel path on a real NCCL communicator (world size 1: the
driver's GPU box has one GPU per call).  Exercises every NCCL call the
multi-GPU bench makes -- the sharded preprocess exchanges and the all-reduce
captured inside the fused training step's CUDA graph -- and checks that they
reproduce the single-process results bit for bit (the mean over one rank is
the identity; the local partial reduction uses the same fixed order)."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


def test_sharded_preprocess_equals_single(nccl_group):
    import paper_2202_13538_b200 as wj
    from paper_2202_13538_b200.distributed import preprocess_sharded

    rng = np.random.default_rng(4)
    g = wj.Graph.from_edges(rng.integers(0, 2000, size=(16000, 2)), 2000)
    a = wj.preprocess(g, 30, 3, 77)
    b = preprocess_sharded(g, 30, 3, 77, group=nccl_group)
    for k in ("walks_d", "offsets_d", "uniq_x_d", "uniq_id_d", "table_keys_d"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    assert np.array_equal(a.dict_vals, b.dict_vals)


@pytest.mark.parametrize("launch", ["graph", "chain"])
def test_dp_fused_step_equals_single(nccl_group, launch):
    """graph: the all-reduce is captured in the step graph; chain: the step
    executor split around it (wj_stepper_grads -> NCCL average ->
    wj_stepper_apply)."""
    import paper_2202_13538_b200 as wj

    rng = np.random.default_rng(5)
    g = wj.Graph.from_edges(rng.integers(0, 3000, size=(30000, 2)), 3000)
    s = wj.preprocess(g, 50, 4, 9)
    q = torch.from_numpy(np.stack([rng.choice(3000, 2, replace=False) for _ in range(330)])).cuda()
    y = torch.from_numpy((np.arange(330) % 11 == 0).astype(np.float32)).cuda()
    out = []
    for group in (None, nccl_group):
        p = wj.init_params(2, 4, dropout=0.1, seed=3)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(s, p, st, mode="fused", seed=12, use_graph=True, process_group=group, launch=launch)
        assert step.fast_tail and step.launch == launch
        losses = [float(step(q, y)) for _ in range(4)]
        out.append((losses, {k: v.clone() for k, v in p.tensors.items()}))
    assert out[0][0] == out[1][0]
    for k in out[0][1]:
        assert torch.equal(out[0][1][k], out[1][1][k]), k
