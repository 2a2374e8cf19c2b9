"""The multi-GPU code paths executed by TWO ranks (two processes) -- on one
GPU, since a driver box has one: gloo collectives on CUDA tensors stand in
for NCCL (same torch.distributed calls, host-staged).  Checks, bit for bit
against the single-process results:

* ``preprocess_sharded``: node-range shards, the distinct-vector merge and the
  store gathered straight into its full-size buffers (``gather_into``) give
  exactly the single-GPU store;
* batch-sharded data parallel (``TrainStep(dp_mode="shard")``, SURVEY §8(e):
  one reference mini-batch split across the ranks): every rank's losses and
  parameters equal one GPU stepping the whole batch, step after step;
* replicated data parallel (the default, ``dp_mode="replicate"``) with the
  same batch on both ranks: the averaged gradients equal one GPU's.
"""

import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = textwrap.dedent(r"""
    import os, sys
    sys.path.insert(0, os.environ["WJ_ROOT"])
    import numpy as np, torch, torch.distributed as dist
    import paper_2202_13538_b200 as wj
    from paper_2202_13538_b200.distributed import preprocess_sharded

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    out = os.environ["WJ_OUT"]
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    # ---- sharded preprocess == single-process preprocess
    rng = np.random.default_rng(4)
    g = wj.Graph.from_edges(rng.integers(0, 2500, size=(20000, 2)), 2500)
    a = wj.preprocess(g, 30, 3, 77)
    b = preprocess_sharded(g, 30, 3, 77)
    for k in ("walks_d", "offsets_d", "uniq_x_d", "uniq_id_d", "uniq_first_d", "slot_idx_d", "table_keys_d"):
        res["pre_" + k] = bool(torch.equal(getattr(a, k), getattr(b, k)))
    res["pre_dicts"] = bool(np.array_equal(a.dict_vals, b.dict_vals) and np.array_equal(a.dict_keys, b.dict_keys))
    # ---- data parallel steps vs one process stepping the whole batch
    s = wj.preprocess(g, 40, 4, 9)
    batches = []
    for B in (330, 1632, 200, 511):
        q = np.stack([rng.choice(2500, 2, replace=False) for _ in range(B)]).astype(np.int64)
        y = (np.arange(B) % 9 == 0).astype(np.float32)
        batches.append((torch.from_numpy(q).cuda(), torch.from_numpy(y).cuda()))
    runs = {}
    for mode in ("single", "shard", "replicate"):
        p = wj.init_params(2, 4, dropout=0.1, seed=3)
        st = wj.AdamState.for_params(p)
        step = wj.TrainStep(s, p, st, seed=12, launch="chain",
                            process_group=None if mode == "single" else dist.group.WORLD,
                            dp_mode="shard" if mode == "shard" else "replicate")
        losses = [float(step(q, y)) for q, y in batches]
        torch.cuda.synchronize()
        runs[mode] = (losses, {k: v.detach().cpu().clone() for k, v in p.tensors.items()})
    for mode in ("shard", "replicate"):
        res[mode + "_losses"] = runs[mode][0] == runs["single"][0]
        res[mode + "_params"] = all(torch.equal(runs[mode][1][k], runs["single"][1][k]) for k in runs["single"][1])
    res["losses"] = {m: runs[m][0] for m in runs}
    import json
    with open(f"{out}.{rank}.json", "w") as fh:
        json.dump(res, fh)
    dist.destroy_process_group()
""")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def two_rank_results(tmp_path_factory):
    import json

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = tmp_path_factory.mktemp("dist2")
    script = d / "worker.py"
    script.write_text(WORKER)
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   WJ_ROOT=ROOT, WJ_OUT=str(d / "res"))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    logs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        logs.append(out)
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{logs[r][-4000:]}"
    return [json.load(open(d / f"res.{r}.json")) for r in range(2)]


def test_two_rank_sharded_preprocess_equals_single(two_rank_results):
    for r, res in enumerate(two_rank_results):
        bad = [k for k, v in res.items() if k.startswith("pre_") and not v]
        assert not bad, (r, bad)


def test_two_rank_batch_sharded_step_equals_single(two_rank_results):
    for r, res in enumerate(two_rank_results):
        assert res["shard_losses"] and res["shard_params"], (r, res["losses"])


def test_two_rank_replicated_step_equals_single(two_rank_results):
    for r, res in enumerate(two_rank_results):
        assert res["replicate_losses"] and res["replicate_params"], (r, res["losses"])
