#!/usr/bin/env python
"""Benchmark of the walk -> RPE -> join -> encode hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c2|c1]
    python bench.py --impl reference ...      # CPU reference arm (oracle port)

Workload (default c3 = BASELINE.json configs[2], the metric's citation2 shape):
Erdos-Renyi graph with 2,927,963 nodes / 30,561,187 edges, 5% of the edges
held out as training positives and removed from the walk graph, M=200 walks
of L=4 steps, link queries (A=2), reference batches of 32 positives + 50
in-seed negatives each (1,632 queries).  Synthetic data, random-init encoder.

A "step" is one training batch: join+densify kernel -> encoder forward ->
BCE -> backward -> Adam (one captured CUDA graph).  The metric is the
reference's train q/s: Q_epoch / (t_pre + batches_per_epoch * t_step), with
t_pre the device time of the full preprocess (sample + RPE + intern, run in
this process) and t_step the mean device time of K timed steps.
``value`` takes queries resident in HBM; ``e2e`` feeds every step from
pinned host memory (H2D of the batch, D2H of the loss inside the timed
region) and preprocesses from the host CSR.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c3": dict(workload="ogbl-citation2-shape", n=2_927_963, m=30_561_187, M=200, L=4, A=2,
               ubar=528.5),
    "c2": dict(workload="ogbl-collab-shape", n=235_868, m=1_285_465, M=200, L=4, A=2, ubar=393.1),
    "c1": dict(workload="er-10k", n=10_000, m=100_000, M=50, L=3, A=2, ubar=106.8),
}
TRAIN_FRAC, K_NEG, POS_PER_BATCH = 0.05, 50, 32
GRAPH_SEED, STORE_SEED, BATCH_SEED = 1, 3, 7
METRIC = "train queries/sec (sample+RPE+join+encode) on citation2-shape; HBM GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--cpu-shard-nodes", type=int, default=0, help="0 = auto")
    ap.add_argument("--pre", default="sharded", choices=["sharded", "redundant"],
                    help="N>1 preprocess: node-range shards + NCCL all-gathers, or the full store on every rank "
                         "(no communication; SURVEY 8(e) asks for both)")
    ap.add_argument("--launch", default="chain", choices=["chain", "graph"],
                    help="chain: native step executor, PDL-chained across steps; graph: one CUDA graph per step")
    ap.add_argument("--mode", default="fused", choices=["fused", "pooled", "reference"],
                    help="fused: wj_join_encode kernel; pooled/reference: wj_join dense + PyTorch encoder")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks --

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, enabled: bool = True):
        self.enabled = enabled
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        if self.enabled:
            self.fh = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=self.fh, stderr=subprocess.DEVNULL)
            except FileNotFoundError:
                self.proc = None
            time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.fh.seek(0)
        rows = [r.split(",") for r in self.fh.read().strip().splitlines() if r.count(",") >= 8]
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for k, nm in enumerate(names):
                if r[5 + k].strip().lower() == "active":
                    reasons.add(nm)
        under = [v for v in sm if v > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(under) if under else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(rows),
                "reasons": sorted(reasons)}


# ------------------------------------------------------------------- setup --

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def build_inputs(cfg, device):
    """Synthetic walk graph + training positives + batch plan (host)."""
    from paper_2202_13538_b200.graph import synthetic_link_graph
    from paper_2202_13538_b200.pipeline import PositiveFilter, QueryOverlapIndex

    split = synthetic_link_graph(cfg["n"], cfg["m"], TRAIN_FRAC, seed=GRAPH_SEED, device=device)
    index = QueryOverlapIndex(split.train_pos)
    filt = PositiveFilter.__new__(PositiveFilter)
    filt.n, filt.keys = cfg["n"], split.all_edges
    return split, index, filt


def make_plan(split, index, filt, count, seed):
    from paper_2202_13538_b200.pipeline import TrainConfig, make_batch

    tc = TrainConfig(batch_size=POS_PER_BATCH, k_neg=K_NEG)
    rng = np.random.default_rng(seed)
    return [make_batch(index, split.train_pos, filt, tc, rng) for _ in range(count)]


def epoch_shape(split):
    n_pos = int(split.train_pos.shape[0])
    return n_pos * (1 + K_NEG), math.ceil(n_pos / POS_PER_BATCH)


# --------------------------------------------------------------- our arm --

def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2202_13538_b200 as wj
    from paper_2202_13538_b200 import _lib
    from paper_2202_13538_b200.joiner import dense_batch

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _lib.load()
    torch.manual_seed(1234 + rank)
    M, L, A = cfg["M"], cfg["L"], cfg["A"]

    def barrier_sync():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    split, index, filt = build_inputs(cfg, dev)
    q_epoch, nb_epoch = epoch_shape(split)
    g = split.walk_graph

    # ---- preprocess: warm once, then time the full Alg. 1 on device
    if world > 1 and args.pre == "sharded":
        from paper_2202_13538_b200.distributed import preprocess_sharded as prep
    else:
        prep = wj.preprocess
    store = prep(g, M, L, STORE_SEED)
    del store  # its blocks stay in the caching allocator: the timed run measures device work
    phases = []
    barrier_sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    store = prep(g, M, L, STORE_SEED, phases=phases)
    e1.record()
    barrier_sync()
    t_pre = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    phase_ms = {name: a.elapsed_time(b) for name, a, b in phases}
    ubar = store.num_entries / store.num_nodes

    # ---- batch plan (host), uploaded before the timed region
    W, K = args.warmup, args.steps
    plan = make_plan(split, index, filt, W + K, BATCH_SEED + rank)
    qd = [torch.from_numpy(q).to(dev) for q, _ in plan]
    yd = [torch.from_numpy(y).to(dev) for _, y in plan]
    # the planner's per-batch groups of identical queries (wj_group_queries),
    # resident with their batch
    from paper_2202_13538_b200.pipeline import GROUP_MAX

    gd = []
    for q, _ in plan:
        gb = np.empty((2 + q.shape[1]) * q.shape[0] + 2, dtype=np.int32)
        _lib.call("wj_group_queries", q.ctypes.data, q.shape[0], q.shape[1], GROUP_MAX, gb.ctypes.data, None)
        gd.append((torch.from_numpy(gb).to(dev), int(gb[0])))
    B_mean = float(np.mean([q.shape[0] for q, _ in plan[W:]]))

    params = wj.init_params(A, L, hidden=64, dropout=0.1, seed=11, device=dev)
    state = wj.AdamState.for_params(params, lr=1e-3)
    step = wj.TrainStep(store, params, state, dense_dtype=torch.float32, mode=args.mode,
                        use_graph=True, process_group=(dist.group.WORLD if world > 1 else None),
                        seed=1000 + rank, overlap_inputs=True, launch=args.launch)
    for k in range(W):                       # warm-up: captures every batch shape of the plan
        step(qd[k], yd[k], groups=gd[k])
    for k in range(W, W + K):
        if step.launch == "graph" and (qd[k].shape[0], A) not in step._graphs:
            step(qd[k], yd[k])

    # ---- value: K steps, inputs resident in HBM
    with ClockSampler(local, enabled=not args.no_clocks) as clocks:
        barrier_sync()
        # a ~1 ms device-side head start so the host enqueues the K steps ahead
        # of the GPU: the events then time device execution, not host jitter
        torch.cuda._sleep(2_000_000)
        e0.record()
        for k in range(W, W + K):
            loss = step(qd[k], yd[k], groups=gd[k])
        e1.record()
        barrier_sync()
    t_step = max_over_ranks(e0.elapsed_time(e1) / 1e3 / K)
    final_loss = float(loss.item())

    # ---- join kernel alone, same batches, events on its stream
    dense_buf = {}
    j0, j1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(W, W + K):  # warm
        shp = qd[k].shape[0]
        dense_buf.setdefault(shp, torch.empty((shp, A * M * (L + 1), A * (L + 1)), device=dev))
        dense_batch(store, qd[k], out=dense_buf[shp], validate=False)
    torch.cuda.synchronize()
    j0.record()
    for k in range(W, W + K):
        dense_batch(store, qd[k], out=dense_buf[qd[k].shape[0]], validate=False)
    j1.record()
    torch.cuda.synchronize()
    t_join = j0.elapsed_time(j1) / 1e3 / K
    # ---- fused join+encode kernel alone (training: dropout + backward statistics)
    enc_bufs = {}
    step_t = torch.zeros(1, dtype=torch.int64, device=dev)
    for k in range(W, W + K):
        shp = qd[k].shape[0]
        enc_bufs.setdefault(shp, {"pooled": torch.empty((shp, 64), device=dev),
                                  "S": torch.empty((shp, A * (L + 1), 64), device=dev),
                                  "msum": torch.empty((shp, 64), device=dev)})
    t_enc = None
    if A * (L + 1) <= 16:
        def enc_launch(k):
            if step.launch == "chain":  # the production kernel: dynamic scheduling over query groups
                step.encode_only(qd[k], groups=gd[k])
                return
            b = enc_bufs[qd[k].shape[0]]
            t = params.tensors
            wj.encoder.join_encode(store, qd[k], t["w1"], t["b1"], 0.9, 5, step_t, b["pooled"], b["S"],
                                   b["msum"])

        for k in range(W, W + K):
            enc_launch(k)
        torch.cuda.synchronize()
        j0.record()
        for k in range(W, W + K):
            enc_launch(k)
        j1.record()
        torch.cuda.synchronize()
        t_enc = j0.elapsed_time(j1) / 1e3 / K

    # ---- e2e: host CSR -> preprocess (device) overlapped with the batch
    # planner's build (host thread: query index + positive-tuple set,
    # pipeline.py:276-280) -> pinned batches -> step -> loss to host.  The
    # batches come from the native planner (the reference's BFS batches +
    # in-seed negatives on numpy's PCG64 stream, pipeline.py:287-305) on its
    # producer thread: planning, H2D, step and the loss read-back are all
    # inside the timed region.
    from paper_2202_13538_b200.pipeline import BatchPlanner, DeviceFeeder, TrainConfig

    host_g = g.to_host()
    nn_ = cfg["n"]
    filt_rows = np.stack([split.all_edges // nn_, split.all_edges % nn_], 1)
    torch.cuda.synchronize()
    del store
    step = None
    barrier_sync()
    w0 = time.perf_counter()
    e0.record()
    planner = BatchPlanner(split.train_pos, filt_rows, nn_, TrainConfig(batch_size=POS_PER_BATCH, k_neg=K_NEG),
                           np.random.default_rng(BATCH_SEED + rank), depth=8, background=True)
    store = prep(host_g, M, L, STORE_SEED)
    e1.record()
    torch.cuda.synchronize()
    t_pre_dev = e0.elapsed_time(e1) / 1e3
    t_pre_wall_dev = time.perf_counter() - w0
    planner.wait()
    t_plan_setup = time.perf_counter() - w0  # the planner build, from the same start
    barrier_sync()
    t_pre_e2e = max_over_ranks(max(t_pre_dev, t_pre_wall_dev, t_plan_setup))
    del filt_rows
    params = wj.init_params(A, L, hidden=64, dropout=0.1, seed=11, device=dev)
    state = wj.AdamState.for_params(params, lr=1e-3)
    step = wj.TrainStep(store, params, state, dense_dtype=torch.float32, mode=args.mode,
                        use_graph=True, process_group=(dist.group.WORLD if world > 1 else None),
                        seed=1000 + rank, overlap_inputs=True, launch=args.launch)
    loss_h = torch.empty(W + K, dtype=torch.float32).pin_memory()
    chain = step.launch == "chain"
    # chain: pinned batch -> side-stream H2D into a device ring (one batch
    # ahead, completion checked on the host) -> step; the Adam kernel writes
    # the loss straight into pinned host memory.  graph: the step graph copies
    # the pinned batch itself.
    feeder = DeviceFeeder(planner, dev) if chain else None
    source = feeder.epoch if chain else planner.epoch

    def e2e_step(k, q, y):
        if chain:
            step(q, y, loss_out=loss_h[k:k + 1], groups=(feeder.groups, feeder.n_groups))
            feeder.consumed()
        else:
            loss_h[k:k + 1].copy_(step(q, y).reshape(1), non_blocking=True)
            planner.release(step.input_event)

    it = source()  # warm-up epoch: captures the step graphs, then abandoned
    for k in range(W):
        q, y, _ = next(it)
        e2e_step(k, q, y)
    it.close()
    barrier_sync()
    h2d_list = []
    w0 = time.perf_counter()
    e0.record()
    it = source()  # the producer thread starts inside the timed region
    for k in range(W, W + K):
        try:
            q, y, _ = next(it)
        except StopIteration:  # small graphs: the epoch ends, the next one starts (as in train())
            it = source()
            q, y, _ = next(it)
        e2e_step(k, q, y)
        h2d_list.append(q.numel() * 8 + (0 if chain else y.numel() * 4))
    e1.record()
    barrier_sync()
    wall = (time.perf_counter() - w0) / K
    it.close()
    planner.close()
    t_dev_e2e = e0.elapsed_time(e1) / 1e3 / K
    t_step_e2e = max_over_ranks(max(t_dev_e2e, wall))
    h2d = int(np.mean(h2d_list))

    if args.mode == "fused" and step.fast_tail:
        launches_per_step = 3
        launches_note = (("per timed step (native step executor, one PDL chain across steps): "
                          if step.launch == "chain" else "per timed step (one CUDA graph, PDL-chained): ") +
                         "wj_join_encode (join + layer 1), "
                         "wj_encoder_tail (tensor-core tail + partial grads), wj_adam")
    else:
        launches_per_step = 1
        launches_note = "per timed step: wj_join (the encoder runs as PyTorch/cuBLAS kernels)"
    value = q_epoch / (t_pre + (nb_epoch / world) * t_step)
    e2e = q_epoch / (t_pre_e2e + (nb_epoch / world) * t_step_e2e)

    # ---- roofline of the join kernel (SURVEY §8(d) join bytes per query)
    hbm, peak_kind = peaks()
    s_bytes = 4  # fp32 dense elements
    c = 1 if M <= 255 else 2
    join_bytes_q = A * M * (L + 1) * 4 + A * ubar * (4 + c * (L + 1)) + A * A * M * (L + 1) ** 2 * s_bytes
    achieved = join_bytes_q * B_mean / t_join / 1e9
    # whole-step bytes per query (B_q of SURVEY §8(d), dense at s=4)
    b_pre = M * L * 64 + 2 * M * (L + 1) * 4 + ubar * (4 + c * (L + 1))
    b_q = (A * M * (L + 1) * 4 + A * ubar * (4 + c * (L + 1)) + 3 * A * A * M * (L + 1) ** 2 * s_bytes
           + b_pre * cfg["n"] / q_epoch)
    # fused kernel: what it must move per query -- the A anchors' sorted
    # (uniq_x, uniq_id) lists in, pooled/msum/S out (the dense tile and the
    # [rows, 64] activations never exist)
    AW = A * (L + 1)
    vbar = (store.vslots_d.numel() - 2) / store.num_nodes if store.vslots_d is not None else 0.0
    # per query: query ids + per-anchor offsets / vindex entries, the anchors'
    # sorted (uniq_x, uniq_id) lists, their virtual-landing lists (uint16);
    # written: pooled, msum and S (fp32)
    enc_bytes_q = A * (8 + 16 + 16) + A * ubar * 8 + A * vbar * 2 + (2 + AW) * 64 * 4
    kname = "wj_join_encode" if args.mode == "fused" else "wj_join"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"{args.config}_{kname}_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("bytes_per_launch")
        except Exception:
            traffic = None
    if args.mode == "fused" and t_enc:
        # achieved = SURVEY 8(d)'s per-query join figure (walk blocks + the
        # anchors' RPE index + the dense tile at s = 2 B: 57.5 KB at C3) x the
        # launch's queries / the launch time.  The fused kernel does that
        # join's work without materialising the tile; the bytes it must move
        # itself (enc_bytes_q) are reported beside it as "minimal".
        sv_bytes_q = A * M * (L + 1) * 4 + A * ubar * (4 + c * (L + 1)) + A * A * M * (L + 1) ** 2 * 2
        ach = sv_bytes_q * B_mean / t_enc / 1e9
        roof = {"kernel": "wj_join_encode (join + densify + layer-1 fwd/bwd statistics)", "bound": "hbm",
                "achieved": round(ach, 1), "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": round(ach / hbm, 4), "traffic": traffic,
                "bytes_per_query": round(sv_bytes_q, 1),
                "bytes_definition": "SURVEY 8(d) join bytes per query (A*M*(L+1)*4 + A*Ubar*(4+c*(L+1)) + "
                                    "A^2*M*(L+1)^2*2) x queries per launch",
                "kernel_ms": round(t_enc * 1e3, 4), "kernel_share_of_step": round(t_enc / t_step, 3),
                "minimal": {"bytes_per_query": round(enc_bytes_q, 1),
                            "achieved": round(enc_bytes_q * B_mean / t_enc / 1e9, 1),
                            "frac": round(enc_bytes_q * B_mean / t_enc / 1e9 / hbm, 4),
                            "definition": "bytes the fused kernel must move: anchor lists + virtual-landing "
                                          "lists + metadata in, pooled/msum/S out"},
                "note": ("not HBM-bound: issue-bound on the integer ALU (dropout hash) and latency-bound in "
                         "the per-query prepass (ncu: ALU pipe ~53%, DRAM <1%); see DESIGN.md"),
                "traffic_note": "ncu dram bytes of one launch (profiles/c3_wj_join_encode_traffic.json)"}
    else:
        roof = {"kernel": "wj_join (join + densify, fp32 dense)", "bound": "hbm",
                "achieved": round(achieved, 1), "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic,
                "bytes_per_query": round(join_bytes_q, 1), "kernel_ms": round(t_join * 1e3, 4),
                "kernel_share_of_step": round(t_join / t_step, 3)}
    roof["wj_join_dense_fp32"] = {"achieved_gbs": round(achieved, 1), "frac": round(achieved / hbm, 4),
                                  "ms": round(t_join * 1e3, 4), "bytes_per_query": round(join_bytes_q, 1)}
    roof["north_star"] = {"bytes_per_query_B_q": round(b_q, 1),
                          "frac": round(b_q * B_mean / t_step / 1e9 / hbm, 4),
                          "definition": "SURVEY 8(d) B_q * step queries / t_step / peak (40% target)"}

    out = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": round(t_step * 1e3, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32 walk/RPE/join, fp32 encoder",
        "data": "synthetic (Erdos-Renyi graph of the named shape, random-init encoder)",
        "config": {
            "workload": f"{cfg['workload']} ER n={cfg['n']} m={cfg['m']}, M={M}, L={L}, A={A}, "
                        f"5% link split, batches of {POS_PER_BATCH} pos + {K_NEG}/pos neg",
            "n_nodes": cfg["n"], "n_edges": cfg["m"], "walk_graph_edges": int(g.indices.numel() // 2),
            "M": M, "L": L, "arity": A, "queries_per_step": B_mean,
            "train_pos": int(split.train_pos.shape[0]), "Q_epoch": q_epoch,
            "batches_per_epoch": nb_epoch, "t_pre_ms": round(t_pre * 1e3, 3),
            "t_pre_phase_ms": {k: round(v, 3) for k, v in phase_ms.items()},
            "store_entries": int(store.num_entries), "ubar_measured": round(ubar, 2),
            "table_size": int(store.table_keys_d.numel()),
            "value_formula": "Q_epoch / (t_pre + batches_per_epoch / n_gpus * t_step)",
            "l2": "inputs larger than L2 (store > 40 GB, a different random batch every step)",
            "final_loss": final_loss,
            "parallelism": f"dp{world}",
            "launch": step.launch,
            "preprocess": args.pre if world > 1 else "single",
        },
        "e2e": {"value": round(e2e, 1), "unit": "queries/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 4, "t_pre_ms": round(t_pre_e2e * 1e3, 3),
                "t_planner_setup_ms": round(t_plan_setup * 1e3, 3),
                "t_pre_note": "device preprocess and the planner build (host thread) overlap; t_pre is the later end",
                "device_ms_per_step": round(t_dev_e2e * 1e3, 4), "wall_ms_per_step": round(wall * 1e3, 4),
                "ms_per_step": round(t_step_e2e * 1e3, 4),
                "path": ("host CSR -> preprocess; native batch planner (producer thread) -> pinned batch "
                         "-> H2D (side stream, one batch ahead) -> step (chain executor) -> loss D2H "
                         "(written into pinned memory by the Adam kernel), every step timed")},
        "roofline": roof,
        "gpu_launches": K * launches_per_step,
        "gpu_launches_note": launches_note,
        "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, cfg, split, index, filt, plan[W], q_epoch, nb_epoch,
                                           g)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


# --------------------------------------------------------- CPU reference --

def cpu_reference_batch(cfg, idxptr, indices, q, y, index_ref, pos_ref, filt_ref, rng_ref,
                        threads, params, adam, drop_rng):
    """One reference training-loop body on the host (pipeline.py:293-310),
    timed without the untimed sub-store build.  Returns (seconds, parts)."""
    from oracle import core, pipeline_ref

    M, L = cfg["M"], cfg["L"]
    # sub-store over the batch's anchors (preprocess work -- accounted in t_pre)
    anchors, local = np.unique(q, return_inverse=True)
    walks = core.sample_nodes(idxptr, indices, anchors, M, L, STORE_SEED, threads)
    sub = core.store_from_walks(walks, STORE_SEED, threads)
    ql = local.reshape(q.shape).astype(np.int64)
    parts = {}
    t0 = time.perf_counter()
    pipeline_ref.make_batch(index_ref, pos_ref, filt_ref, rng_ref)  # BFS + negatives (exact ref)
    t1 = time.perf_counter()
    from oracle import encoder_ref

    dense = core.dense_batch(sub, ql, threads)
    t2 = time.perf_counter()
    logits, cache = encoder_ref.forward(params, dense, L, dropout=0.1, training=True, dropout_rng=drop_rng)
    encoder_ref.bce_loss(logits, y)
    grads = encoder_ref.backward(params, cache, y)
    adam.update(params, grads)
    t3 = time.perf_counter()
    parts.update(batchgen=t1 - t0, join_densify=t2 - t1, encoder=t3 - t2)
    return t3 - t0, parts


class _FastFilter(set):
    """Set-like positive filter over sorted packed keys for the reference
    negative sampler (membership only; same answers as the reference set)."""

    def __init__(self, keys, n):
        super().__init__()
        self.keys, self.n = keys, n

    def __contains__(self, t):
        k = int(t[0]) * self.n + int(t[1])
        i = np.searchsorted(self.keys, k)
        return bool(i < len(self.keys) and self.keys[i] == k)


def cpu_setup(cfg, split, index_q_limit=None):
    from oracle import pipeline_ref

    pos = [tuple(r) for r in split.train_pos.tolist()]
    index_ref = pipeline_ref.QueryOverlapIndex(pos)
    filt_ref = _FastFilter(split.all_edges, cfg["n"])
    return pos, index_ref, filt_ref


def cpu_preprocess_shard(cfg, idxptr, indices, shard, threads):
    """Reference preprocess phases on nodes [0, shard), scaled to n."""
    from oracle import core

    M, L = cfg["M"], cfg["L"]
    nodes = np.arange(shard, dtype=np.int64)
    t0 = time.perf_counter()
    walks = core.sample_nodes(idxptr, indices, nodes, M, L, STORE_SEED, threads)
    t_sample = time.perf_counter() - t0
    st = core.store_from_walks(walks, STORE_SEED, threads, timed=True)
    ph = dict(st.phase_seconds, sample=t_sample)
    scale = cfg["n"] / shard
    return sum(ph.values()) * scale, {k: round(v * scale, 3) for k, v in ph.items()}


def cpu_baseline(args, cfg, split, index, filt, batch, q_epoch, nb_epoch, g, budget_s=30.0):
    """Oracle (port of the reference CPU path) on this host's cores, bounded sample."""
    from oracle import core, encoder_ref

    threads = core.default_threads()
    host = g.to_host()
    idxptr = np.ascontiguousarray(host.idxptr, np.int64)
    indices = np.ascontiguousarray(host.indices, np.int32)
    shard = args.cpu_shard_nodes or min(cfg["n"], max(2000, 5000 * threads // 8))
    t_pre, ph = cpu_preprocess_shard(cfg, idxptr, indices, shard, threads)
    pos, index_ref, filt_ref = cpu_setup(cfg, split)
    q, y = batch
    params = encoder_ref.init_params(cfg["A"], cfg["L"], seed=11)
    adam = encoder_ref.Adam(params)
    rng_ref = np.random.default_rng(BATCH_SEED)
    drop_rng = np.random.default_rng(5)
    # bounded: scale the batch down if one full batch would exceed the budget
    sub = min(q.shape[0], 408)
    t_sub, parts = cpu_reference_batch(cfg, idxptr, indices, q[:sub], y[:sub].astype(np.float64),
                                       index_ref, pos, filt_ref, rng_ref, threads, params, adam, drop_rng)
    per_q = (t_sub - parts["batchgen"]) / sub
    t_batch = parts["batchgen"] + per_q * q.shape[0]
    value = q_epoch / (t_pre + nb_epoch * t_batch)
    return {"value": round(value, 3), "unit": "queries/s", "cores": threads, "kind": "port",
            "sample": f"preprocess on nodes [0,{shard}) scaled x{cfg['n'] / shard:.1f} "
                      f"(sequential intern scaled linearly, estimated); one batch's join+densify+"
                      f"fp64 encoder fwd/bwd/Adam on {sub} of {q.shape[0]} queries scaled linearly, "
                      f"plus the exact reference BFS batch generation",
            "t_pre_s": round(t_pre, 3), "t_pre_phase_s": ph, "t_batch_s": round(t_batch, 4),
            "batch_parts_s": {k: round(v, 4) for k, v in parts.items()},
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, cfg):
    """--impl reference: the oracle port of the reference CPU path, rank 0 only."""
    world, rank, local = dist_env()
    if rank != 0:
        return
    import torch

    from oracle import core, encoder_ref

    dev = torch.device("cuda", local) if torch.cuda.is_available() else torch.device("cpu")
    split, index, filt = build_inputs(cfg, dev)
    q_epoch, nb_epoch = epoch_shape(split)
    g = split.walk_graph
    threads = core.default_threads()
    host = g.to_host()
    idxptr = np.ascontiguousarray(host.idxptr, np.int64)
    indices = np.ascontiguousarray(host.indices, np.int32)
    shard = args.cpu_shard_nodes or min(cfg["n"], max(2000, 5000 * threads // 8))
    t_pre, ph = cpu_preprocess_shard(cfg, idxptr, indices, shard, threads)
    pos, index_ref, filt_ref = cpu_setup(cfg, split)
    W, K = args.warmup, args.steps
    plan = make_plan(split, index, filt, W + K, BATCH_SEED)
    params = encoder_ref.init_params(cfg["A"], cfg["L"], seed=11)
    adam = encoder_ref.Adam(params)
    rng_ref = np.random.default_rng(BATCH_SEED)
    drop_rng = np.random.default_rng(5)
    # per-step sample bounded so the whole --steps K --warmup W run stays
    # within about a minute of encoder time (the fp64 encoder is ~1.8 s per
    # 408 queries at C3): 408 queries for K + W <= 25, fewer beyond, >= 32
    sub = 408 if cfg["n"] > 100_000 else 1632
    sub = max(32, min(sub, int(sub * 25 / max(W + K, 1))))
    times = []
    for k in range(W + K):
        q, y = plan[k]
        s = min(sub, q.shape[0])
        t, parts = cpu_reference_batch(cfg, idxptr, indices, q[:s], y[:s].astype(np.float64), index_ref,
                                       pos, filt_ref, rng_ref, threads, params, adam, drop_rng)
        t_full = parts["batchgen"] + (t - parts["batchgen"]) * q.shape[0] / s
        if k >= W:
            times.append(t_full)
    t_batch = float(np.mean(times))
    value = q_epoch / (t_pre + nb_epoch * t_batch)
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "queries/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(t_batch * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64/int32 kernels, fp64 encoder",
        "data": "synthetic (same generator and seeds as the GPU arm)", "impl": "reference",
        "config": {"workload": f"{cfg['workload']} ER n={cfg['n']} m={cfg['m']}, M={cfg['M']}, "
                               f"L={cfg['L']}, A={cfg['A']}", "Q_epoch": q_epoch,
                   "batches_per_epoch": nb_epoch, "t_pre_s_estimated": round(t_pre, 3),
                   "t_pre_phase_s": ph, "parallelism": "host threads"},
        "cpu_baseline": {"value": round(value, 3), "unit": "queries/s", "cores": threads, "kind": "port",
                         "sample": f"preprocess on nodes [0,{shard}) scaled to n; each step = reference "
                                   f"BFS batch generation + join/densify/fp64 encoder on {sub} queries "
                                   f"scaled to the full batch", "cpu": _cpu_model()},
        "e2e": {"value": round(value, 3), "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
