"""The encoder that consumes the joined RPE tensor, in PyTorch on the device.

Reference: /root/reference/pkg/src/walkjoin/encoder.py (float64 numpy MLP
with hand-written backprop).  Architecture, init, loss and Adam are the
reference's; the math is re-expressed for the GPU:

* ``mode="reference"`` follows the reference op order literally
  (x@W1+b1 -> ReLU -> dropout -> @W2+b2 -> mean over steps -> mean over
  walks -> classifier), fp32 or fp64.
* ``mode="pooled"`` (default) uses the exact identity that the row mean
  commutes with the affine W2 layer (encoder.py:159-161): hq = mean_rows(a1)
  @ W2 + b2, with the row mean accumulated in fp64.  Backward needs only the
  per-query column scale g_b = dhq_b @ W2^T / rows, so no [rows, hidden]
  gradient of W2 is ever formed.

Dropout masks are drawn from a torch generator, not numpy PCG64, so training
trajectories match the reference statistically, not bitwise.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

TENSOR_ORDER = ("w1", "b1", "w2", "b2", "u1", "c1", "u2", "c2")


@dataclass
class ModelParams:
    """Weights of the step encoder and classifier (encoder.py:32-63), device tensors."""

    arity: int
    walk_steps: int
    hidden: int
    feature_dim: int
    dropout: float
    tensors: dict
    version: int = 0

    @property
    def d_in(self) -> int:
        return self.arity * (self.walk_steps + 1) + self.feature_dim

    def __getattr__(self, name):
        if name in TENSOR_ORDER:
            return self.__dict__["tensors"][name]
        raise AttributeError(name)

    def copy(self) -> "ModelParams":
        return ModelParams(self.arity, self.walk_steps, self.hidden, self.feature_dim, self.dropout,
                           {k: v.clone() for k, v in self.tensors.items()}, self.version)

    def numpy(self) -> dict:
        return {k: v.detach().double().cpu().numpy() for k, v in self.tensors.items()}


def _glorot(rng, fan_in, fan_out):
    a = math.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-a, a, size=(fan_in, fan_out))


def init_params(arity, walk_steps, hidden=64, feature_dim=0, dropout=0.1, seed=0,
                device="cuda", dtype=torch.float32) -> ModelParams:
    """Seeded glorot-uniform weights, zero biases -- same draws as encoder.py:87-117."""
    rng = np.random.default_rng(seed)
    d_in = arity * (walk_steps + 1) + feature_dim
    host = {
        "w1": _glorot(rng, d_in, hidden), "b1": np.zeros(hidden),
        "w2": _glorot(rng, hidden, hidden), "b2": np.zeros(hidden),
        "u1": _glorot(rng, hidden, hidden), "c1": np.zeros(hidden),
        "u2": _glorot(rng, hidden, 1)[:, 0], "c2": np.zeros(1),
    }
    return ModelParams(arity, walk_steps, hidden, feature_dim, dropout,
                       {k: torch.tensor(v, dtype=dtype, device=device) for k, v in host.items()})


def flatten_params(p: ModelParams) -> tuple:
    """Move the parameters into one flat fp32 buffer (TENSOR_ORDER) and make
    ``p.tensors`` views of it.  Returns (flat, host int32 offsets
    [w1, b1, w2, b2, u1, c1, u2, c2, total]) for the tail / Adam kernels."""
    sizes = [p.tensors[k].numel() for k in TENSOR_ORDER]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    flat = torch.cat([p.tensors[k].reshape(-1).to(torch.float32) for k in TENSOR_ORDER])
    for k, o, n in zip(TENSOR_ORDER, offs[:-1], sizes):
        p.tensors[k] = flat[o: o + n].view(p.tensors[k].shape)
    return flat, offs


def params_from_numpy(arrays: dict, arity, walk_steps, dropout=0.0, device="cuda",
                      dtype=torch.float32) -> ModelParams:
    t = {k: torch.tensor(np.asarray(arrays[k]), dtype=dtype, device=device) for k in TENSOR_ORDER}
    hidden = t["w1"].shape[1]
    feature_dim = t["w1"].shape[0] - arity * (walk_steps + 1)
    return ModelParams(arity, walk_steps, hidden, feature_dim, dropout, t)


def dropout_mask(shape, keep: float, generator, device, dtype):
    """Inverted-dropout mask {0, 1/keep} (encoder.py:157)."""
    return (torch.rand(shape, generator=generator, device=device) < keep).to(dtype) / keep


def forward(p: ModelParams, dense: torch.Tensor, training: bool = False,
            generator: Optional[torch.Generator] = None, mode: str = "pooled",
            drop_mask: Optional[torch.Tensor] = None):
    """[B, rows, d_in] -> ([B] logits, cache) (encoder.py:126-180)."""
    x = dense if dense.dim() == 3 else dense[None]
    B, rows, d_in = x.shape
    if d_in != p.d_in:
        raise ValueError(f"input width {d_in} does not match model d_in {p.d_in}")
    width = p.walk_steps + 1
    if rows % width != 0:
        raise ValueError(f"row count {rows} is not a multiple of m+1 = {width}")
    t = p.tensors
    dt = t["w1"].dtype
    flat = x.reshape(B * rows, d_in)
    if flat.dtype != dt:
        flat = flat.to(dt)
    z1 = torch.addmm(t["b1"], flat, t["w1"])
    relu1 = z1 > 0
    a1 = torch.relu_(z1)
    mask = drop_mask
    if mask is None and training and p.dropout > 0.0:
        mask = dropout_mask(a1.shape, 1.0 - p.dropout, generator, a1.device, dt)
    if mask is not None:
        a1.mul_(mask.reshape(a1.shape))
    if mode == "reference":
        e = torch.addmm(t["b2"], a1, t["w2"])
        walk_enc = e.reshape(B, rows // width, width, p.hidden).mean(dim=2)
        hq = walk_enc.to(torch.float64).mean(dim=1).to(dt)
        pooled = None
    else:
        pooled = a1.reshape(B, rows, p.hidden).sum(dim=1, dtype=torch.float64).div_(rows).to(dt)
        hq = torch.addmm(t["b2"], pooled, t["w2"])
    z2 = torch.addmm(t["c1"], hq, t["u1"])
    relu2 = z2 > 0
    a2 = torch.relu(z2)
    logits = a2 @ t["u2"] + t["c2"][0]
    cache = dict(x=flat, relu1=relu1, mask=mask, a1d=a1, pooled=pooled, hq=hq, relu2=relu2, a2=a2,
                 logits=logits, rows=rows, B=B, mode=mode, version=p.version)
    return logits, cache


def join_cross(store, q: torch.Tensor, out: Optional[torch.Tensor] = None) -> Optional[torch.Tensor]:
    """Cross RPE ids of every distinct landing of every query anchor
    (wj_join_cross): [B, A, A-1, max_unique] int32, or None for A = 1."""
    from . import _lib

    B, A = q.shape
    if A < 2:
        return None
    mu = max(store.max_unique, 1)
    if out is None:
        out = torch.empty((B, A, A - 1, mu), dtype=torch.int32, device=store.device)
    _lib.call("wj_join_cross", _lib.ptr(q), B, A, _lib.ptr(store.offsets_d), _lib.ptr(store.uniq_x_d),
              _lib.ptr(store.uniq_id_d), mu, _lib.ptr(out), _lib.stream_handle(store.device))
    return out


def join_encode(store, q: torch.Tensor, w1: torch.Tensor, b1: torch.Tensor, keep: float, seed: int,
                step: Optional[torch.Tensor], pooled: torch.Tensor, S: Optional[torch.Tensor] = None,
                msum: Optional[torch.Tensor] = None, simt: bool = False,
                cross: Optional[torch.Tensor] = None) -> None:
    """One wj_join_encode launch (wj_join_encode_simt with ``simt``) on the
    current stream; see include/walkjoin_b200.h for the outputs.  ``cross``
    (from join_cross) lets the tensor-core kernel skip its list searches."""
    from . import _lib

    B, A = q.shape
    args = (_lib.ptr(q), B, A, _lib.ptr(store.offsets_d), _lib.ptr(store.uniq_x_d), _lib.ptr(store.uniq_id_d))
    tail = (store.num_walks, store.walk_steps, store.max_unique, _lib.ptr(store.table_keys_d),
            int(store.table_keys_d.numel()), _lib.ptr(w1), _lib.ptr(b1), int(w1.shape[1]), float(keep),
            int(seed) & ((1 << 64) - 1), _lib.ptr(step), _lib.ptr(pooled), _lib.ptr(S), _lib.ptr(msum),
            _lib.stream_handle(store.device))
    if simt:
        _lib.call("wj_join_encode_simt", *args, *tail)
    else:
        _lib.call("wj_join_encode", *args, _lib.ptr(cross), *store.vindex_ptrs(), *tail)


def score_shared(store, q: torch.Tensor, w1: torch.Tensor, b1: torch.Tensor, pooled: torch.Tensor,
                 S: Optional[torch.Tensor] = None, msum: Optional[torch.Tensor] = None) -> None:
    """One wj_score_shared launch: keep = 1 scoring of a batch whose queries
    come in runs of equal first anchors (a positive and its negatives); the
    same pooled / S / msum as ``join_encode(..., keep=1.0)``, bit for bit."""
    from . import _lib

    _lib.call("wj_score_shared", _lib.ptr(q), q.shape[0], _lib.ptr(store.offsets_d), _lib.ptr(store.uniq_x_d),
              _lib.ptr(store.uniq_id_d), _lib.ptr(store.trow_d), store.num_walks, store.walk_steps,
              store.max_unique, _lib.ptr(w1), _lib.ptr(b1), _lib.ptr(pooled), _lib.ptr(S), _lib.ptr(msum),
              _lib.stream_handle(store.device))


def fused_supported(p: ModelParams, store) -> bool:
    """True when wj_join_encode (tensor-core or SIMT kernel) accepts this
    model / store shape: RPE-only fp32 models whose (arity, L+1, hidden,
    max_unique) fall inside an instantiated kernel.  Probed once per (store,
    arity, hidden) with an empty batch, which runs the library's own envelope
    checks; callers route other shapes to dense_batch + ``forward``."""
    if p.feature_dim or p.w1.dtype != torch.float32:
        return False
    cache = store.__dict__.setdefault("_fused_ok", {})
    key = (p.arity, p.hidden)
    if key not in cache:
        if store.voff_d is None:
            store.build_vindex()
        t = p.tensors
        q = torch.empty((0, p.arity), dtype=torch.int64, device=store.device)
        pooled = torch.empty((1, p.hidden), dtype=torch.float32, device=store.device)
        try:
            join_encode(store, q, t["w1"], t["b1"], 1.0, 0, None, pooled)
            cache[key] = True
        except NotImplementedError:
            cache[key] = False
    return cache[key]


TAIL_AW = (2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 14, 15, 16)  # A*(L+1) instantiated by wj_encoder_tail


class FusedScorer:
    """Scoring without dropout or gradients, two kernels per chunk:
    wj_join_encode at keep = 1 (its no-dropout variant: distinct landings
    weighted by their row counts, no random stream, no S / msum output) ->
    wj_encoder_tail in logits mode (W2 layer, classifier).  Replaces
    pipeline._score_array's _dense_batch -> forward(training=False)
    (pipeline.py:185-198, encoder.py:126-180).  Needs hidden = 64 and an
    instantiated A*(L+1); the parameters are copied into one flat buffer at
    construction (call ``refresh()`` after they change)."""

    def __init__(self, p: ModelParams, store):
        import ctypes

        if not (fused_supported(p, store) and p.hidden == 64 and p.arity * store.width in TAIL_AW):
            raise NotImplementedError("fused scoring needs an RPE-only fp32 model with hidden = 64")
        self.p, self.store = p, store
        sizes = [p.tensors[k].numel() for k in TENSOR_ORDER]
        self.offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
        self.offs_c = (ctypes.c_int32 * 9)(*[int(x) for x in self.offs])
        self.flat = torch.empty(int(self.offs[-1]), dtype=torch.float32, device=store.device)
        self.refresh()
        self._bufs = {}

    def use_shared_runs(self, B: int, runs: Optional[int]) -> bool:
        """wj_score_shared when the B queries come in long runs (``runs`` of
        them) of equal first anchors (arity 2, L + 1 <= 7; WJ_SCORE_SHARED=0/1
        forces it off / on); ``runs`` None: count them on the device."""

        env = os.environ.get("WJ_SCORE_SHARED")
        ok = self.p.arity == 2 and self.store.width <= 7 and self.store.trow_d is not None
        if env is not None:
            return env == "1" and ok
        return ok and B >= 1024 and runs is not None and runs * 32 <= B

    def _use_shared(self, q: torch.Tensor) -> bool:
        B = q.shape[0]
        if not self.use_shared_runs(B, 0):  # decided without the run count: no device read
            return False
        if "WJ_SCORE_SHARED" in os.environ:
            return True
        return self.use_shared_runs(B, 1 + int((q[1:, 0] != q[:-1, 0]).sum()))

    def refresh(self) -> None:
        torch.cat([self.p.tensors[k].reshape(-1).to(torch.float32) for k in TENSOR_ORDER], out=self.flat)
        self.version = getattr(self.p, "version", 0)

    def logits(self, q: torch.Tensor, shared: Optional[bool] = None) -> torch.Tensor:
        """q [B, A] int64 on the store's device (ids already validated);
        ``shared``: the scoring kernel if the caller already chose it."""
        from . import _lib

        B, A = q.shape
        dev = self.store.device
        buf = self._bufs.get(B)
        if buf is None:
            buf = (torch.empty((B, 64), dtype=torch.float32, device=dev),
                   torch.empty(B, dtype=torch.float32, device=dev))
            self._bufs = {B: buf}
        pooled, logits = buf
        t = self.p.tensors
        if shared is None:
            shared = self._use_shared(q)
        if shared:  # runs of equal first anchors: u's part once per run
            score_shared(self.store, q, t["w1"], t["b1"], pooled)
        else:
            join_encode(self.store, q, t["w1"], t["b1"], 1.0, 0, None, pooled)
        scale = 1.0 / (A * self.store.landings)
        _lib.call("wj_encoder_tail", _lib.ptr(pooled), None, None, None, B, A * self.store.width, 64,
                  _lib.ptr(self.flat), self.offs_c, scale, _lib.ptr(logits), None, 0, None, None,
                  _lib.stream_handle(dev))
        return logits


def forward_fused(p: ModelParams, store, q: torch.Tensor, training: bool = False, seed: int = 0,
                  step: Optional[torch.Tensor] = None, need_grad: bool = True, out: dict = None,
                  tail: bool = True):
    """Encoder forward straight from query ids: the wj_join_encode kernel
    joins, densifies and applies layer 1 (+ReLU, dropout, row mean and the
    backward statistics) per query; the [B, 64]-sized rest runs in PyTorch.
    Same math as ``forward`` (mode="pooled"); see csrc/encode.cu."""
    from . import _lib

    if p.feature_dim:
        raise NotImplementedError("fused encoder takes RPE inputs only (use dense_batch + forward)")
    if p.w1.dtype != torch.float32:
        raise NotImplementedError("fused encoder computes in fp32")
    B, A = q.shape
    if A != p.arity:
        raise ValueError(f"queries have arity {A} but model was trained with arity {p.arity}")
    W = store.width
    H, AW = p.hidden, A * W
    dev = store.device
    rows = A * store.landings
    keep = (1.0 - p.dropout) if (training and p.dropout > 0.0) else 1.0
    o = out if out is not None else {}
    pooled = o.get("pooled")
    if pooled is None:
        pooled = torch.empty((B, H), dtype=torch.float32, device=dev)
    S = msum = None
    if need_grad:
        S = o.get("S")
        msum = o.get("msum")
        if S is None:
            S = torch.empty((B, AW, H), dtype=torch.float32, device=dev)
            msum = torch.empty((B, H), dtype=torch.float32, device=dev)
    t = p.tensors
    join_encode(store, q, t["w1"], t["b1"], keep, seed, step, pooled, S, msum, cross=o.get("cross"))
    if not tail:
        return None, None
    pooled_mean = pooled / (keep * rows)
    hq = torch.addmm(t["b2"], pooled_mean, t["w2"])
    z2 = torch.addmm(t["c1"], hq, t["u1"])
    relu2 = z2 > 0
    a2 = torch.relu(z2)
    logits = a2 @ t["u2"] + t["c2"][0]
    cache = dict(pooled=pooled_mean, S=S, msum=msum, keep=keep, hq=hq, relu2=relu2, a2=a2,
                 logits=logits, rows=rows, B=B, mode="fused", version=p.version)
    return logits, cache


def bce_loss(logits: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
    """Numerically stable mean BCE on the logit scale (encoder.py:183-188)."""
    z = logits
    return (torch.clamp_min(z, 0) - z * labels + torch.log1p(torch.exp(-z.abs()))).mean()


def backward(p: ModelParams, cache: dict, labels: torch.Tensor) -> dict:
    """Gradients of the mean BCE (encoder.py:200-233)."""
    if cache["version"] != p.version:
        raise ValueError("stale cache: params were updated after this forward pass")
    t = p.tensors
    logits = cache["logits"]
    B, rows = cache["B"], cache["rows"]
    y = labels.to(logits.dtype)
    dlogit = (torch.sigmoid(logits) - y) / B
    dc2 = dlogit.sum().reshape(1)
    du2 = cache["a2"].t() @ dlogit
    dz2 = torch.outer(dlogit, t["u2"]) * cache["relu2"]
    dc1 = dz2.sum(0)
    du1 = cache["hq"].t() @ dz2
    dhq = dz2 @ t["u1"].t()
    db2 = dhq.sum(0)
    if cache["mode"] == "fused":
        dw2 = cache["pooled"].t() @ dhq
        g = (dhq @ t["w2"].t()) / (rows * cache["keep"])      # [B, h]
        dw1 = torch.einsum("bch,bh->ch", cache["S"], g)
        db1 = (cache["msum"] * g).sum(0)
        return {"w1": dw1, "b1": db1, "w2": dw2, "b2": db2, "u1": du1, "c1": dc1, "u2": du2, "c2": dc2}
    if cache["mode"] == "reference":
        de = (dhq / rows).repeat_interleave(rows, dim=0)
        dw2 = cache["a1d"].t() @ de
        da1 = de @ t["w2"].t()
    else:
        dw2 = cache["pooled"].t() @ dhq
        g = (dhq @ t["w2"].t()) / rows                       # [B, h], same for every row of b
        da1 = g[:, None, :].expand(B, rows, p.hidden).reshape(B * rows, p.hidden)
    dz1 = da1 * cache["relu1"]
    if cache["mask"] is not None:
        dz1 = dz1 * cache["mask"].reshape(dz1.shape)
    db1 = dz1.sum(0)
    dw1 = cache["x"].t() @ dz1
    return {"w1": dw1, "b1": db1, "w2": dw2, "b2": db2, "u1": du1, "c1": dc1, "u2": du2, "c2": dc2}


@dataclass
class AdamState:
    """First/second moments (encoder.py:66-84)."""

    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    step: int = 0
    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)

    @classmethod
    def for_params(cls, p: ModelParams, lr: float = 1e-3) -> "AdamState":
        s = cls(lr=lr)
        for k, v in p.tensors.items():
            s.m[k] = torch.zeros_like(v)
            s.v[k] = torch.zeros_like(v)
        return s


def adam_step(p: ModelParams, grads: dict, state: AdamState) -> None:
    """Bias-corrected Adam, in place, reference op order (encoder.py:236-249)."""
    state.step += 1
    t = state.step
    bc1 = 1.0 - state.beta1 ** t
    bc2 = 1.0 - state.beta2 ** t
    for name in TENSOR_ORDER:
        g = grads[name]
        tensor = p.tensors[name]
        if g.shape != tensor.shape:
            raise ValueError(f"gradient shape {tuple(g.shape)} != param shape {tuple(tensor.shape)} for {name}")
        m, v = state.m[name], state.v[name]
        m.mul_(state.beta1).add_(g, alpha=1.0 - state.beta1)
        v.mul_(state.beta2).addcmul_(g, g, value=1.0 - state.beta2)
        tensor.sub_(state.lr * (m / bc1) / ((v / bc2).sqrt_().add_(state.eps)))
    p.version += 1


def adam_step_graphable(p: ModelParams, grads: dict, state: AdamState, inv_bc: torch.Tensor) -> None:
    """Adam with the bias corrections read from a device tensor
    ``inv_bc = [1/(1-beta1^t), 1/(1-beta2^t)]`` (TrainStep derives it on the
    device from its step counter), so the update can live inside a captured
    CUDA graph."""
    for name in TENSOR_ORDER:
        g = grads[name]
        tensor = p.tensors[name]
        m, v = state.m[name], state.v[name]
        m.mul_(state.beta1).add_(g, alpha=1.0 - state.beta1)
        v.mul_(state.beta2).addcmul_(g, g, value=1.0 - state.beta2)
        mh = m * inv_bc[0]
        vh = v * inv_bc[1]
        tensor.sub_(state.lr * mh / (vh.sqrt_().add_(state.eps)))
