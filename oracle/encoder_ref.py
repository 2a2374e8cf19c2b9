"""float64 numpy restatement of the reference encoder (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/walkjoin/encoder.py line by line:
glorot init (:87-117), forward (:126-180), BCE (:183-188), backward
(:200-233), Adam (:236-249).  Parameters are a plain dict of float64 arrays
keyed w1,b1,w2,b2,u1,c1,u2,c2 (encoder.py:25 tensor order).
"""

from __future__ import annotations

import math
from typing import Optional

import numpy as np

TENSOR_ORDER = ("w1", "b1", "w2", "b2", "u1", "c1", "u2", "c2")


def _glorot(rng, fan_in, fan_out):
    a = math.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-a, a, size=(fan_in, fan_out))


def init_params(arity, walk_steps, hidden=64, feature_dim=0, seed=0) -> dict:
    """encoder.py:87-117 (same rng draw order, so identical weights)."""
    rng = np.random.default_rng(seed)
    d_in = arity * (walk_steps + 1) + feature_dim
    return {
        "w1": _glorot(rng, d_in, hidden),
        "b1": np.zeros(hidden),
        "w2": _glorot(rng, hidden, hidden),
        "b2": np.zeros(hidden),
        "u1": _glorot(rng, hidden, hidden),
        "c1": np.zeros(hidden),
        "u2": _glorot(rng, hidden, 1)[:, 0],
        "c2": np.zeros(1),
    }


def _exact_mean_over_rows(x):
    """encoder.py:120-123."""
    return np.array([math.fsum(x[:, h]) for h in range(x.shape[1])]) / x.shape[0]


def forward(p: dict, dense: np.ndarray, walk_steps: int, dropout: float = 0.0,
            training: bool = False, dropout_rng: Optional[np.random.Generator] = None,
            drop_mask: Optional[np.ndarray] = None):
    """encoder.py:126-180.  ``drop_mask`` (already divided by keep) may be
    passed explicitly so a test can feed the same mask to both sides."""
    x = np.asarray(dense, np.float64)
    batched = x.ndim == 3
    if not batched:
        x = x[None]
    B, rows, d_in = x.shape
    width = walk_steps + 1
    n_walks = rows // width
    hidden = p["w1"].shape[1]
    flat = x.reshape(B * rows, d_in)
    z1 = flat @ p["w1"] + p["b1"]
    a1 = np.maximum(z1, 0.0)
    mask = None
    if drop_mask is not None:
        mask = drop_mask.reshape(a1.shape)
        a1 = a1 * mask
    elif training and dropout > 0.0:
        keep = 1.0 - dropout
        mask = (dropout_rng.random(a1.shape) < keep) / keep
        a1 = a1 * mask
    e = a1 @ p["w2"] + p["b2"]
    walk_enc = e.reshape(B, n_walks, width, hidden).mean(axis=2)
    hq = np.stack([_exact_mean_over_rows(walk_enc[b]) for b in range(B)])
    z2 = hq @ p["u1"] + p["c1"]
    a2 = np.maximum(z2, 0.0)
    logits = a2 @ p["u2"] + p["c2"][0]
    cache = dict(x=flat, relu1=z1 > 0.0, drop_mask=mask, a1d=a1, hq=hq, relu2=z2 > 0.0, a2=a2,
                 logits=logits, n_walks=n_walks, width=width)
    return (logits if batched else float(logits[0])), cache


def bce_loss(logit, label) -> float:
    """encoder.py:183-188."""
    z = np.asarray(logit, np.float64)
    y = np.asarray(label, np.float64)
    return float(np.mean(np.maximum(z, 0.0) - z * y + np.log1p(np.exp(-np.abs(z)))))


def _sigmoid(z):
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def backward(p: dict, cache: dict, label) -> dict:
    """encoder.py:200-233."""
    logits = cache["logits"]
    B = logits.shape[0]
    y = np.atleast_1d(np.asarray(label, np.float64))
    n_walks, width = cache["n_walks"], cache["width"]
    dlogit = (_sigmoid(logits) - y) / B
    dc2 = np.array([dlogit.sum()])
    du2 = cache["a2"].T @ dlogit
    dz2 = np.outer(dlogit, p["u2"]) * cache["relu2"]
    dc1 = dz2.sum(axis=0)
    du1 = cache["hq"].T @ dz2
    dhq = dz2 @ p["u1"].T
    de = np.repeat(dhq / (n_walks * width), n_walks * width, axis=0)
    db2 = de.sum(axis=0)
    dw2 = cache["a1d"].T @ de
    da1 = de @ p["w2"].T
    if cache["drop_mask"] is not None:
        da1 = da1 * cache["drop_mask"]
    dz1 = da1 * cache["relu1"]
    db1 = dz1.sum(axis=0)
    dw1 = cache["x"].T @ dz1
    return {"w1": dw1, "b1": db1, "w2": dw2, "b2": db2, "u1": du1, "c1": dc1, "u2": du2, "c2": dc2}


class Adam:
    """encoder.py:66-84 state + :236-249 update."""

    def __init__(self, p: dict, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
        self.lr, self.beta1, self.beta2, self.eps, self.step = lr, beta1, beta2, eps, 0
        self.m = {k: np.zeros_like(v) for k, v in p.items()}
        self.v = {k: np.zeros_like(v) for k, v in p.items()}

    def update(self, p: dict, g: dict):
        self.step += 1
        t = self.step
        for name in TENSOR_ORDER:
            self.m[name] = self.beta1 * self.m[name] + (1.0 - self.beta1) * g[name]
            self.v[name] = self.beta2 * self.v[name] + (1.0 - self.beta2) * g[name] * g[name]
            m_hat = self.m[name] / (1.0 - self.beta1 ** t)
            v_hat = self.v[name] / (1.0 - self.beta2 ** t)
            p[name] -= self.lr * m_hat / (np.sqrt(v_hat) + self.eps)
