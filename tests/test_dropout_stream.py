"""Statistical checks of the join+encode kernel's dropout stream design
(encode_mma.cu: per lane and tile one hashed 32-bit seed, then 16 draws
x_k = A_k s + C_k -- the LCG a = 747796405, c = 2891336453 jumped k + 1 steps
-- folded to two 14-bit uniforms per draw).  CPU only: the same arithmetic in
numpy over many seeds.  The decisions are Bernoulli(T / 2^14) per unit and
landing; what matters is that every 14-bit field is uniform and that the 32
fields of one (lane, tile) are independent of each other at the thresholds the
kernel uses (keep = 0.9: T = 14746 for 1-row, 16220 / 13271 for 2-row)."""

import numpy as np

M32 = (1 << 32) - 1


def _jump():
    a, c, A, C = 747796405, 2891336453, 1, 0
    ta, tc = [], []
    for _ in range(16):
        A, C = (A * a) & M32, (C * a + c) & M32
        ta.append(A)
        tc.append(C)
    return np.array(ta, np.uint64), np.array(tc, np.uint64)


def _fields(n_seeds=200_000, rng_seed=1):
    """[n_seeds, 32] 14-bit uniforms u (the kernel compares u < T)."""
    rng = np.random.default_rng(rng_seed)
    cq = rng.integers(0, 1 << 32, size=n_seeds, dtype=np.uint64)
    s = (cq * np.uint64(0x7FEB352D)) & np.uint64(M32)
    s ^= s >> np.uint64(15)
    s = (s * np.uint64(0x846CA68B)) & np.uint64(M32)
    s ^= s >> np.uint64(16)
    A, C = _jump()
    x = (s[:, None] * A[None, :] + C[None, :]) & np.uint64(M32)
    y = ~(x ^ (x >> np.uint64(16))) & np.uint64(0x3FFF3FFF)
    up = np.concatenate([(y & np.uint64(0xFFFF)), (y >> np.uint64(16))], axis=1).astype(np.int64)
    return 0x3FFF - up  # u in [0, 2^14)


def test_fields_uniform():
    u = _fields()
    for j in range(u.shape[1]):
        h = np.bincount(u[:, j] >> 8, minlength=64)  # 64 bins of 256
        e = u.shape[0] / 64
        chi2 = ((h - e) ** 2 / e).sum()
        assert chi2 < 120, (j, chi2)  # 63 dof: p ~ 3e-5


def test_decisions_pairwise_independent():
    u = _fields()
    n = u.shape[0]
    for T in (14746, 16220, 13271):
        d = (u < T).astype(np.float64)
        p = d.mean(0)
        assert np.all(np.abs(p - T / 16384) < 5 * np.sqrt(T / 16384 * (1 - T / 16384) / n)), (T, p)
        c = np.corrcoef(d.T)
        off = c[~np.eye(c.shape[0], dtype=bool)]
        # 200K samples: |corr| of independent indicators ~ N(0, 1/sqrt(n)) = 0.0022
        assert np.max(np.abs(off)) < 0.015, (T, np.max(np.abs(off)))


def test_kept_counts_binomial():
    """The number kept among the 32 decisions of a lane is Binomial(32, keep)."""
    u = _fields()
    T = 14746
    k = (u < T).sum(1)
    p = T / 16384
    assert abs(k.mean() - 32 * p) < 0.01
    assert 0.95 < k.var() / (32 * p * (1 - p)) < 1.05
