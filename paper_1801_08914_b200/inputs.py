"""Seeded synthetic inputs of the BASELINE configs.

The stream is the reference's own test RNG, ``oracle::Xorshift``
(tests/test_support.hpp:79-92: xorshift64 13/7/17, uniform = (next >> 11) 2^-53,
log_uniform = exp(uniform(log lo, log hi))), seeded 1000 + config id, drawn in
the documented order: per cell (lexicographic, x fastest) alpha then beta; f_hat
in broken order (cell-major, local dof order); lambda (m values); x_b (nS
values); then, for config 4, the interior vertex displacements.  The CPU oracle
(oracle/hdr_oracle.c hdo_gen_inputs) draws the same stream, so the timed
inputs of bench.py are the parity-tested ones (tests/test_inputs.py checks the
bits).  Every arithmetic step is the C one (no fused multiply-add; exp / log
from the platform libm via ``math``).
"""
from __future__ import annotations

import math

import numpy as np

_M64 = 0xFFFFFFFFFFFFFFFF

# BASELINE.json configs: dim, cells, RT order, coefficient law, seed (1000 + id)
CONFIGS = {
    1: dict(dim=2, cells=(64, 64), k=0, coef=("uniform", 1.0, 1.0), seed=1001,
            desc="cfg1: 2D unit-square 64x64 quads, RT_0, alpha=beta=1"),
    2: dict(dim=3, cells=(64, 64, 64), k=0, coef=("logu", 1e-2, 1e2), seed=1002,
            desc="cfg2: 3D unit-cube 64^3 hexes (262,144 elems), RT_0, alpha,beta log-uniform [1e-2,1e2]"),
    3: dict(dim=3, cells=(48, 48, 48), k=1, coef=("logu", 1e-2, 1e2), seed=1003,
            desc="cfg3: 3D unit-cube 48^3 hexes (110,592 elems), RT_1, alpha,beta log-uniform [1e-2,1e2]"),
    4: dict(dim=3, cells=(24, 24, 24), k=2, coef=("logu", 1e-3, 1e3), seed=1004, perturb=0.2,
            desc="cfg4: 3D 24^3 perturbed trilinear hexes (13,824 elems, interior vertices moved U[-0.2h,0.2h]), "
                 "RT_2 (Piola), alpha,beta log-uniform [1e-3,1e3]"),
    5: dict(dim=3, cells=(32, 32, 32), k=3, coef=("checker", 1e-2, 1e2), seed=1005,
            desc="cfg5: 3D unit-cube 32^3 hexes (32,768 elems), RT_3, 4^3 checkerboard sigma_t in {1e-2,1e2}"),
}


class Xorshift:
    """oracle::Xorshift (tests/test_support.hpp:79-92)."""

    def __init__(self, seed: int):
        self.state = seed if seed else 0x9E3779B97F4A7C15

    def uniforms(self, n: int) -> np.ndarray:
        """n draws of uniform() in [0, 1)."""
        s = self.state
        out = np.empty(n, dtype=np.uint64)
        for i in range(n):
            s ^= (s << 13) & _M64
            s ^= s >> 7
            s ^= (s << 17) & _M64
            out[i] = s >> 11
        self.state = s
        return out.astype(np.float64) * 2.0 ** -53

    def uniform(self, lo: float, hi: float, n: int) -> np.ndarray:
        return lo + (hi - lo) * self.uniforms(n)  # two roundings, as the C expression


def _shape(dim: int, cells, k: int):
    c = list(cells) + [1] * (3 - len(cells))
    dpf = (k + 1) ** (dim - 1)
    n = 2 * dim * dpf + dim * k * dpf
    nfaces, interior = 0, 0
    for a in range(dim):
        cnt, inner = c[a] + 1, c[a] - 1
        for b in range(dim):
            if b != a:
                cnt *= c[b]
                inner *= c[b]
        nfaces += cnt
        interior += inner
    return c, n, dpf, nfaces * dpf, interior * dpf


def make_inputs(dim: int, cells, k: int, coef, seed: int, perturb: float = 0.0, extras: bool = False):
    """(alpha, beta, f_hat[, lambda, x_b, vertices]) of the §8(d) law.  coef =
    (kind, p0, p1) with kind "uniform" | "logu" | "checker" | "softhard" (the
    reference's soft_hard_coefficients, p0 = exponent, src/mesh.cpp:168-191)."""
    c, n, _, n_s, m = _shape(dim, cells, k)
    ncells = c[0] * c[1] * c[2]
    h = [1.0 / c[a] if a < dim else 1.0 for a in range(3)]
    kind, p0, p1 = coef
    r = Xorshift(seed)
    idx = np.arange(ncells)
    co = [idx % c[0], (idx // c[0]) % c[1], idx // (c[0] * c[1])]
    if kind == "uniform":
        alpha, beta = np.full(ncells, float(p0)), np.full(ncells, float(p1))
    elif kind == "logu":
        u = r.uniforms(2 * ncells)
        l0, l1 = math.log(p0), math.log(p1)
        t = l0 + (l1 - l0) * u
        e = np.array([math.exp(x) for x in t.tolist()])
        alpha, beta = e[0::2].copy(), e[1::2].copy()
    elif kind == "checker":  # cfg5: alpha_ref = 1 (divdiv), beta_ref = 1 / (3 sigma_t) (mass), SURVEY.md §8(d)
        reg = np.zeros(ncells, dtype=np.int64)
        for a in range(dim):
            x = 0.0 + (co[a].astype(np.float64) + 0.5) * h[a]
            reg += np.floor(4.0 * x).astype(np.int64)
        sigma = np.where(reg % 2 == 0, float(p0), float(p1))
        alpha, beta = np.ones(ncells), 1.0 / (3.0 * sigma)
    elif kind == "softhard":
        in_lo = np.ones(ncells, bool)
        in_hi = np.ones(ncells, bool)
        for a in range(dim):
            x = 0.0 + (co[a].astype(np.float64) + 0.5) * h[a]
            in_lo &= (x >= 0.25) & (x <= 0.5)
            in_hi &= (x >= 0.5) & (x <= 0.75)
        alpha = np.ones(ncells)
        beta = np.where(in_lo | in_hi, math.pow(10.0, int(p0)), 1.0)
    else:
        raise ValueError(f"unknown coefficient law {kind}")
    f_hat = r.uniform(-1.0, 1.0, ncells * n)
    if not extras and not perturb:
        return alpha, beta, f_hat
    lam = r.uniform(-1.0, 1.0, m)
    x_b = r.uniform(-1.0, 1.0, n_s)
    verts = None
    if perturb and dim == 3:
        nv = [c[a] + 1 for a in range(3)]
        g = np.stack(np.meshgrid(*[np.arange(nv[a]) * h[a] for a in range(3)], indexing="ij"), -1)
        g = np.ascontiguousarray(g.transpose(2, 1, 0, 3))  # (z, y, x, coord), x fastest
        interior = np.zeros((nv[2], nv[1], nv[0]), bool)
        interior[1:-1, 1:-1, 1:-1] = True
        cnt = int(interior.sum()) * 3
        d = r.uniforms(cnt)
        amp = np.array([perturb * h[a] for a in range(3)])
        lo = -amp
        # lo + (hi - lo) u per coordinate, drawn vertex by vertex (x fastest), x then y then z
        disp = (lo[None, :] + (amp - lo)[None, :] * d.reshape(-1, 3))
        g[interior] = g[interior] + disp
        verts = g.reshape(-1, 3)
    if extras:
        return alpha, beta, f_hat, lam, x_b, verts
    return alpha, beta, f_hat, verts


def config_inputs(cfg_id: int, seed: int | None = None):
    """(alpha, beta, f_hat, vertices or None) of BASELINE config cfg_id."""
    cfg = CONFIGS[cfg_id]
    out = make_inputs(cfg["dim"], cfg["cells"], cfg["k"], cfg["coef"], cfg["seed"] if seed is None else seed,
                      perturb=cfg.get("perturb", 0.0))
    if len(out) == 3:
        return out + (None,)
    return out
