"""Seeded, exact (dyadic) synthetic workloads.  No method arithmetic here.

Conventions:
  * pixel (r, c) of an N1 x N2 grid has physical centre
    x = (-1 + (r + 1/2) h, -1 + (c + 1/2) h), h = 2 / N;
  * all masses are integer counts times 2^-E, E = 12 + 2 ceil(log2 N);
  * basic cell i = (i1, i2) covers pixel rows [i1 s, (i1+1) s) and columns
    [i2 s, (i2+1) s); linear index i = i1 * n2 + i2.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

M64 = (1 << 64) - 1


class SplitMix64:
    """SplitMix64 (Steele, Lea, Flood 2014); documented so any language can
    reproduce the same stream.  next_double() returns (z >> 11) * 2^-53."""

    def __init__(self, seed: int):
        self.state = seed & M64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()


def exponent_E(N: int) -> int:
    """Mass quantum exponent: total mass = 2^E counts, mean 4096 counts/pixel."""
    return 12 + 2 * int(math.ceil(math.log2(N)))


def _pixel_centres(N: int):
    h = 2.0 / N
    x = -1.0 + (np.arange(N, dtype=np.float64) + 0.5) * h
    return x, h


def _quantise(rho: np.ndarray, E: int) -> np.ndarray:
    """Integer counts c >= 1 with sum exactly 2^E (largest pixel absorbs the
    rounding residual, lowest linear index among ties)."""
    total = 1 << E
    c = np.maximum(1, np.rint(rho / rho.sum() * total)).astype(np.int64)
    resid = total - int(c.sum())
    k = int(np.argmax(c))
    c.flat[k] += resid
    assert c.min() >= 1 and int(c.sum()) == total
    assert int(c.max()) < (1 << 23), "counts must stay exact in fp32"
    return c


def gaussian_mixture_counts(N: int, seed: int, E: int | None = None) -> np.ndarray:
    """GM(seed): K = 5 + (u0 mod 11) anisotropic Gaussians, means in
    [-0.6, 0.6]^2, per-axis std in [0.05, 0.3], orientation in [0, pi),
    weights in [0.5, 1.5], plus a floor of 1e-3 * mean density so that every
    basic cell has positive mass.  Returns int64 counts (N, N)."""
    if E is None:
        E = exponent_E(N)
    rng = SplitMix64(seed)
    K = 5 + (rng.next_u64() % 11)
    x, _ = _pixel_centres(N)
    X1, X2 = np.meshgrid(x, x, indexing="ij")
    rho = np.zeros((N, N), dtype=np.float64)
    for _ in range(K):
        m1 = rng.uniform(-0.6, 0.6)
        m2 = rng.uniform(-0.6, 0.6)
        sa = rng.uniform(0.05, 0.3)
        sb = rng.uniform(0.05, 0.3)
        phi = rng.uniform(0.0, math.pi)
        wgt = rng.uniform(0.5, 1.5)
        cph, sph = math.cos(phi), math.sin(phi)
        d1, d2 = X1 - m1, X2 - m2
        u = cph * d1 + sph * d2
        v = -sph * d1 + cph * d2
        rho += wgt * np.exp(-0.5 * (u * u / (sa * sa) + v * v / (sb * sb))) / (2 * math.pi * sa * sb)
    rho += 1e-3 * rho.mean()
    return _quantise(rho, E)


def push_T0(a: np.ndarray) -> np.ndarray:
    """Push-forward of a pixel array under T0 (x1, x2) -> (-x2, x1) (Eq. T0,
    PAPER.md:941-947): pixel (r, c) -> (N-1-c, r)."""
    return a[:, ::-1].T.copy()


def four_bumps_counts(N: int, E: int | None = None) -> np.ndarray:
    """Four isotropic bumps at (+-1/2, +-1/2), sigma = 0.2 (paper silent,
    PAPER.md:940; SPEC's constants), plus the 1e-3 floor.  Built from one
    quadrant and its T0 images so that T0_# mu = mu exactly."""
    assert N % 2 == 0
    if E is None:
        E = exponent_E(N)
    x, _ = _pixel_centres(N)
    X1, X2 = np.meshgrid(x, x, indexing="ij")
    rho = np.zeros((N, N))
    for m1 in (-0.5, 0.5):
        for m2 in (-0.5, 0.5):
            rho += np.exp(-((X1 - m1) ** 2 + (X2 - m2) ** 2) / (2 * 0.2 ** 2))
    rho += 1e-3 * rho.mean()
    hN = N // 2
    q = rho[:hN, :hN]
    total = 1 << E
    cq = np.maximum(1, np.rint(q / (4.0 * q.sum()) * total)).astype(np.int64)
    resid = total - 4 * int(cq.sum())
    assert resid % 4 == 0
    cq.flat[int(np.argmax(cq))] += resid // 4
    full = np.zeros((N, N), dtype=np.int64)
    full[:hN, :hN] = cq
    full = full + push_T0(full)
    full = full + push_T0(push_T0(full))
    assert int(full.sum()) == total and full.min() >= 1
    assert np.array_equal(push_T0(full), full)
    return full


def rotation_map(theta_deg: float):
    """T_theta(x) = lam R_theta x with lam = 1/(|cos|+|sin|) so the rotated
    square fits into [-1,1]^2.  Returns (cos, sin, lam)."""
    t = math.radians(theta_deg)
    c, s = math.cos(t), math.sin(t)
    lam = 1.0 / (abs(c) + abs(s))
    return c, s, lam


def splat_coupling(counts: np.ndarray, s: int, theta_deg: float):
    """pi^0 = (id, T_theta)_# mu by integer bilinear splatting (DESIGN.md
    reading R17).  Each source pixel's count is split among the <= 4 target
    pixels around T(x) as floor(weight * count) plus the remainder to the
    largest fractional parts (ties -> lowest target index).  theta = 90 uses
    the exact pixel permutation of Eq. T0.

    Returns (nu_counts, off[I,2], ext[I,2], pos[I], data_counts[...]) where the
    boxes are the per-source-basic-cell Y-marginals nu_i^0 (Eq.
    basic-cell-Y-marginal) in bounding-box form
    (PAPER.md:1115)."""
    N1, N2 = counts.shape
    assert N1 == N2
    N = N1
    n1, n2 = N1 // s, N2 // s
    rr, cc = np.meshgrid(np.arange(N1), np.arange(N2), indexing="ij")
    src_cell = ((rr // s) * n2 + (cc // s)).ravel()
    cnt = counts.ravel().astype(np.int64)
    if abs(theta_deg - 90.0) < 1e-12:
        tr = (N - 1 - cc).ravel()[:, None]
        tc = rr.ravel()[:, None]
        parts = cnt[:, None]
    elif abs(theta_deg) < 1e-12:
        tr = rr.ravel()[:, None]
        tc = cc.ravel()[:, None]
        parts = cnt[:, None]
    else:
        co, si, lam = rotation_map(theta_deg)
        x, h = _pixel_centres(N)
        x1 = x[rr].ravel()
        x2 = x[cc].ravel()
        y1 = lam * (co * x1 - si * x2)
        y2 = lam * (si * x1 + co * x2)
        u1 = (y1 + 1.0) / h - 0.5
        u2 = (y2 + 1.0) / h - 0.5
        a1 = np.floor(u1)
        a2 = np.floor(u2)
        f1 = u1 - a1
        f2 = u2 - a2
        a1 = a1.astype(np.int64)
        a2 = a2.astype(np.int64)
        tr = np.stack([a1, a1, a1 + 1, a1 + 1], axis=1)
        tc = np.stack([a2, a2 + 1, a2, a2 + 1], axis=1)
        wts = np.stack([(1 - f1) * (1 - f2), (1 - f1) * f2, f1 * (1 - f2), f1 * f2], axis=1)
        tr = np.clip(tr, 0, N - 1)
        tc = np.clip(tc, 0, N - 1)
        raw = wts * cnt[:, None]
        base = np.floor(raw).astype(np.int64)
        frac = raw - base
        rem = cnt - base.sum(axis=1)
        tlin = tr * N2 + tc
        order = np.lexsort((tlin, -frac), axis=-1)  # largest frac first, ties lowest index
        rank = np.empty_like(order)
        np.put_along_axis(rank, order, np.arange(4)[None, :].repeat(len(cnt), 0), axis=1)
        parts = base + (rank < rem[:, None]).astype(np.int64)
    assert np.array_equal(parts.sum(axis=1), cnt)
    mask = parts > 0
    cell = np.broadcast_to(src_cell[:, None], parts.shape)[mask]
    r = np.broadcast_to(tr, parts.shape)[mask]
    c = np.broadcast_to(tc, parts.shape)[mask]
    p = parts[mask]
    nu_counts = np.zeros(N1 * N2, dtype=np.int64)
    np.add.at(nu_counts, r * N2 + c, p)
    I = n1 * n2
    r0 = np.full(I, 1 << 30, dtype=np.int64)
    c0 = np.full(I, 1 << 30, dtype=np.int64)
    r1 = np.full(I, -1, dtype=np.int64)
    c1 = np.full(I, -1, dtype=np.int64)
    np.minimum.at(r0, cell, r)
    np.minimum.at(c0, cell, c)
    np.maximum.at(r1, cell, r)
    np.maximum.at(c1, cell, c)
    e1 = r1 - r0 + 1
    e2 = c1 - c0 + 1
    sizes = e1 * e2
    pos = np.zeros(I, dtype=np.int64)
    pos[1:] = np.cumsum(sizes)[:-1]
    data = np.zeros(int(sizes.sum()), dtype=np.int64)
    idx = pos[cell] + (r - r0[cell]) * e2[cell] + (c - c0[cell])
    np.add.at(data, idx, p)
    off = np.stack([r0, c0], axis=1).astype(np.int32)
    ext = np.stack([e1, e2], axis=1).astype(np.int32)
    return nu_counts.reshape(N1, N2), off, ext, pos, data


@dataclass
class Problem:
    """One synthetic instance.  Everything is exact: value = count * 2^-E."""
    name: str
    N: int
    s: int
    eps_factor: float      # eps = (eps_factor * h)^2
    E: int
    mu_counts: np.ndarray  # (N, N) int64
    nu_counts: np.ndarray  # (N, N) int64
    init_off: np.ndarray   # (I, 2) int32 lower (row, col) corner
    init_ext: np.ndarray   # (I, 2) int32 extents
    init_pos: np.ndarray   # (I,) int64 start of cell i in init_counts
    init_counts: np.ndarray  # int64

    @property
    def h(self) -> float:
        return 2.0 / self.N

    @property
    def eps(self) -> float:
        return (self.eps_factor * self.h) ** 2

    @property
    def eps_prime(self) -> float:
        """eps / h^2: regularisation in pixel^2 units."""
        return self.eps_factor ** 2

    @property
    def quantum(self) -> float:
        return 2.0 ** (-self.E)

    @property
    def mu(self) -> np.ndarray:
        return self.mu_counts.astype(np.float64) * self.quantum

    @property
    def nu(self) -> np.ndarray:
        return self.nu_counts.astype(np.float64) * self.quantum

    @property
    def init_data(self) -> np.ndarray:
        return self.init_counts.astype(np.float64) * self.quantum

    @property
    def n(self) -> int:
        return self.N // self.s

    def supplies(self) -> np.ndarray:
        """q_i = m_i 2^E (exact int64 basic-cell supplies)."""
        n = self.n
        return self.mu_counts.reshape(n, self.s, n, self.s).sum(axis=(1, 3)).ravel().astype(np.int64)


def make_problem(kind: str, N: int, s: int, eps_factor: float = 2.0,
                 theta_deg: float = 20.0, seed: int = 0) -> Problem:
    """kind = "gm" (Gaussian mixture GM(seed) pushed by T_theta) or "bumps"
    (four bumps with T0, theta forced to 90 so nu = mu)."""
    E = exponent_E(N)
    if kind == "gm":
        mu = gaussian_mixture_counts(N, seed, E)
        th = theta_deg
    elif kind == "bumps":
        mu = four_bumps_counts(N, E)
        th = 90.0
    else:
        raise ValueError(kind)
    nu, off, ext, pos, data = splat_coupling(mu, s, th)
    if kind == "bumps":
        assert np.array_equal(nu, mu)
    name = f"{kind}{'' if kind != 'gm' else seed}_N{N}_s{s}_eps{eps_factor:g}h_th{th:g}"
    return Problem(name, N, s, float(eps_factor), E, mu, nu, off, ext, pos, data)


# Arc order of the 5-point neighbourhood (Def. neigh):
# 0 = self, 1 = up (i1-1), 2 = down (i1+1), 3 = left (i2-1), 4 = right (i2+1).
ARC_D = ((0, 0), (-1, 0), (1, 0), (0, -1), (0, 1))


def random_flow(q: np.ndarray, n1: int, n2: int, seed: int, n_cycles: int = 200) -> np.ndarray:
    """A random feasible flow w (|I| x 5 int64) satisfying both divergence
    constraints exactly (Eq. div-constraint): start from the
    stationary flow and superpose random integer 2-cycles and 4-cycles, each
    bounded by the remaining self-mass of the nodes it passes through."""
    rng = SplitMix64(seed)
    I = n1 * n2
    w = np.zeros((I, 5), dtype=np.int64)
    w[:, 0] = q
    for _ in range(n_cycles):
        i1 = int(rng.next_u64() % n1)
        i2 = int(rng.next_u64() % n2)
        kind = rng.next_u64() % 3
        if kind == 0 and i2 + 1 < n2:           # 2-cycle right/left
            nodes = [(i1, i2), (i1, i2 + 1)]
            arcs = [4, 3]
        elif kind == 1 and i1 + 1 < n1 and i2 + 1 < n2:   # clockwise plaquette
            nodes = [(i1, i2), (i1, i2 + 1), (i1 + 1, i2 + 1), (i1 + 1, i2)]
            arcs = [4, 2, 3, 1]
        elif kind == 2 and i1 + 1 < n1 and i2 + 1 < n2:   # counter-clockwise
            nodes = [(i1, i2), (i1 + 1, i2), (i1 + 1, i2 + 1), (i1, i2 + 1)]
            arcs = [2, 4, 1, 3]
        else:
            continue
        idx = [a * n2 + b for a, b in nodes]
        cap = min(int(w[k, 0]) for k in idx)
        if cap <= 0:
            continue
        amt = 1 + int(rng.next_u64() % max(1, cap // 2))
        for k, a in zip(idx, arcs):
            w[k, 0] -= amt
            w[k, a] += amt
    return w


def random_mcf_instance(n1: int, n2: int, seed: int, qmax: int = 1000, cmax: int = 1000):
    """Random integer min-cost-flow instance on the n1 x n2 grid graph:
    supplies q_i in [1, qmax], arc costs C_ij in [-cmax, cmax] for the 4
    neighbour arcs, columns in ARC_D order (column 0 = self arc, cost 0; arcs
    leaving the grid get cost 0 and are unusable)."""
    rng = SplitMix64(seed)
    I = n1 * n2
    q = np.array([1 + rng.next_u64() % qmax for _ in range(I)], dtype=np.int64)
    C = np.zeros((I, 5), dtype=np.int64)
    for i in range(I):
        for a in range(1, 5):
            C[i, a] = int(rng.next_u64() % (2 * cmax + 1)) - cmax
    return q, C
