"""O5 — diagnostics of App. A.2.2.  fp64, dense where
needed (small N only).  Test infrastructure (see oracle/__init__.py).

Units: objectives are reported in physical units, c(x, y) = h^2 |k - l|^2
and eps = eps' h^2 (reading R2).
"""
from __future__ import annotations

import numpy as np

from .sinkhorn import lse, sqdist


def marginal_errors(st):
    """L1 marginal errors of the state (Table rows):
    X: sum_x |P_X pi(x) - mu(x)| for the plans of the last sweep
       (pre-balance; equals the sum of per-cell stopping errors);
    Y: sum_y |sum_i nu_i(y) - nu(y)| of the stored basic-cell marginals."""
    ex = float(np.abs(st.last["PX"] - st.mu).sum()) if "PX" in st.last else float("nan")
    tot = np.zeros((st.N1, st.N2))
    for r0, c0, d in st.boxes:
        tot[r0:r0 + d.shape[0], c0:c0 + d.shape[1]] += d
    ey = float(np.abs(tot - st.nu).sum())
    return ex, ey


def transport_cost(st):
    """<c, pi> of the last sweep's plans: h^2 sum_i m_i Q_i (physical units)."""
    return float(st.h * st.h * np.sum(st.m * st.last["Q"]))


def dense_state_plan(st):
    """Materialise the global plan pi = sum_J pi_J of the last sweep (needs
    keep_plans=True; small N).  Returns (N1 N2) x (N1 N2) fp64."""
    P = np.zeros((st.N1 * st.N2, st.N1 * st.N2))
    for (R, C, ly, a, b, plan) in st.last["plans"].values():
        xi = R * st.N2 + C
        yi = ly[:, 0] * st.N2 + ly[:, 1]
        P[np.ix_(xi, yi)] += plan
    return P


def primal_score(st, P=None):
    """E(pi) = <c, pi> + eps KL(pi | mu (x) nu) (Eq. KL
    PAPER.md:154-167 with phi(0) = 1) of the last sweep's plan pi = sum_J
    pi_J (needs keep_plans=True).  With P given, of that dense plan instead.
    The X-blocks of a partition are disjoint, so the sum over cells below is
    the same sum as over the materialised plan (checked in the pins)."""
    if P is not None:
        return _primal_dense(st, P)
    nu = st.nu
    s_pi = s_cost = s_kl = 0.0
    for (R, C, ly, a, b, plan) in st.last["plans"].values():
        d2 = (R[:, None] - ly[None, :, 0]) ** 2 + (C[:, None] - ly[None, :, 1]) ** 2
        ref = st.mu[R, C][:, None] * nu[ly[:, 0], ly[:, 1]][None, :]
        pos = plan > 0
        if np.any(pos & (ref <= 0)):
            return float("inf")
        s_cost += float(np.sum(d2 * plan)) * st.h * st.h
        s_kl += float(np.sum(plan[pos] * np.log(plan[pos] / ref[pos])))
        s_pi += float(plan.sum())
    kl = s_kl - s_pi + float(st.mu.sum()) * float(nu.sum())
    return s_cost + st.eps * kl


def _primal_dense(st, P):
    N1, N2 = st.N1, st.N2
    k = np.stack(np.meshgrid(np.arange(N1), np.arange(N2), indexing="ij"), -1).reshape(-1, 2)
    c = sqdist(k, k) * st.h * st.h
    ref = np.outer(st.mu.ravel(), st.nu.ravel())
    pos = P > 0
    if np.any(pos & (ref <= 0)):
        return float("inf")
    kl = float(np.sum(P[pos] * np.log(P[pos] / ref[pos])) - P.sum() + ref.sum())
    return float(np.sum(c * P) + st.eps * kl)


def dual_score(st, a: np.ndarray, b: np.ndarray):
    """D(alpha, beta) = <alpha, mu> + <beta, nu> + eps <1 - exp((alpha + beta
    - c)/eps), mu (x) nu>, with alpha = eps a,
    beta = eps b given per pixel (b ignored where nu = 0).  Dense."""
    N1, N2 = st.N1, st.N2
    k = np.stack(np.meshgrid(np.arange(N1), np.arange(N2), indexing="ij"), -1).reshape(-1, 2)
    Ce = sqdist(k, k) / st.eps_p
    mu, nu = st.mu.ravel(), st.nu.ravel()
    bb = np.where(nu > 0, b.ravel(), 0.0)
    ex = np.exp(a.ravel()[:, None] + bb[None, :] - Ce)
    val = np.sum(a.ravel() * mu) + np.sum(bb * nu) + np.sum(mu[:, None] * nu[None, :] * (1.0 - ex))
    return float(st.eps * val)


def stitch_alpha(st):
    """Global X-potential alpha† from the cell potentials of the last A and B
    sweeps, following the proof of Prop. convergence-hybrid
    as the stitching of BoSch2020 §6.3 (not reproduced in the paper,
    PAPER.md:1413; reading R15): walk a fixed spanning tree of the partition
    graph (the "comb": A-cell (a1, a2) hangs off A-cell (a1, a2-1) through
    B-cell (a1, a2); A-cell (a1, 0) off A-cell (a1-1, 0) through B-cell
    (a1, 0)).  Across an edge (J, J') sharing basic cell i the offset changes
    by the mu-weighted mean of (a_J' - a_J) over X_i; alpha† = a_J - s_J on
    A-cells.  Returns a† per pixel (nat units)."""
    n1, n2, s = st.n1, st.n2, st.s
    na1, na2 = (n1 + 1) // 2, (n2 + 1) // 2
    nb2 = n2 // 2 + 1
    fa, fb = st.alpha["A"], st.alpha["B"]

    def wmean_diff(pv, pu, i1, i2):
        sl = (slice(i1 * s, (i1 + 1) * s), slice(i2 * s, (i2 + 1) * s))
        wgt = st.mu[sl]
        return float(np.sum(wgt * (pv[sl] - pu[sl])) / np.sum(wgt))

    off = np.zeros((na1, na2))
    for a1 in range(na1):
        if a1 > 0:   # A(a1-1, 0) -> B(a1, 0) -> A(a1, 0)
            off[a1, 0] = (off[a1 - 1, 0] + wmean_diff(fb, fa, 2 * a1 - 1, 0)
                          + wmean_diff(fa, fb, 2 * a1, 0))
        for a2 in range(1, na2):   # A(a1, a2-1) -> B(a1, a2) -> A(a1, a2)
            off[a1, a2] = (off[a1, a2 - 1] + wmean_diff(fb, fa, 2 * a1, 2 * a2 - 1)
                           + wmean_diff(fa, fb, 2 * a1, 2 * a2))
    assert nb2 >= na2
    a = np.zeros((st.N1, st.N2))
    for a1 in range(na1):
        for a2 in range(na2):
            sl = (slice(2 * a1 * s, min(2 * a1 + 2, n1) * s), slice(2 * a2 * s, min(2 * a2 + 2, n2) * s))
            a[sl] = fa[sl] - off[a1, a2]
    return a


def y_response(st, a: np.ndarray):
    """Exact global Y-update b(y) = -log sum_x exp(a(x) - c/eps) mu(x)."""
    N1, N2 = st.N1, st.N2
    k = np.stack(np.meshgrid(np.arange(N1), np.arange(N2), indexing="ij"), -1).reshape(-1, 2)
    Ce = sqdist(k, k) / st.eps_p
    with np.errstate(divide="ignore"):
        logmu = np.log(st.mu.ravel())
    return (-lse(a.ravel()[:, None] + logmu[:, None] - Ce, axis=0)).reshape(N1, N2)


def pd_gap(st, P=None):
    """Relative primal-dual gap (E(pi) - D(alpha†, beta†)) / D
    with alpha† from stitch_alpha and beta† its exact Y-response.
    Returns (E, D, rel_gap)."""
    E = primal_score(st, P)
    a = stitch_alpha(st)
    b = y_response(st, a)
    D = dual_score(st, a, b)
    return E, D, (E - D) / D
