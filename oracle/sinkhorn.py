"""Dense log-domain Sinkhorn (test infrastructure, see oracle/__init__.py).

Potentials are dimensionless: a = alpha/eps, b = beta/eps.  Costs are in
pixel^2 units, so c/eps = |k - l|^2 / eps' with eps' = eps / h^2
(reading R2).  No separable shortcut, no gauge trick: the
(n_x x n_y) kernel is materialised (this is the plain definition the GPU's
separable local-gauge kernel must reproduce, App. A.1).
"""
from __future__ import annotations

import numpy as np


def lse(v: np.ndarray, axis: int) -> np.ndarray:
    """log sum exp along axis (max-shifted; all -inf -> -inf)."""
    m = np.max(v, axis=axis, keepdims=True)
    m_safe = np.where(np.isfinite(m), m, 0.0)
    out = np.log(np.sum(np.exp(v - m_safe), axis=axis, keepdims=True)) + m_safe
    return np.squeeze(out, axis=axis)


def sqdist(kx: np.ndarray, ly: np.ndarray) -> np.ndarray:
    """|k - l|^2 for pixel coordinates kx (n,2) and ly (m,2) (squared
    Euclidean cost)."""
    d1 = kx[:, 0:1].astype(np.float64) - ly[None, :, 0].astype(np.float64)
    d2 = kx[:, 1:2].astype(np.float64) - ly[None, :, 1].astype(np.float64)
    return d1 * d1 + d2 * d2


def cell_sinkhorn(mu_x: np.ndarray, kx: np.ndarray, nu_y: np.ndarray, ly: np.ndarray,
                  eps_p: float, a0: np.ndarray, err: float, fixed_iter: int = 0,
                  max_iter: int = 2000):
    """Entropic OT on one composite cell, Alg. 1 line 4:
    min <c, pi> + eps KL(pi | mu_J (x) nu) over Pi(mu_J, nu_J).  The
    reference measure mu_J (x) nu_J has the same minimiser (
    reading R5).  Log-domain Sinkhorn, alternating
        Y-update  b(l)  = -log sum_k exp(a(k) - c(k,l)/eps) mu(k)
        X-update  a'(k) = -log sum_l exp(b(l) - c(k,l)/eps) nu_J(l)
    Stopping rule (App. A.2.1; per-cell reading R6):
    L1 X-marginal error of the plan (a, b) after the Y-update,
        e = sum_k mu(k) |r - exp(a(k) - a'(k))| <= err * mu(X_J),
    where r = ||nu_J|| / mu(X_J) (reading R6': after a Y-update the plan has
    mass ||nu_J||, which the truncation ledger R9 can make differ from
    mu(X_J); r = 1 for balanced cells, the paper's case),
    or exactly fixed_iter passes (parity mode), or max_iter passes.

    nu_y must be > 0 (zero pixels of the box are excluded, reading R19).
    Returns (a, b, plan, iters, e_first, e_last) with plan = exp(a + b - c/eps)
    mu nu (rows = kx, cols = ly), whose Y-marginal is exactly nu_y.
    """
    C = sqdist(kx, ly) / eps_p
    logmu = np.log(mu_x)
    lognu = np.log(nu_y)
    a = a0.astype(np.float64).copy()
    tol = err * float(mu_x.sum())
    rm1 = (float(nu_y.sum()) - float(mu_x.sum())) / float(mu_x.sum())
    t = 0
    e0 = None
    while True:
        t += 1
        b = -lse(a[:, None] + logmu[:, None] - C, axis=0)
        a_new = -lse(b[None, :] + lognu[None, :] - C, axis=1)
        e = float(np.sum(mu_x * np.abs(np.expm1(a - a_new) - rm1)))
        if e0 is None:
            e0 = e
        if fixed_iter > 0:
            stop = t >= fixed_iter
        else:
            stop = (e <= tol) or (t >= max_iter)
        if stop:
            break
        a = a_new
    plan = np.exp(a[:, None] + b[None, :] - C) * mu_x[:, None] * nu_y[None, :]
    return a, b, plan, t, e0, e


def dense_sinkhorn(mu: np.ndarray, nu: np.ndarray, eps_p: float, tol: float = 1e-13,
                   max_iter: int = 200000, a0=None):
    """Global dense log-domain Sinkhorn on the whole grid problem
    (Eq. entropic-transport) — the brute-force reference
    (O6).  Runs until the L1 X-marginal error after the Y-update is
    <= tol.  Returns (plan (N^2 x N^2 over supports), a, b, xs, ys) with
    xs, ys the flat pixel indices of the supports of mu and nu."""
    N1, N2 = mu.shape
    xs = np.flatnonzero(mu.ravel() > 0)
    ys = np.flatnonzero(nu.ravel() > 0)
    kx = np.stack([xs // N2, xs % N2], axis=1)
    ly = np.stack([ys // N2, ys % N2], axis=1)
    mux = mu.ravel()[xs]
    nuy = nu.ravel()[ys]
    C = sqdist(kx, ly) / eps_p
    logmu, lognu = np.log(mux), np.log(nuy)
    a = np.zeros(len(xs)) if a0 is None else np.asarray(a0, np.float64).ravel()[xs].copy()
    for _ in range(max_iter):
        b = -lse(a[:, None] + logmu[:, None] - C, axis=0)
        a_new = -lse(b[None, :] + lognu[None, :] - C, axis=1)
        e = float(np.sum(mux * np.abs(np.expm1(a - a_new))))
        a = a_new
        if e <= tol:
            break
    b = -lse(a[:, None] + logmu[:, None] - C, axis=0)
    plan = np.exp(a[:, None] + b[None, :] - C) * mux[:, None] * nuy[None, :]
    return plan, a, b, xs, ys


def y_update_at(a: np.ndarray, mu: np.ndarray, eps_p: float, ls) -> np.ndarray:
    """Y-half of the Sinkhorn iteration at selected target pixels only:
    b(l) = -LSE_k [a(k) + log mu(k) - |k - l|^2 / eps'] over supp(mu)
    (the beta-update of Eq. entropic-transport's dual, the
    same formula as the first line of dense_sinkhorn's loop).  a, mu: (N1, N2)
    grids; ls: (m, 2) integer pixel coordinates.  O(N1 N2) per target, so it
    serves sampled checks at full size."""
    N1, N2 = mu.shape
    xs = np.flatnonzero(mu.ravel() > 0)
    kx = np.stack([xs // N2, xs % N2], axis=1)
    base = a.ravel()[xs] + np.log(mu.ravel()[xs])
    ls = np.asarray(ls, dtype=np.int64).reshape(-1, 2)
    out = np.empty(len(ls))
    for j, l in enumerate(ls):
        out[j] = -lse(base - sqdist(kx, l[None, :])[:, 0] / eps_p, axis=0)
    return out
