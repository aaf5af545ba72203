"""f3 — multiscale domain decomposition (App. A.2.1 "Multi-scale and
eps-scaling"; the coarse-to-fine strategy of
[BoSch2020, Section 6.4], which the paper uses but does not reproduce,
PAPER.md:1205).  Test infrastructure (see oracle/__init__.py).

Readings (R23-R25; the paper is silent on the details):
  R23 layers: N_l = N / 2^(L-1-l), l = 0..L-1, same basic cell size s on every
      layer; mu_l, nu_l are 2x2 block sums of the next finer layer (exact on
      the dyadic inputs).
  R24 eps: on every layer eps = eps' h_l^2 with the same eps' (the target
      (2h)^2 gives eps' = 4), so eps drops 4x at each refinement (the paper's
      ladder 2 dx^2 -> dx^2/2 per layer, also spans 4x per
      layer).  Each layer runs the hybrid scheme (Alg. 3)
      until the sweep-entry errors of both partitions are <= conv (reading
      R14) or a cycle cap.
  R25 refinement: the fine coupling keeps the coarse basic-cell marginals and
      distributes them uniformly w.r.t. mu (x) nu inside each coarse pixel
      pair: for a fine basic cell i' inside coarse basic cell i and a fine
      pixel y' inside coarse pixel y,
          nu_i'(y') = (nu_i(y) * (m_i' / m_i)) * (nu(y') / nu_l(y)),
      evaluated in exactly this order in fp64, then truncated at tau with a
      minimal box (a5).  It is a feasible coupling: sum_i' nu_i' = nu and
      ||nu_i'|| = m_i' (up to the truncation ledger, R9), and coarsening it
      back gives the coarse marginals (pinned).
  R25' warm start: the physical dual potential is kept across the
      refinement, so in units of eps (which drops 4x, R24) the fine
      partition-A potential is a_f(x') = 4 a_l(parent(x')) (every fine A-cell
      lies in one coarse A-cell, so the coarse per-cell constants are
      harmless); partition B starts from alpha = 0 (reading R7).
  The coarsest layer starts from the product coupling pi = mu (x) nu, i.e.
  nu_i = m_i nu (a feasible coupling for any pair of measures).
  R24' eps-scaling inside a layer (optional, eps_scale = F > 1; the paper's
      scheme: "the initial regularization strength is eps =
      2 dx^2 ... the final value is dx^2 / 2 ... the final regularization
      strength on a given multiscale layer coincides with the initial one in
      the next layer"): every layer starts at eps' F and halves eps' after
      each stage until eps'; every stage runs cycles until R14 <= conv.
      With F = 4 a layer spans the paper's 4x and its initial eps equals the
      coarser layer's final one.  Changing eps keeps the physical dual
      potential: in units of eps (base 2) alpha scales by eps_old / eps_new
      (set_eps); the refinement transfer of R25' scales by eps_c / eps_f.
"""
from __future__ import annotations

import numpy as np

from .domdec import OracleState, truncate_box
from .diagnostics import marginal_errors
from .domdec import domdec_sweep
from .flow import flow_update
from .partitions import basic_partition


def coarsen(a: np.ndarray) -> np.ndarray:
    """2x2 block sums (R23): a_l(x) = sum of the four finer pixels of x."""
    N1, N2 = a.shape
    assert N1 % 2 == 0 and N2 % 2 == 0
    return a.reshape(N1 // 2, 2, N2 // 2, 2).sum(axis=(1, 3))


def product_state(mu: np.ndarray, nu: np.ndarray, s: int, eps_p: float, h: float, tau: float = 1e-15):
    """State of the product coupling mu (x) nu: nu_i = m_i nu on the minimal
    box of supp(nu), truncated at tau (a5)."""
    N1, N2 = mu.shape
    n1, n2, m = basic_partition(mu, s)
    nz = np.argwhere(nu > 0)
    a1, a2 = nz.min(axis=0)
    b1, b2 = nz.max(axis=0) + 1
    boxes = []
    dropped = 0.0
    for i in range(n1 * n2):
        r0, c0, d, dr = truncate_box(int(a1), int(a2), m[i] * nu[a1:b1, a2:b2], tau)
        boxes.append([r0, c0, d])
        dropped += dr
    st = OracleState(N1, N2, s, float(eps_p), float(h), np.asarray(mu, np.float64), np.asarray(nu, np.float64),
                     m, n1, n2, boxes)
    st.dropped = dropped
    return st


def set_eps(st: OracleState, eps_p: float):
    """R24': change eps' of a state, keeping the physical potentials
    (alpha in units of eps scales by eps_old / eps_new)."""
    f = st.eps_p / float(eps_p)
    for k in list(st.alpha):
        if st.alpha[k] is not None:
            st.alpha[k] = st.alpha[k] * f
    st.eps_p = float(eps_p)


def refine_state(stc: OracleState, mu_f: np.ndarray, nu_f: np.ndarray, tau: float = 1e-15, eps_p_f=None):
    """Fine state from a coarse one (R25).  mu_f, nu_f: the next finer layer
    (coarsen(mu_f) must equal stc.mu, likewise nu); eps_p_f: the fine layer's
    initial eps' (default: the coarse one, R24)."""
    N1, N2 = mu_f.shape
    s = stc.s
    n1, n2, m = basic_partition(mu_f, s)
    nu_c = coarsen(nu_f)
    # ry(y') = nu(y') / nu_l(parent(y')), 0 where the coarse pixel is empty
    par = np.kron(nu_c, np.ones((2, 2)))
    ry = np.zeros_like(nu_f)
    pos = par > 0
    ry[pos] = nu_f[pos] / par[pos]
    boxes = [None] * (n1 * n2)
    dropped = 0.0
    for i in range(stc.n1 * stc.n2):
        i1, i2 = divmod(i, stc.n2)
        r0, c0, d = stc.boxes[i]
        R0, C0 = 2 * r0, 2 * c0
        v = np.kron(d, np.ones((2, 2)))                       # nu_i(parent(y'))
        ryb = ry[R0:R0 + v.shape[0], C0:C0 + v.shape[1]]
        for a in range(2):
            for b in range(2):
                j = (2 * i1 + a) * n2 + (2 * i2 + b)
                rx = m[j] / stc.m[i]
                child = (v * rx) * ryb
                rr, cc, dd, dr = truncate_box(R0, C0, child, tau)
                boxes[j] = [rr, cc, dd]
                dropped += dr
    eps_p_f = stc.eps_p if eps_p_f is None else float(eps_p_f)
    st = OracleState(N1, N2, s, eps_p_f, stc.h / 2.0, np.asarray(mu_f, np.float64),
                     np.asarray(nu_f, np.float64), m, n1, n2, boxes)
    st.dropped = stc.dropped + dropped
    if stc.alpha.get("A") is not None:   # R25': eps_c / eps_f = 4 eps'_c / eps'_f
        st.alpha["A"] = (4.0 * stc.eps_p / eps_p_f) * np.kron(stc.alpha["A"], np.ones((2, 2)))
    return st


def layers(mu: np.ndarray, nu: np.ndarray, levels: int):
    """[(mu_0, nu_0), ..., (mu_{L-1}, nu_{L-1})], coarsest first (R23)."""
    out = [(np.asarray(mu, np.float64), np.asarray(nu, np.float64))]
    for _ in range(levels - 1):
        a, b = out[0]
        out.insert(0, (coarsen(a), coarsen(b)))
    return out


def eps_stages(eps_p: float, eps_scale: float):
    """R24': the eps' of the stages of one layer, eps' F, eps' F / 2, ...,
    eps' (F = eps_scale >= 1)."""
    out = [float(eps_p) * float(eps_scale)]
    while out[-1] > eps_p * (1 + 1e-12):
        out.append(max(float(eps_p), out[-1] / 2.0))
    return out


def multiscale_solve(mu, nu, s: int, eps_p: float, levels: int, E: int, err: float = 1e-4,
                     conv: float = 1e-4, max_cycles: int = 1000, hybrid: bool = True, fixed_iter: int = 0,
                     tau: float = 1e-15, callback=None, eps_scale: float = 1.0, eps_stage_cycles: int = 0):
    """Coarse-to-fine hybrid domain decomposition (R23-R25, R24' for
    eps_scale > 1).  The physical domain is [-1, 1]^2 on every layer
    (h_l = 2 / N_l).  Per layer and eps stage: cycles of (A, B[, FlowUpdate])
    until both sweep-entry errors / ||mu|| <= conv (reading R14) or
    max_cycles (per stage; stages before the last run eps_stage_cycles cycles
    when > 0).  Supplies q_i = m_i 2^E (exact, R11) with the same
    E on every layer.  Returns (final state, per-layer records; "cycles" sums
    the stages, "converged" is the last stage's)."""
    lay = layers(mu, nu, levels)
    hist = []
    st = None
    stages = eps_stages(eps_p, eps_scale)
    for lv, (mu_l, nu_l) in enumerate(lay):
        h = 2.0 / mu_l.shape[0]
        st = (product_state(mu_l, nu_l, s, stages[0], h, tau) if st is None
              else refine_state(st, mu_l, nu_l, tau, eps_p_f=stages[0]))
        q = np.rint(st.m * 2.0 ** E).astype(np.int64)
        total = float(mu_l.sum())
        rec = {"level": lv, "N": mu_l.shape[0], "cycles": 0, "converged": False, "flows": 0}
        for si, ep in enumerate(stages):
            if si > 0:
                set_eps(st, ep)
            rec["converged"] = False
            last = si == len(stages) - 1
            for cyc in range(max_cycles if (last or eps_stage_cycles <= 0) else eps_stage_cycles):
                e0 = []
                for kind in ("A", "B"):
                    r = domdec_sweep(st, kind, err=err, fixed_iter=fixed_iter, tau=tau)
                    e0.append(r["e0_sum"] / total)
                if hybrid:
                    fu = flow_update(st, q, tau=tau)
                    rec["flows"] += int(not fu["stationary"])
                rec["cycles"] += 1
                if callback:
                    callback(lv, rec["cycles"] - 1, st, e0)
                if max(e0) <= conv:
                    rec["converged"] = True
                    break
        rec["l1"] = marginal_errors(st)
        hist.append(rec)
    return st, hist
