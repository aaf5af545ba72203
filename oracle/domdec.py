"""O2 — one domain-decomposition sweep on bounding-box state
(Alg. 1 PAPER.md:261-285 realised as Alg. 4 PAPER.md:1209-1241 without
batching).  Test infrastructure (see oracle/__init__.py).

State = basic-cell Y-marginals nu_i in bounding-box form (PAPER.md:311-322,
1115) plus the X-potential a of the last sweep on each partition (the warm
start alpha^init of Alg. 4, reading R7).  Everything fp64, global gauge.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .partitions import basic_partition, composite_partition
from .sinkhorn import cell_sinkhorn


@dataclass
class OracleState:
    N1: int
    N2: int
    s: int
    eps_p: float          # eps / h^2
    h: float
    mu: np.ndarray        # (N1, N2) fp64
    nu: np.ndarray        # (N1, N2) fp64
    m: np.ndarray         # basic masses (I,)
    n1: int
    n2: int
    boxes: list           # per basic cell: [r0, c0, data (e1, e2) fp64]
    alpha: dict = field(default_factory=lambda: {"A": None, "B": None})
    dropped: float = 0.0  # truncation ledger (reading R9)
    last: dict = field(default_factory=dict)  # by-products of the last sweep

    @property
    def eps(self) -> float:
        return self.eps_p * self.h * self.h


def init_state(mu, nu, s, eps_p, h, off, ext, pos, data) -> OracleState:
    """Initial state from the generator's basic-cell boxes (pi^0, reading R17)."""
    N1, N2 = mu.shape
    n1, n2, m = basic_partition(mu, s)
    boxes = []
    for i in range(n1 * n2):
        e1, e2 = int(ext[i, 0]), int(ext[i, 1])
        d = np.asarray(data[pos[i]:pos[i] + e1 * e2], dtype=np.float64).reshape(e1, e2).copy()
        boxes.append([int(off[i, 0]), int(off[i, 1]), d])
    return OracleState(N1, N2, s, float(eps_p), float(h), np.asarray(mu, np.float64),
                       np.asarray(nu, np.float64), m, n1, n2, boxes)


def basic_to_composite(boxes, members):
    """nu_J = sum_{i in J} nu_i on the hull box (App. A.1 Eq.
    get-composite-cell-marginal PAPER.md:1128-1133; Alg. 1 line 3
    PAPER.md:274).  Summation in member order.  Returns (L1, L2, nuJ)."""
    L1 = min(boxes[i][0] for i in members)
    L2 = min(boxes[i][1] for i in members)
    U1 = max(boxes[i][0] + boxes[i][2].shape[0] for i in members)
    U2 = max(boxes[i][1] + boxes[i][2].shape[1] for i in members)
    nuJ = np.zeros((U1 - L1, U2 - L2))
    for i in members:
        r0, c0, d = boxes[i]
        nuJ[r0 - L1:r0 - L1 + d.shape[0], c0 - L2:c0 - L2 + d.shape[1]] += d
    return L1, L2, nuJ


def balance(parts, targets):
    """Balance (Alg. 4 line 6; the procedure is deferred to
    BoSch2020 §6, PAPER.md:1205 — reading R8).  parts: list of arrays (same
    shape) nu_k, k in J; targets t_k with sum t_k = sum ||nu_k||.  With
    M_k = ||nu_k||, delta_k = M_k - t_k, donors (delta > 0) send
    f_dr = delta_d (-delta_r) / Delta to each receiver r (Delta = sum of the
    donor deltas), pixel by pixel:
        tr_dr(y) = f_dr [ theta_d nu_d(y) nu_r(y) / (nu_J(y) T_dr)
                          + (1 - theta_d) nu_d(y) / M_d ],
        T_dr = sum_y nu_d nu_r / nu_J,  nu_J = sum_k nu_k,
    i.e. mass moves where donor and receiver are both present (overlap
    transfer), blended with a transfer in the donor's own shape only as much
    as needed to stay non-negative: with L_d = sum_r f_dr / T_dr and
    l_d = delta_d / M_d < 1, theta_d = 1 if L_d <= 1, else
    (1 - l_d) / (L_d - l_d) (theta_d = 0 if some T_dr = 0).  The rule is
    continuous in its inputs, preserves sum_k nu_k pointwise, gives
    ||nu_k|| = t_k and keeps nu_k >= 0."""
    mass = np.array([p.sum() for p in parts])
    delta = mass - np.asarray(targets)
    donors = np.flatnonzero(delta > 0)
    recv = np.flatnonzero(delta < 0)
    if len(donors) == 0 or len(recv) == 0:
        return [p.copy() for p in parts]
    D = float(delta[donors].sum())
    nuJ = np.zeros_like(parts[0])
    for p in parts:
        nuJ = nuJ + p
    safe = np.where(nuJ > 0, nuJ, 1.0)
    out = [p.copy() for p in parts]
    for d in donors:
        T = {r: float(np.sum(parts[d] * parts[r] / safe)) for r in recv}
        f = {r: delta[d] * (-delta[r]) / D for r in recv}
        if any(T[r] <= 0 for r in recv):
            theta = 0.0
        else:
            L = sum(f[r] / T[r] for r in recv)
            l = delta[d] / mass[d]
            theta = 1.0 if L <= 1.0 else (1.0 - l) / (L - l)
        for r in recv:
            tr = f[r] * (1.0 - theta) / mass[d] * parts[d]
            if theta > 0:
                tr = tr + f[r] * theta / T[r] * parts[d] * parts[r] / safe
            out[d] = out[d] - tr
            out[r] = out[r] + tr
    return out


def truncate_box(r0: int, c0: int, d: np.ndarray, tau: float):
    """Truncate (Alg. 4 line 7; threshold 1e-15 PAPER.md:1265):
    entries < tau become 0 (reading R9: no renormalisation), then the minimal
    bounding box of the non-zeros (bottom-left corner offset
    PAPER.md:1123).  Returns (r0', c0', d', dropped_mass)."""
    d = d.copy()
    small = d < tau
    dropped = float(d[small].sum())
    d[small] = 0.0
    nz = np.argwhere(d > 0)
    if len(nz) == 0:
        raise ValueError("truncation annihilated a basic cell")
    a1, a2 = nz.min(axis=0)
    b1, b2 = nz.max(axis=0) + 1
    return r0 + int(a1), c0 + int(a2), d[a1:b1, a2:b2].copy(), dropped


def composite_geometry(st: OracleState, members):
    """X-block of a composite cell: pixel rows/cols (row-major) and per pixel
    the member index it belongs to."""
    s, n2 = st.s, st.n2
    rows = sorted({i // n2 for i in members})
    cols = sorted({i % n2 for i in members})
    pr = np.arange(rows[0] * s, (rows[-1] + 1) * s)
    pc = np.arange(cols[0] * s, (cols[-1] + 1) * s)
    R, Cc = np.meshgrid(pr, pc, indexing="ij")
    R, Cc = R.ravel(), Cc.ravel()
    cell_of = (R // s) * n2 + (Cc // s)
    return R, Cc, cell_of


def domdec_sweep(st: OracleState, kind: str, err: float = 1e-4, fixed_iter: int = 0,
                 max_iter: int = 2000, tau: float = 1e-15, keep_plans: bool = False,
                 cells=None):
    """DomDecIter(pi, J_kind) (Alg. 1) in the realisation of
    Alg. 4: for every composite cell J of the partition,
      1. nu_J = BasicToComposite;
      2. warm start a = alpha_kind on X_J, zero on the partition's first sweep
         (reading R7);
      3. cell Sinkhorn until the stopping rule;
      4. CompositeToBasic: nu_i(y) = sum_{x in X_i} pi_J(x, y)
         (direct partial sums);
      5. Balance (reading R8) to t_i = m_i ||nu_J|| / mu(X_J);
      6. Truncate + minimal box;
      7. store a.
    By-products kept in st.last: per basic cell Q_i = <c, pi_i>/m_i in px^2
    and the pre-balance cell marginal nu_i^pre = P_Y pi_i (reading R13), plan
    X-marginal per pixel, per-cell (iters, e0, e).

    cells: optional list of composite-cell indices to process (sampled parity
    at full size); then the state is NOT advanced and the per-cell results are
    returned instead.
    Returns a stats dict.
    """
    comp = composite_partition(st.n1, st.n2, kind)
    s = st.s
    sample_mode = cells is not None
    todo = range(len(comp)) if cells is None else cells
    new_boxes = [None] * (st.n1 * st.n2)
    alpha_old = st.alpha[kind]
    alpha_new = np.zeros((st.N1, st.N2)) if alpha_old is None else alpha_old.copy()
    Q = np.zeros(st.n1 * st.n2)
    nu_pre = [None] * (st.n1 * st.n2)
    PX = np.zeros((st.N1, st.N2))
    stats = {"iters": [], "e0": [], "e": [], "dropped": 0.0, "mass_X": []}
    plans = {}
    results = {}
    for k in todo:
        members = comp[k]
        L1, L2, nuJ = basic_to_composite(st.boxes, members)
        R, Cc, cell_of = composite_geometry(st, members)
        mu_x = st.mu[R, Cc]
        kx = np.stack([R, Cc], axis=1)
        yr, yc = np.nonzero(nuJ > 0)
        ly = np.stack([yr + L1, yc + L2], axis=1)
        nu_y = nuJ[yr, yc]
        a0 = np.zeros(len(R)) if alpha_old is None else alpha_old[R, Cc]
        a, b, plan, it, e0, e = cell_sinkhorn(mu_x, kx, nu_y, ly, st.eps_p, a0, err,
                                              fixed_iter, max_iter)
        massJ = float(nuJ.sum())
        muXJ = float(mu_x.sum())
        parts = []
        for i in members:
            sel = cell_of == i
            part = np.zeros_like(nuJ)
            part[yr, yc] = plan[sel].sum(axis=0)
            parts.append(part)
            nu_pre[i] = (L1, L2, part.copy())
            d2 = (kx[sel, 0:1] - ly[None, :, 0]) ** 2 + (kx[sel, 1:2] - ly[None, :, 1]) ** 2
            Q[i] = float(np.sum(d2 * plan[sel])) / st.m[i]
        PX[R, Cc] = plan.sum(axis=1)
        targets = [st.m[i] * massJ / muXJ for i in members]
        parts = balance(parts, targets)
        cell_out = {}
        for i, p in zip(members, parts):
            r0, c0, d, dr = truncate_box(L1, L2, p, tau)
            new_boxes[i] = [r0, c0, d]
            cell_out[i] = (r0, c0, d)
            stats["dropped"] += dr
        alpha_new[R, Cc] = a
        stats["iters"].append(it)
        stats["e0"].append(e0)
        stats["e"].append(e)
        stats["mass_X"].append(muXJ)
        if keep_plans:
            plans[k] = (R, Cc, ly, a, b, plan)
        if sample_mode:
            results[k] = {"boxes": cell_out, "a": a, "R": R, "C": Cc, "L": (L1, L2), "nuJ": nuJ,
                          "iters": it, "e0": e0, "e": e,
                          "Q": {i: Q[i] for i in members}, "nu_pre": {i: nu_pre[i] for i in members},
                          "PX": plan.sum(axis=1)}
    if sample_mode:
        return results
    st.boxes = new_boxes
    st.alpha[kind] = alpha_new
    st.dropped += stats["dropped"]
    st.last = {"kind": kind, "Q": Q, "PX": PX, "nu_pre": nu_pre, "plans": plans if keep_plans else None}
    stats["e0_sum"] = float(np.sum(stats["e0"]))
    stats["e_sum"] = float(np.sum(stats["e"]))
    return stats
