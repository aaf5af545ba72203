"""O3 — the flow update (§3.2, Def. flow-update) with the
product gluing candidate pi_hat_ij = mu_j/m_j (x) nu_i/m_i (Remark eps-gamma,
PAPER.md:550-552; reading R12) on the 5-point neighbourhood.
Test infrastructure (see oracle/__init__.py).

Steps follow §5.1:
  1. edge costs c_bar_ij = <c, pi_hat_ij - pi_hat_ii> (Eq. edge-cost
     PAPER.md:419-421) by direct double sums;
  2. min-cost flow (Eq. MinCostFlow PAPER.md:378-381 with the divergence
     constraint PAPER.md:350-354) — exact LP on integer data (reading R11);
  3. new basic-cell Y-marginals nu_hat_j = sum_i w_ij nu_i/m_i
     (Lemma, Eq. flow-update-cell-marginals PAPER.md:453-456).
Arc order per source cell: 0 self, 1 up, 2 down, 3 left, 4 right.
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp
from scipy.optimize import linprog

from .domdec import truncate_box

ARC_D = ((0, 0), (-1, 0), (1, 0), (0, -1), (0, 1))
COST_SCALE = 1024.0  # C_ij = round_half_even(c_bar_ij [px^2] * 2^10), reading R11


def neighbour(i: int, a: int, n1: int, n2: int) -> int:
    """Index of the a-th neighbour of basic cell i, or -1 outside the grid."""
    i1, i2 = divmod(i, n2)
    j1, j2 = i1 + ARC_D[a][0], i2 + ARC_D[a][1]
    if 0 <= j1 < n1 and 0 <= j2 < n2:
        return j1 * n2 + j2
    return -1


def edge_costs(st, Q=None, nus=None, cells=None):
    """c_bar (I x 5, px^2 units, NaN for arcs leaving the grid), c_bar_ii = 0.
    For i != j, with the product candidate:
        c_bar_ij = (1/m_i) sum_{x in X_j} sum_y |x - y|^2 (mu(x)/m_j) nu_i(y) - Q_i
    where pi_i is the last sweep's plan on X_i, Q_i = <c, pi_i>/m_i
    (pi_hat_ii = pi_i/m_i) and nu_i = P_Y pi_i its Y-marginal
    (reading R13: the paper instantiates pi_i for this step).
    Direct double sums over pixels (no moment shortcut).  Q and nus (list of
    (r0, c0, array)) may be given explicitly; by default both come from
    st.last.  cells: optional subset of source cells i (other rows stay NaN)."""
    if Q is None:
        Q = st.last["Q"]
        if nus is None:
            nus = st.last["nu_pre"]
    if nus is None:
        nus = st.boxes
    n1, n2, s = st.n1, st.n2, st.s
    I = n1 * n2
    cbar = np.full((I, 5), np.nan)
    for i in (range(I) if cells is None else cells):
        r0, c0, d = nus[i]
        yr, yc = np.nonzero(d > 0)
        vals = d[yr, yc]
        Y1 = (yr + r0).astype(np.float64)
        Y2 = (yc + c0).astype(np.float64)
        cbar[i, 0] = 0.0
        for a in range(1, 5):
            j = neighbour(i, a, n1, n2)
            if j < 0:
                continue
            j1, j2 = divmod(j, n2)
            xr, xc = np.meshgrid(np.arange(j1 * s, (j1 + 1) * s), np.arange(j2 * s, (j2 + 1) * s),
                                 indexing="ij")
            xr, xc = xr.ravel().astype(np.float64), xc.ravel().astype(np.float64)
            mux = st.mu[xr.astype(int), xc.astype(int)]
            d2 = (xr[:, None] - Y1[None, :]) ** 2 + (xc[:, None] - Y2[None, :]) ** 2
            tot = float(np.sum(d2 * mux[:, None] * vals[None, :]))
            cbar[i, a] = tot / (st.m[i] * st.m[j]) - Q[i]
    return cbar


def gamma_conditional(st, i: int, j: int, eps_gamma_p: float, tol: float = 1e-12, max_iter: int = 200000):
    """The plan gamma_ij in Pi(mu_i/m_i, mu_j/m_j) of a gluing edge candidate
    (Def. glued-plan): the optimal entropic plan for the cost
    |x - x'|^2 with regularisation eps_gamma_p (pixel^2 units; Remark
    eps-gamma PAPER.md:543-559: eps -> inf gives the product coupling, eps -> 0
    an optimal plan), by dense log-domain Sinkhorn (with eps-scaling) to an L1
    marginal error <= tol.  Returned as its disintegration against the first marginal,
    gamma~(x' | x) = gamma(x, x') / (mu(x) / m_i) (rows x in X_i, columns
    x' in X_j, both row-major), and the pixel coordinates of X_i and X_j."""
    s, n2 = st.s, st.n2
    from .partitions import cell_pixels
    from .sinkhorn import lse, sqdist
    ri, ci = cell_pixels(i, n2, s)
    rj, cj = cell_pixels(j, n2, s)
    xi = np.stack([ri, ci], 1).astype(np.float64)
    xj = np.stack([rj, cj], 1).astype(np.float64)
    pa = st.mu[ri, ci] / st.m[i]
    pb = st.mu[rj, cj] / st.m[j]
    Cm = sqdist(xi, xj) / eps_gamma_p
    la, lb = np.log(pa), np.log(pb)
    D = sqdist(xi, xj)
    # eps-scaling (a standard device for small eps, whose plain Sinkhorn
    # iteration contracts like 1 - exp(-max c / eps)): halve eps from max c
    # down to eps_gamma_p, warm-starting the potentials (in units of the
    # current eps, rescaled at each stage), then iterate to tol
    eps_stages = []
    e = max(float(D.max()), eps_gamma_p)
    while e > eps_gamma_p:
        eps_stages.append(e)
        e /= 2.0
    eps_stages.append(eps_gamma_p)
    a = np.zeros(len(pa))
    b = np.zeros(len(pb))
    prev = eps_stages[0]
    for k, e in enumerate(eps_stages):
        a *= prev / e
        b *= prev / e
        prev = e
        Cm = D / e
        last = k == len(eps_stages) - 1
        for _ in range(max_iter if last else 200):
            b = -lse(a[:, None] + la[:, None] - Cm, axis=0)
            a = -lse(b[None, :] + lb[None, :] - Cm, axis=1)
            if last:
                g = np.exp(a[:, None] + b[None, :] - Cm + la[:, None] + lb[None, :])
                if np.abs(g.sum(axis=0) - pb).sum() <= tol:
                    break
    g = np.exp(a[:, None] + b[None, :] - Cm + la[:, None] + lb[None, :])
    return g / g.sum(axis=1, keepdims=True), xi, xj


def glued_edge_costs(st, eps_gamma_p: float):
    """c_bar (I x 5, px^2) with gluing edge candidates (Def. glued-plan,
    PAPER.md:531-541) built from entropic plans gamma_ij
    (gamma_conditional) and the last sweep's plans pi_i (keep_plans=True):
        pi_hat_ij(x', y) = (1/m_i) sum_{x in X_i} gamma~(x' | x) pi_i(x, y),
        c_bar_ij = <c, pi_hat_ij> - <c, pi_i>/m_i
                 = (1/m_i) sum_x sum_x' sum_y gamma~(x'|x) pi_i(x,y) (|x'-y|^2 - |x-y|^2)
    by direct sums (reading R26: pi_i enters as is; its X-marginal is mu_i up
    to the Sinkhorn tolerance, the case in which this is exactly Eq.
    glued-plan).  c_bar_ii = 0; NaN on arcs leaving the grid."""
    from .partitions import composite_partition
    from .sinkhorn import sqdist
    plans = st.last.get("plans")
    if not plans:
        raise ValueError("glued_edge_costs needs the last sweep's plans (keep_plans=True)")
    n1, n2 = st.n1, st.n2
    I = n1 * n2
    cbar = np.full((I, 5), np.nan)
    comp = composite_partition(n1, n2, st.last["kind"])
    for k, members in enumerate(comp):
        R, Cc, ly, a, b, plan = plans[k]
        cell_of = (R // st.s) * n2 + (Cc // st.s)
        ly = np.asarray(ly, np.float64)
        for i in members:
            sel = cell_of == i
            P = plan[sel]                                   # pi_i(x, y), rows in X_i row-major
            X = np.stack([R[sel], Cc[sel]], 1).astype(np.float64)
            own = float(np.sum(P * sqdist(X, ly)))           # <c, pi_i> in px^2
            cbar[i, 0] = 0.0
            for aa in range(1, 5):
                j = neighbour(i, aa, n1, n2)
                if j < 0:
                    continue
                gt, xi, xj = gamma_conditional(st, i, j, eps_gamma_p)
                assert np.array_equal(xi, X)
                M = P @ sqdist(xj, ly).T                    # sum_y pi(x, y) |x' - y|^2
                cbar[i, aa] = (float(np.sum(gt * M)) - own) / st.m[i]
    return cbar


def integer_instance(cbar: np.ndarray, q: np.ndarray):
    """Integer data of the min-cost flow (reading R11): C_ij =
    round_half_even(c_bar_ij * 2^10) (0 on self / invalid arcs), q_i exact."""
    C = np.where(np.isnan(cbar), 0.0, np.rint(cbar * COST_SCALE)).astype(np.int64)
    C[:, 0] = 0
    return C, q.astype(np.int64)


def flow_objective(w: np.ndarray, C: np.ndarray) -> int:
    """sum_ij w_ij C_ij in exact (Python) integers."""
    return int(sum(int(a) * int(b) for a, b in zip(w.ravel().tolist(), C.ravel().tolist())))


def check_flow(w: np.ndarray, q: np.ndarray, n1: int, n2: int) -> bool:
    """Both divergence constraints of Eq. div-constraint,
    exactly, and w >= 0, and no mass on arcs leaving the grid."""
    I = n1 * n2
    if np.any(w < 0):
        return False
    out = w.sum(axis=1)
    inn = np.zeros(I, dtype=np.int64)
    for i in range(I):
        for a in range(5):
            j = neighbour(i, a, n1, n2)
            if j < 0:
                if w[i, a] != 0:
                    return False
                continue
            inn[j] += w[i, a]
    return bool(np.array_equal(out, q) and np.array_equal(inn, q))


def min_cost_flow(q: np.ndarray, C: np.ndarray, n1: int, n2: int):
    """Exact optimum of Eq. MinCostFlow on integer data:
    transportation LP (sources i, sinks j, arcs (i, j) in N) solved by a
    library simplex (HiGHS dual simplex — a library primitive; the paper uses
    OR-tools).  The constraint matrix is totally unimodular, so
    the vertex solution is integral; it is rounded and verified exactly.
    Returns (w (I x 5 int64), objective (exact int))."""
    I = n1 * n2
    var_i, var_a, var_j = [], [], []
    for i in range(I):
        for a in range(5):
            j = neighbour(i, a, n1, n2)
            if j >= 0:
                var_i.append(i)
                var_a.append(a)
                var_j.append(j)
    nv = len(var_i)
    cost = np.array([C[i, a] for i, a in zip(var_i, var_a)], dtype=np.float64)
    rows = np.concatenate([np.array(var_i), I + np.array(var_j)])
    cols = np.concatenate([np.arange(nv), np.arange(nv)])
    A = sp.csr_matrix((np.ones(2 * nv), (rows, cols)), shape=(2 * I, nv))
    b = np.concatenate([q, q]).astype(np.float64)
    res = linprog(cost, A_eq=A, b_eq=b, bounds=(0, None), method="highs-ds")
    if res.status != 0:
        raise RuntimeError(f"min-cost flow LP failed: {res.message}")
    x = np.rint(res.x).astype(np.int64)
    w = np.zeros((I, 5), dtype=np.int64)
    for k in range(nv):
        w[var_i[k], var_a[k]] = x[k]
    if not check_flow(w, q, n1, n2):
        raise RuntimeError("rounded LP solution is not an exact flow")
    return w, flow_objective(w, C)


def mcf_bruteforce(q: np.ndarray, C: np.ndarray, n1: int, n2: int):
    """Exhaustive enumeration of all integer flows (tiny instances, <= 6
    nodes, small q).  The LP is totally unimodular, so the integer optimum is
    the LP optimum.  Returns the optimal objective."""
    I = n1 * n2
    arcs = [[(a, neighbour(i, a, n1, n2)) for a in range(5) if neighbour(i, a, n1, n2) >= 0]
            for i in range(I)]

    def compositions(total, k):
        if k == 1:
            yield (total,)
            return
        for first in range(total + 1):
            for rest in compositions(total - first, k - 1):
                yield (first,) + rest

    options = [list(compositions(int(q[i]), len(arcs[i]))) for i in range(I)]
    best = None
    for choice in itertools.product(*options):
        inn = [0] * I
        obj = 0
        for i in range(I):
            for (a, j), v in zip(arcs[i], choice[i]):
                inn[j] += v
                obj += v * int(C[i, a])
        if inn == [int(x) for x in q]:
            if best is None or obj < best:
                best = obj
    return best


def apply_flow(st, w: np.ndarray, q: np.ndarray, tau: float = 1e-15):
    """nu_hat_j = sum_{i in N(j)} w_ij nu_i / m_i (Eq. flow-update-cell-
    marginals), realised as (w_ij / q_i) nu_i with the
    exact supplies q_i = m_i 2^E (reading R11).  Only cells with inflow from a
    neighbour (w_jj < q_j) change; their new box is the hull of the
    contributing boxes, followed by truncate + minimal box.
    Summation order: self, from up, from down, from left, from right.
    Returns the number of rewritten cells."""
    n1, n2 = st.n1, st.n2
    I = n1 * n2
    # source arc a' such that neighbour(i, a') = j, for i = neighbour(j, a)
    rev = {1: 2, 2: 1, 3: 4, 4: 3}
    new_boxes = list(st.boxes)
    changed = 0
    for j in range(I):
        if w[j, 0] == q[j]:
            continue
        changed += 1
        contrib = [(j, float(w[j, 0]) / float(q[j]))] if w[j, 0] > 0 else []
        for a in (1, 2, 3, 4):
            i = neighbour(j, a, n1, n2)
            if i < 0:
                continue
            wij = w[i, rev[a]]
            if wij > 0:
                contrib.append((i, float(wij) / float(q[i])))
        L1 = min(st.boxes[i][0] for i, _ in contrib)
        L2 = min(st.boxes[i][1] for i, _ in contrib)
        U1 = max(st.boxes[i][0] + st.boxes[i][2].shape[0] for i, _ in contrib)
        U2 = max(st.boxes[i][1] + st.boxes[i][2].shape[1] for i, _ in contrib)
        acc = np.zeros((U1 - L1, U2 - L2))
        for i, f in contrib:
            r0, c0, d = st.boxes[i]
            acc[r0 - L1:r0 - L1 + d.shape[0], c0 - L2:c0 - L2 + d.shape[1]] += f * d
        r0, c0, d, dr = truncate_box(L1, L2, acc, tau)
        st.dropped += dr
        new_boxes[j] = [r0, c0, d]
    st.boxes = new_boxes
    return changed


def flow_update(st, q: np.ndarray, tau: float = 1e-15):
    """FlowUpdate(pi) of Alg. 3: edge costs, exact min-cost
    flow, accept iff the optimal objective is strictly negative (the
    stationary flow has objective 0), then apply.
    Returns dict(stationary, objective, changed, w, C, cbar)."""
    cbar = edge_costs(st)
    C, q = integer_instance(cbar, q)
    w, obj = min_cost_flow(q, C, st.n1, st.n2)
    out = {"objective": obj, "w": w, "C": C, "cbar": cbar, "changed": 0}
    if obj < 0:
        out["changed"] = apply_flow(st, w, q, tau)
        out["stationary"] = False
    else:
        out["stationary"] = True
    return out
