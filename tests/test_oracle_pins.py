"""Pins of the oracle against what the paper and mathematics fix (CPU only).

Each test names the passage or fact it pins.  None of them re-types the
oracle's own formula: they use closed forms, brute force, independent
identities (marginals, strong/weak duality, the Lemma identities of §3.2) or
special cases that reduce to a hand formula.
"""
import math

import numpy as np
import pytest

import oracle as O
from oracle.flow import check_flow, neighbour
from oracle.sinkhorn import sqdist
from synth import make_problem, random_flow, random_mcf_instance


def _state(p):
    return O.init_state(p.mu, p.nu, p.s, p.eps_prime, p.h, p.init_off, p.init_ext,
                        p.init_pos, p.init_data)


# ---------------------------------------------------------------- Sinkhorn

def test_dense_sinkhorn_2x2_closed_form(golden):
    """SPEC.md:137 example; closed form from Prop. optimal couplings."""
    g = golden("sinkhorn_2x2.json")
    mu = np.array(g["mu"]).reshape(g["grid_shape"])
    nu = np.array(g["nu"]).reshape(g["grid_shape"])
    plan, a, b, xs, ys = O.dense_sinkhorn(mu, nu, g["eps_prime"], tol=1e-15)
    np.testing.assert_allclose(plan, np.array(g["plan"]), rtol=0, atol=1e-13)


def test_dense_sinkhorn_large_eps_is_product():
    """eps -> infinity: the entropic optimum tends to mu (x) nu (PAPER.md:746
    'pi = mu (x) nu already minimises the relative entropy')."""
    p = make_problem("gm", 8, 2, eps_factor=2.0, theta_deg=20, seed=1)
    prod = None
    devs = []
    for eps_p in (1e8, 1e9):
        plan, a, b, xs, ys = O.dense_sinkhorn(p.mu, p.nu, eps_p, tol=1e-15)
        prod = np.outer(p.mu.ravel()[xs], p.nu.ravel()[ys])
        devs.append(np.max(np.abs(plan / prod - 1)))
    # deviation is O(max c / eps') = O(98 / eps') and shrinks like 1/eps'
    assert devs[1] < 1e-6 and 5 < devs[0] / devs[1] < 20


def test_fig1_semi_discrete_limit():
    """Fig. 1 problem: mu uniform, nu two Diracs symmetric about
    the horizontal midline; as eps -> 0 the optimum splits mu along the
    bisector.  The limit cost is a direct sum over pixels."""
    N = 16
    mu = np.full((N, N), 1.0 / N ** 2)
    nu = np.zeros((N, N))
    ra, rb, cc = 3, 12, 7
    nu[ra, cc] = nu[rb, cc] = 0.5
    plan, a, b, xs, ys = O.dense_sinkhorn(mu, nu, 0.05, tol=1e-14)
    r = np.arange(N)[:, None].repeat(N, 1)
    c = np.arange(N)[None, :].repeat(N, 0)
    tgt = np.where(r <= 7, ra, rb)
    h = 2.0 / N
    limit = float(np.sum(mu * ((r - tgt) ** 2 + (c - cc) ** 2))) * h * h
    kx = np.stack([xs // N, xs % N], 1)
    ly = np.stack([ys // N, ys % N], 1)
    cost = float(np.sum(sqdist(kx, ly) * plan)) * h * h
    assert abs(cost - limit) < 1e-9 * limit


def test_cell_sinkhorn_strong_duality_and_marginals():
    """A cell solve at tight tolerance is optimal: Y-marginal exact after the
    Y-update, X-marginal within tolerance, and primal value
    E = <c,pi> + eps KL(pi|mu (x) nu) equals the dual value
    D = <a,mu> + <b,nu> + <1 - exp(a+b-c), mu (x) nu> (PAPER.md:1400-1410,
    strong duality certifies optimality; weak duality D <= E always)."""
    rng = np.random.default_rng(0)
    kx = np.stack(np.meshgrid(np.arange(4), np.arange(4), indexing="ij"), -1).reshape(-1, 2)
    ly = np.stack(np.meshgrid(np.arange(2, 9), np.arange(-1, 5), indexing="ij"), -1).reshape(-1, 2)
    mu = rng.uniform(0.5, 1.5, len(kx))
    mu /= mu.sum()
    nu = rng.uniform(0.1, 1.5, len(ly))
    nu /= nu.sum()
    eps_p = 4.0
    a, b, plan, it, e0, e = O.cell_sinkhorn(mu, kx, nu, ly, eps_p, np.zeros(len(kx)), 1e-13)
    np.testing.assert_allclose(plan.sum(0), nu, rtol=1e-12)
    assert np.abs(plan.sum(1) - mu).sum() <= 1e-12
    C = sqdist(kx, ly) / eps_p
    ref = np.outer(mu, nu)
    E = np.sum(C * plan) + np.sum(plan * np.log(plan / ref)) - plan.sum() + ref.sum()
    D = np.sum(a * mu) + np.sum(b * nu) + np.sum(ref * (1 - np.exp(a[:, None] + b[None, :] - C)))
    assert abs(E - D) < 1e-10
    # weak duality with perturbed potentials
    D2 = np.sum((a + 0.3) * mu) + np.sum((b - 0.1) * nu) + np.sum(
        ref * (1 - np.exp(a[:, None] + 0.3 + b[None, :] - 0.1 - C)))
    assert D2 <= E + 1e-14


def test_cell_sinkhorn_stopping_rule():
    """Err = 1e-4 stopping rule: the returned X-error is
    <= Err * mu(X_J) and equals the L1 X-marginal error of the plan."""
    rng = np.random.default_rng(1)
    kx = np.stack(np.meshgrid(np.arange(8), np.arange(8), indexing="ij"), -1).reshape(-1, 2)
    ly = np.stack(np.meshgrid(np.arange(-5, 12), np.arange(0, 14), indexing="ij"), -1).reshape(-1, 2)
    mu = rng.uniform(0.5, 1.5, len(kx)) * 1e-3
    nu = rng.uniform(0.1, 1.5, len(ly))
    nu *= mu.sum() / nu.sum()
    a, b, plan, it, e0, e = O.cell_sinkhorn(mu, kx, nu, ly, 4.0, np.zeros(len(kx)), 1e-4)
    assert e <= 1e-4 * mu.sum()
    assert abs(np.abs(plan.sum(1) - mu).sum() - e) < 1e-12 * mu.sum()
    assert it > 1 and e0 > e


# ---------------------------------------------------------------- partitions


def test_cell_sinkhorn_mass_defect():
    """Reading R6': when truncation (R9) leaves ||nu_J|| != mu(X_J), the plan
    after a Y-update has mass ||nu_J|| and the best attainable X-marginal is
    mu ||nu_J|| / mu(X_J).  The rescaled problem has the same minimiser up to
    that factor (the entropic plan of (mu, r nu) is r times the plan of
    (mu, nu) in the mu (x) nu_J reference), so: the solve still meets the
    tolerance, and its plan is exactly r times the balanced plan."""
    rng = np.random.default_rng(5)
    kx = np.array([(i, j) for i in range(4) for j in range(4)])
    mu = rng.uniform(0.5, 1.5, len(kx))
    ly = np.array([(i, j) for i in range(-1, 5) for j in range(-2, 5)])
    nu = rng.uniform(0.5, 1.5, len(ly))
    nu *= mu.sum() / nu.sum()
    r = 1.0 + 3e-4                       # defect above Err: unreachable without R6'
    _, _, p1, it1, _, e1 = O.cell_sinkhorn(mu, kx, nu, ly, 4.0, np.zeros(len(kx)), 1e-10)
    _, _, p2, it2, _, e2 = O.cell_sinkhorn(mu, kx, r * nu, ly, 4.0, np.zeros(len(kx)), 1e-10)
    assert it2 < 2000 and e2 <= 1e-10 * mu.sum()
    assert np.allclose(p2, r * p1, rtol=1e-8, atol=0)
    assert np.allclose(p2.sum(axis=1), r * mu, rtol=1e-9)

@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_partitions(n):
    """Def. partitions, Fig. PAPER.md:250: A and B each
    partition I; staggered grids give a connected partition graph
    (PAPER.md:779-795)."""
    A = O.composite_partition(n, n, "A")
    B = O.composite_partition(n, n, "B")
    assert len(A) == (n // 2) ** 2 and len(B) == (n // 2 + 1) ** 2
    for P in (A, B):
        flat = sorted(i for J in P for i in J)
        assert flat == list(range(n * n))
        assert all(1 <= len(J) <= 4 for J in P)
    assert O.partition_graph_connected(n, n)


def test_partition_graph_hand_cases():
    """Def. PartitionGraph on hand-made partitions of 2x2
    basic cells (n1 = n2 = 2): if B = A, each A-cell only meets its own copy
    (two components per cell pair: disconnected whenever there are >= 2
    cells); a B that straddles the A-cells joins them (connected).  Also a
    1 x 3 strip where B = {0}, {1, 2} and A = {0, 1}, {2}: path A0-B0,
    A0-B1, B1-A1 (connected); with B = {0, 1}, {2} = A it is disconnected."""
    A = [[0, 1], [2, 3]]
    assert not O.partition_graph_connected(2, 2, A=A, B=[[0, 1], [2, 3]])
    assert O.partition_graph_connected(2, 2, A=A, B=[[0], [1, 2], [3]])
    assert not O.partition_graph_connected(2, 2, A=[[0], [1], [2], [3]], B=[[0], [1], [2], [3]])
    assert O.partition_graph_connected(1, 3, A=[[0, 1], [2]], B=[[0], [1, 2]])
    assert not O.partition_graph_connected(1, 3, A=[[0, 1], [2]], B=[[0, 1], [2]])


def test_integer_instance_half_even_hand_case():
    """Reading R11: C_ij = round_half_even(c_bar_ij * 2^10), 0 on the self arc
    and on arcs leaving the grid (NaN); q exact.  Hand values on the exact
    half-integers of the cost quantum: 0.5 -> 0, 1.5 -> 2, 2.5 -> 2,
    -0.5 -> 0, -1.5 -> -2, 3.25 -> 3, -2.75 -> -3 (floor or ceil or round
    half away from zero each fail one of them)."""
    u = 1.0 / 1024.0
    cbar = np.array([[0.0, 0.5 * u, 1.5 * u, 2.5 * u, np.nan],
                     [7.0, -0.5 * u, -1.5 * u, 3.25 * u, -2.75 * u]])
    q = np.array([5, 9], dtype=np.int64)
    C, qq = O.integer_instance(cbar, q)
    assert C.dtype == np.int64 and qq.dtype == np.int64
    assert C.tolist() == [[0, 0, 2, 2, 0], [0, 0, -2, 3, -3]]
    assert qq.tolist() == [5, 9]


def test_zero_mass_cell_rejected():
    """m_i > 0 is required."""
    mu = np.ones((4, 4))
    mu[:2, :2] = 0
    with pytest.raises(ValueError):
        O.basic_partition(mu, 2)


# ---------------------------------------------------------------- bbox ops

def test_basic_to_composite_hull_and_mass():
    """Eq. get-composite-cell-marginal: disjoint boxes
    -> union box, masses add, entries placed at their offsets."""
    boxes = [[2, 3, np.array([[1.0, 2.0]])], [5, 1, np.array([[3.0], [4.0]])]]
    L1, L2, nuJ = O.basic_to_composite(boxes, [0, 1])
    assert (L1, L2) == (2, 1) and nuJ.shape == (5, 4)
    assert nuJ[0, 2] == 1 and nuJ[0, 3] == 2 and nuJ[3, 0] == 3 and nuJ[4, 0] == 4
    assert nuJ.sum() == 10


def test_balance_identities():
    """Balance (reading R8): masses reach the targets, the
    pointwise sum is unchanged, an already balanced cell is untouched."""
    rng = np.random.default_rng(2)
    parts = [rng.uniform(0, 1, (5, 6)) * (rng.uniform() < 0.7) for _ in range(4)]
    parts = [p + 1e-3 for p in parts]
    tot = sum(p.sum() for p in parts)
    t = rng.uniform(0.5, 1.5, 4)
    t *= tot / t.sum()
    out = O.balance(parts, t)
    np.testing.assert_allclose([o.sum() for o in out], t, rtol=1e-13)
    np.testing.assert_allclose(sum(out), sum(parts), rtol=1e-13)
    assert all((o >= 0).all() for o in out)
    same = O.balance(parts, [p.sum() for p in parts])
    for a, b in zip(same, parts):
        assert np.array_equal(a, b)
    # hand example: masses (0.6, 0.4) -> (0.5, 0.5): 0.1 moves
    # from cell 0 to cell 1 at their shared support point.
    p0 = np.array([[0.3, 0.3]])
    p1 = np.array([[0.4, 0.0]])
    o0, o1 = O.balance([p0, p1], [0.5, 0.5])
    np.testing.assert_allclose(o0, [[0.2, 0.3]])
    np.testing.assert_allclose(o1, [[0.5, 0.0]])
    # disjoint supports cannot exchange mass pointwise: the transfer falls
    # back to the donor's own shape (theta = 0)
    q0 = np.array([[0.6, 0.0]])
    q1 = np.array([[0.0, 0.4]])
    r0, r1 = O.balance([q0, q1], [0.5, 0.5])
    np.testing.assert_allclose(r0 + r1, q0 + q1)
    np.testing.assert_allclose([r0.sum(), r1.sum()], [0.5, 0.5])
    assert (r0 >= 0).all() and (r1 >= 0).all()
    np.testing.assert_allclose(r1, [[0.1, 0.4]])
    # continuity of the blend at the overlap-capacity threshold L = 1
    a0 = np.array([[0.5, 0.1]])
    a1 = np.array([[0.1, 0.3]])
    Tov = 0.5 * 0.1 / 0.6 + 0.1 * 0.3 / 0.4
    outs = []
    for dlt in (Tov * (1 - 1e-9), Tov * (1 + 1e-9)):
        m0, m1 = a0.sum(), a1.sum()
        outs.append(O.balance([a0, a1], [m0 - dlt, m1 + dlt]))
    np.testing.assert_allclose(outs[0][0], outs[1][0], rtol=1e-7)
    np.testing.assert_allclose(outs[0][1], outs[1][1], rtol=1e-7)


def test_truncate_box():
    """Truncate at tau and minimal box:
    strict '<', exact-tau survives, tau = 0 is a pure repack, mass ledger."""
    d = np.zeros((5, 6))
    d[1, 2] = 1.0
    d[3, 4] = 1e-15
    d[2, 1] = 0.9e-15
    r0, c0, out, dropped = O.truncate_box(10, 20, d, 1e-15)
    assert (r0, c0) == (11, 22) and out.shape == (3, 3)
    assert out[0, 0] == 1.0 and out[2, 2] == 1e-15 and dropped == 0.9e-15
    r0, c0, out, dropped = O.truncate_box(0, 0, d, 0.0)
    assert (r0, c0, out.shape, dropped) == (1, 1, (3, 4), 0.0)


# ---------------------------------------------------------------- domdec

def test_sweep_invariants_and_monotone_objective():
    """DomDecIter (Alg. 1): every sweep keeps the global
    Y-marginal (sum_i nu_i = nu up to the truncation ledger), sets
    ||nu_i|| = m_i (balance), and never increases the primal objective
    (block coordinate descent)."""
    p = make_problem("gm", 16, 2, eps_factor=2.0, theta_deg=20, seed=0)
    st = _state(p)
    prevE = math.inf
    for k in range(6):
        stt = O.domdec_sweep(st, "AB"[k % 2], err=1e-11, keep_plans=True)
        ex, ey = O.marginal_errors(st)
        assert ey <= 1e-14 + 2 * st.dropped
        masses = np.array([b[2].sum() for b in st.boxes])
        # ||nu_i|| = m_i ||nu_J|| / mu(X_J): exact up to the truncation ledger (R8, R9)
        np.testing.assert_allclose(masses, st.m, rtol=1e-13, atol=st.dropped)
        assert ex <= 1e-11 * 1.01
        E = O.primal_score(st)
        assert E <= prevE + 1e-12
        prevE = E


@pytest.mark.parametrize("kind,hybrid", [("gm", False), ("gm", True), ("bumps", True)])
def test_domdec_converges_to_dense_global_optimum(kind, hybrid):
    """Domain decomposition and the hybrid scheme converge to the unique
    minimiser (Prop. convergence-hybrid):
    brute-force dense global Sinkhorn on the tiny problem is the reference."""
    p = make_problem(kind, 16, 2, eps_factor=2.0, theta_deg=20, seed=0)
    st = _state(p)
    plan, a, b, xs, ys = O.dense_sinkhorn(p.mu, p.nu, p.eps_prime, tol=1e-14)
    N = p.N
    kx = np.stack([xs // N, xs % N], 1)
    ly = np.stack([ys // N, ys % N], 1)
    cost_star = float(np.sum(sqdist(kx, ly) * plan)) * p.h ** 2
    O.run(st, p.supplies(), 70 if kind == "gm" else 100, hybrid=hybrid, err=1e-9)
    cost = O.transport_cost(st)
    assert abs(cost - cost_star) < 1e-6 * cost_star


def test_fixed_point_at_global_optimum():
    """A globally optimal coupling is a fixed point of S_A and S_B
    (PAPER.md:825-827): starting from the dense optimum's basic-cell
    marginals, one A and one B sweep change the marginals by < 1e-8."""
    p = make_problem("gm", 16, 2, eps_factor=2.0, theta_deg=20, seed=3)
    plan, a, b, xs, ys = O.dense_sinkhorn(p.mu, p.nu, p.eps_prime, tol=1e-15)
    N, s, n = p.N, p.s, p.n
    st = _state(p)
    boxes = []
    for i in range(n * n):
        i1, i2 = divmod(i, n)
        rows = np.isin(xs // N // s, [i1]) & np.isin(xs % N // s, [i2])
        nu_i = np.zeros(N * N)
        nu_i[ys] = plan[rows].sum(0)
        boxes.append(O.truncate_box(0, 0, nu_i.reshape(N, N), 1e-15)[:3])
    st.boxes = [list(bx) for bx in boxes]
    before = [bx[2].copy() for bx in st.boxes]
    O.domdec_sweep(st, "A", err=1e-12)
    O.domdec_sweep(st, "B", err=1e-12)
    for (r0, c0, d), d0, bx0 in zip(st.boxes, before, boxes):
        full = np.zeros((N, N))
        full[r0:r0 + d.shape[0], c0:c0 + d.shape[1]] = d
        full0 = np.zeros((N, N))
        full0[bx0[0]:bx0[0] + d0.shape[0], bx0[1]:bx0[1] + d0.shape[1]] = d0
        assert np.abs(full - full0).sum() < 1e-8


# ---------------------------------------------------------------- flow update

def test_singleton_edge_costs_reduce_to_simple_formula():
    """Remark after Def. flow-update: for singleton cells
    (s = 1) the general cost <c, pi_hat_ij - pi_hat_ii> becomes Eq.
    CostCoefficientSimple:
        c_bar_ij = <c(x_j, .) - c(x_i, .), nu_i/m_i>."""
    p = make_problem("gm", 8, 1, eps_factor=2.0, theta_deg=20, seed=4)
    st = _state(p)
    n = p.n
    # pi_i/m_i for a singleton cell is delta_{x_i} (x) nu_i/m_i, so
    # Q_i = <c(x_i, .), nu_i/m_i>.
    Q = np.zeros(n * n)
    for i in range(n * n):
        r0, c0, d = st.boxes[i]
        yr, yc = np.nonzero(d > 0)
        Q[i] = np.sum(((yr + r0 - i // n) ** 2 + (yc + c0 - i % n) ** 2) * d[yr, yc]) / st.m[i]
    cbar = O.edge_costs(st, Q)
    for i in range(n * n):
        r0, c0, d = st.boxes[i]
        yr, yc = np.nonzero(d > 0)
        for a in range(1, 5):
            j = neighbour(i, a, n, n)
            if j < 0:
                continue
            cj = (yr + r0 - j // n) ** 2 + (yc + c0 - j % n) ** 2
            ci = (yr + r0 - i // n) ** 2 + (yc + c0 - i % n) ** 2
            simple = np.sum((cj - ci) * d[yr, yc]) / st.m[i]
            assert abs(cbar[i, a] - simple) < 1e-9 * max(1.0, abs(simple))


def _materialise_flow_plan(st, w, q):
    """pi_hat = sum_j sum_i w_ij pi_hat_ij (Eq. flow-update-new-plan,
    PAPER.md:425-434) with the product candidate mu_j/m_j (x) nu_i/m_i,
    nu_i = P_Y pi_i, for i != j and pi_hat_ii = pi_i/m_i, as a dense matrix."""
    N, s, n = st.N1, st.s, st.n1
    P = O.dense_state_plan(st)
    out = np.zeros_like(P)
    for i in range(n * n):
        i1, i2 = divmod(i, n)
        xi = np.array([(r) * N + c for r in range(i1 * s, (i1 + 1) * s) for c in range(i2 * s, (i2 + 1) * s)])
        r0, c0, d = st.last["nu_pre"][i]
        nu_i = np.zeros(N * N)
        nu_i[(np.arange(r0, r0 + d.shape[0])[:, None] * N + np.arange(c0, c0 + d.shape[1])[None, :]).ravel()] = d.ravel()
        for a in range(5):
            j = neighbour(i, a, n, n)
            if j < 0 or w[i, a] == 0:
                continue
            frac = w[i, a] / q[i]
            if a == 0:
                out[xi, :] += frac * P[xi, :]
            else:
                j1, j2 = divmod(j, n)
                xj = np.array([r * N + c for r in range(j1 * s, (j1 + 1) * s) for c in range(j2 * s, (j2 + 1) * s)])
                out[np.ix_(xj, np.arange(N * N))] += frac * np.outer(st.mu.ravel()[xj] / st.m[j], nu_i / st.m[i] * st.m[i])
    return P, out


def test_transport_change_identity_and_marginals():
    """Lemma transport-non-increasing, Eq. total-cost-update
    (PAPER.md:518-525): <c, pi_hat - pi> = sum w_ij c_bar_ij, and Lemma
    flow-preserves-marginals: pi_hat keeps both marginals
    and its basic-cell Y-marginals are Eq. flow-update-cell-marginals."""
    p = make_problem("gm", 8, 2, eps_factor=2.0, theta_deg=20, seed=5)
    st = _state(p)
    O.domdec_sweep(st, "A", err=1e-13, keep_plans=True)
    q = p.supplies()
    n = p.n
    w = random_flow(q, n, n, seed=7, n_cycles=60)
    assert check_flow(w, q, n, n)
    cbar = O.edge_costs(st)
    P, Phat = _materialise_flow_plan(st, w, q)
    N = p.N
    k = np.stack(np.meshgrid(np.arange(N), np.arange(N), indexing="ij"), -1).reshape(-1, 2)
    c = sqdist(k, k)
    lhs = float(np.sum(c * (Phat - P)))
    rhs = float(np.nansum(w / q[:, None] * st.m[:, None] * cbar))
    assert abs(lhs - rhs) < 1e-9 * (1 + abs(rhs))
    np.testing.assert_allclose(Phat.sum(1), P.sum(1), atol=1e-15)
    np.testing.assert_allclose(Phat.sum(0), P.sum(0), atol=1e-15)
    # apply_flow's cell marginals == P_Y of pi_hat restricted to X_j
    st2_boxes = [list(b) for b in st.boxes]
    O.apply_flow(st, w, q, tau=0.0)
    s = p.s
    for j in range(n * n):
        j1, j2 = divmod(j, n)
        xj = [r * N + cc for r in range(j1 * s, (j1 + 1) * s) for cc in range(j2 * s, (j2 + 1) * s)]
        ref = Phat[xj].sum(0).reshape(N, N)
        r0, c0, d = st.boxes[j]
        got = np.zeros((N, N))
        got[r0:r0 + d.shape[0], c0:c0 + d.shape[1]] = d
        if w[j, 0] == q[j]:
            # untouched cell keeps its stored nu_j (== P_Y pi_j up to balancing)
            r0b, c0b, db = st2_boxes[j]
            assert r0 == r0b and c0 == c0b and np.array_equal(d, db)
        else:
            assert np.abs(got - ref).sum() < 1e-12 + 1e-9 * ref.sum()


def test_product_coupling_costs_are_curl_free():
    """For pi = mu (x) nu every flow update is stationary: with
    the product candidate, c_bar_ij = f(j) - f(i) is a potential difference,
    so c_bar is antisymmetric and sums to zero around every plaquette."""
    N, s = 8, 2
    p = make_problem("gm", N, s, eps_factor=2.0, theta_deg=20, seed=6)
    st = _state(p)
    n = p.n
    nu = p.nu
    r0, c0 = np.nonzero(nu > 0)
    boxes = []
    for i in range(n * n):
        boxes.append(list(O.truncate_box(0, 0, nu * st.m[i], 0.0)[:3]))
    st.boxes = boxes
    # Q_i for pi_i = mu_i (x) nu: <c, mu_i/m_i (x) nu>
    Q = np.zeros(n * n)
    for i in range(n * n):
        i1, i2 = divmod(i, n)
        xr, xc = np.meshgrid(np.arange(i1 * s, (i1 + 1) * s), np.arange(i2 * s, (i2 + 1) * s), indexing="ij")
        mux = p.mu[xr, xc].ravel()
        d2 = (xr.ravel()[:, None] - r0[None, :]) ** 2 + (xc.ravel()[:, None] - c0[None, :]) ** 2
        Q[i] = np.sum(d2 * mux[:, None] * nu[r0, c0][None, :]) / st.m[i]
    cbar = O.edge_costs(st, Q)
    for i in range(n * n):
        for a, ra in ((1, 2), (2, 1), (3, 4), (4, 3)):
            j = neighbour(i, a, n, n)
            if j >= 0:
                assert abs(cbar[i, a] + cbar[j, ra]) < 1e-9 * (1 + abs(cbar[i, a]))
    for i1 in range(n - 1):
        for i2 in range(n - 1):
            i = i1 * n + i2
            cyc = cbar[i, 4] + cbar[i + 1, 2] + cbar[i + 1 + n, 3] + cbar[i + n, 1]
            assert abs(cyc) < 1e-9 * (1 + np.nanmax(np.abs(cbar)))


def test_mcf_two_node_example(golden):
    """SPEC.md:369 worked example of Eq. MinCostFlow."""
    g = golden("mcf_2node.json")
    q = np.array(g["q"], dtype=np.int64)
    C = np.array(g["C"], dtype=np.int64)
    w, obj = O.min_cost_flow(q, C, g["n1"], g["n2"])
    assert obj == g["objective"]
    assert np.array_equal(w, np.array(g["w"]))
    assert O.mcf_bruteforce(q, C, g["n1"], g["n2"]) == g["objective"]


@pytest.mark.parametrize("shape", [(1, 2), (1, 3), (2, 2), (2, 3), (1, 5)])
@pytest.mark.parametrize("seed", range(6))
def test_mcf_matches_bruteforce(shape, seed):
    """Exact LP optimum == exhaustive enumeration on <= 6 nodes;
    the optimum is <= 0 since the stationary flow is feasible."""
    n1, n2 = shape
    q, C = random_mcf_instance(n1, n2, seed=100 + seed, qmax=2 if n1 * n2 > 4 else 3, cmax=9)
    w, obj = O.min_cost_flow(q, C, n1, n2)
    assert check_flow(w, q, n1, n2)
    assert obj <= 0
    assert obj == O.mcf_bruteforce(q, C, n1, n2)


def test_apply_flow_special_cases():
    """Stationary flow -> identity; two singleton cells exchanging all mass
    swap their marginals (Eq. PiHatSimple)."""
    p = make_problem("gm", 4, 1, eps_factor=2.0, theta_deg=20, seed=8)
    st = _state(p)
    q = p.supplies()
    n = p.n
    before = [[b[0], b[1], b[2].copy()] for b in st.boxes]
    w = np.zeros((n * n, 5), dtype=np.int64)
    w[:, 0] = q
    assert O.apply_flow(st, w, q) == 0
    for a, b in zip(st.boxes, before):
        assert a[0] == b[0] and a[1] == b[1] and np.array_equal(a[2], b[2])
    # make cells 0 and 1 equal-mass, then swap them completely
    st.m[1] = st.m[0]
    q2 = q.copy()
    q2[1] = q2[0]
    w = np.zeros((n * n, 5), dtype=np.int64)
    w[:, 0] = q2
    w[0, 0] = 0
    w[1, 0] = 0
    w[0, 4] = q2[0]
    w[1, 3] = q2[1]
    O.apply_flow(st, w, q2, tau=0.0)
    assert st.boxes[0][0] == before[1][0] and st.boxes[0][1] == before[1][1]
    np.testing.assert_allclose(st.boxes[0][2], before[1][2], rtol=1e-15)
    np.testing.assert_allclose(st.boxes[1][2], before[0][2], rtol=1e-15)


def test_hybrid_flow_decreases_objective_and_stops():
    """Flow updates never increase the transport objective (Lemma
    PAPER.md:508-529), and with gluing candidates not the entropic objective
    either (Prop. PAPER.md:735-741); near the optimum they become stationary
    (PAPER.md:996)."""
    p = make_problem("bumps", 16, 2, eps_factor=0.5, theta_deg=90, seed=0)
    st = _state(p)
    q = p.supplies()
    hist = []
    for cyc in range(12):
        O.domdec_sweep(st, "A", err=1e-10)
        O.domdec_sweep(st, "B", err=1e-10, keep_plans=True)
        E0 = O.primal_score(st)
        c0 = O.transport_cost(st)
        fu = O.flow_update(st, q, tau=0.0)
        hist.append(fu["stationary"])
        if not fu["stationary"]:
            assert fu["objective"] < 0
            # the flow step's change of <c, pi> is sum w c_bar < 0 (in px^2):
            dc = float(np.nansum(fu["w"] / q[:, None] * st.m[:, None] * fu["cbar"])) * p.h ** 2
            assert dc < 0
    assert not hist[0]           # the T0 rotation has curl: the first flow moves mass
    assert all(hist[-3:])        # ... and the flows stop near the optimum


def test_y_update_at_dirac_closed_form():
    """mu = Dirac at k0: b(l) = |k0 - l|^2/eps' - a(k0) - log mu(k0) exactly."""
    mu = np.zeros((5, 7))
    mu[2, 3] = 0.5
    a = np.full((5, 7), 0.3)
    ls = [(0, 0), (2, 3), (4, 6), (1, 5)]
    b = O.y_update_at(a, mu, 2.0, ls)
    want = [((2 - r) ** 2 + (3 - c) ** 2) / 2.0 - 0.3 - np.log(0.5) for r, c in ls]
    assert np.allclose(b, want, rtol=0, atol=1e-14)


def test_y_update_at_brute_force_linear_domain():
    """Brute force in the linear domain on a 3x4 grid (plain loops, no LSE):
    exp(-b(l)) = sum_k mu(k) e^{a(k)} e^{-|k-l|^2/eps'}."""
    rng = np.random.default_rng(7)
    mu = rng.random((3, 4))
    mu[1, 2] = 0.0
    a = rng.normal(size=(3, 4))
    eps_p = 1.5
    ls = [(r, c) for r in range(3) for c in range(4)]
    b = O.y_update_at(a, mu, eps_p, ls)
    for j, (r, c) in enumerate(ls):
        s = 0.0
        for k1 in range(3):
            for k2 in range(4):
                s += mu[k1, k2] * np.exp(a[k1, k2]) * np.exp(-((k1 - r) ** 2 + (k2 - c) ** 2) / eps_p)
        assert abs(b[j] - (-np.log(s))) <= 1e-13
