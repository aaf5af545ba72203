"""Pins of the oracle's diagnostics (App. A.2.2): primal
score, stitched dual potential (reading R15), exact Y-response and the
primal-dual gap.  CPU only; each test names the fact it pins (closed forms,
strong/weak duality, invariance under per-cell constants)."""
import types

import numpy as np
import pytest

import oracle as O
from synth import make_problem


def _state(p):
    return O.init_state(p.mu, p.nu, p.s, p.eps_prime, p.h, p.init_off, p.init_ext,
                        p.init_pos, p.init_data)


def _fake_state(n1, n2, s, rng):
    N1, N2 = n1 * s, n2 * s
    mu = rng.uniform(0.5, 1.5, (N1, N2))
    return types.SimpleNamespace(n1=n1, n2=n2, s=s, N1=N1, N2=N2, mu=mu / mu.sum(), alpha={})


def _cell_constants(n1, n2, s, kind, rng):
    """Per-pixel field that is constant on each composite cell of `kind`."""
    out = np.zeros((n1 * s, n2 * s))
    for J in O.composite_partition(n1, n2, kind):
        v = rng.normal() * 10
        for i in J:
            i1, i2 = divmod(i, n2)
            out[i1 * s:(i1 + 1) * s, i2 * s:(i2 + 1) * s] = v
    return out


@pytest.mark.parametrize("n1,n2", [(4, 4), (6, 8), (5, 7), (2, 2), (1, 3)])
def test_stitch_recovers_global_potential(n1, n2):
    """If every cell potential is one global potential plus a cell constant
    (the gauge freedom of each cell problem), stitching
    returns that potential up to one global constant, for any grid shape
    (odd counts clip the last A-cells)."""
    rng = np.random.default_rng(n1 * 10 + n2)
    s = 2
    st = _fake_state(n1, n2, s, rng)
    g = rng.normal(size=(st.N1, st.N2))
    st.alpha["A"] = g + _cell_constants(n1, n2, s, "A", rng)
    st.alpha["B"] = g + _cell_constants(n1, n2, s, "B", rng)
    a = O.stitch_alpha(st)
    d = a - g
    np.testing.assert_allclose(d, d.flat[0], atol=1e-11)


def test_stitch_hand_example():
    """Two A-cells in a row (n = 2 x 4, s = 1): A0 = 0, A1 = 5 everywhere;
    the B-cell joining them (basic columns 1, 2) holds 1 on column 1 and 4 on
    column 2.  Path A0 -> B -> A1: offset = (1 - 0) + (5 - 4) = 2, so
    alpha† = 0 on A0 and 5 - 2 = 3 on A1 (R15 comb tree)."""
    st = types.SimpleNamespace(n1=2, n2=4, s=1, N1=2, N2=4, mu=np.full((2, 4), 1 / 8), alpha={})
    st.alpha["A"] = np.array([[0, 0, 5, 5], [0, 0, 5, 5]], float)
    st.alpha["B"] = np.array([[7, 1, 4, 9], [7, 1, 4, 9]], float)
    a = O.stitch_alpha(st)
    np.testing.assert_allclose(a, [[0, 0, 3, 3], [0, 0, 3, 3]], atol=1e-14)


def test_y_response_dirac_closed_form():
    """mu = delta at x0: b(y) = |x0 - y|^2 / eps' - a(x0) exactly."""
    st = types.SimpleNamespace(N1=6, N2=5, eps_p=3.0)
    mu = np.zeros((6, 5))
    mu[2, 3] = 1.0
    st.mu = mu
    a = np.random.default_rng(0).normal(size=(6, 5))
    b = O.y_response(st, a)
    l1, l2 = np.meshgrid(np.arange(6), np.arange(5), indexing="ij")
    np.testing.assert_allclose(b, ((l1 - 2) ** 2 + (l2 - 3) ** 2) / 3.0 - a[2, 3], atol=1e-12)


def test_dual_equals_primal_at_dense_optimum():
    """Strong duality for entropic OT: at the dense
    Sinkhorn fixed point, y_response(a*) = b* and D(a*, b*) = E(pi*)."""
    p = make_problem("gm", 8, 2, eps_factor=2.0, theta_deg=20, seed=3)
    st = _state(p)
    plan, a, b, xs, ys = O.dense_sinkhorn(p.mu, p.nu, p.eps_prime, tol=1e-14)
    A = np.zeros(p.mu.size)
    A[xs] = a
    A = A.reshape(p.mu.shape)
    by = O.y_response(st, A).ravel()[ys]
    np.testing.assert_allclose(by, b, atol=1e-9)
    P = np.zeros((p.mu.size, p.nu.size))
    P[np.ix_(xs, ys)] = plan
    B = np.zeros(p.nu.size)
    B[ys] = b
    E = O.primal_score(st, P)
    D = O.dual_score(st, A, B.reshape(p.nu.shape))
    assert abs(E - D) <= 1e-10 * abs(E)


def test_primal_cells_equal_dense_and_gap_closes():
    """The per-cell primal equals the primal of the materialised plan (the
    X-blocks are disjoint); weak duality D <= E holds along domdec, and the
    gap closes as domdec converges to the global minimiser (PAPER.md:45,
    212; Table rows)."""
    p = make_problem("gm", 16, 2, eps_factor=2.0, theta_deg=20, seed=0)
    st = _state(p)
    gaps = []
    for k in range(40):
        O.domdec_sweep(st, "AB"[k % 2], err=1e-11, keep_plans=True)
        if k in (1, 9, 39):
            E = O.primal_score(st)
            if k == 1:
                Ed = O.primal_score(st, O.dense_state_plan(st))
                assert abs(E - Ed) <= 1e-12 * abs(E)
            E2, D, gap = O.pd_gap(st)
            assert E2 == E
            assert gap >= -1e-12
            gaps.append(gap)
    # the rotated initial coupling is far from optimal; the gap then decays
    # (geometrically for pure domdec on this tiny problem)
    assert gaps[0] > 1e-4
    assert gaps[0] > gaps[1] > gaps[2]
    assert gaps[2] < 0.1 * gaps[0]
