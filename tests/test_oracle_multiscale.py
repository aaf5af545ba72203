"""Pins of the multiscale oracle (f3, oracle/multiscale.py; readings R23-R25)
against what the definitions and the mathematics fix, independently of the
oracle's own formulas: exact mass bookkeeping of coarsening, feasibility and
the coarse round trip of the refinement, the product coupling as a fixed
point of refinement, and convergence of the whole pipeline to the dense
global optimum (domdec converges to the unique minimiser, PAPER.md:45,
792-795)."""
import numpy as np
import pytest

import oracle as O
from oracle import multiscale as M
from synth import make_problem


def test_coarsen_hand_case_and_exact_mass():
    a = np.arange(16, dtype=np.float64).reshape(4, 4)
    c = M.coarsen(a)
    assert c.tolist() == [[0 + 1 + 4 + 5, 2 + 3 + 6 + 7], [8 + 9 + 12 + 13, 10 + 11 + 14 + 15]]
    p = make_problem("gm", 64, 2, theta_deg=20, seed=3)
    for lv in M.layers(p.mu, p.nu, 4):
        # dyadic counts: every layer sums to exactly 1 in fp64
        assert lv[0].sum() == 1.0 and lv[1].sum() == 1.0
    with pytest.raises(AssertionError):
        M.coarsen(np.ones((3, 4)))


def _y_marginal(st):
    acc = np.zeros((st.N1, st.N2))
    for r0, c0, d in st.boxes:
        acc[r0:r0 + d.shape[0], c0:c0 + d.shape[1]] += d
    return acc


def test_product_state_is_the_product_coupling():
    p = make_problem("gm", 16, 2, theta_deg=20, seed=1)
    st = M.product_state(p.mu, p.nu, 2, 4.0, 2.0 / 16)
    for i, (r0, c0, d) in enumerate(st.boxes):
        full = np.zeros_like(p.nu)
        full[r0:r0 + d.shape[0], c0:c0 + d.shape[1]] = d
        np.testing.assert_allclose(full, st.m[i] * p.nu, rtol=1e-15, atol=0)
    assert np.abs(_y_marginal(st) - p.nu).sum() <= 1e-15


def test_refine_feasible_and_round_trip():
    """R25: the refined coupling is feasible (||nu_i'|| = m_i', sum = nu up
    to the truncation ledger) and coarsening it back (children summed, Y
    pixels 2x2-summed) returns the coarse basic marginals."""
    p = make_problem("gm", 32, 2, theta_deg=20, seed=2)
    mu_c, nu_c = M.coarsen(p.mu), M.coarsen(p.nu)
    stc = M.product_state(mu_c, nu_c, 2, 4.0, 2.0 / 16)
    # a non-trivial coarse state: a few sweeps from the product coupling
    for kind in ("A", "B", "A"):
        O.domdec_sweep(stc, kind, err=1e-6)
    stf = M.refine_state(stc, p.mu, p.nu)
    led = stf.dropped - stc.dropped   # mass truncated by the refinement itself
    # the coarse state's own truncation ledger carries over to the Y-marginal
    assert np.abs(_y_marginal(stf) - p.nu).sum() <= stf.dropped + 1e-14
    for i, (r0, c0, d) in enumerate(stf.boxes):
        assert abs(d.sum() - stf.m[i]) <= 1e-13 * stf.m[i] + led
    for i in range(stc.n1 * stc.n2):
        i1, i2 = divmod(i, stc.n2)
        acc = np.zeros((stf.N1, stf.N2))
        for a in range(2):
            for b in range(2):
                r0, c0, d = stf.boxes[(2 * i1 + a) * stf.n2 + 2 * i2 + b]
                acc[r0:r0 + d.shape[0], c0:c0 + d.shape[1]] += d
        back = M.coarsen(acc)
        r0, c0, d = stc.boxes[i]
        ref = np.zeros_like(back)
        ref[r0:r0 + d.shape[0], c0:c0 + d.shape[1]] = d
        np.testing.assert_allclose(back, ref, rtol=1e-13, atol=led + 1e-300)


def test_refine_of_product_is_product():
    p = make_problem("gm", 32, 2, theta_deg=20, seed=4)
    stc = M.product_state(M.coarsen(p.mu), M.coarsen(p.nu), 2, 4.0, 2.0 / 16)
    stf = M.refine_state(stc, p.mu, p.nu)
    for i, (r0, c0, d) in enumerate(stf.boxes):
        full = np.zeros_like(p.nu)
        full[r0:r0 + d.shape[0], c0:c0 + d.shape[1]] = d
        np.testing.assert_allclose(full, stf.m[i] * p.nu, rtol=1e-14, atol=1e-300)


def test_multiscale_converges_to_dense_optimum():
    """The whole coarse-to-fine hybrid pipeline on a 16^2 GM pair (layers
    8^2, 16^2, s = 2, eps' = 4) reaches the dense global entropic optimum:
    transport cost within 1e-5 relative (the unique minimiser, PAPER.md:212,
    to which domdec converges)."""
    p = make_problem("gm", 16, 2, theta_deg=20, seed=0)
    st, hist = M.multiscale_solve(p.mu, p.nu, 2, 4.0, levels=2, E=p.E, err=1e-9, conv=1e-9, max_cycles=200)
    assert all(r["converged"] for r in hist), hist
    plan, a, b, xs, ys = O.dense_sinkhorn(p.mu, p.nu, 4.0, tol=1e-13)
    from oracle.sinkhorn import sqdist
    N = p.N
    cstar = float(np.sum(sqdist(np.stack([xs // N, xs % N], 1), np.stack([ys // N, ys % N], 1)) * plan)) * p.h ** 2
    assert abs(O.transport_cost(st) - cstar) < 1e-5 * cstar


def test_eps_stages_and_set_eps():
    """R24': stages eps' F, F/2, ..., 1 x eps'; set_eps keeps
    the physical potential alpha * eps'."""
    assert M.eps_stages(4.0, 4.0) == [16.0, 8.0, 4.0]
    assert M.eps_stages(4.0, 1.0) == [4.0]
    assert M.eps_stages(4.0, 3.0) == [12.0, 6.0, 4.0]
    p = make_problem("gm", 16, 2, theta_deg=20, seed=0)
    st = M.product_state(p.mu, p.nu, 2, 16.0, p.h)
    O.domdec_sweep(st, "A", fixed_iter=5)
    phys = st.alpha["A"] * st.eps_p
    M.set_eps(st, 8.0)
    assert st.eps_p == 8.0
    np.testing.assert_allclose(st.alpha["A"] * st.eps_p, phys, rtol=1e-15)


@pytest.mark.parametrize("stage_cycles", [0, 1])
def test_multiscale_eps_scaling_converges_to_dense_optimum(stage_cycles):
    """R24' eps-scaling inside every layer (eps' 16 -> 8 -> 4, the paper's 4x
    span per layer; intermediate stages until R14 or one cycle
    each) reaches the same dense global entropic optimum at the final eps' = 4
    as the fixed-eps pipeline."""
    p = make_problem("gm", 16, 2, theta_deg=20, seed=0)
    st, hist = M.multiscale_solve(p.mu, p.nu, 2, 4.0, levels=2, E=p.E, err=1e-9, conv=1e-9, max_cycles=200,
                                  eps_scale=4.0, eps_stage_cycles=stage_cycles)
    assert all(r["converged"] for r in hist), hist
    assert st.eps_p == 4.0
    plan, a, b, xs, ys = O.dense_sinkhorn(p.mu, p.nu, 4.0, tol=1e-13)
    from oracle.sinkhorn import sqdist
    N = p.N
    cstar = float(np.sum(sqdist(np.stack([xs // N, xs % N], 1), np.stack([ys // N, ys % N], 1)) * plan)) * p.h ** 2
    assert abs(O.transport_cost(st) - cstar) < 1e-5 * cstar
