"""Pins of the gluing edge candidates (Def. glued-plan
PAPER.md:531-541, Remark eps-gamma PAPER.md:543-559) in the oracle, against
what the definitions fix: gamma_ij has the two prescribed marginals; the
eps -> inf limit is the product candidate; with singleton
cells every candidate is the product one (Remark PAPER.md:438-441); for
uniform cells the eps -> 0 plan is the translation and the edge cost has a
closed form."""
import numpy as np

import oracle as O
from oracle import multiscale as M
from oracle.flow import gamma_conditional, glued_edge_costs
from synth import make_problem


def _state_after_sweeps(p, kinds=("A", "B"), keep=True):
    st = O.init_state(p.mu, p.nu, p.s, p.eps_prime, p.h, p.init_off, p.init_ext, p.init_pos, p.init_data)
    for k in kinds:
        O.domdec_sweep(st, k, err=1e-8, keep_plans=keep)
    return st


def test_gamma_marginals():
    p = make_problem("gm", 16, 2, eps_factor=2.0, theta_deg=20, seed=3)
    st = _state_after_sweeps(p, ("A",))
    for i, j, e in [(5, 6, 0.25), (5, 13, 0.25), (20, 19, 4.0), (0, 8, 0.05)]:
        gt, xi, xj = gamma_conditional(st, i, j, e)
        np.testing.assert_allclose(gt.sum(axis=1), 1.0, rtol=0, atol=1e-12)
        wi = st.mu[xi[:, 0].astype(int), xi[:, 1].astype(int)] / st.m[i]
        wj = st.mu[xj[:, 0].astype(int), xj[:, 1].astype(int)] / st.m[j]
        np.testing.assert_allclose((gt * wi[:, None]).sum(axis=0), wj, rtol=0, atol=1e-11)


def test_glued_large_eps_is_product_candidate():
    """Remark eps-gamma: eps -> inf gives gamma = mu_i/m_i (x) mu_j/m_j and the
    glued candidate mu_j/m_j (x) nu_i/m_i."""
    p = make_problem("gm", 16, 2, eps_factor=2.0, theta_deg=20, seed=1)
    st = _state_after_sweeps(p)
    g = glued_edge_costs(st, 1e9)
    pr = O.edge_costs(st)
    ok = ~np.isnan(pr)
    assert np.array_equal(ok, ~np.isnan(g))
    np.testing.assert_allclose(g[ok], pr[ok], rtol=1e-6, atol=1e-6)


def test_glued_singleton_cells_equal_product():
    """Singleton basic cells (s = 1): gamma_ij is the only coupling of two
    Diracs, so every candidate is delta_{x_j} (x) nu_i/m_i (Remark
    PAPER.md:438-441) and the costs equal the product ones."""
    p = make_problem("gm", 8, 1, eps_factor=2.0, theta_deg=20, seed=4)
    st = _state_after_sweeps(p)
    g = glued_edge_costs(st, 0.25)
    pr = O.edge_costs(st)
    ok = ~np.isnan(pr)
    np.testing.assert_allclose(g[ok], pr[ok], rtol=1e-12, atol=1e-10)


def test_glued_translation_closed_form():
    """Uniform mu on every cell: the eps -> 0 optimal plan between two
    neighbouring cells is the translation x -> x + t (t = s e_k), so
    c_bar_ij = (1/m_i) sum_{x, y} pi_i(x, y) (|x + t - y|^2 - |x - y|^2)
             = |t|^2 ||pi_i|| / m_i - (2/m_i) t . sum_{x,y} pi_i(x, y) (y - x)."""
    N, s = 8, 2
    mu = np.full((N, N), 1.0 / (N * N))
    nu = np.roll(mu, 0)
    st = M.product_state(mu, nu, s, 4.0, 2.0 / N)
    O.domdec_sweep(st, "A", err=1e-10, keep_plans=True)
    g = glued_edge_costs(st, 0.005)
    comp = O.composite_partition(st.n1, st.n2, "A")
    for k, members in enumerate(comp):
        R, Cc, ly, a, b, plan = st.last["plans"][k]
        cell_of = (R // s) * st.n2 + (Cc // s)
        for i in members:
            sel = cell_of == i
            P = plan[sel]
            X = np.stack([R[sel], Cc[sel]], 1).astype(np.float64)
            disp = np.array([float(np.sum(P * (ly[None, :, d] - X[:, d:d + 1]))) for d in (0, 1)])
            for aa, t in ((1, (-s, 0)), (2, (s, 0)), (3, (0, -s)), (4, (0, s))):
                j = O.flow.neighbour(i, aa, st.n1, st.n2)
                if j < 0:
                    continue
                t = np.array(t, np.float64)
                ref = (t @ t) * P.sum() / st.m[i] - 2.0 * (t @ disp) / st.m[i]
                assert abs(g[i, aa] - ref) <= 1e-8 * (1 + abs(ref)), (i, aa, g[i, aa], ref)
