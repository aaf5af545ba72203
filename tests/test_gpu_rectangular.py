"""Rectangular grids (N1 != N2; the C-ABI takes both, the paper's images are
square).  The oracle runs three tolerance-mode cycles from the product
coupling (the first passes from a product coupling are a far-from-equilibrium
transient where fp32 and fp64 drift apart by more than the parity bound on
any grid shape, tests/diag/rect_probe.py); a GPU context is then built from
the oracle's state (domdec_init with its boxes, domdec_import_alpha with its
potentials), so both sides sweep identical inputs: K passes per partition,
boxes within the parity bound, transport costs within 1e-5; then a flow
update with the exact min-cost flow on the n1 x n2 cell graph (objective
equal to the oracle LP's, the GPU's flow applied on both sides) and one more
cycle."""
import numpy as np
import pytest

import oracle as O
from oracle import multiscale as M
from parity import compare_states, gpu_transport_cost, rel_tols

gpu = pytest.mark.gpu


def _dyadic(shape, E, seed):
    """Positive counts summing to exactly 2^E (exact in fp32 / fp64)."""
    rng = np.random.default_rng(seed)
    n = shape[0] * shape[1]
    c = rng.integers(20, 60, n)
    rest = (1 << E) - int(c.sum())
    assert rest > 0
    np.add.at(c, rng.integers(0, n, rest), 1)
    return (c / float(1 << E)).reshape(shape)


def _arrays(boxes):
    off = np.array([[b[0], b[1]] for b in boxes], np.int32)
    ext = np.array([list(b[2].shape) for b in boxes], np.int32)
    sizes = ext[:, 0].astype(np.int64) * ext[:, 1]
    pos = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    data = np.concatenate([b[2].ravel() for b in boxes]).astype(np.float64)
    return off, ext, pos, data


@gpu
@pytest.mark.parametrize("shape", [(24, 40), (40, 24)])
def test_rectangular_grid_parity(shape):
    from paper_2405_09400_b200 import DomDec, mincost_flow
    E, s, eps_p = 18, 2, 4.0
    mu, nu = _dyadic(shape, E, 1), _dyadic(shape, E, 2)
    h = 2.0 / shape[0]
    st = M.product_state(mu, nu, s, eps_p, h)
    for _ in range(3):
        O.domdec_sweep(st, "A", err=1e-4)
        O.domdec_sweep(st, "B", err=1e-4)
    K = 10
    off, ext, pos, data = _arrays(st.boxes)
    dd = DomDec(mu, nu, s, eps_p * h * h, h, off, ext, pos, data, E, fixed_iter=K)
    dd.import_alpha("A", st.alpha["A"])
    dd.import_alpha("B", st.alpha["B"])
    n1, n2 = shape[0] // s, shape[1] // s
    q = np.rint(st.m * 2.0 ** E).astype(np.int64)
    rb, rt = rel_tols(eps_p)
    for cyc in range(2):
        for part in "AB":
            O.domdec_sweep(st, part, fixed_iter=K)
            g = dd.sweep(part, stats=True)
            assert g["overflow"] == 0
            cmp = compare_states(dd.boxes(), st.boxes)
            assert cmp["unexplained"] == 0 and cmp["rel_bulk"] < rb and cmp["rel_tail"] < rt, (cyc, part, cmp)
            oc, gc = O.transport_cost(st), gpu_transport_cost(dd, h)
            assert abs(gc - oc) < 1e-5 * oc, (cyc, part, gc, oc)
        _, C, qg = dd.edge_costs()
        assert np.array_equal(qg, q)
        w, obj, _ = mincost_flow(n1, n2, qg, C)
        _, oobj = O.min_cost_flow(qg, C, n1, n2)
        assert obj == min(oobj, 0), (cyc, obj, oobj)
        if obj < 0:
            dd.apply_flow(w)
            O.apply_flow(st, w, qg)
    ex, ey = dd.marginal_error()
    oex, oey = O.marginal_errors(st)
    assert abs(ex - oex) < 1e-6 and abs(ey - oey) < 1e-6
    dd.close()
