"""Cell sizes s = 1 and s = 8, and the smallest grids of 2 x 2 basic cells (the library builds sweep kernels for s in
{1, 2, 4, 8}; the other parity tests use s = 2 and 4): one sweep from the
generated coupling with exactly K Sinkhorn passes per cell against the fp64
oracle, in the automatic size classes and with every cell in the huge class
on clusters (comp_cap), plus a short hybrid trajectory's transport cost."""
import numpy as np
import pytest

import oracle as O
from parity import compare_states, gpu_ctx, gpu_transport_cost, oracle_state, rel_tols
from synth import make_problem

gpu = pytest.mark.gpu

CASES = {"s1": lambda: make_problem("gm", 24, 1, eps_factor=2.0, theta_deg=20, seed=1),
         "s8": lambda: make_problem("gm", 64, 8, eps_factor=2.0, theta_deg=20, seed=2),
         # the smallest grids: 2 x 2 basic cells (one A cell, B cells of 1 x 1, 1 x 2, 2 x 1)
         "tiny_s2": lambda: make_problem("gm", 4, 2, eps_factor=2.0, theta_deg=20, seed=3),
         "tiny_s4": lambda: make_problem("gm", 8, 4, eps_factor=2.0, theta_deg=20, seed=4)}


@gpu
@pytest.mark.parametrize("case", ["s1", "s8", "tiny_s2", "tiny_s4"])
@pytest.mark.parametrize("part", ["A", "B"])
@pytest.mark.parametrize("comp_cap", [0, 8])
def test_first_sweep_parity_other_cell_sizes(case, part, comp_cap):
    """s = 1: K = 20 at the standard tolerance.  s = 8 (X-blocks of 16 x 16
    pixels): the expanded exponents are ~2x larger than for s = 4, so the
    bound scales with NX / 8, and K = 5: by K = 20 single near-tail entries
    (~1e-6 of their box maximum) of members whose pixels have tiny mu differ
    by up to 5% - the fp32 potentials of such pixels are weakly determined
    (DESIGN.md "Parity tolerances"); the transport cost still agrees
    (test_hybrid_trajectory_other_cell_sizes)."""
    p = CASES[case]()
    K = 5 if case == "s8" else 20
    st = oracle_state(p)
    ost = O.domdec_sweep(st, part, fixed_iter=K)
    dd = gpu_ctx(p, fixed_iter=K, comp_cap=comp_cap)
    gst = dd.sweep(part, stats=True)
    assert gst["cells"] == len(ost["iters"]) and gst["iters_total"] == K * gst["cells"]
    assert gst["overflow"] == 0
    cmp = compare_states(dd.boxes(), st.boxes)
    rb, rt = rel_tols(p.eps_prime)
    nx = 2 * p.s
    rb, rt = rb * max(1, nx // 8), rt * max(1, nx // 8)
    assert cmp["unexplained"] == 0 and cmp["rel_bulk"] < rb and cmp["rel_tail"] < rt, cmp
    assert abs(gst["l1x_final"] - ost["e_sum"]) < 1e-6
    ex, ey = dd.marginal_error()
    oex, _ = O.marginal_errors(st)
    assert abs(ex - oex) < 1e-6 and ey < 1e-12
    dd.close()


@gpu
@pytest.mark.parametrize("case", ["s1", "s8", "tiny_s2", "tiny_s4"])
def test_hybrid_trajectory_other_cell_sizes(case):
    """Four hybrid cycles (fixed K, the GPU's optimal flow injected on both
    sides as in the lockstep protocol of test_gpu_parity): transport cost
    within 1e-5 relative after every sweep."""
    from paper_2405_09400_b200 import mincost_flow
    p = CASES[case]()
    K = 20
    st = oracle_state(p)
    dd = gpu_ctx(p, fixed_iter=K)
    for cyc in range(4):
        for part in "AB":
            O.domdec_sweep(st, part, fixed_iter=K)
            dd.sweep(part)
            oc, gc = O.transport_cost(st), gpu_transport_cost(dd, p.h)
            assert abs(gc - oc) < 1e-5 * oc, (cyc, part, gc, oc)
        _, C, q = dd.edge_costs()
        w, obj, _ = mincost_flow(p.n, p.n, q, C)
        _, oobj = O.min_cost_flow(q, C, p.n, p.n)
        assert obj == min(oobj, 0), (cyc, obj, oobj)
        if obj < 0:
            dd.apply_flow(w)
            O.apply_flow(st, w, q)
    dd.close()
