"""GPU parity of the gluing edge candidates (Def.
glued-plan PAPER.md:531-541, reading R26) against the oracle's direct sums
(oracle.flow.glued_edge_costs, pinned in test_oracle_glued.py)."""
import numpy as np
import pytest

import oracle as O
from oracle.flow import glued_edge_costs
from parity import CONFIGS, gpu_ctx, gpu_transport_cost, oracle_state

gpu = pytest.mark.gpu


@gpu
@pytest.mark.parametrize("cfg,eps_g", [("cfg1_gm", 0.25), ("cfg2_gm", 0.25), ("cfg1_gm1", 1e6)])
def test_glued_edge_costs_parity(cfg, eps_g):
    p = CONFIGS[cfg]()
    K = 25
    st = oracle_state(p)
    dd = gpu_ctx(p, fixed_iter=K)
    dd.set_candidate("glued", eps_g)
    for part in ("A", "B"):
        O.domdec_sweep(st, part, fixed_iter=K, keep_plans=True)
        dd.sweep(part)
    cbar, C, q = dd.edge_costs()
    ocbar = glued_edge_costs(st, eps_g)
    valid = ~np.isnan(ocbar)
    assert np.array_equal(valid, ~np.isnan(cbar))
    scale = 1.0 + np.abs(st.last["Q"])[:, None] * np.ones((1, 5))
    err = np.abs(cbar[valid] - ocbar[valid]) / scale[valid]
    assert err.max() < 5e-5, err.max()
    if eps_g > 1e5:   # eps -> inf: the product candidate
        dd.set_candidate("product")
        pc, _, _ = dd.edge_costs()
        assert np.abs(pc[valid] - cbar[valid]).max() < 1e-6 * (1 + np.abs(pc[valid]).max())
    dd.close()


@gpu
def test_glued_hybrid_lockstep():
    """Alg. 3 with gluing candidates, GPU and oracle in lockstep (parity mode,
    the GPU's optimal flow injected into both, optimal flows being
    non-unique): the GPU's integer instance equals the
    oracle's own up to rounding-boundary arcs, the LP optimum matches, and
    the transport costs agree to 1e-5 after every cycle."""
    from paper_2405_09400_b200 import mincost_flow
    p = CONFIGS["cfg1_gm"]()
    K = 20
    st = oracle_state(p)
    dd = gpu_ctx(p, fixed_iter=K)
    dd.set_candidate("glued", 0.25)
    moved = 0
    for cyc in range(4):
        for part in ("A", "B"):
            O.domdec_sweep(st, part, fixed_iter=K, keep_plans=True)
            dd.sweep(part)
        _, C, q = dd.edge_costs()
        oC, oq = O.integer_instance(glued_edge_costs(st, 0.25), q)
        diff = C != oC
        assert np.all(np.abs(C[diff] - oC[diff]) <= 1), cyc
        assert diff.sum() <= max(2, diff.size // 1000), (cyc, diff.sum())
        w, obj, _ = mincost_flow(p.n, p.n, q, C)
        _, oobj = O.min_cost_flow(q, C, p.n, p.n)
        assert obj == min(oobj, 0), (cyc, obj, oobj)
        if obj < 0:
            moved += 1
            dd.apply_flow(w)
            O.apply_flow(st, w, q)
        oc, gc = O.transport_cost(st), gpu_transport_cost(dd, p.h)
        assert abs(gc - oc) < 1e-5 * oc, (cyc, gc, oc)
    assert moved > 0
    dd.close()
