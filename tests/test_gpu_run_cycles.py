"""domdec_run_cycles: the hybrid iteration (Alg. 3; Alg. 2
for flow_every = 0) launched as CUDA-graph units must give the same state as
the same sequence of domdec_sweep / flow_update calls, and stop by the
sweep-entry criterion of reading R14 like the eager loop does."""
import numpy as np
import pytest

from parity import CONFIGS, gpu_ctx

gpu = pytest.mark.gpu


def _same_state(a, b):
    ba, bb = a.boxes(), b.boxes()
    assert len(ba) == len(bb)
    for (r0, c0, d), (s0, t0, e) in zip(ba, bb):
        assert r0 == s0 and c0 == t0 and np.array_equal(d, e)
    for part in "AB":
        assert np.array_equal(a.export_alpha(part), b.export_alpha(part))


def _eager(dd, cycles, flow_every):
    for k in range(cycles):
        dd.sweep("A")
        dd.sweep("B")
        if flow_every and k % flow_every == flow_every - 1:
            dd.flow_update()


@gpu
@pytest.mark.parametrize("flow_every", [0, 1, 2])
def test_run_cycles_bit_identical_to_eager(flow_every):
    """Fixed cycle count (conv = 0 never met): graph replays (three units
    after the eager warm-up unit, plus a second call that reuses the graph)
    equal the eager sequence bit for bit; the counters advance the same."""
    p = CONFIGS["cfg2_gm"]()
    G = 2 if flow_every == 0 else 2 * flow_every
    n1 = 4 * G
    g = gpu_ctx(p, fixed_iter=20)
    n, e, _ = g.run_cycles(n1, flow_every=flow_every, conv=0.0)
    assert n == n1 and np.isfinite(e) and e > 0
    n, _, _ = g.run_cycles(G, flow_every=flow_every, conv=0.0)   # the captured graph, no warm-up
    assert n == G
    r = gpu_ctx(p, fixed_iter=20)
    _eager(r, n1 + G, flow_every)
    _same_state(g, r)
    cg, cr = g.counters(), r.counters()
    assert cg["sweeps"] == cr["sweeps"] == 2 * (n1 + G)
    assert cg["flow_updates"] == cr["flow_updates"]
    # (the L1 sums use fp64 atomics: equal up to summation order, i.e. to a
    # few ulps of the unit total mass)
    for a, b in zip(g.marginal_error(), r.marginal_error()):
        assert abs(a - b) <= 1e-14
    g.close()
    r.close()


@gpu
def test_run_cycles_convergence_matches_eager_criterion():
    """Tolerance mode to conv = 1e-4: run_cycles stops in the graph unit of
    the first cycle whose both entry errors / ||mu|| are <= conv (R14); the
    eager loop with the same criterion stops at that cycle, and its error is
    the one reported (config 1, which converges in tens of cycles)."""
    p = CONFIGS["cfg1_gm"]()
    conv, fe = 1e-4, 1
    G = 2 * fe
    g = gpu_ctx(p)
    n, e, moved = g.run_cycles(200, flow_every=fe, conv=conv)
    assert e <= conv and 0 <= moved <= n // fe
    r = gpu_ctx(p)
    total = float(p.mu.sum())
    k, er = 0, np.inf
    while k < 200:
        ea = r.sweep("A", stats=True)["l1x_entry"]
        eb = r.sweep("B", stats=True)["l1x_entry"]
        r.flow_update()
        k += 1
        er = max(ea, eb) / total
        if er <= conv:
            break
    assert k <= n < k + G, (k, n)
    assert abs(e - er) <= 1e-12 + 1e-9 * er
    g.close()
    r.close()


@gpu
def test_run_cycles_errors_and_stripe_refusal():
    p = CONFIGS["cfg2_gm"]()
    g = gpu_ctx(p, fixed_iter=5)
    with pytest.raises(Exception):
        g.run_cycles(0)
    with pytest.raises(Exception):
        g.run_cycles(4, flow_every=-1)
    g.close()
