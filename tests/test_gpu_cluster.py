"""The huge size class on thread-block clusters (sweep_cluster.cuh): one
composite cell solved by a cluster of CTAs sharing its Y-rows through
distributed shared memory must give the single-CTA result up to the fp32
summation order, and the oracle's within the usual parity tolerances."""
import os

import numpy as np
import pytest

import oracle as O
from parity import CONFIGS, compare_states, gpu_ctx, oracle_state, rel_tols

gpu = pytest.mark.gpu


def _ctx_with(env, p, **kw):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return gpu_ctx(p, **kw)   # the knobs are read when the context is built
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


VARIANTS = {"single": {"DD_H_CLUSTER": "0"}, "cluster8": {"DD_H_CLUSTER": "8"},
            "cluster2": {"DD_H_CLUSTER": "2"}, "fallback": {"DD_H_CLUSTER": "8", "DD_H_CLUSTER_KB": "1"}}


@gpu
@pytest.mark.parametrize("cfg", ["cfg2_gm", "cfg2_bumps"])
@pytest.mark.parametrize("part", ["A", "B"])
def test_cluster_class_matches_oracle_and_single_cta(cfg, part):
    """comp_cap = 8 sends every cell with a hull side > 8 to the huge class.
    Fixed K passes: every variant (single CTA on global scratch, clusters of 8
    and of 2 CTAs, and the leader-only fallback for cells too large for the
    cluster's shared memory) matches the oracle like the shared-memory
    classes do; the cluster runs are deterministic (two runs bit-identical);
    cluster and single-CTA plans agree to fp32 rounding."""
    p = CONFIGS[cfg]()
    K = 20
    st = oracle_state(p)
    O.domdec_sweep(st, part, fixed_iter=K)
    rb, rt = rel_tols(p.eps_prime)
    res = {}
    for name, env in list(VARIANTS.items()) + [("cluster8b", VARIANTS["cluster8"])]:
        dd = _ctx_with(env, p, fixed_iter=K, comp_cap=8)
        gst = dd.sweep(part, stats=True)
        assert gst["overflow"] == 0 and gst["iters_total"] == K * gst["cells"], (name, gst)
        cmp = compare_states(dd.boxes(), st.boxes)
        assert cmp["unexplained"] == 0 and cmp["rel_bulk"] < rb and cmp["rel_tail"] < rt, (name, cmp)
        res[name] = (dd.boxes(), dd.export_alpha(part), gst)
        dd.close()
    for (r0, c0, d), (s0, t0, e) in zip(res["cluster8"][0], res["cluster8b"][0]):
        assert r0 == s0 and c0 == t0 and np.array_equal(d, e)
    assert np.array_equal(res["cluster8"][1], res["cluster8b"][1])
    a_s, a_c = res["single"][1], res["cluster8"][1]
    ok = np.isfinite(a_s) & (a_s != 0)
    assert np.max(np.abs(a_s[ok] - a_c[ok])) < 2e-3
    assert abs(res["single"][2]["l1x_final"] - res["cluster8"][2]["l1x_final"]) < 1e-6


@gpu
def test_cluster_class_tolerance_mode_hybrid():
    """Tolerance mode (Err = 1e-4), hybrid cycles with every cell in the
    huge class on clusters: the trajectory stays healthy (no overflow, no
    iteration cap, finite errors) and reaches the same transport cost and
    X-error level as the automatic classes after 8 cycles."""
    p = CONFIGS["cfg3_gm_eps2"]()
    out = {}
    for name, kw in (("auto", {}), ("cluster", {"comp_cap": 8})):
        dd = _ctx_with(VARIANTS["cluster8"], p, **kw)
        for _ in range(8):
            for part in "AB":
                s = dd.sweep(part, stats=True)
                assert s["overflow"] == 0 and s["nonconverged"] == 0 and np.isfinite(s["l1x_entry"]), (name, s)
            dd.flow_update()
        out[name] = (dd.marginal_error(), dd.export_plan_cost().sum())
        dd.close()
    (ex_a, _), qa = out["auto"]
    (ex_c, _), qc = out["cluster"]
    assert abs(qa - qc) < 1e-4 * abs(qa)
    assert ex_c < 3e-4 and ex_a < 3e-4


@gpu
@pytest.mark.parametrize("part", ["A", "B"])
def test_stale_potentials_exercise_fallbacks(part):
    """A warm start far from the solution (potentials perturbed by +-60 log2
    units per pixel, imported with domdec_import_alpha): from the second pass
    on, the shifts (the previous outputs) are far from the new values, so
    shifted sums can leave [2^-60, 2^60] and take the max-shift fallback
    (single-CTA and cluster paths alike).  The result after K passes matches
    the oracle started from the same potentials."""
    p = CONFIGS["cfg2_gm"]()
    K = 20
    rng = np.random.default_rng(11)
    base = gpu_ctx(p, fixed_iter=5)
    base.sweep("A"); base.sweep("B")
    alpha = base.export_alpha(part) + rng.uniform(-60.0, 60.0, (p.N, p.N)) * np.log(2.0)
    st = oracle_state(p)
    # the oracle from the same coupling (the generated one) and the same potentials
    st.alpha[part] = alpha.copy()
    O.domdec_sweep(st, part, fixed_iter=K)
    rb, rt = rel_tols(p.eps_prime)
    for name, env in (("single", VARIANTS["single"]), ("cluster8", VARIANTS["cluster8"])):
        dd = _ctx_with(env, p, fixed_iter=K, comp_cap=8)
        dd.import_alpha(part, alpha)
        gst = dd.sweep(part, stats=True)
        assert gst["overflow"] == 0 and np.isfinite(gst["l1x_final"]), (name, gst)
        cmp = compare_states(dd.boxes(), st.boxes)
        assert cmp["unexplained"] == 0 and cmp["rel_bulk"] < rb and cmp["rel_tail"] < rt, (name, cmp)
        dd.close()
    base.close()
