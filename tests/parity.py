"""Helpers shared by the GPU parity tests (comparison logic only)."""
import numpy as np

import oracle as O
from synth import make_problem

TAU = 1e-15
# Tolerances: the GPU solves the cell problems
# in fp32 base-2 log domain; exponent magnitudes inside a box are <= ~250
# (log2 units), so a potential carries <= ~250 * 2^-24 * (few ops) ~ 1e-4
# absolute error in log2 units on the far tails and ~1e-6 in the bulk.
REL_BULK = 4e-5      # entries >= 1e-6 * max of the cell, at eps' >= 4
REL_TAIL = 2e-3      # every entry >= tau, at eps' >= 4


def rel_tols(eps_prime):
    """The log-domain exponents scale like 1/eps' (w = log2(e)/eps'), so the
    fp32 absolute error of a potential, and the relative error of an entry,
    grows like max(1, 4/eps')."""
    f = max(1.0, 4.0 / eps_prime)
    return REL_BULK * f, REL_TAIL * f
GUARD = 1e-2         # box mismatches allowed only for entries within (1 +- GUARD) tau


def oracle_state(p):
    return O.init_state(p.mu, p.nu, p.s, p.eps_prime, p.h, p.init_off, p.init_ext, p.init_pos, p.init_data)


def gpu_ctx(p, **kw):
    from paper_2405_09400_b200 import DomDec
    return DomDec.from_problem(p, **kw)


def compare_cell(g, o, tau=TAU):
    """Compare one basic-cell marginal (r0, c0, arr) GPU vs oracle.
    Returns dict(box_equal, guard_ok, rel_bulk, rel_tail)."""
    gr, gc, ga = g
    orr, oc, oa = o
    box_equal = (gr, gc, ga.shape) == (orr, oc, oa.shape)
    r0, c0 = min(gr, orr), min(gc, oc)
    r1 = max(gr + ga.shape[0], orr + oa.shape[0])
    c1 = max(gc + ga.shape[1], oc + oa.shape[1])
    G = np.zeros((r1 - r0, c1 - c0))
    Ov = np.zeros_like(G)
    G[gr - r0:gr - r0 + ga.shape[0], gc - c0:gc - c0 + ga.shape[1]] = ga
    Ov[orr - r0:orr - r0 + oa.shape[0], oc - c0:oc - c0 + oa.shape[1]] = oa
    only = (G > 0) != (Ov > 0)
    guard_ok = bool(np.all(np.maximum(G, Ov)[only] < tau * (1 + GUARD)))
    both = (G > 0) & (Ov > 0)
    mx = Ov.max()
    rel = np.abs(G - Ov) / np.maximum(Ov, 1e-300)
    bulk = both & (Ov >= 1e-6 * mx)
    return {"box_equal": box_equal, "guard_ok": guard_ok,
            "rel_bulk": float(rel[bulk].max()) if bulk.any() else 0.0,
            "rel_tail": float(rel[both].max()) if both.any() else 0.0}


def compare_states(gboxes, oboxes, cells=None):
    idx = range(len(oboxes)) if cells is None else cells
    res = [compare_cell(gboxes[i], oboxes[i]) for i in idx]
    return {"n": len(res),
            "box_mismatch": sum(not r["box_equal"] for r in res),
            "unexplained": sum((not r["box_equal"]) and (not r["guard_ok"]) for r in res) +
                           sum(not r["guard_ok"] for r in res if r["box_equal"]),
            "rel_bulk": max(r["rel_bulk"] for r in res),
            "rel_tail": max(r["rel_tail"] for r in res)}


def gpu_transport_cost(dd, h):
    return float(np.sum(dd.export_plan_cost())) * h * h


CONFIGS = {
    # BASELINE.json configs[0]: 16x16, GM, eps = (2h)^2, s = 2 (oracle in seconds)
    "cfg1_gm": lambda: make_problem("gm", 16, 2, eps_factor=2.0, theta_deg=20, seed=0),
    "cfg1_gm1": lambda: make_problem("gm", 16, 2, eps_factor=2.0, theta_deg=20, seed=1),
    "cfg1_bumps_small_eps": lambda: make_problem("bumps", 16, 2, eps_factor=0.5),
    # configs[1]: 64x64, s = 2 (four bumps with T0 and a GM)
    "cfg2_bumps": lambda: make_problem("bumps", 64, 2, eps_factor=2.0),
    "cfg2_gm": lambda: make_problem("gm", 64, 2, eps_factor=2.0, theta_deg=20, seed=0),
    # configs[2]: 256x256, s = 4, eps sweep
    "cfg3_gm_eps2": lambda: make_problem("gm", 256, 4, eps_factor=2.0, theta_deg=5, seed=0),
    "cfg3_gm_eps4": lambda: make_problem("gm", 256, 4, eps_factor=4.0, theta_deg=5, seed=1),
    "cfg3_gm_eps8": lambda: make_problem("gm", 256, 4, eps_factor=8.0, theta_deg=5, seed=2),
}
