"""O4 — schedules: pure domain decomposition (Alg. 2, PAPER.md:296-305,
A/B alternation) and the hybrid scheme (Alg. 3: A, B,
FlowUpdate, repeat).  Test infrastructure (see oracle/__init__.py)."""
from __future__ import annotations

from .diagnostics import marginal_errors, transport_cost
from .domdec import domdec_sweep
from .flow import flow_update


def run(st, q, n_cycles: int, hybrid: bool = True, err: float = 1e-4, fixed_iter: int = 0,
        max_iter: int = 2000, tau: float = 1e-15, keep_plans: bool = False, callback=None):
    """Run n_cycles of (A, B[, Flow]).  Trajectory time t = #sweeps / n
    (flows take no time).  Returns a list of records."""
    hist = []
    sweeps = 0
    for cyc in range(n_cycles):
        for kind in ("A", "B"):
            stt = domdec_sweep(st, kind, err=err, fixed_iter=fixed_iter, max_iter=max_iter,
                               tau=tau, keep_plans=keep_plans)
            sweeps += 1
            ex, ey = marginal_errors(st)
            rec = {"cycle": cyc, "step": kind, "t": sweeps / st.n1, "e0": stt["e0_sum"],
                   "e": stt["e_sum"], "iters": sum(stt["iters"]), "l1x": ex, "l1y": ey,
                   "cost": transport_cost(st)}
            hist.append(rec)
            if callback:
                callback(rec, st)
        if hybrid:
            fu = flow_update(st, q, tau=tau)
            rec = {"cycle": cyc, "step": "F", "t": sweeps / st.n1, "objective": fu["objective"],
                   "stationary": fu["stationary"], "changed": fu["changed"]}
            hist.append(rec)
            if callback:
                callback(rec, st)
    return hist
