"""Checkpoint / resume through the C-ABI: export the basic-cell marginals
(domdec_export_cells) and both partitions' potentials (domdec_export_alpha),
build a new context from them (domdec_init + domdec_import_alpha) and
continue: the resumed context reproduces the original's next sweeps (warm
start R7) up to the fp32 rounding of the re-gauged
potentials, and fewer Sinkhorn passes are needed than from alpha = 0."""
import numpy as np
import pytest

from parity import CONFIGS, compare_states, gpu_ctx, gpu_transport_cost, rel_tols

gpu = pytest.mark.gpu


def _resume(dd, p, **kw):
    from paper_2405_09400_b200 import DomDec
    off, ext, pos, data = dd.export_cells()
    r = DomDec(p.mu, p.nu, p.s, p.eps, p.h, np.ascontiguousarray(off, np.int32), np.ascontiguousarray(ext, np.int32),
               np.ascontiguousarray(pos, np.int64), np.ascontiguousarray(data, np.float64), p.E, **kw)
    return r


@gpu
@pytest.mark.parametrize("mode", ["fixed", "tolerance"])
def test_resume_from_exported_state(mode):
    p = CONFIGS["cfg2_gm"]()
    kw = {"fixed_iter": 15} if mode == "fixed" else {}
    a = gpu_ctx(p, **kw)
    for _ in range(3):
        a.sweep("A"); a.sweep("B"); a.flow_update()
    r = _resume(a, p, **kw)
    cold = _resume(a, p, **kw)
    r.import_alpha("A", a.export_alpha("A"))
    r.import_alpha("B", a.export_alpha("B"))
    for part in "AB":
        sa = a.sweep(part, stats=True)
        sr = r.sweep(part, stats=True)
        sc = cold.sweep(part, stats=True)
        if mode == "fixed":   # same passes: entries agree to the fp32 parity bound
            rb, rt = rel_tols(p.eps_prime)
            cmp = compare_states(r.boxes(), a.boxes())
            assert cmp["unexplained"] == 0 and cmp["rel_bulk"] < rb and cmp["rel_tail"] < rt, (part, cmp)
        # (tolerance mode: a cell may stop one pass apart, so entries agree to the
        # Sinkhorn tolerance only; the cost and the pass counts are compared)
        ca, cr = gpu_transport_cost(a, p.h), gpu_transport_cost(r, p.h)
        assert abs(ca - cr) < 1e-6 * ca, (part, ca, cr)
        if mode == "tolerance":
            assert abs(sr["iters_total"] - sa["iters_total"]) <= 0.02 * sa["iters_total"] + sa["cells"], (sa, sr)
            assert sc["iters_total"] > sr["iters_total"], (sc["iters_total"], sr["iters_total"])
    with pytest.raises(Exception):
        bad = np.full((p.N, p.N), np.nan)
        r.import_alpha("A", bad)
    for d in (a, r, cold):
        d.close()
