"""ctypes binding of libdomdec (include/domdec.h) — argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libdomdec.so; this
module only converts numpy arrays to pointers and status codes to
exceptions.  There is no CPU fallback: if the shared library is missing or
no CUDA device is usable, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DOMDEC_LIB") or os.path.join(_HERE, "libdomdec.so")

DD_OK, DD_ERR_ARG, DD_ERR_PRECOND, DD_ERR_NUMERIC, DD_ERR_CUDA, DD_ERR_OOM = 0, 1, 2, 3, 4, 6
PART_A, PART_B = 0, 1


class DomDecError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libdomdec status {status}: {msg}")
        self.status = status


class _Problem(C.Structure):
    _fields_ = [("N1", C.c_int32), ("N2", C.c_int32), ("h", C.c_double), ("eps", C.c_double),
                ("cell_size", C.c_int32), ("mu", C.POINTER(C.c_double)), ("nu", C.POINTER(C.c_double)),
                ("init_off", C.POINTER(C.c_int32)), ("init_ext", C.POINTER(C.c_int32)),
                ("init_pos", C.POINTER(C.c_int64)), ("init_data", C.POINTER(C.c_double)),
                ("mass_exponent", C.c_int32)]


class _Options(C.Structure):
    _fields_ = [("err", C.c_double), ("max_iter", C.c_int32), ("fixed_iter", C.c_int32),
                ("trunc", C.c_double), ("slot_cap", C.c_int32), ("comp_cap", C.c_int32),
                ("device", C.c_int32), ("stream", C.c_void_p), ("track_primal", C.c_int32),
                ("row_begin", C.c_int32), ("row_end", C.c_int32)]


class SweepStats(C.Structure):
    _fields_ = [("cells", C.c_int64), ("nonconverged", C.c_int64), ("iters_total", C.c_int64),
                ("iters_max", C.c_int32), ("overflow", C.c_int32), ("l1x_entry", C.c_double),
                ("l1x_final", C.c_double), ("dropped_mass", C.c_double), ("mufu_ops", C.c_double),
                ("bytes", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class FlowStats(C.Structure):
    _fields_ = [("stationary", C.c_int32), ("certificate", C.c_int32), ("refines", C.c_int32),
                ("rounds", C.c_int32), ("label_rounds", C.c_int32), ("objective", C.c_int64),
                ("changed_cells", C.c_int64), ("solver_ms", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class MsOptions(C.Structure):
    _fields_ = [("levels", C.c_int32), ("max_cycles", C.c_int32), ("flow_every", C.c_int32), ("conv", C.c_double),
                ("eps_scale", C.c_double), ("eps_stage_cycles", C.c_int32)]


class MsStats(C.Structure):
    _fields_ = [("levels", C.c_int32), ("N", C.c_int32 * 16), ("cycles", C.c_int32 * 16), ("flows", C.c_int32 * 16),
                ("converged", C.c_int32 * 16), ("entry_error", C.c_double * 16), ("seconds", C.c_double * 16),
                ("init_seconds", C.c_double * 16), ("flow_seconds", C.c_double * 16), ("total_seconds", C.c_double)]

    def as_dict(self):
        L = self.levels
        return {"levels": L, "N": list(self.N[:L]), "cycles": list(self.cycles[:L]), "flows": list(self.flows[:L]),
                "converged": [bool(x) for x in self.converged[:L]], "entry_error": list(self.entry_error[:L]),
                "seconds": list(self.seconds[:L]), "init_seconds": list(self.init_seconds[:L]),
                "flow_seconds": list(self.flow_seconds[:L]), "total_seconds": self.total_seconds}


class Counters(C.Structure):
    _fields_ = [("sweeps", C.c_int64), ("flow_updates", C.c_int64), ("cells", C.c_int64), ("iters", C.c_int64),
                ("mufu_ops", C.c_double), ("bytes", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load libdomdec.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        path = os.environ.get("DD_LIB_PATH", LIB_PATH)   # development A/B builds
        if not os.path.exists(path):
            raise ImportError(f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(path)
        vp = C.c_void_p
        L.domdec_init.argtypes = [C.POINTER(_Problem), C.POINTER(_Options), C.POINTER(vp)]
        L.domdec_sweep.argtypes = [vp, C.c_int, C.POINTER(SweepStats)]
        L.flow_update.argtypes = [vp, C.POINTER(FlowStats)]
        L.marginal_error.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.primal_dual_gap.argtypes = [vp] + [C.POINTER(C.c_double)] * 4
        L.domdec_export_cells.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                          C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_int64)]
        L.domdec_export_alpha.argtypes = [vp, C.c_int, C.POINTER(C.c_double)]
        L.domdec_export_plan_cost.argtypes = [vp, C.POINTER(C.c_double)]
        if hasattr(L, "domdec_import_alpha"):
            L.domdec_import_alpha.argtypes = [vp, C.c_int, C.POINTER(C.c_double)]
        if hasattr(L, "domdec_export_cell_stats"):   # (absent from older development builds)
            L.domdec_export_cell_stats.argtypes = [vp, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                                   C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        L.flow_edge_costs.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.flow_apply.argtypes = [vp, C.POINTER(C.c_int64)]
        L.dd_mincost_flow.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(FlowStats),
                                      C.c_int32, vp]
        pd = C.POINTER(C.c_double)
        L.dd_sinkhorn_global.argtypes = [C.c_int32, C.c_int32, pd, pd, C.c_double, C.c_double, C.c_int32, C.c_int32,
                                         C.c_int32, vp, pd, pd, C.POINTER(C.c_int32), pd, pd]
        L.domdec_halo_pack.argtypes = [vp, C.c_int32, vp, C.c_int64, C.POINTER(C.c_int64)]
        L.domdec_halo_unpack.argtypes = [vp, C.c_int32, vp, C.c_int64]
        L.domdec_destroy.argtypes = [vp]
        if hasattr(L, "flow_solve"):   # (absent from older development builds)
            L.flow_edge_costs_device.argtypes = [vp, vp, vp]
            L.flow_solve.argtypes = [vp, vp, vp, C.POINTER(FlowStats)]
            L.flow_apply_device.argtypes = [vp, vp]
            L.domdec_halo_capacity.argtypes = [vp, C.POINTER(C.c_int64)]
            L.flow_set_candidate.argtypes = [vp, C.c_int32, C.c_double]
        if hasattr(L, "dd_multiscale_solve"):
            L.domdec_init_product.argtypes = [C.POINTER(_Problem), C.POINTER(_Options), C.POINTER(vp)]
            L.domdec_refine.argtypes = [vp, C.POINTER(_Problem), C.POINTER(_Options), C.POINTER(vp)]
            L.dd_multiscale_solve.argtypes = [C.POINTER(_Problem), C.POINTER(_Options), C.POINTER(MsOptions),
                                              C.POINTER(vp), C.POINTER(MsStats)]
        if hasattr(L, "domdec_set_eps"):
            L.domdec_set_eps.argtypes = [vp, C.c_double]
        if hasattr(L, "domdec_run_cycles"):
            L.domdec_run_cycles.argtypes = [vp, C.c_int32, C.c_int32, C.c_double, C.POINTER(C.c_int32),
                                            C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        L.domdec_counters.argtypes = [vp, C.POINTER(Counters)]
        L.domdec_reset_counters.argtypes = [vp]
        L.dd_mufu_peak.argtypes = [C.c_int32, C.POINTER(C.c_double)]
        L.dd_last_error.argtypes = [vp]
        L.dd_last_error.restype = C.c_char_p
        L.dd_version.restype = C.c_char_p
        for fn in ("domdec_init", "domdec_sweep", "flow_update", "marginal_error", "primal_dual_gap",
                   "domdec_export_cells", "domdec_export_alpha", "domdec_export_plan_cost",
                   "domdec_export_cell_stats", "flow_edge_costs", "flow_apply", "dd_mincost_flow", "domdec_destroy", "domdec_counters",
                   "domdec_reset_counters", "dd_mufu_peak", "domdec_halo_pack", "domdec_halo_unpack",
                   "dd_sinkhorn_global", "domdec_init_product", "domdec_refine", "dd_multiscale_solve",
                   "domdec_export_cell_stats", "flow_edge_costs_device", "flow_solve", "flow_apply_device",
                   "domdec_halo_capacity", "flow_set_candidate", "domdec_run_cycles", "domdec_set_eps",
                   "domdec_import_alpha"):
            if hasattr(L, fn):
                getattr(L, fn).restype = C.c_int
        _lib = L
    return _lib


EXPORTED = ("domdec_init", "domdec_sweep", "flow_update", "marginal_error", "primal_dual_gap",
            "domdec_export_cells", "domdec_export_alpha", "domdec_export_plan_cost",
            "domdec_export_cell_stats", "flow_edge_costs", "flow_apply", "dd_mincost_flow", "domdec_destroy",
            "dd_last_error", "dd_version", "domdec_counters", "domdec_reset_counters", "dd_mufu_peak",
            "domdec_halo_pack", "domdec_halo_unpack", "dd_sinkhorn_global", "domdec_init_product",
            "domdec_refine", "dd_multiscale_solve", "flow_edge_costs_device", "flow_solve",
            "flow_apply_device", "domdec_halo_capacity", "flow_set_candidate", "domdec_run_cycles",
            "domdec_set_eps", "domdec_import_alpha")


def _problem(mu, nu, s, eps, h, E, off=None, ext=None, pos=None, data=None):
    N1, N2 = mu.shape
    return _Problem(N1, N2, float(h), float(eps), int(s), _ptr(mu, C.c_double), _ptr(nu, C.c_double),
                    _ptr(off, C.c_int32) if off is not None else None, _ptr(ext, C.c_int32) if ext is not None else None,
                    _ptr(pos, C.c_int64) if pos is not None else None,
                    _ptr(data, C.c_double) if data is not None else None, int(E))


def _options(err=1e-4, max_iter=2000, fixed_iter=0, trunc=1e-15, slot_cap=0, comp_cap=0, device=0, stream=None,
             track_primal=False, row_begin=0, row_end=0):
    return _Options(float(err), int(max_iter), int(fixed_iter), float(trunc), int(slot_cap), int(comp_cap),
                    int(device), C.c_void_p(stream) if stream else None, int(bool(track_primal)),
                    int(row_begin), int(row_end))


def multiscale_solve(mu, nu, cell_size, eps, E, levels, conv=1e-4, max_cycles=1000, flow_every=1, eps_scale=1.0,
                     eps_stage_cycles=0, **opts):
    """dd_multiscale_solve (readings R23-R25): coarse-to-fine
    hybrid domain decomposition of the N1 x N2 problem on [-1, 1]^2 (h = 2/N1,
    eps in physical units, eps' = eps/h^2 kept on every layer).  Returns
    (DomDec of the finest layer, stats dict)."""
    mu_ = np.ascontiguousarray(mu, np.float64)
    nu_ = np.ascontiguousarray(nu, np.float64)
    P = _problem(mu_, nu_, cell_size, eps, 2.0 / mu_.shape[0], E)
    O = _options(**opts)
    M = MsOptions(int(levels), int(max_cycles), int(flow_every), float(conv), float(eps_scale),
                  int(eps_stage_cycles))
    st = MsStats()
    ctx = C.c_void_p()
    _check(lib().dd_multiscale_solve(C.byref(P), C.byref(O), C.byref(M), C.byref(ctx), C.byref(st)), None)
    return DomDec._wrap(ctx, mu_, nu_, cell_size), st.as_dict()


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def _check(status, ctx):
    if status != DD_OK:
        msg = lib().dd_last_error(ctx)
        raise DomDecError(status, msg.decode() if msg else "")


class DomDec:
    """One solver context (device state = basic-cell marginals + potentials).

    Construction copies mu, nu and the initial basic-cell boxes to the GPU
    (domdec_init); all further calls operate on device-resident state."""

    def __init__(self, mu, nu, cell_size, eps, h, init_off, init_ext, init_pos, init_data, mass_exponent,
                 _how="init", _coarse=None, **opts):
        self._keep = [np.ascontiguousarray(mu, np.float64), np.ascontiguousarray(nu, np.float64)]
        if _how == "init":
            self._keep += [np.ascontiguousarray(init_off, np.int32), np.ascontiguousarray(init_ext, np.int32),
                           np.ascontiguousarray(init_pos, np.int64), np.ascontiguousarray(init_data, np.float64)]
        mu_, nu_ = self._keep[:2]
        self.N1, self.N2 = mu_.shape
        self.s = int(cell_size)
        self.n1, self.n2 = self.N1 // self.s, self.N2 // self.s
        self.I = self.n1 * self.n2
        P = _problem(mu_, nu_, self.s, eps, h, mass_exponent, *(self._keep[2:] if _how == "init" else ()))
        O = _options(**opts)
        ctx = C.c_void_p()
        if _how == "init":
            _check(lib().domdec_init(C.byref(P), C.byref(O), C.byref(ctx)), None)
        elif _how == "product":
            _check(lib().domdec_init_product(C.byref(P), C.byref(O), C.byref(ctx)), None)
        else:
            _check(lib().domdec_refine(_coarse._ctx, C.byref(P), C.byref(O), C.byref(ctx)), None)
        self._ctx = ctx

    @classmethod
    def product(cls, mu, nu, cell_size, eps, h, mass_exponent, **opts):
        """Context started from the product coupling mu (x) nu (domdec_init_product)."""
        return cls(mu, nu, cell_size, eps, h, None, None, None, None, mass_exponent, _how="product", **opts)

    def refine(self, mu_f, nu_f, eps_f, mass_exponent, **opts):
        """Context of the next finer layer initialised with the refinement of
        this context's marginals (domdec_refine, readings R23-R25)."""
        N1 = np.asarray(mu_f).shape[0]
        return DomDec(mu_f, nu_f, self.s, eps_f, 2.0 / N1, None, None, None, None, mass_exponent, _how="refine",
                      _coarse=self, **opts)

    @classmethod
    def _wrap(cls, ctx, mu, nu, s):
        self = cls.__new__(cls)
        self._keep = [mu, nu]
        self.N1, self.N2 = mu.shape
        self.s = int(s)
        self.n1, self.n2 = self.N1 // self.s, self.N2 // self.s
        self.I = self.n1 * self.n2
        self._ctx = ctx
        return self

    @classmethod
    def from_problem(cls, p, **kw):
        """Build from a synth.Problem-like object (attributes mu, nu, s, eps, h,
        init_off, init_ext, init_pos, init_data, E)."""
        return cls(p.mu, p.nu, p.s, p.eps, p.h, p.init_off, p.init_ext, p.init_pos, p.init_data, p.E, **kw)

    def sweep(self, part, stats=False):
        st = SweepStats() if stats else None
        _check(lib().domdec_sweep(self._ctx, PART_A if part in ("A", 0) else PART_B,
                                  C.byref(st) if st is not None else None), self._ctx)
        return st.as_dict() if st is not None else None

    def flow_update(self, stats=False):
        st = FlowStats() if stats else None
        _check(lib().flow_update(self._ctx, C.byref(st) if st is not None else None), self._ctx)
        return st.as_dict() if st is not None else None

    def set_eps(self, eps):
        """domdec_set_eps: new eps (physical, <= the construction eps), physical potentials kept."""
        _check(lib().domdec_set_eps(self._ctx, float(eps)), self._ctx)

    def run_cycles(self, max_cycles, flow_every=1, conv=1e-4):
        """Hybrid cycles to convergence on the device (CUDA-graph units):
        returns (cycles executed, entry error, non-stationary flow updates)."""
        n, e, mv = C.c_int32(), C.c_double(), C.c_int32()
        _check(lib().domdec_run_cycles(self._ctx, int(max_cycles), int(flow_every), float(conv), C.byref(n),
                                       C.byref(e), C.byref(mv)), self._ctx)
        return n.value, e.value, mv.value

    def marginal_error(self):
        x, y = C.c_double(), C.c_double()
        _check(lib().marginal_error(self._ctx, C.byref(x), C.byref(y)), self._ctx)
        return x.value, y.value

    def primal_dual_gap(self):
        v = [C.c_double() for _ in range(4)]
        _check(lib().primal_dual_gap(self._ctx, *[C.byref(a) for a in v]), self._ctx)
        return tuple(a.value for a in v)

    def halo_size(self, row):
        """Bytes of the serialised marginals of basic-cell row `row`."""
        n = C.c_int64()
        _check(lib().domdec_halo_pack(self._ctx, int(row), None, 0, C.byref(n)), self._ctx)
        return n.value

    def halo_pack(self, row, dev_ptr, cap):
        """Serialise row `row` into the device buffer at dev_ptr (cap bytes)."""
        n = C.c_int64()
        _check(lib().domdec_halo_pack(self._ctx, int(row), C.c_void_p(dev_ptr), int(cap), C.byref(n)), self._ctx)
        return n.value

    def set_candidate(self, kind="product", eps_gamma_p=0.25):
        """flow_set_candidate: "product" (R12) or "glued" (gluing candidates with
        entropic gamma_ij)."""
        _check(lib().flow_set_candidate(self._ctx, 0 if kind == "product" else 1, float(eps_gamma_p)), self._ctx)

    def halo_capacity(self):
        """Bytes of a halo buffer that holds any row (domdec_halo_capacity)."""
        n = C.c_int64()
        _check(lib().domdec_halo_capacity(self._ctx, C.byref(n)), self._ctx)
        return n.value

    def edge_costs_device(self, cbar_ptr, C_ptr):
        """flow_edge_costs_device: cbar / C into device buffers (asynchronous)."""
        _check(lib().flow_edge_costs_device(self._ctx, C.c_void_p(cbar_ptr) if cbar_ptr else None,
                                            C.c_void_p(C_ptr) if C_ptr else None), self._ctx)

    def flow_solve(self, C_ptr, w_ptr=None, stats=False):
        """flow_solve: warm-started exact min-cost flow of a device instance."""
        st = FlowStats() if stats else None
        _check(lib().flow_solve(self._ctx, C.c_void_p(C_ptr), C.c_void_p(w_ptr) if w_ptr else None,
                                C.byref(st) if st is not None else None), self._ctx)
        return st.as_dict() if st is not None else None

    def apply_flow_device(self, w_ptr):
        _check(lib().flow_apply_device(self._ctx, C.c_void_p(w_ptr)), self._ctx)

    def halo_unpack(self, row, dev_ptr, nbytes):
        """Replace row `row` by a buffer written by halo_pack (device pointer)."""
        _check(lib().domdec_halo_unpack(self._ctx, int(row), C.c_void_p(dev_ptr), int(nbytes)), self._ctx)

    def export_cells(self):
        I = self.I
        off = np.zeros((I, 2), np.int32)
        ext = np.zeros((I, 2), np.int32)
        pos = np.zeros(I, np.int64)
        n = C.c_int64()
        _check(lib().domdec_export_cells(self._ctx, _ptr(off, C.c_int32), _ptr(ext, C.c_int32),
                                         _ptr(pos, C.c_int64), None, 0, C.byref(n)), self._ctx)
        data = np.zeros(max(1, n.value), np.float64)
        _check(lib().domdec_export_cells(self._ctx, _ptr(off, C.c_int32), _ptr(ext, C.c_int32),
                                         _ptr(pos, C.c_int64), _ptr(data, C.c_double), data.size, C.byref(n)),
               self._ctx)
        return off, ext, pos, data[:n.value]

    def boxes(self):
        """Basic-cell marginals as a list of (r0, c0, 2-D array)."""
        off, ext, pos, data = self.export_cells()
        return [(int(off[i, 0]), int(off[i, 1]),
                 data[pos[i]:pos[i] + ext[i, 0] * ext[i, 1]].reshape(ext[i, 0], ext[i, 1]))
                for i in range(self.I)]

    def export_alpha(self, part):
        a = np.zeros((self.N1, self.N2), np.float64)
        _check(lib().domdec_export_alpha(self._ctx, PART_A if part in ("A", 0) else PART_B, _ptr(a, C.c_double)),
               self._ctx)
        return a

    def import_alpha(self, part, alpha):
        """domdec_import_alpha: warm-start potential in the export_alpha format (resume)."""
        a = np.ascontiguousarray(alpha, np.float64)
        assert a.shape == (self.N1, self.N2)
        _check(lib().domdec_import_alpha(self._ctx, PART_A if part in ("A", 0) else PART_B, _ptr(a, C.c_double)),
               self._ctx)

    def cell_stats(self, part):
        """Per composite cell (iters, e0, e) of the last sweep on a partition."""
        pp = PART_A if part in ("A", 0) else PART_B
        n = C.c_int32()
        _check(lib().domdec_export_cell_stats(self._ctx, pp, None, None, None, C.byref(n)), self._ctx)
        it = np.zeros(n.value, np.int32)
        e0 = np.zeros(n.value, np.float64)
        e = np.zeros(n.value, np.float64)
        _check(lib().domdec_export_cell_stats(self._ctx, pp, _ptr(it, C.c_int32), _ptr(e0, C.c_double),
                                              _ptr(e, C.c_double), C.byref(n)), self._ctx)
        return it, e0, e

    def export_plan_cost(self):
        q = np.zeros(self.I, np.float64)
        _check(lib().domdec_export_plan_cost(self._ctx, _ptr(q, C.c_double)), self._ctx)
        return q

    def edge_costs(self):
        cbar = np.zeros((self.I, 5), np.float64)
        Cc = np.zeros((self.I, 5), np.int64)
        q = np.zeros(self.I, np.int64)
        _check(lib().flow_edge_costs(self._ctx, _ptr(cbar, C.c_double), _ptr(Cc, C.c_int64), _ptr(q, C.c_int64)),
               self._ctx)
        return cbar, Cc, q

    def apply_flow(self, w):
        w = np.ascontiguousarray(w, np.int64)
        assert w.shape == (self.I, 5)
        _check(lib().flow_apply(self._ctx, _ptr(w, C.c_int64)), self._ctx)

    def counters(self):
        cnt = Counters()
        _check(lib().domdec_counters(self._ctx, C.byref(cnt)), self._ctx)
        return cnt.as_dict()

    def reset_counters(self):
        _check(lib().domdec_reset_counters(self._ctx), self._ctx)

    def close(self):
        if getattr(self, "_ctx", None):
            lib().domdec_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mufu_peak(device=0):
    """Measured ex2 throughput of the device (ops/s)."""
    v = C.c_double()
    _check(lib().dd_mufu_peak(int(device), C.byref(v)), None)
    return v.value


def mincost_flow(n1, n2, q, Cc, device=0, stream=None):
    """Standalone GPU exact min-cost flow (dd_mincost_flow).  Returns
    (w [I,5] int64, objective, stats dict)."""
    q = np.ascontiguousarray(q, np.int64)
    Cc = np.ascontiguousarray(Cc, np.int64)
    w = np.zeros((n1 * n2, 5), np.int64)
    obj = C.c_int64()
    st = FlowStats()
    _check(lib().dd_mincost_flow(int(n1), int(n2), _ptr(q, C.c_int64), _ptr(Cc, C.c_int64), _ptr(w, C.c_int64),
                                 C.byref(obj), C.byref(st), int(device), C.c_void_p(stream) if stream else None),
           None)
    return w, obj.value, st.as_dict()


def sinkhorn_global(mu, nu, eps_p, err=1e-4, max_iter=100000, check_every=1, alpha0=None, device=0, stream=None):
    """Global separable log-domain Sinkhorn on the GPU (dd_sinkhorn_global,
    the SinkhornGPU comparator).  mu, nu: (N1, N2) float64.  Returns
    (a, b, iters, l1_x, solve_ms) with a, b (N1, N2) float64 in units of eps."""
    mu = np.ascontiguousarray(mu, np.float64)
    nu = np.ascontiguousarray(nu, np.float64)
    N1, N2 = mu.shape
    a = np.zeros((N1, N2)) if alpha0 is None else np.array(alpha0, np.float64, order="C", copy=True)
    b = np.zeros((N1, N2))
    it, e, ms = C.c_int32(), C.c_double(), C.c_double()
    pd = C.c_double
    _check(lib().dd_sinkhorn_global(int(N1), int(N2), _ptr(mu, pd), _ptr(nu, pd), float(eps_p), float(err),
                                    int(max_iter), int(check_every), int(device),
                                    C.c_void_p(stream) if stream else None, _ptr(a, pd), _ptr(b, pd),
                                    C.byref(it), C.byref(e), C.byref(ms)), None)
    return a, b, it.value, e.value, ms.value
