"""Thin ctypes binding of include/ckkt.h (argument marshalling only).

Every numerical step runs inside libckkt.so (CUDA kernels for sm_100a); this
module converts numpy / torch arguments to pointers and back.  It never falls
back to a CPU implementation: if the library or a CUDA device is missing the
calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CKKT_LIB_OVERRIDE") or os.path.join(_HERE, "libckkt.so")  # override: experiments only

CKKT_OK, CKKT_NOT_PD, CKKT_CG_NO_CONVERGENCE, CKKT_REFINE_NOT_CONVERGED = 0, 1, 2, 3
CKKT_PATTERN_ERROR, CKKT_INVALID_ARG, CKKT_CUDA_ERROR, CKKT_OUT_OF_MEMORY = 4, 5, 6, 7
CKKT_LIFTED, CKKT_HYKKT = 0, 1

EXPORTED = ["ckkt_default_options", "ckkt_setup", "ckkt_get_sizes", "ckkt_export_symbolic",
            "ckkt_export_elimination_order", "ckkt_export_analysis", "ckkt_setup_from_analysis", "ckkt_refactor",
            "ckkt_refactor_inertia", "ckkt_fraction_to_boundary",
            "ckkt_solve", "ckkt_iterate_host", "ckkt_profile", "ckkt_phase_times", "ckkt_launch_count",
            "ckkt_destroy", "ckkt_status_str", "ckkt_distillation_eval"]
PHASES = ("condense", "factor", "forward", "backward", "vector")


class ckkt_pattern(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m_e", ctypes.c_int32), ("m_i", ctypes.c_int32),
                ("w_nnz", ctypes.c_int64), ("w_row", ctypes.c_void_p), ("w_col", ctypes.c_void_p),
                ("g_rowptr", ctypes.c_void_p), ("g_col", ctypes.c_void_p),
                ("h_rowptr", ctypes.c_void_p), ("h_col", ctypes.c_void_p)]


class ckkt_options(ctypes.Structure):
    _fields_ = [("strategy", ctypes.c_int32), ("gamma", ctypes.c_double), ("cg_rtol", ctypes.c_double),
                ("cg_maxit", ctypes.c_int32), ("ref_tol", ctypes.c_double), ("ref_maxit", ctypes.c_int32),
                ("batch", ctypes.c_int32), ("leaf", ctypes.c_int32), ("perm", ctypes.c_void_p),
                ("device", ctypes.c_int32), ("stream", ctypes.c_void_p), ("cg_rtol_corr", ctypes.c_double)]


class ckkt_info(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("k_cg", ctypes.c_int32), ("k_cg_total", ctypes.c_int32),
                ("n_ref", ctypes.c_int32), ("rel_res", ctypes.c_double), ("rel_res_unrefined", ctypes.c_double),
                ("res_inf", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ckkt_distillation_params(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("D", ctypes.c_double), ("F", ctypes.c_double),
                ("w_x", ctypes.c_double), ("rho", ctypes.c_double), ("horizon", ctypes.c_double),
                ("x_f", ctypes.c_double), ("xbar1", ctypes.c_double), ("ubar", ctypes.c_double),
                ("feed_tray", ctypes.c_int32), ("M", ctypes.c_double * 32)]


class ckkt_sizes(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m_e", ctypes.c_int32), ("m_i", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("nnz_k", ctypes.c_int64), ("nnz_l", ctypes.c_int64), ("l_storage", ctypes.c_int64),
                ("n_supernodes", ctypes.c_int32), ("n_levels", ctypes.c_int32), ("flops_factor", ctypes.c_double),
                ("device_bytes", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load libckkt.so (built in-tree by __graft_entry__.build()); raises if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        L.ckkt_default_options.argtypes = [ctypes.POINTER(ckkt_options)]
        L.ckkt_default_options.restype = None
        L.ckkt_setup.argtypes = [ctypes.POINTER(ckkt_pattern), ctypes.POINTER(ckkt_options), ctypes.POINTER(P)]
        L.ckkt_setup.restype = ctypes.c_int
        L.ckkt_get_sizes.argtypes = [P, ctypes.POINTER(ckkt_sizes)]
        L.ckkt_get_sizes.restype = ctypes.c_int
        L.ckkt_export_symbolic.argtypes = [P, P, P, P, P, P]
        L.ckkt_export_symbolic.restype = ctypes.c_int
        L.ckkt_export_elimination_order.argtypes = [P, P]
        L.ckkt_export_elimination_order.restype = ctypes.c_int
        L.ckkt_export_analysis.argtypes = [P, P, ctypes.POINTER(ctypes.c_int64)]
        L.ckkt_export_analysis.restype = ctypes.c_int
        L.ckkt_setup_from_analysis.argtypes = [ctypes.POINTER(ckkt_pattern), ctypes.POINTER(ckkt_options), P,
                                               ctypes.c_int64, ctypes.POINTER(P)]
        L.ckkt_setup_from_analysis.restype = ctypes.c_int
        L.ckkt_refactor.argtypes = [P, P, P, P, P, P, P, P, P]
        L.ckkt_refactor.restype = ctypes.c_int
        L.ckkt_refactor_inertia.argtypes = [P] * 11
        L.ckkt_refactor_inertia.restype = ctypes.c_int
        L.ckkt_fraction_to_boundary.argtypes = [ctypes.c_int32, ctypes.c_int64, P, P, ctypes.c_double, P, P]
        L.ckkt_fraction_to_boundary.restype = ctypes.c_int
        L.ckkt_solve.argtypes = [P, P, P, P, P, P, P, P, P, ctypes.POINTER(ckkt_info)]
        L.ckkt_solve.restype = ctypes.c_int
        L.ckkt_iterate_host.argtypes = [P] * 16 + [ctypes.POINTER(ckkt_info)]
        L.ckkt_iterate_host.restype = ctypes.c_int
        L.ckkt_profile.argtypes = [P, ctypes.c_int32]
        L.ckkt_profile.restype = ctypes.c_int
        L.ckkt_phase_times.argtypes = [P, P, P]
        L.ckkt_phase_times.restype = ctypes.c_int
        L.ckkt_launch_count.argtypes = [P]
        L.ckkt_launch_count.restype = ctypes.c_int64
        L.ckkt_destroy.argtypes = [P]
        L.ckkt_destroy.restype = None
        L.ckkt_distillation_eval.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ckkt_distillation_params),
                                             P, P, P, P, ctypes.c_double, P, P, P, P, P]
        L.ckkt_distillation_eval.restype = ctypes.c_int
        L.ckkt_status_str.argtypes = [ctypes.c_int]
        L.ckkt_status_str.restype = ctypes.c_char_p
        _lib = L
    return _lib


def fraction_to_boundary(s, ds, tau: float):
    """ckkt_fraction_to_boundary on [B, len] (or [len]) device FP64 tensors; returns alpha [B] on the device,
    enqueued on torch's current stream."""
    import torch
    if s.shape != ds.shape or s.dtype != torch.float64 or ds.dtype != torch.float64:
        raise ValueError("s and ds: same shape, float64")
    if s.dim() not in (1, 2):
        raise ValueError("s and ds: [len] or [B, len]")
    s2, d2 = (s, ds) if s.dim() == 2 else (s.unsqueeze(0), ds.unsqueeze(0))
    alpha = torch.empty(s2.shape[0], dtype=torch.float64, device=s.device)
    rc = lib().ckkt_fraction_to_boundary(s2.shape[0], s2.shape[1], _dptr(s2), _dptr(d2), float(tau), _dptr(alpha),
                                         ctypes.c_void_p(torch.cuda.current_stream(s.device).cuda_stream))
    if rc:
        raise CKKTError(rc, "ckkt_fraction_to_boundary")
    return alpha


def distillation_params(p) -> ckkt_distillation_params:
    """ckkt_distillation_params from an inputs.distillation.Params-like object (attribute names match)."""
    out = ckkt_distillation_params()
    for name in ("alpha", "D", "F", "w_x", "rho", "horizon", "x_f", "xbar1", "ubar", "feed_tray"):
        setattr(out, name, getattr(p, name))
    for k, mk in enumerate(p.holdups()):
        out.M[k] = float(mk)
    return out


def distillation_eval(N, params, xbar0, v, lam=None, row_scale=None, obj_scale=1.0, j_val=None, w_val=None, c=None,
                      grad_f=None, batch=1):
    """ckkt_distillation_eval on device tensors (outputs preallocated by the caller; any may be None), enqueued
    on torch's current stream."""
    import torch
    prm = distillation_params(params)
    rc = lib().ckkt_distillation_eval(int(N), int(batch), ctypes.byref(prm), _dptr(xbar0), _dptr(v), _dptr(lam),
                                      _dptr(row_scale), float(obj_scale), _dptr(j_val), _dptr(w_val), _dptr(c),
                                      _dptr(grad_f), ctypes.c_void_p(torch.cuda.current_stream(v.device).cuda_stream))
    if rc:
        raise CKKTError(rc, "ckkt_distillation_eval")


class CKKTError(RuntimeError):
    def __init__(self, code, where):
        super().__init__(f"{where}: {lib().ckkt_status_str(code).decode()} ({code})")
        self.code = code


def _np_ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _dptr(t):
    """Device pointer of a contiguous torch CUDA tensor (or None)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device pointer expected (torch CUDA tensor)")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _hptr(a):
    """Host pointer of a numpy array or a CPU torch tensor (pinned or not)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous
        return a.ctypes.data_as(ctypes.c_void_p)
    if a.is_cuda:
        raise ValueError("host pointer expected")
    return ctypes.c_void_p(a.data_ptr())


def default_options(**kw) -> ckkt_options:
    o = ckkt_options()
    lib().ckkt_default_options(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class Context:
    """Owns one ckkt_ctx.  Method names follow the C ABI (ckkt_<name>)."""

    def __init__(self, n, m_e, m_i, w_row, w_col, g_rowptr=None, g_col=None, h_rowptr=None, h_col=None,
                 perm=None, stream=None, analysis=None, **options):
        """analysis: optional bytes from export_analysis() of the same pattern and settings
        (ckkt_setup_from_analysis: no symbolic analysis at setup)."""
        L = lib()
        self._keep = []

        def arr(a):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=np.int32)
            self._keep.append(a)
            return a

        w_row, w_col = arr(w_row), arr(w_col)
        g_rowptr, g_col, h_rowptr, h_col = arr(g_rowptr), arr(g_col), arr(h_rowptr), arr(h_col)
        pat = ckkt_pattern(n=n, m_e=m_e, m_i=m_i, w_nnz=len(w_row), w_row=_np_ptr(w_row), w_col=_np_ptr(w_col),
                           g_rowptr=_np_ptr(g_rowptr), g_col=_np_ptr(g_col), h_rowptr=_np_ptr(h_rowptr),
                           h_col=_np_ptr(h_col))
        opt = default_options(**options)
        if perm is not None:
            perm = arr(perm)
            opt.perm = _np_ptr(perm)
        if stream is not None:
            opt.stream = ctypes.c_void_p(stream)
        self.opt = opt
        self.n, self.m_e, self.m_i, self.batch = n, m_e, m_i, opt.batch
        h = ctypes.c_void_p()
        if analysis is None:
            rc = L.ckkt_setup(ctypes.byref(pat), ctypes.byref(opt), ctypes.byref(h))
        else:
            buf = np.frombuffer(analysis, dtype=np.uint8)  # zero-copy view (bytes or a uint8 array)
            rc = L.ckkt_setup_from_analysis(ctypes.byref(pat), ctypes.byref(opt), buf.ctypes.data_as(ctypes.c_void_p),
                                            buf.size, ctypes.byref(h))
        if rc != CKKT_OK:
            raise CKKTError(rc, "ckkt_setup" if analysis is None else "ckkt_setup_from_analysis")
        self.h = h
        self._keep = []

    def close(self):
        if getattr(self, "h", None):
            lib().ckkt_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- host-side queries
    def get_sizes(self) -> dict:
        s = ckkt_sizes()
        rc = lib().ckkt_get_sizes(self.h, ctypes.byref(s))
        if rc:
            raise CKKTError(rc, "ckkt_get_sizes")
        return s.as_dict()

    def export_symbolic(self, pattern: bool = True):
        sz = self.get_sizes()
        n = sz["n"]
        perm = np.empty(n, np.int32)
        parent = np.empty(n, np.int32)
        cc = np.empty(n, np.int32)
        Lp = np.empty(n + 1, np.int64) if pattern else None
        Li = np.empty(sz["nnz_l"], np.int32) if pattern else None
        rc = lib().ckkt_export_symbolic(self.h, _np_ptr(perm), _np_ptr(parent), _np_ptr(cc), _np_ptr(Lp), _np_ptr(Li))
        if rc:
            raise CKKTError(rc, "ckkt_export_symbolic")
        return perm, parent, cc, Lp, Li

    def export_analysis(self) -> np.ndarray:
        """ckkt_export_analysis: the serialized symbolic analysis as a uint8 array (reusable with
        Context(..., analysis=...); .tofile() / np.fromfile() store it)."""
        size = ctypes.c_int64(0)
        rc = lib().ckkt_export_analysis(self.h, None, ctypes.byref(size))
        if rc:
            raise CKKTError(rc, "ckkt_export_analysis")
        buf = np.empty(size.value, dtype=np.uint8)
        rc = lib().ckkt_export_analysis(self.h, buf.ctypes.data_as(ctypes.c_void_p), ctypes.byref(size))
        if rc:
            raise CKKTError(rc, "ckkt_export_analysis")
        return buf

    def export_elimination_order(self):
        """ckkt_export_elimination_order: order[k] = original index eliminated k-th (min_bad_pivot's order)."""
        order = np.empty(self.n, np.int32)
        rc = lib().ckkt_export_elimination_order(self.h, _np_ptr(order))
        if rc:
            raise CKKTError(rc, "ckkt_export_elimination_order")
        return order

    def profile(self, enable: bool = True):
        rc = lib().ckkt_profile(self.h, int(enable))
        if rc:
            raise CKKTError(rc, "ckkt_profile")

    def phase_times(self) -> dict:
        """{phase: (ms, launches)} accumulated since the previous call (synchronises the stream)."""
        ms = np.zeros(len(PHASES))
        cnt = np.zeros(len(PHASES), np.int64)
        rc = lib().ckkt_phase_times(self.h, _np_ptr(ms), _np_ptr(cnt))
        if rc:
            raise CKKTError(rc, "ckkt_phase_times")
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(PHASES)}

    def launch_count(self) -> int:
        return int(lib().ckkt_launch_count(self.h))

    # ---- device calls (torch CUDA tensors, batch-major)
    def refactor(self, w_val, g_val, h_val, sigma_x, d_s=None, delta_x=None, not_pd=None, min_bad_pivot=None):
        rc = lib().ckkt_refactor(self.h, _dptr(w_val), _dptr(g_val), _dptr(h_val), _dptr(sigma_x), _dptr(d_s),
                                 _dptr(delta_x), _dptr(not_pd), _dptr(min_bad_pivot))
        if rc:
            raise CKKTError(rc, "ckkt_refactor")

    def refactor_inertia(self, w_val, g_val, h_val, sigma_x, d_s, delta_x, delta_last=None, not_pd=None):
        """ckkt_refactor_inertia: delta_x is a device [B] FP64 tensor the library fills (keep it alive
        until the last solve); returns (status, accepted deltas [B], trials [B]) as numpy arrays."""
        dl = None if delta_last is None else np.ascontiguousarray(delta_last, dtype=np.float64)
        dout = np.zeros(self.batch, np.float64)
        tout = np.zeros(self.batch, np.int32)
        rc = lib().ckkt_refactor_inertia(self.h, _dptr(w_val), _dptr(g_val), _dptr(h_val), _dptr(sigma_x),
                                         _dptr(d_s), _hptr(dl), _dptr(delta_x), _hptr(dout), _hptr(tout),
                                         _dptr(not_pd))
        if rc not in (CKKT_OK, CKKT_NOT_PD):
            raise CKKTError(rc, "ckkt_refactor_inertia")
        return rc, dout, tout

    def solve(self, r1, r2, r3, r4, dx, ds, dy, dz, want_info: bool = True):
        infos = (ckkt_info * self.batch)() if want_info else None
        rc = lib().ckkt_solve(self.h, _dptr(r1), _dptr(r2), _dptr(r3), _dptr(r4), _dptr(dx), _dptr(ds), _dptr(dy),
                              _dptr(dz), infos)
        if rc in (CKKT_INVALID_ARG, CKKT_CUDA_ERROR, CKKT_OUT_OF_MEMORY, CKKT_PATTERN_ERROR):
            raise CKKTError(rc, "ckkt_solve")
        return rc, ([i.as_dict() for i in infos] if want_info else None)

    def iterate_host(self, w_val, g_val, h_val, sigma_x, d_s, delta_x, r1, r2, r3, r4, dx, ds, dy, dz, not_pd=None):
        infos = (ckkt_info * self.batch)()
        rc = lib().ckkt_iterate_host(self.h, _hptr(w_val), _hptr(g_val), _hptr(h_val), _hptr(sigma_x), _hptr(d_s),
                                     _hptr(delta_x), _hptr(r1), _hptr(r2), _hptr(r3), _hptr(r4), _hptr(dx), _hptr(ds),
                                     _hptr(dy), _hptr(dz), _hptr(not_pd), infos)
        if rc in (CKKT_INVALID_ARG, CKKT_CUDA_ERROR, CKKT_OUT_OF_MEMORY, CKKT_PATTERN_ERROR):
            raise CKKTError(rc, "ckkt_iterate_host")
        return rc, [i.as_dict() for i in infos]
