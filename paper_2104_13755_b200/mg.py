"""Thin ctypes binding over libmg (include/mg.h), same names as the C ABI.

Argument marshalling only: every step of the method runs in the sm_100a
kernels of libmg.so.  Arrays may be numpy arrays (host) or torch tensors
(host or CUDA); they are passed by pointer, never copied or computed on here.
There is no fallback: if libmg.so is missing or no CUDA device is visible
the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libmg.so")

MG_OK, MG_ERR_INVALID_ARG, MG_ERR_SHAPE, MG_ERR_INPUT, MG_ERR_NOT_SPD, MG_ERR_STATE, MG_ERR_CUDA, \
    MG_ERR_NUMERIC, MG_NOT_CONVERGED = range(9)
STATUS_NAMES = ["MG_OK", "MG_ERR_INVALID_ARG", "MG_ERR_SHAPE", "MG_ERR_INPUT", "MG_ERR_NOT_SPD", "MG_ERR_STATE",
                "MG_ERR_CUDA", "MG_ERR_NUMERIC", "MG_NOT_CONVERGED"]
PROF_CLASSES = ["gs_sweep", "residual_restrict", "prolong", "coarse_solve", "resnorm", "galerkin", "assembly",
                "factor", "permute", "coarse_tail", "alpha"]
PROF_LEVELS = 16


class MGError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS_NAMES[code] if 0 <= code < len(STATUS_NAMES) else code}: {msg}")
        self.code = code


_lib = None
_vp = C.c_void_p


def lib():
    """Load libmg.so (built in-tree by paper_2104_13755_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libmg.so not found at {LIB_PATH}: run `python -m paper_2104_13755_b200.build`")
        L = C.CDLL(LIB_PATH)
        i32, i64, dbl = C.c_int32, C.c_int64, C.c_double
        sig = {
            "mg_create": (C.c_int, [C.POINTER(_vp), C.c_int, _vp]),
            "mg_destroy": (None, [_vp]),
            "mg_last_error": (C.c_char_p, [_vp]),
            "mg_set_options": (C.c_int, [_vp, C.c_int, C.c_int]),
            "mg_hierarchy_load": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]),
            "mg_set_matrix": (C.c_int, [_vp, i32, i64, _vp, _vp, _vp, C.c_int]),
            "mg_set_matrix_cotan": (C.c_int, [_vp, _vp, dbl, dbl]),
            "mg_apply_mass": (C.c_int, [_vp, i32, _vp, _vp]),
            "mg_set_matrix_split": (C.c_int, [_vp, i32, i64, _vp, _vp, _vp, _vp]),
            "mg_set_matrix_split_cotan": (C.c_int, [_vp, _vp]),
            "mg_set_alpha": (C.c_int, [_vp, dbl]),
            "mg_set_smoother": (C.c_int, [_vp, C.c_int, dbl, C.c_int]),
            "mg_set_zero_guess": (C.c_int, [_vp, C.c_int32]),
            "mg_set_dirichlet": (C.c_int, [_vp, i32, _vp]),
            "mg_set_matrix_bilaplacian": (C.c_int, [_vp, _vp, dbl, dbl]),
            "mg_solve_pcg": (C.c_int, [_vp, i32, _vp, _vp, dbl, i32, _vp, _vp]),
            "mg_solve": (C.c_int, [_vp, i32, _vp, _vp, dbl, i32, _vp, _vp]),
            "mg_level_info": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp]),
            "mg_get_level_csr": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp]),
            "mg_get_colouring": (C.c_int, [_vp, C.c_int, _vp]),
            "mg_get_mass": (C.c_int, [_vp, _vp]),
            "mg_get_coarse_factor": (C.c_int, [_vp, _vp]),
            "mg_util_greedy_colouring": (C.c_int, [i32, _vp, _vp, _vp, _vp]),
            "mg_util_galerkin_pattern": (C.c_int, [i32, _vp, _vp, i32, _vp, _vp, _vp, _vp, _vp]),
            "mg_util_one_ring": (C.c_int, [i32, i32, _vp, _vp, _vp, _vp, _vp]),
            "mg_set_profiling": (C.c_int, [_vp, C.c_int]),
            "mg_get_profile": (C.c_int, [_vp, _vp, _vp]),
            "mg_launch_count": (i64, [_vp]),
            "mg_problem_size": (C.c_int, [_vp, _vp, _vp]),
            "mg_set_execution": (C.c_int, [_vp, C.c_int]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ptr(a, dtype):
    """Pointer of a contiguous numpy array / torch tensor of the given dtype."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if a.dtype != dtype or not a.flags.c_contiguous:
            raise TypeError(f"expected C-contiguous {np.dtype(dtype)} array, got {a.dtype}")
        return a.ctypes.data
    # torch tensor
    import torch
    tdt = {np.float64: torch.float64, np.int32: torch.int32, np.int64: torch.int64}[np.dtype(dtype).type]
    if a.dtype != tdt or not a.is_contiguous():
        raise TypeError(f"expected contiguous {tdt} tensor, got {a.dtype}")
    return a.data_ptr()


def mg_problem_size(ctx):
    """(n_full, device) of the loaded hierarchy."""
    n, dev = C.c_int32(), C.c_int32()
    _check(ctx, lib().mg_problem_size(ctx, C.byref(n), C.byref(dev)))
    return n.value, dev.value


def _check_rows(ctx, a, k, name):
    """The C side cannot see extents: B / X / V must be (n_full, k) (or (n_full,)
    for k = 1), and a CUDA tensor must live on the context's device."""
    if a is None:
        return
    n, dev = mg_problem_size(ctx)
    shape = tuple(a.shape)
    if not (shape == (n, k) or (k == 1 and shape == (n,))):
        raise ValueError(f"{name}: expected shape ({n}, {k}), got {shape}")
    if not isinstance(a, np.ndarray) and getattr(a, "is_cuda", False) and a.device.index != dev:
        raise ValueError(f"{name}: tensor on cuda:{a.device.index}, context on cuda:{dev}")


def _check_len(a, count, name):
    if a is not None and int(np.prod(a.shape)) < count:
        raise ValueError(f"{name}: needs at least {count} entries, got {int(np.prod(a.shape))}")


def _check(ctx, rc, allow=()):
    if rc != MG_OK and rc not in allow:
        msg = lib().mg_last_error(ctx).decode() if ctx else ""
        raise MGError(rc, msg)
    return rc


# ---------------------------------------------------------------------------
# C-ABI mirrors


def mg_create(device=0, stream=None):
    """Returns an opaque context handle.  `stream`: a cudaStream_t integer
    (torch.cuda.current_stream().cuda_stream) or None for a private stream."""
    h = _vp()
    rc = lib().mg_create(C.byref(h), int(device), stream or None)
    if rc != MG_OK:
        raise MGError(rc, "mg_create failed (no CUDA device or driver error)")
    return h


def mg_destroy(ctx):
    lib().mg_destroy(ctx)


def mg_last_error(ctx):
    return lib().mg_last_error(ctx).decode()


MG_EXEC_NO_PDL, MG_EXEC_NO_PIPE, MG_EXEC_COARSE_TRSV, MG_EXEC_DEVICE_LOOP = 1, 2, 4, 8


def mg_set_execution(ctx, flags=0):
    """Scheduling options (include/mg.h MG_EXEC_*); call before mg_set_matrix*."""
    return _check(ctx, lib().mg_set_execution(ctx, int(flags)))


def mg_set_options(ctx, mu_pre=2, mu_post=2):
    return _check(ctx, lib().mg_set_options(ctx, int(mu_pre), int(mu_post)))


def mg_hierarchy_load(ctx, levels, P):
    """levels: [(V_l float64 [n_l,3], F_l int32 [m_l,3] or None)], P: [(cols int32 [n_l,3], w float64 [n_l,3])]."""
    nl = len(levels)
    keep = []
    Vs = [np.ascontiguousarray(V, np.float64) for V, _ in levels]
    Fs = [None if F is None else np.ascontiguousarray(F, np.int32) for _, F in levels]
    n_verts = np.array([V.shape[0] for V in Vs], np.int32)
    n_faces = np.array([0 if F is None else F.shape[0] for F in Fs], np.int32)
    Varr = (C.c_void_p * nl)(*[V.ctypes.data for V in Vs])
    Farr = (C.c_void_p * nl)(*[None if F is None else F.ctypes.data for F in Fs])
    Pc = [np.ascontiguousarray(c, np.int32) for c, _ in P[: nl - 1]]
    Pw = [np.ascontiguousarray(w, np.float64) for _, w in P[: nl - 1]]
    Pcarr = (C.c_void_p * max(1, nl - 1))(*[c.ctypes.data for c in Pc])
    Pwarr = (C.c_void_p * max(1, nl - 1))(*[w.ctypes.data for w in Pw])
    keep += [Vs, Fs, Pc, Pw]
    return _check(ctx, lib().mg_hierarchy_load(ctx, nl, n_verts.ctypes.data, n_faces.ctypes.data,
                                               C.cast(Varr, C.c_void_p), C.cast(Farr, C.c_void_p),
                                               C.cast(Pcarr, C.c_void_p), C.cast(Pwarr, C.c_void_p)))


def mg_set_matrix(ctx, n, nnz, row_ptr, col, val, on_device=0):
    _check_len(row_ptr, n + 1, "row_ptr")
    _check_len(col, nnz, "col")
    _check_len(val, nnz, "val")
    return _check(ctx, lib().mg_set_matrix(ctx, int(n), int(nnz), _ptr(row_ptr, np.int32), _ptr(col, np.int32),
                                           _ptr(val, np.float64), int(on_device)))


def mg_set_matrix_cotan(ctx, V, mass_coeff, lap_coeff):
    _check_rows(ctx, V, 3, "V")
    return _check(ctx, lib().mg_set_matrix_cotan(ctx, _ptr(V, np.float64), float(mass_coeff), float(lap_coeff)))


def mg_set_matrix_split(ctx, n, nnz, row_ptr, col, q_val, m_val):
    _check_len(row_ptr, n + 1, "row_ptr")
    for a, nm in ((col, "col"), (q_val, "q_val"), (m_val, "m_val")):
        _check_len(a, nnz, nm)
    return _check(ctx, lib().mg_set_matrix_split(ctx, int(n), int(nnz), _ptr(row_ptr, np.int32), _ptr(col, np.int32),
                                                 _ptr(q_val, np.float64), _ptr(m_val, np.float64)))


def mg_set_matrix_split_cotan(ctx, V):
    _check_rows(ctx, V, 3, "V")
    return _check(ctx, lib().mg_set_matrix_split_cotan(ctx, _ptr(V, np.float64)))


def mg_set_alpha(ctx, alpha):
    return _check(ctx, lib().mg_set_alpha(ctx, float(alpha)))


def mg_apply_mass(ctx, k, X, B):
    _check_rows(ctx, X, k, "X")
    _check_rows(ctx, B, k, "B")
    return _check(ctx, lib().mg_apply_mass(ctx, int(k), _ptr(X, np.float64), _ptr(B, np.float64)))


def mg_solve(ctx, k, B, X, rel_tol, max_cycles, res_hist=None):
    """Returns (status, cycles); status MG_OK or MG_NOT_CONVERGED (others raise).
    res_hist: optional float64 numpy array of (max_cycles+1)*k entries."""
    _check_rows(ctx, B, k, "B")
    _check_rows(ctx, X, k, "X")
    _check_len(res_hist, (int(max_cycles) + 1) * int(k), "res_hist")
    cyc = C.c_int32(0)
    rc = lib().mg_solve(ctx, int(k), _ptr(B, np.float64), _ptr(X, np.float64), float(rel_tol), int(max_cycles),
                        _ptr(res_hist, np.float64), C.byref(cyc))
    _check(ctx, rc, allow=(MG_NOT_CONVERGED,))
    return rc, cyc.value


def mg_set_matrix_bilaplacian(ctx, V, mass_coeff, bilap_coeff):
    _check_rows(ctx, V, 3, "V")
    return _check(ctx, lib().mg_set_matrix_bilaplacian(ctx, _ptr(V, np.float64), float(mass_coeff), float(bilap_coeff)))


def mg_set_dirichlet(ctx, known):
    """Known fine vertices (App. B); an empty list removes the constraints."""
    known = np.ascontiguousarray(np.asarray(known, dtype=np.int32))
    return _check(ctx, lib().mg_set_dirichlet(ctx, int(known.size), known.ctypes.data if known.size else None))


def mg_set_smoother(ctx, kind=0, omega=0.8, symmetric=False):
    """kind 0 multicolour GS, 1 damped Jacobi; symmetric: reversed post colours."""
    return _check(ctx, lib().mg_set_smoother(ctx, int(kind), float(omega), int(bool(symmetric))))


def mg_set_zero_guess(ctx, on=True):
    """Solves start from X0 = 0 and X is output only (not read, no H2D copy)."""
    return _check(ctx, lib().mg_set_zero_guess(ctx, int(bool(on))))


def mg_solve_pcg(ctx, k, B, X, rel_tol, max_iters, res_hist=None):
    """MG-preconditioned CG; returns (status, iterations)."""
    _check_rows(ctx, B, k, "B")
    _check_rows(ctx, X, k, "X")
    _check_len(res_hist, (int(max_iters) + 1) * int(k), "res_hist")
    it = C.c_int32(0)
    rc = lib().mg_solve_pcg(ctx, int(k), _ptr(B, np.float64), _ptr(X, np.float64), float(rel_tol), int(max_iters),
                            _ptr(res_hist, np.float64), C.byref(it))
    _check(ctx, rc, allow=(MG_NOT_CONVERGED,))
    return rc, it.value


def mg_level_info(ctx, l):
    n, nnz, nc = C.c_int32(), C.c_int64(), C.c_int32()
    _check(ctx, lib().mg_level_info(ctx, int(l), C.byref(n), C.byref(nnz), C.byref(nc)))
    return n.value, nnz.value, nc.value


def mg_get_level_csr(ctx, l, values=True):
    n, nnz, _ = mg_level_info(ctx, l)
    rp = np.empty(n + 1, np.int32)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64) if values else None
    _check(ctx, lib().mg_get_level_csr(ctx, int(l), rp.ctypes.data, col.ctypes.data,
                                       None if val is None else val.ctypes.data))
    return rp, col, val


def mg_get_colouring(ctx, l):
    n, _, _ = mg_level_info(ctx, l)
    out = np.empty(n, np.int32)
    _check(ctx, lib().mg_get_colouring(ctx, int(l), out.ctypes.data))
    return out


def mg_get_mass(ctx, n):
    M = np.empty(n, np.float64)
    _check(ctx, lib().mg_get_mass(ctx, M.ctypes.data))
    return M


def mg_get_coarse_factor(ctx, n_coarse):
    L = np.empty((n_coarse, n_coarse), np.float64)
    _check(ctx, lib().mg_get_coarse_factor(ctx, L.ctypes.data))
    return L


def mg_util_greedy_colouring(row_ptr, col):
    row_ptr = np.ascontiguousarray(row_ptr, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    n = row_ptr.shape[0] - 1
    out = np.empty(n, np.int32)
    k = C.c_int32()
    rc = lib().mg_util_greedy_colouring(n, row_ptr.ctypes.data, col.ctypes.data, out.ctypes.data, C.byref(k))
    if rc:
        raise MGError(rc, "mg_util_greedy_colouring")
    return out, k.value


def mg_util_one_ring(n, F, slots=True):
    """(row_ptr, col, slots) of the 1-ring pattern of faces F [nF][3]."""
    F = np.ascontiguousarray(F, np.int32)
    rp = np.zeros(n + 1, np.int32)
    nnz = C.c_int64(0)
    rc = lib().mg_util_one_ring(int(n), F.shape[0], F.ctypes.data, rp.ctypes.data, C.byref(nnz), None, None)
    if rc != MG_OK:
        raise MGError(rc, "mg_util_one_ring")
    col = np.zeros(nnz.value, np.int32)
    sl = np.zeros(nnz.value, np.uint8) if slots else None
    rc = lib().mg_util_one_ring(int(n), F.shape[0], F.ctypes.data, rp.ctypes.data, C.byref(nnz), col.ctypes.data,
                                sl.ctypes.data if slots else None)
    if rc != MG_OK:
        raise MGError(rc, "mg_util_one_ring")
    return rp, col, sl


def mg_util_galerkin_pattern(row_ptr, col, n_coarse, P_cols, P_w):
    row_ptr = np.ascontiguousarray(row_ptr, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    Pc = np.ascontiguousarray(P_cols, np.int32)
    Pw = np.ascontiguousarray(P_w, np.float64)
    n = row_ptr.shape[0] - 1
    crp = np.empty(n_coarse + 1, np.int32)
    nnz = C.c_int64()
    rc = lib().mg_util_galerkin_pattern(n, row_ptr.ctypes.data, col.ctypes.data, int(n_coarse), Pc.ctypes.data,
                                        Pw.ctypes.data, crp.ctypes.data, C.byref(nnz), None)
    if rc:
        raise MGError(rc, "mg_util_galerkin_pattern")
    ccol = np.empty(nnz.value, np.int32)
    rc = lib().mg_util_galerkin_pattern(n, row_ptr.ctypes.data, col.ctypes.data, int(n_coarse), Pc.ctypes.data,
                                        Pw.ctypes.data, crp.ctypes.data, C.byref(nnz), ccol.ctypes.data)
    if rc:
        raise MGError(rc, "mg_util_galerkin_pattern")
    return crp, ccol


def mg_set_profiling(ctx, classes=True):
    """classes: True (all), False (off), an int bit mask, or kernel-class names."""
    if classes is True:
        mask = (1 << len(PROF_CLASSES)) - 1
    elif classes is False or classes is None:
        mask = 0
    elif isinstance(classes, int):
        mask = classes
    else:
        mask = 0
        for name in classes:
            mask |= 1 << PROF_CLASSES.index(name)
    return _check(ctx, lib().mg_set_profiling(ctx, int(mask)))


def mg_get_profile(ctx):
    """Returns {class: {level: (ms, launches)}} accumulated since the last call."""
    ms = np.zeros(len(PROF_CLASSES) * PROF_LEVELS)
    n = np.zeros(len(PROF_CLASSES) * PROF_LEVELS, np.int64)
    _check(ctx, lib().mg_get_profile(ctx, ms.ctypes.data, n.ctypes.data))
    out = {}
    for ci, name in enumerate(PROF_CLASSES):
        d = {l: (float(ms[ci * PROF_LEVELS + l]), int(n[ci * PROF_LEVELS + l]))
             for l in range(PROF_LEVELS) if n[ci * PROF_LEVELS + l]}
        if d:
            out[name] = d
    return out


def mg_launch_count(ctx):
    return int(lib().mg_launch_count(ctx))


# ---------------------------------------------------------------------------
# Convenience object (still marshalling only)


class Solver:
    """RAII wrapper: hierarchy + matrix + solve on one context."""

    def __init__(self, levels, P, device=0, stream=None, mu_pre=2, mu_post=2, execution=0):
        self.ctx = mg_create(device, stream)
        self.levels = levels
        self.n = levels[0][0].shape[0]
        self.sizes = [V.shape[0] for V, _ in levels]
        mg_hierarchy_load(self.ctx, levels, P)
        mg_set_options(self.ctx, mu_pre, mu_post)
        if execution:
            mg_set_execution(self.ctx, execution)

    def close(self):
        if getattr(self, "ctx", None) is not None:
            mg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_matrix(self, row_ptr, col, val):
        return mg_set_matrix(self.ctx, self.n, col.shape[0], row_ptr, col, val)

    def set_matrix_cotan(self, V, mass_coeff, lap_coeff):
        return mg_set_matrix_cotan(self.ctx, V, mass_coeff, lap_coeff)

    def set_matrix_split(self, row_ptr, col, q_val, m_val):
        return mg_set_matrix_split(self.ctx, self.n, col.shape[0], row_ptr, col, q_val, m_val)

    def set_matrix_split_cotan(self, V):
        return mg_set_matrix_split_cotan(self.ctx, V)

    def set_alpha(self, alpha):
        return mg_set_alpha(self.ctx, alpha)

    def apply_mass(self, X, B):
        k = 1 if X.ndim == 1 else X.shape[1]
        return mg_apply_mass(self.ctx, k, X, B)

    def solve(self, B, X, rel_tol=1e-10, max_cycles=100, history=True):
        k = 1 if B.ndim == 1 else B.shape[1]
        hist = np.full((max_cycles + 1) * k, np.nan) if history else None
        rc, cyc = mg_solve(self.ctx, k, B, X, rel_tol, max_cycles, hist)
        if hist is not None:
            hist = hist.reshape(max_cycles + 1, k)[: cyc + 1]
        return rc, cyc, hist

    def set_matrix_bilaplacian(self, V, mass_coeff, bilap_coeff):
        return mg_set_matrix_bilaplacian(self.ctx, V, mass_coeff, bilap_coeff)

    def set_dirichlet(self, known):
        return mg_set_dirichlet(self.ctx, known)

    def set_smoother(self, kind=0, omega=0.8, symmetric=False):
        return mg_set_smoother(self.ctx, kind, omega, symmetric)

    def set_zero_guess(self, on=True):
        return mg_set_zero_guess(self.ctx, on)

    def solve_pcg(self, B, X, rel_tol=1e-10, max_iters=100, history=True):
        k = 1 if B.ndim == 1 else B.shape[1]
        hist = np.full((max_iters + 1) * k, np.nan) if history else None
        rc, it = mg_solve_pcg(self.ctx, k, B, X, rel_tol, max_iters, hist)
        if hist is not None:
            hist = hist.reshape(max_iters + 1, k)[: it + 1]
        return rc, it, hist

    def level(self, l, values=True):
        rp, col, val = mg_get_level_csr(self.ctx, l, values)
        return dict(rowptr=rp, col=col, val=val, colour=mg_get_colouring(self.ctx, l),
                    ncolours=mg_level_info(self.ctx, l)[2])
