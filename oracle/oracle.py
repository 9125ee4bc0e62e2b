"""ctypes wrapper over the plain C++ oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2104_13755_b200) never imports this module, and this module imports
nothing from the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

CXXFLAGS = ["-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def _src_hash():
    import hashlib
    with open(_SRC, "rb") as f:
        return hashlib.sha256(" ".join(CXXFLAGS).encode() + f.read()).hexdigest()


def build(force=False):
    """Compile the oracle (g++, single-threaded, no FMA contraction; reading
    A18).  Rebuilt whenever the source hash recorded beside the library differs."""
    hfile = _LIB + ".sha256"
    h = _src_hash()
    if not force and os.path.exists(_LIB) and os.path.exists(hfile) and open(hfile).read().strip() == h:
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["g++", *CXXFLAGS, _SRC, "-o", tmp])
    os.replace(tmp, _LIB)
    with open(hfile, "w") as f:
        f.write(h + "\n")
    return _LIB


_lib = None
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_vp = C.c_void_p


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        sig = {
            "ora_csr_new": (_vp, [C.c_int32, C.c_int32, _i64p, _i32p, _f64p]),
            "ora_csr_free": (None, [_vp]),
            "ora_csr_rows": (C.c_int32, [_vp]),
            "ora_csr_cols": (C.c_int32, [_vp]),
            "ora_csr_nnz": (C.c_int64, [_vp]),
            "ora_csr_export": (None, [_vp, _i64p, _i32p, _f64p]),
            "ora_cotan_laplacian": (_vp, [C.c_int32, C.c_int32, _f64p, _i32p]),
            "ora_lumped_mass": (None, [C.c_int32, C.c_int32, _f64p, _i32p, _f64p]),
            "ora_mass_plus_laplacian": (_vp, [_vp, _f64p, C.c_double, C.c_double]),
            "ora_spmv": (None, [_vp, C.c_int32, _f64p, _f64p]),
            "ora_prolongation": (_vp, [C.c_int32, C.c_int32, _i32p, _f64p]),
            "ora_galerkin": (_vp, [_vp, _vp]),
            "ora_greedy_colouring": (C.c_int32, [_vp, _i32p]),
            "ora_cholesky": (C.c_int, [C.c_int32, _f64p, _f64p]),
            "ora_cholesky_solve": (None, [C.c_int32, _f64p, C.c_int32, _f64p, _f64p]),
            "ora_gs_sweep": (None, [_vp, _i32p, C.c_int32, C.c_int32, _f64p, _f64p]),
            "ora_mg_new": (_vp, [C.c_int32, _i32p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), _vp,
                                 C.c_int32, C.c_int32]),
            "ora_mg_free": (None, [_vp]),
            "ora_mg_status": (C.c_int, [_vp]),
            "ora_mg_levels": (C.c_int32, [_vp]),
            "ora_mg_level_info": (None, [_vp, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int32)]),
            "ora_mg_level_export": (None, [_vp, C.c_int32, _i64p, _i32p, _f64p, _i32p]),
            "ora_mg_coarse_factor": (None, [_vp, _f64p]),
            "ora_mg_vcycle": (None, [_vp, C.c_int32, _f64p, _f64p]),
            "ora_mg_solve": (C.c_int, [_vp, C.c_int32, _f64p, _f64p, C.c_double, C.c_int32, _f64p,
                                       C.POINTER(C.c_int32)]),
            "ora_mg_set_smoother": (None, [_vp, C.c_int32, C.c_double, C.c_int32]),
            "ora_mg_phase_times": (None, [_vp, _f64p]),
            "ora_jacobi_sweep": (None, [_vp, C.c_int32, _f64p, _f64p, C.c_double]),
            "ora_mg_pcg": (C.c_int, [_vp, C.c_int32, _f64p, _f64p, C.c_double, C.c_int32, _f64p,
                                     C.POINTER(C.c_int32)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class Csr:
    """Owned oracle CSR handle."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ora_csr_free(self.h)
            self.h = None

    @classmethod
    def from_arrays(cls, nrows, ncols, rowptr, col, val):
        return cls(lib().ora_csr_new(nrows, ncols, np.ascontiguousarray(rowptr, np.int64), _i32(col), _f64(val)))

    @classmethod
    def from_scipy(cls, S):
        S = S.tocsr()
        S.sort_indices()
        return cls.from_arrays(S.shape[0], S.shape[1], S.indptr.astype(np.int64), S.indices, S.data)

    @property
    def shape(self):
        return (lib().ora_csr_rows(self.h), lib().ora_csr_cols(self.h))

    @property
    def nnz(self):
        return lib().ora_csr_nnz(self.h)

    def arrays(self):
        n, _ = self.shape
        nnz = self.nnz
        rp = np.empty(n + 1, np.int64)
        col = np.empty(nnz, np.int32)
        val = np.empty(nnz, np.float64)
        lib().ora_csr_export(self.h, rp, col, val)
        return rp, col, val

    def to_scipy(self):
        import scipy.sparse as sp
        rp, col, val = self.arrays()
        return sp.csr_matrix((val, col, rp), shape=self.shape)

    def spmv(self, X):
        X = _f64(X)
        k = 1 if X.ndim == 1 else X.shape[1]
        Y = np.empty((self.shape[0], k))
        lib().ora_spmv(self.h, k, X, Y)
        return Y[:, 0] if X.ndim == 1 else Y


def cotan_laplacian(V, F):
    V, F = _f64(V), _i32(F)
    return Csr(lib().ora_cotan_laplacian(V.shape[0], F.shape[0], V, F))


def lumped_mass(V, F):
    V, F = _f64(V), _i32(F)
    M = np.empty(V.shape[0])
    lib().ora_lumped_mass(V.shape[0], F.shape[0], V, F, M)
    return M


def mass_plus_laplacian(L, M, mass_coeff, lap_coeff):
    return Csr(lib().ora_mass_plus_laplacian(L.h, _f64(M), float(mass_coeff), float(lap_coeff)))


def assemble(V, F, mass_coeff, lap_coeff):
    """A = mass_coeff M + lap_coeff L (and M), both from (V, F)."""
    L = cotan_laplacian(V, F)
    M = lumped_mass(V, F)
    return mass_plus_laplacian(L, M, mass_coeff, lap_coeff), M


def bilaplacian(V, F):
    """Row f3: Q = L M^{-1} L (E_{Delta^2}) from
    the oracle's cotan L and lumped M, one scipy sparse product (a library
    primitive); returns (Q as Csr, M)."""
    import scipy.sparse as sp
    L = cotan_laplacian(V, F).to_scipy()
    M = lumped_mass(V, F)
    Q = (L @ sp.diags(1.0 / M) @ L).tocsr()
    Q.sort_indices()
    return Csr.from_scipy(Q), M


def assemble_bilaplacian(V, F, mass_coeff, bilap_coeff):
    """A = mass_coeff M + bilap_coeff L M^{-1} L on the 2-ring pattern (and M)."""
    import scipy.sparse as sp
    Q, M = bilaplacian(V, F)
    A = (bilap_coeff * Q.to_scipy() + mass_coeff * sp.diags(M)).tocsr()
    A.sort_indices()
    return Csr.from_scipy(A), M


def prolongation(n_coarse, cols, w):
    cols, w = _i32(cols), _f64(w)
    return Csr(lib().ora_prolongation(cols.shape[0], n_coarse, cols, w))


def galerkin(P, A):
    return Csr(lib().ora_galerkin(P.h, A.h))


def greedy_colouring(A):
    col = np.empty(A.shape[0], np.int32)
    k = lib().ora_greedy_colouring(A.h, col)
    return col, k


def cholesky(A):
    A = _f64(A)
    L = np.empty_like(A)
    rc = lib().ora_cholesky(A.shape[0], A, L)
    if rc != 0:
        raise np.linalg.LinAlgError("oracle Cholesky: non-positive pivot")
    return L


def cholesky_solve(L, B):
    B = _f64(B)
    k = 1 if B.ndim == 1 else B.shape[1]
    X = np.empty(B.shape)
    lib().ora_cholesky_solve(L.shape[0], _f64(L), k, B, X)
    return X


def gs_sweep(A, colour, ncolours, B, X):
    """One multicolour GS sweep, X updated in place (must be float64 C-contiguous)."""
    B = _f64(B)
    k = 1 if B.ndim == 1 else B.shape[1]
    assert X.dtype == np.float64 and X.flags.c_contiguous
    lib().ora_gs_sweep(A.h, _i32(colour), int(ncolours), k, B, X)
    return X


def jacobi_sweep(A, B, X, omega=0.8):
    """One damped Jacobi sweep (App. E), X updated in place."""
    B = _f64(B)
    k = 1 if B.ndim == 1 else B.shape[1]
    assert X.dtype == np.float64 and X.flags.c_contiguous
    lib().ora_jacobi_sweep(A.h, k, B, X, float(omega))
    return X


class MG:
    """Oracle multigrid: setup on construction; vcycle / solve."""

    def __init__(self, sizes, Ps, A0, mu_pre=2, mu_post=2):
        self._keep = []
        n_levels = len(sizes)
        cols = (C.c_void_p * max(1, n_levels - 1))()
        ws = (C.c_void_p * max(1, n_levels - 1))()
        for l, (c, w) in enumerate(Ps[: n_levels - 1]):
            c, w = _i32(c), _f64(w)
            self._keep += [c, w]
            cols[l] = c.ctypes.data
            ws[l] = w.ctypes.data
        self.A0 = A0
        self.h = lib().ora_mg_new(n_levels, _i32(sizes), cols, ws, A0.h, mu_pre, mu_post)
        self.status = lib().ora_mg_status(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ora_mg_free(self.h)
            self.h = None

    @property
    def n_levels(self):
        return lib().ora_mg_levels(self.h)

    def level(self, l):
        n, nnz, nc = C.c_int32(), C.c_int64(), C.c_int32()
        lib().ora_mg_level_info(self.h, l, C.byref(n), C.byref(nnz), C.byref(nc))
        rp = np.empty(n.value + 1, np.int64)
        col = np.empty(nnz.value, np.int32)
        val = np.empty(nnz.value)
        colour = np.empty(n.value, np.int32)
        lib().ora_mg_level_export(self.h, l, rp, col, val, colour)
        return dict(n=n.value, nnz=nnz.value, ncolours=nc.value, rowptr=rp, col=col, val=val, colour=colour)

    def phase_times(self):
        """Wall-clock seconds of the setup phases (Galerkin symbolic + numeric,
        colouring, coarsest Cholesky) and of the last solve (V-cycles, residual
        norms).  Timing only (bench.py's CPU baseline)."""
        t = np.zeros(5)
        lib().ora_mg_phase_times(self.h, t)
        return dict(zip(("galerkin_s", "colouring_s", "cholesky_s", "vcycles_s", "norms_s"), map(float, t)))

    def coarse_factor(self):
        n = self.level(self.n_levels - 1)["n"]
        L = np.empty((n, n))
        lib().ora_mg_coarse_factor(self.h, L)
        return L

    def vcycle(self, B, X):
        B = _f64(B)
        k = 1 if B.ndim == 1 else B.shape[1]
        assert X.dtype == np.float64 and X.flags.c_contiguous
        lib().ora_mg_vcycle(self.h, k, B, X)
        return X

    def set_smoother(self, kind=0, omega=0.8, symmetric=False):
        """kind 0 multicolour GS (reading A2), 1 damped Jacobi (App. E);
        symmetric: post-relaxation colours in reverse order (row f4)."""
        lib().ora_mg_set_smoother(self.h, int(kind), float(omega), int(bool(symmetric)))
        return self

    def pcg(self, B, X0=None, rel_tol=1e-10, max_iters=100):
        """MG-preconditioned CG (row f4); returns (X, history, rc)."""
        B = _f64(B)
        k = 1 if B.ndim == 1 else B.shape[1]
        X = np.zeros(B.shape) if X0 is None else _f64(X0).copy()
        hist = np.full((max_iters + 1) * k, np.nan)
        it = C.c_int32()
        rc = lib().ora_mg_pcg(self.h, k, B, X, float(rel_tol), int(max_iters), hist, C.byref(it))
        return X, hist.reshape(max_iters + 1, k)[: it.value + 1], rc

    def solve(self, B, X0=None, rel_tol=1e-10, max_cycles=100):
        B = _f64(B)
        k = 1 if B.ndim == 1 else B.shape[1]
        X = np.zeros(B.shape) if X0 is None else _f64(X0).copy()
        hist = np.full((max_cycles + 1) * k, np.nan)
        cyc = C.c_int32()
        rc = lib().ora_mg_solve(self.h, k, B, X, float(rel_tol), int(max_cycles), hist, C.byref(cyc))
        return X, hist.reshape(max_cycles + 1, k)[: cyc.value + 1], rc


def mcf(sizes, Ps, V0, F, dt, steps, rel_tol=1e-8, max_cycles=100, mu_pre=2, mu_post=2):
    """Implicit mean-curvature flow, config 5 (Fig. mcf, reading A15):
    per step rebuild L_t, M_t from the current positions X_t, A_t = M_t + dt L_t,
    B = M_t X_t, solve with warm start X_0 = X_t, X_{t+1} = X.  The hierarchy
    (Ps) is reused because connectivity is fixed."""
    X = _f64(V0).copy()
    cycles = []
    for _ in range(steps):
        A, M = assemble(X, F, 1.0, dt)
        mg = MG(sizes, Ps, A, mu_pre, mu_post)
        B = M[:, None] * X
        X, hist, rc = mg.solve(B, X0=X, rel_tol=rel_tol, max_cycles=max_cycles)
        cycles.append(hist.shape[0] - 1)
        if rc not in (0,):
            raise RuntimeError(f"oracle mcf: solve returned {rc}")
    return X, cycles


def dirichlet_reduce(sizes, Ps, known):
    """Dirichlet reduction of the hierarchy (App. B; row f2), plain
    numpy.  Returns (u, sizes', Ps', keep) where u = ascending unknown fine
    indices, P_0' = P_{u:} with its coarse columns renumbered, and, at every
    level, coarse columns whose maximum (absolute) weight over the kept rows
    is zero are removed together with "the corresponding rows in the
    prolongation at the next level".  Reading A24: the paper states
    the rule for the second-finest level; it is applied at every level until no
    column is all-zero, and the hierarchy stops at the last non-empty level.
    keep[l] = kept (original) indices of level l."""
    n0 = sizes[0]
    mask = np.ones(n0, bool)
    mask[np.asarray(known, np.int64)] = False
    keep = [np.nonzero(mask)[0]]
    new_sizes = [keep[0].size]
    new_P = []
    for l in range(len(sizes) - 1):
        if keep[-1].size == 0:
            break
        c, w = np.asarray(Ps[l][0]), np.asarray(Ps[l][1], np.float64)
        rows_c, rows_w = c[keep[-1]], w[keep[-1]]
        colmax = np.zeros(sizes[l + 1])
        np.maximum.at(colmax, rows_c.ravel(), np.abs(rows_w).ravel())
        kept_cols = np.nonzero(colmax > 0.0)[0]
        remap = -np.ones(sizes[l + 1], np.int64)
        remap[kept_cols] = np.arange(kept_cols.size)
        nc = np.where(rows_w != 0.0, remap[rows_c], 0)
        assert (nc >= 0).all()
        new_P.append((nc.astype(np.int32), np.where(rows_w != 0.0, rows_w, 0.0)))
        keep.append(kept_cols)
        new_sizes.append(kept_cols.size)
    if new_sizes[-1] == 0 and len(new_sizes) > 1:   # nothing survives below: stop at the last non-empty level
        new_sizes.pop()
        new_P.pop()
        keep.pop()
    return keep[0], new_sizes, new_P, keep


def dirichlet_solve(sizes, Ps, A, B, X0, known, rel_tol=1e-10, max_cycles=100, mu_pre=2, mu_post=2):
    """Constrained solve (App. B): x_k = X0[known] fixed; the reduced system
    A_uu x_u = b_u - A_uk x_k (eq. "reduced LHS/RHS") solved by the V-cycle on
    the reduced hierarchy of dirichlet_reduce.  Returns (X, history, rc,
    reduced MG object or None)."""
    B, X = _f64(B), _f64(X0).copy()
    u, rs, rP, _ = dirichlet_reduce(sizes, Ps, known)
    if u.size == 0:
        k = 1 if B.ndim == 1 else B.shape[1]
        return X, np.zeros((0, k)), 0, None
    S = A.to_scipy().tocsr()
    kn = np.setdiff1d(np.arange(S.shape[0]), u)
    Auu = S[u][:, u]
    bu = B[u] - S[u][:, kn] @ X[kn]
    mg = MG(rs, rP, Csr.from_scipy(Auu), mu_pre, mu_post)
    xu, hist, rc = mg.solve(bu, X0=X[u], rel_tol=rel_tol, max_cycles=max_cycles)
    X[u] = xu
    return X, hist, rc, mg
