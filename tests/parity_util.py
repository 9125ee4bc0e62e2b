"""Helpers shared by the GPU parity tests: run one synthetic problem through
the oracle (oracle/) and through the CUDA path (libmg via its binding), and
apply the tolerance rules of SURVEY.md §8(c.4) / DESIGN.md §4."""
from __future__ import annotations

import numpy as np

U = 2.0 ** -53
X_TOL = 1e-9        # BJ: relative difference in X (per column, normwise)
RHO_TOL = 1e-8      # BJ: relative difference in each cycle's residual norm
VAL_TOL = 1e-12     # internal: coarse operator values, mass (row-normwise)


def oracle_rhs(ora, p, M):
    if p.rhs_kind == "direct":
        return np.ascontiguousarray(p.rhs, np.float64)
    return np.ascontiguousarray(M[:, None] * p.rhs, np.float64)


def oracle_problem(ora, p, mu=(2, 2)):
    V, F = p.levels[0]
    A, M = ora.assemble(V, F, p.mass_coeff, p.lap_coeff)
    mg = ora.MG(p.sizes, p.P, A, *mu)
    return A, M, mg


def gpu_solver(p, mu=(2, 2)):
    from paper_2104_13755_b200 import mg
    return mg.Solver(p.levels, p.P, mu_pre=mu[0], mu_post=mu[1])


def tau_floor(A_scipy, X, B):
    """Rounding floor of rho: 32 u || |A||x| + |b| || / ||b|| per column."""
    absA = abs(A_scipy)
    num = np.linalg.norm(absA @ np.abs(X) + np.abs(B), axis=0)
    den = np.linalg.norm(B, axis=0)
    den = np.where(den > 0, den, 1.0)
    return 32 * U * num / den


def check_history(h_gpu, h_ora, tau):
    """|rho' - rho| <= 1e-8 rho + tau (floor-aware rule, reading A20)."""
    n = min(h_gpu.shape[0], h_ora.shape[0])
    d = np.abs(h_gpu[:n] - h_ora[:n])
    bound = RHO_TOL * h_ora[:n] + tau[None, :]
    assert np.all(d <= bound), f"history mismatch: max excess {np.max(d - bound):.3e}\n{h_gpu[:n]}\n{h_ora[:n]}"
    literal = np.all(d <= RHO_TOL * h_ora[:n])
    return literal


def check_x(Xg, Xo, tol=X_TOL):
    for c in range(Xo.shape[1]):
        den = np.linalg.norm(Xo[:, c])
        err = np.linalg.norm(Xg[:, c] - Xo[:, c]) / (den if den > 0 else 1.0)
        assert err <= tol, f"column {c}: relative X difference {err:.3e} > {tol}"


def check_level_parity(solver, mg_ora, l, values=True):
    g = solver.level(l, values)
    o = mg_ora.level(l)
    assert np.array_equal(g["rowptr"], o["rowptr"].astype(np.int32)), f"level {l}: row_ptr differs"
    assert np.array_equal(g["col"], o["col"]), f"level {l}: columns differ"
    assert g["ncolours"] == o["ncolours"] and np.array_equal(g["colour"], o["colour"]), f"level {l}: colouring differs"
    if values:
        rp = o["rowptr"]
        for i in range(o["n"]):
            pass
        diff = np.abs(g["val"] - o["val"])
        # row-normwise relative error
        rowmax = np.maximum.reduceat(np.abs(o["val"]), rp[:-1].astype(np.int64)) if o["nnz"] else np.zeros(0)
        rows = np.repeat(np.arange(o["n"]), np.diff(rp))
        rel = diff / np.where(rowmax[rows] > 0, rowmax[rows], 1.0)
        assert rel.max(initial=0.0) <= VAL_TOL, f"level {l}: value rel diff {rel.max():.3e}"
    return g, o
