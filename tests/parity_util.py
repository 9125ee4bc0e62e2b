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


def gpu_solver(p, mu=(2, 2), execution=0):
    from paper_2104_13755_b200 import mg
    return mg.Solver(p.levels, p.P, mu_pre=mu[0], mu_post=mu[1], execution=execution)


def tau_floor(A_scipy, X, B):
    """Rounding floor of rho at iterate X: 32 u || |A||x| + |b| || / ||b|| per
    column (reading A20)."""
    absA = abs(A_scipy)
    X2 = X.reshape(X.shape[0], -1)
    B2 = B.reshape(B.shape[0], -1)
    num = np.linalg.norm(absA @ np.abs(X2) + np.abs(B2), axis=0)
    den = np.linalg.norm(B2, axis=0)
    den = np.where(den > 0, den, 1.0)
    return 32 * U * num / den


def oracle_solve_tau(mgo, A_scipy, B, X0=None, rel_tol=0.0, max_cycles=100):
    """The oracle's Alg. 1 loop run cycle by cycle (ora_mg_solve is exactly
    vcycle + residual norm per cycle, oracle.cpp), so that tau_k is taken at
    the iterate x_k it belongs to.  rho_k is the oracle's own residual norm
    (mgo.solve with max_cycles = 0 at x_k).  Returns (X, hist, rc, tau) with
    hist and tau of shape [cycles + 1, k]; rc as ora_mg_solve."""
    B = np.ascontiguousarray(B, np.float64)
    X = np.zeros(B.shape) if X0 is None else np.ascontiguousarray(X0, np.float64).copy()
    hist, taus = [], []

    def rho(Xc):
        _, h, _ = mgo.solve(B, X0=Xc, rel_tol=0.0, max_cycles=0)
        return h[0]

    def done(r):
        return rel_tol > 0.0 and np.all(r <= rel_tol)

    hist.append(rho(X))
    taus.append(tau_floor(A_scipy, X, B))
    rc = 8
    if not np.all(np.isfinite(hist[-1])):
        rc = 7
    elif done(hist[-1]):
        rc = 0
    while rc == 8 and len(hist) - 1 < max_cycles:
        mgo.vcycle(B, X)
        hist.append(rho(X))
        taus.append(tau_floor(A_scipy, X, B))
        if not np.all(np.isfinite(hist[-1])):
            rc = 7
        elif done(hist[-1]):
            rc = 0
    if rc == 8 and not rel_tol > 0.0:
        rc = 0
    return X, np.array(hist), rc, np.array(taus)


def _log_path():
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    return os.environ.get("MG_PARITY_LOG", os.path.join(root, "gpurun_out", "parity_literal.jsonl"))


def check_history(h_gpu, h_ora, tau, tag=None):
    """|rho'_k - rho_k| <= 1e-8 rho_k + tau_k (floor-aware rule, reading A20),
    asserted.  BASELINE's literal rule |rho'_k - rho_k| <= 1e-8 rho_k is
    evaluated per cycle beside it and appended (with tag, the per-cycle
    outcome and the margins) to the parity log (gpurun_out/parity_literal.jsonl
    or $MG_PARITY_LOG).  tau: per cycle [cycles + 1, k] (tau at x_k) or per
    column [k].  Returns the per-cycle literal outcome (all columns)."""
    import inspect
    import json
    import os
    n = min(h_gpu.shape[0], h_ora.shape[0])
    tau = np.asarray(tau, np.float64)
    tau_k = tau[:n] if tau.ndim == 2 else np.broadcast_to(tau[None, :], h_ora[:n].shape)
    d = np.abs(h_gpu[:n] - h_ora[:n])
    bound = RHO_TOL * h_ora[:n] + tau_k
    lit = d <= RHO_TOL * h_ora[:n]
    literal = np.all(lit, axis=1)
    if tag is None:
        fr = inspect.stack()[1]
        tag = f"{os.path.basename(fr.filename)}::{fr.function}"
    rec = {"tag": tag, "cycles": int(n - 1), "literal_all": bool(literal.all()),
           "literal_per_cycle": [bool(v) for v in literal],
           "rel_diff_per_cycle": [float(v) for v in np.max(d / np.where(h_ora[:n] > 0, h_ora[:n], 1.0), axis=1)],
           "rho_oracle": [float(v) for v in np.max(h_ora[:n], axis=1)],
           "tau_over_rho": [float(v) for v in np.max(tau_k / np.where(h_ora[:n] > 0, h_ora[:n], 1.0), axis=1)],
           "a20_pass": bool(np.all(d <= bound))}
    try:
        path = _log_path()
        os.makedirs(os.path.dirname(path), exist_ok=True)
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
    except OSError:
        pass
    assert np.all(d <= bound), f"history mismatch: max excess {np.max(d - bound):.3e}\n{h_gpu[:n]}\n{h_ora[:n]}"
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
        diff = np.abs(g["val"] - o["val"])
        # row-normwise relative error
        rowmax = np.maximum.reduceat(np.abs(o["val"]), rp[:-1].astype(np.int64)) if o["nnz"] else np.zeros(0)
        rows = np.repeat(np.arange(o["n"]), np.diff(rp))
        rel = diff / np.where(rowmax[rows] > 0, rowmax[rows], 1.0)
        assert rel.max(initial=0.0) <= VAL_TOL, f"level {l}: value rel diff {rel.max():.3e}"
    return g, o
