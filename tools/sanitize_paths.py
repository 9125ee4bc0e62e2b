"""Small runs of every libmg path, for compute-sanitizer (one tool per call):
cotan / CSR / split + alpha / bilaplacian / Dirichlet / Jacobi / PCG on
configs 1 and 2 (reduced size) and the cylinder (boundary)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import meshgen  # noqa: E402
from paper_2104_13755_b200 import mg  # noqa: E402

for cid, kw in ((1, {}), (2, {"subdiv": 5}), (3, {"grid": (64, 48)})):
    p = meshgen.make_config(cid, **kw)
    V, F = p.levels[0]
    for k in (1, 3):
        S = mg.Solver(p.levels, p.P)
        S.set_matrix_cotan(V, 1.0, 1e-2)
        B = np.random.default_rng(0).standard_normal((p.n, k))
        X = np.zeros_like(B)
        S.solve(B, X, rel_tol=0.0, max_cycles=2)
        Xt = torch.zeros((p.n, k), dtype=torch.float64, device="cuda")
        S.solve(torch.from_numpy(B).cuda(), Xt, rel_tol=0.0, max_cycles=2)
        S.solve_pcg(B, np.zeros_like(B), rel_tol=0.0, max_iters=2)
        S.set_smoother(1, 0.8, True)
        S.solve(B, np.zeros_like(B), rel_tol=0.0, max_cycles=2)
        S.set_smoother(0, 0.8, False)
        S.set_matrix_split_cotan(V)
        S.set_alpha(0.3)
        S.solve(B, np.zeros_like(B), rel_tol=0.0, max_cycles=1)
        S.set_dirichlet(np.arange(0, p.n, 7))
        S.set_matrix_cotan(V, 1.0, 1e-2)
        S.solve(B, np.zeros_like(B), rel_tol=0.0, max_cycles=2)
        S.set_matrix_bilaplacian(V, 0.9, 0.1)
        S.solve(B, np.zeros_like(B), rel_tol=0.0, max_cycles=1)
        S.set_dirichlet([])
        S.close()
    print("config", cid, "ok", flush=True)
