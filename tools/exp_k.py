"""Experiment: per-level GS time of config 4 for k = 1, 2, 3 right-hand sides
(does the k = 3 iterate, 84 MB with 32-byte rows, stay L2-resident?)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import meshgen  # noqa: E402
from paper_2104_13755_b200 import mg  # noqa: E402

p = meshgen.make_config(4)
S = mg.Solver(p.levels, p.P)
V = torch.from_numpy(np.ascontiguousarray(p.levels[0][0])).cuda()
S.set_matrix_cotan(V, p.mass_coeff, p.lap_coeff)
F = torch.from_numpy(np.ascontiguousarray(p.rhs)).cuda()
B3 = torch.zeros_like(F)
S.apply_mass(F, B3)
for k in (1, 2, 3, 4):
    B = B3[:, :min(k, 3)].contiguous() if k <= 3 else torch.cat([B3, B3[:, :1]], 1).contiguous()
    for rep in range(2):
        X = torch.zeros_like(B)
        mg.mg_set_profiling(S.ctx, True)
        mg.mg_get_profile(S.ctx)
        S.solve(B, X, rel_tol=0.0, max_cycles=3)
        torch.cuda.synchronize()
        prof = mg.mg_get_profile(S.ctx)
        mg.mg_set_profiling(S.ctx, False)
    gs = {l: round(ms / 3, 4) for l, (ms, n) in prof["gs_sweep"].items()}
    rr = {l: round(ms / 3, 4) for l, (ms, n) in prof["residual_restrict"].items()}
    print("k", k, "gs/cycle", gs, "rr/cycle", rr, "norm", round(prof["resnorm"][0][0] / 3, 4), flush=True)
