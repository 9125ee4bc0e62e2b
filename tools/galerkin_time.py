"""Per-level Galerkin rebuild time of one config (CUDA events through the
library's profiler): python tools/galerkin_time.py [config]"""
import os, sys, json, numpy as np, torch
sys.path.insert(0, os.getcwd())
import meshgen
from paper_2104_13755_b200 import mg
p = meshgen.make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
S = mg.Solver(p.levels, p.P)
V = torch.from_numpy(np.ascontiguousarray(p.levels[0][0])).cuda()
def setm():
    try:
        S.set_matrix_cotan(V, p.mass_coeff, p.lap_coeff)
    except mg.MGError:
        pass    # experiment variants that skip a phase leave A_H indefinite
setm()
mg.mg_set_profiling(S.ctx, ["galerkin"]); mg.mg_get_profile(S.ctx)
for _ in range(5): setm()
pr = mg.mg_get_profile(S.ctx)["galerkin"]
print(os.environ.get("MG_GALT_XMODE", "0"), {l: round(ms / n, 4) for l, (ms, n) in pr.items()}, round(sum(ms / n for ms, n in pr.values()), 4))
