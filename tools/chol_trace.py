"""Phase timeline of the coarsest factor (k_chol_grid, CTA 0's globaltimer
stamps) in an experiment build: MG_NVCC_DEFINES=-DMG_CHOL_TRACE.
    python tools/chol_trace.py [config]"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import meshgen
from paper_2104_13755_b200 import mg
p = meshgen.make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
S = mg.Solver(p.levels, p.P)
V = torch.from_numpy(np.ascontiguousarray(p.levels[0][0])).cuda()
for _ in range(3):
    S.set_matrix_cotan(V, p.mass_coeff, p.lap_coeff)
