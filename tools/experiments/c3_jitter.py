# CPU oracle experiment (C3 fidelity): cylinder tangent jitter 0 / 0.15 / 0.3 h with the current scaffold
import math, sys, numpy as np
sys.path.insert(0, '/root/repo')
import meshgen
from oracle import oracle as O
O.build()
orig = meshgen.cylinder_grid
for jit in (0.0, 0.15, 0.3):
    meshgen.cylinder_grid = lambda nt, nz, h, rng=None, jitter=jit, theta0=0.0: orig(nt, nz, h, rng=rng, jitter=jitter, theta0=theta0)
    for n in (128, 256, 512):
        p = meshgen.make_config(3, grid=(n, n))
        V, F = p.levels[0]
        for lap in (1e-2,):
            A, M = O.assemble(V, F, 1.0, lap)
            B = np.random.default_rng(5).standard_normal((V.shape[0], 1))
            mg = O.MG(p.sizes, p.P, A)
            X, hist, rc = mg.solve(B, rel_tol=1e-10, max_cycles=100)
            rates = hist[1:, 0] / hist[:-1, 0]
            print("jitter", jit, n, "cycles", hist.shape[0]-1, "median rate", round(float(np.median(rates)), 3), flush=True)
