# CPU oracle experiment (C3 fidelity): current (independently jittered) vs nested cylinder scaffold (coarse vertices = even (i, j) fine vertices + the top row), rel. residual 1e-10, cycles and median per-cycle rate
import math, sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import meshgen
from meshgen import cylinder_grid, chart_prolongation
from oracle import oracle as O
O.build()

def nested(nt, nz, rng, height=4.0):
    V, F, th, z = cylinder_grid(nt, nz, height, rng=rng)
    levels=[(V,F)]; Ps=[]
    # index grid of the current level
    ti = np.tile(np.arange(nt), nz); tj = np.repeat(np.arange(nz), nt)
    th_f, z_f, ntf, nzf = th, z, nt, nz
    while th_f.shape[0] > 1000:
        rows = sorted(set(range(0, nzf, 2)) | {nzf - 1})
        ntc, nzc = ntf // 2, len(rows)
        sel = np.array([r * ntf + 2 * i for r in rows for i in range(ntc)])
        th_c, z_c = th_f[sel], z_f[sel]
        Vc = np.stack([np.cos(th_c), np.sin(th_c), z_c], 1)
        ii, jj = np.meshgrid(np.arange(ntc), np.arange(nzc - 1), indexing="xy"); ii=ii.ravel(); jj=jj.ravel()
        v00 = jj*ntc+ii; v10 = jj*ntc+(ii+1)%ntc; v11=(jj+1)*ntc+(ii+1)%ntc; v01=(jj+1)*ntc+ii
        Fc = np.concatenate([np.stack([v00,v10,v11],1), np.stack([v00,v11,v01],1)],0)
        Ps.append(chart_prolongation(np.mod(th_f,2*math.pi), z_f, np.mod(th_c,2*math.pi), z_c, ntc, nzc, Fc))
        levels.append((Vc, Fc)); th_f, z_f, ntf, nzf = th_c, z_c, ntc, nzc
    return levels, Ps

for n in (64, 128, 256, 512):
    rng = np.random.default_rng(1)
    b = None
    for kind in ("current", "nested"):
        if kind == "current":
            p = meshgen.make_config(3, grid=(n, n))
            levels, Ps = p.levels, p.P
        else:
            levels, Ps = nested(n, n, np.random.default_rng(210413755 + 3))
        V, F = levels[0]
        A, M = O.assemble(V, F, 1.0, 1e-2)
        B = np.random.default_rng(5).standard_normal((V.shape[0], 1))
        mg = O.MG([l[0].shape[0] for l in levels], Ps, A)
        X, hist, rc = mg.solve(B, rel_tol=1e-10, max_cycles=100)
        rates = hist[1:, 0] / hist[:-1, 0]
        print(n, kind, [l[0].shape[0] for l in levels], "cycles", hist.shape[0]-1, "median rate", round(float(np.median(rates)), 3), flush=True)
