"""Idealised schedule of the tile-dataflow GS smoother (mg_vcycle.cu FlowArgs)
on the real level-0 colouring / tiles of a config: G workers (resident CTAs),
worker b runs positions b, b+G, ... of the sequence, one time unit per tile,
a tile starts when the worker is free and every dependency has finished
(+ `lag` units of publication latency).  Prints makespan / ideal per
candidate skew D (D = ngs: colour-major).  CPU only.

    python tools/flow_order_sim.py --config 5 --G 444
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import meshgen  # noqa: E402
from paper_2104_13755_b200 import mg  # noqa: E402


def morton(V):
    lo, hi = V.min(0), V.max(0)
    q = np.minimum(((V - lo) / np.maximum(hi - lo, 1e-300) * 2097151.0).astype(np.uint64), 2097151)
    def spread(x):
        x = x & np.uint64(0x1fffff)
        x = (x | x << np.uint64(32)) & np.uint64(0x1f00000000ffff)
        x = (x | x << np.uint64(16)) & np.uint64(0x1f0000ff0000ff)
        x = (x | x << np.uint64(8)) & np.uint64(0x100f00f00f00f00f)
        x = (x | x << np.uint64(4)) & np.uint64(0x10c30c30c30c30c3)
        x = (x | x << np.uint64(2)) & np.uint64(0x1249249249249249)
        return x
    return spread(q[:, 0]) | spread(q[:, 1]) << np.uint64(1) | spread(q[:, 2]) << np.uint64(2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--G", type=int, default=444)
    ap.add_argument("--T", type=int, default=256)
    ap.add_argument("--lag", type=float, default=0.3)
    ap.add_argument("--rank", default="z", choices=["morton", "z", "band"])
    ap.add_argument("--bands", type=int, default=64)
    a = ap.parse_args()
    p = meshgen.make_config(a.config)
    V, F = p.levels[0]
    n = V.shape[0]
    import scipy.sparse as sp
    I = np.concatenate([F[:, 0], F[:, 1], F[:, 2], F[:, 1], F[:, 2], F[:, 0], np.arange(n)])
    J = np.concatenate([F[:, 1], F[:, 2], F[:, 0], F[:, 0], F[:, 1], F[:, 2], np.arange(n)])
    A = sp.csr_matrix((np.ones(len(I)), (I, J)), shape=(n, n))
    A.sum_duplicates()
    A.sort_indices()
    col, nc = mg.mg_util_greedy_colouring(A.indptr.astype(np.int32), A.indices.astype(np.int32))
    key = morton(V)
    if a.rank == "band":   # rows of a colour by (height band, Morton)
        z = V[:, 2]
        band = np.minimum(((z - z.min()) / (z.max() - z.min()) * a.bands).astype(np.int64), a.bands - 1)
        perm = np.lexsort((np.arange(n), key, band, col))
    else:
        perm = np.lexsort((np.arange(n), key, col))
    iperm = np.empty(n, np.int64)
    iperm[perm] = np.arange(n)
    co = np.bincount(col, minlength=nc)
    print(f"n {n} colours {nc} sizes {co.tolist()}")
    # colour tiles (internal order)
    tiles, tcol = [], []
    off = 0
    for c in range(nc):
        for r0 in range(off, off + co[c], a.T):
            tiles.append((r0, min(a.T, off + co[c] - r0)))
            tcol.append(c)
        off += co[c]
    ngs = len(tiles)
    tcol = np.array(tcol)
    tile_of = np.empty(n, np.int64)
    for t, (r0, nr) in enumerate(tiles):
        tile_of[r0:r0 + nr] = t
    Ai = A[perm][:, perm].tocsr()
    deps = []
    for t, (r0, nr) in enumerate(tiles):
        cols = Ai.indices[Ai.indptr[r0]:Ai.indptr[r0 + nr]]
        deps.append(np.unique(np.concatenate([[t], tile_of[cols]])))
    if a.rank == "morton":
        mid = np.array([key[perm[r0 + nr // 2]] for r0, nr in tiles])
    elif a.rank == "band":   # normalised position inside the tile's colour
        cstart = np.concatenate([[0], np.cumsum(co)])
        mid = np.array([(r0 + nr / 2 - cstart[tcol[t]]) / co[tcol[t]] for t, (r0, nr) in enumerate(tiles)])
    else:   # sweep line: height of the tile's centroid
        mid = np.array([V[perm[r0:r0 + nr], 2].mean() for r0, nr in tiles])
    rank = np.empty(ngs, np.int64)
    rank[np.argsort(mid, kind="stable")] = np.arange(ngs)
    G = a.G
    print(f"ngs {ngs}  G {G}  ideal (2 sweeps) {2 * ngs / G:.1f}")
    for D in [ngs, ngs // 2, ngs // 4, ngs // 8, ngs // 16, ngs // 32, ngs // 64]:
        k = rank + tcol * D
        seq = np.lexsort((tcol, k))
        pos = np.empty(ngs, np.int64)
        pos[seq] = np.arange(ngs)
        # two sweeps
        tot = 2 * ngs
        fin = np.zeros(tot)
        wfree = np.zeros(G)
        dists = []
        for g in range(tot):
            s, q = divmod(g, ngs)
            t = seq[q]
            st = wfree[g % G]
            for nn in deps[t]:
                if tcol[nn] < tcol[t]:
                    gd = s * ngs + pos[nn]
                else:
                    gd = (s - 1) * ngs + pos[nn]
                if gd >= 0:
                    st = max(st, fin[gd] + a.lag)
                    dists.append(g - gd)
            fin[g] = st + 1.0
            wfree[g % G] = fin[g]
        dists = np.array(dists)
        if dists.min() <= 0:
            print(f"D {D:6d}: not topological (min dist {dists.min()})")
            continue
        print(f"D {D:6d}: makespan {fin.max():7.1f}  (ideal {tot / G:6.1f})  min dist {dists.min()}  "
              f"deps < G {np.mean(dists < G) * 100:.2f}%  < 2G {np.mean(dists < 2 * G) * 100:.2f}%")


if __name__ == "__main__":
    main()
