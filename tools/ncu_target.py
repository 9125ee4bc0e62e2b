"""Short, deterministic driver for ncu captures: one full hot-path step of a
config (GPU assembly -> Galerkin -> Cholesky -> B = M f -> `--cycles` V-cycles).

    python tools/ncu_target.py --config 4 --cycles 2
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--cycles", type=int, default=2)
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    import torch

    import meshgen
    from paper_2104_13755_b200 import mg
    p = meshgen.make_config(args.config)
    S = mg.Solver(p.levels, p.P)
    V = torch.from_numpy(np.ascontiguousarray(p.levels[0][0])).cuda()
    B = torch.zeros((p.n, p.k), dtype=torch.float64, device="cuda")
    F = torch.from_numpy(np.ascontiguousarray(p.rhs if p.rhs_kind != "mcf" else p.levels[0][0])).cuda()
    for _ in range(args.steps):
        S.set_matrix_cotan(V, p.mass_coeff, p.lap_coeff)
        if p.rhs_kind == "direct":
            B.copy_(F)
        else:
            S.apply_mass(F, B)
        X = torch.zeros_like(B)
        rc, cyc, h = S.solve(B, X, rel_tol=0.0, max_cycles=args.cycles)
    torch.cuda.synchronize()
    print("ok", cyc, h[-1].tolist())


if __name__ == "__main__":
    main()
