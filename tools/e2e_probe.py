"""Host-timed breakdown of the e2e step (bench.py Workload.step_host) per API
call, to see where the host<->device path spends its time.

    python tools/e2e_probe.py --config 5
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--steps", type=int, default=4)
    args = ap.parse_args()
    import torch
    import bench
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        W = bench.Workload(args.config, 0, stream)
        W.step()
        torch.cuda.synchronize()
        S, p = W.S, W.p
        for it in range(args.steps):
            t = [time.perf_counter()]
            src = W.hXcur if p.rhs_kind == "mcf" else W.hV
            S.set_matrix_cotan(src, p.mass_coeff, p.lap_coeff)
            torch.cuda.synchronize(); t.append(time.perf_counter())
            if p.rhs_kind == "mcf":
                S.apply_mass(W.hXcur, W.B)
            elif W.hF is not None:
                S.apply_mass(W.hF, W.B)
            torch.cuda.synchronize(); t.append(time.perf_counter())
            if p.rhs_kind == "mcf":
                W.hX.copy_(W.hXcur)
            t.append(time.perf_counter())
            rc, cyc = W.mg.mg_solve(S.ctx, W.k, W.B, W.hX, W.rel_tol, W.max_cycles)
            torch.cuda.synchronize(); t.append(time.perf_counter())
            if p.rhs_kind == "mcf":
                W.hXcur.copy_(W.hX)
            t.append(time.perf_counter())
            d = [round((b - a) * 1e3, 3) for a, b in zip(t, t[1:])]
            print(f"step {it}: set_matrix_cotan {d[0]} ms, apply_mass {d[1]}, host copy {d[2]}, solve {d[3]} "
                  f"({cyc} cycles), host copy {d[4]}; total {round((t[-1] - t[0]) * 1e3, 3)}")
        t0 = time.perf_counter()
        for _ in range(3):
            W.step()
        torch.cuda.synchronize()
        print("device step (host-timed)", round((time.perf_counter() - t0) / 3 * 1e3, 3), "ms")


if __name__ == "__main__":
    main()
