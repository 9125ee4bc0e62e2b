"""Markdown tables from bench.py JSON lines (one per config): headline numbers,
and a split of one step by phase in the categories of the paper's Table
`profile` (prepare P^T A P / relaxation / transfers /
residual norm / others), from the per-class CUDA-event breakdown.
    python tools/profile_table.py profiles/r02/final/bench_c{1,2,3,4,5}.json"""
import json
import sys


def load(p):
    return json.loads(open(p).read().strip().splitlines()[-1])


def cls(d, name):
    return sum(v["ms"] for v in d["breakdown_ms"].get(name, {}).values())


rows = [(p, load(p)) for p in sys.argv[1:]]
print("| config | V-cycles/s | e2e V-cycles/s | ms/step | cycles/step | V-cycle ms | rebuild ms/step | "
      "L0 GS frac | V-cycle frac | clocks (MHz, reasons) |")
print("|---|---|---|---|---|---|---|---|---|---|")
for p, d in rows:
    c = d["config"]["workload"].split(":")[0]
    clk = d.get("clocks") or {}
    cyc = d["cycles_per_step"]
    print(f"| {c} | {d['value']:.1f} | {d['e2e']['value']:.1f} | {d['ms_per_step']:.3f} | "
          f"{sum(cyc) / len(cyc):.0f} | {d['vcycle_ms']:.4f} | {d['rebuild_ms_per_step']:.3f} | "
          f"{d['roofline']['frac']:.3f} | {d['vcycle_roofline']['frac']:.3f} | "
          f"{clk.get('sm_mhz')}, {','.join(clk.get('reasons', [])) or 'none'} |")
print()
print("Split of one step (ms, % of the profiled step) in the categories of Table `profile`:")
print()
print("| config | P^T A P (Galerkin) | relaxation (GS) | transfers (residual+restriction, prolongation) | "
      "residual norm | coarsest solve | others (assembly, factor, permutations) |")
print("|---|---|---|---|---|---|---|")
for p, d in rows:
    c = d["config"]["workload"].split(":")[0]
    parts = [cls(d, "galerkin"), cls(d, "gs_sweep"), cls(d, "residual_restrict") + cls(d, "prolong"),
             cls(d, "resnorm"), cls(d, "coarse_solve"), cls(d, "assembly") + cls(d, "factor") + cls(d, "permute")]
    tot = sum(parts)
    print(f"| {c} | " + " | ".join(f"{x:.3f} ({100 * x / tot:.0f}%)" for x in parts) + " |")
