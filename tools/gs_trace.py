"""Timeline of the GS colour passes inside the production V-cycle graph, from
an experiment build (MG_NVCC_DEFINES=-DMG_GS_TRACE): per CTA the %globaltimer
at kernel entry, after griddepcontrol.wait and at the end of thread 0.  Per
level and kernel: pass period (end of pass c-1 -> end of pass c), the gap from
the previous pass's last CTA end to this pass's first wait release, the
post-wait duration of a CTA (median / max), and how long before the wait
release the CTAs were resident (prologue overlap).

    MG_NVCC_DEFINES=-DMG_GS_TRACE python tools/gs_trace.py [config]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import meshgen
from paper_2104_13755_b200 import build, mg

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p = meshgen.make_config(cfg)
S = mg.Solver(p.levels, p.P)
V = torch.from_numpy(np.ascontiguousarray(p.levels[0][0])).cuda()
S.set_matrix_cotan(V, p.mass_coeff, p.lap_coeff)
k = 3
B = torch.randn(p.n, k, dtype=torch.float64, device="cuda")
X = torch.zeros_like(B)
S.solve(B, X, rel_tol=0.0, max_cycles=3)
lib = ctypes.CDLL(build.LIB)
lib.mg_debug_gs_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
lib.mg_debug_gs_trace(None, 0, 1)
X.zero_()
S.solve(B, X, rel_tol=0.0, max_cycles=1)
cap = 1 << 20
buf = np.zeros((cap, 4), np.uint64)
n = lib.mg_debug_gs_trace(buf.ctypes.data, cap, 1)
buf = buf[:n]
kid = (buf[:, 3] >> np.uint64(56)).astype(np.int64)
key = ((buf[:, 3] >> np.uint64(24)) & np.uint64(0xffffffff)).astype(np.int64)
t0, t1, t2 = (buf[:, i].astype(np.int64) for i in range(3))
base = t0.min()
t0, t1, t2 = t0 - base, t1 - base, t2 - base
names = {1: "k_tile_pipe", 2: "k_tile_pipe_lpr", 3: "k_tile_one_lpr", 4: "k_lpr_sweep"}
# passes: entries of one kernel launch share (kid, key) and are contiguous in time
order = np.argsort(t1, kind="stable")
passes = []
cur = None
for i in order:
    tag = (kid[i], key[i])
    if cur is None or cur["tag"] != tag or t0[i] > cur["end"] + 50000:
        cur = {"tag": tag, "idx": [], "end": 0}
        passes.append(cur)
    cur["idx"].append(i)
    cur["end"] = max(cur["end"], t2[i])
print(f"config {cfg}: {n} CTA records, {len(passes)} passes (one V-cycle); times in us")
print("kernel            ctas  period  prev_end->first_release  release_spread  post_wait med/max  resident_before_release med")
prev_end = None
rows = {}
for ps in passes:
    ix = np.array(ps["idx"])
    s0, s1, s2 = t0[ix], t1[ix], t2[ix]
    end = s2.max()
    rec = dict(ctas=len(ix), period=(end - prev_end) if prev_end is not None else np.nan,
               gap=(s1.min() - prev_end) if prev_end is not None else np.nan, spread=s1.max() - s1.min(),
               pw_med=np.median(s2 - s1), pw_max=(s2 - s1).max(), pre=np.median(s1 - s0))
    prev_end = end
    rows.setdefault((names.get(ps["tag"][0], "?"), rec["ctas"] // 50), []).append(rec)
for (name, _), rs in sorted(rows.items(), key=lambda kv: -kv[1][0]["ctas"]):
    f = lambda key_: np.nanmedian([r[key_] for r in rs]) * 1e-3
    print(f"{name:16s} {int(np.median([r['ctas'] for r in rs])):5d} x{len(rs):4d} {f('period'):7.2f} {f('gap'):10.2f} "
          f"{f('spread'):14.2f} {f('pw_med'):10.2f} /{f('pw_max'):6.2f} {f('pre'):12.2f}")
