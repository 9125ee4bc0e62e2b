"""Group the SASS of one kernel in an ncu report into runs of equal execution
count (basic-block-like) and print the heavy ones with their stall samples.
    python tools/ncu_sass_regions.py REPORT.ncu-rep [min_total_Minstr]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# the export repeats a header line per kernel/launch
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1][:80], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = {h: i for i, h in enumerate(r)}
    elif cur is not None and "hdr" in cur:
        cur["rows"].append(r)
for b in blocks:
    h = b["hdr"]
    seg, c = [], None
    tot_i = tot_s = 0
    for k, r in enumerate(b["rows"]):
        try:
            ie = int(r[h["Instructions Executed"]])
            s = int(r[h["Warp Stall Sampling (All Samples)"]])
        except (ValueError, KeyError):
            continue
        tot_i += ie
        tot_s += s
        if c and c[1] == ie:
            c[2] += 1
            c[3] += s
            c[4] += ie
            c[6] = r[h["Source"]].strip()[:60]
        else:
            if c:
                seg.append(c)
            c = [k, ie, 1, s, ie, r[h["Source"]].strip()[:60], ""]
    seg.append(c)
    print(f"=== {b['name']}  instr {tot_i / 1e6:.1f}M  stall samples {tot_s}")
    for k, ie, n, s, ti, src, last in seg:
        if ti / 1e6 >= thr or s > 0.03 * tot_s:
            print(f"  {k:5d} per={ie:9d} n={n:3d} tot={ti / 1e6:7.1f}M stall={100 * s / max(tot_s, 1):5.1f}%  {src} .. {last}")
