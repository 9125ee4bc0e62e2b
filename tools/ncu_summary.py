"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel name: launches, total time, share of the total, mean time.
The last `--tail N` launches only (e.g. the timed step), else all.

    python tools/ncu_summary.py gpurun_out/.../launches.csv [--tail N] [--skip-torch]
"""
import argparse
import collections
import csv
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--tail", type=int, default=0)
    ap.add_argument("--skip-torch", action="store_true")
    a = ap.parse_args()
    rows = []
    with open(a.csv) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        if a.skip_torch and name.startswith("void at::"):
            continue
        t = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)   # -> us
        short = re.sub(r"\(.*$", "", name).replace("mg::<unnamed>::", "").replace("void ", "")
        rows.append((short, t))
    if a.tail:
        rows = rows[-a.tail:]
    tot = sum(t for _, t in rows)
    agg = collections.OrderedDict()
    for n, t in rows:
        c, s = agg.get(n, (0, 0.0))
        agg[n] = (c + 1, s + t)
    print(f"{len(rows)} launches, {tot:.1f} us total (cold-cache, serialised)")
    print(f"{'kernel':40s} {'launches':>8s} {'total_us':>10s} {'share':>7s} {'mean_us':>9s}")
    for n, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n[:40]:40s} {c:8d} {s:10.1f} {100 * s / tot:6.2f}% {s / c:9.2f}")


if __name__ == "__main__":
    main()
