"""Summarise an ncu --set full report: per launch the headline metrics, the
warp-stall breakdown and the hottest SASS regions.
    python tools/ncu_summary2.py REPORT.ncu-rep [launch-id]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else None


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr = raw[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
idx = {h: i for i, h in enumerate(hdr)}
for li, row in enumerate(raw[2:]):
    if want is not None and str(li) != want:
        continue
    print(f"--- launch {li}")
    for k in keys:
        if k in idx:
            print(f"  {k:70s} {row[idx[k]]}")
    st = [(h, row[i]) for h, i in idx.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and
          not h.endswith("_not_issued")]
    tot = sum(float(v or 0) for _, v in st)
    for h, v in sorted(st, key=lambda x: -float(x[1] or 0))[:8]:
        print(f"  stall {h[33:]:40s} {100 * float(v or 0) / tot:5.1f}%")
