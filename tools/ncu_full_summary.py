"""One line per captured launch of an `ncu --set full` report (key SOL /
occupancy / cache metrics), for profiles/.

    python tools/ncu_full_summary.py gpurun_out/<tag>/full_c4.ncu-rep > profiles/r01/ncu_full_c4_final.txt
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Achieved Occupancy", "Registers Per Thread", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size"]


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    iid, ik, isec, im, iu, iv = (h.index(x) for x in ("ID", "Kernel Name", "Section Name", "Metric Name", "Metric Unit",
                                                       "Metric Value"))
    per = {}
    names = {}
    for r in rows[1:]:
        key = int(r[iid])
        names[key] = r[ik]
        m = r[im]
        if m in KEYS and (m, key) not in per:
            if m == "Memory Throughput" and r[iu] == "%":
                continue
            per[(m, key)] = f"{m}: {r[iv]} {r[iu]}".strip()
    print("# ncu --set full (cold caches; tools/ncu_target.py --config 4 --cycles 1), one line per captured launch")
    for key in sorted(names):
        nm = names[key].split("(")[0].replace("void mg::", "").replace("(anonymous namespace)::", "")
        print(key, nm[:40].ljust(40), " | ".join(per[(m, key)] for m in KEYS if (m, key) in per))


if __name__ == "__main__":
    main()
