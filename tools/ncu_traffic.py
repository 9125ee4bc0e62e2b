"""Write profiles/ncu_traffic.json from an `ncu --set full` report: DRAM bytes
(read + write) per launch of the dominant kernel (level-0 GS colour pass,
k_tile_pipe<3, 0>), which bench.py reports as roofline.traffic.

    python tools/ncu_traffic.py gpurun_out/<tag>/full_c4.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ik = h.index("Kernel Name")
    ir, iw = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = []
    for r in rows[2:]:
        if "k_tile_pipe<3, 0>" in r[ik] or "k_tile_pipe<3, 0, " in r[ik] or "k_tile_pipe<(int)3, (int)0" in r[ik]:
            per.append(float(r[ir].replace(",", "")) * scale[units[ir]] + float(r[iw].replace(",", "")) * scale[units[iw]])
    if not per:
        sys.exit("no k_tile_pipe<3, 0> launch in the report")
    doc = {
        "_about": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from one "
                  "`ncu --set full --clock-control none` capture (%s, tools/ncu_target.py --config 4 --cycles 1). "
                  "ncu flushes the caches before every replayed kernel, so these are COLD-cache numbers: the gathered "
                  "iterate x (84 MB) comes from DRAM instead of L2 as it does inside the timed V-cycle; the "
                  "algorithmic bytes per launch are 69.9 MB (config 4)." % os.path.relpath(rep, ROOT),
        "config4": {"kernel": "k_tile_pipe<3,0,8> (level-0 GS colour pass)", "per_launch_bytes": per,
                    "gs_sweep_level0_bytes_per_launch": sum(per) / len(per)},
    }
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump(doc, f, indent=1)
    print(doc["config4"]["gs_sweep_level0_bytes_per_launch"])


if __name__ == "__main__":
    main()
