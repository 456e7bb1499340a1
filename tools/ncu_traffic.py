"""Update profiles/ncu_traffic.json from ncu --set full captures (units normalised).

    python tools/ncu_traffic.py KEY REP NOTE [KEY REP NOTE ...]
"""
import csv
import io
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6,
         "%": 1.0, "inst": 1.0, "": 1.0}
NAMES = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_sector_hit_rate.pct",
         "smsp__inst_executed.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {}
    for n in NAMES:
        if n in h:
            i = h.index(n)
            d[n] = float(v[i].replace(",", "")) * SCALE.get(u[i], 1.0)
    return d


def main():
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
    J = json.load(open(path))
    a = sys.argv[1:]
    for k in range(0, len(a), 3):
        key, rep, note = a[k:k + 3]
        d = raw(rep)
        rd, wr = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
        J["kernels"][key] = {"duration_us": d["gpu__time_duration.sum"], "dram_bytes_read": rd, "dram_bytes_write": wr,
                             "dram_bytes_per_launch": rd + wr, "l2_hit_pct": d.get("lts__t_sector_hit_rate.pct"),
                             "warp_instructions": d.get("smsp__inst_executed.sum"), "note": note}
        if key.startswith("k_brick_step"):
            J["k_brick_step"] = {"dram_bytes_per_launch": rd + wr, "capture": rep}
    json.dump(J, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
