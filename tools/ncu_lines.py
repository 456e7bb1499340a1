"""Aggregate an ncu `--page source --print-source cuda,sass --csv` export per
CUDA source line: warp-stall samples, instructions executed, top stall reasons.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import csv
import os
import sys

SORTI = os.environ.get("NCU_SORT") == "inst"  # sort by instructions executed


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    fname, header = "?", None
    agg = []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            header = r
            continue
        if header and r[0].isdigit():
            if len(r) != len(header):
                continue  # a source line whose text broke the CSV quoting
            d2 = {header[i]: r[i] for i in range(len(header))}
            try:
                samp = int(d2.get("Warp Stall Sampling (All Samples)", "0") or 0)
                ins = int(d2.get("Instructions Executed", "0") or 0)
            except ValueError:
                continue
            stalls = {k: int(v) for k, v in d2.items() if k.startswith("stall_") and "Not Issued" not in k
                      and v.isdigit() and int(v) > 0}
            agg.append((samp, ins, fname, int(r[0]), r[1][:70], stalls))
    tot_s = sum(a[0] for a in agg) or 1
    tot_i = sum(a[1] for a in agg) or 1
    print(f"total samples {tot_s}, instructions executed (warp) {tot_i}")
    for samp, ins, f, ln, src, st in sorted(agg, key=lambda a: -(a[1] if SORTI else a[0]))[:top]:
        ss = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"{100*samp/tot_s:5.1f}% {100*ins/tot_i:5.1f}%i {f}:{ln:<5} {src:<70} "
              + " ".join(f"{k[6:]}={v}" for k, v in ss))


if __name__ == "__main__":
    main()
