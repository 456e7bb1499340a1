"""Markdown summary of one ncu `--set full` capture for profiles/.

    python tools/ncu_summary.py gpurun_out/brick_r01.ncu-rep "title" [launch index] > profiles/r01_brick_step_ncu.md

Key section metrics, DRAM bytes per launch, and the top source lines by warp
stall samples with their instruction share (needs -lineinfo builds and
--import-source on).
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "No Eligible", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Theoretical Occupancy",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Block Limit Registers", "Block Limit Shared Mem", "Grid Size",
        "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
       "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum"]


LAUNCH = []  # --launch-skip i --launch-count 1 (a report holding several kernels)


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *LAUNCH, *args], capture_output=True, text=True).stdout


def main():
    rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
    if len(sys.argv) > 3:
        LAUNCH[:] = ["--launch-skip", sys.argv[3], "--launch-count", "1"]
    out = [f"# {title}", "", f"Source: `{rep}` (ncu --set full --clock-control none --import-source on).", ""]
    det = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    kname = det[1][4] if len(det) > 1 else "?"
    out += [f"Kernel: `{kname}`", "", "| metric | value | unit |", "|---|---|---|"]
    seen = set()
    for r in det[1:]:
        if len(r) > 14 and r[12] in KEYS and r[12] not in seen:
            seen.add(r[12])
            out.append(f"| {r[12]} | {r[14]} | {r[13]} |")
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    if len(raw) > 2:
        h, units, v = raw[0], raw[1], raw[2]
        out += ["", "| raw metric | value | unit |", "|---|---|---|"]
        for k in RAW:
            if k in h:
                out.append(f"| {k} | {v[h.index(k)]} | {units[h.index(k)]} |")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    fname, header, agg = "?", None, []
    for r in src:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            header = r
            continue
        if header and r[0].isdigit() and len(r) == len(header):
            d = {header[i]: r[i] for i in range(len(header))}
            try:
                s = int(d["Warp Stall Sampling (All Samples)"] or 0)
                n = int(d["Instructions Executed"] or 0)
            except ValueError:
                continue
            st = sorted(((k[6:], int(x)) for k, x in d.items()
                         if k.startswith("stall_") and "Not Issued" not in k and x.isdigit() and int(x) > 0),
                        key=lambda kv: -kv[1])[:3]
            agg.append((s, n, fname, int(r[0]), r[1].strip()[:60], st))
    ts = sum(a[0] for a in agg) or 1
    ti = sum(a[1] for a in agg) or 1
    out += ["", f"Top source lines by warp-stall samples (total {ts} samples, {ti} warp instructions):", "",
            "| stall % | instr % | line | source | top stalls |", "|---|---|---|---|---|"]
    for s, n, f, ln, code, st in sorted(agg, key=lambda a: -a[0])[:25]:
        code = code.replace("|", "\\|")
        out.append(f"| {100 * s / ts:.1f} | {100 * n / ti:.1f} | {f}:{ln} | `{code}` | "
                   + ", ".join(f"{k} {x}" for k, x in st) + " |")
    print("\n".join(out))


if __name__ == "__main__":
    main()
