"""Opcode census of the shipped libtgcu.so cubins (sm_100a SASS).

Counts, per hot kernel, the instructions that show the Blackwell data path:
TMA tile loads/stores (UTMALDG/UTMASTG), bulk copies (UBLKCP), mbarrier
traffic (SYNCS), paired fp32 math (FFMA2/FADD2/FMUL2), fp64 (DFMA), vector
L2 reductions (REDG), shared-memory atomics (ATOMS), cluster barriers
(UCGABAR). Usage: python tools/sass_summary.py [libtgcu.so] > profiles/...md
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2402_14415_b200/libtgcu.so"
OPS = ["UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "SYNCS", "FFMA2", "FADD2", "FMUL2", "FFMA", "DFMA",
       "REDG", "ATOMS", "ATOMG", "SHFL", "BAR.SYNC", "UCGABAR", "LDS", "STS", "LDG", "STG"]
KEEP = ("k_brick_step", "k_eval_brick", "k_eval_direct", "k_qbin", "k_bin_", "k_small_",
        "k_step_finalize", "k_resample", "k_sample_field", "k_render")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    stats = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            stats[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if not m:
            continue
        op = m.group(1)
        stats[cur]["instrs"] += 1
        base = op.split(".")[0]
        for p in OPS:
            if op == p or base == p or (p == "BAR.SYNC" and op.startswith("BAR.SYNC")):
                stats[cur][p] += 1
                break
    names = subprocess.run(["c++filt"], input="\n".join(stats), capture_output=True, text=True).stdout.split("\n")
    print(f"# SASS opcode census of `{LIB}` (cuobjdump -sass; tools/sass_summary.py)\n")
    print("No tcgen05 (UTCMMA) by design: nothing on the path is a contraction (DESIGN §3).\n")
    print("| kernel | instrs | " + " | ".join(OPS) + " |")
    print("|---|---:|" + "---:|" * len(OPS))
    for (raw, c), dm in zip(stats.items(), names):
        if not any(k in dm for k in KEEP):
            continue
        dm = dm.replace("(tgcu::StepArgs)", "").replace("void tgcu::", "")
        print(f"| `{dm[:90]}` | {c['instrs']} | " + " | ".join(str(c[p]) for p in OPS) + " |")


if __name__ == "__main__":
    main()
