"""Per-kernel mean duration from an ncu `--metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_table.py launches.csv [skip_first_n_launches]
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    hdr, agg, seen = None, collections.OrderedDict(), 0
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        seen += 1
        if seen <= skip:
            continue
        a = agg.setdefault(d["Kernel Name"][:70], [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(t for _, t in agg.values())
    print("| launches | mean us | total share | kernel |\n|---|---|---|---|")
    for k, (n, t) in agg.items():
        print(f"| {n} | {t / n / 1000:.1f} | {t / tot:.1%} | `{k}` |")


if __name__ == "__main__":
    main()
