"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel name, the number
of launches, total and mean device time, and the share of the total (cold-cache, serialised)."""
import collections
import csv
import sys


def main(path, skip_names=("reduce", "copy_in", "copy_out")):
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1e-6)
        rows.append((name, v * scale))
    agg = collections.OrderedDict()
    for name, ms in rows:
        short = name.split("(")[0].replace("void ", "")
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += ms
    total = sum(a[1] for a in agg.values())
    print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'mean ms':>9s} {'share':>6s}")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:70]:70s} {n:8d} {ms:10.3f} {ms / n:9.4f} {100 * ms / total:5.1f}%")
    print(f"{'total':70s} {sum(a[0] for a in agg.values()):8d} {total:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
