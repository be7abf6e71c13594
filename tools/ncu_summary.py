"""Summarises an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, total, mean, share."""
import collections
import csv
import sys


def main(path, steps=None):
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    agg, tot = collections.OrderedDict(), 0.0
    for row in csv.DictReader(lines):
        name = row["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(row["Metric Value"].replace(",", ""))
        u = row["Metric Unit"]
        v = v / 1e3 if u == "ns" else (v * 1e3 if u == "ms" else v)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:42s} n={c:4d} total={t:9.1f}us avg={t / c:8.1f}us share={100 * t / tot:5.1f}%")
    print(f"total {tot:.1f} us over {sum(c for c, _ in agg.values())} launches" + (f" = {tot / steps:.1f} us/step" if steps else ""))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
