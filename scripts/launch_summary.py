"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python scripts/launch_summary.py launches.csv "header comment" > profiles/rNN_launches_bench.txt
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    head = sys.argv[2] if len(sys.argv) > 2 else ""
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1000.0 if unit == "ns" else v * 1000.0 if unit == "ms" else v
        rows.append((r["Kernel Name"], us))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for k, us in rows:
        tot[k] += us
        cnt[k] += 1
    total = sum(tot.values())
    if head:
        print("# " + head)
    for k, us in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{us:10.1f} us {100 * us / total:5.1f}% n={cnt[k]:4d} {k[:70]}")
    print(f"total {total:.1f} us")


if __name__ == "__main__":
    main()
