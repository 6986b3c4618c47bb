#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X` launch
list per kernel (launches, total/mean us, share of all launches).

usage: python tools/launch_summary.py launches.csv "title" > summary.md
"""
import collections
import csv
import sys


def main():
    path, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"][:50]
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        tot[k] += float(r["Metric Value"].replace(",", "")) * scale
        cnt[k] += 1
    all_us = sum(tot.values())
    print(f"# ncu launch list: {title}\n")
    print("gpu__time_duration.sum per kernel (cold-cache, serialised, `--clock-control none`); share of all launches.\n")
    print("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
    for k, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| {k} | {cnt[k]} | {t:.1f} | {t / cnt[k]:.1f} | {t / all_us:.3f} |")


if __name__ == "__main__":
    main()
