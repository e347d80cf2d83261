"""Kernel shares from an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python tools/summarize_launches.py LAUNCHES.csv  -> markdown table on stdout"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.defaultdict(lambda: [0, 0.0])
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
             "s": 1e3, "second": 1e3}.get(r[ui], 1e-6)
    t = tot[r[ki][:140]]
    t[0] += 1
    t[1] += float(r[vi].replace(",", "")) * scale
total = sum(v[1] for v in tot.values())
print("| kernel | launches | total ms | share |")
print("|---|---|---|---|")
for k, (n, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"| {k} | {n} | {ms:.2f} | {100 * ms / total:.1f} % |")
print(f"| total | {sum(v[0] for v in tot.values())} | {total:.2f} | |")
