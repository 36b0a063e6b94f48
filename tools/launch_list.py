"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
bench.py into the per-iteration table kept under profiles/: the launches
between the last two L2-flush kernels are one timed ADMM iteration.
usage: python tools/launch_list.py launches.csv [title]"""
import csv, io, sys
from collections import OrderedDict

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else path
lines = [l for l in open(path) if not l.startswith("==")]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
seq = []
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"])
    unit = r.get("Metric Unit", "ns")
    us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v if unit in ("us", "usecond") else v / 1e3
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    seq.append((name, us))
flush = [i for i, (n, _) in enumerate(seq) if "k_flush" in n]
it = seq[flush[-2] + 1:flush[-1]] if len(flush) >= 2 else seq
tot = OrderedDict()
for n, us in it:
    c, t = tot.get(n, (0, 0.0))
    tot[n] = (c + 1, t + us)
s = sum(t for _, t in tot.values())
print(f"# {title}")
print(f"# raw CSV: {len(seq)} launches captured; one timed ADMM iteration between two L2 flushes")
print("# per-launch times are cold-cache and serialised by ncu: compare SHARES with bench.py\n")
print(f"{'kernel':40s} {'launches':>8s} {'total us':>10s} {'share':>7s}")
for n, (c, t) in tot.items():
    print(f"{n[:40]:40s} {c:8d} {t:10.2f} {100 * t / s:6.1f}%")
print(f"{'total':40s} {sum(c for c, _ in tot.values()):8d} {s:10.2f}\n")
print("per-launch sequence:")
for n, us in it:
    print(f"  {n[:40]:40s} {us:8.2f} us")
