"""Summarise an `ncu --csv --metrics ...` launch log: one line per launch
(or, with --group N, the median of every N consecutive launches).
usage: python tools/ncu_csv.py LOG.csv [--skip S] [--group N] [--kernel REGEX]"""
import argparse
import collections
import csv
import re
import statistics

ap = argparse.ArgumentParser()
ap.add_argument("log")
ap.add_argument("--skip", type=int, default=0)
ap.add_argument("--group", type=int, default=1)
ap.add_argument("--kernel", default=None)
a = ap.parse_args()
rows = list(csv.reader(open(a.log)))
h = [x for x in rows if x and x[0] == "ID"][0]
by = collections.OrderedDict()
for x in rows:
    if len(x) == len(h) and x[0] != "ID":
        d = dict(zip(h, x))
        if a.kernel and not re.search(a.kernel, d["Kernel Name"]):
            continue
        e = by.setdefault(d["ID"], {"kernel": d["Kernel Name"][:48]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
launches = list(by.values())[a.skip:]


def fmt(k, v):
    if "bytes" in k:
        return f"{k.split('.')[0].replace('dram__bytes_', 'dram_')}={v / 1e6:.0f}MB"
    if "time_duration" in k:
        return f"t={v / 1e3:.1f}us"
    return f"{k}={v:.4g}"


for i in range(0, len(launches), a.group):
    chunk = launches[i:i + a.group]
    keys = [k for k in chunk[0] if k != "kernel"]
    med = {k: statistics.median(c[k] for c in chunk if k in c) for k in keys}
    print(f"[{i + a.skip}:{i + a.skip + len(chunk)}] {chunk[0]['kernel']:48s} " +
          "  ".join(fmt(k, v) for k, v in med.items()))
