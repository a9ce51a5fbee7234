"""Summarise an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv`
capture: per kernel name, mean time and DRAM bytes.  python tools/ncu_mem_summary.py file.csv"""
import collections
import csv
import io
import sys

import numpy as np

t = open(sys.argv[1]).read()
lines = t[t.index('"ID"'):].splitlines()
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for row in csv.DictReader(io.StringIO("\n".join(lines))):
    agg[row["Kernel Name"].split("(")[0][:70]][row["Metric Name"]].append(float(row["Metric Value"].replace(",", "")))
print(f"{'kernel':70s} {'n':>4s} {'us':>8s} {'rd MB':>8s} {'wr MB':>8s} {'GB/s':>7s}")
for k, v in agg.items():
    d = np.mean(v["gpu__time_duration.sum"])
    rd, wr = np.mean(v["dram__bytes_read.sum"]), np.mean(v["dram__bytes_write.sum"])
    print(f"{k:70s} {len(v['gpu__time_duration.sum']):4d} {d / 1000:8.1f} {rd / 1e6:8.1f} {wr / 1e6:8.1f} "
          f"{(rd + wr) / d:7.0f}")
