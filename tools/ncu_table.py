"""Per-launch table of an ncu --csv metrics log: python tools/ncu_table.py log.csv"""
import collections, csv, sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
per = collections.OrderedDict()
for r in rows:
    k = (r["ID"], r["Kernel Name"].split("(")[0][:34])
    per.setdefault(k, {})[r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
for (i, name), m in per.items():
    t = m.get("gpu__time_duration.sum")
    us = t[0] / 1e3 if t and t[1] in ("ns", "nsecond") else (t[0] if t else 0)
    rd = m.get("dram__bytes_read.sum", (0, ""))
    wr = m.get("dram__bytes_write.sum", (0, ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = rd[0] * scale.get(rd[1], 1) + wr[0] * scale.get(wr[1], 1)
    gbs = tot / (us * 1e-6) / 1e9 if us else 0
    print(f"{i:>4} {name:34s} {us:8.1f} us  dram {tot/1e6:8.1f} MB  {gbs:7.0f} GB/s")
