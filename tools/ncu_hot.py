"""Top stalled SASS lines of one kernel in an ncu report: python tools/ncu_hot.py rep.ncu-rep <kernel-index> [n]"""
import csv, io, subprocess, sys

rep, idx = sys.argv[1], int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
heads = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = heads[idx]
end = heads[idx + 1] - 1 if idx + 1 < len(heads) else len(rows)
hdr = rows[h]
data = [r for r in rows[h + 1:end] if len(r) == len(hdr)]
ia, iw = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iw] or 0) for r in data) or 1
print(rows[h - 1][:2])
for r in sorted(data, key=lambda r: -float(r[iw] or 0))[:n]:
    print(f"{float(r[iw]) / tot * 100:5.1f}%  {r[ia][:110]}")
