"""Key counters of every kernel in an ncu report: python tools/ncu_summary.py rep.ncu-rep [out.csv]

Writes (or prints) one row per kernel launch: duration, DRAM bytes read/written,
DRAM / L2 / L1 throughput %, tensor-pipe (tcgen05 UTCHMMA) utilisation, SM
clock -- the numbers DESIGN.md section 4 cites."""
import csv, io, subprocess, sys

KEYS = {
    "time_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm_ghz": "sm__cycles_elapsed.avg.per_second",
}
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    row = {"kernel": d["Kernel Name"].split("(")[0][:40], "grid": d.get("launch__grid_size", "")}
    for k, m in KEYS.items():
        v = d.get(m, "")
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            row[k] = ""
            continue
        unit = u.get(m, "")
        if k.endswith("_MB"):
            x = x * {"byte": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1.0, "MB": 1.0, "Gbyte": 1e3, "GB": 1e3}.get(unit, 1.0)
        if k == "time_us":
            x = x * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        row[k] = round(x, 3)
    out.append(row)
w = csv.DictWriter(open(sys.argv[2], "w") if len(sys.argv) > 2 else sys.stdout, fieldnames=list(out[0]))
w.writeheader()
w.writerows(out)
