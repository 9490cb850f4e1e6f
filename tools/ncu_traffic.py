"""Reads an ncu --set full report and records the DRAM traffic of one kernel
per launch into profiles/ncu_traffic.json (bench.py's roofline.traffic).
usage: ncu_traffic.py REPORT.ncu-rep KERNEL_SUBSTRING PER_LAUNCH_ALGORITHMIC_BYTES"""
import csv, io, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, kernel, alg = sys.argv[1], sys.argv[2], int(sys.argv[3])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
out = None
for r in data:
    if kernel not in r[col["Kernel Name"]]:
        continue
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        tot += float(r[col[m]].replace(",", "")) * scale.get(units[col[m]], 1)
    out = {"per_launch_bytes": alg, "dram_bytes": int(tot), "dram_over_algorithmic": round(tot / alg, 4),
           "duration_ns": r[col["gpu__time_duration.sum"]] if "gpu__time_duration.sum" in col else None,
           "kernel": r[col["Kernel Name"]], "source": os.path.relpath(rep, ROOT)}
    break
if out is None:
    sys.exit(f"{kernel} not in {rep}")
p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
d = json.load(open(p)) if os.path.exists(p) else {}
d[kernel] = out
json.dump(d, open(p, "w"), indent=1)
print(json.dumps(out))
