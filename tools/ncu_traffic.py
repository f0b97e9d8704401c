"""DRAM bytes and duration per captured launch of every full_*.ncu-rep in a directory
(dram__bytes_read.sum + dram__bytes_write.sum, gpu__time_duration.sum), as JSON."""
import csv, io, json, os, subprocess, sys

d = sys.argv[1]
out = {}
for f in sorted(os.listdir(d)):
    if not (f.startswith("full_") and f.endswith(".ncu-rep")):
        continue
    raw = subprocess.run(["ncu", "-i", os.path.join(d, f), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        m = dict(zip(h, r))
        u = dict(zip(h, units))

        def num(k):
            v = float(m[k].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "usecond": 1,
                     "us": 1, "msecond": 1e3, "ms": 1e3}.get(u.get(k, ""), 1)
            return v * scale
        out[f[:-8]] = {"kernel": m.get("Kernel Name", "")[:80], "dram_bytes": num("dram__bytes_read.sum") + num(
            "dram__bytes_write.sum"), "dram_read": num("dram__bytes_read.sum"), "dram_write": num("dram__bytes_write.sum"),
            "duration_us": num("gpu__time_duration.sum"), "units": {k: u.get(k) for k in (
                "dram__bytes_read.sum", "gpu__time_duration.sum")}}
print(json.dumps(out, indent=1))
