"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel launches,
total/avg duration and share of kernel time. Usage: python tools/launch_summary.py launches.csv"""
import collections, csv, io, re, sys

rows = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(rows) if l.startswith('"ID"'))
agg = collections.OrderedDict()
for d in csv.DictReader(io.StringIO("\n".join(rows[start:]))):
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"^(void )?(carve_dev::)?", "", d["Kernel Name"])
    name = re.sub(r"\(.*$", "", name).replace("(int)", "").replace("(bool)", "")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[d["Metric Unit"]]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(d["Metric Value"].replace(",", "")) * scale
tot = sum(v[1] for v in agg.values()) or 1.0
print(f"{'kernel':46s} {'launches':>9s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}")
for k, (n, us) in agg.items():
    print(f"{k[:46]:46s} {n:9d} {us:10.1f} {us / n:8.2f} {us / tot:6.3f}")
