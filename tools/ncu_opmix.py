"""Dynamic opcode mix and stall reasons of one kernel capture (tools only):
python tools/ncu_opmix.py report.ncu-rep [units]  -> instructions per unit (e.g. warp-rows) by opcode,
stall samples by reason, the costliest source lines (needs --import-source / -lineinfo)."""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]


def n(r, c):
    try:
        return float(r[idx[c]])
    except (KeyError, ValueError):
        return 0.0


tot = sum(n(r, "Instructions Executed") for r in data)
print(f"instructions {tot:.4g}  per unit {tot / units:.1f}")
ops = collections.Counter()
for r in data:
    src = re.sub(r"^@!?U?P\w+\s+", "", r[idx["Source"]].strip())
    ops[src.split()[0] if src else "?"] += n(r, "Instructions Executed")
print(" ".join(f"{k}={v / units:.1f}" for k, v in ops.most_common(40)))
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
st = collections.Counter()
for r in data:
    for c in stall_cols:
        st[c[6:]] += n(r, c)
S = sum(st.values()) or 1
print("stalls", ", ".join(f"{k} {100 * v / S:.1f}%" for k, v in st.most_common(10)))
