"""Stall breakdown + hottest SASS lines of the single kernel in an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(raw)); h = r[0]; d = dict(zip(h, r[2]))
items = []
for k in h:
    if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued'):
        try: items.append((float(d[k].replace(',', '')), k[33:]))
        except ValueError: pass
tot = sum(v for v, _ in items)
print('stalls:', ', '.join('%s %.1f%%' % (k, 100 * v / tot) for v, k in sorted(items, reverse=True)[:10]))
for k in ('gpu__time_duration.sum', 'sm__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
          'sm__warps_active.avg.pct_of_peak_sustained_active'):
    print(k, d.get(k))
src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(src)); hdr = None; data = []
for x in rows:
    if x and x[0] == 'Address': hdr = x; continue
    if hdr and len(x) == len(hdr) and x[0].startswith('0x'): data.append(x)
idx = {k: i for i, k in enumerate(hdr)}
sc = [k for k in hdr if k.startswith('stall_') and 'Not Issued' not in k]
def n(x, c):
    try: return int(x[idx[c]])
    except ValueError: return 0
t = [(sum(n(x, c) for c in sc), x) for x in data]
S = sum(v for v, _ in t)
for v, x in sorted(t, key=lambda z: -z[0])[:top]:
    det = sorted(((n(x, c), c[6:]) for c in sc), reverse=True)[:2]
    print('%5.2f%%' % (100 * v / S), x[idx['Address']][-5:], x[idx['Source']][:58], det)
