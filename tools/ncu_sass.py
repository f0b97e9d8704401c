"""Per-SASS-instruction stall breakdown of kernel #ID from an ncu report (source page)."""
import csv, collections, subprocess, sys, io
rep, kid = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else None)
args = ['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass']
if kid is not None: args[3:3] = ['--print-kernel-base', 'function', '-k', kid] if False else []
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur, hdr = [], [], None
for r in rows:
    if r and r[0] == 'Kernel Name':
        if cur: blocks.append((name, hdr, cur))
        name, cur = r[1], []
    elif r and r[0] == 'Address':
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0].startswith('0x'):
        cur.append(r)
if cur: blocks.append((name, hdr, cur))
for name, hdr, data in blocks:
    if kid and kid not in name: continue
    idx = {h: i for i, h in enumerate(hdr)}
    def n(r, c):
        try: return int(r[idx[c]])
        except: return 0
    sc = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
    tot = collections.Counter()
    for r in data:
        for c in sc: tot[c[6:]] += n(r, c)
    S = sum(tot.values())
    print('==', name[:70], 'samples', S, 'instr', sum(n(r, 'Instructions Executed') for r in data))
    print('   stalls:', ', '.join(f'{k} {100*v/S:.0f}%' for k, v in tot.most_common(8)))
    top = sorted(data, key=lambda r: -n(r, 'Warp Stall Sampling (All Samples)'))[:int(sys.argv[3]) if len(sys.argv) > 3 else 20]
    for r in top:
        st = {c[6:]: n(r, c) for c in sc if n(r, c) > 0}
        print('  ', r[idx['Address']][-5:], str(n(r, 'Warp Stall Sampling (All Samples)')).rjust(5), r[idx['Source']][:60].ljust(60), st)
