"""Aggregate an ncu source page (--print-source cuda,sass CSV) per CUDA source line range (diagnostics).
usage: ncu_by_line.py src.csv  name:lo-hi ..."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[2]
ix = {h: i for i, h in enumerate(hdr)}
cols = ['Warp Stall Sampling (All Samples)', 'Instructions Executed', 'L1 Tag Requests Global',
        'L2 Theoretical Sectors Global', 'L1 Wavefronts Shared']
cols = [c for c in cols if c in ix]
ranges = []
for a in sys.argv[2:]:
    name, r = a.split(':'); lo, hi = map(int, r.split('-')); ranges.append((name, lo, hi))
tot = {n: [0] * len(cols) for n, _, _ in ranges}
stall = {n: {} for n, _, _ in ranges}
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
line = None
fname = rows[0][1]
other = [0] * len(cols)
for r in rows[3:]:
    if r and r[0] == 'File Path': fname = r[1]; line = None; continue
    if len(r) != len(hdr) or r[0] == 'Line No': continue
    if r[0]: line = int(r[0]); continue     # CUDA line summary row
    if line is None: continue
    if not fname.endswith(sys.argv[1 + 0].split('@')[-1] if False else 'chain.cu'):
        for j, c in enumerate(cols):
            try: other[j] += float(r[ix[c]] or 0)
            except ValueError: pass
        continue
    for n, lo, hi in ranges:
        if lo <= line <= hi:
            for j, c in enumerate(cols):
                try: tot[n][j] += float(r[ix[c]] or 0)
                except ValueError: pass
            for h in reasons:
                try: stall[n][h] = stall[n].get(h, 0) + float(r[ix[h]] or 0)
                except ValueError: pass
print('%-10s' % 'role' + ''.join('%16s' % c.split('(')[0][:15] for c in cols))
print('%-10s' % 'inlined' + ''.join('%16.0f' % v for v in other))
for n, _, _ in ranges:
    print('%-10s' % n + ''.join('%16.0f' % v for v in tot[n]))
    top = sorted(stall[n].items(), key=lambda kv: -kv[1])[:5]
    print('           stalls:', ', '.join('%s %.0f' % (k[6:], v) for k, v in top))
