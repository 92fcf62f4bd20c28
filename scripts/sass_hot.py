"""Print SASS lines of an ncu source-page CSV with their warp-stall samples (diagnostics).
usage: sass_hot.py src.csv [pattern-anchor] [before] [after]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
body = [r for r in rows[2:] if len(r) == len(hdr)]
anchor = sys.argv[2] if len(sys.argv) > 2 else 'SHFL'
b, a = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (40, 40)
tot = sum(int(r[ix['Warp Stall Sampling (All Samples)']] or 0) for r in body)
print('total samples', tot)
hits = [i for i, r in enumerate(body) if anchor in r[ix['Source']]]
if not hits: sys.exit('anchor not found')
lo, hi = max(0, hits[0] - b), min(len(body), hits[-1] + a)
for r in body[lo:hi]:
    s = int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
    top = sorted(((int(r[ix[h]] or 0), h[6:]) for h in reasons), reverse=True)[:2]
    tops = ' '.join(f'{h}:{v}' for v, h in top if v)
    print(f"{r[ix['Address']][-5:]} {s:6d} {r[ix['Instructions Executed']]:>9} {r[ix['Source']].strip()[:70]:70s} {tops}")
