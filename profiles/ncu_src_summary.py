"""Summarise an `ncu --page source --csv --print-source sass` export: total
stall samples by reason, and the top-N instructions with their dominant
reasons. Usage: python ncu_src_summary.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
f = lambda r, h: float(r[ix[h]] or 0)
tot = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in data)
print('total samples %.0f, %d SASS lines' % (tot, len(data)))
agg = {h: sum(f(r, h) for r in data) for h in reasons}
print('by reason:', ', '.join('%s %.1f%%' % (h[6:], 100 * v / tot)
                              for h, v in sorted(agg.items(), key=lambda x: -x[1]) if v > 0.005 * tot))
for r in sorted(data, key=lambda r: -f(r, 'Warp Stall Sampling (All Samples)'))[:n]:
    s = f(r, 'Warp Stall Sampling (All Samples)')
    top = sorted(((f(r, h), h[6:]) for h in reasons), reverse=True)[:2]
    print('%5.1f%% %10s  %-60s %s' % (100 * s / tot, r[ix['Instructions Executed']],
                                      r[ix['Source']][:60],
                                      ' '.join('%s:%.0f%%' % (h, 100 * v / max(s, 1)) for v, h in top if v)))
