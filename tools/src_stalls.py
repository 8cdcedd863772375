"""Aggregate an ncu source page (csv, --print-source cuda,sass) per CUDA source line: samples, instructions
and the dominant stall reasons.  Usage: python tools/src_stalls.py page.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
cur = None
last = None
agg = collections.defaultdict(lambda: collections.Counter())
srcs = {}
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if len(r) > 4 and r[0] == 'Line No':
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) // 2:
        continue
    if r[0]:
        last = (cur, int(r[0]))
        srcs[last] = r[1].strip()[:70]
    for i, name in enumerate(hdr):
        if i < 4 or 'Not Issued' in name:
            continue
        if name in ('Warp Stall Sampling (All Samples)', 'Instructions Executed') or name.startswith('stall_'):
            try:
                agg[last][name] += float(r[i].replace(',', '') or 0)
            except ValueError:
                pass
tot = sum(c['Warp Stall Sampling (All Samples)'] for c in agg.values()) or 1
toti = sum(c['Instructions Executed'] for c in agg.values()) or 1
tot_stall = collections.Counter()
for c in agg.values():
    for k, v in c.items():
        if k.startswith('stall_'):
            tot_stall[k] += v
print('samples %.0f  instructions %.3g' % (tot, toti))
print('stalls:', ', '.join('%s %.0f%%' % (k[6:], 100 * v / tot) for k, v in tot_stall.most_common(8)))
for key, c in sorted(agg.items(), key=lambda kv: -kv[1]['Warp Stall Sampling (All Samples)'])[:top]:
    st = [(k[6:], v) for k, v in c.items() if k.startswith('stall_') and v > 0]
    st.sort(key=lambda x: -x[1])
    s = c['Warp Stall Sampling (All Samples)']
    print('%s:%-5d %5.1f%% smp %5.1f%% inst  [%s]  %s' % (key[0], key[1], 100 * s / tot,
          100 * c['Instructions Executed'] / toti, ' '.join('%s:%.0f' % (k, 100 * v / max(s, 1)) for k, v in st[:3]),
          srcs.get(key, '')))
