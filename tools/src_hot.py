"""Aggregate an ncu 'cuda,sass' source page (csv) to CUDA source lines: stall samples + instructions."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None; cur_file = None; agg = collections.defaultdict(lambda: [0.0, 0.0, '']); last_line = None
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]; continue
    if len(r) > 4 and r[0] == 'Line No':
        hdr = r; continue
    if hdr is None or len(r) < 8:
        continue
    line, src = r[0], r[1]
    if line:
        last_line = (cur_file, int(line)); agg[last_line][2] = src.strip()[:80]
    key = last_line
    try:
        agg[key][0] += float(r[4].replace(',', '') or 0)
        agg[key][1] += float(r[7].replace(',', '') or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f'samples {tot:.0f} instructions {toti:.3g}')
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f'{k[0]}:{k[1]:5d} {100*v[0]/tot:5.1f}% smp {100*v[1]/toti:5.1f}% inst  {v[2]}')
