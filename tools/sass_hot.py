"""Top SASS instructions of an ncu source page (--print-source sass --csv) by stall samples / executed."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]
def f(r, k):
    try: return float(r[idx[k]].replace(',', ''))
    except: return 0.0
tot_s = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in data)
tot_i = sum(f(r, 'Instructions Executed') for r in data)
print('total samples', tot_s, 'instructions', tot_i)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for pos, r in enumerate(data):
    r.append(pos)
top = sorted(data, key=lambda r: -f(r, 'Warp Stall Sampling (All Samples)'))[:n]
for r in sorted(top, key=lambda r: r[-1]):
    print(f"{r[-1]:5d} {100*f(r,'Warp Stall Sampling (All Samples)')/tot_s:5.1f}% inst {f(r,'Instructions Executed')/1e6:7.2f}M  {r[idx['Source']].strip()[:90]}")
ops = collections.Counter()
for r in data:
    op = r[idx['Source']].strip().split()[0] if r[idx['Source']].strip() else '?'
    if op.startswith('@'):
        op = r[idx['Source']].strip().split()[1]
    ops[op.split('.')[0]] += f(r, 'Instructions Executed')
print('by opcode:', ', '.join(f'{k}:{v/tot_i*100:.1f}%' for k, v in ops.most_common(20)))
