"""Summarise an ncu report: duration, DRAM, occupancy, top stall reasons, issue stats."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
for row in r[2:]:
    d = dict(zip(h, row))
    print('kernel', d.get('Kernel Name', '')[:60], 'dur(ms)', d.get('gpu__time_duration.sum'))
    for k in ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
              'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
              'smsp__inst_executed.sum', 'launch__registers_per_thread', 'launch__occupancy_limit_registers',
              'lts__t_bytes.sum', 'l1tex__t_bytes.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed']:
        if k in d: print(f'  {k} = {d[k]}')
    vals = []
    for k in h:
        if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued'):
            try: vals.append((float(d[k].replace(',', '')), k.replace('smsp__pcsamp_warps_issue_stalled_', '')))
            except: pass
    tot = sum(v for v, _ in vals) or 1
    print('  stalls:', ' '.join(f'{k}:{100*v/tot:.0f}%' for v, k in sorted(vals, reverse=True)[:8]))
