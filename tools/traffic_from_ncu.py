"""Per-launch DRAM traffic of the sweep / factor kernels from one ncu --set full report -> profiles/traffic.json.
usage: python tools/traffic_from_ncu.py <report.ncu-rep> <source note>"""
import csv, json, subprocess, sys
rep, note = sys.argv[1], sys.argv[2]
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, units = r[0], r[1]
scale = {'byte': 1.0, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'Tbyte': 1e12}
per = {}
for row in r[2:]:
    d = dict(zip(h, row))
    u = dict(zip(h, units))
    name = d['Kernel Name'].split('(')[0].replace('<unnamed>::', '')
    tot = sum(float(d[k].replace(',', '')) * scale[u[k]] for k in ('dram__bytes_read.sum', 'dram__bytes_write.sum'))
    per.setdefault(name, tot)  # first capture of each kernel
fwd = per['k_fwd_tiny'] + per['k_fwd_persist'] + per.get('k_fwd_top', 0.0)
bwd = per.get('k_bwd_top', 0.0) + per['k_bwd_persist'] + per['k_bwd_tiny']
fac = per.get('k_factor_tiny', 0.0) + per['k_factor_persist']
res = {"_source": note, "k_fwd_tiny + k_fwd_persist + k_fwd_top (one forward sweep)": fwd,
       "k_bwd_top + k_bwd_persist + k_bwd_tiny (one backward sweep)": bwd,
       "k_factor_tiny + k_factor_persist (one numeric factorization)": fac,
       "k_condense": next((v for k, v in per.items() if "k_condense" in k), None),
       "_per_kernel": per}
json.dump(res, open('profiles/traffic.json', 'w'), indent=1)
print(json.dumps(res, indent=1))
