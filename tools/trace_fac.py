import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
os.environ['CKKT_TRACE_FACTOR'] = '1'
from inputs import distillation as dist
from paper_2403_15913_b200 import ckkt
L = ckkt.lib()
L.ckkt_debug_get.restype = ctypes.c_int64; L.ckkt_debug_get.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
def get(ctx, what, dt):
    cnt = L.ckkt_debug_get(ctx.h, what, None); a = np.empty(cnt, dt); L.ckkt_debug_get(ctx.h, what, a.ctypes.data_as(ctypes.c_void_p)); return a
N, leaf = int(sys.argv[1]), int(sys.argv[2])
inst = dist.Instance(N); it = inst.iterate(9, 1.5e-4); pat = inst.model.pat
dev = torch.device('cuda:0')
ctx = ckkt.Context(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=leaf, device=0,
                   stream=torch.cuda.current_stream().cuda_stream)
vals = [torch.as_tensor(a, device=dev) for a in (it.w_val, it.j_val, it.sigma_x)]
ctx.refactor(vals[0], vals[1], None, vals[2]); torch.cuda.synchronize()
ns = ctx.get_sizes()['n_supernodes']
ts = np.zeros(4 * ns, np.uint64)
for r in range(2):
    L.ckkt_debug_trace_bwd(ctx.h, ts.ctypes.data_as(ctypes.c_void_p))
ts = ts.reshape(ns, 4).astype(np.float64)
done = ts[:, 0] > 0
t0 = ts[done, 0].min()
wake, end = (ts[:, 1] - t0) / 1e3, (ts[:, 2] - t0) / 1e3
big = ts[:, 3] >= 1000000
sf = get(ctx, 3, np.int32); srp = get(ctx, 4, np.int64); chp = get(ctx, 9, np.int32); chl = get(ctx, 10, np.int32)
w = np.diff(sf); m = np.diff(srp)
proc = end - wake
print('traced', done.sum(), 'of', ns, 'total us', end[done].max())
for name, sel in [('big', done & big), ('small', done & ~big)]:
    print(name, 'count', sel.sum(), 'sum proc us', proc[sel].sum(), 'mean', proc[sel].mean(), 'max', proc[sel].max())
par = -np.ones(ns, int)
for s in range(ns):
    for c in chl[chp[s]:chp[s + 1]]: par[c] = s
s = int(np.argmax(np.where(done, end, -1)))
chain = []
while s >= 0:
    chain.append(s); s = par[s]
print('chain', len(chain))
for s in chain[::-1]:
    if not done[s]: continue
    print(f"s={s:6d} w={w[s]:3d} m={m[s]:4d} wake={wake[s]:8.1f} end={end[s]:8.1f} proc={proc[s]:7.1f} big={int(big[s])}")
# proc time vs size for big
sel = done & big
for lo, hi in [(0, 2000), (2000, 5000), (5000, 10000), (10000, 1e9)]:
    ss = sel & (m * w >= lo) & (m * w < hi)
    if ss.any(): print(f"panel [{lo},{hi}) n={ss.sum()} mean proc {proc[ss].mean():.1f} us")
ph = np.fromfile('/tmp/ckkt_phases.bin', dtype=np.uint64).reshape(ns, 8).astype(np.float64)
issmall = np.zeros(ns, bool)
sel = (ph[:, 0] > 0) & issmall
d = np.diff(ph[sel][:, :7], axis=1) / 1e3
print('SMALL fronts:', sel.sum(), ' '.join(f"{nm}={d[:, k].mean():.1f}" for k, nm in enumerate(['zero+K', 'ext-panel', 'dense', 'syrk+out', '-', 'ext-U'])))
sel = (ph[:, 0] > 0) & ~issmall
d = np.diff(ph[sel][:, :7], axis=1) / 1e3
names = ['zero+K', 'ext-panel', 'dense', 'syrk', 'panel-out', 'ext-U']
pw = (m * w)[sel]
chol = (ph[sel][:, 7] - ph[sel][:, 2]) / 1e3
for lo, hi in [(0, 2000), (2000, 5000), (5000, 1e9)]:
    ss = (pw >= lo) & (pw < hi)
    print(f"panel [{lo},{hi}) n={ss.sum()} " + ' '.join(f"{nm}={d[ss, k].mean():.1f}" for k, nm in enumerate(names)) + f" (chol+inv {chol[ss].mean():.1f}) mean w {w[sel][ss].mean():.1f}")
