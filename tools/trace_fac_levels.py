"""Factor timeline by tree height at C3 (debug trace build of k_factor_persist): per height, the number
of traced supernodes, first wake / last end (us from the first ticket) and the summed processing time.
Usage: python tools/trace_fac_levels.py N leaf"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ['CKKT_TRACE_FACTOR'] = '1'
from inputs import distillation as dist
from paper_2403_15913_b200 import ckkt
L = ckkt.lib()
L.ckkt_debug_get.restype = ctypes.c_int64
L.ckkt_debug_get.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]


def get(ctx, what, dt):
    cnt = L.ckkt_debug_get(ctx.h, what, None)
    a = np.empty(cnt, dt)
    L.ckkt_debug_get(ctx.h, what, a.ctypes.data_as(ctypes.c_void_p))
    return a


N, leaf = int(sys.argv[1]), int(sys.argv[2])
inst = dist.Instance(N)
it = inst.iterate(9, 1.5e-4)
pat = inst.model.pat
dev = torch.device('cuda:0')
ctx = ckkt.Context(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=leaf, device=0,
                   stream=torch.cuda.current_stream().cuda_stream)
vals = [torch.as_tensor(a, device=dev) for a in (it.w_val, it.j_val, it.sigma_x)]
ctx.refactor(vals[0], vals[1], None, vals[2])
torch.cuda.synchronize()
ns = ctx.get_sizes()['n_supernodes']
ts = np.zeros(4 * ns, np.uint64)
for r in range(2):
    L.ckkt_debug_trace_bwd(ctx.h, ts.ctypes.data_as(ctypes.c_void_p))
ts = ts.reshape(ns, 4).astype(np.float64)
done = ts[:, 0] > 0
t0 = ts[done, 0].min()
tick, wake, end = (ts[:, 0] - t0) / 1e3, (ts[:, 1] - t0) / 1e3, (ts[:, 2] - t0) / 1e3
big = ts[:, 3] >= 1000000
sf = get(ctx, 3, np.int32)
srp = get(ctx, 4, np.int64)
chp = get(ctx, 9, np.int32)
chl = get(ctx, 10, np.int32)
w = np.diff(sf)
m = np.diff(srp)
h = np.zeros(ns, int)
for s in range(ns):
    c = chl[chp[s]:chp[s + 1]]
    if len(c):
        h[s] = h[c].max() + 1
print('traced', done.sum(), 'of', ns, 'total us %.1f' % end[done].max())
print(' h   count  big  first_tick  first_wake  last_end   sum_wait   sum_proc  mean_proc  mean_m mean_w')
for lv in range(h.max() + 1):
    sel = done & (h == lv)
    if not sel.any():
        continue
    print('%2d %7d %5d %10.1f %10.1f %10.1f %10.1f %10.1f %8.2f %7.1f %5.1f' % (
        lv, sel.sum(), (sel & big).sum(), tick[sel].min(), wake[sel].min(), end[sel].max(),
        (wake - tick)[sel].sum(), (end - wake)[sel].sum(), (end - wake)[sel].mean(), m[sel].mean(), w[sel].mean()))
