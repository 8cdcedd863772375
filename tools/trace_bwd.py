import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
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
for r in range(3):
    L.ckkt_debug_trace_bwd(ctx.h, ts.ctypes.data_as(ctypes.c_void_p))
ts = ts.reshape(ns, 4).astype(np.float64)
t0 = ts[:, 0][ts[:, 0] > 0].min()
tick, wake, end = (ts[:, 0] - t0) / 1e3, (ts[:, 1] - t0) / 1e3, (ts[:, 2] - t0) / 1e3
sf = get(ctx, 3, np.int32); srp = get(ctx, 4, np.int64); chp = get(ctx, 9, np.int32); chl = get(ctx, 10, np.int32)
par = -np.ones(ns, int)
for s in range(ns):
    for c in chl[chp[s]:chp[s + 1]]: par[c] = s
print('total us', end.max(), 'mean proc us', np.mean(end - wake), 'max proc', np.max(end - wake))
# critical path: follow latest-ending leaf upwards
s = int(np.argmax(end))
chain = []
while s >= 0:
    chain.append(s); s = par[s]
print('chain len', len(chain))
for s in chain[::-1][:40]:
    w = sf[s + 1] - sf[s]; m = srp[s + 1] - srp[s]
    print(f"s={s:6d} w={w:3d} m={m:4d} tick={tick[s]:8.1f} wake={wake[s]:8.1f} end={end[s]:8.1f} proc={end[s]-wake[s]:6.1f} waitpar={wake[s] - (end[par[s]] if par[s] >= 0 else 0):7.1f} warp={int(ts[s,3])}")
