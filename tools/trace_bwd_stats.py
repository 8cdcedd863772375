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
done = ts[:, 0] > 0
t0 = ts[done, 0].min()
tick, wake, end = (ts[:, 0] - t0) / 1e3, (ts[:, 1] - t0) / 1e3, (ts[:, 2] - t0) / 1e3
sf = get(ctx, 3, np.int32); srp = get(ctx, 4, np.int64)
w = np.diff(sf); m = np.diff(srp); pw = m * w
proc = end - wake; waitt = wake - tick
print('traced', done.sum(), 'span us', end[done].max())
for lo, hi in [(0, 256), (256, 512), (512, 2000), (2000, 5000), (5000, 1e9)]:
    ss = done & (pw >= lo) & (pw < hi)
    if ss.any():
        print(f"panel [{lo},{hi}) n={ss.sum()} proc mean {proc[ss].mean():.1f} p50 {np.median(proc[ss]):.1f} p90 {np.percentile(proc[ss],90):.1f}  wait mean {waitt[ss].mean():.1f}  warp-time share {proc[ss].sum()/proc[done].sum():.2f}")
kind = ts[:, 3]
for k in [0, 1]:
    ss = done & (kind == k)
    if ss.any():
        print(f"mode {'warp' if k == 0 else 'cta'}: n={ss.sum()} wake range [{wake[ss].min():.0f},{wake[ss].max():.0f}] end max {end[ss].max():.0f} proc sum {proc[ss].sum():.0f} us")
hist, edges = np.histogram(end[done], bins=10)
print('completions per time bin:', list(zip(np.round(edges[:-1]).astype(int), hist)))
chp = get(ctx, 9, np.int32); chl = get(ctx, 10, np.int32)
h = np.zeros(len(w), np.int32)
for s in range(len(w)):  # children precede parents (postorder)
    c = chl[chp[s]:chp[s + 1]]
    if len(c): h[s] = h[c].max() + 1
print('height: count traced, tick min, wake min/max, end max, proc mean, bytes MB')
for lv in range(h.max() + 1):
    ss = done & (h == lv)
    if ss.any():
        st = ss & (kind == 1)
        print(f"  h={lv:2d} n={ss.sum():7d} top {st.sum():6d} tick [{tick[ss].min():6.0f}] wake [{wake[ss].min():6.0f},{wake[ss].max():6.0f}] end {end[ss].max():6.0f} proc {proc[ss].mean():5.1f} MB {pw[ss].sum()*8/1e6:7.1f}" + (f" top: start [{tick[st].min():5.0f},{tick[st].max():5.0f}] end [{end[st].min():5.0f},{end[st].max():5.0f}] wait {(wake-tick)[st].mean():4.1f} proc {proc[st].mean():4.1f}" if st.any() else ""))
