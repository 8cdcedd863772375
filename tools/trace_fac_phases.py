"""Per-phase times of the CTA fronts of one C3 factorization (debug trace build: factor_big stamps
zero+K / panel extend-add / dense / update tiles / panel out / update extend-add).  Usage:
python tools/trace_fac_phases.py N leaf"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ['CKKT_TRACE_FACTOR'] = '1'
from inputs import distillation as dist  # noqa: E402
from paper_2403_15913_b200 import ckkt  # noqa: E402

L = ckkt.lib()
L.ckkt_debug_get.restype = ctypes.c_int64
L.ckkt_debug_get.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]


def get(ctx, what, dt):
    cnt = L.ckkt_debug_get(ctx.h, what, None)
    a = np.empty(cnt, dt)
    L.ckkt_debug_get(ctx.h, what, a.ctypes.data_as(ctypes.c_void_p))
    return a


N, leaf = int(sys.argv[1]), int(sys.argv[2])
it = dist.Instance(N).iterate(9, 1.5e-4)
pat = dist.build_pattern(N)
dev = torch.device('cuda:0')
ctx = ckkt.Context(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=leaf, device=0,
                   stream=torch.cuda.current_stream().cuda_stream)
vals = [torch.as_tensor(a, device=dev) for a in (it.w_val, it.j_val, it.sigma_x)]
ctx.refactor(vals[0], vals[1], None, vals[2])
torch.cuda.synchronize()
ns = ctx.get_sizes()['n_supernodes']
ts = np.zeros(4 * ns, np.uint64)
L.ckkt_debug_trace_bwd(ctx.h, ts.ctypes.data_as(ctypes.c_void_p))
ph = np.fromfile('/tmp/ckkt_phases.bin', dtype=np.uint64).reshape(ns, 8).astype(np.float64)
sf = get(ctx, 3, np.int32)
srp = get(ctx, 4, np.int64)
chp = get(ctx, 9, np.int32)
w = np.diff(sf)
m = np.diff(srp)
nch = np.diff(chp)
sel = ph[:, 0] > 0
d = np.diff(ph[sel][:, :7], axis=1) / 1e3
names = ['zero+K', 'ext-panel', 'dense', 'upd-tiles', 'panel-out', 'ext-U']
pw = (m * w)[sel]
print('CTA fronts traced:', sel.sum())
for lo, hi in [(0, 1024), (1024, 2048), (2048, 4096), (4096, 8192), (8192, 1 << 30)]:
    ss = (pw >= lo) & (pw < hi)
    if ss.any():
        print(f"panel [{lo:5d},{hi if hi < 1e9 else 'inf'}) n={ss.sum():6d} mean m {m[sel][ss].mean():5.1f} w "
              f"{w[sel][ss].mean():4.1f} children {nch[sel][ss].mean():.1f} | " +
              ' '.join(f"{nm}={d[ss, k].mean():6.1f}" for k, nm in enumerate(names)) +
              f" | total {d[ss].sum(axis=1).mean():6.1f} us")
