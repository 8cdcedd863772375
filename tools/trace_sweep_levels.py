"""Sweep timeline by tree height (debug trace of the sweep kernels, g_debug_ts): per height the number of
supernodes, how many are in the top set / tiny subtrees, first ticket / last end (us from the first
ticket), summed wait (ticket -> children ready) and processing (children ready -> end) time.
Usage: python tools/trace_sweep_levels.py N leaf fwd|bwd"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if sys.argv[3] == "fwd":
    os.environ["CKKT_TRACE_FWD"] = "1"
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
inst = dist.Instance(N)
it = inst.iterate(9, 1.5e-4)
pat = inst.model.pat
dev = torch.device("cuda:0")
ctx = ckkt.Context(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=leaf, device=0,
                   stream=torch.cuda.current_stream().cuda_stream)
vals = [torch.as_tensor(a, device=dev) for a in (it.w_val, it.j_val, it.sigma_x)]
ctx.refactor(vals[0], vals[1], None, vals[2])
torch.cuda.synchronize()
ns = ctx.get_sizes()["n_supernodes"]
ts = np.zeros(4 * ns, np.uint64)
for r in range(3):
    L.ckkt_debug_trace_bwd(ctx.h, ts.ctypes.data_as(ctypes.c_void_p))
ts = ts.reshape(ns, 4).astype(np.float64)
done = ts[:, 0] > 0
t0 = ts[done, 0].min()
tick, wake, end = (ts[:, 0] - t0) / 1e3, (ts[:, 1] - t0) / 1e3, (ts[:, 2] - t0) / 1e3
tag = ts[:, 3]
top = tag == 1  # the top kernels write 1, the persistent kernels 1e6 + CTA or the warp id, tiny 0
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
print(sys.argv[3], "traced", done.sum(), "of", ns, "total us %.1f" % end[done].max(),
      "top set", top.sum(), "panels MB %.1f" % ((m * w)[top].sum() * 8e-6), "of %.1f" % ((m * w).sum() * 8e-6))
print(" h   count   top first_tick  last_end   sum_wait   sum_proc  mean_proc  mean_m mean_w")
for lv in range(h.max() + 1):
    sel = done & (h == lv)
    if not sel.any():
        continue
    print("%2d %7d %5d %10.1f %10.1f %10.1f %10.1f %8.2f %7.1f %5.1f" % (
        lv, sel.sum(), (sel & top).sum(), tick[sel].min(), end[sel].max(), (wake - tick)[sel].sum(),
        (end - wake)[sel].sum(), (end - wake)[sel].mean(), m[sel].mean(), w[sel].mean()))
for name, sel in (("top", done & top), ("other", done & ~top)):
    if sel.any():
        print("%s: %d supernodes, span %.1f .. %.1f us, mean wait %.2f us, mean proc %.2f us" % (
            name, sel.sum(), tick[sel].min(), end[sel].max(), (wake - tick)[sel].mean(), (end - wake)[sel].mean()))
