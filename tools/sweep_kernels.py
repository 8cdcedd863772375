"""Per-kernel durations of one forward + backward sweep at size N (run under ncu --metrics
gpu__time_duration.sum; with CKKT_NOWAIT=1 the dependency waits are skipped: throughput-only timing).
Usage: python tools/sweep_kernels.py N"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import distillation as dist  # noqa: E402
from paper_2403_15913_b200 import ckkt  # noqa: E402

N = int(sys.argv[1])
cache = f"/tmp/ckkt_iter_{N}.npz"
pat = dist.build_pattern(N)
if os.path.exists(cache):
    z = np.load(cache)
    w_val, j_val, sig = z["w"], z["j"], z["s"]
else:
    it = dist.Instance(N).iterate(9, 1.5e-4)
    w_val, j_val, sig = it.w_val, it.j_val, it.sigma_x
    np.savez(cache, w=w_val, j=j_val, s=sig)
L = ckkt.lib()
L.ckkt_debug_time.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
dev = torch.device("cuda:0")
ctx = ckkt.Context(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=1072, device=0,
                   stream=torch.cuda.current_stream().cuda_stream)
v = [torch.as_tensor(a, device=dev) for a in (w_val, j_val, sig)]
ctx.refactor(v[0], v[1], None, v[2])
torch.cuda.synchronize()
out = np.zeros(3)
L.ckkt_debug_time(ctx.h, 3, out.ctypes.data_as(ctypes.c_void_p))
print("fwd %.3f ms bwd %.3f ms" % (out[0], out[1]))
