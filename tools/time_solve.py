"""Time one triangular-solve pair and one refactor for a distillation config (debug entry point)."""
import ctypes, sys, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from inputs import distillation as dist
from paper_2403_15913_b200 import ckkt
L = ckkt.lib(); L.ckkt_debug_time.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
for arg in sys.argv[1:]:
    N, leaf = [int(x) for x in arg.split(':')]
    inst = dist.Instance(N); it = inst.iterate(9, 1.5e-4); pat = inst.model.pat
    dev = torch.device('cuda:0')
    ctx = ckkt.Context(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=leaf, device=0,
                       stream=torch.cuda.current_stream().cuda_stream)
    vals = [torch.as_tensor(a, device=dev) for a in (it.w_val, it.j_val, it.sigma_x)]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for r in range(3):
        ev[0].record(); ctx.refactor(vals[0], vals[1], None, vals[2]); ev[1].record(); torch.cuda.synchronize()
    fac = ev[0].elapsed_time(ev[1])
    out = np.zeros(3)
    L.ckkt_debug_time(ctx.h, 3, out.ctypes.data_as(ctypes.c_void_p))
    L.ckkt_debug_time(ctx.h, 10, out.ctypes.data_as(ctypes.c_void_p))
    sz = ctx.get_sizes()
    lb = sz['l_storage'] * 8
    print(f"N={N} leaf={leaf} refactor={fac:.3f}ms fwd={out[0]:.3f}ms bwd={out[1]:.3f}ms  L={lb/1e9:.3f}GB  fwd GB/s={lb/out[0]/1e6:.0f} bwd GB/s={lb/out[1]/1e6:.0f} ns={sz['n_supernodes']} levels={sz['n_levels']}", flush=True)
    ctx.close()
