"""Refactor (and optionally solve) one C3-sized iterate a few times: a short driver for ncu captures of the
factor / sweep kernels.  Usage: python tools/one_refactor.py N [reps] [solve]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import distillation as dist  # noqa: E402
from paper_2403_15913_b200 import ckkt  # noqa: E402

N = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
solve = len(sys.argv) > 3 and sys.argv[3] == "solve"
inst = dist.Instance(N)
it = inst.iterate(9, 1.5e-4)
pat = inst.model.pat
dev = torch.device("cuda:0")
ctx = ckkt.Context(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=1072, device=0,
                   stream=torch.cuda.current_stream().cuda_stream)
vals = [torch.as_tensor(a, device=dev) for a in (it.w_val, it.j_val, it.sigma_x)]
rng = np.random.default_rng(3000)
r1 = torch.as_tensor(rng.standard_normal(pat.n), device=dev)
r3 = torch.as_tensor(rng.standard_normal(pat.m), device=dev)
dx = torch.empty(pat.n, dtype=torch.float64, device=dev)
dy = torch.empty(pat.m, dtype=torch.float64, device=dev)
for r in range(reps):
    ctx.refactor(vals[0], vals[1], None, vals[2])
    if solve:
        ctx.solve(r1, None, r3, None, dx, None, dy, None)
torch.cuda.synchronize()
print("ok", ctx.get_sizes()["n_supernodes"])
