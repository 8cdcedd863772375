"""Experiment: the correction passes' CG tolerance (cg_rtol_corr, reading R6) at the default ref_tol; mean
IPM-iteration time over trajectory iterates at size N.  Usage: python tools/exp_corr_tol.py N"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import distillation as dist  # noqa: E402
from paper_2403_15913_b200 import ckkt  # noqa: E402

N = int(sys.argv[1])
inst = dist.Instance(N)
mus = dist.mu_schedule()
pat = inst.model.pat
dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
T = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
ks = [1, 4, 7, 10, 13, 16]
its = {k: inst.iterate(k, mus[k // 3]) for k in ks}
rng = np.random.default_rng(3000)
r1, ra = T(rng.standard_normal(pat.n)), T(rng.standard_normal(pat.m))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for tol in (1e-6, 1e-5, 1e-4, 1e-3, 1e-2):
    ctx = ckkt.Context(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=1072,
                       device=0, stream=st.cuda_stream, cg_rtol_corr=tol)
    tot, nref, kct, worst = 0.0, [], [], 0.0
    for k in ks:
        it = its[k]
        vals = [T(it.w_val), T(it.j_val), None, T(it.sigma_x)]
        dx = torch.empty(pat.n, dtype=torch.float64, device=dev)
        dy = torch.empty(pat.m, dtype=torch.float64, device=dev)
        ctx.refactor(*vals)
        rc, info = ctx.solve(r1, None, ra, None, dx, None, dy, None)
        ev[0].record(st)
        ctx.refactor(*vals)
        ctx.solve(r1, None, ra, None, dx, None, dy, None, want_info=False)
        ev[1].record(st)
        torch.cuda.synchronize()
        tot += ev[0].elapsed_time(ev[1])
        nref.append(info[0]["n_ref"])
        kct.append(info[0]["k_cg_total"])
        worst = max(worst, info[0]["rel_res"])
    print(f"cg_rtol_corr {tol:.0e}: mean {tot / len(ks):6.2f} ms  n_ref {nref}  k_cg_total {kct}  worst omega {worst:.1e}",
          flush=True)
    ctx.close()
