"""Experiment: HyKKT refinement target ref_tol vs work and step accuracy at size N (compared with the
ref_tol = 1e-14 step).  Usage: python tools/exp_reftol.py N"""
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
ks = [2, 5, 9, 13, 16]
its = {k: inst.iterate(k, mus[k // 3]) for k in ks}
rng = np.random.default_rng(3000)
r1, ra = rng.standard_normal(pat.n), rng.standard_normal(pat.m)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ref = {}
for tol in (1e-14, 1e-12, 1e-10):
    ctx = ckkt.Context(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=1072,
                       device=0, stream=st.cuda_stream, ref_tol=tol)
    for k in ks:
        it = its[k]
        vals = [T(it.w_val), T(it.j_val), None, T(it.sigma_x)]
        dx = torch.empty(pat.n, dtype=torch.float64, device=dev)
        dy = torch.empty(pat.m, dtype=torch.float64, device=dev)
        ctx.refactor(*vals)
        rc, info = ctx.solve(T(r1), None, T(ra), None, dx, None, dy, None)
        ev[0].record(st)
        for _ in range(3):
            ctx.refactor(*vals)
            ctx.solve(T(r1), None, T(ra), None, dx, None, dy, None, want_info=False)
        ev[1].record(st)
        torch.cuda.synchronize()
        x = np.concatenate([dx.cpu().numpy(), dy.cpu().numpy()])
        if tol == 1e-14:
            ref[k] = x
        e = np.linalg.norm(x - ref[k]) / np.linalg.norm(ref[k])
        print(f"ref_tol {tol:.0e} iterate {k:2d}: {ev[0].elapsed_time(ev[1]) / 3:6.2f} ms n_ref {info[0]['n_ref']} "
              f"k_cg_total {info[0]['k_cg_total']} omega {info[0]['rel_res']:.1e} status {info[0]['status']} "
              f"step diff vs 1e-14: {e:.1e}", flush=True)
    ctx.close()
