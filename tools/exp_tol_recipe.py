"""Experiments (not part of the product): (1) HyKKT first-pass CG tolerance vs total work and accuracy;
(2) Lifted-KKT slack recipes (reading of SURVEY §8(d)) vs refinement passes.  Usage: python tools/exp_tol_recipe.py N"""
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
ks = [2, 9, 16]
its = {k: inst.iterate(k, mus[k // 3]) for k in ks}
rng = np.random.default_rng(3000)
r1 = rng.standard_normal(pat.n)
ra = rng.standard_normal(pat.m)
rb = rng.standard_normal(pat.m)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def run(ctx, k, me, lifted_d=None, reps=3):
    it = its[k]
    vals = [T(it.w_val), T(it.j_val) if me else None, None if me else T(it.j_val), T(it.sigma_x),
            None if me else T(lifted_d)]
    dx = torch.empty(pat.n, dtype=torch.float64, device=dev)
    dy = torch.empty(pat.m, dtype=torch.float64, device=dev) if me else None
    ds = None if me else torch.empty(pat.m, dtype=torch.float64, device=dev)
    dz = None if me else torch.empty(pat.m, dtype=torch.float64, device=dev)
    args = (T(r1), None if me else T(ra), T(ra) if me else None, None if me else T(rb), dx, ds, dy, dz)
    ctx.refactor(*vals)
    rc, info = ctx.solve(*args)
    ev[0].record(st)
    for _ in range(reps):
        ctx.refactor(*vals)
        ctx.solve(*args, want_info=False)
    ev[1].record(st)
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps, info[0], dx.cpu().numpy()


print("== HyKKT first-pass CG tolerance")
ref = {}
for tol in (() if "lifted" in sys.argv else (1e-10, 1e-8, 1e-6, 1e-4)):
    ctx = ckkt.Context(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=1072,
                       device=0, stream=st.cuda_stream, cg_rtol=tol)
    for k in ks:
        ms, info, dx = run(ctx, k, True)
        if tol == 1e-10:
            ref[k] = dx
        err = np.linalg.norm(dx - ref[k]) / np.linalg.norm(ref[k])
        print(f"tol {tol:.0e} iterate {k:2d}: {ms:7.2f} ms  k_cg {info['k_cg']:3d} k_cg_total {info['k_cg_total']:3d} "
              f"n_ref {info['n_ref']} omega0 {info['rel_res_unrefined']:.1e} omega {info['rel_res']:.1e} "
              f"|dx-dx(1e-10)| {err:.1e}", flush=True)
    ctx.close()
print("== Lifted-KKT slack recipes")
tau = dist.TAU
ctx = ckkt.Context(pat.n, 0, pat.m, pat.w_row, pat.w_col, None, None, pat.j_rowptr, pat.j_col, leaf=1072,
                   strategy=ckkt.CKKT_LIFTED, device=0, stream=st.cuda_stream)
for k in ks:
    it = its[k]
    mu = it.mu
    g = inst.model.residual(it.v, inst.xbar0) * inst.row_scale
    recipes = {"uniform(-0.9tau,0.9tau) [current]": it.d_lifted,
               "clip(g, +-0.9tau) [SURVEY 8(d)]": None,
               "s = 0 (D = 2mu/tau^2)": np.full(pat.m, 2 * mu / tau ** 2)}
    s_clip = np.clip(g, -0.9 * tau, 0.9 * tau)
    recipes["clip(g, +-0.9tau) [SURVEY 8(d)]"] = mu / (s_clip + tau) ** 2 + mu / (tau - s_clip) ** 2
    for name, d in recipes.items():
        ms, info, dx = run(ctx, k, False, lifted_d=d)
        print(f"iterate {k:2d} mu {mu:.1e} {name:38s}: {ms:6.2f} ms n_ref {info['n_ref']} omega0 "
              f"{info['rel_res_unrefined']:.1e} omega {info['rel_res']:.1e} status {info['status']}  "
              f"D in [{d.min():.1e}, {d.max():.1e}], frac(|g|>0.9tau) {np.mean(np.abs(g) > 0.9 * tau):.2f}",
              flush=True)
