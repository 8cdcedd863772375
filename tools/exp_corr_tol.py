"""Experiment: the correction passes' CG tolerance (cg_rtol_corr, reading R6) at the default ref_tol; mean
IPM-iteration time (refactor + solve, CUDA events) over all 18 positions of bench.py's trajectory at size N.
Usage: python tools/exp_corr_tol.py N [tol ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2403_15913_b200 import ckkt  # noqa: E402

N = int(sys.argv[1])
tols = [float(a) for a in sys.argv[2:]] or [1e-6, 1e-5, 1e-4]
dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
data = bench.build_inputs(N, [0], dev)
pat, n, m = data["pat"], data["n"], data["m"]
T = data["w"].shape[0]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
dx = torch.empty((1, n), dtype=torch.float64, device=dev)
dy = torch.empty((1, m), dtype=torch.float64, device=dev)
for tol in tols:
    ctx = ckkt.Context(n, m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=1072,
                       device=0, stream=st.cuda_stream, cg_rtol_corr=tol)
    tot, nref, kct, worst = 0.0, [], [], 0.0
    for k in range(T):
        args = (data["w"][k], data["j"][k], None, data["sig"][k], None, None, None, None)
        ctx.refactor(*args)
        rc, info = ctx.solve(data["r1"][k], None, data["ra"][k], None, dx, None, dy, None, want_info=True)
        ev[0].record(st)
        ctx.refactor(*args)
        ctx.solve(data["r1"][k], None, data["ra"][k], None, dx, None, dy, None, want_info=False)
        ev[1].record(st)
        torch.cuda.synchronize()
        tot += ev[0].elapsed_time(ev[1])
        nref.append(info[0]["n_ref"])
        kct.append(info[0]["k_cg_total"])
        worst = max(worst, info[0]["rel_res"])
    print(f"cg_rtol_corr {tol:.0e}: mean {tot / T:6.2f} ms  n_ref mean {sum(nref) / T:.2f} {nref}  k_cg_total "
          f"{kct}  worst omega {worst:.1e}", flush=True)
    ctx.close()
