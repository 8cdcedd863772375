"""NEXT-1: iteration counts of the filter line-search IPM with HyKKT (exact KKT system) and
with Lifted-KKT (relaxed problem, tau = 1e-6) through libckkt, tol 1e-6, from the simulated
start of the input recipe.  One JSON line per N.  Usage: python tools/ipm_lifted_vs_hykkt.py N [N ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import distillation as dist  # noqa: E402
from paper_2403_15913_b200 import ipm  # noqa: E402

for N in [int(a) for a in sys.argv[1:]]:
    out = {"N": N}
    nlp = dist.NLP(dist.Instance(N))
    p = nlp.pat
    t = time.time()
    rh = ipm.solve_nlp(nlp, ipm.GpuKKT(nlp.n, nlp.m, p.w_row, p.w_col, p.j_rowptr, p.j_col, leaf=1072), max_iter=300)
    out["hykkt"] = {"status": rh.status, "iterations": rh.iterations, "objective": rh.objective,
                    "kkt_error": rh.kkt_error, "wall_s": time.time() - t}
    lnlp = ipm.LiftedNLP(dist.NLP(dist.Instance(N)))
    t = time.time()
    rl = ipm.solve_nlp(lnlp, ipm.LiftedGpuKKT(lnlp.nv, lnlp.m, p.w_row, p.w_col, p.j_rowptr, p.j_col, leaf=1072),
                       max_iter=300)
    out["lifted"] = {"status": rl.status, "iterations": rl.iterations, "objective": rl.objective,
                     "kkt_error": rl.kkt_error, "wall_s": time.time() - t}
    out["ratio_lifted_over_hykkt"] = rl.iterations / max(rh.iterations, 1)
    print(json.dumps(out), flush=True)
