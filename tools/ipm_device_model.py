"""IPM wall time per iteration with the model derivatives on the host (numpy, inputs.distillation.NLP) vs on
the GPU (ipm.DeviceDistillationNLP, ckkt_distillation_eval; NEXT-4 inside NEXT-1).  Same HyKKT solve
(libckkt) in both; prints one JSON line per (N, model).  Usage: python tools/ipm_device_model.py N [N ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from inputs import distillation as dist  # noqa: E402
from paper_2403_15913_b200 import ipm  # noqa: E402

for N in [int(a) for a in sys.argv[1:]] or [1000, 5000]:
    for model in ("host", "device"):
        base = dist.NLP(dist.Instance(N))
        nlp = ipm.DeviceDistillationNLP(base) if model == "device" else base
        p = nlp.pat
        kkt = ipm.GpuKKT(nlp.n, nlp.m, p.w_row, p.w_col, p.j_rowptr, p.j_col, leaf=1072)
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = ipm.solve_nlp(nlp, kkt, max_iter=100)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(json.dumps({"N": N, "model": model, "status": res.status, "iterations": res.iterations,
                          "objective": res.objective, "kkt_error": res.kkt_error, "wall_s": dt,
                          "ms_per_iteration": 1e3 * dt / max(res.iterations, 1)}), flush=True)
