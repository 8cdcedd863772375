"""Table II-style run: the filter line-search IPM (paper_2403_15913_b200/ipm.py) on the
distillation NLP to tol 1e-6 with the libckkt HyKKT solve; reports iterations, the setup
("init": symbolic analysis + device allocation) and the summed linear-solve time (inertia-corrected
refactor + solve, synchronised wall time per call), next to the whole IPM wall time (which includes
the numpy model evaluation standing in for ExaModels AD).
usage: python tools/ipm_table2.py [N ...]  -> one JSON line per N"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from inputs import distillation as dist  # noqa: E402
from paper_2403_15913_b200 import ipm  # noqa: E402


class TimedKKT(ipm.GpuKKT):
    def __init__(self, *a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        super().__init__(*a, **k)
        torch.cuda.synchronize()
        self.init_s = time.perf_counter() - t
        self.lin_s = 0.0

    def _timed(self, f, *a):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = f(*a)
        torch.cuda.synchronize()
        self.lin_s += time.perf_counter() - t
        return out

    def refactor(self, *a):
        return self._timed(super().refactor, *a)

    def solve(self, *a):
        return self._timed(super().solve, *a)


def main():
    Ns = [int(x) for x in sys.argv[1:]] or [1000, 5000, 50000]
    for N in Ns:
        t0 = time.perf_counter()
        nlp = dist.NLP(dist.Instance(N))
        gen_s = time.perf_counter() - t0
        p = nlp.pat
        kkt = TimedKKT(nlp.n, nlp.m, p.w_row, p.w_col, p.j_rowptr, p.j_col, leaf=1072 if N >= 1000 else 64)
        t1 = time.perf_counter()
        res = ipm.solve_nlp(nlp, kkt, max_iter=200)
        ipm_s = time.perf_counter() - t1
        print(json.dumps({
            "N": N, "n": nlp.n, "m": nlp.m, "status": res.status, "iterations": res.iterations,
            "objective": res.objective, "kkt_error": res.kkt_error,
            "init_s": kkt.init_s, "linsolve_s": kkt.lin_s, "ipm_wall_s": ipm_s, "gen_s": gen_s,
            "linsolve_ms_per_iter": 1e3 * kkt.lin_s / max(res.iterations, 1),
            "delta_x": [h["delta_x"] for h in res.history], "k_cg": [h["k_cg"] for h in res.history],
            "ls": [h["ls"] for h in res.history],
            "note": "strategy HyKKT gamma=1e7; model evaluation in numpy on the host (not timed as linsolve)"}),
            flush=True)


if __name__ == "__main__":
    main()
