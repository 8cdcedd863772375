"""Config-1 HyKKT and Lifted-KKT refactor+solve (N=50) for compute-sanitizer runs (memcheck / racecheck /
synccheck, one tool per run).  Usage: compute-sanitizer --tool memcheck python tools/sanitize_c1.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from kkt_cases import distillation_case, run_gpu  # noqa: E402

for strategy in (1, 0):
    case = distillation_case(50, strategy, iterates=[3, 12])
    g = run_gpu(case, strategy, leaf=64)
    for b in range(case.B):
        assert g["info"][b]["status"] == 0, g["info"][b]
        assert g["info"][b]["rel_res"] <= 1e-10
    print("strategy", strategy, "ok", [i["k_cg"] for i in g["info"]], flush=True)
print("sanitize_c1 done")
