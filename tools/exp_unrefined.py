"""Unrefined accuracy of the CUDA path vs the oracle on identical C3 iterates (VERDICT r01 item 4:
does the explicit L11^-1 of the sweeps cost accuracy?).  The oracle factors with a plain sparse
Cholesky and solves with triangular substitutions, so equal unrefined errors mean the stored
inverse diagonal blocks cost nothing.  Usage: python tools/exp_unrefined.py [N] [iterates...]"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import distillation as dist  # noqa: E402
from kkt_cases import distillation_case, run_gpu, run_oracle  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
its = [int(a) for a in sys.argv[2:]] or [3, 9, 15]
inst = dist.Instance(N)
for strategy, name in ((1, "hykkt"), (0, "lifted")):
    for k in its:
        case = distillation_case(N, strategy, iterates=[k], inst_obj=inst)
        g = run_gpu(case, strategy, leaf=1072)["info"][0]
        t = time.time()
        _, d, o = run_oracle(case, 0, strategy, gamma=1e7, leaf=1072)
        print(f"{name} N={N} iterate {k}: unrefined omega gpu {g['rel_res_unrefined']:.3e} oracle "
              f"{o.rel_res_unrefined:.3e} | k_cg gpu {g['k_cg']} oracle {o.k_cg} | n_ref gpu {g['n_ref']} "
              f"oracle {o.n_ref} | refined gpu {g['rel_res']:.2e} oracle {o.rel_res:.2e} "
              f"(oracle {time.time() - t:.0f} s)", flush=True)
