import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from kkt_cases import distillation_case, run_gpu
for N in [5, 20, 50]:
    for leaf in [16, 64, 268]:
        for strat in [1, 0]:
            case = distillation_case(N, strat, iterates=[4])
            g = run_gpu(case, strat, leaf=leaf)
            sz = g['ctx'].get_sizes()
            print(N, leaf, strat, g['rc'], g['info'][0]['rel_res_unrefined'], g['info'][0]['rel_res'], sz['n_supernodes'], sz['n_levels'], flush=True)
