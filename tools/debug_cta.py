import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from kkt_cases import random_case, run_gpu
case = random_case(41, 0, 12, seeds=[11])
g = run_gpu(case, 0, gamma=0.0, leaf=8)
print('notpd', g['notpd'], 'minpiv', g['minpiv'], g['info'])
