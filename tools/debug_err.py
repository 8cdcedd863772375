import sys, ctypes
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from kkt_cases import random_case, run_gpu
from paper_2403_15913_b200 import ckkt
L = ckkt.lib(); L.ckkt_debug_error_string.restype = ctypes.c_char_p
case = random_case(int(sys.argv[1]), 0, int(sys.argv[2]), seeds=[11])
try:
    g = run_gpu(case, 0, gamma=0.0, leaf=8)
    print('ok', g['info'])
except Exception as e:
    print('EXC', e, L.ckkt_debug_error_string())
