"""Cycles of the dense-front warp Cholesky+inversion and the DMMA TRSM (debug entry point)."""
import ctypes, sys
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2403_15913_b200 import ckkt
L = ckkt.lib()
L.ckkt_debug_bench_chol.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
for w, m in [(4, 20), (8, 40), (13, 60), (16, 80), (24, 110), (32, 140), (48, 180), (55, 200), (64, 250)]:
    out = np.zeros(2, np.int64)
    L.ckkt_debug_bench_chol(w, m, 20, out.ctypes.data_as(ctypes.c_void_p))
    print(f"w={w:3d} m={m:4d}: chol+inv {out[0]:7d} cycles ({out[0]/w:6.0f}/col)  trsm {out[1]:7d} cycles")
