"""MatrixMarket dump of the condensed matrix K_gamma for oracle cross-checks (SURVEY §5 config/flags: the
SPEC's SOLVER_DEBUG_DUMP).  Refactors one distillation iterate through libckkt, reads the device's K values
(internal lower CSC, debug export) back in the ORIGINAL ordering, builds the oracle's K_gamma from the
same inputs, writes both as symmetric (lower) .mtx files and prints the largest relative entry difference.
Usage: python tools/dump_mm.py N iterate outdir [strategy: 1 = HyKKT, 0 = Lifted]"""
import ctypes
import os
import sys

import numpy as np
import scipy.io
import scipy.sparse as sp
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from kkt_cases import distillation_case  # noqa: E402
from oracle import kkt as OK  # noqa: E402
from paper_2403_15913_b200 import ckkt  # noqa: E402

N, k, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
strategy = int(sys.argv[4]) if len(sys.argv) > 4 else 1
os.makedirs(out, exist_ok=True)
case = distillation_case(N, strategy, iterates=[k])
L = ckkt.lib()
L.ckkt_debug_get.restype = ctypes.c_int64
L.ckkt_debug_get.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]


def get(ctx, what, dt):
    cnt = L.ckkt_debug_get(ctx.h, what, None)
    a = np.empty(cnt, dt)
    L.ckkt_debug_get(ctx.h, what, a.ctypes.data_as(ctypes.c_void_p))
    return a


dev = torch.device("cuda:0")
T = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev) if a.size else None
ctx = ckkt.Context(case.n, case.m_e, case.m_i, case.w_row, case.w_col,
                   case.g_rowptr if case.m_e else None, case.g_col if case.m_e else None,
                   case.h_rowptr if case.m_i else None, case.h_col if case.m_i else None,
                   strategy=strategy, gamma=1e7, leaf=1072, device=0,
                   stream=torch.cuda.current_stream().cuda_stream)
vals = [T(case.w_val[0]), T(case.g_val[0]), T(case.h_val[0]), T(case.sigma_x[0]), T(case.d_s[0]),
        T(case.delta_x[:1])]
ctx.refactor(*vals)
torch.cuda.synchronize()
kval = get(ctx, 1, np.float64)
kp, ki, perm2 = get(ctx, 7, np.int64), get(ctx, 8, np.int32), get(ctx, 2, np.int32)
n = case.n
cols = np.repeat(np.arange(n), np.diff(kp))
r, c = perm2[ki], perm2[cols]  # internal -> original indices
lo_r, lo_c = np.maximum(r, c), np.minimum(r, c)
K_gpu = sp.coo_matrix((kval, (lo_r, lo_c)), shape=(n, n)).tocsr()
o = OK.SparseKKT(case.n, case.m_e, case.m_i, case.w_row, case.w_col,
                 case.g_rowptr if case.m_e else np.zeros(1, np.int32), case.g_col if case.m_e else np.zeros(0, np.int32),
                 case.h_rowptr if case.m_i else np.zeros(1, np.int32), case.h_col if case.m_i else np.zeros(0, np.int32),
                 strategy=strategy, gamma=1e7, leaf=1072)
o.refactor(case.w_val[0], case.g_val[0], case.h_val[0], case.sigma_x[0], case.d_s[0], float(case.delta_x[0]))
K_or = sp.coo_matrix((o.Ax, (np.maximum(o.k_row, o.k_col), np.minimum(o.k_row, o.k_col))), shape=(n, n)).tocsr()
tag = f"N{N}_it{k}_{'hykkt' if strategy == 1 else 'lifted'}"
scipy.io.mmwrite(os.path.join(out, f"K_gpu_{tag}.mtx"), K_gpu, symmetry="symmetric")
scipy.io.mmwrite(os.path.join(out, f"K_oracle_{tag}.mtx"), K_or, symmetry="symmetric")
d = abs(K_gpu - K_or)
scale = abs(K_or).max()
print(f"{tag}: n {n}, nnz(lower) gpu {K_gpu.nnz} oracle {K_or.nnz}, max |K_gpu - K_oracle| / max|K| = "
      f"{d.max() / scale:.2e}; written to {out}")
