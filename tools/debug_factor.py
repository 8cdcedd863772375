import sys, ctypes, numpy as np, scipy.sparse as sp
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from kkt_cases import distillation_case, random_case, run_gpu, run_oracle
from paper_2403_15913_b200 import ckkt
L = ckkt.lib(); L.ckkt_debug_get.restype = ctypes.c_int64; L.ckkt_debug_get.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
def get(ctx, what, dt):
    cnt = L.ckkt_debug_get(ctx.h, what, None); a = np.empty(cnt, dt); L.ckkt_debug_get(ctx.h, what, a.ctypes.data_as(ctypes.c_void_p)); return a
for (name, case, strat, leaf) in [("dist5", distillation_case(5, 1, [4]), 1, 16), ("rand41", random_case(41, 0, 12, seeds=[11]), 0, 8), ("dist300", distillation_case(300, 1, [4]), 1, 268)]:
    g = run_gpu(case, strat, leaf=leaf, gamma=1e7 if strat else 0.0)
    ctx = g['ctx']
    Lst = get(ctx, 0, np.float64); Kv = get(ctx, 1, np.float64); perm2 = get(ctx, 2, np.int32)
    sf = get(ctx, 3, np.int32); srp = get(ctx, 4, np.int64); sr = get(ctx, 5, np.int32); pofs = get(ctx, 6, np.int64)
    kp = get(ctx, 7, np.int64); ki = get(ctx, 8, np.int32)
    n = case.n
    K = sp.csc_matrix((Kv, ki, kp), shape=(n, n)).toarray(); K = K + np.tril(K, -1).T
    Ld = np.zeros((n, n))
    for s in range(len(sf) - 1):
        f, w = sf[s], sf[s+1]-sf[s]; rows = sr[srp[s]:srp[s+1]]; m = len(rows)
        P = Lst[pofs[s]:pofs[s]+m*w].reshape(w, m).T
        for c in range(w):
            Ld[rows[c:], f + c] = P[c:, c]
    E = np.abs(Ld @ Ld.T - K)
    print(name, 'LLt-K', E.max() / np.abs(K).max(), 'ns', len(sf)-1, 'nan', np.isnan(Ld).sum(), 'rel_res', g['info'][0]['rel_res_unrefined'], flush=True)
    o, d, info = run_oracle(case, 0, strat, gamma=1e7 if strat else 0.0, leaf=leaf)
    Ko = sp.csc_matrix((o.Ax, o.Ai, o.Ap), shape=(n, n)).toarray(); Ko = Ko + np.tril(Ko, -1).T
    Korig = np.empty_like(Ko); Korig[np.ix_(o.perm, o.perm)] = Ko
    Kint = Korig[np.ix_(perm2, perm2)]
    print('   K vs oracle K', np.abs(Kint - K).max() / np.abs(K).max(), flush=True)
    bad = np.where(E.max(axis=0) > 1e-8 * np.abs(K).max())[0]
    print('   bad cols', bad[:20], len(bad), flush=True)
