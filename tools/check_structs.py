"""Host-side consistency check of the internal supernodal structures (debug export)."""
import ctypes, sys
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2403_15913_b200 import ckkt
from inputs.random_kkt import random_instance
from inputs.distillation import build_pattern
L = ckkt.lib(); L.ckkt_debug_get.restype = ctypes.c_int64; L.ckkt_debug_get.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
def get(ctx, what, dt):
    cnt = L.ckkt_debug_get(ctx.h, what, None); a = np.empty(cnt, dt); L.ckkt_debug_get(ctx.h, what, a.ctypes.data_as(ctypes.c_void_p)); return a
def check(ctx):
    sf = get(ctx,3,np.int32); srp = get(ctx,4,np.int64); sr = get(ctx,5,np.int32); pofs = get(ctx,6,np.int64)
    kp = get(ctx,7,np.int64); ki = get(ctx,8,np.int32); chp = get(ctx,9,np.int32); chl = get(ctx,10,np.int32)
    relofs = get(ctx,11,np.int64); relmap = get(ctx,12,np.int32); uofs = get(ctx,13,np.int64); kmap = get(ctx,15,np.int32)
    ns = len(sf)-1; n = sf[-1]
    par = -np.ones(ns, int)
    for s in range(ns):
        for c in chl[chp[s]:chp[s+1]]: par[c] = s
    for s in range(ns):
        f, w = sf[s], sf[s+1]-sf[s]; rows = sr[srp[s]:srp[s+1]]; m = len(rows)
        assert w >= 1 and m >= w, (s, w, m)
        assert np.array_equal(rows[:w], np.arange(f, f+w)), (s, rows[:w], f, w)
        assert np.all(np.diff(rows) > 0)
        assert pofs[s+1]-pofs[s] == m*w
        for j in range(f, f+w):
            for k in range(kp[j], kp[j+1]):
                assert 0 <= kmap[k] < m*w, (s, j, k, kmap[k], m, w)
                col, row = divmod(kmap[k], m); assert col == j-f and rows[row] == ki[k]
        if par[s] >= 0:
            p = par[s]; prow = sr[srp[p]:srp[p+1]]
            rel = relmap[relofs[s]:relofs[s]+m-w]
            assert np.array_equal(prow[rel], rows[w:]), s
            assert p > s
        else:
            assert m == w
    print('ok ns', ns, 'n', n, 'max w', np.diff(sf).max())
inst = random_instance(10, 0, 3, seed=11)
check(ckkt.Context(10, 0, 3, inst.w_row, inst.w_col, None, None, inst.h_rowptr, inst.h_col, leaf=8, device=-1, strategy=0))
inst = random_instance(41, 0, 12, seed=11)
check(ckkt.Context(41, 0, 12, inst.w_row, inst.w_col, None, None, inst.h_rowptr, inst.h_col, leaf=8, device=-1, strategy=0))
pat = build_pattern(30)
check(ckkt.Context(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=268, device=-1))
