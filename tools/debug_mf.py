"""Emulate the multifrontal factorization on the host with the library's own internal structures
(debug export) and report the first supernode whose GPU panel / update matrix differs."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
from kkt_cases import distillation_case, random_case, run_gpu  # noqa: E402
from paper_2403_15913_b200 import ckkt  # noqa: E402

L = ckkt.lib()
L.ckkt_debug_get.restype = ctypes.c_int64
L.ckkt_debug_get.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]


def get(ctx, what, dt):
    cnt = L.ckkt_debug_get(ctx.h, what, None)
    a = np.empty(cnt, dt)
    L.ckkt_debug_get(ctx.h, what, a.ctypes.data_as(ctypes.c_void_p))
    return a


if len(sys.argv) < 2:
    case, strat, gamma, leaf = random_case(41, 0, 12, seeds=[11]), 0, 0.0, 8
else:
    case, strat, gamma, leaf = distillation_case(int(sys.argv[1]), 1, [4]), 1, 1e7, 64
g = run_gpu(case, strat, gamma=gamma, leaf=leaf)
ctx = g['ctx']
print('notpd', g['notpd'], 'minpiv', g['minpiv'])
Lg = get(ctx, 0, np.float64)
Kv = get(ctx, 1, np.float64)
Ug = get(ctx, 14, np.float64)
sf = get(ctx, 3, np.int32)
srp = get(ctx, 4, np.int64)
pofs = get(ctx, 6, np.int64)
kp = get(ctx, 7, np.int64)
chp = get(ctx, 9, np.int32)
chl = get(ctx, 10, np.int32)
relofs = get(ctx, 11, np.int64)
relmap = get(ctx, 12, np.int32)
uofs = get(ctx, 13, np.int64)
kmap = get(ctx, 15, np.int32)
ns = len(sf) - 1
Ue = {}
for s in range(ns):
    f, w = sf[s], sf[s + 1] - sf[s]
    m = srp[s + 1] - srp[s]
    mu = m - w
    F = np.zeros((m, m))
    P = np.zeros(m * w)
    for k in range(kp[f], kp[f + w]):
        P[kmap[k]] = Kv[k]
    F[:, :w] = P.reshape(w, m).T
    for ci in range(chp[s], chp[s + 1]):
        c = chl[ci]
        mc = (srp[c + 1] - srp[c]) - (sf[c + 1] - sf[c])
        rel = relmap[relofs[c]:relofs[c] + mc]
        Uc = Ue[c]
        for j in range(mc):
            for i in range(j, mc):
                F[rel[i], rel[j]] += Uc[i, j]
    F = np.tril(F) + np.tril(F, -1).T
    if not np.all(np.linalg.eigvalsh(F[:w, :w]) > 0):
        print('emulation NOT PD at supernode', s, 'f', f, 'w', w, 'm', m)
        break
    L11 = np.linalg.cholesky(F[:w, :w])
    L21 = np.linalg.solve(L11, F[w:, :w].T).T
    Ue[s] = np.tril(F[w:, w:] - L21 @ L21.T)
    Pg = Lg[pofs[s]:pofs[s] + m * w].reshape(w, m).T
    Z = np.linalg.inv(L11)
    e1 = np.abs(np.tril(Pg[:w]) - np.tril(Z)).max() / max(1, np.abs(Z).max())
    e2 = np.abs(Pg[w:] - L21).max() / max(1, np.abs(L21).max()) if mu else 0
    Ugs = Ug[uofs[s]:uofs[s] + mu * mu].reshape(mu, mu).T if mu else np.zeros((0, 0))
    e3 = np.abs(np.tril(Ugs) - Ue[s]).max() / max(1, np.abs(Ue[s]).max()) if mu else 0
    if max(e1, e2, e3) > 1e-8:
        print('MISMATCH supernode', s, 'f', f, 'w', w, 'm', m, 'children', list(chl[chp[s]:chp[s + 1]]), 'errs', e1,
              e2, e3)
        print(' Z emu', np.round(Z[:4, :4], 4))
        print(' Z gpu', np.round(Pg[:4, :4], 4))
        print(' L21 emu', np.round(L21[:3, :4], 4))
        print(' L21 gpu', np.round(Pg[w:w + 3, :4], 4))
        break
else:
    print('all', ns, 'supernodes match')
