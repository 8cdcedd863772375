"""Experiment (not part of the product): dx = -t - sum_k alpha_k K^{-1} G^T p_k accumulated during
CG (no separate dx solve) vs the fresh solve dx = K^{-1}(-r_gamma - G^T dy); refinement counts."""
import sys
import numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__)))); sys.path.insert(0, __import__('os').path.join(__import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))), 'tests'))
from oracle import kkt as OK
from kkt_cases import distillation_case, E32

class Acc(OK.SparseKKT):
    acc = False
    def _cg_acc(self, b):
        x = np.zeros(self.m_e); z = np.zeros(self.n)
        bnorm = np.linalg.norm(b)
        if bnorm == 0.0:
            return x, z, 0, True
        r = b.copy(); p = r.copy(); rr = r @ r
        for k in range(1, self.cg_maxit + 1):
            vn = self.kgamma_solve(self.G.T @ p)
            q = self.G @ vn
            alpha = rr / (p @ q)
            x += alpha * p; z += alpha * vn
            r -= alpha * q
            rr_new = r @ r
            if np.sqrt(rr_new) <= self.cg_rtol * bnorm:
                return x, z, k, True
            p = r + (rr_new / rr) * p
            rr = rr_new
        return x, z, self.cg_maxit, False

    def solve_once(self, r1, r2, r3, r4):
        if not self.acc:
            return super().solve_once(r1, r2, r3, r4)
        rt = r1 + self.H.T @ (self.d_s * r4 - r2)
        rg = rt + self.gamma * (self.G.T @ r3)
        t = self.kgamma_solve(rg)
        b = r3 - self.G @ t
        dy, z, k, conv = self._cg_acc(b)
        dx = -t - z
        ds = -r4 - self.H @ dx
        dz = -r2 - self.d_s * ds
        return dx, ds, dy, dz, k, conv

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
case = distillation_case(N, 1, iterates=[3, 9, 15])
for acc in (False, True):
    for b in range(case.B):
        o = Acc(case.n, case.m_e, case.m_i, case.w_row, case.w_col, case.g_rowptr, case.g_col, E32, E32[:0],
                strategy=1, gamma=1e7, leaf=1072)
        o.acc = acc
        o.refactor(case.w_val[b], case.g_val[b], case.h_val[b], case.sigma_x[b], case.d_s[b], case.delta_x[b])
        d, info = o.solve(case.r1[b], case.r2[b], case.r3[b], case.r4[b])
        print('acc' if acc else 'solve', 'iterate', b, 'k_cg', info.k_cg, 'total', info.k_cg_total, 'n_ref', info.n_ref,
              'omega0 %.2e' % info.rel_res_unrefined, 'omega %.2e' % info.rel_res)
