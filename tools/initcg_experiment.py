"""Experiment (not part of the product): CG iterations of the refinement passes with a warm start
projected onto the first pass's Krylov directions (Init-CG / deflation) vs the plain x0 = 0."""
import sys
import numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__)))); sys.path.insert(0, __import__('os').path.join(__import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))), 'tests'))
from oracle import kkt as OK
from kkt_cases import distillation_case, E32

class RecCG(OK.SparseKKT):
    mode = 'plain'
    def _cg(self, b):
        bnorm = np.linalg.norm(b)
        x = np.zeros(self.m_e)
        if bnorm == 0.0:
            return x, 0, True
        store = not hasattr(self, 'P') or self.mode == 'init2'
        if hasattr(self, 'P') and self.mode != 'plain':
            # x0 = P (P^T S P)^{-1} P^T b with S p_i = q_i, P^T S P diagonal (CG conjugacy)
            for p, q, pq in zip(self.P, self.Q, self.PQ):
                x += (p @ b) / pq * p
            r = b - sum(((p @ b) / pq) * q for p, q, pq in zip(self.P, self.Q, self.PQ))
        else:
            r = b.copy()
        if store:
            self.P, self.Q, self.PQ = [], [], []  # (init2: each pass replaces the store)
        p = r.copy(); rr = r @ r
        if not store and self.mode == 'aug':
            for pi, qi, pqi in zip(self.P, self.Q, self.PQ):
                p -= (qi @ r) / pqi * pi
        for k in range(1, self.cg_maxit + 1):
            if np.sqrt(rr) <= self.cg_rtol * bnorm:
                return x, k - 1, True
            q = self.G @ self.kgamma_solve(self.G.T @ p)
            pq = p @ q
            if store:
                self.P.append(p.copy()); self.Q.append(q.copy()); self.PQ.append(pq)
            if not store and self.mode == 'aug' and getattr(self, 'append', False) and len(self.P) < 64:
                self.P2.append(p.copy()); self.Q2.append(q.copy()); self.PQ2.append(pq)
            alpha = rr / pq
            x += alpha * p
            r -= alpha * q
            rr_new = r @ r
            if np.sqrt(rr_new) <= self.cg_rtol * bnorm:
                return x, k, True
            p = r + (rr_new / rr) * p
            if not store and self.mode == 'aug':
                # AugCG: keep the new direction S-conjugate to the stored ones
                for pi, qi, pqi in zip(self.P, self.Q, self.PQ):
                    p -= (qi @ r) / pqi * pi
            rr = rr_new
        return x, self.cg_maxit, False

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
case = distillation_case(N, 1, iterates=[3, 9, 15])
for mode in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['plain', 'init', 'aug']):
    for b in range(case.B):
        o = RecCG(case.n, case.m_e, case.m_i, case.w_row, case.w_col, case.g_rowptr, case.g_col, E32, E32[:0],
                  strategy=1, gamma=1e7, leaf=1072)
        o.mode = mode
        o.refactor(case.w_val[b], case.g_val[b], case.h_val[b], case.sigma_x[b], case.d_s[b], case.delta_x[b])
        d, info = o.solve(case.r1[b], case.r2[b], case.r3[b], case.r4[b])
        print(mode, 'iterate', b, 'k_cg', info.k_cg, 'total', info.k_cg_total, 'n_ref', info.n_ref, 'omega', info.rel_res)
