"""Tier S oracle: the sparse Newton-step solve (TEST INFRASTRUCTURE ONLY).

Follows PAPER.md §IV-§V in the paper's order and notation:

  setup     : K pattern = pattern(W) ∪ pattern(G^T G) ∪ pattern(H^T H) ∪ diag
              (fixed across iterations); ordering;
              symbolic analysis
  refactor  : K_gamma = W + Sigma_x + delta_x I + H^T D_s H + gamma G^T G
              (gamma = 0 for Lifted-KKT), Cholesky;
              breakdown = wrong inertia (Haynsworth P:317-321)
  solve     : condensed rhs r~ = r1 + H^T (D_s r4 - r2)
              Lifted-KKT: K dx = -r~   (Eq. liftedkkt)
              HyKKT: r_gamma = r~ + gamma G^T r3;
                     CG on S_gamma dy = r3 - G K_gamma^{-1} r_gamma (Eq. schurcomp,
                     P:389-392, matrix-free, no preconditioner);
                     K_gamma dx = -r_gamma - G^T dy (reading R2 of P:394)
              recovery ds = -r4 - H dx, dz = -r2 - D_s ds
              Richardson refinement on K_aug (reading R7)

Library primitives used as single steps: scipy.sparse products / matvecs and
numpy dot products.  The Cholesky, triangular solves, ordering and symbolic
analysis are the plain C of oracle/csrc/sparse_oracle.c.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.sparse as sp

from . import sparse as S

LIFTED, HYKKT = 0, 1


@dataclasses.dataclass
class Info:
    k_cg: int = 0            # CG iterations of the first (unrefined) solve
    k_cg_total: int = 0      # CG iterations over all refinement passes
    n_ref: int = 0           # Richardson corrections applied
    rel_res: float = np.nan  # componentwise backward error of the returned step
    rel_res_unrefined: float = np.nan
    res_inf: float = np.nan  # ||K_aug d + r||_inf
    cg_converged: bool = True


def csr(m, n, rp, ci, v=None):
    if v is None:
        v = np.ones(len(ci))
    return sp.csr_matrix((np.asarray(v, dtype=np.float64), np.asarray(ci), np.asarray(rp)), shape=(m, n))


class SparseKKT:
    """Sparse oracle for one pattern.  Arguments follow include/ckkt.h."""

    def __init__(self, n, m_e, m_i, w_row, w_col, g_rowptr, g_col, h_rowptr, h_col,
                 strategy=HYKKT, leaf=64, perm=None, gamma=1e7,
                 cg_rtol=1e-10, cg_maxit=200, ref_tol=1e-14, ref_maxit=10):
        self.n, self.m_e, self.m_i = n, m_e, m_i
        self.strategy = strategy
        if strategy == LIFTED and m_e != 0:
            raise ValueError("Lifted-KKT requires m_e = 0 (all equalities relaxed, P:333-346)")
        self.gamma = gamma if strategy == HYKKT else 0.0
        self.cg_rtol, self.cg_maxit = cg_rtol, cg_maxit
        self.ref_tol, self.ref_maxit = ref_tol, ref_maxit
        self.w_row = np.asarray(w_row, dtype=np.int64)
        self.w_col = np.asarray(w_col, dtype=np.int64)
        self.Gp = csr(m_e, n, g_rowptr, g_col)
        self.Hp = csr(m_i, n, h_rowptr, h_col)
        self.g_rowptr, self.g_col = np.asarray(g_rowptr), np.asarray(g_col)
        self.h_rowptr, self.h_col = np.asarray(h_rowptr), np.asarray(h_col)
        # --- K pattern (structural union, all-positive weights: no cancellation)
        Wp = sp.coo_matrix((np.ones(len(self.w_row)), (self.w_row, self.w_col)), shape=(n, n)).tocsr()
        Kp = (Wp + Wp.T + self.Gp.T @ self.Gp + self.Hp.T @ self.Hp + sp.eye(n, format="csr")).tocsr()
        Kp.sum_duplicates()
        Kp.sort_indices()
        self.Kp = Kp
        # adjacency without self loops
        A = Kp.tolil()
        A.setdiag(0)
        A = A.tocsr()
        A.eliminate_zeros()
        A.sort_indices()
        self.xadj = A.indptr.astype(np.int32)
        self.adj = A.indices.astype(np.int32)
        # --- ordering
        self.perm = S.nd_order(self.xadj, self.adj, leaf) if perm is None else np.asarray(perm, dtype=np.int32)
        self.iperm = np.empty(n, dtype=np.int32)
        self.iperm[self.perm] = np.arange(n, dtype=np.int32)
        # --- permuted lower CSC pattern of P K P^T
        coo = Kp.tocoo()
        pi, pj = self.iperm[coo.row], self.iperm[coo.col]
        keep = pi >= pj
        self.k_row, self.k_col = coo.row[keep], coo.col[keep]   # original (row, col) of each slot
        pi, pj = pi[keep], pj[keep]
        order = np.lexsort((pi, pj))
        self.k_row, self.k_col, pi, pj = self.k_row[order], self.k_col[order], pi[order], pj[order]
        self.Ai = pi.astype(np.int32)
        self.Ap = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(pj, minlength=n), out=self.Ap[1:])
        # --- symbolic analysis
        self.parent, self.colcount, self.Lp, self.Li = S.symbolic(self.Ap, self.Ai)
        self.Lx = None

    # ------------------------------------------------------------------
    def refactor(self, w_val, g_val, h_val, sigma_x, d_s, delta_x):
        n = self.n
        self.W = sp.coo_matrix((np.asarray(w_val, dtype=np.float64), (self.w_row, self.w_col)), shape=(n, n)).tocsr()
        Wl = self.W
        self.Wsym = (Wl + Wl.T - sp.diags(Wl.diagonal())).tocsr()
        self.diag = np.asarray(sigma_x, dtype=np.float64) + float(delta_x)
        self.G = csr(self.m_e, n, self.g_rowptr, self.g_col, g_val)
        self.H = csr(self.m_i, n, self.h_rowptr, self.h_col, h_val)
        self.d_s = np.asarray(d_s, dtype=np.float64)
        # K_gamma = W + Sigma + delta I + H^T D_s H + gamma G^T G
        K = self.Wsym + sp.diags(self.diag) + self.H.T @ sp.diags(self.d_s) @ self.H
        if self.m_e:
            K = K + self.gamma * (self.G.T @ self.G)
        K = K.tocsr()
        Kd = K.todok() if n < 2000 else None
        if Kd is not None:
            Ax = np.array([Kd.get((r, c), 0.0) for r, c in zip(self.k_row, self.k_col)])
        else:
            K.sum_duplicates()
            K.sort_indices()
            Ax = _gather_csr(K, self.k_row, self.k_col)
        self.Ax = Ax
        self.Lx, fail = S.cholesky(self.Ap, self.Ai, Ax, self.Lp, self.Li)
        self.fail = fail
        return fail

    def kgamma_solve(self, b):
        """x = K_gamma^{-1} b = P^T L^{-T} L^{-1} P b."""
        y = S.lsolve(self.Lp, self.Li, self.Lx, b[self.perm])
        y = S.ltsolve(self.Lp, self.Li, self.Lx, y)
        x = np.empty(self.n)
        x[self.perm] = y
        return x

    # ------------------------------------------------------------------
    def _cg(self, b):
        """Unpreconditioned CG on S_gamma = G K_gamma^{-1} G^T, x0 = 0 (reading R6)."""
        x = np.zeros(self.m_e)
        bnorm = np.linalg.norm(b)
        if bnorm == 0.0:
            return x, 0, True
        r = b.copy()
        p = r.copy()
        rr = r @ r
        for k in range(1, self.cg_maxit + 1):
            q = self.G @ self.kgamma_solve(self.G.T @ p)
            alpha = rr / (p @ q)
            x += alpha * p
            r -= alpha * q
            rr_new = r @ r
            if np.sqrt(rr_new) <= self.cg_rtol * bnorm:
                return x, k, True
            p = r + (rr_new / rr) * p
            rr = rr_new
        return x, self.cg_maxit, False

    def solve_once(self, r1, r2, r3, r4):
        """One unrefined pass of the strategy: returns (dx, ds, dy, dz, k_cg, converged)."""
        rt = r1 + self.H.T @ (self.d_s * r4 - r2)
        k, conv = 0, True
        if self.m_e:
            rg = rt + self.gamma * (self.G.T @ r3)
            b = r3 - self.G @ self.kgamma_solve(rg)          # Eq. schurcomp rhs
            dy, k, conv = self._cg(b)
            dx = self.kgamma_solve(-rg - self.G.T @ dy)      # reading R2
        else:
            dy = np.zeros(0)
            dx = self.kgamma_solve(-rt)                      # Eq. liftedkkt
        ds = -r4 - self.H @ dx
        dz = -r2 - self.d_s * ds
        return dx, ds, dy, dz, k, conv

    def kaug_residual(self, r, d):
        """rho = -r - K_aug d and the componentwise backward error
        omega = max_i |rho_i| / (|K_aug| |d| + |r|)_i  (reading R7)."""
        r1, r2, r3, r4 = r
        dx, ds, dy, dz = d
        Wd = self.Wsym @ dx + self.diag * dx
        aWd = abs(self.Wsym) @ abs(dx) + abs(self.diag * dx)
        rho1 = -r1 - (Wd + self.G.T @ dy + self.H.T @ dz)
        a1 = aWd + abs(self.G.T) @ abs(dy) + abs(self.H.T) @ abs(dz) + abs(r1)
        rho2 = -r2 - (self.d_s * ds + dz)
        a2 = abs(self.d_s * ds) + abs(dz) + abs(r2)
        rho3 = -r3 - self.G @ dx
        a3 = abs(self.G) @ abs(dx) + abs(r3)
        rho4 = -r4 - (self.H @ dx + ds)
        a4 = abs(self.H) @ abs(dx) + abs(ds) + abs(r4)
        rho = np.concatenate([rho1, rho2, rho3, rho4])
        a = np.concatenate([a1, a2, a3, a4])
        with np.errstate(invalid="ignore", divide="ignore"):
            w = np.where(a > 0, np.abs(rho) / a, np.where(rho == 0, 0.0, np.inf))
        omega = float(w.max()) if len(w) else 0.0
        return (rho1, rho2, rho3, rho4), omega, float(np.abs(rho).max()) if len(rho) else 0.0

    def solve(self, r1, r2, r3, r4):
        """Newton step solving K_aug d = -r with Richardson refinement."""
        if self.Lx is None or self.fail >= 0:
            raise RuntimeError("refactor failed or not called")
        r = (np.asarray(r1, float), np.asarray(r2, float), np.asarray(r3, float), np.asarray(r4, float))
        info = Info()
        dx, ds, dy, dz, k, conv = self.solve_once(*r)
        info.k_cg = info.k_cg_total = k
        info.cg_converged = conv
        d = [dx, ds, dy, dz]
        rho, omega, rinf = self.kaug_residual(r, d)
        info.rel_res_unrefined = omega
        best = (omega, rinf, [x.copy() for x in d])
        prev = omega
        for it in range(self.ref_maxit):
            if omega <= self.ref_tol:
                break
            c = self.solve_once(*(-x for x in rho))
            info.k_cg_total += c[4]
            d = [d[0] + c[0], d[1] + c[1], d[2] + c[2], d[3] + c[3]]
            info.n_ref += 1
            rho, omega, rinf = self.kaug_residual(r, d)
            if omega < best[0]:
                best = (omega, rinf, [x.copy() for x in d])
            if omega > 0.5 * prev:      # stagnation: keep the best iterate
                break
            prev = omega
        info.rel_res, info.res_inf = best[0], best[1]
        return tuple(best[2]), info


def inertia_correction(kkt: SparseKKT, w_val, g_val, h_val, sigma_x, d_s, delta_last=0.0,
                       delta_first=1e-4, kappa_plus=8.0, delta_min=1e-20, delta_max=1e40):
    """Inertia correction around the refactorization ("(delta_x, delta_c) are computed so
    as the regularized system satisfies (8)"; Cholesky success <=> correct inertia).
    Schedule = DESIGN.md reading R15 (SPEC inertia_correction): try delta = 0; on failure start at
    delta_first * max(1, ||W||_inf) if delta_last == 0, else max(delta_min, delta_last / 3) (kappa_minus = 1/3);
    multiply by kappa_plus after each further failure; give up above delta_max.
    Returns (delta, trials, failed)."""
    delta, trials = 0.0, 0
    while True:
        trials += 1
        if kkt.refactor(w_val, g_val, h_val, sigma_x, d_s, delta) < 0:
            return delta, trials, False
        if delta == 0.0:
            if delta_last == 0.0:
                w_inf = float(abs(kkt.Wsym).sum(axis=1).max()) if kkt.Wsym.nnz else 0.0   # ||W||_inf
                # max(1, ||W||_inf); a NaN norm propagates (NaN values never factor: give up)
                d = delta_first * (w_inf if not w_inf <= 1.0 else 1.0)
            else:
                d = max(delta_min, delta_last / 3.0)
        else:
            d = kappa_plus * delta
        if not d <= delta_max:
            return delta, trials, True
        delta = d


def _gather_csr(K, rows, cols):
    """K[rows[i], cols[i]] for a csr matrix with sorted indices (0 where absent)."""
    out = np.zeros(len(rows))
    indptr, indices, data = K.indptr, K.indices, K.data
    # process row by row via searchsorted on the concatenated keys
    key = rows.astype(np.int64) * K.shape[1] + cols.astype(np.int64)
    rr = np.repeat(np.arange(K.shape[0], dtype=np.int64), np.diff(indptr))
    kkey = rr * K.shape[1] + indices.astype(np.int64)
    pos = np.searchsorted(kkey, key)
    pos_c = np.minimum(pos, len(kkey) - 1)
    hit = (pos < len(kkey)) & (kkey[pos_c] == key)
    out[hit] = data[pos_c[hit]]
    return out


def fraction_to_boundary(s, ds, tau):
    """Largest alpha in (0, 1] with s + alpha ds >= (1 - tau) s, for s > 0 (the step
    length is "computed using a fraction-to-boundary rule"; SPEC fraction_to_boundary):
    alpha = min(1, min over ds_i < 0 of tau s_i / (-ds_i)).  Entries whose ratio is NaN are
    skipped (Python's min keeps the running value against NaN)."""
    alpha = 1.0
    for si, di in zip(np.asarray(s, dtype=np.float64).tolist(), np.asarray(ds, dtype=np.float64).tolist()):
        if di < 0:
            alpha = min(alpha, tau * si / -di)
    return alpha
