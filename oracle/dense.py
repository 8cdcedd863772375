"""Tier T oracle: dense formulas for tiny systems (TEST INFRASTRUCTURE ONLY).

Every function writes out a definition from PAPER.md; no blocking, fusion or
reordering beyond the definition.  Inputs are inputs.random_kkt.KKTInstance
(or anything with the same fields).

Notation: W_eff = W + diag(Sigma_x) + delta_x I — the paper's W_k with the
variable-bound barrier term folded in and the primal regularization of
P:239-244 (reading R3).
"""
from __future__ import annotations

import math

import numpy as np

BK_ALPHA = (1.0 + math.sqrt(17.0)) / 8.0


# --------------------------------------------------------------------------
# K_aug and its blocks
# --------------------------------------------------------------------------
def W_eff(inst) -> np.ndarray:
    return inst.W_dense() + np.diag(inst.sigma_x) + inst.delta_x * np.eye(inst.n)


def assemble_kaug(inst) -> np.ndarray:
    """K_aug of Eq. kkt:augmented, unknown order (dx, ds, dy, dz)."""
    n, me, mi = inst.n, inst.m_e, inst.m_i
    G, H = inst.G_dense(), inst.H_dense()
    N = n + mi + me + mi
    K = np.zeros((N, N))
    ix, is_, iy, iz = slice(0, n), slice(n, n + mi), slice(n + mi, n + mi + me), slice(n + mi + me, N)
    K[ix, ix] = W_eff(inst)
    K[ix, iy] = G.T
    K[ix, iz] = H.T
    K[is_, is_] = np.diag(inst.d_s)
    K[is_, iz] = np.eye(mi)
    K[iy, ix] = G
    K[iz, ix] = H
    K[iz, is_] = np.eye(mi)
    return K


def rhs_vector(inst) -> np.ndarray:
    """r = (r1, r2, r3, r4); the step solves K_aug d = -r."""
    return np.concatenate([inst.r1, inst.r2, inst.r3, inst.r4])


def split_step(inst, d):
    n, me, mi = inst.n, inst.m_e, inst.m_i
    return d[:n], d[n:n + mi], d[n + mi:n + mi + me], d[n + mi + me:]


def assemble_kcond(inst, K=None) -> np.ndarray:
    """K_cond = [K G^T; G 0] of Eq. kkt:condensed."""
    K = condensed_matrix(inst) if K is None else K
    G = inst.G_dense()
    n, me = inst.n, inst.m_e
    Kc = np.zeros((n + me, n + me))
    Kc[:n, :n] = K
    Kc[:n, n:] = G.T
    Kc[n:, :n] = G
    return Kc


# --------------------------------------------------------------------------
# Bunch–Kaufman LDL^T with inertia (textbook partial pivoting)
# --------------------------------------------------------------------------
class BunchKaufman:
    """P A P^T = L D L^T, D block diagonal with 1x1 / 2x2 blocks.

    Pivot choice: Bunch & Kaufman (1977) with alpha = (1 + sqrt 17)/8.
    """

    def __init__(self, A: np.ndarray):
        A = np.array(A, dtype=np.float64, copy=True)
        n = A.shape[0]
        assert A.shape == (n, n)
        self.n = n
        self.scale = np.max(np.abs(A)) if n else 0.0
        L = np.eye(n)
        perm = np.arange(n)
        blocks = []  # (k, size)
        k = 0

        def swap(i, j):
            if i == j:
                return
            A[[i, j], :] = A[[j, i], :]
            A[:, [i, j]] = A[:, [j, i]]
            L[[i, j], :k] = L[[j, i], :k]
            perm[[i, j]] = perm[[j, i]]

        while k < n:
            akk = abs(A[k, k])
            if k == n - 1:
                size = 1
            else:
                col = np.abs(A[k + 1:, k])
                r = k + 1 + int(np.argmax(col))
                lam = col.max()
                if max(akk, lam) == 0.0:
                    size = 1
                elif akk >= BK_ALPHA * lam:
                    size = 1
                else:
                    rowr = np.abs(A[k:, r]).copy()
                    rowr[r - k] = 0.0
                    sig = rowr.max()
                    if akk * sig >= BK_ALPHA * lam * lam:
                        size = 1
                    elif abs(A[r, r]) >= BK_ALPHA * sig:
                        swap(k, r)
                        size = 1
                    else:
                        swap(k + 1, r)
                        size = 2
            if size == 1:
                d = A[k, k]
                if d != 0.0:
                    l = A[k + 1:, k] / d
                    A[k + 1:, k + 1:] -= d * np.outer(l, l)
                    L[k + 1:, k] = l
                blocks.append((k, 1))
                k += 1
            else:
                E = A[k:k + 2, k:k + 2].copy()
                C = A[k + 2:, k:k + 2]
                Lb = C @ np.linalg.inv(E)
                A[k + 2:, k + 2:] -= Lb @ C.T
                L[k + 2:, k:k + 2] = Lb
                blocks.append((k, 2))
                k += 2
        self.L = L
        self.perm = perm
        self.blocks = blocks
        self.Dblocks = []
        for (k, s) in blocks:
            self.Dblocks.append(A[k:k + s, k:k + s].copy())

    def inertia(self, rtol: float = 1e-10):
        """(n_plus, n_zero, n_minus); |eigenvalue of a D block| <= rtol*max|A| counts as zero."""
        tol = rtol * self.scale
        pos = zero = neg = 0
        for D in self.Dblocks:
            for ev in np.linalg.eigvalsh(D):
                if abs(ev) <= tol:
                    zero += 1
                elif ev > 0:
                    pos += 1
                else:
                    neg += 1
        return pos, zero, neg

    def solve(self, b: np.ndarray) -> np.ndarray:
        y = b[self.perm].astype(np.float64).copy()
        n = self.n
        # L z = y (unit lower)
        for j in range(n):
            y[j + 1:] -= self.L[j + 1:, j] * y[j]
        # D w = z
        for (k, s), D in zip(self.blocks, self.Dblocks):
            y[k:k + s] = np.linalg.solve(D, y[k:k + s])
        # L^T x = w
        for j in range(n - 1, -1, -1):
            y[j] -= self.L[j + 1:, j] @ y[j + 1:]
        x = np.empty(n)
        x[self.perm] = y
        return x


def eig_inertia(A: np.ndarray, rtol: float = 1e-10):
    """Inertia by a dense symmetric eigendecomposition (library routine)."""
    ev = np.linalg.eigvalsh(A)
    tol = rtol * max(np.max(np.abs(A)), 1e-300)
    return int((ev > tol).sum()), int((np.abs(ev) <= tol).sum()), int((ev < -tol).sum())


# --------------------------------------------------------------------------
# Step definitions
# --------------------------------------------------------------------------
def augmented_step(inst):
    """The Newton step as defined: K_aug d = -r, by Bunch–Kaufman.
    Returns (dx, ds, dy, dz), inertia triple."""
    K = assemble_kaug(inst)
    bk = BunchKaufman(K)
    d = bk.solve(-rhs_vector(inst))
    return split_step(inst, d), bk.inertia()


def condensed_matrix(inst) -> np.ndarray:
    """K_k = W_k + delta_x I + H^T D_s H, W_k incl. Sigma_x."""
    H = inst.H_dense()
    return W_eff(inst) + H.T @ np.diag(inst.d_s) @ H


def condensed_rhs(inst) -> np.ndarray:
    """r1 + H^T (D_s r4 - r2); the condensed system is K_cond d = -[this; r3]."""
    H = inst.H_dense()
    return inst.r1 + H.T @ (inst.d_s * inst.r4 - inst.r2)


def recover_slack_dual(inst, dx):
    """d_s = -r4 - H dx ; d_z = -r2 - D_s d_s."""
    H = inst.H_dense()
    ds = -inst.r4 - H @ dx
    dz = -inst.r2 - inst.d_s * ds
    return ds, dz


def hykkt_matrix(inst, gamma: float) -> np.ndarray:
    """K_gamma = K_k + gamma G^T G."""
    G = inst.G_dense()
    return condensed_matrix(inst) + gamma * G.T @ G


def hykkt_rhs(inst, gamma: float) -> np.ndarray:
    """r_gamma = r1 + H^T (D_s r4 - r2) + gamma G^T r3."""
    return condensed_rhs(inst) + gamma * inst.G_dense().T @ inst.r3


def schur_matrix(inst, gamma: float) -> np.ndarray:
    """S_gamma = G K_gamma^{-1} G^T, formed densely (tiny systems only)."""
    G = inst.G_dense()
    return G @ np.linalg.solve(hykkt_matrix(inst, gamma), G.T)


def hykkt_step_dense(inst, gamma: float):
    """HyKKT by dense block elimination of Eq. hykkt:
    S_gamma dy = r3 - G K_gamma^{-1} r_gamma (Eq. schurcomp);
    K_gamma dx = -r_gamma - G^T dy (reading R2 of the printed sign)."""
    G = inst.G_dense()
    Kg = hykkt_matrix(inst, gamma)
    rg = hykkt_rhs(inst, gamma)
    S = G @ np.linalg.solve(Kg, G.T)
    dy = np.linalg.solve(S, inst.r3 - G @ np.linalg.solve(Kg, rg)) if inst.m_e else np.zeros(0)
    dx = np.linalg.solve(Kg, -rg - G.T @ dy)
    ds, dz = recover_slack_dual(inst, dx)
    return dx, ds, dy, dz


def lifted_step_dense(inst):
    """Lifted-KKT (Eq. liftedkkt): K_k dx = -r1 - H^T(D_s r4 - r2); m_e = 0."""
    assert inst.m_e == 0
    dx = np.linalg.solve(condensed_matrix(inst), -condensed_rhs(inst))
    ds, dz = recover_slack_dual(inst, dx)
    return dx, ds, np.zeros(0), dz
