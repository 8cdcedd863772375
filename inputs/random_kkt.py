"""Small random saddle-point instances for unit tests (seeded).

An instance carries the inputs of one Newton-step solve of P:179-201:
W (sparse symmetric, indefinite), G (m_e x n), H (m_i x n), Sigma_x (n),
D_s (m_i, > 0), delta_x, and right-hand sides r1..r4.  Instances satisfy
LICQ (G full row rank) and SOSC on null(G) by construction: W's
diagonal is shifted until Z^T (W + Sigma + delta I + H^T D_s H) Z >= margin,
which keeps W itself indefinite in general.  This is test-data generation,
not the method: the dense linear algebra used here only *certifies* the
assumptions.
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass
class KKTInstance:
    n: int
    m_e: int
    m_i: int
    w_row: np.ndarray   # lower COO (row >= col), int32
    w_col: np.ndarray
    w_val: np.ndarray
    g_rowptr: np.ndarray
    g_col: np.ndarray
    g_val: np.ndarray
    h_rowptr: np.ndarray
    h_col: np.ndarray
    h_val: np.ndarray
    sigma_x: np.ndarray
    d_s: np.ndarray
    delta_x: float
    r1: np.ndarray
    r2: np.ndarray
    r3: np.ndarray
    r4: np.ndarray

    def W_dense(self) -> np.ndarray:
        W = np.zeros((self.n, self.n))
        for r, c, v in zip(self.w_row, self.w_col, self.w_val):
            W[r, c] += v
            if r != c:
                W[c, r] += v
        return W

    def G_dense(self) -> np.ndarray:
        return _csr_dense(self.m_e, self.n, self.g_rowptr, self.g_col, self.g_val)

    def H_dense(self) -> np.ndarray:
        return _csr_dense(self.m_i, self.n, self.h_rowptr, self.h_col, self.h_val)


def _csr_dense(m, n, rp, ci, v):
    A = np.zeros((m, n))
    for i in range(m):
        for p in range(rp[i], rp[i + 1]):
            A[i, ci[p]] += v[p]
    return A


def _dense_to_csr(A):
    m, n = A.shape
    rp = [0]
    ci, vv = [], []
    for i in range(m):
        nz = np.nonzero(A[i])[0]
        ci += list(nz)
        vv += list(A[i, nz])
        rp.append(len(ci))
    return (np.array(rp, dtype=np.int32), np.array(ci, dtype=np.int32), np.array(vv, dtype=np.float64))


def random_instance(n: int, m_e: int, m_i: int, seed: int, density: float = 0.3,
                    sigma_range=(1e-2, 1e2), d_range=(1e-2, 1e2), margin: float = 1e-1,
                    delta_x: float = 0.0) -> KKTInstance:
    """Random instance with LICQ + SOSC.  sigma/d ranges are log-uniform."""
    rng = np.random.default_rng(seed)
    # G: full row rank, sparse: one guaranteed "pivot" column per row
    G = np.zeros((m_e, n))
    piv = rng.permutation(n)[:m_e]
    for i in range(m_e):
        mask = rng.uniform(size=n) < density
        G[i, mask] = rng.standard_normal(mask.sum())
        G[i, piv[i]] = 2.0 + rng.uniform()
    H = np.zeros((m_i, n))
    for i in range(m_i):
        mask = rng.uniform(size=n) < density
        mask[rng.integers(n)] = True
        H[i, mask] = rng.standard_normal(mask.sum())
    W = np.zeros((n, n))
    for i in range(n):
        for j in range(i):
            if rng.uniform() < density:
                W[i, j] = W[j, i] = rng.standard_normal()
        W[i, i] = rng.standard_normal()
    sigma = np.exp(rng.uniform(np.log(sigma_range[0]), np.log(sigma_range[1]), n)) if sigma_range else np.zeros(n)
    d = np.exp(rng.uniform(np.log(d_range[0]), np.log(d_range[1]), m_i))
    K = W + np.diag(sigma) + delta_x * np.eye(n) + H.T @ (d[:, None] * H)
    if m_e > 0:
        _, _, vt = np.linalg.svd(G)
        Z = vt[m_e:].T
    else:
        Z = np.eye(n)
    lam_min = np.linalg.eigvalsh(Z.T @ K @ Z).min() if Z.shape[1] > 0 else margin
    if lam_min < margin:
        shift = margin - lam_min
        W += shift * np.eye(n)
    rows, cols = np.nonzero(np.tril(W))
    # include the full diagonal in the pattern (explicit zeros allowed)
    diag_missing = [i for i in range(n) if W[i, i] == 0.0]
    rows = np.concatenate([rows, diag_missing]).astype(np.int32)
    cols = np.concatenate([cols, diag_missing]).astype(np.int32)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    gr = _dense_to_csr(G)
    hr = _dense_to_csr(H)
    return KKTInstance(n=n, m_e=m_e, m_i=m_i,
                       w_row=rows, w_col=cols, w_val=W[rows, cols].copy(),
                       g_rowptr=gr[0], g_col=gr[1], g_val=gr[2],
                       h_rowptr=hr[0], h_col=hr[1], h_val=hr[2],
                       sigma_x=sigma, d_s=d, delta_x=delta_x,
                       r1=rng.standard_normal(n), r2=rng.standard_normal(m_i),
                       r3=rng.standard_normal(m_e), r4=rng.standard_normal(m_i))
