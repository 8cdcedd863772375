"""Distillation-column NLP of PAPER.md §VI.A: patterns and values.

Reading "A" of the model:

* stages t = 0..N, each with the 67 variables x_1..x_32, y_1..y_32, u, L, V
  (S_t = F + L_t eliminated symbolically), so n = 67(N+1) — Table I's n
   exactly;
* 66 equality rows per stage, stage-major: stage 0 = 32 initial conditions
  x_{n,0} = xbar_{n,0}, then for every stage the L-row L = uD, the
  V-row V = L + D, 32 VLE rows and, for t >= 1, the 32
  implicit-Euler material balances with Δt = 10/N;
* objective  sum_{t=1..N} w_x (x_{1,t} - xbar_1)^2 + rho (u_t - ubar)^2,
  w_x = 1000, rho = 1 (the paper calls w_x "gamma", renamed here
  because gamma is also the HyKKT parameter);
* bounds 1 <= u_t <= 5 for every stage, which enter the KKT system
  only through the barrier diagonal Sigma_x on the u entries.

Constants the paper does not state (C14): M_1 = M_32 = 5, other
M_n = 1; x_f = 0.5; xbar_1 = 0.98; ubar = 2; initial profile = steady state
at ubar.  The garbled reboiler balance is read as
  dx_32/dt = (S x_31 - (F - D) x_32 - V y_32) / M_32.

This module computes the model's residual g, Jacobian J = dg/dx, gradient of
f and Hessian of the Lagrangian W = ∇²f + Σ λ_r ∇²g_r.  None of that is the
method under test (condensation, Cholesky, CG, refinement live in oracle/ and
in the CUDA library); it is the problem data both sides consume.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

NV = 67  # variables per stage
NR = 66  # equality rows per stage
NT = 32  # trays
# variable offsets inside a stage
OX, OY, OU, OL, OV = 0, 32, 64, 65, 66


@dataclasses.dataclass(frozen=True)
class Params:
    alpha: float = 1.6        # relative volatility
    D: float = 0.2            # distillate flow
    F: float = 0.4            # feed flow
    w_x: float = 1000.0       # objective weight on x_1 (paper's "gamma")
    rho: float = 1.0          # objective weight on u
    horizon: float = 10.0     # Δt = 10/N
    feed_tray: int = 17
    x_f: float = 0.5          # unstated (C14)
    xbar1: float = 0.98       # unstated (C14)
    ubar: float = 2.0         # unstated (C14)
    u_lo: float = 1.0
    u_hi: float = 5.0

    def holdups(self) -> np.ndarray:
        M = np.ones(NT)
        M[0] = 5.0
        M[NT - 1] = 5.0
        return M


def dimensions(N: int) -> tuple[int, int]:
    """(n, m_e) = (67(N+1), 66(N+1)); n matches Table I."""
    return NV * (N + 1), NR * (N + 1)


def _stage_rows(t: int):
    """Row templates of stage t: list of (kind, tray) in row order."""
    rows = []
    if t == 0:
        rows += [("ic", k) for k in range(1, NT + 1)]
    rows += [("Lrow", 0), ("Vrow", 0)]
    rows += [("vle", k) for k in range(1, NT + 1)]
    if t >= 1:
        rows += [("bal", k) for k in range(1, NT + 1)]
    return rows


def _row_cols(kind: str, k: int):
    """Column offsets (relative to the stage base b = 67 t; -67+.. = previous
    stage) of one row, strictly increasing."""
    if kind == "ic":
        return [OX + k - 1]
    if kind == "Lrow":
        return [OU, OL]
    if kind == "Vrow":
        return [OL, OV]
    if kind == "vle":
        return [OX + k - 1, OY + k - 1]
    # balance row of tray k at stage t >= 1
    prev = -NV + OX + k - 1
    if k == 1:
        return [prev, OX + 0, OY + 1, OV]
    if k == NT:
        return [prev, OX + NT - 2, OX + NT - 1, OY + NT - 1, OL, OV]
    return [prev, OX + k - 2, OX + k - 1, OY + k - 1, OY + k, OL, OV]


def _w_stage_entries(t: int):
    """Lower-triangular W entries (row_off, col_off) of stage t, row >= col."""
    ent = [(OX + k, OX + k) for k in range(NT)]
    if t >= 1:
        ent.append((OU, OU))
        ent += [(OL, OX + k) for k in range(NT - 1)]          # (L, x_1..x_31)
        ent.append((OV, OX + 0))                              # (V, x_1)
        ent += [(OV, OY + k) for k in range(1, NT)]           # (V, y_2..y_32)
    return ent


@dataclasses.dataclass
class Pattern:
    N: int
    n: int
    m: int
    w_row: np.ndarray   # int32 [nnz_W], lower triangle (row >= col)
    w_col: np.ndarray
    j_rowptr: np.ndarray  # int32 [m+1], CSR of J = dg/dx
    j_col: np.ndarray     # int32 [nnz_J], strictly increasing per row


def build_pattern(N: int) -> Pattern:
    if N < 1:
        raise ValueError("N >= 1 required")
    n, m = dimensions(N)
    # J pattern
    row_lens0 = [len(_row_cols(*r)) for r in _stage_rows(0)]
    row_lens1 = [len(_row_cols(*r)) for r in _stage_rows(1)]
    cols0 = np.concatenate([np.array(_row_cols(*r)) for r in _stage_rows(0)])
    cols1 = np.concatenate([np.array(_row_cols(*r)) for r in _stage_rows(1)])
    nnz0, nnz1 = len(cols0), len(cols1)
    base = (np.arange(1, N + 1) * NV)[:, None]
    j_col = np.concatenate([cols0, (cols1[None, :] + base).ravel()]).astype(np.int32)
    lens = np.concatenate([np.array(row_lens0), np.tile(np.array(row_lens1), N)])
    j_rowptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(lens, out=j_rowptr[1:])
    assert j_rowptr[-1] == nnz0 + N * nnz1 == 288 * N + 100
    # W pattern (sorted by (row, col) within the whole matrix for determinism)
    w0 = np.array(_w_stage_entries(0))
    w1 = np.array(_w_stage_entries(1))
    w_all = np.concatenate([w0, (w1[None, :, :] + np.arange(1, N + 1)[:, None, None] * NV).reshape(-1, 2)])
    order = np.lexsort((w_all[:, 1], w_all[:, 0]))
    w_all = w_all[order]
    return Pattern(N=N, n=n, m=m,
                   w_row=w_all[:, 0].astype(np.int32), w_col=w_all[:, 1].astype(np.int32),
                   j_rowptr=j_rowptr.astype(np.int32), j_col=j_col)


class Model:
    """Values of the distillation NLP at a full variable vector v (length n)."""

    def __init__(self, N: int, params: Params = Params()):
        self.N = N
        self.p = params
        self.pat = build_pattern(N)
        self.n, self.m = self.pat.n, self.pat.m
        self.dt = params.horizon / N
        self.M = params.holdups()
        # permutation that maps the W entry order produced by _w_values (stage-major,
        # template order) to the sorted pattern order of build_pattern
        w0 = np.array(_w_stage_entries(0))
        w1 = np.array(_w_stage_entries(1))
        w_all = np.concatenate([w0, (w1[None, :, :] + np.arange(1, N + 1)[:, None, None] * NV).reshape(-1, 2)])
        self._w_order = np.lexsort((w_all[:, 1], w_all[:, 0]))

    # ---- helpers -------------------------------------------------------
    def split(self, v: np.ndarray):
        S = v.reshape(self.N + 1, NV)
        return S[:, OX:OX + NT], S[:, OY:OY + NT], S[:, OU], S[:, OL], S[:, OV]

    def vle(self, x):
        a = self.p.alpha
        return a * x / (1.0 + (a - 1.0) * x)

    def vle_d1(self, x):
        a = self.p.alpha
        return a / (1.0 + (a - 1.0) * x) ** 2

    def vle_d2(self, x):
        a = self.p.alpha
        return -2.0 * a * (a - 1.0) / (1.0 + (a - 1.0) * x) ** 3

    def xdot(self, x, y, L, V):
        """Right-hand sides of the material balances, arrays [..., 32]."""
        p, M = self.p, self.M
        S = p.F + L
        L = np.asarray(L)[..., None]
        V = np.asarray(V)[..., None]
        S = np.asarray(S)[..., None]
        xd = np.empty_like(x)
        xd[..., 0] = V[..., 0] * (y[..., 1] - x[..., 0]) / M[0]
        k = np.arange(1, 16)  # trays 2..16
        xd[..., k] = (L * (x[..., k - 1] - x[..., k]) - V * (y[..., k] - y[..., k + 1])) / M[k]
        f = p.feed_tray - 1
        xd[..., f] = (p.F * p.x_f + L[..., 0] * x[..., f - 1] - S[..., 0] * x[..., f]
                      - V[..., 0] * (y[..., f] - y[..., f + 1])) / M[f]
        k = np.arange(17, 31)  # trays 18..31
        xd[..., k] = (S * (x[..., k - 1] - x[..., k]) - V * (y[..., k] - y[..., k + 1])) / M[k]
        xd[..., 31] = (S[..., 0] * x[..., 30] - (p.F - p.D) * x[..., 31] - V[..., 0] * y[..., 31]) / M[31]
        return xd

    def xdot_jac(self, x, u):
        """d xdot / d x with y = VLE(x) eliminated; dense [..., 32, 32]."""
        p, M = self.p, self.M
        L = u * p.D
        V = L + p.D
        S = p.F + L
        yp = self.vle_d1(x)
        Jm = np.zeros(x.shape + (NT,))
        Jm[..., 0, 0] = -V / M[0]
        Jm[..., 0, 1] = V * yp[..., 1] / M[0]
        for k in range(1, NT):
            flow = L if k < p.feed_tray - 1 else S  # trays 2..16 use L; 17 uses L on x16
            if k == p.feed_tray - 1:
                Jm[..., k, k - 1] = L / M[k]
                Jm[..., k, k] = (-S - V * yp[..., k]) / M[k]
            elif k == NT - 1:
                Jm[..., k, k - 1] = S / M[k]
                Jm[..., k, k] = (-(p.F - p.D) - V * yp[..., k]) / M[k]
                continue
            else:
                Jm[..., k, k - 1] = flow / M[k]
                Jm[..., k, k] = (-flow - V * yp[..., k]) / M[k]
            Jm[..., k, k + 1] = V * yp[..., k + 1] / M[k]
        return Jm

    # ---- simulation (implicit Euler) -----------------------------
    def steady_state(self, u: float) -> np.ndarray:
        """Steady state profile x (32,) at constant u, by pseudo-transient
        continuation (implicit Euler with growing steps) + Newton."""
        x = np.full(NT, 0.5)
        for h in [0.1, 1.0, 10.0, 100.0, 1e3, 1e4, 1e6, 1e9, 1e12, 1e15]:
            for _ in range(60):
                xd = self.xdot(x, self.vle(x), u * self.p.D, u * self.p.D + self.p.D)
                r = (x - x) / h - xd
                Jn = np.eye(NT) / h - self.xdot_jac(x, u)
                dx = np.linalg.solve(Jn, -r)
                x = np.clip(x + dx, 1e-6, 1 - 1e-6)
                if np.max(np.abs(dx)) < 1e-15:
                    break
        res = self.xdot(x, self.vle(x), u * self.p.D, u * self.p.D + self.p.D)
        assert np.max(np.abs(res)) < 1e-10, res
        return x

    def simulate(self, x0: np.ndarray, u: np.ndarray) -> np.ndarray:
        """Implicit-Euler trajectory X[t] (t = 0..N) from x0 under controls u[t]."""
        N, dt = self.N, self.dt
        X = np.empty((N + 1, NT))
        X[0] = x0
        x = x0.copy()
        for t in range(1, N + 1):
            xprev = X[t - 1]
            L = u[t] * self.p.D
            V = L + self.p.D
            for _ in range(20):
                r = (x - xprev) / dt - self.xdot(x, self.vle(x), L, V)
                Jn = np.eye(NT) / dt - self.xdot_jac(x, u[t])
                dx = np.linalg.solve(Jn, -r)
                x = x + dx
                if np.max(np.abs(dx)) < 1e-14:
                    break
            X[t] = x
        return X

    def full_vector(self, X: np.ndarray, u: np.ndarray) -> np.ndarray:
        """Assemble v with y, L, V from the algebraic rows."""
        v = np.empty((self.N + 1, NV))
        v[:, OX:OX + NT] = X
        v[:, OY:OY + NT] = self.vle(X)
        v[:, OU] = u
        v[:, OL] = u * self.p.D
        v[:, OV] = v[:, OL] + self.p.D
        return v.ravel()

    # ---- residual, Jacobian, gradient, Hessian --------------------------
    def residual(self, v: np.ndarray, xbar0: np.ndarray) -> np.ndarray:
        x, y, u, L, V = self.split(v)
        p = self.p
        g = np.empty((self.N + 1, NR))
        # stage 0: IC rows then L, V, VLE
        g0 = np.concatenate([x[0] - xbar0, [L[0] - u[0] * p.D, V[0] - L[0] - p.D], y[0] - self.vle(x[0])])
        out = [g0]
        if self.N >= 1:
            xd = self.xdot(x[1:], y[1:], L[1:], V[1:])
            bal = (x[1:] - x[:-1]) / self.dt - xd
            rest = np.concatenate([(L[1:] - u[1:] * p.D)[:, None], (V[1:] - L[1:] - p.D)[:, None],
                                   y[1:] - self.vle(x[1:]), bal], axis=1)
            out.append(rest.ravel())
        g = np.concatenate(out)
        assert g.shape == (self.m,)
        return g

    def jacobian_values(self, v: np.ndarray) -> np.ndarray:
        """Values of J in the CSR order of build_pattern (row-major, cols increasing)."""
        x, y, u, L, V = self.split(v)
        p, M, dt = self.p, self.M, self.dt
        N = self.N
        # stage 0
        s0 = [np.ones(NT), [-p.D, 1.0], [-1.0, 1.0]]
        vle0 = np.stack([-self.vle_d1(x[0]), np.ones(NT)], axis=1).ravel()
        out0 = np.concatenate([s0[0], s0[1], s0[2], vle0])
        if N == 0:
            return out0
        T = slice(1, N + 1)
        xs, ys, Ls, Vs = x[T], y[T], L[T], V[T]
        S = p.F + Ls
        one = np.ones(N)
        blocks = [np.stack([-p.D * one, one], 1), np.stack([-one, one], 1)]
        vle = np.stack([-self.vle_d1(xs), np.ones_like(xs)], axis=2).reshape(N, 2 * NT)
        blocks.append(vle)
        # balances
        bal = []
        k = 0  # tray 1: [x1-, x1, y2, V]
        bal.append(np.stack([-one / dt, 1 / dt + Vs / M[0], -Vs / M[0], -(ys[:, 1] - xs[:, 0]) / M[0]], 1))
        for k in range(1, NT - 1):
            if k < p.feed_tray - 1:       # trays 2..16: flow L
                flow = Ls
            elif k == p.feed_tray - 1:    # feed tray 17: L on x16, S on x17
                flow = None
            else:                          # trays 18..31: flow S
                flow = S
            if flow is None:
                c_prev_tray = -Ls / M[k]
                c_self = 1 / dt + S / M[k]
            else:
                c_prev_tray = -flow / M[k]
                c_self = 1 / dt + flow / M[k]
            bal.append(np.stack([-one / dt, c_prev_tray, c_self, Vs / M[k], -Vs / M[k],
                                 -(xs[:, k - 1] - xs[:, k]) / M[k],
                                 (ys[:, k] - ys[:, k + 1]) / M[k]], 1))
        k = NT - 1  # reboiler: [x32-, x31, x32, y32, L, V]
        bal.append(np.stack([-one / dt, -S / M[k], (1 / dt + (p.F - p.D) / M[k]) * one, Vs / M[k],
                             -xs[:, k - 1] / M[k], ys[:, k] / M[k]], 1))
        blocks += bal
        rest = np.concatenate(blocks, axis=1)
        assert rest.shape == (N, 288)
        return np.concatenate([out0, rest.ravel()])

    def grad_f(self, v: np.ndarray) -> np.ndarray:
        x, y, u, L, V = self.split(v)
        g = np.zeros((self.N + 1, NV))
        g[1:, OX] = 2 * self.p.w_x * (x[1:, 0] - self.p.xbar1)
        g[1:, OU] = 2 * self.p.rho * (u[1:] - self.p.ubar)
        return g.ravel()

    def objective(self, v: np.ndarray) -> float:
        x, y, u, L, V = self.split(v)
        return float(np.sum(self.p.w_x * (x[1:, 0] - self.p.xbar1) ** 2 + self.p.rho * (u[1:] - self.p.ubar) ** 2))

    def hessian_values(self, v: np.ndarray, lam: np.ndarray, obj_weight: float = 1.0) -> np.ndarray:
        """W = obj_weight ∇²f + Σ_r λ_r ∇²g_r in the sorted lower pattern order of build_pattern."""
        x, y, u, L, V = self.split(v)
        p, M, N = self.p, self.M, self.N
        lam = lam.reshape(N + 1, NR)
        # multipliers of VLE rows and balance rows per stage
        lv = np.empty((N + 1, NT))
        lv[0] = lam[0, NT + 2:NT + 2 + NT]
        lv[1:] = lam[1:, 2:2 + NT]
        lb = lam[1:, 2 + NT:2 + 2 * NT]  # [N, 32]
        vals = []
        # stage 0: (x_n, x_n) VLE curvature. g_vle = y - vle(x) -> d2 = -vle''
        vals.append(-lv[0] * self.vle_d2(x[0]))
        if N >= 1:
            xs = x[1:]
            dxx = -lv[1:] * self.vle_d2(xs)
            dxx[:, 0] += 2 * p.w_x * obj_weight
            duu = np.full(N, 2 * p.rho * obj_weight)
            # (L, x_k), k = 1..31 (0-based 0..30)
            dLx = np.zeros((N, NT - 1))
            for k0 in range(NT - 1):         # x_{k0+1}
                n_next = k0 + 1               # tray index (0-based) of row n = k+1
                dLx[:, k0] += -lb[:, n_next] / M[n_next]      # (L, x_{n-1}) of row n, n = 2..32
                if 1 <= k0 <= NT - 2:
                    dLx[:, k0] += lb[:, k0] / M[k0]           # (L, x_n) of row n, n = 2..31
            dVx1 = lb[:, 0] / M[0]
            dVy = np.zeros((N, NT - 1))       # (V, y_k), k = 2..32
            for k0 in range(1, NT):
                j = k0 - 1
                if k0 == 1:
                    dVy[:, j] += -lb[:, 0] / M[0]             # condenser (V, y2)
                dVy[:, j] += lb[:, k0] / M[k0]                # (V, y_n) of row n
                if k0 >= 2:
                    dVy[:, j] += -lb[:, k0 - 1] / M[k0 - 1]   # (V, y_{n+1}) of row n = k-1
            stage = np.concatenate([dxx, duu[:, None], dLx, dVx1[:, None], dVy], axis=1)
            vals.append(stage.ravel())
        w = np.concatenate(vals)
        return w[self._w_order]


# ---------------------------------------------------------------------------
# Synthetic interior-point iterates (DESIGN.md §3 "input recipe")
# ---------------------------------------------------------------------------
TAU = 1e-6          # Lifted-KKT relaxation


def mu_schedule(mu0: float = 0.1, tol: float = 1e-6, kappa: float = 0.2, theta: float = 1.5):
    """Monotone barrier schedule mu' = max(tol/10, min(kappa mu, mu^theta))
     from mu0 down to tol/10."""
    mus = [mu0]
    while mus[-1] > tol / 10 * (1 + 1e-12):
        mu = mus[-1]
        mus.append(max(tol / 10, min(kappa * mu, mu ** theta)))
    return mus


@dataclasses.dataclass
class Iterate:
    mu: float
    v: np.ndarray        # primal point (n)
    lam: np.ndarray      # equality multipliers (m)
    w_val: np.ndarray    # W values (nnz_W)
    j_val: np.ndarray    # J values (nnz_J)
    sigma_x: np.ndarray  # barrier diagonal (n), nonzero on u only
    d_lifted: np.ndarray # slack diagonal D of the relaxed rows (m), Lifted-KKT


MAX_GRADIENT = 100.0  # gradient-based NLP scaling of MadNLP/Ipopt (reading R14)


class Instance:
    """One NMPC instance (initial state seeded by 1000 + i) with its base
    trajectory, multipliers and IPM-like iterates.

    scaled=True (default, reading R14): the iterates are those of the gradient-scaled NLP that an
    Ipopt-style solver such as MadNLP factorizes by default (P:62 cites [wachter2006implementation];
    the paper only sets tol and gamma): objective scale s_f = min(1, 100/||grad f(x0)||_inf) and
    constraint row scales s_r = min(1, 100/||grad g_r(x0)||_inf), fixed at the base point.  J rows
    are multiplied by s_r, the multipliers are those of the scaled problem and
    W = s_f grad^2 f + sum_r lam_r s_r grad^2 g_r."""

    def __init__(self, N: int, instance: int = 0, params: Params = Params(), lsqr_iters: int = 60,
                 scaled: bool = True):
        self.model = Model(N, params)
        md = self.model
        p = params
        xs = md.steady_state(p.ubar)
        rng = np.random.default_rng(1000 + instance)
        self.xbar0 = np.clip(xs + 0.05 * rng.uniform(-1, 1, NT), 0.01, 0.99)
        tt = np.arange(N + 1) * md.dt
        phase = 2 * math.pi * rng.uniform()
        self.u = p.ubar + 0.5 * np.sin(0.7 * tt + phase)
        X = md.simulate(self.xbar0, self.u)
        self.v = md.full_vector(X, self.u)
        # equality multipliers: least squares on ∇f + Jᵀλ = 0 (fixed LSQR budget)
        from scipy.sparse import csr_matrix
        from scipy.sparse.linalg import lsqr
        pat = md.pat
        jv = md.jacobian_values(self.v)
        self.rows_of_entries = np.repeat(np.arange(md.m), np.diff(pat.j_rowptr))
        if scaled:
            rowmax = np.zeros(md.m)
            np.maximum.at(rowmax, self.rows_of_entries, np.abs(jv))
            self.row_scale = np.minimum(1.0, MAX_GRADIENT / np.maximum(rowmax, 1e-300))
            gmax = np.abs(md.grad_f(self.v)).max()
            self.obj_scale = min(1.0, MAX_GRADIENT / gmax) if gmax > 0 else 1.0
        else:
            self.row_scale = np.ones(md.m)
            self.obj_scale = 1.0
        J = csr_matrix((jv * self.row_scale[self.rows_of_entries], pat.j_col, pat.j_rowptr), shape=(md.m, md.n))
        self.lam = lsqr(J.T.tocsr(), -self.obj_scale * md.grad_f(self.v), atol=0, btol=0, iter_lim=lsqr_iters)[0]
        self.instance = instance

    def iterate(self, k: int, mu: float) -> Iterate:
        md = self.model
        p = md.p
        rng = np.random.default_rng(2000 + 7919 * self.instance + k)
        scale = 1e-2 * math.sqrt(mu / 0.1)
        v = self.v.copy().reshape(md.N + 1, NV)
        v[:, OX:OX + NT] = np.clip(v[:, OX:OX + NT] + scale * rng.standard_normal((md.N + 1, NT)), 1e-3, 1 - 1e-3)
        v[:, OY:OY + NT] = np.clip(v[:, OY:OY + NT] + scale * rng.standard_normal((md.N + 1, NT)), 1e-3, 1 - 1e-3)
        v[:, OU] = np.clip(v[:, OU] + scale * rng.standard_normal(md.N + 1), p.u_lo + 0.05, p.u_hi - 0.05)
        v = v.ravel()
        lam = self.lam + 0.1 * rng.standard_normal(md.m)
        sigma = np.zeros((md.N + 1, NV))
        u = v.reshape(md.N + 1, NV)[:, OU]
        sigma[:, OU] = mu / (u - p.u_lo) ** 2 + mu / (p.u_hi - u) ** 2
        s = 0.9 * TAU * rng.uniform(-1, 1, md.m)
        d = mu / (s + TAU) ** 2 + mu / (TAU - s) ** 2
        rs = self.row_scale
        return Iterate(mu=mu, v=v, lam=lam, w_val=md.hessian_values(v, lam * rs, self.obj_scale),
                       j_val=md.jacobian_values(v) * rs[self.rows_of_entries], sigma_x=sigma.ravel(), d_lifted=d)

    def trajectory(self, per_mu: int = 3):
        """~18 iterates: 3 per barrier value of mu_schedule()."""
        out = []
        k = 0
        for mu in mu_schedule():
            for _ in range(per_mu):
                out.append(self.iterate(k, mu))
                k += 1
        return out


def random_rhs(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal(n)


class NLP:
    """The (gradient-scaled, reading R14) distillation NLP of one instance as the callbacks the IPM
    driver (paper_2403_15913_b200/ipm.py) needs: min s_f f(v) s.t. S_r c(v) = 0, u_lo <= u <= u_hi."""

    def __init__(self, inst: "Instance"):
        from scipy.sparse import csr_matrix
        md = inst.model
        self.inst, self.md = inst, md
        self.n, self.m = md.n, md.m
        self.pat = md.pat
        self.bidx = np.arange(md.N + 1) * NV + OU
        self.lo = np.full(md.N + 1, md.p.u_lo)
        self.hi = np.full(md.N + 1, md.p.u_hi)
        self.x0 = inst.v.copy()
        self.lam0 = inst.lam.copy()
        self.sf, self.rs = inst.obj_scale, inst.row_scale
        self._rse = inst.row_scale[inst.rows_of_entries]
        self._csr = lambda jv: csr_matrix((jv, self.pat.j_col, self.pat.j_rowptr), shape=(md.m, md.n))

    def f(self, v):
        return self.sf * self.md.objective(v)

    def grad_f(self, v):
        return self.sf * self.md.grad_f(v)

    def c(self, v):
        return self.rs * self.md.residual(v, self.inst.xbar0)

    def jac(self, v):
        return self.md.jacobian_values(v) * self._rse

    def jac_t(self, v, jv, y):
        return self._csr(jv).T @ y

    def hess(self, v, lam):
        return self.md.hessian_values(v, lam * self.rs, self.sf)
