"""Interior-point loop around the C ABI (host driver, not the hot path).

The paper runs MadNLP's filter line-search interior-point method ([17] = Wächter and
Biegler) with the condensed-KKT Newton step on the GPU.  This module is that loop for NLPs of the
form  min f(v)  s.t.  c(v) = 0,  lo <= v_B <= hi  (bounds on a subset B of the variables),
with the per-iteration linear algebra entirely in libckkt — HyKKT (GpuKKT: m_e = m, m_i = 0), or Lifted-KKT
on the relaxed problem of P:333-346 (LiftedNLP + LiftedGpuKKT: m_e = 0, every row relaxed with a slack):

  * inertia correction: ckkt_refactor_inertia (reading R15);
  * Newton step: ckkt_solve of  [W + Sigma_x + delta_x I, J^T; J, 0] [dx; dlam] = -[r1; r3]  with
    r1 = grad f + J^T lam - mu/(v_B - lo) + mu/(hi - v_B)  (primal-dual barrier gradient)
    and Sigma_x = z_L/(v_B - lo) + z_U/(hi - v_B);
  * step lengths: ckkt_fraction_to_boundary on the bound slacks and on the bound duals (tau =
    max(0.99, 1 - mu));
  * line search: the Wächter–Biegler filter (switching condition, Armijo on the barrier objective,
    sufficient decrease of theta = ||c||_1 or phi, filter augmentation), without second-order
    corrections or feasibility restoration (a step below alpha_min stops with status "restoration");
  * barrier update (SPEC update_mu): mu' = max(tol/10, min(0.2 mu, mu^1.5)) once
    E_mu <= 10 mu; stop when E_0 <= tol (tol = 1e-6).

Host arithmetic here is O(n) vector bookkeeping in numpy on iterates copied back from the device;
the model evaluation (f, c, J, W) is the caller's `problem`: the host model (inputs.distillation.NLP) or
DeviceDistillationNLP, whose J and W come from the GPU kernel ckkt_distillation_eval (NEXT-4) and go to
the KKT solve without leaving the device (general AD as in ExaModels is out of scope, §8(f) 4).
"""
from __future__ import annotations

import dataclasses
import math
import warnings

import numpy as np

# Wächter–Biegler constants ([17], Ipopt defaults)
GAMMA_THETA, GAMMA_PHI, DELTA_SW, S_THETA, S_PHI, ETA_PHI = 1e-5, 1e-5, 1.0, 1.1, 2.3, 1e-4
KAPPA_EPS, KAPPA_MU, THETA_MU, KAPPA_SIGMA = 10.0, 0.2, 1.5, 1e10


@dataclasses.dataclass
class IPMResult:
    status: str                 # "converged" | "max_iter" | "restoration" | "inertia_failure" | "linear_solver_failure"
    iterations: int
    v: np.ndarray
    lam: np.ndarray
    z_lo: np.ndarray
    z_hi: np.ndarray
    objective: float
    kkt_error: float
    history: list               # per iteration: dict(mu, theta, phi, alpha, delta_x, k_cg, trials, ls)


class GpuKKT:
    """The per-iteration solve through libckkt (HyKKT).  refactor(w, j, sigma, delta_last) ->
    (ok, delta, trials); solve(r1, r3) -> (dx, dlam, info)."""

    def __init__(self, n, m, w_row, w_col, j_rowptr, j_col, gamma=1e7, leaf=64, device=0):
        import torch
        from . import ckkt
        self.torch, self.ckkt = torch, ckkt
        self.dev = torch.device("cuda", device)
        self.n, self.m = n, m
        self.ctx = ckkt.Context(n, m, 0, w_row, w_col, j_rowptr, j_col, None, None, strategy=ckkt.CKKT_HYKKT,
                                gamma=gamma, leaf=leaf, device=device,
                                stream=torch.cuda.current_stream(self.dev).cuda_stream)
        self.delta = torch.zeros(1, dtype=torch.float64, device=self.dev)

    def _t(self, a):
        if isinstance(a, self.torch.Tensor):  # device values (DeviceDistillationNLP): no host round trip
            return a.to(device=self.dev, dtype=self.torch.float64).contiguous()
        return self.torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=self.dev)

    def refactor(self, w_val, j_val, sigma_x, delta_last):
        self._vals = [self._t(w_val), self._t(j_val), None, self._t(sigma_x), None]  # zero-copy: keep alive
        rc, d, t = self.ctx.refactor_inertia(*self._vals, self.delta, np.array([delta_last]))
        return rc == self.ckkt.CKKT_OK, float(d[0]), int(t[0])

    def solve(self, r1, r3):
        T = self.torch
        dx = T.empty(self.n, dtype=T.float64, device=self.dev)
        dy = T.empty(self.m, dtype=T.float64, device=self.dev)
        rc, info = self.ctx.solve(self._t(r1), None, self._t(r3), None, dx, None, dy, None)
        # CG / refinement non-convergence still returns the best iterate (include/ckkt.h); reported per step
        return dx.cpu().numpy(), dy.cpu().numpy(), dict(info[0], rc=int(rc))

    def fraction_to_boundary(self, s, ds, tau):
        a = self.ckkt.fraction_to_boundary(self._t(s), self._t(ds), tau)
        return float(a.cpu().numpy()[0])


def transpose_pattern(j_rowptr, j_col, n):
    """CSR pattern of J^T from J's (rowptr, col): (ptr [n+1], col [nnz] = J's row of each entry, perm [nnz])
    with values_T = values_J[perm] (entries of a J column in increasing row order)."""
    j_rowptr, j_col = np.asarray(j_rowptr), np.asarray(j_col)
    rows = np.repeat(np.arange(j_rowptr.size - 1), np.diff(j_rowptr))
    perm = np.lexsort((rows, j_col))
    ptr = np.concatenate([[0], np.cumsum(np.bincount(j_col, minlength=n))])
    return ptr, rows[perm], perm


class DeviceDistillationNLP:
    """The distillation NLP with its derivatives evaluated on the GPU (the
    paper evaluates the model with ExaModels on the device, so J and W never cross to the host).  Same
    callbacks as the host model `base` (inputs.distillation.NLP), except that jac / hess return device
    tensors from ckkt_distillation_eval, which GpuKKT / LiftedGpuKKT hand to libckkt without a copy; c and
    grad_f are evaluated on the device and copied back (O(n) vectors for the line search); J^T y is a
    device CSR product of the transposed pattern (host-driver bookkeeping, not the hot path); f stays the
    host objective of `base`."""

    def __init__(self, base, device=0):
        import torch
        from . import ckkt
        inst = base.inst
        self.base, self.torch, self.ckkt = base, torch, ckkt
        self.dev = torch.device("cuda", device)
        self.N, self.params = base.md.N, base.md.p
        self.n, self.m, self.pat = base.n, base.m, base.pat
        self.bidx, self.lo, self.hi = base.bidx, base.lo, base.hi
        self.x0, self.lam0 = base.x0.copy(), base.lam0.copy()
        T = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=self.dev)
        self._T = T
        self._xbar0, self._rs, self._sf = T(inst.xbar0), T(inst.row_scale), float(inst.obj_scale)
        t_ptr, t_col, perm = transpose_pattern(self.pat.j_rowptr, self.pat.j_col, self.n)
        self._t_ptr, self._t_col, self._t_perm = (T(a, torch.int64) for a in (t_ptr, t_col, perm))

    def _eval(self, v, lam=None, j=False, w=False, c=False, g=False):
        torch = self.torch
        e = lambda k: torch.empty(k, dtype=torch.float64, device=self.dev)
        out = dict(j=e(self.pat.j_col.size) if j else None, w=e(self.pat.w_row.size) if w else None,
                   c=e(self.m) if c else None, g=e(self.n) if g else None)
        self.ckkt.distillation_eval(self.N, self.params, self._xbar0, self._T(v), None if lam is None else self._T(lam),
                                    self._rs, self._sf, out["j"], out["w"], out["c"], out["g"])
        return out

    def f(self, v):
        return self.base.f(v)

    def grad_f(self, v):
        return self._eval(v, g=True)["g"].cpu().numpy()

    def c(self, v):
        return self._eval(v, c=True)["c"].cpu().numpy()

    def jac(self, v):
        return self._eval(v, j=True)["j"]

    def jac_t(self, v, jv, y):
        torch = self.torch
        vals = self._T(jv) if not isinstance(jv, torch.Tensor) else jv
        with warnings.catch_warnings():  # (torch's "sparse CSR is beta" notice)
            warnings.simplefilter("ignore", UserWarning)
            jt = torch.sparse_csr_tensor(self._t_ptr, self._t_col, vals[self._t_perm], size=(self.n, self.m),
                                         check_invariants=False)
            return (jt @ self._T(y)).cpu().numpy()

    def hess(self, v, lam):
        return self._eval(v, lam=lam, w=True)["w"]


class LiftedNLP:
    """The relaxed problem of Lifted-KKT (Eq. problemrelaxation): min f(v) s.t. -tau <= c(v) <= tau
    and the variable bounds, written with one slack per row as an NLP in w = (v, s):
        min f(v)  s.t.  c(v) + s = 0,  lo <= v_B <= hi,  -tau <= s <= tau      (tau = 1e-6).
    Its primal-dual Newton system [W + Sigma_v, 0, J^T; 0, Sigma_s, I; J, I, 0] is exactly the ABI's K_aug
    of the Lifted strategy with H = J and D_s = Sigma_s (LiftedGpuKKT maps the calls), so solve_nlp
    drives it unchanged: the slack rows of the gradient become r2, the constraint residual c + s becomes
    r4, the multipliers of the relaxed rows are the ABI's dz."""

    def __init__(self, nlp, tau=1e-6):
        self.base, self.tau = nlp, tau
        n, m = nlp.n, nlp.m
        self.nv, self.m = n, m
        self.n = n + m
        self.pat = nlp.pat
        self.bidx = np.concatenate([nlp.bidx, n + np.arange(m)])
        self.lo = np.concatenate([nlp.lo, np.full(m, -tau)])
        self.hi = np.concatenate([nlp.hi, np.full(m, tau)])
        s0 = np.clip(-nlp.c(nlp.x0), -0.9 * tau, 0.9 * tau)  # feasible start: s = -c(x0) inside the box
        self.x0 = np.concatenate([nlp.x0, s0])
        self.lam0 = nlp.lam0.copy()

    def f(self, w):
        return self.base.f(w[:self.nv])

    def grad_f(self, w):
        return np.concatenate([self.base.grad_f(w[:self.nv]), np.zeros(self.m)])

    def c(self, w):
        return self.base.c(w[:self.nv]) + w[self.nv:]

    def jac(self, w):  # values of J (the slack part of [J I] is the identity)
        return self.base.jac(w[:self.nv])

    def jac_t(self, w, jv, y):
        return np.concatenate([self.base.jac_t(w[:self.nv], jv, y), y])

    def hess(self, w, lam):  # W of the v block (f and c are linear in s)
        return self.base.hess(w[:self.nv], lam)


class LiftedGpuKKT:
    """The per-iteration solve of LiftedNLP through libckkt with the Lifted-KKT strategy (m_e = 0, H = J,
    D_s = Sigma_s): refactor(w, j, sigma_w, delta_last) -> (ok, delta, trials); solve(r1_w, c_w) ->
    (dw, dlam, info)."""

    def __init__(self, n, m, w_row, w_col, j_rowptr, j_col, leaf=64, device=0):
        import torch
        from . import ckkt
        self.torch, self.ckkt = torch, ckkt
        self.dev = torch.device("cuda", device)
        self.n, self.m = n, m
        self.ctx = ckkt.Context(n, 0, m, w_row, w_col, None, None, j_rowptr, j_col, strategy=ckkt.CKKT_LIFTED,
                                leaf=leaf, device=device, stream=torch.cuda.current_stream(self.dev).cuda_stream)
        self.delta = torch.zeros(1, dtype=torch.float64, device=self.dev)

    def _t(self, a):
        if isinstance(a, self.torch.Tensor):  # device values (DeviceDistillationNLP): no host round trip
            return a.to(device=self.dev, dtype=self.torch.float64).contiguous()
        return self.torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=self.dev)

    def refactor(self, w_val, j_val, sigma_w, delta_last):
        n = self.n
        self._vals = [self._t(w_val), None, self._t(j_val), self._t(sigma_w[:n]), self._t(sigma_w[n:])]
        rc, d, t = self.ctx.refactor_inertia(*self._vals, self.delta, np.array([delta_last]))
        return rc == self.ckkt.CKKT_OK, float(d[0]), int(t[0])

    def solve(self, r1_w, c_w):
        T, n, m = self.torch, self.n, self.m
        dx = T.empty(n, dtype=T.float64, device=self.dev)
        ds = T.empty(m, dtype=T.float64, device=self.dev)
        dz = T.empty(m, dtype=T.float64, device=self.dev)
        rc, info = self.ctx.solve(self._t(r1_w[:n]), self._t(r1_w[n:]), None, self._t(c_w), dx, ds, None, dz)
        dw = np.concatenate([dx.cpu().numpy(), ds.cpu().numpy()])
        return dw, dz.cpu().numpy(), dict(info[0], rc=int(rc))

    def fraction_to_boundary(self, s, ds, tau):
        a = self.ckkt.fraction_to_boundary(self._t(s), self._t(ds), tau)
        return float(a.cpu().numpy()[0])


def solve_nlp(problem, kkt, mu0=0.1, tol=1e-6, max_iter=200, alpha_min_frac=0.05, verbose=False) -> IPMResult:
    """Filter line-search IPM (see the module docstring).  `problem` provides n, m, bidx (indices of
    the bounded variables), lo, hi, x0, lam0, f(v), grad_f(v), c(v), jac(v) (J values in the
    pattern's CSR order), jac_t(v, jv, y) (J^T y) and hess(v, lam) (W values
    of f + lam^T c).  `kkt` provides refactor / solve / fraction_to_boundary (GpuKKT)."""
    P = problem
    b, lo, hi = P.bidx, P.lo, P.hi
    v = P.x0.copy()
    lam = P.lam0.copy()
    mu = mu0
    sl, su = v[b] - lo, hi - v[b]
    z_lo, z_hi = mu / sl, mu / su
    delta_last = 0.0
    hist = []

    def barrier(vv, mu_):
        return P.f(vv) - mu_ * (np.log(vv[b] - lo).sum() + np.log(hi - vv[b]).sum())

    def kkt_error(vv, ll, zl, zu, jv, mu_):
        g = P.grad_f(vv) + P.jac_t(vv, jv, ll)
        g[b] += -zl + zu
        comp = max(np.abs((vv[b] - lo) * zl - mu_).max(initial=0.0), np.abs((hi - vv[b]) * zu - mu_).max(initial=0.0))
        return max(np.abs(g).max(initial=0.0), np.abs(P.c(vv)).max(initial=0.0), comp)

    cv = P.c(v)
    theta0 = np.abs(cv).sum()
    theta_max, theta_min = 1e4 * max(1.0, theta0), 1e-4 * max(1.0, theta0)
    filt = []
    status = "max_iter"
    it = 0
    for it in range(max_iter + 1):
        jv = P.jac(v)
        err0 = kkt_error(v, lam, z_lo, z_hi, jv, 0.0)
        if err0 <= tol:
            status = "converged"
            break
        while kkt_error(v, lam, z_lo, z_hi, jv, mu) <= KAPPA_EPS * mu and mu > tol / 10 * (1 + 1e-12):
            mu = max(tol / 10, min(KAPPA_MU * mu, mu ** THETA_MU))   # SPEC update_mu
            filt = []
        if it == max_iter:
            break
        sl, su = v[b] - lo, hi - v[b]
        sigma = np.zeros(P.n)
        sigma[b] = z_lo / sl + z_hi / su
        ok, delta, trials = kkt.refactor(P.hess(v, lam), jv, sigma, delta_last)
        if not ok:
            status = "inertia_failure"
            break
        if delta > 0:
            delta_last = delta
        r1 = P.grad_f(v) + P.jac_t(v, jv, lam)
        r1[b] += -mu / sl + mu / su
        cv = P.c(v)
        dx, dlam, info = kkt.solve(r1, cv)
        # a step the linear solver could not deliver (NOT_PD / CG non-convergence, or non-finite values)
        # must not reach the line search; REFINE_NOT_CONVERGED still returns the best (finite) iterate
        rc = int(info.get("rc", 0))
        if rc not in (0, 3) or not (np.all(np.isfinite(dx)) and np.all(np.isfinite(dlam))):
            status = "linear_solver_failure"
            hist.append(dict(mu=mu, delta_x=delta, trials=trials, k_cg=int(info.get("k_cg", 0)), solve_rc=rc))
            break
        dzl = mu / sl - z_lo - (z_lo / sl) * dx[b]
        dzu = mu / su - z_hi + (z_hi / su) * dx[b]
        tau = max(0.99, 1.0 - mu)
        a_max = min(kkt.fraction_to_boundary(np.concatenate([sl, su]), np.concatenate([dx[b], -dx[b]]), tau), 1.0)
        a_z = kkt.fraction_to_boundary(np.concatenate([z_lo, z_hi]), np.concatenate([dzl, dzu]), tau)
        # ---- filter line search (Wächter–Biegler)
        theta = np.abs(cv).sum()
        phi = barrier(v, mu)
        gphi = P.grad_f(v)
        gphi[b] += -mu / sl + mu / su
        dphi = float(gphi @ dx)
        alpha, ls, accepted, armijo = a_max, 0, False, False
        a_lo = alpha_min_frac * a_max * min(GAMMA_THETA, GAMMA_PHI * theta / max(-dphi, 1e-300)) if dphi < 0 \
            else alpha_min_frac * a_max * GAMMA_THETA
        while alpha >= a_lo and alpha > 1e-16:
            vt = v + alpha * dx
            tt = np.abs(P.c(vt)).sum()
            pt = barrier(vt, mu)
            if math.isfinite(pt) and tt <= theta_max and not any(tt >= ft and pt >= fp for ft, fp in filt):
                switching = dphi < 0 and alpha * (-dphi) ** S_PHI > DELTA_SW * theta ** S_THETA
                if theta <= theta_min and switching:
                    if pt <= phi + ETA_PHI * alpha * dphi:
                        accepted, armijo = True, True
                elif tt <= (1 - GAMMA_THETA) * theta or pt <= phi - GAMMA_PHI * theta:
                    accepted = True
            if accepted:
                break
            alpha *= 0.5
            ls += 1
        if not accepted:
            status = "restoration"
            break
        if not armijo:
            filt.append(((1 - GAMMA_THETA) * theta, phi - GAMMA_PHI * theta))
        v = v + alpha * dx
        lam = lam + alpha * dlam
        z_lo = z_lo + a_z * dzl
        z_hi = z_hi + a_z * dzu
        # keep the bound duals within KAPPA_SIGMA of mu / slack (Ipopt's safeguard)
        sl, su = v[b] - lo, hi - v[b]
        z_lo = np.clip(z_lo, mu / (KAPPA_SIGMA * sl), KAPPA_SIGMA * mu / sl)
        z_hi = np.clip(z_hi, mu / (KAPPA_SIGMA * su), KAPPA_SIGMA * mu / su)
        hist.append(dict(mu=mu, theta=theta, phi=phi, alpha=alpha, alpha_z=a_z, delta_x=delta, trials=trials,
                         k_cg=int(info.get("k_cg", 0)), solve_rc=int(info.get("rc", 0)), ls=ls))
        if verbose:
            print(f"it {it:3d} mu {mu:.2e} theta {theta:.2e} phi {phi:.6e} alpha {alpha:.3e} delta {delta:.1e} "
                  f"ls {ls}")
    return IPMResult(status=status, iterations=it, v=v, lam=lam, z_lo=z_lo, z_hi=z_hi, objective=P.f(v),
                     kkt_error=kkt_error(v, lam, z_lo, z_hi, P.jac(v), 0.0), history=hist)
