"""IPM loop around the ABI (paper_2403_15913_b200/ipm.py): host logic on CPU
with the oracle as the linear solver, and on the GPU through libckkt with iteration parity against
the oracle-driven run (HyKKT reaches the iteration counts of an exact factorization)."""
from __future__ import annotations

import numpy as np
import pytest

from inputs import distillation as dist
from kkt_cases import E32
from oracle import kkt as K
from paper_2403_15913_b200 import ipm


class OracleKKT:
    """Test adapter: the same refactor / solve / fraction_to_boundary calls served by the oracle."""

    def __init__(self, nlp, gamma=1e7):
        p = nlp.pat
        self.o = K.SparseKKT(nlp.n, nlp.m, 0, p.w_row, p.w_col, p.j_rowptr, p.j_col, E32, E32[:0],
                             strategy=K.HYKKT, gamma=gamma, leaf=64)

    def refactor(self, w_val, j_val, sigma_x, delta_last):
        d, t, failed = K.inertia_correction(self.o, w_val, j_val, [], sigma_x, [], delta_last=delta_last)
        return not failed, d, t

    def solve(self, r1, r3):
        (dx, ds, dy, dz), info = self.o.solve(r1, np.zeros(0), r3, np.zeros(0))
        return dx, dy, {"k_cg": info.k_cg}

    def fraction_to_boundary(self, s, ds, tau):
        return K.fraction_to_boundary(s, ds, tau)


class OracleLiftedKKT:
    """Test adapter of ipm.LiftedGpuKKT served by the oracle (Lifted-KKT: m_e = 0, H = J, D_s = Sigma_s)."""

    def __init__(self, nlp):
        p = nlp.pat
        self.n, self.m = nlp.nv, nlp.m
        self.o = K.SparseKKT(self.n, 0, self.m, p.w_row, p.w_col, E32, E32[:0], p.j_rowptr, p.j_col,
                             strategy=K.LIFTED, leaf=64)

    def refactor(self, w_val, j_val, sigma_w, delta_last):
        n = self.n
        d, t, failed = K.inertia_correction(self.o, w_val, [], j_val, sigma_w[:n], sigma_w[n:], delta_last=delta_last)
        return not failed, d, t

    def solve(self, r1_w, c_w):
        n = self.n
        (dx, ds, dy, dz), info = self.o.solve(r1_w[:n], r1_w[n:], np.zeros(0), c_w)
        return np.concatenate([dx, ds]), dz, {"k_cg": 0}

    def fraction_to_boundary(self, s, ds, tau):
        return K.fraction_to_boundary(s, ds, tau)


class _Pat:
    def __init__(self, w_row, w_col, j_rowptr, j_col):
        self.w_row, self.w_col = np.asarray(w_row, np.int32), np.asarray(w_col, np.int32)
        self.j_rowptr, self.j_col = np.asarray(j_rowptr, np.int32), np.asarray(j_col, np.int32)


class RosenNLP:
    """Nonconvex toy: min (1-x)^2 + 100 (y - x^2)^2 + (u - 2)^2  s.t.  x - u + 1 = 0,  1 <= u <= 5.
    Optimum (1, 1, 2), f = 0.  From (0.5, 1.5, 1.5) the reduced Hessian is indefinite, so the loop
    needs the inertia correction (delta_x > 0) and the line search backtracks."""
    n, m = 3, 1
    pat = _Pat([0, 1, 1, 2], [0, 0, 1, 2], [0, 2], [0, 2])
    bidx = np.array([2])
    lo, hi = np.array([1.0]), np.array([5.0])

    def __init__(self):
        self.x0 = np.array([0.5, 1.5, 1.5])
        self.lam0 = np.zeros(1)

    def f(self, v):
        x, y, u = v
        return (1 - x) ** 2 + 100 * (y - x * x) ** 2 + (u - 2) ** 2

    def grad_f(self, v):
        x, y, u = v
        return np.array([-2 * (1 - x) - 400 * x * (y - x * x), 200 * (y - x * x), 2 * (u - 2)])

    def c(self, v):
        return np.array([v[0] - v[2] + 1])

    def jac(self, v):
        return np.array([1.0, -1.0])

    def jac_t(self, v, jv, y):
        return np.array([jv[0] * y[0], 0.0, jv[1] * y[0]])

    def hess(self, v, lam):
        x, y, u = v
        return np.array([2 - 400 * y + 1200 * x * x, -400 * x, 200.0, 2.0])


def test_ipm_oracle_nonconvex_uses_inertia_correction():
    nlp = RosenNLP()
    res = ipm.solve_nlp(nlp, OracleKKT(nlp), max_iter=100)
    assert res.status == "converged", res
    assert np.allclose(res.v, [1.0, 1.0, 2.0], atol=1e-5)
    assert any(h["delta_x"] > 0 for h in res.history)
    assert any(h["trials"] > 1 for h in res.history)


@pytest.mark.gpu
def test_ipm_gpu_nonconvex_parity():
    """The nonconvex toy through libckkt: same iterations, deltas and trial counts as the oracle."""
    r_o = ipm.solve_nlp(RosenNLP(), OracleKKT(RosenNLP()), max_iter=100)
    p = RosenNLP.pat
    r_g = ipm.solve_nlp(RosenNLP(), ipm.GpuKKT(3, 1, p.w_row, p.w_col, p.j_rowptr, p.j_col, leaf=4), max_iter=100)
    assert r_g.status == r_o.status == "converged"
    assert r_g.iterations == r_o.iterations
    assert [h["trials"] for h in r_g.history] == [h["trials"] for h in r_o.history]
    np.testing.assert_allclose([h["delta_x"] for h in r_g.history], [h["delta_x"] for h in r_o.history], rtol=1e-12)
    assert np.abs(r_g.v - r_o.v).max() <= 1e-8


def _check_solution(nlp, res):
    assert res.status == "converged", (res.status, res.iterations)
    assert res.kkt_error <= 1e-6
    assert np.abs(nlp.c(res.v)).max() <= 1e-6
    u = res.v[nlp.bidx]
    assert np.all(u > nlp.lo) and np.all(u < nlp.hi)


def test_ipm_oracle_converges_distillation():
    """Host logic: the filter line-search IPM converges on the N = 4 distillation NLP to tol 1e-6
     from the simulated start, with bound multipliers >= 0 and u strictly inside its bounds."""
    nlp = dist.NLP(dist.Instance(4))
    res = ipm.solve_nlp(nlp, OracleKKT(nlp), max_iter=100)
    _check_solution(nlp, res)
    assert np.all(res.z_lo > 0) and np.all(res.z_hi > 0)
    assert res.history[-1]["mu"] <= 1e-6


@pytest.mark.gpu
def test_ipm_gpu_iteration_parity():
    """The same IPM with the libckkt HyKKT solve (inertia correction and fraction-to-boundary on
    the device) converges on N = 10 in the same number of iterations as with the oracle solve, to
    the same optimum."""
    nlp = dist.NLP(dist.Instance(10))
    r_o = ipm.solve_nlp(nlp, OracleKKT(nlp), max_iter=100)
    nlp_g = dist.NLP(dist.Instance(10))
    r_g = ipm.solve_nlp(nlp_g, ipm.GpuKKT(nlp_g.n, nlp_g.m, nlp_g.pat.w_row, nlp_g.pat.w_col, nlp_g.pat.j_rowptr,
                                          nlp_g.pat.j_col), max_iter=100)
    _check_solution(nlp, r_o)
    _check_solution(nlp_g, r_g)
    assert r_g.iterations == r_o.iterations
    assert abs(r_g.objective - r_o.objective) <= 1e-8 * max(1.0, abs(r_o.objective))
    assert np.abs(r_g.v - r_o.v).max() <= 1e-6


def _check_lifted(lnlp, res):
    assert res.status == "converged", (res.status, res.iterations)
    assert res.kkt_error <= 1e-6
    v, sl = res.v[:lnlp.nv], res.v[lnlp.nv:]
    c = lnlp.base.c(v)
    assert np.abs(c + sl).max() <= 1e-6                     # c(v) + s = 0
    assert np.all(np.abs(sl) < lnlp.tau)                     # -tau < s < tau: the relaxed rows hold
    assert np.abs(c).max() <= lnlp.tau + 1e-6


def test_ipm_oracle_lifted_relaxation_converges():
    """NEXT-1: the same filter line-search IPM on the relaxed problem of Lifted-KKT
    (-tau <= c(v) <= tau, tau = 1e-6, one slack per row) converges on the N = 4 distillation NLP to
    tol 1e-6; the relaxed optimum is within O(tau) of the HyKKT one.  Iteration counts are recorded for the
    paper's comparison ("Lifted-KKT ... requires twice as much iterations")."""
    nlp = dist.NLP(dist.Instance(4))
    res_h = ipm.solve_nlp(nlp, OracleKKT(nlp), max_iter=200)
    lnlp = ipm.LiftedNLP(dist.NLP(dist.Instance(4)))
    res_l = ipm.solve_nlp(lnlp, OracleLiftedKKT(lnlp), max_iter=200)
    _check_solution(nlp, res_h)
    _check_lifted(lnlp, res_l)
    assert abs(res_l.objective - res_h.objective) <= 1e-3 * max(1.0, abs(res_h.objective))
    print(f"iterations: HyKKT {res_h.iterations}, Lifted-KKT {res_l.iterations}")


@pytest.mark.gpu
def test_ipm_gpu_lifted_iteration_parity():
    """Lifted-KKT IPM through libckkt (inertia correction, Lifted solve with K_aug refinement and
    fraction-to-boundary on the device): the same iteration count as the oracle-driven run on N = 10."""
    def run(kkt_cls):
        lnlp = ipm.LiftedNLP(dist.NLP(dist.Instance(10)))
        p = lnlp.pat
        kkt = kkt_cls(lnlp) if kkt_cls is OracleLiftedKKT else kkt_cls(lnlp.nv, lnlp.m, p.w_row, p.w_col, p.j_rowptr,
                                                                        p.j_col)
        return lnlp, ipm.solve_nlp(lnlp, kkt, max_iter=200)
    lo, r_o = run(OracleLiftedKKT)
    lg, r_g = run(ipm.LiftedGpuKKT)
    _check_lifted(lo, r_o)
    _check_lifted(lg, r_g)
    assert r_g.iterations == r_o.iterations
    assert abs(r_g.objective - r_o.objective) <= 1e-8 * max(1.0, abs(r_o.objective))


@pytest.mark.gpu
@pytest.mark.parametrize("lifted", [False, True])
def test_ipm_gpu_device_model(lifted):
    """NEXT-4 inside NEXT-1: the IPM with the model derivatives evaluated on the GPU
    (ipm.DeviceDistillationNLP: J and W from ckkt_distillation_eval go to libckkt without a host round
    trip) takes the same iterations to the same optimum as with the host model, for HyKKT and for
    Lifted-KKT on the relaxed problem (N = 10)."""
    def run(device_model):
        base = dist.NLP(dist.Instance(10))
        nlp = ipm.DeviceDistillationNLP(base) if device_model else base
        if lifted:
            nlp = ipm.LiftedNLP(nlp)
            p = nlp.pat
            kkt = ipm.LiftedGpuKKT(nlp.nv, nlp.m, p.w_row, p.w_col, p.j_rowptr, p.j_col)
        else:
            p = nlp.pat
            kkt = ipm.GpuKKT(nlp.n, nlp.m, p.w_row, p.w_col, p.j_rowptr, p.j_col)
        return nlp, ipm.solve_nlp(nlp, kkt, max_iter=200)
    nh, rh = run(False)
    nd, rd = run(True)
    if lifted:
        _check_lifted(nh, rh)
        _check_lifted(nd, rd)
    else:
        _check_solution(nh, rh)
        _check_solution(nd.base, rd)
    assert rd.iterations == rh.iterations
    assert abs(rd.objective - rh.objective) <= 1e-8 * max(1.0, abs(rh.objective))
    # both runs stop at the IPM tolerance 1e-6; the relaxed problem's slacks / duals are less
    # well determined, so its iterates agree to O(tol) rather than better
    assert np.abs(rd.v - rh.v).max() <= (1e-5 if lifted else 1e-6)


def test_transpose_pattern_matches_scipy():
    """The J^T pattern DeviceDistillationNLP multiplies with (host logic, no GPU): values gathered through
    perm reproduce scipy's transpose of the distillation Jacobian pattern."""
    from scipy.sparse import csr_matrix
    pat = dist.build_pattern(7)
    rng = np.random.default_rng(5)
    jv = rng.standard_normal(pat.j_col.size)
    ptr, col, perm = ipm.transpose_pattern(pat.j_rowptr, pat.j_col, pat.n)
    ref = csr_matrix((jv, pat.j_col, pat.j_rowptr), shape=(pat.m, pat.n)).T.tocsr()
    ref.sort_indices()
    assert np.array_equal(ptr, ref.indptr) and np.array_equal(col, ref.indices)
    assert np.array_equal(jv[perm], ref.data)
    y = rng.standard_normal(pat.m)
    got = np.array([jv[perm][ptr[i]:ptr[i + 1]] @ y[col[ptr[i]:ptr[i + 1]]] for i in range(pat.n)])
    assert np.allclose(got, ref @ y, rtol=1e-14, atol=1e-14)
