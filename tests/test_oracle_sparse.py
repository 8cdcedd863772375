"""Pins of the Tier S oracle (oracle/sparse.py, oracle/kkt.py): brute force on tiny
inputs, library routines, hand-derived orderings, 40-digit references."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from inputs import distillation as dist
from inputs.random_kkt import random_instance
from oracle import dense as D
from oracle import kkt as K
from oracle import sparse as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


# ----------------------------------------------------------------------------
# helpers (brute force, written independently of the oracle)
# ----------------------------------------------------------------------------
def lower_csc(A_bool):
    n = A_bool.shape[0]
    Ap, Ai = [0], []
    for j in range(n):
        rows = [i for i in range(j, n) if A_bool[i, j] or i == j]
        Ai += rows
        Ap.append(len(Ai))
    return np.array(Ap, np.int64), np.array(Ai, np.int32)


def brute_symbolic(A_bool):
    """Dense boolean Gaussian elimination: filled pattern F, parent(j) = min{i>j: F_ij}."""
    n = A_bool.shape[0]
    F = np.array(A_bool | A_bool.T, dtype=bool)
    np.fill_diagonal(F, True)
    for j in range(n):
        rows = [i for i in range(j + 1, n) if F[i, j]]
        for a in rows:
            for b in rows:
                F[a, b] = True
    L = np.tril(F)
    parent = np.array([min([i for i in range(j + 1, n) if L[i, j]], default=-1) for j in range(n)])
    return L, parent


def brute_md(adj_sets, verts):
    """Exact minimum degree with lowest-index ties, Python sets."""
    G = {v: set(a for a in adj_sets[v] if a in verts) for v in verts}
    order = []
    while G:
        v = min(G, key=lambda x: (len(G[x]), x))
        nb = G.pop(v)
        for a in nb:
            G[a] |= nb
            G[a].discard(a)
            G[a].discard(v)
        order.append(v)
    return order


def adjacency(A_bool):
    n = A_bool.shape[0]
    xadj, adj = [0], []
    for i in range(n):
        nb = [j for j in range(n) if j != i and (A_bool[i, j] or A_bool[j, i])]
        adj += nb
        xadj.append(len(adj))
    return np.array(xadj, np.int32), np.array(adj, np.int32)


def random_pattern(n, dens, seed):
    rng = np.random.default_rng(seed)
    A = rng.uniform(size=(n, n)) < dens
    A = A | A.T
    np.fill_diagonal(A, True)
    return A


# ----------------------------------------------------------------------------
# symbolic analysis
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(20))
def test_symbolic_vs_boolean_elimination(seed):
    n = 5 + seed * 3
    A = random_pattern(n, 0.08 + 0.01 * (seed % 5), seed)
    Ap, Ai = lower_csc(A)
    parent, cc, Lp, Li = S.symbolic(Ap, Ai)
    L, par_ref = brute_symbolic(A)
    assert np.array_equal(parent, par_ref)
    assert np.array_equal(cc, L.sum(axis=0))
    for j in range(n):
        assert np.array_equal(Li[Lp[j]:Lp[j + 1]], np.nonzero(L[:, j])[0])


def test_symbolic_worked_examples():
    n = 10
    T = np.eye(n, dtype=bool) | np.eye(n, k=1, dtype=bool) | np.eye(n, k=-1, dtype=bool)
    assert S.symbolic(*lower_csc(T))[3].size == GOLD["symbolic_tridiagonal"]["nnz_L"]
    arrow_first = np.eye(n, dtype=bool)
    arrow_first[0, :] = arrow_first[:, 0] = True
    arrow_last = np.eye(n, dtype=bool)
    arrow_last[-1, :] = arrow_last[:, -1] = True
    g = GOLD["symbolic_arrow"]
    assert S.symbolic(*lower_csc(arrow_last))[3].size == g["nnz_L_arrow_last"]
    assert S.symbolic(*lower_csc(arrow_first))[3].size == g["nnz_L_arrow_first"]
    Dg = np.eye(n, dtype=bool)
    parent, cc, Lp, Li = S.symbolic(*lower_csc(Dg))
    assert np.all(parent == -1) and np.all(cc == 1)


def test_symbolic_distillation_vs_brute():
    pat = dist.build_pattern(1)
    o = K.SparseKKT(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col,
                    np.zeros(1, np.int32), np.zeros(0, np.int32), leaf=16)
    Kd = o.Kp.toarray() != 0
    P = Kd[np.ix_(o.perm, o.perm)]
    L, par = brute_symbolic(P)
    assert np.array_equal(o.parent, par)
    assert o.Li.size == L.sum()


# ----------------------------------------------------------------------------
# ordering
# ----------------------------------------------------------------------------
def test_nd_path_graph_hand_derived():
    """Path 0-1-2-3-4-5-6, leaf 2: separator {3}, then {1} and {5} (derivation in DESIGN.md §5)."""
    n = 7
    A = np.eye(n, dtype=bool) | np.eye(n, k=1, dtype=bool) | np.eye(n, k=-1, dtype=bool)
    xadj, adj = adjacency(A)
    assert S.nd_order(xadj, adj, 2).tolist() == [0, 2, 1, 4, 6, 5, 3]


def test_nd_components_order():
    """Two disjoint paths {0,2,4} and {1,3}: components ordered by smallest vertex; leaf >= size -> MD."""
    A = np.eye(5, dtype=bool)
    for a, b in [(0, 2), (2, 4), (1, 3)]:
        A[a, b] = A[b, a] = True
    xadj, adj = adjacency(A)
    # MD on {0,2,4}: degrees 1,2,1 -> 0 first (lowest index), then 2 (deg 1, tie with 4 -> 2), then 4
    assert S.nd_order(xadj, adj, 10).tolist() == [0, 2, 4, 1, 3]


@pytest.mark.parametrize("seed", range(8))
def test_md_leaf_vs_python_sets(seed):
    n = 12 + 4 * seed
    A = random_pattern(n, 0.15, 50 + seed)
    xadj, adj = adjacency(A)
    adj_sets = {i: set(adj[xadj[i]:xadj[i + 1]]) for i in range(n)}
    # leaf >= n: whole components ordered by MD, components by smallest vertex
    got = S.nd_order(xadj, adj, n).tolist()
    seen, comps = set(), []
    for v in range(n):
        if v in seen:
            continue
        comp, stack = {v}, [v]
        while stack:
            x = stack.pop()
            for a in adj_sets[x]:
                if a not in comp:
                    comp.add(a); stack.append(a)
        seen |= comp
        comps.append(comp)
    ref = []
    for c in comps:
        ref += brute_md(adj_sets, c)
    assert got == ref


def test_nd_ordering_properties_distillation():
    pat = dist.build_pattern(30)
    args = (pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, np.zeros(1, np.int32), np.zeros(0, np.int32))
    o = K.SparseKKT(*args, leaf=268)
    assert np.array_equal(np.sort(o.perm), np.arange(pat.n))
    o2 = K.SparseKKT(*args, leaf=268)
    assert np.array_equal(o.perm, o2.perm)  # deterministic
    nat = K.SparseKKT(*args, perm=np.arange(pat.n, dtype=np.int32))
    assert o.Li.size < nat.Li.size  # fill reduction


# ----------------------------------------------------------------------------
# numeric Cholesky and triangular solves
# ----------------------------------------------------------------------------
def _spd_from_pattern(A_bool, seed):
    rng = np.random.default_rng(seed)
    n = A_bool.shape[0]
    M = np.where(A_bool, rng.standard_normal((n, n)), 0.0)
    M = (M + M.T) / 2
    M += np.diag(np.abs(M).sum(axis=1) + 1.0)
    return M


def _lower_vals(M, Ap, Ai):
    n = len(Ap) - 1
    return np.array([M[Ai[p], j] for j in range(n) for p in range(Ap[j], Ap[j + 1])])


@pytest.mark.parametrize("seed", range(10))
def test_cholesky_vs_lapack(seed):
    n = 10 + 5 * seed
    A = random_pattern(n, 0.1, 200 + seed)
    M = _spd_from_pattern(A, seed)
    Ap, Ai = lower_csc(A)
    parent, cc, Lp, Li = S.symbolic(Ap, Ai)
    Lx, fail = S.cholesky(Ap, Ai, _lower_vals(M, Ap, Ai), Lp, Li)
    assert fail == -1
    Ld = np.zeros((n, n))
    for j in range(n):
        Ld[Li[Lp[j]:Lp[j + 1]], j] = Lx[Lp[j]:Lp[j + 1]]
    Lref = np.linalg.cholesky(M)
    assert np.abs(Ld - Lref).max() <= 1e-12 * np.abs(Lref).max()
    b = np.random.default_rng(seed).standard_normal(n)
    x = S.ltsolve(Lp, Li, Lx, S.lsolve(Lp, Li, Lx, b))
    assert np.linalg.norm(M @ x - b) <= 1e-12 * np.linalg.norm(b) * np.linalg.cond(M)


def test_cholesky_worked_examples():
    g = GOLD["cholesky_identity"]
    A = np.array(g["A"], float)
    Ap, Ai = lower_csc(A != 0)
    _, _, Lp, Li = S.symbolic(Ap, Ai)
    Lx, fail = S.cholesky(Ap, Ai, _lower_vals(A, Ap, Ai), Lp, Li)
    assert fail == -1 and np.array_equal(Lx, np.ones(3))
    g = GOLD["cholesky_not_pd"]
    A = np.array(g["A"], float)
    Ap, Ai = lower_csc(A != 0)
    _, _, Lp, Li = S.symbolic(Ap, Ai)
    assert S.cholesky(Ap, Ai, _lower_vals(A, Ap, Ai), Lp, Li)[1] == g["pivot"]
    g = GOLD["trisolve_diag"]
    A = np.array(g["A"], float)
    Ap, Ai = lower_csc(A != 0)
    _, _, Lp, Li = S.symbolic(Ap, Ai)
    Lx, _ = S.cholesky(Ap, Ai, _lower_vals(A, Ap, Ai), Lp, Li)
    x = S.ltsolve(Lp, Li, Lx, S.lsolve(Lp, Li, Lx, np.array(g["b"], float)))
    assert np.allclose(x, g["x"], atol=1e-15)


def test_cholesky_nan_pivot_fails():
    A = np.array([[1.0, 0.0], [0.0, np.nan]])
    Ap, Ai = lower_csc(np.ones((2, 2), bool))
    _, _, Lp, Li = S.symbolic(Ap, Ai)
    assert S.cholesky(Ap, Ai, np.array([1.0, 0.0, np.nan]), Lp, Li)[1] == 1


def test_refactorization_reuse():
    """20 refills against one symbolic analysis equal LAPACK on each."""
    pat = dist.build_pattern(2)
    inst = dist.Instance(2)
    o = K.SparseKKT(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col,
                    np.zeros(1, np.int32), np.zeros(0, np.int32), gamma=1e4, leaf=32)
    for k, it in enumerate(inst.trajectory()[:20]):
        assert o.refactor(it.w_val, it.j_val, np.zeros(0), it.sigma_x, np.zeros(0), 0.0) == -1
        Kd = sp.csc_matrix((o.Ax, o.Ai, o.Ap), shape=(pat.n, pat.n)).toarray()
        Kd = Kd + np.tril(Kd, -1).T
        Lref = np.linalg.cholesky(Kd)
        Ld = sp.csc_matrix((o.Lx, o.Li, o.Lp), shape=(pat.n, pat.n)).toarray()
        assert np.abs(Ld - Lref).max() <= 1e-10 * np.abs(Lref).max()


# ----------------------------------------------------------------------------
# CG on S_gamma
# ----------------------------------------------------------------------------
def _diag_instance(kdiag, gamma):
    n = len(kdiag)
    W = np.diag(kdiag)
    rows, cols = np.arange(n, dtype=np.int32), np.arange(n, dtype=np.int32)
    eye_rp = np.arange(n + 1, dtype=np.int32)
    o = K.SparseKKT(n, n, 0, rows, cols, eye_rp, np.arange(n, dtype=np.int32), np.zeros(1, np.int32),
                    np.zeros(0, np.int32), gamma=gamma, cg_rtol=1e-12, leaf=4)
    o.refactor(np.array(kdiag, float), np.ones(n), np.zeros(0), np.zeros(n), np.zeros(0), 0.0)
    return o


def test_cg_worked_examples():
    """G = I: S_gamma = (K + gamma I)^{-1}.  K = I -> 1 iteration; K = diag(1,2,3) -> <= 3."""
    o = _diag_instance([1.0, 1.0, 1.0], 1.0)
    x, k, conv = o._cg(np.array([1.0, 2.0, 3.0]))
    assert conv and k == 1 and np.allclose(x, 2 * np.array([1.0, 2.0, 3.0]))
    o = _diag_instance([1.0, 2.0, 3.0], 1.0)
    x, k, conv = o._cg(np.array([1.0, 2.0, 3.0]))
    assert conv and k <= 3 and np.allclose(x, np.array([2.0, 6.0, 12.0]))
    x, k, conv = o._cg(np.zeros(3))
    assert k == 0 and np.all(x == 0)


def test_cg_krylov_bound():
    """k distinct eigenvalues -> <= k iterations, here with 4 distinct values."""
    kd = np.repeat([1.0, 5.0, 9.0, 20.0], 6)
    o = _diag_instance(kd, 0.5)
    b = np.random.default_rng(1).standard_normal(len(kd))
    x, k, conv = o._cg(b)
    assert conv and k <= 4 + 1
    assert np.allclose(x, (kd + 0.5) * b, rtol=1e-10)


# ----------------------------------------------------------------------------
# full Newton step vs the definition
# ----------------------------------------------------------------------------
def _oracle_for(inst, strategy, gamma=1e7, leaf=8):
    o = K.SparseKKT(inst.n, inst.m_e, inst.m_i, inst.w_row, inst.w_col, inst.g_rowptr, inst.g_col,
                    inst.h_rowptr, inst.h_col, strategy=strategy, gamma=gamma, leaf=leaf)
    fail = o.refactor(inst.w_val, inst.g_val, inst.h_val, inst.sigma_x, inst.d_s, inst.delta_x)
    return o, fail


def mp_reference(inst, dps=40):
    """K_aug d = -r solved in 40-digit arithmetic (mpmath LU)."""
    import mpmath
    mpmath.mp.dps = dps
    Ka = D.assemble_kaug(inst)
    r = D.rhs_vector(inst)
    A = mpmath.matrix(Ka.tolist())
    b = mpmath.matrix((-r).tolist())
    x = mpmath.lu_solve(A, b)
    return np.array([float(v) for v in x])


@pytest.mark.parametrize("seed", range(8))
def test_hykkt_sparse_vs_mpmath(seed):
    """Wide-range Sigma (1e-8..1e8) and D_s: refined HyKKT step within 1e-9 of the 40-digit step."""
    inst = random_instance(14, 5, 4, seed=seed, sigma_range=(1e-8, 1e8), d_range=(1e-4, 1e8))
    ref = mp_reference(inst)
    for gamma in (1e4, 1e7):
        o, fail = _oracle_for(inst, K.HYKKT, gamma=gamma)
        assert fail == -1
        d, info = o.solve(inst.r1, inst.r2, inst.r3, inst.r4)
        got = np.concatenate(d)
        assert np.linalg.norm(got - ref) <= 1e-9 * np.linalg.norm(ref), (gamma, info)
        assert info.rel_res <= 1e-12


@pytest.mark.parametrize("seed", range(8))
def test_lifted_sparse_vs_mpmath(seed):
    """Lifted-KKT with D_s in [1e5, 1e12] (tau = 1e-6 regime): refinement restores accuracy."""
    inst = random_instance(16, 0, 10, seed=seed, d_range=(1e5, 1e12))
    ref = mp_reference(inst)
    o, fail = _oracle_for(inst, K.LIFTED)
    assert fail == -1
    d, info = o.solve(inst.r1, inst.r2, inst.r3, inst.r4)
    got = np.concatenate(d)
    for a, b in zip(D.split_step(inst, got), D.split_step(inst, ref)):
        if len(b):
            assert np.linalg.norm(a - b) <= 1e-9 * np.linalg.norm(b)
    assert info.rel_res <= 1e-12


def test_not_pd_flag():
    """An indefinite K (negative Sigma) makes the Cholesky fail: wrong inertia."""
    inst = random_instance(12, 0, 3, seed=4)
    inst.sigma_x = inst.sigma_x - 1e3
    o, fail = _oracle_for(inst, K.LIFTED)
    assert fail >= 0
    Kc = D.condensed_matrix(inst)
    assert np.linalg.eigvalsh(Kc).min() < 0


def _bk_refined_reference(inst):
    """BK solve + 3 refinement steps with the residual in extended precision (x87 long double)."""
    Ka = D.assemble_kaug(inst)
    r = D.rhs_vector(inst)
    bk = D.BunchKaufman(Ka)
    x = bk.solve(-r)
    KL = Ka.astype(np.longdouble)
    for _ in range(3):
        res = (-r.astype(np.longdouble) - KL @ x.astype(np.longdouble)).astype(np.float64)
        x = x + bk.solve(res)
    return x


class _DistInst:
    def __init__(self, N, it, strategy, rhs_seed=3000):
        md = dist.Model(N)
        pat = md.pat
        self.n = pat.n
        rng = np.random.default_rng(rhs_seed)
        if strategy == K.HYKKT:
            self.m_e, self.m_i = pat.m, 0
            self.g_rowptr, self.g_col, self.g_val = pat.j_rowptr, pat.j_col, it.j_val
            self.h_rowptr, self.h_col, self.h_val = np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0)
            self.d_s = np.zeros(0)
        else:
            self.m_e, self.m_i = 0, pat.m
            self.h_rowptr, self.h_col, self.h_val = pat.j_rowptr, pat.j_col, it.j_val
            self.g_rowptr, self.g_col, self.g_val = np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0)
            self.d_s = it.d_lifted
        self.w_row, self.w_col, self.w_val = pat.w_row, pat.w_col, it.w_val
        self.sigma_x, self.delta_x = it.sigma_x, 0.0
        self.r1 = rng.standard_normal(self.n)
        self.r2 = rng.standard_normal(self.m_i)
        self.r3 = rng.standard_normal(self.m_e)
        self.r4 = rng.standard_normal(self.m_i)

    def W_dense(self):
        W = np.zeros((self.n, self.n))
        W[self.w_row, self.w_col] = self.w_val
        return W + np.tril(W, -1).T

    def G_dense(self):
        return sp.csr_matrix((self.g_val, self.g_col, self.g_rowptr), shape=(self.m_e, self.n)).toarray()

    def H_dense(self):
        return sp.csr_matrix((self.h_val, self.h_col, self.h_rowptr), shape=(self.m_i, self.n)).toarray()


@pytest.mark.parametrize("strategy", [K.HYKKT, K.LIFTED])
@pytest.mark.parametrize("k", [0, 17])
def test_distillation_step_vs_dense_reference(strategy, k):
    """N = 2 distillation iterates (mu = 0.1 and 1e-7): refined sparse step within 1e-8 per block
    of the extended-precision-refined dense Bunch–Kaufman step."""
    inst_d = dist.Instance(2)
    it = inst_d.trajectory()[k]
    inst = _DistInst(2, it, strategy)
    ref = _bk_refined_reference(inst)
    o, fail = _oracle_for(inst, strategy, leaf=32)
    assert fail == -1
    d, info = o.solve(inst.r1, inst.r2, inst.r3, inst.r4)
    for a, b in zip(d, D.split_step(inst, ref)):
        if len(b):
            assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b), info
    assert info.rel_res <= 1e-12


def test_cg_iterations_distillation_gamma_1e7():
    """CG on S_gamma converges in < 10 iterations on average at gamma = 1e7."""
    inst_d = dist.Instance(50)
    pat = inst_d.model.pat
    o = K.SparseKKT(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col,
                    np.zeros(1, np.int32), np.zeros(0, np.int32), gamma=1e7, leaf=268)
    ks = []
    for it in inst_d.trajectory()[::2]:
        assert o.refactor(it.w_val, it.j_val, np.zeros(0), it.sigma_x, np.zeros(0), 0.0) == -1
        r1 = np.random.default_rng(1).standard_normal(pat.n)
        r3 = np.random.default_rng(2).standard_normal(pat.m)
        d, info = o.solve(r1, np.zeros(0), r3, np.zeros(0))
        ks.append(info.k_cg)
        assert info.rel_res <= 1e-12
    assert np.mean(ks) < 10


def test_hykkt_gamma_robustness_sparse():
    """Steps identical across gamma in {1e4, 1e6, 1e8} after refinement."""
    inst_d = dist.Instance(5)
    it = inst_d.trajectory()[9]
    inst = _DistInst(5, it, K.HYKKT)
    steps = []
    for gamma in (1e4, 1e6, 1e8):
        o, fail = _oracle_for(inst, K.HYKKT, gamma=gamma, leaf=64)
        assert fail == -1
        d, info = o.solve(inst.r1, inst.r2, inst.r3, inst.r4)
        steps.append(np.concatenate(d))
    for s in steps[1:]:
        assert np.linalg.norm(s - steps[0]) <= 1e-8 * np.linalg.norm(steps[0])


@pytest.mark.parametrize("seed", range(6))
def test_unrefined_pass_matches_dense_formulas(seed):
    """The unrefined sparse pass (condensation, CG, recovery) equals the Tier T formulas
    of P:306-313 / P:377-394 on its own, so refinement cannot mask a wrong term."""
    inst = random_instance(18, 6, 5, seed=300 + seed)
    o, fail = _oracle_for(inst, K.HYKKT, gamma=1e3)
    assert fail == -1
    o.cg_rtol = 1e-14
    dx, ds, dy, dz, k, conv = o.solve_once(inst.r1, inst.r2, inst.r3, inst.r4)
    ref = D.hykkt_step_dense(inst, 1e3)
    for a, b in zip((dx, ds, dy, dz), ref):
        assert np.linalg.norm(a - b) <= 1e-9 * max(np.linalg.norm(b), 1e-300)
    inst = random_instance(18, 0, 7, seed=400 + seed)
    o, fail = _oracle_for(inst, K.LIFTED)
    dx, ds, dy, dz, k, conv = o.solve_once(inst.r1, inst.r2, inst.r3, inst.r4)
    ref = D.lifted_step_dense(inst)
    for a, b in zip((dx, ds, dz), (ref[0], ref[1], ref[3])):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
