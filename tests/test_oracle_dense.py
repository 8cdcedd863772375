"""Pins of the Tier T oracle (oracle/dense.py) against library routines,
closed forms and the worked examples of tests/golden/."""
import json
import os

import numpy as np
import pytest

from inputs.random_kkt import random_instance
from oracle import dense as D

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


class _Tiny:
    """Hand-written instance from dense blocks (worked examples)."""

    def __init__(self, W, G=None, H=None, sigma=None, d_s=None, r1=None, r2=None, r3=None, r4=None, delta=0.0):
        W = np.array(W, float)
        self.n = W.shape[0]
        self._W = W
        self._G = np.zeros((0, self.n)) if G is None else np.array(G, float)
        self._H = np.zeros((0, self.n)) if H is None else np.array(H, float)
        self.m_e, self.m_i = self._G.shape[0], self._H.shape[0]
        self.sigma_x = np.zeros(self.n) if sigma is None else np.array(sigma, float)
        self.d_s = np.zeros(self.m_i) if d_s is None else np.array(d_s, float)
        self.delta_x = delta
        z = lambda v, k: np.zeros(k) if v is None else np.array(v, float)
        self.r1, self.r2, self.r3, self.r4 = z(r1, self.n), z(r2, self.m_i), z(r3, self.m_e), z(r4, self.m_i)

    def W_dense(self):
        return self._W

    def G_dense(self):
        return self._G

    def H_dense(self):
        return self._H


@pytest.mark.parametrize("seed", range(20))
def test_bunch_kaufman_solve_matches_lapack(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40))
    A = rng.standard_normal((n, n))
    A = A + A.T
    if seed % 3 == 0:
        A[np.diag_indices(n)] = 0.0  # forces 2x2 pivots
    b = rng.standard_normal(n)
    x = D.BunchKaufman(A).solve(b)
    xr = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xr) <= 1e-9 * np.linalg.norm(xr)


def test_bunch_kaufman_inertia_vs_eigen():
    """Sylvester: BK inertia equals eigenvalue sign counts on 100 matrices."""
    rng = np.random.default_rng(11)
    for _ in range(100):
        n = int(rng.integers(1, 30))
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        ev = rng.standard_normal(n) * np.exp(rng.uniform(-3, 3, n))
        k0 = int(rng.integers(0, 3))
        ev[:k0] = 0.0
        A = (Q * ev) @ Q.T
        A = (A + A.T) / 2
        assert D.BunchKaufman(A).inertia() == D.eig_inertia(A)


def test_inertia_worked_examples():
    for A, expect in GOLD["inertia_small"]["cases"]:
        assert D.BunchKaufman(np.array(A, float)).inertia() == tuple(expect)


def _gen(seed, n=None, me=None, mi=None, **kw):
    rng = np.random.default_rng(seed + 100)
    n = n or int(rng.integers(4, 20))
    me = int(rng.integers(0, n // 2 + 1)) if me is None else me
    mi = int(rng.integers(0, n)) if mi is None else mi
    return random_instance(n, me, mi, seed=seed, **kw)


@pytest.mark.parametrize("seed", range(25))
def test_augmented_step_inertia_and_residual(seed):
    """Eq. inertia holds for LICQ+SOSC instances; BK step solves K_aug d = -r."""
    inst = _gen(seed)
    (dx, ds, dy, dz), inert = D.augmented_step(inst)
    assert inert == (inst.n + inst.m_i, 0, inst.m_i + inst.m_e)
    K = D.assemble_kaug(inst)
    d = np.concatenate([dx, ds, dy, dz])
    r = D.rhs_vector(inst)
    assert np.linalg.norm(K @ d + r) <= 1e-10 * (np.linalg.norm(K) * np.linalg.norm(d) + np.linalg.norm(r))


def test_haynsworth_equivalence():
    """In(K_aug) = (n+m_i, 0, m_i+m_e)  <=>  In(K_cond) = (n, 0, m_e), 100 instances,
    half of them made indefinite on null(G) by a negative diagonal shift."""
    rng = np.random.default_rng(3)
    hits = {True: 0, False: 0}
    for s in range(100):
        inst = _gen(1000 + s)
        if s % 2:
            inst.sigma_x = inst.sigma_x - rng.uniform(0.5, 20.0)
        Ka, Kc = D.assemble_kaug(inst), D.assemble_kcond(inst)
        a = D.eig_inertia(Ka) == (inst.n + inst.m_i, 0, inst.m_i + inst.m_e)
        c = D.eig_inertia(Kc) == (inst.n, 0, inst.m_e)
        assert a == c
        hits[a] += 1
    assert hits[True] > 10 and hits[False] > 10


@pytest.mark.parametrize("seed", range(15))
def test_condensed_and_hykkt_equal_augmented(seed):
    """Block elimination and HyKKT reproduce the K_aug step;
    HyKKT is gamma-independent."""
    inst = _gen(seed)
    (dx, ds, dy, dz), _ = D.augmented_step(inst)
    ref = np.concatenate([dx, ds, dy, dz])
    for gamma in (1e-3, 1.0, 1e4, 1e6, 1e8):
        h = np.concatenate(D.hykkt_step_dense(inst, gamma))
        tol = 1e-8 if gamma <= 1e4 else 1e-6
        assert np.linalg.norm(h - ref) <= tol * np.linalg.norm(ref), gamma


@pytest.mark.parametrize("seed", range(10))
def test_lifted_equals_relaxed_augmented(seed):
    """Eq. liftedkkt is the relaxed problem's K_aug step (moderate D_s)."""
    inst = _gen(seed, me=0)
    (dx, ds, dy, dz), inert = D.augmented_step(inst)
    ref = np.concatenate([dx, ds, dy, dz])
    got = np.concatenate(D.lifted_step_dense(inst))
    assert np.linalg.norm(got - ref) <= 1e-9 * np.linalg.norm(ref)


def test_lifted_unrefined_loses_accuracy_with_large_D():
    """with D_s ~ 1/tau^2 the unrefined Lifted step is inaccurate and "has to be
    refined" -- the unrefined dense step departs from the K_aug step by >> FP64 eps."""
    errs = []
    for seed in range(6):
        inst = _gen(seed, me=0, d_range=(1e5, 1e12))
        (dx, ds, dy, dz), _ = D.augmented_step(inst)
        ref = np.concatenate([dx, ds, dy, dz])
        got = np.concatenate(D.lifted_step_dense(inst))
        errs.append(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    assert max(errs) > 1e-10


def test_worked_examples_hykkt():
    g = GOLD["hykkt_rank_one"]
    t = _Tiny(g["K"], G=g["G"])
    assert np.allclose(D.hykkt_matrix(t, g["gamma"]), np.array(g["K_gamma"]), atol=0, rtol=0)
    g = GOLD["hykkt_hand_solved"]
    for gamma in g["gammas"]:
        t = _Tiny(g["K"], G=g["G"], r1=g["r1"], r3=g["r3"])
        dx, ds, dy, dz = D.hykkt_step_dense(t, gamma)
        assert np.allclose(dx, g["dx"], atol=1e-9) and np.allclose(dy, g["dy"], atol=1e-9)
        (ax, _, ay, _), _ = D.augmented_step(t)
        assert np.allclose(ax, g["dx"], atol=1e-12) and np.allclose(ay, g["dy"], atol=1e-12)


def test_worked_example_recovery_and_rhs():
    g = GOLD["recover_slack_dual"]
    t = _Tiny([[1.0]], H=g["H"], d_s=g["D_s"], r2=g["r2"], r4=g["r4"])
    ds, dz = D.recover_slack_dual(t, np.array(g["dx"], float))
    assert ds.tolist() == g["ds"] and dz.tolist() == g["dz"]
    r1 = np.array(GOLD["condensed_rhs_identity"]["r1"])
    n = len(r1)
    t = _Tiny(np.eye(n), H=np.eye(n), d_s=np.ones(n), r1=r1, r2=np.zeros(n), r4=np.ones(n))
    assert np.allclose(-D.condensed_rhs(t), -(r1 + 1.0), atol=0)


def test_condensation_special_cases():
    """H = 0, delta = 0 -> K = W;  W = 0, H = I, D_s = diag(d) -> K = diag(d);
    G = 0 -> K_gamma = K and r_gamma = condensed rhs."""
    rng = np.random.default_rng(0)
    W = rng.standard_normal((5, 5)); W = W + W.T
    t = _Tiny(W, H=np.zeros((2, 5)), d_s=np.ones(2))
    assert np.array_equal(D.condensed_matrix(t), W)
    d = rng.uniform(1, 2, 5)
    t = _Tiny(np.zeros((5, 5)), H=np.eye(5), d_s=d)
    assert np.allclose(D.condensed_matrix(t), np.diag(d), atol=0)
    t = _Tiny(W, G=np.zeros((2, 5)), r1=rng.standard_normal(5), r3=rng.standard_normal(2))
    assert np.array_equal(D.hykkt_matrix(t, 1e7), D.condensed_matrix(t))
    assert np.array_equal(D.hykkt_rhs(t, 1e7), D.condensed_rhs(t))


@pytest.mark.parametrize("seed", range(5))
def test_schur_eigenvalues_closed_form(seed):
    """Sherman–Morrison–Woodbury: eig(S_gamma) = mu_i / (1 + gamma mu_i), mu_i = eig(G K^{-1} G^T)
    when K is SPD; hence gamma S_gamma -> I."""
    inst = _gen(seed, n=12, me=5, mi=3)
    K = D.condensed_matrix(inst)
    K = K + (1.0 - min(0.0, np.linalg.eigvalsh(K).min())) * np.eye(inst.n)
    G = inst.G_dense()
    mu = np.linalg.eigvalsh(G @ np.linalg.solve(K, G.T))
    spreads = []
    for gamma in (1e3, 1e5, 1e7):
        S = G @ np.linalg.solve(K + gamma * G.T @ G, G.T)
        ev = np.sort(np.linalg.eigvalsh((S + S.T) / 2))
        expect = np.sort(mu / (1 + gamma * mu))
        assert np.allclose(ev, expect, rtol=1e-6, atol=0)
        spreads.append(ev.max() / ev.min())
    assert spreads[0] > spreads[1] > spreads[2] and spreads[2] < 1 + 1e-3
