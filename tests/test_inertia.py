"""Inertia correction (reading R15): the oracle's delta_x search
pinned to closed forms and to dense eigenvalues, and the C-ABI ckkt_refactor_inertia against it."""
from __future__ import annotations

import math

import numpy as np
import pytest
import scipy.sparse as sp

from inputs.random_kkt import random_instance
from oracle import kkt as K
from kkt_cases import E32, distillation_case, random_case


def _diag_kkt(wdiag, strategy=K.HYKKT):
    n = len(wdiag)
    idx = np.arange(n, dtype=np.int32)
    o = K.SparseKKT(n, 0, 0, idx, idx, E32, E32[:0], E32, E32[:0], strategy=strategy, leaf=4)
    return o, np.asarray(wdiag, float)


def test_pd_needs_no_regularization():
    """W > 0: accepted at delta = 0 after one factorization."""
    o, w = _diag_kkt([2.0, 1.0, 3.0])
    assert K.inertia_correction(o, w, [], [], np.zeros(3), []) == (0.0, 1, False)


def test_diag_minus_one_closed_form():
    """W = diag(-1, 1), no constraints (SPEC example): K = W + delta I is PD iff delta > 1.
    ||W||_inf = 1, so the schedule is 0, 1e-4 * 8^k; the first value above 1 has
    k = ceil(log_8(1e4)) = 5, i.e. delta = 1e-4 * 8^5 = 3.2768 after k + 2 = 7 factorizations."""
    o, w = _diag_kkt([-1.0, 1.0])
    delta, trials, failed = K.inertia_correction(o, w, [], [], np.zeros(2), [])
    k = math.ceil(math.log(1e4, 8))
    assert not failed and trials == k + 2
    assert delta == pytest.approx(1e-4 * 8 ** k, rel=1e-15) and delta == pytest.approx(3.2768, rel=1e-15)


def test_norm_scales_first_delta():
    """W = diag(-50, 30): ||W||_inf = 50, schedule 5e-3 * 8^k; first above 50: k = 5 (163.84)."""
    o, w = _diag_kkt([-50.0, 30.0])
    delta, trials, failed = K.inertia_correction(o, w, [], [], np.zeros(2), [])
    assert (trials, failed) == (7, False) and delta == pytest.approx(5e-3 * 8 ** 5, rel=1e-15)


def test_warm_start_from_last_delta():
    """delta_last = 0.9: first nonzero trial 0.3 (fails, needs > 1), then 2.4."""
    o, w = _diag_kkt([-1.0, 1.0])
    delta, trials, failed = K.inertia_correction(o, w, [], [], np.zeros(2), [], delta_last=0.9)
    assert (trials, failed) == (3, False) and delta == pytest.approx(2.4, rel=1e-15)


def test_gives_up_on_non_finite():
    """A NaN in W can never give a positive pivot; its NaN norm ends the search after one trial."""
    o, w = _diag_kkt([np.nan, 1.0])
    assert K.inertia_correction(o, w, [], [], np.zeros(2), []) == (0.0, 1, True)


def test_gives_up_above_cap():
    """W = diag(-5e40, 1): schedule 0, 5e36 * 8^k; PD needs delta > 5e40 but 5e36 * 8^4 = 2.048e40
    exceeds the 1e40 cap, so the search stops after 5 factorizations at delta = 2.56e39."""
    o, w = _diag_kkt([-5e40, 1.0])
    delta, trials, failed = K.inertia_correction(o, w, [], [], np.zeros(2), [])
    assert failed and trials == 5 and delta == pytest.approx(2.56e39, rel=1e-15)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_accepted_delta_minimal_and_inertia(seed):
    """Random HyKKT instances made indefinite by a negative Sigma shift.  By dense eigenvalues:
    K_gamma(delta) > 0 at the accepted delta and not at the schedule's previous value; and the
    unreduced [K(delta) G^T; G 0] then has inertia (n, 0, m_e) (congruence, reading R9)."""
    n, me = 14, 5
    inst = random_instance(n, me, 0, seed=seed)
    shift = [-3.0, -30.0, -0.5, -300.0][seed]
    sig = inst.sigma_x + shift
    gamma = 1e2
    o = K.SparseKKT(n, me, 0, inst.w_row, inst.w_col, inst.g_rowptr, inst.g_col, E32, E32[:0],
                    strategy=K.HYKKT, gamma=gamma, leaf=4)
    delta, trials, failed = K.inertia_correction(o, inst.w_val, inst.g_val, [], sig, [])
    assert not failed and trials >= 2
    W = sp.coo_matrix((inst.w_val, (inst.w_row, inst.w_col)), shape=(n, n)).toarray()
    W = W + np.tril(W, -1).T
    G = sp.csr_matrix((inst.g_val, inst.g_col, inst.g_rowptr), shape=(me, n)).toarray()
    Kg = lambda d: W + np.diag(sig + d) + gamma * G.T @ G
    assert np.linalg.eigvalsh(Kg(delta)).min() > 0
    prev = 0.0 if trials == 2 else delta / 8
    assert np.linalg.eigvalsh(Kg(prev)).min() < 0
    Ka = np.block([[W + np.diag(sig + delta), G.T], [G, np.zeros((me, me))]])
    ev = np.linalg.eigvalsh(Ka)
    assert (ev > 0).sum() == n and (ev < 0).sum() == me


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", [K.HYKKT, K.LIFTED])
def test_gpu_inertia_vs_oracle(strategy):
    """ckkt_refactor_inertia on a batch of distillation iterates with Sigma shifted by
    (0, -1, -40, -3000): per instance the same trial count and delta as the oracle (delta to 1e-13:
    ||W||_inf is summed in another order), NOT_PD cleared, and the step at that delta matches the
    oracle's within the parity bar."""
    import torch
    from paper_2403_15913_b200 import ckkt
    case = distillation_case(12, strategy, [2, 5, 9, 14])
    shifts = np.array([0.0, -1.0, -40.0, -3000.0])
    case.sigma_x = case.sigma_x + shifts[:, None]
    dev = torch.device("cuda:0")
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev) if a.size else None
    B = case.B
    ctx = ckkt.Context(case.n, case.m_e, case.m_i, case.w_row, case.w_col,
                       case.g_rowptr if case.m_e else None, case.g_col if case.m_e else None,
                       case.h_rowptr if case.m_i else None, case.h_col if case.m_i else None,
                       strategy=strategy, leaf=64, batch=B, device=0,
                       stream=torch.cuda.current_stream().cuda_stream)
    vals = [T(case.w_val), T(case.g_val), T(case.h_val), T(case.sigma_x), T(case.d_s)]
    dx_delta = torch.zeros(B, dtype=torch.float64, device=dev)
    notpd = torch.ones(B, dtype=torch.int32, device=dev)
    rc, deltas, trials = ctx.refactor_inertia(*vals, dx_delta, None, notpd)
    assert rc == ckkt.CKKT_OK and not notpd.cpu().numpy().any()
    assert np.array_equal(dx_delta.cpu().numpy(), deltas)
    dx = torch.empty((B, case.n), dtype=torch.float64, device=dev)
    ds = torch.empty((B, case.m_i), dtype=torch.float64, device=dev) if case.m_i else None
    dy = torch.empty((B, case.m_e), dtype=torch.float64, device=dev) if case.m_e else None
    dz = torch.empty((B, case.m_i), dtype=torch.float64, device=dev) if case.m_i else None
    ctx.solve(T(case.r1), T(case.r2), T(case.r3), T(case.r4), dx, ds, dy, dz)
    torch.cuda.synchronize()
    assert trials[0] == 1 and deltas[0] == 0.0 and trials[-1] > 2
    for b in range(B):
        o = K.SparseKKT(case.n, case.m_e, case.m_i, case.w_row, case.w_col,
                        case.g_rowptr if case.m_e else E32, case.g_col if case.m_e else E32[:0],
                        case.h_rowptr if case.m_i else E32, case.h_col if case.m_i else E32[:0],
                        strategy=strategy, leaf=64)
        d_o, t_o, f_o = K.inertia_correction(o, case.w_val[b], case.g_val[b], case.h_val[b], case.sigma_x[b],
                                             case.d_s[b])
        assert not f_o and trials[b] == t_o, (b, trials[b], t_o)
        assert deltas[b] == pytest.approx(d_o, rel=1e-13, abs=0)
        d_ref, _ = o.solve(case.r1[b], case.r2[b], case.r3[b], case.r4[b])
        ref = d_ref[0]
        got = dx[b].cpu().numpy()
        assert np.linalg.norm(got - ref) <= 1e-8 * max(np.linalg.norm(ref), 1e-300), b


@pytest.mark.gpu
def test_gpu_inertia_warm_start_and_failure():
    """delta_last warm start (first nonzero delta = delta_last / 3) and a NaN instance that gives up
    (CKKT_NOT_PD, flag set) while the other instance of the batch is accepted."""
    import torch
    from paper_2403_15913_b200 import ckkt
    case = random_case(16, 4, 0, [7, 8])
    case.sigma_x = case.sigma_x - np.array([[60.0], [0.0]])
    case.w_val[1, 0] = np.nan
    dev = torch.device("cuda:0")
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev) if a.size else None
    ctx = ckkt.Context(case.n, case.m_e, 0, case.w_row, case.w_col, case.g_rowptr, case.g_col, None, None,
                       strategy=ckkt.CKKT_HYKKT, leaf=8, batch=2, device=0,
                       stream=torch.cuda.current_stream().cuda_stream)
    vals = [T(case.w_val), T(case.g_val), None, T(case.sigma_x), None]
    dd = torch.zeros(2, dtype=torch.float64, device=dev)
    notpd = torch.zeros(2, dtype=torch.int32, device=dev)
    rc, deltas, trials = ctx.refactor_inertia(*vals, dd, np.array([1.0, 0.0]), notpd)
    assert rc == ckkt.CKKT_NOT_PD
    assert notpd.cpu().numpy().tolist() == [0, 1]
    o = K.SparseKKT(case.n, case.m_e, 0, case.w_row, case.w_col, case.g_rowptr, case.g_col, E32, E32[:0],
                    strategy=K.HYKKT, leaf=8)
    d_o, t_o, f_o = K.inertia_correction(o, case.w_val[0], case.g_val[0], [], case.sigma_x[0], [], delta_last=1.0)
    assert not f_o and trials[0] == t_o and deltas[0] == d_o  # warm start: exact (no norm involved)
    assert deltas[0] == pytest.approx(8.0 ** (t_o - 2) / 3.0, rel=1e-15)
    d1, t1, f1 = K.inertia_correction(o, case.w_val[1], case.g_val[1], [], case.sigma_x[1], [])
    assert f1 and trials[1] == t1
