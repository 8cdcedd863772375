"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars (north_star): per block relative step error <= 1e-8, componentwise KKT backward
error <= 1e-10, integer arrays bit-exact, NOT_PD flag identical, k_CG within +-1."""
import numpy as np
import pytest

from kkt_cases import (Case, block_errors, distillation_case, elementwise_errors, host_kaug_backward_error,
                        random_case, run_gpu, run_oracle)

pytestmark = pytest.mark.gpu

STEP_TOL = 1e-8
RES_TOL = 1e-10


def _check(case, strategy, gamma=1e7, leaf=64, step_tol=STEP_TOL):
    g = run_gpu(case, strategy, gamma=gamma, leaf=leaf)
    for b in range(case.B):
        o, d, info = run_oracle(case, b, strategy, gamma=gamma, leaf=leaf)
        if d is None:
            assert g["notpd"][b] == 1
            continue
        assert g["notpd"][b] == 0
        if not info.cg_converged:
            # out of contract (reading R6 cap): both sides must report CG non-convergence
            assert g["info"][b]["status"] == 2 and g["info"][b]["k_cg"] == info.k_cg
            continue
        errs = block_errors(g, b, d)
        assert max(errs) <= step_tol, (b, errs, g["info"][b], info)
        assert max(elementwise_errors(g, b, d)) <= step_tol, (b, elementwise_errors(g, b, d))
        gi = g["info"][b]
        assert gi["rel_res"] <= RES_TOL, gi
        assert abs(gi["k_cg"] - info.k_cg) <= 1, (gi, info)
        got = (g["dx"][b], g["ds"][b], g["dy"][b], g["dz"][b])
        assert host_kaug_backward_error(case, b, got) <= RES_TOL
    return g


@pytest.mark.parametrize("shape", [(30, 8, 6), (41, 0, 12), (25, 10, 0), (60, 20, 15), (1, 0, 0), (7, 3, 0)])
@pytest.mark.parametrize("strategy", [0, 1])
def test_random_instances(shape, strategy):
    n, me, mi = shape
    if strategy == 0 and me > 0:
        pytest.skip("Lifted needs m_e = 0")
    case = random_case(n, me, mi, seeds=[11, 12, 13], sigma_range=(1e-4, 1e4), d_range=(1e-2, 1e6))
    _check(case, strategy, gamma=1e4 if strategy else 0.0, leaf=8)


def test_random_wide_range_lifted():
    case = random_case(40, 0, 20, seeds=[5, 6], d_range=(1e5, 1e12), sigma_range=(1e-8, 1e8))
    _check(case, 0, leaf=16)


@pytest.mark.parametrize("strategy", [0, 1])
def test_distillation_c1(strategy):
    """Config 1 (N=50), several iterates of the synthetic trajectory in one batch."""
    case = distillation_case(50, strategy, iterates=[0, 5, 9, 13, 17])
    _check(case, strategy)


@pytest.mark.parametrize("leaf", [16, 268, 1072])
def test_distillation_leaf_sizes(leaf):
    case = distillation_case(60, 1, iterates=[2, 16])
    _check(case, 1, leaf=leaf)


def test_symbolic_bit_exact_on_device_context():
    """perm, etree, column counts and L pattern exported by a device context equal the oracle."""
    from oracle import kkt as OK
    case = distillation_case(120, 1, iterates=[0])
    g = run_gpu(case, 1, leaf=268)
    perm, parent, cc, Lp, Li = g["ctx"].export_symbolic()
    o = OK.SparseKKT(case.n, case.m_e, 0, case.w_row, case.w_col, case.g_rowptr, case.g_col,
                     np.zeros(1, np.int32), np.zeros(0, np.int32), leaf=268)
    assert np.array_equal(perm, o.perm) and np.array_equal(parent, o.parent)
    assert np.array_equal(cc, o.colcount) and np.array_equal(Lp, o.Lp) and np.array_equal(Li, o.Li)


def test_not_pd_flag_matches_oracle():
    case = random_case(20, 0, 5, seeds=[3, 4, 5])
    case.sigma_x[1] -= 1e3   # instance 1 indefinite
    g = run_gpu(case, 0, leaf=8)
    assert g["notpd"].tolist() == [0, 1, 0]
    assert g["info"][1]["status"] == 1 and np.all(np.isnan(g["dx"][1]))
    o, d, _ = run_oracle(case, 1, 0, leaf=8)
    assert d is None
    for b in (0, 2):
        o, d, info = run_oracle(case, b, 0, leaf=8)
        assert max(block_errors(g, b, d)) <= STEP_TOL


def test_not_pd_instance_in_hykkt_batch():
    """A non-PD instance in a HyKKT batch: flagged and NaN-filled, while the other instances run the
    CG (first pass, Init-CG correction passes, accumulated dx) unaffected and match the oracle."""
    case = random_case(30, 8, 0, seeds=[7, 8, 9])
    case.sigma_x[1] -= 1e9
    g = run_gpu(case, 1, gamma=1e4, leaf=8)
    assert g["notpd"].tolist() == [0, 1, 0]
    assert np.all(np.isnan(g["dx"][1]))
    for b in (0, 2):
        o, d, info = run_oracle(case, b, 1, gamma=1e4, leaf=8)
        assert max(block_errors(g, b, d)) <= STEP_TOL
        assert g["info"][b]["rel_res"] <= RES_TOL


@pytest.mark.parametrize("n,small_panel", [(22, "512"), (30, "1536"), (60, "512")])
def test_dense_fronts_wider_than_16(n, small_panel, monkeypatch):
    """Dense instances whose single front runs the blocked dense path with several 16-column diagonal
    blocks: 16 < w <= 32 on the one-warp path, w = 60 on a whole CTA."""
    monkeypatch.setenv("CKKT_SMALL_PANEL", small_panel)
    case = random_case(n, 4, 0, seeds=[21, 22], density=1.0)
    _check(case, 1, gamma=1e4, leaf=n)
    _check(case, 0, leaf=n) if case.m_i else None


def test_gamma_sweep_stress():
    """Config 5: Sigma log-uniform over [1e-8, 1e8] on all variables, gamma in 1e4..1e8."""
    case = distillation_case(40, 1, iterates=[12])
    rng = np.random.default_rng(4000)
    case.sigma_x[:] = np.exp(rng.uniform(np.log(1e-8), np.log(1e8), case.sigma_x.shape))
    for gamma in (1e4, 1e5, 1e6, 1e7, 1e8):
        _check(case, 1, gamma=gamma)


@pytest.mark.gpu
def test_correction_cg_tolerance_does_not_change_the_step():
    """Reading R6: the refinement passes' CG tolerance (cg_rtol_corr) only changes the work, not the
    result: at 1e-10 and at the default 1e-6 the refined steps meet the same bars and agree."""
    case = distillation_case(50, 1, iterates=[3, 11, 16])
    g_tight = run_gpu(case, 1, cg_rtol_corr=1e-10)
    g_loose = run_gpu(case, 1)
    for b in range(case.B):
        for g in (g_tight, g_loose):
            assert g["info"][b]["rel_res"] <= RES_TOL
        assert g_loose["info"][b]["k_cg"] == g_tight["info"][b]["k_cg"]      # first pass unchanged
        ref = g_tight["dx"][b]
        assert np.linalg.norm(g_loose["dx"][b] - ref) <= STEP_TOL * np.linalg.norm(ref)


def _oracle_first_failure(case, b, strategy, order, gamma=1e7):
    """Position of the first failing pivot of the oracle's column Cholesky run in `order`, or -1."""
    from oracle import kkt as OK
    E32 = np.zeros(1, np.int32)
    o = OK.SparseKKT(case.n, case.m_e, case.m_i, case.w_row, case.w_col,
                     case.g_rowptr if case.m_e else E32, case.g_col if case.m_e else E32[:0],
                     case.h_rowptr if case.m_i else E32, case.h_col if case.m_i else E32[:0],
                     strategy=strategy, gamma=gamma, perm=order)
    return o.refactor(case.w_val[b], case.g_val[b], case.h_val[b], case.sigma_x[b], case.d_s[b], case.delta_x[b])


def _shift_some(case, rng, per_instance=3, shift=1e12):
    """Make each instance indefinite by a large negative shift of Sigma_x on a few random variables;
    the first of them in the elimination order is where a sequential Cholesky first fails."""
    for b in range(case.B):
        idx = rng.choice(case.n, size=per_instance, replace=False)
        case.sigma_x[b, idx] -= shift


@pytest.mark.parametrize("kind", ["random_lifted", "random_hykkt", "distillation_hykkt", "distillation_lifted"])
def test_min_bad_pivot_matches_oracle_first_failure(kind):
    """Reading R9: min_bad_pivot is the original index of the failing column that comes first in
    the internal elimination order.  The oracle's sequential column Cholesky, run in the exported order,
    must fail first at exactly that column (every earlier pivot is a pivot of a PD leading block)."""
    import torch
    rng = np.random.default_rng(hash(kind) % 2**32)
    if kind == "random_lifted":
        case, strategy, gamma, leaf = random_case(60, 0, 20, seeds=[31, 32, 33, 34]), 0, 0.0, 8
    elif kind == "random_hykkt":
        case, strategy, gamma, leaf = random_case(60, 15, 0, seeds=[41, 42, 43]), 1, 1e4, 8
    elif kind == "distillation_hykkt":
        case, strategy, gamma, leaf = distillation_case(50, 1, iterates=[2, 9, 15]), 1, 1e7, 64
    else:
        case, strategy, gamma, leaf = distillation_case(50, 0, iterates=[4, 12]), 0, 0.0, 64
    _shift_some(case, rng)
    g = run_gpu(case, strategy, gamma=gamma if gamma else 1e7, leaf=leaf)
    order = g["ctx"].export_elimination_order()
    assert sorted(order.tolist()) == list(range(case.n))
    for b in range(case.B):
        k = _oracle_first_failure(case, b, strategy, order, gamma=gamma if gamma else 1e7)
        assert k >= 0 and g["notpd"][b] == 1
        assert g["minpiv"][b] == order[k], (b, k, g["minpiv"][b], order[k])
    # a positive definite instance reports -1
    case2 = distillation_case(50, 1, iterates=[5])
    g2 = run_gpu(case2, 1, leaf=64)
    assert g2["notpd"][0] == 0 and g2["minpiv"][0] == -1


def test_refactor_with_new_value_buffers_matches_fresh_context():
    """Zero-copy ABI: a second refactor on the same context with DIFFERENT value buffers (the first ones
    freed) must give exactly what a fresh context gives on those values: the captured CG graph reads
    only context-owned copies."""
    import torch
    from paper_2403_15913_b200 import ckkt
    dev = torch.device("cuda:0")
    case = distillation_case(60, 1, iterates=[3, 14])
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)

    def solve(ctx, k):
        vals = [T(case.w_val[k]), T(case.g_val[k]), None, T(case.sigma_x[k]), None, None]
        ctx.refactor(*vals)
        dx = torch.empty(case.n, dtype=torch.float64, device=dev)
        dy = torch.empty(case.m_e, dtype=torch.float64, device=dev)
        rc, info = ctx.solve(T(case.r1[k]), None, T(case.r3[k]), None, dx, None, dy, None)
        torch.cuda.synchronize()
        del vals
        return dx.cpu().numpy(), dy.cpu().numpy(), info[0]

    mk = lambda: ckkt.Context(case.n, case.m_e, 0, case.w_row, case.w_col, case.g_rowptr, case.g_col, None, None,
                              strategy=1, device=0, stream=torch.cuda.current_stream().cuda_stream)
    ctx = mk()
    solve(ctx, 0)
    torch.cuda.empty_cache()
    _ = torch.full((4 * case.g_val.shape[1],), float("nan"), dtype=torch.float64, device=dev)  # reuse freed blocks
    dx1, dy1, i1 = solve(ctx, 1)
    dx2, dy2, i2 = solve(mk(), 1)
    assert i1["k_cg"] == i2["k_cg"] and i1["rel_res_unrefined"] == i2["rel_res_unrefined"], (i1, i2)
    assert np.array_equal(dx1, dx2) and np.array_equal(dy1, dy2)


@pytest.mark.parametrize("strategy", [1, 0])
def test_k_shard_bit_identity(strategy):
    """per-instance results do not depend on how a batch is sharded.  8 instances solved as
    1 context x 8, 2 x 4 and 8 x 1 give bit-identical steps (deterministic kernels, same arithmetic for
    every batch size)."""
    cases = [distillation_case(60, strategy, iterates=[k], rhs_seed=3000 + k) for k in (0, 2, 5, 7, 9, 11, 14, 17)]
    c0 = cases[0]

    def stack(sel):
        f = {k: getattr(c0, k) for k in ("n", "m_e", "m_i", "w_row", "w_col", "g_rowptr", "g_col", "h_rowptr",
                                         "h_col")}
        for name in ("w_val", "g_val", "h_val", "sigma_x", "d_s", "delta_x", "r1", "r2", "r3", "r4"):
            f[name] = np.concatenate([getattr(cases[i], name) for i in sel], axis=0)
        return Case(**f)

    results = {}
    for per in (8, 4, 1):
        outs = []
        for s0 in range(0, 8, per):
            g = run_gpu(stack(range(s0, s0 + per)), strategy, leaf=64)
            outs.append(np.concatenate([g["dx"], g["ds"], g["dy"], g["dz"]], axis=1))
            for b in range(per):
                assert g["info"][b]["status"] == 0, g["info"][b]
        results[per] = np.concatenate(outs, axis=0)
    assert np.array_equal(results[8].view(np.int64), results[4].view(np.int64))
    assert np.array_equal(results[8].view(np.int64), results[1].view(np.int64))


@pytest.mark.parametrize("strategy", [1, 0])
def test_front_paths_bit_identical(strategy, monkeypatch):
    """The factorization's front paths (one-warp fronts and whole-CTA fronts) use the same arithmetic in the
    same order, so moving every front onto the CTA path (CKKT_SMALL_PANEL=64) or letting more fronts onto
    the one-warp path must not change a single bit of the step."""
    case = distillation_case(120, strategy, iterates=[4, 13])
    ref = run_gpu(case, strategy, leaf=268)
    for panel in ("64", "1536"):
        monkeypatch.setenv("CKKT_SMALL_PANEL", panel)
        g = run_gpu(case, strategy, leaf=268)
        for name in ("dx", "ds", "dy", "dz"):
            assert np.array_equal(g[name].view(np.int64), ref[name].view(np.int64)), (panel, name)


@pytest.mark.parametrize("strategy", [1, 0])
def test_iterate_host_matches_device_calls(strategy):
    """ckkt_iterate_host (values and right-hand sides from pinned HOST buffers, the right-hand sides on the
    context's second stream during the factorization) returns bit-for-bit the step and info of
    ckkt_refactor + ckkt_solve on device buffers, on a batch of two distillation iterates, twice in a row
    (the staging buffers are reused)."""
    import torch
    case = distillation_case(50, strategy, iterates=[2, 11])
    g = run_gpu(case, strategy, leaf=64)
    ctx, B = g["ctx"], case.B
    P = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).pin_memory() if a.size else None
    E = lambda k: torch.empty((B, k), dtype=torch.float64).pin_memory() if k else None
    hv = [P(case.w_val), P(case.g_val), P(case.h_val), P(case.sigma_x), P(case.d_s), P(case.delta_x)]
    hr = [P(case.r1), P(case.r2), P(case.r3), P(case.r4)]
    for _ in range(2):
        out = [E(case.n), E(case.m_i), E(case.m_e), E(case.m_i)]
        rc, info = ctx.iterate_host(*hv, *hr, *out)
        assert rc == g["rc"]
        for name, t in zip(("dx", "ds", "dy", "dz"), out):
            if t is not None:
                assert np.array_equal(t.numpy(), g[name]), name
        for b in range(B):
            assert info[b] == g["info"][b]
