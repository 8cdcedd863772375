"""GPU parity at the bench's sizes and launch configuration (leaf 1072, HyKKT gamma = 1e7 / Lifted).

* config 2 (N = 1000): element-wise against the oracle on several iterates of the trajectory;
* config 3 (N = 50 000, the size bench.py times): element-wise against the oracle for one HyKKT
  iterate (the oracle's sparse Cholesky finishes in well under a minute at this size), and the
  size-independent properties for both strategies — status OK, componentwise backward error of the
  unreduced system <= 1e-10, recomputed on the host from the definition (scipy), independent of
  both the CUDA path and the oracle;
* a batch of independent NMPC instances (different initial states, one pattern) in one context,
  the single-GPU slice of config 4, each instance against the oracle.
"""
import numpy as np
import pytest

from inputs import distillation as dist
from kkt_cases import (Case, block_errors, distillation_case, elementwise_errors, host_kaug_backward_error, run_gpu,
                        run_oracle)

pytestmark = pytest.mark.gpu

STEP_TOL = 1e-8
RES_TOL = 1e-10
LEAF = 1072  # bench.py's launch configuration


def _compare(case, strategy, g, b, oracle_leaf=LEAF):
    o, d, info = run_oracle(case, b, strategy, gamma=1e7, leaf=oracle_leaf)
    assert d is not None and g["notpd"][b] == 0
    errs = block_errors(g, b, d)
    assert max(errs) <= STEP_TOL, (b, errs, g["info"][b], info)
    ew = elementwise_errors(g, b, d)
    assert max(ew) <= STEP_TOL, (b, ew)
    assert abs(g["info"][b]["k_cg"] - info.k_cg) <= 1, (g["info"][b], info)


@pytest.mark.parametrize("strategy", [1, 0])
def test_c2_trajectory_vs_oracle(strategy):
    case = distillation_case(1000, strategy, iterates=[0, 9, 17])
    g = run_gpu(case, strategy, leaf=LEAF)
    for b in range(case.B):
        assert g["info"][b]["status"] == 0, g["info"][b]
        assert g["info"][b]["rel_res"] <= RES_TOL
        _compare(case, strategy, g, b)


@pytest.fixture(scope="module")
def c3_instance():
    return dist.Instance(50000)


def test_c3_full_size_hykkt_vs_oracle(c3_instance):
    case = distillation_case(50000, 1, iterates=[9], inst_obj=c3_instance)
    g = run_gpu(case, 1, leaf=LEAF)
    info = g["info"][0]
    assert info["status"] == 0 and info["rel_res"] <= RES_TOL, info
    got = (g["dx"][0], g["ds"][0], g["dy"][0], g["dz"][0])
    assert host_kaug_backward_error(case, 0, got) <= RES_TOL
    _compare(case, 1, g, 0)


def test_c3_full_size_lifted_vs_oracle(c3_instance):
    case = distillation_case(50000, 0, iterates=[9], inst_obj=c3_instance)
    g = run_gpu(case, 0, leaf=LEAF)
    info = g["info"][0]
    assert info["status"] == 0 and info["rel_res"] <= RES_TOL, info
    got = (g["dx"][0], g["ds"][0], g["dy"][0], g["dz"][0])
    assert host_kaug_backward_error(case, 0, got) <= RES_TOL
    assert np.all(np.isfinite(g["dx"][0]))
    _compare(case, 0, g, 0)


def test_c3_run_to_run_bit_identical(c3_instance):
    """Five refactor+solve calls on the same C3 inputs (bench.py's launch configuration) return
    bit-identical steps: every reduction has a fixed order and the persistent kernels' cross-CTA
    dependencies are acquire/release synchronised (a race would show up as run-to-run noise)."""
    import torch
    case = distillation_case(50000, 1, iterates=[13], inst_obj=c3_instance)
    g = run_gpu(case, 1, leaf=LEAF)
    ctx, vals = g["ctx"], g["vals"]
    dev = torch.device("cuda:0")
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
    r1, r3 = T(case.r1), T(case.r3)
    ref = (g["dx"][0].copy(), g["dy"][0].copy())
    for rep in range(5):
        ctx.refactor(*vals)
        dx = torch.empty((1, case.n), dtype=torch.float64, device=dev)
        dy = torch.empty((1, case.m_e), dtype=torch.float64, device=dev)
        rc, info = ctx.solve(r1, None, r3, None, dx, None, dy, None)
        assert rc == 0
        assert np.array_equal(dx.cpu().numpy()[0], ref[0]) and np.array_equal(dy.cpu().numpy()[0], ref[1]), rep


def _batch_of_instances(N, instances, iterate, strategy):
    """One iterate of each instance's trajectory, stacked into one batch on the shared pattern."""
    cases = [distillation_case(N, strategy, iterates=[iterate], instance=i, rhs_seed=3000 + i) for i in instances]
    c0 = cases[0]
    stack = lambda name: np.concatenate([getattr(c, name) for c in cases], axis=0)
    fields = {f: getattr(c0, f) for f in ("n", "m_e", "m_i", "w_row", "w_col", "g_rowptr", "g_col", "h_rowptr",
                                          "h_col")}
    for name in ("w_val", "g_val", "h_val", "sigma_x", "d_s", "delta_x", "r1", "r2", "r3", "r4"):
        fields[name] = stack(name)
    return Case(**fields)


def test_batched_instances_vs_oracle():
    case = _batch_of_instances(200, instances=[0, 1, 2, 3], iterate=12, strategy=1)
    g = run_gpu(case, 1, leaf=LEAF)
    assert case.B == 4
    for b in range(case.B):
        assert g["info"][b]["status"] == 0 and g["info"][b]["rel_res"] <= RES_TOL, g["info"][b]
        _compare(case, 1, g, b)
