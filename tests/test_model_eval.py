"""NEXT-4 (the model derivatives are evaluated on the GPU): the distillation
model's Jacobian, Lagrangian Hessian, residual and objective gradient by the CUDA kernel
(ckkt_distillation_eval) against the host generator inputs/distillation.py — itself pinned against FP64
autograd in tests/test_inputs.py — on iterates of the trajectory, with the gradient scaling of R14."""
import ctypes

import numpy as np
import pytest

from inputs import distillation as dist
from paper_2403_15913_b200 import ckkt


def test_argument_checks():
    """Argument validation happens before any device work (no GPU needed)."""
    L = ckkt.lib()
    prm = ckkt.distillation_params(dist.Params())
    dummy = ctypes.c_void_p(8)
    assert L.ckkt_distillation_eval(0, 1, ctypes.byref(prm), dummy, dummy, None, None, 1.0, None, None, None, None,
                                    None) == ckkt.CKKT_INVALID_ARG
    assert L.ckkt_distillation_eval(5, 0, ctypes.byref(prm), dummy, dummy, None, None, 1.0, None, None, None, None,
                                    None) == ckkt.CKKT_INVALID_ARG
    assert L.ckkt_distillation_eval(5, 1, None, dummy, dummy, None, None, 1.0, None, None, None, None,
                                    None) == ckkt.CKKT_INVALID_ARG
    assert L.ckkt_distillation_eval(5, 1, ctypes.byref(prm), dummy, None, None, None, 1.0, None, None, None, None,
                                    None) == ckkt.CKKT_INVALID_ARG
    bad = ckkt.distillation_params(dist.Params())
    bad.feed_tray = 40
    assert L.ckkt_distillation_eval(5, 1, ctypes.byref(bad), dummy, dummy, None, None, 1.0, None, None, None, None,
                                    None) == ckkt.CKKT_INVALID_ARG
    bad = ckkt.distillation_params(dist.Params())
    bad.M[3] = 0.0
    assert L.ckkt_distillation_eval(5, 1, ctypes.byref(bad), dummy, dummy, None, None, 1.0, None, None, None, None,
                                    None) == ckkt.CKKT_INVALID_ARG
    # c needs xbar0
    assert L.ckkt_distillation_eval(5, 1, ctypes.byref(prm), None, dummy, None, None, 1.0, None, None, dummy, None,
                                    None) == ckkt.CKKT_INVALID_ARG


def _close(got, ref, tol=4e-15):
    scale = max(np.max(np.abs(ref)), 1e-300)
    return float(np.max(np.abs(got - ref)) / scale) <= tol


@pytest.mark.gpu
@pytest.mark.parametrize("N", [1, 50, 1000])
def test_gpu_model_eval_matches_host_generator(N):
    import torch
    dev = torch.device("cuda:0")
    inst = dist.Instance(N, 3)
    md = inst.model
    mus = dist.mu_schedule()
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
    for k in (1, 10):
        it = inst.iterate(k, mus[k // 3])
        lam = it.lam
        rs, sf = inst.row_scale, inst.obj_scale
        jv = torch.empty(md.pat.j_col.size, dtype=torch.float64, device=dev)
        wv = torch.empty(md.pat.w_row.size, dtype=torch.float64, device=dev)
        c = torch.empty(md.m, dtype=torch.float64, device=dev)
        g = torch.empty(md.n, dtype=torch.float64, device=dev)
        ckkt.distillation_eval(N, md.p, T(inst.xbar0), T(it.v), T(lam), T(rs), sf, jv, wv, c, g)
        torch.cuda.synchronize()
        j_ref = md.jacobian_values(it.v) * rs[inst.rows_of_entries]
        w_ref = md.hessian_values(it.v, lam * rs, sf)
        c_ref = rs * md.residual(it.v, inst.xbar0)
        g_ref = sf * md.grad_f(it.v)
        assert _close(jv.cpu().numpy(), j_ref)
        assert _close(wv.cpu().numpy(), w_ref)
        assert _close(g.cpu().numpy(), g_ref)
        # the residual is a difference of O(1) terms that cancel to ~1e-2 at these iterates: absolute bar
        assert np.max(np.abs(c.cpu().numpy() - c_ref)) <= 1e-12
        # the iterate's own values (the GPU path's inputs) are reproduced: J and W equal the generator's
        assert _close(jv.cpu().numpy(), it.j_val) and _close(wv.cpu().numpy(), it.w_val)


@pytest.mark.gpu
def test_gpu_model_eval_batch_and_defaults():
    """Batch-major evaluation of several instances in one launch equals per-instance calls; NULL lam /
    row_scale mean 0 / 1."""
    import torch
    dev = torch.device("cuda:0")
    N = 40
    insts = [dist.Instance(N, i) for i in range(3)]
    md = insts[0].model
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
    V = T(np.stack([i.v for i in insts]))
    jv = torch.empty((3, md.pat.j_col.size), dtype=torch.float64, device=dev)
    wv = torch.empty((3, md.pat.w_row.size), dtype=torch.float64, device=dev)
    ckkt.distillation_eval(N, md.p, T(insts[0].xbar0), V, None, None, 1.0, jv, wv, None, None, batch=3)
    torch.cuda.synchronize()
    for b, inst in enumerate(insts):
        assert _close(jv[b].cpu().numpy(), md.jacobian_values(inst.v))
        assert _close(wv[b].cpu().numpy(), md.hessian_values(inst.v, np.zeros(md.m), 1.0))
