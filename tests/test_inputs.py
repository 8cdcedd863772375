"""Generator pins: dimensions from Table I, derivatives against autograd."""
import json
import os

import numpy as np
import pytest

from inputs import distillation as dist

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def test_table1_dimensions():
    """n = 67(N+1) reproduces Table I's n column exactly."""
    g = GOLD["table1_dimensions"]
    for N, n in zip(g["N"], g["n"]):
        assert dist.dimensions(N)[0] == n


@pytest.mark.parametrize("N", [1, 2, 7, 100])
def test_pattern_counts(N):
    pat = dist.build_pattern(N)
    assert pat.n == 67 * (N + 1) and pat.m == 66 * (N + 1)
    assert pat.j_rowptr[-1] == 288 * N + 100
    assert len(pat.w_row) == 96 * N + 32
    assert np.all(pat.w_row >= pat.w_col)
    for i in range(pat.m):
        c = pat.j_col[pat.j_rowptr[i]:pat.j_rowptr[i + 1]]
        assert np.all(np.diff(c) > 0) and c.min() >= 0 and c.max() < pat.n
    # block-banded: no coordinate couples stages more than one apart
    rows = np.repeat(np.arange(pat.m), np.diff(pat.j_rowptr))
    st_row = rows // 66
    st_col = pat.j_col // 67
    assert np.all((st_col == st_row) | (st_col == st_row - 1))


def _torch_model(md, xbar0):
    import torch
    p, M = md.p, md.M

    def g_fn(v):
        S = v.reshape(md.N + 1, 67)
        x, y, u, L, V = S[:, :32], S[:, 32:64], S[:, 64], S[:, 65], S[:, 66]
        a = p.alpha
        vle = a * x / (1 + (a - 1) * x)
        out = [torch.cat([x[0] - torch.as_tensor(xbar0), (L[0] - u[0] * p.D)[None], (V[0] - L[0] - p.D)[None], y[0] - vle[0]])]
        for t in range(1, md.N + 1):
            Lt, Vt = L[t], V[t]
            St = p.F + Lt
            xt, yt, xp = x[t], y[t], x[t - 1]
            xd = []
            xd.append(Vt * (yt[1] - xt[0]) / M[0])
            for k in range(1, 31):
                if k < 16:
                    xd.append((Lt * (xt[k - 1] - xt[k]) - Vt * (yt[k] - yt[k + 1])) / M[k])
                elif k == 16:
                    xd.append((p.F * p.x_f + Lt * xt[15] - St * xt[16] - Vt * (yt[16] - yt[17])) / M[k])
                else:
                    xd.append((St * (xt[k - 1] - xt[k]) - Vt * (yt[k] - yt[k + 1])) / M[k])
            xd.append((St * xt[30] - (p.F - p.D) * xt[31] - Vt * yt[31]) / M[31])
            bal = (xt - xp) / md.dt - torch.stack(xd)
            out.append(torch.cat([(Lt - u[t] * p.D)[None], (Vt - Lt - p.D)[None], yt - vle[t], bal]))
        return torch.cat(out)

    def f_fn(v):
        S = v.reshape(md.N + 1, 67)
        return (p.w_x * (S[1:, 0] - p.xbar1) ** 2 + p.rho * (S[1:, 64] - p.ubar) ** 2).sum()

    return g_fn, f_fn


@pytest.mark.parametrize("N", [1, 3])
def test_derivatives_vs_autograd(N):
    """J and W = ∇²f + Σλ∇²g of the hand-coded generator equal FP64 autograd."""
    import torch
    md = dist.Model(N)
    rng = np.random.default_rng(5)
    v = rng.uniform(0.1, 0.9, md.n)
    v.reshape(N + 1, 67)[:, 64] = rng.uniform(1.5, 3.0, N + 1)
    lam = rng.standard_normal(md.m)
    xbar0 = rng.uniform(0.1, 0.9, 32)
    g_fn, f_fn = _torch_model(md, xbar0)
    vt = torch.tensor(v, dtype=torch.float64)
    g_ref = g_fn(vt).numpy()
    assert np.allclose(md.residual(v, xbar0), g_ref, atol=1e-12, rtol=0)
    Jref = torch.autograd.functional.jacobian(g_fn, vt).numpy()
    pat = md.pat
    J = np.zeros((md.m, md.n))
    rows = np.repeat(np.arange(md.m), np.diff(pat.j_rowptr))
    J[rows, pat.j_col] = md.jacobian_values(v)
    assert np.abs(J - Jref).max() < 1e-10
    assert np.all(Jref[J == 0] == 0)  # pattern covers every structural nonzero
    lt = torch.tensor(lam)
    Href = torch.autograd.functional.hessian(lambda z: f_fn(z) + lt @ g_fn(z), vt).numpy()
    W = np.zeros((md.n, md.n))
    W[pat.w_row, pat.w_col] = md.hessian_values(v, lam)
    W = W + np.tril(W, -1).T
    assert np.abs(W - Href).max() < 1e-10 * max(1.0, np.abs(Href).max())
    assert np.all(np.abs(Href[W == 0]) < 1e-12)
    vv = vt.clone().requires_grad_()
    f_fn(vv).backward()
    assert np.allclose(md.grad_f(v), vv.grad.numpy(), atol=1e-10)


def test_trajectory_feasible_and_bounded():
    inst = dist.Instance(20)
    md = inst.model
    assert np.abs(md.residual(inst.v, inst.xbar0)).max() < 1e-10
    its = inst.trajectory()
    assert len(its) == 18
    mus = [it.mu for it in its]
    assert mus[0] == 0.1 and abs(mus[-1] - 1e-7) < 1e-20 and all(a >= b for a, b in zip(mus, mus[1:]))
    for it in its:
        u = it.v.reshape(21, 67)[:, 64]
        assert np.all((u > 1) & (u < 5))
        sig = it.sigma_x.reshape(21, 67)
        assert np.all(sig[:, 64] > 0) and np.all(sig[:, :64] == 0) and np.all(sig[:, 65:] == 0)
        assert np.all(it.d_lifted >= 2 * it.mu / dist.TAU ** 2 * (1 - 1e-12))


def test_mu_schedule_formula():
    """mu' = max(tol/10, min(0.2 mu, mu^1.5)): 0.1 -> 0.02; 0.01 -> 0.001."""
    mus = dist.mu_schedule()
    assert abs(mus[1] - 0.02) < 1e-15
    assert abs(max(1e-7, min(0.2 * 0.01, 0.01 ** 1.5)) - 0.001) < 1e-15


def test_gradient_scaling_reading_r14():
    """Scaled iterates: every Jacobian row has max |entry| <= 100 at the base point, and the
    scaled W equals s_f grad^2 f + sum_r (lam_r s_r) grad^2 g_r (autograd on the scaled Lagrangian)."""
    import torch
    inst = dist.Instance(3)
    md = inst.model
    it = inst.iterate(0, 0.1)
    base = md.jacobian_values(inst.v) * inst.row_scale[inst.rows_of_entries]
    rowmax = np.zeros(md.m)
    np.maximum.at(rowmax, inst.rows_of_entries, np.abs(base))
    assert rowmax.max() <= 100.0 * (1 + 1e-12)
    g_fn, f_fn = _torch_model(md, inst.xbar0)
    vt = torch.tensor(it.v)
    sl = torch.tensor(it.lam * inst.row_scale)
    Href = torch.autograd.functional.hessian(lambda z: inst.obj_scale * f_fn(z) + sl @ g_fn(z), vt).numpy()
    pat = md.pat
    W = np.zeros((md.n, md.n))
    W[pat.w_row, pat.w_col] = it.w_val
    W = W + np.tril(W, -1).T
    assert np.abs(W - Href).max() < 1e-9 * max(1.0, np.abs(Href).max())
    Jref = torch.autograd.functional.jacobian(g_fn, vt).numpy() * inst.row_scale[:, None]
    J = np.zeros((md.m, md.n))
    J[inst.rows_of_entries, pat.j_col] = it.j_val
    assert np.abs(J - Jref).max() < 1e-10
