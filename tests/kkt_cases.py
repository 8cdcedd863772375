"""Shared test helpers: build instances, run the CUDA path through the C ABI and the oracle."""
from __future__ import annotations

import dataclasses

import numpy as np

from inputs import distillation as dist
from inputs.random_kkt import random_instance

E32 = np.zeros(1, np.int32)


@dataclasses.dataclass
class Case:
    """One pattern + B value sets (batch-major arrays)."""
    n: int
    m_e: int
    m_i: int
    w_row: np.ndarray
    w_col: np.ndarray
    g_rowptr: np.ndarray
    g_col: np.ndarray
    h_rowptr: np.ndarray
    h_col: np.ndarray
    w_val: np.ndarray   # [B, nnzW]
    g_val: np.ndarray   # [B, nnzG]
    h_val: np.ndarray
    sigma_x: np.ndarray  # [B, n]
    d_s: np.ndarray      # [B, m_i]
    delta_x: np.ndarray  # [B]
    r1: np.ndarray
    r2: np.ndarray
    r3: np.ndarray
    r4: np.ndarray

    @property
    def B(self):
        return self.w_val.shape[0]


def distillation_case(N, strategy, iterates, instance=0, rhs_seed=3000, inst_obj=None):
    """strategy 1 = HyKKT (rows in G), 0 = Lifted (rows relaxed into H with D)."""
    inst = inst_obj or dist.Instance(N, instance)
    traj = inst.trajectory()
    its = [traj[k] for k in iterates]
    pat = inst.model.pat
    n, m = pat.n, pat.m
    B = len(its)
    rng = np.random.default_rng(rhs_seed)
    r1 = rng.standard_normal((B, n))
    ra = rng.standard_normal((B, m))
    rb = rng.standard_normal((B, m))
    J = np.stack([it.j_val for it in its])
    common = dict(n=n, w_row=pat.w_row, w_col=pat.w_col, w_val=np.stack([it.w_val for it in its]),
                  sigma_x=np.stack([it.sigma_x for it in its]), delta_x=np.zeros(B), r1=r1)
    if strategy == 1:
        return Case(m_e=m, m_i=0, g_rowptr=pat.j_rowptr, g_col=pat.j_col, h_rowptr=E32, h_col=E32[:0],
                    g_val=J, h_val=np.zeros((B, 0)), d_s=np.zeros((B, 0)), r2=np.zeros((B, 0)), r3=ra,
                    r4=np.zeros((B, 0)), **common)
    return Case(m_e=0, m_i=m, g_rowptr=E32, g_col=E32[:0], h_rowptr=pat.j_rowptr, h_col=pat.j_col,
                g_val=np.zeros((B, 0)), h_val=J, d_s=np.stack([it.d_lifted for it in its]), r2=ra,
                r3=np.zeros((B, 0)), r4=rb, **common)


def random_case(n, m_e, m_i, seeds, **kw):
    """B random instances on ONE pattern: the first seed fixes the pattern, values of the others
    are re-drawn on it (with their own SOSC shift)."""
    base = random_instance(n, m_e, m_i, seed=seeds[0], **kw)
    insts = [base]
    for s in seeds[1:]:
        rng = np.random.default_rng(s)
        o = random_instance(n, m_e, m_i, seed=seeds[0], **kw)
        o.w_val = base.w_val * rng.uniform(0.5, 1.5, len(base.w_val))
        o.g_val = base.g_val * rng.uniform(0.5, 1.5, len(base.g_val))
        o.h_val = base.h_val * rng.uniform(0.5, 1.5, len(base.h_val))
        diag = base.w_row == base.w_col
        o.w_val[diag] += 5.0 + 20.0 * rng.uniform()
        o.sigma_x = base.sigma_x * rng.uniform(0.5, 2.0, n)
        o.d_s = base.d_s * rng.uniform(0.5, 2.0, m_i)
        o.r1, o.r2, o.r3, o.r4 = (rng.standard_normal(n), rng.standard_normal(m_i), rng.standard_normal(m_e),
                                  rng.standard_normal(m_i))
        insts.append(o)
    st = lambda f: np.stack([getattr(i, f) for i in insts])
    return Case(n=n, m_e=m_e, m_i=m_i, w_row=base.w_row, w_col=base.w_col, g_rowptr=base.g_rowptr,
                g_col=base.g_col, h_rowptr=base.h_rowptr, h_col=base.h_col, w_val=st("w_val"), g_val=st("g_val"),
                h_val=st("h_val"), sigma_x=st("sigma_x"), d_s=st("d_s"),
                delta_x=np.array([i.delta_x for i in insts], float), r1=st("r1"), r2=st("r2"), r3=st("r3"),
                r4=st("r4"))


def run_oracle(case: Case, b: int, strategy: int, gamma=1e7, leaf=64, perm=None):
    from oracle import kkt as OK
    o = OK.SparseKKT(case.n, case.m_e, case.m_i, case.w_row, case.w_col,
                     case.g_rowptr if case.m_e else E32, case.g_col if case.m_e else E32[:0],
                     case.h_rowptr if case.m_i else E32, case.h_col if case.m_i else E32[:0],
                     strategy=strategy, gamma=gamma, leaf=leaf, perm=perm)
    fail = o.refactor(case.w_val[b], case.g_val[b], case.h_val[b], case.sigma_x[b], case.d_s[b], case.delta_x[b])
    if fail >= 0:
        return o, None, None
    d, info = o.solve(case.r1[b], case.r2[b], case.r3[b], case.r4[b])
    return o, d, info


def run_gpu(case: Case, strategy: int, gamma=1e7, leaf=64, **opts):
    import torch
    from paper_2403_15913_b200 import ckkt
    dev = torch.device("cuda:0")
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev) if a.size else None
    B = case.B
    ctx = ckkt.Context(case.n, case.m_e, case.m_i, case.w_row, case.w_col,
                       case.g_rowptr if case.m_e else None, case.g_col if case.m_e else None,
                       case.h_rowptr if case.m_i else None, case.h_col if case.m_i else None,
                       strategy=strategy, gamma=gamma, leaf=leaf, batch=B, device=0,
                       stream=torch.cuda.current_stream().cuda_stream, **opts)
    notpd = torch.zeros(B, dtype=torch.int32, device=dev)
    minpiv = torch.zeros(B, dtype=torch.int32, device=dev)
    # value arrays must stay alive until the solve completes (zero-copy ABI, include/ckkt.h)
    vals = [T(case.w_val), T(case.g_val), T(case.h_val), T(case.sigma_x), T(case.d_s), T(case.delta_x)]
    ctx.refactor(*vals, notpd, minpiv)
    dx = torch.empty((B, case.n), dtype=torch.float64, device=dev)
    ds = torch.empty((B, case.m_i), dtype=torch.float64, device=dev) if case.m_i else None
    dy = torch.empty((B, case.m_e), dtype=torch.float64, device=dev) if case.m_e else None
    dz = torch.empty((B, case.m_i), dtype=torch.float64, device=dev) if case.m_i else None
    rc, info = ctx.solve(T(case.r1), T(case.r2), T(case.r3), T(case.r4), dx, ds, dy, dz)
    torch.cuda.synchronize()
    em = lambda t, k: t.cpu().numpy() if t is not None else np.zeros((B, 0))
    out = dict(rc=rc, info=info, notpd=notpd.cpu().numpy(), minpiv=minpiv.cpu().numpy(),
               dx=em(dx, case.n), ds=em(ds, case.m_i), dy=em(dy, case.m_e), dz=em(dz, case.m_i), ctx=ctx, vals=vals)
    return out


def block_errors(gpu, b, d_oracle):
    errs = []
    for name, ref in zip(("dx", "ds", "dy", "dz"), d_oracle):
        if len(ref) == 0:
            continue
        got = gpu[name][b]
        errs.append(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))
    return errs


def elementwise_errors(gpu, b, d_oracle):
    """Per block: max_i |d_gpu,i - d_oracle,i| / max_i |d_oracle,i| (every element against the block's
    scale, so no component can hide inside a 2-norm)."""
    errs = []
    for name, ref in zip(("dx", "ds", "dy", "dz"), d_oracle):
        if len(ref) == 0:
            continue
        got = gpu[name][b]
        errs.append(float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300)))
    return errs


def host_kaug_backward_error(case: Case, b: int, d):
    """Componentwise backward error of a step computed on the host from the definition (independent
    of both the GPU path and the oracle): max_i |rho_i| / (|K_aug||d| + |r|)_i."""
    import scipy.sparse as sp
    n, me, mi = case.n, case.m_e, case.m_i
    dx, ds, dy, dz = d
    W = sp.coo_matrix((case.w_val[b], (case.w_row, case.w_col)), shape=(n, n)).tocsr()
    Ws = (W + W.T - sp.diags(W.diagonal())).tocsr()
    G = sp.csr_matrix((case.g_val[b], case.g_col, case.g_rowptr), shape=(me, n)) if me else sp.csr_matrix((0, n))
    H = sp.csr_matrix((case.h_val[b], case.h_col, case.h_rowptr), shape=(mi, n)) if mi else sp.csr_matrix((0, n))
    dg = case.sigma_x[b] + case.delta_x[b]
    r1, r2, r3, r4 = case.r1[b], case.r2[b], case.r3[b], case.r4[b]
    A = abs
    rho1 = -r1 - (Ws @ dx + dg * dx + G.T @ dy + H.T @ dz)
    a1 = A(Ws) @ A(dx) + A(dg * dx) + A(G.T) @ A(dy) + A(H.T) @ A(dz) + A(r1)
    rho2 = -r2 - (case.d_s[b] * ds + dz)
    a2 = A(case.d_s[b] * ds) + A(dz) + A(r2)
    rho3 = -r3 - G @ dx
    a3 = A(G) @ A(dx) + A(r3)
    rho4 = -r4 - (H @ dx + ds)
    a4 = A(H) @ A(dx) + A(ds) + A(r4)
    rho = np.concatenate([rho1, rho2, rho3, rho4])
    a = np.concatenate([a1, a2, a3, a4])
    return float(np.max(np.abs(rho) / np.where(a > 0, a, 1.0)))
