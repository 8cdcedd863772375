"""CPU checks of the C ABI: libckkt.so loads, exports every symbol include/ckkt.h declares, and its
host-only symbolic analysis (device = -1) is bit-exact with the oracle's independent implementation."""
import ctypes
import os
import re

import numpy as np
import pytest

from inputs import distillation as dist
from inputs.random_kkt import random_instance
from oracle import kkt as OK
from paper_2403_15913_b200 import ckkt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
E32 = np.zeros(1, np.int32)


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "ckkt.h")).read()
    return sorted(set(re.findall(r"\b(ckkt_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = ckkt.lib()
    syms = _declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(ckkt.EXPORTED) == syms


def test_struct_layouts_match_header():
    # sizes of the ABI structs (x86-64 SysV), cross-checked against offsets computed by ctypes
    assert ctypes.sizeof(ckkt.ckkt_pattern) == 4 * 3 + 4 + 8 + 8 * 6
    assert ctypes.sizeof(ckkt.ckkt_info) == 4 * 4 + 8 * 3
    o = ckkt.default_options()
    assert o.strategy == ckkt.CKKT_HYKKT and o.gamma == 1e7 and o.cg_rtol == 1e-10 and o.cg_maxit == 200 and o.cg_rtol_corr == 1e-6
    assert o.batch == 1 and o.ref_maxit == 10


def _host_ctx(n, me, mi, w_row, w_col, g_rp, g_c, h_rp, h_c, **kw):
    return ckkt.Context(n, me, mi, w_row, w_col, g_rp, g_c, h_rp, h_c, device=-1, **kw)


@pytest.mark.parametrize("N,leaf", [(3, 16), (50, 64), (200, 268), (300, 1072)])
def test_symbolic_bit_exact_distillation(N, leaf):
    pat = dist.build_pattern(N)
    ctx = _host_ctx(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=leaf)
    perm, parent, cc, Lp, Li = ctx.export_symbolic()
    o = OK.SparseKKT(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, E32, E32[:0], leaf=leaf)
    assert np.array_equal(perm, o.perm)
    assert np.array_equal(parent, o.parent)
    assert np.array_equal(cc, o.colcount)
    assert np.array_equal(Lp, o.Lp) and np.array_equal(Li, o.Li)
    sz = ctx.get_sizes()
    assert sz["nnz_l"] == len(o.Li) and sz["nnz_k"] == len(o.Ai)


def test_symbolic_bit_exact_lifted_pattern_equals_hykkt_pattern():
    """Lifted (rows in H) and HyKKT (rows in G) share the K pattern (SURVEY §8 note); same symbolic."""
    pat = dist.build_pattern(30)
    a = _host_ctx(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=128)
    b = _host_ctx(pat.n, 0, pat.m, pat.w_row, pat.w_col, None, None, pat.j_rowptr, pat.j_col, leaf=128,
                  strategy=ckkt.CKKT_LIFTED)
    for x, y in zip(a.export_symbolic(), b.export_symbolic()):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("seed", range(10))
def test_symbolic_bit_exact_random(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 80))
    me = int(rng.integers(0, n // 2))
    mi = int(rng.integers(0, n))
    inst = random_instance(n, me, mi, seed=seed, density=float(rng.uniform(0.03, 0.2)))
    leaf = int(rng.integers(2, 20))
    ctx = _host_ctx(n, me, mi, inst.w_row, inst.w_col, inst.g_rowptr, inst.g_col, inst.h_rowptr, inst.h_col,
                    leaf=leaf)
    perm, parent, cc, Lp, Li = ctx.export_symbolic()
    o = OK.SparseKKT(n, me, mi, inst.w_row, inst.w_col, inst.g_rowptr, inst.g_col, inst.h_rowptr, inst.h_col,
                     leaf=leaf)
    assert np.array_equal(perm, o.perm) and np.array_equal(parent, o.parent)
    assert np.array_equal(Lp, o.Lp) and np.array_equal(Li, o.Li)


def test_caller_perm_is_used():
    pat = dist.build_pattern(5)
    perm = np.random.default_rng(0).permutation(pat.n).astype(np.int32)
    ctx = _host_ctx(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, perm=perm)
    p, parent, cc, Lp, Li = ctx.export_symbolic()
    assert np.array_equal(p, perm)
    o = OK.SparseKKT(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, E32, E32[:0], perm=perm)
    assert np.array_equal(parent, o.parent) and np.array_equal(Li, o.Li)


def test_pattern_errors():
    with pytest.raises(ckkt.CKKTError) as e:
        _host_ctx(3, 0, 0, np.array([0, 1]), np.array([1, 0]), None, None, None, None)  # upper entry
    assert e.value.code == ckkt.CKKT_PATTERN_ERROR
    with pytest.raises(ckkt.CKKTError) as e:
        _host_ctx(3, 1, 0, np.array([0]), np.array([0]), np.array([0, 2]), np.array([2, 1]), None, None)  # unsorted
    assert e.value.code == ckkt.CKKT_PATTERN_ERROR
    with pytest.raises(ckkt.CKKTError) as e:  # Lifted with equality rows
        _host_ctx(3, 1, 0, np.array([0]), np.array([0]), np.array([0, 1]), np.array([1]), None, None,
                  strategy=ckkt.CKKT_LIFTED)
    assert e.value.code == ckkt.CKKT_INVALID_ARG
    with pytest.raises(ckkt.CKKTError) as e:
        _host_ctx(3, 0, 0, np.array([0]), np.array([0]), None, None, None, None, perm=np.array([0, 0, 1]))
    assert e.value.code == ckkt.CKKT_INVALID_ARG


def test_device_calls_refuse_host_only_context():
    ctx = _host_ctx(3, 0, 0, np.array([0, 1, 2]), np.array([0, 1, 2]), None, None, None, None)
    assert ckkt.lib().ckkt_refactor(ctx.h, None, None, None, None, None, None, None, None) == ckkt.CKKT_INVALID_ARG
    assert ckkt.lib().ckkt_refactor_inertia(ctx.h, None, None, None, None, None, None, None, None, None,
                                            None) == ckkt.CKKT_INVALID_ARG


def test_fraction_to_boundary_argument_checks():
    """Argument validation happens before any device work (no GPU needed): tau outside (0, 1),
    negative sizes, missing pointers -> CKKT_INVALID_ARG; an empty batch is a no-op."""
    L = ckkt.lib()
    dummy = ctypes.c_void_p(8)
    assert L.ckkt_fraction_to_boundary(1, 4, dummy, dummy, 1.0, dummy, None) == ckkt.CKKT_INVALID_ARG
    assert L.ckkt_fraction_to_boundary(1, 4, dummy, dummy, 0.0, dummy, None) == ckkt.CKKT_INVALID_ARG
    assert L.ckkt_fraction_to_boundary(1, -1, dummy, dummy, 0.99, dummy, None) == ckkt.CKKT_INVALID_ARG
    assert L.ckkt_fraction_to_boundary(1, 4, None, dummy, 0.99, dummy, None) == ckkt.CKKT_INVALID_ARG
    assert L.ckkt_fraction_to_boundary(1, 4, dummy, dummy, 0.99, None, None) == ckkt.CKKT_INVALID_ARG
    assert L.ckkt_fraction_to_boundary(0, 4, None, None, 0.99, None, None) == ckkt.CKKT_OK


def test_option_validation():
    """tolerances must be finite and > 0 (cg_rtol_corr = 0 means the default), caps >= 0."""
    args = (3, 0, 0, np.array([0, 1, 2]), np.array([0, 1, 2]), None, None, None, None)
    for bad in (dict(cg_rtol=0.0), dict(cg_rtol=float("nan")), dict(cg_rtol_corr=-1.0),
                dict(cg_rtol_corr=float("inf")), dict(ref_tol=0.0), dict(cg_maxit=-1), dict(ref_maxit=-2),
                dict(gamma=0.0)):
        with pytest.raises(ckkt.CKKTError) as e:
            _host_ctx(*args, **bad)
        assert e.value.code == ckkt.CKKT_INVALID_ARG, bad
    _host_ctx(*args, cg_rtol_corr=0.0)          # zero-initialised field: the default
    _host_ctx(*args, gamma=0.0, strategy=ckkt.CKKT_LIFTED)  # gamma is ignored by Lifted


def test_elimination_order_is_a_postorder_of_perm():
    """ckkt_export_elimination_order (the order min_bad_pivot refers to, reading R9) is a permutation that
    is a postorder of the exported ordering's elimination tree: every column comes after its descendants and
    the L pattern it induces has the same size as the exported one (R11)."""
    pat = dist.build_pattern(30)
    ctx = _host_ctx(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=64)
    order = ctx.export_elimination_order()
    perm, parent, cc, Lp, Li = ctx.export_symbolic()
    assert sorted(order.tolist()) == list(range(pat.n))
    pos_in_perm = np.empty(pat.n, np.int64)
    pos_in_perm[perm] = np.arange(pat.n)
    pos = np.empty(pat.n, np.int64)
    pos[order] = np.arange(pat.n)
    for j in range(pat.n):                     # j indexes perm positions; parent[j] is a perm position
        p = parent[j]
        if p >= 0:
            assert pos[perm[j]] < pos[perm[p]]
    o = OK.SparseKKT(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, E32, E32[:0], perm=order)
    assert len(o.Li) == len(Li)
    assert ckkt.lib().ckkt_export_elimination_order(ctx.h, None) == ckkt.CKKT_INVALID_ARG


def test_analysis_blob_round_trip():
    """NEXT-2 (the analysis can be done offline): a context set up from an exported analysis
    has exactly the arrays of a freshly analysed one; a blob of another pattern, leaf or ordering is
    refused; a truncated blob is refused."""
    pat = dist.build_pattern(40)
    args = (pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None)
    ctx = _host_ctx(*args, leaf=64)
    blob = ctx.export_analysis()
    assert len(blob) > 1000
    ctx2 = _host_ctx(*args, leaf=64, analysis=blob)
    a, b = ctx.export_symbolic(), ctx2.export_symbolic()
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert np.array_equal(ctx.export_elimination_order(), ctx2.export_elimination_order())
    assert ctx.get_sizes() == ctx2.get_sizes()
    assert np.array_equal(ctx2.export_analysis(), blob)
    for bad in (dict(leaf=65, analysis=blob), dict(leaf=64, analysis=blob[:-8]), dict(leaf=64, analysis=np.full(64, 7, np.uint8))):
        with pytest.raises(ckkt.CKKTError) as e:
            _host_ctx(*args, **bad)
        assert e.value.code == ckkt.CKKT_INVALID_ARG
    other = dist.build_pattern(41)
    with pytest.raises(ckkt.CKKTError):
        _host_ctx(other.n, other.m, 0, other.w_row, other.w_col, other.j_rowptr, other.j_col, None, None, leaf=64,
                  analysis=blob)
    perm = np.arange(pat.n, dtype=np.int32)[::-1].copy()
    with pytest.raises(ckkt.CKKTError):  # blob of the built-in ordering used with a caller ordering
        _host_ctx(*args, leaf=64, perm=perm, analysis=blob)


@pytest.mark.parametrize("N,leaf", [(1500, 64), (2500, 1072)])
def test_parallel_analysis_matches_oracle_and_thread_count(N, leaf, monkeypatch):
    """The multithreaded analysis (parallel nested-dissection levels, leaf minimum degree, pattern and map
    construction) reproduces the specified ordering and symbolic arrays exactly: against the oracle, and
    with one thread against many."""
    pat = dist.build_pattern(N)
    args = (pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None)
    many = _host_ctx(*args, leaf=leaf)
    monkeypatch.setenv("CKKT_THREADS", "1")
    one = _host_ctx(*args, leaf=leaf)
    assert np.array_equal(many.export_analysis(), one.export_analysis())
    perm, parent, cc, Lp, Li = many.export_symbolic()
    o = OK.SparseKKT(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, E32, E32[:0], leaf=leaf)
    assert np.array_equal(perm, o.perm) and np.array_equal(parent, o.parent) and np.array_equal(cc, o.colcount)
    assert np.array_equal(Lp, o.Lp) and np.array_equal(Li, o.Li)


def _debug_get(ctx, what, dt):
    L = ckkt.lib()
    L.ckkt_debug_get.restype = ctypes.c_int64
    L.ckkt_debug_get.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    cnt = L.ckkt_debug_get(ctx.h, what, None)
    a = np.empty(cnt, dt)
    L.ckkt_debug_get(ctx.h, what, a.ctypes.data_as(ctypes.c_void_p))
    return a


@pytest.mark.parametrize("case", ["dist3", "dist40", "rand0", "rand1", "rand2", "rand3"])
def test_supernode_row_structures_cover_the_factor(case):
    """The supernodes' row lists (built by a postorder merge over the fundamental-supernode tree, not
    from the L pattern) against the exact L pattern of the internal order, obtained from the exported
    (oracle-pinned) symbolic relabelled by the postorder: every supernode lists its own columns first,
    rows ascending and unique, and contains the L structure of each of its columns (amalgamated
    supernodes may hold more rows: their explicit zeros)."""
    if case.startswith("dist"):
        pat = dist.build_pattern(int(case[4:]))
        ctx = _host_ctx(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=64)
        n = pat.n
    else:
        seed = int(case[4:])
        rng = np.random.default_rng(100 + seed)
        n = int(rng.integers(20, 120))
        me, mi = int(rng.integers(0, n // 2)), int(rng.integers(0, n))
        inst = random_instance(n, me, mi, seed=seed, density=float(rng.uniform(0.03, 0.15)))
        ctx = _host_ctx(n, me, mi, inst.w_row, inst.w_col, inst.g_rowptr, inst.g_col, inst.h_rowptr, inst.h_col,
                        leaf=int(rng.integers(2, 20)))
    perm, parent, cc, Lp, Li = ctx.export_symbolic()
    perm2 = _debug_get(ctx, 2, np.int32)
    sfirst = _debug_get(ctx, 3, np.int32)
    srp = _debug_get(ctx, 4, np.int64)
    srows = _debug_get(ctx, 5, np.int32)
    iperm = np.empty(n, np.int64)
    iperm[perm] = np.arange(n)
    post = iperm[perm2]                 # internal column k = exported column post[k]
    ipost = np.empty(n, np.int64)
    ipost[post] = np.arange(n)
    for s in range(sfirst.size - 1):
        f, l = int(sfirst[s]), int(sfirst[s + 1])
        rows = srows[srp[s]:srp[s + 1]]
        assert np.array_equal(rows[:l - f], np.arange(f, l))
        assert np.all(np.diff(rows) > 0)
        have = set(rows.tolist())
        for k in range(f, l):
            j = post[k]
            struct = ipost[Li[Lp[j]:Lp[j + 1]]]
            assert struct.min() == k and set(struct.tolist()) <= have, (s, k)
