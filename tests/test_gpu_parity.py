"""GPU parity: the sm_100a kernels (through the C ABI) against the C oracle
(oracle/mpmg_oracle.c, itself pinned bitwise to the compiled reference).

Bar (BASELINE.json north_star): per-kernel results identical to the
reference value-for-value (binary16/32/64 values compared exactly; the only
tolerated difference is the sign of an exact zero, which no later operation
can turn into a nonzero value); full solves: same outer iteration count
within +-1 and final solution within 1e-9 relative L2.
"""
import numpy as np
import pytest

import paper_2007_07539_b200 as mg
from oracle import FP16, FP32, FP64, Oracle

pytestmark = pytest.mark.gpu

O = Oracle()
POLICIES = [(True, True, False), (False, True, False), (True, False, False), (False, False, False),
            (True, True, True), (False, True, True)]


def same(a, b):
    a = np.asarray(a); b = np.asarray(b)
    return a.shape == b.shape and np.array_equal(a, b, equal_nan=True)


def mismatch(a, b):
    a = np.asarray(a); b = np.asarray(b)
    bad = ~((a == b) | (np.isnan(a) & np.isnan(b)))
    idx = np.nonzero(bad)[0]
    return f"{idx.size} mismatches, first {idx[:5]}: gpu {a[idx[:5]]} oracle {b[idx[:5]]}"


def rand_level(rng, n, prec, ftz, scale=1.0):
    x = (rng.random(n) * 2.0 - 1.0) * scale
    return O.round_vec(x, prec, ftz)


@pytest.fixture(scope="module")
def rng():
    return np.random.default_rng(1234)


_OH = {}


def oracle_h(dim, n, L, variant, ftz):
    key = (dim, n, L, variant, ftz)
    if key not in _OH:
        _OH[key] = O.hierarchy(dim, n, L, variant, ftz=ftz)
    return _OH[key]


# (variant, dim, nodes, levels, level under test): binary16 and binary64
# streaming levels of deep hierarchies, binary32 levels of HSD/DSH cascades
CASES = [(v, 3, 129, 7, l) for v in ("h_mg", "d_mg") for l in (6, 5)] + \
        [(v, 3, 97, 6, l) for v in ("h_mg", "d_mg") for l in (5, 4)] + \
        [(v, 2, 257, 8, l) for v in ("h_mg", "d_mg") for l in (7, 6)] + \
        [(v, d, n, 3, 2) for v in ("hsd_mg", "dsh_mg") for d, n in ((2, 257), (3, 129))]


@pytest.mark.parametrize("variant,dim,n,L,l", CASES)
@pytest.mark.parametrize("ftz,fma,acc32", POLICIES)
def test_level_kernels(variant, dim, n, L, l, ftz, fma, acc32, rng):
    h = mg.Hierarchy(dim, n, L, variant, ftz=ftz, fma=fma, acc32=acc32)
    ho = oracle_h(dim, n, L, variant, ftz)
    if acc32 and ho.prec(l) != FP16:
        pytest.skip("binary32 accumulation only changes binary16 levels")
    ctx = O.ctx(ftz, fma, acc32)
    prec = ho.prec(l)
    N = ho.rows(l)
    cols, vals = ho.matrix(l, 0)
    # magnitudes spanning the binary16 subnormal range (as scaled residuals do)
    u = rand_level(rng, N, prec, ftz, 1e-3)
    b = rand_level(rng, N, prec, ftz, 1.0)
    y_o = O.spmv(cols, vals, prec, u, ctx)
    y_g = h.spmv(l, u)
    assert same(y_g, y_o), "spmv " + mismatch(y_g, y_o)
    r_o = O.axpy(prec, -1.0, y_o, b, ctx)
    r_g = h.defect(l, b, u)
    assert same(r_g, r_o), "defect " + mismatch(r_g, r_o)
    j_o = ho.jacobi(l, b, u, 2, ctx=ctx)
    j_g = h.jacobi(l, b, u, 2)
    assert same(j_g, j_o), "jacobi " + mismatch(j_g, j_o)
    z_o = ho.jacobi(l, b, np.zeros(N), 3, ctx=ctx)
    z_g = h.jacobi(l, b, None, 3)  # first step from zero (fused form)
    assert same(z_g, z_o), "jacobi-from-zero " + mismatch(z_g, z_o)
    # transfers between l and l-1
    rc_o, _ = ho.restrict(l, b, False, ctx=ctx)
    rc_g = h.restrict(l, b)
    assert same(rc_g, rc_o), "restrict " + mismatch(rc_g, rc_o)
    pc = ho.prec(l - 1)
    c = rand_level(rng, ho.rows(l - 1), pc, ftz, 0.5)
    t_o = ho.prolong(l, c, 1.0, ctx=ctx)
    p_o = O.axpy(prec, 1.0, t_o, u, ctx)
    p_g = h.prolong_correct(l, c, u)
    assert same(p_g, p_o), "prolong " + mismatch(p_g, p_o)


@pytest.mark.parametrize("variant", ["h_mg", "hsd_mg", "d_mg", "dsh_mg"])
# (73 and 145: non-power-of-two grids whose coarse cluster kernel has a
# binary16 slab level with P = 18, whose planes are not 16-byte multiples)
@pytest.mark.parametrize("dim,n,L", [(3, 65, 6), (2, 257, 8), (3, 33, 5), (3, 97, 6), (3, 73, 4), (3, 145, 5)])
@pytest.mark.parametrize("ftz", [True, False])
def test_v_cycle(variant, dim, n, L, ftz, rng):
    h = mg.Hierarchy(dim, n, L, variant, ftz=ftz)
    ho = O.hierarchy(dim, n, L, variant, ftz=ftz)
    ctx = O.ctx(ftz, True, False)
    fp = ho.prec(L - 1)
    b = O.rhs(dim, n)
    rl = O.cast(b, fp, O.norm2(b) if variant != "d_mg" else 1.0, ctx)
    c_o = ho.v_cycle(rl, ctx)
    c_g = h.v_cycle(rl)
    assert same(c_g, c_o), "v_cycle " + mismatch(c_g, c_o)


def test_coarse_solve_matches_cg(rng):
    for variant in ["h_mg", "d_mg", "hsd_mg"]:
        for dim, n, L in [(2, 65, 3), (3, 33, 3)]:  # base grids with 15^2 / 7^3 unknowns
            h = mg.Hierarchy(dim, n, L, variant, ftz=True)
            ho = O.hierarchy(dim, n, L, variant, ftz=True)
            p0 = ho.prec(0)
            b = rand_level(rng, ho.rows(0), p0, True, 1.0)
            u_o, it, conv, res = ho.cg(0, b)
            u_g = h.coarse_solve(b)
            assert same(u_g, u_o), f"cg {variant} {dim} " + mismatch(u_g, u_o)


@pytest.mark.parametrize("variant", ["h_mg", "hsd_mg", "d_mg", "dsh_mg"])
@pytest.mark.parametrize("dim,n,L", [(3, 65, 6), (2, 257, 8), (3, 97, 6), (3, 145, 5)])
@pytest.mark.parametrize("ftz", [True, False])
@pytest.mark.parametrize("graph", [True, False])
def test_ir_solve(variant, dim, n, L, ftz, graph):
    h = mg.Hierarchy(dim, n, L, variant, ftz=ftz)
    ho = O.hierarchy(dim, n, L, variant, ftz=ftz)
    b = O.rhs(dim, n)
    tol = 1e-10 * O.norm2(b)
    try:
        so = ho.ir_solve(b, tol=tol, ctx=O.ctx(ftz, True, False))
    except FloatingPointError:
        # the reference's H_MG diverges on some non-power-of-two grids (145^3
        # FTZ off: a non-finite residual norm); the GPU solve must throw the
        # same DivergedError (ir_solver.cpp:99-101)
        with pytest.raises(mg.DivergedError):
            h.ir_solve(b, mg.IrConfig(outer_tolerance=tol, use_graph=graph))
        return
    u, rep = h.ir_solve(b, mg.IrConfig(outer_tolerance=tol, use_graph=graph))
    assert rep.converged == so["converged"]
    assert abs(rep.iterations - so["iterations"]) <= 1
    rel = np.linalg.norm(u - so["u"]) / np.linalg.norm(so["u"])
    assert rel <= 1e-9, rel
    # the first residual is the same FP64 defect of u0 = 0 -> identical
    assert rep.residual_history[0] == pytest.approx(so["history"][0], rel=1e-13)
    assert rep.final_residual < tol


def test_ir_solve_random_guess_and_refresh():
    dim, n, L = 3, 65, 6
    h = mg.Hierarchy(dim, n, L, "h_mg", ftz=False)
    ho = O.hierarchy(dim, n, L, "h_mg", ftz=False)
    b = O.rhs(dim, n)
    for refresh in (10, 3, 0):
        so = ho.ir_solve(b, tol=1e-9, random_guess=True, seed=42, refresh=refresh, ctx=O.ctx(False))
        u, rep = h.ir_solve(b, mg.IrConfig(outer_tolerance=1e-9, random_initial_guess=True, seed=42,
                                           residual_refresh_interval=refresh))
        # the random initial guess is SplitMix64 (rng.hpp), identical bits -> same first residual
        assert rep.residual_history[0] == pytest.approx(so["history"][0], rel=1e-13)
        assert abs(rep.iterations - so["iterations"]) <= 1
        assert np.linalg.norm(u - so["u"]) / np.linalg.norm(so["u"]) <= 1e-9


def test_max_iterations_not_an_error():
    h = mg.Hierarchy(3, 33, 5, "h_mg")
    b = O.rhs(3, 33)
    u, rep = h.ir_solve(b, mg.IrConfig(outer_tolerance=1e-30, max_outer_iterations=3))
    assert not rep.converged and rep.iterations == 3 and len(rep.residual_history) == 4


def test_zero_rhs_converges_immediately():
    h = mg.Hierarchy(3, 33, 5, "h_mg")
    u, rep = h.ir_solve(np.zeros(31 ** 3))
    assert rep.converged and rep.iterations == 0 and not u.any()


def test_scaling_forced_off_stagnates_h_mg():
    # SPEC acceptance 5: without residuum scaling the FP16 cast flushes the
    # residual once it drops below the binary16 range; with it, converges.
    dim, n, L = 2, 257, 8
    h = mg.Hierarchy(dim, n, L, "h_mg")
    b = O.rhs(dim, n)
    _, on = h.ir_solve(b, mg.IrConfig(outer_tolerance=1e-9, max_outer_iterations=40))
    _, off = h.ir_solve(b, mg.IrConfig(outer_tolerance=1e-9, max_outer_iterations=40, scaling=2))
    assert on.converged and not off.converged


@pytest.mark.parametrize("variant,refresh,max_it,tol", [
    ("h_mg", 10, 100, 1e-10),   # the benchmark schedule: one fold at the refresh
    ("h_mg", 3, 100, 1e-10),    # a fold every 3 iterations
    ("hsd_mg", 0, 14, 1e-30),   # no refresh: folds when the 10-slot ring fills, then at the end
    ("h_mg", 10, 14, 1e-30),    # fold at 10, 4 parked corrections folded after the loop
])
@pytest.mark.parametrize("graph", [True, False])
@pytest.mark.parametrize("dim,n,L", [(3, 65, 6), (2, 257, 8), (3, 97, 6)])
def test_deferred_corrections_bitwise(variant, refresh, max_it, tol, graph, dim, n, L, monkeypatch):
    """The deferred u += a c (ring of parked corrections, mpmg_solver.cu) gives
    the bitwise solution, residual history and iteration count of the fused
    per-iteration update_residuum_correction (kernels.cpp:300-341) -- with the
    plane UPDATE_R (3D 65^3) and the streaming one (2D; pitch 96)."""
    b = mg.problem_rhs(dim, n)
    out = []
    for defer in ("1", "0"):
        monkeypatch.setenv("MPMG_DEFER_U", defer)
        h = mg.Hierarchy(dim, n, L, variant, ftz=False)
        cfg = mg.IrConfig(outer_tolerance=tol * float(np.linalg.norm(b)), max_outer_iterations=max_it,
                          residual_refresh_interval=refresh, use_graph=graph)
        out.append(h.ir_solve(b, cfg))
        h.close()
    (u1, r1), (u0, r0) = out
    assert r1.iterations == r0.iterations and r1.converged == r0.converged
    assert same(u1.view(np.uint64), u0.view(np.uint64))
    assert same(r1.residual_history, r0.residual_history)
    assert r1.final_residual == r0.final_residual


@pytest.mark.parametrize("refresh", [1, 3, 0])
def test_final_residual_is_residual_norm(refresh):
    """SolveReport.final_residual == residual_norm(A, u, b) (ir_solver.cpp:21-49) of
    the returned u, whether the last iteration refreshed r (its defect's sum of
    squares is reused) or not (a fresh residual-norm pass)."""
    dim, n, L = 3, 33, 5
    b = mg.problem_rhs(dim, n)
    h = mg.Hierarchy(dim, n, L, "h_mg", ftz=False)
    cfg = mg.IrConfig(outer_tolerance=1e-10 * float(np.linalg.norm(b)), residual_refresh_interval=refresh)
    u, rep = h.ir_solve(b, cfg)
    h.close()
    cols, vals = O.stiffness(dim, n)
    t = O.spmv(cols, vals, FP64, u, O.ctx(False))
    r = b - t
    assert rep.final_residual == pytest.approx(float(np.sqrt(np.dot(r, r))), rel=1e-12)


@pytest.mark.parametrize("n", [129, 65])
def test_asymmetric_binary16_stencil(n, rng):
    """The binary16 plane / direct kernels keep one register per tap class
    (sym16): a stencil whose edge taps are not all one value must take the
    general stencil kernels and still match the oracle bitwise (C ABI defect
    with one edge tap perturbed; pitch 128 = plane kernel, 64 = direct)."""
    import ctypes as C
    import torch
    Lb = mg.lib()
    ctx = O.ctx(False, True, False)
    pol = mg.policy_word(False, True, False)
    A = mg.level_stencil(3, n, FP16, False)
    ho = oracle_h(3, n, 2, "h_mg", False)
    cols, vals = ho.matrix(1, 0)
    m = n - 2
    k = 1  # (dz, dy, dx) = (-1, -1, 0): an edge tap
    off = -m * m - m
    new = A.taps[k] * 1.5
    A.taps[k] = new
    rows = np.arange(cols.shape[0])[:, None]
    vals = np.where((cols - rows == off) & (vals != 0), O.round_vec([new], FP16, False)[0], vals)
    N = m ** 3
    u = rand_level(rng, N, FP16, False, 1e-2)
    b = rand_level(rng, N, FP16, False, 1.0)
    plen = Lb.mpmg_padded_len(3, n)

    def pack(x):
        out = torch.zeros(plen, dtype=torch.float16, device="cuda")
        src = torch.from_numpy(x).to("cuda").half()
        mg._check(Lb.mpmg_gpu_pack(3, n, FP16, src.data_ptr(), out.data_ptr(), None), "pack")
        return out

    ud, bd = pack(u), pack(b)
    rd = torch.zeros_like(ud)
    assert Lb.mpmg_gpu_defect(C.byref(A), bd.data_ptr(), ud.data_ptr(), rd.data_ptr(), pol, None) == 0
    comp = torch.zeros(N, dtype=torch.float16, device="cuda")
    mg._check(Lb.mpmg_gpu_unpack(3, n, FP16, rd.data_ptr(), comp.data_ptr(), None), "unpack")
    rg = comp.double().cpu().numpy()
    ro = O.axpy(FP16, -1.0, O.spmv(cols, vals, FP16, u, ctx), b, ctx)
    assert same(rg, ro), mismatch(rg, ro)
    # and the perturbation matters (the symmetric kernels would have ignored it)
    r0 = O.axpy(FP16, -1.0, O.spmv(*ho.matrix(1, 0), FP16, u, ctx), b, ctx)
    assert not same(ro, r0)
