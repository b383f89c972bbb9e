"""GPU parity at the paper's 193^3 grid: its finest pitch
192 is not a power of two, so the plane kernels run their W = 6 instantiation
(three binary16 pairs / six binary64 values per lane, 4-byte-word row loads),
while the coarser pitches 96, 48, 24, 12, 6 take the streaming k_stencil and the
coarse cluster kernel. Bitwise against the oracle: every level kernel of the
finest level, whole V-cycles, the outer FP64 kernels through the C ABI, and an
H_MG solve (iterations, history, solution)."""
import ctypes as C

import numpy as np
import pytest

import paper_2007_07539_b200 as mg
from oracle import FP16, FP32, FP64, Oracle

pytestmark = pytest.mark.gpu

O = Oracle()
DIM, N, L = 3, 193, 7


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
    return O.cast(x, prec, 1.0, O.ctx(ftz))


_OH = {}


def oracle_h(variant, ftz):
    key = (variant, ftz)
    if key not in _OH:
        _OH.clear()
        _OH[key] = O.hierarchy(DIM, N, L, variant, ftz=ftz, implicit=True)
    return _OH[key]


@pytest.fixture(scope="module")
def rng():
    return np.random.default_rng(193)


@pytest.mark.parametrize("variant,ftz", [("h_mg", False), ("h_mg", True), ("d_mg", False)])
def test_level_kernels_193(variant, ftz, rng):
    l = L - 1  # pitch 192
    h = mg.Hierarchy(DIM, N, L, variant, ftz=ftz)
    ho = oracle_h(variant, ftz)
    ctx = O.ctx(ftz, True, False)
    prec = ho.prec(l)
    Nl = ho.rows(l)
    A = ho.o.L.orc_level_matrix(ho.h, l, 0).contents
    u = rand_level(rng, Nl, prec, ftz, 1e-3)
    b = rand_level(rng, Nl, prec, ftz, 1.0)
    y_o = O.spmv_e(A, u, ctx)
    r_o = O.axpy(prec, -1.0, y_o, b, ctx)
    r_g = h.defect(l, b, u)
    assert same(r_g, r_o), "defect " + mismatch(r_g, r_o)
    j_o = ho.jacobi(l, b, u, 2, ctx=ctx)
    j_g = h.jacobi(l, b, u, 2)
    assert same(j_g, j_o), "jacobi " + mismatch(j_g, j_o)
    z_o = ho.jacobi(l, b, np.zeros(Nl), 3, ctx=ctx)
    z_g = h.jacobi(l, b, None, 3)
    assert same(z_g, z_o), "jacobi-from-zero " + mismatch(z_g, z_o)
    rc_o, _ = ho.restrict(l, b, False, ctx=ctx)
    rc_g = h.restrict(l, b)
    assert same(rc_g, rc_o), "restrict " + mismatch(rc_g, rc_o)
    c = rand_level(rng, ho.rows(l - 1), ho.prec(l - 1), ftz, 0.5)
    p_o = O.axpy(prec, 1.0, ho.prolong(l, c, 1.0, ctx=ctx), u, ctx)
    p_g = h.prolong_correct(l, c, u)
    assert same(p_g, p_o), "prolong " + mismatch(p_g, p_o)
    h.close()


@pytest.mark.parametrize("variant", ["h_mg", "hsd_mg", "d_mg"])
def test_v_cycle_193(variant):
    h = mg.Hierarchy(DIM, N, L, variant, ftz=False)
    ho = oracle_h(variant, False)
    ctx = O.ctx(False, True, False)
    b = O.rhs(DIM, N)
    fp = ho.prec(L - 1)
    rl = O.cast(b, fp, O.norm2(b) if variant != "d_mg" else 1.0, ctx)
    c_o = ho.v_cycle(rl, ctx)
    c_g = h.v_cycle(rl)
    assert same(c_g, c_o), "v_cycle " + mismatch(c_g, c_o)
    h.close()


@pytest.mark.parametrize("cprec", [FP16, FP64])
def test_outer_kernels_193(cprec, rng):
    """FP64 defect and the fused update at pitch 192 (W = 6 binary64 rows)"""
    import torch
    Lb = mg.lib()
    ctx = O.ctx(False, True, False)
    pol = mg.policy_word(False, True, False)
    A64s = mg.level_stencil(DIM, N, FP64, False)
    A64 = O.stiffness_implicit(DIM, N)
    Nn = mg.unknowns(DIM, N)
    plen = Lb.mpmg_padded_len(DIM, N)
    tdt = {FP16: torch.float16, FP64: torch.float64}

    def pack(x, prec):
        out = torch.zeros(plen, dtype=tdt[prec], device="cuda")
        src = torch.from_numpy(x).cuda().to(tdt[prec])
        mg._check(Lb.mpmg_gpu_pack(DIM, N, prec, src.data_ptr(), out.data_ptr(), None), "pack")
        return out

    def unpack(d, prec):
        comp = torch.zeros(Nn, dtype=tdt[prec], device="cuda")
        mg._check(Lb.mpmg_gpu_unpack(DIM, N, prec, d.data_ptr(), comp.data_ptr(), None), "unpack")
        torch.cuda.synchronize()
        return comp.double().cpu().numpy()

    u = rng.random(Nn) * 2 - 1
    b = rng.random(Nn) * 2 - 1
    ud, bd = pack(u, FP64), pack(b, FP64)
    rd = torch.zeros_like(bd)
    part = torch.zeros(max(Lb.mpmg_gpu_partials_len(DIM, N), 1), dtype=torch.float64, device="cuda")
    assert Lb.mpmg_gpu_defect_f64(C.byref(A64s), bd.data_ptr(), ud.data_ptr(), rd.data_ptr(), part.data_ptr(),
                                  None) == 0
    r_g = unpack(rd, FP64)
    r_o = O.axpy(FP64, -1.0, O.spmv_e(A64, u, ctx), b, ctx)
    assert same(r_g, r_o), "defect64 " + mismatch(r_g, r_o)
    c = rand_level(rng, Nn, cprec, False, 1.0)
    cd = pack(c, cprec)
    alpha = 3.7e-3
    ad = torch.tensor([alpha], dtype=torch.float64, device="cuda")
    assert Lb.mpmg_gpu_update_rc(C.byref(A64s), cd.data_ptr(), cprec, rd.data_ptr(), ud.data_ptr(), ad.data_ptr(),
                                 part.data_ptr(), pol, None) == 0
    r2, u2 = unpack(rd, FP64), unpack(ud, FP64)
    ro = O.axpy(FP64, -alpha, O.spmv_e(A64, c, ctx), r_g, ctx)
    uo = O.axpy(FP64, alpha, c, u, ctx)
    assert same(r2, ro), "update r " + mismatch(r2, ro)
    assert same(u2, uo), "update u " + mismatch(u2, uo)


def test_ir_solve_193_h_mg():
    ctx = O.ctx(False, True, False)
    b = O.rhs(DIM, N)
    tol = 1e-10 * O.norm2(b)
    ho = oracle_h("h_mg", False)
    so = ho.ir_solve(b, tol=tol, ctx=ctx)
    h = mg.Hierarchy(DIM, N, L, "h_mg", ftz=False)
    u, rep = h.ir_solve(b, mg.IrConfig(outer_tolerance=tol))
    h.close()
    assert rep.converged and so["converged"]
    assert abs(rep.iterations - so["iterations"]) <= 1
    # the trajectory agrees to the rounding level of each entry (the norm's
    # summation grouping differs in the last bit, so a binary16 scaled cast may
    # round one ulp apart); the contract is iterations +-1 and the solution
    n = min(len(rep.residual_history), len(so["history"]))
    np.testing.assert_allclose(rep.residual_history[:n], so["history"][:n], rtol=1e-3)
    assert np.linalg.norm(u - so["u"]) / np.linalg.norm(so["u"]) <= 1e-9
