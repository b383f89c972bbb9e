"""GPU parity at BASELINE configs[4]'s grid on one B200: 3D 1025^3 (pitch
1024, 1,070,599,167 unknowns) -- the level kernels of the two finest levels
(pitch 1024 and 512: four and two warps per row, the 8-warp FP64 outer
update shape), the transfers between them and the outer FP64 kernels.

A whole oracle pass at this size takes minutes per operation, so each
operation is checked bitwise on SAMPLED output planes (the first two, the
last two, and planes around the quarter / half points, where the z-chunks
and halo handling of the launches change) against the oracle's row-range
restatement (orc_spmv_rows / orc_transfer_rows, the same per-row arithmetic
as the whole-vector oracle, tests/test_oracle.py).
"""
import ctypes as C

import numpy as np
import pytest

import paper_2007_07539_b200 as mg
from oracle import FP16, FP64, Oracle

pytestmark = pytest.mark.gpu

O = Oracle()
DIM, NF = 3, 1025


def same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def mismatch(a, b, r0):
    bad = np.nonzero(~(np.asarray(a) == np.asarray(b)))[0]
    return f"{bad.size} mismatches, first rows {bad[:5] + r0}: gpu {np.asarray(a)[bad[:5]]} oracle {np.asarray(b)[bad[:5]]}"


def torch_():
    import torch
    return torch


def tdt(prec):
    t = torch_()
    return {FP16: t.float16, FP64: t.float64}[prec]


def planes(P):
    m = P - 1
    zs = sorted({1, 2, P // 4, P // 4 + 1, P // 2, P // 2 + 1, 3 * P // 4, m - 1, m})
    return [z for z in zs if 1 <= z <= m]


def pack(n, comp, prec):
    """compact value-domain host array -> padded device vector"""
    t = torch_()
    Lb = mg.lib()
    out = t.zeros(Lb.mpmg_padded_len(DIM, n), dtype=tdt(prec), device="cuda")
    src = t.from_numpy(comp).to("cuda").to(tdt(prec))
    mg._check(Lb.mpmg_gpu_pack(DIM, n, prec, src.data_ptr(), out.data_ptr(), None), "pack")
    del src
    return out


def unpack(n, dev, prec):
    t = torch_()
    comp = t.zeros(mg.unknowns(DIM, n), dtype=tdt(prec), device="cuda")
    mg._check(mg.lib().mpmg_gpu_unpack(DIM, n, prec, dev.data_ptr(), comp.data_ptr(), None), "unpack")
    t.cuda.synchronize()
    return comp.double().cpu().numpy()


def rand(rng, n, prec, scale):
    x = (rng.random(mg.unknowns(DIM, n)) * 2 - 1) * scale
    return O.cast(x, prec, 1.0, O.ctx(False))


def rows_of(n, z):
    m = n - 2
    return (z - 1) * m * m, z * m * m


@pytest.fixture(scope="module")
def rng():
    return np.random.default_rng(1025)


@pytest.mark.parametrize("prec", [FP64, FP16])
@pytest.mark.parametrize("n", [1025, 513])
def test_level_kernels_1025(prec, n, rng):
    Lb = mg.lib()
    ctx = O.ctx(False, True, False)
    pol = mg.policy_word(False, True, False)
    A = mg.level_stencil(DIM, n, prec, False)
    # the oracle's level operator in precision prec (implicit rows)
    hl = O.hierarchy(DIM, n, 2, "h_mg" if prec == FP16 else "d_mg", ftz=False, implicit=True)
    Al = hl.o.L.orc_level_matrix(hl.h, 1, 0).contents
    u = rand(rng, n, prec, 1e-3)
    b = rand(rng, n, prec, 1.0)
    ud, bd = pack(n, u, prec), pack(n, b, prec)
    t = torch_()
    out = t.zeros_like(ud)
    # one Jacobi step and the defect
    assert Lb.mpmg_gpu_jacobi(C.byref(A), bd.data_ptr(), ud.data_ptr(), out.data_ptr(), 2.0 / 3.0, pol, None) == 0
    jg = unpack(n, out, prec)
    assert Lb.mpmg_gpu_defect(C.byref(A), bd.data_ptr(), ud.data_ptr(), out.data_ptr(), pol, None) == 0
    dg = unpack(n, out, prec)
    # the pre-smoother's fused steps 1 + 2 from u = 0 (JACOBI_Z)
    tmp = t.zeros_like(ud)
    assert Lb.mpmg_gpu_jacobi_from_zero2(C.byref(A), bd.data_ptr(), tmp.data_ptr(), out.data_ptr(), 2.0 / 3.0, pol,
                                         None) == 0
    zg = unpack(n, out, prec)
    del tmp, out
    w = O.round_vec([2.0 / 3.0], prec, False)[0]
    dinv = O.round_vec([A.inv_diag], prec, False)[0]  # the level's D^-1 (already in prec)
    for z in planes(n - 1):
        r0, r1 = rows_of(n, z)
        tt = O.spmv_rows(Al, u, r0, r1, ctx)
        r = O.axpy(prec, -1.0, tt, b[r0:r1], ctx)
        assert same(dg[r0:r1], r), f"defect plane {z}: " + mismatch(dg[r0:r1], r, r0)
        dr = O.vec_multiply(prec, np.full(r1 - r0, dinv), r, ctx)
        jo = O.axpy(prec, w, dr, u[r0:r1], ctx)
        assert same(jg[r0:r1], jo), f"jacobi plane {z}: " + mismatch(jg[r0:r1], jo, r0)
    # step 1 from zero: u1 = w (d b) (pointwise, whole vector), step 2 on the sampled planes
    u1 = O.axpy(prec, w, O.vec_multiply(prec, np.full(b.size, dinv), b, ctx), np.zeros(b.size), ctx)
    for z in planes(n - 1):
        r0, r1 = rows_of(n, z)
        r = O.axpy(prec, -1.0, O.spmv_rows(Al, u1, r0, r1, ctx), b[r0:r1], ctx)
        zo = O.axpy(prec, w, O.vec_multiply(prec, np.full(r1 - r0, dinv), r, ctx), u1[r0:r1], ctx)
        assert same(zg[r0:r1], zo), f"jacobi-from-zero plane {z}: " + mismatch(zg[r0:r1], zo, r0)


@pytest.mark.parametrize("prec", [FP64, FP16])
def test_transfers_1025(prec, rng):
    """restriction 1025 -> 513 and prolongation + correction 513 -> 1025"""
    Lb = mg.lib()
    ctx = O.ctx(False, True, False)
    pol = mg.policy_word(False, True, False)
    nc = (NF + 1) // 2
    hl = O.hierarchy(DIM, NF, 2, "h_mg" if prec == FP16 else "d_mg", ftz=False, implicit=True)
    R = hl.o.L.orc_level_matrix(hl.h, 0, 2).contents
    P = hl.o.L.orc_level_matrix(hl.h, 0, 1).contents
    t = torch_()
    rf = rand(rng, NF, prec, 1e-2)
    rfd = pack(NF, rf, prec)
    rcd = t.zeros(Lb.mpmg_padded_len(DIM, nc), dtype=tdt(prec), device="cuda")
    assert Lb.mpmg_gpu_restrict(DIM, NF, prec, prec, rfd.data_ptr(), rcd.data_ptr(), None, pol, None) == 0
    rcg = unpack(nc, rcd, prec)
    for z in planes(nc - 1):
        r0, r1 = rows_of(nc, z)
        ro = O.cast(O.transfer_rows(R, rf, prec, r0, r1, ctx), prec, 1.0, ctx)
        assert same(rcg[r0:r1], ro), f"restrict plane {z}: " + mismatch(rcg[r0:r1], ro, r0)
    del rfd, rf
    c = rand(rng, nc, prec, 0.5)
    u = rand(rng, NF, prec, 1e-2)
    cd, ud = pack(nc, c, prec), pack(NF, u, prec)
    assert Lb.mpmg_gpu_prolong_correct(DIM, NF, prec, prec, cd.data_ptr(), ud.data_ptr(), None, pol, None) == 0
    pg = unpack(NF, ud, prec)
    for z in planes(NF - 1):
        r0, r1 = rows_of(NF, z)
        tp = O.cast(O.transfer_rows(P, c, prec, r0, r1, ctx), prec, 1.0, ctx)
        po = O.axpy(prec, 1.0, tp, u[r0:r1], ctx)
        assert same(pg[r0:r1], po), f"prolong plane {z}: " + mismatch(pg[r0:r1], po, r0)


def test_v_cycle_513_d_mg():
    """One whole D_MG V-cycle at 513^3 (L = 9: two streaming levels above the
    pitch-256 ones, pitch 512 with two warps per row) bitwise against the
    oracle -- the composition, not only the kernels."""
    n, L = 513, 9
    ctx = O.ctx(False, True, False)
    h = mg.Hierarchy(DIM, n, L, "d_mg", ftz=False)
    ho = O.hierarchy(DIM, n, L, "d_mg", ftz=False, implicit=True)
    b = mg.problem_rhs(DIM, n)
    cg, co = h.v_cycle(b), ho.v_cycle(b, ctx)
    h.close()
    bad = np.count_nonzero(cg != co)
    assert bad == 0, f"{bad} mismatches, rel {np.linalg.norm(cg - co) / np.linalg.norm(co):.3e}"


@pytest.mark.parametrize("cprec", [FP64, FP16])
def test_outer_kernels_1025(cprec, rng):
    """FP64 defect and the fused update r -= a A c, u += a c (the D_MG outer
    update runs the 8-warp-per-row shape at pitch 1024)"""
    Lb = mg.lib()
    t = torch_()
    ctx = O.ctx(False, True, False)
    pol = mg.policy_word(False, True, False)
    A64s = mg.level_stencil(DIM, NF, FP64, False)
    A64 = O.stiffness_implicit(DIM, NF)
    N = mg.unknowns(DIM, NF)
    u = rng.random(N) * 2 - 1
    b = rng.random(N) * 2 - 1
    ud, bd = pack(NF, u, FP64), pack(NF, b, FP64)
    rd = t.zeros_like(bd)
    part = t.zeros(max(Lb.mpmg_gpu_partials_len(DIM, NF), 1), dtype=t.float64, device="cuda")
    assert Lb.mpmg_gpu_defect_f64(C.byref(A64s), bd.data_ptr(), ud.data_ptr(), rd.data_ptr(), part.data_ptr(),
                                  None) == 0
    rg = unpack(NF, rd, FP64)
    for z in planes(NF - 1):
        r0, r1 = rows_of(NF, z)
        ro = O.axpy(FP64, -1.0, O.spmv_rows(A64, u, r0, r1, ctx), b[r0:r1], ctx)
        assert same(rg[r0:r1], ro), f"defect64 plane {z}: " + mismatch(rg[r0:r1], ro, r0)
    del bd, b
    c = rand(rng, NF, cprec, 1.0)
    cd = pack(NF, c, cprec)
    alpha = 3.7e-3
    ad = t.tensor([alpha], dtype=t.float64, device="cuda")
    assert Lb.mpmg_gpu_update_rc(C.byref(A64s), cd.data_ptr(), cprec, rd.data_ptr(), ud.data_ptr(), ad.data_ptr(),
                                 part.data_ptr(), pol, None) == 0
    rg2, ug2 = unpack(NF, rd, FP64), unpack(NF, ud, FP64)
    for z in planes(NF - 1):
        r0, r1 = rows_of(NF, z)
        s = O.spmv_rows(A64, c, r0, r1, ctx)  # A c in FP64 (c widened)
        ro = O.axpy(FP64, -alpha, s, rg[r0:r1], ctx)  # r = fma(-a, (A c)_i, r)
        uo = O.axpy(FP64, alpha, c[r0:r1], u[r0:r1], ctx)
        assert same(rg2[r0:r1], ro), f"update r plane {z}: " + mismatch(rg2[r0:r1], ro, r0)
        assert same(ug2[r0:r1], uo), f"update u plane {z}: " + mismatch(ug2[r0:r1], uo, r0)
