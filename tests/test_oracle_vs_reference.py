"""The oracle restatement against the unmodified reference (oracle/_ref),
bitwise, on fresh seeded inputs at sizes beyond the golden fixtures. Skipped
where the compiled reference is absent."""
import numpy as np
import pytest

from oracle import FP16, FP32, FP64, Oracle, Reference, ref_available

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref/libmpmg_ref.so not built")

O = Oracle()


def same_bits(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.fixture(scope="module")
def R():
    return Reference()


def test_fp16_scalars(R):
    rng = np.random.default_rng(5)
    xs = np.concatenate([rng.standard_normal(5000) * 10.0 ** rng.integers(-9, 5, 5000), [0.0, -0.0, 65520.0]])
    for ftz in (0, 1):
        assert same_bits([O.q16(x, ftz) for x in xs], [R.q16(x, ftz) for x in xs])
    a = O.round_vec(rng.standard_normal(3000), FP16, False)
    b = O.round_vec(rng.standard_normal(3000) * 1e-3, FP16, False)
    c = O.round_vec(rng.standard_normal(3000) * 1e-5, FP16, False)
    for ftz in (0, 1):
        for fma in (0, 1):
            mine = [O.fma16(x, y, z, ftz, fma) for x, y, z in zip(a, b, c)]
            ref = [R.fma16(x, y, z, ftz, fma) for x, y, z in zip(a, b, c)]
            assert same_bits(mine, ref)


@pytest.mark.parametrize("variant", ["h_mg", "hsd_mg", "dsh_mg", "d_mg"])
@pytest.mark.parametrize("ftz", [0, 1])
def test_level_ops_3d_33(R, variant, ftz):
    dim, n, L = 3, 33, 5
    ho = O.hierarchy(dim, n, L, variant, ftz=bool(ftz))
    hr = R.hierarchy(dim, n, L, variant, ftz=ftz)
    rng = np.random.default_rng(7)
    for l in (L - 1, L - 2):
        p = ho.prec(l)
        N = ho.rows(l)
        assert p == hr.prec(l) and N == hr.rows(l)
        co, vo = ho.matrix(l, 0)
        cr, vr = hr.matrix(l, 0)
        assert np.array_equal(co, cr) and same_bits(vo, vr)
        assert same_bits(ho.invdiag(l), hr.invdiag(l))
        b = O.round_vec(rng.standard_normal(N), p, ftz)
        u = O.round_vec(rng.standard_normal(N) * 1e-3, p, ftz)
        for acc32 in (0, 1):
            ctx = O.ctx(ftz, True, acc32)
            assert same_bits(O.spmv(co, vo, p, u, ctx), hr.spmv(l, u, acc32=bool(acc32)))
            assert same_bits(ho.jacobi(l, b, u, 2, ctx=ctx), hr.jacobi(l, b, u, 2, acc32=bool(acc32)))
        ro, so = ho.restrict(l, b, rescale=True, ctx=O.ctx(ftz))
        rr, sr = hr.restrict(l, b, rescale=True)
        assert same_bits(ro, rr) and so == sr
        c = O.round_vec(rng.standard_normal(ho.rows(l - 1)), ho.prec(l - 1), ftz)
        assert same_bits(ho.prolong(l, c, 0.5, ctx=O.ctx(ftz)), hr.prolong(l, c, 0.5))


@pytest.mark.parametrize("dim,n,L", [(3, 65, 6), (2, 129, 7)])
@pytest.mark.parametrize("variant", ["h_mg", "hsd_mg", "dsh_mg"])
def test_v_cycle_and_update(R, dim, n, L, variant):
    ho = O.hierarchy(dim, n, L, variant, ftz=False)
    hr = R.hierarchy(dim, n, L, variant, ftz=0)
    b = O.rhs(dim, n)
    rb, _ = R.rhs(dim, n)
    assert same_bits(b, rb)
    fp = ho.prec(L - 1)
    rl = O.cast(b, fp, O.norm2(b), O.ctx(False))
    assert same_bits(rl, R.cast(b, FP64, fp, R.norm2(b), ftz=0))
    c = ho.v_cycle(rl, O.ctx(False))
    assert same_bits(c, hr.v_cycle(rl))
    cols, vals = O.stiffness(dim, n)
    r0 = np.array(b); u0 = np.zeros_like(b)
    ro, uo = O.update_rc(cols, vals, r0, u0, c, 0.37, O.ctx(False))
    rr, ur = R.update_rc(dim, n, r0, u0, c, fp, 0.37, ftz=0)
    assert same_bits(ro, rr) and same_bits(uo, ur)


def test_ir_solve_random_guess(R):
    dim, n, L = 3, 33, 5
    ho = O.hierarchy(dim, n, L, "h_mg", ftz=False)
    hr = R.hierarchy(dim, n, L, "h_mg", ftz=0)
    b = O.rhs(dim, n)
    for refresh in (10, 3, 0):
        so = ho.ir_solve(b, tol=1e-9, random_guess=True, seed=42, refresh=refresh, ctx=O.ctx(False))
        sr = hr.ir_solve(rel_tol=0, abs_tol=1e-9, random_guess=True, seed=42, refresh=refresh)
        assert so["iterations"] == sr["iterations"]
        assert same_bits(so["history"], sr["history"])
        assert same_bits(so["u"], sr["u"])
