"""CPU tests of the parity oracle (oracle/mpmg_oracle.c).

The oracle is pinned three ways before any GPU result is compared with it:
  1. the reference's own known-answer tests, restated
     (proj/tests/test_precision.cpp, proj/tests/test_kernels.cpp), with an
     independent binary16 rounding (numpy's float64 -> float16 cast and exact
     rational arithmetic) standing in for the MPFR oracle (oracles.hpp:20-78);
  2. the golden fixtures in tests/golden/*.npz, generated from the unmodified
     reference library by tests/golden/make_golden.py;
  3. when oracle/_ref/libmpmg_ref.so is present, the reference itself on
     fresh seeded inputs (test_oracle_vs_reference.py).
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import FP16, FP32, FP64, Oracle

O = Oracle()
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"))


def same_bits(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


class SplitMix64:
    """rng.hpp:9-25."""

    def __init__(self, seed):
        self.s = seed & 0xFFFFFFFFFFFFFFFF

    def next_u64(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)

    def next_double(self):
        return (self.next_u64() >> 11) * 2.0 ** -53


# ---------------------------------------------------------------------------
# independent binary16 rounding of an exact rational (stands in for MPFR)
# ---------------------------------------------------------------------------
def round_q16(q: Fraction, ftz: bool) -> float:
    if q == 0:
        return 0.0
    s = -1.0 if q < 0 else 1.0
    a = abs(q)
    e = math.floor(math.log2(a.numerator) - math.log2(a.denominator))
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, -14)  # subnormal spacing 2^-24
    ulp = Fraction(2) ** (e - 10)
    m = a / ulp
    fl = math.floor(m)
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    v = float(fl * ulp)
    if v >= 65520.0 or v > 65504.0:
        return s * math.inf
    if ftz and v < 2.0 ** -14:
        return math.copysign(0.0, s)
    return s * v


def np16(x):
    return float(np.float64(x).astype(np.float16))


# ---------------------------------------------------------------------------
# 1. binary16 semantics (test_precision.cpp restated)
# ---------------------------------------------------------------------------
def test_limits_and_unit_roundoff():  # test_precision.cpp:43-66
    assert O.q16(65504.0) == 65504.0
    assert O.q16(65520.0) == math.inf and O.q16(65519.999999) == 65504.0
    assert O.q16(2.0 ** -24, ftz=False) == 2.0 ** -24
    assert O.q16(2.0 ** -25, ftz=False) == 0.0  # tie to even (zero)
    assert O.q16(1.0 + 2.0 ** -12) == 1.0
    assert O.fma16(1.0, 1.0, 2.0 ** -12, ftz=False) == 1.0


def test_exhaustive_round_trip_and_flush():  # test_precision.cpp:68-92
    L = O.L
    for bits in range(0x10000):
        w = L.orc_widen_fp16(bits)
        exp = (bits >> 10) & 0x1F
        man = bits & 0x3FF
        if exp == 0x1F and man:
            assert math.isnan(w)
            continue
        assert L.orc_pack_fp16(O.q16(w, ftz=False)) == bits
        f = O.q16(w, ftz=True)
        if exp == 0 and man:  # subnormal -> signed zero
            assert f == 0.0 and math.copysign(1.0, f) == (-1.0 if bits & 0x8000 else 1.0)
        else:
            assert L.orc_pack_fp16(f) == bits


def test_rounding_matches_independent_rne():  # test_precision.cpp:94-135
    cases = [0.0, -0.0, 1.0, -1.0, 65504.0, 65519.999999, 65520.0, 65521.0, 1e6, -1e6, 2.0 ** -14, 2.0 ** -24,
             2.0 ** -25, 1.5 * 2.0 ** -24, 2.0 ** -26, 2048.5, 2049.5, 0.1, -0.1, 3.14159265358979, 2.0 ** -130,
             -(2.0 ** -130), 1e300, math.inf, -math.inf]
    for e in range(-14, 16):
        for m in (0, 1, 2, 511, 512, 1022, 1023):
            half = 2.0 ** (e - 11)
            base = 2.0 ** e * (1.0 + m / 1024.0)
            cases += [base + half, np.nextafter(base + half, 0.0), np.nextafter(base + half, 1e308), -(base + half)]
    for m in range(1024):
        cases += [(m + 0.5) * 2.0 ** -24, -(m + 0.5) * 2.0 ** -24]
    rng = SplitMix64(0xC0FFEE)
    for _ in range(200000):
        ex = int(rng.next_u64() % 48) - 30
        mant = 1.0 + rng.next_double()
        sign = -1.0 if rng.next_u64() & 1 else 1.0
        cases.append(sign * math.ldexp(mant, ex))
    xs = np.array(cases)
    with np.errstate(over="ignore"):
        ref = xs.astype(np.float16).astype(np.float64)  # numpy: one correct RNE rounding
    mine = np.array([O.q16(x, ftz=False) for x in xs])
    assert same_bits(mine, ref)


def test_add_mul_fma_match_exact_rounding():  # test_precision.cpp:137-183
    rng = SplitMix64(0xABCDEF)

    def rnd16():
        bits = int(rng.next_u64() & 0xFFFF)
        if (bits >> 10) & 0x1F == 0x1F:
            bits &= 0xFBFF  # finite
        return O.L.orc_widen_fp16(bits)

    for _ in range(20000):
        a, b, c = rnd16(), rnd16(), rnd16()
        for ftz in (False, True):
            exact_fma = Fraction(a) * Fraction(b) + Fraction(c)
            assert O.fma16(a, b, c, ftz, True) == round_q16(exact_fma, ftz) or (
                exact_fma == 0 and O.fma16(a, b, c, ftz, True) == 0.0)
            assert O.L.orc_fp16_add(a, b, int(ftz)) == round_q16(Fraction(a) + Fraction(b), ftz) or a + b == 0
            assert O.L.orc_fp16_mul(a, b, int(ftz)) == round_q16(Fraction(a) * Fraction(b), ftz) or a * b == 0
            # commutativity (test_precision.cpp:160-163)
            assert same_bits(O.L.orc_fp16_add(a, b, int(ftz)), O.L.orc_fp16_add(b, a, int(ftz)))


def test_fused_versus_unfused_known_answers():  # test_precision.cpp:185-222
    a = 1.0 + 2.0 ** -10
    assert O.fma16(a, a, -1.0, False, True) == 2.0 ** -9
    assert O.fma16(a, a, -1.0, False, False) == 2.0 ** -9
    b = 1.0 - 2.0 ** -10
    assert O.fma16(a, b, -1.0, False, True) == -(2.0 ** -20)
    assert O.fma16(a, b, -1.0, False, False) == 0.0
    f = O.fma16(a, b, -1.0, True, True)
    assert f == 0.0 and math.copysign(1.0, f) == -1.0


def test_monotone_and_roundtrip_bound():  # test_precision.cpp:224-251
    rng = SplitMix64(0x12345)
    for _ in range(20000):
        ex = int(rng.next_u64() % 40) - 24
        x = math.ldexp(1.0 + rng.next_double(), ex)
        y = math.ldexp(1.0 + rng.next_double(), ex + int(rng.next_u64() % 3))
        if rng.next_u64() & 1:
            x, y = -x, -y
        if x > y:
            x, y = y, x
        assert O.q16(x, False) <= O.q16(y, False)
        assert O.q16(x, True) <= O.q16(y, True)
        if 2.0 ** -14 <= abs(x) <= 65504.0:
            assert abs(O.q16(x, True) - x) <= 2.0 ** -11 * abs(x)


def test_special_values():  # test_precision.cpp:267-279
    assert math.isnan(O.L.orc_fp16_add(math.inf, -math.inf, 0))
    assert O.L.orc_fp16_add(math.inf, 1.0, 0) == math.inf
    assert O.L.orc_fp16_mul(-math.inf, 2.0, 0) == -math.inf
    assert O.L.orc_pack_fp16(O.q16(math.nan)) == 0x7E00
    assert O.L.orc_pack_fp16(O.q16(-0.0)) == 0x8000
    assert O.L.orc_pack_fp16(O.q16(0.0)) == 0x0000


# ---------------------------------------------------------------------------
# 2. kernels (test_kernels.cpp restated) and golden fixtures
# ---------------------------------------------------------------------------
def test_spmv_identity_bitwise():  # test_kernels.cpp:92-106
    rng = np.random.default_rng(1)
    for p in (FP16, FP32, FP64):
        x = O.round_vec(rng.random(12) * 2 - 1, p)
        cols = np.arange(12, dtype=np.int32)[:, None]
        vals = np.ones((12, 1))
        assert same_bits(O.spmv(cols, vals, p, x), x)


def test_spmv_golden():  # test_kernels.cpp:108-145 restated on reference outputs
    g = gold("kernels")
    for k in range(int(g["spmv_count"])):
        cols, vals, x, prec = g[f"spmv_{k}_cols"], g[f"spmv_{k}_vals"], g[f"spmv_{k}_x"], int(g[f"spmv_{k}_prec"])
        for ftz in (0, 1):
            for fma in (0, 1):
                for acc32 in ((0, 1) if prec == FP16 else (0,)):
                    ctx = O.ctx(ftz, fma, acc32)
                    xr = O.round_vec(x, prec, ftz)
                    vr = np.array([O.round_vec(r, prec, ftz) for r in vals])
                    y = O.spmv(cols, vr, prec, xr, ctx)
                    assert same_bits(y, g[f"spmv_{k}_y_{ftz}{fma}{acc32}"]), (k, ftz, fma, acc32)


def test_spmv_fp32_accumulation_mode():  # test_kernels.cpp:129-145
    rng = SplitMix64(7)
    n = 16
    cols = np.zeros((n, 5), dtype=np.int32); vals = np.zeros((n, 5))
    for i in range(n):
        cs = sorted({int(rng.next_u64() % n) for _ in range(5)})
        for s in range(5):
            cols[i, s] = cs[s] if s < len(cs) else i
            vals[i, s] = O.q16(2 * rng.next_double() - 1) if s < len(cs) else 0.0
    x = O.round_vec([2 * rng.next_double() - 1 for _ in range(n)], FP16)
    y = O.spmv(cols, vals, FP16, x, O.ctx(True, True, True))
    for i in range(n):
        acc = np.float32(0.0)
        for s in range(5):  # fmaf chain (exact product of two binary16 in binary64, one rounding)
            acc = np.float32(float(np.float32(vals[i, s])) * float(np.float32(x[cols[i, s]])) + float(acc))
        assert y[i] == O.q16(float(acc), True)


def test_axpy_and_vec_multiply_known_answers():  # test_kernels.cpp:147-195
    rng = np.random.default_rng(3)
    for p in (FP16, FP32, FP64):
        x = O.round_vec(rng.random(33) * 2 - 1, p); y = O.round_vec(rng.random(33) * 2 - 1, p)
        assert same_bits(O.axpy(p, 0.0, x, y), y)
        neg = O.axpy(p, -2.0, x, x)
        assert not O.axpy(p, 1.0, x, neg).any()
        assert same_bits(O.vec_multiply(p, x, np.ones(33)), x)
    assert math.isinf(O.vec_multiply(FP16, [300.0], [300.0])[0])
    x16 = O.round_vec(rng.random(200) * 1.5 + 0.5, FP16); y16 = O.round_vec(rng.random(200) * 1.5 + 0.5, FP16)
    z = O.axpy(FP16, 0.7, x16, y16)
    a16 = O.q16(0.7)
    exact = y16 + a16 * x16
    assert np.all(np.abs(z - exact) <= 2.0 ** -10 * np.abs(exact))


def test_update_rc_golden_and_unfused_identity():  # test_kernels.cpp:197-247, kernels.cpp:300-341
    g = gold("kernels")
    for j in range(int(g["urc_count"])):
        dim, n, cp, ftz, alpha = g[f"urc_{j}_meta"]
        cols, vals = O.stiffness(int(dim), int(n))
        ctx = O.ctx(bool(ftz), True, False)
        r, u = O.update_rc(cols, vals, g[f"urc_{j}_r"], g[f"urc_{j}_u"], g[f"urc_{j}_c"], alpha, ctx)
        assert same_bits(r, g[f"urc_{j}_r_out"]) and same_bits(u, g[f"urc_{j}_u_out"])
        # fused == cast + axpy + spmv + axpy (bitwise)
        wc = g[f"urc_{j}_c"]
        u_ref = O.axpy(FP64, alpha, wc, g[f"urc_{j}_u"], ctx)
        Ac = O.spmv(cols, vals, FP64, wc, ctx)
        r_ref = O.axpy(FP64, -alpha, Ac, g[f"urc_{j}_r"], ctx)
        assert same_bits(r, r_ref) and same_bits(u, u_ref)


def test_cast_golden_and_flush_boundary():  # test_kernels.cpp:249-289
    g = gold("kernels")
    x = g["cast_x"]
    nx = O.norm2(x)
    assert nx == float(g["cast_norm"])
    for ftz in (0, 1):
        for tgt in (FP16, FP32):
            ctx = O.ctx(bool(ftz))
            s = O.cast(x, tgt, nx, ctx)
            assert same_bits(s, g[f"cast_{tgt}_{ftz}_scaled"])
            assert same_bits(O.cast(x, tgt, 1.0, ctx), g[f"cast_{tgt}_{ftz}_unscaled"])
    s = O.cast(x, FP16, nx)
    keep = np.abs(x) >= 2.0 ** -14 * nx
    assert np.all(s[keep] != 0)
    assert 1 - 2.0 ** -9 <= O.norm2(s) <= 1 + 2.0 ** -9
    assert not O.cast(x, FP16, 1.0).any()
    for bad in (0.0, -1.0, math.inf):
        with pytest.raises(ValueError):
            O.cast(x, FP16, bad)


def test_norm_against_compensated():  # test_kernels.cpp:331-339
    rng = np.random.default_rng(23)
    x = rng.random(256) * 2 - 1
    s = Fraction(0)
    for v in x:
        s += Fraction(v) * Fraction(v)
    ref = math.sqrt(float(s))
    assert abs(O.norm2(x) - ref) <= 1e-14 * ref


# ---------------------------------------------------------------------------
# 3. hierarchy, V-cycle, CG and IR against the reference's own outputs
# ---------------------------------------------------------------------------
VARIANTS = ["d_mg", "h_mg", "dsh_mg", "hsd_mg"]


@pytest.mark.parametrize("dim,n,L", [(2, 17, 4), (3, 9, 3), (2, 65, 6), (3, 33, 5)])
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("ftz", [0, 1])
def test_hierarchy_golden(dim, n, L, variant, ftz):  # multigrid.cpp:282-323, mesh_fem.cpp:71-295
    g = gold("hierarchy")
    key = f"{dim}_{n}_{variant}_{ftz}"
    h = O.hierarchy(dim, n, L, variant, ftz=bool(ftz))
    assert [h.prec(l) for l in range(L)] == list(g[f"{key}_prec"])
    assert [h.rows(l) for l in range(L)] == list(g[f"{key}_rows"])
    for l in range(L):
        cols, vals = h.matrix(l, 0)
        assert same_bits(h.invdiag(l), g[f"{key}_l{l}_invdiag"])
        if n <= 17:
            assert np.array_equal(cols, g[f"{key}_l{l}_A_cols"])
            assert same_bits(vals, g[f"{key}_l{l}_A_vals"])
            if l < L - 1:
                for w, nm in ((1, "P"), (2, "R")):
                    c2, v2 = h.matrix(l, w)
                    assert np.array_equal(c2, g[f"{key}_l{l}_{nm}_cols"]), nm
                    assert same_bits(v2, g[f"{key}_l{l}_{nm}_vals"]), nm
        else:
            m = (n - 1) >> (L - 1 - l)
            c = (m - 2) // 2
            row = c + (m - 1) * c + ((m - 1) ** 2 * c if dim == 3 else 0)
            assert same_bits(vals[row], g[f"{key}_l{l}_A_row"])


def test_stencil_and_rhs_golden():  # mesh_fem.cpp:71-202
    g = gold("hierarchy")
    for dim, n in ((2, 5), (2, 9), (2, 33), (2, 257), (3, 5), (3, 9), (3, 17), (3, 65), (3, 129), (3, 257)):
        assert same_bits(O.stencil(dim, n), g[f"stencil_{dim}_{n}"]), (dim, n)
    for dim, n in ((2, 33), (3, 17)):
        assert same_bits(O.rhs(dim, n), g[f"rhs_{dim}_{n}"])
        assert same_bits(O.exact(dim, n), g[f"exact_{dim}_{n}"])


def test_v_cycle_golden():  # multigrid.cpp:354-393
    g = gold("cycles")
    n_checked = 0
    for dim, n, L in ((2, 33, 5), (3, 17, 4), (3, 33, 5)):
        for variant in VARIANTS:
            for ftz in (0, 1):
                for acc32 in (0, 1):
                    key = f"{dim}_{n}_{variant}_{ftz}_{acc32}"
                    if f"vc_{key}_in" not in g:
                        continue
                    h = O.hierarchy(dim, n, L, variant, ftz=bool(ftz))
                    c = h.v_cycle(g[f"vc_{key}_in"], O.ctx(bool(ftz), True, bool(acc32)))
                    assert same_bits(c, g[f"vc_{key}_out"]), key
                    n_checked += 1
    assert n_checked == 36


def test_cg_golden():  # multigrid.cpp:91-151
    g = gold("cycles")
    for dim, n in ((2, 65), (3, 33)):
        for variant in ("d_mg", "h_mg", "hsd_mg"):
            key = f"cg_{dim}_{n}_{variant}"
            h = O.hierarchy(dim, n, 3, variant, ftz=True)
            u, it, conv, res = h.cg(0, g[f"{key}_b"])
            assert same_bits(u, g[f"{key}_u"])
            assert [it, int(conv)] == [int(v) for v in g[f"{key}_meta"][:2]]
            assert res == g[f"{key}_meta"][2]


SOLVES = ["cfg0", "3_65_h_mg_ftz0", "3_65_h_mg_ftz1", "3_65_hsd_mg_ftz0", "3_65_dsh_mg_ftz0", "3_65_d_mg_ftz0",
          "2_257_h_mg_ftz0", "2_257_hsd_mg_ftz1", "3_33_h_mg_ftz0"]


@pytest.mark.parametrize("name", SOLVES)
def test_ir_solve_golden(name):  # ir_solver.cpp:51-127
    g = gold("solves")
    dim, n, L, v, pre, post, ftz, its, conv = [int(x) for x in g[f"{name}_meta"]]
    h = O.hierarchy(dim, n, L, VARIANTS[v], pre=pre, post=post, ftz=bool(ftz))
    b = O.rhs(dim, n)
    s = h.ir_solve(b, rel_tol=1e-10, ctx=O.ctx(bool(ftz)))
    assert s["iterations"] == its and s["converged"] == bool(conv)
    assert same_bits(s["history"], g[f"{name}_history"])
    assert s["final_residual"] == float(g[f"{name}_final"])
    if f"{name}_u" in g:
        assert same_bits(s["u"], g[f"{name}_u"])


@pytest.mark.parametrize("dim,n,L", [(2, 17, 4), (3, 9, 3), (3, 17, 4), (2, 33, 5)])
@pytest.mark.parametrize("variant", ["d_mg", "h_mg", "hsd_mg", "dsh_mg"])
@pytest.mark.parametrize("ftz", [0, 1])
def test_implicit_operators_equal_assembled(dim, n, L, variant, ftz):
    """The oracle's implicit level operators (rows generated on demand, used
    at 257^3 where the assembled ELL is GBs) are the assembled ELL matrices
    row for row -- columns, values and padding -- and give bitwise the same
    V-cycle (mesh_fem.cpp:124-150, 204-295; ell_matrix.cpp:90-92)."""
    he = O.hierarchy(dim, n, L, variant, ftz=ftz)
    hi = O.hierarchy(dim, n, L, variant, ftz=ftz, implicit=True)
    for l in range(L):
        assert same_bits(he.invdiag(l), hi.invdiag(l))
        for which in (0, 1, 2):
            a, b = he.matrix(l, which), hi.matrix(l, which)
            if a is None:
                assert b is None
                continue
            assert np.array_equal(a[0], b[0]) and same_bits(a[1], b[1]), (l, which)
    b = O.rhs(dim, n)
    ctx = O.ctx(ftz)
    rl = O.cast(b, he.prec(L - 1), O.norm2(b) if variant != "d_mg" else 1.0, ctx)
    assert same_bits(he.v_cycle(rl, ctx), hi.v_cycle(rl, ctx))
    A = O.stiffness(dim, n)
    Ai = O.stiffness_implicit(dim, n)
    u = np.random.default_rng(3).random(len(b))
    assert same_bits(O.spmv(A[0], A[1], FP64, u), O.spmv_e(Ai, u))
    assert O.L.orc_residual_norm(Ai, u, b) == O.residual_norm_e(Ai, u, b)


def test_implicit_ir_solve_equals_assembled():
    ho = O.hierarchy(3, 33, 5, "h_mg", ftz=False)
    hi = O.hierarchy(3, 33, 5, "h_mg", ftz=False, implicit=True)
    b = O.rhs(3, 33)
    s1 = ho.ir_solve(b, ctx=O.ctx(False))
    s2 = hi.ir_solve(b, ctx=O.ctx(False))
    assert s1["iterations"] == s2["iterations"]
    assert same_bits(s1["history"], s2["history"]) and same_bits(s1["u"], s2["u"])
