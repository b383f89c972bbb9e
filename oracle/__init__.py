"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product.

ctypes bindings for
  * ``Oracle``: the plain-C restatement of the reference (``mpmg_oracle.c``),
  * ``Reference``: the unmodified reference library compiled from
    /root/reference by ``oracle/Makefile`` (``_ref/libmpmg_ref.so``) behind our
    extern "C" shim (``ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package. The product
(``paper_2007_07539_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmpmg_ref.so")

FP16, FP32, FP64 = 0, 1, 2
D_MG, H_MG, DSH_MG, HSD_MG = 0, 1, 2, 3
VARIANTS = {"d_mg": D_MG, "h_mg": H_MG, "dsh_mg": DSH_MG, "hsd_mg": HSD_MG}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def build(quiet: bool = True) -> None:
    """Compile the oracle (and, when /root/reference is present, the reference)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def unknowns(dim: int, n: int) -> int:
    m = n - 2
    return m * m if dim == 2 else m * m * m


def nodes_at_level(n: int, levels: int, l: int) -> int:
    return ((n - 1) >> (levels - 1 - l)) + 1


class _Ctx(C.Structure):
    _fields_ = [("ftz", C.c_int), ("fma", C.c_int), ("acc32", C.c_int)]


class _Ell(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("rw", C.c_int), ("prec", C.c_int),
                ("col", C.POINTER(C.c_int32)), ("val", C.POINTER(C.c_double)),
                ("gen", C.c_int), ("gdim", C.c_int), ("gn", C.c_int), ("gtaps", C.c_double * 27)]


def _ell_to_numpy(e: _Ell, lib=None):
    n = e.rows * e.rw
    if e.gen:  # implicit operator: generate the rows
        cols = np.zeros((e.rows, e.rw), dtype=np.int32)
        vals = np.zeros((e.rows, e.rw))
        lib.orc_ell_rows(C.byref(e), cols, vals)
        return cols, vals
    cols = np.ctypeslib.as_array(e.col, shape=(n,)).copy().reshape(e.rows, e.rw)
    vals = np.ctypeslib.as_array(e.val, shape=(n,)).copy().reshape(e.rows, e.rw)
    return cols, vals


class Oracle:
    """The C restatement (mpmg_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        d, i, i64 = C.c_double, C.c_int, C.c_int64
        L.orc_quantize_fp16.restype = d; L.orc_quantize_fp16.argtypes = [d, i]
        L.orc_fp16_fma.restype = d; L.orc_fp16_fma.argtypes = [d, d, d, i, i]
        L.orc_fp16_add.restype = d; L.orc_fp16_add.argtypes = [d, d, i]
        L.orc_fp16_mul.restype = d; L.orc_fp16_mul.argtypes = [d, d, i]
        L.orc_pack_fp16.restype = C.c_uint; L.orc_pack_fp16.argtypes = [d]
        L.orc_widen_fp16.restype = d; L.orc_widen_fp16.argtypes = [C.c_uint]
        L.orc_round.restype = d; L.orc_round.argtypes = [d, i, i]
        L.orc_spmv.argtypes = [C.POINTER(_Ell), _dp, _dp, _Ctx]
        L.orc_axpy.argtypes = [i, d, _dp, _dp, _dp, i64, _Ctx]
        L.orc_vec_multiply.argtypes = [i, _dp, _dp, _dp, i64, _Ctx]
        L.orc_update_rc.argtypes = [_dp, _dp, C.POINTER(_Ell), _dp, d, _Ctx]
        L.orc_cast.restype = i; L.orc_cast.argtypes = [_dp, i64, i, d, _dp, _Ctx]
        L.orc_dot.restype = d; L.orc_dot.argtypes = [_dp, _dp, i64]
        L.orc_norm2.restype = d; L.orc_norm2.argtypes = [_dp, i64]
        L.orc_stiffness.restype = i; L.orc_stiffness.argtypes = [i, i, C.POINTER(_Ell)]
        L.orc_stencil.restype = i; L.orc_stencil.argtypes = [i, i, _dp]
        L.orc_transfer.restype = i; L.orc_transfer.argtypes = [i, i, C.POINTER(_Ell), C.POINTER(_Ell)]
        L.orc_rhs.argtypes = [i, i, i, _dp]
        L.orc_exact.argtypes = [i, i, i, _dp]
        L.orc_ell_free.argtypes = [C.POINTER(_Ell)]
        L.orc_ell_rows.argtypes = [C.POINTER(_Ell), _ip, _dp]
        L.orc_spmv_rows.argtypes = [C.POINTER(_Ell), _dp, _dp, i64, i64, _Ctx]
        L.orc_transfer_rows.argtypes = [C.POINTER(_Ell), _dp, i, _dp, i64, i64, _Ctx]
        L.orc_stiffness_implicit.restype = i; L.orc_stiffness_implicit.argtypes = [i, i, C.POINTER(_Ell)]
        L.orc_hier_build_ex.restype = C.c_void_p
        L.orc_hier_build_ex.argtypes = [i, i, i, i, i, i, d, d, i, i, i, i, C.POINTER(C.c_int), i]
        L.orc_hier_build.restype = C.c_void_p
        L.orc_hier_build.argtypes = [i, i, i, i, i, i, d, d, i, i, i, i, C.POINTER(C.c_int)]
        L.orc_hier_free.argtypes = [C.c_void_p]
        L.orc_hier_levels.restype = i; L.orc_hier_levels.argtypes = [C.c_void_p]
        L.orc_level_prec.restype = i; L.orc_level_prec.argtypes = [C.c_void_p, i]
        L.orc_level_rows.restype = i64; L.orc_level_rows.argtypes = [C.c_void_p, i]
        L.orc_level_matrix.restype = C.POINTER(_Ell); L.orc_level_matrix.argtypes = [C.c_void_p, i, i]
        L.orc_level_invdiag.restype = C.POINTER(C.c_double); L.orc_level_invdiag.argtypes = [C.c_void_p, i]
        L.orc_jacobi.argtypes = [C.c_void_p, i, _dp, _dp, i, d, _Ctx]
        L.orc_restrict.restype = d; L.orc_restrict.argtypes = [C.c_void_p, i, _dp, i, _dp, _Ctx]
        L.orc_prolong.restype = i; L.orc_prolong.argtypes = [C.c_void_p, i, _dp, d, _dp, _Ctx]
        L.orc_cg.restype = i; L.orc_cg.argtypes = [C.c_void_p, i, _dp, _dp, C.POINTER(C.c_int), C.POINTER(C.c_double), _Ctx]
        L.orc_v_cycle.argtypes = [C.c_void_p, _dp, _dp, _Ctx]
        L.orc_residual_norm.restype = d; L.orc_residual_norm.argtypes = [C.POINTER(_Ell), _dp, _dp]
        L.orc_ir_solve.restype = i
        L.orc_ir_solve.argtypes = [C.c_void_p, C.POINTER(_Ell), _dp, d, i, i, C.c_uint64, i, i, _Ctx, _dp, _dp, i,
                                   C.POINTER(C.c_int), C.POINTER(C.c_double)]

    @staticmethod
    def ctx(ftz=True, fma=True, acc32=False):
        return _Ctx(int(ftz), int(fma), int(acc32))

    # --- scalars
    def q16(self, x, ftz=True):
        return self.L.orc_quantize_fp16(float(x), int(ftz))

    def fma16(self, a, b, c, ftz=True, fma=True):
        return self.L.orc_fp16_fma(float(a), float(b), float(c), int(ftz), int(fma))

    def round_vec(self, xs, prec, ftz=True):
        f = self.L.orc_round
        return np.array([f(float(x), prec, int(ftz)) for x in np.asarray(xs, dtype=np.float64)])

    # --- assembly
    def stiffness(self, dim, n):
        e = _Ell()
        if self.L.orc_stiffness(dim, n, C.byref(e)):
            raise ValueError("stiffness")
        out = _ell_to_numpy(e)
        self.L.orc_ell_free(C.byref(e))
        return out

    def stencil(self, dim, n):
        taps = np.zeros(27)
        k = self.L.orc_stencil(dim, n, taps)
        return taps[:k].copy()

    def stiffness_implicit(self, dim, n):
        """The FP64 operator as an implicit row generator (bitwise the
        assembled ELL; for 257^3 and up, where the slot arrays are GBs)."""
        e = _Ell()
        if self.L.orc_stiffness_implicit(dim, n, C.byref(e)):
            raise ValueError("stiffness")
        return e

    def transfer(self, dim, nf):
        P, R = _Ell(), _Ell()
        if self.L.orc_transfer(dim, nf, C.byref(P), C.byref(R)):
            raise ValueError("transfer")
        out = (_ell_to_numpy(P), _ell_to_numpy(R))
        self.L.orc_ell_free(C.byref(P)); self.L.orc_ell_free(C.byref(R))
        return out

    def rhs(self, dim, n, k=1):
        b = np.zeros(unknowns(dim, n))
        self.L.orc_rhs(dim, n, k, b)
        return b

    def exact(self, dim, n, k=1):
        u = np.zeros(unknowns(dim, n))
        self.L.orc_exact(dim, n, k, u)
        return u

    def norm2(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self.L.orc_norm2(x, x.size)

    # --- generic ELL kernels on numpy arrays
    def spmv(self, cols, vals, prec, x, ctx=None, n_cols=None):
        cols = np.ascontiguousarray(cols, dtype=np.int32); vals = np.ascontiguousarray(vals, dtype=np.float64)
        rows, rw = cols.shape
        e = _Ell(rows, n_cols or len(x), rw, prec, cols.ctypes.data_as(C.POINTER(C.c_int32)),
                 vals.ctypes.data_as(C.POINTER(C.c_double)))
        y = np.zeros(rows)
        self.L.orc_spmv(C.byref(e), np.ascontiguousarray(x, dtype=np.float64), y, ctx or self.ctx())
        return y

    # --- kernels on an _Ell (explicit or implicit, e.g. stiffness_implicit)
    def spmv_e(self, e, x, ctx=None):
        y = np.zeros(e.rows)
        self.L.orc_spmv(C.byref(e), np.ascontiguousarray(x, dtype=np.float64), y, ctx or self.ctx())
        return y

    def spmv_rows(self, e, x, r0, r1, ctx=None):
        """rows [r0, r1) of A x (sampled checks at sizes where a whole pass is slow)"""
        y = np.zeros(r1 - r0)
        self.L.orc_spmv_rows(C.byref(e), np.ascontiguousarray(x, dtype=np.float64), y, r0, r1, ctx or self.ctx())
        return y

    def transfer_rows(self, e, x, prec, r0, r1, ctx=None):
        """rows [r0, r1) of the transfer product (restriction / prolongation) in precision prec"""
        y = np.zeros(r1 - r0)
        self.L.orc_transfer_rows(C.byref(e), np.ascontiguousarray(x, dtype=np.float64), prec, y, r0, r1,
                                 ctx or self.ctx())
        return y

    def update_rc_e(self, e, r, u, c, alpha, ctx=None):
        r = np.array(r, dtype=np.float64); u = np.array(u, dtype=np.float64)
        self.L.orc_update_rc(r, u, C.byref(e), np.ascontiguousarray(c, dtype=np.float64), float(alpha),
                             ctx or self.ctx())
        return r, u

    def residual_norm_e(self, e, u, b):
        return self.L.orc_residual_norm(C.byref(e), np.ascontiguousarray(u, dtype=np.float64),
                                        np.ascontiguousarray(b, dtype=np.float64))

    def update_rc(self, cols, vals, r, u, c, alpha, ctx=None):
        cols = np.ascontiguousarray(cols, dtype=np.int32); vals = np.ascontiguousarray(vals, dtype=np.float64)
        rows, rw = cols.shape
        e = _Ell(rows, rows, rw, FP64, cols.ctypes.data_as(C.POINTER(C.c_int32)),
                 vals.ctypes.data_as(C.POINTER(C.c_double)))
        r = np.array(r, dtype=np.float64); u = np.array(u, dtype=np.float64)
        self.L.orc_update_rc(r, u, C.byref(e), np.ascontiguousarray(c, dtype=np.float64), float(alpha),
                             ctx or self.ctx())
        return r, u

    def cast(self, x, target, scale=1.0, ctx=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros_like(x)
        if self.L.orc_cast(x, x.size, target, float(scale), out, ctx or self.ctx()):
            raise ValueError("cast_vector: scale must be positive and finite")
        return out

    def axpy(self, prec, alpha, x, y, ctx=None):
        x = np.ascontiguousarray(x, dtype=np.float64); y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.zeros_like(x)
        self.L.orc_axpy(prec, float(alpha), x, y, out, x.size, ctx or self.ctx())
        return out

    def vec_multiply(self, prec, a, b, ctx=None):
        a = np.ascontiguousarray(a, dtype=np.float64); b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.zeros_like(a)
        self.L.orc_vec_multiply(prec, a, b, out, a.size, ctx or self.ctx())
        return out

    def hierarchy(self, dim, n, levels, variant, pre=3, post=3, omega=2.0 / 3.0, base_tol=1e-4, base_mode=0,
                  base_maxit=0, ftz=True, fma=True, implicit=False):
        return OracleHierarchy(self, dim, n, levels, variant, pre, post, omega, base_tol, base_mode, base_maxit,
                               ftz, fma, implicit)


class OracleHierarchy:
    def __init__(self, o: Oracle, dim, n, levels, variant, pre, post, omega, base_tol, base_mode, base_maxit,
                 ftz, fma, implicit=False):
        self.o, self.dim, self.n, self.L = o, dim, n, levels
        self.implicit = bool(implicit)
        err = C.c_int(-1)
        if isinstance(variant, str):
            variant = VARIANTS[variant]
        self.variant = variant
        self.h = o.L.orc_hier_build_ex(dim, n, levels, variant, pre, post, omega, base_tol, base_mode,
                                       base_maxit, int(ftz), int(fma), C.byref(err), int(implicit))
        if not self.h:
            raise RuntimeError(f"oracle hierarchy build failed (level {err.value})")

    def __del__(self):
        if getattr(self, "h", None):
            self.o.L.orc_hier_free(self.h)
            self.h = None

    def prec(self, l):
        return self.o.L.orc_level_prec(self.h, l)

    def rows(self, l):
        return self.o.L.orc_level_rows(self.h, l)

    def matrix(self, l, which=0):
        p = self.o.L.orc_level_matrix(self.h, l, which)
        if not p:
            return None
        return _ell_to_numpy(p.contents, self.o.L)

    def invdiag(self, l):
        p = self.o.L.orc_level_invdiag(self.h, l)
        return np.ctypeslib.as_array(p, shape=(self.rows(l),)).copy()

    def jacobi(self, l, b, u, steps, omega=2.0 / 3.0, ctx=None):
        u = np.array(u, dtype=np.float64)
        self.o.L.orc_jacobi(self.h, l, np.ascontiguousarray(b, dtype=np.float64), u, steps, omega,
                            ctx or self.o.ctx())
        return u

    def restrict(self, l, r_fine, rescale=False, ctx=None):
        out = np.zeros(self.rows(l - 1))
        s = self.o.L.orc_restrict(self.h, l, np.ascontiguousarray(r_fine, dtype=np.float64), int(rescale), out,
                                  ctx or self.o.ctx())
        return out, s

    def prolong(self, l, c_coarse, scale=1.0, ctx=None):
        out = np.zeros(self.rows(l))
        self.o.L.orc_prolong(self.h, l, np.ascontiguousarray(c_coarse, dtype=np.float64), float(scale), out,
                             ctx or self.o.ctx())
        return out

    def cg(self, l, b, ctx=None):
        u = np.zeros(self.rows(l))
        conv, res = C.c_int(0), C.c_double(0)
        it = self.o.L.orc_cg(self.h, l, np.ascontiguousarray(b, dtype=np.float64), u, C.byref(conv), C.byref(res),
                             ctx or self.o.ctx())
        return u, it, bool(conv.value), res.value

    def v_cycle(self, b, ctx=None):
        c = np.zeros(self.rows(self.L - 1))
        self.o.L.orc_v_cycle(self.h, np.ascontiguousarray(b, dtype=np.float64), c, ctx or self.o.ctx())
        return c

    def ir_solve(self, b, A=None, tol=None, rel_tol=1e-10, max_it=100, random_guess=False, seed=0, scaling=0,
                 refresh=10, ctx=None):
        """Returns dict(iterations, history, converged, final_residual, u)."""
        if A is None and self.implicit:
            e = self.o.stiffness_implicit(self.dim, self.n)
            rows = e.rows
        else:
            if A is None:
                A = self.o.stiffness(self.dim, self.n)
            cols = np.ascontiguousarray(A[0], dtype=np.int32); vals = np.ascontiguousarray(A[1], dtype=np.float64)
            rows, rw = cols.shape
            e = _Ell(rows, rows, rw, FP64, cols.ctypes.data_as(C.POINTER(C.c_int32)),
                     vals.ctypes.data_as(C.POINTER(C.c_double)))
        b = np.ascontiguousarray(b, dtype=np.float64)
        if tol is None:
            tol = rel_tol * self.o.norm2(b)
        u = np.zeros(rows); hist = np.zeros(max_it + 2)
        conv, fres = C.c_int(0), C.c_double(0)
        its = self.o.L.orc_ir_solve(self.h, C.byref(e), b, tol, max_it, int(random_guess), seed, scaling, refresh,
                                    ctx or self.o.ctx(), u, hist, max_it + 2, C.byref(conv), C.byref(fres))
        if its == -2:
            raise FloatingPointError("ir_solve diverged")
        if its < 0:
            raise ValueError("ir_solve usage error")
        return dict(iterations=its, history=hist[:its + 1].copy(), converged=bool(conv.value),
                    final_residual=fres.value, u=u)


class Reference:
    """The unmodified reference (oracle/_ref/libmpmg_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        d, i, i64, vp = C.c_double, C.c_int, C.c_int64, C.c_void_p
        L.ref_quantize_fp16.restype = d; L.ref_quantize_fp16.argtypes = [d, i]
        L.ref_fp16_fma.restype = d; L.ref_fp16_fma.argtypes = [d, d, d, i, i]
        L.ref_round_to_fp16_bits.restype = C.c_uint; L.ref_round_to_fp16_bits.argtypes = [d, i]
        L.ref_widen_bits.restype = d; L.ref_widen_bits.argtypes = [C.c_uint]
        L.ref_unknowns.restype = i64; L.ref_unknowns.argtypes = [i, i]
        L.ref_problem_rhs.restype = i; L.ref_problem_rhs.argtypes = [i, i, i, _dp, _dp]
        L.ref_stencil.restype = i; L.ref_stencil.argtypes = [i, i, _dp]
        L.ref_stiffness.restype = i; L.ref_stiffness.argtypes = [i, i, C.c_void_p, C.c_void_p]
        L.ref_hier_build.restype = vp
        L.ref_hier_build.argtypes = [i, i, i, i, i, i, i, d, d, i, i, i, i]
        L.ref_hier_free.argtypes = [vp]
        L.ref_hier_build_seconds.restype = d; L.ref_hier_build_seconds.argtypes = [vp]
        L.ref_hier_levels.restype = i; L.ref_hier_levels.argtypes = [vp]
        L.ref_level_prec.restype = i; L.ref_level_prec.argtypes = [vp, i]
        L.ref_level_rows.restype = i64; L.ref_level_rows.argtypes = [vp, i]
        L.ref_level_matrix_shape.restype = i
        L.ref_level_matrix_shape.argtypes = [vp, i, i, C.POINTER(i64), C.POINTER(i64)]
        L.ref_level_matrix.restype = i; L.ref_level_matrix.argtypes = [vp, i, i, _ip, _dp]
        L.ref_level_invdiag.restype = i; L.ref_level_invdiag.argtypes = [vp, i, _dp]
        L.ref_level_spmv.restype = i; L.ref_level_spmv.argtypes = [vp, i, _dp, _dp, i, i, i]
        L.ref_level_jacobi.restype = i; L.ref_level_jacobi.argtypes = [vp, i, _dp, _dp, i, d, i, i, i]
        L.ref_level_defect.restype = i; L.ref_level_defect.argtypes = [vp, i, _dp, _dp, _dp, i, i, i]
        L.ref_level_restrict.restype = d; L.ref_level_restrict.argtypes = [vp, i, _dp, i, _dp, i, i]
        L.ref_level_prolong.restype = i; L.ref_level_prolong.argtypes = [vp, i, _dp, d, _dp, i, i]
        L.ref_level_cg.restype = i
        L.ref_level_cg.argtypes = [vp, i, _dp, _dp, C.POINTER(i), C.POINTER(i), C.POINTER(d), i, i]
        L.ref_v_cycle.restype = i; L.ref_v_cycle.argtypes = [vp, _dp, _dp, i, i, i]
        L.ref_update_rc.restype = i; L.ref_update_rc.argtypes = [i, i, _dp, _dp, _dp, i, d, i, i]
        L.ref_defect64.restype = i; L.ref_defect64.argtypes = [i, i, _dp, _dp, _dp]
        L.ref_cast.restype = i; L.ref_cast.argtypes = [_dp, i64, i, i, d, _dp, i]
        L.ref_norm2.restype = d; L.ref_norm2.argtypes = [_dp, i64, i]
        L.ref_ell_spmv.restype = i; L.ref_ell_spmv.argtypes = [i64, i64, i, _ip, _dp, i, _dp, _dp, i, i, i]
        L.ref_ir_solve.restype = i
        L.ref_ir_solve.argtypes = [vp, d, d, i, i, C.c_uint64, i, i, i, i, i, C.c_void_p, _dp, i,
                                   C.POINTER(i), C.POINTER(d), C.POINTER(d), C.POINTER(d)]

    def q16(self, x, ftz=True):
        return self.L.ref_quantize_fp16(float(x), int(ftz))

    def fma16(self, a, b, c, ftz=True, fma=True):
        return self.L.ref_fp16_fma(float(a), float(b), float(c), int(ftz), int(fma))

    def rhs(self, dim, n, k=1):
        N = self.L.ref_unknowns(dim, n)
        b = np.zeros(N); u = np.zeros(N)
        self.L.ref_problem_rhs(dim, k, n, b, u)
        return b, u

    def stencil(self, dim, n):
        taps = np.zeros(27)
        k = self.L.ref_stencil(dim, n, taps)
        return taps[:k].copy()

    def stiffness(self, dim, n):
        N = self.L.ref_unknowns(dim, n)
        rw = 9 if dim == 2 else 27
        cols = np.zeros(N * rw, dtype=np.int32); vals = np.zeros(N * rw)
        self.L.ref_stiffness(dim, n, cols.ctypes.data, vals.ctypes.data)
        return cols.reshape(N, rw), vals.reshape(N, rw)

    def hierarchy(self, dim, n, levels, variant, pre=3, post=3, omega=2.0 / 3.0, base_tol=1e-4, base_mode=0,
                  base_maxit=0, ftz=True, fma=True, k=1):
        return RefHierarchy(self, dim, n, levels, variant, pre, post, omega, base_tol, base_mode, base_maxit,
                            ftz, fma, k)

    def cast(self, x, src, dst, scale, ftz=True):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros_like(x)
        if self.L.ref_cast(x, x.size, src, dst, float(scale), out, int(ftz)):
            raise ValueError("cast_vector")
        return out

    def norm2(self, x, prec=FP64):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self.L.ref_norm2(x, x.size, prec)

    def update_rc(self, dim, n, r, u, c, c_prec, alpha, ftz=True, fma=True):
        r = np.array(r, dtype=np.float64); u = np.array(u, dtype=np.float64)
        if self.L.ref_update_rc(dim, n, r, u, np.ascontiguousarray(c, dtype=np.float64), c_prec, float(alpha),
                                int(ftz), int(fma)):
            raise RuntimeError("update_rc")
        return r, u

    def defect64(self, dim, n, b, u):
        r = np.zeros(len(b))
        self.L.ref_defect64(dim, n, np.ascontiguousarray(b, dtype=np.float64),
                            np.ascontiguousarray(u, dtype=np.float64), r)
        return r

    def ell_spmv(self, cols, vals, prec, x, ftz=True, fma=True, acc32=False, n_cols=None):
        cols = np.ascontiguousarray(cols, dtype=np.int32); vals = np.ascontiguousarray(vals, dtype=np.float64)
        rows, rw = cols.shape
        y = np.zeros(rows)
        self.L.ref_ell_spmv(rows, n_cols or len(x), rw, cols.reshape(-1), vals.reshape(-1), prec,
                            np.ascontiguousarray(x, dtype=np.float64), y, int(ftz), int(fma), int(acc32))
        return y


class RefHierarchy:
    def __init__(self, r: Reference, dim, n, levels, variant, pre, post, omega, base_tol, base_mode, base_maxit,
                 ftz, fma, k):
        if isinstance(variant, str):
            variant = VARIANTS[variant]
        self.r, self.dim, self.n, self.L, self.ftz, self.fma = r, dim, n, levels, ftz, fma
        self.h = r.L.ref_hier_build(dim, k, n, levels, variant, pre, post, omega, base_tol, base_mode, base_maxit,
                                    int(ftz), int(fma))
        if not self.h:
            raise RuntimeError("reference hierarchy build failed")
        self.build_seconds = r.L.ref_hier_build_seconds(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.r.L.ref_hier_free(self.h)
            self.h = None

    def prec(self, l):
        return self.r.L.ref_level_prec(self.h, l)

    def rows(self, l):
        return self.r.L.ref_level_rows(self.h, l)

    def matrix(self, l, which=0):
        rows, cols = C.c_int64(), C.c_int64()
        rw = self.r.L.ref_level_matrix_shape(self.h, l, which, C.byref(rows), C.byref(cols))
        if rw < 0:
            return None
        c = np.zeros(rows.value * rw, dtype=np.int32); v = np.zeros(rows.value * rw)
        self.r.L.ref_level_matrix(self.h, l, which, c, v)
        return c.reshape(rows.value, rw), v.reshape(rows.value, rw)

    def invdiag(self, l):
        out = np.zeros(self.rows(l))
        self.r.L.ref_level_invdiag(self.h, l, out)
        return out

    def spmv(self, l, x, acc32=False):
        y = np.zeros(self.rows(l))
        self.r.L.ref_level_spmv(self.h, l, np.ascontiguousarray(x, dtype=np.float64), y, int(self.ftz),
                                int(self.fma), int(acc32))
        return y

    def jacobi(self, l, b, u, steps, omega=2.0 / 3.0, acc32=False):
        u = np.array(u, dtype=np.float64)
        self.r.L.ref_level_jacobi(self.h, l, np.ascontiguousarray(b, dtype=np.float64), u, steps, omega,
                                  int(self.ftz), int(self.fma), int(acc32))
        return u

    def defect(self, l, b, u, acc32=False):
        r = np.zeros(self.rows(l))
        self.r.L.ref_level_defect(self.h, l, np.ascontiguousarray(b, dtype=np.float64),
                                  np.ascontiguousarray(u, dtype=np.float64), r, int(self.ftz), int(self.fma),
                                  int(acc32))
        return r

    def restrict(self, l, r_fine, rescale=False):
        out = np.zeros(self.rows(l - 1))
        s = self.r.L.ref_level_restrict(self.h, l, np.ascontiguousarray(r_fine, dtype=np.float64), int(rescale),
                                        out, int(self.ftz), int(self.fma))
        return out, s

    def prolong(self, l, c_coarse, scale=1.0):
        out = np.zeros(self.rows(l))
        self.r.L.ref_level_prolong(self.h, l, np.ascontiguousarray(c_coarse, dtype=np.float64), float(scale), out,
                                   int(self.ftz), int(self.fma))
        return out

    def cg(self, l, b):
        u = np.zeros(self.rows(l))
        it, conv, res = C.c_int(), C.c_int(), C.c_double()
        self.r.L.ref_level_cg(self.h, l, np.ascontiguousarray(b, dtype=np.float64), u, C.byref(it), C.byref(conv),
                              C.byref(res), int(self.ftz), int(self.fma))
        return u, it.value, bool(conv.value), res.value

    def v_cycle(self, b, acc32=False):
        c = np.zeros(self.rows(self.L - 1))
        self.r.L.ref_v_cycle(self.h, np.ascontiguousarray(b, dtype=np.float64), c, int(self.ftz), int(self.fma),
                             int(acc32))
        return c

    def ir_solve(self, rel_tol=1e-10, abs_tol=1e-9, max_it=100, random_guess=False, seed=0, scaling=0, refresh=10,
                 acc32=False, want_u=True):
        N = self.rows(self.L - 1)
        u = np.zeros(N) if want_u else None
        hist = np.zeros(max_it + 2)
        conv, fres, wall, err = C.c_int(), C.c_double(), C.c_double(), C.c_double()
        its = self.r.L.ref_ir_solve(self.h, rel_tol, abs_tol, max_it, int(random_guess), seed, scaling, refresh,
                                    int(self.ftz), int(self.fma), int(acc32),
                                    u.ctypes.data if want_u else None, hist, max_it + 2,
                                    C.byref(conv), C.byref(fres), C.byref(wall), C.byref(err))
        if its == -2:
            raise FloatingPointError("reference ir_solve diverged")
        if its < 0:
            raise RuntimeError("reference ir_solve failed")
        return dict(iterations=its, history=hist[:its + 1].copy(), converged=bool(conv.value),
                    final_residual=fres.value, wall_s=wall.value, err_l2=err.value, u=u)
