"""B200-native mixed-precision iterative refinement + geometric multigrid.

Host-side Python mirror of the reference's solver API (arxiv 2007.07539,
``mpmg``: ``MgHierarchy::build`` multigrid.hpp:104-107, ``v_cycle``
multigrid.hpp:119, ``ir_solve`` ir_solver.hpp:57-60) over the C ABI in
``include/mpmg_gpu.h``; every operation runs in the hand-written sm_100a
kernels of ``libmpmg_b200.so`` (built in-tree by ``build()``).

There is no CPU fallback: constructing a :class:`Hierarchy` without the
compiled library or without a CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libmpmg_b200.so")

FP16, FP32, FP64 = 0, 1, 2
D_MG, H_MG, DSH_MG, HSD_MG = 0, 1, 2, 3
VARIANTS = {"d_mg": D_MG, "h_mg": H_MG, "dsh_mg": DSH_MG, "hsd_mg": HSD_MG}
MPMG_FTZ, MPMG_FMA, MPMG_ACC32 = 1, 2, 4
OP_SPMV, OP_JACOBI, OP_DEFECT, OP_RESTRICT, OP_PROLONG, OP_COARSE_SOLVE = range(6)

ERRORS = {0: "ok", -1: "invalid argument", -2: "non-finite residual", -3: "CUDA error", -4: "binary16 overflow",
          -5: "out of memory", -6: "unsupported"}


class HierarchyBuildError(RuntimeError):
    """binary16 overflow while casting a level (errors.hpp:10-19)."""

    def __init__(self, level, msg):
        super().__init__(msg)
        self.level = level


class DivergedError(RuntimeError):
    """non-finite residual norm in the outer loop (errors.hpp:21-29)."""

    def __init__(self, iteration, msg):
        super().__init__(msg)
        self.iteration = iteration


def build(verbose: bool = False) -> str:
    """Compile libmpmg_b200.so for sm_100a (nvcc; no GPU needed)."""
    for sub in ("csrc", "cpp"):  # the sm_100a library, then the C++ drop-in layer over it
        out = subprocess.run(["make", "-C", os.path.join(HERE, sub), "-j8"], capture_output=True, text=True)
        if verbose:
            print(out.stdout[-4000:], out.stderr[-4000:])
        if out.returncode != 0:
            raise RuntimeError(f"{sub} build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    return LIB_PATH


class Stencil(C.Structure):
    _fields_ = [("dim", C.c_int32), ("nodes", C.c_int32), ("prec", C.c_int32), ("ntaps", C.c_int32),
                ("taps", C.c_double * 27), ("inv_diag", C.c_double)]

    def taps_array(self):
        return np.array(self.taps[: self.ntaps])


class SolverConfig(C.Structure):
    _fields_ = [("dim", C.c_int32), ("k", C.c_int32), ("nodes", C.c_int32), ("levels", C.c_int32),
                ("variant", C.c_int32), ("pre_steps", C.c_int32), ("post_steps", C.c_int32),
                ("omega", C.c_double), ("base_tol", C.c_double), ("base_mode", C.c_int32),
                ("base_max_iterations", C.c_int32), ("policy", C.c_uint32), ("device", C.c_int32)]


class SolveParams(C.Structure):
    _fields_ = [("outer_tolerance", C.c_double), ("max_outer_iterations", C.c_int32),
                ("random_initial_guess", C.c_int32), ("seed", C.c_uint64), ("scaling", C.c_int32),
                ("residual_refresh_interval", C.c_int32), ("use_graph", C.c_int32)]


class SolveReportC(C.Structure):
    _fields_ = [("converged", C.c_int32), ("iterations", C.c_int32), ("final_residual", C.c_double),
                ("device_seconds", C.c_double), ("wall_seconds", C.c_double), ("used_graph", C.c_int32),
                ("graph_error", C.c_int32)]


_lib = None


def lib():
    """Load libmpmg_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run paper_2007_07539_b200.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    d, i, i32, u32, vp, sz = C.c_double, C.c_int, C.c_int32, C.c_uint32, C.c_void_p, C.c_size_t
    dp = C.POINTER(C.c_double)
    L.mpmg_padded_len.restype = sz; L.mpmg_padded_len.argtypes = [i32, i32]
    L.mpmg_interior_len.restype = sz; L.mpmg_interior_len.argtypes = [i32, i32]
    L.mpmg_bytes_per_value.restype = i; L.mpmg_bytes_per_value.argtypes = [i32]
    L.mpmg_last_error.restype = C.c_char_p
    L.mpmg_build_stencil.restype = i; L.mpmg_build_stencil.argtypes = [i32, i32, i32, u32, C.POINTER(Stencil)]
    L.mpmg_round_fp16.restype = d; L.mpmg_round_fp16.argtypes = [d, i32]
    L.mpmg_problem_rhs.restype = i; L.mpmg_problem_rhs.argtypes = [i32, i32, i32, dp]
    L.mpmg_solver_default_config.argtypes = [C.POINTER(SolverConfig)]
    L.mpmg_solve_default_params.argtypes = [C.POINTER(SolveParams)]
    L.mpmg_solver_create.restype = vp
    L.mpmg_solver_create.argtypes = [C.POINTER(SolverConfig), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.mpmg_solver_destroy.argtypes = [vp]
    L.mpmg_solver_levels.restype = i; L.mpmg_solver_levels.argtypes = [vp]
    L.mpmg_solver_level_info.restype = i; L.mpmg_solver_level_info.argtypes = [vp, i, C.POINTER(Stencil)]
    L.mpmg_solver_unknowns.restype = sz; L.mpmg_solver_unknowns.argtypes = [vp]
    L.mpmg_solver_stream.restype = vp; L.mpmg_solver_stream.argtypes = [vp]
    L.mpmg_solver_device_buffers.restype = i
    L.mpmg_solver_device_buffers.argtypes = [vp, C.POINTER(dp), C.POINTER(dp)]
    L.mpmg_solver_solve.restype = i
    L.mpmg_solver_solve.argtypes = [vp, vp, vp, C.POINTER(SolveParams), dp, i32, C.POINTER(SolveReportC)]
    L.mpmg_solver_solve_device.restype = i
    L.mpmg_solver_solve_device.argtypes = [vp, vp, vp, C.POINTER(SolveParams), dp, i32, C.POINTER(SolveReportC)]
    L.mpmg_solver_v_cycle.restype = i; L.mpmg_solver_v_cycle.argtypes = [vp, dp, dp]
    L.mpmg_solver_level_op.restype = i
    L.mpmg_solver_level_op.argtypes = [vp, i, i, dp, dp, dp, i32, d]
    # layer 1: kernel entry points on raw device pointers (padded layout)
    sp = C.POINTER(Stencil)
    L.mpmg_gpu_pack.restype = i; L.mpmg_gpu_pack.argtypes = [i32, i32, i32, vp, vp, vp]
    L.mpmg_gpu_unpack.restype = i; L.mpmg_gpu_unpack.argtypes = [i32, i32, i32, vp, vp, vp]
    L.mpmg_gpu_jacobi.restype = i; L.mpmg_gpu_jacobi.argtypes = [sp, vp, vp, vp, d, u32, vp]
    L.mpmg_gpu_jacobi_from_zero2.restype = i
    L.mpmg_gpu_jacobi_from_zero2.argtypes = [sp, vp, vp, vp, d, u32, vp]
    L.mpmg_gpu_defect.restype = i; L.mpmg_gpu_defect.argtypes = [sp, vp, vp, vp, u32, vp]
    L.mpmg_gpu_spmv.restype = i; L.mpmg_gpu_spmv.argtypes = [sp, vp, vp, u32, vp]
    L.mpmg_gpu_restrict.restype = i
    L.mpmg_gpu_restrict.argtypes = [i32, i32, i32, i32, vp, vp, vp, u32, vp]
    L.mpmg_gpu_prolong_correct.restype = i
    L.mpmg_gpu_prolong_correct.argtypes = [i32, i32, i32, i32, vp, vp, vp, u32, vp]
    L.mpmg_gpu_defect_f64.restype = i; L.mpmg_gpu_defect_f64.argtypes = [sp, vp, vp, vp, vp, vp]
    L.mpmg_gpu_update_rc.restype = i; L.mpmg_gpu_update_rc.argtypes = [sp, vp, i32, vp, vp, vp, vp, u32, vp]
    L.mpmg_gpu_update_r.restype = i
    L.mpmg_gpu_update_r.argtypes = [sp, vp, i32, vp, vp, vp, vp, C.c_int64, vp, vp, u32, vp]
    L.mpmg_gpu_jacobi_slot.restype = i
    L.mpmg_gpu_jacobi_slot.argtypes = [sp, vp, vp, vp, C.c_int64, vp, d, u32, vp]
    L.mpmg_gpu_update_r_partials.restype = i; L.mpmg_gpu_update_r_partials.argtypes = [i32, i32, i32]
    L.mpmg_gpu_fold.restype = i; L.mpmg_gpu_fold.argtypes = [C.c_int64, vp, vp, C.c_int64, i32, vp, vp, u32, vp]
    L.mpmg_gpu_scale_downcast.restype = i
    L.mpmg_gpu_scale_downcast.argtypes = [i32, i32, vp, vp, i32, vp, i32, u32, vp]
    L.mpmg_gpu_partials_len.restype = i; L.mpmg_gpu_partials_len.argtypes = [i32, i32]
    L.mpmg_gpu_norm2_f64.restype = i; L.mpmg_gpu_norm2_f64.argtypes = [i32, i32, vp, vp, vp, vp]
    L.mpmg_gpu_norm_finalize.restype = i; L.mpmg_gpu_norm_finalize.argtypes = [vp, i32, vp, vp]
    i64 = C.c_int64
    L.mpmg_gpu_ell_spmv.restype = i; L.mpmg_gpu_ell_spmv.argtypes = [i64, i32, vp, vp, i32, vp, vp, u32, vp]
    L.mpmg_gpu_axpy.restype = i; L.mpmg_gpu_axpy.argtypes = [i64, i32, d, vp, vp, vp, u32, vp]
    L.mpmg_gpu_vec_multiply.restype = i; L.mpmg_gpu_vec_multiply.argtypes = [i64, i32, vp, vp, vp, u32, vp]
    L.mpmg_gpu_ell_transfer.restype = i
    L.mpmg_gpu_ell_transfer.argtypes = [i64, i32, vp, vp, i32, vp, i32, i32, vp, i32, vp, vp, u32, vp]
    L.mpmg_gpu_ell_update_rc.restype = i
    L.mpmg_gpu_ell_update_rc.argtypes = [i64, i32, vp, vp, vp, i32, vp, vp, vp, u32, vp]
    L.mpmg_gpu_cast.restype = i; L.mpmg_gpu_cast.argtypes = [i64, vp, i32, vp, i32, vp, d, u32, vp]
    L.mpmg_gpu_dot_seq.restype = i; L.mpmg_gpu_dot_seq.argtypes = [i64, vp, i32, vp, i32, vp, i32, vp]
    L.mpmg_dev_count.restype = i
    _lib = L
    return L


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _check(rc, what):
    if rc != 0:
        msg = lib().mpmg_last_error().decode(errors="replace")
        raise RuntimeError(f"{what}: {ERRORS.get(rc, rc)} ({msg})")


def policy_word(ftz=True, fma=True, acc32=False) -> int:
    return (MPMG_FTZ if ftz else 0) | (MPMG_FMA if fma else 0) | (MPMG_ACC32 if acc32 else 0)


def level_stencil(dim, nodes, prec, ftz=True) -> Stencil:
    """Per-level operator of MgHierarchy::build (host setup, no GPU needed)."""
    s = Stencil()
    rc = lib().mpmg_build_stencil(dim, nodes, prec, policy_word(ftz), C.byref(s))
    if rc == -4:
        raise HierarchyBuildError(-1, "binary16 overflow")
    _check(rc, "mpmg_build_stencil")
    return s


def problem_rhs(dim, nodes, k=1) -> np.ndarray:
    """Manufactured load vector (assemble_rhs, mesh_fem.cpp:157-202)."""
    m = nodes - 2
    b = np.zeros(m ** dim)
    _check(lib().mpmg_problem_rhs(dim, nodes, k, _dp(b)), "mpmg_problem_rhs")
    return b


def unknowns(dim, nodes):
    return (nodes - 2) ** dim


@dataclass
class SolveReport:
    """SolveReport (ir_solver.hpp:26-44)."""
    converged: bool
    iterations: int
    residual_history: np.ndarray
    final_residual: float
    device_seconds: float
    wall_seconds: float
    used_graph: bool = False
    graph_error: int = 0


@dataclass
class IrConfig:
    """IrConfig (ir_solver.hpp:12-24)."""
    outer_tolerance: float = 1e-9
    max_outer_iterations: int = 100
    random_initial_guess: bool = False
    seed: int = 0
    scaling: int = 0  # 0 VariantDefault, 1 ForceOn, 2 ForceOff
    residual_refresh_interval: int = 10
    use_graph: bool = True

    def c(self) -> SolveParams:
        p = SolveParams()
        p.outer_tolerance = self.outer_tolerance
        p.max_outer_iterations = self.max_outer_iterations
        p.random_initial_guess = int(self.random_initial_guess)
        p.seed = self.seed
        p.scaling = self.scaling
        p.residual_refresh_interval = self.residual_refresh_interval
        p.use_graph = int(self.use_graph)
        return p


class Hierarchy:
    """Device-resident MgHierarchy (multigrid.hpp:96-140) for the Poisson model
    problem, plus the finest FP64 operator used by ir_solve."""

    def __init__(self, dim, nodes, levels, variant="h_mg", pre=3, post=3, omega=2.0 / 3.0, base_tol=1e-4,
                 base_mode=0, base_max_iterations=0, ftz=True, fma=True, acc32=False, k=1, device=0):
        L = lib()
        cfg = SolverConfig()
        L.mpmg_solver_default_config(C.byref(cfg))
        cfg.dim, cfg.k, cfg.nodes, cfg.levels = dim, k, nodes, levels
        cfg.variant = VARIANTS[variant] if isinstance(variant, str) else variant
        cfg.pre_steps, cfg.post_steps, cfg.omega = pre, post, omega
        cfg.base_tol, cfg.base_mode, cfg.base_max_iterations = base_tol, base_mode, base_max_iterations
        cfg.policy = policy_word(ftz, fma, acc32)
        cfg.device = device
        err, lvl = C.c_int(0), C.c_int(-1)
        self._h = L.mpmg_solver_create(C.byref(cfg), C.byref(err), C.byref(lvl))
        if not self._h:
            if err.value == -4:
                raise HierarchyBuildError(lvl.value, f"binary16 overflow while casting level {lvl.value}")
            _check(err.value or -3, "mpmg_solver_create")
        self.dim, self.nodes, self.levels, self.k = dim, nodes, levels, k
        self.variant = cfg.variant
        self.policy = cfg.policy

    def close(self):
        if getattr(self, "_h", None):
            lib().mpmg_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def level_nodes(self, l):
        return ((self.nodes - 1) >> (self.levels - 1 - l)) + 1

    def level(self, l) -> Stencil:
        s = Stencil()
        _check(lib().mpmg_solver_level_info(self._h, l, C.byref(s)), "level_info")
        return s

    def unknowns(self, l=None):
        n = self.nodes if l is None else self.level_nodes(l)
        return unknowns(self.dim, n)

    def device_buffers(self):
        b, u = C.POINTER(C.c_double)(), C.POINTER(C.c_double)()
        _check(lib().mpmg_solver_device_buffers(self._h, C.byref(b), C.byref(u)), "device_buffers")
        return C.cast(b, C.c_void_p).value, C.cast(u, C.c_void_p).value

    def stream(self):
        return lib().mpmg_solver_stream(self._h)

    # --- per-level kernels on host value-domain arrays (parity tests) -----
    def _op(self, op, l, in0, in1, out_len, steps=0, scale=1.0):
        out = np.zeros(out_len)
        a = None if in0 is None else np.ascontiguousarray(in0, dtype=np.float64)
        b = None if in1 is None else np.ascontiguousarray(in1, dtype=np.float64)
        rc = lib().mpmg_solver_level_op(self._h, op, l, _dp(a), _dp(b), _dp(out), steps, float(scale))
        _check(rc, f"level_op({op})")
        return out

    def spmv(self, l, x):
        return self._op(OP_SPMV, l, x, None, self.unknowns(l))

    def defect(self, l, b, u):
        return self._op(OP_DEFECT, l, u, b, self.unknowns(l))

    def jacobi(self, l, b, u, steps):
        return self._op(OP_JACOBI, l, u, b, self.unknowns(l), steps=steps)

    def restrict(self, l, r_fine, scale=1.0):
        return self._op(OP_RESTRICT, l, r_fine, None, self.unknowns(l - 1), scale=scale)

    def prolong_correct(self, l, c_coarse, u_fine, scale=1.0):
        return self._op(OP_PROLONG, l, c_coarse, u_fine, self.unknowns(l), scale=scale)

    def coarse_solve(self, b):
        return self._op(OP_COARSE_SOLVE, 0, b, None, self.unknowns(0))

    def v_cycle(self, b):
        """MgHierarchy::v_cycle on finest-precision value-domain arrays."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        c = np.zeros_like(b)
        _check(lib().mpmg_solver_v_cycle(self._h, _dp(b), _dp(c)), "v_cycle")
        return c

    # --- ir_solve -----------------------------------------------------------
    def ir_solve(self, b, config: IrConfig = None, u_out=None):
        """ir_solve (ir_solver.cpp:51-127) with host buffers; returns (u, report)."""
        config = config or IrConfig()
        b = np.ascontiguousarray(b, dtype=np.float64)
        u = u_out if u_out is not None else np.zeros_like(b)
        hist = np.zeros(config.max_outer_iterations + 2)
        rep = SolveReportC()
        p = config.c()
        rc = lib().mpmg_solver_solve(self._h, b.ctypes.data, u.ctypes.data, C.byref(p), _dp(hist),
                                     len(hist), C.byref(rep))
        if rc == -2:
            raise DivergedError(rep.iterations, lib().mpmg_last_error().decode())
        _check(rc, "ir_solve")
        return u, SolveReport(bool(rep.converged), rep.iterations, hist[: rep.iterations + 1].copy(),
                              rep.final_residual, rep.device_seconds, rep.wall_seconds, bool(rep.used_graph),
                              rep.graph_error)

    def ir_solve_ptr(self, b_ptr, u_ptr, config: IrConfig = None, device=False):
        """ir_solve on raw pointers (host pinned buffers, or device padded
        vectors when device=True). Returns the SolveReport without history."""
        config = config or IrConfig()
        rep = SolveReportC()
        p = config.c()
        f = lib().mpmg_solver_solve_device if device else lib().mpmg_solver_solve
        rc = f(self._h, b_ptr, u_ptr, C.byref(p), None, 0, C.byref(rep))
        if rc == -2:
            raise DivergedError(rep.iterations, lib().mpmg_last_error().decode())
        _check(rc, "ir_solve")
        return SolveReport(bool(rep.converged), rep.iterations, np.zeros(0), rep.final_residual,
                           rep.device_seconds, rep.wall_seconds, bool(rep.used_graph), rep.graph_error)
