"""Multi-GPU z-slab decomposition of the mixed-precision IR-MG solve
(BASELINE.json configs[4]).

One process per GPU (``torch.distributed``: NCCL over NVLink for the GPU
path, gloo in the CPU tests). The fine levels of the hierarchy are cut into
z-slabs: rank r owns the global interior planes [max(1, r P_l/R), (r+1) P_l/R)
of level l, stored with one halo plane on each side (include/mpmg_gpu.h,
``mpmg_slab``). Coarse plane k coincides with fine plane 2k, so the slabs of
consecutive levels nest: the restriction needs only the fine lower halo and
the prolongation only the coarse upper halo. Every stencil application is
preceded by a one-plane halo exchange with each neighbour. Levels with fewer
than ``min_planes`` planes per rank (or a pitch below the plane kernels'
minimum) are agglomerated: the restricted right-hand side of the first such
level is gathered on rank 0, which runs the remaining V-cycle (and the CG base
solve) with the single-GPU solver, and the correction is scattered back.

Per-point arithmetic is the same as on one GPU, so a V-cycle is bitwise
independent of the rank count; the outer residual norm is a sum of per-rank
partial sums combined in rank order on every rank (deterministic for a given
rank count; SURVEY §7 hard part 7 covers the last-bit difference to the
reference's sequential order).

The kernels are reached through an ``ops`` object: :class:`CudaOps` calls the
sm_100a C ABI; the CPU tests substitute a NumPy model of the same slab
operations to check the decomposition, halo and agglomeration logic with
world_size 2 on gloo.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Slab:
    nz: int
    z_lo: int
    halo_lo: int
    halo_hi: int


class SlabPlan:
    """Which levels are distributed and how their planes map to ranks."""

    def __init__(self, nodes, levels, world, min_planes=4, min_pitch=32, max_pitch=1024):
        self.nodes, self.levels, self.world = nodes, levels, world
        self.P = [((nodes - 1) >> (levels - 1 - l)) for l in range(levels)]
        self.dist = [False] * levels
        for l in range(levels - 1, -1, -1):
            P = self.P[l]
            if not (min_pitch <= P <= max_pitch and P % world == 0 and P // world >= min_planes):
                break
            self.dist[l] = True
        if not self.dist[-1]:
            raise ValueError(f"finest pitch {self.P[-1]} cannot be split over {world} ranks")
        # the agglomeration level: the finest level solved on rank 0
        self.agg = max(l for l in range(levels) if not self.dist[l]) if not all(self.dist) else -1
        if self.agg < 0:
            raise ValueError("no coarse level left for the agglomerated solve")
        # the agglomeration level is restricted into slab-wise too: its planes
        # must split evenly, or coarse planes would be left out (and the last
        # rank's prolongation would read past its slab)
        if self.P[self.agg] % world != 0:
            raise ValueError(f"agglomeration pitch {self.P[self.agg]} is not divisible by {world} ranks")
        try:
            self.check()
        except AssertionError as ex:
            raise ValueError(f"invalid slab decomposition: {ex}") from None

    def nodes_at(self, l):
        return self.P[l] + 1

    def slab(self, l, rank):
        """owned planes of level l on `rank` (also defined for the
        agglomeration level: the planes a rank restricts into)."""
        P = self.P[l]
        chunk = P // self.world
        lo = max(1, rank * chunk)
        hi = (rank + 1) * chunk
        return Slab(hi - lo, lo, int(rank > 0), int(rank < self.world - 1))

    def slab_len(self, l, rank):
        P = self.P[l]
        return (self.slab(l, rank).nz + 2) * P * P + P + 1

    def check(self):
        """invariants the kernels rely on (tests)"""
        for l in range(self.agg, self.levels):
            cover = []
            for r in range(self.world):
                s = self.slab(l, r)
                assert s.nz >= (1 if l > self.agg else 0)  # an agglomeration slab may be empty
                cover.extend(range(s.z_lo, s.z_lo + s.nz))
            assert cover == list(range(1, self.P[l])), (l, cover[:5])
            if l > self.agg:
                for r in range(self.world):
                    f, c = self.slab(l, r), self.slab(l - 1, r)
                    # restriction: coarse k reads fine 2k-1..2k+1 within [lo_f - 1, hi_f]
                    assert 2 * c.z_lo - 1 >= f.z_lo - 1 and 2 * (c.z_lo + c.nz - 1) + 1 <= f.z_lo + f.nz
                    # prolongation: fine F reads coarse F//2 .. (F+1)//2 within [lo_c - 1, hi_c]
                    assert f.z_lo // 2 >= c.z_lo - 1 and (f.z_lo + f.nz) // 2 <= c.z_lo + c.nz
        return True


# ---------------------------------------------------------------------------
# communication
# ---------------------------------------------------------------------------
class Comm:
    """Halo exchange, gathers and scalar sums over torch.distributed. With
    gloo, device tensors are staged through host memory."""

    def __init__(self, dist_mod, rank, world, device_tensors):
        self.d, self.rank, self.world = dist_mod, rank, world
        self.stage = device_tensors and dist_mod.get_backend() == "gloo"

    def _ops(self, pairs):
        """pairs: list of ('send'|'recv', tensor, peer); runs them as one batch"""
        if not pairs:
            return
        if self.stage:
            hosts, reqs = [], []
            for kind, t, peer in pairs:
                h = t.detach().cpu() if kind == "send" else t.new_empty(t.shape, device="cpu")
                hosts.append((kind, t, h))
                reqs.append(self.d.isend(h, peer) if kind == "send" else self.d.irecv(h, peer))
            for q in reqs:
                q.wait()
            for kind, t, h in hosts:
                if kind == "recv":
                    t.copy_(h)
            return
        P2P = self.d.P2POp
        ops = [P2P(self.d.isend if kind == "send" else self.d.irecv, t, peer) for kind, t, peer in pairs]
        for q in self.d.batch_isend_irecv(ops):
            q.wait()

    def exchange(self, t, plane, nz, which="both"):
        """fill halo planes 0 / nz+1 of slab array t from the neighbours"""
        pl = lambda q: t[q * plane:(q + 1) * plane]  # noqa: E731
        pairs = []
        lo, hi = self.rank - 1, self.rank + 1
        if which in ("both", "lo"):  # my lower halo <- lower rank's top plane
            if lo >= 0:
                pairs.append(("recv", pl(0), lo))
            if hi < self.world:
                pairs.append(("send", pl(nz), hi))
        if which in ("both", "hi"):  # my upper halo <- upper rank's first plane
            if hi < self.world:
                pairs.append(("recv", pl(nz + 1), hi))
            if lo >= 0:
                pairs.append(("send", pl(1), lo))
        self._ops(pairs)

    def gather_planes(self, local, s, full, plane):
        """owned planes of every rank's slab -> rank 0's whole-level array"""
        if self.rank == 0:
            full[s.z_lo * plane:(s.z_lo + s.nz) * plane].copy_(local[plane:(1 + s.nz) * plane])
            pairs = []
            for r in range(1, self.world):
                sr = self.slabs[r]
                pairs.append(("recv", full[sr.z_lo * plane:(sr.z_lo + sr.nz) * plane], r))
            self._ops(pairs)
        else:
            self._ops([("send", local[plane:(1 + s.nz) * plane], 0)])

    def scatter_planes(self, full, s, local, plane):
        """rank 0's whole-level array -> every rank's owned planes + both halos"""
        if self.rank == 0:
            local[:(s.nz + 2) * plane].copy_(full[(s.z_lo - 1) * plane:(s.z_lo + s.nz + 1) * plane])
            pairs = []
            for r in range(1, self.world):
                sr = self.slabs[r]
                pairs.append(("send", full[(sr.z_lo - 1) * plane:(sr.z_lo + sr.nz + 1) * plane], r))
            self._ops(pairs)
        else:
            self._ops([("recv", local[:(s.nz + 2) * plane], 0)])

    def sum_scalar(self, x, like):
        """sum of one double per rank, in rank order (deterministic)"""
        if self.world == 1:
            return float(x)
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64, device=like.device)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        self.d.all_gather(out, t)
        s = 0.0
        for v in out:
            s += float(v.item())
        return s


# ---------------------------------------------------------------------------
# kernels: the sm_100a C ABI on z-slabs
# ---------------------------------------------------------------------------
class SlabC(C.Structure):
    _fields_ = [("nz", C.c_int32), ("z_lo", C.c_int32), ("halo_lo", C.c_int32), ("halo_hi", C.c_int32)]


class CudaOps:
    """Slab operations through include/mpmg_gpu.h (device pointers of torch
    tensors, on torch's current stream)."""

    def __init__(self, plan, variant, ftz, pre=3, post=3, omega=2.0 / 3.0, device=None):
        import torch

        from . import FP16, FP32, FP64, lib, level_stencil, policy_word
        self.torch, self.L, self.plan = torch, lib(), plan
        self.FP16, self.FP32, self.FP64 = FP16, FP32, FP64
        L = self.L
        vp, i32, u32, d = C.c_void_p, C.c_int32, C.c_uint32, C.c_double
        sp = C.POINTER(SlabC)
        from . import Stencil
        st = C.POINTER(Stencil)
        for name, args in (("mpmg_gpu_slab_jacobi", [st, sp, vp, vp, vp, d, u32, vp]),
                           ("mpmg_gpu_slab_defect", [st, sp, vp, vp, vp, u32, vp]),
                           ("mpmg_gpu_slab_restrict", [i32, sp, sp, i32, i32, vp, vp, u32, vp]),
                           ("mpmg_gpu_slab_prolong_correct", [i32, sp, sp, i32, i32, vp, vp, u32, vp]),
                           ("mpmg_gpu_slab_defect_f64", [st, sp, vp, vp, vp, vp, i32, vp]),
                           ("mpmg_gpu_slab_update_rc", [st, sp, vp, i32, vp, vp, vp, vp, u32, vp]),
                           ("mpmg_gpu_slab_scale_downcast", [i32, sp, vp, vp, i32, vp, i32, u32, vp]),
                           ("mpmg_gpu_slab_partials_len", [i32, sp, i32, i32]),
                           ("mpmg_gpu_partials_sum", [vp, i32, vp, vp])):
            f = getattr(L, name)
            f.restype = C.c_int
            f.argtypes = args
        self.variant, self.ftz = variant, ftz
        self.pre, self.post, self.omega = pre, post, omega
        self.policy = policy_word(ftz, True, False)
        self.prec = [_variant_prec(variant, l, plan.levels) for l in range(plan.levels)]
        self.A = [level_stencil(3, plan.nodes_at(l), self.prec[l], ftz) for l in range(plan.levels)]
        self.A64 = level_stencil(3, plan.nodes, FP64, ftz)
        self.dt = {FP16: torch.float16, FP32: torch.float32, FP64: torch.float64}

    def _s(self, s):
        return C.byref(SlabC(s.nz, s.z_lo, s.halo_lo, s.halo_hi))

    def _stream(self):
        # torch's default stream is the legacy NULL stream (handle 0); pass
        # cudaStreamLegacy explicitly -- NULL means "the solver's own stream"
        # to the mpmg_solver_* entry points
        s = self.torch.cuda.current_stream().cuda_stream
        return s if s else 1

    def _ok(self, rc, what):
        if rc != 0:
            raise RuntimeError(f"{what}: code {rc} ({self.L.mpmg_last_error().decode()})")

    def zeros(self, n, prec):
        return self.torch.zeros(n, dtype=self.dt[prec], device="cuda")

    def jacobi(self, l, s, b, u_in, u_out):
        self._ok(self.L.mpmg_gpu_slab_jacobi(C.byref(self.A[l]), self._s(s), b.data_ptr(),
                                             None if u_in is None else u_in.data_ptr(), u_out.data_ptr(),
                                             self.omega, self.policy, self._stream()), "slab_jacobi")

    def defect(self, l, s, b, u, r):
        self._ok(self.L.mpmg_gpu_slab_defect(C.byref(self.A[l]), self._s(s), b.data_ptr(), u.data_ptr(),
                                             r.data_ptr(), self.policy, self._stream()), "slab_defect")

    def restrict(self, l, sf, sc, r_f, b_c):
        self._ok(self.L.mpmg_gpu_slab_restrict(self.plan.nodes_at(l), self._s(sf), self._s(sc), self.prec[l],
                                               self.prec[l - 1], r_f.data_ptr(), b_c.data_ptr(), self.policy,
                                               self._stream()), "slab_restrict")

    def prolong(self, l, sf, sc, c_c, u_f):
        self._ok(self.L.mpmg_gpu_slab_prolong_correct(self.plan.nodes_at(l), self._s(sf), self._s(sc),
                                                      self.prec[l], self.prec[l - 1], c_c.data_ptr(), u_f.data_ptr(),
                                                      self.policy, self._stream()), "slab_prolong")

    def partials(self, s, update):
        n = self.L.mpmg_gpu_slab_partials_len(self.plan.nodes, self._s(s), self.prec[-1], int(update))
        return self.torch.zeros(max(n, 1), dtype=self.torch.float64, device="cuda"), n

    def local_sumsq(self, part, n):
        out = self.torch.zeros(1, dtype=self.torch.float64, device="cuda")
        self._ok(self.L.mpmg_gpu_partials_sum(part.data_ptr(), n, out.data_ptr(), self._stream()), "partials_sum")
        return float(out.item())

    def defect64(self, s, b, u, r, part, resnorm=False):
        self._ok(self.L.mpmg_gpu_slab_defect_f64(C.byref(self.A64), self._s(s), b.data_ptr(), u.data_ptr(),
                                                 None if r is None else r.data_ptr(), part.data_ptr(), int(resnorm),
                                                 self._stream()), "slab_defect_f64")

    def update(self, s, c, r, u, alpha_dev, part):
        self._ok(self.L.mpmg_gpu_slab_update_rc(C.byref(self.A64), self._s(s), c.data_ptr(), self.prec[-1],
                                                r.data_ptr(), u.data_ptr(), alpha_dev.data_ptr(), part.data_ptr(),
                                                self.policy, self._stream()), "slab_update_rc")

    def downcast(self, s, r, out, alpha_dev, scale_enabled):
        self._ok(self.L.mpmg_gpu_slab_scale_downcast(self.plan.nodes, self._s(s), r.data_ptr(), out.data_ptr(),
                                                     self.prec[-1], alpha_dev.data_ptr(), int(scale_enabled),
                                                     self.policy, self._stream()), "slab_downcast")

    def coarse_solver(self):
        """the single-GPU solver for levels 0..agg (rank 0)"""
        from . import Hierarchy
        a = self.plan.agg
        self._coarse = Hierarchy(3, self.plan.nodes_at(a), a + 1, self.variant, pre=self.pre, post=self.post,
                                 ftz=self.ftz)
        L = self.L
        L.mpmg_solver_v_cycle_device.restype = C.c_int
        L.mpmg_solver_v_cycle_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        return self._coarse

    def coarse_cycle(self, b_full, c_full):
        self._ok(self.L.mpmg_solver_v_cycle_device(self._coarse.handle, b_full.data_ptr(), c_full.data_ptr(),
                                                   self._stream()), "coarse v_cycle")


def _variant_prec(variant, l, levels):
    """VariantConfig::make (multigrid.cpp:54-77); level 0 = coarsest"""
    v = variant if isinstance(variant, str) else {0: "d_mg", 1: "h_mg", 2: "dsh_mg", 3: "hsd_mg"}[variant]
    if v == "d_mg":
        return 2
    if v == "h_mg":
        return 0
    if v == "hsd_mg":
        return 2 if l <= 1 else (1 if l == 2 else 0)
    return 0 if l <= 1 else (1 if l == 2 else 2)  # dsh_mg


# ---------------------------------------------------------------------------
# the distributed solver
# ---------------------------------------------------------------------------
class SlabSolver:
    """ir_solve (ir_solver.cpp:51-127) over z-slabs of the finest grid.
    Supports u0 = 0, variants without DSH restriction rescaling."""

    def __init__(self, plan, ops, comm):
        self.plan, self.ops, self.comm = plan, ops, comm
        if getattr(ops, "variant", "h_mg") in ("dsh_mg", 2):
            raise NotImplementedError("DSH restriction rescaling is not distributed")
        r, W = comm.rank, comm.world
        comm.slabs = [plan.slab(plan.agg, q) for q in range(W)]
        self.lv = {}
        for l in range(plan.agg, plan.levels):
            s = plan.slab(l, r)
            n = plan.slab_len(l, r)
            p = ops.prec[l]
            self.lv[l] = dict(s=s, u=ops.zeros(n, p), u2=ops.zeros(n, p), b=ops.zeros(n, p), r=ops.zeros(n, p),
                              plane=plan.P[l] ** 2)
        F = plan.levels - 1
        sF = plan.slab(F, r)
        n = plan.slab_len(F, r)
        self.u, self.r, self.b = ops.zeros(n, 2), ops.zeros(n, 2), ops.zeros(n, 2)
        self.partU, self.nU = ops.partials(sF, True)
        self.partD, self.nD = ops.partials(sF, False)
        a = plan.agg
        if r == 0:
            Pa = plan.P[a]
            full = Pa ** 3 + Pa ** 2 + Pa + 1
            self.bfull, self.cfull = ops.zeros(full, ops.prec[a]), ops.zeros(full, ops.prec[a])
            ops.coarse_solver()

    # V-cycle on the distributed levels; the rhs of level l is lv[l]['b'];
    # returns the slab array holding the correction (halos exchanged)
    def cycle(self, l):
        P, ops, comm = self.plan, self.ops, self.comm
        X = self.lv[l]
        s, plane = X["s"], X["plane"]
        if l == P.agg:  # gather -> rank 0 solves levels 0..agg -> scatter
            comm.gather_planes(X["b"], s, self.bfull if comm.rank == 0 else None, plane)
            if comm.rank == 0:
                ops.coarse_cycle(self.bfull, self.cfull)
            comm.scatter_planes(self.cfull if comm.rank == 0 else None, s, X["u"], plane)
            return X["u"]
        cur, other = X["u"], X["u2"]
        if ops.pre > 0:
            ops.jacobi(l, s, X["b"], None, cur)
            comm.exchange(cur, plane, s.nz)
            for _ in range(ops.pre - 1):
                ops.jacobi(l, s, X["b"], cur, other)
                comm.exchange(other, plane, s.nz)
                cur, other = other, cur
        else:
            cur.zero_()
        ops.defect(l, s, X["b"], cur, X["r"])
        comm.exchange(X["r"], plane, s.nz, "lo")
        C_ = self.lv[l - 1]
        ops.restrict(l, s, C_["s"], X["r"], C_["b"])
        cc = self.cycle(l - 1)
        if l - 1 != P.agg:
            comm.exchange(cc, C_["plane"], C_["s"].nz, "hi")
        ops.prolong(l, s, C_["s"], cc, cur)
        comm.exchange(cur, plane, s.nz)
        for _ in range(ops.post):
            ops.jacobi(l, s, X["b"], cur, other)
            comm.exchange(other, plane, s.nz)
            cur, other = other, cur
        return cur

    def solve(self, b_slab, tol, max_it=100, refresh=10, scaling=0):
        """b_slab: this rank's FP64 slab of the rhs (owned planes filled).
        Returns (u slab, iterations, history, converged, final residual)."""
        import torch
        P, ops, comm = self.plan, self.ops, self.comm
        F = P.levels - 1
        s = P.slab(F, comm.rank)
        plane = P.P[F] ** 2
        self.b.copy_(b_slab)
        self.u.zero_()
        scale_enabled = scaling == 1 or (scaling == 0 and getattr(ops, "variant", "h_mg") not in ("d_mg", 0))
        alpha_dev = torch.zeros(1, dtype=torch.float64, device=self.u.device)
        ops.defect64(s, self.b, self.u, self.r, self.partD)
        alpha = math.sqrt(comm.sum_scalar(ops.local_sumsq(self.partD, self.nD), self.u))
        hist, its, conv = [alpha], 0, False
        rlow = self.lv[F]["b"]
        while True:
            if not math.isfinite(alpha):
                raise FloatingPointError(f"non-finite residual norm at iteration {its}")
            if alpha < tol:
                conv = True
                break
            if its >= max_it:
                break
            sc = alpha if (scale_enabled and alpha > 0) else 1.0
            alpha_dev.fill_(sc)
            ops.downcast(s, self.r, rlow, alpha_dev, 1)
            c = self.cycle(F)
            ops.update(s, c, self.r, self.u, alpha_dev, self.partU)
            its += 1
            if refresh > 0 and its % refresh == 0:
                comm.exchange(self.u, plane, s.nz)
                ops.defect64(s, self.b, self.u, self.r, self.partD)
                ss = ops.local_sumsq(self.partD, self.nD)
            else:
                ss = ops.local_sumsq(self.partU, self.nU)
            alpha = math.sqrt(comm.sum_scalar(ss, self.u))
            hist.append(alpha)
        comm.exchange(self.u, plane, s.nz)
        ops.defect64(s, self.b, self.u, None, self.partD, resnorm=True)
        final = math.sqrt(comm.sum_scalar(ops.local_sumsq(self.partD, self.nD), self.u))
        return self.u, its, hist, conv, final


def slab_of_compact(b_compact, plan, rank, torch_mod, device):
    """this rank's FP64 slab of a compact (reference-ordered) 3D vector"""
    F = plan.levels - 1
    s = plan.slab(F, rank)
    P = plan.P[F]
    m = P - 1
    out = torch_mod.zeros(plan.slab_len(F, rank), dtype=torch_mod.float64)
    v = out[: (s.nz + 2) * P * P].view(s.nz + 2, P, P)
    src = torch_mod.from_numpy(np.asarray(b_compact).reshape(m, m, m))
    v[1:1 + s.nz, 1:P, 1:P] = src[s.z_lo - 1:s.z_lo - 1 + s.nz]
    return out.to(device)


def compact_of_slabs(slabs, plan, torch_mod=None):
    """gather helper for tests: owned planes of every rank (numpy arrays or
    tensors) -> compact order"""
    F = plan.levels - 1
    P = plan.P[F]
    m = P - 1
    out = np.zeros((m, m, m))
    for rank, t in enumerate(slabs):
        s = plan.slab(F, rank)
        a = t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)
        v = a[: (s.nz + 2) * P * P].reshape(s.nz + 2, P, P)
        out[s.z_lo - 1:s.z_lo - 1 + s.nz] = v[1:1 + s.nz, 1:P, 1:P]
    return out.reshape(-1)


# ---------------------------------------------------------------------------
# the C++ multi-GPU solver (csrc/mpmg_dist.cu, include/mpmg_gpu.h mpmg_dist_*)
# ---------------------------------------------------------------------------
class DistSolver:
    """One rank of the C++ z-slab solver: peer-memory halos / gather / norms,
    one CUDA graph per solve (device WHILE loop). `exchange(blob) -> list of
    all ranks' blobs` moves the connection blobs (torch.distributed
    all_gather_object across processes; a plain list within one process)."""

    def __init__(self, nodes, levels, variant, rank, world, ftz=False, pre=3, post=3, device=0, min_planes=4):
        from . import SolverConfig, VARIANTS, lib, policy_word
        L = lib()
        vp, i32, sz = C.c_void_p, C.c_int32, C.c_size_t
        L.mpmg_dist_create.restype = vp
        L.mpmg_dist_create.argtypes = [C.POINTER(SolverConfig), i32, i32, i32, vp, sz, C.POINTER(sz),
                                       C.POINTER(C.c_int)]
        L.mpmg_dist_connect.restype = C.c_int; L.mpmg_dist_connect.argtypes = [vp, vp, sz]
        L.mpmg_dist_destroy.argtypes = [vp]
        L.mpmg_dist_info.restype = C.c_int
        L.mpmg_dist_info.argtypes = [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32), C.POINTER(sz)]
        L.mpmg_dist_buffers.restype = C.c_int
        L.mpmg_dist_buffers.argtypes = [vp, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
        L.mpmg_dist_stream.restype = vp; L.mpmg_dist_stream.argtypes = [vp]
        L.mpmg_dist_exchange_stats.restype = C.c_int
        L.mpmg_dist_exchange_stats.argtypes = [vp, C.POINTER(i32), C.POINTER(i32)]
        L.mpmg_dist_graph_kernels.restype = C.c_int
        L.mpmg_dist_graph_kernels.argtypes = [vp, C.POINTER(i32), C.POINTER(i32)]
        from . import SolveParams, SolveReportC
        L.mpmg_dist_prepare.restype = C.c_int
        L.mpmg_dist_prepare.argtypes = [vp, C.POINTER(SolveParams)]
        L.mpmg_dist_solve_device.restype = C.c_int
        L.mpmg_dist_solve_device.argtypes = [vp, C.POINTER(SolveParams), C.POINTER(C.c_double), i32,
                                             C.POINTER(SolveReportC)]
        self.L, self.nodes, self.levels, self.rank, self.world = L, nodes, levels, rank, world
        cfg = SolverConfig()
        L.mpmg_solver_default_config(C.byref(cfg))
        cfg.dim, cfg.nodes, cfg.levels = 3, nodes, levels
        cfg.variant = VARIANTS[variant] if isinstance(variant, str) else variant
        cfg.pre_steps, cfg.post_steps = pre, post
        cfg.policy = policy_word(ftz, True, False)
        cfg.device = device
        blob = (C.c_ubyte * 256)()
        n = C.c_size_t(0)
        err = C.c_int(0)
        self.h = L.mpmg_dist_create(C.byref(cfg), rank, world, min_planes, blob, 256, C.byref(n), C.byref(err))
        if not self.h:
            raise RuntimeError(f"mpmg_dist_create: code {err.value} ({L.mpmg_last_error().decode()})")
        self.blob = bytes(blob[: n.value])
        agg, zlo, nz, slen = C.c_int32(), C.c_int32(), C.c_int32(), C.c_size_t()
        L.mpmg_dist_info(self.h, C.byref(agg), C.byref(zlo), C.byref(nz), C.byref(slen))
        self.agg, self.z_lo, self.nz, self.slab_len = agg.value, zlo.value, nz.value, slen.value

    def connect(self, blobs):
        allb = b"".join(blobs)
        buf = (C.c_ubyte * len(allb)).from_buffer_copy(allb)
        rc = self.L.mpmg_dist_connect(self.h, buf, len(self.blob))
        if rc != 0:
            raise RuntimeError(f"mpmg_dist_connect: code {rc} ({self.L.mpmg_last_error().decode()})")

    def exchange_stats(self):
        """(fused, copied): halo exchanges in the last captured solve graph done
        by the producing kernel's peer stores / by a separate peer copy"""
        f, c = C.c_int32(), C.c_int32()
        self.L.mpmg_dist_exchange_stats(self.h, C.byref(f), C.byref(c))
        return f.value, c.value

    def graph_kernels(self):
        """(outer, per_iteration): kernel nodes of the captured solve graph;
        a solve of k iterations launches outer + k * per_iteration kernels"""
        o, b = C.c_int32(), C.c_int32()
        rc = self.L.mpmg_dist_graph_kernels(self.h, C.byref(o), C.byref(b))
        return (o.value, b.value) if rc == 0 else None

    def buffers(self):
        b, u = C.c_void_p(), C.c_void_p()
        self.L.mpmg_dist_buffers(self.h, C.byref(b), C.byref(u))
        return b.value, u.value

    def _params(self, tol, max_it, refresh, scaling):
        from . import IrConfig
        return IrConfig(outer_tolerance=tol, max_outer_iterations=max_it, residual_refresh_interval=refresh,
                        scaling=scaling).c()

    def prepare(self, tol, max_it=100, refresh=10, scaling=0):
        p = self._params(tol, max_it, refresh, scaling)
        rc = self.L.mpmg_dist_prepare(self.h, C.byref(p))
        if rc != 0:
            raise RuntimeError(f"mpmg_dist_prepare: code {rc} ({self.L.mpmg_last_error().decode()})")

    def solve(self, tol, max_it=100, refresh=10, scaling=0):
        """every rank calls it (same arguments); returns (report, history)"""
        from . import SolveReportC
        p = self._params(tol, max_it, refresh, scaling)
        hist = (C.c_double * (max_it + 2))()
        rep = SolveReportC()
        rc = self.L.mpmg_dist_solve_device(self.h, C.byref(p), hist, max_it + 2, C.byref(rep))
        if rc != 0:
            raise RuntimeError(f"mpmg_dist_solve_device: code {rc} ({self.L.mpmg_last_error().decode()})")
        return rep, np.array(hist[: rep.iterations + 1])

    def close(self):
        if getattr(self, "h", None):
            self.L.mpmg_dist_destroy(self.h)
            self.h = None
