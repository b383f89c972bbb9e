// TMA-staged plane kernels of the outer FP64 refinement (ir_solver.cpp:
// 51-127): FP64 defect (+ ||r||^2 partials), final residual norm, and the
// fused update u += a c, r -= a A c with c widened from the finest level
// precision (kernels.cpp:300-341).
#include <cuda_runtime.h>

#include <cstdlib>

#include "mpmg_plane_launch.cuh"

namespace mpmg_impl {

int plane_num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// CTA shape of the FP64 outer updates: 4 values per lane, two warps per
// 256-wide row (PlaneCfg V = 10) -- fewer registers per thread and more CTAs
// than 8 values per lane (UPDATE_R 73.6 -> 69.9 us at 257^3; the D_MG solve
// with the fused UPDATE 7.66 -> 7.28 ms)
constexpr int OV = 10;
// DEFECT64 / RESNORM shape (MPMG_DEF64_SHAPE: 0 = 8 values per lane, the
// default -- 84 vs 91 us at 257^3 --, else OV)
static int def_shape() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MPMG_DEF64_SHAPE");
    v = e ? std::atoi(e) : 0;
  }
  return v;
}

bool plane_outer_supported(int dim, int nodes) {
  if (dim != 3) return false;
  return with_pitch(pitch(nodes), [](auto) {});
}

bool plane_defect64(const mpmg_stencil& A64, const double* b, const double* u, double* r, double* partials,
                    bool fma, bool resnorm, cudaStream_t s, const int* gate, cudaError_t* err, const mpmg_slab* slab) {
  if (!plane_outer_supported(A64.dim, A64.nodes) || !aligned16(b) || !aligned16(u) || !aligned16(r)) return false;
  PlaneArgs a = plane_args(A64, slab);
  a.x = u; a.b = b; a.out = r; a.partials = partials; a.gate = gate;
  return with_pitch(a.P, [&](auto pc) {
    constexpr int PP = decltype(pc)::value;
    if (def_shape() == 0) {
      if (resnorm) *err = PlaneLaunch<P64, P64, P64, POP_RESNORM, false, true, PP>::run(a, s);
      else if (fma) *err = PlaneLaunch<P64, P64, P64, POP_DEFECT64, false, true, PP>::run(a, s);
      else *err = PlaneLaunch<P64, P64, P64, POP_DEFECT64, false, false, PP>::run(a, s);
      return;
    }
    if (resnorm) *err = PlaneLaunch<P64, P64, P64, POP_RESNORM, false, true, PP, OV>::run(a, s);  // ir_solver.cpp:38
    else if (fma) *err = PlaneLaunch<P64, P64, P64, POP_DEFECT64, false, true, PP, OV>::run(a, s);
    else *err = PlaneLaunch<P64, P64, P64, POP_DEFECT64, false, false, PP, OV>::run(a, s);
  });
}

bool plane_update_rc(const mpmg_stencil& A64, const void* c, int c_prec, double* r, double* u,
                     const double* alpha_dev, double* partials, bool fma, cudaStream_t s, cudaError_t* err,
                     const mpmg_slab* slab) {
  if (!plane_outer_supported(A64.dim, A64.nodes) || !aligned16(c) || !aligned16(r) || !aligned16(u)) return false;
  PlaneArgs a = plane_args(A64, slab);
  a.x = c; a.r64 = r; a.u64 = u; a.alpha = alpha_dev; a.partials = partials;
  return with_pitch(a.P, [&](auto pc) {
    constexpr int PP = decltype(pc)::value;
    auto go = [&](auto lpc) {
      constexpr int L = decltype(lpc)::value;
      *err = fma ? PlaneLaunch<L, P64, P64, POP_UPDATE, false, true, PP, OV>::run(a, s)
                 : PlaneLaunch<L, P64, P64, POP_UPDATE, false, false, PP, OV>::run(a, s);
    };
    switch (c_prec) {
      case MPMG_FP16: go(std::integral_constant<int, P16>{}); break;
      case MPMG_FP32: go(std::integral_constant<int, P32>{}); break;
      default: go(std::integral_constant<int, P64>{}); break;
    }
  });
}

// r -= a A c (+ ||r||^2 partials) and c -> ring slot *slot (deferred
// u += a c, see mpmg_solver.cu); binary16/32 c only
bool plane_update_r(const mpmg_stencil& A64, const void* c, int c_prec, double* r, const double* alpha_dev,
                    double* partials, void* ring, long long ring_len, const int* slot, double* ring_scale, bool fma,
                    cudaStream_t s, cudaError_t* err, const mpmg_slab* slab) {
  if (c_prec == MPMG_FP64 || !plane_outer_supported(A64.dim, A64.nodes) || !aligned16(c) || !aligned16(r) ||
      !aligned16(ring) || (ring_len * mpmg_bytes_per_value(c_prec)) % 16 != 0)
    return false;
  PlaneArgs a = plane_args(A64, slab);
  a.x = c; a.r64 = r; a.alpha = alpha_dev; a.partials = partials;
  a.ring = ring; a.ring_len = ring_len; a.ring_slot = slot; a.ring_scale = ring_scale;
  return with_pitch(a.P, [&](auto pc) {
    constexpr int PP = decltype(pc)::value;
    auto go = [&](auto lpc) {
      constexpr int L = decltype(lpc)::value;
      *err = fma ? PlaneLaunch<L, P64, P64, POP_UPDATE_R, false, true, PP, OV>::run(a, s)
                 : PlaneLaunch<L, P64, P64, POP_UPDATE_R, false, false, PP, OV>::run(a, s);
    };
    if (c_prec == MPMG_FP16) go(std::integral_constant<int, P16>{});
    else go(std::integral_constant<int, P32>{});
  });
}

int plane_update_r_partials(int dim, int nodes, int lp, int pz) {
  if (!plane_outer_supported(dim, nodes) || lp == MPMG_FP64) return -1;
  int n = -1;
  if (pz <= 0) pz = pitch(nodes);
  with_pitch(pitch(nodes), [&](auto pc) {
    constexpr int PP = decltype(pc)::value;
    n = lp == MPMG_FP16 ? PlaneLaunch<P16, P64, P64, POP_UPDATE_R, false, true, PP, OV>::partials(pz)
                        : PlaneLaunch<P32, P64, P64, POP_UPDATE_R, false, true, PP, OV>::partials(pz);
  });
  return n;
}

// partial sums written per launch: UPDATE with operand precision lp, or the
// FP64 defect / residual norm (lp == FP64); -1 when not covered
// (FMA on/off and DEFECT64/RESNORM instantiations share the shared-memory
// footprint, hence the occupancy and the grid)
int plane_partials(int dim, int nodes, int lp, bool update, int pz) {
  if (!plane_outer_supported(dim, nodes)) return -1;
  int n = -1;
  if (pz <= 0) pz = pitch(nodes);
  with_pitch(pitch(nodes), [&](auto pc) {
    constexpr int PP = decltype(pc)::value;
    if (!update) {
      n = def_shape() == 0 ? PlaneLaunch<P64, P64, P64, POP_DEFECT64, false, true, PP>::partials(pz)
                           : PlaneLaunch<P64, P64, P64, POP_DEFECT64, false, true, PP, OV>::partials(pz);
      return;
    }
    switch (lp) {
      case MPMG_FP16: n = PlaneLaunch<P16, P64, P64, POP_UPDATE, false, true, PP, OV>::partials(pz); break;
      case MPMG_FP32: n = PlaneLaunch<P32, P64, P64, POP_UPDATE, false, true, PP, OV>::partials(pz); break;
      default: n = PlaneLaunch<P64, P64, P64, POP_UPDATE, false, true, PP, OV>::partials(pz); break;
    }
  });
  return n;
}

}  // namespace mpmg_impl
