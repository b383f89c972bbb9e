// Host launchers of the streaming stencil kernels. Included by one
// translation unit per storage precision (mpmg_stencil_f16/f32/f64.cu) so the
// policy-templated instantiations compile in parallel.
#pragma once

#include <algorithm>
#include <type_traits>

#include "mpmg_internal.h"
#include "mpmg_stencil.cuh"

namespace mpmg_impl {

using namespace mpmg_dev;

inline __half2 half2_of(double v) {
  const __half h = __double2half(v);
  return __halves2half2(h, h);
}

inline StencilArgs make_args(const mpmg_stencil& A, int zc) {
  StencilArgs a{};
  a.P = pitch(A.nodes);
  a.zc = zc;
  a.plane = A.dim == 3 ? (long long)a.P * a.P : (long long)a.P;
  for (int i = 0; i < 27; ++i) {
    const double t = i < A.ntaps ? A.taps[i] : 0.0;
    a.t16[i] = half2_of(t);
    a.t32[i] = (float)t;
    a.t64[i] = t;
  }
  a.d16 = half2_of(A.inv_diag);
  a.d32 = (float)A.inv_diag;
  a.d64 = A.inv_diag;
  return a;
}

template <int DIM, int LP, int CP, int EP, int OP, bool FTZ, bool FMA>
cudaError_t run_stencil(const StencilArgs& a, cudaStream_t s) {
  using G = Geo<LP, CP>;
  const dim3 block(32, G::BW);
  if constexpr (!OpTraits<OP>::kNorm && DIM == 3) {
    // level ops on pitches the plane kernels do not take (not a power of two:
    // 192, 96, 48, ...): z-chunks short enough for about four CTAs per SM --
    // the fixed 16-plane chunks left 9 to 288 CTAs at these sizes. (The norm
    // ops keep ZC: their partial-sum count is sized from it.)
    const dim3 g0 = stencil_grid(DIM, a.P, G::W, G::RY, G::BW, G::ZC);
    const long long xy = (long long)g0.x * g0.y, target = 4LL * 148;
    int zc = (int)std::min<long long>(G::ZC, std::max<long long>(1, (long long)(a.P - 1) * xy / target));
    StencilArgs b = a;
    b.zc = zc;
    const dim3 grid = stencil_grid(DIM, a.P, G::W, G::RY, G::BW, zc);
    k_stencil<DIM, LP, CP, EP, OP, FTZ, FMA, G::RY, G::BW><<<grid, block, 0, s>>>(b);
    return cudaGetLastError();
  }
  const dim3 grid = stencil_grid(DIM, a.P, G::W, G::RY, G::BW, G::ZC);
  k_stencil<DIM, LP, CP, EP, OP, FTZ, FMA, G::RY, G::BW><<<grid, block, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename F>
inline cudaError_t with_policy(uint32_t policy, F&& f) {
  const bool ftz = policy & MPMG_FTZ, fma = policy & MPMG_FMA;
  if (ftz && fma) return f(std::true_type{}, std::true_type{});
  if (ftz) return f(std::true_type{}, std::false_type{});
  if (fma) return f(std::false_type{}, std::true_type{});
  return f(std::false_type{}, std::false_type{});
}

// level-precision op (SpMV / defect / Jacobi) for storage precision LP
template <int LP>
cudaError_t level_op_impl(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                          uint32_t policy, cudaStream_t s) {
  {  // TMA-staged plane kernels first (3D, pitch a multiple of 32)
    cudaError_t pe = cudaSuccess;
    bool done = false;
    if constexpr (LP == P16) done = plane_level_op_f16(op, A, x, b, out, omega, policy, s, &pe);
    else if constexpr (LP == P32) done = plane_level_op_f32(op, A, x, b, out, omega, policy, s, &pe);
    else done = plane_level_op_f64(op, A, x, b, out, omega, policy, s, &pe);
    if (done) return pe;
  }
  StencilArgs a = make_args(A, Geo<LP, LP>::ZC);
  a.x = x; a.b = b; a.out = out;
  const bool ftz = policy & MPMG_FTZ;
  const double w = round_to(omega, LP, ftz);
  a.w16 = half2_of(w); a.w32 = (float)w; a.w64 = w;
  const bool acc32 = LP == P16 && (policy & MPMG_ACC32);
  return with_policy(policy, [&](auto FT, auto FM) -> cudaError_t {
    constexpr bool kF = decltype(FT)::value, kM = decltype(FM)::value;
    auto go = [&](auto dimc, auto cpc) -> cudaError_t {
      constexpr int D = decltype(dimc)::value, C = decltype(cpc)::value;
      switch (op) {
        case 0: return run_stencil<D, LP, C, LP, OP_SPMV, kF, kM>(a, s);
        case 1: return run_stencil<D, LP, C, LP, OP_DEFECT, kF, kM>(a, s);
        default: return run_stencil<D, LP, C, LP, OP_JACOBI, kF, kM>(a, s);
      }
    };
    using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>;
    using CL = std::integral_constant<int, LP>;
    if constexpr (LP == P16) {
      using C32 = std::integral_constant<int, P32>;
      if (acc32) return A.dim == 3 ? go(I3{}, C32{}) : go(I2{}, C32{});
    }
    return A.dim == 3 ? go(I3{}, CL{}) : go(I2{}, CL{});
  });
}

}  // namespace mpmg_impl
