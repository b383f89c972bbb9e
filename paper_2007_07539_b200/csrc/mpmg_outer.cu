// Outer FP64 refinement kernels (ir_solver.cpp:51-127): defect, fused
// update of u and r with the widened low-precision correction, and the final
// from-scratch residual norm. Instantiations of the streaming stencil.
#include "mpmg_stencil_launch.cuh"

namespace mpmg_impl {

cudaError_t launch_defect64(const mpmg_stencil& A64, const double* b, const double* u, double* r, double* partials,
                            bool fma, bool resnorm, cudaStream_t s, const int* gate) {
  cudaError_t pe = cudaSuccess;
  if (plane_defect64(A64, b, u, r, partials, fma, resnorm, s, gate, &pe)) return pe;
  StencilArgs a = make_args(A64, Geo<P64, P64>::ZC);
  a.x = u; a.b = b; a.out = r; a.partials = partials; a.gate = gate;
  using I2 = std::integral_constant<int, 2>;
  using I3 = std::integral_constant<int, 3>;
  auto go = [&](auto dimc) -> cudaError_t {
    constexpr int D = decltype(dimc)::value;
    if (resnorm) return run_stencil<D, P64, P64, P64, OP_RESNORM, false, true>(a, s);  // ir_solver.cpp:38 std::fma
    if (fma) return run_stencil<D, P64, P64, P64, OP_DEFECT64, false, true>(a, s);
    return run_stencil<D, P64, P64, P64, OP_DEFECT64, false, false>(a, s);
  };
  return A64.dim == 3 ? go(I3{}) : go(I2{});
}

cudaError_t launch_update_rc(const mpmg_stencil& A64, const void* c, int c_prec, double* r, double* u,
                             const double* alpha_dev, double* partials, bool fma, cudaStream_t s) {
  cudaError_t pe = cudaSuccess;
  if (plane_update_rc(A64, c, c_prec, r, u, alpha_dev, partials, fma, s, &pe)) return pe;
  using I2 = std::integral_constant<int, 2>;
  using I3 = std::integral_constant<int, 3>;
  auto go = [&](auto dimc, auto lpc, auto fmc) -> cudaError_t {
    constexpr int D = decltype(dimc)::value, L = decltype(lpc)::value;
    constexpr bool M = decltype(fmc)::value;
    StencilArgs a = make_args(A64, Geo<L, P64>::ZC);
    a.x = c; a.r64 = r; a.u64 = u; a.alpha = alpha_dev; a.partials = partials;
    return run_stencil<D, L, P64, P64, OP_UPDATE, false, M>(a, s);
  };
  auto by_prec = [&](auto dimc, auto fmc) -> cudaError_t {
    switch (c_prec) {
      case MPMG_FP16: return go(dimc, std::integral_constant<int, P16>{}, fmc);
      case MPMG_FP32: return go(dimc, std::integral_constant<int, P32>{}, fmc);
      default: return go(dimc, std::integral_constant<int, P64>{}, fmc);
    }
  };
  auto by_fma = [&](auto dimc) -> cudaError_t {
    return fma ? by_prec(dimc, std::true_type{}) : by_prec(dimc, std::false_type{});
  };
  return A64.dim == 3 ? by_fma(I3{}) : by_fma(I2{});
}

// r -= a A c (+ partials) and c into ring slot *slot: the streaming form of
// plane_update_r for shapes the plane kernels do not take (2D levels, pitches
// that are not a power of two); binary16/32 c only
bool stencil_update_r(const mpmg_stencil& A64, const void* c, int c_prec, double* r, const double* alpha_dev,
                      double* partials, void* ring, long long ring_len, const int* slot, double* ring_scale, bool fma,
                      cudaStream_t s, cudaError_t* err) {
  if (c_prec == MPMG_FP64) return false;
  using I2 = std::integral_constant<int, 2>;
  using I3 = std::integral_constant<int, 3>;
  auto go = [&](auto dimc, auto lpc, auto fmc) -> cudaError_t {
    constexpr int D = decltype(dimc)::value, L = decltype(lpc)::value;
    constexpr bool M = decltype(fmc)::value;
    StencilArgs a = make_args(A64, Geo<L, P64>::ZC);
    a.x = c; a.r64 = r; a.alpha = alpha_dev; a.partials = partials;
    a.ring = ring; a.ring_len = ring_len; a.ring_slot = slot; a.ring_scale = ring_scale;
    return run_stencil<D, L, P64, P64, OP_UPDATE_R, false, M>(a, s);
  };
  auto by_prec = [&](auto dimc, auto fmc) -> cudaError_t {
    return c_prec == MPMG_FP16 ? go(dimc, std::integral_constant<int, P16>{}, fmc)
                               : go(dimc, std::integral_constant<int, P32>{}, fmc);
  };
  auto by_fma = [&](auto dimc) -> cudaError_t {
    return fma ? by_prec(dimc, std::true_type{}) : by_prec(dimc, std::false_type{});
  };
  *err = A64.dim == 3 ? by_fma(I3{}) : by_fma(I2{});
  return true;
}

// partial sums written by the FP64-epilogue kernels (update: stencil operand
// in precision lp; defect64/resnorm: lp == FP64)
int stencil_partials(int dim, int nodes, int lp, bool update) {
  const int pp = plane_partials(dim, nodes, lp, update);
  if (pp > 0) return pp;
  const int P = pitch(nodes);
  dim3 g;
  if (!update) lp = MPMG_FP64;
  switch (lp) {
    case MPMG_FP16: { using G = Geo<P16, P64>; g = stencil_grid(dim, P, G::W, G::RY, G::BW, G::ZC); break; }
    case MPMG_FP32: { using G = Geo<P32, P64>; g = stencil_grid(dim, P, G::W, G::RY, G::BW, G::ZC); break; }
    default: { using G = Geo<P64, P64>; g = stencil_grid(dim, P, G::W, G::RY, G::BW, G::ZC); break; }
  }
  return (int)(g.x * g.y * g.z);
}

bool stencil_supported(int dim, int nodes, int prec) {
  const int P = pitch(nodes);
  const int W = prec == MPMG_FP64 ? 2 : 4;
  (void)dim;
  return P >= 16 && P % W == 0;
}

// two Jacobi steps from u = 0 (steps 1+2 of the pre-smoother, multigrid.cpp:
// 376-377): one fused plane-kernel pass over b when covered, else the
// pointwise first step into `tmp` followed by a streaming step
cudaError_t launch_jacobi_zero2(const mpmg_stencil& A, const void* b, void* tmp, void* out, double omega,
                                double omega_r, uint32_t policy, cudaStream_t s) {
  cudaError_t pe = cudaSuccess;
  bool done = false;
  if (A.prec == MPMG_FP16) done = plane_level_op_f16(3, A, b, b, out, omega, policy, s, &pe);
  else if (A.prec == MPMG_FP32) done = plane_level_op_f32(3, A, b, b, out, omega, policy, s, &pe);
  else done = plane_level_op_f64(3, A, b, b, out, omega, policy, s, &pe);
  if (done) return pe;
  cudaError_t e = launch_jacobi_zero(A.dim, A.nodes, A.prec, b, tmp, omega_r, A.inv_diag, policy, s);
  if (e == cudaSuccess) e = launch_level_op(2, A, tmp, b, out, omega, policy, s);
  return e;
}

cudaError_t launch_level_op(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                            uint32_t policy, cudaStream_t s) {
  switch (A.prec) {
    case MPMG_FP16: return launch_level_op_f16(op, A, x, b, out, omega, policy, s);
    case MPMG_FP32: return launch_level_op_f32(op, A, x, b, out, omega, policy, s);
    default: return launch_level_op_f64(op, A, x, b, out, omega, policy, s);
  }
}

}  // namespace mpmg_impl
