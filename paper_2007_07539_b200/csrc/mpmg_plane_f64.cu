// TMA-staged plane-kernel instantiations for binary64 levels (mpmg_plane.cuh).
#include "mpmg_plane_launch.cuh"

namespace mpmg_impl {
bool plane_level_op_f64(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                       uint32_t policy, cudaStream_t s, cudaError_t* err, const mpmg_slab* slab) {
  return plane_level_op<mpmg_dev::P64>(op, A, x, b, out, omega, policy, s, err, slab);
}
bool plane_level_op_push_f64(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                              uint32_t policy, cudaStream_t s, cudaError_t* err, const mpmg_slab* slab, void* push_lo,
                              void* push_hi) {
  return plane_level_op_push<mpmg_dev::P64>(op, A, x, b, out, omega, policy, s, err, slab, push_lo, push_hi);
}
}  // namespace mpmg_impl
