// TMA-staged plane-kernel instantiations for binary16 levels (mpmg_plane.cuh).
#include "mpmg_plane_launch.cuh"

namespace mpmg_impl {
bool plane_level_op_f16(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                       uint32_t policy, cudaStream_t s, cudaError_t* err, const mpmg_slab* slab) {
  return plane_level_op<mpmg_dev::P16>(op, A, x, b, out, omega, policy, s, err, slab);
}
// one Jacobi step whose output goes to slot *slot of a ring (stride values)
bool plane_jacobi_slot_f16(const mpmg_stencil& A, const void* x, const void* b, void* ring, long long stride,
                          const int* slot, double omega, uint32_t policy, cudaStream_t s, cudaError_t* err) {
  return plane_level_op<mpmg_dev::P16>(2, A, x, b, ring, omega, policy, s, err, nullptr, slot, stride);
}
bool plane_level_op_push_f16(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                              uint32_t policy, cudaStream_t s, cudaError_t* err, const mpmg_slab* slab, void* push_lo,
                              void* push_hi) {
  return plane_level_op_push<mpmg_dev::P16>(op, A, x, b, out, omega, policy, s, err, slab, push_lo, push_hi);
}
}  // namespace mpmg_impl
