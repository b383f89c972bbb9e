// Streaming stencil instantiations for binary32 levels (see mpmg_stencil.cuh).
#include "mpmg_stencil_launch.cuh"

namespace mpmg_impl {
cudaError_t launch_level_op_f32(int op, const mpmg_stencil& A, const void* x, const void* b, void* out,
                                double omega, uint32_t policy, cudaStream_t s) {
  return level_op_impl<mpmg_dev::P32>(op, A, x, b, out, omega, policy, s);
}
}  // namespace mpmg_impl
