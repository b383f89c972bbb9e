// Coarse-level kernel dispatcher (kernels: mpmg_coarse.cuh).
#include "mpmg_coarse.cuh"

namespace mpmg_impl {

cudaError_t launch_coarse_cycle(const CoarseArgs& a, uint32_t policy, cudaStream_t s) {
  return (policy & MPMG_FTZ) ? launch_coarse_ftz1(a, policy, s) : launch_coarse_ftz0(a, policy, s);
}

}  // namespace mpmg_impl
