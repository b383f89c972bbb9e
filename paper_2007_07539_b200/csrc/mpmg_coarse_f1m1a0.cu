// Coarse-level kernel instantiations: flush_subnormals_to_zero = true,
// fused_multiply_add = true, binary32 accumulation of binary16 = false (one
// translation unit per policy so the eight compile in parallel).
#include "mpmg_coarse.cuh"

namespace mpmg_impl {

cudaError_t launch_coarse_f1m1a0(const CoarseArgs& a, cudaStream_t s) {
  return coarse_detail::launch_t<true, true, false>(a, s);
}

}  // namespace mpmg_impl
