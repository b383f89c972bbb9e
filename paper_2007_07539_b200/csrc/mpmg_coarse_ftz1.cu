// Coarse-level kernel instantiations, flush_subnormals_to_zero = true.
#include "mpmg_coarse.cuh"

namespace mpmg_impl {

using namespace coarse_detail;

cudaError_t launch_coarse_ftz1(const CoarseArgs& a, uint32_t policy, cudaStream_t s) {
  const bool fma = policy & MPMG_FMA, acc = policy & MPMG_ACC32;
  if (fma) return acc ? launch_t<true, true, true>(a, s) : launch_t<true, true, false>(a, s);
  return acc ? launch_t<true, false, true>(a, s) : launch_t<true, false, false>(a, s);
}

}  // namespace mpmg_impl
