// Coarse-level kernel dispatcher (kernels: mpmg_coarse.cuh).
#include "mpmg_coarse.cuh"

namespace mpmg_impl {

cudaError_t launch_coarse_cycle(const CoarseArgs& a, uint32_t policy, cudaStream_t s) {
  const int k = ((policy & MPMG_FTZ) ? 4 : 0) + ((policy & MPMG_FMA) ? 2 : 0) + ((policy & MPMG_ACC32) ? 1 : 0);
  switch (k) {
    case 0: return launch_coarse_f0m0a0(a, s);
    case 1: return launch_coarse_f0m0a1(a, s);
    case 2: return launch_coarse_f0m1a0(a, s);
    case 3: return launch_coarse_f0m1a1(a, s);
    case 4: return launch_coarse_f1m0a0(a, s);
    case 5: return launch_coarse_f1m0a1(a, s);
    case 6: return launch_coarse_f1m1a0(a, s);
    default: return launch_coarse_f1m1a1(a, s);
  }
}

}  // namespace mpmg_impl
