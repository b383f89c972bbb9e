// Internal host-side declarations shared by the CUDA translation units of the
// B200 hot path. Not part of the public ABI (see include/mpmg_gpu.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "mpmg_gpu.h"

namespace mpmg_impl {

inline int pitch(int nodes) { return nodes - 1; }

// C-ABI entry points start from a clean error state: a non-sticky error
// left behind by an unrelated runtime call of the host process (it would
// otherwise surface as this call's launch error through cudaGetLastError).
// Sticky device faults persist and are still reported.
inline void clear_stale_error() { (void)cudaGetLastError(); }

// launch with programmatic dependent launch enabled (MPMG_PDL=0 disables);
// the kernel must call mpmg_dev::pdl_wait() before reading predecessor data
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// binary16 RNE rounding with optional flush-after-rounding, in the binary64
// value domain (same contract as the reference's quantize_fp16,
// precision.cpp:23-48); host side, used to round per-level scalars.
double round_fp16(double x, bool ftz);
// PVector::set rounding (vector.hpp:43-55) to precision `prec`.
double round_to(double x, int prec, bool ftz);
uint16_t fp16_bits(double v);  // exact binary16 value -> bits
double fp16_value(uint16_t bits);

// ---- stencil family (mpmg_stencil_*.cu, mpmg_outer.cu) -------------------
// level ops: op in {0 spmv, 1 defect, 2 jacobi}; level precision A.prec
cudaError_t launch_level_op(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                            uint32_t policy, cudaStream_t s);
cudaError_t launch_jacobi_zero2(const mpmg_stencil& A, const void* b, void* tmp, void* out, double omega,
                                double omega_r, uint32_t policy, cudaStream_t s);
cudaError_t launch_level_op_f16(int op, const mpmg_stencil& A, const void* x, const void* b, void* out,
                                double omega, uint32_t policy, cudaStream_t s);
cudaError_t launch_level_op_f32(int op, const mpmg_stencil& A, const void* x, const void* b, void* out,
                                double omega, uint32_t policy, cudaStream_t s);
cudaError_t launch_level_op_f64(int op, const mpmg_stencil& A, const void* x, const void* b, void* out,
                                double omega, uint32_t policy, cudaStream_t s);
// outer FP64 ops
cudaError_t launch_defect64(const mpmg_stencil& A64, const double* b, const double* u, double* r, double* partials,
                            bool fma, bool resnorm, cudaStream_t s, const int* gate = nullptr);
cudaError_t launch_update_rc(const mpmg_stencil& A64, const void* c, int c_prec, double* r, double* u,
                             const double* alpha_dev, double* partials, bool fma, cudaStream_t s);
// number of partial sums one launch writes: the fused update with operand
// precision lp (update = true), or the FP64 defect / residual norm
int stencil_partials(int dim, int nodes, int lp, bool update);
// TMA-staged plane kernels (mpmg_plane_*.cu): return false when the shape
// or policy is not covered (the caller then uses the streaming kernels)
// (slab: a z-slab of the level, include/mpmg_gpu.h; nullptr = the whole level)
// z-slab JACOBI (op 2) / DEFECT (op 1) that also stores the boundary output
// planes into the neighbours' halo planes (multi-GPU, mpmg_dist.cu)
bool plane_level_op_push_f16(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                             uint32_t policy, cudaStream_t s, cudaError_t* err, const mpmg_slab* slab, void* push_lo,
                             void* push_hi);
bool plane_level_op_push_f32(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                             uint32_t policy, cudaStream_t s, cudaError_t* err, const mpmg_slab* slab, void* push_lo,
                             void* push_hi);
bool plane_level_op_push_f64(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                             uint32_t policy, cudaStream_t s, cudaError_t* err, const mpmg_slab* slab, void* push_lo,
                             void* push_hi);
bool plane_level_op_f16(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                        uint32_t policy, cudaStream_t s, cudaError_t* err, const mpmg_slab* slab = nullptr);
bool plane_level_op_f32(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                        uint32_t policy, cudaStream_t s, cudaError_t* err, const mpmg_slab* slab = nullptr);
bool plane_level_op_f64(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                        uint32_t policy, cudaStream_t s, cudaError_t* err, const mpmg_slab* slab = nullptr);
bool plane_jacobi_slot_f16(const mpmg_stencil& A, const void* x, const void* b, void* ring, long long stride,
                           const int* slot, double omega, uint32_t policy, cudaStream_t s, cudaError_t* err);
bool plane_jacobi_slot_f32(const mpmg_stencil& A, const void* x, const void* b, void* ring, long long stride,
                           const int* slot, double omega, uint32_t policy, cudaStream_t s, cudaError_t* err);
bool plane_defect64(const mpmg_stencil& A64, const double* b, const double* u, double* r, double* partials,
                    bool fma, bool resnorm, cudaStream_t s, const int* gate, cudaError_t* err,
                    const mpmg_slab* slab = nullptr);
bool plane_update_rc(const mpmg_stencil& A64, const void* c, int c_prec, double* r, double* u,
                     const double* alpha_dev, double* partials, bool fma, cudaStream_t s, cudaError_t* err,
                     const mpmg_slab* slab = nullptr);
int plane_partials(int dim, int nodes, int lp, bool update, int pz = 0);
bool plane_update_r(const mpmg_stencil& A64, const void* c, int c_prec, double* r, const double* alpha_dev,
                    double* partials, void* ring, long long ring_len, const int* slot, double* ring_scale, bool fma,
                    cudaStream_t s, cudaError_t* err, const mpmg_slab* slab = nullptr);
int plane_update_r_partials(int dim, int nodes, int lp, int pz = 0);
bool stencil_update_r(const mpmg_stencil& A64, const void* c, int c_prec, double* r, const double* alpha_dev,
                      double* partials, void* ring, long long ring_len, const int* slot, double* ring_scale, bool fma,
                      cudaStream_t s, cudaError_t* err);
// true when the streaming stencil kernels support this level shape
bool stencil_supported(int dim, int nodes, int prec);

// ---- pointwise / transfer (mpmg_pointwise.cu) -----------------------------
cudaError_t launch_pack(int dim, int nodes, int prec, const void* compact, void* padded, bool unpack,
                        cudaStream_t s);
cudaError_t launch_jacobi_zero(int dim, int nodes, int prec, const void* b, void* u, double omega_r,
                               double invdiag_r, uint32_t policy, cudaStream_t s);
cudaError_t launch_restrict(int dim, int fine_nodes, int fine_prec, int coarse_prec, const void* r_fine,
                            void* r_coarse, const double* scale_dev, uint32_t policy, cudaStream_t s);
cudaError_t launch_prolong(int dim, int fine_nodes, int fine_prec, int coarse_prec, const void* c_coarse,
                           void* u_fine, const double* scale_dev, uint32_t policy, cudaStream_t s);
cudaError_t launch_jacobi_zero_len(size_t len, int prec, const void* b, void* u, double omega_r, double invdiag_r,
                                   uint32_t policy, cudaStream_t s);
cudaError_t launch_downcast_len(size_t len, const double* x, void* out, int prec, const double* alpha_dev,
                                int scale_enabled, uint32_t policy, cudaStream_t s);
cudaError_t launch_restrict_slab(int fine_nodes, const mpmg_slab& sf, const mpmg_slab& sc, int fine_prec,
                                 int coarse_prec, const void* r_fine, void* r_coarse, uint32_t policy, cudaStream_t s);
cudaError_t launch_prolong_slab(int fine_nodes, const mpmg_slab& sf, const mpmg_slab& sc, int fine_prec,
                                int coarse_prec, const void* c_coarse, void* u_fine, uint32_t policy, cudaStream_t s);
cudaError_t launch_downcast(int dim, int nodes, const double* x, void* out, int prec, const double* alpha_dev,
                            int scale_enabled, uint32_t policy, cudaStream_t s);
cudaError_t launch_norm2(size_t len, const double* x, double* partials, double* out, cudaStream_t s);
cudaError_t launch_norm_finalize(const double* partials, int n, double* out, cudaStream_t s);
cudaError_t launch_partials_sum(const double* partials, int n, double* out, cudaStream_t s);
int norm2_partials(size_t len);
cudaError_t launch_copy_sumsq(size_t len, const double* x, double* y, double* partials, cudaStream_t s);
cudaError_t launch_fold(size_t len, double* u, const void* ring, long long ring_len, int prec, const double* scales,
                        const int* count, int extra, const int* gate, bool fma, cudaStream_t s,
                        const int* uzero = nullptr);
cudaError_t launch_fill_random01(double* padded_u, int dim, int nodes, uint64_t seed, cudaStream_t s);

// ---- coarse sub-hierarchy (mpmg_coarse.cu) --------------------------------
constexpr int kMaxCoarseLevels = 16;
struct CoarseLevel {
  int dim, nodes, prec;
  double taps[27];
  double inv_diag;  // rounded to prec
  double omega;     // rounded to prec
  void *u, *u2, *b, *r;  // padded vectors of this level
  double* prod;          // binary64 scratch (restriction products), interior-sized padded
};
struct CoarseArgs {
  int nlev;          // levels 0..nlev-1 handled by the kernel
  int pre, post;
  int rescale;       // DSH restriction rescaling (multigrid.cpp:383)
  double base_tol;
  int base_mode, base_maxit;
  CoarseLevel lv[kMaxCoarseLevels];
  // CG scratch on level 0 (padded, level-0 precision) + best iterate
  void *cg_r, *cg_p, *cg_ap, *cg_s, *cg_best;
  int* cg_iterations;  // optional diagnostics (device)
  int cta_points;      // levels with <= this many unknowns run on CTA 0 out of shared memory
  int debug;           // MPMG_COARSE_DEBUG=1: record per-phase clock64 stamps
  long long* dbg;      // device buffer for them (64 entries) or nullptr
  // cluster slab mode shared-memory layout, filled by the launcher (slab_smem)
  unsigned long long slab_off[kMaxCoarseLevels + 1], slab_sz[kMaxCoarseLevels], slab_total;
};
cudaError_t launch_coarse_cycle(const CoarseArgs& a, uint32_t policy, cudaStream_t s);

// ---- IR control (mpmg_solver.cu) ------------------------------------------
struct IrState {
  double alpha;       // current ||r||
  double scale;       // scale used by the current iteration
  int iterations;
  int converged;
  int diverged;
  int active;         // loop still running
  int refresh_now;    // next refresh due
  int pending;        // deferred corrections stored in the ring, not yet folded into u
  int fold_now;       // the current iteration folds the ring into u (refresh due or ring full)
  int final_pending;  // residual_norm still to compute (0: the last iteration's refresh defect
                      // left exactly its partial sums in the buffer)
  int u_zero;         // deferred corrections: u is still the zero initial guess (never written)
};

std::string& last_error();
int set_cuda_error(cudaError_t e);

}  // namespace mpmg_impl
