// Layer-1 C ABI (include/mpmg_gpu.h): one entry point per kernel family, on
// device pointers in the padded layout. Argument checks mirror the
// reference's `require` preconditions (kernels.cpp:243-395,
// multigrid.cpp:79-280) and map to MPMG_EINVAL instead of exceptions.
#include "mpmg_host.h"
#include "mpmg_internal.h"

using namespace mpmg_impl;

namespace {

bool valid_prec(int p) { return p == MPMG_FP16 || p == MPMG_FP32 || p == MPMG_FP64; }

bool valid_stencil(const mpmg_stencil* A) {
  return A && (A->dim == 2 || A->dim == 3) && A->nodes >= 3 && valid_prec(A->prec) &&
         A->ntaps == (A->dim == 3 ? 27 : 9);
}

int rc(cudaError_t e) { return e == cudaSuccess ? MPMG_OK : set_cuda_error(e); }

}  // namespace

extern "C" {

int mpmg_gpu_pack(int32_t dim, int32_t nodes, int32_t prec, const void* compact, void* padded, void* stream) {
  clear_stale_error();
  if ((dim != 2 && dim != 3) || nodes < 3 || !valid_prec(prec) || !compact || !padded) return MPMG_EINVAL;
  return rc(launch_pack(dim, nodes, prec, compact, padded, false, (cudaStream_t)stream));
}

int mpmg_gpu_unpack(int32_t dim, int32_t nodes, int32_t prec, const void* padded, void* compact, void* stream) {
  clear_stale_error();
  if ((dim != 2 && dim != 3) || nodes < 3 || !valid_prec(prec) || !compact || !padded) return MPMG_EINVAL;
  return rc(launch_pack(dim, nodes, prec, compact, const_cast<void*>(padded), true, (cudaStream_t)stream));
}

int mpmg_gpu_jacobi(const mpmg_stencil* A, const void* b, const void* u_in, void* u_out, double omega,
                    uint32_t policy, void* stream) {
  clear_stale_error();
  if (!valid_stencil(A) || !b || !u_out || u_in == u_out) return MPMG_EINVAL;
  if (!(omega > 0.0 && omega <= 1.0)) return MPMG_EINVAL;  // multigrid.cpp:82
  if (!stencil_supported(A->dim, A->nodes, A->prec)) return MPMG_EUNSUPPORTED;
  const cudaStream_t s = (cudaStream_t)stream;
  if (!u_in)
    return rc(launch_jacobi_zero(A->dim, A->nodes, A->prec, b, u_out, round_to(omega, A->prec, policy & MPMG_FTZ),
                                 A->inv_diag, policy, s));
  return rc(launch_level_op(2, *A, u_in, b, u_out, omega, policy, s));
}

int mpmg_gpu_jacobi_from_zero2(const mpmg_stencil* A, const void* b, void* tmp, void* u_out, double omega,
                               uint32_t policy, void* stream) {
  clear_stale_error();
  if (!valid_stencil(A) || !b || !tmp || !u_out || tmp == u_out || b == u_out) return MPMG_EINVAL;
  if (!(omega > 0.0 && omega <= 1.0)) return MPMG_EINVAL;  // multigrid.cpp:82
  if (!stencil_supported(A->dim, A->nodes, A->prec)) return MPMG_EUNSUPPORTED;
  const double wr = round_to(omega, A->prec, policy & MPMG_FTZ);
  return rc(launch_jacobi_zero2(*A, b, tmp, u_out, omega, wr, policy, (cudaStream_t)stream));
}

int mpmg_gpu_defect(const mpmg_stencil* A, const void* b, const void* u, void* r, uint32_t policy, void* stream) {
  clear_stale_error();
  if (!valid_stencil(A) || !b || !u || !r || u == r) return MPMG_EINVAL;
  if (!stencil_supported(A->dim, A->nodes, A->prec)) return MPMG_EUNSUPPORTED;
  return rc(launch_level_op(1, *A, u, b, r, 1.0, policy, (cudaStream_t)stream));
}

int mpmg_gpu_spmv(const mpmg_stencil* A, const void* x, void* y, uint32_t policy, void* stream) {
  clear_stale_error();
  if (!valid_stencil(A) || !x || !y || x == y) return MPMG_EINVAL;  // kernels.cpp:248 aliasing
  if (!stencil_supported(A->dim, A->nodes, A->prec)) return MPMG_EUNSUPPORTED;
  return rc(launch_level_op(0, *A, x, nullptr, y, 1.0, policy, (cudaStream_t)stream));
}

int mpmg_gpu_restrict(int32_t dim, int32_t fine_nodes, int32_t fine_prec, int32_t coarse_prec, const void* r_fine,
                      void* r_coarse, const double* scale_dev, uint32_t policy, void* stream) {
  clear_stale_error();
  if ((dim != 2 && dim != 3) || fine_nodes < 5 || (fine_nodes - 1) % 2 || !valid_prec(fine_prec) ||
      !valid_prec(coarse_prec) || !r_fine || !r_coarse)
    return MPMG_EINVAL;
  return rc(launch_restrict(dim, fine_nodes, fine_prec, coarse_prec, r_fine, r_coarse, scale_dev, policy,
                            (cudaStream_t)stream));
}

int mpmg_gpu_prolong_correct(int32_t dim, int32_t fine_nodes, int32_t fine_prec, int32_t coarse_prec,
                             const void* c_coarse, void* u_fine, const double* scale_dev, uint32_t policy,
                             void* stream) {
  clear_stale_error();
  if ((dim != 2 && dim != 3) || fine_nodes < 5 || (fine_nodes - 1) % 2 || !valid_prec(fine_prec) ||
      !valid_prec(coarse_prec) || !c_coarse || !u_fine)
    return MPMG_EINVAL;
  return rc(launch_prolong(dim, fine_nodes, fine_prec, coarse_prec, c_coarse, u_fine, scale_dev, policy,
                           (cudaStream_t)stream));
}

int mpmg_gpu_defect_f64(const mpmg_stencil* A64, const double* b, const double* u, double* r, double* partials,
                        void* stream) {
  clear_stale_error();
  if (!valid_stencil(A64) || A64->prec != MPMG_FP64 || !b || !u || !r) return MPMG_EINVAL;
  if (!stencil_supported(A64->dim, A64->nodes, MPMG_FP64)) return MPMG_EUNSUPPORTED;
  return rc(launch_defect64(*A64, b, u, r, partials, true, false, (cudaStream_t)stream));
}

int mpmg_gpu_update_rc(const mpmg_stencil* A64, const void* c, int32_t c_prec, double* r, double* u,
                       const double* alpha_dev, double* partials, uint32_t policy, void* stream) {
  clear_stale_error();
  if (!valid_stencil(A64) || A64->prec != MPMG_FP64 || !c || !valid_prec(c_prec) || !r || !u || !alpha_dev)
    return MPMG_EINVAL;
  if (!stencil_supported(A64->dim, A64->nodes, c_prec)) return MPMG_EUNSUPPORTED;
  return rc(launch_update_rc(*A64, c, c_prec, r, u, alpha_dev, partials, policy & MPMG_FMA, (cudaStream_t)stream));
}

int mpmg_gpu_update_r(const mpmg_stencil* A64, const void* c, int32_t c_prec, double* r, const double* alpha_dev,
                      double* partials, void* ring, int64_t ring_len, const int32_t* slot_dev, double* ring_scale,
                      uint32_t policy, void* stream) {
  clear_stale_error();
  if (!valid_stencil(A64) || A64->prec != MPMG_FP64 || !c || !valid_prec(c_prec) || !r || !alpha_dev || !ring ||
      ring_len < (int64_t)mpmg_padded_len(A64->dim, A64->nodes) || !slot_dev || !ring_scale)
    return MPMG_EINVAL;
  cudaError_t e = cudaSuccess;
  if (!plane_update_r(*A64, c, c_prec, r, alpha_dev, partials, ring, (long long)ring_len, slot_dev, ring_scale,
                      policy & MPMG_FMA, (cudaStream_t)stream, &e))
    return MPMG_EUNSUPPORTED;
  return rc(e);
}

int mpmg_gpu_jacobi_slot(const mpmg_stencil* A, const void* b, const void* u_in, void* ring, int64_t ring_len,
                         const int32_t* slot_dev, double omega, uint32_t policy, void* stream) {
  clear_stale_error();
  if (!valid_stencil(A) || !b || !u_in || !ring || !slot_dev) return MPMG_EINVAL;
  if (!(omega > 0.0 && omega <= 1.0)) return MPMG_EINVAL;  // multigrid.cpp:82
  if (ring_len < (int64_t)mpmg_padded_len(A->dim, A->nodes)) return MPMG_EINVAL;
  cudaError_t e = cudaSuccess;
  bool done = false;
  if (A->prec == MPMG_FP16)
    done = plane_jacobi_slot_f16(*A, u_in, b, ring, (long long)ring_len, slot_dev, omega, policy, (cudaStream_t)stream, &e);
  else if (A->prec == MPMG_FP32)
    done = plane_jacobi_slot_f32(*A, u_in, b, ring, (long long)ring_len, slot_dev, omega, policy, (cudaStream_t)stream, &e);
  if (!done) return MPMG_EUNSUPPORTED;
  return rc(e);
}

int mpmg_gpu_update_r_partials(int32_t dim, int32_t nodes, int32_t c_prec) {
  clear_stale_error();
  const int n = plane_update_r_partials(dim, nodes, c_prec);
  return n > 0 ? n : MPMG_EUNSUPPORTED;
}

int mpmg_gpu_fold(int64_t len, double* u, const void* ring, int64_t ring_len, int32_t c_prec,
                  const double* ring_scale, const int32_t* count_dev, uint32_t policy, void* stream) {
  clear_stale_error();
  if (len < 1 || !u || !ring || ring_len < len || !valid_prec(c_prec) || !ring_scale || !count_dev) return MPMG_EINVAL;
  return rc(launch_fold((size_t)len, u, ring, (long long)ring_len, c_prec, ring_scale, count_dev, 0, nullptr,
                        policy & MPMG_FMA, (cudaStream_t)stream));
}

int mpmg_gpu_scale_downcast(int32_t dim, int32_t nodes, const double* x, void* out, int32_t prec,
                            const double* alpha_dev, int32_t scale_enabled, uint32_t policy, void* stream) {
  clear_stale_error();
  if ((dim != 2 && dim != 3) || nodes < 3 || !x || !out || !valid_prec(prec) || !alpha_dev) return MPMG_EINVAL;
  return rc(launch_downcast(dim, nodes, x, out, prec, alpha_dev, scale_enabled, policy, (cudaStream_t)stream));
}

int mpmg_gpu_partials_len(int32_t dim, int32_t nodes) {
  clear_stale_error();
  int m = norm2_partials(mpmg_padded_len(dim, nodes));
  for (int lp : {MPMG_FP16, MPMG_FP32, MPMG_FP64})
    for (bool up : {false, true}) {
      const int v = stencil_partials(dim, nodes, lp, up);
      m = m > v ? m : v;
    }
  return m;
}

int mpmg_gpu_norm2_f64(int32_t dim, int32_t nodes, const double* x, double* partials, double* out_dev,
                       void* stream) {
  clear_stale_error();
  if ((dim != 2 && dim != 3) || nodes < 3 || !x || !partials || !out_dev) return MPMG_EINVAL;
  return rc(launch_norm2(mpmg_padded_len(dim, nodes), x, partials, out_dev, (cudaStream_t)stream));
}

int mpmg_gpu_norm_finalize(const double* partials, int32_t n_partials, double* out_dev, void* stream) {
  clear_stale_error();
  if (!partials || n_partials < 0 || !out_dev) return MPMG_EINVAL;
  return rc(launch_norm_finalize(partials, n_partials, out_dev, (cudaStream_t)stream));
}

// level-0-style stencil for a grid/precision (MgHierarchy::build per level)
int mpmg_build_stencil(int32_t dim, int32_t nodes, int32_t prec, uint32_t policy, mpmg_stencil* out) {
  if (!out || !valid_prec(prec)) return MPMG_EINVAL;
  return build_level_stencil(dim, nodes, prec, policy & MPMG_FTZ, out);
}

double mpmg_round_fp16(double x, int32_t ftz) { return round_fp16(x, ftz != 0); }

int mpmg_dev_count(void) {
  clear_stale_error();
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void* mpmg_dev_alloc(size_t bytes) {
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, bytes < 16 ? 16 : bytes);
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return nullptr;
  }
  return p;
}

void mpmg_dev_free(void* p) {
  if (p) cudaFree(p);
}

int mpmg_dev_h2d(void* dst, const void* src, size_t bytes) {
  clear_stale_error();
  if (!bytes) return MPMG_OK;
  if (!dst || !src) return MPMG_EINVAL;
  return rc(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
}

int mpmg_dev_d2h(void* dst, const void* src, size_t bytes) {
  clear_stale_error();
  if (!bytes) return MPMG_OK;
  if (!dst || !src) return MPMG_EINVAL;
  return rc(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
}

int mpmg_dev_memset0(void* p, size_t bytes) {
  clear_stale_error();
  if (!bytes) return MPMG_OK;
  if (!p) return MPMG_EINVAL;
  return rc(cudaMemset(p, 0, bytes));
}

int mpmg_dev_sync(void) { return rc(cudaDeviceSynchronize()); }

}  // extern "C"

// ---- z-slab entry points (multi-GPU slab decomposition) -------------------
namespace {

bool valid_slab(const mpmg_stencil* A, const mpmg_slab* s) {
  return valid_stencil(A) && A->dim == 3 && s && s->nz >= 1 && s->z_lo >= 1 && s->z_lo + s->nz <= A->nodes - 1 &&
         (A->nodes - 1) % 32 == 0;
}

}  // namespace

extern "C" {

size_t mpmg_slab_len(int32_t nodes, int32_t nz) {
  const size_t P = (size_t)(nodes - 1);
  return (size_t)(nz + 2) * P * P + P + 1;
}

int mpmg_gpu_slab_jacobi(const mpmg_stencil* A, const mpmg_slab* s, const void* b, const void* u_in, void* u_out,
                         double omega, uint32_t policy, void* stream) {
  clear_stale_error();
  if (!valid_slab(A, s) || !b || !u_out || u_in == u_out || !(omega > 0.0 && omega <= 1.0)) return MPMG_EINVAL;
  const cudaStream_t q = (cudaStream_t)stream;
  const bool ftz = policy & MPMG_FTZ;
  if (!u_in) {  // owned planes only: the halo planes may be receiving a neighbour's copy right now
    const size_t pl = (size_t)(A->nodes - 1) * (A->nodes - 1);
    const size_t off = pl * (size_t)mpmg_bytes_per_value(A->prec);
    return rc(launch_jacobi_zero_len(pl * (size_t)s->nz, A->prec, static_cast<const unsigned char*>(b) + off,
                                     static_cast<unsigned char*>(u_out) + off, round_to(omega, A->prec, ftz),
                                     A->inv_diag, policy, q));
  }
  cudaError_t e = cudaSuccess;
  bool done = false;
  if (A->prec == MPMG_FP16) done = plane_level_op_f16(2, *A, u_in, b, u_out, omega, policy, q, &e, s);
  else if (A->prec == MPMG_FP32) done = plane_level_op_f32(2, *A, u_in, b, u_out, omega, policy, q, &e, s);
  else done = plane_level_op_f64(2, *A, u_in, b, u_out, omega, policy, q, &e, s);
  return done ? rc(e) : MPMG_EUNSUPPORTED;
}

int mpmg_gpu_slab_defect(const mpmg_stencil* A, const mpmg_slab* s, const void* b, const void* u, void* r,
                         uint32_t policy, void* stream) {
  clear_stale_error();
  if (!valid_slab(A, s) || !b || !u || !r || u == r) return MPMG_EINVAL;
  const cudaStream_t q = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  bool done = false;
  if (A->prec == MPMG_FP16) done = plane_level_op_f16(1, *A, u, b, r, 1.0, policy, q, &e, s);
  else if (A->prec == MPMG_FP32) done = plane_level_op_f32(1, *A, u, b, r, 1.0, policy, q, &e, s);
  else done = plane_level_op_f64(1, *A, u, b, r, 1.0, policy, q, &e, s);
  return done ? rc(e) : MPMG_EUNSUPPORTED;
}

int mpmg_gpu_slab_restrict(int32_t fine_nodes, const mpmg_slab* sf, const mpmg_slab* sc, int32_t fine_prec,
                           int32_t coarse_prec, const void* r_fine, void* r_coarse, uint32_t policy, void* stream) {
  clear_stale_error();
  if (!sf || !sc || !r_fine || !r_coarse || !valid_prec(fine_prec) || !valid_prec(coarse_prec) ||
      (fine_nodes - 1) % 2 || 2 * sc->z_lo < sf->z_lo || 2 * (sc->z_lo + sc->nz - 1) + 1 > sf->z_lo + sf->nz)
    return MPMG_EINVAL;
  return rc(launch_restrict_slab(fine_nodes, *sf, *sc, fine_prec, coarse_prec, r_fine, r_coarse, policy,
                                 (cudaStream_t)stream));
}

int mpmg_gpu_slab_prolong_correct(int32_t fine_nodes, const mpmg_slab* sf, const mpmg_slab* sc, int32_t fine_prec,
                                  int32_t coarse_prec, const void* c_coarse, void* u_fine, uint32_t policy,
                                  void* stream) {
  clear_stale_error();
  if (!sf || !sc || !c_coarse || !u_fine || !valid_prec(fine_prec) || !valid_prec(coarse_prec) || (fine_nodes - 1) % 8)
    return MPMG_EINVAL;
  return rc(launch_prolong_slab(fine_nodes, *sf, *sc, fine_prec, coarse_prec, c_coarse, u_fine, policy,
                                (cudaStream_t)stream));
}

int mpmg_gpu_slab_defect_f64(const mpmg_stencil* A64, const mpmg_slab* s, const double* b, const double* u,
                             double* r, double* partials, int32_t resnorm, void* stream) {
  clear_stale_error();
  if (!valid_slab(A64, s) || A64->prec != MPMG_FP64 || !b || !u || (!r && !resnorm)) return MPMG_EINVAL;
  cudaError_t e = cudaSuccess;
  return plane_defect64(*A64, b, u, r, partials, true, resnorm != 0, (cudaStream_t)stream, nullptr, &e, s)
             ? rc(e)
             : MPMG_EUNSUPPORTED;
}

int mpmg_gpu_slab_update_rc(const mpmg_stencil* A64, const mpmg_slab* s, const void* c, int32_t c_prec, double* r,
                            double* u, const double* alpha_dev, double* partials, uint32_t policy, void* stream) {
  clear_stale_error();
  if (!valid_slab(A64, s) || A64->prec != MPMG_FP64 || !c || !valid_prec(c_prec) || !r || !u || !alpha_dev)
    return MPMG_EINVAL;
  cudaError_t e = cudaSuccess;
  return plane_update_rc(*A64, c, c_prec, r, u, alpha_dev, partials, policy & MPMG_FMA, (cudaStream_t)stream, &e, s)
             ? rc(e)
             : MPMG_EUNSUPPORTED;
}

int mpmg_gpu_slab_scale_downcast(int32_t nodes, const mpmg_slab* s, const double* x, void* out, int32_t prec,
                                 const double* alpha_dev, int32_t scale_enabled, uint32_t policy, void* stream) {
  clear_stale_error();
  if (!s || s->nz < 1 || nodes < 3 || !x || !out || !valid_prec(prec) || !alpha_dev) return MPMG_EINVAL;
  return rc(launch_downcast_len(mpmg_slab_len(nodes, s->nz), x, out, prec, alpha_dev, scale_enabled, policy,
                                (cudaStream_t)stream));
}

int mpmg_gpu_slab_partials_len(int32_t nodes, const mpmg_slab* s, int32_t c_prec, int32_t update) {
  clear_stale_error();
  if (!s || s->nz < 1) return MPMG_EINVAL;
  return plane_partials(3, nodes, c_prec, update != 0, s->nz + 1);
}

int mpmg_gpu_partials_sum(const double* partials, int32_t n, double* out_dev, void* stream) {
  clear_stale_error();
  if (!partials || n < 0 || !out_dev) return MPMG_EINVAL;
  return rc(launch_partials_sum(partials, n, out_dev, (cudaStream_t)stream));
}

}  // extern "C"
