// Generic ELLPACK device path: the reference's operator format
// (EllMatrix, ell_matrix.hpp:18-74) for systems that are not the Poisson
// stencil hierarchy (MgHierarchy::from_levels, multigrid.hpp:109-111, and the
// public kernel API, kernels.hpp:11-38). Matrices live on the device
// slot-major (val[s * rows + r]) so a warp reading slot s of 32 consecutive
// rows is one coalesced access; the per-row summation order is the
// reference's slot order, every operation rounded like Arith<P>
// (kernels.cpp:18-67).
#include <algorithm>

#include "mpmg_arith.cuh"
#include "mpmg_internal.h"

namespace mpmg_impl {

using namespace mpmg_dev;

namespace {

constexpr int kT = 256;

template <int PREC> struct E;
template <> struct E<P16> { using T = __half; };
template <> struct E<P32> { using T = float; };
template <> struct E<P64> { using T = double; };

// Arith<P> on scalars, policy as template flags
template <int PREC, bool FTZ, bool FMA> struct Ar;
template <bool FTZ, bool FMA> struct Ar<P16, FTZ, FMA> {
  using T = __half;
  static __device__ __forceinline__ T fma(T a, T b, T c) { return fma16s<FTZ, FMA>(a, b, c); }
  static __device__ __forceinline__ T mul(T a, T b) { return mul16s<FTZ>(a, b); }
  static __device__ __forceinline__ T from(double v) { return round16<FTZ>(v); }
  static __device__ __forceinline__ double wide(T v) { return (double)__half2float(v); }
  static __device__ __forceinline__ T zero() { return __ushort_as_half((unsigned short)0); }
};
template <bool FTZ, bool FMA> struct Ar<P32, FTZ, FMA> {
  using T = float;
  static __device__ __forceinline__ T fma(T a, T b, T c) { return fma32<FTZ, FMA>(a, b, c); }
  static __device__ __forceinline__ T mul(T a, T b) { return mul32<FTZ>(a, b); }
  static __device__ __forceinline__ T from(double v) { return round32<FTZ>(v); }
  static __device__ __forceinline__ double wide(T v) { return (double)v; }
  static __device__ __forceinline__ T zero() { return 0.0f; }
};
template <bool FTZ, bool FMA> struct Ar<P64, FTZ, FMA> {
  using T = double;
  static __device__ __forceinline__ T fma(T a, T b, T c) { return fma64<FMA>(a, b, c); }
  static __device__ __forceinline__ T mul(T a, T b) { return mul64(a, b); }
  static __device__ __forceinline__ T from(double v) { return v; }
  static __device__ __forceinline__ double wide(T v) { return v; }
  static __device__ __forceinline__ T zero() { return 0.0; }
};

template <int PREC>
__device__ __forceinline__ double wide_any(const void* p, long long i) {
  if constexpr (PREC == P16) return (double)__half2float(static_cast<const __half*>(p)[i]);
  else if constexpr (PREC == P32) return (double)static_cast<const float*>(p)[i];
  else return static_cast<const double*>(p)[i];
}

// y = A x (spmv_impl, kernels.cpp:137-193); ACC32: binary16 data with a
// binary32 fma chain and one final rounding (kernels.cpp:151-162)
template <int PREC, bool FTZ, bool FMA, bool ACC32>
__global__ void k_ell_spmv(long long rows, int rw, const int* __restrict__ col, const void* __restrict__ val,
                           const void* __restrict__ x, void* __restrict__ y) {
  using A = Ar<PREC, FTZ, FMA>;
  using T = typename A::T;
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const T* v = static_cast<const T*>(val);
  const T* xv = static_cast<const T*>(x);
  if constexpr (ACC32) {
    float acc = 0.0f;
    for (int s = 0; s < rw; ++s)
      acc = fma32<FTZ, FMA>(__half2float(v[s * rows + r]), __half2float(xv[col[s * rows + r]]), acc);
    static_cast<T*>(y)[r] = f16s<FTZ>(__float2half_rn(acc));
  } else {
    T acc = A::zero();
    for (int s = 0; s < rw; ++s) acc = A::fma(v[s * rows + r], xv[col[s * rows + r]], acc);
    static_cast<T*>(y)[r] = acc;
  }
}

// out = y + alpha x (axpy_impl, kernels.cpp:195-212): alpha rounded first
template <int PREC, bool FTZ, bool FMA>
__global__ void k_axpy(long long n, double alpha, const void* x, const void* y, void* out) {
  using A = Ar<PREC, FTZ, FMA>;
  using T = typename A::T;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T a = A::from(alpha);
  static_cast<T*>(out)[i] = A::fma(a, static_cast<const T*>(x)[i], static_cast<const T*>(y)[i]);
}

// out = a .* b (vec_multiply_impl, kernels.cpp:214-229)
template <int PREC, bool FTZ, bool FMA>
__global__ void k_vmul(long long n, const void* a, const void* b, void* out) {
  using A = Ar<PREC, FTZ, FMA>;
  using T = typename A::T;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  static_cast<T*>(out)[i] = A::mul(static_cast<const T*>(a)[i], static_cast<const T*>(b)[i]);
}

// transfer_product<CP> (multigrid.cpp:155-205) + store_scaled (:220-232):
// product in the precision CP of x with the matrix value re-rounded to CP,
// then out = round_OP(prod / scale) (divide) or round_OP(prod * scale);
// optionally the binary64 products for the DSH norm
template <int CP, int MP, int OP, bool FTZ, bool FMA>
__global__ void k_ell_transfer(long long rows, int rw, const int* __restrict__ col, const void* __restrict__ val,
                               const void* __restrict__ x, const double* scale_dev, int divide, void* out,
                               double* prod) {
  using A = Ar<CP, FTZ, FMA>;
  using T = typename A::T;
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const T* xv = static_cast<const T*>(x);
  T acc = A::zero();
  for (int s = 0; s < rw; ++s) {
    const double mv = wide_any<MP>(val, s * rows + r);
    if constexpr (CP == P32) {  // multigrid.cpp:178-184: the unfused product rounds to binary32, only the sum flushes
      const float m = (float)mv, xx = xv[col[s * rows + r]];
      acc = f32<FTZ>(FMA ? __fmaf_rn(m, xx, acc) : __fadd_rn(__fmul_rn(m, xx), acc));
    } else {
      acc = A::fma(A::from(mv), xv[col[s * rows + r]], acc);
    }
  }
  const double p = A::wide(acc);
  if (prod) prod[r] = p;
  if (out) {
    const double sc = scale_dev ? *scale_dev : 1.0;
    const double v = divide ? p / sc : p * sc;
    if constexpr (OP == P16) static_cast<__half*>(out)[r] = round16<FTZ>(v);
    else if constexpr (OP == P32) static_cast<float*>(out)[r] = round32<FTZ>(v);
    else static_cast<double*>(out)[r] = v;
  }
}

// update_residuum_correction on a generic FP64 ELL (kernels.cpp:300-341)
template <int CP, bool FMA>
__global__ void k_ell_update(long long rows, int rw, const int* __restrict__ col, const double* __restrict__ val,
                             const void* __restrict__ c, double* r, double* u, const double* alpha_dev) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const double al = *alpha_dev;
  u[i] = fma64<FMA>(al, wide_any<CP>(c, i), u[i]);
  double s = 0.0;
  for (int k = 0; k < rw; ++k) s = fma64<FMA>(val[k * rows + i], wide_any<CP>(c, col[k * rows + i]), s);
  r[i] = fma64<FMA>(-al, s, r[i]);
}

// cast_vector (kernels.cpp:231-239, 343-360): out = round_OP(x / scale)
template <int XP, int OP, bool FTZ>
__global__ void k_cast(long long n, const void* x, void* out, const double* scale_dev, double scale) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double s = scale_dev ? *scale_dev : scale;
  const double v = wide_any<XP>(x, i) / s;
  if constexpr (OP == P16) static_cast<__half*>(out)[i] = round16<FTZ>(v);
  else if constexpr (OP == P32) static_cast<float*>(out)[i] = round32<FTZ>(v);
  else static_cast<double*>(out)[i] = v;
}

// dot_fp64 / norm2_fp64 (kernels.cpp:368-395): ONE thread, sequential fma in
// index order -- bitwise the reference's value. (The IR hot path uses the
// deterministic tree reduction instead, SURVEY §7 hard part 7.)
template <int XP, int YP>
__global__ void k_dot_seq(long long n, const void* x, const void* y, double* out, int sqrt_it) {
  double acc = 0.0;
  for (long long i = 0; i < n; ++i) acc = __fma_rn(wide_any<XP>(x, i), wide_any<YP>(y, i), acc);
  *out = sqrt_it ? sqrt(acc) : acc;
}

// validate mode (kernels.cpp:90-113, multigrid.cpp:259-265): the smallest
// index holding a non-finite value (binary16: exponent field all ones), or
// n when every entry is finite
template <int XP>
__global__ void k_find_nonfinite(long long n, const void* x, unsigned long long* first) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool bad;
  if constexpr (XP == P16) bad = (__half_as_ushort(static_cast<const __half*>(x)[i]) & 0x7C00u) == 0x7C00u;
  else if constexpr (XP == P32) bad = !isfinite(static_cast<const float*>(x)[i]);
  else bad = !isfinite(static_cast<const double*>(x)[i]);
  if (bad) atomicMin(first, (unsigned long long)i);
}

template <typename F>
cudaError_t by_prec(int p, F&& f) {
  switch (p) {
    case MPMG_FP16: return f(std::integral_constant<int, P16>{});
    case MPMG_FP32: return f(std::integral_constant<int, P32>{});
    default: return f(std::integral_constant<int, P64>{});
  }
}
template <typename F>
cudaError_t by_pol(uint32_t policy, F&& f) {
  const bool ftz = policy & MPMG_FTZ, fma = policy & MPMG_FMA;
  if (ftz && fma) return f(std::true_type{}, std::true_type{});
  if (ftz) return f(std::true_type{}, std::false_type{});
  if (fma) return f(std::false_type{}, std::true_type{});
  return f(std::false_type{}, std::false_type{});
}
inline unsigned nb(long long n) { return (unsigned)std::max<long long>(1, (n + kT - 1) / kT); }
inline bool vp(int p) { return p == MPMG_FP16 || p == MPMG_FP32 || p == MPMG_FP64; }
int rc(cudaError_t e) { return e == cudaSuccess ? MPMG_OK : set_cuda_error(e); }

}  // namespace
}  // namespace mpmg_impl

using namespace mpmg_impl;

extern "C" {

int mpmg_gpu_ell_spmv(int64_t rows, int32_t rw, const int32_t* col, const void* val, int32_t prec, const void* x,
                      void* y, uint32_t policy, void* stream) {
  clear_stale_error();
  if (rows < 0 || rw < 1 || !vp(prec) || !col || !val || !x || !y || x == y) return MPMG_EINVAL;
  if (rows == 0) return MPMG_OK;
  const cudaStream_t s = (cudaStream_t)stream;
  return rc(by_prec(prec, [&](auto pc) -> cudaError_t {
    return by_pol(policy, [&](auto ft, auto fm) -> cudaError_t {
      constexpr int PR = decltype(pc)::value;
      constexpr bool F = decltype(ft)::value, M = decltype(fm)::value;
      if (PR == P16 && (policy & MPMG_ACC32))
        k_ell_spmv<P16, F, M, true><<<nb(rows), kT, 0, s>>>(rows, rw, col, val, x, y);
      else
        k_ell_spmv<PR, F, M, false><<<nb(rows), kT, 0, s>>>(rows, rw, col, val, x, y);
      return cudaGetLastError();
    });
  }));
}

int mpmg_gpu_axpy(int64_t n, int32_t prec, double alpha, const void* x, const void* y, void* out, uint32_t policy,
                  void* stream) {
  clear_stale_error();
  if (n < 0 || !vp(prec) || !x || !y || !out) return MPMG_EINVAL;
  if (n == 0) return MPMG_OK;
  return rc(by_prec(prec, [&](auto pc) -> cudaError_t {
    return by_pol(policy, [&](auto ft, auto fm) -> cudaError_t {
      k_axpy<decltype(pc)::value, decltype(ft)::value, decltype(fm)::value>
          <<<nb(n), kT, 0, (cudaStream_t)stream>>>(n, alpha, x, y, out);
      return cudaGetLastError();
    });
  }));
}

int mpmg_gpu_vec_multiply(int64_t n, int32_t prec, const void* a, const void* b, void* out, uint32_t policy,
                          void* stream) {
  clear_stale_error();
  if (n < 0 || !vp(prec) || !a || !b || !out) return MPMG_EINVAL;
  if (n == 0) return MPMG_OK;
  return rc(by_prec(prec, [&](auto pc) -> cudaError_t {
    return by_pol(policy, [&](auto ft, auto fm) -> cudaError_t {
      k_vmul<decltype(pc)::value, decltype(ft)::value, decltype(fm)::value>
          <<<nb(n), kT, 0, (cudaStream_t)stream>>>(n, a, b, out);
      return cudaGetLastError();
    });
  }));
}

int mpmg_gpu_ell_transfer(int64_t rows, int32_t rw, const int32_t* col, const void* val, int32_t mat_prec,
                          const void* x, int32_t x_prec, int32_t out_prec, const double* scale_dev, int32_t divide,
                          void* out, double* prod, uint32_t policy, void* stream) {
  clear_stale_error();
  if (rows < 0 || rw < 1 || !col || !val || !x || !vp(mat_prec) || !vp(x_prec) || !vp(out_prec) || (!out && !prod))
    return MPMG_EINVAL;
  if (rows == 0) return MPMG_OK;
  return rc(by_prec(x_prec, [&](auto cp) -> cudaError_t {
    return by_prec(mat_prec, [&](auto mp) -> cudaError_t {
      return by_prec(out_prec, [&](auto op) -> cudaError_t {
        return by_pol(policy, [&](auto ft, auto fm) -> cudaError_t {
          k_ell_transfer<decltype(cp)::value, decltype(mp)::value, decltype(op)::value, decltype(ft)::value,
                         decltype(fm)::value>
              <<<nb(rows), kT, 0, (cudaStream_t)stream>>>(rows, rw, col, val, x, scale_dev, divide, out, prod);
          return cudaGetLastError();
        });
      });
    });
  }));
}

int mpmg_gpu_ell_update_rc(int64_t rows, int32_t rw, const int32_t* col, const double* val, const void* c,
                           int32_t c_prec, double* r, double* u, const double* alpha_dev, uint32_t policy,
                           void* stream) {
  clear_stale_error();
  if (rows < 0 || rw < 1 || !col || !val || !c || !vp(c_prec) || !r || !u || !alpha_dev) return MPMG_EINVAL;
  if (rows == 0) return MPMG_OK;
  return rc(by_prec(c_prec, [&](auto cp) -> cudaError_t {
    constexpr int C = decltype(cp)::value;
    if (policy & MPMG_FMA)
      k_ell_update<C, true><<<nb(rows), kT, 0, (cudaStream_t)stream>>>(rows, rw, col, val, c, r, u, alpha_dev);
    else
      k_ell_update<C, false><<<nb(rows), kT, 0, (cudaStream_t)stream>>>(rows, rw, col, val, c, r, u, alpha_dev);
    return cudaGetLastError();
  }));
}

int mpmg_gpu_cast(int64_t n, const void* x, int32_t x_prec, void* out, int32_t out_prec, const double* scale_dev,
                  double scale, uint32_t policy, void* stream) {
  clear_stale_error();
  if (n < 0 || !x || !out || !vp(x_prec) || !vp(out_prec)) return MPMG_EINVAL;
  if (!scale_dev && !(scale > 0.0 && scale < INFINITY)) return MPMG_EINVAL;  // kernels.cpp:345
  if (n == 0) return MPMG_OK;
  const bool ftz = policy & MPMG_FTZ;
  return rc(by_prec(x_prec, [&](auto xp) -> cudaError_t {
    return by_prec(out_prec, [&](auto op) -> cudaError_t {
      constexpr int X = decltype(xp)::value, O = decltype(op)::value;
      if (ftz) k_cast<X, O, true><<<nb(n), kT, 0, (cudaStream_t)stream>>>(n, x, out, scale_dev, scale);
      else k_cast<X, O, false><<<nb(n), kT, 0, (cudaStream_t)stream>>>(n, x, out, scale_dev, scale);
      return cudaGetLastError();
    });
  }));
}

int mpmg_gpu_dot_seq(int64_t n, const void* x, int32_t x_prec, const void* y, int32_t y_prec, double* out_dev,
                     int32_t take_sqrt, void* stream) {
  clear_stale_error();
  if (n < 0 || !x || !y || !out_dev || !vp(x_prec) || !vp(y_prec)) return MPMG_EINVAL;
  return rc(by_prec(x_prec, [&](auto xp) -> cudaError_t {
    return by_prec(y_prec, [&](auto yp) -> cudaError_t {
      k_dot_seq<decltype(xp)::value, decltype(yp)::value><<<1, 1, 0, (cudaStream_t)stream>>>(n, x, y, out_dev,
                                                                                            take_sqrt);
      return cudaGetLastError();
    });
  }));
}

int mpmg_gpu_find_nonfinite(int64_t n, const void* x, int32_t x_prec, int64_t* index, void* stream) {
  clear_stale_error();
  if (n < 0 || !x || !vp(x_prec) || !index) return MPMG_EINVAL;
  *index = -1;
  if (n == 0) return MPMG_OK;
  const cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, 8, s);
  const unsigned long long init = (unsigned long long)n;
  if (e == cudaSuccess) e = cudaMemcpyAsync(d, &init, 8, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = by_prec(x_prec, [&](auto xp) -> cudaError_t {
      k_find_nonfinite<decltype(xp)::value><<<nb(n), kT, 0, s>>>(n, x, d);
      return cudaGetLastError();
    });
  unsigned long long first = init;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&first, d, 8, cudaMemcpyDeviceToHost, s);
  if (d) {
    const cudaError_t ef = cudaFreeAsync(d, s);
    if (e == cudaSuccess) e = ef;
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return rc(e);
  *index = first < init ? (int64_t)first : -1;
  return MPMG_OK;
}

}  // extern "C"
