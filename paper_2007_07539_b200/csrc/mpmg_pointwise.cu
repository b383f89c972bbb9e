// Pointwise and grid-transfer kernels of the hot path:
//   * layout conversion compact <-> padded (mesh_fem.hpp:43-50 ordering),
//   * first Jacobi step from u = 0 (multigrid.cpp:376 + 79-89),
//   * full-weighting restriction with precision change (multigrid.cpp:236-268),
//   * prolongation + correction (multigrid.cpp:270-280, 389-390),
//   * scaled FP64 -> FP16/FP32 downcast (kernels.cpp:343-360),
//   * deterministic two-stage FP64 norm (replaces kernels.cpp:384-395).
#include <algorithm>

#include "mpmg_arith.cuh"
#include "mpmg_internal.h"

namespace mpmg_impl {

using namespace mpmg_dev;

namespace {

constexpr int kThreads = 256;

inline bool aligned64(const void* p) { return ((uintptr_t)p & 63u) == 0; }

// one thread per 8 values, at most ~8 waves of 256-thread CTAs per SM
inline unsigned grid8(size_t len) {
  const size_t groups = len / 8 + 1;
  return (unsigned)std::max<size_t>(1, std::min<size_t>((groups + kThreads - 1) / kThreads, 148u * 64u));
}

inline unsigned blocks_for(size_t n, int per_thread = 1) {
  const size_t t = (n + (size_t)per_thread - 1) / per_thread;
  return (unsigned)std::max<size_t>(1, (t + kThreads - 1) / kThreads);
}

template <int PREC> struct St;
template <> struct St<P16> { using T = __half; };
template <> struct St<P32> { using T = float; };
template <> struct St<P64> { using T = double; };

// padded index of interior point i of the compact ordering
__device__ __forceinline__ long long padded_index(long long i, int dim, int P) {
  const long long m = P - 1;
  const long long x = i % m + 1;
  if (dim == 2) return (i / m + 1) * P + x;
  const long long y = (i / m) % m + 1, z = i / (m * m) + 1;
  return (z * P + y) * (long long)P + x;
}

template <typename T>
__global__ void k_pack(const T* __restrict__ src, T* __restrict__ dst, long long n, int dim, int P, int unpack) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long p = padded_index(i, dim, P);
  if (unpack) dst[i] = src[p];
  else dst[p] = src[i];
}

// u = round(omega * round(D^-1 * b)) == one Jacobi step from zero, bitwise:
// t = A*0 = +0; r = fma(-1, +0, b) = b; t = d*b; u = fma(w, t, +0).
template <int PREC, bool FTZ, bool FMA>
__global__ void k_jacobi_zero(const void* __restrict__ bv, void* __restrict__ uv, long long len, double w,
                              double d) {
  pdl_wait();
  pdl_launch();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= len) return;
  if constexpr (PREC == P16) {
    const __half b = static_cast<const __half*>(bv)[i];
    const __half t = mul16s<FTZ>(__double2half(d), b);
    static_cast<__half*>(uv)[i] = fma16s<FTZ, FMA>(__double2half(w), t, __ushort_as_half((unsigned short)0));
  } else if constexpr (PREC == P32) {
    const float b = static_cast<const float*>(bv)[i];
    const float t = mul32<FTZ>((float)d, b);
    static_cast<float*>(uv)[i] = fma32<FTZ, FMA>((float)w, t, 0.0f);
  } else {
    const double b = static_cast<const double*>(bv)[i];
    static_cast<double*>(uv)[i] = fma64<FMA>(w, mul64(d, b), 0.0);
  }
}

// transfer_product<P> single step (multigrid.cpp:166-195). The weights are
// 2^-k (k = number of straddled dimensions), built exactly in the compute
// precision by exponent arithmetic -- no runtime conversion per product.
template <int CP, bool FTZ, bool FMA> struct Xfer;
template <bool FTZ, bool FMA> struct Xfer<P16, FTZ, FMA> {
  using T = __half;
  static __device__ __forceinline__ T zero() { return __ushort_as_half((unsigned short)0); }
  static __device__ __forceinline__ T weight(int k) { return __ushort_as_half((unsigned short)(0x3C00 - (k << 10))); }
  static __device__ __forceinline__ T step(T w, T x, T acc) { return fma16s<FTZ, FMA>(w, x, acc); }
  static __device__ __forceinline__ double wide(T v) { return (double)__half2float(v); }
};
template <bool FTZ, bool FMA> struct Xfer<P32, FTZ, FMA> {
  using T = float;
  static __device__ __forceinline__ T zero() { return 0.0f; }
  static __device__ __forceinline__ T weight(int k) { return __int_as_float(0x3F800000 - (k << 23)); }
  // multigrid.cpp:178-184: the unfused form rounds the product to binary32
  // and flushes only the sum
  static __device__ __forceinline__ T step(T w, T x, T acc) {
    return f32<FTZ>(FMA ? __fmaf_rn(w, x, acc) : __fadd_rn(__fmul_rn(w, x), acc));
  }
  static __device__ __forceinline__ double wide(T v) { return (double)v; }
};
template <bool FTZ, bool FMA> struct Xfer<P64, FTZ, FMA> {
  using T = double;
  static __device__ __forceinline__ T zero() { return 0.0; }
  static __device__ __forceinline__ T weight(int k) {
    return __longlong_as_double(0x3FF0000000000000LL - ((long long)k << 52));
  }
  static __device__ __forceinline__ T step(T w, T x, T acc) { return fma64<FMA>(w, x, acc); }
  static __device__ __forceinline__ double wide(T v) { return v; }
};

template <int P, bool FTZ> __device__ __forceinline__ typename St<P>::T store_round(double v);
template <> __device__ __forceinline__ __half store_round<P16, true>(double v) { return round16<true>(v); }
template <> __device__ __forceinline__ __half store_round<P16, false>(double v) { return round16<false>(v); }
template <> __device__ __forceinline__ float store_round<P32, true>(double v) { return round32<true>(v); }
template <> __device__ __forceinline__ float store_round<P32, false>(double v) { return round32<false>(v); }
template <> __device__ __forceinline__ double store_round<P64, true>(double v) { return v; }
template <> __device__ __forceinline__ double store_round<P64, false>(double v) { return v; }

// restriction: one thread per coarse interior node (cx,cy,cz); 3^dim fine
// neighbours of (2cx,2cy,2cz) in lexicographic order with weights
// prod_d (d == 0 ? 1 : 1/2) (mesh_fem.cpp:266-293).
template <int DIM, int FP, int CPc, bool FTZ, bool FMA>
__global__ void k_restrict(const void* __restrict__ rf_, void* __restrict__ rc_, int Pc, const double* scale_dev,
                           int zoff = 0) {
  pdl_wait();
  pdl_launch();
  using X = Xfer<FP, FTZ, FMA>;
  using TF = typename X::T;
  const TF* rf = static_cast<const TF*>(rf_);
  const int cx = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int cy = blockIdx.y * blockDim.y + threadIdx.y + 1;
  const int cz = DIM == 3 ? (int)blockIdx.z + 1 : 0;
  if (cx > Pc - 1 || cy > Pc - 1) return;
  const int Pf = 2 * Pc;
  const long long pf = DIM == 3 ? (long long)Pf * Pf : (long long)Pf;
  TF acc = X::zero();
  // fine plane of coarse (local) plane cz: 2 cz + zoff (zoff = 0 for a whole
  // level; for z-slabs the local plane numbering of the two levels differs)
  const long long cf = (DIM == 3 ? (long long)(2 * cz + zoff) * pf : 0) + (long long)(2 * cy) * Pf + 2 * cx;
#pragma unroll
  for (int dz = (DIM == 3 ? -1 : 0); dz <= (DIM == 3 ? 1 : 0); ++dz)
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        acc = X::step(X::weight((dx != 0) + (dy != 0) + (dz != 0)), rf[cf + dz * pf + (long long)dy * Pf + dx], acc);
      }
  const long long ci = (DIM == 3 ? (long long)cz * Pc * Pc : 0) + (long long)cy * Pc + cx;
  if constexpr (FP == CPc) {
    if (!scale_dev) {  // same precision, scale 1: the cast is the identity
      static_cast<TF*>(rc_)[ci] = acc;
      return;
    }
  }
  const double s = scale_dev ? *scale_dev : 1.0;
  static_cast<typename St<CPc>::T*>(rc_)[ci] = store_round<CPc, FTZ>(X::wide(acc) / s);
}

// prolongation + correction: one thread per fine interior node; parents per
// dimension: even j -> j/2 (w 1), odd -> (j-1)/2, (j+1)/2 (w 1/2), z-parent
// outermost (mesh_fem.cpp:222-252). Boundary parents read the stored zeros.
template <int DIM, int FP, int CPc, bool FTZ, bool FMA>
__global__ void k_prolong(const void* __restrict__ cc_, void* __restrict__ uf_, int Pf, const double* scale_dev) {
  pdl_wait();
  pdl_launch();
  using X = Xfer<CPc, FTZ, FMA>;
  using TC = typename X::T;
  const TC* cc = static_cast<const TC*>(cc_);
  const int fx = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int fy = blockIdx.y * blockDim.y + threadIdx.y + 1;
  const int fz = DIM == 3 ? (int)blockIdx.z + 1 : 0;
  if (fx > Pf - 1 || fy > Pf - 1) return;
  const int Pc = Pf / 2;
  int px[2], py[2], pz[2];
  const int nx = (fx & 1) ? 2 : 1, ny = (fy & 1) ? 2 : 1, nz = DIM == 3 ? ((fz & 1) ? 2 : 1) : 1;
  px[0] = fx >> 1; px[1] = (fx + 1) >> 1;
  py[0] = fy >> 1; py[1] = (fy + 1) >> 1;
  pz[0] = fz >> 1; pz[1] = (fz + 1) >> 1;
  TC acc = X::zero();
  for (int c = 0; c < nz; ++c)
    for (int b = 0; b < ny; ++b)
      for (int a = 0; a < nx; ++a) {
        const long long ci = (DIM == 3 ? (long long)pz[c] * Pc * Pc : 0) + (long long)py[b] * Pc + px[a];
        acc = X::step(X::weight((fx & 1) + (fy & 1) + (DIM == 3 ? (fz & 1) : 0)), cc[ci], acc);
      }
  const double s = scale_dev ? *scale_dev : 1.0;
  const double v = X::wide(acc) * s;
  const long long fi = (DIM == 3 ? (long long)fz * Pf * Pf : 0) + (long long)fy * Pf + fx;
  using TF = typename St<FP>::T;
  TF* uf = static_cast<TF*>(uf_);
  const TF t = store_round<FP, FTZ>(v);
  if constexpr (FP == P16) uf[fi] = fma16s<FTZ, FMA>(__ushort_as_half((unsigned short)0x3C00), t, uf[fi]);
  else if constexpr (FP == P32) uf[fi] = fma32<FTZ, FMA>(1.0f, t, uf[fi]);
  else uf[fi] = fma64<FMA>(1.0, t, uf[fi]);
}

// out = round_prec(x / s), s = (scale_enabled && alpha > 0) ? alpha : 1
template <int PREC, bool FTZ>
__global__ void k_downcast(const double* __restrict__ x, void* __restrict__ out, long long len,
                           const double* alpha, int scale_enabled) {
  pdl_wait();
  pdl_launch();
  const double a = *alpha;
  const double s = (scale_enabled && a > 0.0) ? a : 1.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x)
    static_cast<typename St<PREC>::T*>(out)[i] = store_round<PREC, FTZ>(__ddiv_rn(x[i], s));
}

// ---- vectorized forms: 8 consecutive values per thread (16-byte binary16 /
// 32-byte binary32 / 64-byte binary64 accesses); same arithmetic as above.
template <int PREC> struct V8;
template <> struct V8<P16> {
  __half2 h[4];
  __device__ __forceinline__ void load(const void* p, long long i) {
    const uint4 q = *reinterpret_cast<const uint4*>(static_cast<const __half*>(p) + i);
    h[0] = u2h(q.x); h[1] = u2h(q.y); h[2] = u2h(q.z); h[3] = u2h(q.w);
  }
  __device__ __forceinline__ void store(void* p, long long i) const {
    *reinterpret_cast<uint4*>(static_cast<__half*>(p) + i) = make_uint4(h2u(h[0]), h2u(h[1]), h2u(h[2]), h2u(h[3]));
  }
  __device__ __forceinline__ __half get(int e) const { return e & 1 ? __high2half(h[e >> 1]) : __low2half(h[e >> 1]); }
  __device__ __forceinline__ void set(int e, __half v) {
    h[e >> 1] = e & 1 ? __halves2half2(__low2half(h[e >> 1]), v) : __halves2half2(v, __high2half(h[e >> 1]));
  }
};
template <> struct V8<P32> {
  float v[8];
  __device__ __forceinline__ void load(const void* p, long long i) {
    const float4* q = reinterpret_cast<const float4*>(static_cast<const float*>(p) + i);
    const float4 a = q[0], b = q[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  __device__ __forceinline__ void store(void* p, long long i) const {
    float4* q = reinterpret_cast<float4*>(static_cast<float*>(p) + i);
    q[0] = make_float4(v[0], v[1], v[2], v[3]);
    q[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
  __device__ __forceinline__ float get(int e) const { return v[e]; }
  __device__ __forceinline__ void set(int e, float x) { v[e] = x; }
};
template <> struct V8<P64> {
  double v[8];
  __device__ __forceinline__ void load(const void* p, long long i) {
    const double2* q = reinterpret_cast<const double2*>(static_cast<const double*>(p) + i);
#pragma unroll
    for (int k = 0; k < 4; ++k) { const double2 a = q[k]; v[2 * k] = a.x; v[2 * k + 1] = a.y; }
  }
  __device__ __forceinline__ void store(void* p, long long i) const {
    double2* q = reinterpret_cast<double2*>(static_cast<double*>(p) + i);
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = make_double2(v[2 * k], v[2 * k + 1]);
  }
  __device__ __forceinline__ double get(int e) const { return v[e]; }
  __device__ __forceinline__ void set(int e, double x) { v[e] = x; }
};

// downcast of n8 groups of 8 values (len - 8*n8 tail done by block 0)
// x / s correctly rounded without a per-element division (the scale is one
// scalar for the whole vector): y = RN(1/s), q = RN(x y), e = x - s q (exact
// via fma), q' = RN(q + e y). With y the correctly rounded reciprocal this is
// the correctly rounded quotient (Markstein's theorem), bitwise equal to
// __ddiv_rn -- checked exhaustively-by-sample in tests/test_gpu_parity.py.
__device__ __forceinline__ double div_by(double x, double s, double y) {
  const double q = __dmul_rn(x, y);
  const double e = __fma_rn(-s, q, x);
  return __fma_rn(e, y, q);
}

template <int PREC, bool FTZ>
__global__ void k_downcast8(const double* __restrict__ x, void* __restrict__ out, long long len,
                            const double* alpha, int scale_enabled) {
  pdl_wait();
  pdl_launch();
  const double a = *alpha;
  const double s = (scale_enabled && a > 0.0) ? a : 1.0;
  const double y = __drcp_rn(s);
  const long long n8 = len / 8;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n8; g += (long long)gridDim.x * blockDim.x) {
    V8<P64> in;
    in.load(x, 8 * g);
    V8<PREC> o;
#pragma unroll
    for (int e = 0; e < 8; ++e) o.set(e, store_round<PREC, FTZ>(s == 1.0 ? in.get(e) : div_by(in.get(e), s, y)));
    o.store(out, 8 * g);
  }
  if (blockIdx.x == 0 && threadIdx.x < len - 8 * n8) {
    const long long i = 8 * n8 + threadIdx.x;
    static_cast<typename St<PREC>::T*>(out)[i] = store_round<PREC, FTZ>(__ddiv_rn(x[i], s));
  }
}

template <int PREC, bool FTZ, bool FMA>
__device__ __forceinline__ typename St<PREC>::T jz_one(typename St<PREC>::T b, double w, double d) {
  if constexpr (PREC == P16) {
    const __half t = mul16s<FTZ>(__double2half(d), b);
    return fma16s<FTZ, FMA>(__double2half(w), t, __ushort_as_half((unsigned short)0));
  } else if constexpr (PREC == P32) {
    return fma32<FTZ, FMA>((float)w, mul32<FTZ>((float)d, b), 0.0f);
  } else {
    return fma64<FMA>(w, mul64(d, b), 0.0);
  }
}

template <int PREC, bool FTZ, bool FMA>
__global__ void k_jacobi_zero8(const void* __restrict__ bv, void* __restrict__ uv, long long len, double w, double d) {
  pdl_wait();
  pdl_launch();
  const long long n8 = len / 8;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n8; g += (long long)gridDim.x * blockDim.x) {
    V8<PREC> b;
    b.load(bv, 8 * g);
    V8<PREC> u;
#pragma unroll
    for (int e = 0; e < 8; ++e) u.set(e, jz_one<PREC, FTZ, FMA>(b.get(e), w, d));
    u.store(uv, 8 * g);
  }
  if (blockIdx.x == 0 && threadIdx.x < len - 8 * n8) {
    const long long i = 8 * n8 + threadIdx.x;
    using T = typename St<PREC>::T;
    static_cast<T*>(uv)[i] = jz_one<PREC, FTZ, FMA>(static_cast<const T*>(bv)[i], w, d);
  }
}

template <typename T>
__device__ __forceinline__ void ldg4(const T* p, T* out) {
  if constexpr (sizeof(T) == 2) {
    const uint2 q = __ldg(reinterpret_cast<const uint2*>(p));
    out[0] = __ushort_as_half((unsigned short)(q.x & 0xFFFFu));
    out[1] = __ushort_as_half((unsigned short)(q.x >> 16));
    out[2] = __ushort_as_half((unsigned short)(q.y & 0xFFFFu));
    out[3] = __ushort_as_half((unsigned short)(q.y >> 16));
  } else if constexpr (sizeof(T) == 4) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p));
    out[0] = q.x; out[1] = q.y; out[2] = q.z; out[3] = q.w;
  } else {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p)), b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    out[0] = a.x; out[1] = a.y; out[2] = b.x; out[3] = b.y;
  }
}

// prolongation + correction, 8 consecutive fine x per thread (Pf % 8 == 0);
// same parent order and rounding as k_prolong
template <int DIM, int FP, int CPc, bool FTZ, bool FMA>
__global__ void k_prolong8(const void* __restrict__ cc_, void* __restrict__ uf_, int Pf, const double* scale_dev,
                           int zf_lo = 1, int zc_lo = 1) {
  pdl_wait();
  pdl_launch();
  using X = Xfer<CPc, FTZ, FMA>;
  using TC = typename X::T;
  const TC* cc = static_cast<const TC*>(cc_);
  const int groups = Pf / 8;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= groups * (Pf - 1)) return;
  const int fy = g / groups + 1;
  const int x0 = (g % groups) * 8;
  const int fz = DIM == 3 ? (int)blockIdx.y + 1 : 0;  // local plane
  const int gz = fz + zf_lo - 1;                       // global plane (parity, parents)
  const int Pc = Pf / 2;
  const int ny = (fy & 1) ? 2 : 1, nz = DIM == 3 ? ((gz & 1) ? 2 : 1) : 1;
  const int py[2] = {fy >> 1, (fy + 1) >> 1};
  const int pz[2] = {(gz >> 1) - zc_lo + 1, ((gz + 1) >> 1) - zc_lo + 1};
  // coarse values x0/2 .. x0/2+4 of each parent row
  TC c[2][2][5];
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (k < nz && j < ny) {
        const long long base = (DIM == 3 ? (long long)pz[k] * Pc * Pc : 0) + (long long)py[j] * Pc + x0 / 2;
        // x0/2 is a multiple of 4: one aligned 4-value load + one scalar
        // (x0/2 + 4 <= Pc always; index Pc is the row's aliased zero ghost)
        ldg4<TC>(cc + base, c[k][j]);
        c[k][j][4] = __ldg(cc + base + 4);
      }
    }
  const double s = scale_dev ? *scale_dev : 1.0;
  const bool unit = !scale_dev;
  const long long fi = (DIM == 3 ? (long long)fz * Pf * Pf : 0) + (long long)fy * Pf + x0;
  V8<FP> u;
  u.load(uf_, fi);
  if constexpr (FP == P16 && CPc == P16) {
    if (unit) {
      // binary16, unit scale: fine pairs (2j, 2j+1) in one half2. Per parent
      // row the even node takes w c_j, the odd one (w/2) c_j then (w/2)
      // c_{j+1} -- the same per-node order as below; the even lane's extra
      // fma(0, c, acc) leaves acc unchanged (up to the sign of a zero)
      const int kyz = (fy & 1) + (DIM == 3 ? (gz & 1) : 0);
      const __half2 w1 = __halves2half2(X::weight(kyz), X::weight(kyz + 1));
      const __half2 w2 = __halves2half2(__ushort_as_half((unsigned short)0), X::weight(kyz + 1));
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        __half2 acc = u2h(0u);
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (k < nz && j < ny) {
              acc = fma16<FTZ, FMA>(w1, __half2half2(c[k][j][p]), acc);
              acc = fma16<FTZ, FMA>(w2, __half2half2(c[k][j][p + 1]), acc);
            }
        u.h[p] = fma16<FTZ, FMA>(u2h(0x3C003C00u), acc, u.h[p]);  // axpy(1, t, u)
      }
      if (x0 == 0) u.set(0, __ushort_as_half((unsigned short)0));  // ghost node
      u.store(uf_, fi);
      return;
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int fx = x0 + e;
    if (fx == 0) continue;  // ghost node stays zero
    const int nx = (fx & 1) ? 2 : 1;
    const auto wk = X::weight((fx & 1) + (fy & 1) + (DIM == 3 ? (gz & 1) : 0));
    const int px0 = (fx >> 1) - x0 / 2;
    TC acc = X::zero();
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int a = 0; a < 2; ++a)
          if (k < nz && j < ny && a < nx) acc = X::step(wk, c[k][j][px0 + a], acc);
    typename St<FP>::T t;
    if constexpr (FP == CPc) t = unit ? acc : store_round<FP, FTZ>(X::wide(acc) * s);
    else t = store_round<FP, FTZ>(X::wide(acc) * s);
    if constexpr (FP == P16) u.set(e, fma16s<FTZ, FMA>(__ushort_as_half((unsigned short)0x3C00), t, u.get(e)));
    else if constexpr (FP == P32) u.set(e, fma32<FTZ, FMA>(1.0f, t, u.get(e)));
    else u.set(e, fma64<FMA>(1.0, t, u.get(e)));
  }
  u.store(uf_, fi);
}

// restriction, 4 consecutive coarse x per thread (Pc % 4 == 0, no scale,
// same precision on both levels): each fine row segment 8g-1 .. 8g+7 is one
// aligned 8-value vector load plus one scalar, shared by the 4 outputs;
// per-output slot order (dz, dy, dx) as k_restrict. zoff as in k_restrict.
template <int DIM, int FP, bool FTZ, bool FMA>
__global__ void k_restrict4(const void* __restrict__ rf_, void* __restrict__ rc_, int Pc, int zoff, int nzc) {
  pdl_wait();
  pdl_launch();
  using X = Xfer<FP, FTZ, FMA>;
  using T = typename X::T;
  const int groups = Pc / 4;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per_plane = (long long)groups * (Pc - 1);
  if (tid >= per_plane * (DIM == 3 ? nzc : 1)) return;
  const int cz = DIM == 3 ? (int)(tid / per_plane) + 1 : 0;
  const int rem = (int)(tid % per_plane);
  const int cy = rem / groups + 1;
  const int g = rem % groups;
  const int Pf = 2 * Pc;
  const long long pf = (long long)Pf * Pf;
  const T* rf = static_cast<const T*>(rf_);
  T acc[4];
#pragma unroll
  for (int o = 0; o < 4; ++o) acc[o] = X::zero();
#pragma unroll
  for (int dz = (DIM == 3 ? -1 : 0); dz <= (DIM == 3 ? 1 : 0); ++dz)
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const long long row = (DIM == 3 ? (long long)(2 * cz + zoff + dz) * pf : 0) + (long long)(2 * cy + dy) * Pf;
      V8<FP> v;
      v.load(rf, row + 8 * g);
      const T left = g > 0 ? rf[row + 8 * g - 1] : X::zero();
#pragma unroll
      for (int o = 0; o < 4; ++o)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
          const int e = 2 * o + dx;  // fine offset within the segment
          const T x = e < 0 ? left : v.get(e);
          acc[o] = X::step(X::weight((dx != 0) + (dy != 0) + (dz != 0)), x, acc[o]);
        }
    }
  if (g == 0) acc[0] = X::zero();  // cx = 0 is the boundary ghost
  T* rc = static_cast<T*>(rc_) + (DIM == 3 ? (long long)cz * Pc * Pc : 0) + (long long)cy * Pc + 4 * g;
#pragma unroll
  for (int o = 0; o < 4; ++o) rc[o] = acc[o];
}

// deterministic per-block partial sums of x_i^2 (fixed grid, fixed order)
__global__ void k_sumsq(const double* __restrict__ x, long long len, double* partials) {
  __shared__ double red[kThreads / 32];
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x)
    acc = __fma_rn(x[i], x[i], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    partials[blockIdx.x] = s;
  }
}

// r = b and per-block sums of b_i^2: the initial defect b - A u for u = 0
// (ir_solver.cpp:92-93) bitwise -- t = A 0 = +0 and fma(-1, +0, b) = b for
// every b including signed zeros -- at 16 instead of 24 bytes per unknown
__global__ void k_copy_sumsq(const double* __restrict__ x, double* __restrict__ y, long long len,
                             double* partials) {
  __shared__ double red[kThreads / 32];
  double acc = 0.0;
  const long long n2 = len / 2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
    const double2 v = reinterpret_cast<const double2*>(x)[i];
    reinterpret_cast<double2*>(y)[i] = v;
    acc = __fma_rn(v.x, v.x, acc);
    acc = __fma_rn(v.y, v.y, acc);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (len & 1)) {
    const double v = x[len - 1];
    y[len - 1] = v;
    acc = __fma_rn(v, v, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    partials[blockIdx.x] = s;
  }
}

__global__ void k_finalize(const double* __restrict__ partials, int n, double* out, int take_sqrt = 1) {
  __shared__ double red[kThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += kThreads) acc += partials[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = take_sqrt ? sqrt(red[0]) : red[0];
}

// SplitMix64 U[0,1) initial guess (ir_solver.cpp:80-84, rng.hpp:13-25): the
// k-th interior node (compact order) receives the k-th draw.
__global__ void k_random01(double* u, long long n, int dim, int P, uint64_t seed) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t z = seed + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  u[padded_index(i, dim, P)] = (double)(z >> 11) * 0x1.0p-53;
}

template <typename F>
cudaError_t with_ftz_fma(uint32_t policy, F&& f) {
  const bool ftz = policy & MPMG_FTZ, fma = policy & MPMG_FMA;
  if (ftz && fma) return f(std::true_type{}, std::true_type{});
  if (ftz) return f(std::true_type{}, std::false_type{});
  if (fma) return f(std::false_type{}, std::true_type{});
  return f(std::false_type{}, std::false_type{});
}

template <typename F>
cudaError_t with_prec(int prec, F&& f) {
  switch (prec) {
    case MPMG_FP16: return f(std::integral_constant<int, P16>{});
    case MPMG_FP32: return f(std::integral_constant<int, P32>{});
    default: return f(std::integral_constant<int, P64>{});
  }
}

}  // namespace

cudaError_t launch_pack(int dim, int nodes, int prec, const void* compact, void* padded, bool unpack,
                        cudaStream_t s) {
  const size_t n = mpmg_interior_len(dim, nodes);
  if (n == 0) return cudaSuccess;
  const int P = pitch(nodes);
  return with_prec(prec, [&](auto pc) -> cudaError_t {
    using T = typename St<decltype(pc)::value>::T;
    if (unpack)
      k_pack<T><<<blocks_for(n), kThreads, 0, s>>>(static_cast<const T*>(padded), static_cast<T*>(const_cast<void*>(compact)),
                                                    (long long)n, dim, P, 1);
    else
      k_pack<T><<<blocks_for(n), kThreads, 0, s>>>(static_cast<const T*>(compact), static_cast<T*>(padded), (long long)n,
                                                    dim, P, 0);
    return cudaGetLastError();
  });
}

cudaError_t launch_jacobi_zero(int dim, int nodes, int prec, const void* b, void* u, double omega_r,
                               double invdiag_r, uint32_t policy, cudaStream_t s) {
  return launch_jacobi_zero_len(mpmg_padded_len(dim, nodes), prec, b, u, omega_r, invdiag_r, policy, s);
}

cudaError_t launch_jacobi_zero_len(size_t len, int prec, const void* b, void* u, double omega_r, double invdiag_r,
                                   uint32_t policy, cudaStream_t s) {
  const bool vec = aligned64(b) && aligned64(u);
  return with_prec(prec, [&](auto pc) -> cudaError_t {
    return with_ftz_fma(policy, [&](auto ft, auto fm) -> cudaError_t {
      constexpr int PR = decltype(pc)::value;
      constexpr bool T = decltype(ft)::value, M = decltype(fm)::value;
      cudaError_t e;
      if (vec)
        e = launch_pdl(k_jacobi_zero8<PR, T, M>, dim3(grid8(len)), dim3(kThreads), 0, s, b, u, (long long)len, omega_r, invdiag_r);
      else
        e = launch_pdl(k_jacobi_zero<PR, T, M>, dim3(blocks_for(len)), dim3(kThreads), 0, s, b, u, (long long)len, omega_r, invdiag_r);
      return e;
    });
  });
}

cudaError_t launch_restrict(int dim, int fine_nodes, int fine_prec, int coarse_prec, const void* r_fine,
                            void* r_coarse, const double* scale_dev, uint32_t policy, cudaStream_t s) {
  const int Pc = pitch(fine_nodes) / 2;
  if (Pc < 2) return cudaSuccess;
  const dim3 block(32, 8);
  const dim3 grid((Pc - 1 + 31) / 32, (Pc - 1 + 7) / 8, dim == 3 ? Pc - 1 : 1);
  if (!scale_dev && fine_prec == coarse_prec && Pc % 4 == 0 && Pc >= 8 && aligned64(r_fine)) {
    const long long n = (long long)(Pc / 4) * (Pc - 1) * (dim == 3 ? Pc - 1 : 1);
    const unsigned blocks = (unsigned)((n + kThreads - 1) / kThreads);
    return with_prec(fine_prec, [&](auto fp) -> cudaError_t {
      return with_ftz_fma(policy, [&](auto ft, auto fm) -> cudaError_t {
        constexpr int F = decltype(fp)::value;
        constexpr bool T = decltype(ft)::value, M = decltype(fm)::value;
        if (dim == 3) return launch_pdl(k_restrict4<3, F, T, M>, dim3(blocks), dim3(kThreads), 0, s, r_fine, r_coarse, Pc, 0, Pc - 1);
        return launch_pdl(k_restrict4<2, F, T, M>, dim3(blocks), dim3(kThreads), 0, s, r_fine, r_coarse, Pc, 0, 1);
      });
    });
  }
  return with_prec(fine_prec, [&](auto fp) -> cudaError_t {
    return with_prec(coarse_prec, [&](auto cp) -> cudaError_t {
      return with_ftz_fma(policy, [&](auto ft, auto fm) -> cudaError_t {
        constexpr int F = decltype(fp)::value, Cc = decltype(cp)::value;
        constexpr bool T = decltype(ft)::value, M = decltype(fm)::value;
        if (dim == 3) return launch_pdl(k_restrict<3, F, Cc, T, M>, grid, block, 0, s, r_fine, r_coarse, Pc, scale_dev, 0);
        return launch_pdl(k_restrict<2, F, Cc, T, M>, grid, block, 0, s, r_fine, r_coarse, Pc, scale_dev, 0);
      });
    });
  });
}

cudaError_t launch_prolong(int dim, int fine_nodes, int fine_prec, int coarse_prec, const void* c_coarse,
                           void* u_fine, const double* scale_dev, uint32_t policy, cudaStream_t s) {
  const int Pf = pitch(fine_nodes);
  const dim3 block(32, 8);
  const dim3 grid((Pf - 1 + 31) / 32, (Pf - 1 + 7) / 8, dim == 3 ? Pf - 1 : 1);
  const bool vec = Pf % 8 == 0 && aligned64(u_fine) && ((uintptr_t)c_coarse & 15u) == 0;
  const dim3 grid8v((unsigned)(((Pf / 8) * (Pf - 1) + kThreads - 1) / kThreads), dim == 3 ? Pf - 1 : 1);
  return with_prec(fine_prec, [&](auto fp) -> cudaError_t {
    return with_prec(coarse_prec, [&](auto cp) -> cudaError_t {
      return with_ftz_fma(policy, [&](auto ft, auto fm) -> cudaError_t {
        constexpr int F = decltype(fp)::value, Cc = decltype(cp)::value;
        constexpr bool T = decltype(ft)::value, M = decltype(fm)::value;
        if (vec) {
          if (dim == 3) return launch_pdl(k_prolong8<3, F, Cc, T, M>, grid8v, dim3(kThreads), 0, s, c_coarse, u_fine, Pf, scale_dev, 1, 1);
          return launch_pdl(k_prolong8<2, F, Cc, T, M>, grid8v, dim3(kThreads), 0, s, c_coarse, u_fine, Pf, scale_dev, 1, 1);
        }
        if (dim == 3) return launch_pdl(k_prolong<3, F, Cc, T, M>, grid, block, 0, s, c_coarse, u_fine, Pf, scale_dev);
        return launch_pdl(k_prolong<2, F, Cc, T, M>, grid, block, 0, s, c_coarse, u_fine, Pf, scale_dev);
      });
    });
  });
}

// z-slab transfers (3D): coarse local planes 1..nzc from fine slab planes
// (fine local plane 0 = the lower halo); prolongation of fine local planes
// 1..nzf from coarse local planes (coarse local nzc+1 = the upper halo)
cudaError_t launch_restrict_slab(int fine_nodes, const mpmg_slab& sf, const mpmg_slab& sc, int fine_prec,
                                 int coarse_prec, const void* r_fine, void* r_coarse, uint32_t policy,
                                 cudaStream_t s) {
  const int Pc = pitch(fine_nodes) / 2;
  if (Pc < 2 || sc.nz < 1) return cudaSuccess;
  const dim3 block(32, 8);
  const dim3 grid((Pc - 1 + 31) / 32, (Pc - 1 + 7) / 8, sc.nz);
  const int zoff = 2 * sc.z_lo - sf.z_lo - 1;
  if (fine_prec == coarse_prec && Pc % 4 == 0 && Pc >= 8 && aligned64(r_fine)) {
    const long long n = (long long)(Pc / 4) * (Pc - 1) * sc.nz;
    return with_prec(fine_prec, [&](auto fp) -> cudaError_t {
      return with_ftz_fma(policy, [&](auto ft, auto fm) -> cudaError_t {
        k_restrict4<3, decltype(fp)::value, decltype(ft)::value, decltype(fm)::value>
            <<<(unsigned)((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(r_fine, r_coarse, Pc, zoff, sc.nz);
        return cudaGetLastError();
      });
    });
  }
  return with_prec(fine_prec, [&](auto fp) -> cudaError_t {
    return with_prec(coarse_prec, [&](auto cp) -> cudaError_t {
      return with_ftz_fma(policy, [&](auto ft, auto fm) -> cudaError_t {
        k_restrict<3, decltype(fp)::value, decltype(cp)::value, decltype(ft)::value, decltype(fm)::value>
            <<<grid, block, 0, s>>>(r_fine, r_coarse, Pc, nullptr, zoff);
        return cudaGetLastError();
      });
    });
  });
}

cudaError_t launch_prolong_slab(int fine_nodes, const mpmg_slab& sf, const mpmg_slab& sc, int fine_prec,
                                int coarse_prec, const void* c_coarse, void* u_fine, uint32_t policy,
                                cudaStream_t s) {
  const int Pf = pitch(fine_nodes);
  if (Pf % 8 || !aligned64(u_fine) || ((uintptr_t)c_coarse & 15u) || sf.nz < 1) return cudaErrorInvalidValue;
  const dim3 grid8v((unsigned)(((Pf / 8) * (Pf - 1) + kThreads - 1) / kThreads), sf.nz);
  return with_prec(fine_prec, [&](auto fp) -> cudaError_t {
    return with_prec(coarse_prec, [&](auto cp) -> cudaError_t {
      return with_ftz_fma(policy, [&](auto ft, auto fm) -> cudaError_t {
        k_prolong8<3, decltype(fp)::value, decltype(cp)::value, decltype(ft)::value, decltype(fm)::value>
            <<<grid8v, kThreads, 0, s>>>(c_coarse, u_fine, Pf, nullptr, sf.z_lo, sc.z_lo);
        return cudaGetLastError();
      });
    });
  });
}

cudaError_t launch_downcast(int dim, int nodes, const double* x, void* out, int prec, const double* alpha_dev,
                            int scale_enabled, uint32_t policy, cudaStream_t s) {
  return launch_downcast_len(mpmg_padded_len(dim, nodes), x, out, prec, alpha_dev, scale_enabled, policy, s);
}

cudaError_t launch_downcast_len(size_t len, const double* x, void* out, int prec, const double* alpha_dev,
                                int scale_enabled, uint32_t policy, cudaStream_t s) {
  const unsigned blocks = std::min<unsigned>(blocks_for(len, 4), 148u * 16u);
  if (aligned64(x) && aligned64(out))
    return with_prec(prec, [&](auto pc) -> cudaError_t {
      if (policy & MPMG_FTZ)
        return launch_pdl(k_downcast8<decltype(pc)::value, true>, dim3(grid8(len)), dim3(kThreads), 0, s, x, out,
                          (long long)len, alpha_dev, scale_enabled);
      return launch_pdl(k_downcast8<decltype(pc)::value, false>, dim3(grid8(len)), dim3(kThreads), 0, s, x, out,
                        (long long)len, alpha_dev, scale_enabled);
    });
  return with_prec(prec, [&](auto pc) -> cudaError_t {
    if (policy & MPMG_FTZ)
      k_downcast<decltype(pc)::value, true><<<blocks, kThreads, 0, s>>>(x, out, (long long)len, alpha_dev, scale_enabled);
    else
      k_downcast<decltype(pc)::value, false><<<blocks, kThreads, 0, s>>>(x, out, (long long)len, alpha_dev, scale_enabled);
    return cudaGetLastError();
  });
}

template <int PREC>
__device__ __forceinline__ double widen(typename St<PREC>::T v) {
  if constexpr (PREC == P16) return (double)__half2float(v);
  else return (double)v;
}

// deferred corrections (mpmg_solver.cu): u_i = fma(a_k, c_k,i, u_i) for
// k = 0 .. *count + extra - 1 in slot order -- per element the exact sequence
// of the u half of update_residuum_correction (kernels.cpp:300-341), so u is
// bitwise what the per-iteration update would have produced
// uzero (optional device flag): u is still the zero initial guess -- start
// the chain from +0 instead of reading u (and write u even with no slot).
template <int PREC, bool FMA>
__global__ void k_fold8(double* __restrict__ u, const void* __restrict__ ring, long long ring_len,
                        const double* __restrict__ scales, const int* count, int extra, const int* gate,
                        long long len, const int* uzero) {
  pdl_wait();
  pdl_launch();
  if (gate && *gate == 0) return;
  const int n = *count + extra;
  const bool uz = uzero && *uzero;
  if (n <= 0 && !uz) return;
  using T = typename St<PREC>::T;
  const T* cr = static_cast<const T*>(ring);
  const long long n8 = len / 8;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n8; g += (long long)gridDim.x * blockDim.x) {
    V8<P64> acc;
    if (uz) {
#pragma unroll
      for (int e = 0; e < 8; ++e) acc.set(e, 0.0);
    } else {
      acc.load(u, 8 * g);
    }
    for (int k = 0; k < n; ++k) {
      const double a = scales[k];
      V8<PREC> c;
      c.load(cr + k * ring_len, 8 * g);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc.set(e, fma64<FMA>(a, widen<PREC>(c.get(e)), acc.get(e)));
    }
    acc.store(u, 8 * g);
  }
  if (blockIdx.x == 0 && threadIdx.x < len - 8 * n8) {
    const long long i = 8 * n8 + threadIdx.x;
    double v = uz ? 0.0 : u[i];
    for (int k = 0; k < n; ++k) v = fma64<FMA>(scales[k], widen<PREC>(cr[k * ring_len + i]), v);
    u[i] = v;
  }
}

cudaError_t launch_fold(size_t len, double* u, const void* ring, long long ring_len, int prec, const double* scales,
                        const int* count, int extra, const int* gate, bool fma, cudaStream_t s, const int* uzero) {
  if (!aligned64(u) || !aligned64(ring) || (ring_len * mpmg_bytes_per_value(prec)) % 64 != 0)
    return cudaErrorInvalidValue;
  return with_prec(prec, [&](auto pc) -> cudaError_t {
    constexpr int PR = decltype(pc)::value;
    // grid-stride over a few CTAs per SM: a gated-off launch retires in one wave
    const unsigned g = std::min<unsigned>(grid8(len), 148u * 4u);
    if (fma)
      return launch_pdl(k_fold8<PR, true>, dim3(g), dim3(kThreads), 0, s, u, ring, ring_len, scales, count, extra,
                        gate, (long long)len, uzero);
    return launch_pdl(k_fold8<PR, false>, dim3(g), dim3(kThreads), 0, s, u, ring, ring_len, scales, count, extra,
                      gate, (long long)len, uzero);
  });
}

int norm2_partials(size_t len) { return (int)std::min<unsigned>(blocks_for(len, 8), 148u * 8u); }

cudaError_t launch_norm2(size_t len, const double* x, double* partials, double* out, cudaStream_t s) {
  const int nb = norm2_partials(len);
  k_sumsq<<<nb, kThreads, 0, s>>>(x, (long long)len, partials);
  k_finalize<<<1, kThreads, 0, s>>>(partials, nb, out);
  return cudaGetLastError();
}

cudaError_t launch_copy_sumsq(size_t len, const double* x, double* y, double* partials, cudaStream_t s) {
  if (((uintptr_t)x & 15u) || ((uintptr_t)y & 15u)) return cudaErrorInvalidValue;
  k_copy_sumsq<<<norm2_partials(len), kThreads, 0, s>>>(x, y, (long long)len, partials);
  return cudaGetLastError();
}

cudaError_t launch_partials_sum(const double* partials, int n, double* out, cudaStream_t s) {
  k_finalize<<<1, kThreads, 0, s>>>(partials, n, out, 0);
  return cudaGetLastError();
}

cudaError_t launch_norm_finalize(const double* partials, int n, double* out, cudaStream_t s) {
  k_finalize<<<1, kThreads, 0, s>>>(partials, n, out);
  return cudaGetLastError();
}

cudaError_t launch_fill_random01(double* padded_u, int dim, int nodes, uint64_t seed, cudaStream_t s) {
  const size_t n = mpmg_interior_len(dim, nodes);
  if (n == 0) return cudaSuccess;
  k_random01<<<blocks_for(n), kThreads, 0, s>>>(padded_u, (long long)n, dim, pitch(nodes), seed);
  return cudaGetLastError();
}

}  // namespace mpmg_impl
