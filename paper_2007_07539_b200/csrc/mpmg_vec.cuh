// Per-lane value vectors for the streaming stencil kernels.
//
// A lane owns W consecutive x-values of one grid row: 8 bytes of binary16
// (W = 4, two half2), 16 bytes of binary32 (W = 4) or binary64 (W = 2), so
// every row load is one coalesced 64/128-bit access per lane. Values are
// held in a "compute" precision CP that may be wider than the storage
// precision (binary16 storage widened to binary32 for Fp16Accum::FP32, or to
// binary64 for the FP64 outer update).
#pragma once

#include "mpmg_arith.cuh"

namespace mpmg_dev {

template <int SP> struct LaneWidth;
template <> struct LaneWidth<P16> { static constexpr int W = 4; };
template <> struct LaneWidth<P32> { static constexpr int W = 4; };
template <> struct LaneWidth<P64> { static constexpr int W = 2; };

template <int CP, int W> struct Vec;
template <int W> struct Vec<P16, W> { __half2 h[W / 2]; };
template <int W> struct Vec<P32, W> { float v[W]; };
template <int W> struct Vec<P64, W> { double v[W]; };

template <int CP> struct Scalar;
template <> struct Scalar<P16> { using T = __half; };
template <> struct Scalar<P32> { using T = float; };
template <> struct Scalar<P64> { using T = double; };

template <int CP, int W>
__device__ __forceinline__ Vec<CP, W> vzero() {
  Vec<CP, W> r;
  if constexpr (CP == P16) {
#pragma unroll
    for (int i = 0; i < W / 2; ++i) r.h[i] = u2h(0u);
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = 0;
  }
  return r;
}

// ---- loads of W storage values (SP) at element index idx, widened to CP ----
template <int SP, int CP, int W>
__device__ __forceinline__ Vec<CP, W> vload(const void* base, long long idx, bool valid) {
  Vec<CP, W> r;
  if constexpr (SP == P16) {
    static_assert(W == 4, "binary16 lanes hold 4 values");
    uint2 raw = make_uint2(0u, 0u);
    if (valid) raw = __ldg(reinterpret_cast<const uint2*>(static_cast<const __half*>(base) + idx));
    if constexpr (CP == P16) {
      r.h[0] = u2h(raw.x);
      r.h[1] = u2h(raw.y);
    } else {
      const float2 a = __half22float2(u2h(raw.x)), b = __half22float2(u2h(raw.y));
      r.v[0] = a.x; r.v[1] = a.y; r.v[2] = b.x; r.v[3] = b.y;
    }
  } else if constexpr (SP == P32) {
    static_assert(CP != P16, "no narrowing loads");
#pragma unroll
    for (int i = 0; i < W; i += 4) {
      float4 raw = make_float4(0.f, 0.f, 0.f, 0.f);
      if (valid) raw = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(base) + idx + i));
      r.v[i] = raw.x; r.v[i + 1] = raw.y; r.v[i + 2] = raw.z; r.v[i + 3] = raw.w;
    }
  } else {
    static_assert(CP == P64, "binary64 storage computes in binary64");
#pragma unroll
    for (int i = 0; i < W; i += 2) {
      double2 raw = make_double2(0.0, 0.0);
      if (valid) raw = __ldg(reinterpret_cast<const double2*>(static_cast<const double*>(base) + idx + i));
      r.v[i] = raw.x; r.v[i + 1] = raw.y;
    }
  }
  return r;
}

// plain (non-__ldg) load for buffers the same kernel also writes
template <int SP, int W>
__device__ __forceinline__ Vec<SP, W> vload_rw(const void* base, long long idx, bool valid) {
  Vec<SP, W> r = vzero<SP, W>();
  if (!valid) return r;
  if constexpr (SP == P16) {
    const uint2 raw = *reinterpret_cast<const uint2*>(static_cast<const __half*>(base) + idx);
    r.h[0] = u2h(raw.x); r.h[1] = u2h(raw.y);
  } else if constexpr (SP == P32) {
#pragma unroll
    for (int i = 0; i < W; i += 4) {
      const float4 raw = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + idx + i);
      r.v[i] = raw.x; r.v[i + 1] = raw.y; r.v[i + 2] = raw.z; r.v[i + 3] = raw.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < W; i += 2) {
      const double2 raw = *reinterpret_cast<const double2*>(static_cast<const double*>(base) + idx + i);
      r.v[i] = raw.x; r.v[i + 1] = raw.y;
    }
  }
  return r;
}

template <int SP, int W>
__device__ __forceinline__ void vstore(void* base, long long idx, const Vec<SP, W>& v) {
  if constexpr (SP == P16) {
    *reinterpret_cast<uint2*>(static_cast<__half*>(base) + idx) = make_uint2(h2u(v.h[0]), h2u(v.h[1]));
  } else if constexpr (SP == P32) {
#pragma unroll
    for (int i = 0; i < W; i += 4)
      *reinterpret_cast<float4*>(static_cast<float*>(base) + idx + i) =
          make_float4(v.v[i], v.v[i + 1], v.v[i + 2], v.v[i + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < W; i += 2)
      *reinterpret_cast<double2*>(static_cast<double*>(base) + idx + i) = make_double2(v.v[i], v.v[i + 1]);
  }
}

// scalar load of one storage value widened to CP (edge lanes' halo values)
template <int SP, int CP>
__device__ __forceinline__ typename Scalar<CP>::T sload(const void* base, long long idx, bool valid) {
  using T = typename Scalar<CP>::T;
  if constexpr (SP == P16) {
    __half h = __ushort_as_half((unsigned short)0);
    if (valid) h = __ldg(static_cast<const __half*>(base) + idx);
    if constexpr (CP == P16) return h;
    else return static_cast<T>(__half2float(h));
  } else if constexpr (SP == P32) {
    float f = 0.f;
    if (valid) f = __ldg(static_cast<const float*>(base) + idx);
    return static_cast<T>(f);
  } else {
    double d = 0.0;
    if (valid) d = __ldg(static_cast<const double*>(base) + idx);
    return static_cast<T>(d);
  }
}

// first / last value of a lane vector (sent to the neighbouring lanes)
template <int CP, int W>
__device__ __forceinline__ typename Scalar<CP>::T vfirst(const Vec<CP, W>& v) {
  if constexpr (CP == P16) return __low2half(v.h[0]);
  else return v.v[0];
}
template <int CP, int W>
__device__ __forceinline__ typename Scalar<CP>::T vlast(const Vec<CP, W>& v) {
  if constexpr (CP == P16) return __high2half(v.h[W / 2 - 1]);
  else return v.v[W - 1];
}

template <typename T>
__device__ __forceinline__ T shfl_up1(T v) { return __shfl_up_sync(0xffffffffu, v, 1); }
template <typename T>
__device__ __forceinline__ T shfl_dn1(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }
template <>
__device__ __forceinline__ __half shfl_up1<__half>(__half v) {
  return __ushort_as_half((unsigned short)__shfl_up_sync(0xffffffffu, (unsigned)__half_as_ushort(v), 1));
}
template <>
__device__ __forceinline__ __half shfl_dn1<__half>(__half v) {
  return __ushort_as_half((unsigned short)__shfl_down_sync(0xffffffffu, (unsigned)__half_as_ushort(v), 1));
}

// x-1 / x+1 shifted neighbour vectors of a lane vector
template <int CP, int W>
__device__ __forceinline__ void vshift(const Vec<CP, W>& c, typename Scalar<CP>::T prev, typename Scalar<CP>::T next,
                                       Vec<CP, W>& L, Vec<CP, W>& R) {
  if constexpr (CP == P16) {
    static_assert(W == 4, "");
    const uint32_t c0 = h2u(c.h[0]), c1 = h2u(c.h[1]);
    const uint32_t pv = (uint32_t)__half_as_ushort(prev), nx = (uint32_t)__half_as_ushort(next);
    L.h[0] = u2h(__byte_perm(pv, c0, 0x5410));  // (prev, v0)
    const uint32_t mid = __byte_perm(c0, c1, 0x5432);  // (v1, v2)
    L.h[1] = u2h(mid);
    R.h[0] = u2h(mid);
    R.h[1] = u2h(__byte_perm(c1, nx, 0x5432));  // (v3, next)
  } else {
    L.v[0] = prev;
#pragma unroll
    for (int i = 1; i < W; ++i) L.v[i] = c.v[i - 1];
#pragma unroll
    for (int i = 0; i < W - 1; ++i) R.v[i] = c.v[i + 1];
    R.v[W - 1] = next;
  }
}

// ---- elementwise Arith<P> on lane vectors, constant first operand ---------
template <int CP> struct Coef;
template <> struct Coef<P16> { using T = __half2; };
template <> struct Coef<P32> { using T = float; };
template <> struct Coef<P64> { using T = double; };

template <int CP, bool FTZ, bool FMA, int W>
__device__ __forceinline__ void vfma(typename Coef<CP>::T a, const Vec<CP, W>& x, Vec<CP, W>& acc) {
  if constexpr (CP == P16) {
#pragma unroll
    for (int i = 0; i < W / 2; ++i) acc.h[i] = fma16<FTZ, FMA>(a, x.h[i], acc.h[i]);
  } else if constexpr (CP == P32) {
#pragma unroll
    for (int i = 0; i < W; ++i) acc.v[i] = fma32<FTZ, FMA>(a, x.v[i], acc.v[i]);
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) acc.v[i] = fma64<FMA>(a, x.v[i], acc.v[i]);
  }
}

// acc = fma(a, x, y) with vector x and y
template <int CP, bool FTZ, bool FMA, int W>
__device__ __forceinline__ Vec<CP, W> vfma3(typename Coef<CP>::T a, const Vec<CP, W>& x, const Vec<CP, W>& y) {
  Vec<CP, W> r = y;
  vfma<CP, FTZ, FMA, W>(a, x, r);
  return r;
}

template <int CP, bool FTZ, int W>
__device__ __forceinline__ Vec<CP, W> vmul(typename Coef<CP>::T a, const Vec<CP, W>& x) {
  Vec<CP, W> r;
  if constexpr (CP == P16) {
#pragma unroll
    for (int i = 0; i < W / 2; ++i) r.h[i] = mul16<FTZ>(a, x.h[i]);
  } else if constexpr (CP == P32) {
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = mul32<FTZ>(a, x.v[i]);
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = mul64(a, x.v[i]);
  }
  return r;
}

// binary32 accumulators -> binary16 (Fp16Accum::FP32 final rounding)
template <bool FTZ, int W>
__device__ __forceinline__ Vec<P16, W> vquant16(const Vec<P32, W>& a) {
  Vec<P16, W> r;
#pragma unroll
  for (int i = 0; i < W / 2; ++i) r.h[i] = round16x2<FTZ>(a.v[2 * i], a.v[2 * i + 1]);
  return r;
}

// zero the element at lane-local position 0 (the x = 0 boundary node)
template <int CP, int W>
__device__ __forceinline__ void vzero_first(Vec<CP, W>& v) {
  if constexpr (CP == P16) v.h[0] = u2h(h2u(v.h[0]) & 0xFFFF0000u);
  else v.v[0] = 0;
}

template <int CP, int W>
__device__ __forceinline__ double vsumsq(const Vec<CP, W>& v, double acc) {
  static_assert(CP == P64, "norms are taken of binary64 vectors");
#pragma unroll
  for (int i = 0; i < W; ++i) acc = __fma_rn(v.v[i], v.v[i], acc);
  return acc;
}

}  // namespace mpmg_dev
