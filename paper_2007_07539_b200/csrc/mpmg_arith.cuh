// Device arithmetic that reproduces the reference's rounding semantics on
// sm_100a hardware, value for value:
//   * binary16: per-operation round-to-nearest-even with gradual underflow,
//     then the reference's flush-after-rounding (quantize_fp16,
//     precision.cpp:23-48): native fma.rn.f16x2 / mul.rn / add.rn (no .ftz)
//     followed by an explicit |v| < 2^-14 -> +-0 select when FTZ is on.
//   * binary32: fma.rn.f32 / mul.rn / add.rn + explicit ftz_fp32
//     (precision.hpp:78-83), kernels.cpp:34-50.
//   * binary64: fma.rn.f64 or mul.rn + add.rn (kernels.cpp:21-32).
// The translation unit is compiled with -fmad=false so that only these
// explicit intrinsics fuse, like the reference's -ffp-contract=off
// (proj/CMakeLists.txt:12).
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

namespace mpmg_dev {

enum { P16 = 0, P32 = 1, P64 = 2 };

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor
// drains; pdl_wait() blocks until the predecessor grid has completed and its
// writes are visible, so it must precede every read of predecessor output.
// pdl_launch() lets the successor grid be scheduled early. Both are no-ops
// for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint32_t h2u(__half2 v) { return *reinterpret_cast<uint32_t*>(&v); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

// ---- flush helpers -------------------------------------------------------
// binary16: |v| < 2^-14 (exponent field zero, value nonzero) -> signed zero.
// Implemented as v * (|v| >= 2^-14 ? 1 : 0): the product is exact and keeps
// the sign of v, NaN/inf pass through (NaN compares false -> NaN*0 = NaN).
__device__ __forceinline__ __half2 flush16(__half2 v) {
  const __half2 mn = u2h(0x04000400u);  // 2^-14 in both halves
  return __hmul2_rn(v, __hge2(__habs2(v), mn));
}
__device__ __forceinline__ __half flush16s(__half v) {
  const uint16_t u = __half_as_ushort(v);
  return __ushort_as_half((u & 0x7C00u) ? u : (uint16_t)(u & 0x8000u));
}
__device__ __forceinline__ float flush32(float v) {
  // ftz_fp32: v != 0 && |v| < FLT_MIN -> copysign(0, v)
  const uint32_t u = __float_as_uint(v);
  return (u & 0x7F800000u) ? v : __uint_as_float(u & 0x80000000u);
}

template <bool FTZ> __device__ __forceinline__ __half2 f16(__half2 v) { return FTZ ? flush16(v) : v; }
template <bool FTZ> __device__ __forceinline__ __half f16s(__half v) { return FTZ ? flush16s(v) : v; }
template <bool FTZ> __device__ __forceinline__ float f32(float v) { return FTZ ? flush32(v) : v; }

// ---- Arith<P> (kernels.cpp:18-67) on packed / scalar registers ------------
template <bool FTZ, bool FMA>
__device__ __forceinline__ __half2 fma16(__half2 a, __half2 b, __half2 c) {
  if (FMA) return f16<FTZ>(__hfma2(a, b, c));
  return f16<FTZ>(__hadd2_rn(f16<FTZ>(__hmul2_rn(a, b)), c));
}
template <bool FTZ>
__device__ __forceinline__ __half2 mul16(__half2 a, __half2 b) { return f16<FTZ>(__hmul2_rn(a, b)); }

template <bool FTZ, bool FMA>
__device__ __forceinline__ __half fma16s(__half a, __half b, __half c) {
  if (FMA) return f16s<FTZ>(__hfma(a, b, c));
  return f16s<FTZ>(__hadd_rn(f16s<FTZ>(__hmul_rn(a, b)), c));
}
template <bool FTZ>
__device__ __forceinline__ __half mul16s(__half a, __half b) { return f16s<FTZ>(__hmul_rn(a, b)); }

template <bool FTZ, bool FMA>
__device__ __forceinline__ float fma32(float a, float b, float c) {
  if (FMA) return f32<FTZ>(__fmaf_rn(a, b, c));
  return f32<FTZ>(__fadd_rn(f32<FTZ>(__fmul_rn(a, b)), c));
}
template <bool FTZ>
__device__ __forceinline__ float mul32(float a, float b) { return f32<FTZ>(__fmul_rn(a, b)); }

template <bool FMA>
__device__ __forceinline__ double fma64(double a, double b, double c) {
  if (FMA) return __fma_rn(a, b, c);
  return __dadd_rn(__dmul_rn(a, b), c);
}
__device__ __forceinline__ double mul64(double a, double b) { return __dmul_rn(a, b); }

// ---- PVector::set rounding from binary64 (vector.hpp:43-55) ---------------
// cvt.rn.f16.f64 rounds once (no double->float->half double rounding).
template <bool FTZ>
__device__ __forceinline__ __half round16(double v) { return f16s<FTZ>(__double2half(v)); }
template <bool FTZ>
__device__ __forceinline__ float round32(double v) { return f32<FTZ>(__double2float_rn(v)); }

// quantize a binary32 accumulator to binary16 (kernels.cpp:160-161):
// float -> half RNE is a single rounding of the exact float value.
template <bool FTZ>
__device__ __forceinline__ __half2 round16x2(float lo, float hi) {
  return f16<FTZ>(__floats2half2_rn(lo, hi));
}

}  // namespace mpmg_dev
