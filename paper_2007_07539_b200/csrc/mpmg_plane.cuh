// TMA-staged 27-point stencil kernels for 3D levels whose pitch P is a
// multiple of 32 (every streaming level of a max-depth hierarchy).
//
// Same operations and bitwise arithmetic as mpmg_stencil.cuh (SpMV, level
// defect, damped Jacobi, FP64 defect / residual norm, fused outer update;
// reference: kernels.cpp:137-193, 300-341, multigrid.cpp:79-89, 379-380,
// ir_solver.cpp:21-49, 92-93), re-tiled for sm_100a:
//
//   * A CTA owns a tile of TY = WY*RY consecutive output rows (full x width)
//     and a chunk of ZC consecutive output planes. It streams the planes of
//     the operand through an NS-stage shared-memory ring: for every plane one
//     elected thread issues ONE cp.async.bulk (TMA bulk copy) of the TY+2
//     contiguous operand rows and one per epilogue operand (b, or r and u),
//     completing on an mbarrier with a transaction count. No per-thread
//     address arithmetic or predication is spent on loads, and NS-1 planes
//     are in flight per CTA.
//   * A lane owns W = P/(32*WX) consecutive x values of a row; the warp's
//     halo values come from its neighbour lanes (shuffles) or, across warps,
//     from shared memory. Each operand row is read from shared memory once
//     per plane and feeds up to 3 output rows x 3 output planes from
//     registers (three rotating accumulator slots).
//   * Summation order per output is the reference's ELL slot order
//     (dz, dy, dx ascending, mesh_fem.cpp:124-150); boundary neighbours are
//     either the stored zero ghosts or skipped (ghost planes), which changes
//     nothing but the sign of an exact zero. binary16 levels skip the six
//     face taps when they round to zero (their FP64 values are ~1e-18
//     roundoff residues): fma(0, x, acc) == acc for every
//     nonzero acc.
#pragma once

#include <type_traits>

#include "mpmg_arith.cuh"

namespace mpmg_dev {

enum { POP_SPMV = 0, POP_DEFECT = 1, POP_JACOBI = 2, POP_DEFECT64 = 3, POP_RESNORM = 4, POP_UPDATE = 5,
       POP_JACOBI_Z = 6, POP_UPDATE_R = 7 };
// JACOBI_Z: steps 1 and 2 from u = 0 fused (operand = b, u1 = w D^-1 b on the fly)
// UPDATE_R: the r half of UPDATE (r -= a A c) plus a copy of c into slot
//   *ring_slot of the correction ring, whose u += a c updates are applied
//   later in the same order (deferred correction, mpmg_solver.cu)

struct PlaneArgs {
  int P;             // pitch
  int zc;            // output planes per CTA
  int pz;            // index of the last local plane: outputs are planes 1 .. pz-1
                     // (a whole level: pz = P; a z-slab of nz owned planes: nz + 1)
  int load_lo;       // plane 0 holds data (a neighbour's halo) -- else a zero ghost, skipped
  int load_hi;       // plane pz holds data
  int ty;            // output rows per CTA (WY*RY)
  long long plane;   // P*P
  __half2 t16[27];
  float t32[27];
  double t64[27];
  __half2 d16, w16;
  float d32, w32;
  double d64, w64;
  const void* x;        // stencil operand (u, or c for UPDATE)
  const void* b;        // DEFECT / JACOBI / DEFECT64 / RESNORM right-hand side
  void* out;            // SPMV / DEFECT / JACOBI / DEFECT64 output
  double* r64;          // UPDATE in/out
  double* u64;          // UPDATE in/out
  const double* alpha;  // UPDATE scale (device scalar)
  double* partials;     // per-CTA sum of squares (DEFECT64 / RESNORM / UPDATE)
  const int* gate;      // optional device flag: no-op unless *gate != 0
  void* ring;           // UPDATE_R: correction ring (slots of ring_len values, precision LP)
  long long ring_len;
  const int* ring_slot; // UPDATE_R: device slot index
  double* ring_scale;   // UPDATE_R: per-slot scale (= *alpha)
  // optional: out += *out_slot * out_stride values (a Jacobi step writing
  // straight into the correction ring); UPDATE_R with x == nullptr reads c
  // from ring slot *ring_slot and skips the copy
  const int* out_slot;
  long long out_stride;
  // OPT bit 3 (z-slab level ops of the multi-GPU solver): the first owned
  // output plane is also stored into push_lo (the lower neighbour's top halo
  // plane, over NVLink peer memory) and the last into push_hi (the upper
  // neighbour's bottom halo plane) -- the halo exchange fused into the
  // producing kernel
  void* push_lo;
  void* push_hi;
};

// ---- PTX: mbarrier + bulk copy ------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "MPMG_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra MPMG_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---- per-lane rows: W values in compute precision CP ---------------------
template <int CP, int W> struct Row;
template <int W> struct Row<P16, W> {  // W >= 2: packed pairs
  static_assert(W % 2 == 0, "");
  __half2 h[W / 2];
};
template <> struct Row<P16, 1> { __half h; };
template <int W> struct Row<P32, W> { float v[W]; };
template <int W> struct Row<P64, W> { double v[W]; };

template <int CP> struct Sc;
template <> struct Sc<P16> { using T = __half; };
template <> struct Sc<P32> { using T = float; };
template <> struct Sc<P64> { using T = double; };

template <int SP> struct Bytes { static constexpr int v = SP == P16 ? 2 : (SP == P32 ? 4 : 8); };

template <int CP, int W>
__device__ __forceinline__ void rzero(Row<CP, W>& r) {
  if constexpr (CP == P16) {
    if constexpr (W == 1) r.h = __ushort_as_half((unsigned short)0);
    else {
#pragma unroll
      for (int i = 0; i < W / 2; ++i) r.h[i] = u2h(0u);
    }
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = 0;
  }
}

// load W storage values (SP) from shared memory, widened to CP
template <int SP, int CP, int W>
__device__ __forceinline__ void rload(const unsigned char* s, Row<CP, W>& r) {
  if constexpr (SP == P16) {
    if constexpr (CP == P16) {
      if constexpr (W == 1) r.h = *reinterpret_cast<const __half*>(s);
      else if constexpr (W % 8 == 0) {
#pragma unroll
        for (int i = 0; i < W / 8; ++i) {
          const uint4 q = *reinterpret_cast<const uint4*>(s + 16 * i);
          r.h[4 * i + 0] = u2h(q.x); r.h[4 * i + 1] = u2h(q.y); r.h[4 * i + 2] = u2h(q.z); r.h[4 * i + 3] = u2h(q.w);
        }
      } else if constexpr (W % 4 == 0) {
#pragma unroll
        for (int i = 0; i < W / 4; ++i) {
          const uint2 q = *reinterpret_cast<const uint2*>(s + 8 * i);
          r.h[2 * i] = u2h(q.x); r.h[2 * i + 1] = u2h(q.y);
        }
      } else {  // W = 2, 6: 4-byte words (a lane's row segment is only 4-byte aligned)
#pragma unroll
        for (int i = 0; i < W / 2; ++i) r.h[i] = u2h(*reinterpret_cast<const uint32_t*>(s + 4 * i));
      }
    } else {  // widen (exact)
      const __half* hp = reinterpret_cast<const __half*>(s);
      if constexpr (W == 1) r.v[0] = (typename Sc<CP>::T)__half2float(hp[0]);
      else {
        __half2 tmp[W / 2];
        if constexpr (W % 8 == 0) {
#pragma unroll
          for (int i = 0; i < W / 8; ++i) {
            const uint4 q = *reinterpret_cast<const uint4*>(s + 16 * i);
            tmp[4 * i + 0] = u2h(q.x); tmp[4 * i + 1] = u2h(q.y); tmp[4 * i + 2] = u2h(q.z); tmp[4 * i + 3] = u2h(q.w);
          }
        } else if constexpr (W % 4 == 0) {
#pragma unroll
          for (int i = 0; i < W / 4; ++i) {
            const uint2 q = *reinterpret_cast<const uint2*>(s + 8 * i);
            tmp[2 * i] = u2h(q.x); tmp[2 * i + 1] = u2h(q.y);
          }
        } else {
#pragma unroll
          for (int i = 0; i < W / 2; ++i) tmp[i] = u2h(*reinterpret_cast<const uint32_t*>(s + 4 * i));
        }
#pragma unroll
        for (int i = 0; i < W / 2; ++i) {
          const float2 f = __half22float2(tmp[i]);
          r.v[2 * i] = (typename Sc<CP>::T)f.x;
          r.v[2 * i + 1] = (typename Sc<CP>::T)f.y;
        }
      }
    }
  } else if constexpr (SP == P32) {
    const float* fp = reinterpret_cast<const float*>(s);
    if constexpr (W % 4 == 0) {
#pragma unroll
      for (int i = 0; i < W / 4; ++i) {
        const float4 q = *reinterpret_cast<const float4*>(fp + 4 * i);
        r.v[4 * i] = q.x; r.v[4 * i + 1] = q.y; r.v[4 * i + 2] = q.z; r.v[4 * i + 3] = q.w;
      }
    } else if constexpr (W % 2 == 0) {
#pragma unroll
      for (int i = 0; i < W / 2; ++i) {
        const float2 q = *reinterpret_cast<const float2*>(fp + 2 * i);
        r.v[2 * i] = q.x; r.v[2 * i + 1] = q.y;
      }
    } else {
      r.v[0] = fp[0];
    }
  } else {
    const double* dp = reinterpret_cast<const double*>(s);
    if constexpr (W >= 2) {
#pragma unroll
      for (int i = 0; i < W / 2; ++i) {
        const double2 q = *reinterpret_cast<const double2*>(dp + 2 * i);
        r.v[2 * i] = q.x; r.v[2 * i + 1] = q.y;
      }
    } else {
      r.v[0] = dp[0];
    }
  }
}

template <int SP, int CP>
__device__ __forceinline__ typename Sc<CP>::T sload_s(const unsigned char* s) {
  if constexpr (SP == P16) {
    const __half h = *reinterpret_cast<const __half*>(s);
    if constexpr (CP == P16) return h;
    else return (typename Sc<CP>::T)__half2float(h);
  } else if constexpr (SP == P32) {
    return (typename Sc<CP>::T) * reinterpret_cast<const float*>(s);
  } else {
    return *reinterpret_cast<const double*>(s);
  }
}

template <int CP, int W>
__device__ __forceinline__ typename Sc<CP>::T rfirst(const Row<CP, W>& r) {
  if constexpr (CP == P16) {
    if constexpr (W == 1) return r.h;
    else return __low2half(r.h[0]);
  } else return r.v[0];
}
template <int CP, int W>
__device__ __forceinline__ typename Sc<CP>::T rlast(const Row<CP, W>& r) {
  if constexpr (CP == P16) {
    if constexpr (W == 1) return r.h;
    else return __high2half(r.h[W / 2 - 1]);
  } else return r.v[W - 1];
}

template <typename T>
__device__ __forceinline__ T shup(T v) { return __shfl_up_sync(0xffffffffu, v, 1); }
template <typename T>
__device__ __forceinline__ T shdn(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }
template <>
__device__ __forceinline__ __half shup<__half>(__half v) {
  return __ushort_as_half((unsigned short)__shfl_up_sync(0xffffffffu, (unsigned)__half_as_ushort(v), 1));
}
template <>
__device__ __forceinline__ __half shdn<__half>(__half v) {
  return __ushort_as_half((unsigned short)__shfl_down_sync(0xffffffffu, (unsigned)__half_as_ushort(v), 1));
}

// x-1 / x+1 neighbour rows
template <int CP, int W>
__device__ __forceinline__ void rshift(const Row<CP, W>& c, typename Sc<CP>::T prev, typename Sc<CP>::T next,
                                       Row<CP, W>& L, Row<CP, W>& R) {
  if constexpr (CP == P16 && W == 1) {
    L.h = prev;
    R.h = next;
  } else if constexpr (CP == P16) {
    const uint32_t pv = (uint32_t)__half_as_ushort(prev), nx = (uint32_t)__half_as_ushort(next);
    uint32_t cu[W / 2];
#pragma unroll
    for (int i = 0; i < W / 2; ++i) cu[i] = h2u(c.h[i]);
    // pairs hold (v[2i] low, v[2i+1] high); L pair i = (v[2i-1], v[2i]),
    // R pair i = (v[2i+1], v[2i+2])
    L.h[0] = u2h(__byte_perm(pv, cu[0], 0x5410));  // (prev, lo(cu0))
#pragma unroll
    for (int i = 1; i < W / 2; ++i) L.h[i] = u2h(__byte_perm(cu[i - 1], cu[i], 0x5432));
#pragma unroll
    for (int i = 0; i < W / 2; ++i) {
      const uint32_t hi = i == W / 2 - 1 ? nx : cu[i + 1];
      R.h[i] = u2h(__byte_perm(cu[i], hi, 0x5432));  // (hi(cu), lo(hi))
    }
  } else {
    L.v[0] = prev;
#pragma unroll
    for (int i = 1; i < W; ++i) L.v[i] = c.v[i - 1];
#pragma unroll
    for (int i = 0; i < W - 1; ++i) R.v[i] = c.v[i + 1];
    R.v[W - 1] = next;
  }
}

// acc = fma(t, x, acc) elementwise, Arith<CP> rounding
template <int CP, bool FTZ, bool FMA, int W, typename TT>
__device__ __forceinline__ void rfma(TT t, const Row<CP, W>& x, Row<CP, W>& acc) {
  if constexpr (CP == P16) {
    if constexpr (W == 1) acc.h = fma16s<FTZ, FMA>(__low2half(t), x.h, acc.h);
    else {
#pragma unroll
      for (int i = 0; i < W / 2; ++i) acc.h[i] = fma16<FTZ, FMA>(t, x.h[i], acc.h[i]);
    }
  } else if constexpr (CP == P32) {
#pragma unroll
    for (int i = 0; i < W; ++i) acc.v[i] = fma32<FTZ, FMA>(t, x.v[i], acc.v[i]);
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) acc.v[i] = fma64<FMA>(t, x.v[i], acc.v[i]);
  }
}

template <int CP>
__device__ __forceinline__ auto tap(const PlaneArgs& a, int k) {
  if constexpr (CP == P16) return a.t16[k];
  else if constexpr (CP == P32) return a.t32[k];
  else return a.t64[k];
}

// store W values of precision SP from row r (same precision) to global
template <int SP, int W>
__device__ __forceinline__ void gstore(void* base, long long idx, const Row<SP, W>& r) {
  if constexpr (SP == P16) {
    __half* p = static_cast<__half*>(base) + idx;
    if constexpr (W == 1) *p = r.h;
    else if constexpr (W % 8 == 0) {
#pragma unroll
      for (int i = 0; i < W / 8; ++i)
        reinterpret_cast<uint4*>(p)[i] =
            make_uint4(h2u(r.h[4 * i]), h2u(r.h[4 * i + 1]), h2u(r.h[4 * i + 2]), h2u(r.h[4 * i + 3]));
    } else if constexpr (W % 4 == 0) {
#pragma unroll
      for (int i = 0; i < W / 4; ++i) reinterpret_cast<uint2*>(p)[i] = make_uint2(h2u(r.h[2 * i]), h2u(r.h[2 * i + 1]));
    } else {
#pragma unroll
      for (int i = 0; i < W / 2; ++i) reinterpret_cast<uint32_t*>(p)[i] = h2u(r.h[i]);
    }
  } else if constexpr (SP == P32) {
    float* p = static_cast<float*>(base) + idx;
    if constexpr (W % 4 == 0) {
#pragma unroll
      for (int i = 0; i < W / 4; ++i)
        reinterpret_cast<float4*>(p)[i] = make_float4(r.v[4 * i], r.v[4 * i + 1], r.v[4 * i + 2], r.v[4 * i + 3]);
    } else if constexpr (W % 2 == 0) {
#pragma unroll
      for (int i = 0; i < W / 2; ++i) reinterpret_cast<float2*>(p)[i] = make_float2(r.v[2 * i], r.v[2 * i + 1]);
    } else *p = r.v[0];
  } else {
    double* p = static_cast<double*>(base) + idx;
    if constexpr (W >= 2) {
#pragma unroll
      for (int i = 0; i < W / 2; ++i) reinterpret_cast<double2*>(p)[i] = make_double2(r.v[2 * i], r.v[2 * i + 1]);
    } else *p = r.v[0];
  }
}

// load W values of precision SP from global (read-only path)
template <int SP, int W>
__device__ __forceinline__ void gload(const void* base, long long idx, Row<SP, W>& r) {
  if constexpr (SP == P16) {
    const __half* p = static_cast<const __half*>(base) + idx;
    if constexpr (W == 1) r.h = __ldg(p);
    else if constexpr (W % 8 == 0) {
#pragma unroll
      for (int i = 0; i < W / 8; ++i) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(p) + i);
        r.h[4 * i] = u2h(q.x); r.h[4 * i + 1] = u2h(q.y); r.h[4 * i + 2] = u2h(q.z); r.h[4 * i + 3] = u2h(q.w);
      }
    } else if constexpr (W % 4 == 0) {
#pragma unroll
      for (int i = 0; i < W / 4; ++i) {
        const uint2 q = __ldg(reinterpret_cast<const uint2*>(p) + i);
        r.h[2 * i] = u2h(q.x); r.h[2 * i + 1] = u2h(q.y);
      }
    } else {
#pragma unroll
      for (int i = 0; i < W / 2; ++i) r.h[i] = u2h(__ldg(reinterpret_cast<const unsigned int*>(p) + i));
    }
  } else if constexpr (SP == P32) {
    const float* p = static_cast<const float*>(base) + idx;
    if constexpr (W % 4 == 0) {
#pragma unroll
      for (int i = 0; i < W / 4; ++i) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(p) + i);
        r.v[4 * i] = q.x; r.v[4 * i + 1] = q.y; r.v[4 * i + 2] = q.z; r.v[4 * i + 3] = q.w;
      }
    } else if constexpr (W % 2 == 0) {
#pragma unroll
      for (int i = 0; i < W / 2; ++i) {
        const float2 q = __ldg(reinterpret_cast<const float2*>(p) + i);
        r.v[2 * i] = q.x; r.v[2 * i + 1] = q.y;
      }
    } else r.v[0] = __ldg(p);
  } else {
    const double* p = static_cast<const double*>(base) + idx;
    if constexpr (W >= 2) {
#pragma unroll
      for (int i = 0; i < W / 2; ++i) {
        const double2 q = __ldg(reinterpret_cast<const double2*>(p) + i);
        r.v[2 * i] = q.x; r.v[2 * i + 1] = q.y;
      }
    } else r.v[0] = __ldg(p);
  }
}

// zero lane-local element 0 (the x = 0 ghost node)
template <int CP, int W>
__device__ __forceinline__ void rzero_first(Row<CP, W>& r) {
  if constexpr (CP == P16) {
    if constexpr (W == 1) r.h = __ushort_as_half((unsigned short)0);
    else r.h[0] = u2h(h2u(r.h[0]) & 0xFFFF0000u);
  } else r.v[0] = 0;
}

// elementwise epilogue helpers in the level precision EP
template <int EP, bool FTZ, bool FMA, int W, typename TT>
__device__ __forceinline__ Row<EP, W> efma(TT a, const Row<EP, W>& x, const Row<EP, W>& y) {
  Row<EP, W> r = y;
  rfma<EP, FTZ, FMA, W>(a, x, r);
  return r;
}
template <int EP, bool FTZ, int W, typename TT>
__device__ __forceinline__ Row<EP, W> emul(TT a, const Row<EP, W>& x) {
  Row<EP, W> r;
  if constexpr (EP == P16) {
    if constexpr (W == 1) r.h = mul16s<FTZ>(__low2half(a), x.h);
    else {
#pragma unroll
      for (int i = 0; i < W / 2; ++i) r.h[i] = mul16<FTZ>(a, x.h[i]);
    }
  } else if constexpr (EP == P32) {
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = mul32<FTZ>(a, x.v[i]);
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = mul64(a, x.v[i]);
  }
  return r;
}
// first Jacobi step from zero, elementwise: u1 = fma(w, d*b, +0) (the
// fused form of t = A*0, r = b - t, t = d r, u = 0 + w t; multigrid.cpp:79-89)
template <int CP, bool FTZ, bool FMA, int W, typename TT>
__device__ __forceinline__ void jz_row(TT d, TT w, Row<CP, W>& x) {
  Row<CP, W> zero;
  rzero(zero);
  x = efma<CP, FTZ, FMA, W>(w, emul<CP, FTZ, W>(d, x), zero);
}
template <int CP, bool FTZ, bool FMA, typename ST, typename TT>
__device__ __forceinline__ ST jz_scalar(TT d, TT w, ST v) {
  if constexpr (CP == P16) return fma16s<FTZ, FMA>(__low2half(w), mul16s<FTZ>(__low2half(d), v), __ushort_as_half((unsigned short)0));
  else if constexpr (CP == P32) return fma32<FTZ, FMA>(w, mul32<FTZ>(d, v), 0.0f);
  else return fma64<FMA>(w, mul64(d, v), 0.0);
}

// binary32 accumulators -> binary16 (Fp16Accum::FP32, kernels.cpp:160-161)
template <bool FTZ, int W>
__device__ __forceinline__ Row<P16, W> quant16(const Row<P32, W>& a) {
  Row<P16, W> r;
  if constexpr (W == 1) r.h = f16s<FTZ>(__float2half_rn(a.v[0]));
  else {
#pragma unroll
    for (int i = 0; i < W / 2; ++i) r.h[i] = round16x2<FTZ>(a.v[2 * i], a.v[2 * i + 1]);
  }
  return r;
}

__device__ __forceinline__ bool is_face(int k) {
  return k == 4 || k == 10 || k == 12 || k == 14 || k == 16 || k == 22;
}

// tap k = 9 (dz+1) + 3 (dy+1) + (dx+1) by its number of nonzero offsets:
// 0 centre, 1 face, 2 edge, 3 corner. The binary16 kernels only run on
// stencils whose faces are zero and whose edge / corner taps are each one
// value (sym16 in the launcher: every hierarchy level), so they pin three
// tap registers instead of 21 -- the registers the plane loop needs.
__host__ __device__ constexpr int tap_class(int k) {
  return (k / 9 != 1) + ((k / 3) % 3 != 1) + (k % 3 != 1);
}
__host__ __device__ constexpr int tap_rep(int c) { return c == 0 ? 13 : (c == 1 ? 4 : (c == 2 ? 1 : 0)); }

// ---- the kernel ----------------------------------------------------------
// LP storage precision of the stencil operand; CP accumulation precision;
// EP epilogue/output precision; W values per lane; WX warps per row;
// WY warp-rows per CTA; RY rows per thread; NS pipeline stages.
// OPT bit 0: stage b through shared memory (instead of the register prefetch);
// bit 2: output to ring slot *out_slot (PlaneArgs::out_slot / out_stride)
template <int LP, int CP, int EP, int OP, bool FTZ, bool FMA, bool SKIPF, int W, int WX, int WY, int RY, int NS,
          int OPT = 0>
struct PlaneK {
  static constexpr int kThreads = 32 * WX * WY;
  static constexpr int TY = WY * RY;
  static constexpr bool kB = OP == POP_DEFECT || OP == POP_JACOBI || OP == POP_DEFECT64 || OP == POP_RESNORM;
  static constexpr bool kNorm = OP == POP_DEFECT64 || OP == POP_RESNORM || OP == POP_UPDATE || OP == POP_UPDATE_R;
  // binary16/32 level ops prefetch b into registers one plane ahead (global
  // loads); the FP64 epilogue operands are staged through shared memory
  static constexpr bool kBReg = (OP == POP_DEFECT || OP == POP_JACOBI) && EP != P64 && !(OPT & 1);
  static constexpr bool kJZ = OP == POP_JACOBI_Z;  // b is the stencil operand: nothing else staged
  static constexpr int kEpiBytes =
      OP == POP_UPDATE ? 16 : (OP == POP_UPDATE_R ? 8 : ((kB && !kBReg) ? Bytes<EP>::v : 0));  // per value
  static constexpr int kP = 32 * WX * W;  // pitch (compile-time)
  static constexpr int kXRow = kP * Bytes<LP>::v;
  static constexpr int kXBytes = (TY + 2) * kXRow;
  static constexpr int kEpiRow = kP * kEpiBytes;
  static constexpr int kStage = kXBytes + TY * kEpiRow;
  static constexpr int kSmem = 128 + NS * kStage;
};

template <int LP, int CP, int EP, int OP, bool FTZ, bool FMA, bool SKIPF, int W, int WX, int WY, int RY, int NS,
          int OPT = 0>
__global__ void __launch_bounds__(32 * WX * WY, (CP == P16 && 32 * WX * WY == 128) ? 4 : 1)
    k_plane(const __grid_constant__ PlaneArgs a) {
  using K = PlaneK<LP, CP, EP, OP, FTZ, FMA, SKIPF, W, WX, WY, RY, NS, OPT>;
  using ST = typename Sc<CP>::T;
  constexpr int P = K::kP;
  constexpr int TY = K::TY;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  unsigned char* stages = smem + 128;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wx = warp % WX, wy = warp / WX;
  const int x0 = (wx * 32 + lane) * W;
  const int tr = wy * RY;  // tile row of this thread's first output row (minus 1)
  const int y0 = 1 + (int)blockIdx.x * TY;
  const int z0 = 1 + (int)blockIdx.y * a.zc;
  const int z1 = min(z0 + a.zc, a.pz);  // outputs [z0, z1)
  const int NQ = z1 - z0 + 2;        // planes z0-1 .. z1
  const long long plane = (long long)P * P;
  const int xrows = min(y0 + TY, P) - y0 + 2;  // operand rows y0-1 .. min(y0+TY, P)
  const int erows = min(TY, P - y0);           // epilogue rows y0 .. y0+erows-1

  const unsigned char* xsrc = static_cast<const unsigned char*>(a.x);  // set after the gate (ring slot)
  auto issue = [&](int k) {  // one elected thread: plane k into stage k % NS
    const int q = z0 - 1 + k;
    if ((q == 0 && !a.load_lo) || (q == a.pz && !a.load_hi)) return;  // zero ghost planes are never loaded
    unsigned char* st = stages + (k % NS) * K::kStage;
    uint64_t* bar = full + (k % NS);
    const uint32_t xb = (uint32_t)(xrows * K::kXRow);
    const uint32_t eb = (uint32_t)(erows * P * (K::kEpiBytes ? Bytes<EP>::v : 0));
    uint32_t tot = xb;
    if constexpr (OP == POP_UPDATE) tot += 2 * (uint32_t)(erows * P * 8);
    else if constexpr (OP == POP_UPDATE_R) tot += (uint32_t)(erows * P * 8);
    else if constexpr (K::kB && !K::kBReg) tot += eb;
    mbar_arrive_tx(bar, tot);
    const long long xo = q * plane + (long long)(y0 - 1) * P;
    bulk_g2s(st, xsrc + xo * Bytes<LP>::v, xb, bar);
    const long long eo = q * plane + (long long)y0 * P;
    if constexpr (OP == POP_UPDATE) {
      bulk_g2s(st + K::kXBytes, a.r64 + eo, (uint32_t)(erows * P * 8), bar);
      bulk_g2s(st + K::kXBytes + TY * P * 8, a.u64 + eo, (uint32_t)(erows * P * 8), bar);
    } else if constexpr (OP == POP_UPDATE_R) {
      bulk_g2s(st + K::kXBytes, a.r64 + eo, (uint32_t)(erows * P * 8), bar);
    } else if constexpr (K::kB && !K::kBReg) {
      bulk_g2s(st + K::kXBytes, static_cast<const unsigned char*>(a.b) + eo * Bytes<EP>::v, eb, bar);
    }
  };

  pdl_wait();    // predecessor output visible from here on
  pdl_launch();  // let the next kernel's CTAs be scheduled as ours retire
  if (a.gate && *a.gate == 0) return;  // uniform across the grid
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_init(full + s, 1);
    fence_barrier_init();
  }
  __syncthreads();
  long long ring_off = 0;
  bool ring_copy = false;
  if constexpr (OP == POP_UPDATE_R) {
    const int slot = *a.ring_slot;
    ring_off = (long long)slot * a.ring_len;
    if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) a.ring_scale[slot] = *a.alpha;
    ring_copy = a.x != nullptr;
    if (!ring_copy) xsrc = static_cast<const unsigned char*>(a.ring) + ring_off * Bytes<LP>::v;
  }
  // OPT bit 2: the output goes to slot *out_slot of a ring (a separate
  // instantiation, so the common kernels carry no extra registers)
  void* outp = a.out;
  if constexpr ((OPT & 4) != 0)
    outp = static_cast<unsigned char*>(a.out) + (long long)*a.out_slot * a.out_stride * Bytes<EP>::v;
  // output row store (+ the fused halo push of a slab's boundary planes)
  auto put = [&](long long gi, int zo, const Row<EP, W>& row) {
    gstore<EP, W>(outp, gi, row);
    if constexpr ((OPT & 8) != 0) {
      const long long in_plane = gi - zo * plane;
      if (zo == 1 && a.push_lo) gstore<EP, W>(a.push_lo, in_plane, row);
      if (zo == a.pz - 1 && a.push_hi) gstore<EP, W>(a.push_hi, in_plane, row);
    }
  };
  if (tid == 0) {
    for (int k = 0; k < NS - 1 && k < NQ; ++k) issue(k);
  }

  // binary16 taps pinned in registers (HFMA2 takes no constant-bank operand)
  // (read once from shared memory: a constant-bank value would be
  // rematerialised by ptxas with an LDC per use)
  __shared__ uint32_t s_taps[27];
  if (CP == P16 && tid < 27) s_taps[tid] = h2u(a.t16[tid]);
  __syncthreads();
  static_assert(CP != P16 || SKIPF, "binary16 plane kernels take the symmetric (sym16) stencil form");
  uint32_t tk[4];  // binary16: by tap class (face taps are skipped)
  if constexpr (CP == P16) {
#pragma unroll
    for (int c = 0; c < 4; ++c) tk[c] = c == 1 ? 0u : s_taps[tap_rep(c)];
  }
  // JACOBI_Z: D^-1 and omega in the compute precision
  const auto jd = [&] {
    if constexpr (CP == P16) return a.d16;
    else if constexpr (CP == P32) return a.d32;
    else return a.d64;
  }();
  const auto jw = [&] {
    if constexpr (CP == P16) return a.w16;
    else if constexpr (CP == P32) return a.w32;
    else return a.w64;
  }();
  (void)jd; (void)jw;
  auto tapk = [&](int k) {
    if constexpr (CP == P16) return u2h(tk[tap_class(k)]);
    else return tap<CP>(a, k);
  };

  // kBReg: b rows of the next output plane, prefetched into registers
  Row<EP, W> bcur[K::kBReg ? RY : 1], bnext[K::kBReg ? RY : 1];
  auto prefetch_b = [&](int zq) {
    if constexpr (K::kBReg) {
#pragma unroll
      for (int i = 0; i < RY; ++i) {
        const int y = y0 + tr + i;
        if (zq >= z0 && zq < z1 && y <= P - 1) gload<EP, W>(a.b, zq * plane + (long long)y * P + x0, bnext[i]);
      }
    }
  };

  Row<CP, W> acc0[RY], acc1[RY], acc2[RY];
#pragma unroll
  for (int i = 0; i < RY; ++i) { rzero(acc0[i]); rzero(acc1[i]); rzero(acc2[i]); }
  double sq = 0.0;
  uint32_t phase = 0;

  // contributions of one operand plane (stage s) to the three output planes;
  // bit d of the compile-time mask M selects output plane A_d (M = 7 on the
  // interior planes of a chunk, partial masks on its first / last two)
  auto accumulate = [&](auto mask_c, const unsigned char* st, Row<CP, W>* A0, Row<CP, W>* A1, Row<CP, W>* A2) {
    constexpr int M = decltype(mask_c)::value;
#pragma unroll
    for (int j = 0; j < RY + 2; ++j) {
      const unsigned char* rp = st + (tr + j) * K::kXRow;
      Row<CP, W> c, L, R;
      rload<LP, CP, W>(rp + x0 * Bytes<LP>::v, c);
      if constexpr (K::kJZ) jz_row<CP, FTZ, FMA, W>(jd, jw, c);
      ST prev = shup(rlast<CP, W>(c));
      ST next = shdn(rfirst<CP, W>(c));
      if constexpr (WX > 1) {
        // the neighbour warps' edge values, read raw from the staged row (the
        // shuffled ones above are already transformed for JACOBI_Z)
        if (lane == 0) {
          prev = x0 > 0 ? sload_s<LP, CP>(rp + (x0 - 1) * Bytes<LP>::v) : ST(0);
          if constexpr (K::kJZ) prev = jz_scalar<CP, FTZ, FMA, ST>(jd, jw, prev);
        }
        if (lane == 31) {
          next = x0 + W < P ? sload_s<LP, CP>(rp + (x0 + W) * Bytes<LP>::v) : ST(0);
          if constexpr (K::kJZ) next = jz_scalar<CP, FTZ, FMA, ST>(jd, jw, next);
        }
      } else {
        if (lane == 0) prev = ST(0);   // x = -1: only feeds the ghost output x = 0
        if (lane == 31) next = ST(0);  // x = P: the aliased ghost (zero)
      }
      rshift<CP, W>(c, prev, next, L, R);
#pragma unroll
      for (int i = 0; i < RY; ++i) {
        const int dyi = j - i;  // 0,1,2 <-> dy = -1, 0, +1
        if (dyi < 0 || dyi > 2) continue;
#pragma unroll
        for (int dz = 0; dz < 3; ++dz) {
          // operand plane q is dz=+1 for output q-1 (A0), 0 for q (A1), -1 for q+1 (A2)
          Row<CP, W>* Acc = dz == 0 ? A0 : (dz == 1 ? A1 : A2);
          const int tz = 2 - dz;  // tap plane index: dz_tap + 1
          if (((M >> dz) & 1) == 0) continue;
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) {
            const int k = tz * 9 + dyi * 3 + dx;
            if (SKIPF && is_face(k)) continue;
            rfma<CP, FTZ, FMA, W>(tapk(k), dx == 0 ? L : (dx == 1 ? c : R), Acc[i]);
          }
        }
      }
    }
  };

  // epilogue of output plane zo from the stage that holds plane zo
  auto epilogue = [&](const unsigned char* st, int zo, Row<CP, W>* Acc) {
#pragma unroll
    for (int i = 0; i < RY; ++i) {
      const int y = y0 + tr + i;
      const bool v = y <= P - 1;
      const long long gi = zo * plane + (long long)y * P + x0;
      Row<EP, W> t;
      if constexpr (CP == EP) t = Acc[i];
      else if constexpr (EP == P16) t = quant16<FTZ, W>(Acc[i]);
      if constexpr (OP == POP_SPMV) {
        if (x0 == 0) rzero_first<EP, W>(t);
        if (v) put(gi, zo, t);
      } else if constexpr (OP == POP_DEFECT || OP == POP_JACOBI || OP == POP_JACOBI_Z) {
        Row<EP, W> bb;
        if constexpr (K::kJZ) rload<LP, EP, W>(st + (tr + i + 1) * K::kXRow + x0 * Bytes<LP>::v, bb);  // b centre
        else if constexpr (K::kBReg) bb = bcur[i];
        else rload<EP, EP, W>(st + K::kXBytes + (tr + i) * K::kEpiRow + x0 * Bytes<EP>::v, bb);
        if constexpr (EP == P16) {
          const __half2 m1 = u2h(0xBC00BC00u);
          Row<EP, W> r = efma<EP, FTZ, FMA, W>(m1, t, bb);  // axpy(-1, t, b)
          if constexpr (OP == POP_DEFECT) {
            if (x0 == 0) rzero_first<EP, W>(r);
            if (v) put(gi, zo, r);
          } else {
            const Row<EP, W> dr = emul<EP, FTZ, W>(a.d16, r);  // vec_multiply(inv_diag, r)
            Row<EP, W> uc;
            if constexpr (K::kJZ) {
              uc = bb;
              jz_row<EP, FTZ, FMA, W>(a.d16, a.w16, uc);
            } else rload<LP, EP, W>(st + (tr + i + 1) * K::kXRow + x0 * Bytes<LP>::v, uc);
            Row<EP, W> un = efma<EP, FTZ, FMA, W>(a.w16, dr, uc);  // axpy(omega, t, u)
            if (x0 == 0) rzero_first<EP, W>(un);
            if (v) put(gi, zo, un);
          }
        } else {
          using ET = typename Sc<EP>::T;
          const ET m1 = ET(-1), dd = EP == P32 ? (ET)a.d32 : (ET)a.d64, ww = EP == P32 ? (ET)a.w32 : (ET)a.w64;
          Row<EP, W> r = efma<EP, FTZ, FMA, W>(m1, t, bb);
          if constexpr (OP == POP_DEFECT) {
            if (x0 == 0) rzero_first<EP, W>(r);
            if (v) put(gi, zo, r);
          } else {
            const Row<EP, W> dr = emul<EP, FTZ, W>(dd, r);
            Row<EP, W> uc;
            if constexpr (K::kJZ) {
              uc = bb;
              jz_row<EP, FTZ, FMA, W>(dd, ww, uc);
            } else rload<LP, EP, W>(st + (tr + i + 1) * K::kXRow + x0 * Bytes<LP>::v, uc);
            Row<EP, W> un = efma<EP, FTZ, FMA, W>(ww, dr, uc);
            if (x0 == 0) rzero_first<EP, W>(un);
            if (v) put(gi, zo, un);
          }
        }
      } else if constexpr (OP == POP_DEFECT64 || OP == POP_RESNORM) {
        Row<P64, W> bb, r;
        rload<P64, P64, W>(st + K::kXBytes + (tr + i) * K::kEpiRow + x0 * 8, bb);
#pragma unroll
        for (int e = 0; e < W; ++e)
          r.v[e] = OP == POP_RESNORM ? __dsub_rn(bb.v[e], t.v[e]) : fma64<FMA>(-1.0, t.v[e], bb.v[e]);
        if (x0 == 0) rzero_first<P64, W>(r);
        if (v) {
          if (OP == POP_DEFECT64 && a.out) gstore<P64, W>(outp, gi, r);
#pragma unroll
          for (int e = 0; e < W; ++e) sq = __fma_rn(r.v[e], r.v[e], sq);
        }
      } else if constexpr (OP == POP_UPDATE_R) {
        const double al = *a.alpha;
        Row<P64, W> rr, rn;
        Row<LP, W> craw;
        rload<P64, P64, W>(st + K::kXBytes + (tr + i) * (P * 8) + x0 * 8, rr);
        rload<LP, LP, W>(st + (tr + i + 1) * K::kXRow + x0 * Bytes<LP>::v, craw);
#pragma unroll
        for (int e = 0; e < W; ++e) rn.v[e] = fma64<FMA>(-al, t.v[e], rr.v[e]);
        if (x0 == 0) rzero_first<P64, W>(rn);
        if (v) {
          gstore<P64, W>(a.r64, gi, rn);
          if (ring_copy) gstore<LP, W>(a.ring, ring_off + gi, craw);  // c unchanged (x = 0 ghost is zero)
#pragma unroll
          for (int e = 0; e < W; ++e) sq = __fma_rn(rn.v[e], rn.v[e], sq);
        }
      } else if constexpr (OP == POP_UPDATE) {
        const double al = *a.alpha;
        Row<P64, W> rr, uu, cc, un, rn;
        rload<P64, P64, W>(st + K::kXBytes + (tr + i) * (P * 8) + x0 * 8, rr);
        rload<P64, P64, W>(st + K::kXBytes + TY * P * 8 + (tr + i) * (P * 8) + x0 * 8, uu);
        rload<LP, P64, W>(st + (tr + i + 1) * K::kXRow + x0 * Bytes<LP>::v, cc);
#pragma unroll
        for (int e = 0; e < W; ++e) {
          un.v[e] = fma64<FMA>(al, cc.v[e], uu.v[e]);
          rn.v[e] = fma64<FMA>(-al, t.v[e], rr.v[e]);
        }
        if (x0 == 0) { rzero_first<P64, W>(un); rzero_first<P64, W>(rn); }
        if (v) {
          gstore<P64, W>(a.u64, gi, un);
          gstore<P64, W>(a.r64, gi, rn);
#pragma unroll
          for (int e = 0; e < W; ++e) sq = __fma_rn(rn.v[e], rn.v[e], sq);
        }
      }
    }
  };

  // plane loop; the accumulator slots rotate by register moves (a 3x unrolled
  // loop renaming them statically spills at the 128-register cap and measured
  // slower). Operand plane k feeds output planes q-1 (acc0, ours iff k >= 2),
  // q (acc1, 1 <= k <= NQ-2) and q+1 (acc2, k <= NQ-3): the chunk's first and
  // last two planes take statically specialised partial accumulations instead
  // of per-tap guards.
  for (int k = 0; k < NQ; ++k) {
    const int q = z0 - 1 + k;
    const int s = k % NS;
    const unsigned char* st = stages + s * K::kStage;
    prefetch_b(q);
    if ((q > 0 || a.load_lo) && (q < a.pz || a.load_hi)) {
      mbar_wait(full + s, (phase >> s) & 1u);
      phase ^= 1u << s;
      const int m = (k >= 2) | (k >= 1 && k <= NQ - 2) << 1 | (k <= NQ - 3) << 2;
      switch (m) {  // CTA-uniform; mask 5 cannot occur
        case 7: accumulate(std::integral_constant<int, 7>{}, st, acc0, acc1, acc2); break;
        case 6: accumulate(std::integral_constant<int, 6>{}, st, acc0, acc1, acc2); break;
        case 4: accumulate(std::integral_constant<int, 4>{}, st, acc0, acc1, acc2); break;
        case 3: accumulate(std::integral_constant<int, 3>{}, st, acc0, acc1, acc2); break;
        case 2: accumulate(std::integral_constant<int, 2>{}, st, acc0, acc1, acc2); break;
        case 1: accumulate(std::integral_constant<int, 1>{}, st, acc0, acc1, acc2); break;
        default: break;
      }
    }
    if (k >= 2) epilogue(stages + ((k - 1) % NS) * K::kStage, q - 1, acc0);
    if constexpr (K::kBReg) {
#pragma unroll
      for (int i = 0; i < RY; ++i) bcur[i] = bnext[i];
    }
#pragma unroll
    for (int i = 0; i < RY; ++i) {
      acc0[i] = acc1[i];
      acc1[i] = acc2[i];
      rzero(acc2[i]);
    }
    __syncthreads();
    if (tid == 0 && k + NS - 1 < NQ) {
      fence_proxy_async();
      issue(k + NS - 1);
    }
  }

  if constexpr (K::kNorm) {
    if (a.partials) {
      __shared__ double red[32];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
      if (lane == 0) red[warp] = sq;
      __syncthreads();
      if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < K::kThreads / 32; ++w) s += red[w];
        a.partials[blockIdx.y * gridDim.x + blockIdx.x] = s;
      }
    }
  }
}

// ---- direct-load variant for small L2-resident levels ---------------------
// One warp per output row (x width P = 32 W), no shared-memory staging: each
// lane loads its W values of the 9 neighbour rows straight from L2 and shifts
// them like k_plane (WX = 1). Same per-output slot order and epilogue as
// k_plane, so the results are bitwise those of the plane kernel; it trades
// 9x L2 reads for no pipeline fill, which wins on the latency-bound levels.
template <int LP, int OP, bool FTZ, bool FMA, bool SKIPF, int W>
__global__ void __launch_bounds__(128) k_direct(const __grid_constant__ PlaneArgs a) {
  using ST = typename Sc<LP>::T;
  constexpr int P = 32 * W;
  constexpr bool kJZ = OP == POP_JACOBI_Z;
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31;
  const int rr = (int)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (rr >= (P - 1) * (P - 1)) return;  // warp-uniform
  const int y = 1 + rr % (P - 1), z = 1 + rr / (P - 1);
  const int x0 = lane * W;
  const long long plane = (long long)P * P;
  static_assert(LP != P16 || SKIPF, "binary16 direct kernels take the symmetric (sym16) stencil form");
  uint32_t tk[4];  // binary16: by tap class (see tap_class)
  if constexpr (LP == P16) {
#pragma unroll
    for (int c = 0; c < 4; ++c) tk[c] = c == 1 ? 0u : h2u(a.t16[tap_rep(c)]);
  }
  auto tapk = [&](int k) {
    if constexpr (LP == P16) return u2h(tk[tap_class(k)]);
    else return tap<LP>(a, k);
  };
  const auto jd = [&] {
    if constexpr (LP == P16) return a.d16;
    else if constexpr (LP == P32) return a.d32;
    else return a.d64;
  }();
  const auto jw = [&] {
    if constexpr (LP == P16) return a.w16;
    else if constexpr (LP == P32) return a.w32;
    else return a.w64;
  }();
  (void)jd; (void)jw;
  const long long gi = z * plane + (long long)y * P + x0;
  void* const outp = a.out;
  Row<LP, W> acc, ctr;
  rzero(acc);
  rzero(ctr);
#pragma unroll
  for (int tz = 0; tz < 3; ++tz)
#pragma unroll
    for (int ty = 0; ty < 3; ++ty) {
      Row<LP, W> c, L, R;
      gload<LP, W>(a.x, gi + (tz - 1) * plane + (ty - 1) * P, c);
      if constexpr (kJZ) jz_row<LP, FTZ, FMA, W>(jd, jw, c);
      if (tz == 1 && ty == 1) ctr = c;
      ST prev = shup(rlast<LP, W>(c));
      ST next = shdn(rfirst<LP, W>(c));
      if (lane == 0) prev = ST(0);   // x = -1: only feeds the ghost output x = 0
      if (lane == 31) next = ST(0);  // x = P: the aliased ghost (zero)
      rshift<LP, W>(c, prev, next, L, R);
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int k = tz * 9 + ty * 3 + dx;
        if (SKIPF && is_face(k)) continue;
        rfma<LP, FTZ, FMA, W>(tapk(k), dx == 0 ? L : (dx == 1 ? c : R), acc);
      }
    }
  Row<LP, W> bb;
  if constexpr (kJZ) gload<LP, W>(a.x, gi, bb);  // operand == b
  else gload<LP, W>(a.b, gi, bb);
  if constexpr (LP == P16) {
    const __half2 m1 = u2h(0xBC00BC00u);
    Row<LP, W> r = efma<LP, FTZ, FMA, W>(m1, acc, bb);
    if constexpr (OP == POP_DEFECT) {
      if (x0 == 0) rzero_first<LP, W>(r);
      gstore<LP, W>(outp, gi, r);
    } else {
      const Row<LP, W> dr = emul<LP, FTZ, W>(a.d16, r);
      Row<LP, W> un = efma<LP, FTZ, FMA, W>(a.w16, dr, ctr);  // ctr: u, or u1 = w D^-1 b (JACOBI_Z)
      if (x0 == 0) rzero_first<LP, W>(un);
      gstore<LP, W>(outp, gi, un);
    }
  } else {
    const ST m1 = ST(-1), dd = LP == P32 ? (ST)a.d32 : (ST)a.d64, ww = LP == P32 ? (ST)a.w32 : (ST)a.w64;
    Row<LP, W> r = efma<LP, FTZ, FMA, W>(m1, acc, bb);
    if constexpr (OP == POP_DEFECT) {
      if (x0 == 0) rzero_first<LP, W>(r);
      gstore<LP, W>(outp, gi, r);
    } else {
      const Row<LP, W> dr = emul<LP, FTZ, W>(dd, r);
      Row<LP, W> un = efma<LP, FTZ, FMA, W>(ww, dr, ctr);
      if (x0 == 0) rzero_first<LP, W>(un);
      gstore<LP, W>(outp, gi, un);
    }
  }
}

}  // namespace mpmg_dev
