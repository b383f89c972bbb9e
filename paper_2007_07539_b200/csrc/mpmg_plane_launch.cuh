// Host launchers of the TMA-staged plane kernels (mpmg_plane.cuh). Included
// by one translation unit per operand precision so the instantiations
// compile in parallel.
#pragma once

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "mpmg_internal.h"
#include "mpmg_plane.cuh"
#include "mpmg_row2d.cuh"

namespace mpmg_impl {

using namespace mpmg_dev;

// CTA shape per (operand precision, compute precision, op, pitch); V > 0
// selects an alternative shape for tuning (MPMG_PLANE_VARIANT, binary16
// Jacobi only)
template <int LP, int CP, int OP, int P, int V = 0>
struct PlaneCfg {
  // (P = 192, the finest pitch of the paper's 193^3 grid: W = 6 everywhere)
  static constexpr int W = (V == 10 && P >= 128 && (P / 32) % 4 == 0) ? 4 : (P >= 256 ? 8 : P / 32);
  static constexpr int WX = P / (32 * W);
  static constexpr bool kWide = CP == P64 || (CP == P32 && LP != P16) || OP == POP_UPDATE || OP == POP_UPDATE_R;
  // output rows per thread and warp-rows per CTA
  static constexpr int RY0 = kWide ? 2 : 4;
  static constexpr int WY0 = WX >= 4 ? 1 : (WX == 2 ? 2 : 4);
  static constexpr int NS0 = kWide && W == 8 ? 3 : 4;
  static constexpr int RY = V == 1 ? 2 : (V == 2 ? 2 : (V == 3 ? 4 : (V == 5 ? 1 : RY0)));
  static constexpr int WY = V == 2 ? 8 : (V == 3 ? 2 : (V == 5 ? 8 : WY0));
  // (V = 10 at P = 1024: 3 stages, or the FP64 UPDATE stage (r, u rows of
  // 8 KB + c rows) would need 256 KB of shared memory)
  static constexpr int NS = V == 2 ? 3 : (V == 4 ? 3 : (V == 10 ? (P >= 1024 ? 3 : 4) : NS0));
  static constexpr int OPT = V == 4 ? 1 : (V == 11 ? 4 : (V == 12 ? 8 : 0));
};

inline int plane_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MPMG_PLANE_VARIANT");
    v = e ? std::atoi(e) : 0;
    if (v < 0 || v > 5) v = 0;
  }
  return v;
}

inline int plane_variant128() {  // the same shapes for the pitch-128 Jacobi (MPMG_PLANE_VARIANT128)
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MPMG_PLANE_VARIANT128");
    v = e ? std::atoi(e) : 0;
    if (v < 0 || v > 5) v = 0;
  }
  return v;
}

inline int outer_waves() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MPMG_OUTER_WAVES");
    v = e ? std::atoi(e) : 1;
    if (v < 1 || v > 64) v = 1;
  }
  return v;
}

// largest pitch run by the direct-load kernel (MPMG_DIRECT_MAX_P; measured:
// 3.65 vs 4.2 us per Jacobi step at 65^3, slower than k_plane from 129^3 up)
inline int direct_max_pitch() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MPMG_DIRECT_MAX_P");
    v = e ? std::atoi(e) : 64;
  }
  return v;
}

// smallest pitch the plane kernels take level ops for (MPMG_PLANE_MIN_P,
// tuning; below it the streaming stencil kernels run)
inline int plane_min_pitch() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MPMG_PLANE_MIN_P");
    v = e ? std::atoi(e) : 0;
  }
  return v;
}

// minimum output planes per CTA below pitch 256 (MPMG_ZMIN_SMALL, tuning)
inline int small_zmin() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MPMG_ZMIN_SMALL");
    v = e ? std::atoi(e) : 1;
    if (v < 1 || v > 64) v = 1;
  }
  return v;
}

inline __half2 h2_of(double v) {
  const __half h = __double2half(v);
  return __halves2half2(h, h);
}

// slab: nz owned planes with halo flags, or nullptr for the whole level
inline PlaneArgs plane_args(const mpmg_stencil& A, const mpmg_slab* slab = nullptr) {
  PlaneArgs a{};
  a.P = pitch(A.nodes);
  a.pz = slab ? slab->nz + 1 : a.P;
  a.load_lo = slab ? slab->halo_lo : 0;
  a.load_hi = slab ? slab->halo_hi : 0;
  a.plane = (long long)a.P * a.P;
  for (int i = 0; i < 27; ++i) {
    const double t = i < A.ntaps ? A.taps[i] : 0.0;
    a.t16[i] = h2_of(t);
    a.t32[i] = (float)t;
    a.t64[i] = t;
  }
  a.d16 = h2_of(A.inv_diag);
  a.d32 = (float)A.inv_diag;
  a.d64 = A.inv_diag;
  return a;
}

// number of SMs of the current device (cached)
int plane_num_sms();

template <int LP, int CP, int EP, int OP, bool FTZ, bool FMA, int P, int V = 0>
struct PlaneLaunch {
  using C = PlaneCfg<LP, CP, OP, P, V>;
  static constexpr bool SKIPF = CP == P16;
  using K = PlaneK<LP, CP, EP, OP, FTZ, FMA, SKIPF, C::W, C::WX, C::WY, C::RY, C::NS, C::OPT>;
  static constexpr auto kernel = k_plane<LP, CP, EP, OP, FTZ, FMA, SKIPF, C::W, C::WX, C::WY, C::RY, C::NS, C::OPT>;
  static_assert(K::kSmem + 512 <= 227 * 1024, "plane-kernel shared memory exceeds the sm_100a per-CTA limit");

  // grid: y-tiles x z-chunks, z-chunks sized so the grid is about one wave.
  // The wave is that of the FTZ-off/FMA-on build for every policy, so the
  // grid -- and the number of norm partials the FP64-epilogue ops write --
  // does not depend on the policy's register footprint (k_control sums
  // exactly the count mpmg_solver_create sized).
  static dim3 grid(int* zc, int pz = P) {
    static int per_sm = -1;
    if (per_sm < 0) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, K::kSmem);
      constexpr auto ref = k_plane<LP, CP, EP, OP, false, true, SKIPF, C::W, C::WX, C::WY, C::RY, C::NS, C::OPT>;
      cudaFuncSetAttribute(ref, cudaFuncAttributeMaxDynamicSharedMemorySize, K::kSmem);
      int n = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, ref, K::kThreads, K::kSmem);
      per_sm = n > 0 ? n : 1;
    }
    const int ytiles = (P - 1 + K::TY - 1) / K::TY;
    int cap = per_sm * plane_num_sms();
    // FP64 outer kernels (no z-halo on their FP64 streams): several waves of
    // shorter chunks even out the per-SM tail
    if constexpr (OP == POP_UPDATE || OP == POP_UPDATE_R || OP == POP_DEFECT64 || OP == POP_RESNORM)
      cap *= outer_waves();
    int chunks = cap / ytiles;
    if (chunks < 1) chunks = 1;
    if (chunks > pz - 1) chunks = pz - 1;
    int z = (pz - 1 + chunks - 1) / chunks;
    // small grids are latency-bound: as many CTAs as possible; large grids
    // keep >= 2 planes per chunk so the z-halo re-reads stay small
    const int zmin = P >= 256 ? 2 : small_zmin();
    if (z < zmin) z = zmin;
    *zc = z;
    return dim3(ytiles, (pz - 1 + z - 1) / z, 1);
  }

  static cudaError_t run(PlaneArgs a, cudaStream_t s) {
    int zc = 0;
    const dim3 g = grid(&zc, a.pz);
    a.zc = zc;
    a.ty = K::TY;
    return launch_pdl(kernel, g, dim3(K::kThreads), K::kSmem, s, a);
  }

  static int partials(int pz = P) {
    int zc = 0;
    const dim3 g = grid(&zc, pz);
    return (int)(g.x * g.y);
  }
};

// 2D levels through k_row2d: 16 bytes per lane, a 6-stage ring per warp,
// 4 warps per CTA, persistent grid of >= 8-row runs per warp
template <int LP, int OP, bool FTZ>
struct Row2dLaunch {
  static constexpr int W = 16 / Bytes<LP>::v;
  static constexpr int NS = 6, WPB = 4;
  using K = R2<LP, OP, W, NS>;
  static constexpr int kSmem = WPB * K::WARP_SMEM;
  static constexpr auto kernel = k_row2d<LP, OP, FTZ, W, NS, WPB>;
  static int blocks() {
    static int nb = -1;
    if (nb < 0) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
      int n = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, 32 * WPB, kSmem);
      nb = (n > 0 ? n : 1) * plane_num_sms();
    }
    return nb;
  }
  static cudaError_t run(const PlaneArgs& a, cudaStream_t s) {
    const long long T = (long long)(a.P / K::SEG) * (a.P - 1);
    long long nb = blocks();
    const long long want = (T / 8 + WPB - 1) / WPB;
    if (want < nb) nb = want > 0 ? want : 1;
    return launch_pdl(kernel, dim3((unsigned)nb), dim3(32 * WPB), kSmem, s, a);
  }
};

// smallest 2D pitch k_row2d takes (MPMG_ROW2D_MINP; 0 disables it)
inline int row2d_min_pitch() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MPMG_ROW2D_MINP");
    v = e ? std::atoi(e) : 64;
  }
  return v;
}

// dispatch on the pitch; returns false when the plane kernels do not cover P
template <typename F>
inline bool with_pitch(int P, F&& f) {
  switch (P) {
    case 32: f(std::integral_constant<int, 32>{}); return true;
    case 64: f(std::integral_constant<int, 64>{}); return true;
    case 128: f(std::integral_constant<int, 128>{}); return true;
    case 192: f(std::integral_constant<int, 192>{}); return true;
    case 256: f(std::integral_constant<int, 256>{}); return true;
    case 512: f(std::integral_constant<int, 512>{}); return true;
    case 1024: f(std::integral_constant<int, 1024>{}); return true;
    default: return false;
  }
}

inline bool aligned16(const void* p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; }

// the binary16 plane / direct kernels drop the six face taps and keep one
// value per tap class (tap_class): they run only when, in binary16, the faces
// are exactly zero and the 12 edge and the 8 corner taps are each one value
// (true on every level of the hierarchy); anything else takes the stencil
// kernels
inline bool sym16(const mpmg_stencil& A) {
  if (A.ntaps != 27) return false;
  uint16_t rep[4] = {0, 0, 0, 0};
  bool seen[4] = {false, false, false, false};
  for (int k = 0; k < 27; ++k) {
    const __half h = __double2half(A.taps[k]);
    uint16_t bits;
    memcpy(&bits, &h, 2);
    const int c = tap_class(k);
    if (c == 1) {
      if (__half2float(h) != 0.0f) return false;
      continue;
    }
    if (!seen[c]) { seen[c] = true; rep[c] = bits; }
    else if (rep[c] != bits) return false;
  }
  return true;
}

// level op (1 DEFECT / 2 JACOBI / 3 two JACOBI steps from zero, x = b) through
// the plane kernels; false if not covered
// z-slab level op whose boundary output planes are also pushed into the
// neighbours' halo planes (push_lo / push_hi, either may be null): JACOBI
// (op 2) and DEFECT (op 1) on 3D slabs; false if not covered
template <int LP>
bool plane_level_op_push(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                         uint32_t policy, cudaStream_t s, cudaError_t* err, const mpmg_slab* slab, void* push_lo,
                         void* push_hi) {
  if (A.dim != 3 || !slab || (op != 1 && op != 2)) return false;
  if (!(policy & MPMG_FMA) || (LP == P16 && (policy & MPMG_ACC32))) return false;
  if (LP == P16 && !sym16(A)) return false;
  if (!aligned16(x) || !aligned16(b) || !aligned16(out) || !aligned16(push_lo) || !aligned16(push_hi)) return false;
  PlaneArgs a = plane_args(A, slab);
  a.x = x; a.b = b; a.out = out;
  a.push_lo = push_lo; a.push_hi = push_hi;
  const bool ftz = policy & MPMG_FTZ;
  const double w = round_to(omega, LP, ftz);
  a.w16 = h2_of(w); a.w32 = (float)w; a.w64 = w;
  return with_pitch(a.P, [&](auto pc) {
    constexpr int PP = decltype(pc)::value;
    if (op == 1) *err = ftz ? PlaneLaunch<LP, LP, LP, POP_DEFECT, true, true, PP, 12>::run(a, s)
                            : PlaneLaunch<LP, LP, LP, POP_DEFECT, false, true, PP, 12>::run(a, s);
    else *err = ftz ? PlaneLaunch<LP, LP, LP, POP_JACOBI, true, true, PP, 12>::run(a, s)
                    : PlaneLaunch<LP, LP, LP, POP_JACOBI, false, true, PP, 12>::run(a, s);
  });
}

template <int LP>
bool plane_level_op(int op, const mpmg_stencil& A, const void* x, const void* b, void* out, double omega,
                    uint32_t policy, cudaStream_t s, cudaError_t* err, const mpmg_slab* slab = nullptr,
                    const int* out_slot = nullptr, long long out_stride = 0) {
  if (A.dim == 2 && (op == 1 || op == 2 || op == 3) && !slab && !out_slot && (policy & MPMG_FMA) &&
      !(LP == P16 && (policy & MPMG_ACC32))) {
    const int P = pitch(A.nodes);
    constexpr int SEG = 32 * 16 / Bytes<LP>::v;
    if (row2d_min_pitch() > 0 && P >= row2d_min_pitch() && P >= SEG && P % SEG == 0 && aligned16(x) &&
        aligned16(b) && aligned16(out)) {
      PlaneArgs a = plane_args(A, nullptr);
      a.x = x; a.b = b; a.out = out;
      const bool ftz = policy & MPMG_FTZ;
      const double w = round_to(omega, LP, ftz);
      a.w16 = h2_of(w); a.w32 = (float)w; a.w64 = w;
      auto go = [&](auto opc) {
        constexpr int O = decltype(opc)::value;
        *err = ftz ? Row2dLaunch<LP, O, true>::run(a, s) : Row2dLaunch<LP, O, false>::run(a, s);
      };
      if (op == 1) go(std::integral_constant<int, POP_DEFECT>{});
      else if (op == 3) go(std::integral_constant<int, POP_JACOBI_Z>{});
      else go(std::integral_constant<int, POP_JACOBI>{});
      return true;
    }
  }
  if (A.dim != 3 || (op != 1 && op != 2 && op != 3)) return false;
  if (pitch(A.nodes) < plane_min_pitch()) return false;
  if (!(policy & MPMG_FMA) || (LP == P16 && (policy & MPMG_ACC32))) return false;
  if (LP == P16 && !sym16(A)) return false;
  if (!aligned16(x) || !aligned16(b) || !aligned16(out)) return false;
  PlaneArgs a = plane_args(A, slab);
  a.x = x; a.b = b; a.out = out;
  a.out_slot = out_slot; a.out_stride = out_stride;
  const bool ftz = policy & MPMG_FTZ;
  const double w = round_to(omega, LP, ftz);
  a.w16 = h2_of(w); a.w32 = (float)w; a.w64 = w;
  return with_pitch(a.P, [&](auto pc) {
    constexpr int PP = decltype(pc)::value;
    if (out_slot) {  // Jacobi step into a ring slot (V = 11: the OPT bit-2 instantiation)
      *err = ftz ? PlaneLaunch<LP, LP, LP, POP_JACOBI, true, true, PP, 11>::run(a, s)
                 : PlaneLaunch<LP, LP, LP, POP_JACOBI, false, true, PP, 11>::run(a, s);
      return;
    }
    if constexpr (PP <= 256) {
      if (!slab && PP <= direct_max_pitch()) {  // small L2-resident level: direct loads
        constexpr int W = PP / 32;
        constexpr bool SK = LP == P16;
        const dim3 g((unsigned)(((PP - 1) * (PP - 1) + 3) / 4));
        auto go = [&](auto kern) { *err = launch_pdl(kern, g, dim3(128), 0, s, a); };
        if (op == 1) ftz ? go(k_direct<LP, POP_DEFECT, true, true, SK, W>) : go(k_direct<LP, POP_DEFECT, false, true, SK, W>);
        else if (op == 3) ftz ? go(k_direct<LP, POP_JACOBI_Z, true, true, SK, W>)
                              : go(k_direct<LP, POP_JACOBI_Z, false, true, SK, W>);
        else ftz ? go(k_direct<LP, POP_JACOBI, true, true, SK, W>) : go(k_direct<LP, POP_JACOBI, false, true, SK, W>);
        return;
      }
    }
    if (op == 1) *err = ftz ? PlaneLaunch<LP, LP, LP, POP_DEFECT, true, true, PP>::run(a, s)
                            : PlaneLaunch<LP, LP, LP, POP_DEFECT, false, true, PP>::run(a, s);
    else if (op == 3) *err = ftz ? PlaneLaunch<LP, LP, LP, POP_JACOBI_Z, true, true, PP>::run(a, s)
                                 : PlaneLaunch<LP, LP, LP, POP_JACOBI_Z, false, true, PP>::run(a, s);
    else {
      if constexpr (LP == P16 && (PP == 256 || PP == 128)) {  // tuning shapes (MPMG_PLANE_VARIANT[128])
        const int pv = PP == 256 ? plane_variant() : plane_variant128();
        if (!ftz && pv > 0) {
          switch (pv) {
            case 1: *err = PlaneLaunch<LP, LP, LP, POP_JACOBI, false, true, PP, 1>::run(a, s); break;
            case 2: *err = PlaneLaunch<LP, LP, LP, POP_JACOBI, false, true, PP, 2>::run(a, s); break;
            case 3: *err = PlaneLaunch<LP, LP, LP, POP_JACOBI, false, true, PP, 3>::run(a, s); break;
            case 4: *err = PlaneLaunch<LP, LP, LP, POP_JACOBI, false, true, PP, 4>::run(a, s); break;
            default: *err = PlaneLaunch<LP, LP, LP, POP_JACOBI, false, true, PP, 5>::run(a, s); break;
          }
          return;
        }
      }
      *err = ftz ? PlaneLaunch<LP, LP, LP, POP_JACOBI, true, true, PP>::run(a, s)
                 : PlaneLaunch<LP, LP, LP, POP_JACOBI, false, true, PP>::run(a, s);
    }
  });
}

}  // namespace mpmg_impl
