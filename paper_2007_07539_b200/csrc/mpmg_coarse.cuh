#pragma once
// Coarse part of the V-cycle in ONE persistent cooperative launch: every
// level with <= kCoarsePoints interior unknowns (127^3 / 1447^2 and below:
// the levels whose per-launch work is too small to hide a kernel launch and
// a pipeline ramp) runs inside a single grid -- pre-smoothing, defect,
// restriction (with the DSH rescale), the CG base solve on level 0,
// prolongation + correction and post-smoothing -- separated by grid-wide
// barriers instead of kernel launches. Levels with <= kCtaPoints unknowns
// are worked by CTA 0 alone out of shared memory with __syncthreads; the
// other CTAs wait at the next grid barrier. This replaces the coarse part of
// the reference's recursion (cycle_at, multigrid.cpp:362-393) and cg_solve
// (multigrid.cpp:91-151).
//
// Arithmetic is the same per-operation rounding as the streaming kernels
// (policy as template parameters). The grid levels live in global memory
// (L2-resident at these sizes; grid.sync() orders and publishes the writes
// of one step to the next). Reductions the reference accumulates
// sequentially (dot_fp64 / norm2_fp64, kernels.cpp:368-395; the DSH
// restriction norm, multigrid.cpp:246-250) run on one thread in the
// reference's lexicographic order, so the base solve is bitwise identical to
// the reference.
#include <cooperative_groups.h>

#include <type_traits>

#include "mpmg_arith.cuh"
#include "mpmg_internal.h"

#include <algorithm>
#include <cstdlib>

namespace mpmg_impl {

using namespace mpmg_dev;

namespace coarse_detail {

constexpr int kThreads = 512;
constexpr int kCtaPoints = 4096;

template <int PR> struct T_;
template <> struct T_<P16> { using T = __half; };
template <> struct T_<P32> { using T = float; };
template <> struct T_<P64> { using T = double; };

// loads of data written earlier in this launch (plain loads: grid.sync()
// and __syncthreads order them after the writes)
template <typename T>
__device__ __forceinline__ T ldcg(const T* p) { return *p; }

template <int PR, bool FTZ, bool FMA, bool ACC32>
struct Lv {
  using T = typename T_<PR>::T;
  static __device__ __forceinline__ T from(double v) {
    if constexpr (PR == P16) return round16<FTZ>(v);
    else if constexpr (PR == P32) return round32<FTZ>(v);
    else return v;
  }
  static __device__ __forceinline__ double wide(T v) {
    if constexpr (PR == P16) return (double)__half2float(v);
    else return (double)v;
  }
  static __device__ __forceinline__ T zero() { return T(0); }
  static __device__ __forceinline__ T fma(T a, T b, T c) {
    if constexpr (PR == P16) return fma16s<FTZ, FMA>(a, b, c);
    else if constexpr (PR == P32) return fma32<FTZ, FMA>(a, b, c);
    else return fma64<FMA>(a, b, c);
  }
  static __device__ __forceinline__ T mul(T a, T b) {
    if constexpr (PR == P16) return mul16s<FTZ>(a, b);
    else if constexpr (PR == P32) return mul32<FTZ>(a, b);
    else return mul64(a, b);
  }
  // transfer weight 2^-k, exact in the compute precision (no conversion)
  static __device__ __forceinline__ T weight(int k) {
    if constexpr (PR == P16) return __ushort_as_half((unsigned short)(0x3C00 - (k << 10)));
    else if constexpr (PR == P32) return __int_as_float(0x3F800000 - (k << 23));
    else return __longlong_as_double(0x3FF0000000000000LL - ((long long)k << 52));
  }
  // transfer_product step (multigrid.cpp:166-195): FP32 unfused flushes only the sum
  static __device__ __forceinline__ T xfer(T w, T x, T acc) {
    if constexpr (PR == P32) return f32<FTZ>(FMA ? __fmaf_rn(w, x, acc) : __fadd_rn(__fmul_rn(w, x), acc));
    else return fma(w, x, acc);
  }
  // the level's taps in the compute precision, converted once per operation
  struct Taps {
    T t[27];
    float f[27];
  };
  // (t16/t32: the level's taps pre-rounded once per launch in shared memory)
  static __device__ __forceinline__ Taps taps(const CoarseLevel& L, const __half* t16, const float* t32) {
    Taps k;
#pragma unroll
    for (int t = 0; t < 27; ++t) {
      if constexpr (PR == P16) k.t[t] = t16[t];
      else if constexpr (PR == P32) k.t[t] = t32[t];
      else k.t[t] = L.taps[t];
      k.f[t] = t32[t];
    }
    return k;
  }
  // A x at one point (all 3^dim taps in slot order; ghosts are zero);
  // ld(dz, dy, dx) returns the neighbour value
  template <int DIM, typename LD>
  static __device__ __forceinline__ T apply_f(const Taps& k, LD&& ld) {
    if constexpr (PR == P16 && ACC32) {  // Fp16Accum::FP32 (kernels.cpp:151-162)
      float acc = 0.0f;
      int t = 0;
#pragma unroll
      for (int dz = (DIM == 3 ? -1 : 0); dz <= (DIM == 3 ? 1 : 0); ++dz)
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
          for (int dx = -1; dx <= 1; ++dx, ++t) acc = fma32<FTZ, FMA>(k.f[t], __half2float(ld(dz, dy, dx)), acc);
      return f16s<FTZ>(__float2half_rn(acc));
    } else {
      T acc = zero();
      int t = 0;
#pragma unroll
      for (int dz = (DIM == 3 ? -1 : 0); dz <= (DIM == 3 ? 1 : 0); ++dz)
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
          for (int dx = -1; dx <= 1; ++dx, ++t) acc = fma(k.t[t], ld(dz, dy, dx), acc);
      return acc;
    }
  }
  template <int DIM>
  static __device__ __forceinline__ T apply_d(const Taps& k, const T* x, int i, int P) {
    const int pl = DIM == 3 ? P * P : 0;
    return apply_f<DIM>(k, [&](int dz, int dy, int dx) { return ldcg(x + i + dz * pl + dy * P + dx); });
  }
  static __device__ __forceinline__ T apply(const Taps& k, int dim, const T* x, int i, int P) {
    return dim == 3 ? apply_d<3>(k, x, i, P) : apply_d<2>(k, x, i, P);
  }
  // A x on a one-unknown level: every neighbour is a (zero) ghost, so
  // apply()'s chain is +0 until the centre tap and unchanged after it (the
  // taps are finite: fma(t, +0, acc) = acc + (+-0) = acc for acc != 0, and
  // acc = +0 stays +0) -- bitwise the centre term alone, on a register.
  static __device__ __forceinline__ T apply1(const Taps& k, int dim, T x) {
    const int c = dim == 3 ? 13 : 4;
    if constexpr (PR == P16 && ACC32) return f16s<FTZ>(__float2half_rn(fma32<FTZ, FMA>(k.f[c], __half2float(x), 0.0f)));
    else return fma(k.t[c], x, zero());
  }
};

struct Pt {
  int n, m, P, dim;
  unsigned magic;  // ceil(2^32 / m): k / m == umulhi(k, magic) for k < 2^32 / m
  // compact k -> interior coordinates (1-based; z = 0 in 2D)
  __device__ __forceinline__ void xyz(int k, int& x, int& y, int& z) const {
    const unsigned q = __umulhi((unsigned)k, magic);
    x = k - (int)q * m + 1;
    if (dim == 2) { y = (int)q + 1; z = 0; return; }
    const unsigned zz = __umulhi(q, magic);
    y = (int)(q - zz * m) + 1;
    z = (int)zz + 1;
  }
  __device__ __forceinline__ int idx(int k) const {  // compact k -> padded index
    const unsigned q = __umulhi((unsigned)k, magic);
    const int x = k - (int)q * m + 1;
    if (dim == 2) return ((int)q + 1) * P + x;
    const unsigned z = __umulhi(q, magic);
    return (((int)z + 1) * P + (int)(q - z * m) + 1) * P + x;
  }
};

__device__ __forceinline__ Pt points(const CoarseLevel& L) {
  Pt p;
  p.P = L.nodes - 1;
  p.m = p.P - 1;
  p.dim = L.dim;
  p.n = L.dim == 3 ? p.m * p.m * p.m : p.m * p.m;
  p.magic = 0xFFFFFFFFu / (unsigned)p.m + 1u;
  return p;
}

__device__ __forceinline__ void grid_sync() { cooperative_groups::this_grid().sync(); }
// all CTAs of the (single-cluster) grid: the hardware cluster barrier, with
// release/acquire at cluster scope ordering the global-memory level data
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}

// ---- cluster slab mode ----------------------------------------------------
// One thread-block cluster of C CTAs runs the coarse cycle with every level
// above the CTA-0 levels split into z-slabs that live in the CTAs' shared
// memory (one halo plane each side, pushed to the neighbours through
// distributed shared memory after every operation) -- an operation is local
// shared-memory work plus one hardware cluster barrier instead of L2 round
// trips plus a grid-wide barrier. Ownership nests: CTA r owns planes
// [lo_T(r), lo_T(r+1)) of the top level T, lo_T(r) = 1 + r (P_T - 1) / C, and
// coarse plane k wherever it owns fine plane 2k: lo_l(r) = ceil(lo_T(r) / 2^(T-l)).
__host__ __device__ inline int slab_lo(int P_top, int C, int shift, int r) {
  const int lt = 1 + (r * (P_top - 1)) / C;
  return (lt + (1 << shift) - 1) >> shift;
}
// elements of one slab buffer of a level with pitch P and at most nz owned planes
// (halo planes included; the top halo plane's aliased x = P / y = P ghosts
// reach P + 1 values past it)
__host__ __device__ inline long long slab_elems(int P, int nz) { return (long long)(nz + 2) * P * P + P + 1; }
__host__ __device__ inline int slab_max_nz(int P_top, int C, int shift) {
  int m = 0;
  for (int r = 0; r < C; ++r) {
    const int nz = slab_lo(P_top, C, shift, r + 1) - slab_lo(P_top, C, shift, r);
    m = nz > m ? nz : m;
  }
  return m;
}

// halo pushes of one CTA on one slab level: plane src (local plane index) to
// CTA t's local plane dst; CTA t reads planes lo_t - 1 and hi_t
struct PushTab {
  int n;
  signed char t[8], src[8], dst[8];
};

// UP: the one precision of every level (P16/P32/P64: H_MG, D_MG -- a single
// code path, a third of the instruction footprint), or 3 for mixed cascades
template <bool FTZ, bool FMA, bool ACC32, int UP>
struct Coarse {
  const CoarseArgs& a;
  unsigned rank, ncta;
  CoarseLevel* lv;  // level table in shared memory: CTA 0's small levels point into shared memory
  void* const* cgp;  // CG scratch r, p, ap, s, best
  const __half (*t16)[27];
  const float (*t32)[27];
  const bool slab;  // cluster slab mode (else a cooperative grid, level data in global memory)
  // per-level point geometry and CTA-0 flag, computed once per launch (shared
  // memory) -- points() divides, and every operation asks several times
  const Pt* spt = nullptr;
  const unsigned char* ssmall = nullptr;
  __device__ const Pt& pt(const CoarseLevel& L) const { return spt[&L - lv]; }
  __device__ Coarse(const CoarseArgs& args, CoarseLevel* table, void* const* cg, const __half (*a16)[27],
                    const float (*a32)[27], bool cluster)
      : a(args), rank(blockIdx.x), ncta(gridDim.x), lv(table), cgp(cg), t16(a16), t32(a32), slab(cluster) {}
  __device__ void gsync() {
    if (slab) cluster_sync();
    else grid_sync();
  }
  // slab mode: owned planes [lo(l, r), lo(l, r + 1)) of level l (table in
  // shared memory, filled at kernel start)
  const short (*slo)[17] = nullptr;
  const PushTab* push = nullptr;  // per level: planes this CTA pushes, and to whom
  __device__ int lo(int l, int r) const { return slo[l][r]; }

  template <int PR>
  __device__ typename Lv<PR, FTZ, FMA, ACC32>::Taps taps_of(const CoarseLevel& L) const {
    const int l = (int)(&L - lv);
    return Lv<PR, FTZ, FMA, ACC32>::taps(L, t16[l], t32[l]);
  }

  template <int PR> using O = Lv<PR, FTZ, FMA, ACC32>;

  __device__ bool small(const CoarseLevel& L) const { return ssmall[&L - lv] != 0; }
  long long t0 = 0;
  int nst = 0;
  // phase timestamps (MPMG_COARSE_DEBUG): code*1e12 + cycles since start,
  // kept in registers by thread 0 of CTA 0 and written to a.dbg at the end
  // (MPMG_COARSE_DEBUG = 3 + r records CTA r's stamps, with the fine-grained ones)
  __device__ unsigned stamp_rank() const { return a.debug >= 3 ? (unsigned)(a.debug - 3) : 0u; }
  __device__ void stamp(int code, int l) {
    if (a.dbg && rank == stamp_rank() && threadIdx.x == 0 && nst < 63)
      a.dbg[1 + nst++] = (long long)(code * 100 + l) * 1000000000000LL + (clock64() - t0);
  }
  __device__ void stamps_done() {
    if (a.dbg && rank == stamp_rank() && threadIdx.x == 0) a.dbg[0] = nst;
  }
  // team of a level: the whole grid, or CTA 0 alone
  __device__ bool in_team(const CoarseLevel& L) const { return !small(L) || rank == 0; }
  __device__ void sync(const CoarseLevel& L) {
    if (small(L)) __syncthreads();
    else gsync();
  }

  template <typename F>
  __device__ void for_points(const CoarseLevel& L, F&& f) {
    for_points_by(L, small(L) ? 0 : (slab ? 2 : 1), f);
  }
  // mode 0: each CTA walks every point; 1: the points are spread over the
  // grid; 2 (slab mode): this CTA's planes
  // as for_points_by, with the point's coordinates: f(i, x, y, z, P)
  template <typename F>
  __device__ void for_points_xyz(const CoarseLevel& L, int mode, F&& f) {
    const Pt p = pt(L);
    int start = threadIdx.x, stride = blockDim.x, end = p.n;
    if (mode == 1) { start += (int)rank * blockDim.x; stride *= (int)ncta; }
    if (mode == 2) {
      const int l = (int)(&L - lv);
      const int m2 = p.m * p.m;
      start += (lo(l, (int)rank) - 1) * m2;
      end = (lo(l, (int)rank + 1) - 1) * m2;
    }
    for (int k = start; k < end; k += stride) {
      int x, y, z;
      p.xyz(k, x, y, z);
      f((z * p.P + y) * p.P + x, x, y, z, p.P);
    }
  }
  template <typename F>
  __device__ void for_points_by(const CoarseLevel& L, int mode, F&& f) {
    const Pt p = pt(L);
    int start = threadIdx.x, stride = blockDim.x, end = p.n;
    if (mode == 1) { start += (int)rank * blockDim.x; stride *= (int)ncta; }
    if (mode == 2) {
      const int l = (int)(&L - lv);
      const int m2 = p.m * p.m;
      start += (lo(l, (int)rank) - 1) * m2;
      end = (lo(l, (int)rank + 1) - 1) * m2;
    }
    for (int k = start; k < end; k += stride) f(p.idx(k), p.P);
  }
  // slab mode: push this CTA's first / last owned plane of buffer x (level l)
  // into the halo planes of every CTA that reads it -- CTA t reads planes
  // lo_t - 1 and hi_t (also when its own slab is empty) -- then a cluster
  // barrier. Halo planes outside 1..P-1 are ghost planes and stay zero.
  __device__ void exchange(int l, void* x) {
    const CoarseLevel& L = lv[l];
    const int P = L.nodes - 1;
    const int bytes = L.prec == MPMG_FP16 ? 2 : (L.prec == MPMG_FP32 ? 4 : 8);
    const int pl = P * P * bytes;  // plane bytes: a multiple of 8 (P is even on a slab level)
    const int zlo = lo(l, (int)rank);
    __syncthreads();
    const int cnt = push[l].n;
    if (cnt > 0 && (pl & 15) != 0) {  // binary16 with P = 2 mod 4: 8-byte words
      const uint32_t real = (uint32_t)__cvta_generic_to_shared(static_cast<unsigned char*>(x) + (long long)(zlo - 1) * pl);
      const int n8 = pl / 8;
      for (int i = threadIdx.x; i < cnt * n8; i += blockDim.x) {
        const int k = i / n8, c = i - k * n8;
        uint32_t dst;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                     : "=r"(dst) : "r"(real + (uint32_t)push[l].dst[k] * (uint32_t)pl), "r"((int)push[l].t[k]));
        uint2 v;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                     : "=r"(v.x), "=r"(v.y) : "r"(real + (uint32_t)push[l].src[k] * (uint32_t)pl + 8u * c));
        asm volatile("st.shared::cluster.v2.u32 [%0], {%1, %2};" :: "r"(dst + 8u * c), "r"(v.x), "r"(v.y) : "memory");
      }
    } else if (cnt > 0) {
      // shared-window addresses: ld.shared locally, st.shared::cluster remotely
      const uint32_t real = (uint32_t)__cvta_generic_to_shared(static_cast<unsigned char*>(x) + (long long)(zlo - 1) * pl);
      const int n16 = pl / 16;
      for (int i = threadIdx.x; i < cnt * n16; i += blockDim.x) {
        const int k = i / n16, c = i - k * n16;
        uint32_t dst;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                     : "=r"(dst) : "r"(real + (uint32_t)push[l].dst[k] * (uint32_t)pl), "r"((int)push[l].t[k]));
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(real + (uint32_t)push[l].src[k] * (uint32_t)pl + 16u * c));
        asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};"
                     :: "r"(dst + 16u * c), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
      }
    }
    if (a.debug > 1) stamp(9, l);
    cluster_sync();
  }

  template <typename F>
  __device__ void by_prec(int prec, F&& f) {
    if constexpr (UP < 3) {
      (void)prec;
      f(std::integral_constant<int, UP>{});
    } else {
      if (prec == MPMG_FP16) f(std::integral_constant<int, P16>{});
      else if (prec == MPMG_FP32) f(std::integral_constant<int, P32>{});
      else f(std::integral_constant<int, P64>{});
    }
  }

  // binary16 slab levels (3D): two x-neighbours per thread in one half2 --
  // three aligned 32-bit loads per stencil row, the x-1 / x+1 pairs by byte
  // permutes, HFMA2 on both nodes in the slot order of apply() (each lane is
  // the scalar chain, bitwise). DEF: defect r = b - A u, else a Jacobi step.
  // The pair (0, 1) computes the x = 0 ghost and stores it as zero.
  template <bool DEF>
  __device__ void pairs16(const CoarseLevel& L, const void* bv, const void* uv, void* ov, bool from_zero) {
    using OP = O<P16>;
    const int l = (int)(&L - lv);
    const int P = L.nodes - 1, P2 = P * P, hp = P / 2;
    // a slab level: this CTA's planes; a CTA-0 level (in CTA 0's shared memory): all
    const bool whole = small(L);
    const int zlo = whole ? 1 : lo(l, (int)rank), nz = whole ? P - 1 : lo(l, (int)rank + 1) - zlo;
    const int np = (P - 1) * hp;  // pairs per plane
    // 32-bit shared-window addresses of the virtual bases (global plane z at
    // base + 2 z P^2; modular arithmetic, only in-slab addresses are formed)
    const uint32_t su = (uint32_t)__cvta_generic_to_shared(static_cast<const __half*>(uv) + (long long)(zlo - 1) * P2) -
                        (uint32_t)((zlo - 1) * P2 * 2);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(static_cast<const __half*>(bv) + (long long)(zlo - 1) * P2) -
                        (uint32_t)((zlo - 1) * P2 * 2);
    const uint32_t so = (uint32_t)__cvta_generic_to_shared(static_cast<__half*>(ov) + (long long)(zlo - 1) * P2) -
                        (uint32_t)((zlo - 1) * P2 * 2);
    const auto tk = taps_of<P16>(L);
    __half2 t2[27];
#pragma unroll
    for (int t = 0; t < 27; ++t) t2[t] = __half2half2(tk.t[t]);
    int roff[9];  // byte offsets of the 9 stencil rows
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy) roff[(dz + 1) * 3 + dy + 1] = 2 * (dz * P2 + dy * P);
    const __half2 m1 = u2h(0xBC00BC00u);
    const __half2 w = __half2half2(OP::from(L.omega)), d = __half2half2(OP::from(L.inv_diag));
    const __half2 z2 = u2h(0u);
    for (int t = threadIdx.x; t < np * nz; t += blockDim.x) {  // (pair, plane) items
      const int zq = t / np, k = t - zq * np;
      const int y = 1 + k / hp, x = 2 * (k - (y - 1) * hp);
      {
        const uint32_t off = 2u * (uint32_t)((zlo + zq) * P2 + y * P + x);
        __half2 acc = z2, uc = z2;
        if (DEF || !from_zero) {
#pragma unroll
          for (int rw = 0; rw < 9; ++rw) {
            const uint32_t a0 = su + off + (uint32_t)roff[rw];
            uint32_t w0, w1, w2;
            asm volatile("ld.shared.u32 %0, [%1+-4];" : "=r"(w0) : "r"(a0));
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w1) : "r"(a0));
            asm volatile("ld.shared.u32 %0, [%1+4];" : "=r"(w2) : "r"(a0));
            const __half2 lft = u2h(__byte_perm(w0, w1, 0x5432)), rgt = u2h(__byte_perm(w1, w2, 0x5432));
            acc = fma16<FTZ, FMA>(t2[3 * rw], lft, acc);
            acc = fma16<FTZ, FMA>(t2[3 * rw + 1], u2h(w1), acc);
            acc = fma16<FTZ, FMA>(t2[3 * rw + 2], rgt, acc);
            if (rw == 4) uc = u2h(w1);
          }
        }
        uint32_t bw;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(bw) : "r"(sb + off));
        const __half2 r = fma16<FTZ, FMA>(m1, acc, u2h(bw));
        __half2 out = DEF ? r : fma16<FTZ, FMA>(w, mul16<FTZ>(d, r), uc);
        uint32_t ow = h2u(out);
        if (x == 0) ow &= 0xFFFF0000u;  // ghost node stays +0
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(so + off), "r"(ow) : "memory");
      }
    }
  }
  // slab mode: every 3D level with an even pitch -- slab levels, and CTA 0's
  // levels (whose buffers CTA 0 addresses as plain shared memory)
  __device__ bool pairs_ok(const CoarseLevel& L) const {
    return slab && (!small(L) || rank == 0) && L.dim == 3 && ((L.nodes - 1) & 1) == 0;
  }

  template <int PR>
  __device__ void jacobi(const CoarseLevel& L, const void* bv, const void* uin, void* uout, bool from_zero) {
    if constexpr (PR == P16 && !ACC32) {
      if (pairs_ok(L)) { pairs16<false>(L, bv, uin, uout, from_zero); return; }
    }
    using OP = O<PR>;
    using T = typename OP::T;
    const T* b = static_cast<const T*>(bv);
    const T* u = static_cast<const T*>(uin);
    T* o = static_cast<T*>(uout);
    const T w = OP::from(L.omega), d = OP::from(L.inv_diag), m1 = OP::from(-1.0);
    const auto tk = taps_of<PR>(L);
    for_points(L, [&](int i, int P) {
      const T t = from_zero ? OP::zero() : OP::apply(tk, L.dim, u, i, P);
      const T r = OP::fma(m1, t, ldcg(b + i));
      o[i] = OP::fma(w, OP::mul(d, r), from_zero ? OP::zero() : ldcg(u + i));
    });
  }

  template <int PR>
  __device__ void defect(const CoarseLevel& L, const void* bv, const void* uv, void* rv) {
    if constexpr (PR == P16 && !ACC32) {
      if (pairs_ok(L)) { pairs16<true>(L, bv, uv, rv, false); return; }
    }
    using OP = O<PR>;
    using T = typename OP::T;
    const T m1 = OP::from(-1.0);
    const auto tk = taps_of<PR>(L);
    for_points(L, [&](int i, int P) {
      static_cast<T*>(rv)[i] = OP::fma(m1, OP::apply(tk, L.dim, static_cast<const T*>(uv), i, P), ldcg(static_cast<const T*>(bv) + i));
    });
  }

  // R r_f (product in the fine precision FP) -> coarse b; when `keep`, the
  // binary64 products go to C.prod first (DSH rescale norm)
  // A grid level restricting into a CTA-0 level (the entry level) spreads
  // the coarse points over the grid and writes the global copy of C.b, which
  // stage_in then brings into CTA 0's shared memory.
  template <int FP>
  __device__ void restrict_to(const CoarseLevel& F, const CoarseLevel& Cin, const void* rfv, bool keep) {
    using OF = O<FP>;
    using T = typename OF::T;
    const T* rf = static_cast<const T*>(rfv);
    const int Pf = F.nodes - 1;
    const int pf = F.dim == 3 ? Pf * Pf : 0;
    const bool spread = !keep && !small(F) && small(Cin) && !slab;
    const CoarseLevel& C = Cin;
    void* const cb = spread ? a.lv[&Cin - lv].b : C.b;
    // slab mode: coarse plane k is computed by the owner of fine plane 2k
    // (and written to CTA 0's shared memory when the coarse level is a CTA-0 level)
    const int mode = (slab && !small(F)) ? 2 : ((spread || !small(C)) ? 1 : 0);
    for_points_xyz(C, mode, [&](int ci, int cx, int cy, int cz, int Pc) {
      const int cf = cz * 2 * pf + cy * 2 * Pf + cx * 2;
      T acc = OF::zero();
      for (int dz = (F.dim == 3 ? -1 : 0); dz <= (F.dim == 3 ? 1 : 0); ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            acc = OF::xfer(OF::weight((dx != 0) + (dy != 0) + (dz != 0)), ldcg(rf + cf + dz * pf + dy * Pf + dx), acc);
          }
      if (keep) C.prod[ci] = OF::wide(acc);
      else by_prec(C.prec, [&](auto cp) {
        using OC = O<decltype(cp)::value>;
        static_cast<typename OC::T*>(cb)[ci] = OC::from(OF::wide(acc));  // scale 1
      });
    });
  }

  template <int CPc>
  __device__ void restrict_store(const CoarseLevel& C, double scale) {
    using OC = O<CPc>;
    for_points(C, [&](int ci, int) {
      static_cast<typename OC::T*>(C.b)[ci] = OC::from(C.prod[ci] / scale);
    });
  }

  // u_f += round_f(scale * P c) (product in the coarse precision)
  template <int FP, int CPc>
  __device__ void prolong(const CoarseLevel& F, const CoarseLevel& C, const void* ccv, void* ufv, double scale) {
    using OC = O<CPc>;
    using OF = O<FP>;
    using TC = typename OC::T;
    using TF = typename OF::T;
    const TC* cc = static_cast<const TC*>(ccv);
    TF* uf = static_cast<TF*>(ufv);
    const int Pc = C.nodes - 1;
    for_points_xyz(F, small(F) ? 0 : (slab ? 2 : 1), [&](int fi, int fx, int fy, int fz, int Pf) {
      const int nx = (fx & 1) ? 2 : 1, ny = (fy & 1) ? 2 : 1, nz = F.dim == 3 ? ((fz & 1) ? 2 : 1) : 1;
      const int px[2] = {fx >> 1, (fx + 1) >> 1}, py[2] = {fy >> 1, (fy + 1) >> 1}, pz[2] = {fz >> 1, (fz + 1) >> 1};
      const TC w = OC::weight((fx & 1) + (fy & 1) + (F.dim == 3 ? (fz & 1) : 0));
      TC acc = OC::zero();
      for (int c = 0; c < nz; ++c)
        for (int b = 0; b < ny; ++b)
          for (int aa = 0; aa < nx; ++aa) {
            const int ci = (F.dim == 3 ? pz[c] * Pc * Pc : 0) + py[b] * Pc + px[aa];
            acc = OC::xfer(w, ldcg(cc + ci), acc);
          }
      const TF t = OF::from(OC::wide(acc) * scale);
      uf[fi] = OF::fma(OF::from(1.0), t, ldcg(uf + fi));
    });
  }

  // sequential fma dot in lexicographic interior order (kernels.cpp:368-382)
  template <typename TA, typename TB>
  __device__ double dot_seq(const Pt& p, const TA* x, const TB* y) {
    double acc = 0.0;
    for (int k = 0; k < p.n; ++k) {
      const int i = p.idx(k);
      acc = __fma_rn((double)wide_v(ldcg(x + i)), (double)wide_v(ldcg(y + i)), acc);
    }
    return acc;
  }
  template <typename T>
  static __device__ __forceinline__ double wide_v(T v) {
    if constexpr (std::is_same<T, __half>::value) return (double)__half2float(v);
    else return (double)v;
  }

  // CG on level 0 (multigrid.cpp:91-151), CTA 0 only; a base level of <= 32
  // unknowns (every max-depth hierarchy) runs on warp 0 alone with warp
  // barriers and shuffles instead of CTA-wide barriers
  template <int PR>
  __device__ void cg(const CoarseLevel& L, const void* bv, void* uv) {
    if (pt(L).n == 1) cg_one<PR>(L, bv, uv);
    else if (pt(L).n <= 32) cg_impl<PR, true>(L, bv, uv);
    else cg_impl<PR, false>(L, bv, uv);
  }
  // cg_impl on a one-unknown base level (every max-depth hierarchy): the
  // identical operation sequence, every vector a register of thread 0, so an
  // iteration is a short dependent chain instead of barriers and shared
  // memory round trips (an FP16 base level runs all 10 iterations)
  template <int PR>
  __device__ void cg_one(const CoarseLevel& L, const void* bv, void* uv) {
    using OP = O<PR>;
    using T = typename OP::T;
    if (threadIdx.x != 0) return;
    const Pt pt = this->pt(L);
    const int i0 = pt.idx(0);
    const T b = ldcg(static_cast<const T*>(bv) + i0);
    T* uo = static_cast<T*>(uv) + i0;
    const double bw = wide_v(b);
    const double norm_b = sqrt(__fma_rn(bw, bw, 0.0));
    T u = OP::zero(), r = b, p = b, best = OP::zero();
    if (norm_b == 0.0) {
      *uo = u;
      return;
    }
    const int max_it = a.base_maxit > 0 ? a.base_maxit : 10;
    const double thr = a.base_mode == 0 ? a.base_tol * norm_b : a.base_tol;
    double rz = __fma_rn(wide_v(r), wide_v(r), 0.0);
    double true_res = norm_b, best_res = norm_b;
    int it = 0;
    const T m1 = OP::from(-1.0);
    const auto tk = taps_of<PR>(L);
    while (true_res >= thr && it < max_it) {
      const T ap = OP::apply1(tk, L.dim, p);
      const double pAp = __fma_rn(wide_v(p), wide_v(ap), 0.0);
      if (!(pAp > 0.0) || !isfinite(pAp)) break;
      const double alpha = rz / pAp;
      const T al = OP::from(alpha), mal = OP::from(-alpha);
      u = OP::fma(al, p, u);
      r = OP::fma(mal, ap, r);
      const double rz_new = __fma_rn(wide_v(r), wide_v(r), 0.0);
      ++it;
      const T sc = OP::fma(m1, OP::apply1(tk, L.dim, u), b);
      true_res = sqrt(__fma_rn(wide_v(sc), wide_v(sc), 0.0));
      if (true_res < best_res) {
        best_res = true_res;
        best = u;
      }
      if (rz == 0.0) break;
      const T be = OP::from(rz_new / rz);
      p = OP::fma(be, p, r);
      rz = rz_new;
    }
    *uo = true_res > best_res ? best : u;
    if (a.cg_iterations) *a.cg_iterations = it;
  }
  template <int PR, bool WARP>
  __device__ void cg_impl(const CoarseLevel& L, const void* bv, void* uv) {
    using OP = O<PR>;
    using T = typename OP::T;
    if (WARP && threadIdx.x >= 32) return;
    __shared__ double sh;
    const T* b = static_cast<const T*>(bv);
    T* u = static_cast<T*>(uv);
    T* r = static_cast<T*>(cgp[0]);
    T* p = static_cast<T*>(cgp[1]);
    T* ap = static_cast<T*>(cgp[2]);
    T* sc = static_cast<T*>(cgp[3]);
    T* best = static_cast<T*>(cgp[4]);
    const Pt pt = this->pt(L);
    auto dot = [&](const T* x, const T* y) -> double {
      if constexpr (WARP) {
        __syncwarp();
        double v = 0.0;
        if (threadIdx.x == 0) v = dot_seq(pt, x, y);
        return __shfl_sync(0xffffffffu, v, 0);
      } else {
        __syncthreads();
        if (threadIdx.x == 0) sh = dot_seq(pt, x, y);
        __syncthreads();
        const double v = sh;
        __syncthreads();
        return v;
      }
    };
    auto each = [&](auto&& f) {
      for (int k = threadIdx.x; k < pt.n; k += (WARP ? 32 : (int)blockDim.x)) f(pt.idx(k));
      if constexpr (WARP) __syncwarp();
      else __syncthreads();
    };
    const int max_it = a.base_maxit > 0 ? a.base_maxit : 10 * pt.n;
    each([&](int i) {
      u[i] = OP::zero();
      r[i] = ldcg(b + i);
      p[i] = ldcg(b + i);
      best[i] = OP::zero();
    });
    const double norm_b = sqrt(dot(b, b));
    if (norm_b == 0.0) return;
    const double thr = a.base_mode == 0 ? a.base_tol * norm_b : a.base_tol;
    double rz = dot(r, r);
    double true_res = norm_b, best_res = norm_b;
    int it = 0;
    const T m1 = OP::from(-1.0);
    const auto tk = taps_of<PR>(L);
    while (true_res >= thr && it < max_it) {
      each([&](int i) { ap[i] = OP::apply(tk, L.dim, p, i, pt.P); });
      const double pAp = dot(p, ap);
      if (!(pAp > 0.0) || !isfinite(pAp)) break;
      const double alpha = rz / pAp;
      const T al = OP::from(alpha), mal = OP::from(-alpha);
      each([&](int i) {
        u[i] = OP::fma(al, ldcg(p + i), ldcg(u + i));
        r[i] = OP::fma(mal, ldcg(ap + i), ldcg(r + i));
      });
      const double rz_new = dot(r, r);
      ++it;
      each([&](int i) { sc[i] = OP::apply(tk, L.dim, u, i, pt.P); });
      each([&](int i) { sc[i] = OP::fma(m1, ldcg(sc + i), ldcg(b + i)); });
      true_res = sqrt(dot(sc, sc));
      if (true_res < best_res) {
        best_res = true_res;
        each([&](int i) { best[i] = ldcg(u + i); });
      }
      if (rz == 0.0) break;
      const T be = OP::from(rz_new / rz);
      each([&](int i) { p[i] = OP::fma(be, ldcg(p + i), ldcg(r + i)); });
      rz = rz_new;
    }
    if (true_res > best_res) each([&](int i) { u[i] = ldcg(best + i); });
    if (threadIdx.x == 0 && a.cg_iterations) *a.cg_iterations = it;
  }

  __device__ void copy_level(const CoarseLevel& L, const void* src, void* dst) {
    for_points(L, [&](int i, int) {
      if (L.prec == MPMG_FP16) static_cast<uint16_t*>(dst)[i] = static_cast<const uint16_t*>(src)[i];
      else if (L.prec == MPMG_FP32) static_cast<uint32_t*>(dst)[i] = static_cast<const uint32_t*>(src)[i];
      else static_cast<uint64_t*>(dst)[i] = static_cast<const uint64_t*>(src)[i];
    });
  }

  // barrier after an operation on level L that wrote buffer x (slab mode:
  // halo exchange + cluster barrier for a slab level)
  __device__ void after(const CoarseLevel& L, void* x) {
    if (slab && !small(L)) {
      if (a.debug > 1) { __syncthreads(); stamp(7, (int)(&L - lv)); }
      exchange((int)(&L - lv), x);
      if (a.debug > 1) stamp(8, (int)(&L - lv));
    } else {
      sync(L);
      if (a.debug > 1) stamp(7, (int)(&L - lv));
    }
  }

  // ping-pong smoothing between L.u and L.u2; returns the result buffer
  __device__ void* smooth(const CoarseLevel& L, void* cur, int steps) {
    for (int s = 0; s < steps; ++s) {
      void* out = (cur == L.u) ? L.u2 : L.u;
      const bool z = cur == nullptr;
      if (in_team(L)) by_prec(L.prec, [&](auto pc) { jacobi<decltype(pc)::value>(L, L.b, z ? L.b : cur, out, z); });
      after(L, out);
      cur = out;
    }
    return cur;
  }

  // Every CTA walks the same schedule; an op on a small level is worked by
  // CTA 0 only and followed by __syncthreads, an op on a big level by the
  // whole grid and followed by a grid barrier. The one extra grid
  // barrier before prolongating a small level's correction into a big level
  // publishes CTA 0's small-level results.
  int entry = -1;  // highest level worked by CTA 0 alone (its b arrives in global memory)

  // global b of the entry level -> CTA 0's shared copy
  __device__ void stage_in(int l) {
    if (rank == 0) copy_level(lv[l], a.lv[l].b, lv[l].b);
    __syncthreads();
  }
  __device__ void stage_out(int l, const void* src) {
    if (rank == 0) copy_level(lv[l], src, a.lv[l].u);
    __syncthreads();
  }

  // slab mode schedule (3D, one precision, no DSH rescaling, level 0 a CTA-0 level)
  __device__ void run_slab() {
    void* cur[kMaxCoarseLevels];
    const int top = a.nlev - 1;
    if (t0 == 0) t0 = clock64();
    stamp(10, 0);    // (debug: t0 = kernel entry, so this is the set-up time)
    cluster_sync();  // every CTA's shared memory is laid out and zeroed
    copy_level(lv[top], a.lv[top].b, lv[top].b);  // own planes of the top rhs
    __syncthreads();
    for (int l = top; l >= 1; --l) {
      const CoarseLevel& L = lv[l];
      const CoarseLevel& C = lv[l - 1];
      stamp(1, l);
      void* u = smooth(L, nullptr, a.pre);
      if (u == nullptr) {  // pre_steps == 0: u = 0
        if (in_team(L)) for_points(L, [&](int i, int) {
          if (L.prec == MPMG_FP16) static_cast<uint16_t*>(L.u)[i] = 0;
          else if (L.prec == MPMG_FP32) static_cast<float*>(L.u)[i] = 0.f;
          else static_cast<double*>(L.u)[i] = 0.0;
        });
        after(L, L.u);
        u = L.u;
      }
      cur[l] = u;
      stamp(4, l);
      if (in_team(L)) by_prec(L.prec, [&](auto pc) { defect<decltype(pc)::value>(L, L.b, u, L.r); });
      after(L, L.r);
      stamp(5, l);
      if (in_team(L)) by_prec(L.prec, [&](auto pc) { restrict_to<decltype(pc)::value>(L, C, L.r, false); });
      if (small(L)) __syncthreads();
      else cluster_sync();  // coarse rhs complete (a CTA-0 level's in CTA 0)
    }
    if (rank == 0) by_prec(lv[0].prec, [&](auto pc) { cg<decltype(pc)::value>(lv[0], lv[0].b, lv[0].u); });
    __syncthreads();
    cur[0] = lv[0].u;
    stamp(2, 0);
    for (int l = 1; l <= top; ++l) {
      const CoarseLevel& L = lv[l];
      const CoarseLevel& C = lv[l - 1];
      if (!small(L) && small(C)) cluster_sync();  // CTA 0's correction visible cluster-wide
      if (in_team(L)) {
        by_prec(L.prec, [&](auto fp) {
          by_prec(C.prec, [&](auto cp) {
            prolong<decltype(fp)::value, decltype(cp)::value>(L, C, cur[l - 1], cur[l], 1.0);
          });
        });
      }
      after(L, cur[l]);
      stamp(6, l);
      cur[l] = smooth(L, cur[l], a.post);
      stamp(3, l);
    }
    copy_level(lv[top], cur[top], a.lv[top].u);  // own planes of the top correction
    stamp(12, top);
    stamps_done();
  }

  __device__ void run() {
    __shared__ double scales[kMaxCoarseLevels];
    void* cur[kMaxCoarseLevels];
    const int top = a.nlev - 1;
    t0 = clock64();
    for (int l = top; l >= 0; --l)
      if (small(lv[l])) { entry = l; break; }
    // down-sweep (cycle_at before the recursive call)
    for (int l = top; l >= 1; --l) {
      const CoarseLevel& L = lv[l];
      const CoarseLevel& C = lv[l - 1];
      stamp(1, l);
      if (small(L) && l == entry) stage_in(l);
      void* u = smooth(L, nullptr, a.pre);
      if (u == nullptr) {  // pre_steps == 0: u = 0
        if (in_team(L)) for_points(L, [&](int i, int) {
          if (L.prec == MPMG_FP16) static_cast<uint16_t*>(L.u)[i] = 0;
          else if (L.prec == MPMG_FP32) static_cast<float*>(L.u)[i] = 0.f;
          else static_cast<double*>(L.u)[i] = 0.0;
        });
        sync(L);
        u = L.u;
      }
      cur[l] = u;
      stamp(4, l);
      if (in_team(L)) by_prec(L.prec, [&](auto pc) { defect<decltype(pc)::value>(L, L.b, u, L.r); });
      sync(L);
      stamp(5, l);
      const bool rescale = a.rescale && C.prec == MPMG_FP16;  // multigrid.cpp:383
      if (in_team(L)) by_prec(L.prec, [&](auto pc) { restrict_to<decltype(pc)::value>(L, C, L.r, rescale); });
      sync(L);
      if (threadIdx.x == 0) {
        double sc = 1.0;
        if (rescale && in_team(L)) {  // multigrid.cpp:246-250, sequential fma order
          const Pt pc = pt(C);
          double acc = 0.0;
          for (int k = 0; k < pc.n; ++k) {
            const double v = C.prod[pc.idx(k)];
            acc = __fma_rn(v, v, acc);
          }
          const double nrm = sqrt(acc);
          if (nrm > 0.0 && isfinite(nrm)) sc = nrm;
        }
        scales[l - 1] = sc;
      }
      __syncthreads();
      if (rescale) {
        if (in_team(L)) by_prec(C.prec, [&](auto cp) { restrict_store<decltype(cp)::value>(C, scales[l - 1]); });
        sync(L);
      }
    }
    // base solve on CTA 0
    if (top == 0 && entry == 0) {
      // single-level call (OP_COARSE_SOLVE): result to global
      stage_in(0);
      if (rank == 0) by_prec(lv[0].prec, [&](auto pc) { cg<decltype(pc)::value>(lv[0], lv[0].b, lv[0].u); });
      __syncthreads();
      if (rank == 0) copy_level(lv[0], lv[0].u, a.lv[0].u);
      __syncthreads();
      return;
    }
    {
      const CoarseLevel& B = lv[0];
      if (entry == 0) stage_in(0);
      if (rank == 0) by_prec(B.prec, [&](auto pc) { cg<decltype(pc)::value>(B, B.b, B.u); });
      __syncthreads();
      if (!small(B)) gsync();
      cur[0] = B.u;
      stamp(2, 0);
    }
    // up-sweep
    for (int l = 1; l <= top; ++l) {
      const CoarseLevel& L = lv[l];
      const CoarseLevel& C = lv[l - 1];
      if (!small(L) && small(C)) {
        stage_out(l - 1, cur[l - 1]);  // CTA 0's shared-memory correction -> global
        cur[l - 1] = a.lv[l - 1].u;
        gsync();
      }
      if (in_team(L)) {
        by_prec(L.prec, [&](auto fp) {
          by_prec(C.prec, [&](auto cp) {
            prolong<decltype(fp)::value, decltype(cp)::value>(L, C, cur[l - 1], cur[l], scales[l - 1]);
          });
        });
      }
      sync(L);
      stamp(6, l);
      void* u = smooth(L, cur[l], a.post);
      if (l == top && u != a.lv[top].u) {  // the caller reads the top correction from global L.u
        if (in_team(L)) copy_level(L, u, a.lv[top].u);
        sync(L);
        u = a.lv[top].u;
      }
      cur[l] = u;
      stamp(3, l);
    }
    stamps_done();
  }
};

__host__ __device__ inline long long padded_of(const CoarseLevel& L) {
  const long long P = L.nodes - 1;
  return L.dim == 3 ? P * P * P + P * P + P + 1 : P * P + P + 1;
}
__host__ __device__ inline int bytes_of(int prec) { return prec == MPMG_FP16 ? 2 : (prec == MPMG_FP32 ? 4 : 8); }
__host__ __device__ inline bool small_level(const CoarseLevel& L, int cta_points) {
  const long long m = L.nodes - 2;
  return (L.dim == 3 ? m * m * m : m * m) <= cta_points;
}

// shared bytes for CTA 0's small levels (u, u2, b, r each, 16-byte aligned)
// plus the CG scratch of level 0
__host__ __device__ inline size_t coarse_smem(const CoarseArgs& a) {
  size_t n = 0;
  for (int l = 0; l < a.nlev; ++l)
    if (small_level(a.lv[l], a.cta_points)) n += 4 * ((padded_of(a.lv[l]) * bytes_of(a.lv[l].prec) + 15) / 16 * 16);
  if (small_level(a.lv[0], a.cta_points)) n += 5 * ((padded_of(a.lv[0]) * bytes_of(a.lv[0].prec) + 15) / 16 * 16);
  return n;
}

// slab mode shared-memory layout (identical in every CTA of the cluster):
// per level, CTA-0 levels as full padded vectors and slab levels as C-way
// z-slabs, 4 buffers each (u, u2, b, r), then the CG scratch of level 0.
// off[l] = byte offset of level l's buffers, sz[l] = bytes per buffer.
__host__ __device__ inline size_t slab_smem(const CoarseArgs& a, int C, size_t* off, size_t* sz) {
  size_t n = 0;
  const int T = a.nlev - 1;
  for (int l = 0; l < a.nlev; ++l) {
    const CoarseLevel& L = a.lv[l];
    const long long P = L.nodes - 1;
    long long elems = padded_of(L);
    if (!small_level(L, a.cta_points)) elems = slab_elems((int)P, slab_max_nz((int)(a.lv[T].nodes - 1), C, T - l));
    const size_t b = ((size_t)elems * bytes_of(L.prec) + 15) / 16 * 16;
    if (off) off[l] = n;
    if (sz) sz[l] = b;
    n += 4 * b;
  }
  if (off) off[a.nlev] = n;
  n += 5 * ((padded_of(a.lv[0]) * bytes_of(a.lv[0].prec) + 15) / 16 * 16);
  return n;
}

template <bool FTZ, bool FMA, bool ACC32, int UP>
__global__ void __launch_bounds__(kThreads) k_coarse(const __grid_constant__ CoarseArgs a, int use_smem, int cluster) {
  const long long t_entry = a.dbg ? clock64() : 0;
  __shared__ CoarseLevel table[kMaxCoarseLevels];
  __shared__ __half t16[kMaxCoarseLevels][27];
  __shared__ float t32[kMaxCoarseLevels][27];
  for (int i = threadIdx.x; i < a.nlev * 27; i += blockDim.x) {
    const double v = a.lv[i / 27].taps[i % 27];
    t16[i / 27][i % 27] = round16<FTZ>(v);
    t32[i / 27][i % 27] = round32<FTZ>(v);
  }
  __shared__ void* cg[5];
  __shared__ Pt s_pt[kMaxCoarseLevels];
  __shared__ unsigned char s_small[kMaxCoarseLevels];
  if (threadIdx.x < a.nlev) {
    s_pt[threadIdx.x] = points(a.lv[threadIdx.x]);
    s_small[threadIdx.x] = small_level(a.lv[threadIdx.x], a.cta_points) ? 1 : 0;
  }
  extern __shared__ __align__(16) unsigned char dyn[];
  // level table: a parallel word copy of the launch parameters (a serial
  // struct copy by one thread cost microseconds); pointers patched below
  static_assert(sizeof(CoarseLevel) % 8 == 0, "");
  for (int i = threadIdx.x; i < a.nlev * (int)(sizeof(CoarseLevel) / 8); i += blockDim.x)
    reinterpret_cast<unsigned long long*>(table)[i] = reinterpret_cast<const unsigned long long*>(a.lv)[i];
  __shared__ short slo_tab[kMaxCoarseLevels][17];
  __shared__ PushTab push_tab[kMaxCoarseLevels];
  if (cluster)  // slab mode: plane ownership of every level and CTA
    for (int i = threadIdx.x; i < a.nlev * 17; i += blockDim.x) {
      const int T = a.nlev - 1, l = i / 17, r = i % 17;
      slo_tab[l][r] = (short)(r <= (int)gridDim.x ? slab_lo((int)(a.lv[T].nodes - 1), (int)gridDim.x, T - l, r) : 0);
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    cg[0] = a.cg_r; cg[1] = a.cg_p; cg[2] = a.cg_ap; cg[3] = a.cg_s; cg[4] = a.cg_best;
    if (use_smem && blockIdx.x == 0 && !cluster) {
      unsigned char* p = dyn;
      for (int l = 0; l < a.nlev; ++l) {
        if (!small_level(a.lv[l], a.cta_points)) continue;
        const size_t b = (padded_of(a.lv[l]) * bytes_of(a.lv[l].prec) + 15) / 16 * 16;
        table[l].u = p; p += b;
        table[l].u2 = p; p += b;
        table[l].b = p; p += b;
        table[l].r = p; p += b;
      }
      if (small_level(a.lv[0], a.cta_points)) {
        const size_t b = (padded_of(a.lv[0]) * bytes_of(a.lv[0].prec) + 15) / 16 * 16;
        for (int k = 0; k < 5; ++k) { cg[k] = p; p += b; }
      }
    }
  }
  if (cluster) {  // slab mode: every CTA lays out its slabs (and CTA 0's levels)
    // (one set-up phase: level buffers by thread l, push tables by thread 32 + l,
    // zero fill by everyone -- the launcher computed the layout)
    if (threadIdx.x < a.nlev) {
      const int l = threadIdx.x;
      unsigned char* q[4];
      for (int k = 0; k < 4; ++k) q[k] = dyn + a.slab_off[l] + k * a.slab_sz[l];
      if (small_level(a.lv[l], a.cta_points)) {  // CTA 0's full vectors, reached through DSMEM
        // (CTA 0 itself keeps the plain shared-memory addresses: its small-level
        // operations are latency chains, and a cluster-window access is slower)
        if (blockIdx.x != 0) {
          cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
          for (int k = 0; k < 4; ++k) q[k] = static_cast<unsigned char*>(cl.map_shared_rank((void*)q[k], 0));
        }
      } else {  // virtual base: global plane z of the slab at base + z * plane bytes
        const long long P = a.lv[l].nodes - 1;
        const long long shift = (long long)(slo_tab[l][blockIdx.x] - 1) * P * P * bytes_of(a.lv[l].prec);
        for (int k = 0; k < 4; ++k) q[k] -= shift;
      }
      table[l].u = q[0]; table[l].u2 = q[1]; table[l].b = q[2]; table[l].r = q[3];
      if (l == 0) {
        const size_t b0 = (padded_of(a.lv[0]) * bytes_of(a.lv[0].prec) + 15) / 16 * 16;
        for (int k = 0; k < 5; ++k) cg[k] = dyn + a.slab_off[a.nlev] + k * b0;
      }
    } else if (threadIdx.x >= 32 && threadIdx.x < 32 + a.nlev) {  // push tables
      const int l = threadIdx.x - 32, C = (int)gridDim.x, r = blockIdx.x;
      PushTab& pt = push_tab[l];
      int n = 0;
      const int zlo = slo_tab[l][r], zhi = slo_tab[l][r + 1];
      if (!small_level(a.lv[l], a.cta_points))
        for (int t = 0; t < C; ++t) {
          if (t == r) continue;
          const int tlo = slo_tab[l][t], thi = slo_tab[l][t + 1];
          for (int side = 0; side < 2; ++side) {
            const int z = side == 0 ? tlo - 1 : thi;
            if (z < zlo || z >= zhi || n >= 8) continue;
            pt.t[n] = (signed char)t;
            pt.src[n] = (signed char)(z - (zlo - 1));
            pt.dst[n] = (signed char)(z - (tlo - 1));
            ++n;
          }
        }
      pt.n = n;
    }
    const size_t n = a.slab_total / 16;
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) reinterpret_cast<uint4*>(dyn)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    Coarse<FTZ, FMA, ACC32, UP> c(a, table, cg, t16, t32, true);
    c.spt = s_pt;
    c.ssmall = s_small;
    c.slo = slo_tab;
    c.push = push_tab;
    c.t0 = t_entry;
    c.run_slab();
    return;
  }
  if (use_smem && blockIdx.x == 0) {  // ghosts must read as zero
    const size_t n = coarse_smem(a) / 16;
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) reinterpret_cast<uint4*>(dyn)[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  Coarse<FTZ, FMA, ACC32, UP> c(a, table, cg, t16, t32, false);
  c.spt = s_pt;
  c.ssmall = s_small;
  c.run();
}

template <bool FTZ, bool FMA, bool ACC32, int UP>
cudaError_t launch_u(const CoarseArgs& a, cudaStream_t s) {
  auto kern = k_coarse<FTZ, FMA, ACC32, UP>;
  const CoarseLevel& T = a.lv[a.nlev - 1];
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  // (no programmatic dependent launch: measured, an early-resident 16-CTA
  // cluster slows the FP64 cascade's predecessors by ~60 us per V-cycle)
  cudaLaunchAttribute at[1];
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static size_t attr_set = 0;
  auto want_smem = [&](size_t bytes) {
    if (bytes > attr_set) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      attr_set = bytes;
    }
  };
  // slab mode: one cluster (16, else 8 CTAs) when every level is 3D, without
  // DSH rescaling (its restriction norm spans the cluster), and the base level
  // is a CTA-0 level; mixed cascades (HSD) too unless MPMG_COARSE_MIXED_SLAB=0
  static int cl_env = -1, mixed_env = -1;
  if (cl_env < 0) {
    const char* e = std::getenv("MPMG_COARSE_CLUSTER");
    cl_env = e ? std::atoi(e) : 16;
    const char* m = std::getenv("MPMG_COARSE_MIXED_SLAB");
    mixed_env = m ? std::atoi(m) : 1;
  }
  bool slab_ok = cl_env > 1 && (UP < 3 || mixed_env != 0) && !a.rescale && !small_level(T, a.cta_points) &&
                 small_level(a.lv[0], a.cta_points);
  for (int l = 0; l < a.nlev && slab_ok; ++l) slab_ok = a.lv[l].dim == 3 && a.lv[l].nodes - 1 >= 2;
  if (slab_ok) {
    static int tried = 0, ok16 = 0, ok8 = 0;
    if (!tried) {
      tried = 1;
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    for (int c = std::min(cl_env, 16); c >= 8; c /= 2) {
      const size_t smem = slab_smem(a, c, nullptr, nullptr);
      if (smem > 212 * 1024) continue;  // + ~10 KB of static tables <= 227 KB per CTA
      int& ok = c == 16 ? ok16 : ok8;
      want_smem(smem);
      if (ok == 0) {  // can a cluster of c CTAs with this footprint be resident?
        cudaLaunchConfig_t q = cfg;
        q.gridDim = dim3(c);
        q.dynamicSmemBytes = smem;
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = c;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        q.attrs = qa;
        int nc = 0;
        ok = (cudaOccupancyMaxActiveClusters(&nc, kern, &q) == cudaSuccess && nc > 0) ? 1 : -1;
        cudaGetLastError();
      }
      if (ok < 0) continue;
      cfg.gridDim = dim3(c);
      cfg.dynamicSmemBytes = smem;
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      CoarseArgs ac = a;
      size_t off[kMaxCoarseLevels + 1], sz[kMaxCoarseLevels];
      ac.slab_total = slab_smem(a, c, off, sz);
      for (int l = 0; l <= a.nlev; ++l) ac.slab_off[l] = off[l];
      for (int l = 0; l < a.nlev; ++l) ac.slab_sz[l] = sz[l];
      return cudaLaunchKernelEx(&cfg, kern, ac, 1, c);
    }
  }
  const size_t smem = coarse_smem(a);
  const int use_smem = smem <= 200 * 1024 ? 1 : 0;
  const size_t dyn = use_smem ? smem : 0;
  if (use_smem) want_smem(smem);
  // grid: one CTA when every level is a CTA-0 level, else every co-resident
  // CTA as a cooperative grid
  unsigned grid = 1;
  if (!small_level(T, a.cta_points)) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kThreads, dyn);
    static int per_env = -1;  // MPMG_COARSE_PER_SM: CTAs per SM (<= occupancy)
    if (per_env < 0) {
      const char* e = std::getenv("MPMG_COARSE_PER_SM");
      per_env = e ? std::atoi(e) : 0;
    }
    if (per_env > 0) per = std::min(per, per_env);
    grid = (unsigned)std::max(1, per) * (unsigned)std::max(1, sms);
  }
  cfg.gridDim = dim3(grid);
  cfg.dynamicSmemBytes = dyn;
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, use_smem, 0);
}

template <bool FTZ, bool FMA, bool ACC32>
cudaError_t launch_t(const CoarseArgs& a, cudaStream_t s) {
  bool uni = true;
  for (int l = 1; l < a.nlev; ++l) uni = uni && a.lv[l].prec == a.lv[0].prec;
  if (!uni) return launch_u<FTZ, FMA, ACC32, 3>(a, s);
  switch (a.lv[0].prec) {
    case MPMG_FP16: return launch_u<FTZ, FMA, ACC32, P16>(a, s);
    case MPMG_FP32: return launch_u<FTZ, FMA, ACC32, P32>(a, s);
    default: return launch_u<FTZ, FMA, ACC32, P64>(a, s);
  }
}

}  // namespace coarse_detail

// one translation unit per policy (mpmg_coarse_f<ftz>m<fma>a<acc32>.cu)
#define MPMG_COARSE_DECL(F, M, A) cudaError_t launch_coarse_f##F##m##M##a##A(const CoarseArgs& a, cudaStream_t s);
MPMG_COARSE_DECL(0, 0, 0) MPMG_COARSE_DECL(0, 0, 1) MPMG_COARSE_DECL(0, 1, 0) MPMG_COARSE_DECL(0, 1, 1)
MPMG_COARSE_DECL(1, 0, 0) MPMG_COARSE_DECL(1, 0, 1) MPMG_COARSE_DECL(1, 1, 0) MPMG_COARSE_DECL(1, 1, 1)
#undef MPMG_COARSE_DECL

}  // namespace mpmg_impl
