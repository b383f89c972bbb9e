// Coarse sub-hierarchy in ONE thread block: every level too small for the
// streaming kernels (pitch below the warp footprint) runs inside a single
// persistent CTA — pre-smoothing, defect, restriction (with the DSH rescale),
// the CG base solve on level 0, prolongation + correction and post-smoothing
// — separated by __syncthreads instead of kernel launches. This replaces the
// coarse part of the reference's recursion (cycle_at, multigrid.cpp:362-393)
// and cg_solve (multigrid.cpp:91-151).
//
// Arithmetic is the same per-operation rounding as the streaming kernels.
// Reductions that the reference accumulates sequentially (dot_fp64 /
// norm2_fp64, kernels.cpp:368-395; the DSH restriction norm,
// multigrid.cpp:246-250) are done by one thread in the reference's
// lexicographic order when the level has <= kSeqDot unknowns, so the base
// solve is bitwise identical to the reference there.
#include <type_traits>

#include "mpmg_arith.cuh"
#include "mpmg_internal.h"

namespace mpmg_impl {

using namespace mpmg_dev;

namespace {

constexpr int kCoarseThreads = 512;
constexpr long long kSeqDot = 32768;

template <int PR> struct T_;
template <> struct T_<P16> { using T = __half; };
template <> struct T_<P32> { using T = float; };
template <> struct T_<P64> { using T = double; };

// Policy is a runtime value here: the coarse kernel is latency-bound, and a
// single instantiation keeps the build fast.
struct Pol {
  bool ftz, fma, acc32;
};

__device__ __forceinline__ __half rfma16(Pol p, __half a, __half b, __half c) {
  __half r;
  if (p.fma) r = __hfma(a, b, c);
  else {
    __half m = __hmul_rn(a, b);
    if (p.ftz) m = flush16s(m);
    r = __hadd_rn(m, c);
  }
  return p.ftz ? flush16s(r) : r;
}
__device__ __forceinline__ float rfma32(Pol p, float a, float b, float c) {
  float r;
  if (p.fma) r = __fmaf_rn(a, b, c);
  else {
    float m = __fmul_rn(a, b);
    if (p.ftz) m = flush32(m);
    r = __fadd_rn(m, c);
  }
  return p.ftz ? flush32(r) : r;
}

template <int PR>
struct Lv {
  using T = typename T_<PR>::T;
  static __device__ __forceinline__ T from(Pol p, double v) {
    if constexpr (PR == P16) return p.ftz ? round16<true>(v) : round16<false>(v);
    else if constexpr (PR == P32) return p.ftz ? round32<true>(v) : round32<false>(v);
    else return v;
  }
  static __device__ __forceinline__ double wide(T v) {
    if constexpr (PR == P16) return (double)__half2float(v);
    else return (double)v;
  }
  static __device__ __forceinline__ T zero() { return T(0); }
  static __device__ __forceinline__ T fma(Pol p, T a, T b, T c) {
    if constexpr (PR == P16) return rfma16(p, a, b, c);
    else if constexpr (PR == P32) return rfma32(p, a, b, c);
    else return p.fma ? __fma_rn(a, b, c) : __dadd_rn(__dmul_rn(a, b), c);
  }
  static __device__ __forceinline__ T mul(Pol p, T a, T b) {
    if constexpr (PR == P16) { const __half m = __hmul_rn(a, b); return p.ftz ? flush16s(m) : m; }
    else if constexpr (PR == P32) { const float m = __fmul_rn(a, b); return p.ftz ? flush32(m) : m; }
    else return __dmul_rn(a, b);
  }
  // transfer_product step (multigrid.cpp:166-195): FP32 unfused flushes only the sum
  static __device__ __forceinline__ T xfer(Pol p, double w, T x, T acc) {
    if constexpr (PR == P32) {
      const float r = p.fma ? __fmaf_rn((float)w, x, acc) : __fadd_rn(__fmul_rn((float)w, x), acc);
      return p.ftz ? flush32(r) : r;
    } else return fma(p, from(p, w), x, acc);
  }
  // A x at padded index i (all 3^dim taps; ghosts are zero)
  static __device__ __forceinline__ T apply(Pol p, const CoarseLevel& L, const T* x, long long i, int P) {
    const long long pl = L.dim == 3 ? (long long)P * P : 0;
    if constexpr (PR == P16) {
      if (p.acc32) {  // Fp16Accum::FP32 (kernels.cpp:151-162)
        float acc = 0.0f;
        int t = 0;
        for (int dz = (L.dim == 3 ? -1 : 0); dz <= (L.dim == 3 ? 1 : 0); ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx, ++t)
              acc = rfma32(p, (float)L.taps[t], __half2float(x[i + dz * pl + (long long)dy * P + dx]), acc);
        const __half h = __float2half_rn(acc);
        return p.ftz ? flush16s(h) : h;
      }
    }
    T acc = zero();
    int t = 0;
    for (int dz = (L.dim == 3 ? -1 : 0); dz <= (L.dim == 3 ? 1 : 0); ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx, ++t)
          acc = fma(p, from(p, L.taps[t]), x[i + dz * pl + (long long)dy * P + dx], acc);
    return acc;
  }
};

struct Pt {
  long long n;  // interior points
  int P, dim;
  __device__ __forceinline__ long long idx(long long k) const {
    const long long m = P - 1;
    const long long x = k % m + 1;
    if (dim == 2) return (k / m + 1) * P + x;
    return ((k / (m * m) + 1) * P + (k / m) % m + 1) * (long long)P + x;
  }
};

__device__ __forceinline__ Pt points(const CoarseLevel& L) {
  Pt p;
  p.P = L.nodes - 1;
  p.dim = L.dim;
  const long long m = p.P - 1;
  p.n = L.dim == 3 ? m * m * m : m * m;
  return p;
}

// sequential fma dot in lexicographic interior order (kernels.cpp:368-382)
template <typename TA, typename TB, typename W1, typename W2>
__device__ double dot_seq(const Pt& p, const TA* x, const TB* y, W1 wx, W2 wy) {
  double acc = 0.0;
  for (long long k = 0; k < p.n; ++k) {
    const long long i = p.idx(k);
    acc = __fma_rn(wx(x[i]), wy(y[i]), acc);
  }
  return acc;
}

struct Coarse {
  const CoarseArgs& a;
  Pol pol;
  __device__ Coarse(const CoarseArgs& args, Pol p) : a(args), pol(p) {}

  template <typename F>
  __device__ void for_points(const CoarseLevel& L, F&& f) {
    const Pt p = points(L);
    for (long long k = threadIdx.x; k < p.n; k += blockDim.x) f(p.idx(k), p.P);
  }

  template <int PR>
  __device__ void jacobi(const CoarseLevel& L, const void* bv, const void* uin, void* uout, bool from_zero) {
    using O = Lv<PR>;
    using T = typename O::T;
    const T* b = static_cast<const T*>(bv);
    const T* u = static_cast<const T*>(uin);
    T* o = static_cast<T*>(uout);
    const T w = O::from(pol, L.omega), d = O::from(pol, L.inv_diag), m1 = O::from(pol, -1.0);
    for_points(L, [&](long long i, int P) {
      const T t = from_zero ? O::zero() : O::apply(pol, L, u, i, P);
      const T r = O::fma(pol, m1, t, b[i]);
      o[i] = O::fma(pol, w, O::mul(pol, d, r), from_zero ? O::zero() : u[i]);
    });
  }

  template <int PR>
  __device__ void defect(const CoarseLevel& L, const void* bv, const void* uv, void* rv) {
    using O = Lv<PR>;
    using T = typename O::T;
    const T m1 = O::from(pol, -1.0);
    for_points(L, [&](long long i, int P) {
      static_cast<T*>(rv)[i] = O::fma(pol, m1, O::apply(pol, L, static_cast<const T*>(uv), i, P), static_cast<const T*>(bv)[i]);
    });
  }

  // R r_f into C.prod (binary64 value domain of the fine-precision product)
  template <int FP>
  __device__ void restrict_prod(const CoarseLevel& F, const CoarseLevel& C, const void* rfv) {
    using O = Lv<FP>;
    using T = typename O::T;
    const T* rf = static_cast<const T*>(rfv);
    const int Pf = F.nodes - 1;
    const long long pf = F.dim == 3 ? (long long)Pf * Pf : 0;
    for_points(C, [&](long long ci, int Pc) {
      const long long m = Pc;
      const long long cx = ci % m, cy = (ci / m) % m, cz = F.dim == 3 ? ci / (m * m) : 0;
      const long long cf = cz * 2 * pf + cy * 2 * Pf + cx * 2;
      T acc = O::zero();
      for (int dz = (F.dim == 3 ? -1 : 0); dz <= (F.dim == 3 ? 1 : 0); ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const double w = (dx == 0 ? 1.0 : 0.5) * (dy == 0 ? 1.0 : 0.5) * (dz == 0 ? 1.0 : 0.5);
            const T x = rf[cf + dz * pf + (long long)dy * Pf + dx];
            acc = O::xfer(pol, w, x, acc);
          }
      C.prod[ci] = O::wide(acc);
    });
  }

  template <int CPc>
  __device__ void restrict_store(const CoarseLevel& C, double scale) {
    using O = Lv<CPc>;
    using T = typename O::T;
    for_points(C, [&](long long ci, int) { static_cast<T*>(C.b)[ci] = O::from(pol, C.prod[ci] / scale); });
  }

  // u_f += round_f(scale * P c) (prod in coarse precision)
  template <int FP, int CPc>
  __device__ void prolong(const CoarseLevel& F, const CoarseLevel& C, const void* ccv, void* ufv, double scale) {
    using OC = Lv<CPc>;
    using OF = Lv<FP>;
    using TC = typename OC::T;
    using TF = typename OF::T;
    const TC* cc = static_cast<const TC*>(ccv);
    TF* uf = static_cast<TF*>(ufv);
    const int Pc = C.nodes - 1;
    for_points(F, [&](long long fi, int Pf) {
      const long long m = Pf;
      const int fx = (int)(fi % m), fy = (int)((fi / m) % m), fz = F.dim == 3 ? (int)(fi / (m * m)) : 0;
      const int nx = (fx & 1) ? 2 : 1, ny = (fy & 1) ? 2 : 1, nz = F.dim == 3 ? ((fz & 1) ? 2 : 1) : 1;
      const int px[2] = {fx >> 1, (fx + 1) >> 1}, py[2] = {fy >> 1, (fy + 1) >> 1}, pz[2] = {fz >> 1, (fz + 1) >> 1};
      const double w = ((fx & 1) ? 0.5 : 1.0) * ((fy & 1) ? 0.5 : 1.0) * (F.dim == 3 && (fz & 1) ? 0.5 : 1.0);
      TC acc = OC::zero();
      for (int c = 0; c < nz; ++c)
        for (int b = 0; b < ny; ++b)
          for (int aa = 0; aa < nx; ++aa) {
            const long long ci = (F.dim == 3 ? (long long)pz[c] * Pc * Pc : 0) + (long long)py[b] * Pc + px[aa];
            acc = OC::xfer(pol, w, cc[ci], acc);
          }
      const TF t = OF::from(pol, OC::wide(acc) * scale);
      uf[fi] = OF::fma(pol, OF::from(pol, 1.0), t, uf[fi]);
    });
  }

  // CG on level 0 (multigrid.cpp:91-151)
  template <int PR>
  __device__ void cg(const CoarseLevel& L, const void* bv, void* uv) {
    using O = Lv<PR>;
    using T = typename O::T;
    __shared__ double sh[4];
    __shared__ double red[kCoarseThreads];
    const T* b = static_cast<const T*>(bv);
    T* u = static_cast<T*>(uv);
    T* r = static_cast<T*>(a.cg_r);
    T* p = static_cast<T*>(a.cg_p);
    T* ap = static_cast<T*>(a.cg_ap);
    T* sc = static_cast<T*>(a.cg_s);
    T* best = static_cast<T*>(a.cg_best);
    const Pt pt = points(L);
    const auto wd = [](T v) { return O::wide(v); };
    auto dot = [&](const T* x, const T* y) -> double {
      // returns the value on thread 0 only; caller broadcasts
      if (pt.n <= kSeqDot) {
        if (threadIdx.x == 0) sh[3] = dot_seq(pt, x, y, wd, wd);
      } else {
        double acc = 0.0;
        for (long long k = threadIdx.x; k < pt.n; k += blockDim.x) {
          const long long i = pt.idx(k);
          acc = __fma_rn(O::wide(x[i]), O::wide(y[i]), acc);
        }
        red[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
          double s = 0.0;
          for (int t = 0; t < (int)blockDim.x; ++t) s += red[t];
          sh[3] = s;
        }
      }
      __syncthreads();
      const double v = sh[3];
      __syncthreads();
      return v;
    };
    const int max_it = a.base_maxit > 0 ? a.base_maxit : 10 * (int)pt.n;
    for_points(L, [&](long long i, int) {
      u[i] = O::zero();
      r[i] = b[i];
      p[i] = b[i];
      best[i] = O::zero();
    });
    __syncthreads();
    const double norm_b = sqrt(dot(b, b));
    if (norm_b == 0.0) return;
    const double thr = a.base_mode == 0 ? a.base_tol * norm_b : a.base_tol;
    double rz = dot(r, r);
    double true_res = norm_b, best_res = norm_b;
    int it = 0;
    while (true_res >= thr && it < max_it) {
      for_points(L, [&](long long i, int P) { ap[i] = O::apply(pol, L, p, i, P); });
      __syncthreads();
      const double pAp = dot(p, ap);
      if (!(pAp > 0.0) || !isfinite(pAp)) break;
      const double alpha = rz / pAp;
      const T al = O::from(pol, alpha), mal = O::from(pol, -alpha);
      for_points(L, [&](long long i, int) {
        u[i] = O::fma(pol, al, p[i], u[i]);
        r[i] = O::fma(pol, mal, ap[i], r[i]);
      });
      __syncthreads();
      const double rz_new = dot(r, r);
      ++it;
      for_points(L, [&](long long i, int P) { sc[i] = O::apply(pol, L, u, i, P); });
      __syncthreads();
      const T m1 = O::from(pol, -1.0);
      for_points(L, [&](long long i, int) { sc[i] = O::fma(pol, m1, sc[i], b[i]); });
      __syncthreads();
      true_res = sqrt(dot(sc, sc));
      if (true_res < best_res) {
        best_res = true_res;
        for_points(L, [&](long long i, int) { best[i] = u[i]; });
        __syncthreads();
      }
      if (rz == 0.0) break;
      const T be = O::from(pol, rz_new / rz);
      for_points(L, [&](long long i, int) { p[i] = O::fma(pol, be, p[i], r[i]); });
      __syncthreads();
      rz = rz_new;
    }
    if (true_res > best_res) {
      for_points(L, [&](long long i, int) { u[i] = best[i]; });
      __syncthreads();
    }
    if (threadIdx.x == 0 && a.cg_iterations) *a.cg_iterations = it;
  }

  template <typename F>
  __device__ void by_prec(int prec, F&& f) {
    if (prec == MPMG_FP16) f(std::integral_constant<int, P16>{});
    else if (prec == MPMG_FP32) f(std::integral_constant<int, P32>{});
    else f(std::integral_constant<int, P64>{});
  }

  __device__ void copy_level(const CoarseLevel& L, const void* src, void* dst) {
    const int bytes = mpmg_dev_bytes(L.prec);
    const Pt p = points(L);
    for (long long k = threadIdx.x; k < p.n; k += blockDim.x) {
      const long long i = p.idx(k);
      if (bytes == 2) static_cast<uint16_t*>(dst)[i] = static_cast<const uint16_t*>(src)[i];
      else if (bytes == 4) static_cast<uint32_t*>(dst)[i] = static_cast<const uint32_t*>(src)[i];
      else static_cast<uint64_t*>(dst)[i] = static_cast<const uint64_t*>(src)[i];
    }
  }
  static __device__ __forceinline__ int mpmg_dev_bytes(int prec) { return prec == MPMG_FP16 ? 2 : (prec == MPMG_FP32 ? 4 : 8); }

  // smoothing with ping-pong between L.u and L.u2; returns the buffer that
  // holds the result. `cur` is the current iterate buffer (or null: zero).
  __device__ void* smooth(const CoarseLevel& L, void* cur, int steps) {
    for (int s = 0; s < steps; ++s) {
      void* out = (cur == L.u) ? L.u2 : L.u;
      const bool z = cur == nullptr;
      by_prec(L.prec, [&](auto pc) { jacobi<decltype(pc)::value>(L, L.b, z ? L.b : cur, out, z); });
      __syncthreads();
      cur = out;
    }
    return cur;
  }

  __device__ void run() {
    __shared__ double scales[kMaxCoarseLevels];
    void* cur[kMaxCoarseLevels];
    const int top = a.nlev - 1;
    // down-sweep (cycle_at before the recursive call)
    for (int l = top; l >= 1; --l) {
      const CoarseLevel& L = a.lv[l];
      void* u = smooth(L, nullptr, a.pre);
      if (u == nullptr) {  // pre_steps == 0: u = 0
        for_points(L, [&](long long i, int) {
          if (L.prec == MPMG_FP16) static_cast<uint16_t*>(L.u)[i] = 0;
          else if (L.prec == MPMG_FP32) static_cast<float*>(L.u)[i] = 0.f;
          else static_cast<double*>(L.u)[i] = 0.0;
        });
        __syncthreads();
        u = L.u;
      }
      cur[l] = u;
      by_prec(L.prec, [&](auto pc) { defect<decltype(pc)::value>(L, L.b, u, L.r); });
      __syncthreads();
      const CoarseLevel& C = a.lv[l - 1];
      by_prec(L.prec, [&](auto pc) { restrict_prod<decltype(pc)::value>(L, C, L.r); });
      __syncthreads();
      if (threadIdx.x == 0) {
        double s = 1.0;
        if (a.rescale && C.prec == MPMG_FP16) {  // multigrid.cpp:246-250
          const Pt pc = points(C);
          double acc = 0.0;
          for (long long k = 0; k < pc.n; ++k) {
            const double v = C.prod[pc.idx(k)];
            acc = __fma_rn(v, v, acc);
          }
          const double nrm = sqrt(acc);
          if (nrm > 0.0 && isfinite(nrm)) s = nrm;
        }
        scales[l - 1] = s;
      }
      __syncthreads();
      by_prec(C.prec, [&](auto pc) { restrict_store<decltype(pc)::value>(C, scales[l - 1]); });
      __syncthreads();
    }
    // base solve
    {
      const CoarseLevel& B = a.lv[0];
      by_prec(B.prec, [&](auto pc) { cg<decltype(pc)::value>(B, B.b, B.u); });
      __syncthreads();
      cur[0] = B.u;
    }
    // up-sweep
    for (int l = 1; l <= top; ++l) {
      const CoarseLevel& L = a.lv[l];
      const CoarseLevel& C = a.lv[l - 1];
      by_prec(L.prec, [&](auto fp) {
        by_prec(C.prec, [&](auto cp) {
          prolong<decltype(fp)::value, decltype(cp)::value>(L, C, cur[l - 1], cur[l], scales[l - 1]);
        });
      });
      __syncthreads();
      void* u = smooth(L, cur[l], a.post);
      if (u != L.u) {
        copy_level(L, u, L.u);
        __syncthreads();
        u = L.u;
      }
      cur[l] = u;
    }
  }
};

__global__ void __launch_bounds__(kCoarseThreads) k_coarse(const __grid_constant__ CoarseArgs a, Pol p) {
  Coarse c(a, p);
  c.run();
}

}  // namespace

cudaError_t launch_coarse_cycle(const CoarseArgs& a, uint32_t policy, cudaStream_t s) {
  const Pol p{(policy & MPMG_FTZ) != 0, (policy & MPMG_FMA) != 0, (policy & MPMG_ACC32) != 0};
  k_coarse<<<1, kCoarseThreads, 0, s>>>(a, p);
  return cudaGetLastError();
}

}  // namespace mpmg_impl
