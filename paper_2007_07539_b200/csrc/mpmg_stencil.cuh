// Streaming 27-point (3D) / 9-point (2D) stencil kernels on the ghost-aliased
// pitch layout (include/mpmg_gpu.h).
//
// One kernel template implements every "SpMV + pointwise epilogue" of the hot
// path. The reference computes each of these as separate ELL passes
// (kernels.cpp:137-193 then axpy/vec_multiply); here the stencil sum and its
// epilogue are one pass over HBM:
//
//   OP_SPMV     y = A x                                  (kernels.cpp:137-193)
//   OP_DEFECT   r = b - A u                               (multigrid.cpp:379-380)
//   OP_JACOBI   u' = u + w D^-1 (b - A u)                 (multigrid.cpp:79-89)
//   OP_DEFECT64 r = b - A u in FP64 (+ ||r||^2 partials)  (ir_solver.cpp:92-93,115-119)
//   OP_RESNORM  ||b - A u||^2 partials, fma chain         (ir_solver.cpp:21-49)
//   OP_UPDATE   u += a c, r -= a A c (+ partials)         (kernels.cpp:300-341)
//
// Work decomposition: a lane owns W consecutive x-values (one 64/128-bit
// access per row); a warp covers 32*W values of a row; in 3D each thread owns
// RY consecutive rows and streams along z through a block-private range of
// ZC planes, keeping three accumulator slots (outputs z-1, z, z+1). Each
// loaded plane row therefore feeds three outputs from registers; x-neighbours
// come from lane shuffles (one halo value per warp edge). The summation order
// of every output is exactly the reference's ELL slot order: dz, dy, dx
// ascending (mesh_fem.cpp:124-150), each product rounded per
// operation. Boundary neighbours read the stored zeros of the ghost nodes: an
// extra fma(a, 0, acc) leaves every nonzero acc unchanged (it can only flip
// the sign of an exactly-zero acc), so results equal the reference's
// compacted-row results value-for-value.
#pragma once

#include "mpmg_vec.cuh"

namespace mpmg_dev {

enum { OP_SPMV = 0, OP_DEFECT = 1, OP_JACOBI = 2, OP_DEFECT64 = 3, OP_RESNORM = 4, OP_UPDATE = 5, OP_UPDATE_R = 6 };
// OP_UPDATE_R: the r half of OP_UPDATE (r -= a A c, + partials) and c copied
//   into ring slot *ring_slot (deferred u += a c, as POP_UPDATE_R in
//   mpmg_plane.cuh; the streaming form serves 2D and non-plane pitches)

struct StencilArgs {
  int P;             // pitch (nodes - 1)
  int zc;            // planes per block
  long long plane;   // plane stride: P*P (3D) or P (2D)
  __half2 t16[27];   // taps, broadcast binary16 pairs
  float t32[27];
  double t64[27];
  __half2 d16, w16;  // D^-1 and omega rounded to binary16
  float d32, w32;
  double d64, w64;
  const void* x;     // stencil operand (u, or c for OP_UPDATE)
  const void* b;     // right-hand side (OP_DEFECT/JACOBI/DEFECT64/RESNORM)
  void* out;         // output vector (y / r / u')
  double* r64;       // OP_UPDATE in/out
  double* u64;       // OP_UPDATE in/out
  const double* alpha;  // OP_UPDATE scale (device scalar)
  double* partials;  // optional per-block sum of squares
  const int* gate;   // optional device flag: kernel is a no-op unless *gate != 0
  void* ring;          // OP_UPDATE_R: correction ring (slots of ring_len values, precision LP)
  long long ring_len;
  const int* ring_slot;
  double* ring_scale;  // per-slot scale (= *alpha)
};

template <int CP> struct Taps;
template <> struct Taps<P16> { static __device__ __forceinline__ __half2 get(const StencilArgs& a, int i) { return a.t16[i]; } };
template <> struct Taps<P32> { static __device__ __forceinline__ float get(const StencilArgs& a, int i) { return a.t32[i]; } };
template <> struct Taps<P64> { static __device__ __forceinline__ double get(const StencilArgs& a, int i) { return a.t64[i]; } };

template <int OP> struct OpTraits {
  static constexpr bool kNeedB = OP == OP_DEFECT || OP == OP_JACOBI || OP == OP_DEFECT64 || OP == OP_RESNORM;
  static constexpr bool kNorm = OP == OP_DEFECT64 || OP == OP_RESNORM || OP == OP_UPDATE || OP == OP_UPDATE_R;
};

// block-level deterministic sum of one double per thread -> partials[block]
template <int NT>
__device__ __forceinline__ void block_partial(double v, double* partials) {
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < NT / 32; ++w) s += red[w];
    partials[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s;
  }
}

// DIM: 2/3. LP: storage precision of the stencil operand. CP: accumulation
// precision. EP: epilogue/output precision. BW warps per block.
template <int DIM, int LP, int CP, int EP, int OP, bool FTZ, bool FMA, int RY, int BW>
__global__ void __launch_bounds__(32 * BW) k_stencil(const __grid_constant__ StencilArgs a) {
  constexpr int W = LaneWidth<LP>::W;
  constexpr int NR = DIM == 3 ? RY + 2 : 1;  // rows loaded per plane
  constexpr int NO = DIM == 3 ? RY : 1;      // output rows per thread
  constexpr int TPP = DIM == 3 ? 9 : 3;      // taps per plane
  using S = typename Scalar<CP>::T;

  if (a.gate && *a.gate == 0) return;  // uniform across the grid
  if constexpr (OP == OP_UPDATE_R) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0 && threadIdx.y == 0)
      a.ring_scale[*a.ring_slot] = *a.alpha;
  }
  const int lane = threadIdx.x;
  const int P = a.P;
  const long long xchunk = DIM == 3 ? (long long)blockIdx.x * 32 + lane
                                    : ((long long)blockIdx.x * BW + threadIdx.y) * 32 + lane;
  const int x0 = (int)(xchunk * W);
  const bool xvalid = x0 < P;
  const int y0 = DIM == 3 ? 1 + (int)(blockIdx.y * BW + threadIdx.y) * RY : 0;
  const int z0 = 1 + (int)blockIdx.z * a.zc;
  const int z1 = min(z0 + a.zc, P);  // outputs [z0, z1)
  const long long plane = a.plane;

  double sq = 0.0;  // sum of squares for OpTraits::kNorm

  // rows of one plane: lane vector + halo scalar (lane 0: x0-1, lane 31: x0+W)
  Vec<CP, W> cur[NR], nxt[NR];
  S ecur[NR], enxt[NR];
  auto load_plane = [&](int q, Vec<CP, W>* rows, S* edge) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const int y = DIM == 3 ? y0 - 1 + j : 0;
      const bool yv = DIM == 3 ? (y <= P) : true;
      const long long base = (long long)q * plane + (long long)y * (DIM == 3 ? P : 0);
      rows[j] = vload<LP, CP, W>(a.x, base + x0, yv && xvalid);
      const int ex = lane == 0 ? x0 - 1 : x0 + W;
      const bool ev = yv && (lane == 0 || lane == 31) && ex >= 0 && ex < P;
      edge[j] = sload<LP, CP>(a.x, base + ex, ev);
    }
  };

  Vec<CP, W> acc0[NO], acc1[NO], acc2[NO];  // outputs q-1, q, q+1
  Vec<CP, W> cen[NO];                        // centre values of plane q-1
#pragma unroll
  for (int i = 0; i < NO; ++i) {
    acc0[i] = vzero<CP, W>(); acc1[i] = vzero<CP, W>(); acc2[i] = vzero<CP, W>(); cen[i] = vzero<CP, W>();
  }

  const bool active = (DIM == 3 ? y0 <= P - 1 : true) && z0 <= P - 1;
  if (active) load_plane(z0 - 1, cur, ecur);

  for (int q = z0 - 1; active && q <= z1; ++q) {
    if (q + 1 <= z1) load_plane(q + 1, nxt, enxt);

    // epilogue operands of output plane q-1 (issued early)
    const int zo = q - 1;
    const bool emit = zo >= z0;
    Vec<EP, W> bo[NO];
    Vec<P64, W> uo[NO], ro[NO];
    if (emit) {
#pragma unroll
      for (int i = 0; i < NO; ++i) {
        const int y = DIM == 3 ? y0 + i : 0;
        const bool v = xvalid && (DIM == 3 ? y <= P - 1 : true);
        const long long idx = (long long)zo * plane + (long long)y * (DIM == 3 ? P : 0) + x0;
        if constexpr (OpTraits<OP>::kNeedB) bo[i] = vload<EP, EP, W>(a.b, idx, v);
        if constexpr (OP == OP_UPDATE) {
          uo[i] = vload_rw<P64, W>(a.u64, idx, v);
          ro[i] = vload_rw<P64, W>(a.r64, idx, v);
        }
        if constexpr (OP == OP_UPDATE_R) ro[i] = vload_rw<P64, W>(a.r64, idx, v);
      }
    }

    // x-shifted neighbours of this plane's rows
    Vec<CP, W> Lr[NR], Rr[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const S up = shfl_up1(vlast<CP, W>(cur[j]));
      const S dn = shfl_dn1(vfirst<CP, W>(cur[j]));
      const S prev = lane == 0 ? ecur[j] : up;
      const S next = lane == 31 ? ecur[j] : dn;
      vshift<CP, W>(cur[j], prev, next, Lr[j], Rr[j]);
    }

    // accumulate: slot 0 gets dz=+1 taps, slot 1 dz=0, slot 2 dz=-1
#pragma unroll
    for (int i = 0; i < NO; ++i) {
#pragma unroll
      for (int dy = 0; dy < (DIM == 3 ? 3 : 1); ++dy) {
        const int j = DIM == 3 ? i + dy : 0;
        const int tb = DIM == 3 ? dy * 3 : 0;
        vfma<CP, FTZ, FMA, W>(Taps<CP>::get(a, 2 * TPP + tb + 0), Lr[j], acc0[i]);
        vfma<CP, FTZ, FMA, W>(Taps<CP>::get(a, 2 * TPP + tb + 1), cur[j], acc0[i]);
        vfma<CP, FTZ, FMA, W>(Taps<CP>::get(a, 2 * TPP + tb + 2), Rr[j], acc0[i]);
        vfma<CP, FTZ, FMA, W>(Taps<CP>::get(a, 1 * TPP + tb + 0), Lr[j], acc1[i]);
        vfma<CP, FTZ, FMA, W>(Taps<CP>::get(a, 1 * TPP + tb + 1), cur[j], acc1[i]);
        vfma<CP, FTZ, FMA, W>(Taps<CP>::get(a, 1 * TPP + tb + 2), Rr[j], acc1[i]);
        vfma<CP, FTZ, FMA, W>(Taps<CP>::get(a, 0 * TPP + tb + 0), Lr[j], acc2[i]);
        vfma<CP, FTZ, FMA, W>(Taps<CP>::get(a, 0 * TPP + tb + 1), cur[j], acc2[i]);
        vfma<CP, FTZ, FMA, W>(Taps<CP>::get(a, 0 * TPP + tb + 2), Rr[j], acc2[i]);
      }
    }

    // epilogue of output plane q-1
    if (emit) {
#pragma unroll
      for (int i = 0; i < NO; ++i) {
        const int y = DIM == 3 ? y0 + i : 0;
        const bool v = xvalid && (DIM == 3 ? y <= P - 1 : true);
        const long long idx = (long long)zo * plane + (long long)y * (DIM == 3 ? P : 0) + x0;
        Vec<EP, W> t;
        if constexpr (CP == EP) t = acc0[i];
        else t = vquant16<FTZ, W>(acc0[i]);  // binary32 accumulation -> binary16
        if constexpr (OP == OP_SPMV) {
          if (x0 == 0) vzero_first<EP, W>(t);
          if (v) vstore<EP, W>(a.out, idx, t);
        } else if constexpr (OP == OP_DEFECT || OP == OP_JACOBI) {
          typename Coef<EP>::T m1, dd, ww;
          if constexpr (EP == P16) { m1 = u2h(0xBC00BC00u); dd = a.d16; ww = a.w16; }
          else if constexpr (EP == P32) { m1 = -1.0f; dd = a.d32; ww = a.w32; }
          else { m1 = -1.0; dd = a.d64; ww = a.w64; }
          Vec<EP, W> r = vfma3<EP, FTZ, FMA, W>(m1, t, bo[i]);  // axpy(-1, t, b)
          if constexpr (OP == OP_DEFECT) {
            if (x0 == 0) vzero_first<EP, W>(r);
            if (v) vstore<EP, W>(a.out, idx, r);
          } else {
            const Vec<EP, W> dr = vmul<EP, FTZ, W>(dd, r);     // vec_multiply(inv_diag, r)
            Vec<EP, W> uc;
            if constexpr (CP == EP) uc = cen[i];
            else {
#pragma unroll
              for (int k = 0; k < W / 2; ++k) uc.h[k] = __floats2half2_rn(cen[i].v[2 * k], cen[i].v[2 * k + 1]);
            }
            Vec<EP, W> un = vfma3<EP, FTZ, FMA, W>(ww, dr, uc);  // axpy(omega, t, u)
            if (x0 == 0) vzero_first<EP, W>(un);
            if (v) vstore<EP, W>(a.out, idx, un);
          }
        } else if constexpr (OP == OP_DEFECT64 || OP == OP_RESNORM) {
          Vec<P64, W> r;
#pragma unroll
          for (int k = 0; k < W; ++k)
            r.v[k] = OP == OP_RESNORM ? __dsub_rn(bo[i].v[k], t.v[k]) : fma64<FMA>(-1.0, t.v[k], bo[i].v[k]);
          if (x0 == 0) vzero_first<P64, W>(r);
          if (v) {
            if (OP == OP_DEFECT64 && a.out) vstore<P64, W>(a.out, idx, r);
            sq = vsumsq<P64, W>(r, sq);
          }
        } else if constexpr (OP == OP_UPDATE) {
          const double al = *a.alpha;
          Vec<P64, W> un, rn;
#pragma unroll
          for (int k = 0; k < W; ++k) {
            un.v[k] = fma64<FMA>(al, cen[i].v[k], uo[i].v[k]);
            rn.v[k] = fma64<FMA>(-al, t.v[k], ro[i].v[k]);
          }
          if (x0 == 0) { vzero_first<P64, W>(un); vzero_first<P64, W>(rn); }
          if (v) {
            vstore<P64, W>(a.u64, idx, un);
            vstore<P64, W>(a.r64, idx, rn);
            sq = vsumsq<P64, W>(rn, sq);
          }
        } else if constexpr (OP == OP_UPDATE_R) {
          const double al = *a.alpha;
          Vec<P64, W> rn;
#pragma unroll
          for (int k = 0; k < W; ++k) rn.v[k] = fma64<FMA>(-al, t.v[k], ro[i].v[k]);
          if (x0 == 0) vzero_first<P64, W>(rn);
          if (v) {
            vstore<P64, W>(a.r64, idx, rn);
            sq = vsumsq<P64, W>(rn, sq);
            // c unchanged into the ring slot (its x = 0 ghost is zero)
            const Vec<LP, W> craw = vload_rw<LP, W>(a.x, idx, true);
            vstore<LP, W>(static_cast<unsigned char*>(a.ring) +
                              (long long)*a.ring_slot * a.ring_len * (LP == P16 ? 2 : (LP == P32 ? 4 : 8)),
                          idx, craw);
          }
        }
      }
    }

    // rotate accumulators and plane buffers
#pragma unroll
    for (int i = 0; i < NO; ++i) {
      acc0[i] = acc1[i];
      acc1[i] = acc2[i];
      acc2[i] = vzero<CP, W>();
      cen[i] = cur[DIM == 3 ? i + 1 : 0];
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) { cur[j] = nxt[j]; ecur[j] = enxt[j]; }
  }

  if constexpr (OpTraits<OP>::kNorm) {
    if (a.partials) block_partial<32 * BW>(sq, a.partials);
  }
}

// ---- launch geometry (shared by the launcher and the partials sizing) ----
template <int LP, int CP> struct Geo {
  static constexpr int W = LaneWidth<LP>::W;
  static constexpr int RY = (LP == P16 && CP == P16) ? 4 : 2;
  static constexpr int BW = 4;
  static constexpr int ZC = 16;
};

inline dim3 stencil_grid(int dim, int P, int W, int RY, int BW, int ZC) {
  const int xch = (P + W - 1) / W;
  const int zb = (P - 1 + ZC - 1) / ZC;
  if (dim == 3) {
    const int rg = (P - 1 + RY - 1) / RY;
    return dim3((xch + 31) / 32, (rg + BW - 1) / BW, zb);
  }
  return dim3((xch + 32 * BW - 1) / (32 * BW), 1, zb);
}

}  // namespace mpmg_dev
