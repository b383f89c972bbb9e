// TMA-staged 9-point stencil kernel for 2D levels (pitch P >= 32 W, a power
// of two): SpMV, level defect, damped Jacobi and the fused first two Jacobi
// steps from u = 0 in binary16 / binary32 / binary64. Reference arithmetic:
// kernels.cpp:137-212 (spmv, axpy: per-operation rounding, FTZ after
// rounding), multigrid.cpp:79-89 (jacobi_smooth), 376-380.
//
// 2D levels are HBM bound (9 taps per unknown against 3 streamed operands),
// so the kernel is built for bytes in flight:
//   * a warp owns an x segment of 32 W values (16 B per lane) and a
//     contiguous run of rows; it streams the operand rows of its segment
//     (plus one 16-byte halo each side) through its own NS-stage shared
//     memory ring, one cp.async.bulk (TMA) per row and one per b row,
//     completing on per-warp mbarriers -- no CTA barrier in the loop;
//   * each operand row is read from shared memory once and pushes its
//     contributions into the three output rows it touches (dy = +1, 0, -1
//     of rows y-1, y, y+1); output row y is finished by input row y+1, so
//     per output the FMA order is the reference's slot order (dy, dx
//     ascending, mesh_fem.cpp:124-150) -- bitwise k_stencil's results;
//   * the grid is persistent (one wave); the (segment, row) space is split
//     into equal contiguous runs per warp (>= 8 rows each).
#pragma once

#include "mpmg_plane.cuh"

namespace mpmg_dev {

template <int LP, int OP, int W, int NS>
struct R2 {
  static constexpr int B = Bytes<LP>::v;
  static constexpr int SEG = 32 * W;                // values per warp segment
  static constexpr int HALO = 16 / B;               // halo values per side (16 B)
  static constexpr int ROWB = (SEG + 2 * HALO) * B;  // staged row bytes
  static constexpr bool kB = OP == POP_DEFECT || OP == POP_JACOBI;
  static constexpr int STAGE = ROWB * (kB ? 2 : 1);  // operand row (+ b row)
  static constexpr int BARS = 128;
  static constexpr int WARP_SMEM = BARS + NS * STAGE;
  static_assert(NS >= 3 && NS * 8 <= BARS, "");
  static_assert(ROWB % 16 == 0, "");
};

template <int LP, int OP, bool FTZ, int W, int NS, int WPB>
__global__ void __launch_bounds__(32 * WPB) k_row2d(const __grid_constant__ PlaneArgs a) {
  using K = R2<LP, OP, W, NS>;
  using ST = typename Sc<LP>::T;
  constexpr bool kJZ = OP == POP_JACOBI_Z;
  extern __shared__ __align__(128) unsigned char smem[];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wbase = smem + warp * K::WARP_SMEM;
  uint64_t* full = reinterpret_cast<uint64_t*>(wbase);
  unsigned char* stages = wbase + K::BARS;
  const int P = a.P;

  pdl_wait();
  pdl_launch();
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_init(full + s, 1);
    fence_barrier_init();
  }
  __syncwarp();
  // taps (dy, dx) in slot order, and the Jacobi scalars, in LP
  using TT = decltype(tap<LP>(a, 0));
  TT tk[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) tk[k] = tap<LP>(a, k);
  const TT dd = [&] {
    if constexpr (LP == P16) return a.d16;
    else if constexpr (LP == P32) return a.d32;
    else return a.d64;
  }();
  const TT ww = [&] {
    if constexpr (LP == P16) return a.w16;
    else if constexpr (LP == P32) return a.w32;
    else return a.w64;
  }();

  const unsigned char* xg = static_cast<const unsigned char*>(a.x);
  const unsigned char* bg = static_cast<const unsigned char*>(a.b);
  const int nseg = P / K::SEG;
  const int NY = P - 1;  // output rows 1 .. P-1
  const long long T = (long long)nseg * NY;
  const long long NW = (long long)gridDim.x * WPB;
  const long long gw = (long long)blockIdx.x * WPB + warp;
  long long lo = gw * T / NW;
  const long long hi = (gw + 1) * T / NW;
  uint32_t it = 0, phase = 0;

  while (lo < hi) {
    const int xs = (int)(lo / NY);
    const int ys = (int)(lo % NY) + 1;
    const int ye = ys + (int)min((long long)(NY - (ys - 1)), hi - lo);  // outputs [ys, ye)
    lo += ye - ys;
    const int xseg = xs * K::SEG;
    const int x0 = xseg + lane * W;
    const int HL = xseg > 0 ? K::HALO : 0;
    const int HR = xseg + K::SEG < P ? K::HALO : 0;
    const uint32_t nb = (uint32_t)((K::SEG + HL + HR) * K::B);
    const int NQ = ye - ys + 2;  // input rows ys-1 .. ye

    // the halo the copies leave untouched at the level edges reads as zero
    // (x = P ghost; the x = -1 value only feeds the ghost output x = 0)
    if (HR == 0 || HL == 0) {
      __syncwarp();
      for (int s = lane; s < NS; s += 32) {
        if (HR == 0) *reinterpret_cast<uint4*>(stages + s * K::STAGE + (K::HALO + K::SEG) * K::B) = make_uint4(0, 0, 0, 0);
        if (HL == 0) *reinterpret_cast<uint4*>(stages + s * K::STAGE) = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
    }
    // lane 0: input row k (y = ys - 1 + k; rows 0 and P are the zero ghost rows,
    // stored in the padded layout) and the b row of output ys - 2 + k
    auto issue = [&](int k) {
      const int y = ys - 1 + k;
      const uint32_t s = (it + k) % NS;
      unsigned char* st = stages + s * K::STAGE;
      const bool bop = K::kB && k >= 1;
      mbar_arrive_tx(full + s, nb * (bop ? 2u : 1u));
      bulk_g2s(st + (K::HALO - HL) * K::B, xg + ((long long)y * P + xseg - HL) * K::B, nb, full + s);
      if (bop)
        bulk_g2s(st + K::ROWB + (K::HALO - HL) * K::B, bg + ((long long)(y - 1) * P + xseg - HL) * K::B, nb, full + s);
    };
    if (lane == 0) {
      fence_proxy_async();
      for (int k = 0; k < NS - 1 && k < NQ; ++k) issue(k);
    }

    Row<LP, W> acc[3];  // outputs y-1 (finish), y (middle), y+1 (start)
#pragma unroll
    for (int m = 0; m < 3; ++m) rzero(acc[m]);
    for (int k = 0; k < NQ; ++k) {
      const uint32_t s = (it + k) % NS;
      const unsigned char* st = stages + s * K::STAGE;
      mbar_wait(full + s, (phase >> s) & 1u);
      phase ^= 1u << s;
      const unsigned char* rp = st + (K::HALO + lane * W) * K::B;
      Row<LP, W> c, L, R;
      rload<LP, LP, W>(rp, c);
      ST prev = sload_s<LP, LP>(rp - K::B);
      ST next = sload_s<LP, LP>(rp + W * K::B);
      if constexpr (kJZ) {
        jz_row<LP, FTZ, true, W>(dd, ww, c);
        prev = jz_scalar<LP, FTZ, true, ST>(dd, ww, prev);
        next = jz_scalar<LP, FTZ, true, ST>(dd, ww, next);
      }
      rshift<LP, W>(c, prev, next, L, R);
      const bool fin = k >= 2, mid = k >= 1 && k <= NQ - 2, sta = k <= NQ - 3;
#pragma unroll
      for (int role = 0; role < 3; ++role) {  // finish: dy=+1 taps 6..8; middle: 3..5; start: 0..2
        if (!(role == 0 ? fin : (role == 1 ? mid : sta))) continue;
        const int t0 = (2 - role) * 3;
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) rfma<LP, FTZ, true, W>(tk[t0 + dx], dx == 0 ? L : (dx == 1 ? c : R), acc[role]);
      }
      if (fin) {  // output row y - 1: its b row is in this stage, its centre u in the previous one
        const int yo = ys - 2 + k;
        const long long gi = (long long)yo * P + x0;
        Row<LP, W> t = acc[0];
        const unsigned char* prv = stages + ((it + k + NS - 1) % NS) * K::STAGE + (K::HALO + lane * W) * K::B;
        if constexpr (OP == POP_SPMV) {
          if (x0 == 0) rzero_first<LP, W>(t);
          gstore<LP, W>(a.out, gi, t);
        } else {
          Row<LP, W> bb;
          if constexpr (kJZ) rload<LP, LP, W>(prv, bb);
          else rload<LP, LP, W>(st + K::ROWB + (K::HALO + lane * W) * K::B, bb);
          Row<LP, W> r;
          if constexpr (LP == P16) r = efma<LP, FTZ, true, W>(u2h(0xBC00BC00u), t, bb);  // axpy(-1, t, b)
          else r = efma<LP, FTZ, true, W>(ST(-1), t, bb);
          if constexpr (OP == POP_DEFECT) {
            if (x0 == 0) rzero_first<LP, W>(r);
            gstore<LP, W>(a.out, gi, r);
          } else {
            const Row<LP, W> dr = emul<LP, FTZ, W>(dd, r);  // vec_multiply(inv_diag, r)
            Row<LP, W> uc;
            if constexpr (kJZ) {
              uc = bb;
              jz_row<LP, FTZ, true, W>(dd, ww, uc);
            } else {
              rload<LP, LP, W>(prv, uc);
            }
            Row<LP, W> un = efma<LP, FTZ, true, W>(ww, dr, uc);  // axpy(omega, t, u)
            if (x0 == 0) rzero_first<LP, W>(un);
            gstore<LP, W>(a.out, gi, un);
          }
        }
      }
      acc[0] = acc[1];
      acc[1] = acc[2];
      rzero(acc[2]);
      __syncwarp();
      if (lane == 0 && k + NS - 1 < NQ) {
        fence_proxy_async();
        issue(k + NS - 1);  // into the stage of row k-1, free now
      }
    }
    it += NQ;
  }
}

}  // namespace mpmg_dev
