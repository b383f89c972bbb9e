// Host-side setup of the hot path: per-level stencil coefficients, binary16
// rounding of per-level scalars and the manufactured right-hand side. Runs
// once per hierarchy (the reference's MgHierarchy::build, multigrid.cpp:
// 282-323, which assembles full ELL matrices; here only the 3^dim distinct
// coefficients of each level are needed because every row of the assembled
// operator carries the same values).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numbers>
#include <thread>
#include <vector>

#include "mpmg_host.h"

namespace mpmg_impl {

namespace {

uint64_t dbits(double x) { uint64_t u; std::memcpy(&u, &x, 8); return u; }
double bitsd(uint64_t u) { double x; std::memcpy(&x, &u, 8); return x; }

// 2-point Gauss rule on [0,1] (mesh_fem.cpp:13-17)
constexpr double kGaussOff = 0.28867513459481287;
double gauss(int i) { return i == 0 ? 0.5 - kGaussOff : 0.5 + kGaussOff; }
double phi1(int node, double t) { return node == 0 ? 1.0 - t : t; }
double dphi1(int node) { return node == 0 ? -1.0 : 1.0; }

// element stiffness entry on the reference cell (mesh_fem.cpp:21-51):
// sum over Gauss points of w * grad(phi_a) . grad(phi_b)
double cell_entry(int dim, int a, int b) {
  double acc = 0.0;
  for (int g = 0; g < (1 << dim); ++g) {
    double xi[3] = {0.0, 0.0, 0.0};
    for (int d = 0; d < dim; ++d) xi[d] = gauss((g >> d) & 1);
    double w = 1.0;
    for (int d = 0; d < dim; ++d) w *= 0.5;
    double dot = 0.0;
    for (int d = 0; d < dim; ++d) {
      double ga = dphi1((a >> d) & 1), gb = dphi1((b >> d) & 1);
      for (int e = 0; e < dim; ++e) {
        if (e == d) continue;
        ga *= phi1((a >> e) & 1, xi[e]);
        gb *= phi1((b >> e) & 1, xi[e]);
      }
      dot += ga * gb;
    }
    acc += w * dot;
  }
  return acc;
}

}  // namespace

double round_fp16(double x, bool ftz) {
  const uint64_t u = dbits(x);
  const uint64_t mag = u & 0x7FFFFFFFFFFFFFFFull;
  if (mag == 0) return x;
  if (mag >= 0x7FF0000000000000ull) return mag > 0x7FF0000000000000ull ? std::nan("") : x;
  if (mag >= 0x40EFFE0000000000ull) return (u >> 63) ? -INFINITY : INFINITY;  // >= 65520
  if (mag < 0x3F20000000000000ull) {  // below 2^-13 the grid is 2^-24 apart
    const double q = std::ldexp(std::nearbyint(std::ldexp(std::fabs(x), 24)), -24);
    if (q == 0.0 || (ftz && q < 0x1p-14)) return std::copysign(0.0, x);
    return std::copysign(q, x);
  }
  // 11 significant bits: round the low 42 fraction bits to nearest even
  const uint64_t keep = u & ~0x3FFFFFFFFFFull, rest = u & 0x3FFFFFFFFFFull, half = 0x20000000000ull;
  uint64_t r = keep;
  if (rest > half || (rest == half && (keep & 0x40000000000ull))) r += 0x40000000000ull;
  return bitsd(r);
}

double round_to(double x, int prec, bool ftz) {
  if (prec == MPMG_FP16) return round_fp16(x, ftz);
  if (prec == MPMG_FP32) {
    const float f = static_cast<float>(x);
    if (ftz && f != 0.0f && std::fabs(f) < 1.17549435e-38f) return std::copysign(0.0, static_cast<double>(f));
    return static_cast<double>(f);
  }
  return x;
}

uint16_t fp16_bits(double v) {
  const uint64_t u = dbits(v);
  const uint16_t sign = static_cast<uint16_t>((u >> 48) & 0x8000u);
  if ((u & 0x7FFFFFFFFFFFFFFFull) == 0) return sign;
  if (std::isnan(v)) return 0x7E00;
  if (std::isinf(v)) return static_cast<uint16_t>(sign | 0x7C00);
  const int e = static_cast<int>((u >> 52) & 0x7FF) - 1023;
  if (e < -14) return static_cast<uint16_t>(sign | static_cast<uint16_t>(std::fabs(v) * 0x1p24));
  return static_cast<uint16_t>(sign | ((e + 15) << 10) | ((u >> 42) & 0x3FF));
}

double fp16_value(uint16_t h) {
  const int e = (h >> 10) & 0x1F, m = h & 0x3FF;
  double v;
  if (e == 31) v = m ? std::nan("") : INFINITY;
  else if (e == 0) v = m * 0x1p-24;
  else v = std::ldexp(1.0 + m / 1024.0, e - 15);
  return (h & 0x8000) ? -v : v;
}

// The 3^dim coefficients of an interior row of the Q1 stiffness on a grid with
// n nodes per dimension, accumulated exactly as the element loop of
// assemble_stiffness (mesh_fem.cpp:88-123) adds them for one node: elements in
// (ez, ey, ex) order, the node's local index a fixed per element, partner b.
int stencil_taps(int dim, int n, double* taps) {
  if ((dim != 2 && dim != 3) || n < 3) return -1;
  const int ln = 1 << dim, ntaps = dim == 3 ? 27 : 9;
  const double h = 1.0 / (n - 1);
  const double hs = dim == 2 ? 1.0 : h;  // element matrix = h^(dim-2) * reference cell
  double el[64];
  for (int a = 0; a < ln; ++a)
    for (int b = 0; b < ln; ++b) el[a * ln + b] = hs * cell_entry(dim, a, b);
  for (int t = 0; t < ntaps; ++t) taps[t] = 0.0;
  // the node sits at local corner a = (1-ex, 1-ey, 1-ez) of the element whose
  // lower corner is offset (ex-1, ey-1, ez-1) from it
  for (int ez = 0; ez < (dim == 3 ? 2 : 1); ++ez)
    for (int ey = 0; ey < 2; ++ey)
      for (int ex = 0; ex < 2; ++ex) {
        const int a = (1 - ex) | ((1 - ey) << 1) | (dim == 3 ? (1 - ez) << 2 : 0);
        for (int b = 0; b < ln; ++b) {
          const int dx = (b & 1) - (a & 1), dy = ((b >> 1) & 1) - ((a >> 1) & 1);
          const int dz = dim == 3 ? ((b >> 2) & 1) - ((a >> 2) & 1) : 0;
          const int t = dim == 3 ? ((dz + 1) * 3 + (dy + 1)) * 3 + (dx + 1) : (dy + 1) * 3 + (dx + 1);
          taps[t] += el[a * ln + b];
        }
      }
  return ntaps;
}

// assemble_rhs (mesh_fem.cpp:157-202) into the compact interior ordering
// Manufactured load vector (assemble_rhs, mesh_fem.cpp:157-202): the same
// element-order accumulation b[node] += w * f * phi, bitwise, but
//   * the per-dimension sine factors sin(k pi h (e + xi)) and the Gauss
//     weights / shape values come from tables computed with the identical
//     expressions (f = amp * S_x * S_y [* S_z] in the same order);
//   * element layers (the outermost element index) are split over threads.
//     A node plane shared by two threads' ranges receives the lower range's
//     terms first: each thread first adds the terms of its first layer that
//     land on the plane ABOVE it and all of its other layers, and only after
//     every thread is done the terms of its first layer on the plane at its
//     own lower boundary -- per node the additions happen in the sequential
//     order, so every entry is bitwise the single-threaded sum (a minute at
//     1025^3 instead of ~10).
void problem_rhs(int dim, int n, int k, double* b) {
  const double h = 1.0 / (n - 1);
  const double kpi = k * std::numbers::pi;
  const double amp = dim * kpi * kpi;
  double jac = 1.0;
  for (int d = 0; d < dim; ++d) jac *= h;
  const long long m = n - 2;
  const long long N = dim == 3 ? m * m * m : m * m;
  std::memset(b, 0, static_cast<size_t>(N) * sizeof(double));
  const int ng = 1 << dim;
  double w = jac;
  for (int d = 0; d < dim; ++d) w *= 0.5;
  // sin(kpi * h * (e + xi)) for e in [0, n-1), xi = gauss(0|1)
  std::vector<double> S(static_cast<size_t>(n - 1) * 2);
  for (int e = 0; e < n - 1; ++e)
    for (int q = 0; q < 2; ++q) S[static_cast<size_t>(e) * 2 + q] = std::sin(kpi * h * (e + gauss(q)));
  double phiT[8][8];  // [g][a]
  for (int g = 0; g < ng; ++g)
    for (int a = 0; a < ng; ++a) {
      double phi = 1.0;
      for (int d = 0; d < dim; ++d) phi *= phi1((a >> d) & 1, gauss((g >> d) & 1));
      phiT[g][a] = phi;
    }
  auto interior = [n](int i) { return i >= 1 && i <= n - 2; };
  const int outer = dim - 1;  // the element index split over threads (z in 3D, y in 2D)
  // element layer lo (outer index) restricted to the nodes whose outer offset
  // is `sel` (0 or 1; 2 = both)
  auto layer = [&](int lo, int sel) {
    const int e2 = dim == 3 ? lo : 0;
    const int ylo = dim == 3 ? 0 : lo, yhi = dim == 3 ? n - 1 : lo + 1;
    for (int ey = ylo; ey < yhi; ++ey)
      for (int ex = 0; ex < n - 1; ++ex) {
        const int e[3] = {ex, ey, e2};
        for (int g = 0; g < ng; ++g) {
          double f = amp;
          for (int d = 0; d < dim; ++d) f *= S[static_cast<size_t>(e[d]) * 2 + ((g >> d) & 1)];
          const double wf = w * f;
          for (int a = 0; a < ng; ++a) {
            const int off = (a >> outer) & 1;
            if (sel != 2 && off != sel) continue;
            const int ax = ex + (a & 1), ay = ey + ((a >> 1) & 1), az = dim == 3 ? e2 + ((a >> 2) & 1) : 1;
            if (!interior(ax) || !interior(ay) || (dim == 3 && !interior(az))) continue;
            long long idx = static_cast<long long>(ay - 1) * m + (ax - 1);
            if (dim == 3) idx += static_cast<long long>(az - 1) * m * m;
            b[idx] += wf * phiT[g][a];
          }
        }
      }
  };
  const int layers = n - 1;
  int nt = static_cast<int>(std::thread::hardware_concurrency());
  if (const char* e = std::getenv("MPMG_RHS_THREADS")) nt = std::atoi(e);
  nt = std::max(1, std::min(nt, layers / 4));
  if (nt == 1) {
    for (int l = 0; l < layers; ++l) layer(l, 2);
    return;
  }
  auto lo_of = [&](int t) { return static_cast<int>(static_cast<long long>(layers) * t / nt); };
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)  // phase 1
    th.emplace_back([&, t] {
      const int l0 = lo_of(t), l1 = lo_of(t + 1);
      layer(l0, t == 0 ? 2 : 1);
      for (int l = l0 + 1; l < l1; ++l) layer(l, 2);
    });
  for (auto& x : th) x.join();
  th.clear();
  for (int t = 1; t < nt; ++t) th.emplace_back([&, t] { layer(lo_of(t), 0); });  // phase 2
  for (auto& x : th) x.join();
}

int variant_precision(int variant, int l) {  // VariantConfig::make, multigrid.cpp:54-77
  switch (variant) {
    case MPMG_D_MG: return MPMG_FP64;
    case MPMG_H_MG: return MPMG_FP16;
    case MPMG_HSD_MG: return l <= 1 ? MPMG_FP64 : (l == 2 ? MPMG_FP32 : MPMG_FP16);
    default: return l <= 1 ? MPMG_FP16 : (l == 2 ? MPMG_FP32 : MPMG_FP64);
  }
}

int build_level_stencil(int dim, int nodes, int prec, bool ftz, mpmg_stencil* out) {
  double taps[27];
  const int nt = stencil_taps(dim, nodes, taps);
  if (nt < 0) return MPMG_EINVAL;
  std::memset(out, 0, sizeof(*out));
  out->dim = dim;
  out->nodes = nodes;
  out->prec = prec;
  out->ntaps = nt;
  const int centre = nt / 2;
  // cast_checked (multigrid.cpp:25-33): binary16 overflow of any stored entry.
  // With a single interior node only the centre coefficient is stored.
  if (prec == MPMG_FP16) {
    double mx = 0.0;
    for (int t = 0; t < nt; ++t)
      if (nodes > 3 || t == centre) mx = std::fmax(mx, std::fabs(taps[t]));
    if (mx > 65504.0) return MPMG_EBUILD;
  }
  for (int t = 0; t < nt; ++t) out->taps[t] = round_to(taps[t], prec, ftz);
  // inverse diagonal from the FP64 diagonal, then cast (multigrid.cpp:296-310)
  out->inv_diag = round_to(1.0 / taps[centre], prec, ftz);
  return MPMG_OK;
}

}  // namespace mpmg_impl
