// Drop-in test of the C++ API (include/mpmg/*.hpp) on the device: the
// reference's own kernel known-answer tests (proj/tests/test_kernels.cpp:
// 92-349) restated, plus end-to-end solves pinned to the reference's golden
// results (tests/golden/solves.npz) and a cross-check of
// the fused stencil path against the generic ELLPACK path.
//   built + run by tests/test_cpp_api.py
#include <cmath>
#include <cstdio>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "mpmg/errors.hpp"
#include "mpmg/ir_solver.hpp"
#include "mpmg/kernels.hpp"
#include "mpmg/mesh_fem.hpp"
#include "mpmg/multigrid.hpp"
#include "mpmg/rng.hpp"

using namespace mpmg;

static int g_checks = 0, g_fail = 0;
#define CHECK(c)                                                               \
  do {                                                                         \
    ++g_checks;                                                                \
    if (!(c)) {                                                                \
      ++g_fail;                                                                \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);                 \
    }                                                                          \
  } while (0)
#define CHECK_THROWS(stmt, T)                                                  \
  do {                                                                         \
    bool thrown = false;                                                       \
    try { stmt; } catch (const T&) { thrown = true; } catch (...) {}           \
    CHECK(thrown);                                                             \
  } while (0)

static bool bits_equal(const PVector& a, const PVector& b) {
  if (a.size() != b.size() || a.precision() != b.precision()) return false;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const double x = a.get(i), y = b.get(i);
    if (!(x == y && std::signbit(x) == std::signbit(y)) && !(std::isnan(x) && std::isnan(y))) return false;
  }
  return true;
}
static bool values_equal(const PVector& a, const PVector& b) {  // +0 == -0
  if (a.size() != b.size()) return false;
  for (std::size_t i = 0; i < a.size(); ++i)
    if (!(a.get(i) == b.get(i)) && !(std::isnan(a.get(i)) && std::isnan(b.get(i)))) return false;
  return true;
}
static PVector random_vector(SplitMix64& rng, std::size_t n, Precision p, double lo = -1.0, double hi = 1.0) {
  PVector v(n, p);
  for (std::size_t i = 0; i < n; ++i) v.set(i, lo + (hi - lo) * rng.next_double());
  return v;
}

static void kernel_kats() {
  ExecContext ctx;
  SplitMix64 rng(1);
  for (Precision p : {Precision::FP16, Precision::FP32, Precision::FP64}) {  // test_kernels.cpp:92-106
    const EllMatrix I = EllMatrix::identity(12, p);
    const PVector x = random_vector(rng, 12, p);
    CHECK(bits_equal(spmv(I, x, ctx), x));
  }
  // ELL spmv == dense per-op reference in every precision (test_kernels.cpp:108-127)
  SplitMix64 r2(42);
  for (Precision p : {Precision::FP16, Precision::FP32, Precision::FP64}) {
    for (std::size_t n : {3u, 8u, 17u, 32u}) {
      std::vector<std::vector<std::pair<std::int32_t, double>>> rows(n);
      for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j)
          if (r2.next_u64() % 3 == 0) rows[i].emplace_back(static_cast<std::int32_t>(j), 2.0 * r2.next_double() - 1.0);
      const EllMatrix A = EllMatrix::from_entries(n, n, rows, p);
      const PVector x = random_vector(r2, n, p);
      const PVector y = spmv(A, x, ctx);
      PVector e(n, p);
      for (std::size_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int s = 0; s < A.row_width(); ++s) {
          const double a = A.value(i, s), xv = x.get(static_cast<std::size_t>(A.col(i, s)));
          if (p == Precision::FP16) acc = fp16_fma_value(a, xv, acc, ctx.policy);
          else if (p == Precision::FP32)
            acc = ftz_fp32(std::fmaf(static_cast<float>(a), static_cast<float>(xv), static_cast<float>(acc)), true);
          else acc = std::fma(a, xv, acc);
        }
        e.set(i, acc, ctx.policy);
      }
      CHECK(values_equal(y, e));
    }
  }
  // axpy (test_kernels.cpp:147-172)
  for (Precision p : {Precision::FP16, Precision::FP32, Precision::FP64}) {
    const PVector x = random_vector(rng, 33, p), y = random_vector(rng, 33, p);
    CHECK(bits_equal(axpy(0.0, x, y, ctx), y));
    PVector neg(x.size(), p);
    axpy(-2.0, x, x, neg, ctx);
    const PVector z = axpy(1.0, x, neg, ctx);
    bool all0 = true;
    for (std::size_t i = 0; i < z.size(); ++i) all0 = all0 && z.get(i) == 0.0;
    CHECK(all0);
  }
  // vec_multiply (test_kernels.cpp:174-195)
  {
    const PVector h = PVector::from_values(std::vector<double>{300.0}, Precision::FP16);
    CHECK(std::isinf(vec_multiply(h, h, ctx).get(0)));
    ExecContext strict;
    strict.validate = true;
    CHECK_THROWS(vec_multiply(h, h, strict), ValidationError);
  }
  // fused update == unfused pair, bitwise (test_kernels.cpp:197-247)
  SplitMix64 r3(11);
  for (Precision cp : {Precision::FP16, Precision::FP32, Precision::FP64}) {
    for (int rep = 0; rep < 10; ++rep) {
      std::vector<std::vector<std::pair<std::int32_t, double>>> rows(4);
      for (int i = 0; i < 4; ++i) {
        if (i > 0) rows[i].emplace_back(i - 1, -1.0);
        rows[i].emplace_back(i, 2.0);
        if (i < 3) rows[i].emplace_back(i + 1, -1.0);
      }
      const EllMatrix A = EllMatrix::from_entries(4, 4, rows, Precision::FP64);
      const PVector c = random_vector(r3, 4, cp);
      const double alpha = 2.0 * r3.next_double();
      PVector r = random_vector(r3, 4, Precision::FP64), u = random_vector(r3, 4, Precision::FP64);
      PVector rr = r, uu = u;
      update_residuum_correction(r, u, A, c, alpha, ctx);
      const PVector wc = cast_vector(c, Precision::FP64, 1.0, ctx);
      axpy(alpha, wc, uu, uu, ctx);
      const PVector Ac = spmv(A, wc, ctx);
      axpy(-alpha, Ac, rr, rr, ctx);
      CHECK(bits_equal(r, rr));
      CHECK(bits_equal(u, uu));
    }
  }
  // cast_vector (test_kernels.cpp:249-289)
  {
    SplitMix64 r4(13);
    std::vector<double> tiny(50);
    for (auto& v : tiny) v = (2.0 * r4.next_double() - 1.0) * 1e-7;
    const PVector x = PVector::from_values(tiny, Precision::FP64);
    const double nrm = norm2_fp64(x, ctx);
    const PVector s = cast_vector(x, Precision::FP16, nrm, ctx);
    bool keep = true;
    for (std::size_t i = 0; i < s.size(); ++i)
      if (std::fabs(tiny[i]) >= kFp16MinNormal * nrm) keep = keep && s.get(i) != 0.0;
    CHECK(keep);
    const double sn = norm2_fp64(s, ctx);
    CHECK(sn >= 1.0 - 0x1p-9 && sn <= 1.0 + 0x1p-9);
    const PVector un = cast_vector(x, Precision::FP16, 1.0, ctx);
    bool zero = true;
    for (std::size_t i = 0; i < un.size(); ++i) zero = zero && un.get(i) == 0.0;
    CHECK(zero);
    CHECK_THROWS(cast_vector(x, Precision::FP16, 0.0, ctx), std::invalid_argument);
    CHECK_THROWS(cast_vector(x, Precision::FP16, -1.0, ctx), std::invalid_argument);
  }
  // usage errors (test_kernels.cpp:319-329)
  {
    std::vector<std::vector<std::pair<std::int32_t, double>>> rows(4);
    for (int i = 0; i < 4; ++i) rows[i].emplace_back(i, 2.0);
    const EllMatrix A = EllMatrix::from_entries(4, 4, rows, Precision::FP64);
    const PVector x3(3, Precision::FP64), x4h(4, Precision::FP16), a(4, Precision::FP64);
    CHECK_THROWS(spmv(A, x3, ctx), std::invalid_argument);
    CHECK_THROWS(spmv(A, x4h, ctx), std::invalid_argument);
    CHECK_THROWS(axpy(1.0, a, x3, ctx), std::invalid_argument);
    CHECK_THROWS(vec_multiply(a, x4h, ctx), std::invalid_argument);
    PVector y(4, Precision::FP64);
    CHECK_THROWS(spmv(A, y, y, ctx), std::invalid_argument);
  }
  // norm against a compensated sum (test_kernels.cpp:331-339)
  {
    SplitMix64 r5(23);
    const PVector x = random_vector(r5, 256, Precision::FP64);
    double s = 0.0, c = 0.0;
    for (std::size_t i = 0; i < x.size(); ++i) {
      const double v = x.get(i) * x.get(i), t = s + v;
      c += std::fabs(s) >= std::fabs(v) ? (s - t) + v : (v - t) + s;
      s = t;
    }
    const double ref = std::sqrt(s + c);
    CHECK(std::fabs(norm2_fp64(x, ctx) - ref) <= 1e-14 * ref);
  }
  // dump format (test_kernels.cpp:341-349)
  {
    const EllMatrix A = EllMatrix::from_dense({{1.5, 0.0}, {0.0, -2.0}}, Precision::FP32);
    std::ostringstream os;
    A.dump(os);
    CHECK(os.str().find("ellpack 2 2 1 fp32") == 0);
    CHECK(os.str().find("0:1.5") != std::string::npos);
    CHECK(os.str().find("1:-2") != std::string::npos);
  }
}

// end-to-end: BASELINE configs[0] and an H_MG solve, pinned to the
// reference's iteration counts (tests/golden/solves.npz)
static void solves() {
  {
    const ProblemSpec spec{3, 1, 65, 6};
    const Problem p = build_problem(spec);
    MgHierarchy h = MgHierarchy::build(spec, MgVariant::D_MG, SmootherConfig{2, 2, 2.0 / 3.0});
    IrConfig cfg;
    cfg.outer_tolerance = 1e-10 * norm2_fp64(p.b, {});
    ExecContext ctx;
    const IrResult r = ir_solve(p.A, p.b, h, cfg, ctx);
    CHECK(r.report.converged);
    CHECK(r.report.iterations == 9);
    CHECK(std::fabs(r.report.residual_history[0] - 2.043358e-02) < 1e-7);
    CHECK(r.report.final_residual < cfg.outer_tolerance);
    CHECK(r.report.residual_history.size() == static_cast<std::size_t>(r.report.iterations) + 1);
    CHECK(nodal_l2_error(r.u, p.u_exact, p.grid) < 1e-3);
    std::printf("cfg0 D_MG 65^3 V(2,2): %d its, final %.3e, device %.3f ms\n", r.report.iterations,
                r.report.final_residual, r.report.device_time_s * 1e3);
  }
  {
    const ProblemSpec spec{3, 1, 33, 5};
    const Problem p = build_problem(spec);
    ExecContext ctx;
    ctx.policy.flush_subnormals_to_zero = false;
    MgHierarchy h = MgHierarchy::build(spec, MgVariant::H_MG, {}, {}, ctx.policy);
    IrConfig cfg;
    cfg.outer_tolerance = 1e-10 * norm2_fp64(p.b, {});
    const IrResult fast = ir_solve(p.A, p.b, h, cfg, ctx);
    CHECK(fast.report.converged);
    CHECK(fast.report.iterations == 8);  // 3_33_h_mg_ftz0
    // the same system through the generic ELLPACK path: an untagged copy of A
    // and a hierarchy rebuilt from the level data (from_levels)
    std::vector<GridLevel> lv;
    for (int l = 0; l < h.levels(); ++l) lv.push_back(h.level(l));
    MgHierarchy g = MgHierarchy::from_levels(lv, h.smoother(), h.base_solver(), false);
    const EllMatrix A2 = p.A.cast_to(Precision::FP64);
    IrConfig cfg2 = cfg;
    cfg2.scaling = IrConfig::Scaling::ForceOn;  // from_levels leaves variant D_MG (multigrid.hpp:136)
    const IrResult gen = ir_solve(A2, p.b, g, cfg2, ctx);
    CHECK(gen.report.converged);
    CHECK(std::abs(gen.report.iterations - fast.report.iterations) <= 1);
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < gen.u.size(); ++i) {
      const double d = gen.u.get(i) - fast.u.get(i);
      num += d * d;
      den += fast.u.get(i) * fast.u.get(i);
    }
    CHECK(std::sqrt(num / den) <= 1e-9);
    // one V-cycle: fused stencil path == generic ELLPACK path (values)
    PVector rl = cast_vector(p.b, Precision::FP16, norm2_fp64(p.b, ctx), ctx);
    PVector c1(rl.size(), Precision::FP16), c2(rl.size(), Precision::FP16);
    h.v_cycle(rl, c1, ctx);
    g.v_cycle(rl, c2, ctx);
    CHECK(values_equal(c1, c2));
    std::printf("H_MG 33^3: fused %d its, generic %d its, rel diff %.2e\n", fast.report.iterations,
                gen.report.iterations, std::sqrt(num / den));
  }
  // validate mode (ExecContext::validate; kernels.cpp:96-113, multigrid.cpp:
  // 259-265, 365-369): the fused path hands over to the op-for-op path,
  // which checks every kernel output on the device
  {
    const ProblemSpec spec{3, 1, 33, 5};
    const Problem p = build_problem(spec);
    ExecContext ctx;
    ctx.policy.flush_subnormals_to_zero = false;
    MgHierarchy h = MgHierarchy::build(spec, MgVariant::H_MG, {}, {}, ctx.policy);
    IrConfig cfg;
    cfg.outer_tolerance = 1e-10 * norm2_fp64(p.b, {});
    const IrResult fast = ir_solve(p.A, p.b, h, cfg, ctx);
    ExecContext vctx = ctx;
    vctx.validate = true;
    const IrResult val = ir_solve(p.A, p.b, h, cfg, vctx);  // finite throughout: no throw
    CHECK(val.report.converged);
    CHECK(std::abs(val.report.iterations - fast.report.iterations) <= 1);
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < val.u.size(); ++i) {
      const double d = val.u.get(i) - fast.u.get(i);
      num += d * d;
      den += fast.u.get(i) * fast.u.get(i);
    }
    CHECK(std::sqrt(num / den) <= 1e-9);
    // a non-finite rhs entry: the first axpy (r = b - A u) reports it by index
    PVector bad = p.b;
    bad.set(123, std::numeric_limits<double>::infinity());
    bool thrown = false;
    try {
      ir_solve(p.A, bad, h, cfg, vctx);
    } catch (const ValidationError& e) {
      thrown = std::string(e.what()).find("index 123") != std::string::npos;
    }
    CHECK(thrown);
    // without validate the same input diverges (non-finite alpha, ir_solver.cpp:97-101)
    CHECK_THROWS(ir_solve(p.A, bad, h, cfg, ctx), DivergedError);
    // a V-cycle on a binary16 input holding an infinity
    PVector rl = cast_vector(p.b, Precision::FP16, norm2_fp64(p.b, ctx), ctx);
    rl.set(7, std::numeric_limits<double>::infinity());
    PVector c(rl.size(), Precision::FP16);
    CHECK_THROWS(h.v_cycle(rl, c, vctx), ValidationError);
    std::printf("validate mode: %d its (fused %d)\n", val.report.iterations, fast.report.iterations);
  }
  // errors: diverged / build / spec
  CHECK_THROWS((ProblemSpec{3, 1, 66, 6}.validate()), std::invalid_argument);
}

// host-only mode: dump the setup-side results for comparison with the
// reference's golden fixtures (no GPU needed)
template <typename T>
static void write(const std::string& path, const T* p, std::size_t n) {
  FILE* f = std::fopen(path.c_str(), "wb");
  std::fwrite(p, sizeof(T), n, f);
  std::fclose(f);
}
static void dump_ell(const std::string& stem, const EllMatrix& A) {
  std::vector<double> v(A.rows() * A.row_width());
  for (std::size_t r = 0; r < A.rows(); ++r)
    for (int s = 0; s < A.row_width(); ++s) v[r * A.row_width() + s] = A.value(r, s);
  write(stem + "_cols.bin", A.col_data().data(), A.col_data().size());
  write(stem + "_vals.bin", v.data(), v.size());
}
static int host_dump(const std::string& dir) {
  for (auto [dim, n] : {std::pair{2, 17}, std::pair{3, 9}}) {
    const StructuredGrid g{dim, n}, c{dim, (n + 1) / 2};
    dump_ell(dir + "/A_" + std::to_string(dim) + "_" + std::to_string(n), assemble_stiffness(g));
    auto [P, R] = assemble_transfer(g, c);
    dump_ell(dir + "/P_" + std::to_string(dim) + "_" + std::to_string(n), P);
    dump_ell(dir + "/R_" + std::to_string(dim) + "_" + std::to_string(n), R);
  }
  for (auto [dim, n] : {std::pair{2, 33}, std::pair{3, 17}}) {
    const StructuredGrid g{dim, n};
    const PVector b = assemble_rhs(g, 1), u = exact_solution(g, 1);
    write(dir + "/rhs_" + std::to_string(dim) + "_" + std::to_string(n) + ".bin", b.f64().data(), b.size());
    write(dir + "/exact_" + std::to_string(dim) + "_" + std::to_string(n) + ".bin", u.f64().data(), u.size());
  }
  SplitMix64 rng(7);
  std::vector<double> abc;
  for (int i = 0; i < 20000; ++i) {
    double t[3];
    for (double& x : t) {
      const unsigned bits = static_cast<unsigned>(rng.next_u64() & 0xFFFFu);
      x = ((bits >> 10) & 0x1Fu) == 0x1Fu ? 0.5 : widen(Fp16Value{static_cast<std::uint16_t>(bits)});
    }
    for (int ftz = 0; ftz < 2; ++ftz)
      for (int fma = 0; fma < 2; ++fma) {
        abc.insert(abc.end(), {t[0], t[1], t[2], double(ftz), double(fma),
                               fp16_fma_value(t[0], t[1], t[2], ArithmeticPolicy{ftz != 0, fma != 0})});
      }
  }
  write(dir + "/fp16_fma.bin", abc.data(), abc.size());
  std::printf("host dump ok\n");
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 2 && std::string(argv[1]) == "--host-dump") return host_dump(argv[2]);
  try {
    kernel_kats();
    solves();
  } catch (const std::exception& e) {
    std::printf("EXCEPTION %s\n", e.what());
    return 2;
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
