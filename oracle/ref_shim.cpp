// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (arxiv 2007.07539's
// `mpmg`, compiled from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libmpmg_ref.so). It only calls the reference's public C++ API
// (core/include/mpmg/*.hpp) so Python tests, the golden-fixture script and
// `bench.py --impl reference` can drive the real reference:
//   * hierarchy / level data   -> MgHierarchy::build  (multigrid.cpp:282-323)
//   * per-kernel goldens       -> kernels.hpp:11-38, multigrid.hpp:73-94
//   * full solves              -> ir_solve            (ir_solver.cpp:51-127)
// Vectors cross the boundary as binary64 "value domain" arrays (every stored
// binary16/binary32 value is exactly representable in binary64).

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "mpmg/ell_matrix.hpp"
#include "mpmg/errors.hpp"
#include "mpmg/ir_solver.hpp"
#include "mpmg/kernels.hpp"
#include "mpmg/mesh_fem.hpp"
#include "mpmg/multigrid.hpp"
#include "mpmg/precision.hpp"

using namespace mpmg;

namespace {

Precision prec_of(int p) { return p == 0 ? Precision::FP16 : (p == 1 ? Precision::FP32 : Precision::FP64); }
int prec_code(Precision p) { return static_cast<int>(p); }

ExecContext make_ctx(int ftz, int fma, int acc32) {
  ExecContext c;
  c.policy.flush_subnormals_to_zero = ftz != 0;
  c.policy.fused_multiply_add = fma != 0;
  c.fp16_accumulation = acc32 ? Fp16Accum::FP32 : Fp16Accum::FP16;
  return c;
}

PVector vec_from(const double* xs, std::size_t n, int prec, const ArithmeticPolicy& pol) {
  PVector v(n, prec_of(prec));
  for (std::size_t i = 0; i < n; ++i) v.set(i, xs[i], pol);
  return v;
}

void vec_to(const PVector& v, double* out) {
  for (std::size_t i = 0; i < v.size(); ++i) out[i] = v.get(i);
}

struct Handle {
  ProblemSpec spec;
  MgHierarchy h;
  ArithmeticPolicy policy;
  double build_s = 0.0;
};

EllMatrix ell_from(std::int64_t rows, std::int64_t cols, int rw, const std::int32_t* c, const double* v,
                   int prec, const ArithmeticPolicy& pol) {
  EllMatrix m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols), rw, prec_of(prec));
  for (std::int64_t r = 0; r < rows; ++r)
    for (int s = 0; s < rw; ++s) m.set_slot(r, s, c[r * rw + s], v[r * rw + s], pol);
  return m;
}

const EllMatrix& level_matrix(const GridLevel& g, int which) {
  return which == 0 ? g.A : (which == 1 ? g.prolong_to_finer : g.restrict_from_finer);
}

}  // namespace

extern "C" {

// ---- precision primitives (precision.cpp) ---------------------------------
double ref_quantize_fp16(double x, int ftz) { return quantize_fp16(x, ftz != 0); }
double ref_fp16_fma(double a, double b, double c, int ftz, int fma) {
  return fp16_fma_value(a, b, c, ArithmeticPolicy{ftz != 0, fma != 0});
}
double ref_fp16_add(double a, double b, int ftz) { return fp16_add_value(a, b, ftz != 0); }
double ref_fp16_mul(double a, double b, int ftz) { return fp16_mul_value(a, b, ftz != 0); }
unsigned ref_round_to_fp16_bits(double x, int ftz) {
  return round_to_fp16(x, ArithmeticPolicy{ftz != 0, true}).bits;
}
double ref_widen_bits(unsigned bits) { return widen(Fp16Value{static_cast<std::uint16_t>(bits)}); }

// ---- problem (mesh_fem.cpp) -------------------------------------------------
std::int64_t ref_unknowns(int dim, int n) { return static_cast<std::int64_t>(StructuredGrid{dim, n}.unknowns()); }

int ref_problem_rhs(int dim, int k, int n, double* b, double* u_exact) {
  try {
    const StructuredGrid g{dim, n};
    if (b) vec_to(assemble_rhs(g, k), b);
    if (u_exact) vec_to(exact_solution(g, k), u_exact);
    return 0;
  } catch (...) { return -1; }
}

// Assembled FP64 stiffness of one grid: row width and, optionally, the ELL
// arrays (mesh_fem.cpp:71-155).
int ref_stiffness(int dim, int n, std::int32_t* cols, double* vals) {
  try {
    const EllMatrix A = assemble_stiffness(StructuredGrid{dim, n});
    const auto c = A.col_data();
    const auto v = A.f64();
    if (cols) std::memcpy(cols, c.data(), c.size() * sizeof(std::int32_t));
    if (vals) std::memcpy(vals, v.data(), v.size() * sizeof(double));
    return A.row_width();
  } catch (...) { return -1; }
}

// One interior row's 3^dim stencil (lexicographic dz,dy,dx) of the assembled
// FP64 stiffness: read from the row of the grid's centre node.
int ref_stencil(int dim, int n, double* taps) {
  try {
    const StructuredGrid g{dim, n};
    const EllMatrix A = assemble_stiffness(g);
    const int c = (n - 1) / 2;
    const std::size_t row = g.interior_index(c, c, c);
    for (int s = 0; s < A.row_width(); ++s) taps[s] = A.value(row, s);
    return A.row_width();
  } catch (...) { return -1; }
}

// ---- hierarchy (multigrid.cpp:282-342) -------------------------------------
void* ref_hier_build(int dim, int k, int n, int levels, int variant, int pre, int post, double omega,
                     double base_tol, int base_mode, int base_maxit, int ftz, int fma) {
  try {
    auto* hd = new Handle{};
    hd->spec = ProblemSpec{dim, k, n, levels};
    hd->policy = ArithmeticPolicy{ftz != 0, fma != 0};
    BaseSolverConfig base;
    base.tolerance = base_tol;
    base.max_iterations = base_maxit;
    base.mode = base_mode ? BaseSolverConfig::ToleranceMode::Absolute
                          : BaseSolverConfig::ToleranceMode::RelativeToRhs;
    const auto t0 = std::chrono::steady_clock::now();
    hd->h = MgHierarchy::build(hd->spec, static_cast<MgVariant>(variant), SmootherConfig{pre, post, omega},
                               base, hd->policy);
    hd->build_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return hd;
  } catch (const HierarchyBuildError& e) {
    return nullptr;
  } catch (...) { return nullptr; }
}

void ref_hier_free(void* h) { delete static_cast<Handle*>(h); }
double ref_hier_build_seconds(void* h) { return static_cast<Handle*>(h)->build_s; }
int ref_hier_levels(void* h) { return static_cast<Handle*>(h)->h.levels(); }
int ref_level_prec(void* h, int l) { return prec_code(static_cast<Handle*>(h)->h.level(l).precision); }
std::int64_t ref_level_rows(void* h, int l) { return static_cast<std::int64_t>(static_cast<Handle*>(h)->h.level(l).A.rows()); }

// which: 0 = A, 1 = prolong_to_finer, 2 = restrict_from_finer
int ref_level_matrix_shape(void* h, int l, int which, std::int64_t* rows, std::int64_t* cols) {
  const GridLevel& g = static_cast<Handle*>(h)->h.level(l);
  if (which != 0 && !g.has_finer) return -1;
  const EllMatrix& m = level_matrix(g, which);
  *rows = static_cast<std::int64_t>(m.rows());
  *cols = static_cast<std::int64_t>(m.cols());
  return m.row_width();
}

int ref_level_matrix(void* h, int l, int which, std::int32_t* cols, double* vals) {
  const GridLevel& g = static_cast<Handle*>(h)->h.level(l);
  if (which != 0 && !g.has_finer) return -1;
  const EllMatrix& m = level_matrix(g, which);
  for (std::size_t r = 0; r < m.rows(); ++r)
    for (int s = 0; s < m.row_width(); ++s) {
      cols[r * m.row_width() + s] = m.col(r, s);
      vals[r * m.row_width() + s] = m.value(r, s);
    }
  return 0;
}

int ref_level_invdiag(void* h, int l, double* out) {
  vec_to(static_cast<Handle*>(h)->h.level(l).inv_diag, out);
  return 0;
}

// ---- per-kernel goldens on a level of a built hierarchy ---------------------
int ref_level_spmv(void* hp, int l, const double* x, double* y, int ftz, int fma, int acc32) {
  try {
    auto* hd = static_cast<Handle*>(hp);
    GridLevel& g = hd->h.level(l);
    const ExecContext ctx = make_ctx(ftz, fma, acc32);
    const int p = prec_code(g.precision);
    const PVector xv = vec_from(x, g.unknowns(), p, ctx.policy);
    PVector yv(g.unknowns(), g.precision);
    spmv(g.A, xv, yv, ctx);
    vec_to(yv, y);
    return 0;
  } catch (...) { return -1; }
}

int ref_level_jacobi(void* hp, int l, const double* b, double* u, int steps, double omega, int ftz, int fma,
                     int acc32) {
  try {
    auto* hd = static_cast<Handle*>(hp);
    GridLevel& g = hd->h.level(l);
    const ExecContext ctx = make_ctx(ftz, fma, acc32);
    const int p = prec_code(g.precision);
    const PVector bv = vec_from(b, g.unknowns(), p, ctx.policy);
    PVector uv = vec_from(u, g.unknowns(), p, ctx.policy);
    jacobi_smooth(g, bv, uv, steps, omega, ctx);
    vec_to(uv, u);
    return 0;
  } catch (...) { return -1; }
}

// level defect r = b - A u in the level precision (multigrid.cpp:379-380)
int ref_level_defect(void* hp, int l, const double* b, const double* u, double* r, int ftz, int fma, int acc32) {
  try {
    auto* hd = static_cast<Handle*>(hp);
    GridLevel& g = hd->h.level(l);
    const ExecContext ctx = make_ctx(ftz, fma, acc32);
    const int p = prec_code(g.precision);
    const PVector bv = vec_from(b, g.unknowns(), p, ctx.policy);
    const PVector uv = vec_from(u, g.unknowns(), p, ctx.policy);
    PVector t(g.unknowns(), g.precision), rv(g.unknowns(), g.precision);
    spmv(g.A, uv, t, ctx);
    axpy(-1.0, t, bv, rv, ctx);
    vec_to(rv, r);
    return 0;
  } catch (...) { return -1; }
}

// restrict from level l (fine) into level l-1 (coarse); returns the scale
double ref_level_restrict(void* hp, int l, const double* r_fine, int rescale, double* r_coarse, int ftz, int fma) {
  auto* hd = static_cast<Handle*>(hp);
  GridLevel& f = hd->h.level(l);
  GridLevel& c = hd->h.level(l - 1);
  const ExecContext ctx = make_ctx(ftz, fma, 0);
  const PVector rf = vec_from(r_fine, f.unknowns(), prec_code(f.precision), ctx.policy);
  PVector rc(c.unknowns(), c.precision);
  const double s = restrict_with_cast(c.restrict_from_finer, rf, c.precision, rescale != 0, rc, ctx);
  vec_to(rc, r_coarse);
  return s;
}

// prolong from level l-1 (coarse) to level l (fine): c_fine = cast(scale * P c)
int ref_level_prolong(void* hp, int l, const double* c_coarse, double scale, double* c_fine, int ftz, int fma) {
  try {
    auto* hd = static_cast<Handle*>(hp);
    GridLevel& f = hd->h.level(l);
    GridLevel& c = hd->h.level(l - 1);
    const ExecContext ctx = make_ctx(ftz, fma, 0);
    const PVector cc = vec_from(c_coarse, c.unknowns(), prec_code(c.precision), ctx.policy);
    PVector cf(f.unknowns(), f.precision);
    prolong_with_cast(c.prolong_to_finer, cc, f.precision, scale, cf, ctx);
    vec_to(cf, c_fine);
    return 0;
  } catch (...) { return -1; }
}

int ref_level_cg(void* hp, int l, const double* b, double* u, int* iters, int* converged, double* res, int ftz,
                 int fma) {
  try {
    auto* hd = static_cast<Handle*>(hp);
    GridLevel& g = hd->h.level(l);
    const ExecContext ctx = make_ctx(ftz, fma, 0);
    const PVector bv = vec_from(b, g.unknowns(), prec_code(g.precision), ctx.policy);
    PVector uv(g.unknowns(), g.precision);
    const CgResult r = cg_solve(g.A, bv, uv, hd->h.base_solver(), ctx);
    vec_to(uv, u);
    *iters = r.iterations;
    *converged = r.converged;
    *res = r.final_residual;
    return 0;
  } catch (...) { return -1; }
}

int ref_v_cycle(void* hp, const double* b, double* c, int ftz, int fma, int acc32) {
  try {
    auto* hd = static_cast<Handle*>(hp);
    const ExecContext ctx = make_ctx(ftz, fma, acc32);
    const int L = hd->h.levels();
    const std::size_t n = hd->h.level(L - 1).unknowns();
    const int p = prec_code(hd->h.finest_precision());
    const PVector bv = vec_from(b, n, p, ctx.policy);
    PVector cv(n, hd->h.finest_precision());
    hd->h.v_cycle(bv, cv, ctx);
    vec_to(cv, c);
    return 0;
  } catch (...) { return -1; }
}

// ---- outer FP64 kernels on the finest assembled operator -------------------
// update_residuum_correction (kernels.cpp:300-341) with A = assembled FP64
// stiffness of (dim, n); c given in precision c_prec.
int ref_update_rc(int dim, int n, double* r, double* u, const double* c, int c_prec, double alpha, int ftz, int fma) {
  try {
    const EllMatrix A = assemble_stiffness(StructuredGrid{dim, n});
    const ExecContext ctx = make_ctx(ftz, fma, 0);
    const std::size_t N = A.rows();
    PVector rv = vec_from(r, N, 2, ctx.policy), uv = vec_from(u, N, 2, ctx.policy);
    const PVector cv = vec_from(c, N, c_prec, ctx.policy);
    update_residuum_correction(rv, uv, A, cv, alpha, ctx);
    vec_to(rv, r);
    vec_to(uv, u);
    return 0;
  } catch (...) { return -1; }
}

// outer defect r = b - A u (ir_solver.cpp:92-93): spmv + axpy(-1)
int ref_defect64(int dim, int n, const double* b, const double* u, double* r) {
  try {
    const EllMatrix A = assemble_stiffness(StructuredGrid{dim, n});
    ExecContext ctx;
    const std::size_t N = A.rows();
    const PVector bv = vec_from(b, N, 2, ctx.policy), uv = vec_from(u, N, 2, ctx.policy);
    PVector t(N, Precision::FP64), rv(N, Precision::FP64);
    spmv(A, uv, t, ctx);
    axpy(-1.0, t, bv, rv, ctx);
    vec_to(rv, r);
    return 0;
  } catch (...) { return -1; }
}

int ref_cast(const double* x, std::int64_t n, int src_prec, int dst_prec, double scale, double* out, int ftz) {
  try {
    ExecContext ctx = make_ctx(ftz, 1, 0);
    const PVector xv = vec_from(x, static_cast<std::size_t>(n), src_prec, ctx.policy);
    PVector o(static_cast<std::size_t>(n), prec_of(dst_prec));
    cast_vector(xv, prec_of(dst_prec), scale, o, ctx);
    vec_to(o, out);
    return 0;
  } catch (...) { return -1; }
}

double ref_norm2(const double* x, std::int64_t n, int prec) {
  ExecContext ctx;
  const PVector xv = vec_from(x, static_cast<std::size_t>(n), prec, ArithmeticPolicy{false, true});
  return norm2_fp64(xv, ctx);
}

// generic ELL spmv (kernels.cpp:137-193) on caller-provided ELL arrays
int ref_ell_spmv(std::int64_t rows, std::int64_t cols, int rw, const std::int32_t* c, const double* v, int prec,
                 const double* x, double* y, int ftz, int fma, int acc32) {
  try {
    const ExecContext ctx = make_ctx(ftz, fma, acc32);
    const EllMatrix A = ell_from(rows, cols, rw, c, v, prec, ctx.policy);
    const PVector xv = vec_from(x, static_cast<std::size_t>(cols), prec, ctx.policy);
    PVector yv(static_cast<std::size_t>(rows), prec_of(prec));
    spmv(A, xv, yv, ctx);
    vec_to(yv, y);
    return 0;
  } catch (...) { return -1; }
}

// ---- full solve (ir_solver.cpp:51-127) -------------------------------------
// rel_tol > 0: tolerance = rel_tol * ||b|| (BASELINE metric); else abs_tol.
// Returns iterations, or -1 on error, -2 on DivergedError.
int ref_ir_solve(void* hp, double rel_tol, double abs_tol, int max_it, int random_guess, std::uint64_t seed,
                 int scaling, int refresh, int ftz, int fma, int acc32, double* u_out, double* hist, int hist_cap,
                 int* converged, double* final_res, double* wall_s, double* err_l2) {
  try {
    auto* hd = static_cast<Handle*>(hp);
    const ExecContext ctx = make_ctx(ftz, fma, acc32);
    const Problem p = build_problem(hd->spec);
    IrConfig cfg;
    cfg.outer_tolerance = rel_tol > 0 ? rel_tol * norm2_fp64(p.b, ExecContext{}) : abs_tol;
    cfg.max_outer_iterations = max_it;
    cfg.initial_guess = random_guess ? IrConfig::InitialGuess::SeededRandom01 : IrConfig::InitialGuess::Zeros;
    cfg.seed = seed;
    cfg.scaling = static_cast<IrConfig::Scaling>(scaling);
    cfg.residual_refresh_interval = refresh;
    const IrResult res = ir_solve(p.A, p.b, hd->h, cfg, ctx);
    if (u_out) vec_to(res.u, u_out);
    const auto& h = res.report.residual_history;
    for (int i = 0; i < hist_cap && i < static_cast<int>(h.size()); ++i) hist[i] = h[static_cast<std::size_t>(i)];
    *converged = res.report.converged;
    *final_res = res.report.final_residual;
    *wall_s = res.report.wall_time_s;
    if (err_l2) *err_l2 = nodal_l2_error(res.u, p.u_exact, p.grid);
    return res.report.iterations;
  } catch (const DivergedError& e) {
    return -2;
  } catch (...) { return -1; }
}

}  // extern "C"
