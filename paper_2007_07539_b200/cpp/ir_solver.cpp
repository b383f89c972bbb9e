// Iterative refinement (ir_solver.hpp), ir_solver.cpp:21-127 semantics.
//
// Fast path: a build() hierarchy solving its own assembled operator (the
// EllMatrix carries the stencil tag of assemble_stiffness) runs the whole
// solve on the device -- one CUDA graph with a device-side WHILE loop
// (mpmg_solver_solve). Otherwise: the same loop with generic device ELLPACK
// kernels, host-orchestrated, sequential-order norms (bitwise the reference).
#include "mpmg/ir_solver.hpp"

#include <chrono>
#include <cmath>
#include <stdexcept>
#include <string>

#include "device.hpp"
#include "generic.hpp"
#include "mpmg/errors.hpp"
#include "mpmg/rng.hpp"

namespace mpmg {

using namespace detail;

namespace {

void require(bool cond, const char* msg) {
  if (!cond) throw std::invalid_argument(msg);
}

bool scale_on(const IrConfig& c, const MgHierarchy& h) {
  if (c.scaling == IrConfig::Scaling::ForceOn) return true;
  if (c.scaling == IrConfig::Scaling::ForceOff) return false;
  return h.variant() != MgVariant::D_MG;  // ir_solver.cpp:70-76
}

// ||b - A u||: fma row sums, b - s, sequential fma of squares (ir_solver.cpp:21-49)
double dev_residual_norm(const EllMatrix& A, const DevVec& u, const DevVec& b) {
  DevVec s(A.rows(), Precision::FP64), r(A.rows(), Precision::FP64);
  ExecContext fused;
  fused.policy.fused_multiply_add = true;
  dev_spmv(A, u, s, fused);
  dev_axpy(-1.0, s, b, r, fused);  // fma(-1, s, b) == b - s, one rounding
  return dev_norm(r, fused);
}

}  // namespace

double residual_norm(const EllMatrix& A, const PVector& u, const PVector& b, const ExecContext& ctx) {
  require(A.precision() == Precision::FP64 && u.precision() == Precision::FP64 && b.precision() == Precision::FP64,
          "residual_norm: binary64 operands required");
  require(A.rows() == A.cols() && u.size() == A.rows() && b.size() == A.rows(), "residual_norm: dimension mismatch");
  DevVec du(u), db(b);
  const double v = dev_residual_norm(A, du, db);
  const std::uint64_t n = A.rows(), slots = n * static_cast<std::uint64_t>(A.row_width());
  add(ctx.traffic, slots * 16 + n * 8, 0, slots * 4, 2 * slots + 3 * n + 1);
  return v;
}

IrResult ir_solve(const EllMatrix& A_high, const PVector& b_high, MgHierarchy& h, const IrConfig& config,
                  const ExecContext& caller_ctx) {
  require(A_high.precision() == Precision::FP64 && b_high.precision() == Precision::FP64,
          "ir_solve: the outer system must be binary64");
  require(A_high.rows() == A_high.cols() && b_high.size() == A_high.rows(), "ir_solve: dimension mismatch");
  require(A_high.rows() == h.level(h.levels() - 1).unknowns(), "ir_solve: hierarchy does not match the system size");
  require(config.outer_tolerance > 0.0, "ir_solve: tolerance must be positive");
  const auto t0 = std::chrono::steady_clock::now();
  IrResult result;
  SolveReport& rep = result.report;
  const ExecContext ctx = caller_ctx.with_counter(&rep.outer_traffic);
  h.reset_traffic();
  const std::size_t n = A_high.rows();
  result.u = PVector(n, Precision::FP64);
  const bool scale_enabled = scale_on(config, h);

  const auto& tag = A_high.stencil_tag();
  // validate mode checks every kernel's output (kernels.cpp:96-113): it runs
  // op for op on the generic device path, which checks each result
  const bool fast = !caller_ctx.validate && h.spec() && tag.dim == h.spec()->dim &&
                    tag.nodes == h.spec()->finest_nodes_per_dim;
  if (fast) {
    auto* s = static_cast<mpmg_solver*>(h.device_solver(caller_ctx));
    mpmg_solve_params p{};
    mpmg_solve_default_params(&p);
    p.outer_tolerance = config.outer_tolerance;
    p.max_outer_iterations = config.max_outer_iterations;
    p.random_initial_guess = config.initial_guess == IrConfig::InitialGuess::SeededRandom01;
    p.seed = config.seed;
    p.scaling = static_cast<int>(config.scaling);
    p.residual_refresh_interval = config.residual_refresh_interval;
    std::vector<double> hist(static_cast<std::size_t>(config.max_outer_iterations) + 2);
    mpmg_solve_report r{};
    const int code = mpmg_solver_solve(s, b_high.f64().data(), result.u.f64().data(), &p, hist.data(),
                                       static_cast<int32_t>(hist.size()), &r);
    if (code == MPMG_ENONFINITE)
      throw DivergedError(r.iterations, "ir_solve: non-finite residual norm at iteration " + std::to_string(r.iterations));
    check(code, "ir_solve");
    rep.converged = r.converged;
    rep.iterations = r.iterations;
    rep.residual_history.assign(hist.begin(), hist.begin() + r.iterations + 1);
    rep.final_residual = r.final_residual;
    rep.device_time_s = r.device_seconds;
    // traffic model of the same loop (ir_solver.cpp accounting)
    const std::uint64_t slots = n * static_cast<std::uint64_t>(A_high.row_width());
    const std::uint64_t lp = static_cast<std::uint64_t>(bytes_per_value(h.finest_precision()));
    const int its = r.iterations, refresh = config.residual_refresh_interval > 0 ? its / config.residual_refresh_interval : 0;
    add(ctx.traffic, (1 + refresh) * (slots * 16 + 2 * n * 8), (1 + refresh) * 2 * n * 8, (1 + refresh) * slots * 4,
        (1 + refresh) * (2 * slots + 2 * n));
    add(ctx.traffic, (its + 1) * n * 8, 0, 0, (its + 1) * (2 * n + 1));                       // norms
    add(ctx.traffic, its * n * 8, its * n * lp, 0, its * n);                                   // casts
    add(ctx.traffic, its * (slots * 8 + 2 * n * 8 + n * lp), its * 2 * n * 8, its * slots * 4,
        its * (2 * slots + 4 * n));                                                            // updates
    add(ctx.traffic, slots * 16 + n * 8, 0, slots * 4, 2 * slots + 3 * n + 1);                 // residual_norm
    std::vector<TrafficCounter> lt(static_cast<std::size_t>(h.levels()));
    ExecContext dummy;
    for (int i = 0; i < its; ++i) add_cycle_traffic(h, lt, dummy);
    rep.level_traffic = lt;
    rep.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return result;
  }

  // generic device loop (ir_solver.cpp:78-125)
  require_device();
  const Precision mg = h.finest_precision();
  if (config.initial_guess == IrConfig::InitialGuess::SeededRandom01) {
    SplitMix64 rng(config.seed);
    auto ud = result.u.f64();
    for (std::size_t i = 0; i < n; ++i) ud[i] = rng.next_double();
  }
  DevVec u(result.u), b(b_high), r(n, Precision::FP64), t(n, Precision::FP64), rl(n, mg), cl(n, mg);
  DevHierarchy dh(h);
  std::vector<TrafficCounter> lt(static_cast<std::size_t>(h.levels()));
  dev_spmv(A_high, u, t, ctx);
  dev_axpy(-1.0, t, b, r, ctx);
  DevBuf al(8);
  const DeviceEll& DA = A_high.device();
  while (true) {
    const double alpha = dev_norm(r, ctx);
    rep.residual_history.push_back(alpha);
    if (!std::isfinite(alpha))
      throw DivergedError(rep.iterations, "ir_solve: non-finite residual norm at iteration " + std::to_string(rep.iterations));
    if (alpha < config.outer_tolerance) {
      rep.converged = true;
      break;
    }
    if (rep.iterations >= config.max_outer_iterations) break;
    const double scale = scale_enabled && alpha > 0.0 ? alpha : 1.0;
    check(mpmg_gpu_cast(static_cast<int64_t>(n), r.get(), MPMG_FP64, rl.get(), prec_code(mg), nullptr, scale,
                        policy_word(ctx), nullptr),
          "cast_vector");
    add(ctx.traffic, n * 8, n * static_cast<std::uint64_t>(bytes_per_value(mg)), 0, n);
    dh.cycle(h.levels() - 1, rl, cl, caller_ctx, lt);
    al.upload(&scale, 8);
    check(mpmg_gpu_ell_update_rc(DA.rows, DA.rw, DA.col.as<int32_t>(), DA.val.as<double>(), cl.get(), prec_code(mg),
                                 static_cast<double*>(r.get()), static_cast<double*>(u.get()), al.as<double>(),
                                 policy_word(ctx), nullptr),
          "update_residuum_correction");
    if (ctx.validate) {  // kernels.cpp:337-340
      dev_validate(r, "update_residuum_correction");
      dev_validate(u, "update_residuum_correction");
    }
    const std::uint64_t slots = n * static_cast<std::uint64_t>(A_high.row_width());
    add(ctx.traffic, slots * 8 + 2 * n * 8 + n * static_cast<std::uint64_t>(bytes_per_value(mg)), 2 * n * 8, slots * 4,
        2 * slots + 4 * n);
    ++rep.iterations;
    if (config.residual_refresh_interval > 0 && rep.iterations % config.residual_refresh_interval == 0) {
      dev_spmv(A_high, u, t, ctx);
      dev_axpy(-1.0, t, b, r, ctx);
    }
  }
  rep.final_residual = dev_residual_norm(A_high, u, b);
  u.to(result.u);
  rep.level_traffic = lt;
  rep.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return result;
}

}  // namespace mpmg
