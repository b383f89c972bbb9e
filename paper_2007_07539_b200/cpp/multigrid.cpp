// Multigrid API (multigrid.hpp) of the drop-in layer.
//
//  * MgHierarchy::build: the reference's per-level host data (multigrid.cpp:
//    282-323) plus a device solver per arithmetic policy (mpmg_solver_*,
//    the fused sm_100a stencil V-cycle) used by v_cycle and ir_solve.
//  * Everything else (from_levels hierarchies, jacobi_smooth, cg_solve,
//    restrict_with_cast, prolong_with_cast) runs the generic device ELLPACK
//    kernels with device-resident operands, in the reference's operation
//    order (multigrid.cpp:79-393).
#include "mpmg/multigrid.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>
#include <string>
#include <utility>

#include "device.hpp"
#include "generic.hpp"
#include "mpmg/errors.hpp"

namespace mpmg {

using namespace detail;

namespace {

void require(bool cond, const char* msg) {
  if (!cond) throw std::invalid_argument(msg);
}

EllMatrix cast_checked(const EllMatrix& m, Precision target, const ArithmeticPolicy& policy, int level) {
  if (target == Precision::FP16 && m.max_abs_value() > kFp16Max)
    throw HierarchyBuildError(level, "binary16 overflow while casting level " + std::to_string(level) +
                                         " (max |entry| = " + std::to_string(m.max_abs_value()) + ")");
  return m.cast_to(target, policy);
}

}  // namespace

std::string_view variant_name(MgVariant v) {
  switch (v) {
    case MgVariant::D_MG: return "d_mg";
    case MgVariant::H_MG: return "h_mg";
    case MgVariant::DSH_MG: return "dsh_mg";
    default: return "hsd_mg";
  }
}

std::optional<MgVariant> parse_variant(std::string_view name) {
  for (MgVariant v : {MgVariant::D_MG, MgVariant::H_MG, MgVariant::DSH_MG, MgVariant::HSD_MG})
    if (name == variant_name(v)) return v;
  return std::nullopt;
}

VariantConfig VariantConfig::make(MgVariant v, int levels) {
  require(levels >= 1, "VariantConfig: level count must be positive");
  VariantConfig c;
  c.variant = v;
  c.level_precision.resize(static_cast<std::size_t>(levels));
  for (int l = 0; l < levels; ++l) {
    Precision p = Precision::FP64;
    if (v == MgVariant::H_MG) p = Precision::FP16;
    else if (v == MgVariant::HSD_MG) p = l <= 1 ? Precision::FP64 : (l == 2 ? Precision::FP32 : Precision::FP16);
    else if (v == MgVariant::DSH_MG) p = l <= 1 ? Precision::FP16 : (l == 2 ? Precision::FP32 : Precision::FP64);
    c.level_precision[static_cast<std::size_t>(l)] = p;
  }
  c.rescale_fp16_restrictions = v == MgVariant::DSH_MG;
  return c;
}

// ---- public level operations (device-resident inside each call) ---------

void jacobi_smooth(GridLevel& level, const PVector& b, PVector& u, int steps, double omega, const ExecContext& ctx) {
  require(steps >= 0, "jacobi_smooth: steps must be non-negative");
  require(omega > 0.0 && omega <= 1.0, "jacobi_smooth: omega must be in (0, 1]");
  if (steps == 0) return;
  DevVec db(b), du(u), dr(u.size(), u.precision()), dt(u.size(), u.precision()), dd(level.inv_diag);
  dev_jacobi(level.A, dd, db, du, dr, dt, steps, omega, ctx);
  du.to(u);
}

CgResult cg_solve(const EllMatrix& A, const PVector& b, PVector& u, const BaseSolverConfig& cfg,
                  const ExecContext& ctx) {
  require(A.rows() == A.cols(), "cg_solve: A must be square");
  require(A.precision() == b.precision(), "cg_solve: precision mismatch");
  require(b.size() == A.rows() && u.size() == A.rows(), "cg_solve: dimension mismatch");
  require(u.precision() == b.precision(), "cg_solve: precision mismatch");
  require(cfg.tolerance > 0.0, "cg_solve: tolerance must be positive");
  DevVec db(b), du(u.size(), u.precision());
  const CgResult r = dev_cg(A, db, du, cfg, ctx);
  du.to(u);
  return r;
}

double restrict_with_cast(const EllMatrix& R, const PVector& r_fine, Precision coarse_precision, bool rescale,
                          PVector& r_coarse, const ExecContext& ctx) {
  require(R.cols() == r_fine.size(), "restrict_with_cast: dimension mismatch");
  require(R.rows() == r_coarse.size(), "restrict_with_cast: output dimension mismatch");
  require(r_coarse.precision() == coarse_precision, "restrict_with_cast: output precision mismatch");
  DevVec df(r_fine), dc(r_coarse.size(), coarse_precision);
  const double s = dev_restrict(R, df, dc, rescale, ctx);
  dc.to(r_coarse);
  if (ctx.validate)
    for (std::size_t i = 0; i < r_coarse.size(); ++i)
      if (!std::isfinite(r_coarse.get(i)))
        throw ValidationError("restrict_with_cast: non-finite entry at index " + std::to_string(i));
  return s;
}

void prolong_with_cast(const EllMatrix& P, const PVector& c_coarse, Precision fine_precision, double scale,
                       PVector& c_fine, const ExecContext& ctx) {
  require(P.cols() == c_coarse.size(), "prolong_with_cast: dimension mismatch");
  require(P.rows() == c_fine.size(), "prolong_with_cast: output dimension mismatch");
  require(c_fine.precision() == fine_precision, "prolong_with_cast: output precision mismatch");
  require(scale > 0.0 && std::isfinite(scale), "prolong_with_cast: scale must be positive");
  DevVec dc(c_coarse), df(c_fine.size(), fine_precision);
  dev_prolong(P, dc, df, scale, ctx);
  df.to(c_fine);
}

// ---- hierarchy -------------------------------------------------------------

MgHierarchy MgHierarchy::build(const ProblemSpec& spec, MgVariant variant, const SmootherConfig& smoother,
                               const BaseSolverConfig& base, const ArithmeticPolicy& policy) {
  spec.validate();
  require(spec.levels >= 2, "MgHierarchy: at least two levels required");
  const VariantConfig vc = VariantConfig::make(variant, spec.levels);
  std::vector<GridLevel> levels(static_cast<std::size_t>(spec.levels));
  for (int l = 0; l < spec.levels; ++l) {
    GridLevel& g = levels[static_cast<std::size_t>(l)];
    g.precision = vc.level_precision[static_cast<std::size_t>(l)];
    const StructuredGrid grid{spec.dim, spec.nodes_at_level(l)};
    const EllMatrix A64 = assemble_stiffness(grid);
    // inverse of the assembled diagonal (multigrid.cpp:296-306), cast to the
    // level precision. Every row of the generated operator carries the same
    // diagonal coefficient, so it is read from one row (the slot whose column
    // is the row itself) and broadcast.
    std::vector<std::int32_t> cols(static_cast<std::size_t>(A64.row_width()));
    std::vector<double> vals(cols.size());
    A64.row(0, cols.data(), vals.data());
    double diag = 0.0;
    for (std::size_t s = 0; s < cols.size(); ++s)
      if (cols[s] == 0) { diag = vals[s]; break; }
    PVector d(A64.rows(), g.precision);
    d.set(0, 1.0 / diag, policy);
    if (g.precision == Precision::FP16) std::fill(d.f16().begin(), d.f16().end(), d.f16()[0]);
    else if (g.precision == Precision::FP32) std::fill(d.f32().begin(), d.f32().end(), d.f32()[0]);
    else std::fill(d.f64().begin(), d.f64().end(), d.f64()[0]);
    g.A = cast_checked(A64, g.precision, policy, l);
    g.inv_diag = std::move(d);
    if (l < spec.levels - 1) {
      auto [P, R] = assemble_transfer(StructuredGrid{spec.dim, spec.nodes_at_level(l + 1)}, grid);
      g.prolong_to_finer = cast_checked(P, g.precision, policy, l);
      g.restrict_from_finer = cast_checked(R, g.precision, policy, l);
      g.has_finer = true;
    }
  }
  MgHierarchy h = from_levels(std::move(levels), smoother, base, vc.rescale_fp16_restrictions);
  h.variant_ = variant;
  h.spec_ = spec;
  auto sv = std::make_shared<DeviceSolvers>();
  mpmg_solver_default_config(&sv->base);
  sv->base.dim = spec.dim;
  sv->base.k = spec.k;
  sv->base.nodes = spec.finest_nodes_per_dim;
  sv->base.levels = spec.levels;
  sv->base.variant = static_cast<int>(variant);
  sv->base.pre_steps = smoother.pre_steps;
  sv->base.post_steps = smoother.post_steps;
  sv->base.omega = smoother.omega;
  sv->base.base_tol = base.tolerance;
  sv->base.base_mode = base.mode == BaseSolverConfig::ToleranceMode::Absolute ? 1 : 0;
  sv->base.base_max_iterations = base.max_iterations;
  h.solvers_ = sv;
  return h;
}

MgHierarchy MgHierarchy::from_levels(std::vector<GridLevel> levels, const SmootherConfig& smoother,
                                     const BaseSolverConfig& base, bool rescale_fp16_restrictions) {
  require(!levels.empty(), "MgHierarchy: empty level list");
  MgHierarchy h;
  h.levels_ = std::move(levels);
  h.smoother_ = smoother;
  h.base_ = base;
  h.rescale_fp16_restrictions_ = rescale_fp16_restrictions;
  for (auto& g : h.levels_) {
    const std::size_t n = g.A.rows();
    g.u = PVector(n, g.precision);
    g.b = PVector(n, g.precision);
    g.r = PVector(n, g.precision);
    g.t = PVector(n, g.precision);
  }
  h.level_traffic_.assign(h.levels_.size(), TrafficCounter{});
  return h;
}

void MgHierarchy::reset_traffic() {
  for (auto& t : level_traffic_) t.reset();
}

TrafficCounter MgHierarchy::cycle_traffic() const {
  TrafficCounter t;
  for (const auto& l : level_traffic_) t += l;
  return t;
}

mpmg_solver* DeviceSolvers::get(uint32_t policy) {
  for (auto& e : items)
    if (e.policy == policy) return e.s;
  require_device();
  mpmg_solver_config c = base;
  c.policy = policy;
  int err = 0, lvl = -1;
  mpmg_solver* s = mpmg_solver_create(&c, &err, &lvl);
  if (!s) {
    if (err == MPMG_EBUILD) throw HierarchyBuildError(lvl, "binary16 overflow while casting level " + std::to_string(lvl));
    raise(err ? err : MPMG_ECUDA, "mpmg_solver_create");
  }
  items.push_back({policy, s});
  return s;
}

void* MgHierarchy::device_solver(const ExecContext& ctx) {
  if (!solvers_) return nullptr;
  return solvers_->get(policy_word(ctx));
}

void MgHierarchy::v_cycle(const PVector& b, PVector& c, const ExecContext& ctx) {
  require(b.precision() == finest_precision(), "v_cycle: rhs precision mismatch");
  require(c.precision() == finest_precision(), "v_cycle: output precision mismatch");
  require(b.size() == levels_.back().unknowns(), "v_cycle: dimension mismatch");
  require(c.size() == levels_.back().unknowns(), "v_cycle: output dimension mismatch");
  if (solvers_ && !ctx.validate) {
    // the fused stencil V-cycle on the device: the vectors move in their
    // storage precision (compact -> padded on the device, no host value
    // loop); validate mode runs op for op (every kernel's output checked)
    auto* s = static_cast<mpmg_solver*>(device_solver(ctx));
    const int dim = spec_->dim, nodes = spec_->finest_nodes_per_dim, pc = prec_code(b.precision());
    const std::size_t plen = mpmg_padded_len(dim, nodes), vb = static_cast<std::size_t>(bytes_per_value(b.precision()));
    DevVec db(b), dc(c.size(), c.precision());
    DevBuf pb(plen * vb), pcv(plen * vb);
    check(mpmg_dev_memset0(pb.get(), plen * vb), "v_cycle");
    check(mpmg_gpu_pack(dim, nodes, pc, db.get(), pb.get(), nullptr), "v_cycle pack");
    check(mpmg_dev_sync(), "v_cycle");
    check(mpmg_solver_v_cycle_device(s, pb.get(), pcv.get(), mpmg_solver_stream(s)), "v_cycle");
    check(mpmg_dev_sync(), "v_cycle");
    check(mpmg_gpu_unpack(dim, nodes, pc, pcv.get(), dc.get(), nullptr), "v_cycle unpack");
    check(mpmg_dev_sync(), "v_cycle");
    dc.to(c);
    add_cycle_traffic(*this, level_traffic_, ctx);
    return;
  }
  DevVec db(b), dc(c.size(), c.precision());
  DevHierarchy dh(*this);
  dh.cycle(levels() - 1, db, dc, ctx, level_traffic_);
  dc.to(c);
}

void MgHierarchy::cycle_at(int l, const PVector& rhs, PVector& u, const ExecContext& ctx) {
  DevVec db(rhs), du(u.size(), u.precision());
  DevHierarchy dh(*this);
  dh.cycle(l, db, du, ctx, level_traffic_);
  du.to(u);
}

}  // namespace mpmg
