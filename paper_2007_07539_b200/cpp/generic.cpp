// Device-resident generic ELLPACK multigrid (generic.hpp).
#include "generic.hpp"

#include <cmath>
#include <stdexcept>
#include <string>

#include "mpmg/errors.hpp"

namespace mpmg::detail {

namespace {
std::uint64_t vb(Precision p) { return static_cast<std::uint64_t>(bytes_per_value(p)); }
}  // namespace

// validate mode: the reference's validate_finite (kernels.cpp:90-113) on a
// device vector -- the first non-finite index, found on the device
void dev_validate(const DevVec& v, const char* what) {
  int64_t idx = -1;
  check(mpmg_gpu_find_nonfinite(static_cast<int64_t>(v.n), v.get(), prec_code(v.prec), &idx, nullptr), what);
  if (idx >= 0) throw ValidationError(std::string(what) + ": non-finite entry at index " + std::to_string(idx));
}

void dev_spmv(const EllMatrix& A, const DevVec& x, DevVec& y, const ExecContext& ctx) {
  const DeviceEll& D = A.device();
  check(mpmg_gpu_ell_spmv(D.rows, D.rw, D.col.as<int32_t>(), D.val.get(), prec_code(A.precision()), x.get(), y.get(),
                          policy_word(ctx), nullptr),
        "spmv");
  const std::uint64_t slots = A.rows() * static_cast<std::uint64_t>(A.row_width());
  add(ctx.traffic, slots * vb(x.prec) * 2, A.rows() * vb(y.prec), slots * 4, slots * 2);
  if (ctx.validate) dev_validate(y, "spmv");  // kernels.cpp:254
}

void dev_axpy(double alpha, const DevVec& x, const DevVec& y, DevVec& out, const ExecContext& ctx) {
  check(mpmg_gpu_axpy(static_cast<int64_t>(x.n), prec_code(x.prec), alpha, x.get(), y.get(), out.get(),
                      policy_word(ctx), nullptr),
        "axpy");
  add(ctx.traffic, 2 * x.n * vb(x.prec), x.n * vb(x.prec), 0, 2 * x.n);
  if (ctx.validate) dev_validate(out, "axpy");  // kernels.cpp:273
}

void dev_vmul(const DevVec& a, const DevVec& b, DevVec& out, const ExecContext& ctx) {
  check(mpmg_gpu_vec_multiply(static_cast<int64_t>(a.n), prec_code(a.prec), a.get(), b.get(), out.get(),
                              policy_word(ctx), nullptr),
        "vec_multiply");
  add(ctx.traffic, 2 * a.n * vb(a.prec), a.n * vb(a.prec), 0, a.n);
  if (ctx.validate) dev_validate(out, "vec_multiply");  // kernels.cpp:291
}

static double seq(const DevVec& x, const DevVec& y, int take_sqrt) {
  DevBuf out(8);
  check(mpmg_gpu_dot_seq(static_cast<int64_t>(x.n), x.get(), prec_code(x.prec), y.get(), prec_code(y.prec),
                         out.as<double>(), take_sqrt, nullptr),
        "dot");
  double v = 0.0;
  out.download(&v, 8);
  return v;
}

double dev_dot(const DevVec& x, const DevVec& y, const ExecContext& ctx) {
  add(ctx.traffic, x.n * vb(x.prec) + y.n * vb(y.prec), 0, 0, 2 * x.n);
  return seq(x, y, 0);
}

double dev_norm(const DevVec& x, const ExecContext& ctx) {
  add(ctx.traffic, x.n * vb(x.prec), 0, 0, 2 * x.n + 1);
  return seq(x, x, 1);
}

void dev_copy(const DevVec& src, DevVec& dst) {
  check(mpmg_gpu_cast(static_cast<int64_t>(src.n), src.get(), prec_code(src.prec), dst.get(), prec_code(dst.prec),
                      nullptr, 1.0, 0u, nullptr),
        "copy");
}

// multigrid.cpp:79-89
void dev_jacobi(const EllMatrix& A, const DevVec& inv_diag, const DevVec& b, DevVec& u, DevVec& r, DevVec& t, int steps,
                double omega, const ExecContext& ctx) {
  for (int s = 0; s < steps; ++s) {
    dev_spmv(A, u, t, ctx);
    dev_axpy(-1.0, t, b, r, ctx);
    dev_vmul(inv_diag, r, t, ctx);
    dev_axpy(omega, t, u, u, ctx);
  }
}

// multigrid.cpp:91-151
CgResult dev_cg(const EllMatrix& A, const DevVec& b, DevVec& u, const BaseSolverConfig& cfg, const ExecContext& ctx) {
  const std::size_t n = A.rows();
  const Precision p = b.prec;
  const int max_it = cfg.max_iterations > 0 ? cfg.max_iterations : 10 * static_cast<int>(n);
  check(mpmg_dev_memset0(u.get(), n * bytes_per_value(p)), "cg");
  DevVec r(n, p), pv(n, p), Ap(n, p), scratch(n, p), best(n, p);
  dev_copy(b, r);  // r = b - A*0 (cast_vector copies are counted by the reference)
  add(ctx.traffic, n * vb(p), n * vb(p), 0, n);
  dev_copy(r, pv);
  add(ctx.traffic, n * vb(p), n * vb(p), 0, n);
  check(mpmg_dev_memset0(best.get(), n * bytes_per_value(p)), "cg");
  const double norm_b = dev_norm(b, ctx);
  if (norm_b == 0.0) return {0, true, 0.0};
  const double thr = cfg.mode == BaseSolverConfig::ToleranceMode::RelativeToRhs ? cfg.tolerance * norm_b : cfg.tolerance;
  double rz = dev_dot(r, r, ctx);
  double true_res = norm_b, best_res = true_res;
  int it = 0;
  while (true_res >= thr && it < max_it) {
    dev_spmv(A, pv, Ap, ctx);
    const double pAp = dev_dot(pv, Ap, ctx);
    if (!(pAp > 0.0) || !std::isfinite(pAp)) break;
    const double alpha = rz / pAp;
    dev_axpy(alpha, pv, u, u, ctx);
    dev_axpy(-alpha, Ap, r, r, ctx);
    const double rz_new = dev_dot(r, r, ctx);
    ++it;
    dev_spmv(A, u, scratch, ctx);
    dev_axpy(-1.0, scratch, b, scratch, ctx);
    true_res = dev_norm(scratch, ctx);
    if (true_res < best_res) {
      best_res = true_res;
      dev_copy(u, best);
    }
    if (rz == 0.0) break;
    dev_axpy(rz_new / rz, pv, r, pv, ctx);
    rz = rz_new;
  }
  if (true_res > best_res) {
    dev_copy(best, u);
    true_res = best_res;
  }
  return {it, true_res < thr, true_res};
}

// multigrid.cpp:236-268 (transfer_product :155-205, store_scaled :220-232)
double dev_restrict(const EllMatrix& R, const DevVec& r_fine, DevVec& r_coarse, bool rescale, const ExecContext& ctx) {
  const DeviceEll& D = R.device();
  const std::uint64_t slots = R.rows() * static_cast<std::uint64_t>(R.row_width());
  add(ctx.traffic, slots * vb(R.precision()) + slots * vb(r_fine.prec), 0, slots * 4, 2 * slots);
  double scale = 1.0;
  if (rescale && r_coarse.prec == Precision::FP16) {
    DevVec prod(R.rows(), Precision::FP64);
    check(mpmg_gpu_ell_transfer(D.rows, D.rw, D.col.as<int32_t>(), D.val.get(), prec_code(R.precision()), r_fine.get(),
                                prec_code(r_fine.prec), prec_code(r_coarse.prec), nullptr, 1, nullptr,
                                static_cast<double*>(prod.get()), policy_word(ctx), nullptr),
          "restrict");
    const double nrm = seq(prod, prod, 1);  // multigrid.cpp:246-250: sequential fma
    if (nrm > 0.0 && std::isfinite(nrm)) scale = nrm;
    add(ctx.traffic, R.rows() * vb(r_fine.prec), 0, 0, 2 * R.rows() + 1);
    check(mpmg_gpu_cast(D.rows, prod.get(), MPMG_FP64, r_coarse.get(), prec_code(r_coarse.prec), nullptr, scale,
                        policy_word(ctx), nullptr),
          "restrict store");
  } else {
    check(mpmg_gpu_ell_transfer(D.rows, D.rw, D.col.as<int32_t>(), D.val.get(), prec_code(R.precision()), r_fine.get(),
                                prec_code(r_fine.prec), prec_code(r_coarse.prec), nullptr, 1, r_coarse.get(), nullptr,
                                policy_word(ctx), nullptr),
          "restrict");
  }
  add(ctx.traffic, 0, R.rows() * vb(r_coarse.prec), 0, R.rows());
  if (ctx.validate) dev_validate(r_coarse, "restrict_with_cast");  // multigrid.cpp:259-265
  return scale;
}

// multigrid.cpp:270-280
void dev_prolong(const EllMatrix& P, const DevVec& c_coarse, DevVec& c_fine, double scale, const ExecContext& ctx) {
  const DeviceEll& D = P.device();
  DevBuf sc(8);
  sc.upload(&scale, 8);
  check(mpmg_gpu_ell_transfer(D.rows, D.rw, D.col.as<int32_t>(), D.val.get(), prec_code(P.precision()), c_coarse.get(),
                              prec_code(c_coarse.prec), prec_code(c_fine.prec), sc.as<double>(), 0, c_fine.get(), nullptr,
                              policy_word(ctx), nullptr),
        "prolong");
  const std::uint64_t slots = P.rows() * static_cast<std::uint64_t>(P.row_width());
  add(ctx.traffic, slots * vb(P.precision()) + slots * vb(c_coarse.prec), P.rows() * vb(c_fine.prec), slots * 4,
      2 * slots + P.rows());
}

DevHierarchy::DevHierarchy(MgHierarchy& hh) : h(hh) {
  lv.reserve(static_cast<std::size_t>(h.levels()));
  for (int l = 0; l < h.levels(); ++l) {
    const GridLevel& g = h.level(l);
    Lv x;
    x.inv_diag = DevVec(g.inv_diag);
    x.u = DevVec(g.unknowns(), g.precision);
    x.b = DevVec(g.unknowns(), g.precision);
    x.r = DevVec(g.unknowns(), g.precision);
    x.t = DevVec(g.unknowns(), g.precision);
    lv.push_back(std::move(x));
  }
}

// multigrid.cpp:362-393
void DevHierarchy::cycle(int l, const DevVec& rhs, DevVec& u, const ExecContext& caller, std::vector<TrafficCounter>& traffic) {
  GridLevel& g = h.level(l);
  Lv& L = lv[static_cast<std::size_t>(l)];
  const ExecContext ctx = caller.with_counter(&traffic[static_cast<std::size_t>(l)]);
  if (caller.validate && (rhs.prec != g.precision || u.prec != g.precision))
    throw ValidationError("v_cycle: vector precision does not match level " + std::to_string(l));
  if (l == 0) {
    dev_cg(g.A, rhs, u, h.base_solver(), ctx);
    return;
  }
  check(mpmg_dev_memset0(u.get(), u.n * bytes_per_value(u.prec)), "fill_zero");
  const SmootherConfig& sm = h.smoother();
  dev_jacobi(g.A, L.inv_diag, rhs, u, L.r, L.t, sm.pre_steps, sm.omega, ctx);
  dev_spmv(g.A, u, L.t, ctx);
  dev_axpy(-1.0, L.t, rhs, L.r, ctx);
  GridLevel& c = h.level(l - 1);
  Lv& C = lv[static_cast<std::size_t>(l - 1)];
  const bool rescale = h.rescales() && c.precision == Precision::FP16;
  const double scale = dev_restrict(c.restrict_from_finer, L.r, C.b, rescale, ctx);
  cycle(l - 1, C.b, C.u, caller, traffic);
  dev_prolong(c.prolong_to_finer, C.u, L.t, scale, ctx);
  dev_axpy(1.0, L.t, u, u, ctx);
  dev_jacobi(g.A, L.inv_diag, rhs, u, L.r, L.t, sm.post_steps, sm.omega, ctx);
}

void add_cycle_traffic(const MgHierarchy& h, std::vector<TrafficCounter>& traffic, const ExecContext& ctx) {
  const SmootherConfig& sm = h.smoother();
  for (int l = 1; l < h.levels(); ++l) {
    const GridLevel& g = h.level(l);
    const GridLevel& c = h.level(l - 1);
    TrafficCounter* t = &traffic[static_cast<std::size_t>(l)];
    const std::uint64_t n = g.unknowns(), slots = n * static_cast<std::uint64_t>(g.A.row_width()), b = vb(g.precision);
    const int spmvs = sm.pre_steps + sm.post_steps + 1;
    const int axpys = 2 * (sm.pre_steps + sm.post_steps) + 2;
    add(t, spmvs * slots * b * 2, spmvs * n * b, spmvs * slots * 4, spmvs * slots * 2);
    add(t, axpys * 2 * n * b, axpys * n * b, 0, axpys * 2 * n);
    add(t, (sm.pre_steps + sm.post_steps) * 2 * n * b, (sm.pre_steps + sm.post_steps) * n * b, 0,
        (sm.pre_steps + sm.post_steps) * n);
    const EllMatrix& R = c.restrict_from_finer;
    const std::uint64_t rs = R.rows() * static_cast<std::uint64_t>(R.row_width());
    add(t, rs * vb(R.precision()) + rs * b, R.rows() * vb(c.precision), rs * 4, 2 * rs + R.rows());
    const EllMatrix& P = c.prolong_to_finer;
    const std::uint64_t ps = P.rows() * static_cast<std::uint64_t>(P.row_width());
    add(t, ps * vb(P.precision()) + ps * vb(c.precision), P.rows() * b, ps * 4, 2 * ps + P.rows());
  }
  (void)ctx;
}

}  // namespace mpmg::detail
