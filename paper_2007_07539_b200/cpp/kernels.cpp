// Public kernel API (kernels.hpp) over the device ELLPACK kernels
// (csrc/mpmg_ell.cu). Argument checks and the traffic model follow the
// reference (kernels.cpp:243-395); the arithmetic runs on the GPU.
#include "mpmg/kernels.hpp"

#include <cmath>
#include <stdexcept>
#include <string>

#include "device.hpp"
#include "mpmg/errors.hpp"

namespace mpmg {

using namespace detail;

namespace {

void require(bool cond, const char* msg) {
  if (!cond) throw std::invalid_argument(msg);
}

void validate_finite(const PVector& v, const char* what) {
  for (std::size_t i = 0; i < v.size(); ++i)
    if (!std::isfinite(v.get(i)))
      throw ValidationError(std::string(what) + ": non-finite entry at index " + std::to_string(i));
}

std::uint64_t vb(const PVector& v) { return static_cast<std::uint64_t>(bytes_per_value(v.precision())); }

}  // namespace

void spmv(const EllMatrix& A, const PVector& x, PVector& y, const ExecContext& ctx) {
  require(A.cols() == x.size(), "spmv: dimension mismatch between A and x");
  require(A.rows() == y.size(), "spmv: dimension mismatch between A and y");
  require(A.precision() == x.precision(), "spmv: precision mismatch between A and x");
  require(x.precision() == y.precision(), "spmv: precision mismatch between x and y");
  require(&x != &y, "spmv: output must not alias the input");
  const DeviceEll& D = A.device();
  DevVec dx(x), dy(y.size(), y.precision());
  check(mpmg_gpu_ell_spmv(D.rows, D.rw, D.col.as<int32_t>(), D.val.get(), prec_code(A.precision()), dx.get(),
                          dy.get(), policy_word(ctx), nullptr),
        "spmv");
  dy.to(y);
  const std::uint64_t slots = A.rows() * static_cast<std::uint64_t>(A.row_width());
  add(ctx.traffic, slots * vb(x) * 2, A.rows() * vb(y), slots * 4, slots * 2);
  if (ctx.validate) validate_finite(y, "spmv");
}

PVector spmv(const EllMatrix& A, const PVector& x, const ExecContext& ctx) {
  PVector y(A.rows(), A.precision());
  spmv(A, x, y, ctx);
  return y;
}

void axpy(double alpha, const PVector& x, const PVector& y, PVector& out, const ExecContext& ctx) {
  require(x.size() == y.size() && x.size() == out.size(), "axpy: dimension mismatch");
  require(x.precision() == y.precision() && x.precision() == out.precision(), "axpy: precision mismatch");
  DevVec dx(x), dy(y), dout(out.size(), out.precision());
  check(mpmg_gpu_axpy(static_cast<int64_t>(x.size()), prec_code(x.precision()), alpha, dx.get(), dy.get(), dout.get(),
                      policy_word(ctx), nullptr),
        "axpy");
  dout.to(out);
  add(ctx.traffic, 2 * x.size() * vb(x), x.size() * vb(x), 0, 2 * x.size());
  if (ctx.validate) validate_finite(out, "axpy");
}

PVector axpy(double alpha, const PVector& x, const PVector& y, const ExecContext& ctx) {
  PVector out(x.size(), x.precision());
  axpy(alpha, x, y, out, ctx);
  return out;
}

void vec_multiply(const PVector& a, const PVector& b, PVector& out, const ExecContext& ctx) {
  require(a.size() == b.size() && a.size() == out.size(), "vec_multiply: dimension mismatch");
  require(a.precision() == b.precision() && a.precision() == out.precision(), "vec_multiply: precision mismatch");
  DevVec da(a), db(b), dout(out.size(), out.precision());
  check(mpmg_gpu_vec_multiply(static_cast<int64_t>(a.size()), prec_code(a.precision()), da.get(), db.get(), dout.get(),
                              policy_word(ctx), nullptr),
        "vec_multiply");
  dout.to(out);
  add(ctx.traffic, 2 * a.size() * vb(a), a.size() * vb(a), 0, a.size());
  if (ctx.validate) validate_finite(out, "vec_multiply");
}

PVector vec_multiply(const PVector& a, const PVector& b, const ExecContext& ctx) {
  PVector out(a.size(), a.precision());
  vec_multiply(a, b, out, ctx);
  return out;
}

void update_residuum_correction(PVector& r, PVector& u, const EllMatrix& A, const PVector& c, double alpha,
                                const ExecContext& ctx) {
  require(r.precision() == Precision::FP64 && u.precision() == Precision::FP64,
          "update_residuum_correction: r and u must be binary64");
  require(A.precision() == Precision::FP64, "update_residuum_correction: A must be binary64");
  require(A.rows() == A.cols(), "update_residuum_correction: A must be square");
  require(r.size() == A.rows() && u.size() == A.rows() && c.size() == A.rows(),
          "update_residuum_correction: dimension mismatch");
  const DeviceEll& D = A.device();
  DevVec dr(r), du(u), dc(c);
  DevBuf al(8);
  al.upload(&alpha, 8);
  check(mpmg_gpu_ell_update_rc(D.rows, D.rw, D.col.as<int32_t>(), D.val.as<double>(), dc.get(), prec_code(c.precision()),
                               static_cast<double*>(dr.get()), static_cast<double*>(du.get()), al.as<double>(),
                               policy_word(ctx), nullptr),
        "update_residuum_correction");
  dr.to(r);
  du.to(u);
  const std::uint64_t n = A.rows(), slots = n * static_cast<std::uint64_t>(A.row_width());
  add(ctx.traffic, slots * 8 + 2 * n * 8 + n * vb(c), 2 * n * 8, slots * 4, 2 * slots + 4 * n);
  if (ctx.validate) {
    validate_finite(r, "update_residuum_correction");
    validate_finite(u, "update_residuum_correction");
  }
}

void cast_vector(const PVector& x, Precision target, double scale, PVector& out, const ExecContext& ctx) {
  require(scale > 0.0 && std::isfinite(scale), "cast_vector: scale must be positive and finite");
  require(out.size() == x.size(), "cast_vector: dimension mismatch");
  require(out.precision() == target, "cast_vector: output precision mismatch");
  DevVec dx(x), dout(out.size(), target);
  check(mpmg_gpu_cast(static_cast<int64_t>(x.size()), dx.get(), prec_code(x.precision()), dout.get(), prec_code(target),
                      nullptr, scale, policy_word(ctx), nullptr),
        "cast_vector");
  dout.to(out);
  add(ctx.traffic, x.size() * vb(x), x.size() * static_cast<std::uint64_t>(bytes_per_value(target)), 0, x.size());
}

PVector cast_vector(const PVector& x, Precision target, double scale, const ExecContext& ctx) {
  PVector out(x.size(), target);
  cast_vector(x, target, scale, out, ctx);
  return out;
}

double dot_fp64(const PVector& x, const PVector& y, const ExecContext& ctx) {
  require(x.size() == y.size(), "dot: dimension mismatch");
  DevVec dx(x), dy(y);
  DevBuf out(8);
  check(mpmg_gpu_dot_seq(static_cast<int64_t>(x.size()), dx.get(), prec_code(x.precision()), dy.get(),
                         prec_code(y.precision()), out.as<double>(), 0, nullptr),
        "dot_fp64");
  double v = 0.0;
  out.download(&v, 8);
  add(ctx.traffic, x.size() * vb(x) + y.size() * vb(y), 0, 0, 2 * x.size());
  return v;
}

double norm2_fp64(const PVector& x, const ExecContext& ctx) {
  DevVec dx(x);
  DevBuf out(8);
  check(mpmg_gpu_dot_seq(static_cast<int64_t>(x.size()), dx.get(), prec_code(x.precision()), dx.get(),
                         prec_code(x.precision()), out.as<double>(), 1, nullptr),
        "norm2_fp64");
  double v = 0.0;
  out.download(&v, 8);
  add(ctx.traffic, x.size() * vb(x), 0, 0, 2 * x.size() + 1);
  return v;
}

}  // namespace mpmg
