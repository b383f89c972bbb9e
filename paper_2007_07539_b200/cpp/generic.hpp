// Device-resident generic ELLPACK multigrid (internal to the C++ layer):
// the reference's level operations (multigrid.cpp:79-280) and V-cycle
// recursion (:354-393) on device buffers, one C-ABI kernel per reference
// kernel call, so results match the reference op for op.
#pragma once

#include <vector>

#include "device.hpp"
#include "mpmg/multigrid.hpp"

namespace mpmg::detail {

// validate mode: throws ValidationError("<what>: non-finite entry at index i")
void dev_validate(const DevVec& v, const char* what);
// y = A x, r = b - A u etc. on device vectors of matching precision
void dev_spmv(const EllMatrix& A, const DevVec& x, DevVec& y, const ExecContext& ctx);
void dev_axpy(double alpha, const DevVec& x, const DevVec& y, DevVec& out, const ExecContext& ctx);
void dev_vmul(const DevVec& a, const DevVec& b, DevVec& out, const ExecContext& ctx);
double dev_dot(const DevVec& x, const DevVec& y, const ExecContext& ctx);
double dev_norm(const DevVec& x, const ExecContext& ctx);
void dev_copy(const DevVec& src, DevVec& dst);  // same precision, untracked

void dev_jacobi(const EllMatrix& A, const DevVec& inv_diag, const DevVec& b, DevVec& u, DevVec& r, DevVec& t, int steps,
                double omega, const ExecContext& ctx);
CgResult dev_cg(const EllMatrix& A, const DevVec& b, DevVec& u, const BaseSolverConfig& cfg, const ExecContext& ctx);
double dev_restrict(const EllMatrix& R, const DevVec& r_fine, DevVec& r_coarse, bool rescale, const ExecContext& ctx);
void dev_prolong(const EllMatrix& P, const DevVec& c_coarse, DevVec& c_fine, double scale, const ExecContext& ctx);

/// per-level device scratch of a hierarchy for one generic V-cycle
struct DevHierarchy {
  struct Lv {
    DevVec inv_diag, u, b, r, t;
  };
  MgHierarchy& h;
  std::vector<Lv> lv;
  explicit DevHierarchy(MgHierarchy& hh);
  /// cycle_at(l) with rhs / result on the device
  void cycle(int l, const DevVec& rhs, DevVec& u, const ExecContext& ctx, std::vector<TrafficCounter>& traffic);
};

/// the reference's traffic model for one V-cycle of a build() hierarchy
/// (the device solver runs it fused; CG iterations are not included)
void add_cycle_traffic(const MgHierarchy& h, std::vector<TrafficCounter>& traffic, const ExecContext& ctx);

}  // namespace mpmg::detail
