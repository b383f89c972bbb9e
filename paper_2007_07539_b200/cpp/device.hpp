// Internal glue of the C++ drop-in layer: RAII device buffers over the C ABI
// (include/mpmg_gpu.h), error-code -> exception mapping, and the device
// mirrors of ELLPACK matrices. No CUDA headers: this layer only calls the
// C ABI, like any other FFI host.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "mpmg/ell_matrix.hpp"
#include "mpmg/errors.hpp"
#include "mpmg/traffic.hpp"
#include "mpmg/vector.hpp"
#include "mpmg_gpu.h"

namespace mpmg::detail {

inline int prec_code(Precision p) { return static_cast<int>(p); }

inline uint32_t policy_word(const ExecContext& ctx) {
  uint32_t w = 0;
  if (ctx.policy.flush_subnormals_to_zero) w |= MPMG_FTZ;
  if (ctx.policy.fused_multiply_add) w |= MPMG_FMA;
  if (ctx.fp16_accumulation == Fp16Accum::FP32) w |= MPMG_ACC32;
  return w;
}

[[noreturn]] inline void raise(int code, const char* what) {
  const std::string msg = std::string(what) + ": " + mpmg_last_error();
  switch (code) {
    case MPMG_EINVAL: throw std::invalid_argument(msg);
    case MPMG_ENONFINITE: throw ValidationError(msg);
    default: throw DeviceError(msg + " (code " + std::to_string(code) + ")");
  }
}
inline void check(int code, const char* what) {
  if (code != MPMG_OK) raise(code, what);
}

/// fails loudly when no CUDA device is visible: there is no CPU fallback
inline void require_device() {
  if (mpmg_dev_count() <= 0) throw DeviceError("mpmg: no CUDA device visible (the B200 path has no CPU fallback)");
}

class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(std::size_t bytes) : bytes_(bytes) {
    require_device();
    p_ = mpmg_dev_alloc(bytes);
    if (!p_) raise(MPMG_ENOMEM, "mpmg_dev_alloc");
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), bytes_(o.bytes_) { o.p_ = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      mpmg_dev_free(p_);
      p_ = o.p_;
      bytes_ = o.bytes_;
      o.p_ = nullptr;
    }
    return *this;
  }
  ~DevBuf() { mpmg_dev_free(p_); }
  void* get() const { return p_; }
  template <typename T> T* as() const { return static_cast<T*>(p_); }
  std::size_t bytes() const { return bytes_; }
  void upload(const void* src, std::size_t n) { check(mpmg_dev_h2d(p_, src, n), "h2d"); }
  void download(void* dst, std::size_t n) const { check(mpmg_dev_d2h(dst, p_, n), "d2h"); }

 private:
  void* p_ = nullptr;
  std::size_t bytes_ = 0;
};

/// a PVector staged on the device for one call
struct DevVec {
  DevBuf buf;
  std::size_t n = 0;
  Precision prec = Precision::FP64;
  DevVec() = default;
  DevVec(std::size_t len, Precision p) : buf(len * bytes_per_value(p)), n(len), prec(p) {}
  explicit DevVec(const PVector& v) : DevVec(v.size(), v.precision()) { buf.upload(v.raw(), n * bytes_per_value(prec)); }
  void to(PVector& v) const { buf.download(v.raw(), n * bytes_per_value(prec)); }
  void* get() const { return buf.get(); }
};

/// slot-major device copy of an EllMatrix
struct DeviceEll {
  DevBuf col, val;
  std::int64_t rows = 0;
  int rw = 0;
  Precision prec = Precision::FP64;
};

std::shared_ptr<DeviceEll> make_device_ell(const EllMatrix& A);

/// traffic model of the reference kernels (kernels.cpp / multigrid.cpp)
inline void add(TrafficCounter* t, std::uint64_t rd, std::uint64_t wr, std::uint64_t idx, std::uint64_t flops) {
  if (!t) return;
  t->value_bytes_read += rd;
  t->value_bytes_written += wr;
  t->index_bytes_read += idx;
  t->flops += flops;
}

/// device solver handles of a build() hierarchy, one per policy word
struct DeviceSolvers {
  mpmg_solver_config base{};
  struct Entry {
    uint32_t policy;
    mpmg_solver* s;
  };
  std::vector<Entry> items;
  ~DeviceSolvers() {
    for (auto& e : items) mpmg_solver_destroy(e.s);
  }
  mpmg_solver* get(uint32_t policy);
};

}  // namespace mpmg::detail
