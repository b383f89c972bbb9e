// Solver engine: device-resident level hierarchy, V-cycle schedule and the
// FP64 iterative-refinement loop (the reference's MgHierarchy::build /
// v_cycle, multigrid.cpp:282-393, and ir_solve, ir_solver.cpp:51-127),
// re-designed for one B200:
//   * every level vector lives in HBM in the ghost-aliased pitch layout;
//   * a level with more than kCoarsePoints unknowns runs the streaming
//     stencil kernels; all coarser levels (and the CG base solve) run inside
//     one persistent cooperative kernel (mpmg_coarse.cu);
//   * the outer loop runs on the device: a control kernel reduces ||r||,
//     applies the reference's stopping rules and sets the condition of a CUDA
//     graph WHILE node, so a whole solve is one graph launch with no host
//     round trip per iteration (fallback: host loop over a captured
//     iteration graph).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "mpmg_host.h"
#include "mpmg_internal.h"

namespace mpmg_impl {

thread_local std::string g_err;

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MPMG_PDL");
    v = e ? std::atoi(e) : 0;  // off by default: no measured gain inside the graph
  }
  return v != 0;
}
std::string& last_error() { return g_err; }
int set_cuda_error(cudaError_t e) {
  g_err = cudaGetErrorString(e);
  return MPMG_ECUDA;
}

namespace {

// levels with more interior unknowns than this run the streaming (plane)
// kernels, one launch per operation; the rest run inside the one persistent
// cooperative coarse kernel (mpmg_coarse.cu)
constexpr long long kCoarsePoints = 32768;
// (MPMG_COARSE_POINTS / MPMG_CTA_POINTS override both thresholds for tuning)
long long env_ll(const char* name, long long dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoll(v) : dflt;
}
constexpr int kCtlThreads = 256;

struct Level {
  mpmg_stencil A{};
  double omega_r = 0.0;
  size_t len = 0;
  int bytes = 8;
  bool big = false;
  void *u = nullptr, *u2 = nullptr, *b = nullptr, *r = nullptr;
  double* prod = nullptr;   // binary64 restriction product (DSH rescale / coarse kernel)
  double* scale = nullptr;  // device scalar: scale of the restriction into this level
};

// sums the selected partial-sum buffer (fixed order), sets alpha = sqrt and
// applies ir_solver.cpp:95-120 to the device IR state
__global__ void k_control(IrState* st, const double* p_main, int n_main, const double* p_ref, int n_ref,
                          double* hist, int hist_cap, double tol, int max_it, int scale_enabled, int refresh,
                          int increment, cudaGraphConditionalHandle cond, int use_cond, int ring_k,
                          int reuse_refresh) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // pdl_wait (mpmg_arith.cuh)
  __shared__ double red[kCtlThreads];
  const bool ref = increment && st->refresh_now;
  const double* p = ref ? p_ref : p_main;
  const int n = ref ? n_ref : n_main;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += kCtlThreads) acc += p[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kCtlThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double alpha = sqrt(red[0]);
    // deferred corrections: this iteration stored one more c in the ring,
    // or folded all of them (and its own) into u
    if (increment && ring_k > 0) {
      if (st->fold_now) st->u_zero = 0;
      st->pending = st->fold_now ? 0 : st->pending + 1;
    }
    if (increment) st->iterations += 1;
    const int it = st->iterations;
    if (hist && it < hist_cap) hist[it] = alpha;
    st->alpha = alpha;
    int active = 0;
    if (!isfinite(alpha)) st->diverged = 1;                 // DivergedError
    else if (alpha < tol) st->converged = 1;
    else if (it >= max_it) active = 0;                       // budget exhausted, not an error
    else {
      active = 1;
      st->scale = (scale_enabled && alpha > 0.0) ? alpha : 1.0;  // ir_solver.cpp:109
    }
    st->active = active;
    st->refresh_now = (refresh > 0 && (it + 1) % refresh == 0) ? 1 : 0;
    // the next iteration folds the ring into u when it refreshes r = b - A u
    // or when its c fills the last slot
    st->fold_now = ring_k > 0 && (st->refresh_now || st->pending + 1 >= ring_k) ? 1 : 0;
    // residual_norm (ir_solver.cpp:21-49) of an iterate whose refresh defect
    // just ran is that defect's sum of squares: fma(-1, t, b) and b - t round
    // identically and both use the FMA product A u
    st->final_pending = (increment && ref && reuse_refresh) ? 0 : 1;
    if (use_cond) cudaGraphSetConditional(cond, active ? 1u : 0u);
  }
}

__global__ void k_state_reset(IrState* st, int u_zero) {
  st->alpha = 0.0;
  st->scale = 1.0;
  st->iterations = 0;
  st->converged = 0;
  st->diverged = 0;
  st->active = 0;
  st->refresh_now = 0;
  st->pending = 0;
  st->fold_now = 0;
  st->final_pending = 1;
  st->u_zero = u_zero;
}

__global__ void k_sanitize_scale(double* s) {
  const double v = *s;
  if (!(v > 0.0) || !isfinite(v)) *s = 1.0;  // multigrid.cpp:250
}

__global__ void k_fill_one(double* s) { *s = 1.0; }

}  // namespace
}  // namespace mpmg_impl

using namespace mpmg_impl;

struct mpmg_solver {
  mpmg_solver_config cfg{};
  std::vector<Level> lv;
  mpmg_stencil A64{};
  int nc = 0;  // levels [0, nc) run in the coarse kernel
  CoarseArgs cargs{};
  size_t len = 0;  // finest padded length
  double *u = nullptr, *r = nullptr, *b = nullptr;
  double* stage = nullptr;  // compact host-I/O staging (padded buffers keep zero ghosts)
  void* rlow = nullptr;  // finest-precision scaled residual (== lv.back().b)
  bool rlow_alias = false;
  double *partU = nullptr, *partD = nullptr;
  int nU = 0, nD = 0;
  // deferred corrections (binary16/32 finest level): the r half of
  // update_residuum_correction runs every iteration and parks c in a ring;
  // u += a_k c_k is applied for all parked k at once, in order, when r is
  // refreshed from u, when the ring is full and at the end of the solve --
  // per element the same fma sequence, so u is bitwise unchanged, while each
  // iteration skips the FP64 read + write of u (16 of 34 bytes per unknown)
  int ring_k = 0;  // 0: fused update (FP64 finest level or unsupported shape)
  bool ring_cycle = false;  // while enqueueing an IR iteration: the V-cycle may end in the ring
  void* ring = nullptr;
  long long ring_len = 0;
  double* ring_scale = nullptr;
  IrState* st = nullptr;
  IrState* st_h = nullptr;
  double* hist = nullptr;
  int hist_cap = 0;
  double* final_d = nullptr;
  double* final_h = nullptr;
  double* one = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  std::vector<void*> allocs;
  // captured solve graph and the parameters it was captured with
  cudaGraphExec_t exec = nullptr;
  mpmg_solve_params gkey{};
  bool gvalid = false;

  ~mpmg_solver() {
    if (exec) cudaGraphExecDestroy(exec);
    for (void* p : allocs) cudaFree(p);
    if (st_h) cudaFreeHost(st_h);
    if (final_h) cudaFreeHost(final_h);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (s) cudaStreamDestroy(s);
  }

  template <typename T>
  cudaError_t alloc(T** p, size_t bytes) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(q, 0, std::max<size_t>(bytes, 16), s);
    allocs.push_back(q);
    *p = static_cast<T*>(q);
    return e;
  }

  uint32_t policy() const { return cfg.policy; }
  bool fma() const { return cfg.policy & MPMG_FMA; }
  int finest() const { return (int)lv.size() - 1; }

  // ---- V-cycle schedule (cycle_at, multigrid.cpp:362-393) ----------------
  cudaError_t run_coarse(cudaStream_t q) { return launch_coarse_cycle(cargs, policy(), q); }

  // returns the buffer holding the level-l correction
  cudaError_t cycle(int l, cudaStream_t q, void** result) {
    Level& L = lv[l];
    if (!L.big) {  // this level and everything below: one CTA
      cudaError_t e = run_coarse(q);
      *result = L.u;
      return e;
    }
    cudaError_t e = cudaSuccess;
    void* cur = nullptr;
    int k = 0;
    if (cfg.pre_steps >= 2) {  // steps 1+2 from zero in one pass (result in u2, like the unfused pair)
      e = launch_jacobi_zero2(L.A, L.b, L.u, L.u2, cfg.omega, L.omega_r, policy(), q);
      cur = L.u2;
      k = 2;
    }
    for (; k < cfg.pre_steps && e == cudaSuccess; ++k) {
      void* out = (cur == L.u) ? L.u2 : L.u;
      if (!cur) e = launch_jacobi_zero(L.A.dim, L.A.nodes, L.A.prec, L.b, out, L.omega_r, L.A.inv_diag, policy(), q);
      else e = launch_level_op(2, L.A, cur, L.b, out, cfg.omega, policy(), q);
      cur = out;
    }
    if (e != cudaSuccess) return e;
    if (!cur) {
      e = cudaMemsetAsync(L.u, 0, L.len * L.bytes, q);
      cur = L.u;
    }
    if (e == cudaSuccess) e = launch_level_op(1, L.A, cur, L.b, L.r, cfg.omega, policy(), q);
    Level& C = lv[l - 1];
    const bool rescale = cfg.variant == MPMG_DSH_MG && C.A.prec == MPMG_FP16;  // multigrid.cpp:383
    if (e == cudaSuccess) {
      if (rescale) {
        // R r_f kept exactly in binary64, scale = ||R r_f||, then the scaled cast
        e = launch_restrict(L.A.dim, L.A.nodes, L.A.prec, MPMG_FP64, L.r, C.prod, nullptr, policy(), q);
        if (e == cudaSuccess) e = launch_norm2(C.len, C.prod, partD, C.scale, q);
        if (e == cudaSuccess) { k_sanitize_scale<<<1, 1, 0, q>>>(C.scale); e = cudaGetLastError(); }
        if (e == cudaSuccess) e = launch_downcast(C.A.dim, C.A.nodes, C.prod, C.b, C.A.prec, C.scale, 1, policy(), q);
      } else {
        e = launch_restrict(L.A.dim, L.A.nodes, L.A.prec, C.A.prec, L.r, C.b, nullptr, policy(), q);
      }
    }
    if (e != cudaSuccess) return e;
    void* cc = nullptr;
    e = cycle(l - 1, q, &cc);
    if (e != cudaSuccess) return e;
    // scale of the restriction into C (the coarse kernel keeps its own
    // internal scales; this one crosses from a streaming level)
    const double* sc = rescale ? C.scale : nullptr;
    e = launch_prolong(L.A.dim, L.A.nodes, L.A.prec, C.A.prec, cc, cur, sc, policy(), q);
    for (int k = 0; k < cfg.post_steps && e == cudaSuccess; ++k) {
      void* out = (cur == L.u) ? L.u2 : L.u;
      if (ring_cycle && l == finest() && k == cfg.post_steps - 1) {
        // the correction goes straight into the deferred-correction ring slot
        // (read there by UPDATE_R, which then skips its copy)
        bool done = false;
        if (L.A.prec == MPMG_FP16)
          done = plane_jacobi_slot_f16(L.A, cur, L.b, ring, ring_len, &st->pending, cfg.omega, policy(), q, &e);
        else if (L.A.prec == MPMG_FP32)
          done = plane_jacobi_slot_f32(L.A, cur, L.b, ring, ring_len, &st->pending, cfg.omega, policy(), q, &e);
        if (done) {
          *result = nullptr;
          return e;
        }
      }
      e = launch_level_op(2, L.A, cur, L.b, out, cfg.omega, policy(), q);
      cur = out;
    }
    *result = cur;
    return e;
  }

  cudaError_t v_cycle(cudaStream_t q, void** result) { return cycle(finest(), q, result); }

  // ---- IR loop pieces --------------------------------------------------------
  int scale_enabled(const mpmg_solve_params& p) const {
    if (p.scaling == 1) return 1;
    if (p.scaling == 2) return 0;
    return cfg.variant != MPMG_D_MG;  // ir_solver.cpp:70-76
  }

  cudaError_t enqueue_init(const mpmg_solve_params& p, cudaStream_t q, cudaGraphConditionalHandle h, int use_cond) {
    // deferred corrections from u0 = 0: u is first written by a fold, which
    // starts from +0 instead of reading it (no zero fill, no first read)
    const int uz = ring_k > 0 && !p.random_initial_guess;
    k_state_reset<<<1, 1, 0, q>>>(st, uz);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && !uz) e = cudaMemsetAsync(u, 0, len * sizeof(double), q);
    if (e == cudaSuccess && p.random_initial_guess)
      e = launch_fill_random01(u, cfg.dim, cfg.nodes, p.seed, q);
    int n0 = nD;  // ir_solver.cpp:92-93: r = b - A u
    if (e == cudaSuccess && p.random_initial_guess) e = launch_defect64(A64, b, u, r, partD, fma(), false, q);
    else if (e == cudaSuccess) {  // u = 0: r = b bitwise
      e = launch_copy_sumsq(len, b, r, partD, q);
      n0 = norm2_partials(len);
    }
    if (e == cudaSuccess) {
      k_control<<<1, kCtlThreads, 0, q>>>(st, partD, n0, partD, n0, hist, hist_cap, p.outer_tolerance,
                                            p.max_outer_iterations, scale_enabled(p),
                                            p.residual_refresh_interval, 0, h, use_cond, ring_k, 0);
      e = cudaGetLastError();
    }
    return e;
  }

  cudaError_t enqueue_iteration(const mpmg_solve_params& p, cudaStream_t q, cudaGraphConditionalHandle h,
                                int use_cond) {
    cudaError_t e = cudaSuccess;
    const int fp = lv.back().A.prec;
    if (!rlow_alias)  // cast_vector(r, mg_precision, scale, r_low), ir_solver.cpp:109-110
      e = launch_downcast(cfg.dim, cfg.nodes, r, rlow, fp, &st->scale, 1, policy(), q);
    void* c = nullptr;
    ring_cycle = ring_k > 0;
    if (e == cudaSuccess) e = v_cycle(q, &c);  // ir_solver.cpp:111 (c == nullptr: in the ring slot)
    ring_cycle = false;
    if (ring_k > 0) {  // ir_solver.cpp:112, the u half deferred
      if (e == cudaSuccess && !plane_update_r(A64, c, fp, r, &st->scale, partU, ring, ring_len, &st->pending,
                                              ring_scale, fma(), q, &e) &&
          !stencil_update_r(A64, c, fp, r, &st->scale, partU, ring, ring_len, &st->pending, ring_scale, fma(), q,
                            &e))
        e = cudaErrorInvalidValue;
      if (e == cudaSuccess)
        e = launch_fold(len, u, ring, ring_len, fp, ring_scale, &st->pending, 1, &st->fold_now, fma(), q, &st->u_zero);
    } else if (e == cudaSuccess) {  // ir_solver.cpp:112
      e = launch_update_rc(A64, c, fp, r, u, &st->scale, partU, fma(), q);
    }
    if (e == cudaSuccess && p.residual_refresh_interval > 0)  // ir_solver.cpp:115-119 (gated on device)
      e = launch_defect64(A64, b, u, r, partD, fma(), false, q, &st->refresh_now);
    if (e == cudaSuccess) {
      e = launch_pdl(k_control, dim3(1), dim3(kCtlThreads), 0, q, st, (const double*)partU, nU,
                     (const double*)partD, nD, hist, hist_cap, p.outer_tolerance, p.max_outer_iterations,
                     scale_enabled(p), p.residual_refresh_interval, 1, h, use_cond, ring_k, fma() ? 1 : 0);
    }
    return e;
  }

  cudaError_t enqueue_final(cudaStream_t q) {  // residual_norm, ir_solver.cpp:21-49 / :122
    cudaError_t e = cudaSuccess;
    if (ring_k > 0)  // corrections still parked
      e = launch_fold(len, u, ring, ring_len, lv.back().A.prec, ring_scale, &st->pending, 0, nullptr, fma(), q,
                      &st->u_zero);
    if (e == cudaSuccess) e = launch_defect64(A64, b, u, nullptr, partD, true, true, q, &st->final_pending);
    if (e == cudaSuccess) e = launch_norm_finalize(partD, nD, final_d, q);
    return e;
  }

  static bool same_params(const mpmg_solve_params& a, const mpmg_solve_params& b) {
    return a.outer_tolerance == b.outer_tolerance && a.max_outer_iterations == b.max_outer_iterations &&
           a.random_initial_guess == b.random_initial_guess && a.seed == b.seed && a.scaling == b.scaling &&
           a.residual_refresh_interval == b.residual_refresh_interval;
  }

  // whole solve as one graph: init -> WHILE(active){iteration} -> final norm
  cudaError_t build_graph(const mpmg_solve_params& p) {
    if (exec) { cudaGraphExecDestroy(exec); exec = nullptr; }
    gvalid = false;
    cudaStream_t body_s = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&body_s, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
    cudaGraph_t g = nullptr;
    e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    cudaGraphConditionalHandle h{};
    cudaGraph_t cg = nullptr;
    if (e == cudaSuccess) {
      cudaStreamCaptureStatus stt;
      const cudaGraphNode_t* deps = nullptr;
      size_t nd = 0;
      e = cudaStreamGetCaptureInfo(s, &stt, nullptr, &cg, &deps, &nd);
      if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault);
      if (e == cudaSuccess) e = enqueue_init(p, s, h, 1);
      cudaGraphNode_t node = nullptr;
      cudaGraph_t body = nullptr;
      if (e == cudaSuccess) e = cudaStreamGetCaptureInfo(s, &stt, nullptr, &cg, &deps, &nd);
      if (e == cudaSuccess) {
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        e = cudaGraphAddNode(&node, cg, deps, nd, &cp);
        if (e == cudaSuccess) body = cp.conditional.phGraph_out[0];
      }
      if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
      if (e == cudaSuccess) {
        e = cudaStreamBeginCaptureToGraph(body_s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess) {
          const cudaError_t e2 = enqueue_iteration(p, body_s, h, 1);
          cudaGraph_t dummy = nullptr;
          const cudaError_t e3 = cudaStreamEndCapture(body_s, &dummy);
          e = e2 != cudaSuccess ? e2 : e3;
        }
      }
      if (e == cudaSuccess) e = enqueue_final(s);
      cudaGraph_t out = nullptr;
      const cudaError_t e4 = cudaStreamEndCapture(s, &out);
      if (e == cudaSuccess) e = e4;
      g = e4 == cudaSuccess ? out : nullptr;  // an invalidated capture hands back no graph to destroy
    }
    cudaStreamDestroy(body_s);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, g, 0);
    if (g) cudaGraphDestroy(g);
    if (e == cudaSuccess) {
      gkey = p;
      gvalid = true;
    } else {
      cudaGetLastError();  // clear sticky capture errors
      exec = nullptr;
    }
    return e;
  }
};

namespace {

int finish(cudaError_t e) { return e == cudaSuccess ? MPMG_OK : set_cuda_error(e); }

}  // namespace

extern "C" {

size_t mpmg_padded_len(int32_t dim, int32_t nodes) {
  const size_t P = (size_t)(nodes - 1);
  return dim == 3 ? P * P * P + P * P + P + 1 : P * P + P + 1;
}

size_t mpmg_interior_len(int32_t dim, int32_t nodes) {
  const size_t m = nodes > 2 ? (size_t)(nodes - 2) : 0;
  return dim == 3 ? m * m * m : m * m;
}

int mpmg_bytes_per_value(int32_t prec) { return prec == MPMG_FP16 ? 2 : (prec == MPMG_FP32 ? 4 : 8); }

const char* mpmg_last_error(void) { return g_err.c_str(); }

void mpmg_solver_default_config(mpmg_solver_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->dim = 3; c->k = 1; c->nodes = 65; c->levels = 6; c->variant = MPMG_H_MG;
  c->pre_steps = 3; c->post_steps = 3; c->omega = 2.0 / 3.0;  // SmootherConfig{3,3,2/3}
  c->base_tol = 1e-4; c->base_mode = 0; c->base_max_iterations = 0;  // BaseSolverConfig{}
  c->policy = MPMG_FTZ | MPMG_FMA;  // ArithmeticPolicy{} default
  c->device = 0;
}

void mpmg_solve_default_params(mpmg_solve_params* p) {
  std::memset(p, 0, sizeof(*p));
  p->outer_tolerance = 1e-9;  // IrConfig{} (ir_solver.hpp:16-23)
  p->max_outer_iterations = 100;
  p->residual_refresh_interval = 10;
  p->use_graph = 1;
}

int mpmg_problem_rhs(int32_t dim, int32_t nodes, int32_t k, double* b_out) {
  if ((dim != 2 && dim != 3) || nodes < 3 || k < 1 || !b_out) return MPMG_EINVAL;
  problem_rhs(dim, nodes, k, b_out);
  return MPMG_OK;
}

mpmg_solver* mpmg_solver_create(const mpmg_solver_config* cfg, int* err, int* err_level) {
  clear_stale_error();
  auto fail = [&](int code, int level) -> mpmg_solver* {
    if (err) *err = code;
    if (err_level) *err_level = level;
    return nullptr;
  };
  if (err) *err = MPMG_OK;
  if (err_level) *err_level = -1;
  if (!cfg) return fail(MPMG_EINVAL, -1);
  const mpmg_solver_config c = *cfg;
  // ProblemSpec::validate (mesh_fem.cpp:57-69) + build preconditions (multigrid.cpp:285-286)
  if ((c.dim != 2 && c.dim != 3) || c.k < 1 || c.levels < 2 || c.levels > 30 || c.nodes < 3 ||
      (c.nodes - 1) % (1 << (c.levels - 1)) != 0 || ((c.nodes - 1) >> (c.levels - 1)) + 1 < 3) {
    last_error() = "invalid ProblemSpec";
    return fail(MPMG_EINVAL, -1);
  }
  if (c.pre_steps < 0 || c.post_steps < 0 || !(c.omega > 0.0 && c.omega <= 1.0) || !(c.base_tol > 0.0)) {
    last_error() = "invalid smoother/base-solver config";
    return fail(MPMG_EINVAL, -1);
  }
  cudaError_t e = cudaSetDevice(c.device);
  if (e != cudaSuccess) { set_cuda_error(e); return fail(MPMG_ECUDA, -1); }
  auto* S = new mpmg_solver();
  S->cfg = c;
  const bool ftz = c.policy & MPMG_FTZ;
  e = cudaStreamCreateWithFlags(&S->s, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&S->e0);
  if (e == cudaSuccess) e = cudaEventCreate(&S->e1);
  if (e != cudaSuccess) { set_cuda_error(e); delete S; return fail(MPMG_ECUDA, -1); }

  S->lv.resize(c.levels);
  for (int l = 0; l < c.levels; ++l) {
    Level& L = S->lv[l];
    const int nl = ((c.nodes - 1) >> (c.levels - 1 - l)) + 1;  // nodes_at_level, mesh_fem.hpp:20-22
    const int prec = variant_precision(c.variant, l);
    const int rc = build_level_stencil(c.dim, nl, prec, ftz, &L.A);
    if (rc != MPMG_OK) { delete S; return fail(rc, l); }
    L.omega_r = round_to(c.omega, prec, ftz);
    L.len = mpmg_padded_len(c.dim, nl);
    L.bytes = mpmg_bytes_per_value(prec);
    L.big = (long long)mpmg_interior_len(c.dim, nl) > env_ll("MPMG_COARSE_POINTS", kCoarsePoints) &&
            stencil_supported(c.dim, nl, prec);
  }
  // big levels must be a suffix (finest levels)
  for (int l = c.levels - 1; l >= 1; --l)
    if (!S->lv[l].big) { for (int k = 0; k < l; ++k) S->lv[k].big = false; break; }
  for (int l = 0; l < c.levels; ++l)
    if (!S->lv[l].big) S->nc = l + 1;
  if (S->nc > kMaxCoarseLevels) { last_error() = "too many coarse levels"; delete S; return fail(MPMG_EUNSUPPORTED, -1); }

  // finest FP64 operator (A_high of ir_solve)
  build_level_stencil(c.dim, c.nodes, MPMG_FP64, ftz, &S->A64);
  S->len = mpmg_padded_len(c.dim, c.nodes);
  const int F = c.levels - 1;
  const int fprec = S->lv[F].A.prec;
  e = S->alloc(&S->u, S->len * 8);
  if (e == cudaSuccess) e = S->alloc(&S->r, S->len * 8);
  if (e == cudaSuccess) e = S->alloc(&S->b, S->len * 8);
  if (e == cudaSuccess) e = S->alloc(&S->stage, mpmg_interior_len(c.dim, c.nodes) * 8);
  // D_MG without forced scaling casts r to FP64 with scale 1: a bitwise copy,
  // so the finest rhs aliases r. Decided per solve below; we keep
  // a separate buffer too so ForceOn scaling works.
  for (int l = 0; l < c.levels && e == cudaSuccess; ++l) {
    Level& L = S->lv[l];
    const size_t bytes = L.len * L.bytes;
    e = S->alloc(&L.u, bytes);
    if (e == cudaSuccess) e = S->alloc(&L.u2, bytes);
    if (e == cudaSuccess) e = S->alloc(&L.b, bytes);
    if (e == cudaSuccess) e = S->alloc(&L.r, bytes);
    if (e == cudaSuccess && l < F) e = S->alloc(&L.prod, L.len * 8);
    if (e == cudaSuccess) e = S->alloc(&L.scale, 8);
    if (e == cudaSuccess) { k_fill_one<<<1, 1, 0, S->s>>>(L.scale); e = cudaGetLastError(); }
  }
  S->rlow = S->lv[F].b;
  (void)fprec;
  // partial-sum buffers
  S->nU = stencil_partials(c.dim, c.nodes, fprec, true);
  S->nD = stencil_partials(c.dim, c.nodes, MPMG_FP64, false);
  if (env_ll("MPMG_DEFER_U", 1) != 0 && fprec != MPMG_FP64) {
    int nr = plane_update_r_partials(c.dim, c.nodes, fprec);
    if (nr <= 0 && stencil_supported(c.dim, c.nodes, fprec))  // the streaming UPDATE_R (2D, other pitches)
      nr = stencil_partials(c.dim, c.nodes, fprec, true);
    if (nr > 0) {
      S->ring_k = 10;
      S->nU = nr;
      S->ring_len = (long long)((S->len + 63) / 64 * 64);
    }
  }
  if (e == cudaSuccess && S->ring_k > 0)
    e = S->alloc(&S->ring, (size_t)S->ring_k * (size_t)S->ring_len * (size_t)mpmg_bytes_per_value(fprec));
  if (e == cudaSuccess && S->ring_k > 0) e = S->alloc(&S->ring_scale, (size_t)S->ring_k * 8);
  const int npart = std::max({S->nU, S->nD, norm2_partials(S->lv[F].len)});
  if (e == cudaSuccess) e = S->alloc(&S->partU, (size_t)npart * 8);
  if (e == cudaSuccess) e = S->alloc(&S->partD, (size_t)npart * 8);
  if (e == cudaSuccess) e = S->alloc(&S->st, sizeof(IrState));
  S->hist_cap = 1024;
  if (e == cudaSuccess) e = S->alloc(&S->hist, (size_t)S->hist_cap * 8);
  if (e == cudaSuccess) e = S->alloc(&S->final_d, 8);
  if (e == cudaSuccess) e = cudaMallocHost(&S->st_h, sizeof(IrState));
  if (e == cudaSuccess) e = cudaMallocHost(&S->final_h, 8);
  // coarse kernel arguments
  if (e == cudaSuccess && S->nc > 0) {
    CoarseArgs& A = S->cargs;
    A.nlev = S->nc;
    A.pre = c.pre_steps;
    A.post = c.post_steps;
    A.rescale = c.variant == MPMG_DSH_MG;
    A.base_tol = c.base_tol;
    A.base_mode = c.base_mode;
    A.base_maxit = c.base_max_iterations;
    // levels up to 512 unknowns (7^3) run on CTA 0 out of shared memory; a
    // grid-wide step (barrier-bound, ~2.5 us) beats one SM from 15^3 up
    A.cta_points = (int)env_ll("MPMG_CTA_POINTS", 512);
    A.debug = (int)env_ll("MPMG_COARSE_DEBUG", 0);
    A.dbg = nullptr;
    if (A.debug) e = S->alloc(&A.dbg, 64 * sizeof(long long));
    for (int l = 0; l < S->nc; ++l) {
      const Level& L = S->lv[l];
      CoarseLevel& C = A.lv[l];
      C.dim = c.dim; C.nodes = L.A.nodes; C.prec = L.A.prec;
      std::memcpy(C.taps, L.A.taps, sizeof(C.taps));
      C.inv_diag = L.A.inv_diag;
      C.omega = L.omega_r;
      C.u = L.u; C.u2 = L.u2; C.b = L.b; C.r = L.r; C.prod = L.prod;
    }
    const size_t b0 = S->lv[0].len * S->lv[0].bytes;
    e = S->alloc(&A.cg_r, b0);
    if (e == cudaSuccess) e = S->alloc(&A.cg_p, b0);
    if (e == cudaSuccess) e = S->alloc(&A.cg_ap, b0);
    if (e == cudaSuccess) e = S->alloc(&A.cg_s, b0);
    if (e == cudaSuccess) e = S->alloc(&A.cg_best, b0);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(S->s);
  if (e != cudaSuccess) {
    set_cuda_error(e);
    delete S;
    return fail(e == cudaErrorMemoryAllocation ? MPMG_ENOMEM : MPMG_ECUDA, -1);
  }
  return S;
}

void mpmg_solver_destroy(mpmg_solver* s) { delete s; }

int mpmg_solver_levels(const mpmg_solver* s) { return s ? (int)s->lv.size() : 0; }

int mpmg_solver_level_info(const mpmg_solver* s, int level, mpmg_stencil* out) {
  if (!s || !out || level < -1 || level >= (int)s->lv.size()) return MPMG_EINVAL;
  *out = level == -1 ? s->A64 : s->lv[level].A;
  return MPMG_OK;
}

size_t mpmg_solver_unknowns(const mpmg_solver* s) { return s ? mpmg_interior_len(s->cfg.dim, s->cfg.nodes) : 0; }

void* mpmg_solver_stream(mpmg_solver* s) { return s ? (void*)s->s : nullptr; }

int mpmg_solver_device_buffers(mpmg_solver* s, double** b_dev, double** u_dev) {
  if (!s) return MPMG_EINVAL;
  if (b_dev) *b_dev = s->b;
  if (u_dev) *u_dev = s->u;
  return MPMG_OK;
}

int mpmg_solver_solve_device(mpmg_solver* S, const double* b_dev, double* u_dev, const mpmg_solve_params* pp,
                             double* hist, int32_t hist_cap, mpmg_solve_report* rep) {
  clear_stale_error();
  if (!S || !pp || !(pp->outer_tolerance > 0.0) || pp->max_outer_iterations < 0) return MPMG_EINVAL;
  const mpmg_solve_params p = *pp;
  cudaStream_t q = S->s;
  if (p.max_outer_iterations + 1 > S->hist_cap) {  // history sized per solve (any max_outer_iterations)
    cudaError_t ea = cudaStreamSynchronize(q);
    if (ea == cudaSuccess) {
      S->allocs.erase(std::remove(S->allocs.begin(), S->allocs.end(), (void*)S->hist), S->allocs.end());
      ea = cudaFree(S->hist);
      S->hist = nullptr;
    }
    if (ea == cudaSuccess) ea = S->alloc(&S->hist, (size_t)(p.max_outer_iterations + 1) * 8);
    if (ea != cudaSuccess) return finish(ea);
    S->hist_cap = p.max_outer_iterations + 1;
    S->gvalid = false;  // the graph captured the old history pointer
  }
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaSuccess;
  if (b_dev && b_dev != S->b) e = cudaMemcpyAsync(S->b, b_dev, S->len * 8, cudaMemcpyDeviceToDevice, q);
  // D_MG with unit scale: r_low == r bitwise (cast_vector with scale 1 is a copy)
  const bool alias = S->lv.back().A.prec == MPMG_FP64 && !S->scale_enabled(p);
  if (alias != S->rlow_alias) {
    S->rlow_alias = alias;
    S->lv.back().b = alias ? (void*)S->r : S->rlow;
    if (S->nc == (int)S->lv.size()) S->cargs.lv[S->nc - 1].b = S->lv.back().b;
    S->gvalid = false;
  }
  if (e == cudaSuccess) e = cudaEventRecord(S->e0, q);
  bool graph_ok = false;
  cudaError_t gerr = cudaSuccess;
  if (e == cudaSuccess && p.use_graph) {
    if (!S->gvalid || !mpmg_solver::same_params(S->gkey, p)) gerr = S->build_graph(p);
    if (S->gvalid) {
      e = cudaGraphLaunch(S->exec, q);
      graph_ok = e == cudaSuccess;
    }
  }
  if (e == cudaSuccess && !graph_ok) {
    cudaGraphConditionalHandle none{};
    e = S->enqueue_init(p, q, none, 0);
    while (e == cudaSuccess) {
      e = cudaMemcpyAsync(S->st_h, S->st, sizeof(IrState), cudaMemcpyDeviceToHost, q);
      if (e == cudaSuccess) e = cudaStreamSynchronize(q);
      if (e != cudaSuccess || !S->st_h->active) break;
      e = S->enqueue_iteration(p, q, none, 0);
    }
    if (e == cudaSuccess) e = S->enqueue_final(q);
  }
  if (e == cudaSuccess) e = cudaEventRecord(S->e1, q);
  if (e == cudaSuccess && u_dev && u_dev != S->u) e = cudaMemcpyAsync(u_dev, S->u, S->len * 8, cudaMemcpyDeviceToDevice, q);
  if (e == cudaSuccess) e = cudaMemcpyAsync(S->st_h, S->st, sizeof(IrState), cudaMemcpyDeviceToHost, q);
  if (e == cudaSuccess) e = cudaMemcpyAsync(S->final_h, S->final_d, 8, cudaMemcpyDeviceToHost, q);
  if (e == cudaSuccess) e = cudaStreamSynchronize(q);
  if (e != cudaSuccess) return set_cuda_error(e);
  const IrState st = *S->st_h;
  if (hist && hist_cap > 0) {
    const int n = std::min(hist_cap, st.iterations + 1);
    e = cudaMemcpy(hist, S->hist, (size_t)n * 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return set_cuda_error(e);
  }
  if (rep) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, S->e0, S->e1);
    rep->converged = st.converged;
    rep->iterations = st.iterations;
    rep->final_residual = *S->final_h;
    rep->device_seconds = ms * 1e-3;
    rep->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rep->used_graph = graph_ok ? 1 : 0;
    rep->graph_error = (int32_t)gerr;
  }
  if (st.diverged) {
    last_error() = "ir_solve: non-finite residual norm at iteration " + std::to_string(st.iterations);
    return MPMG_ENONFINITE;
  }
  return MPMG_OK;
}

int mpmg_solver_solve(mpmg_solver* S, const double* b_host, double* u_host, const mpmg_solve_params* p,
                      double* hist, int32_t hist_cap, mpmg_solve_report* rep) {
  clear_stale_error();
  if (!S || !b_host) return MPMG_EINVAL;
  const auto t0 = std::chrono::steady_clock::now();
  const size_t n = mpmg_interior_len(S->cfg.dim, S->cfg.nodes);
  cudaStream_t q = S->s;
  // compact host rhs -> compact staging (the u buffer) -> padded b
  cudaError_t e = cudaMemcpyAsync(S->stage, b_host, n * 8, cudaMemcpyHostToDevice, q);
  if (e == cudaSuccess) e = launch_pack(S->cfg.dim, S->cfg.nodes, MPMG_FP64, S->stage, S->b, false, q);
  if (e != cudaSuccess) return set_cuda_error(e);
  int rc = mpmg_solver_solve_device(S, S->b, S->u, p, hist, hist_cap, rep);
  if (rc != MPMG_OK && rc != MPMG_ENONFINITE) return rc;
  if (u_host) {
    e = launch_pack(S->cfg.dim, S->cfg.nodes, MPMG_FP64, S->stage, S->u, true, q);
    if (e == cudaSuccess) e = cudaMemcpyAsync(u_host, S->stage, n * 8, cudaMemcpyDeviceToHost, q);
    if (e == cudaSuccess) e = cudaStreamSynchronize(q);
    if (e != cudaSuccess) return set_cuda_error(e);
  }
  if (rep) rep->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return rc;
}

}  // extern "C"

// ---- host value-domain helpers for the per-level test entry points --------
namespace {

cudaError_t upload_values(mpmg_solver* S, int dim, int nodes, int prec, const double* vals, void* padded) {
  const size_t n = mpmg_interior_len(dim, nodes);
  std::vector<unsigned char> host(n * 8);
  for (size_t i = 0; i < n; ++i) {
    if (prec == MPMG_FP16) reinterpret_cast<uint16_t*>(host.data())[i] = fp16_bits(vals[i]);
    else if (prec == MPMG_FP32) reinterpret_cast<float*>(host.data())[i] = (float)vals[i];
    else reinterpret_cast<double*>(host.data())[i] = vals[i];
  }
  void* stage = nullptr;
  cudaError_t e = cudaMalloc(&stage, std::max<size_t>(n * 8, 16));
  if (e == cudaSuccess) e = cudaMemcpyAsync(stage, host.data(), n * mpmg_bytes_per_value(prec), cudaMemcpyHostToDevice, S->s);
  if (e == cudaSuccess) e = launch_pack(dim, nodes, prec, stage, padded, false, S->s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(S->s);
  cudaFree(stage);
  return e;
}

cudaError_t download_values(mpmg_solver* S, int dim, int nodes, int prec, const void* padded, double* vals) {
  const size_t n = mpmg_interior_len(dim, nodes);
  std::vector<unsigned char> host(n * 8);
  void* stage = nullptr;
  cudaError_t e = cudaMalloc(&stage, std::max<size_t>(n * 8, 16));
  if (e == cudaSuccess) e = launch_pack(dim, nodes, prec, stage, const_cast<void*>(padded), true, S->s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(host.data(), stage, n * mpmg_bytes_per_value(prec), cudaMemcpyDeviceToHost, S->s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(S->s);
  cudaFree(stage);
  if (e != cudaSuccess) return e;
  for (size_t i = 0; i < n; ++i) {
    if (prec == MPMG_FP16) vals[i] = fp16_value(reinterpret_cast<uint16_t*>(host.data())[i]);
    else if (prec == MPMG_FP32) vals[i] = (double)reinterpret_cast<float*>(host.data())[i];
    else vals[i] = reinterpret_cast<double*>(host.data())[i];
  }
  return cudaSuccess;
}

}  // namespace

extern "C" {

int mpmg_solver_v_cycle(mpmg_solver* S, const double* b_host, double* c_host) {
  clear_stale_error();
  if (!S || !b_host || !c_host) return MPMG_EINVAL;
  Level& F = S->lv.back();
  // use the dedicated rlow buffer as the finest rhs
  void* saved = F.b;
  F.b = S->rlow;
  if (S->nc == (int)S->lv.size()) S->cargs.lv[S->nc - 1].b = F.b;
  S->gvalid = false;
  cudaError_t e = upload_values(S, F.A.dim, F.A.nodes, F.A.prec, b_host, F.b);
  void* c = nullptr;
  if (e == cudaSuccess) e = S->v_cycle(S->s, &c);
  if (e == cudaSuccess) e = download_values(S, F.A.dim, F.A.nodes, F.A.prec, c, c_host);
  F.b = saved;
  if (S->nc == (int)S->lv.size()) S->cargs.lv[S->nc - 1].b = saved;
  return finish(e);
}

int mpmg_solver_coarse_debug(mpmg_solver* S, long long* out, int32_t cap) {
  if (!S || !out || cap < 1) return MPMG_EINVAL;
  if (!S->cargs.dbg) return MPMG_EUNSUPPORTED;
  cudaError_t e = cudaStreamSynchronize(S->s);
  if (e == cudaSuccess) e = cudaMemcpy(out, S->cargs.dbg, (size_t)(cap < 64 ? cap : 64) * 8, cudaMemcpyDeviceToHost);
  return finish(e);
}

int mpmg_solver_v_cycle_device(mpmg_solver* S, const void* b_dev, void* c_dev, void* stream) {
  clear_stale_error();
  if (!S || !b_dev || !c_dev) return MPMG_EINVAL;
  Level& F = S->lv.back();
  const cudaStream_t q = stream ? (cudaStream_t)stream : S->s;
  void* saved = F.b;
  F.b = S->rlow;
  if (S->nc == (int)S->lv.size()) S->cargs.lv[S->nc - 1].b = F.b;
  S->gvalid = false;
  const size_t bytes = F.len * F.bytes;
  cudaError_t e = cudaMemcpyAsync(F.b, b_dev, bytes, cudaMemcpyDeviceToDevice, q);
  void* c = nullptr;
  if (e == cudaSuccess) e = S->v_cycle(q, &c);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c_dev, c, bytes, cudaMemcpyDeviceToDevice, q);
  F.b = saved;
  if (S->nc == (int)S->lv.size()) S->cargs.lv[S->nc - 1].b = saved;
  return finish(e);
}

// Per-level ops on host value-domain buffers (parity tests):
//  SPMV     out = A_l in0
//  JACOBI   out = `steps` Jacobi steps on A_l u = in1 from u = in0 (in0 NULL: from zero)
//  DEFECT   out = in1 - A_l in0
//  RESTRICT out (level l-1) = restrict(in0 at level l), product scale `scale`
//  PROLONG  out (level l) = in1 + round(scale * P in0), in0 at level l-1
//  COARSE_SOLVE out = CG solution of A_0 u = in0 (level must be 0)
int mpmg_solver_level_op(mpmg_solver* S, int op, int l, const double* in0, const double* in1, double* out,
                         int32_t steps, double scale) {
  clear_stale_error();
  if (!S || l < 0 || l >= (int)S->lv.size() || !out) return MPMG_EINVAL;
  Level& L = S->lv[l];
  const int dim = L.A.dim, nodes = L.A.nodes, prec = L.A.prec;
  cudaStream_t q = S->s;
  cudaError_t e = cudaSuccess;
  double* sdev = nullptr;
  switch (op) {
    case MPMG_OP_SPMV:
      e = upload_values(S, dim, nodes, prec, in0, L.u);
      if (e == cudaSuccess) {
        if (stencil_supported(dim, nodes, prec)) e = launch_level_op(0, L.A, L.u, nullptr, L.r, S->cfg.omega, S->policy(), q);
        else return MPMG_EUNSUPPORTED;
      }
      if (e == cudaSuccess) e = download_values(S, dim, nodes, prec, L.r, out);
      break;
    case MPMG_OP_DEFECT:
      if (!stencil_supported(dim, nodes, prec)) return MPMG_EUNSUPPORTED;
      e = upload_values(S, dim, nodes, prec, in0, L.u);
      if (e == cudaSuccess) e = upload_values(S, dim, nodes, prec, in1, L.b);
      if (e == cudaSuccess) e = launch_level_op(1, L.A, L.u, L.b, L.r, S->cfg.omega, S->policy(), q);
      if (e == cudaSuccess) e = download_values(S, dim, nodes, prec, L.r, out);
      break;
    case MPMG_OP_JACOBI: {
      if (!stencil_supported(dim, nodes, prec)) return MPMG_EUNSUPPORTED;
      e = upload_values(S, dim, nodes, prec, in1, L.b);
      void* cur = nullptr;
      if (e == cudaSuccess && in0) { e = upload_values(S, dim, nodes, prec, in0, L.u); cur = L.u; }
      int k = 0;
      if (e == cudaSuccess && !in0 && steps >= 2) {  // the fused first two steps (as in the V-cycle)
        e = launch_jacobi_zero2(L.A, L.b, L.u, L.u2, S->cfg.omega, L.omega_r, S->policy(), q);
        cur = L.u2;
        k = 2;
      }
      for (; k < steps && e == cudaSuccess; ++k) {
        void* o = (cur == L.u) ? L.u2 : L.u;
        if (!cur) e = launch_jacobi_zero(dim, nodes, prec, L.b, o, L.omega_r, L.A.inv_diag, S->policy(), q);
        else e = launch_level_op(2, L.A, cur, L.b, o, S->cfg.omega, S->policy(), q);
        cur = o;
      }
      if (!cur) { e = cudaMemsetAsync(L.u, 0, L.len * L.bytes, q); cur = L.u; }
      if (e == cudaSuccess) e = download_values(S, dim, nodes, prec, cur, out);
      break;
    }
    case MPMG_OP_RESTRICT: {
      if (l < 1) return MPMG_EINVAL;
      Level& C = S->lv[l - 1];
      e = upload_values(S, dim, nodes, prec, in0, L.r);
      if (e == cudaSuccess) e = cudaMalloc(&sdev, 8);
      if (e == cudaSuccess) e = cudaMemcpy(sdev, &scale, 8, cudaMemcpyHostToDevice);
      if (e == cudaSuccess)
        e = launch_restrict(dim, nodes, prec, C.A.prec, L.r, C.b, sdev, S->policy(), q);
      if (e == cudaSuccess) e = download_values(S, dim, C.A.nodes, C.A.prec, C.b, out);
      break;
    }
    case MPMG_OP_PROLONG: {
      if (l < 1) return MPMG_EINVAL;
      Level& C = S->lv[l - 1];
      e = upload_values(S, dim, C.A.nodes, C.A.prec, in0, C.u);
      if (e == cudaSuccess) e = upload_values(S, dim, nodes, prec, in1, L.u);
      if (e == cudaSuccess) e = cudaMalloc(&sdev, 8);
      if (e == cudaSuccess) e = cudaMemcpy(sdev, &scale, 8, cudaMemcpyHostToDevice);
      if (e == cudaSuccess)
        e = launch_prolong(dim, nodes, prec, C.A.prec, C.u, L.u, sdev, S->policy(), q);
      if (e == cudaSuccess) e = download_values(S, dim, nodes, prec, L.u, out);
      break;
    }
    case MPMG_OP_COARSE_SOLVE: {
      if (l != 0) return MPMG_EINVAL;
      CoarseArgs a = S->cargs;
      a.nlev = 1;
      e = upload_values(S, dim, nodes, prec, in0, L.b);
      if (e == cudaSuccess) e = launch_coarse_cycle(a, S->policy(), q);
      if (e == cudaSuccess) e = download_values(S, dim, nodes, prec, L.u, out);
      break;
    }
    default: return MPMG_EINVAL;
  }
  if (sdev) cudaFree(sdev);
  if (e == cudaSuccess) e = cudaStreamSynchronize(q);
  return finish(e);
}

}  // extern "C"
