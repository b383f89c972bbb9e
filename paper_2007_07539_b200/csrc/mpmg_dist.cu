// Multi-GPU z-slab solver: one process per GPU, the fine levels
// split into z-slabs, halos and the coarse rhs moved over NVLink / NVSwitch
// by peer-memory copies, the coarse levels agglomerated (replicated on every
// rank), the whole IR loop one CUDA graph with a device-side WHILE node on
// every rank -- no host round trip and no NCCL call per iteration.
//
// Peer memory: every rank allocates its buffers in ONE arena with the same
// layout on every rank (slabs sized for the largest slab), exports it with
// cudaIpcGetMemHandle and maps the other ranks' arenas (mpmg_dist_connect).
// A peer's copy of a buffer is then peer_base + (local offset). Ranks of the
// same process (tests) exchange raw pointers instead of IPC handles.
//
// Ordering: a sender copies boundary planes into the receivers' halo planes
// (cudaMemcpyAsync on mapped peer pointers -- copy engines over NVLink), then
// k_signal publishes a per-(sender, receiver) sequence number in the
// receiver's flag word (release, system scope); the receiver's k_wait
// spins until it sees the number it expects (acquire). Sequence counters live
// in device memory, so a captured graph replays correctly. Every exchange is
// a full handshake with both neighbours, so no rank runs more than one
// exchange ahead: a halo is never overwritten while its receiver still
// reads the previous one (write-after-read), nor read before it arrives.
//
// Determinism: per-point arithmetic does not depend on the rank count; the
// residual norm is each rank's fixed-order partial sum, published to every
// rank and summed in rank order -- alpha, the stopping decisions and the
// whole control flow are identical on all ranks and run to run.
//
// Reference: ir_solver.cpp:51-127 (the IR loop), multigrid.cpp:354-393 (the
// V-cycle) -- the same operations as the single-GPU solver (mpmg_solver.cu),
// slab-restricted (mpmg_gpu_slab_*).
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "mpmg_host.h"
#include "mpmg_internal.h"

using namespace mpmg_impl;

namespace {

constexpr int kMaxWorld = 64;

struct DState {  // device IR state (ir_solver.cpp:95-120)
  double alpha, scale;
  int iterations, converged, diverged, active, refresh_now, final_pending;
  int pending, fold_now;  // deferred corrections (as IrState, mpmg_solver.cu)
};

struct Comm {  // device-resident exchange bookkeeping (part of the arena)
  unsigned long long flags[kMaxWorld];   // written by the peers: their sequence number for us
  unsigned long long sent[kMaxWorld];    // our next sequence number per receiver
  unsigned long long expect[kMaxWorld];  // what we wait for per sender
  double slot[kMaxWorld];                // the ranks' partial sums of squares
};

__global__ void k_signal(Comm* self, Comm* const* peers, int rank, const int* to, int n) {
  // every copy enqueued before this kernel on the stream has completed
  __threadfence_system();
  for (int k = 0; k < n; ++k) {
    const int t = to[k];
    const unsigned long long v = ++self->sent[t];
    unsigned long long* f = &peers[t]->flags[rank];
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
  }
}

__global__ void k_wait(Comm* self, const int* from, int n) {
  for (int k = 0; k < n; ++k) {
    const int s = from[k];
    const unsigned long long want = ++self->expect[s];
    unsigned long long v;
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(&self->flags[s]) : "memory");
    } while (v < want);
  }
}

// this rank's partial sum (fixed order) -> every rank's slot[rank], then signal all
__global__ void k_publish(Comm* self, Comm* const* peers, int rank, int world, const double* part, int n,
                          const int* refresh_now, const double* part2, int n2) {
  __shared__ double red[256];
  const bool alt = refresh_now && *refresh_now;
  const double* p = alt ? part2 : part;
  const int m = alt ? n2 : n;
  double acc = 0.0;
  for (int i = threadIdx.x; i < m; i += 256) acc += p[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int t = 0; t < world; ++t) {
      double* d = t == rank ? &self->slot[rank] : &peers[t]->slot[rank];
      asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(d), "d"(red[0]) : "memory");
    }
    __threadfence_system();
    for (int t = 0; t < world; ++t) {
      if (t == rank) continue;
      const unsigned long long v = ++self->sent[t];
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&peers[t]->flags[rank]), "l"(v) : "memory");
    }
  }
}

// alpha = sqrt(sum of the ranks' slots in rank order); ir_solver.cpp:95-120
__global__ void k_dcontrol(DState* st, const Comm* self, int world, double* hist, int hist_cap, double tol,
                           int max_it, int scale_enabled, int refresh, int increment,
                           cudaGraphConditionalHandle cond, int use_cond, int ring_k) {
  double s = 0.0;
  for (int t = 0; t < world; ++t) s += self->slot[t];
  const double alpha = sqrt(s);
  // deferred corrections: this iteration parked one more c, or folded them all
  if (increment && ring_k > 0) st->pending = st->fold_now ? 0 : st->pending + 1;
  if (increment) st->iterations += 1;
  const int it = st->iterations;
  if (hist && it < hist_cap) hist[it] = alpha;
  st->alpha = alpha;
  int active = 0;
  if (!isfinite(alpha)) st->diverged = 1;
  else if (alpha < tol) st->converged = 1;
  else if (it < max_it) {
    active = 1;
    st->scale = (scale_enabled && alpha > 0.0) ? alpha : 1.0;  // ir_solver.cpp:109
  }
  st->active = active;
  st->refresh_now = (refresh > 0 && (it + 1) % refresh == 0) ? 1 : 0;
  // the next iteration folds the ring into u when it refreshes r or fills the ring
  st->fold_now = ring_k > 0 && (st->refresh_now || st->pending + 1 >= ring_k) ? 1 : 0;
  if (use_cond) cudaGraphSetConditional(cond, active ? 1u : 0u);
}

__global__ void k_dreset(DState* st) {
  st->alpha = 0.0;
  st->scale = 1.0;
  st->iterations = st->converged = st->diverged = st->active = st->refresh_now = 0;
  st->pending = st->fold_now = 0;
  st->final_pending = 1;
}

__global__ void k_dfinal(const Comm* self, int world, double* out) {
  double s = 0.0;
  for (int t = 0; t < world; ++t) s += self->slot[t];
  *out = sqrt(s);
}

int prec_of(int variant, int l) { return variant_precision(variant, l); }
int bytes_of(int prec) { return prec == MPMG_FP16 ? 2 : (prec == MPMG_FP32 ? 4 : 8); }

struct Blob {  // what a rank publishes for its peers
  int pid, device;
  size_t arena_bytes;
  void* raw;  // same-process ranks
  cudaIpcMemHandle_t handle;
};

}  // namespace

struct DLevel {
  int l = 0, P = 0, prec = 0, bytes = 0;
  mpmg_stencil A{};
  mpmg_slab s{};
  int nz_max = 0;
  size_t slab_len = 0;  // elements (sized for nz_max)
  size_t u = 0, u2 = 0, b = 0, r = 0;  // arena offsets
};

struct mpmg_dist {
  mpmg_solver_config cfg{};
  int rank = 0, world = 1, levels = 0, agg = -1, top = 0;
  std::vector<DLevel> lv;  // index = level (agg .. top used)
  mpmg_stencil A64{};
  mpmg_solver* coarse = nullptr;  // levels 0..agg, replicated
  unsigned char* arena = nullptr;
  size_t arena_bytes = 0;
  size_t off_comm = 0, off_bfull = 0, off_cfull = 0, off_u = 0, off_r = 0, off_b = 0;
  size_t full_len = 0;  // agg level padded length
  std::vector<unsigned char*> peer;  // peer arena bases (index = rank; own = arena)
  Comm** peers_dev = nullptr;        // device array of peer Comm pointers
  int* nb_dev = nullptr;             // device index lists: [lo, hi] neighbours, all others
  int n_lo_hi = 0, n_lo = 0, n_hi = 0, n_all = 0;
  int *lo_dev = nullptr, *hi_dev = nullptr, *all_dev = nullptr;
  double *partU = nullptr, *partD = nullptr;
  int nU = 0, nD = 0;
  // deferred corrections (binary16/32 finest level, as mpmg_solver.cu): the
  // iteration's c is parked in ring slot `pending` by UPDATE_R (r only) and
  // folded into the owned planes of u at a refresh, a full ring and the end
  int ring_k = 0;
  void* ring = nullptr;  // ring_k slots of ring_len values (the finest slab layout)
  long long ring_len = 0;
  double* ring_scale = nullptr;
  DState* st = nullptr;
  double* hist = nullptr;
  int hist_cap = 0;
  double* final_d = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaGraphExec_t exec = nullptr;
  mpmg_solve_params gkey{};
  bool gvalid = false;
  bool connected = false;
  bool fuse_halos = true;         // MPMG_DIST_FUSE_HALOS=0: kernel + copy exchange
  bool fuse_jz = true;            // MPMG_DIST_JZ=0: pointwise step 1 + stencil step 2
  int n_fused = 0, n_copied = 0;  // halo exchanges recorded in the last graph
  int n_kern_outer = -1, n_kern_body = -1;  // its kernel nodes: init + final, one iteration

  template <typename T = void>
  T* at(size_t off) { return reinterpret_cast<T*>(arena + off); }
  template <typename T = void>
  T* peer_at(int r, size_t off) { return reinterpret_cast<T*>(peer[r] + off); }
  Comm* comm() { return at<Comm>(off_comm); }
  uint32_t policy() const { return cfg.policy; }
  bool fma() const { return cfg.policy & MPMG_FMA; }

  ~mpmg_dist() {
    if (exec) cudaGraphExecDestroy(exec);
    if (coarse) mpmg_solver_destroy(coarse);
    for (int r = 0; r < (int)peer.size(); ++r)
      if (r != rank && peer[r] && peer_ipc[r]) cudaIpcCloseMemHandle(peer[r]);
    for (void* p : {(void*)ring, (void*)ring_scale, (void*)arena, (void*)peers_dev, (void*)lo_dev, (void*)hi_dev, (void*)all_dev, (void*)partU,
                    (void*)partD, (void*)st, (void*)hist, (void*)final_d})
      if (p) cudaFree(p);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (s) cudaStreamDestroy(s);
  }
  std::vector<int> peer_ipc;

  // slab of level l on rank q (SlabPlan, dist.py: chunk = P / world)
  mpmg_slab slab_of(int l, int q) const {
    const int P = lv[l].P, chunk = P / world;
    mpmg_slab t{};
    t.z_lo = std::max(1, q * chunk);
    t.nz = (q + 1) * chunk - t.z_lo;
    t.halo_lo = q > 0;
    t.halo_hi = q < world - 1;
    return t;
  }

  // halo exchange of buffer `off` of level l. fill_lo: every rank's bottom
  // halo plane (plane 0) receives its lower neighbour's last owned plane --
  // we send our last plane up and receive from below; fill_hi: every rank's
  // top halo plane (nz + 1) receives its upper neighbour's first owned plane.
  cudaError_t exchange(int l, size_t off, bool fill_lo, bool fill_hi, cudaStream_t q, int bytes = 0) {
    ++n_copied;
    const DLevel& L = lv[l];
    const size_t pl = (size_t)L.P * L.P * (bytes ? bytes : L.bytes);
    cudaError_t e = cudaSuccess;
    if (fill_lo && rank + 1 < world)  // our last owned plane -> upper neighbour's plane 0
      e = cudaMemcpyAsync(peer_at<unsigned char>(rank + 1, off), at<unsigned char>(off) + (size_t)L.s.nz * pl, pl,
                          cudaMemcpyDeviceToDevice, q);
    if (e == cudaSuccess && fill_hi && rank > 0) {  // our first owned plane -> lower neighbour's top halo
      const mpmg_slab t = slab_of(l, rank - 1);
      e = cudaMemcpyAsync(peer_at<unsigned char>(rank - 1, off) + (size_t)(t.nz + 1) * pl, at<unsigned char>(off) + pl,
                          pl, cudaMemcpyDeviceToDevice, q);
    }
    if (e != cudaSuccess) return e;
    return handshake(fill_lo, fill_hi, q);
  }

  // signal whom we wrote halos to, wait for whoever writes ours (see exchange)
  cudaError_t handshake(bool fill_lo, bool fill_hi, cudaStream_t q) {
    cudaError_t e = cudaSuccess;
    const int* to = fill_lo && fill_hi ? nb_dev : (fill_lo ? hi_dev : lo_dev);
    const int nto = fill_lo && fill_hi ? n_lo_hi : (fill_lo ? n_hi : n_lo);
    const int* from = fill_lo && fill_hi ? nb_dev : (fill_lo ? lo_dev : hi_dev);
    const int nfrom = fill_lo && fill_hi ? n_lo_hi : (fill_lo ? n_lo : n_hi);
    if (e == cudaSuccess && nto > 0) {
      k_signal<<<1, 1, 0, q>>>(comm(), peers_dev, rank, to, nto);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess && nfrom > 0) {
      k_wait<<<1, 1, 0, q>>>(comm(), from, nfrom);
      e = cudaGetLastError();
    }
    return e;
  }

  // a slab JACOBI (op 2) / DEFECT (op 1) of level l writing buffer `out`,
  // with the halo exchange fused into the kernel: its first / last owned
  // output planes are also stored straight into the neighbours' halo planes
  // (peer memory over NVLink), then only the handshake runs. Falls back to
  // the kernel + copy exchange where the fused kernel does not cover the level.
  cudaError_t op_push(int op, int l, size_t b, size_t in, size_t out, bool fill_lo, bool fill_hi, cudaStream_t q) {
    DLevel& L = lv[l];
    const size_t pl = (size_t)L.P * L.P * L.bytes;
    void* push_lo = nullptr;  // our first plane -> lower neighbour's top halo (fill_hi)
    void* push_hi = nullptr;  // our last plane -> upper neighbour's plane 0 (fill_lo)
    if (fill_hi && rank > 0) push_lo = peer_at<unsigned char>(rank - 1, out) + (size_t)(slab_of(l, rank - 1).nz + 1) * pl;
    if (fill_lo && rank + 1 < world) push_hi = peer_at<unsigned char>(rank + 1, out);
    cudaError_t e = cudaSuccess;
    bool done = false;
    if (fuse_halos) {
      if (L.prec == MPMG_FP16)
        done = plane_level_op_push_f16(op, L.A, at(in), at(b), at(out), cfg.omega, policy(), q, &e, &L.s, push_lo, push_hi);
      else if (L.prec == MPMG_FP32)
        done = plane_level_op_push_f32(op, L.A, at(in), at(b), at(out), cfg.omega, policy(), q, &e, &L.s, push_lo, push_hi);
      else
        done = plane_level_op_push_f64(op, L.A, at(in), at(b), at(out), cfg.omega, policy(), q, &e, &L.s, push_lo, push_hi);
    }
    if (done) {
      ++n_fused;
      return e == cudaSuccess ? handshake(fill_lo, fill_hi, q) : e;
    }
    const int rc = op == 2 ? mpmg_gpu_slab_jacobi(&L.A, &L.s, at(b), at(in), at(out), cfg.omega, policy(), q)
                           : mpmg_gpu_slab_defect(&L.A, &L.s, at(b), at(in), at(out), policy(), q);
    if (rc != MPMG_OK) return cudaErrorUnknown;
    return exchange(l, out, fill_lo, fill_hi, q);
  }

  // the agglomeration level: our owned planes of the restricted rhs into every
  // rank's full vector, then the replicated coarse V-cycle, then our slab of
  // the correction (owned planes and halos) from the full correction
  cudaError_t agglomerate(cudaStream_t q) {
    const DLevel& L = lv[agg];
    const size_t pl = (size_t)L.P * L.P * L.bytes;
    cudaError_t e = cudaSuccess;
    if (L.s.nz > 0) {
      for (int t = 0; t < world && e == cudaSuccess; ++t) {
        unsigned char* dst = (t == rank ? at<unsigned char>(off_bfull) : peer_at<unsigned char>(t, off_bfull)) +
                             (size_t)L.s.z_lo * pl;
        e = cudaMemcpyAsync(dst, at<unsigned char>(L.b) + pl, (size_t)L.s.nz * pl, cudaMemcpyDeviceToDevice, q);
      }
    }
    if (e == cudaSuccess && n_all > 0) {
      k_signal<<<1, 1, 0, q>>>(comm(), peers_dev, rank, all_dev, n_all);
      e = cudaGetLastError();
      if (e == cudaSuccess) {
        k_wait<<<1, 1, 0, q>>>(comm(), all_dev, n_all);
        e = cudaGetLastError();
      }
    }
    if (e == cudaSuccess) {
      const int rc = mpmg_solver_v_cycle_device(coarse, at(off_bfull), at(off_cfull), q);
      if (rc != MPMG_OK) return cudaErrorUnknown;
    }
    // planes z_lo - 1 .. z_lo + nz of the full correction = the slab with halos
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(at<unsigned char>(L.u), at<unsigned char>(off_cfull) + (size_t)(L.s.z_lo - 1) * pl,
                          (size_t)(L.s.nz + 2) * pl, cudaMemcpyDeviceToDevice, q);
    return e;
  }

  // V-cycle of the distributed levels (dist.py SlabSolver.cycle); returns the
  // offset of the buffer holding level l's correction (halos exchanged)
  cudaError_t cycle(int l, cudaStream_t q, size_t* res) {
    if (l == agg) {
      *res = lv[agg].u;
      return agglomerate(q);
    }
    DLevel& L = lv[l];
    size_t cur = L.u, other = L.u2;
    cudaError_t e = cudaSuccess;
    auto ok = [&](int rc) {
      if (rc != MPMG_OK && e == cudaSuccess) e = cudaErrorUnknown;
    };
    if (cfg.pre_steps > 0) {
      int done = 1;  // pre-smoothing steps taken
      bool jz = false;
      if (cfg.pre_steps >= 2 && fuse_jz) {
        // steps 1 + 2 from u = 0 in one JACOBI_Z sweep (u1 = w D^-1 b formed on
        // the fly from the staged b): needs b's halo planes instead of u1's
        e = exchange(l, L.b, true, true, q);
        cudaError_t pe = cudaSuccess;
        if (e == cudaSuccess) {
          if (L.prec == MPMG_FP16)
            jz = plane_level_op_f16(3, L.A, at(L.b), at(L.b), at(cur), cfg.omega, policy(), q, &pe, &L.s);
          else if (L.prec == MPMG_FP32)
            jz = plane_level_op_f32(3, L.A, at(L.b), at(L.b), at(cur), cfg.omega, policy(), q, &pe, &L.s);
          else
            jz = plane_level_op_f64(3, L.A, at(L.b), at(L.b), at(cur), cfg.omega, policy(), q, &pe, &L.s);
          if (jz) e = pe;
        }
        if (jz) done = 2;
      }
      if (!jz && e == cudaSuccess) ok(mpmg_gpu_slab_jacobi(&L.A, &L.s, at(L.b), nullptr, at(cur), cfg.omega, policy(), q));
      if (e == cudaSuccess) e = exchange(l, cur, true, true, q);
      for (int k = done; k < cfg.pre_steps && e == cudaSuccess; ++k) {
        e = op_push(2, l, L.b, cur, other, true, true, q);
        std::swap(cur, other);
      }
    } else {
      e = cudaMemsetAsync(at(cur), 0, L.slab_len * L.bytes, q);
    }
    if (e == cudaSuccess) e = op_push(1, l, L.b, cur, L.r, true, false, q);  // the restriction reads the lower halo
    DLevel& C = lv[l - 1];
    if (e == cudaSuccess && C.s.nz > 0)  // (an agglomeration slab may own no plane)
      ok(mpmg_gpu_slab_restrict(L.P + 1, &L.s, &C.s, L.prec, C.prec, at(L.r), at(C.b), policy(), q));
    size_t cc = 0;
    if (e == cudaSuccess) e = cycle(l - 1, q, &cc);
    if (e == cudaSuccess && l - 1 != agg) e = exchange(l - 1, cc, false, true, q);  // prolongation: upper halo
    if (e == cudaSuccess)
      ok(mpmg_gpu_slab_prolong_correct(L.P + 1, &L.s, &C.s, L.prec, C.prec, at(cc), at(cur), policy(), q));
    if (e == cudaSuccess) e = exchange(l, cur, true, true, q);
    for (int k = 0; k < cfg.post_steps && e == cudaSuccess; ++k) {
      e = op_push(2, l, L.b, cur, other, true, true, q);
      std::swap(cur, other);
    }
    *res = cur;
    return e;
  }

  int scale_enabled(const mpmg_solve_params& p) const {
    if (p.scaling == 1) return 1;
    if (p.scaling == 2) return 0;
    return cfg.variant != MPMG_D_MG;
  }

  cudaError_t publish_and_control(const mpmg_solve_params& p, cudaStream_t q, bool increment,
                                  cudaGraphConditionalHandle h, int use_cond, const double* part, int n,
                                  const double* part2, int n2, const int* alt) {
    k_publish<<<1, 256, 0, q>>>(comm(), peers_dev, rank, world, part, n, alt, part2, n2);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && n_all > 0) {
      k_wait<<<1, 1, 0, q>>>(comm(), all_dev, n_all);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
      k_dcontrol<<<1, 1, 0, q>>>(st, comm(), world, hist, hist_cap, p.outer_tolerance, p.max_outer_iterations,
                                 scale_enabled(p), p.residual_refresh_interval, increment ? 1 : 0, h, use_cond,
                                 ring_k);
      e = cudaGetLastError();
    }
    return e;
  }

  cudaError_t enqueue_init(const mpmg_solve_params& p, cudaStream_t q, cudaGraphConditionalHandle h, int use_cond) {
    k_dreset<<<1, 1, 0, q>>>(st);
    cudaError_t e = cudaGetLastError();
    const DLevel& F = lv[top];
    const size_t n = F.slab_len * 8;
    if (e == cudaSuccess) e = cudaMemsetAsync(at(off_u), 0, n, q);
    if (e == cudaSuccess && mpmg_gpu_slab_defect_f64(&A64, &F.s, at<double>(off_b), at<double>(off_u),
                                                     at<double>(off_r), partD, 0, q) != MPMG_OK)
      e = cudaErrorUnknown;
    if (e == cudaSuccess) e = publish_and_control(p, q, false, h, use_cond, partD, nD, partD, nD, nullptr);
    return e;
  }

  cudaError_t enqueue_iteration(const mpmg_solve_params& p, cudaStream_t q, cudaGraphConditionalHandle h,
                                int use_cond) {
    DLevel& F = lv[top];
    cudaError_t e = cudaSuccess;
    // cast_vector(r, mg precision, scale) over the owned planes (ir_solver.cpp:109-110;
    // b's halo planes belong to the neighbours' exchanges)
    {
      const size_t pl = (size_t)F.P * F.P;
      e = launch_downcast_len((size_t)F.s.nz * pl, at<double>(off_r) + pl, at<unsigned char>(F.b) + pl * F.bytes,
                              F.prec, &st->scale, 1, policy(), q);
      if (e != cudaSuccess) return e;
    }
    size_t c = 0;
    e = cycle(top, q, &c);
    // update_residuum_correction (ir_solver.cpp:112): c's halos are exchanged
    if (ring_k > 0) {  // r -= a A c now, u += a c deferred (bitwise the same u)
      if (e == cudaSuccess && !plane_update_r(A64, at(c), F.prec, at<double>(off_r), &st->scale, partU, ring,
                                              ring_len, &st->pending, ring_scale, fma(), q, &e, &F.s))
        e = cudaErrorNotSupported;
      if (e == cudaSuccess) e = fold(1, &st->fold_now, q);
    } else if (e == cudaSuccess && mpmg_gpu_slab_update_rc(&A64, &F.s, at(c), F.prec, at<double>(off_r),
                                                           at<double>(off_u), &st->scale, partU, policy(),
                                                           q) != MPMG_OK) {
      e = cudaErrorUnknown;
    }
    // the refresh r = b - A u every refresh-th iteration (ir_solver.cpp:115-119),
    // gated on the device; u's halos first
    if (e == cudaSuccess && p.residual_refresh_interval > 0) {
      e = exchange(top, off_u, true, true, q, 8);  // the FP64 iterate
      cudaError_t pe = cudaSuccess;
      if (e == cudaSuccess && !plane_defect64(A64, at<double>(off_b), at<double>(off_u), at<double>(off_r), partD,
                                              fma(), false, q, &st->refresh_now, &pe, &F.s))
        e = cudaErrorNotSupported;
      if (e == cudaSuccess) e = pe;
    }
    if (e == cudaSuccess) e = publish_and_control(p, q, true, h, use_cond, partU, nU, partD, nD, &st->refresh_now);
    return e;
  }

  // the parked corrections (+ this iteration's when extra = 1) into u's owned
  // planes only: a neighbour may be storing into u's halo planes meanwhile
  cudaError_t fold(int extra, const int* gate, cudaStream_t q) {
    const DLevel& F = lv[top];
    const size_t pl = (size_t)F.P * F.P;
    return launch_fold((size_t)F.s.nz * pl, at<double>(off_u) + pl,
                       static_cast<unsigned char*>(ring) + pl * bytes_of(F.prec), ring_len, F.prec, ring_scale,
                       &st->pending, extra, gate, fma(), q);
  }

  cudaError_t enqueue_final(cudaStream_t q) {  // residual_norm (ir_solver.cpp:21-49)
    const DLevel& F = lv[top];
    cudaError_t e = ring_k > 0 ? fold(0, nullptr, q) : cudaSuccess;  // corrections still parked
    if (e == cudaSuccess) e = exchange(top, off_u, true, true, q, 8);
    if (e == cudaSuccess && mpmg_gpu_slab_defect_f64(&A64, &F.s, at<double>(off_b), at<double>(off_u), nullptr,
                                                     partD, 1, q) != MPMG_OK)
      e = cudaErrorUnknown;
    if (e == cudaSuccess) {
      k_publish<<<1, 256, 0, q>>>(comm(), peers_dev, rank, world, partD, nD, nullptr, partD, nD);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess && n_all > 0) {
      k_wait<<<1, 1, 0, q>>>(comm(), all_dev, n_all);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
      k_dfinal<<<1, 1, 0, q>>>(comm(), world, final_d);
      e = cudaGetLastError();
    }
    return e;
  }

  // kernel nodes of a captured graph (top level: the WHILE node's body counted apart)
  static int kernel_nodes(cudaGraph_t gr) {
    size_t n = 0;
    if (cudaGraphGetNodes(gr, nullptr, &n) != cudaSuccess) { cudaGetLastError(); return -1; }
    std::vector<cudaGraphNode_t> nodes(n);
    if (n && cudaGraphGetNodes(gr, nodes.data(), &n) != cudaSuccess) { cudaGetLastError(); return -1; }
    int k = 0;
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType t;
      if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
    }
    return k;
  }

  cudaError_t build_graph(const mpmg_solve_params& p) {
    n_kern_outer = n_kern_body = -1;
    if (exec) { cudaGraphExecDestroy(exec); exec = nullptr; }
    gvalid = false;
    n_fused = n_copied = 0;
    cudaStream_t body_s = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&body_s, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
    cudaGraph_t g = nullptr;
    e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      cudaGraphConditionalHandle h{};
      cudaGraph_t cg = nullptr;
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
          if (e == cudaSuccess) n_kern_body = kernel_nodes(body);
        }
      }
      if (e == cudaSuccess) e = enqueue_final(s);
      cudaGraph_t out = nullptr;
      const cudaError_t e4 = cudaStreamEndCapture(s, &out);
      if (e == cudaSuccess) e = e4;
      g = e4 == cudaSuccess ? out : nullptr;
      if (g) n_kern_outer = kernel_nodes(g);
    }
    cudaStreamDestroy(body_s);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, g, 0);
    if (g) cudaGraphDestroy(g);
    if (e == cudaSuccess) {
      gkey = p;
      gvalid = true;
    } else {
      cudaGetLastError();
      exec = nullptr;
    }
    return e;
  }
};

namespace {
bool same_params(const mpmg_solve_params& a, const mpmg_solve_params& b) {
  return a.outer_tolerance == b.outer_tolerance && a.max_outer_iterations == b.max_outer_iterations &&
         a.scaling == b.scaling && a.residual_refresh_interval == b.residual_refresh_interval;
}
}  // namespace

extern "C" {

mpmg_dist* mpmg_dist_create(const mpmg_solver_config* cfg, int32_t rank, int32_t world, int32_t min_planes,
                            void* blob, size_t blob_cap, size_t* blob_len, int* err) {
  clear_stale_error();
  auto fail = [&](int code) -> mpmg_dist* {
    if (err) *err = code;
    return nullptr;
  };
  if (err) *err = MPMG_OK;
  if (!cfg || world < 1 || world > kMaxWorld || rank < 0 || rank >= world || !blob_len) return fail(MPMG_EINVAL);
  const mpmg_solver_config c = *cfg;
  if (c.dim != 3 || c.levels < 2 || c.levels > 30 || (c.nodes - 1) % (1 << (c.levels - 1)) != 0 ||
      ((c.nodes - 1) >> (c.levels - 1)) + 1 < 3 || c.variant == MPMG_DSH_MG)
    return fail(MPMG_EINVAL);
  if (min_planes < 1) min_planes = 4;
  *blob_len = sizeof(Blob);
  if (!blob || blob_cap < sizeof(Blob)) return fail(MPMG_EINVAL);
  cudaError_t e = cudaSetDevice(c.device);
  if (e != cudaSuccess) return fail(set_cuda_error(e));
  auto* D = new mpmg_dist();
  D->cfg = c;
  if (const char* fe = std::getenv("MPMG_DIST_FUSE_HALOS")) D->fuse_halos = std::atoi(fe) != 0;
  if (const char* je = std::getenv("MPMG_DIST_JZ")) D->fuse_jz = std::atoi(je) != 0;
  D->rank = rank;
  D->world = world;
  D->levels = c.levels;
  D->top = c.levels - 1;
  D->lv.resize(c.levels);
  const bool ftz = c.policy & MPMG_FTZ;
  // distributed levels: from the finest down while the pitch splits evenly
  // into >= min_planes planes per rank on a plane-kernel pitch (SlabPlan)
  for (int l = c.levels - 1; l >= 0; --l) {
    DLevel& L = D->lv[l];
    L.l = l;
    L.P = (c.nodes - 1) >> (c.levels - 1 - l);
    L.prec = prec_of(c.variant, l);
    L.bytes = bytes_of(L.prec);
    if (build_level_stencil(3, L.P + 1, L.prec, ftz, &L.A) != MPMG_OK) { delete D; return fail(MPMG_EBUILD); }
  }
  int agg = -1;
  for (int l = c.levels - 1; l >= 0; --l) {
    const int P = D->lv[l].P;
    if (!(P >= 32 && P <= 1024 && P % world == 0 && P / world >= min_planes)) { agg = l; break; }
  }
  if (agg < 0 || agg == c.levels - 1 || D->lv[agg].P % world != 0) { delete D; return fail(MPMG_EINVAL); }
  D->agg = agg;
  build_level_stencil(3, c.nodes, MPMG_FP64, ftz, &D->A64);
  // arena layout (identical on every rank: slabs sized for the largest slab)
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) / 256 * 256;
    return o;
  };
  D->off_comm = take(sizeof(Comm));
  for (int l = agg; l < c.levels; ++l) {
    DLevel& L = D->lv[l];
    L.s = D->slab_of(l, rank);
    L.nz_max = L.P / world;
    L.slab_len = mpmg_slab_len(L.P + 1, L.nz_max);
    const size_t bytes = L.slab_len * L.bytes;
    L.u = take(bytes); L.u2 = take(bytes); L.b = take(bytes); L.r = take(bytes);
  }
  const DLevel& A = D->lv[agg];
  D->full_len = mpmg_padded_len(3, A.P + 1);
  D->off_bfull = take(D->full_len * A.bytes);
  D->off_cfull = take(D->full_len * A.bytes);
  const size_t fl = D->lv[D->top].slab_len * 8;
  D->off_u = take(fl); D->off_r = take(fl); D->off_b = take(fl);
  D->arena_bytes = off;
  e = cudaMalloc(&D->arena, D->arena_bytes);
  if (e == cudaSuccess) e = cudaMemset(D->arena, 0, D->arena_bytes);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&D->s, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&D->e0);
  if (e == cudaSuccess) e = cudaEventCreate(&D->e1);
  // partial sums of the finest slab kernels
  const DLevel& F = D->lv[D->top];
  D->nU = std::max(1, mpmg_gpu_slab_partials_len(c.nodes, &F.s, F.prec, 1));
  D->nD = std::max(1, mpmg_gpu_slab_partials_len(c.nodes, &F.s, F.prec, 0));
  if (F.prec != MPMG_FP64) {
    const char* de = std::getenv("MPMG_DEFER_U");
    const int nr = (de && std::atoi(de) == 0) ? -1 : plane_update_r_partials(3, c.nodes, F.prec, F.s.nz + 1);
    if (nr > 0) {
      D->ring_k = 10;
      D->nU = nr;
      D->ring_len = (long long)((F.slab_len + 63) / 64 * 64);
    }
  }
  if (e == cudaSuccess && D->ring_k > 0) {
    const size_t rb = (size_t)D->ring_k * (size_t)D->ring_len * (size_t)F.bytes;
    e = cudaMalloc(&D->ring, rb);
    if (e == cudaSuccess) e = cudaMemset(D->ring, 0, rb);
    if (e == cudaSuccess) e = cudaMalloc(&D->ring_scale, (size_t)D->ring_k * 8);
  }
  const int np = std::max(D->nU, D->nD);
  if (e == cudaSuccess) e = cudaMalloc(&D->partU, np * 8);
  if (e == cudaSuccess) e = cudaMalloc(&D->partD, np * 8);
  if (e == cudaSuccess) e = cudaMalloc(&D->st, sizeof(DState));
  D->hist_cap = 1024;
  if (e == cudaSuccess) e = cudaMalloc(&D->hist, D->hist_cap * 8);
  if (e == cudaSuccess) e = cudaMalloc(&D->final_d, 8);
  if (e != cudaSuccess) { set_cuda_error(e); delete D; return fail(MPMG_ECUDA); }
  // the replicated coarse solver: levels 0..agg of the same variant
  mpmg_solver_config cc = c;
  cc.nodes = A.P + 1;
  cc.levels = agg + 1;
  int cerr = 0, clev = -1;
  D->coarse = mpmg_solver_create(&cc, &cerr, &clev);
  if (!D->coarse) { delete D; return fail(cerr ? cerr : MPMG_ECUDA); }
  Blob bl{};
  bl.pid = (int)getpid();
  bl.device = c.device;
  bl.arena_bytes = D->arena_bytes;
  bl.raw = D->arena;
  e = cudaIpcGetMemHandle(&bl.handle, D->arena);
  if (e != cudaSuccess) { cudaGetLastError(); std::memset(&bl.handle, 0, sizeof(bl.handle)); }
  std::memcpy(blob, &bl, sizeof(Blob));
  return D;
}

int mpmg_dist_connect(mpmg_dist* D, const void* blobs, size_t blob_len) {
  clear_stale_error();
  if (!D || !blobs || blob_len != sizeof(Blob)) return MPMG_EINVAL;
  const int W = D->world, R = D->rank;
  D->peer.assign(W, nullptr);
  D->peer_ipc.assign(W, 0);
  const int me = (int)getpid();
  for (int q = 0; q < W; ++q) {
    Blob b;
    std::memcpy(&b, static_cast<const unsigned char*>(blobs) + (size_t)q * sizeof(Blob), sizeof(Blob));
    if (b.arena_bytes != D->arena_bytes) return MPMG_EINVAL;  // every rank must lay out the same arena
    if (q == R) { D->peer[q] = D->arena; continue; }
    if (b.pid == me) {  // same process (tests): the pointer itself
      D->peer[q] = static_cast<unsigned char*>(b.raw);
      if (b.device != D->cfg.device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return set_cuda_error(e);
        cudaGetLastError();
      }
      continue;
    }
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return set_cuda_error(e);
    D->peer[q] = static_cast<unsigned char*>(p);
    D->peer_ipc[q] = 1;
  }
  // device tables: peer Comm pointers, neighbour lists
  std::vector<Comm*> pc(W);
  for (int q = 0; q < W; ++q) pc[q] = reinterpret_cast<Comm*>(D->peer[q] + D->off_comm);
  std::vector<int> lohi, lo, hi, all;
  if (R > 0) { lohi.push_back(R - 1); lo.push_back(R - 1); }
  if (R < W - 1) { lohi.push_back(R + 1); hi.push_back(R + 1); }
  for (int q = 0; q < W; ++q)
    if (q != R) all.push_back(q);
  D->n_lo_hi = (int)lohi.size(); D->n_lo = (int)lo.size(); D->n_hi = (int)hi.size(); D->n_all = (int)all.size();
  auto upload = [](const std::vector<int>& v, int** dst) -> cudaError_t {
    cudaError_t e = cudaMalloc(dst, std::max<size_t>(1, v.size()) * sizeof(int));
    if (e == cudaSuccess && !v.empty()) e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice);
    return e;
  };
  cudaError_t e = cudaMalloc(&D->peers_dev, W * sizeof(Comm*));
  if (e == cudaSuccess) e = cudaMemcpy(D->peers_dev, pc.data(), W * sizeof(Comm*), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = upload(lohi, &D->nb_dev);
  if (e == cudaSuccess) e = upload(lo, &D->lo_dev);
  if (e == cudaSuccess) e = upload(hi, &D->hi_dev);
  if (e == cudaSuccess) e = upload(all, &D->all_dev);
  if (e != cudaSuccess) return set_cuda_error(e);
  D->connected = true;
  return MPMG_OK;
}

void mpmg_dist_destroy(mpmg_dist* D) { delete D; }

int mpmg_dist_info(const mpmg_dist* D, int32_t* agg_level, int32_t* z_lo, int32_t* nz, size_t* slab_len) {
  if (!D) return MPMG_EINVAL;
  const DLevel& F = D->lv[D->top];
  if (agg_level) *agg_level = D->agg;
  if (z_lo) *z_lo = F.s.z_lo;
  if (nz) *nz = F.s.nz;
  if (slab_len) *slab_len = F.slab_len;
  return MPMG_OK;
}

int mpmg_dist_exchange_stats(const mpmg_dist* D, int32_t* fused, int32_t* copied) {
  if (!D) return MPMG_EINVAL;
  if (fused) *fused = D->n_fused;
  if (copied) *copied = D->n_copied;
  return MPMG_OK;
}

int mpmg_dist_graph_kernels(const mpmg_dist* D, int32_t* outer, int32_t* per_iteration) {
  if (!D || D->n_kern_outer < 0 || D->n_kern_body < 0) return MPMG_EINVAL;
  if (outer) *outer = D->n_kern_outer;
  if (per_iteration) *per_iteration = D->n_kern_body;
  return MPMG_OK;
}

int mpmg_dist_buffers(mpmg_dist* D, double** b_slab, double** u_slab) {
  if (!D) return MPMG_EINVAL;
  if (b_slab) *b_slab = D->at<double>(D->off_b);
  if (u_slab) *u_slab = D->at<double>(D->off_u);
  return MPMG_OK;
}

void* mpmg_dist_stream(mpmg_dist* D) { return D ? (void*)D->s : nullptr; }

int mpmg_dist_agg_buffers(mpmg_dist* D, void** b_full, void** c_full, size_t* len) {
  if (!D) return MPMG_EINVAL;
  if (b_full) *b_full = D->at(D->off_bfull);
  if (c_full) *c_full = D->at(D->off_cfull);
  if (len) *len = D->full_len;
  return MPMG_OK;
}

int mpmg_dist_prepare(mpmg_dist* D, const mpmg_solve_params* pp) {
  clear_stale_error();
  if (!D || !D->connected || !pp || !(pp->outer_tolerance > 0.0) || pp->max_outer_iterations < 0) return MPMG_EINVAL;
  const mpmg_solve_params p = *pp;
  if (p.max_outer_iterations + 1 > D->hist_cap) {
    cudaError_t e = cudaStreamSynchronize(D->s);
    if (e == cudaSuccess) e = cudaFree(D->hist);
    D->hist = nullptr;
    if (e == cudaSuccess) e = cudaMalloc(&D->hist, (size_t)(p.max_outer_iterations + 1) * 8);
    if (e != cudaSuccess) return set_cuda_error(e);
    D->hist_cap = p.max_outer_iterations + 1;
    D->gvalid = false;
  }
  if (!D->gvalid || !same_params(D->gkey, p)) {
    const cudaError_t e = D->build_graph(p);
    if (e != cudaSuccess) return set_cuda_error(e);
  }
  return MPMG_OK;
}

int mpmg_dist_solve_device(mpmg_dist* D, const mpmg_solve_params* pp, double* hist, int32_t hist_cap,
                           mpmg_solve_report* rep) {
  clear_stale_error();
  if (!D || !D->connected || !pp || !(pp->outer_tolerance > 0.0) || pp->max_outer_iterations < 0 ||
      pp->random_initial_guess)
    return MPMG_EINVAL;
  // (re)building the graph allocates and may synchronize the device: done
  // here only if the caller did not prepare this solve
  const int prc = mpmg_dist_prepare(D, pp);
  if (prc != MPMG_OK) return prc;
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaEventRecord(D->e0, D->s);
  if (e == cudaSuccess) e = cudaGraphLaunch(D->exec, D->s);
  if (e == cudaSuccess) e = cudaEventRecord(D->e1, D->s);
  DState st{};
  double fin = 0.0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&st, D->st, sizeof(DState), cudaMemcpyDeviceToHost, D->s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&fin, D->final_d, 8, cudaMemcpyDeviceToHost, D->s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(D->s);
  if (e != cudaSuccess) return set_cuda_error(e);
  if (hist && hist_cap > 0) {
    const int n = std::min(hist_cap, st.iterations + 1);
    e = cudaMemcpy(hist, D->hist, (size_t)n * 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return set_cuda_error(e);
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, D->e0, D->e1);
  if (rep) {
    rep->converged = st.converged;
    rep->iterations = st.iterations;
    rep->final_residual = fin;
    rep->device_seconds = ms * 1e-3;
    rep->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rep->used_graph = 1;
    rep->graph_error = 0;
  }
  if (st.diverged) {
    last_error() = "ir_solve: non-finite residual norm";
    return MPMG_ENONFINITE;
  }
  return MPMG_OK;
}

}  // extern "C"
