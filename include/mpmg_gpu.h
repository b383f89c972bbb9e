/* mpmg_gpu.h — C ABI of the B200-native mixed-precision IR + geometric
 * multigrid hot path (arxiv 2007.07539, BASELINE.json north_star).
 *
 * Two layers, both plain C (no torch or C++ types in any signature):
 *
 *  1. mpmg_gpu_*  — one entry point per fused sm_100a kernel family. Device
 *     pointers, sizes, a precision code, a policy word and a cudaStream_t
 *     (passed as void*). Asynchronous on the stream; never throws; returns
 *     MPMG_OK or a negative MPMG_E* code. Scalars that are produced on the
 *     device (alpha = ||r||, restriction scales) are passed as device pointers.
 *     These replace the reference's kernel layer (core/include/mpmg/kernels.hpp
 *     :11-38 and the level operations of multigrid.hpp:73-94); see each entry.
 *
 *  2. mpmg_solver_* — handle API over the whole hot path (hierarchy build,
 *     V-cycle, IR solve) with HOST buffers, mirroring MgHierarchy::build
 *     (multigrid.hpp:104-107), MgHierarchy::v_cycle (multigrid.hpp:119) and
 *     ir_solve (ir_solver.hpp:57-60). This is what an FFI (ctypes/cgo/JNI)
 *     binds; the C++ drop-in API (include/mpmg/ headers) is built on it.
 *
 * Device vector layout ("ghost-aliased pitch layout"). A level with n nodes
 * per dimension (boundary included) has pitch P = n - 1 and stores node
 * (x, y[, z]) with x, y, z in [0, P] at x + P*y (+ P*P*z). Node x = P of one
 * row aliases node x = 0 of the next row; both are Dirichlet boundary nodes,
 * stored as zero and never written, so the stencil needs no boundary
 * branches. Allocation: P^3 + P^2 + P + 1 (3D) or P^2 + P + 1 (2D) values.
 * The reference's compact interior ordering (mesh_fem.hpp:43-50, x fastest)
 * converts with mpmg_gpu_pack / mpmg_gpu_unpack.
 */
#ifndef MPMG_GPU_H
#define MPMG_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Precision codes == mpmg::Precision (precision.hpp:12). */
enum { MPMG_FP16 = 0, MPMG_FP32 = 1, MPMG_FP64 = 2 };

/* Variant codes == mpmg::MgVariant (multigrid.hpp:19). */
enum { MPMG_D_MG = 0, MPMG_H_MG = 1, MPMG_DSH_MG = 2, MPMG_HSD_MG = 3 };

/* Policy word: ArithmeticPolicy (precision.hpp:32-35) + Fp16Accum
 * (traffic.hpp:35). Reference default = MPMG_FTZ | MPMG_FMA. */
enum { MPMG_FTZ = 1u, MPMG_FMA = 2u, MPMG_ACC32 = 4u };

/* Return codes. */
enum {
  MPMG_OK = 0,
  MPMG_EINVAL = -1,      /* std::invalid_argument in the reference */
  MPMG_ENONFINITE = -2,  /* DivergedError / ValidationError */
  MPMG_ECUDA = -3,       /* CUDA runtime failure */
  MPMG_EBUILD = -4,      /* HierarchyBuildError (binary16 overflow) */
  MPMG_ENOMEM = -5,
  MPMG_EUNSUPPORTED = -6
};

/* One level's operator: the reference's per-level ELL matrix is a constant
 * stencil (every row's slot value for a given offset is bitwise identical,
 * SURVEY §8a-R0; checked against the reference in tests/test_hierarchy.py).
 * taps are lexicographic (dz, dy, dx), already rounded to `prec`. */
typedef struct mpmg_stencil {
  int32_t dim;      /* 2 or 3 */
  int32_t nodes;    /* nodes per dimension incl. boundary; pitch P = nodes-1 */
  int32_t prec;     /* storage == arithmetic precision of this level */
  int32_t ntaps;    /* 9 or 27 */
  double taps[27];  /* value domain, rounded to prec */
  double inv_diag;  /* Jacobi D^-1 (per-level constant), rounded to prec */
} mpmg_stencil;

/* A z-slab of a 3D level (multi-GPU slab decomposition): the
 * rank owns global interior planes z_lo .. z_lo+nz-1, stored as local planes
 * 1..nz of a slab array in the padded layout with one halo plane on each
 * side: local plane 0 = global z_lo-1, local plane nz+1 = global z_lo+nz.
 * A halo plane holds the neighbour's plane (halo_* = 1) or, at the domain
 * boundary, the zero Dirichlet ghost (halo_* = 0, never read). Allocation:
 * mpmg_slab_len values. A whole level is the slab {P-1, 1, 0, 0}. */
typedef struct mpmg_slab {
  int32_t nz;
  int32_t z_lo;
  int32_t halo_lo;
  int32_t halo_hi;
} mpmg_slab;

/* (nz + 2) P^2 + P + 1 */
size_t mpmg_slab_len(int32_t nodes, int32_t nz);

/* Number of values of a padded level vector. */
size_t mpmg_padded_len(int32_t dim, int32_t nodes);
/* Number of interior unknowns ((n-2)^dim). */
size_t mpmg_interior_len(int32_t dim, int32_t nodes);
/* Bytes per value of a precision code (precision.hpp:14-20). */
int mpmg_bytes_per_value(int32_t prec);

/* Last CUDA error string of this thread (for diagnostics). */
const char* mpmg_last_error(void);

/* ---- layer 1: kernels (device pointers, padded layout) -------------------*/

/* compact interior (reference ordering) <-> padded; ghosts written as zero */
int mpmg_gpu_pack(int32_t dim, int32_t nodes, int32_t prec, const void* compact, void* padded, void* stream);
int mpmg_gpu_unpack(int32_t dim, int32_t nodes, int32_t prec, const void* padded, void* compact, void* stream);

/* One damped-Jacobi step u_out = u_in + w D^-1 (b - A u_in), every operation
 * rounded to the level precision in the reference's order:
 * jacobi_smooth multigrid.cpp:79-89 = spmv (kernels.cpp:137-193), axpy(-1)
 * (:195-212), vec_multiply (:214-229), axpy(omega). u_in == NULL means the
 * step starts from u = 0 (multigrid.cpp:376). u_in and u_out must differ. */
int mpmg_gpu_jacobi(const mpmg_stencil* A, const void* b, const void* u_in, void* u_out, double omega,
                    uint32_t policy, void* stream);

/* Level defect r = b - A u in the level precision (multigrid.cpp:379-380). */
/* Steps 1 and 2 of jacobi_smooth from u = 0 (multigrid.cpp:376-377), as the
 * V-cycle's pre-smoother runs them: one fused pass over b where the plane /
 * row kernels cover the level (u1 = w D^-1 b formed on the fly), else the
 * pointwise first step into `tmp` and a streaming second step. */
int mpmg_gpu_jacobi_from_zero2(const mpmg_stencil* A, const void* b, void* tmp, void* u_out, double omega,
                               uint32_t policy, void* stream);
int mpmg_gpu_defect(const mpmg_stencil* A, const void* b, const void* u, void* r, uint32_t policy, void* stream);

/* y = A x in the level precision (kernels.cpp:137-193). */
int mpmg_gpu_spmv(const mpmg_stencil* A, const void* x, void* y, uint32_t policy, void* stream);

/* Full-weighting restriction with precision change (restrict_with_cast,
 * multigrid.cpp:236-268): r_c = round_{coarse_prec}(R r_f / scale), the
 * product accumulated in fine_prec with per-op rounding. `scale_dev` is a
 * device double (NULL = 1.0). fine grid has `fine_nodes` nodes per dim. */
int mpmg_gpu_restrict(int32_t dim, int32_t fine_nodes, int32_t fine_prec, int32_t coarse_prec, const void* r_fine,
                      void* r_coarse, const double* scale_dev, uint32_t policy, void* stream);

/* Prolongation + correction (prolong_with_cast multigrid.cpp:270-280 and
 * axpy(1) :389-390): u_f = round_f(u_f + round_f(scale * (P c_c))), P c_c in
 * coarse_prec with per-op rounding. `scale_dev` device double (NULL = 1.0). */
int mpmg_gpu_prolong_correct(int32_t dim, int32_t fine_nodes, int32_t fine_prec, int32_t coarse_prec,
                             const void* c_coarse, void* u_fine, const double* scale_dev, uint32_t policy,
                             void* stream);

/* Outer FP64 defect r = b - A u (ir_solver.cpp:92-93); when `partials` is
 * non-NULL also writes per-block partial sums of r_i^2 for mpmg_gpu_norm_finalize. */
int mpmg_gpu_defect_f64(const mpmg_stencil* A64, const double* b, const double* u, double* r, double* partials,
                        void* stream);

/* Fused update (update_residuum_correction kernels.cpp:300-341): u += a*c,
 * r -= a * A c, all FP64 with c (precision c_prec) widened on read. `alpha_dev`
 * is a device double. Optional norm partials of the new r. */
int mpmg_gpu_update_rc(const mpmg_stencil* A64, const void* c, int32_t c_prec, double* r, double* u,
                       const double* alpha_dev, double* partials, uint32_t policy, void* stream);

/* Deferred-correction halves of update_residuum_correction (kernels.cpp:
 * 300-341), as the solver runs them for binary16/32 finest levels:
 * update_r: r_i = fma(-alpha, (A c)_i, r_i) (+ partial sums of r_i^2 as in
 *   update_rc) and c copied into ring slot *slot_dev (ring_len values per
 *   slot, ring_len * bytes a multiple of 64), ring_scale[*slot_dev] = alpha.
 *   3D levels with pitch 32..1024 only (MPMG_EUNSUPPORTED otherwise).
 * fold: u_i = fma(ring_scale[k], c_k,i, u_i) for k = 0 .. *count_dev - 1 in
 *   order -- bitwise the u half of the per-iteration update. len = padded
 *   length of u. */
int mpmg_gpu_update_r(const mpmg_stencil* A64, const void* c, int32_t c_prec, double* r, const double* alpha_dev,
                      double* partials, void* ring, int64_t ring_len, const int32_t* slot_dev, double* ring_scale,
                      uint32_t policy, void* stream);
int mpmg_gpu_update_r_partials(int32_t dim, int32_t nodes, int32_t c_prec);
/* The last finest post-smoothing step of a deferred-correction cycle
 * (jacobi_smooth, multigrid.cpp:79-89, one step): u_out = the Jacobi step of
 * u_in written straight into ring slot *slot_dev (ring + *slot_dev *
 * ring_len values), where update_r then reads c. binary16/32 3D levels with
 * pitch 32..1024 and FMA on; MPMG_EUNSUPPORTED otherwise. */
int mpmg_gpu_jacobi_slot(const mpmg_stencil* A, const void* b, const void* u_in, void* ring, int64_t ring_len,
                         const int32_t* slot_dev, double omega, uint32_t policy, void* stream);
int mpmg_gpu_fold(int64_t len, double* u, const void* ring, int64_t ring_len, int32_t c_prec,
                  const double* ring_scale, const int32_t* count_dev, uint32_t policy, void* stream);

/* Scaled downcast (cast_vector kernels.cpp:343-360): out = round_prec(x / s)
 * with s = *alpha_dev if (scale_enabled && *alpha_dev > 0) else 1. */
int mpmg_gpu_scale_downcast(int32_t dim, int32_t nodes, const double* x, void* out, int32_t prec,
                            const double* alpha_dev, int32_t scale_enabled, uint32_t policy, void* stream);

/* Number of partial sums written by the partial-producing kernels. */
int mpmg_gpu_partials_len(int32_t dim, int32_t nodes);
/* Norm of a padded FP64 vector: deterministic two-stage reduction (fixed
 * block partition, fixed-order final sum). Writes sqrt(sum) to *out_dev. */
int mpmg_gpu_norm2_f64(int32_t dim, int32_t nodes, const double* x, double* partials, double* out_dev,
                       void* stream);
int mpmg_gpu_norm_finalize(const double* partials, int32_t n_partials, double* out_dev, void* stream);

/* ---- z-slab kernels (3D; pitch P = nodes-1 in {32,...,1024}) ------------
 * Same arithmetic as the whole-level entry points above, restricted to the
 * slab's owned planes; halo planes must have been exchanged beforehand. */

/* one Jacobi step on the owned planes; u_in NULL = first step from zero
 * (pointwise, owned planes only -- the halo planes are left to the exchange) */
int mpmg_gpu_slab_jacobi(const mpmg_stencil* A, const mpmg_slab* s, const void* b, const void* u_in, void* u_out,
                         double omega, uint32_t policy, void* stream);
int mpmg_gpu_slab_defect(const mpmg_stencil* A, const mpmg_slab* s, const void* b, const void* u, void* r,
                         uint32_t policy, void* stream);
/* coarse slab sc from fine slab sf (needs the fine LOWER halo of r_fine);
 * product accumulated in fine_prec, stored in coarse_prec (scale 1) */
int mpmg_gpu_slab_restrict(int32_t fine_nodes, const mpmg_slab* sf, const mpmg_slab* sc, int32_t fine_prec,
                           int32_t coarse_prec, const void* r_fine, void* r_coarse, uint32_t policy, void* stream);
/* u_fine += P c_coarse on the fine owned planes (needs the coarse UPPER halo) */
int mpmg_gpu_slab_prolong_correct(int32_t fine_nodes, const mpmg_slab* sf, const mpmg_slab* sc, int32_t fine_prec,
                                  int32_t coarse_prec, const void* c_coarse, void* u_fine, uint32_t policy,
                                  void* stream);
/* FP64 defect r = b - A u of the owned planes + per-CTA sums of r^2
 * (resnorm != 0: the residual_norm form b - s, no store) */
int mpmg_gpu_slab_defect_f64(const mpmg_stencil* A64, const mpmg_slab* s, const double* b, const double* u,
                             double* r, double* partials, int32_t resnorm, void* stream);
int mpmg_gpu_slab_update_rc(const mpmg_stencil* A64, const mpmg_slab* s, const void* c, int32_t c_prec, double* r,
                            double* u, const double* alpha_dev, double* partials, uint32_t policy, void* stream);
/* out = round(x / alpha) over the whole local slab array */
int mpmg_gpu_slab_scale_downcast(int32_t nodes, const mpmg_slab* s, const double* x, void* out, int32_t prec,
                                 const double* alpha_dev, int32_t scale_enabled, uint32_t policy, void* stream);
/* partial sums written by slab_defect_f64 (update = 0) or slab_update_rc
 * (update = 1, c precision c_prec) */
int mpmg_gpu_slab_partials_len(int32_t nodes, const mpmg_slab* s, int32_t c_prec, int32_t update);
/* *out_dev = sum of partials[0..n) in index order (no square root) */
int mpmg_gpu_partials_sum(const double* partials, int32_t n, double* out_dev, void* stream);

/* ---- generic ELLPACK path (from_levels hierarchies, public kernel API) ----
 * Device matrices are SLOT-MAJOR: val[s*rows + r], col[s*rows + r] (the
 * reference's row-major EllMatrix, ell_matrix.hpp:18-74, transposed on
 * upload so that a warp's 32 rows read one coalesced segment per slot).
 * Vectors are dense device arrays in their storage precision. */

/* y = A x in precision prec, per-slot rounding in slot order (spmv_impl,
 * kernels.cpp:137-193); MPMG_ACC32 in `policy` selects Fp16Accum::FP32 for
 * binary16 data. x and y must differ (kernels.cpp:248). */
int mpmg_gpu_ell_spmv(int64_t rows, int32_t rw, const int32_t* col, const void* val, int32_t prec, const void* x,
                      void* y, uint32_t policy, void* stream);
/* out = y + round(alpha) x (axpy_impl, kernels.cpp:195-212); out may alias */
int mpmg_gpu_axpy(int64_t n, int32_t prec, double alpha, const void* x, const void* y, void* out, uint32_t policy,
                  void* stream);
/* out = a .* b (vec_multiply_impl, kernels.cpp:214-229); out may alias */
int mpmg_gpu_vec_multiply(int64_t n, int32_t prec, const void* a, const void* b, void* out, uint32_t policy,
                          void* stream);
/* transfer_product + store_scaled (multigrid.cpp:155-232): the product M x in
 * x's precision (matrix values re-rounded to it), then out = round_out(prod /
 * scale) when divide != 0 (restriction) or round_out(prod * scale)
 * (prolongation). scale_dev NULL = 1. prod (optional, binary64) receives the
 * products for the DSH rescale norm. */
int mpmg_gpu_ell_transfer(int64_t rows, int32_t rw, const int32_t* col, const void* val, int32_t mat_prec,
                          const void* x, int32_t x_prec, int32_t out_prec, const double* scale_dev, int32_t divide,
                          void* out, double* prod, uint32_t policy, void* stream);
/* update_residuum_correction on a generic binary64 ELL (kernels.cpp:300-341) */
int mpmg_gpu_ell_update_rc(int64_t rows, int32_t rw, const int32_t* col, const double* val, const void* c,
                           int32_t c_prec, double* r, double* u, const double* alpha_dev, uint32_t policy,
                           void* stream);
/* cast_vector (kernels.cpp:343-360): out = round_out(x / s), s = *scale_dev
 * when non-NULL else `scale` (must be positive and finite) */
int mpmg_gpu_cast(int64_t n, const void* x, int32_t x_prec, void* out, int32_t out_prec, const double* scale_dev,
                  double scale, uint32_t policy, void* stream);
/* dot_fp64 / norm2_fp64 (kernels.cpp:368-395): sequential fma accumulation in
 * index order on one device thread -- bitwise the reference's value. */
/* Validate mode (ExecContext::validate; kernels.cpp:90-113 validate_finite,
 * multigrid.cpp:259-265): *index = the smallest i with x[i] non-finite (NaN
 * or +-inf; binary16: exponent field all ones), or -1. Synchronous on
 * `stream` (the result is a host value). */
int mpmg_gpu_find_nonfinite(int64_t n, const void* x, int32_t x_prec, int64_t* index, void* stream);
int mpmg_gpu_dot_seq(int64_t n, const void* x, int32_t x_prec, const void* y, int32_t y_prec, double* out_dev,
                     int32_t take_sqrt, void* stream);

/* ---- device memory helpers for FFI hosts (the C++ drop-in layer, ctypes)
 * All synchronous on the legacy default stream (stream argument NULL of the
 * kernel entry points). */
int mpmg_dev_count(void);                                    /* CUDA devices visible */
void* mpmg_dev_alloc(size_t bytes);                          /* NULL on failure */
void mpmg_dev_free(void* p);
int mpmg_dev_h2d(void* dst_dev, const void* src_host, size_t bytes);
int mpmg_dev_d2h(void* dst_host, const void* src_dev, size_t bytes);
int mpmg_dev_memset0(void* p, size_t bytes);
int mpmg_dev_sync(void);

/* The per-level operator of MgHierarchy::build (multigrid.cpp:290-310) for a
 * grid of `nodes` nodes per dimension in precision `prec`: the assembled Q1
 * coefficients (mesh_fem.cpp:71-155) rounded per policy, and D^-1. Returns
 * MPMG_EBUILD on binary16 overflow (cast_checked, multigrid.cpp:25-33). */
int mpmg_build_stencil(int32_t dim, int32_t nodes, int32_t prec, uint32_t policy, mpmg_stencil* out);

/* quantize_fp16 (precision.cpp:23-48) on the host. */
double mpmg_round_fp16(double x, int32_t ftz);

/* ---- layer 2: solver handle (host buffers) --------------------------------*/

typedef struct mpmg_solver mpmg_solver;

typedef struct mpmg_solver_config {
  int32_t dim, k, nodes, levels, variant;
  int32_t pre_steps, post_steps;  /* SmootherConfig (multigrid.hpp:31-35) */
  double omega;
  double base_tol;                /* BaseSolverConfig (multigrid.hpp:41-46) */
  int32_t base_mode;              /* 0 RelativeToRhs, 1 Absolute */
  int32_t base_max_iterations;    /* 0 = 10 x base unknowns */
  uint32_t policy;                /* MPMG_FTZ | MPMG_FMA | MPMG_ACC32 */
  int32_t device;
} mpmg_solver_config;

typedef struct mpmg_solve_params {   /* IrConfig (ir_solver.hpp:12-24) */
  double outer_tolerance;            /* absolute ||r||_2 bound */
  int32_t max_outer_iterations;
  int32_t random_initial_guess;      /* InitialGuess::SeededRandom01 */
  uint64_t seed;
  int32_t scaling;                   /* 0 VariantDefault, 1 ForceOn, 2 ForceOff */
  int32_t residual_refresh_interval;
  int32_t use_graph;                 /* capture the loop as one CUDA graph */
} mpmg_solve_params;

typedef struct mpmg_solve_report {   /* SolveReport (ir_solver.hpp:26-44) */
  int32_t converged;
  int32_t iterations;
  double final_residual;
  double device_seconds;             /* CUDA-event time of the solve */
  double wall_seconds;
  int32_t used_graph;                /* 1: the solve ran as one CUDA graph */
  int32_t graph_error;               /* cudaError_t of a failed graph build (0: none) */
} mpmg_solve_report;

void mpmg_solver_default_config(mpmg_solver_config* cfg);
void mpmg_solve_default_params(mpmg_solve_params* p);

/* Builds the device-resident hierarchy (MgHierarchy::build semantics) and
 * the FP64 finest operator. Returns NULL on error; *err receives the code and
 * *err_level the offending level for MPMG_EBUILD. */
mpmg_solver* mpmg_solver_create(const mpmg_solver_config* cfg, int* err, int* err_level);
void mpmg_solver_destroy(mpmg_solver* s);

int mpmg_solver_levels(const mpmg_solver* s);
int mpmg_solver_level_info(const mpmg_solver* s, int level, mpmg_stencil* out);
size_t mpmg_solver_unknowns(const mpmg_solver* s);
void* mpmg_solver_stream(mpmg_solver* s);

/* Manufactured right-hand side of the problem (assemble_rhs, mesh_fem.cpp:
 * 157-202), computed on the host in binary64, compact ordering. */
int mpmg_problem_rhs(int32_t dim, int32_t nodes, int32_t k, double* b_out);

/* ir_solve with host buffers (b compact FP64 in, u compact FP64 out). The
 * residual history (iterations+1 entries) is written when hist != NULL. */
int mpmg_solver_solve(mpmg_solver* s, const double* b_host, double* u_host, const mpmg_solve_params* p,
                      double* hist, int32_t hist_cap, mpmg_solve_report* rep);

/* The solver's own device-resident padded FP64 rhs and solution buffers. */
int mpmg_solver_device_buffers(mpmg_solver* s, double** b_dev, double** u_dev);

/* Same, on device-resident padded FP64 vectors (b_dev, u_dev); passing the
 * solver's own buffers (mpmg_solver_device_buffers) avoids any copy. */
int mpmg_solver_solve_device(mpmg_solver* s, const double* b_dev, double* u_dev, const mpmg_solve_params* p,
                             double* hist, int32_t hist_cap, mpmg_solve_report* rep);

/* One V-cycle on host buffers: b, c compact in the finest level precision,
 * passed as binary64 value-domain arrays (MgHierarchy::v_cycle). */
int mpmg_solver_v_cycle(mpmg_solver* s, const double* b_host, double* c_host);

/* Diagnostics: per-phase clock64 stamps of the last coarse-kernel run
 * (solver created with MPMG_COARSE_DEBUG=1 in the environment). out[0] =
 * count, out[1..] = (phase*100 + level) * 1e12 + cycles. */
int mpmg_solver_coarse_debug(mpmg_solver* s, long long* out, int32_t cap);

/* One V-cycle on device buffers: b_dev, c_dev padded arrays of the finest
 * level's precision, on `stream` (NULL: the solver's stream). Used by the
 * multi-GPU driver for the agglomerated coarse levels. */
int mpmg_solver_v_cycle_device(mpmg_solver* s, const void* b_dev, void* c_dev, void* stream);

/* Per-level operations on host value-domain buffers (for parity tests of the
 * level kernels through the same device code the solver runs). */
int mpmg_solver_level_op(mpmg_solver* s, int op, int level, const double* in0, const double* in1, double* out,
                         int32_t steps, double scale);
enum { MPMG_OP_SPMV = 0, MPMG_OP_JACOBI = 1, MPMG_OP_DEFECT = 2, MPMG_OP_RESTRICT = 3, MPMG_OP_PROLONG = 4,
       MPMG_OP_COARSE_SOLVE = 5 };

/* ---- multi-GPU z-slab solver (one process per GPU) -------------------------
 * SURVEY §8e; no reference counterpart (the reference is single-threaded,
 * multigrid.hpp:96-98). The fine levels are split into z-slabs over `world`
 * ranks (while the pitch splits into >= min_planes planes per rank), the
 * coarser levels are agglomerated: every rank gathers the restricted rhs of
 * the agglomeration level over peer memory and runs the coarse V-cycle
 * itself (replicated, bitwise identical). Halos, the gather and the norm
 * partials move by peer-memory copies / stores over NVLink (CUDA IPC handles;
 * raw pointers between ranks of one process) with device-side sequence flags;
 * a solve is one CUDA graph with a device WHILE loop per rank.
 *   create : builds rank `rank`'s buffers and writes its exchange blob
 *            (*blob_len bytes) -- transport it to every rank (any channel);
 *   connect: all ranks' blobs concatenated in rank order;
 *   buffers: this rank's FP64 rhs / solution slabs (local planes 0..nz+1 of
 *            the finest level, P^2 values each; owned planes 1..nz are global
 *            planes z_lo..z_lo+nz-1); fill b's owned planes before a solve;
 *   solve  : every rank calls it; same params on all ranks. u0 = 0 only.
 * Variants D_MG / H_MG / HSD_MG (no DSH rescaling); 3D. */
typedef struct mpmg_dist mpmg_dist;
mpmg_dist* mpmg_dist_create(const mpmg_solver_config* cfg, int32_t rank, int32_t world, int32_t min_planes,
                            void* blob, size_t blob_cap, size_t* blob_len, int* err);
int mpmg_dist_connect(mpmg_dist* d, const void* blobs, size_t blob_len);
void mpmg_dist_destroy(mpmg_dist* d);
int mpmg_dist_info(const mpmg_dist* d, int32_t* agg_level, int32_t* z_lo, int32_t* nz, size_t* slab_len);
int mpmg_dist_buffers(mpmg_dist* d, double** b_slab, double** u_slab);
/* halo exchanges recorded in the last captured solve graph: those fused into
 * the producing slab kernel (stores into the neighbours' halo planes) and
 * those done as kernel + peer copy (MPMG_DIST_FUSE_HALOS=0, or levels the
 * fused kernel does not cover: pitch <= 64, FP64 u, agglomeration) */
int mpmg_dist_exchange_stats(const mpmg_dist* d, int32_t* fused, int32_t* copied);
/* kernel launches of the captured solve graph: init + final (outer) and one
 * IR iteration (the WHILE body); a solve of k iterations launches
 * outer + k * per_iteration kernels. MPMG_EINVAL before the graph exists. */
int mpmg_dist_graph_kernels(const mpmg_dist* d, int32_t* outer, int32_t* per_iteration);
void* mpmg_dist_stream(mpmg_dist* d);
/* the agglomeration level's replicated rhs / correction (full padded vectors
 * in that level's precision), after a solve: the last cycle's */
int mpmg_dist_agg_buffers(mpmg_dist* d, void** b_full, void** c_full, size_t* len);
/* builds (captures) the solve graph for these params without running it --
 * allocation and capture may synchronize the device, so ranks sharing one
 * GPU (tests) prepare before any of them solves */
int mpmg_dist_prepare(mpmg_dist* d, const mpmg_solve_params* p);
int mpmg_dist_solve_device(mpmg_dist* d, const mpmg_solve_params* p, double* hist, int32_t hist_cap,
                           mpmg_solve_report* rep);

#ifdef __cplusplus
}
#endif
#endif /* MPMG_GPU_H */
