/* TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
 *
 * Plain-C restatement of the reference (arxiv 2007.07539 `mpmg`, C++20 at
 * /root/reference/proj/core) for the hot path named by BASELINE.json:
 * FP64 iterative refinement around a mixed-precision geometric-multigrid
 * V-cycle. Every function cites the reference file:line it restates.
 *
 * Pinning: tests/test_oracle_*.py check this restatement against (1) the
 * reference's own known-answer tests (proj/tests/test_precision.cpp,
 * test_kernels.cpp), restated, and (2) the unmodified reference compiled by
 * oracle/Makefile into oracle/_ref/libmpmg_ref.so, bitwise, plus committed
 * golden fixtures generated from it (tests/golden/make_golden.py).
 *
 * Representation: vectors are binary64 arrays in the "value domain" (every
 * binary16 / binary32 value is exact in binary64) tagged with a precision;
 * ELLPACK matrices are row-major (row*rw+slot) like ell_matrix.hpp:18-74.
 */
#ifndef MPMG_ORACLE_H
#define MPMG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_FP16 = 0, ORC_FP32 = 1, ORC_FP64 = 2 };
enum { ORC_D_MG = 0, ORC_H_MG = 1, ORC_DSH_MG = 2, ORC_HSD_MG = 3 };

typedef struct {
  int ftz;   /* ArithmeticPolicy::flush_subnormals_to_zero (precision.hpp:32-35) */
  int fma;   /* ArithmeticPolicy::fused_multiply_add */
  int acc32; /* ExecContext::fp16_accumulation == FP32 (traffic.hpp:35-44) */
} orc_ctx;

typedef struct {
  int64_t rows, cols;
  int rw, prec;
  int32_t* col;
  double* val; /* value domain, already rounded to prec */
  /* implicit operators (col == val == NULL): rows are generated on demand in
   * exactly the slot order and padding of the assembled ELL (mesh_fem.cpp:
   * 124-150, 204-295; ell_matrix.cpp:26-28, 90-92), so a 257^3 or larger
   * level needs no multi-GB slot arrays. gen: 0 explicit, 1 stiffness A,
   * 2 prolongation P, 3 restriction R; gdim/gn: dimension and the node
   * count of the row grid (A), or of the FINE grid (P, R); gtaps: the
   * per-offset coefficients (A: the level stencil, rounded to prec). */
  int gen, gdim, gn;
  double gtaps[27];
} orc_ell;

/* precision.cpp */
double orc_quantize_fp16(double x, int ftz);
double orc_fp16_fma(double a, double b, double c, int ftz, int fma);
double orc_fp16_add(double a, double b, int ftz);
double orc_fp16_mul(double a, double b, int ftz);
unsigned orc_pack_fp16(double v);
double orc_widen_fp16(unsigned bits);
float orc_ftz_fp32(float v, int ftz);
double orc_round(double v, int prec, int ftz);

/* ell_matrix.cpp */
int orc_ell_alloc(orc_ell* m, int64_t rows, int64_t cols, int rw, int prec);
void orc_ell_free(orc_ell* m);
/* row r of any (explicit or implicit) ELL: rw columns and values */
void orc_ell_row(const orc_ell* m, int64_t r, int32_t* cols, double* vals);
void orc_ell_rows(const orc_ell* m, int32_t* cols, double* vals); /* all rows, row-major */

/* kernels.cpp */
void orc_spmv(const orc_ell* A, const double* x, double* y, orc_ctx ctx);
void orc_spmv_rows(const orc_ell* A, const double* x, double* y, int64_t r0, int64_t r1, orc_ctx ctx);
void orc_transfer_rows(const orc_ell* M, const double* x, int prec, double* out, int64_t r0, int64_t r1,
                       orc_ctx ctx);
void orc_axpy(int prec, double alpha, const double* x, const double* y, double* out, int64_t n, orc_ctx ctx);
void orc_vec_multiply(int prec, const double* a, const double* b, double* out, int64_t n, orc_ctx ctx);
void orc_update_rc(double* r, double* u, const orc_ell* A, const double* c, double alpha, orc_ctx ctx);
int orc_cast(const double* x, int64_t n, int target, double scale, double* out, orc_ctx ctx);
double orc_dot(const double* x, const double* y, int64_t n);
double orc_norm2(const double* x, int64_t n);

/* mesh_fem.cpp */
int64_t orc_unknowns(int dim, int n);
int orc_stiffness(int dim, int n, orc_ell* A);
/* the same operator as an implicit row generator (no slot arrays) */
int orc_stiffness_implicit(int dim, int n, orc_ell* A);
int orc_stencil(int dim, int n, double* taps);
int orc_transfer(int dim, int nf, orc_ell* P, orc_ell* R);
void orc_rhs(int dim, int n, int k, double* b);
void orc_exact(int dim, int n, int k, double* u);
double orc_nodal_l2(const double* u, const double* v, int64_t len, int dim, int n);

/* multigrid.cpp */
typedef struct orc_hier orc_hier;
/* implicit = 1: every level operator (A, P, R) is an implicit row generator
 * (bitwise the assembled ELL, tests/test_oracle.py); 0: assembled ELL */
orc_hier* orc_hier_build_ex(int dim, int n, int levels, int variant, int pre, int post, double omega,
                            double base_tol, int base_mode, int base_maxit, int ftz, int fma, int* err_level,
                            int implicit);
orc_hier* orc_hier_build(int dim, int n, int levels, int variant, int pre, int post, double omega,
                         double base_tol, int base_mode, int base_maxit, int ftz, int fma, int* err_level);
void orc_hier_free(orc_hier* h);
int orc_hier_levels(const orc_hier* h);
int orc_level_prec(const orc_hier* h, int l);
int64_t orc_level_rows(const orc_hier* h, int l);
const orc_ell* orc_level_matrix(const orc_hier* h, int l, int which); /* 0=A 1=P 2=R */
const double* orc_level_invdiag(const orc_hier* h, int l);
void orc_jacobi(orc_hier* h, int l, const double* b, double* u, int steps, double omega, orc_ctx ctx);
double orc_restrict(orc_hier* h, int l, const double* r_fine, int rescale, double* r_coarse, orc_ctx ctx);
int orc_prolong(orc_hier* h, int l, const double* c_coarse, double scale, double* c_fine, orc_ctx ctx);
int orc_cg(orc_hier* h, int l, const double* b, double* u, int* converged, double* res, orc_ctx ctx);
void orc_v_cycle(orc_hier* h, const double* b, double* c, orc_ctx ctx);

/* ir_solver.cpp */
double orc_residual_norm(const orc_ell* A, const double* u, const double* b);
/* returns iterations, -2 on divergence (DivergedError), -1 on usage error */
int orc_ir_solve(orc_hier* h, const orc_ell* A, const double* b, double tol, int max_it, int random_guess,
                 uint64_t seed, int scaling, int refresh, orc_ctx ctx, double* u_out, double* hist, int hist_cap,
                 int* converged, double* final_res);

/* rng.hpp */
uint64_t orc_splitmix_next(uint64_t* state);
double orc_splitmix_double(uint64_t* state);

#ifdef __cplusplus
}
#endif
#endif
