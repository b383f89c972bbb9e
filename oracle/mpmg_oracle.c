/* TEST INFRASTRUCTURE ONLY — see mpmg_oracle.h. Compiled with
 * -ffp-contract=off (proj/CMakeLists.txt:12) so only explicit fma() fuses. */
#include "mpmg_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* precision (core/src/precision.cpp, core/include/mpmg/precision.hpp)       */
/* ------------------------------------------------------------------------ */

static uint64_t dbits(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static double bitsd(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }

static const double kMinNormal16 = 6.103515625e-5; /* 2^-14, precision.hpp:44 */

/* precision.cpp:23-48: RNE to binary16 in the binary64 domain; overflow to
 * inf at >= 65520; NaN canonicalised; FTZ applied after rounding. */
double orc_quantize_fp16(double x, int ftz) {
  uint64_t u = dbits(x);
  const uint64_t mag = u & 0x7FFFFFFFFFFFFFFFull;
  if (mag == 0) return x;
  if (mag >= 0x7FF0000000000000ull) return mag > 0x7FF0000000000000ull ? NAN : x;
  if (mag >= 0x40EFFE0000000000ull) return (u >> 63) ? -INFINITY : INFINITY;
  if (mag < 0x3F20000000000000ull) { /* |x| < 2^-13: uniform 2^-24 grid */
    const double magic = (u >> 63) ? -402653184.0 : 402653184.0;
    const double r = (x + magic) - magic;
    if (r == 0.0 || (ftz && fabs(r) < kMinNormal16)) return copysign(0.0, x);
    return r;
  }
  u += 0x1FFFFFFFFFFull + ((u >> 42) & 1u);
  u &= ~0x3FFFFFFFFFFull;
  return bitsd(u);
}

/* precision.cpp:69-83 */
unsigned orc_pack_fp16(double v) {
  const uint64_t u = dbits(v);
  const unsigned sign = (unsigned)((u >> 48) & 0x8000u);
  if ((u & 0x7FFFFFFFFFFFFFFFull) == 0) return sign;
  if (isnan(v)) return 0x7E00u;
  if (isinf(v)) return sign | 0x7C00u;
  const int e = (int)((u >> 52) & 0x7FF) - 1023;
  if (e < -14) return sign | (unsigned)(fabs(v) * 0x1p24);
  return sign | ((unsigned)(e + 15) << 10) | (unsigned)((u >> 42) & 0x3FF);
}

/* precision.cpp:50-65 */
double orc_widen_fp16(unsigned bits) {
  const unsigned e = (bits >> 10) & 0x1F, m = bits & 0x3FF;
  double v;
  if (e == 31) v = m ? NAN : INFINITY;
  else if (e == 0) v = (double)m * 0x1p-24;
  else v = bitsd(((uint64_t)(e - 15 + 1023) << 52) | ((uint64_t)m << 42));
  return (bits >> 15) ? -v : v;
}

/* precision.cpp:89-97 */
double orc_fp16_add(double a, double b, int ftz) { return orc_quantize_fp16(a + b, ftz); }
double orc_fp16_mul(double a, double b, int ftz) { return orc_quantize_fp16(a * b, ftz); }

/* precision.cpp:99-121: single rounding via round-to-odd of the binary64 sum */
double orc_fp16_fma(double a, double b, double c, int ftz, int fused) {
  if (!fused) return orc_quantize_fp16(orc_quantize_fp16(a * b, ftz) + c, ftz);
  const double prod = a * b;
  double s = prod + c;
  if (isfinite(s)) {
    const double bv = s - prod;
    const double err = (prod - (s - bv)) + (c - bv);
    if (err != 0.0 && (dbits(s) & 1u) == 0) s = nextafter(s, err > 0 ? INFINITY : -INFINITY);
  }
  return orc_quantize_fp16(s, ftz);
}

/* precision.hpp:78-83 */
float orc_ftz_fp32(float v, int ftz) {
  if (ftz && v != 0.0f && fabsf(v) < FLT_MIN) return copysignf(0.0f, v);
  return v;
}

/* PVector::set (vector.hpp:43-55) == Arith<P>::from_double (kernels.cpp:27,40,58) */
double orc_round(double v, int prec, int ftz) {
  if (prec == ORC_FP16) return orc_quantize_fp16(v, ftz);
  if (prec == ORC_FP32) return (double)orc_ftz_fp32((float)v, ftz);
  return v;
}

/* Arith<P>::fma (kernels.cpp:29-31, 46-49, 64-66) */
static double ar_fma(int prec, double a, double b, double c, orc_ctx x) {
  if (prec == ORC_FP64) return x.fma ? fma(a, b, c) : a * b + c;
  if (prec == ORC_FP32) {
    const float fa = (float)a, fb = (float)b, fc = (float)c;
    if (x.fma) return (double)orc_ftz_fp32(fmaf(fa, fb, fc), x.ftz);
    return (double)orc_ftz_fp32(orc_ftz_fp32(fa * fb, x.ftz) + fc, x.ftz);
  }
  return orc_fp16_fma(a, b, c, x.ftz, x.fma);
}

/* Arith<P>::mul (kernels.cpp:28, 43-45, 61-63) */
static double ar_mul(int prec, double a, double b, orc_ctx x) {
  if (prec == ORC_FP64) return a * b;
  if (prec == ORC_FP32) return (double)orc_ftz_fp32((float)a * (float)b, x.ftz);
  return orc_fp16_mul(a, b, x.ftz);
}

/* ------------------------------------------------------------------------ */
/* ELLPACK container (core/src/ell_matrix.cpp)                               */
/* ------------------------------------------------------------------------ */

/* ell_matrix.cpp:10-28: every slot padded (value 0, col = min(row, cols-1)) */
int orc_ell_alloc(orc_ell* m, int64_t rows, int64_t cols, int rw, int prec) {
  memset(m, 0, sizeof(*m));
  m->rows = rows; m->cols = cols; m->rw = rw; m->prec = prec;
  m->col = (int32_t*)malloc((size_t)(rows * rw) * sizeof(int32_t));
  m->val = (double*)calloc((size_t)(rows * rw), sizeof(double));
  if (!m->col || !m->val) return -1;
  for (int64_t r = 0; r < rows; ++r)
    for (int s = 0; s < rw; ++s) m->col[r * rw + s] = (int32_t)(r < cols - 1 ? r : cols - 1);
  return 0;
}

void orc_ell_free(orc_ell* m) {
  free(m->col); free(m->val);
  m->col = NULL; m->val = NULL;
}

static void ell_set(orc_ell* m, int64_t row, int slot, int32_t col, double v, int ftz) {
  m->col[row * m->rw + slot] = col;                       /* ell_matrix.cpp:79-88 */
  m->val[row * m->rw + slot] = orc_round(v, m->prec, ftz);
}

static void ell_pad(orc_ell* m, int64_t row, int from) {  /* ell_matrix.cpp:90-92 */
  const int32_t pc = (int32_t)(row < m->cols - 1 ? row : m->cols - 1);
  for (int s = from; s < m->rw; ++s) { m->col[row * m->rw + s] = pc; m->val[row * m->rw + s] = 0.0; }
}

/* ell_matrix.cpp:102-118 (+ multigrid.cpp:25-33 overflow check) */
static int ell_cast(const orc_ell* src, orc_ell* dst, int prec, int ftz) {
  if (prec == ORC_FP16) {
    double mx = 0.0;
    for (int64_t i = 0; i < src->rows * src->rw; ++i) mx = fmax(mx, fabs(src->val[i]));
    if (mx > 65504.0) return -1;
  }
  if (orc_ell_alloc(dst, src->rows, src->cols, src->rw, prec)) return -2;
  memcpy(dst->col, src->col, (size_t)(src->rows * src->rw) * sizeof(int32_t));
  for (int64_t i = 0; i < src->rows * src->rw; ++i) dst->val[i] = orc_round(src->val[i], prec, ftz);
  return 0;
}

/* Implicit operators: row r generated in the slot order and padding of the
 * assembled matrices. A: orc_stiffness below (mesh_fem.cpp:124-150): the
 * in-domain neighbours in lexicographic (dz, dy, dx) order carrying the
 * level's per-offset coefficient, then (col = row, 0) padding. P / R:
 * orc_transfer (mesh_fem.cpp:204-295). */
static void decode_row(int dim, int n, int64_t r, int* ix, int* iy, int* iz) {
  const int64_t m = n - 2;
  *ix = (int)(r % m) + 1;
  *iy = (int)((r / m) % m) + 1;
  *iz = dim == 3 ? (int)(r / (m * m)) + 1 : 1;
}

void orc_ell_row(const orc_ell* m, int64_t r, int32_t* cols, double* vals) {
  const int rw = m->rw;
  if (m->gen == 0) {
    memcpy(cols, m->col + r * rw, (size_t)rw * sizeof(int32_t));
    memcpy(vals, m->val + r * rw, (size_t)rw * sizeof(double));
    return;
  }
  const int dim = m->gdim, n = m->gn;
  int out = 0;
  if (m->gen == 1) {
    int ix, iy, iz;
    decode_row(dim, n, r, &ix, &iy, &iz);
    const int zlo = dim == 3 ? -1 : 0, zhi = dim == 3 ? 1 : 0;
    for (int dz = zlo; dz <= zhi; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int jx = ix + dx, jy = iy + dy, jz = iz + dz;
          if (!(jx >= 1 && jx <= n - 2) || !(jy >= 1 && jy <= n - 2) || (dim == 3 && !(jz >= 1 && jz <= n - 2)))
            continue;
          const int slot = ((dim == 3 ? dz + 1 : 0) * 3 + (dy + 1)) * 3 + (dx + 1);
          const int64_t mm = n - 2;
          cols[out] = (int32_t)((int64_t)(jy - 1) * mm + (jx - 1) + (dim == 3 ? (int64_t)(jz - 1) * mm * mm : 0));
          vals[out++] = m->gtaps[slot];
        }
  } else if (m->gen == 2) { /* P: fine row, parents per dimension ascending */
    const int nf = n, mc = (nf + 1) / 2 - 2;
    int f[3];
    decode_row(dim, nf, r, &f[0], &f[1], &f[2]);
    int cnt[3], idx[3][2];
    double w[3][2];
    for (int d = 0; d < 3; ++d) {
      if (d == 2 && dim == 2) { cnt[d] = 1; idx[d][0] = 1; w[d][0] = 1.0; continue; }
      if (f[d] % 2 == 0) { cnt[d] = 1; idx[d][0] = f[d] / 2; w[d][0] = 1.0; }
      else {
        cnt[d] = 0;
        for (int s2 = 0; s2 < 2; ++s2) {
          const int jc = (f[d] - 1) / 2 + s2;
          if (jc >= 1 && jc <= mc) { idx[d][cnt[d]] = jc; w[d][cnt[d]] = 0.5; ++cnt[d]; }
        }
      }
    }
    const int64_t mmc = mc;
    for (int c = 0; c < cnt[2]; ++c)
      for (int b = 0; b < cnt[1]; ++b)
        for (int a = 0; a < cnt[0]; ++a) {
          cols[out] = (int32_t)((int64_t)(idx[1][b] - 1) * mmc + (idx[0][a] - 1) +
                                (dim == 3 ? (int64_t)(idx[2][c] - 1) * mmc * mmc : 0));
          vals[out++] = orc_round(w[0][a] * w[1][b] * (dim == 3 ? w[2][c] : 1.0), m->prec, 0);
        }
  } else { /* R: coarse row, the 3^dim fine neighbours of node 2i */
    const int nf = n, nc = (nf + 1) / 2;
    int cx, cy, cz;
    decode_row(dim, nc, r, &cx, &cy, &cz);
    const int zlo = dim == 3 ? -1 : 0, zhi = dim == 3 ? 1 : 0;
    const int64_t mf = nf - 2;
    for (int dz = zlo; dz <= zhi; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          double ww = (dx == 0 ? 1.0 : 0.5) * (dy == 0 ? 1.0 : 0.5);
          if (dim == 3) ww *= dz == 0 ? 1.0 : 0.5;
          const int fx = 2 * cx + dx, fy = 2 * cy + dy, fz = dim == 3 ? 2 * cz + dz : 1;
          cols[out] = (int32_t)((int64_t)(fy - 1) * mf + (fx - 1) + (dim == 3 ? (int64_t)(fz - 1) * mf * mf : 0));
          vals[out++] = orc_round(ww, m->prec, 0);
        }
  }
  const int32_t pc = (int32_t)(r < m->cols - 1 ? r : m->cols - 1); /* ell_matrix.cpp:90-92 */
  for (; out < rw; ++out) { cols[out] = pc; vals[out] = 0.0; }
}

void orc_ell_rows(const orc_ell* m, int32_t* cols, double* vals) {
  for (int64_t r = 0; r < m->rows; ++r) orc_ell_row(m, r, cols + r * m->rw, vals + r * m->rw);
}

/* row pointers without a copy for assembled matrices */
#define ELL_ROW(m, r, c, v)                                           \
  int32_t c##_buf[27];                                                \
  double v##_buf[27];                                                 \
  const int32_t* c;                                                   \
  const double* v;                                                    \
  if ((m)->gen == 0) {                                                \
    c = (m)->col + (r) * (m)->rw;                                     \
    v = (m)->val + (r) * (m)->rw;                                     \
  } else {                                                            \
    orc_ell_row((m), (r), c##_buf, v##_buf);                          \
    c = c##_buf;                                                      \
    v = v##_buf;                                                      \
  }

/* ------------------------------------------------------------------------ */
/* sparse kernels (core/src/kernels.cpp)                                     */
/* ------------------------------------------------------------------------ */

/* kernels.cpp:137-193 */
void orc_spmv(const orc_ell* A, const double* x, double* y, orc_ctx ctx) {
  const int rw = A->rw;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < A->rows; ++r) {
    ELL_ROW(A, r, c, v)
    if (A->prec == ORC_FP16 && ctx.acc32) { /* kernels.cpp:151-162 */
      float acc = 0.0f;
      orc_ctx c32 = ctx;
      for (int j = 0; j < rw; ++j) acc = (float)ar_fma(ORC_FP32, (float)v[j], (float)x[c[j]], acc, c32);
      y[r] = orc_quantize_fp16((double)acc, ctx.ftz);
    } else {
      double acc = 0.0;
      for (int j = 0; j < rw; ++j) acc = ar_fma(A->prec, v[j], x[c[j]], acc, ctx);
      y[r] = acc;
    }
  }
}

/* rows [r0, r1) of y = A x only (the sampled-row checks at 1025^3, where a
 * whole oracle pass is minutes): the same per-row arithmetic as orc_spmv */
void orc_spmv_rows(const orc_ell* A, const double* x, double* y, int64_t r0, int64_t r1, orc_ctx ctx) {
  const int rw = A->rw;
#pragma omp parallel for schedule(static)
  for (int64_t r = r0; r < r1; ++r) {
    ELL_ROW(A, r, c, v)
    if (A->prec == ORC_FP16 && ctx.acc32) {
      float acc = 0.0f;
      for (int j = 0; j < rw; ++j) acc = (float)ar_fma(ORC_FP32, (float)v[j], (float)x[c[j]], acc, ctx);
      y[r - r0] = orc_quantize_fp16((double)acc, ctx.ftz);
    } else {
      double acc = 0.0;
      for (int j = 0; j < rw; ++j) acc = ar_fma(A->prec, v[j], x[c[j]], acc, ctx);
      y[r - r0] = acc;
    }
  }
}

/* kernels.cpp:195-212: alpha rounded into the precision first */
void orc_axpy(int prec, double alpha, const double* x, const double* y, double* out, int64_t n, orc_ctx ctx) {
  const double a = orc_round(alpha, prec, ctx.ftz);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = ar_fma(prec, a, x[i], y[i], ctx);
}

/* kernels.cpp:214-229 */
void orc_vec_multiply(int prec, const double* a, const double* b, double* out, int64_t n, orc_ctx ctx) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = ar_mul(prec, a[i], b[i], ctx);
}

/* kernels.cpp:300-341: r, u, A binary64; c widened once */
void orc_update_rc(double* r, double* u, const orc_ell* A, const double* c, double alpha, orc_ctx ctx) {
  const int rw = A->rw;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < A->rows; ++i) {
    u[i] = ar_fma(ORC_FP64, alpha, c[i], u[i], ctx);
    ELL_ROW(A, i, ac, av)
    double s = 0.0;
    for (int j = 0; j < rw; ++j) s = ar_fma(ORC_FP64, av[j], c[ac[j]], s, ctx);
    r[i] = ar_fma(ORC_FP64, -alpha, s, r[i], ctx);
  }
}

/* kernels.cpp:231-239, 343-360: division in binary64, one rounding */
int orc_cast(const double* x, int64_t n, int target, double scale, double* out, orc_ctx ctx) {
  if (!(scale > 0.0) || !isfinite(scale)) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = orc_round(x[i] / scale, target, ctx.ftz);
  return 0;
}

/* kernels.cpp:368-395: sequential fma accumulation */
double orc_dot(const double* x, const double* y, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc = fma(x[i], y[i], acc);
  return acc;
}

double orc_norm2(const double* x, int64_t n) { return sqrt(orc_dot(x, x, n)); }

/* ------------------------------------------------------------------------ */
/* mesh_fem (core/src/mesh_fem.cpp, core/include/mpmg/mesh_fem.hpp)          */
/* ------------------------------------------------------------------------ */

static const double kGaussHalfSpread = 0.28867513459481287; /* mesh_fem.cpp:14 */

static double gauss_point(int i) { return i == 0 ? 0.5 - kGaussHalfSpread : 0.5 + kGaussHalfSpread; }
static double shape1d(int node, double t) { return node == 0 ? 1.0 - t : t; }
static double dshape1d(int node) { return node == 0 ? -1.0 : 1.0; }

/* mesh_fem.cpp:21-51 */
static double ref_stiffness_entry(int dim, int a, int b) {
  const int npts = dim == 2 ? 4 : 8;
  double acc = 0.0;
  for (int g = 0; g < npts; ++g) {
    double xi[3] = {0, 0, 0};
    int gg = g;
    for (int d = 0; d < dim; ++d) { xi[d] = gauss_point(gg & 1); gg >>= 1; }
    double w = 1.0;
    for (int d = 0; d < dim; ++d) w *= 0.5;
    double dot = 0.0;
    for (int d = 0; d < dim; ++d) {
      double da = dshape1d((a >> d) & 1), db = dshape1d((b >> d) & 1);
      for (int e = 0; e < dim; ++e) {
        if (e == d) continue;
        da *= shape1d((a >> e) & 1, xi[e]);
        db *= shape1d((b >> e) & 1, xi[e]);
      }
      dot += da * db;
    }
    acc += w * dot;
  }
  return acc;
}

/* mesh_fem.hpp:43-50 */
static int64_t interior_index(int n, int dim, int ix, int iy, int iz) {
  const int64_t m = n - 2;
  int64_t idx = (int64_t)(iy - 1) * m + (ix - 1);
  if (dim == 3) idx += (int64_t)(iz - 1) * m * m;
  return idx;
}
static int is_interior(int n, int i) { return i >= 1 && i <= n - 2; }

int64_t orc_unknowns(int dim, int n) {
  const int64_t m = n - 2;
  return dim == 2 ? m * m : m * m * m;
}

static void element_matrix(int dim, int n, double* el) {
  const double h = 1.0 / (n - 1);
  const double hs = dim == 2 ? 1.0 : h; /* mesh_fem.cpp:80 */
  const int ln = 1 << dim;
  for (int a = 0; a < ln; ++a)
    for (int b = 0; b < ln; ++b) el[a * ln + b] = hs * ref_stiffness_entry(dim, a, b);
}

/* mesh_fem.cpp:71-155: element-order accumulation into delta slots, then
 * compaction of the in-domain slots (ascending column) + padding */
int orc_stiffness(int dim, int n, orc_ell* A) {
  if ((dim != 2 && dim != 3) || n < 3) return -1;
  const int ln = 1 << dim, slots = dim == 2 ? 9 : 27;
  double el[64];
  element_matrix(dim, n, el);
  const int64_t N = orc_unknowns(dim, n);
  double* acc = (double*)calloc((size_t)(N * slots), sizeof(double));
  if (!acc) return -2;
  const int ezc = dim == 3 ? n - 1 : 1;
  for (int ez = 0; ez < ezc; ++ez)
    for (int ey = 0; ey < n - 1; ++ey)
      for (int ex = 0; ex < n - 1; ++ex)
        for (int a = 0; a < ln; ++a) {
          const int ax = ex + (a & 1), ay = ey + ((a >> 1) & 1), az = dim == 3 ? ez + ((a >> 2) & 1) : 1;
          if (!is_interior(n, ax) || !is_interior(n, ay) || (dim == 3 && !is_interior(n, az))) continue;
          const int64_t row = interior_index(n, dim, ax, ay, az);
          for (int b = 0; b < ln; ++b) {
            const int bx = ex + (b & 1), by = ey + ((b >> 1) & 1), bz = dim == 3 ? ez + ((b >> 2) & 1) : 1;
            if (!is_interior(n, bx) || !is_interior(n, by) || (dim == 3 && !is_interior(n, bz))) continue;
            const int dz = dim == 3 ? bz - az + 1 : 0;
            const int slot = (dz * 3 + (by - ay + 1)) * 3 + (bx - ax + 1);
            acc[row * slots + slot] += el[a * ln + b];
          }
        }
  if (orc_ell_alloc(A, N, N, slots, ORC_FP64)) { free(acc); return -2; }
  const int m = n - 2, zlo = dim == 3 ? -1 : 0, zhi = dim == 3 ? 1 : 0, izc = dim == 3 ? m : 1;
  for (int iz = 1; iz <= izc; ++iz)
    for (int iy = 1; iy <= m; ++iy)
      for (int ix = 1; ix <= m; ++ix) {
        const int64_t row = interior_index(n, dim, ix, iy, iz);
        int out = 0;
        for (int dz = zlo; dz <= zhi; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              const int jx = ix + dx, jy = iy + dy, jz = iz + dz;
              if (!is_interior(n, jx) || !is_interior(n, jy) || (dim == 3 && !is_interior(n, jz))) continue;
              const int slot = ((dim == 3 ? dz + 1 : 0) * 3 + (dy + 1)) * 3 + (dx + 1);
              ell_set(A, row, out++, (int32_t)interior_index(n, dim, jx, jy, jz), acc[row * slots + slot], 0);
            }
        ell_pad(A, row, out);
      }
  free(acc);
  return 0;
}

/* The 3^dim delta coefficients any interior row receives from the same
 * element-order accumulation as mesh_fem.cpp:92-123, restricted to the
 * 2^dim elements around one node (identical for every interior row). */
int orc_stencil(int dim, int n, double* taps) {
  if ((dim != 2 && dim != 3) || n < 3) return -1;
  const int ln = 1 << dim, slots = dim == 2 ? 9 : 27;
  double el[64];
  element_matrix(dim, n, el);
  for (int s = 0; s < slots; ++s) taps[s] = 0.0;
  const int c = 1; /* node at (1,1,1) of a local 3^dim patch */
  const int ezlo = dim == 3 ? 0 : 0, ezhi = dim == 3 ? 1 : 0;
  for (int ez = ezlo; ez <= ezhi; ++ez)
    for (int ey = 0; ey <= 1; ++ey)
      for (int ex = 0; ex <= 1; ++ex)
        for (int a = 0; a < ln; ++a) {
          const int ax = ex + (a & 1), ay = ey + ((a >> 1) & 1), az = dim == 3 ? ez + ((a >> 2) & 1) : c;
          if (ax != c || ay != c || az != c) continue;
          for (int b = 0; b < ln; ++b) {
            const int bx = ex + (b & 1), by = ey + ((b >> 1) & 1), bz = dim == 3 ? ez + ((b >> 2) & 1) : c;
            const int dz = dim == 3 ? bz - az + 1 : 0;
            taps[(dz * 3 + (by - ay + 1)) * 3 + (bx - ax + 1)] += el[a * ln + b];
          }
        }
  return slots;
}

/* mesh_fem.cpp:204-295 */
int orc_transfer(int dim, int nf, orc_ell* P, orc_ell* R) {
  const int nc = (nf + 1) / 2;
  if (nf != 2 * nc - 1) return -1;
  const int mf = nf - 2, mc = nc - 2;
  const int64_t Nf = orc_unknowns(dim, nf), Nc = orc_unknowns(dim, nc);
  if (orc_ell_alloc(P, Nf, Nc, 1 << dim, ORC_FP64)) return -2;
  const int fzc = dim == 3 ? mf : 1;
  for (int fz = 1; fz <= fzc; ++fz)
    for (int fy = 1; fy <= mf; ++fy)
      for (int fx = 1; fx <= mf; ++fx) {
        int cnt[3], idx[3][2];
        double w[3][2];
        const int f[3] = {fx, fy, fz};
        for (int d = 0; d < 3; ++d) {
          if (d == 2 && dim == 2) { cnt[d] = 1; idx[d][0] = 1; w[d][0] = 1.0; continue; }
          if (f[d] % 2 == 0) { cnt[d] = 1; idx[d][0] = f[d] / 2; w[d][0] = 1.0; }
          else {
            cnt[d] = 0;
            for (int s = 0; s < 2; ++s) {
              const int jc = (f[d] - 1) / 2 + s;
              if (jc >= 1 && jc <= mc) { idx[d][cnt[d]] = jc; w[d][cnt[d]] = 0.5; ++cnt[d]; }
            }
          }
        }
        const int64_t row = interior_index(nf, dim, fx, fy, fz);
        int slot = 0;
        for (int c = 0; c < cnt[2]; ++c)
          for (int b = 0; b < cnt[1]; ++b)
            for (int a = 0; a < cnt[0]; ++a)
              ell_set(P, row, slot++, (int32_t)interior_index(nc, dim, idx[0][a], idx[1][b], idx[2][c]),
                      w[0][a] * w[1][b] * (dim == 3 ? w[2][c] : 1.0), 0);
        ell_pad(P, row, slot);
      }
  if (orc_ell_alloc(R, Nc, Nf, dim == 2 ? 9 : 27, ORC_FP64)) return -2;
  const int czc = dim == 3 ? mc : 1;
  for (int cz = 1; cz <= czc; ++cz)
    for (int cy = 1; cy <= mc; ++cy)
      for (int cx = 1; cx <= mc; ++cx) {
        const int64_t row = interior_index(nc, dim, cx, cy, cz);
        int slot = 0;
        const int zlo = dim == 3 ? -1 : 0, zhi = dim == 3 ? 1 : 0;
        for (int dz = zlo; dz <= zhi; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              double ww = (dx == 0 ? 1.0 : 0.5) * (dy == 0 ? 1.0 : 0.5);
              if (dim == 3) ww *= dz == 0 ? 1.0 : 0.5;
              ell_set(R, row, slot++,
                      (int32_t)interior_index(nf, dim, 2 * cx + dx, 2 * cy + dy, dim == 3 ? 2 * cz + dz : 1), ww, 0);
            }
        ell_pad(R, row, slot);
      }
  return 0;
}

/* mesh_fem.cpp:157-202 */
void orc_rhs(int dim, int n, int k, double* b) {
  const double h = 1.0 / (n - 1);
  const double kpi = k * 3.141592653589793;
  const double amp = dim * kpi * kpi;
  const int ln = 1 << dim, npts = 1 << dim;
  double jac = 1.0;
  for (int d = 0; d < dim; ++d) jac *= h;
  memset(b, 0, (size_t)orc_unknowns(dim, n) * sizeof(double));
  const int ezc = dim == 3 ? n - 1 : 1;
  for (int ez = 0; ez < ezc; ++ez)
    for (int ey = 0; ey < n - 1; ++ey)
      for (int ex = 0; ex < n - 1; ++ex) {
        const int e[3] = {ex, ey, ez};
        for (int g = 0; g < npts; ++g) {
          double xi[3] = {0, 0, 0}, w = jac;
          for (int d = 0; d < dim; ++d) { xi[d] = gauss_point((g >> d) & 1); w *= 0.5; }
          double f = amp;
          for (int d = 0; d < dim; ++d) f *= sin(kpi * h * (e[d] + xi[d]));
          for (int a = 0; a < ln; ++a) {
            const int ax = ex + (a & 1), ay = ey + ((a >> 1) & 1), az = dim == 3 ? ez + ((a >> 2) & 1) : 1;
            if (!is_interior(n, ax) || !is_interior(n, ay) || (dim == 3 && !is_interior(n, az))) continue;
            double phi = 1.0;
            for (int d = 0; d < dim; ++d) phi *= shape1d((a >> d) & 1, xi[d]);
            b[interior_index(n, dim, ax, ay, az)] += w * f * phi;
          }
        }
      }
}

/* mesh_fem.cpp:297-315 */
void orc_exact(int dim, int n, int k, double* u) {
  const int m = n - 2, izc = dim == 3 ? m : 1;
  const double h = 1.0 / (n - 1), kpi = k * 3.141592653589793;
  for (int iz = 1; iz <= izc; ++iz)
    for (int iy = 1; iy <= m; ++iy)
      for (int ix = 1; ix <= m; ++ix) {
        double v = sin(kpi * ix * h) * sin(kpi * iy * h);
        if (dim == 3) v *= sin(kpi * iz * h);
        u[interior_index(n, dim, ix, iy, iz)] = v;
      }
}

/* mesh_fem.cpp:317-327 */
double orc_nodal_l2(const double* u, const double* v, int64_t len, int dim, int n) {
  double acc = 0.0;
  for (int64_t i = 0; i < len; ++i) { const double d = u[i] - v[i]; acc = fma(d, d, acc); }
  double s = 1.0;
  for (int d = 0; d < dim; ++d) s *= 1.0 / (n - 1);
  return sqrt(s * acc);
}

/* ------------------------------------------------------------------------ */
/* multigrid (core/src/multigrid.cpp, core/include/mpmg/multigrid.hpp)       */
/* ------------------------------------------------------------------------ */

typedef struct {
  int prec, has_finer;
  int64_t n;
  orc_ell A, P, R;
  double* inv_diag;
  double *u, *b, *r, *t; /* scratch, multigrid.cpp:333-339 */
} orc_level;

struct orc_hier {
  int levels, variant, pre, post, rescale;
  double omega, base_tol;
  int base_mode, base_maxit;
  orc_level* lv;
};

/* multigrid.cpp:54-77 */
static int variant_prec(int v, int l) {
  switch (v) {
    case ORC_D_MG: return ORC_FP64;
    case ORC_H_MG: return ORC_FP16;
    case ORC_HSD_MG: return l <= 1 ? ORC_FP64 : (l == 2 ? ORC_FP32 : ORC_FP16);
    default: return l <= 1 ? ORC_FP16 : (l == 2 ? ORC_FP32 : ORC_FP64);
  }
}

/* multigrid.cpp:282-342 (ProblemSpec::validate: mesh_fem.cpp:57-69) */
/* an implicit A / P / R of precision prec (the ell_cast rounding of the
 * assembled FP64 values: the stencil taps; transfer weights are powers of 2) */
static void implicit_ell(orc_ell* m, int gen, int dim, int n, int prec, int ftz) {
  memset(m, 0, sizeof(*m));
  const int nc = (n + 1) / 2;
  const int64_t N = orc_unknowns(dim, n), Nc = gen == 1 ? N : orc_unknowns(dim, nc);
  m->gen = gen; m->gdim = dim; m->gn = n; m->prec = prec;
  if (gen == 1) {
    m->rows = N; m->cols = N; m->rw = dim == 2 ? 9 : 27;
    double t[27];
    orc_stencil(dim, n, t);
    for (int k = 0; k < m->rw; ++k) m->gtaps[k] = orc_round(t[k], prec, ftz);
  } else {
    m->rows = gen == 2 ? N : Nc; m->cols = gen == 2 ? Nc : N;
    m->rw = gen == 2 ? (1 << dim) : (dim == 2 ? 9 : 27);
    (void)ftz; /* transfer weights are powers of two >= 2^-3: exact in every precision */
  }
}

int orc_stiffness_implicit(int dim, int n, orc_ell* A) {
  if ((dim != 2 && dim != 3) || n < 3) return -1;
  implicit_ell(A, 1, dim, n, ORC_FP64, 0);
  return 0;
}

orc_hier* orc_hier_build(int dim, int n, int levels, int variant, int pre, int post, double omega,
                         double base_tol, int base_mode, int base_maxit, int ftz, int fma_, int* err_level) {
  return orc_hier_build_ex(dim, n, levels, variant, pre, post, omega, base_tol, base_mode, base_maxit, ftz, fma_,
                           err_level, 0);
}

orc_hier* orc_hier_build_ex(int dim, int n, int levels, int variant, int pre, int post, double omega,
                            double base_tol, int base_mode, int base_maxit, int ftz, int fma_, int* err_level,
                            int implicit) {
  (void)fma_;
  if (err_level) *err_level = -1;
  if (levels < 2 || (n - 1) % (1 << (levels - 1)) != 0 || ((n - 1) >> (levels - 1)) + 1 < 3) return NULL;
  orc_hier* h = (orc_hier*)calloc(1, sizeof(orc_hier));
  h->levels = levels; h->variant = variant; h->pre = pre; h->post = post; h->omega = omega;
  h->base_tol = base_tol; h->base_mode = base_mode; h->base_maxit = base_maxit;
  h->rescale = variant == ORC_DSH_MG;
  h->lv = (orc_level*)calloc((size_t)levels, sizeof(orc_level));
  for (int l = 0; l < levels; ++l) {
    orc_level* L = &h->lv[l];
    L->prec = variant_prec(variant, l);
    const int nl = ((n - 1) >> (levels - 1 - l)) + 1; /* mesh_fem.hpp:20-22 */
    if (implicit) {
      implicit_ell(&L->A, 1, dim, nl, L->prec, ftz);
      L->n = L->A.rows;
      double t[27];
      orc_stencil(dim, nl, t);
      const double inv = orc_round(1.0 / t[dim == 2 ? 4 : 13], L->prec, ftz); /* multigrid.cpp:296-306 */
      L->inv_diag = (double*)malloc((size_t)L->n * sizeof(double));
      for (int64_t r = 0; r < L->n; ++r) L->inv_diag[r] = inv;
      if (l < levels - 1) {
        const int nf = ((n - 1) >> (levels - 2 - l)) + 1;
        implicit_ell(&L->P, 2, dim, nf, L->prec, ftz);
        implicit_ell(&L->R, 3, dim, nf, L->prec, ftz);
        L->has_finer = 1;
      }
      L->u = (double*)calloc((size_t)L->n, sizeof(double));
      L->b = (double*)calloc((size_t)L->n, sizeof(double));
      L->r = (double*)calloc((size_t)L->n, sizeof(double));
      L->t = (double*)calloc((size_t)L->n, sizeof(double));
      continue;
    }
    orc_ell A64;
    orc_stiffness(dim, nl, &A64);
    L->n = A64.rows;
    L->inv_diag = (double*)malloc((size_t)L->n * sizeof(double));
    for (int64_t r = 0; r < A64.rows; ++r) { /* multigrid.cpp:296-306 */
      double diag = 0.0;
      for (int s = 0; s < A64.rw; ++s)
        if (A64.col[r * A64.rw + s] == (int32_t)r) { diag = A64.val[r * A64.rw + s]; break; }
      L->inv_diag[r] = orc_round(1.0 / diag, L->prec, ftz); /* cast_vector(.,1.0) */
    }
    if (ell_cast(&A64, &L->A, L->prec, ftz)) { if (err_level) *err_level = l; orc_ell_free(&A64); orc_hier_free(h); return NULL; }
    orc_ell_free(&A64);
    if (l < levels - 1) {
      orc_ell P64, R64;
      orc_transfer(dim, ((n - 1) >> (levels - 2 - l)) + 1, &P64, &R64);
      if (ell_cast(&P64, &L->P, L->prec, ftz) || ell_cast(&R64, &L->R, L->prec, ftz)) {
        if (err_level) *err_level = l;
        orc_ell_free(&P64); orc_ell_free(&R64); orc_hier_free(h); return NULL;
      }
      orc_ell_free(&P64); orc_ell_free(&R64);
      L->has_finer = 1;
    }
    L->u = (double*)calloc((size_t)L->n, sizeof(double));
    L->b = (double*)calloc((size_t)L->n, sizeof(double));
    L->r = (double*)calloc((size_t)L->n, sizeof(double));
    L->t = (double*)calloc((size_t)L->n, sizeof(double));
  }
  return h;
}

void orc_hier_free(orc_hier* h) {
  if (!h) return;
  for (int l = 0; l < h->levels; ++l) {
    orc_level* L = &h->lv[l];
    orc_ell_free(&L->A); orc_ell_free(&L->P); orc_ell_free(&L->R);
    free(L->inv_diag); free(L->u); free(L->b); free(L->r); free(L->t);
  }
  free(h->lv);
  free(h);
}

int orc_hier_levels(const orc_hier* h) { return h->levels; }
int orc_level_prec(const orc_hier* h, int l) { return h->lv[l].prec; }
int64_t orc_level_rows(const orc_hier* h, int l) { return h->lv[l].n; }
const orc_ell* orc_level_matrix(const orc_hier* h, int l, int which) {
  if (which == 0) return &h->lv[l].A;
  if (!h->lv[l].has_finer) return NULL;
  return which == 1 ? &h->lv[l].P : &h->lv[l].R;
}
const double* orc_level_invdiag(const orc_hier* h, int l) { return h->lv[l].inv_diag; }

/* multigrid.cpp:79-89 */
static void jacobi_level(orc_level* L, const double* b, double* u, int steps, double omega, orc_ctx ctx) {
  for (int s = 0; s < steps; ++s) {
    orc_spmv(&L->A, u, L->t, ctx);
    orc_axpy(L->prec, -1.0, L->t, b, L->r, L->n, ctx);
    orc_vec_multiply(L->prec, L->inv_diag, L->r, L->t, L->n, ctx);
    orc_axpy(L->prec, omega, L->t, u, u, L->n, ctx);
  }
}

void orc_jacobi(orc_hier* h, int l, const double* b, double* u, int steps, double omega, orc_ctx ctx) {
  jacobi_level(&h->lv[l], b, u, steps, omega, ctx);
}

/* multigrid.cpp:155-205: product in the compute precision, per-op rounding,
 * matrix entries re-rounded on the fly (exact for powers of two) */
static void transfer_product(const orc_ell* M, const double* x, int prec, double* out, orc_ctx ctx) {
  const int rw = M->rw;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < M->rows; ++r) {
    ELL_ROW(M, r, c, v)
    if (prec == ORC_FP16) {
      double acc = 0.0;
      for (int j = 0; j < rw; ++j) acc = orc_fp16_fma(orc_quantize_fp16(v[j], ctx.ftz), x[c[j]], acc, ctx.ftz, ctx.fma);
      out[r] = acc;
    } else if (prec == ORC_FP32) {
      float acc = 0.0f;
      for (int j = 0; j < rw; ++j)
        acc = orc_ftz_fp32(ctx.fma ? fmaf((float)v[j], (float)x[c[j]], acc) : (float)v[j] * (float)x[c[j]] + acc,
                           ctx.ftz);
      out[r] = (double)acc;
    } else {
      double acc = 0.0;
      for (int j = 0; j < rw; ++j) acc = ctx.fma ? fma(v[j], x[c[j]], acc) : v[j] * x[c[j]] + acc;
      out[r] = acc;
    }
  }
}

/* rows [r0, r1) of the transfer product M x (precision prec, per-op
 * rounding), the restriction / prolongation of multigrid.cpp:155-205 */
void orc_transfer_rows(const orc_ell* M, const double* x, int prec, double* out, int64_t r0, int64_t r1,
                       orc_ctx ctx) {
  const int rw = M->rw;
#pragma omp parallel for schedule(static)
  for (int64_t r = r0; r < r1; ++r) {
    ELL_ROW(M, r, c, v)
    double acc = 0.0;
    if (prec == ORC_FP16) {
      for (int j = 0; j < rw; ++j) acc = orc_fp16_fma(orc_quantize_fp16(v[j], ctx.ftz), x[c[j]], acc, ctx.ftz, ctx.fma);
    } else if (prec == ORC_FP32) {
      float a = 0.0f;
      for (int j = 0; j < rw; ++j)
        a = orc_ftz_fp32(ctx.fma ? fmaf((float)v[j], (float)x[c[j]], a) : (float)v[j] * (float)x[c[j]] + a, ctx.ftz);
      acc = (double)a;
    } else {
      for (int j = 0; j < rw; ++j) acc = ctx.fma ? fma(v[j], x[c[j]], acc) : v[j] * x[c[j]] + acc;
    }
    out[r - r0] = acc;
  }
}

/* multigrid.cpp:236-268 (+ store_scaled :220-232) */
static double restrict_level(const orc_ell* R, const double* r_fine, int fine_prec, int coarse_prec, int rescale,
                             double* r_coarse, orc_ctx ctx) {
  double* prod = (double*)malloc((size_t)R->rows * sizeof(double));
  transfer_product(R, r_fine, fine_prec, prod, ctx);
  double scale = 1.0;
  if (rescale && coarse_prec == ORC_FP16) {
    const double nrm = orc_norm2(prod, R->rows);
    if (nrm > 0.0 && isfinite(nrm)) scale = nrm;
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < R->rows; ++i) r_coarse[i] = orc_round(prod[i] / scale, coarse_prec, ctx.ftz);
  free(prod);
  return scale;
}

double orc_restrict(orc_hier* h, int l, const double* r_fine, int rescale, double* r_coarse, orc_ctx ctx) {
  return restrict_level(&h->lv[l - 1].R, r_fine, h->lv[l].prec, h->lv[l - 1].prec, rescale, r_coarse, ctx);
}

/* multigrid.cpp:270-280 */
static int prolong_level(const orc_ell* P, const double* c_coarse, int coarse_prec, int fine_prec, double scale,
                         double* c_fine, orc_ctx ctx) {
  if (!(scale > 0.0) || !isfinite(scale)) return -1;
  double* prod = (double*)malloc((size_t)P->rows * sizeof(double));
  transfer_product(P, c_coarse, coarse_prec, prod, ctx);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < P->rows; ++i) c_fine[i] = orc_round(prod[i] * scale, fine_prec, ctx.ftz);
  free(prod);
  return 0;
}

int orc_prolong(orc_hier* h, int l, const double* c_coarse, double scale, double* c_fine, orc_ctx ctx) {
  return prolong_level(&h->lv[l - 1].P, c_coarse, h->lv[l - 1].prec, h->lv[l].prec, scale, c_fine, ctx);
}

/* multigrid.cpp:91-151 */
static int cg_level(const orc_ell* A, const double* b, double* u, int prec, double tol, int mode, int maxit_cfg,
                    int* converged, double* final_res, orc_ctx ctx) {
  const int64_t n = A->rows;
  const int max_it = maxit_cfg > 0 ? maxit_cfg : 10 * (int)n;
  memset(u, 0, (size_t)n * sizeof(double));
  double* r = (double*)malloc((size_t)n * sizeof(double));
  double* p = (double*)malloc((size_t)n * sizeof(double));
  double* Ap = (double*)malloc((size_t)n * sizeof(double));
  double* sc = (double*)malloc((size_t)n * sizeof(double));
  double* best = (double*)calloc((size_t)n, sizeof(double));
  orc_cast(b, n, prec, 1.0, r, ctx);
  orc_cast(r, n, prec, 1.0, p, ctx);
  const double norm_b = orc_norm2(b, n);
  int it = 0;
  if (norm_b == 0.0) {
    *converged = 1; *final_res = 0.0;
    free(r); free(p); free(Ap); free(sc); free(best);
    return 0;
  }
  const double thr = mode == 0 ? tol * norm_b : tol;
  double rz = orc_dot(r, r, n), true_res = norm_b, best_res = true_res;
  while (true_res >= thr && it < max_it) {
    orc_spmv(A, p, Ap, ctx);
    const double pAp = orc_dot(p, Ap, n);
    if (!(pAp > 0.0) || !isfinite(pAp)) break;
    const double alpha = rz / pAp;
    orc_axpy(prec, alpha, p, u, u, n, ctx);
    orc_axpy(prec, -alpha, Ap, r, r, n, ctx);
    const double rz_new = orc_dot(r, r, n);
    ++it;
    orc_spmv(A, u, sc, ctx);
    orc_axpy(prec, -1.0, sc, b, sc, n, ctx);
    true_res = orc_norm2(sc, n);
    if (true_res < best_res) { best_res = true_res; memcpy(best, u, (size_t)n * sizeof(double)); }
    if (rz == 0.0) break;
    const double beta = rz_new / rz;
    orc_axpy(prec, beta, p, r, p, n, ctx);
    rz = rz_new;
  }
  if (true_res > best_res) { memcpy(u, best, (size_t)n * sizeof(double)); true_res = best_res; }
  *converged = true_res < thr;
  *final_res = true_res;
  free(r); free(p); free(Ap); free(sc); free(best);
  return it;
}

int orc_cg(orc_hier* h, int l, const double* b, double* u, int* converged, double* res, orc_ctx ctx) {
  return cg_level(&h->lv[l].A, b, u, h->lv[l].prec, h->base_tol, h->base_mode, h->base_maxit, converged, res, ctx);
}

/* multigrid.cpp:362-393 */
static void cycle_at(orc_hier* h, int l, const double* rhs, double* u, orc_ctx ctx) {
  orc_level* L = &h->lv[l];
  if (l == 0) {
    int conv; double res;
    cg_level(&L->A, rhs, u, L->prec, h->base_tol, h->base_mode, h->base_maxit, &conv, &res, ctx);
    return;
  }
  memset(u, 0, (size_t)L->n * sizeof(double));
  jacobi_level(L, rhs, u, h->pre, h->omega, ctx);
  orc_spmv(&L->A, u, L->t, ctx);
  orc_axpy(L->prec, -1.0, L->t, rhs, L->r, L->n, ctx);
  orc_level* C = &h->lv[l - 1];
  const int rescale = h->rescale && C->prec == ORC_FP16;
  const double scale = restrict_level(&C->R, L->r, L->prec, C->prec, rescale, C->b, ctx);
  cycle_at(h, l - 1, C->b, C->u, ctx);
  prolong_level(&C->P, C->u, C->prec, L->prec, scale, L->t, ctx);
  orc_axpy(L->prec, 1.0, L->t, u, u, L->n, ctx);
  jacobi_level(L, rhs, u, h->post, h->omega, ctx);
}

void orc_v_cycle(orc_hier* h, const double* b, double* c, orc_ctx ctx) { cycle_at(h, h->levels - 1, b, c, ctx); }

/* ------------------------------------------------------------------------ */
/* ir_solver (core/src/ir_solver.cpp) + rng.hpp                               */
/* ------------------------------------------------------------------------ */

uint64_t orc_splitmix_next(uint64_t* s) { /* rng.hpp:13-18 */
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
double orc_splitmix_double(uint64_t* s) { return (double)(orc_splitmix_next(s) >> 11) * 0x1.0p-53; }

/* ir_solver.cpp:21-49 */
double orc_residual_norm(const orc_ell* A, const double* u, const double* b) {
  double* rr = (double*)malloc((size_t)A->rows * sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < A->rows; ++i) {
    ELL_ROW(A, i, c, v)
    double s = 0.0;
    for (int j = 0; j < A->rw; ++j) s = fma(v[j], u[c[j]], s);
    rr[i] = b[i] - s;
  }
  double acc = 0.0; /* sequential, in row order */
  for (int64_t i = 0; i < A->rows; ++i) acc = fma(rr[i], rr[i], acc);
  free(rr);
  return sqrt(acc);
}

/* ir_solver.cpp:51-127. scaling: 0 VariantDefault, 1 ForceOn, 2 ForceOff */
int orc_ir_solve(orc_hier* h, const orc_ell* A, const double* b, double tol, int max_it, int random_guess,
                 uint64_t seed, int scaling, int refresh, orc_ctx ctx, double* u, double* hist, int hist_cap,
                 int* converged, double* final_res) {
  const int64_t n = A->rows;
  if (A->prec != ORC_FP64 || n != h->lv[h->levels - 1].n || !(tol > 0.0)) return -1;
  const int mgp = h->lv[h->levels - 1].prec;
  const int scale_on = scaling == 1 ? 1 : (scaling == 2 ? 0 : h->variant != ORC_D_MG);
  memset(u, 0, (size_t)n * sizeof(double));
  if (random_guess) {
    uint64_t st = seed;
    for (int64_t i = 0; i < n; ++i) u[i] = orc_splitmix_double(&st);
  }
  double* r = (double*)malloc((size_t)n * sizeof(double));
  double* t = (double*)malloc((size_t)n * sizeof(double));
  double* rl = (double*)malloc((size_t)n * sizeof(double));
  double* cl = (double*)calloc((size_t)n, sizeof(double));
  orc_spmv(A, u, t, ctx);
  orc_axpy(ORC_FP64, -1.0, t, b, r, n, ctx);
  int its = 0, rc = 0;
  *converged = 0;
  for (;;) {
    const double alpha = orc_norm2(r, n);
    if (hist && its < hist_cap) hist[its] = alpha;
    if (!isfinite(alpha)) { rc = -2; break; }
    if (alpha < tol) { *converged = 1; break; }
    if (its >= max_it) break;
    const double scale = scale_on && alpha > 0.0 ? alpha : 1.0;
    orc_cast(r, n, mgp, scale, rl, ctx);
    orc_v_cycle(h, rl, cl, ctx);
    orc_update_rc(r, u, A, cl, scale, ctx);
    ++its;
    if (refresh > 0 && its % refresh == 0) {
      orc_spmv(A, u, t, ctx);
      orc_axpy(ORC_FP64, -1.0, t, b, r, n, ctx);
    }
  }
  *final_res = orc_residual_norm(A, u, b);
  free(r); free(t); free(rl); free(cl);
  return rc ? rc : its;
}
