// Host-side setup helpers (mpmg_host.cpp).
#pragma once

#include <stdint.h>

#include "mpmg_gpu.h"

namespace mpmg_impl {

double round_fp16(double x, bool ftz);
double round_to(double x, int prec, bool ftz);
uint16_t fp16_bits(double v);
double fp16_value(uint16_t bits);

// 3^dim stencil of an interior row (mesh_fem.cpp:71-155 accumulation order)
int stencil_taps(int dim, int n, double* taps);
// assemble_rhs (mesh_fem.cpp:157-202), compact interior order
void problem_rhs(int dim, int n, int k, double* b);
// VariantConfig::make (multigrid.cpp:54-77)
int variant_precision(int variant, int level);
// per-level operator in precision `prec` (MgHierarchy::build, multigrid.cpp:290-310)
int build_level_stencil(int dim, int nodes, int prec, bool ftz, mpmg_stencil* out);

}  // namespace mpmg_impl
