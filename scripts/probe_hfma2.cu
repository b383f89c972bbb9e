// Microbenchmark: HFMA2 issue rate on sm_100a for the operand forms the
// binary16 stencil can use (tap in a register / tap as an immediate), with
// and without a shared (reused) x operand. Prints warp-instructions per
// cycle per SM sub-partition.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cuda_fp16.h>
#include <cstdio>

template <int MODE>
__global__ void kern(const __half2* __restrict__ in, __half2* out, int iters, long long* cyc) {
  __half2 x[8], acc[16], t[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = in[threadIdx.x + i * 32];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = in[threadIdx.x + 256 + i];
#pragma unroll
  for (int i = 0; i < 4; ++i) t[i] = in[512 + i];
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (MODE == 0) acc[j] = __hfma2(t[(j + k) & 3], x[(j * 3 + k) & 7], acc[j]);      // distinct operands
        else if (MODE == 1) acc[j] = __hfma2(t[j & 3], x[k], acc[j]);                      // x shared by 16 FMAs
        else if (MODE == 2) acc[j] = __hfma2(__floats2half2_rn(0.375f, 0.375f), x[(j * 3 + k) & 7], acc[j]);  // imm
        else acc[j] = __hfma2(__floats2half2_rn(0.375f, 0.375f), x[k], acc[j]);            // imm + shared x
      }
    }
  }
  long long c1 = clock64();
  __half2 s = acc[0];
#pragma unroll
  for (int i = 1; i < 16; ++i) s = __hadd2(s, acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = c1 - c0;
}

int main() {
  __half2 *in, *out;
  long long* cyc;
  cudaMalloc(&in, 4096 * 4);
  cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, 148 * 2048 * 4 * 8);
  cudaMalloc(&cyc, 8);
  const int iters = 2000;
  for (int mode = 0; mode < 4; ++mode) {
    for (int warps = 4; warps <= 32; warps *= 2) {
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      auto k = mode == 0 ? kern<0> : mode == 1 ? kern<1> : mode == 2 ? kern<2> : kern<3>;
      k<<<148, warps * 32>>>(in, out, 10, cyc);
      cudaEventRecord(a);
      k<<<148, warps * 32>>>(in, out, iters, cyc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double inst = (double)iters * 128 * warps;  // warp-instructions per SM
      printf("mode %d warps/SM %2d: %.3f HFMA2 warp-inst / clk / SMSP (clock64 %lld cyc, %.3f ms)\n", mode, warps,
             inst / 4.0 / (double)c, c, ms);
    }
  }
  return 0;
}
