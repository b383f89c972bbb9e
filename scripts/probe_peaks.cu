// Hierarchical-roofline denominators not in MEASURED_PEAKS.json, measured on
// the B200: L2 read bandwidth (a 48 MiB working set read repeatedly: L2
// resident), shared-memory (L1) read bandwidth, and the DFMA / HFMA2 issue
// rates (FP64 and binary16 non-tensor FMA peaks).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probe_peaks.bin scripts/probe_peaks.cu
#include <cuda_fp16.h>
#include <cstdio>

__global__ void l2_read(const uint4* __restrict__ p, size_t n16, int reps, uint4* out) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
      uint4 v;
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if (acc.x == 0x12345678u) out[0] = acc;
}

__global__ void smem_read(int reps, unsigned* out) {
  __shared__ uint4 s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_uint4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  uint4 acc = make_uint4(0, 0, 0, 0);
  int j = threadIdx.x;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 8
    for (int k = 0; k < 8; ++k) {
      const uint4 v = s[(j + k * 128) & 2047];
      acc.x ^= v.x; acc.y += v.y; acc.z ^= v.z; acc.w += v.w;
    }
    j = (j + 32) & 2047;
  }
  if (acc.x == 0x12345678u) out[0] = acc.x + acc.y + acc.z + acc.w;
}

__global__ void dfma_rate(double x, int iters, double* out) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999999, 1e-9);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 123.0) out[0] = s;
}

int main() {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // L2: 48 MiB, read 40 times
  const size_t bytes = 48ull << 20, n16 = bytes / 16;
  uint4 *buf, *out;
  cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes); cudaMalloc(&out, 64);
  l2_read<<<148 * 8, 512>>>(buf, n16, 2, out);
  cudaEventRecord(e0);
  l2_read<<<148 * 8, 512>>>(buf, n16, 40, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("l2_read_gbs %.1f\n", 40.0 * bytes / (ms * 1e-3) / 1e9);
  // shared memory: 16 B per thread per load
  const int reps = 4096;
  smem_read<<<148 * 4, 512>>>(16, (unsigned*)out);
  cudaEventRecord(e0);
  smem_read<<<148 * 4, 512>>>(reps, (unsigned*)out);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("smem_read_gbs %.1f\n", 148.0 * 4 * 512 * reps * 8 * 16 / (ms * 1e-3) / 1e9);
  // FP64 FMA
  const int iters = 1 << 14;
  dfma_rate<<<148 * 4, 512>>>(1.0, 16, (double*)out);
  cudaEventRecord(e0);
  dfma_rate<<<148 * 4, 512>>>(1.0, iters, (double*)out);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("fp64_fma_tflops %.2f\n", 2.0 * 148 * 4 * 512 * (double)iters * 8 / (ms * 1e-3) / 1e12);
  printf("fp16_fma_tflops_nontensor %.2f (from the HFMA2 probe: 0.5 warp-inst/clk/SMSP at 1965 MHz)\n",
         148.0 * 4 * 0.5 * 32 * 2 * 2 * 1.965e9 / 1e12);
  return 0;
}
