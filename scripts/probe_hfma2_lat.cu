// HFMA2 dependent-issue latency on sm_100a: K independent accumulator chains
// per warp, one warp per SM sub-partition; rate = min(0.5, K / latency).
#include <cuda_fp16.h>
#include <cstdio>

template <int K>
__global__ void chains(const __half2* __restrict__ in, __half2* out, int iters, long long* cyc) {
  __half2 acc[K], t = in[0], x = in[1];
#pragma unroll
  for (int i = 0; i < K; ++i) acc[i] = in[2 + i];
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 32; ++r)
#pragma unroll
      for (int i = 0; i < K; ++i) acc[i] = __hfma2(t, x, acc[i]);
  }
  long long c1 = clock64();
  __half2 s = acc[0];
#pragma unroll
  for (int i = 1; i < K; ++i) s = __hadd2(s, acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = c1 - c0;
}

template <int K>
void run(__half2* in, __half2* out, long long* cyc) {
  const int iters = 4000;
  chains<K><<<148, 128>>>(in, out, 10, cyc);
  chains<K><<<148, 128>>>(in, out, iters, cyc);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double inst = (double)iters * 32 * K;  // per warp
  printf("K=%2d chains: %.3f HFMA2/clk per warp -> latency ~ %.2f cyc\n", K, inst / c, K * c / inst);
}

int main() {
  __half2 *in, *out;
  long long* cyc;
  cudaMalloc(&in, 4096);
  cudaMemset(in, 0, 4096);
  cudaMalloc(&out, 148 * 128 * 4);
  cudaMalloc(&cyc, 8);
  run<1>(in, out, cyc); run<2>(in, out, cyc); run<3>(in, out, cyc); run<4>(in, out, cyc);
  run<6>(in, out, cyc); run<8>(in, out, cyc); run<12>(in, out, cyc); run<16>(in, out, cyc);
  return 0;
}
