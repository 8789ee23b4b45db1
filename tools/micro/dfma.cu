// Microbenchmark: DFMA dependent-chain latency and throughput per SM at a
// given number of warps (8 = k_blocked's occupancy).  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void k(double* out, int iters, long long* cycles) {
  double a[CHAINS];
  for (int c = 0; c < CHAINS; ++c) a[c] = threadIdx.x * 1e-3 + c;
  const double m = 0.999999, b = 1e-7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) a[c] = fma(a[c], m, b);
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int CHAINS>
void run(int warps_per_sm, int sms) {
  const int iters = 4096;
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * sms * warps_per_sm * 32);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  k<CHAINS><<<sms, warps_per_sm * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  const double dfma_per_sm = double(iters) * CHAINS * warps_per_sm * 32;
  printf("chains %2d warps/SM %2d: %.2f cycles per dependent DFMA, %.1f DFMA lanes/clk/SM\n",
         CHAINS, warps_per_sm, double(c) / (iters), dfma_per_sm / double(c));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1>(1, sms);
  run<1>(8, sms);
  run<4>(8, sms);
  run<8>(8, sms);
  run<16>(8, sms);
  run<8>(16, sms);
  run<16>(16, sms);
  return 0;
}
