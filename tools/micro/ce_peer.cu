// Copy-engine peer bandwidth on two GPUs (one process): can a qubit swap run
// on the copy engines, beside an SM-saturating kernel, fast enough to hide it?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o ce_peer ce_peer.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_busy(double2* a, size_t n, int reps) {  // HBM streaming, every SM
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
      double2 v = a[i];
      v.x = v.x * 1.0000001 + 1e-9;
      a[i] = v;
    }
}

int main() {
  const size_t bytes = size_t(4) << 30, rows = 64, pitch = size_t(128) << 20;  // 2D: 64 rows of 64 MiB, pitch 128 MiB
  void *a[2], *b[2], *big[2];
  cudaStream_t s[2], k[2];
  for (int d = 0; d < 2; ++d) {
    cudaSetDevice(d);
    cudaDeviceEnablePeerAccess(1 - d, 0);
    cudaMalloc(&a[d], bytes); cudaMalloc(&b[d], bytes); cudaMalloc(&big[d], size_t(16) << 30);
    cudaMemset(a[d], 1, bytes); cudaMemset(big[d], 0, size_t(16) << 30);
    cudaStreamCreateWithFlags(&s[d], cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&k[d], cudaStreamNonBlocking);
  }
  cudaEvent_t e0, e1; cudaSetDevice(0); cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto sync = [&] { for (int d = 0; d < 2; ++d) { cudaSetDevice(d); cudaDeviceSynchronize(); } };
  auto timed = [&](const char* name, auto&& body, double moved) {
    sync();
    cudaSetDevice(0); cudaEventRecord(e0, 0);
    body();
    sync();
    cudaSetDevice(0); cudaEventRecord(e1, 0); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-58s %8.2f ms  %7.1f GB/s  %s\n", name, ms, moved / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
  };
  timed("peer copy 0->1, 4 GiB, one stream", [&] { cudaSetDevice(0); cudaMemcpyPeerAsync(b[1], 1, a[0], 0, bytes, s[0]); }, bytes);
  timed("peer copy both directions, 4 GiB each", [&] {
    for (int d = 0; d < 2; ++d) { cudaSetDevice(d); cudaMemcpyPeerAsync(b[1 - d], 1 - d, a[d], d, bytes, s[d]); } }, bytes);
  timed("peer copy both directions, 4 x 1 GiB streams each way", [&] {
    for (int d = 0; d < 2; ++d) { cudaSetDevice(d);
      for (int c = 0; c < 4; ++c) cudaMemcpyPeerAsync((char*)b[1 - d] + (size_t(c) << 30), 1 - d, (char*)a[d] + (size_t(c) << 30), d, size_t(1) << 30, c % 2 ? s[d] : k[d]); } }, bytes);
  timed("2D peer copy both directions (64 x 32 MiB rows)", [&] {
    for (int d = 0; d < 2; ++d) { cudaSetDevice(d);
      cudaMemcpy2DAsync(b[1 - d], pitch / 2, a[d], pitch / 2, size_t(32) << 20, rows, cudaMemcpyDefault, s[d]); } }, double(rows) * (32 << 20));
  for (size_t w : {size_t(512), size_t(2048), size_t(8192), size_t(32768), size_t(262144)}) {
    char name[96];
    const size_t nrows = (size_t(1) << 31) / w;  // 2 GiB per direction, pitch 2 w
    snprintf(name, sizeof name, "2D peer copy both directions, rows of %zu B", w);
    timed(name, [&] {
      for (int d = 0; d < 2; ++d) { cudaSetDevice(d);
        cudaMemcpy2DAsync(b[1 - d], w, a[d], 2 * w, w, nrows, cudaMemcpyDefault, s[d]); } }, double(nrows) * w);
  }
  timed("local D2D copy 4 GiB (CE)", [&] { cudaSetDevice(0); cudaMemcpyAsync(b[0], a[0], bytes, cudaMemcpyDeviceToDevice, s[0]); }, 2.0 * bytes);
  const size_t n = (size_t(16) << 30) / 16;
  timed("busy kernel alone (16 GiB r+w x 4), both GPUs", [&] {
    for (int d = 0; d < 2; ++d) { cudaSetDevice(d); k_busy<<<148 * 8, 256, 0, k[d]>>>((double2*)big[d], n, 4); } }, 4.0 * 2 * (16.0 * (1 << 30)));
  timed("busy kernel + peer copies both ways (4 GiB each)", [&] {
    for (int d = 0; d < 2; ++d) { cudaSetDevice(d); k_busy<<<148 * 8, 256, 0, k[d]>>>((double2*)big[d], n, 4);
      cudaMemcpyPeerAsync(b[1 - d], 1 - d, a[d], d, bytes, s[d]); } }, 4.0 * 2 * (16.0 * (1 << 30)));
  // peer copy time under the busy kernel, measured on the copy stream
  sync();
  for (int d = 0; d < 2; ++d) { cudaSetDevice(d); k_busy<<<148 * 8, 256, 0, k[d]>>>((double2*)big[d], n, 8); }
  cudaSetDevice(0);
  cudaEvent_t c0, c1; cudaEventCreate(&c0); cudaEventCreate(&c1);
  cudaEventRecord(c0, s[0]);
  cudaMemcpyPeerAsync(b[1], 1, a[0], 0, bytes, s[0]);
  cudaEventRecord(c1, s[0]);
  cudaSetDevice(1); cudaMemcpyPeerAsync(b[0], 0, a[1], 1, bytes, s[1]);
  sync();
  float ms; cudaEventElapsedTime(&ms, c0, c1);
  printf("%-58s %8.2f ms  %7.1f GB/s\n", "peer copy 0->1 (4 GiB) while both GPUs run the busy kernel", ms, bytes / (ms * 1e6));
  return 0;
}
