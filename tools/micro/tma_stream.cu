// TMA streaming micro-benchmark for the HBM tile pattern of k_blocked: each of
// 296 CTAs (2 per SM) moves 32 KiB tiles of a 2^28-amplitude state through
// shared memory (load, then store back) with `depth` loads in flight, for
// several box shapes.  Reports GB/s of (load + store) bytes.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o tma_stream tma_stream.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstring>

struct Map { CUtensorMap m; int rank, box_bits, nl; int start[5], ebits[5]; uint64_t left; };
using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                         const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                         CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                         CUtensorMapFloatOOBfill);
static Map encode(const int* tq, int n, void* amps, int promo) {
  Map T; memset(&T, 0, sizeof T);
  int start[5] = {0}, len[5] = {3}, rank = 1, b = 3;
  if (tq[3] != 3) { start[rank] = 3; len[rank++] = 0; }
  while (b < 11) { int e = b + 1; while (e < 11 && tq[e] == tq[e - 1] + 1) ++e;
    if (rank < 5) { start[rank] = tq[b]; len[rank++] = e - b; } else for (int j = b; j < e; ++j) T.left |= 1ull << tq[j];
    b = e; }
  cuuint64_t dim[5], stride[4]; cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  dim[0] = 16; box[0] = 16; int bb = 3;
  for (int i = 1; i < rank; ++i) { int top = i + 1 < rank ? start[i + 1] : n; T.start[i] = start[i]; T.ebits[i] = top - start[i];
    dim[i] = 1ull << (top - start[i]); stride[i - 1] = 16ull << start[i]; box[i] = 1u << len[i]; bb += len[i]; }
  T.rank = rank; T.box_bits = bb; T.nl = __builtin_popcountll(T.left);
  void* f; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  CUtensorMapL2promotion pr[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
  reinterpret_cast<Enc>(f)(&T.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, amps, dim, stride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, pr[promo], CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return T;
}
__device__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ void tcopy(bool st, uint32_t sm, const void* map, uint32_t bar, int rank, const int* c) {
  if (!st) {
    switch (rank) {
      case 2: asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(sm), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]) : "memory"); break;
      case 3: asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(sm), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]) : "memory"); break;
      case 4: asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(sm), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory"); break;
      default: asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(sm), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
    }
  } else {
    switch (rank) {
      case 2: asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map), "r"(sm), "r"(c[0]), "r"(c[1]) : "memory"); break;
      case 3: asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map), "r"(sm), "r"(c[0]), "r"(c[1]), "r"(c[2]) : "memory"); break;
      case 4: asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(map), "r"(sm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory"); break;
      default: asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(map), "r"(sm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
    }
  }
}
__device__ void tile(bool st, const Map& T, uint64_t base, uint32_t sm, uint32_t bar) {
  for (int v = 0; v < (1 << T.nl); ++v) {
    uint64_t g = base; int j = 0;
    for (uint64_t m = T.left; m; m &= m - 1, ++j) if (v >> j & 1) g |= m & (0 - m);
    int c[5] = {0, 0, 0, 0, 0};
    for (int i = 1; i < T.rank; ++i) c[i] = int((g >> T.start[i]) & ((1ull << T.ebits[i]) - 1));
    tcopy(st, sm + (uint32_t(v) << (T.box_bits + 4)), &T.m, bar, T.rank, c);
  }
}
// depth: loads in flight (buffers = depth + 1); store: write each tile back
__global__ void __launch_bounds__(128, 2) k_stream(const __grid_constant__ Map T, int n, uint64_t omask, int depth, int store) {
  extern __shared__ __align__(128) double2 raw[];
  double2* buf = raw + ((1024u - (su32(raw) & 1023u)) & 1023u) / 16;
  __shared__ __align__(8) uint64_t bars[4];
  const uint64_t n_tiles = 1ull << (n - 11);
  const uint64_t per = n_tiles / gridDim.x, t0 = blockIdx.x * per;
  const int nbuf = depth + 1;
  auto base_of = [&](uint64_t t) { uint64_t b = 0; int j = 0; for (uint64_t m = omask; m; m &= m - 1, ++j) if (t >> j & 1) b |= m & (0 - m); return b; };
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  unsigned ph = 0;
  if (threadIdx.x == 0)
    for (int d = 0; d < depth && d < int(per); ++d) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[d])), "r"(32768));
      tile(false, T, base_of(t0 + d), su32(buf + d * 2048), su32(&bars[d]));
    }
  for (uint64_t i = 0; i < per; ++i) {
    const int b = int(i % nbuf);
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(&bars[b])), "r"((ph >> b) & 1) : "memory");
    ph ^= 1u << b;
    __syncthreads();
    if (threadIdx.x == 0) {
      if (store) { tile(true, T, base_of(t0 + i), su32(buf + b * 2048), 0); asm volatile("cp.async.bulk.commit_group;"); }
      if (i + depth < per) {
        const int nb = int((i + depth) % nbuf);
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // the store from buffer nb (issued depth tiles ago)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[nb])), "r"(32768));
        tile(false, T, base_of(t0 + i + depth), su32(buf + nb * 2048), su32(&bars[nb]));
      }
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
int main() {
  const int n = 28;
  void* amps; cudaMalloc(&amps, 16ull << n); cudaMemset(amps, 0, 16ull << n);
  const int cases[4][11] = {{0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10}, {0, 1, 2, 5, 9, 13, 17, 20, 22, 24, 27},
                            {0, 1, 2, 3, 4, 8, 9, 14, 15, 20, 21}, {0, 1, 2, 6, 7, 8, 9, 14, 15, 16, 17}};
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int ci = 0; ci < 4; ++ci)
    for (int promo : {0, 2, 3})
      for (int depth : {1, 2})
        for (int store : {0, 1}) {
          uint64_t tm = 0; for (int i = 0; i < 11; ++i) tm |= 1ull << cases[ci][i];
          Map T = encode(cases[ci], n, amps, promo);
          const uint64_t om = ((1ull << n) - 1) & ~tm;
          const size_t sm = size_t(depth + 1) * 32768 + 1024;
          k_stream<<<296, 128, sm>>>(T, n, om, depth, store);
          cudaEventRecord(e0);
          for (int r = 0; r < 3; ++r) k_stream<<<296, 128, sm>>>(T, n, om, depth, store);
          cudaEventRecord(e1); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          const double bytes = 3.0 * (16ull << n) * (store ? 2 : 1) * (double((1ull << (n - 11)) / 296 * 296) / (1ull << (n - 11)));
          printf("case %d rank %d copies %d promo %d depth %d store %d: %.2f ms  %.0f GB/s  %s\n", ci, T.rank, 1 << T.nl, promo, depth, store,
                 ms / 3, bytes / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
        }
  return 0;
}
