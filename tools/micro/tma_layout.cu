// Micro check of the TMA tile layout k_blocked assumes (planner.h "TMA
// tiles"): a tile of an n-qubit state at physical base `base`, tile qubits tq,
// loaded by cp.async.bulk.tensor with the per-pass map of device.cu, must land
// at swz_tma(l) for tile-local index l; a TMA store of a known buffer must
// write amplitude base | scatter(l) from slot swz_tma(l).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o tma_layout tma_layout.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>
#include <utility>

struct TmaInfo {
  CUtensorMap map;
  uint64_t left;
  int start[5], ebits[5], rank, box_bits;
};

using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                         const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                         CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                         CUtensorMapFloatOOBfill);

static bool g_reverse = false;  // list the run dims in reverse qubit order
static TmaInfo encode(const int* tq, int k, int n, void* amps) {
  TmaInfo T;
  memset(&T, 0, sizeof T);
  int start[5] = {0}, len[5] = {3}, rank = 1, b = 3;
  if (tq[3] != 3) { start[rank] = 3; len[rank++] = 0; }
  while (b < k) {
    int e = b + 1;
    while (e < k && tq[e] == tq[e - 1] + 1) ++e;
    if (rank < 5) { start[rank] = tq[b]; len[rank++] = e - b; }
    else for (int j = b; j < e; ++j) T.left |= 1ull << tq[j];
    b = e;
  }
  cuuint64_t dim[5], stride[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  dim[0] = 16; box[0] = 16;
  int bb = 3;
  for (int i = 1; i < rank; ++i) {
    int top = i + 1 < rank ? start[i + 1] : n;
    T.start[i] = start[i]; T.ebits[i] = top - start[i];
    dim[i] = 1ull << (top - start[i]); stride[i - 1] = 16ull << start[i];
    box[i] = 1u << len[i]; bb += len[i];
  }
  if (g_reverse) {  // dims 1..rank-1 in reverse order
    for (int i = 1, j = rank - 1; i < j; ++i, --j) {
      std::swap(T.start[i], T.start[j]); std::swap(T.ebits[i], T.ebits[j]);
      std::swap(dim[i], dim[j]); std::swap(stride[i - 1], stride[j - 1]); std::swap(box[i], box[j]);
    }
  }
  T.rank = rank; T.box_bits = bb;
  void* f; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  CUresult r = reinterpret_cast<Enc>(f)(&T.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, amps, dim,
                                        stride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("rank %d box_bits %d left %llx encode rc %d dims:", rank, bb, (unsigned long long)T.left, int(r));
  for (int i = 0; i < rank; ++i) printf(" [%llu box %u]", (unsigned long long)dim[i], box[i]);
  printf("\n");
  return T;
}

__device__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }


__device__ void tld(uint32_t dst, const void* map, uint32_t bar, int rank, const int* c) {
  switch (rank) {
    case 2: asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]) : "memory"); break;
    case 3: asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]) : "memory"); break;
    case 4: asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory"); break;
    default: asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
  }
}
__device__ void tst(const void* map, uint32_t src, int rank, const int* c) {
  switch (rank) {
    case 2: asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map), "r"(src), "r"(c[0]), "r"(c[1]) : "memory"); break;
    case 3: asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map), "r"(src), "r"(c[0]), "r"(c[1]), "r"(c[2]) : "memory"); break;
    case 4: asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(map), "r"(src), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory"); break;
    default: asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(map), "r"(src), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
  }
}

__global__ void k_test(const __grid_constant__ TmaInfo T, uint64_t base, double2* out, int store) {
  extern __shared__ __align__(128) double2 raw[];
  double2* buf = raw + ((1024u - (su32(raw) & 1023u)) & 1023u) / 16;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = su32(&bar), dst = su32(buf);
  if (!store) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(32768));
      int nl = __popcll(T.left);
      for (int v = 0; v < (1 << nl); ++v) {
        uint64_t g = base; int j = 0;
        for (uint64_t m = T.left; m; m &= m - 1, ++j) if (v >> j & 1) g |= m & (0 - m);
        int c[5] = {0, 0, 0, 0, 0};
        for (int i = 1; i < T.rank; ++i) c[i] = int((g >> T.start[i]) & ((1ull << T.ebits[i]) - 1));
        uint32_t at = dst + (uint32_t(v) << (T.box_bits + 4));
        tld(at, &T.map, b, T.rank, c);
      }
    }
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(b) : "memory");
    for (int s = threadIdx.x; s < 2048; s += blockDim.x) out[s] = buf[s];
  } else {
    for (int s = threadIdx.x; s < 2048; s += blockDim.x) buf[s] = make_double2(double(s), -1.0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      int nl = __popcll(T.left);
      for (int v = 0; v < (1 << nl); ++v) {
        uint64_t g = base; int j = 0;
        for (uint64_t m = T.left; m; m &= m - 1, ++j) if (v >> j & 1) g |= m & (0 - m);
        int c[5] = {0, 0, 0, 0, 0};
        for (int i = 1; i < T.rank; ++i) c[i] = int((g >> T.start[i]) & ((1ull << T.ebits[i]) - 1));
        uint32_t at = dst + (uint32_t(v) << (T.box_bits + 4));
        tst(&T.map, at, T.rank, c);
      }
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }
}

static uint64_t scatter(uint64_t l, const int* tq, int k) {
  uint64_t g = 0;
  for (int i = 0; i < k; ++i) if (l >> i & 1) g |= 1ull << tq[i];
  return g;
}

// smem (pre-swizzle) index of tile-local l: dim0 bits, then each dim's box
// bits in dim order, then the leftover qubits (ascending)
static int smem_of(int l, const int* tq, const TmaInfo& T) {
  int out = l & 7, pos = 3;
  for (int i = 1; i < T.rank; ++i) {
    // the dim's box bits: tile qubits start..start+len-1 where the box is 2^len
    for (int b = 3; b < 11; ++b) {
      const int q = tq[b];
      if (q >= T.start[i] && q < T.start[i] + T.ebits[i] && !(T.left >> q & 1)) {
        // inside this dim's coordinate range and a box bit (lowest run bits)
        if (l >> b & 1) out |= 1 << (pos + (q - T.start[i]));
      }
    }
    int blen = 0;
    for (int b = 3; b < 11; ++b) { const int q = tq[b]; if (q >= T.start[i] && q < T.start[i] + T.ebits[i] && !(T.left >> q & 1)) ++blen; }
    pos += blen;
  }
  for (int b = 3; b < 11; ++b) if (T.left >> tq[b] & 1) { if (l >> b & 1) out |= 1 << pos; ++pos; }
  return out;
}

int main() {
  const int n = 20;
  double2* amps; double2* out;
  cudaMalloc(&amps, sizeof(double2) << n);
  cudaMalloc(&out, sizeof(double2) * 2048);
  std::vector<double2> h(1 << n);
  const int cases[4][11] = {{0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10},
                            {0, 1, 2, 4, 6, 8, 10, 12, 14, 16, 18},
                            {0, 1, 2, 3, 4, 6, 7, 9, 10, 12, 13},
                            {0, 1, 2, 4, 6, 8, 10, 12, 13, 14, 15}};
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  for (int rev = 0; rev < 2; ++rev)
  for (int ci = 0; ci < 4; ++ci) {
    g_reverse = rev;
    const int* tq = cases[ci];
    uint64_t tmask = scatter(2047, tq, 11), omask = ((1ull << n) - 1) & ~tmask;
    TmaInfo T = encode(tq, 11, n, amps);
    const uint64_t bases[4] = {uint64_t(0), omask, omask & 0x5555555555ull, omask & 0xaaaaaaaaull};
    for (uint64_t base : bases) {
      for (int i = 0; i < (1 << n); ++i) h[i] = make_double2(double(i), 0.0);
      cudaMemcpy(amps, h.data(), sizeof(double2) << n, cudaMemcpyHostToDevice);
      k_test<<<1, 128, 32768 + 1024>>>(T, base, out, 0);
      std::vector<double2> o(2048);
      cudaMemcpy(o.data(), out, sizeof(double2) * 2048, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int l = 0; l < 2048; ++l) {
        int s = smem_of(l, tq, T) ^ ((smem_of(l, tq, T) >> 3) & 7);
        uint64_t want = base | scatter(l, tq, 11);
        if (o[s].x != double(want)) { if (bad < 4) printf("  load base %llx l %d slot %d got %.0f want %llu\n", (unsigned long long)base, l, s, o[s].x, (unsigned long long)want); ++bad; }
      }
      // store
      cudaMemset(amps, 0, sizeof(double2) << n);
      k_test<<<1, 128, 32768 + 1024>>>(T, base, out, 1);
      cudaMemcpy(h.data(), amps, sizeof(double2) << n, cudaMemcpyDeviceToHost);
      int sbad = 0;
      for (int l = 0; l < 2048; ++l) {
        int s = smem_of(l, tq, T) ^ ((smem_of(l, tq, T) >> 3) & 7);
        uint64_t g = base | scatter(l, tq, 11);
        if (h[g].x != double(s) || h[g].y != -1.0) { if (sbad < 4) printf("  store base %llx l %d got %.0f want slot %d\n", (unsigned long long)base, l, h[g].x, s); ++sbad; }
      }
      printf("rev %d case %d base %llx: load bad %d, store bad %d (%s)\n", rev, ci, (unsigned long long)base, bad, sbad,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
