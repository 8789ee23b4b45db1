// sm_100a kernels and the device half of the C ABI.
//
// Reference hot path (nucsim/engine.py) and its replacement here:
//   apply_1q / apply_2q / apply_dense (92-156)  -> k_apply1 / k_apply2 / k_applyk
//   _branch_probability (159-161)               -> k_half_norm + k_sum_fixed
//   _project (164-167)                          -> k_project
//   sample's |a|^2 (215)                        -> k_probabilities (no FMA)
//   expectation_pauli (225-239)                 -> k_pauli_term
//   run()'s gate loop + MMA asserts (414-423)   -> k_blocked: ONE persistent
//       cooperative launch walks the whole fused gate stream; each pass moves
//       the state through shared memory once (global traffic 32 B/amplitude)
//       and applies every gate of the pass in registers, stage by stage;
//       mid-circuit assertions are epilogue reductions + prologue collapses
//       separated by grid-wide barriers.
// The state is complex128 in HBM as double2 (16-byte vector loads/stores).
#include <cooperative_groups.h>
#include <cuda.h>  // CUtensorMap types only: the encoder comes from cudaGetDriverEntryPoint
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is resolved at run time (shard_nccl)

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>

#include "device.cuh"
#include "planner_host.h"

namespace cg = cooperative_groups;

namespace nsb {
namespace dev {

constexpr int kReduceThreads = 256;
constexpr int kReduceBlocks = 1184;  // 8 x 148 SMs: fixed => deterministic sums

// ---------------------------------------------------------------------------
// per-op kernels

__global__ void k_vacuum(double2* __restrict__ a, uint64_t n_amps) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n_amps;
       i += uint64_t(gridDim.x) * blockDim.x)
    a[i] = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
}

struct M2 {
  double2 m[4];
};
struct M4 {
  double2 m[16];
};

__global__ void k_apply1(double2* __restrict__ a, uint64_t n_pairs, int q, M2 u) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n_pairs;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i0 = insert_zero(i, q), i1 = i0 | (uint64_t(1) << q);
    const double2 x = a[i0], y = a[i1];
    double2 o0 = make_double2(0.0, 0.0), o1 = o0;
    cmac(o0, u.m[0], x);
    cmac(o0, u.m[1], y);
    cmac(o1, u.m[2], x);
    cmac(o1, u.m[3], y);
    a[i0] = o0;
    a[i1] = o1;
  }
}

// p < q; matrix index = bit(p) + 2 bit(q)  (engine.py:104-121)
__global__ void k_apply2(double2* __restrict__ a, uint64_t n_quads, int p, int q, M4 u) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n_quads;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t b = insert_zero(insert_zero(i, p), q);
    const uint64_t idx[4] = {b, b | (uint64_t(1) << p), b | (uint64_t(1) << q),
                             b | (uint64_t(1) << p) | (uint64_t(1) << q)};
    double2 x[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = a[idx[c]];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double2 o = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < 4; ++c) cmac(o, u.m[4 * r + c], x[c]);
      a[idx[r]] = o;
    }
  }
}

struct KQ {
  int k;
  int slot_q[5];    // qubit of matrix slot j
  int sorted_q[5];  // same qubits ascending (for zero insertion)
};

// dense k-qubit matrix (k <= 5) on arbitrary qubits (engine.py:130-156)
__global__ void k_applyk(double2* __restrict__ a, uint64_t n_groups, KQ g,
                         const double2* __restrict__ m) {
  const int dim = 1 << g.k;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n_groups;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t base = i;
    for (int j = 0; j < g.k; ++j) base = insert_zero(base, g.sorted_q[j]);
    double2 x[32], o[32];
    uint64_t idx[32];
    for (int s = 0; s < dim; ++s) {
      uint64_t e = base;
      for (int j = 0; j < g.k; ++j)
        if (s >> j & 1) e |= uint64_t(1) << g.slot_q[j];
      idx[s] = e;
      x[s] = a[e];
    }
    for (int r = 0; r < dim; ++r) {
      double2 acc = make_double2(0.0, 0.0);
      for (int c = 0; c < dim; ++c) cmac(acc, __ldg(m + r * dim + c), x[c]);
      o[r] = acc;
    }
    for (int s = 0; s < dim; ++s) a[idx[s]] = o[s];
  }
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w];
  return s;  // valid in thread 0
}

// sum |a_i|^2 over indices with bit q == outcome, per-block partials
__global__ void k_half_norm(const double2* __restrict__ a, uint64_t n_half, int q, int outcome,
                            double* __restrict__ partials) {
  __shared__ double red[32];
  double s = 0.0;
  const uint64_t bit = uint64_t(outcome) << q;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n_half;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const double2 v = a[insert_zero(i, q) | bit];
    s = fma(v.x, v.x, s);
    s = fma(v.y, v.y, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void k_norm2(const double2* __restrict__ a, uint64_t n, double* __restrict__ partials) {
  __shared__ double red[32];
  double s = 0.0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const double2 v = a[i];
    s = fma(v.x, v.x, s);
    s = fma(v.y, v.y, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// fixed-order (sequential per lane, then butterfly) sum of `count` values
__global__ void k_sum_fixed(const double* __restrict__ in, int count, int stride_out,
                            double* __restrict__ out) {
  const int lane = threadIdx.x;
  double s = 0.0;
  for (int i = lane; i < count; i += 32) s += in[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) out[0] = s;
  (void)stride_out;
}

__global__ void k_project(double2* __restrict__ a, uint64_t n, int q, int outcome, double scale) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    double2 v = a[i];
    if (int((i >> q) & 1) != outcome) {
      v = make_double2(0.0, 0.0);
    } else {
      v.x = v.x * scale;
      v.y = v.y * scale;
    }
    a[i] = v;
  }
}

// numpy: amps.real**2 + amps.imag**2 -- two roundings per product, one per
// sum, no contraction (engine.py:215)
__global__ void k_probabilities(const double2* __restrict__ a, uint64_t n, double* __restrict__ p) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const double2 v = a[i];
    p[i] = __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y));
  }
}

// sum_j conj(a_j) (-1)^popc(j & zmask) a_{j ^ xmask}, per-block complex partials
// Per-chunk sums of |a_i|^2 (chunks of 2^clog amplitudes) for sampling a
// sharded state (sample, engine.py:207-222): one warp per chunk, each lane a
// sequential sum of its strided slice, then a fixed shuffle tree, so the sums
// are deterministic.  Probabilities as in k_probabilities (no contraction).
__global__ void k_prob_chunk_sums(const double2* __restrict__ a, uint64_t n_chunks, int clog,
                                  double* __restrict__ out) {
  const uint64_t lane = threadIdx.x & 31;
  const uint64_t w0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t len = uint64_t(1) << clog;
  for (uint64_t c = w0; c < n_chunks; c += nw) {
    const double2* base = a + (c << clog);
    double s = 0.0;
    for (uint64_t i = lane; i < len; i += 32) {
      const double2 v = base[i];
      s = __dadd_rn(s, __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
    if (lane == 0) out[c] = s;
  }
}

__global__ void k_pauli_term(const double2* __restrict__ a, uint64_t n, uint64_t xmask,
                             uint64_t zmask, double* __restrict__ partials) {
  __shared__ double red[32];
  double sr = 0.0, si = 0.0;
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < n;
       j += uint64_t(gridDim.x) * blockDim.x) {
    const double2 u = a[j], v = a[j ^ xmask];
    double pr = fma(u.x, v.x, u.y * v.y);  // conj(u) * v
    double pi = fma(u.x, v.y, -(u.y * v.x));
    if (__popcll(j & zmask) & 1) {
      pr = -pr;
      pi = -pi;
    }
    sr += pr;
    si += pi;
  }
  sr = block_sum(sr, red);
  si = block_sum(si, red);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = sr;
    partials[2 * blockIdx.x + 1] = si;
  }
}

__global__ void k_sum_fixed2(const double* __restrict__ in, int count, double* __restrict__ out) {
  const int lane = threadIdx.x;
  double sr = 0.0, si = 0.0;
  for (int i = lane; i < count; i += 32) {
    sr += in[2 * i];
    si += in[2 * i + 1];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, off);
    si += __shfl_xor_sync(0xffffffffu, si, off);
  }
  if (lane == 0) {
    out[0] = sr;
    out[1] = si;
  }
}

// ---------------------------------------------------------------------------
// blocked gate-stream kernel

// ---- TMA tiles (planner.h "TMA tiles") --------------------------------------
// Per pass: a tensor map over the whole state whose dims are the tile's qubit
// runs.  dim 0 = qubits 0..2 as 16 doubles (128 bytes, the swizzle span);
// dim i >= 1 covers qubits start[i] .. start[i] + ebits[i] - 1 with the box
// over its lowest run bits (dim 1 starts at qubit 3: a short gap below the
// first run is a traversal stride, a long one a dim with a box of one); the
// last dim reaches qubit n - 1, so tile qubits beyond five dims (`left`) are
// coordinate bits of it, one copy per value, each copy 2^box_bits amplitudes.
// rank 0: the pass's tiles need too many copies and move by cp.async.
struct alignas(64) TmaPass {
  CUtensorMap map;  // 128 bytes
  uint64_t left;
  int8_t start[5];
  int8_t ebits[5];
  int8_t rank;
  int8_t box_bits;
  uint8_t pad[44];
};
static_assert(sizeof(TmaPass) == 192, "TmaPass layout");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred done;\n"
      "NSB_MBAR_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      "@!done bra NSB_MBAR_WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void tma_load(uint32_t dst, const void* map, uint32_t bar, int rank,
                                         const int* c) {
  switch (rank) {
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1])
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]),
          "r"(c[2])
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]),
          "r"(c[1]), "r"(c[2]), "r"(c[3])
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]),
          "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
          : "memory");
      break;
  }
}
// shared -> global, one bulk group per tile (cp.async.bulk.commit_group)
__device__ __forceinline__ void tma_store(const void* map, uint32_t src, int rank, const int* c) {
  switch (rank) {
    case 2:
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];"
                   ::"l"(map), "r"(src), "r"(c[0]), "r"(c[1]) : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
          ::"l"(map), "r"(src), "r"(c[0]), "r"(c[1]), "r"(c[2]) : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];"
          ::"l"(map), "r"(src), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group"
          " [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(map), "r"(src), "r"(c[0]), "r"(c[1]),
          "r"(c[2]), "r"(c[3]), "r"(c[4])
          : "memory");
      break;
  }
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// planner.h swz_tma: the 128-byte TMA swizzle in 16-byte slots
__device__ __forceinline__ int swz_tma(int l) { return l ^ ((l >> 3) & 7); }

struct BlockedParams {
  double2* amps;
  int n;
  const PassDesc* passes;
  int pass_begin, pass_end;
  const GroupDesc* groups;
  const GateOp* ops;
  const double2* mats;
  double* partials;  // 2 * gridDim
  double* record;    // p0 per assertion step
  int* fail;         // [0] flag, [1] step
  unsigned* bar;     // grid-barrier arrival counter (zeroed before each launch)
  double eps;
  int debug;         // timing experiments only (NSB_DEBUG_BLOCKED): 1 skip sweeps, 2 skip HBM,
                     // 4 no CTA rotation
  // chunk restriction (overlapped qubit swaps, nsb_shard_swap_overlap): only
  // the tiles whose physical bits at cmask (out-of-tile qubits of every pass
  // of the launch) equal cval; cbits = popcount(cmask).  0: every tile.
  uint64_t cmask, cval;
  int cbits;
  const TmaPass* tmaps;  // per pass of `passes` (TMA plans, planner.h); else null
  int tma_store;         // TMA passes store their tiles by TMA (else by the threads)
};

// ---- octet sweeps over a shared-memory batch -------------------------------
// A group (planner.h) is applied in one sweep: thread t loads the octet
// {A_t ^ c0 m0 ^ c1 m1 ^ c2 m2} into x[c] (through the read map on the load
// side), applies the group's gates in registers -- x's index c spells the
// octet's logical axis bits, so every gate touches compile-time register
// indices for its axis pattern -- and stores the octet.  Batches live in
// shared memory under the XOR swizzle swz (device.cuh); all offsets are
// swizzled per-bit values precomputed by the planner, combined by XOR.

// (x, y) <- [[m0, m1], [m2, m3]] (x, y)
__device__ __forceinline__ void mix2(double2& x, double2& y, const double2 m0, const double2 m1,
                                     const double2 m2, const double2 m3) {
  double2 ox = make_double2(0.0, 0.0), oy = ox;
  cmac(ox, m0, x);
  cmac(ox, m1, y);
  cmac(oy, m2, x);
  cmac(oy, m3, y);
  x = ox;
  y = oy;
}

// (x, y) <- [[a0, a1], [a2, a3]] (x, y) with real a: the imaginary parts of
// the payload are exact zeros (kPair*r), two multiply-adds per output part
__device__ __forceinline__ void mix2r(double2& x, double2& y, const double a0, const double a1,
                                      const double a2, const double a3) {
  const double2 ox = make_double2(fma(a0, x.x, a1 * y.x), fma(a0, x.y, a1 * y.y));
  const double2 oy = make_double2(fma(a2, x.x, a3 * y.x), fma(a2, x.y, a3 * y.y));
  x = ox;
  y = oy;
}

__device__ __forceinline__ double2 pick(const double2 x0, const double2 x1, const double2 x2,
                                        const double2 x3, int c) {
  double2 r = x0;
  r = c == 1 ? x1 : r;
  r = c == 2 ? x2 : r;
  r = c == 3 ? x3 : r;
  return r;
}

// 2q gate with slot 0 on axis P and slot 1 on axis Q (P < Q) on each of the
// thread's NO octets: two quads per octet, member s of quad h at register
// h | bit(s,0) << P | bit(s,1) << Q.  Matrix entries are read once per gate.
template <int P, int Q, int C, int NO>
__device__ __forceinline__ void gate2(double2 (&xs)[NO][8], const GateOp o,
                                      const double2* __restrict__ m) {
  constexpr int R = 3 - P - Q;
  constexpr int A = 1 << P, B = 1 << Q, H = 1 << R;
  switch (C) {
    case kCX01:  // swaps members 1, 3
#pragma unroll
      for (int q = 0; q < NO; ++q)
#pragma unroll
        for (int h = 0; h <= H; h += H) {
          const double2 t = xs[q][h | A];
          xs[q][h | A] = xs[q][h | A | B];
          xs[q][h | A | B] = t;
        }
      break;
    case kCX10:  // swaps members 2, 3
#pragma unroll
      for (int q = 0; q < NO; ++q)
#pragma unroll
        for (int h = 0; h <= H; h += H) {
          const double2 t = xs[q][h | B];
          xs[q][h | B] = xs[q][h | A | B];
          xs[q][h | A | B] = t;
        }
      break;
    case kSwap:  // swaps members 1, 2
#pragma unroll
      for (int q = 0; q < NO; ++q)
#pragma unroll
        for (int h = 0; h <= H; h += H) {
          const double2 t = xs[q][h | A];
          xs[q][h | A] = xs[q][h | B];
          xs[q][h | B] = t;
        }
      break;
    case kPairQ:
    case kPairP:
    case kPairX: {  // blocks: Q (0,2),(1,3); P (0,1),(2,3); X (0,3),(1,2)
      constexpr int u1 = C == kPairQ ? B : (C == kPairP ? A : A | B);
      constexpr int u2 = C == kPairQ ? A : (C == kPairP ? B : A);
      constexpr int u3 = C == kPairQ ? A | B : (C == kPairP ? A | B : B);
      const double2 m0 = m[0], m1 = m[1], m2 = m[2], m3 = m[3];
      const double2 n0 = m[4], n1 = m[5], n2 = m[6], n3 = m[7];
#pragma unroll
      for (int q = 0; q < NO; ++q)
#pragma unroll
        for (int h = 0; h <= H; h += H) {
          mix2(xs[q][h], xs[q][h | u1], m0, m1, m2, m3);
          mix2(xs[q][h | u2], xs[q][h | u3], n0, n1, n2, n3);
        }
      break;
    }
    case kPairQr:
    case kPairPr:
    case kPairXr: {
      constexpr int u1 = C == kPairQr ? B : (C == kPairPr ? A : A | B);
      constexpr int u2 = C == kPairQr ? A : (C == kPairPr ? B : A);
      constexpr int u3 = C == kPairQr ? A | B : (C == kPairPr ? A | B : B);
      const double a0 = m[0].x, a1 = m[1].x, a2 = m[2].x, a3 = m[3].x;
      const double b0 = m[4].x, b1 = m[5].x, b2 = m[6].x, b3 = m[7].x;
#pragma unroll
      for (int q = 0; q < NO; ++q)
#pragma unroll
        for (int h = 0; h <= H; h += H) {
          mix2r(xs[q][h], xs[q][h | u1], a0, a1, a2, a3);
          mix2r(xs[q][h | u2], xs[q][h | u3], b0, b1, b2, b3);
        }
      break;
    }
    case kDiag2: {
      const double2 d0 = m[0], d1 = m[1], d2 = m[2], d3 = m[3];
#pragma unroll
      for (int q = 0; q < NO; ++q)
#pragma unroll
        for (int h = 0; h <= H; h += H) {
          xs[q][h] = cmul(d0, xs[q][h]);
          xs[q][h | A] = cmul(d1, xs[q][h | A]);
          xs[q][h | B] = cmul(d2, xs[q][h | B]);
          xs[q][h | A | B] = cmul(d3, xs[q][h | A | B]);
        }
      break;
    }
    case kMono2: {
      const double2 v0 = m[0], v1 = m[1], v2 = m[2], v3 = m[3];
      const int c0 = o.cols & 3, c1 = (o.cols >> 2) & 3, c2 = (o.cols >> 4) & 3,
                c3 = (o.cols >> 6) & 3;
#pragma unroll
      for (int q = 0; q < NO; ++q)
#pragma unroll
        for (int h = 0; h <= H; h += H) {
          const double2 x0 = xs[q][h], x1 = xs[q][h | A], x2 = xs[q][h | B],
                        x3 = xs[q][h | A | B];
          xs[q][h] = cmul(v0, pick(x0, x1, x2, x3, c0));
          xs[q][h | A] = cmul(v1, pick(x0, x1, x2, x3, c1));
          xs[q][h | B] = cmul(v2, pick(x0, x1, x2, x3, c2));
          xs[q][h | A | B] = cmul(v3, pick(x0, x1, x2, x3, c3));
        }
      break;
    }
    case kSparse2: {
      const unsigned cols = o.cols;
      double2 out[NO][2][4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double2 ma = m[2 * r], mb = m[2 * r + 1];
        const int ca = (cols >> (4 * r)) & 3, cb = (cols >> (4 * r + 2)) & 3;
#pragma unroll
        for (int q = 0; q < NO; ++q)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int h = hh * H;
            const double2 x0 = xs[q][h], x1 = xs[q][h | A], x2 = xs[q][h | B],
                          x3 = xs[q][h | A | B];
            double2 acc = make_double2(0.0, 0.0);
            cmac(acc, ma, pick(x0, x1, x2, x3, ca));
            cmac(acc, mb, pick(x0, x1, x2, x3, cb));
            out[q][hh][r] = acc;
          }
      }
#pragma unroll
      for (int q = 0; q < NO; ++q)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int h = hh * H;
          xs[q][h] = out[q][hh][0];
          xs[q][h | A] = out[q][hh][1];
          xs[q][h | B] = out[q][hh][2];
          xs[q][h | A | B] = out[q][hh][3];
        }
      break;
    }
    default: {  // kDense2
      double2 out[NO][2][4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double2 w0 = m[4 * r], w1 = m[4 * r + 1], w2 = m[4 * r + 2], w3 = m[4 * r + 3];
#pragma unroll
        for (int q = 0; q < NO; ++q)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int h = hh * H;
#ifdef NSB_DENSE_ROWS
            double2 acc = make_double2(0.0, 0.0);
            cmac(acc, w0, xs[q][h]);
            cmac(acc, w1, xs[q][h | A]);
            cmac(acc, w2, xs[q][h | B]);
            cmac(acc, w3, xs[q][h | A | B]);
            out[q][hh][r] = acc;
#else
            out[q][hh][r] = make_double2(0.0, 0.0);
#endif
          }
#ifndef NSB_DENSE_ROWS
        // column-major: consecutive multiply-adds share the matrix operand
        // (register reuse; measured 1.4 % faster on rand28 than row chains)
        const double2 wc[4] = {w0, w1, w2, w3};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int cm = ((c & 1) ? A : 0) | ((c & 2) ? B : 0);
#pragma unroll
          for (int q = 0; q < NO; ++q)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) out[q][hh][r].x = fma(wc[c].x, xs[q][hh * H | cm].x, out[q][hh][r].x);
#pragma unroll
          for (int q = 0; q < NO; ++q)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) out[q][hh][r].x = fma(-wc[c].y, xs[q][hh * H | cm].y, out[q][hh][r].x);
#pragma unroll
          for (int q = 0; q < NO; ++q)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) out[q][hh][r].y = fma(wc[c].x, xs[q][hh * H | cm].y, out[q][hh][r].y);
#pragma unroll
          for (int q = 0; q < NO; ++q)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) out[q][hh][r].y = fma(wc[c].y, xs[q][hh * H | cm].x, out[q][hh][r].y);
        }
#endif
      }
#pragma unroll
      for (int q = 0; q < NO; ++q)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int h = hh * H;
          xs[q][h] = out[q][hh][0];
          xs[q][h | A] = out[q][hh][1];
          xs[q][h | B] = out[q][hh][2];
          xs[q][h | A | B] = out[q][hh][3];
        }
      break;
    }
  }
}

// 1q gate on axis P: pairs (c, c | 1 << P) of each octet
template <int P, int C, int NO>
__device__ __forceinline__ void gate1(double2 (&xs)[NO][8], const GateOp,
                                      const double2* __restrict__ m) {
  constexpr int A = 1 << P;
  constexpr int L0 = P == 0 ? 2 : 1, L1 = P == 2 ? 2 : 4;  // the other two axes
  if (C == kDiag1) {
    const double2 d0 = m[0], d1 = m[1];
#pragma unroll
    for (int q = 0; q < NO; ++q)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c = ((i & 1) ? L0 : 0) | ((i & 2) ? L1 : 0);
        xs[q][c] = cmul(d0, xs[q][c]);
        xs[q][c | A] = cmul(d1, xs[q][c | A]);
      }
  } else {
    const double2 m0 = m[0], m1 = m[1], m2 = m[2], m3 = m[3];
#pragma unroll
    for (int q = 0; q < NO; ++q)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c = ((i & 1) ? L0 : 0) | ((i & 2) ? L1 : 0);
        mix2(xs[q][c], xs[q][c | A], m0, m1, m2, m3);
      }
  }
}

// Whole-octet ops (planner group fusion, planner.h kPatT* / kPatAll).
// 2x2 on axis T with one block per value of the other two axes (L0 lower).
template <int T, int NO>
__device__ __forceinline__ void gate_octet_axis(double2 (&xs)[NO][8],
                                                const double2* __restrict__ m) {
  constexpr int A = 1 << T;
  constexpr int L0 = T == 0 ? 2 : 1, L1 = T == 2 ? 2 : 4;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int c = ((b & 1) ? L0 : 0) | ((b & 2) ? L1 : 0);
    const double2 m0 = m[4 * b], m1 = m[4 * b + 1], m2 = m[4 * b + 2], m3 = m[4 * b + 3];
#pragma unroll
    for (int q = 0; q < NO; ++q) mix2(xs[q][c], xs[q][c | A], m0, m1, m2, m3);
  }
}

// 4x4 on axes (P, Q) with one block per value of the third axis (whole-octet
// op of planner group fusion, kPatD*): block hh at m + 16 hh, column-major
template <int P, int Q, int NO>
__device__ __forceinline__ void gate_octet_pair(double2 (&xs)[NO][8],
                                                const double2* __restrict__ m) {
  constexpr int A = 1 << P, B = 1 << Q, H = 7 ^ A ^ B;
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int h = hh ? H : 0;
    const double2* w = m + 16 * hh;
    double2 out[NO][4];
#pragma unroll
    for (int q = 0; q < NO; ++q)
#pragma unroll
      for (int r = 0; r < 4; ++r) out[q][r] = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double2 wc = w[4 * r + c];
        const int cm = h | ((c & 1) ? A : 0) | ((c & 2) ? B : 0);
#pragma unroll
        for (int q = 0; q < NO; ++q) cmac(out[q][r], wc, xs[q][cm]);
      }
#pragma unroll
    for (int q = 0; q < NO; ++q) {
      xs[q][h] = out[q][0];
      xs[q][h | A] = out[q][1];
      xs[q][h | B] = out[q][2];
      xs[q][h | A | B] = out[q][3];
    }
  }
}

// Register-axis exchange (four-axis groups): octet position P <-> octet index
// (the planner emits these only for the two-octet layout: a no-op otherwise)
template <int P, int NO>
__device__ __forceinline__ void swap_axis_q(double2 (&xs)[NO][8]) {
  if constexpr (NO == 2) {
    constexpr int A = 1 << P;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (!(c & A)) {
        const double2 t = xs[0][c | A];
        xs[0][c | A] = xs[NO - 1][c];
        xs[NO - 1][c] = t;
      }
  }
}

// Register CX (four-axis groups): registers c' = c with bit K ^= bit J over
// the 16 registers of the two octets (bit 3 = octet index)
template <int J, int K, int NO>
__device__ __forceinline__ void reg_cx(double2 (&xs)[NO][8]) {
  if constexpr (NO == 2 || (J < 3 && K < 3)) {  // octet-index bits need two octets
#pragma unroll
    for (int c = 0; c < 8 * NO; ++c)
      if ((c >> J & 1) && !(c >> K & 1)) {
        const int e = c | (1 << K);
        const double2 t = xs[c >> 3][c & 7];
        xs[c >> 3][c & 7] = xs[e >> 3][e & 7];
        xs[e >> 3][e & 7] = t;
      }
  }
}

template <int NO>
__device__ __forceinline__ void gate_octet_diag(double2 (&xs)[NO][8],
                                                const double2* __restrict__ m) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double2 d = m[c];
#pragma unroll
    for (int q = 0; q < NO; ++q) xs[q][c] = cmul(d, xs[q][c]);
  }
}

// Per pass, the thread part of every group's octet address is tabulated:
// entry e of table 0 (table 1) is the XOR of the swizzled offsets of thread
// bits 0..3 (4..7) set in e -- store side in bits 0..15, load side (through
// the read map) in bits 16..31.
__device__ __forceinline__ uint32_t thread_table_entry(const GroupDesc& d, int e) {
  const int half = e >> 4, bits = e & 15;
  uint32_t v = 0;
  for (int b = 0; b < 4; ++b)
    if (bits >> b & 1) {
      const int tb = 4 * half + b;
      v ^= d.tcol[tb];
      v ^= static_cast<uint32_t>(d.rtcol[tb]) << 16;
    }
  return v;
}

// One octet sweep: src -> registers -> dst (different buffers).  Thread t
// owns octets t + j T (j < kOctets, T = kPassThreads; octet-index bit
// kThreadBits selects the second octet -- a fourth axis in four-axis
// groups).  `kap` holds 8 parity bits per tile of the batch (the axes'
// out-of-tile rows): 4 for the load placement, 4 for the store placement.
template <int NO>
__device__ __forceinline__ void apply_group(const double2* __restrict__ src,
                                            double2* __restrict__ dst, int k, int nvalid,
                                            const GroupDesc& G, const GateOp* __restrict__ ops,
                                            const double2* __restrict__ mats, unsigned kap,
                                            const uint32_t* ttab) {
  constexpr int TB = NO == 2 ? 7 : 8;  // thread bits of the layout (planner.cpp)
  const int t = threadIdx.x;
  const int cb = k - 3;
  // Every thread sweeps both of its octets.  Octets past the batch's valid
  // tiles (a short last batch, or k < 8) address the unused part of the
  // 2^11-amplitude buffer: they move garbage that is never stored to global
  // memory, which is cheaper than predicating every load and store (a warp
  // none of whose octets is valid skips the sweep altogether: see k_blocked).

  const GateOp first = ops[0];  // (unused by read-map-only sweeps)
  const uint32_t v = ttab[t & 15] ^ ttab[16 + (t >> 4)];
  const int m0 = G.am[0], m1 = G.am[1], m2 = G.am[2];
  const int r0 = G.ram[0], r1 = G.ram[1], r2 = G.ram[2];
  int a[NO], r[NO];
#pragma unroll
  for (int q = 0; q < NO; ++q) {
    const int oi = t + (q << TB);
    a[q] = (v & 0xffffu) ^ (q ? G.tcol[TB] : 0);
    r[q] = (v >> 16) ^ (q ? G.rtcol[TB] : 0);
    const int sh = 8 * (oi >> cb);  // tiles >= 4 exist only as garbage octets
    const unsigned kp = sh < 32 ? (kap >> sh) & 0xffu : 0u;
    if (kp & 1) r[q] ^= r0;
    if (kp & 2) r[q] ^= r1;
    if (kp & 4) r[q] ^= r2;
    if (NO == 2 && (kp & 8)) r[q] ^= G.rtcol[NO == 2 ? TB : 0];
    if (kp & 16) a[q] ^= m0;
    if (kp & 32) a[q] ^= m1;
    if (kp & 64) a[q] ^= m2;
    if (NO == 2 && (kp & 128)) a[q] ^= G.tcol[NO == 2 ? TB : 0];
  }
  double2 x[NO][8];
#pragma unroll
  for (int q = 0; q < NO; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c)
#ifdef NSB_SWEEP_NOMEM  // timing experiment (tools/sweep_exp.sh): gate arithmetic only
      x[q][c] = make_double2(double(r[q] + c), double(a[q] - c));
#else
      x[q][c] = src[r[q] ^ ((c & 1) ? r0 : 0) ^ ((c & 2) ? r1 : 0) ^ ((c & 4) ? r2 : 0)];
#endif
  const int n_ops = G.n_ops();
  auto store = [&]() {
#pragma unroll
    for (int q = 0; q < NO; ++q)
#pragma unroll
      for (int c = 0; c < 8; ++c)
#ifdef NSB_SWEEP_NOMEM
        if (x[q][c].x == 1234.5678) dst[a[q] ^ c] = x[q][c];
#else
        dst[a[q] ^ ((c & 1) ? m0 : 0) ^ ((c & 2) ? m1 : 0) ^ ((c & 4) ? m2 : 0)] = x[q][c];
#endif
  };
  // Gate dispatch: pattern * 16 + class selects straight-line register code.
  // The LAST gate of a group stores its octets from inside its own case, so
  // the common one-gate group never merges the 64-register octet pair across
  // the dispatch (the merge costs the allocator a full copy).
  auto dispatch = [&](const GateOp o, bool last) __attribute__((always_inline)) {
    const double2* m = mats + o.mat;
#ifndef NSB_NO_HOTPATH
    // the dominant kinds first (deep21: whole-octet 2x2 51 %, 4x4-per-third-axis
    // 18 %; rand28: dense 4x4 on axes 0,1 66 %), ahead of the switch's
    // compare-and-branch tree
    if (o.kind == op_kind(kPatT0, kDense1)) {
      gate_octet_axis<0, NO>(x, m);
      if (last) store();
      return;
    }
    if (o.kind == op_kind(kPatD01, kDense2)) {
      gate_octet_pair<0, 1, NO>(x, m);
      if (last) store();
      return;
    }
    if (o.kind == op_kind(kPat01, kDense2)) {
      gate2<0, 1, kDense2, NO>(x, o, m);
      if (last) store();
      return;
    }
#endif
    switch (o.kind) {
#define NSB_G2(P, Q, PAT, C)                                             \
  case op_kind(PAT, C):                                                     \
    gate2<P, Q, C, NO>(x, o, m);                                         \
    if (last) store();                                                   \
    break;
#define NSB_G2ALL(P, Q, PAT)                                             \
  NSB_G2(P, Q, PAT, kDense2) NSB_G2(P, Q, PAT, kSparse2)                 \
  NSB_G2(P, Q, PAT, kMono2) NSB_G2(P, Q, PAT, kDiag2)                    \
  NSB_G2(P, Q, PAT, kCX01) NSB_G2(P, Q, PAT, kCX10)                      \
  NSB_G2(P, Q, PAT, kPairQ) NSB_G2(P, Q, PAT, kPairP)                    \
  NSB_G2(P, Q, PAT, kPairX) NSB_G2(P, Q, PAT, kSwap)                    \
  NSB_G2(P, Q, PAT, kPairQr) NSB_G2(P, Q, PAT, kPairPr)                  \
  NSB_G2(P, Q, PAT, kPairXr)
#define NSB_G1(P, PAT, C)                                                \
  case op_kind(PAT, C):                                                     \
    gate1<P, C, NO>(x, o, m);                                            \
    if (last) store();                                                   \
    break;
      NSB_G2ALL(0, 1, kPat01)
      NSB_G2ALL(0, 2, kPat02)
      NSB_G2ALL(1, 2, kPat12)
      NSB_G1(0, kPat0, kDense1) NSB_G1(0, kPat0, kDiag1)
      NSB_G1(1, kPat1, kDense1) NSB_G1(1, kPat1, kDiag1)
      NSB_G1(2, kPat2, kDense1) NSB_G1(2, kPat2, kDiag1)
#define NSB_GT(T)                                                        \
  case op_kind(kPatT0 + T, kDense1):                                      \
    gate_octet_axis<T, NO>(x, m);                                        \
    if (last) store();                                                   \
    break;
      NSB_GT(0) NSB_GT(1) NSB_GT(2)
#define NSB_GD(P, Q, PAT)                                                \
  case op_kind(PAT, kDense2):                                            \
    gate_octet_pair<P, Q, NO>(x, m);                                     \
    if (last) store();                                                   \
    break;
      NSB_GD(0, 1, kPatD01) NSB_GD(0, 2, kPatD02) NSB_GD(1, 2, kPatD12)
#undef NSB_GD
      case op_kind(kPatAll, kDiag1):
        gate_octet_diag<NO>(x, m);
        if (last) store();
        break;
#if NSB_OCTETS == 2
#define NSB_GQ(P)                                                        \
  case reg_swap_kind(P):                                                 \
    swap_axis_q<P, NO>(x);                                               \
    if (last) store();                                                   \
    break;
      NSB_GQ(0) NSB_GQ(1) NSB_GQ(2)
#undef NSB_GQ
#endif
#define NSB_RCX(J, K)                                                    \
  case reg_cx_kind(J, K):                                                \
    reg_cx<J, K, NO>(x);                                                 \
    if (last) store();                                                   \
    break;
      NSB_RCX(0, 1) NSB_RCX(0, 2) NSB_RCX(1, 0) NSB_RCX(1, 2) NSB_RCX(2, 0) NSB_RCX(2, 1)
#if NSB_OCTETS == 2
      NSB_RCX(0, 3) NSB_RCX(1, 3) NSB_RCX(2, 3) NSB_RCX(3, 0) NSB_RCX(3, 1) NSB_RCX(3, 2)
#endif
#undef NSB_RCX
#undef NSB_GT
#undef NSB_G1
#undef NSB_G2ALL
#undef NSB_G2
      default:
        if (last) store();
        break;
    }
  };
#ifdef NSB_SWEEP_NOOPS  // timing experiment (tools/sweep_exp.sh): loads and stores only
  if (true) {
#else
  if (n_ops == 0) {
#endif
    store();
    return;
  }
#ifndef NSB_NO_PREFETCH
  // each op's descriptor is read one op ahead (the first one before the
  // octet loads), so the dispatch branch does not wait on a shared load
  GateOp o = first;
#pragma unroll 1
  for (int i = 0; i + 1 < n_ops; ++i) {
    const GateOp nx = ops[i + 1];
    dispatch(o, false);
    o = nx;
  }
  dispatch(o, true);
#else
#pragma unroll 1
  for (int i = 0; i + 1 < n_ops; ++i) dispatch(ops[i], false);
  dispatch(ops[n_ops - 1], true);
#endif
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// One persistent CTA per SM; while the gate sweeps of tile i run, tile i+1 of
// the same pass streams into the other shared-memory buffer with cp.async.
constexpr size_t kBlockedSmemBytes = sizeof(double2) * (3 * kTileAmpsMax + kMaxPassMats) +
                                     sizeof(GroupDesc) * kMaxPassGates +
                                     sizeof(GateOp) * kMaxPassOps;
// TMA plans: the batch buffers start on a 1024-byte boundary (128-byte swizzle)
constexpr size_t kBlockedSmemBytesTma = kBlockedSmemBytes + 1024;

// kChunk: the chunk-restricted instantiation (overlapped swaps); the plain
// one compiles the restriction away (its address math is the hot loop's).
// kTma: a TMA plan (planner.h): tiles hold qubits 0..2, k = kTileQubitsMax,
// the pass-edge layout is swz_tma.  Without kChunk the tiles move by
// cp.async.bulk.tensor (one elected thread issues, an mbarrier per buffer
// counts the bytes in, bulk groups track the stores); the chunk-restricted
// instantiation keeps per-thread cp.async under the same layout.
// kOct: the thread layout the plan was laid out for (HostPlan::octets): two
// octets per thread and 128 threads, or one octet and 256 threads (small
// states)
template <bool kChunk, bool kTma, int kOct = kOctets>
__global__ void __launch_bounds__(kOct == 2 ? (1 << NSB_THREAD_BITS) : 256, kCtasPerSm)
    k_blocked(BlockedParams p) {
  constexpr bool kHw = kTma && !kChunk;
  constexpr int kThreadBits = kOct == 2 ? nsb::kThreadBits : 8;  // the layout's (shadows planner.h)
  constexpr int kPassThreads = 1 << kThreadBits;
  const uint64_t c_mask = kChunk ? p.cmask : 0, c_val = kChunk ? p.cval : 0;
  const int c_bits = kChunk ? p.cbits : 0;
  // dynamic shared memory: 3 batch buffers (current, gate-sweep target,
  // prefetch) | pass matrices | pass group descriptors | gate ops
  extern __shared__ __align__(128) double2 smem_raw[];
  double2* smem = smem_raw;
  if constexpr (kTma) smem += ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) / sizeof(double2);
  // shared-memory slot of a tile-local amplitude at the pass edges (loads,
  // collapse, stores): the TMA layout in a TMA pass (sp.tma) of a TMA plan
  double2* s_mats = smem + 3 * kTileAmpsMax;
  GroupDesc* s_groups = reinterpret_cast<GroupDesc*>(s_mats + kMaxPassMats);
  GateOp* s_ops = reinterpret_cast<GateOp*>(s_groups + kMaxPassGates);
  __shared__ PassDesc sp;
  __shared__ uint64_t s_hi[1 << (kTileQubitsMax - 7)];  // offsets of tile bits >= kThreadBits
  __shared__ unsigned s_gm[kMaxPassGates];  // per group: out-of-tile axis parities per batch tile
  __shared__ uint32_t s_ttab[kMaxPassGates][32];  // per group: thread-address tables
  __shared__ double red[32];
  __shared__ double s_p0;
  __shared__ uint64_t s_omask;  // physical mask of the pass's out-of-tile qubits
  __shared__ __align__(8) uint64_t s_mbar[3];  // TMA: bytes landed per batch buffer
  __shared__ uint64_t s_tleft;                 // TMA: the pass's TmaPass fields
  __shared__ int8_t s_tstart[5], s_tebits[5], s_trank, s_tbox;
  const int tid = threadIdx.x;
  double carry_p0 = 1.0;  // p0 of the previous pass's assertion (collapse input)
  unsigned n_bar = 0;     // grid barriers passed in this launch
  unsigned mph = 0;       // TMA: mbarrier phase to wait for, per buffer (bit b)
  // slot of tile-local amplitude (b << k) + tid + (j << kThreadBits): in a TMA
  // pass the copy layout permutes the tile bits (PassDesc::tperm) under swz_tma
  bool etma = false;
  int k_cur = 0;   // the pass's tile qubits
  int pi_tid = 0;  // TMA pass: the permuted index of this thread's bits
  __shared__ int s_pij[1 << (kTileQubitsMax - 7)];  // ... of j << kThreadBits
  auto eslot = [&](int b, int j) {
    if (kTma && etma) return swz_tma(pi_tid ^ s_pij[j]);
    return swz((b << k_cur) + tid + (j << kThreadBits));
  };
  if constexpr (kHw) {
    if (tid == 0) {
      for (int b = 0; b < 3; ++b) mbar_init(smem_u32(&s_mbar[b]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // (stage() below opens with a CTA barrier)
  }

  // Stage pass pi's descriptors in shared memory.  Called for the next pass
  // right before the grid barrier, so the copy overlaps the wait.
  auto stage = [&](int pi) {
    __syncthreads();  // the previous pass is done with sp and the tables
    if (tid < int(sizeof(PassDesc) / sizeof(int)))
      reinterpret_cast<int*>(&sp)[tid] = reinterpret_cast<const int*>(p.passes + pi)[tid];
    __syncthreads();
    const int n_mat = sp.mat_count;
    for (int i = tid; i < n_mat; i += kPassThreads) s_mats[i] = p.mats[sp.mat_begin + i];
    const int n_words = (sp.group_end - sp.group_begin) * int(sizeof(GroupDesc) / 8);
    const uint64_t* src = reinterpret_cast<const uint64_t*>(p.groups + sp.group_begin);
    uint64_t* dst = reinterpret_cast<uint64_t*>(s_groups);
    for (int i = tid; i < n_words; i += kPassThreads) dst[i] = src[i];
    const int n_ow = sp.op_end - sp.op_begin;
    const uint64_t* osrc = reinterpret_cast<const uint64_t*>(p.ops + sp.op_begin);
    uint64_t* odst = reinterpret_cast<uint64_t*>(s_ops);
    for (int i = tid; i < n_ow; i += kPassThreads) odst[i] = osrc[i];
    __syncthreads();
    const int n_entries = (sp.group_end - sp.group_begin) * 32;
    for (int e = tid; e < n_entries; e += kPassThreads)
      s_ttab[e >> 5][e & 31] = thread_table_entry(s_groups[e >> 5], e & 31);
    if (tid == 0) {
      uint64_t m = 0;
      for (int b = 0; b < p.n - sp.k; ++b) m |= uint64_t(1) << sp.oq[b];
      s_omask = m & ~c_mask;
      if constexpr (kHw) {
        const TmaPass& T = p.tmaps[pi];
        s_tleft = T.left;
        for (int i = 0; i < 5; ++i) {
          s_tstart[i] = T.start[i];
          s_tebits[i] = T.ebits[i];
        }
        s_trank = T.rank;
        s_tbox = T.box_bits;
      }
    }
    constexpr int kHi = kTileQubitsMax - kThreadBits;
    if (kTma && sp.tma && tid < (1 << kHi)) {
      int v = 0;
      for (int b = 0; b < kHi; ++b)
        if (tid >> b & 1) v |= 1 << sp.tperm[kThreadBits + b];
      s_pij[tid] = v;
    }
    if (tid < (1 << kHi)) {
      uint64_t h = 0;
      for (int b = 0; b < kHi; ++b)
        if ((tid >> b & 1) && kThreadBits + b < sp.k) h |= uint64_t(1) << sp.tq[kThreadBits + b];
      s_hi[tid] = h;
    }
    __syncthreads();
  };
  if (p.eps >= 0.0 && p.fail[0]) return;  // an earlier launch of this MMA run failed its assertion
  if (p.pass_begin < p.pass_end) stage(p.pass_begin);
  // a launch that starts with a collapse (streamed MMA runs: one launch per
  // part between assertions) takes p0 from the record the previous launch wrote
  if (p.pass_begin < p.pass_end && sp.collapse_q >= 0) carry_p0 = p.record[sp.collapse_slot];

  for (int pi = p.pass_begin; pi < p.pass_end; ++pi) {
    const int k = sp.k;
    const int lo_bits = k < kThreadBits ? k : kThreadBits;
    uint64_t lo = 0;  // global offset of this thread's low tile-local bits
    for (int b = 0; b < lo_bits; ++b)
      if (tid >> b & 1) lo |= uint64_t(1) << sp.tq[b];
    __syncthreads();
    const int n_out = p.n - k;
    const uint64_t n_tiles = uint64_t(1) << (n_out - c_bits);
    const int n_j = k > kThreadBits ? 1 << (k - kThreadBits) : 1;
    const bool loader = tid < (1 << lo_bits);
    const double cscale = sp.collapse_q >= 0 ? 1.0 / sqrt(carry_p0) : 1.0;
    const int n_groups = sp.group_end - sp.group_begin;
    double msum = 0.0;
    // TMA plans: this pass's tiles move by TMA (the planner's choice, sp.tma);
    // the chunk-restricted instantiation moves them by cp.async in that layout
    etma = kTma && sp.tma;
    k_cur = k;
    const bool tp = kHw && etma;
    // ... and are stored by TMA too (p.tma_store), else by the threads (the
    // next tile is then requested at the start of a tile, not after its first
    // sweep: no store is reading the buffer it lands in)
    const bool ts = tp && p.tma_store;
    if (kTma && etma) {
      pi_tid = 0;
      for (int b = 0; b < kThreadBits; ++b)
        if (tid >> b & 1) pi_tid |= 1 << sp.tperm[b];
    }

    auto tile_base = [&](uint64_t t) {  // physical index bits of tile t (no tile-local bits)
      uint64_t base = 0;
      if constexpr (!kChunk) {
        for (int b = 0; b < n_out; ++b)
          if (t >> b & 1) base |= uint64_t(1) << sp.oq[b];
      } else {
        base = c_val;
        for (int b = 0, j = 0; b < n_out; ++b) {
          const uint64_t qb = uint64_t(1) << sp.oq[b];
          if (c_mask & qb) continue;  // a chunk bit: fixed to cval
          if (t >> j++ & 1) base |= qb;
        }
      }
      return base;
    };
    // contiguous tile range of this CTA, processed in batches of nb tiles
    const int nb = k >= kTileQubitsMax ? 1 : min(1 << (kTileQubitsMax - k), 4);
    const uint64_t per = n_tiles / gridDim.x, extra = n_tiles % gridDim.x;
    // the CTAs holding the extra tiles alternate between passes, so the CTA
    // that arrived last at a barrier (and stages after arriving) is not
    // again the slowest in the next pass
    const unsigned vb = (p.debug & 4) ? blockIdx.x
                                      : (blockIdx.x + ((pi & 1) ? gridDim.x / 2 : 0)) % gridDim.x;
    const uint64_t t_begin = vb * per + (vb < extra ? vb : extra);
    const uint64_t t_end = t_begin + per + (vb < extra ? 1 : 0);
    // tile t+1's base from tile t's: increment within the out-of-tile mask
    const uint64_t omask = s_omask;
    auto next_base = [&](uint64_t b) {
      if constexpr (!kChunk) return ((b | ~omask) + 1) & omask;
      return (((b | ~omask) + 1) & omask) | c_val;
    };
    auto issue_batch = [&](uint64_t t0, uint64_t base0, double2* buf) {
      if (!loader || (p.debug & 2)) return;
      uint64_t base = base0 | lo;
#pragma unroll 1
      for (int b = 0; b < nb && t0 + b < t_end; ++b) {
        double2* dst = buf;
#pragma unroll 2
        for (int j = 0; j < n_j; ++j)
          cp_async16(dst + eslot(b, j), p.amps + (base | s_hi[j]));
        base = next_base(base & omask) | lo;
      }
    };
    // TMA (one thread): the tile at physical base `base` <-> buffer bi, one
    // copy per value of the tile qubits beyond the map's dims
    auto tma_tile = [&](bool store, uint64_t base, int bi) {
      const void* map = &p.tmaps[pi].map;
      const uint64_t left = s_tleft;
      const int rank = s_trank, box = s_tbox;
      const uint32_t buf = smem_u32(smem + bi * kTileAmpsMax);
      const uint32_t bar = smem_u32(&s_mbar[bi]);
      if (!store) mbar_expect_tx(bar, kTileAmpsMax * sizeof(double2));
      const int nl = __popcll(left);
#pragma unroll 1
      for (int v = 0; v < (1 << nl); ++v) {
        uint64_t g = base;
        int j = 0;
        for (uint64_t m = left; m; m &= m - 1, ++j)
          if (v >> j & 1) g |= m & (0 - m);
        int c[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int i = 1; i < 5; ++i)
          if (i < rank) c[i] = static_cast<int>((g >> s_tstart[i]) & ((uint64_t(1) << s_tebits[i]) - 1));
        const uint32_t at = buf + (static_cast<uint32_t>(v) << (box + 4));
        if (store)
          tma_store(map, at, rank, c);
        else
          tma_load(at, map, bar, rank, c);
      }
      if (store) bulk_commit();
    };

    int cur = 0, pre = 1, spare = 2;  // buffer roles (rotate)
    uint64_t bnext = t_begin < t_end ? tile_base(t_begin) : 0;  // base of the batch's first tile
    if (tp) {
      if (tid == 0 && t_begin < t_end && !(p.debug & 2)) tma_tile(false, bnext, 0);
    } else {
      if (t_begin < t_end) issue_batch(t_begin, bnext, smem);
      cp_async_commit();
    }
    for (uint64_t t0 = t_begin; t0 < t_end; t0 += nb) {
      double2* tile = smem + cur * kTileAmpsMax;
      const int nvalid = t_end - t0 < uint64_t(nb) ? static_cast<int>(t_end - t0) : nb;
      uint64_t tbase[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        tbase[b] = b < nvalid ? bnext : 0;
        if (b < nb) bnext = next_base(bnext);  // ends as the next batch's first base
      }
      // TMA: the next tile is requested after this tile's first sweep (its
      // buffer is the one the previous tile's TMA store is still reading)
      const bool pending = tp && t0 + nb < t_end && !(p.debug & 2);
      const bool early = !ts || (p.debug & 16);  // request at the tile start
      auto request_next = [&]() {
        if (tid == 0) {
          bulk_wait_read0();
          tma_tile(false, bnext, pre);
        }
      };
      if (tp) {
        if (!(p.debug & 2)) mbar_wait(smem_u32(&s_mbar[cur]), (mph >> cur) & 1u);
        mph ^= 1u << cur;
        if (pending && early) request_next();
      } else {
        if (t0 + nb < t_end) issue_batch(t0 + nb, bnext, smem + pre * kTileAmpsMax);
        cp_async_commit();
        cp_async_wait<1>();  // this batch has landed (the next may be in flight)
      }
      if (tid < n_groups) {  // out-of-tile axis parities per (group, tile of the batch)
        const GroupDesc& d = s_groups[tid];
        unsigned gm = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (b < nvalid) {
            unsigned kl = 0;  // per axis (= load position)
#pragma unroll
            for (int i = 0; i < 4; ++i) kl |= (__popcll(tbase[b] & d.r_out[i]) & 1u) << i;
            unsigned ks = 0;  // per store position: parity of the load rows summing to its row
#pragma unroll
            for (int j = 0; j < 4; ++j) ks |= (__popc(kl & (d.kmat >> (4 * j)) & 15u) & 1u) << j;
            gm |= (kl | ks << 4) << (8 * b);
          }
        }
        s_gm[tid] = gm;
      }
      __syncthreads();
      if (sp.collapse_q >= 0) {  // pending collapse (engine.py:164-167)
        const int cq = sp.collapse_q;
        uint64_t bb = tbase[0];
        if (loader)
#pragma unroll 1
          for (int b = 0; b < 4; ++b, bb = next_base(bb))
#pragma unroll 1
            for (int j = 0; j < n_j && b < nvalid; ++j) {
              const uint64_t g = bb | lo | s_hi[j];
              double2& v = tile[eslot(b, j)];
              if ((g >> cq) & 1) {
                v = make_double2(0.0, 0.0);
              } else {
                v.x *= cscale;
                v.y *= cscale;
              }
            }
        __syncthreads();
      }
      // small states (8 qubits fill 32 octets): warps without a valid octet
      // skip the sweeps (valid octets only ever address valid tiles)
#ifndef NSB_NO_SKIP
      const bool warp_idle = (tid & ~31) >= (nvalid << (k - 3));
#else
      const bool warp_idle = false;
#endif
#pragma unroll 1
      for (int g = 0; g < ((p.debug & 1) ? 0 : n_groups); ++g) {
        const GroupDesc& d = s_groups[g];
        const bool cta_sync = d.sync();  // read before the sweep: no load latency after it
        double2* out = smem + spare * kTileAmpsMax;
        if (!warp_idle)
          apply_group<kOct>(tile, out, k, nvalid, d, s_ops + d.op_begin, s_mats, s_gm[g], s_ttab[g]);
        if (pending && g == 0 && !early) request_next();
        const int tmp = cur;
        cur = spare;
        spare = tmp;
        tile = out;
        if (cta_sync || (kHw && (p.debug & 8)))
          __syncthreads();
        else
          __syncwarp();  // the next sweep reads only this warp's amplitudes
      }
      if (ts) {
        if (pending && !early && (n_groups == 0 || (p.debug & 1))) request_next();
        // assertion epilogue partial sums from the final buffer, then ONE
        // thread stores the tile (TMA reads the swz_tma layout)
        const int mq = sp.measure_q;
        if (mq >= 0 && !(p.debug & 2)) {
          const uint64_t base = tbase[0] | lo;
#pragma unroll 2
          for (int j = 0; j < n_j; ++j) {
            const uint64_t g = base | s_hi[j];
            if (!((g >> mq) & 1)) {
              const double2 v = tile[eslot(0, j)];
              msum = fma(v.x, v.x, msum);
              msum = fma(v.y, v.y, msum);
            }
          }
        }
        fence_async_shared();  // this thread's sweep stores -> the TMA store's reads
        __syncthreads();
        if (tid == 0 && !(p.debug & 2)) tma_tile(true, tbase[0], cur);
      } else {
      // shared -> global (+ assertion epilogue partial sums)
      if (loader && !(p.debug & 2)) {
        const int mq = sp.measure_q;
        uint64_t bb = tbase[0];  // advanced in registers (no dynamic index into tbase)
#pragma unroll 1
        for (int b = 0; b < 4; ++b, bb = next_base(bb)) {
          if (b >= nvalid) break;
          const uint64_t base = bb | lo;
#pragma unroll 2
          for (int j = 0; j < n_j; ++j) {
            const uint64_t g = base | s_hi[j];
            const double2 v = tile[eslot(b, j)];
            p.amps[g] = v;
            if (mq >= 0 && !((g >> mq) & 1)) {
              msum = fma(v.x, v.x, msum);
              msum = fma(v.y, v.y, msum);
            }
          }
        }
      }
      __syncthreads();  // buffer `cur` is free for the batch issued next iteration
      }
      const int done = cur;  // next batch lives in `pre`; `done` takes the next prefetch
      cur = pre;
      pre = done;
    }
    if (ts) {
      if (tid == 0) {  // the pass's tile stores are complete before the grid barrier
        bulk_wait0();
        fence_async_global();
      }
    } else {
      cp_async_wait<0>();
    }
    const int mq = sp.measure_q;
    const int mslot = sp.measure_slot;
    if (mq >= 0) {
      const double bs = block_sum(msum, red);
      if (tid == 0) p.partials[(mslot & 1) * gridDim.x + blockIdx.x] = bs;
    }
    // split grid barrier: arrive, stage the next pass's descriptors while the
    // other CTAs finish, then wait (co-residency from the cooperative launch)
#ifdef NSB_FENCE_ALL
    __threadfence();
    __syncthreads();
    ++n_bar;
    if (tid == 0) atomicAdd(p.bar, 1u);
#else
    // the CTA barrier orders every thread's stores before thread 0's gpu-scope
    // fence, which is cumulative (the cooperative-groups grid barrier pattern)
    __syncthreads();
    ++n_bar;
    if (tid == 0 && gridDim.x > 1) {
      __threadfence();
      atomicAdd(p.bar, 1u);
    }
#endif
    if (pi + 1 < p.pass_end) stage(pi + 1);
    if (tid == 0 && gridDim.x > 1) {  // one CTA (n <= 11): the CTA barrier suffices
      const unsigned target = n_bar * gridDim.x;
      unsigned seen;
      // relaxed polling (no L1 invalidation per iteration), one acquire fence after
      do {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(p.bar) : "memory");
      } while (seen < target);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    if (kHw && tid == 0) fence_async_global();  // other CTAs' stores -> this CTA's TMA loads
    __syncthreads();
    if (mq >= 0) {
      if (tid < 32) {
        const double* part = p.partials + (mslot & 1) * gridDim.x;
        double s = 0.0;
        for (int i = tid; i < int(gridDim.x); i += 32) s += part[i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (tid == 0) s_p0 = s;
      }
      __syncthreads();
      carry_p0 = s_p0;
      if (blockIdx.x == 0 && tid == 0) {
        p.record[mslot] = carry_p0;
        if (carry_p0 < p.eps && !p.debug) {
          p.fail[0] = 1;
          p.fail[1] = mslot;
        }
      }
      if (carry_p0 < p.eps && !p.debug) return;  // every block saw the same p0
    }
  }
}

// ---------------------------------------------------------------------------
// sharded state: the half of the local shard that changes owner when a global
// qubit and local qubit L trade places (bit L == v), packed in index order.

__global__ void k_shard_pack(const double2* __restrict__ a, double2* __restrict__ out,
                             uint64_t off, uint64_t count, int L, int v) {
  const uint64_t vb = uint64_t(v) << L;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = a[insert_zero(off + i, L) | vb];
}

__global__ void k_shard_unpack(double2* __restrict__ a, const double2* __restrict__ in,
                               uint64_t off, uint64_t count, int L, int v) {
  const uint64_t vb = uint64_t(v) << L;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x)
    a[insert_zero(off + i, L) | vb] = in[i];
}

// Qubit swap through peer memory (NVLink): element k of this rank's outgoing
// half (bit L == v_mine) trades places with element k of the partner's
// (bit L == v_peer).  Chunks of 2^clog element pairs alternate between the
// two ranks (chunk parity), so every pair is read and written by exactly one
// GPU: one local and one remote load, one local and one remote store, four
// independent pairs in flight per thread.
__global__ void k_shard_swap_p2p(double2* __restrict__ mine, double2* __restrict__ peer,
                                 uint64_t half, int L, int v_mine, int v_peer, int parity,
                                 int clog) {
  const uint64_t clen = uint64_t(1) << clog;
  const uint64_t n_chunks = (half + clen - 1) >> clog;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  // owned elements, enumerated densely: e -> chunk 2 * (e >> clog) + parity
  const uint64_t owned_chunks = (n_chunks + 1 - parity) >> 1;
  const uint64_t n_owned = owned_chunks << clog;
  for (uint64_t e0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e0 < n_owned;
       e0 += 4 * stride) {
    uint64_t km[4], kp[4];
    double2 x[4], y[4];
    bool ok[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t e = e0 + u * stride;
      const uint64_t k = ((2 * (e >> clog) + parity) << clog) | (e & (clen - 1));
      ok[u] = e < n_owned && k < half;
      km[u] = insert_zero(k, L) | (uint64_t(v_mine) << L);
      kp[u] = insert_zero(k, L) | (uint64_t(v_peer) << L);
      if (ok[u]) {
        x[u] = mine[km[u]];
        y[u] = peer[kp[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (ok[u]) {
        mine[km[u]] = y[u];
        peer[kp[u]] = x[u];
      }
  }
  __threadfence_system();
}

// One chunk of an overlapped qubit swap (nsb_shard_swap_overlap): the
// element pairs of k_shard_swap_p2p whose bits at the chunk qubits equal the
// chunk's value.  Pair index k (the bits other than L and the chunk qubits)
// is spread by inserting zeros at pos[0..npos) (ascending: the chunk qubits
// and L), then the fixed bits are set.  Sub-chunks of 2^clog pairs alternate
// between the two partners as in k_shard_swap_p2p.
struct SwapChunk {
  int npos;
  int pos[8];
  uint64_t fixed_mine, fixed_peer;  // chunk value | (v << L) on each side
  uint64_t n_pairs;
};
constexpr int kSwapThreads = 256;
__global__ void __launch_bounds__(kSwapThreads, 2)
    k_shard_swap_chunk(double2* __restrict__ mine, double2* __restrict__ peer, SwapChunk sc,
                       int parity, int clog) {
  const uint64_t clen = uint64_t(1) << clog;
  const uint64_t n_sub = (sc.n_pairs + clen - 1) >> clog;
  const uint64_t n_owned = ((n_sub + 1 - parity) >> 1) << clog;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  constexpr int U = 4;
  for (uint64_t e0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e0 < n_owned;
       e0 += U * stride) {
    uint64_t km[U], kp[U];
    double2 x[U], y[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t e = e0 + u * stride;
      uint64_t k = ((2 * (e >> clog) + parity) << clog) | (e & (clen - 1));
      ok[u] = e < n_owned && k < sc.n_pairs;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < sc.npos) k = insert_zero(k, sc.pos[i]);
      km[u] = k | sc.fixed_mine;
      kp[u] = k | sc.fixed_peer;
      if (ok[u]) {
        x[u] = mine[km[u]];
        y[u] = peer[kp[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok[u]) {
        mine[km[u]] = y[u];
        peer[kp[u]] = x[u];
      }
  }
}

// Chunk-landed flags of overlapped swaps, in each shard allocation behind its
// amplitudes (kShardFlagWords words; slot 2 c + side).  The signal runs on
// the swap stream after the chunk's kernel (whose stores, local and remote,
// are complete at its end) and writes both partners' copies; the wait holds
// the gate stream until both sides' kernels for the chunk are done.
constexpr int kShardFlagWords = 256;
__global__ void k_flag_signal(unsigned* mine, unsigned* peer, int slot, unsigned epoch) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(mine + slot), "r"(epoch) : "memory");
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peer + slot), "r"(epoch) : "memory");
}
__global__ void k_flag_wait(const unsigned* f, int s0, int s1, unsigned epoch) {
  if (threadIdx.x == 0) {
    unsigned v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f + s0) : "memory");
    } while (v < epoch);
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f + s1) : "memory");
    } while (v < epoch);
    __threadfence_system();
  }
}

}  // namespace dev
}  // namespace nsb

// ===========================================================================
// host side

using namespace nsb;

namespace {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define NSB_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));              \
  } while (0)

template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t count = 0;
  // non-null: stream-ordered allocation from the context's private plan pool
  // (cudaMallocFromPoolAsync / cudaFreeAsync on `stream`), so releasing a
  // plan's buffers does not synchronise the device
  cudaStream_t stream = nullptr;
  void alloc(size_t n, cudaStream_t s = nullptr, cudaMemPool_t pool = nullptr) {
    release();
    if (n == 0) n = 1;
    cudaError_t e = s ? cudaMallocFromPoolAsync(reinterpret_cast<void**>(&ptr), n * sizeof(T),
                                                pool, s)
                      : cudaMalloc(&ptr, n * sizeof(T));
    if (e != cudaSuccess) {
      ptr = nullptr;
      throw std::bad_alloc();
    }
    stream = s;
    count = n;
  }
  void upload(const T* src, size_t n, cudaStream_t s, cudaMemPool_t pool) {
    alloc(n, s, pool);
    if (n) NSB_CUDA(cudaMemcpyAsync(ptr, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void release() {
    if (ptr) {
      if (stream)
        cudaFreeAsync(ptr, stream);
      else
        cudaFree(ptr);
    }
    ptr = nullptr;
    stream = nullptr;
    count = 0;
  }
  ~DevBuf() { release(); }
};

}  // namespace

struct nsb_ctx {
  // one reference held by the owner (nsb_ctx_destroy drops it) and one by
  // every live plan, so a plan never outlives the context it runs on
  std::atomic<int> refs{1};
  int device = 0;
  cudaMemPool_t plan_pool = nullptr;  // private stream-ordered pool for plan buffers
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t tev0 = nullptr, tev1 = nullptr;  // nsb_timer_start / stop
  int sm_count = 0;
  int blocked_grid = 0;  // co-resident CTAs of k_blocked
  bool tma_ok = false;   // the TMA instantiation is co-resident on the same grid
  bool o1_ok = false;    // ... and the one-octet layout
  int n = 0;
  uint64_t n_amps = 0;
  DevBuf<double2> amps;
  DevBuf<double> scratch;  // reductions
  DevBuf<double> probs;    // nsb_probabilities (kept between calls)
  double* pinned = nullptr;
  size_t pinned_bytes = 0;
  // sharded state (nsb_comm_init): this process holds rank `rank` of `nranks`
  void* comm = nullptr;  // ncclComm_t
  double2* peers[64] = {};  // IPC-mapped shards of the other ranks (nsb_shard_open_peers)
  int rank = 0, nranks = 1;
  // qubit swaps: pack / unpack on `stream`, NCCL on `xfer`, double-buffered
  cudaStream_t xfer = nullptr;
  cudaEvent_t ev_packed[2] = {}, ev_moved[2] = {}, ev_unpacked[2] = {};
  DevBuf<double2> stage_send[2], stage_recv[2];
  // overlapped swaps (nsb_shard_swap_overlap): epoch of the chunk flags
  unsigned swap_epoch = 0;
  cudaEvent_t ev_ov0 = nullptr, ev_ov1 = nullptr;
  // copy-engine swaps (nsb_shard_swap_overlap_ce): two staging slots, one
  // event per chunk
  DevBuf<double2> ce_stage;
  cudaEvent_t ev_chunk[16] = {};
  cudaStream_t xfer2 = nullptr;  // local copies (pulls on xfer)
  cudaEvent_t ev_pulled[2] = {}, ev_local[2] = {};  // per staging slot
};

struct nsb_plan {
  nsb_ctx* ctx = nullptr;  // holds a reference (ctx->refs)
  int n = 0;               // qubit count the plan was built for
  // persistent CTAs of this plan's k_blocked launches: the co-resident grid,
  // but no more than the tiles of a pass -- a state of one tile (n <= 11) runs
  // on ONE CTA with no grid barrier at all, a 16-qubit state on 32
  int grid = 0;
  HostPlan host;
  DevBuf<PassDesc> passes, mma_passes;
  DevBuf<GroupDesc> groups;
  DevBuf<GateOp> ops;
  DevBuf<double2> mats, dense;
  DevBuf<double> record, partials;
  DevBuf<int> fail;
  DevBuf<unsigned> bar;
  // TMA plans: tensor maps per pass of `passes` [0] and `mma_passes` [1],
  // encoded for the state buffer tm_amps (re-encoded if the state moves)
  std::vector<dev::TmaPass> tm_host[2];
  DevBuf<dev::TmaPass> tm_dev[2];
  const double2* tm_amps[2] = {nullptr, nullptr};
  double last_ms = 0.0;
  int64_t last_launches = 0;
  // the plan's own stream for releasing its buffers: stream-ordered frees
  // (no device-wide synchronise) that do not depend on the context outliving
  // the plan; every run synchronises the context stream before returning
  int device = 0;
  cudaStream_t rel = nullptr;
  ~nsb_plan() {
    if (rel) cudaSetDevice(device);
    passes.release(); mma_passes.release(); groups.release(); ops.release();
    mats.release(); dense.release(); record.release(); partials.release();
    fail.release(); bar.release();
    tm_dev[0].release(); tm_dev[1].release();
    if (rel) cudaStreamDestroy(rel);
  }
};

namespace {

// NCCL is resolved at run time from the process's libnccl.so.2 (torch's copy
// when torch is loaded, else the system library), so the library keeps
// loading on machines without NCCL and never carries a second NCCL instance.
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string error;
};

const NcclApi& shard_nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
#define NSB_NCCL_SYM(field, name)                                     \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, #name));     \
  if (!a.field) a.error = "libnccl lacks " #name;
    NSB_NCCL_SYM(get_unique_id, ncclGetUniqueId)
    NSB_NCCL_SYM(comm_init_rank, ncclCommInitRank)
    NSB_NCCL_SYM(comm_destroy, ncclCommDestroy)
    NSB_NCCL_SYM(send, ncclSend)
    NSB_NCCL_SYM(recv, ncclRecv)
    NSB_NCCL_SYM(all_gather, ncclAllGather)
    NSB_NCCL_SYM(group_start, ncclGroupStart)
    NSB_NCCL_SYM(group_end, ncclGroupEnd)
    NSB_NCCL_SYM(error_string, ncclGetErrorString)
#undef NSB_NCCL_SYM
    return a;
  }();
  if (!api.error.empty()) throw CudaError(api.error);
  return api;
}

#define NSB_NCCL(call)                                                                 \
  do {                                                                                 \
    const ncclResult_t r_ = (call);                                                    \
    if (r_ != ncclSuccess)                                                             \
      throw CudaError(std::string(#call) + ": " + shard_nccl().error_string(r_));      \
  } while (0)

void shard_comm_destroy(nsb_ctx* c) {
  for (double2*& p : c->peers)
    if (p) {
      cudaIpcCloseMemHandle(p);
      p = nullptr;
    }
  if (c->comm) shard_nccl().comm_destroy(static_cast<ncclComm_t>(c->comm));
  c->comm = nullptr;
  c->rank = 0;
  c->nranks = 1;
}

int fail_status(nsb_status* st, int code, const std::string& msg) {
  set_status(st, code, msg);
  return code;
}

// A failed MMA assertion inside a guarded call (-> NSB_EASSERT with step, p0).
struct AssertFailure {
  int step;
  double prob;
  std::string msg;
};

// Runs f, mapping exceptions to status codes.  The return value is the
// status code whether or not the caller passed a status struct (a NULL st
// is replaced by a local one, so a failure set inside f is still returned).
template <class F>
int guarded(nsb_status* st, F&& f) {
  nsb_status local;
  if (!st) st = &local;
  set_status(st, NSB_OK, "");
  try {
    f();
  } catch (const AssertFailure& a) {
    set_status(st, NSB_EASSERT, a.msg, a.step, a.prob);
    return NSB_EASSERT;
  } catch (const CudaError& e) {
    return fail_status(st, NSB_EDEVICE, e.what());
  } catch (const std::bad_alloc&) {
    return fail_status(st, NSB_ERESOURCE, "out of device or host memory");
  } catch (const std::invalid_argument& e) {
    return fail_status(st, NSB_EINVAL, e.what());
  } catch (const std::exception& e) {
    return fail_status(st, NSB_EDEVICE, e.what());
  }
  return st->code;
}

void ctx_free(nsb_ctx* ctx);
void ctx_release(nsb_ctx* ctx) {
  if (ctx && ctx->refs.fetch_sub(1) == 1) ctx_free(ctx);
}

// Host programs of destroyed plans (hundreds of MB for long circuits) are
// released by ONE long-lived worker thread, off the caller's path; small
// ones inline.  The singleton is never destroyed (no exit-order hazard).
struct Reclaimer {
  std::mutex mu;
  std::condition_variable cv;
  std::deque<HostPlan*> queue;
  Reclaimer() {
    std::thread([this] {
      for (;;) {
        HostPlan* h;
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [this] { return !queue.empty(); });
          h = queue.front();
          queue.pop_front();
        }
        delete h;
      }
    }).detach();
  }
  static Reclaimer& get() {
    static Reclaimer* r = new Reclaimer();
    return *r;
  }
  void push(HostPlan* h) {
    {
      std::lock_guard<std::mutex> lk(mu);
      queue.push_back(h);
    }
    cv.notify_one();
  }
};

size_t host_plan_bytes(const HostPlan& H) {
  return H.groups.size() * sizeof(GroupDesc) + H.gate_ops.size() * sizeof(GateOp) +
         (H.matrices.size() + H.packed_all.size() + H.dense_mats.size()) * sizeof(double) +
         (H.passes.size() + H.mma_passes.size()) * sizeof(PassDesc);
}

// state vector allocation; on out-of-memory the plan pool's cached blocks
// are returned to the device and the allocation retried once
// (plus the zeroed chunk-flag words of overlapped swaps behind the amplitudes)
constexpr uint64_t kFlagAmps = dev::kShardFlagWords * sizeof(unsigned) / sizeof(double2);
void alloc_state(nsb_ctx* c, uint64_t n_amps) {
  try {
    c->amps.alloc(n_amps + kFlagAmps);
  } catch (const std::bad_alloc&) {
    cudaGetLastError();
    NSB_CUDA(cudaDeviceSynchronize());
    if (c->plan_pool) NSB_CUDA(cudaMemPoolTrimTo(c->plan_pool, 0));
    c->amps.alloc(n_amps + kFlagAmps);
  }
  NSB_CUDA(cudaMemsetAsync(c->amps.ptr + n_amps, 0, kFlagAmps * sizeof(double2), c->stream));
}

unsigned* shard_flags(double2* amps, uint64_t n_amps) {
  return reinterpret_cast<unsigned*>(amps + n_amps);
}

unsigned grid_for(uint64_t work, int threads, const nsb_ctx* c) {
  const uint64_t want = (work + threads - 1) / threads;
  const uint64_t cap = uint64_t(c->sm_count) * 8;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min(want, cap)));
}

void require_state(const nsb_ctx* c) {
  if (!c || !c->amps.ptr) throw std::invalid_argument("state not initialised");
}

void ensure_pinned(nsb_ctx* c, size_t bytes) {
  if (c->pinned_bytes >= bytes) return;
  if (c->pinned) cudaFreeHost(c->pinned);
  c->pinned = nullptr;
  c->pinned_bytes = 0;
  NSB_CUDA(cudaMallocHost(&c->pinned, bytes));
  c->pinned_bytes = bytes;
}

// Host <-> device through the context's pinned staging buffer (16 MiB chunks):
// pageable copies make the driver stage and pin on every call, with erratic
// latency (observed 5 ms .. 0.9 s for 16 MiB on the same box).
void copy_d2h(nsb_ctx* c, void* dst, const void* src, size_t bytes) {
  const size_t chunk = size_t(16) << 20;
  ensure_pinned(c, std::min(bytes, chunk));
  for (size_t off = 0; off < bytes; off += chunk) {
    const size_t nb = std::min(chunk, bytes - off);
    NSB_CUDA(cudaMemcpyAsync(c->pinned, static_cast<const char*>(src) + off, nb,
                             cudaMemcpyDeviceToHost, c->stream));
    NSB_CUDA(cudaStreamSynchronize(c->stream));
    std::memcpy(static_cast<char*>(dst) + off, c->pinned, nb);
  }
}

void copy_h2d(nsb_ctx* c, void* dst, const void* src, size_t bytes) {
  const size_t chunk = size_t(16) << 20;
  ensure_pinned(c, std::min(bytes, chunk));
  for (size_t off = 0; off < bytes; off += chunk) {
    const size_t nb = std::min(chunk, bytes - off);
    NSB_CUDA(cudaStreamSynchronize(c->stream));  // staging free again
    std::memcpy(c->pinned, static_cast<const char*>(src) + off, nb);
    NSB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, c->pinned, nb,
                             cudaMemcpyHostToDevice, c->stream));
  }
  NSB_CUDA(cudaStreamSynchronize(c->stream));
}

// deterministic half-norm: fixed grid, then fixed-order sum
double half_norm(nsb_ctx* c, int q, int outcome) {
  const uint64_t n_half = c->n_amps >> 1;
  dev::k_half_norm<<<dev::kReduceBlocks, dev::kReduceThreads, 0, c->stream>>>(
      c->amps.ptr, n_half, q, outcome, c->scratch.ptr);
  dev::k_sum_fixed<<<1, 32, 0, c->stream>>>(c->scratch.ptr, dev::kReduceBlocks, 0,
                                             c->scratch.ptr + 2 * dev::kReduceBlocks);
  double out = 0.0;
  NSB_CUDA(cudaMemcpyAsync(&out, c->scratch.ptr + 2 * dev::kReduceBlocks, sizeof(double),
                           cudaMemcpyDeviceToHost, c->stream));
  NSB_CUDA(cudaStreamSynchronize(c->stream));
  return out;
}

void project(nsb_ctx* c, int q, int outcome, double prob) {
  const double scale = 1.0 / std::sqrt(prob);
  dev::k_project<<<grid_for(c->n_amps, 256, c), 256, 0, c->stream>>>(c->amps.ptr, c->n_amps, q,
                                                                      outcome, scale);
  NSB_CUDA(cudaGetLastError());
}

void apply_matrix(nsb_ctx* c, const double* u, const int32_t* qubits, int k,
                  const double2* dev_mat /* optional, for k >= 3 */) {
  for (int j = 0; j < k; ++j) {
    if (qubits[j] < 0 || qubits[j] >= c->n) throw std::invalid_argument("qubit out of range");
    for (int i = 0; i < j; ++i)
      if (qubits[i] == qubits[j]) throw std::invalid_argument("duplicate qubit");
  }
  if (k == 1) {
    dev::M2 m;
    std::memcpy(m.m, u, sizeof(m.m));
    dev::k_apply1<<<grid_for(c->n_amps >> 1, 256, c), 256, 0, c->stream>>>(
        c->amps.ptr, c->n_amps >> 1, qubits[0], m);
  } else if (k == 2) {
    dev::M4 m;
    int p = qubits[0], q = qubits[1];
    if (p < q) {
      std::memcpy(m.m, u, sizeof(m.m));
    } else {  // swap_conjugate (engine.py:124-127)
      static const int perm[4] = {0, 2, 1, 3};
      for (int r = 0; r < 4; ++r)
        for (int col = 0; col < 4; ++col) {
          m.m[4 * r + col].x = u[2 * (perm[r] * 4 + perm[col])];
          m.m[4 * r + col].y = u[2 * (perm[r] * 4 + perm[col]) + 1];
        }
      std::swap(p, q);
    }
    dev::k_apply2<<<grid_for(c->n_amps >> 2, 256, c), 256, 0, c->stream>>>(
        c->amps.ptr, c->n_amps >> 2, p, q, m);
  } else {
    if (k > 5 || k > c->n) throw std::invalid_argument("at most 5 qubits per dense gate");
    dev::KQ g;
    g.k = k;
    for (int j = 0; j < k; ++j) g.slot_q[j] = g.sorted_q[j] = qubits[j];
    std::sort(g.sorted_q, g.sorted_q + k);
    const double2* m = dev_mat;
    DevBuf<double2> tmp;
    if (!m) {
      tmp.upload(reinterpret_cast<const double2*>(u), size_t(1) << (2 * k), c->stream, c->plan_pool);
      m = tmp.ptr;
    }
    dev::k_applyk<<<grid_for(c->n_amps >> k, 128, c), 128, 0, c->stream>>>(
        c->amps.ptr, c->n_amps >> k, g, m);
    NSB_CUDA(cudaGetLastError());
    if (!dev_mat) NSB_CUDA(cudaStreamSynchronize(c->stream));  // tmp lifetime
  }
  NSB_CUDA(cudaGetLastError());
}

// ---- stream memory operations (copy-engine swaps) --------------------------
// cuStreamWriteValue32 / cuStreamWaitValue32 from the driver: flag words
// written and awaited by the stream front end, no kernel (no SM) involved
struct StreamMem {
  using Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  Fn write_fn = nullptr, wait_fn = nullptr;
  void write(cudaStream_t s, unsigned* addr, unsigned v) const {
    const CUresult r = write_fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v,
                                0 /* CU_STREAM_WRITE_VALUE_DEFAULT: after a memory barrier */);
    if (r != CUDA_SUCCESS) throw CudaError("cuStreamWriteValue32 failed (" + std::to_string(int(r)) + ")");
  }
  void wait(cudaStream_t s, unsigned* addr, unsigned v) const {
    const CUresult r = wait_fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v,
                               CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) throw CudaError("cuStreamWaitValue32 failed (" + std::to_string(int(r)) + ")");
  }
};
const StreamMem& stream_mem() {
  static const StreamMem sm = [] {
    StreamMem m;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    NSB_CUDA(cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q));
    m.write_fn = reinterpret_cast<StreamMem::Fn>(f);
    NSB_CUDA(cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q));
    m.wait_fn = reinterpret_cast<StreamMem::Fn>(f);
    if (!m.write_fn || !m.wait_fn) throw std::runtime_error("stream memory operations unavailable");
    return m;
  }();
  return sm;
}

// ---- TMA tensor maps (planner.h "TMA tiles", dev::TmaPass) -----------------
using TensorMapEncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                          const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                          const cuuint32_t*, CUtensorMapInterleave,
                                          CUtensorMapSwizzle, CUtensorMapL2promotion,
                                          CUtensorMapFloatOOBfill);
TensorMapEncodeTiled tensor_map_encoder() {
  static TensorMapEncodeTiled fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    NSB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess)
      throw std::runtime_error("cuTensorMapEncodeTiled is not available");
    return reinterpret_cast<TensorMapEncodeTiled>(f);
  }();
  return fn;
}

// L2 sector promotion of the tile copies: the 128-byte rows are whole lines
// already (NSB_TMA_PROMO = 0 none, 1 64B, 2 128B, 3 256B)
CUtensorMapL2promotion tma_l2_promotion() {
  static const int v = [] {
    const char* e = std::getenv("NSB_TMA_PROMO");
    return e ? std::atoi(e) : 2;
  }();
  return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
       : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
       : v == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
}

// TMA passes store their tiles by TMA (1, NSB_TMA_STORE) or by the threads (0)
int tma_store_mode() {
  static const int v = [] {
    const char* e = std::getenv("NSB_TMA_STORE");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

// the tensor map of pass P over an n-qubit state at `amps` (rank 0: the
// planner left the pass on cp.async, PassDesc::tma = 0)
void encode_tma_pass(const PassDesc& P, int n, const double2* amps, dev::TmaPass& T) {
  std::memset(&T, 0, sizeof T);
  if (!P.tma) return;
  TmaLayout L;  // the planner's choice: the dim order whose layout is P.tperm
  if (!tma_layout(P, n, 0, L)) throw std::logic_error("TMA pass tile is not TMA-shaped");
  const int n_orders = L.n_orders;
  int o = 0;
  while (std::memcmp(L.perm, P.tperm, sizeof L.perm) != 0) {
    if (++o >= n_orders) throw std::logic_error("TMA pass copy layout not found");
    tma_layout(P, n, o, L);
  }
  T.left = L.left;
  cuuint64_t dim[5], stride[4];
  cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
  dim[0] = 16;  // qubits 0..2 as re/im doubles: 128 bytes
  box[0] = 16;
  int box_bits = 3;
  for (int i = 1; i < L.rank; ++i) {
    T.start[i] = static_cast<int8_t>(L.start[i]);
    T.ebits[i] = static_cast<int8_t>(L.ebits[i]);
    dim[i] = cuuint64_t(1) << L.ebits[i];
    stride[i - 1] = cuuint64_t(sizeof(double2)) << L.start[i];
    box[i] = 1u << (L.len[i] + L.gap[i]);
    estr[i] = 1u << L.gap[i];
    box_bits += L.len[i];
  }
  T.rank = static_cast<int8_t>(L.rank);
  T.box_bits = static_cast<int8_t>(box_bits);
  const CUresult r = tensor_map_encoder()(
      &T.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, static_cast<cuuint32_t>(L.rank),
      const_cast<double2*>(amps), dim, stride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, tma_l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

// device tensor maps of `passes` for the current state (plans: cached per array)
void encode_tma_passes(const std::vector<PassDesc>& passes, int n, const double2* amps,
                       std::vector<dev::TmaPass>& out) {
  out.resize(passes.size());
  for (size_t i = 0; i < passes.size(); ++i) encode_tma_pass(passes[i], n, amps, out[i]);
}

const dev::TmaPass* plan_tma(nsb_ctx* c, nsb_plan* P, const PassDesc* passes) {
  if (!P->host.tma) return nullptr;
  const int w = passes == P->mma_passes.ptr ? 1 : 0;
  if (P->tm_amps[w] != c->amps.ptr || !P->tm_dev[w].ptr) {
    encode_tma_passes(w ? P->host.mma_passes : P->host.passes, c->n, c->amps.ptr, P->tm_host[w]);
    P->tm_dev[w].upload(P->tm_host[w].data(), P->tm_host[w].size(), c->stream, c->plan_pool);
    P->tm_dev[w].stream = P->rel;  // released with the plan's other buffers
    P->tm_amps[w] = c->amps.ptr;
  }
  return P->tm_dev[w].ptr;
}

template <int O>
void* blocked_kernel_o(bool chunk, bool tma) {
  return chunk ? (tma ? reinterpret_cast<void*>(dev::k_blocked<true, true, O>)
                      : reinterpret_cast<void*>(dev::k_blocked<true, false, O>))
               : (tma ? reinterpret_cast<void*>(dev::k_blocked<false, true, O>)
                      : reinterpret_cast<void*>(dev::k_blocked<false, false, O>));
}
void* blocked_kernel(bool chunk, bool tma, int octets = 2) {
  return octets == 1 ? blocked_kernel_o<1>(chunk, tma) : blocked_kernel_o<2>(chunk, tma);
}
// threads per CTA of a plan's kernel layout
unsigned blocked_threads(int octets) { return octets == 1 ? 256u : unsigned(kPassThreads); }

// launch k_blocked over [pb, pe) of `passes` cooperatively
void launch_blocked(nsb_ctx* c, nsb_plan* P, const PassDesc* passes, int pb, int pe, double eps,
                    int grid = 0, uint64_t cmask = 0, uint64_t cval = 0) {
  dev::BlockedParams bp;
  bp.amps = c->amps.ptr;
  bp.n = c->n;
  bp.passes = passes;
  bp.pass_begin = pb;
  bp.pass_end = pe;
  bp.groups = P->groups.ptr;
  bp.ops = P->ops.ptr;
  bp.mats = P->mats.ptr;
  bp.partials = P->partials.ptr;
  bp.record = P->record.ptr;
  bp.fail = P->fail.ptr;
  bp.bar = P->bar.ptr;
  NSB_CUDA(cudaMemsetAsync(P->bar.ptr, 0, sizeof(unsigned), c->stream));
  bp.eps = eps;
  static const int debug = [] {
    const char* e = std::getenv("NSB_DEBUG_BLOCKED");
    return e ? std::atoi(e) : 0;
  }();
  bp.debug = debug;
  bp.cmask = cmask;
  bp.cval = cval;
  bp.cbits = __builtin_popcountll(cmask);
  const bool tma = P->host.tma;
  bp.tmaps = tma && !cmask ? plan_tma(c, P, passes) : nullptr;
  bp.tma_store = tma_store_mode();
  void* args[] = {&bp};
  const int oct = P->host.octets;
  NSB_CUDA(cudaLaunchCooperativeKernel(
      blocked_kernel(cmask != 0, tma, oct), dim3(grid > 0 ? grid : P->grid),
      dim3(blocked_threads(oct)), args, tma ? dev::kBlockedSmemBytesTma : dev::kBlockedSmemBytes,
      c->stream));
  P->last_launches += 1;
}

// bits of v spread over the set bits of mask (ascending)
uint64_t deposit_bits(uint64_t v, uint64_t mask) {
  uint64_t out = 0;
  for (int j = 0; mask; mask &= mask - 1, ++j)
    if (v >> j & 1) out |= mask & (0 - mask);
  return out;
}

double p0_scale(const HostPlan& H, int step) {
  return step >= 0 && step < static_cast<int>(H.p0_scale.size()) ? H.p0_scale[step] : 1.0;
}

void run_item(nsb_ctx* c, nsb_plan* P, const Item& it) {
  if (it.kind == Item::kGates) {
    launch_blocked(c, P, P->passes.ptr, it.pass_begin, it.pass_end, -1.0);
  } else if (it.kind == Item::kDense) {
    const double* u = P->host.dense_mats.data() + 2 * it.mat_off;
    apply_matrix(c, u, it.qs, it.k, it.k >= 3 ? P->dense.ptr + it.mat_off : nullptr);
    P->last_launches += 1;
  }
}

}  // namespace

extern "C" {

int nsb_device_count(int32_t* n) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
  if (n) *n = c;
  return NSB_OK;
}

int nsb_ctx_create(int32_t device, nsb_ctx** out, nsb_status* st) {
  if (!out) return fail_status(st, NSB_EINVAL, "null out pointer");
  *out = nullptr;
  auto ctx = std::make_unique<nsb_ctx>();
  const int rc = guarded(st, [&] {
    int count = 0;
    NSB_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw std::invalid_argument("no such CUDA device");
    ctx->device = device;
    NSB_CUDA(cudaSetDevice(device));
    NSB_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    {  // plan buffers come from a private stream-ordered pool that keeps up to
       // 8 GiB cached across plans (the device's default pool is left alone);
       // state allocations trim it on out-of-memory (alloc_state)
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      NSB_CUDA(cudaMemPoolCreate(&ctx->plan_pool, &props));
      uint64_t keep = uint64_t(8) << 30;
      NSB_CUDA(cudaMemPoolSetAttribute(ctx->plan_pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    NSB_CUDA(cudaEventCreate(&ctx->ev0));
    NSB_CUDA(cudaEventCreate(&ctx->ev1));
    NSB_CUDA(cudaEventCreate(&ctx->tev0));
    NSB_CUDA(cudaEventCreate(&ctx->tev1));
    NSB_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
    const int smem = static_cast<int>(dev::kBlockedSmemBytes);
    const int smem_tma = static_cast<int>(dev::kBlockedSmemBytesTma);
    for (int oct : {1, 2})
      for (bool chunk : {false, true})
        for (bool tma : {false, true})
          NSB_CUDA(cudaFuncSetAttribute(blocked_kernel(chunk, tma, oct),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        tma ? smem_tma : smem));
    int per_sm = 0, per_sm_tma = 0;
    NSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::k_blocked<false, false>,
                                                           kPassThreads, smem));
    NSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm_tma, dev::k_blocked<false, true>, kPassThreads, smem_tma));
    if (per_sm < 1) throw std::runtime_error("k_blocked cannot be resident");
    ctx->blocked_grid = per_sm * ctx->sm_count;
    // TMA plans run on the same persistent grid (NSB_TMA=0 or a smaller
    // residency: per-thread cp.async under the usual layout)
    ctx->tma_ok = per_sm_tma == per_sm;
    int per_sm_o1 = 0;  // the one-octet layout (256 threads) on the same grid
    NSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm_o1, dev::k_blocked<false, false, 1>, 256, smem));
    ctx->o1_ok = per_sm_o1 == per_sm;
    ctx->scratch.alloc(4 * dev::kReduceBlocks + 64);
  });
  if (rc == NSB_OK) *out = ctx.release();
  return rc;
}

void nsb_ctx_destroy(nsb_ctx* ctx) { ctx_release(ctx); }

}  // extern "C"

namespace {
void ctx_free(nsb_ctx* ctx) {
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->comm) shard_comm_destroy(ctx);
  ctx->amps.release();
  ctx->scratch.release();
  ctx->probs.release();
  for (int b = 0; b < 2; ++b) {
    ctx->stage_send[b].release();
    ctx->stage_recv[b].release();
    if (ctx->ev_packed[b]) cudaEventDestroy(ctx->ev_packed[b]);
    if (ctx->ev_moved[b]) cudaEventDestroy(ctx->ev_moved[b]);
    if (ctx->ev_unpacked[b]) cudaEventDestroy(ctx->ev_unpacked[b]);
  }
  if (ctx->xfer) cudaStreamDestroy(ctx->xfer);
  if (ctx->ev_ov0) cudaEventDestroy(ctx->ev_ov0);
  if (ctx->ev_ov1) cudaEventDestroy(ctx->ev_ov1);
  for (cudaEvent_t& e : ctx->ev_chunk)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (ctx->ev_pulled[i]) cudaEventDestroy(ctx->ev_pulled[i]);
    if (ctx->ev_local[i]) cudaEventDestroy(ctx->ev_local[i]);
  }
  if (ctx->xfer2) cudaStreamDestroy(ctx->xfer2);
  ctx->ce_stage.release();
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->tev0) cudaEventDestroy(ctx->tev0);
  if (ctx->tev1) cudaEventDestroy(ctx->tev1);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->plan_pool) cudaMemPoolDestroy(ctx->plan_pool);  // deferred by CUDA until freed
  delete ctx;
}
}  // namespace

extern "C" {

int nsb_state_init(nsb_ctx* c, int32_t n_qubits, nsb_status* st) {
  if (!c) return fail_status(st, NSB_EINVAL, "null context");
  if (n_qubits < 1 || n_qubits > kMaxQubits)
    return fail_status(st, NSB_EINVAL, "qubit count out of range");
  return guarded(st, [&] {
    NSB_CUDA(cudaSetDevice(c->device));
    const uint64_t n_amps = uint64_t(1) << n_qubits;
    if (c->n != n_qubits || !c->amps.ptr) {
      for (int r = 0; r < 64; ++r)
        if (c->peers[r])
          throw std::invalid_argument(
              "state size change while peer shards are mapped (re-open peers after init)");
      c->amps.release();
      c->n = 0;
      alloc_state(c, n_amps);
      c->n = n_qubits;
      c->n_amps = n_amps;
    }
    dev::k_vacuum<<<grid_for(n_amps, 256, c), 256, 0, c->stream>>>(c->amps.ptr, n_amps);
    NSB_CUDA(cudaGetLastError());
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int nsb_state_reset(nsb_ctx* c, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    NSB_CUDA(cudaSetDevice(c->device));
    dev::k_vacuum<<<grid_for(c->n_amps, 256, c), 256, 0, c->stream>>>(c->amps.ptr, c->n_amps);
    NSB_CUDA(cudaGetLastError());
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int nsb_state_upload(nsb_ctx* c, const double* amps, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!amps) throw std::invalid_argument("null host buffer");
    NSB_CUDA(cudaSetDevice(c->device));
    copy_h2d(c, c->amps.ptr, amps, c->n_amps * sizeof(double2));
  });
}

int nsb_state_download(nsb_ctx* c, double* amps, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!amps) throw std::invalid_argument("null host buffer");
    NSB_CUDA(cudaSetDevice(c->device));
    copy_d2h(c, amps, c->amps.ptr, c->n_amps * sizeof(double2));
  });
}

int nsb_state_norm2(nsb_ctx* c, double* out, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    NSB_CUDA(cudaSetDevice(c->device));
    dev::k_norm2<<<dev::kReduceBlocks, dev::kReduceThreads, 0, c->stream>>>(
        c->amps.ptr, c->n_amps, c->scratch.ptr);
    dev::k_sum_fixed<<<1, 32, 0, c->stream>>>(c->scratch.ptr, dev::kReduceBlocks, 0,
                                               c->scratch.ptr + 2 * dev::kReduceBlocks);
    NSB_CUDA(cudaMemcpyAsync(out, c->scratch.ptr + 2 * dev::kReduceBlocks, sizeof(double),
                             cudaMemcpyDeviceToHost, c->stream));
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int nsb_apply_matrix(nsb_ctx* c, const double* u, const int32_t* qubits, int32_t k,
                     nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!u || !qubits || k < 1) throw std::invalid_argument("bad matrix arguments");
    NSB_CUDA(cudaSetDevice(c->device));
    apply_matrix(c, u, qubits, k, nullptr);
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int nsb_branch_probability(nsb_ctx* c, int32_t q, int32_t outcome, double* p, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (q < 0 || q >= c->n || (outcome != 0 && outcome != 1) || !p)
      throw std::invalid_argument("bad measurement arguments");
    NSB_CUDA(cudaSetDevice(c->device));
    *p = half_norm(c, q, outcome);
  });
}

int nsb_project(nsb_ctx* c, int32_t q, int32_t outcome, double prob, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (q < 0 || q >= c->n || (outcome != 0 && outcome != 1))
      throw std::invalid_argument("bad projection arguments");
    NSB_CUDA(cudaSetDevice(c->device));
    project(c, q, outcome, prob);
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int nsb_probabilities(nsb_ctx* c, double* out, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!out) throw std::invalid_argument("null output");
    NSB_CUDA(cudaSetDevice(c->device));
    if (c->probs.count < c->n_amps) c->probs.alloc(c->n_amps);
    dev::k_probabilities<<<grid_for(c->n_amps, 256, c), 256, 0, c->stream>>>(
        c->amps.ptr, c->n_amps, c->probs.ptr);
    NSB_CUDA(cudaGetLastError());
    copy_d2h(c, out, c->probs.ptr, c->n_amps * sizeof(double));
  });
}

int nsb_prob_chunk_sums(nsb_ctx* c, int32_t chunk_log2, double* out, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!out) throw std::invalid_argument("null output");
    if (chunk_log2 < 0 || chunk_log2 > c->n) throw std::invalid_argument("bad chunk size");
    NSB_CUDA(cudaSetDevice(c->device));
    const uint64_t n_chunks = c->n_amps >> chunk_log2;
    if (c->probs.count < n_chunks) c->probs.alloc(n_chunks);
    const uint64_t warps = std::min<uint64_t>(n_chunks, uint64_t(c->sm_count) * 64);
    dev::k_prob_chunk_sums<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, c->stream>>>(
        c->amps.ptr, n_chunks, chunk_log2, c->probs.ptr);
    NSB_CUDA(cudaGetLastError());
    copy_d2h(c, out, c->probs.ptr, n_chunks * sizeof(double));
  });
}

int nsb_probabilities_range(nsb_ctx* c, uint64_t offset, uint64_t count, double* out,
                            nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!out && count) throw std::invalid_argument("null output");
    if (offset > c->n_amps || count > c->n_amps - offset)
      throw std::invalid_argument("range outside the state");
    if (!count) return;
    NSB_CUDA(cudaSetDevice(c->device));
    if (c->probs.count < count) c->probs.alloc(count);
    dev::k_probabilities<<<grid_for(count, 256, c), 256, 0, c->stream>>>(c->amps.ptr + offset,
                                                                         count, c->probs.ptr);
    NSB_CUDA(cudaGetLastError());
    copy_d2h(c, out, c->probs.ptr, count * sizeof(double));
  });
}

int nsb_expectation_pauli(nsb_ctx* c, const uint64_t* xmask, const uint64_t* zmask,
                          const double* coeffs, int64_t n_terms, double* out_re, double* out_im,
                          nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (n_terms < 0 || (n_terms > 0 && (!xmask || !zmask || !coeffs)) || !out_re || !out_im)
      throw std::invalid_argument("bad expectation arguments");
    NSB_CUDA(cudaSetDevice(c->device));
    double acc_re = 0.0, acc_im = 0.0;
    for (int64_t t = 0; t < n_terms; ++t) {
      dev::k_pauli_term<<<dev::kReduceBlocks, dev::kReduceThreads, 0, c->stream>>>(
          c->amps.ptr, c->n_amps, xmask[t], zmask[t], c->scratch.ptr);
      dev::k_sum_fixed2<<<1, 32, 0, c->stream>>>(c->scratch.ptr, dev::kReduceBlocks,
                                                  c->scratch.ptr + 2 * dev::kReduceBlocks + 8);
      double s[2];
      NSB_CUDA(cudaMemcpyAsync(s, c->scratch.ptr + 2 * dev::kReduceBlocks + 8, sizeof s,
                               cudaMemcpyDeviceToHost, c->stream));
      NSB_CUDA(cudaStreamSynchronize(c->stream));
      // acc += coeff * s   (coeff complex: phase of the Y letters folded in)
      const double cr = coeffs[2 * t], ci = coeffs[2 * t + 1];
      acc_re += cr * s[0] - ci * s[1];
      acc_im += cr * s[1] + ci * s[0];
    }
    *out_re = acc_re;
    *out_im = acc_im;
  });
}

int nsb_plan_create(nsb_ctx* c, const nsb_op* ops, int64_t n_ops, const double* params,
                    const double* payloads, nsb_plan** out, nsb_status* st) {
  return nsb_plan_create_ex(c, ops, n_ops, params, payloads, 0, out, st);
}

int nsb_plan_create_ex(nsb_ctx* c, const nsb_op* ops, int64_t n_ops, const double* params,
                       const double* payloads, int32_t flags, nsb_plan** out, nsb_status* st) {
  if (!out) return fail_status(st, NSB_EINVAL, "null out pointer");
  *out = nullptr;
  auto P = std::make_unique<nsb_plan>();
  const int rc = guarded(st, [&] {
    require_state(c);
    if (n_ops < 0 || (n_ops > 0 && !ops)) throw std::invalid_argument("bad op list");
    NSB_CUDA(cudaSetDevice(c->device));
    P->device = c->device;
    P->n = c->n;
    NSB_CUDA(cudaStreamCreateWithFlags(&P->rel, cudaStreamNonBlocking));
    if (flags & NSB_PLAN_EXACT) P->host.identity_budget = 0.0;
    P->host.allow_tma = c->tma_ok;
    P->host.octets = c->o1_ok ? plan_octets(c->n) : 2;
    P->host.build(ops, n_ops, params, payloads, c->n, c->blocked_grid);
    HostPlan& H = P->host;
    {
      uint64_t tiles = 1;
      for (const auto* v : {&H.passes, &H.mma_passes})
        for (const PassDesc& pd : *v) tiles = std::max(tiles, uint64_t(1) << (c->n - pd.k));
      // the full persistent grid even when a pass has fewer tiles than CTAs:
      // the CTAs without a tile in pass p arrive at once and stage pass p+1
      // while the others work, and the extra-tile roles alternate between
      // passes, so the next pass's CTAs start staged (ucc8 0.833 vs 0.886 ms,
      // mcm16 5.43 vs 5.62 ms against a grid of one CTA per tile;
      // NSB_TILE_GRID=1 restores that)
      P->grid = c->blocked_grid;
      if (std::getenv("NSB_TILE_GRID"))
        P->grid = static_cast<int>(std::min<uint64_t>(tiles, uint64_t(c->blocked_grid)));
    }
    cudaMemPool_t pool = c->plan_pool;
    P->passes.upload(H.passes.data(), H.passes.size(), c->stream, pool);
    P->mma_passes.upload(H.mma_passes.data(), H.mma_passes.size(), c->stream, pool);
    P->groups.upload(H.groups.data(), H.groups.size(), c->stream, pool);
    P->ops.upload(H.gate_ops.data(), H.gate_ops.size(), c->stream, pool);
    P->mats.upload(reinterpret_cast<const double2*>(H.matrices.data()), H.matrices.size() / 2,
                   c->stream, pool);
    P->dense.upload(reinterpret_cast<const double2*>(H.dense_mats.data()),
                    H.dense_mats.size() / 2, c->stream, pool);
    P->record.alloc(std::max<int64_t>(H.n_measures, 1), c->stream, pool);
    P->partials.alloc(2 * size_t(std::max(c->blocked_grid, 1)), c->stream, pool);
    P->fail.alloc(2, c->stream, pool);
    P->bar.alloc(1, c->stream, pool);
    NSB_CUDA(cudaStreamSynchronize(c->stream));
    for (cudaStream_t* bs : {&P->passes.stream, &P->mma_passes.stream, &P->groups.stream,
                             &P->ops.stream, &P->mats.stream, &P->dense.stream,
                             &P->record.stream, &P->partials.stream, &P->fail.stream,
                             &P->bar.stream})
      *bs = P->rel;
  });
  if (rc == NSB_OK) {
    c->refs.fetch_add(1);
    P->ctx = c;
    *out = P.release();
  }
  return rc;
}

void nsb_plan_destroy(nsb_plan* plan) {
  if (!plan) return;
  cudaSetDevice(plan->device);
  // the host-side program is handed to the reclaimer thread when large
  if (host_plan_bytes(plan->host) > (size_t(8) << 20)) {
    HostPlan* host = nullptr;
    try {
      host = new HostPlan(std::move(plan->host));
      Reclaimer::get().push(host);
    } catch (...) {
      delete host;  // release inline
    }
  }
  nsb_ctx* c = plan->ctx;
  delete plan;
  ctx_release(c);
}

int nsb_plan_info_get(const nsb_plan* plan, nsb_plan_info* info) {
  if (!plan || !info) return NSB_EINVAL;
  plan_info(plan->host, info);
  return NSB_OK;
}

int nsb_plan_run_mma(nsb_ctx* c, nsb_plan* P, double eps, double* assert_probs,
                     nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!P || P->ctx != c) throw std::invalid_argument("plan belongs to another context");
    if (P->n != c->n) throw std::invalid_argument("plan was built for another qubit count");
    NSB_CUDA(cudaSetDevice(c->device));
    HostPlan& H = P->host;
    P->last_launches = 0;
    NSB_CUDA(cudaMemsetAsync(P->fail.ptr, 0, 2 * sizeof(int), c->stream));
    NSB_CUDA(cudaEventRecord(c->ev0, c->stream));
    if (H.mma_ok) {
      if (!H.mma_passes.empty())
        launch_blocked(c, P, P->mma_passes.ptr, 0, static_cast<int>(H.mma_passes.size()), eps);
      NSB_CUDA(cudaEventRecord(c->ev1, c->stream));
      int fail[2] = {0, 0};
      NSB_CUDA(cudaMemcpyAsync(fail, P->fail.ptr, sizeof fail, cudaMemcpyDeviceToHost,
                               c->stream));
      std::vector<double> rec(std::max<int64_t>(H.n_measures, 1));
      NSB_CUDA(cudaMemcpyAsync(rec.data(), P->record.ptr, rec.size() * sizeof(double),
                               cudaMemcpyDeviceToHost, c->stream));
      NSB_CUDA(cudaStreamSynchronize(c->stream));
      float ms = 0.f;
      NSB_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
      P->last_ms = ms;
      const int n_ok = fail[0] ? fail[1] : static_cast<int>(H.n_measures);
      // the reference's P(|0>) includes the norm carried by the near-identity
      // gates the plan does not execute (planner_host.h p0_scale)
      for (int s = 0; s < static_cast<int>(H.n_measures) && s < static_cast<int>(rec.size()); ++s)
        rec[s] *= p0_scale(H, s);
      if (assert_probs)
        for (int s = 0; s < n_ok; ++s) assert_probs[s] = rec[s];
      if (fail[0]) {
        char buf[128];
        std::snprintf(buf, sizeof buf, "assertion failed at step %d: P(|0>) = %.3e", fail[1],
                      rec[fail[1]]);
        throw AssertFailure{fail[1], rec[fail[1]], buf};
      }
      return;
    }
    // item-by-item: k-qubit gates or the unblocked (n < 6) path
    for (const Item& it : H.items) {
      if (it.kind == Item::kMeasure) {
        const double p0 = half_norm(c, it.qubit, 0);
        const double p0_ref = p0 * p0_scale(H, it.step);
        if (p0 < eps) {
          char buf[128];
          std::snprintf(buf, sizeof buf, "assertion failed at step %d: P(|0>) = %.3e", it.step,
                        p0_ref);
          throw AssertFailure{it.step, p0_ref, buf};
        }
        if (assert_probs) assert_probs[it.step] = p0_ref;
        project(c, it.qubit, 0, p0);
        P->last_launches += 3;
      } else if (it.kind != Item::kReset) {
        run_item(c, P, it);
      }
    }
    NSB_CUDA(cudaEventRecord(c->ev1, c->stream));
    NSB_CUDA(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    NSB_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    P->last_ms = ms;
  });
}

int nsb_plan_run_segment(nsb_ctx* c, nsb_plan* P, int64_t seg, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!P || P->ctx != c) throw std::invalid_argument("plan belongs to another context");
    if (P->n != c->n) throw std::invalid_argument("plan was built for another qubit count");
    if (seg < 0 || seg >= static_cast<int64_t>(P->host.items.size()))
      throw std::invalid_argument("item index out of range");
    NSB_CUDA(cudaSetDevice(c->device));
    run_item(c, P, P->host.items[seg]);
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

// Rejection mode (engine.py:431-474) through the C ABI.  The caller supplies
// its Philox uniforms (rng.random() draws in order); they are consumed exactly
// as the reference consumes them: one per executed MEASURE, one per executed
// RESET, one per accepted shot's sample (engine.py:443, 452, 462).
// Filter-shaped circuits (every MEASURE followed by a RESET of the same qubit,
// every RESET after such a MEASURE) are replayed: ONE device pass along the
// all-zero path records P(0) at every marker (with the reset's
// renormalisation, engine.py:455), and the shots are decided on the host from
// the draws; a reset draw of 1 leaves that path and the shot is simulated
// explicitly from its forced outcomes on.  Other circuits (or flags & 1) run
// every shot on the device.
int nsb_plan_run_rejection(nsb_ctx* c, nsb_plan* P, const double* uniforms, int64_t n_uniforms,
                           int64_t shots, int32_t flags, int64_t* consumed, int64_t* accepted,
                           int64_t* step_rejections, int64_t* sample_index, double* first_state,
                           nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!P || P->ctx != c) throw std::invalid_argument("plan belongs to another context");
    if (P->n != c->n) throw std::invalid_argument("plan was built for another qubit count");
    if (shots < 0 || (shots > 0 && (!uniforms || !sample_index)) || !consumed || !accepted)
      throw std::invalid_argument("bad rejection arguments");
    NSB_CUDA(cudaSetDevice(c->device));
    const HostPlan& H = P->host;
    if (H.n_identity_gates) throw std::invalid_argument("rejection mode needs an exact plan");
    const std::vector<Item>& items = H.items;
    int64_t cur = 0;
    auto draw = [&]() -> double {
      if (cur >= n_uniforms) throw std::invalid_argument("uniform stream exhausted");
      return uniforms[cur++];
    };
    for (int64_t s = 0; s < H.n_measures; ++s) step_rejections[s] = 0;
    *accepted = 0;
    std::vector<double> cum;
    auto cumsum = [&]() {  // np.cumsum of re*re + im*im (sequential, engine.py:215-216)
      if (c->probs.count < c->n_amps) c->probs.alloc(c->n_amps);
      dev::k_probabilities<<<grid_for(c->n_amps, 256, c), 256, 0, c->stream>>>(
          c->amps.ptr, c->n_amps, c->probs.ptr);
      NSB_CUDA(cudaGetLastError());
      cum.resize(c->n_amps);
      copy_d2h(c, cum.data(), c->probs.ptr, c->n_amps * sizeof(double));
      for (uint64_t i = 1; i < c->n_amps; ++i) cum[i] = cum[i - 1] + cum[i];
    };
    auto sample_one = [&](double u) -> int64_t {  // searchsorted(side="right"), clipped
      const double x = u * cum.back();
      int64_t idx = std::upper_bound(cum.begin(), cum.end(), x) - cum.begin();
      return std::min<int64_t>(idx, static_cast<int64_t>(cum.size()) - 1);
    };
    auto restart = [&]() {
      dev::k_vacuum<<<grid_for(c->n_amps, 256, c), 256, 0, c->stream>>>(c->amps.ptr, c->n_amps);
      NSB_CUDA(cudaGetLastError());
    };
    static const double kX[8] = {0, 0, 1, 0, 1, 0, 0, 0};
    bool kept = false;
    auto keep = [&]() {
      if (first_state && !kept) {
        copy_d2h(c, first_state, c->amps.ptr, c->n_amps * sizeof(double2));
        kept = true;
      }
    };
    // one shot on the device from |0...0> (engine.py:436-463); the first
    // forced.size() marker outcomes are given (their draws were taken)
    auto explicit_shot = [&](const std::vector<int>& forced, int64_t shot) {
      restart();
      size_t j = 0;
      for (size_t i = 0; i < items.size(); ++i) {
        const Item& it = items[i];
        if (it.kind == Item::kMeasure || it.kind == Item::kReset) {
          const double p0 = half_norm(c, it.qubit, 0);
          const int outcome = j < forced.size() ? forced[j] : (draw() < p0 ? 0 : 1);
          ++j;
          if (it.kind == Item::kMeasure) {
            if (outcome) {
              ++step_rejections[it.step];
              sample_index[shot] = -1;
              return;
            }
            project(c, it.qubit, 0, p0);
          } else {
            project(c, it.qubit, outcome, outcome == 0 ? p0 : 1.0 - p0);
            if (outcome) apply_matrix(c, kX, &it.qubit, 1, nullptr);
          }
        } else {
          run_item(c, P, it);
        }
      }
      ++*accepted;
      cumsum();
      sample_index[shot] = sample_one(draw());
      keep();
    };
    bool replay = !(flags & 1);
    {  // filter-shaped: MEASURE q, RESET q pairs only (engine._replayable)
      std::vector<const Item*> marks;
      for (const Item& it : items)
        if (it.kind == Item::kMeasure || it.kind == Item::kReset) marks.push_back(&it);
      if (marks.empty() || marks.size() % 2) replay = false;
      for (size_t i = 0; replay && i < marks.size(); i += 2)
        replay = marks[i]->kind == Item::kMeasure && marks[i + 1]->kind == Item::kReset &&
                 marks[i]->qubit == marks[i + 1]->qubit;
    }
    if (!replay) {
      for (int64_t s = 0; s < shots; ++s) explicit_shot({}, s);
      *consumed = cur;
      NSB_CUDA(cudaStreamSynchronize(c->stream));
      return;
    }
    // one pass along the accepted path
    struct Mark {
      bool measure;
      int step;
      double p;
    };
    std::vector<Mark> path;
    bool reachable = true;
    restart();
    for (const Item& it : items) {
      if (it.kind == Item::kMeasure) {
        const double p0 = half_norm(c, it.qubit, 0);
        path.push_back({true, it.step, p0});
        if (p0 <= 0.0) {
          reachable = false;  // every shot stops here
          break;
        }
        project(c, it.qubit, 0, p0);
      } else if (it.kind == Item::kReset) {
        const double p0 = half_norm(c, it.qubit, 0);
        path.push_back({false, -1, p0});
        project(c, it.qubit, 0, p0);
      } else {
        run_item(c, P, it);
      }
    }
    if (reachable) {
      cumsum();
      keep();
    }
    std::vector<double> path_cum = cum;
    for (int64_t s = 0; s < shots; ++s) {
      std::vector<int> forced;
      int outcome = -1;  // >= 0: rejected at that step; -2: left the path
      for (const Mark& m : path) {
        const double u = draw();
        if (m.measure) {
          if (!(u < m.p)) {
            outcome = m.step;
            break;
          }
          forced.push_back(0);
        } else if (!(u < m.p)) {  // reset drew 1
          forced.push_back(1);
          outcome = -2;
          break;
        } else {
          forced.push_back(0);
        }
      }
      if (outcome >= 0) {
        ++step_rejections[outcome];
        sample_index[s] = -1;
        continue;
      }
      if (outcome == -2) {
        explicit_shot(forced, s);
        cum = path_cum;
        continue;
      }
      ++*accepted;
      sample_index[s] = sample_one(draw());
    }
    *consumed = cur;
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

// MMA run with planning streamed behind execution (engine.run's MMA path, the
// reference-facing call): the op list is cut at its MEASURE / RESET markers
// (the relabeling frame is flushed there, so the parts are independent
// planning problems); a host thread plans the parts in order, each with all
// cores on its passes, and the caller's thread uploads part s and launches
// its passes (one cooperative k_blocked launch per part, pass descriptors with
// the assertion epilogue / collapse prologue of the markers around it) while
// part s+1 is being planned.  A launch that starts with a collapse takes p0
// from the record; a failed assertion makes the later launches return at once.
// Reported p0 carry the parts' near-identity norm factors as in
// nsb_plan_run_mma.  Circuits with k >= 3 dense gates or fewer than 6 qubits
// are not streamed (NSB_EINVAL: use nsb_plan_create + nsb_plan_run_mma).
int nsb_run_mma_streamed(nsb_ctx* c, const nsb_op* ops, int64_t n_ops, const double* params,
                         const double* payloads, double eps, double* assert_probs,
                         int64_t* n_measures, double* device_ms, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (n_ops < 0 || (n_ops > 0 && !ops) || !n_measures) throw std::invalid_argument("bad op list");
    if (c->n < 6) throw std::invalid_argument("streamed MMA runs need >= 6 qubits");
    NSB_CUDA(cudaSetDevice(c->device));
    std::vector<int64_t> marks;
    int64_t n_meas = 0;
    for (int64_t i = 0; i < n_ops; ++i) {
      if (ops[i].kind == NSB_OP_MEASURE || ops[i].kind == NSB_OP_RESET) marks.push_back(i);
      if (ops[i].kind == NSB_OP_MEASURE) ++n_meas;
      if (ops[i].kind == NSB_OP_GATE && ops[i].nq >= 3)
        throw std::invalid_argument("streamed MMA runs take 1q / 2q gates only");
    }
    *n_measures = n_meas;
    // parts: the gate runs between markers; the first run is also cut at 1/16,
    // 1/8, 1/4 and 1/2 of its length (an exact frame flush at each cut) so the
    // device starts after a short plan instead of a whole filter step
    struct Range {
      int64_t b, e;
      int64_t mark;  // index of the marker ending the part, -1: an artificial cut
    };
    std::vector<Range> ranges;
    for (size_t s = 0; s <= marks.size(); ++s) {
      const int64_t b = s == 0 ? 0 : marks[s - 1] + 1, e = s < marks.size() ? marks[s] : n_ops;
      const int64_t mk = s < marks.size() ? marks[s] : -1;
      if (s == 0 && e - b >= 4096) {
        int64_t at = b;
        for (int64_t div : {16, 8, 4, 2}) {
          const int64_t cut = b + (e - b) / div;
          if (cut > at) {
            ranges.push_back({at, cut, -1});
            at = cut;
          }
        }
        ranges.push_back({at, e, mk});
      } else {
        ranges.push_back({b, e, mk});
      }
    }
    const size_t n_parts = ranges.size();
    const double budget = default_identity_budget_value();
    // producer: parts planned in order on a host thread
    std::vector<std::unique_ptr<HostPlan>> parts(n_parts);
    std::vector<std::exception_ptr> errs(n_parts);
    std::mutex mu;
    std::condition_variable cv;
    size_t ready = 0;
    std::atomic<bool> stop{false};
    std::thread producer([&] {
      for (size_t s = 0; s < n_parts && !stop.load(); ++s) {
        const int64_t b = ranges[s].b, e = ranges[s].e;
        auto H = std::make_unique<HostPlan>();
        try {
          H->identity_budget = n_ops ? budget * static_cast<double>(e - b) / n_ops : 0.0;
          H->allow_tma = c->tma_ok;
          H->octets = c->o1_ok ? plan_octets(c->n) : 2;
          H->build_segment(ops + b, e - b, params, payloads, c->n, c->blocked_grid);
        } catch (...) {
          errs[s] = std::current_exception();
        }
        {
          std::lock_guard<std::mutex> lk(mu);
          parts[s] = std::move(H);
          ready = s + 1;
        }
        cv.notify_one();
      }
    });
    struct PartDev {
      DevBuf<dev::TmaPass> tmaps;  // TMA parts: tensor maps per pass
      DevBuf<PassDesc> passes;
      DevBuf<GroupDesc> groups;
      DevBuf<GateOp> ops;
      DevBuf<double2> mats;
    };
    std::vector<PartDev> dev(n_parts + 1);
    DevBuf<double> record, partials;
    DevBuf<int> fail;
    DevBuf<unsigned> bar;
    cudaMemPool_t pool = c->plan_pool;
    record.alloc(std::max<int64_t>(n_meas, 1), c->stream, pool);
    partials.alloc(2 * size_t(std::max(c->blocked_grid, 1)), c->stream, pool);
    fail.alloc(2, c->stream, pool);
    bar.alloc(1, c->stream, pool);
    NSB_CUDA(cudaMemsetAsync(fail.ptr, 0, 2 * sizeof(int), c->stream));
    NSB_CUDA(cudaEventRecord(c->ev0, c->stream));
    static const int debug = [] {
      const char* e = std::getenv("NSB_DEBUG_BLOCKED");
      return e ? std::atoi(e) : 0;
    }();
    int grid = 0;
    auto launch = [&](PartDev& d, int count, bool tma, int oct) {
      dev::BlockedParams bp;
      bp.amps = c->amps.ptr;
      bp.n = c->n;
      bp.passes = d.passes.ptr;
      bp.pass_begin = 0;
      bp.pass_end = count;
      bp.groups = d.groups.ptr;
      bp.ops = d.ops.ptr;
      bp.mats = d.mats.ptr;
      bp.partials = partials.ptr;
      bp.record = record.ptr;
      bp.fail = fail.ptr;
      bp.bar = bar.ptr;
      bp.eps = eps;
      bp.debug = debug;
      bp.cmask = bp.cval = 0;
      bp.cbits = 0;
      bp.tmaps = tma ? d.tmaps.ptr : nullptr;
      bp.tma_store = tma_store_mode();
      NSB_CUDA(cudaMemsetAsync(bar.ptr, 0, sizeof(unsigned), c->stream));
      void* args[] = {&bp};
      NSB_CUDA(cudaLaunchCooperativeKernel(
          blocked_kernel(false, tma, oct), dim3(grid), dim3(blocked_threads(oct)), args,
          tma ? dev::kBlockedSmemBytesTma : dev::kBlockedSmemBytes, c->stream));
    };
    std::vector<double> scale(std::max<int64_t>(n_meas, 1), 1.0);
    double running = 1.0;
    int pending_q = -1, pending_slot = -1, step = 0;
    int k_tile = 0;
    auto fresh = [&]() {
      PassDesc P{};
      P.k = k_tile;
      P.measure_q = P.collapse_q = -1;
      P.measure_slot = P.collapse_slot = -1;
      int t = 0, o = 0;
      for (int q = 0; q < c->n; ++q) {
        if (q < k_tile)
          P.tq[t++] = static_cast<int8_t>(q);
        else
          P.oq[o++] = static_cast<int8_t>(q);
      }
      return P;
    };
    try {
      for (size_t s = 0; s < n_parts; ++s) {
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return ready > s; });
        }
        if (errs[s]) std::rethrow_exception(errs[s]);
        HostPlan& H = *parts[s];
        if (!H.blocked) throw std::invalid_argument("streamed MMA runs need a blocked plan");
        for (const Item& it : H.items)
          if (it.kind == Item::kDense) throw std::invalid_argument("dense k-qubit item in a stream");
        if (!grid) {
          k_tile = H.tile_qubits;
          grid = c->blocked_grid;  // as nsb_plan_create_ex: the full grid
          if (std::getenv("NSB_TILE_GRID"))
            grid = static_cast<int>(std::min<uint64_t>(uint64_t(1) << (c->n - k_tile),
                                                       uint64_t(c->blocked_grid)));
        }
        std::vector<PassDesc> mp = H.passes;  // one kGates item at most: all passes in order
        if (!mp.empty() && pending_q >= 0) {
          mp.front().collapse_q = pending_q;
          mp.front().collapse_slot = pending_slot;
          pending_q = -1;
        }
        running *= H.tail_scale2;
        const int64_t mk = ranges[s].mark;
        if (mk >= 0 && ops[mk].kind == NSB_OP_MEASURE) {
          if (mp.empty() || pending_q >= 0) {
            PassDesc P = fresh();
            if (pending_q >= 0) {
              P.collapse_q = pending_q;
              P.collapse_slot = pending_slot;
              pending_q = -1;
            }
            mp.push_back(P);
          }
          mp.back().measure_q = ops[mk].q[0];
          mp.back().measure_slot = step;
          pending_q = ops[mk].q[0];
          pending_slot = step;
          scale[step] = running;
          running = 1.0;
          ++step;
        }
        if (s + 1 == n_parts && pending_q >= 0) {  // the last collapse
          PassDesc P = fresh();
          P.collapse_q = pending_q;
          P.collapse_slot = pending_slot;
          mp.push_back(P);
        }
        if (!mp.empty()) {
          PartDev& d = dev[s];
          d.passes.upload(mp.data(), mp.size(), c->stream, pool);
          d.groups.upload(H.groups.data(), H.groups.size(), c->stream, pool);
          d.ops.upload(H.gate_ops.data(), H.gate_ops.size(), c->stream, pool);
          d.mats.upload(reinterpret_cast<const double2*>(H.matrices.data()),
                        H.matrices.size() / 2, c->stream, pool);
          if (H.tma) {
            std::vector<dev::TmaPass> tm;
            encode_tma_passes(mp, c->n, c->amps.ptr, tm);
            d.tmaps.upload(tm.data(), tm.size(), c->stream, pool);
          }
          launch(d, static_cast<int>(mp.size()), H.tma, H.octets);
        }
        if (s > 0) {  // planned parts already uploaded: release their host programs
          std::lock_guard<std::mutex> lk(mu);
          parts[s - 1].reset();
        }
      }
    } catch (...) {
      stop = true;
      producer.join();
      throw;
    }
    producer.join();
    NSB_CUDA(cudaEventRecord(c->ev1, c->stream));
    int fl[2] = {0, 0};
    NSB_CUDA(cudaMemcpyAsync(fl, fail.ptr, sizeof fl, cudaMemcpyDeviceToHost, c->stream));
    std::vector<double> rec(std::max<int64_t>(n_meas, 1));
    NSB_CUDA(cudaMemcpyAsync(rec.data(), record.ptr, rec.size() * sizeof(double),
                             cudaMemcpyDeviceToHost, c->stream));
    NSB_CUDA(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    NSB_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    if (device_ms) *device_ms = ms;
    for (int64_t i = 0; i < n_meas; ++i) rec[i] *= scale[i];
    const int64_t n_ok = fl[0] ? fl[1] : n_meas;
    if (assert_probs)
      for (int64_t i = 0; i < n_ok; ++i) assert_probs[i] = rec[i];
    for (PartDev& d : dev) {  // stream-ordered frees on the context stream
      d.tmaps.release();
      d.passes.release();
      d.groups.release();
      d.ops.release();
      d.mats.release();
    }
    if (fl[0]) {
      char buf[128];
      std::snprintf(buf, sizeof buf, "assertion failed at step %d: P(|0>) = %.3e", fl[1], rec[fl[1]]);
      throw AssertFailure{fl[1], rec[fl[1]], buf};
    }
  });
}

int nsb_plan_segment_marker(const nsb_plan* P, int64_t seg, int32_t* kind, int32_t* qubit,
                            int32_t* step) {
  if (!P || seg < 0 || seg >= static_cast<int64_t>(P->host.items.size()) || !kind || !qubit ||
      !step)
    return NSB_EINVAL;
  const Item& it = P->host.items[seg];
  *kind = it.kind == Item::kMeasure ? NSB_OP_MEASURE
                                    : (it.kind == Item::kReset ? NSB_OP_RESET : NSB_OP_GATE);
  *qubit = it.qubit;
  *step = it.step;
  return NSB_OK;
}

int nsb_plan_p0_scale(const nsb_plan* P, int32_t step, double* scale) {
  if (!P || !scale || step < 0 || step >= P->host.n_measures) return NSB_EINVAL;
  *scale = p0_scale(P->host, step);
  return NSB_OK;
}

int nsb_plan_last_timing(const nsb_plan* P, double* ms, int64_t* launches) {
  if (!P) return NSB_EINVAL;
  if (ms) *ms = P->last_ms;
  if (launches) *launches = P->last_launches;
  return NSB_OK;
}

int nsb_timer_start(nsb_ctx* c, nsb_status* st) {
  return guarded(st, [&] {
    if (!c) throw std::invalid_argument("null context");
    NSB_CUDA(cudaSetDevice(c->device));
    NSB_CUDA(cudaEventRecord(c->tev0, c->stream));
  });
}

int nsb_timer_stop(nsb_ctx* c, double* ms, nsb_status* st) {
  return guarded(st, [&] {
    if (!c || !ms) throw std::invalid_argument("null argument");
    NSB_CUDA(cudaSetDevice(c->device));
    NSB_CUDA(cudaEventRecord(c->tev1, c->stream));
    NSB_CUDA(cudaEventSynchronize(c->tev1));
    float f = 0.f;
    NSB_CUDA(cudaEventElapsedTime(&f, c->tev0, c->tev1));
    *ms = f;
  });
}

// ---------------------------------------------------------------------------
// sharded state

int nsb_comm_unique_id(uint8_t* id, nsb_status* st) {
  return guarded(st, [&] {
    if (!id) throw std::invalid_argument("null id buffer");
    ncclUniqueId u;
    NSB_NCCL(shard_nccl().get_unique_id(&u));
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

int nsb_comm_init(nsb_ctx* c, const uint8_t* id, int32_t nranks, int32_t rank, nsb_status* st) {
  if (!c || !id) return fail_status(st, NSB_EINVAL, "null argument");
  if (nranks < 1 || (nranks & (nranks - 1)) || rank < 0 || rank >= nranks)
    return fail_status(st, NSB_EINVAL, "rank count must be a power of two and rank < count");
  return guarded(st, [&] {
    NSB_CUDA(cudaSetDevice(c->device));
    if (c->comm) shard_comm_destroy(c);
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t comm = nullptr;
    NSB_NCCL(shard_nccl().comm_init_rank(&comm, nranks, u, rank));
    c->comm = comm;
    c->rank = rank;
    c->nranks = nranks;
    if (!c->xfer) {
      NSB_CUDA(cudaStreamCreateWithFlags(&c->xfer, cudaStreamNonBlocking));
      for (int b = 0; b < 2; ++b) {
        NSB_CUDA(cudaEventCreateWithFlags(&c->ev_packed[b], cudaEventDisableTiming));
        NSB_CUDA(cudaEventCreateWithFlags(&c->ev_moved[b], cudaEventDisableTiming));
        NSB_CUDA(cudaEventCreateWithFlags(&c->ev_unpacked[b], cudaEventDisableTiming));
      }
    }
  });
}

int nsb_shard_swap(nsb_ctx* c, int32_t global_bit, int32_t local_q, int64_t chunk_amps,
                   nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!c->comm) throw std::invalid_argument("no communicator (nsb_comm_init)");
    if (global_bit < 0 || (1 << global_bit) >= c->nranks || local_q < 0 || local_q >= c->n)
      throw std::invalid_argument("bad shard swap qubits");
    NSB_CUDA(cudaSetDevice(c->device));
    const NcclApi& api = shard_nccl();
    const int peer = c->rank ^ (1 << global_bit);
    const int v = 1 - ((c->rank >> global_bit) & 1);  // the half that changes owner
    const uint64_t half = c->n_amps >> 1;
    const uint64_t chunk =
        std::min<uint64_t>(half, chunk_amps > 0 ? uint64_t(chunk_amps) : (uint64_t(1) << 25));
    // pack / unpack run beside NCCL's copy kernels: leave most SMs to them
    const unsigned pgrid = static_cast<unsigned>(std::max(1, c->sm_count / 2));
    for (int b = 0; b < 2; ++b)
      if (c->stage_send[b].count < chunk) {
        c->stage_send[b].alloc(chunk);
        c->stage_recv[b].alloc(chunk);
      }
    auto comm = static_cast<ncclComm_t>(c->comm);
    // Pipeline over chunks j: pack(j) and unpack(j) on the compute stream,
    // the exchange of j on the transfer stream, so pack(j+1) and unpack(j-1)
    // overlap the NVLink transfer of j.  Staging buffers alternate (j & 1).
    const uint64_t n_chunks = (half + chunk - 1) / chunk;
    auto count = [&](uint64_t j) { return std::min(chunk, half - j * chunk); };
    auto pack = [&](uint64_t j) {
      const int b = static_cast<int>(j & 1);
      const uint64_t cnt = count(j);
      dev::k_shard_pack<<<pgrid, 512, 0, c->stream>>>(c->amps.ptr, c->stage_send[b].ptr,
                                                      j * chunk, cnt, local_q, v);
      NSB_CUDA(cudaGetLastError());
      NSB_CUDA(cudaEventRecord(c->ev_packed[b], c->stream));
    };
    NSB_CUDA(cudaEventRecord(c->ev_unpacked[0], c->stream));  // buffers free
    NSB_CUDA(cudaEventRecord(c->ev_unpacked[1], c->stream));
    pack(0);
    for (uint64_t j = 0; j < n_chunks; ++j) {
      const int b = static_cast<int>(j & 1);
      const uint64_t cnt = count(j);
      NSB_CUDA(cudaStreamWaitEvent(c->xfer, c->ev_packed[b], 0));
      NSB_CUDA(cudaStreamWaitEvent(c->xfer, c->ev_unpacked[b], 0));
      NSB_NCCL(api.group_start());
      NSB_NCCL(api.send(c->stage_send[b].ptr, 2 * cnt, ncclFloat64, peer, comm, c->xfer));
      NSB_NCCL(api.recv(c->stage_recv[b].ptr, 2 * cnt, ncclFloat64, peer, comm, c->xfer));
      NSB_NCCL(api.group_end());
      NSB_CUDA(cudaEventRecord(c->ev_moved[b], c->xfer));
      if (j + 1 < n_chunks) {  // the send buffer of j+1 was last read by exchange j-1
        NSB_CUDA(cudaStreamWaitEvent(c->stream, c->ev_moved[b ^ 1], 0));
        pack(j + 1);
      }
      NSB_CUDA(cudaStreamWaitEvent(c->stream, c->ev_moved[b], 0));
      dev::k_shard_unpack<<<pgrid, 512, 0, c->stream>>>(c->amps.ptr, c->stage_recv[b].ptr,
                                                        j * chunk, cnt, local_q, v);
      NSB_CUDA(cudaGetLastError());
      NSB_CUDA(cudaEventRecord(c->ev_unpacked[b], c->stream));
    }
    NSB_CUDA(cudaStreamSynchronize(c->stream));
    NSB_CUDA(cudaStreamSynchronize(c->xfer));
  });
}

int nsb_shard_ipc_handle(nsb_ctx* c, uint8_t* handle, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!handle) throw std::invalid_argument("null handle");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    NSB_CUDA(cudaSetDevice(c->device));
    cudaIpcMemHandle_t h;
    NSB_CUDA(cudaIpcGetMemHandle(&h, c->amps.ptr));
    std::memcpy(handle, &h, sizeof h);
  });
}

int nsb_shard_open_peers(nsb_ctx* c, const uint8_t* handles, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!c->comm) throw std::invalid_argument("no communicator (nsb_comm_init)");
    if (!handles) throw std::invalid_argument("null handles");
    if (c->nranks > 64) throw std::invalid_argument("too many ranks for peer mapping");
    NSB_CUDA(cudaSetDevice(c->device));
    {  // every rank's shard must have this rank's size
      double* buf = c->scratch.ptr + 2 * dev::kReduceBlocks + 8;
      if (c->scratch.count < size_t(2 * dev::kReduceBlocks + 8 + 1 + c->nranks))
        throw std::invalid_argument("rank count exceeds scratch");
      const double mine = static_cast<double>(c->n_amps);
      NSB_CUDA(cudaMemcpyAsync(buf, &mine, sizeof mine, cudaMemcpyHostToDevice, c->stream));
      NSB_NCCL(shard_nccl().all_gather(buf, buf + 1, 1, ncclFloat64,
                                       static_cast<ncclComm_t>(c->comm), c->stream));
      std::vector<double> sizes(c->nranks);
      NSB_CUDA(cudaMemcpyAsync(sizes.data(), buf + 1, sizeof(double) * c->nranks,
                               cudaMemcpyDeviceToHost, c->stream));
      NSB_CUDA(cudaStreamSynchronize(c->stream));
      for (double v : sizes)
        if (v != mine) throw std::invalid_argument("peer shards differ in size");
    }
    for (int r = 0; r < c->nranks; ++r) {
      if (r == c->rank) continue;
      if (c->peers[r]) {  // re-open: the partner may have reallocated its shard
        NSB_CUDA(cudaIpcCloseMemHandle(c->peers[r]));
        c->peers[r] = nullptr;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + 64 * r, sizeof h);
      void* p = nullptr;
      NSB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      c->peers[r] = static_cast<double2*>(p);
    }
  });
}

// stream-ordered rendezvous of all ranks (an 8-byte all-gather on the stream)
void comm_barrier(nsb_ctx* c) {
  double* buf = c->scratch.ptr + 2 * dev::kReduceBlocks + 8;
  NSB_NCCL(shard_nccl().all_gather(buf, buf + 1, 1, ncclFloat64,
                                   static_cast<ncclComm_t>(c->comm), c->stream));
}

// Collective: unmap the partners' shards, then a rendezvous, so no rank frees
// (or reallocates) its exported shard while another still maps it.
int nsb_shard_close_peers(nsb_ctx* c, nsb_status* st) {
  return guarded(st, [&] {
    if (!c || !c->comm) throw std::invalid_argument("no communicator (nsb_comm_init)");
    NSB_CUDA(cudaSetDevice(c->device));
    NSB_CUDA(cudaStreamSynchronize(c->stream));
    for (double2*& p : c->peers)
      if (p) {
        NSB_CUDA(cudaIpcCloseMemHandle(p));
        p = nullptr;
      }
    comm_barrier(c);
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int nsb_shard_swap_p2p(nsb_ctx* c, int32_t global_bit, int32_t local_q, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!c->comm) throw std::invalid_argument("no communicator (nsb_comm_init)");
    if (global_bit < 0 || (1 << global_bit) >= c->nranks || local_q < 0 || local_q >= c->n)
      throw std::invalid_argument("bad shard swap qubits");
    const int partner = c->rank ^ (1 << global_bit);
    if (!c->peers[partner]) throw std::invalid_argument("peer shard not mapped (nsb_shard_open_peers)");
    if (c->scratch.count < size_t(2 * dev::kReduceBlocks + 8 + 1 + c->nranks))
      throw std::invalid_argument("barrier exceeds scratch");
    NSB_CUDA(cudaSetDevice(c->device));
    const int b = (c->rank >> global_bit) & 1;
    const uint64_t half = c->n_amps >> 1;
    const int clog = static_cast<int>(std::min<uint64_t>(16, c->n - 1));
    comm_barrier(c);  // both shards are final before either is touched
    dev::k_shard_swap_p2p<<<static_cast<unsigned>(c->sm_count * 4), 256, 0, c->stream>>>(
        c->amps.ptr, c->peers[partner], half, local_q, 1 - b, b, b, clog);
    NSB_CUDA(cudaGetLastError());
    comm_barrier(c);  // both halves of the exchange landed before either continues
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int nsb_plan_run_segment_chunked(nsb_ctx* c, nsb_plan* P, int64_t seg, int32_t chunk_bits,
                                 int32_t* n_chunked, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!P || P->ctx != c) throw std::invalid_argument("plan belongs to another context");
    if (P->n != c->n) throw std::invalid_argument("plan was built for another qubit count");
    if (seg < 0 || seg >= static_cast<int64_t>(P->host.items.size()))
      throw std::invalid_argument("item index out of range");
    NSB_CUDA(cudaSetDevice(c->device));
    uint64_t cm = 0;
    const int np = chunk_prefix(P->host, seg, -1, chunk_bits, &cm);
    if (n_chunked) *n_chunked = np;
    const Item& it = P->host.items[static_cast<size_t>(seg)];
    if (np == 0) {
      run_item(c, P, it);
    } else {
      const int cb = __builtin_popcountll(cm);
      for (uint64_t ch = 0; ch < (uint64_t(1) << cb); ++ch)
        launch_blocked(c, P, P->passes.ptr, it.pass_begin, it.pass_begin + np, -1.0, 0, cm,
                       deposit_bits(ch, cm));
      if (it.pass_begin + np < it.pass_end)
        launch_blocked(c, P, P->passes.ptr, it.pass_begin + np, it.pass_end, -1.0);
    }
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

// Overlapped qubit swap (header): the chunk pipeline.  Swap stream: chunk
// kernels back to back, each followed by its flag signal; gate stream: per
// chunk, wait for both partners' flags, then the item's chunkable passes on
// that chunk (grid reduced by the swap CTAs, which share the SMs); then the
// rest of the item on every tile.
int nsb_shard_swap_overlap(nsb_ctx* c, int32_t global_bit, int32_t local_q, nsb_plan* P,
                           int64_t seg, int32_t chunk_bits, int32_t swap_ctas,
                           int32_t* n_chunked, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!c->comm) throw std::invalid_argument("no communicator (nsb_comm_init)");
    if (global_bit < 0 || (1 << global_bit) >= c->nranks || local_q < 0 || local_q >= c->n)
      throw std::invalid_argument("bad shard swap qubits");
    if (!P || P->ctx != c) throw std::invalid_argument("plan belongs to another context");
    if (P->n != c->n) throw std::invalid_argument("plan was built for another qubit count");
    if (seg < 0 || seg >= static_cast<int64_t>(P->host.items.size()))
      throw std::invalid_argument("item index out of range");
    const int partner = c->rank ^ (1 << global_bit);
    if (!c->peers[partner]) throw std::invalid_argument("peer shard not mapped (nsb_shard_open_peers)");
    NSB_CUDA(cudaSetDevice(c->device));
    uint64_t cm = 0;
    const int np = chunk_prefix(P->host, seg, local_q, chunk_bits, &cm);
    if (n_chunked) *n_chunked = np;
    const Item& it = P->host.items[static_cast<size_t>(seg)];
    const int b = (c->rank >> global_bit) & 1;
    const uint64_t half = c->n_amps >> 1;
    if (np == 0) {  // nothing chunkable: swap, then the item
      const int clog = static_cast<int>(std::min<uint64_t>(16, c->n - 1));
      comm_barrier(c);
      dev::k_shard_swap_p2p<<<static_cast<unsigned>(c->sm_count * 4), 256, 0, c->stream>>>(
          c->amps.ptr, c->peers[partner], half, local_q, 1 - b, b, b, clog);
      NSB_CUDA(cudaGetLastError());
      comm_barrier(c);
      run_item(c, P, it);
      NSB_CUDA(cudaStreamSynchronize(c->stream));
      return;
    }
    if (!c->xfer) NSB_CUDA(cudaStreamCreateWithFlags(&c->xfer, cudaStreamNonBlocking));
    if (!c->ev_ov0) NSB_CUDA(cudaEventCreateWithFlags(&c->ev_ov0, cudaEventDisableTiming));
    if (!c->ev_ov1) NSB_CUDA(cudaEventCreateWithFlags(&c->ev_ov1, cudaEventDisableTiming));
    const int cb = __builtin_popcountll(cm);
    const int n_ch = 1 << cb;
    if (2 * n_ch > dev::kShardFlagWords) throw std::invalid_argument("too many swap chunks");
    const int ctas = swap_ctas > 0 ? swap_ctas : 32;
    const int grid = std::max(1, P->grid - ctas);
    const unsigned epoch = ++c->swap_epoch;
    unsigned* f_mine = shard_flags(c->amps.ptr, c->n_amps);
    unsigned* f_peer = shard_flags(c->peers[partner], c->n_amps);
    dev::SwapChunk sc{};
    {
      std::vector<int> pos;
      for (uint64_t m = cm | (uint64_t(1) << local_q); m; m &= m - 1) pos.push_back(__builtin_ctzll(m));
      sc.npos = static_cast<int>(pos.size());
      for (int i = 0; i < sc.npos; ++i) sc.pos[i] = pos[i];
      sc.n_pairs = half >> cb;
    }
    const int clog = static_cast<int>(std::min<uint64_t>(16, c->n - 1 - cb));
    // timing experiments only (wrong states): 1 = no swap kernels, 2 = no chunked passes
    static const int ov_debug = [] {
      const char* e = std::getenv("NSB_OVERLAP_DEBUG");
      return e ? std::atoi(e) : 0;
    }();
    comm_barrier(c);  // both shards are final before either is touched
    NSB_CUDA(cudaEventRecord(c->ev_ov0, c->stream));
    NSB_CUDA(cudaStreamWaitEvent(c->xfer, c->ev_ov0, 0));
    for (int ch = 0; ch < n_ch; ++ch) {
      const uint64_t cv = deposit_bits(static_cast<uint64_t>(ch), cm);
      sc.fixed_mine = cv | (uint64_t(1 - b) << local_q);
      sc.fixed_peer = cv | (uint64_t(b) << local_q);
      if (!(ov_debug & 1)) {
        dev::k_shard_swap_chunk<<<static_cast<unsigned>(ctas), dev::kSwapThreads, 0, c->xfer>>>(
            c->amps.ptr, c->peers[partner], sc, b, clog);
        NSB_CUDA(cudaGetLastError());
      }
      dev::k_flag_signal<<<1, 1, 0, c->xfer>>>(f_mine, f_peer, 2 * ch + b, epoch);
      NSB_CUDA(cudaGetLastError());
    }
    for (int ch = 0; ch < n_ch; ++ch) {
      dev::k_flag_wait<<<1, 32, 0, c->stream>>>(f_mine, 2 * ch, 2 * ch + 1, epoch);
      NSB_CUDA(cudaGetLastError());
      if (!(ov_debug & 2))
        launch_blocked(c, P, P->passes.ptr, it.pass_begin, it.pass_begin + np, -1.0, grid, cm,
                       deposit_bits(static_cast<uint64_t>(ch), cm));
    }
    if (it.pass_begin + np < it.pass_end)
      launch_blocked(c, P, P->passes.ptr, it.pass_begin + np, it.pass_end, -1.0);
    NSB_CUDA(cudaEventRecord(c->ev_ov1, c->xfer));
    NSB_CUDA(cudaStreamWaitEvent(c->stream, c->ev_ov1, 0));
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int nsb_shard_swap_overlap_ce(nsb_ctx* c, int32_t global_bit, int32_t local_q, nsb_plan* P,
                              int64_t seg, int32_t chunk_bits, int64_t stage_bytes,
                              int32_t* n_chunked, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    if (!c->comm) throw std::invalid_argument("no communicator (nsb_comm_init)");
    if (global_bit < 0 || (1 << global_bit) >= c->nranks || local_q < 0 || local_q >= c->n)
      throw std::invalid_argument("bad shard swap qubits");
    if (!P || P->ctx != c) throw std::invalid_argument("plan belongs to another context");
    if (P->n != c->n) throw std::invalid_argument("plan was built for another qubit count");
    if (seg < 0 || seg >= static_cast<int64_t>(P->host.items.size()))
      throw std::invalid_argument("item index out of range");
    const int partner = c->rank ^ (1 << global_bit);
    if (!c->peers[partner]) throw std::invalid_argument("peer shard not mapped (nsb_shard_open_peers)");
    NSB_CUDA(cudaSetDevice(c->device));
    const StreamMem& sm = stream_mem();
    uint64_t cm = 0;
    int np = chunk_prefix(P->host, seg, local_q, std::min(chunk_bits, 4), &cm);
    // The copy engines move about 1.5 G rows per second: regions of short runs
    // (a low chunk or swap qubit) would take them longer than the SM swap
    // kernel takes the whole exchange (tools/r2_ce_dbg.sh: 512-byte runs, local
    // copies at 0.7 TB/s).  Those swaps run on the SMs, not overlapped.
    static const int min_run_log2 = [] {
      const char* e = std::getenv("NSB_CE_MIN_RUN");
      return e ? std::atoi(e) : 12;
    }();
    if (np > 0 && __builtin_ctzll(cm | (uint64_t(1) << local_q)) < min_run_log2) np = 0;
    if (n_chunked) *n_chunked = np;
    const Item& it = P->host.items[static_cast<size_t>(seg)];
    const int b = (c->rank >> global_bit) & 1;
    const uint64_t half = c->n_amps >> 1;
    auto sm_swap_then_item = [&]() {
      const int clog = static_cast<int>(std::min<uint64_t>(16, c->n - 1));
      comm_barrier(c);
      dev::k_shard_swap_p2p<<<static_cast<unsigned>(c->sm_count * 4), 256, 0, c->stream>>>(
          c->amps.ptr, c->peers[partner], half, local_q, 1 - b, b, b, clog);
      NSB_CUDA(cudaGetLastError());
      comm_barrier(c);
      run_item(c, P, it);
      NSB_CUDA(cudaStreamSynchronize(c->stream));
      if (n_chunked) *n_chunked = 0;
    };
    if (np == 0) {  // nothing chunkable (or short runs): the SM swap, then the item
      sm_swap_then_item();
      return;
    }
    if (!c->xfer) NSB_CUDA(cudaStreamCreateWithFlags(&c->xfer, cudaStreamNonBlocking));
    if (!c->ev_ov0) NSB_CUDA(cudaEventCreateWithFlags(&c->ev_ov0, cudaEventDisableTiming));
    if (!c->ev_ov1) NSB_CUDA(cudaEventCreateWithFlags(&c->ev_ov1, cudaEventDisableTiming));
    const int cb = __builtin_popcountll(cm);
    const int n_ch = 1 << cb;
    for (int ch = 0; ch < n_ch; ++ch)
      if (!c->ev_chunk[ch]) NSB_CUDA(cudaEventCreateWithFlags(&c->ev_chunk[ch], cudaEventDisableTiming));
    if (!c->xfer2) NSB_CUDA(cudaStreamCreateWithFlags(&c->xfer2, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      if (!c->ev_pulled[i]) NSB_CUDA(cudaEventCreateWithFlags(&c->ev_pulled[i], cudaEventDisableTiming));
      if (!c->ev_local[i]) NSB_CUDA(cudaEventCreateWithFlags(&c->ev_local[i], cudaEventDisableTiming));
    }
    // The exchanged region of chunk ch: bits F = cm + local_q fixed (mine:
    // local_q = 1 - b, the partner's: local_q = b), the other bits free,
    // paired element for element in one fixed order.  It is a set of runs of
    // 2^p1 amplitudes (p1 = the lowest fixed bit); the free bits above p1 form
    // groups of consecutive bits between fixed ones.  One 3-D copy covers the
    // run, the group right above it as height (rows at twice the run's pitch:
    // the copy engine reads every other run of one contiguous span) and the
    // largest group above that as depth; a host loop enumerates the other
    // groups' bits; copies are split into staging blocks of at most a slot.
    const uint64_t F = cm | (uint64_t(1) << local_q);
    const int p1 = __builtin_ctzll(F);
    struct Group {
      int lo, bits;
    };
    std::vector<Group> groups;
    for (int q = p1 + 1; q < c->n;) {
      if (F >> q & 1) {
        ++q;
        continue;
      }
      int e = q;
      while (e < c->n && !(F >> e & 1)) ++e;
      groups.push_back({q, e - q});
      q = e;
    }
    static int max_pitch = 0;
    if (!max_pitch) NSB_CUDA(cudaDeviceGetAttribute(&max_pitch, cudaDevAttrMaxPitch, c->device));
    int gh = -1, gd = -1;  // height and depth groups
    if (!groups.empty() && (uint64_t(sizeof(double2)) << groups[0].lo) <= uint64_t(max_pitch)) gh = 0;
    for (int i = 0; i < static_cast<int>(groups.size()); ++i)
      if (i != gh && groups[i].lo > (gh >= 0 ? groups[gh].lo : -1) &&
          (gd < 0 || groups[i].bits > groups[gd].bits))
        gd = i;
    uint64_t other = 0;  // free bits enumerated on the host
    for (int i = 0; i < static_cast<int>(groups.size()); ++i)
      if (i != gh && i != gd)
        for (int t = 0; t < groups[i].bits; ++t) other |= uint64_t(1) << (groups[i].lo + t);
    const uint64_t run = uint64_t(1) << p1;
    const uint64_t H = gh >= 0 ? uint64_t(1) << groups[gh].bits : 1;
    const uint64_t D = gd >= 0 ? uint64_t(1) << groups[gd].bits : 1;
    // strides (log2 amplitudes); no height group: one run per row (pitch = width)
    const int hs = gh >= 0 ? groups[gh].lo : p1;
    const int ds = gd >= 0 ? groups[gd].lo : hs + (gh >= 0 ? groups[gh].bits : 0);
    const uint64_t n_outer = uint64_t(1) << __builtin_popcountll(other);
    if (n_outer > 4096) {  // too many copies to enqueue (both partners decide alike)
      sm_swap_then_item();
      return;
    }
    const uint64_t cap = std::max<uint64_t>(run, (stage_bytes > 0 ? static_cast<uint64_t>(stage_bytes)
                                                                  : (uint64_t(4) << 30)) / sizeof(double2));
    const uint64_t chunk_amps = half >> cb;
    const uint64_t slot = std::min<uint64_t>(chunk_amps, cap);
    if (c->ce_stage.count < 2 * slot) {
      c->ce_stage.release();
      c->ce_stage.alloc(2 * slot);
    }
    // one chunk's pieces: (outer value, depth range, height range), each a 3-D
    // copy of whole runs, in the fixed element order
    struct Piece {
      uint64_t outer, d0, nd, h0, nh;
    };
    std::vector<Piece> pieces;
    const uint64_t slice = H * run;  // amplitudes per depth slice
    for (uint64_t o = 0; o < n_outer; ++o) {
      if (slice <= slot) {
        const uint64_t per = slot / slice;  // depth slices per piece
        for (uint64_t d0 = 0; d0 < D; d0 += per) pieces.push_back({o, d0, std::min(per, D - d0), 0, H});
      } else {
        const uint64_t per = std::max<uint64_t>(1, slot / run);  // rows per piece
        for (uint64_t d0 = 0; d0 < D; ++d0)
          for (uint64_t h0 = 0; h0 < H; h0 += per) pieces.push_back({o, d0, 1, h0, std::min(per, H - h0)});
      }
    }
    {  // staging blocks per swap (one flag word each): else the SM swap
      int blocks = 0;
      for (size_t p0 = 0; p0 < pieces.size(); ++blocks) {
        uint64_t used = 0;
        size_t q = p0;
        for (; q < pieces.size(); ++q) {
          const uint64_t amps = pieces[q].nd * pieces[q].nh * run;
          if (used + amps > slot) break;
          used += amps;
        }
        p0 = q;
      }
      if (blocks * n_ch > dev::kShardFlagWords) {
        sm_swap_then_item();
        return;
      }
    }
    auto copy3d_on = [&](cudaStream_t strm, double2* dst, bool dst_dense, const double2* src,
                         bool src_dense, const Piece& pc, cudaMemcpyKind kind) {
      if (run >= (uint64_t(1) << 20)) {  // long runs: plain 1-D copies, run by run
        const uint64_t sh = uint64_t(1) << hs, sd = uint64_t(1) << ds;
        uint64_t off = 0;
        for (uint64_t d = 0; d < pc.nd; ++d)
          for (uint64_t r = 0; r < pc.nh; ++r, off += run) {
            const uint64_t strided = d * sd + r * sh;
            NSB_CUDA(cudaMemcpyAsync(dst + (dst_dense ? off : strided), src + (src_dense ? off : strided),
                                     run * sizeof(double2), kind, strm));
          }
        return;
      }
      cudaMemcpy3DParms m{};
      const size_t wb = run * sizeof(double2);
      const size_t sp = size_t(sizeof(double2)) << hs;
      const size_t sy = size_t(1) << (ds - hs);
      m.srcPtr = src_dense ? make_cudaPitchedPtr(const_cast<double2*>(src), wb, wb, pc.nh)
                           : make_cudaPitchedPtr(const_cast<double2*>(src), sp, wb, sy);
      m.dstPtr = dst_dense ? make_cudaPitchedPtr(dst, wb, wb, pc.nh) : make_cudaPitchedPtr(dst, sp, wb, sy);
      m.extent = make_cudaExtent(wb, pc.nh, pc.nd);
      m.kind = kind;
      NSB_CUDA(cudaMemcpy3DAsync(&m, strm));
    };
    auto copy3d = [&](double2* dst, bool dst_dense, const double2* src, bool src_dense,
                      const Piece& pc, cudaMemcpyKind kind) {
      copy3d_on(c->xfer, dst, dst_dense, src, src_dense, pc, kind);
    };
    auto region_off = [&](uint64_t fix, const Piece& pc) {
      return fix | deposit_bits(pc.outer, other) | (pc.d0 << ds) | (pc.h0 << hs);
    };
    // timing experiments only (wrong states): 2 = no chunked passes, 4 = no
    // flag words, 8 = no local copies, 16 = no peer pulls
    static const int ov_debug = [] {
      const char* e = std::getenv("NSB_OVERLAP_DEBUG");
      return e ? std::atoi(e) : 0;
    }();
    const unsigned epoch = ++c->swap_epoch;
    unsigned* f_mine = shard_flags(c->amps.ptr, c->n_amps);
    unsigned* f_peer = shard_flags(c->peers[partner], c->n_amps);
    comm_barrier(c);  // both shards are final before either is touched
    NSB_CUDA(cudaEventRecord(c->ev_ov0, c->stream));
    NSB_CUDA(cudaStreamWaitEvent(c->xfer, c->ev_ov0, 0));
    NSB_CUDA(cudaStreamWaitEvent(c->xfer2, c->ev_ov0, 0));
    // per block k: pulls on xfer, then the flag word to the partner; local
    // copies on xfer2 once the pull landed and the partner's word arrived, so
    // block k's local copy (HBM) runs beside block k+1's pull (NVLink); a
    // slot is pulled into again only after its local copy (ev_local)
    int k = 0;  // staging block: flag word, slot k & 1
    for (int ch = 0; ch < n_ch; ++ch) {
      const uint64_t cv = deposit_bits(static_cast<uint64_t>(ch), cm);
      const uint64_t fix_mine = cv | (uint64_t(1 - b) << local_q);
      const uint64_t fix_peer = cv | (uint64_t(b) << local_q);
      for (size_t p0 = 0; p0 < pieces.size(); ++k) {
        if (k >= dev::kShardFlagWords) throw std::invalid_argument("too many swap blocks");
        double2* sbuf = c->ce_stage.ptr + static_cast<uint64_t>(k & 1) * slot;
        if (k >= 2) NSB_CUDA(cudaStreamWaitEvent(c->xfer, c->ev_local[k & 1], 0));
        size_t p = p0;
        uint64_t used = 0;
        for (; p < pieces.size(); ++p) {  // pull: the partner's half into the slot
          const uint64_t amps = pieces[p].nd * pieces[p].nh * run;
          if (used + amps > slot) break;
          if (!(ov_debug & 16))
            copy3d(sbuf + used, true, c->peers[partner] + region_off(fix_peer, pieces[p]), false,
                   pieces[p], cudaMemcpyDefault);
          used += amps;
        }
        if (!(ov_debug & 4)) sm.write(c->xfer, f_peer + k, epoch);  // "your block k is read"
        NSB_CUDA(cudaEventRecord(c->ev_pulled[k & 1], c->xfer));
        NSB_CUDA(cudaStreamWaitEvent(c->xfer2, c->ev_pulled[k & 1], 0));
        if (!(ov_debug & 4)) sm.wait(c->xfer2, f_mine + k, epoch);  // ... and mine
        used = 0;
        for (size_t q = p0; q < p && !(ov_debug & 8); ++q) {  // the slot into my half
          copy3d_on(c->xfer2, c->amps.ptr + region_off(fix_mine, pieces[q]), false, sbuf + used, true,
                    pieces[q], cudaMemcpyDeviceToDevice);
          used += pieces[q].nd * pieces[q].nh * run;
        }
        NSB_CUDA(cudaEventRecord(c->ev_local[k & 1], c->xfer2));
        p0 = p;
      }
      NSB_CUDA(cudaEventRecord(c->ev_chunk[ch], c->xfer2));
    }
    for (int ch = 0; ch < n_ch; ++ch) {
      NSB_CUDA(cudaStreamWaitEvent(c->stream, c->ev_chunk[ch], 0));
      if (!(ov_debug & 2))
        launch_blocked(c, P, P->passes.ptr, it.pass_begin, it.pass_begin + np, -1.0, 0, cm,
                       deposit_bits(static_cast<uint64_t>(ch), cm));
    }
    if (it.pass_begin + np < it.pass_end)
      launch_blocked(c, P, P->passes.ptr, it.pass_begin + np, it.pass_end, -1.0);
    NSB_CUDA(cudaEventRecord(c->ev_ov1, c->xfer));
    NSB_CUDA(cudaStreamWaitEvent(c->stream, c->ev_ov1, 0));
    NSB_CUDA(cudaEventRecord(c->ev_ov1, c->xfer2));
    NSB_CUDA(cudaStreamWaitEvent(c->stream, c->ev_ov1, 0));
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int nsb_shard_reset(nsb_ctx* c, nsb_status* st) {
  return guarded(st, [&] {
    require_state(c);
    NSB_CUDA(cudaSetDevice(c->device));
    if (c->rank == 0) {
      dev::k_vacuum<<<grid_for(c->n_amps, 256, c), 256, 0, c->stream>>>(c->amps.ptr, c->n_amps);
      NSB_CUDA(cudaGetLastError());
    } else {
      NSB_CUDA(cudaMemsetAsync(c->amps.ptr, 0, c->n_amps * sizeof(double2), c->stream));
    }
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int nsb_shard_allgather(nsb_ctx* c, const double* in, int32_t count, double* out,
                        nsb_status* st) {
  return guarded(st, [&] {
    if (!c || !c->comm) throw std::invalid_argument("no communicator (nsb_comm_init)");
    if (!in || !out || count < 1) throw std::invalid_argument("bad gather size");
    NSB_CUDA(cudaSetDevice(c->device));
    const size_t need = size_t(count) * (c->nranks + 1);
    DevBuf<double> big;  // large gathers (sampled indices): a temporary buffer
    double* d_in = c->scratch.ptr + 2 * dev::kReduceBlocks + 8;
    if (count > 64 || c->scratch.count < size_t(2 * dev::kReduceBlocks + 8) + need) {
      big.alloc(need);
      d_in = big.ptr;
    }
    double* d_out = d_in + count;
    NSB_CUDA(cudaMemcpyAsync(d_in, in, count * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    NSB_NCCL(shard_nccl().all_gather(d_in, d_out, count, ncclFloat64,
                                     static_cast<ncclComm_t>(c->comm), c->stream));
    NSB_CUDA(cudaMemcpyAsync(out, d_out, size_t(count) * c->nranks * sizeof(double),
                             cudaMemcpyDeviceToHost, c->stream));
    NSB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"
