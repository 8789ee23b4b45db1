// Device program produced by the host planner (planner.cpp) and executed by
// the blocked gate-stream kernel (device.cu).
//
// Two ideas carry the design:
//  1. Relabeling frame.  Exact CX and SWAP payloads are permutations that are
//     linear over GF(2) on basis indices.  The planner does not move data for
//     them: it keeps a linear map M with psi(v) = phi(M v) between the
//     logical state psi and the physical array phi, and rewrites every later
//     gate on logical qubit j to act along the physical XOR mask M e_j.  At
//     every measurement / reset / dense k-qubit gate and at the end of the
//     program the frame is flushed back to the identity with a short
//     sequence of physical CX gates (exact data movement), so everything
//     outside a gate run sees the reference's ordinary little-endian state.
//  2. Passes.  The state is cut into 2^(n-k) tiles of 2^k amplitudes over a
//     physical tile qubit set T (|T| = k <= kTileQubitsMax, always holding
//     qubits 0..2 so global accesses are whole 128-byte lines).  A pass
//     streams every tile through shared memory once and applies its gates as
//     octet sweeps (below): each sweep moves the tile through registers once
//     and applies a group of up to three-axis gates there.  Global traffic is
//     32 B per amplitude per pass.
// Mid-circuit measurements end a pass: the pass epilogue writes per-CTA
// partial sums of |a|^2 over the |0> half, the grid agrees on p0 after the
// barrier, and the next pass's prologue applies the collapse.
#pragma once

#include <cstdint>

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

namespace nsb {

#ifndef NSB_TILE_MAX
#define NSB_TILE_MAX 11
#endif
constexpr int kTileQubitsMax = NSB_TILE_MAX;     // 2048 amplitudes = 32 KiB per buffer
constexpr int kTileAmpsMax = 1 << kTileQubitsMax;
#ifndef NSB_OCTETS
#define NSB_OCTETS 2
#endif
constexpr int kOctets = NSB_OCTETS;              // octets per thread per sweep (1 or 2)
#ifndef NSB_THREAD_BITS  // build variants: 12-qubit tiles take 256 threads (8 warps, one CTA per SM)
#define NSB_THREAD_BITS (kOctets == 2 ? 7 : 8)
#endif
constexpr int kThreadBits = NSB_THREAD_BITS;
constexpr int kPassThreads = 1 << kThreadBits;  // 4 (8) warps per CTA, two CTAs per SM
constexpr int kCtasPerSm = kPassThreads > 128 ? 1 : 2;
constexpr int kIndexBits = kThreadBits + (kOctets == 2 ? 1 : 0);  // octet-index bits of a batch
constexpr int kIndexSlots = kIndexBits > 8 ? 10 : 8;  // GroupDesc offset slots
static_assert(kIndexBits <= kIndexSlots, "GroupDesc index-bit offsets");
constexpr int kLowQubits = 3;                    // always-tiled qubits 0..2 (128 B runs)
// States up to this many qubits stay L2-resident inside a launch: their
// tiles need not hold qubits 0..2 (sector efficiency matters less than the
// extra free tile qubit slots, which cut the pass count by a third).
constexpr int kL2ResidentQubits = 22;
// ... but qubits 0, 1 (64-byte runs: half the L2 requests of 32-byte runs)
// still pay: deep21 measured 862 ms with 2, 878 ms with 1, 924 ms with 3.
constexpr int kLowQubitsL2 = 2;
constexpr int kMaxQubits = 40;
// TMA tiles.  When every tile holds qubits 0..2 at full size (the HBM
// policy), a tile moves between HBM and shared memory by cp.async.bulk.tensor:
// the tile's qubit runs are the dims of a <= 5-D tensor map (per pass; qubits
// 0..2 and re/im the 128-byte inner dim, runs beyond five dims as separate
// copies), landing under the hardware's 128-byte swizzle
//   swz_tma(l) = l ^ ((l >> 3) & 7)      (16-byte slots, 1024-byte aligned)
// instead of swz.  Both are linear over XOR, so only the pass edges change:
// the FIRST group of a pass loads with swz_tma offsets, the LAST one stores
// with them (the TMA store reads that layout); the sweeps in between keep swz.
// Coordinates are int32 and a dim spans at most 2^31 values: n <= 34.
// Per pass, only where it pays: a tile of few copies (a copy costs the TMA
// unit a fixed few hundred cycles) whose first / last sweep keeps all eight
// 16-byte bank groups under swz_tma (the hardware swizzle mixes slot bits
// 3..5 only, so axes on tile bits j and j + 3 alias); else cp.async and swz.
constexpr int kTmaMaxQubits = 34;
constexpr int kTmaMaxCopies = 2;

// Payload classes, chosen by exact-zero structure (skipping an exact zero
// term is bit-identical to multiplying by it).
enum GateClass : uint8_t {
  kDense1 = 0,    // 2x2                                  (4 complex values)
  kDiag1 = 1,     // 2x2 diagonal                         (2)
  kDense2 = 2,    // 4x4 dense                            (16)
  kSparse2 = 3,   // 4x4, <= 2 nonzeros per row, any cols (8 + column codes)
  kMono2 = 4,     // 4x4, <= 1 nonzero per row            (4 + column codes)
  kDiag2 = 5,     // 4x4 diagonal                         (4)
  kCX01 = 6,      // exact CX, slot 0 controls slot 1: swaps members 1,3  (0)
  kCX10 = 7,      // exact CX, slot 1 controls slot 0: swaps members 2,3  (0)
  kPairQ = 8,     // 2x2 blocks on members (0,2) and (1,3)                (8)
  kPairP = 9,     // 2x2 blocks on members (0,1) and (2,3)                (8)
  kPairX = 10,    // 2x2 blocks on members (0,3) and (1,2)                (8)
  kSwap = 11,     // exact SWAP: swaps members 1,2                        (0)
  kPermute = 12,  // identity sweep that only applies its read map      (0)
  kPairQr = 13,   // kPairQ with real entries (imaginary parts exactly 0)  (8)
  kPairPr = 14,   // kPairP, real                                          (8)
  kPairXr = 15,   // kPairX, real                                          (8)
  kNumClasses = 16
};

// A gate on logical qubits (a, b) acts on physical cosets of span{ma, mb}
// (ma = M e_a, mb = M e_b).  The coset member whose LOGICAL bits a, b are
// zero is found with the dual rows ra, rb of M^-1 (logical bit a of physical
// index p = parity(p & ra)).
//
// Octet sweeps.  Consecutive gates of a pass that together touch at most
// three logical axes (m_i, r_i) -- tile-local physical masks with their dual
// rows, r_i(m_j) = delta_ij -- form a GROUP, executed as ONE shared-memory
// sweep: every thread loads one octet {A ^ c0 m0 ^ c1 m1 ^ c2 m2} into eight
// registers, applies all of the group's gates there (register index c = the
// octet's logical bits, fixed at compile time per axis pattern) and stores
// it back.  The octet bases A range over C = ker(r_0) ^ ker(r_1) ^ ker(r_2)
// inside the tile, so the logical bits of an octet member never depend on A
// -- only on the tile (out-of-tile parts of the rows, folded into A per tile
// as the parity bits kappa).  Groups with fewer than three axes are padded
// with a free tile axis.  The planner orders C's basis so the first three
// thread bits hit different 16-byte bank groups under the shared-memory
// swizzle swz(l) = l ^ ((l>>3 ^ l>>6 ^ l>>9) & 7); because swz and all maps
// are linear over XOR, the planner stores swizzled per-bit offsets and the
// kernel only XORs.
//
// Read maps: physical permutations (the CX gates that shrink the relabeling
// frame) are not executed as sweeps of their own.  The group that follows
// them in a pass reads its octets through their composition R (a linear map
// of tile-local indices) and writes in place order, so the r* fields hold
// the same offsets mapped through R (equal to the plain ones when R = I).
//
// Four-axis groups (full 11-qubit tiles): a thread's two octets are the two
// values of a FOURTH logical axis -- its 16 registers are the coset of a
// four-dimensional subspace -- so a run of gates touching up to four axes is
// one sweep.  Gates still address the octet positions 0..2 only: before a
// gate that needs the fourth axis, a register-axis exchange op (kPermute with
// pattern kPatQ0..2, straight register moves, no arithmetic) swaps it with a
// position the gate does not use.  Loads place axis i at position i (axis 3
// on the octet index); stores use the final placement `perm`.  The
// out-of-tile parity bits kappa are therefore taken per axis for the loads
// and permuted for the stores.
struct GroupDesc {        // 80 bytes
  uint16_t am[3];         // swizzled masks of the axes at positions 0..2 after the ops (store)
  uint16_t ram[3];        // axes 0..2 through the read map R (load side)
  uint16_t tcol[kIndexSlots];   // swizzled offsets of octet-index bits (store side):
                                // thread bits, then the octet index (a fourth axis, or a free vector)
  uint16_t rtcol[kIndexSlots];  // load side
  uint8_t op_begin;       // first GateOp (relative to the pass's op_begin)
  uint8_t n_ops_sync;     // bits 0..6: gate ops (0: a pure read-map sweep); bit 7: CTA
                          // barrier after this sweep (else warp-local, __syncwarp)
  uint16_t kmat;          // store parity map: bits 4j..4j+3 = the load rows whose sum
                          // is the final row at position j
  uint64_t r_out[4];      // out-of-tile parts of the load basis rows (position 3: 0 if none)
  __host__ __device__ int n_ops() const { return n_ops_sync & 127; }
  __host__ __device__ bool sync() const { return n_ops_sync >> 7; }
};
static_assert(sizeof(GroupDesc) == (kIndexSlots > 8 ? 88 : 80), "GroupDesc layout");

// One gate of a group: class, axis pattern, payload.  Two-qubit gates are
// stored with slot 0 on the lower axis (the planner exchanges the slots of
// the payload when needed).
enum AxisPattern : uint8_t {
  kPat01 = 0, kPat02 = 1, kPat12 = 2,  // 2q: (slot0 axis, slot1 axis)
  kPat0 = 3, kPat1 = 4, kPat2 = 5,     // 1q: axis
  // Whole-octet ops, the product of a group's gates (planner group fusion):
  // kPatT0..T2 with class kDense1 = a 2x2 on axis t whose matrix depends on
  // the other two axes (four blocks, block index = their bits, lower axis
  // first; 16 complex values); kPatAll with class kDiag1 = 8x8 diagonal (8).
  kPatT0 = 6, kPatT1 = 7, kPatT2 = 8, kPatAll = 9,
  // kPatD01/D02/D12 with class kDense2: a 4x4 on the two axes (slot 0 the
  // lower) with one block per value of the third axis (32 complex values)
  kPatD01 = 10, kPatD02 = 11, kPatD12 = 12,
  // kPatQ0..Q2 with class kPermute: exchange register position 0..2 with the
  // octet index (four-axis groups; no matrix)
  kPatQ0 = 13, kPatQ1 = 14, kPatQ2 = 15
};
// Dense dispatch keys (GateOp::kind): consecutive small integers, so the
// kernel's switch compiles to one indirect branch through a jump table
// instead of a compare-and-branch tree over pat * 16 + cls.
#ifndef NSB_SPARSE_KINDS
__host__ __device__ constexpr int op_kind(int pat, int cls) {
  // 2q patterns: 13 classes each (kPermute and the 1q classes never occur there)
  return pat <= kPat12 ? pat * 13 + (cls < kPermute ? cls - kDense2 : cls - kDense2 - 1)
       : pat <= kPat2 ? 39 + (pat - kPat0) * 2 + (cls == kDiag1 ? 1 : 0)
       : pat <= kPatT2 ? 45 + (pat - kPatT0)
       : pat == kPatAll ? 48
       : pat <= kPatD12 ? 49 + (pat - kPatD01)
       : 67;
}
__host__ __device__ constexpr int reg_swap_kind(int p) { return 52 + p; }
__host__ __device__ constexpr int reg_cx_kind(int j, int k) { return 55 + j * 3 + (k < j ? k : k - 1); }
#else  // A/B: the sparse keys of round 1
__host__ __device__ constexpr int op_kind(int pat, int cls) { return pat * 16 + cls; }
__host__ __device__ constexpr int reg_swap_kind(int p) { return (kPatQ0 + p) * 16 + kPermute; }
__host__ __device__ constexpr int reg_cx_kind(int j, int k) { return 208 + j * 3 + (k < j ? k : k - 1); }
#endif

struct GateOp {           // 8 bytes
  int16_t mat;            // offset (complex elements) in the pass's matrix block
  uint8_t cls;            // GateClass
  uint8_t pat;            // AxisPattern
  uint16_t cols;          // kSparse2 / kMono2: 2-bit column codes
  uint8_t kind;           // pat * 16 + cls (the kernel's dispatch key)
  uint8_t pad;
};
static_assert(sizeof(GateOp) == 8, "GateOp layout");

// Per pass the kernel stages the group descriptors, gate ops and the pass's
// own block of packed matrices in shared memory (bounded by these limits).
constexpr int kMaxPassGates = 40;   // gates per pass (and groups per pass)
constexpr int kMaxPassOps = 80;     // gate ops per pass, register-axis exchanges included
constexpr int kMaxPassMats = 384;   // complex elements (6 KiB)

struct PassDesc {         // 112 bytes
  int32_t group_begin, group_end;
  int32_t op_begin, op_end;
  int32_t mat_begin, mat_count;  // the pass's matrix block (complex elements)
  int32_t k;              // tile qubits used (<= kTileQubitsMax)
  int32_t measure_q;      // epilogue: partial P(q=0) sums (-1: none)
  int32_t measure_slot;   // index into the probability record
  int32_t collapse_q;     // prologue: collapse onto q=0 using the carried p0
  int32_t collapse_slot;
  int32_t tma;            // 1: tiles move by TMA; the first group loads and the last
                          // group stores under swz_tma (TMA plans, "TMA tiles")
  int8_t tq[16];          // tile-local bit i -> physical qubit (ascending)
  int8_t oq[32];          // tile-index bit j -> physical qubit (ascending)
  int8_t tperm[16];       // TMA passes: tile-local bit i -> bit of the copy layout in
                          // shared memory (before swz_tma); the order of the map's dims
};
static_assert(sizeof(PassDesc) == 112, "PassDesc layout");

}  // namespace nsb
