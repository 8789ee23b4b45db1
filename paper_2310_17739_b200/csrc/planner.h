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
//     streams every tile through shared memory once and applies each of its
//     gates as one shared-memory sweep (pairs / quads along the gate's
//     tile-local XOR masks).  Global traffic is 32 B per amplitude per pass.
// Mid-circuit measurements end a pass: the pass epilogue writes per-CTA
// partial sums of |a|^2 over the |0> half, the grid agrees on p0 after the
// barrier, and the next pass's prologue applies the collapse.
#pragma once

#include <cstdint>

namespace nsb {

constexpr int kTileQubitsMax = 11;               // 2048 amplitudes = 32 KiB per buffer
constexpr int kTileAmpsMax = 1 << kTileQubitsMax;
constexpr int kThreadBits = 8;
constexpr int kPassThreads = 1 << kThreadBits;  // 8 warps per CTA, two CTAs per SM
constexpr int kLowQubits = 3;                    // always-tiled qubits 0..2 (128 B runs)
constexpr int kMaxQubits = 40;

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
  kNumClasses = 13
};

// A gate on logical qubits (a, b) acts on physical cosets of span{ma, mb}
// (ma = M e_a, mb = M e_b).  The coset member whose LOGICAL bits a, b are
// zero is found with the dual rows ra, rb of M^-1 (logical bit a of physical
// index p = parity(p & ra)).
//
// Work split: a sweep covers one batch (nb tiles stored back to back, batch
// index = tile-local index | tile-in-batch << k).  Item j (a quad or a pair)
// of the batch is j = t + T i (thread t, iteration i, T = kPassThreads); its
// representative is the batch index whose bits at the pivot positions are
// zero and whose other bits are j's bits, placed at the planner-chosen free
// positions pos[0..].  pos[0..2] are picked with distinct residues mod 3, so
// the 8 lanes of a quarter-warp hit 8 different 16-byte bank groups under
// the shared-memory swizzle swz(l) = l ^ ((l>>3 ^ l>>6 ^ l>>9) & 7).  Because
// swz, the placement and the parities are all linear over XOR, the planner
// stores swizzled per-bit offsets and parity masks and the kernel only XORs.
//
// Read maps: physical permutations (the CX gates that shrink the relabeling
// frame) are not executed as sweeps of their own.  A gate that follows them in
// a pass reads its members through their composition R (a linear map of
// tile-local indices) and writes in place order, so the r* fields hold the
// same offsets mapped through R (equal to the plain ones when R = I).
struct GateDesc {     // 96 bytes
  int32_t mat;        // offset (complex elements) in the pass's matrix block
  uint8_t cls;        // GateClass
  uint8_t nq;         // 1 or 2
  uint8_t tla, tlb;   // thread bits whose position carries a ra / rb bit
  uint16_t sa, sb;    // swizzled masks of slot 0 / slot 1
  uint16_t st1, st2, st3;   // swizzled offsets of iteration bits 0, 1, 2
  uint16_t cols;      // kSparse2 / kMono2: 2-bit column codes
  uint8_t spar;       // ra / rb parities of iteration bits (la1 lb1 la2 lb2 la3 lb3)
  uint8_t pad0[3];
  uint16_t tcol[8];   // swizzled offsets of thread bits 0..7
  uint16_t rsa, rsb, rst1, rst2, rst3;  // the same, read through R
  uint16_t rtcol[8];
  uint8_t pad1[14];
  uint64_t ra_out, rb_out;  // out-of-tile parts of the dual rows (physical bits)
};
static_assert(sizeof(GateDesc) == 96, "GateDesc layout");

// Per pass the kernel stages the gate descriptors and the pass's own block
// of packed matrices in shared memory (bounded by these limits).
constexpr int kMaxPassGates = 40;
constexpr int kMaxPassMats = 384;   // complex elements (6 KiB)

struct PassDesc {         // 112 bytes
  int32_t gate_begin, gate_end;
  int32_t mat_begin, mat_count;  // the pass's matrix block (complex elements)
  int32_t k;              // tile qubits used (<= kTileQubitsMax)
  int32_t measure_q;      // epilogue: partial P(q=0) sums (-1: none)
  int32_t measure_slot;   // index into the probability record
  int32_t collapse_q;     // prologue: collapse onto q=0 using the carried p0
  int32_t collapse_slot;
  int32_t pad[3];
  int8_t tq[16];          // tile-local bit i -> physical qubit (ascending)
  int8_t oq[48];          // tile-index bit j -> physical qubit (ascending)
};

}  // namespace nsb
