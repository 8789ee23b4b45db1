// Device program produced by the host planner (planner.cpp) and executed by
// the blocked gate-stream kernel (device.cu).
//
// Hierarchy:
//   pass   = one sweep of the state through shared memory: the state is cut
//            into 2^(n-k) tiles of 2^k amplitudes over a tile qubit set T
//            (|T| = k <= kTileQubits, always containing qubits 0..2 so every
//            global access is a full 128-byte line);
//   stage  = one shared-memory round trip inside a pass: every thread pulls a
//            16-amplitude group spanned by 4 tile-local qubits R into registers
//            and applies all stage gates (on qubits of R) there;
//   gate   = a 1q / 2q payload in group-local bit positions plus its sparsity
//            class (dense, <=2 nnz per row, monomial, diagonal).
// Mid-circuit measurements end a pass: the pass epilogue writes per-tile
// partial sums of |a|^2 over the |0> half, the grid agrees on p0 after the
// barrier, and the next pass's prologue applies the collapse.
#pragma once

#include <cstdint>

namespace nsb {

constexpr int kTileQubits = 12;                  // 4096 amplitudes = 64 KiB tile
constexpr int kTileAmps = 1 << kTileQubits;
constexpr int kGroupQubits = 4;                  // 16 amplitudes per thread
constexpr int kGroupAmps = 1 << kGroupQubits;
constexpr int kPassThreads = kTileAmps / kGroupAmps;  // 256
constexpr int kLowQubits = 3;                    // always-tiled qubits 0..2 (128 B runs)
constexpr int kMaxQubits = 40;

// Payload classes, chosen by exact-zero structure (skipping an exact zero
// term is bit-identical to multiplying by it).  Ordered cheapest first.
enum GateClass : uint8_t {
  kDense1 = 0,    // 2x2                                  (4 complex values)
  kDiag1 = 1,     // 2x2 diagonal                         (2)
  kDense2 = 2,    // 4x4 dense                            (16)
  kSparse2 = 3,   // 4x4, <= 2 nonzeros per row, any cols (8 + column codes)
  kMono2 = 4,     // 4x4, <= 1 nonzero per row            (4 + column codes)
  kDiag2 = 5,     // 4x4 diagonal                         (4)
  kCX01 = 6,      // exact CX, slot 0 controls slot 1: swaps |01>,|11>  (0)
  kCX10 = 7,      // exact CX, slot 1 controls slot 0: swaps |10>,|11>  (0)
  kPairQ = 8,     // 2x2 on slot 1 selected by slot 0: (0,2) and (1,3)  (8)
  kPairP = 9,     // 2x2 on slot 0 selected by slot 1: (0,1) and (2,3)  (8)
  kPairX = 10,    // 2x2 on the anti-diagonal pairs (0,3) and (1,2)     (8)
  kNumClasses = 11
};

struct GateDesc {     // 16 bytes
  int32_t mat;        // offset (complex elements) into the matrix pool
  uint8_t cls;        // GateClass
  uint8_t a, b;       // group bit of slot 0 / slot 1 (a < b after planning)
  uint8_t pad;
  uint16_t cols;      // sparse classes: 2 bits per (row, nz#) column index
  uint16_t pad2;
  int32_t pad3;
};

struct StageDesc {    // 16 bytes
  int32_t gate_begin, gate_end;
  int8_t rpos[kGroupQubits];                  // tile-local bit of group bit j
  uint32_t tperm;                             // packed 4-bit tile-local positions
};                                            // of thread bits 0..7 (non-R)

struct PassDesc {
  int32_t stage_begin, stage_end;
  int32_t k;              // tile qubits used (<= kTileQubits)
  int32_t measure_q;      // epilogue: partial P(q=0) sums (-1: none)
  int32_t measure_slot;   // index into the probability record
  int32_t collapse_q;     // prologue: collapse onto q=0 using record[collapse_slot]
  int32_t collapse_slot;
  int32_t pad;
  int8_t tq[16];          // tile-local bit i -> global qubit (ascending)
  int8_t oq[48];          // tile-index bit j -> global qubit (ascending)
};

}  // namespace nsb
