// Host-side plan container (see planner.cpp for the scheduling algorithm).
#pragma once

#include <cstring>
#include <unordered_map>
#include <vector>

#include "host_common.h"
#include "planner.h"

namespace nsb {

struct Key {
  std::vector<uint64_t> bits;
  bool operator==(const Key& o) const { return bits == o.bits; }
};
struct KeyHash {
  size_t operator()(const Key& k) const {
    uint64_t h = 1469598103934665603ull;
    for (uint64_t b : k.bits) {
      h ^= b;
      h *= 1099511628211ull;
      h ^= h >> 29;
    }
    return static_cast<size_t>(h);
  }
};

struct PoolBuilder {
  std::vector<double>& pool;
  std::unordered_map<Key, int32_t, KeyHash> seen;
  int32_t add(const double* v, int n_complex) {
    Key k;
    k.bits.resize(2 * n_complex + 1);
    std::memcpy(k.bits.data(), v, sizeof(double) * 2 * n_complex);
    k.bits.back() = static_cast<uint64_t>(n_complex);
    auto it = seen.find(k);
    if (it != seen.end()) return it->second;
    const int32_t off = static_cast<int32_t>(pool.size() / 2);
    pool.insert(pool.end(), v, v + 2 * n_complex);
    seen.emplace(std::move(k), off);
    return off;
  }
};

struct PhysGate {
  uint8_t cls = 0;
  int nq = 0;
  uint64_t ma = 0, mb = 0;  // physical XOR masks of slot 0 / slot 1
  uint64_t ra = 0, rb = 0;  // dual rows: logical slot bits as physical parities
  int32_t mat = 0;          // packed payload: offset into HostPlan::packed_all
  int32_t n_mat = 0;        // complex elements
  uint16_t cols = 0;
};

struct Item {
  enum Kind { kGates, kDense, kMeasure, kReset } kind;
  int32_t pass_begin = 0, pass_end = 0;  // kGates: passes[pass_begin, pass_end)
  int32_t k = 0, qs[5] = {0, 0, 0, 0, 0};
  int64_t mat_off = 0;                   // kDense: offset (complex) into dense_mats
  int32_t qubit = -1, step = -1;         // kMeasure / kReset
};

struct HostPlan {
  int n_qubits = 0;
  int tile_qubits = 0;
  int low_qubits = kLowQubits;  // qubits 0..low-1 are in every pass's tile
  bool blocked = false;   // blocked pass kernel (n >= 6); else per-op kernels
  bool mma_ok = false;    // whole MMA run fits one cooperative launch
  int64_t n_gates = 0, n_measures = 0;
  int64_t n_frame_gates = 0;  // exact CX/SWAP absorbed by the relabeling frame
  int64_t n_flush_gates = 0;  // physical CX emitted to flush the frame
  int64_t n_frame_flushes = 0;  // flushes forced by a wide support
  int64_t n_folded_gates = 0;   // physical CXs folded into read maps
  int64_t n_ops = 0;            // gate ops executed on the device (all groups)
  int64_t n_warp_syncs = 0;     // sweeps followed by __syncwarp instead of a CTA barrier
  int64_t n_fused_group_ops = 0;  // gate ops removed by group fusion (fuse_group)
  int64_t n_axis_swaps = 0;       // register-axis exchanges of four-axis groups
  bool fuse_groups = true;      // NSB_NO_GROUP_FUSION=1 turns group fusion off
  // tiles move by TMA (planner.h "TMA tiles"): the first group of every pass
  // loads under swz_tma, the last one stores under it
  bool tma = false;
  bool allow_tma = true;  // set by the caller: the device runs the TMA kernel
  // octets per thread of the blocked kernel this plan is laid out for (set by
  // the caller, plan_octets): 2 (128 threads) or 1 (256 threads: small states)
  int octets = kOctets;
  // Gates within rounding of a scalar identity s I (e.g. the fused H.H / S.Sdg
  // products between consecutive JW terms, 1 + 2^-52 on the diagonal) are not
  // executed.  Their scalar is kept: the reference's state carries the product
  // of the |s|^2 in its norm until the next measurement renormalises it, so
  // each reported P(|0>) is multiplied by that product (p0_scale; a real
  // positive s makes the post-collapse states agree exactly).  What is not
  // compensated -- the residuals ||U - s I||_F, the phases |s/|s| - 1| and the
  // norm drift after the last measurement -- is summed in identity_error and
  // kept within identity_budget: for unitaries ||U_N..U_1 - U'_N..U'_1|| <=
  // sum ||U_i - U'_i||, so the state moves by at most identity_error relative
  // L2 (default budget 3e-11, under a third of the 1e-10 parity bound;
  // NSB_IDENTITY_BUDGET=0 executes every gate).
  double identity_budget = -1.0;  // < 0: the default / environment
  int64_t n_identity_gates = 0;
  double identity_error = 0.0;
  std::vector<double> p0_scale;   // per assertion step: product of |s|^2 since the last one
  double tail_scale2 = 1.0;       // product of |s|^2 after the last measurement
  double tail_error = 0.0;        // sum of | |s| - 1 | after the last measurement
  double tail_error_total = 0.0;  // its final value (parts of a parallel build)
  int64_t flops = 0;
  int64_t class_count[kNumClasses] = {};

  std::vector<Item> items;
  std::vector<PassDesc> passes;      // plain gate passes (items reference ranges)
  std::vector<PassDesc> mma_passes;  // whole-circuit MMA program
  std::vector<GroupDesc> groups;    // octet sweeps
  std::vector<GateOp> gate_ops;     // their gates
  std::vector<double> matrices;      // packed payloads, one block per pass
  std::vector<double> packed_all;    // packed payloads of the current run
  std::vector<double> dense_mats;    // k-qubit / unblocked matrices (full)
  std::vector<int32_t> items_flat;   // nsb_host_plan_view export

  // workers: persistent CTAs of the pass kernel (tile-size choice)
  void build(const nsb_op* ops, int64_t n_ops, const double* params, const double* payloads,
             int n, int workers);
  // one gate run between two markers (no MEASURE / RESET inside): the unit of
  // the parallel build and of streamed MMA runs (nsb_run_mma_streamed)
  void build_segment(const nsb_op* ops, int64_t n_ops, const double* params,
                     const double* payloads, int n, int workers) {
    build_serial(ops, n_ops, params, payloads, n, workers);
  }

 private:
  void build_serial(const nsb_op* ops, int64_t n_ops, const double* params,
                    const double* payloads, int n, int workers);
  void schedule_run(std::vector<PhysGate>& run, int k);
  void build_mma();
};

// The TMA copy layout of a pass's tile (planner.h "TMA tiles", dev::TmaPass):
// dim 0 = qubits 0..2; dims 1.. = the (up to four) longest runs of consecutive
// tile qubits, listed in a chosen order -- the order of their bits in shared
// memory -- each dim's coordinate spanning its run and the out-of-tile qubits
// above it (the lowest one starting at qubit 3: a gap of <= 3 qubits below its
// run is a traversal stride, a longer one takes a dim with a box of one);
// the other runs are `left`, coordinate bits of the dim below them, one copy
// per value, their bits on top of the copy layout.  perm: tile-local bit ->
// bit of the copy layout.  `order` < n_orders picks the order of the run dims.
// False: the pass's tile is not TMA-shaped (k < kTileQubitsMax, qubits 0..2
// not all tiled, n > kTmaMaxQubits).
struct TmaLayout {
  int rank = 0;                      // dims, dim 0 included
  int start[5] = {0}, ebits[5] = {0}, len[5] = {0}, gap[5] = {0};
  uint64_t left = 0;
  int8_t perm[16] = {0};
  int n_orders = 0;
};
bool tma_layout(const PassDesc& P, int n, int order, TmaLayout& L);

void plan_info(const HostPlan& H, nsb_plan_info* info);
// the thread layout for an n-qubit state: one octet per thread up to
// kSmallStateQubits (more warps on the few tiles of a small state; filter
// circuits, tools/oct_sweep.py: 16 q 4.78 vs 4.91 ms, 18 q 6.51 vs 8.15 ms,
// 19 q 8.74 vs 8.62 ms, 21 q 30.8 vs 29.5 ms), two above; NSB_PLAN_OCTETS
// overrides
constexpr int kSmallStateQubits = 18;
int plan_octets(int n);
inline int plan_thread_bits(int octets) { return octets == 2 ? 7 : 8; }
double default_identity_budget_value();  // NSB_IDENTITY_BUDGET or 3e-11
// passes of item `item` runnable chunk by chunk over the qubits *cmask (planner.cpp)
int chunk_prefix(const HostPlan& H, int64_t item, int avoid_q, int want_bits, uint64_t* cmask);

}  // namespace nsb
