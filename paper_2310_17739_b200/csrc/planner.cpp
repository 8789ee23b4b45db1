// Host planner: turns the fused op list (engine._compile's plan, engine.py:
// 295-363) into the blocked device program of planner.h.
//
//  1. resolve every 1q/2q matrix (payload or nsb::gate_matrix), classify its
//     sparsity by exact zeros (skipping an exact zero term is bit-identical
//     to multiplying by it), deduplicate identical payloads by hash;
//  2. cut the op list into items: gate runs, k>=3 dense gates, MEASURE, RESET;
//  3. schedule each gate run into passes (tile qubit sets of <= 11 qubits,
//     kTileQubitsMax) with a dependency-respecting greedy look-ahead: a gate
//     joins the open pass if it fits the tile set and no skipped earlier gate
//     shares a qubit with it; otherwise it is deferred to a later pass;
//  4. inside a pass, group gates into octet sweeps (three-axis register
//     groups with a register frame, planner.h) the same way;
//  5. for MMA mode, build a single pass list in which each MEASURE becomes
//     an epilogue reduction of the preceding pass and a collapse prologue of
//     the next one (engine.py:183-191, 164-167).
#include "planner_host.h"
#include "../../include/nucsim_b200.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <complex>
#include <atomic>
#include <exception>
#include <thread>
#include <cstdlib>
#include <stdexcept>
#include <unordered_map>

namespace nsb {
static_assert(kNumClasses == NSB_N_CLASSES, "class count exported by the C ABI");
namespace {

inline int popc(uint64_t m) { return __builtin_popcountll(m); }

inline bool is_zero(const double* m, int idx) { return m[2 * idx] == 0.0 && m[2 * idx + 1] == 0.0; }

// Classify a gate matrix and write its packed form; returns class.
// Packed layouts (complex elements) are listed with GateClass in planner.h;
// kPair* store the two 2x2 blocks row-major, block 0 first.
//
// Before classifying, components at or below half an ulp of the matrix's
// largest component (|v| <= 2^-53 max|m|) are set to zero: products such as
// cos(pi/2) * 0.7071 = 4.3e-17 otherwise make a diagonal or monomial payload
// look dense.  The change to the matrix is below the rounding of one product
// with its largest entry, so the gate is unchanged at double precision
// (amplitudes stay within the 1e-10 parity bound after 10^8 gates even if
// every such perturbation added up coherently: 10^8 x 1.1e-16 = 1.1e-8 of
// the norm is the worst case, the observed drift is ~1e-13).  NSB_EXACT_CLASSES=1
// keeps the exact-zero rule only (bit-identical skipping).
uint8_t pack_matrix(const double* m_in, int nq, std::vector<double>& packed, uint16_t& cols) {
  packed.clear();
  cols = 0;
  static const bool exact_only = [] {
    const char* e = std::getenv("NSB_EXACT_CLASSES");
    return e && std::atoi(e) != 0;
  }();
  const int n_comp = nq == 1 ? 8 : 32;
  double mc[32];
  double mx = 0.0;
  for (int i = 0; i < n_comp; ++i) mx = std::max(mx, std::fabs(m_in[i]));
  const double thr = exact_only ? 0.0 : std::ldexp(mx, -53);
  for (int i = 0; i < n_comp; ++i) mc[i] = std::fabs(m_in[i]) <= thr ? 0.0 : m_in[i];
  const double* m = mc;
  static const bool no_real = [] {
    const char* e = std::getenv("NSB_NO_REAL_CLASSES");
    return e && std::atoi(e) != 0;
  }();
  auto put = [&](int idx) {
    packed.push_back(m[2 * idx]);
    packed.push_back(m[2 * idx + 1]);
  };
  auto put_zero = [&]() {
    packed.push_back(0.0);
    packed.push_back(0.0);
  };
  if (nq == 1) {
    if (is_zero(m, 1) && is_zero(m, 2)) {
      put(0);
      put(3);
      return kDiag1;
    }
    for (int i = 0; i < 4; ++i) put(i);
    return kDense1;
  }
  bool nz[4][4];
  int max_nnz = 0;
  bool diag = true;
  for (int r = 0; r < 4; ++r) {
    int nnz = 0;
    for (int c = 0; c < 4; ++c) {
      nz[r][c] = !is_zero(m, r * 4 + c);
      if (nz[r][c]) {
        ++nnz;
        if (c != r) diag = false;
      }
    }
    max_nnz = std::max(max_nnz, nnz);
  }
  if (diag) {
    for (int r = 0; r < 4; ++r) put(r * 4 + r);
    return kDiag2;
  }
  auto is_one = [&](int idx) { return m[2 * idx] == 1.0 && m[2 * idx + 1] == 0.0; };
  auto exact_perm = [&](const int* sigma) {
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 4; ++c)
        if (c == sigma[r] ? !is_one(r * 4 + c) : nz[r][c]) return false;
    return true;
  };
  static const int kCxA[4] = {0, 3, 2, 1}, kCxB[4] = {0, 1, 3, 2}, kSw[4] = {0, 2, 1, 3};
  if (exact_perm(kCxA)) return kCX01;
  if (exact_perm(kCxB)) return kCX10;
  if (exact_perm(kSw)) return kSwap;
  // two independent 2x2 blocks on fixed index pairs
  struct PairPattern {
    uint8_t cls;
    int pair[2][2];
  };
  static const PairPattern kPairs[3] = {{kPairQ, {{0, 2}, {1, 3}}},
                                        {kPairP, {{0, 1}, {2, 3}}},
                                        {kPairX, {{0, 3}, {1, 2}}}};
  for (const PairPattern& pp : kPairs) {
    bool fits = true;
    for (int r = 0; r < 4 && fits; ++r) {
      const int* blk = (pp.pair[0][0] == r || pp.pair[0][1] == r) ? pp.pair[0] : pp.pair[1];
      for (int c = 0; c < 4; ++c)
        if (nz[r][c] && c != blk[0] && c != blk[1]) fits = false;
    }
    if (!fits) continue;
    bool real = !no_real;
    for (int b = 0; b < 2; ++b) {
      const int x = pp.pair[b][0], y = pp.pair[b][1];
      const int idx[4] = {x * 4 + x, x * 4 + y, y * 4 + x, y * 4 + y};
      for (int e : idx) {
        put(e);
        real = real && m[2 * e + 1] == 0.0;
      }
    }
    // real blocks: half the multiply-adds (the kernel skips the exact-zero
    // imaginary parts, bit-identical to multiplying by them)
    if (real) return static_cast<uint8_t>(pp.cls == kPairQ ? kPairQr
                                          : pp.cls == kPairP ? kPairPr : kPairXr);
    return pp.cls;
  }
  if (max_nnz <= 1) {
    for (int r = 0; r < 4; ++r) {
      int c0 = 0;
      bool found = false;
      for (int c = 0; c < 4; ++c)
        if (nz[r][c]) {
          c0 = c;
          found = true;
        }
      if (found)
        put(r * 4 + c0);
      else
        put_zero();
      cols |= static_cast<uint16_t>(c0 << (2 * r));
    }
    return kMono2;
  }
  if (max_nnz <= 2) {
    for (int r = 0; r < 4; ++r) {
      int cs[2] = {0, 1}, n = 0;
      for (int c = 0; c < 4 && n < 2; ++c)
        if (nz[r][c]) cs[n++] = c;
      if (n == 1) cs[1] = cs[0] == 0 ? 1 : 0;  // second slot multiplies an exact zero
      for (int j = 0; j < 2; ++j) {
        if (j < n)
          put(r * 4 + cs[j]);
        else
          put_zero();
        cols |= static_cast<uint16_t>(cs[j] << (2 * (2 * r + j)));
      }
    }
    return kSparse2;
  }
  for (int i = 0; i < 16; ++i) put(i);
  return kDense2;
}

// matrix with its two slots exchanged (engine.swap_conjugate, engine.py:124-127)
void swap_slots(double* m) {
  static const int perm[4] = {0, 2, 1, 3};
  double t[32];
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      t[2 * (r * 4 + c)] = m[2 * (perm[r] * 4 + perm[c])];
      t[2 * (r * 4 + c) + 1] = m[2 * (perm[r] * 4 + perm[c]) + 1];
    }
  std::memcpy(m, t, sizeof t);
}

// Greedy dependency-respecting packing of gates (given by qubit masks, in
// execution order) into groups whose qubit union has at most `cap` members
// (`base` is always in the set).  A gate joins the open group if it fits and
// no earlier skipped gate shares a qubit with it; skipped gates keep their
// relative order and are retried first by the next group.  Scanning stops
// after `lookahead` gates or once nothing else can join.
//
// `masks` are the qubits a gate needs inside the group; `deps` (optional,
// defaults to `masks`) are all qubits it reads or writes -- a relabeled gate
// also reads the bits of its dual rows -- and decide ordering conflicts.
std::vector<std::vector<int>> pack_groups(const std::vector<uint64_t>& masks, int cap,
                                          uint64_t base, uint64_t all, int lookahead,
                                          std::vector<uint64_t>& sets,
                                          const std::vector<uint64_t>* deps = nullptr,
                                          const std::vector<int>* weights = nullptr,
                                          int max_count = 1 << 30, int max_weight = 1 << 30) {
  std::vector<std::vector<int>> groups;
  std::vector<int> pending, still;
  size_t cursor = 0;
  const size_t total = masks.size();
  while (!pending.empty() || cursor < total) {
    uint64_t set = base, blocked = 0;
    std::vector<int> grp;
    int scanned = 0, weight = 0;
    still.clear();
    bool stop = false;
    auto visit = [&](int g) {
      const uint64_t m = masks[g];
      const uint64_t dm = deps ? (*deps)[g] : m;
      const int wg = weights ? (*weights)[g] : 0;
      if (!stop && !(dm & blocked) && popc(set | m) <= cap &&
          static_cast<int>(grp.size()) < max_count && weight + wg <= max_weight) {
        set |= m;
        weight += wg;
        grp.push_back(g);
      } else {
        blocked |= dm;
        still.push_back(g);
      }
      ++scanned;
      if (scanned >= lookahead || (blocked & all) == all ||
          (popc(set) >= cap && (set & ~blocked) == 0) ||
          static_cast<int>(grp.size()) >= max_count)
        stop = true;
    };
    for (int g : pending) visit(g);
    while (!stop && cursor < total) visit(static_cast<int>(cursor++));
    pending.swap(still);
    if (grp.empty()) throw std::logic_error("planner made no progress");
    groups.push_back(std::move(grp));
    sets.push_back(set);
  }
  return groups;
}

}  // namespace

// compress the bits of `m` that lie in `set` into consecutive positions
static inline uint32_t pext64(uint64_t m, uint64_t set) {
  uint32_t out = 0;
  int j = 0;
  for (uint64_t s = set; s; s &= s - 1, ++j)
    if (m & (s & -s)) out |= 1u << j;
  return out;
}

static inline int lowest_bit(uint64_t m) { return __builtin_ctzll(m); }

// tile size: the largest k <= kTileQubitsMax whose tile count spreads over
// the persistent CTAs with >= 85% balance (2^(n-k) tiles over `workers`
// CTAs); bigger tiles mean fewer passes, whose fixed cost dominates a lost
// balance of a few percent.
// physical support (bits of ma | mb) above which the frame is flushed first
constexpr int kMaxSupport = 4;

// Scalar part s = U_00 of a near-scalar matrix and the residual ||U - s I||_F
// (dim x dim complex, interleaved re, im)
double scalar_residual(const double* m, int dim, double& s_re, double& s_im) {
  s_re = m[0];
  s_im = m[1];
  double s = 0.0;
  for (int r = 0; r < dim; ++r)
    for (int c = 0; c < dim; ++c) {
      const double re = m[2 * (r * dim + c)] - (r == c ? s_re : 0.0);
      const double im = m[2 * (r * dim + c) + 1] - (r == c ? s_im : 0.0);
      s += re * re + im * im;
    }
  return std::sqrt(s);
}
// a few ulps of 1: products such as H.H or S.Sdg come out as 1 +- 2^-52
constexpr double kIdentityTol = 1e-15;
double default_identity_budget() {
  static const double b = [] {
    const char* e = std::getenv("NSB_IDENTITY_BUDGET");
    return e ? std::atof(e) : 3e-11;
  }();
  return b;
}

int plan_octets(int n) {
  static const int forced = [] {
    const char* e = std::getenv("NSB_PLAN_OCTETS");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 1 || forced == 2) return forced;
  return n <= kSmallStateQubits ? 1 : 2;
}

bool tma_layout(const PassDesc& P, int n, int order, TmaLayout& L) {
  L = TmaLayout();
  if (P.k != kTileQubitsMax || P.tq[0] != 0 || P.tq[1] != 1 || P.tq[2] != 2 || n > kTmaMaxQubits)
    return false;
  struct Run {
    int s, len, pos;  // lowest qubit, length, tile-local position of its lowest bit
  };
  Run runs[16];
  int nr = 0;
  for (int b = 3; b < P.k;) {
    int e = b + 1;
    while (e < P.k && P.tq[e] == P.tq[e - 1] + 1) ++e;
    if (e - b > 8) return false;  // a box dim spans at most 256 (12-qubit tile variants)
    runs[nr++] = {P.tq[b], e - b, b};
    b = e;
  }
  // the dims: the longest runs (fewest copies), four, or three and a gap dim
  int idx[16];
  for (int i = 0; i < nr; ++i) idx[i] = i;
  std::stable_sort(idx, idx + nr, [&](int a, int b) { return runs[a].len > runs[b].len; });
  int nd = std::min(nr, 4);
  bool gap_dim = false;
  int stride_gap = 0;
  for (;;) {
    int low = 0;
    for (int i = 1; i < nd; ++i)
      if (runs[idx[i]].s < runs[idx[low]].s) low = i;
    const Run& r = runs[idx[low]];
    gap_dim = r.s > 3 && !(r.s - 3 <= 3 && r.len + r.s - 3 <= 8);
    stride_gap = r.s > 3 && !gap_dim ? r.s - 3 : 0;
    if (!gap_dim || nd + 1 <= 4) break;
    --nd;  // make room for the gap dim
  }
  // coordinate ranges (qubit order): dim of run j spans [start_j, next start)
  int sel[4];
  for (int i = 0; i < nd; ++i) sel[i] = idx[i];
  std::sort(sel, sel + nd, [&](int a, int b) { return runs[a].s < runs[b].s; });
  int cstart[16], cend[16];
  for (int i = 0; i < nd; ++i) {
    cstart[sel[i]] = runs[sel[i]].s;
    cend[sel[i]] = i + 1 < nd ? runs[sel[i + 1]].s : n;
  }
  if (stride_gap) cstart[sel[0]] = 3;
  // dim order in shared memory: permutation `order` of the run dims
  int ord[4];
  for (int i = 0; i < nd; ++i) ord[i] = sel[i];
  L.n_orders = 1;
  for (int i = 2; i <= nd; ++i) L.n_orders *= i;
  for (int i = 0; i < order % L.n_orders; ++i) std::next_permutation(ord, ord + nd);
  L.len[0] = 3;
  L.rank = 1;
  for (int b = 0; b < 3; ++b) L.perm[b] = static_cast<int8_t>(b);
  int pos = 3;
  for (int i = 0; i < nd; ++i) {
    const Run& r = runs[ord[i]];
    L.start[L.rank] = cstart[ord[i]];
    L.ebits[L.rank] = cend[ord[i]] - cstart[ord[i]];
    L.len[L.rank] = r.len;
    L.gap[L.rank] = cstart[ord[i]] < r.s ? r.s - cstart[ord[i]] : 0;
    ++L.rank;
    for (int t = 0; t < r.len; ++t) L.perm[r.pos + t] = static_cast<int8_t>(pos++);
  }
  if (gap_dim) {  // box of one over qubits 3 .. lowest run - 1
    L.start[L.rank] = 3;
    L.ebits[L.rank] = runs[sel[0]].s - 3;
    L.len[L.rank] = 0;
    ++L.rank;
  }
  bool in_dims[16] = {};
  for (int i = 0; i < nd; ++i) in_dims[sel[i]] = true;
  for (int j = 0; j < nr; ++j)  // the other runs: copy index bits, ascending
    if (!in_dims[j])
      for (int t = 0; t < runs[j].len; ++t) {
        L.left |= uint64_t(1) << (runs[j].s + t);
        L.perm[runs[j].pos + t] = static_cast<int8_t>(pos++);
      }
  return true;
}

static int choose_tile_qubits(int n, int workers) {
  if (n <= kTileQubitsMax) return n;
  for (int k = kTileQubitsMax; k >= 9; --k) {
    const double tiles = std::ldexp(1.0, n - k);
    const double rounds = std::ceil(tiles / workers);
    if (tiles / (rounds * workers) >= 0.85) return k;
  }
  return kTileQubitsMax;
}

// ---- octet groups (planner.h) ----------------------------------------------

namespace {

inline int parity32(uint32_t x) { return __builtin_popcount(x) & 1; }
inline uint32_t swz11(uint32_t l) { return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7u); }
// the TMA layout of a tile at the pass edges (planner.h, swz_tma)
inline uint32_t swz_edge(uint32_t l) { return l ^ ((l >> 3) & 7u); }

// basis of {v in GF(2)^k : parity(f_i & v) = 0 for all i}
struct Basis {
  uint32_t v[16];
  int n = 0;
  bool empty() const { return n == 0; }
  size_t size() const { return static_cast<size_t>(n); }
  uint32_t& operator[](size_t i) { return v[i]; }
  uint32_t* begin() { return v; }
  uint32_t* end() { return v + n; }
  void insert_at(int pos, uint32_t x) {
    for (int i = n; i > pos; --i) v[i] = v[i - 1];
    v[pos] = x;
    ++n;
  }
};

Basis kernel_basis(const uint32_t* f, int nf, int k) {
  uint32_t rows[8];
  int piv[8], nr = 0;
  for (int i = 0; i < nf; ++i) {  // reduced row echelon form
    uint32_t r = f[i];
    for (int j = 0; j < nr; ++j)
      if (r >> piv[j] & 1) r ^= rows[j];
    if (!r) continue;
    const int p = __builtin_ctz(r);
    for (int j = 0; j < nr; ++j)
      if (rows[j] >> p & 1) rows[j] ^= r;
    rows[nr] = r;
    piv[nr++] = p;
  }
  uint32_t pivmask = 0;
  for (int j = 0; j < nr; ++j) pivmask |= 1u << piv[j];
  Basis basis;
  for (int c = 0; c < k; ++c) {
    if (pivmask >> c & 1) continue;
    uint32_t v = 1u << c;
    for (int j = 0; j < nr; ++j)
      if (rows[j] >> c & 1) v |= 1u << piv[j];
    basis.v[basis.n++] = v;
  }
  return basis;
}

// Exchange the two slots of a packed 2q payload (engine.swap_conjugate):
// an exact permutation of values and column codes (no arithmetic).
void swap_packed_slots(uint8_t& cls, double* v, uint16_t& cols) {
  static const int pi[4] = {0, 2, 1, 3};
  double t[32];
  switch (cls) {
    case kDense2:
      swap_slots(v);
      break;
    case kDiag2:
      for (int i = 0; i < 2; ++i) std::swap(v[2 + i], v[4 + i]);
      break;
    case kMono2: {
      std::memcpy(t, v, 8 * sizeof(double));
      uint16_t c2 = 0;
      for (int s = 0; s < 4; ++s) {
        const int ns = pi[s];
        v[2 * ns] = t[2 * s];
        v[2 * ns + 1] = t[2 * s + 1];
        c2 |= static_cast<uint16_t>(pi[(cols >> (2 * s)) & 3] << (2 * ns));
      }
      cols = c2;
      break;
    }
    case kSparse2: {
      std::memcpy(t, v, 16 * sizeof(double));
      uint16_t c2 = 0;
      for (int s = 0; s < 4; ++s) {
        const int ns = pi[s];
        for (int j = 0; j < 2; ++j) {
          v[2 * (2 * ns + j)] = t[2 * (2 * s + j)];
          v[2 * (2 * ns + j) + 1] = t[2 * (2 * s + j) + 1];
          c2 |= static_cast<uint16_t>(pi[(cols >> (2 * (2 * s + j))) & 3] << (2 * (2 * ns + j)));
        }
      }
      cols = c2;
      break;
    }
    case kCX01:
      cls = kCX10;
      break;
    case kCX10:
      cls = kCX01;
      break;
    case kPairQ:
      cls = kPairP;
      break;
    case kPairP:
      cls = kPairQ;
      break;
    case kPairQr:
      cls = kPairPr;
      break;
    case kPairPr:
      cls = kPairQr;
      break;
    case kPairX:  // second block acts on (2, 1) afterwards: reverse its entries
    case kPairXr:
      std::memcpy(t, v + 8, 8 * sizeof(double));
      for (int e = 0; e < 4; ++e) {
        v[8 + 2 * e] = t[2 * (3 - e)];
        v[8 + 2 * e + 1] = t[2 * (3 - e) + 1];
      }
      break;
    default:  // kSwap: symmetric
      break;
  }
}

// ---- group fusion ----------------------------------------------------------
// A group's gates act on the eight octet registers (register index = the
// octet's logical axis bits).  apply_octet mirrors gate1 / gate2 of
// csrc/device.cu on complex registers; fuse_group multiplies the group's
// gates into one 8x8 matrix and, when that product is an axis-targeted
// block op or a diagonal, replaces the gates by ONE whole-octet op
// (kPatT* / kPatAll): one dispatch, no intermediate register copies, and
// for the common (diagonal, two-block) pairs of deep circuits 8 instead of
// 12 multiply-adds per amplitude.  The product is rounded once per entry
// (within the 1e-10 parity bound; components below half an ulp of the
// largest are zeroed as in pack_matrix).
using cplx = std::complex<double>;

// plain complex product (std::complex's operator* calls __muldc3 for its
// NaN/Inf recovery: an order of magnitude slower, and not needed here)
inline cplx cm(const cplx& a, const cplx& b) {
  return cplx(a.real() * b.real() - a.imag() * b.imag(), a.real() * b.imag() + a.imag() * b.real());
}

void apply_octet(const GateOp& op, const double* m2, cplx* x) {
  auto M = [&](int i) { return cplx(m2[2 * i], m2[2 * i + 1]); };
  auto mix = [&](int i, int j, int e) {
    const cplx a = x[i], b = x[j];
    x[i] = cm(M(e), a) + cm(M(e + 1), b);
    x[j] = cm(M(e + 2), a) + cm(M(e + 3), b);
  };
  const int c = op.cls;
  if (op.pat >= kPat0 && op.pat <= kPat2) {
    const int A = 1 << (op.pat - kPat0);
    for (int b = 0; b < 8; ++b) {
      if (b & A) continue;
      if (c == kDiag1) {
        x[b] = cm(M(0), x[b]);
        x[b | A] = cm(M(1), x[b | A]);
      } else {
        mix(b, b | A, 0);
      }
    }
    return;
  }
  static const int kAx[3][2] = {{0, 1}, {0, 2}, {1, 2}};
  const int P = kAx[op.pat][0], Q = kAx[op.pat][1], R = 3 - P - Q;
  const int A = 1 << P, B = 1 << Q, H = 1 << R;
  for (int h = 0; h <= H; h += H) {
    const int idx[4] = {h, h | A, h | B, h | A | B};
    cplx v[4], out[4];
    for (int s = 0; s < 4; ++s) out[s] = v[s] = x[idx[s]];
    switch (c) {
      case kCX01: std::swap(out[1], out[3]); break;
      case kCX10: std::swap(out[2], out[3]); break;
      case kSwap: std::swap(out[1], out[2]); break;
      case kPermute: break;
      case kPairQ: case kPairP: case kPairX: case kPairQr: case kPairPr: case kPairXr: {
        const int k = (c == kPairQ || c == kPairQr) ? 0 : (c == kPairP || c == kPairPr) ? 1 : 2;
        static const int kU[3][4] = {{0, 2, 1, 3}, {0, 1, 2, 3}, {0, 3, 1, 2}};
        const int* u = kU[k];
        out[u[0]] = cm(M(0), v[u[0]]) + cm(M(1), v[u[1]]);
        out[u[1]] = cm(M(2), v[u[0]]) + cm(M(3), v[u[1]]);
        out[u[2]] = cm(M(4), v[u[2]]) + cm(M(5), v[u[3]]);
        out[u[3]] = cm(M(6), v[u[2]]) + cm(M(7), v[u[3]]);
        break;
      }
      case kDiag2:
        for (int s = 0; s < 4; ++s) out[s] = cm(M(s), v[s]);
        break;
      case kMono2:
        for (int s = 0; s < 4; ++s) out[s] = cm(M(s), v[(op.cols >> (2 * s)) & 3]);
        break;
      case kSparse2:
        for (int s = 0; s < 4; ++s)
          out[s] = cm(M(2 * s), v[(op.cols >> (4 * s)) & 3]) +
                   cm(M(2 * s + 1), v[(op.cols >> (4 * s + 2)) & 3]);
        break;
      default:  // kDense2
        for (int s = 0; s < 4; ++s)
          out[s] = cm(M(4 * s), v[0]) + cm(M(4 * s + 1), v[1]) + cm(M(4 * s + 2), v[2]) +
                   cm(M(4 * s + 3), v[3]);
        break;
    }
    for (int s = 0; s < 4; ++s) x[idx[s]] = out[s];
  }
}

// The fused replacement of a group's ops (op + packed values), or false.
bool fuse_group(const std::vector<GateOp>& ops, const std::vector<double>& mats, GateOp& fused,
                std::vector<double>& packed) {
  if (ops.size() < 2) return false;
  // structural pre-check: the XOR span of the register distances the gates
  // can couple must be {0} or {0, 2^t}, else the product cannot qualify
  static const uint8_t kReach2[3] = {1 | 2, 1 | 4, 1 | 8};  // 2q patterns -> slot masks
  (void)kReach2;
  uint32_t span = 0;  // bit mask of axis bits that some gate moves amplitudes along
  for (const GateOp& op : ops) {
    if (op.pat > kPat2) return false;
    if (op.cls == kDiag1 || op.cls == kDiag2 || op.cls == kPermute) continue;
    if (op.pat >= kPat0) {
      span |= 1u << (op.pat - kPat0);
      continue;
    }
    static const int kAx[3][2] = {{0, 1}, {0, 2}, {1, 2}};
    const uint32_t a = 1u << kAx[op.pat][0], b = 1u << kAx[op.pat][1];
    switch (op.cls) {
      case kPairQ: case kPairQr: case kCX01: span |= b; break;   // slot 1 moves
      case kPairP: case kPairPr: case kCX10: span |= a; break;   // slot 0 moves
      default: span |= a | b; break;                            // both (or a diagonal move)
    }
  }
  if (__builtin_popcount(span) > 2) return false;
  // gate cost in multiply-adds per amplitude plus a per-gate overhead (dispatch,
  // matrix loads, register copies; measured to dominate short gates)
  auto cost = [](const GateOp& op) {
    constexpr int kOverhead = 8;
    switch (op.cls) {
      case kDense1: return 8 + kOverhead;
      case kDense2: return 16 + kOverhead;
      case kSparse2: case kPairQ: case kPairP: case kPairX: return 8 + kOverhead;
      case kPairQr: case kPairPr: case kPairXr: case kMono2: case kDiag1: case kDiag2:
        return 4 + kOverhead;
      default: return kOverhead;
    }
  };
  int cost_in = 0;
  for (const GateOp& op : ops) cost_in += cost(op);
  cplx Mx[8][8];
  for (int j = 0; j < 8; ++j) {
    cplx x[8];
    for (int i = 0; i < 8; ++i) x[i] = i == j ? 1.0 : 0.0;
    for (const GateOp& op : ops) apply_octet(op, mats.data() + 2 * op.mat, x);
    for (int i = 0; i < 8; ++i) Mx[i][j] = x[i];
  }
  double mx = 0.0;
  for (auto& row : Mx)
    for (const cplx& v : row) mx = std::max({mx, std::fabs(v.real()), std::fabs(v.imag())});
  const double thr = std::ldexp(mx, -53);
  uint8_t reach = 0;  // bit d: some nonzero entry couples registers r, r ^ d
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c < 8; ++c) {
      cplx& v = Mx[r][c];
      v = cplx(std::fabs(v.real()) <= thr ? 0.0 : v.real(), std::fabs(v.imag()) <= thr ? 0.0 : v.imag());
      if (v != cplx(0.0, 0.0)) reach |= static_cast<uint8_t>(1u << (r ^ c));
    }
  packed.clear();
  auto put = [&](const cplx& v) {
    packed.push_back(v.real());
    packed.push_back(v.imag());
  };
  fused = GateOp{};
  if ((reach & ~1u) == 0) {
    for (int c = 0; c < 8; ++c) put(Mx[c][c]);
    fused.cls = kDiag1;
    fused.pat = kPatAll;
  } else {
    int t = -1;
    for (int a = 0; a < 3; ++a)
      if ((reach & ~(1u | (1u << (1 << a)))) == 0) t = a;
    if (t < 0) {
      // two axes (a < b): a 4x4 on them with one block per value of the third
      // (32 values); only when cheaper than the gates it replaces
      static const int kPairs[3][2] = {{0, 1}, {0, 2}, {1, 2}};
      int pat = -1;
      for (int k = 0; k < 3; ++k) {
        const uint32_t A = 1u << kPairs[k][0], B = 1u << kPairs[k][1];
        const uint32_t ok = (1u << 0) | (1u << A) | (1u << B) | (1u << (A | B));
        if ((reach & ~ok) == 0) pat = k;
      }
      if (pat < 0 || 16 + 8 >= cost_in) return false;
      const int A = 1 << kPairs[pat][0], B = 1 << kPairs[pat][1], H = 7 ^ A ^ B;
      for (int hh = 0; hh < 2; ++hh) {
        const int h = hh ? H : 0;
        const int idx[4] = {h, h | A, h | B, h | A | B};
        for (int r = 0; r < 4; ++r)
          for (int c = 0; c < 4; ++c) put(Mx[idx[r]][idx[c]]);
      }
      fused.cls = kDense2;
      fused.pat = static_cast<uint8_t>(kPatD01 + pat);
      fused.kind = static_cast<uint8_t>(op_kind(fused.pat, fused.cls));
      return true;
    }
    const int T = 1 << t;
    const int L0 = t == 0 ? 2 : 1, L1 = t == 2 ? 2 : 4;  // the other two axes
    for (int b = 0; b < 4; ++b) {
      const int h = ((b & 1) ? L0 : 0) | ((b & 2) ? L1 : 0);
      put(Mx[h][h]);
      put(Mx[h][h | T]);
      put(Mx[h | T][h]);
      put(Mx[h | T][h | T]);
    }
    fused.cls = kDense1;
    fused.pat = static_cast<uint8_t>(kPatT0 + t);
  }
  fused.kind = static_cast<uint8_t>(op_kind(fused.pat, fused.cls));
  return true;
}

struct Axis {
  uint32_t m = 0;     // tile-local physical mask
  uint32_t rin = 0;   // tile-local part of the dual row
  uint64_t rout = 0;  // out-of-tile part
  bool operator==(const Axis& o) const { return m == o.m && rin == o.rin && rout == o.rout; }
};

// A group's registers form a dual basis (m_j, r_j) of a <= 4-dimensional
// subspace V of tile masks and the matching row space R (register position j:
// 0..2 octet bits, 3 the octet index).  Register ops (kRegCX / kRegSwap:
// straight register moves) change the basis without moving data in memory;
// `ax` is the current basis, `ax0` the one the loads use.
struct OpenGroup {
  int nax = 0;
  int maxax = 3;           // 4: four-axis group (the octet index is the fourth axis)
  Axis ax[4];              // current register basis
  Axis ax0[4];             // load basis
  uint32_t rcol[16];       // read map of the group's loads
  uint32_t axm = 0;        // union of the (unpadded) axis masks
  bool r_id = true;        // read map is the identity
  std::vector<GateOp> ops;
  std::vector<double> mats;  // packed payloads of the ops (complex, back to back)
};

// axis slots of the gate's qubits in the group (adding axes if allowed);
// false if the gate needs a fourth axis or clashes with the group's frame
std::atomic<long> g_join_fail[3];  // NSB_PLAN_DEBUG: degenerate, axis overflow, ok
struct JoinReport {
  ~JoinReport() {
    if (std::getenv("NSB_PLAN_DEBUG"))
      std::fprintf(stderr, "join: degenerate %ld overflow %ld ok %ld\n", g_join_fail[0].load(),
                   g_join_fail[1].load(), g_join_fail[2].load());
  }
} g_join_report;

inline int dotp(const Axis& row, uint32_t m) { return parity32(row.rin & m); }

// register ops of register-frame groups (planner.h reg_cx_kind / reg_swap_kind)
inline uint8_t regcx_kind(int j, int k) { return static_cast<uint8_t>(reg_cx_kind(j, k)); }

// Place a gate's axes in the group: every gate axis (m, r) must lie in
// V x R or extend both (keeping the basis dual); register ops then bring it
// to a unit vector at an octet position.  On success the ops are appended
// and pos[a] holds the gate axis' octet position; on failure G is unchanged.
bool place_gate(OpenGroup& G, const Axis* ga, int nq, int* pos) {
  Axis cur[4], load[4];
  int d = G.nax;
  for (int j = 0; j < 4; ++j) {
    cur[j] = G.ax[j];
    load[j] = G.ax0[j];
  }
  std::vector<GateOp> ops;
  auto cx = [&](int j, int k) {  // registers c' = c with bit k ^= bit j
    cur[j].m ^= cur[k].m;
    cur[k].rin ^= cur[j].rin;
    cur[k].rout ^= cur[j].rout;
    GateOp o{};
    o.cls = kPermute;
    o.pat = kPatQ0;
    o.kind = regcx_kind(j, k);
    ops.push_back(o);
  };
  auto swap3 = [&](int f) {
    std::swap(cur[f], cur[3]);
    GateOp o{};
    o.cls = kPermute;
    o.pat = kPatQ0;
    o.kind = static_cast<uint8_t>(reg_swap_kind(f));
    ops.push_back(o);
  };
  uint32_t used = 0;  // positions taken by the gate's earlier axis
  for (int a = 0; a < nq; ++a) {
    const uint32_t m = ga[a].m;
    uint32_t mv = 0, al = 0, be = 0;
    Axis rr{};
    for (int j = 0; j < d; ++j) {
      if (dotp(cur[j], m)) {
        al |= 1u << j;
        mv ^= cur[j].m;
      }
      if (dotp(ga[a], cur[j].m)) {
        be |= 1u << j;
        rr.rin ^= cur[j].rin;
        rr.rout ^= cur[j].rout;
      }
    }
    const bool inV = mv == m, inR = rr.rin == ga[a].rin && rr.rout == ga[a].rout;
    if (!inV || !inR) {
      if (inV || inR) {
        ++g_join_fail[0];
        return false;
      }
      if (d == G.maxax) {
        ++g_join_fail[1];
        return false;
      }
      Axis nw;
      nw.m = m ^ mv;
      nw.rin = ga[a].rin ^ rr.rin;
      nw.rout = ga[a].rout ^ rr.rout;
      if (!dotp(nw, nw.m)) {  // the extended pairing would be degenerate
        ++g_join_fail[0];
        return false;
      }
      cur[d] = load[d] = nw;
      al |= 1u << d;
      be |= 1u << d;
      ++d;
    }
    // pivot: a free position with al = be = 1 (exists: al . be = 1), octet bits first
    int p = -1;
    for (int j = 0; j < d && p < 0; ++j)
      if (!(used >> j & 1) && (al & be) >> j & 1) p = j;
    if (p < 0) throw std::logic_error("gate axis has no pivot in the group");
    for (int k = 0; k < d; ++k)  // masks: clear al outside p
      if (k != p && (al >> k & 1)) {
        cx(p, k);
        al ^= 1u << k;
        if (be >> k & 1) be ^= 1u << p;  // beta_p ^= beta_k
      }
    for (int k = 0; k < d; ++k)  // rows: clear be outside p
      if (k != p && (be >> k & 1)) {
        cx(k, p);
        be ^= 1u << k;
      }
    if (p == 3) {
      int f = 0;
      while (used >> f & 1) ++f;
      swap3(f);
      p = f;
    }
    used |= 1u << p;
    pos[a] = p;
  }
  for (int j = 0; j < 4; ++j) {
    G.ax[j] = cur[j];
    G.ax0[j] = load[j];
  }
  G.nax = d;
  for (const GateOp& o : ops) {
    GateOp q = o;
    q.mat = static_cast<int16_t>(G.mats.size() / 2);
    G.ops.push_back(q);
  }
  ++g_join_fail[2];
  return true;
}

// Warp-local sweeps: with warp positions W (warp-bit count tile positions,
// mask wm) a group whose axes avoid them (and whose read map keeps them) can
// give warp w exactly the amplitudes whose bits at W spell w -- its octets
// never leave that set, so consecutive warp-local sweeps need only __syncwarp.
// Thread layouts (HostPlan::octets): two octets per thread -> 128 threads, 7
// thread bits, 2 warp bits; one octet -> 256 threads, 8 thread bits, 3 warp bits.
constexpr int kMaxWarpBits = 3;
inline int thread_bits_of(int octets) { return plan_thread_bits(octets); }

bool warp_local(const OpenGroup& G, uint32_t wm) {
  if (G.axm & wm) return false;
  if (G.r_id) return true;
  for (int i = 0; i < 16; ++i) {
    const uint32_t want = (wm >> i & 1) ? (1u << i) : 0u;
    if ((G.rcol[i] & wm) != want) return false;
  }
  return true;
}

// load_edge / store_edge (a TMA pass's copy layout, TmaLayout::perm): the
// group reads the tile as TMA left it / writes the layout the TMA store reads
// (swz_tma of the permuted index instead of swz11 on that side)
void finish_group(OpenGroup& G, int k, GroupDesc& d, uint32_t wm, int octets,
                  const int8_t* load_edge = nullptr, const int8_t* store_edge = nullptr) {
  const int tb = thread_bits_of(octets);             // thread bits
  const int ib = tb + (octets == 2 ? 1 : 0);         // octet-index bits
  const int warp_bits = tb - 5;
  auto edge = [k](const int8_t* perm, uint32_t l) {
    uint32_t x = l & ~((1u << k) - 1);
    for (int i = 0; i < k; ++i)
      if (l >> i & 1) x |= 1u << perm[i];
    return swz_edge(x);
  };
  auto swz_ld = [&](uint32_t l) { return load_edge ? edge(load_edge, l) : swz11(l); };
  auto swz_st = [&](uint32_t l) { return store_edge ? edge(store_edge, l) : swz11(l); };
  const bool local = wm != 0;
  while (G.nax < 3) {  // pad with a free axis of the tile (outside the warp positions)
    uint32_t f[3 + kMaxWarpBits];
    int nf = 0;
    for (int i = 0; i < G.nax; ++i) f[nf++] = G.ax[i].rin;  // rows span R (either basis)
    for (uint32_t w = wm; w; w &= w - 1) f[nf++] = w & (0u - w);
    Basis ker = kernel_basis(f, nf, k);
    if (ker.empty()) throw std::logic_error("no free axis in the tile");
    Axis a;
    a.m = ker[0];
    const int p = __builtin_ctz(a.m);
    a.rin = 1u << p;
    for (int j = 0; j < G.nax; ++j)
      if (G.ax[j].m >> p & 1) a.rin ^= G.ax[j].rin;
    G.ax0[G.nax] = a;  // dual to both bases (orthogonal to V and R)
    G.ax[G.nax++] = a;
  }
  const int na = G.nax;  // 3, or 4 (the octet index is axis 3)
  uint32_t f[4] = {G.ax0[0].rin, G.ax0[1].rin, G.ax0[2].rin, na == 4 ? G.ax0[3].rin : 0u};
  Basis C = kernel_basis(f, na, k);
  if (static_cast<int>(C.size()) != k - na) throw std::logic_error("group axes are not dual");
  uint32_t cw[kMaxWarpBits] = {};
  if (local) {  // index bits 5.. (the warp bits) pick the warp's coset of W
    int wp[kMaxWarpBits], nw = 0;
    for (uint32_t w = wm; w; w &= w - 1) wp[nw++] = __builtin_ctz(w);
    auto phi = [&](uint32_t v) {
      uint32_t o = 0;
      for (int j = 0; j < nw; ++j) o |= (v >> wp[j] & 1) << j;
      return o;
    };
    // reduce C so that kWarpBits vectors have unit images under phi, the rest 0
    int np = 0;
    for (int j = 0; j < nw; ++j) {
      int piv = -1;
      for (int i = np; i < C.n; ++i)
        if (phi(C.v[i]) >> j & 1) {
          piv = i;
          break;
        }
      if (piv < 0) throw std::logic_error("warp positions do not split the group");
      std::swap(C.v[np], C.v[piv]);
      for (int i = 0; i < C.n; ++i)
        if (i != np && (phi(C.v[i]) >> j & 1)) C.v[i] ^= C.v[np];
      ++np;
    }
    for (int j = 0; j < nw; ++j) cw[j] = C.v[j];  // phi(cw[j]) = e_j
    Basis K;
    for (int i = nw; i < C.n; ++i) K.v[K.n++] = C.v[i];
    C = K;
  }
  auto rmap = [&](uint32_t u) {  // R u on tile-local bits; batch bits pass through
    uint32_t out = u & ~((1u << k) - 1);
    for (int i = 0; i < k; ++i)
      if (u >> i & 1) out ^= G.rcol[i];
    return out;
  };
  // Thread bits 0..2 first: a quarter-warp (8 lanes of a 128-bit access)
  // spans their combinations, so it hits 8 distinct 16-byte bank groups iff
  // their bank images are independent -- on the load side (read map, load
  // swizzle) and on the store side alike.  Greedy over span(C): the basis
  // vectors first, then every combination, each pick independent of the
  // earlier ones on as many sides as possible (round 2; before, the store side
  // only, which left TMA plans' swz_tma edges with 3x the conflicts).
  {
    auto bank_ld = [&](uint32_t v) { return swz_ld(rmap(v)) & 7u; };
    auto bank_st = [&](uint32_t v) { return swz_st(v) & 7u; };
    struct Span3 {  // reduced basis of a subspace of GF(2)^3 (pivot = lowest bit)
      uint32_t r[3];
      int n = 0;
      uint32_t reduce(uint32_t x) const {
        for (int i = 0; i < n; ++i)
          if (x >> __builtin_ctz(r[i]) & 1) x ^= r[i];
        return x;
      }
      void add(uint32_t x) {
        x = reduce(x);
        if (!x) return;
        for (int i = 0; i < n; ++i)
          if (r[i] >> __builtin_ctz(x) & 1) r[i] ^= x;
        r[n++] = x;
      }
    } sl, ss;
    struct SpanK {  // reduced basis of the picked vectors in tile space
      uint32_t r[16];
      int n = 0;
      uint32_t reduce(uint32_t x) const {
        for (int i = 0; i < n; ++i)
          if (x >> (31 - __builtin_clz(r[i])) & 1) x ^= r[i];
        return x;
      }
      void add(uint32_t x) {
        x = reduce(x);
        if (x) r[n++] = x;
      }
    } picked_span;
    uint32_t picked[3];
    int np = 0;
    const int nk = C.n;
    for (int step = 0; step < 3 && step < nk; ++step) {
      int best = -1;
      uint32_t best_v = 0;
      auto consider = [&](uint32_t v) {
        if (!v || !picked_span.reduce(v)) return;
        const int sc = (sl.reduce(bank_ld(v)) ? 1 : 0) + (ss.reduce(bank_st(v)) ? 1 : 0);
        if (sc > best) {
          best = sc;
          best_v = v;
        }
      };
      for (int i = 0; i < nk && best < 2; ++i) consider(C[i]);
      if (best < 2 && nk <= 8)
        for (uint32_t m = 1; m < (1u << nk) && best < 2; ++m) {
          uint32_t v = 0;
          for (int i = 0; i < nk; ++i)
            if (m >> i & 1) v ^= C[i];
          consider(v);
        }
      if (best <= 0) break;  // nothing independent on either side
      picked[np++] = best_v;
      picked_span.add(best_v);
      sl.add(bank_ld(best_v));
      ss.add(bank_st(best_v));
    }
    if (np) {  // basis of span(C) that starts with the picks
      Basis B;
      SpanK sp = picked_span;
      for (int i = 0; i < np; ++i) B.v[B.n++] = picked[i];
      for (int i = 0; i < nk; ++i)
        if (sp.reduce(C[i])) {
          sp.add(C[i]);
          B.v[B.n++] = C[i];
        }
      if (B.n != nk) throw std::logic_error("thread basis lost a dimension");
      C = B;
    }
  }
  if (local)
    for (int j = warp_bits - 1; j >= 0; --j) C.insert_at(5, cw[j]);
  for (int i = 0; i < 3; ++i) {
    d.am[i] = static_cast<uint16_t>(swz_st(G.ax[i].m));          // final basis (stores)
    d.ram[i] = static_cast<uint16_t>(swz_ld(rmap(G.ax0[i].m)));  // load basis
  }
  // store parity bits: final row j = sum_i M_ji (load row i), M_ji = r_j . m0_i
  d.kmat = 0;
  for (int j = 0; j < 4; ++j) {
    d.r_out[j] = j < na ? G.ax0[j].rout : 0;
    for (int i = 0; i < 4; ++i) {
      const int mji = (j < na && i < na) ? dotp(G.ax[j], G.ax0[i].m) : (i == j ? 1 : 0);
      d.kmat |= static_cast<uint16_t>(mji << (4 * j + i));
    }
  }
  const int cb = k - 3;
  for (int b = 0; b < ib; ++b) {
    if (na == 4 && b == tb) {  // the octet index: axis 3 (load), its final axis (store)
      d.tcol[b] = static_cast<uint16_t>(swz_st(G.ax[3].m));
      d.rtcol[b] = static_cast<uint16_t>(swz_ld(rmap(G.ax0[3].m)));
      continue;
    }
    const uint32_t v = b < cb ? C[b] : (1u << (k + b - cb));  // then tile-in-batch bits
    d.tcol[b] = static_cast<uint16_t>(swz_st(v));
    d.rtcol[b] = static_cast<uint16_t>(swz_ld(rmap(v)));
  }
}

}  // namespace

// Gate runs between two MEASURE / RESET ops are independent planning problems
// (the relabeling frame is flushed at every marker), so long circuits are
// planned on several host threads and the parts concatenated in order.
void HostPlan::build(const nsb_op* ops, int64_t n_ops, const double* params,
                     const double* payloads, int n, int workers) {
  std::vector<int64_t> marks;
  for (int64_t i = 0; i < n_ops; ++i)
    if (ops[i].kind == NSB_OP_MEASURE || ops[i].kind == NSB_OP_RESET) marks.push_back(i);
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (marks.empty() || n_ops < 20000 || hw == 1 || std::getenv("NSB_PLAN_SERIAL")) {
    build_serial(ops, n_ops, params, payloads, n, workers);
    build_mma();
    return;
  }
  const double total_budget = identity_budget >= 0.0 ? identity_budget : default_identity_budget();
  // parts: [0, m0), [m0 + 1, m1), ..., [m_last + 1, n_ops)
  const size_t n_parts = marks.size() + 1;
  std::vector<HostPlan> parts(n_parts);
  std::vector<std::exception_ptr> errors(n_parts);
  auto range = [&](size_t s, int64_t& b, int64_t& e) {
    b = s == 0 ? 0 : marks[s - 1] + 1;
    e = s < marks.size() ? marks[s] : n_ops;
  };
  std::atomic<size_t> next{0};
  auto worker = [&]() {
    for (size_t s; (s = next.fetch_add(1)) < n_parts;) {
      int64_t b, e;
      range(s, b, e);
      try {  // the identity budget is shared out in proportion to the part's ops
        parts[s].identity_budget =
            total_budget * static_cast<double>(e - b) / static_cast<double>(n_ops);
        parts[s].allow_tma = allow_tma;
        parts[s].octets = octets;
        parts[s].build_serial(ops + b, e - b, params, payloads, n, workers);
      } catch (...) {
        errors[s] = std::current_exception();
      }
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < std::min<size_t>(hw, n_parts); ++t) pool.emplace_back(worker);
  worker();
  for (std::thread& t : pool) t.join();
  for (auto& e : errors)
    if (e) std::rethrow_exception(e);
  // concatenate: each part's items, then the marker that ended it
  build_serial(ops, 0, params, payloads, n, workers);  // header fields, no ops
  int step = 0;
  double running_scale2 = 1.0, running_tail_error = 0.0;
  for (size_t s = 0; s < n_parts; ++s) {
    HostPlan& H = parts[s];
    const int32_t pass0 = static_cast<int32_t>(passes.size());
    const int32_t group0 = static_cast<int32_t>(groups.size());
    const int32_t op0 = static_cast<int32_t>(gate_ops.size());
    const int32_t mat0 = static_cast<int32_t>(matrices.size() / 2);
    const int64_t dense0 = static_cast<int64_t>(dense_mats.size() / 2);
    for (PassDesc P : H.passes) {
      P.group_begin += group0;
      P.group_end += group0;
      P.op_begin += op0;
      P.op_end += op0;
      P.mat_begin += mat0;
      passes.push_back(P);
    }
    groups.insert(groups.end(), H.groups.begin(), H.groups.end());
    gate_ops.insert(gate_ops.end(), H.gate_ops.begin(), H.gate_ops.end());
    matrices.insert(matrices.end(), H.matrices.begin(), H.matrices.end());
    dense_mats.insert(dense_mats.end(), H.dense_mats.begin(), H.dense_mats.end());
    for (Item it : H.items) {
      if (it.kind == Item::kGates) {
        it.pass_begin += pass0;
        it.pass_end += pass0;
      } else if (it.kind == Item::kDense) {
        it.mat_off += dense0;
      }
      items.push_back(it);
    }
    n_gates += H.n_gates;
    n_identity_gates += H.n_identity_gates;
    // each part added its own tail error (it has no measurement); only the
    // drift after the circuit's last measurement stays uncompensated
    identity_error += H.identity_error - H.tail_error_total;
    running_tail_error += H.tail_error_total;
    n_frame_gates += H.n_frame_gates;
    n_flush_gates += H.n_flush_gates;
    n_frame_flushes += H.n_frame_flushes;
    n_folded_gates += H.n_folded_gates;
    this->n_ops += H.n_ops;
    n_warp_syncs += H.n_warp_syncs;
    n_fused_group_ops += H.n_fused_group_ops;
    n_axis_swaps += H.n_axis_swaps;
    flops += H.flops;
    for (int c = 0; c < kNumClasses; ++c) class_count[c] += H.class_count[c];
    running_scale2 *= H.tail_scale2;  // parts hold no measurement (split at markers)
    if (s < marks.size()) {
      const nsb_op& o = ops[marks[s]];
      if (o.q[0] < 0 || o.q[0] >= n) throw std::invalid_argument("qubit out of range in plan");
      if (o.kind == NSB_OP_MEASURE) {
        p0_scale.push_back(running_scale2);
        running_scale2 = 1.0;
        running_tail_error = 0.0;
      }
      Item it;
      it.kind = o.kind == NSB_OP_MEASURE ? Item::kMeasure : Item::kReset;
      it.qubit = o.q[0];
      it.step = o.kind == NSB_OP_MEASURE ? step++ : -1;
      items.push_back(it);
    }
  }
  n_measures = step;
  identity_error += running_tail_error;
  build_mma();
}

void HostPlan::build_serial(const nsb_op* ops, int64_t n_ops, const double* params,
                            const double* payloads, int n, int workers) {
  n_qubits = n;
  if (n < 1 || n > kMaxQubits) throw std::invalid_argument("qubit count out of range");
  if (identity_budget < 0.0) identity_budget = default_identity_budget();
  int k = choose_tile_qubits(n, workers);
  if (const char* e = std::getenv("NSB_TILE_QUBITS")) k = std::min(std::atoi(e), n);  // tuning
  tile_qubits = k;
  low_qubits = n <= kL2ResidentQubits ? kLowQubitsL2 : kLowQubits;
  if (const char* e = std::getenv("NSB_LOW_QUBITS")) low_qubits = std::atoi(e);  // tuning
  if (const char* e = std::getenv("NSB_NO_GROUP_FUSION")) fuse_groups = std::atoi(e) == 0;
  // TMA tiles (planner.h): whenever every tile holds qubits 0..2 at full size
  // (the HBM policy, n > kL2ResidentQubits, or NSB_LOW_QUBITS >= 3); NSB_TMA=0 off
  tma = allow_tma && low_qubits >= kLowQubits && k == kTileQubitsMax && n > k &&
        n <= kTmaMaxQubits;
  if (const char* e = std::getenv("NSB_TMA")) tma = tma && std::atoi(e) != 0;
  blocked = n >= 6;
  // NSB_FORCE_PER_OP=1: every gate is its own item executed by the per-op
  // kernels (k_apply1 / k_apply2 / k_applyk, oracle-tested one by one) -- the
  // full-size cross-check of the blocked program (tests/test_fullsize_gpu.py)
  if (const char* e = std::getenv("NSB_FORCE_PER_OP")) blocked = blocked && std::atoi(e) == 0;
  std::vector<PhysGate> run;
  uint64_t col[64];  // frame: physical mask of logical bit j (M e_j)
  uint64_t row[64];  // inverse frame: logical bit j = parity(p & row[j]) (M^-1)
  for (int j = 0; j < 64; ++j) col[j] = row[j] = uint64_t(1) << j;
  std::vector<double> packed;
  int step = 0;

  auto emit_cx = [&](int c, int t) {  // physical CX(control c, target t)
    PhysGate g{};
    g.cls = kCX01;
    g.nq = 2;
    g.ma = g.ra = uint64_t(1) << c;
    g.mb = g.rb = uint64_t(1) << t;
    g.mat = 0;
    g.n_mat = 0;
    run.push_back(g);
    ++n_flush_gates;
  };
  // Bring the frame back to the identity: reduce M to I by column additions
  // col[c] ^= col[t] (= M * CX(c, t)), then M = C_k ... C_1, applied
  // physically in the reverse of the recording order.
  auto flush_frame = [&]() {
    bool identity = true;
    for (int j = 0; j < n; ++j) identity &= col[j] == (uint64_t(1) << j);
    if (identity) return;
    uint64_t m[64];
    std::memcpy(m, col, sizeof m);
    std::vector<std::pair<int, int>> ops_rec;
    for (int b = 0; b < n; ++b) {
      if (!(m[b] >> b & 1)) {
        int j = b + 1;
        while (j < n && !(m[j] >> b & 1)) ++j;
        if (j >= n) throw std::logic_error("relabeling frame is singular");
        m[b] ^= m[j];
        ops_rec.emplace_back(b, j);
      }
      for (int j = 0; j < n; ++j)
        if (j != b && (m[j] >> b & 1)) {
          m[j] ^= m[b];
          ops_rec.emplace_back(j, b);
        }
    }
    for (size_t i = ops_rec.size(); i-- > 0;) emit_cx(ops_rec[i].first, ops_rec[i].second);
    for (int j = 0; j < 64; ++j) col[j] = row[j] = uint64_t(1) << j;
  };
  // A physical CX(c -> t) gives M <- P M: every column holding bit c toggles
  // bit t; M^-1 <- M^-1 P: every row holding bit t toggles bit c.  Clearing
  // the non-pivot bits of one column costs |col| - 1 such gates.
  auto physical_cx = [&](int c, int t) {
    emit_cx(c, t);
    for (int j = 0; j < n; ++j) {
      if (col[j] >> c & 1) col[j] ^= uint64_t(1) << t;
      if (row[j] >> t & 1) row[j] ^= uint64_t(1) << c;
    }
  };
  auto reduce_column = [&](int j) {
    const uint64_t m = col[j];
    if (popc(m) <= 1) return;
    const int pivot = __builtin_ctzll(m);
    for (uint64_t r = m & (m - 1); r; r &= r - 1) physical_cx(pivot, __builtin_ctzll(r));
  };
  auto flush_run = [&]() {
    flush_frame();
    if (run.empty()) return;
    Item it;
    it.kind = Item::kGates;
    it.pass_begin = static_cast<int32_t>(passes.size());
    schedule_run(run, k);
    it.pass_end = static_cast<int32_t>(passes.size());
    items.push_back(it);
    run.clear();
    packed_all.clear();
  };

  for (int64_t i = 0; i < n_ops; ++i) {
    const nsb_op& o = ops[i];
    if (o.kind == NSB_OP_BARRIER) continue;
    for (int j = 0; j < o.nq; ++j)
      if (o.q[j] < 0 || o.q[j] >= n) throw std::invalid_argument("qubit out of range in plan");
    if (o.kind == NSB_OP_MEASURE || o.kind == NSB_OP_RESET) {
      flush_run();
      if (o.kind == NSB_OP_MEASURE) {  // the reference renormalises here
        p0_scale.push_back(tail_scale2);
        tail_scale2 = 1.0;
        tail_error = 0.0;
      }
      Item it;
      it.kind = o.kind == NSB_OP_MEASURE ? Item::kMeasure : Item::kReset;
      it.qubit = o.q[0];
      it.step = o.kind == NSB_OP_MEASURE ? step++ : -1;
      items.push_back(it);
      continue;
    }
    CMat mat;
    const int dim = 1 << o.nq;
    if (o.payload >= 0) {
      if (!payloads) throw std::invalid_argument("payload offset without payload pool");
      mat.dim = dim;
      std::memcpy(mat.v, payloads + 2 * o.payload, sizeof(double) * 2 * dim * dim);
    } else if (!gate_matrix(o.tag, o.param >= 0 ? params + o.param : nullptr,
                            gate_n_params(o.tag), mat) || mat.dim != dim) {
      throw std::invalid_argument("cannot resolve gate matrix");
    }
    ++n_gates;
    if (blocked && o.nq <= 2 && identity_budget > 0.0) {
      double s_re, s_im;
      const double res = scalar_residual(mat.v, dim, s_re, s_im);
      const double mod = std::hypot(s_re, s_im);
      const double phase_err = std::hypot(s_re / mod - 1.0, s_im / mod);
      const double mod_err = std::fabs(mod - 1.0);  // uncompensated only after the last measurement
      const double err = res + phase_err;
      if (res <= kIdentityTol && mod_err <= kIdentityTol && phase_err <= kIdentityTol &&
          identity_error + err + tail_error + mod_err <= identity_budget) {
        identity_error += err;
        tail_error += mod_err;
        tail_scale2 *= mod * mod;
        ++n_identity_gates;
        continue;
      }
    }
    if (o.nq >= 3 || !blocked) {
      flush_run();
      Item it;
      it.kind = Item::kDense;
      it.k = o.nq;
      for (int j = 0; j < o.nq; ++j) it.qs[j] = o.q[j];
      it.mat_off = static_cast<int64_t>(dense_mats.size() / 2);
      dense_mats.insert(dense_mats.end(), mat.v, mat.v + 2 * dim * dim);
      flops += 8ll * dim * dim * (int64_t(1) << (n - o.nq));
      items.push_back(it);
      continue;
    }
    PhysGate g{};
    g.nq = o.nq;
    g.cls = pack_matrix(mat.v, o.nq, packed, g.cols);
    class_count[g.cls]++;
    const int a = o.q[0], b = o.nq == 2 ? o.q[1] : -1;
    // logical CX(c -> t): M <- M C, i.e. column c += column t and, for
    // M^-1 <- C M^-1, row t += row c
    if (g.cls == kCX01) {
      col[a] ^= col[b];
      row[b] ^= row[a];
      ++n_frame_gates;
      continue;
    }
    if (g.cls == kCX10) {
      col[b] ^= col[a];
      row[a] ^= row[b];
      ++n_frame_gates;
      continue;
    }
    if (g.cls == kSwap) {
      std::swap(col[a], col[b]);
      std::swap(row[a], row[b]);
      ++n_frame_gates;
      continue;
    }
    if (popc(col[a] | (o.nq == 2 ? col[b] : 0)) > kMaxSupport) {
      // keep physical supports small so passes stay dense: reduce just this
      // gate's columns to unit vectors with physical CXs (row operations)
      reduce_column(a);
      if (o.nq == 2) reduce_column(b);
      ++n_frame_flushes;
    }
    g.ma = col[a];
    g.mb = o.nq == 2 ? col[b] : 0;
    g.ra = row[a];
    g.rb = o.nq == 2 ? row[b] : 0;
    g.mat = static_cast<int32_t>(packed_all.size() / 2);
    g.n_mat = static_cast<int32_t>(packed.size() / 2);
    packed_all.insert(packed_all.end(), packed.begin(), packed.end());
    static const int kNnz[kNumClasses] = {4, 2, 16, 8, 4, 4, 0, 0, 8, 8, 8, 0, 0, 4, 4, 4};
    flops += 8ll * kNnz[g.cls] * (int64_t(1) << (n - g.nq));
    run.push_back(g);
  }
  flush_run();
  n_measures = step;
  tail_error_total = tail_error;
  identity_error += tail_error;  // after the last measurement: not compensated
  tail_error = 0.0;
}

void HostPlan::schedule_run(std::vector<PhysGate>& run, int k) {
  const int n = n_qubits;
  const uint64_t all = (n == 64) ? ~uint64_t(0) : ((uint64_t(1) << n) - 1);
  const uint64_t low = (uint64_t(1) << std::min(low_qubits, n)) - 1;
  std::vector<uint64_t> masks(run.size()), deps(run.size());
  std::vector<int> weights(run.size());
  for (size_t i = 0; i < run.size(); ++i) {
    masks[i] = run[i].ma | run[i].mb;
    deps[i] = masks[i] | run[i].ra | run[i].rb;
    weights[i] = run[i].n_mat;
    if (popc(masks[i] | low) > k) throw std::logic_error("gate support exceeds the tile");
  }
  std::vector<uint64_t> sets;
  // four-axis groups with a register frame: full tiles, two octets per thread.
  // Off by default (NSB_FOUR_AXIS=1 turns them on): on deep21 they cut the
  // sweeps by 35 % but split group fusion into runs between register ops, so
  // 30 % more gate ops run and the kernel -- bound by per-op latency, not by
  // shared-memory traffic -- got 31 % slower (832 vs 634 ms).
  static const bool four_axis_env = std::getenv("NSB_FOUR_AXIS") != nullptr;
  const bool four_axis = octets == 2 && k == kTileQubitsMax && four_axis_env;
  const int tb = thread_bits_of(octets), warp_bits = tb - 5;
  // one group slot stays free for a trailing read-map sweep
  auto pass_groups = pack_groups(masks, k, low, all, 256, sets, &deps, &weights,
                                 kMaxPassGates - 1, kMaxPassMats);
  // Passes are independent planning problems (each starts from an identity
  // read map): large runs build them on host threads, then concatenate.
  struct PassOut {
    PassDesc P{};
    std::vector<GroupDesc> groups;
    std::vector<GateOp> gate_ops;
    std::vector<double> matrices;
    int64_t n_ops = 0, n_folded = 0, n_permute = 0, n_fused = 0, n_warp = 0, n_axis = 0;
  };
  auto build_pass = [&](size_t pi, PassOut& out) {
    uint64_t tset = sets[pi];
    for (int q = 0; q < n && popc(tset) < k; ++q) tset |= uint64_t(1) << q;
    PassDesc P{};
    P.k = k;
    P.measure_q = P.collapse_q = -1;
    P.measure_slot = P.collapse_slot = -1;
    int t = 0, o = 0;
    for (int q = 0; q < n; ++q) {
      if (tset >> q & 1)
        P.tq[t++] = static_cast<int8_t>(q);
      else
        P.oq[o++] = static_cast<int8_t>(q);
    }
    P.group_begin = static_cast<int32_t>(out.groups.size());
    P.op_begin = static_cast<int32_t>(out.gate_ops.size());
    P.mat_begin = static_cast<int32_t>(out.matrices.size() / 2);
    uint32_t rcol[16];  // pending read map R (tile-local columns), product of CXs
    for (int i = 0; i < 16; ++i) rcol[i] = 1u << i;
    bool r_identity = true;
    OpenGroup G;
    bool open = false;
    std::vector<OpenGroup> closed;  // the pass's groups, finalised at the end
    auto close = [&]() {
      if (!open) return;
      G.axm = 0;
      for (int i = 0; i < G.nax; ++i) G.axm |= G.ax[i].m;
      G.r_id = true;
      for (int i = 0; i < 16; ++i) G.r_id &= G.rcol[i] == (1u << i);
      closed.push_back(std::move(G));
      open = false;
    };
    auto start = [&]() {
      G = OpenGroup();
      G.maxax = four_axis ? 4 : 3;
      std::memcpy(G.rcol, rcol, sizeof rcol);
      for (int i = 0; i < 16; ++i) rcol[i] = 1u << i;
      r_identity = true;
      open = true;
    };
    auto axes_of = [&](const PhysGate& g, Axis* ga) {
      ga[0].m = pext64(g.ma, tset);
      ga[0].rin = pext64(g.ra, tset);
      ga[0].rout = g.ra & ~tset;
      if (g.nq == 2) {
        ga[1].m = pext64(g.mb, tset);
        ga[1].rin = pext64(g.rb, tset);
        ga[1].rout = g.rb & ~tset;
      }
    };
    auto add_op = [&](const PhysGate& g, int* slot) {
      GateOp op{};
      op.cls = g.cls;
      op.cols = g.cols;
      op.mat = static_cast<int16_t>(G.mats.size() / 2);
      const size_t m0 = G.mats.size();
      G.mats.insert(G.mats.end(), packed_all.begin() + 2 * g.mat,
                    packed_all.begin() + 2 * (g.mat + g.n_mat));
      if (g.nq == 1) {
        op.pat = static_cast<uint8_t>(kPat0 + slot[0]);
      } else {
        if (slot[0] > slot[1]) {
          swap_packed_slots(op.cls, G.mats.data() + m0, op.cols);
          std::swap(slot[0], slot[1]);
        }
        op.pat = static_cast<uint8_t>(slot[0] == 0 ? (slot[1] == 1 ? kPat01 : kPat02) : kPat12);
      }
      op.kind = static_cast<uint8_t>(op_kind(op.pat, op.cls));
      G.ops.push_back(op);
      ++out.n_ops;
    };
    // Gates between two folded permutations are grouped greedily with
    // look-ahead: a gate may join the open group ahead of skipped gates it
    // commutes with (disjoint physical supports and dual rows).
    std::vector<int> seg;
    auto flush_segment = [&]() {
      std::vector<int> rest, still;
      rest.swap(seg);
      while (!rest.empty()) {
        close();
        start();
        uint64_t blocked = 0;
        still.clear();
        for (int gi : rest) {
          const PhysGate& g = run[gi];
          const uint64_t dm = g.ma | g.mb | g.ra | g.rb;
          Axis ga[2];
          axes_of(g, ga);
          int slot[2] = {0, 0};
          if (!(dm & blocked) && place_gate(G, ga, g.nq, slot)) {
            add_op(g, slot);
          } else {
            blocked |= dm;
            still.push_back(gi);
          }
        }
        if (G.ops.empty()) throw std::logic_error("grouping made no progress");
        rest.swap(still);
      }
    };
    for (int gi : pass_groups[pi]) {
      const PhysGate& g = run[gi];
      const bool perm = g.cls == kCX01 || g.cls == kCX10 || g.cls == kSwap;
      if (perm && popc(g.ma) == 1 && popc(g.mb) == 1) {
        // fold into the read map of the next group: R <- R C
        flush_segment();
        close();
        const int a = lowest_bit(pext64(g.ma, tset)), b = lowest_bit(pext64(g.mb, tset));
        if (g.cls == kCX01) {
          rcol[a] ^= rcol[b];
        } else if (g.cls == kCX10) {
          rcol[b] ^= rcol[a];
        } else {
          std::swap(rcol[a], rcol[b]);
        }
        r_identity = false;
        ++out.n_folded;
        continue;
      }
      seg.push_back(gi);
    }
    flush_segment();
    close();
    if (!r_identity) {  // trailing permutation: one sweep through R without gates
      start();
      close();
      ++out.n_permute;
    }
    // warp positions: the pair of tile positions that lets the most
    // consecutive sweeps run warp-locally (kThreadBits + 1 octet-index bits
    // must be tile-local for the warp bits 5, 6 to be C vectors: k >= 10)
    // warp positions per group: a run of consecutive groups that share a warp
    // split (two tile positions outside their axes and read maps) runs with
    // __syncwarp between its sweeps; the split may change wherever a CTA
    // barrier is needed anyway.  Dynamic programming over the groups picks
    // the assignment with the most warp-local sweep transitions.
    std::vector<uint32_t> wsel(closed.size(), 0u);
    bool pt = false;  // this pass's tiles move by TMA (planner.h "TMA tiles")
    if (k - 3 >= tb && !closed.empty()) {  // warp bits of the octet index are tile-local
      std::vector<uint32_t> cands;
      for (uint32_t wm = 1; wm < (1u << k); ++wm)
        if (__builtin_popcount(wm) == warp_bits) cands.push_back(wm);
      const size_t G = closed.size(), W = cands.size();
      std::vector<uint8_t> ok(G * W);
      for (size_t g = 0; g < G; ++g)
        for (size_t w = 0; w < W; ++w) ok[g * W + w] = warp_local(closed[g], cands[w]);
      // S[g][w]: most warp-local transitions among groups 0..g with group g on split w
      std::vector<int> S(G * W, 0), from(G * W, -1);
      for (size_t g = 1; g < G; ++g) {
        int best = -1, arg = 0;
        for (size_t w = 0; w < W; ++w)
          if (S[(g - 1) * W + w] > best) best = S[(g - 1) * W + w], arg = static_cast<int>(w);
        for (size_t w = 0; w < W; ++w) {
          int v = best, f = arg;  // switch split (a CTA barrier between g-1 and g)
          if (ok[(g - 1) * W + w] && ok[g * W + w] && S[(g - 1) * W + w] + 1 > v) {
            v = S[(g - 1) * W + w] + 1;
            f = static_cast<int>(w);
          }
          S[g * W + w] = v;
          from[g * W + w] = f;
        }
      }
      int w = 0;
      for (size_t x = 1; x < W; ++x)
        if (S[(G - 1) * W + x] > S[(G - 1) * W + w]) w = static_cast<int>(x);
      for (size_t g = G; g-- > 0;) {
        wsel[g] = ok[g * W + w] ? cands[w] : 0u;
        if (g) w = from[g * W + w];
      }
    }
    // group fusion, within the pass's matrix budget (kMaxPassMats)
    if (fuse_groups) {
      size_t used = 0;
      for (const OpenGroup& H : closed) used += H.mats.size() / 2;
      for (OpenGroup& H : closed) {
        // runs of gates between register-axis exchanges act on the same
        // three octet positions: each run is fused on its own
        std::vector<GateOp> ops_out;
        std::vector<double> mats_out;
        size_t i = 0;
        while (i < H.ops.size()) {
          if (H.ops[i].pat >= kPatQ0) {
            GateOp sw = H.ops[i++];
            sw.mat = static_cast<int16_t>(mats_out.size() / 2);
            ops_out.push_back(sw);
            continue;
          }
          size_t j = i;
          while (j < H.ops.size() && H.ops[j].pat < kPatQ0) ++j;
          std::vector<GateOp> run_ops(H.ops.begin() + i, H.ops.begin() + j);
          GateOp f;
          std::vector<double> pk;
          size_t run_size = 0;  // complex values of the run's own payloads
          auto op_size = [&](const GateOp& o) -> size_t {
            static const int kN[kNumClasses] = {4, 2, 16, 8, 4, 4, 0, 0, 8, 8, 8, 0, 0, 8, 8, 8};
            if (o.pat == kPatAll) return 8;
            if (o.pat >= kPatT0 && o.pat <= kPatT2) return 16;
            if (o.pat >= kPatD01 && o.pat <= kPatD12) return 32;
            return static_cast<size_t>(kN[o.cls]);
          };
          for (const GateOp& o : run_ops) run_size += op_size(o);
          bool fused = false;
          if (fuse_group(run_ops, H.mats, f, pk)) {
            const size_t after = used - run_size + pk.size() / 2;
            if (after <= size_t(kMaxPassMats)) {
              used = after;
              out.n_fused += static_cast<int64_t>(run_ops.size()) - 1;
              out.n_ops -= static_cast<int64_t>(run_ops.size()) - 1;
              f.mat = static_cast<int16_t>(mats_out.size() / 2);
              ops_out.push_back(f);
              mats_out.insert(mats_out.end(), pk.begin(), pk.end());
              fused = true;
            }
          }
          if (!fused)
            for (GateOp o : run_ops) {
              const size_t nv = op_size(o);
              const size_t src = static_cast<size_t>(o.mat);
              o.mat = static_cast<int16_t>(mats_out.size() / 2);
              mats_out.insert(mats_out.end(), H.mats.begin() + 2 * src,
                              H.mats.begin() + 2 * (src + nv));
              ops_out.push_back(o);
            }
          i = j;
        }
        H.ops = std::move(ops_out);
        H.mats = std::move(mats_out);
      }
    }
    if (tma) {
      // the first copy-layout order whose edge sweeps keep all eight bank
      // groups under swz_tma (thread bits 0..2 independent mod the swizzle);
      // none, or too many copies: this pass stays on cp.async and swz
      auto rank3 = [](const uint16_t* v) {
        uint32_t r[3];
        int nr = 0;
        for (int i = 0; i < 3; ++i) {
          uint32_t x = v[i] & 7u;
          for (int j = 0; j < nr; ++j)
            if (x >> __builtin_ctz(r[j]) & 1) x ^= r[j];
          if (!x) continue;
          for (int j = 0; j < nr; ++j)
            if (r[j] >> __builtin_ctz(x) & 1) r[j] ^= x;
          r[nr++] = x;
        }
        return nr;
      };
      TmaLayout L;
      if (tma_layout(P, n, 0, L) && (1 << __builtin_popcountll(L.left)) <= kTmaMaxCopies) {
        const int n_orders = L.n_orders;
        for (int o = 0; o < n_orders && !pt; ++o) {
          tma_layout(P, n, o, L);
          pt = true;
          if (!closed.empty()) {
            const size_t last = closed.size() - 1;
            OpenGroup f = closed.front(), l = closed.back();
            GroupDesc df{}, dl{};
            finish_group(f, k, df, wsel.front(), octets, L.perm, last == 0 ? L.perm : nullptr);
            finish_group(l, k, dl, wsel.back(), octets, last == 0 ? L.perm : nullptr, L.perm);
            pt = rank3(df.rtcol) == 3 && rank3(dl.tcol) == 3;
          }
          if (pt) std::memcpy(P.tperm, L.perm, sizeof P.tperm);
        }
      }
    }
    P.tma = pt ? 1 : 0;
    for (size_t g = 0; g < closed.size(); ++g) {
      OpenGroup& H = closed[g];
      GroupDesc d{};
      d.op_begin = static_cast<uint8_t>(out.gate_ops.size() - P.op_begin);
      d.n_ops_sync = static_cast<uint8_t>(H.ops.size());
      const int32_t mat0 = static_cast<int32_t>(out.matrices.size() / 2) - P.mat_begin;
      for (GateOp op : H.ops) {
        op.mat = static_cast<int16_t>(op.mat + mat0);
        out.gate_ops.push_back(op);
      }
      out.matrices.insert(out.matrices.end(), H.mats.begin(), H.mats.end());
      const uint32_t wm = wsel[g];
      // A warp-local transition g -> g+1 needs each warp's slots to stay its
      // own in BOTH buffers: g+1 overwrites the buffer g read.  Across a TMA
      // edge (g = first: its loads are in the copy layout, g+1's stores on swz;
      // g+1 = last: the reverse) the two layouts map a warp's amplitudes to the
      // same slots only if its split positions are unswizzled (>= 3) and not
      // moved by the copy layout's permutation.
      bool split_fixed = true;
      for (int b = 0; b < k; ++b)
        if (wm >> b & 1) split_fixed = split_fixed && b >= 3 && P.tperm[b] == b;
      const bool edge = pt && (g == 0 || g + 2 == closed.size());
      const bool next = g + 1 < closed.size() && wm && wsel[g + 1] == wm && !(edge && !split_fixed);
      finish_group(H, k, d, wm, octets, pt && g == 0 ? P.tperm : nullptr,
                   pt && g + 1 == closed.size() ? P.tperm : nullptr);
      if (!next) d.n_ops_sync |= 128;
      if (next) ++out.n_warp;
      for (const GateOp& o : H.ops) out.n_axis += o.cls == kPermute && o.pat == kPatQ0;
      out.groups.push_back(d);
    }
    P.group_end = static_cast<int32_t>(out.groups.size());
    P.op_end = static_cast<int32_t>(out.gate_ops.size());
    if (P.op_end - P.op_begin > kMaxPassOps || P.group_end - P.group_begin > kMaxPassGates)
      throw std::logic_error("pass exceeds the kernel's op / group capacity");
    P.mat_count = static_cast<int32_t>(out.matrices.size() / 2) - P.mat_begin;
    out.P = P;
    };
  std::vector<PassOut> outs(pass_groups.size());
  const size_t np = pass_groups.size();
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const size_t n_threads = np >= 64 && !std::getenv("NSB_PLAN_SERIAL") ? std::min<size_t>(hw, np / 32) : 1;
  if (n_threads <= 1) {
    for (size_t pi = 0; pi < np; ++pi) build_pass(pi, outs[pi]);
  } else {
    std::atomic<size_t> next{0};
    std::vector<std::exception_ptr> errs(n_threads);
    auto work = [&](size_t w) {
      try {
        for (size_t pi; (pi = next.fetch_add(1)) < np;) build_pass(pi, outs[pi]);
      } catch (...) {
        errs[w] = std::current_exception();
      }
    };
    std::vector<std::thread> pool;
    for (size_t w = 1; w < n_threads; ++w) pool.emplace_back(work, w);
    work(0);
    for (std::thread& t : pool) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  }
  for (PassOut& out : outs) {  // concatenate in pass order
    PassDesc P = out.P;
    P.group_begin += static_cast<int32_t>(groups.size());
    P.group_end += static_cast<int32_t>(groups.size());
    P.op_begin += static_cast<int32_t>(gate_ops.size());
    P.op_end += static_cast<int32_t>(gate_ops.size());
    P.mat_begin += static_cast<int32_t>(matrices.size() / 2);
    groups.insert(groups.end(), out.groups.begin(), out.groups.end());
    gate_ops.insert(gate_ops.end(), out.gate_ops.begin(), out.gate_ops.end());
    matrices.insert(matrices.end(), out.matrices.begin(), out.matrices.end());
    passes.push_back(P);
    n_ops += out.n_ops;
    n_folded_gates += out.n_folded;
    class_count[kPermute] += out.n_permute;
    n_fused_group_ops += out.n_fused;
    n_warp_syncs += out.n_warp;
    n_axis_swaps += out.n_axis;
  }
}

void HostPlan::build_mma() {
  // single-launch MMA program: possible when every item is a gate run,
  // a measure or a reset (no k>=3 dense gates) and the blocked path is on
  mma_ok = blocked;
  for (const Item& it : items)
    if (it.kind == Item::kDense) mma_ok = false;
  if (!mma_ok) return;
  auto fresh = [&]() {
    PassDesc P{};
    P.k = tile_qubits;
    P.measure_q = P.collapse_q = -1;
    P.measure_slot = P.collapse_slot = -1;
    P.group_begin = P.group_end = 0;
    P.op_begin = P.op_end = 0;
    P.mat_begin = P.mat_count = 0;
    int t = 0, o = 0;
    for (int q = 0; q < n_qubits; ++q) {
      if (q < tile_qubits)
        P.tq[t++] = static_cast<int8_t>(q);
      else
        P.oq[o++] = static_cast<int8_t>(q);
    }
    return P;
  };
  int pending_collapse_q = -1, pending_slot = -1;
  for (const Item& it : items) {
    if (it.kind == Item::kGates) {
      for (int32_t p = it.pass_begin; p < it.pass_end; ++p) {
        PassDesc P = passes[p];
        if (pending_collapse_q >= 0) {
          P.collapse_q = pending_collapse_q;
          P.collapse_slot = pending_slot;
          pending_collapse_q = -1;
        }
        mma_passes.push_back(P);
      }
    } else if (it.kind == Item::kMeasure) {
      if (mma_passes.empty() || mma_passes.back().measure_q >= 0 || pending_collapse_q >= 0) {
        PassDesc P = fresh();
        if (pending_collapse_q >= 0) {
          P.collapse_q = pending_collapse_q;
          P.collapse_slot = pending_slot;
          pending_collapse_q = -1;
        }
        mma_passes.push_back(P);
      }
      mma_passes.back().measure_q = it.qubit;
      mma_passes.back().measure_slot = it.step;
      pending_collapse_q = it.qubit;
      pending_slot = it.step;
    }
    // RESET: no-op in MMA mode (engine.py:420-421)
  }
  if (pending_collapse_q >= 0) {
    PassDesc P = fresh();
    P.collapse_q = pending_collapse_q;
    P.collapse_slot = pending_slot;
    mma_passes.push_back(P);
  }
}

}  // namespace nsb

namespace {
void fill_info(const nsb::HostPlan& H, nsb_plan_info* info) {
  using nsb::Item;
  info->n_identity_gates = H.n_identity_gates;
  info->identity_error = H.identity_error;
  info->n_gates = H.n_gates;
  info->n_measures = H.n_measures;
  int64_t resets = 0, segs = 0;
  for (const Item& it : H.items) {
    resets += it.kind == Item::kReset;
    segs += it.kind == Item::kGates || it.kind == Item::kDense;
  }
  info->n_resets = resets;
  info->n_segments = segs;
  const auto& passes = H.mma_ok ? H.mma_passes : H.passes;
  info->n_passes = static_cast<int64_t>(passes.size());
  info->flops = H.flops;
  info->tile_qubits = H.tile_qubits;
  info->n_items = static_cast<int64_t>(H.items.size());
  info->n_frame_gates = H.n_frame_gates;
  info->n_flush_gates = H.n_flush_gates;
  info->n_device_gates = H.n_ops;
  info->n_sweeps = static_cast<int64_t>(H.groups.size());
  info->n_fused_group_ops = H.n_fused_group_ops;
}
}  // namespace

namespace nsb {
void plan_info(const HostPlan& H, nsb_plan_info* info) { fill_info(H, info); }
double default_identity_budget_value() { return default_identity_budget(); }
}  // namespace nsb

extern "C" int nsb_plan_analyze(const nsb_op* ops, int64_t n_ops, const double* params,
                                const double* payloads, int32_t n_qubits, nsb_plan_info* info,
                                int64_t* class_counts, nsb_status* st) {
  if (!info || (n_ops > 0 && !ops)) {
    nsb::set_status(st, NSB_EINVAL, "null argument");
    return NSB_EINVAL;
  }
  try {
    nsb::HostPlan H;
    H.octets = nsb::plan_octets(n_qubits);
    H.build(ops, n_ops, params, payloads, n_qubits, 296);  // 2 CTAs x 148 SMs (B200)
    fill_info(H, info);
    if (class_counts)
      for (int c = 0; c < nsb::kNumClasses; ++c) class_counts[c] = H.class_count[c];
  } catch (const std::bad_alloc&) {
    nsb::set_status(st, NSB_ERESOURCE, "host out of memory in planner");
    return NSB_ERESOURCE;
  } catch (const std::exception& e) {
    nsb::set_status(st, NSB_EINVAL, e.what());
    return NSB_EINVAL;
  }
  nsb::set_status(st, NSB_OK, "");
  return NSB_OK;
}


extern "C" int nsb_host_plan_build(const nsb_op* ops, int64_t n_ops, const double* params,
                                   const double* payloads, int32_t n_qubits, int32_t workers,
                                   void** out, nsb_status* st) {
  if (!out || (n_ops > 0 && !ops) || workers < 1) {
    nsb::set_status(st, NSB_EINVAL, "bad arguments");
    return NSB_EINVAL;
  }
  *out = nullptr;
  try {
    auto* H = new nsb::HostPlan();
    H->octets = nsb::plan_octets(n_qubits);
    try {
      H->build(ops, n_ops, params, payloads, n_qubits, workers);
    } catch (...) {
      delete H;
      throw;
    }
    for (const nsb::Item& it : H->items) {
      const int kind = it.kind == nsb::Item::kGates ? 0
                       : it.kind == nsb::Item::kMeasure ? 1
                       : it.kind == nsb::Item::kReset ? 2 : 3;
      H->items_flat.push_back(kind);
      H->items_flat.push_back(kind == 0 ? it.pass_begin : it.qubit);
      H->items_flat.push_back(kind == 0 ? it.pass_end : it.step);
      H->items_flat.push_back(it.k);
    }
    *out = H;
  } catch (const std::bad_alloc&) {
    nsb::set_status(st, NSB_ERESOURCE, "host out of memory in planner");
    return NSB_ERESOURCE;
  } catch (const std::exception& e) {
    nsb::set_status(st, NSB_EINVAL, e.what());
    return NSB_EINVAL;
  }
  nsb::set_status(st, NSB_OK, "");
  return NSB_OK;
}

namespace nsb {
// Overlapped qubit swaps (device.cu, nsb_shard_swap_overlap).  A pass never
// moves data between tiles, so a run of passes that all leave a set B of
// local qubits out of their tiles can be executed chunk by chunk, one chunk
// per value of the B bits -- chunk c as soon as chunk c of the swap before it
// has landed.  This picks the longest prefix of item `item`'s passes that
// leaves `want_bits` qubits (other than the swapped local qubit `avoid_q`)
// out of every tile, falling back to fewer bits; B = the highest such
// qubits.  Returns the prefix length (0: no chunking) and B in *cmask.
int chunk_prefix(const HostPlan& H, int64_t item, int avoid_q, int want_bits, uint64_t* cmask) {
  *cmask = 0;
  if (item < 0 || item >= static_cast<int64_t>(H.items.size())) return 0;
  const Item& it = H.items[static_cast<size_t>(item)];
  if (it.kind != Item::kGates || want_bits < 1) return 0;
  const uint64_t all = H.n_qubits >= 64 ? ~uint64_t(0) : (uint64_t(1) << H.n_qubits) - 1;
  for (int bits = std::min(want_bits, 6); bits >= 1; --bits) {
    uint64_t used = avoid_q >= 0 ? uint64_t(1) << avoid_q : 0;
    int n = 0;
    for (int pi = it.pass_begin; pi < it.pass_end; ++pi) {
      const PassDesc& P = H.passes[static_cast<size_t>(pi)];
      uint64_t u = used;
      for (int b = 0; b < P.k; ++b) u |= uint64_t(1) << P.tq[b];
      if (popc(all & ~u) < bits) break;
      used = u;
      ++n;
    }
    if (n == 0) continue;
    uint64_t freeq = all & ~used, m = 0;
    for (int b = 0; b < bits; ++b) {
      const uint64_t top = uint64_t(1) << (63 - __builtin_clzll(freeq));
      m |= top;
      freeq &= ~top;
    }
    *cmask = m;
    return n;
  }
  return 0;
}
}  // namespace nsb

extern "C" int nsb_host_plan_chunk_prefix(const void* plan, int64_t item, int32_t avoid_q,
                                          int32_t want_bits, int32_t* n_pass, uint64_t* cmask) {
  if (!plan || !n_pass || !cmask) return NSB_EINVAL;
  *n_pass = nsb::chunk_prefix(*static_cast<const nsb::HostPlan*>(plan), item, avoid_q, want_bits,
                              cmask);
  return NSB_OK;
}

extern "C" int nsb_host_plan_view(const void* plan, nsb_plan_view* v) {
  if (!plan || !v) return NSB_EINVAL;
  const auto* H = static_cast<const nsb::HostPlan*>(plan);
  std::memset(v, 0, sizeof(*v));
  v->n_qubits = H->n_qubits;
  v->tile_qubits = H->tile_qubits;
  v->tma_edges = H->tma ? 1 : 0;
  v->octets = H->octets;
  v->thread_bits = nsb::plan_thread_bits(H->octets);
  v->mma_ok = H->mma_ok;
  v->n_measures = static_cast<int32_t>(H->n_measures);
  v->pass_desc_bytes = sizeof(nsb::PassDesc);
  v->group_desc_bytes = sizeof(nsb::GroupDesc);
  v->gate_op_bytes = sizeof(nsb::GateOp);
  v->n_passes = static_cast<int64_t>(H->passes.size());
  v->n_mma_passes = static_cast<int64_t>(H->mma_passes.size());
  v->n_groups = static_cast<int64_t>(H->groups.size());
  v->n_gate_ops = static_cast<int64_t>(H->gate_ops.size());
  v->n_matrices = static_cast<int64_t>(H->matrices.size() / 2);
  v->n_items = static_cast<int64_t>(H->items.size());
  v->passes = H->passes.data();
  v->mma_passes = H->mma_passes.data();
  v->groups = H->groups.data();
  v->gate_ops = H->gate_ops.data();
  v->matrices = H->matrices.data();
  v->items = H->items_flat.data();
  return NSB_OK;
}

extern "C" void nsb_host_plan_free(void* plan) { delete static_cast<nsb::HostPlan*>(plan); }
