// Four-pass 1q/2q gate fusion, bit-exact against the reference pipeline
// (nucsim/fusion.py:101-251):
//   merge_1q            fusion.py:101-131
//   absorb_1q (+sweep)  fusion.py:134-184
//   normalize_2q_order  fusion.py:187-199
//   fuse_2q             fusion.py:202-237
// Walls, slot placement, product order and the per-pass gate counts follow
// the reference exactly; every matrix product uses the host's zgemm FMA
// order (host_common.h) so payloads compare equal with np.array_equal.
//
// Complexity is O(N) per pass with O(1) per-qubit state: a qubit belongs to
// at most one pending run in merge_1q and fuse_2q (a gate touching it
// flushes the others), so the reference's dict scans become array lookups.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <string>
#include <thread>
#include <new>
#include <stdexcept>

#include "host_common.h"

namespace nsb {
namespace {

constexpr int kMaxQ = 64;

struct Fuser {
  const double* params;
  int variant;
  std::vector<double> pool;  // complex payloads, interleaved
  // read-only payloads shared by the segments of a parallel fusion; offsets
  // below n_base index `base`, the rest this fuser's own pool
  const double* base = nullptr;
  int64_t n_base = 0;

  int64_t push_payload(const double* m, int dim) {
    const int64_t off = n_base + static_cast<int64_t>(pool.size() / 2);
    pool.insert(pool.end(), m, m + 2 * dim * dim);
    return off;
  }

  const double* payload(int64_t off) const {
    return off < n_base ? base + 2 * off : pool.data() + 2 * (off - n_base);
  }

  // resolved_matrix (circuit.py:42-46) of a 1- or 2-qubit op
  void matrix(const nsb_op& op, double* out) const {
    const int dim = 1 << op.nq;
    if (op.payload >= 0) {
      std::memcpy(out, payload(op.payload), sizeof(double) * 2 * dim * dim);
      return;
    }
    CMat m;
    const double* p = op.param >= 0 ? params + op.param : nullptr;
    if (!gate_matrix(op.tag, p, gate_n_params(op.tag), m))
      throw std::runtime_error("gate without closed-form matrix reached fusion");
    std::memcpy(out, m.v, sizeof(double) * 2 * dim * dim);
  }

  nsb_op payload_op(int tag, int nq, const int32_t* q, const double* m) {
    nsb_op o{};
    o.kind = NSB_OP_GATE;
    o.tag = tag;
    o.nq = nq;
    o.cbit = -1;
    o.src = -1;
    o.param = -1;
    o.mask = 0;
    for (int j = 0; j < 5; ++j) o.q[j] = j < nq ? q[j] : -1;
    for (int j = 0; j < nq; ++j) o.mask |= uint64_t(1) << q[j];
    o.payload = push_payload(m, 1 << nq);
    return o;
  }
};

inline bool is_gate(const nsb_op& o) { return o.kind == NSB_OP_GATE; }

template <class F>
inline void for_each_qubit(const nsb_op& o, F f) {
  uint64_t m = o.mask;
  while (m) {
    const int q = __builtin_ctzll(m);
    f(q);
    m &= m - 1;
  }
}

// _lift (fusion.py:96-98): slot 0 -> kron(I, V), slot 1 -> kron(V, I)
void lift(const double* v, int slot, double* out) {
  std::memset(out, 0, sizeof(double) * 32);
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      const int rs = slot == 0 ? (r & 1) : (r >> 1), cs = slot == 0 ? (c & 1) : (c >> 1);
      const int ro = slot == 0 ? (r >> 1) : (r & 1), co = slot == 0 ? (c >> 1) : (c & 1);
      if (ro != co) continue;
      out[2 * (r * 4 + c)] = v[2 * (rs * 2 + cs)];
      out[2 * (r * 4 + c) + 1] = v[2 * (rs * 2 + cs) + 1];
    }
}

int64_t count_gates(const std::vector<nsb_op>& ops) {
  int64_t n = 0;
  for (const nsb_op& o : ops) n += is_gate(o);
  return n;
}

std::vector<nsb_op> merge_1q(Fuser& F, const std::vector<nsb_op>& in) {
  std::vector<nsb_op> out;
  out.reserve(in.size());
  struct Run {
    int64_t slot = -1;
    double acc[8];
  };
  std::vector<Run> pending(kMaxQ);
  auto flush = [&](int q) {
    Run& r = pending[q];
    if (r.slot < 0) return;
    const int32_t qs[1] = {q};
    out[r.slot] = F.payload_op(NSB_GATE_C1, 1, qs, r.acc);
    r.slot = -1;
  };
  double u[8], tmp[8];
  for (const nsb_op& ins : in) {
    if (is_gate(ins) && ins.nq == 1) {
      Run& r = pending[ins.q[0]];
      F.matrix(ins, u);
      if (r.slot < 0) {
        r.slot = static_cast<int64_t>(out.size());
        out.push_back(ins);
        std::memcpy(r.acc, u, sizeof u);
      } else {
        matmul(u, r.acc, tmp, 2, F.variant);  // later gate on the left
        std::memcpy(r.acc, tmp, sizeof tmp);
      }
    } else {
      for_each_qubit(ins, flush);
      out.push_back(ins);
    }
  }
  for (int q = 0; q < kMaxQ; ++q) flush(q);
  return out;
}

bool absorb_sweep(Fuser& F, const std::vector<nsb_op>& in, std::vector<nsb_op>& out) {
  std::vector<nsb_op> dest;
  std::vector<char> dead;
  dest.reserve(in.size());
  dead.reserve(in.size());
  std::vector<int64_t> last(kMaxQ, -1);
  bool changed = false;
  double v[8], lifted[32], m[32], tmp[32];
  for (const nsb_op& src : in) {
    nsb_op ins = src;
    if (is_gate(ins) && ins.nq == 1) {
      const int q = ins.q[0];
      const int64_t j = last[q];
      if (j >= 0 && !dead[j] && is_gate(dest[j]) && dest[j].nq == 2) {
        // forward absorption: C2 <- lift(V, slot) @ U  (fusion.py:156-165)
        const nsb_op& prev = dest[j];
        const int slot = prev.q[0] == q ? 0 : 1;
        F.matrix(ins, v);
        lift(v, slot, lifted);
        F.matrix(prev, m);
        matmul(lifted, m, tmp, 4, F.variant);
        dest[j] = F.payload_op(NSB_GATE_C2, 2, prev.q, tmp);
        changed = true;
        continue;
      }
    } else if (is_gate(ins) && ins.nq == 2) {
      // backward absorption, slot 0 then slot 1 (fusion.py:166-178)
      bool have = false;
      for (int slot = 0; slot < 2; ++slot) {
        const int64_t j = last[ins.q[slot]];
        if (j >= 0 && !dead[j] && is_gate(dest[j]) && dest[j].nq == 1) {
          if (!have) {
            F.matrix(ins, m);
            have = true;
          }
          F.matrix(dest[j], v);
          lift(v, slot, lifted);
          matmul(m, lifted, tmp, 4, F.variant);
          std::memcpy(m, tmp, sizeof tmp);
          dead[j] = 1;
          changed = true;
        }
      }
      if (have) ins = F.payload_op(NSB_GATE_C2, 2, ins.q, m);
    }
    dest.push_back(ins);
    dead.push_back(0);
    const int64_t here = static_cast<int64_t>(dest.size()) - 1;
    for_each_qubit(ins, [&](int q) { last[q] = here; });
  }
  out.clear();
  out.reserve(dest.size());
  for (size_t i = 0; i < dest.size(); ++i)
    if (!dead[i]) out.push_back(dest[i]);
  return changed;
}

std::vector<nsb_op> absorb_1q(Fuser& F, const std::vector<nsb_op>& in) {
  std::vector<nsb_op> cur = in, nxt;
  while (absorb_sweep(F, cur, nxt)) cur.swap(nxt);
  return nxt;
}

std::vector<nsb_op> normalize_2q(Fuser& F, const std::vector<nsb_op>& in) {
  static const int perm[4] = {0, 2, 1, 3};
  std::vector<nsb_op> out;
  out.reserve(in.size());
  double m[32], p[32];
  for (const nsb_op& ins : in) {
    if (is_gate(ins) && ins.nq == 2 && ins.q[0] > ins.q[1]) {
      F.matrix(ins, m);
      for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
          p[2 * (r * 4 + c)] = m[2 * (perm[r] * 4 + perm[c])];
          p[2 * (r * 4 + c) + 1] = m[2 * (perm[r] * 4 + perm[c]) + 1];
        }
      const int32_t qs[2] = {ins.q[1], ins.q[0]};
      out.push_back(F.payload_op(NSB_GATE_C2, 2, qs, p));
    } else {
      out.push_back(ins);
    }
  }
  return out;
}

std::vector<nsb_op> fuse_2q(Fuser& F, const std::vector<nsb_op>& in) {
  std::vector<nsb_op> out;
  out.reserve(in.size());
  struct Run {
    int32_t a, b;
    int64_t slot;
    double acc[32];
  };
  std::vector<Run> runs;          // pending runs (slot < 0 = free entry)
  std::vector<int> owner(kMaxQ, -1);  // qubit -> pending run index
  auto flush = [&](int r) {
    Run& run = runs[r];
    const int32_t qs[2] = {run.a, run.b};
    out[run.slot] = F.payload_op(NSB_GATE_C2, 2, qs, run.acc);
    owner[run.a] = owner[run.b] = -1;
    run.slot = -1;
  };
  auto flush_touching = [&](const nsb_op& ins, int keep) {
    for_each_qubit(ins, [&](int q) {
      const int r = owner[q];
      if (r >= 0 && r != keep) flush(r);
    });
  };
  double u[32], tmp[32];
  for (const nsb_op& ins : in) {
    if (is_gate(ins) && ins.nq == 2) {
      const int a = ins.q[0], b = ins.q[1];
      int keep = -1;
      if (owner[a] >= 0 && owner[a] == owner[b] && runs[owner[a]].a == a && runs[owner[a]].b == b)
        keep = owner[a];
      flush_touching(ins, keep);
      F.matrix(ins, u);
      if (keep < 0) {
        int r = -1;
        for (size_t i = 0; i < runs.size(); ++i)
          if (runs[i].slot < 0) {
            r = static_cast<int>(i);
            break;
          }
        if (r < 0) {
          runs.emplace_back();
          r = static_cast<int>(runs.size()) - 1;
        }
        Run& run = runs[r];
        run.a = a;
        run.b = b;
        run.slot = static_cast<int64_t>(out.size());
        std::memcpy(run.acc, u, sizeof u);
        owner[a] = owner[b] = r;
        out.push_back(ins);
      } else {
        Run& run = runs[keep];
        matmul(u, run.acc, tmp, 4, F.variant);
        std::memcpy(run.acc, tmp, sizeof tmp);
      }
    } else {
      flush_touching(ins, -1);
      out.push_back(ins);
    }
  }
  for (size_t r = 0; r < runs.size(); ++r)
    if (runs[r].slot >= 0) flush(static_cast<int>(r));
  return out;
}

using Pass = std::vector<nsb_op> (*)(Fuser&, const std::vector<nsb_op>&);
const Pass kPasses[4] = {merge_1q, absorb_1q, normalize_2q, fuse_2q};

void run_passes(Fuser& F, std::vector<nsb_op>& cur, int pass_mask, int64_t* before,
                int64_t* after) {
  for (int p = 0; p < 4; ++p) {
    before[p] = count_gates(cur);
    if (pass_mask & (1 << p)) cur = kPasses[p](F, cur);
    after[p] = count_gates(cur);
  }
}

inline uint64_t op_mask(const nsb_op& o) {
  uint64_t m = o.mask;
  if (m == 0)
    for (int j = 0; j < o.nq; ++j) m |= uint64_t(1) << o.q[j];
  return m;
}

// Input record i as the passes see it (checked by validate_input first).
inline nsb_op input_op(const nsb_op* ops, int64_t i) {
  nsb_op o = ops[i];
  o.mask = op_mask(o);
  o.src = static_cast<int32_t>(i);
  return o;
}

// The serial loop's checks, in its order (first bad record wins); returns
// the union qubit mask and the extent of the input payload pool.
uint64_t validate_input(const nsb_op* ops, int64_t n_ops, const double* payloads,
                        int64_t* n_base) {
  uint64_t all = 0;
  int64_t ext = 0;
  for (int64_t i = 0; i < n_ops; ++i) {
    const nsb_op& o = ops[i];
    if (o.nq < 0 || o.nq > 5) throw std::invalid_argument("op with bad qubit count");
    if (o.kind == NSB_OP_GATE && o.payload >= 0) {
      if (!payloads) throw std::invalid_argument("payload offset without payload pool");
      ext = std::max<int64_t>(ext, o.payload + (int64_t(1) << (2 * o.nq)));
    } else if (o.kind == NSB_OP_GATE && o.nq <= 2 && gate_arity(o.tag) != o.nq) {
      throw std::invalid_argument("gate tag / qubit count mismatch");
    }
    all |= op_mask(o);
  }
  *n_base = ext;
  return all;
}

// Segment boundaries for parallel fusion: just after every barrier whose qubit
// set covers every qubit of the circuit.  Such a barrier flushes every pending
// run of merge_1q and fuse_2q and resets absorb_1q's last-op table
// (fusion.py:127, 149-150, 233), so no pass carries state across it and the
// segments fuse independently to exactly the sequential result.  Small
// circuits stay on one segment.
std::vector<int64_t> segment_cuts(const nsb_op* ops, int64_t n_ops, uint64_t all) {
  constexpr int64_t kMinSegmentOps = 1 << 15;
  std::vector<int64_t> cuts{0};
  if (n_ops >= 2 * kMinSegmentOps)
    for (int64_t i = 0; i < n_ops; ++i)
      if (ops[i].kind == NSB_OP_BARRIER && (op_mask(ops[i]) & all) == all &&
          i + 1 - cuts.back() >= kMinSegmentOps && n_ops - (i + 1) >= kMinSegmentOps)
        cuts.push_back(i + 1);
  cuts.push_back(n_ops);
  return cuts;
}

// The segments on host threads: each builds its records straight from the
// input, runs the four passes with its own payload pool over the shared input
// payloads (offsets below n_base unchanged), and copies its ops and pool into
// the output at its offset (payload offsets rebased); pass counts summed.
void fuse_segments(const nsb_op* ops, const double* params, const double* payloads,
                   int64_t n_base, const std::vector<int64_t>& cuts, int pass_mask,
                   int variant, nsb_fused* out) {
  const size_t n_seg = cuts.size() - 1;
  struct Seg {
    std::vector<nsb_op> ops;
    Fuser fz;
    int64_t before[4], after[4];
    int64_t op_off = 0, pool_off = 0;  // complex units, after n_base
    std::string err;
    bool oom = false;
  };
  std::vector<Seg> segs(n_seg);
  for (Seg& sg : segs) {
    sg.fz.params = params;
    sg.fz.variant = variant;
    sg.fz.base = payloads;
    sg.fz.n_base = n_base;
  }
  const size_t hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  auto parallel = [&](auto&& body) {
    std::atomic<size_t> next{0};
    auto worker = [&]() {
      for (size_t s; (s = next.fetch_add(1)) < n_seg;) {
        try {
          body(s);
        } catch (const std::bad_alloc&) {
          segs[s].oom = true;
        } catch (const std::exception& e) {
          segs[s].err = e.what();
        }
      }
    };
    std::vector<std::thread> threads;
    for (size_t t = 1; t < std::min(hw, n_seg); ++t) threads.emplace_back(worker);
    worker();
    for (std::thread& t : threads) t.join();
    for (const Seg& sg : segs) {  // the earliest segment's failure, as the serial order
      if (sg.oom) throw std::bad_alloc();
      if (!sg.err.empty()) throw std::runtime_error(sg.err);
    }
  };
  parallel([&](size_t s) {
    Seg& sg = segs[s];
    sg.ops.reserve(cuts[s + 1] - cuts[s]);
    for (int64_t i = cuts[s]; i < cuts[s + 1]; ++i) sg.ops.push_back(input_op(ops, i));
    run_passes(sg.fz, sg.ops, pass_mask, sg.before, sg.after);
  });
  int64_t n_out = 0, n_pool = n_base;
  for (Seg& sg : segs) {
    sg.op_off = n_out;
    sg.pool_off = n_pool;
    n_out += static_cast<int64_t>(sg.ops.size());
    n_pool += static_cast<int64_t>(sg.fz.pool.size() / 2);
  }
  for (int p = 0; p < 4; ++p) {
    out->pass_before[p] = out->pass_after[p] = 0;
    for (const Seg& sg : segs) {
      out->pass_before[p] += sg.before[p];
      out->pass_after[p] += sg.after[p];
    }
  }
  out->gates_before = out->pass_before[0];
  out->n_ops = n_out;
  out->n_payload = n_pool;
  out->ops = static_cast<nsb_op*>(std::malloc(sizeof(nsb_op) * std::max<int64_t>(n_out, 1)));
  out->payloads = static_cast<double*>(std::malloc(sizeof(double) * 2 * std::max<int64_t>(n_pool, 1)));
  if (!out->ops || !out->payloads) throw std::bad_alloc();
  if (n_base > 0) std::memcpy(out->payloads, payloads, sizeof(double) * 2 * n_base);
  parallel([&](size_t s) {
    Seg& sg = segs[s];
    const int64_t shift = sg.pool_off - n_base;
    nsb_op* dst = out->ops + sg.op_off;
    for (size_t i = 0; i < sg.ops.size(); ++i) {
      nsb_op o = sg.ops[i];
      if (o.payload >= n_base) o.payload += shift;
      dst[i] = o;
    }
    if (!sg.fz.pool.empty())
      std::memcpy(out->payloads + 2 * sg.pool_off, sg.fz.pool.data(),
                  sizeof(double) * sg.fz.pool.size());
    std::vector<nsb_op>().swap(sg.ops);
    std::vector<double>().swap(sg.fz.pool);
  });
}

}  // namespace

int fuse(const nsb_op* ops, int64_t n_ops, const double* params, const double* payloads,
         int pass_mask, int variant, nsb_fused* out, nsb_status* st) {
  if (!out || (n_ops > 0 && !ops)) {
    set_status(st, NSB_EINVAL, "null argument");
    return NSB_EINVAL;
  }
  if (variant != NSB_BLAS_CHAIN2 && variant != NSB_BLAS_FOUR) {
    set_status(st, NSB_EINVAL, "unknown blas variant");
    return NSB_EINVAL;
  }
  std::memset(out, 0, sizeof(*out));
  try {
    int64_t n_base = 0;
    const uint64_t all = validate_input(ops, n_ops, payloads, &n_base);
    const std::vector<int64_t> cuts = segment_cuts(ops, n_ops, all);
    if (cuts.size() > 2 && !std::getenv("NSB_FUSE_SERIAL")) {  // (serial: parity tests)
      fuse_segments(ops, params, payloads, n_base, cuts, pass_mask, variant, out);
      set_status(st, NSB_OK, "");
      return NSB_OK;
    }
    Fuser F{params, variant, {}};
    std::vector<nsb_op> cur;
    cur.reserve(n_ops);
    for (int64_t i = 0; i < n_ops; ++i) {
      nsb_op o = ops[i];
      if (o.nq < 0 || o.nq > 5) throw std::invalid_argument("op with bad qubit count");
      if (o.mask == 0)
        for (int j = 0; j < o.nq; ++j) o.mask |= uint64_t(1) << o.q[j];
      o.src = static_cast<int32_t>(i);
      if (o.kind == NSB_OP_GATE && o.payload >= 0) {
        if (!payloads) throw std::invalid_argument("payload offset without payload pool");
        const int dim = 1 << o.nq;
        o.payload = F.push_payload(payloads + 2 * o.payload, dim);
      } else if (o.kind == NSB_OP_GATE && o.nq <= 2 && gate_arity(o.tag) != o.nq) {
        throw std::invalid_argument("gate tag / qubit count mismatch");
      }
      cur.push_back(o);
    }
    out->gates_before = count_gates(cur);
    run_passes(F, cur, pass_mask, out->pass_before, out->pass_after);
    out->n_ops = static_cast<int64_t>(cur.size());
    out->ops = static_cast<nsb_op*>(std::malloc(sizeof(nsb_op) * std::max<size_t>(cur.size(), 1)));
    out->n_payload = static_cast<int64_t>(F.pool.size() / 2);
    out->payloads =
        static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(F.pool.size(), 1)));
    if (!out->ops || !out->payloads) throw std::bad_alloc();
    std::memcpy(out->ops, cur.data(), sizeof(nsb_op) * cur.size());
    std::memcpy(out->payloads, F.pool.data(), sizeof(double) * F.pool.size());
  } catch (const std::bad_alloc&) {
    nsb_fused_free(out);
    set_status(st, NSB_ERESOURCE, "host out of memory during fusion");
    return NSB_ERESOURCE;
  } catch (const std::exception& e) {
    nsb_fused_free(out);
    set_status(st, NSB_EINVAL, e.what());
    return NSB_EINVAL;
  }
  set_status(st, NSB_OK, "");
  return NSB_OK;
}

}  // namespace nsb

extern "C" {

int nsb_fuse(const nsb_op* ops, int64_t n_ops, const double* params, const double* payloads,
             int32_t pass_mask, int32_t blas_variant, nsb_fused* out, nsb_status* st) {
  return nsb::fuse(ops, n_ops, params, payloads, pass_mask, blas_variant, out, st);
}

void nsb_fused_free(nsb_fused* f) {
  if (!f) return;
  std::free(f->ops);
  std::free(f->payloads);
  f->ops = nullptr;
  f->payloads = nullptr;
  f->n_ops = f->n_payload = 0;
}

int nsb_gate_matrix(int32_t tag, const double* params, int32_t n_params, double* out) {
  nsb::CMat m;
  if (!out || !nsb::gate_matrix(tag, params, n_params, m)) return NSB_EINVAL;
  std::memcpy(out, m.v, sizeof(double) * 2 * m.dim * m.dim);
  return NSB_OK;
}

void nsb_free(void* p) { std::free(p); }

}  // extern "C"
