// Native projection-filter circuit emitter: the instruction stream of the
// reference's build_filter_circuit (nucsim/projection.py:215-255) with its
// per-term rotation body _rotation (projection.py:191-212), written straight
// into the packed op list so 10^8-gate workloads never become Python objects.
// Parameters are deduplicated: every (filter step, term) pair shares one
// params-pool slot across its Trotter slices.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <stdexcept>

#include "host_common.h"

namespace nsb {
namespace {

struct Emitter {
  // the op list is written straight into the malloc'd output buffer (10^8
  // records are GBs: no second copy); `cap` is an upper bound fixed up front
  nsb_op* ops = nullptr;
  size_t n_ops = 0, cap = 0;
  std::vector<double> params;
  int n;  // register width (system + ancilla)

  ~Emitter() { std::free(ops); }
  void reserve(size_t c) {
    ops = static_cast<nsb_op*>(std::malloc(sizeof(nsb_op) * std::max<size_t>(c, 1)));
    if (!ops) throw std::bad_alloc();
    cap = c;
  }
  void push(const nsb_op& o) {
    if (n_ops == cap) throw std::logic_error("generator op count bound exceeded");
    ops[n_ops++] = o;
  }
  // append `times` copies of records [b, e) (identical Trotter slices)
  void repeat(size_t b, size_t e, int64_t times) {
    const size_t len = e - b;
    if (n_ops + len * static_cast<size_t>(times) > cap)
      throw std::logic_error("generator op count bound exceeded");
    for (int64_t r = 0; r < times; ++r, n_ops += len)
      std::memcpy(ops + n_ops, ops + b, sizeof(nsb_op) * len);
  }

  void gate(int tag, int a, int b = -1, int64_t param = -1) {
    nsb_op o{};
    o.kind = NSB_OP_GATE;
    o.tag = tag;
    o.nq = b < 0 ? 1 : 2;
    o.cbit = -1;
    for (int j = 0; j < 5; ++j) o.q[j] = -1;
    o.q[0] = a;
    o.q[1] = b;
    o.src = -1;
    o.param = param;
    o.payload = -1;
    o.mask = (uint64_t(1) << a) | (b >= 0 ? uint64_t(1) << b : 0);
    push(o);
  }
  void marker(int kind, int q, int cbit) {
    nsb_op o{};
    o.kind = kind;
    o.tag = kind == NSB_OP_MEASURE ? NSB_GATE_MEASURE
                                   : (kind == NSB_OP_RESET ? NSB_GATE_RESET : NSB_GATE_BARRIER);
    o.nq = kind == NSB_OP_BARRIER ? 0 : 1;
    o.cbit = cbit;
    for (int j = 0; j < 5; ++j) o.q[j] = -1;
    if (q >= 0) o.q[0] = q;
    o.src = -1;
    o.param = -1;
    o.payload = -1;
    o.mask = kind == NSB_OP_BARRIER ? ((n == 64) ? ~uint64_t(0) : (uint64_t(1) << n) - 1)
                                    : uint64_t(1) << q;
    push(o);
  }
  int64_t param(double v) {
    params.push_back(v);
    return static_cast<int64_t>(params.size()) - 1;
  }
};

}  // namespace

int generate_filter(int n_system, const uint8_t* letters, const double* coeffs, int64_t n_terms,
                    const double* steps, int n_steps, int64_t trotter, const uint8_t* trial,
                    nsb_fused* out, double** params_out, int64_t* n_params_out, nsb_status* st) {
  if (n_system < 1 || n_system + 1 > 64 || n_steps < 1 || trotter < 1 || !out || !params_out ||
      !n_params_out || (n_terms > 0 && (!letters || !coeffs)) || !steps) {
    set_status(st, NSB_EINVAL, "invalid generator arguments");
    return NSB_EINVAL;
  }
  std::memset(out, 0, sizeof(*out));
  try {
    Emitter E;
    E.n = n_system + 1;
    const int anc = n_system;
    // per-term layout, reused across slices
    std::vector<std::vector<int>> involved(n_terms);
    int64_t body_gates = 0;
    for (int64_t t = 0; t < n_terms; ++t) {
      for (int q = 0; q < n_system; ++q) {
        const uint8_t c = letters[t * n_system + q];
        if (c > 3) throw std::invalid_argument("Pauli letter code must be 0..3");
        if (c != 0) involved[t].push_back(q);
      }
      const int m = static_cast<int>(involved[t].size());
      body_gates += m == 0 ? 1 : 2 * m + 5 + 4 * m;
    }
    E.reserve(static_cast<size_t>(n_steps * (trotter * body_gates + 5) + n_system + 1 + 64));
    if (trial)
      for (int q = 0; q < n_system; ++q)
        if (trial[q]) E.gate(NSB_GATE_X, q);
    std::vector<int64_t> theta_slot(n_terms);
    for (int i = 0; i < n_steps; ++i) {
      const double t_i = steps[2 * i], delta = steps[2 * i + 1];
      for (int64_t t = 0; t < n_terms; ++t) {
        const double theta = coeffs[t] * t_i / static_cast<double>(trotter);
        theta_slot[t] = E.param(2.0 * theta);
      }
      // every slice of a step is the same record sequence (the step's
      // parameter slots are shared): emit one, copy it trotter - 1 times
      const size_t slice0 = E.n_ops;
      {
        for (int64_t t = 0; t < n_terms; ++t) {
          const std::vector<int>& inv = involved[t];
          const uint8_t* L = letters + t * n_system;
          if (inv.empty()) {
            E.gate(NSB_GATE_RY, anc, -1, theta_slot[t]);
            continue;
          }
          for (int q : inv) {  // basis change in: X -> h, Y -> sdg h
            if (L[q] == 1) E.gate(NSB_GATE_H, q);
            if (L[q] == 2) {
              E.gate(NSB_GATE_SDG, q);
              E.gate(NSB_GATE_H, q);
            }
          }
          E.gate(NSB_GATE_SDG, anc);
          E.gate(NSB_GATE_H, anc);
          for (size_t j = 0; j < inv.size(); ++j)
            E.gate(NSB_GATE_CX, inv[j], j + 1 < inv.size() ? inv[j + 1] : anc);
          E.gate(NSB_GATE_RZ, anc, -1, theta_slot[t]);
          for (size_t j = inv.size(); j-- > 0;)
            E.gate(NSB_GATE_CX, inv[j], j + 1 < inv.size() ? inv[j + 1] : anc);
          E.gate(NSB_GATE_H, anc);
          E.gate(NSB_GATE_S, anc);
          for (size_t j = inv.size(); j-- > 0;) {  // basis change out: X -> h, Y -> h s
            const int q = inv[j];
            if (L[q] == 1) E.gate(NSB_GATE_H, q);
            if (L[q] == 2) {
              E.gate(NSB_GATE_H, q);
              E.gate(NSB_GATE_S, q);
            }
          }
        }
      }
      E.repeat(slice0, E.n_ops, trotter - 1);
      E.gate(NSB_GATE_RY, anc, -1, E.param(2.0 * delta));
      E.marker(NSB_OP_MEASURE, anc, i);
      E.marker(NSB_OP_BARRIER, -1, -1);
      E.marker(NSB_OP_RESET, anc, -1);
      E.marker(NSB_OP_BARRIER, -1, -1);
    }
    for (int q = 0; q <= n_system; ++q) E.marker(NSB_OP_MEASURE, q, n_steps + q);
    *params_out = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(1, E.params.size())));
    if (!*params_out) throw std::bad_alloc();
    std::memcpy(*params_out, E.params.data(), sizeof(double) * E.params.size());
    *n_params_out = static_cast<int64_t>(E.params.size());
    int64_t g = 0;
    for (size_t i = 0; i < E.n_ops; ++i) g += E.ops[i].kind == NSB_OP_GATE;
    out->gates_before = g;
    out->n_ops = static_cast<int64_t>(E.n_ops);
    nsb_op* shrunk = static_cast<nsb_op*>(std::realloc(E.ops, sizeof(nsb_op) * std::max<size_t>(E.n_ops, 1)));
    out->ops = shrunk ? shrunk : E.ops;
    E.ops = nullptr;  // owned by out
  } catch (const std::bad_alloc&) {
    std::free(out->ops);
    out->ops = nullptr;
    set_status(st, NSB_ERESOURCE, "host out of memory in generator");
    return NSB_ERESOURCE;
  } catch (const std::exception& e) {
    std::free(out->ops);
    out->ops = nullptr;
    set_status(st, NSB_EINVAL, e.what());
    return NSB_EINVAL;
  }
  set_status(st, NSB_OK, "");
  return NSB_OK;
}

}  // namespace nsb

extern "C" int nsb_generate_filter(int32_t n_system, const uint8_t* letters, const double* coeffs,
                                   int64_t n_terms, const double* steps, int32_t n_steps,
                                   int64_t trotter, const uint8_t* trial_bits, nsb_fused* out,
                                   double** params_out, int64_t* n_params_out, nsb_status* st) {
  return nsb::generate_filter(n_system, letters, coeffs, n_terms, steps, n_steps, trotter,
                              trial_bits, out, params_out, n_params_out, st);
}
