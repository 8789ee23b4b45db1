// Native gate vocabulary: dense matrices bit-identical to the reference's
// gate_matrix (nucsim/gates.py:111-291).  Used by the fusion pass and the
// native filter-circuit generator so 10^8-gate circuits never touch Python.
//
// Exactness notes (verified by tests/test_gates.py against golden vectors):
//  * e^{ix} is (cos x, sin x) from libm, what np.exp(1j*x) returns;
//  * complex * real scalar in numpy is (re*s, im*s) -- no rounding beyond
//    the single product, so we form the products directly;
//  * RCCX / RC3X compose lifted matrices with numpy `@`, i.e. zgemm's
//    four-accumulator order (host_common.h matmul_four).
#include <cstdio>

#include "host_common.h"

namespace nsb {
namespace {

struct Tag {
  int arity, n_params;
};

constexpr Tag kTags[NSB_GATE_COUNT] = {
    {1, 3}, {1, 2}, {1, 1}, {2, 0}, {1, 0}, {1, 0}, {1, 0}, {1, 0}, {1, 0}, {1, 0},
    {1, 0}, {1, 0}, {1, 0}, {1, 1}, {1, 1}, {1, 1}, {2, 0}, {2, 0}, {2, 0}, {2, 0},
    {3, 0}, {3, 0}, {2, 1}, {2, 1}, {2, 1}, {2, 1}, {2, 3}, {2, 1}, {2, 1}, {3, 0},
    {4, 0}, {4, 0}, {4, 0}, {5, 0}, {1, 0}, {2, 0}, {1, 0}, {1, 0}, {0, 0}};

struct C {
  double r, i;
};

// (u00, u01, u10, u11) of a one-qubit tag
bool one_qubit(int tag, const double* p, C u[4]) {
  const double R = std::sqrt(0.5);
  auto set = [&](C a, C b, C c, C d) {
    u[0] = a;
    u[1] = b;
    u[2] = c;
    u[3] = d;
  };
  auto u3 = [&](double theta, double phi, double lam) {
    const double h = theta / 2;
    const double c = std::cos(h), s = std::sin(h);
    const double cl = std::cos(lam), sl = std::sin(lam);
    const double cp = std::cos(phi), sp = std::sin(phi);
    const double pl = phi + lam;
    const double cpl = std::cos(pl), spl = std::sin(pl);
    set({c, 0.0}, {-cl * s, -sl * s}, {cp * s, sp * s}, {cpl * c, spl * c});
  };
  switch (tag) {
    case NSB_GATE_U3: u3(p[0], p[1], p[2]); return true;
    case NSB_GATE_U2: u3(M_PI / 2, p[0], p[1]); return true;
    case NSB_GATE_U1: set({1, 0}, {0, 0}, {0, 0}, {std::cos(p[0]), std::sin(p[0])}); return true;
    case NSB_GATE_RX: {
      const double h = p[0] / 2, c = std::cos(h), s = std::sin(h);
      set({c, 0}, {0, -s}, {0, -s}, {c, 0});
      return true;
    }
    case NSB_GATE_RY: {
      const double h = p[0] / 2, c = std::cos(h), s = std::sin(h);
      set({c, 0}, {-s, 0}, {s, 0}, {c, 0});
      return true;
    }
    case NSB_GATE_RZ: {
      const double h = p[0] / 2, c = std::cos(h), s = std::sin(h);
      set({c, -s}, {0, 0}, {0, 0}, {c, s});
      return true;
    }
    case NSB_GATE_ID: set({1, 0}, {0, 0}, {0, 0}, {1, 0}); return true;
    case NSB_GATE_X: set({0, 0}, {1, 0}, {1, 0}, {0, 0}); return true;
    case NSB_GATE_Y: set({0, 0}, {0, -1}, {0, 1}, {0, 0}); return true;
    case NSB_GATE_Z: set({1, 0}, {0, 0}, {0, 0}, {-1, 0}); return true;
    case NSB_GATE_H: set({R, 0}, {R, 0}, {R, 0}, {-R, 0}); return true;
    case NSB_GATE_S: set({1, 0}, {0, 0}, {0, 0}, {0, 1}); return true;
    case NSB_GATE_SDG: set({1, 0}, {0, 0}, {0, 0}, {0, -1}); return true;
    case NSB_GATE_T:
      set({1, 0}, {0, 0}, {0, 0}, {std::cos(M_PI / 4), std::sin(M_PI / 4)});
      return true;
    case NSB_GATE_TDG:
      set({1, 0}, {0, 0}, {0, 0}, {std::cos(M_PI / 4), -std::sin(M_PI / 4)});
      return true;
    default: return false;
  }
}

void identity(CMat& m, int dim) {
  m.dim = dim;
  std::memset(m.v, 0, sizeof(double) * 2 * dim * dim);
  for (int d = 0; d < dim; ++d) m.re(d, d) = 1.0;
}

void controlled(const C u[4], int n_controls, CMat& m) {
  const int dim = 2 << n_controls;
  identity(m, dim);
  const int lo = (1 << n_controls) - 1, hi = lo | (1 << n_controls);
  const int idx[4][2] = {{lo, lo}, {lo, hi}, {hi, lo}, {hi, hi}};
  for (int e = 0; e < 4; ++e) {
    m.re(idx[e][0], idx[e][1]) = u[e].r;
    m.im(idx[e][0], idx[e][1]) = u[e].i;
  }
}

// scatter a k-slot gate into a width-slot register (exact placement)
void embed(const CMat& u, const int* slots, int k, int width, CMat& out) {
  const int dim = 1 << width;
  out.dim = dim;
  std::memset(out.v, 0, sizeof(double) * 2 * dim * dim);
  for (int col = 0; col < dim; ++col) {
    int sub_col = 0, rest = col;
    for (int j = 0; j < k; ++j) {
      sub_col |= ((col >> slots[j]) & 1) << j;
      rest &= ~(1 << slots[j]);
    }
    for (int sr = 0; sr < (1 << k); ++sr) {
      const double vr = u.re(sr, sub_col), vi = u.im(sr, sub_col);
      if (vr == 0.0 && vi == 0.0) continue;
      int row = rest;
      for (int j = 0; j < k; ++j) row |= ((sr >> j) & 1) << slots[j];
      out.re(row, col) += vr;
      out.im(row, col) += vi;
    }
  }
}

void relative_phase_toffoli(bool four_controls, CMat& out) {
  C hl[4], t[4], tdg[4], xs[4] = {{0, 0}, {1, 0}, {1, 0}, {0, 0}};
  one_qubit(NSB_GATE_U2, (const double[]){0.0, M_PI}, hl);
  one_qubit(NSB_GATE_U1, (const double[]){M_PI / 4}, t);
  one_qubit(NSB_GATE_U1, (const double[]){-M_PI / 4}, tdg);
  CMat H, T, TD, CX;
  auto to_mat = [](const C u[4], CMat& m) {
    m.dim = 2;
    for (int e = 0; e < 4; ++e) {
      m.v[2 * e] = u[e].r;
      m.v[2 * e + 1] = u[e].i;
    }
  };
  to_mat(hl, H);
  to_mat(t, T);
  to_mat(tdg, TD);
  controlled(xs, 1, CX);
  struct Step {
    const CMat* u;
    int s0, s1;  // s1 < 0: one slot
  };
  const int a = 0, b = 1, c = 2, d = 3;
  std::vector<Step> body;
  int width;
  if (!four_controls) {
    width = 3;
    body = {{&H, c, -1}, {&T, c, -1}, {&CX, b, c}, {&TD, c, -1}, {&CX, a, c},
            {&T, c, -1}, {&CX, b, c}, {&TD, c, -1}, {&H, c, -1}};
  } else {
    width = 4;
    body = {{&H, d, -1}, {&T, d, -1}, {&CX, c, d}, {&TD, d, -1}, {&H, d, -1},
            {&CX, a, d}, {&T, d, -1}, {&CX, b, d}, {&TD, d, -1}, {&CX, a, d},
            {&T, d, -1}, {&CX, b, d}, {&TD, d, -1}, {&H, d, -1}, {&T, d, -1},
            {&CX, c, d}, {&TD, d, -1}, {&H, d, -1}};
  }
  CMat acc, lifted, next;
  identity(acc, 1 << width);
  for (const Step& s : body) {
    const int slots[2] = {s.s0, s.s1};
    embed(*s.u, slots, s.s1 < 0 ? 1 : 2, width, lifted);
    next.dim = acc.dim;
    matmul_four(lifted.v, acc.v, next.v, acc.dim);
    std::memcpy(acc.v, next.v, sizeof(double) * 2 * acc.dim * acc.dim);
  }
  out = acc;
}

}  // namespace

int gate_arity(int tag) { return (tag >= 0 && tag < NSB_GATE_COUNT) ? kTags[tag].arity : -1; }
int gate_n_params(int tag) {
  return (tag >= 0 && tag < NSB_GATE_COUNT) ? kTags[tag].n_params : -1;
}

bool gate_matrix(int tag, const double* p, int n_params, CMat& out) {
  if (tag < 0 || tag >= NSB_GATE_COUNT || n_params != kTags[tag].n_params) return false;
  C u[4];
  if (kTags[tag].arity == 1 && one_qubit(tag, p, u)) {
    out.dim = 2;
    for (int e = 0; e < 4; ++e) {
      out.v[2 * e] = u[e].r;
      out.v[2 * e + 1] = u[e].i;
    }
    return true;
  }
  static const C X[4] = {{0, 0}, {1, 0}, {1, 0}, {0, 0}};
  switch (tag) {
    case NSB_GATE_CX: controlled(X, 1, out); return true;
    case NSB_GATE_CY: one_qubit(NSB_GATE_Y, p, u); controlled(u, 1, out); return true;
    case NSB_GATE_CZ: one_qubit(NSB_GATE_Z, p, u); controlled(u, 1, out); return true;
    case NSB_GATE_CH: one_qubit(NSB_GATE_H, p, u); controlled(u, 1, out); return true;
    case NSB_GATE_CRX: one_qubit(NSB_GATE_RX, p, u); controlled(u, 1, out); return true;
    case NSB_GATE_CRY: one_qubit(NSB_GATE_RY, p, u); controlled(u, 1, out); return true;
    case NSB_GATE_CRZ: one_qubit(NSB_GATE_RZ, p, u); controlled(u, 1, out); return true;
    case NSB_GATE_CU1: one_qubit(NSB_GATE_U1, p, u); controlled(u, 1, out); return true;
    case NSB_GATE_CU3: one_qubit(NSB_GATE_U3, p, u); controlled(u, 1, out); return true;
    case NSB_GATE_SWAP: {
      identity(out, 4);
      out.re(1, 1) = out.re(2, 2) = 0.0;
      out.re(1, 2) = out.re(2, 1) = 1.0;
      return true;
    }
    case NSB_GATE_RXX: {
      const double h = p[0] / 2, c = std::cos(h), s = std::sin(h);
      out.dim = 4;
      std::memset(out.v, 0, sizeof(double) * 32);
      for (int d = 0; d < 4; ++d) {
        out.re(d, d) = c;
        out.im(d, 3 - d) = -s;
      }
      return true;
    }
    case NSB_GATE_RZZ: {
      identity(out, 4);
      const double c = std::cos(p[0]), s = std::sin(p[0]);
      out.re(1, 1) = out.re(2, 2) = c;
      out.im(1, 1) = out.im(2, 2) = s;
      return true;
    }
    case NSB_GATE_CCX: controlled(X, 2, out); return true;
    case NSB_GATE_C3X: controlled(X, 3, out); return true;
    case NSB_GATE_C4X: controlled(X, 4, out); return true;
    case NSB_GATE_C3SQRTX: {
      const C sx[4] = {{0.5, 0.5}, {0.5, -0.5}, {0.5, -0.5}, {0.5, 0.5}};
      controlled(sx, 3, out);
      return true;
    }
    case NSB_GATE_CSWAP: {
      identity(out, 8);
      out.re(3, 3) = out.re(5, 5) = 0.0;
      out.re(3, 5) = out.re(5, 3) = 1.0;
      return true;
    }
    case NSB_GATE_RCCX: relative_phase_toffoli(false, out); return true;
    case NSB_GATE_RC3X: relative_phase_toffoli(true, out); return true;
    default: return false;
  }
}

void set_status(nsb_status* st, int code, const std::string& msg, int step, double prob) {
  if (!st) return;
  st->code = code;
  st->step = step;
  st->prob = prob;
  std::snprintf(st->msg, sizeof(st->msg), "%s", msg.c_str());
}

}  // namespace nsb
