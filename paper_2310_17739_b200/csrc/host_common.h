// Host-side helpers shared by the gate vocabulary, fusion and planner.
// Compiled with -ffp-contract=off: every fused multiply-add below is an
// explicit std::fma so the products reproduce OpenBLAS zgemm bit-for-bit
// (oracle/zgemm_order.c restates the same orders).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/nucsim_b200.h"

namespace nsb {

// dim x dim complex, row-major, interleaved (re, im)
struct CMat {
  int dim = 0;
  double v[2 * 32 * 32];  // up to 5 qubits
  double& re(int r, int c) { return v[2 * (r * dim + c)]; }
  double& im(int r, int c) { return v[2 * (r * dim + c) + 1]; }
  double re(int r, int c) const { return v[2 * (r * dim + c)]; }
  double im(int r, int c) const { return v[2 * (r * dim + c) + 1]; }
};

// C = A @ B with the accumulation order OpenBLAS's zgemm kernel uses.
//  - "chain": one accumulator per element, k ascending,
//      re = fma(-ai, bi, re); re = fma(ar, br, re); im = fma(ai, br, im); im = fma(ar, bi, im)
//  - "four": four accumulators rr/ii/ri/ir, then re = rr - ii, im = ri + ir
// (numpy `@` -> cblas_zgemm; reference fusion.py:124, 162, 174, 231 and
// gates.py:176).  `chain` is only ever used for 2x2 on CHAIN2 hosts.
inline void matmul_chain(const double* a, const double* b, double* c, int n) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double re = 0.0, im = 0.0;
      for (int k = 0; k < n; ++k) {
        const double ar = a[2 * (i * n + k)], ai = a[2 * (i * n + k) + 1];
        const double br = b[2 * (k * n + j)], bi = b[2 * (k * n + j) + 1];
        re = std::fma(-ai, bi, re);
        re = std::fma(ar, br, re);
        im = std::fma(ai, br, im);
        im = std::fma(ar, bi, im);
      }
      c[2 * (i * n + j)] = re;
      c[2 * (i * n + j) + 1] = im;
    }
}

inline void matmul_four(const double* a, const double* b, double* c, int n) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double rr = 0.0, ii = 0.0, ri = 0.0, ir = 0.0;
      for (int k = 0; k < n; ++k) {
        const double ar = a[2 * (i * n + k)], ai = a[2 * (i * n + k) + 1];
        const double br = b[2 * (k * n + j)], bi = b[2 * (k * n + j) + 1];
        rr = std::fma(ar, br, rr);
        ii = std::fma(ai, bi, ii);
        ri = std::fma(ar, bi, ri);
        ir = std::fma(ai, br, ir);
      }
      c[2 * (i * n + j)] = rr - ii;
      c[2 * (i * n + j) + 1] = ri + ir;
    }
}

inline void matmul(const double* a, const double* b, double* c, int n, int variant) {
  if (n == 2 && variant == NSB_BLAS_CHAIN2)
    matmul_chain(a, b, c, n);
  else
    matmul_four(a, b, c, n);
}

// matrix of a named gate; returns false for tags without a closed form
bool gate_matrix(int tag, const double* p, int n_params, CMat& out);
int gate_arity(int tag);
int gate_n_params(int tag);

void set_status(nsb_status* st, int code, const std::string& msg, int step = 0,
                double prob = 0.0);

}  // namespace nsb
