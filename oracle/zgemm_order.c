/*
 * ORACLE (test infrastructure only -- never linked into the product).
 *
 * C restatement of the accumulation order OpenBLAS 0.3.30's zgemm kernels use
 * for the small complex products the reference's fusion pass computes with
 * numpy `@` (nucsim/fusion.py:124, 162, 174, 231; gates.py:176).  numpy
 * routes complex128 `@` to cblas_zgemm of its bundled OpenBLAS, so these are
 * restatements of that third-party algorithm (scipy-openblas64 0.3.30,
 * DYNAMIC_ARCH), pinned by tests/golden/ fixtures generated from the
 * reference itself:
 *   oracle_mm_chain : SkylakeX / SapphireRapids 2x2 -- one accumulator per
 *                     element, k ascending, re -= ai*bi then re += ar*br,
 *                     im += ai*br then im += ar*bi (each a fused multiply-add)
 *   oracle_mm_four  : every other size / core -- four accumulators
 *                     rr, ii, ri, ir; re = rr - ii, im = ri + ir
 * Compiled with -ffp-contract=off so only the explicit fma() calls fuse.
 */
#include <math.h>

void oracle_mm_chain(int n, const double* a, const double* b, double* c) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double re = 0.0, im = 0.0;
      for (int k = 0; k < n; ++k) {
        const double* x = a + 2 * (i * n + k);
        const double* y = b + 2 * (k * n + j);
        re = fma(-x[1], y[1], re);
        re = fma(x[0], y[0], re);
        im = fma(x[1], y[0], im);
        im = fma(x[0], y[1], im);
      }
      c[2 * (i * n + j)] = re;
      c[2 * (i * n + j) + 1] = im;
    }
}

void oracle_mm_four(int n, const double* a, const double* b, double* c) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double rr = 0.0, ii = 0.0, ri = 0.0, ir = 0.0;
      for (int k = 0; k < n; ++k) {
        const double* x = a + 2 * (i * n + k);
        const double* y = b + 2 * (k * n + j);
        rr = fma(x[0], y[0], rr);
        ii = fma(x[1], y[1], ii);
        ri = fma(x[0], y[1], ri);
        ir = fma(x[1], y[0], ir);
      }
      c[2 * (i * n + j)] = rr - ii;
      c[2 * (i * n + j) + 1] = ri + ir;
    }
}
