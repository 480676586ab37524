/* Error anatomy of the FP32 Barnes-Hut sum (analysis tool, not product).
 * Same DFS and fp64 MAC decisions as the oracle (_kernels.py:17-48); for the
 * accepted nodes the force is summed under arithmetic variants:
 *   v0  fp64 (the reference)
 *   v1  fp32 coordinates (q, com rounded), fp32 terms, correctly rounded rsqrt, fp32 sum
 *   v2  dx rounded from the fp64 difference, fp32 terms and sum
 *   v3  v1 terms, fp64 sum
 *   v4  v1 with an fp32 rsqrt of 2^-22.9 relative error (worst-case sign +)
 * build: gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC -o /tmp/fp32err.so tools/fp32_error.c -lm */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifndef H5T
#define H5T float
#endif

/* v5 (fold): v1 with the partial folded into a second fp32 sum whenever the
 * node's mirrored-preorder index (mir, the device traversal order) passes a
 * multiple of `fold`, or every `fold_terms` accepted terms when fold < 0. */
void fp32_error(const int64_t* children, const double* com, const double* mass,
                const double* length, const double* q, const double* qm, int64_t m, double theta,
                double G, double eps2, const int64_t* mir, int64_t fold,
                double* out /* m x 6 x 3 */) {
  const double th2 = theta * theta;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < m; i++) {
    int64_t stack[256];
    int sp = 0;
    stack[sp++] = 0;
    double f0[3] = {0, 0, 0}, f3[3] = {0, 0, 0};
    float f1[3] = {0, 0, 0}, f2[3] = {0, 0, 0}, f4[3] = {0, 0, 0};
    float p5[3] = {0, 0, 0};
    H5T h5[3] = {0, 0, 0};
    int64_t lim = fold > 0 ? fold : 0, nterms = 0;
    const double* qq = q + 3 * i;
    const float q32[3] = {(float)qq[0], (float)qq[1], (float)qq[2]};
    const float e2f = (float)eps2;
    while (sp > 0) {
      const int64_t nd = stack[--sp];
      const double* c = com + 3 * nd;
      double d[3], d2 = 0.0;
      for (int k = 0; k < 3; k++) {
        d[k] = qq[k] - c[k];
        d2 += d[k] * d[k];
      }
      int leaf = 1;
      for (int k = 0; k < 8; k++) leaf &= children[8 * nd + k] < 0;
      if (leaf || length[nd] * length[nd] < th2 * d2) {
        const double den = d2 + eps2;
        if (den > 0) {
          const double w = G * qm[i] * mass[nd] / (den * sqrt(den));
          for (int k = 0; k < 3; k++) f0[k] -= w * d[k];
        }
        /* fp32 variants: a = m * inv^3 * (com - q) accumulated, times G m_q */
        float dx1[3], dx2[3];
        for (int k = 0; k < 3; k++) {
          dx1[k] = (float)c[k] - q32[k];
          dx2[k] = (float)(c[k] - qq[k]);
        }
        const float m32 = (float)mass[nd];
        {
          const float r2 = dx1[0] * dx1[0] + dx1[1] * dx1[1] + dx1[2] * dx1[2] + e2f;
          const float inv = 1.0f / sqrtf(r2);
          const float w = m32 * (inv * inv * inv);
          const float inva = inv * (1.0f + 1.27e-7f);
          const float wa = m32 * (inva * inva * inva);
          if (fold > 0 && mir[nd] >= lim) {
            for (int k = 0; k < 3; k++) { h5[k] += p5[k]; p5[k] = 0.f; }
            lim = (mir[nd] / fold + 1) * fold;
          } else if (fold < 0 && nterms > 0 && nterms % (-fold) == 0) {
            for (int k = 0; k < 3; k++) { h5[k] += p5[k]; p5[k] = 0.f; }
          }
          nterms++;
          for (int k = 0; k < 3; k++) {
            p5[k] = fmaf(w, dx1[k], p5[k]);
            f1[k] = fmaf(w, dx1[k], f1[k]);
            f3[k] += (double)(w * dx1[k]);
            f4[k] = fmaf(wa, dx1[k], f4[k]);
          }
        }
        {
          const float r2 = dx2[0] * dx2[0] + dx2[1] * dx2[1] + dx2[2] * dx2[2] + e2f;
          const float inv = 1.0f / sqrtf(r2);
          const float w = m32 * (inv * inv * inv);
          for (int k = 0; k < 3; k++) f2[k] = fmaf(w, dx2[k], f2[k]);
        }
      } else {
        for (int k = 0; k < 8; k++) {
          const int64_t ch = children[8 * nd + k];
          if (ch >= 0) stack[sp++] = ch;
        }
      }
    }
    const double gq = G * qm[i];
    double* o = out + 18 * i;
    for (int k = 0; k < 3; k++) o[15 + k] = gq * (double)(h5[k] + p5[k]);
    for (int k = 0; k < 3; k++) {
      o[k] = f0[k];
      o[3 + k] = gq * f1[k];
      o[6 + k] = gq * f2[k];
      o[9 + k] = gq * f3[k];
      o[12 + k] = gq * f4[k];
    }
  }
}
