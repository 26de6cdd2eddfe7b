/* Plain-C restatement of the reference CSR reduction order -- TEST
 * INFRASTRUCTURE ONLY (oracle/, never linked into the product).
 *
 * The reference aggregates each CSR row with np.add.reduceat over
 * contrib = fl32(val * x[col]) (kernels.py:112-113, :187-188).  numpy
 * evaluates one reduceat segment c[0..m) as  c[0] + P(c[1..m))  where P is
 * numpy's pairwise_sum (numpy/_core/src/umath/loops_utils.h.src):
 *   n < 8     r = -0.0; r += a[i] in order
 *   n <= 128  8 accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), tail in order
 *   n > 128   m = n/2 - (n/2)%8 ; P(a[:m]) + P(a[m:])
 * tests/test_oracle.py checks this file bit-for-bit against np.add.reduceat,
 * which pins the order the CUDA kernel (csrc/ag_spmm.cu) implements.
 * Compiled with -ffp-contract=off so no FMA is formed. */
#include <stdint.h>
#include <string.h>

static float pw(const float *a, int64_t n, int64_t stride) {
  if (n < 8) {
    float r = -0.0f;
    for (int64_t i = 0; i < n; ++i) r += a[i * stride];
    return r;
  }
  if (n <= 128) {
    float r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j * stride];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[(i + j) * stride];
    float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i * stride];
    return res;
  }
  int64_t m = n / 2;
  m -= m % 8;
  return pw(a, m, stride) + pw(a + m * stride, n - m, stride);
}

/* y[V,F] = reduceat-order CSR aggregation (sum); rows without edges are 0.
 * scratch must hold max_row_len * F floats. */
void oracle_csr_sum(int64_t V, int64_t F, const int32_t *row_ptr, const int32_t *col,
                    const float *val, const float *x, float *y, float *scratch) {
  for (int64_t r = 0; r < V; ++r) {
    const int64_t s = row_ptr[r], e = row_ptr[r + 1];
    float *out = y + r * F;
    if (e == s) {
      memset(out, 0, (size_t)F * sizeof(float));
      continue;
    }
    const int64_t m = e - s;
    for (int64_t k = 0; k < m; ++k) {
      const float v = val ? val[s + k] : 1.0f;
      const float *xr = x + (int64_t)col[s + k] * F;
      for (int64_t f = 0; f < F; ++f) scratch[k * F + f] = v * xr[f];
    }
    for (int64_t f = 0; f < F; ++f) {
      out[f] = (m == 1) ? scratch[f] : scratch[f] + pw(scratch + F + f, m - 1, F);
    }
  }
}
