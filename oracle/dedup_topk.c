/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into or called by the product path.
 *
 * Plain-C restatement of the reference's native proof kernel
 *   /root/reference/pkg/src/symgrad/_dtkpcore.pyx:17-96  (dedup_topk)
 * with the same argument meaning and byte layout:
 *   member u8 [M][R][I], present u8 [M][R], p f64 [M][I]  ->
 *   out_member u8 [M][k][I], out_present u8 [M][k]   (caller zero-initialises outputs)
 * Per segment m: skip absent rows; pack the row's nonzero bytes into 64-bit words and
 * multiply p[m][j] over member columns in ascending j (pyx:51-57); drop rows whose packed
 * words equal an earlier kept row (first occurrence wins, pyx:58-72); select up to k rows
 * by probability descending, original row index ascending on exact ties (pyx:74-94);
 * copy the selected source rows' bytes (pyx:91-94).
 * Parity pinned against the compiled reference and tests/golden (see tests/test_oracle.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int oracle_dedup_topk(const uint8_t* member, const uint8_t* present, const double* p, int64_t M, int64_t R,
                      int64_t I, int64_t k, uint8_t* out_member, uint8_t* out_present) {
  if (M <= 0 || R <= 0 || k <= 0) return 0;
  const int64_t W = (I + 63) >> 6;
  const int64_t WW = W > 0 ? W : 1;
  uint64_t* words = (uint64_t*)calloc((size_t)(R * WW), sizeof(uint64_t));
  double* probs = (double*)calloc((size_t)R, sizeof(double));
  int64_t* idx = (int64_t*)calloc((size_t)R, sizeof(int64_t));
  if (!words || !probs || !idx) {
    free(words);
    free(probs);
    free(idx);
    return -1;
  }
  for (int64_t m = 0; m < M; ++m) {
    int64_t nd = 0;
    for (int64_t r = 0; r < R; ++r) {
      if (!present[m * R + r]) continue;
      uint64_t* wr = words + nd * WW;
      memset(wr, 0, (size_t)WW * sizeof(uint64_t));
      double prob = 1.0;
      const uint8_t* row = member + (m * R + r) * I;
      for (int64_t j = 0; j < I; ++j) {
        if (row[j]) {
          wr[j >> 6] |= (uint64_t)1 << (j & 63);
          prob *= p[m * I + j];
        }
      }
      int dup = 0;
      for (int64_t d = 0; d < nd && !dup; ++d) {
        int same = 1;
        for (int64_t w = 0; w < W; ++w) {
          if (words[d * WW + w] != wr[w]) {
            same = 0;
            break;
          }
        }
        dup = same;
      }
      if (dup) continue;
      probs[nd] = prob;
      idx[nd] = r;
      ++nd;
    }
    const int64_t nsel = k < nd ? k : nd;
    for (int64_t a = 0; a < nsel; ++a) {
      int64_t best = a;
      for (int64_t c = a + 1; c < nd; ++c) {
        if (probs[c] > probs[best] || (probs[c] == probs[best] && idx[c] < idx[best])) best = c;
      }
      if (best != a) {
        double tp = probs[a];
        probs[a] = probs[best];
        probs[best] = tp;
        int64_t ti = idx[a];
        idx[a] = idx[best];
        idx[best] = ti;
      }
      out_present[m * k + a] = 1;
      memcpy(out_member + (m * k + a) * I, member + (m * R + idx[a]) * I, (size_t)I);
    }
  }
  free(words);
  free(probs);
  free(idx);
  return 0;
}
