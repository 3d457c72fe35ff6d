/*
 * C restatement of the reference's routing-surrogate kernels — TEST
 * INFRASTRUCTURE ONLY (see oracle/__init__.py). Built by
 * __graft_entry__.build() into oracle/_build/liboracle.so.
 *
 *  oracle_uniform_union_counts   moesim/kernels.py:73-103
 *      per token: partial Fisher-Yates on an identity pool,
 *      j = i + (int)(u * (E - i)), swap, pick pool[i]; pool restored after
 *      the token; per-trial union size.
 *  oracle_weighted_union_counts  moesim/kernels.py:106-145
 *      per token: k sequential weighted draws without replacement with a
 *      running cumulative sum in expert order; round-off fallback picks the
 *      highest-index undrawn expert (kernels.py:133-138).
 *
 * Pinned against outputs of the reference itself (tests/golden/union_counts.npz,
 * produced by tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int oracle_uniform_union_counts(const double* u, int64_t trials, int64_t batch, int64_t k, int64_t E,
                                int64_t* out) {
  int64_t* pool = (int64_t*)malloc(sizeof(int64_t) * (size_t)E);
  int64_t* swaps = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k > 0 ? k : 1));
  int64_t* stamp = (int64_t*)calloc((size_t)E, sizeof(int64_t));
  if (!pool || !swaps || !stamp) return 1;
  for (int64_t e = 0; e < E; ++e) pool[e] = e;
  for (int64_t t = 0; t < trials; ++t) {
    int64_t uni = 0;
    for (int64_t b = 0; b < batch; ++b) {
      const double* ub = u + (t * batch + b) * k;
      for (int64_t i = 0; i < k; ++i) {
        const int64_t j = i + (int64_t)(ub[i] * (double)(E - i));
        swaps[i] = j;
        const int64_t tmp = pool[i];
        pool[i] = pool[j];
        pool[j] = tmp;
        const int64_t e = pool[i];
        if (stamp[e] != t + 1) {
          stamp[e] = t + 1;
          ++uni;
        }
      }
      for (int64_t i = k - 1; i >= 0; --i) {
        const int64_t j = swaps[i];
        const int64_t tmp = pool[i];
        pool[i] = pool[j];
        pool[j] = tmp;
      }
    }
    out[t] = uni;
  }
  free(pool);
  free(swaps);
  free(stamp);
  return 0;
}

int oracle_weighted_union_counts(const double* u, int64_t trials, int64_t batch, int64_t k, int64_t E,
                                 const double* weights, int64_t* out) {
  int64_t* drawn = (int64_t*)malloc(sizeof(int64_t) * (size_t)E);
  int64_t* stamp = (int64_t*)calloc((size_t)E, sizeof(int64_t));
  if (!drawn || !stamp) return 1;
  for (int64_t e = 0; e < E; ++e) drawn[e] = -1;
  double total_w = 0.0;
  for (int64_t e = 0; e < E; ++e) total_w += weights[e];
  for (int64_t t = 0; t < trials; ++t) {
    int64_t uni = 0;
    for (int64_t b = 0; b < batch; ++b) {
      const int64_t tok = t * batch + b;
      const double* ub = u + tok * k;
      double w_rem = total_w;
      for (int64_t i = 0; i < k; ++i) {
        const double target = ub[i] * w_rem;
        double cum = 0.0;
        int64_t sel = -1;
        for (int64_t e = 0; e < E; ++e) {
          if (drawn[e] == tok) continue;
          cum += weights[e];
          if (cum > target) {
            sel = e;
            break;
          }
        }
        if (sel < 0) {
          for (int64_t e = E - 1; e >= 0; --e)
            if (drawn[e] != tok) {
              sel = e;
              break;
            }
        }
        drawn[sel] = tok;
        w_rem -= weights[sel];
        if (stamp[sel] != t + 1) {
          stamp[sel] = t + 1;
          ++uni;
        }
      }
    }
    out[t] = uni;
  }
  free(drawn);
  free(stamp);
  return 0;
}
