/* Plain-C restatement of the reference's integer products -- TEST
 * INFRASTRUCTURE ONLY (the fast checker at BASELINE sizes; never linked into
 * the product).
 *   oracle_db_matvec:  b[c] = sum_i db[i][c] * qu[i] mod 2^32
 *                      (ServerGlobalState.db_matvec, protocol.py:242-257)
 *   oracle_hint_cols:  H[j][k] = -(sum_i db[i][cols[j]] * A[i][k]) mod 2^32
 *                      (_global_hint_fast/_slow, protocol.py:195-217)
 * uint32 wrapping arithmetic is exact mod 2^32 (= mod q for q = 2^32). */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

void oracle_db_matvec(const uint8_t* db, int64_t d0, int64_t d1, const uint32_t* qu, uint32_t* b) {
  const int64_t BS = 1024;
#pragma omp parallel for schedule(static)
  for (int64_t c0 = 0; c0 < d1; c0 += BS) {
    const int64_t c1 = c0 + BS < d1 ? c0 + BS : d1;
    uint32_t acc[1024];
    memset(acc, 0, sizeof(acc));
    for (int64_t i = 0; i < d0; ++i) {
      const uint8_t* row = db + i * d1;
      const uint32_t q = qu[i];
      for (int64_t c = c0; c < c1; ++c) acc[c - c0] += (uint32_t)row[c] * q;
    }
    for (int64_t c = c0; c < c1; ++c) b[c] = acc[c - c0];
  }
}

void oracle_hint_cols(const uint8_t* db, int64_t d0, int64_t d1, const uint32_t* A, int64_t n,
                      const int64_t* cols, int64_t ncols, uint32_t* H) {
#pragma omp parallel for schedule(dynamic)
  for (int64_t j = 0; j < ncols; ++j) {
    uint32_t* h = H + j * n;
    memset(h, 0, (size_t)n * 4);
    const int64_t c = cols[j];
    for (int64_t i = 0; i < d0; ++i) {
      const uint32_t v = db[i * d1 + c];
      if (!v) continue;
      const uint32_t* a = A + i * n;
      for (int64_t k = 0; k < n; ++k) h[k] += v * a[k];
    }
    for (int64_t k = 0; k < n; ++k) h[k] = 0u - h[k];
  }
}

/* H rows [c_lo, c_hi) of -(db^T A) mod 2^32 (same restatement as
 * oracle_hint_cols), cache-blocked 64 DB rows at a time so the whole 1 GiB
 * global hint is a checker of seconds, not hours. */
__attribute__((target_clones("avx2", "default")))
void oracle_hint_rows(const uint8_t* db, int64_t d0, int64_t d1, const uint32_t* A, int64_t n,
                      int64_t c_lo, int64_t c_hi, uint32_t* H) {
  const int64_t BS = 64;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t c0 = c_lo; c0 < c_hi; c0 += BS) {
    const int64_t c1 = c0 + BS < c_hi ? c0 + BS : c_hi;
    uint32_t* h = H + (c0 - c_lo) * n;
    memset(h, 0, (size_t)(c1 - c0) * n * 4);
    for (int64_t i = 0; i < d0; ++i) {
      const uint8_t* row = db + i * d1;
      const uint32_t* a = A + i * n;
      for (int64_t c = c0; c < c1; ++c) {
        const uint32_t v = row[c];
        if (!v) continue;
        uint32_t* hc = h + (c - c0) * n;
        for (int64_t k = 0; k < n; ++k) hc[k] += v * a[k];
      }
    }
    for (int64_t j = 0; j < (c1 - c0) * n; ++j) h[j] = 0u - h[j];
  }
}
