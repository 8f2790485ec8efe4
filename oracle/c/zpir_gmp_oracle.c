/* GMP-backed restatement of the reference's big-integer server arithmetic --
 * TEST INFRASTRUCTURE ONLY (the checker at BASELINE sizes, where the Python
 * restatement in oracle/ref.py would take hours). Never linked into the
 * product. Links libgmp.so.10 (GMP 6.3, the library gmpy2 wraps -- the
 * reference's pinned big-integer dependency, pyproject.toml:10-14); the image
 * ships no gmp.h, so the few mpz entry points used are declared here.
 *
 *   oracle_gmp_multiexp:  prod_k bases[k]^exps[r][k] mod M for every row r,
 *                         by the reference's own algorithm: w = 6-bit windows
 *                         (w = maxbits below 7), buckets 1..2^w-1, running-sum
 *                         combine, w squarings between windows; 1 when every
 *                         exponent is zero (paillier.py:134-193); rows in
 *                         parallel (OpenMP) -- paillier_matmul, :196-203
 *   oracle_gmp_answer_t:  t_g = (sum_j gamma^j (b_c + y_c)) mod m with
 *                         y_c = sum_k H[c][k] ck_o[k], c = g cap + j
 *                         (protocol.py:343-350; identity of SURVEY 8c(ii),
 *                         pinned against the reference by the golden t)
 *   oracle_gmp_combine:   K_g = ((1 + (t_g mod m) m) mod m^2) k_g mod m^2
 *                         (protocol.py:354-358, paillier.py:104-106, :120-123)
 * All big integers cross the boundary as little-endian u32 limb rows. */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned long mp_limb_t;
typedef struct {
  int _mp_alloc;
  int _mp_size;
  mp_limb_t* _mp_d;
} mpz_struct;
typedef mpz_struct mpz_t[1];

extern void __gmpz_init(mpz_struct*);
extern void __gmpz_clear(mpz_struct*);
extern void __gmpz_set(mpz_struct*, const mpz_struct*);
extern void __gmpz_set_ui(mpz_struct*, unsigned long);
extern void __gmpz_mul(mpz_struct*, const mpz_struct*, const mpz_struct*);
extern void __gmpz_mod(mpz_struct*, const mpz_struct*, const mpz_struct*);
extern void __gmpz_add(mpz_struct*, const mpz_struct*, const mpz_struct*);
extern void __gmpz_addmul_ui(mpz_struct*, const mpz_struct*, unsigned long);
extern void __gmpz_import(mpz_struct*, size_t, int, size_t, int, size_t, const void*);
extern void* __gmpz_export(void*, size_t*, int, size_t, int, size_t, const mpz_struct*);
extern size_t __gmpz_sizeinbase(const mpz_struct*, int);
extern int __gmpz_cmp_ui(const mpz_struct*, unsigned long);

static void from_limbs(mpz_struct* z, const uint32_t* limbs, int64_t L) {
  __gmpz_import(z, (size_t)L, -1, 4, -1, 0, limbs);
}

/* writes exactly L limbs (zero-padded); returns -1 if z does not fit */
static int to_limbs(uint32_t* out, int64_t L, const mpz_struct* z) {
  memset(out, 0, (size_t)L * 4);
  if (z->_mp_size == 0) return 0;
  size_t need = (__gmpz_sizeinbase(z, 2) + 31) / 32;
  if ((int64_t)need > L) return -1;
  size_t cnt = 0;
  __gmpz_export(out, &cnt, -1, 4, -1, 0, z);
  return 0;
}

static int bitlen_limbs(const uint32_t* e, int64_t L) {
  for (int64_t i = L - 1; i >= 0; --i)
    if (e[i]) return (int)(32 * i + 32 - __builtin_clz(e[i]));
  return 0;
}

static unsigned digit_at(const uint32_t* e, int64_t L, int shift, unsigned mask) {
  int64_t w = shift >> 5;
  int s = shift & 31;
  uint64_t v = 0;
  if (w < L) v = e[w];
  if (w + 1 < L) v |= (uint64_t)e[w + 1] << 32;
  return (unsigned)(v >> s) & mask;
}

int oracle_gmp_multiexp(const uint32_t* bases, int64_t n, int64_t Lb, const uint32_t* exps,
                        int64_t rows, int64_t Le, const uint32_t* mod, int64_t Lm, uint32_t* out,
                        int64_t Lo) {
  int err = 0;
#pragma omp parallel
  {
    mpz_t M, acc, running, total, tmp;
    __gmpz_init(M);
    __gmpz_init(acc);
    __gmpz_init(running);
    __gmpz_init(total);
    __gmpz_init(tmp);
    from_limbs(M, mod, Lm);
    mpz_struct* B = (mpz_struct*)malloc(sizeof(mpz_struct) * (size_t)n);
    mpz_struct* bk = (mpz_struct*)malloc(sizeof(mpz_struct) * 64);
    char* have = (char*)malloc(64);
    for (int64_t k = 0; k < n; ++k) {
      __gmpz_init(&B[k]);
      from_limbs(&B[k], bases + k * Lb, Lb);
    }
    for (int i = 0; i < 64; ++i) __gmpz_init(&bk[i]);
#pragma omp for schedule(dynamic, 1)
    for (int64_t r = 0; r < rows; ++r) {
      const uint32_t* E = exps + r * n * Le;
      int maxbits = 0;
      for (int64_t k = 0; k < n; ++k) {
        int b = bitlen_limbs(E + k * Le, Le);
        if (b > maxbits) maxbits = b;
      }
      if (maxbits == 0) {
        __gmpz_set_ui(acc, 1);
      } else {
        const int w = maxbits > 6 ? 6 : maxbits;
        const int nwin = (maxbits + w - 1) / w;
        const unsigned mask = (1u << w) - 1;
        int acc_one = 1;
        for (int win = nwin - 1; win >= 0; --win) {
          if (!acc_one)
            for (int s = 0; s < w; ++s) {
              __gmpz_mul(tmp, acc, acc);
              __gmpz_mod(acc, tmp, M);
            }
          memset(have, 0, 64);
          for (int64_t k = 0; k < n; ++k) {
            unsigned d = digit_at(E + k * Le, Le, win * w, mask);
            if (!d) continue;
            if (!have[d]) {
              __gmpz_set(&bk[d], &B[k]);
              have[d] = 1;
            } else {
              __gmpz_mul(tmp, &bk[d], &B[k]);
              __gmpz_mod(&bk[d], tmp, M);
            }
          }
          int run_set = 0, tot_set = 0;
          for (int d = (int)mask; d >= 1; --d) {
            if (have[d]) {
              if (!run_set) {
                __gmpz_set(running, &bk[d]);
                run_set = 1;
              } else {
                __gmpz_mul(tmp, running, &bk[d]);
                __gmpz_mod(running, tmp, M);
              }
            }
            if (run_set) {
              if (!tot_set) {
                __gmpz_set(total, running);
                tot_set = 1;
              } else {
                __gmpz_mul(tmp, total, running);
                __gmpz_mod(total, tmp, M);
              }
            }
          }
          if (tot_set) {
            if (acc_one) {
              __gmpz_set(acc, total);
              acc_one = 0;
            } else {
              __gmpz_mul(tmp, acc, total);
              __gmpz_mod(acc, tmp, M);
            }
          }
        }
        if (acc_one) __gmpz_set_ui(acc, 1);
        __gmpz_mod(tmp, acc, M);
        __gmpz_set(acc, tmp);
      }
      if (to_limbs(out + r * Lo, Lo, acc)) {
#pragma omp atomic write
        err = -1;
      }
    }
    for (int64_t k = 0; k < n; ++k) __gmpz_clear(&B[k]);
    for (int i = 0; i < 64; ++i) __gmpz_clear(&bk[i]);
    free(B);
    free(bk);
    free(have);
    __gmpz_clear(M);
    __gmpz_clear(acc);
    __gmpz_clear(running);
    __gmpz_clear(total);
    __gmpz_clear(tmp);
  }
  return err;
}

int oracle_gmp_answer_t(const uint32_t* H, const uint32_t* b, int64_t d1, int64_t n,
                        const uint32_t* cko, int64_t Lc, const uint32_t* m, int64_t Lm,
                        const uint32_t* gamma, int64_t Lg, int64_t cap, uint32_t* t, int64_t Lt) {
  const int64_t groups = (d1 + cap - 1) / cap;
  int err = 0;
#pragma omp parallel
  {
    mpz_t Mz, G, acc, y, tmp;
    __gmpz_init(Mz);
    __gmpz_init(G);
    __gmpz_init(acc);
    __gmpz_init(y);
    __gmpz_init(tmp);
    from_limbs(Mz, m, Lm);
    from_limbs(G, gamma, Lg);
    mpz_struct* C = (mpz_struct*)malloc(sizeof(mpz_struct) * (size_t)n);
    for (int64_t k = 0; k < n; ++k) {
      __gmpz_init(&C[k]);
      from_limbs(&C[k], cko + k * Lc, Lc);
    }
#pragma omp for schedule(dynamic, 1)
    for (int64_t g = 0; g < groups; ++g) {
      const int64_t lo = g * cap;
      const int64_t hi = lo + cap < d1 ? lo + cap : d1;
      __gmpz_set_ui(acc, 0);
      for (int64_t c = hi - 1; c >= lo; --c) {     /* Horner in gamma, top slot first */
        __gmpz_set_ui(y, b[c]);
        const uint32_t* hc = H + c * n;
        for (int64_t k = 0; k < n; ++k)
          if (hc[k]) __gmpz_addmul_ui(y, &C[k], hc[k]);
        __gmpz_mul(tmp, acc, G);
        __gmpz_add(acc, tmp, y);
      }
      __gmpz_mod(tmp, acc, Mz);
      if (to_limbs(t + g * Lt, Lt, tmp)) {
#pragma omp atomic write
        err = -1;
      }
    }
    for (int64_t k = 0; k < n; ++k) __gmpz_clear(&C[k]);
    free(C);
    __gmpz_clear(Mz);
    __gmpz_clear(G);
    __gmpz_clear(acc);
    __gmpz_clear(y);
    __gmpz_clear(tmp);
  }
  return err;
}

int oracle_gmp_combine(const uint32_t* t, int64_t Lt, const uint32_t* k, int64_t Lk, int64_t groups,
                       const uint32_t* m, int64_t Lm, uint32_t* K, int64_t LK) {
  int err = 0;
  mpz_t Mz, M2, x, y, tmp;
  __gmpz_init(Mz);
  __gmpz_init(M2);
  __gmpz_init(x);
  __gmpz_init(y);
  __gmpz_init(tmp);
  from_limbs(Mz, m, Lm);
  __gmpz_mul(M2, Mz, Mz);
  for (int64_t g = 0; g < groups; ++g) {
    from_limbs(x, t + g * Lt, Lt);
    __gmpz_mod(tmp, x, Mz);
    __gmpz_mul(x, tmp, Mz);
    __gmpz_set_ui(tmp, 1);
    __gmpz_add(y, x, tmp);
    __gmpz_mod(x, y, M2);            /* trivial_encrypt(t) = 1 + t m mod m^2 */
    from_limbs(y, k + g * Lk, Lk);
    __gmpz_mul(tmp, x, y);
    __gmpz_mod(x, tmp, M2);
    if (to_limbs(K + g * LK, LK, x)) err = -1;
  }
  __gmpz_clear(Mz);
  __gmpz_clear(M2);
  __gmpz_clear(x);
  __gmpz_clear(y);
  __gmpz_clear(tmp);
  return err;
}
