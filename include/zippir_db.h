/* Handle-level C ABI of libzpir_b200.so: HOST buffers in and out.
 *
 * This is the minimum export set of SURVEY.md section 8(b) -- what a
 * non-Python caller (or the reference's own code through ctypes, see
 * INTEGRATION.md) binds to replace the server hot path without managing
 * device memory, streams or Montgomery constants itself:
 *
 *   (1) zpir_db_create / zpir_db_destroy   DB handle from host u8 (d0, d1)
 *   (2) zpir_db_matvec (nvec = 1)          b = db^T qu mod q
 *   (3) zpir_db_matvec (nvec > 1)          B = db^T Q  mod q (batched queries)
 *   (4) zpir_db_global_hint                H = -db^T A mod q
 *   (5) zpir_db_answer                     t_g = (bs_g + hv_g) mod m
 *       zpir_db_answer_combined            K_g = Enc~(t_g) * k_g mod m^2
 *   (6) zpir_montmul_batch                 a_i * b_i mod N
 *   (7) zpir_multiexp_batch                prod_k bases_k^e(g,k) mod N
 *   (8) zpir_db_update_rows                replace db columns, refresh H rows
 *   +   zpir_db_client_hint                k_g = prod_k ck_r[k]^H_scaled[g][k] mod m^2
 *
 * Conventions: every pointer argument is HOST memory (pageable is fine;
 * copies are staged internally), big integers are little-endian u32 limb
 * rows of the stated width, matrices are row-major. Status codes and
 * zpir_last_error() as in zippir_b200.h (1 = bad input -> ValueError,
 * 2 = CUDA failure, 3 = unsupported width). Calls on one handle are
 * serialised by a per-handle lock; different handles (and the device-pointer
 * ABI) may be used concurrently from any thread. The calling thread's
 * current CUDA device is preserved.
 */
#ifndef ZIPPIR_DB_H
#define ZIPPIR_DB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct zpir_db zpir_db;

/* ProtocolParams (protocol.py:40-95) as the device path needs them. */
typedef struct zpir_db_params {
  int64_t d0;          /* records: db has d0 rows */
  int64_t d1;          /* record size: db has d1 columns (= DB rows of DB = db^T) */
  int64_t n;           /* LWE dimension */
  int32_t log2q;       /* q = 2^log2q, 1 <= log2q <= 32 */
  int32_t p;           /* plaintext modulus: every db symbol must be < p */
  int32_t cap;         /* slots per group (ProtocolParams.capacity, protocol.py:66-78) */
  int32_t gamma_bits;  /* bit length of the batch scale gamma (<= 256) */
  uint32_t gamma[8];   /* gamma (compress.py:36-43) as LE u32 words */
  int32_t device;      /* CUDA device ordinal */
  int32_t engine;      /* 0 = tcgen05 tensor cores (default), 1 = CUDA cores */
} zpir_db_params;

/* (1) Build the device state from a host db (d0 x ld_db bytes, first d1 used):
 * transposed u8 DB, public matrix A and the global hint H. A is either a
 * host (d0 x n) u32 array or NULL, in which case it is generated on the
 * device from the 16-byte a_seed exactly as ProtocolParams.public_matrix
 * (protocol.py:91-95, prg.py:23-57). Replaces ServerGlobalState.__init__
 * (protocol.py:162-193). ValueError cases as the reference: shape, symbol
 * >= p (protocol.py:166-169). */
int zpir_db_create(const zpir_db_params* params, const uint8_t* db, int64_t ld_db,
                   const uint32_t* A, const uint8_t* a_seed, zpir_db** out);
int zpir_db_destroy(zpir_db* h);

/* groups = d1' = ceil(d1 / cap); rows = padded DB rows on the device. */
int zpir_db_info(const zpir_db* h, int64_t* groups, int64_t* rows);

/* (4) H (d1 x n) u32 = -db^T A mod q (protocol.py:195-217). */
int zpir_db_global_hint(zpir_db* h, uint32_t* H);

/* (2)/(3) b[v*d1 + c] = sum_i db[i,c] qu[v*d0 + i] mod q for v < nvec
 * (protocol.py:242-257; nvec > 1 is the batched GEMM, 64 vectors per pass). */
int zpir_db_matvec(zpir_db* h, const uint32_t* qu, int64_t nvec, uint32_t* b);

/* (5) One online answer, SEPARATE mode: t (groups x L) with
 * t_g = (scaled_b(b)_g + sum_k H_scaled[g][k] ck_o[k]) mod m, b = db_matvec(qu)
 * (protocol.py:333-351; rns.rns_matmul_mod rns.py:163-188). qu: d0 u32;
 * ck_o: n x L limbs (< m); m: L limbs (odd). */
int zpir_db_answer(zpir_db* h, const uint32_t* qu, const uint32_t* ck_o, const uint32_t* m, int L,
                   uint32_t* t);

/* COMBINED mode: K (groups x 2L) = ((1 + t_g m) mod m^2) k_g mod m^2 for the
 * stored hint entries k (groups x 2L limbs) (protocol.py:352-358). */
int zpir_db_answer_combined(zpir_db* h, const uint32_t* qu, const uint32_t* ck_o,
                            const uint32_t* m, int L, const uint32_t* k, uint32_t* K);

/* Per-client hint for one query index: k (groups x 2L) with
 * k_g = prod_k ck_r[k]^H_scaled[g][k] mod m^2 and
 * ck_r[k] = Stream(seed, 1, (query_index << 32) | k).below(m^2), sampled on
 * the device (protocol.py:285-296, paillier.py:134-208). */
int zpir_db_client_hint(zpir_db* h, const uint32_t* m, int L, const uint8_t* seed,
                        int64_t seed_len, uint64_t query_index, uint32_t* k);

/* (8) Replace db columns cols[i] (= DB rows) with values[i*d0 .. +d0) and
 * recompute only those rows of H. Afterwards the handle equals a fresh
 * zpir_db_create on the updated db (server.py:115-124 rebuilds everything). */
int zpir_db_update_rows(zpir_db* h, const int64_t* cols, int64_t count, const uint8_t* values);

/* (6) out[i] = a[i] * b[i] mod N, count rows of L limbs, a, b < N, N odd
 * (paillier.add, paillier.py:120-123). */
int zpir_montmul_batch(const uint32_t* a, const uint32_t* b, int64_t count, const uint32_t* N,
                       int L, uint32_t* out, int device);

/* (7) out[g] (L limbs) = prod_k bases[k]^e(g,k) mod N for g < rows;
 * bases n x L (< N), exponents rows x n x Le limbs; all-zero rows give 1
 * (paillier.multiexp / paillier_matmul, paillier.py:134-203). */
int zpir_multiexp_batch(const uint32_t* bases, int64_t n, const uint32_t* exps, int64_t rows,
                        int Le, const uint32_t* N, int L, uint32_t* out, int device);

#ifdef __cplusplus
}
#endif

#endif /* ZIPPIR_DB_H */
