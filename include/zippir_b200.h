/* C ABI of the B200-native ZipPIR server hot path (libzpir_b200.so).
 *
 * Plain pointers and sizes only: every buffer argument is DEVICE memory on
 * the current CUDA device, every `stream` is a cudaStream_t passed as void*
 * (NULL = legacy default stream). Limbs are little-endian uint32 words.
 * Every entry point returns 0 on success or a nonzero status
 * (1 = bad input -> Python ValueError, 2 = CUDA failure, 3 = unsupported
 * width); zpir_last_error() returns the calling thread's last message.
 * Nothing throws across this boundary; all entry points are re-entrant
 * (no global mutable state besides the thread-local error string), so the
 * reference's connection threads and hint-worker thread may call them
 * concurrently on their own streams (server.py:215-228, :72-84).
 *
 * The reference (Python, /root/reference/pkg/src/zippir) has no FFI of its
 * own; each function below names the reference code it replaces, and the
 * ctypes binding a maintainer would add is in INTEGRATION.md
 * (paper_2603_09190_b200/_lib.py is that binding).
 */
#ifndef ZIPPIR_B200_H
#define ZIPPIR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZPIR_ABI_VERSION 1

int zpir_abi_version(void);
const char* zpir_last_error(void);

/* Database layout: dbt[c*ld + i] = db[i*ld_src + c] for i < d0, c < d1,
 * zero padding up to rows x ld (rows % 128 == 0, ld % 64 == 0).
 * Replaces the centered float64 copy _dbt_c built in
 * ServerGlobalState.__init__ (protocol.py:190-193). */
int zpir_transpose_db(const uint8_t* db, int64_t d0, int64_t d1, int64_t ld_src,
                      uint8_t* dbt, int64_t rows, int64_t ld, void* stream);

/* Global hint H[c,k] = qmask & -(sum_i dbt[c,i] * A[i,k]), A is (ld x lda)
 * row-major u32 with zero rows >= d0 and zero columns >= n, H is (rows x n).
 * Replaces ServerGlobalState._global_hint_fast / _global_hint_slow
 * (protocol.py:195-217). */
int zpir_global_hint(const uint8_t* dbt, int64_t rows, int64_t ld, const uint32_t* A,
                     int64_t lda, int64_t n, uint32_t* H, uint32_t qmask, void* stream);

/* Online GEMV b = qmask & (dbt * qu) for nvec query vectors qu[v*ld + i]
 * (zero-padded to ld), b[v*rows + c]. workspace: zpir_gemv_workspace_bytes.
 * Replaces ServerGlobalState.db_matvec (protocol.py:242-257). */
int64_t zpir_gemv_workspace_bytes(int64_t ld, int64_t nvec);
int zpir_gemv(const uint8_t* dbt, int64_t rows, int64_t ld, const uint32_t* qu, int64_t nvec,
              uint32_t* b, uint32_t qmask, void* workspace, void* stream);

/* Answer compression, row stage: z[c, 0..lm+4) = sum_k H[c,k] * cko[k, 0..lm)
 * exactly (rows % 32 == 0, lm % 32 == 0); b and qmask are accepted for
 * ABI stability and ignored (the group stage adds b).
 * Replaces rns.rns_matmul_mod's residue products (rns.py:163-188). */
int zpir_answer_rows(const uint32_t* H, int64_t rows, int64_t n, const uint32_t* b,
                     uint32_t qmask, const uint32_t* cko, int lm, uint32_t* z, void* stream);

/* Answer compression, group stage:
 * t[g] = (sum_j 2^(32j) ((b[c] & qmask) + z[c])) mod m, c = g*cap + j < d1;
 * m given as lm limbs with np = -m^-1 mod 2^32 and rpow[s] = R^(s+1) mod m
 * (R = 2^(32 lm)) for s < nchunks (2 or 3); fast0 = 1 iff R < 2m. t rows
 * have stride t_ld (zero-extended). Replaces Garner reconstruction +
 * scaled_b + the final add (rns.py:94-127, protocol.py:259-269, :349-350)
 * for gamma = q = 2^32. */
int zpir_answer_groups(const uint32_t* z, const uint32_t* b, uint32_t qmask, int64_t d1, int cap,
                       int64_t groups, int lm, const uint32_t* m, uint32_t np,
                       const uint32_t* rpow, int nchunks, int fast0, uint32_t* t, int64_t t_ld,
                       void* stream);

/* COMBINED response K[g] = (1 + t[g] m) k[g] mod m^2; m^2 as l2 limbs with
 * np2, r2 = R^2 mod m^2, mr = m R mod m^2 (R = 2^(32 l2)); t zero-extended
 * to l2 limbs. Replaces the trivial_encrypt + add loop of respond()
 * (protocol.py:354-358; paillier.py:104-106, :120-123). */
int zpir_combine(const uint32_t* t, const uint32_t* k, int64_t groups, int l2,
                 const uint32_t* m2, uint32_t np2, const uint32_t* r2, const uint32_t* mr,
                 uint32_t* out, void* stream);

/* out[i] = a[i] * b[i] mod N (canonical), limbs % 32 == 0, r2 = R^2 mod N.
 * Batched paillier.add (paillier.py:120-123). */
int zpir_mulmod(const uint32_t* a, const uint32_t* b, int64_t count, int limbs, const uint32_t* N,
                uint32_t np, const uint32_t* r2, uint32_t* out, void* stream);

/* Multi-exponentiation out[g] = prod_k bases[k]^{e(g,k)} mod N for rows g,
 * bases (n x limbs, canonical < N), exponent limb j of (g,k) at
 * exps[g*row_stride + k*base_stride + j*limb_stride], j < elimbs.
 * Replaces paillier.multiexp / paillier_matmul (paillier.py:134-203), as
 * called by protocol.hint (protocol.py:291-296). */
int64_t zpir_multiexp_workspace_bytes(int64_t n, int64_t rows, int elimbs, int limbs);
int zpir_multiexp(const uint32_t* bases, int64_t n, const uint32_t* exps, int64_t rows,
                  int64_t row_stride, int64_t base_stride, int64_t limb_stride, int elimbs,
                  int limbs, const uint32_t* N, uint32_t np, const uint32_t* r2, uint32_t* out,
                  void* workspace, int64_t ws_bytes, void* stream);

/* ---- tcgen05 (UMMA kind::i8) engine -------------------------------------
 * Query byte planes: planes[(4v+l)*ld + i] = byte l of qu[v*ld + i], rows
 * 4*nvec .. prow-1 zeroed (prow = 16 for nvec <= 4, 256 for nvec <= 64). */
int zpir_query_planes(const uint32_t* qu, int64_t ld, int64_t nvec, uint8_t* planes, int64_t prow,
                      void* stream);

/* b[v*rows + r] = (dbt * qu_v)[r] mod 2^32 on the tensor cores (stream-K
 * split, wrapping atomics). Same contract as zpir_gemv (protocol.py:242-257),
 * planes from zpir_query_planes. nvec <= 64 (batched queries). ctas caps the
 * persistent grid (0 = one CTA per SM) so the compression GEMM can run
 * concurrently on the remaining SMs. */
int zpir_umma_gemv(const uint8_t* dbt, int64_t rows, int64_t ld, const uint8_t* planes,
                   int64_t nvec, uint32_t* b, int ctas, void* stream);

/* A byte planes: aplanes[(4k+l)*ld + i] = byte l of A[i*lda + k]. */
int zpir_build_aplanes(const uint32_t* A, int64_t ld, int64_t lda, int64_t n, uint8_t* aplanes,
                       void* stream);

/* Global hint on the tensor cores, H[r*n + k] = qmask & -(dbt A)[r,k]
 * (protocol.py:195-217); n % 64 == 0. */
int zpir_umma_global_hint(const uint8_t* dbt, int64_t rows, int64_t ld, const uint8_t* aplanes,
                          int64_t n, uint32_t* H, uint32_t qmask, void* stream);

/* Compression operand: bc[b*4n + 4k + a] = byte (b-a) of ck_o[k], b < nb
 * (nb = 16*ceil((4 lm + 3)/16): 144 / 272 / 400 for lm = 32 / 64 / 96). */
int zpir_build_bc(const uint32_t* cko, int64_t n, int lm, int nb, uint8_t* bc, void* stream);

/* Row stage of the answer compression on the tensor cores: same contract as
 * zpir_answer_rows (b unused) with wz = lm + 4 (rns.py:163-188 replacement). */
int zpir_umma_answer_rows(const uint32_t* H, int64_t rows, int64_t n, const uint8_t* bc, int nb,
                          const uint32_t* b, uint32_t qmask, int wz, uint32_t* z, int ctas,
                          void* stream);

/* ---- planar compression (default for lm = 32 / 64) ------------------------
 * H byte planes: hp[r*4np + a*np + k] = byte a of H[r*n + k], np = n rounded up
 * to 128 (zero padded); built once per DB version. */
int zpir_h_planes(const uint32_t* H, int64_t rows, int64_t n, uint8_t* hp, void* stream);
/* ck_o byte rows for nq queries: bp[q*(4 lm)*np + j*np + k] = byte j of cko[q][k]. */
int zpir_build_bcp(const uint32_t* cko, int64_t n, int lm, int nq, uint8_t* bp, void* stream);
/* z[q*rows*wz + r*wz + i] = limbs of sum_k H[r,k] * ck_q[k] (wz = lm + 4), as
 * zpir_umma_answer_rows, via z = sum_a 2^(8a) sum_j 2^(8j) (Hp_a Bp^T)[r, j]: one
 * N = 4 lm tcgen05 MMA per 32-byte k-step, four plane passes per tile
 * (rns.py:163-188 replacement); lm in {32, 64}, n <= 33025. */
int zpir_umma_answer_rows_planar(const uint8_t* hp, int64_t rows, int64_t n, const uint8_t* bp,
                                 int lm, int nq, int wz, uint32_t* z, int ctas, void* stream);

/* ---- batched queries (BASELINE configs[3]; no reference counterpart: the
 * reference answers strictly one query at a time, protocol.py:333) ---------
 * nq stacked compression operands (nq x nb x 4n bytes) from nq ck_o limb rows. */
int zpir_build_bc_batch(const uint32_t* cko, int64_t n, int lm, int nb, int nq, uint8_t* bc,
                        void* stream);
/* z[q*rows*wz + r*wz + i] for nq queries in one tcgen05 launch (H tiles are
 * reused from L2 across the queries of a row block). */
int zpir_umma_answer_rows_batch(const uint32_t* H, int64_t rows, int64_t n, const uint8_t* bc,
                                int nb, int nq, int wz, uint32_t* z, void* stream);
/* Group stage for nq queries: z / b strides zq / bq, per-query modulus limbs
 * mods[q*lm], n' nps[q], R-power tables rpows[q*nchunks*lm], fast0s[q];
 * t[q*groups*t_ld + g*t_ld]. */
int zpir_answer_groups_batch(const uint32_t* z, int64_t zq, const uint32_t* b, int64_t bq,
                             uint32_t qmask, int64_t d1, int cap, int64_t groups, int lm,
                             const uint32_t* mods, const uint32_t* nps, const uint32_t* rpows,
                             int nchunks, const uint8_t* fast0s, uint32_t* t, int64_t t_ld, int nq,
                             int stride, void* stream);

/* Split group stage (lets the Montgomery work overlap the GEMV):
 * tz[q][g] = (sum_j 2^(32j) z[c]) mod m_q  -- needs only the compression output;
 * t[q][g]  = (tz[q][g] + sum_j 2^(32j) (b[q][c] & qmask)) mod m_q -- after the
 * GEMV; exact because sum_j 2^(32j) b_c < gamma^cap < m (protocol.py:66-78).
 * Same per-query arrays as zpir_answer_groups_batch; tz and t share t_ld.
 * stride = slot stride in 32-bit limbs (gamma = 2^(32 stride): 1 for the
 * binary-key quarter-delta layout, 2 for the uniform-key one). */
int zpir_groups_z(const uint32_t* z, int64_t zq, int64_t d1, int cap, int64_t groups, int lm,
                  const uint32_t* mods, const uint32_t* nps, const uint32_t* rpows, int nchunks,
                  const uint8_t* fast0s, uint32_t* tz, int64_t t_ld, int nq, int stride,
                  void* stream);
int zpir_groups_finish(const uint32_t* tz, const uint32_t* b, int64_t bq, uint32_t qmask,
                       int64_t d1, int cap, int64_t groups, int lm, const uint32_t* mods,
                       uint32_t* t, int64_t t_ld, int nq, int stride, void* stream);

/* ---- device ChaCha20 streams (prg.py:23-57), key32/iv16 are HOST byte arrays
 * (key = SHA-256(seed), iv = domain || 15-byte LE index) --------------------
 * Public matrix A (protocol.py:91-95): out[r*ld + c] = mask & low32(u64 word
 * r*cols + c) of the stream. */
int zpir_chacha_words32(const uint8_t* key32, const uint8_t* iv16, int64_t rows, int64_t cols,
                        uint32_t* out, int64_t ld, uint32_t mask, void* stream);
/* ck_r (paillier.py:206-208, protocol.py:285-288): out[k] = Stream(seed, domain,
 * (query_index << 32) | k).below(bound) for k < n, as `limbs` u32 limbs;
 * bits = bitlen(bound - 1); bound is a device limb array. */
int zpir_chacha_below(const uint8_t* key32, uint32_t domain, uint64_t query_index, int64_t n,
                      const uint32_t* bound, int limbs, int bits, uint32_t* out, void* stream);

/* Python-int boundary helpers: regroup CPython's 30-bit digits (copied raw by
 * the host) into 32-bit limbs and back (limbs rows have stride ld). */
int zpir_digits_to_limbs(const uint32_t* digits, int64_t count, int ndig, uint32_t* limbs, int nl,
                         void* stream);
int zpir_limbs_to_digits(const uint32_t* limbs, int64_t count, int nl, int64_t ld,
                         uint32_t* digits, int ndig, void* stream);

/* ---- slot-decomposed hints and incremental DB update (BASELINE configs[4];
 * the reference rebuilds everything on update, server.py:115-124) ---------
 * Multiexp over an explicit list of exponent rows (row_ids, nullable = 0..rows-1);
 * out[row_ids[i]] gets row i's product, kept in Montgomery form when keep_mont
 * (all-zero rows then get one_m = R mod N). */
int zpir_multiexp_rows(const uint32_t* bases, int64_t n, const uint32_t* exps,
                       const int32_t* row_ids, int64_t rows, int64_t row_stride,
                       int64_t base_stride, int64_t limb_stride, int elimbs, int limbs,
                       const uint32_t* N, uint32_t np, const uint32_t* r2, const uint32_t* one_m,
                       int keep_mont, uint32_t* out, void* workspace, int64_t ws_bytes,
                       void* stream);
/* k[g] = prod_j W[g*cap + j]^(gamma^j) mod N (W in Montgomery form; k canonical)
 * for the groups in group_ids (nullable = all ngroups), by Horner in gamma
 * (gamma = HOST array of ceil(gamma_bits/32) u32 words, gamma_bits <= 256; for
 * gamma = 2^32 that is 32 squarings per slot): the hint entry
 * k_g = prod_k ck_r[k]^H_scaled[g][k] (paillier.py:134-203) rebuilt from its
 * per-DB-row factors W[c] = prod_k ck_r[k]^H[c][k]. */
int zpir_slot_combine(const uint32_t* W, int cap, const int32_t* group_ids, int64_t ngroups,
                      int limbs, const uint32_t* N, uint32_t np, const uint32_t* gamma,
                      int gamma_bits, uint32_t* out, void* stream);
/* zpir_slot_combine for `clients` keys of the same width in one launch (host
 * arrays of device pointers W / N / out and of n' values; shared group ids):
 * the hint worker's batch (protocol.hints). */
int zpir_slot_combine_many(int clients, const uint32_t* const* W, const uint32_t* const* N,
                           const uint32_t* np, uint32_t* const* out, int cap,
                           const int32_t* group_ids, int64_t ngroups, int limbs,
                           const uint32_t* gamma, int gamma_bits, void* stream);
/* Group stage for a general batch scale gamma (not 2^32 / 2^64):
 * t[g] = sum_j (gamma^j mod m) ((b[c] & qmask) + z[c]) mod m, with
 * ctab[j] = {gamma^j R mod m, gamma^j R^2 mod m} (lm limbs each) and w a
 * workspace of d1 x lm limbs (protocol.py:219-238, :259-269 generic paths). */
int zpir_answer_general(const uint32_t* z, const uint32_t* b, uint32_t qmask, int64_t d1, int cap,
                        int64_t groups, int lm, const uint32_t* m, uint32_t np,
                        const uint32_t* ctab, uint32_t* w, uint32_t* t, int64_t t_ld,
                        void* stream);
/* Fixed-base table for 32-bit exponents: P[i*n + k] = bases[k]^(2^(8 i)) in
 * Montgomery form, i < 4. */
int zpir_pow8_table(const uint32_t* bases, int64_t n, int limbs, const uint32_t* N, uint32_t np,
                    const uint32_t* r2, uint32_t* P, void* stream);
/* W[r] = prod_k bases[k]^exps[r*row_stride + k] (Montgomery form) for the
 * listed rows (row_ids nullable = 0..rows-1), one 255-bucket Pippenger over
 * the 4n byte digits per row using P; all-zero rows get one_m. */
int zpir_slot_fixed(const uint32_t* P, int64_t n, const uint32_t* exps, int64_t row_stride,
                    const int32_t* row_ids, int64_t rows, int limbs, const uint32_t* N,
                    uint32_t np, const uint32_t* one_m, uint32_t* W, void* stream);
/* zpir_slot_fixed for rows 0..rows-1 with the Pippenger bucket updates on the
 * tensor cores (position-major: each position multiplies one bucket per row by
 * the same y = P[pos]; X y mod N = sum_i x_i (y 256^i mod N) over the bytes x_i
 * of X is one int8 GEMM against the table of reduced byte shifts of y, left
 * unreduced in 515 bytes); 4096-bit N only (limbs = 128).
 * P is the pow8 table of zpir_pow8_table (only its first n entries, the
 * Montgomery bases, are read). Transient workspace:
 * zpir_slot_fixed_tc_workspace(n, rows, 1) bytes (~34 KB per row + ~1.7 GB per
 * client at n = 1024). */
int zpir_slot_fixed_tc(const uint32_t* P, int64_t n, const uint32_t* E, int64_t rs, int64_t rows,
                       int limbs, const uint32_t* N, uint32_t np, const uint32_t* one_m,
                       uint32_t* W, void* stream);
/* zpir_slot_fixed_tc for `clients` independent keys in one launch (the hint
 * worker's batch; also the incremental refresh): client c's table P[c]
 * (4n x 128 limbs), N[c] / one_m[c] (128 limbs each) and output
 * rows W[c] are device addresses passed in HOST arrays; np is a host array.
 * Rows r < rows read exponent row e = row_ids ? row_ids[r] : r and write
 * W[c][e]. Replaces paillier.multiexp (paillier.py:134-193) as called by
 * protocol.hint (protocol.py:291-296) for each client of a batch.
 * Transient workspace: zpir_slot_fixed_tc_workspace(n, rows, clients) bytes. */
int zpir_slot_fixed_tc_many(int clients, const uint64_t* P, const uint64_t* N, const uint32_t* np,
                            const uint64_t* one_m, const uint64_t* W, int64_t n,
                            const uint32_t* E, int64_t rs, const int32_t* row_ids, int64_t rows,
                            void* stream);
int64_t zpir_slot_fixed_tc_workspace(int64_t n, int64_t rows, int clients);
/* flags[r] = (row r of a != row r of b), rows of ld bytes. */
int zpir_rows_differ(const uint8_t* a, const uint8_t* b, int64_t rows, int64_t ld, uint32_t* flags,
                     void* stream);
/* Row gather (scatter = 0: dst[i] = src[ids[i]]) / scatter (dst[ids[i]] = src[i]). */
int zpir_move_rows(const uint8_t* src, uint8_t* dst, int64_t pitch, const int32_t* ids,
                   int64_t nrows, int scatter, void* stream);

/* Record a cudaEvent_t on `stream`; inside stream capture as an external
 * event-record node, so timing events around a kernel fire on every replay
 * of the captured graph (bench.py's in-step roofline). */
int zpir_event_record(void* event, void* stream);

/* Make `stream` wait for `event`; inside stream capture as an external
 * event-wait node (the answer's second graph waits for the GEMV graph). */
int zpir_stream_wait_event(void* stream, void* event);
/* cudaGraphLaunch of an instantiated graph (cudaGraphExec_t) on `stream`:
 * the low-overhead replay respond() uses. */
int zpir_graph_launch(void* graph_exec, void* stream);

/* The device address of pinned host memory (cudaHostGetDevicePointer); the
 * zero-copy answer graphs pass host buffers to kernels only where it equals
 * the host address (UVA), else they take the copy-node path. */
int zpir_host_device_pointer(void* host, void** dev);

/* Async pinned-host <-> device copy (kind 0 = H2D, 1 = D2H) on `stream`. */
int zpir_memcpy_async(void* dst, const void* src, int64_t bytes, int kind, void* stream);

/* Residues of the batch-scaled hint matrix modulo a prime basis: the
 * reference's H_rns = rns.matrix_to_rns(basis, H_scaled) (rns.py:148-154,
 * protocol.py:188), built on demand from the device H. Entry (g, k) =
 * sum_{j < cap} 2^(32 stride j) S[g cap + j][k] over the `rows` valid rows of
 * S (rows x n u32); weights[i][j] = 2^(32 stride j) mod primes[i] (count x cap
 * u64); out (count, groups, n) float64. Replaces the host to_rns (rns.py:70-86). */
int zpir_rns_residues(const uint32_t* S, int64_t rows, int64_t n, int cap, int stride,
                      const uint32_t* primes, const uint64_t* weights, int count, int64_t groups,
                      double* out, void* stream);

/* The reference multiexp's group-multiplication count (paillier.py:134-193,
 * counter bump :192) for each hint entry prod_k base_k^E[g][k] with
 * E[g][k] = sum_j 2^(sbits j) S[g cap + j][k] (gamma = 2^sbits, slots below
 * 2^min(sbits, 32)); out: groups int64. Lets the drop-in's counters report
 * what the reference would (golden hint_group_mults). */
int zpir_multiexp_opcount(const uint32_t* S, int64_t rows, int64_t n, int cap, int sbits,
                          int64_t groups, int64_t* out, void* stream);

/* Roofline probe: time `iters` x 16 32-bit IMADs per thread on blocks x 256
 * threads (CUDA events); the IMAD peak the bignum kernels are measured against. */
int zpir_probe_imad(int blocks, int iters, float* ms);
/* Roofline probe: `iters` rounds of 4 tcgen05 kind::i8 MMAs (M = 128, N = n,
 * K = 32) per CTA from resident smem, blocks CTAs; ops = blocks*iters*4*2*128*n*32.
 * The int8 tensor rate the compression / hint GEMMs are measured against. */
int zpir_probe_umma_i8(int blocks, int iters, int n, float* ms);

#ifdef __cplusplus
}
#endif

#endif /* ZIPPIR_B200_H */
