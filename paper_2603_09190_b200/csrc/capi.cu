// extern "C" boundary (include/zippir_b200.h): status codes + thread-local
// error string; no exceptions cross this boundary.
#include <cstdarg>
#include <cstdio>

#include "../../include/zippir_b200.h"
#include "zpir_common.cuh"

namespace zpir {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int transpose_db_launch(const uint8_t*, int64_t, int64_t, int64_t, uint8_t*, int64_t, int64_t,
                        cudaStream_t);
int hint_gemm_launch(const uint8_t*, int64_t, int64_t, const uint32_t*, int64_t, int64_t,
                     uint32_t*, uint32_t, cudaStream_t);
int gemv_launch(const uint8_t*, int64_t, int64_t, const uint32_t*, int64_t, uint32_t*, uint32_t,
                uint32_t*, cudaStream_t);
int answer_rows_launch(const uint32_t*, int64_t, int64_t, const uint32_t*, uint32_t,
                       const uint32_t*, int, uint32_t*, cudaStream_t);
int answer_groups_launch(const uint32_t*, const uint32_t*, uint32_t, int64_t, int, int64_t, int,
                         const uint32_t*, uint32_t, const uint32_t*, int, int, uint32_t*, int64_t,
                         cudaStream_t);
int combine_launch(const uint32_t*, const uint32_t*, int64_t, int, const uint32_t*, uint32_t,
                   const uint32_t*, const uint32_t*, uint32_t*, cudaStream_t);
int mulmod_launch(const uint32_t*, const uint32_t*, int64_t, int, const uint32_t*, uint32_t,
                  const uint32_t*, uint32_t*, cudaStream_t);
int64_t multiexp_workspace_bytes(int64_t, int64_t, int, int);
int multiexp_launch(const uint32_t*, int64_t, const uint32_t*, int64_t, int64_t, int64_t, int64_t,
                    int, int, const uint32_t*, uint32_t, const uint32_t*, uint32_t*, void*,
                    int64_t, cudaStream_t);

int query_planes_launch(const uint32_t*, int64_t, int64_t, uint8_t*, int64_t, cudaStream_t);
int umma_gemv_launch(const uint8_t*, int64_t, int64_t, const uint8_t*, int64_t, uint32_t*, int,
                     cudaStream_t);
int umma_hint_launch(const uint8_t*, int64_t, int64_t, const uint8_t*, int64_t, uint32_t*,
                     uint32_t, cudaStream_t);
int umma_answer_rows_launch(const uint32_t*, int64_t, int64_t, const uint8_t*, int,
                            const uint32_t*, uint32_t, int, uint32_t*, int, cudaStream_t);
int build_bc_launch(const uint32_t*, int64_t, int, int, uint8_t*, cudaStream_t);
int build_aplanes_launch(const uint32_t*, int64_t, int64_t, int64_t, uint8_t*, cudaStream_t);
int imad_probe(int, int, float*);
int rns_residues_launch(const uint32_t*, int64_t, int64_t, int, int, const uint32_t*,
                        const unsigned long long*, int, int64_t, double*, cudaStream_t);
int multiexp_opcount_launch(const uint32_t*, int64_t, int64_t, int, int, int64_t, long long*,
                            cudaStream_t);
int tc_slot_fixed_launch(const uint32_t*, int64_t, const uint32_t*, int64_t, int64_t,
                         const uint32_t*, uint32_t, const uint32_t*, uint32_t*, cudaStream_t);
int tc_slot_fixed_many_launch(int, const uint32_t* const*, const uint32_t* const*, const uint32_t*,
                              const uint32_t* const*, uint32_t* const*, int64_t, const uint32_t*,
                              int64_t, const int32_t*, int64_t, cudaStream_t);
int64_t tc_slot_fixed_workspace(int64_t, int64_t, int);
int h_planes_launch(const uint32_t*, int64_t, int64_t, uint8_t*, cudaStream_t);
int build_bcp_launch(const uint32_t*, int64_t, int, int, uint8_t*, cudaStream_t);
int umma_planar_launch(const uint8_t*, int64_t, int64_t, const uint8_t*, int, int, int, uint32_t*,
                       int, cudaStream_t);
int umma_probe(int, int, int, float*);
int multiexp_rows_launch(const uint32_t*, int64_t, const uint32_t*, const int32_t*, int64_t, int64_t,
                         int64_t, int64_t, int, int, const uint32_t*, uint32_t, const uint32_t*,
                         const uint32_t*, int, uint32_t*, void*, int64_t, cudaStream_t);
int slot_combine_many_launch(int, const uint32_t* const*, const uint32_t* const*, const uint32_t*,
                             uint32_t* const*, int, const int32_t*, int64_t, int, const uint32_t*,
                             int, cudaStream_t);
int slot_combine_launch(const uint32_t*, int, const int32_t*, int64_t, int, const uint32_t*,
                        uint32_t, const uint32_t*, int, uint32_t*, cudaStream_t);
int answer_general_launch(const uint32_t*, const uint32_t*, uint32_t, int64_t, int, int64_t, int,
                          const uint32_t*, uint32_t, const uint32_t*, uint32_t*, uint32_t*, int64_t,
                          cudaStream_t);
int pow8_table_launch(const uint32_t*, int64_t, int, const uint32_t*, uint32_t, const uint32_t*,
                      uint32_t*, cudaStream_t);
int slot_fixed_launch(const uint32_t*, int64_t, const uint32_t*, int64_t, const int32_t*, int64_t,
                      int, const uint32_t*, uint32_t, const uint32_t*, uint32_t*, cudaStream_t);
int groups_z_launch(const uint32_t*, int64_t, int64_t, int, int64_t, int, const uint32_t*,
                    const uint32_t*, const uint32_t*, int, const uint8_t*, uint32_t*, int64_t, int,
                    int, cudaStream_t);
int groups_finish_launch(const uint32_t*, const uint32_t*, int64_t, uint32_t, int64_t, int, int64_t,
                         int, const uint32_t*, uint32_t*, int64_t, int, int, cudaStream_t);
int chacha_words32_launch(const uint8_t*, const uint8_t*, int64_t, int64_t, uint32_t*, int64_t,
                          uint32_t, cudaStream_t);
int chacha_below_launch(const uint8_t*, uint32_t, uint64_t, int64_t, const uint32_t*, int, int,
                        uint32_t*, cudaStream_t);
int digits_to_limbs_launch(const uint32_t*, int64_t, int, uint32_t*, int, cudaStream_t);
int limbs_to_digits_launch(const uint32_t*, int64_t, int, int64_t, uint32_t*, int, cudaStream_t);
int rows_differ_launch(const uint8_t*, const uint8_t*, int64_t, int64_t, uint32_t*, cudaStream_t);
int move_rows_launch(const uint8_t*, uint8_t*, int64_t, const int32_t*, int64_t, int, cudaStream_t);
int build_bc_batch_launch(const uint32_t*, int64_t, int, int, int, uint8_t*, cudaStream_t);
int umma_answer_rows_batch_launch(const uint32_t*, int64_t, int64_t, const uint8_t*, int, int, int,
                                  uint32_t*, cudaStream_t);
int answer_groups_batch_launch(const uint32_t*, int64_t, const uint32_t*, int64_t, uint32_t, int64_t,
                               int, int64_t, int, const uint32_t*, const uint32_t*,
                               const uint32_t*, int, const uint8_t*, uint32_t*, int64_t, int, int,
                               cudaStream_t);

}  // namespace zpir

using namespace zpir;

#define ZPIR_GUARD(expr)                              \
  do {                                                \
    try {                                             \
      return (expr);                                  \
    } catch (...) {                                   \
      set_error("unexpected C++ exception");          \
      return kErrCuda;                                \
    }                                                 \
  } while (0)

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int zpir_abi_version(void) { return ZPIR_ABI_VERSION; }

const char* zpir_last_error(void) { return g_err; }

int zpir_transpose_db(const uint8_t* db, int64_t d0, int64_t d1, int64_t ld_src, uint8_t* dbt,
                      int64_t rows, int64_t ld, void* stream) {
  ZPIR_GUARD(transpose_db_launch(db, d0, d1, ld_src, dbt, rows, ld, S(stream)));
}

int zpir_global_hint(const uint8_t* dbt, int64_t rows, int64_t ld, const uint32_t* A, int64_t lda,
                     int64_t n, uint32_t* H, uint32_t qmask, void* stream) {
  ZPIR_GUARD(hint_gemm_launch(dbt, rows, ld, A, lda, n, H, qmask, S(stream)));
}

int64_t zpir_gemv_workspace_bytes(int64_t ld, int64_t nvec) { return ld * nvec * 4; }

int zpir_gemv(const uint8_t* dbt, int64_t rows, int64_t ld, const uint32_t* qu, int64_t nvec,
              uint32_t* b, uint32_t qmask, void* workspace, void* stream) {
  ZPIR_GUARD(gemv_launch(dbt, rows, ld, qu, nvec, b, qmask, static_cast<uint32_t*>(workspace),
                         S(stream)));
}

int zpir_answer_rows(const uint32_t* H, int64_t rows, int64_t n, const uint32_t* b, uint32_t qmask,
                     const uint32_t* cko, int lm, uint32_t* z, void* stream) {
  ZPIR_GUARD(answer_rows_launch(H, rows, n, b, qmask, cko, lm, z, S(stream)));
}

int zpir_answer_groups(const uint32_t* z, const uint32_t* b, uint32_t qmask, int64_t d1, int cap,
                       int64_t groups, int lm, const uint32_t* m, uint32_t np,
                       const uint32_t* rpow, int nchunks, int fast0, uint32_t* t, int64_t t_ld,
                       void* stream) {
  ZPIR_GUARD(answer_groups_launch(z, b, qmask, d1, cap, groups, lm, m, np, rpow, nchunks, fast0, t,
                                  t_ld, S(stream)));
}

int zpir_combine(const uint32_t* t, const uint32_t* k, int64_t groups, int l2, const uint32_t* m2,
                 uint32_t np2, const uint32_t* r2, const uint32_t* mr, uint32_t* out,
                 void* stream) {
  ZPIR_GUARD(combine_launch(t, k, groups, l2, m2, np2, r2, mr, out, S(stream)));
}

int zpir_mulmod(const uint32_t* a, const uint32_t* b, int64_t count, int limbs, const uint32_t* N,
                uint32_t np, const uint32_t* r2, uint32_t* out, void* stream) {
  ZPIR_GUARD(mulmod_launch(a, b, count, limbs, N, np, r2, out, S(stream)));
}

int64_t zpir_multiexp_workspace_bytes(int64_t n, int64_t rows, int elimbs, int limbs) {
  return multiexp_workspace_bytes(n, rows, elimbs, limbs);
}

int zpir_multiexp(const uint32_t* bases, int64_t n, const uint32_t* exps, int64_t rows,
                  int64_t row_stride, int64_t base_stride, int64_t limb_stride, int elimbs,
                  int limbs, const uint32_t* N, uint32_t np, const uint32_t* r2, uint32_t* out,
                  void* workspace, int64_t ws_bytes, void* stream) {
  ZPIR_GUARD(multiexp_launch(bases, n, exps, rows, row_stride, base_stride, limb_stride, elimbs,
                             limbs, N, np, r2, out, workspace, ws_bytes, S(stream)));
}

int zpir_query_planes(const uint32_t* qu, int64_t ld, int64_t nvec, uint8_t* planes, int64_t prow,
                      void* stream) {
  ZPIR_GUARD(query_planes_launch(qu, ld, nvec, planes, prow, S(stream)));
}

int zpir_umma_gemv(const uint8_t* dbt, int64_t rows, int64_t ld, const uint8_t* planes,
                   int64_t nvec, uint32_t* b, int ctas, void* stream) {
  ZPIR_GUARD(umma_gemv_launch(dbt, rows, ld, planes, nvec, b, ctas, S(stream)));
}

int zpir_build_aplanes(const uint32_t* A, int64_t ld, int64_t lda, int64_t n, uint8_t* aplanes,
                       void* stream) {
  ZPIR_GUARD(build_aplanes_launch(A, ld, lda, n, aplanes, S(stream)));
}

int zpir_umma_global_hint(const uint8_t* dbt, int64_t rows, int64_t ld, const uint8_t* aplanes,
                          int64_t n, uint32_t* H, uint32_t qmask, void* stream) {
  ZPIR_GUARD(umma_hint_launch(dbt, rows, ld, aplanes, n, H, qmask, S(stream)));
}

int zpir_build_bc(const uint32_t* cko, int64_t n, int lm, int nb, uint8_t* bc, void* stream) {
  ZPIR_GUARD(build_bc_launch(cko, n, lm, nb, bc, S(stream)));
}

int zpir_umma_answer_rows(const uint32_t* H, int64_t rows, int64_t n, const uint8_t* bc, int nb,
                          const uint32_t* b, uint32_t qmask, int wz, uint32_t* z, int ctas,
                          void* stream) {
  ZPIR_GUARD(umma_answer_rows_launch(H, rows, n, bc, nb, b, qmask, wz, z, ctas, S(stream)));
}

int zpir_probe_imad(int blocks, int iters, float* ms) { ZPIR_GUARD(imad_probe(blocks, iters, ms)); }

int zpir_slot_fixed_tc(const uint32_t* P, int64_t n, const uint32_t* E, int64_t rs, int64_t rows,
                       int limbs, const uint32_t* N, uint32_t np, const uint32_t* one_m,
                       uint32_t* W, void* stream) {
  if (limbs != 128) {
    set_error("slot_fixed_tc: the tensor-core path is built for 4096-bit N (limbs=%d)", limbs);
    return kErrUnsupported;
  }
  ZPIR_GUARD(tc_slot_fixed_launch(P, n, E, rs, rows, N, np, one_m, W, S(stream)));
}

int zpir_slot_fixed_tc_many(int clients, const uint64_t* P, const uint64_t* N, const uint32_t* np,
                            const uint64_t* one_m, const uint64_t* W, int64_t n,
                            const uint32_t* E, int64_t rs, const int32_t* row_ids, int64_t rows,
                            void* stream) {
  if (!P || !N || !np || !one_m || !W) {
    set_error("slot_fixed_tc_many: null client array");
    return kErrInput;
  }
  ZPIR_GUARD(tc_slot_fixed_many_launch(
      clients, reinterpret_cast<const uint32_t* const*>(P), reinterpret_cast<const uint32_t* const*>(N),
      np, reinterpret_cast<const uint32_t* const*>(one_m), reinterpret_cast<uint32_t* const*>(W), n,
      E, rs, row_ids, rows, S(stream)));
}

int64_t zpir_slot_fixed_tc_workspace(int64_t n, int64_t rows, int clients) {
  return tc_slot_fixed_workspace(n, rows, clients);
}

int zpir_h_planes(const uint32_t* H, int64_t rows, int64_t n, uint8_t* hp, void* stream) {
  ZPIR_GUARD(h_planes_launch(H, rows, n, hp, S(stream)));
}

int zpir_build_bcp(const uint32_t* cko, int64_t n, int lm, int nq, uint8_t* bp, void* stream) {
  ZPIR_GUARD(build_bcp_launch(cko, n, lm, nq, bp, S(stream)));
}

int zpir_umma_answer_rows_planar(const uint8_t* hp, int64_t rows, int64_t n, const uint8_t* bp,
                                 int lm, int nq, int wz, uint32_t* z, int ctas, void* stream) {
  ZPIR_GUARD(umma_planar_launch(hp, rows, n, bp, lm, nq, wz, z, ctas, S(stream)));
}

int zpir_probe_umma_i8(int blocks, int iters, int n, float* ms) {
  ZPIR_GUARD(umma_probe(blocks, iters, n, ms));
}

int zpir_build_bc_batch(const uint32_t* cko, int64_t n, int lm, int nb, int nq, uint8_t* bc,
                        void* stream) {
  ZPIR_GUARD(build_bc_batch_launch(cko, n, lm, nb, nq, bc, S(stream)));
}

int zpir_umma_answer_rows_batch(const uint32_t* H, int64_t rows, int64_t n, const uint8_t* bc,
                                int nb, int nq, int wz, uint32_t* z, void* stream) {
  ZPIR_GUARD(umma_answer_rows_batch_launch(H, rows, n, bc, nb, nq, wz, z, S(stream)));
}

int zpir_answer_groups_batch(const uint32_t* z, int64_t zq, const uint32_t* b, int64_t bq,
                             uint32_t qmask, int64_t d1, int cap, int64_t groups, int lm,
                             const uint32_t* mods, const uint32_t* nps, const uint32_t* rpows,
                             int nchunks, const uint8_t* fast0s, uint32_t* t, int64_t t_ld, int nq,
                             int stride, void* stream) {
  ZPIR_GUARD(answer_groups_batch_launch(z, zq, b, bq, qmask, d1, cap, groups, lm, mods, nps, rpows,
                                        nchunks, fast0s, t, t_ld, nq, stride, S(stream)));
}

int zpir_multiexp_rows(const uint32_t* bases, int64_t n, const uint32_t* exps,
                       const int32_t* row_ids, int64_t rows, int64_t row_stride,
                       int64_t base_stride, int64_t limb_stride, int elimbs, int limbs,
                       const uint32_t* N, uint32_t np, const uint32_t* r2, const uint32_t* one_m,
                       int keep_mont, uint32_t* out, void* workspace, int64_t ws_bytes,
                       void* stream) {
  ZPIR_GUARD(multiexp_rows_launch(bases, n, exps, row_ids, rows, row_stride, base_stride,
                                  limb_stride, elimbs, limbs, N, np, r2, one_m, keep_mont, out,
                                  workspace, ws_bytes, S(stream)));
}

int zpir_slot_combine_many(int clients, const uint32_t* const* W, const uint32_t* const* N,
                           const uint32_t* np, uint32_t* const* out, int cap,
                           const int32_t* group_ids, int64_t ngroups, int limbs,
                           const uint32_t* gamma, int gamma_bits, void* stream) {
  ZPIR_GUARD(slot_combine_many_launch(clients, W, N, np, out, cap, group_ids, ngroups, limbs,
                                      gamma, gamma_bits, S(stream)));
}

int zpir_slot_combine(const uint32_t* W, int cap, const int32_t* group_ids, int64_t ngroups,
                      int limbs, const uint32_t* N, uint32_t np, const uint32_t* gamma,
                      int gamma_bits, uint32_t* out, void* stream) {
  ZPIR_GUARD(slot_combine_launch(W, cap, group_ids, ngroups, limbs, N, np, gamma, gamma_bits, out,
                                 S(stream)));
}

int zpir_answer_general(const uint32_t* z, const uint32_t* b, uint32_t qmask, int64_t d1, int cap,
                        int64_t groups, int lm, const uint32_t* m, uint32_t np,
                        const uint32_t* ctab, uint32_t* w, uint32_t* t, int64_t t_ld,
                        void* stream) {
  ZPIR_GUARD(answer_general_launch(z, b, qmask, d1, cap, groups, lm, m, np, ctab, w, t, t_ld,
                                   S(stream)));
}

int zpir_pow8_table(const uint32_t* bases, int64_t n, int limbs, const uint32_t* N, uint32_t np,
                    const uint32_t* r2, uint32_t* P, void* stream) {
  ZPIR_GUARD(pow8_table_launch(bases, n, limbs, N, np, r2, P, S(stream)));
}

int zpir_slot_fixed(const uint32_t* P, int64_t n, const uint32_t* exps, int64_t row_stride,
                    const int32_t* row_ids, int64_t rows, int limbs, const uint32_t* N,
                    uint32_t np, const uint32_t* one_m, uint32_t* W, void* stream) {
  ZPIR_GUARD(slot_fixed_launch(P, n, exps, row_stride, row_ids, rows, limbs, N, np, one_m, W,
                               S(stream)));
}

int zpir_groups_z(const uint32_t* z, int64_t zq, int64_t d1, int cap, int64_t groups, int lm,
                  const uint32_t* mods, const uint32_t* nps, const uint32_t* rpows, int nchunks,
                  const uint8_t* fast0s, uint32_t* tz, int64_t t_ld, int nq, int stride,
                  void* stream) {
  ZPIR_GUARD(groups_z_launch(z, zq, d1, cap, groups, lm, mods, nps, rpows, nchunks, fast0s, tz, t_ld,
                             nq, stride, S(stream)));
}

int zpir_groups_finish(const uint32_t* tz, const uint32_t* b, int64_t bq, uint32_t qmask,
                       int64_t d1, int cap, int64_t groups, int lm, const uint32_t* mods,
                       uint32_t* t, int64_t t_ld, int nq, int stride, void* stream) {
  ZPIR_GUARD(groups_finish_launch(tz, b, bq, qmask, d1, cap, groups, lm, mods, t, t_ld, nq, stride,
                                  S(stream)));
}

int zpir_chacha_words32(const uint8_t* key32, const uint8_t* iv16, int64_t rows, int64_t cols,
                        uint32_t* out, int64_t ld, uint32_t mask, void* stream) {
  ZPIR_GUARD(chacha_words32_launch(key32, iv16, rows, cols, out, ld, mask, S(stream)));
}

int zpir_host_device_pointer(void* host, void** dev) {
  if (!host || !dev) {
    set_error("zpir_host_device_pointer: null argument");
    return kErrInput;
  }
  const cudaError_t e = cudaHostGetDevicePointer(dev, host, 0);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("cudaHostGetDevicePointer: %s", cudaGetErrorString(e));
    return kErrCuda;
  }
  return kOk;
}

int zpir_rns_residues(const uint32_t* smat, int64_t rows, int64_t n, int cap, int stride,
                      const uint32_t* primes, const uint64_t* weights, int count, int64_t groups,
                      double* out, void* stream) {
  ZPIR_GUARD(rns_residues_launch(smat, rows, n, cap, stride, primes,
                                 reinterpret_cast<const unsigned long long*>(weights), count,
                                 groups, out, S(stream)));
}

int zpir_multiexp_opcount(const uint32_t* smat, int64_t rows, int64_t n, int cap, int sbits,
                          int64_t groups, int64_t* out, void* stream) {
  ZPIR_GUARD(multiexp_opcount_launch(smat, rows, n, cap, sbits, groups,
                                     reinterpret_cast<long long*>(out), S(stream)));
}

int zpir_chacha_below(const uint8_t* key32, uint32_t domain, uint64_t query_index, int64_t n,
                      const uint32_t* bound, int limbs, int bits, uint32_t* out, void* stream) {
  ZPIR_GUARD(chacha_below_launch(key32, domain, query_index, n, bound, limbs, bits, out,
                                 S(stream)));
}

int zpir_digits_to_limbs(const uint32_t* digits, int64_t count, int ndig, uint32_t* limbs, int nl,
                         void* stream) {
  ZPIR_GUARD(digits_to_limbs_launch(digits, count, ndig, limbs, nl, S(stream)));
}

int zpir_limbs_to_digits(const uint32_t* limbs, int64_t count, int nl, int64_t ld,
                         uint32_t* digits, int ndig, void* stream) {
  ZPIR_GUARD(limbs_to_digits_launch(limbs, count, nl, ld, digits, ndig, S(stream)));
}

int zpir_rows_differ(const uint8_t* a, const uint8_t* b, int64_t rows, int64_t ld, uint32_t* flags,
                     void* stream) {
  ZPIR_GUARD(rows_differ_launch(a, b, rows, ld, flags, S(stream)));
}

int zpir_move_rows(const uint8_t* src, uint8_t* dst, int64_t pitch, const int32_t* ids,
                   int64_t nrows, int scatter, void* stream) {
  ZPIR_GUARD(move_rows_launch(src, dst, pitch, ids, nrows, scatter, S(stream)));
}

// Async copy between pinned host and device memory (kind: 0 = H2D, 1 = D2H)
// on the caller's stream; lets the API layer skip framework overhead per query.
int zpir_event_record(void* event, void* stream) {
  // external record: inside stream capture this becomes an event-record node
  // that fires on every graph replay (plain records only order the capture)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(S(stream), &cs) != cudaSuccess) return check_launch("event_record");
  const unsigned flags = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
  if (cudaEventRecordWithFlags(reinterpret_cast<cudaEvent_t>(event), S(stream), flags) !=
      cudaSuccess)
    return check_launch("event_record");
  return kOk;
}

int zpir_stream_wait_event(void* stream, void* event) {
  // inside stream capture: an external event-wait node (waits, at every
  // replay, for the event's latest record made outside the graph)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(S(stream), &cs) != cudaSuccess) return check_launch("stream_wait");
  const unsigned flags = cs == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0u;
  if (cudaStreamWaitEvent(S(stream), reinterpret_cast<cudaEvent_t>(event), flags) != cudaSuccess)
    return check_launch("stream_wait");
  return kOk;
}

int zpir_graph_launch(void* graph_exec, void* stream) {
  if (cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(graph_exec), S(stream)) != cudaSuccess)
    return check_launch("graph_launch");
  return kOk;
}

int zpir_memcpy_async(void* dst, const void* src, int64_t bytes, int kind, void* stream) {
  const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  if (cudaMemcpyAsync(dst, src, (size_t)bytes, k, S(stream)) != cudaSuccess)
    return check_launch("memcpy_async");
  return kOk;
}

}  // extern "C"
