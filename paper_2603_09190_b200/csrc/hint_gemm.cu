// Server setup: DB layout transform and the global hint H = -DB * A mod q.
//
// Reference: ServerGlobalState.__init__ / _global_hint_fast (protocol.py:162-207)
// computes H = -db^T A mod q with two exact float64 GEMMs (A split 16/16)
// and falls back to Python triple loops when d0 > 32768 (protocol.py:209-217).
// Here the product is exact integer arithmetic mod 2^32 for any d0.
//
// CUDA-core version: 128x128 output tiles, 8x8 register blocking per thread,
// 32-deep K slabs staged in shared memory; u8 x u32 -> u32 wrapping IMAD.
#include "zpir_common.cuh"

namespace zpir {

// dbt[c * ld + i] = db[i * d1 + c]; zero in the padding (rows >= d1, i >= d0).
__global__ void __launch_bounds__(256)
transpose_db_kernel(const uint8_t* __restrict__ db, int64_t d0, int64_t d1, int64_t ld_src,
                    uint8_t* __restrict__ dbt, int64_t rows, int64_t ld) {
  __shared__ uint8_t tile[64][65];
  const int64_t i0 = (int64_t)blockIdx.x * 64;  // along d0 (K)
  const int64_t c0 = (int64_t)blockIdx.y * 64;  // along d1 (rows of DB)
  const int t = threadIdx.x;
#pragma unroll 4
  for (int rr = 0; rr < 16; ++rr) {
    const int i = rr * 4 + (t >> 6), c = t & 63;
    const int64_t gi = i0 + i, gc = c0 + c;
    tile[i][c] = (gi < d0 && gc < d1) ? db[gi * ld_src + gc] : (uint8_t)0;
  }
  __syncthreads();
#pragma unroll 4
  for (int rr = 0; rr < 16; ++rr) {
    const int c = rr * 4 + (t >> 6), i = t & 63;
    const int64_t gi = i0 + i, gc = c0 + c;
    if (gc < rows && gi < ld) dbt[gc * ld + gi] = tile[i][c];
  }
}

int transpose_db_launch(const uint8_t* db, int64_t d0, int64_t d1, int64_t ld_src, uint8_t* dbt,
                        int64_t rows, int64_t ld, cudaStream_t st) {
  if (rows < d1 || ld < d0 || rows % 64 || ld % 64) {
    set_error("transpose_db: bad padding (rows=%lld ld=%lld d0=%lld d1=%lld)", (long long)rows,
              (long long)ld, (long long)d0, (long long)d1);
    return kErrInput;
  }
  dim3 grid((unsigned)(ld / 64), (unsigned)(rows / 64));
  transpose_db_kernel<<<grid, 256, 0, st>>>(db, d0, d1, ld_src, dbt, rows, ld);
  return check_launch("transpose_db");
}

// H[c, k] = qmask & -(sum_i dbt[c, i] * A[i, k]); A is (ld x lda) with
// lda a multiple of 128 and zero columns >= n; H is (rows x n).
__global__ void __launch_bounds__(256, 2)
hint_gemm_kernel(const uint8_t* __restrict__ dbt, int64_t ld, const uint32_t* __restrict__ A,
                 int64_t lda, int64_t n, uint32_t* __restrict__ H, uint32_t qmask) {
  __shared__ __align__(16) uint8_t sD[32][128 + 16];
  __shared__ __align__(16) uint32_t sA[32][128];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int64_t row0 = (int64_t)blockIdx.y * 128, col0 = (int64_t)blockIdx.x * 128;
  uint32_t acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0;

  for (int64_t k0 = 0; k0 < ld; k0 += 32) {
    {
      const int row = t >> 1, half = t & 1;
      const uint4 v = *reinterpret_cast<const uint4*>(dbt + (row0 + row) * ld + k0 + half * 16);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int b = 0; b < 16; ++b) sD[half * 16 + b][row] = (uint8_t)(w[b >> 2] >> (8 * (b & 3)));
    }
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int idx = t + it * 256, k = idx >> 5, c4 = (idx & 31) * 4;
      *reinterpret_cast<uint4*>(&sA[k][c4]) =
          *reinterpret_cast<const uint4*>(A + (k0 + k) * lda + col0 + c4);
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      const uint2 dv = *reinterpret_cast<const uint2*>(&sD[kk][ty * 8]);
      const uint4 a0 = *reinterpret_cast<const uint4*>(&sA[kk][tx * 4]);
      const uint4 a1 = *reinterpret_cast<const uint4*>(&sA[kk][64 + tx * 4]);
      const uint32_t av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const uint32_t byte = ((r < 4 ? dv.x : dv.y) >> (8 * (r & 3))) & 0xffu;
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] += byte * av[c];
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int64_t row = row0 + ty * 8 + r;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int64_t col = col0 + (c < 4 ? tx * 4 + c : 64 + tx * 4 + (c - 4));
      if (col < n) H[row * n + col] = (0u - acc[r][c]) & qmask;
    }
  }
}

int hint_gemm_launch(const uint8_t* dbt, int64_t rows, int64_t ld, const uint32_t* A, int64_t lda,
                     int64_t n, uint32_t* H, uint32_t qmask, cudaStream_t st) {
  if (rows % 128 || ld % 32 || lda % 128 || lda < n || n <= 0) {
    set_error("global_hint: bad shapes (rows=%lld ld=%lld lda=%lld n=%lld)", (long long)rows,
              (long long)ld, (long long)lda, (long long)n);
    return kErrInput;
  }
  dim3 grid((unsigned)(lda / 128), (unsigned)(rows / 128));
  hint_gemm_kernel<<<grid, 256, 0, st>>>(dbt, ld, A, lda, n, H, qmask);
  return check_launch("global_hint");
}

// ---- incremental database update helpers (server.py:115-124 does a full
// rebuild; here only the DB rows that changed are re-multiplied) -----------

// flags[r] = 1 iff rows r of a and b (ld bytes, ld % 16 == 0) differ.
__global__ void __launch_bounds__(256)
rows_differ_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t ld,
                   uint32_t* __restrict__ flags) {
  const int64_t r = blockIdx.x;
  const uint4* pa = reinterpret_cast<const uint4*>(a + r * ld);
  const uint4* pb = reinterpret_cast<const uint4*>(b + r * ld);
  int diff = 0;
  for (int64_t i = threadIdx.x; i < ld / 16; i += blockDim.x) {
    const uint4 x = pa[i], y = pb[i];
    diff |= (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
  }
  diff = __syncthreads_or(diff);
  if (threadIdx.x == 0) flags[r] = diff ? 1u : 0u;
}

// dst row i = src row ids[i] (gather) or dst row ids[i] = src row i (scatter),
// rows of `pitch` bytes (pitch % 16 == 0).
__global__ void move_rows_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                 int64_t pitch, const int32_t* __restrict__ ids, int scatter) {
  const int64_t i = blockIdx.x;
  const int64_t si = scatter ? i : (int64_t)ids[i];
  const int64_t di = scatter ? (int64_t)ids[i] : i;
  const uint4* s = reinterpret_cast<const uint4*>(src + si * pitch);
  uint4* d = reinterpret_cast<uint4*>(dst + di * pitch);
  for (int64_t k = threadIdx.x; k < pitch / 16; k += blockDim.x) d[k] = s[k];
}

int rows_differ_launch(const uint8_t* a, const uint8_t* b, int64_t rows, int64_t ld,
                       uint32_t* flags, cudaStream_t st) {
  if (ld % 16 || rows <= 0) {
    set_error("rows_differ: ld %% 16 required");
    return kErrInput;
  }
  rows_differ_kernel<<<(unsigned)rows, 256, 0, st>>>(a, b, ld, flags);
  return check_launch("rows_differ");
}

int move_rows_launch(const uint8_t* src, uint8_t* dst, int64_t pitch, const int32_t* ids,
                     int64_t nrows, int scatter, cudaStream_t st) {
  if (pitch % 16 || nrows < 0) {
    set_error("move_rows: pitch %% 16 required");
    return kErrInput;
  }
  if (nrows == 0) return kOk;
  move_rows_kernel<<<(unsigned)nrows, 256, 0, st>>>(src, dst, pitch, ids, scatter);
  return check_launch("move_rows");
}

}  // namespace zpir
