// Online answer, compression half: t_g = (bs_g + hv_g) mod m, and COMBINED.
//
// Reference: respond() (protocol.py:333-365) computes hv = H_scaled * ck_o
// mod m through a 240-prime RNS engine (rns.py:163-188) over H_rns (240 x d1'
// x n float64, ~1 GB at 1 GiB) and adds bs = scaled_b(b) (protocol.py:259-269).
// For gamma = q = 2^32 the batch-scaled hint is the little-endian
// concatenation of H's 32-bit words (protocol.py:223-230), so
//   t_g = ( sum_j 2^(32 j) * (b_c + y_c) ) mod m,   c = g*cap + j,
//   y_c = sum_k H[c,k] * ck_o[k]        (exact, < n 2^32 m)
// (SURVEY 8c(ii)); the device reads H (4 bytes/entry, 128 MB at 1 GiB)
// instead of H_rns.
//
//   answer_rows   z_c = y_c as Lm + 4 32-bit limbs (top two always zero;
//                 the padding keeps z rows 16-byte aligned), Lm = limbs of m.
//   answer_groups X_g = sum_j 2^(32j) (b_c + z_c); t_g = X_g mod m via
//                 t = sum_s mont(X_s, R^(s+1) mod m) over Lm-limb chunks X_s.
//   combine       K_g = (1 + t_g m) * k_g mod m^2 (paillier.py:104-123).
#include <cstdlib>

#include "bignum.cuh"

namespace zpir {

// z[c, 0..Lm+4) = y_c = sum_k H[c,k] * cko[k, 0..Lm) (b is added by the group stage)
// 128 threads, tile = 32 rows x 64 limbs, each thread 4 rows x 4 limbs with
// 96-bit accumulators; row-wise carry propagation in shared memory.
__global__ void __launch_bounds__(128)
answer_rows_kernel(const uint32_t* __restrict__ H, int64_t n, const uint32_t* __restrict__ b,
                   uint32_t qmask, const uint32_t* __restrict__ cko, int lm,
                   uint32_t* __restrict__ z) {
  __shared__ __align__(16) uint32_t sH[16][32];
  __shared__ __align__(16) uint32_t sC[16][64];
  __shared__ uint32_t sS[32][64][3];
  const int t = threadIdx.x, tr = t >> 4, tc = t & 15;
  const int64_t row0 = (int64_t)blockIdx.x * 32;
  const int wz = lm + 4;
  // row-carry state, owned by threads 0..31 (one row each)
  unsigned __int128 carry = 0;
  (void)b;
  (void)qmask;

  for (int ch = 0; ch < lm; ch += 64) {
    uint32_t lo[4][4], mi[4][4], hi[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) lo[r][c] = mi[r][c] = hi[r][c] = 0;
    for (int64_t k0 = 0; k0 < n; k0 += 16) {
      {
        const int row = t >> 2, kq = (t & 3) * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t k = k0 + kq + i;
          sH[kq + i][row] = (k < n) ? H[(row0 + row) * n + k] : 0u;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int idx = t + i * 128, kk = idx >> 6, l = idx & 63;
        const int64_t k = k0 + kk;
        sC[kk][l] = (k < n && ch + l < lm) ? cko[k * lm + ch + l] : 0u;
      }
      __syncthreads();
#pragma unroll 4
      for (int kk = 0; kk < 16; ++kk) {
        const uint4 hv = *reinterpret_cast<const uint4*>(&sH[kk][tr * 4]);
        const uint32_t h[4] = {hv.x, hv.y, hv.z, hv.w};
        uint32_t c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = sC[kk][tc + 16 * j];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
                "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
                "addc.u32 %2, %2, 0;"
                : "+r"(lo[r][j]), "+r"(mi[r][j]), "+r"(hi[r][j])
                : "r"(h[r]), "r"(c[j]));
      }
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        sS[tr * 4 + r][tc + 16 * j][0] = lo[r][j];
        sS[tr * 4 + r][tc + 16 * j][1] = mi[r][j];
        sS[tr * 4 + r][tc + 16 * j][2] = hi[r][j];
      }
    __syncthreads();
    if (t < 32) {
      uint32_t* zr = z + (row0 + t) * wz;
      const int lim = min(64, lm - ch);
      for (int l = 0; l < lim; ++l) {
        const unsigned __int128 s = (unsigned __int128)sS[t][l][0] |
                                    ((unsigned __int128)sS[t][l][1] << 32) |
                                    ((unsigned __int128)sS[t][l][2] << 64);
        const unsigned __int128 v = s + carry;
        zr[ch + l] = (uint32_t)v;
        carry = v >> 32;
      }
    }
    __syncthreads();
  }
  if (t < 32) {
    uint32_t* zr = z + (row0 + t) * wz;
    zr[lm] = (uint32_t)carry;
    zr[lm + 1] = (uint32_t)(carry >> 32);
    zr[lm + 2] = (uint32_t)(carry >> 64);
    zr[lm + 3] = 0;
  }
}

// One CTA (4 warps) per group g, latency-oriented (521 groups at 1 GiB):
//   1. all threads: position sums S[P] = sum_j z[g*cap + j][P - j] (+ b at
//      P < rows of the group), split as lo/hi 32-bit words in shared memory
//   2. warp 0: X = LO + (HI << 32) with a ballot carry-lookahead add
//      (NCH*LM limbs held as LPL*NCH limbs per lane)
//   3. warp s < NCH: r_s = mont(X_s, R^(s+1) mod m) -- the chunk products run
//      concurrently in different warps; chunk 0 only needs a conditional
//      subtraction when R < 2m (m of exactly 32*LM bits)
//   4. warp 0: t = sum_s r_s mod m
// Batched over queries with blockIdx.y = query q: z, b, t, the modulus, its
// R-power table, n' and fast0 are offset by the per-query strides (zero
// strides and a single n'/fast0 for the one-query call).
struct GroupBatch {
  int64_t zq, bq, tq, mq, rq;
  const uint32_t* nps;     // per-query n' (nullptr: use np)
  const uint8_t* fast0s;   // per-query fast0 (nullptr: use fast0)
  int stride = 1;          // slot stride in 32-bit limbs: gamma = 2^(32 stride)
};

template <int LPL, int NCH, bool WITH_B = true>
__global__ void __launch_bounds__(128)
answer_groups_kernel(const uint32_t* __restrict__ z, const uint32_t* __restrict__ b,
                     uint32_t qmask, int64_t d1, int cap, int64_t groups,
                     const uint32_t* __restrict__ mod, uint32_t np,
                     const uint32_t* __restrict__ rpow, int fast0, uint32_t* __restrict__ t,
                     int64_t t_ld, GroupBatch bt) {
  {
    const int64_t q = blockIdx.y;
    z += q * bt.zq;
    b += q * bt.bq;
    t += q * bt.tq;
    mod += q * bt.mq;
    rpow += q * bt.rq;
    if (bt.nps) np = bt.nps[q];
    if (bt.fast0s) fast0 = bt.fast0s[q];
  }
  constexpr int LM = 32 * LPL;
  constexpr int NX = NCH * LM;
  constexpr int LX = NCH * LPL;
  __shared__ __align__(16) uint32_t lo[NX], hi[NX + 1], X[NX], R[NCH][LM];
  extern __shared__ uint32_t zs[];  // the group's z rows (cap x wz), staged
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t g = blockIdx.x;
  const int wz = LM + 4;
  const int64_t c0 = g * cap;
  const int nrows = (int)(((int64_t)cap < d1 - c0) ? (int64_t)cap : d1 - c0);
  {
    // coalesced 16-byte copy of the group's rows (contiguous in z)
    const uint4* src = reinterpret_cast<const uint4*>(z + c0 * wz);
    uint4* dst = reinterpret_cast<uint4*>(zs);
    const int n16 = nrows * wz / 4;
    for (int i = tid; i < n16; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  // position sums X_P = b_P + sum_j z_j[P - j], split into lo/hi words
  const int sd = bt.stride;
  for (int P = tid; P < NX; P += blockDim.x) {
    unsigned long long s = (WITH_B && P % sd == 0 && P / sd < nrows)
                               ? (unsigned long long)(b[c0 + P / sd] & qmask)
                               : 0ull;
    const int jlo = max(0, (P - wz + sd) / sd), jhi = min(nrows - 1, P / sd);
    for (int j = jlo; j <= jhi; ++j) s += zs[j * wz + (P - sd * j)];
    lo[P] = (uint32_t)s;
    hi[P + 1] = (uint32_t)(s >> 32);
  }
  if (tid == 0) hi[0] = 0;
  __syncthreads();
  if (warp == 0) {
    uint32_t x[LX], y[LX];
#pragma unroll
    for (int i = 0; i < LX; ++i) {
      x[i] = lo[lane * LX + i];
      y[i] = hi[lane * LX + i];
    }
    big_add<LX>(x, y, lane);
#pragma unroll
    for (int i = 0; i < LX; ++i) X[lane * LX + i] = x[i];
  }
  __syncthreads();
  if (warp < NCH) {
    uint32_t n_[LPL], x[LPL], rp[LPL];
    big_load<LPL>(n_, mod, lane);
#pragma unroll
    for (int i = 0; i < LPL; ++i) x[i] = X[warp * LM + lane * LPL + i];
    if (warp == 0 && fast0) {
      big_cond_sub<LPL>(x, 0u, n_, lane);  // X_0 < R < 2m
    } else {
      big_load<LPL>(rp, rpow + (size_t)warp * LM, lane);
      mont_mul<LPL>(x, x, rp, n_, np, lane);
    }
#pragma unroll
    for (int i = 0; i < LPL; ++i) R[warp][lane * LPL + i] = x[i];
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t n_[LPL], res[LPL], x[LPL];
    big_load<LPL>(n_, mod, lane);
#pragma unroll
    for (int i = 0; i < LPL; ++i) res[i] = R[0][lane * LPL + i];
#pragma unroll
    for (int s = 1; s < NCH; ++s) {
#pragma unroll
      for (int i = 0; i < LPL; ++i) x[i] = R[s][lane * LPL + i];
      const uint32_t cy = big_add<LPL>(res, x, lane);
      big_cond_sub<LPL>(res, cy, n_, lane);
    }
    uint32_t* out = t + g * t_ld;
    big_store<LPL>(out, res, lane);
    for (int64_t i = LM + lane; i < t_ld; i += 32) out[i] = 0;
  }
}

// Finish stage: t_g = (tz_g + B_g) mod m with B_g = sum_j 2^(32 j) (b_c & qmask)
// < gamma^cap < m (capacity bound, protocol.py:66-78), so one addition and one
// conditional subtraction suffice. tz_g = (sum_j 2^(32j) z_c) mod m comes from
// answer_groups_kernel<..., WITH_B = false>, which therefore does not wait for
// the GEMV. One warp per group; per-query strides as in GroupBatch.
template <int LPL>
__global__ void __launch_bounds__(128)
groups_finish_kernel(const uint32_t* __restrict__ tz, const uint32_t* __restrict__ b,
                     uint32_t qmask, int64_t d1, int cap, int64_t groups,
                     const uint32_t* __restrict__ mod, uint32_t* __restrict__ t, int64_t t_ld,
                     GroupBatch bt) {
  constexpr int LM = 32 * LPL;
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= groups) return;
  const int64_t q = blockIdx.y;
  tz += q * groups * t_ld;
  b += q * bt.bq;
  t += q * bt.tq;
  mod += q * bt.mq;
  const int64_t c0 = g * cap;
  const int nrows = (int)(((int64_t)cap < d1 - c0) ? (int64_t)cap : d1 - c0);
  uint32_t n_[LPL], x[LPL], y[LPL];
  big_load<LPL>(n_, mod, lane);
  big_load<LPL>(x, tz + g * t_ld, lane);
#pragma unroll
  for (int i = 0; i < LPL; ++i) {
    const int j = lane * LPL + i;
    y[i] = (j % bt.stride == 0 && j / bt.stride < nrows) ? (b[c0 + j / bt.stride] & qmask) : 0u;
  }
  const uint32_t cy = big_add<LPL>(x, y, lane);
  big_cond_sub<LPL>(x, cy, n_, lane);
  uint32_t* out = t + g * t_ld;
  big_store<LPL>(out, x, lane);
  for (int64_t i = LM + lane; i < t_ld; i += 32) out[i] = 0;
}

// ---- general gamma (not a power of 2^32): t_g = sum_j (gamma^j mod m)(b_c + z_c)
// mod m (protocol.py:219-238, :259-269 with the reference's generic loops).
// rows_weighted: one warp per row c = g*cap + j (< d1): u = z_c + (b_c & qmask)
// as LM + 4 limbs, w_c = mont(u_lo, gamma^j R mod m) + mont(u_hi, gamma^j R^2
// mod m) mod m with u = u_lo + R u_hi. ctab[j] = {gamma^j R, gamma^j R^2} mod m.
template <int LPL>
__global__ void __launch_bounds__(128)
rows_weighted_kernel(const uint32_t* __restrict__ z, const uint32_t* __restrict__ b,
                     uint32_t qmask, int64_t d1, int cap, const uint32_t* __restrict__ mod,
                     uint32_t np, const uint32_t* __restrict__ ctab, uint32_t* __restrict__ w) {
  constexpr int LM = 32 * LPL;
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= d1) return;
  const int j = (int)(c % cap);
  const uint32_t* zr = z + c * (LM + 4);
  uint32_t n_[LPL], lo[LPL], hi[LPL], cc[LPL];
  big_load<LPL>(n_, mod, lane);
  big_load<LPL>(lo, zr, lane);
#pragma unroll
  for (int i = 0; i < LPL; ++i) {
    const int li = lane * LPL + i;
    hi[i] = (li < 4) ? zr[LM + li] : 0u;
    cc[i] = (li == 0) ? (b[c] & qmask) : 0u;
  }
  const uint32_t cy = big_add<LPL>(lo, cc, lane);     // lo += b_c, carry into hi
  big_set_small<LPL>(cc, cy, lane);
  big_add<LPL>(hi, cc, lane);
  big_load<LPL>(cc, ctab + (size_t)j * 2 * LM, lane);
  mont_mul<LPL>(lo, lo, cc, n_, np, lane);
  big_load<LPL>(cc, ctab + (size_t)j * 2 * LM + LM, lane);
  mont_mul<LPL>(hi, hi, cc, n_, np, lane);
  const uint32_t c2 = big_add<LPL>(lo, hi, lane);
  big_cond_sub<LPL>(lo, c2, n_, lane);
  big_store<LPL>(w + c * LM, lo, lane);
}

// t_g = sum_{j < rows of g} w[g*cap + j] mod m, one warp per group.
template <int LPL>
__global__ void __launch_bounds__(128)
group_sum_kernel(const uint32_t* __restrict__ w, int64_t d1, int cap, int64_t groups,
                 const uint32_t* __restrict__ mod, uint32_t* __restrict__ t, int64_t t_ld) {
  constexpr int LM = 32 * LPL;
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= groups) return;
  const int64_t c0 = g * cap;
  const int nrows = (int)(((int64_t)cap < d1 - c0) ? (int64_t)cap : d1 - c0);
  uint32_t n_[LPL], acc[LPL], x[LPL];
  big_load<LPL>(n_, mod, lane);
  big_set_small<LPL>(acc, 0, lane);
  for (int j = 0; j < nrows; ++j) {
    big_load<LPL>(x, w + (c0 + j) * LM, lane);
    const uint32_t cy = big_add<LPL>(acc, x, lane);
    big_cond_sub<LPL>(acc, cy, n_, lane);
  }
  uint32_t* out = t + g * t_ld;
  big_store<LPL>(out, acc, lane);
  for (int64_t i = LM + lane; i < t_ld; i += 32) out[i] = 0;
}

// K_g = (1 + t_g m) k_g mod m^2, one warp per group, with m^2 context
// (n2, np2), r2 = R^2 mod m^2, mr = m R mod m^2.
template <int LPL>
__global__ void __launch_bounds__(128)
combine_kernel(const uint32_t* __restrict__ t, const uint32_t* __restrict__ k, int64_t groups,
               const uint32_t* __restrict__ n2, uint32_t np2, const uint32_t* __restrict__ r2,
               const uint32_t* __restrict__ mr, uint32_t* __restrict__ out) {
  constexpr int L = 32 * LPL;
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= groups) return;
  uint32_t n_[LPL], a[LPL], b[LPL], one[LPL];
  big_load<LPL>(n_, n2, lane);
  big_load<LPL>(a, t + g * L, lane);
  big_load<LPL>(b, mr, lane);
  mont_mul<LPL>(a, a, b, n_, np2, lane);  // t m  (< m^2, exact)
  big_set_small<LPL>(one, 1, lane);
  big_add<LPL>(a, one, lane);             // 1 + t m  (< m^2, no carry out)
  big_load<LPL>(b, k + g * L, lane);
  mont_mul<LPL>(a, a, b, n_, np2, lane);  // (1 + t m) k R^-1
  big_load<LPL>(b, r2, lane);
  mont_mul<LPL>(a, a, b, n_, np2, lane);  // (1 + t m) k
  big_store<LPL>(out + g * L, a, lane);
}

// out[i] = a[i] * b[i] mod N (canonical), one warp per product: two Montgomery
// products, the second against R^2 mod N. Backs paillier.add-style batches.
template <int LPL>
__global__ void __launch_bounds__(128)
mulmod_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, int64_t count,
              const uint32_t* __restrict__ n, uint32_t np, const uint32_t* __restrict__ r2,
              uint32_t* __restrict__ out) {
  constexpr int L = 32 * LPL;
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= count) return;
  uint32_t n_[LPL], x[LPL], y[LPL];
  big_load<LPL>(n_, n, lane);
  big_load<LPL>(x, a + i * L, lane);
  big_load<LPL>(y, b + i * L, lane);
  mont_mul<LPL>(x, x, y, n_, np, lane);
  big_load<LPL>(y, r2, lane);
  mont_mul<LPL>(x, x, y, n_, np, lane);
  big_store<LPL>(out + i * L, x, lane);
}

int answer_rows_launch(const uint32_t* H, int64_t rows, int64_t n, const uint32_t* b,
                       uint32_t qmask, const uint32_t* cko, int lm, uint32_t* z, cudaStream_t st) {
  if (rows % 32 || n <= 0 || lm <= 0 || lm % 32) {
    set_error("answer_rows: bad shapes (rows=%lld n=%lld lm=%d)", (long long)rows, (long long)n, lm);
    return kErrInput;
  }
  answer_rows_kernel<<<(unsigned)(rows / 32), 128, 0, st>>>(H, n, b, qmask, cko, lm, z);
  return check_launch("answer_rows");
}

#define ZPIR_LPL_DISPATCH(LPLV, ...)                                   \
  switch (LPLV) {                                                      \
    case 1: { constexpr int LPL = 1; __VA_ARGS__; } break;            \
    case 2: { constexpr int LPL = 2; __VA_ARGS__; } break;            \
    case 3: { constexpr int LPL = 3; __VA_ARGS__; } break;            \
    case 4: { constexpr int LPL = 4; __VA_ARGS__; } break;            \
    case 6: { constexpr int LPL = 6; __VA_ARGS__; } break;            \
    case 8: { constexpr int LPL = 8; __VA_ARGS__; } break;            \
    default:                                                           \
      set_error("unsupported limb width %d (limbs per lane)", LPLV); \
      return kErrUnsupported;                                          \
  }

static int answer_groups_launch_ex(const uint32_t* z, const uint32_t* b, uint32_t qmask,
                                   int64_t d1, int cap, int64_t groups, int lm,
                                   const uint32_t* mod, uint32_t np, const uint32_t* rpow,
                                   int nchunks, int fast0, uint32_t* t, int64_t t_ld,
                                   cudaStream_t st, int nq, GroupBatch bt) {
  if (lm % 32 || nchunks * lm < bt.stride * cap + lm + 4 || t_ld < lm || cap <= 0 || nchunks < 2 ||
      nchunks > 3) {
    set_error("answer_groups: bad layout (lm=%d cap=%d nchunks=%d)", lm, cap, nchunks);
    return kErrInput;
  }
  const dim3 grid((unsigned)groups, (unsigned)nq);
  const size_t zsm = (size_t)cap * (lm + 4) * sizeof(uint32_t);
#define ZPIR_GROUPS(NCHV)                                                                    \
  ZPIR_LPL_DISPATCH(lm / 32, {                                                               \
    cudaFuncSetAttribute(answer_groups_kernel<LPL, NCHV>,                                    \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zsm);             \
    answer_groups_kernel<LPL, NCHV><<<grid, 128, zsm, st>>>(z, b, qmask, d1, cap, groups,    \
                                                            mod, np, rpow, fast0, t, t_ld,   \
                                                            bt);                             \
  })
  if (nchunks == 2) {
    ZPIR_GROUPS(2);
  } else {
    ZPIR_GROUPS(3);
  }
#undef ZPIR_GROUPS
  return check_launch("answer_groups");
}

// Group stage without b (tz = (sum_j 2^(32j) z_c) mod m) and the finish stage.
int groups_z_launch(const uint32_t* z, int64_t zq, int64_t d1, int cap, int64_t groups, int lm,
                    const uint32_t* mods, const uint32_t* nps, const uint32_t* rpows, int nchunks,
                    const uint8_t* fast0s, uint32_t* tz, int64_t t_ld, int nq, int stride,
                    cudaStream_t st) {
  if (lm % 32 || stride < 1 || nchunks * lm < stride * cap + lm + 4 || t_ld < lm || cap <= 0 ||
      nchunks < 2 || nchunks > 3 || stride * cap >= lm) {
    set_error("groups_z: bad layout (lm=%d cap=%d nchunks=%d stride=%d)", lm, cap, nchunks,
              stride);
    return kErrInput;
  }
  GroupBatch bt{zq, 0, groups * t_ld, lm, (int64_t)nchunks * lm, nps, fast0s, stride};
  const dim3 grid((unsigned)groups, (unsigned)nq);
  size_t zsm = (size_t)cap * (lm + 4) * sizeof(uint32_t);
#define ZPIR_GZ(NCHV)                                                                          \
  ZPIR_LPL_DISPATCH(lm / 32, {                                                                 \
    cudaFuncSetAttribute(answer_groups_kernel<LPL, NCHV, false>,                               \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zsm);               \
    answer_groups_kernel<LPL, NCHV, false><<<grid, 128, zsm, st>>>(                            \
        z, nullptr, 0u, d1, cap, groups, mods, 0u, rpows, 0, tz, t_ld, bt);                    \
  })
  if (nchunks == 2) {
    ZPIR_GZ(2);
  } else {
    ZPIR_GZ(3);
  }
#undef ZPIR_GZ
  return check_launch("groups_z");
}

int groups_finish_launch(const uint32_t* tz, const uint32_t* b, int64_t bq, uint32_t qmask,
                         int64_t d1, int cap, int64_t groups, int lm, const uint32_t* mods,
                         uint32_t* t, int64_t t_ld, int nq, int stride, cudaStream_t st) {
  if (lm % 32 || t_ld < lm || stride < 1 || stride * cap > lm) {
    set_error("groups_finish: bad layout");
    return kErrInput;
  }
  GroupBatch bt{0, bq, groups * t_ld, lm, 0, nullptr, nullptr, stride};
  const dim3 grid((unsigned)ceil_div(groups, 4), (unsigned)nq);
  ZPIR_LPL_DISPATCH(lm / 32, {
    groups_finish_kernel<LPL><<<grid, 128, 0, st>>>(tz, b, qmask, d1, cap, groups, mods, t, t_ld,
                                                    bt);
  });
  return check_launch("groups_finish");
}

// Batched group stage: nq queries sharing d1/cap/lm, per-query moduli.
int answer_groups_batch_launch(const uint32_t* z, int64_t zq, const uint32_t* b, int64_t bq,
                               uint32_t qmask, int64_t d1, int cap, int64_t groups, int lm,
                               const uint32_t* mods, const uint32_t* nps, const uint32_t* rpows,
                               int nchunks, const uint8_t* fast0s, uint32_t* t, int64_t t_ld,
                               int nq, int stride, cudaStream_t st) {
  GroupBatch bt{zq, bq, groups * t_ld, lm, (int64_t)nchunks * lm, nps, fast0s, stride};
  return answer_groups_launch_ex(z, b, qmask, d1, cap, groups, lm, mods, 0, rpows, nchunks, 0, t,
                                 t_ld, st, nq, bt);
}

int answer_groups_launch(const uint32_t* z, const uint32_t* b, uint32_t qmask, int64_t d1,
                         int cap, int64_t groups, int lm, const uint32_t* mod, uint32_t np,
                         const uint32_t* rpow, int nchunks, int fast0, uint32_t* t, int64_t t_ld,
                         cudaStream_t st) {
  return answer_groups_launch_ex(z, b, qmask, d1, cap, groups, lm, mod, np, rpow, nchunks, fast0,
                                 t, t_ld, st, 1, GroupBatch{0, 0, 0, 0, 0, nullptr, nullptr});
}

// General-gamma group stage; w = workspace of d1 x lm limbs.
int answer_general_launch(const uint32_t* z, const uint32_t* b, uint32_t qmask, int64_t d1, int cap,
                          int64_t groups, int lm, const uint32_t* mod, uint32_t np,
                          const uint32_t* ctab, uint32_t* w, uint32_t* t, int64_t t_ld,
                          cudaStream_t st) {
  if (lm % 32 || t_ld < lm || cap <= 0 || d1 <= 0) {
    set_error("answer_general: bad layout");
    return kErrInput;
  }
  ZPIR_LPL_DISPATCH(lm / 32, {
    rows_weighted_kernel<LPL><<<(unsigned)ceil_div(d1, 4), 128, 0, st>>>(z, b, qmask, d1, cap, mod,
                                                                        np, ctab, w);
    if (int e = check_launch("rows_weighted")) return e;
    group_sum_kernel<LPL><<<(unsigned)ceil_div(groups, 4), 128, 0, st>>>(w, d1, cap, groups, mod,
                                                                        t, t_ld);
  });
  return check_launch("group_sum");
}

int combine_launch(const uint32_t* t, const uint32_t* k, int64_t groups, int l2, const uint32_t* n2,
                   uint32_t np2, const uint32_t* r2, const uint32_t* mr, uint32_t* out,
                   cudaStream_t st) {
  if (l2 % 32) {
    set_error("combine: limb count %d not a multiple of 32", l2);
    return kErrInput;
  }
  const unsigned grid = (unsigned)ceil_div(groups, 4);
  ZPIR_LPL_DISPATCH(l2 / 32, {
    combine_kernel<LPL><<<grid, 128, 0, st>>>(t, k, groups, n2, np2, r2, mr, out);
  });
  return check_launch("combine");
}

int mulmod_launch(const uint32_t* a, const uint32_t* b, int64_t count, int limbs, const uint32_t* n,
                  uint32_t np, const uint32_t* r2, uint32_t* out, cudaStream_t st) {
  if (limbs % 32) {
    set_error("mulmod: limb count %d not a multiple of 32", limbs);
    return kErrInput;
  }
  const unsigned grid = (unsigned)ceil_div(count, 4);
  ZPIR_LPL_DISPATCH(limbs / 32, {
    mulmod_kernel<LPL><<<grid, 128, 0, st>>>(a, b, count, n, np, r2, out);
  });
  return check_launch("mulmod");
}

}  // namespace zpir
