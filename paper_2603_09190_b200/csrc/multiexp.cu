// Per-client compressed hint: k_g = prod_k ck_r[k]^{H_scaled[g][k]} mod m^2.
//
// Reference: hint() (protocol.py:291-296) -> paillier_matmul (paillier.py:
// 196-203) -> multiexp (paillier.py:134-193): w=6 windows, buckets 1..63,
// running-sum combine, one row at a time in gmpy2 (361,620 4096-bit group
// multiplications per entry at BASELINE parameters).
//
// B200 design (exact, same group element, canonical output < m^2):
//   to_mont       bases -> Montgomery form (one warp per base).
//   window        one warp per (row g, window w): counting-sort the 6-bit
//                 digits of the n exponents into buckets in shared memory,
//                 then for d = 63..1 form bucket_d = prod of its bases,
//                 running *= bucket_d, total *= running, all in registers
//                 (the running product never leaves the warp); write the
//                 window total W[g][w].
//   combine       one warp per row: acc = acc^(2^6) * W[g][w] from the top
//                 window down, then out of Montgomery form.
// Exponents are read in place through a strided-limb view: limb j of
// exponent (g, k) is E[g*rs + k*bs + j*ls]. For the hint that view is H
// itself (rs = cap*n, bs = 1, ls = n), since with gamma = 2^32 the limbs of
// H_scaled[g][k] are H[g*cap + j][k] (protocol.py:223-230); no H_scaled is
// ever materialised.
#include <algorithm>
#include <cstdlib>

#include <vector>

#include "bignum.cuh"

namespace zpir {

constexpr int kWin = 6;
constexpr int kBuckets = 1 << kWin;

__device__ __forceinline__ uint32_t exp_digit(const uint32_t* __restrict__ E, int64_t off,
                                              int64_t ls, int elimbs, int bitpos) {
  const int j = bitpos >> 5, sh = bitpos & 31;
  if (j >= elimbs) return 0u;
  uint32_t v = E[off + j * ls] >> sh;
  if (sh > 32 - kWin && j + 1 < elimbs) v |= E[off + (j + 1) * ls] << (32 - sh);
  return v & (kBuckets - 1);
}

template <int LPL>
__global__ void __launch_bounds__(128)
to_mont_kernel(const uint32_t* __restrict__ x, int64_t count, const uint32_t* __restrict__ n,
               uint32_t np, const uint32_t* __restrict__ r2, uint32_t* __restrict__ out) {
  constexpr int L = 32 * LPL;
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= count) return;
  uint32_t n_[LPL], a[LPL], b[LPL];
  big_load<LPL>(n_, n, lane);
  big_load<LPL>(a, x + i * L, lane);
  big_load<LPL>(b, r2, lane);
  mont_mul<LPL>(a, a, b, n_, np, lane);
  big_store<LPL>(out + i * L, a, lane);
}

// Shared memory per warp: cnt[64] + off[64] (u32) + list[n] (u32).
template <int LPL>
__global__ void __launch_bounds__(128)
window_kernel(const uint32_t* __restrict__ bases, int64_t n, const uint32_t* __restrict__ E,
              int64_t rows, int64_t rs, int64_t bs, int64_t ls, int elimbs, int nwin,
              const uint32_t* __restrict__ N, uint32_t np, uint32_t* __restrict__ W,
              uint8_t* __restrict__ flags, const int32_t* __restrict__ row_ids) {
  constexpr int L = 32 * LPL;
  extern __shared__ uint32_t smem_u32[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  uint32_t* cnt = smem_u32 + (size_t)wid * (2 * kBuckets + n);
  uint32_t* off = cnt + kBuckets;
  uint32_t* list = off + kBuckets;
  uint32_t n_[LPL];
  big_load<LPL>(n_, N, lane);
  const int64_t tasks = rows * nwin;
  for (int64_t task = (int64_t)blockIdx.x * wpb + wid; task < tasks;
       task += (int64_t)gridDim.x * wpb) {
    const int64_t gi = task / nwin;
    const int win = (int)(task - gi * nwin);
    const int64_t g = row_ids ? (int64_t)row_ids[gi] : gi;  // exponent row
    const int bitpos = win * kWin;
    cnt[lane] = 0;
    cnt[lane + 32] = 0;
    __syncwarp();
    for (int64_t k = lane; k < n; k += 32) {
      const uint32_t d = exp_digit(E, g * rs + k * bs, ls, elimbs, bitpos);
      if (d) atomicAdd(&cnt[d], 1u);
    }
    __syncwarp();
    // exclusive scan of cnt[0..63]: lane holds entries 2*lane, 2*lane+1
    const uint32_t c0 = cnt[2 * lane], c1 = cnt[2 * lane + 1];
    uint32_t incl = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(ZPIR_FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const uint32_t excl = incl - c0 - c1;
    off[2 * lane] = excl;
    off[2 * lane + 1] = excl + c0;
    __syncwarp();
    for (int64_t k = lane; k < n; k += 32) {
      const uint32_t d = exp_digit(E, g * rs + k * bs, ls, elimbs, bitpos);
      if (d) list[atomicAdd(&off[d], 1u)] = (uint32_t)k;
    }
    __syncwarp();
    // off[d] is now the end of bucket d
    bool has_run = false, has_tot = false;
    uint32_t run[LPL], tot[LPL], bkt[LPL], x[LPL];
    for (int d = kBuckets - 1; d >= 1; --d) {
      const uint32_t c = cnt[d];
      if (c) {
        const uint32_t e = off[d], s = e - c;
        big_load<LPL>(bkt, bases + (size_t)list[s] * L, lane);
        for (uint32_t i = s + 1; i < e; ++i) {
          big_load<LPL>(x, bases + (size_t)list[i] * L, lane);
          mont_mul<LPL>(bkt, bkt, x, n_, np, lane);
        }
        if (has_run) mont_mul<LPL>(run, run, bkt, n_, np, lane);
        else big_copy<LPL>(run, bkt);
        has_run = true;
      }
      if (has_run) {
        if (has_tot) mont_mul<LPL>(tot, tot, run, n_, np, lane);
        else big_copy<LPL>(tot, run);
        has_tot = true;
      }
    }
    if (has_tot) big_store<LPL>(W + (size_t)task * L, tot, lane);
    if (lane == 0) flags[task] = has_tot ? 1 : 0;
    __syncwarp();
  }
}

template <int LPL>
__global__ void __launch_bounds__(128)
combine_windows_kernel(const uint32_t* __restrict__ W, const uint8_t* __restrict__ flags,
                       int64_t rows, int nwin, const uint32_t* __restrict__ N, uint32_t np,
                       uint32_t* __restrict__ out, const int32_t* __restrict__ row_ids,
                       int keep_mont, const uint32_t* __restrict__ one_m) {
  constexpr int L = 32 * LPL;
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= rows) return;
  uint32_t n_[LPL], acc[LPL], x[LPL];
  big_load<LPL>(n_, N, lane);
  bool has = false;
  for (int w = nwin - 1; w >= 0; --w) {
    if (has)
      for (int s = 0; s < kWin; ++s) mont_mul<LPL>(acc, acc, acc, n_, np, lane);
    const int64_t task = g * nwin + w;
    if (flags[task]) {
      big_load<LPL>(x, W + (size_t)task * L, lane);
      if (has) mont_mul<LPL>(acc, acc, x, n_, np, lane);
      else big_copy<LPL>(acc, x);
      has = true;
    }
  }
  if (keep_mont) {
    if (!has) big_load<LPL>(acc, one_m, lane);   // Montgomery form of 1
  } else if (has) {
    big_set_small<LPL>(x, 1, lane);
    mont_mul<LPL>(acc, acc, x, n_, np, lane);  // leave Montgomery form
  } else {
    big_set_small<LPL>(acc, 1, lane);          // all exponents zero -> 1 (paillier.py:145-146)
  }
  const int64_t orow = row_ids ? (int64_t)row_ids[g] : g;
  big_store<LPL>(out + orow * L, acc, lane);
}

// Slot-decomposed hint: k_g = prod_j W[g*cap + j]^(2^(32 j)) mod N, with the
// per-slot products W (Montgomery form) from a 32-bit multiexp per DB row.
// Horner from the top slot: acc = acc^(2^32) * W_j. One warp per group.
// Exponent of the Horner step (gamma), up to 256 bits, passed by value.
struct GammaExp {
  uint32_t w[8];
  int nbits;
};

// One client's slot-combine operands (the batched launch reads them per blockIdx.y).
struct SlotClient {
  const uint32_t* W;
  const uint32_t* N;
  uint32_t* out;
  uint32_t np;
};

template <int LPL>
__global__ void __launch_bounds__(128)
slot_combine_kernel(const SlotClient* __restrict__ cls, SlotClient one, int cap,
                    const int32_t* __restrict__ group_ids, int64_t ngroups, GammaExp gm) {
  constexpr int L = 32 * LPL;
// latency-bound (one warp per group, few groups): the 4x-unrolled CIOS is
// 17.4 -> 15.1 ms for one client at 1 GiB (tools/slot_probe.py, bit-identical)
#define MM(...) mont_mul<LPL, 4>(__VA_ARGS__)
  const int lane = threadIdx.x & 31;
  const int64_t gi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gi >= ngroups) return;
  const SlotClient c = cls ? cls[blockIdx.y] : one;
  const uint32_t np = c.np;
  const int64_t g = group_ids ? (int64_t)group_ids[gi] : gi;
  uint32_t n_[LPL], acc[LPL], x[LPL];
  big_load<LPL>(n_, c.N, lane);
  const uint32_t* Wg = c.W + (size_t)g * cap * L;
  big_load<LPL>(acc, Wg + (size_t)(cap - 1) * L, lane);
  uint32_t base[LPL];
  for (int j = cap - 2; j >= 0; --j) {
    // acc = acc^gamma (left-to-right binary; gamma = 2^32 is 32 squarings)
    big_copy<LPL>(base, acc);
    for (int bit = gm.nbits - 2; bit >= 0; --bit) {
      MM(acc, acc, acc, n_, np, lane);
      if ((gm.w[bit >> 5] >> (bit & 31)) & 1u) MM(acc, acc, base, n_, np, lane);
    }
    big_load<LPL>(x, Wg + (size_t)j * L, lane);
    MM(acc, acc, x, n_, np, lane);
  }
  big_set_small<LPL>(x, 1, lane);
  MM(acc, acc, x, n_, np, lane);  // leave Montgomery form
  big_store<LPL>(c.out + g * L, acc, lane);
}
#undef MM

// ---- fixed-base slot multiexp (w = 8) -------------------------------------
// P[i][k] = ck_k^(2^(8 i)) in Montgomery form (i < 4), one warp per base.
template <int LPL>
__global__ void __launch_bounds__(128)
pow8_table_kernel(const uint32_t* __restrict__ bases, int64_t n, const uint32_t* __restrict__ N,
                  uint32_t np, const uint32_t* __restrict__ r2, uint32_t* __restrict__ P) {
  constexpr int L = 32 * LPL;
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= n) return;
  uint32_t n_[LPL], a[LPL], b[LPL];
  big_load<LPL>(n_, N, lane);
  big_load<LPL>(a, bases + k * L, lane);
  big_load<LPL>(b, r2, lane);
  mont_mul<LPL>(a, a, b, n_, np, lane);
  big_store<LPL>(P + (size_t)k * L, a, lane);
  for (int i = 1; i < 4; ++i) {
    for (int s = 0; s < 8; ++s) mont_mul<LPL>(a, a, a, n_, np, lane);
    big_store<LPL>(P + ((size_t)i * n + k) * L, a, lane);
  }
}

// W[r] = prod_{i<4, k<n} P[i][k]^(byte_i(H[r][k])) -- one Pippenger with 255
// buckets over the 4n (i, k) digit pairs of the 32-bit exponent row r: no
// per-window squarings, ~4n + 510 multiplications. One warp per row; the
// digits are counting-sorted in shared memory (u16 indices i*n + k).
// Smem per warp: cnt[256] + off[256] (u32) + list[4n] (u16).
template <int LPL>
__global__ void __launch_bounds__(128)
slot_fixed_kernel(const uint32_t* __restrict__ P, int64_t n, const uint32_t* __restrict__ E,
                  int64_t rs, const int32_t* __restrict__ row_ids, int64_t rows,
                  const uint32_t* __restrict__ N, uint32_t np, const uint32_t* __restrict__ one_m,
                  uint32_t* __restrict__ out, int S, uint32_t* __restrict__ part) {
  constexpr int L = 32 * LPL;
  extern __shared__ uint32_t smem_u32[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const int64_t per_warp = 512 + (4 * n + 1) / 2;
  uint32_t* cnt = smem_u32 + (size_t)wid * per_warp;
  uint32_t* off = cnt + 256;
  uint16_t* list = reinterpret_cast<uint16_t*>(off + 256);
  uint32_t n_[LPL];
  big_load<LPL>(n_, N, lane);
  // S > 1 (few rows): digit range s of the row's 255 buckets per warp,
  // partial products to part[(gi*S + s)], multiplied together by slot_parts_kernel
  for (int64_t wi = (int64_t)blockIdx.x * wpb + wid; wi < rows * S;
       wi += (int64_t)gridDim.x * wpb) {
    const int64_t gi = wi / S;
    const int sp = (int)(wi - gi * S);
    const uint32_t lo = 1u + (uint32_t)(255 * sp / S), hi = (uint32_t)(255 * (sp + 1) / S);
    const int64_t r = row_ids ? (int64_t)row_ids[gi] : gi;
    const uint32_t* er = E + r * rs;
#pragma unroll
    for (int q = 0; q < 8; ++q) cnt[lane * 8 + q] = 0;
    __syncwarp();
    for (int64_t k = lane; k < n; k += 32) {
      const uint32_t w = er[k];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t d = (w >> (8 * i)) & 0xffu;
        if (d >= lo && d <= hi) atomicAdd(&cnt[d], 1u);
      }
    }
    __syncwarp();
    // exclusive scan of cnt[0..255]: lane holds entries 8*lane .. 8*lane+7
    uint32_t c[8], run = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      c[q] = cnt[lane * 8 + q];
      run += c[q];
    }
    uint32_t incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(ZPIR_FULL, incl, o);
      if (lane >= o) incl += v;
    }
    uint32_t base = incl - run;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      off[lane * 8 + q] = base;
      base += c[q];
    }
    __syncwarp();
    for (int64_t k = lane; k < n; k += 32) {
      const uint32_t w = er[k];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t d = (w >> (8 * i)) & 0xffu;
        if (d >= lo && d <= hi) list[atomicAdd(&off[d], 1u)] = (uint16_t)(i * n + k);
      }
    }
    __syncwarp();
    bool has_run = false, has_tot = false;
    uint32_t run_[LPL], tot[LPL], bkt[LPL], x[LPL];
    for (int d = (int)hi; d >= (int)lo; --d) {
      const uint32_t cd = cnt[d];
      if (cd) {
        const uint32_t e = off[d], s0 = e - cd;
        big_load<LPL>(bkt, P + (size_t)list[s0] * L, lane);
        for (uint32_t i = s0 + 1; i < e; ++i) {
          big_load<LPL>(x, P + (size_t)list[i] * L, lane);
          mont_mul<LPL>(bkt, bkt, x, n_, np, lane);
        }
        if (has_run) mont_mul<LPL>(run_, run_, bkt, n_, np, lane);
        else big_copy<LPL>(run_, bkt);
        has_run = true;
      }
      if (has_run) {
        if (has_tot) mont_mul<LPL>(tot, tot, run_, n_, np, lane);
        else big_copy<LPL>(tot, run_);
        has_tot = true;
      }
    }
    if (!has_tot) big_load<LPL>(tot, one_m, lane);
    if (S == 1) {
      big_store<LPL>(out + r * L, tot, lane);
    } else {
      // tot = prod_{d in [lo, hi]} B_d^(d - lo + 1); times run^(lo - 1) gives
      // prod B_d^d over the range (left-to-right binary, lo - 1 < 256)
      if (has_run && lo > 1) {
        const uint32_t e = lo - 1;
        big_copy<LPL>(x, run_);
        for (int b = 30 - __clz(e); b >= 0; --b) {
          mont_mul<LPL>(x, x, x, n_, np, lane);
          if ((e >> b) & 1u) mont_mul<LPL>(x, x, run_, n_, np, lane);
        }
        mont_mul<LPL>(tot, tot, x, n_, np, lane);
      }
      big_store<LPL>(part + (gi * S + sp) * L, tot, lane);
    }
    __syncwarp();
  }
}

// out[row_ids[gi] or gi] = prod_s part[gi*S + s] (Montgomery form), one warp per row.
template <int LPL>
__global__ void __launch_bounds__(128)
slot_parts_kernel(const uint32_t* __restrict__ part, int S, const int32_t* __restrict__ row_ids,
                  int64_t rows, const uint32_t* __restrict__ N, uint32_t np,
                  uint32_t* __restrict__ out) {
  constexpr int L = 32 * LPL;
  const int lane = threadIdx.x & 31;
  const int64_t gi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gi >= rows) return;
  uint32_t n_[LPL], acc[LPL], x[LPL];
  big_load<LPL>(n_, N, lane);
  big_load<LPL>(acc, part + gi * S * L, lane);
  for (int sp = 1; sp < S; ++sp) {
    big_load<LPL>(x, part + (gi * S + sp) * L, lane);
    mont_mul<LPL>(acc, acc, x, n_, np, lane);
  }
  const int64_t r = row_ids ? (int64_t)row_ids[gi] : gi;
  big_store<LPL>(out + r * L, acc, lane);
}

int64_t multiexp_workspace_bytes(int64_t n, int64_t rows, int elimbs, int limbs) {
  const int64_t nwin = ceil_div((int64_t)32 * elimbs, kWin);
  const int64_t a = ((n * limbs * 4 + 255) / 256) * 256;
  const int64_t w = ((rows * nwin * limbs * 4 + 255) / 256) * 256;
  const int64_t f = ((rows * nwin + 255) / 256) * 256;
  return a + w + f;
}

#define ZPIR_LPL_DISPATCH2(LPLV, ...)                                  \
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

int multiexp_rows_launch(const uint32_t* bases, int64_t n, const uint32_t* E,
                         const int32_t* row_ids, int64_t rows, int64_t rs, int64_t bs, int64_t ls,
                         int elimbs, int limbs, const uint32_t* N, uint32_t np,
                         const uint32_t* r2, const uint32_t* one_m, int keep_mont, uint32_t* out,
                         void* ws, int64_t ws_bytes, cudaStream_t st) {
  if (limbs % 32 || n <= 0 || rows <= 0 || elimbs <= 0 || (keep_mont && !one_m)) {
    set_error("multiexp: bad shapes (n=%lld rows=%lld elimbs=%d limbs=%d)", (long long)n,
              (long long)rows, elimbs, limbs);
    return kErrInput;
  }
  if (ws_bytes < multiexp_workspace_bytes(n, rows, elimbs, limbs)) {
    set_error("multiexp: workspace too small");
    return kErrInput;
  }
  const int nwin = (int)ceil_div((int64_t)32 * elimbs, kWin);
  uint8_t* p = static_cast<uint8_t*>(ws);
  uint32_t* bm = reinterpret_cast<uint32_t*>(p);
  p += ((n * limbs * 4 + 255) / 256) * 256;
  uint32_t* W = reinterpret_cast<uint32_t*>(p);
  p += ((rows * nwin * limbs * 4 + 255) / 256) * 256;
  uint8_t* flags = p;
  const size_t smem = (size_t)4 * (2 * kBuckets + n) * sizeof(uint32_t);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  ZPIR_LPL_DISPATCH2(limbs / 32, {
    to_mont_kernel<LPL><<<(unsigned)ceil_div(n, 4), 128, 0, st>>>(bases, n, N, np, r2, bm);
    if (int e = check_launch("multiexp to_mont")) return e;
    cudaFuncSetAttribute(window_kernel<LPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    const int64_t tasks = rows * nwin;
    const int64_t grid = std::min<int64_t>(ceil_div(tasks, 4), (int64_t)sms * 32);
    window_kernel<LPL><<<(unsigned)grid, 128, smem, st>>>(bm, n, E, rows, rs, bs, ls, elimbs,
                                                          nwin, N, np, W, flags, row_ids);
    if (int e = check_launch("multiexp window")) return e;
    combine_windows_kernel<LPL><<<(unsigned)ceil_div(rows, 4), 128, 0, st>>>(
        W, flags, rows, nwin, N, np, out, row_ids, keep_mont, one_m);
  });
  return check_launch("multiexp combine");
}

int multiexp_launch(const uint32_t* bases, int64_t n, const uint32_t* E, int64_t rows, int64_t rs,
                    int64_t bs, int64_t ls, int elimbs, int limbs, const uint32_t* N, uint32_t np,
                    const uint32_t* r2, uint32_t* out, void* ws, int64_t ws_bytes,
                    cudaStream_t st) {
  return multiexp_rows_launch(bases, n, E, nullptr, rows, rs, bs, ls, elimbs, limbs, N, np, r2,
                              nullptr, 0, out, ws, ws_bytes, st);
}

// P = pow8 table (4 x n x limbs) of the canonical bases (Montgomery form).
int pow8_table_launch(const uint32_t* bases, int64_t n, int limbs, const uint32_t* N, uint32_t np,
                      const uint32_t* r2, uint32_t* P, cudaStream_t st) {
  if (limbs % 32 || n <= 0) {
    set_error("pow8_table: bad shapes");
    return kErrInput;
  }
  ZPIR_LPL_DISPATCH2(limbs / 32, {
    pow8_table_kernel<LPL><<<(unsigned)ceil_div(n, 4), 128, 0, st>>>(bases, n, N, np, r2, P);
  });
  return check_launch("pow8_table");
}

// W[row] (Montgomery form) for the listed 32-bit exponent rows E[row*rs + k].
int slot_fixed_launch(const uint32_t* P, int64_t n, const uint32_t* E, int64_t rs,
                      const int32_t* row_ids, int64_t rows, int limbs, const uint32_t* N,
                      uint32_t np, const uint32_t* one_m, uint32_t* W, cudaStream_t st) {
  if (limbs % 32 || n <= 0 || rows <= 0 || 4 * n > 65536) {
    set_error("slot_fixed: bad shapes (n=%lld rows=%lld)", (long long)n, (long long)rows);
    return kErrInput;
  }
  const size_t smem = (size_t)4 * (512 + (4 * n + 1) / 2) * sizeof(uint32_t);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // split each row's buckets over S warps when there are too few rows to fill
  // the GPU (small DBs, incremental refreshes of a few hundred rows)
  const int64_t target = (int64_t)sms * 32;
  int S = 1;
  while (S < 8 && rows * S < target) S *= 2;
  uint32_t* part = nullptr;
  if (S > 1 && cudaMallocAsync(reinterpret_cast<void**>(&part), (size_t)rows * S * limbs * 4, st) !=
                   cudaSuccess) {
    cudaGetLastError();
    S = 1;
    part = nullptr;
  }
  ZPIR_LPL_DISPATCH2(limbs / 32, {
    cudaFuncSetAttribute(slot_fixed_kernel<LPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    const int64_t grid = std::min<int64_t>(ceil_div(rows * S, 4), (int64_t)sms * 16);
    slot_fixed_kernel<LPL><<<(unsigned)grid, 128, smem, st>>>(P, n, E, rs, row_ids, rows, N, np,
                                                              one_m, W, S, part);
    if (S > 1)
      slot_parts_kernel<LPL><<<(unsigned)ceil_div(rows, 4), 128, 0, st>>>(part, S, row_ids, rows,
                                                                          N, np, W);
  });
  if (part) cudaFreeAsync(part, st);
  return check_launch("slot_fixed");
}

static int slot_combine_run(const SlotClient* cls, SlotClient one, int clients, int cap,
                            const int32_t* group_ids, int64_t ngroups, int limbs,
                            const uint32_t* gamma, int gamma_bits, cudaStream_t st) {
  if (limbs % 32 || cap <= 0 || ngroups <= 0 || gamma_bits < 1 || gamma_bits > 256 ||
      clients <= 0 || clients > 65535) {
    set_error("slot_combine: bad shapes (gamma_bits=%d clients=%d)", gamma_bits, clients);
    return kErrInput;
  }
  GammaExp gm{};
  for (int i = 0; i < (gamma_bits + 31) / 32; ++i) gm.w[i] = gamma[i];
  gm.nbits = gamma_bits;
  const dim3 grid((unsigned)ceil_div(ngroups, 4), (unsigned)clients);
  ZPIR_LPL_DISPATCH2(limbs / 32, {
    slot_combine_kernel<LPL><<<grid, 128, 0, st>>>(cls, one, cap, group_ids, ngroups, gm);
  });
  return check_launch("slot_combine");
}

int slot_combine_launch(const uint32_t* W, int cap, const int32_t* group_ids, int64_t ngroups,
                        int limbs, const uint32_t* N, uint32_t np, const uint32_t* gamma,
                        int gamma_bits, uint32_t* out, cudaStream_t st) {
  const SlotClient one{W, N, out, np};
  return slot_combine_run(nullptr, one, 1, cap, group_ids, ngroups, limbs, gamma, gamma_bits, st);
}

// Several clients (same key width, same groups) in one launch, blockIdx.y =
// client: the latency-bound Horner chains of all clients fill the GPU together.
int slot_combine_many_launch(int clients, const uint32_t* const* W, const uint32_t* const* N,
                             const uint32_t* np, uint32_t* const* out, int cap,
                             const int32_t* group_ids, int64_t ngroups, int limbs,
                             const uint32_t* gamma, int gamma_bits, cudaStream_t st) {
  if (clients <= 0) {
    set_error("slot_combine_many: no clients");
    return kErrInput;
  }
  std::vector<SlotClient> h(clients);
  for (int c = 0; c < clients; ++c) h[c] = {W[c], N[c], out[c], np[c]};
  SlotClient* d = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(SlotClient) * clients, st) !=
          cudaSuccess ||
      cudaMemcpyAsync(d, h.data(), sizeof(SlotClient) * clients, cudaMemcpyHostToDevice, st) !=
          cudaSuccess) {
    if (d) cudaFreeAsync(d, st);
    return check_launch("slot_combine_many setup");
  }
  const int rc = slot_combine_run(d, h[0], clients, cap, group_ids, ngroups, limbs, gamma,
                                  gamma_bits, st);
  cudaFreeAsync(d, st);
  return rc;
}

}  // namespace zpir
