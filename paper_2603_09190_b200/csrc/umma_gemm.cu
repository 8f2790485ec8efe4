// tcgen05 (UMMA) int8 GEMM with byte-limb epilogues -- the tensor-core engine
// behind the online GEMV, batched queries, the global hint and the answer
// compression.
//
//   P[r, j] = sum_k A[r, k] * B[j, k]      u8 x u8 -> s32 in TMEM (kind::i8)
//
// A = DB (rows x ld bytes) or H viewed as bytes (rows x 4n); B holds byte
// planes of the other operand so that every 32-bit quantity is an exact sum
// of shifted byte products:
//   * u32 vector x (query qu, or a column of A): plane l = byte l of x, and
//     sum_l 2^(8l) P[r, 4v+l] = (A x_v)[r] (mod 2^32)          -> LIMB modes
//   * big integer ck_o[k] (lm 32-bit limbs): H[r,k] = sum_a 2^(8a) byte_a,
//     B[b, (k,a)] = byte_(b-a)(ck_o[k]) so sum_b 2^(8b) P[r, b]
//     = sum_k H[r,k] ck_o[k] = y_r exactly                      -> BIGINT mode
// Every product is < 2^16 and the K extents keep s32 partial sums far below
// 2^31 for the BIGINT mode (4n <= 2^14 bytes: < 2^30); the LIMB modes only
// need sums mod 2^32, which wrapping s32 accumulation (no .satfinite) gives.
//
// Kernel structure (one CTA per SM, 192 threads, persistent):
//   warp 0  TMA producer: A tile 128 x 128 B and B tile NT x 128 B per stage,
//           SWIZZLE_128B, mbarrier complete_tx
//   warp 1  TMEM allocator + single-thread MMA issuer: 4 x (M=128, N<=256,
//           K=32) MMAs per 128-byte k-block, tcgen05.commit frees the stage
//   warps 2-5  epilogue: tcgen05.ld 32x32b (warp w owns TMEM lanes 32(w%4)..)
//           -> limb recombination -> global (store or wrapping atomic add)
// Work: persistent CTAs walk a contiguous range of (tile, k-block) units
// ("stream-K", split = 1; exact because the LIMB outputs are sums mod 2^32
// and are combined with wrapping atomics) or of whole tiles (split = 0).
#include <cudaTypedefs.h>
#include <cstdlib>

#include <algorithm>

#include "umma.cuh"

namespace zpir {

using namespace sm100;

enum UmmaMode : int {
  kLimbCols = 0,     // out[(n*NT/4 + j) * ldo + r]  (+)= sum_l P[r,4j+l] << 8l
  kLimbRowsNeg = 1,  // out[r * ldo + n*NT/4 + j]  = qmask & -(sum_l ...)   (whole tiles)
  kBigint = 2        // z[r * wz + i] = limbs of sum_b P[r,b] << 8b
};

struct UmmaArgs {
  int m_tiles, n_tiles, kblocks;
  int split;
  uint32_t* out;
  int64_t ldo;
  int nout;
  uint32_t qmask;
  const uint32_t* b;
  int wz;
  int64_t zq;  // BIGINT: per-N-tile (= per query) stride of z
  int a_keep;  // BIGINT pair kernel: L2 evict_last for the A operand (H)
};

constexpr int kBM = 128;   // rows per tile (TMEM lanes)
constexpr int kBK = 128;   // bytes of K per stage (one 128-byte swizzle row)
constexpr int kThreads = 192;

template <int NT>
struct UmmaCfg {
  static constexpr int kABytes = kBM * kBK;
  static constexpr int kBBytes = NT * kBK;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = std::min(12, (200 * 1024) / kStageBytes);
  // Two accumulator buffers when they fit side by side in the 512 TMEM
  // columns; for 256 < NT <= 272 they overlap by kOv = 2 NT - 512 <= 32
  // columns at [512 - NT, NT): the epilogue drains that overlap first and
  // releases it early (bar "oempty") so the next tile's MMAs can start.
  static constexpr int kAcc = (2 * NT <= 512 + 32) ? 2 : 1;
  static constexpr int kOv = (kAcc == 2 && 2 * NT > 512) ? 2 * NT - 512 : 0;
  static constexpr int kAccOff1 = (kOv > 0) ? 512 - NT : NT;
  static constexpr int kTmemCols = (kAcc * NT <= 32) ? 32 : (kAcc * NT <= 64) ? 64
                                 : (kAcc * NT <= 128) ? 128 : (kAcc * NT <= 256) ? 256 : 512;
  // TMA box height for B: largest multiple-of-8 divisor of NT that is <= 256
  static constexpr int boxB() {
    for (int h = 256; h >= 8; h -= 8)
      if (NT % h == 0) return h;
    return 8;
  }
  static constexpr int kBoxB = boxB();
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
};

struct SegIter {
  int64_t u, u1;
  int kb;
  bool split;
  __device__ bool next(int64_t& t, int& k0, int& k1) {
    if (u >= u1) return false;
    if (split) {
      t = u / kb;
      k0 = (int)(u - t * kb);
      const int64_t left = u1 - u;
      k1 = (int)((int64_t)kb < k0 + left ? (int64_t)kb : k0 + left);
      u += k1 - k0;
    } else {
      t = u;
      k0 = 0;
      k1 = kb;
      u += 1;
    }
    return true;
  }
};

__device__ __forceinline__ SegIter seg_range(const UmmaArgs& a) {
  const int64_t T = (int64_t)a.m_tiles * a.n_tiles;
  const int64_t U = a.split ? T * a.kblocks : T;
  const int64_t G = gridDim.x, s = blockIdx.x;
  SegIter it;
  it.u = s * U / G;
  it.u1 = (s + 1) * U / G;
  it.kb = a.kblocks;
  it.split = a.split != 0;
  return it;
}

template <int NT, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
umma_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                 const UmmaArgs args) {
  using C = UmmaCfg<NT>;
  static_assert(C::kOv == 0 || MODE == kBigint, "overlapped accumulators need the BIGINT epilogue");
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::kStages * C::kBBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kAcc;
  uint64_t* oempty = tempty + C::kAcc;
  uint32_t* tbase_smem = reinterpret_cast<uint32_t*>(oempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::kAcc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    mbar_init(oempty, 128);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tbase_smem, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tbase_smem;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      const uint64_t pol_a = l2_evict_first();
      SegIter it = seg_range(args);
      int64_t t;
      int k0, k1, stage = 0;
      uint32_t phase = 0;
      while (it.next(t, k0, k1)) {
        const int m = (int)(t / args.n_tiles), n = (int)(t % args.n_tiles);
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::kStageBytes);
          tma_load_2d_hint(sA + stage * C::kABytes, &mapA, &full[stage], kb * kBK, m * kBM, pol_a);
#pragma unroll
          for (int p = 0; p < NT / C::kBoxB; ++p)
            tma_load_2d(sB + stage * C::kBBytes + p * C::kBoxB * kBK, &mapB, &full[stage],
                        kb * kBK, n * NT + p * C::kBoxB);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      SegIter it = seg_range(args);
      int64_t t;
      int k0, k1, stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      int seg = 0;
      while (it.next(t, k0, k1)) {
        mbar_wait(&tempty[acc], aphase ^ 1);
        if constexpr (C::kOv > 0) {
          // the previous segment (other buffer) must have drained the overlap
          if (seg > 0) mbar_wait(oempty, (uint32_t)((seg - 1) & 1));
        }
        tc_fence_after();
        const uint32_t d = tbase + (uint32_t)(acc * C::kAccOff1);
        ++seg;
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * C::kABytes);
          const uint32_t b0 = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / 32; ++k) {
            const uint64_t ad = desc_sw128(a0 + k * 32);
            // N > 256: two MMAs of balanced width (multiples of 16), e.g. 144 + 128
            constexpr int kN0 = NT <= 256 ? NT : ((NT / 2 + 15) / 16) * 16;
            const uint32_t acc_on = (kb > k0 || k > 0) ? 1u : 0u;
            umma_i8(d, ad, desc_sw128(b0 + k * 32), idesc_u8(kBM, kN0), acc_on);
            if constexpr (NT > kN0)
              umma_i8(d + kN0, ad, desc_sw128(b0 + kN0 * kBK + k * 32),
                      idesc_u8(kBM, NT - kN0), acc_on);
          }
          umma_commit(&empty[stage]);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        if (++acc == C::kAcc) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5, 128 threads) ----------------
    const int quarter = warp & 3;
    const int lrow = quarter * 32 + lane;
    SegIter it = seg_range(args);
    int64_t t;
    int k0, k1, acc = 0;
    uint32_t aphase = 0;
    while (it.next(t, k0, k1)) {
      const int m = (int)(t / args.n_tiles), n = (int)(t % args.n_tiles);
      const int64_t row = (int64_t)m * kBM + lrow;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t taddr = tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * C::kAccOff1);
      if constexpr (MODE == kLimbCols || MODE == kLimbRowsNeg) {
        const bool partial = args.split != 0;
#pragma unroll 1
        for (int c0 = 0; c0 < NT; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(taddr + c0, r);
          tmem_wait_ld();
          uint32_t v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            v[j] = r[4 * j] + (r[4 * j + 1] << 8) + (r[4 * j + 2] << 16) + (r[4 * j + 3] << 24);
          const int jg = n * (NT / 4) + c0 / 4;
          if constexpr (MODE == kLimbCols) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (c0 / 4 + j < args.nout) {
                uint32_t* dst = args.out + (int64_t)(jg + j) * args.ldo + row;
                if (partial) atomicAdd(dst, v[j]);
                else *dst = v[j];
              }
            }
          } else {
            uint4 w = make_uint4((0u - v[0]) & args.qmask, (0u - v[1]) & args.qmask,
                                 (0u - v[2]) & args.qmask, (0u - v[3]) & args.qmask);
            if (jg + 3 < args.nout) {
              *reinterpret_cast<uint4*>(args.out + row * args.ldo + jg) = w;
            } else {
              const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
              for (int j = 0; j < 4; ++j)
                if (jg + j < args.nout) args.out[row * args.ldo + jg + j] = wv[j];
            }
          }
        }
      } else {
        // BIGINT: z_r = sum_b P[r, b] 2^(8b), carry-propagated (b is added by
        // the group stage, so this GEMM does not depend on the GEMV)
        constexpr int kOvChunks = C::kOv / 16;
        uint32_t ov[kOvChunks > 0 ? kOvChunks : 1][16];
        const int first = (acc == 0) ? (NT - C::kOv) : 0;
        if constexpr (kOvChunks > 0) {
          // drain the TMEM columns shared with the other buffer first
#pragma unroll
          for (int q = 0; q < kOvChunks; ++q) tmem_ld16(taddr + first + 16 * q, ov[q]);
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive(oempty);
        }
        unsigned long long carry = 0;
        uint32_t* zr = args.out + (int64_t)n * args.zq + row * args.wz;
#pragma unroll 1
        for (int c0 = 0; c0 < NT; c0 += 16) {
          uint32_t r[16];
          const bool in_ov = kOvChunks > 0 && c0 >= first && c0 < first + C::kOv;
          if (in_ov) {
            const int qi = (c0 - first) >> 4;
#pragma unroll
            for (int q = 0; q < (kOvChunks > 0 ? kOvChunks : 1); ++q)
              if (q == qi)
#pragma unroll
                for (int i = 0; i < 16; ++i) r[i] = ov[q][i];
          } else {
            tmem_ld16(taddr + c0, r);
            tmem_wait_ld();
          }
          uint32_t limb[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const unsigned long long s = (unsigned long long)r[4 * i] +
                                         ((unsigned long long)r[4 * i + 1] << 8) +
                                         ((unsigned long long)r[4 * i + 2] << 16) +
                                         ((unsigned long long)r[4 * i + 3] << 24) + carry;
            limb[i] = (uint32_t)s;
            carry = s >> 32;
          }
          const int li = c0 / 4;
          if (li + 3 < args.wz) {
            *reinterpret_cast<uint4*>(zr + li) = make_uint4(limb[0], limb[1], limb[2], limb[3]);
          } else {
            for (int i = 0; i < 4; ++i)
              if (li + i < args.wz) zr[li + i] = limb[i];
          }
        }
        for (int li = NT / 4; li < args.wz; ++li) {
          zr[li] = (uint32_t)carry;
          carry >>= 32;
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == C::kAcc) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, C::kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// CTA-pair variant of the BIGINT (answer compression) GEMM: tcgen05.mma
// cta_group::2, M = 256 rows per pair tile (128 per CTA, its own TMEM lanes),
// B split by N halves (each CTA stages NT/2 rows of every k-block: half the
// per-SM operand feed of the single-CTA kernel, which is feed-bound).
// Cluster (2,1,1) = one TPC. The leader (rank 0) owns full[] and issues the
// MMAs; both CTAs' TMA loads signal the leader's full[s]; the leader's
// commits arrive on empty[] / tfull[] of both CTAs (multicast); both CTAs'
// epilogues arrive on the leader's tempty[] / oempty.
template <int NT>
struct PairCfg {
  static constexpr int kP0 = NT < 256 ? NT : 256;          // first MMA's N
  static constexpr int kP1 = NT - kP0;                     // second MMA's N (0 if none)
  static constexpr int kH0 = kP0 / 2, kH1 = kP1 / 2;       // rows per CTA of each part
  static constexpr int kABytes = kBM * kBK;
  static constexpr int kBBytes = (kH0 + kH1) * kBK;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = std::min(12, (200 * 1024) / kStageBytes);
  static constexpr int kAcc = UmmaCfg<NT>::kAcc;
  static constexpr int kOv = UmmaCfg<NT>::kOv;
  static constexpr int kAccOff1 = UmmaCfg<NT>::kAccOff1;
  static constexpr int kTmemCols = UmmaCfg<NT>::kTmemCols;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
  static_assert(kH0 % 8 == 0 && kH1 % 8 == 0, "B halves must be whole 8-row swizzle atoms");
};

template <int NT>
__global__ void __launch_bounds__(kThreads, 1)
umma_pair_bigint_kernel(const __grid_constant__ CUtensorMap mapA,
                        const __grid_constant__ CUtensorMap mapB0,
                        const __grid_constant__ CUtensorMap mapB1, const UmmaArgs args,
                        int64_t rows) {
  using C = PairCfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::kStages * C::kBBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kAcc;
  uint64_t* oempty = tempty + C::kAcc;
  uint32_t* tbase_smem = reinterpret_cast<uint32_t*>(oempty + 1);

  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB0);
    if (C::kH1) tma_prefetch(&mapB1);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::kAcc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 256);
    }
    mbar_init(oempty, 256);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(tbase_smem, C::kTmemCols);
  tc_fence_before();
  cluster_sync();   // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tbase = *tbase_smem;

  // pair work list: units = (pair tile, n) over m_tiles pair tiles of 256 rows
  UmmaArgs pa = args;
  const int npairs = (int)(gridDim.x >> 1), pid = (int)(blockIdx.x >> 1);
  SegIter it;
  {
    const int64_t T = (int64_t)pa.m_tiles * pa.n_tiles;
    it.u = pid * T / npairs;
    it.u1 = (pid + 1) * T / npairs;
    it.kb = pa.kblocks;
    it.split = false;
  }

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs) ----------------
      // H (the A operand, 4 bytes x n per DB row) is kept in L2 across
      // queries when args.a_keep: the concurrent GEMV streams the DB with
      // evict_first, so H lines survive and the answer reads less HBM
      const uint64_t pol_a = pa.a_keep ? l2_evict_last() : l2_evict_first();
      const uint64_t pol_b = l2_evict_last();
      int64_t t;
      int k0, k1, stage = 0;
      uint32_t phase = 0;
      while (it.next(t, k0, k1)) {
        const int m = (int)(t / pa.n_tiles), n = (int)(t % pa.n_tiles);
        const int arow = m * 2 * kBM + (int)rank * kBM;
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
          if (leader) mbar_expect_tx(&full[stage], 2 * C::kStageBytes);
          uint8_t* b = sB + stage * C::kBBytes;
          tma_load_2d_pair(sA + stage * C::kABytes, &mapA, fb, kb * kBK, arow, pol_a);
          tma_load_2d_pair(b, &mapB0, fb, kb * kBK, n * NT + (int)rank * C::kH0, pol_b);
          if (C::kH1)
            tma_load_2d_pair(b + C::kH0 * kBK, &mapB1, fb, kb * kBK,
                             n * NT + C::kP0 + (int)rank * C::kH1, pol_b);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader only) ----------------
      int64_t t;
      int k0, k1, stage = 0, acc = 0, seg = 0;
      uint32_t phase = 0, aphase = 0;
      while (it.next(t, k0, k1)) {
        mbar_wait(&tempty[acc], aphase ^ 1);
        if constexpr (C::kOv > 0) {
          if (seg > 0) mbar_wait(oempty, (uint32_t)((seg - 1) & 1));
        }
        tc_fence_after();
        const uint32_t d = tbase + (uint32_t)(acc * C::kAccOff1);
        ++seg;
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * C::kABytes);
          const uint32_t b0 = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / 32; ++k) {
            const uint64_t ad = desc_sw128(a0 + k * 32);
            const uint32_t acc_on = (kb > k0 || k > 0) ? 1u : 0u;
            umma_i8_pair(d, ad, desc_sw128(b0 + k * 32), idesc_u8(2 * kBM, C::kP0), acc_on);
            if (C::kP1)
              umma_i8_pair(d + C::kP0, ad, desc_sw128(b0 + C::kH0 * kBK + k * 32),
                           idesc_u8(2 * kBM, C::kP1 ? C::kP1 : 16), acc_on);
          }
          umma_commit_pair(&empty[stage], 0x3);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&tfull[acc], 0x3);
        if (++acc == C::kAcc) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5 of both CTAs) ----------------
    const int quarter = warp & 3;
    const int lrow = quarter * 32 + lane;
    const uint32_t tempty_l0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const uint32_t tempty_l1 = mapa_shared(smem_u32(&tempty[C::kAcc - 1]), 0);
    const uint32_t oempty_l = mapa_shared(smem_u32(oempty), 0);
    int64_t t;
    int k0, k1, acc = 0;
    uint32_t aphase = 0;
    while (it.next(t, k0, k1)) {
      const int m = (int)(t / pa.n_tiles), n = (int)(t % pa.n_tiles);
      const int64_t row = (int64_t)m * 2 * kBM + (int64_t)rank * kBM + lrow;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t taddr = tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * C::kAccOff1);
      constexpr int kOvChunks = C::kOv / 16;
      uint32_t ov[kOvChunks > 0 ? kOvChunks : 1][16];
      const int first = (acc == 0) ? (NT - C::kOv) : 0;
      if constexpr (kOvChunks > 0) {
#pragma unroll
        for (int q = 0; q < kOvChunks; ++q) tmem_ld16(taddr + first + 16 * q, ov[q]);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive_remote(oempty_l);
      }
      const bool live = row < rows;
      unsigned long long carry = 0;
      uint32_t* zr = pa.out + (int64_t)n * pa.zq + row * pa.wz;
#pragma unroll 1
      for (int c0 = 0; c0 < NT; c0 += 16) {
        uint32_t r[16];
        const bool in_ov = kOvChunks > 0 && c0 >= first && c0 < first + C::kOv;
        if (in_ov) {
          const int qi = (c0 - first) >> 4;
#pragma unroll
          for (int q = 0; q < (kOvChunks > 0 ? kOvChunks : 1); ++q)
            if (q == qi)
#pragma unroll
              for (int i = 0; i < 16; ++i) r[i] = ov[q][i];
        } else {
          tmem_ld16(taddr + c0, r);
          tmem_wait_ld();
        }
        uint32_t limb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const unsigned long long s = (unsigned long long)r[4 * i] +
                                       ((unsigned long long)r[4 * i + 1] << 8) +
                                       ((unsigned long long)r[4 * i + 2] << 16) +
                                       ((unsigned long long)r[4 * i + 3] << 24) + carry;
          limb[i] = (uint32_t)s;
          carry = s >> 32;
        }
        const int li = c0 / 4;
        if (live) {
          if (li + 3 < pa.wz) {
            *reinterpret_cast<uint4*>(zr + li) = make_uint4(limb[0], limb[1], limb[2], limb[3]);
          } else {
            for (int i = 0; i < 4; ++i)
              if (li + i < pa.wz) zr[li + i] = limb[i];
          }
        }
      }
      if (live)
        for (int li = NT / 4; li < pa.wz; ++li) {
          zr[li] = (uint32_t)carry;
          carry >>= 32;
        }
      tc_fence_before();
      mbar_arrive_remote(acc ? tempty_l1 : tempty_l0);
      if (++acc == C::kAcc) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
  tc_fence_before();
  cluster_sync();   // all MMAs consumed, all TMEM reads done in both CTAs
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tbase, C::kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// Planar BIGINT GEMM (the answer compression, default for lm = 32 / 64):
//   z_r = sum_a 2^(8a) * sum_j 2^(8j) P_a[r, j],  P_a[r, j] = sum_k Hp[r, a, k] * Bp[j, k]
// with Hp[r, a, k] = byte a of H[r, k] (byte planes, plane pitch np = n rounded
// up to 128) and Bp[j, k] = byte j of ck_o[k] (N = 4 lm = 128 / 256 rows). One
// tile = 4 passes (a = 0..3) of K = np into alternating TMEM buffers; every MMA
// is a single N = 4 lm instruction (no N = 16 remainder: the tensor pipe spends
// ~95 cycles on any MMA up to N ~ 144 and ~146 on N = 256, tools/probe_umma.py),
// 128 MMAs per 128-row tile instead of 256. The epilogue carry-propagates each
// pass's 4 lm columns and adds them, shifted by 8a bits, into the row's z limbs
// held in registers. |P_a| <= n * 255^2 < 2^31 for n <= 33025.
template <int NT>
__global__ void __launch_bounds__(kThreads, 1)
umma_planar_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const UmmaArgs args, int64_t np) {
  using C = UmmaCfg<NT>;
  static_assert(NT % 16 == 0 && NT <= 256 && C::kAcc == 2 && C::kOv == 0, "planar: N <= 256");
  constexpr int kLimbs = NT / 4;          // limbs of one pass's column block
  constexpr int kZ = kLimbs + 4;          // z row width (lm + 4)
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::kStages * C::kBBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kAcc;
  uint32_t* tbase_smem = reinterpret_cast<uint32_t*>(tempty + C::kAcc + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::kAcc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tbase_smem, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tbase_smem;
  const int kbp = (int)(np / kBK);        // k-blocks per plane pass

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      // batches: every H tile is re-read once per query by the same CTA (pair),
      // so H stays in L2 (the working set is ~1 MB per pair tile in flight)
      const uint64_t pol_a = args.a_keep ? l2_evict_last() : l2_evict_first();
      const uint64_t pol_b = l2_evict_last();
      SegIter it = seg_range(args);
      int64_t t;
      int k0, k1, stage = 0;
      uint32_t phase = 0;
      while (it.next(t, k0, k1)) {
        const int m = (int)(t / args.n_tiles), n = (int)(t % args.n_tiles);
        for (int a = 0; a < 4; ++a)
          for (int kb = 0; kb < kbp; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], C::kStageBytes);
            tma_load_2d_hint(sA + stage * C::kABytes, &mapA, &full[stage],
                             (int)(a * np) + kb * kBK, m * kBM, pol_a);
            tma_load_2d_hint(sB + stage * C::kBBytes, &mapB, &full[stage], kb * kBK, n * NT,
                             pol_b);
            if (++stage == C::kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: one accumulation group per (tile, plane) ----------------
      SegIter it = seg_range(args);
      int64_t t;
      int k0, k1, stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      const uint32_t idesc = idesc_u8(kBM, NT);
      while (it.next(t, k0, k1)) {
        for (int a = 0; a < 4; ++a) {
          mbar_wait(&tempty[acc], aphase ^ 1);
          tc_fence_after();
          const uint32_t d = tbase + (uint32_t)(acc * C::kAccOff1);
          for (int kb = 0; kb < kbp; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint64_t ad = desc_sw128(smem_u32(sA + stage * C::kABytes));
            const uint64_t bd = desc_sw128(smem_u32(sB + stage * C::kBBytes));
#pragma unroll
            for (int k = 0; k < kBK / 32; ++k)   // +32 bytes = +2 in the start-address field
              umma_i8(d, ad + 2 * k, bd + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
            umma_commit(&empty[stage]);
            if (++stage == C::kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit(&tfull[acc]);
          if (++acc == C::kAcc) {
            acc = 0;
            aphase ^= 1;
          }
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5): z row in registers ----------------
    const int quarter = warp & 3;
    const int lrow = quarter * 32 + lane;
    SegIter it = seg_range(args);
    int64_t t;
    int k0, k1, acc = 0;
    uint32_t aphase = 0;
    while (it.next(t, k0, k1)) {
      const int m = (int)(t / args.n_tiles), n = (int)(t % args.n_tiles);
      const int64_t row = (int64_t)m * kBM + lrow;
      uint32_t z[kZ];
#pragma unroll
      for (int i = 0; i < kZ; ++i) z[i] = 0;
#pragma unroll 1
      for (int a = 0; a < 4; ++a) {
        mbar_wait(&tfull[acc], aphase);
        tc_fence_after();
        const uint32_t taddr =
            tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * C::kAccOff1);
        const uint32_t sh = 8u * (uint32_t)a;
        unsigned long long carry = 0;   // column carry of this pass
        uint32_t prev = 0, c2 = 0;       // previous limb (for the shift), carry into z
#pragma unroll
        for (int c = 0; c < NT / 16; ++c) {
          uint32_t r[16];
          tmem_ld16(taddr + 16 * c, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const unsigned long long sum = (unsigned long long)r[4 * i] +
                                           ((unsigned long long)r[4 * i + 1] << 8) +
                                           ((unsigned long long)r[4 * i + 2] << 16) +
                                           ((unsigned long long)r[4 * i + 3] << 24) + carry;
            const uint32_t v = (uint32_t)sum;
            carry = sum >> 32;
            const uint32_t w = __funnelshift_l(prev, v, sh);
            const unsigned long long zz = (unsigned long long)z[4 * c + i] + w + c2;
            z[4 * c + i] = (uint32_t)zz;
            c2 = (uint32_t)(zz >> 32);
            prev = v;
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        // high limbs: the pass's final carry (< 2^32), then the shifted-out bits
        {
          const uint32_t v0 = (uint32_t)carry, v1 = (uint32_t)(carry >> 32);
          const uint32_t w[4] = {__funnelshift_l(prev, v0, sh), __funnelshift_l(v0, v1, sh),
                                 __funnelshift_l(v1, 0u, sh), 0u};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const unsigned long long zz = (unsigned long long)z[kLimbs + i] + w[i] + c2;
            z[kLimbs + i] = (uint32_t)zz;
            c2 = (uint32_t)(zz >> 32);
          }
        }
        if (++acc == C::kAcc) {
          acc = 0;
          aphase ^= 1;
        }
      }
      uint32_t* zr = args.out + (int64_t)n * args.zq + row * args.wz;
#pragma unroll
      for (int i = 0; i < kZ; i += 4) {
        if (args.a_keep)   // batches: stream z past L2 so the H tiles stay resident
          __stcs(reinterpret_cast<uint4*>(zr + i), make_uint4(z[i], z[i + 1], z[i + 2], z[i + 3]));
        else
          *reinterpret_cast<uint4*>(zr + i) = make_uint4(z[i], z[i + 1], z[i + 2], z[i + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, C::kTmemCols);
  }
}

// Planar BIGINT GEMM on CTA pairs (cta_group::2) for batches of queries: the
// umma_planar_kernel contract with M = 256 rows per pair tile (128 per CTA, each
// CTA's own TMEM lanes) and the ck_o byte rows (B, N = 4 lm) split by N halves.
//
// The B operand of a query -- its half, (NT / 2) x np bytes, 128 KB at n = 1024
// and 2048-bit m -- stays RESIDENT in shared memory while the pair sweeps row
// tiles, so a unit (pair tile, query) streams only its four H plane tiles
// through the ring: 512 KB per SM and 128 MMAs instead of 1 MB (the streaming
// form was bound by L2 -> SM traffic at ~0.5 of the tensor rate). Units are
// taken block of row tiles by block, each block's (query, tile) units split
// evenly over the pairs: a pair sees one or two queries per block (one or two B
// loads), and every block's H planes (<= 48 MB) are read from HBM once and then
// from L2 by all queries.
// Both CTAs' TMA loads complete on the leader's barriers; the leader's commits
// multicast to both CTAs; both epilogues arrive on the leader's tempty.
template <int NT>
struct PlanarPairCfg {
  static constexpr int kH = NT / 2;                       // B rows per CTA
  static constexpr int kABytes = kBM * kBK;               // one H plane k-block (16 KB)
  static constexpr int kBResMax = 128 * 1024;             // resident B half
  static constexpr int kStages = 6;
  static constexpr int kAcc = 2;
  static constexpr int kTmemCols = 512;
  static constexpr int kSmem = kBResMax + kStages * kABytes + 1024 + 256;
};

// The units (pair tile m, query q) of one pair, block of row tiles by block:
// every block's units, in (query, tile) order, are split evenly over all pairs,
// so the whole GPU works on one block's H planes at a time.
struct PlanarUnits {
  int m_tiles, nq, tb;   // tb = row tiles per block
  int npairs, pid;
  int blk = 0, t = 0;    // current block, its tile count
  int64_t r = 0, r1 = 0; // position / end of this pair's range in the block
  __device__ PlanarUnits(int m_tiles_, int nq_, int tb_, int npairs_, int pid_)
      : m_tiles(m_tiles_), nq(nq_), tb(tb_), npairs(npairs_), pid(pid_) {
    open();
  }
  __device__ void open() {
    t = min(tb, m_tiles - blk * tb);
    const int64_t U = t > 0 ? (int64_t)t * nq : 0;
    r = pid * U / npairs;
    r1 = (pid + 1) * U / npairs;
  }
  // next unit; `lastq` = the following unit (if any) belongs to another query
  __device__ bool next(int& m, int& q, bool& lastq) {
    while (t > 0 && r >= r1) {
      ++blk;
      open();
    }
    if (t <= 0) return false;
    q = (int)(r / t);
    m = blk * tb + (int)(r - (int64_t)q * t);
    ++r;
    lastq = r >= r1 || (int)(r / t) != q;
    return true;
  }
};

template <int NT>
__global__ void __launch_bounds__(kThreads, 1)
umma_planar_pair_kernel(const __grid_constant__ CUtensorMap mapA,
                        const __grid_constant__ CUtensorMap mapB, const UmmaArgs args,
                        int64_t np, int64_t rows, int tb) {
  using C = PlanarPairCfg<NT>;
  constexpr int kLimbs = NT / 4;
  constexpr int kZ = kLimbs + 4;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sB = smem;                                     // resident: kbp k-blocks of kH x 128 B
  uint8_t* sA = smem + C::kBResMax;
  uint64_t* full = reinterpret_cast<uint64_t*>(sA + C::kStages * C::kABytes);   // leader
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kAcc;                     // leader
  uint64_t* bfull = tempty + C::kAcc;                     // leader: the query's B landed in both CTAs
  uint64_t* bfree = bfull + 1;                            // every MMA reading the resident B done
  uint32_t* tbase_smem = reinterpret_cast<uint32_t*>(bfree + 1);

  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::kAcc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 256);
    }
    mbar_init(bfull, 1);
    mbar_init(bfree, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(tbase_smem, C::kTmemCols);
  tc_fence_before();
  cluster_sync();   // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tbase = *tbase_smem;
  const int kbp = (int)(np / kBK);        // k-blocks per plane pass

  PlanarUnits units(args.m_tiles, args.n_tiles, tb, (int)(gridDim.x >> 1), (int)(blockIdx.x >> 1));
  int m, q;
  bool lastq;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs) ----------------
      const uint64_t pol_a = args.a_keep ? l2_evict_last() : l2_evict_first();
      const uint64_t pol_b = l2_evict_last();
      int stage = 0, qcur = -1;
      uint32_t phase = 0, bph = 0;
      bool fresh = true;                   // the next unit starts a new resident B
      while (units.next(m, q, lastq)) {
        if (fresh) {
          // the resident B changes: wait until no MMA reads the old one
          if (qcur >= 0) {
            mbar_wait(bfree, bph);
            bph ^= 1;
          }
          qcur = q;
          const uint32_t fb = mapa_shared(smem_u32(bfull), 0);
          if (leader) mbar_expect_tx(bfull, 2u * (uint32_t)(kbp * C::kH * kBK));
          for (int kb = 0; kb < kbp; ++kb)
            tma_load_2d_pair(sB + kb * (C::kH * kBK), &mapB, fb, kb * kBK,
                             q * NT + (int)rank * C::kH, pol_b);
        }
        const int arow = m * 2 * kBM + (int)rank * kBM;
        for (int a = 0; a < 4; ++a)
          for (int kb = 0; kb < kbp; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (leader) mbar_expect_tx(&full[stage], 2 * C::kABytes);
            tma_load_2d_pair(sA + stage * C::kABytes, &mapA, mapa_shared(smem_u32(&full[stage]), 0),
                             (int)(a * np) + kb * kBK, arow, pol_a);
            if (++stage == C::kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        fresh = lastq;
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader): one group per (unit, plane) ----------------
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0, bph = 0;
      const uint32_t idesc = idesc_u8(2 * kBM, NT);
      bool fresh = true;
      while (units.next(m, q, lastq)) {
        if (fresh) {
          mbar_wait(bfull, bph);
          bph ^= 1;
          tc_fence_after();
        }
        for (int a = 0; a < 4; ++a) {
          mbar_wait(&tempty[acc], aphase ^ 1);
          tc_fence_after();
          const uint32_t d = tbase + (uint32_t)(acc * 256);
          for (int kb = 0; kb < kbp; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint64_t ad = desc_sw128(smem_u32(sA + stage * C::kABytes));
            const uint64_t bd = desc_sw128(smem_u32(sB + kb * (C::kH * kBK)));
#pragma unroll
            for (int k = 0; k < kBK / 32; ++k)
              umma_i8_pair(d, ad + 2 * k, bd + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
            umma_commit_pair(&empty[stage], 0x3);
            if (++stage == C::kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit_pair(&tfull[acc], 0x3);
          if (++acc == C::kAcc) {
            acc = 0;
            aphase ^= 1;
          }
        }
        // last unit on this resident B: it may be replaced once these MMAs are done
        if (lastq) umma_commit_pair(bfree, 0x3);
        fresh = lastq;
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5 of both CTAs): z row in registers ----------------
    const int quarter = warp & 3;
    const int lrow = quarter * 32 + lane;
    const uint32_t tempty_l[2] = {mapa_shared(smem_u32(&tempty[0]), 0),
                                  mapa_shared(smem_u32(&tempty[1]), 0)};
    int acc = 0;
    uint32_t aphase = 0;
    int n;
    while (units.next(m, n, lastq)) {
      const int64_t row = (int64_t)m * 2 * kBM + (int64_t)rank * kBM + lrow;
      uint32_t z[kZ];
#pragma unroll
      for (int i = 0; i < kZ; ++i) z[i] = 0;
#pragma unroll 1
      for (int a = 0; a < 4; ++a) {
        mbar_wait(&tfull[acc], aphase);
        tc_fence_after();
        const uint32_t taddr = tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * 256);
        const uint32_t sh = 8u * (uint32_t)a;
        unsigned long long carry = 0;
        uint32_t prev = 0, c2 = 0;
#pragma unroll
        for (int c = 0; c < NT / 16; ++c) {
          uint32_t r[16];
          tmem_ld16(taddr + 16 * c, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const unsigned long long sum = (unsigned long long)r[4 * i] +
                                           ((unsigned long long)r[4 * i + 1] << 8) +
                                           ((unsigned long long)r[4 * i + 2] << 16) +
                                           ((unsigned long long)r[4 * i + 3] << 24) + carry;
            const uint32_t v = (uint32_t)sum;
            carry = sum >> 32;
            const uint32_t w = __funnelshift_l(prev, v, sh);
            const unsigned long long zz = (unsigned long long)z[4 * c + i] + w + c2;
            z[4 * c + i] = (uint32_t)zz;
            c2 = (uint32_t)(zz >> 32);
            prev = v;
          }
        }
        tc_fence_before();
        mbar_arrive_remote(tempty_l[acc]);
        {
          const uint32_t v0 = (uint32_t)carry, v1 = (uint32_t)(carry >> 32);
          const uint32_t w[4] = {__funnelshift_l(prev, v0, sh), __funnelshift_l(v0, v1, sh),
                                 __funnelshift_l(v1, 0u, sh), 0u};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const unsigned long long zz = (unsigned long long)z[kLimbs + i] + w[i] + c2;
            z[kLimbs + i] = (uint32_t)zz;
            c2 = (uint32_t)(zz >> 32);
          }
        }
        if (++acc == C::kAcc) {
          acc = 0;
          aphase ^= 1;
        }
      }
      if (row < rows) {
        uint32_t* zr = args.out + (int64_t)n * args.zq + row * args.wz;
#pragma unroll
        for (int i = 0; i < kZ; i += 4)
          __stcs(reinterpret_cast<uint4*>(zr + i), make_uint4(z[i], z[i + 1], z[i + 2], z[i + 3]));
      }
    }
  }
  tc_fence_before();
  cluster_sync();   // all MMAs consumed, all TMEM reads done in both CTAs
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tbase, C::kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// operand builders

// Bc[b * (4n) + 4k + a] = byte (b - a) of ck_o[k] (0 outside [0, 4 lm)), b < nb.
// One CTA per 32 values of k and 32 rows b: the 32 ck_o rows are staged in
// shared memory (row pitch lm + 1 words against bank conflicts), each warp
// then writes 32 consecutive output words of one row b.
__global__ void __launch_bounds__(256)
build_bc_kernel(const uint32_t* __restrict__ cko, int64_t n, int lm, int nb,
                uint32_t* __restrict__ bc) {
  extern __shared__ uint32_t sck[];
  cko += (int64_t)blockIdx.z * n * lm;   // query q = blockIdx.z
  bc += (int64_t)blockIdx.z * nb * n;
  const int64_t k0 = (int64_t)blockIdx.x * 32;
  const int pitch = lm + 1;
  for (int idx = threadIdx.x; idx < 32 * lm; idx += blockDim.x) {
    const int kk = idx / lm, j = idx - kk * lm;
    sck[kk * pitch + j] = (k0 + kk < n) ? cko[(k0 + kk) * lm + j] : 0u;
  }
  __syncthreads();
  const int kk = threadIdx.x & 31;
  const uint8_t* by = reinterpret_cast<const uint8_t*>(sck + kk * pitch);
  if (k0 + kk >= n) return;
  const int b1 = min(nb, (int)(blockIdx.y + 1) * 32);
  for (int bb = blockIdx.y * 32 + (threadIdx.x >> 5); bb < b1; bb += blockDim.x >> 5) {
    uint32_t w = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int j = bb - a;
      if (j >= 0 && j < 4 * lm) w |= (uint32_t)by[j] << (8 * a);
    }
    bc[(int64_t)bb * n + k0 + kk] = w;
  }
}

// Ap[(4k + l) * ld + i] = byte l of A[i * lda + k], k < n, i < ld.
__global__ void __launch_bounds__(256)
build_aplanes_kernel(const uint32_t* __restrict__ A, int64_t ld, int64_t lda, int64_t n,
                     uint8_t* __restrict__ ap) {
  __shared__ uint32_t tile[64][33];
  const int64_t i0 = (int64_t)blockIdx.x * 64, k0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 64; r += 8) {
    const int64_t i = i0 + r, k = k0 + tx;
    tile[r][tx] = (i < ld && k < n) ? A[i * lda + k] : 0u;
  }
  __syncthreads();
  // thread -> (k = k0 + c, quad q of 4 consecutive i), writes 4 plane words
  for (int idx = threadIdx.x; idx < 32 * 16; idx += 256) {
    const int c = idx >> 4, q = idx & 15;
    const int64_t k = k0 + c;
    if (k >= n || i0 + 4 * q >= ld) continue;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      uint32_t w = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) w |= ((tile[4 * q + e][c] >> (8 * l)) & 0xffu) << (8 * e);
      *reinterpret_cast<uint32_t*>(ap + (4 * k + l) * ld + i0 + 4 * q) = w;
    }
  }
}

// ---------------------------------------------------------------------------
// host side

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2D u8 tensor (rows x cols, row pitch `pitch` bytes), box = box_rows x 128 bytes.
static int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t pitch,
                    int box_rows) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return kErrCuda;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): rows=%lld cols=%lld pitch=%lld box=%d", (int)r,
              (long long)rows, (long long)cols, (long long)pitch, box_rows);
    return kErrCuda;
  }
  return kOk;
}

static int num_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <int NT, int MODE>
static int umma_run(const uint8_t* A, int64_t rows, int64_t K, int64_t lda_bytes, const uint8_t* B,
                    int64_t brows, int64_t ldb_bytes, UmmaArgs args, cudaStream_t st,
                    int max_ctas = 0) {
  using Cfg = UmmaCfg<NT>;
  if (rows % kBM || brows % NT) {
    set_error("umma: rows %% 128 / brows %% NT (rows=%lld brows=%lld NT=%d)", (long long)rows,
              (long long)brows, NT);
    return kErrInput;
  }
  CUtensorMap ma, mb;
  if (int e = make_map(&ma, A, rows, K, lda_bytes, kBM)) return e;
  if (int e = make_map(&mb, B, brows, K, ldb_bytes, Cfg::kBoxB)) return e;
  args.m_tiles = (int)(rows / kBM);
  args.n_tiles = (int)(brows / NT);
  args.kblocks = (int)ceil_div(K, kBK);
  const int64_t T = (int64_t)args.m_tiles * args.n_tiles;
  const int64_t U = args.split ? T * args.kblocks : T;
  const int sms = num_sms();
  const int cap = (max_ctas > 0 && max_ctas < sms) ? max_ctas : sms;
  const int grid = (int)std::min<int64_t>(cap, U);
  auto kern = umma_gemm_kernel<NT, MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
  if (max_ctas > 0 && grid % 2 == 0) {
    // sharing the GPU with a CTA-pair kernel: occupy whole TPCs (clusters of
    // 2) so the remaining SMs stay pairable
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Cfg::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, ma, mb, args) != cudaSuccess)
      return check_launch("umma_gemm cluster launch");
    return check_launch("umma_gemm");
  }
  kern<<<grid, kThreads, Cfg::kSmem, st>>>(ma, mb, args);
  return check_launch("umma_gemm");
}

// CTA-pair BIGINT GEMM launch: clusters of 2, grid = 2 x pairs.
template <int NT>
static int umma_pair_run(const uint8_t* A, int64_t rows, int64_t K, int64_t lda_bytes,
                         const uint8_t* B, int64_t brows, int64_t ldb_bytes, UmmaArgs args,
                         cudaStream_t st, int max_ctas) {
  using C = PairCfg<NT>;
  if (rows % kBM || brows % NT) {
    set_error("umma_pair: rows %% 128 / brows %% NT (rows=%lld brows=%lld NT=%d)",
              (long long)rows, (long long)brows, NT);
    return kErrInput;
  }
  CUtensorMap ma, mb0, mb1;
  if (int e = make_map(&ma, A, rows, K, lda_bytes, kBM)) return e;
  if (int e = make_map(&mb0, B, brows, K, ldb_bytes, C::kH0)) return e;
  if (int e = make_map(&mb1, B, brows, K, ldb_bytes, C::kH1 ? C::kH1 : C::kH0)) return e;
  args.m_tiles = (int)ceil_div(rows, 2 * kBM);
  args.n_tiles = (int)(brows / NT);
  args.a_keep = 1;   // H rows: L2 evict_last (re-read once per query of a batch)
  args.kblocks = (int)ceil_div(K, kBK);
  args.split = 0;
  const int64_t T = (int64_t)args.m_tiles * args.n_tiles;
  const int sms = num_sms();
  const int cap = (max_ctas > 0 && max_ctas < sms) ? max_ctas : sms;
  const int pairs = (int)std::min<int64_t>(cap / 2, T);
  auto kern = umma_pair_bigint_kernel<NT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * (pairs > 0 ? pairs : 1));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, ma, mb0, mb1, args, rows) != cudaSuccess)
    return check_launch("umma_pair_bigint launch");
  return check_launch("umma_pair_bigint");
}


// b[v * rows + r] = qmask & (DB qu_v)[r] for nvec <= 4 (N = 16) or 64 (N = 256)
int umma_gemv_launch(const uint8_t* dbt, int64_t rows, int64_t ld, const uint8_t* qplanes,
                     int64_t nvec, uint32_t* out, int ctas, cudaStream_t st) {
  if (cudaMemsetAsync(out, 0, rows * nvec * sizeof(uint32_t), st) != cudaSuccess)
    return check_launch("umma_gemv memset");
  UmmaArgs a{};
  a.split = 1;
  a.out = out;
  a.ldo = rows;
  a.nout = (int)nvec;
  a.qmask = 0xffffffffu;
  if (nvec <= 4) return umma_run<16, kLimbCols>(dbt, rows, ld, ld, qplanes, 16, ld, a, st, ctas);
  if (nvec <= 64)
    return umma_run<256, kLimbCols>(dbt, rows, ld, ld, qplanes, 256, ld, a, st, ctas);
  set_error("umma_gemv: at most 64 query vectors per launch (got %lld)", (long long)nvec);
  return kErrInput;
}

// H[r * n + k] = qmask & -(DB A)[r, k]; aplanes = (4n x ld) byte planes of A.
int umma_hint_launch(const uint8_t* dbt, int64_t rows, int64_t ld, const uint8_t* aplanes,
                     int64_t n, uint32_t* H, uint32_t qmask, cudaStream_t st) {
  if ((4 * n) % 256) {
    set_error("umma_hint: 4n must be a multiple of 256 (n=%lld)", (long long)n);
    return kErrUnsupported;
  }
  UmmaArgs a{};
  a.split = 0;
  a.out = H;
  a.ldo = n;
  a.nout = (int)n;
  a.qmask = qmask;
  return umma_run<256, kLimbRowsNeg>(dbt, rows, ld, ld, aplanes, 4 * n, ld, a, st);
}

// z[r * wz + i] = limbs of sum_k H[r,k] ck_o[k] (b is added by the group stage); bc from build_bc.
int umma_answer_rows_launch(const uint32_t* H, int64_t rows, int64_t n, const uint8_t* bc, int nb,
                            const uint32_t* b, uint32_t qmask, int wz, uint32_t* z, int ctas,
                            cudaStream_t st) {
  UmmaArgs a{};
  a.split = 0;
  a.out = z;
  a.b = b;
  a.qmask = qmask;
  a.wz = wz;
  const uint8_t* Ab = reinterpret_cast<const uint8_t*>(H);
  // CTA pairs (cta_group::2, M = 256): half the B operand traffic per SM
  switch (nb) {
    case 144: return umma_pair_run<144>(Ab, rows, 4 * n, 4 * n, bc, 144, 4 * n, a, st, ctas);
    case 272: return umma_pair_run<272>(Ab, rows, 4 * n, 4 * n, bc, 272, 4 * n, a, st, ctas);
    case 400: return umma_pair_run<400>(Ab, rows, 4 * n, 4 * n, bc, 400, 4 * n, a, st, ctas);
    default:
      set_error("umma_answer_rows: unsupported B width %d", nb);
      return kErrUnsupported;
  }
}

static int build_bc_launch_ex(const uint32_t* cko, int64_t n, int lm, int nb, uint8_t* bc,
                              cudaStream_t st, int nq) {
  const size_t smem = (size_t)32 * (lm + 1) * sizeof(uint32_t);
  dim3 grid((unsigned)ceil_div(n, 32), (unsigned)ceil_div(nb, 32), (unsigned)nq);
  build_bc_kernel<<<grid, 256, smem, st>>>(cko, n, lm, nb,
                                                               reinterpret_cast<uint32_t*>(bc));
  return check_launch("build_bc");
}

int build_bc_launch(const uint32_t* cko, int64_t n, int lm, int nb, uint8_t* bc, cudaStream_t st) {
  return build_bc_launch_ex(cko, n, lm, nb, bc, st, 1);
}

int build_bc_batch_launch(const uint32_t* cko, int64_t n, int lm, int nb, int nq, uint8_t* bc,
                          cudaStream_t st) {
  return build_bc_launch_ex(cko, n, lm, nb, bc, st, nq);
}

// z[q][r * wz + i] for nq queries (bc = nq stacked operands): one launch,
// tiles = (row block, query) with consecutive tiles sharing the H rows.
int umma_answer_rows_batch_launch(const uint32_t* H, int64_t rows, int64_t n, const uint8_t* bc,
                                  int nb, int nq, int wz, uint32_t* z, cudaStream_t st) {
  UmmaArgs a{};
  a.split = 0;
  a.out = z;
  a.wz = wz;
  a.zq = rows * wz;
  const uint8_t* Ab = reinterpret_cast<const uint8_t*>(H);
  switch (nb) {
    case 144: return umma_pair_run<144>(Ab, rows, 4 * n, 4 * n, bc, 144LL * nq, 4 * n, a, st, 0);
    case 272: return umma_pair_run<272>(Ab, rows, 4 * n, 4 * n, bc, 272LL * nq, 4 * n, a, st, 0);
    case 400: return umma_pair_run<400>(Ab, rows, 4 * n, 4 * n, bc, 400LL * nq, 4 * n, a, st, 0);
    default:
      set_error("umma_answer_rows_batch: unsupported B width %d", nb);
      return kErrUnsupported;
  }
}

// Hp[r * 4np + a * np + k] = byte a of H[r * n + k] (zero for k >= n): the
// compression's A operand, one 128-byte-aligned byte plane per H byte.
__global__ void __launch_bounds__(256)
h_planes_kernel(const uint32_t* __restrict__ H, int64_t rows, int64_t n, int64_t np,
                uint8_t* __restrict__ hp) {
  const int64_t r = blockIdx.y;
  const int64_t k4 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;  // 4 k per thread
  if (r >= rows || k4 >= np) return;
  uint32_t w[4] = {0u, 0u, 0u, 0u};   // w[a] = bytes a of H[r, k4 .. k4+3]
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t h = (k4 + e < n) ? H[r * n + k4 + e] : 0u;
#pragma unroll
    for (int a = 0; a < 4; ++a) w[a] |= ((h >> (8 * a)) & 0xffu) << (8 * e);
  }
  uint8_t* dst = hp + r * 4 * np + k4;
#pragma unroll
  for (int a = 0; a < 4; ++a) *reinterpret_cast<uint32_t*>(dst + a * np) = w[a];
}

// Bp[q][j * np + k] = byte j of ck_q[k] (j < 4 lm; zero for k >= n)
__global__ void __launch_bounds__(256)
build_bcp_kernel(const uint32_t* __restrict__ cko, int64_t n, int lm, int64_t np,
                 uint8_t* __restrict__ bp) {
  __shared__ uint32_t tile[32][33];
  const int64_t q = blockIdx.z;
  cko += q * n * lm;
  bp += q * (int64_t)(4 * lm) * np;
  const int64_t k0 = (int64_t)blockIdx.x * 32;
  const int l0 = blockIdx.y * 32;   // limb block
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = ty; i < 32; i += 8) {
    const int64_t k = k0 + i;
    tile[i][tx] = (k < n && l0 + tx < lm) ? cko[k * lm + l0 + tx] : 0u;
  }
  __syncthreads();
  // thread -> (limb l0 + li, byte e): row j = 4 (l0 + li) + e, 32 consecutive k
  for (int idx = ty; idx < 32 * 4; idx += 8) {
    const int li = idx >> 2, e = idx & 3;
    if (l0 + li >= lm) continue;
    const int64_t k = k0 + tx;
    if (k >= np) continue;
    bp[(int64_t)(4 * (l0 + li) + e) * np + k] = (uint8_t)(tile[tx][li] >> (8 * e));
  }
}

int h_planes_launch(const uint32_t* H, int64_t rows, int64_t n, uint8_t* hp, cudaStream_t st) {
  const int64_t np = ceil_div(n, kBK) * kBK;
  if (rows <= 0 || rows > 65535 * 64) {
    set_error("h_planes: bad rows %lld", (long long)rows);
    return kErrInput;
  }
  for (int64_t r0 = 0; r0 < rows; r0 += 65535) {
    const int64_t rr = (rows - r0) < 65535 ? (rows - r0) : 65535;
    dim3 grid((unsigned)ceil_div(np / 4, 256), (unsigned)rr);
    h_planes_kernel<<<grid, 256, 0, st>>>(H + r0 * n, rr, n, np, hp + r0 * 4 * np);
  }
  return check_launch("h_planes");
}

int build_bcp_launch(const uint32_t* cko, int64_t n, int lm, int nq, uint8_t* bp, cudaStream_t st) {
  const int64_t np = ceil_div(n, kBK) * kBK;
  dim3 grid((unsigned)ceil_div(np, 32), (unsigned)ceil_div(lm, 32), (unsigned)nq);
  build_bcp_kernel<<<grid, 256, 0, st>>>(cko, n, lm, np, bp);
  return check_launch("build_bcp");
}

// The CTA-pair planar kernel keeps a query's B half resident in shared memory:
// whenever that fits (n <= 1024 at 2048-bit m). Single queries use it too (the
// answer step on a 36 / 112 SM split: 194-195 us against 201-206 us with the
// single-CTA kernel, A/B on one box); larger n falls back to the single-CTA
// kernel below.
static bool use_planar_pair(int NT, int64_t np) {
  return (int64_t)(NT / 2) * np <= PlanarPairCfg<256>::kBResMax;
}

// z (nq x rows x wz) from the planar operands; lm in {32, 64}.
int umma_planar_launch(const uint8_t* hp, int64_t rows, int64_t n, const uint8_t* bp, int lm,
                       int nq, int wz, uint32_t* z, int ctas, cudaStream_t st) {
  const int64_t np = ceil_div(n, kBK) * kBK;
  if (wz != lm + 4 || rows % kBM || (lm != 32 && lm != 64) || n > 33025) {
    set_error("umma_planar: unsupported shape (lm=%d wz=%d rows=%lld n=%lld)", lm, wz,
              (long long)rows, (long long)n);
    return kErrUnsupported;
  }
  UmmaArgs a{};
  a.split = 0;
  a.out = z;
  a.wz = wz;
  a.zq = rows * wz;
  a.a_keep = nq > 1 ? 1 : 0;
  const int NT = 4 * lm;
  CUtensorMap ma, mb;
  if (int e = make_map(&ma, hp, rows, 4 * np, 4 * np, kBM)) return e;
  if (int e = make_map(&mb, bp, (int64_t)NT * nq, np, np, NT)) return e;
  a.m_tiles = (int)(rows / kBM);
  a.n_tiles = nq;
  a.kblocks = (int)(4 * np / kBK);
  const int64_t T = (int64_t)a.m_tiles * a.n_tiles;
  const int sms = num_sms();
  const int cap = (ctas > 0 && ctas < sms) ? ctas : sms;
  const int grid = (int)std::min<int64_t>(cap, T);
  if (use_planar_pair(NT, np) && cap >= 2) {
    CUtensorMap mbp;
    if (int e = make_map(&mbp, bp, (int64_t)NT * nq, np, np, NT / 2)) return e;
    a.m_tiles = (int)ceil_div(rows, 2 * kBM);
    const int64_t Tp = (int64_t)a.m_tiles * a.n_tiles;
    const int pairs = (int)std::max<int64_t>(1, std::min<int64_t>(cap / 2, Tp));
    // blocks of row tiles whose H planes (2 kBM x 4 np bytes per pair tile) stay in L2
    // (<= 48 MB); among the block sizes of at least half that, the one whose
    // (query, tile) units split most evenly over the pairs, block by block
    const int64_t tile_bytes = 2ll * kBM * 4 * np;
    int tb = a.m_tiles;
    if (nq > 1) {
      const int tmax = (int)std::max<int64_t>(1, std::min<int64_t>(a.m_tiles, (48ll << 20) / tile_bytes));
      int64_t best = -1;
      for (int t = tmax; t >= std::max(1, tmax / 2); --t) {
        int64_t steps = 0;                 // units of the busiest pair, summed over the blocks
        for (int left = a.m_tiles; left > 0; left -= t)
          steps += ceil_div((int64_t)std::min(left, t) * nq, (int64_t)pairs);
        if (best < 0 || steps < best) {
          best = steps;
          tb = t;
        }
      }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (NT == 256) {
      auto kern = umma_planar_pair_kernel<256>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           PlanarPairCfg<256>::kSmem);
      cfg.dynamicSmemBytes = PlanarPairCfg<256>::kSmem;
      e = cudaLaunchKernelEx(&cfg, kern, ma, mbp, a, np, rows, tb);
    } else {
      auto kern = umma_planar_pair_kernel<128>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           PlanarPairCfg<128>::kSmem);
      cfg.dynamicSmemBytes = PlanarPairCfg<128>::kSmem;
      e = cudaLaunchKernelEx(&cfg, kern, ma, mbp, a, np, rows, tb);
    }
    if (e != cudaSuccess) return check_launch("umma_planar_pair launch");
    return check_launch("umma_planar_pair");
  }
  if (NT == 256) {
    auto kern = umma_planar_kernel<256>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, UmmaCfg<256>::kSmem);
    kern<<<grid, kThreads, UmmaCfg<256>::kSmem, st>>>(ma, mb, a, np);
  } else {
    auto kern = umma_planar_kernel<128>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, UmmaCfg<128>::kSmem);
    kern<<<grid, kThreads, UmmaCfg<128>::kSmem, st>>>(ma, mb, a, np);
  }
  return check_launch("umma_planar");
}

int build_aplanes_launch(const uint32_t* A, int64_t ld, int64_t lda, int64_t n, uint8_t* ap,
                         cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(ld, 64), (unsigned)ceil_div(n, 32));
  build_aplanes_kernel<<<grid, 256, 0, st>>>(A, ld, lda, n, ap);
  return check_launch("build_aplanes");
}

}  // namespace zpir
