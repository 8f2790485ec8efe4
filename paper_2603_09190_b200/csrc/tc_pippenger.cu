// Per-client hint on the tensor cores: the Pippenger bucket updates of
// slot_fixed (multiexp.cu) as Montgomery multiplications by a FIXED multiplier.
//
// W[r] = prod_{pos < 4n} P[pos]^{digit(r, pos)}, digit(r, pos) = byte (pos / n)
// of H[r][pos % n], P[pos] = ck_r[pos % n]^(2^(8 (pos / n))) (pow8_table, Montgomery
// form mod N = m^2). Position-major Pippenger: at every position each row
// multiplies ONE of its 255 buckets by the same P[pos], so a position is a
// batch "X (rows) times fixed Y mod N" -- three Toeplitz int8 GEMMs:
//   u = X * Y' mod R          (Y' = Y * N' mod R, N' = -N^-1 mod R, R = 2^4096)
//   Z = (X * Y + u * N) / R   (< 2N; one conditional subtraction)
// with a byte-Toeplitz B operand Toep(y)[j][a] = byte_{j-a}(y). Tiles of
// Toep(y) (256 output columns x 128 K bytes) depend only on delta = c0 - a0, so
// each multiplier is stored as 6 SW128 tiles (delta = -128 .. 512). One CTA per
// 128-row tile per position: 30 k-blocks (120 N = 256 MMAs, ~146 cycles each),
// three TMEM drains with carry chains in registers; X (gathered from the
// buckets) and u live in shared memory as the MMAs' A operands.
// The bucket combine (prod_d B_d^d, running sums, per-row operands) stays on
// the IMAD warp-Montgomery path.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "bignum.cuh"
#include "umma.cuh"

namespace zpir {

using namespace sm100;

namespace tcp {

constexpr int kL = 128;            // limbs of N = m^2 (2048-bit m)
constexpr int kRows = 128;         // rows per tile (TMEM lanes)
constexpr int kBK = 128;           // K bytes per k-block
constexpr int kTile = 256 * kBK;   // one Toeplitz tile: 256 columns x 128 K bytes
constexpr int kTY = 6;             // tiles per multiplier (delta = -128 .. 512)
constexpr int kTYp = 4;            // tiles of Y' (columns < 512: delta = -128 .. 256)
constexpr int kStages = 3;
constexpr int kThreads = 192;
constexpr int kABytes = kRows * 512;     // one 128 x 512-byte A operand (4 k-blocks)
constexpr int kSmem = 2 * kABytes + kStages * kTile + 1024 + 1024;

// The static MMA schedule: (phase, TMEM chunk, A = X (0) / U (1), k-block,
// B source (0 = Y', 1 = Y, 2 = N), tile index t = 2 cc - ka + 1).
struct Step {
  int8_t phase, chunk, a, ka, src, t;
};
__constant__ Step kSched[30];
constexpr int kNSteps = 30;

}  // namespace tcp

// tiles[(c * T + t) * 256 + j][a] = byte_{128 (t - 1) + j - a}(y_c), zero outside [0, 512)
__global__ void __launch_bounds__(256)
toep_tiles_kernel(const uint32_t* __restrict__ Y, int T, uint8_t* __restrict__ tiles) {
  const int64_t ct = blockIdx.x;                 // c * T + t
  const int64_t c = ct / T;
  const int t = (int)(ct - c * T);
  const int j = threadIdx.x;
  const uint8_t* y = reinterpret_cast<const uint8_t*>(Y + c * tcp::kL);
  const int delta = 128 * (t - 1);
  uint8_t* row = tiles + (ct * 256 + j) * tcp::kBK;
#pragma unroll 1
  for (int a0 = 0; a0 < tcp::kBK; a0 += 16) {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t v = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int idx = delta + j - (a0 + 4 * q + e);
        const uint32_t byte = (idx >= 0 && idx < 512) ? y[idx] : 0u;
        v |= byte << (8 * e);
      }
      w[q] = v;
    }
    *reinterpret_cast<uint4*>(row + a0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// out[c] = Y[c] * Np mod 2^4096, one thread per value (product scanning).
__global__ void __launch_bounds__(128)
mul_lo_kernel(const uint32_t* __restrict__ Y, int64_t count, const uint32_t* __restrict__ Np,
              uint32_t* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= count) return;
  const uint32_t* y = Y + c * tcp::kL;
  uint32_t* o = out + c * tcp::kL;
  unsigned long long lo = 0, hi = 0;  // 128-bit column accumulator (lo, hi)
  for (int k = 0; k < tcp::kL; ++k) {
    for (int i = 0; i <= k; ++i) {
      const unsigned long long p = (unsigned long long)y[i] * Np[k - i];
      const unsigned long long s = lo + p;
      hi += (s < lo);
      lo = s;
    }
    o[k] = (uint32_t)lo;
    lo = (lo >> 32) | (hi << 32);
    hi >>= 32;
  }
}

__global__ void bucket_fill_kernel(uint32_t* __restrict__ B, int64_t count,
                                   const uint32_t* __restrict__ one) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // u32 index
  if (i < count * tcp::kL) B[i] = one[i % tcp::kL];
}

// W[r] = prod_d B[r][d]^d (running sums from d = 255 down), Montgomery form.
// Buckets are stored lazily reduced: flag F[r][d] set means "subtract N (mod R)".
__global__ void __launch_bounds__(128)
bucket_combine_kernel(const uint32_t* __restrict__ B, const uint8_t* __restrict__ F, int64_t rows,
                      const uint32_t* __restrict__ N, uint32_t np, uint32_t* __restrict__ W) {
  constexpr int LPL = tcp::kL / 32;
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  uint32_t n_[LPL], run[LPL], tot[LPL], x[LPL];
  big_load<LPL>(n_, N, lane);
  const uint32_t* br = B + r * 255 * tcp::kL;
  const uint8_t* fr = F + r * 255;
  big_load<LPL>(run, br + 254 * tcp::kL, lane);
  if (fr[254]) big_cond_sub<LPL>(run, 1u, n_, lane);
  big_copy<LPL>(tot, run);
  for (int d = 254; d >= 1; --d) {
    big_load<LPL>(x, br + (d - 1) * tcp::kL, lane);
    if (fr[d - 1]) big_cond_sub<LPL>(x, 1u, n_, lane);
    mont_mul<LPL>(run, run, x, n_, np, lane);
    mont_mul<LPL>(tot, tot, run, n_, np, lane);
  }
  big_store<LPL>(W + r * tcp::kL, tot, lane);
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Carry-propagate 16 TMEM columns (byte positions) into 4 u32 limbs.
__device__ __forceinline__ void carry4(const uint32_t (&v)[16], unsigned long long& carry,
                                       uint32_t (&limb)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned long long s = (unsigned long long)v[4 * i] +
                                 ((unsigned long long)v[4 * i + 1] << 8) +
                                 ((unsigned long long)v[4 * i + 2] << 16) +
                                 ((unsigned long long)v[4 * i + 3] << 24) + carry;
    limb[i] = (uint32_t)s;
    carry = s >> 32;
  }
}

// Pippenger positions pos0..pos1-1 for one 128-row tile per CTA (tiles are
// independent: a row only touches its own buckets):
//   B[r][d - 1] *= P[pos] for d = digit(r, pos) != 0.
// Per position, six 256-column tasks alternate between two TMEM buffers so
// the epilogue drains one while the MMA warp fills the other:
//   U0, U1: columns 0..255 / 256..511 of X * Y'    -> u (mod R) into smem
//   L0, L1: columns 0..511 of X * Y + u * N        -> carry out of bit 4096
//   H0, H1: columns 512..1023                       -> Z (< 2N), kept in registers
__global__ void __launch_bounds__(tcp::kThreads, 1)
tc_step_kernel(const __grid_constant__ CUtensorMap mapYp, const __grid_constant__ CUtensorMap mapY,
               const __grid_constant__ CUtensorMap mapN, const uint32_t* __restrict__ E,
               int64_t rs, int64_t n, int pos0, int pos1, int64_t rows, uint32_t* __restrict__ Bk,
               uint8_t* __restrict__ Fk, const uint32_t* __restrict__ Nlimbs) {
  using namespace tcp;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* XA = smem;                       // X (4 k-blocks of 128 x 128 B, SW128)
  uint8_t* UA = smem + kABytes;             // u, same layout
  uint8_t* BS = smem + 2 * kABytes;         // B tile stages
  uint64_t* full = reinterpret_cast<uint64_t*>(BS + kStages * kTile);
  uint64_t* empty = full + kStages;
  uint64_t* xfull = empty + kStages;
  uint64_t* uready = xfull + 1;             // [2]: u bytes 0..255 / 256..511 written
  uint64_t* tfull = uready + 2;             // [2] per TMEM buffer
  uint64_t* tempty = tfull + 2;             // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t* sN = tslot + 4;                 // N limbs (512 B)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapYp);
    tma_prefetch(&mapY);
    tma_prefetch(&mapN);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(xfull, 128);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&uready[b], 128);
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < kL; i += blockDim.x) sN[i] = Nlimbs[i];
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const int64_t row0 = (int64_t)blockIdx.x * kRows;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: the 30 B tiles of every position ----------------
      const uint64_t pol = l2_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int pos = pos0; pos < pos1; ++pos)
        for (int s = 0; s < kNSteps; ++s) {
          const Step st = kSched[s];
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], kTile);
          uint8_t* dst = BS + stage * kTile;
          if (st.src == 0)
            tma_load_2d_hint(dst, &mapYp, &full[stage], 0, (pos * kTYp + st.t) * 256, pol);
          else if (st.src == 1)
            tma_load_2d_hint(dst, &mapY, &full[stage], 0, (pos * kTY + st.t) * 256, pol);
          else
            tma_load_2d_hint(dst, &mapN, &full[stage], 0, st.t * 256, pol);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: tasks 0..5 per position, buffer = task & 1 ----------------
      const uint32_t idesc = idesc_u8(kRows, 256);
      int stage = 0;
      uint32_t phase = 0, xph = 0;
      uint32_t eph[2] = {0, 0};
      bool used[2] = {false, false};
      for (int pos = pos0; pos < pos1; ++pos) {
        int cur = -1;
        bool first = true, uwait = false;
        for (int s = 0; s < kNSteps; ++s) {
          const Step st = kSched[s];
          const int buf = st.phase & 1;
          if (st.phase != cur) {
            if (cur >= 0) umma_commit(&tfull[cur & 1]);
            if (used[buf]) {                  // the epilogue has drained this buffer
              mbar_wait(&tempty[buf], eph[buf]);
              eph[buf] ^= 1;
            }
            used[buf] = true;
            if (st.phase == 0) mbar_wait(xfull, xph);
            tc_fence_after();
            cur = st.phase;
            first = true;
            uwait = false;
          }
          if (st.a && !uwait) {               // u * N: u bytes of this column range ready
            mbar_wait(&uready[st.phase == 2 ? 0 : 1], xph);
            tc_fence_after();
            uwait = true;
          }
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32((st.a ? UA : XA) + st.ka * (kRows * kBK));
          const uint64_t ad = desc_sw128(a0);
          const uint64_t bd = desc_sw128(smem_u32(BS + stage * kTile));
          const uint32_t d = tbase + (uint32_t)(buf * 256);
#pragma unroll
          for (int k = 0; k < kBK / 32; ++k)
            umma_i8(d, ad + 2 * k, bd + 2 * k, idesc, (first && k == 0) ? 0u : 1u);
          first = false;
          umma_commit(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[cur & 1]);
        xph ^= 1;
      }
    }
  } else {
    // ---------------- epilogue: one row per thread ----------------
    const int quarter = warp & 3;
    const int t = quarter * 32 + lane;          // row within the tile = TMEM lane
    const int64_t r = row0 + t;
    const uint32_t lanebase = tbase + ((uint32_t)(quarter * 32) << 16);
    uint32_t fph[2] = {0, 0};
    for (int pos = pos0; pos < pos1; ++pos) {
      const int dig_i = pos / (int)n;
      const int64_t dig_k = pos - (int64_t)dig_i * n;
      uint32_t dg = 0;
      if (r < rows) dg = (E[r * rs + dig_k] >> (8 * dig_i)) & 0xffu;
      const int64_t bidx = (r * 255) + (dg ? dg - 1 : 0);
      uint32_t* brow = Bk + bidx * kL;
      // gather X = B[r][dg - 1] into the SW128 A layout (zero rows for dg == 0);
      // the previous position's MMAs are complete (its last tfull was waited).
      // A set flag means the stored value is Z with Z - N still to be taken (mod R).
      {
        const bool lazy = dg && Fk[bidx];
        uint4 v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c)
          v[c] = dg ? *reinterpret_cast<const uint4*>(brow + 4 * c) : make_uint4(0u, 0u, 0u, 0u);
        if (lazy) {
          uint32_t bw = 0;
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            uint32_t* w = reinterpret_cast<uint32_t*>(&v[c]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const unsigned long long dlt = (unsigned long long)w[i] - sN[4 * c + i] - bw;
              w[i] = (uint32_t)dlt;
              bw = (uint32_t)(dlt >> 63);
            }
          }
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int kb = c >> 3, ch = c & 7;
          *reinterpret_cast<uint4*>(XA + kb * (kRows * kBK) + t * kBK + ((ch ^ (t & 7)) << 4)) =
              v[c];
        }
      }
      fence_async_smem();
      mbar_arrive(xfull);
      unsigned long long carry = 0;
      uint32_t zb = 0;                        // borrow chain of Z - N, low limbs up
#pragma unroll 1
      for (int task = 0; task < 6; ++task) {
        const int buf = task & 1;
        mbar_wait(&tfull[buf], fph[buf]);
        fph[buf] ^= 1;
        tc_fence_after();
        const uint32_t taddr = lanebase + (uint32_t)(buf * 256);
        if (task == 2) carry = 0;             // the low-column chain of X*Y + u*N starts
#pragma unroll 2
        for (int c = 0; c < 16; ++c) {
          uint32_t v[16], limb[4];
          tmem_ld16(taddr + 16 * c, v);
          tmem_wait_ld();
          carry4(v, carry, limb);
          if (task < 2) {                     // u bytes -> UA (SW128 A operand)
            const int cc = task * 16 + c;     // 16-byte chunk of u
            const int kb = cc >> 3, ch = cc & 7;
            *reinterpret_cast<uint4*>(UA + kb * (kRows * kBK) + t * kBK + ((ch ^ (t & 7)) << 4)) =
                make_uint4(limb[0], limb[1], limb[2], limb[3]);
          } else if (task >= 4) {             // Z limbs: unreduced to the bucket, borrow chain
            const int li = (task - 4) * 64 + 4 * c;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const unsigned long long dlt = (unsigned long long)limb[i] - sN[li + i] - zb;
              zb = (uint32_t)(dlt >> 63);
            }
            if (dg)
              *reinterpret_cast<uint4*>(brow + li) = make_uint4(limb[0], limb[1], limb[2], limb[3]);
          }
        }
        if (task < 2) {
          fence_async_smem();
          mbar_arrive(&uready[task]);
        }
        tc_fence_before();
        mbar_arrive(&tempty[buf]);
      }
      // Z = z + 2^4096 * carry < 2N: Z >= N iff the top carry is set or Z - N does
      // not borrow; the subtraction is deferred to the bucket's next reader (flag)
      if (dg) Fk[bidx] = (carry != 0 || zb == 0) ? 1 : 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 tcp_encode() {
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

static int tile_map(CUtensorMap* map, const void* base, int64_t rows) {
  auto fn = tcp_encode();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return kErrCuda;
  }
  cuuint64_t dims[2] = {(cuuint64_t)tcp::kBK, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)tcp::kBK};
  cuuint32_t box[2] = {(cuuint32_t)tcp::kBK, 256};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (tiles) failed (%d)", (int)r);
    return kErrCuda;
  }
  return kOk;
}

static int upload_schedule() {
  static bool done = false;
  if (done) return kOk;
  tcp::Step h[tcp::kNSteps];
  int k = 0;
  // tasks 0, 1 (U0, U1): global 256-column chunks 0, 1 of X * Y'
  for (int gc = 0; gc < 2; ++gc)
    for (int ka = 0; ka < 4; ++ka) {
      const int t = 2 * gc - ka + 1;
      if (t >= 0 && t < tcp::kTYp) h[k++] = {(int8_t)gc, (int8_t)(gc & 1), 0, (int8_t)ka, 0, (int8_t)t};
    }
  // tasks 2..5 (L0, L1, H0, H1): chunk gc = task - 2 of X * Y + u * N, the
  // X * Y k-blocks first (they do not wait for u)
  for (int gc = 0; gc < 4; ++gc) {
    const int task = gc + 2;
    for (int a = 0; a < 2; ++a)
      for (int ka = 0; ka < 4; ++ka) {
        const int t = 2 * gc - ka + 1;
        if (t < 0 || t >= tcp::kTY) continue;
        h[k++] = {(int8_t)task, (int8_t)(task & 1), (int8_t)a, (int8_t)ka, (int8_t)(a ? 2 : 1),
                  (int8_t)t};
      }
  }
  if (k != tcp::kNSteps) {
    set_error("tc_pippenger: schedule has %d steps", k);
    return kErrCuda;
  }
  if (cudaMemcpyToSymbol(tcp::kSched, h, sizeof(h)) != cudaSuccess) return check_launch("schedule");
  done = true;
  return kOk;
}

// W[r] (Montgomery form, 4096-bit N) for rows r < rows of 32-bit exponent rows
// E[r * rs + k]: the slot_fixed contract, with the bucket updates on tcgen05.
int tc_slot_fixed_launch(const uint32_t* P, int64_t n, const uint32_t* E, int64_t rs, int64_t rows,
                         const uint32_t* N, uint32_t np, const uint32_t* one_m,
                         const uint32_t* Nprime, uint32_t* W, cudaStream_t st) {
  using namespace tcp;
  const int64_t npos = 4 * n;
  if (n <= 0 || rows <= 0 || npos > 65536) {
    set_error("tc_slot_fixed: bad shapes (n=%lld rows=%lld)", (long long)n, (long long)rows);
    return kErrInput;
  }
  if (int e = upload_schedule()) return e;
  {
    // keep the multi-GB workspace in the stream-ordered pool between clients
    static bool pool_set = false;
    if (!pool_set) {
      int dev = 0;
      cudaMemPool_t pool;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      cudaGetLastError();
      pool_set = true;
    }
  }
  const int64_t tiles = ceil_div(rows, kRows);
  const int64_t rows_p = tiles * kRows;
  uint32_t *Yp = nullptr, *Bk = nullptr;
  uint8_t *tY = nullptr, *tYp = nullptr, *tN = nullptr, *Fk = nullptr;
  auto fail = [&](const char* what) {
    if (Yp) cudaFreeAsync(Yp, st);
    if (Bk) cudaFreeAsync(Bk, st);
    if (tY) cudaFreeAsync(tY, st);
    if (tYp) cudaFreeAsync(tYp, st);
    if (tN) cudaFreeAsync(tN, st);
    if (Fk) cudaFreeAsync(Fk, st);
    cudaGetLastError();
    set_error("tc_slot_fixed: %s", what);
    return kErrCuda;
  };
  if (cudaMallocAsync(reinterpret_cast<void**>(&Yp), (size_t)npos * kL * 4, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&tY), (size_t)npos * kTY * kTile, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&tYp), (size_t)npos * kTYp * kTile, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&tN), (size_t)kTY * kTile, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&Bk), (size_t)rows_p * 255 * kL * 4, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&Fk), (size_t)rows_p * 255, st) != cudaSuccess)
    return fail("workspace allocation");
  if (cudaMemsetAsync(Fk, 0, (size_t)rows_p * 255, st) != cudaSuccess) return fail("memset");
  mul_lo_kernel<<<(unsigned)ceil_div(npos, 128), 128, 0, st>>>(P, npos, Nprime, Yp);
  toep_tiles_kernel<<<(unsigned)(npos * kTY), 256, 0, st>>>(P, kTY, tY);
  toep_tiles_kernel<<<(unsigned)(npos * kTYp), 256, 0, st>>>(Yp, kTYp, tYp);
  toep_tiles_kernel<<<(unsigned)kTY, 256, 0, st>>>(N, kTY, tN);
  {
    const int64_t cnt = rows_p * 255;
    bucket_fill_kernel<<<(unsigned)ceil_div(cnt * kL, 256), 256, 0, st>>>(Bk, cnt, one_m);
  }
  if (int e = check_launch("tc_slot_fixed setup")) return fail("setup kernels");
  CUtensorMap mYp, mY, mN;
  if (tile_map(&mYp, tYp, npos * kTYp * 256) || tile_map(&mY, tY, npos * kTY * 256) ||
      tile_map(&mN, tN, (int64_t)kTY * 256))
    return fail("tensor maps");
  cudaFuncSetAttribute(tc_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  // one launch walks every position (tiles are independent); chunked so a
  // launch stays well under a second
  static int64_t chunk = -1;
  if (chunk < 0) {
    const char* e = getenv("ZPIR_TC_CHUNK");
    chunk = e ? std::max<int64_t>(1, atoll(e)) : 1024;
  }
  for (int64_t p0 = 0; p0 < npos; p0 += chunk) {
    const int64_t p1 = std::min<int64_t>(npos, p0 + chunk);
    tc_step_kernel<<<(unsigned)tiles, kThreads, kSmem, st>>>(mYp, mY, mN, E, rs, n, (int)p0,
                                                             (int)p1, rows, Bk, Fk, N);
  }
  if (check_launch("tc_step")) return fail("tc_step launch");
  bucket_combine_kernel<<<(unsigned)ceil_div(rows, 4), 128, 0, st>>>(Bk, Fk, rows, N, np, W);
  if (check_launch("bucket_combine")) return fail("bucket_combine");
  cudaFreeAsync(Yp, st);
  cudaFreeAsync(Bk, st);
  cudaFreeAsync(tY, st);
  cudaFreeAsync(tYp, st);
  cudaFreeAsync(tN, st);
  cudaFreeAsync(Fk, st);
  return check_launch("tc_slot_fixed");
}

}  // namespace zpir
