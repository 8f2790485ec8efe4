// Per-client hint on the tensor cores: the Pippenger bucket updates of
// slot_fixed (multiexp.cu) as modular multiplications by a FIXED multiplier,
// each one a plain int8 GEMM against a table of reduced shifts of the multiplier.
//
// W[r] = prod_{pos < D n} P[pos]^{digit(r, pos)}: every 32-bit exponent word
// H[r][k] is cut into D digits (DigitSpec), pos = i n + k, digit(r, pos) =
// digit i of H[r][k] and P[pos] = ck_r[k]^(2^off_i). Position-major Pippenger:
// at every position each row multiplies ONE of its 2^w - 1 buckets by the same
// y = P[pos] (standard form), so a position is a batch "X (rows) times y mod N".
// With X = sum_i x_i 256^i (bytes) and the table T_i = y 256^i mod N,
//   X y = sum_i x_i T_i  (mod N)          -- one u8 x u8 -> s32 GEMM, K = bytes of X,
// and the byte columns of the product (each < 515 * 255^2 < 2^25) carry-propagate
// to V = sum_i x_i T_i < 515 * 255 * N < 2^4114: 515 bytes. V is NOT reduced; it
// is the next X of its bucket as it stands (K = 515 bytes, padded to 544 = 17
// MMA k-steps), and the bound is closed under the operation because every T_i
// is < N whatever the size of X was. No Montgomery reduction, no quotient, no
// dependency between the MMAs of one position: per position and 128-row tile
//   task A: columns   0..255 (17 N = 256 MMAs) -> limbs 0..63
//   task B: columns 256..511 (17 MMAs)          -> limbs 64..127 and the carry, limb 128
// into two TMEM buffers, drained by the epilogue while the other one fills.
// The bucket combine reduces each bucket once (quotient estimate from the top
// limbs, bignum.cuh) before its IMAD running products.
//
// Buckets hold Montgomery-form values and y is in standard form, so products
// stay in Montgomery form. A row whose digit repeats at the next position gets
// its next X forwarded from this position's output by its own thread.
//
// Several clients (independent keys) run in one launch: blockIdx.y = client,
// every client with its own tables, buckets and output rows; rows may be a
// subset of the exponent rows (row ids), which is the incremental refresh.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "bignum.cuh"
#include "umma.cuh"

namespace zpir {

using namespace sm100;

#ifdef ZPIR_TC_TRACE
// debug timeline of CTA (0, 0): per position, 16 clock64 stamps (tools/tc_trace.py)
__device__ unsigned long long g_tc_trace[64 * 16];
#define TC_STAMP(pos, k)                                                                      \
  do {                                                                                        \
    if (blockIdx.x == 0 && blockIdx.y == 0 && (pos) - pos0 < 64)                              \
      g_tc_trace[((pos) - pos0) * 16 + (k)] = clock64();                                      \
  } while (0)
#else
#define TC_STAMP(pos, k) \
  do {                   \
  } while (0)
#endif

namespace tcp {

constexpr int kL = 128;            // limbs of N = m^2 (2048-bit m)
constexpr int kXL = 136;           // limbs per stored bucket (129 used; 544 B = 17 sectors)
constexpr int kRows = 128;         // rows per tile (TMEM lanes)
constexpr int kBK = 128;           // K bytes per full k-block
constexpr int kKB = 4;             // full k-blocks: bytes 0..511 of X
constexpr int kKT = 32;            // tail k-step: bytes 512..543 (512..514 used)
constexpr int kTK = kKB * kBK + kKT;   // table row pitch = K bytes per position (544)
constexpr int kUsedK = 515;        // bytes of X that can be non-zero
constexpr int kCols = 512;         // byte columns of the product = table rows per position
constexpr int kTile = 256 * kBK;   // B stage: 256 columns x 128 K bytes (SW128)
constexpr int kTail = 256 * kKT;   // B tail stage: 256 columns x 32 K bytes (SW32)
constexpr int kStages = 4;
constexpr int kTStages = 3;
constexpr int kThreads = 192;
constexpr int kABytes = kRows * kKB * kBK;   // X bytes 0..511: 4 k-blocks of 128 x 128 B (SW128)
constexpr int kATail = kRows * kKT;          // X bytes 512..543 (SW32)
constexpr int kSmem = kABytes + kATail + kStages * kTile + kTStages * kTail + 1024 + 1024;

}  // namespace tcp

// Per-client arguments of one batched launch (device copy).
struct TcClient {
  const uint32_t* P;        // (npos, 128) Montgomery multipliers
  const uint32_t* N;        // 128 limbs of N = m^2
  const uint32_t* one;      // R mod N
  uint32_t* W;              // output rows (Montgomery form), indexed by exponent row
  uint32_t np;              // -N^-1 mod 2^32
};

// Radix of the exponent digits: D digits per 32-bit exponent word, digit i
// = bits off[i] .. off[i] + width[i] - 1; nb = 2^max(width) - 1 buckets per row.
// Fewer, wider digits mean fewer positions (tensor-core work) but more buckets
// to combine on the IMAD path (2 nb Montgomery products per row).
struct DigitSpec {
  int D, nb;
  int off[8], width[8];
};

// Pd[c][i * n + k] = base_k^(2^off[i]) (Montgomery form), base_k = P_c[k] (the
// first block of the client's pow8 table): one warp per base, squarings only.
__global__ void __launch_bounds__(128)
powtab_kernel(const TcClient* __restrict__ cl, int64_t n, DigitSpec ds, uint32_t* __restrict__ Pd) {
  constexpr int LPL = tcp::kL / 32;
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.y;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= n) return;
  uint32_t n_[LPL], a[LPL];
  big_load<LPL>(n_, cl[c].N, lane);
  big_load<LPL>(a, cl[c].P + k * tcp::kL, lane);
  const uint32_t np = cl[c].np;
  uint32_t* out = Pd + (int64_t)c * ds.D * n * tcp::kL;
  int cur = 0;
  for (int i = 0; i < ds.D; ++i) {
    for (; cur < ds.off[i]; ++cur) mont_mul<LPL>(a, a, a, n_, np, lane);
    big_store<LPL>(out + ((int64_t)i * n + k) * tcp::kL, a, lane);
  }
}

// The multiplier tables: T[((c * npos + p) * 512 + j) * 544 + i] = byte j of
// (y_{c,p} 256^i mod N_c), y = Pd[c][p] taken out of Montgomery form; zero for
// i >= 515. One warp per position walks i upwards, t <- 256 t mod N (a byte
// shift and one quotient-estimate reduction); every lane keeps the last 16 i's
// of its 16 byte rows in registers and writes them as 16-byte row segments.
__global__ void __launch_bounds__(128)
table_kernel(const TcClient* __restrict__ cl, const uint32_t* __restrict__ Pd, int64_t npos,
             uint8_t* __restrict__ T) {
  constexpr int LPL = tcp::kL / 32;
  static_assert(LPL == 4, "16 bytes per lane");
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.y;
  const int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= npos) return;
  uint32_t n_[LPL], t[LPL], e1[LPL];
  big_load<LPL>(n_, cl[c].N, lane);
  big_load<LPL>(t, Pd + ((int64_t)c * npos + p) * tcp::kL, lane);
  big_set_small<LPL>(e1, 1u, lane);
  mont_mul<LPL>(t, t, e1, n_, cl[c].np, lane);        // y in standard form, < N
  const uint32_t nt8 = (__shfl_sync(ZPIR_FULL, n_[LPL - 1], 31) >> 8) + 1u;
  uint8_t* out = T + (((int64_t)c * npos + p) * tcp::kCols + 16 * lane) * tcp::kTK;
#pragma unroll 1
  for (int blk = 0; blk < tcp::kTK / 16; ++blk) {
    uint32_t acc[16][4];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const bool live = 16 * blk + s < tcp::kUsedK;
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        // byte b of this lane's 16 bytes into byte s of the row segment
        const uint32_t src = live ? t[b >> 2] : 0u;
        const uint32_t byte = (src >> (8 * (b & 3))) & 0xffu;
        if ((s & 3) == 0) acc[b][s >> 2] = byte;
        else acc[b][s >> 2] |= byte << (8 * (s & 3));
      }
      // t <- 256 t mod N
      uint32_t prev = __shfl_up_sync(ZPIR_FULL, t[LPL - 1], 1);
      prev = lane == 0 ? 0u : prev;
      const uint32_t top = __shfl_sync(ZPIR_FULL, t[LPL - 1], 31);
      const uint32_t tb = top >> 24;
#pragma unroll
      for (int k = LPL - 1; k >= 1; --k) t[k] = (t[k] << 8) | (t[k - 1] >> 24);
      t[0] = (t[0] << 8) | (prev >> 24);
      // quotient estimate from the top 40 bits over the top 24 bits of N (+1):
      // never too large, at most one too small
      const uint32_t xt8 = (tb << 24) | ((top << 8) >> 8);   // (tb 2^32 + new top limb) >> 8
      big_reduce_top<LPL>(t, tb, xt8 / nt8, n_, lane);
    }
#pragma unroll
    for (int b = 0; b < 16; ++b)
      *reinterpret_cast<uint4*>(out + (int64_t)b * tcp::kTK + 16 * blk) =
          make_uint4(acc[b][0], acc[b][1], acc[b][2], acc[b][3]);
  }
}

// Buckets start at 1 (Montgomery form): limbs 0..127 = R mod N, 128..135 = 0.
__global__ void bucket_fill_kernel(const TcClient* __restrict__ cl, uint32_t* __restrict__ B,
                                   int64_t count) {
  const int c = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // u32 index
  if (i < count * tcp::kXL) {
    const int l = (int)(i % tcp::kXL);
    B[(int64_t)c * count * tcp::kXL + i] = l < tcp::kL ? cl[c].one[l] : 0u;
  }
}

// W[row] = prod_d B[r][d]^d (running sums from d = nb down), Montgomery form.
// Buckets are stored unreduced (129 limbs, < 2^4114): reduced mod N on load.
__global__ void __launch_bounds__(128)
bucket_combine_kernel(const TcClient* __restrict__ cl, const uint32_t* __restrict__ Ball, int nb,
                      int64_t rows, int64_t rows_p, const int32_t* __restrict__ rid) {
  constexpr int LPL = tcp::kL / 32;
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.y;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const uint32_t np = cl[c].np;
  uint32_t n_[LPL], run[LPL], tot[LPL], x[LPL];
  big_load<LPL>(n_, cl[c].N, lane);
  const uint64_t nt1 = (uint64_t)__shfl_sync(ZPIR_FULL, n_[LPL - 1], 31) + 1u;
  const uint32_t* br = Ball + ((int64_t)c * rows_p + r) * nb * tcp::kXL;
  auto load = [&](uint32_t (&v)[LPL], int d) {
    const uint32_t* q = br + (int64_t)d * tcp::kXL;
    big_load<LPL>(v, q, lane);
    const uint32_t h = q[tcp::kL];
    const uint64_t xt = ((uint64_t)h << 32) | __shfl_sync(ZPIR_FULL, v[LPL - 1], 31);
    big_reduce_top<LPL>(v, h, (uint32_t)(xt / nt1), n_, lane);
  };
  load(run, nb - 1);
  big_copy<LPL>(tot, run);
  for (int d = nb - 1; d >= 1; --d) {
    load(x, d - 1);
    mont_mul<LPL>(run, run, x, n_, np, lane);
    mont_mul<LPL>(tot, tot, run, n_, np, lane);
  }
  const int64_t orow = rid ? (int64_t)rid[r] : r;
  big_store<LPL>(cl[c].W + orow * tcp::kL, tot, lane);
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 32 lanes x 32 bit, 32 consecutive columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// Wait for this thread's outstanding TMEM loads, ordered after `dep` (the
// last value computed from the previous batch) so the compiler keeps that
// work ahead of the wait.
__device__ __forceinline__ void tmem_wait_after(unsigned long long dep) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::"l"(dep) : "memory");
}
__device__ __forceinline__ void regs_ready(uint32_t (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(v[i]));
}

// Drain 256 TMEM columns of this thread's lane in eight 32-column batches,
// double-buffered: batch g + 1 is in flight while batch g is processed.
// f(g, v) consumes columns 32 g .. 32 g + 31; it updates `carry`, which also
// orders the next wait after the processing.
template <class F>
__device__ __forceinline__ void drain256(uint32_t taddr, unsigned long long& carry, F&& f) {
  uint32_t va[32], vb[32];
  tmem_ld32(taddr, va);
  tmem_wait_after(carry);
  regs_ready(va);
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    uint32_t (&cur)[32] = (g & 1) ? vb : va;
    uint32_t (&nxt)[32] = (g & 1) ? va : vb;
    if (g < 7) tmem_ld32(taddr + 32 * (g + 1), nxt);
    f(g, cur);
    if (g < 7) {
      tmem_wait_after(carry);
      regs_ready(nxt);
    }
  }
}

// Four byte columns (s32 sums) + carry -> one 32-bit limb.
__device__ __forceinline__ uint32_t limb4(const uint32_t* v, unsigned long long& carry) {
  const unsigned long long s = (unsigned long long)v[0] + ((unsigned long long)v[1] << 8) +
                               ((unsigned long long)v[2] << 16) +
                               ((unsigned long long)v[3] << 24) + carry;
  carry = s >> 32;
  return (uint32_t)s;
}

// K-major operand tile with SWIZZLE_32B: rows of 32 bytes, 8-row (256 B) atoms.
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;            // SBO = 256 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;                     // SWIZZLE_32B
  return d;
}

// Pippenger positions pos0..pos1-1 for one 128-row tile of one client per CTA
// (tiles are independent: a row only touches its own buckets):
//   B[r][d - 1] <- B[r][d - 1] * y[pos] for d = digit(r, pos) != 0.
__global__ void __launch_bounds__(tcp::kThreads, 1)
tc_step_kernel(const __grid_constant__ CUtensorMap mapT, const __grid_constant__ CUtensorMap mapTail,
               const __grid_constant__ DigitSpec ds, const uint32_t* __restrict__ E, int64_t rs,
               const int32_t* __restrict__ rid, int64_t n, int64_t npos, int pos0, int pos1,
               int64_t rows, int64_t rows_p, uint32_t* __restrict__ Ball) {
  using namespace tcp;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* XA = smem;                       // X bytes 0..511: 4 k-blocks of 128 x 128 B, SW128
  uint8_t* XT = smem + kABytes;             // X bytes 512..543: 128 x 32 B, SW32
  uint8_t* BS = XT + kATail;                // table stages (256 x 128 B)
  uint8_t* BT = BS + kStages * kTile;       // table tail stages (256 x 32 B)
  uint64_t* full = reinterpret_cast<uint64_t*>(BT + kTStages * kTail);
  uint64_t* empty = full + kStages;
  uint64_t* tlfull = empty + kStages;       // tail ring
  uint64_t* tlempty = tlfull + kTStages;
  uint64_t* xfull = tlempty + kTStages;     // X of the position complete in shared memory
  uint64_t* xfree = xfull + 1;              // every MMA reading X of the position done
  uint64_t* tfull = xfree + 1;              // [2] per TMEM buffer
  uint64_t* tempty = tfull + 2;             // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int client = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapT);
    tma_prefetch(&mapTail);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kTStages; ++s) {
      mbar_init(&tlfull[s], 1);
      mbar_init(&tlempty[s], 1);
    }
    mbar_init(xfull, 128);
    mbar_init(xfree, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    fence_mbar_init();
  }
  // bytes 516..543 of every X stay zero
  for (int i = threadIdx.x; i < kATail / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(XT)[i] = make_uint4(0u, 0u, 0u, 0u);
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const int64_t row0 = (int64_t)blockIdx.x * kRows;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: the table of every position, by column half ----------------
      const uint64_t pol = l2_evict_last();
      const int64_t cpos = (int64_t)client * npos;
      int stage = 0, ts = 0;
      uint32_t phase = 0, tph = 0;
      for (int pos = pos0; pos < pos1; ++pos)
        for (int task = 0; task < 2; ++task) {
          const int trow = (int)(((cpos + pos) * 2 + task) * 256);
          for (int kb = 0; kb < kKB; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], kTile);
            tma_load_2d_hint(BS + stage * kTile, &mapT, &full[stage], kb * kBK, trow, pol);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          mbar_wait(&tlempty[ts], tph ^ 1);
          mbar_expect_tx(&tlfull[ts], kTail);
          tma_load_2d_hint(BT + ts * kTail, &mapTail, &tlfull[ts], kKB * kBK, trow, pol);
          if (++ts == kTStages) {
            ts = 0;
            tph ^= 1;
          }
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: task A -> TMEM buffer 0, task B -> buffer 1 ----------------
      const uint32_t idesc = idesc_u8(kRows, 256);
      const uint64_t xtd = desc_sw32(smem_u32(XT));
      int stage = 0, ts = 0;
      uint32_t phase = 0, tph = 0, xph = 0;
      uint32_t eph[2] = {0, 0};
#ifdef ZPIR_TC_TRACE
      unsigned long long fwait = 0;   // cycles the MMA thread waited for table tiles this position
#endif
      for (int pos = pos0; pos < pos1; ++pos) {
        for (int task = 0; task < 2; ++task) {
          if (task == 0) {
            mbar_wait(xfull, xph);
            xph ^= 1;
          }
          if (pos > pos0) {                              // the buffer's previous drain
            mbar_wait(&tempty[task], eph[task]);
            eph[task] ^= 1;
          }
          tc_fence_after();
          TC_STAMP(pos, 11 + task);
          const uint32_t d = tbase + (uint32_t)(task * 256);
          for (int kb = 0; kb < kKB; ++kb) {
#ifdef ZPIR_TC_TRACE
            const unsigned long long tw0 = clock64();
            mbar_wait(&full[stage], phase);
            fwait += clock64() - tw0;
#else
            mbar_wait(&full[stage], phase);
#endif
            tc_fence_after();
            const uint64_t ad = desc_sw128(smem_u32(XA + kb * (kRows * kBK)));
            const uint64_t bd = desc_sw128(smem_u32(BS + stage * kTile));
#pragma unroll
            for (int k = 0; k < kBK / 32; ++k)
              umma_i8(d, ad + 2 * k, bd + 2 * k, idesc, (kb == 0 && k == 0) ? 0u : 1u);
            umma_commit(&empty[stage]);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          mbar_wait(&tlfull[ts], tph);
          tc_fence_after();
          umma_i8(d, xtd, desc_sw32(smem_u32(BT + ts * kTail)), idesc, 1u);
          umma_commit(&tlempty[ts]);
          if (++ts == kTStages) {
            ts = 0;
            tph ^= 1;
          }
          if (task == 1) umma_commit(xfree);             // X no longer read
          umma_commit(&tfull[task]);
        }
        TC_STAMP(pos, 13);
#ifdef ZPIR_TC_TRACE
        if (blockIdx.x == 0 && blockIdx.y == 0 && pos - pos0 < 64) g_tc_trace[(pos - pos0) * 16 + 15] = fwait;
        fwait = 0;
#endif
      }
    }
  } else {
    // ---------------- epilogue: one row per thread (TMEM lane), 4 warps ----------------
    const int quarter = warp & 3;
    const int t = quarter * 32 + lane;          // row within the tile = TMEM lane
    const int64_t r = row0 + t;
    const int64_t er = r < rows ? (rid ? (int64_t)rid[r] : r) : 0;
    const int nb = ds.nb;
    uint32_t* Bc = Ball + (int64_t)client * rows_p * nb * kXL;
    const uint32_t lanebase = tbase + ((uint32_t)(quarter * 32) << 16);
    uint32_t fph[2] = {0, 0}, xfph = 0;
    const int kbl = lane >> 3, chl = lane & 7;  // this lane's 16-byte chunk of bytes 0..511
    const uint32_t xa_l = smem_u32(XA) + kbl * (kRows * kBK) + (uint32_t)(quarter * 32) * kBK;
    const uint32_t xa_t = smem_u32(XA) + t * kBK;                        // + k-block, chunk
    const uint32_t xt_t = smem_u32(XT) + t * kKT + (((t >> 2) & 1) << 4);  // chunk 0 of the tail row
    uint8_t* xa_row = XA + t * kBK;
    uint8_t* xt_row = XT + t * kKT + (((t >> 2) & 1) << 4);
    const int64_t rbase = row0 + quarter * 32;
    auto digit_at = [&](int p) -> uint32_t {
      if (r >= rows) return 0u;
      const int di = p / (int)n;
      return (E[er * rs + (p - (int64_t)di * n)] >> ds.off[di]) & ((1u << ds.width[di]) - 1u);
    };
    // X rows of the warp from their buckets, warp-cooperative async copies: lane
    // c moves bytes 16c..16c+15 of each of the warp's 32 rows into the SW128 A
    // layout (zero fill for digit 0), and the tail chunk of its own row. A row
    // with `fwd` set (digit repeats) is copied by its own thread instead: the low
    // half from the bucket it has just stored, the high half straight from the
    // drain of task B.
    auto gather_issue = [&](uint32_t dgv, uint32_t fwd) {
      const uint32_t sk = __ballot_sync(0xffffffffu, fwd != 0);
#pragma unroll 8
      for (int i = 0; i < 32; ++i) {
        const uint32_t d_i = __shfl_sync(0xffffffffu, dgv, i);
        if ((sk >> i) & 1u) continue;
        const uint32_t* src = Bc + ((rbase + i) * nb + (d_i ? d_i - 1 : 0)) * kXL + 4 * lane;
        const uint32_t dst = xa_l + i * kBK + ((chl ^ (i & 7)) << 4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                     "r"(d_i ? 16u : 0u)
                     : "memory");
      }
      const uint32_t* own = Bc + (r * nb + (dgv ? dgv - 1 : 0)) * kXL;
      if (!fwd) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(xt_t), "l"(own + kL),
                     "r"(dgv ? 16u : 0u)
                     : "memory");
      } else {
#pragma unroll 4
        for (int cc = 0; cc < 16; ++cc)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           xa_t + (cc >> 3) * (kRows * kBK) + (((cc & 7) ^ (t & 7)) << 4)),
                       "l"(own + 4 * cc)
                       : "memory");
      }
    };
    auto gather_publish = [&]() {
      asm volatile("cp.async.wait_all;" ::: "memory");
      fence_async_smem();
      mbar_arrive(xfull);
    };
    auto prefetch_bucket = [&](uint32_t d) {
      if (!d) return;
      const uint32_t* pb = Bc + (r * nb + d - 1) * kXL;
#pragma unroll
      for (int j = 0; j < 5; ++j) asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + 32 * j));
    };

    // prologue: X of the first position
    uint32_t dg = digit_at(pos0);
    gather_issue(dg, 0u);
    gather_publish();
    uint32_t dg_n = pos0 + 1 < pos1 ? digit_at(pos0 + 1) : 0u;
    prefetch_bucket(dg_n);

    for (int pos = pos0; pos < pos1; ++pos) {
      const bool last = pos + 1 >= pos1;
      const bool tr = threadIdx.x == 64;
      if (tr) TC_STAMP(pos, 0);
      uint32_t* brow = Bc + ((r * nb) + (dg ? dg - 1 : 0)) * kXL;
      // the next position's bucket is this position's (digit repeats): its X is
      // this position's output
      const uint32_t fwd = (!last && dg && dg_n == dg) ? 1u : 0u;
      // limbs awaiting a 32-byte store (one 256-bit STG per 8 limbs: whole sectors)
      uint32_t pend[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      unsigned long long carry = 0;
      // ---- task A: limbs 0..63
      mbar_wait(&tfull[0], fph[0]);
      fph[0] ^= 1;
      if (tr) TC_STAMP(pos, 1);
      tc_fence_after();
      drain256(lanebase, carry, [&](int g, const uint32_t (&v)[32]) {
#pragma unroll
        for (int k = 0; k < 8; ++k) pend[k] = limb4(v + 4 * k, carry);
        if (dg)
          asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(brow + 8 * g),
                       "r"(pend[0]), "r"(pend[1]), "r"(pend[2]), "r"(pend[3]), "r"(pend[4]),
                       "r"(pend[5]), "r"(pend[6]), "r"(pend[7])
                       : "memory");
      });
      if (tr) TC_STAMP(pos, 2);
      tc_fence_before();
      mbar_arrive(&tempty[0]);
      // ---- the next position's gather, once no MMA reads X any more; it lands
      // while task B is drained
      if (!last) {
        mbar_wait(xfree, xfph);
        xfph ^= 1;
        if (tr) TC_STAMP(pos, 3);
        gather_issue(dg_n, fwd);
        if (tr) TC_STAMP(pos, 4);
      }
      // ---- task B: limbs 64..127 and the carry out (limb 128)
      mbar_wait(&tfull[1], fph[1]);
      fph[1] ^= 1;
      if (tr) TC_STAMP(pos, 5);
      tc_fence_after();
      drain256(lanebase + 256u, carry, [&](int g, const uint32_t (&v)[32]) {
#pragma unroll
        for (int k = 0; k < 8; ++k) pend[k] = limb4(v + 4 * k, carry);
        if (dg)
          asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(brow + 64 + 8 * g),
                       "r"(pend[0]), "r"(pend[1]), "r"(pend[2]), "r"(pend[3]), "r"(pend[4]),
                       "r"(pend[5]), "r"(pend[6]), "r"(pend[7])
                       : "memory");
        if (fwd) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int cc = 16 + 2 * g + h, kb = cc >> 3, ch = cc & 7;
            *reinterpret_cast<uint4*>(xa_row + kb * (kRows * kBK) + ((ch ^ (t & 7)) << 4)) =
                make_uint4(pend[4 * h], pend[4 * h + 1], pend[4 * h + 2], pend[4 * h + 3]);
          }
        }
      });
      {
        const uint4 top = make_uint4((uint32_t)carry, 0u, 0u, 0u);
        if (dg) *reinterpret_cast<uint4*>(brow + kL) = top;
        if (fwd) *reinterpret_cast<uint4*>(xt_row) = top;
      }
      if (tr) TC_STAMP(pos, 6);
      tc_fence_before();
      mbar_arrive(&tempty[1]);
      if (!last) {
        gather_publish();                       // xfull for the next position
        if (tr) TC_STAMP(pos, 7);
        dg = dg_n;
        dg_n = pos + 2 < pos1 ? digit_at(pos + 2) : 0u;
        prefetch_bucket(dg_n);
      }
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

// (rows x 544) u8 table matrix, boxes of 256 rows x box_k K bytes.
static int table_map(CUtensorMap* map, const void* base, int64_t rows, int box_k,
                     CUtensorMapSwizzle sw) {
  auto fn = tcp_encode();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return kErrCuda;
  }
  cuuint64_t dims[2] = {(cuuint64_t)tcp::kTK, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)tcp::kTK};
  cuuint32_t box[2] = {(cuuint32_t)box_k, 256};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (tables) failed (%d)", (int)r);
    return kErrCuda;
  }
  return kOk;
}

// Digits per 32-bit exponent word; balanced widths, wider digits first.
static DigitSpec digit_spec() {
  constexpr int D = 6;
  DigitSpec ds{};
  ds.D = D;
  int off = 0, maxw = 0;
  for (int i = 0; i < D; ++i) {
    const int w = 32 / D + (i < 32 % D ? 1 : 0);
    ds.off[i] = off;
    ds.width[i] = w;
    off += w;
    maxw = std::max(maxw, w);
  }
  ds.nb = (1 << maxw) - 1;
  return ds;
}

int64_t tc_slot_fixed_workspace(int64_t n, int64_t rows, int clients) {
  using namespace tcp;
  const DigitSpec ds = digit_spec();
  const int64_t npos = ds.D * n;
  const int64_t rows_p = ceil_div(rows, kRows) * kRows;
  return (int64_t)clients * (npos * kL * 4 + npos * kCols * kTK + rows_p * ds.nb * kXL * 4);
}

// W_c[rid[r] or r] (Montgomery form, 4096-bit N_c) for rows r < rows of 32-bit
// exponent rows E[(rid[r] or r) * rs + k], for `clients` independent keys in one
// launch: the slot_fixed contract (P_c = the client's pow8 table, of which the
// first n entries -- the Montgomery bases -- are read) with the bucket updates
// on tcgen05.
int tc_slot_fixed_many_launch(int clients, const uint32_t* const* P, const uint32_t* const* N,
                              const uint32_t* np, const uint32_t* const* one_m,
                              uint32_t* const* W, int64_t n, const uint32_t* E, int64_t rs,
                              const int32_t* rid, int64_t rows, cudaStream_t st) {
  using namespace tcp;
  const DigitSpec ds = digit_spec();
  const int nb = ds.nb;
  const int64_t npos = ds.D * n;
  if (clients <= 0 || clients > 65535 || n <= 0 || rows <= 0 || npos > 65536 ||
      (int64_t)clients * npos * kCols >= (1ll << 31)) {
    set_error("tc_slot_fixed: bad shapes (clients=%d n=%lld rows=%lld)", clients, (long long)n,
              (long long)rows);
    return kErrInput;
  }
  {
    // keep the multi-GB workspace in the stream-ordered pool between calls
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
  const int C = clients;
  const int64_t tiles = ceil_div(rows, kRows);
  const int64_t rows_p = tiles * kRows;
  std::vector<TcClient> hc(C);
  for (int c = 0; c < C; ++c) hc[c] = {P[c], N[c], one_m[c], W[c], np[c]};
  TcClient* dcl = nullptr;
  uint32_t *Pd = nullptr, *Bk = nullptr;
  uint8_t* T = nullptr;
  auto release = [&]() {
    if (dcl) cudaFreeAsync(dcl, st);
    if (Pd) cudaFreeAsync(Pd, st);
    if (T) cudaFreeAsync(T, st);
    if (Bk) cudaFreeAsync(Bk, st);
  };
  auto fail = [&](const char* what) {
    release();
    cudaGetLastError();
    set_error("tc_slot_fixed: %s", what);
    return kErrCuda;
  };
  if (cudaMallocAsync(reinterpret_cast<void**>(&dcl), sizeof(TcClient) * C, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&Pd), (size_t)C * npos * kL * 4, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&T), (size_t)C * npos * kCols * kTK, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&Bk), (size_t)C * rows_p * nb * kXL * 4, st) != cudaSuccess)
    return fail("workspace allocation");
  // the host vector is read at enqueue time for pageable memory (synchronous copy)
  if (cudaMemcpyAsync(dcl, hc.data(), sizeof(TcClient) * C, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return fail("client table");
  powtab_kernel<<<dim3((unsigned)ceil_div(n, 4), C), 128, 0, st>>>(dcl, n, ds, Pd);
  table_kernel<<<dim3((unsigned)ceil_div(npos, 4), C), 128, 0, st>>>(dcl, Pd, npos, T);
  {
    const int64_t cnt = rows_p * nb;
    bucket_fill_kernel<<<dim3((unsigned)ceil_div(cnt * kXL, 256), C), 256, 0, st>>>(dcl, Bk, cnt);
  }
  if (check_launch("tc_slot_fixed setup")) return fail("setup kernels");
  CUtensorMap mT, mTail;
  if (table_map(&mT, T, (int64_t)C * npos * kCols, kBK, CU_TENSOR_MAP_SWIZZLE_128B) ||
      table_map(&mTail, T, (int64_t)C * npos * kCols, kKT, CU_TENSOR_MAP_SWIZZLE_32B))
    return fail("tensor maps");
  cudaFuncSetAttribute(tc_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  // one launch walks every position (tiles are independent); chunked so a
  // launch stays well under a second
  constexpr int64_t chunk = 4096;
  const int64_t ck = std::max<int64_t>(1, chunk / std::max<int64_t>(1, ceil_div(tiles * C, 2 * 148)));
  for (int64_t p0 = 0; p0 < npos; p0 += ck) {
    const int64_t p1 = std::min<int64_t>(npos, p0 + ck);
    tc_step_kernel<<<dim3((unsigned)tiles, C), kThreads, kSmem, st>>>(
        mT, mTail, ds, E, rs, rid, n, npos, (int)p0, (int)p1, rows, rows_p, Bk);
  }
  if (check_launch("tc_step")) return fail("tc_step launch");
  bucket_combine_kernel<<<dim3((unsigned)ceil_div(rows, 4), C), 128, 0, st>>>(dcl, Bk, nb, rows,
                                                                             rows_p, rid);
  if (check_launch("bucket_combine")) return fail("bucket_combine");
  release();
  return check_launch("tc_slot_fixed");
}

#ifdef ZPIR_TC_TRACE
extern "C" int zpir_tc_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_tc_trace, sizeof(g_tc_trace)) == cudaSuccess ? 0 : 2;
}
#endif

// Single-client form (the original entry point).
int tc_slot_fixed_launch(const uint32_t* P, int64_t n, const uint32_t* E, int64_t rs, int64_t rows,
                         const uint32_t* N, uint32_t np, const uint32_t* one_m, uint32_t* W,
                         cudaStream_t st) {
  return tc_slot_fixed_many_launch(1, &P, &N, &np, &one_m, &W, n, E, rs, nullptr, rows, st);
}

}  // namespace zpir
