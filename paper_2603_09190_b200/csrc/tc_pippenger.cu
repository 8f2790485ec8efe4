// Per-client hint on the tensor cores: the Pippenger bucket updates of
// slot_fixed (multiexp.cu) as Montgomery multiplications by a FIXED multiplier.
//
// W[r] = prod_{pos < D n} P[pos]^{digit(r, pos)}: every 32-bit exponent word
// H[r][k] is cut into D digits (DigitSpec, default D = 6: widths 6,6,5,5,5,5),
// pos = i n + k, digit(r, pos) = digit i of H[r][k] and P[pos] = ck_r[k]^(2^off_i)
// (powtab_kernel, Montgomery form mod N = m^2). Position-major Pippenger: at
// every position each row multiplies ONE of its 2^w - 1 buckets by the same
// Y = P[pos], so a position is a batch "X (rows) times fixed Y mod N" --
// Toeplitz int8 GEMMs:
//   u = X * Y' mod R          (Y' = Y * N' mod R, N' = -N^-1 mod R, R = 2^4096)
//   Z = (X * Y + u * N) / R   (< 2N; the conditional subtraction is deferred)
// with a byte-Toeplitz B operand Toep(y)[j][a] = byte_{delta + j - a}(y).
//
// Only 1028 of the 1536 byte columns of u and X*Y + u*N are ever drained from
// TMEM: S = X*Y + u*N is an exact multiple of R, every column sum is < 2^27,
// so the carry out of the low half is ceil(low4 / 2^32) with low4 the 4 byte
// columns 508..511 (the columns below add e < 2^20 to low4 / 2^32 and the total
// is an integer). Per position and 128-row tile: four 256-column tasks
//   U0, U1: columns 0..255 / 256..511 of X * Y'        -> u into shared memory
//   H0:     columns 508..763 of X * Y + u * N           -> carry, Z limbs 0..62
//   H1:     columns 764..1019                           -> Z limbs 63..126
// and the three top columns 1020..1022 (12 byte products) on the CUDA cores.
// 20 k-blocks (80 N = 256 MMAs) per position; the tasks ping-pong two TMEM
// buffers so the epilogue drains one while the MMA warp fills the other. The
// X * Y parts of H0 and H1 are issued before the u * N parts, so the next
// position's bucket gather (cp.async) overlaps the H drains; a row whose digit
// repeats gets its next X forwarded from Z by its own thread.
//
// Several clients (independent keys) run in one launch: blockIdx.y = client,
// every client with its own Toeplitz tiles, buckets and output rows; rows may be
// a subset of the exponent rows (row ids), which is the incremental refresh.
// The bucket combine (prod_d B_d^d, running sums) stays on the IMAD warp path.
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
constexpr int kRows = 128;         // rows per tile (TMEM lanes)
constexpr int kBK = 128;           // K bytes per k-block
constexpr int kTile = 256 * kBK;   // one Toeplitz tile: 256 columns x 128 K bytes
constexpr int kTYp = 4;            // Y' tiles: delta = -128 + 128 t (U0, U1)
constexpr int kDeltaYp = -128;
constexpr int kTY = 5;             // Y / N tiles: delta = 124 + 128 t (H0, H1)
constexpr int kDeltaY = 124;
constexpr int kStages = 3;
constexpr int kThreads = 192;
constexpr int kABytes = kRows * 512;     // one 128 x 512-byte A operand (4 k-blocks)
constexpr int kSmem = 2 * kABytes + kStages * kTile + 1024 + 1024;
constexpr int kNSteps = 20;

// The static MMA schedule: task (0 U0, 1 U1, 2 H0, 3 H1; TMEM buffer = task & 1),
// A operand (0 = X, 1 = u), k-block, B source (0 = Y', 1 = Y, 2 = N), tile t,
// issue segment: 0 U0, 1 U1, 2 H0 X*Y, 3 H1 X*Y (then X is free), 4 H0 u*N, 5 H1 u*N.
struct Step {
  int8_t task, a, ka, src, t, seg;
};
__constant__ Step kSched[kNSteps];

}  // namespace tcp

// Per-client arguments of one batched launch (device copy).
struct TcClient {
  const uint32_t* P;        // (npos, 128) Montgomery multipliers
  const uint32_t* N;        // 128 limbs of N = m^2
  const uint32_t* one;      // R mod N
  const uint32_t* Nprime;   // -N^-1 mod R
  uint32_t* W;              // output rows (Montgomery form), indexed by exponent row
  uint32_t np;              // -N^-1 mod 2^32
};

// Radix of the exponent digits: D digits per 32-bit exponent word, digit i
// = bits off[i] .. off[i] + width[i] - 1; nb = 2^max(width) - 1 buckets per row.
// Fewer, wider digits mean fewer positions (tensor-core work, 4n at D = 4) but
// more buckets to combine on the IMAD path (2 nb Montgomery products per row).
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

// tiles[((c * npos + p) * T + t) * 256 + j][a] = byte_{delta0 + 128 t + j - a}(y_{c,p}),
// zero outside [0, 512); y = Y[c][p] (which = 1, fixed stride) or the client's N.
__global__ void __launch_bounds__(256)
toep_tiles_kernel(const TcClient* __restrict__ cl, int which, const uint32_t* __restrict__ Ybase,
                  int64_t npos, int T, int delta0, uint8_t* __restrict__ tiles) {
  const int64_t pt = blockIdx.x;                 // p * T + t
  const int c = blockIdx.y;
  const int64_t p = pt / T;
  const int t = (int)(pt - p * T);
  const int j = threadIdx.x;
  const uint32_t* ysrc = which == 1 ? Ybase + ((int64_t)c * npos + p) * tcp::kL : cl[c].N;
  const uint8_t* y = reinterpret_cast<const uint8_t*>(ysrc);
  const int delta = delta0 + 128 * t;
  uint8_t* row = tiles + (((int64_t)c * npos * T + pt) * 256 + j) * tcp::kBK;
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

// out[c][p] = Pd_c[p] * Nprime_c mod 2^4096, one thread per value (product scanning).
__global__ void __launch_bounds__(128)
mul_lo_kernel(const TcClient* __restrict__ cl, const uint32_t* __restrict__ Pd, int64_t npos,
              uint32_t* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (p >= npos) return;
  const uint32_t* y = Pd + ((int64_t)c * npos + p) * tcp::kL;
  const uint32_t* Np = cl[c].Nprime;
  uint32_t* o = out + ((int64_t)c * npos + p) * tcp::kL;
  unsigned long long lo = 0, hi = 0;  // 128-bit column accumulator (lo, hi)
  for (int k = 0; k < tcp::kL; ++k) {
    for (int i = 0; i <= k; ++i) {
      const unsigned long long pr = (unsigned long long)y[i] * Np[k - i];
      const unsigned long long s = lo + pr;
      hi += (s < lo);
      lo = s;
    }
    o[k] = (uint32_t)lo;
    lo = (lo >> 32) | (hi << 32);
    hi >>= 32;
  }
}

__global__ void bucket_fill_kernel(const TcClient* __restrict__ cl, uint32_t* __restrict__ B,
                                   int64_t count) {
  const int c = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // u32 index
  if (i < count * tcp::kL) B[(int64_t)c * count * tcp::kL + i] = cl[c].one[i % tcp::kL];
}

// W[row] = prod_d B[r][d]^d (running sums from d = nb down), Montgomery form.
// Buckets are stored lazily reduced: flag F[r][d] set means "subtract N (mod R)".
__global__ void __launch_bounds__(128)
bucket_combine_kernel(const TcClient* __restrict__ cl, const uint32_t* __restrict__ Ball,
                      const uint8_t* __restrict__ Fall, int nb, int64_t rows, int64_t rows_p,
                      const int32_t* __restrict__ rid) {
  constexpr int LPL = tcp::kL / 32;
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.y;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const uint32_t np = cl[c].np;
  uint32_t n_[LPL], run[LPL], tot[LPL], x[LPL];
  big_load<LPL>(n_, cl[c].N, lane);
  const uint32_t* br = Ball + ((int64_t)c * rows_p + r) * nb * tcp::kL;
  const uint8_t* fr = Fall + ((int64_t)c * rows_p + r) * nb;
  big_load<LPL>(run, br + (nb - 1) * tcp::kL, lane);
  if (fr[nb - 1]) big_cond_sub<LPL>(run, 1u, n_, lane);
  big_copy<LPL>(tot, run);
  for (int d = nb - 1; d >= 1; --d) {
    big_load<LPL>(x, br + (d - 1) * tcp::kL, lane);
    if (fr[d - 1]) big_cond_sub<LPL>(x, 1u, n_, lane);
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

// Pippenger positions pos0..pos1-1 for one 128-row tile of one client per CTA
// (tiles are independent: a row only touches its own buckets):
//   B[r][d - 1] *= P[pos] for d = digit(r, pos) != 0.
__global__ void __launch_bounds__(tcp::kThreads, 1)
tc_step_kernel(const __grid_constant__ CUtensorMap mapYp, const __grid_constant__ CUtensorMap mapY,
               const __grid_constant__ CUtensorMap mapN, const TcClient* __restrict__ cl,
               const uint32_t* __restrict__ Pd, const __grid_constant__ DigitSpec ds,
               const uint32_t* __restrict__ E, int64_t rs, const int32_t* __restrict__ rid,
               int64_t n, int64_t npos, int pos0, int pos1, int64_t rows, int64_t rows_p,
               uint32_t* __restrict__ Ball, uint8_t* __restrict__ Fall) {
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
  uint64_t* uready = xfull + 1;             // all 512 bytes of u written
  uint64_t* tfull = uready + 1;             // [2] per TMEM buffer
  uint64_t* tempty = tfull + 2;             // [2]
  uint64_t* xfree = tempty + 2;             // every MMA reading X of this position done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(xfree + 2);
  uint32_t* sN = tslot + 4;                 // N limbs (512 B)

  const int client = blockIdx.y;
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
    mbar_init(uready, 128);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    mbar_init(xfree, 1);
    fence_mbar_init();
  }
  const uint32_t* Ncl = cl[client].N;
  for (int i = threadIdx.x; i < kL; i += blockDim.x) sN[i] = Ncl[i];
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const int64_t row0 = (int64_t)blockIdx.x * kRows;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: the 20 B tiles of every position ----------------
      const uint64_t pol = l2_evict_last();
      const int64_t cpos = (int64_t)client * npos;
      int stage = 0;
      uint32_t phase = 0;
      for (int pos = pos0; pos < pos1; ++pos)
        for (int s = 0; s < kNSteps; ++s) {
          const Step st = kSched[s];
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], kTile);
          uint8_t* dst = BS + stage * kTile;
          if (st.src == 0)
            tma_load_2d_hint(dst, &mapYp, &full[stage], 0, (int)(((cpos + pos) * kTYp + st.t) * 256),
                             pol);
          else if (st.src == 1)
            tma_load_2d_hint(dst, &mapY, &full[stage], 0, (int)(((cpos + pos) * kTY + st.t) * 256),
                             pol);
          else
            tma_load_2d_hint(dst, &mapN, &full[stage], 0, (client * kTY + st.t) * 256, pol);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: six segments per position, buffer = task & 1 ----------------
      const uint32_t idesc = idesc_u8(kRows, 256);
      int stage = 0;
      uint32_t phase = 0, xph = 0;
      uint32_t eph[2] = {0, 0};
      bool used0 = false, used1 = false;
#ifdef ZPIR_TC_TRACE
      unsigned long long fwait = 0;   // cycles the MMA thread waited for B tiles this position
#endif
      for (int pos = pos0; pos < pos1; ++pos) {
        int cur = -1;
        bool first = true;
        for (int s = 0; s < kNSteps; ++s) {
          const Step st = kSched[s];
          const int buf = st.task & 1;
          if (st.seg != cur) {
            if (cur == 0) umma_commit(&tfull[0]);          // U0 -> epilogue
            else if (cur == 1) umma_commit(&tfull[1]);     // U1
            else if (cur == 3) umma_commit(xfree);         // X no longer read
            else if (cur == 4) umma_commit(&tfull[0]);     // H0
            switch (st.seg) {
              case 0:                                      // buffer 0 after H0(pos-1) drained
                if (used0) { mbar_wait(&tempty[0], eph[0]); eph[0] ^= 1; }
                used0 = true;
                mbar_wait(xfull, xph);
                break;
              case 1:                                      // buffer 1 after H1(pos-1) drained
                if (used1) { mbar_wait(&tempty[1], eph[1]); eph[1] ^= 1; }
                used1 = true;
                break;
              case 2:                                      // U0 drained
                mbar_wait(&tempty[0], eph[0]); eph[0] ^= 1;
                break;
              case 3:                                      // U1 drained
                mbar_wait(&tempty[1], eph[1]); eph[1] ^= 1;
                break;
              case 4:                                      // all of u written
                mbar_wait(uready, xph);
                break;
              default:
                break;
            }
            tc_fence_after();
            cur = st.seg;
            if (cur < 4) TC_STAMP(pos, 11 + cur);
            first = cur <= 3;                              // u * N accumulates onto X * Y
          }
#ifdef ZPIR_TC_TRACE
          const unsigned long long tw0 = clock64();
          mbar_wait(&full[stage], phase);
          fwait += clock64() - tw0;
#else
          mbar_wait(&full[stage], phase);
#endif
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
        umma_commit(&tfull[1]);                            // H1
#ifdef ZPIR_TC_TRACE
        if (blockIdx.x == 0 && blockIdx.y == 0 && pos - pos0 < 64) g_tc_trace[(pos - pos0) * 16 + 15] = fwait;
        fwait = 0;
#endif
        xph ^= 1;
      }
    }
  } else {
    // ---------------- epilogue: one row per thread (TMEM lane), 4 warps ----------------
    const int quarter = warp & 3;
    const int t = quarter * 32 + lane;          // row within the tile = TMEM lane
    const int64_t r = row0 + t;
    const int64_t er = r < rows ? (rid ? (int64_t)rid[r] : r) : 0;
    const int nb = ds.nb;
    uint32_t* Bc = Ball + (int64_t)client * rows_p * nb * kL;
    uint8_t* Fc = Fall + (int64_t)client * rows_p * nb;
    const uint32_t* Pc = Pd + (int64_t)client * npos * kL;
    const uint32_t lanebase = tbase + ((uint32_t)(quarter * 32) << 16);
    uint32_t nl[4];                             // N limbs 4 lane .. 4 lane + 3 (gather)
#pragma unroll
    for (int i = 0; i < 4; ++i) nl[i] = sN[4 * lane + i];
    const uint32_t ntop = sN[kL - 1], n126 = sN[kL - 2];
    uint32_t fph[2] = {0, 0}, xfph = 0;
    const int kbl = lane >> 3, chl = lane & 7;  // this lane's 16-byte chunk of a row
    const uint32_t xa_l = smem_u32(XA) + kbl * (kRows * kBK) + (uint32_t)(quarter * 32) * kBK;
    const int64_t rbase = row0 + quarter * 32;
    auto digit_at = [&](int p) -> uint32_t {
      if (r >= rows) return 0u;
      const int di = p / (int)n;
      return (E[er * rs + (p - (int64_t)di * n)] >> ds.off[di]) & ((1u << ds.width[di]) - 1u);
    };
    // X rows of the warp from their buckets, warp-cooperative async copies: lane
    // c moves bytes 16c..16c+15 of each of the warp's 32 rows into the SW128 A
    // layout (zero fill for digit 0); rows with `skip` set are written by their
    // own thread instead (bucket updated at this very position).
    auto gather_issue = [&](uint32_t dgv, uint32_t skip) {
      const uint32_t sk = __ballot_sync(0xffffffffu, skip != 0);
#pragma unroll 8
      for (int i = 0; i < 32; ++i) {
        const uint32_t d_i = __shfl_sync(0xffffffffu, dgv, i);
        if ((sk >> i) & 1u) continue;
        const uint32_t* src = Bc + ((rbase + i) * nb + (d_i ? d_i - 1 : 0)) * kL + 4 * lane;
        const uint32_t dst = xa_l + i * kBK + ((chl ^ (i & 7)) << 4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                     "r"(d_i ? 16u : 0u)
                     : "memory");
      }
    };
    // copies landed; lazily reduced buckets: a set flag means the stored value
    // is Z with Z - N still to be taken (mod R)
    // gather_land: the copies landed, lazily reduced buckets reduced in place;
    // gather_publish: X complete (conflict rows forwarded) -> the MMA warp
    auto gather_land = [&](uint32_t lz) {
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncwarp();
      uint32_t lzm = __ballot_sync(0xffffffffu, lz != 0);
      while (lzm) {
        const int i = __ffs(lzm) - 1;
        lzm &= lzm - 1;
        uint8_t* q = XA + kbl * (kRows * kBK) + (quarter * 32 + i) * kBK + ((chl ^ (i & 7)) << 4);
        uint4 w = *reinterpret_cast<const uint4*>(q);
        uint32_t v[4] = {w.x, w.y, w.z, w.w};
        big_cond_sub<4>(v, 1u, nl, lane);       // x - N mod R (warp-uniform)
        *reinterpret_cast<uint4*>(q) = make_uint4(v[0], v[1], v[2], v[3]);
      }
    };
    auto gather_publish = [&]() {
      fence_async_smem();
      mbar_arrive(xfull);
      __syncwarp();
    };
    auto gather_finish = [&](uint32_t lz) {
      gather_land(lz);
      gather_publish();
    };
    // bytes 508..511 of this row's X (k-block 3, chunk 7)
    const uint32_t* xtop_p =
        reinterpret_cast<const uint32_t*>(XA + 3 * (kRows * kBK) + t * kBK + ((7 ^ (t & 7)) << 4) + 12);
    auto prefetch_bucket = [&](uint32_t d) {
      if (!d) return;
      const uint32_t* pb = Bc + (r * nb + d - 1) * kL;
#pragma unroll
      for (int j = 0; j < 4; ++j) asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + 32 * j));
    };

    // prologue: X of the first position
    uint32_t dg = digit_at(pos0);
    gather_issue(dg, 0u);
    gather_finish((dg && Fc[r * nb + dg - 1]) ? 1u : 0u);
    uint32_t xtop = *xtop_p;
    uint32_t dg_n = pos0 + 1 < pos1 ? digit_at(pos0 + 1) : 0u;
    prefetch_bucket(dg_n);

    for (int pos = pos0; pos < pos1; ++pos) {
      const bool last = pos + 1 >= pos1;
      const bool tr = threadIdx.x == 64;
      if (tr) TC_STAMP(pos, 0);
      const int64_t bidx = (r * nb) + (dg ? dg - 1 : 0);
      uint32_t* brow = Bc + bidx * kL;
      const uint32_t ytop = Pc[(int64_t)pos * kL + kL - 1];
      // the next position's bucket is this position's (digit repeats): its X is
      // this position's Z, written into the A layout by this thread below
      const uint32_t conflict = (!last && dg && dg_n == dg) ? 1u : 0u;
      const uint32_t lazy_n = (!last && dg_n && !conflict && Fc[r * nb + dg_n - 1]) ? 1u : 0u;

      unsigned long long carry = 0;
      uint32_t utop = 0;
      // ---- U0, U1: u = X * Y' mod R, limbs into the SW128 A layout of u
#pragma unroll 1
      for (int task = 0; task < 2; ++task) {
        mbar_wait(&tfull[task], fph[task]);
        fph[task] ^= 1;
        if (tr) TC_STAMP(pos, 1 + 2 * task);
        tc_fence_after();
        const uint32_t taddr = lanebase + (uint32_t)(task * 256);
        drain256(taddr, carry, [&](int g, const uint32_t (&v)[32]) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {        // 16-byte chunk of u: 4 limbs
            uint32_t l[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) l[i] = limb4(v + 16 * j + 4 * i, carry);
            const int cc = task * 16 + 2 * g + j;
            const int kb = cc >> 3, ch = cc & 7;
            *reinterpret_cast<uint4*>(UA + kb * (kRows * kBK) + t * kBK + ((ch ^ (t & 7)) << 4)) =
                make_uint4(l[0], l[1], l[2], l[3]);
            utop = l[3];
          }
        });
        if (tr) TC_STAMP(pos, 2 + 2 * task);
        if (task == 1) {
          fence_async_smem();
          mbar_arrive(uready);
        }
        tc_fence_before();
        mbar_arrive(&tempty[task]);
      }
      // ---- the next position's gather, once no MMA reads X any more; it lands
      // while H0 / H1 are computed and drained
      if (!last) {
        mbar_wait(xfree, xfph);
        xfph ^= 1;
        if (tr) TC_STAMP(pos, 5);
        gather_issue(dg_n, conflict);
        // land + reduce the gathered rows now: the epilogue would otherwise
        // idle until H0 is computed, and this work leaves the critical path
        gather_land(lazy_n);
      }
      // ---- H0, H1: Z = (X * Y + u * N) / R from columns 508..1019 (+ 1020..1022)
      // Z limbs awaiting a 32-byte store (one 256-bit STG per 8 limbs: whole
      // sectors, half the store instructions of 16-byte stores)
      uint32_t pend[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      auto emit = [&](int li) {               // limbs li-7..li complete
        if (dg)
          asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(brow + li - 7),
                       "r"(pend[0]), "r"(pend[1]), "r"(pend[2]), "r"(pend[3]), "r"(pend[4]),
                       "r"(pend[5]), "r"(pend[6]), "r"(pend[7])
                       : "memory");
        if (conflict) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int cc = ((li - 7) >> 2) + h, kb = cc >> 3, ch = cc & 7;
            *reinterpret_cast<uint4*>(XA + kb * (kRows * kBK) + t * kBK + ((ch ^ (t & 7)) << 4)) =
                make_uint4(pend[4 * h], pend[4 * h + 1], pend[4 * h + 2], pend[4 * h + 3]);
          }
        }
      };
      carry = 0;
      {
        mbar_wait(&tfull[0], fph[0]);
        fph[0] ^= 1;
        if (tr) TC_STAMP(pos, 6);
        tc_fence_after();
        const uint32_t taddr = lanebase;
        drain256(taddr, carry, [&](int g, const uint32_t (&v)[32]) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int slot = 8 * g + k;        // columns 508 + 4 slot ..
            if (slot == 0) {
              // low4 = columns 508..511 as one number (< 2^54)
              const unsigned long long low4 =
                  (unsigned long long)v[0] + ((unsigned long long)v[1] << 8) +
                  ((unsigned long long)v[2] << 16) + ((unsigned long long)v[3] << 24);
              carry = (low4 + 0xffffffffull) >> 32;
              continue;
            }
            const int li = slot - 1;           // Z limb
            pend[li & 7] = limb4(v + 4 * k, carry);
            if ((li & 7) == 7) emit(li);
          }
        });
        if (tr) TC_STAMP(pos, 7);
        tc_fence_before();
        mbar_arrive(&tempty[0]);
      }
      {
        mbar_wait(&tfull[1], fph[1]);
        fph[1] ^= 1;
        if (tr) TC_STAMP(pos, 8);
        tc_fence_after();
        const uint32_t taddr = lanebase + 256u;
        drain256(taddr, carry, [&](int g, const uint32_t (&v)[32]) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int li = 63 + 8 * g + k;     // columns 764 + 4 (li - 63) ..
            pend[li & 7] = limb4(v + 4 * k, carry);
            if ((li & 7) == 7) emit(li);
          }
        });
        if (tr) TC_STAMP(pos, 9);
        tc_fence_before();
        mbar_arrive(&tempty[1]);
      }
      // columns 1020..1022 (1023 is empty): bytes 509..511 of X, Y, u, N
      {
        const uint32_t x9 = (xtop >> 8) & 0xffu, x10 = (xtop >> 16) & 0xffu, x11 = xtop >> 24;
        const uint32_t y9 = (ytop >> 8) & 0xffu, y10 = (ytop >> 16) & 0xffu, y11 = ytop >> 24;
        const uint32_t u9 = (utop >> 8) & 0xffu, u10 = (utop >> 16) & 0xffu, u11 = utop >> 24;
        const uint32_t n9 = (ntop >> 8) & 0xffu, n10 = (ntop >> 16) & 0xffu, n11 = ntop >> 24;
        const uint32_t c0 = x9 * y11 + x10 * y10 + x11 * y9 + u9 * n11 + u10 * n10 + u11 * n9;
        const uint32_t c1 = x10 * y11 + x11 * y10 + u10 * n11 + u11 * n10;
        const uint32_t c2 = x11 * y11 + u11 * n11;
        const unsigned long long s = (unsigned long long)c0 + ((unsigned long long)c1 << 8) +
                                     ((unsigned long long)c2 << 16) + carry;
        const uint32_t z = (uint32_t)s;
        const uint32_t top = (uint32_t)(s >> 32);
        pend[7] = z;
        emit(kL - 1);
        // Z = z + 2^4096 * top < 2N: Z >= N iff the top carry is set or z >= N,
        // decided by the top two limbs unless both equal N's (then by all of
        // them, read back). The bucket keeps Z and a flag (the subtraction is
        // deferred to its next reader); the forwarded X is reduced right here.
        uint32_t f;
        if (top) {
          f = 1u;
        } else if (pend[7] != ntop || pend[6] != n126) {
          f = (pend[7] > ntop || (pend[7] == ntop && pend[6] > n126)) ? 1u : 0u;
        } else {
          f = 1u;                                // z == N so far: equal counts as >=
          const uint32_t* zs = conflict ? nullptr : brow;
          for (int li = kL - 3; li >= 0; --li) {
            uint32_t zl;
            if (zs) {
              zl = zs[li];
            } else {
              const int cc = li >> 2, kb = cc >> 3, ch = cc & 7;
              zl = reinterpret_cast<const uint32_t*>(
                  XA + kb * (kRows * kBK) + t * kBK + ((ch ^ (t & 7)) << 4))[li & 3];
            }
            if (zl != sN[li]) {
              f = zl > sN[li] ? 1u : 0u;
              break;
            }
          }
        }
        if (dg) Fc[bidx] = (uint8_t)f;
        if (conflict && f) {
          uint32_t bw = 0;
#pragma unroll 1
          for (int cc = 0; cc < 32; ++cc) {
            const int kb = cc >> 3, ch = cc & 7;
            uint4* q = reinterpret_cast<uint4*>(XA + kb * (kRows * kBK) + t * kBK + ((ch ^ (t & 7)) << 4));
            uint4 w = *q;
            uint32_t v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const unsigned long long d = (unsigned long long)v[i] - sN[4 * cc + i] - bw;
              v[i] = (uint32_t)d;
              bw = (uint32_t)(d >> 63);
            }
            *q = make_uint4(v[0], v[1], v[2], v[3]);
          }
        }
      }
      if (!last) {
        gather_publish();                       // xfull for the next position
        if (tr) TC_STAMP(pos, 10);
        xtop = *xtop_p;
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
  // U0, U1: output columns 256 gc .. of X * Y', tile delta = 256 gc - 128 ka
  for (int gc = 0; gc < 2; ++gc)
    for (int ka = 0; ka < 4; ++ka) {
      const int delta = 256 * gc - 128 * ka;
      const int t = (delta - tcp::kDeltaYp) / 128;
      if (delta - 127 < 512 && delta + 255 >= 0 && t >= 0 && t < tcp::kTYp)
        h[k++] = {(int8_t)gc, 0, (int8_t)ka, 0, (int8_t)t, (int8_t)gc};
    }
  // H0, H1 (output columns c0 = 508 / 764 of X * Y + u * N): both X * Y parts
  // first (after them X is no longer read: the next position's gather may
  // start), then both u * N parts (they wait for u)
  for (int a = 0; a < 2; ++a)
    for (int hh = 0; hh < 2; ++hh) {
      const int c0 = 508 + 256 * hh;
      for (int ka = 0; ka < 4; ++ka) {
        const int delta = c0 - 128 * ka;
        if (delta - 127 >= 512) continue;           // window entirely above byte 511
        const int t = (delta - tcp::kDeltaY) / 128;
        h[k++] = {(int8_t)(2 + hh), (int8_t)a, (int8_t)ka, (int8_t)(a ? 2 : 1), (int8_t)t,
                  (int8_t)(2 + 2 * a + hh)};
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

// Digits per 32-bit exponent word: 6 (widths
// 6,6,5,5,5,5 and 63 buckets per row); balanced widths, wider digits first.
static DigitSpec digit_spec() {
  constexpr int D = 6;   // measured optimum of D = 4..7
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
  return (int64_t)clients * (2 * npos * kL * 4 + npos * (kTY + kTYp) * kTile + kTY * kTile +
                             rows_p * ds.nb * (kL * 4 + 1));
}

// W_c[rid[r] or r] (Montgomery form, 4096-bit N_c) for rows r < rows of 32-bit
// exponent rows E[(rid[r] or r) * rs + k], for `clients` independent keys in one
// launch: the slot_fixed contract (P_c = the client's pow8 table, of which the
// first n entries -- the Montgomery bases -- are read) with the bucket updates
// on tcgen05.
int tc_slot_fixed_many_launch(int clients, const uint32_t* const* P, const uint32_t* const* N,
                              const uint32_t* np, const uint32_t* const* one_m,
                              const uint32_t* const* Nprime, uint32_t* const* W, int64_t n,
                              const uint32_t* E, int64_t rs, const int32_t* rid, int64_t rows,
                              cudaStream_t st) {
  using namespace tcp;
  const DigitSpec ds = digit_spec();
  const int nb = ds.nb;
  const int64_t npos = ds.D * n;
  if (clients <= 0 || clients > 65535 || n <= 0 || rows <= 0 || npos > 65536 ||
      (int64_t)clients * npos * kTY * 256 >= (1ll << 31)) {
    set_error("tc_slot_fixed: bad shapes (clients=%d n=%lld rows=%lld)", clients, (long long)n,
              (long long)rows);
    return kErrInput;
  }
  if (int e = upload_schedule()) return e;
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
  for (int c = 0; c < C; ++c) hc[c] = {P[c], N[c], one_m[c], Nprime[c], W[c], np[c]};
  TcClient* dcl = nullptr;
  uint32_t *Pd = nullptr, *Yp = nullptr, *Bk = nullptr;
  uint8_t *tY = nullptr, *tYp = nullptr, *tN = nullptr, *Fk = nullptr;
  auto release = [&]() {
    if (dcl) cudaFreeAsync(dcl, st);
    if (Pd) cudaFreeAsync(Pd, st);
    if (Yp) cudaFreeAsync(Yp, st);
    if (Bk) cudaFreeAsync(Bk, st);
    if (tY) cudaFreeAsync(tY, st);
    if (tYp) cudaFreeAsync(tYp, st);
    if (tN) cudaFreeAsync(tN, st);
    if (Fk) cudaFreeAsync(Fk, st);
  };
  auto fail = [&](const char* what) {
    release();
    cudaGetLastError();
    set_error("tc_slot_fixed: %s", what);
    return kErrCuda;
  };
  if (cudaMallocAsync(reinterpret_cast<void**>(&dcl), sizeof(TcClient) * C, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&Pd), (size_t)C * npos * kL * 4, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&Yp), (size_t)C * npos * kL * 4, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&tY), (size_t)C * npos * kTY * kTile, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&tYp), (size_t)C * npos * kTYp * kTile, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&tN), (size_t)C * kTY * kTile, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&Bk), (size_t)C * rows_p * nb * kL * 4, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&Fk), (size_t)C * rows_p * nb, st) != cudaSuccess)
    return fail("workspace allocation");
  // the host vector is read at enqueue time for pageable memory (synchronous copy)
  if (cudaMemcpyAsync(dcl, hc.data(), sizeof(TcClient) * C, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemsetAsync(Fk, 0, (size_t)C * rows_p * nb, st) != cudaSuccess)
    return fail("client table / flags");
  powtab_kernel<<<dim3((unsigned)ceil_div(n, 4), C), 128, 0, st>>>(dcl, n, ds, Pd);
  mul_lo_kernel<<<dim3((unsigned)ceil_div(npos, 128), C), 128, 0, st>>>(dcl, Pd, npos, Yp);
  toep_tiles_kernel<<<dim3((unsigned)(npos * kTY), C), 256, 0, st>>>(dcl, 1, Pd, npos, kTY,
                                                                     kDeltaY, tY);
  toep_tiles_kernel<<<dim3((unsigned)(npos * kTYp), C), 256, 0, st>>>(dcl, 1, Yp, npos, kTYp,
                                                                      kDeltaYp, tYp);
  toep_tiles_kernel<<<dim3((unsigned)kTY, C), 256, 0, st>>>(dcl, 2, nullptr, 1, kTY, kDeltaY, tN);
  {
    const int64_t cnt = rows_p * nb;
    bucket_fill_kernel<<<dim3((unsigned)ceil_div(cnt * kL, 256), C), 256, 0, st>>>(dcl, Bk, cnt);
  }
  if (check_launch("tc_slot_fixed setup")) return fail("setup kernels");
  CUtensorMap mYp, mY, mN;
  if (tile_map(&mYp, tYp, C * npos * kTYp * 256) || tile_map(&mY, tY, C * npos * kTY * 256) ||
      tile_map(&mN, tN, (int64_t)C * kTY * 256))
    return fail("tensor maps");
  cudaFuncSetAttribute(tc_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  // one launch walks every position (tiles are independent); chunked so a
  // launch stays well under a second
  constexpr int64_t chunk = 1024;
  const int64_t ck = std::max<int64_t>(1, chunk / std::max<int64_t>(1, ceil_div(tiles * C, 2 * 148)));
  for (int64_t p0 = 0; p0 < npos; p0 += ck) {
    const int64_t p1 = std::min<int64_t>(npos, p0 + ck);
    tc_step_kernel<<<dim3((unsigned)tiles, C), kThreads, kSmem, st>>>(
        mYp, mY, mN, dcl, Pd, ds, E, rs, rid, n, npos, (int)p0, (int)p1, rows, rows_p, Bk, Fk);
  }
  if (check_launch("tc_step")) return fail("tc_step launch");
  bucket_combine_kernel<<<dim3((unsigned)ceil_div(rows, 4), C), 128, 0, st>>>(dcl, Bk, Fk, nb, rows,
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
                         const uint32_t* N, uint32_t np, const uint32_t* one_m,
                         const uint32_t* Nprime, uint32_t* W, cudaStream_t st) {
  return tc_slot_fixed_many_launch(1, &P, &N, &np, &one_m, &Nprime, &W, n, E, rs, nullptr, rows, st);
}

}  // namespace zpir
