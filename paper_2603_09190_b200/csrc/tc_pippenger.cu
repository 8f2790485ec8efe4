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
// into two TMEM buffers (34 MMAs and 512 drained columns per position; the
// Montgomery form of this step needed 80 MMAs in a three-product chain and 1028
// drained columns). The bucket combine reduces each bucket once (quotient
// estimate from the top limbs, bignum.cuh) before its IMAD running products.
//
// Buckets hold Montgomery-form values and y is in standard form, so products
// stay in Montgomery form. A row whose digit repeats at the next position gets
// its next X forwarded from this position's output by its own thread.
//
// What bounds the step is the movement of the buckets, not the tensor pipe:
// every live row reads (cp.async) and writes (scattered 32-byte stores) one
// 544-byte bucket per position, 2.5e11 bytes per client at n = 1024, far beyond
// L2 (DRAM 43%, L2 61%, int8 tensor 55% of peak under ncu).
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
constexpr int kHalf = 128;         // table columns staged per CTA of a pair and task
constexpr int kTile = kHalf * kBK; // table stage: 128 columns x 128 K bytes (SW128)
constexpr int kTail = kHalf * kKT; // table tail stage: 128 columns x 32 K bytes (SW32)
constexpr int kStages = 4;
constexpr int kTStages = 4;
constexpr int kThreads = 320;     // tile X warps 0-3, tile Y warps 4-7, TMA warp 8, MMA warp 9
constexpr int kABytes = kRows * kKB * kBK;   // X bytes 0..511: 4 k-blocks of 128 x 128 B (SW128)
constexpr int kATail = kRows * kKT;          // X bytes 512..543 (SW32)
constexpr int kXBytes = kABytes + kATail;    // X of one tile
constexpr int kSmem = 2 * kXBytes + kStages * kTile + kTStages * kTail + 1024 + 1024;

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
// shift and one quotient-estimate reduction). A lane owns 16 byte rows (its 16
// bytes of t); it keeps 32 steps of 8 of them in registers and writes them as
// whole 32-byte sectors, walking the chain once per half of its rows (16-byte
// stores of all 16 rows in one walk leave every sector half written: 4.1 ms per
// client at n = 1024 against 2.9 ms for the two walks).
template <int HALF>
__device__ __forceinline__ void table_walk(uint32_t (&t)[4], const uint32_t (&n_)[4], uint32_t nt8,
                                           uint8_t* __restrict__ out, int lane) {
  constexpr int LPL = 4;
#pragma unroll 1
  for (int blk = 0; blk < tcp::kTK / 32; ++blk) {
    uint32_t acc[8][8];
#pragma unroll
    for (int s = 0; s < 32; ++s) {
      const bool live = 32 * blk + s < tcp::kUsedK;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        // byte 8 HALF + b of this lane's 16 bytes into byte s of the row segment
        const int bb = 8 * HALF + b;
        const uint32_t src = live ? t[bb >> 2] : 0u;
        const uint32_t byte = (src >> (8 * (bb & 3))) & 0xffu;
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
    for (int b = 0; b < 8; ++b)
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(
                       out + (int64_t)(8 * HALF + b) * tcp::kTK + 32 * blk),
                   "r"(acc[b][0]), "r"(acc[b][1]), "r"(acc[b][2]), "r"(acc[b][3]), "r"(acc[b][4]),
                   "r"(acc[b][5]), "r"(acc[b][6]), "r"(acc[b][7])
                   : "memory");
  }
}

__global__ void __launch_bounds__(128)
table_kernel(const TcClient* __restrict__ cl, const uint32_t* __restrict__ Pd, int64_t npos,
             uint8_t* __restrict__ T) {
  constexpr int LPL = tcp::kL / 32;
  static_assert(LPL == 4, "16 bytes per lane");
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.y;
  const int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= npos) return;
  uint32_t n_[LPL], y[LPL], t[LPL], e1[LPL];
  big_load<LPL>(n_, cl[c].N, lane);
  big_load<LPL>(y, Pd + ((int64_t)c * npos + p) * tcp::kL, lane);
  big_set_small<LPL>(e1, 1u, lane);
  mont_mul<LPL>(y, y, e1, n_, cl[c].np, lane);        // y in standard form, < N
  const uint32_t nt8 = (__shfl_sync(ZPIR_FULL, n_[LPL - 1], 31) >> 8) + 1u;
  uint8_t* out = T + (((int64_t)c * npos + p) * tcp::kCols + 16 * lane) * tcp::kTK;
  big_copy<LPL>(t, y);
  table_walk<0>(t, n_, nt8, out, lane);
  big_copy<LPL>(t, y);
  table_walk<1>(t, n_, nt8, out, lane);
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
__device__ __forceinline__ void tmem_wait_after(uint32_t dep) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::"r"(dep) : "memory");
}
__device__ __forceinline__ void regs_ready(uint32_t (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(v[i]));
}

// Drain 256 TMEM columns of this thread's lane in eight 32-column batches,
// double-buffered: batch g + 1 is in flight while batch g is processed.
// f(g, v) consumes columns 32 g .. 32 g + 31; it updates `carry`, which also
// orders the next wait after the processing. (Three buffers with two loads in
// flight shorten a drain by ~0.6k cycles and change nothing end to end: the
// position is bound by the load-store unit.)
template <class F>
__device__ __forceinline__ void drain256(uint32_t taddr, uint32_t& carry, F&& f) {
  uint32_t va[32], vb[32];
  tmem_ld32(taddr, va);
  tmem_wait_after(carry);
  regs_ready(va);
#pragma unroll 1
  for (int g = 0; g < 8; g += 2) {
    tmem_ld32(taddr + 32 * (g + 1), vb);
    f(g, va);
    tmem_wait_after(carry);
    regs_ready(vb);
    if (g < 6) tmem_ld32(taddr + 32 * (g + 2), va);
    f(g + 1, vb);
    if (g < 6) {
      tmem_wait_after(carry);
      regs_ready(va);
    }
  }
}

// 32 byte columns (s32 sums < 2^25) + carry in -> eight 32-bit limbs + carry
// out (< 2^26). Per limb s = v0 + 2^8 v1 + 2^16 v2 + 2^24 v3 in 32-bit pieces:
// lo = s mod 2^32 by wrapping shift-adds, hi = floor(s / 2^32) through the
// exact floors w1 = (v0 >> 8) + v1, w2 = (w1 >> 8) + v2, w3 = (w2 >> 8) + v3,
// hi = w3 >> 8 (64-bit multiply-adds run at a fraction of the 32-bit rate, and
// the drains are issue-bound). The eight (lo, hi) pairs are independent; only
// the final add-with-carry chain lo_k + hi_{k-1} is sequential.
__device__ __forceinline__ void limbs8(const uint32_t* v, uint32_t& cin, uint32_t (&out)[8]) {
  uint32_t lo[8], hi[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t v0 = v[4 * k], v1 = v[4 * k + 1], v2 = v[4 * k + 2], v3 = v[4 * k + 3];
    lo[k] = v0 + (v1 << 8) + (v2 << 16) + (v3 << 24);
    const uint32_t w1 = (v0 >> 8) + v1;
    const uint32_t w2 = (w1 >> 8) + v2;
    const uint32_t w3 = (w2 >> 8) + v3;
    hi[k] = w3 >> 8;
  }
  asm volatile(
      "add.cc.u32 %0, %9, %17;\n\t"
      "addc.cc.u32 %1, %10, %18;\n\t"
      "addc.cc.u32 %2, %11, %19;\n\t"
      "addc.cc.u32 %3, %12, %20;\n\t"
      "addc.cc.u32 %4, %13, %21;\n\t"
      "addc.cc.u32 %5, %14, %22;\n\t"
      "addc.cc.u32 %6, %15, %23;\n\t"
      "addc.cc.u32 %7, %16, %24;\n\t"
      "addc.u32 %8, %25, 0;"
      : "=r"(out[0]), "=r"(out[1]), "=r"(out[2]), "=r"(out[3]), "=r"(out[4]), "=r"(out[5]),
        "=r"(out[6]), "=r"(out[7]), "=r"(cin)
      : "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]),
        "r"(lo[7]), "r"(cin), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3]), "r"(hi[4]),
        "r"(hi[5]), "r"(hi[6]), "r"(hi[7]));
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

// Pippenger positions pos0..pos1-1 for TWO 128-row tiles of one client per CTA
// (tiles are independent: a row only touches its own buckets):
//   B[r][d - 1] <- B[r][d - 1] * y[pos] for d = digit(r, pos) != 0.
//
// CTA pairs (clusters of 2 on one TPC, tcgen05 cta_group::2): the leader issues
// M = 256 MMAs over both CTAs' X tiles, every CTA stages its own HALF of the
// table columns of a task (128 of 256: half the L2 -> SM and shared-memory
// traffic per MMA) and drains its own 128 TMEM lanes. The two tiles X and Y of a
// CTA alternate on the tensor pipe, position by position:
//   X.A(p) -> TMEM 0, X.B(p) -> TMEM 1, Y.A(p) -> TMEM 0, Y.B(p) -> TMEM 1, X.A(p+1) ...
// so everything a tile's next position depends on -- the drain of its task B
// (forwarded rows), the gather of its next X from the buckets, the drain that
// frees a TMEM buffer -- happens under the other tile's MMAs. Per CTA:
//   warps 0-3  tile X, one row per thread: drains, gather (cp.async)
//   warps 4-7  tile Y
//   warp 8     TMA producer (its table halves; completion on the leader's barrier)
//   warp 9     MMA issuer (leader only)
// (a scheduler serves its highest warp id first: the two single-thread warps
// must not wait behind the draining warps.)
__global__ void __launch_bounds__(tcp::kThreads, 1)
tc_step_kernel(const __grid_constant__ CUtensorMap mapT, const __grid_constant__ CUtensorMap mapTail,
               const __grid_constant__ DigitSpec ds, const uint32_t* __restrict__ E, int64_t rs,
               const int32_t* __restrict__ rid, int64_t n, int64_t npos, int pos0, int pos1,
               int64_t rows, int64_t rows_p, uint32_t* __restrict__ Ball) {
  using namespace tcp;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* XB = smem;                       // per tile: X bytes 0..511 (4 k-blocks of 128 x 128 B,
                                            // SW128), X bytes 512..543 (128 x 32 B, SW32)
  uint8_t* BS = XB + 2 * kXBytes;           // table stages (128 x 128 B)
  uint8_t* BT = BS + kStages * kTile;       // table tail stages (128 x 32 B)
  uint64_t* full = reinterpret_cast<uint64_t*>(BT + kTStages * kTail);   // leader
  uint64_t* empty = full + kStages;
  uint64_t* tlfull = empty + kStages;       // tail ring (leader)
  uint64_t* tlempty = tlfull + kTStages;
  uint64_t* xfull = tlempty + kTStages;     // [tile] leader: X of the tile complete in both CTAs
  uint64_t* tfull = xfull + 2;              // [tile][task] accumulator complete
  uint64_t* tempty = tfull + 4;             // [tile][task] leader: accumulator drained in both CTAs
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 4);

  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int client = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 8 && lane == 0) {
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
    for (int b = 0; b < 2; ++b) {
      mbar_init(&xfull[b], 2 * 128);
    }
    for (int b = 0; b < 4; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * 128);
    }
    fence_mbar_init();
  }
  // bytes 516..543 of every X stay zero
  for (int i = threadIdx.x; i < 2 * kATail / 16; i += blockDim.x) {
    const int b = i / (kATail / 16), j = i % (kATail / 16);
    reinterpret_cast<uint4*>(XB + b * kXBytes + kABytes)[j] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (warp == 9) tmem_alloc_pair(tslot, 512);
  tc_fence_before();
  cluster_sync();   // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 8) {
    if (lane == 0) {
      // ---------------- TMA producer: this CTA's half of the table columns of each task ----------------
      const uint64_t pol = l2_evict_last();
      const int64_t cpos = (int64_t)client * npos;
      int stage = 0, ts = 0;
      uint32_t phase = 0, tph = 0;
      for (int pos = pos0; pos < pos1; ++pos)
#pragma unroll 1
        for (int tt = 0; tt < 4; ++tt) {                  // (tile X, Y) x (task A, B)
          const int trow = (int)(((cpos + pos) * 2 + (tt & 1)) * 256) + (int)rank * kHalf;
#pragma unroll 1
          for (int kb = 0; kb < kKB; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (leader) mbar_expect_tx(&full[stage], 2 * kTile);
            tma_load_2d_pair(BS + stage * kTile, &mapT, mapa_shared(smem_u32(&full[stage]), 0),
                             kb * kBK, trow, pol);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          mbar_wait(&tlempty[ts], tph ^ 1);
          if (leader) mbar_expect_tx(&tlfull[ts], 2 * kTail);
          tma_load_2d_pair(BT + ts * kTail, &mapTail, mapa_shared(smem_u32(&tlfull[ts]), 0),
                           kKB * kBK, trow, pol);
          if (++ts == kTStages) {
            ts = 0;
            tph ^= 1;
          }
        }
    }
  } else if (warp == 9) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer: task A -> TMEM buffer 0, task B -> buffer 1, tiles alternating ----------------
      const uint32_t idesc = idesc_u8(2 * kRows, 256);
      int stage = 0, ts = 0;
      uint32_t phase = 0, tph = 0, xph = 0, eph = 0;
#ifdef ZPIR_TC_TRACE
      unsigned long long fwait = 0;   // cycles the MMA thread waited for table tiles this position
#endif
      for (int pos = pos0; pos < pos1; ++pos) {
        for (int tile = 0; tile < 2; ++tile) {
          const uint8_t* XA = XB + tile * kXBytes;
          const uint64_t xtd = desc_sw32(smem_u32(XA + kABytes));
          for (int task = 0; task < 2; ++task) {
            if (task == 0) mbar_wait(&xfull[tile], xph);
            // the buffer's previous drain: the other tile's, of this position (tile Y) or
            // the previous one (tile X)
            if (pos > pos0 || tile == 1)
              mbar_wait(&tempty[2 * (tile ^ 1) + task], tile ? eph : eph ^ 1);
            tc_fence_after();
            if (tile == 0) TC_STAMP(pos, 11 + task);
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
                umma_i8_pair(d, ad + 2 * k, bd + 2 * k, idesc, (kb == 0 && k == 0) ? 0u : 1u);
              umma_commit_pair(&empty[stage], 0x3);
              if (++stage == kStages) {
                stage = 0;
                phase ^= 1;
              }
            }
            mbar_wait(&tlfull[ts], tph);
            tc_fence_after();
            umma_i8_pair(d, xtd, desc_sw32(smem_u32(BT + ts * kTail)), idesc, 1u);
            umma_commit_pair(&tlempty[ts], 0x3);
            if (++ts == kTStages) {
              ts = 0;
              tph ^= 1;
            }
            umma_commit_pair(&tfull[2 * tile + task], 0x3);
          }
          if (tile == 0) TC_STAMP(pos, 13);
        }
        xph ^= 1;
        eph ^= 1;
        TC_STAMP(pos, 14);
#ifdef ZPIR_TC_TRACE
        if (blockIdx.x == 0 && blockIdx.y == 0 && pos - pos0 < 64) g_tc_trace[(pos - pos0) * 16 + 15] = fwait;
        fwait = 0;
#endif
      }
    }
  } else {
    // ---------------- epilogue: one row per thread (TMEM lane), warps 0-3 tile X, 4-7 tile Y ----------------
    const int tile = warp >> 2;
    const int quarter = warp & 3;
    const int t = quarter * 32 + lane;          // row within the tile = TMEM lane
    const int64_t row0 = ((int64_t)blockIdx.x * 2 + tile) * kRows;
    const int64_t r = row0 + t;
    const int64_t er = r < rows ? (rid ? (int64_t)rid[r] : r) : 0;
    const int nb = ds.nb;
    uint32_t* Bc = Ball + (int64_t)client * rows_p * nb * kXL;
    const uint32_t lanebase = tbase + ((uint32_t)(quarter * 32) << 16);
    uint8_t* XA = XB + tile * kXBytes;
    uint8_t* xa_row = XA + t * kBK;
    uint8_t* xt_row = XA + kABytes + t * kKT + (((t >> 2) & 1) << 4);   // chunk 0 of the tail row
    const uint32_t xfull_l = mapa_shared(smem_u32(&xfull[tile]), 0);
    const uint32_t tempty_a = mapa_shared(smem_u32(&tempty[2 * tile]), 0);
    const uint32_t tempty_b = mapa_shared(smem_u32(&tempty[2 * tile + 1]), 0);
    uint64_t* tfull_a = &tfull[2 * tile];
    uint64_t* tfull_b = &tfull[2 * tile + 1];
    auto digit_at = [&](int p) -> uint32_t {
      if (r >= rows || p >= pos1) return 0u;
      const int di = p / (int)n;
      return (E[er * rs + (p - (int64_t)di * n)] >> ds.off[di]) & ((1u << ds.width[di]) - 1u);
    };
    auto store8 = [&](uint32_t* dst, const uint32_t (&v)[8]) {
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(v[0]),
                   "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                   : "memory");
    };
    // X rows of the warp from their buckets, warp-cooperative async copies: eight
    // lanes per row, lane q of them moving the 16-byte chunk q of each of the
    // row's four 128-byte k-block segments into the SW128 A layout (whole
    // 128-byte lines in global memory, conflict-free in shared memory; zero fill
    // for digit 0), and lane 0 the tail chunk. A row with `fwd` set (digit
    // repeats) is copied by its own thread instead: the low half from the bucket
    // it has just stored, the high half straight from the drain of task B.
    const int gj = lane >> 3, gq = lane & 7;
    const uint4* wsrc = reinterpret_cast<const uint4*>(Bc + (row0 + quarter * 32) * nb * kXL) + gq;
    const uint32_t rstride = (uint32_t)nb * (kXL / 4);   // one row's buckets, in 16-byte units
    const uint32_t xa_w = smem_u32(XA) + (uint32_t)(quarter * 32) * kBK;
    const uint32_t xt_w = smem_u32(XA) + kABytes + (uint32_t)(quarter * 32) * kKT;
    auto gather_issue = [&](uint32_t dgv, uint32_t fwd, const uint32_t* own) {
      // bucket index | live (digit != 0) | forwarded, of this lane's row
      const uint32_t pk = (dgv ? dgv - 1u : 0u) | (dgv ? 0x100u : 0u) | (fwd ? 0x200u : 0u);
#pragma unroll 2
      for (int it = 0; it < 8; ++it) {
        const int i = 4 * it + gj;                         // row of the warp
        const uint32_t p_i = __shfl_sync(0xffffffffu, pk, i);
        if (p_i & 0x200u) continue;
        const uint4* src = wsrc + ((uint32_t)i * rstride + (p_i & 0xffu) * (kXL / 4));
        const uint32_t dst = xa_w + i * kBK + ((gq ^ (i & 7)) << 4);
        const uint32_t sz = (p_i >> 4) & 16u;
#pragma unroll
        for (int kb = 0; kb < kKB; ++kb)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + kb * (kRows * kBK)),
                       "l"(src + 8 * kb), "r"(sz)
                       : "memory");
        if (gq == 0)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                           xt_w + i * kKT + (((i >> 2) & 1) << 4)),
                       "l"(src + 32), "r"(sz)
                       : "memory");
      }
      if (fwd) {
#pragma unroll 4
        for (int cc = 0; cc < 16; ++cc)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           smem_u32(xa_row) + (cc >> 3) * (kRows * kBK) + (((cc & 7) ^ (t & 7)) << 4)),
                       "l"(own + 4 * cc)
                       : "memory");
      }
    };
    auto publish = [&]() {
      asm volatile("cp.async.wait_all;" ::: "memory");
      fence_async_smem();
      mbar_arrive_remote(xfull_l);
    };
    auto prefetch_bucket = [&](uint32_t d) {
      if (!d) return;
      const uint32_t* pb = Bc + (r * nb + d - 1) * kXL;
#pragma unroll
      for (int j = 0; j < 5; ++j) asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + 32 * j));
    };

    // prologue: X of the first position
    uint32_t dg = digit_at(pos0), dg_n = digit_at(pos0 + 1);
    gather_issue(dg, 0u, nullptr);
    publish();
    prefetch_bucket(dg_n);
    uint32_t fph = 0;
    for (int pos = pos0; pos < pos1; ++pos) {
      const bool last = pos + 1 >= pos1;
      const bool tr = threadIdx.x == 0;
      if (tr) TC_STAMP(pos, 0);
      uint32_t* brow = Bc + ((r * nb) + (dg ? dg - 1 : 0)) * kXL;
      // the next position's bucket is this position's (digit repeats): its X is
      // this position's output
      const uint32_t fwd = (!last && dg && dg_n == dg) ? 1u : 0u;
      uint32_t carry = 0;
      // ---- task A: limbs 0..63
      mbar_wait(tfull_a, fph);
      if (tr) TC_STAMP(pos, 1);
      tc_fence_after();
      drain256(lanebase, carry, [&](int g, const uint32_t (&v)[32]) {
        uint32_t pend[8];
        limbs8(v, carry, pend);
        if (dg) store8(brow + 8 * g, pend);
      });
      if (tr) TC_STAMP(pos, 2);
      tc_fence_before();
      mbar_arrive_remote(tempty_a);
      // ---- task B: limbs 64..127 and the carry out (limb 128). Once it is complete
      // no MMA reads X any more: forwarded rows go straight into X
      mbar_wait(tfull_b, fph);
      fph ^= 1;
      if (tr) TC_STAMP(pos, 5);
      tc_fence_after();
      drain256(lanebase + 256u, carry, [&](int g, const uint32_t (&v)[32]) {
        uint32_t pend[8];
        limbs8(v, carry, pend);
        if (dg) store8(brow + 64 + 8 * g, pend);
        if (fwd) {
          const int cc = 16 + 2 * g;
          *reinterpret_cast<uint4*>(xa_row + (cc >> 3) * (kRows * kBK) + (((cc & 7) ^ (t & 7)) << 4)) =
              make_uint4(pend[0], pend[1], pend[2], pend[3]);
          *reinterpret_cast<uint4*>(xa_row + (cc >> 3) * (kRows * kBK) + ((((cc + 1) & 7) ^ (t & 7)) << 4)) =
              make_uint4(pend[4], pend[5], pend[6], pend[7]);
        }
      });
      {
        // limb 128 and the row's zero padding as one whole 32-byte sector
        const uint32_t topv[8] = {carry, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        if (dg) store8(brow + kL, topv);
        if (fwd) *reinterpret_cast<uint4*>(xt_row) = make_uint4(carry, 0u, 0u, 0u);
      }
      if (tr) TC_STAMP(pos, 6);
      tc_fence_before();
      mbar_arrive_remote(tempty_b);
      if (!last) {
        // ---- the next position's gather; it lands under the other tile's MMAs
        __syncwarp();
        gather_issue(dg_n, fwd, brow);
        if (tr) TC_STAMP(pos, 4);
        publish();                              // xfull for the tile's next position
        if (tr) TC_STAMP(pos, 7);
        dg = dg_n;
        dg_n = digit_at(pos + 2);
        prefetch_bucket(dg_n);
      }
    }
  }
  tc_fence_before();
  cluster_sync();   // all MMAs consumed, all TMEM reads done in both CTAs
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc_pair(tbase, 512);
  }
}

// the IMAD kernel of the same contract (multiexp.cu)
int slot_fixed_launch(const uint32_t* P, int64_t n, const uint32_t* E, int64_t rs,
                      const int32_t* row_ids, int64_t rows, int limbs, const uint32_t* N,
                      uint32_t np, const uint32_t* one_m, uint32_t* W, cudaStream_t st);

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

// (rows x 544) u8 table matrix, boxes of 128 rows (one CTA's half of a task) x box_k K bytes.
static int table_map(CUtensorMap* map, const void* base, int64_t rows, int box_k,
                     CUtensorMapSwizzle sw) {
  auto fn = tcp_encode();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return kErrCuda;
  }
  cuuint64_t dims[2] = {(cuuint64_t)tcp::kTK, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)tcp::kTK};
  cuuint32_t box[2] = {(cuuint32_t)box_k, (cuuint32_t)tcp::kHalf};
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
  // measured optimum of D = 5..11: more digits mean more positions
  // but fewer buckets (IMAD combine; more of them found in L2)
  constexpr int D = 7;
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
  const int64_t rows_p = ceil_div(rows, 4 * kRows) * 4 * kRows;
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
                              const int32_t* rid, int64_t rows_all, cudaStream_t st) {
  using namespace tcp;
  // A CTA pair takes 512 rows. A short remainder (at most a quarter of a pair, next
  // to at least one full pair) goes to the IMAD kernel instead of a pair of its own:
  // 32823 rows are 64 pairs + 55 rows, and 16 clients x 128 CTAs are 13.8 waves of
  // 148 SMs where 16 x 130 are 14.05.
  const int64_t rem = rows_all % (4 * kRows);
  const bool tail = rows_all > 4 * kRows && rem > 0 && rem <= kRows && 4 * n <= 65536;
  const int64_t rows = tail ? rows_all - rem : rows_all;
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
  const int64_t ctas = 2 * ceil_div(rows, 4 * kRows);    // whole CTA pairs, two tiles per CTA
  const int64_t tiles = 2 * ctas;
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
  const int64_t ck = std::max<int64_t>(1, chunk / std::max<int64_t>(1, ceil_div(ctas * C, 148)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ctas, C);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int64_t p0 = 0; p0 < npos; p0 += ck) {
    const int64_t p1 = std::min<int64_t>(npos, p0 + ck);
    if (cudaLaunchKernelEx(&cfg, tc_step_kernel, mT, mTail, ds, E, rs, rid, n, npos, (int)p0,
                           (int)p1, rows, rows_p, Bk) != cudaSuccess)
      return fail("tc_step launch");
  }
  if (check_launch("tc_step")) return fail("tc_step launch");
  bucket_combine_kernel<<<dim3((unsigned)ceil_div(rows, 4), C), 128, 0, st>>>(dcl, Bk, nb, rows,
                                                                             rows_p, rid);
  if (check_launch("bucket_combine")) return fail("bucket_combine");
  release();
  if (tail)
    for (int c = 0; c < C; ++c) {
      // rows [rows, rows_all): by position in the row-id list, or by row
      const int e = rid ? slot_fixed_launch(P[c], n, E, rs, rid + rows, rem, kL, N[c], np[c],
                                            one_m[c], W[c], st)
                        : slot_fixed_launch(P[c], n, E + rows * rs, rs, nullptr, rem, kL, N[c], np[c],
                                            one_m[c], W[c] + rows * kL, st);
      if (e) return e;
    }
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
