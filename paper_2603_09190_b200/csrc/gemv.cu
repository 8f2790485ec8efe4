// Online answer, first matrix product: b = DB * qu mod 2^32 (u8 x u32).
//
// Reference: ServerGlobalState.db_matvec (protocol.py:242-257), which runs an
// exact centered float64 BLAS GEMV over an 8-byte-per-element copy of db^T.
// Here DB = db^T is held once as u8 (rows = d1 padded to 128, ld = d0 padded
// to 64) and streamed from HBM exactly once per query.
//
// Arithmetic: qu is split into four byte planes qu = sum_l 2^(8l) qu_l, so
//   b[c] = sum_l 2^(8l) * (sum_i DB[c,i] * qu_l[i])  (mod 2^32)
// and each inner sum is a chain of IDP4A (4 x u8*u8 + u32) instructions on
// 32-bit words of DB and of the packed planes: one instruction per DB byte,
// no byte unpacking. Wrapping u32 accumulation is exact mod 2^32.
//
// Work split: a warp owns R consecutive rows over one K-chunk; lanes read 16
// contiguous bytes per row per step (coalesced 128-bit loads, R loads in
// flight), the query planes come from L1/L2 (they are re-read by every row
// group, 4*d0 bytes, L2-resident). Partial row sums are warp-reduced and
// atomically added (wrapping add commutes, so the split-K is exact).
#include "zpir_common.cuh"

namespace zpir {

// qp[l * (ld/4) + w] = byte l of qu[4w], qu[4w+1], qu[4w+2], qu[4w+3]
__global__ void qplanes_kernel(const uint32_t* __restrict__ qu, int64_t words,
                               int64_t nvec, uint32_t* __restrict__ qp) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= words) return;
  for (int64_t v = 0; v < nvec; ++v) {
    const uint4 x = reinterpret_cast<const uint4*>(qu + v * words * 4)[w];
    uint32_t* dst = qp + v * 4 * words;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const uint32_t sel = (uint32_t)l | ((uint32_t)(l + 4) << 4);
      const uint32_t lo = __byte_perm(x.x, x.y, sel);  // [x.b_l, y.b_l, ...]
      const uint32_t hi = __byte_perm(x.z, x.w, sel);
      dst[l * words + w] = __byte_perm(lo, hi, 0x5410);
    }
  }
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int R>
__global__ void __launch_bounds__(256)
gemv_dp4a_kernel(const uint8_t* __restrict__ dbt, int64_t rows, int64_t ld,
                 const uint32_t* __restrict__ qp, uint32_t* __restrict__ out,
                 int64_t kchunk, int64_t nkc) {
  const int lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nrg = rows / R;
  const int64_t kc = item / nrg;
  const int64_t rg = item - kc * nrg;
  if (kc >= nkc) return;
  const int64_t k0 = kc * kchunk;
  const int64_t k1 = min(k0 + kchunk, ld);
  const int64_t words = ld >> 2;
  const uint8_t* base = dbt + rg * R * ld;

  uint32_t acc[R][4];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int l = 0; l < 4; ++l) acc[r][l] = 0;

#pragma unroll 2
  for (int64_t k = k0 + lane * 16; k < k1; k += 512) {
    uint4 d[R];
#pragma unroll
    for (int r = 0; r < R; ++r) d[r] = ldg_stream(base + r * ld + k);
    uint4 q[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) q[l] = __ldg(reinterpret_cast<const uint4*>(qp + l * words + (k >> 2)));
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        acc[r][l] = __dp4a(d[r].x, q[l].x, acc[r][l]);
        acc[r][l] = __dp4a(d[r].y, q[l].y, acc[r][l]);
        acc[r][l] = __dp4a(d[r].z, q[l].z, acc[r][l]);
        acc[r][l] = __dp4a(d[r].w, q[l].w, acc[r][l]);
      }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    uint32_t v = acc[r][0] + (acc[r][1] << 8) + (acc[r][2] << 16) + (acc[r][3] << 24);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(ZPIR_FULL, v, o);
    if (lane == 0) atomicAdd(out + rg * R + r, v);
  }
}

__global__ void mask_kernel(uint32_t* x, int64_t count, uint32_t mask) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) x[i] &= mask;
}

// planes (prow x ld bytes): rows 4v+l = byte plane l of query v, zero rows
// 4*nvec .. prow-1 (the B operand of the tcgen05 GEMV).
int query_planes_launch(const uint32_t* qu, int64_t ld, int64_t nvec, uint8_t* planes,
                        int64_t prow, cudaStream_t st) {
  if (ld % 64 || prow < 4 * nvec) {
    set_error("query_planes: ld %% 64 and prow >= 4 nvec required");
    return kErrInput;
  }
  const int64_t words = ld / 4;
  if (prow > 4 * nvec &&
      cudaMemsetAsync(planes + 4 * nvec * ld, 0, (prow - 4 * nvec) * ld, st) != cudaSuccess)
    return check_launch("query_planes memset");
  qplanes_kernel<<<(unsigned)ceil_div(words, 256), 256, 0, st>>>(
      qu, words, nvec, reinterpret_cast<uint32_t*>(planes));
  return check_launch("query_planes");
}

int gemv_launch(const uint8_t* dbt, int64_t rows, int64_t ld, const uint32_t* qu, int64_t nvec,
                uint32_t* out, uint32_t qmask, uint32_t* qp, cudaStream_t st) {
  constexpr int R = 8;
  if (rows <= 0 || ld <= 0 || rows % 128 || ld % 64 || nvec <= 0) {
    set_error("gemv: rows must be a positive multiple of 128 and ld of 64 (rows=%lld ld=%lld)",
              (long long)rows, (long long)ld);
    return kErrInput;
  }
  const int64_t words = ld / 4;
  qplanes_kernel<<<(unsigned)ceil_div(words, 256), 256, 0, st>>>(qu, words, nvec, qp);
  if (int e = check_launch("qplanes")) return e;
  const int64_t kchunk = 8192;
  const int64_t nkc = ceil_div(ld, kchunk);
  const int64_t items = (rows / R) * nkc;
  for (int64_t v = 0; v < nvec; ++v) {
    if (cudaMemsetAsync(out + v * rows, 0, rows * sizeof(uint32_t), st) != cudaSuccess)
      return check_launch("gemv memset");
    gemv_dp4a_kernel<R><<<(unsigned)ceil_div(items, 8), 256, 0, st>>>(
        dbt, rows, ld, qp + v * 4 * words, out + v * rows, kchunk, nkc);
    if (int e = check_launch("gemv")) return e;
    if (qmask != 0xffffffffu) {
      mask_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(out + v * rows, rows, qmask);
      if (int e = check_launch("gemv mask")) return e;
    }
  }
  return kOk;
}

}  // namespace zpir
