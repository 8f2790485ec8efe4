// 30-bit digit <-> 32-bit limb regrouping on the device, so the host side of
// the API boundary is a memcpy of CPython's int digits (csrc/pyconv.c) instead
// of a per-int conversion loop (1024 x 2048-bit ck_o per query, 521 results).
#include "zpir_common.cuh"

namespace zpir {

// limbs[i][l] = bits [32 l, 32 l + 32) of the integer with 30-bit digits digits[i][*]
__global__ void digits_to_limbs_kernel(const uint32_t* __restrict__ digits, int64_t count,
                                       int ndig, uint32_t* __restrict__ limbs, int nl) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count * nl) return;
  const int64_t i = idx / nl;
  const int l = (int)(idx - i * nl);
  const uint32_t* d = digits + i * ndig;
  const int bit = 32 * l;
  const int d0 = bit / 30, off = bit - 30 * d0;
  uint64_t acc = 0;
  int have = 0;
  for (int q = d0; q < ndig && have - off < 32; ++q) {
    acc |= (uint64_t)d[q] << have;
    have += 30;
  }
  limbs[idx] = (uint32_t)(acc >> off);
}

// digits[i][q] = bits [30 q, 30 q + 30) of the integer with 32-bit limbs limbs[i][*]
__global__ void limbs_to_digits_kernel(const uint32_t* __restrict__ limbs, int64_t count, int nl,
                                       int64_t ld, uint32_t* __restrict__ digits, int ndig) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count * ndig) return;
  const int64_t i = idx / ndig;
  const int q = (int)(idx - i * ndig);
  const uint32_t* x = limbs + i * ld;
  const int bit = 30 * q;
  const int l0 = bit / 32, off = bit - 32 * l0;
  uint64_t acc = 0;
  if (l0 < nl) acc = x[l0];
  if (l0 + 1 < nl) acc |= (uint64_t)x[l0 + 1] << 32;
  digits[idx] = (uint32_t)(acc >> off) & 0x3fffffffu;
}

int digits_to_limbs_launch(const uint32_t* digits, int64_t count, int ndig, uint32_t* limbs, int nl,
                           cudaStream_t st) {
  if (count <= 0 || ndig <= 0 || nl <= 0) {
    set_error("digits_to_limbs: bad shape");
    return kErrInput;
  }
  const int64_t total = count * nl;
  digits_to_limbs_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, st>>>(digits, count, ndig,
                                                                          limbs, nl);
  return check_launch("digits_to_limbs");
}

int limbs_to_digits_launch(const uint32_t* limbs, int64_t count, int nl, int64_t ld,
                           uint32_t* digits, int ndig, cudaStream_t st) {
  if (count <= 0 || ndig <= 0 || nl <= 0 || ld < nl) {
    set_error("limbs_to_digits: bad shape");
    return kErrInput;
  }
  const int64_t total = count * ndig;
  limbs_to_digits_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, st>>>(limbs, count, nl, ld,
                                                                          digits, ndig);
  return check_launch("limbs_to_digits");
}

}  // namespace zpir
