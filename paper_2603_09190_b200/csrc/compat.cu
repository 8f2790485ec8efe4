// Reference-API compatibility kernels (off the online hot path).
//
//   rns_residues   residues of the batch-scaled hint matrix modulo a prime
//                  basis -- the reference's H_rns = matrix_to_rns(basis,
//                  H_scaled) (rns.py:148-154, protocol.py:188), produced
//                  from the device H on demand (the answer path never needs
//                  it: it reads H in place). Entry (g, k) of the scaled
//                  matrix is sum_j 2^(32 stride j) S[g cap + j][k]; output
//                  (count, groups, n) float64, each residue < 2^27.
//   multiexp_opcount  the reference's group-multiplication count of each
//                  hint entry (paillier.py:134-193: w = 6-bit windows, w
//                  squarings between windows, bucket products, running-sum
//                  and window-total products), from the digits of the
//                  exponents read in place from H -- so counters report what
//                  the reference's own multiexp would have counted.
#include "zpir_common.cuh"

namespace zpir {

// grid (ceil(n / 128), groups), 128 threads, dynamic smem cap * 128 u32
__global__ void __launch_bounds__(128)
rns_residues_kernel(const uint32_t* __restrict__ S, int64_t rows, int64_t n, int cap, int stride,
                    const uint32_t* __restrict__ primes, const unsigned long long* __restrict__ w,
                    int count, int64_t groups, double* __restrict__ out) {
  extern __shared__ uint32_t sv[];   // [cap][128]
  const int64_t g = blockIdx.y;
  const int64_t k = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int64_t c0 = g * cap;
  const int nr = (int)((rows - c0) < cap ? (rows - c0) : cap);
  for (int j = 0; j < nr; ++j) sv[j * 128 + threadIdx.x] = (k < n) ? S[(c0 + j) * n + k] : 0u;
  if (k >= n) return;
  for (int i = 0; i < count; ++i) {
    const uint32_t p = primes[i];
    const unsigned long long* wi = w + (size_t)i * cap;
    unsigned long long acc = 0;
    for (int j = 0; j < nr; ++j) {
      acc += (unsigned long long)(sv[j * 128 + threadIdx.x] % p) * wi[j];
      if ((j & 511) == 511) acc %= p;     // < 2^54 per term: 512 terms stay below 2^63
    }
    out[((size_t)i * groups + g) * n + k] = (double)(acc % p);
  }
  (void)stride;
}

int rns_residues_launch(const uint32_t* S, int64_t rows, int64_t n, int cap, int stride,
                        const uint32_t* primes, const unsigned long long* w, int count,
                        int64_t groups, double* out, cudaStream_t st) {
  if (cap <= 0 || n <= 0 || count <= 0 || groups <= 0 || cap > 384) {
    set_error("rns_residues: bad shape (cap=%d n=%lld count=%d)", cap, (long long)n, count);
    return kErrInput;
  }
  const size_t smem = (size_t)cap * 128 * 4;
  cudaFuncSetAttribute(rns_residues_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  dim3 grid((unsigned)ceil_div(n, 128), (unsigned)groups);
  rns_residues_kernel<<<grid, 128, smem, st>>>(S, rows, n, cap, stride, primes, w, count, groups,
                                               out);
  return check_launch("rns_residues");
}

// bit `off` of exponent (g, k) = sum_j 2^(sbits j) S[g cap + j][k] (slot j holds
// a value below 2^min(sbits, 32): H < q <= gamma = 2^sbits)
__device__ __forceinline__ uint32_t exp_bit(const uint32_t* S, int64_t c0, int nr, int64_t n,
                                            int64_t k, int sbits, int off) {
  const int j = off / sbits, b = off - j * sbits;
  if (j >= nr || b >= 32) return 0u;
  return (S[(c0 + j) * n + k] >> b) & 1u;
}

// one CTA (256 threads) per group: the reference's multiexp op count for
// prod_k base_k^{E[g][k]}, E[g][k] = sum_j 2^(sbits j) S[g cap + j][k]
__global__ void __launch_bounds__(256)
multiexp_opcount_kernel(const uint32_t* __restrict__ S, int64_t rows, int64_t n, int cap,
                        int sbits, long long* __restrict__ out) {
  __shared__ int s_max;
  __shared__ unsigned s_mask[2];
  __shared__ int s_nnz, s_dmax;
  const int64_t g = blockIdx.x;
  const int64_t c0 = g * cap;
  const int nr = (int)((rows - c0) < cap ? (rows - c0) : cap);
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  int mb = 0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    for (int j = nr - 1; j >= 0; --j) {
      const uint32_t v = S[(c0 + j) * n + k];
      if (v) {
        mb = max(mb, sbits * j + 32 - __clz(v));
        break;
      }
    }
  }
  atomicMax(&s_max, mb);
  __syncthreads();
  const int maxbits = s_max;
  if (maxbits == 0) {
    if (threadIdx.x == 0) out[g] = 0;
    return;
  }
  const int w = maxbits > 6 ? 6 : maxbits;
  const int nwin = (maxbits + w - 1) / w;
  long long nmul = 0;
  bool acc_one = true;
  for (int win = nwin - 1; win >= 0; --win) {
    if (threadIdx.x == 0) {
      s_mask[0] = s_mask[1] = 0u;
      s_nnz = 0;
      s_dmax = 0;
    }
    __syncthreads();
    int nnz = 0, dmax = 0;
    unsigned m0 = 0, m1 = 0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
      unsigned d = 0;
      for (int i = 0; i < w; ++i) d |= exp_bit(S, c0, nr, n, k, sbits, win * w + i) << i;
      if (d) {
        ++nnz;
        dmax = max(dmax, (int)d);
        if (d < 32) m0 |= 1u << d; else m1 |= 1u << (d - 32);
      }
    }
    atomicAdd(&s_nnz, nnz);
    atomicMax(&s_dmax, dmax);
    if (m0) atomicOr(&s_mask[0], m0);
    if (m1) atomicOr(&s_mask[1], m1);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (!acc_one) nmul += w;                       // w squarings
      const int D = __popc(s_mask[0]) + __popc(s_mask[1]);
      if (D > 0) {
        nmul += (s_nnz - D)                          // bucket products
              + (D - 1)                              // running sum
              + (s_dmax - 1);                        // window total
        if (acc_one) acc_one = false; else nmul += 1;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[g] = nmul;
}

int multiexp_opcount_launch(const uint32_t* S, int64_t rows, int64_t n, int cap, int sbits,
                            int64_t groups, long long* out, cudaStream_t st) {
  if (cap <= 0 || n <= 0 || sbits < 1 || groups <= 0) {
    set_error("multiexp_opcount: bad shape");
    return kErrInput;
  }
  multiexp_opcount_kernel<<<(unsigned)groups, 256, 0, st>>>(S, rows, n, cap, sbits, out);
  return check_launch("multiexp_opcount");
}

}  // namespace zpir
