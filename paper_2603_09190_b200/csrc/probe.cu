// Microbenchmarks for the roofline denominators MEASURED_PEAKS.json lacks:
// the IMAD throughput the bignum kernels are bound by (32-bit IMAD.LO/HI as
// emitted by the CIOS loop), measured on the device with CUDA events.
#include "umma.cuh"

namespace zpir {
using namespace sm100;

// tcgen05 kind::i8 throughput: each CTA (one per SM) issues `iters` rounds of
// 4 MMAs (M = 128, N = n, K = 32 bytes) from one resident smem stage into
// TMEM (NACC independent accumulators, MMA k of a round -> accumulator k % NACC),
// committing to an mbarrier every 8 rounds so the queue stays bounded.
// Descriptors are hoisted: the loop body is the bare issue sequence.
// ops = blocks * iters * 4 * 2 * 128 * n * 32.
template <int NACC>
__global__ void __launch_bounds__(128, 1) umma_probe_kernel(int iters, int n) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * 128;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + 256 * 128);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x9E3779B9u * (i + 1) ^ blockIdx.x;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = *tslot;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    const uint32_t idesc = idesc_u8(128, n);
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ad[k] = desc_sw128(a0 + k * 32);
      bd[k] = desc_sw128(b0 + k * 32);
    }
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        umma_i8(d + (uint32_t)((k % NACC) * n), ad[k], bd[k], idesc, 1u);
      if ((it & 7) == 7 || it == iters - 1) {
        umma_commit(bar);
        mbar_wait(bar, phase);
        phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(d, 512);
  }
}

int umma_probe(int blocks, int iters, int n, float* ms) {
  const int nacc = n >= 1000 ? n / 1000 : 1;  // n = nacc * 1000 + N selects accumulators
  n %= 1000;
  if (n < 16 || n > 256 || n % 16 || nacc * n > 512 || (nacc != 1 && nacc != 2 && nacc != 4)) {
    set_error("umma_probe: n multiple of 16 in [16, 256], nacc in {1,2,4}, nacc * n <= 512");
    return kErrInput;
  }
  const int smem = (128 + 256) * 128 + 1024 + 64;
  auto kern = nacc == 1 ? umma_probe_kernel<1> : nacc == 2 ? umma_probe_kernel<2>
                                                           : umma_probe_kernel<4>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, 128, smem>>>(iters / 10 + 1, n);  // warm-up
  cudaEventRecord(e0);
  kern<<<blocks, 128, smem>>>(iters, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return check_launch("umma_probe");
}

// 8 independent mad.lo/mad.hi chains per thread; one "op" = one 32x32 multiply-add.
__global__ void __launch_bounds__(256) imad_probe_kernel(uint32_t* out, int iters, uint32_t seed) {
  uint32_t a[8], c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = seed * (threadIdx.x + 1) + i;
    c[i] = i ^ blockIdx.x;
  }
  const uint32_t b = seed | 1;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(c[i]) : "r"(a[i]), "r"(b));
      asm volatile("mad.hi.u32 %0, %1, %2, %0;" : "+r"(a[i]) : "r"(c[i]), "r"(b));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i] ^ c[i];
  if (s == 0x12345678u) out[0] = s;
}

// returns ms for `iters` iterations on blocks x 256 threads; ops = blocks*256*iters*16
int imad_probe(int blocks, int iters, float* ms) {
  uint32_t* out = nullptr;
  if (cudaMalloc(&out, 4) != cudaSuccess) return check_launch("probe malloc");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  imad_probe_kernel<<<blocks, 256>>>(out, iters / 10 + 1, 3u);  // warm-up
  cudaEventRecord(e0);
  imad_probe_kernel<<<blocks, 256>>>(out, iters, 7u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return check_launch("imad_probe");
}

}  // namespace zpir
