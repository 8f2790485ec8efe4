// Microbenchmarks for the roofline denominators MEASURED_PEAKS.json lacks:
// the IMAD throughput the bignum kernels are bound by (32-bit IMAD.LO/HI as
// emitted by the CIOS loop), measured on the device with CUDA events.
#include "zpir_common.cuh"

namespace zpir {

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
