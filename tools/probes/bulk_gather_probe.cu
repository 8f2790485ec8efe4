// Gather throughput probe (B200): every CTA (one per SM) gathers ROWS scattered
// 544-byte rows of a large global array into shared memory per iteration, either
// with cp.async (16-byte chunks, eight lanes per row: the tc_step gather) or with
// cp.async.bulk (four 128-byte copies and one 32-byte copy per row, one thread per
// row, mbarrier complete_tx). Prints cycles per iteration and bytes / cycle / SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bulk_probe tools/probes/bulk_gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int ROWS = 128, ROWB = 544;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) probe(const uint8_t* __restrict__ src, int64_t nrows,
                                                int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(128));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t ph = 0;
  uint64_t seed = 0x9e3779b97f4a7c15ull * (blockIdx.x * 131 + t + 1);
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    seed = seed * 6364136223846793005ull + 1442695040888963407ull;
    const int64_t row = (int64_t)((seed >> 20) % (uint64_t)nrows);   // this thread's row
    if (MODE == 0) {
      // cp.async: lanes 8j..8j+7 move row 4 it2 + j of the warp's 32 rows
      for (int it2 = 0; it2 < 8; ++it2) {
        const int i = 4 * it2 + (lane >> 3);
        const int64_t r = __shfl_sync(0xffffffffu, row, i);
        const uint8_t* s = src + r * ROWB + (lane & 7) * 16;
        const uint32_t d = smem_u32(sm) + (warp * 32 + i) * 128 + (lane & 7) * 16;
#pragma unroll
        for (int kb = 0; kb < 4; ++kb)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + kb * 16384), "l"(s + 128 * kb)
                       : "memory");
        if ((lane & 7) == 0)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           smem_u32(sm) + 65536 + (warp * 32 + i) * 32),
                       "l"(s + 512)
                       : "memory");
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
    } else {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(ROWB)
                   : "memory");
      const uint8_t* s = src + row * ROWB;
#pragma unroll
      for (int kb = 0; kb < 4; ++kb)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];" ::"r"(
                smem_u32(sm) + kb * 16384 + t * 128),
            "l"(s + 128 * kb), "r"(smem_u32(&bar))
            : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32, [%2];" ::"r"(
              smem_u32(sm) + 65536 + t * 32),
          "l"(s + 512), "r"(smem_u32(&bar))
          : "memory");
      uint32_t ok = 0;
      while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(&bar)), "r"(ph)
            : "memory");
      ph ^= 1;
    }
  }
  const unsigned long long t1 = clock64();
  if (t == 0) cyc[blockIdx.x] = t1 - t0;
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // rows of the source array: 4 M = 2.3 GB (far beyond L2) by default; e.g. 100000 = 54 MB stays in L2
  const int64_t nrows = argc > 1 ? atoll(argv[1]) : (4 << 20);
  uint8_t* src;
  unsigned long long* cyc;
  cudaMalloc(&src, nrows * ROWB);
  cudaMemset(src, 1, nrows * ROWB);
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  const int smem = 65536 + 4096 + 1024;
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) probe<0><<<sms, 128, smem>>>(src, nrows, iters, cyc);
      else probe<1><<<sms, 128, smem>>>(src, nrows, iters, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    }
    unsigned long long h[256];
    cudaMemcpy(h, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += (double)h[i];
    avg /= sms * (double)iters;
    printf("%s: %.0f cycles per %d-row gather, %.1f B/clk/SM (%.0f MB of rows, %d SMs)\n",
           mode == 0 ? "cp.async 16 B x 8 lanes per row" : "cp.async.bulk 4 x 128 B + 32 B per row",
           avg, ROWS, ROWS * ROWB / avg, nrows * ROWB / 1e6, sms);
  }
  return 0;
}
