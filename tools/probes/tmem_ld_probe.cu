// TMEM -> register load throughput probe (B200): W warps per CTA (one CTA per
// SM), each warp reads all 512 columns of its 32-lane quarter with
// tcgen05.ld.sync.aligned.32x32b.x{16,32,64}, DEPTH loads in flight before
// tcgen05.wait::ld. Prints bytes / cycle / SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_probe tools/probes/tmem_ld_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int X>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ld<16>(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
                 "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
}
template <>
__device__ __forceinline__ void ld<32>(uint32_t taddr, uint32_t* r) {
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

template <int X, int DEPTH>
__global__ void __launch_bounds__(256, 1) probe(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  const int nw = blockDim.x >> 5;
  const int half = warp >> 2;      // with 8 warps, two warps per quarter split the columns
  const int c0 = (nw > 4) ? half * 256 : 0, c1 = (nw > 4) ? c0 + 256 : 512;
  uint32_t acc = 0;
  uint32_t r[DEPTH][X];
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = c0; c < c1; c += X * DEPTH) {
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) ld<X>(base + c + X * d, r[d]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int d = 0; d < DEPTH; ++d)
#pragma unroll
        for (int i = 0; i < X; ++i) acc += r[d][i];
    }
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x9e3779b9u) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
  }
}

template <int X, int DEPTH>
void run(int threads, int iters) {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 4);
  probe<X, DEPTH><<<148, threads>>>(iters / 10 + 1, cyc, sink);
  probe<X, DEPTH><<<148, threads>>>(iters, cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += h[i];
  mean /= 148;
  const double bytes = (double)iters * 128 * 512 * 4;   // all 512 columns x 128 lanes per iter
  printf("x%-2d depth %d warps %d: %.1f B/cycle/SM (%s)\n", X, DEPTH, threads / 32, bytes / mean,
         cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  const int iters = 2000;
  run<16, 1>(128, iters);
  run<16, 4>(128, iters);
  run<32, 1>(128, iters);
  run<32, 2>(128, iters);
  run<32, 4>(128, iters);
  run<32, 2>(256, iters);
  run<16, 4>(256, iters);
  return 0;
}
