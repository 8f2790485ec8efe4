// Shared helpers for the ZipPIR B200 server-path kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define ZPIR_FULL 0xffffffffu

namespace zpir {

// Status codes returned by every extern "C" entry point (include/zippir_b200.h).
enum Status : int {
  kOk = 0,
  kErrInput = 1,      // maps to Python ValueError (reference: protocol.py:166-169, :337-338)
  kErrCuda = 2,       // CUDA runtime failure (launch, memory, device)
  kErrUnsupported = 3 // shape / limb width outside what the kernels are built for
};

void set_error(const char* fmt, ...);

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return kErrCuda;
  }
  return kOk;
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace zpir
