// Small host helpers shared by the CUDA translation units.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "status.h"

namespace nif {

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

#ifdef __CUDACC__
// device-wide nanosecond clock (diagnostic timelines; comparable across SMs)
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

// Launch errors are reported synchronously (configuration errors); device
// faults surface at the caller's next synchronisation as usual.
inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(NIF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return NIF_OK;
}

}  // namespace nif
