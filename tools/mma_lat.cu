// Microbenchmark: tcgen05.mma (kind::f16, M=128) issue -> commit ->
// mbarrier round-trip latency vs N, K steps, operand source (SS / TS) and
// CTAs resident per SM. Thread 0 of every CTA issues `steps` MMAs of
// K=16, commits, waits, and records clock64 deltas.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2306_07191_b200/csrc \
//        -I../include mma_lat.cu -o mma_lat
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "tc.cuh"

using namespace nif;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc));
}

__global__ void lat_kernel(int N, int steps, int iters, int ts, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  if (tid < 32) tc::tmem_alloc<256>(&tslot);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tb = tslot;
  const uint32_t sa = tc::smem_u32(smem);
  const uint32_t idesc = tc::idesc_f16(N);
  uint32_t phase = 0;
  for (int it = 0; it < iters; ++it) {
    long long t0 = clock64();
    if (tid == 0) {
      tc::fence_after_sync();
      for (int s = 0; s < steps; ++s) {
        const uint64_t bd = tc::smem_desc(sa + 8192 + s * 256, 128, 1024);
        if (ts)
          mma_ts(tb, tb + 128 + s * 8, bd, idesc, s > 0);
        else
          tc::mma_f16(tb, tc::smem_desc(sa + s * 256, 128, 1024), bd, idesc, s > 0);
      }
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    long long t1 = clock64();
    if (tid == 0) out[(size_t)blockIdx.x * iters + it] = t1 - t0;
    tc::fence_before_sync();
    __syncthreads();
  }
  __syncthreads();
  if (tid < 32) tc::tmem_dealloc(tb, 256);
}

int main() {
  int sms = 148;
  const int iters = 64;
  printf("mode   N  steps  ctas/SM  median_cycles  p90\n");
  for (int ts = 0; ts < 2; ++ts)
    for (int N : {16, 48, 64, 128})
      for (int steps : {1, 4})
        for (int per_sm : {1, 2, 4}) {
          const int grid = sms * per_sm;
          const size_t smem_bytes = 200 * 1024 / per_sm;  // force per_sm CTAs per SM
          cudaFuncSetAttribute(lat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem_bytes);
          long long* d;
          cudaMalloc(&d, sizeof(long long) * grid * iters);
          lat_kernel<<<grid, 128, smem_bytes>>>(N, steps, iters, ts, d);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
          }
          std::vector<long long> h((size_t)grid * iters);
          cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
          cudaFree(d);
          std::vector<long long> v;
          for (int b = 0; b < grid; ++b)
            for (int i = 8; i < iters; ++i) v.push_back(h[(size_t)b * iters + i]);
          std::sort(v.begin(), v.end());
          printf("%s %4d %5d %7d %12lld %8lld\n", ts ? "TS" : "SS", N, steps, per_sm,
                 v[v.size() / 2], v[v.size() * 9 / 10]);
        }
  return 0;
}
