// Host staging bandwidth probe (GPU box): pageable -> pinned copy with T
// threads (plain memcpy vs AVX2 streaming stores), pinned -> device DMA
// alone, and both at once -- is the drop-in e2e path bound by host DRAM?
//   nvcc -O2 -Xcompiler -mavx2 -o /tmp/staging_bw tools/staging_bw.cu && /tmp/staging_bw
#include <cuda_runtime.h>
#include <immintrin.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static void copy_nt(uint8_t* dst, const uint8_t* src, size_t n) {
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    __m256i a = _mm256_loadu_si256((const __m256i*)(src + i));
    __m256i b = _mm256_loadu_si256((const __m256i*)(src + i + 32));
    __m256i c = _mm256_loadu_si256((const __m256i*)(src + i + 64));
    __m256i d = _mm256_loadu_si256((const __m256i*)(src + i + 96));
    _mm256_stream_si256((__m256i*)(dst + i), a);
    _mm256_stream_si256((__m256i*)(dst + i + 32), b);
    _mm256_stream_si256((__m256i*)(dst + i + 64), c);
    _mm256_stream_si256((__m256i*)(dst + i + 96), d);
  }
  std::memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static double par_copy(uint8_t* dst, const uint8_t* src, size_t n, int T, bool nt) {
  double t0 = now();
  std::vector<std::thread> th;
  size_t per = (n / T + 4095) / 4096 * 4096;
  for (int i = 0; i < T; ++i) {
    size_t a = i * per, b = std::min(n, a + per);
    if (a >= b) break;
    th.emplace_back([=] { nt ? copy_nt(dst + a, src + a, b - a) : (void)std::memcpy(dst + a, src + a, b - a); });
  }
  for (auto& t : th) t.join();
  return n / (now() - t0) / 1e9;
}

int main() {
  const size_t n = 73289328;
  std::vector<uint8_t> src(n, 1);
  uint8_t *pin, *pin2, *dev;
  cudaHostAlloc((void**)&pin, n, 0);
  cudaHostAlloc((void**)&pin2, n, 0);
  cudaMalloc((void**)&dev, n);
  std::memset(pin, 0, n);
  std::memset(pin2, 0, n);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int T : {1, 2, 4, 8, 12, 16})
    for (int nt : {0, 1}) {
      double best = 0;
      for (int r = 0; r < 5; ++r) best = std::max(best, par_copy(pin, src.data(), n, T, nt));
      printf("{\"copy\": \"%s\", \"threads\": %d, \"gbs\": %.1f}\n", nt ? "nt" : "memcpy", T, best);
    }
  auto dma = [&](uint8_t* p) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    cudaMemcpyAsync(dev, p, n, cudaMemcpyHostToDevice, s);
    cudaEventRecord(b, s);
    return std::make_pair(a, b);
  };
  for (int r = 0; r < 3; ++r) {
    auto ev = dma(pin2);
    cudaEventSynchronize(ev.second);
    float ms;
    cudaEventElapsedTime(&ms, ev.first, ev.second);
    printf("{\"dma_alone_gbs\": %.1f}\n", n / (ms * 1e-3) / 1e9);
  }
  for (int T : {4, 8, 16}) {
    auto ev = dma(pin2);
    double g = par_copy(pin, src.data(), n, T, true);
    cudaEventSynchronize(ev.second);
    float ms;
    cudaEventElapsedTime(&ms, ev.first, ev.second);
    printf("{\"concurrent_threads\": %d, \"copy_gbs\": %.1f, \"dma_gbs\": %.1f}\n", T, g, n / (ms * 1e-3) / 1e9);
  }
  return 0;
}
