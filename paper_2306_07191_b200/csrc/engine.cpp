// Native visibility engine: the whole split pass behind one C-ABI object
// (SURVEY.md §8b "nif_occluded (fused whole path)"), for FFI callers that
// hold rays in (pageable) host memory -- the drop-in for
// PredictorBackend.occluded (renderer.py:675-683) / NifBackend
// (nif.py:486-499) from a ctypes stub.
//
// The engine owns every device buffer of the pass for a fixed ray capacity:
// rays, the gather's record queues and workspace, the per-ray answer and,
// for per_object models, the bucketing scratch of each family -- plus a
// ring of pinned host staging slots. One call streams the caller's rays
// through the ring in chunks:
//
//   host threads: memcpy chunk k (pageable -> pinned slot k % S)
//   copy stream : H2D of slot k                      (overlaps chunk k-1's pass)
//   main stream : gather -> outer || inner query of chunk k
//   d2h stream  : the chunk's answer bytes -> pinned out slot -> caller
//
// so the PCIe upload, the staging memcpy (spread over a small pool of host
// threads) and the device pass of neighbouring chunks all overlap.
//
// Record queues hold `slots_per_ray` records per ray of a chunk (a bound, not
// the worst case n_obj): the gather never writes past it and always reports
// the true totals, so a chunk that overflowed is detected from its counts
// and re-run after the queues grow.
//
// Scene and model stay owned by the caller (views of device memory). After
// an optimiser step, repack (nif_fast_pack_dev) and call
// nif_engine_update_model with the stream the pack was enqueued on: the
// engine's streams wait for it before the next query.
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "kernels.h"
#include "nif_b200.h"
#include "status.h"

namespace {

// A few persistent host threads for the pageable <-> pinned staging copies.
class CopyPool {
 public:
  explicit CopyPool(int n) {
    for (int i = 0; i < n; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    stop_flag_.store(true);
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  int size() const { return (int)threads_.size() + 1; }
  // runs fn(i) for i in [0, parts) on the pool plus the calling thread
  void run(int parts, const std::function<void(int)>& fn) {
    if (threads_.empty() || parts <= 1) {
      for (int i = 0; i < parts; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_ = &fn;
      next_ = 0;
      parts_ = parts;
      pending_ = parts;
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      int i;
      const std::function<void(int)>* fn;
      {
        std::lock_guard<std::mutex> g(mu_);
        if (fn_ == nullptr || next_ >= parts_) return;
        i = next_++;
        fn = fn_;
      }
      (*fn)(i);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      // spin briefly before sleeping: staging jobs arrive every ~0.2 ms
      // within a call and calls come back to back, so a condvar wake-up
      // (tens of us) would otherwise sit in front of every chunk
      const auto t0 = std::chrono::steady_clock::now();
      while (gen_.load(std::memory_order_acquire) == seen && !stop_flag_.load() &&
             std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(kSpinUs))
        _mm_pause();
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || gen_.load() != seen; });
        if (stop_) return;
        seen = gen_.load();
      }
      work();
    }
  }
  static constexpr int kSpinUs = 300;
  std::atomic<bool> stop_flag_{false};
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int next_ = 0, parts_ = 0, pending_ = 0;
  std::atomic<uint64_t> gen_{0};
  bool stop_ = false;
};

// One persistent thread that runs a job (the staging loop of one call) while
// the calling thread issues uploads and launches: the staging copy of chunk
// k+1 proceeds while chunk k's launches are being enqueued.
class Stager {
 public:
  Stager() : t_([this] { loop(); }) {}
  ~Stager() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    t_.join();
  }
  void start(std::function<void()> job) {
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = std::move(job);
      busy_ = true;
    }
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [this] { return !busy_; });
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [this] { return stop_ || (busy_ && job_); });
        if (stop_) return;
        job = std::move(job_);
        job_ = nullptr;
      }
      job();
      {
        std::lock_guard<std::mutex> g(mu_);
        busy_ = false;
      }
      done_cv_.notify_all();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::function<void()> job_;
  bool busy_ = false, stop_ = false;
  std::thread t_;
};

// spin (then yield) until counter >= target or abort is set
inline bool wait_counter(const std::atomic<int>& counter, int target,
                         const std::atomic<bool>& abort) {
  for (int spins = 0; counter.load(std::memory_order_acquire) < target; ++spins) {
    if (abort.load(std::memory_order_relaxed)) return false;
    if (spins < 4096) _mm_pause();
    else std::this_thread::yield();
  }
  return true;
}

// Pageable -> pinned copy with non-temporal (streaming) stores: the pinned
// slot is read next by the DMA engine, not by this core, so write-allocate
// reads of the destination lines would only add host-DRAM traffic (which
// the staging copy shares with the upload itself).
__attribute__((target("avx2"))) void copy_nt_avx2(uint8_t* dst, const uint8_t* src, size_t n) {
  size_t head = (32 - ((uintptr_t)dst & 31)) & 31;
  if (head > n) head = n;
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256((const __m256i*)(src + i));
    const __m256i b = _mm256_loadu_si256((const __m256i*)(src + i + 32));
    const __m256i c = _mm256_loadu_si256((const __m256i*)(src + i + 64));
    const __m256i d = _mm256_loadu_si256((const __m256i*)(src + i + 96));
    _mm256_stream_si256((__m256i*)(dst + i), a);
    _mm256_stream_si256((__m256i*)(dst + i + 32), b);
    _mm256_stream_si256((__m256i*)(dst + i + 64), c);
    _mm256_stream_si256((__m256i*)(dst + i + 96), d);
  }
  std::memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}

bool use_nt_copy() {
  static const bool v = [] {
    const char* e = std::getenv("NIF_STAGING_NT");
    if (e != nullptr && e[0] == '0') return false;
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx2") != 0;
  }();
  return v;
}

void stage_copy(void* dst, const void* src, size_t n) {
  if (use_nt_copy()) copy_nt_avx2((uint8_t*)dst, (const uint8_t*)src, n);
  else std::memcpy(dst, src, n);
}

constexpr int kMaxSlots = 16;  // staging ring depth bound (NIF_STAGING_SLOTS)
constexpr int kDefaultSlots = 3;
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e != nullptr && std::atoi(e) > 0 ? std::atoi(e) : dflt;
}
int64_t chunk_rays_default() {  // default chunk: 256K rays, 14.7 MB in (NIF_STAGING_CHUNK)
  const char* e = std::getenv("NIF_STAGING_CHUNK");
  return e != nullptr && std::atoll(e) > 0 ? std::atoll(e) : (int64_t)1 << 18;
}
constexpr int kMaxChunks = 4096;

}  // namespace

struct nif_engine {
  nif_scene_view scene;
  nif_family_view outer, inner;
  const uint8_t* route;  // device
  int64_t capacity = 0;  // rays
  int n_net = 0;
  int64_t chunk_cap = 0;       // rays per chunk (staging slot size)
  int64_t slots_per_ray = 0;   // record slots per ray of a chunk, per queue
  int64_t qcap = 0;            // record slots per queue = chunk_cap * slots_per_ray
  double* org = nullptr;
  double* dir = nullptr;
  double* tms = nullptr;
  uint8_t* occ = nullptr;  // per-ray answer (the gather seeds it with bvh_occ)
  void* queues = nullptr;
  void* workspace = nullptr;
  size_t ws_bytes = 0;
  void* bucket[2] = {nullptr, nullptr};
  int64_t* counts = nullptr;     // device [4]
  nif_gather_out out{};
  // pinned staging ring
  int slots = 0;                     // staging ring depth
  bool ramp = true;                  // geometric first chunks
  uint8_t* pin_in[kMaxSlots] = {};   // chunk_cap * 56 B: o | d | t
  uint8_t* pin_out[kMaxSlots] = {};  // chunk_cap B
  int64_t* pin_counts = nullptr;  // [kMaxChunks][4] per-chunk record totals
  cudaEvent_t ev_in[kMaxSlots] = {};    // H2D of the slot done (slot reusable)
  cudaEvent_t ev_out[kMaxSlots] = {};   // D2H into the out slot done
  cudaEvent_t ev_pass[kMaxSlots] = {};  // pass of the slot's chunk done (main)
  cudaStream_t main = nullptr, side = nullptr, copy = nullptr, d2h = nullptr;
  cudaEvent_t ev_side = nullptr, ev_join = nullptr, ev_model = nullptr;
  CopyPool* pool = nullptr;
  Stager* stager = nullptr;
  int64_t overflow_reruns = 0;
};

namespace {

template <typename T>
int dev_alloc(T** p, size_t bytes) {
  if (cudaMalloc((void**)p, bytes > 0 ? bytes : 1) != cudaSuccess)
    return nif::fail(NIF_ERR_CUDA, "engine: cudaMalloc of %zu bytes failed", bytes);
  return NIF_OK;
}

void free_queues(nif_engine* e) {
  for (void** p : {&e->queues, &e->bucket[0], &e->bucket[1]})
    if (*p) {
      cudaFree(*p);
      *p = nullptr;
    }
}

void release(nif_engine* e) {
  free_queues(e);
  for (void* p : {(void*)e->org, (void*)e->dir, (void*)e->tms, (void*)e->occ, e->workspace,
                  (void*)e->counts})
    if (p) cudaFree(p);
  for (int s = 0; s < kMaxSlots; ++s) {
    if (e->pin_in[s]) cudaFreeHost(e->pin_in[s]);
    if (e->pin_out[s]) cudaFreeHost(e->pin_out[s]);
    for (cudaEvent_t ev : {e->ev_in[s], e->ev_out[s], e->ev_pass[s]})
      if (ev) cudaEventDestroy(ev);
  }
  if (e->pin_counts) cudaFreeHost(e->pin_counts);
  for (cudaEvent_t ev : {e->ev_side, e->ev_join, e->ev_model})
    if (ev) cudaEventDestroy(ev);
  for (cudaStream_t s : {e->main, e->side, e->copy, e->d2h})
    if (s) cudaStreamDestroy(s);
  delete e->stager;
  delete e->pool;
  delete e;
}

// (re)allocate the record queues for qcap slots each
int alloc_queues(nif_engine* e, int64_t slots_per_ray) {
  free_queues(e);
  e->slots_per_ray = slots_per_ray;
  const int64_t cap = e->chunk_cap * slots_per_ray;
  e->qcap = cap;
  // outer obj/ray/coord4, inner obj/ray/coord4/r; 7 arrays, 256 B aligned
  const size_t qbytes = (size_t)cap * (4 + 4 + 16) + (size_t)cap * (4 + 4 + 16 + 4) + 8 * 256;
  int rc = dev_alloc(&e->queues, qbytes);
  if (rc) return rc;
  if (e->outer.n_heads > 1) {
    const size_t nb = nif_bucket_scratch_bytes(cap, e->outer.n_obj);
    if ((rc = dev_alloc(&e->bucket[0], nb)) || (rc = dev_alloc(&e->bucket[1], nb))) return rc;
    // zero-filled once: the bucketed query re-zeroes its histogram itself
    if (cudaMemset(e->bucket[0], 0, nb) != cudaSuccess ||
        cudaMemset(e->bucket[1], 0, nb) != cudaSuccess)
      return nif::fail(NIF_ERR_CUDA, "engine: bucket scratch memset failed");
  }
  uint8_t* q = (uint8_t*)e->queues;
  auto carve = [&](size_t bytes) {
    uint8_t* p = q;
    q += (bytes + 255) / 256 * 256;
    return p;
  };
  e->out.outer_obj = (int32_t*)carve((size_t)cap * 4);
  e->out.outer_ray = (int32_t*)carve((size_t)cap * 4);
  e->out.outer_coord = (float*)carve((size_t)cap * 16);
  e->out.inner_obj = (int32_t*)carve((size_t)cap * 4);
  e->out.inner_ray = (int32_t*)carve((size_t)cap * 4);
  e->out.inner_coord = (float*)carve((size_t)cap * 16);
  e->out.inner_r = (float*)carve((size_t)cap * 4);
  if ((size_t)(q - (uint8_t*)e->queues) > qbytes)
    return nif::fail(NIF_ERR_CUDA, "engine: queue carve overflow");
  e->out.cap_outer = cap;
  e->out.cap_inner = cap;
  e->out.counts = e->counts;
  return NIF_OK;
}

// the engine's streams wait for work the caller enqueued on `producer`
// (e.g. nif_fast_pack_dev of the model the engine is about to read)
void wait_producer(nif_engine* e, void* producer) {
  cudaEventRecord(e->ev_model, (cudaStream_t)producer);
  cudaStreamWaitEvent(e->main, e->ev_model, 0);
  cudaStreamWaitEvent(e->side, e->ev_model, 0);
}

}  // namespace

extern "C" int nif_engine_create(const nif_scene_view* scene, const uint8_t* route_dev,
                                 int32_t n_net_obj, const nif_family_view* outer,
                                 const nif_family_view* inner, int64_t capacity,
                                 void* producer_stream, nif_engine** out_engine) {
  if (out_engine == nullptr) return nif::fail(NIF_ERR_VALUE, "engine: null output handle");
  *out_engine = nullptr;
  if (capacity <= 0) return nif::fail(NIF_ERR_VALUE, "engine capacity must be positive");
  if (outer == nullptr || inner == nullptr || outer->fast == nullptr || inner->fast == nullptr)
    return nif::fail(NIF_ERR_VALUE, "engine needs both families packed (nif_fast_pack_dev)");
  if (outer->sigmoid_head != 1 || inner->sigmoid_head != 1)
    return nif::fail(NIF_ERR_VALUE, "model was built with the geometry head");
  nif_engine* e = new (std::nothrow) nif_engine();
  if (e == nullptr) return nif::fail(NIF_ERR_CUDA, "engine: out of host memory");
  e->scene = *scene;
  e->outer = *outer;
  e->inner = *inner;
  e->route = route_dev;
  e->capacity = capacity;
  e->n_net = n_net_obj > 0 ? n_net_obj : 1;
  e->chunk_cap = std::min<int64_t>(capacity, chunk_rays_default());
  int rc = NIF_OK;
  e->ws_bytes = nif_gather_workspace_bytes(e->chunk_cap);
  if ((rc = dev_alloc(&e->org, (size_t)capacity * 24)) ||
      (rc = dev_alloc(&e->dir, (size_t)capacity * 24)) ||
      (rc = dev_alloc(&e->tms, (size_t)capacity * 8)) ||
      (rc = dev_alloc(&e->occ, (size_t)capacity)) ||
      (rc = dev_alloc(&e->workspace, e->ws_bytes)) ||
      (rc = dev_alloc(&e->counts, 4 * sizeof(int64_t)))) {
    release(e);
    return rc;
  }
  // the gather workspace starts zero-filled (its hot-path counters re-arm)
  if (cudaMemset(e->workspace, 0, e->ws_bytes) != cudaSuccess) {
    release(e);
    return nif::fail(NIF_ERR_CUDA, "engine: workspace memset failed");
  }
  // a shadow ray meets only a few network-routed boxes; start at 4 slots per
  // ray (C2: 1.16 records per ray) and grow on overflow
  if ((rc = alloc_queues(e, std::min(e->n_net, 4)))) {
    release(e);
    return rc;
  }
  e->slots = std::min(kMaxSlots, env_int("NIF_STAGING_SLOTS", kDefaultSlots));
  const char* ramp_env = std::getenv("NIF_STAGING_RAMP");
  e->ramp = ramp_env == nullptr || ramp_env[0] != '0';
  for (int s = 0; s < e->slots; ++s) {
    if (cudaHostAlloc((void**)&e->pin_in[s], (size_t)e->chunk_cap * 56, cudaHostAllocDefault) !=
            cudaSuccess ||
        cudaHostAlloc((void**)&e->pin_out[s], (size_t)e->chunk_cap, cudaHostAllocDefault) !=
            cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_in[s], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_out[s], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_pass[s], cudaEventDisableTiming) != cudaSuccess) {
      release(e);
      return nif::fail(NIF_ERR_CUDA, "engine: pinned staging allocation failed");
    }
  }
  if (cudaHostAlloc((void**)&e->pin_counts, sizeof(int64_t) * 4 * kMaxChunks,
                    cudaHostAllocDefault) != cudaSuccess ||
      cudaStreamCreateWithFlags(&e->main, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&e->copy, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&e->d2h, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->ev_side, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->ev_model, cudaEventDisableTiming) != cudaSuccess) {
    release(e);
    return nif::fail(NIF_ERR_CUDA, "engine: stream / event creation failed");
  }
  const unsigned hw = std::thread::hardware_concurrency();
  int threads = (int)std::max(1u, std::min(8u, hw > 1 ? hw / 2 : 1u));
  if (const char* env = std::getenv("NIF_STAGING_THREADS")) threads = std::max(1, std::atoi(env));
  // the stager thread joins the copy pool's workers in every staging copy
  e->pool = new (std::nothrow) CopyPool(threads - 1);
  e->stager = new (std::nothrow) Stager();
  if (e->pool == nullptr || e->stager == nullptr) {
    release(e);
    return nif::fail(NIF_ERR_CUDA, "engine: out of host memory");
  }
  wait_producer(e, producer_stream);
  *out_engine = e;
  return NIF_OK;
}

extern "C" int nif_engine_update_model(nif_engine* e, const nif_family_view* outer,
                                       const nif_family_view* inner, void* producer_stream) {
  if (e == nullptr) return nif::fail(NIF_ERR_VALUE, "engine: null handle");
  if (outer == nullptr || inner == nullptr || outer->fast == nullptr || inner->fast == nullptr)
    return nif::fail(NIF_ERR_VALUE, "engine needs both families packed (nif_fast_pack_dev)");
  if (outer->sigmoid_head != 1 || inner->sigmoid_head != 1)
    return nif::fail(NIF_ERR_VALUE, "model was built with the geometry head");
  e->outer = *outer;
  e->inner = *inner;
  wait_producer(e, producer_stream);
  return NIF_OK;
}

extern "C" int nif_engine_info(const nif_engine* e, int64_t* out4) {
  if (e == nullptr || out4 == nullptr) return nif::fail(NIF_ERR_VALUE, "engine: null argument");
  out4[0] = e->chunk_cap;
  out4[1] = e->slots_per_ray;
  out4[2] = e->pool->size();
  out4[3] = e->overflow_reruns;
  return NIF_OK;
}

namespace {

// the pass over rays [s0, s1) of the resident buffers, on e->main (outer
// family forked onto e->side and joined back); ray ids are chunk-relative
int run_range(nif_engine* e, int64_t s0, int64_t s1) {
  const int64_t n = s1 - s0;
  nif_gather_out out = e->out;
  out.bvh_occ = e->occ + s0;
  int rc = nif_gather_dev(&e->scene, e->route, e->org + 3 * s0, e->dir + 3 * s0, e->tms + s0, n,
                          &out, e->workspace, e->ws_bytes, e->main);
  if (rc != NIF_OK) return rc;
  cudaEventRecord(e->ev_side, e->main);
  cudaStreamWaitEvent(e->side, e->ev_side, 0);
  const int64_t cap = out.cap_outer;
  if (e->outer.n_heads > 1) {
    rc = nif_query_bucketed_dev(&e->outer, out.outer_obj, out.outer_ray, out.outer_coord, nullptr,
                                e->counts, cap, e->occ + s0, nullptr, e->bucket[0], e->side);
    if (rc == NIF_OK)
      rc = nif_query_bucketed_dev(&e->inner, out.inner_obj, out.inner_ray, out.inner_coord,
                                  out.inner_r, e->counts + 1, cap, e->occ + s0, nullptr,
                                  e->bucket[1], e->main);
  } else {
    rc = nif_query_dev(&e->outer, out.outer_obj, out.outer_ray, out.outer_coord, nullptr,
                       e->counts, cap, e->occ + s0, nullptr, NIF_IMPL_AUTO, e->side);
    if (rc == NIF_OK)
      rc = nif_query_dev(&e->inner, out.inner_obj, out.inner_ray, out.inner_coord, out.inner_r,
                         e->counts + 1, cap, e->occ + s0, nullptr, NIF_IMPL_AUTO, e->main);
  }
  cudaEventRecord(e->ev_join, e->side);
  cudaStreamWaitEvent(e->main, e->ev_join, 0);
  return rc;
}

// pageable -> pinned (or back) over the copy pool, in ~1 MB pieces
void pooled_copy(CopyPool* pool, std::vector<std::pair<void*, const void*>>& dst_src,
                 std::vector<size_t>& bytes) {
  constexpr size_t kPiece = 1 << 20;
  struct Piece {
    uint8_t* d;
    const uint8_t* s;
    size_t n;
  };
  std::vector<Piece> pieces;
  for (size_t k = 0; k < bytes.size(); ++k)
    for (size_t off = 0; off < bytes[k]; off += kPiece)
      pieces.push_back({(uint8_t*)dst_src[k].first + off, (const uint8_t*)dst_src[k].second + off,
                        std::min(kPiece, bytes[k] - off)});
  pool->run((int)pieces.size(), [&](int i) { stage_copy(pieces[i].d, pieces[i].s, pieces[i].n); });
}

}  // namespace

extern "C" int nif_engine_occluded_host(nif_engine* e, const double* origins,
                                        const double* dirs, const double* tmaxs, int64_t n,
                                        uint8_t* occ_out, int32_t chunks) {
  if (e == nullptr) return nif::fail(NIF_ERR_VALUE, "engine: null handle");
  if (n < 0) return nif::fail(NIF_ERR_VALUE, "ray count cannot be negative");
  if (n > e->capacity)
    return nif::fail(NIF_ERR_VALUE, "%lld rays exceed the engine capacity %lld", (long long)n,
                     (long long)e->capacity);
  if (n == 0) return NIF_OK;
  // chunk boundaries. Default: geometric ramp-up (slot/8, slot/4, slot/2,
  // then whole slots) so the first upload starts after a short staging copy
  // and the pipeline fill costs little; chunks > 0: uniform chunks.
  int64_t step = e->chunk_cap;
  if (chunks > 0) step = std::min(step, (n + chunks - 1) / chunks);
  step = std::max<int64_t>(step, (n + kMaxChunks - 1) / kMaxChunks);
  if (step > e->chunk_cap) return nif::fail(NIF_ERR_VALUE, "engine: too many rays per call");
  std::vector<int64_t> bound{0};
  for (int64_t size = chunks > 0 || !e->ramp ? step : std::max<int64_t>(1, step / 8);
       bound.back() < n;
       size = std::min(step, 2 * size)) {
    if ((int)bound.size() > kMaxChunks) return nif::fail(NIF_ERR_VALUE, "engine: too many chunks");
    bound.push_back(std::min(n, bound.back() + size));
  }
  const int nc = (int)bound.size() - 1;
  int rc = NIF_OK;
  auto drain = [&](int k) {  // chunk k's answer: pinned out slot -> caller
    const int s = k % e->slots;
    const int64_t s0 = bound[k], s1 = bound[k + 1];
    cudaEventSynchronize(e->ev_out[s]);
    std::memcpy(occ_out + s0, e->pin_out[s], (size_t)(s1 - s0));
  };
  // Staging runs on the stager thread (+ copy pool), one chunk ahead of the
  // uploads: it fills slot k % S once the upload of chunk k - S (the slot's
  // previous tenant) has been issued and has completed, then publishes
  // `staged` = k + 1. This thread waits for `staged`, issues the upload and
  // the chunk's pass, and publishes `issued`.
  std::atomic<int> staged{0}, issued{0};
  std::atomic<bool> abort{false};
  // NIF_STAGING_TRACE=1: host timeline of the call on stderr (diagnostics)
  static const bool trace = std::getenv("NIF_STAGING_TRACE") != nullptr;
  using clk = std::chrono::steady_clock;
  const auto t_call = clk::now();
  std::vector<double> t_staged(trace ? nc : 0), t_issued(trace ? nc : 0);
  auto us = [&] { return std::chrono::duration<double, std::micro>(clk::now() - t_call).count(); };
  e->stager->start([&] {
    for (int k = 0; k < nc; ++k) {
      const int s = k % e->slots;
      if (k >= e->slots) {
        if (!wait_counter(issued, k - e->slots + 1, abort)) return;
        cudaEventSynchronize(e->ev_in[s]);  // the slot's previous upload is done
      }
      const int64_t s0 = bound[k], m = bound[k + 1] - s0;
      uint8_t* pin = e->pin_in[s];
      std::vector<std::pair<void*, const void*>> ds = {
          {pin, origins + 3 * s0}, {pin + m * 24, dirs + 3 * s0}, {pin + m * 48, tmaxs + s0}};
      std::vector<size_t> bytes = {(size_t)m * 24, (size_t)m * 24, (size_t)m * 8};
      pooled_copy(e->pool, ds, bytes);
      if (trace) t_staged[k] = us();
      staged.store(k + 1, std::memory_order_release);
    }
  });
  for (int k = 0; k < nc && rc == NIF_OK; ++k) {
    const int s = k % e->slots;
    const int64_t s0 = bound[k], s1 = bound[k + 1], m = s1 - s0;
    if (k >= e->slots) drain(k - e->slots);  // the out slot's previous answer is out
    wait_counter(staged, k + 1, abort);
    uint8_t* pin = e->pin_in[s];
    cudaMemcpyAsync(e->org + 3 * s0, pin, (size_t)m * 24, cudaMemcpyHostToDevice, e->copy);
    cudaMemcpyAsync(e->dir + 3 * s0, pin + m * 24, (size_t)m * 24, cudaMemcpyHostToDevice,
                    e->copy);
    cudaMemcpyAsync(e->tms + s0, pin + m * 48, (size_t)m * 8, cudaMemcpyHostToDevice, e->copy);
    cudaEventRecord(e->ev_in[s], e->copy);
    issued.store(k + 1, std::memory_order_release);
    cudaStreamWaitEvent(e->main, e->ev_in[s], 0);
    rc = run_range(e, s0, s1);
    if (rc != NIF_OK) break;
    cudaMemcpyAsync(e->pin_counts + 4 * k, e->counts, 4 * sizeof(int64_t),
                    cudaMemcpyDeviceToHost, e->main);
    cudaEventRecord(e->ev_pass[s], e->main);
    cudaStreamWaitEvent(e->d2h, e->ev_pass[s], 0);
    cudaMemcpyAsync(e->pin_out[s], e->occ + s0, (size_t)m, cudaMemcpyDeviceToHost, e->d2h);
    cudaEventRecord(e->ev_out[s], e->d2h);
    if (trace) t_issued[k] = us();
  }
  if (rc != NIF_OK) abort.store(true);
  e->stager->wait();
  if (rc == NIF_OK)
    for (int k = std::max(0, nc - e->slots); k < nc; ++k) drain(k);
  if (trace) {
    std::fprintf(stderr, "{\"staging_trace_us\": {\"chunks\": %d, \"staged\": [", nc);
    for (int k = 0; k < nc; ++k) std::fprintf(stderr, "%s%.1f", k ? "," : "", t_staged[k]);
    std::fprintf(stderr, "], \"issued\": [");
    for (int k = 0; k < nc; ++k) std::fprintf(stderr, "%s%.1f", k ? "," : "", t_issued[k]);
    std::fprintf(stderr, "], \"drained\": %.1f}}\n", us());
  }
  const cudaError_t err = cudaStreamSynchronize(e->main);
  cudaStreamSynchronize(e->copy);
  cudaStreamSynchronize(e->d2h);
  if (rc != NIF_OK) return rc;
  if (err != cudaSuccess) return nif::fail(NIF_ERR_CUDA, "engine: %s", cudaGetErrorString(err));
  // overflowed chunks: grow the queues to the largest total seen and re-run
  // them (their rays are still resident)
  const int64_t qcap_run = e->qcap;
  auto total = [&](int k) { return std::max(e->pin_counts[4 * k], e->pin_counts[4 * k + 1]); };
  int64_t need = 0;
  for (int k = 0; k < nc; ++k) need = std::max(need, total(k));
  if (need > qcap_run) {
    // a chunk holds at most chunk_cap * n_net records per queue
    const int64_t want = (need + need / 4 + e->chunk_cap - 1) / e->chunk_cap;
    if ((rc = alloc_queues(e, std::min<int64_t>(e->n_net, want)))) return rc;
    for (int k = 0; k < nc; ++k) {
      if (total(k) <= qcap_run) continue;
      const int64_t s0 = bound[k], s1 = bound[k + 1];
      ++e->overflow_reruns;
      if ((rc = run_range(e, s0, s1))) return rc;
      cudaMemcpyAsync(occ_out + s0, e->occ + s0, (size_t)(s1 - s0), cudaMemcpyDeviceToHost,
                      e->main);
      if (cudaStreamSynchronize(e->main) != cudaSuccess)
        return nif::fail(NIF_ERR_CUDA, "engine: re-run failed");
    }
  }
  return NIF_OK;
}

extern "C" int nif_engine_destroy(nif_engine* e) {
  if (e == nullptr) return NIF_OK;
  cudaStreamSynchronize(e->main);
  cudaStreamSynchronize(e->side);
  cudaStreamSynchronize(e->copy);
  cudaStreamSynchronize(e->d2h);
  release(e);
  return NIF_OK;
}
