// Native visibility engine: the whole split pass behind one C-ABI object
// (SURVEY.md §8b "nif_occluded (fused whole path)"), for FFI callers that
// hold rays in host memory -- the drop-in for PredictorBackend.occluded
// (renderer.py:675-683) / NifBackend (nif.py:486-499) from a ctypes stub.
//
// The engine owns every device buffer of the pass for a fixed ray capacity:
// rays, the gather's record queues and workspace, the per-ray answer and,
// for per_object models, the bucketing scratch of each family. One call
// copies a chunk of rays in, runs gather -> outer / inner query (the two
// families on two streams) and copies the chunk's answer out; chunk k+1's
// host->device copy is issued on a copy stream while chunk k computes.
// Scene and model stay owned by the caller (views of device memory, e.g.
// built by the Python package); call nif_fast_pack_dev after each optimiser
// step before the next query, as for nif_query_dev.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>

#include "kernels.h"
#include "nif_b200.h"
#include "status.h"

struct nif_engine {
  nif_scene_view scene;
  nif_family_view outer, inner;
  const uint8_t* route;  // device
  int64_t capacity = 0;
  int n_net = 0;
  double* org = nullptr;
  double* dir = nullptr;
  double* tms = nullptr;
  uint8_t* occ = nullptr;  // per-ray answer (the gather seeds it with bvh_occ)
  void* queues = nullptr;
  void* workspace = nullptr;
  size_t ws_bytes = 0;
  void* bucket[2] = {nullptr, nullptr};
  int64_t* counts = nullptr;
  nif_gather_out out{};
  cudaStream_t main = nullptr, side = nullptr, copy = nullptr;
  cudaEvent_t ev_side = nullptr, ev_join = nullptr;
};

namespace {

template <typename T>
int dev_alloc(T** p, size_t bytes) {
  if (cudaMalloc((void**)p, bytes > 0 ? bytes : 1) != cudaSuccess)
    return nif::fail(NIF_ERR_CUDA, "engine: cudaMalloc of %zu bytes failed", bytes);
  return NIF_OK;
}

void release(nif_engine* e) {
  for (void* p : {(void*)e->org, (void*)e->dir, (void*)e->tms, (void*)e->occ, e->queues,
                  e->workspace, e->bucket[0], e->bucket[1], (void*)e->counts})
    if (p) cudaFree(p);
  if (e->ev_side) cudaEventDestroy(e->ev_side);
  if (e->ev_join) cudaEventDestroy(e->ev_join);
  for (cudaStream_t s : {e->main, e->side, e->copy})
    if (s) cudaStreamDestroy(s);
  delete e;
}

}  // namespace

extern "C" int nif_engine_create(const nif_scene_view* scene, const uint8_t* route_dev,
                                 int32_t n_net_obj, const nif_family_view* outer,
                                 const nif_family_view* inner, int64_t capacity,
                                 nif_engine** out_engine) {
  if (out_engine == nullptr) return nif::fail(NIF_ERR_VALUE, "engine: null output handle");
  *out_engine = nullptr;
  if (capacity <= 0) return nif::fail(NIF_ERR_VALUE, "engine capacity must be positive");
  if (outer == nullptr || inner == nullptr || outer->fast == nullptr || inner->fast == nullptr)
    return nif::fail(NIF_ERR_VALUE, "engine needs both families packed (nif_fast_pack_dev)");
  nif_engine* e = new (std::nothrow) nif_engine();
  if (e == nullptr) return nif::fail(NIF_ERR_CUDA, "engine: out of host memory");
  e->scene = *scene;
  e->outer = *outer;
  e->inner = *inner;
  e->route = route_dev;
  e->capacity = capacity;
  e->n_net = n_net_obj > 0 ? n_net_obj : 1;
  const int64_t cap = capacity * e->n_net;  // record slots per queue (gather bound)
  int rc = NIF_OK;
  // queues: outer obj/ray/coord4, inner obj/ray/coord4/r
  // 7 arrays, each rounded up to 256 B by carve()
  const size_t qbytes = (size_t)cap * (4 + 4 + 16) + (size_t)cap * (4 + 4 + 16 + 4) + 8 * 256;
  e->ws_bytes = nif_gather_workspace_bytes(capacity);
  if ((rc = dev_alloc(&e->org, (size_t)capacity * 24)) || (rc = dev_alloc(&e->dir, (size_t)capacity * 24)) ||
      (rc = dev_alloc(&e->tms, (size_t)capacity * 8)) || (rc = dev_alloc(&e->occ, (size_t)capacity)) ||
      (rc = dev_alloc(&e->queues, qbytes)) || (rc = dev_alloc(&e->workspace, e->ws_bytes)) ||
      (rc = dev_alloc(&e->counts, 4 * sizeof(int64_t)))) {
    release(e);
    return rc;
  }
  if (outer->n_heads > 1) {
    const size_t nb = nif_bucket_scratch_bytes(cap, outer->n_obj);
    if ((rc = dev_alloc(&e->bucket[0], nb)) || (rc = dev_alloc(&e->bucket[1], nb))) {
      release(e);
      return rc;
    }
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
  if ((size_t)(q - (uint8_t*)e->queues) > qbytes) {
    release(e);
    return nif::fail(NIF_ERR_CUDA, "engine: queue carve overflow");
  }
  e->out.cap_outer = cap;
  e->out.cap_inner = cap;
  e->out.counts = e->counts;
  if (cudaStreamCreateWithFlags(&e->main, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&e->copy, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->ev_side, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    release(e);
    return nif::fail(NIF_ERR_CUDA, "engine: stream / event creation failed");
  }
  *out_engine = e;
  return NIF_OK;
}

extern "C" int nif_engine_update_model(nif_engine* e, const nif_family_view* outer,
                                       const nif_family_view* inner) {
  if (e == nullptr) return nif::fail(NIF_ERR_VALUE, "engine: null handle");
  e->outer = *outer;
  e->inner = *inner;
  return NIF_OK;
}

namespace {

// the pass over rays [s0, s1) of the resident buffers, on e->main (outer
// family forked onto e->side and joined back)
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
  if (chunks < 1) chunks = 1;
  const int64_t step = (n + chunks - 1) / chunks;
  cudaEvent_t ready[64];
  const int nc = (int)std::min<int64_t>((n + step - 1) / step, 64);
  const int64_t step2 = (n + nc - 1) / nc;
  for (int k = 0; k < nc; ++k) cudaEventCreateWithFlags(&ready[k], cudaEventDisableTiming);
  for (int k = 0; k < nc; ++k) {  // all copies in, in order, on the copy stream
    const int64_t s0 = k * step2, s1 = std::min(n, s0 + step2);
    cudaMemcpyAsync(e->org + 3 * s0, origins + 3 * s0, (size_t)(s1 - s0) * 24,
                    cudaMemcpyHostToDevice, e->copy);
    cudaMemcpyAsync(e->dir + 3 * s0, dirs + 3 * s0, (size_t)(s1 - s0) * 24,
                    cudaMemcpyHostToDevice, e->copy);
    cudaMemcpyAsync(e->tms + s0, tmaxs + s0, (size_t)(s1 - s0) * 8, cudaMemcpyHostToDevice,
                    e->copy);
    cudaEventRecord(ready[k], e->copy);
  }
  int rc = NIF_OK;
  for (int k = 0; k < nc && rc == NIF_OK; ++k) {  // chunk k computes as k+1 streams in
    const int64_t s0 = k * step2, s1 = std::min(n, s0 + step2);
    cudaStreamWaitEvent(e->main, ready[k], 0);
    rc = run_range(e, s0, s1);
    if (rc == NIF_OK)
      cudaMemcpyAsync(occ_out + s0, e->occ + s0, (size_t)(s1 - s0), cudaMemcpyDeviceToHost,
                      e->main);
  }
  const cudaError_t err = cudaStreamSynchronize(e->main);
  cudaStreamSynchronize(e->copy);
  for (int k = 0; k < nc; ++k) cudaEventDestroy(ready[k]);
  if (rc != NIF_OK) return rc;
  if (err != cudaSuccess) return nif::fail(NIF_ERR_CUDA, "engine: %s", cudaGetErrorString(err));
  return NIF_OK;
}

extern "C" int nif_engine_destroy(nif_engine* e) {
  if (e == nullptr) return NIF_OK;
  cudaStreamSynchronize(e->main);
  cudaStreamSynchronize(e->side);
  cudaStreamSynchronize(e->copy);
  release(e);
  return NIF_OK;
}
