// GPU binned-SAH BVH build that reproduces the reference builder node for
// node (bvh.py:34-303 _build_sah; host twin: sah_builder.cpp).
//
// Level-synchronous: every node of one tree level is one CTA. A CTA reduces
// its segment's bounds, bins the centroids of every axis at once (warp-
// private shared-memory bins), evaluates the reference's sweeps and SAH
// costs on one thread in the reference's order, and stably partitions its
// segment (block-wide scans over the segment in order), so each segment's
// contents and order evolve exactly as in the reference's depth-first loop.
// The reference numbers nodes in depth-first processing order (the k-th
// split node in preorder gives its children ids 2k+1, 2k+2); after the
// build, subtree internal-node counts (bottom-up) and preorder ranks
// (top-down) recover those ids. Arithmetic as in the host builder:
// -fmad=false, the reference's expression order, first-occurrence ties for
// the node bounds (the reference's sequential `if x < best` scans).
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.h"
#include "kernels.h"
#include "nif_b200.h"
#include "status.h"

namespace nif {
namespace {

constexpr int kBT = 256;       // threads per segment CTA
constexpr int kWarps = kBT / 32;
constexpr int kMaxBins = 32;

struct SahIn {
  const double* lo;
  const double* hi;
  const double* ce;
  int64_t max_leaf;
  int n_bins;
  double c_trav, c_isect;
};

struct BfsNodes {  // indexed by build (BFS-allocation) id
  double* lo;      // [cap][3]
  double* hi;
  int64_t* start;
  int64_t* count;
  int32_t* left;
  int32_t* right;
  uint8_t* leaf;
};

struct LevelIO {
  const int64_t* s_start;
  const int64_t* s_end;
  const int32_t* s_id;
  int64_t* n_start;
  int64_t* n_end;
  int32_t* n_id;
  int* n_next;
  int* id_counter;
  const int64_t* order_in;
  int64_t* order_out;
  int64_t* order_final;
};

__device__ __forceinline__ int bin_of(double c, double cmin, double ext, int n_bins) {
  // bvh.py:148  b = int(n_bins * (ce[p, axis] - cmin) / ext), clamped
  long long b = (long long)((double)n_bins * (c - cmin) / ext);
  if (b >= n_bins) b = n_bins - 1;
  if (b < 0) b = 0;
  return (int)b;
}

// total order on doubles for the bin bounds (the sign of a zero bound never
// changes a surface area, so -0 < +0 is harmless there)
__device__ __forceinline__ unsigned long long dkey(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dval(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// value + scan position: IEEE comparison, ties (incl. -0 == +0) to the
// earliest position -- what the reference's sequential scan keeps
struct VI {
  double v;
  long long i;
};
__device__ __forceinline__ void vi_min(VI& a, double v, long long i) {
  if (v < a.v || (!(a.v < v) && i < a.i)) {
    a.v = v;
    a.i = i;
  }
}
__device__ __forceinline__ void vi_max(VI& a, double v, long long i) {
  if (v > a.v || (!(a.v > v) && i < a.i)) {
    a.v = v;
    a.i = i;
  }
}

__global__ void __launch_bounds__(kBT) sah_level_kernel(SahIn P, LevelIO L, BfsNodes N) {
  const int64_t start = L.s_start[blockIdx.x], end = L.s_end[blockIdx.x];
  const int id = L.s_id[blockIdx.x];
  const int64_t count = end - start;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = P.n_bins;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);

  __shared__ VI s_b[kWarps][6];
  __shared__ double s_c[kWarps][6];
  __shared__ int s_cnt[kWarps][3][kMaxBins];
  __shared__ unsigned long long s_blo[kWarps][3][kMaxBins][3];
  __shared__ unsigned long long s_bhi[kWarps][3][kMaxBins][3];
  __shared__ double s_cmin[3], s_ext[3];
  __shared__ int s_bin_axes, s_mode, s_axis, s_k;  // mode: 0 leaf, 1 bin split, 2 halve
  __shared__ long long s_nl;
  __shared__ int s_scan[kWarps];

  // ---- 1. node bounds (first occurrence) and centroid bounds ---------------
  VI bl[3], bh[3];
  double cl[3], ch[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    bl[c] = {inf, (long long)0x7fffffffffffffffll};
    bh[c] = {-inf, (long long)0x7fffffffffffffffll};
    cl[c] = inf;
    ch[c] = -inf;
  }
  for (int64_t i = start + tid; i < end; i += kBT) {
    const int64_t p = L.order_in[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      vi_min(bl[c], P.lo[p * 3 + c], i);
      vi_max(bh[c], P.hi[p * 3 + c], i);
      const double cc = P.ce[p * 3 + c];
      cl[c] = cc < cl[c] ? cc : cl[c];
      ch[c] = cc > ch[c] ? cc : ch[c];
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double v0 = __shfl_xor_sync(0xffffffffu, bl[c].v, off);
      const long long i0 = __shfl_xor_sync(0xffffffffu, bl[c].i, off);
      vi_min(bl[c], v0, i0);
      const double v1 = __shfl_xor_sync(0xffffffffu, bh[c].v, off);
      const long long i1 = __shfl_xor_sync(0xffffffffu, bh[c].i, off);
      vi_max(bh[c], v1, i1);
      const double c0 = __shfl_xor_sync(0xffffffffu, cl[c], off);
      const double c1 = __shfl_xor_sync(0xffffffffu, ch[c], off);
      cl[c] = c0 < cl[c] ? c0 : cl[c];
      ch[c] = c1 > ch[c] ? c1 : ch[c];
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      s_b[warp][c] = bl[c];
      s_b[warp][3 + c] = bh[c];
      s_c[warp][c] = cl[c];
      s_c[warp][3 + c] = ch[c];
    }
  }
  // clear the warp-private bins meanwhile
  for (int e = tid; e < kWarps * 3 * kMaxBins; e += kBT) {
    (&s_cnt[0][0][0])[e] = 0;
    for (int c = 0; c < 3; ++c) {
      (&s_blo[0][0][0][0])[e * 3 + c] = 0xffffffffffffffffull;
      (&s_bhi[0][0][0][0])[e * 3 + c] = 0ull;
    }
  }
  __syncthreads();
  if (tid == 0) {
    VI B[6];
    double Cl[3], Ch[3];
    for (int c = 0; c < 6; ++c) B[c] = s_b[0][c];
    for (int c = 0; c < 3; ++c) {
      Cl[c] = s_c[0][c];
      Ch[c] = s_c[0][3 + c];
    }
    for (int w = 1; w < kWarps; ++w)
      for (int c = 0; c < 3; ++c) {
        vi_min(B[c], s_b[w][c].v, s_b[w][c].i);
        vi_max(B[3 + c], s_b[w][3 + c].v, s_b[w][3 + c].i);
        Cl[c] = s_c[w][c] < Cl[c] ? s_c[w][c] : Cl[c];
        Ch[c] = s_c[w][3 + c] > Ch[c] ? s_c[w][3 + c] : Ch[c];
      }
    for (int c = 0; c < 3; ++c) {
      N.lo[(int64_t)id * 3 + c] = B[c].v;
      N.hi[(int64_t)id * 3 + c] = B[3 + c].v;
    }
    int axes = 0;
    if (count > 1) {
      const double dx = B[3].v - B[0].v, dy = B[4].v - B[1].v, dz = B[5].v - B[2].v;
      const double sa_node = 2.0 * (dx * dy + dy * dz + dz * dx);
      if (sa_node > 1e-300)
        for (int a = 0; a < 3; ++a) {
          s_cmin[a] = Cl[a];
          s_ext[a] = Ch[a] - Cl[a];
          if (s_ext[a] > 0.0) axes |= 1 << a;
        }
      // stash the node surface area for the cost pass in s_c (reuse)
      s_c[0][0] = sa_node;
    }
    s_bin_axes = axes;
  }
  __syncthreads();
  const int axes = s_bin_axes;

  // ---- 2. centroid bins of every live axis ----------------------------------
  if (axes) {
    for (int64_t i = start + tid; i < end; i += kBT) {
      const int64_t p = L.order_in[i];
      for (int a = 0; a < 3; ++a) {
        if (!(axes & (1 << a))) continue;
        const int b = bin_of(P.ce[p * 3 + a], s_cmin[a], s_ext[a], nb);
        atomicAdd(&s_cnt[warp][a][b], 1);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          atomicMin(&s_blo[warp][a][b][c], dkey(P.lo[p * 3 + c]));
          atomicMax(&s_bhi[warp][a][b][c], dkey(P.hi[p * 3 + c]));
        }
      }
    }
  }
  __syncthreads();

  // ---- 3. sweeps, costs, split decision (one thread, reference order) ------
  if (tid == 0) {
    int best_axis = -1, best_k = -1;
    double best_cost = inf;
    long long best_nl = 0;
    if (axes) {
      const double sa_node = s_c[0][0];
      for (int a = 0; a < 3; ++a) {
        if (!(axes & (1 << a))) continue;
        long long cnt[kMaxBins];
        double blo[kMaxBins][3], bhi[kMaxBins][3];
        for (int k = 0; k < nb; ++k) {
          long long cc = 0;
          unsigned long long kl[3] = {0xffffffffffffffffull, 0xffffffffffffffffull,
                                      0xffffffffffffffffull};
          unsigned long long kh[3] = {0ull, 0ull, 0ull};
          for (int w = 0; w < kWarps; ++w) {
            cc += s_cnt[w][a][k];
            for (int c = 0; c < 3; ++c) {
              kl[c] = s_blo[w][a][k][c] < kl[c] ? s_blo[w][a][k][c] : kl[c];
              kh[c] = s_bhi[w][a][k][c] > kh[c] ? s_bhi[w][a][k][c] : kh[c];
            }
          }
          cnt[k] = cc;
          for (int c = 0; c < 3; ++c) {
            blo[k][c] = cc ? dval(kl[c]) : inf;
            bhi[k][c] = cc ? dval(kh[c]) : -inf;
          }
        }
        double left_sa[kMaxBins], right_sa[kMaxBins];
        long long left_n[kMaxBins], right_n[kMaxBins];
        double ax = inf, ay = inf, az = inf, bx = -inf, by = -inf, bz = -inf;
        long long c0 = 0;
        for (int k = 0; k < nb; ++k) {  // bvh.py:159-189
          if (cnt[k] > 0) {
            if (blo[k][0] < ax) ax = blo[k][0];
            if (blo[k][1] < ay) ay = blo[k][1];
            if (blo[k][2] < az) az = blo[k][2];
            if (bhi[k][0] > bx) bx = bhi[k][0];
            if (bhi[k][1] > by) by = bhi[k][1];
            if (bhi[k][2] > bz) bz = bhi[k][2];
          }
          c0 += cnt[k];
          left_n[k] = c0;
          if (c0 > 0) {
            const double ex = bx - ax, ey = by - ay, ez = bz - az;
            left_sa[k] = 2.0 * (ex * ey + ey * ez + ez * ex);
          } else {
            left_sa[k] = 0.0;
          }
        }
        ax = ay = az = inf;
        bx = by = bz = -inf;
        c0 = 0;
        for (int k = nb - 1; k >= 0; --k) {  // bvh.py:190-219
          if (cnt[k] > 0) {
            if (blo[k][0] < ax) ax = blo[k][0];
            if (blo[k][1] < ay) ay = blo[k][1];
            if (blo[k][2] < az) az = blo[k][2];
            if (bhi[k][0] > bx) bx = bhi[k][0];
            if (bhi[k][1] > by) by = bhi[k][1];
            if (bhi[k][2] > bz) bz = bhi[k][2];
          }
          c0 += cnt[k];
          right_n[k] = c0;
          if (c0 > 0) {
            const double ex = bx - ax, ey = by - ay, ez = bz - az;
            right_sa[k] = 2.0 * (ex * ey + ey * ez + ez * ex);
          } else {
            right_sa[k] = 0.0;
          }
        }
        for (int k = 0; k < nb - 1; ++k) {  // bvh.py:220-229
          const long long nl = left_n[k], nr = right_n[k + 1];
          if (nl == 0 || nr == 0) continue;
          const double cost = P.c_trav + (left_sa[k] * (double)nl + right_sa[k + 1] * (double)nr) *
                                             P.c_isect / sa_node;
          if (cost < best_cost) {
            best_cost = cost;
            best_axis = a;
            best_k = k;
            best_nl = nl;
          }
        }
      }
    }
    int mode = 0;
    if (best_axis >= 0 && (count > P.max_leaf || best_cost < P.c_isect * (double)count))
      mode = 1;
    else if (count > P.max_leaf)
      mode = 2;
    s_mode = mode;
    s_axis = best_axis;
    s_k = best_k;
    s_nl = mode == 1 ? best_nl : count / 2;
  }
  __syncthreads();
  const int mode = s_mode;

  // ---- 4. leaf / stable partition / halving ---------------------------------
  if (mode == 0) {
    for (int64_t i = start + tid; i < end; i += kBT) L.order_final[i] = L.order_in[i];
    if (tid == 0) {
      N.leaf[id] = 1;
      N.start[id] = start;
      N.count[id] = count;
    }
    return;
  }
  const long long nl = s_nl;
  if (mode == 2) {
    for (int64_t i = start + tid; i < end; i += kBT) L.order_out[i] = L.order_in[i];
  } else {
    const int a = s_axis, kk = s_k;
    const double cmin = s_cmin[a], ext = s_ext[a];
    long long lbase = 0, rbase = 0;
    for (int64_t c0 = start; c0 < end; c0 += kBT) {
      const int64_t i = c0 + tid;
      const bool valid = i < end;
      int64_t p = 0;
      bool left = false;
      if (valid) {
        p = L.order_in[i];
        left = bin_of(P.ce[p * 3 + a], cmin, ext, nb) <= kk;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, valid && left);
      const unsigned bar = __ballot_sync(0xffffffffu, valid && !left);
      if (lane == 0) s_scan[warp] = __popc(bal) | (__popc(bar) << 16);
      __syncthreads();
      int lw = 0, rw = 0, lt = 0, rt = 0;
      for (int w = 0; w < kWarps; ++w) {
        const int v = s_scan[w];
        if (w < warp) {
          lw += v & 0xffff;
          rw += v >> 16;
        }
        lt += v & 0xffff;
        rt += v >> 16;
      }
      const unsigned below = (1u << lane) - 1u;
      if (valid) {
        if (left)
          L.order_out[start + lbase + lw + __popc(bal & below)] = p;
        else
          L.order_out[start + nl + rbase + rw + __popc(bar & below)] = p;
      }
      lbase += lt;
      rbase += rt;
      __syncthreads();
    }
  }
  if (tid == 0) {
    const int base = atomicAdd(L.id_counter, 2);
    N.leaf[id] = 0;
    N.left[id] = base;
    N.right[id] = base + 1;
    const int j = atomicAdd(L.n_next, 2);
    const int64_t mid = start + nl;
    L.n_start[j] = start;
    L.n_end[j] = mid;
    L.n_id[j] = base;
    L.n_start[j + 1] = mid;
    L.n_end[j + 1] = end;
    L.n_id[j + 1] = base + 1;
  }
}

__global__ void iota_kernel(int64_t* o, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = i;
}

// bottom-up: internal-node count of each subtree (one tree level per launch)
__global__ void sah_isub_kernel(const int32_t* ids, int n, BfsNodes N, int32_t* isub) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int v = ids[j];
  isub[v] = N.leaf[v] ? 0 : 1 + isub[N.left[v]] + isub[N.right[v]];
}

// top-down: preorder rank among internal nodes -> the reference's node ids
__global__ void sah_rank_kernel(const int32_t* ids, int n, BfsNodes N, const int32_t* isub,
                                int32_t* rank, int32_t* ref_id) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int v = ids[j];
  if (N.leaf[v]) return;
  const int k = rank[v];
  const int l = N.left[v], r = N.right[v];
  ref_id[l] = 1 + 2 * k;
  ref_id[r] = 2 + 2 * k;
  rank[l] = k + 1;
  rank[r] = k + 1 + isub[l];
}

__global__ void sah_emit_kernel(int n_nodes, BfsNodes N, const int32_t* ref_id, double* node_lo,
                                double* node_hi, int64_t* node_a, int64_t* node_b,
                                uint8_t* node_leaf) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n_nodes) return;
  const int r = ref_id[v];
  for (int c = 0; c < 3; ++c) {
    node_lo[(int64_t)r * 3 + c] = N.lo[(int64_t)v * 3 + c];
    node_hi[(int64_t)r * 3 + c] = N.hi[(int64_t)v * 3 + c];
  }
  node_leaf[r] = N.leaf[v];
  if (N.leaf[v]) {
    node_a[r] = N.start[v];
    node_b[r] = N.count[v];
  } else {
    node_a[r] = ref_id[N.left[v]];
    node_b[r] = ref_id[N.right[v]];
  }
}

template <typename T>
T* dalloc(size_t count, cudaStream_t st) {
  void* p = nullptr;
  if (cudaMallocAsync(&p, count * sizeof(T) + 16, st) != cudaSuccess) return nullptr;
  return (T*)p;
}

}  // namespace
}  // namespace nif

using namespace nif;

extern "C" int nif_build_sah_dev(const double* lo, const double* hi, const double* ce, int64_t n,
                                 int64_t max_leaf, int64_t n_bins, double c_trav, double c_isect,
                                 double* node_lo, double* node_hi, int64_t* node_a,
                                 int64_t* node_b, uint8_t* node_leaf, int64_t* order,
                                 int64_t* n_nodes_out, void* stream) {
  if (n <= 0) return fail(NIF_ERR_VALUE, "cannot build a tree over zero primitives");
  if (n_bins < 2 || n_bins > kMaxBins || max_leaf < 1)
    return fail(NIF_ERR_VALUE, "bad SAH parameters (2 <= n_bins <= %d)", kMaxBins);
  if (n >= (int64_t)1 << 30) return fail(NIF_ERR_VALUE, "GPU SAH build supports < 2^30 primitives");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t cap = 2 * n;
  BfsNodes N{dalloc<double>(cap * 3, st), dalloc<double>(cap * 3, st), dalloc<int64_t>(cap, st),
             dalloc<int64_t>(cap, st),    dalloc<int32_t>(cap, st),    dalloc<int32_t>(cap, st),
             dalloc<uint8_t>(cap, st)};
  int64_t* ord_a = dalloc<int64_t>(n, st);
  int64_t* ord_b = dalloc<int64_t>(n, st);
  // per-level segment lists, stacked: every node id appears in exactly one
  int64_t* seg_s = dalloc<int64_t>(cap, st);
  int64_t* seg_e = dalloc<int64_t>(cap, st);
  int32_t* seg_i = dalloc<int32_t>(cap, st);
  int* counters = dalloc<int>(2, st);  // [0] id counter, [1] next-level count
  int32_t* isub = dalloc<int32_t>(cap, st);
  int32_t* rank = dalloc<int32_t>(cap, st);
  int32_t* ref_id = dalloc<int32_t>(cap, st);
  if (!N.lo || !N.hi || !N.start || !N.count || !N.left || !N.right || !N.leaf || !ord_a ||
      !ord_b || !seg_s || !seg_e || !seg_i || !counters || !isub || !rank || !ref_id)
    return fail(NIF_ERR_CUDA, "GPU SAH build: device allocation failed");
  iota_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ord_a, n);
  const int64_t root_s = 0;
  const int32_t root_i = 0;
  cudaMemcpyAsync(seg_s, &root_s, 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(seg_e, &n, 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(seg_i, &root_i, 4, cudaMemcpyHostToDevice, st);
  const int init[2] = {1, 0};
  cudaMemcpyAsync(counters, init, 8, cudaMemcpyHostToDevice, st);
  SahIn P{lo, hi, ce, max_leaf, (int)n_bins, c_trav, c_isect};
  std::vector<std::pair<int64_t, int>> levels;  // (offset into the stacked lists, count)
  int64_t off = 0;
  int n_seg = 1;
  int64_t* oin = ord_a;
  int64_t* oout = ord_b;
  while (n_seg > 0) {
    levels.push_back({off, n_seg});
    LevelIO L{seg_s + off, seg_e + off, seg_i + off, seg_s + off + n_seg, seg_e + off + n_seg,
              seg_i + off + n_seg, counters + 1, counters, oin, oout, order};
    cudaMemsetAsync(counters + 1, 0, 4, st);
    sah_level_kernel<<<(unsigned)n_seg, kBT, 0, st>>>(P, L, N);
    int next = 0;
    cudaMemcpyAsync(&next, counters + 1, 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("nif_build_sah_dev(level)");
    off += n_seg;
    n_seg = next;
    int64_t* t = oin;
    oin = oout;
    oout = t;
  }
  int n_nodes = 0;
  cudaMemcpyAsync(&n_nodes, counters, 4, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  // reference numbering
  for (int lv = (int)levels.size() - 1; lv >= 0; --lv) {
    const int cnt = levels[lv].second;
    sah_isub_kernel<<<(cnt + 255) / 256, 256, 0, st>>>(seg_i + levels[lv].first, cnt, N, isub);
  }
  const int zero = 0;
  cudaMemcpyAsync(rank, &zero, 4, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(ref_id, &zero, 4, cudaMemcpyHostToDevice, st);
  for (size_t lv = 0; lv < levels.size(); ++lv) {
    const int cnt = levels[lv].second;
    sah_rank_kernel<<<(cnt + 255) / 256, 256, 0, st>>>(seg_i + levels[lv].first, cnt, N, isub,
                                                       rank, ref_id);
  }
  sah_emit_kernel<<<(n_nodes + 255) / 256, 256, 0, st>>>(n_nodes, N, ref_id, node_lo, node_hi,
                                                         node_a, node_b, node_leaf);
  for (void* p : {(void*)N.lo, (void*)N.hi, (void*)N.start, (void*)N.count, (void*)N.left,
                  (void*)N.right, (void*)N.leaf, (void*)ord_a, (void*)ord_b, (void*)seg_s,
                  (void*)seg_e, (void*)seg_i, (void*)counters, (void*)isub, (void*)rank,
                  (void*)ref_id})
    cudaFreeAsync(p, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("nif_build_sah_dev");
  *n_nodes_out = n_nodes;
  return check_launch("nif_build_sah_dev");
}
