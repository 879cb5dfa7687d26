// GPU binned-SAH BVH build that reproduces the reference builder node for
// node (bvh.py:34-303 _build_sah; host twin: sah_builder.cpp).
//
// Level-synchronous: all nodes of one tree level are processed by one round
// of launches, each node by the unit its size calls for:
//   * small segments (<= 32 primitives): one warp, one primitive per lane;
//     bins are accumulated lane-per-bin in the reference's sequential order;
//   * medium segments (<= 8192): one CTA; warp-private shared-memory bins;
//   * huge segments: chunks of 2048 primitives spread over many CTAs, with
//     per-chunk partial bounds / bins reduced per segment, per-chunk left
//     counts and a stable chunked scatter.
// The bin sweeps and SAH costs (bvh.py:159-229) run lane-per-bin as warp
// scans; bounds unions are order-independent min/max (the sign of a zero
// bin bound never changes a surface area) and the costs use the reference's
// expression order (-fmad=false), so every cost, hence every split, is the
// reference's. Node bounds keep the first occurrence in segment order of
// each extreme (the reference's `if x < best` scans), so even the sign of a
// zero bound matches. Each segment is stably partitioned, so segment
// contents and order evolve exactly as in the reference's depth-first loop.
// The reference numbers nodes in depth-first processing order (the k-th
// split node in preorder gives its children ids 2k+1, 2k+2); build ids are
// handed out level by level (each level's ids are one contiguous range), so
// subtree internal-node counts (bottom-up) and preorder ranks (top-down)
// over those ranges recover the reference ids.
#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.h"
#include "kernels.h"
#include "nif_b200.h"
#include "status.h"

namespace nif {
namespace {

constexpr int kBT = 256;  // threads per CTA
constexpr int kWarps = kBT / 32;
constexpr int kMaxBins = 32;
constexpr int kSmall = 32;    // segments up to this size: one warp
constexpr int kHuge = 8192;   // segments above this size: chunked over CTAs
constexpr int kChunk = 2048;  // primitives per chunk of a huge segment

__device__ __forceinline__ double d_inf() { return __longlong_as_double(0x7ff0000000000000ll); }

struct SahIn {
  const double* lo;
  const double* hi;
  const double* ce;
  int64_t max_leaf;
  int n_bins;
  double c_trav, c_isect;
};

struct BfsNodes {  // indexed by build id
  double* lo;      // [cap][3]
  double* hi;
  int64_t* start;
  int64_t* count;
  int32_t* left;
  int32_t* right;
  uint8_t* leaf;
};

struct Seg {
  int32_t s, e, id;
};

struct Emit {       // next level's segment lists
  Seg* med;         // medium: med[j]
  Seg* small_top;   // small: small_top[-1 - j] (the same buffer, from the back)
  Seg* huge;        // huge: huge[j]
  int* ctr;         // [0] build ids handed out, [1] medium, [2] small, [3] huge
};

struct Orders {
  const int64_t* in;
  int64_t* out;    // split segments, for the next level
  int64_t* final;  // leaves
};

__device__ __forceinline__ int bin_of(double c, double cmin, double ext, int n_bins) {
  // bvh.py:148  b = int(n_bins * (ce[p, axis] - cmin) / ext), clamped
  long long b = (long long)((double)n_bins * (c - cmin) / ext);
  if (b >= n_bins) b = n_bins - 1;
  if (b < 0) b = 0;
  return (int)b;
}

__device__ __forceinline__ double surface(double ax, double ay, double az, double bx, double by,
                                          double bz) {
  const double ex = bx - ax, ey = by - ay, ez = bz - az;
  return 2.0 * (ex * ey + ey * ez + ez * ex);
}

// total order on doubles for the bin bounds
__device__ __forceinline__ unsigned long long dkey(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dval(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// ---- node bounds: value + position, ties to the earliest position ----------
struct VI {
  double v;
  long long i;
};
__device__ __forceinline__ void vi_min(VI& a, double v, long long i) {
  if (v < a.v || (!(a.v < v) && i < a.i)) a = {v, i};
}
__device__ __forceinline__ void vi_max(VI& a, double v, long long i) {
  if (v > a.v || (!(a.v > v) && i < a.i)) a = {v, i};
}

struct Bounds {
  VI b[6];      // lo xyz (min), hi xyz (max)
  double c[6];  // centroid min xyz, max xyz
};

__device__ __forceinline__ void bounds_init(Bounds& B) {
  for (int c = 0; c < 3; ++c) {
    B.b[c] = {d_inf(), 0x7fffffffffffffffll};
    B.b[3 + c] = {-d_inf(), 0x7fffffffffffffffll};
    B.c[c] = d_inf();
    B.c[3 + c] = -d_inf();
  }
}
__device__ __forceinline__ void bounds_add(Bounds& B, const SahIn& P, int64_t p, long long i) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    vi_min(B.b[c], P.lo[p * 3 + c], i);
    vi_max(B.b[3 + c], P.hi[p * 3 + c], i);
    const double cc = P.ce[p * 3 + c];
    B.c[c] = cc < B.c[c] ? cc : B.c[c];
    B.c[3 + c] = cc > B.c[3 + c] ? cc : B.c[3 + c];
  }
}
__device__ __forceinline__ void bounds_merge(Bounds& B, const Bounds& O) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    vi_min(B.b[c], O.b[c].v, O.b[c].i);
    vi_max(B.b[3 + c], O.b[3 + c].v, O.b[3 + c].i);
    B.c[c] = O.c[c] < B.c[c] ? O.c[c] : B.c[c];
    B.c[3 + c] = O.c[3 + c] > B.c[3 + c] ? O.c[3 + c] : B.c[3 + c];
  }
}
__device__ __forceinline__ void bounds_warp_reduce(Bounds& B) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Bounds O;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      O.b[c].v = __shfl_xor_sync(0xffffffffu, B.b[c].v, off);
      O.b[c].i = __shfl_xor_sync(0xffffffffu, B.b[c].i, off);
      O.c[c] = __shfl_xor_sync(0xffffffffu, B.c[c], off);
    }
    bounds_merge(B, O);
  }
}

// block-wide bounds of order[r0, r1); result valid in every thread
__device__ void block_bounds(const SahIn& P, const int64_t* order, int64_t r0, int64_t r1,
                             Bounds& out) {
  __shared__ Bounds s_bd[kWarps];
  Bounds B;
  bounds_init(B);
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kBT) bounds_add(B, P, order[i], i);
  bounds_warp_reduce(B);
  if ((threadIdx.x & 31) == 0) s_bd[threadIdx.x >> 5] = B;
  __syncthreads();
  out = s_bd[0];
  for (int w = 1; w < kWarps; ++w) bounds_merge(out, s_bd[w]);
  __syncthreads();
}

// ---- the split decision inputs of a node ------------------------------------
struct NodeGeo {
  double cmin[3], ext[3], sa;
  int axes;  // axes with a positive centroid extent, 0 if no split search
  int pad;   // explicit, so whole-struct copies read initialised bytes
};

__device__ __forceinline__ NodeGeo node_geo(const Bounds& B, int64_t count) {
  NodeGeo G;
  G.axes = 0;
  G.pad = 0;
  G.sa = 0.0;
  for (int a = 0; a < 3; ++a) {
    G.cmin[a] = B.c[a];
    G.ext[a] = B.c[3 + a] - B.c[a];
  }
  if (count > 1) {  // bvh.py:133-146
    G.sa = surface(B.b[0].v, B.b[1].v, B.b[2].v, B.b[3].v, B.b[4].v, B.b[5].v);
    if (G.sa > 1e-300)
      for (int a = 0; a < 3; ++a)
        if (G.ext[a] > 0.0) G.axes |= 1 << a;
  }
  return G;
}

// ---- lane-per-bin sweep of one axis (bvh.py:159-229) --------------------------
struct AxisBest {
  double cost;
  int k;  // -1: no valid split on this axis
  long long nl;
};

__device__ AxisBest warp_sweep(long long cnt, const double lo[3], const double hi[3], int nb,
                               double sa_node, double c_trav, double c_isect) {
  const int lane = threadIdx.x & 31;
  const double inf = d_inf();
  double la[3], lb[3], ra[3], rb[3];
  for (int c = 0; c < 3; ++c) {
    la[c] = ra[c] = lo[c];
    lb[c] = rb[c] = hi[c];
  }
  long long ln = cnt, rn = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const long long ol = __shfl_up_sync(0xffffffffu, ln, d);
    const long long orr = __shfl_down_sync(0xffffffffu, rn, d);
    if (lane >= d) ln += ol;
    if (lane + d < 32) rn += orr;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double a0 = __shfl_up_sync(0xffffffffu, la[c], d);
      const double b0 = __shfl_up_sync(0xffffffffu, lb[c], d);
      const double a1 = __shfl_down_sync(0xffffffffu, ra[c], d);
      const double b1 = __shfl_down_sync(0xffffffffu, rb[c], d);
      if (lane >= d) {
        la[c] = a0 < la[c] ? a0 : la[c];
        lb[c] = b0 > lb[c] ? b0 : lb[c];
      }
      if (lane + d < 32) {
        ra[c] = a1 < ra[c] ? a1 : ra[c];
        rb[c] = b1 > rb[c] ? b1 : rb[c];
      }
    }
  }
  const double left_sa = ln > 0 ? surface(la[0], la[1], la[2], lb[0], lb[1], lb[2]) : 0.0;
  const double right_sa = rn > 0 ? surface(ra[0], ra[1], ra[2], rb[0], rb[1], rb[2]) : 0.0;
  const long long nr = __shfl_down_sync(0xffffffffu, rn, 1);
  const double rsa = __shfl_down_sync(0xffffffffu, right_sa, 1);
  double cost = inf;
  if (lane < nb - 1 && ln != 0 && nr != 0)
    cost = c_trav + (left_sa * (double)ln + rsa * (double)nr) * c_isect / sa_node;
  int k = cost < inf ? lane : 64;
  if (k == 64) cost = inf;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double oc = __shfl_xor_sync(0xffffffffu, cost, off);
    const int ok = __shfl_xor_sync(0xffffffffu, k, off);
    if (oc < cost || (oc == cost && ok < k)) {
      cost = oc;
      k = ok;
    }
  }
  const long long nl = __shfl_sync(0xffffffffu, ln, k & 31);
  return {cost, k == 64 ? -1 : k, nl};
}

// bvh.py:230-275: split by the best bin, else halve when over the leaf size
struct Decision {
  int mode;  // 0 leaf, 1 bin split, 2 halve
  int axis, k;
  int pad;  // explicit, so whole-struct copies read initialised bytes
  long long nl;
};
__device__ __forceinline__ Decision decide(const SahIn& P, int64_t count, int axis,
                                           const AxisBest& b) {
  if (axis >= 0 && (count > P.max_leaf || b.cost < P.c_isect * (double)count))
    return {1, axis, b.k, 0, b.nl};
  if (count > P.max_leaf) return {2, -1, -1, 0, (long long)(count / 2)};
  return {0, -1, -1, 0, 0};
}

__device__ __forceinline__ void push_seg(const Emit& E, int s, int e, int id) {
  const Seg g{s, e, id};
  const int c = e - s;
  if (c <= kSmall)
    E.small_top[-1 - atomicAdd(&E.ctr[2], 1)] = g;
  else if (c <= kHuge)
    E.med[atomicAdd(&E.ctr[1], 1)] = g;
  else
    E.huge[atomicAdd(&E.ctr[3], 1)] = g;
}

__device__ __forceinline__ void emit_split(const Emit& E, const BfsNodes& N, const Seg& g,
                                           long long nl) {
  const int base = atomicAdd(&E.ctr[0], 2);
  N.leaf[g.id] = 0;
  N.left[g.id] = base;
  N.right[g.id] = base + 1;
  const int mid = g.s + (int)nl;
  push_seg(E, g.s, mid, base);
  push_seg(E, mid, g.e, base + 1);
}

__device__ __forceinline__ void write_node_bounds(const BfsNodes& N, int id, const Bounds& B) {
  for (int c = 0; c < 3; ++c) {
    N.lo[(int64_t)id * 3 + c] = B.b[c].v;
    N.hi[(int64_t)id * 3 + c] = B.b[3 + c].v;
  }
}

// ---- block-level binning ----------------------------------------------------
struct BinSmem {
  int cnt[kWarps][3][kMaxBins];
  unsigned long long lo[kWarps][3][kMaxBins][3];
  unsigned long long hi[kWarps][3][kMaxBins][3];
};

__device__ void bins_clear(BinSmem& S) {
  for (int e = threadIdx.x; e < kWarps * 3 * kMaxBins; e += kBT) {
    (&S.cnt[0][0][0])[e] = 0;
    for (int c = 0; c < 3; ++c) {
      (&S.lo[0][0][0][0])[e * 3 + c] = 0xffffffffffffffffull;
      (&S.hi[0][0][0][0])[e * 3 + c] = 0ull;
    }
  }
}

__device__ void bins_add(BinSmem& S, const SahIn& P, const int64_t* order, int64_t r0, int64_t r1,
                         const NodeGeo& G) {
  const int warp = threadIdx.x >> 5;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kBT) {
    const int64_t p = order[i];
    unsigned long long kl[3], kh[3];
    for (int c = 0; c < 3; ++c) {
      kl[c] = dkey(P.lo[p * 3 + c]);
      kh[c] = dkey(P.hi[p * 3 + c]);
    }
    for (int a = 0; a < 3; ++a) {
      if (!(G.axes & (1 << a))) continue;
      const int b = bin_of(P.ce[p * 3 + a], G.cmin[a], G.ext[a], P.n_bins);
      atomicAdd(&S.cnt[warp][a][b], 1);
      for (int c = 0; c < 3; ++c) {
        atomicMin(&S.lo[warp][a][b][c], kl[c]);
        atomicMax(&S.hi[warp][a][b][c], kh[c]);
      }
    }
  }
}

// lane k of warp a: bin k of axis a summed over the warp-private copies
__device__ __forceinline__ void bins_merge(const BinSmem& S, int a, int k, long long& cnt,
                                           unsigned long long kl[3], unsigned long long kh[3]) {
  cnt = 0;
  for (int c = 0; c < 3; ++c) {
    kl[c] = 0xffffffffffffffffull;
    kh[c] = 0ull;
  }
  for (int w = 0; w < kWarps; ++w) {
    cnt += S.cnt[w][a][k];
    for (int c = 0; c < 3; ++c) {
      kl[c] = S.lo[w][a][k][c] < kl[c] ? S.lo[w][a][k][c] : kl[c];
      kh[c] = S.hi[w][a][k][c] > kh[c] ? S.hi[w][a][k][c] : kh[c];
    }
  }
}

__device__ __forceinline__ void keys_to_bounds(long long cnt, const unsigned long long kl[3],
                                               const unsigned long long kh[3], double lo[3],
                                               double hi[3]) {
  for (int c = 0; c < 3; ++c) {
    lo[c] = cnt ? dval(kl[c]) : d_inf();
    hi[c] = cnt ? dval(kh[c]) : -d_inf();
  }
}

// stable block partition of order.in[r0, r1) by the chosen bin: left
// elements go to lbase.., right ones to rbase.. (absolute positions)
__device__ void block_partition(const SahIn& P, const Orders& O, int64_t r0, int64_t r1,
                                int64_t lbase, int64_t rbase, int axis, int kk, double cmin,
                                double ext) {
  __shared__ int s_scan[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t c0 = r0; c0 < r1; c0 += kBT) {
    const int64_t i = c0 + threadIdx.x;
    const bool valid = i < r1;
    int64_t p = 0;
    bool left = false;
    if (valid) {
      p = O.in[i];
      left = bin_of(P.ce[p * 3 + axis], cmin, ext, P.n_bins) <= kk;
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
        O.out[lbase + lw + __popc(bal & below)] = p;
      else
        O.out[rbase + rw + __popc(bar & below)] = p;
    }
    lbase += lt;
    rbase += rt;
    __syncthreads();
  }
}

// ============================================================================
// small segments: one warp each
// ============================================================================
__global__ void __launch_bounds__(kBT) sah_small_kernel(SahIn P, const Seg* list, int n_list,
                                                        Emit E, Orders O, BfsNodes N) {
  const int w = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (w >= n_list) return;  // whole warps leave together
  const Seg g = list[w];
  const int lane = threadIdx.x & 31;
  const int count = g.e - g.s;
  const bool valid = lane < count;
  const double inf = d_inf();
  int64_t p = 0;
  double lo[3], hi[3];
  Bounds B;
  bounds_init(B);
  if (valid) {
    p = O.in[g.s + lane];
    bounds_add(B, P, p, lane);
    for (int c = 0; c < 3; ++c) {
      lo[c] = P.lo[p * 3 + c];
      hi[c] = P.hi[p * 3 + c];
    }
  } else {
    for (int c = 0; c < 3; ++c) {
      lo[c] = inf;
      hi[c] = -inf;
    }
  }
  bounds_warp_reduce(B);
  if (lane == 0) write_node_bounds(N, g.id, B);
  const NodeGeo G = node_geo(B, count);
  AxisBest best{inf, -1, 0};
  int best_axis = -1;
  int packed = 0;
  if (G.axes) {
    for (int a = 0; a < 3; ++a)
      if (valid && (G.axes & (1 << a)))
        packed |= bin_of(P.ce[p * 3 + a], G.cmin[a], G.ext[a], P.n_bins) << (5 * a);
    // lane = bin; elements in segment order, as the reference's scan
    for (int a = 0; a < 3; ++a) {
      if (!(G.axes & (1 << a))) continue;
      long long cnt = 0;
      double blo[3] = {inf, inf, inf}, bhi[3] = {-inf, -inf, -inf};
      for (int j = 0; j < count; ++j) {
        const int bj = (__shfl_sync(0xffffffffu, packed, j) >> (5 * a)) & 31;
        double jl[3], jh[3];
        for (int c = 0; c < 3; ++c) {
          jl[c] = __shfl_sync(0xffffffffu, lo[c], j);
          jh[c] = __shfl_sync(0xffffffffu, hi[c], j);
        }
        if (bj != lane) continue;
        cnt += 1;
        for (int c = 0; c < 3; ++c) {
          if (jl[c] < blo[c]) blo[c] = jl[c];
          if (jh[c] > bhi[c]) bhi[c] = jh[c];
        }
      }
      // lanes >= n_bins hold empty bins (no element maps there)
      const AxisBest r = warp_sweep(cnt, blo, bhi, P.n_bins, G.sa, P.c_trav, P.c_isect);
      if (r.k >= 0 && r.cost < best.cost) {
        best = r;
        best_axis = a;
      }
    }
  }
  const Decision D = decide(P, count, best_axis, best);
  if (D.mode == 0) {
    if (valid) O.final[g.s + lane] = p;
    if (lane == 0) {
      N.leaf[g.id] = 1;
      N.start[g.id] = g.s;
      N.count[g.id] = count;
    }
    return;
  }
  if (D.mode == 2) {
    if (valid) O.out[g.s + lane] = p;
  } else {
    const bool left = valid && ((packed >> (5 * D.axis)) & 31) <= D.k;
    const unsigned bal = __ballot_sync(0xffffffffu, left);
    const unsigned bar = __ballot_sync(0xffffffffu, valid && !left);
    const unsigned below = (1u << lane) - 1u;
    if (valid)
      O.out[g.s + (left ? __popc(bal & below) : (int)D.nl + __popc(bar & below))] = p;
  }
  if (lane == 0) emit_split(E, N, g, D.nl);
}

// ============================================================================
// medium segments: one CTA each
// ============================================================================
__global__ void __launch_bounds__(kBT) sah_medium_kernel(SahIn P, const Seg* list, Emit E,
                                                         Orders O, BfsNodes N) {
  __shared__ BinSmem S;
  __shared__ AxisBest s_best[3];
  __shared__ Decision s_dec;
  const Seg g = list[blockIdx.x];
  const int64_t count = g.e - g.s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  bins_clear(S);
  Bounds B;
  block_bounds(P, O.in, g.s, g.e, B);  // (syncs: also orders the clear)
  const NodeGeo G = node_geo(B, count);
  if (threadIdx.x == 0) write_node_bounds(N, g.id, B);
  if (G.axes) {
    bins_add(S, P, O.in, g.s, g.e, G);
    __syncthreads();
    if (warp < 3) {
      AxisBest r{d_inf(), -1, 0};
      if (G.axes & (1 << warp)) {
        long long cnt;
        unsigned long long kl[3], kh[3];
        double lo[3], hi[3];
        bins_merge(S, warp, lane < P.n_bins ? lane : 0, cnt, kl, kh);
        if (lane >= P.n_bins) cnt = 0;
        keys_to_bounds(cnt, kl, kh, lo, hi);
        r = warp_sweep(cnt, lo, hi, P.n_bins, G.sa, P.c_trav, P.c_isect);
      }
      if (lane == 0) s_best[warp] = r;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    AxisBest best{d_inf(), -1, 0};
    int best_axis = -1;
    if (G.axes)
      for (int a = 0; a < 3; ++a)
        if (s_best[a].k >= 0 && s_best[a].cost < best.cost) {
          best = s_best[a];
          best_axis = a;
        }
    s_dec = decide(P, count, best_axis, best);
  }
  __syncthreads();
  const Decision D = s_dec;
  if (D.mode == 0) {
    for (int64_t i = g.s + threadIdx.x; i < g.e; i += kBT) O.final[i] = O.in[i];
    if (threadIdx.x == 0) {
      N.leaf[g.id] = 1;
      N.start[g.id] = g.s;
      N.count[g.id] = count;
    }
    return;
  }
  if (D.mode == 2) {
    for (int64_t i = g.s + threadIdx.x; i < g.e; i += kBT) O.out[i] = O.in[i];
  } else {
    block_partition(P, O, g.s, g.e, g.s, g.s + D.nl, D.axis, D.k, G.cmin[D.axis],
                    G.ext[D.axis]);
  }
  if (threadIdx.x == 0) emit_split(E, N, g, D.nl);
}

// ============================================================================
// huge segments: chunked over CTAs
// ============================================================================
struct Chunk {
  int32_t seg, r0, r1;
};

struct HugeState {
  const Seg* segs;       // this level's huge segments
  const Chunk* chunks;   // [n_chunks]
  const int32_t* first;  // [n_segs] first chunk of each segment
  const int32_t* nch;    // [n_segs]
  Bounds* part;          // [n_chunks]
  NodeGeo* geo;          // [n_segs]
  Decision* dec;         // [n_segs]
  int* pcnt;             // [n_chunks][3][kMaxBins]
  unsigned long long* plo;  // [n_chunks][3][kMaxBins][3]
  unsigned long long* phi;
  int32_t* chunk_nl;     // [n_chunks]
};

__global__ void __launch_bounds__(kBT) huge_bounds_kernel(SahIn P, HugeState H, Orders O) {
  const Chunk ch = H.chunks[blockIdx.x];
  Bounds B;
  block_bounds(P, O.in, ch.r0, ch.r1, B);
  if (threadIdx.x == 0) H.part[blockIdx.x] = B;
}

__global__ void __launch_bounds__(32) huge_geo_kernel(SahIn P, HugeState H, BfsNodes N) {
  const Seg g = H.segs[blockIdx.x];
  const int f = H.first[blockIdx.x], nc = H.nch[blockIdx.x];
  Bounds B;
  bounds_init(B);
  for (int j = threadIdx.x; j < nc; j += 32) bounds_merge(B, H.part[f + j]);
  bounds_warp_reduce(B);
  if (threadIdx.x == 0) {
    write_node_bounds(N, g.id, B);
    H.geo[blockIdx.x] = node_geo(B, g.e - g.s);
  }
}

__global__ void __launch_bounds__(kBT) huge_bin_kernel(SahIn P, HugeState H, Orders O) {
  __shared__ BinSmem S;
  const Chunk ch = H.chunks[blockIdx.x];
  const NodeGeo G = H.geo[ch.seg];
  if (!G.axes) return;
  bins_clear(S);
  __syncthreads();
  bins_add(S, P, O.in, ch.r0, ch.r1, G);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < 3 && lane < P.n_bins && (G.axes & (1 << warp))) {
    long long cnt;
    unsigned long long kl[3], kh[3];
    bins_merge(S, warp, lane, cnt, kl, kh);
    const int64_t e = ((int64_t)blockIdx.x * 3 + warp) * kMaxBins + lane;
    H.pcnt[e] = (int)cnt;
    for (int c = 0; c < 3; ++c) {
      H.plo[e * 3 + c] = kl[c];
      H.phi[e * 3 + c] = kh[c];
    }
  }
}

__global__ void __launch_bounds__(96) huge_decide_kernel(SahIn P, HugeState H, Emit E,
                                                         BfsNodes N) {
  __shared__ AxisBest s_best[3];
  const int s = blockIdx.x;
  const Seg g = H.segs[s];
  const NodeGeo G = H.geo[s];
  const int lane = threadIdx.x & 31, a = threadIdx.x >> 5;
  AxisBest r{d_inf(), -1, 0};
  if (G.axes & (1 << a)) {
    long long cnt = 0;
    unsigned long long kl[3] = {~0ull, ~0ull, ~0ull}, kh[3] = {0ull, 0ull, 0ull};
    if (lane < P.n_bins) {
      const int f = H.first[s], nc = H.nch[s];
      for (int j = 0; j < nc; ++j) {
        const int64_t e = ((int64_t)(f + j) * 3 + a) * kMaxBins + lane;
        cnt += H.pcnt[e];
        for (int c = 0; c < 3; ++c) {
          const unsigned long long l = H.plo[e * 3 + c], h = H.phi[e * 3 + c];
          kl[c] = l < kl[c] ? l : kl[c];
          kh[c] = h > kh[c] ? h : kh[c];
        }
      }
    }
    double lo[3], hi[3];
    keys_to_bounds(cnt, kl, kh, lo, hi);
    r = warp_sweep(cnt, lo, hi, P.n_bins, G.sa, P.c_trav, P.c_isect);
  }
  if (lane == 0) s_best[a] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    AxisBest best{d_inf(), -1, 0};
    int best_axis = -1;
    if (G.axes)
      for (int x = 0; x < 3; ++x)
        if (s_best[x].k >= 0 && s_best[x].cost < best.cost) {
          best = s_best[x];
          best_axis = x;
        }
    const Decision D = decide(P, g.e - g.s, best_axis, best);
    H.dec[s] = D;
    // huge segments exceed any leaf size, so D.mode != 0
    emit_split(E, N, g, D.nl);
  }
}

__global__ void __launch_bounds__(kBT) huge_count_kernel(SahIn P, HugeState H, Orders O) {
  __shared__ int s_n[kWarps];
  const Chunk ch = H.chunks[blockIdx.x];
  const Decision D = H.dec[ch.seg];
  if (D.mode != 1) return;
  const NodeGeo G = H.geo[ch.seg];
  int n = 0;
  for (int64_t i = ch.r0 + threadIdx.x; i < ch.r1; i += kBT)
    n += bin_of(P.ce[O.in[i] * 3 + D.axis], G.cmin[D.axis], G.ext[D.axis], P.n_bins) <= D.k;
  n = __reduce_add_sync(0xffffffffu, n);
  if ((threadIdx.x & 31) == 0) s_n[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kWarps; ++w) t += s_n[w];
    H.chunk_nl[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kBT) huge_scatter_kernel(SahIn P, HugeState H, Orders O) {
  __shared__ int s_before;
  const Chunk ch = H.chunks[blockIdx.x];
  const Decision D = H.dec[ch.seg];
  if (D.mode == 2) {
    for (int64_t i = ch.r0 + threadIdx.x; i < ch.r1; i += kBT) O.out[i] = O.in[i];
    return;
  }
  const NodeGeo G = H.geo[ch.seg];
  const Seg g = H.segs[ch.seg];
  if (threadIdx.x < 32) {
    int t = 0;
    for (int j = H.first[ch.seg] + threadIdx.x; j < (int)blockIdx.x; j += 32) t += H.chunk_nl[j];
    t = __reduce_add_sync(0xffffffffu, t);
    if (threadIdx.x == 0) s_before = t;
  }
  __syncthreads();
  const int64_t before = s_before;
  block_partition(P, O, ch.r0, ch.r1, g.s + before, g.s + D.nl + (ch.r0 - g.s - before), D.axis,
                  D.k, G.cmin[D.axis], G.ext[D.axis]);
}

// ============================================================================
// reference numbering
// ============================================================================
__global__ void iota_kernel(int64_t* o, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = i;
}

// bottom-up: internal-node count of each subtree (ids of one level)
__global__ void sah_isub_kernel(int v0, int v1, BfsNodes N, int32_t* isub) {
  const int v = v0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= v1) return;
  isub[v] = N.leaf[v] ? 0 : 1 + isub[N.left[v]] + isub[N.right[v]];
}

// top-down: preorder rank among internal nodes -> the reference's node ids
__global__ void sah_rank_kernel(int v0, int v1, BfsNodes N, const int32_t* isub, int32_t* rank,
                                int32_t* ref_id) {
  const int v = v0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= v1 || N.leaf[v]) return;
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

// one device allocation carved into the build's arrays
struct Arena {
  char* base = nullptr;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    T* p = (T*)(base ? base + off : nullptr);
    off += (count * sizeof(T) + 255) / 256 * 256;
    return p;
  }
};

}  // namespace
}  // namespace nif

namespace nif {
namespace {

// every device array of one build, carved from one workspace
struct Work {
  BfsNodes N;
  Seg *lists[2], *huge[2];
  int64_t *ord_a, *ord_b;
  int* ctr;
  int32_t *isub, *rank, *ref_id;
  HugeState H;
  Chunk* chunks;
  int32_t *first, *nch;
};

size_t carve(Arena& A, int64_t n, Work& W) {
  const int64_t cap = 2 * n;
  const int64_t max_huge = n / kHuge + 2;  // huge segments of one level
  const int64_t max_chunks = n / kChunk + max_huge + 1;
  A.off = 0;
  W.N = {A.take<double>(cap * 3), A.take<double>(cap * 3), A.take<int64_t>(cap),
         A.take<int64_t>(cap),    A.take<int32_t>(cap),    A.take<int32_t>(cap),
         A.take<uint8_t>(cap)};
  W.lists[0] = A.take<Seg>(n + 2);
  W.lists[1] = A.take<Seg>(n + 2);
  W.huge[0] = A.take<Seg>(max_huge);
  W.huge[1] = A.take<Seg>(max_huge);
  W.ord_a = A.take<int64_t>(n);
  W.ord_b = A.take<int64_t>(n);
  W.ctr = A.take<int>(4);
  W.isub = A.take<int32_t>(cap);
  W.rank = A.take<int32_t>(cap);
  W.ref_id = A.take<int32_t>(cap);
  W.chunks = A.take<Chunk>(max_chunks);
  W.first = A.take<int32_t>(max_huge);
  W.nch = A.take<int32_t>(max_huge);
  W.H.part = A.take<Bounds>(max_chunks);
  W.H.geo = A.take<NodeGeo>(max_huge);
  W.H.dec = A.take<Decision>(max_huge);
  W.H.pcnt = A.take<int>(max_chunks * 3 * kMaxBins);
  W.H.plo = A.take<unsigned long long>(max_chunks * 3 * kMaxBins * 3);
  W.H.phi = A.take<unsigned long long>(max_chunks * 3 * kMaxBins * 3);
  W.H.chunk_nl = A.take<int32_t>(max_chunks);
  return A.off;
}

}  // namespace
}  // namespace nif

using namespace nif;

extern "C" size_t nif_build_sah_workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  Arena A;
  Work W;
  return carve(A, n, W) + 256;
}

extern "C" int nif_build_sah_dev(const double* lo, const double* hi, const double* ce, int64_t n,
                                 int64_t max_leaf, int64_t n_bins, double c_trav, double c_isect,
                                 double* node_lo, double* node_hi, int64_t* node_a,
                                 int64_t* node_b, uint8_t* node_leaf, int64_t* order,
                                 int64_t* n_nodes_out, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  if (n <= 0) return fail(NIF_ERR_VALUE, "cannot build a tree over zero primitives");
  if (n_bins < 2 || n_bins > kMaxBins || max_leaf < 1)
    return fail(NIF_ERR_VALUE, "bad SAH parameters (2 <= n_bins <= %d)", kMaxBins);
  if (n >= (int64_t)1 << 30) return fail(NIF_ERR_VALUE, "GPU SAH build supports < 2^30 primitives");
  if (max_leaf >= kHuge) return fail(NIF_ERR_VALUE, "max_leaf must be below %d", kHuge);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t need = nif_build_sah_workspace_bytes(n);
  Arena A;
  Work W;
  void* owned = nullptr;
  if (workspace == nullptr) {
    if (cudaMallocAsync(&owned, need, st) != cudaSuccess)
      return fail(NIF_ERR_CUDA, "GPU SAH build: device allocation of %zu bytes failed", need);
    workspace = owned;
  } else if (workspace_bytes < need) {
    return fail(NIF_ERR_VALUE, "SAH workspace of %zu bytes is below the %zu required",
                workspace_bytes, need);
  }
  A.base = (char*)(((uintptr_t)workspace + 255) / 256 * 256);
  carve(A, n, W);
  BfsNodes N = W.N;
  Seg** lists = W.lists;
  Seg** huge = W.huge;
  int64_t *ord_a = W.ord_a, *ord_b = W.ord_b;
  int* ctr = W.ctr;
  int32_t *isub = W.isub, *rank = W.rank, *ref_id = W.ref_id;
  HugeState H = W.H;
  Chunk* chunks = W.chunks;
  int32_t *first = W.first, *nch = W.nch;
  H.chunks = chunks;
  H.first = first;
  H.nch = nch;
  SahIn P{lo, hi, ce, max_leaf, (int)n_bins, c_trav, c_isect};

  iota_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ord_a, n);
  // level 0: the root segment in its size class
  const Seg root{0, (int32_t)n, 0};
  int n_med = 0, n_small = 0, n_huge = 0;
  std::vector<Seg> h_huge;
  if (n <= kSmall) {
    cudaMemcpyAsync(lists[0] + (n + 2) - 1, &root, sizeof(Seg), cudaMemcpyHostToDevice, st);
    n_small = 1;
  } else if (n <= kHuge) {
    cudaMemcpyAsync(lists[0], &root, sizeof(Seg), cudaMemcpyHostToDevice, st);
    n_med = 1;
  } else {
    cudaMemcpyAsync(huge[0], &root, sizeof(Seg), cudaMemcpyHostToDevice, st);
    h_huge.push_back(root);
    n_huge = 1;
  }
  int h_ctr[4] = {1, 0, 0, 0};
  cudaMemcpyAsync(ctr, h_ctr, sizeof(h_ctr), cudaMemcpyHostToDevice, st);
  std::vector<int> id_end{1};  // level L's ids are [id_end[L-1], id_end[L]) (level 0: [0, 1))
  const bool prof = std::getenv("NIF_SAH_PROFILE") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (prof) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
  }
  std::vector<Chunk> h_chunks;
  std::vector<int32_t> h_first, h_nch;
  int cur = 0, level = 0;
  int64_t* oin = ord_a;
  int64_t* oout = ord_b;
  while (n_med + n_small + n_huge > 0) {
    const int nxt = cur ^ 1;
    Emit E{lists[nxt], lists[nxt] + (n + 2), huge[nxt], ctr};
    Orders O{oin, oout, order};
    cudaMemsetAsync(ctr + 1, 0, 3 * sizeof(int), st);
    if (prof) cudaEventRecord(e0, st);
    if (n_huge) {
      h_chunks.clear();
      h_first.clear();
      h_nch.clear();
      for (int s = 0; s < n_huge; ++s) {
        const Seg g = h_huge[s];
        h_first.push_back((int32_t)h_chunks.size());
        for (int32_t r = g.s; r < g.e; r += kChunk)
          h_chunks.push_back({s, r, r + kChunk < g.e ? r + kChunk : g.e});
        h_nch.push_back((int32_t)h_chunks.size() - h_first.back());
      }
      const int nc = (int)h_chunks.size();
      cudaMemcpyAsync(chunks, h_chunks.data(), nc * sizeof(Chunk), cudaMemcpyHostToDevice, st);
      cudaMemcpyAsync(first, h_first.data(), n_huge * 4, cudaMemcpyHostToDevice, st);
      cudaMemcpyAsync(nch, h_nch.data(), n_huge * 4, cudaMemcpyHostToDevice, st);
      H.segs = huge[cur];
      huge_bounds_kernel<<<nc, kBT, 0, st>>>(P, H, O);
      huge_geo_kernel<<<n_huge, 32, 0, st>>>(P, H, N);
      huge_bin_kernel<<<nc, kBT, 0, st>>>(P, H, O);
      huge_decide_kernel<<<n_huge, 96, 0, st>>>(P, H, E, N);
      huge_count_kernel<<<nc, kBT, 0, st>>>(P, H, O);
      huge_scatter_kernel<<<nc, kBT, 0, st>>>(P, H, O);
    }
    if (n_med) sah_medium_kernel<<<n_med, kBT, 0, st>>>(P, lists[cur], E, O, N);
    if (n_small)
      sah_small_kernel<<<(n_small + kWarps - 1) / kWarps, kBT, 0, st>>>(
          P, lists[cur] + (n + 2) - n_small, n_small, E, O, N);
    if (prof) cudaEventRecord(e1, st);
    cudaMemcpyAsync(h_ctr, ctr, sizeof(h_ctr), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) {
      if (owned) cudaFreeAsync(owned, st);
      return check_launch("nif_build_sah_dev(level)");
    }
    if (prof) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      std::fprintf(stderr, "sah level %d: huge %d med %d small %d, %.3f ms\n", level, n_huge,
                   n_med, n_small, ms);
    }
    id_end.push_back(h_ctr[0]);
    n_med = h_ctr[1];
    n_small = h_ctr[2];
    n_huge = h_ctr[3];
    if (n_huge) {
      h_huge.resize(n_huge);
      cudaMemcpyAsync(h_huge.data(), huge[nxt], n_huge * sizeof(Seg), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
    }
    cur = nxt;
    int64_t* t = oin;
    oin = oout;
    oout = t;
    ++level;
  }
  if (prof) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  const int n_nodes = id_end.back();
  // id_end has one entry per processed level plus the trailing (empty) one
  const int n_levels = (int)id_end.size() - 1;
  auto range = [&](int L, int& v0, int& v1) {
    v0 = L == 0 ? 0 : id_end[L - 1];
    v1 = id_end[L];
  };
  for (int L = n_levels - 1; L >= 0; --L) {
    int v0, v1;
    range(L, v0, v1);
    if (v1 > v0) sah_isub_kernel<<<(v1 - v0 + 255) / 256, 256, 0, st>>>(v0, v1, N, isub);
  }
  const int zero = 0;
  cudaMemcpyAsync(rank, &zero, 4, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(ref_id, &zero, 4, cudaMemcpyHostToDevice, st);
  for (int L = 0; L < n_levels; ++L) {
    int v0, v1;
    range(L, v0, v1);
    if (v1 > v0)
      sah_rank_kernel<<<(v1 - v0 + 255) / 256, 256, 0, st>>>(v0, v1, N, isub, rank, ref_id);
  }
  sah_emit_kernel<<<(n_nodes + 255) / 256, 256, 0, st>>>(n_nodes, N, ref_id, node_lo, node_hi,
                                                         node_a, node_b, node_leaf);
  const int rc = check_launch("nif_build_sah_dev");
  if (owned) cudaFreeAsync(owned, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("nif_build_sah_dev");
  *n_nodes_out = n_nodes;
  if (prof)
    std::fprintf(stderr, "sah build: %d levels, %.3f ms wall\n", n_levels,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                           t_start).count());
  return rc;
}
