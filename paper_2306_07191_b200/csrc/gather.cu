// Phase 1 of the split visibility pass as ONE kernel (bvh.py:772-901
// _k_gather_queries + renderer.py:613-644 gather_queries):
//   per ray: fp64 top-level classification of every object (slab test with
//   the ray's reciprocal direction computed once, containment against
//   per-object pre-widened bounds), hybrid any-hit for objects routed to
//   their own trees, then ordered compaction into the outer / inner record
//   queues through a decoupled look-back scan over 128-ray tiles, so rays
//   are read from HBM once and classified once.
// Results are bit-identical to the reference's classification: 1.0 / d,
// lo - tol and hi + tol are deterministic IEEE operations, so hoisting them
// out of the object loop changes no value. Compiled with -fmad=false.
//
// Coordinates: the interleaved API output (QueryRecords, fp64) uses the
// reference's fp64 transforms; the hot-path queues store fp32 coordinates,
// evaluated as fp32 atan2/acos of the fp64 box-relative vector (the
// classification and degenerate test stay fp64). The per-ray direction
// coordinates are computed once per ray, not once per record.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "common.h"
#include "geom.cuh"
#include "kernels.h"
#include "nif_b200.h"
#include "status.h"

namespace nif {
namespace {

constexpr int kThreads = 256;    // rays per tile (one per thread)
#ifndef NIF_BUNDLE_SIGN
#define NIF_BUNDLE_SIGN 1  // warp-bundle cull: two sign-selected products per axis instead of eight
#endif
#ifndef NIF_NF_LEAN
#define NIF_NF_LEAN 1  // slab_nf / classify_nf without the first-axis compares and short circuits (A/B)
#endif
#ifndef NIF_EMIT_UNIFIED
#define NIF_EMIT_UNIFIED 1  // hot-path record emission: one path for outer and inner records (A/B)
#endif
#ifndef NIF_SLAB_NF
#define NIF_SLAB_NF 1  // hot path: sign-selected slab planes (slab_nf) for rays with |d_a| > 1e-20
#endif
#ifndef NIF_GATHER_MINB
#define NIF_GATHER_MINB 3        // resident CTAs per SM the register budget targets
#endif
constexpr int kMaxObjFused = 32; // 2 bits per object in a 64-bit mask

struct ObjC {
  double lo[3], hi[3];  // box
  double lt[3], ht[3];  // lo - tol, hi + tol  (geometry.py:260-262)
  double c[3];          // 0.5 * (lo + hi)     (geometry.py:275-277, 295-297)
  double hn;            // |half diagonal|      (geometry.py:302-305)
  int id, route, root;
  float hinv;           // 1 / (float)hn: the hot path's fp32 r' = |o - c| / hn
};

struct RayX {
  double ox, oy, oz, dx, dy, dz, tmax;
  double ix, iy, iz;  // 1 / d where d != 0
};

// geometry.py:152-196 with the reciprocal hoisted (inv = 1.0 / d is the
// same value the reference recomputes per box).
__device__ __forceinline__ Hit3 slab(const RayX& r, const ObjC& b) {
  double t0 = -CUDART_INF, t1 = CUDART_INF;
  if (r.dx != 0.0) {
    double ta = (b.lo[0] - r.ox) * r.ix, tb = (b.hi[0] - r.ox) * r.ix;
    if (ta > tb) { double q = ta; ta = tb; tb = q; }
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  } else if (r.ox < b.lo[0] || r.ox > b.hi[0]) {
    return {false, 0.0, 0.0};
  }
  if (r.dy != 0.0) {
    double ta = (b.lo[1] - r.oy) * r.iy, tb = (b.hi[1] - r.oy) * r.iy;
    if (ta > tb) { double q = ta; ta = tb; tb = q; }
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  } else if (r.oy < b.lo[1] || r.oy > b.hi[1]) {
    return {false, 0.0, 0.0};
  }
  if (r.dz != 0.0) {
    double ta = (b.lo[2] - r.oz) * r.iz, tb = (b.hi[2] - r.oz) * r.iz;
    if (ta > tb) { double q = ta; ta = tb; tb = q; }
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  } else if (r.oz < b.lo[2] || r.oz > b.hi[2]) {
    return {false, 0.0, 0.0};
  }
  if (t1 < t0 || t1 < 0.0) return {false, t0, t1};
  return {true, t0, t1};
}

// slab() for rays with every |d_a| > 1e-20 (finite, nonzero reciprocals):
// the entry plane of each axis is known from the reciprocal's sign, so the
// per-axis swap (a DSETP and four 32-bit selects per axis) becomes a
// shared-memory load at a per-ray offset. Exact: with finite operands
// (lo - o) * inv <= (hi - o) * inv for inv > 0 and >= for inv < 0 (rounding
// is monotone), so the reference's swap picks the same pair; where the two
// are equal they are the same bits (a zero here is lo == hi == o, and
// (+0) * inv has one sign). lh points at ObjC::lo (hi follows it);
// s3 = 3 * [inv_a < 0] packed per axis (bits 0-1 x, 2-3 y, 4-5 z).
__device__ __forceinline__ Hit3 slab_nf(const RayX& r, const ObjC& b, int s3) {
  const double* lh = b.lo;
  const int sx = s3 & 3, sy = (s3 >> 2) & 3, sz = s3 >> 4;
#if NIF_NF_LEAN
  // first axis: the reference's max(-inf, ta) / min(+inf, tb) are ta / tb
  // (no NaN here: finite origin and reciprocal)
  double t0 = (lh[sx] - r.ox) * r.ix, t1 = (lh[3 - sx] - r.ox) * r.ix;
#else
  double t0 = -CUDART_INF, t1 = CUDART_INF;
  {
    const double ta = (lh[sx] - r.ox) * r.ix, tb = (lh[3 - sx] - r.ox) * r.ix;
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  }
#endif
  {
    const double ta = (lh[1 + sy] - r.oy) * r.iy, tb = (lh[4 - sy] - r.oy) * r.iy;
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  }
  {
    const double ta = (lh[2 + sz] - r.oz) * r.iz, tb = (lh[5 - sz] - r.oz) * r.iz;
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  }
  return {!((t1 < t0) | (t1 < 0.0)), t0, t1};
}

__device__ __forceinline__ int classify_nf(const RayX& r, const ObjC& b, bool test_box,
                                           double tol, int s3) {
  const Hit3 h = slab_nf(r, b, s3);
#if NIF_NF_LEAN
  // the same predicates without short-circuit branches (no side effects)
  if (test_box & !(h.hit & (h.t0 <= r.tmax) & (h.t1 >= -tol))) return 0;
  const bool inside = (b.lt[0] <= r.ox) & (r.ox <= b.ht[0]) & (b.lt[1] <= r.oy) &
                      (r.oy <= b.ht[1]) & (b.lt[2] <= r.oz) & (r.oz <= b.ht[2]);
  return inside ? 2 : ((h.hit & (h.t0 > 0.0) & (h.t0 < r.tmax)) ? 1 : 0);
#else
  if (test_box && !(h.hit && h.t0 <= r.tmax && h.t1 >= -tol)) return 0;
  if (b.lt[0] <= r.ox && r.ox <= b.ht[0] && b.lt[1] <= r.oy && r.oy <= b.ht[1] &&
      b.lt[2] <= r.oz && r.oz <= b.ht[2])
    return 2;
  if (h.hit && h.t0 > 0.0 && h.t0 < r.tmax) return 1;
  return 0;
#endif
}

// 0 none, 1 outer, 2 inner (see trace.cu classify())
__device__ __forceinline__ int classify_obj(const RayX& r, const ObjC& b, bool test_box,
                                            double tol, double* t0) {
  const Hit3 h = slab(r, b);
  if (test_box && !(h.hit && h.t0 <= r.tmax && h.t1 >= -tol)) return 0;
  if (b.lt[0] <= r.ox && r.ox <= b.ht[0] && b.lt[1] <= r.oy && r.oy <= b.ht[1] &&
      b.lt[2] <= r.oz && r.oz <= b.ht[2])
    return 2;
  if (h.hit && h.t0 > 0.0 && h.t0 < r.tmax) {
    *t0 = h.t0;
    return 1;
  }
  return 0;
}

// Hot-path spherical map (geometry.py:233-246) with minimax polynomials in
// place of atan2f / acosf (a quarter of the gather's instructions):
//   atan(a) = a * P(a^2) on [0, 1], |err| < 1e-7 rad (degree 7 in a^2);
//   acos(z) = sqrt(1 - z) * Q(z) on [0, 1], |err| < 3e-8 (degree 7),
// with the quadrant / sign logic of atan2 (signed zeros included, so
// atan2(+0, -0) = pi as in the reference) and acos(-z) = pi - acos(z).
// The queue coordinates stay within 2e-7 of the fp64 reference map.
__device__ __forceinline__ float fast_atan2(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  const float a = mx > 0.f ? __fdividef(mn, mx) : 0.f;
  const float s = a * a;
  float p = -0.0047803754f;
  p = fmaf(p, s, 0.02455685f);
  p = fmaf(p, s, -0.059904344f);
  p = fmaf(p, s, 0.09942734f);
  p = fmaf(p, s, -0.14029412f);
  p = fmaf(p, s, 0.19971374f);
  p = fmaf(p, s, -0.33332095f);
  p = fmaf(p, s, 0.99999994f);
  float r = p * a;
  if (ay > ax) r = 1.57079632679f - r;
  if (signbit(x)) r = 3.14159265359f - r;
  return copysignf(r, y);
}

__device__ __forceinline__ float fast_acos(float z) {
  const float za = fminf(fabsf(z), 1.0f);
  float q = -0.0012628123f;
  q = fmaf(q, za, 0.006671229f);
  q = fmaf(q, za, -0.017089725f);
  q = fmaf(q, za, 0.030892996f);
  q = fmaf(q, za, -0.050174695f);
  q = fmaf(q, za, 0.08897905f);
  q = fmaf(q, za, -0.2145988f);
  q = fmaf(q, za, 1.5707963f);
  const float x = 1.0f - za;
  // sqrt(x) as x * rsqrt(x): MUFU.RSQ alone (within 2 ulp; the map's
  // tolerance is 2e-7), exact 0 at the pole
  const float r = (x > 0.f ? x * rsqrtf(x) : 0.f) * q;
  return z < 0.f ? 3.14159265359f - r : r;
}

// ninv: 1 / |(x, y, z)| (1 for unit directions)
__device__ __forceinline__ void sph32f(float x, float y, float z, float ninv, float* u, float* v) {
  float uu = fmaf(fast_atan2(y, x), 0.5f / CUDART_PI_F, 0.5f);
  if (uu >= 1.0f) uu -= 1.0f;
  else if (uu < 0.0f) uu += 1.0f;
  const float zz = fminf(fmaxf(z * ninv, -1.0f), 1.0f);
  *u = uu;
  *v = fast_acos(zz) * (1.0f / CUDART_PI_F);
}

// The reference's degenerate test sqrt(r.r) < 1e-9 in fp64, exactly,
// without the square root: the squared norm is the reference's expression,
// and since the fp64 sqrt is correctly rounded and monotone,
// sqrt(r2) < 1e-9  <=>  r2 < T for T the least double with sqrt(T) >= 1e-9,
// which is the double nearest 1e-18 (0x1.2725dd1d243acp-60; checked with a
// nextafter search around it). The returned norm is fp32 (it only feeds
// fp32 coordinates).
__device__ __forceinline__ bool degenerate_f32(double rx, double ry, double rz, float* rn,
                                               float* rinv) {
  static_assert(kDegenerateRadius == 1e-9, "threshold below is derived for 1e-9");
  const double r2 = rx * rx + ry * ry + rz * rz;
  // fp32 norm and inverse from one MUFU.RSQ (within 2 ulp; both only feed
  // fp32 coordinates); not used for a degenerate record (r2 < 1e-18 keeps
  // (float)r2 a normal number otherwise)
  const float r2f = (float)r2;
  const float ri = rsqrtf(r2f);
  *rn = r2f * ri;
  *rinv = ri;
  return r2 < 1e-18;
}

constexpr uint64_t kFlagA = 1ull << 62;
constexpr uint64_t kFlagP = 2ull << 62;
constexpr uint64_t kCntMask = (1ull << 31) - 1;

__device__ __forceinline__ uint64_t pack(uint64_t flag, uint64_t o, uint64_t i) {
  return flag | (o << 31) | i;
}

// Conservative fp32 prefilter of the top-level candidate test. The fp32
// slab interval is widened by dt = 1e-5 * S * max|1/d| (S bounds every
// coordinate involved), which exceeds the fp32 rounding error of each slab
// bound (< 3 * 2^-24 * S * |1/d_a|) fifty-fold; an object it rejects can
// therefore never pass the reference's fp64 test _window_hit(-tol, tmax),
// and every object it accepts is re-classified exactly in fp64. Used only
// for multi-object scenes (the single-object root is never box-tested) and
// rays with no |d_a| below 1e-20 (fp32 reciprocal overflow).
struct RayF {
  float ix, iy, iz, ox_i, oy_i, oz_i, dt, tmax_ru;
  float ox, oy, oz;
};

__device__ __forceinline__ bool prefilter(const RayF& q, const float4 lo, const float4 hi) {
  const float ax = fmaf(lo.x, q.ix, q.ox_i), bx = fmaf(hi.x, q.ix, q.ox_i);
  const float ay = fmaf(lo.y, q.iy, q.oy_i), by = fmaf(hi.y, q.iy, q.oy_i);
  const float az = fmaf(lo.z, q.iz, q.oz_i), bz = fmaf(hi.z, q.iz, q.oz_i);
  const float t0 = fmaxf(fmaxf(fminf(ax, bx), fminf(ay, by)), fminf(az, bz)) - q.dt;
  const float t1 = fminf(fminf(fmaxf(ax, bx), fmaxf(ay, by)), fmaxf(az, bz)) + q.dt;
  return t1 >= t0 && t1 >= -1e-6f && t0 <= q.tmax_ru;
}

// Warp-level conservative culling. With origins in [ol, oh], reciprocal
// directions in [il, ih] (one sign per axis) and t_max <= tm over the
// warp, interval arithmetic bounds every ray's slab entry from below (E)
// and exit from above (X) per box; a box is a candidate for some ray only if
// max_a E_a <= min_a X_a, min_a X_a >= -tol and max_a E_a <= tm, which is
// what the per-ray candidate test requires (axes decoupled: conservative).
// The same dt margin as the per-ray prefilter covers fp32 rounding. Lane k
// evaluates object k; the ballot is the warp-uniform survivor mask.
__device__ __forceinline__ float wmin(float v) {
  float r;
  asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float wmax(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

__device__ __forceinline__ void interval_slab(float lo, float hi, float ol, float oh, float il,
                                              float ih, float& E, float& X) {
  if (!(il > 0.f || ih < 0.f)) return;  // mixed signs: no bound from this axis
#if NIF_BUNDLE_SIGN
  // The sign of the reciprocals (warp-uniform) says which plane is the
  // entry and which corner of [o] x [inv] bounds each product, so only the
  // two extremal products are formed. They are the same fp32 products the
  // four-corner form below takes the min / max of (rounding is monotone),
  // and its min(ta, tb) / max(ta, tb) pick the entry / exit side because
  // hi - o >= lo - o: E and X are bit-identical.
  if (il > 0.f) {  // entry lo, exit hi
    const float v0 = lo - oh, u1 = hi - ol;
    E = fmaxf(E, v0 * (v0 >= 0.f ? il : ih));
    X = fminf(X, u1 * (u1 >= 0.f ? ih : il));
  } else {         // entry hi, exit lo
    const float u1 = hi - ol, v0 = lo - oh;
    E = fmaxf(E, u1 * (u1 >= 0.f ? il : ih));
    X = fminf(X, v0 * (v0 <= 0.f ? il : ih));
  }
  return;
#endif
  const float a0 = lo - oh, a1 = lo - ol, b0 = hi - oh, b1 = hi - ol;
  const float p0 = a0 * il, p1 = a0 * ih, p2 = a1 * il, p3 = a1 * ih;
  const float q0 = b0 * il, q1 = b0 * ih, q2 = b1 * il, q3 = b1 * ih;
  const float ta_lo = fminf(fminf(p0, p1), fminf(p2, p3)), ta_hi = fmaxf(fmaxf(p0, p1), fmaxf(p2, p3));
  const float tb_lo = fminf(fminf(q0, q1), fminf(q2, q3)), tb_hi = fmaxf(fmaxf(q0, q1), fmaxf(q2, q3));
  E = fmaxf(E, fminf(ta_lo, tb_lo));
  X = fminf(X, fmaxf(ta_hi, tb_hi));
}

__device__ __forceinline__ uint32_t warp_bundle_mask(const RayF& q, bool use_pf, bool valid,
                                                     int lane, int n_obj, const float4* flo,
                                                     const float4* fhi, uint32_t all_obj,
                                                     float absmax) {
  const unsigned full = 0xffffffffu;
  const uint32_t vmask = __ballot_sync(full, valid);
  if (n_obj <= 1 || vmask == 0 || !__all_sync(full, use_pf || !valid)) return all_obj;
  float ox = q.ox, oy = q.oy, oz = q.oz, ix = q.ix, iy = q.iy, iz = q.iz, tm = q.tmax_ru;
  if (vmask != full) {  // (the last chunk only) invalid lanes borrow the first
                        // valid lane's ray: neutral for the min/max below
    const int src = __ffs(vmask) - 1;
    const float sox = __shfl_sync(full, ox, src), soy = __shfl_sync(full, oy, src),
                soz = __shfl_sync(full, oz, src), six = __shfl_sync(full, ix, src),
                siy = __shfl_sync(full, iy, src), siz = __shfl_sync(full, iz, src),
                stm = __shfl_sync(full, tm, src);
    if (!valid) {
      ox = sox; oy = soy; oz = soz;
      ix = six; iy = siy; iz = siz;
      tm = stm;
    }
  }
  const float oxl = wmin(ox), oxh = wmax(ox), oyl = wmin(oy), oyh = wmax(oy);
  const float ozl = wmin(oz), ozh = wmax(oz);
  const float ixl = wmin(ix), ixh = wmax(ix), iyl = wmin(iy), iyh = wmax(iy);
  const float izl = wmin(iz), izh = wmax(iz);
  const float tmh = wmax(tm);
  // margin from warp-wide maxima: every interval endpoint product pairs some
  // lane's origin with some lane's reciprocal
  const float omax = fmaxf(fmaxf(fmaxf(fabsf(oxl), fabsf(oxh)), fmaxf(fabsf(oyl), fabsf(oyh))),
                           fmaxf(fabsf(ozl), fabsf(ozh)));
  const float imax = fmaxf(fmaxf(fmaxf(fabsf(ixl), fabsf(ixh)), fmaxf(fabsf(iyl), fabsf(iyh))),
                           fmaxf(fabsf(izl), fabsf(izh)));
  const float dth = 1e-5f * (absmax + omax + 1e-30f) * imax;
  if (!isfinite(dth)) return all_obj;
  bool pass = false;
  if (lane < n_obj) {
    const float4 lo = flo[lane], hi = fhi[lane];
    float E = -CUDART_INF_F, X = CUDART_INF_F;
    interval_slab(lo.x, hi.x, oxl, oxh, ixl, ixh, E, X);
    interval_slab(lo.y, hi.y, oyl, oyh, iyl, iyh, E, X);
    interval_slab(lo.z, hi.z, ozl, ozh, izl, izh, E, X);
    E -= dth;
    X += dth;
    pass = E <= X && X >= -1e-6f && E <= tmh;
  }
  uint32_t m = __ballot_sync(full, pass);
  if (n_obj > 32) m = 0xffffffffu;
  return m;
}

template <bool EXACT>
__global__ void __launch_bounds__(kThreads, NIF_GATHER_MINB)
gather_fused_kernel(nif_scene_view s, const uint8_t* __restrict__ route,
                    const double* __restrict__ org, const double* __restrict__ dir,
                    const double* __restrict__ tms, int64_t n, nif_gather_out out,
                    unsigned long long* __restrict__ status, int* __restrict__ tile_ctr,
                    int64_t n_tiles, long long* __restrict__ prof) {
  __shared__ ObjC objs[kMaxObjFused];
  __shared__ float4 flo[kMaxObjFused], fhi[kMaxObjFused];
  __shared__ float s_absmax;
  __shared__ int s_tile;
  __shared__ int s_warp[kThreads / 32];
  __shared__ unsigned long long s_excl;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int n_obj = s.n_obj;
  if (tid == 0) s_absmax = 0.f;
  __syncthreads();
  if (tid < n_obj) {
    ObjC& b = objs[tid];
    const int ob = s.t_order[tid];  // leaf (DFS) order
    const double* bx = s.obox + (size_t)ob * 6;
    float am = 0.f;
    for (int a = 0; a < 3; ++a) {
      b.lo[a] = bx[a];
      b.hi[a] = bx[3 + a];
      b.lt[a] = bx[a] - s.tol;
      b.ht[a] = bx[3 + a] + s.tol;
      b.c[a] = 0.5 * (bx[a] + bx[3 + a]);
      am = fmaxf(am, fmaxf(fabsf((float)bx[a]), fabsf((float)bx[3 + a])));
    }
    flo[tid] = make_float4((float)bx[0], (float)bx[1], (float)bx[2], 0.f);
    fhi[tid] = make_float4((float)bx[3], (float)bx[4], (float)bx[5], 0.f);
    const double hx = 0.5 * (bx[3] - bx[0]), hy = 0.5 * (bx[4] - bx[1]),
                 hz = 0.5 * (bx[5] - bx[2]);
    b.hn = sqrt(hx * hx + hy * hy + hz * hz);
    b.hinv = 1.0f / (float)b.hn;
    b.id = ob;
    b.route = route[ob];
    b.root = s.roots[ob];
    atomicMax(reinterpret_cast<int*>(&s_absmax), __float_as_int(am));
  }
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t i = tile * kThreads + tid;
  const bool valid = i < n;
#define NIF_GPROF(k) \
  if (prof != nullptr && tid == 0 && tile < 8192) prof[tile * 8 + (k)] = clock64();
  NIF_GPROF(0);

  RayX r{};
  RayF q{};
  bool use_pf = false;
  if (valid) {
    r.ox = org[i * 3 + 0];
    r.oy = org[i * 3 + 1];
    r.oz = org[i * 3 + 2];
    r.dx = dir[i * 3 + 0];
    r.dy = dir[i * 3 + 1];
    r.dz = dir[i * 3 + 2];
    r.tmax = tms[i];
    r.ix = r.dx != 0.0 ? 1.0 / r.dx : 0.0;
    r.iy = r.dy != 0.0 ? 1.0 / r.dy : 0.0;
    r.iz = r.dz != 0.0 ? 1.0 / r.dz : 0.0;
    use_pf = n_obj > 1 && fabs(r.dx) > 1e-20 && fabs(r.dy) > 1e-20 && fabs(r.dz) > 1e-20;
    if (use_pf) {
      q.ix = (float)r.ix;
      q.iy = (float)r.iy;
      q.iz = (float)r.iz;
      q.ox = (float)r.ox;
      q.oy = (float)r.oy;
      q.oz = (float)r.oz;
      q.ox_i = -(float)r.ox * q.ix;
      q.oy_i = -(float)r.oy * q.iy;
      q.oz_i = -(float)r.oz * q.iz;
      const float S = s_absmax + fmaxf(fmaxf(fabsf((float)r.ox), fabsf((float)r.oy)),
                                       fabsf((float)r.oz)) + 1e-30f;
      const float imax = fmaxf(fmaxf(fabsf(q.ix), fabsf(q.iy)), fabsf(q.iz));
      q.dt = 1e-5f * S * imax;
      q.tmax_ru = __double2float_ru(r.tmax);
      use_pf = isfinite(q.dt);
    }
  }
  // ---- classify (once) --------------------------------------------------
  uint64_t mask = 0;   // 2 bits per object slot: 1 outer, 2 inner
  uint32_t hyb = 0;    // routed-away candidates
  int n_out = 0, n_in = 0;
  const bool test_box = n_obj > 1;
  const uint32_t all_obj = n_obj >= 32 ? 0xffffffffu : ((1u << n_obj) - 1u);
  // (1) warp-cooperative culling: lane k tests object k against the whole
  //     warp's ray bundle (warp_bundle_mask); (2) per-ray fp32 prefilter over
  //     the survivors; (3) exact fp64 classification of what is left.
  const uint32_t wmask =
      warp_bundle_mask(q, use_pf, valid, lane, n_obj, flo, fhi, all_obj, s_absmax);
  uint32_t pmask = 0;
  if (valid) {
    if (use_pf) {
      uint32_t w = wmask;
      while (w) {
        const int k = __ffs(w) - 1;
        w &= w - 1;
        pmask |= (uint32_t)prefilter(q, flo[k], fhi[k]) << k;
      }
    } else {
      pmask = all_obj;
    }
    while (pmask) {
      const int k = __ffs(pmask) - 1;
      pmask &= pmask - 1;
      double t0;
      const int kind = classify_obj(r, objs[k], test_box, s.tol, &t0);
      if (kind == 0) continue;
      if (objs[k].route == 1) {
        mask |= (uint64_t)kind << (2 * k);
        if (kind == 1) ++n_out;
        else ++n_in;
      } else {
        hyb |= 1u << k;
      }
    }
  }
  NIF_GPROF(1);
  // ---- block scan of (outer, inner) counts, packed 16|16 ------------------
  const int packed = (n_out << 16) | n_in;
  int incl = packed;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  NIF_GPROF(2);
  int warp_base = 0, block_total = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    if (w < warp) warp_base += s_warp[w];
    block_total += s_warp[w];
  }
  const int excl_in_block = warp_base + incl - packed;
  // ---- publish the tile aggregate, then the hybrid any-hit ----------------
  const uint64_t agg_o = (uint32_t)block_total >> 16, agg_i = (uint32_t)block_total & 0xffff;
  if (tid == 0)
    atomicExch(status + tile, pack(tile == 0 ? kFlagP : kFlagA, agg_o, agg_i));
  if (valid) {
    bool occ = false;
    uint32_t h = hyb;
    while (h != 0 && !occ) {
      const int k = __ffs(h) - 1;
      h &= h - 1;
      occ = occluded_in_object(s.nodes, s.tris, objs[k].root, r.ox, r.oy, r.oz, r.dx, r.dy, r.dz,
                               s.eps, r.tmax);
    }
    out.bvh_occ[i] = occ ? 1 : 0;
  }
  NIF_GPROF(3);
  // ---- decoupled look-back, one warp, 32 predecessors per probe -----------
  if (warp == 0) {
    uint32_t ex_o = 0, ex_i = 0;
    if (tile > 0) {
      int64_t base = tile - 1;
      while (true) {
        const int64_t j = base - lane;
        uint64_t v = kFlagP;  // before tile 0: an inclusive prefix of zero
        if (j >= 0) {
          do {
            v = *reinterpret_cast<volatile unsigned long long*>(status + j);
          } while ((v >> 62) == 0);
        }
        const uint32_t pm = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        const int stop = pm ? __ffs(pm) - 1 : 31;
        const uint32_t co = lane <= stop ? (uint32_t)((v >> 31) & kCntMask) : 0u;
        const uint32_t ci = lane <= stop ? (uint32_t)(v & kCntMask) : 0u;
        ex_o += __reduce_add_sync(0xffffffffu, co);
        ex_i += __reduce_add_sync(0xffffffffu, ci);
        if (pm) break;
        base -= 32;
      }
      if (lane == 0) atomicExch(status + tile, pack(kFlagP, ex_o + agg_o, ex_i + agg_i));
    }
    if (lane == 0) {
      if (tile == n_tiles - 1) {
        out.counts[0] = (int64_t)(ex_o + agg_o);
        out.counts[1] = (int64_t)(ex_i + agg_i);
        out.counts[2] = (int64_t)(ex_o + agg_o) + (int64_t)(ex_i + agg_i);
      }
      s_excl = ((uint64_t)ex_o << 32) | ex_i;
    }
  }
  NIF_GPROF(4);
  __syncthreads();
  NIF_GPROF(5);
  if (!valid) return;
  // ---- write records -------------------------------------------------------
  int64_t jo = (int64_t)(s_excl >> 32) + (excl_in_block >> 16);
  int64_t ji = (int64_t)(s_excl & 0xffffffffu) + (excl_in_block & 0xffff);
  int64_t jt = jo + ji;
  float du = 0.f, dv = 0.f;
  if (!EXACT && mask != 0) sph32f((float)r.dx, (float)r.dy, (float)r.dz, 1.0f, &du, &dv);
  int deg_count = 0;
  uint64_t m = mask;
  while (m != 0) {
    const int bit = __ffsll((long long)m) - 1;
    const int k = bit >> 1;
    const int kind = (int)((m >> (2 * k)) & 3);
    m &= ~(3ull << (2 * k));
    const ObjC& b = objs[k];
    double cc[5];
    float c4[4], rr = 0.f;
    bool deg;
    if (kind == 1) {
      const Hit3 hh = slab(r, b);
      if (EXACT) {
        deg = transform_outer(r.ox, r.oy, r.oz, r.dx, r.dy, r.dz, b.lo, b.hi, hh.t0, cc);
        cc[4] = 0.0;
      } else {
        const double ex = r.ox + hh.t0 * r.dx, ey = r.oy + hh.t0 * r.dy,
                     ez = r.oz + hh.t0 * r.dz;
        const double rx = ex - b.c[0], ry = ey - b.c[1], rz = ez - b.c[2];
        float rnf, rinvf;
        deg = degenerate_f32(rx, ry, rz, &rnf, &rinvf);
        if (deg) { c4[0] = 0.5f; c4[1] = 0.5f; }
        else sph32f((float)rx, (float)ry, (float)rz, rinvf, &c4[0], &c4[1]);
        c4[2] = du;
        c4[3] = dv;
      }
    } else {
      if (EXACT) {
        deg = transform_inner(r.ox, r.oy, r.oz, r.dx, r.dy, r.dz, b.lo, b.hi, cc);
      } else {
        const double rx = r.ox - b.c[0], ry = r.oy - b.c[1], rz = r.oz - b.c[2];
        float rnf, rinvf;
        deg = degenerate_f32(rx, ry, rz, &rnf, &rinvf);
        if (deg) { c4[0] = 0.5f; c4[1] = 0.5f; rr = 0.f; }
        else {
          sph32f((float)rx, (float)ry, (float)rz, rinvf, &c4[0], &c4[1]);
          rr = fminf(rnf * b.hinv, 1.0f);
        }
        c4[2] = du;
        c4[3] = dv;
      }
    }
    if (EXACT) {
      c4[0] = (float)cc[0];
      c4[1] = (float)cc[1];
      c4[2] = (float)cc[2];
      c4[3] = (float)cc[3];
      rr = (float)cc[4];
    }
    if (kind == 1) {
      if (jo < out.cap_outer) {
        out.outer_obj[jo] = b.id;
        out.outer_ray[jo] = (int32_t)i;
        reinterpret_cast<float4*>(out.outer_coord)[jo] = make_float4(c4[0], c4[1], c4[2], c4[3]);
      }
      ++jo;
    } else {
      if (ji < out.cap_inner) {
        out.inner_obj[ji] = b.id;
        out.inner_ray[ji] = (int32_t)i;
        reinterpret_cast<float4*>(out.inner_coord)[ji] = make_float4(c4[0], c4[1], c4[2], c4[3]);
        out.inner_r[ji] = rr;
      }
      ++ji;
    }
    if (EXACT && out.rec_kind != nullptr && jt < out.cap_total) {
      out.rec_kind[jt] = kind == 1 ? 0 : 1;
      out.rec_obj[jt] = b.id;
      out.rec_ray[jt] = (int32_t)i;
      for (int q = 0; q < 5; ++q) out.rec_coord[jt * 5 + q] = cc[q];
    }
    ++jt;
    deg_count += deg ? 1 : 0;
  }
  NIF_GPROF(6);
  if (deg_count) atomicAdd((unsigned long long*)(out.counts + 3), (unsigned long long)deg_count);
}

// ===========================================================================
// Persistent, software-pipelined variant of the hot-path gather (queues only).
//
// Each CTA claims 256-ray tiles in increasing order and keeps three in
// flight: the rays of tile j+1 (and j+2) stream into shared memory through
// cp.async.bulk (TMA bulk copies completing on an mbarrier) while tile j is
// classified; tile j's records are written one iteration later, after its
// decoupled look-back, so the look-back wait overlaps tile j+1's
// classification instead of stalling the CTA. Deadlock-free: a CTA waiting
// on the predecessors of tile a only holds unpublished tiles claimed after
// a (larger ids), so waits always point to smaller tiles.
// ===========================================================================
__device__ __forceinline__ uint32_t tc_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int kStages = 3;
constexpr int kRayBytes = 56;  // origin 24 + direction 24 + tmax 8
constexpr int kStageBytes = kThreads * kRayBytes;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(tc_smem(dst)),
      "l"(src), "r"(bytes), "r"(tc_smem(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc_smem(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITG_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITG_%=;\n\t}" ::"r"(tc_smem(bar)),
      "r"(parity)
      : "memory");
}

struct TileRays {
  const double* o;  // origins of ray 0 of the tile (smem or global)
  const double* d;
  const double* t;
};

__device__ __forceinline__ TileRays tile_rays(uint8_t* stage, bool staged, const double* org,
                                              const double* dir, const double* tms,
                                              int64_t tile) {
  if (staged) {
    return {reinterpret_cast<const double*>(stage),
            reinterpret_cast<const double*>(stage + kThreads * 24),
            reinterpret_cast<const double*>(stage + kThreads * 48)};
  }
  const int64_t r0 = tile * kThreads;
  return {org + r0 * 3, dir + r0 * 3, tms + r0};
}

__global__ void __launch_bounds__(kThreads, NIF_GATHER_MINB)
gather_persist_kernel(nif_scene_view s, const uint8_t* __restrict__ route,
                      const double* __restrict__ org, const double* __restrict__ dir,
                      const double* __restrict__ tms, int64_t n, nif_gather_out out,
                      unsigned long long* __restrict__ status, int* __restrict__ tile_ctr,
                      int64_t n_tiles) {
  extern __shared__ __align__(128) uint8_t dsm[];  // kStages x kStageBytes ray buffers
  __shared__ ObjC objs[kMaxObjFused];
  __shared__ float4 flo[kMaxObjFused], fhi[kMaxObjFused];
  __shared__ float s_absmax;
  __shared__ int s_warp[kThreads / 32];
  __shared__ unsigned long long s_excl;
  __shared__ uint64_t sbar[kStages];
  __shared__ long long s_tiles[kStages];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int n_obj = s.n_obj;
  const int64_t n_full = n / kThreads;  // tiles whose rays are bulk-copied
  if (tid == 0) s_absmax = 0.f;
  __syncthreads();
  if (tid < n_obj) {
    ObjC& b = objs[tid];
    const int ob = s.t_order[tid];
    const double* bx = s.obox + (size_t)ob * 6;
    float am = 0.f;
    for (int a = 0; a < 3; ++a) {
      b.lo[a] = bx[a];
      b.hi[a] = bx[3 + a];
      b.lt[a] = bx[a] - s.tol;
      b.ht[a] = bx[3 + a] + s.tol;
      b.c[a] = 0.5 * (bx[a] + bx[3 + a]);
      am = fmaxf(am, fmaxf(fabsf((float)bx[a]), fabsf((float)bx[3 + a])));
    }
    flo[tid] = make_float4((float)bx[0], (float)bx[1], (float)bx[2], 0.f);
    fhi[tid] = make_float4((float)bx[3], (float)bx[4], (float)bx[5], 0.f);
    const double hx = 0.5 * (bx[3] - bx[0]), hy = 0.5 * (bx[4] - bx[1]),
                 hz = 0.5 * (bx[5] - bx[2]);
    b.hn = sqrt(hx * hx + hy * hy + hz * hz);
    b.hinv = 1.0f / (float)b.hn;
    b.id = ob;
    b.route = route[ob];
    b.root = s.roots[ob];
    atomicMax(reinterpret_cast<int*>(&s_absmax), __float_as_int(am));
  }
  auto claim = [&](int st) {  // thread 0: claim the next tile for stage st
    const long long t = atomicAdd(tile_ctr, 1);
    s_tiles[st] = t < n_tiles ? t : -1;
    if (t < n_full) {
      uint8_t* dst = dsm + st * kStageBytes;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(sbar + st, kStageBytes);
      bulk_g2s(dst, org + t * kThreads * 3, kThreads * 24, sbar + st);
      bulk_g2s(dst + kThreads * 24, dir + t * kThreads * 3, kThreads * 24, sbar + st);
      bulk_g2s(dst + kThreads * 48, tms + t * kThreads, kThreads * 8, sbar + st);
    }
  };
  if (tid == 0) {
    for (int st = 0; st < kStages; ++st)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc_smem(sbar + st)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    claim(0);
    claim(1);
  }
  __syncthreads();
  const bool test_box = n_obj > 1;
  const uint32_t all_obj = n_obj >= 32 ? 0xffffffffu : ((1u << n_obj) - 1u);
  uint32_t phases = 0;  // parity bit per stage

  // state of the previous tile (written one iteration late)
  long long p_tile = -1;
  uint64_t p_mask = 0;
  int p_excl = 0;
  uint32_t p_agg = 0;

  for (int j = 0;; ++j) {
    const int st = j % kStages;
    const long long tile = s_tiles[st];
    long long cur_tile = tile;
    uint64_t mask = 0;
    int excl_in_block = 0;
    uint32_t block_total = 0;
    if (tile >= 0) {
      const bool staged = tile < n_full;
      if (staged) {
        mbar_wait_parity(sbar + st, (phases >> st) & 1u);
        phases ^= 1u << st;
      }
      const TileRays tr = tile_rays(dsm + st * kStageBytes, staged, org, dir, tms, tile);
      const int64_t i = tile * kThreads + tid;
      const bool valid = i < n;
      RayX r{};
      RayF q{};
      bool use_pf = false;
      if (valid) {
        r.ox = tr.o[tid * 3 + 0];
        r.oy = tr.o[tid * 3 + 1];
        r.oz = tr.o[tid * 3 + 2];
        r.dx = tr.d[tid * 3 + 0];
        r.dy = tr.d[tid * 3 + 1];
        r.dz = tr.d[tid * 3 + 2];
        r.tmax = tr.t[tid];
        r.ix = r.dx != 0.0 ? 1.0 / r.dx : 0.0;
        r.iy = r.dy != 0.0 ? 1.0 / r.dy : 0.0;
        r.iz = r.dz != 0.0 ? 1.0 / r.dz : 0.0;
        use_pf = n_obj > 1 && fabs(r.dx) > 1e-20 && fabs(r.dy) > 1e-20 && fabs(r.dz) > 1e-20;
        if (use_pf) {
          q.ix = (float)r.ix;
          q.iy = (float)r.iy;
          q.iz = (float)r.iz;
          q.ox = (float)r.ox;
          q.oy = (float)r.oy;
          q.oz = (float)r.oz;
          q.ox_i = -(float)r.ox * q.ix;
          q.oy_i = -(float)r.oy * q.iy;
          q.oz_i = -(float)r.oz * q.iz;
          const float S = s_absmax + fmaxf(fmaxf(fabsf(q.ox), fabsf(q.oy)), fabsf(q.oz)) + 1e-30f;
          const float imax = fmaxf(fmaxf(fabsf(q.ix), fabsf(q.iy)), fabsf(q.iz));
          q.dt = 1e-5f * S * imax;
          q.tmax_ru = __double2float_ru(r.tmax);
          use_pf = isfinite(q.dt);
        }
      }
      uint32_t hyb = 0;
      int n_out = 0, n_in = 0;
      const uint32_t wmask =
          warp_bundle_mask(q, use_pf, valid, lane, n_obj, flo, fhi, all_obj, s_absmax);
      if (valid) {
        uint32_t pmask = 0;
        if (use_pf) {
          uint32_t w = wmask;
          while (w) {
            const int k = __ffs(w) - 1;
            w &= w - 1;
            pmask |= (uint32_t)prefilter(q, flo[k], fhi[k]) << k;
          }
        } else {
          pmask = all_obj;
        }
        while (pmask) {
          const int k = __ffs(pmask) - 1;
          pmask &= pmask - 1;
          double t0;
          const int kind = classify_obj(r, objs[k], test_box, s.tol, &t0);
          if (kind == 0) continue;
          if (objs[k].route == 1) {
            mask |= (uint64_t)kind << (2 * k);
            if (kind == 1) ++n_out;
            else ++n_in;
          } else {
            hyb |= 1u << k;
          }
        }
      }
      const int packed = (n_out << 16) | n_in;
      int incl = packed;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
      }
      if (lane == 31) s_warp[warp] = incl;
      __syncthreads();
      int warp_base = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) {
        if (w < warp) warp_base += s_warp[w];
        tot += s_warp[w];
      }
      excl_in_block = warp_base + incl - packed;
      block_total = (uint32_t)tot;
      if (tid == 0)
        atomicExch(status + tile, pack(tile == 0 ? kFlagP : kFlagA, block_total >> 16,
                                       block_total & 0xffff));
      if (valid) {
        bool occ = false;
        uint32_t h = hyb;
        while (h != 0 && !occ) {
          const int k = __ffs(h) - 1;
          h &= h - 1;
          occ = occluded_in_object(s.nodes, s.tris, objs[k].root, r.ox, r.oy, r.oz, r.dx, r.dy,
                                   r.dz, s.eps, r.tmax);
        }
        out.bvh_occ[i] = occ ? 1 : 0;
      }
    }
    // ---- previous tile: look-back, then its records -------------------------
    if (p_tile >= 0) {
      if (warp == 0) {
        const uint64_t agg_o = p_agg >> 16, agg_i = p_agg & 0xffff;
        uint32_t ex_o = 0, ex_i = 0;
        if (p_tile > 0) {
          int64_t base = p_tile - 1;
          while (true) {
            const int64_t jj = base - lane;
            uint64_t v = kFlagP;
            if (jj >= 0) {
              do {
                v = *reinterpret_cast<volatile unsigned long long*>(status + jj);
              } while ((v >> 62) == 0);
            }
            const uint32_t pm = __ballot_sync(0xffffffffu, (v >> 62) == 2);
            const int stop = pm ? __ffs(pm) - 1 : 31;
            const uint32_t co = lane <= stop ? (uint32_t)((v >> 31) & kCntMask) : 0u;
            const uint32_t ci = lane <= stop ? (uint32_t)(v & kCntMask) : 0u;
            ex_o += __reduce_add_sync(0xffffffffu, co);
            ex_i += __reduce_add_sync(0xffffffffu, ci);
            if (pm) break;
            base -= 32;
          }
          if (lane == 0) atomicExch(status + p_tile, pack(kFlagP, ex_o + agg_o, ex_i + agg_i));
        }
        if (lane == 0) {
          if (p_tile == n_tiles - 1) {
            out.counts[0] = (int64_t)(ex_o + agg_o);
            out.counts[1] = (int64_t)(ex_i + agg_i);
            out.counts[2] = (int64_t)(ex_o + agg_o) + (int64_t)(ex_i + agg_i);
          }
          s_excl = ((uint64_t)ex_o << 32) | ex_i;
        }
      }
      __syncthreads();
      const int64_t i = p_tile * kThreads + tid;
      if (i < n && p_mask != 0) {
        const int pst = (j + kStages - 1) % kStages;
        const TileRays tr =
            tile_rays(dsm + pst * kStageBytes, p_tile < n_full, org, dir, tms, p_tile);
        RayX r{};
        r.ox = tr.o[tid * 3 + 0];
        r.oy = tr.o[tid * 3 + 1];
        r.oz = tr.o[tid * 3 + 2];
        r.dx = tr.d[tid * 3 + 0];
        r.dy = tr.d[tid * 3 + 1];
        r.dz = tr.d[tid * 3 + 2];
        r.tmax = tr.t[tid];
        int64_t jo = (int64_t)(s_excl >> 32) + (p_excl >> 16);
        int64_t ji = (int64_t)(s_excl & 0xffffffffu) + (p_excl & 0xffff);
        float du, dv;
        sph32f((float)r.dx, (float)r.dy, (float)r.dz, 1.0f, &du, &dv);
        bool have_inv = false;
        int deg_count = 0;
        uint64_t m = p_mask;
        while (m != 0) {
          const int bit = __ffsll((long long)m) - 1;
          const int k = bit >> 1;
          const int kind = (int)((m >> (2 * k)) & 3);
          m &= ~(3ull << (2 * k));
          const ObjC& b = objs[k];
          float c0, c1, rr = 0.f;
          float rnf, rinvf;
          bool deg;
          if (kind == 1) {
            if (!have_inv) {
              r.ix = r.dx != 0.0 ? 1.0 / r.dx : 0.0;
              r.iy = r.dy != 0.0 ? 1.0 / r.dy : 0.0;
              r.iz = r.dz != 0.0 ? 1.0 / r.dz : 0.0;
              have_inv = true;
            }
            const Hit3 hh = slab(r, b);
            const double ex = r.ox + hh.t0 * r.dx, ey = r.oy + hh.t0 * r.dy,
                         ez = r.oz + hh.t0 * r.dz;
            const double rx = ex - b.c[0], ry = ey - b.c[1], rz = ez - b.c[2];
            deg = degenerate_f32(rx, ry, rz, &rnf, &rinvf);
            if (deg) { c0 = 0.5f; c1 = 0.5f; }
            else sph32f((float)rx, (float)ry, (float)rz, rinvf, &c0, &c1);
            if (jo < out.cap_outer) {
              out.outer_obj[jo] = b.id;
              out.outer_ray[jo] = (int32_t)i;
              reinterpret_cast<float4*>(out.outer_coord)[jo] = make_float4(c0, c1, du, dv);
            }
            ++jo;
          } else {
            const double rx = r.ox - b.c[0], ry = r.oy - b.c[1], rz = r.oz - b.c[2];
            deg = degenerate_f32(rx, ry, rz, &rnf, &rinvf);
            if (deg) { c0 = 0.5f; c1 = 0.5f; rr = 0.f; }
            else {
              sph32f((float)rx, (float)ry, (float)rz, rinvf, &c0, &c1);
              rr = fminf(rnf * b.hinv, 1.0f);
            }
            if (ji < out.cap_inner) {
              out.inner_obj[ji] = b.id;
              out.inner_ray[ji] = (int32_t)i;
              reinterpret_cast<float4*>(out.inner_coord)[ji] = make_float4(c0, c1, du, dv);
              out.inner_r[ji] = rr;
            }
            ++ji;
          }
          deg_count += deg ? 1 : 0;
        }
        if (deg_count)
          atomicAdd((unsigned long long*)(out.counts + 3), (unsigned long long)deg_count);
      }
    }
    if (cur_tile < 0) break;  // uniform: no tile this iteration, previous drained
    __syncthreads();          // stage (j-1) % kStages fully consumed
    if (tid == 0) claim((j + 2) % kStages);
    p_tile = cur_tile;
    p_mask = mask;
    p_excl = excl_in_block;
    p_agg = block_total;
    __syncthreads();          // s_tiles of the next iterations visible
  }
}


// ===========================================================================
// Hot-path gather with unordered (warp-granular) compaction.
//
// The visibility pass only needs, per ray, the OR of its records' bits, so
// the hot-path queues need not be in the reference's ray-major order (the
// API gather above keeps it). Each warp takes 32-ray chunks (static stride,
// no CTA-wide barriers at all), classifies exactly as above, reserves its
// records with one atomicAdd per queue, and writes them contiguously (rays
// of a chunk stay adjacent, which keeps the query kernels' latent gathers
// coherent). No scan, no look-back, no staging: a warp never waits on
// another. Per-ray results are identical to the ordered kernels.
// ===========================================================================
#ifndef NIF_GATHER_MINB_U
#define NIF_GATHER_MINB_U 3
#endif
#ifndef NIF_RAY_PREFILTER
// per-ray fp32 prefilter after the warp-bundle cull: 0 = the bundle's
// survivors go straight to the exact fp64 test (C2: 1.52 bundle survivors
// per ray, 1.21 after the prefilter -- the prefilter cost more than the fp64
// tests it saved: gather 70.1 -> 68.6 us)
#define NIF_RAY_PREFILTER 0
#endif
#ifdef NIF_GATHER_STATS
// diagnostics build only: rays, bundle survivors, prefilter survivors, hits
__device__ unsigned long long g_gstats[4];
#endif

__global__ void __launch_bounds__(kThreads, NIF_GATHER_MINB_U)
gather_warp_kernel(nif_scene_view s, const uint8_t* __restrict__ route,
                   const double* __restrict__ org, const double* __restrict__ dir,
                   const double* __restrict__ tms, int64_t n, nif_gather_out out,
                   unsigned long long* __restrict__ reserve, unsigned int* __restrict__ done,
                   unsigned int* __restrict__ tail, unsigned long long* __restrict__ deg_acc,
                   int dyn_rounds, unsigned long long* __restrict__ tl) {
  __shared__ ObjC objs[kMaxObjFused];
  __shared__ float4 flo[kMaxObjFused], fhi[kMaxObjFused];
  __shared__ float s_absmax;
  // programmatic dependent launch: the query kernel queued behind this one
  // may start its prologue (weights -> smem, TMEM) on SMs this persistent
  // grid leaves free; it reads the queues only after griddepcontrol.wait,
  // i.e. after this grid has completed and flushed
  asm volatile("griddepcontrol.launch_dependents;");
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int n_obj = s.n_obj;
  // diagnostic timeline (nif_debug_set_timeline_gather): per warp entry,
  // after the prologue, exit, chunks processed
  unsigned long long* wtl =
      tl != nullptr && lane == 0 ? tl + ((int64_t)blockIdx.x * (kThreads / 32) + warp) * 4 : nullptr;
  if (wtl) wtl[0] = globaltimer();
  int n_done = 0;
  if (tid == 0) s_absmax = 0.f;
  __syncthreads();
  if (tid < n_obj) {
    ObjC& b = objs[tid];
    const int ob = s.t_order[tid];
    const double* bx = s.obox + (size_t)ob * 6;
    float am = 0.f;
    for (int a = 0; a < 3; ++a) {
      b.lo[a] = bx[a];
      b.hi[a] = bx[3 + a];
      b.lt[a] = bx[a] - s.tol;
      b.ht[a] = bx[3 + a] + s.tol;
      b.c[a] = 0.5 * (bx[a] + bx[3 + a]);
      am = fmaxf(am, fmaxf(fabsf((float)bx[a]), fabsf((float)bx[3 + a])));
    }
    flo[tid] = make_float4((float)bx[0], (float)bx[1], (float)bx[2], 0.f);
    fhi[tid] = make_float4((float)bx[3], (float)bx[4], (float)bx[5], 0.f);
    const double hx = 0.5 * (bx[3] - bx[0]), hy = 0.5 * (bx[4] - bx[1]),
                 hz = 0.5 * (bx[5] - bx[2]);
    b.hn = sqrt(hx * hx + hy * hy + hz * hz);
    b.hinv = 1.0f / (float)b.hn;
    b.id = ob;
    b.route = route[ob];
    b.root = s.roots[ob];
    atomicMax(reinterpret_cast<int*>(&s_absmax), __float_as_int(am));
  }
  __syncthreads();
  const bool test_box = n_obj > 1;
  const uint32_t all_obj = n_obj >= 32 ? 0xffffffffu : ((1u << n_obj) - 1u);
  const int64_t n_chunks = (n + 31) / 32;
  const int64_t nw = (int64_t)gridDim.x * (kThreads / 32);
  const float absmax = s_absmax;
  int deg_count = 0;
  // every warp takes n_chunks / nw chunks statically (interleaved), the
  // remainder is handed out one chunk at a time on demand, so warps that
  // drew cheap chunks absorb the tail instead of idling
  const int64_t wid = (int64_t)blockIdx.x * (kThreads / 32) + warp;
  const int64_t rounds = max((int64_t)0, n_chunks / nw - dyn_rounds);
  if (wtl) wtl[1] = globaltimer();
  for (int64_t k = 0;; ++k) {
    int64_t c;
    if (k < rounds) {
      c = wid + k * nw;
    } else {
      unsigned int t = 0;
      if (lane == 0) t = atomicAdd(tail, 1u);
      c = rounds * nw + __shfl_sync(0xffffffffu, t, 0);
      if (c >= n_chunks) break;
    }
    ++n_done;
    const int64_t i = c * 32 + lane;
    const bool valid = i < n;
    RayX r;  // written for valid lanes; invalid lanes never read their ray
    RayF q;
    bool use_pf = false;
    int s3 = -1;  // entry-plane offsets for slab_nf, -1: the general slab
    if (valid) {
      r.ox = __ldg(org + i * 3 + 0);
      r.oy = __ldg(org + i * 3 + 1);
      r.oz = __ldg(org + i * 3 + 2);
      r.dx = __ldg(dir + i * 3 + 0);
      r.dy = __ldg(dir + i * 3 + 1);
      r.dz = __ldg(dir + i * 3 + 2);
      r.tmax = __ldg(tms + i);
      r.ix = r.dx != 0.0 ? 1.0 / r.dx : 0.0;
      r.iy = r.dy != 0.0 ? 1.0 / r.dy : 0.0;
      r.iz = r.dz != 0.0 ? 1.0 / r.dz : 0.0;
      use_pf = n_obj > 1 && fabs(r.dx) > 1e-20 && fabs(r.dy) > 1e-20 && fabs(r.dz) > 1e-20;
      if (use_pf) {
        q.ix = (float)r.ix;
        q.iy = (float)r.iy;
        q.iz = (float)r.iz;
        q.ox = (float)r.ox;
        q.oy = (float)r.oy;
        q.oz = (float)r.oz;
        q.ox_i = -q.ox * q.ix;
        q.oy_i = -q.oy * q.iy;
        q.oz_i = -q.oz * q.iz;
        const float S = absmax + fmaxf(fmaxf(fabsf(q.ox), fabsf(q.oy)), fabsf(q.oz)) + 1e-30f;
        const float imax = fmaxf(fmaxf(fabsf(q.ix), fabsf(q.iy)), fabsf(q.iz));
        q.dt = 1e-5f * S * imax;
        q.tmax_ru = __double2float_ru(r.tmax);
        use_pf = isfinite(q.dt);
        // finite origin and reciprocals (dt is finite): no NaN in slab_nf
        if (use_pf) s3 = (r.ix < 0.0 ? 3 : 0) | (r.iy < 0.0 ? 12 : 0) | (r.iz < 0.0 ? 48 : 0);
      }
    }
    uint64_t mask = 0;
    uint32_t hyb = 0;
    int n_out = 0, n_in = 0;
    const uint32_t wmask = warp_bundle_mask(q, use_pf, valid, lane, n_obj, flo, fhi, all_obj, absmax);
    if (valid) {
      uint32_t pmask = 0;
      if (use_pf) {
#if NIF_RAY_PREFILTER
        uint32_t w = wmask;
        while (w) {
          const int k = __ffs(w) - 1;
          w &= w - 1;
          pmask |= (uint32_t)prefilter(q, flo[k], fhi[k]) << k;
        }
#else
        pmask = wmask;
#endif
      } else {
        pmask = all_obj;
      }
#ifdef NIF_GATHER_STATS
      atomicAdd(&g_gstats[0], 1ull);
      atomicAdd(&g_gstats[1], (unsigned long long)__popc(wmask));
      atomicAdd(&g_gstats[2], (unsigned long long)__popc(pmask));
#endif
      while (pmask) {
        const int k = __ffs(pmask) - 1;
        pmask &= pmask - 1;
        int kind;
        if (NIF_SLAB_NF && s3 >= 0) {
          kind = classify_nf(r, objs[k], test_box, s.tol, s3);
        } else {
          double t0;
          kind = classify_obj(r, objs[k], test_box, s.tol, &t0);
        }
        if (kind == 0) continue;
#ifdef NIF_GATHER_STATS
        atomicAdd(&g_gstats[3], 1ull);
#endif
        if (objs[k].route == 1) {
          mask |= (uint64_t)kind << (2 * k);
          if (kind == 1) ++n_out;
          else ++n_in;
        } else {
          hyb |= 1u << k;
        }
      }
      bool occ = false;
      uint32_t h = hyb;
      while (h != 0 && !occ) {
        const int k = __ffs(h) - 1;
        h &= h - 1;
        occ = occluded_in_object(s.nodes, s.tris, objs[k].root, r.ox, r.oy, r.oz, r.dx, r.dy,
                                 r.dz, s.eps, r.tmax);
      }
      out.bvh_occ[i] = occ ? 1 : 0;
    }
    // warp-level reservation of this chunk's records
    const int packed = (n_out << 16) | n_in;
    int incl = packed;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    if (tot == 0) continue;
    // one 64-bit atomic per chunk reserves both queues: outer count in the
    // high word, inner in the low word (each < 2^31 by the slot bound)
    unsigned long long base = 0;
    if (lane == 0)
      base = atomicAdd(reserve, ((unsigned long long)(tot >> 16) << 32) |
                                    (unsigned long long)(tot & 0xffff));
    base = __shfl_sync(0xffffffffu, base, 0);
    const int64_t base_o = (int64_t)(base >> 32);
    const int64_t base_i = (int64_t)(base & 0xffffffffull);
    const int excl = incl - packed;
    int64_t jo = base_o + (excl >> 16);
    int64_t ji = base_i + (excl & 0xffff);
    float du = 0.f, dv = 0.f;
    if (mask != 0) sph32f((float)r.dx, (float)r.dy, (float)r.dz, 1.0f, &du, &dv);
    uint64_t m = mask;
    while (m != 0) {
      const int bit = __ffsll((long long)m) - 1;
      const int k = bit >> 1;
      const int kind = (int)((m >> (2 * k)) & 3);
      m &= ~(3ull << (2 * k));
      const ObjC& b = objs[k];
#if NIF_EMIT_UNIFIED
      // one path for both kinds (a warp mixing outer and inner records no
      // longer runs the map twice): the record point is the entry point
      // o + t0 d (outer, same fp64 expression) or the origin (inner)
      const bool outer = kind == 1;
      double px = r.ox, py = r.oy, pz = r.oz;
      if (outer) {
        const Hit3 hh = (NIF_SLAB_NF && s3 >= 0) ? slab_nf(r, b, s3) : slab(r, b);
        px = r.ox + hh.t0 * r.dx;
        py = r.oy + hh.t0 * r.dy;
        pz = r.oz + hh.t0 * r.dz;
      }
      const double rx = px - b.c[0], ry = py - b.c[1], rz = pz - b.c[2];
      float rnf, rinvf, c0 = 0.5f, c1 = 0.5f, rr = 0.f;
      const bool deg = degenerate_f32(rx, ry, rz, &rnf, &rinvf);
      if (!deg) {
        sph32f((float)rx, (float)ry, (float)rz, rinvf, &c0, &c1);
        rr = fminf(rnf * b.hinv, 1.0f);  // within 1 ulp of rnf / hn (fp32); inner only
      }
      const int64_t j = outer ? jo : ji;
      if (j < (outer ? out.cap_outer : out.cap_inner)) {
        (outer ? out.outer_obj : out.inner_obj)[j] = b.id;
        (outer ? out.outer_ray : out.inner_ray)[j] = (int32_t)i;
        reinterpret_cast<float4*>(outer ? out.outer_coord : out.inner_coord)[j] =
            make_float4(c0, c1, du, dv);
        if (!outer) out.inner_r[j] = rr;
      }
      jo += outer ? 1 : 0;
      ji += outer ? 0 : 1;
      deg_count += deg ? 1 : 0;
#else
      float c0, c1, rr = 0.f;
      float rnf, rinvf;
      bool deg;
      if (kind == 1) {
        const Hit3 hh = (NIF_SLAB_NF && s3 >= 0) ? slab_nf(r, b, s3) : slab(r, b);
        const double ex = r.ox + hh.t0 * r.dx, ey = r.oy + hh.t0 * r.dy, ez = r.oz + hh.t0 * r.dz;
        const double rx = ex - b.c[0], ry = ey - b.c[1], rz = ez - b.c[2];
        deg = degenerate_f32(rx, ry, rz, &rnf, &rinvf);
        if (deg) { c0 = 0.5f; c1 = 0.5f; }
        else sph32f((float)rx, (float)ry, (float)rz, rinvf, &c0, &c1);
        if (jo < out.cap_outer) {
          out.outer_obj[jo] = b.id;
          out.outer_ray[jo] = (int32_t)i;
          reinterpret_cast<float4*>(out.outer_coord)[jo] = make_float4(c0, c1, du, dv);
        }
        ++jo;
      } else {
        const double rx = r.ox - b.c[0], ry = r.oy - b.c[1], rz = r.oz - b.c[2];
        deg = degenerate_f32(rx, ry, rz, &rnf, &rinvf);
        if (deg) { c0 = 0.5f; c1 = 0.5f; rr = 0.f; }
        else {
          sph32f((float)rx, (float)ry, (float)rz, rinvf, &c0, &c1);
          rr = fminf(rnf * b.hinv, 1.0f);  // within 1 ulp of rnf / hn (fp32)
        }
        if (ji < out.cap_inner) {
          out.inner_obj[ji] = b.id;
          out.inner_ray[ji] = (int32_t)i;
          reinterpret_cast<float4*>(out.inner_coord)[ji] = make_float4(c0, c1, du, dv);
          out.inner_r[ji] = rr;
        }
        ++ji;
      }
      deg_count += deg ? 1 : 0;
#endif
    }
  }
  const int dsum = __reduce_add_sync(0xffffffffu, deg_count);
  if (lane == 0 && dsum) atomicAdd(deg_acc, (unsigned long long)dsum);
  if (wtl) {
    wtl[2] = globaltimer();
    wtl[3] = (unsigned long long)n_done;
  }
  // the last CTA to finish publishes the queue lengths
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last && tid == 0) {
    const unsigned long long v = atomicAdd(reserve, 0ull);
    out.counts[0] = (int64_t)(v >> 32);
    out.counts[1] = (int64_t)(v & 0xffffffffull);
    out.counts[2] = out.counts[0] + out.counts[1];
    out.counts[3] = (int64_t)atomicAdd(deg_acc, 0ull);
    // every other CTA is done: re-arm the counters for the next call
    *reserve = 0ull;
    *deg_acc = 0ull;
    *tail = 0u;
    *done = 0u;
  }
}

long long* g_gprof = nullptr;  // diagnostic phase stamps (nif_debug_set_prof_gather)
int g_gather_cpsm = 0;     // CTAs per SM of the hot-path gather grid (0: NIF_GATHER_MINB_U)
int g_gather_dyn = 0;      // static rounds of the hot-path gather handed out on demand instead
unsigned long long* g_tl_gather = nullptr;  // nif_debug_set_timeline_gather
int g_gather_variant = 0;  // 0 unordered warp chunks, 1 one tile per CTA, 2 persistent ordered

size_t fused_ws(int64_t n) {
  const int64_t tiles = (n + kThreads - 1) / kThreads;
  return align_up((size_t)(tiles > 0 ? tiles : 1) * 8, 256) + 256;
}

}  // namespace
}  // namespace nif

using namespace nif;

// Workspace: a fixed header [0, kGatherHdr) -- the hot-path kernel's
// counters (reservation, CTA done, degenerate sum; the remainder-chunk tail
// on its own line), zero on entry (zero-filled workspace, re-armed by the
// kernel's last CTA) -- then the per-variant scratch (look-back status
// words / two-pass buffers).
constexpr size_t kGatherHdr = 256;

extern "C" size_t nif_gather_workspace_bytes(int64_t n) {
  const size_t a = gather_two_pass_workspace(n), b = fused_ws(n);
  return kGatherHdr + (a > b ? a : b);
}

extern "C" int nif_gather_dev(const nif_scene_view* s, const uint8_t* route,
                              const double* origins, const double* dirs, const double* tmaxs,
                              int64_t n, const nif_gather_out* out, void* workspace,
                              size_t workspace_bytes, void* stream) {
  if (n < 0) return fail(NIF_ERR_VALUE, "ray count cannot be negative");
  if (n >= (int64_t)1 << 31) return fail(NIF_ERR_VALUE, "at most 2^31-1 rays per gather");
  if ((uint64_t)n * (uint64_t)(s->n_obj > 0 ? s->n_obj : 1) >= ((uint64_t)1 << 31))
    return fail(NIF_ERR_VALUE, "gather exceeds 2^31 record slots; split the ray batch");
  if (workspace_bytes < nif_gather_workspace_bytes(n))
    return fail(NIF_ERR_VALUE, "gather workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* hdr = (uint8_t*)workspace;
  uint8_t* ws = hdr + kGatherHdr;
  const size_t ws_bytes = workspace_bytes - kGatherHdr;
  const bool unordered = out->rec_kind == nullptr && g_gprof == nullptr && g_gather_variant == 0;
  const bool warp_path = n > 0 && s->n_obj <= kMaxObjFused && unordered;
  // the hot-path kernel writes all four counts itself
  if (!warp_path) cudaMemsetAsync(out->counts, 0, 4 * sizeof(int64_t), st);
  // the hot-path kernel re-arms its own counters (its last CTA zeroes them
  // after publishing the counts): no memset node in front of it (-2 us per
  // pass at C2); every other path zeroes the header itself
  if (!warp_path) cudaMemsetAsync(hdr, 0, kGatherHdr, st);
  int rc = NIF_OK;
  if (n == 0) {
    rc = check_launch("gather(empty)");
  } else if (s->n_obj > kMaxObjFused) {
    rc = gather_two_pass(s, route, origins, dirs, tmaxs, n, out, ws, ws_bytes, st);
  } else if (warp_path) {
    const int64_t chunks = (n + 31) / 32;
    int64_t grid = (int64_t)sm_count() * (g_gather_cpsm > 0 ? g_gather_cpsm : NIF_GATHER_MINB_U);
    if (grid * (kThreads / 32) > chunks) grid = (chunks + kThreads / 32 - 1) / (kThreads / 32);
    gather_warp_kernel<<<(unsigned)grid, kThreads, 0, st>>>(
        *s, route, origins, dirs, tmaxs, n, *out, (unsigned long long*)hdr,
        (unsigned int*)(hdr + 8), (unsigned int*)(hdr + 128), (unsigned long long*)(hdr + 16),
        g_gather_dyn, g_tl_gather);
    rc = check_launch("nif_gather_dev");
  } else {
    const int64_t tiles = (n + kThreads - 1) / kThreads;
    unsigned long long* status = (unsigned long long*)ws;
    int* ctr = (int*)(ws + align_up((size_t)tiles * 8, 256));
    cudaMemsetAsync(ws, 0, align_up((size_t)tiles * 8, 256) + 256, st);
    if (out->rec_kind != nullptr)
      gather_fused_kernel<true><<<(unsigned)tiles, kThreads, 0, st>>>(
          *s, route, origins, dirs, tmaxs, n, *out, status, ctr, tiles, g_gprof);
    else if (g_gprof != nullptr || g_gather_variant == 1)
      gather_fused_kernel<false><<<(unsigned)tiles, kThreads, 0, st>>>(
          *s, route, origins, dirs, tmaxs, n, *out, status, ctr, tiles, g_gprof);
    else {
      const int smem = kStages * kStageBytes;
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(gather_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem);
        attr = true;
      }
      int64_t grid = (int64_t)sm_count() * NIF_GATHER_MINB;
      if (grid > tiles) grid = tiles;
      gather_persist_kernel<<<(unsigned)grid, kThreads, smem, st>>>(
          *s, route, origins, dirs, tmaxs, n, *out, status, ctr, tiles);
    }
    rc = check_launch("nif_gather_dev");
  }
  return rc;
}

extern "C" int nif_debug_set_prof_gather(void* buf) {
  g_gprof = (long long*)buf;
  return NIF_OK;
}

extern "C" int nif_debug_gather_stats(unsigned long long* out) {
#ifdef NIF_GATHER_STATS
  cudaMemcpyFromSymbol(out, g_gstats, sizeof(unsigned long long) * 4);
  unsigned long long z[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(g_gstats, z, sizeof(z));
  return NIF_OK;
#else
  (void)out;
  return fail(NIF_ERR_UNSUPPORTED, "built without NIF_GATHER_STATS");
#endif
}

extern "C" int nif_debug_set_timeline_gather(void* buf) {
  g_tl_gather = (unsigned long long*)buf;
  return NIF_OK;
}

extern "C" int nif_debug_set_gather_dynamic(int rounds) {
  g_gather_dyn = rounds < 0 ? 0 : rounds;
  return NIF_OK;
}

extern "C" int nif_debug_set_gather_grid(int ctas_per_sm) {
  g_gather_cpsm = ctas_per_sm;
  return NIF_OK;
}

extern "C" int nif_debug_set_gather_variant(int v) {
  g_gather_variant = v;
  return NIF_OK;
}
