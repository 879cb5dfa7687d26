// fp64 geometry cores shared by the gather, label, comparator and
// primary-ray kernels. Each function restates a reference numba core in the
// same operation order; the translation units that include this header are
// compiled with -fmad=false so no multiply-add is contracted (numba emits
// none), which keeps slab tests, containment and Moller-Trumbore bit-exact.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "nif_b200.h"

namespace nif {

constexpr double kPi = 3.141592653589793;
constexpr double kTwoPi = 2.0 * 3.141592653589793;
constexpr double kDegenerateRadius = 1e-9;  // geometry.py:22
constexpr int kStack = 120;  // device traversal stack: bvh.py:26 MAX_DEPTH

struct Hit3 {
  bool hit;
  double t0, t1;
};

// geometry.py:152-196 (_ray_aabb)
__device__ __forceinline__ Hit3 ray_aabb(double ox, double oy, double oz, double dx, double dy,
                                         double dz, double lx, double ly, double lz, double hx,
                                         double hy, double hz) {
  double t0 = -CUDART_INF, t1 = CUDART_INF;
  if (dx != 0.0) {
    double inv = 1.0 / dx;
    double ta = (lx - ox) * inv, tb = (hx - ox) * inv;
    if (ta > tb) { double s = ta; ta = tb; tb = s; }
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  } else if (ox < lx || ox > hx) {
    return {false, 0.0, 0.0};
  }
  if (dy != 0.0) {
    double inv = 1.0 / dy;
    double ta = (ly - oy) * inv, tb = (hy - oy) * inv;
    if (ta > tb) { double s = ta; ta = tb; tb = s; }
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  } else if (oy < ly || oy > hy) {
    return {false, 0.0, 0.0};
  }
  if (dz != 0.0) {
    double inv = 1.0 / dz;
    double ta = (lz - oz) * inv, tb = (hz - oz) * inv;
    if (ta > tb) { double s = ta; ta = tb; tb = s; }
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  } else if (oz < lz || oz > hz) {
    return {false, 0.0, 0.0};
  }
  if (t1 < t0 || t1 < 0.0) return {false, t0, t1};
  return {true, t0, t1};
}

// bvh.py:446-451 (_window_hit)
__device__ __forceinline__ bool window_hit(double ox, double oy, double oz, double dx, double dy,
                                           double dz, const double* lo, const double* hi,
                                           double t_floor, double t_cap, double* t0_out) {
  Hit3 h = ray_aabb(ox, oy, oz, dx, dy, dz, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
  if (t0_out) *t0_out = h.t0;
  return h.hit && h.t0 <= t_cap && h.t1 >= t_floor;
}

// geometry.py:199-230 (_ray_triangle): returns t (< 0 on miss)
__device__ __forceinline__ double ray_triangle(double ox, double oy, double oz, double dx,
                                               double dy, double dz, const double* v,
                                               double* b1_out = nullptr,
                                               double* b2_out = nullptr) {
  const double ax = v[0], ay = v[1], az = v[2];
  const double e1x = v[3] - ax, e1y = v[4] - ay, e1z = v[5] - az;
  const double e2x = v[6] - ax, e2y = v[7] - ay, e2z = v[8] - az;
  const double px = dy * e2z - dz * e2y;
  const double py = dz * e2x - dx * e2z;
  const double pz = dx * e2y - dy * e2x;
  const double det = e1x * px + e1y * py + e1z * pz;
  if (-1e-12 < det && det < 1e-12) return -1.0;
  const double inv = 1.0 / det;
  const double sx = ox - ax, sy = oy - ay, sz = oz - az;
  const double b1 = (sx * px + sy * py + sz * pz) * inv;
  if (b1 < 0.0 || b1 > 1.0) return -1.0;
  const double qx = sy * e1z - sz * e1y;
  const double qy = sz * e1x - sx * e1z;
  const double qz = sx * e1y - sy * e1x;
  const double b2 = (dx * qx + dy * qy + dz * qz) * inv;
  if (b2 < 0.0 || b1 + b2 > 1.0) return -1.0;
  const double t = (e2x * qx + e2y * qy + e2z * qz) * inv;
  if (t <= 0.0) return -1.0;
  if (b1_out) *b1_out = b1;
  if (b2_out) *b2_out = b2;
  return t;
}

// geometry.py:233-246 (_dir_to_spherical)
__device__ __forceinline__ void dir_to_spherical(double dx, double dy, double dz, double* u,
                                                 double* v) {
  double uu = (atan2(dy, dx) + kPi) / kTwoPi;
  if (uu >= 1.0) uu -= 1.0;
  else if (uu < 0.0) uu += 1.0;
  double z = dz;
  if (z > 1.0) z = 1.0;
  else if (z < -1.0) z = -1.0;
  *u = uu;
  *v = acos(z) / kPi;
}

// geometry.py:257-263 (_box_contains)
__device__ __forceinline__ bool box_contains(double px, double py, double pz, const double* lo,
                                             const double* hi, double tol) {
  return (lo[0] - tol <= px && px <= hi[0] + tol) && (lo[1] - tol <= py && py <= hi[1] + tol) &&
         (lo[2] - tol <= pz && pz <= hi[2] + tol);
}

// geometry.py:266-289 (_transform_outer); returns degenerate flag
__device__ __forceinline__ bool transform_outer(double ox, double oy, double oz, double dx,
                                                double dy, double dz, const double* lo,
                                                const double* hi, double t_enter, double c[4]) {
  const double ex = ox + t_enter * dx, ey = oy + t_enter * dy, ez = oz + t_enter * dz;
  const double cx = 0.5 * (lo[0] + hi[0]), cy = 0.5 * (lo[1] + hi[1]), cz = 0.5 * (lo[2] + hi[2]);
  const double rx = ex - cx, ry = ey - cy, rz = ez - cz;
  const double rn = sqrt(rx * rx + ry * ry + rz * rz);
  bool deg;
  if (rn < kDegenerateRadius) {
    c[0] = 0.5;
    c[1] = 0.5;
    deg = true;
  } else {
    dir_to_spherical(rx / rn, ry / rn, rz / rn, &c[0], &c[1]);
    deg = false;
  }
  dir_to_spherical(dx, dy, dz, &c[2], &c[3]);
  return deg;
}

// geometry.py:292-317 (_transform_inner); c[4] = r'
__device__ __forceinline__ bool transform_inner(double px, double py, double pz, double dx,
                                                double dy, double dz, const double* lo,
                                                const double* hi, double c[5]) {
  const double cx = 0.5 * (lo[0] + hi[0]), cy = 0.5 * (lo[1] + hi[1]), cz = 0.5 * (lo[2] + hi[2]);
  const double rx = px - cx, ry = py - cy, rz = pz - cz;
  const double rn = sqrt(rx * rx + ry * ry + rz * rz);
  const double hx = 0.5 * (hi[0] - lo[0]), hy = 0.5 * (hi[1] - lo[1]), hz = 0.5 * (hi[2] - lo[2]);
  const double hn = sqrt(hx * hx + hy * hy + hz * hz);
  bool deg;
  if (rn < kDegenerateRadius) {
    c[0] = 0.5;
    c[1] = 0.5;
    c[4] = 0.0;
    deg = true;
  } else {
    dir_to_spherical(rx / rn, ry / rn, rz / rn, &c[0], &c[1]);
    double r = rn / hn;
    if (r > 1.0) r = 1.0;
    c[4] = r;
    deg = false;
  }
  dir_to_spherical(dx, dy, dz, &c[2], &c[3]);
  return deg;
}

// bvh.py:524-576 (_occluded_in_object): any-hit in one object's subtree
// with t in (eps, t_max); children visited left first, right pushed.
static __device__ __noinline__ bool occluded_in_object(const nif_node* __restrict__ nodes,
                                                const double* __restrict__ tris, int root,
                                                double ox, double oy, double oz, double dx,
                                                double dy, double dz, double eps,
                                                double t_max) {
  int stack[kStack];
  int sp = 0;
  int node = root;
  while (node >= 0) {
    int descend = -1;
    const nif_node& nd = nodes[node];
    if (nd.leaf == 1) {
      const int first = nd.a, cnt = nd.b;
      for (int i = first; i < first + cnt; ++i) {
        const double t = ray_triangle(ox, oy, oz, dx, dy, dz, tris + (size_t)i * 9);
        if (t > eps && t < t_max) return true;
      }
    } else {
      const int l = nd.a, r = nd.b;
      const bool hl = window_hit(ox, oy, oz, dx, dy, dz, nodes[l].lo, nodes[l].hi, eps, t_max,
                                 nullptr);
      const bool hr = window_hit(ox, oy, oz, dx, dy, dz, nodes[r].lo, nodes[r].hi, eps, t_max,
                                 nullptr);
      if (hl && hr) {
        stack[sp++] = r;
        descend = l;
      } else if (hl) {
        descend = l;
      } else if (hr) {
        descend = r;
      }
    }
    if (descend >= 0) node = descend;
    else if (sp > 0) node = stack[--sp];
    else node = -1;
  }
  return false;
}

// bvh.py:454-521 (_closest_in_object): nearest triangle with t in
// (eps, t_best); near child first, far child pushed with its entry t.
static __device__ __noinline__ int closest_in_object(const nif_node* __restrict__ nodes,
                                              const double* __restrict__ tris, int root, double ox,
                                              double oy, double oz, double dx, double dy,
                                              double dz, double eps, double* t_best_io,
                                              double* bu_out, double* bv_out) {
  int stack[kStack];
  double tstack[kStack];
  double t_best = *t_best_io;
  int best = -1;
  double bu = 0.0, bv = 0.0;
  int sp = 0;
  int node = root;
  while (node >= 0) {
    int descend = -1;
    const nif_node& nd = nodes[node];
    if (nd.leaf == 1) {
      const int first = nd.a, cnt = nd.b;
      for (int i = first; i < first + cnt; ++i) {
        double u, v;
        const double t = ray_triangle(ox, oy, oz, dx, dy, dz, tris + (size_t)i * 9, &u, &v);
        if (t > eps && t < t_best) {
          t_best = t;
          best = i;
          bu = u;
          bv = v;
        }
      }
    } else {
      int l = nd.a, r = nd.b;
      double tl, tr;
      const bool hl = window_hit(ox, oy, oz, dx, dy, dz, nodes[l].lo, nodes[l].hi, eps, t_best,
                                 &tl);
      const bool hr = window_hit(ox, oy, oz, dx, dy, dz, nodes[r].lo, nodes[r].hi, eps, t_best,
                                 &tr);
      if (hl && hr) {
        if (tl > tr) {
          int s = l; l = r; r = s;
          double st = tl; tl = tr; tr = st;
        }
        stack[sp] = r;
        tstack[sp] = tr;
        ++sp;
        descend = l;
      } else if (hl) {
        descend = l;
      } else if (hr) {
        descend = r;
      }
    }
    if (descend >= 0) {
      node = descend;
    } else {
      node = -1;
      while (sp > 0) {
        --sp;
        if (tstack[sp] < t_best) {
          node = stack[sp];
          break;
        }
      }
    }
  }
  *t_best_io = t_best;
  *bu_out = bu;
  *bv_out = bv;
  return best;
}

}  // namespace nif
