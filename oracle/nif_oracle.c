/*
 * TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT.
 *
 * CPU restatement of the reference NIF path (niftrace, pure Python + numba
 * at /root/reference/pkg/src/niftrace) used as the parity oracle by tests/,
 * __graft_entry__.smoke() and the cpu_baseline leg of bench.py only. Each
 * function cites the reference lines it follows and keeps their operation
 * order; compiled with -ffp-contract=off (numba emits no FMA), so results
 * are bit-identical to the reference's kernels. Pinned against golden
 * vectors produced by the reference itself (tests/golden/make_golden.py).
 *
 * Array layouts are the reference's ScenePack layout (bvh.py:958-997):
 * separate [n][3] float64 arrays, int64 node words, uint8 leaf flags.
 * Loops over rays / records are OpenMP-parallel; every item is
 * independent, so results do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAX_DEPTH 120 /* bvh.py:26 */
#define CONTAINMENT_TOL 1e-6
#define DEGENERATE_RADIUS 1e-9
#define PI 3.141592653589793
#define TWO_PI (2.0 * 3.141592653589793)

/* ---- geometry.py:152-196 (_ray_aabb) ---------------------------------- */
static int ray_aabb(double ox, double oy, double oz, double dx, double dy, double dz,
                    double lx, double ly, double lz, double hx, double hy, double hz,
                    double* t0o, double* t1o) {
  double t0 = -INFINITY, t1 = INFINITY, inv, ta, tb, s;
  if (dx != 0.0) {
    inv = 1.0 / dx; ta = (lx - ox) * inv; tb = (hx - ox) * inv;
    if (ta > tb) { s = ta; ta = tb; tb = s; }
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  } else if (ox < lx || ox > hx) { *t0o = 0.0; *t1o = 0.0; return 0; }
  if (dy != 0.0) {
    inv = 1.0 / dy; ta = (ly - oy) * inv; tb = (hy - oy) * inv;
    if (ta > tb) { s = ta; ta = tb; tb = s; }
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  } else if (oy < ly || oy > hy) { *t0o = 0.0; *t1o = 0.0; return 0; }
  if (dz != 0.0) {
    inv = 1.0 / dz; ta = (lz - oz) * inv; tb = (hz - oz) * inv;
    if (ta > tb) { s = ta; ta = tb; tb = s; }
    if (ta > t0) t0 = ta;
    if (tb < t1) t1 = tb;
  } else if (oz < lz || oz > hz) { *t0o = 0.0; *t1o = 0.0; return 0; }
  *t0o = t0; *t1o = t1;
  if (t1 < t0 || t1 < 0.0) return 0;
  return 1;
}

/* ---- bvh.py:446-451 (_window_hit) -------------------------------------- */
static int window_hit(double ox, double oy, double oz, double dx, double dy, double dz,
                      const double* lo, const double* hi, double t_floor, double t_cap,
                      double* t0o) {
  double t0, t1;
  int hit = ray_aabb(ox, oy, oz, dx, dy, dz, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], &t0, &t1);
  *t0o = t0;
  return hit && t0 <= t_cap && t1 >= t_floor;
}

/* ---- geometry.py:199-230 (_ray_triangle) ------------------------------- */
static double ray_triangle(double ox, double oy, double oz, double dx, double dy, double dz,
                           const double* a, const double* b, const double* c,
                           double* b1o, double* b2o) {
  double e1x = b[0] - a[0], e1y = b[1] - a[1], e1z = b[2] - a[2];
  double e2x = c[0] - a[0], e2y = c[1] - a[1], e2z = c[2] - a[2];
  double px = dy * e2z - dz * e2y;
  double py = dz * e2x - dx * e2z;
  double pz = dx * e2y - dy * e2x;
  double det = e1x * px + e1y * py + e1z * pz;
  if (-1e-12 < det && det < 1e-12) return -1.0;
  double inv = 1.0 / det;
  double sx = ox - a[0], sy = oy - a[1], sz = oz - a[2];
  double b1 = (sx * px + sy * py + sz * pz) * inv;
  if (b1 < 0.0 || b1 > 1.0) return -1.0;
  double qx = sy * e1z - sz * e1y;
  double qy = sz * e1x - sx * e1z;
  double qz = sx * e1y - sy * e1x;
  double b2 = (dx * qx + dy * qy + dz * qz) * inv;
  if (b2 < 0.0 || b1 + b2 > 1.0) return -1.0;
  double t = (e2x * qx + e2y * qy + e2z * qz) * inv;
  if (t <= 0.0) return -1.0;
  if (b1o) *b1o = b1;
  if (b2o) *b2o = b2;
  return t;
}

/* ---- geometry.py:233-246 (_dir_to_spherical) --------------------------- */
static void dir_to_spherical(double dx, double dy, double dz, double* u, double* v) {
  double uu = (atan2(dy, dx) + PI) / TWO_PI;
  if (uu >= 1.0) uu -= 1.0;
  else if (uu < 0.0) uu += 1.0;
  double z = dz;
  if (z > 1.0) z = 1.0;
  else if (z < -1.0) z = -1.0;
  *u = uu;
  *v = acos(z) / PI;
}

/* ---- geometry.py:257-263 ------------------------------------------------ */
static int box_contains(double px, double py, double pz, const double* lo, const double* hi,
                        double tol) {
  return (lo[0] - tol <= px && px <= hi[0] + tol) && (lo[1] - tol <= py && py <= hi[1] + tol) &&
         (lo[2] - tol <= pz && pz <= hi[2] + tol);
}

/* ---- geometry.py:266-289 ------------------------------------------------ */
static int transform_outer(double ox, double oy, double oz, double dx, double dy, double dz,
                           const double* lo, const double* hi, double t_enter, double* c) {
  double ex = ox + t_enter * dx, ey = oy + t_enter * dy, ez = oz + t_enter * dz;
  double cx = 0.5 * (lo[0] + hi[0]), cy = 0.5 * (lo[1] + hi[1]), cz = 0.5 * (lo[2] + hi[2]);
  double rx = ex - cx, ry = ey - cy, rz = ez - cz;
  double rn = sqrt(rx * rx + ry * ry + rz * rz);
  int deg;
  if (rn < DEGENERATE_RADIUS) { c[0] = 0.5; c[1] = 0.5; deg = 1; }
  else { dir_to_spherical(rx / rn, ry / rn, rz / rn, &c[0], &c[1]); deg = 0; }
  dir_to_spherical(dx, dy, dz, &c[2], &c[3]);
  return deg;
}

/* ---- geometry.py:292-317 ------------------------------------------------ */
static int transform_inner(double px, double py, double pz, double dx, double dy, double dz,
                           const double* lo, const double* hi, double* c) {
  double cx = 0.5 * (lo[0] + hi[0]), cy = 0.5 * (lo[1] + hi[1]), cz = 0.5 * (lo[2] + hi[2]);
  double rx = px - cx, ry = py - cy, rz = pz - cz;
  double rn = sqrt(rx * rx + ry * ry + rz * rz);
  double hx = 0.5 * (hi[0] - lo[0]), hy = 0.5 * (hi[1] - lo[1]), hz = 0.5 * (hi[2] - lo[2]);
  double hn = sqrt(hx * hx + hy * hy + hz * hz);
  int deg;
  if (rn < DEGENERATE_RADIUS) { c[0] = 0.5; c[1] = 0.5; c[4] = 0.0; deg = 1; }
  else {
    dir_to_spherical(rx / rn, ry / rn, rz / rn, &c[0], &c[1]);
    double r = rn / hn;
    if (r > 1.0) r = 1.0;
    c[4] = r;
    deg = 0;
  }
  dir_to_spherical(dx, dy, dz, &c[2], &c[3]);
  return deg;
}

/* Scene arrays in the reference ScenePack layout. */
typedef struct {
  const double *t_lo, *t_hi;
  const int64_t *t_a, *t_b;
  const uint8_t* t_leaf;
  const int64_t* t_order;
  const int64_t* roots;
  const double *b_lo, *b_hi;
  const int64_t *b_a, *b_b;
  const uint8_t* b_leaf;
  const double *v0, *v1, *v2, *n0, *n1, *n2;
  const double *obox_lo, *obox_hi;
  int64_t n_obj;
  double eps;
} oscene;

/* ---- bvh.py:524-576 (_occluded_in_object) ------------------------------ */
static int occluded_in_object(const oscene* s, int64_t root, double ox, double oy, double oz,
                              double dx, double dy, double dz, double eps, double t_max) {
  int64_t stack[MAX_DEPTH];
  int sp = 0;
  int64_t node = root;
  double tl, tr;
  while (node >= 0) {
    int64_t descend = -1;
    if (s->b_leaf[node] == 1) {
      int64_t first = s->b_a[node];
      for (int64_t i = first; i < first + s->b_b[node]; ++i) {
        double t = ray_triangle(ox, oy, oz, dx, dy, dz, s->v0 + 3 * i, s->v1 + 3 * i,
                                s->v2 + 3 * i, NULL, NULL);
        if (t > eps && t < t_max) return 1;
      }
    } else {
      int64_t l = s->b_a[node], r = s->b_b[node];
      int hl = window_hit(ox, oy, oz, dx, dy, dz, s->b_lo + 3 * l, s->b_hi + 3 * l, eps, t_max, &tl);
      int hr = window_hit(ox, oy, oz, dx, dy, dz, s->b_lo + 3 * r, s->b_hi + 3 * r, eps, t_max, &tr);
      if (hl && hr) { stack[sp++] = r; descend = l; }
      else if (hl) descend = l;
      else if (hr) descend = r;
    }
    if (descend >= 0) node = descend;
    else if (sp > 0) node = stack[--sp];
    else node = -1;
  }
  return 0;
}

/* ---- bvh.py:454-521 (_closest_in_object) ------------------------------- */
static int64_t closest_in_object(const oscene* s, int64_t root, double ox, double oy, double oz,
                                 double dx, double dy, double dz, double eps, double* t_best_io,
                                 double* bu_o, double* bv_o) {
  int64_t stack[MAX_DEPTH];
  double tstack[MAX_DEPTH];
  double t_best = *t_best_io, bu = 0.0, bv = 0.0, tl, tr, u, v;
  int64_t best = -1;
  int sp = 0;
  int64_t node = root;
  while (node >= 0) {
    int64_t descend = -1;
    if (s->b_leaf[node] == 1) {
      int64_t first = s->b_a[node];
      for (int64_t i = first; i < first + s->b_b[node]; ++i) {
        double t = ray_triangle(ox, oy, oz, dx, dy, dz, s->v0 + 3 * i, s->v1 + 3 * i,
                                s->v2 + 3 * i, &u, &v);
        if (t > eps && t < t_best) { t_best = t; best = i; bu = u; bv = v; }
      }
    } else {
      int64_t l = s->b_a[node], r = s->b_b[node];
      int hl = window_hit(ox, oy, oz, dx, dy, dz, s->b_lo + 3 * l, s->b_hi + 3 * l, eps, t_best, &tl);
      int hr = window_hit(ox, oy, oz, dx, dy, dz, s->b_lo + 3 * r, s->b_hi + 3 * r, eps, t_best, &tr);
      if (hl && hr) {
        if (tl > tr) { int64_t q = l; l = r; r = q; double qt = tl; tl = tr; tr = qt; }
        stack[sp] = r; tstack[sp] = tr; ++sp; descend = l;
      } else if (hl) descend = l;
      else if (hr) descend = r;
    }
    if (descend >= 0) node = descend;
    else {
      node = -1;
      while (sp > 0) { --sp; if (tstack[sp] < t_best) { node = stack[sp]; break; } }
    }
  }
  *t_best_io = t_best; *bu_o = bu; *bv_o = bv;
  return best;
}

/* ---- bvh.py:579-647 (_scene_closest) ----------------------------------- */
static int64_t scene_closest(const oscene* s, double ox, double oy, double oz, double dx,
                             double dy, double dz, double eps, double* t_o, int64_t* obj_o,
                             double* bu_o, double* bv_o) {
  int64_t stack[MAX_DEPTH];
  double tstack[MAX_DEPTH];
  double t_best = INFINITY, bu = 0.0, bv = 0.0, tl, tr;
  int64_t best_obj = -1, best_slot = -1;
  int sp = 0;
  int64_t node = 0;
  while (node >= 0) {
    int64_t descend = -1;
    if (s->t_leaf[node] == 1) {
      int64_t first = s->t_a[node];
      for (int64_t i = first; i < first + s->t_b[node]; ++i) {
        int64_t o = s->t_order[i];
        double t = t_best, u, v;
        int64_t slot = closest_in_object(s, s->roots[o], ox, oy, oz, dx, dy, dz, eps, &t, &u, &v);
        if (slot >= 0) { t_best = t; best_obj = o; best_slot = slot; bu = u; bv = v; }
      }
    } else {
      int64_t l = s->t_a[node], r = s->t_b[node];
      int hl = window_hit(ox, oy, oz, dx, dy, dz, s->t_lo + 3 * l, s->t_hi + 3 * l, eps, t_best, &tl);
      int hr = window_hit(ox, oy, oz, dx, dy, dz, s->t_lo + 3 * r, s->t_hi + 3 * r, eps, t_best, &tr);
      if (hl && hr) {
        if (tl > tr) { int64_t q = l; l = r; r = q; double qt = tl; tl = tr; tr = qt; }
        stack[sp] = r; tstack[sp] = tr; ++sp; descend = l;
      } else if (hl) descend = l;
      else if (hr) descend = r;
    }
    if (descend >= 0) node = descend;
    else {
      node = -1;
      while (sp > 0) { --sp; if (tstack[sp] < t_best) { node = stack[sp]; break; } }
    }
  }
  *t_o = t_best; *obj_o = best_obj; *bu_o = bu; *bv_o = bv;
  return best_slot;
}

/* ---- bvh.py:650-700 (_scene_occluded), bvh.py:744-756 (_k_occluded) --- */
static int scene_occluded(const oscene* s, double ox, double oy, double oz, double dx, double dy,
                          double dz, double eps, double t_max) {
  int64_t stack[MAX_DEPTH];
  int sp = 0;
  int64_t node = 0;
  double tl, tr;
  while (node >= 0) {
    int64_t descend = -1;
    if (s->t_leaf[node] == 1) {
      int64_t first = s->t_a[node];
      for (int64_t i = first; i < first + s->t_b[node]; ++i) {
        int64_t o = s->t_order[i];
        if (occluded_in_object(s, s->roots[o], ox, oy, oz, dx, dy, dz, eps, t_max)) return 1;
      }
    } else {
      int64_t l = s->t_a[node], r = s->t_b[node];
      int hl = window_hit(ox, oy, oz, dx, dy, dz, s->t_lo + 3 * l, s->t_hi + 3 * l, eps, t_max, &tl);
      int hr = window_hit(ox, oy, oz, dx, dy, dz, s->t_lo + 3 * r, s->t_hi + 3 * r, eps, t_max, &tr);
      if (hl && hr) { stack[sp++] = r; descend = l; }
      else if (hl) descend = l;
      else if (hr) descend = r;
    }
    if (descend >= 0) node = descend;
    else if (sp > 0) node = stack[--sp];
    else node = -1;
  }
  return 0;
}

void oracle_occluded(const oscene* s, const double* o, const double* d, const double* tm,
                     int64_t n, uint8_t* out) {
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i)
    out[i] = (uint8_t)scene_occluded(s, o[3 * i], o[3 * i + 1], o[3 * i + 2], d[3 * i],
                                     d[3 * i + 1], d[3 * i + 2], s->eps, tm[i]);
}

/* ---- bvh.py:904-916 (_k_label_visible) --------------------------------- */
void oracle_label_visible(const oscene* s, const int32_t* rec_obj, const int32_t* rec_ray,
                          int64_t m, const double* o, const double* d, const double* tm,
                          uint8_t* vis) {
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t j = 0; j < m; ++j) {
    int64_t i = rec_ray[j];
    int occ = occluded_in_object(s, s->roots[rec_obj[j]], o[3 * i], o[3 * i + 1], o[3 * i + 2],
                                 d[3 * i], d[3 * i + 1], d[3 * i + 2], s->eps, tm[i]);
    vis[j] = occ ? 0 : 1;
  }
}

/* ---- bvh.py:772-901 (_k_gather_queries) --------------------------------
 * Dense per-ray slots [i*n_obj, (i+1)*n_obj) exactly as the reference; the
 * caller compacts by rec_kind != 255 (renderer.py:636-643). Top-level DFS
 * traversal as written in the reference (not the per-object shortcut the
 * CUDA kernel uses), so the parity test checks that shortcut.            */
void oracle_gather(const oscene* s, const uint8_t* route, const double* org, const double* dir,
                   const double* tms, int64_t n, double tol, uint8_t* rec_kind, int32_t* rec_obj,
                   int32_t* rec_ray, double* rec_coord, uint8_t* bvh_occ, int64_t* n_deg) {
  const int64_t n_obj = s->n_obj;
  int64_t deg_total = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : deg_total)
  for (int64_t i = 0; i < n; ++i) {
    int64_t cand[4096];
    int64_t stack[MAX_DEPTH];
    double ox = org[3 * i], oy = org[3 * i + 1], oz = org[3 * i + 2];
    double dx = dir[3 * i], dy = dir[3 * i + 1], dz = dir[3 * i + 2];
    double tmax = tms[i], tl, tr;
    int occ = 0;
    int64_t n_cand = 0;
    int sp = 0;
    int64_t node = 0;
    while (node >= 0) {
      int64_t descend = -1;
      if (s->t_leaf[node] == 1) {
        int64_t first = s->t_a[node];
        for (int64_t k = first; k < first + s->t_b[node]; ++k) cand[n_cand++] = s->t_order[k];
      } else {
        int64_t l = s->t_a[node], r = s->t_b[node];
        int hl = window_hit(ox, oy, oz, dx, dy, dz, s->t_lo + 3 * l, s->t_hi + 3 * l, -tol, tmax, &tl);
        int hr = window_hit(ox, oy, oz, dx, dy, dz, s->t_lo + 3 * r, s->t_hi + 3 * r, -tol, tmax, &tr);
        if (hl && hr) { stack[sp++] = r; descend = l; }
        else if (hl) descend = l;
        else if (hr) descend = r;
      }
      if (descend >= 0) node = descend;
      else if (sp > 0) node = stack[--sp];
      else node = -1;
    }
    int64_t base = i * n_obj, n_rec = 0;
    for (int64_t k = 0; k < n_cand; ++k) {
      int64_t o = cand[k];
      const double* lo = s->obox_lo + 3 * o;
      const double* hi = s->obox_hi + 3 * o;
      double c[5];
      if (box_contains(ox, oy, oz, lo, hi, tol)) {
        if (route[o] == 1) {
          int deg = transform_inner(ox, oy, oz, dx, dy, dz, lo, hi, c);
          int64_t slot = base + n_rec;
          rec_kind[slot] = 1; rec_obj[slot] = (int32_t)o; rec_ray[slot] = (int32_t)i;
          for (int q = 0; q < 5; ++q) rec_coord[slot * 5 + q] = c[q];
          ++n_rec;
          deg_total += deg;
        } else if (!occ) {
          occ = occluded_in_object(s, s->roots[o], ox, oy, oz, dx, dy, dz, s->eps, tmax);
        }
      } else {
        double t0, t1;
        int hit = ray_aabb(ox, oy, oz, dx, dy, dz, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], &t0, &t1);
        if (hit && t0 > 0.0 && t0 < tmax) {
          if (route[o] == 1) {
            int deg = transform_outer(ox, oy, oz, dx, dy, dz, lo, hi, t0, c);
            int64_t slot = base + n_rec;
            rec_kind[slot] = 0; rec_obj[slot] = (int32_t)o; rec_ray[slot] = (int32_t)i;
            for (int q = 0; q < 4; ++q) rec_coord[slot * 5 + q] = c[q];
            rec_coord[slot * 5 + 4] = 0.0;
            ++n_rec;
            deg_total += deg;
          } else if (!occ) {
            occ = occluded_in_object(s, s->roots[o], ox, oy, oz, dx, dy, dz, s->eps, tmax);
          }
        }
      }
    }
    for (int64_t k = n_rec; k < n_obj; ++k) rec_kind[base + k] = 255;
    bvh_occ[i] = occ ? 1 : 0;
  }
  *n_deg = deg_total;
}

/* ---- renderer.py:86-105 (stateless RNG) -------------------------------- */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static double rand01(uint64_t seed, uint64_t pixel, uint64_t sample, uint64_t draw) {
  uint64_t x = seed + 0x9E3779B97F4A7C15ull;
  x = mix64(x + pixel * 0xBF58476D1CE4E5B9ull);
  x = mix64(x + sample * 0x94D049BB133111EBull);
  x = mix64(x + draw * 0x9E3779B97F4A7C15ull);
  return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

/* ---- renderer.py:453-506 (_k_primary) + 509-532 (_k_light_sample) +
 *      535-547 (_k_uniform_dirs), point and area lights ------------------ */
void oracle_sample_pass(const oscene* s, const double* cam /* pos fwd right up tan aspect */,
                        int64_t width, int64_t height, const uint8_t* l_kind,
                        const double* l_data, const double* cum, int64_t n_lights,
                        uint64_t seed, uint64_t sample, int sampler, uint8_t* hit, double* t_out,
                        int32_t* obj_out, double* point, double* normal, double* pdir,
                        double* ldir, double* tmax_o, double* pdf_o, double* emit) {
  const int64_t n = width * height;
  const double cpx = cam[0], cpy = cam[1], cpz = cam[2];
  const double fx = cam[3], fy = cam[4], fz = cam[5];
  const double rx = cam[6], ry = cam[7], rz = cam[8];
  const double ux = cam[9], uy = cam[10], uz = cam[11];
  const double tan_half = cam[12], aspect = cam[13];
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i) {
    int64_t px = i % width, py = i / width;
    double jx = rand01(seed, i, sample, 0), jy = rand01(seed, i, sample, 1);
    double sx = (((double)px + jx) / (double)width) * 2.0 - 1.0;
    double sy = 1.0 - (((double)py + jy) / (double)height) * 2.0;
    double dx = fx + sx * tan_half * aspect * rx + sy * tan_half * ux;
    double dy = fy + sx * tan_half * aspect * ry + sy * tan_half * uy;
    double dz = fz + sx * tan_half * aspect * rz + sy * tan_half * uz;
    double dn = sqrt(dx * dx + dy * dy + dz * dz);
    dx /= dn; dy /= dn; dz /= dn;
    pdir[3 * i] = dx; pdir[3 * i + 1] = dy; pdir[3 * i + 2] = dz;
    double t, bu, bv;
    int64_t o;
    int64_t slot = scene_closest(s, cpx, cpy, cpz, dx, dy, dz, s->eps, &t, &o, &bu, &bv);
    double P[3] = {0, 0, 0}, N[3] = {0, 0, 0};
    if (slot >= 0) {
      hit[i] = 1; t_out[i] = t; obj_out[i] = (int32_t)o;
      P[0] = cpx + t * dx; P[1] = cpy + t * dy; P[2] = cpz + t * dz;
      double b0 = 1.0 - bu - bv;
      double nx = b0 * s->n0[3 * slot] + bu * s->n1[3 * slot] + bv * s->n2[3 * slot];
      double ny = b0 * s->n0[3 * slot + 1] + bu * s->n1[3 * slot + 1] + bv * s->n2[3 * slot + 1];
      double nz = b0 * s->n0[3 * slot + 2] + bu * s->n1[3 * slot + 2] + bv * s->n2[3 * slot + 2];
      double nn = sqrt(nx * nx + ny * ny + nz * nz);
      if (nn > 0.0) { nx /= nn; ny /= nn; nz /= nn; }
      N[0] = nx; N[1] = ny; N[2] = nz;
    } else {
      hit[i] = 0; t_out[i] = INFINITY; obj_out[i] = -1;
    }
    for (int c = 0; c < 3; ++c) { point[3 * i + c] = P[c]; normal[3 * i + c] = N[c]; }
    double ld[3] = {0, 0, 0}, em[3] = {0, 0, 0}, tmax = 0.0, pdf = 0.0;
    if (sampler == 1) {
      em[0] = em[1] = em[2] = 1.0;
      if (slot >= 0) {
        double u_a = rand01(seed, i, sample, 2), u_b = rand01(seed, i, sample, 3);
        double z = 1.0 - 2.0 * u_a;
        double q = 1.0 - z * z;
        double sq = sqrt(q > 0.0 ? q : 0.0);
        double phi = (2.0 * PI) * u_b;
        ld[0] = cos(phi) * sq; ld[1] = sin(phi) * sq; ld[2] = z;
        tmax = INFINITY; pdf = 1.0 / (4.0 * PI);
      }
    } else if (slot >= 0 && n_lights > 0) {
      double u_sel = rand01(seed, i, sample, 2), u_a = rand01(seed, i, sample, 3),
             u_b = rand01(seed, i, sample, 4);
      int64_t li = 0;
      while (li < n_lights && cum[li] <= u_sel) ++li;
      if (li >= n_lights) li = n_lights - 1;
      double sel_pmf = cum[li] - (li > 0 ? cum[li - 1] : 0.0);
      const double* L = l_data + 16 * li;
      if (l_kind[li] == 0) {
        double vx = L[0] - P[0], vy = L[1] - P[1], vz = L[2] - P[2];
        double dd = sqrt(vx * vx + vy * vy + vz * vz);
        if (dd <= 0.0) { ld[2] = 1.0; pdf = 1.0; }
        else {
          double inv = 1.0 / dd, inv2 = inv * inv;
          ld[0] = vx * inv; ld[1] = vy * inv; ld[2] = vz * inv;
          tmax = dd; pdf = sel_pmf;
          em[0] = L[3] * inv2; em[1] = L[4] * inv2; em[2] = L[5] * inv2;
        }
      } else {
        double sxp = L[0] + u_a * L[3] + u_b * L[6];
        double syp = L[1] + u_a * L[4] + u_b * L[7];
        double szp = L[2] + u_a * L[5] + u_b * L[8];
        double vx = sxp - P[0], vy = syp - P[1], vz = szp - P[2];
        double d2 = vx * vx + vy * vy + vz * vz;
        double dd = sqrt(d2);
        if (dd <= 0.0) { ld[2] = 1.0; pdf = 1.0; }
        else {
          double inv = 1.0 / dd;
          ld[0] = vx * inv; ld[1] = vy * inv; ld[2] = vz * inv;
          tmax = dd;
          double cos_l = -(ld[0] * L[12] + ld[1] * L[13] + ld[2] * L[14]);
          if (cos_l <= 0.0) pdf = sel_pmf;
          else { pdf = sel_pmf * d2 / (L[15] * cos_l); em[0] = L[9]; em[1] = L[10]; em[2] = L[11]; }
        }
      }
    }
    for (int c = 0; c < 3; ++c) { ldir[3 * i + c] = ld[c]; emit[3 * i + c] = em[c]; }
    tmax_o[i] = tmax; pdf_o[i] = pdf;
  }
}

/* ---- grids.py:125-162 / 187-191 + nif.py:286-311 (encode_*_arrays) ----- */
static void axis_indices(double x, int64_t R, int wrap, int64_t* i0o, int64_t* i1o, double* w) {
  double xc = x * (double)R - 0.5;
  double x0 = floor(xc);
  *w = xc - x0;
  int64_t i0 = (int64_t)x0, i1 = i0 + 1;
  if (wrap) { i0 = ((i0 % R) + R) % R; i1 = ((i1 % R) + R) % R; }
  else {
    i0 = i0 < 0 ? 0 : (i0 > R - 1 ? R - 1 : i0);
    i1 = i1 < 0 ? 0 : (i1 > R - 1 ? R - 1 : i1);
  }
  *i0o = i0; *i1o = i1;
}

static void lookup_2d(const float* g, int64_t R, int64_t N, double u, double v, double* out) {
  int64_t iu0, iu1, iv0, iv1;
  double wu, wv;
  axis_indices(u, R, 1, &iu0, &iu1, &wu);
  axis_indices(v, R, 0, &iv0, &iv1, &wv);
  double w00 = (1.0 - wu) * (1.0 - wv), w01 = (1.0 - wu) * wv, w10 = wu * (1.0 - wv), w11 = wu * wv;
  for (int64_t k = 0; k < N; ++k) {
    double s = w00 * (double)g[(iu0 * R + iv0) * N + k] + w01 * (double)g[(iu0 * R + iv1) * N + k] +
               w10 * (double)g[(iu1 * R + iv0) * N + k] + w11 * (double)g[(iu1 * R + iv1) * N + k];
    out[k] = (double)(float)s;
  }
}

static void lookup_1d(const float* g, int64_t R, int64_t N, double x, double* out) {
  int64_t i0, i1;
  double w;
  axis_indices(x, R, 0, &i0, &i1, &w);
  for (int64_t k = 0; k < N; ++k) {
    double s = (1.0 - w) * (double)g[i0 * N + k] + w * (double)g[i1 * N + k];
    out[k] = (double)(float)s;
  }
}

/* pos/dir: [n_obj][R][R][N]; dist: [n_obj][Rd][Nd] or NULL (outer). */
void oracle_encode(const float* pos, const float* dirg, const float* dist, int64_t R, int64_t N,
                   int64_t Rd, int64_t Nd, const int64_t* obj, const double* coord, int64_t m,
                   int64_t cw, double* out) {
  const int64_t in_dim = 2 * N + (dist ? Nd : 0);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < m; ++j) {
    const int64_t o = obj[j];
    const double* c = coord + j * cw;
    double* y = out + j * in_dim;
    lookup_2d(pos + o * R * R * N, R, N, c[0], c[1], y);
    lookup_2d(dirg + o * R * R * N, R, N, c[2], c[3], y + N);
    if (dist) lookup_1d(dist + o * Rd * Nd, Rd, Nd, c[4], y + 2 * N);
  }
}

/* ---- nif.py:321-359 (_k_dense_forward), rows [0, m) ------------------- */
void oracle_dense_forward(const float* w_flat, const float* b_flat, const int64_t* dims,
                          int64_t n_dims, int sigmoid_head, const double* x, int64_t m,
                          double* out) {
  int64_t md = 0;
  for (int64_t i = 0; i < n_dims; ++i) if (dims[i] > md) md = dims[i];
  const int64_t nl = n_dims - 1;
#pragma omp parallel
  {
    double* bufa0 = (double*)malloc(sizeof(double) * md);
    double* bufb0 = (double*)malloc(sizeof(double) * md);
#pragma omp for schedule(static)
    for (int64_t j = 0; j < m; ++j) {
      double *bufa = bufa0, *bufb = bufb0, *tmp;
      for (int64_t k = 0; k < dims[0]; ++k) bufa[k] = x[j * dims[0] + k];
      int64_t wo = 0, bo = 0;
      for (int64_t layer = 0; layer < nl; ++layer) {
        int64_t nin = dims[layer], nout = dims[layer + 1];
        for (int64_t o = 0; o < nout; ++o) {
          double acc = (double)b_flat[bo + o];
          int64_t base = wo + o * nin;
          for (int64_t k = 0; k < nin; ++k) acc += (double)w_flat[base + k] * bufa[k];
          if (layer < nl - 1) bufb[o] = acc > 0.0 ? acc : 0.01 * acc;
          else if (sigmoid_head == 1) {
            if (acc >= 0.0) bufb[o] = 1.0 / (1.0 + exp(-acc));
            else { double e = exp(acc); bufb[o] = e / (1.0 + e); }
          } else bufb[o] = acc;
        }
        wo += nin * nout;
        bo += nout;
        tmp = bufa; bufa = bufb; bufb = tmp;
      }
      for (int64_t k = 0; k < dims[nl]; ++k) out[j * dims[nl] + k] = bufa[k];
    }
    free(bufa0);
    free(bufb0);
  }
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---- bvh.py:34-303 (_build_sah) ----------------------------------------
 * Binned SAH, depth-first with an explicit stack, stable partition by bin
 * index, "halve by current order" when centroids collapse. Outputs sized
 * for 2n nodes; returns the node count. Single-threaded like the reference
 * (the order of the node ids is the reference's stack discipline). */
static int sah_bin(double c, double cmin, double ext, int64_t n_bins) {
  int64_t b = (int64_t)((double)n_bins * (c - cmin) / ext);
  if (b >= n_bins) b = n_bins - 1;
  if (b < 0) b = 0;
  return (int)b;
}

int64_t oracle_build_sah(const double* lo, const double* hi, const double* ce, int64_t n,
                         int64_t max_leaf, int64_t n_bins, double c_trav, double c_isect,
                         double* node_lo, double* node_hi, int64_t* node_a, int64_t* node_b,
                         uint8_t* node_leaf, int64_t* order) {
  int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t* stack = (int64_t*)malloc(sizeof(int64_t) * 3 * (size_t)(2 * n + 8));
  int64_t* bin_cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_bins);
  double* bin_lo = (double*)malloc(sizeof(double) * 3 * (size_t)n_bins);
  double* bin_hi = (double*)malloc(sizeof(double) * 3 * (size_t)n_bins);
  double* left_sa = (double*)malloc(sizeof(double) * (size_t)n_bins);
  double* right_sa = (double*)malloc(sizeof(double) * (size_t)n_bins);
  int64_t* left_n = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_bins);
  int64_t* right_n = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_bins);
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  for (int64_t i = 0; i < 2 * n; ++i) {
    node_a[i] = 0;
    node_b[i] = 0;
    node_leaf[i] = 0;
  }
  stack[0] = 0;
  stack[1] = 0;
  stack[2] = n;
  int64_t sp = 1, n_nodes = 1;
  while (sp > 0) {
    --sp;
    const int64_t idx = stack[3 * sp], start = stack[3 * sp + 1], end = stack[3 * sp + 2];
    const int64_t count = end - start;
    double bl[3] = {INFINITY, INFINITY, INFINITY}, bh[3] = {-INFINITY, -INFINITY, -INFINITY};
    double cl[3] = {INFINITY, INFINITY, INFINITY}, chh[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = start; i < end; ++i) {
      const int64_t p = order[i];
      for (int c = 0; c < 3; ++c) {
        if (lo[3 * p + c] < bl[c]) bl[c] = lo[3 * p + c];
        if (hi[3 * p + c] > bh[c]) bh[c] = hi[3 * p + c];
      }
      for (int c = 0; c < 3; ++c) {
        if (ce[3 * p + c] < cl[c]) cl[c] = ce[3 * p + c];
        if (ce[3 * p + c] > chh[c]) chh[c] = ce[3 * p + c];
      }
    }
    for (int c = 0; c < 3; ++c) {
      node_lo[3 * idx + c] = bl[c];
      node_hi[3 * idx + c] = bh[c];
    }
    double best_cost = INFINITY;
    int best_axis = -1;
    int64_t best_k = -1;
    if (count > 1) {
      const double dx = bh[0] - bl[0], dy = bh[1] - bl[1], dz = bh[2] - bl[2];
      const double sa_node = 2.0 * (dx * dy + dy * dz + dz * dx);
      if (sa_node > 1e-300) {
        for (int axis = 0; axis < 3; ++axis) {
          const double cmin = cl[axis], ext = chh[axis] - cl[axis];
          if (ext <= 0.0) continue;
          for (int64_t k = 0; k < n_bins; ++k) {
            bin_cnt[k] = 0;
            for (int c = 0; c < 3; ++c) {
              bin_lo[3 * k + c] = INFINITY;
              bin_hi[3 * k + c] = -INFINITY;
            }
          }
          for (int64_t i = start; i < end; ++i) {
            const int64_t p = order[i];
            const int b = sah_bin(ce[3 * p + axis], cmin, ext, n_bins);
            bin_cnt[b] += 1;
            for (int c = 0; c < 3; ++c) {
              if (lo[3 * p + c] < bin_lo[3 * b + c]) bin_lo[3 * b + c] = lo[3 * p + c];
              if (hi[3 * p + c] > bin_hi[3 * b + c]) bin_hi[3 * b + c] = hi[3 * p + c];
            }
          }
          for (int dir = 0; dir < 2; ++dir) {  /* left sweep, then right sweep */
            double a[3] = {INFINITY, INFINITY, INFINITY}, bb[3] = {-INFINITY, -INFINITY, -INFINITY};
            int64_t cnt = 0;
            for (int64_t j = 0; j < n_bins; ++j) {
              const int64_t k = dir == 0 ? j : n_bins - 1 - j;
              if (bin_cnt[k] > 0)
                for (int c = 0; c < 3; ++c) {
                  if (bin_lo[3 * k + c] < a[c]) a[c] = bin_lo[3 * k + c];
                  if (bin_hi[3 * k + c] > bb[c]) bb[c] = bin_hi[3 * k + c];
                }
              cnt += bin_cnt[k];
              double sa = 0.0;
              if (cnt > 0) {
                const double ex = bb[0] - a[0], ey = bb[1] - a[1], ez = bb[2] - a[2];
                sa = 2.0 * (ex * ey + ey * ez + ez * ex);
              }
              if (dir == 0) {
                left_n[k] = cnt;
                left_sa[k] = sa;
              } else {
                right_n[k] = cnt;
                right_sa[k] = sa;
              }
            }
          }
          for (int64_t k = 0; k < n_bins - 1; ++k) {
            const int64_t nl = left_n[k], nr = right_n[k + 1];
            if (nl == 0 || nr == 0) continue;
            const double cost =
                c_trav + (left_sa[k] * (double)nl + right_sa[k + 1] * (double)nr) * c_isect / sa_node;
            if (cost < best_cost) {
              best_cost = cost;
              best_axis = axis;
              best_k = k;
            }
          }
        }
      }
    }
    int do_split = 0;
    int64_t mid = start;
    if (best_axis >= 0 && (count > max_leaf || best_cost < c_isect * (double)count)) {
      const double cmin = cl[best_axis], ext = chh[best_axis] - cl[best_axis];
      int64_t nl = 0;
      for (int64_t i = start; i < end; ++i) {
        const int64_t p = order[i];
        if (sah_bin(ce[3 * p + best_axis], cmin, ext, n_bins) <= best_k) tmp[nl++] = p;
      }
      int64_t nr = nl;
      for (int64_t i = start; i < end; ++i) {
        const int64_t p = order[i];
        if (sah_bin(ce[3 * p + best_axis], cmin, ext, n_bins) > best_k) tmp[nr++] = p;
      }
      for (int64_t i = 0; i < count; ++i) order[start + i] = tmp[i];
      mid = start + nl;
      do_split = 1;
    } else if (count > max_leaf) {
      mid = start + count / 2;
      do_split = 1;
    }
    if (do_split) {
      const int64_t left = n_nodes, right = n_nodes + 1;
      n_nodes += 2;
      node_a[idx] = left;
      node_b[idx] = right;
      node_leaf[idx] = 0;
      stack[3 * sp] = right;
      stack[3 * sp + 1] = mid;
      stack[3 * sp + 2] = end;
      ++sp;
      stack[3 * sp] = left;
      stack[3 * sp + 1] = start;
      stack[3 * sp + 2] = mid;
      ++sp;
    } else {
      node_a[idx] = start;
      node_b[idx] = count;
      node_leaf[idx] = 1;
    }
  }
  free(tmp);
  free(stack);
  free(bin_cnt);
  free(bin_lo);
  free(bin_hi);
  free(left_sa);
  free(right_sa);
  free(left_n);
  free(right_n);
  return n_nodes;
}

/* thread count of the following parallel regions (the bench's reference arm
   runs under torchrun, which starts its workers with OMP_NUM_THREADS=1) */
void oracle_set_threads(int n) {
#ifdef _OPENMP
  extern void omp_set_num_threads(int);
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
