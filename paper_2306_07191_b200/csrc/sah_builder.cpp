// Binned-SAH BVH builder (host side, one-time scene preprocessing).
//
// The GPU traversal kernels consume the flat node arrays this produces. The
// build reproduces the reference builder node for node (same bin index
// arithmetic, same split choice, same stable partition, same DFS node
// numbering), so the device any-hit kernels walk exactly the tree the
// reference walks and labels stay bit-exact by construction.
//   reference: pkg/src/niftrace/bvh.py:34-303 (_build_sah)
//
// Compile with -ffp-contract=off: the reference (numba, no fastmath) emits no
// FMAs, and every cost/bin expression below keeps its left-to-right order.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#include "nif_b200.h"
#include "status.h"

namespace {

struct Range {
  int64_t idx, start, end;
};

inline int64_t bin_of(double c, double cmin, double ext, int64_t n_bins) {
  // bvh.py:148  b = int(n_bins * (ce[p, axis] - cmin) / ext), clamped
  int64_t b = (int64_t)((double)n_bins * (c - cmin) / ext);
  if (b >= n_bins) b = n_bins - 1;
  if (b < 0) b = 0;
  return b;
}

}  // namespace

extern "C" int nif_build_sah(const double* lo, const double* hi, const double* ce,
                             int64_t n, int64_t max_leaf, int64_t n_bins,
                             double c_trav, double c_isect, double* node_lo,
                             double* node_hi, int64_t* node_a, int64_t* node_b,
                             uint8_t* node_leaf, int64_t* order,
                             int64_t* n_nodes_out) {
  if (n <= 0) return nif::fail(NIF_ERR_VALUE, "cannot build a tree over zero primitives");
  if (n_bins < 2 || max_leaf < 1) return nif::fail(NIF_ERR_VALUE, "bad SAH parameters");
  const double inf = std::numeric_limits<double>::infinity();
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  std::vector<int64_t> tmp(n);
  std::vector<Range> stack;
  stack.reserve(128);
  std::vector<int64_t> bin_cnt(n_bins), left_n(n_bins), right_n(n_bins);
  std::vector<double> bin_lo(n_bins * 3), bin_hi(n_bins * 3), left_sa(n_bins),
      right_sa(n_bins);

  stack.push_back({0, 0, n});
  int64_t n_nodes = 1;
  while (!stack.empty()) {
    Range r = stack.back();
    stack.pop_back();
    const int64_t idx = r.idx, start = r.start, end = r.end;
    const int64_t count = end - start;
    double bl[3] = {inf, inf, inf}, bh[3] = {-inf, -inf, -inf};
    double cl[3] = {inf, inf, inf}, chh[3] = {-inf, -inf, -inf};
    for (int64_t i = start; i < end; ++i) {
      const int64_t p = order[i];
      for (int c = 0; c < 3; ++c) {
        if (lo[p * 3 + c] < bl[c]) bl[c] = lo[p * 3 + c];
        if (hi[p * 3 + c] > bh[c]) bh[c] = hi[p * 3 + c];
        if (ce[p * 3 + c] < cl[c]) cl[c] = ce[p * 3 + c];
        if (ce[p * 3 + c] > chh[c]) chh[c] = ce[p * 3 + c];
      }
    }
    for (int c = 0; c < 3; ++c) {
      node_lo[idx * 3 + c] = bl[c];
      node_hi[idx * 3 + c] = bh[c];
    }

    double best_cost = inf;
    int best_axis = -1;
    int64_t best_k = -1;
    if (count > 1) {
      const double dx = bh[0] - bl[0], dy = bh[1] - bl[1], dz = bh[2] - bl[2];
      const double sa_node = 2.0 * (dx * dy + dy * dz + dz * dx);
      if (sa_node > 1e-300) {
        for (int axis = 0; axis < 3; ++axis) {
          const double cmin = cl[axis];
          const double ext = chh[axis] - cl[axis];
          if (ext <= 0.0) continue;
          for (int64_t k = 0; k < n_bins; ++k) {
            bin_cnt[k] = 0;
            for (int c = 0; c < 3; ++c) {
              bin_lo[k * 3 + c] = inf;
              bin_hi[k * 3 + c] = -inf;
            }
          }
          for (int64_t i = start; i < end; ++i) {
            const int64_t p = order[i];
            const int64_t b = bin_of(ce[p * 3 + axis], cmin, ext, n_bins);
            bin_cnt[b] += 1;
            for (int c = 0; c < 3; ++c) {
              if (lo[p * 3 + c] < bin_lo[b * 3 + c]) bin_lo[b * 3 + c] = lo[p * 3 + c];
              if (hi[p * 3 + c] > bin_hi[b * 3 + c]) bin_hi[b * 3 + c] = hi[p * 3 + c];
            }
          }
          // left sweep: union of bins [0..k]      (bvh.py:159-189)
          double a[3] = {inf, inf, inf}, bb[3] = {-inf, -inf, -inf};
          int64_t cnt = 0;
          for (int64_t k = 0; k < n_bins; ++k) {
            if (bin_cnt[k] > 0) {
              for (int c = 0; c < 3; ++c) {
                if (bin_lo[k * 3 + c] < a[c]) a[c] = bin_lo[k * 3 + c];
                if (bin_hi[k * 3 + c] > bb[c]) bb[c] = bin_hi[k * 3 + c];
              }
            }
            cnt += bin_cnt[k];
            left_n[k] = cnt;
            if (cnt > 0) {
              const double ex = bb[0] - a[0], ey = bb[1] - a[1], ez = bb[2] - a[2];
              left_sa[k] = 2.0 * (ex * ey + ey * ez + ez * ex);
            } else {
              left_sa[k] = 0.0;
            }
          }
          // right sweep: union of bins [k..]     (bvh.py:190-219)
          for (int c = 0; c < 3; ++c) {
            a[c] = inf;
            bb[c] = -inf;
          }
          cnt = 0;
          for (int64_t k = n_bins - 1; k >= 0; --k) {
            if (bin_cnt[k] > 0) {
              for (int c = 0; c < 3; ++c) {
                if (bin_lo[k * 3 + c] < a[c]) a[c] = bin_lo[k * 3 + c];
                if (bin_hi[k * 3 + c] > bb[c]) bb[c] = bin_hi[k * 3 + c];
              }
            }
            cnt += bin_cnt[k];
            right_n[k] = cnt;
            if (cnt > 0) {
              const double ex = bb[0] - a[0], ey = bb[1] - a[1], ez = bb[2] - a[2];
              right_sa[k] = 2.0 * (ex * ey + ey * ez + ez * ex);
            } else {
              right_sa[k] = 0.0;
            }
          }
          for (int64_t k = 0; k < n_bins - 1; ++k) {
            const int64_t nl = left_n[k];
            const int64_t nr = right_n[k + 1];
            if (nl == 0 || nr == 0) continue;
            // bvh.py:226 cost = c_trav + (lsa*nl + rsa*nr) * c_isect / sa_node
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

    bool do_split = false;
    int64_t mid = start;
    if (best_axis >= 0 && (count > max_leaf || best_cost < c_isect * (double)count)) {
      // stable partition by bin index (bvh.py:235-270)
      const double cmin = cl[best_axis];
      const double ext = chh[best_axis] - cl[best_axis];
      int64_t nl = 0;
      for (int64_t i = start; i < end; ++i) {
        const int64_t p = order[i];
        if (bin_of(ce[p * 3 + best_axis], cmin, ext, n_bins) <= best_k) tmp[nl++] = p;
      }
      int64_t nr = nl;
      for (int64_t i = start; i < end; ++i) {
        const int64_t p = order[i];
        if (bin_of(ce[p * 3 + best_axis], cmin, ext, n_bins) > best_k) tmp[nr++] = p;
      }
      std::memcpy(order + start, tmp.data(), sizeof(int64_t) * count);
      mid = start + nl;
      do_split = true;
    } else if (count > max_leaf) {
      // centroids collapsed; halve by current order (bvh.py:271-274)
      mid = start + count / 2;
      do_split = true;
    }

    if (do_split) {
      const int64_t left = n_nodes, right = n_nodes + 1;
      n_nodes += 2;
      node_a[idx] = left;
      node_b[idx] = right;
      node_leaf[idx] = 0;
      stack.push_back({right, mid, end});
      stack.push_back({left, start, mid});
    } else {
      node_a[idx] = start;
      node_b[idx] = count;
      node_leaf[idx] = 1;
    }
  }
  *n_nodes_out = n_nodes;
  return NIF_OK;
}
