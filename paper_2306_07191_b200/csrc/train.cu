// Online training step on the device: per-object batch counts, the fused
// encode -> MLP forward -> L2 loss -> backward -> grid-gradient scatter
// kernel, and the multi-tensor Adam (nif.py:682-749 _train_batch,
// mlp.py:82-167, grids.py:31-56 / 153-202).
//
// Compiled with -fmad=false so the grid interpolation weights and the
// Adam update evaluate exactly the reference's fp64 expressions; the MLP
// accumulations use explicit fmaf (fp32, like the reference's sgemm).
//
// Layout of the fused kernel: one CTA per RB rows (one row per thread).
// Pre-activations of every hidden layer stay in shared memory (rows padded
// to W+1 floats: conflict-free per-row access), so the backward pass needs
// no recomputation; weight gradients are CTA-level reductions over the RB
// rows (dz^T a), flushed with one fp32 atomic per weight per CTA. Grid
// gradients are fp32 atomics of (fp64 weight * upstream) rounded to fp32,
// the reference's np.add.at contributions.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cstdlib>
#include <stdint.h>

#include "common.h"
#include "kernels.h"
#include "nif_b200.h"
#include "status.h"

namespace nif {
namespace {

constexpr float kSlope = 0.01f;
constexpr int kMaxIn = 16;
constexpr int kMaxOut = 4;

__device__ __forceinline__ float leaky(float z) { return z > 0.f ? z : z * kSlope; }

struct Axis {
  int i0, i1;
  double w;
};

// grids.py:125-138
__device__ __forceinline__ Axis axis_indices(double x, int R, bool wrap) {
  const double xc = x * (double)R - 0.5;
  const double x0 = floor(xc);
  Axis a;
  a.w = xc - x0;
  long long i0 = (long long)x0, i1 = i0 + 1;
  if (wrap) {
    i0 = ((i0 % R) + R) % R;
    i1 = ((i1 % R) + R) % R;
  } else {
    i0 = i0 < 0 ? 0 : (i0 > R - 1 ? R - 1 : i0);
    i1 = i1 < 0 ? 0 : (i1 > R - 1 ? R - 1 : i1);
  }
  a.i0 = (int)i0;
  a.i1 = (int)i1;
  return a;
}

struct Bil64 {
  int c[4];        // flat cell index of corners 00, 01, 10, 11
  double w[4];
};

__device__ __forceinline__ Bil64 bil64(double u, double v, int R) {
  const Axis au = axis_indices(u, R, true), av = axis_indices(v, R, false);
  Bil64 b;
  b.c[0] = au.i0 * R + av.i0;
  b.c[1] = au.i0 * R + av.i1;
  b.c[2] = au.i1 * R + av.i0;
  b.c[3] = au.i1 * R + av.i1;
  b.w[0] = (1.0 - au.w) * (1.0 - av.w);
  b.w[1] = (1.0 - au.w) * av.w;
  b.w[2] = au.w * (1.0 - av.w);
  b.w[3] = au.w * av.w;
  return b;
}

struct TrainArgs {
  nif_family_view f;
  nif_train_view t;
  const int64_t* obj;
  const double* coord;
  const float* label;
  const int64_t* idx;
  int64_t n_rows, row0, row_step;
  double* sq_err;
  const int64_t* cursor;  // device row offset added to idx (graph-replayed steps), or NULL
  // gradient sinks (nif_train_fwdbwd_ex_dev): MLP gradients go to mlp_dst
  // ([w | pad | b], the family buffer's layout from off_w) by fp32 atomics,
  // or -- deterministic mode -- as this CTA's partial sums into row
  // blockIdx.x of mlp_part ([n_cta][n_mlp], reduced in CTA order after the
  // kernel); with dx_out set, the input gradient of batch row g is stored at
  // dx_out[g * IN + k] instead of being scattered into the grids
  float* mlp_dst;
  float* mlp_part;
  int64_t n_mlp;
  float* dx_out;
  int64_t part_cap;  // floats in mlp_part
};

thread_local unsigned g_last_ctas = 0;  // CTAs of the last fwd/bwd launch (host)

__device__ __forceinline__ void mlp_put(const TrainArgs& a, float* dst, float s) {
  if (a.mlp_part != nullptr)
    a.mlp_part[(size_t)blockIdx.x * a.n_mlp + (size_t)(dst - a.mlp_dst)] = s;
  else
    atomicAdd(dst, s);
}

// idx + *cursor: a CUDA graph of one optimiser step is replayed per batch
// while the batch start lives on the device
__device__ __forceinline__ const int64_t* batch_idx(const int64_t* idx, const int64_t* cursor) {
  return (idx != nullptr && cursor != nullptr) ? idx + *cursor : idx;
}

template <int W>
__global__ void train_fwdbwd_kernel(TrainArgs a) {
  extern __shared__ float sm[];
  const int RB = blockDim.x;
  const int tid = threadIdx.x;
  const int WP = W + 1;
  const nif_family_view& f = a.f;
  const int L = f.n_layers - 1;    // hidden layers
  const int IN = f.dims[0];
  const int OUT = f.dims[f.n_layers];
  float* zs = sm;                          // [L][RB][WP]
  float* dzA = zs + (size_t)L * RB * WP;   // [RB][WP]
  float* dzB = dzA + (size_t)RB * WP;      // [RB][WP]
  float* xs = dzB + (size_t)RB * WP;       // [RB][kMaxIn]
  float* dh = xs + (size_t)RB * kMaxIn;    // [RB][kMaxOut]
  // per_object sharing: the weight gradients of a CTA are reduced per head
  // over that head's rows only (rows of a batch belong to several objects)
  int* s_rhead = reinterpret_cast<int*>(dh + (size_t)RB * kMaxOut);  // [RB]
  int* s_uniq = s_rhead + RB;                                         // [RB]
  __shared__ int s_nuniq;

  const int64_t k_row = (int64_t)blockIdx.x * RB + tid;
  const int64_t g = a.row0 + k_row * a.row_step;
  const bool valid = k_row * a.row_step + a.row0 < a.n_rows && g < a.n_rows;
  const int64_t* bidx = batch_idx(a.idx, a.cursor);
  const int64_t row = valid ? (bidx ? bidx[g] : g) : 0;
  const int o = valid ? (int)a.obj[row] : 0;
  const int head = f.n_heads > 1 ? o : 0;
  s_rhead[tid] = valid ? head : -1;
  __syncthreads();
  if (tid == 0) {
    int nu = 0;
    for (int r = 0; r < RB; ++r) {
      const int h = s_rhead[r];
      if (h < 0) continue;
      bool seen = false;
      for (int q = 0; q < nu; ++q) seen = seen || s_uniq[q] == h;
      if (!seen) s_uniq[nu++] = h;
    }
    s_nuniq = nu;
  }
  __syncthreads();
  const int n_uniq = s_nuniq;
  const float* Wt = f.w + (size_t)head * f.w_stride;
  const float* Bt = f.b + (size_t)head * f.b_stride;
  float* gW0 = a.mlp_dst;
  float* gB0 = a.mlp_dst + (a.t.off_b - a.t.off_w);
  const int cw = f.family == NIF_FAMILY_OUTER ? 4 : 5;

  // ---- encode (grids.py:141-191: fp64 weights, fp64 sum, fp32 result) ----
  float x[kMaxIn];
#pragma unroll
  for (int k = 0; k < kMaxIn; ++k) x[k] = 0.f;
  Bil64 bp{}, bd{};
  Axis ad{};
  if (valid) {
    const double* c = a.coord + row * cw;
    const size_t g2 = (size_t)f.R * f.R * f.N;
    const float* gp = f.pos + (size_t)o * g2;
    const float* gd = f.dir + (size_t)o * g2;
    bp = bil64(c[0], c[1], f.R);
    bd = bil64(c[2], c[3], f.R);
    for (int k = 0; k < f.N; ++k) {
      const double sp = bp.w[0] * (double)gp[(size_t)bp.c[0] * f.N + k] +
                        bp.w[1] * (double)gp[(size_t)bp.c[1] * f.N + k] +
                        bp.w[2] * (double)gp[(size_t)bp.c[2] * f.N + k] +
                        bp.w[3] * (double)gp[(size_t)bp.c[3] * f.N + k];
      const double sd = bd.w[0] * (double)gd[(size_t)bd.c[0] * f.N + k] +
                        bd.w[1] * (double)gd[(size_t)bd.c[1] * f.N + k] +
                        bd.w[2] * (double)gd[(size_t)bd.c[2] * f.N + k] +
                        bd.w[3] * (double)gd[(size_t)bd.c[3] * f.N + k];
      x[k] = (float)sp;
      x[f.N + k] = (float)sd;
    }
    if (f.family == NIF_FAMILY_INNER) {
      ad = axis_indices(c[4], f.Rd, false);
      const float* gr = f.dist + (size_t)o * f.Rd * f.Nd;
      for (int k = 0; k < f.Nd; ++k) {
        const double s = (1.0 - ad.w) * (double)gr[(size_t)ad.i0 * f.Nd + k] +
                         ad.w * (double)gr[(size_t)ad.i1 * f.Nd + k];
        x[2 * f.N + k] = (float)s;
      }
    }
  }
  for (int k = 0; k < IN; ++k) xs[tid * kMaxIn + k] = x[k];

  // ---- forward -------------------------------------------------------------
  {  // layer 0
    float* z = zs + (size_t)tid * WP;
    for (int j = 0; j < W; ++j) {
      float acc = __ldg(Bt + j);
      const float* wr = Wt + (size_t)j * IN;
      for (int k = 0; k < IN; ++k) acc = fmaf(__ldg(wr + k), x[k], acc);
      z[j] = acc;
    }
  }
  size_t wo = (size_t)IN * W, bo = W;
  for (int l = 1; l < L; ++l) {
    const float* zp = zs + ((size_t)(l - 1) * RB + tid) * WP;
    float* z = zs + ((size_t)l * RB + tid) * WP;
    for (int j = 0; j < W; ++j) {
      float acc = __ldg(Bt + bo + j);
      const float* wr = Wt + wo + (size_t)j * W;
      for (int k = 0; k < W; ++k) acc = fmaf(__ldg(wr + k), leaky(zp[k]), acc);
      z[j] = acc;
    }
    wo += (size_t)W * W;
    bo += W;
  }
  // head + loss (mlp.py:91-101, 159-167)
  const size_t wo_h = wo, bo_h = bo;
  {
    const float* zp = zs + ((size_t)(L - 1) * RB + tid) * WP;
    const int n_o = valid ? a.t.counts[o] : 1;
    const float scale = (float)(2.0 / ((double)n_o * OUT));  // pred.dtype.type(2.0/diff.size)
    double sq = 0.0;
    for (int q = 0; q < OUT; ++q) {
      float acc = __ldg(Bt + bo_h + q);
      const float* wr = Wt + wo_h + (size_t)q * W;
      for (int k = 0; k < W; ++k) acc = fmaf(__ldg(wr + k), leaky(zp[k]), acc);
      float out, dz;
      const float lab = valid ? a.label[row * OUT + q] : 0.f;
      if (f.sigmoid_head) {
        out = acc >= 0.f ? 1.f / (1.f + expf(-acc)) : expf(acc) / (1.f + expf(acc));
        const float diff = out - lab;
        sq += (double)diff * (double)diff;
        const float gout = diff * scale;
        dz = gout * out * (1.f - out);
      } else {
        out = acc;
        const float diff = out - lab;
        sq += (double)diff * (double)diff;
        dz = diff * scale;
      }
      dh[tid * kMaxOut + q] = valid ? dz : 0.f;
    }
    if (valid) atomicAdd(a.sq_err, sq);
  }
  // da for the last hidden layer -> dz_{L-1}
  {
    const float* zp = zs + ((size_t)(L - 1) * RB + tid) * WP;
    float* dz = dzA + (size_t)tid * WP;
    for (int k = 0; k < W; ++k) {
      float da = 0.f;
      for (int q = 0; q < OUT; ++q) da = fmaf(dh[tid * kMaxOut + q], __ldg(Wt + wo_h + q * W + k), da);
      dz[k] = zp[k] > 0.f ? da : da * kSlope;
    }
  }
  __syncthreads();
  // head gradients: gW[q][k] = sum_r dh[r][q] * a_{L-1}[r][k]
  for (int hi = 0; hi < n_uniq; ++hi) {
    const int hh = s_uniq[hi];
    float* gW = gW0 + (size_t)hh * f.w_stride;
    float* gB = gB0 + (size_t)hh * f.b_stride;
    for (int e = tid; e < OUT * (W + 1); e += RB) {
      const int q = e / (W + 1), k = e % (W + 1);
      float s = 0.f;
      if (k < W) {
        for (int r = 0; r < RB; ++r)
          if (s_rhead[r] == hh)
            s = fmaf(dh[r * kMaxOut + q], leaky(zs[((size_t)(L - 1) * RB + r) * WP + k]), s);
        mlp_put(a, gW + wo_h + q * W + k, s);
      } else {
        for (int r = 0; r < RB; ++r)
          if (s_rhead[r] == hh) s += dh[r * kMaxOut + q];
        mlp_put(a, gB + bo_h + q, s);
      }
    }
  }
  // hidden layers L-1 .. 1
  float* dzc = dzA;
  float* dzn = dzB;
  for (int l = L - 1; l >= 1; --l) {
    wo -= (size_t)W * W;
    bo -= W;
    // weight grads of dense layer l: sum_r dz_l[r][j] * a_{l-1}[r][k]
    for (int hi = 0; hi < n_uniq; ++hi) {
      const int hh = s_uniq[hi];
      float* gW = gW0 + (size_t)hh * f.w_stride;
      float* gB = gB0 + (size_t)hh * f.b_stride;
      for (int e = tid; e < W * (W + 1); e += RB) {
        const int j = e / (W + 1), k = e % (W + 1);
        float s = 0.f;
        if (k < W) {
          for (int r = 0; r < RB; ++r)
            if (s_rhead[r] == hh)
              s = fmaf(dzc[(size_t)r * WP + j], leaky(zs[((size_t)(l - 1) * RB + r) * WP + k]),
                       s);
          mlp_put(a, gW + wo + (size_t)j * W + k, s);
        } else {
          for (int r = 0; r < RB; ++r)
            if (s_rhead[r] == hh) s += dzc[(size_t)r * WP + j];
          mlp_put(a, gB + bo + j, s);
        }
      }
    }
    // dz_{l-1} = mask(z_{l-1}) * (dz_l W_l)
    {
      const float* zp = zs + ((size_t)(l - 1) * RB + tid) * WP;
      const float* dc = dzc + (size_t)tid * WP;
      float* dn = dzn + (size_t)tid * WP;
      for (int k = 0; k < W; ++k) {
        float da = 0.f;
        for (int j = 0; j < W; ++j) da = fmaf(dc[j], __ldg(Wt + wo + (size_t)j * W + k), da);
        dn[k] = zp[k] > 0.f ? da : da * kSlope;
      }
    }
    __syncthreads();
    float* tmp = dzc;
    dzc = dzn;
    dzn = tmp;
  }
  // layer 0 weight grads: sum_r dz_0[r][j] * x[r][k]
  for (int hi = 0; hi < n_uniq; ++hi) {
    const int hh = s_uniq[hi];
    float* gW = gW0 + (size_t)hh * f.w_stride;
    float* gB = gB0 + (size_t)hh * f.b_stride;
    for (int e = tid; e < W * (IN + 1); e += RB) {
      const int j = e / (IN + 1), k = e % (IN + 1);
      float s = 0.f;
      if (k < IN) {
        for (int r = 0; r < RB; ++r)
          if (s_rhead[r] == hh) s = fmaf(dzc[(size_t)r * WP + j], xs[r * kMaxIn + k], s);
        mlp_put(a, gW + (size_t)j * IN + k, s);
      } else {
        for (int r = 0; r < RB; ++r)
          if (s_rhead[r] == hh) s += dzc[(size_t)r * WP + j];
        mlp_put(a, gB + j, s);
      }
    }
  }
  if (!valid) return;
  // input gradient dx = dz_0 W_0 -> grid scatter (grids.py:171-202)
  float dx[kMaxIn];
  for (int k = 0; k < IN; ++k) {
    float s = 0.f;
    const float* dc = dzc + (size_t)tid * WP;
    for (int j = 0; j < W; ++j) s = fmaf(dc[j], __ldg(Wt + (size_t)j * IN + k), s);
    dx[k] = s;
  }
  if (a.dx_out != nullptr) {  // data-parallel / deterministic: the scatter runs later
    for (int k = 0; k < IN; ++k) a.dx_out[g * IN + k] = dx[k];
    return;
  }
  const size_t g2 = (size_t)f.R * f.R * f.N;
  float* gpos = a.t.grad + a.t.off_pos + (size_t)o * g2;
  float* gdir = a.t.grad + a.t.off_dir + (size_t)o * g2;
  for (int c = 0; c < 4; ++c)
    for (int k = 0; k < f.N; ++k) {
      atomicAdd(gpos + (size_t)bp.c[c] * f.N + k, (float)(bp.w[c] * (double)dx[k]));
      atomicAdd(gdir + (size_t)bd.c[c] * f.N + k, (float)(bd.w[c] * (double)dx[f.N + k]));
    }
  if (f.family == NIF_FAMILY_INNER) {
    float* gr = a.t.grad + a.t.off_dist + (size_t)o * f.Rd * f.Nd;
    for (int k = 0; k < f.Nd; ++k) {
      atomicAdd(gr + (size_t)ad.i0 * f.Nd + k, (float)((1.0 - ad.w) * (double)dx[2 * f.N + k]));
      atomicAdd(gr + (size_t)ad.i1 * f.Nd + k, (float)(ad.w * (double)dx[2 * f.N + k]));
    }
  }
}

__global__ void batch_counts_kernel(const int64_t* __restrict__ obj, const int64_t* __restrict__ idx,
                                    int64_t n, int n_obj, int32_t* __restrict__ counts,
                                    const int64_t* __restrict__ cursor) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  idx = batch_idx(idx, cursor);
  const int64_t o = obj[idx ? idx[r] : r];
  if (o >= 0 && o < n_obj) atomicAdd(counts + o, 1);
}

// numba's float ** int (int_power_impl): binary exponentiation, libm pow
// beyond 0x10000.
__device__ __forceinline__ double int_power(double a, long long e) {
  if (e > 0x10000) return pow(a, (double)e);
  double r = 1.0;
  while (e) {
    if (e & 1) r *= a;
    e >>= 1;
    a *= a;
  }
  return r;
}

struct AdamSeg {
  int64_t off, per, n_units;  // element offset, elements per unit, units
  int kind;                   // 0 grid (unit = object), 1 mlp (unit = head)
};

__global__ void adam_steps_kernel(nif_train_view t, int n_obj, int n_heads, int shared) {
  const int i = threadIdx.x + blockIdx.x * blockDim.x;
  if (i < n_obj && t.counts[i] > 0) t.grid_steps[i] += 1;
  if (i < n_heads) {
    const bool touched = shared ? true : t.counts[i] > 0;
    if (touched) t.mlp_steps[i] += 1;
  }
}

__global__ void cursor_advance_kernel(int64_t* cursor, int64_t delta) { *cursor += delta; }

// One step's prologue for graph replay, one CTA: the batch's per-object row
// counts (overwritten, so no clearing kernel is needed) and the Adam step
// counters of the touched objects / heads (adam_steps_kernel's rule).
__global__ void __launch_bounds__(1024) train_prologue_kernel(const int64_t* __restrict__ obj,
                                                              const int64_t* __restrict__ idx,
                                                              const int64_t* __restrict__ cursor,
                                                              int64_t n, nif_train_view t,
                                                              int n_obj, int n_heads,
                                                              int shared) {
  extern __shared__ int hist[];
  // the step's fused fwd/bwd (programmatic dependent launch) may start now:
  // it reads the counts written here only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  for (int i = threadIdx.x; i < n_obj; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  idx = batch_idx(idx, cursor);
  // four rows per thread per round, their index and object loads issued
  // together (the step's latency is two dependent global loads, not eight)
  for (int64_t r0 = threadIdx.x; r0 < n; r0 += 4 * (int64_t)blockDim.x) {
    int64_t rows[4], o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t r = r0 + k * (int64_t)blockDim.x;
      rows[k] = r < n ? (idx ? idx[r] : r) : -1;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = rows[k] >= 0 ? obj[rows[k]] : -1;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (o[k] >= 0 && o[k] < n_obj) atomicAdd(hist + o[k], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_obj || i < n_heads; i += blockDim.x) {
    if (i < n_obj) {
      t.counts[i] = hist[i];
      if (hist[i] > 0) t.grid_steps[i] += 1;
    }
    if (i < n_heads && (shared || hist[i] > 0)) t.mlp_steps[i] += 1;
  }
}

// grids.py:31-45 _adam_update per element
__global__ void adam_kernel(nif_train_view t, AdamSeg s0, AdamSeg s1, AdamSeg s2, AdamSeg s3,
                            AdamSeg s4, int nseg, int shared, double lr, double b1, double b2,
                            double eps) {
  const AdamSeg segs[5] = {s0, s1, s2, s3, s4};
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;; e += (int64_t)gridDim.x * blockDim.x) {
    // locate the segment
    int64_t base = 0;
    int sid = -1;
    int64_t local = 0;
    for (int q = 0; q < nseg; ++q) {
      const int64_t len = segs[q].per * segs[q].n_units;
      if (e < base + len) {
        sid = q;
        local = e - base;
        break;
      }
      base += len;
    }
    if (sid < 0) return;
    const AdamSeg& sg = segs[sid];
    const int64_t unit = local / sg.per;
    int64_t step;
    if (sg.kind == 0) {
      if (t.counts[unit] <= 0) continue;
      step = t.grid_steps[unit];
    } else {
      if (!shared && t.counts[unit] <= 0) continue;
      step = t.mlp_steps[unit];
    }
    const double c1 = 1.0 - int_power(b1, step);
    const double c2 = 1.0 - int_power(b2, step);
    const int64_t p = sg.off + local;
    const double g = (double)t.grad[p] * 1.0;
    const double mi = b1 * ((double)t.m[p] * 1.0) + (1.0 - b1) * g;
    const double vi = b2 * ((double)t.v[p] * 1.0) + (1.0 - b2) * g * g;
    t.m[p] = (float)mi;
    t.v[p] = (float)vi;
    const double mh = mi / c1;
    const double vh = vi / c2;
    t.params[p] = (float)((double)t.params[p] - lr * mh / (sqrt(vh) + eps));
    t.grad[p] = 0.f;
  }
}


// Dense Adam, unit-major: blockIdx.z = segment (pos, dir, dist, w, b),
// blockIdx.y = unit (object grid set or head), blockIdx.x = chunk of the
// unit's elements. Untouched units exit per block (no per-element test),
// the bias corrections c1 / c2 are computed once per block, and segments
// whose per-unit length is a multiple of 4 move p / g / m / v as float4.
// Per element the reference's fp64 expression (grids.py:33-45) is kept.
// x, or 1.0 where x is +-0 -- as PTX, so the compiler cannot fold it back
// into the division it guards
__device__ __forceinline__ double nonzero(double x) {
  double r;
  asm("{\n .reg .pred z;\n setp.eq.f64 z, %1, 0d0000000000000000;\n"
      " selp.f64 %0, 0d3FF0000000000000, %1, z;\n}"
      : "=d"(r)
      : "d"(x));
  return r;
}

template <int V>
__device__ __forceinline__ void adam_elem(float& p, float& gr, float& m, float& v, double lr,
                                          double b1, double b2, double eps, double c1,
                                          double c2) {
  const double g = (double)gr * 1.0;
  const double mi = b1 * ((double)m * 1.0) + (1.0 - b1) * g;
  const double vi = b2 * ((double)v * 1.0) + (1.0 - b2) * g * g;
  m = (float)mi;
  v = (float)vi;
  if constexpr (V == 1) {  // the plain expression (variant for measurement)
    const double mh = mi / c1;
    const double vh = vi / c2;
    p = (float)((double)p - lr * mh / (sqrt(vh) + eps));
  } else {
    // Zero operands are resolved by selects: x / c for x = +-0 and c > 0 is
    // x itself, and vi == 0 is +0 (so sqrt(vi / c2) + eps == eps); the
    // divisions and the square root only ever see non-zero operands (1.0
    // stands in), which keeps them on their fast path -- most cells of a
    // sparsely touched grid hold zero moments, and a zero operand sends a
    // division into its slow special-operand subroutine. Bit-identical.
    const double mh = mi == 0.0 ? mi : nonzero(mi) / c1;
    const double num = lr * mh;
    const double den = vi == 0.0 ? eps : sqrt(nonzero(vi) / c2) + eps;
    const double q = num == 0.0 ? num : nonzero(num) / den;
    p = (float)((double)p - q);
  }
  gr = 0.f;
}

__device__ __forceinline__ bool changed4(const float4& a, const float4& b) {
  return (__float_as_uint(a.x) ^ __float_as_uint(b.x)) | (__float_as_uint(a.y) ^ __float_as_uint(b.y)) |
         (__float_as_uint(a.z) ^ __float_as_uint(b.z)) | (__float_as_uint(a.w) ^ __float_as_uint(b.w));
}

template <int AV>
__global__ void __launch_bounds__(256, 4) adam_units_kernel(nif_train_view t, AdamSeg s0, AdamSeg s1,
                                                         AdamSeg s2, AdamSeg s3, AdamSeg s4,
                                                         int shared, double lr, double b1,
                                                         double b2, double eps,
                                                         int64_t* cursor, int64_t delta) {
  // graph replay: the batch cursor moves on here (the step's readers of it
  // have finished: they precede this kernel on the stream)
  if (cursor && (blockIdx.x | blockIdx.y | blockIdx.z | threadIdx.x) == 0) *cursor += delta;
  const unsigned z = blockIdx.z;  // uniform selects (no local-memory array)
  const AdamSeg sg = z == 0 ? s0 : z == 1 ? s1 : z == 2 ? s2 : z == 3 ? s3 : s4;
  const int64_t unit = blockIdx.y;
  if (unit >= sg.n_units) return;
  int64_t step;
  if (sg.kind == 0) {
    if (t.counts[unit] <= 0) return;
    step = t.grid_steps[unit];
  } else {
    if (!shared && t.counts[unit] <= 0) return;
    step = t.mlp_steps[unit];
  }
  __shared__ double s_c[2];
  if (threadIdx.x == 0) {
    s_c[0] = 1.0 - int_power(b1, step);
    s_c[1] = 1.0 - int_power(b2, step);
  }
  __syncthreads();
  const double c1 = s_c[0], c2 = s_c[1];
  const int64_t base = sg.off + unit * sg.per;
  if ((sg.per & 3) == 0 && (base & 3) == 0) {
    const int64_t n4 = sg.per >> 2;
    float4* P = reinterpret_cast<float4*>(t.params + base);
    float4* G = reinterpret_cast<float4*>(t.grad + base);
    float4* M = reinterpret_cast<float4*>(t.m + base);
    float4* V = reinterpret_cast<float4*>(t.v + base);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4;
         e += (int64_t)gridDim.x * blockDim.x) {
      const float4 p0 = P[e], g0 = G[e], m0 = M[e], v0 = V[e];
      float4 p = p0, g = g0, m = m0, v = v0;
      adam_elem<AV>(p.x, g.x, m.x, v.x, lr, b1, b2, eps, c1, c2);
      adam_elem<AV>(p.y, g.y, m.y, v.y, lr, b1, b2, eps, c1, c2);
      adam_elem<AV>(p.z, g.z, m.z, v.z, lr, b1, b2, eps, c1, c2);
      adam_elem<AV>(p.w, g.w, m.w, v.w, lr, b1, b2, eps, c1, c2);
      // store only what changed bit-wise: cells a step did not touch keep
      // g == +0 (and, never touched so far, p / m / v too), so most of the
      // write traffic of a sparsely touched grid is skipped
      if (changed4(p, p0)) P[e] = p;
      if (changed4(g, g0)) G[e] = g;
      if (changed4(m, m0)) M[e] = m;
      if (changed4(v, v0)) V[e] = v;
    }
  } else {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < sg.per;
         e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t q = base + e;
      adam_elem<AV>(t.params[q], t.grad[q], t.m[q], t.v[q], lr, b1, b2, eps, c1, c2);
    }
  }
}

__global__ void clear_counts_kernel(int32_t* counts, int n) {
  const int i = threadIdx.x + blockIdx.x * blockDim.x;
  if (i < n) counts[i] = 0;
}


// ---------------------------------------------------------------------------
// Tiled variant (shared MLP, hidden width a multiple of 16): 32 rows per CTA
// of 128 threads, every dense layer a small CTA-wide SIMT GEMM with 4 x W/16
// register tiles over the rows' activations in shared memory and the layer's
// weights staged in shared memory (transposed for the forward pass). Each
// output accumulates bias-first and k ascending with fmaf, exactly the
// per-row kernel's order, so forward values and the per-row backward
// quantities are bit-identical to it; only the CTA partial sums of the
// weight gradients (32 rows instead of 128 per atomic) differ in rounding.
// 4x more CTAs per batch and ~W/16x less serial work per thread.
// ---------------------------------------------------------------------------
// RB rows per CTA, TT threads: 16 column groups x (TT/16) row groups of
// RPT = 16 RB / TT rows each
// shared-memory carve of the tiled kernel (floats unless noted)
struct TiledSmem {
  int zs, dzA, dzB, xs, dh, sw, sb, rwd, rwi, total_bytes;
  int o_h1, o_head;  // offsets of the hidden / head weights inside sw
};
__host__ __device__ inline TiledSmem tiled_smem(int W, int RB, int L, int IN, int OUT) {
  TiledSmem t;
  const int WP = W + 1;
  t.zs = 0;
  t.dzA = t.zs + L * RB * WP;
  t.dzB = t.dzA + RB * WP;
  t.xs = t.dzB + RB * WP;
  t.dh = t.xs + RB * kMaxIn;
  t.sw = t.dh + RB * kMaxOut;
  t.o_h1 = W * (IN + 1);
  t.o_head = t.o_h1 + (L - 1) * W * WP;
  t.sb = t.sw + t.o_head + OUT * WP;
  const int end_f = t.sb + L * W + kMaxOut;
  t.rwd = (end_f + 1) / 2;  // in doubles: [RB][9] corner weights of each row
  t.rwi = (t.rwd + RB * 9) * 2;  // in ints: [RB][11] corner cells, object (-1: no row)
  t.total_bytes = (t.rwi + RB * 11) * 4;
  return t;
}

template <int W, int RB, int TT>
__global__ void __launch_bounds__(TT) train_fwdbwd_tiled_kernel(TrainArgs a) {
  constexpr int RPT = RB * 16 / TT;
  static_assert(RPT >= 1 && RB * 16 == RPT * TT && TT >= RB * kMaxOut, "tiling");
  constexpr int WP = W + 1;
  constexpr int CPT = W / 16;  // output columns per thread (16 column groups)
  extern __shared__ float sm[];
  const int tid = threadIdx.x;
  const nif_family_view& f = a.f;
  const int L = f.n_layers - 1;
  const int IN = f.dims[0];
  const int INP = IN + 1;
  const int OUT = f.dims[f.n_layers];
  const TiledSmem T = tiled_smem(W, RB, L, IN, OUT);
  float* zs = sm + T.zs;    // [L][RB][WP] activations leaky(z)
  float* dzA = sm + T.dzA;  // [RB][WP]
  float* dzB = sm + T.dzB;  // [RB][WP]
  float* xs = sm + T.xs;    // [RB][kMaxIn]
  float* dh = sm + T.dh;    // [RB][kMaxOut]
  float* sw = sm + T.sw;    // every layer's weights, natural [j][k], rows padded to K + 1
  float* sb = sm + T.sb;    // every layer's biases
  double* rwd = reinterpret_cast<double*>(sm) + T.rwd;
  int* rwi = reinterpret_cast<int*>(sm) + T.rwi;
  float* gW = a.mlp_dst;
  float* gB = a.mlp_dst + (a.t.off_b - a.t.off_w);
  const int cw = f.family == NIF_FAMILY_OUTER ? 4 : 5;
  const int tc = tid & 15, tr = tid >> 4;  // 16 column groups x TT/16 row groups of RPT

  // ---- stage the whole MLP once (its loads overlap the encode's) -----------
  {
    const int n0 = W * IN;
    for (int e = tid; e < n0; e += TT) {  // layer 0: rows of IN (odd) floats
      const int j = e / IN;
      sw[j * INP + (e - j * IN)] = __ldg(f.w + e);
    }
    // hidden layers and head: rows of W floats (W % 16 == 0), read as float4
    constexpr int Q = W / 4;
    const int rows = (L - 1) * W + OUT;
    const float4* src = reinterpret_cast<const float4*>(f.w + n0);
    for (int e = tid; e < rows * Q; e += TT) {
      const int rr = e / Q, c4 = e - (e / Q) * Q;
      const float4 v = __ldg(src + e);
      const int d = (rr < (L - 1) * W ? T.o_h1 + (rr / W) * W * WP + (rr % W) * WP
                                      : T.o_head + (rr - (L - 1) * W) * WP) + 4 * c4;
      sw[d] = v.x;
      sw[d + 1] = v.y;
      sw[d + 2] = v.z;
      sw[d + 3] = v.w;
    }
    for (int e = tid; e < L * W + OUT; e += TT) sb[e] = __ldg(f.b + e);
  }

  // ---- encode: row setup on threads 0..RB-1 (corner cells and weights into
  // shared memory), then one (row, input) feature per thread -----------------
  if (tid < RB) {
    const int64_t k_row = (int64_t)blockIdx.x * RB + tid;
    const int64_t g = a.row0 + k_row * a.row_step;
    const bool valid = g < a.n_rows;
    const int64_t* bidx = batch_idx(a.idx, a.cursor);
    const int64_t row = valid ? (bidx ? bidx[g] : g) : 0;
    const int o = valid ? (int)a.obj[row] : 0;
    Bil64 bp{}, bd{};
    Axis ad{};
    if (valid) {
      const double* c = a.coord + row * cw;
      bp = bil64(c[0], c[1], f.R);
      bd = bil64(c[2], c[3], f.R);
      if (f.family == NIF_FAMILY_INNER) ad = axis_indices(c[4], f.Rd, false);
    }
    // the row's corner cells / weights: the features below and the
    // backward pass's grid scatter both read them
    for (int c = 0; c < 4; ++c) {
      rwd[tid * 9 + c] = bp.w[c];
      rwd[tid * 9 + 4 + c] = bd.w[c];
      rwi[tid * 11 + c] = bp.c[c];
      rwi[tid * 11 + 4 + c] = bd.c[c];
    }
    rwd[tid * 9 + 8] = ad.w;
    rwi[tid * 11 + 8] = ad.i0;
    rwi[tid * 11 + 9] = ad.i1;
    rwi[tid * 11 + 10] = valid ? o : -1;
  }
  __syncthreads();
  {
    const int IN_ = f.family == NIF_FAMILY_INNER ? 2 * f.N + f.Nd : 2 * f.N;
    const size_t g2 = (size_t)f.R * f.R * f.N;
    for (int e = tid; e < RB * kMaxIn; e += TT) {
      const int r = e / kMaxIn, k = e % kMaxIn;
      const int o = rwi[r * 11 + 10];
      float x = 0.f;
      if (o >= 0 && k < IN_) {
        // nif.py:286-311 per feature, the reference's corner order in fp64
        if (k < 2 * f.N) {
          const bool is_pos = k < f.N;
          const float* gg = (is_pos ? f.pos : f.dir) + (size_t)o * g2;
          const int kk = is_pos ? k : k - f.N;
          const int cb = is_pos ? 0 : 4;
          const double s = rwd[r * 9 + cb + 0] * (double)gg[(size_t)rwi[r * 11 + cb + 0] * f.N + kk] +
                           rwd[r * 9 + cb + 1] * (double)gg[(size_t)rwi[r * 11 + cb + 1] * f.N + kk] +
                           rwd[r * 9 + cb + 2] * (double)gg[(size_t)rwi[r * 11 + cb + 2] * f.N + kk] +
                           rwd[r * 9 + cb + 3] * (double)gg[(size_t)rwi[r * 11 + cb + 3] * f.N + kk];
          x = (float)s;
        } else {
          const int kk = k - 2 * f.N;
          const float* gr = f.dist + (size_t)o * f.Rd * f.Nd;
          const double w = rwd[r * 9 + 8];
          const double s = (1.0 - w) * (double)gr[(size_t)rwi[r * 11 + 8] * f.Nd + kk] +
                           w * (double)gr[(size_t)rwi[r * 11 + 9] * f.Nd + kk];
          x = (float)s;
        }
      }
      xs[r * kMaxIn + k] = x;
    }
  }

  // ---- forward: Z_l = bias + act(prev) . W_l^T (k ascending) ---------------
  for (int l = 0; l < L; ++l) {
    const int K = l == 0 ? IN : W;
    const int KP = K + 1;
    const float* wl = l == 0 ? sw : sw + T.o_h1 + (l - 1) * W * WP;
    __syncthreads();  // weights, x / the previous layer's outputs visible
    float acc[RPT][CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const float bj = sb[l * W + tc + 16 * c];
#pragma unroll
      for (int i = 0; i < RPT; ++i) acc[i][c] = bj;
    }
    const float* prev = l == 0 ? xs : zs + (size_t)(l - 1) * RB * WP;
    const int ps = l == 0 ? kMaxIn : WP;
    for (int k = 0; k < K; ++k) {
      float av[RPT];
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const float v = prev[(tr * RPT + i) * ps + k];
        av[i] = v;  // x, or the previous layer's activation
      }
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const float wv = wl[(tc + 16 * c) * KP + k];
#pragma unroll
        for (int i = 0; i < RPT; ++i) acc[i][c] = fmaf(wv, av[i], acc[i][c]);
      }
    }
    float* z = zs + (size_t)l * RB * WP;
#pragma unroll
    for (int i = 0; i < RPT; ++i)
#pragma unroll
      for (int c = 0; c < CPT; ++c) z[(tr * RPT + i) * WP + tc + 16 * c] = leaky(acc[i][c]);
  }
  // the hidden layers hold activations leaky(z), stored once by their
  // producer (same sign as z, so the backward masks `z > 0` read them
  // unchanged)
  __syncthreads();
  // the batch counts (per-object loss scale) come from the step's prologue
  // kernel; everything above overlaps it under programmatic dependent launch
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // ---- head + loss: one (row, q) per thread --------------------------------
  const size_t wo_h = (size_t)W * IN + (size_t)(L - 1) * W * W, bo_h = (size_t)L * W;
  const float* swh = sw + T.o_head;
  const float* zl = zs + (size_t)(L - 1) * RB * WP;
  {
    const int r = tid % RB, q = tid / RB;
    if (q < OUT) {
      const int64_t k_row = (int64_t)blockIdx.x * RB + r;
      const int64_t g = a.row0 + k_row * a.row_step;
      const bool v = g < a.n_rows;
      const int64_t* bidx = batch_idx(a.idx, a.cursor);
      const int64_t rw = v ? (bidx ? bidx[g] : g) : 0;
      const int ob = v ? (int)a.obj[rw] : 0;
      float acc = sb[bo_h + q];
      for (int k = 0; k < W; ++k) acc = fmaf(swh[q * WP + k], zl[r * WP + k], acc);
      const int n_o = v ? a.t.counts[ob] : 1;
      const float scale = (float)(2.0 / ((double)n_o * OUT));
      const float lab = v ? a.label[rw * OUT + q] : 0.f;
      float out, dz;
      if (f.sigmoid_head) {
        out = acc >= 0.f ? 1.f / (1.f + expf(-acc)) : expf(acc) / (1.f + expf(acc));
        const float diff = out - lab;
        if (v) atomicAdd(a.sq_err, (double)diff * (double)diff);
        dz = diff * scale * out * (1.f - out);
      } else {
        out = acc;
        const float diff = out - lab;
        if (v) atomicAdd(a.sq_err, (double)diff * (double)diff);
        dz = diff * scale;
      }
      dh[r * kMaxOut + q] = v ? dz : 0.f;
    }
  }
  __syncthreads();
  // dZ_{L-1}[r][k] = mask * sum_q dh[r][q] Wh[q][k]
  for (int e = tid; e < RB * W; e += TT) {
    const int r = e / W, k = e % W;
    float da = 0.f;
    for (int q = 0; q < OUT; ++q) da = fmaf(dh[r * kMaxOut + q], swh[q * WP + k], da);
    dzA[r * WP + k] = zl[r * WP + k] > 0.f ? da : da * kSlope;
  }
  // head gradients
  for (int e = tid; e < OUT * (W + 1); e += TT) {
    const int q = e / (W + 1), k = e % (W + 1);
    float s = 0.f;
    if (k < W) {
      for (int r = 0; r < RB; ++r) s = fmaf(dh[r * kMaxOut + q], zl[r * WP + k], s);
      mlp_put(a, gW + wo_h + q * W + k, s);
    } else {
      for (int r = 0; r < RB; ++r) s += dh[r * kMaxOut + q];
      mlp_put(a, gB + bo_h + q, s);
    }
  }
  __syncthreads();
  float* dzc = dzA;
  float* dzn = dzB;
  for (int l = L - 1; l >= 1; --l) {
    const size_t wo = (size_t)W * IN + (size_t)(l - 1) * W * W, bo = (size_t)l * W;
    const float* wl = sw + T.o_h1 + (l - 1) * W * WP;
    const float* zp = zs + (size_t)(l - 1) * RB * WP;
    // weight grads of dense layer l: gW[j][k] += sum_r dz[r][j] a[r][k]
    if constexpr (TT == 256) {
      // 16 x 16 threads, each a CPT x CPT register tile (j = tj + 16 cj,
      // k = tk + 16 ck), rows ascending as in the per-element loop
      const int tj = tid >> 4, tk = tid & 15;
      float g[CPT][CPT];
#pragma unroll
      for (int cj = 0; cj < CPT; ++cj)
#pragma unroll
        for (int ck = 0; ck < CPT; ++ck) g[cj][ck] = 0.f;
      for (int r = 0; r < RB; ++r) {
        float dj[CPT], ak[CPT];
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          dj[c] = dzc[r * WP + tj + 16 * c];
          ak[c] = zp[r * WP + tk + 16 * c];
        }
#pragma unroll
        for (int cj = 0; cj < CPT; ++cj)
#pragma unroll
          for (int ck = 0; ck < CPT; ++ck) g[cj][ck] = fmaf(dj[cj], ak[ck], g[cj][ck]);
      }
#pragma unroll
      for (int cj = 0; cj < CPT; ++cj)
#pragma unroll
        for (int ck = 0; ck < CPT; ++ck)
          mlp_put(a, gW + wo + (size_t)(tj + 16 * cj) * W + tk + 16 * ck, g[cj][ck]);
      if (tid < W) {
        float sbias = 0.f;
        for (int r = 0; r < RB; ++r) sbias += dzc[r * WP + tid];
        mlp_put(a, gB + bo + tid, sbias);
      }
    } else {
      for (int e = tid; e < W * (W + 1); e += TT) {
        const int j = e / (W + 1), k = e % (W + 1);
        float s = 0.f;
        if (k < W) {
          for (int r = 0; r < RB; ++r) s = fmaf(dzc[r * WP + j], zp[r * WP + k], s);
          mlp_put(a, gW + wo + (size_t)j * W + k, s);
        } else {
          for (int r = 0; r < RB; ++r) s += dzc[r * WP + j];
          mlp_put(a, gB + bo + j, s);
        }
      }
    }
    // dZ_{l-1} = mask . (dZ_l W_l), j ascending
    float acc[RPT][CPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i)
#pragma unroll
      for (int c = 0; c < CPT; ++c) acc[i][c] = 0.f;
    for (int j = 0; j < W; ++j) {
      float dv[RPT];
#pragma unroll
      for (int i = 0; i < RPT; ++i) dv[i] = dzc[(tr * RPT + i) * WP + j];
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const float wv = wl[j * WP + tc + 16 * c];
#pragma unroll
        for (int i = 0; i < RPT; ++i) acc[i][c] = fmaf(dv[i], wv, acc[i][c]);
      }
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i)
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int r = tr * RPT + i, k = tc + 16 * c;
        dzn[r * WP + k] = zp[r * WP + k] > 0.f ? acc[i][c] : acc[i][c] * kSlope;
      }
    __syncthreads();
    float* tmp = dzc;
    dzc = dzn;
    dzn = tmp;
  }
  // layer 0 weight grads
  for (int e = tid; e < W * (IN + 1); e += TT) {
    const int j = e / (IN + 1), k = e % (IN + 1);
    float s = 0.f;
    if (k < IN) {
      for (int r = 0; r < RB; ++r) s = fmaf(dzc[r * WP + j], xs[r * kMaxIn + k], s);
      mlp_put(a, gW + (size_t)j * IN + k, s);
    } else {
      for (int r = 0; r < RB; ++r) s += dzc[r * WP + j];
      mlp_put(a, gB + j, s);
    }
  }
  // dx = dZ_0 W_0, one (row, input) per thread -> grid scatter
  // (grids.py:171-202); j ascending as in the per-row kernel
  const size_t g2 = (size_t)f.R * f.R * f.N;
  for (int e = tid; e < RB * IN; e += TT) {
    const int r = e / IN, k = e - (e / IN) * IN;
    const int o = rwi[r * 11 + 10];
    if (o < 0) continue;
    float s = 0.f;
    const float* dc = dzc + (size_t)r * WP;
    for (int j = 0; j < W; ++j) s = fmaf(dc[j], sw[j * INP + k], s);
    if (a.dx_out != nullptr) {  // data-parallel / deterministic: the scatter runs later
      const int64_t g = a.row0 + ((int64_t)blockIdx.x * RB + r) * a.row_step;
      a.dx_out[g * IN + k] = s;
      continue;
    }
    const double dx = (double)s;
    if (k < 2 * f.N) {
      const bool is_pos = k < f.N;
      float* gg = a.t.grad + (is_pos ? a.t.off_pos : a.t.off_dir) + (size_t)o * g2;
      const int kk = is_pos ? k : k - f.N;
      const int cb = is_pos ? 0 : 4;
      for (int c = 0; c < 4; ++c)
        atomicAdd(gg + (size_t)rwi[r * 11 + cb + c] * f.N + kk,
                  (float)(rwd[r * 9 + cb + c] * dx));
    } else {
      const int kk = k - 2 * f.N;
      const double w = rwd[r * 9 + 8];
      float* gr = a.t.grad + a.t.off_dist + (size_t)o * f.Rd * f.Nd;
      atomicAdd(gr + (size_t)rwi[r * 11 + 8] * f.Nd + kk, (float)((1.0 - w) * dx));
      atomicAdd(gr + (size_t)rwi[r * 11 + 9] * f.Nd + kk, (float)(w * dx));
    }
  }
}

int g_train_variant = 0;  // 0 tiled where it applies, 1 per-row kernel, 2/3 other tilings,
                          // 4 plain Adam expression (nif_debug_set_train_variant)

template <int W, int RB, int TT>
int launch_fwdbwd_tiled_rb(const TrainArgs& a, cudaStream_t st) {
  const int L = a.f.n_layers - 1;
  const size_t smem =
      (size_t)tiled_smem(W, RB, L, a.f.dims[0], a.f.dims[a.f.n_layers]).total_bytes;
  if (smem > 200 * 1024) return fail(NIF_ERR_UNSUPPORTED, "MLP too large for the training kernel");
  auto kern = train_fwdbwd_tiled_kernel<W, RB, TT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t my_rows = (a.n_rows - a.row0 + a.row_step - 1) / a.row_step;
  if (my_rows <= 0) return NIF_OK;
  const unsigned grid = (unsigned)((my_rows + RB - 1) / RB);
  if (a.mlp_part != nullptr && (int64_t)grid * a.n_mlp > a.part_cap)
    return fail(NIF_ERR_VALUE, "MLP partials buffer too small (%lld CTAs)", (long long)grid);
  g_last_ctas = grid;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a);
  return check_launch("nif_train_fwdbwd_dev(tiled)");
}

// 16 rows x 256 threads (one row per thread-row): twice the CTAs and eight
// warps each, against the latency of the small per-layer GEMMs
// (nif_debug_set_train_variant 2 selects the 32-row / 128-thread tiling)
template <int W>
int launch_fwdbwd_tiled(const TrainArgs& a, cudaStream_t st) {
  if (g_train_variant == 2) return launch_fwdbwd_tiled_rb<W, 32, 128>(a, st);
  if (g_train_variant == 3) return launch_fwdbwd_tiled_rb<W, 32, 256>(a, st);
  return launch_fwdbwd_tiled_rb<W, 16, 256>(a, st);
}

template <int W>
int launch_fwdbwd(const TrainArgs& a, cudaStream_t st) {
  const int L = a.f.n_layers - 1;
  int rb = 128;
  auto smem_for = [&](int r) {
    return ((size_t)L * r * (W + 1) + 2 * (size_t)r * (W + 1) + (size_t)r * kMaxIn +
            (size_t)r * kMaxOut) * sizeof(float) + 2 * (size_t)r * sizeof(int);
  };
  while (rb > 32 && smem_for(rb) > 200 * 1024) rb /= 2;
  const size_t smem = smem_for(rb);
  if (smem > 220 * 1024) return fail(NIF_ERR_UNSUPPORTED, "MLP too large for the training kernel");
  auto kern = train_fwdbwd_kernel<W>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t my_rows = (a.n_rows - a.row0 + a.row_step - 1) / a.row_step;
  if (my_rows <= 0) return NIF_OK;
  const unsigned grid = (unsigned)((my_rows + rb - 1) / rb);
  if (a.mlp_part != nullptr && (int64_t)grid * a.n_mlp > a.part_cap)
    return fail(NIF_ERR_VALUE, "MLP partials buffer too small (%lld CTAs)", (long long)grid);
  if (a.mlp_part != nullptr)  // per-head partials: a CTA writes only its own heads' rows
    cudaMemsetAsync(a.mlp_part, 0, (size_t)grid * a.n_mlp * sizeof(float), st);
  g_last_ctas = grid;
  kern<<<grid, rb, smem, st>>>(a);
  return check_launch("nif_train_fwdbwd_dev");
}

}  // namespace
}  // namespace nif

namespace nif {
namespace {
int launch_fwdbwd_any(const TrainArgs& a, cudaStream_t st);
}
}  // namespace nif

using namespace nif;

extern "C" int nif_batch_counts_cur_dev(const int64_t* obj, const int64_t* idx,
                                        const int64_t* cursor, int64_t n_rows, int32_t n_obj,
                                        int32_t* counts, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_rows <= 0) return NIF_OK;
  batch_counts_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, st>>>(obj, idx, n_rows, n_obj,
                                                                        counts, cursor);
  return check_launch("nif_batch_counts_dev");
}

extern "C" int nif_batch_counts_dev(const int64_t* obj, const int64_t* idx, int64_t n_rows,
                                    int32_t n_obj, int32_t* counts, void* stream) {
  return nif_batch_counts_cur_dev(obj, idx, nullptr, n_rows, n_obj, counts, stream);
}

extern "C" int nif_cursor_advance_dev(int64_t* cursor, int64_t delta, void* stream) {
  cursor_advance_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(cursor, delta);
  return check_launch("nif_cursor_advance_dev");
}

extern "C" int nif_train_fwdbwd_cur_dev(const nif_family_view* f, const nif_train_view* t,
                                        const int64_t* obj, const double* coord,
                                        const float* label, const int64_t* idx,
                                        const int64_t* cursor, int64_t n_rows, int64_t row0,
                                        int64_t row_step, double* sq_err, void* stream);

extern "C" int nif_train_fwdbwd_dev(const nif_family_view* f, const nif_train_view* t,
                                    const int64_t* obj, const double* coord, const float* label,
                                    const int64_t* idx, int64_t n_rows, int64_t row0,
                                    int64_t row_step, double* sq_err, void* stream) {
  return nif_train_fwdbwd_cur_dev(f, t, obj, coord, label, idx, nullptr, n_rows, row0, row_step,
                                  sq_err, stream);
}

extern "C" int nif_train_fwdbwd_cur_dev(const nif_family_view* f, const nif_train_view* t,
                                        const int64_t* obj, const double* coord,
                                        const float* label, const int64_t* idx,
                                        const int64_t* cursor, int64_t n_rows, int64_t row0,
                                        int64_t row_step, double* sq_err, void* stream) {
  TrainArgs a{*f, *t, obj, coord, label, idx, n_rows, row0, row_step, sq_err, cursor,
              t->grad + t->off_w, nullptr, 0, nullptr, 0};
  return launch_fwdbwd_any(a, (cudaStream_t)stream);
}

namespace nif {
namespace {
int launch_fwdbwd_any(const TrainArgs& a, cudaStream_t st) {
  const nif_family_view* f = &a.f;
  g_last_ctas = 0;
  if (a.n_rows <= 0) return NIF_OK;
  if (f->n_layers < 2) return fail(NIF_ERR_UNSUPPORTED, "training needs at least one hidden layer");
  if (f->dims[0] > kMaxIn) return fail(NIF_ERR_UNSUPPORTED, "input width above %d", kMaxIn);
  if (f->dims[f->n_layers] > kMaxOut) return fail(NIF_ERR_UNSUPPORTED, "head wider than %d", kMaxOut);
  for (int i = 2; i < f->n_layers; ++i)
    if (f->dims[i] != f->dims[1]) return fail(NIF_ERR_UNSUPPORTED, "hidden widths must match");
  if (a.row_step < 1 || a.row0 < 0) return fail(NIF_ERR_VALUE, "bad row partition");
  if (g_train_variant != 1 && f->n_heads == 1) {
    switch (f->dims[1]) {
      case 16: return launch_fwdbwd_tiled<16>(a, st);
      case 32: return launch_fwdbwd_tiled<32>(a, st);
      case 48: return launch_fwdbwd_tiled<48>(a, st);
      case 64: return launch_fwdbwd_tiled<64>(a, st);
      case 96: return launch_fwdbwd_tiled<96>(a, st);
      case 128: return launch_fwdbwd_tiled<128>(a, st);
      default: break;
    }
  }
  switch (f->dims[1]) {
    case 8: return launch_fwdbwd<8>(a, st);
    case 16: return launch_fwdbwd<16>(a, st);
    case 32: return launch_fwdbwd<32>(a, st);
    case 48: return launch_fwdbwd<48>(a, st);
    case 64: return launch_fwdbwd<64>(a, st);
    case 96: return launch_fwdbwd<96>(a, st);
    case 128: return launch_fwdbwd<128>(a, st);
    default: return fail(NIF_ERR_UNSUPPORTED, "hidden width %d not instantiated", f->dims[1]);
  }
}
}  // namespace
}  // namespace nif

extern "C" int nif_debug_set_train_variant(int v) {
  g_train_variant = v;
  return NIF_OK;
}

namespace {

// the dense update of every touched unit; cursor: advanced by delta (graph replay)
void launch_adam_units(const nif_family_view* f, const nif_train_view* t, double lr,
                       double beta1, double beta2, double eps, int64_t* cursor, int64_t delta,
                       cudaStream_t st) {
  const int n_heads = f->n_heads;
  const int shared = n_heads == 1;
  AdamSeg s[5];
  int ns = 0;
  const int64_t g2 = (int64_t)f->R * f->R * f->N;
  s[ns++] = {t->off_pos, g2, f->n_obj, 0};
  s[ns++] = {t->off_dir, g2, f->n_obj, 0};
  if (f->family == NIF_FAMILY_INNER) s[ns++] = {t->off_dist, (int64_t)f->Rd * f->Nd, f->n_obj, 0};
  s[ns++] = {t->off_w, f->w_stride, n_heads, 1};
  s[ns++] = {t->off_b, f->b_stride, n_heads, 1};
  while (ns < 5) s[ns++] = {0, 1, 0, 1};
  if (g_train_variant == 1) {
    int64_t total = 0;
    for (int q = 0; q < 5; ++q) total += s[q].per * s[q].n_units;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    adam_kernel<<<(unsigned)(blocks > 0 ? blocks : 1), 256, 0, st>>>(
        *t, s[0], s[1], s[2], s[3], s[4], 5, shared, lr, beta1, beta2, eps);
    if (cursor) cursor_advance_kernel<<<1, 1, 0, st>>>(cursor, delta);
    return;
  }
  int64_t per_max = 0, units = 0;
  for (int q = 0; q < 5; ++q) {
    if (s[q].per > per_max) per_max = s[q].per;
    if (s[q].n_units > units) units = s[q].n_units;
  }
  // ~4 float4 per thread per block: enough blocks to fill the GPU for the
  // touched units without a per-element segment search
  // (1, 2, 8, 16 float4 per thread measured slower at C2: 20 / 18 / 22 / 36 us
  // against 16 us for the inner family)
  int64_t bx = (per_max / 4 + 1023) / 1024;
  if (bx < 1) bx = 1;
  dim3 grid((unsigned)bx, (unsigned)(units > 0 ? units : 1), 5);
  if (g_train_variant == 4)
    adam_units_kernel<1><<<grid, 256, 0, st>>>(*t, s[0], s[1], s[2], s[3], s[4], shared, lr,
                                               beta1, beta2, eps, cursor, delta);
  else
    adam_units_kernel<0><<<grid, 256, 0, st>>>(*t, s[0], s[1], s[2], s[3], s[4], shared, lr,
                                               beta1, beta2, eps, cursor, delta);
}

}  // namespace

extern "C" int nif_adam_dev(const nif_family_view* f, const nif_train_view* t, double lr,
                            double beta1, double beta2, double eps, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int n_heads = f->n_heads;
  const int n = f->n_obj > n_heads ? f->n_obj : n_heads;
  adam_steps_kernel<<<(n + 127) / 128, 128, 0, st>>>(*t, f->n_obj, n_heads, n_heads == 1);
  launch_adam_units(f, t, lr, beta1, beta2, eps, nullptr, 0, st);
  clear_counts_kernel<<<(f->n_obj + 127) / 128, 128, 0, st>>>(t->counts, f->n_obj);
  return check_launch("nif_adam_dev");
}

extern "C" int nif_train_prologue_cur_dev(const nif_family_view* f, const nif_train_view* t,
                                          const int64_t* obj, const int64_t* idx,
                                          const int64_t* cursor, int64_t n_rows, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int n_obj = f->n_obj, n_heads = f->n_heads;
  if (n_obj > 12 * 1024) {  // histogram beyond one CTA's shared memory
    clear_counts_kernel<<<(n_obj + 127) / 128, 128, 0, st>>>(t->counts, n_obj);
    if (n_rows > 0)
      batch_counts_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, st>>>(obj, idx, n_rows,
                                                                            n_obj, t->counts,
                                                                            cursor);
    const int n = n_obj > n_heads ? n_obj : n_heads;
    adam_steps_kernel<<<(n + 127) / 128, 128, 0, st>>>(*t, n_obj, n_heads, n_heads == 1);
    return check_launch("nif_train_prologue_cur_dev");
  }
  train_prologue_kernel<<<1, 1024, (size_t)n_obj * sizeof(int), st>>>(
      obj, idx, cursor, n_rows, *t, n_obj, n_heads, n_heads == 1);
  return check_launch("nif_train_prologue_cur_dev");
}

extern "C" int nif_adam_units_dev(const nif_family_view* f, const nif_train_view* t, double lr,
                                  double beta1, double beta2, double eps, int64_t* cursor,
                                  int64_t delta, void* stream) {
  launch_adam_units(f, t, lr, beta1, beta2, eps, cursor, delta, (cudaStream_t)stream);
  return check_launch("nif_adam_units_dev");
}

// ---------------------------------------------------------------------------
// Gradient sinks for data-parallel and deterministic training
// ---------------------------------------------------------------------------
namespace nif {
namespace {

// dst[i] += sum_c part[c][i], CTAs in order (deterministic MLP gradients);
// the [w | pad | b] padding is skipped
__global__ void mlp_reduce_kernel(const float* __restrict__ part, int n_cta, int64_t n_mlp,
                                  int64_t w_end, int64_t b_begin, float* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_mlp || (i >= w_end && i < b_begin)) return;
  float s = 0.f;
  for (int c = 0; c < n_cta; ++c) s += part[(size_t)c * n_mlp + i];
  dst[i] += s;
}

struct ScatterArgs {
  nif_family_view f;
  nif_train_view t;
  const int64_t* obj;
  const double* coord;
  const int64_t* idx;
  const int64_t* cursor;
  int64_t n_rows;
  const float* dx;  // [n_rows][IN]
  int slots;        // 8 (outer: 4 pos + 4 dir corners) or 10 (+ 2 dist)
};

// One contribution slot of batch row g: the grid cell (element offset of its
// first latent in the family buffer), the latent count, the fp64 corner
// weight and the offset of the matching inputs in dx -- grids.py:125-150
// corner order 00, 01, 10, 11 (2-D), i0, i1 (1-D)
struct Contrib {
  int64_t elem;
  int n, kbase;
  double w;
};

__device__ __forceinline__ Contrib contrib(const ScatterArgs& a, int64_t g, int slot) {
  const nif_family_view& f = a.f;
  const int64_t* bidx = batch_idx(a.idx, a.cursor);
  const int64_t row = bidx ? bidx[g] : g;
  const int o = (int)a.obj[row];
  const int cw = f.family == NIF_FAMILY_OUTER ? 4 : 5;
  const double* c = a.coord + row * cw;
  Contrib r;
  if (slot < 8) {
    const bool pos = slot < 4;
    const Bil64 b = pos ? bil64(c[0], c[1], f.R) : bil64(c[2], c[3], f.R);
    const int q = slot & 3;
    r.elem = (pos ? a.t.off_pos : a.t.off_dir) + ((int64_t)o * f.R * f.R + b.c[q]) * f.N;
    r.n = f.N;
    r.kbase = pos ? 0 : f.N;
    r.w = b.w[q];
  } else {
    const Axis ax = axis_indices(c[4], f.Rd, false);
    const bool hi = slot == 9;
    r.elem = a.t.off_dist + ((int64_t)o * f.Rd + (hi ? ax.i1 : ax.i0)) * f.Nd;
    r.n = f.Nd;
    r.kbase = 2 * f.N;
    r.w = hi ? ax.w : 1.0 - ax.w;
  }
  return r;
}

// Atomic scatter, warp-aggregated: a warp takes 32 consecutive batch rows
// of one slot; lanes that hit the same cell are combined (lane order) with
// __match_any_sync and the group's leader issues one fp32 atomic per latent.
__global__ void __launch_bounds__(256) scatter_atomic_kernel(ScatterArgs a) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t wid = t >> 5;
  const int slot = (int)(wid % a.slots);
  const int64_t g = (wid / a.slots) * 32 + lane;
  const bool valid = g < a.n_rows;
  const int IN = a.f.dims[0];
  Contrib c{};
  if (valid) c = contrib(a, g, slot);
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const unsigned peers = __match_any_sync(act, c.elem);
  const int leader = __ffs(peers) - 1;
  float* dst = a.t.grad + c.elem;
  for (int k = 0; k < c.n; ++k) {
    // grids.py:175: (w * up).astype(f32), then added into the fp32 grad
    float v = (float)(c.w * (double)a.dx[g * IN + c.kbase + k]);
    // leader accumulates its peers in ascending lane order
    unsigned rest = peers & ~(1u << lane);
    float sum = v;
    while (__any_sync(act, rest != 0u)) {
      const int src = rest ? __ffs(rest) - 1 : lane;
      const float pv = __shfl_sync(act, v, src);
      if (rest) {
        sum += pv;
        rest &= rest - 1;
      }
    }
    if (lane == leader) atomicAdd(dst + k, sum);
  }
}

// ---- deterministic=2: order-independent fixed-point scatter ---------------
// Every contribution (float)(w * dx) is scaled by 2^S (exact in fp64) and
// rounded to an int64; int64 atomic sums are associative, so the result is
// bit-identical whatever the atomics' order -- on every run and on every
// data-parallel rank -- at about the atomic scatter's cost. S is chosen per
// batch from max |dx| so no cell can overflow: |sum| <= 4 * n_rows * max|dx|
// < 2^62. The first contribution to a cell claims it (a per-cell tag) and
// lists it; each listed cell is then rounded once to fp32 (__ll2float_rn,
// then an exact power-of-two scale) and added into the grad, and its
// accumulator and tag cleared. Workspace: int64 per family element, uint32
// tag per element, the cell list, {max |dx| bits, list length, blocks done}
// -- zeroed once before first use; every call leaves it zeroed again.
struct FxWs {
  unsigned long long* acc;
  uint32_t* tag;
  uint32_t* list;
  uint32_t* state;  // [0] max |dx| (fp32 bits), [1] listed cells, [2] convert blocks done
};

__device__ __forceinline__ int fx_shift(const uint32_t* state, int64_t n_rows) {
  const float m = __uint_as_float(state[0]);
  int e = 0;
  const double bound = 4.0 * (double)n_rows * (double)m;  // bound < 2^e
  if (bound > 0.0) frexp(bound, &e);
  const int S = 62 - e;
  return S < 0 ? 0 : (S > 100 ? 100 : S);
}

__global__ void __launch_bounds__(256) fx_max_kernel(const float* __restrict__ dx, int64_t n,
                                                     uint32_t* state) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(dx[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(state, __float_as_uint(m));  // m >= 0
}

__device__ __forceinline__ long long fx_q(float v, int S) {
  return __double2ll_rn(ldexp((double)v, S));
}

// pass 2: warp-aggregated int64 atomics (exact sums, any order); the first
// contribution to each cell lists it
__global__ void __launch_bounds__(256) scatter_fx_add_kernel(ScatterArgs a, FxWs w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t wid = t >> 5;
  const int slot = (int)(wid % a.slots);
  const int64_t g = (wid / a.slots) * 32 + lane;
  const bool valid = g < a.n_rows;
  const int IN = a.f.dims[0];
  const int S = fx_shift(w.state, a.n_rows);
  Contrib c{};
  if (valid) c = contrib(a, g, slot);
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const unsigned peers = __match_any_sync(act, c.elem);
  const int leader = __ffs(peers) - 1;
  for (int k = 0; k < c.n; ++k) {
    const long long q = fx_q((float)(c.w * (double)a.dx[g * IN + c.kbase + k]), S);
    unsigned rest = peers & ~(1u << lane);
    long long sum = q;
    while (__any_sync(act, rest != 0u)) {
      const int src = rest ? __ffs(rest) - 1 : lane;
      const long long pv = __shfl_sync(act, q, src);
      if (rest) {
        sum += pv;
        rest &= rest - 1;
      }
    }
    if (lane == leader) atomicAdd(w.acc + c.elem + k, (unsigned long long)sum);
  }
  if (lane == leader && atomicExch(w.tag + c.elem, 1u) == 0u)
    w.list[atomicAdd(w.state + 1, 1u)] = (uint32_t)c.elem;
}

// pass 3: each listed cell, int64 -> fp32 once; the last block re-zeroes the state
template <int NL>
__device__ __forceinline__ void fx_convert_cell(unsigned long long* __restrict__ acc,
                                                float* __restrict__ grad, float inv) {
  long long q[NL];
  float g[NL];
#pragma unroll
  for (int k = 0; k < NL; ++k) {  // every load in flight before the first store
    q[k] = (long long)acc[k];
    g[k] = grad[k];
  }
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    acc[k] = 0ull;
    grad[k] = g[k] + __fmul_rn(__ll2float_rn(q[k]), inv);
  }
}

__global__ void __launch_bounds__(256) scatter_fx_convert_kernel(ScatterArgs a, FxWs w) {
  const int S = fx_shift(w.state, a.n_rows);
  const float inv = __int_as_float((127 - S) << 23);  // 2^-S, exact (0 <= S <= 100)
  const uint32_t n_cells = w.state[1];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_cells;
       i += gridDim.x * blockDim.x) {
    const int64_t elem = w.list[i];
    const bool dist = a.f.family == NIF_FAMILY_INNER && elem >= a.t.off_dist;
    const int n = dist ? a.f.Nd : a.f.N;
    unsigned long long* acc = w.acc + elem;
    float* grad = a.t.grad + elem;
    switch (n) {
      case 1: fx_convert_cell<1>(acc, grad, inv); break;
      case 2: fx_convert_cell<2>(acc, grad, inv); break;
      case 3: fx_convert_cell<3>(acc, grad, inv); break;
      case 4: fx_convert_cell<4>(acc, grad, inv); break;
      case 5: fx_convert_cell<5>(acc, grad, inv); break;
      case 6: fx_convert_cell<6>(acc, grad, inv); break;
      case 7: fx_convert_cell<7>(acc, grad, inv); break;
      default: fx_convert_cell<8>(acc, grad, inv); break;
    }
    w.tag[elem] = 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(w.state + 2, 1u) == gridDim.x - 1) {  // every block has read the state
      w.state[0] = 0u;
      w.state[1] = 0u;
      w.state[2] = 0u;
    }
  }
}

constexpr int kLatStride = 8;  // floats per precomputed contribution (N, Nd <= 8)

// Deterministic scatter, pass 1: per contribution t = g * slots + slot, its
// fp32 values (float)(w * dx) per latent and a 32-bit sort key (cell
// element << 2 | corner). The keys are written in t order, i.e. batch-row
// major, and the radix sort is stable, so equal keys stay in batch order:
// sorted by (cell, corner, row) -- np.add.at's order for that cell.
__global__ void scatter_keys_kernel(ScatterArgs a, uint32_t* __restrict__ keys,
                                    uint32_t* __restrict__ ids, float* __restrict__ vals) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.n_rows * a.slots) return;
  const int64_t g = t / a.slots;
  const int slot = (int)(t - g * a.slots);
  const Contrib c = contrib(a, g, slot);
  const int corner = slot < 8 ? (slot & 3) : slot - 8;
  keys[t] = ((uint32_t)c.elem << 2) | (uint32_t)corner;
  ids[t] = (uint32_t)t;
  const int IN = a.f.dims[0];
  float* v = vals + t * kLatStride;
  for (int k = 0; k < c.n; ++k) v[k] = (float)(c.w * (double)a.dx[g * IN + c.kbase + k]);
}

// pass 2: one warp per sorted position; the warp whose position starts a
// cell's run walks the run 32 contributions at a time (lanes load in
// parallel, coalesced) and adds them in sorted order into fp32
// accumulators seeded with the grad: one sequential fp32 sum per latent,
// exactly np.add.at's. (Runs can be hundreds long -- e.g. the outer
// direction grid, where one light makes most shadow rays of an object hit
// the same few cells -- so a thread-serial walk would be latency-bound.)
template <int NL>
__device__ __forceinline__ void seg_sum_warp(float* dst, const uint32_t* keys,
                                             const uint32_t* ids, const float* vals, int64_t i,
                                             int64_t n_keys, uint32_t cell, int lane) {
  float acc[NL];
#pragma unroll
  for (int k = 0; k < NL; ++k) acc[k] = dst[k];
  for (int64_t j0 = i;; j0 += 32) {
    const int64_t j = j0 + lane;
    const bool in = j < n_keys && (keys[j] >> 2) == cell;
    const unsigned m = __ballot_sync(0xffffffffu, in);  // a prefix of the lanes (sorted)
    float v[NL];
    if (in) {
      const float* src = vals + (size_t)ids[j] * kLatStride;
#pragma unroll
      for (int k = 0; k < NL; ++k) v[k] = src[k];
    }
    const int cnt = __popc(m);
    for (int q = 0; q < cnt; ++q)
#pragma unroll
      for (int k = 0; k < NL; ++k) acc[k] += __shfl_sync(0xffffffffu, v[k], q);
    if (cnt < 32) break;
  }
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NL; ++k) dst[k] = acc[k];
}

__global__ void __launch_bounds__(256) scatter_segments_kernel(
    ScatterArgs a, const uint32_t* __restrict__ keys, const uint32_t* __restrict__ ids,
    const float* __restrict__ vals, int64_t n_keys) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n_keys) return;
  const uint32_t cell = keys[i] >> 2;
  if (i > 0 && (keys[i - 1] >> 2) == cell) return;  // warp-uniform
  const bool dist = a.f.family == NIF_FAMILY_INNER && (int64_t)cell >= a.t.off_dist;
  const int n = dist ? a.f.Nd : a.f.N;
  float* dst = a.t.grad + cell;
  switch (n) {
    case 1: seg_sum_warp<1>(dst, keys, ids, vals, i, n_keys, cell, lane); break;
    case 2: seg_sum_warp<2>(dst, keys, ids, vals, i, n_keys, cell, lane); break;
    case 3: seg_sum_warp<3>(dst, keys, ids, vals, i, n_keys, cell, lane); break;
    case 4: seg_sum_warp<4>(dst, keys, ids, vals, i, n_keys, cell, lane); break;
    case 5: seg_sum_warp<5>(dst, keys, ids, vals, i, n_keys, cell, lane); break;
    case 6: seg_sum_warp<6>(dst, keys, ids, vals, i, n_keys, cell, lane); break;
    case 7: seg_sum_warp<7>(dst, keys, ids, vals, i, n_keys, cell, lane); break;
    default: seg_sum_warp<8>(dst, keys, ids, vals, i, n_keys, cell, lane); break;
  }
}

int bits_for(uint64_t v) {
  int b = 0;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

struct ScatterWs {
  uint32_t *keys_in, *keys_out, *ids_in, *ids_out;
  float* vals;
  void* temp;
  size_t temp_bytes, total;
};

size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

ScatterWs scatter_ws(int64_t n_keys, int end_bit, void* base) {
  ScatterWs w{};
  size_t temp = 0;
  const int nk = (int)(n_keys > 0 ? n_keys : 1);
  cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, nk, 0, end_bit);
  const size_t kb = al256((size_t)nk * 4);
  uint8_t* p = (uint8_t*)base;
  w.keys_in = (uint32_t*)p;
  w.keys_out = (uint32_t*)(p + kb);
  w.ids_in = (uint32_t*)(p + 2 * kb);
  w.ids_out = (uint32_t*)(p + 3 * kb);
  w.vals = (float*)(p + 4 * kb);
  const size_t vb = al256((size_t)nk * kLatStride * 4);
  w.temp = p + 4 * kb + vb;
  w.temp_bytes = temp;
  w.total = 4 * kb + vb + al256(temp);
  return w;
}

int scatter_slots(const nif_family_view* f) { return f->family == NIF_FAMILY_INNER ? 10 : 8; }

}  // namespace
}  // namespace nif

extern "C" int nif_train_fwdbwd_ex_dev(const nif_family_view* f, const nif_train_view* t,
                                       const int64_t* obj, const double* coord,
                                       const float* label, const int64_t* idx,
                                       const int64_t* cursor, int64_t n_rows, int64_t row0,
                                       int64_t row_step, double* sq_err, float* dx_out,
                                       float* mlp_grad, float* mlp_part, int64_t part_floats,
                                       void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n_mlp = t->off_b - t->off_w + (int64_t)f->n_heads * f->b_stride;
  float* dst = mlp_grad ? mlp_grad : t->grad + t->off_w;
  TrainArgs a{*f, *t, obj, coord, label, idx, n_rows, row0, row_step, sq_err, cursor,
              dst, mlp_part, n_mlp, dx_out, part_floats};
  int rc = launch_fwdbwd_any(a, st);
  if (rc != NIF_OK || mlp_part == nullptr || g_last_ctas == 0) return rc;
  const int64_t w_end = (int64_t)f->n_heads * f->w_stride, b_begin = t->off_b - t->off_w;
  mlp_reduce_kernel<<<(unsigned)((n_mlp + 255) / 256), 256, 0, st>>>(
      mlp_part, (int)g_last_ctas, n_mlp, w_end, b_begin, dst);
  return check_launch("nif_train_fwdbwd_ex_dev(reduce)");
}

extern "C" int64_t nif_train_part_floats(const nif_family_view* f, const nif_train_view* t,
                                         int64_t n_rows) {
  // worst case over the kernels: 16 rows per CTA (tiled), 32 (per-row floor)
  const int64_t n_mlp = t->off_b - t->off_w + (int64_t)f->n_heads * f->b_stride;
  return ((n_rows + 15) / 16) * n_mlp;
}

extern "C" size_t nif_grid_scatter_ws_bytes(const nif_family_view* f, const nif_train_view* t,
                                            int64_t n_rows, int deterministic) {
  if (deterministic == 2)  // acc, tag, list, state
    return al256((size_t)t->numel * 8) + al256((size_t)t->numel * 4) +
           al256((size_t)(n_rows * scatter_slots(f)) * 4) + 256;
  if (deterministic == 1)
    return scatter_ws(n_rows * scatter_slots(f), bits_for((uint64_t)t->numel) + 2, nullptr).total;
  return 0;
}

extern "C" int nif_grid_scatter_dev(const nif_family_view* f, const nif_train_view* t,
                                    const int64_t* obj, const double* coord, const int64_t* idx,
                                    const int64_t* cursor, int64_t n_rows, const float* dx,
                                    int deterministic, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_rows <= 0) return NIF_OK;
  if (f->N > kLatStride || f->Nd > kLatStride)
    return fail(NIF_ERR_UNSUPPORTED, "more than %d latents per cell", kLatStride);
  ScatterArgs a{*f, *t, obj, coord, idx, cursor, n_rows, dx, scatter_slots(f)};
  const int64_t n_keys = n_rows * a.slots;
  if (!deterministic) {
    const int64_t threads = ((n_rows + 31) / 32) * 32 * a.slots;
    scatter_atomic_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(a);
    return check_launch("nif_grid_scatter_dev(atomic)");
  }
  if (deterministic == 2) {
    const size_t need = nif_grid_scatter_ws_bytes(f, t, n_rows, 2);
    if (ws == nullptr || ws_bytes < need)
      return fail(NIF_ERR_VALUE, "scatter workspace needs %zu bytes", need);
    // [state | acc | tag | list]: the list last, so calls with fewer rows
    // than the workspace was sized for see the same state / accumulators
    uint8_t* p = (uint8_t*)ws;
    const size_t o1 = 256, o2 = o1 + al256((size_t)t->numel * 8);
    const size_t o3 = o2 + al256((size_t)t->numel * 4);
    FxWs w{(unsigned long long*)(p + o1), (uint32_t*)(p + o2), (uint32_t*)(p + o3),
           (uint32_t*)p};
    const int64_t n_dx = n_rows * f->dims[0];
    int64_t mb = (n_dx + 1023) / 1024;
    if (mb > sm_count()) mb = sm_count();
    fx_max_kernel<<<(unsigned)(mb > 0 ? mb : 1), 256, 0, st>>>(dx, n_dx, w.state);
    const int64_t threads = ((n_rows + 31) / 32) * 32 * a.slots;
    scatter_fx_add_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(a, w);
    int64_t cb = (n_keys + 255) / 256;
    if (cb > 2 * sm_count()) cb = 2 * sm_count();
    scatter_fx_convert_kernel<<<(unsigned)cb, 256, 0, st>>>(a, w);
    return check_launch("nif_grid_scatter_dev(fixed point)");
  }
  const int end_bit = bits_for((uint64_t)t->numel) + 2;
  if (end_bit > 32 || n_keys > INT32_MAX)
    return fail(NIF_ERR_UNSUPPORTED, "deterministic scatter: family buffer above 2^30 floats");
  ScatterWs w = scatter_ws(n_keys, end_bit, ws);
  if (ws == nullptr || ws_bytes < w.total)
    return fail(NIF_ERR_VALUE, "scatter workspace needs %zu bytes", w.total);
  const unsigned blocks = (unsigned)((n_keys + 255) / 256);
  scatter_keys_kernel<<<blocks, 256, 0, st>>>(a, w.keys_in, w.ids_in, w.vals);
  size_t tb = w.temp_bytes;
  // stable: equal (cell, corner) keys keep batch-row order
  if (cub::DeviceRadixSort::SortPairs(w.temp, tb, w.keys_in, w.keys_out, w.ids_in, w.ids_out,
                                      (int)n_keys, 0, end_bit, st) != cudaSuccess)
    return check_launch("nif_grid_scatter_dev(sort)");
  scatter_segments_kernel<<<(unsigned)((n_keys + 7) / 8), 256, 0, st>>>(a, w.keys_out, w.ids_out,
                                                                       w.vals, n_keys);
  return check_launch("nif_grid_scatter_dev(deterministic)");
}
