// Phase 2 of the split visibility pass: per-record grid encoding, the
// visibility MLP, the p < 0.5 threshold and the per-ray OR
// (nif.py:467-483 infer_records, renderer.py:675-683 PredictorBackend).
//
// Two implementations behind nif_query_dev:
//  * query_tc_kernel  -- persistent, 128 records per tile (M = 128 rows of
//    tcgen05.mma kind::f16), features/activations staged fp16 in shared
//    memory in the UMMA canonical K-major layout, fp32 accumulators in TMEM,
//    biases folded into the GEMMs through a constant-one input column, the
//    N=1 head run as an N=16 MMA. Weights live in shared memory for the
//    kernel's lifetime; latent tables are fp16 (nif_fast_pack_dev).
//  * query_simt_kernel -- fp32 CUDA-core kernel over the fp32 master
//    tables; the numerical anchor for the tensor-core path and the path for
//    configurations the tensor-core kernel does not cover (per-object MLPs,
//    the geometry head, very wide inputs).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdlib>
#include <stdint.h>

#include "common.h"
#include "kernels.h"
#include "nif_b200.h"
#include "status.h"
#include "tc.cuh"

namespace nif {
namespace {

constexpr float kSlope = 0.01f;  // mlp.py:17 HIDDEN_SLOPE
constexpr int kTileRows = 128;
constexpr int kK1 = 16;          // padded layer-1 K (features + bias column)
// Tiles of 128 records a CTA advances in lockstep (one barrier / commit per
// layer for all of them). Measured on B200 at C2: 1 beats 2 (more CTAs per
// SM hide the MMA round trip better than batching it).
constexpr int kTpc = 1;

#ifndef NIF_TS_PROF
#define NIF_TS_PROF 0  // 1: clock64 phase stamps in query_ts_kernel (nif_debug_set_prof)
#endif

// ---------------------------------------------------------------------------
// fast blob layout
// ---------------------------------------------------------------------------

#ifndef NIF_CPACK8
#define NIF_CPACK8 1  // corner-packed 64 B entries for 8-latent tables (inner family)
#endif
struct FastLayout {
  int W, L, in_dim, Kp, NP, NPd, R, Rd, N, Nd, n_obj;
  int HD;  // head outputs: 1 (occlusion logit) or 4 (geometry: normal + depth)
  size_t off_w1, off_hidden, off_head, off_headf, w_bytes;
  size_t w_stride_blob;  // bytes between the weight blocks of two heads
  int n_heads;
  size_t off_pos, off_dir, off_dist, total;
  int tmem_cols;
  bool tc_ok;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 255) / 256 * 256; }

__host__ __device__ inline FastLayout make_layout(const nif_family_view& f) {
  FastLayout l{};
  l.in_dim = f.dims[0];
  l.W = f.dims[1];
  l.L = f.n_layers - 1;
  l.Kp = ((l.W + 1) + 15) / 16 * 16;
  l.N = f.N;
  l.Nd = f.Nd;
  l.NP = f.N <= 4 ? 4 : 8;
  l.NPd = 4;
  l.R = f.R;
  l.Rd = f.Rd;
  l.n_obj = f.n_obj;
  l.off_w1 = 0;
  l.off_hidden = l.off_w1 + (size_t)l.W * kK1 * 2;
  l.off_head = l.off_hidden + (size_t)(l.L > 0 ? l.L - 1 : 0) * l.W * l.Kp * 2;
  // fp32 head rows [HD][W] then the HD biases (CUDA-core head)
  l.HD = f.dims[f.n_layers];
  l.off_headf = l.off_head + (size_t)16 * l.Kp * 2;
  l.w_bytes = l.off_headf + ((size_t)l.HD * (l.W + 1) * 4 + 15) / 16 * 16;
  // one weight block per head (per_object sharing: one MLP per object)
  l.n_heads = f.n_heads;
  l.w_stride_blob = al16(l.w_bytes);
  l.off_pos = l.w_stride_blob * (size_t)(f.n_heads > 0 ? f.n_heads : 1);
  // 2-D tables with 4 latents per cell (outer) are corner-packed: one
  // 32 B entry per (u cell, v cell + 1) holding the four bilinear corners
  // (u wrap and v clamp applied), so a lookup is one sector and two 16 B
  // loads. With 8 latents per cell (inner) the packed entry would be 64 B
  // for the same four 16 B loads and a 4x larger footprint (measured
  // slower at R <= 128), so those stay one cell per 16 B. 1-D: corner pairs.
  const size_t tab = (l.NP == 4 || NIF_CPACK8) ? (size_t)f.n_obj * f.R * (f.R + 1) * 4 * l.NP * 2
                                              : (size_t)f.n_obj * f.R * f.R * l.NP * 2;
  l.off_dir = al16(l.off_pos + tab);
  l.off_dist = al16(l.off_dir + tab);
  const size_t dtab =
      f.family == NIF_FAMILY_INNER ? (size_t)f.n_obj * (f.Rd + 1) * 2 * l.NPd * 2 : 0;
  l.total = al16(l.off_dist + dtab);
  int cols = kTpc * ((l.W + 31) / 32 * 32);  // kTpc tiles x W accumulator columns
  l.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  bool hidden_same = true;
  for (int i = 1; i < f.n_layers; ++i) hidden_same = hidden_same && f.dims[i] == l.W;
  const bool inst = (f.family == NIF_FAMILY_OUTER && (f.N == 2 || f.N == 3 || f.N == 4)) ||
                    (f.family == NIF_FAMILY_INNER &&
                     ((f.N == 5 && (f.Nd == 3 || f.Nd == 4)) || (f.N == 4 && f.Nd == 3)));
  const bool head_ok = (f.sigmoid_head == 1 && l.HD == 1) || (f.sigmoid_head == 0 && l.HD == 4);
  l.tc_ok = inst && f.n_heads >= 1 && head_ok &&
            l.L >= 1 && hidden_same && l.W % 16 == 0 && l.W >= 16 && l.W <= 240 &&
            l.in_dim + 1 <= kK1;
  return l;
}

// byte offset of element (r, k) in a K-major canonical tile with K = kp
__host__ __device__ inline size_t canon_off(int r, int k, int kp) {
  return (size_t)(r >> 3) * (kp * 16) + (size_t)(k >> 3) * 128 + (size_t)(r & 7) * 16 +
         (size_t)(k & 7) * 2;
}

// weights -> fp16 canonical tiles with the bias folded into column `in`
__global__ void pack_weights_kernel(nif_family_view f, FastLayout l, uint8_t* blob) {
  // blockIdx.y = head: per_object sharing packs one weight block per object
  blob += (size_t)blockIdx.y * l.w_stride_blob;
  f.w += (size_t)blockIdx.y * f.w_stride;
  f.b += (size_t)blockIdx.y * f.b_stride;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int n1 = l.W * kK1;
  const int nh = (l.L - 1) * l.W * l.Kp;
  const int nhead = 16 * l.Kp;
  if (idx >= n1 + nh + nhead + l.HD * (l.W + 1)) return;
  if (idx >= n1 + nh + nhead) {  // fp32 copy of the head rows [HD][W], then the HD biases
    const int k = idx - n1 - nh - nhead;
    const size_t wo = (size_t)f.dims[0] * l.W + (size_t)(l.L - 1) * l.W * l.W;
    reinterpret_cast<float*>(blob + l.off_headf)[k] =
        k < l.HD * l.W ? f.w[wo + k] : f.b[(size_t)l.W * l.L + (k - l.HD * l.W)];
    return;
  }
  float val = 0.f;
  size_t off;
  if (idx < n1) {
    const int r = idx / kK1, k = idx % kK1;
    const int nin = f.dims[0];
    if (k < nin) val = f.w[(size_t)r * nin + k];
    else if (k == nin) val = f.b[r];
    off = l.off_w1 + canon_off(r, k, kK1);
  } else if (idx < n1 + nh) {
    const int j = idx - n1;
    const int layer = j / (l.W * l.Kp);  // hidden tile index -> dense layer layer+1
    const int rem = j % (l.W * l.Kp);
    const int r = rem / l.Kp, k = rem % l.Kp;
    size_t wo = (size_t)f.dims[0] * l.W + (size_t)layer * l.W * l.W;
    size_t bo = (size_t)l.W * (layer + 1);
    if (k < l.W) val = f.w[wo + (size_t)r * l.W + k];
    else if (k == l.W) val = f.b[bo + r];
    off = l.off_hidden + (size_t)layer * l.W * l.Kp * 2 + canon_off(r, k, l.Kp);
  } else {
    const int j = idx - n1 - nh;
    const int r = j / l.Kp, k = j % l.Kp;
    size_t wo = (size_t)f.dims[0] * l.W + (size_t)(l.L - 1) * l.W * l.W;
    size_t bo = (size_t)l.W * l.L;
    if (r == 0 && k < l.W) val = f.w[wo + k];
    else if (r == 0 && k == l.W) val = f.b[bo];
    off = l.off_head + canon_off(r, k, l.Kp);
  }
  *reinterpret_cast<__half*>(blob + off) = __float2half_rn(val);
}

// fp32 master latents -> corner-packed fp16 tables (one thread per corner
// of an entry). 2-D entry (iu, jq), jq in [0, R]: corners (iu, jv0),
// (iu, jv1), (iu+1 mod R, jv0), (iu+1 mod R, jv1) with jv0 = clamp(jq-1),
// jv1 = clamp(jq) -- exactly the four cells grids.py:125-150 combines for
// floor(v R - 0.5) = jq - 1. 1-D entry jq in [0, Rd]: (clamp(jq-1), clamp(jq)).
__global__ void pack_tables_kernel(nif_family_view f, FastLayout l, uint8_t* blob) {
  const int R = l.R, Rd = l.Rd;
  const bool quad = l.NP == 4 || NIF_CPACK8;
  const int64_t ent2 = quad ? (int64_t)l.n_obj * R * (R + 1) * 4 : (int64_t)l.n_obj * R * R;
  const int64_t ent1 = f.family == NIF_FAMILY_INNER ? (int64_t)l.n_obj * (Rd + 1) * 2 : 0;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < 2 * ent2 && !quad) {
    const bool is_dir = idx >= ent2;
    const int64_t c = is_dir ? idx - ent2 : idx;
    const float* src = (is_dir ? f.dir : f.pos) + c * l.N;
    __half* dst = reinterpret_cast<__half*>(blob + (is_dir ? l.off_dir : l.off_pos)) + c * l.NP;
    for (int k = 0; k < l.NP; ++k) dst[k] = __float2half_rn(k < l.N ? src[k] : 0.f);
  } else if (idx < 2 * ent2) {
    const bool is_dir = idx >= ent2;
    const int64_t e = is_dir ? idx - ent2 : idx;  // ((o * R + iu) * (R+1) + jq) * 4 + c
    const int c = (int)(e & 3);
    const int64_t q = e >> 2;
    const int jq = (int)(q % (R + 1));
    const int64_t oi = q / (R + 1);
    const int iu = (int)(oi % R);
    const int64_t o = oi / R;
    const int u = (c >> 1) ? (iu + 1 == R ? 0 : iu + 1) : iu;
    int jv = (c & 1) ? jq : jq - 1;
    jv = jv < 0 ? 0 : (jv > R - 1 ? R - 1 : jv);
    const float* src = (is_dir ? f.dir : f.pos) + (((size_t)o * R + u) * R + jv) * l.N;
    __half* dst = reinterpret_cast<__half*>(blob + (is_dir ? l.off_dir : l.off_pos)) + e * l.NP;
    for (int k = 0; k < l.NP; ++k) dst[k] = __float2half_rn(k < l.N ? src[k] : 0.f);
  } else if (idx < 2 * ent2 + ent1) {
    const int64_t e = idx - 2 * ent2;  // ((o * (Rd+1)) + jq) * 2 + c
    const int c = (int)(e & 1);
    const int64_t q = e >> 1;
    const int jq = (int)(q % (Rd + 1));
    const int64_t o = q / (Rd + 1);
    int j = c ? jq : jq - 1;
    j = j < 0 ? 0 : (j > Rd - 1 ? Rd - 1 : j);
    const float* src = f.dist + ((size_t)o * Rd + j) * l.Nd;
    __half* dst = reinterpret_cast<__half*>(blob + l.off_dist) + e * l.NPd;
    for (int k = 0; k < l.NPd; ++k) dst[k] = __float2half_rn(k < l.Nd ? src[k] : 0.f);
  }
}

// ---------------------------------------------------------------------------
// interpolation helpers (fp32 coordinates, cell-centred, u wraps, v clamps)
// ---------------------------------------------------------------------------

struct Bil {
  int iu0, iu1, iv0, iv1;
  float w00, w01, w10, w11;
};

__device__ __forceinline__ Bil bilinear(float u, float v, int R) {
  Bil b;
  u = u - floorf(u);  // wrap period 1 in u == wrap period R in the index
  const float xu = u * (float)R - 0.5f;
  const float fu = floorf(xu);
  const float wu = xu - fu;
  int i0 = (int)fu, i1 = i0 + 1;
  if (i0 < 0) i0 += R;
  if (i1 >= R) i1 -= R;
  const float xv = v * (float)R - 0.5f;
  const float fv = floorf(xv);
  const float wv = xv - fv;
  int j0 = (int)fv, j1 = j0 + 1;
  j0 = min(max(j0, 0), R - 1);
  j1 = min(max(j1, 0), R - 1);
  b.iu0 = i0;
  b.iu1 = i1;
  b.iv0 = j0;
  b.iv1 = j1;
  b.w00 = (1.f - wu) * (1.f - wv);
  b.w01 = (1.f - wu) * wv;
  b.w10 = wu * (1.f - wv);
  b.w11 = wu * wv;
  return b;
}

struct Lin {
  int i0, i1;
  float w;
};

__device__ __forceinline__ Lin linear1(float x, int R) {
  const float xc = x * (float)R - 0.5f;
  const float f0 = floorf(xc);
  Lin l;
  l.w = xc - f0;
  int i0 = (int)f0, i1 = i0 + 1;
  l.i0 = min(max(i0, 0), R - 1);
  l.i1 = min(max(i1, 0), R - 1);
  return l;
}

// ---------------------------------------------------------------------------
// SIMT fp32 query kernel
// ---------------------------------------------------------------------------

constexpr int kSimtMaxIn = 64;
constexpr int kSimtMaxW = 256;

__global__ void __launch_bounds__(128)
query_simt_kernel(nif_family_view f, const int32_t* __restrict__ obj,
                  const int32_t* __restrict__ ray, const float* __restrict__ coord4,
                  const float* __restrict__ rr, const int64_t* __restrict__ count, int64_t cap,
                  uint8_t* __restrict__ occ, float* __restrict__ logits) {
  const int64_t n = min(*count, cap);
  float x[kSimtMaxIn];
  float a[kSimtMaxW], b[kSimtMaxW];
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int o = obj[j];
    const float4 c = reinterpret_cast<const float4*>(coord4)[j];
    const size_t g2 = (size_t)f.R * f.R * f.N;
    const float* gp = f.pos + (size_t)o * g2;
    const float* gd = f.dir + (size_t)o * g2;
    Bil bp = bilinear(c.x, c.y, f.R), bd = bilinear(c.z, c.w, f.R);
    for (int k = 0; k < f.N; ++k) {
      x[k] = bp.w00 * gp[((size_t)bp.iu0 * f.R + bp.iv0) * f.N + k] +
             bp.w01 * gp[((size_t)bp.iu0 * f.R + bp.iv1) * f.N + k] +
             bp.w10 * gp[((size_t)bp.iu1 * f.R + bp.iv0) * f.N + k] +
             bp.w11 * gp[((size_t)bp.iu1 * f.R + bp.iv1) * f.N + k];
      x[f.N + k] = bd.w00 * gd[((size_t)bd.iu0 * f.R + bd.iv0) * f.N + k] +
                   bd.w01 * gd[((size_t)bd.iu0 * f.R + bd.iv1) * f.N + k] +
                   bd.w10 * gd[((size_t)bd.iu1 * f.R + bd.iv0) * f.N + k] +
                   bd.w11 * gd[((size_t)bd.iu1 * f.R + bd.iv1) * f.N + k];
    }
    if (f.family == NIF_FAMILY_INNER) {
      const Lin l = linear1(rr[j], f.Rd);
      const float* gr = f.dist + (size_t)o * f.Rd * f.Nd;
      for (int k = 0; k < f.Nd; ++k)
        x[2 * f.N + k] = (1.f - l.w) * gr[(size_t)l.i0 * f.Nd + k] + l.w * gr[(size_t)l.i1 * f.Nd + k];
    }
    const int head = f.n_heads > 1 ? o : 0;
    const float* W = f.w + (size_t)head * f.w_stride;
    const float* B = f.b + (size_t)head * f.b_stride;
    for (int k = 0; k < f.dims[0]; ++k) a[k] = x[k];
    int wo = 0, bo = 0;
    for (int layer = 0; layer < f.n_layers; ++layer) {
      const int nin = f.dims[layer], nout = f.dims[layer + 1];
      for (int q = 0; q < nout; ++q) {
        float acc = __ldg(B + bo + q);
        const float* wr = W + wo + q * nin;
        for (int k = 0; k < nin; ++k) acc = fmaf(__ldg(wr + k), a[k], acc);
        b[q] = (layer < f.n_layers - 1) ? (acc > 0.f ? acc : kSlope * acc) : acc;
      }
      wo += nin * nout;
      bo += nout;
      for (int q = 0; q < nout; ++q) a[q] = b[q];
    }
    const int od = f.dims[f.n_layers];
    if (logits)
      for (int q = 0; q < od; ++q) logits[j * od + q] = a[q];
    if (occ && f.sigmoid_head == 1 && a[0] < 0.f) occ[ray[j]] = 1;
  }
}

// ---------------------------------------------------------------------------
// tcgen05 fused query kernel
// ---------------------------------------------------------------------------

struct TcArgs {
  const uint8_t* blob;
  FastLayout l;
  const int32_t* obj;
  const int32_t* ray;
  const float* coord4;
  const float* rr;
  const int64_t* count;
  int64_t cap;
  uint8_t* occ;
  float* logits;
  long long* prof;  // diagnostic phase timestamps (nif_debug_set_prof), or NULL
  // per_object sharing: records bucketed by object into 128-row tiles
  const int32_t* perm;      // [tile * 128 + row] -> record index, -1 = padding
  const int32_t* tile_obj;  // [tile] -> object (= head)
  const int64_t* n_tiles;   // device count of bucketed tiles
  // diagnostic timeline (nif_debug_set_timeline), or NULL: per warpgroup
  // globaltimer at entry, after the grid dependency wait, after the first
  // tile, at exit, and the tile count
  unsigned long long* tl;
};

long long* g_prof = nullptr;
unsigned long long* g_tl_query = nullptr;
int g_query_variant = 0;  // nif_debug_set_query_variant
int g_query_cpsm = 0;     // CTAs per SM cap of the fused query grids (0: TMEM/occupancy bound)

__device__ __forceinline__ void store_chunk(uint8_t* base, int row, int chunk, int kp,
                                            uint4 v) {
  *reinterpret_cast<uint4*>(base + (size_t)(row >> 3) * (kp * 16) + chunk * 128 +
                            (row & 7) * 16) = v;
}

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// Two-stage software pipeline of the per-record inputs: while tile k runs
// its MMA chain, the latent-table corners of tile k+1 are in flight
// (issued right after tile k's first MMA) and the record words of tile
// k+2 are being fetched, so the dependent gathers (record -> indices ->
// corners) never sit on the critical path of a tile.
struct RecIn {
  int obj, ray, rec;  // rec: record index (differs from the row for bucketed tiles)
  float4 c;
  float r;
  bool valid;
};

// Raw corner data of one record, gathered a tile ahead: NP/2 16-byte loads
// per 2-D lookup (outer NP=4: two corners per load; inner NP=8: one) and
// one for the 1-D distance pair.
template <int N, int ND>
struct EncIn {
  static constexpr int NP = N <= 4 ? 4 : 8;
  static constexpr int NQ = NP / 2;  // 16 B loads per 2-D lookup (2 packed / 4 cells)
  uint4 qp[NQ], qd[NQ], qr;
  float wp[4], wd[4], wr;
  int ray, rec;
  bool valid;
};

// 32-byte read-only load (LDG.256 on sm_100) of an aligned entry
__device__ __forceinline__ void ldg256(const uint4* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z),
                 "=r"(b.w)
               : "l"(p));
}

// bilinear entry of the corner-packed table: (u cell) x (v cell + 1)
struct BilQ {
  int q;
  float w00, w01, w10, w11;
};

__device__ __forceinline__ BilQ bilinear_q(float u, float v, int R) {
  BilQ b;
  u = u - floorf(u);
  const float xu = u * (float)R - 0.5f;
  const float fu = floorf(xu);
  const float wu = xu - fu;
  int i0 = (int)fu;
  if (i0 < 0) i0 += R;
  if (i0 > R - 1) i0 = R - 1;
  const float xv = v * (float)R - 0.5f;
  const float fv = floorf(xv);
  const float wv = xv - fv;
  const int jq = (int)fminf(fmaxf(fv + 1.0f, 0.0f), (float)R);
  b.q = i0 * (R + 1) + jq;
  b.w00 = (1.f - wu) * (1.f - wv);
  b.w01 = (1.f - wu) * wv;
  b.w10 = wu * (1.f - wv);
  b.w11 = wu * wv;
  return b;
}

__device__ __forceinline__ RecIn load_rec(const TcArgs& a, int64_t tile, int tid, int64_t n,
                                          bool inner) {
  RecIn r;
  const int64_t row = tile * kTileRows + tid;
  r.valid = row < n;
  r.obj = 0;
  r.ray = 0;
  r.rec = (int)row;
  r.c = make_float4(0.f, 0.f, 0.f, 0.f);
  r.r = 0.f;
  if (r.valid) {
    r.obj = __ldg(a.obj + row);
    r.ray = __ldg(a.ray + row);
    r.c = __ldg(reinterpret_cast<const float4*>(a.coord4) + row);
    if (inner) r.r = __ldg(a.rr + row);
  }
  return r;
}

// record of a bucketed tile (per_object sharing): row -> record index via
// perm, -1 = padding
__device__ __forceinline__ RecIn load_rec_perm(const TcArgs& a, int64_t tile, int tid,
                                               int64_t t_end, bool inner) {
  RecIn r;
  r.valid = false;
  r.obj = 0;
  r.ray = 0;
  r.rec = -1;
  r.c = make_float4(0.f, 0.f, 0.f, 0.f);
  r.r = 0.f;
  if (tile < t_end) {
    const int idx = __ldg(a.perm + tile * kTileRows + tid);
    if (idx >= 0) {
      r.valid = true;
      r.rec = idx;
      r.obj = __ldg(a.obj + idx);
      r.ray = __ldg(a.ray + idx);
      r.c = __ldg(reinterpret_cast<const float4*>(a.coord4) + idx);
      if (inner) r.r = __ldg(a.rr + idx);
    }
  }
  return r;
}

template <int N, int ND>
__device__ __forceinline__ void issue_enc(EncIn<N, ND>& e, const RecIn& r, const __half* tpos,
                                          const __half* tdir, const __half* tdist, int R, int Rd) {
  constexpr int NP = EncIn<N, ND>::NP, NQ = EncIn<N, ND>::NQ;
  e.valid = r.valid;
  e.ray = r.ray;
  e.rec = r.rec;
  if (!r.valid) return;
  if constexpr (NP == 4 || NIF_CPACK8) {  // corner-packed entries: 32 B (NP 4) or 64 B (NP 8)
    const size_t g2 = (size_t)R * (R + 1) * NQ;  // uint4 per object table
    const BilQ bp = bilinear_q(r.c.x, r.c.y, R), bd = bilinear_q(r.c.z, r.c.w, R);
    const uint4* P = reinterpret_cast<const uint4*>(tpos) + (size_t)r.obj * g2 + (size_t)bp.q * NQ;
    const uint4* D = reinterpret_cast<const uint4*>(tdir) + (size_t)r.obj * g2 + (size_t)bd.q * NQ;
    ldg256(P, e.qp[0], e.qp[1]);
    ldg256(D, e.qd[0], e.qd[1]);
    if constexpr (NQ == 4) {
      ldg256(P + 2, e.qp[2], e.qp[3]);
      ldg256(D + 2, e.qd[2], e.qd[3]);
    }
    e.wp[0] = bp.w00; e.wp[1] = bp.w01; e.wp[2] = bp.w10; e.wp[3] = bp.w11;
    e.wd[0] = bd.w00; e.wd[1] = bd.w01; e.wd[2] = bd.w10; e.wd[3] = bd.w11;
  } else {  // one 16 B cell per corner
    const size_t g2 = (size_t)R * R;
    const Bil bp = bilinear(r.c.x, r.c.y, R), bd = bilinear(r.c.z, r.c.w, R);
    const uint4* P = reinterpret_cast<const uint4*>(tpos) + (size_t)r.obj * g2;
    const uint4* D = reinterpret_cast<const uint4*>(tdir) + (size_t)r.obj * g2;
    e.qp[0] = __ldg(P + (size_t)bp.iu0 * R + bp.iv0);
    e.qp[1] = __ldg(P + (size_t)bp.iu0 * R + bp.iv1);
    e.qp[2] = __ldg(P + (size_t)bp.iu1 * R + bp.iv0);
    e.qp[3] = __ldg(P + (size_t)bp.iu1 * R + bp.iv1);
    e.qd[0] = __ldg(D + (size_t)bd.iu0 * R + bd.iv0);
    e.qd[1] = __ldg(D + (size_t)bd.iu0 * R + bd.iv1);
    e.qd[2] = __ldg(D + (size_t)bd.iu1 * R + bd.iv0);
    e.qd[3] = __ldg(D + (size_t)bd.iu1 * R + bd.iv1);
    e.wp[0] = bp.w00; e.wp[1] = bp.w01; e.wp[2] = bp.w10; e.wp[3] = bp.w11;
    e.wd[0] = bd.w00; e.wd[1] = bd.w01; e.wd[2] = bd.w10; e.wd[3] = bd.w11;
  }
  if constexpr (ND > 0) {
    const float xc = r.r * (float)Rd - 0.5f;
    const float f0 = floorf(xc);
    const int jq = (int)fminf(fmaxf(f0 + 1.0f, 0.0f), (float)Rd);
    e.qr = __ldg(reinterpret_cast<const uint4*>(tdist) + (size_t)r.obj * (Rd + 1) + jq);
    e.wr = xc - f0;
  }
  (void)NP;
}

__device__ __forceinline__ unsigned long long f2pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2unpack(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// one corner's latent pair (fp16x2) times its fp32 weight, accumulated in
// fp32x2 with one FFMA2 (the same fp32 fma per element as two FFMAs)
__device__ __forceinline__ void acc_h2(uint32_t u, unsigned long long w2, unsigned long long& a) {
  const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&u));
  a = ffma2(f2pack(f.x, f.y), w2, a);
}

// corner c of a packed entry: NP=4 -> words (2c, 2c+1) of the entry's 8,
// NP=8 -> the four words of uint4 c; acc holds NP/2 packed latent pairs
template <int NP, int NQ>
__device__ __forceinline__ void acc_entry(const uint4 (&q)[NQ], const float (&w)[4],
                                          unsigned long long* acc) {
  if constexpr (NP == 4) {
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      const unsigned long long w0 = f2pack(w[2 * i], w[2 * i]);
      const unsigned long long w1 = f2pack(w[2 * i + 1], w[2 * i + 1]);
      acc_h2(q[i].x, w0, acc[0]);
      acc_h2(q[i].y, w0, acc[1]);
      acc_h2(q[i].z, w1, acc[0]);
      acc_h2(q[i].w, w1, acc[1]);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const unsigned long long wc = f2pack(w[c], w[c]);
      acc_h2(q[c].x, wc, acc[0]);
      acc_h2(q[c].y, wc, acc[1]);
      acc_h2(q[c].z, wc, acc[2]);
      acc_h2(q[c].w, wc, acc[3]);
    }
  }
}

#ifndef NIF_INTERP_FHFMA
// 1: interpolation with the mixed-precision FMA (f16 latent x f16 weight +
// f32 accumulator, one FHFMA per latent: no separate f16 -> f32 conversion
// and no work on the padding latents): C2 pass -1.3 us, but the bilinear
// weights rounded to f16 grow the logit error ~1.5x (1-epoch model: 0.0088
// vs 0.0066 max, 10-epoch |l| < 1: 0.009 vs 0.004); 0 (default): convert
// the latent pairs and interpolate with fp32 weights (FFMA2)
#define NIF_INTERP_FHFMA 0
#endif

// d = h(a) * h(b) + c with f16 operands taken from the low (L) / high (H)
// halves of two 32-bit registers; the f16 x f16 product is exact in fp32
#define NIF_FHFMA(NAME, AS, BS)                                                      \
  __device__ __forceinline__ float NAME(uint32_t a2, uint32_t b2, float c) {         \
    float d;                                                                         \
    asm("{.reg .f16 a0, a1, b0, b1;\n\t"                                            \
        "mov.b32 {a0, a1}, %1;\n\t"                                                  \
        "mov.b32 {b0, b1}, %2;\n\t"                                                  \
        "fma.rn.f32.f16 %0, " AS ", " BS ", %3;}"                                     \
        : "=f"(d) : "r"(a2), "r"(b2), "f"(c));                                      \
    return d;                                                                        \
  }
NIF_FHFMA(fhfma_ll, "a0", "b0")
NIF_FHFMA(fhfma_lh, "a0", "b1")
NIF_FHFMA(fhfma_hl, "a1", "b0")
NIF_FHFMA(fhfma_hh, "a1", "b1")
#undef NIF_FHFMA

// latent i (0..7) of a corner held in words (w0, w1, w2, w3), times the
// weight in half `wh` (0 low, 1 high) of the f16 pair `wp`, into acc
__device__ __forceinline__ float fh_latent(int i, uint32_t w0, uint32_t w1, uint32_t w2,
                                           uint32_t w3, uint32_t wp, int wh, float acc) {
  const uint32_t word = i < 2 ? w0 : i < 4 ? w1 : i < 6 ? w2 : w3;
  if (i & 1) return wh ? fhfma_hh(word, wp, acc) : fhfma_hl(word, wp, acc);
  return wh ? fhfma_lh(word, wp, acc) : fhfma_ll(word, wp, acc);
}

// the N real latents of one 2-D lookup (corner-packed entry; corner c's
// weight w[c] in f16), accumulated in fp32 over the corners in order
template <int N, int NP, int NQ>
__device__ __forceinline__ void fh_entry(const uint4 (&q)[NQ], const float (&w)[4],
                                         float (&acc)[8]) {
  const uint32_t wa = h2u(__floats2half2_rn(w[0], w[1]));
  const uint32_t wb = h2u(__floats2half2_rn(w[2], w[3]));
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t wp = c < 2 ? wa : wb;
    uint32_t w0, w1, w2 = 0u, w3 = 0u;
    if constexpr (NP == 4) {  // corner c: words (2c, 2c + 1) of the 8
      const uint4& u = q[c >> 1];
      w0 = (c & 1) ? u.z : u.x;
      w1 = (c & 1) ? u.w : u.y;
    } else {
      w0 = q[c].x;
      w1 = q[c].y;
      w2 = q[c].z;
      w3 = q[c].w;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = fh_latent(i, w0, w1, w2, w3, wp, c & 1, acc[i]);
  }
}

template <int N, int ND>
__device__ __forceinline__ void finish_enc(const EncIn<N, ND>& e, float (&x)[16]) {
  constexpr int NP = EncIn<N, ND>::NP, NQ = EncIn<N, ND>::NQ;
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = 0.f;
#if NIF_INTERP_FHFMA
  if (e.valid) {
    float ap[8], ad[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) ap[i] = ad[i] = 0.f;
    fh_entry<N, NP, NQ>(e.qp, e.wp, ap);
    fh_entry<N, NP, NQ>(e.qd, e.wd, ad);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      x[i] = ap[i];
      x[N + i] = ad[i];
    }
    if constexpr (ND > 0) {  // 1-D distance pair: corner 0 in words x, y; corner 1 in z, w
      const uint32_t wr = h2u(__floats2half2_rn(1.f - e.wr, e.wr));
#pragma unroll
      for (int i = 0; i < ND; ++i) {
        float a = fh_latent(i, e.qr.x, e.qr.y, 0u, 0u, wr, 0, 0.f);
        a = fh_latent(i, e.qr.z, e.qr.w, 0u, 0u, wr, 1, a);
        x[2 * N + i] = a;
      }
    }
  }
  x[2 * N + ND] = 1.f;
  return;
#endif
  if (e.valid) {
    unsigned long long ap[NP / 2], ad[NP / 2];
#pragma unroll
    for (int i = 0; i < NP / 2; ++i) ap[i] = ad[i] = 0ull;  // (+0, +0)
    acc_entry<NP, NQ>(e.qp, e.wp, ap);
    acc_entry<NP, NQ>(e.qd, e.wd, ad);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const float2 p2 = f2unpack(ap[i >> 1]), d2 = f2unpack(ad[i >> 1]);
      x[i] = (i & 1) ? p2.y : p2.x;
      x[N + i] = (i & 1) ? d2.y : d2.x;
    }
    if constexpr (ND > 0) {
      unsigned long long ar[2] = {0ull, 0ull};
      const unsigned long long w0 = f2pack(1.f - e.wr, 1.f - e.wr), w1 = f2pack(e.wr, e.wr);
      acc_h2(e.qr.x, w0, ar[0]);
      acc_h2(e.qr.y, w0, ar[1]);
      acc_h2(e.qr.z, w1, ar[0]);
      acc_h2(e.qr.w, w1, ar[1]);
#pragma unroll
      for (int i = 0; i < ND; ++i) {
        const float2 r2 = f2unpack(ar[i >> 1]);
        x[2 * N + i] = (i & 1) ? r2.y : r2.x;
      }
    }
  }
  x[2 * N + ND] = 1.f;
}

// kTpc tiles of 128 records per CTA advance in lockstep: one barrier, one
// batch of MMAs (one M=128 MMA chain per tile, issued back to back) and
// one commit per layer cover kTpc*128 rows. Each tile owns W TMEM columns;
// the N=16 head accumulates into the first 16 of them once the last hidden
// layer has been drained.

template <int N, int ND>
__global__ void __launch_bounds__(128 * kTpc) query_tc_kernel(TcArgs a) {
  constexpr bool INNER = ND > 0;
  constexpr int IN = 2 * N + ND;
  static_assert(IN + 1 <= 16, "layer-1 inputs plus bias must fit K = 16");
  extern __shared__ __align__(1024) uint8_t smem[];
  const FastLayout& l = a.l;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int tt = warp >> 2;             // tile of this warpgroup
  const int trow = tid & (kTileRows - 1);
  const int W = l.W, Kp = l.Kp, L = l.L;
  const size_t w_al = al16(l.w_bytes);
  const size_t a1_bytes = (size_t)kTileRows * kK1 * 2, a2_bytes = (size_t)kTileRows * Kp * 2;
  uint8_t* sW = smem;
  uint8_t* sA1 = smem + w_al + (size_t)tt * (a1_bytes + a2_bytes);
  uint8_t* sA2 = sA1 + a1_bytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + w_al + kTpc * (a1_bytes + a2_bytes));
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);

  const __half* tpos = reinterpret_cast<const __half*>(a.blob + l.off_pos);
  const __half* tdir = reinterpret_cast<const __half*>(a.blob + l.off_dir);
  const __half* tdist = reinterpret_cast<const __half*>(a.blob + l.off_dist);
  const int64_t n = min(*a.count, a.cap);
  const int64_t n_super = (n + kTpc * kTileRows - 1) / (kTpc * kTileRows);
  const int64_t stride = gridDim.x;
  auto tile_of = [&](int64_t sup) { return sup * kTpc + tt; };

  // prologue of the input pipeline (overlaps the setup below)
  EncIn<N, ND> ea;
  issue_enc<N, ND>(ea, load_rec(a, tile_of(blockIdx.x), trow, n, INNER), tpos, tdir, tdist, l.R,
                   l.Rd);
  RecIn rb = load_rec(a, tile_of(blockIdx.x + stride), trow, n, INNER);

  // weights -> smem (resident for the kernel's lifetime)
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.blob);
    uint4* dst = reinterpret_cast<uint4*>(sW);
    for (size_t i = tid; i < l.w_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  // constant tail of the activation tile: column W = 1 (bias), rest 0
  for (int c = W / 8; c < Kp / 8; ++c) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (c == W / 8) v.x = h2u(__halves2half2(__float2half_rn(1.f), __float2half_rn(0.f)));
    store_chunk(sA2, trow, c, Kp, v);
  }
  if (tid == 0) {
    tc::mbar_init(bar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc_dyn(tslot, l.tmem_cols);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = *tslot;
  const int Wc = (W + 31) / 32 * 32;  // TMEM column stride per tile
  const uint32_t my_acc = tbase + (uint32_t)(tt * Wc);
  const uint32_t lane_base = my_acc + ((uint32_t)((warp & 3) * 32) << 16);

  const uint32_t base_a = tc::smem_u32(smem + w_al), sWa = tc::smem_u32(sW);
  const uint32_t tile_stride = (uint32_t)(a1_bytes + a2_bytes);
  const uint64_t dW1 = tc::smem_desc(sWa + (uint32_t)l.off_w1, 128, kK1 * 16);
  const uint32_t idW = tc::idesc_f16(W), id16 = tc::idesc_f16(16);
  const __half2 slope2 = __float2half2_rn(kSlope);

  uint32_t phase = 0;
  int it = 0;
#define NIF_PROF(k)                                                      \
  if (a.prof != nullptr && tid == 0 && it < 4)                          \
    a.prof[((int64_t)blockIdx.x * 4 + it) * 16 + (k)] = clock64();
  for (int64_t sup = blockIdx.x; sup < n_super; sup += stride, ++it) {
    NIF_PROF(0);
    const int64_t row = tile_of(sup) * kTileRows + trow;
    const bool valid = ea.valid;
    const int my_ray = ea.ray;
    // ---- encode: 16 fp16 inputs (features, 1, zeros) ------------------------
    {
      float x[16];
      finish_enc<N, ND>(ea, x);
      uint4 v0, v1;
      v0.x = h2u(__floats2half2_rn(x[0], x[1]));
      v0.y = h2u(__floats2half2_rn(x[2], x[3]));
      v0.z = h2u(__floats2half2_rn(x[4], x[5]));
      v0.w = h2u(__floats2half2_rn(x[6], x[7]));
      v1.x = h2u(__floats2half2_rn(x[8], x[9]));
      v1.y = h2u(__floats2half2_rn(x[10], x[11]));
      v1.z = h2u(__floats2half2_rn(x[12], x[13]));
      v1.w = h2u(__floats2half2_rn(x[14], x[15]));
      store_chunk(sA1, trow, 0, kK1, v0);
      store_chunk(sA1, trow, 1, kK1, v1);
    }
    NIF_PROF(1);
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    NIF_PROF(2);
    if (tid == 0) {
      tc::fence_after_sync();
#pragma unroll
      for (int q = 0; q < kTpc; ++q)
        tc::mma_f16(tbase + q * Wc, tc::smem_desc(base_a + q * tile_stride, 128, kK1 * 16), dW1,
                    idW, 0);
      tc::mma_commit(bar);
    }
    // next tiles' inputs go in flight while this tile's MMA chain runs
    issue_enc<N, ND>(ea, rb, tpos, tdir, tdist, l.R, l.Rd);
    rb = load_rec(a, tile_of(sup + 2 * stride), trow, n, INNER);
    NIF_PROF(3);
    tc::mbar_spin(bar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    NIF_PROF(4);

    for (int layer = 1; layer <= L; ++layer) {
      // epilogue: TMEM accumulators -> leaky ReLU (fp16) -> next A tile
      for (int cc = 0; cc < W / 16; ++cc) {
        float v[16];
        tc::tmem_ld16(lane_base + cc * 16, v);
        uint32_t h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          __half2 q = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
          q = __hmax2(q, __hmul2(q, slope2));
          h[i] = h2u(q);
        }
        store_chunk(sA2, trow, 2 * cc, Kp, make_uint4(h[0], h[1], h[2], h[3]));
        store_chunk(sA2, trow, 2 * cc + 1, Kp, make_uint4(h[4], h[5], h[6], h[7]));
      }
      NIF_PROF(3 + 3 * layer);
      tc::fence_async_smem();
      tc::fence_before_sync();
      __syncthreads();
      NIF_PROF(4 + 3 * layer);
      if (tid == 0) {
        tc::fence_after_sync();
        const int steps = Kp / 16;
        const bool hid = layer < L;
        const uint32_t wb = hid ? sWa + (uint32_t)(l.off_hidden + (size_t)(layer - 1) * W * Kp * 2)
                                : sWa + (uint32_t)l.off_head;
        for (int q = 0; q < kTpc; ++q) {
          const uint32_t a2 = base_a + q * tile_stride + (uint32_t)a1_bytes;
          for (int s = 0; s < steps; ++s)
            tc::mma_f16(tbase + q * Wc, tc::smem_desc(a2 + s * 256, 128, Kp * 16),
                        tc::smem_desc(wb + s * 256, 128, Kp * 16), hid ? idW : id16, s > 0);
        }
        tc::mma_commit(bar);
      }
      tc::mbar_spin(bar, phase);
      phase ^= 1;
      tc::fence_after_sync();
      NIF_PROF(5 + 3 * layer);
    }
    const float logit = tc::tmem_ld1(lane_base);
    if (valid) {
      if (a.logits) a.logits[row] = logit;
      if (a.occ && logit < 0.f) a.occ[my_ray] = 1;
    }
    tc::fence_before_sync();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, l.tmem_cols);
}

__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
  uint32_t y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}


// Last hidden layer + N=1 head on the CUDA cores: logit = b + sum_k
// w_k * lrelu(z_k) with z read straight from TMEM (fp32 activations, fp32
// accumulation), which saves the head MMA round trip and its barrier.
template <int W, int CH = 32>
__device__ __forceinline__ float head_simt(uint32_t taddr, const float* __restrict__ hw) {
  unsigned long long acc = f2pack(hw[W], 0.f);
  const unsigned long long slope = f2pack(kSlope, kSlope);
#pragma unroll
  for (int g0 = 0; g0 < W; g0 += CH) {
    uint32_t r[CH];
    const int gw = (W - g0) < CH ? (W - g0) : CH;
    tc::tmem_ld16_nw(taddr + g0, r);
    if (CH > 16 && gw > 16) tc::tmem_ld16_nw(taddr + g0 + 16, r + (CH > 16 ? 16 : 0));
    tc::tmem_ld_fence<CH>(r);
#pragma unroll
    for (int c = 0; c < CH; c += 4) {
      if (c >= gw) break;
      const float4 w4 = *reinterpret_cast<const float4*>(hw + g0 + c);
      const unsigned long long z01 = f2pack(__uint_as_float(r[c]), __uint_as_float(r[c + 1]));
      const unsigned long long z23 = f2pack(__uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
      const float2 t01 = f2unpack(fmul2(z01, slope)), t23 = f2unpack(fmul2(z23, slope));
      const unsigned long long a01 =
          f2pack(fmaxf(__uint_as_float(r[c]), t01.x), fmaxf(__uint_as_float(r[c + 1]), t01.y));
      const unsigned long long a23 = f2pack(fmaxf(__uint_as_float(r[c + 2]), t23.x),
                                            fmaxf(__uint_as_float(r[c + 3]), t23.y));
      acc = ffma2(a01, f2pack(w4.x, w4.y), acc);
      acc = ffma2(a23, f2pack(w4.z, w4.w), acc);
    }
  }
  const float2 s = f2unpack(acc);
  return s.x + s.y;
}

// HD-output head (geometry: 4-wide identity head) from the same fp32
// accumulator columns: each activation chunk is loaded once and feeds all
// HD dot products. Rows at hw + j * W, biases at hw + HD * W; for HD = 1 the
// arithmetic (and its order) is head_simt's.
template <int W, int CH, int HD>
__device__ __forceinline__ void head_simt_n(uint32_t taddr, const float* __restrict__ hw,
                                            float (&out)[HD]) {
  // leaky(x) = A x + B |x| (A = (1 + slope) / 2, B = (1 - slope) / 2), so
  // w . leaky(z) = A (w . z) + B (w . |z|): one packed FFMA2 per pair for
  // the linear sum and one FFMA per element with the |.| operand modifier,
  // instead of the product, max and FFMA of max(z, slope z)
  unsigned long long lin[HD];
  float mag[HD], mag2[HD];  // two partial sums: shorter dependent chains
#pragma unroll
  for (int j = 0; j < HD; ++j) {
    lin[j] = 0ull;
    mag[j] = mag2[j] = 0.f;
  }
#pragma unroll
  for (int g0 = 0; g0 < W; g0 += CH) {
    uint32_t r[CH];
    const int gw = (W - g0) < CH ? (W - g0) : CH;
    tc::tmem_ld16_nw(taddr + g0, r);
    if (CH > 16 && gw > 16) tc::tmem_ld16_nw(taddr + g0 + 16, r + (CH > 16 ? 16 : 0));
    tc::tmem_ld_fence<CH>(r);
#pragma unroll
    for (int c = 0; c < CH; c += 4) {
      if (c >= gw) break;
      const float z0 = __uint_as_float(r[c]), z1 = __uint_as_float(r[c + 1]);
      const float z2 = __uint_as_float(r[c + 2]), z3 = __uint_as_float(r[c + 3]);
#pragma unroll
      for (int j = 0; j < HD; ++j) {
        const float4 w4 = *reinterpret_cast<const float4*>(hw + j * W + g0 + c);
        lin[j] = ffma2(f2pack(z0, z1), f2pack(w4.x, w4.y), lin[j]);
        lin[j] = ffma2(f2pack(z2, z3), f2pack(w4.z, w4.w), lin[j]);
        mag[j] = fmaf(fabsf(z0), w4.x, mag[j]);
        mag2[j] = fmaf(fabsf(z1), w4.y, mag2[j]);
        mag[j] = fmaf(fabsf(z2), w4.z, mag[j]);
        mag2[j] = fmaf(fabsf(z3), w4.w, mag2[j]);
      }
    }
  }
  constexpr float kA = 0.5f * (1.0f + kSlope), kB = 0.5f * (1.0f - kSlope);
#pragma unroll
  for (int j = 0; j < HD; ++j) {
    const float2 s = f2unpack(lin[j]);
    out[j] = fmaf(kB, mag[j] + mag2[j], fmaf(kA, s.x + s.y, hw[HD * W + j]));
  }
}

// ---------------------------------------------------------------------------
// Split path: standalone grid encoding -> tcgen05 MLP
//
// encode_tiles_kernel: one thread per record, fp16 latent corners gathered
// from the L2-resident tables, fp32 interpolation, 16 fp16 features per
// record (features, the constant-one bias column, zeros) written straight
// into 128-row tiles of the UMMA canonical K-major layout (4 KB per tile;
// each warp writes one contiguous 1 KB block).
// mlp_tiles_kernel: G independent 128-row tile pipelines per CTA; the
// layer-1 operand of each tile arrives by one 4 KB TMA bulk copy into a
// two-slot ring (issued a tile ahead by the MMA-issuing thread), so the MLP
// warps hold no gather state and run 8 tiles per SM in 64 registers.
// ---------------------------------------------------------------------------

constexpr int kFeatTileBytes = kTileRows * kK1 * 2;  // 4096


template <int N, int ND>
__device__ __forceinline__ RecIn load_rec_row(const int32_t* __restrict__ obj,
                                              const float* __restrict__ coord4,
                                              const float* __restrict__ rr, int64_t row,
                                              int64_t n) {
  RecIn r;
  r.valid = row < n;
  r.obj = 0;
  r.ray = 0;
  r.rec = (int)row;
  r.c = make_float4(0.f, 0.f, 0.f, 0.f);
  r.r = 0.f;
  if (r.valid) {
    r.obj = __ldg(obj + row);
    r.c = __ldg(reinterpret_cast<const float4*>(coord4) + row);
    if (ND > 0) r.r = __ldg(rr + row);
  }
  return r;
}

// feature row width in 16 B words: the layer-1 inputs plus the bias column
// in 8 fp16 (outer, 2N + 1 <= 8) -> one word, else two. The MLP kernel
// zero-fills the missing half of the K = 16 operand.
template <int N, int ND>
__host__ __device__ constexpr int feat_words() {
  return 2 * N + ND + 1 <= 8 ? 1 : 2;
}

template <int N, int ND>
__device__ __forceinline__ void store_feat(const EncIn<N, ND>& e, uint8_t* feat, int64_t row) {
  constexpr int FW = feat_words<N, ND>();
  float x[16];
  finish_enc<N, ND>(e, x);
  uint4 v0, v1;
  v0.x = h2u(__floats2half2_rn(x[0], x[1]));
  v0.y = h2u(__floats2half2_rn(x[2], x[3]));
  v0.z = h2u(__floats2half2_rn(x[4], x[5]));
  v0.w = h2u(__floats2half2_rn(x[6], x[7]));
  uint4* p = reinterpret_cast<uint4*>(feat) + FW * row;
  __stcg(p, v0);
  if constexpr (FW == 2) {
    v1.x = h2u(__floats2half2_rn(x[8], x[9]));
    v1.y = h2u(__floats2half2_rn(x[10], x[11]));
    v1.z = h2u(__floats2half2_rn(x[12], x[13]));
    v1.w = h2u(__floats2half2_rn(x[14], x[15]));
    __stcg(p + 1, v1);
  }
}

// Grid-stride over records, K records per thread per iteration and the
// next iteration's record words prefetched, so each thread keeps K
// corner-gather round trips and K record fetches in flight.
template <int N, int ND, int K>
__global__ void __launch_bounds__(256) encode_tiles_kernel(const uint8_t* __restrict__ blob,
                                                           FastLayout l,
                                                           const int32_t* __restrict__ obj,
                                                           const float* __restrict__ coord4,
                                                           const float* __restrict__ rr,
                                                           const int64_t* __restrict__ count,
                                                           int64_t cap, uint8_t* __restrict__ feat) {
  const int64_t n = min(*count, cap);
  const int64_t n_pad = (n + kTileRows - 1) / kTileRows * kTileRows;
  const __half* tpos = reinterpret_cast<const __half*>(blob + l.off_pos);
  const __half* tdir = reinterpret_cast<const __half*>(blob + l.off_dir);
  const __half* tdist = reinterpret_cast<const __half*>(blob + l.off_dist);
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  RecIn rq[K];
#pragma unroll
  for (int k = 0; k < K; ++k) rq[k] = load_rec_row<N, ND>(obj, coord4, rr, row + k * nt, n);
  for (; row < n_pad; row += K * nt) {
    EncIn<N, ND> e[K];
#pragma unroll
    for (int k = 0; k < K; ++k) issue_enc<N, ND>(e[k], rq[k], tpos, tdir, tdist, l.R, l.Rd);
#pragma unroll
    for (int k = 0; k < K; ++k)
      rq[k] = load_rec_row<N, ND>(obj, coord4, rr, row + (K + k) * nt, n);
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (row + k * nt < n_pad) store_feat<N, ND>(e[k], feat, row + k * nt);
  }
}

struct MlpArgs {
  const uint8_t* blob;  // fast blob (weights at offset 0)
  const uint8_t* feat;  // encoded features, fw x 16 B (8 fp16 each) per record
  int fw;               // 1 (outer shapes, 2N + 1 <= 8) or 2
  const int32_t* ray;
  const int64_t* count;
  int64_t cap;
  uint8_t* occ;
  float* logits;
  long long* prof;  // diagnostic phase stamps (nif_debug_set_prof), or NULL
};

// TMEM per tile: fp32 accumulator [0, W) and the fp16 A operand (two per
// column) [AOFF, AOFF + Kp/2). Keeping A in TMEM means the tensor core reads
// only the weights from shared memory: with N = 48-64 the A tile re-read
// per K step would otherwise make the MLP shared-memory-bandwidth bound.
template <int W, int L, int G, int HD = 1>
struct MlpCfg {
  static constexpr int Kp = ((W + 1) + 15) / 16 * 16;
  static constexpr int AOFF = (W + 15) / 16 * 16;
  static constexpr int STRIDE = (AOFF + Kp / 2 + 15) / 16 * 16;
  static constexpr int COLS_RAW = G * STRIDE;
  static constexpr int COLS = COLS_RAW <= 32 ? 32 : COLS_RAW <= 64 ? 64 : COLS_RAW <= 128 ? 128
                              : COLS_RAW <= 256 ? 256 : 512;
  static constexpr size_t OFF_HEADF =
      (size_t)W * kK1 * 2 + (size_t)(L - 1) * W * Kp * 2 + (size_t)16 * Kp * 2;
  static constexpr size_t W_BYTES = OFF_HEADF + ((size_t)HD * (W + 1) * 4 + 15) / 16 * 16;
  static constexpr size_t W_AL = (W_BYTES + 1023) / 1024 * 1024;
  static constexpr size_t SMEM = W_AL + 128;
  static_assert(W % 16 == 0 && L >= 2, "shape");
  static_assert(COLS_RAW <= 512, "TMEM");
  static_assert(Kp / 2 - W / 2 == 8, "one 8-column constant tail");
};

template <int W>
__device__ __forceinline__ void epilogue_act_tmem(uint32_t acc, uint32_t a_op, __half2 slope2) {
  // W fp32 accumulator columns -> leaky ReLU -> W/2 packed fp16 columns of A
#pragma unroll
  for (int g0 = 0; g0 < W; g0 += 32) {
    uint32_t r[32];
    const int gw = (W - g0) < 32 ? (W - g0) : 32;
    tc::tmem_ld16_nw(acc + g0, r);
    if (gw > 16) tc::tmem_ld16_nw(acc + g0 + 16, r + 16);
    tc::tmem_ld_fence<32>(r);
#pragma unroll
    for (int c = 0; c < 32; c += 16) {
      if (c >= gw) break;
      uint32_t h[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        __half2 q = __floats2half2_rn(__uint_as_float(r[c + 2 * i]), __uint_as_float(r[c + 2 * i + 1]));
        q = __hmax2(q, __hmul2(q, slope2));
        h[i] = h2u(q);
      }
      tc::tmem_st8(a_op + (g0 + c) / 2, h);
    }
  }
  tc::tmem_wait_st();
}

template <int W, int L, int G, int TPS>
__global__ void __launch_bounds__(128 * G, TPS / G) mlp_tiles_kernel(MlpArgs a) {
  using C = MlpCfg<W, L, G>;
  constexpr int Kp = C::Kp;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  const int wg = tid >> 7;
  const int trow = tid & (kTileRows - 1);
  const int quad = (tid >> 5) & 3;
  const bool leader = trow == 0;
  uint8_t* sW = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::W_AL);
  uint64_t* bar = bars + wg;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + G);

  const int64_t n = min(*a.count, a.cap);
  const int64_t n_tiles = (n + kTileRows - 1) / kTileRows;
  const int64_t stride = (int64_t)gridDim.x * G;
  const int64_t first = (int64_t)blockIdx.x * G + wg;

  if (tid == 0) {
    for (int g = 0; g < G; ++g) tc::mbar_init(bars + g, 1);
    tc::fence_barrier_init();
  }
  // the first tile's features are in flight while the weights are staged
  const uint4* F = reinterpret_cast<const uint4*>(a.feat);
  uint4 f0 = make_uint4(0, 0, 0, 0), f1 = f0;
  {
    const int64_t row = first * kTileRows + trow;
    if (first < n_tiles && row < n) {
      f0 = __ldg(F + a.fw * row);
      if (a.fw == 2) f1 = __ldg(F + 2 * row + 1);
    }
  }
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.blob);
    uint4* dst = reinterpret_cast<uint4*>(sW);
    for (int i = tid; i < (int)(C::W_BYTES / 16); i += blockDim.x) dst[i] = __ldg(src + i);
  }
  if (tid < 32) tc::tmem_alloc<C::COLS>(tslot);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
  const uint32_t acc = *tslot + (uint32_t)(wg * C::STRIDE);
  const uint32_t a_op = acc + C::AOFF;
  const uint32_t lane_acc = acc + lane_off, lane_a = a_op + lane_off;
  {  // constant tail of A: column K = W is the bias input (1), the rest 0
    uint32_t tail[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    tail[0] = h2u(__halves2half2(__float2half_rn(1.f), __float2half_rn(0.f)));
    tc::tmem_st8(lane_a + W / 2, tail);
  }
  const uint32_t sWa = tc::smem_u32(sW);
  constexpr uint32_t off_hidden = (uint32_t)W * kK1 * 2;
  const uint32_t idW = tc::idesc_f16(W);
  const __half2 slope2 = __float2half2_rn(kSlope);
  const uint32_t bar_id = 1 + wg;
  const float* headw = reinterpret_cast<const float*>(sW + C::OFF_HEADF);

  uint32_t phase = 0;
  int it = 0;
  long long* prof = a.prof;
#define MLP_PROF(k)                                                                       \
  if (prof != nullptr && trow == 0 && it < 4)                                             \
    prof[(((int64_t)blockIdx.x * G + wg) * 4 + it) * 16 + (k)] = clock64();
  if (prof != nullptr && trow == 0) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    prof[(((int64_t)blockIdx.x * G + wg) * 4) * 16 + 11] = (long long)gt;
  }
  for (int64_t t = first; t < n_tiles; t += stride, ++it) {
    MLP_PROF(0);
    const int64_t row = t * kTileRows + trow;
    const bool valid = row < n;
    {
      const uint32_t fv[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
      tc::tmem_st8(lane_a, fv);
    }
    const int my_ray = valid ? __ldg(a.ray + row) : 0;
    {  // next tile's features stream in under this tile's chain
      const int64_t nrow = row + stride * kTileRows;
      f0 = make_uint4(0, 0, 0, 0);
      f1 = f0;
      if (nrow < n) {
        f0 = __ldg(F + a.fw * nrow);
        if (a.fw == 2) f1 = __ldg(F + 2 * nrow + 1);
      }
    }
    tc::tmem_wait_st();
    tc::fence_before_sync();
    tc::named_sync(bar_id, 128);
    MLP_PROF(1);
    if (leader) {
      tc::fence_after_sync();
      tc::mma_f16_ts(acc, a_op, tc::smem_desc(opaque_u32(sWa), 128, kK1 * 16), idW, 0);
      tc::mma_commit(bar);
    }
    tc::mbar_wait_sleep(bar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    MLP_PROF(2);
#pragma unroll
    for (int layer = 1; layer < L; ++layer) {
      epilogue_act_tmem<W>(lane_acc, lane_a, slope2);
      tc::fence_before_sync();
      MLP_PROF(3 * layer);
      tc::named_sync(bar_id, 128);
      MLP_PROF(3 * layer + 1);
      if (leader) {
        tc::fence_after_sync();
        const uint32_t wb = opaque_u32(sWa + off_hidden + (uint32_t)((layer - 1) * W * Kp * 2));
#pragma unroll
        for (int s = 0; s < Kp / 16; ++s)
          tc::mma_f16_ts(acc, a_op + s * 8, tc::smem_desc(wb + s * 256, 128, Kp * 16), idW, s > 0);
        tc::mma_commit(bar);
      }
      tc::mbar_wait_sleep(bar, phase);
      phase ^= 1;
      tc::fence_after_sync();
      MLP_PROF(3 * layer + 2);
    }
    const float logit = head_simt<W>(lane_acc, headw);
    MLP_PROF(15);
    if (valid) {
      if (a.logits) a.logits[row] = logit;
      if (a.occ && logit < 0.f) a.occ[my_ray] = 1;
    }
    tc::fence_before_sync();
  }
  if (prof != nullptr && trow == 0) {  // whole-loop span and tile count of this warpgroup
    prof[(((int64_t)blockIdx.x * G + wg) * 4) * 16 + 13] = it;
    prof[(((int64_t)blockIdx.x * G + wg) * 4) * 16 + 14] = clock64();
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    prof[(((int64_t)blockIdx.x * G + wg) * 4) * 16 + 12] = (long long)gt;
  }
#undef MLP_PROF
  __syncthreads();
  if (tid < 32) tc::tmem_dealloc(*tslot, C::COLS);
}


// ---------------------------------------------------------------------------
// Fused query, A operand in TMEM (the production path for the default and
// C5 shapes): per 128-record tile one warpgroup gathers and interpolates the
// latent corners (issued a tile ahead, under the previous tile's last MMA),
// stores the 16 fp16 layer-1 inputs of its row straight into TMEM, and runs
// the MLP chain with A in TMEM and only the weights in shared memory; the
// last layer and the N=1 head run on the CUDA cores from the fp32
// accumulator. 6 (W=48) / 4 (W=64) tiles in flight per SM, bounded by TMEM.
// ---------------------------------------------------------------------------
// PO (per_object sharing): records arrive bucketed by object into 128-row
// tiles (nif_query_bucketed_dev); each warpgroup walks a contiguous range of
// tiles and keeps its own copy of the current object's weights, reloading
// it only when the object changes.
// EI: where the next tile's record loads and corner gathers are issued --
// 0 under the last hidden layer's MMA, k >= 1 under the k-th, -1 right after
// the first layer's MMA (the earliest; needs the registers of G = 1 CTAs)
template <int N, int ND, int W, int L, int G, int TPS, bool PO = false, int HD = 1, int EI = 0>
__global__ void __launch_bounds__(128 * G, TPS / G) query_ts_kernel(TcArgs a) {
  using C = MlpCfg<W, L, G, HD>;
  constexpr bool INNER = ND > 0;
  constexpr int Kp = C::Kp;
  extern __shared__ __align__(1024) uint8_t smem[];
  const FastLayout& l = a.l;
  const int tid = threadIdx.x;
  const int wg = tid >> 7;
  const int trow = tid & (kTileRows - 1);
  const int quad = (tid >> 5) & 3;
  const bool leader = trow == 0;
  uint8_t* sW = smem + (PO ? (size_t)wg * C::W_AL : 0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (PO ? G : 1) * C::W_AL);
  uint64_t* bar = bars + wg;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + G);

  const __half* tpos = reinterpret_cast<const __half*>(a.blob + l.off_pos);
  const __half* tdir = reinterpret_cast<const __half*>(a.blob + l.off_dir);
  const __half* tdist = reinterpret_cast<const __half*>(a.blob + l.off_dist);
  unsigned long long* tl =
      a.tl != nullptr && trow == 0 ? a.tl + ((int64_t)blockIdx.x * G + wg) * 5 : nullptr;
  if (tl) tl[0] = globaltimer();
  // prologue first (barriers, weights -> smem, TMEM): under programmatic
  // dependent launch it overlaps the tail of the gather that fills the queues
  if (tid == 0) {
    for (int g = 0; g < G; ++g) tc::mbar_init(bars + g, 1);
    tc::fence_barrier_init();
  }
  if constexpr (!PO) {
    const uint4* src = reinterpret_cast<const uint4*>(a.blob);
    uint4* dst = reinterpret_cast<uint4*>(sW);
    for (int i = tid; i < (int)(C::W_BYTES / 16); i += blockDim.x) dst[i] = __ldg(src + i);
  }
  if (tid < 32) tc::tmem_alloc<C::COLS>(tslot);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the queues are final from here
  if (tl) tl[1] = globaltimer();
  const int64_t n = min(*a.count, a.cap);
  int64_t n_tiles, stride, first;
  if constexpr (PO) {  // contiguous tile range per warpgroup (objects change rarely)
    const int64_t nt = *a.n_tiles;
    const int64_t gw = (int64_t)gridDim.x * G;
    const int64_t per = (nt + gw - 1) / gw;
    first = ((int64_t)blockIdx.x * G + wg) * per;
    n_tiles = min(first + per, nt);
    stride = 1;
  } else {
    n_tiles = (n + kTileRows - 1) / kTileRows;
    stride = (int64_t)gridDim.x * G;
    first = (int64_t)blockIdx.x * G + wg;
  }
  auto fetch = [&](int64_t t) {
    if constexpr (PO) return load_rec_perm(a, t, trow, n_tiles, INNER);
    else return load_rec(a, t, trow, n, INNER);
  };

  EncIn<N, ND> ea;
  issue_enc<N, ND>(ea, fetch(first), tpos, tdir, tdist, l.R, l.Rd);
  RecIn rb = fetch(first + stride);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
  const uint32_t acc = *tslot + (uint32_t)(wg * C::STRIDE);
  const uint32_t a_op = acc + C::AOFF;
  const uint32_t lane_acc = acc + lane_off, lane_a = a_op + lane_off;
  {
    uint32_t tail[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    tail[0] = h2u(__halves2half2(__float2half_rn(1.f), __float2half_rn(0.f)));
    tc::tmem_st8(lane_a + W / 2, tail);
  }
  const uint32_t sWa = tc::smem_u32(sW);
  constexpr uint32_t off_hidden = (uint32_t)W * kK1 * 2;
  const uint32_t idW = tc::idesc_f16(W);
  const __half2 slope2 = __float2half2_rn(kSlope);
  const uint32_t bar_id = 1 + wg;
  const float* headw = reinterpret_cast<const float*>(sW + C::OFF_HEADF);

  uint32_t phase = 0;
#if NIF_TS_PROF  // diagnostic phase stamps (tools/probe_phases.py; costs ~8 %)
  int it = 0;
  long long* prof = a.prof;
#define TS_PROF(k)                                                                     \
  if (prof != nullptr && trow == 0 && it < 8)                                          \
    prof[(((int64_t)blockIdx.x * G + wg) * 8 + it) * 16 + (k)] = clock64();
#define TS_PROF_NEXT() ++it
#else
#define TS_PROF(k)
#define TS_PROF_NEXT()
#endif
  int cur_obj = -1;
  for (int64_t t = first; t < n_tiles; t += stride) {
    TS_PROF(0);
    const int64_t row = ea.rec;
    const bool valid = ea.valid;
    const int my_ray = ea.ray;
    if constexpr (PO) {  // this tile's object MLP -> the warpgroup's weight buffer
      const int ot = __ldg(a.tile_obj + t);
      if (ot != cur_obj) {
        tc::named_sync(bar_id, 128);  // every thread is done with the previous head weights
        const uint4* src = reinterpret_cast<const uint4*>(a.blob + (size_t)ot * l.w_stride_blob);
        uint4* dst = reinterpret_cast<uint4*>(sW);
        for (int i = trow; i < (int)(C::W_BYTES / 16); i += kTileRows) dst[i] = __ldg(src + i);
        tc::fence_async_smem();
        cur_obj = ot;
      }
    }
    {
      float x[16];
      finish_enc<N, ND>(ea, x);
      uint32_t fv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) fv[i] = h2u(__floats2half2_rn(x[2 * i], x[2 * i + 1]));
      tc::tmem_st8(lane_a, fv);
    }
    tc::tmem_wait_st();
    TS_PROF(1);
    tc::fence_before_sync();
    tc::named_sync(bar_id, 128);
    TS_PROF(2);
    if (leader) {
      tc::fence_after_sync();
      tc::mma_f16_ts(acc, a_op, tc::smem_desc(opaque_u32(sWa), 128, kK1 * 16), idW, 0);
      tc::mma_commit(bar);
    }
    if constexpr (EI < 0) {  // next tile's gathers in flight under the whole MLP chain
      issue_enc<N, ND>(ea, rb, tpos, tdir, tdist, l.R, l.Rd);
      rb = fetch(t + 2 * stride);
    }
    tc::mbar_wait_sleep(bar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    TS_PROF(3);
#pragma unroll
    for (int layer = 1; layer < L; ++layer) {
      epilogue_act_tmem<W>(lane_acc, lane_a, slope2);
      TS_PROF(1 + 3 * layer);
      tc::fence_before_sync();
      tc::named_sync(bar_id, 128);
      TS_PROF(2 + 3 * layer);
      if (leader) {
        tc::fence_after_sync();
        const uint32_t wb = opaque_u32(sWa + off_hidden + (uint32_t)((layer - 1) * W * Kp * 2));
#pragma unroll
        for (int s = 0; s < Kp / 16; ++s)
          tc::mma_f16_ts(acc, a_op + s * 8, tc::smem_desc(wb + s * 256, 128, Kp * 16), idW, s > 0);
        tc::mma_commit(bar);
      }
      if (EI >= 0 && layer == (EI > 0 && EI < L ? EI : L - 1)) {
        // next tile's gathers in flight under the remaining MMAs + head
        issue_enc<N, ND>(ea, rb, tpos, tdir, tdist, l.R, l.Rd);
        rb = fetch(t + 2 * stride);
      }
      tc::mbar_wait_sleep(bar, phase);
      phase ^= 1;
      tc::fence_after_sync();
      TS_PROF(3 + 3 * layer);
    }
    float hout[HD];
    head_simt_n<W, 16, HD>(lane_acc, headw, hout);
    if (valid) {
      if constexpr (HD == 1) {
        if (a.logits) a.logits[row] = hout[0];
        if (a.occ && hout[0] < 0.f) a.occ[my_ray] = 1;
      } else if (a.logits) {  // geometry head: raw (normal, depth) outputs
#pragma unroll
        for (int j = 0; j < HD; ++j) a.logits[row * HD + j] = hout[j];
      }
    }
    tc::fence_before_sync();
    TS_PROF(15);
    TS_PROF_NEXT();
    if (tl && t == first) tl[2] = globaltimer();
  }
#undef TS_PROF
#undef TS_PROF_NEXT
  if (tl) {
    tl[3] = globaltimer();
    tl[4] = (unsigned long long)(n_tiles > first ? (n_tiles - first + stride - 1) / stride : 0);
  }
  __syncthreads();
  if (tid < 32) tc::tmem_dealloc(*tslot, C::COLS);
}

template <int N, int ND, int W, int L, int G, int TPS, bool PO = false, int HD = 1, int EI = 0>
int launch_ts(const TcArgs& a, cudaStream_t st) {
  using C = MlpCfg<W, L, G, HD>;
  auto kern = query_ts_kernel<N, ND, W, L, G, TPS, PO, HD, EI>;
  const size_t smem = C::SMEM + (PO ? (size_t)(G - 1) * C::W_AL : 0);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return check_launch("query_ts: smem attribute");
  const int per_sm_tmem = 512 / C::COLS;
  int per_sm = per_sm_tmem < TPS / G ? per_sm_tmem : TPS / G;
  if (g_query_cpsm > 0 && per_sm > g_query_cpsm) per_sm = g_query_cpsm;
  if (per_sm < 1) per_sm = 1;
  const int64_t max_tiles = (a.cap + kTileRows - 1) / kTileRows;
  int64_t grid = (int64_t)sm_count() * per_sm;
  const int64_t need = (max_tiles + G - 1) / G;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  // programmatic dependent launch behind the gather (see query_ts_kernel)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(128 * G);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a);
  return check_launch("nif_query_dev(tcgen05 TS)");
}

// per_object sharing (bucketed tiles): default shapes; 0 = launched
int launch_ts_po(const TcArgs& a, const nif_family_view& f, cudaStream_t st, int* rc) {
  const int W = a.l.W, L = a.l.L;
  if (a.l.HD != 1) return 1;
  if (f.family == NIF_FAMILY_OUTER && f.N == 3 && W == 64 && L == 2) {
    *rc = launch_ts<3, 0, 64, 2, 2, 4, true>(a, st);
    return 0;
  }
  if (f.family == NIF_FAMILY_INNER && f.N == 5 && f.Nd == 3 && W == 48 && L == 3) {
    *rc = launch_ts<5, 3, 48, 3, 1, 4, true, 1, 1>(a, st);
    return 0;
  }
  return 1;
}

// 0 = launched, 1 = no specialisation
int launch_ts_any(const TcArgs& a, const nif_family_view& f, cudaStream_t st, int* rc) {
  const int W = a.l.W, L = a.l.L;
  if (a.l.HD == 4) {  // geometry head (infer_geometry), default shapes
    if (f.family == NIF_FAMILY_OUTER && f.N == 3 && W == 64 && L == 2) {
      *rc = launch_ts<3, 0, 64, 2, 2, 4, false, 4>(a, st);
      return 0;
    }
    if (f.family == NIF_FAMILY_INNER && f.N == 5 && f.Nd == 3 && W == 48 && L == 3) {
      *rc = launch_ts<5, 3, 48, 3, 1, 4, false, 4, 1>(a, st);
      return 0;
    }
    return 1;
  }
#define NIF_TS(NN, NDD, WW, LL, GG, TT)                                        \
  if (f.N == NN && (NDD == 0 ? f.family == NIF_FAMILY_OUTER                    \
                             : (f.family == NIF_FAMILY_INNER && f.Nd == NDD)) && \
      W == WW && L == LL) {                                                    \
    *rc = launch_ts<NN, NDD, WW, LL, GG, TT>(a, st);                           \
    return 0;                                                                  \
  }
  if (g_query_variant == 11) {
    NIF_TS(3, 0, 64, 2, 1, 4)
    NIF_TS(5, 3, 48, 3, 1, 6)
  }
  if (g_query_variant == 12) {  // round-1 inner configuration: 2 CTAs x 3 warpgroups per SM
    NIF_TS(5, 3, 48, 3, 3, 6)
  }
  NIF_TS(3, 0, 64, 2, 2, 4)
  // inner default: one warpgroup per CTA, 4 CTAs per SM (TMEM: 80 columns
  // per tile, allocated as 128), 128 registers per thread -- no spills --
  // and the next tile's gathers issued under the first hidden layer's MMA.
  // C2: 51.9 us vs 57.1 us for 2 CTAs x 3 warpgroups (6 tiles per SM at the
  // 80-register cap, spilling; variant 12)
  if (f.N == 5 && f.family == NIF_FAMILY_INNER && f.Nd == 3 && W == 48 && L == 3) {
    *rc = launch_ts<5, 3, 48, 3, 1, 4, false, 1, 1>(a, st);
    return 0;
  }
  // C5 sweep shapes (TMEM: W=48 -> 80 columns per tile, 64 -> 112, 128 -> 208)
  NIF_TS(3, 0, 64, 3, 2, 4)
  NIF_TS(3, 0, 64, 4, 2, 4)
  NIF_TS(3, 0, 128, 2, 1, 2)
  NIF_TS(3, 0, 128, 3, 1, 2)
  NIF_TS(3, 0, 128, 4, 1, 2)
  NIF_TS(5, 3, 48, 2, 3, 6)
  NIF_TS(5, 3, 48, 4, 3, 6)
  NIF_TS(5, 3, 64, 2, 2, 4)
  NIF_TS(5, 3, 64, 3, 2, 4)
  NIF_TS(5, 3, 64, 4, 2, 4)
  NIF_TS(5, 3, 128, 2, 1, 2)
  NIF_TS(5, 3, 128, 3, 1, 2)
  NIF_TS(5, 3, 128, 4, 1, 2)
#undef NIF_TS
  return 1;
}

template <int N, int ND>
int launch_encode_tiles(const uint8_t* blob, const FastLayout& l, const int32_t* obj,
                        const float* coord4, const float* r, const int64_t* count, int64_t cap,
                        uint8_t* feat, cudaStream_t st) {
  const int64_t rows = (cap + kTileRows - 1) / kTileRows * kTileRows;
  int64_t blocks = (rows + 255) / 256;
  const int64_t max_blocks = (int64_t)sm_count() * 8;  // grid-stride: the count lives on the device
  if (blocks > max_blocks) blocks = max_blocks;
  // two records in flight per thread (1: same speed, 4: slower -- C5 sweep)
  encode_tiles_kernel<N, ND, 2><<<(unsigned)blocks, 256, 0, st>>>(blob, l, obj, coord4, r, count,
                                                                  cap, feat);
  return check_launch("nif_encode_tiles");
}

template <int W, int L, int G, int TPS>
int launch_mlp_tiles(const MlpArgs& a, cudaStream_t st) {
  using C = MlpCfg<W, L, G>;
  auto kern = mlp_tiles_kernel<W, L, G, TPS>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) !=
      cudaSuccess)
    return check_launch("mlp_tiles: smem attribute");
  const int per_sm_tmem = 512 / C::COLS;
  const int per_sm_smem = (int)((228 * 1024) / (C::SMEM + 1024));
  int per_sm = per_sm_tmem < per_sm_smem ? per_sm_tmem : per_sm_smem;
  if (per_sm > TPS / G) per_sm = TPS / G;
  if (per_sm < 1) per_sm = 1;
  const int64_t max_tiles = (a.cap + kTileRows - 1) / kTileRows;
  int64_t grid = (int64_t)sm_count() * per_sm;
  const int64_t need = (max_tiles + G - 1) / G;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, 128 * G, C::SMEM, st>>>(a);
  return check_launch("nif_mlp_tiles");
}

bool mlp_shape_ok(int W, int L) {
  return ((W == 48 || W == 64) && L >= 2 && L <= 4) || (W == 128 && L >= 2 && L <= 4);
}

// 0 = launched, 1 = no specialisation for this shape
int launch_split(const nif_family_view& f, const FastLayout& l, const int32_t* obj,
                 const int32_t* ray, const float* coord4, const float* r, const int64_t* count,
                 int64_t cap, uint8_t* occ, float* logits, uint8_t* feat, int flags,
                 cudaStream_t st, int* rc) {
  const bool outer = f.family == NIF_FAMILY_OUTER;
  if (!mlp_shape_ok(l.W, l.L)) return 1;
  int erc = NIF_OK;
  const uint8_t* blob = (const uint8_t*)f.fast;
  const bool enc_only = (flags & 2) != 0, mlp_only = (flags & 4) != 0;
  if (mlp_only) goto mlp;
  if (outer && f.N == 3) erc = launch_encode_tiles<3, 0>(blob, l, obj, coord4, r, count, cap, feat, st);
  else if (!outer && f.N == 5 && f.Nd == 3)
    erc = launch_encode_tiles<5, 3>(blob, l, obj, coord4, r, count, cap, feat, st);
  else if (outer && f.N == 2) erc = launch_encode_tiles<2, 0>(blob, l, obj, coord4, r, count, cap, feat, st);
  else if (outer && f.N == 4) erc = launch_encode_tiles<4, 0>(blob, l, obj, coord4, r, count, cap, feat, st);
  else if (!outer && f.N == 4 && f.Nd == 3)
    erc = launch_encode_tiles<4, 3>(blob, l, obj, coord4, r, count, cap, feat, st);
  else if (!outer && f.N == 5 && f.Nd == 4)
    erc = launch_encode_tiles<5, 4>(blob, l, obj, coord4, r, count, cap, feat, st);
  else return 1;
  if (erc != NIF_OK || enc_only) {
    *rc = erc;
    return 0;
  }
mlp:
  const int in1 = 2 * f.N + (outer ? 0 : f.Nd) + 1;  // layer-1 inputs + bias (feat_words)
  MlpArgs m{blob, feat, in1 <= 8 ? 1 : 2, ray, count, cap, occ, logits, g_prof};
#define NIF_MLP(WW, LL, GG, TT)                                              \
  if (l.W == WW && l.L == LL) {                                              \
    *rc = launch_mlp_tiles<WW, LL, GG, TT>(m, st);                           \
    return 0;                                                                \
  }
  // tiles per SM bounded by TMEM: W=48 -> 80 columns/tile, W=64 -> 112,
  // W=128 -> 208
  NIF_MLP(64, 2, 2, 4)
  NIF_MLP(48, 3, 3, 6)
  NIF_MLP(64, 3, 2, 4)
  NIF_MLP(64, 4, 2, 4)
  NIF_MLP(48, 2, 3, 6)
  NIF_MLP(48, 4, 3, 6)
  NIF_MLP(128, 2, 1, 2)
  NIF_MLP(128, 3, 1, 2)
  NIF_MLP(128, 4, 1, 2)
#undef NIF_MLP
  return 1;
}

__global__ void occ_init_kernel(const uint8_t* __restrict__ src, int64_t n,
                                uint8_t* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src ? src[i] : 0;
}

size_t tc_smem_bytes(const FastLayout& l) {
  return al16(l.w_bytes) + kTpc * ((size_t)kTileRows * kK1 * 2 + (size_t)kTileRows * l.Kp * 2) +
         64;
}

template <int N, int ND>
int launch_tc(const TcArgs& a, cudaStream_t st) {
  const size_t smem = tc_smem_bytes(a.l);
  auto kern = query_tc_kernel<N, ND>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return check_launch("query_tc: smem attribute");
  const int per_sm_tmem = 512 / a.l.tmem_cols;
  const int per_sm_smem = (int)((227 * 1024) / (smem + 1024));
  int per_sm = per_sm_tmem < per_sm_smem ? per_sm_tmem : per_sm_smem;
  if (per_sm > 8) per_sm = 8;
  if (per_sm < 1) per_sm = 1;
  const int64_t max_super = (a.cap + kTpc * kTileRows - 1) / (kTpc * kTileRows);
  int64_t grid = (int64_t)sm_count() * per_sm;
  if (grid > max_super) grid = max_super;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, 128 * kTpc, smem, st>>>(a);
  return check_launch("nif_query_dev(tcgen05)");
}


// ---------------------------------------------------------------------------
// Bucketing by object (per_object sharing): counting sort of a record queue
// into per-object segments padded to whole 128-row tiles, so every tile of
// the tensor-core kernel runs one object's MLP. Order inside a segment is
// arbitrary (the pass only ORs per ray).
//   scratch: hist i32[n_obj] | cursor i32[n_obj] | tile_off i64[n_obj + 1] |
//            n_tiles i64 | tile_obj i32[max_tiles] | perm i32[max_tiles*128]
// ---------------------------------------------------------------------------
struct BucketWs {
  int32_t* hist;
  int32_t* cursor;
  int64_t* tile_off;
  int64_t* n_tiles;
  int32_t* tile_obj;
  int32_t* perm;
  int64_t max_tiles;
};

__host__ __device__ inline int64_t bucket_max_tiles(int64_t capacity, int n_obj) {
  return (capacity + kTileRows - 1) / kTileRows + n_obj;
}

inline BucketWs bucket_ws(void* scratch, int64_t capacity, int n_obj) {
  BucketWs w;
  uint8_t* p = (uint8_t*)scratch;
  const size_t o4 = ((size_t)n_obj * 4 + 255) / 256 * 256;
  w.hist = (int32_t*)p;
  w.cursor = (int32_t*)(p + o4);
  w.tile_off = (int64_t*)(p + 2 * o4);
  const size_t o8 = ((size_t)(n_obj + 1) * 8 + 255) / 256 * 256;
  w.n_tiles = (int64_t*)(p + 2 * o4 + o8);
  w.max_tiles = bucket_max_tiles(capacity, n_obj);
  w.tile_obj = (int32_t*)(p + 2 * o4 + o8 + 256);
  const size_t ot = ((size_t)w.max_tiles * 4 + 255) / 256 * 256;
  w.perm = (int32_t*)(p + 2 * o4 + o8 + 256 + ot);
  return w;
}

// tile offsets (exclusive scan of padded counts), tile -> object, and the
// -1 padding rows of each object's last tile; run by one block
__device__ void bucket_scan_block(const BucketWs& w, int n_obj) {
  if (n_obj <= 32) {  // one warp: lane o scans object o (no serial chain)
    if (threadIdx.x < 32) {
      const int o = threadIdx.x;
      const int64_t tiles = o < n_obj ? (__ldcg(w.hist + o) + kTileRows - 1) / kTileRows : 0;
      int64_t incl = tiles;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int64_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (o >= d) incl += v;
      }
      if (o < n_obj) {
        w.tile_off[o] = incl - tiles;
        w.cursor[o] = 0;
      }
      if (o == n_obj - 1) {
        w.tile_off[n_obj] = incl;
        *w.n_tiles = incl;
      }
    }
  } else if (threadIdx.x == 0) {
    int64_t off = 0;
    for (int o = 0; o < n_obj; ++o) {
      w.tile_off[o] = off;
      off += (__ldcg(w.hist + o) + kTileRows - 1) / kTileRows;
      w.cursor[o] = 0;
    }
    w.tile_off[n_obj] = off;
    *w.n_tiles = off;
  }
  __syncthreads();
  for (int o = 0; o < n_obj; ++o) {
    const int64_t t0 = w.tile_off[o], t1 = w.tile_off[o + 1];
    for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) w.tile_obj[t] = o;
    // every other slot of the used tiles is written by the scatter
    for (int64_t p = t0 * kTileRows + __ldcg(w.hist + o) + threadIdx.x; p < t1 * kTileRows;
         p += blockDim.x)
      w.perm[p] = -1;
  }
  __syncthreads();
  // the histogram is consumed: re-zero it for the next call (no memset
  // node in front of the histogram kernel; the scratch starts zero-filled)
  for (int o = threadIdx.x; o < n_obj; o += blockDim.x) w.hist[o] = 0;
}

__global__ void bucket_hist_kernel(const int32_t* __restrict__ obj,
                                   const int64_t* __restrict__ count, int64_t cap, int n_obj,
                                   int32_t* __restrict__ hist) {
  extern __shared__ int32_t sh[];
  for (int o = threadIdx.x; o < n_obj; o += blockDim.x) sh[o] = 0;
  __syncthreads();
  const int64_t n = min(*count, cap);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(sh + __ldg(obj + i), 1);
  __syncthreads();
  for (int o = threadIdx.x; o < n_obj; o += blockDim.x)
    if (sh[o]) atomicAdd(hist + o, sh[o]);
}

// one block (a separate launch measured faster than a last-block scan
// folded into the histogram kernel)
__global__ void bucket_scan_kernel(BucketWs w, int n_obj) { bucket_scan_block(w, n_obj); }

__global__ void bucket_scatter_kernel(const int32_t* __restrict__ obj,
                                      const int64_t* __restrict__ count, int64_t cap,
                                      BucketWs w) {
  const int64_t n = min(*count, cap);
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const bool v = i < n;
    const int o = v ? __ldg(obj + i) : -1;
    // warp-aggregated reservation: one atomic per distinct object per warp
    const unsigned peers = __match_any_sync(0xffffffffu, o);
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (v && lane == leader) base = atomicAdd(w.cursor + o, __popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (v) {
      const int rank = __popc(peers & ((1u << lane) - 1u));
      w.perm[w.tile_off[o] * kTileRows + base + rank] = (int32_t)i;
    }
  }
}

// Block-aggregated scatter: a block takes a chunk of kBucketChunk records,
// counts them per object in shared memory, reserves each object's range
// with one global atomic per (chunk, object) -- not one per (warp, object):
// a dozen objects made the per-warp reservations serialise on a dozen
// addresses -- and places each record at its reserved base plus a
// shared-memory rank. Order within a bucket is irrelevant (per-record
// logits, OR per ray).
constexpr int kBucketChunk = 1024;

__device__ __forceinline__ int warp_agg_add(int* ctr, int o, bool v) {
  const int lane = threadIdx.x & 31;
  const unsigned peers = __match_any_sync(0xffffffffu, v ? o : -1);
  const int leader = __ffs(peers) - 1;
  int base = 0;
  if (v && lane == leader) base = atomicAdd(ctr + o, __popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  return base + __popc(peers & ((1u << lane) - 1u));
}

__global__ void __launch_bounds__(256) bucket_scatter_block_kernel(
    const int32_t* __restrict__ obj, const int64_t* __restrict__ count, int64_t cap, BucketWs w,
    int n_obj) {
  extern __shared__ int sm_b[];
  int* s_cnt = sm_b;              // [n_obj] records per object in this chunk
  int* s_base = sm_b + n_obj;     // [n_obj] reserved base in the object's bucket
  int* s_rank = sm_b + 2 * n_obj;  // [n_obj] placement counters
  const int64_t n = min(*count, cap);
  for (int64_t c0 = (int64_t)blockIdx.x * kBucketChunk; c0 < n;
       c0 += (int64_t)gridDim.x * kBucketChunk) {
    const int64_t c1 = min(c0 + (int64_t)kBucketChunk, n);
    for (int o = threadIdx.x; o < n_obj; o += blockDim.x) s_cnt[o] = s_rank[o] = 0;
    __syncthreads();
    for (int64_t b = c0; b < c1; b += blockDim.x) {
      const int64_t i = b + threadIdx.x;
      const bool v = i < c1;
      warp_agg_add(s_cnt, v ? __ldg(obj + i) : 0, v);
    }
    __syncthreads();
    for (int o = threadIdx.x; o < n_obj; o += blockDim.x)
      if (s_cnt[o]) s_base[o] = atomicAdd(w.cursor + o, s_cnt[o]);
    __syncthreads();
    for (int64_t b = c0; b < c1; b += blockDim.x) {
      const int64_t i = b + threadIdx.x;
      const bool v = i < c1;
      const int o = v ? __ldg(obj + i) : 0;
      const int r = warp_agg_add(s_rank, o, v);
      if (v) w.perm[w.tile_off[o] * kTileRows + s_base[o] + r] = (int32_t)i;
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace nif

using namespace nif;

extern "C" size_t nif_fast_pack_bytes(const nif_family_view* f) {
  return make_layout(*f).total;
}

extern "C" int nif_fast_pack_dev(const nif_family_view* f, void* blob, void* stream) {
  const FastLayout l = make_layout(*f);
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(blob, 0, l.total, st);
  if (l.tc_ok) {
    const int nw = l.W * kK1 + (l.L - 1) * l.W * l.Kp + 16 * l.Kp + l.HD * (l.W + 1);
    pack_weights_kernel<<<dim3((nw + 255) / 256, f->n_heads), 256, 0, st>>>(*f, l,
                                                                            (uint8_t*)blob);
  }
  const int64_t cells = 2 * ((l.NP == 4 || NIF_CPACK8) ? (int64_t)l.n_obj * l.R * (l.R + 1) * 4
                                      : (int64_t)l.n_obj * l.R * l.R) +
                        (f->family == NIF_FAMILY_INNER ? (int64_t)l.n_obj * (l.Rd + 1) * 2 : 0);
  pack_tables_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, st>>>(*f, l, (uint8_t*)blob);
  return check_launch("nif_fast_pack_dev");
}

extern "C" int nif_query_dev(const nif_family_view* f, const int32_t* obj, const int32_t* ray,
                             const float* coord4, const float* r, const int64_t* count_dev,
                             int64_t capacity, uint8_t* occ_ray, float* logits, int32_t impl,
                             void* stream) {
  if (capacity <= 0) return NIF_OK;
  if (f->family == NIF_FAMILY_INNER && r == nullptr)
    return fail(NIF_ERR_VALUE, "inner queries need the radial coordinate");
  cudaStream_t st = (cudaStream_t)stream;
  const FastLayout l = make_layout(*f);
  // one MLP per object needs the bucketed records of nif_query_bucketed_dev
  // to run on the tensor cores; unbucketed it runs on the SIMT kernel
  const bool shared_mlp = f->n_heads == 1;
  if (!shared_mlp && (impl == NIF_IMPL_TCGEN05 || impl == NIF_IMPL_TCGEN05_GENERIC))
    return fail(NIF_ERR_UNSUPPORTED, "per-object MLPs on tensor cores need nif_query_bucketed_dev");
  const bool want_tc = impl == NIF_IMPL_TCGEN05 || impl == NIF_IMPL_TCGEN05_GENERIC ||
                       (impl == NIF_IMPL_AUTO && l.tc_ok && shared_mlp && f->fast);
  if (want_tc) {
    if (!l.tc_ok)
      return fail(NIF_ERR_UNSUPPORTED, "configuration not covered by the tcgen05 kernel");
    if (!f->fast) return fail(NIF_ERR_VALUE, "tcgen05 path needs nif_fast_pack_dev first");
    TcArgs a{(const uint8_t*)f->fast, l, obj, ray, coord4, r, count_dev, capacity, occ_ray,
             logits, g_prof};
    a.tl = g_tl_query;
    if (l.HD != 1) {  // geometry head: the TMEM-operand kernel only
      int rc = NIF_OK;
      if (launch_ts_any(a, *f, st, &rc) == 0) return rc;
      if (impl != NIF_IMPL_AUTO)
        return fail(NIF_ERR_UNSUPPORTED, "no tcgen05 geometry-head kernel for W=%d L=%d", l.W, l.L);
      goto simt;
    }
    if (impl != NIF_IMPL_TCGEN05_GENERIC && (g_prof == nullptr || NIF_TS_PROF) &&
        g_query_variant != 2) {
      int rc = NIF_OK;
      if (launch_ts_any(a, *f, st, &rc) == 0) return rc;
    }
    if (f->family == NIF_FAMILY_OUTER && f->N == 3) return launch_tc<3, 0>(a, st);
    if (f->family == NIF_FAMILY_INNER && f->N == 5 && f->Nd == 3) return launch_tc<5, 3>(a, st);
    if (f->family == NIF_FAMILY_OUTER && f->N == 2) return launch_tc<2, 0>(a, st);
    if (f->family == NIF_FAMILY_OUTER && f->N == 4) return launch_tc<4, 0>(a, st);
    if (f->family == NIF_FAMILY_INNER && f->N == 4 && f->Nd == 3) return launch_tc<4, 3>(a, st);
    if (f->family == NIF_FAMILY_INNER && f->N == 5 && f->Nd == 4) return launch_tc<5, 4>(a, st);
    return fail(NIF_ERR_UNSUPPORTED, "no tcgen05 instantiation for N=%d Nd=%d", f->N, f->Nd);
  }
simt:
  if (f->dims[0] > kSimtMaxIn) return fail(NIF_ERR_UNSUPPORTED, "input width above %d", kSimtMaxIn);
  for (int i = 1; i <= f->n_layers; ++i)
    if (f->dims[i] > kSimtMaxW) return fail(NIF_ERR_UNSUPPORTED, "width above %d", kSimtMaxW);
  int64_t blocks = (capacity + 127) / 128;
  const int64_t max_blocks = (int64_t)sm_count() * 16;
  if (blocks > max_blocks) blocks = max_blocks;
  query_simt_kernel<<<(unsigned)blocks, 128, 0, st>>>(*f, obj, ray, coord4, r, count_dev,
                                                      capacity, occ_ray, logits);
  return check_launch("nif_query_dev(simt)");
}


extern "C" size_t nif_bucket_scratch_bytes(int64_t capacity, int32_t n_obj) {
  const int64_t mt = bucket_max_tiles(capacity, n_obj);
  const size_t o4 = ((size_t)n_obj * 4 + 255) / 256 * 256;
  const size_t o8 = ((size_t)(n_obj + 1) * 8 + 255) / 256 * 256;
  const size_t ot = ((size_t)mt * 4 + 255) / 256 * 256;
  return 2 * o4 + o8 + 256 + ot + (size_t)mt * kTileRows * 4;
}

extern "C" int nif_query_bucketed_dev(const nif_family_view* f, const int32_t* obj,
                                      const int32_t* ray, const float* coord4, const float* r,
                                      const int64_t* count_dev, int64_t capacity,
                                      uint8_t* occ_ray, float* logits, void* scratch,
                                      void* stream) {
  if (capacity <= 0) return NIF_OK;
  if (f->family == NIF_FAMILY_INNER && r == nullptr)
    return fail(NIF_ERR_VALUE, "inner queries need the radial coordinate");
  if (scratch == nullptr) return fail(NIF_ERR_VALUE, "bucketed query needs a scratch buffer");
  const FastLayout l = make_layout(*f);
  if (!l.tc_ok) return fail(NIF_ERR_UNSUPPORTED, "configuration not covered by the tcgen05 kernels");
  if (!f->fast) return fail(NIF_ERR_VALUE, "tcgen05 path needs nif_fast_pack_dev first");
  cudaStream_t st = (cudaStream_t)stream;
  const BucketWs w = bucket_ws(scratch, capacity, f->n_obj);  // hist zero on entry
  int64_t blocks = (capacity + 255) / 256;
  const int64_t cap_blocks = (int64_t)sm_count() * 8;
  if (blocks > cap_blocks) blocks = cap_blocks;
  bucket_hist_kernel<<<(unsigned)blocks, 256, (size_t)f->n_obj * 4, st>>>(obj, count_dev, capacity,
                                                                          f->n_obj, w.hist);
  bucket_scan_kernel<<<1, 256, 0, st>>>(w, f->n_obj);
  if (f->n_obj <= 4096) {
    int64_t cb = (capacity + kBucketChunk - 1) / kBucketChunk;
    if (cb > cap_blocks) cb = cap_blocks;
    bucket_scatter_block_kernel<<<(unsigned)(cb > 0 ? cb : 1), 256, (size_t)f->n_obj * 12, st>>>(
        obj, count_dev, capacity, w, f->n_obj);
  } else {
    bucket_scatter_kernel<<<(unsigned)blocks, 256, 0, st>>>(obj, count_dev, capacity, w);
  }
  TcArgs a{(const uint8_t*)f->fast, l, obj, ray, coord4, r, count_dev, capacity, occ_ray,
           logits, nullptr, w.perm, w.tile_obj, w.n_tiles};
  // the tile range is bounded by max_tiles (read from the device count in-kernel)
  a.cap = w.max_tiles * kTileRows;
  int rc = NIF_OK;
  if (launch_ts_po(a, *f, st, &rc) != 0)
    return fail(NIF_ERR_UNSUPPORTED, "no per-object tensor-core specialisation for W=%d L=%d",
                l.W, l.L);
  return rc;
}

extern "C" size_t nif_feat_scratch_bytes(int64_t capacity) {
  return (size_t)((capacity + kTileRows - 1) / kTileRows) * kTileRows * 32;
}

extern "C" int nif_query_split_dev(const nif_family_view* f, const int32_t* obj,
                                   const int32_t* ray, const float* coord4, const float* r,
                                   const int64_t* count_dev, int64_t capacity, uint8_t* occ_ray,
                                   float* logits, void* feat, int32_t flags, void* stream) {
  if (capacity <= 0) return NIF_OK;
  if (f->family == NIF_FAMILY_INNER && r == nullptr)
    return fail(NIF_ERR_VALUE, "inner queries need the radial coordinate");
  if (feat == nullptr) return fail(NIF_ERR_VALUE, "split query needs a feature scratch buffer");
  const FastLayout l = make_layout(*f);
  if (!l.tc_ok || l.HD != 1)
    return fail(NIF_ERR_UNSUPPORTED, "configuration not covered by the tcgen05 kernels");
  if (!f->fast) return fail(NIF_ERR_VALUE, "tcgen05 path needs nif_fast_pack_dev first");
  int rc = NIF_OK;
  if (launch_split(*f, l, obj, ray, coord4, r, count_dev, capacity, occ_ray, logits,
                   (uint8_t*)feat, flags, (cudaStream_t)stream, &rc) != 0)
    return fail(NIF_ERR_UNSUPPORTED, "no split-path specialisation for W=%d L=%d", l.W, l.L);
  return rc;
}

extern "C" int nif_occ_init_dev(const uint8_t* bvh_occ, int64_t n, uint8_t* occ_ray,
                                void* stream) {
  if (n <= 0) return NIF_OK;
  occ_init_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(bvh_occ, n,
                                                                                  occ_ray);
  return check_launch("nif_occ_init_dev");
}

extern "C" int nif_debug_set_query_grid(int ctas_per_sm) {
  g_query_cpsm = ctas_per_sm;
  return NIF_OK;
}

extern "C" int nif_debug_set_query_variant(int v) {
  g_query_variant = v;
  return NIF_OK;
}

extern "C" int nif_debug_set_timeline_query(void* buf) {
  g_tl_query = (unsigned long long*)buf;
  return NIF_OK;
}

extern "C" int nif_debug_set_prof(void* buf) {
  g_prof = (long long*)buf;
  return NIF_OK;
}
