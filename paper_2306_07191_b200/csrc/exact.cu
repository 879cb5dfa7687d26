// Reference-exact array API kernels: grid encoding with fp64 interpolation
// weights (grids.py:125-206, nif.py:286-311) and the row-sequential dense
// forward with fp64 accumulation (nif.py:321-359). Compiled with
// -fmad=false; the output equals the reference's arrays bit for bit (the
// sigmoid head may differ in the last ulp of exp()).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.h"
#include "nif_b200.h"
#include "status.h"

namespace nif {
namespace {

struct Axis {
  int i0, i1;
  double w;
};

// grids.py:125-138 (_axis_indices)
__device__ __forceinline__ Axis axis_indices(double x, int R, bool wrap) {
  const double xc = x * (double)R - 0.5;
  const double x0 = floor(xc);
  Axis a;
  a.w = xc - x0;
  long long i0 = (long long)x0;
  long long i1 = i0 + 1;
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

// grids.py:141-162 (_bilinear + lookup_2d_batch), written into out[0..N)
__device__ __forceinline__ void lookup_2d(const float* __restrict__ g, int R, int N, double u,
                                          double v, double* out) {
  const Axis au = axis_indices(u, R, true);
  const Axis av = axis_indices(v, R, false);
  const double wu = au.w, wv = av.w;
  const double w00 = (1.0 - wu) * (1.0 - wv);
  const double w01 = (1.0 - wu) * wv;
  const double w10 = wu * (1.0 - wv);
  const double w11 = wu * wv;
  const float* g00 = g + ((size_t)au.i0 * R + av.i0) * N;
  const float* g01 = g + ((size_t)au.i0 * R + av.i1) * N;
  const float* g10 = g + ((size_t)au.i1 * R + av.i0) * N;
  const float* g11 = g + ((size_t)au.i1 * R + av.i1) * N;
  for (int k = 0; k < N; ++k) {
    const double s = w00 * (double)g00[k] + w01 * (double)g01[k] + w10 * (double)g10[k] +
                     w11 * (double)g11[k];
    out[k] = (double)(float)s;  // .astype(grid.dtype)
  }
}

// grids.py:187-191 (lookup_1d_batch)
__device__ __forceinline__ void lookup_1d(const float* __restrict__ g, int R, int N, double x,
                                          double* out) {
  const Axis a = axis_indices(x, R, false);
  const float* g0 = g + (size_t)a.i0 * N;
  const float* g1 = g + (size_t)a.i1 * N;
  for (int k = 0; k < N; ++k) {
    const double s = (1.0 - a.w) * (double)g0[k] + a.w * (double)g1[k];
    out[k] = (double)(float)s;
  }
}

__global__ void encode_kernel(nif_family_view f, const int64_t* __restrict__ obj,
                              const double* __restrict__ coord, int64_t m,
                              double* __restrict__ out, int* __restrict__ bad) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int64_t o = obj[j];
  if (o < 0 || o >= f.n_obj) {
    atomicMax(bad, 1);
    return;
  }
  const int cw = f.family == NIF_FAMILY_OUTER ? 4 : 5;
  const double* c = coord + j * cw;
  const int in_dim = f.dims[0];
  double* y = out + j * in_dim;
  const size_t g2 = (size_t)f.R * f.R * f.N;
  lookup_2d(f.pos + (size_t)o * g2, f.R, f.N, c[0], c[1], y);
  lookup_2d(f.dir + (size_t)o * g2, f.R, f.N, c[2], c[3], y + f.N);
  if (f.family == NIF_FAMILY_INNER)
    lookup_1d(f.dist + (size_t)o * f.Rd * f.Nd, f.Rd, f.Nd, c[4], y + 2 * f.N);
}

constexpr int kMaxWidth = 256;

// nif.py:321-359 (_k_dense_forward), one row per thread
__global__ void dense_forward_kernel(nif_family_view f, const int64_t* __restrict__ obj,
                                     const double* __restrict__ x, int64_t m, int sigmoid_head,
                                     double* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int head = f.n_heads > 1 ? (int)obj[j] : 0;
  const float* W = f.w + (size_t)head * f.w_stride;
  const float* B = f.b + (size_t)head * f.b_stride;
  double bufa[kMaxWidth], bufb[kMaxWidth];
  for (int k = 0; k < f.dims[0]; ++k) bufa[k] = x[j * f.dims[0] + k];
  int wo = 0, bo = 0;
  const int nl = f.n_layers;
  for (int layer = 0; layer < nl; ++layer) {
    const int nin = f.dims[layer], nout = f.dims[layer + 1];
    for (int o = 0; o < nout; ++o) {
      double acc = (double)__ldg(B + bo + o);
      const float* wr = W + wo + o * nin;
      for (int k = 0; k < nin; ++k) acc += (double)__ldg(wr + k) * bufa[k];
      if (layer < nl - 1) {
        bufb[o] = acc > 0.0 ? acc : 0.01 * acc;
      } else if (sigmoid_head == 1) {
        if (acc >= 0.0) {
          bufb[o] = 1.0 / (1.0 + exp(-acc));
        } else {
          const double e = exp(acc);
          bufb[o] = e / (1.0 + e);
        }
      } else {
        bufb[o] = acc;
      }
    }
    wo += nin * nout;
    bo += nout;
    for (int o = 0; o < nout; ++o) bufa[o] = bufb[o];
  }
  for (int k = 0; k < f.dims[nl]; ++k) out[j * f.dims[nl] + k] = bufa[k];
}

}  // namespace
}  // namespace nif

using namespace nif;

namespace {
int check_family(const nif_family_view* f) {
  if (f->n_layers < 1 || f->n_layers > NIF_MAX_LAYERS)
    return fail(NIF_ERR_VALUE, "layer count must be in [1, %d]", NIF_MAX_LAYERS);
  for (int i = 0; i <= f->n_layers; ++i)
    if (f->dims[i] < 1 || f->dims[i] > kMaxWidth)
      return fail(NIF_ERR_UNSUPPORTED, "layer width %d outside [1, %d]", f->dims[i], kMaxWidth);
  return NIF_OK;
}
}  // namespace

extern "C" int nif_encode_dev(const nif_family_view* f, const int64_t* obj, const double* coord,
                              int64_t m, double* out, void* stream) {
  int rc = check_family(f);
  if (rc) return rc;
  if (m <= 0) return NIF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int* bad = nullptr;
  if (cudaMallocAsync(&bad, sizeof(int), st) != cudaSuccess)
    return fail(NIF_ERR_CUDA, "encode: allocation failed");
  cudaMemsetAsync(bad, 0, sizeof(int), st);
  encode_kernel<<<(unsigned)((m + 127) / 128), 128, 0, st>>>(*f, obj, coord, m, out, bad);
  int hbad = 0;
  cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(bad, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("nif_encode_dev");
  if (hbad) return fail(NIF_ERR_VALUE, "object id out of range (model covers %d)", f->n_obj);
  return check_launch("nif_encode_dev");
}

extern "C" int nif_forward_dev(const nif_family_view* f, const int64_t* obj, const double* x,
                               int64_t m, int32_t sigmoid_head, double* out, void* stream) {
  int rc = check_family(f);
  if (rc) return rc;
  if (m <= 0) return NIF_OK;
  dense_forward_kernel<<<(unsigned)((m + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      *f, obj, x, m, sigmoid_head, out);
  return check_launch("nif_forward_dev");
}
