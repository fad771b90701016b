// Convolution gradients (training path): input / weight / bias gradients of
// the direct NHWC convolution for an upstream gradient, restating reference
// `conv2d_grads_nhwc` (`ops.py:167-197`).  Used on the gathered block stacks by
// sparse_conv2d_grads (`layers.py:50-65`) and sparse_residual_unit_grads (`layers.py:232-270`),
// and by conv2d_direct_grads.
//
//   dx[n, y, x, c]  = sum over taps (i, j) in order of  sum_k g[n, oy, ox, k] * W[i, j, c, k]
//                     with y = oy*sh + i - ph, x = ox*sw + j - pw   (one thread per dx element)
//   dw[i, j, c, k]  = sum over (n, oy, ox) of x[n, y, x, c] * g[n, oy, ox, k]
//   db[k]           = sum over (n, oy, ox) of g[n, oy, ox, k]
//
// The reductions over output positions are deterministic: positions are cut into fixed
// segments, each segment's partial sum is written to the caller's workspace, and a second
// pass adds the segments in order (no atomics), so repeated calls are bit-identical.
// Accumulation is in the compute type of the dtype (fp32 for f32 / bf16, fp64 for f64).
#include "common.cuh"

namespace sbn {
namespace {

constexpr int kGThreads = 256;
constexpr int kSeg = 2048;  // output positions per partial sum of dw / db

struct GradGeo {
  int n, h, w, cin, oh, ow, cout, kh, kw, sh, sw, ph, pw;
};

template <typename T>
__global__ void __launch_bounds__(kGThreads) conv_grad_input_kernel(const T* __restrict__ g, const T* __restrict__ wt,
                                                                    GradGeo q, T* __restrict__ dx) {
  using A = typename Acc<T>::type;
  const long total = (long)q.n * q.h * q.w * q.cin;
  for (long e = blockIdx.x * (long)kGThreads + threadIdx.x; e < total; e += (long)gridDim.x * kGThreads) {
    const int c = (int)(e % q.cin);
    long r = e / q.cin;
    const int x = (int)(r % q.w);
    r /= q.w;
    const int y = (int)(r % q.h);
    const int n = (int)(r / q.h);
    A acc = A(0);
    for (int i = 0; i < q.kh; ++i) {
      const int ty = y + q.ph - i;
      if (ty < 0 || ty % q.sh) continue;
      const int oy = ty / q.sh;
      if (oy >= q.oh) continue;
      for (int j = 0; j < q.kw; ++j) {
        const int tx = x + q.pw - j;
        if (tx < 0 || tx % q.sw) continue;
        const int ox = tx / q.sw;
        if (ox >= q.ow) continue;
        const T* gp = g + (((long)n * q.oh + oy) * q.ow + ox) * q.cout;
        const T* wp = wt + ((long)(i * q.kw + j) * q.cin + c) * q.cout;
        A tap = A(0);
        for (int k = 0; k < q.cout; ++k) tap += to_acc(__ldg(gp + k)) * to_acc(__ldg(wp + k));
        acc += tap;
      }
    }
    dx[e] = from_acc<T>(acc);
  }
}

// partial dw (and db as the extra "tap" index kh*kw when with_bias) over one segment of
// output positions; grid.y = segment
template <typename T>
__global__ void __launch_bounds__(kGThreads) conv_grad_weight_partial_kernel(
    const T* __restrict__ x, const T* __restrict__ g, GradGeo q, bool with_bias,
    typename Acc<T>::type* __restrict__ part) {
  using A = typename Acc<T>::type;
  const long nw = (long)q.kh * q.kw * q.cin * q.cout;
  const long nout = nw + (with_bias ? q.cout : 0);
  const long P = (long)q.n * q.oh * q.ow;
  const long p0 = (long)blockIdx.y * kSeg, p1 = p0 + kSeg < P ? p0 + kSeg : P;
  for (long e = blockIdx.x * (long)kGThreads + threadIdx.x; e < nout; e += (long)gridDim.x * kGThreads) {
    A acc = A(0);
    if (e < nw) {
      const int k = (int)(e % q.cout);
      long r = e / q.cout;
      const int c = (int)(r % q.cin);
      r /= q.cin;
      const int j = (int)(r % q.kw);
      const int i = (int)(r / q.kw);
      for (long p = p0; p < p1; ++p) {
        const int ox = (int)(p % q.ow);
        const long t = p / q.ow;
        const int oy = (int)(t % q.oh);
        const int n = (int)(t / q.oh);
        const int y = oy * q.sh + i - q.ph, xx = ox * q.sw + j - q.pw;
        if ((unsigned)y >= (unsigned)q.h || (unsigned)xx >= (unsigned)q.w) continue;
        acc += to_acc(__ldg(x + (((long)n * q.h + y) * q.w + xx) * q.cin + c)) * to_acc(__ldg(g + p * q.cout + k));
      }
    } else {
      const int k = (int)(e - nw);
      for (long p = p0; p < p1; ++p) acc += to_acc(__ldg(g + p * q.cout + k));
    }
    part[(long)blockIdx.y * nout + e] = acc;
  }
}

template <typename T>
__global__ void __launch_bounds__(kGThreads) conv_grad_weight_reduce_kernel(const typename Acc<T>::type* __restrict__ part,
                                                                            long nw, long nout, int segs, T* __restrict__ dw,
                                                                            T* __restrict__ db) {
  using A = typename Acc<T>::type;
  for (long e = blockIdx.x * (long)kGThreads + threadIdx.x; e < nout; e += (long)gridDim.x * kGThreads) {
    A s = A(0);
    for (int sg = 0; sg < segs; ++sg) s += part[(long)sg * nout + e];  // segments in order
    if (e < nw)
      dw[e] = from_acc<T>(s);
    else
      db[e - nw] = from_acc<T>(s);
  }
}

int grid_for(long items) {
  const long g = (items + kGThreads - 1) / kGThreads, cap = (long)sm_count() * 8;
  return (int)(g < 1 ? 1 : g > cap ? cap : g);
}

int check_grad_geo(const GradGeo& q) {
  SBN_CHECK_ARG(q.n >= 0 && q.h > 0 && q.w > 0 && q.cin > 0 && q.cout > 0, SBN_ERR_SHAPE, "bad conv-grad dims");
  SBN_CHECK_ARG(q.kh > 0 && q.kw > 0 && q.sh > 0 && q.sw > 0 && q.ph >= 0 && q.pw >= 0, SBN_ERR_INVALID,
                "bad kernel / stride / padding");
  SBN_CHECK_ARG(q.oh == (q.h + 2 * q.ph - q.kh) / q.sh + 1 && q.ow == (q.w + 2 * q.pw - q.kw) / q.sw + 1,
                SBN_ERR_SHAPE, "gradient dims %dx%d do not match the conv output", q.oh, q.ow);
  return SBN_OK;
}

size_t acc_size(int dtype) { return dtype == SBN_F64 ? 8 : 4; }

}  // namespace
}  // namespace sbn

using namespace sbn;

extern "C" int sbn_conv_grad_input(const void* g, int dtype, int n, int h, int w, int cin, int oh, int ow, int cout,
                                   const void* wt, int kh, int kw, int sh, int sw, int ph, int pw, void* dx,
                                   sbn_stream_t stream) {
  GradGeo q{n, h, w, cin, oh, ow, cout, kh, kw, sh, sw, ph, pw};
  int st = check_grad_geo(q);
  if (st) return st;
  SBN_CHECK_ARG(dtype_size(dtype) > 0, SBN_ERR_UNSUPPORTED, "unsupported dtype %d", dtype);
  if (n == 0) return SBN_OK;
  SBN_CHECK_ARG(g && wt && dx, SBN_ERR_INVALID, "null pointer argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = grid_for((long)n * h * w * cin);
  switch (dtype) {
    case SBN_F32: conv_grad_input_kernel<float><<<grid, kGThreads, 0, s>>>((const float*)g, (const float*)wt, q, (float*)dx); break;
    case SBN_F64: conv_grad_input_kernel<double><<<grid, kGThreads, 0, s>>>((const double*)g, (const double*)wt, q, (double*)dx); break;
    default:
      conv_grad_input_kernel<__nv_bfloat16><<<grid, kGThreads, 0, s>>>((const __nv_bfloat16*)g, (const __nv_bfloat16*)wt, q,
                                                                      (__nv_bfloat16*)dx);
  }
  return launch_status("conv_grad_input");
}

extern "C" size_t sbn_conv_grad_weight_workspace(int dtype, int n, int oh, int ow, int cin, int cout, int kh, int kw) {
  const long P = (long)n * oh * ow;
  const long segs = P > 0 ? (P + kSeg - 1) / kSeg : 1;
  return (size_t)segs * ((size_t)kh * kw * cin * cout + cout) * acc_size(dtype);
}

extern "C" int sbn_conv_grad_weight(const void* x, const void* g, int dtype, int n, int h, int w, int cin, int oh,
                                    int ow, int cout, int kh, int kw, int sh, int sw, int ph, int pw, void* dw,
                                    void* db, void* ws, size_t ws_bytes, sbn_stream_t stream) {
  GradGeo q{n, h, w, cin, oh, ow, cout, kh, kw, sh, sw, ph, pw};
  int st = check_grad_geo(q);
  if (st) return st;
  SBN_CHECK_ARG(dtype_size(dtype) > 0, SBN_ERR_UNSUPPORTED, "unsupported dtype %d", dtype);
  SBN_CHECK_ARG((n == 0 || (x && g)) && dw, SBN_ERR_INVALID, "null pointer argument");
  const size_t need = sbn_conv_grad_weight_workspace(dtype, n, oh, ow, cin, cout, kh, kw);
  SBN_CHECK_ARG(ws && ws_bytes >= need, SBN_ERR_WORKSPACE, "conv weight gradient needs a %zu-byte workspace", need);
  cudaStream_t s = (cudaStream_t)stream;
  const long P = (long)n * oh * ow;
  const int segs = P > 0 ? (int)((P + kSeg - 1) / kSeg) : 1;
  const long nw = (long)kh * kw * cin * cout, nout = nw + (db ? cout : 0);
  const dim3 grid1((unsigned)grid_for(nout), (unsigned)segs);
  const int grid2 = grid_for(nout);
#define LAUNCH(T)                                                                                          \
  {                                                                                                        \
    using A = typename Acc<T>::type;                                                                       \
    conv_grad_weight_partial_kernel<T><<<grid1, kGThreads, 0, s>>>((const T*)x, (const T*)g, q, db != nullptr, \
                                                                   (A*)ws);                                \
    conv_grad_weight_reduce_kernel<T><<<grid2, kGThreads, 0, s>>>((const A*)ws, nw, nout, segs, (T*)dw, (T*)db); \
  }
  switch (dtype) {
    case SBN_F32: LAUNCH(float) break;
    case SBN_F64: LAUNCH(double) break;
    default: LAUNCH(__nv_bfloat16)
  }
#undef LAUNCH
  note_launch();  // two launches
  return launch_status("conv_grad_weight");
}
