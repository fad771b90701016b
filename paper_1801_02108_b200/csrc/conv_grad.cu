// Training path: the direct NHWC convolution forward and its input / weight /
// bias gradients, and the branch's BN + ReLU (+ in-bounds map) forward / adjoint, so the
// unit backward's recomputation and products run natively (no cuDNN, no torch arithmetic).
// Convolution gradients: input / weight / bias gradients of
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

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// direct NHWC convolution (the forward half of the training path's recomputation; reference
// `conv2d_nhwc`, `ops.py:145-164`): one thread per output element, output channel fastest
// (coalesced weight reads, broadcast input reads); taps accumulated in the reference's
// order (tap by tap, each tap's channel sum added to the running total), then + bias
template <typename T>
__global__ void __launch_bounds__(kGThreads) conv_forward_kernel(const T* __restrict__ x, const T* __restrict__ wt,
                                                                 const T* __restrict__ bias, GradGeo q, T* __restrict__ y) {
  using A = typename Acc<T>::type;
  const long total = (long)q.n * q.oh * q.ow * q.cout;
  for (long e = blockIdx.x * (long)kGThreads + threadIdx.x; e < total; e += (long)gridDim.x * kGThreads) {
    const int k = (int)(e % q.cout);
    long r = e / q.cout;
    const int ox = (int)(r % q.ow);
    r /= q.ow;
    const int oy = (int)(r % q.oh);
    const int n = (int)(r / q.oh);
    A acc = A(0);
    for (int i = 0; i < q.kh; ++i) {
      const int yy = oy * q.sh + i - q.ph;
      if ((unsigned)yy >= (unsigned)q.h) continue;
      for (int j = 0; j < q.kw; ++j) {
        const int xx = ox * q.sw + j - q.pw;
        if ((unsigned)xx >= (unsigned)q.w) continue;
        const T* xp = x + (((long)n * q.h + yy) * q.w + xx) * q.cin;
        const T* wp = wt + (long)(i * q.kw + j) * q.cin * q.cout + k;
        A tap = A(0);
        for (int c = 0; c < q.cin; ++c) tap += to_acc(__ldg(xp + c)) * to_acc(__ldg(wp + (long)c * q.cout));
        acc += tap;
      }
    }
    if (bias) acc += to_acc(__ldg(bias + k));
    y[e] = from_acc<T>(acc);
  }
}

// inference BN + ReLU of the recomputed branch (reference `ops.py:213-216`, `:233-234`):
// pre = x * s + t (a rounded multiply, then a rounded add, as numpy), post = relu(pre) * valid
// (valid: per-pixel 0 / 1, or none)
template <typename T>
__global__ void __launch_bounds__(kGThreads) bn_relu_kernel(const T* __restrict__ x, long count, int c,
                                                            const T* __restrict__ s, const T* __restrict__ t,
                                                            const T* __restrict__ valid, T* __restrict__ pre,
                                                            T* __restrict__ post) {
  for (long e = blockIdx.x * (long)kGThreads + threadIdx.x; e < count; e += (long)gridDim.x * kGThreads) {
    const int ch = (int)(e % c);
    const T b = add_rn(mul_rn(x[e], __ldg(s + ch)), __ldg(t + ch));  // no FMA contraction
    if (pre) pre[e] = b;
    T r = b > T(0) ? b : T(0);
    if (valid) r = r * __ldg(valid + e / c);
    post[e] = r;
  }
}

// its adjoint: out = g * valid * (pre > 0) * s  (valid / the ReLU mask are exact 0 / 1 factors)
template <typename T>
__global__ void __launch_bounds__(kGThreads) bn_relu_grad_kernel(const T* __restrict__ g, const T* __restrict__ pre,
                                                                 long count, int c, const T* __restrict__ s,
                                                                 const T* __restrict__ valid, T* __restrict__ out) {
  for (long e = blockIdx.x * (long)kGThreads + threadIdx.x; e < count; e += (long)gridDim.x * kGThreads) {
    const bool on = pre[e] > T(0) && (!valid || __ldg(valid + e / c) != T(0));
    out[e] = on ? mul_rn(g[e], __ldg(s + e % c)) : T(0);
  }
}

template <typename T>
__global__ void __launch_bounds__(kGThreads) add_kernel(const T* __restrict__ a, const T* __restrict__ b, long count,
                                                        T* __restrict__ out) {
  for (long e = blockIdx.x * (long)kGThreads + threadIdx.x; e < count; e += (long)gridDim.x * kGThreads)
    out[e] = a[e] + b[e];
}

// train-mode batch statistics of the gathered blocks (reference `sparse_batch_norm`,
// `layers.py:68-82`): per-channel mean, then the mean of squared deviations (population
// variance), each as fixed row segments reduced in order (deterministic); and the
// normalisation (x - mean) * (gamma / sqrt(var + eps)) + beta
template <typename T>
__global__ void __launch_bounds__(kGThreads) channel_sum_partial_kernel(const T* __restrict__ x, long rows, int c,
                                                                        const typename Acc<T>::type* __restrict__ mean,
                                                                        typename Acc<T>::type* __restrict__ part) {
  using A = typename Acc<T>::type;
  const long r0 = (long)blockIdx.y * kSeg, r1 = r0 + kSeg < rows ? r0 + kSeg : rows;
  for (int ch = blockIdx.x * kGThreads + threadIdx.x; ch < c; ch += gridDim.x * kGThreads) {
    A acc = A(0);
    const A m = mean ? mean[ch] : A(0);
    for (long r = r0; r < r1; ++r) {
      const A v = to_acc(__ldg(x + r * c + ch));
      acc += mean ? (v - m) * (v - m) : v;
    }
    part[(long)blockIdx.y * c + ch] = acc;
  }
}

template <typename A>
__global__ void __launch_bounds__(kGThreads) channel_sum_reduce_kernel(const A* __restrict__ part, int segs, int c,
                                                                       long rows, A* __restrict__ out) {
  for (int ch = blockIdx.x * kGThreads + threadIdx.x; ch < c; ch += gridDim.x * kGThreads) {
    A s = A(0);
    for (int sg = 0; sg < segs; ++sg) s += part[(long)sg * c + ch];
    out[ch] = s / A(rows);
  }
}

template <typename T>
__global__ void __launch_bounds__(kGThreads) bn_train_apply_kernel(const T* __restrict__ x, long count, int c,
                                                                   const typename Acc<T>::type* __restrict__ mean,
                                                                   const typename Acc<T>::type* __restrict__ var,
                                                                   const T* __restrict__ gamma, const T* __restrict__ beta,
                                                                   double eps, T* __restrict__ out) {
  using A = typename Acc<T>::type;
  for (long e = blockIdx.x * (long)kGThreads + threadIdx.x; e < count; e += (long)gridDim.x * kGThreads) {
    const int ch = (int)(e % c);
    const A sc = to_acc(gamma[ch]) / sqrt(var[ch] + A(eps));
    out[e] = from_acc<T>((to_acc(x[e]) - mean[ch]) * sc + to_acc(beta[ch]));
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

extern "C" int sbn_conv_forward(const void* x, int dtype, int n, int h, int w, int cin, int oh, int ow, int cout,
                                const void* wt, int kh, int kw, int sh, int sw, int ph, int pw, const void* bias,
                                void* y, sbn_stream_t stream) {
  GradGeo q{n, h, w, cin, oh, ow, cout, kh, kw, sh, sw, ph, pw};
  int st = check_grad_geo(q);
  if (st) return st;
  SBN_CHECK_ARG(dtype == SBN_F32 || dtype == SBN_F64, SBN_ERR_UNSUPPORTED, "conv forward: float32 / float64 only");
  if (n == 0) return SBN_OK;
  SBN_CHECK_ARG(x && wt && y, SBN_ERR_INVALID, "null pointer argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = grid_for((long)n * oh * ow * cout);
  if (dtype == SBN_F32)
    conv_forward_kernel<float><<<grid, kGThreads, 0, s>>>((const float*)x, (const float*)wt, (const float*)bias, q, (float*)y);
  else
    conv_forward_kernel<double><<<grid, kGThreads, 0, s>>>((const double*)x, (const double*)wt, (const double*)bias, q,
                                                           (double*)y);
  return launch_status("conv_forward");
}

extern "C" int sbn_bn_relu(const void* x, int dtype, long count, int c, const void* scale, const void* shift,
                           const void* valid, void* pre, void* post, sbn_stream_t stream) {
  SBN_CHECK_ARG(dtype == SBN_F32 || dtype == SBN_F64, SBN_ERR_UNSUPPORTED, "bn_relu: float32 / float64 only");
  SBN_CHECK_ARG(count >= 0 && c > 0 && count % c == 0, SBN_ERR_SHAPE, "bad element count / channels");
  if (count == 0) return SBN_OK;
  SBN_CHECK_ARG(x && scale && shift && post, SBN_ERR_INVALID, "null pointer argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = grid_for(count);
  if (dtype == SBN_F32)
    bn_relu_kernel<float><<<grid, kGThreads, 0, s>>>((const float*)x, count, c, (const float*)scale, (const float*)shift,
                                                     (const float*)valid, (float*)pre, (float*)post);
  else
    bn_relu_kernel<double><<<grid, kGThreads, 0, s>>>((const double*)x, count, c, (const double*)scale,
                                                      (const double*)shift, (const double*)valid, (double*)pre,
                                                      (double*)post);
  return launch_status("bn_relu");
}

extern "C" int sbn_bn_relu_grad(const void* g, const void* pre, int dtype, long count, int c, const void* scale,
                                const void* valid, void* out, sbn_stream_t stream) {
  SBN_CHECK_ARG(dtype == SBN_F32 || dtype == SBN_F64, SBN_ERR_UNSUPPORTED, "bn_relu_grad: float32 / float64 only");
  SBN_CHECK_ARG(count >= 0 && c > 0 && count % c == 0, SBN_ERR_SHAPE, "bad element count / channels");
  if (count == 0) return SBN_OK;
  SBN_CHECK_ARG(g && pre && scale && out, SBN_ERR_INVALID, "null pointer argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = grid_for(count);
  if (dtype == SBN_F32)
    bn_relu_grad_kernel<float><<<grid, kGThreads, 0, s>>>((const float*)g, (const float*)pre, count, c,
                                                          (const float*)scale, (const float*)valid, (float*)out);
  else
    bn_relu_grad_kernel<double><<<grid, kGThreads, 0, s>>>((const double*)g, (const double*)pre, count, c,
                                                           (const double*)scale, (const double*)valid, (double*)out);
  return launch_status("bn_relu_grad");
}

extern "C" int sbn_add(const void* a, const void* b, int dtype, long count, void* out, sbn_stream_t stream) {
  SBN_CHECK_ARG(dtype == SBN_F32 || dtype == SBN_F64, SBN_ERR_UNSUPPORTED, "add: float32 / float64 only");
  if (count <= 0) return SBN_OK;
  SBN_CHECK_ARG(a && b && out, SBN_ERR_INVALID, "null pointer argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = grid_for(count);
  if (dtype == SBN_F32)
    add_kernel<float><<<grid, kGThreads, 0, s>>>((const float*)a, (const float*)b, count, (float*)out);
  else
    add_kernel<double><<<grid, kGThreads, 0, s>>>((const double*)a, (const double*)b, count, (double*)out);
  return launch_status("add");
}

extern "C" size_t sbn_bn_train_workspace(int dtype, long rows, int c) {
  const long segs = rows > 0 ? (rows + kSeg - 1) / kSeg : 1;
  return (size_t)(segs + 2) * c * acc_size(dtype);
}

extern "C" int sbn_bn_train(const void* x, int dtype, long rows, int c, const void* gamma, const void* beta,
                            double eps, void* out, void* mean, void* var, void* ws, size_t ws_bytes,
                            sbn_stream_t stream) {
  SBN_CHECK_ARG(dtype == SBN_F32 || dtype == SBN_F64, SBN_ERR_UNSUPPORTED, "bn_train: float32 / float64 only");
  SBN_CHECK_ARG(rows > 0 && c > 0 && eps > 0, SBN_ERR_SHAPE, "bn_train needs rows > 0, c > 0, eps > 0");
  SBN_CHECK_ARG(x && gamma && beta && out && mean && var, SBN_ERR_INVALID, "null pointer argument");
  SBN_CHECK_ARG(ws && ws_bytes >= sbn_bn_train_workspace(dtype, rows, c), SBN_ERR_WORKSPACE,
                "bn_train needs a %zu-byte workspace", sbn_bn_train_workspace(dtype, rows, c));
  cudaStream_t s = (cudaStream_t)stream;
  const int segs = (int)((rows + kSeg - 1) / kSeg);
  const dim3 g1((unsigned)((c + kGThreads - 1) / kGThreads), (unsigned)segs);
  const int g2 = (c + kGThreads - 1) / kGThreads;
  const long count = rows * c;
#define LAUNCH(T)                                                                                                   \
  {                                                                                                                 \
    using A = typename Acc<T>::type;                                                                                \
    A* part = (A*)ws;                                                                                               \
    A* m = part + (size_t)segs * c;                                                                                 \
    A* v = m + c;                                                                                                   \
    channel_sum_partial_kernel<T><<<g1, kGThreads, 0, s>>>((const T*)x, rows, c, nullptr, part);                   \
    channel_sum_reduce_kernel<A><<<g2, kGThreads, 0, s>>>(part, segs, c, rows, m);                                  \
    channel_sum_partial_kernel<T><<<g1, kGThreads, 0, s>>>((const T*)x, rows, c, m, part);                         \
    channel_sum_reduce_kernel<A><<<g2, kGThreads, 0, s>>>(part, segs, c, rows, v);                                  \
    bn_train_apply_kernel<T><<<grid_for(count), kGThreads, 0, s>>>((const T*)x, count, c, m, v, (const T*)gamma,    \
                                                                 (const T*)beta, eps, (T*)out);                     \
    cudaMemcpyAsync(mean, m, (size_t)c * sizeof(A), cudaMemcpyDeviceToDevice, s);                                   \
    cudaMemcpyAsync(var, v, (size_t)c * sizeof(A), cudaMemcpyDeviceToDevice, s);                                    \
  }
  if (dtype == SBN_F32) LAUNCH(float) else LAUNCH(double)
#undef LAUNCH
  note_launch(4);  // five launches (launch_status counts the last)
  return launch_status("bn_train");
}
