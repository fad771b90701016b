// Generic fused sparse convolution (SIMT): gather -> valid conv -> scatter in one kernel.
//
// Covers every configuration the reference accepts (`verify.py:60-76`: any kh, kw,
// strides <= kernel, any channel counts, VALID/SAME, f32/f64/bf16).  It is the exact-
// precision path (fp32 FFMA / fp64 DFMA) used for the reference's 1e-5..1e-4 parity
// tolerances; the bf16 tensor-core path is conv_tc.cu.
//
// Work item = (active block, output slice): a block's obh*obw*cout outputs are split over
// `splits` CTAs so small batches still fill the GPU (config 1: 12 blocks x 6 slices).  Each
// CTA stages the block's input window once in shared memory with zero-filled halo (the
// gather of `blocks.py:57-74`) and, when they fit, the whole filter bank (staged once per
// CTA; both operands then come from shared memory: a warp's threads read consecutive
// output channels of one pixel, so weight reads are conflict-free and window reads are
// broadcasts).  Each output keeps the per-tap accumulation order of `ops.py:145-164`
// (sum over input channels per tap, taps added in (i, j) order, bias last) and is stored
// straight into the block's clipped, disjoint output window (the scatter of
// `blocks.py:125-142`).  Persistent grid over the items (device-side block count).
#include "common.cuh"

namespace sbn {
namespace {

constexpr int kThreads = 256;
constexpr size_t kWeightSmemMax = 64 * 1024;  // stage the filter bank when it fits next to the window

template <typename T, bool SMEM, bool WSMEM>
__global__ void __launch_bounds__(kThreads)
sparse_conv_simt_kernel(const T* __restrict__ x, Geo g, int cin, int cout, int kh, int kw, int sh,
                        int sw, const T* __restrict__ w, const T* __restrict__ bias,
                        const int32_t* __restrict__ idx, const int32_t* __restrict__ count,
                        int cap, T* __restrict__ dst, int splits) {
  using A = typename Acc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* win = reinterpret_cast<A*>(smem_raw);
  const int win_elems = SMEM ? g.bh * g.bw * cin : 0;
  A* wts = win + win_elems;
  if (WSMEM) {  // filter bank (HWIO), once per CTA
    const int nw = kh * kw * cin * cout;
    for (int e = threadIdx.x; e < nw; e += kThreads) wts[e] = to_acc(__ldg(w + e));
    // (made visible by the __syncthreads after the first window)
  }
  const int B = ld_count(count, cap);
  const int total = g.obh * g.obw * cout;
  int staged = -1;  // block whose window is in smem
  for (int it = blockIdx.x; it < B * splits; it += gridDim.x) {
    const int b = it / splits, sl = it - b * splits;
    const int n = __ldg(idx + 3 * b), by = __ldg(idx + 3 * b + 1), bx = __ldg(idx + 3 * b + 2);
    const int ys = g.oy + by * g.sy, xs = g.ox + bx * g.sx;
    if (SMEM && staged != b) {
      if (staged >= 0) __syncthreads();  // previous block's reads are done
      for (int e = threadIdx.x; e < win_elems; e += kThreads) {
        const int ci = e % cin;
        const int p = e / cin;
        const int wy = p / g.bw, wx = p - wy * g.bw;
        const int y = ys + wy, xx = xs + wx;
        A v = A(0);
        if (y >= 0 && y < g.h && xx >= 0 && xx < g.w)
          v = to_acc(x[(((size_t)n * g.h + y) * g.w + xx) * cin + ci]);
        win[e] = v;
      }
      __syncthreads();
      staged = b;
    } else if (WSMEM && !SMEM && staged < 0) {
      __syncthreads();
      staged = b;
    }
    for (int o = sl * kThreads + threadIdx.x; o < total; o += splits * kThreads) {
      const int co = o % cout;
      const int p = o / cout;
      const int oyb = p / g.obw, oxb = p - oyb * g.obw;
      const int Y = by * g.obh + oyb, X = bx * g.obw + oxb;
      if (Y >= g.oh || X >= g.ow) continue;
      A acc = A(0);
      for (int i = 0; i < kh; ++i) {
        const int wy = oyb * sh + i;
        for (int j = 0; j < kw; ++j) {
          const int wx = oxb * sw + j;
          const size_t wo = ((size_t)(i * kw + j) * cin) * cout + co;
          A tap = A(0);
          if (SMEM) {
            const A* xp = win + (wy * g.bw + wx) * cin;
            if (WSMEM) {
              const A* wp = wts + wo;
#pragma unroll 4
              for (int ci = 0; ci < cin; ++ci) tap += xp[ci] * wp[(size_t)ci * cout];
            } else {
              const T* wp = w + wo;
#pragma unroll 4
              for (int ci = 0; ci < cin; ++ci) tap += xp[ci] * to_acc(__ldg(wp + (size_t)ci * cout));
            }
          } else {
            const int y = ys + wy, xx = xs + wx;
            if (y < 0 || y >= g.h || xx < 0 || xx >= g.w) continue;
            const T* xp = x + (((size_t)n * g.h + y) * g.w + xx) * cin;
            for (int ci = 0; ci < cin; ++ci)
              tap += to_acc(__ldg(xp + ci)) * (WSMEM ? wts[wo + (size_t)ci * cout] : to_acc(__ldg(w + wo + (size_t)ci * cout)));
          }
          acc += tap;
        }
      }
      if (bias) acc += to_acc(__ldg(bias + co));
      dst[(((size_t)n * g.oh + Y) * g.ow + X) * cout + co] = from_acc<T>(acc);
    }
  }
}

template <typename T, bool SMEM, bool WSMEM>
void launch_conv_simt_variant(size_t smem, int grid, cudaStream_t s, const void* x, Geo g, int cin, int cout, int kh,
                              int kw, int sh, int sw, const void* w, const void* bias, const int32_t* idx,
                              const int32_t* count, int cap, void* dst, int splits) {
  auto k = sparse_conv_simt_kernel<T, SMEM, WSMEM>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, kThreads, smem, s>>>((const T*)x, g, cin, cout, kh, kw, sh, sw, (const T*)w, (const T*)bias, idx, count,
                                 cap, (T*)dst, splits);
}

template <typename T>
int launch_conv_simt(const void* x, int cin, int cout, int kh, int kw, int sh, int sw, Geo g,
                     const void* w, const void* bias, const int32_t* idx, const int32_t* count,
                     int cap, void* dst, cudaStream_t s) {
  using A = typename Acc<T>::type;
  const size_t win_b = (size_t)g.bh * g.bw * cin * sizeof(A);
  const size_t w_b = (size_t)kh * kw * cin * cout * sizeof(A);
  // slices per block: about two outputs per thread, at most 16 CTAs per block
  const long total = (long)g.obh * g.obw * cout;
  int splits = (int)((total + 2 * kThreads - 1) / (2 * kThreads));
  splits = splits < 1 ? 1 : splits > 16 ? 16 : splits;
  const int grid = persistent_grid((int)((long)cap * splits < (1L << 30) ? (long)cap * splits : (1L << 30)), 4);
  const bool wsm = w_b <= kWeightSmemMax;
  if (win_b + (wsm ? w_b : 0) <= 96 * 1024) {
    if (wsm)
      launch_conv_simt_variant<T, true, true>(win_b + w_b, grid, s, x, g, cin, cout, kh, kw, sh, sw, w, bias, idx,
                                              count, cap, dst, splits);
    else
      launch_conv_simt_variant<T, true, false>(win_b, grid, s, x, g, cin, cout, kh, kw, sh, sw, w, bias, idx,
                                               count, cap, dst, splits);
  } else if (wsm) {
    launch_conv_simt_variant<T, false, true>(w_b, grid, s, x, g, cin, cout, kh, kw, sh, sw, w, bias, idx, count, cap,
                                             dst, splits);
  } else {
    launch_conv_simt_variant<T, false, false>(0, grid, s, x, g, cin, cout, kh, kw, sh, sw, w, bias, idx, count, cap,
                                              dst, splits);
  }
  return launch_status("sparse_conv_simt");
}

}  // namespace

int sparse_conv_tc_masked(const void* x, const uint8_t* mask, int cin, int cout, Geo g, const void* wpk,
                          const void* bias, int cap, void* dst, cudaStream_t s, unsigned* slotw, int32_t* gidx);
int sparse_conv_tc(const void* x, int cin, int cout, Geo g, const void* wpk, const void* bias,
                   const int32_t* idx, const int32_t* count, int cap, void* dst, cudaStream_t s);
size_t sparse_conv_tc_packed_bytes(int cin, int cout);
int sparse_conv_tc_pack(const void* w, int cin, int cout, void* img, cudaStream_t s);
bool sparse_conv_tma_supported(int dtype, int cin, int cout, int kh, int kw, int sh, int sw, const Geo& g);
size_t sparse_conv_tma_packed_bytes(int cin, int cout, int k);
int sparse_conv_tma_pack(const void* w, int cin, int cout, int k, void* img, cudaStream_t s);
int sparse_conv_tma(const void* x, int cin, int cout, int k, int sh, int sw, const Geo& g, const void* wpk,
                    const void* bias, const int32_t* idx, const int32_t* count, int cap, void* dst,
                    cudaStream_t s);
bool sparse_conv_tc_supported(int dtype, int cin, int cout, int kh, int kw, int sh, int sw,
                              const Geo& g);
int sparse_conv_tma_masked(const void* x, const uint8_t* mask, int cin, int cout, int k, int sh, int sw,
                           const Geo& g, const void* wpk, const void* bias, void* dst, cudaStream_t s,
                           unsigned* slotw, int32_t* gidx);

}  // namespace sbn

using namespace sbn;

// tensor-core variant for a sparse conv: 1 = single-window row-shift kernel (conv_tc.cu,
// 3x3 stride 1, blocks 8 / 16), 2 = strided-TMA tap GEMM (conv_dense_tc.cu, 1x1 / 3x3 / 5x5,
// stride <= 3, any out block: several tiles per block above 128 pixels), 0 = none (SIMT)
static int conv_tc_kind(int dtype, int cin, int cout, int kh, int kw, int sh, int sw, const Geo& g) {
  if (!(debug_flags() & kDebugConvTma) && sparse_conv_tc_supported(dtype, cin, cout, kh, kw, sh, sw, g)) return 1;
  if (sparse_conv_tma_supported(dtype, cin, cout, kh, kw, sh, sw, g)) return 2;
  return 0;
}

extern "C" int sbn_sparse_conv_algo(int dtype, int cin, int cout, int kh, int kw, int sh, int sw,
                                    const sbn_geometry* gp) {
  if (!gp) return SBN_ALGO_SIMT;
  return conv_tc_kind(dtype, cin, cout, kh, kw, sh, sw, to_geo(gp)) ? SBN_ALGO_TCGEN05 : SBN_ALGO_SIMT;
}

extern "C" size_t sbn_sparse_conv_packed_bytes(int dtype, int cin, int cout, int kh, int kw,
                                               int sh, int sw, const sbn_geometry* gp) {
  if (!gp) return 0;
  switch (conv_tc_kind(dtype, cin, cout, kh, kw, sh, sw, to_geo(gp))) {
    case 1: return sparse_conv_tc_packed_bytes(cin, cout);
    case 2: return sparse_conv_tma_packed_bytes(cin, cout, kh);
    default: return 0;
  }
}

extern "C" int sbn_sparse_conv_pack(const void* w, int dtype, int cin, int cout, int kh, int kw,
                                    int sh, int sw, const sbn_geometry* gp, void* packed,
                                    sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  const int kind = conv_tc_kind(dtype, cin, cout, kh, kw, sh, sw, to_geo(gp));
  SBN_CHECK_ARG(kind != 0, SBN_ERR_UNSUPPORTED, "tcgen05 sparse conv does not support this config");
  SBN_CHECK_ARG(w && packed, SBN_ERR_INVALID, "null argument");
  if (kind == 2) return sparse_conv_tma_pack(w, cin, cout, kh, packed, (cudaStream_t)stream);
  return sparse_conv_tc_pack(w, cin, cout, packed, (cudaStream_t)stream);
}

extern "C" int sbn_sparse_conv(const void* x, int dtype, int cin, int cout, int kh, int kw, int sh,
                               int sw, const sbn_geometry* gp, const void* w, const void* bias,
                               const void* w_packed, const int32_t* idx, const int32_t* count,
                               int cap, void* dst, void* ws, size_t ws_bytes, int algo,
                               sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  SBN_CHECK_ARG(cin > 0 && cout > 0, SBN_ERR_SHAPE, "channels must be > 0");
  SBN_CHECK_ARG(kh > 0 && kw > 0 && sh > 0 && sw > 0 && sh <= kh && sw <= kw, SBN_ERR_INVALID,
                "bad kernel/stride");
  SBN_CHECK_ARG(gp->bh >= kh && gp->bw >= kw, SBN_ERR_INVALID, "block smaller than kernel");
  SBN_CHECK_ARG((gp->bh - kh) / sh + 1 == gp->obh && (gp->bw - kw) / sw + 1 == gp->obw,
                SBN_ERR_INVALID, "out block size inconsistent with kernel/stride");
  if (cap <= 0) return SBN_OK;
  SBN_CHECK_ARG(x && w && idx && count && dst, SBN_ERR_INVALID, "null pointer argument");
  Geo g = to_geo(gp);
  cudaStream_t s = (cudaStream_t)stream;
  const int kind = conv_tc_kind(dtype, cin, cout, kh, kw, sh, sw, g);
  if (algo == SBN_ALGO_TCGEN05) {
    SBN_CHECK_ARG(kind != 0, SBN_ERR_UNSUPPORTED, "tcgen05 sparse conv does not support this config");
  }
  if (kind != 0 && algo != SBN_ALGO_SIMT) {
    const void* wpk = w_packed;
    if (!wpk) {
      const size_t nb = kind == 1 ? sparse_conv_tc_packed_bytes(cin, cout) : sparse_conv_tma_packed_bytes(cin, cout, kh);
      SBN_CHECK_ARG(ws && ws_bytes >= nb, SBN_ERR_WORKSPACE,
                    "tcgen05 sparse conv without a packed weight image needs a %zu-byte workspace", nb);
      int st2 = kind == 1 ? sparse_conv_tc_pack(w, cin, cout, ws, s) : sparse_conv_tma_pack(w, cin, cout, kh, ws, s);
      if (st2) return st2;
      wpk = ws;
    }
    if (kind == 2) return sparse_conv_tma(x, cin, cout, kh, sh, sw, g, wpk, bias, idx, count, cap, dst, s);
    return sparse_conv_tc(x, cin, cout, g, wpk, bias, idx, count, cap, dst, s);
  }
  switch (dtype) {
    case SBN_F32:
      return launch_conv_simt<float>(x, cin, cout, kh, kw, sh, sw, g, w, bias, idx, count, cap, dst, s);
    case SBN_F64:
      return launch_conv_simt<double>(x, cin, cout, kh, kw, sh, sw, g, w, bias, idx, count, cap, dst, s);
    case SBN_BF16:
      return launch_conv_simt<__nv_bfloat16>(x, cin, cout, kh, kw, sh, sw, g, w, bias, idx, count,
                                             cap, dst, s);
    default:
      set_error("unsupported dtype %d", dtype);
      return SBN_ERR_UNSUPPORTED;
  }
}

// ---- sparse_conv2d from the mask (reference `layers.py:27-47`, MAX pool with the default
// threshold): on the tcgen05 double-buffered path the mask reduction runs inside the conv
// kernel (one launch); otherwise sbn_reduce_mask + sbn_sparse_conv.
//   sync_ws (zeroed ONCE by the caller, kept between calls, fixed layout so calls of any
//   geometry may share it): [256 B reserved | reduce_mask ws (fallback path)]
//   ws (scratch): [index list cap*12 | count 256 B | packed weights when none are given]
static size_t al256c(size_t v) { return (v + 255) / 256 * 256; }

extern "C" size_t sbn_sparse_conv_masked_sync_bytes(const sbn_geometry* gp) {
  return gp ? 256 + al256c(sbn_reduce_mask_workspace(gp)) : 0;
}

extern "C" size_t sbn_sparse_conv_masked_workspace(int dtype, int cin, int cout, int kh, int kw, int sh, int sw,
                                                   const sbn_geometry* gp) {
  if (!gp) return 0;
  const size_t cap = (size_t)gp->n * gp->gy * gp->gx;
  return al256c(cap * 12) + 256 + al256c(sbn_sparse_conv_packed_bytes(dtype, cin, cout, kh, kw, sh, sw, gp));
}

extern "C" int sbn_sparse_conv_masked(const void* x, const uint8_t* mask, int dtype, int cin, int cout, int kh,
                                      int kw, int sh, int sw, const sbn_geometry* gp, const void* w,
                                      const void* bias, const void* w_packed, void* dst, void* sync_ws,
                                      size_t sync_bytes, void* ws, size_t ws_bytes, int algo, sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  SBN_CHECK_ARG(x && mask && w && dst, SBN_ERR_INVALID, "null pointer argument");
  SBN_CHECK_ARG(sync_ws && sync_bytes >= sbn_sparse_conv_masked_sync_bytes(gp), SBN_ERR_WORKSPACE,
                "sparse_conv2d (masked) needs a %zu-byte zeroed sync workspace", sbn_sparse_conv_masked_sync_bytes(gp));
  const size_t need = sbn_sparse_conv_masked_workspace(dtype, cin, cout, kh, kw, sh, sw, gp);
  SBN_CHECK_ARG(ws && ws_bytes >= need, SBN_ERR_WORKSPACE, "sparse_conv2d (masked) needs a %zu-byte workspace", need);
  const int cap = gp->n * gp->gy * gp->gx;
  if (cap <= 0) return SBN_OK;
  uint8_t* rmws = (uint8_t*)sync_ws + 256;
  const size_t rmb = sync_bytes - 256;
  uint8_t* w8 = (uint8_t*)ws;
  int32_t* idx = (int32_t*)w8;
  int32_t* count = (int32_t*)(w8 + al256c((size_t)cap * 12));
  uint8_t* pk = w8 + al256c((size_t)cap * 12) + 256;
  const size_t pkb = ws_bytes - al256c((size_t)cap * 12) - 256;
  cudaStream_t s = (cudaStream_t)stream;
  Geo g = to_geo(gp);
  const int kind = conv_tc_kind(dtype, cin, cout, kh, kw, sh, sw, g);
  if (kind == 1 && algo != SBN_ALGO_SIMT) {
    const void* wpk = w_packed;
    if (!wpk) {
      st = sparse_conv_tc_pack(w, cin, cout, pk, s);
      if (st) return st;
      wpk = pk;
    }
    // slot words: the first 64 bytes of the (zeroed-once) sync workspace; list rows: idx
    st = sparse_conv_tc_masked(x, mask, cin, cout, g, wpk, bias, cap, dst, s, (unsigned*)sync_ws, idx);
    if (st != SBN_ERR_UNSUPPORTED) return st;
  }
  // (a global list in this launch, as for the kernel above, measured slower here than
  // reduce_mask + conv: config 3, 32x32 blocks, 26.1 vs 23.4 us at 5 %, 90 vs 82 at 30 %)
  if (kind == 2 && algo != SBN_ALGO_SIMT && (long)cap <= 64L * sm_count()) {  // one launch (local or global list)
    const void* wpk = w_packed;
    if (!wpk) {
      st = sparse_conv_tma_pack(w, cin, cout, kh, pk, s);
      if (st) return st;
      wpk = pk;
    }
    st = sparse_conv_tma_masked(x, mask, cin, cout, kh, sh, sw, g, wpk, bias, dst, s, (unsigned*)sync_ws, idx);
    if (st != SBN_ERR_UNSUPPORTED) return st;
  }
  st = sbn_reduce_mask(mask, gp, SBN_POOL_MAX, 1.0 / ((double)gp->bh * gp->bw), idx, count, rmws, rmb, stream);
  if (st) return st;
  return sbn_sparse_conv(x, dtype, cin, cout, kh, kw, sh, sw, gp, w, bias, w_packed, idx, count, cap, dst,
                         w_packed ? nullptr : pk, w_packed ? 0 : pkb, algo, stream);
}
