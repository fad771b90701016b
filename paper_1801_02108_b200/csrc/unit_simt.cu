// Generic fused sparse residual unit (SIMT) + rim snapshot + the C-ABI dispatcher.
//
// Restates reference `sparse_residual_unit` (`layers.py:203-229`) and `_unit_branch`
// (`layers.py:137-179`) as one kernel per unit: per active block, the window is
// gathered (zero-filled halo), the bottleneck chain runs on-chip, and the result is
// scatter-added into `out` (the reference's `scatter_add(branch, x)`), never
// materialising the block stack.  Pre- and post-activation chains, any halo >= 0
// (conv2 pad 1 for halo 0, crop halo-1 otherwise), f32/f64/bf16.  BN is applied as
// separate rounded multiply and add, as numpy's `arr * scale + shift` (`ops.py:213-216`).
#include "unit.cuh"

namespace sbn {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <typename A>
__device__ __forceinline__ A bn(A v, const A* s, const A* t, int ch) {
  return add_rn(mul_rn(v, s[ch]), t[ch]);
}
template <typename A>
__device__ __forceinline__ A relu(A v) {
  return v > A(0) ? v : A(0);
}
// round an intermediate to the activation dtype (identity for f32/f64)
template <typename T, typename A>
__device__ __forceinline__ A rnd(A v) {
  return to_acc(from_acc<T>(v));
}

template <typename T>
struct UnitArgs {
  const T* x;
  T* out;
  const T* rim;  // non-null: in-place mode (x == out), rim snapshot holds the halo
  Geo g;
  int c, m, halo, pre;
  const T *w1, *b1, *w2, *b2, *w3, *b3;
  UnitFold<typename Acc<T>::type> f;
  const int32_t* idx;
  const int32_t* count;
  int cap;
  typename Acc<T>::type* gscratch;  // null -> dynamic shared memory
  size_t scratch_elems;              // per CTA
};

template <typename T>
__global__ void __launch_bounds__(kThreads) unit_simt_kernel(UnitArgs<T> a) {
  using A = typename Acc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* base = a.gscratch ? a.gscratch + (size_t)blockIdx.x * a.scratch_elems
                       : reinterpret_cast<A*>(smem_raw);
  const Geo& g = a.g;
  const int c = a.c, m = a.m;
  const int npix = g.bh * g.bw;
  A* s0 = base;                       // window (npix x c)
  A* s1 = s0 + (size_t)npix * c;      // stage 1 (npix x m)
  A* s2 = s1 + (size_t)npix * m;      // stage 2 (obh*obw x m)
  const int pad2 = a.halo >= 1 ? 0 : 1;
  const int crop = a.halo >= 1 ? a.halo - 1 : 0;
  const Rim rim{g.bh, g.bw, a.halo};
  const int P = rim.pixels();
  const int B = ld_count(a.count, a.cap);

  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    const int n = __ldg(a.idx + 3 * b), by = __ldg(a.idx + 3 * b + 1), bx = __ldg(a.idx + 3 * b + 2);
    const int ys = g.oy + by * g.sy, xs = g.ox + bx * g.sx;
    // ---- gather (+ pre-activation BN1/ReLU)
    for (int e = threadIdx.x; e < npix * c; e += kThreads) {
      const int ci = e % c, p = e / c;
      const int wy = p / g.bw, wx = p - wy * g.bw;
      const int y = ys + wy, xx = xs + wx;
      A v = A(0);
      if (a.rim && !rim.interior(wy, wx)) {
        v = to_acc(a.rim[((size_t)b * P + rim.index(wy, wx)) * c + ci]);
      } else if (y >= 0 && y < g.h && xx >= 0 && xx < g.w) {
        v = to_acc(a.x[(((size_t)n * g.h + y) * g.w + xx) * c + ci]);
      }
      if (a.pre) v = rnd<T>(relu(bn(v, a.f.s1, a.f.t1, ci)));
      s0[e] = v;
    }
    __syncthreads();
    // ---- stage 1: 1x1 c->m (+b1), BN, ReLU, x in-bounds
    for (int e = threadIdx.x; e < npix * m; e += kThreads) {
      const int j = e % m, p = e / m;
      const A* xp = s0 + (size_t)p * c;
      A acc = A(0);
      for (int ci = 0; ci < c; ++ci) acc += xp[ci] * to_acc(__ldg(a.w1 + (size_t)ci * m + j));
      acc = rnd<T>(acc + to_acc(__ldg(a.b1 + j)));
      acc = a.pre ? rnd<T>(relu(bn(acc, a.f.s2, a.f.t2, j))) : rnd<T>(relu(bn(acc, a.f.s1, a.f.t1, j)));
      const int wy = p / g.bw, wx = p - wy * g.bw;
      const int y = ys + wy, xx = xs + wx;
      const bool valid = (y >= 0 && y < g.h && xx >= 0 && xx < g.w);
      s1[e] = valid ? acc : A(0);
    }
    __syncthreads();
    // ---- stage 2: 3x3 m->m on the window (valid, or pad 1 for halo 0), cropped to the
    //      block's output window, (+b2), BN, ReLU
    const int nq = g.obh * g.obw;
    for (int e = threadIdx.x; e < nq * m; e += kThreads) {
      const int j = e % m, q = e / m;
      const int qy = q / g.obw + crop, qx = q % g.obw + crop;
      A acc = A(0);
      for (int ky = 0; ky < 3; ++ky) {
        const int sy = qy + ky - pad2;
        if (sy < 0 || sy >= g.bh) continue;
        for (int kx = 0; kx < 3; ++kx) {
          const int sx = qx + kx - pad2;
          if (sx < 0 || sx >= g.bw) continue;
          const A* ip = s1 + (size_t)(sy * g.bw + sx) * m;
          const T* wp = a.w2 + (size_t)((ky * 3 + kx) * m) * m + j;
          A tap = A(0);
          for (int ci = 0; ci < m; ++ci) tap += ip[ci] * to_acc(__ldg(wp + (size_t)ci * m));
          acc += tap;
        }
      }
      acc = rnd<T>(acc + to_acc(__ldg(a.b2 + j)));
      acc = a.pre ? relu(bn(acc, a.f.s3, a.f.t3, j)) : relu(bn(acc, a.f.s2, a.f.t2, j));
      s2[e] = rnd<T>(acc);
    }
    __syncthreads();
    // ---- stage 3: 1x1 m->c (+b3) [post: BN3], scatter-add into out
    for (int e = threadIdx.x; e < nq * c; e += kThreads) {
      const int co = e % c, q = e / c;
      const int qy = q / g.obw, qx = q - qy * g.obw;
      const int Y = by * g.obh + qy, X = bx * g.obw + qx;
      if (Y >= g.oh || X >= g.ow) continue;
      const A* ip = s2 + (size_t)q * m;
      A acc = A(0);
      for (int j = 0; j < m; ++j) acc += ip[j] * to_acc(__ldg(a.w3 + (size_t)j * c + co));
      acc = rnd<T>(acc + to_acc(__ldg(a.b3 + co)));
      if (!a.pre) acc = rnd<T>(bn(acc, a.f.s3, a.f.t3, co));
      T* op = a.out + (((size_t)n * g.oh + Y) * g.ow + X) * c + co;
      *op = from_acc<T>(add_rn(to_acc(*op), acc));
    }
    __syncthreads();
  }
}

template <int VS>
__global__ void __launch_bounds__(kThreads)
rim_kernel(const uint8_t* __restrict__ x, Geo g, Rim rim, int pix_bytes,
           const int32_t* __restrict__ idx, const int32_t* __restrict__ count, int cap,
           uint8_t* __restrict__ out) {
  // CTA per active block (grid-strided over the device-side count), 32-bit index math:
  // the rim of one block is P pixels x vpp vectors (config-4 stage 0: 60 x 12)
  using V = typename std::conditional<VS == 16, uint4, typename std::conditional<VS == 8, uint2, uint32_t>::type>::type;
  const int B = ld_count(count, cap);
  const int P = rim.pixels();
  const int vpp = pix_bytes / VS;
  const int per = P * vpp;
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    const int n = __ldg(idx + 3 * b);
    const int y0 = g.oy + __ldg(idx + 3 * b + 1) * g.sy, x0 = g.ox + __ldg(idx + 3 * b + 2) * g.sx;
    V* dst = reinterpret_cast<V*>(out) + (size_t)b * per;
    for (int i = threadIdx.x; i < per; i += kThreads) {
      const int r = i / vpp, k = i - r * vpp;
      int wy, wx;
      rim.coord(r, wy, wx);
      const int y = y0 + wy, xx = x0 + wx;
      V v;
      if (y >= 0 && y < g.h && xx >= 0 && xx < g.w)
        v = *(reinterpret_cast<const V*>(x + (((size_t)n * g.h + y) * g.w + xx) * pix_bytes) + k);
      else
        memset(&v, 0, sizeof(V));
      dst[i] = v;
    }
  }
}

template <typename A>
size_t simt_scratch_elems(int c, int m, const Geo& g) {
  return (size_t)g.bh * g.bw * (c + m) + (size_t)g.obh * g.obw * m;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

size_t rim_bytes(int es, int c, const Geo& g, int halo, int cap) {
  Rim r{g.bh, g.bw, halo};
  return align_up((size_t)cap * r.pixels() * c * es, 256);
}

template <typename T>
int launch_unit_simt(const void* x, void* out, const void* rim, int c, int m, const Geo& g,
                     int halo, int pre, const sbn_unit_params* p, const int32_t* idx,
                     const int32_t* count, int cap, void* ws, cudaStream_t s) {
  using A = typename Acc<T>::type;
  UnitArgs<T> a;
  a.x = (const T*)x;
  a.out = (T*)out;
  a.rim = (const T*)rim;
  a.g = g;
  a.c = c; a.m = m; a.halo = halo; a.pre = pre;
  a.w1 = (const T*)p->w1; a.b1 = (const T*)p->b1;
  a.w2 = (const T*)p->w2; a.b2 = (const T*)p->b2;
  a.w3 = (const T*)p->w3; a.b3 = (const T*)p->b3;
  a.f = UnitFold<A>{(const A*)p->bn1_scale, (const A*)p->bn1_shift, (const A*)p->bn2_scale,
                    (const A*)p->bn2_shift, (const A*)p->bn3_scale, (const A*)p->bn3_shift};
  a.idx = idx; a.count = count; a.cap = cap;
  a.scratch_elems = simt_scratch_elems<A>(c, m, g);
  const size_t smem = a.scratch_elems * sizeof(A);
  int grid;
  if ((int)smem <= max_smem_optin()) {
    a.gscratch = nullptr;
    grid = persistent_grid(cap, smem <= 100 * 1024 ? 2 : 1);
    auto k = unit_simt_kernel<T>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, kThreads, smem, s>>>(a);
  } else {
    grid = persistent_grid(cap, 1);
    a.gscratch = reinterpret_cast<A*>(ws);
    unit_simt_kernel<T><<<grid, kThreads, 0, s>>>(a);
  }
  return launch_status("residual_unit_simt");
}

}  // namespace

int unit_rim_snapshot(const void* x, int es, int c, const Geo& g, int halo, const int32_t* idx,
                      const int32_t* count, int cap, void* rim, cudaStream_t s) {
  Rim r{g.bh, g.bw, halo};
  const int pix = c * es;
  long grid = cap < (long)sm_count() * 8 ? cap : (long)sm_count() * 8;  // CTAs stride over the blocks
  if (grid < 1) grid = 1;
  const uintptr_t al = (uintptr_t)x | (uintptr_t)rim;
  if (pix % 16 == 0 && al % 16 == 0)
    rim_kernel<16><<<(unsigned)grid, kThreads, 0, s>>>((const uint8_t*)x, g, r, pix, idx, count,
                                                       cap, (uint8_t*)rim);
  else if (pix % 8 == 0 && al % 8 == 0)
    rim_kernel<8><<<(unsigned)grid, kThreads, 0, s>>>((const uint8_t*)x, g, r, pix, idx, count, cap,
                                                      (uint8_t*)rim);
  else if (pix % 4 == 0 && al % 4 == 0)
    rim_kernel<4><<<(unsigned)grid, kThreads, 0, s>>>((const uint8_t*)x, g, r, pix, idx, count, cap,
                                                      (uint8_t*)rim);
  else {
    set_error("rim snapshot needs 4-byte aligned pixels (c*elem_size=%d)", pix);
    return SBN_ERR_UNSUPPORTED;
  }
  return launch_status("unit_rim_snapshot");
}

// Workspace layout: [256 B grid-barrier words (zeroed once by the caller, self-resetting)
//                    | rim snapshot (in-place calls) | packed tc image or SIMT scratch]
constexpr size_t kBarBytes = 256;

// wide tcgen05 path: [256 B | S1/S2 stacks | packed image (when none is given)]
size_t unit_workspace_wide(int c, int m, const Geo& g) {
  return kBarBytes + unit_wide_stack_bytes(m, g) + align_up(unit_wide_packed_bytes(c, m), 256);
}

// which tensor-core variant applies: 1 single-kernel unit, 2 wide (pipelined persistent
// launches), 0 none.  The single kernel walks one block's latency chain per CTA; past ~4K
// candidate blocks the pipelined wide unit (one launch for 16x16 blocks) is faster even
// where the single kernel fits (tools/wide_vs_fused.py, config-2 shapes, mask-fused public
// path, single vs wide: 10 % density 34.9 vs 45.9 us at 4 frames (3.4K candidates), 48.3 vs
// 47.0 at 6, 60.7 vs 54.3 at 8, 402.8 vs 242.8 at 64; 20 %: 49.9 vs 50.8 at 4, 76.4 vs 63.4
// at 6, 724.9 vs 425.5 at 64).  Where the wide unit is still three launches (blocks other
// than 16x16) the crossover is ~8K candidates (8 frames: 91 vs 102 us at 20 %).
int unit_tc_kind(int dtype, int c, int m, const Geo& g, int halo, int pre_act) {
  const long cand = (long)g.n * g.gy * g.gx;
  const long max_single = unit_wide_one_launch(c, m, g) ? 4096 : 8192;
  if (!(debug_flags() & kDebugForceWide) &&
      (cand <= max_single || (debug_flags() & kDebugForceFused)) &&
      unit_tc_supported(dtype, c, m, g, halo, pre_act))
    return 1;
  if (unit_tc_supported(dtype, c, m, g, halo, pre_act) && !unit_wide_supported(dtype, c, m, g, halo, pre_act))
    return 1;
  if (unit_wide_supported(dtype, c, m, g, halo, pre_act)) return 2;
  return 0;
}

// a caller-supplied packed image must have been built for the variant this call runs
static int check_packed(const sbn_unit_params* p, int variant, size_t want) {
  SBN_CHECK_ARG(!p->tc_packed || (p->tc_packed_variant == variant && p->tc_packed_bytes == want), SBN_ERR_INVALID,
                "tc_packed image (variant %d, %zu bytes) does not match this call's variant %d (%zu bytes): "
                "it was packed for another block size or batch size",
                p->tc_packed_variant, p->tc_packed_bytes, variant, want);
  return SBN_OK;
}

size_t unit_workspace(int dtype, int c, int m, const Geo& g, int halo, int algo, bool tc) {
  const int es = dtype_size(dtype);
  const int cap = g.n * g.gy * g.gx;
  if (tc && unit_tc_kind(dtype, c, m, g, halo, 1) == 2) return unit_workspace_wide(c, m, g);
  size_t ws = kBarBytes + rim_bytes(es, c, g, halo, cap);
  if (tc) ws += align_up(unit_tc_packed_bytes(c, m, g), 256);  // packing when no image given
  if (!tc) {
    const size_t ae = dtype == SBN_F64 ? 8 : 4;
    const size_t per = simt_scratch_elems<float>(c, m, g) * ae;
    if ((long)per > (long)max_smem_optin()) ws += align_up(per, 256) * (size_t)persistent_grid(cap, 1);
  }
  (void)algo;
  return ws;
}

}  // namespace sbn

using namespace sbn;

extern "C" int sbn_residual_unit_algo(int dtype, int c, int m, const sbn_geometry* gp, int halo,
                                      int pre_act) {
  if (!gp) return SBN_ALGO_SIMT;
  return unit_tc_kind(dtype, c, m, to_geo(gp), halo, pre_act) ? SBN_ALGO_TCGEN05 : SBN_ALGO_SIMT;
}

extern "C" size_t sbn_residual_unit_packed_bytes(int dtype, int c, int m, const sbn_geometry* gp,
                                                 int halo, int pre_act) {
  if (!gp) return 0;
  Geo g = to_geo(gp);
  switch (unit_tc_kind(dtype, c, m, g, halo, pre_act)) {
    case 1: return unit_tc_packed_bytes(c, m, g);
    case 2: return unit_wide_packed_bytes(c, m);
    default: return 0;
  }
}

extern "C" int sbn_residual_unit_packed_variant(int dtype, int c, int m, const sbn_geometry* gp,
                                                int halo, int pre_act) {
  if (!gp) return 0;
  return unit_tc_kind(dtype, c, m, to_geo(gp), halo, pre_act);
}

extern "C" int sbn_residual_unit_pack(const sbn_unit_params* p, int dtype, int c, int m,
                                      const sbn_geometry* gp, int halo, int pre_act, void* packed,
                                      sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  Geo g = to_geo(gp);
  const int kind = unit_tc_kind(dtype, c, m, g, halo, pre_act);
  SBN_CHECK_ARG(kind != 0, SBN_ERR_UNSUPPORTED, "tcgen05 residual unit does not support this config");
  SBN_CHECK_ARG(p && packed, SBN_ERR_INVALID, "null argument");
  if (kind == 2) return unit_wide_pack(p, c, m, packed, (cudaStream_t)stream);
  return unit_tc_pack(p, c, m, g, packed, (cudaStream_t)stream);
}

extern "C" size_t sbn_residual_unit_workspace(int dtype, int c, int m, const sbn_geometry* gp,
                                              int halo, int algo) {
  if (!gp || dtype_size(dtype) == 0) return 0;
  Geo g = to_geo(gp);
  const bool tc = algo != SBN_ALGO_SIMT && unit_tc_kind(dtype, c, m, g, halo, 1) != 0;
  return unit_workspace(dtype, c, m, g, halo, algo, tc);
}

extern "C" int sbn_residual_unit(const void* x, int dtype, int c, int m, const sbn_geometry* gp,
                                 int halo, int pre_act, const sbn_unit_params* p,
                                 const int32_t* idx, const int32_t* count, int cap, void* out,
                                 void* ws, size_t ws_bytes, int algo, sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  SBN_CHECK_ARG(dtype_size(dtype) > 0, SBN_ERR_UNSUPPORTED, "unsupported dtype %d", dtype);
  SBN_CHECK_ARG(c > 0 && m > 0, SBN_ERR_SHAPE, "channels must be > 0");
  SBN_CHECK_ARG(halo >= 0, SBN_ERR_INVALID, "halo must be >= 0");
  SBN_CHECK_ARG(gp->sy == gp->obh && gp->sx == gp->obw && gp->bh - 2 * halo == gp->obh && gp->bw - 2 * halo == gp->obw
                    && gp->oh == gp->h && gp->ow == gp->w,
                SBN_ERR_INVALID, "geometry is not a residual-unit (SAME, stride 1, halo %d) spec",
                halo);
  SBN_CHECK_ARG(p && p->w1 && p->b1 && p->w2 && p->b2 && p->w3 && p->b3 && p->bn1_scale &&
                    p->bn1_shift && p->bn2_scale && p->bn2_shift && p->bn3_scale && p->bn3_shift,
                SBN_ERR_INVALID, "null unit parameter");
  if (cap <= 0) return SBN_OK;
  SBN_CHECK_ARG(x && out && idx && count, SBN_ERR_INVALID, "null pointer argument");
  Geo g = to_geo(gp);
  cudaStream_t s = (cudaStream_t)stream;
  const int kind = unit_tc_kind(dtype, c, m, g, halo, pre_act);
  if (algo == SBN_ALGO_TCGEN05)
    SBN_CHECK_ARG(kind != 0, SBN_ERR_UNSUPPORTED, "tcgen05 residual unit does not support this config");
  const bool use_tc = kind != 0 && algo != SBN_ALGO_SIMT;
  const size_t need = unit_workspace(dtype, c, m, g, halo, algo, use_tc);
  const bool inplace = (x == out);
  const void* rim = nullptr;
  uint8_t* wsb = (uint8_t*)ws;
  if (use_tc && kind == 2) {  // wide: three launches; kernel order resolves the in-place rims
    SBN_CHECK_ARG(ws && ws_bytes >= need, SBN_ERR_WORKSPACE,
                  "residual unit needs a %zu-byte workspace", need);
    uint8_t* stacks = wsb + kBarBytes;
    st = check_packed(p, 2, unit_wide_packed_bytes(c, m));
    if (st) return st;
    const void* packed = p->tc_packed;
    if (!packed) {
      packed = stacks + unit_wide_stack_bytes(m, g);
      st = unit_wide_pack(p, c, m, (void*)packed, s);
      if (st) return st;
    }
    return unit_wide_launch(x, out, c, m, g, packed, idx, count, cap, stacks, s);
  }
  const size_t rb = kBarBytes + rim_bytes(dtype_size(dtype), c, g, halo, cap);
  if (inplace && halo > 0) {
    SBN_CHECK_ARG(ws && ws_bytes >= need, SBN_ERR_WORKSPACE,
                  "in-place residual unit needs a %zu-byte workspace", need);
    if (!use_tc) {  // the tcgen05 kernel handles the rim itself (grid barrier)
      st = unit_rim_snapshot(x, dtype_size(dtype), c, g, halo, idx, count, cap, wsb + kBarBytes, s);
      if (st) return st;
      rim = wsb + kBarBytes;
    }
  }
  if (use_tc) {
    st = check_packed(p, 1, unit_tc_packed_bytes(c, m, g));
    if (st) return st;
    const void* packed = p->tc_packed;
    if (!packed) {
      SBN_CHECK_ARG(ws && ws_bytes >= need, SBN_ERR_WORKSPACE,
                    "residual unit needs a %zu-byte workspace", need);
      st = unit_tc_pack(p, c, m, g, wsb + rb, s);
      if (st) return st;
      packed = wsb + rb;
    }
    return unit_tc_launch(x, out, inplace ? wsb + kBarBytes : nullptr,
                          inplace ? reinterpret_cast<unsigned int*>(wsb) : nullptr, c, m, g, p,
                          packed, idx, count, cap, s);
  }
  void* scratch = nullptr;
  if (need > rb) {
    SBN_CHECK_ARG(ws && ws_bytes >= need, SBN_ERR_WORKSPACE,
                  "residual unit needs a %zu-byte workspace", need);
    scratch = wsb + rb;
  }
  switch (dtype) {
    case SBN_F32:
      return launch_unit_simt<float>(x, out, rim, c, m, g, halo, pre_act, p, idx, count, cap, scratch, s);
    case SBN_F64:
      return launch_unit_simt<double>(x, out, rim, c, m, g, halo, pre_act, p, idx, count, cap, scratch, s);
    default:
      return launch_unit_simt<__nv_bfloat16>(x, out, rim, c, m, g, halo, pre_act, p, idx, count, cap,
                                             scratch, s);
  }
}

// ---- whole sparse_residual_unit (`layers.py:203-229`): mask -> active blocks -> fused unit.
// tcgen05 path: ONE kernel (reduce_mask fused into the unit, unordered active list).
// Otherwise: ordered sbn_reduce_mask + sbn_residual_unit.
// sync_ws (zeroed once, left zeroed): [unit barrier words (256 B) | reduce_mask ws]
// ws (scratch):                      [idx (cap*12) | count | rim | packed image / SIMT scratch]
static size_t al256(size_t v) { return (v + 255) / 256 * 256; }

// sync ws: [barrier/epoch words (256 B) | epoch look-back status (8 B x 4096 CTAs) | reduce_mask ws]
constexpr size_t kCstBytes = 8 * (size_t)kEpochMaxCtas;

extern "C" size_t sbn_sparse_residual_unit_sync_bytes(const sbn_geometry* gp) {
  if (!gp) return 0;
  return kBarBytes + kCstBytes + al256(sbn_reduce_mask_workspace(gp));
}

extern "C" size_t sbn_sparse_residual_unit_workspace(int dtype, int c, int m, const sbn_geometry* gp,
                                                     int halo, int algo) {
  if (!gp || dtype_size(dtype) == 0) return 0;
  const size_t cap = (size_t)gp->n * gp->gy * gp->gx;
  return 256 + al256(cap * 8) + 256 + al256(cap * 12) + sbn_residual_unit_workspace(dtype, c, m, gp, halo, algo);
}

extern "C" int sbn_sparse_residual_unit(const void* x, const uint8_t* mask, int dtype, int c, int m,
                                        const sbn_geometry* gp, int halo, int pre_act,
                                        const sbn_unit_params* p, void* out, void* sync_ws,
                                        size_t sync_bytes, void* ws, size_t ws_bytes, int algo,
                                        sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  SBN_CHECK_ARG(x && mask && out && p, SBN_ERR_INVALID, "null pointer argument");
  SBN_CHECK_ARG(sync_ws && sync_bytes >= sbn_sparse_residual_unit_sync_bytes(gp), SBN_ERR_WORKSPACE,
                "sparse_residual_unit needs a %zu-byte zeroed sync workspace",
                sbn_sparse_residual_unit_sync_bytes(gp));
  const size_t need = sbn_sparse_residual_unit_workspace(dtype, c, m, gp, halo, algo);
  SBN_CHECK_ARG(ws && ws_bytes >= need, SBN_ERR_WORKSPACE,
                "sparse_residual_unit needs a %zu-byte workspace", need);
  const int cap = gp->n * gp->gy * gp->gx;
  if (cap <= 0) return SBN_OK;
  // [slot words 256 B | tagged entries cap*8 | count 256 B | index list cap*12 | unit ws]: the
  // slot words (launch epoch) and the tagged entries sit at fixed offsets from the start, so
  // calls with different geometries sharing one workspace never see each other's index
  // data where they look for tags (a smaller cap's entry range is a prefix of a larger one's)
  uint8_t* w8 = (uint8_t*)ws;
  unsigned int* slotw = (unsigned int*)w8;
  unsigned long long* etag = (unsigned long long*)(w8 + 256);
  int32_t* count = (int32_t*)(w8 + 256 + al256((size_t)cap * 8));
  int32_t* idx = (int32_t*)(w8 + 256 + al256((size_t)cap * 8) + 256);
  uint8_t* uws = w8 + 256 + al256((size_t)cap * 8) + 256 + al256((size_t)cap * 12);  // [bar | rim | pack]
  uint8_t* sync8 = (uint8_t*)sync_ws;
  unsigned int* gbar = reinterpret_cast<unsigned int*>(sync8);
  unsigned long long* cst = reinterpret_cast<unsigned long long*>(sync8 + kBarBytes);
  uint8_t* rmws = sync8 + kBarBytes + kCstBytes;
  Geo g = to_geo(gp);
  cudaStream_t s = (cudaStream_t)stream;
  const bool tc = algo != SBN_ALGO_SIMT && unit_tc_kind(dtype, c, m, g, halo, pre_act) == 1;
  if (algo == SBN_ALGO_TCGEN05)
    SBN_CHECK_ARG(unit_tc_kind(dtype, c, m, g, halo, pre_act) != 0, SBN_ERR_UNSUPPORTED,
                  "tcgen05 residual unit does not support this config");
  if (tc) {
    SBN_CHECK_ARG(gp->sy == gp->obh && gp->sx == gp->obw && gp->bh - 2 * halo == gp->obh &&
                      gp->oh == gp->h && gp->ow == gp->w,
                  SBN_ERR_INVALID, "geometry is not a residual-unit spec");
    const size_t rb = kBarBytes + rim_bytes(dtype_size(dtype), c, g, halo, cap);
    st = check_packed(p, 1, unit_tc_packed_bytes(c, m, g));
    if (st) return st;
    const void* packed = p->tc_packed;
    if (!packed) {
      st = unit_tc_pack(p, c, m, g, uws + rb, s);
      if (st) return st;
      packed = uws + rb;
    }
    const bool inplace = x == out;
    return unit_tc_launch(x, out, inplace ? uws + kBarBytes : nullptr, gbar, c, m, g, p, packed,
                          idx, count, cap, s, mask, idx, count, cst, etag, slotw);
  }
  st = sbn_reduce_mask(mask, gp, SBN_POOL_MAX, 1.0 / ((double)gp->bh * gp->bw), idx, count, rmws,
                       sync_bytes - kBarBytes - kCstBytes, stream);
  if (st) return st;
  // the two-launch path needs zeroed barrier words at the start of its workspace: the
  // 256 barrier bytes of sync_ws are followed by the (zeroed) reduce_mask words, so point
  // the unit at a scratch region whose first 256 bytes we clear here
  cudaMemsetAsync(uws, 0, kBarBytes, s);
  return sbn_residual_unit(x, dtype, c, m, gp, halo, pre_act, p, idx, count, cap, out, uws,
                           ws_bytes - (size_t)(uws - w8), algo, stream);
}
