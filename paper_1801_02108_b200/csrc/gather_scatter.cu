// gather / gather_transpose / scatter / scatter_add / scatter_transpose.
//
// Restates reference `blocks.py:57-159`.  NHWC rows are contiguous on both sides of
// every copy (a window row of bw pixels x C channels in the source, one stack row in
// the destination), so each warp streams whole rows with the widest vector (16 B when
// C*elem_size and the base pointers allow it), zero-filling the out-of-image halo.
// Scatter writes only each block's disjoint, clipped output window: no atomics, and
// the result is bit-exact (add mode does exactly one add in the tensor dtype per
// element, as numpy's `+=`).
#include "common.cuh"

namespace sbn {
namespace {

constexpr int kThreads = 256;

template <int VS> struct VecT;
template <> struct VecT<16> { using type = uint4; };
template <> struct VecT<8> { using type = uint2; };
template <> struct VecT<4> { using type = uint32_t; };
template <> struct VecT<2> { using type = uint16_t; };
template <> struct VecT<1> { using type = uint8_t; };

template <int VS>
__global__ void __launch_bounds__(kThreads)
gather_rows_kernel(const uint8_t* __restrict__ x, Geo g, int pix_bytes,
                   const int32_t* __restrict__ idx, const int32_t* __restrict__ count, int cap,
                   uint8_t* __restrict__ out) {
  using V = typename VecT<VS>::type;
  const int B = ld_count(count, cap);
  const int lane = threadIdx.x & 31;
  const long nwarps = (long)gridDim.x * (kThreads / 32);
  const int vpp = pix_bytes / VS;  // vectors per pixel
  const int nvec = g.bw * vpp;
  for (long r = blockIdx.x * (long)(kThreads / 32) + (threadIdx.x >> 5); r < (long)B * g.bh;
       r += nwarps) {
    const int b = (int)(r / g.bh), wy = (int)(r - (long)b * g.bh);
    const int n = __ldg(idx + 3 * b), by = __ldg(idx + 3 * b + 1), bx = __ldg(idx + 3 * b + 2);
    const int y = g.oy + by * g.sy + wy;
    const int xs = g.ox + bx * g.sx;
    const bool row_ok = (y >= 0 && y < g.h);
    V* dst = reinterpret_cast<V*>(out + (size_t)r * g.bw * pix_bytes);
    const V* src = reinterpret_cast<const V*>(x + ((size_t)n * g.h + (row_ok ? y : 0)) * g.w *
                                                      (size_t)pix_bytes);
    for (int k = lane; k < nvec; k += 32) {
      const int wx = k / vpp;
      const int xx = xs + wx;
      V v;
      if (row_ok && xx >= 0 && xx < g.w) {
        v = __ldg(src + (size_t)xx * vpp + (k - wx * vpp));
      } else {
        memset(&v, 0, sizeof(V));
      }
      dst[k] = v;
    }
  }
}

// Frame-to-frame copy of each active block's region at identical coordinates: region 0 =
// the input window clipped to the image, region 1 = the clipped output (write) window.
// Used to move only the bytes a sparse layer touches between a host-resident frame
// (pinned, UVA) and its device staging copy; warp per region row, 16-B vectors.
template <int VS>
__global__ void __launch_bounds__(kThreads)
copy_regions_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, Geo g, int pix_bytes,
                    const int32_t* __restrict__ idx, const int32_t* __restrict__ count, int cap, int region) {
  using V = typename VecT<VS>::type;
  const int B = ld_count(count, cap);
  const int lane = threadIdx.x & 31;
  const long nwarps = (long)gridDim.x * (kThreads / 32);
  const int rh = region == 0 ? g.bh : g.obh;
  const int fh = region == 0 ? g.h : g.oh, fw = region == 0 ? g.w : g.ow;
  const int rh2 = region == 1 ? g.obh : g.bh;
  for (long r = blockIdx.x * (long)(kThreads / 32) + (threadIdx.x >> 5); r < (long)B * rh2; r += nwarps) {
    const int b = (int)(r / rh2), ry = (int)(r - (long)b * rh2);
    const int n = __ldg(idx + 3 * b), by = __ldg(idx + 3 * b + 1), bx = __ldg(idx + 3 * b + 2);
    const int y = region != 1 ? g.oy + by * g.sy + ry : by * g.obh + ry;
    if (y < 0 || y >= fh) continue;
    int x0 = region != 1 ? g.ox + bx * g.sx : bx * g.obw;
    int x1 = x0 + (region != 1 ? g.bw : g.obw);
    if (region == 2) {
      // union of windows: skip the parts of this window that an active block earlier in
      // the (ascending) list also covers — its left neighbour (columns < overlap), the
      // block above (rows < overlap), above-left / above-right (corner squares).  Those
      // are the entries just before b: scan the last gx + 1 of them, one per lane.
      const int ovy = g.bh - g.sy, ovx = g.bw - g.sx;
      const long key = ((long)n * g.gy + by) * g.gx + bx;
      bool L = false, T = false, TL = false, TR = false;
      for (int k0 = 0; k0 <= g.gx; k0 += 32) {
        const int k = k0 + lane, e = b - 1 - k;
        long kk = -1;
        if (k <= g.gx && e >= 0)
          kk = ((long)__ldg(idx + 3 * e) * g.gy + __ldg(idx + 3 * e + 1)) * g.gx + __ldg(idx + 3 * e + 2);
        L |= __any_sync(0xffffffffu, bx > 0 && kk == key - 1);
        T |= __any_sync(0xffffffffu, by > 0 && kk == key - g.gx);
        TL |= __any_sync(0xffffffffu, by > 0 && bx > 0 && kk == key - g.gx - 1);
        TR |= __any_sync(0xffffffffu, by > 0 && bx < g.gx - 1 && kk == key - g.gx + 1);
      }
      if (ry < ovy && T) continue;
      const int lo = (L || (ry < ovy && TL)) ? ovx : 0, hi = (ry < ovy && TR) ? g.sx : g.bw;
      x1 = x0 + hi;
      x0 += lo;
    }
    x0 = max(x0, 0);
    x1 = min(x1, fw);
    if (x1 <= x0) continue;
    const size_t off = (((size_t)n * fh + y) * fw + x0) * pix_bytes;
    const V* s = reinterpret_cast<const V*>(src + off);
    V* d = reinterpret_cast<V*>(dst + off);
    const int nvec = (x1 - x0) * pix_bytes / VS;
    for (int k = lane; k < nvec; k += 32) d[k] = s[k];
  }
}

// Window regions between a CHANNELS_FIRST (n, c, h, w) tensor and a CHANNELS_LAST staging
// tensor of the same logical dims (dir 0: NCHW -> NHWC, dir 1: NHWC -> NCHW), so the NHWC
// tensor-core paths serve CHANNELS_FIRST callers at sparse cost (only the active windows
// are transposed).  One CTA per (block, window row), transposed through shared memory:
// the NCHW side moves one element per lane along a channel row (16 lanes x 16 channels,
// no index divisions), the NHWC side moves 16-byte vectors of VEC channels along a pixel.
// A pure copy, bit-exact.
template <typename E>
__global__ void __launch_bounds__(256) copy_regions_t_kernel(const E* __restrict__ src, E* __restrict__ dst, Geo g,
                                                             int c, const int32_t* __restrict__ idx,
                                                             const int32_t* __restrict__ count, int cap, int region,
                                                             int dir) {
  constexpr int VEC = 16 / sizeof(E);  // channels per 16-byte vector (host checks c % VEC == 0)
  extern __shared__ __align__(16) uint8_t sm_raw[];
  E* tile = reinterpret_cast<E*>(sm_raw);  // [c][LP]
  const int B = ld_count(count, cap);
  const int rh = region == 1 ? g.obh : g.bh, rw = region == 1 ? g.obw : g.bw;
  const int fh = region == 1 ? g.oh : g.h, fw = region == 1 ? g.ow : g.w;
  const int LP = rw + 1;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // NCHW side: 16 pixels x 16 channels
  const int CV = c / VEC;                                    // NHWC side: vectors per pixel
  for (long item = blockIdx.x; item < (long)B * rh; item += gridDim.x) {
    const int b = (int)(item / rh), ry = (int)(item - (long)b * rh);
    const int n = __ldg(idx + 3 * b), by = __ldg(idx + 3 * b + 1), bx = __ldg(idx + 3 * b + 2);
    const int y = region == 1 ? by * g.obh + ry : g.oy + by * g.sy + ry;
    if (y < 0 || y >= fh) continue;  // uniform per CTA
    int x0 = region == 1 ? bx * g.obw : g.ox + bx * g.sx;
    const int x1 = min(x0 + rw, fw);
    x0 = max(x0, 0);
    const int L = x1 - x0;
    if (L <= 0) continue;
    const size_t plane = (size_t)fh * fw;
    if (dir == 0) {  // NCHW -> tile -> NHWC
      for (int x = tx; x < L; x += 16)
        for (int ch = ty; ch < c; ch += 16) tile[ch * LP + x] = src[((size_t)n * c + ch) * plane + (size_t)y * fw + x0 + x];
      __syncthreads();
      uint4* d = reinterpret_cast<uint4*>(dst + (((size_t)n * fh + y) * fw + x0) * c);
      for (int j = threadIdx.x; j < L * CV; j += blockDim.x) {
        const int x = j / CV, k = j - x * CV;
        __align__(16) E v[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) v[e] = tile[(k * VEC + e) * LP + x];
        d[j] = *reinterpret_cast<const uint4*>(v);
      }
    } else {  // NHWC -> tile -> NCHW
      const uint4* sv = reinterpret_cast<const uint4*>(src + (((size_t)n * fh + y) * fw + x0) * c);
      for (int j = threadIdx.x; j < L * CV; j += blockDim.x) {
        const int x = j / CV, k = j - x * CV;
        const uint4 q = sv[j];
        const E* v = reinterpret_cast<const E*>(&q);
#pragma unroll
        for (int e = 0; e < VEC; ++e) tile[(k * VEC + e) * LP + x] = v[e];
      }
      __syncthreads();
      for (int x = tx; x < L; x += 16)
        for (int ch = ty; ch < c; ch += 16) dst[((size_t)n * c + ch) * plane + (size_t)y * fw + x0 + x] = tile[ch * LP + x];
    }
    __syncthreads();
  }
}

// gather_grad (`blocks.py:162-188`): block table (frame, by, bx) -> stack row, -1 inactive.
__global__ void block_table_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ count, int cap,
                                   Geo g, int32_t* __restrict__ table) {
  const int B = ld_count(count, cap);
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    const int n = idx[3 * b], by = idx[3 * b + 1], bx = idx[3 * b + 2];
    table[((size_t)n * g.gy + by) * g.gx + bx] = b;
  }
}

// Pixel-centric adjoint of gather: every element of dx is written once — the sum of the
// covering blocks' gradient values in ascending stack order (= ascending (by, bx) within
// the frame), starting from zero.  That is the reference's `out += blk` sequence in index
// order, so f32/f64 results are bit-exact and no atomics are needed (bf16 accumulates
// in fp32 and rounds once).
template <typename T>
__global__ void __launch_bounds__(kThreads)
gather_grad_kernel(const T* __restrict__ gblk, Geo g, int c, const int32_t* __restrict__ table,
                   T* __restrict__ dx) {
  using A = typename Acc<T>::type;
  const long total = (long)g.n * g.h * g.w * c;
  for (long i = blockIdx.x * (long)kThreads + threadIdx.x; i < total; i += (long)gridDim.x * kThreads) {
    const int ch = (int)(i % c);
    long p = i / c;
    const int x = (int)(p % g.w);
    p /= g.w;
    const int y = (int)(p % g.h);
    const int n = (int)(p / g.h);
    // covering grid rows: oy + by*sy <= y < oy + by*sy + bh
    const int ry = y - g.oy, rx = x - g.ox;
    int by0 = ry - g.bh + 1 > 0 ? (ry - g.bh + 1 + g.sy - 1) / g.sy : 0;
    int by1 = ry / g.sy;
    int bx0 = rx - g.bw + 1 > 0 ? (rx - g.bw + 1 + g.sx - 1) / g.sx : 0;
    int bx1 = rx / g.sx;
    by1 = min(by1, g.gy - 1);
    bx1 = min(bx1, g.gx - 1);
    T acc = T(0);
    A accf = A(0);
    for (int by = by0; by <= by1; ++by)
      for (int bx = bx0; bx <= bx1; ++bx) {
        const int b = __ldg(table + ((size_t)n * g.gy + by) * g.gx + bx);
        if (b < 0) continue;
        const int wy = ry - by * g.sy, wx = rx - bx * g.sx;
        const T v = __ldg(gblk + (((size_t)b * g.bh + wy) * g.bw + wx) * c + ch);
        if constexpr (sizeof(T) == 2) accf += to_acc(v);
        else acc = acc + v;
      }
    if constexpr (sizeof(T) == 2) dx[i] = from_acc<T>(accf);
    else dx[i] = acc;
  }
}

template <typename E>
__global__ void __launch_bounds__(kThreads)
gather_transpose_kernel(const E* __restrict__ x, Geo g, int c, const int32_t* __restrict__ idx,
                        const int32_t* __restrict__ count, int cap, E* __restrict__ out) {
  const int B = ld_count(count, cap);
  const long per = (long)c * g.bh * g.bw;
  const long total = (long)B * per;
  for (long i = blockIdx.x * (long)kThreads + threadIdx.x; i < total;
       i += (long)gridDim.x * kThreads) {
    const int wx = (int)(i % g.bw);
    long r = i / g.bw;
    const int wy = (int)(r % g.bh);
    r /= g.bh;
    const int ch = (int)(r % c);
    const int b = (int)(r / c);
    const int n = __ldg(idx + 3 * b);
    const int y = g.oy + __ldg(idx + 3 * b + 1) * g.sy + wy;
    const int xx = g.ox + __ldg(idx + 3 * b + 2) * g.sx + wx;
    E v = E(0);
    if (y >= 0 && y < g.h && xx >= 0 && xx < g.w)
      v = __ldg(x + (((size_t)n * g.h + y) * g.w + xx) * c + ch);
    out[i] = v;
  }
}

template <typename T>
__device__ __forceinline__ T add_elem(T a, T b) {
  return a + b;
}
template <>
__device__ __forceinline__ __nv_bfloat16 add_elem<__nv_bfloat16>(__nv_bfloat16 a,
                                                                   __nv_bfloat16 b) {
  return __float2bfloat16_rn(__bfloat162float(a) + __bfloat162float(b));
}

// ADD=false: plain vector copy of each clipped output row; ADD=true: typed add with
// 16-byte vectors of T when VS == 16, else element-wise.
template <int VS, typename T, bool ADD>
__global__ void __launch_bounds__(kThreads)
scatter_rows_kernel(const uint8_t* __restrict__ blk, Geo g, int pix_bytes,
                    const int32_t* __restrict__ idx, const int32_t* __restrict__ count, int cap,
                    uint8_t* __restrict__ dst) {
  using V = typename VecT<VS>::type;
  const int B = ld_count(count, cap);
  const int lane = threadIdx.x & 31;
  const long nwarps = (long)gridDim.x * (kThreads / 32);
  for (long r = blockIdx.x * (long)(kThreads / 32) + (threadIdx.x >> 5); r < (long)B * g.obh;
       r += nwarps) {
    const int b = (int)(r / g.obh), oy = (int)(r - (long)b * g.obh);
    const int n = __ldg(idx + 3 * b), by = __ldg(idx + 3 * b + 1), bx = __ldg(idx + 3 * b + 2);
    const int Y = by * g.obh + oy;
    if (Y >= g.oh) continue;
    const int X0 = bx * g.obw;
    const int npix = min(g.obw, g.ow - X0);
    if (npix <= 0) continue;
    const int nvec = npix * pix_bytes / VS;
    const V* src = reinterpret_cast<const V*>(blk + (size_t)r * g.obw * pix_bytes);
    V* out = reinterpret_cast<V*>(dst + (((size_t)n * g.oh + Y) * g.ow + X0) * pix_bytes);
    for (int k = lane; k < nvec; k += 32) {
      V v = __ldg(src + k);
      if constexpr (ADD) {
        V d = out[k];
        constexpr int ne = VS / sizeof(T);
        T* dv = reinterpret_cast<T*>(&d);
        const T* sv = reinterpret_cast<const T*>(&v);
#pragma unroll
        for (int e = 0; e < ne; ++e) dv[e] = add_elem<T>(dv[e], sv[e]);
        out[k] = d;
      } else {
        out[k] = v;
      }
    }
  }
}

template <typename E>
__global__ void __launch_bounds__(kThreads)
scatter_transpose_kernel(const E* __restrict__ blk, Geo g, int c, const int32_t* __restrict__ idx,
                         const int32_t* __restrict__ count, int cap, E* __restrict__ dst) {
  const int B = ld_count(count, cap);
  const long per = (long)g.obh * g.obw * c;
  const long total = (long)B * per;
  for (long i = blockIdx.x * (long)kThreads + threadIdx.x; i < total;
       i += (long)gridDim.x * kThreads) {
    const int ch = (int)(i % c);
    long r = i / c;
    const int ox = (int)(r % g.obw);
    r /= g.obw;
    const int oy = (int)(r % g.obh);
    const int b = (int)(r / g.obh);
    const int Y = __ldg(idx + 3 * b + 1) * g.obh + oy;
    const int X = __ldg(idx + 3 * b + 2) * g.obw + ox;
    if (Y >= g.oh || X >= g.ow) continue;
    const int n = __ldg(idx + 3 * b);
    dst[(((size_t)n * g.oh + Y) * g.ow + X) * c + ch] =
        blk[(((size_t)b * c + ch) * g.obh + oy) * g.obw + ox];
  }
}

int pick_vec(size_t pix_bytes, const void* a, const void* b) {
  const uintptr_t al = (uintptr_t)a | (uintptr_t)b;
  for (int vs = 16; vs > 1; vs >>= 1)
    if (pix_bytes % vs == 0 && al % vs == 0) return vs;
  return 1;
}

long grid_for(long work_items, int per_cta) {
  long b = (work_items + per_cta - 1) / per_cta;
  long cap = (long)sm_count() * 16;
  if (b > cap) b = cap;
  return b < 1 ? 1 : b;
}

template <int VS>
void launch_gather(const void* x, Geo g, int pix, const int32_t* idx, const int32_t* count,
                   int cap, void* out, cudaStream_t s) {
  gather_rows_kernel<VS><<<(unsigned)grid_for((long)cap * g.bh, kThreads / 32), kThreads, 0, s>>>(
      (const uint8_t*)x, g, pix, idx, count, cap, (uint8_t*)out);
}

template <int VS, typename T, bool ADD>
void launch_scatter(const void* blk, Geo g, int pix, const int32_t* idx, const int32_t* count,
                    int cap, void* dst, cudaStream_t s) {
  scatter_rows_kernel<VS, T, ADD>
      <<<(unsigned)grid_for((long)cap * g.obh, kThreads / 32), kThreads, 0, s>>>(
          (const uint8_t*)blk, g, pix, idx, count, cap, (uint8_t*)dst);
}

template <typename T>
int scatter_add_typed(const void* blk, Geo g, int c, const int32_t* idx, const int32_t* count,
                      int cap, void* dst, cudaStream_t s) {
  const int pix = c * (int)sizeof(T);
  if (pick_vec(pix, blk, dst) == 16)
    launch_scatter<16, T, true>(blk, g, pix, idx, count, cap, dst, s);
  else
    launch_scatter<sizeof(T), T, true>(blk, g, pix, idx, count, cap, dst, s);
  return launch_status("scatter_add");
}

}  // namespace
}  // namespace sbn

using namespace sbn;

extern "C" int sbn_gather(const void* x, int dtype, int c, const sbn_geometry* gp,
                          const int32_t* idx, const int32_t* count, int cap, int transpose,
                          void* out, sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  const int es = dtype_size(dtype);
  SBN_CHECK_ARG(es > 0, SBN_ERR_UNSUPPORTED, "unsupported dtype %d", dtype);
  SBN_CHECK_ARG(c > 0, SBN_ERR_SHAPE, "channels must be > 0");
  if (cap <= 0) return SBN_OK;
  SBN_CHECK_ARG(x && idx && count && out, SBN_ERR_INVALID, "null pointer argument");
  Geo g = to_geo(gp);
  cudaStream_t s = (cudaStream_t)stream;
  if (transpose) {
    const unsigned grid = (unsigned)grid_for((long)cap * c * g.bh * g.bw, kThreads);
    if (es == 2)
      gather_transpose_kernel<uint16_t><<<grid, kThreads, 0, s>>>((const uint16_t*)x, g, c, idx,
                                                                  count, cap, (uint16_t*)out);
    else if (es == 4)
      gather_transpose_kernel<uint32_t><<<grid, kThreads, 0, s>>>((const uint32_t*)x, g, c, idx,
                                                                  count, cap, (uint32_t*)out);
    else
      gather_transpose_kernel<uint64_t><<<grid, kThreads, 0, s>>>((const uint64_t*)x, g, c, idx,
                                                                  count, cap, (uint64_t*)out);
    return launch_status("gather_transpose");
  }
  const int pix = c * es;
  switch (pick_vec(pix, x, out)) {
    case 16: launch_gather<16>(x, g, pix, idx, count, cap, out, s); break;
    case 8: launch_gather<8>(x, g, pix, idx, count, cap, out, s); break;
    case 4: launch_gather<4>(x, g, pix, idx, count, cap, out, s); break;
    default: launch_gather<2>(x, g, pix, idx, count, cap, out, s); break;
  }
  return launch_status("gather");
}

extern "C" int sbn_scatter(const void* blk, int dtype, int c, const sbn_geometry* gp,
                           const int32_t* idx, const int32_t* count, int cap, int add,
                           int transpose, void* dst, sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  const int es = dtype_size(dtype);
  SBN_CHECK_ARG(es > 0, SBN_ERR_UNSUPPORTED, "unsupported dtype %d", dtype);
  SBN_CHECK_ARG(c > 0, SBN_ERR_SHAPE, "channels must be > 0");
  SBN_CHECK_ARG(!(add && transpose), SBN_ERR_UNSUPPORTED, "scatter_transpose has no add mode");
  if (cap <= 0) return SBN_OK;
  SBN_CHECK_ARG(blk && idx && count && dst, SBN_ERR_INVALID, "null pointer argument");
  Geo g = to_geo(gp);
  cudaStream_t s = (cudaStream_t)stream;
  if (transpose) {
    const unsigned grid = (unsigned)grid_for((long)cap * c * g.obh * g.obw, kThreads);
    if (es == 2)
      scatter_transpose_kernel<uint16_t><<<grid, kThreads, 0, s>>>((const uint16_t*)blk, g, c, idx,
                                                                   count, cap, (uint16_t*)dst);
    else if (es == 4)
      scatter_transpose_kernel<uint32_t><<<grid, kThreads, 0, s>>>((const uint32_t*)blk, g, c, idx,
                                                                   count, cap, (uint32_t*)dst);
    else
      scatter_transpose_kernel<uint64_t><<<grid, kThreads, 0, s>>>((const uint64_t*)blk, g, c, idx,
                                                                   count, cap, (uint64_t*)dst);
    return launch_status("scatter_transpose");
  }
  if (add) {
    switch (dtype) {
      case SBN_F32: return scatter_add_typed<float>(blk, g, c, idx, count, cap, dst, s);
      case SBN_F64: return scatter_add_typed<double>(blk, g, c, idx, count, cap, dst, s);
      default: return scatter_add_typed<__nv_bfloat16>(blk, g, c, idx, count, cap, dst, s);
    }
  }
  const int pix = c * es;
  switch (pick_vec(pix, blk, dst)) {
    case 16: launch_scatter<16, uint8_t, false>(blk, g, pix, idx, count, cap, dst, s); break;
    case 8: launch_scatter<8, uint8_t, false>(blk, g, pix, idx, count, cap, dst, s); break;
    case 4: launch_scatter<4, uint8_t, false>(blk, g, pix, idx, count, cap, dst, s); break;
    default: launch_scatter<2, uint8_t, false>(blk, g, pix, idx, count, cap, dst, s); break;
  }
  return launch_status("scatter");
}

extern "C" int sbn_copy_block_regions(const void* src, void* dst, int dtype, int c, const sbn_geometry* gp,
                                      const int32_t* idx, const int32_t* count, int cap, int region,
                                      sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  const int es = dtype_size(dtype);
  SBN_CHECK_ARG(es > 0, SBN_ERR_UNSUPPORTED, "unsupported dtype %d", dtype);
  SBN_CHECK_ARG(c > 0, SBN_ERR_SHAPE, "channels must be > 0");
  SBN_CHECK_ARG(region >= 0 && region <= 2, SBN_ERR_INVALID,
                "region must be 0 (window), 1 (output) or 2 (union of windows)");
  if (region == 2 && (2 * (gp->bh - gp->sy) > gp->bh || 2 * (gp->bw - gp->sx) > gp->bw)) region = 0;
  if (cap <= 0) return SBN_OK;
  SBN_CHECK_ARG(src && dst && idx && count, SBN_ERR_INVALID, "null pointer argument");
  Geo g = to_geo(gp);
  cudaStream_t s = (cudaStream_t)stream;
  const int pix = c * es;
  const long rows = (long)cap * (region != 1 ? g.bh : g.obh);
  const unsigned grid = (unsigned)grid_for(rows * 32, kThreads);
  switch (pick_vec(pix, src, dst)) {
    case 16: copy_regions_kernel<16><<<grid, kThreads, 0, s>>>((const uint8_t*)src, (uint8_t*)dst, g, pix, idx, count, cap, region); break;
    case 8: copy_regions_kernel<8><<<grid, kThreads, 0, s>>>((const uint8_t*)src, (uint8_t*)dst, g, pix, idx, count, cap, region); break;
    case 4: copy_regions_kernel<4><<<grid, kThreads, 0, s>>>((const uint8_t*)src, (uint8_t*)dst, g, pix, idx, count, cap, region); break;
    default: copy_regions_kernel<2><<<grid, kThreads, 0, s>>>((const uint8_t*)src, (uint8_t*)dst, g, pix, idx, count, cap, region); break;
  }
  return launch_status("copy_block_regions");
}

extern "C" int sbn_copy_block_regions_t(const void* src, void* dst, int dtype, int c, const sbn_geometry* gp,
                                        const int32_t* idx, const int32_t* count, int cap, int region, int dir,
                                        sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  const int es = dtype_size(dtype);
  SBN_CHECK_ARG(es > 0, SBN_ERR_UNSUPPORTED, "unsupported dtype %d", dtype);
  SBN_CHECK_ARG(c > 0, SBN_ERR_SHAPE, "channels must be > 0");
  SBN_CHECK_ARG(region == 0 || region == 1, SBN_ERR_INVALID, "region must be 0 (window) or 1 (output)");
  SBN_CHECK_ARG(dir == 0 || dir == 1, SBN_ERR_INVALID, "dir must be 0 (NCHW -> NHWC) or 1 (NHWC -> NCHW)");
  if (cap <= 0) return SBN_OK;
  SBN_CHECK_ARG(src && dst && idx && count, SBN_ERR_INVALID, "null pointer argument");
  Geo g = to_geo(gp);
  const int rw = region == 1 ? g.obw : g.bw;
  const size_t smem = (size_t)c * (rw + 1) * es;
  SBN_CHECK_ARG(smem <= 96 * 1024, SBN_ERR_UNSUPPORTED, "row tile of %zu bytes too large", smem);
  SBN_CHECK_ARG((c * es) % 16 == 0 && ((uintptr_t)src % 16) == 0 && ((uintptr_t)dst % 16) == 0, SBN_ERR_UNSUPPORTED,
                "channels-first window copy needs 16-byte pixel rows (c * elem_size %% 16 == 0)");
  cudaStream_t s = (cudaStream_t)stream;
  const long items = (long)cap * (region == 1 ? g.obh : g.bh);
  const unsigned grid = (unsigned)(items < (long)sm_count() * 8 ? (items < 1 ? 1 : items) : (long)sm_count() * 8);
#define LAUNCH(E)                                                                                          \
  {                                                                                                        \
    auto kern = copy_regions_t_kernel<E>;                                                                  \
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    kern<<<grid, 256, smem, s>>>((const E*)src, (E*)dst, g, c, idx, count, cap, region, dir);              \
  }
  if (es == 2) LAUNCH(uint16_t) else if (es == 4) LAUNCH(uint32_t) else LAUNCH(uint64_t)
#undef LAUNCH
  return launch_status("copy_block_regions_t");
}

extern "C" size_t sbn_gather_grad_workspace(const sbn_geometry* gp) {
  if (!gp) return 0;
  return (size_t)gp->n * gp->gy * gp->gx * sizeof(int32_t);
}

extern "C" int sbn_gather_grad(const void* gblk, int dtype, int c, const sbn_geometry* gp, const int32_t* idx,
                               const int32_t* count, int cap, void* dx, void* ws, size_t ws_bytes,
                               sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  const int es = dtype_size(dtype);
  SBN_CHECK_ARG(es > 0, SBN_ERR_UNSUPPORTED, "unsupported dtype %d", dtype);
  SBN_CHECK_ARG(c > 0, SBN_ERR_SHAPE, "channels must be > 0");
  SBN_CHECK_ARG(dx && idx && count, SBN_ERR_INVALID, "null pointer argument");
  SBN_CHECK_ARG(ws && ws_bytes >= sbn_gather_grad_workspace(gp), SBN_ERR_WORKSPACE,
                "gather_grad needs a %zu-byte workspace", sbn_gather_grad_workspace(gp));
  SBN_CHECK_ARG(cap <= 0 || gblk, SBN_ERR_INVALID, "null block gradient");
  Geo g = to_geo(gp);
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* table = (int32_t*)ws;
  cudaMemsetAsync(table, 0xFF, sbn_gather_grad_workspace(gp), s);
  if (cap > 0) {
    block_table_kernel<<<(unsigned)grid_for(cap, kThreads), kThreads, 0, s>>>(idx, count, cap, g, table);
    st = launch_status("gather_grad_table");
    if (st) return st;
  }
  const unsigned grid = (unsigned)grid_for((long)g.n * g.h * g.w * c, kThreads);
  switch (dtype) {
    case SBN_F32: gather_grad_kernel<float><<<grid, kThreads, 0, s>>>((const float*)gblk, g, c, table, (float*)dx); break;
    case SBN_F64: gather_grad_kernel<double><<<grid, kThreads, 0, s>>>((const double*)gblk, g, c, table, (double*)dx); break;
    default: gather_grad_kernel<__nv_bfloat16><<<grid, kThreads, 0, s>>>((const __nv_bfloat16*)gblk, g, c, table, (__nv_bfloat16*)dx); break;
  }
  return launch_status("gather_grad");
}
