// Mask kernels: reduce_mask (ordered active-block list), downsample_mask, in_bounds_map.
//
// reduce_mask restates reference `tiling.py:120-160` (window sums + argwhere) as ONE
// kernel launch:
//   * one CTA per tile = one block row (frame n, block-row by); tiles are taken in
//     ascending order through an atomic ticket so every earlier tile is resident or done;
//   * the CTA column-reduces the bh mask rows its window row spans (coalesced byte
//     loads, one pass over the mask), then window-reduces columns per block;
//   * MAX: count > 0, AVG: count/(bh*bw) >= thr - 1e-12 in float64 (as the reference);
//   * warp-ballot + popc compaction gives each active block its rank inside the tile;
//     the tile's global offset comes from a decoupled look-back over earlier tiles, so
//     the output is exactly argwhere's ascending (n, by, bx) order without a sort;
//   * the last CTA to finish zeroes the workspace, so it can be reused (and captured
//     in a CUDA graph) without a memset.
#include "common.cuh"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace sbn {
namespace {

constexpr int kMaskThreads = 256;
constexpr int kColBuf = 4096;  // column-sum buffer (ints) per chunk

struct MaskWs {
  unsigned int ticket;
  unsigned int done;
  unsigned long long status[1];  // [tiles] : (flag << 32) | value
};

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__device__ __forceinline__ int block_sum(int v, int* red) {
  // 256-thread block reduction; result broadcast to all threads
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int t = 0;
#pragma unroll
  for (int i = 0; i < kMaskThreads / 32; ++i) t += red[i];
  return t;
}

__global__ void __launch_bounds__(kMaskThreads)
reduce_mask_kernel(const uint8_t* __restrict__ mask, Geo g, int pool, double thr, int chunk,
                   int32_t* __restrict__ idx, int32_t* __restrict__ count, MaskWs* ws, int tiles) {
  // dependents launched with PDL (the conv / unit kernels) may start their prologues and
  // weight copies now; they read the list only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ int colsum[kColBuf];
  __shared__ int red[kMaskThreads / 32];
  __shared__ int woff[kMaskThreads / 32];
  __shared__ unsigned int s_tile;
  __shared__ int s_prefix;
  __shared__ int s_last;
  extern __shared__ uint8_t flags[];  // [gx]

  if (threadIdx.x == 0) s_tile = atomicAdd(&ws->ticket, 1u);
  __syncthreads();
  const int tile = (int)s_tile;
  const int n = tile / g.gy;
  const int by = tile - n * g.gy;

  const int wy0 = g.oy + by * g.sy;
  const int y0 = max(wy0, 0), y1 = min(wy0 + g.bh, g.h);
  const uint8_t* mrow = mask + (size_t)n * g.h * g.w;
  const double area = (double)g.bh * (double)g.bw;

  int tile_count = 0;
  const bool vec = ((g.w & 3) == 0) && ((reinterpret_cast<uintptr_t>(mask) & 3) == 0) && (y1 - y0) < 256;
  for (int bx0 = 0; bx0 < g.gx; bx0 += chunk) {
    const int bx1 = min(bx0 + chunk, g.gx);
    int cx0 = max(g.ox + bx0 * g.sx, 0);
    const int cx1 = min(g.ox + (bx1 - 1) * g.sx + g.bw, g.w);
    __syncthreads();
    if (vec) {
      // 4 columns per thread: a 32-bit word of 0/1 bytes is four packed column counters
      // (no carry between bytes for < 256 rows); every row load is issued before use.
      cx0 &= ~3;
      const int nw = (cx1 - cx0 + 3) >> 2;
      const uint32_t* base = reinterpret_cast<const uint32_t*>(mrow) + (cx0 >> 2);
      const int wpr = g.w >> 2;
      for (int wi = threadIdx.x; wi < nw; wi += kMaskThreads) {
        uint32_t acc = 0;
        int y = y0;
        for (; y + 8 <= y1; y += 8) {
          uint32_t v[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) v[r] = __ldg(base + (size_t)(y + r) * wpr + wi);
#pragma unroll
          for (int r = 0; r < 8; ++r) acc += v[r];
        }
        for (; y < y1; ++y) acc += __ldg(base + (size_t)y * wpr + wi);
        const int x = cx0 + 4 * wi;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (x + e < cx1) colsum[x + e - cx0] = (acc >> (8 * e)) & 0xffu;
      }
    } else {
      for (int x = cx0 + (int)threadIdx.x; x < cx1; x += kMaskThreads) {
        int sum = 0;
        for (int y = y0; y < y1; ++y) sum += __ldg(mrow + (size_t)y * g.w + x);
        colsum[x - cx0] = sum;
      }
    }
    __syncthreads();
    int local = 0;
    for (int bx = bx0 + (int)threadIdx.x; bx < bx1; bx += kMaskThreads) {
      const int wx0 = g.ox + bx * g.sx;
      const int xa = max(wx0, 0), xb = min(wx0 + g.bw, g.w);
      int cnt = 0;
      if (y1 > y0)
        for (int x = xa; x < xb; ++x) cnt += colsum[x - cx0];
      bool on;
      if (pool == SBN_POOL_MAX) on = cnt > 0;
      else on = ((double)cnt / area) >= thr - 1e-12;
      flags[bx] = on ? 1 : 0;
      local += on ? 1 : 0;
    }
    tile_count += block_sum(local, red);
  }

  // ---- decoupled look-back: exclusive prefix of active blocks over earlier tiles.
  //      Warp 0 inspects 32 predecessors per round (lane i -> tile - 1 - i): it sums the
  //      published aggregates up to the nearest inclusive prefix, retrying the window
  //      while any needed predecessor has not published yet.
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (lane == 0)
      atomicExch(&ws->status[tile], ((tile == 0 ? 2ull : 1ull) << 32) | (unsigned)tile_count);
    int prefix = 0;
    int j = tile - 1;
    while (j >= 0) {
      const int k = j - lane;
      unsigned long long st = k >= 0 ? ld_volatile(&ws->status[k]) : (2ull << 32);
      const unsigned flag = (unsigned)(st >> 32);
      const unsigned incl = __ballot_sync(0xffffffffu, flag == 2);
      const unsigned none = __ballot_sync(0xffffffffu, flag == 0);
      const int first = incl ? __ffs(incl) - 1 : 31;
      const unsigned need = first >= 31 ? 0xffffffffu : ((2u << first) - 1u);
      if (none & need) {
        __nanosleep(32);
        continue;
      }
      int v = lane <= first ? (int)(unsigned)(st & 0xffffffffull) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      prefix += v;
      if (incl) break;
      j -= 32;
    }
    if (lane == 0) {
      if (tile > 0) {
        __threadfence();
        atomicExch(&ws->status[tile], (2ull << 32) | (unsigned)(prefix + tile_count));
      }
      s_prefix = prefix;
      if (tile == tiles - 1) *count = prefix + tile_count;
    }
  }
  __syncthreads();

  // ---- ordered compaction: ballot/popc ranks inside the tile
  int base = s_prefix;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int bx0 = 0; bx0 < g.gx; bx0 += kMaskThreads) {
    const int bx = bx0 + (int)threadIdx.x;
    const bool on = bx < g.gx && flags[bx];
    const unsigned bal = __ballot_sync(0xffffffffu, on);
    if (lane == 0) woff[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int i = 0; i < kMaskThreads / 32; ++i) {
      before += (i < warp) ? woff[i] : 0;
      total += woff[i];
    }
    if (on) {
      const int pos = base + before + __popc(bal & ((1u << lane) - 1u));
      idx[3 * pos + 0] = n;
      idx[3 * pos + 1] = by;
      idx[3 * pos + 2] = bx;
    }
    base += total;
    __syncthreads();
  }

  // ---- self-cleaning workspace: the last CTA out resets ticket/done/status
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = (atomicAdd(&ws->done, 1u) == (unsigned)(tiles - 1));
  }
  __syncthreads();
  if (s_last) {
    for (int t = threadIdx.x; t < tiles; t += kMaskThreads) ws->status[t] = 0ull;
    if (threadIdx.x == 0) {
      ws->ticket = 0u;
      ws->done = 0u;
    }
    __threadfence();
  }
}

// Moderate problems: ONE thread-block cluster (kClusterMax CTAs).  CTA r owns a contiguous
// range of block rows; the per-CTA active counts are exchanged through distributed shared
// memory (CTA 0's smem) with two cluster barriers — no global atomics, no look-back, no
// workspace.  Each thread column-reduces one (block row, 4-column word) item with all of
// its row loads in flight.
constexpr int kClusterMax = 16;
constexpr int kClusterThreads = 256;

__global__ void __launch_bounds__(kClusterThreads, 1)
reduce_mask_cluster_kernel(const uint8_t* __restrict__ mask, Geo g, int pool, double thr, int per,
                           int32_t* __restrict__ idx, int32_t* __restrict__ count, int vec) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // (see reduce_mask_kernel)
  // launched with PDL itself (under the previous kernel's tail): the mask may be that
  // kernel's output
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ int s_cnt[kClusterMax];
  __shared__ int wsum[kClusterThreads / 32];
  __shared__ int s_base;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int ncl = (int)cl.num_blocks();
  const int tiles = g.n * g.gy;
  const int t0 = rank * per, t1 = min(t0 + per, tiles);
  const int mt = max(t1 - t0, 0);
  int* colsum = reinterpret_cast<int*>(sm);                 // [per][w]
  uint8_t* flag = sm + (size_t)per * g.w * 4;                // [per * gx]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double area = (double)g.bh * (double)g.bw;
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // "I have started"

  if (vec) {
    const int wpr = g.w >> 2;
    for (int i = tid; i < mt * wpr; i += kClusterThreads) {
      const int tl = i / wpr, wi = i - tl * wpr;
      const int t = t0 + tl;
      const int n = t / g.gy, by = t - n * g.gy;
      const int wy0 = g.oy + by * g.sy;
      const int y0 = max(wy0, 0), y1 = min(wy0 + g.bh, g.h);
      const uint32_t* base = reinterpret_cast<const uint32_t*>(mask + (size_t)n * g.h * g.w) + wi;
      uint32_t acc = 0;
      for (int y = y0; y < y1; y += 16) {
        uint32_t v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = (y + r < y1) ? __ldg(base + (size_t)(y + r) * wpr) : 0u;
#pragma unroll
        for (int r = 0; r < 16; ++r) acc += v[r];
      }
      int* cs = colsum + (size_t)tl * g.w + 4 * wi;
#pragma unroll
      for (int e = 0; e < 4; ++e) cs[e] = (acc >> (8 * e)) & 0xffu;
    }
  } else {
    for (int i = tid; i < mt * g.w; i += kClusterThreads) {
      const int tl = i / g.w, x = i - tl * g.w;
      const int t = t0 + tl;
      const int n = t / g.gy, by = t - n * g.gy;
      const int wy0 = g.oy + by * g.sy;
      const int y0 = max(wy0, 0), y1 = min(wy0 + g.bh, g.h);
      int acc = 0;
      for (int y = y0; y < y1; ++y) acc += __ldg(mask + ((size_t)n * g.h + y) * g.w + x);
      colsum[i] = acc;
    }
  }
  __syncthreads();
  const int T = mt * g.gx;
  for (int c = tid; c < T; c += kClusterThreads) {
    const int tl = c / g.gx, bx = c - tl * g.gx;
    const int t = t0 + tl;
    const int by = t % g.gy;
    const int wy0 = g.oy + by * g.sy;
    const bool rows = max(wy0, 0) < min(wy0 + g.bh, g.h);
    const int wx0 = g.ox + bx * g.sx;
    const int xa = max(wx0, 0), xb = min(wx0 + g.bw, g.w);
    int cnt = 0;
    if (rows)
      for (int x = xa; x < xb; ++x) cnt += colsum[(size_t)tl * g.w + x];
    flag[c] = pool == SBN_POOL_MAX ? (cnt > 0) : (((double)cnt / area) >= thr - 1e-12);
  }
  __syncthreads();
  // per-thread contiguous run of candidates -> in-CTA exclusive scan
  const int pc = (T + kClusterThreads - 1) / kClusterThreads;
  const int c0 = min(tid * pc, T), c1 = min(c0 + pc, T);
  int mine = 0;
  for (int c = c0; c < c1; ++c) mine += flag[c];
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  // every CTA of the cluster must have started before CTA 0's shared memory is written
  // remotely (arrived right at kernel entry, so this wait is normally already satisfied)
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  if (warp == 0) {
    const int ws = lane < kClusterThreads / 32 ? wsum[lane] : 0;
    int wi = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += v;
    }
    if (lane < kClusterThreads / 32) wsum[lane] = wi - ws;
    if (lane == 31) {  // CTA total -> CTA 0's table (distributed shared memory)
      int* remote = cl.map_shared_rank(s_cnt, 0);
      remote[rank] = wi;
    }
  }
  cl.sync();
  if (tid == 0) {
    const int* table = cl.map_shared_rank(s_cnt, 0);
    int base = 0, total = 0;
    for (int r = 0; r < ncl; ++r) {
      const int v = table[r];
      if (r < rank) base += v;
      total += v;
    }
    s_base = base;
    if (rank == 0) *count = total;
  }
  cl.sync();  // CTA 0's table stays alive until everyone has read it
  int pos = s_base + wsum[warp] + incl - mine;
  for (int c = c0; c < c1; ++c) {
    if (flag[c]) {
      const int tl = c / g.gx, bx = c - tl * g.gx;
      const int t = t0 + tl;
      const int n = t / g.gy, by = t - n * g.gy;
      idx[3 * pos] = n;
      idx[3 * pos + 1] = by;
      idx[3 * pos + 2] = bx;
      ++pos;
    }
  }
}

// Large problems (many block rows, e.g. 64 frames): CTA r (in ticket order) owns `per`
// consecutive block rows — the cluster kernel's column-reduce / window-reduce / in-CTA scan
// over all of its rows with every row load of a (row, 4-column word) item in flight — and
// its count joins the ordered list through the decoupled look-back of reduce_mask_kernel
// over the earlier ranges (ws->status[range]).  A few hundred CTAs with several block rows
// each instead of one CTA (ticket, look-back step, done atomic) per block row.
constexpr int kRangeThreads = 256;

__global__ void __launch_bounds__(kRangeThreads)
reduce_mask_ranges_kernel(const uint8_t* __restrict__ mask, Geo g, int pool, double thr, int per,
                          int32_t* __restrict__ idx, int32_t* __restrict__ count, MaskWs* ws, int ranges,
                          int vec, unsigned long long* tr) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // (see reduce_mask_kernel)
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ int wsum[kRangeThreads / 32];
  __shared__ unsigned int s_range;
  __shared__ int s_prefix, s_total, s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long tt0 = tr ? gtimer() : 0;
  if (tid == 0) s_range = atomicAdd(&ws->ticket, 1u);
  __syncthreads();
  const int range = (int)s_range;
  unsigned long long* trc = tr && tid == 0 ? tr + (size_t)range * 8 : nullptr;
  if (trc) { trc[0] = tt0; trc[1] = gtimer(); }
  const int tiles = g.n * g.gy;
  const int t0 = range * per, t1 = min(t0 + per, tiles);
  const int mt = max(t1 - t0, 0);
  int* colsum = reinterpret_cast<int*>(sm);   // [per][w]
  uint8_t* flag = sm + (size_t)per * g.w * 4;  // [per * gx]
  const double area = (double)g.bh * (double)g.bw;

  if (vec) {
    const int wpr = g.w >> 2;
    for (int i = tid; i < mt * wpr; i += kRangeThreads) {
      const int tl = i / wpr, wi = i - tl * wpr;
      const int t = t0 + tl;
      const int n = t / g.gy, by = t - n * g.gy;
      const int wy0 = g.oy + by * g.sy;
      const int y0 = max(wy0, 0), y1 = min(wy0 + g.bh, g.h);
      const uint32_t* base = reinterpret_cast<const uint32_t*>(mask + (size_t)n * g.h * g.w) + wi;
      uint32_t acc = 0;
      for (int y = y0; y < y1; y += 16) {
        uint32_t v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = (y + r < y1) ? __ldg(base + (size_t)(y + r) * wpr) : 0u;
#pragma unroll
        for (int r = 0; r < 16; ++r) acc += v[r];
      }
      int* cs = colsum + (size_t)tl * g.w + 4 * wi;
#pragma unroll
      for (int e = 0; e < 4; ++e) cs[e] = (acc >> (8 * e)) & 0xffu;
    }
  } else {
    for (int i = tid; i < mt * g.w; i += kRangeThreads) {
      const int tl = i / g.w, x = i - tl * g.w;
      const int t = t0 + tl;
      const int n = t / g.gy, by = t - n * g.gy;
      const int wy0 = g.oy + by * g.sy;
      const int y0 = max(wy0, 0), y1 = min(wy0 + g.bh, g.h);
      int acc = 0;
      for (int y = y0; y < y1; ++y) acc += __ldg(mask + ((size_t)n * g.h + y) * g.w + x);
      colsum[i] = acc;
    }
  }
  __syncthreads();
  if (trc) trc[2] = gtimer();
  const int T = mt * g.gx;
  for (int c = tid; c < T; c += kRangeThreads) {
    const int tl = c / g.gx, bx = c - tl * g.gx;
    const int by = (t0 + tl) % g.gy;
    const int wy0 = g.oy + by * g.sy;
    const bool rows = max(wy0, 0) < min(wy0 + g.bh, g.h);
    const int wx0 = g.ox + bx * g.sx;
    const int xa = max(wx0, 0), xb = min(wx0 + g.bw, g.w);
    int cnt = 0;
    if (rows)
      for (int x = xa; x < xb; ++x) cnt += colsum[(size_t)tl * g.w + x];
    flag[c] = pool == SBN_POOL_MAX ? (cnt > 0) : (((double)cnt / area) >= thr - 1e-12);
  }
  __syncthreads();
  // per-thread contiguous run of candidates -> in-CTA exclusive scan
  const int pc = (T + kRangeThreads - 1) / kRangeThreads;
  const int c0 = min(tid * pc, T), c1 = min(c0 + pc, T);
  int mine = 0;
  for (int c = c0; c < c1; ++c) mine += flag[c];
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (trc) trc[3] = gtimer();
  if (warp == 0) {
    const int w_s = lane < kRangeThreads / 32 ? wsum[lane] : 0;
    int wi = w_s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += v;
    }
    if (lane < kRangeThreads / 32) wsum[lane] = wi - w_s;
    if (lane == 31) s_total = wi;
  }
  __syncthreads();
  // decoupled look-back over the earlier ranges with the WHOLE CTA: thread i inspects range
  // j - i, so each round covers 256 predecessors (the one-warp look-back of
  // reduce_mask_kernel advances 32 per memory round trip, which over hundreds of ranges
  // published at about the same time becomes a chain of round trips)
  __shared__ int s_incl[kRangeThreads / 32], s_none[kRangeThreads / 32], s_val[kRangeThreads / 32];
  const int total = s_total;
  if (tid == 0) atomicExch(&ws->status[range], ((range == 0 ? 2ull : 1ull) << 32) | (unsigned)total);
  int prefix = 0;
  for (int j = range - 1; j >= 0;) {
    const int k = j - tid;
    const unsigned long long st = k >= 0 ? ld_volatile(&ws->status[k]) : (2ull << 32);
    const unsigned fl = (unsigned)(st >> 32);
    const unsigned inc_b = __ballot_sync(0xffffffffu, fl == 2);
    const unsigned non_b = __ballot_sync(0xffffffffu, fl == 0);
    if (lane == 0) {
      s_incl[warp] = inc_b ? 32 * warp + __ffs(inc_b) - 1 : 1 << 30;  // nearest inclusive in this warp
      s_none[warp] = non_b ? 32 * warp + __ffs(non_b) - 1 : 1 << 30;  // nearest missing
    }
    __syncthreads();
    int first = 1 << 30, miss = 1 << 30;
#pragma unroll
    for (int w = 0; w < kRangeThreads / 32; ++w) {
      first = min(first, s_incl[w]);
      miss = min(miss, s_none[w]);
    }
    const int upto = first < kRangeThreads ? first : kRangeThreads - 1;
    __syncthreads();
    if (miss <= upto) {  // a needed predecessor has not published yet: retry the window
      __nanosleep(64);
      continue;
    }
    int v = tid <= upto ? (int)(unsigned)(st & 0xffffffffull) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_val[warp] = v;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kRangeThreads / 32; ++w) prefix += s_val[w];
    __syncthreads();
    if (first < kRangeThreads) break;
    j -= kRangeThreads;
  }
  if (tid == 0) {
    if (range > 0) {
      __threadfence();
      atomicExch(&ws->status[range], (2ull << 32) | (unsigned)(prefix + total));
    }
    s_prefix = prefix;
    if (range == ranges - 1) *count = prefix + total;
  }
  __syncthreads();
  if (trc) trc[4] = gtimer();
  int pos = s_prefix + wsum[warp] + incl - mine;
  for (int c = c0; c < c1; ++c) {
    if (flag[c]) {
      const int tl = c / g.gx, bx = c - tl * g.gx;
      const int t = t0 + tl;
      const int n = t / g.gy, by = t - n * g.gy;
      idx[3 * pos] = n;
      idx[3 * pos + 1] = by;
      idx[3 * pos + 2] = bx;
      ++pos;
    }
  }
  // self-cleaning workspace: the last CTA out resets ticket / done / status
  if (tid == 0) {
    __threadfence();
    s_last = (atomicAdd(&ws->done, 1u) == (unsigned)(ranges - 1));
  }
  __syncthreads();
  if (trc) trc[5] = gtimer();
  if (s_last) {
    for (int t = tid; t < ranges; t += kRangeThreads) ws->status[t] = 0ull;
    if (tid == 0) {
      ws->ticket = 0u;
      ws->done = 0u;
    }
    __threadfence();
  }
}

__global__ void downsample_kernel(const uint8_t* __restrict__ in, int n, int h, int w, int f,
                                  int oh, int ow, uint8_t* __restrict__ out, int vec4) {
  const long total = (long)n * oh * ow;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int ox = (int)(i % ow);
    const long r = i / ow;
    const int oy = (int)(r % oh);
    const int fr = (int)(r / oh);
    const int ya = oy * f, yb = min(ya + f, h), xa = ox * f, xb = min(xa + f, w);
    const uint8_t* p = in + (size_t)fr * h * w;
    // no early exit: every row's loads are independent, so they stay in flight together
    // (an any-found exit made the f rows f serial round trips)
    uint32_t m4 = 0;
    if (vec4) {  // 4-byte words: w, f and the base are multiples of 4 (so are xa and xb)
      for (int y = ya; y < yb; ++y)
        for (int x = xa; x < xb; x += 4) m4 = __vmaxu4(m4, __ldg(reinterpret_cast<const uint32_t*>(p + (size_t)y * w + x)));
      m4 = max(max(m4 & 0xffu, (m4 >> 8) & 0xffu), max((m4 >> 16) & 0xffu, m4 >> 24));
    } else {
      for (int y = ya; y < yb; ++y)
        for (int x = xa; x < xb; ++x) m4 = max(m4, (uint32_t)__ldg(p + (size_t)y * w + x));
    }
    out[i] = (uint8_t)m4;
  }
}

__global__ void in_bounds_kernel(Geo g, const int32_t* __restrict__ idx,
                                 const int32_t* __restrict__ count, int cap,
                                 uint8_t* __restrict__ out) {
  const int B = ld_count(count, cap);
  const long per = (long)g.bh * g.bw;
  const long total = (long)B * per;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int b = (int)(i / per);
    const int r = (int)(i - (long)b * per);
    const int wy = r / g.bw, wx = r - wy * g.bw;
    const int y = g.oy + idx[3 * b + 1] * g.sy + wy;
    const int x = g.ox + idx[3 * b + 2] * g.sx + wx;
    out[i] = (y >= 0 && y < g.h && x >= 0 && x < g.w) ? 1 : 0;
  }
}

}  // namespace
}  // namespace sbn

using namespace sbn;

extern "C" size_t sbn_reduce_mask_workspace(const sbn_geometry* g) {
  if (!g) return 0;
  const size_t tiles = (size_t)g->n * (size_t)g->gy;
  return 16 + 8 * (tiles > 0 ? tiles : 1);
}

// The cluster kernel (one cluster, up to 16 CTAs) wins only while each CTA has a few block
// rows; beyond that the one-CTA-per-row look-back kernel is faster (tools/reduce_mask_time.py:
// 8 x 400x350, 16x16 blocks: 20.6 -> 9.1 us; 800x700, 8x8: 9.5 -> 6.8 us; 800x700, 16x16
// (4 rows / CTA) stays on the cluster: 5.6 us vs 6.7).
constexpr int kClusterMaxRowsPerCta = 4;

extern "C" int sbn_reduce_mask(const uint8_t* mask, const sbn_geometry* gp, int pool,
                               double threshold, int32_t* idx, int32_t* count, void* ws,
                               size_t ws_bytes, sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  SBN_CHECK_ARG(pool == SBN_POOL_MAX || pool == SBN_POOL_AVG, SBN_ERR_INVALID, "bad pool mode %d",
                pool);
  SBN_CHECK_ARG(mask && idx && count, SBN_ERR_INVALID, "null pointer argument");
  SBN_CHECK_ARG(ws_bytes >= sbn_reduce_mask_workspace(gp) && ws, SBN_ERR_WORKSPACE,
                "reduce_mask workspace too small (%zu < %zu)", ws_bytes,
                sbn_reduce_mask_workspace(gp));
  cudaStream_t s = (cudaStream_t)stream;
  Geo g = to_geo(gp);
  const long tiles = (long)g.n * g.gy;
  if (tiles == 0) {
    cudaMemsetAsync(count, 0, sizeof(int32_t), s);
    return launch_status("reduce_mask(empty)");
  }
  SBN_CHECK_ARG(tiles < (1l << 31), SBN_ERR_INVALID, "too many block rows");
  {
    // one cluster of up to 16 CTAs when each CTA's block rows fit its shared memory
    int cl = (int)(tiles < kClusterMax ? tiles : kClusterMax);
    const int per = (int)((tiles + cl - 1) / cl);
    cl = (int)((tiles + per - 1) / per);
    const size_t smem = (size_t)per * g.w * 4 + (size_t)per * g.gx;
    if (smem <= 160 * 1024 && per <= kClusterMaxRowsPerCta) {
      const int vec = ((g.w & 3) == 0) && (((uintptr_t)mask & 3) == 0) && g.bh < 256;
      static PerDeviceOnce attr;
      attr([] {
        cudaFuncSetAttribute(reduce_mask_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             160 * 1024 + 16);
        cudaFuncSetAttribute(reduce_mask_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      });
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cl);
      cfg.blockDim = dim3(kClusterThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = (debug_flags() & kDebugNoMaskPdl) ? 0 : 1;
      cfg.numAttrs = 2;
      if (cudaLaunchKernelEx(&cfg, reduce_mask_cluster_kernel, mask, g, pool, threshold, per, idx,
                             count, vec) == cudaSuccess)
        return launch_status("reduce_mask(cluster)");
      cudaGetLastError();  // cluster launch refused: fall through to the look-back kernel
    }
  }
  {
    // several block rows per CTA (about four CTAs per SM), ordered by the look-back
    long per = (tiles + 4L * sm_count() - 1) / (4L * sm_count());
    if (per < 1) per = 1;
    const size_t smem = (size_t)per * g.w * 4 + (size_t)per * g.gx;
    // (at one row per CTA the row kernel below is as fast or faster: tools/reduce_mask_ab.py)
    if (per >= 2 && smem <= 48 * 1024 && !(debug_flags() & kDebugRowReduceMask)) {
      const int vec = ((g.w & 3) == 0) && (((uintptr_t)mask & 3) == 0) && g.bh < 256;
      const int ranges = (int)((tiles + per - 1) / per);
      reduce_mask_ranges_kernel<<<(unsigned)ranges, kRangeThreads, smem, s>>>(
          mask, g, pool, threshold, (int)per, idx, count, reinterpret_cast<MaskWs*>(ws), ranges, vec,
          trace_buffer());
      return launch_status("reduce_mask(ranges)");
    }
  }
  // chunk of block columns whose column range fits the column-sum buffer
  int chunk = g.gx;
  if ((long)(chunk - 1) * g.sx + g.bw + 3 > kColBuf) chunk = (kColBuf - 3 - g.bw) / g.sx + 1;
  SBN_CHECK_ARG(chunk >= 1, SBN_ERR_UNSUPPORTED, "block width %d too large for reduce_mask", g.bw);
  const size_t dyn = (size_t)g.gx;
  SBN_CHECK_ARG(dyn <= 48 * 1024 - 20 * 1024, SBN_ERR_UNSUPPORTED, "grid width %d too large", g.gx);
  reduce_mask_kernel<<<(unsigned)tiles, kMaskThreads, dyn, s>>>(
      mask, g, pool, threshold, chunk, idx, count, reinterpret_cast<MaskWs*>(ws), (int)tiles);
  return launch_status("reduce_mask");
}

extern "C" int sbn_downsample_mask(const uint8_t* in, int n, int h, int w, int factor,
                                   uint8_t* out, sbn_stream_t stream) {
  SBN_CHECK_ARG(factor >= 1, SBN_ERR_INVALID, "factor must be >= 1, got %d", factor);
  SBN_CHECK_ARG(n >= 0 && h > 0 && w > 0, SBN_ERR_SHAPE, "bad mask dims");
  const int oh = (h + factor - 1) / factor, ow = (w + factor - 1) / factor;
  const long total = (long)n * oh * ow;
  if (total == 0) return SBN_OK;
  const int threads = 256;
  long blocks = (total + threads - 1) / threads;
  if (blocks > (long)sm_count() * 32) blocks = (long)sm_count() * 32;
  const int vec4 = (w % 4 == 0) && (factor % 4 == 0) && ((uintptr_t)in % 4 == 0);
  downsample_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(in, n, h, w, factor,
                                                                           oh, ow, out, vec4);
  return launch_status("downsample_mask");
}

extern "C" int sbn_in_bounds(const sbn_geometry* gp, const int32_t* idx, const int32_t* count,
                             int cap, uint8_t* out, sbn_stream_t stream) {
  int st = check_geo(gp);
  if (st) return st;
  if (cap <= 0) return SBN_OK;
  Geo g = to_geo(gp);
  long total = (long)cap * g.bh * g.bw;
  long blocks = (total + 255) / 256;
  if (blocks > (long)sm_count() * 16) blocks = (long)sm_count() * 16;
  in_bounds_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(g, idx, count, cap, out);
  return launch_status("in_bounds");
}
