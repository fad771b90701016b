// tcgen05 / TMEM dense 3x3 convolution with any stride and the bias fused into the
// epilogue (bf16 in/out, fp32 accumulate): the stage-transition projection of
// `run_stage` (reference `layers.py:316-318`, a dense stride-s 3x3 conv + bias) for the
// BASELINE config-4 backbone, which otherwise runs cuDNN plus a separate bias-add pass
// over the whole output.
//
// Implicit GEMM without im2col: a tile is 8 x 16 output pixels (M = 128 rows).  For each
// (K-chunk, tap) the A operand is ONE 4-D TMA box of x — (KC channels, 16*s, 8*s, 1)
// with element strides (1, s, s, 1) at (kc*KC, s*ox0 + kx - pad, s*oy0 + ky - pad, n):
// exactly the 128 input pixels the tap reads, zero-filled outside the image (= SAME /
// VALID padding), landing as swizzled KC-channel rows (SWIZZLE_128B for KC=64, 64B for
// KC=32).  B is the tap's (COUT x KC) weight chunk, pre-packed in the K-major plane
// layout, resident in smem when all 9*CIN*COUT fit, streamed through a ring otherwise.
//
// Warp roles per persistent CTA (320 threads): warps 0-7 epilogue (TMEM lane quarter =
// warp % 4, two warps per quarter split the columns; +bias -> bf16 staged in smem, then
// copied out along whole output pixel rows, coalesced), warp 8 TMA / bulk loader, warp 9
// MMA issuer.  Double-buffered accumulators when 2*COUT <= 512 columns.
#include "tma_util.cuh"

#include <cstring>

namespace sbn {
namespace {

constexpr int kCE = 256;                 // epilogue threads
constexpr int kCThreads = kCE + 64;
#ifndef SBN_DENSE_BUDGET_KB
#define SBN_DENSE_BUDGET_KB 220
#endif
#ifndef SBN_DENSE_RES_STAGES
#define SBN_DENSE_RES_STAGES 3  // resident weights need only a 3-deep A ring (c=96: 166 KB of weights stay resident)
#endif
constexpr int kCBudget = SBN_DENSE_BUDGET_KB * 1024;
#ifndef SBN_DENSE_HALF_BUDGET_KB
#define SBN_DENSE_HALF_BUDGET_KB 108
#endif
constexpr int kHalfBudget = SBN_DENSE_HALF_BUDGET_KB * 1024;  // per CTA at two CTAs / SM
#ifndef SBN_DENSE_MAX_STREAM
#define SBN_DENSE_MAX_STREAM 8
#endif
constexpr int kMaxStream = SBN_DENSE_MAX_STREAM;  // streamed-weights ring depth cap

// weights resident in smem with 64-channel K-chunks?  (otherwise they stream through a ring
// in 32-channel chunks, which keeps the per-stage footprint small enough for a deep ring)
// channel counts padded to the UMMA granule (16): K padding is zero-filled by TMA (the box
// runs past the tensor's channel extent) and by the packed weights, N padding is dropped
// by the epilogue
constexpr int pad16(int c) { return (c + 15) / 16 * 16; }
constexpr int dense_kc(int cp) { return cp % 64 == 0 ? 64 : cp % 32 == 0 ? 32 : 16; }

template <int CIN, int COUT, int KS>
constexpr bool dense_resident() {
  constexpr int cp = pad16(CIN), np = pad16(COUT);
  constexpr int kc = dense_kc(cp);
  constexpr int gs = np <= 192 ? np : 128;
  return (long)SBN_DENSE_RES_STAGES * 128 * kc * 2 + (long)KS * KS * cp * np * 2 + 128L * (gs * 2 + 16) + np * 4 + 128 <= kCBudget;
}

template <int CIN, int COUT, int KS>
struct CCfg {
  static constexpr int TAPS = KS * KS;
  // 64-channel K-chunks whenever CIN allows: each TMA box row is then 128 B (SWIZZLE_128B)
  // per pixel; 32-channel chunks (64-B rows) made the per-tap boxes TMA-issue bound
  // (block-32 sparse conv 348 -> 219 us at 100 %, 192->256 projection 84 -> 68 us)
  // (16-channel chunks, 32-B rows, SWIZZLE_32B, for CIN = 16 / 48 / 80 ...)
  static constexpr int CP = pad16(CIN), NP = pad16(COUT);  // padded K / N extents
  static constexpr int KC = dense_kc(CP);
  static_assert(CP % KC == 0, "K chunking");
  static_assert(COUT % 8 == 0, "output pixel rows must be whole 16-byte chunks");
  static constexpr int NKC = CP / KC;
  static constexpr int ROWB = KC * 2;
  static constexpr uint32_t SWZ = KC == 64 ? 2u : KC == 32 ? 4u : 6u;
  static constexpr int ACH = 128 * ROWB;
  static constexpr int PW = NP * 16;
  static constexpr int WCH = (KC / 8) * PW;
  static constexpr int CHUNKS = NKC * TAPS;
  static constexpr long WBYTES = (long)CHUNKS * WCH;
  static constexpr int NSPLIT = NP > 256 ? 2 : 1;
  static constexpr int NS = NP / NSPLIT;
  static_assert(NP % NSPLIT == 0 && NS % 16 == 0 && NS <= 256, "UMMA N");
  static constexpr int NACC = 2 * NP <= 512 ? 2 : 1;
  static constexpr int TCOLS = NACC * NP;
  static constexpr int TALLOC = TCOLS <= 32 ? 32 : TCOLS <= 64 ? 64 : TCOLS <= 128 ? 128 : TCOLS <= 256 ? 256 : 512;
  static constexpr int GS = NP <= 192 ? NP : 128;  // staged columns per pass
  static_assert(NP % GS == 0, "staging groups");
  static constexpr int SPITCH = GS * 2 + 16;
  static constexpr int STGB = 128 * SPITCH;
  static constexpr int PARB = (NP * 4 + 127) / 128 * 128;
  static constexpr bool RES = dense_resident<CIN, COUT, KS>();
  // A boxes are small and latency-bound (strided gathers): keep up to 12 in flight; the
  // streamed case pairs every A box with a weight chunk, so both rings get the same depth
  static constexpr int SA_R = (int)((kCBudget - WBYTES - STGB - PARB) / ACH);
  static constexpr int SS = (int)((kCBudget - STGB - PARB) / (ACH + WCH));
  // small shapes (resident weights, >= 4 A stages within half the SM's shared memory) run
  // two CTAs per SM: twice the tiles in flight for the latency-bound small-channel convs
  static constexpr int SA_2 = RES ? (int)((kHalfBudget - WBYTES - STGB - PARB) / ACH) : 0;
  static constexpr int CPS = SA_2 >= 4 ? 2 : 1;  // CTAs per SM
  static constexpr int SA = CPS == 2 ? (SA_2 > 12 ? 12 : SA_2)
                                     : RES ? (SA_R > 12 ? 12 : SA_R) : (SS > kMaxStream ? kMaxStream : SS);
  static constexpr int SW = RES ? 0 : SA;
  static constexpr long WREG = RES ? WBYTES : (long)SW * WCH;
  static_assert(SA >= 2 && SA * ACH + WREG + STGB + PARB <= kCBudget, "shared memory budget");
  static constexpr int OFF_W = SA * ACH;
  static constexpr int OFF_STG = OFF_W + (int)WREG;
  static constexpr int OFF_PAR = OFF_STG + STGB;
  static constexpr int SMEM = OFF_PAR + PARB;
};

struct __align__(64) CArgs {
  CUtensorMap tmap;       // x as (C, W, H, N), box (KC, tw*s, th*s, 1), element strides (1, s, s, 1)
  __nv_bfloat16* out;     // (n, oh, ow, COUT)
  const uint8_t* wpk;     // packed weight chunks (kc, tap)
  const float* bias;      // COUT floats (dense mode) ...
  const __nv_bfloat16* bias_bf16;  // ... or bf16 / null (sparse mode, sparse_conv2d's FilterBank)
  int n, oh, ow, sy, sx, py, px;
  int tiles_y, tiles_x;   // dense mode: 8 x 16 output tiles
  int th, tw;             // output rows / cols per tile (dense 8 x 16; sparse: <= the out block)
  // sparse mode (idx != null): active block j of the list is covered by subs_y x subs_x
  // tiles of th x tw outputs (one tile when obh*obw <= 128); its window starts at
  // (goy + by*gsy, gox + bx*gsx) and its output block (obh x obw) at (by*obh, bx*obw)
  const int32_t* idx;
  const int32_t* count;
  int cap, gsy, gsx, goy, gox;
  int obh, obw, subs_y, subs_x;
  // mask-fused sparse mode (mask != null, idx == null): the work units are (candidate
  // block, sub-tile) pairs; CTA c owns units c, c + G, ... (at most kMaxLocalTma), tests
  // each unit's candidate window against the mask itself and convolves the active ones —
  // no reduce_mask launch, no grid-wide step (used when every CTA owns <= 2 units, so the
  // local lists are as balanced as a striped global list)
  const uint8_t* mask;
  int gy, gx, wbh, wbw;   // candidate grid and window (= block) size
  int n_h, n_w;           // input (= mask) height / width
  // mask-fused GLOBAL-list mode (mask and gidx set, list-mode kernel): every CTA tests its
  // candidates (c, c + G, ...), publishes the active ones into gidx, and after all G CTAs have
  // published the CTAs stride through the list as in list mode — one launch for grids too
  // big for the local lists.  sw: [0] launch epoch, [4 + 4 * (tag & 1) + {0 claimed, 1 done}]
  unsigned* sw;
  int32_t* gidx;
};

constexpr int kMaxLocalTma = 4;
constexpr int kMaxGlobTma = 64;  // candidates per CTA in the global-list mode
#ifndef SBN_FUSED_UNITS_PER_CTA
#define SBN_FUSED_UNITS_PER_CTA 4  // mask-fused mode only while every CTA owns <= this many units (2 vs 4: conv-3 block 16 12.3 vs 8.7 us)
#endif
static_assert(SBN_FUSED_UNITS_PER_CTA <= kMaxLocalTma, "local list size");

// tile -> (frame, first output row / col, first input row / col of tap (0, 0)); ly / lx:
// rows / cols of the tile inside its block's output window (sparse) or th / tw (dense)
template <bool LOCAL>
__device__ __forceinline__ void conv_tile(const CArgs& a, const int32_t* lidx, int tile, int& n, int& oy0, int& ox0,
                                          int& iy0, int& ix0, int& ly, int& lx) {
  ly = a.th;
  lx = a.tw;
  if (LOCAL || a.idx || a.gidx) {
    int by, bx, sub;
    if constexpr (LOCAL) {  // this CTA's local list in shared memory: (n, by, bx, sub) per unit
      n = lidx[4 * tile];
      by = lidx[4 * tile + 1];
      bx = lidx[4 * tile + 2];
      sub = lidx[4 * tile + 3];
    } else {
      const int subs = a.subs_y * a.subs_x;
      const int j = tile / subs;
      sub = tile - j * subs;
      if (a.gidx) {  // written in this launch: coherent loads
        n = a.gidx[3 * j];
        by = a.gidx[3 * j + 1];
        bx = a.gidx[3 * j + 2];
      } else {
        n = __ldg(a.idx + 3 * j);
        by = __ldg(a.idx + 3 * j + 1);
        bx = __ldg(a.idx + 3 * j + 2);
      }
    }
    const int ty = sub / a.subs_x, tx = sub - ty * a.subs_x;
    oy0 = by * a.obh + ty * a.th;
    ox0 = bx * a.obw + tx * a.tw;
    iy0 = a.goy + by * a.gsy + ty * a.th * a.sy;
    ix0 = a.gox + bx * a.gsx + tx * a.tw * a.sx;
    ly = min(a.th, a.obh - ty * a.th);
    lx = min(a.tw, a.obw - tx * a.tw);
  } else {
    const int tx = tile % a.tiles_x, ty = (tile / a.tiles_x) % a.tiles_y;
    n = tile / (a.tiles_x * a.tiles_y);
    oy0 = ty * a.th;
    ox0 = tx * a.tw;
    iy0 = oy0 * a.sy - a.py;
    ix0 = ox0 * a.sx - a.px;
  }
}

template <int CIN, int COUT, int KS, bool LOCAL>
__global__ void __launch_bounds__(kCThreads, CCfg<CIN, COUT, KS>::CPS) conv_dense_kernel(const __grid_constant__ CArgs a) {
  using Q = CCfg<CIN, COUT, KS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int SWB = Q::SW > 0 ? Q::SW : 1;
  __shared__ uint64_t a_full[Q::SA], a_empty[Q::SA], w_full[SWB], w_empty[SWB];
  __shared__ uint64_t acc_full[Q::NACC], acc_empty[Q::NACC];
  __shared__ uint32_t tslot;
  __shared__ long long rowdst[128];
  uint8_t* Aring = smem;
  uint8_t* Wring = smem + Q::OFF_W;
  uint8_t* stg = smem + Q::OFF_STG;
  float* bias = reinterpret_cast<float*>(smem + Q::OFF_PAR);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kLWarp = kCE / 32, kMWarp = kLWarp + 1;

  if (tid == 0) {
    for (int s = 0; s < Q::SA; ++s) {
      tc::mbar_init(&a_full[s], 1);
      tc::mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < SWB; ++s) {
      tc::mbar_init(&w_full[s], 1);
      tc::mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < Q::NACC; ++s) {
      tc::mbar_init(&acc_full[s], 1);
      tc::mbar_init(&acc_empty[s], kCE);
    }
    tc::mbar_fence_init();
  }
  if (tid == kLWarp * 32) asm volatile("prefetch.tensormap [%0];" ::"l"(&a.tmap) : "memory");
  for (int i = tid; i < COUT; i += kCThreads)
    bias[i] = a.bias ? a.bias[i] : a.bias_bf16 ? __bfloat162float(a.bias_bf16[i]) : 0.f;
  if constexpr (Q::NP != COUT)
    for (int i = COUT + tid; i < Q::NP; i += kCThreads) bias[i] = 0.f;
  if (warp == 0) tc::tmem_alloc<Q::TALLOC>(&tslot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  tc::pdl_trigger();
  if (Q::RES && tid == kLWarp * 32) {  // weights do not depend on the previous launch
    tc::mbar_expect_tx(&w_full[0], (uint32_t)Q::WBYTES);
    for (int c = 0; c < Q::CHUNKS; ++c)
      tc::bulk_g2s(Wring + (size_t)c * Q::WCH, a.wpk + (size_t)c * Q::WCH, Q::WCH, &w_full[0]);
  }
  tc::pdl_wait();
  __shared__ int32_t s_idx[LOCAL ? 4 * kMaxLocalTma : 1];
  __shared__ int s_nloc;
  if constexpr (LOCAL) {  // reference tiling.py:138-160 (MAX pool): active iff any window pixel is set
    const int subs = a.subs_y * a.subs_x;
    const int U = a.n * a.gy * a.gx * subs, G = gridDim.x, gyx = a.gy * a.gx, area = a.wbh * a.wbw;
    if (tid == 0) s_nloc = 0;
    __syncthreads();
    for (int k = 0; k < kMaxLocalTma; ++k) {
      const int unit = (int)blockIdx.x + k * G;
      if (unit >= U) break;  // uniform
      const int cand = unit / subs, sub = unit - cand * subs;
      const int fr = cand / gyx, rr = cand - fr * gyx, by = rr / a.gx, bx = rr - by * a.gx;
      const int y0 = a.goy + by * a.gsy, x0 = a.gox + bx * a.gsx;
      bool any = false;
      for (int p = tid; p < area; p += kCThreads) {
        const int y = y0 + p / a.wbw, xx = x0 + p % a.wbw;
        if (y >= 0 && y < a.n_h && xx >= 0 && xx < a.n_w) any |= __ldg(a.mask + ((size_t)fr * a.n_h + y) * a.n_w + xx) != 0;
      }
      if (__syncthreads_or(any) && tid == 0) {
        s_idx[4 * s_nloc] = fr;
        s_idx[4 * s_nloc + 1] = by;
        s_idx[4 * s_nloc + 2] = bx;
        s_idx[4 * s_nloc + 3] = sub;
        ++s_nloc;
      }
    }
    __syncthreads();
  }
  if constexpr (!LOCAL) {
    if (a.gidx) {  // mask-fused global list (reference tiling.py:138-160, MAX pool)
      __shared__ uint8_t s_flag[kMaxGlobTma];
      __shared__ int s_base;
      __shared__ unsigned s_tag;
      const int T = a.n * a.gy * a.gx, G = gridDim.x, gyx = a.gy * a.gx, area = a.wbh * a.wbw;
      const int nc = T > (int)blockIdx.x ? min((T - (int)blockIdx.x + G - 1) / G, kMaxGlobTma) : 0;
      if (tid == 0) s_tag = *reinterpret_cast<volatile unsigned*>(a.sw) + 1u;
      constexpr int NW = kCThreads / 32;
      for (int j = warp; j < nc; j += NW) {  // one warp per candidate, all its loads in flight
        const int cand = (int)blockIdx.x + j * G;
        const int fr = cand / gyx, rr = cand - fr * gyx, by = rr / a.gx, bx = rr - by * a.gx;
        const int y0 = a.goy + by * a.gsy, x0 = a.gox + bx * a.gsx;
        uint32_t v = 0;
#pragma unroll 8
        for (int p = lane; p < area; p += 32) {
          const int y = y0 + p / a.wbw, xx = x0 + p % a.wbw;
          const bool ok = y >= 0 && y < a.n_h && xx >= 0 && xx < a.n_w;
          v |= tc::ld_u8_pred(a.mask + ((size_t)fr * a.n_h + (ok ? y : 0)) * a.n_w + (ok ? xx : 0), ok);
        }
        const bool any = __any_sync(0xffffffffu, v != 0);
        if (lane == 0) s_flag[j] = any;
      }
      __syncthreads();
      const unsigned tag = s_tag;
      unsigned* ring = a.sw + 4 + 4 * (tag & 1u);
      if (warp == 0) {  // compact this CTA's active candidates, claim slots, publish rows
        int nl = 0;
        for (int c0 = 0; c0 < nc; c0 += 32) nl += __popc(__ballot_sync(0xffffffffu, c0 + lane < nc && s_flag[c0 + lane]));
        int base = 0;
        if (lane == 0 && nl) base = (int)atomicAdd(ring, (unsigned)nl);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int c0 = 0; c0 < nc; c0 += 32) {
          const bool on = c0 + lane < nc && s_flag[c0 + lane];
          const unsigned bal = __ballot_sync(0xffffffffu, on);
          if (on) {
            const int q = base + __popc(bal & ((1u << lane) - 1u));
            const int cand = (int)blockIdx.x + (c0 + lane) * G;
            const int fr = cand / gyx, rr = cand - fr * gyx;
            a.gidx[3 * q] = fr;
            a.gidx[3 * q + 1] = rr / a.gx;
            a.gidx[3 * q + 2] = rr % a.gx;
          }
          base += __popc(bal);
        }
      }
      __syncthreads();
      if (tid == 0) {
        unsigned old;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(ring + 1) : "memory");
        if (old == gridDim.x - 1) {  // last to publish: recycle the other slot, advance the epoch
          unsigned* other = a.sw + 4 + 4 * ((tag + 1u) & 1u);
          other[0] = 0u;
          other[1] = 0u;
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.sw), "r"(tag) : "memory");
        }
        SpinGuard sg;
        unsigned d;
        while (true) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(d) : "l"(ring + 1) : "memory");
          if (d == gridDim.x) break;
          __nanosleep(32);
          sg.tick(kSpinSlotDone);
        }
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(d) : "l"(ring) : "memory");
        s_nloc = (int)d;
      }
      __syncthreads();
    }
  }
  const int32_t* lidx = s_idx;  // read only in LOCAL mode
  const int ntiles = LOCAL ? s_nloc
                           : a.gidx ? s_nloc * a.subs_y * a.subs_x
                           : a.idx ? ld_count(a.count, a.cap) * a.subs_y * a.subs_x : a.n * a.tiles_y * a.tiles_x;

  if (warp < kLWarp) {
    // ------------------------------------------------ epilogue
    const int qd = warp & 3, half = warp >> 2;
    const int r = qd * 32 + lane;
    constexpr int CHR = Q::GS * 2 / 16;
    constexpr int IT2 = (128 * CHR + kCE - 1) / kCE;
    constexpr int BATCH = IT2 < 8 ? IT2 : 8;
    int k = 0;
    for (int tile = LOCAL ? 0 : blockIdx.x; tile < ntiles; tile += LOCAL ? 1 : gridDim.x, ++k) {
      const int buf = Q::NACC == 2 ? (k & 1) : 0;
      const int use = Q::NACC == 2 ? (k >> 1) : k;
      int n, oy0, ox0, iy0, ix0, ly, lx;
      conv_tile<LOCAL>(a, lidx, tile, n, oy0, ox0, iy0, ix0, ly, lx);
      const int Y = oy0 + r / a.tw, X = ox0 + r % a.tw;
      if (half == 0)
        rowdst[r] = (r < a.th * a.tw && r / a.tw < ly && r % a.tw < lx && Y < a.oh && X < a.ow)
                        ? (((long long)n * a.oh + Y) * a.ow + X) * COUT : -1;
      const uint32_t acc = tmem + ((uint32_t)(qd * 32) << 16) + buf * Q::NP;
      tc::mbar_wait(&acc_full[buf], use & 1);
      tc::fence_after();
      for (int g0 = 0; g0 < Q::NP; g0 += Q::GS) {
#pragma unroll
        for (int e = 0; e < (Q::GS / 16 + 1) / 2; ++e) {
          const int cg = 16 * (2 * e + half);
          if (cg >= Q::GS) break;  // warp-uniform
          float v[16];
          tc::tmem_ld16(acc + g0 + cg, v);
          uint32_t o[8];
#pragma unroll
          for (int q = 0; q < 8; q += 2) {
            const float4 b4 = *reinterpret_cast<const float4*>(bias + g0 + cg + 2 * q);
            o[q] = tc::pack_bf16(v[2 * q] + b4.x, v[2 * q + 1] + b4.y);
            o[q + 1] = tc::pack_bf16(v[2 * q + 2] + b4.z, v[2 * q + 3] + b4.w);
          }
          uint4* sp = reinterpret_cast<uint4*>(stg + r * Q::SPITCH + cg * 2);
          sp[0] = make_uint4(o[0], o[1], o[2], o[3]);
          sp[1] = make_uint4(o[4], o[5], o[6], o[7]);
        }
        if (g0 + Q::GS >= Q::NP) {  // accumulator drained: the next tile's MMAs may start
          tc::fence_before();
          tc::mbar_arrive(&acc_empty[buf]);
        }
        tc::named_bar<1, kCE>();
        // copy out: consecutive threads take consecutive 16-B chunks of one output row
#pragma unroll 1
        for (int jb = 0; jb < IT2; jb += BATCH) {
#pragma unroll
          for (int jj = 0; jj < BATCH; ++jj) {
            const int it = tid + (jb + jj) * kCE;
            if (jb + jj >= IT2 || it >= 128 * CHR) break;
            const int row = it / CHR, ch = it % CHR;
            const long long off = rowdst[row];
            if (off < 0 || (Q::NP != COUT && g0 * 2 / 16 + ch >= COUT * 2 / 16)) continue;  // N padding
            reinterpret_cast<uint4*>(a.out + off + g0)[ch] =
                *reinterpret_cast<const uint4*>(stg + row * Q::SPITCH + ch * 16);
          }
        }
        tc::named_bar<1, kCE>();  // staging / rowdst reuse
      }
    }
  } else if (warp == kLWarp) {
    // ------------------------------------------------ loader
    if (lane == 0) {
      int c = 0, wit = 0;
      for (int tile = LOCAL ? 0 : blockIdx.x; tile < ntiles; tile += LOCAL ? 1 : gridDim.x) {
        int n, oy0, ox0, y0, x0, ly, lx;
        conv_tile<LOCAL>(a, lidx, tile, n, oy0, ox0, y0, x0, ly, lx);
        const uint32_t bytes = (uint32_t)(a.th * a.tw * Q::ROWB);
        for (int kc = 0; kc < Q::NKC; ++kc)
          for (int tap = 0; tap < Q::TAPS; ++tap, ++c) {
            const int s = c % Q::SA;
            tc::mbar_wait(&a_empty[s], ((c / Q::SA) & 1) ^ 1);
            tc::mbar_expect_tx(&a_full[s], bytes);
            tma_4d(Aring + s * Q::ACH, &a.tmap, kc * Q::KC, x0 + tap % KS, y0 + tap / KS, n, &a_full[s]);
            if (!Q::RES) {
              const int sw = wit % SWB;
              tc::mbar_wait(&w_empty[sw], ((wit / SWB) & 1) ^ 1);
              tc::mbar_expect_tx(&w_full[sw], Q::WCH);
              tc::bulk_g2s(Wring + sw * Q::WCH, a.wpk + (size_t)(kc * Q::TAPS + tap) * Q::WCH, Q::WCH, &w_full[sw]);
              ++wit;
            }
          }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(128, Q::NS);
      if (Q::RES) tc::mbar_wait(&w_full[0], 0);
      int c = 0, wit = 0, k = 0;
      for (int tile = LOCAL ? 0 : blockIdx.x; tile < ntiles; tile += LOCAL ? 1 : gridDim.x, ++k) {
        const int buf = Q::NACC == 2 ? (k & 1) : 0;
        const int use = Q::NACC == 2 ? (k >> 1) : k;
        tc::mbar_wait(&acc_empty[buf], (use & 1) ^ 1);
        tc::fence_after();
        const uint32_t acc = tmem + buf * Q::NP;
        for (int kc = 0; kc < Q::NKC; ++kc)
          for (int tap = 0; tap < Q::TAPS; ++tap, ++c) {
            const int s = c % Q::SA;
            tc::mbar_wait(&a_full[s], (c / Q::SA) & 1);
            const int sw = Q::RES ? 0 : wit % SWB;
            if (!Q::RES) tc::mbar_wait(&w_full[sw], (wit / SWB) & 1);
            tc::fence_after();
            const uint64_t ad = tc::desc_kmajor_swz(tc::smem_u32(Aring + s * Q::ACH), 8 * Q::ROWB, Q::SWZ);
            const uint64_t wd = tc::desc_kmajor_noswz(
                tc::smem_u32(Wring + (Q::RES ? (kc * Q::TAPS + tap) * Q::WCH : sw * Q::WCH)), Q::PW, 128);
#pragma unroll
            for (int kk = 0; kk < Q::KC / 16; ++kk)
#pragma unroll
              for (int h = 0; h < Q::NSPLIT; ++h)
                tc::mma_bf16(acc + h * Q::NS, tc::desc_add(ad, kk * 32), tc::desc_add(wd, 2 * kk * Q::PW + h * Q::NS * 16),
                             idesc, (kc | tap | kk) > 0);
            tc::mma_commit(&a_empty[s]);
            if (!Q::RES) {
              tc::mma_commit(&w_empty[sw]);
              ++wit;
            }
          }
        tc::mma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  }
  if (Q::RES && tid == kLWarp * 32) tc::mbar_wait(&w_full[0], 0);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_free<Q::TALLOC>(tmem);
}

// ---- CTA-pair (cta_group::2) dense projection: two 8 x 16 output tiles per pair as ONE
// M = 256 UMMA issued by rank 0.  B is split along N (rank r holds output channels
// [r*NS/2, (r+1)*NS/2) of every N-slice of every weight chunk), so each SM stores / streams
// half of the weights: the config-4 stage-1 projection (96 -> 192) keeps its half (166 KB)
// resident for the whole launch, and the wider ones (192 -> 256, 256 -> 384) stream half the
// bytes per tile.  (The single-CTA kernel re-streams all 9 * CIN * COUT weights from L2 for
// every 128-pixel tile once they exceed shared memory: 332 KB per tile at 96 -> 192.)
// Handshakes (rank 0 owns what its MMA issuer waits on):
//   a_full[s]    both ranks' A boxes of stage s landed (rank 1's TMA completes on it)   rank 0
//   w_full[s]    both weight halves of stage s landed (streamed)                       rank 0
//   *_empty[s]   MMAs reading stage s done (multicast commit)                          both
//   acc_full[b]  accumulator b complete (multicast commit)                             both
//   acc_empty[b] 2 x kCE epilogue arrivals (rank 1's arrive remotely)                  rank 0
//   wpeer        rank 1's resident half landed (remote arrive)                         rank 0
template <int CIN, int COUT, int KS>
struct PCfg {
  using Q = CCfg<CIN, COUT, KS>;
  static constexpr int TAPS = Q::TAPS, KC = Q::KC, NKC = Q::NKC, ROWB = Q::ROWB, ACH = Q::ACH;
  static constexpr uint32_t SWZ = Q::SWZ;
  static constexpr int NP = Q::NP, NSPLIT = Q::NSPLIT, NS = Q::NS, NHS = NS / 2;
  static constexpr int PWR = (NP / 2) * 16;      // plane stride of a rank's half chunk
  static constexpr int WCHR = (KC / 8) * PWR;    // one (kc, tap) half chunk
  static constexpr int CHUNKS = Q::CHUNKS;
  static constexpr long WBYTESR = (long)CHUNKS * WCHR;
  static constexpr int GS = NP % 64 == 0 ? 64 : NP;  // staged columns per pass (small staging buffer)
  static constexpr int SPITCH = GS * 2 + 16;
  static constexpr int STGB = 128 * SPITCH;
  static constexpr int PARB = Q::PARB;
  static constexpr int NACC = Q::NACC, TALLOC = Q::TALLOC;
  static constexpr bool RES = 3L * ACH + WBYTESR + STGB + PARB <= kCBudget;
  static constexpr int SA_R = (int)((kCBudget - WBYTESR - STGB - PARB) / ACH);
  static constexpr int SS = (int)((kCBudget - STGB - PARB) / (ACH + WCHR));
  static constexpr int SA = RES ? (SA_R > 12 ? 12 : SA_R) : (SS > kMaxStream ? kMaxStream : SS);
  static constexpr int SW = RES ? 0 : SA;
  static constexpr long WREG = RES ? WBYTESR : (long)SW * WCHR;
  static constexpr int OFF_W = SA * ACH;
  static constexpr int OFF_STG = OFF_W + (int)WREG;
  static constexpr int OFF_PAR = OFF_STG + STGB;
  static constexpr int SMEM = OFF_PAR + PARB;
  static constexpr int WBOXR = WCHR / 128;      // a half chunk as a TMA box of 128-byte rows
  // used for the dense projections whose weights the single-CTA kernel must stream, when the
  // pair still keeps >= 5 A boxes in flight: these convs are bound by the TMA box rate (one
  // box of 128 strided pixel rows per (K-chunk, tap)), so a shallower A ring loses more than
  // the halved weight stream saves (96 -> 192 with resident halves and 4 A stages: stage 1 of
  // the backbone 0.546 -> 0.549 ms; 192 -> 256 / 256 -> 384 streamed: 0.353 -> 0.346,
  // 0.204 -> 0.199 ms)
  static constexpr bool USE = !Q::RES && NHS % 8 == 0 && SA >= 5 && WBOXR <= 256 && WCHR % 128 == 0 &&
                              SMEM <= 227 * 1024;
};

struct __align__(64) PArgs {
  CArgs c;
  CUtensorMap wmap;  // the pair copy of the packed weights as 128-byte rows, box = one half chunk
};

template <int CIN, int COUT, int KS>
__global__ void __launch_bounds__(kCThreads, 1) conv_dense_pair_kernel(const __grid_constant__ PArgs pa) {
  using P = PCfg<CIN, COUT, KS>;
  const CArgs& a = pa.c;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int SWB = P::SW > 0 ? P::SW : 1;
  __shared__ uint64_t a_full[P::SA], a_empty[P::SA], w_full[SWB], w_empty[SWB];
  __shared__ uint64_t acc_full[P::NACC], acc_empty[P::NACC], wres, wpeer;
  __shared__ uint32_t tslot;
  __shared__ long long rowdst[128];
  uint8_t* Aring = smem;
  uint8_t* Wring = smem + P::OFF_W;
  uint8_t* stg = smem + P::OFF_STG;
  float* bias = reinterpret_cast<float*>(smem + P::OFF_PAR);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = tc::cluster_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  constexpr int kLWarp = kCE / 32;

  if (tid == 0) {
    for (int s = 0; s < P::SA; ++s) {
      tc::mbar_init(&a_full[s], 1);
      tc::mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < SWB; ++s) {
      tc::mbar_init(&w_full[s], 1);
      tc::mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < P::NACC; ++s) {
      tc::mbar_init(&acc_full[s], 1);
      tc::mbar_init(&acc_empty[s], 2 * kCE);
    }
    tc::mbar_init(&wres, 1);
    tc::mbar_init(&wpeer, 1);
    tc::mbar_fence_init();
  }
  if (tid == kLWarp * 32) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&a.tmap) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&pa.wmap) : "memory");
  }
  for (int i = tid; i < COUT; i += kCThreads) bias[i] = a.bias ? a.bias[i] : 0.f;
  if constexpr (P::NP != COUT)
    for (int i = COUT + tid; i < P::NP; i += kCThreads) bias[i] = 0.f;
  if (warp == 0) tc::tmem_alloc_cg2<P::TALLOC>(&tslot);
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();  // both CTAs' barriers exist before any remote arrive / multicast commit
  tc::fence_after();
  const uint32_t tmem = tslot;
  tc::pdl_trigger();
  const uint8_t* wpair = a.wpk + (size_t)P::Q::WBYTES;  // the pair copy follows the single image
  if (P::RES && tid == kLWarp * 32) {  // my half of every chunk, resident (independent of the previous launch)
    tc::mbar_expect_tx(&wres, (uint32_t)P::WBYTESR);
    for (int c = 0; c < P::CHUNKS; ++c)
      tc::bulk_g2s(Wring + (size_t)c * P::WCHR, wpair + ((size_t)c * 2 + rank) * P::WCHR, P::WCHR, &wres);
  }
  tc::pdl_wait();
  const int ntiles = a.n * a.tiles_y * a.tiles_x;
  const int nptiles = (ntiles + 1) / 2;  // an odd last tile pairs with an empty (zero) one

  if (warp < kLWarp) {
    // ------------------------------------------------ epilogue (my tile of each pair tile)
    const int qd = warp & 3, half = warp >> 2;
    const int r = qd * 32 + lane;
    constexpr int CHR = P::GS * 2 / 16;
    constexpr int IT2 = (128 * CHR + kCE - 1) / kCE;
    int k = 0;
    for (int pt = pair; pt < nptiles; pt += npairs, ++k) {
      const int buf = P::NACC == 2 ? (k & 1) : 0;
      const int use = P::NACC == 2 ? (k >> 1) : k;
      const int tile = 2 * pt + (int)rank;
      int n, oy0, ox0, iy0, ix0, ly, lx;
      conv_tile<false>(a, nullptr, tile, n, oy0, ox0, iy0, ix0, ly, lx);
      const int Y = oy0 + r / a.tw, X = ox0 + r % a.tw;
      if (half == 0)
        rowdst[r] = (tile < ntiles && r < a.th * a.tw && Y < a.oh && X < a.ow)
                        ? (((long long)n * a.oh + Y) * a.ow + X) * COUT : -1;
      const uint32_t acc = tmem + ((uint32_t)(qd * 32) << 16) + buf * P::NP;
      tc::mbar_wait(&acc_full[buf], use & 1);
      tc::fence_after();
      for (int g0 = 0; g0 < P::NP; g0 += P::GS) {
#pragma unroll
        for (int e = 0; e < (P::GS / 16 + 1) / 2; ++e) {
          const int cg = 16 * (2 * e + half);
          if (cg >= P::GS) break;  // warp-uniform
          float v[16];
          tc::tmem_ld16(acc + g0 + cg, v);
          uint32_t o[8];
#pragma unroll
          for (int q = 0; q < 8; q += 2) {
            const float4 b4 = *reinterpret_cast<const float4*>(bias + g0 + cg + 2 * q);
            o[q] = tc::pack_bf16(v[2 * q] + b4.x, v[2 * q + 1] + b4.y);
            o[q + 1] = tc::pack_bf16(v[2 * q + 2] + b4.z, v[2 * q + 3] + b4.w);
          }
          uint4* sp = reinterpret_cast<uint4*>(stg + r * P::SPITCH + cg * 2);
          sp[0] = make_uint4(o[0], o[1], o[2], o[3]);
          sp[1] = make_uint4(o[4], o[5], o[6], o[7]);
        }
        if (g0 + P::GS >= P::NP) {  // accumulator drained: the next pair tile's MMAs may start
          tc::fence_before();
          if (rank == 0) tc::mbar_arrive(&acc_empty[buf]);
          else tc::mbar_arrive_cluster(&acc_empty[buf], 0);
        }
        tc::named_bar<1, kCE>();
#pragma unroll
        for (int jj = 0; jj < IT2; ++jj) {
          const int it = tid + jj * kCE;
          if (it >= 128 * CHR) break;
          const int row = it / CHR, ch = it % CHR;
          const long long off = rowdst[row];
          if (off < 0 || (P::NP != COUT && g0 * 2 / 16 + ch >= COUT * 2 / 16)) continue;  // N padding
          reinterpret_cast<uint4*>(a.out + off + g0)[ch] = *reinterpret_cast<const uint4*>(stg + row * P::SPITCH + ch * 16);
        }
        tc::named_bar<1, kCE>();  // staging / rowdst reuse
      }
    }
  } else if (warp == kLWarp) {
    // ------------------------------------------------ loader: my tile's A boxes, my weight halves
    if (lane == 0) {
      if (P::RES && rank == 1) {  // tell rank 0's issuer that my resident half has landed
        tc::mbar_wait(&wres, 0);
        tc::mbar_arrive_cluster(&wpeer, 0);
      }
      int c = 0, wit = 0;
      const uint32_t bytes = (uint32_t)(a.th * a.tw * P::ROWB);
      for (int pt = pair; pt < nptiles; pt += npairs) {
        const int tile = 2 * pt + (int)rank;
        int n, oy0, ox0, y0, x0, ly, lx;
        conv_tile<false>(a, nullptr, tile < ntiles ? tile : 0, n, oy0, ox0, y0, x0, ly, lx);
        if (tile >= ntiles) n = a.n;  // past the last frame: TMA zero-fills the whole box
        for (int kc = 0; kc < P::NKC; ++kc)
          for (int tap = 0; tap < P::TAPS; ++tap, ++c) {
            const int s = c % P::SA;
            tc::mbar_wait(&a_empty[s], ((c / P::SA) & 1) ^ 1);
            if (rank == 0) {
              tc::mbar_expect_tx(&a_full[s], 2 * bytes);
              tma_4d(Aring + s * P::ACH, &a.tmap, kc * P::KC, x0 + tap % KS, y0 + tap / KS, n, &a_full[s]);
            } else {
              tma_4d_cg2(Aring + s * P::ACH, &a.tmap, kc * P::KC, x0 + tap % KS, y0 + tap / KS, n, &a_full[s], 0);
            }
            if (!P::RES) {
              const int sw = wit % SWB;
              tc::mbar_wait(&w_empty[sw], ((wit / SWB) & 1) ^ 1);
              const int row = ((kc * P::TAPS + tap) * 2 + (int)rank) * P::WBOXR;
              if (rank == 0) {
                tc::mbar_expect_tx(&w_full[sw], 2 * P::WCHR);
                tma_2d(Wring + sw * P::WCHR, &pa.wmap, 0, row, &w_full[sw]);
              } else {
                tma_2d_cg2(Wring + sw * P::WCHR, &pa.wmap, 0, row, &w_full[sw], 0);
              }
              ++wit;
            }
          }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ MMA issuer (rank 0): M = 256 over the pair
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(256, P::NS);
      if (P::RES) {
        tc::mbar_wait(&wres, 0);
        tc::mbar_wait(&wpeer, 0);
      }
      int c = 0, wit = 0, k = 0;
      for (int pt = pair; pt < nptiles; pt += npairs, ++k) {
        const int buf = P::NACC == 2 ? (k & 1) : 0;
        const int use = P::NACC == 2 ? (k >> 1) : k;
        tc::mbar_wait(&acc_empty[buf], (use & 1) ^ 1);
        tc::fence_after();
        const uint32_t acc = tmem + buf * P::NP;
        for (int kc = 0; kc < P::NKC; ++kc)
          for (int tap = 0; tap < P::TAPS; ++tap, ++c) {
            const int s = c % P::SA;
            tc::mbar_wait(&a_full[s], (c / P::SA) & 1);
            const int sw = P::RES ? 0 : wit % SWB;
            if (!P::RES) tc::mbar_wait(&w_full[sw], (wit / SWB) & 1);
            tc::fence_after();
            const uint64_t ad = tc::desc_kmajor_swz(tc::smem_u32(Aring + s * P::ACH), 8 * P::ROWB, P::SWZ);
            const uint64_t wd = tc::desc_kmajor_noswz(
                tc::smem_u32(Wring + (P::RES ? (kc * P::TAPS + tap) * P::WCHR : sw * P::WCHR)), P::PWR, 128);
#pragma unroll
            for (int kk = 0; kk < P::KC / 16; ++kk)
#pragma unroll
              for (int h = 0; h < P::NSPLIT; ++h)
                tc::mma_bf16_cg2(acc + h * P::NS, tc::desc_add(ad, kk * 32), tc::desc_add(wd, 2 * kk * P::PWR + h * P::NHS * 16),
                                 idesc, (kc | tap | kk) > 0);
            tc::mma_commit_mc(&a_empty[s], 3);
            if (!P::RES) {
              tc::mma_commit_mc(&w_empty[sw], 3);
              ++wit;
            }
          }
        tc::mma_commit_mc(&acc_full[buf], 3);
      }
    }
    __syncwarp();
  }
  if (P::RES && tid == kLWarp * 32 && rank == 0) tc::mbar_wait(&wres, 0);
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();  // the peer's MMAs / remote arrivals are done before TMEM is freed
  tc::fence_after();
  if (warp == 0) tc::tmem_free_cg2<P::TALLOC>(tmem);
}

template <int CIN, int COUT, int KS>
int launch_dense_pair(const CArgs& c, cudaStream_t s) {
  using P = PCfg<CIN, COUT, KS>;
  if constexpr (P::USE) {
    PArgs pa;
    memset(&pa, 0, sizeof(pa));
    pa.c = c;
    const uint64_t wdims[2] = {64, (uint64_t)P::CHUNKS * 2 * P::WBOXR};  // every half chunk, 128-byte rows
    const uint64_t wstr[1] = {128};
    const uint32_t wbox[2] = {64, (uint32_t)P::WBOXR};
    int st = encode_map(&pa.wmap, c.wpk + (size_t)P::Q::WBYTES, 2, wdims, wstr, wbox, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (st) return st;
    auto kern = conv_dense_pair_kernel<CIN, COUT, KS>;
    static PerDeviceOnce once;
    once([&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM); });
    const long nptiles = ((long)c.n * c.tiles_y * c.tiles_x + 1) / 2;
    const long maxp = sm_count() / 2;
    const long npairs = nptiles < maxp ? (nptiles < 1 ? 1 : nptiles) : maxp;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * npairs));
    cfg.blockDim = dim3(kCThreads);
    cfg.dynamicSmemBytes = P::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, kern, pa);
    return launch_status("dense_conv_tcgen05_pair");
  } else {
    (void)c;
    (void)s;
    return SBN_ERR_UNSUPPORTED;
  }
}

// W (KS, KS, CIN, COUT) HWIO -> chunks (kc, tap) of (COUT rows x KC) in the K-major plane layout
// (+ for the CTA-pair shapes, a second copy after it: chunk (kc, tap) split into the two
// ranks' halves, rank r holding rows [r*NS/2, (r+1)*NS/2) of every N-slice)
template <int CIN, int COUT, int KS>
__global__ void conv_dense_pack_kernel(const __nv_bfloat16* __restrict__ w, uint8_t* __restrict__ img) {
  using Q = CCfg<CIN, COUT, KS>;
  using P = PCfg<CIN, COUT, KS>;
  constexpr int CP = Q::CP, NP = Q::NP;  // padded entries are written as zeros
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < KS * KS * CP * NP; i += gridDim.x * blockDim.x) {
    const int tap = i / (CP * NP), rr = i % (CP * NP), ci = rr / NP, co = rr % NP;
    const int kc = ci / Q::KC, kq = ci % Q::KC;
    const __nv_bfloat16 v = ci < CIN && co < COUT ? w[((size_t)tap * CIN + ci) * COUT + co] : __float2bfloat16(0.f);
    *reinterpret_cast<__nv_bfloat16*>(img + (size_t)(kc * Q::TAPS + tap) * Q::WCH + (kq / 8) * Q::PW + co * 16 +
                                      (kq % 8) * 2) = v;
    if constexpr (P::USE) {
      const int h = co / P::NS, within = co % P::NS, rk = within / P::NHS, row = h * P::NHS + within % P::NHS;
      *reinterpret_cast<__nv_bfloat16*>(img + Q::WBYTES + ((size_t)(kc * Q::TAPS + tap) * 2 + rk) * P::WCHR +
                                        (kq / 8) * P::PWR + row * 16 + (kq % 8) * 2) = v;
    }
  }
}

// Sparse mode: tile an obh x obw output block with the fewest th x tw tiles (th*tw <= 128
// GEMM rows, TMA box extents tw*sx, th*sy <= 256); one tile when the block fits.
static bool sparse_tile_shape(int obh, int obw, int sy, int sx, int& th, int& tw, int& subs_y, int& subs_x) {
  int best = 1 << 30;
  for (int h = 1; h <= obh && h <= 128 && h * sy <= 256; ++h) {
    const int w = min(min(obw, 128 / h), 256 / sx);
    if (w < 1) continue;
    const int t = ((obh + h - 1) / h) * ((obw + w - 1) / w);
    if (t < best || (t == best && h * w > th * tw)) {
      best = t;
      th = h;
      tw = w;
    }
  }
  if (best == (1 << 30)) return false;
  subs_y = (obh + th - 1) / th;
  subs_x = (obw + tw - 1) / tw;
  return true;
}

template <int CIN, int COUT, int KS>
int launch_dense(const void* x, int n, int h, int w, int sy, int sx, int py, int px, int oh, int ow,
                 const void* wpk, const float* bias, void* out, cudaStream_t s,
                 const Geo* sparse = nullptr, const int32_t* idx = nullptr, const int32_t* count = nullptr,
                 int cap = 0, const __nv_bfloat16* bias_bf16 = nullptr, const uint8_t* mask = nullptr,
                 unsigned* slotw = nullptr, int32_t* gidx = nullptr) {
  using Q = CCfg<CIN, COUT, KS>;
  CArgs a;
  memset(&a, 0, sizeof(a));
  int th = 8, tw = 16, subs_y = 1, subs_x = 1;
  if (sparse) sparse_tile_shape(sparse->obh, sparse->obw, sy, sx, th, tw, subs_y, subs_x);
  const uint64_t dims[4] = {(uint64_t)CIN, (uint64_t)w, (uint64_t)h, (uint64_t)n};
  const uint64_t str[3] = {(uint64_t)CIN * 2, (uint64_t)w * CIN * 2, (uint64_t)h * w * CIN * 2};
  const uint32_t box[4] = {(uint32_t)Q::KC, (uint32_t)(tw * sx), (uint32_t)(th * sy), 1};
  const uint32_t es[4] = {1, (uint32_t)sx, (uint32_t)sy, 1};
  int st = encode_map(&a.tmap, x, 4, dims, str, box,
                      Q::KC == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : Q::KC == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B, es);
  if (st) return st;
  a.out = (__nv_bfloat16*)out;
  a.wpk = (const uint8_t*)wpk;
  a.bias = bias;
  a.n = n;
  a.oh = oh;
  a.ow = ow;
  a.sy = sy;
  a.sx = sx;
  a.py = py;
  a.px = px;
  a.bias_bf16 = bias_bf16;
  a.th = th;
  a.tw = tw;
  a.tiles_y = (oh + th - 1) / th;
  a.tiles_x = (ow + tw - 1) / tw;
  long tiles = (long)n * a.tiles_y * a.tiles_x;
  if (sparse) {
    a.idx = idx;
    a.count = count;
    a.cap = cap;
    a.gsy = sparse->sy;
    a.gsx = sparse->sx;
    a.goy = sparse->oy;
    a.gox = sparse->ox;
    a.obh = sparse->obh;
    a.obw = sparse->obw;
    a.subs_y = subs_y;
    a.subs_x = subs_x;
    tiles = (long)cap * subs_y * subs_x;
    if (mask) {  // one CTA per candidate up to the SM count, <= kMaxLocalTma candidates each
      a.idx = nullptr;
      a.mask = mask;
      a.gy = sparse->gy;
      a.gx = sparse->gx;
      a.wbh = sparse->bh;
      a.wbw = sparse->bw;
      a.n_h = h;
      a.n_w = w;
      tiles = (long)sparse->n * sparse->gy * sparse->gx * subs_y * subs_x;  // (candidate, sub-tile) units
      if (gidx) {  // global-list mode: every co-resident CTA tests candidates and strides the list
        const long slots = (long)Q::CPS * sm_count();
        const long cands = (long)sparse->n * sparse->gy * sparse->gx;
        if ((cands + slots - 1) / slots > kMaxGlobTma) {
          set_error("mask-fused tap-GEMM conv: %ld candidates exceed %d per CTA", cands, kMaxGlobTma);
          return SBN_ERR_UNSUPPORTED;
        }
        a.gidx = gidx;
        a.sw = slotw;
        tiles = slots;
      } else if (tiles > (long)kMaxLocalTma * Q::CPS * sm_count()) {
        set_error("mask-fused tap-GEMM conv: %ld units exceed %d per CTA", tiles, kMaxLocalTma);
        return SBN_ERR_UNSUPPORTED;
      }
    }
  }
  if (!sparse && PCfg<CIN, COUT, KS>::USE && !(debug_flags() & kDebugDenseSingle)) return launch_dense_pair<CIN, COUT, KS>(a, s);
  auto kern = mask && !gidx ? conv_dense_kernel<CIN, COUT, KS, true> : conv_dense_kernel<CIN, COUT, KS, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Q::SMEM);
  cudaLaunchConfig_t cfg = {};
  const long slots = (long)Q::CPS * sm_count();
  cfg.gridDim = dim3((unsigned)(tiles < slots ? (tiles < 1 ? 1 : tiles) : slots));
  cfg.blockDim = dim3(kCThreads);
  cfg.dynamicSmemBytes = Q::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a);
  return launch_status(sparse ? "sparse_conv_tcgen05_tma" : "dense_conv_tcgen05");
}

// (CIN, COUT, KS): the config-4 stage projections (3x3) and square shapes at 1x1 / 3x3 / 5x5
#define SBN_DENSE_CONV_CONFIGS(X) \
  X(32, 96, 3)                    \
  X(96, 192, 3)                   \
  X(192, 256, 3)                  \
  X(256, 384, 3)                  \
  X(32, 32, 3)                    \
  X(64, 64, 3)                    \
  X(128, 128, 3)                  \
  X(64, 64, 1)                    \
  X(128, 128, 1)                  \
  X(32, 32, 5)                    \
  X(64, 64, 5)                    \
  X(24, 24, 3)                    \
  X(48, 48, 3)                    \
  X(96, 96, 3)

}  // namespace

// Sparse KxK conv (K = 1, 3, 5; stride <= K) through the same kernel: tile = active
// block, the out block (obh x obw <= 128 pixels) = one strided TMA box per (K-chunk, tap).
bool sparse_conv_tma_supported(int dtype, int cin, int cout, int kh, int kw, int sh, int sw, const Geo& g) {
  if (dtype != SBN_BF16 || kh != kw || sh != sw || sh < 1 || sh > kh || sh > 3) return false;
  int th = 0, tw = 0, subs_y = 0, subs_x = 0;
  if (!sparse_tile_shape(g.obh, g.obw, sh, sw, th, tw, subs_y, subs_x)) return false;
#define X(CI, CO, KS) if (cin == CI && cout == CO && kh == KS) return CCfg<CI, CO, KS>::SMEM <= max_smem_optin();
  SBN_DENSE_CONV_CONFIGS(X)
#undef X
  return false;
}

size_t sparse_conv_tma_packed_bytes(int cin, int cout, int k) {
#define X(CI, CO, KS) \
  if (cin == CI && cout == CO && k == KS) return (size_t)CCfg<CI, CO, KS>::WBYTES * (PCfg<CI, CO, KS>::USE ? 2 : 1);
  SBN_DENSE_CONV_CONFIGS(X)
#undef X
  return 0;
}

int sparse_conv_tma_pack(const void* w, int cin, int cout, int k, void* img, cudaStream_t s) {
#define X(CI, CO, KS)                                                                                      \
  if (cin == CI && cout == CO && k == KS) {                                                                \
    conv_dense_pack_kernel<CI, CO, KS><<<128, 256, 0, s>>>((const __nv_bfloat16*)w, (uint8_t*)img);      \
    return launch_status("conv_tma_pack");                                                                 \
  }
  SBN_DENSE_CONV_CONFIGS(X)
#undef X
  set_error("no tcgen05 tap-GEMM conv instantiation for cin=%d cout=%d kernel=%d", cin, cout, k);
  return SBN_ERR_UNSUPPORTED;
}

int sparse_conv_tma(const void* x, int cin, int cout, int k, int sh, int sw, const Geo& g, const void* wpk,
                    const void* bias, const int32_t* idx, const int32_t* count, int cap, void* dst,
                    cudaStream_t s) {
#define X(CI, CO, KS)                                                                                            \
  if (cin == CI && cout == CO && k == KS)                                                                        \
    return launch_dense<CI, CO, KS>(x, g.n, g.h, g.w, sh, sw, 0, 0, g.oh, g.ow, wpk, nullptr, dst, s, &g, idx, \
                                    count, cap, (const __nv_bfloat16*)bias);
  SBN_DENSE_CONV_CONFIGS(X)
#undef X
  set_error("no tcgen05 tap-GEMM conv instantiation for cin=%d cout=%d kernel=%d", cin, cout, k);
  return SBN_ERR_UNSUPPORTED;
}

// Mask-fused variant for small grids (<= 2 (candidate, sub-tile) units per SM: the local lists
// are then as balanced as a striped global list); SBN_ERR_UNSUPPORTED above that, and the
// caller reduces the mask separately.
int sparse_conv_tma_masked(const void* x, const uint8_t* mask, int cin, int cout, int k, int sh, int sw,
                           const Geo& g, const void* wpk, const void* bias, void* dst, cudaStream_t s,
                           unsigned* slotw, int32_t* gidx) {
  int th = 0, tw = 0, subs_y = 1, subs_x = 1;
  if (!sparse_tile_shape(g.obh, g.obw, sh, sw, th, tw, subs_y, subs_x)) return SBN_ERR_UNSUPPORTED;
  const long units = (long)g.n * g.gy * g.gx * subs_y * subs_x;
  // local lists while every CTA slot owns few units; otherwise the global list (when the
  // caller passed its sync words and list buffer); otherwise the caller reduces the mask
  // (default for windows of 128..512 pixels, where one warp's test of a candidate is one
  // round of loads and the conv is short: Table-1 conv-2 with 16x16 blocks 13.1 -> 12.1 us;
  // 8x8 and 32x32 windows measured as fast or faster with reduce_mask + the list launch;
  // SBN_DEBUG_TMA_GLOBAL_LIST forces it for any window)
  const int area = g.bh * g.bw;
  const bool glob_ok = slotw && gidx && ((debug_flags() & kDebugTmaGlobalList) || (area >= 128 && area <= 512));
#define X(CI, CO, KS)                                                                                            \
  if (cin == CI && cout == CO && k == KS) {                                                                      \
    const bool local = units <= (long)SBN_FUSED_UNITS_PER_CTA * CCfg<CI, CO, KS>::CPS * sm_count();           \
    if (!local && !glob_ok) return SBN_ERR_UNSUPPORTED;                                                        \
    return launch_dense<CI, CO, KS>(x, g.n, g.h, g.w, sh, sw, 0, 0, g.oh, g.ow, wpk, nullptr, dst, s, &g, nullptr, \
                                    nullptr, g.n * g.gy * g.gx, (const __nv_bfloat16*)bias, mask,              \
                                    local ? nullptr : slotw, local ? nullptr : gidx);                          \
  }
  SBN_DENSE_CONV_CONFIGS(X)
#undef X
  return SBN_ERR_UNSUPPORTED;
}

}  // namespace sbn

using namespace sbn;

extern "C" int sbn_dense_conv_supported(int dtype, int cin, int cout, int kh, int kw, int sh, int sw) {
  if (dtype != SBN_BF16 || kh != kw || sh != sw || sh < 1 || sh > kh || sh > 3) return 0;
#define X(CI, CO, KS) if (cin == CI && cout == CO && kh == KS) return CCfg<CI, CO, KS>::SMEM <= max_smem_optin() ? 1 : 0;
  SBN_DENSE_CONV_CONFIGS(X)
#undef X
  return 0;
}

extern "C" size_t sbn_dense_conv_packed_bytes(int cin, int cout, int k) { return sparse_conv_tma_packed_bytes(cin, cout, k); }

extern "C" int sbn_dense_conv_pack(const void* w, int cin, int cout, int k, void* packed, sbn_stream_t stream) {
  SBN_CHECK_ARG(w && packed, SBN_ERR_INVALID, "null argument");
  return sparse_conv_tma_pack(w, cin, cout, k, packed, (cudaStream_t)stream);
}

extern "C" int sbn_dense_conv(const void* x, int n, int h, int w, int cin, int cout, int k, int sh, int sw,
                              int ph, int pw, int oh, int ow, const void* packed, const float* bias, void* out,
                              sbn_stream_t stream) {
  SBN_CHECK_ARG(x && packed && bias && out, SBN_ERR_INVALID, "null pointer argument");
  SBN_CHECK_ARG(n > 0 && h > 0 && w > 0 && oh > 0 && ow > 0, SBN_ERR_SHAPE, "bad dims");
  SBN_CHECK_ARG(sbn_dense_conv_supported(SBN_BF16, cin, cout, k, k, sh, sw), SBN_ERR_UNSUPPORTED,
                "tcgen05 dense conv does not support cin=%d cout=%d kernel %d stride (%d,%d)", cin, cout, k, sh, sw);
  cudaStream_t s = (cudaStream_t)stream;
#define X(CI, CO, KS)                                                                                       \
  if (cin == CI && cout == CO && k == KS)                                                                   \
    return launch_dense<CI, CO, KS>(x, n, h, w, sh, sw, ph, pw, oh, ow, packed, bias, out, s);
  SBN_DENSE_CONV_CONFIGS(X)
#undef X
  return SBN_ERR_UNSUPPORTED;
}
