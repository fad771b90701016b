// tcgen05 / TMEM sparse residual unit for wide channel counts (bf16, pre-activation,
// halo 1): the bottleneck of reference `_unit_branch` (`layers.py:155-169`) as three
// warp-specialised implicit-GEMM launches over the stacked active windows.
//
// The single-kernel unit (unit_tc.cu) keeps the whole window, A2/A3 and all three
// weight sets resident in one CTA's shared memory; that stops fitting beyond c ~ 128
// (c=384/m=192: 1 MB of weights, 196 KB of window).  The backbone stages of BASELINE
// config 4 (c = 96/192/256/384, m = c/2) run here instead.  Rows are the pixels of the
// active windows stacked "tall" (block j's window pixel (wy, wx) is row j*b*b + wy*b + wx),
// so small blocks pack densely into 128-row UMMA tiles and the 3x3 stays a row-shifted
// view of one staged operand:
//
//   IN   rows = window pixels      A = relu(bn1(x window))       (gathered, zero-filled)
//        D = A . W1  -> +b1, bn2, relu, x in-bounds -> S1 [B*b*b, m]   (bf16 stack)
//   MID  rows = window pixels q    D[q] = sum_taps S1[q + ky*b + kx] . W2[ky,kx]
//        -> +b2, bn3, relu -> S2 [B*(b-2)^2, m] (only q with oy, ox < b-2 are kept)
//   OUT  rows = output pixels      D = S2 . W3 -> +b3, + x  -> out at the block's
//        interior, clipped (the scatter-add of `layers.py:224-229`)
//
// Kernel order resolves the in-place hazard (IN reads every window before OUT writes any
// interior), so there is no rim snapshot and no grid barrier.  Launches chain with
// programmatic dependent launch; S1/S2 stay mostly in L2.
//
// Operands arrive by TMA (cp.async.bulk.tensor): one box per 16-byte channel plane lands
// as R rows x 16 B — exactly the K-major plane layout of tc_util.cuh.  IN gathers straight
// from x with a 4-D map (C, W, H, N) and a box of (8 ch, b, hb rows, 1 frame) at the
// block's (possibly negative) window origin: TMA zero-fills out-of-image pixels, so the
// gather's halo semantics (`blocks.py:66-73`) come for free.  MID/OUT read the stacks
// through 2-D maps.
//
// Warp roles per persistent CTA (576 threads):
//   warps 0-7   IN only: BN1 + ReLU in place on each landed chunk (pair-of-planes
//               mapping, conflict-free)
//   warps 8-15  epilogue: tcgen05.ld of the accumulator (TMEM lane quarter = warp % 4,
//               two warps per quarter split the columns), transform, vector stores;
//               double-buffered accumulators when 2*N <= 512
//   warp 16     loader: TMA boxes of A chunks into an SA-deep ring, weight chunks (all
//               resident, or streamed through an SW ring)
//   warp 17     MMA issuer (one thread): tcgen05.mma M=128, N<=256 per instruction
#include "unit.cuh"
#include "tc_util.cuh"

#include "tma_util.cuh"

#include <cstring>

namespace sbn {
namespace {

constexpr int kAThreads = 256;
constexpr int kEThreads = 256;
constexpr int kWideThreads = kAThreads + kEThreads + 64;
constexpr int kOutCopy = kAThreads + kEThreads;  // OUT: threads in the staged copy phase
#ifndef SBN_WIDE_MAX_ROWS
#define SBN_WIDE_MAX_ROWS 200
#endif
constexpr int kMaxRows = SBN_WIDE_MAX_ROWS;  // staged rows of a MID tile: 128 + 2*b + 2 (200: b <= 35; backbone time unchanged vs 168)

enum { kIn = 1, kMid = 2, kOut = 3 };

constexpr int kBudget = 216 * 1024;

// K-chunk choice: the largest of {K (<= 96), 64, 32, 16} that keeps ALL weight chunks
// resident in shared memory next to a 3-deep A ring; 0 when no chunking does (weights
// are then streamed through a ring).
// OUT with N <= 96: the residual tiles are prefetched into shared memory by the (otherwise
// idle) A warps, two tiles ahead of the epilogue.  Wider N would have to give up A-ring depth
// for the buffers (measured slower at N = 192 with one buffer), so they keep the copy phase.
constexpr int out_res_bufs(int mode, int n) { return mode != kOut || n > 96 ? 0 : 2; }
constexpr long out_res_bytes(int mode, int n) { return (long)out_res_bufs(mode, n) * 128L * (n * 2 + 16); }

template <int K, int N, int MODE>
constexpr int resident_kc() {
  constexpr int taps = MODE == kMid ? 9 : 1;
  constexpr int ra = MODE == kMid ? kMaxRows : 128;
  constexpr long wbytes = (long)taps * K * N * 2;
  // IN stages its operand as swizzled rows of KC channels (64 -> SWIZZLE_128B, 32 ->
  // SWIZZLE_64B); MID/OUT use the 16-byte plane layout
  constexpr int pref = MODE == kIn ? (K % 64 == 0 ? 64 : 32) : K <= 96 ? K : (K % 64 == 0 ? 64 : 32);
  constexpr int cands[4] = {pref, 64, 32, 16};
  for (int i = 0; i < 4; ++i) {
    const int kc = cands[i];
    if (kc > pref || K % kc != 0 || kc % 16 != 0 || (MODE == kIn && kc != 64 && kc != 32)) continue;
    const long ach = (long)(kc / 8) * ra * 16;
    const long stg = (MODE == kOut ? 128L * ((N <= 192 ? N : 128) * 2 + 16) : 0) + out_res_bytes(MODE, N);
    if (2 * ach + wbytes + 8192 + stg <= kBudget) return kc;
  }
  return 0;
}

template <int K, int N, int MODE>
struct WCfg {
  static constexpr int TAPS = MODE == kMid ? 9 : 1;
  static constexpr int RKC = resident_kc<K, N, MODE>();
  static constexpr bool RES = RKC != 0;  // weights resident for the whole kernel
  static constexpr int KC = RES ? RKC : (K % 64 == 0 ? 64 : 32);
  static_assert(K % KC == 0 && KC % 16 == 0, "K chunking");
  static_assert(MODE != kIn || KC == 64 || KC == 32, "IN: swizzled 128-B / 64-B rows");
  static constexpr int ROWB = KC * 2;                      // IN: bytes per staged row
  static constexpr uint32_t SWZ = KC == 64 ? 2u : 4u;      // IN: UMMA layout type (SW128 / SW64)
  static constexpr int NKC = K / KC;
  static constexpr int P = KC / 8;         // 16-byte planes per chunk
  static constexpr int RA = MODE == kMid ? kMaxRows : 128;
  static constexpr int PA = RA * 16;       // A plane stride (multiple of 128: TMA destination)
  static constexpr int ACH = P * PA;
  static constexpr int PW = N * 16;
  static constexpr int WCH = P * PW;
  static constexpr int NSPLIT = N > 256 ? 2 : 1;
  static constexpr int NS = N / NSPLIT;
  static_assert(N % NSPLIT == 0 && NS % 16 == 0 && NS <= 256, "UMMA N");
  static constexpr int NACC = 2 * N <= 512 ? 2 : 1;
  static constexpr int TCOLS = NACC * N;
  static_assert(TCOLS <= 512, "TMEM budget");
  static constexpr int TALLOC = TCOLS <= 32 ? 32 : TCOLS <= 64 ? 64 : TCOLS <= 128 ? 128 : TCOLS <= 256 ? 256 : 512;
  static constexpr int NPAR = MODE == kIn ? 2 * K + 3 * N : MODE == kMid ? 3 * N : N;
  static constexpr int al(int v) { return (v + 127) / 128 * 128; }
  static constexpr int PARB = al(NPAR * 4);
  // OUT: the epilogue stages bf16(acc + b3) for GS columns at a time, then copies whole
  // pixel rows with the residual add (coalesced 16-B lanes along each row)
  static constexpr int GS = MODE != kOut ? 0 : (N <= 192 ? N : 128);
  static constexpr int SPITCH = GS * 2 + 16;
  static constexpr int STGB = MODE == kOut ? 128 * SPITCH : 0;
  static constexpr int NRB = out_res_bufs(MODE, N);      // prefetched residual tiles (OUT)
  static constexpr bool PF = NRB > 0;
  static constexpr int RESB = 128 * SPITCH;              // one residual tile, same pitch as stg
  static constexpr int CHUNKS = NKC * TAPS;                       // weight chunks per tile
  static constexpr size_t WBYTES = (size_t)CHUNKS * WCH;          // packed weight bytes
  // resident: A ring as deep as fits (<= 6); streamed: A ring 2..4, W ring 2..4
  static constexpr int BUD = kBudget - STGB - NRB * RESB;
  static constexpr int SA = RES ? ((int)((BUD - (long)WBYTES - PARB) / ACH) > 6 ? 6 : (int)((BUD - (long)WBYTES - PARB) / ACH))
                                : (4 * ACH + 2 * WCH + PARB <= BUD) ? 4 : (3 * ACH + 2 * WCH + PARB <= BUD) ? 3 : 2;
  static constexpr int SW = RES ? 0 : (SA * ACH + 4 * WCH + PARB <= BUD) ? 4 : (SA * ACH + 3 * WCH + PARB <= BUD) ? 3 : 2;
  static constexpr long WREG = RES ? (long)WBYTES : (long)SW * WCH;
  static_assert(SA >= 2 && SA * ACH + WREG + PARB <= BUD, "shared memory budget");
  static constexpr int OFF_W = SA * ACH;
  static constexpr int OFF_PAR = OFF_W + (int)WREG;
  static constexpr int OFF_STG = OFF_PAR + PARB;
  static constexpr int OFF_RES = OFF_STG + STGB;
  static constexpr int SMEM = OFF_RES + NRB * RESB;
  static constexpr int ITEMS = (128 * P + kAThreads / 2 - 1) / (kAThreads / 2);  // IN pieces per thread
  // column slices (OUT): when a launch has too few tiles to fill the grid, each tile is done
  // as two work items of N/2 output columns on different CTAs (same A, half the weights).
  // The k-step order of every accumulator column is unchanged, so results are identical.
  // (Measured on the config-4 stage-3 unit: OUT 13.4 -> 11.4 us; IN and MID got slower —
  // the duplicated A / BN work and MID's streamed weights in plane pieces cost more than the
  // shorter makespan saves — so only OUT slices.)
  static constexpr bool SPL = MODE == kOut && !PF && N >= 128 && (N / 2) % 16 == 0;
  static constexpr int N2 = N / 2;
  static constexpr int NSPLIT2 = N2 > 256 ? 2 : 1;
  static constexpr int NS2 = SPL ? N2 / NSPLIT2 : NS;
  static constexpr int GSH = MODE != kOut || !SPL ? (GS > 0 ? GS : 16) : N2 <= GS ? N2 : N2 % GS == 0 ? GS : N2 / 2;
  static_assert(!SPL || MODE != kOut || (N2 % GSH == 0 && GSH % 16 == 0 && GSH <= GS), "slice staging groups");
};

// Stacks S1 / S2 are stored PLANE-MAJOR: plane k (channels 8k..8k+7) of row r at
// (k * rows_alloc + r) * 16 bytes, so a tile's plane is one contiguous run (a 1-D bulk
// copy) and the epilogues' row-per-lane stores are coalesced.  rows_alloc carries
// kStackPad spare rows so MID's over-reading last tile stays inside the allocation.
constexpr int kStackPad = 256;

struct __align__(64) WArgs {
  CUtensorMap tmap;          // IN: x as (C, W, H, N), swizzled KC-channel boxes
  __nv_bfloat16* dst;        // IN: S1   MID: S2    OUT: out
  const uint8_t* wpk;        // this GEMM's packed weight chunks
  const float* par;          // this GEMM's parameter vectors
  const uint8_t* wpk2;       // fused unit: W2 chunks
  const float* par2;         // fused unit: MID's parameter vectors
  const uint8_t* wpk3;       // fused unit: W3 chunks
  const float* par3;         // fused unit: OUT's parameter vectors
  const __nv_bfloat16* rim;  // fused unit in place: rim snapshot (cap, 60, C), else null
  Geo g;
  const int32_t* idx;
  const int32_t* count;
  int cap;
  int hb, S, G;              // IN: window rows per slab, slabs per block, slabs per tile
  int slab_rows;             // IN: tile rows per slab (hb*b rounded to 8: 128-B aligned TMA boxes)
  int box_rows;              // MID: rows per A box (128 + 2b + 2, rounded to 8)
  const uint8_t* stack;      // MID / OUT: plane-major source stack
  long src_rows;             // MID / OUT: rows_alloc of the source stack (plane stride / 16)
  long dst_rows;             // IN / MID: rows_alloc of the destination stack
  unsigned long long* trace; // diagnostics: CTA 0 event stamps (sbn_debug_set_trace)
  int split;                 // column slices allowed (WCfg::SPL launches with few tiles)
};

// CTA 0 event log (diagnostics): slot ev*64 + tile, tiles < 64
enum { kEvPub = 0, kEvMma = 1, kEvAcc = 2, kEvEpi = 3, kEvIss = 4, kEvLoad = 5, kEvCIss = 7, kEvCData = 8, kEvCPub = 11 };
// (diagnostics build only: the stamps' checks and live registers slow the single-thread
// MMA issuers; tools/build_variant.sh trace -DSBN_TRACE_WIDE, then SBN_LIB_PATH=tools/bin/trace.so)
__device__ __forceinline__ void wtrace(const WArgs& a, int ev, int t) {
#ifdef SBN_TRACE_WIDE
  if (a.trace && blockIdx.x == 0 && t < 64) {
    a.trace[ev * 64 + t] = gtimer();
    a.trace[1024 + ev * 64 + t] = clock64();
  }
#else
  (void)a;
  (void)ev;
  (void)t;
#endif
}

// tiles of the GEMM for B active blocks of size b
template <int MODE>
__device__ __forceinline__ int tile_count(const WArgs& a, int B, int b) {
  if (MODE == kIn) return (B * a.S + a.G - 1) / a.G;
  const long rows = MODE == kOut ? (long)B * (b - 2) * (b - 2) : (long)B * b * b;
  return (int)((rows + 127) / 128);
}

// OUT copy phase, shared by the idle A warps and the epilogue warps (kOutCopy threads,
// copy index `ct`): wait for the staged bf16(acc + b3) group, then along whole output pixel
// rows load the residual, add, store (coalesced 16-B vectors), and release the staging
// buffer.  Inlined at both call sites, so the barrier is the non-.aligned form.
template <int SPITCH, int CHR, int IT2>
__device__ __forceinline__ void out_copy_phase(__nv_bfloat16* dst, const uint8_t* stg, const long long* rowdst, int g0,
                                            int ct) {
  constexpr int BATCH = IT2 < 6 ? IT2 : 6;  // residual loads in flight per thread
  tc::named_bar_any<3, kOutCopy>();
#pragma unroll 1
  for (int jb = 0; jb < IT2; jb += BATCH) {
    uint4 xr[BATCH];
#pragma unroll
    for (int jj = 0; jj < BATCH; ++jj) {
      const int it = ct + (jb + jj) * kOutCopy;
      const long long off = (jb + jj < IT2 && it < 128 * CHR) ? rowdst[it / CHR] : -1;
      xr[jj] = tc::ld_v4_pred(reinterpret_cast<const uint4*>(dst + (off >= 0 ? off + g0 : 0)) + it % CHR, off >= 0);
    }
#pragma unroll
    for (int jj = 0; jj < BATCH; ++jj) {
      const int it = ct + (jb + jj) * kOutCopy;
      if (jb + jj >= IT2 || it >= 128 * CHR) break;
      const int row = it / CHR, ch = it % CHR;
      const long long off = rowdst[row];
      if (off < 0) continue;
      const uint4 sv = *reinterpret_cast<const uint4*>(stg + row * SPITCH + ch * 16);
      const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xr[jj]);
      const __nv_bfloat162* uh = reinterpret_cast<const __nv_bfloat162*>(&sv);
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 xf = __bfloat1622float2(xh[q]), uf = __bfloat1622float2(uh[q]);
        o[q] = tc::pack_bf16(xf.x + uf.x, xf.y + uf.y);
      }
      reinterpret_cast<uint4*>(dst + off + g0)[ch] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
  tc::named_bar_any<3, kOutCopy>();  // staging / rowdst reuse
}

template <int K, int N, int MODE>
__global__ void __launch_bounds__(kWideThreads, 1) unit_wide_kernel(const __grid_constant__ WArgs a) {
  using Q = WCfg<K, N, MODE>;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int SWB = Q::SW > 0 ? Q::SW : 1;
  __shared__ uint64_t a_load[Q::SA], a_full[Q::SA], a_empty[Q::SA], w_full[SWB], w_empty[SWB];
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tslot;
  __shared__ long long rowdst[MODE == kOut ? 128 : 1];  // OUT: element offset of a row's pixel, -1 skip
  constexpr int NRBS = Q::NRB > 0 ? Q::NRB : 1;
  __shared__ long long rowres[NRBS][Q::PF ? 128 : 1];    // OUT prefetch: row offsets of a buffered tile
  __shared__ uint64_t res_full[NRBS], res_empty[NRBS];
  uint8_t* Aring = smem;
  uint8_t* Wring = smem + Q::OFF_W;
  float* par = reinterpret_cast<float*>(smem + Q::OFF_PAR);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Geo& g = a.g;
  const int b = g.bh;
  constexpr int kLWarp = (kAThreads + kEThreads) / 32, kMWarp = kLWarp + 1;

  if (tid == 0) {
    for (int s = 0; s < Q::SA; ++s) {
      tc::mbar_init(&a_load[s], 1);
      tc::mbar_init(&a_full[s], MODE == kIn ? kAThreads / 2 : 1);
      tc::mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < SWB; ++s) {
      tc::mbar_init(&w_full[s], 1);
      tc::mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < NRBS; ++s) {
      tc::mbar_init(&res_full[s], 2 * kAThreads);  // a st.shared release + a cp.async completion per A thread
      tc::mbar_init(&res_empty[s], kEThreads);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&acc_full[s], 1);
      tc::mbar_init(&acc_empty[s], kEThreads);
    }
    tc::mbar_fence_init();
  }
  if (MODE == kIn && tid == kLWarp * 32) asm volatile("prefetch.tensormap [%0];" ::"l"(&a.tmap) : "memory");
  for (int i = tid; i < Q::NPAR; i += kWideThreads) par[i] = a.par[i];
  if (warp == 0) tc::tmem_alloc<Q::TALLOC>(&tslot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  tc::pdl_trigger();
  if (Q::RES && tid == kLWarp * 32) {
    // resident weights: every chunk lands once, under the previous kernel's tail (weights
    // do not depend on it), completion on w_full[0]
    tc::mbar_expect_tx(&w_full[0], (uint32_t)Q::WBYTES);
    for (int c = 0; c < Q::CHUNKS; ++c)
      tc::bulk_g2s(Wring + (size_t)c * Q::WCH, a.wpk + (size_t)c * Q::WCH, Q::WCH, &w_full[0]);
  }
  tc::pdl_wait();  // the previous launch's S1 / S2 / x and the index list are visible
  const int B = ld_count(a.count, a.cap);
  const int ntiles = tile_count<MODE>(a, B, b);
  // column slices (WCfg::SPL): ns = 2 work items per tile when that shortens the makespan
  // (a half-width item costs ~0.6 of a tile: same A operand, half the MMA columns)
  int ns = 1;
  if constexpr (Q::SPL) {
    const int G = gridDim.x, r1 = (ntiles + G - 1) / G, r2 = (2 * ntiles + G - 1) / G;
    if (a.split && 3 * r2 < 5 * r1) ns = 2;
  }
  const int lg = ns - 1;                     // tile = w >> lg, slice = w & lg
  const int nwork = ntiles << lg;
  const int W = N >> lg;                     // output columns per work item
  const int nacc = lg ? (2 * W <= Q::TALLOC ? 2 : 1) : Q::NACC;

  if (tid < kAThreads) {
    // ------------------------------------------------ IN: BN1 + ReLU on landed chunks
    if (MODE == kIn) {
      // one 16-B piece per item: consecutive threads walk the pieces of consecutive rows
      // (conflict-free); the piece in physical slot q of row r holds channel group
      // q ^ swizzle(r) of the chunk
      // two groups of 4 warps take alternate chunks, so two chunks are in flight
      const float* s1 = par;  // packed sign / shift pairs (see unit_wide_pack_kernel)
      constexpr int PR = Q::ROWB / 16;  // pieces per row
      constexpr int TG = kAThreads / 2;
      const int grp_id = tid / TG, gt = tid % TG;
      int c = 0;
      for (int w = blockIdx.x; w < nwork; w += gridDim.x)
        for (int kc = 0; kc < Q::NKC; ++kc, ++c) {
          if ((c & 1) != grp_id) continue;
          const int s = c % Q::SA;
          tc::mbar_wait(&a_load[s], (c / Q::SA) & 1);
          if (gt == 0) wtrace(a, kEvCData, c);
          uint8_t* A = Aring + s * Q::ACH;
          uint4 raw[Q::ITEMS];
#pragma unroll
          for (int j = 0; j < Q::ITEMS; ++j) {
            const int i = gt + j * TG;
            if (i < 128 * PR)
              asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(raw[j].x), "=r"(raw[j].y), "=r"(raw[j].z), "=r"(raw[j].w)
                           : "r"(tc::smem_u32(A + i * 16)));
          }
#pragma unroll
          for (int j = 0; j < Q::ITEMS; ++j) {
            const int i = gt + j * TG;
            if (i >= 128 * PR) break;
            const int r = i / PR, qp = i % PR;
            const int grp = qp ^ (Q::KC == 64 ? (r & 7) : ((r >> 1) & 3));
            // relu(sgn * x + v) in packed bf16 (|s1| lives in W1)
            const uint4 sg4 = *reinterpret_cast<const uint4*>(s1 + (kc * Q::KC + grp * 8) / 2);
            const uint4 vv4 = *reinterpret_cast<const uint4*>(s1 + K / 2 + (kc * Q::KC + grp * 8) / 2);
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[j]);
            const __nv_bfloat162* hs = reinterpret_cast<const __nv_bfloat162*>(&sg4);
            const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&vv4);
            const __nv_bfloat162 z2 = __float2bfloat162_rn(0.f);
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const __nv_bfloat162 y = __hmax2(__hfma2(h[e], hs[e], hv[e]), z2);
              o[e] = *reinterpret_cast<const uint32_t*>(&y);
            }
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(tc::smem_u32(A + i * 16)), "r"(o[0]),
                         "r"(o[1]), "r"(o[2]), "r"(o[3])
                         : "memory");
          }
          tc::fence_async_smem();
          tc::mbar_arrive(&a_full[s]);
          if (gt == 0 && kc == Q::NKC - 1) wtrace(a, kEvPub, c / Q::NKC);
          if (gt == 0) wtrace(a, kEvCPub, c);
        }
    }
    if constexpr (MODE == kOut && Q::PF) {
      // OUT, one staging group: these warps prefetch each tile's residual (x at the output
      // pixels, in place) into a shared buffer NRB tiles ahead of the epilogue — row
      // offsets from the block list, then 16-byte cp.async along pixel rows — so the
      // epilogue's copy reads both operands from shared memory and only stores.  Tiles are
      // disjoint in the output, so reading x ahead of earlier tiles' stores is safe; IN read
      // every window before this launch began (kernel order).
      constexpr int CHR = N * 2 / 16;
      const int ob = b - 2;
      const long TR = (long)B * ob * ob;
      int kk = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++kk) {
        const int rb = kk % Q::NRB;
        tc::mbar_wait(&res_empty[rb], ((kk / Q::NRB) & 1) ^ 1);
        if (tid < 128) {
          const long gr = (long)tile * 128 + tid;
          long long off = -1;
          if (gr < TR) {
            const int j = (int)(gr / (ob * ob)), pp = (int)(gr - (long)j * ob * ob);
            const int Y = __ldg(a.idx + 3 * j + 1) * g.obh + pp / ob, X = __ldg(a.idx + 3 * j + 2) * g.obw + pp % ob;
            if (Y < g.oh && X < g.ow) off = (((long long)__ldg(a.idx + 3 * j) * g.oh + Y) * g.ow + X) * N;
          }
          rowres[rb][tid] = off;
        }
        tc::named_bar<4, kAThreads>();  // this tile's row offsets are visible to every A thread
        uint8_t* rbuf = smem + Q::OFF_RES + rb * Q::RESB;
        for (int it = tid; it < 128 * CHR; it += kAThreads) {
          const int row = it / CHR, ch = it - row * CHR;
          const long long off = rowres[rb][row];
          tc::cp_async16(rbuf + row * Q::SPITCH + ch * 16, a.dst + (off >= 0 ? off + ch * 8 : 0), off >= 0);
        }
        tc::mbar_arrive(&res_full[rb]);  // releases the row offsets
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&res_full[rb]))
                     : "memory");
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if constexpr (MODE == kOut) {
      // OUT: these warps have no operand transform; they join the epilogue's staged copy
      // phase (residual add along pixel rows), same barrier sequence as the epilogue warps
      constexpr int GS = Q::GS, CHR = GS * 2 / 16;
      constexpr int IT2 = (128 * CHR + kOutCopy - 1) / kOutCopy;
      const uint8_t* stg = smem + Q::OFF_STG;
      for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
        if (Q::SPL && lg) {
          constexpr int CHRH = Q::GSH * 2 / 16, IT2H = (128 * CHRH + kOutCopy - 1) / kOutCopy;
          for (int g0 = 0; g0 < Q::N2; g0 += Q::GSH)
            out_copy_phase<Q::SPITCH, CHRH, IT2H>(a.dst + (w & 1) * Q::N2, stg, rowdst, g0, tid);
        } else {
          for (int g0 = 0; g0 < N; g0 += GS) out_copy_phase<Q::SPITCH, CHR, IT2>(a.dst, stg, rowdst, g0, tid);
        }
      }
    }
  } else if (tid < kAThreads + kEThreads) {
    // ------------------------------------------------ epilogue
    // warp w drains TMEM lane quarter w % 4; the two warps of a quarter take alternate
    // 16-column chunks.  IN: relu(acc*s2 + t2'), x in-bounds (t2' = b1*s2 + t2, folded at
    // pack time); MID: relu(acc*s3 + t3'); OUT: x + acc + b3.  One bf16 rounding each.
    const int ew = warp - kAThreads / 32;
    const int qd = warp & 3, half = ew >> 2;
    const int r = qd * 32 + lane;
    const int bb = b * b, ob = b - 2;
    const long TR = MODE == kOut ? (long)B * ob * ob : (long)B * bb;
    constexpr int NCH = N / 16;                 // 16-column chunks
    constexpr int MYCH = (NCH + 1) / 2;         // chunks of this half (upper bound)
    const float* sc = MODE == kIn ? par + 2 * K + N : par + N;  // IN: s2 | MID: s3
    const float* sh = sc + N;                                     // t2' | t3'
    // per-row metadata of a tile; the block-index loads (IN, OUT) are issued one tile
    // ahead (idx_next) and consumed by meta() after the current tile's drain
    int xn = 0, xby = 0, xbx = 0;
    auto idx_next = [&](int tile) {
      const long gr = (long)tile * 128 + r;
      int j = -1;
      if (MODE == kIn) {
        const int i = r / a.slab_rows, sl = tile * a.G + i;
        if (i < a.G && sl < B * a.S) j = sl / a.S;
      } else if (MODE == kOut && gr < TR) {
        j = (int)(gr / (ob * ob));
      }
      if (j >= 0) {
        xn = __ldg(a.idx + 3 * j);
        xby = __ldg(a.idx + 3 * j + 1);
        xbx = __ldg(a.idx + 3 * j + 2);
      }
    };
    bool store = false, valid = true;
    __nv_bfloat16* dp = a.dst;   // OUT: the output pixel row
    long drow = 0;               // IN / MID: destination row of the plane-major stack
    auto meta = [&](int tile) {
      const long gr = (long)tile * 128 + r;
      store = (MODE == kIn || gr < TR) && tile < ntiles;
      valid = true;
      dp = a.dst;
      if (!store) return;
      if (MODE == kIn) {
        // tile = G slabs of hb window rows; this row -> (block j, window row wy, col wx)
        const int i = r / a.slab_rows, rr = r - i * a.slab_rows;
        const int sl = tile * a.G + i;
        const int j = sl / a.S, q = sl - j * a.S;
        const int wy = q * a.hb + rr / b, wx = rr % b;
        store = i < a.G && sl < B * a.S && rr < a.hb * b && wy < b;
        const int y = g.oy + xby * g.sy + wy, x = g.ox + xbx * g.sx + wx;
        valid = y >= 0 && y < g.h && x >= 0 && x < g.w;
        drow = (long)j * bb + wy * b + wx;
      } else if (MODE == kMid) {
        const int j = (int)(gr / bb), p = (int)(gr - (long)j * bb);
        const int oy = p / b, ox = p % b;
        store = oy < ob && ox < ob;
        drow = (long)j * ob * ob + oy * ob + ox;
      } else {
        const int j = (int)(gr / (ob * ob)), p = (int)(gr - (long)j * ob * ob);
        const int oy = p / ob, ox = p % ob;
        const int Y = xby * g.obh + oy, X = xbx * g.obw + ox;
        store = Y < g.oh && X < g.ow;
        dp = a.dst + (((long)xn * g.oh + Y) * g.ow + X) * N;  // residual read from the same row
      }
    };
    idx_next(blockIdx.x >> lg);
    meta(blockIdx.x >> lg);
    int k = 0;
    for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++k) {
      const int buf = nacc == 2 ? (k & 1) : 0;
      const int use = nacc == 2 ? (k >> 1) : k;
      const int nxt = (w + (int)gridDim.x) >> lg;  // the next work item's tile
      const int choff = (w & lg) * W;              // first output column of this item
      idx_next(nxt);
      const uint32_t acc = tmem + ((uint32_t)(qd * 32) << 16) + buf * W;
      tc::mbar_wait(&acc_full[buf], use & 1);
      tc::fence_after();
      if (ew == 0 && lane == 0) wtrace(a, kEvAcc, k);
      if constexpr (MODE == kOut) {
        // staged OUT epilogue: phase 1 writes bf16(acc + b3) of GS columns of this row to
        // smem; phase 2 walks (row, 16-B chunk) items so consecutive lanes cover one pixel
        // row: residual loads and stores are coalesced 16-B vectors
        static_assert(N % Q::GS == 0, "staging groups");
        uint8_t* stg = smem + Q::OFF_STG;
        const float* b3 = par + choff;
        if (half == 0) rowdst[r] = store ? (long long)(dp - a.dst) : -1;
        auto drain = [&](auto gs_c) {
        constexpr int GS = decltype(gs_c)::value, CHR = GS * 2 / 16;
        constexpr int IT2 = (128 * CHR + kOutCopy - 1) / kOutCopy;
        for (int g0 = 0; g0 < W; g0 += GS) {
#pragma unroll
          for (int e = 0; e < (GS / 16 + 1) / 2; ++e) {
            const int cg = 16 * (2 * e + half);  // column inside the group
            if (cg >= GS) break;                 // warp-uniform
            float v[16];
            tc::tmem_ld16(acc + g0 + cg, v);
            uint32_t o[8];
#pragma unroll
            for (int q = 0; q < 8; q += 2) {
              const float4 b4 = *reinterpret_cast<const float4*>(b3 + g0 + cg + 2 * q);
              o[q] = tc::pack_bf16(v[2 * q] + b4.x, v[2 * q + 1] + b4.y);
              o[q + 1] = tc::pack_bf16(v[2 * q + 2] + b4.z, v[2 * q + 3] + b4.w);
            }
            uint4* sp = reinterpret_cast<uint4*>(stg + r * Q::SPITCH + cg * 2);
            sp[0] = make_uint4(o[0], o[1], o[2], o[3]);
            sp[1] = make_uint4(o[4], o[5], o[6], o[7]);
          }
          if (g0 + GS >= W) {  // TMEM fully drained: release the accumulator early
            tc::fence_before();
            tc::mbar_arrive(&acc_empty[buf]);
          }
          if constexpr (Q::PF) {
            // staged bf16(acc + b3) + the prefetched residual -> out, coalesced along rows
            const int et = tid - kAThreads, rb = k % Q::NRB;
            tc::named_bar<5, kEThreads>();               // the whole tile is staged
            tc::mbar_wait(&res_full[rb], (k / Q::NRB) & 1);  // its residual has landed
            const uint8_t* rbuf = smem + Q::OFF_RES + rb * Q::RESB;
            for (int it = et; it < 128 * CHR; it += kEThreads) {
              const int row = it / CHR, ch = it - row * CHR;
              const long long off = rowres[rb][row];
              if (off < 0) continue;
              const uint4 sv = *reinterpret_cast<const uint4*>(stg + row * Q::SPITCH + ch * 16);
              const uint4 xv = *reinterpret_cast<const uint4*>(rbuf + row * Q::SPITCH + ch * 16);
              const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xv);
              const __nv_bfloat162* uh = reinterpret_cast<const __nv_bfloat162*>(&sv);
              uint32_t o[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float2 xf = __bfloat1622float2(xh[q]), uf = __bfloat1622float2(uh[q]);
                o[q] = tc::pack_bf16(xf.x + uf.x, xf.y + uf.y);
              }
              reinterpret_cast<uint4*>(a.dst + off)[ch] = make_uint4(o[0], o[1], o[2], o[3]);
            }
            tc::mbar_arrive(&res_empty[rb]);
            tc::named_bar<5, kEThreads>();  // staging buffer reuse
          } else {
            out_copy_phase<Q::SPITCH, CHR, IT2>(a.dst + choff, stg, rowdst, g0, tid);
          }
        }
        };
        if (Q::SPL && lg)
          drain(std::integral_constant<int, Q::GSH>());
        else
          drain(std::integral_constant<int, Q::GS>());
        if (ew == 0 && lane == 0) wtrace(a, kEvEpi, k);
        meta(nxt);
        continue;
      }
#pragma unroll
      for (int e = 0; e < MYCH; ++e) {
        const int c0 = 16 * (2 * e + half);
        if (c0 >= W) break;  // warp-uniform
        float v[16];
        tc::tmem_ld16(acc + c0, v);
        if (!store) continue;
        const int cc = choff + c0;  // output channel
        uint32_t o[8];
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          const float4 s4 = *reinterpret_cast<const float4*>(sc + cc + 2 * q);
          const float4 t4 = *reinterpret_cast<const float4*>(sh + cc + 2 * q);
          const float u0 = fmaxf(fmaf(v[2 * q], s4.x, t4.x), 0.f);
          const float u1 = fmaxf(fmaf(v[2 * q + 1], s4.y, t4.y), 0.f);
          const float u2 = fmaxf(fmaf(v[2 * q + 2], s4.z, t4.z), 0.f);
          const float u3 = fmaxf(fmaf(v[2 * q + 3], s4.w, t4.w), 0.f);
          o[q] = valid ? tc::pack_bf16(u0, u1) : 0u;
          o[q + 1] = valid ? tc::pack_bf16(u2, u3) : 0u;
        }
        // plane-major stack: lanes hold consecutive rows -> coalesced 16-B stores
        uint4* pl = reinterpret_cast<uint4*>(a.dst) + (long)(cc / 8) * a.dst_rows + drow;
        pl[0] = make_uint4(o[0], o[1], o[2], o[3]);
        pl[a.dst_rows] = make_uint4(o[4], o[5], o[6], o[7]);
      }
      tc::fence_before();
      tc::mbar_arrive(&acc_empty[buf]);
      if (ew == 0 && lane == 0) wtrace(a, kEvEpi, k);
      meta(nxt);
    }
  } else if (warp == kLWarp) {
    // ------------------------------------------------ loader: A boxes (+ streamed weights)
    if (lane == 0) {
      const int bb = b * b;
      int c = 0, wit = 0;
      // IN: the block-index triples of the NEXT tile's slabs are loaded one tile ahead
      int nj[4], nn[4], nby[4], nbx[4];
      auto idx_load = [&](int tile) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int sl = tile * a.G + i;
          nj[i] = (i < a.G && sl < B * a.S) ? sl : -1;
          if (nj[i] >= 0) {
            const int j = sl / a.S;
            nn[i] = __ldg(a.idx + 3 * j);
            nby[i] = __ldg(a.idx + 3 * j + 1);
            nbx[i] = __ldg(a.idx + 3 * j + 2);
          }
        }
      };
      if (MODE == kIn) idx_load(blockIdx.x >> lg);
      for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
        const int tile = w >> lg;
        int cj[4], cn[4], cby[4], cbx[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          cj[i] = nj[i];
          cn[i] = nn[i];
          cby[i] = nby[i];
          cbx[i] = nbx[i];
        }
        if (MODE == kIn) idx_load((w + (int)gridDim.x) >> lg);
        if (c % Q::NKC == 0) wtrace(a, kEvIss, c / Q::NKC);
        for (int kc = 0; kc < Q::NKC; ++kc, ++c) {
          const int s = c % Q::SA;
          tc::mbar_wait(&a_empty[s], ((c / Q::SA) & 1) ^ 1);
          uint8_t* A = Aring + s * Q::ACH;
          uint64_t* bar = MODE == kIn ? &a_load[s] : &a_full[s];
          wtrace(a, kEvCIss, c);
          if (MODE == kIn) {
            int boxes = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) boxes += cj[i] >= 0;
            tc::mbar_expect_tx(bar, (uint32_t)(boxes * Q::ROWB * b * a.hb));
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              if (cj[i] < 0) continue;
              const int q = cj[i] - (cj[i] / a.S) * a.S;
              const int x0 = g.ox + cbx[i] * g.sx, y0 = g.oy + cby[i] * g.sy + q * a.hb;
              // one box of (KC ch, b, hb rows) lands as swizzled KC-channel rows
              tma_4d(A + i * a.slab_rows * Q::ROWB, &a.tmap, kc * Q::KC, x0, y0, cn[i], bar);
            }
          } else {
            const int rows = MODE == kMid ? a.box_rows : 128;
            tc::mbar_expect_tx(bar, (uint32_t)(Q::P * 16 * rows));
            for (int k8 = 0; k8 < Q::P; ++k8)
              tc::bulk_g2s(A + k8 * Q::PA,
                           a.stack + ((long)(kc * Q::P + k8) * a.src_rows + (long)tile * 128) * 16,
                           (uint32_t)(rows * 16), bar);
          }
          if (!Q::RES) {  // streamed weights: this chunk's taps (a slice: its columns of every plane)
            for (int tap = 0; tap < Q::TAPS; ++tap, ++wit) {
              const int sw = wit % SWB;
              tc::mbar_wait(&w_empty[sw], ((wit / SWB) & 1) ^ 1);
              const uint8_t* wsrc = a.wpk + (size_t)(kc * Q::TAPS + tap) * Q::WCH;
              if (Q::SPL && lg) {
                const int co = (w & 1) * Q::N2 * 16;
                tc::mbar_expect_tx(&w_full[sw], Q::P * Q::N2 * 16);
                for (int p = 0; p < Q::P; ++p)
                  tc::bulk_g2s(Wring + sw * Q::WCH + p * Q::PW + co, wsrc + p * Q::PW + co, Q::N2 * 16, &w_full[sw]);
              } else {
                tc::mbar_expect_tx(&w_full[sw], Q::WCH);
                tc::bulk_g2s(Wring + sw * Q::WCH, wsrc, Q::WCH, &w_full[sw]);
              }
            }
          }
        }
        (void)bb;
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(128, Q::NS);
      constexpr uint32_t idesc2 = tc::idesc_bf16_f32(128, Q::NS2);
      int ait = 0, wit = 0, k = 0;
      if (Q::RES) tc::mbar_wait(&w_full[0], 0);
      for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++k) {
        const int buf = nacc == 2 ? (k & 1) : 0;
        const int use = nacc == 2 ? (k >> 1) : k;
        const uint32_t wcol = (uint32_t)((w & lg) * W) * 16;  // this slice's B rows
        tc::mbar_wait(&acc_empty[buf], (use & 1) ^ 1);
        tc::fence_after();
        wtrace(a, kEvMma, k);
        const uint32_t acc = tmem + buf * W;
        for (int kc = 0; kc < Q::NKC; ++kc, ++ait) {
          const int sa = ait % Q::SA;
          tc::mbar_wait(&a_full[sa], (ait / Q::SA) & 1);
          tc::fence_after();
          if (MODE != kIn && kc == Q::NKC - 1) wtrace(a, kEvPub, k);
          if (MODE != kIn) wtrace(a, kEvCData, ait);
          const uint32_t abase = tc::smem_u32(Aring + sa * Q::ACH);
#pragma unroll
          for (int tap = 0; tap < Q::TAPS; ++tap, ++wit) {
            const int sw = Q::RES ? 0 : wit % SWB;
            if (!Q::RES) {
              tc::mbar_wait(&w_full[sw], (wit / SWB) & 1);
              tc::fence_after();
            }
            const int shift = MODE == kMid ? (tap / 3) * b + (tap % 3) : 0;
            const uint32_t wbase = tc::smem_u32(Wring + (Q::RES ? (kc * Q::TAPS + tap) * Q::WCH : sw * Q::WCH));
            // one descriptor per operand and tap, immediate offsets per MMA (the issuer shares
            // its scheduler with the busy BN / epilogue warps)
            const uint64_t ad = MODE == kIn ? tc::desc_kmajor_swz(abase, 8 * Q::ROWB, Q::SWZ)
                                            : tc::desc_kmajor_noswz(abase + shift * 16, Q::PA, 128);
            const uint64_t wd = tc::desc_kmajor_noswz(wbase + wcol, Q::PW, 128);
            if (Q::SPL && lg) {
#pragma unroll
              for (int kk = 0; kk < Q::KC / 16; ++kk)
#pragma unroll
                for (int h = 0; h < Q::NSPLIT2; ++h)
                  tc::mma_bf16(acc + h * Q::NS2, tc::desc_add(ad, MODE == kIn ? kk * 32 : 2 * kk * Q::PA),
                               tc::desc_add(wd, 2 * kk * Q::PW + h * Q::NS2 * 16), idesc2, (kc | tap | kk) > 0);
            } else {
#pragma unroll
              for (int kk = 0; kk < Q::KC / 16; ++kk)
#pragma unroll
                for (int h = 0; h < Q::NSPLIT; ++h)
                  tc::mma_bf16(acc + h * Q::NS, tc::desc_add(ad, MODE == kIn ? kk * 32 : 2 * kk * Q::PA),
                               tc::desc_add(wd, 2 * kk * Q::PW + h * Q::NS * 16), idesc, (kc | tap | kk) > 0);
            }
            if (!Q::RES) tc::mma_commit(&w_empty[sw]);
          }
          tc::mma_commit(&a_empty[sa]);
          if (MODE != kIn) wtrace(a, kEvCPub, ait);  // MID/OUT: chunk's MMAs issued
        }
        tc::mma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  }
  if (Q::RES && tid == kLWarp * 32) tc::mbar_wait(&w_full[0], 0);  // no copy in flight at exit
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_free<Q::TALLOC>(tmem);
}

// ---- fused unit for 16x16 blocks: IN, MID and OUT in one launch, S1 / S2 never leave
// shared memory.
// A block's window is exactly two 128-row tiles (window rows 0-7 and 8-15), so one CTA
// runs the whole bottleneck of a block on its own: GEMM1 of both tiles -> A2 (the S1 rows
// of the block, plane layout) -> GEMM2 as 9 row-shifted views of A2 -> A3 (the S2 rows) ->
// GEMM3 -> + b3 + x -> the block's interior.  Persistent CTAs take blocks
// j = blockIdx.x + k * gridDim.x; the tensor pipe runs GEMM1(k+1), GEMM2(k), GEMM3(k-1)
// back to back while the epilogues of the other blocks drain TMEM.  The MMA order per
// accumulator equals IN's / MID's / OUT's (k-steps of GEMM1 and GEMM3; (K-chunk, tap,
// k-step) of GEMM2) and the roundings are the same, so the output is bit-identical to the
// three-launch path.
// In place (x == out) a block's window rim is its neighbours' interior, which other CTAs
// overwrite while this launch runs: the rims of all active blocks are snapshotted first
// (unit_rim_snapshot, a separate launch) and the BN warps take rim pixels from the
// snapshot.  Interior pixels are written only by their own block, after it read them.
//   warps 0-3   BN1 + ReLU on landed window tiles (rim pixels from the snapshot)
//   warps 4-7   epilogue 3: TMEM -> x + bf16(acc + b3) -> out (the block's interior)
//   warps 8-11  epilogue 1: TMEM -> relu(acc*s2 + t2') * in-bounds -> A2 (bf16, smem)
//   warps 12-15 epilogue 2: TMEM -> relu(acc*s3 + t3') -> A3 (smem)
//   warp 16     loader: window tiles by 4-D TMA (NKC1 boxes per tile); weights resident
//   warp 17     MMA issuer
constexpr int kFB = 16;                  // block size of the fused variant
constexpr int kFBnThreads = 128;         // BN warps 0-3
// CTA-0 event stamps per block k (diagnostics, tools/trace_fused.py)
enum { kFevLoad = 0, kFevLanded = 1, kFevBn = 2, kFevG1 = 3, kFevE1 = 4, kFevG2 = 5, kFevE2a = 6, kFevE2 = 7,
       kFevG1s = 8, kFevG3 = 9, kFevE1s = 10, kFevE3 = 11 };
constexpr int kFR2 = 296;                // A2 rows: 256 + 2*16 + 2 = 290, rounded to 8
constexpr int kFPA2 = kFR2 * 16;         // A2 plane stride
constexpr int kFPA3 = 256 * 16;          // A3 plane stride (rows q = oy*16 + ox of both tiles)
constexpr int kFBudget = 232448 - 1024;  // opt-in dynamic smem minus the static barriers

#ifndef SBN_FUSED_SA_MAX
#define SBN_FUSED_SA_MAX 4
#endif
template <int C, int M>
struct FCfg {
  using Q1 = WCfg<C, M, kIn>;
  using Q2 = WCfg<M, M, kMid>;
  using Q3 = WCfg<M, C, kOut>;
  static constexpr int KC1 = Q1::KC, NKC1 = C / KC1, ROWB = KC1 * 2;
  static constexpr uint32_t SWZ = Q1::SWZ;
  static constexpr int ACH = 128 * ROWB;          // one window chunk: 128 rows x KC1 ch (swizzled)
  static constexpr int WCH1 = Q1::WCH, PW1 = Q1::PW;
  static constexpr int W1B = (int)Q1::WBYTES;
  static constexpr int KC2 = Q2::KC, NKC2 = M / KC2, P2 = KC2 / 8;
  static constexpr int WCH2 = Q2::WCH, PW2 = Q2::PW;
  static constexpr int W2B = (int)Q2::WBYTES;
  static constexpr int PW3 = Q3::PW, W3B = (int)Q3::WBYTES;
  static constexpr int A2B = (M / 8) * kFPA2;
  static constexpr int A3B = (M / 8) * kFPA3;
  static constexpr int PAR1 = Q1::NPAR, PAR2 = Q2::NPAR, PAR3 = Q3::NPAR;
  static constexpr int PARB = (PAR1 + PAR2 + PAR3) * 4 / 128 * 128 + 128;
  // the window ring holds whole tiles: a slot = NKC1 chunks (one TMA box each) completing
  // on one barrier, BN'd by one group, consumed by one MMA wait and released by one commit
  // (the single MMA thread spends ~500 cycles of wait + commit latency per ring step)
  static constexpr int TSB = NKC1 * ACH;
  static constexpr long FIX = 2L * A2B + A3B + W1B + W2B + W3B + PARB;
  static constexpr int SAF = (int)((kFBudget - FIX) / TSB);
  static constexpr int SA = SAF > SBN_FUSED_SA_MAX ? SBN_FUSED_SA_MAX : SAF;  // window ring depth (tiles)
  // TMEM: NB1 GEMM1 tile accumulators (M columns each), two GEMM2 block accumulators (2M),
  // one GEMM3 block accumulator (2C)
  static constexpr int NB1R = (512 - 4 * M - 2 * C) / M;
  static constexpr int NB1 = NB1R >= 4 ? 4 : NB1R;
  // (the in-place rim snapshot, 60 pixels x C per block, reuses the S1 stack: b*b x M per block)
  static constexpr bool OK = M % 16 == 0 && C % 16 == 0 && C <= 256 && NB1 >= 1 && SA >= 2 && C % KC1 == 0 &&
                             60 * C <= 256 * M;
  static constexpr int COL2 = (NB1 > 0 ? NB1 : 1) * M;
  static constexpr int COL3 = COL2 + 4 * M;
  // GEMM3 accumulators: two when TMEM allows (epilogue 3 — the residual loads and the
  // block's stores — then overlaps the next block's GEMM3; it bounds the period otherwise)
  static constexpr int NB3 = COL3 + 4 * C <= 512 ? 2 : 1;
  static constexpr int TCOLS = COL3 + NB3 * 2 * C;
  static constexpr int TALLOC = TCOLS <= 32 ? 32 : TCOLS <= 64 ? 64 : TCOLS <= 128 ? 128 : TCOLS <= 256 ? 256 : 512;
  static constexpr bool BOTH_FIRST = NB1 >= 4;  // GEMM1 of both tiles of k+1 before GEMM2 of k
  static constexpr int OFF_A2 = (SA > 0 ? SA : 1) * TSB;
  static constexpr int OFF_A3 = OFF_A2 + 2 * A2B;
  static constexpr int OFF_W1 = OFF_A3 + A3B;
  static constexpr int OFF_W2 = OFF_W1 + W1B;
  static constexpr int OFF_W3 = OFF_W2 + W2B;
  static constexpr int OFF_PAR = OFF_W3 + W3B;
  static constexpr int SMEM = OFF_PAR + PARB;
};

// per-block stamps (CTA 0), diagnostics build only (see wtrace)
//   tools/build_variant.sh trace -DSBN_TRACE_WIDE; SBN_LIB_PATH=tools/bin/trace.so python tools/trace_fused.py
__device__ __forceinline__ void ftrace(const WArgs& a, int ev, int k) { wtrace(a, ev, k); }

// The issue order shared by the loader and the MMA issuer: GEMM1 tiles g1(k, t), GEMM2
// blocks g2(k), GEMM3 blocks g3(k), k over this CTA's nb blocks.
template <bool BOTH_FIRST, typename G1, typename G2, typename G3>
__device__ __forceinline__ void fused_schedule(int nb, G1&& g1, G2&& g2, G3&& g3) {
  if (nb <= 0) return;
  g1(0, 0);
  g1(0, 1);
  for (int k = 0; k < nb; ++k) {
    const bool more = k + 1 < nb;
    if (more) g1(k + 1, 0);
    if (BOTH_FIRST) {
      if (more) g1(k + 1, 1);
      g2(k);
    } else {
      g2(k);
      if (more) g1(k + 1, 1);
    }
    if (k > 0) g3(k - 1);
  }
  g3(nb - 1);
}

// 32 accumulator columns [g0, g0 + 32) of this thread's TMEM lane (16 when only 16 remain)
template <int N>
__device__ __forceinline__ void tmem_ld_group(uint32_t acc, int g0, float (&v)[32]) {
  if (g0 + 32 <= N) {
    tc::tmem_ld32(acc + g0, v);
  } else {
    float h[16];
    tc::tmem_ld16(acc + g0, h);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = h[i];
#pragma unroll
    for (int i = 16; i < 32; ++i) v[i] = 0.f;
  }
}

template <int C, int M>
__global__ void __launch_bounds__(kWideThreads, 1) unit_wide_fused_kernel(const __grid_constant__ WArgs a) {
  using F = FCfg<C, M>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t a_load[F::SA], a_full[F::SA], a_empty[F::SA], wres;
  __shared__ uint64_t a2_full[2], a2_empty[2], acc1_full[F::NB1], acc1_empty[F::NB1];
  __shared__ uint64_t acc2_full[2], acc2_empty[2], a3_full, a3_empty, acc3_full[F::NB3], acc3_empty[F::NB3];
  __shared__ uint32_t tslot;
  uint8_t* A1 = smem;
  uint8_t* A2 = smem + F::OFF_A2;
  uint8_t* A3 = smem + F::OFF_A3;
  uint8_t* W1 = smem + F::OFF_W1;
  uint8_t* W2 = smem + F::OFF_W2;
  uint8_t* W3 = smem + F::OFF_W3;
  float* par1 = reinterpret_cast<float*>(smem + F::OFF_PAR);
  float* par2 = par1 + F::PAR1;
  float* par3 = par2 + F::PAR2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Geo& g = a.g;
  constexpr int kLWarp = 16, kMWarp = 17;
  constexpr int OB = kFB - 2;

  if (tid == 0) {
    for (int s = 0; s < F::SA; ++s) {
      tc::mbar_init(&a_load[s], 1);
      tc::mbar_init(&a_full[s], kFBnThreads);
      tc::mbar_init(&a_empty[s], 1);
    }
    tc::mbar_init(&wres, 1);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&a2_full[s], 128);
      tc::mbar_init(&a2_empty[s], 1);
      tc::mbar_init(&acc2_full[s], 1);
      tc::mbar_init(&acc2_empty[s], 128);
    }
    for (int s = 0; s < F::NB1; ++s) {
      tc::mbar_init(&acc1_full[s], 1);
      tc::mbar_init(&acc1_empty[s], 128);
    }
    tc::mbar_init(&a3_full, 128);
    tc::mbar_init(&a3_empty, 1);
    for (int b = 0; b < F::NB3; ++b) {
      tc::mbar_init(&acc3_full[b], 1);
      tc::mbar_init(&acc3_empty[b], 128);
    }
    tc::mbar_fence_init();
  }
  if (tid == kLWarp * 32) asm volatile("prefetch.tensormap [%0];" ::"l"(&a.tmap) : "memory");
  for (int i = tid; i < F::PAR1; i += kWideThreads) par1[i] = a.par[i];
  for (int i = tid; i < F::PAR2; i += kWideThreads) par2[i] = a.par2[i];
  for (int i = tid; i < F::PAR3; i += kWideThreads) par3[i] = a.par3[i];
  if (warp == 0) tc::tmem_alloc<F::TALLOC>(&tslot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  tc::pdl_trigger();
  if (tid == kLWarp * 32) {
    // resident weights land under the previous kernel's tail (they do not depend on it)
    tc::mbar_expect_tx(&wres, (uint32_t)(F::W1B + F::W2B + F::W3B));
    for (int c = 0; c < F::Q1::CHUNKS; ++c)
      tc::bulk_g2s(W1 + (size_t)c * F::WCH1, a.wpk + (size_t)c * F::WCH1, F::WCH1, &wres);
    for (int c = 0; c < F::Q2::CHUNKS; ++c)
      tc::bulk_g2s(W2 + (size_t)c * F::WCH2, a.wpk2 + (size_t)c * F::WCH2, F::WCH2, &wres);
    for (int c = 0; c < F::Q3::CHUNKS; ++c)
      tc::bulk_g2s(W3 + (size_t)c * F::Q3::WCH, a.wpk3 + (size_t)c * F::Q3::WCH, F::Q3::WCH, &wres);
  }
  tc::pdl_wait();  // x, the rim snapshot and the index list of the previous launches are visible
  const int B = ld_count(a.count, a.cap);
  const int G = gridDim.x;
  const int nb = B > (int)blockIdx.x ? (B - 1 - (int)blockIdx.x) / G + 1 : 0;

  if (warp < 4) {
    // ------------------------------------------------ BN1 + ReLU on landed tiles (as IN)
    // all BN threads work on one tile at a time (the loader runs SA tiles ahead)
    const float* s1 = par1;
    constexpr int PR = F::ROWB / 16;
    constexpr int TG = kFBnThreads;
    constexpr int IT = 128 * PR / TG;  // pieces per thread per chunk
    constexpr int BATCH = IT < 8 ? IT : 8;
    static_assert(IT % BATCH == 0 && TG % PR == 0, "BN batches");
    // physical 16-B slot of logical channel group q in row r (the TMA swizzle)
    auto swz = [](int r) { return F::KC1 == 64 ? (r & 7) : ((r >> 1) & 3); };
    const int gt = tid;
    const Rim rim{kFB, kFB, 1};
    // In place, the window's rim pixels (its neighbours' interiors, which other CTAs overwrite
    // during this launch) are replaced by the snapshot with one 16-B cp.async per piece into
    // the landed tile.  Tile tl+1's copies are issued (once it has landed) before tile tl is
    // transformed, so their L2 round trip overlaps that work instead of preceding it.
    auto land = [&](int tl2) {
      tc::mbar_wait(&a_load[tl2 % F::SA], (tl2 / F::SA) & 1);
      if (!a.rim) return;
      const int k2 = tl2 >> 1, t2 = tl2 & 1, j2 = (int)blockIdx.x + k2 * G;
#pragma unroll 1
      for (int kc = 0; kc < F::NKC1; ++kc) {
        uint8_t* A = A1 + (tl2 % F::SA) * F::TSB + kc * F::ACH;
#pragma unroll 4
        for (int jj = 0; jj < IT; ++jj) {
          const int i = gt + jj * TG;
          const int r = i / PR, grp = i % PR;
          const int wy = 8 * t2 + (r >> 4), wx = r & 15;
          if (wy == 0 || wy == kFB - 1 || wx == 0 || wx == kFB - 1)
            tc::cp_async16(A + r * F::ROWB + (grp ^ swz(r)) * 16,
                           a.rim + ((size_t)j2 * rim.pixels() + rim.index(wy, wx)) * C + kc * F::KC1 + grp * 8, true);
        }
      }
      tc::cp_async_commit();
    };
    int tl = 0;
    if (nb > 0) land(0);
    for (int k = 0; k < nb; ++k) {
      for (int t = 0; t < 2; ++t, ++tl) {
        const int s = tl % F::SA;
        if (tl + 1 < 2 * nb) {
          land(tl + 1);
          tc::cp_async_wait<1>();  // this tile's rim copies (the group before the one just issued)
        } else {
          tc::cp_async_wait<0>();
        }
        if (gt == 0 && t == 0) ftrace(a, kFevLanded, k);
#pragma unroll 1
        for (int kc = 0; kc < F::NKC1; ++kc) {
          uint8_t* A = A1 + s * F::TSB + kc * F::ACH;
          // this thread's logical channel group is fixed (TG % PR == 0): its BN vectors
          // are loaded once per chunk
          const int grp = gt % PR;
          const uint4 sg4 = *reinterpret_cast<const uint4*>(s1 + (kc * F::KC1 + grp * 8) / 2);
          const uint4 vv4 = *reinterpret_cast<const uint4*>(s1 + C / 2 + (kc * F::KC1 + grp * 8) / 2);
#pragma unroll 1
          for (int b0 = 0; b0 < IT; b0 += BATCH) {
            uint4 raw[BATCH];
#pragma unroll
            for (int jj = 0; jj < BATCH; ++jj) {
              const int r = (gt + (b0 + jj) * TG) / PR;
              asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(raw[jj].x), "=r"(raw[jj].y), "=r"(raw[jj].z), "=r"(raw[jj].w)
                           : "r"(tc::smem_u32(A + r * F::ROWB + (grp ^ swz(r)) * 16)));
            }
#pragma unroll
            for (int jj = 0; jj < BATCH; ++jj) {
              const int r = (gt + (b0 + jj) * TG) / PR;
              const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[jj]);
              const __nv_bfloat162* hs = reinterpret_cast<const __nv_bfloat162*>(&sg4);
              const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&vv4);
              const __nv_bfloat162 z2 = __float2bfloat162_rn(0.f);
              uint32_t o[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const __nv_bfloat162 y = __hmax2(__hfma2(h[e], hs[e], hv[e]), z2);
                o[e] = *reinterpret_cast<const uint32_t*>(&y);
              }
              asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(tc::smem_u32(A + r * F::ROWB + (grp ^ swz(r)) * 16)),
                           "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3])
                           : "memory");
            }
          }
        }
        tc::fence_async_smem();
        tc::mbar_arrive(&a_full[s]);
        if (gt == 0 && t == 1) ftrace(a, kFevBn, k);
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------ epilogue 3: TMEM -> x + bf16(acc + b3) -> out
    // OUT's epilogue at the block's clipped interior; the residual is read from out (= x in
    // place, the clone of x otherwise).  Each thread issues its row's C / 8 residual loads
    // before it drains the accumulator, so they are all in flight at once.
    const int qd = warp & 3, r = qd * 32 + lane;
    const uint32_t lanes = (uint32_t)(qd * 32) << 16;
    const float* b3 = par3;
    for (int k = 0; k < nb; ++k) {
      const int j = (int)blockIdx.x + k * G;
      const int n = __ldg(a.idx + 3 * j), by = __ldg(a.idx + 3 * j + 1), bx = __ldg(a.idx + 3 * j + 2);
      const int b3i = k % F::NB3;
      tc::mbar_wait(&acc3_full[b3i], (k / F::NB3) & 1);
      tc::fence_after();
#pragma unroll 1
      for (int u = 0; u < 2; ++u) {
        const int q = u * 128 + r, oy = q >> 4, ox = q & 15;
        const int Y = by * g.obh + oy, X = bx * g.obw + ox;
        const bool store = oy < OB && ox < OB && Y < g.oh && X < g.ow;
        uint4* dp = reinterpret_cast<uint4*>(a.dst + (((long)n * g.oh + (store ? Y : 0)) * g.ow + (store ? X : 0)) * C);
        uint4 xr[C / 8];
#pragma unroll
        for (int e = 0; e < C / 8; ++e) xr[e] = tc::ld_v4_pred(dp + e, store);
        const uint32_t acc = tmem + lanes + F::COL3 + b3i * 2 * C + u * C;
#pragma unroll
        for (int c0 = 0; c0 < C; c0 += 16) {
          float v[16];
          tc::tmem_ld16(acc + c0, v);
          uint32_t o[8];
#pragma unroll
          for (int q2 = 0; q2 < 8; ++q2) {
            const float2 bb = *reinterpret_cast<const float2*>(b3 + c0 + 2 * q2);
            const __nv_bfloat162 st = __floats2bfloat162_rn(v[2 * q2] + bb.x, v[2 * q2 + 1] + bb.y);
            const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xr[c0 / 8 + q2 / 4]);
            const float2 uf = __bfloat1622float2(st), xf = __bfloat1622float2(xh[q2 % 4]);
            o[q2] = tc::pack_bf16(xf.x + uf.x, xf.y + uf.y);
          }
          if (store) {
            dp[c0 / 8] = make_uint4(o[0], o[1], o[2], o[3]);
            dp[c0 / 8 + 1] = make_uint4(o[4], o[5], o[6], o[7]);
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&acc3_empty[b3i]);
      if (r == 0) ftrace(a, kFevE3, k);
    }
  } else if (warp < 12) {
    // ------------------------------------------------ epilogue 1: TMEM -> A2 (S1 rows)
    const int qd = warp & 3, r = qd * 32 + lane;
    const float* sc = par1 + 2 * C + M;  // s2
    const float* sh = sc + M;            // t2' (b1 folded)
    for (int k = 0; k < nb; ++k) {
      const int j = (int)blockIdx.x + k * G;
      const int by = __ldg(a.idx + 3 * j + 1), bx = __ldg(a.idx + 3 * j + 2);
      const int ab = k & 1;
      tc::mbar_wait(&a2_empty[ab], ((k >> 1) & 1) ^ 1);
      uint8_t* A2b = A2 + ab * F::A2B;
      for (int t = 0; t < 2; ++t) {
        const int ti = 2 * k + t, b1 = ti % F::NB1;
        const int p = t * 128 + r, wy = p >> 4, wx = p & 15;
        const int y = g.oy + by * g.sy + wy, x = g.ox + bx * g.sx + wx;
        const bool valid = y >= 0 && y < g.h && x >= 0 && x < g.w;
        tc::mbar_wait(&acc1_full[b1], (ti / F::NB1) & 1);
        tc::fence_after();
        if (t == 0 && r == 0) ftrace(a, kFevE1s, k);
        const uint32_t acc = tmem + ((uint32_t)(qd * 32) << 16) + b1 * M;
#pragma unroll
        for (int g0 = 0; g0 < M; g0 += 32) {
          float v[32];
          tmem_ld_group<M>(acc, g0, v);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int c0 = g0 + 16 * hh;
            if (c0 >= M) break;
            const float* w = v + 16 * hh;
            uint32_t o[8];
#pragma unroll
            for (int q = 0; q < 8; q += 2) {
              const float4 s4 = *reinterpret_cast<const float4*>(sc + c0 + 2 * q);
              const float4 t4 = *reinterpret_cast<const float4*>(sh + c0 + 2 * q);
              const float u0 = fmaxf(fmaf(w[2 * q], s4.x, t4.x), 0.f);
              const float u1 = fmaxf(fmaf(w[2 * q + 1], s4.y, t4.y), 0.f);
              const float u2 = fmaxf(fmaf(w[2 * q + 2], s4.z, t4.z), 0.f);
              const float u3 = fmaxf(fmaf(w[2 * q + 3], s4.w, t4.w), 0.f);
              o[q] = valid ? tc::pack_bf16(u0, u1) : 0u;
              o[q + 1] = valid ? tc::pack_bf16(u2, u3) : 0u;
            }
            uint8_t* pl = A2b + (c0 / 8) * kFPA2 + p * 16;
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(tc::smem_u32(pl)), "r"(o[0]), "r"(o[1]),
                         "r"(o[2]), "r"(o[3])
                         : "memory");
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(tc::smem_u32(pl + kFPA2)), "r"(o[4]),
                         "r"(o[5]), "r"(o[6]), "r"(o[7])
                         : "memory");
          }
        }
        tc::fence_before();
        tc::mbar_arrive(&acc1_empty[b1]);
      }
      tc::fence_async_smem();
      tc::mbar_arrive(&a2_full[ab]);
      if (r == 0) ftrace(a, kFevE1, k);
    }
  } else if (warp < 16) {
    // ------------------------------------------------ epilogue 2: TMEM -> A3 (S2 rows)
    const int qd = warp & 3, r = qd * 32 + lane;
    const uint32_t lanes = (uint32_t)(qd * 32) << 16;
    auto epi2 = [&](int k) {
      const float* sc = par2 + M;  // s3
      const float* sh = sc + M;    // t3' (b2 folded)
      const int b2 = k & 1;
      tc::mbar_wait(&acc2_full[b2], (k >> 1) & 1);
      tc::mbar_wait(&a3_empty, (k & 1) ^ 1);  // GEMM3 of the previous block has read A3
      tc::fence_after();
      if (r == 0) ftrace(a, kFevE2a, k);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int q = u * 128 + r;
        const uint32_t acc = tmem + lanes + F::COL2 + b2 * 2 * M + u * M;
#pragma unroll
        for (int g0 = 0; g0 < M; g0 += 32) {
          float v[32];
          tmem_ld_group<M>(acc, g0, v);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int c0 = g0 + 16 * hh;
            if (c0 >= M) break;
            const float* w = v + 16 * hh;
            uint32_t o[8];
#pragma unroll
            for (int q2 = 0; q2 < 8; q2 += 2) {
              const float4 s4 = *reinterpret_cast<const float4*>(sc + c0 + 2 * q2);
              const float4 t4 = *reinterpret_cast<const float4*>(sh + c0 + 2 * q2);
              o[q2] = tc::pack_bf16(fmaxf(fmaf(w[2 * q2], s4.x, t4.x), 0.f), fmaxf(fmaf(w[2 * q2 + 1], s4.y, t4.y), 0.f));
              o[q2 + 1] =
                  tc::pack_bf16(fmaxf(fmaf(w[2 * q2 + 2], s4.z, t4.z), 0.f), fmaxf(fmaf(w[2 * q2 + 3], s4.w, t4.w), 0.f));
            }
            uint8_t* pl = A3 + (c0 / 8) * kFPA3 + q * 16;
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(tc::smem_u32(pl)), "r"(o[0]), "r"(o[1]),
                         "r"(o[2]), "r"(o[3])
                         : "memory");
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(tc::smem_u32(pl + kFPA3)), "r"(o[4]),
                         "r"(o[5]), "r"(o[6]), "r"(o[7])
                         : "memory");
          }
        }
      }
      tc::fence_async_smem();
      tc::mbar_arrive(&a3_full);
      tc::fence_before();
      tc::mbar_arrive(&acc2_empty[b2]);
      if (r == 0) ftrace(a, kFevE2, k);
    };
    for (int k = 0; k < nb; ++k) epi2(k);
  } else if (warp == kLWarp) {
    // ------------------------------------------------ loader
    if (lane == 0) {
      int tl = 0;
      int cur_k = -1, cn = 0, cy = 0, cx = 0;
      auto g1 = [&](int k, int t) {
        if (k != cur_k) {
          const int j = (int)blockIdx.x + k * G;
          cn = __ldg(a.idx + 3 * j);
          cy = g.oy + __ldg(a.idx + 3 * j + 1) * g.sy;
          cx = g.ox + __ldg(a.idx + 3 * j + 2) * g.sx;
          cur_k = k;
        }
        const int s = tl % F::SA;
        tc::mbar_wait(&a_empty[s], ((tl / F::SA) & 1) ^ 1);
        if (t == 0) ftrace(a, kFevLoad, k);
        tc::mbar_expect_tx(&a_load[s], (uint32_t)F::TSB);
        for (int kc = 0; kc < F::NKC1; ++kc)
          tma_4d(A1 + s * F::TSB + kc * F::ACH, &a.tmap, kc * F::KC1, cx, cy + 8 * t, cn, &a_load[s]);
        ++tl;
      };
      fused_schedule<F::BOTH_FIRST>(nb, g1, [](int) {}, [](int) {});
    }
    __syncwarp();
  } else if (warp == kMWarp) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      int tl = 0;
      tc::mbar_wait(&wres, 0);
      auto g1 = [&](int k, int t) {
        constexpr uint32_t idesc = tc::idesc_bf16_f32(128, M);
        const int ti = 2 * k + t, b1 = ti % F::NB1;
        tc::mbar_wait(&acc1_empty[b1], ((ti / F::NB1) & 1) ^ 1);
        tc::fence_after();
        if (t == 0) ftrace(a, kFevG1s, k);
        const uint32_t acc = tmem + b1 * M;
        const int s = tl % F::SA;
        tc::mbar_wait(&a_full[s], (tl / F::SA) & 1);
        tc::fence_after();
#pragma unroll
        for (int kc = 0; kc < F::NKC1; ++kc) {
          const uint32_t abase = tc::smem_u32(A1 + s * F::TSB + kc * F::ACH);
          const uint32_t wbase = tc::smem_u32(W1 + kc * F::WCH1);
#pragma unroll
          for (int kk = 0; kk < F::KC1 / 16; ++kk)
            tc::mma_bf16(acc, tc::desc_kmajor_swz(abase + kk * 32, 8 * F::ROWB, F::SWZ),
                         tc::desc_kmajor_noswz(wbase + 2 * kk * F::PW1, F::PW1, 128), idesc, (kc | kk) > 0);
        }
        tc::mma_commit(&a_empty[s]);
        ++tl;
        tc::mma_commit(&acc1_full[b1]);
        if (t == 1) ftrace(a, kFevG1, k);
      };
      auto g2 = [&](int k) {
        constexpr uint32_t idesc = tc::idesc_bf16_f32(128, M);
        const int b2 = k & 1;
        tc::mbar_wait(&acc2_empty[b2], ((k >> 1) & 1) ^ 1);
        tc::mbar_wait(&a2_full[b2], (k >> 1) & 1);
        tc::fence_after();
        ftrace(a, kFevG2, k);
        const uint32_t acc = tmem + F::COL2 + b2 * 2 * M;
        // one base descriptor per operand, offset per (K-chunk, tap) and per MMA (the issuer
        // shares its scheduler with busy warps: instructions per MMA matter)
        const uint64_t a2d = tc::desc_kmajor_noswz(tc::smem_u32(A2 + b2 * F::A2B), kFPA2, 128);
        const uint64_t w2d = tc::desc_kmajor_noswz(tc::smem_u32(W2), F::PW2, 128);
#pragma unroll 1
        for (int kc = 0; kc < F::NKC2; ++kc)
#pragma unroll 1
          for (int tap = 0; tap < 9; ++tap) {  // (rolled: the unrolled tap loop made the issuer spill)
            const int shift = (tap / 3) * kFB + (tap % 3);
            const uint64_t at = tc::desc_add(a2d, kc * F::P2 * kFPA2 + shift * 16);
            const uint64_t wt = tc::desc_add(w2d, (kc * 9 + tap) * F::WCH2);
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
              for (int kk = 0; kk < F::KC2 / 16; ++kk)
                tc::mma_bf16(acc + u * M, tc::desc_add(at, 2 * kk * kFPA2 + u * 128 * 16),
                             tc::desc_add(wt, 2 * kk * F::PW2), idesc, (kc | tap | kk) > 0);
          }
        tc::mma_commit(&a2_empty[b2]);
        tc::mma_commit(&acc2_full[b2]);
      };
      auto g3 = [&](int k) {
        constexpr uint32_t idesc = tc::idesc_bf16_f32(128, C);
        const int b3i = k % F::NB3;
        tc::mbar_wait(&acc3_empty[b3i], ((k / F::NB3) & 1) ^ 1);
        tc::mbar_wait(&a3_full, k & 1);
        tc::fence_after();
        ftrace(a, kFevG3, k);
        const uint32_t a3base = tc::smem_u32(A3), wbase = tc::smem_u32(W3);
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int kk = 0; kk < M / 16; ++kk)
            tc::mma_bf16(tmem + F::COL3 + b3i * 2 * C + u * C,
                         tc::desc_kmajor_noswz(a3base + 2 * kk * kFPA3 + u * 128 * 16, kFPA3, 128),
                         tc::desc_kmajor_noswz(wbase + 2 * kk * F::PW3, F::PW3, 128), idesc, kk > 0);
        tc::mma_commit(&a3_empty);
        tc::mma_commit(&acc3_full[b3i]);
      };
      fused_schedule<F::BOTH_FIRST>(nb, g1, g2, g3);
    }
    __syncwarp();
  }
  if (tid == kLWarp * 32) tc::mbar_wait(&wres, 0);  // no copy in flight at exit
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_free<F::TALLOC>(tmem);
}

// ---- packed image: [W1 chunks | W2 chunks | W3 chunks | params], regions 128-B aligned.
// A chunk c of a GEMM with K-chunk KC, N columns: KC/8 planes of N rows x 16 B,
// element (n, k) at (k/8)*N*16 + n*16 + (k%8)*2 — the kernel's B-operand layout.  MID
// chunks are ordered (kc, tap).
//   params (floats): IN  sgn|v (bf16x2) t1 [c] b1 s2 t2' [m]   MID b2 s3 t3' [m]   OUT b3 [c]
//   (t2' = b1*s2 + t2, t3' = b2*s3 + t3: the conv bias folded into the next BN)
struct WLayout {
  size_t w1, w2, w3, p1, p2, p3, total;
};

template <int C, int M>
constexpr WLayout wide_layout() {
  using Q1 = WCfg<C, M, kIn>;
  using Q2 = WCfg<M, M, kMid>;
  using Q3 = WCfg<M, C, kOut>;
  WLayout L{};
  auto al = [](size_t v) { return (v + 127) / 128 * 128; };
  L.w1 = 0;
  L.w2 = al(L.w1 + Q1::WBYTES);
  L.w3 = al(L.w2 + Q2::WBYTES);
  L.p1 = al(L.w3 + Q3::WBYTES);
  L.p2 = al(L.p1 + (size_t)Q1::NPAR * 4);
  L.p3 = al(L.p2 + (size_t)Q2::NPAR * 4);
  L.total = al(L.p3 + (size_t)Q3::NPAR * 4);
  return L;
}

template <int C, int M>
__global__ void unit_wide_pack_kernel(sbn_unit_params p, uint8_t* __restrict__ img) {
  using Q1 = WCfg<C, M, kIn>;
  using Q2 = WCfg<M, M, kMid>;
  using Q3 = WCfg<M, C, kOut>;
  constexpr WLayout L = wide_layout<C, M>();
  const __nv_bfloat16* w1 = (const __nv_bfloat16*)p.w1;
  const __nv_bfloat16* w2 = (const __nv_bfloat16*)p.w2;
  const __nv_bfloat16* w3 = (const __nv_bfloat16*)p.w3;
  const int stride = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  // BN1 + ReLU is applied in packed bf16 as relu(sgn*x + v) with the per-channel scale
  // |s1| folded into W1's rows: relu(x*s1 + t1) = |s1| * relu(sgn(s1)*x + t1/|s1|).
  const float* s1v = (const float*)p.bn1_scale;
  const float* t1v = (const float*)p.bn1_shift;
  // W1 (1, 1, C, M): B[n = co][k = ci] = W1[ci, co] * |s1[ci]|
  for (int i = t0; i < C * M; i += stride) {
    const int ci = i / M, co = i % M;
    const int kc = ci / Q1::KC, k = ci % Q1::KC;
    *reinterpret_cast<__nv_bfloat16*>(img + L.w1 + (size_t)kc * Q1::WCH + (k / 8) * Q1::PW + co * 16 + (k % 8) * 2) =
        __float2bfloat16_rn(__bfloat162float(w1[i]) * fabsf(s1v[ci]));
  }
  // W2 (3, 3, M, M): chunk (kc, tap)
  for (int i = t0; i < 9 * M * M; i += stride) {
    const int tap = i / (M * M), r = i % (M * M), ci = r / M, co = r % M;
    const int kc = ci / Q2::KC, k = ci % Q2::KC;
    *reinterpret_cast<__nv_bfloat16*>(img + L.w2 + (size_t)(kc * 9 + tap) * Q2::WCH + (k / 8) * Q2::PW + co * 16 + (k % 8) * 2) = w2[i];
  }
  // W3 (1, 1, M, C)
  for (int i = t0; i < M * C; i += stride) {
    const int ci = i / C, co = i % C;
    const int kc = ci / Q3::KC, k = ci % Q3::KC;
    *reinterpret_cast<__nv_bfloat16*>(img + L.w3 + (size_t)kc * Q3::WCH + (k / 8) * Q3::PW + co * 16 + (k % 8) * 2) = w3[i];
  }
  float* p1 = reinterpret_cast<float*>(img + L.p1);
  float* p2 = reinterpret_cast<float*>(img + L.p2);
  float* p3 = reinterpret_cast<float*>(img + L.p3);
  auto bf = [](const void* q, int i) { return __bfloat162float(((const __nv_bfloat16*)q)[i]); };
  // IN params: words [0, C/2) sign pairs, [C/2, C) v = t1/|s1| pairs (bf16x2); [C, 2C) t1
  __nv_bfloat16* sg = reinterpret_cast<__nv_bfloat16*>(p1);
  __nv_bfloat16* vv = reinterpret_cast<__nv_bfloat16*>(p1 + C / 2);
  for (int i = t0; i < C; i += stride) {
    const float a = fabsf(s1v[i]);
    sg[i] = __float2bfloat16_rn(s1v[i] < 0.f ? -1.f : 1.f);
    vv[i] = __float2bfloat16_rn(a > 0.f ? t1v[i] / a : 0.f);
    p1[C + i] = t1v[i];
    p3[i] = bf(p.b3, i);
  }
  for (int i = t0; i < M; i += stride) {  // conv bias folded into the following BN shift
    const float s2 = ((const float*)p.bn2_scale)[i], s3 = ((const float*)p.bn3_scale)[i];
    // channels with s1 == 0 contribute the constant relu(t1) * W1 (their W1 rows are zero)
    float extra = 0.f;
    for (int c = 0; c < C; ++c)
      if (s1v[c] == 0.f) extra += fmaxf(t1v[c], 0.f) * __bfloat162float(w1[c * M + i]);
    p1[2 * C + i] = bf(p.b1, i);
    p1[2 * C + M + i] = s2;
    p1[2 * C + 2 * M + i] = fmaf(bf(p.b1, i) + extra, s2, ((const float*)p.bn2_shift)[i]);
    p2[i] = bf(p.b2, i);
    p2[M + i] = s3;
    p2[2 * M + i] = fmaf(bf(p.b2, i), s3, ((const float*)p.bn3_shift)[i]);
  }
}

template <int K, int N, int MODE>
int launch_wide(const WArgs& a, long max_tiles, cudaStream_t s, const char* what) {
  using Q = WCfg<K, N, MODE>;
  auto kern = unit_wide_kernel<K, N, MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Q::SMEM);
  cudaLaunchConfig_t cfg = {};
  if (Q::SPL) max_tiles *= 2;  // room for column slices
  cfg.gridDim = dim3((unsigned)(max_tiles < sm_count() ? (max_tiles < 1 ? 1 : max_tiles) : sm_count()));
  cfg.blockDim = dim3(kWideThreads);
  cfg.dynamicSmemBytes = Q::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a);
  return launch_status(what);
}

// the fused one-launch unit applies to 16x16 blocks when its buffers fit
template <int C, int M>
bool fused_ok(int b) {
  if constexpr (FCfg<C, M>::OK) {
    return b == kFB && FCfg<C, M>::SMEM <= max_smem_optin() && !(debug_flags() & kDebugWideUnfused);
  } else {
    (void)b;
    return false;
  }
}

template <int C, int M>
int launch_fused(const WArgs& a, long cap, cudaStream_t s) {
  if constexpr (FCfg<C, M>::OK) {
    using F = FCfg<C, M>;
    auto kern = unit_wide_fused_kernel<C, M>;
    static PerDeviceOnce once;
    once([&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, F::SMEM); });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(cap < sm_count() ? (cap < 1 ? 1 : cap) : sm_count()));
    cfg.blockDim = dim3(kWideThreads);
    cfg.dynamicSmemBytes = F::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a);
    return launch_status("residual_unit_wide_fused");
  } else {
    (void)a;
    (void)cap;
    (void)s;
    return SBN_ERR_UNSUPPORTED;
  }
}

template <int C, int M>
int run_wide(const void* x, void* out, const Geo& g, const uint8_t* img, const int32_t* idx,
             const int32_t* count, int cap, uint8_t* s1, uint8_t* s2, cudaStream_t s) {
  constexpr WLayout L = wide_layout<C, M>();
  const int b = g.bh;
  WArgs a;
  memset(&a, 0, sizeof(a));
  a.g = g;
  a.idx = idx;
  a.count = count;
  a.cap = cap;
  // IN slabs: hb window rows of one block per slab, G slabs per 128-row tile
  a.hb = b * b <= 128 ? b : 128 / b;
  a.S = (b + a.hb - 1) / a.hb;
  a.slab_rows = (a.hb * b + 7) / 8 * 8;
  a.G = 128 / a.slab_rows < 4 ? 128 / a.slab_rows : 4;
  a.box_rows = (128 + 2 * b + 2 + 7) / 8 * 8;
  a.split = !(debug_flags() & kDebugWideNoSplit);
  // diagnostics: stamps of ONE of the three launches, selected by debug flag bits 3-4
  const int tsel = (debug_flags() >> 3) & 3;
  unsigned long long* tb = trace_buffer();
  a.trace = tsel == 0 ? tb : nullptr;
  const long rows1 = (long)cap * b * b + kStackPad, rows2 = (long)cap * (b - 2) * (b - 2) + kStackPad;
  // IN: x windows -> S1 (4-D map, box = KC channels x b x hb rows, swizzled rows)
  {
    using Q = WCfg<C, M, kIn>;
    const uint64_t dims[4] = {(uint64_t)C, (uint64_t)g.w, (uint64_t)g.h, (uint64_t)g.n};
    const uint64_t str[3] = {(uint64_t)C * 2, (uint64_t)g.w * C * 2, (uint64_t)g.h * g.w * C * 2};
    const uint32_t box[4] = {(uint32_t)Q::KC, (uint32_t)b, (uint32_t)a.hb, 1};
    int st = encode_map(&a.tmap, x, 4, dims, str, box,
                        Q::KC == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
    if (st) return st;
  }
  int st = 0;
  if (fused_ok<C, M>(b)) {
    // the whole unit in one launch; in place, the rims of the active windows are
    // snapshotted first (into the S1 stack, which this path does not use)
    if (x == out) {
      st = unit_rim_snapshot(x, 2, C, g, 1, idx, count, cap, s1, s);
      if (st) return st;
      a.rim = (const __nv_bfloat16*)s1;
    }
    a.dst = (__nv_bfloat16*)out;
    a.wpk = img + L.w1;
    a.par = (const float*)(img + L.p1);
    a.wpk2 = img + L.w2;
    a.par2 = (const float*)(img + L.p2);
    a.wpk3 = img + L.w3;
    a.par3 = (const float*)(img + L.p3);
    return launch_fused<C, M>(a, cap, s);
  }
  a.dst = (__nv_bfloat16*)s1;
  a.dst_rows = rows1;
  a.wpk = img + L.w1;
  a.par = (const float*)(img + L.p1);
  st = launch_wide<C, M, kIn>(a, ((long)cap * a.S + a.G - 1) / a.G, s, "residual_unit_wide_in");
  if (st) return st;
  // MID: S1 -> S2 (3x3 valid); plane runs by 1-D bulk copies
  a.stack = s1;
  a.src_rows = rows1;
  a.dst = (__nv_bfloat16*)s2;
  a.dst_rows = rows2;
  a.wpk = img + L.w2;
  a.par = (const float*)(img + L.p2);
  a.trace = tsel == 1 ? tb : nullptr;
  st = launch_wide<M, M, kMid>(a, ((long)cap * b * b + 127) / 128, s, "residual_unit_wide_mid");
  if (st) return st;
  // OUT: S2 -> out (+ residual), in place or into the clone
  a.stack = s2;
  a.src_rows = rows2;
  a.dst = (__nv_bfloat16*)out;
  a.wpk = img + L.w3;
  a.par = (const float*)(img + L.p3);
  a.trace = tsel == 2 ? tb : nullptr;
  return launch_wide<M, C, kOut>(a, ((long)cap * (b - 2) * (b - 2) + 127) / 128, s, "residual_unit_wide_out");
}

// (c, m) instantiations: BASELINE config-4 stages (m = c/2) and the small unit shapes
#define SBN_UNIT_WIDE_CONFIGS(X) \
  X(32, 16)                      \
  X(64, 32)                      \
  X(96, 48)                      \
  X(128, 64)                     \
  X(192, 96)                     \
  X(256, 128)                    \
  X(384, 192)

template <int C, int M>
bool fits() {
  const int mx = max_smem_optin();
  return WCfg<C, M, kIn>::SMEM <= mx && WCfg<M, M, kMid>::SMEM <= mx && WCfg<M, C, kOut>::SMEM <= mx;
}

}  // namespace

bool unit_wide_supported(int dtype, int c, int m, const Geo& g, int halo, int pre_act) {
  if (dtype != SBN_BF16 || halo != 1 || !pre_act || g.bh != g.bw || g.bh < 3 ||
      128 + 2 * g.bh + 2 > kMaxRows)
    return false;
#define X(C_, M_) if (c == C_ && m == M_) return fits<C_, M_>();
  SBN_UNIT_WIDE_CONFIGS(X)
#undef X
  return false;
}

bool unit_wide_one_launch(int c, int m, const Geo& g) {
  if (g.bh != g.bw) return false;
#define X(C_, M_) if (c == C_ && m == M_) return fused_ok<C_, M_>(g.bh);
  SBN_UNIT_WIDE_CONFIGS(X)
#undef X
  return false;
}

size_t unit_wide_packed_bytes(int c, int m) {
#define X(C_, M_) if (c == C_ && m == M_) return wide_layout<C_, M_>().total;
  SBN_UNIT_WIDE_CONFIGS(X)
#undef X
  return 0;
}

static size_t stack1_bytes(int m, const Geo& g) {
  const size_t cap = (size_t)g.n * g.gy * g.gx, b = g.bh;
  return ((cap * b * b + kStackPad) * m * 2 + 255) / 256 * 256;
}
static size_t stack2_bytes(int m, const Geo& g) {
  const size_t cap = (size_t)g.n * g.gy * g.gx, b = g.bh;
  return ((cap * (b - 2) * (b - 2) + kStackPad) * m * 2 + 255) / 256 * 256;
}

size_t unit_wide_stack_bytes(int m, const Geo& g) { return stack1_bytes(m, g) + stack2_bytes(m, g); }

int unit_wide_pack(const sbn_unit_params* p, int c, int m, void* img, cudaStream_t s) {
#define X(C_, M_)                                                                        \
  if (c == C_ && m == M_) {                                                              \
    cudaMemsetAsync(img, 0, wide_layout<C_, M_>().total, s);                             \
    unit_wide_pack_kernel<C_, M_><<<64, 256, 0, s>>>(*p, (uint8_t*)img);                 \
    return launch_status("residual_unit_wide_pack");                                     \
  }
  SBN_UNIT_WIDE_CONFIGS(X)
#undef X
  set_error("no wide tcgen05 unit instantiation for c=%d m=%d", c, m);
  return SBN_ERR_UNSUPPORTED;
}

int unit_wide_launch(const void* x, void* out, int c, int m, const Geo& g, const void* packed,
                     const int32_t* idx, const int32_t* count, int cap, void* stacks, cudaStream_t s) {
  uint8_t* s1 = (uint8_t*)stacks;
  uint8_t* s2 = s1 + stack1_bytes(m, g);
#define X(C_, M_) \
  if (c == C_ && m == M_) return run_wide<C_, M_>(x, out, g, (const uint8_t*)packed, idx, count, cap, s1, s2, s);
  SBN_UNIT_WIDE_CONFIGS(X)
#undef X
  set_error("no wide tcgen05 unit instantiation for c=%d m=%d", c, m);
  return SBN_ERR_UNSUPPORTED;
}

}  // namespace sbn
