// tcgen05 / TMEM fused sparse residual unit (bf16 activations, fp32 accumulate).
//
// One persistent CTA (256 threads) walks the active blocks (device-side count).  Per
// block the bottleneck of reference `_unit_branch` (`layers.py:155-169`, pre-activation)
// runs as three tensor-core GEMMs whose operands never leave shared memory / TMEM:
//
//   stage   : window (BS x BS pixels x C) gathered from x (rim from the snapshot when
//             in place), BN1 + ReLU applied in registers -> A1 [pixels x C] bf16
//   GEMM1   : C1[pixels x MC]  = A1 . W1            (UMMA M=128 tiles, N=MC, K=C)
//   epi 1   : +b1, BN2, ReLU, x in-bounds  -> A2 [pixels x MC] bf16
//   GEMM2   : C2[q x MC] = sum_taps A2[q + ky*BS + kx] . W2[ky,kx]
//             (3x3 valid conv as 9 row-shifted views of A2 — "full-width" implicit GEMM:
//              output row q = oy*BS + ox, columns ox >= BS-2 are computed and dropped)
//   epi 2   : +b2, BN3, ReLU -> A3 [q x MC] bf16 (aliases A1)
//   GEMM3   : C3[q x C] = A3 . W3
//   epi 3   : +b3, + x (residual, this block's own interior) -> out, clipped
//
// Operands use the K-major SWIZZLE_NONE plane layout of tc_util.cuh; plane strides are
// padded by 16 B so the 16-byte staging stores of 8 consecutive threads hit 8 distinct
// bank groups.  Accumulators live in TMEM (tcgen05.ld in the epilogues); MMAs are
// issued by one thread and completion is signalled through an mbarrier
// (tcgen05.commit).  Two CTAs per SM overlap one block's global traffic with the other's
// tensor-core work.
#include "unit.cuh"
#include "tc_util.cuh"

#include <cooperative_groups.h>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace sbn {
namespace {

constexpr int kThreads = 256;
int g_last_occ[8] = {0};  // diagnostics: occ single, clusters pair, regs, static smem, max dyn, dyn

template <int C, int MC, int BS>
struct Cfg {
  static_assert(C % 16 == 0 && MC % 16 == 0 && C <= 256 && MC <= 256, "channel constraints");
  static constexpr int NPIX = BS * BS;
  static constexpr int NT1 = (NPIX + 127) / 128;
  static constexpr int NQ = (BS - 2) * BS;
  static constexpr int NT2 = (NQ + 127) / 128;
  static constexpr int R1 = NT1 * 128;
  static constexpr int R2a = NT2 * 128 + 2 * BS + 2;
  static constexpr int R2 = (((R2a > R1 ? R2a : R1) + 7) / 8) * 8;
  static constexpr int R3 = NT2 * 128;
  static constexpr int PAD = 16;
  static constexpr int P1 = R1 * 16 + PAD;   // A1 plane stride
  static constexpr int P2 = R2 * 16 + PAD;   // A2 plane stride
  static constexpr int P3 = R3 * 16 + PAD;   // A3 plane stride (aliases A1)
  static constexpr int PB1 = MC * 16;        // W1^T: MC rows, K = C
  static constexpr int PB2 = MC * 16;        // W2^T per tap: MC rows, K = MC
  static constexpr int TAPB = (MC / 8) * PB2;
  static constexpr int PB3 = C * 16;         // W3^T: C rows, K = MC
  static constexpr int al(int v) { return (v + 127) / 128 * 128; }
  static constexpr int SZ_A1 = al((C / 8) * P1 > (MC / 8) * P3 ? (C / 8) * P1 : (MC / 8) * P3);
  static constexpr int SZ_A2 = al((MC / 8) * P2);
  static constexpr int SZ_B1 = al((C / 8) * PB1);
  static constexpr int SZ_B2 = al(9 * TAPB);
  static constexpr int SZ_B3 = al((MC / 8) * PB3);
  static constexpr int NPAR = 4 * C + 6 * MC;  // s1 t1 b3 + b1 s2 t2 b2 s3 t3 (floats)
  static constexpr int OFF_A2 = SZ_A1;
  static constexpr int OFF_B1 = OFF_A2 + SZ_A2;
  static constexpr int OFF_B2 = OFF_B1 + SZ_B1;
  static constexpr int OFF_B3 = OFF_B2 + SZ_B2;
  static constexpr int OFF_PAR = OFF_B3 + SZ_B3;
  static constexpr int SMEM = OFF_PAR + al(NPAR * 4);
  static constexpr int COL1 = 0;
  static constexpr int COL2 = NT1 * MC;
  static constexpr int COL3 = COL2 + NT2 * MC;
  static constexpr int TCOLS = COL3 + NT2 * C;
  static_assert(TCOLS <= 512, "TMEM budget");
  static constexpr int TALLOC = TCOLS <= 32 ? 32 : TCOLS <= 64 ? 64 : TCOLS <= 128 ? 128 : TCOLS <= 256 ? 256 : 512;
  static constexpr int OCC = (SMEM <= 110 * 1024 && TALLOC <= 256) ? 2 : 1;
};

struct TcArgs {
  const __nv_bfloat16* x;
  __nv_bfloat16* out;
  const __nv_bfloat16* rim;
  Geo g;
  const __nv_bfloat16 *w1, *b1, *w2, *b2, *w3, *b3;
  const float *s1, *t1, *s2, *t2, *s3, *t3;
  const uint8_t* packed;  // smem image of [B1 | B2 | B3 | params] (unit_tc_pack)
  __nv_bfloat16* rim_buf;  // in place, more blocks than CTAs: halo rims snapshotted here
  unsigned int* gbar;      // grid-barrier words (in place only)
  unsigned long long* trace;
  const uint8_t* mask;     // non-null: fused reduce_mask (MAX) + compaction into idx/count
  unsigned long long* cst; // (unused; reserved)
  unsigned long long* etag;  // slot compaction: per-entry (launch tag << 32 | candidate) word
  unsigned int* sw;          // slot words: [0] epoch, [4 + 4 * (tag & 1) + {0 slot, 1 done, 2 staged}]
                             // (same workspace as etag, fixed offsets: reset together)
  int32_t* idx_out;
  int32_t* count_out;
  const int32_t* idx;
  const int32_t* count;
  int cap;
  int early_mask;  // fused: test the first round of candidates before griddepcontrol.wait
};

__device__ __forceinline__ float bf(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// ---- slot compaction (fused mask reduction of the single-kernel sparse_residual_unit).
// Producers: CTA c tests candidates c, c+G, ... against the mask, claims list slots for its
// active ones with ONE atomic per round, publishes each entry as one 64-bit word
// (launch tag << 32 | candidate: a single-copy-atomic store, so no release fence and no
// second read on the consumer side), then increments `done`.  (An L2 prefetch of the
// window issued here by the producer measured slower: it delays `done`, which gates the
// in-place stores.)  Consumers only wait for the entry
// they process (or for done == G to learn that no more entries are coming).  In place,
// the halo hazard is resolved just before the first store (slot_before_store).  Nothing is
// reset on the critical path and no CTA does a global atomic on its way out: the counters
// of launch `tag` live in ring slot tag & 1, and the LAST producer (its `done` increment
// returns G-1, so every CTA has read the epoch) publishes the block count, bumps the epoch
// and zeroes the other slot (its launch completed before this one passed
// griddepcontrol.wait; the next launch will use it).  Tags make stale entries invisible.
//   words: sw[0] epoch, sw[4 + 4 * (tag & 1) + {0 slot counter, 1 done, 2 staged}] (at the
//   start of the unit workspace, before the tagged entries); sync ws [13..14] grid barrier
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release(unsigned* p, unsigned v) {
  asm volatile("red.add.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned* slot_ring(const TcArgs& a, unsigned tag) { return a.sw + 4 + 4 * (tag & 1u); }
// Entry word: hashed launch tag (odd multiplier: a bijection, and far from the small
// integers / activation bits other users of a shared workspace leave behind) << 32 | candidate.
__device__ __forceinline__ unsigned tag_hash(unsigned tag) { return tag * 0x9E3779B1u; }
__device__ __forceinline__ unsigned long long slot_word(unsigned tag, int cand) {
  return ((unsigned long long)tag_hash(tag) << 32) | (unsigned)cand;
}
__device__ __forceinline__ bool slot_match(unsigned long long e, unsigned tag) {
  return (unsigned)(e >> 32) == tag_hash(tag);
}

// Flags of one round of this CTA's candidates (r0 + j*G, j < 32) in shared memory.
struct SlotSmem {
  int flag[32], fr[32], y0[32], x0[32];
  int base;
  unsigned tag;
};

template <int C, int BS>
__device__ __forceinline__ void slot_test(const TcArgs& a, SlotSmem& ss, int r0) {
  const Geo& g = a.g;
  const int tid = threadIdx.x;
  const int T = g.n * g.gy * g.gx;
  constexpr int area = BS * BS;  // the unit's window (bh == bw == BS)
  const int G = gridDim.x;
  const int nj = min(32, (T - r0 + G - 1) / G);
  if (tid < 32) {
    ss.flag[tid] = 0;
    const int cand = r0 + tid * G;
    const int fr = cand / (g.gy * g.gx), rr = cand - fr * (g.gy * g.gx);
    const int cy = rr / g.gx, cx = rr - cy * g.gx;
    ss.fr[tid] = fr;
    ss.y0[tid] = g.oy + cy * g.sy;
    ss.x0[tid] = g.ox + cx * g.sx;
  }
  __syncthreads();
  constexpr int U = 4;  // loads in flight per thread before any is tested
  for (int e0 = tid; e0 < nj * area; e0 += U * kThreads) {
    uint8_t v[U];
    int jj[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kThreads;
      const int j = min(e / area, 31), p = e % area;
      const int fr = ss.fr[j];
      const int y = ss.y0[j] + p / BS, xx = ss.x0[j] + p % BS;
      jj[u] = j;
      v[u] = (e < nj * area && y >= 0 && y < g.h && xx >= 0 && xx < g.w)
                 ? __ldg(a.mask + ((size_t)fr * g.h + y) * g.w + xx) : (uint8_t)0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v[u]) ss.flag[jj[u]] = 1;
  }
  __syncthreads();
}

// Returns this launch's tag (epoch + 1).  Thread 32 gets the old value of its `done`
// increment in `done_old`; it is only consumed by slot_last_producer, after the CTA has
// polled for its entry (the round trip overlaps).  `pretested`: the first round's flags are
// already in `ss` — the kernels test their first round of candidates BEFORE
// griddepcontrol.wait, overlapping the previous kernel's tail (the mask, like the packed
// weights, is never written by a kernel that triggers its dependents early).
template <int C, int BS>
__device__ __forceinline__ unsigned slot_produce(const TcArgs& a, SlotSmem& ss, bool pretested, unsigned& done_old) {
  const Geo& g = a.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned ep = 0;
  if (tid == 0) ep = ld_relaxed_u32(a.sw);
  const int T = g.n * g.gy * g.gx;
  const int G = gridDim.x;
  for (int r0 = blockIdx.x; r0 < T; r0 += 32 * G) {
    const int nj = min(32, (T - r0 + G - 1) / G);
    if (!(pretested && r0 == (int)blockIdx.x)) slot_test<C, BS>(a, ss, r0);
    if (tid == 0) ss.tag = ep + 1u;
    __syncthreads();
    trace(a.trace, 12);
    const unsigned tag = ss.tag;
    if (warp == 0) {
      const bool on = lane < nj && ss.flag[lane];
      const unsigned bal = __ballot_sync(0xffffffffu, on);
      if (lane == 0) ss.base = bal ? (int)atomicAdd(slot_ring(a, tag), (unsigned)__popc(bal)) : 0;
      __syncwarp();
      if (bal) trace(a.trace, 19);
      if (on) {
        const int pos = ss.base + __popc(bal & ((1u << lane) - 1u));
        const int cand = r0 + lane * G;
        const int fr = cand / (g.gy * g.gx), rr = cand - fr * (g.gy * g.gx);
        const int by = rr / g.gx, bx = rr % g.gx;
        st_relaxed_u64(&a.etag[pos], slot_word(tag, cand));
        a.idx_out[3 * pos] = fr;
        a.idx_out[3 * pos + 1] = by;
        a.idx_out[3 * pos + 2] = bx;
      }
    }
    __syncthreads();  // warp 0's reads of this round's flags before the next round's test
  }
  if (T <= (int)blockIdx.x && tid == 0) ss.tag = ep + 1u;  // no candidate for this CTA
  __syncthreads();
  const unsigned tag = ss.tag;
  if (tid == 32) done_old = atom_add_release(slot_ring(a, tag) + 1, 1u);
  trace(a.trace, 14);
  return tag;
}

// the kernels' early half of slot_produce: the first round of mask tests, before
// griddepcontrol.wait
template <int C, int BS>
__device__ __forceinline__ bool slot_pretest(const TcArgs& a, SlotSmem& ss) {
  if (a.mask == nullptr || (int)blockIdx.x >= a.g.n * a.g.gy * a.g.gx || !a.early_mask) return false;
  slot_test<C, BS>(a, ss, blockIdx.x);
  return true;
}

// The last producer (done_old == G - 1: every CTA has read the epoch) publishes the block
// count, zeroes the other ring slot and bumps the epoch.
__device__ __forceinline__ void slot_last_producer(const TcArgs& a, unsigned tag, unsigned done_old) {
  if (threadIdx.x == 32 && done_old == gridDim.x - 1) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const unsigned nb = ld_relaxed_u32(slot_ring(a, tag));
    *a.count_out = (int)nb;
    slot_ring(a, tag)[3] = nb + 1u;  // final block count (+1: 0 = not yet), for slot_before_store
    unsigned* other = slot_ring(a, tag + 1u);
    other[0] = 0u;
    other[1] = 0u;
    other[2] = 0u;
    other[3] = 0u;  // spare ring word: kept zero like the others
    a.sw[0] = tag;
  }
}

// In-place fused: called by every consumer CTA once its FIRST window is read, i.e. after
// the barrier that follows the A1 staging (every thread has consumed its loaded registers,
// so every window load has returned its value).  The in-place hazard is write-after-read
// only (a neighbour's store into this window must not reach a load of it), and a load that
// has returned cannot observe a later store, so a relaxed increment issued after that
// barrier suffices; the reader (slot_before_store) issues its stores only after observing
// the count (control dependency; stores are never issued speculatively).  The release /
// acquire pair this replaced cost ~0.45 us per fence on the critical path of every step.
__device__ __forceinline__ void slot_staged(const TcArgs& a, unsigned tag) {
  if (threadIdx.x == 32) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(slot_ring(a, tag) + 2) : "memory");
}

// In-place fused, before the first store of the first block.  If every block had its own
// consumer (B <= ncons) all windows were staged from x before any store: wait until all
// B * ctas_per_block consumers have staged.  Otherwise (more blocks than consumers) the
// rims of the blocks processed in later rounds are snapshotted now, by all CTAs, behind a
// grid barrier (every CTA is active then).  Returns true when later rounds must read rims
// from the snapshot.
template <int C, int BS>
__device__ __forceinline__ bool slot_before_store(const TcArgs& a, unsigned tag, int ncons, int ctas_per_block,
                                                  int& nblocks) {
  __shared__ int s_B;
  __syncthreads();
  if (threadIdx.x == 0) {
    // ring[3] = final block count + 1 (slot_last_producer) and ring[2] = staged consumers,
    // both polled in one round trip (no fence: see slot_staged)
    unsigned* ring = slot_ring(a, tag);
    SpinGuard sg;
    unsigned f, st;
    while (true) {
      f = ld_relaxed_u32(ring + 3);
      st = ld_relaxed_u32(ring + 2);
      if (f != 0u && (f - 1u > (unsigned)ncons || st >= (f - 1u) * (unsigned)ctas_per_block)) break;
      __nanosleep(32);
      sg.tick(kSpinSlotStaged);
    }
    s_B = (int)(f - 1u);
  }
  __syncthreads();
  const int B = s_B;
  nblocks = B;
  if (B <= ncons) return false;
  const Geo& g = a.g;
  const Rim r{BS, BS, 1};
  const int Pr = r.pixels();
  for (int blk = ncons + blockIdx.x; blk < B; blk += gridDim.x) {
    const int n = __ldcg(a.idx_out + 3 * blk), by = __ldcg(a.idx_out + 3 * blk + 1), bx = __ldcg(a.idx_out + 3 * blk + 2);
    const int ys = g.oy + by * g.sy, xs = g.ox + bx * g.sx;
    for (int i = threadIdx.x; i < Pr * (C / 8); i += kThreads) {
      const int rp = i / (C / 8), k = i % (C / 8);
      int wy, wx;
      r.coord(rp, wy, wx);
      const int y = ys + wy, xx = xs + wx;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (y >= 0 && y < g.h && xx >= 0 && xx < g.w)
        v = *(reinterpret_cast<const uint4*>(a.x) + (((size_t)n * g.h + y) * g.w + xx) * (C / 8) + k);
      reinterpret_cast<uint4*>(a.rim_buf)[((size_t)blk * Pr + rp) * (C / 8) + k] = v;
    }
  }
  grid_barrier(a.gbar + 13, gridDim.x);
  return true;
}

#ifndef SBN_ENTRY_POLL_NS
#define SBN_ENTRY_POLL_NS 64  // back-off per entry poll: config 2 at 10 % 11.75 -> 11.56 us (tools/poll_ab.sh)
#endif
// Entry `blk` of this launch: returns false when the list is complete and shorter.
__device__ __forceinline__ bool slot_entry(const TcArgs& a, unsigned tag, int blk, int& n, int& by,
                                           int& bx) {
  __shared__ int s_e[4];
  if (blk >= a.g.n * a.g.gy * a.g.gx) return false;  // more consumers than candidates
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* ring = slot_ring(a, tag);
    int ok = 0;
    unsigned long long e = 0;
    SpinGuard sg;
    while (true) {  // both words in flight per iteration: one round trip per poll
      sg.tick(kSpinSlotEntry);
#if SBN_ENTRY_POLL_NS > 0
      __nanosleep(SBN_ENTRY_POLL_NS);  // back off the L2 line the producers' `done` atomics hit
#endif
      e = ld_relaxed_u64(&a.etag[blk]);
      const unsigned d = ld_relaxed_u32(ring + 1);
      if (slot_match(e, tag)) {
        ok = 1;
        break;
      }
      if (d == gridDim.x) {  // all producers done: re-read the entry after an acquire
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        e = ld_relaxed_u64(&a.etag[blk]);
        ok = slot_match(e, tag) ? 1 : 0;
        break;
      }
    }
    s_e[3] = ok;
    if (ok) {
      const Geo& g = a.g;
      const int cand = (int)(unsigned)e;
      const int fr = cand / (g.gy * g.gx), rr = cand - fr * (g.gy * g.gx);
      s_e[0] = fr;
      s_e[1] = rr / g.gx;
      s_e[2] = rr % g.gx;
    }
  }
  __syncthreads();
  n = s_e[0];
  by = s_e[1];
  bx = s_e[2];
  return s_e[3] != 0;
}

// Prefetch block `blk`'s in-image window rows into L2 (one bulk prefetch per row), so the
// next iteration's window loads hit L2.  Fused mode: only if the entry is already published.
template <int C, int BS>
__device__ __forceinline__ void prefetch_window(const TcArgs& a, const int32_t* idx, unsigned tag,
                                                int blk) {
  const Geo& g = a.g;
  if (threadIdx.x >= 32 || blk >= g.n * g.gy * g.gx) return;
  int n, by, bx;
  if (tag) {
    const unsigned long long e = ld_relaxed_u64(&a.etag[blk]);
    if (!slot_match(e, tag)) return;
    const int cand = (int)(unsigned)e;
    n = cand / (g.gy * g.gx);
    const int rr = cand - n * (g.gy * g.gx);
    by = rr / g.gx;
    bx = rr % g.gx;
  } else {
    if (blk >= ld_count(a.count, a.cap)) return;
    n = __ldcg(idx + 3 * blk), by = __ldcg(idx + 3 * blk + 1), bx = __ldcg(idx + 3 * blk + 2);
  }
  const int ys = g.oy + by * g.sy, xs = g.ox + bx * g.sx;
  const int x0 = max(xs, 0), x1 = min(xs + BS, g.w);
  const int wy = threadIdx.x;
  const int y = ys + wy;
  if (wy < BS && y >= 0 && y < g.h && x1 > x0)
    tc::prefetch_l2(a.x + (((size_t)n * g.h + y) * g.w + x0) * C, (uint32_t)((x1 - x0) * C * 2));
}

template <int C, int MC, int BS>
__global__ void __launch_bounds__(kThreads, Cfg<C, MC, BS>::OCC) unit_tc_kernel(TcArgs a) {
  using K = Cfg<C, MC, BS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* A1 = smem;
  uint8_t* A2 = smem + K::OFF_A2;
  uint8_t* A3 = smem;  // alias: A1 is dead once GEMM1 has completed
  uint8_t* B1 = smem + K::OFF_B1;
  uint8_t* B2 = smem + K::OFF_B2;
  uint8_t* B3 = smem + K::OFF_B3;
  float* par = reinterpret_cast<float*>(smem + K::OFF_PAR);
  float* s1 = par;
  float* t1 = s1 + C;
  float* b3 = t1 + C;
  float* b1 = b3 + C;
  float* s2 = b1 + MC;
  float* t2 = s2 + MC;
  float* b2 = t2 + MC;
  float* s3 = b2 + MC;
  float* t3 = s3 + MC;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Geo& g = a.g;

  trace(a.trace, 0);
  // ---- prologue: one bulk (TMA) copy of the pre-packed weight/param image; it lands
  //      while the first window is being loaded
  __shared__ uint64_t wbar;
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&wbar, 1);
    tc::mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
    constexpr uint32_t bytes = K::SMEM - K::OFF_B1;
    tc::mbar_expect_tx(&wbar, bytes);
    tc::bulk_g2s(B1, a.packed, bytes, &wbar);
  }
  __shared__ SlotSmem ss;
  const bool pretested = slot_pretest<C, BS>(a, ss);  // under the previous kernel's tail
  if (warp == 0) tc::tmem_alloc<K::TALLOC>(&tslot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  uint32_t phase = 0;
  bool weights_ready = false;

  trace(a.trace, 1);
  // everything above overlaps the previous kernel (reduce_mask) under PDL; the next
  // launch may start its own prologue now (its griddepcontrol.wait still waits for this
  // grid to complete and flush)
  tc::pdl_trigger();
  tc::pdl_wait();
  int n0 = 0, by0 = 0, bx0 = 0;
  int B = 0;
  const int32_t* idx = a.idx;
  unsigned tag = 0;
  const bool inplace = a.x == a.out;
  const bool fused = a.mask != nullptr;
  bool have;
  if (fused) {  // mask -> blocks in this kernel (slot compaction), see slot_produce
    unsigned done_old = 0;
    tag = slot_produce<C, BS>(a, ss, pretested, done_old);
    idx = a.idx_out;
    have = slot_entry(a, tag, blockIdx.x, n0, by0, bx0);
    slot_last_producer(a, tag, done_old);
  } else {
    if ((int)blockIdx.x < a.cap) {  // speculative: the first block's row, loaded alongside the count
      n0 = __ldg(idx + 3 * blockIdx.x);
      by0 = __ldg(idx + 3 * blockIdx.x + 1);
      bx0 = __ldg(idx + 3 * blockIdx.x + 2);
    }
    B = ld_count(a.count, a.cap);
    have = (int)blockIdx.x < B;
  }
  trace(a.trace, 2);
  // In place, a block's halo rim is its neighbours' interior, which they overwrite.
  //  fused:     windows are staged straight from x; before the first store,
  //             slot_before_store waits until every block's consumer has staged (or, with
  //             more blocks than consumers, snapshots the later rounds' rims).
  //  resident (B <= grid): every block has its own CTA; all windows are staged before
  //                        any CTA writes (split grid barrier: arrive after staging, wait
  //                        before epilogue 3).
  //  streamed (B > grid):  rims of all blocks are snapshotted first (grid barrier),
  //                        then windows read interiors from x and rims from the snapshot.
  const bool resident = !fused && B <= (int)gridDim.x;
  const __nv_bfloat16* rimsrc = a.rim;
  bool first_store = fused && inplace;  // slot_before_store still pending
  int known_B = -1;                     // block count, once slot_before_store has read it
  if (!fused && inplace && !resident) {
    const Rim r{BS, BS, 1};
    const int Pr = r.pixels();
    for (int blk = blockIdx.x; blk < B; blk += gridDim.x) {
      const int n = __ldcg(idx + 3 * blk), by = __ldcg(idx + 3 * blk + 1), bx = __ldcg(idx + 3 * blk + 2);
      const int ys = g.oy + by * g.sy, xs = g.ox + bx * g.sx;
      for (int i = tid; i < Pr * (C / 8); i += kThreads) {
        const int rp = i / (C / 8), k = i % (C / 8);
        int wy, wx;
        r.coord(rp, wy, wx);
        const int y = ys + wy, xx = xs + wx;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (y >= 0 && y < g.h && xx >= 0 && xx < g.w)
          v = *(reinterpret_cast<const uint4*>(a.x) + (((size_t)n * g.h + y) * g.w + xx) * (C / 8) + k);
        reinterpret_cast<uint4*>(a.rim_buf)[((size_t)blk * Pr + rp) * (C / 8) + k] = v;
      }
    }
    grid_barrier(a.gbar, gridDim.x);
    rimsrc = a.rim_buf;
  }
  if (!have) {  // idle CTA: drain the weight copy, release TMEM
    tc::mbar_wait(&wbar, 0);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == 0) tc::tmem_free<K::TALLOC>(tmem);
    return;
  }

  const Rim rim{BS, BS, 1};
  const int P = rim.pixels();
  const int q = warp & 3;           // TMEM lane quarter of this warp
  const int tpar = warp >> 2;       // tile parity handled by this warp

  for (int blk = blockIdx.x;;) {
    const int n = n0, by = by0, bx = bx0;
    const int ys = g.oy + by * g.sy, xs = g.ox + bx * g.sx;

    // ---- 1. stage the window: all loads in flight first, then BN1 + ReLU -> bf16 planes
    constexpr int TOT = K::NPIX * (C / 8);
    constexpr int ITEMS = (TOT + kThreads - 1) / kThreads;
    uint4 raw[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const int i = tid + it * kThreads;
      const int p = i / (C / 8), k = i % (C / 8);
      const int wy = p / BS, wx = p % BS;
      const int y = ys + wy, xx = xs + wx;
      const bool from_rim = rimsrc && !rim.interior(wy, wx);
      const bool inb = y >= 0 && y < g.h && xx >= 0 && xx < g.w;
      const uint4* src = from_rim
          ? reinterpret_cast<const uint4*>(rimsrc) + ((size_t)blk * P + rim.index(wy, wx)) * (C / 8) + k
          : reinterpret_cast<const uint4*>(a.x) + (((size_t)n * g.h + (inb ? y : 0)) * g.w + (inb ? xx : 0)) * (C / 8) + k;
      raw[it] = tc::ld_v4_pred(src, (i < TOT) && (from_rim || inb));
    }
    trace(a.trace, 3);
    prefetch_window<C, BS>(a, idx, tag, blk + gridDim.x);  // after this block's loads are issued
    // in place + resident: announce "my window is read"; the matching wait sits right
    // before the first store of epilogue 3, so it overlaps the three GEMMs
    if (inplace && resident) grid_arrive(a.gbar);
    trace(a.trace, 4);
    if (!weights_ready) {
      tc::mbar_wait(&wbar, 0);
      weights_ready = true;
    }
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const int i = tid + it * kThreads;
      if (i >= TOT) break;
      const int p = i / (C / 8), k = i % (C / 8);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[it]);
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        const int ch = k * 8 + 2 * e;
        const float v0 = fmaxf(__fadd_rn(__fmul_rn(f.x, s1[ch]), t1[ch]), 0.f);
        const float v1 = fmaxf(__fadd_rn(__fmul_rn(f.y, s1[ch + 1]), t1[ch + 1]), 0.f);
        o[e] = tc::pack_bf16(v0, v1);
      }
      *reinterpret_cast<uint4*>(A1 + k * K::P1 + p * 16) = make_uint4(o[0], o[1], o[2], o[3]);
    }
    tc::fence_async_smem();
    __syncthreads();
    if (first_store) slot_staged(a, tag);  // window read (see slot_staged)
    trace(a.trace, 5);

    // ---- 2. GEMM1: C1 = A1 . W1
    if (tid == 0) {
      tc::fence_after();
      constexpr uint32_t id1 = tc::idesc_bf16_f32(128, MC);
#pragma unroll
      for (int t = 0; t < K::NT1; ++t)
#pragma unroll
        for (int k = 0; k < C / 16; ++k)
          tc::mma_bf16(tmem + K::COL1 + t * MC,
                       tc::desc_add(tc::desc_kmajor_noswz(tc::smem_u32(A1), K::P1, 128), 2 * k * K::P1 + t * 128 * 16),
                       tc::desc_add(tc::desc_kmajor_noswz(tc::smem_u32(B1), K::PB1, 128), 2 * k * K::PB1), id1, k > 0);
      tc::mma_commit(&bar);
      trace(a.trace, 12);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after();

    trace(a.trace, 6);
    // ---- 3. epilogue 1: +b1, BN2, ReLU, x in-bounds -> A2
    for (int t = tpar; t < K::NT1; t += 2) {
      const int r = t * 128 + q * 32 + lane;
      const int wy = r / BS, wx = r % BS;
      const int y = ys + wy, xx = xs + wx;
      const bool valid = r < K::NPIX && y >= 0 && y < g.h && xx >= 0 && xx < g.w;
#pragma unroll
      for (int c0 = 0; c0 < MC; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + K::COL1 + t * MC + c0, v);
        uint32_t o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float u0 = __bfloat162float(__float2bfloat16_rn(v[2 * e] + b1[c0 + 2 * e]));
          float u1 = __bfloat162float(__float2bfloat16_rn(v[2 * e + 1] + b1[c0 + 2 * e + 1]));
          u0 = fmaxf(__fadd_rn(__fmul_rn(u0, s2[c0 + 2 * e]), t2[c0 + 2 * e]), 0.f);
          u1 = fmaxf(__fadd_rn(__fmul_rn(u1, s2[c0 + 2 * e + 1]), t2[c0 + 2 * e + 1]), 0.f);
          o[e] = valid ? tc::pack_bf16(u0, u1) : 0u;
        }
        *reinterpret_cast<uint4*>(A2 + (c0 / 8) * K::P2 + r * 16) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(A2 + (c0 / 8 + 1) * K::P2 + r * 16) = make_uint4(o[4], o[5], o[6], o[7]);
      }
    }
    tc::fence_before();
    tc::fence_async_smem();
    __syncthreads();

    trace(a.trace, 7);
    // ---- 4. GEMM2: 3x3 valid conv as 9 row-shifted views of A2
    if (tid == 0) {
      tc::fence_after();
      constexpr uint32_t id2 = tc::idesc_bf16_f32(128, MC);
#pragma unroll
      for (int t = 0; t < K::NT2; ++t)
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const int shift = (tap / 3) * BS + (tap % 3);
#pragma unroll
          for (int k = 0; k < MC / 16; ++k)
            tc::mma_bf16(tmem + K::COL2 + t * MC,
                         tc::desc_add(tc::desc_kmajor_noswz(tc::smem_u32(A2), K::P2, 128), 2 * k * K::P2 + (t * 128 + shift) * 16),
                         tc::desc_add(tc::desc_kmajor_noswz(tc::smem_u32(B2), K::PB2, 128), tap * K::TAPB + 2 * k * K::PB2),
                         id2, (tap | k) > 0);
        }
      tc::mma_commit(&bar);
      trace(a.trace, 13);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after();

    trace(a.trace, 8);
    // ---- 5. epilogue 2: +b2, BN3, ReLU -> A3; prefetch this row's residual (x at the
    //      output pixel) so its latency hides under GEMM3
    constexpr bool kPrefetch = K::NT2 <= 2;
    uint4 res[kPrefetch ? C / 8 : 1];
    if (kPrefetch && tpar < K::NT2) {
      const int r = tpar * 128 + q * 32 + lane;
      const int oy = r / BS, ox = r % BS;
      const int Y = by * g.obh + oy, X = bx * g.obw + ox;
      const bool st = oy < BS - 2 && ox < BS - 2 && Y < g.oh && X < g.ow;
      const uint4* op = reinterpret_cast<const uint4*>(a.out) +
                        (((size_t)n * g.oh + (st ? Y : 0)) * g.ow + (st ? X : 0)) * (C / 8);
#pragma unroll
      for (int k = 0; k < (kPrefetch ? C / 8 : 1); ++k) res[k] = tc::ld_v4_pred(op + k, st);
    }
    for (int t = tpar; t < K::NT2; t += 2) {
      const int r = t * 128 + q * 32 + lane;
#pragma unroll
      for (int c0 = 0; c0 < MC; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + K::COL2 + t * MC + c0, v);
        uint32_t o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float u0 = __bfloat162float(__float2bfloat16_rn(v[2 * e] + b2[c0 + 2 * e]));
          float u1 = __bfloat162float(__float2bfloat16_rn(v[2 * e + 1] + b2[c0 + 2 * e + 1]));
          u0 = fmaxf(__fadd_rn(__fmul_rn(u0, s3[c0 + 2 * e]), t3[c0 + 2 * e]), 0.f);
          u1 = fmaxf(__fadd_rn(__fmul_rn(u1, s3[c0 + 2 * e + 1]), t3[c0 + 2 * e + 1]), 0.f);
          o[e] = tc::pack_bf16(u0, u1);
        }
        *reinterpret_cast<uint4*>(A3 + (c0 / 8) * K::P3 + r * 16) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(A3 + (c0 / 8 + 1) * K::P3 + r * 16) = make_uint4(o[4], o[5], o[6], o[7]);
      }
    }
    tc::fence_before();
    tc::fence_async_smem();
    __syncthreads();

    trace(a.trace, 9);
    // ---- 6. GEMM3: C3 = A3 . W3
    if (tid == 0) {
      tc::fence_after();
      constexpr uint32_t id3 = tc::idesc_bf16_f32(128, C);
#pragma unroll
      for (int t = 0; t < K::NT2; ++t)
#pragma unroll
        for (int k = 0; k < MC / 16; ++k)
          tc::mma_bf16(tmem + K::COL3 + t * C,
                       tc::desc_add(tc::desc_kmajor_noswz(tc::smem_u32(A3), K::P3, 128), 2 * k * K::P3 + t * 128 * 16),
                       tc::desc_add(tc::desc_kmajor_noswz(tc::smem_u32(B3), K::PB3, 128), 2 * k * K::PB3), id3, k > 0);
      tc::mma_commit(&bar);
      trace(a.trace, 14);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after();

    if (inplace && resident) grid_wait(a.gbar, (unsigned)B);  // neighbours have read my rim
    if (first_store) {  // fused in place: neighbours staged / later rims snapshotted
      if (slot_before_store<C, BS>(a, tag, (int)gridDim.x, 1, known_B)) rimsrc = a.rim_buf;
      first_store = false;
    }
    trace(a.trace, 10);
    // ---- 7. epilogue 3: +b3, + residual, store the block's clipped output window
    for (int t = tpar; t < K::NT2; t += 2) {
      const int r = t * 128 + q * 32 + lane;
      const int oy = r / BS, ox = r % BS;
      const int Y = by * g.obh + oy, X = bx * g.obw + ox;
      const bool store = oy < BS - 2 && ox < BS - 2 && Y < g.oh && X < g.ow;
      uint4* op = reinterpret_cast<uint4*>(a.out) + (((size_t)n * g.oh + (store ? Y : 0)) * g.ow + (store ? X : 0)) * (C / 8);
#pragma unroll
      for (int c0 = 0; c0 < C; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + K::COL3 + t * C + c0, v);
        if (store) {
          uint4 xr[2];
          if constexpr (kPrefetch) {
            xr[0] = res[c0 / 8];
            xr[1] = res[c0 / 8 + 1];
          } else {
            xr[0] = op[c0 / 8];
            xr[1] = op[c0 / 8 + 1];
          }
          const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(xr);
          uint32_t o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float2 xf = __bfloat1622float2(xh[e]);
            const float u0 = __bfloat162float(__float2bfloat16_rn(v[2 * e] + b3[c0 + 2 * e]));
            const float u1 = __bfloat162float(__float2bfloat16_rn(v[2 * e + 1] + b3[c0 + 2 * e + 1]));
            o[e] = tc::pack_bf16(__fadd_rn(xf.x, u0), __fadd_rn(xf.y, u1));
          }
          op[c0 / 8] = make_uint4(o[0], o[1], o[2], o[3]);
          op[c0 / 8 + 1] = make_uint4(o[4], o[5], o[6], o[7]);
        }
      }
    }
    tc::fence_before();
    __syncthreads();
    trace(a.trace, 11);
    blk += gridDim.x;
    if (fused) {
      // the block count is known after the in-place wait: no poll when the list is done
      if ((known_B >= 0 && blk >= known_B) || !slot_entry(a, tag, blk, n0, by0, bx0)) break;
    } else {
      if (blk >= B) break;
      n0 = __ldcg(idx + 3 * blk);
      by0 = __ldcg(idx + 3 * blk + 1);
      bx0 = __ldcg(idx + 3 * blk + 2);
    }
  }

  tc::fence_after();
  if (warp == 0) tc::tmem_free<K::TALLOC>(tmem);
}

// Pre-pack W1/W2/W3 (transposed into the K-major plane layout) and the float params into
// the exact shared-memory image the kernel bulk-copies in its prologue.
template <int C, int MC, int BS>
__global__ void unit_tc_pack_kernel(TcArgs a, uint8_t* __restrict__ img) {
  using K = Cfg<C, MC, BS>;
  uint8_t* B1 = img;
  uint8_t* B2 = img + (K::OFF_B2 - K::OFF_B1);
  uint8_t* B3 = img + (K::OFF_B3 - K::OFF_B1);
  float* par = reinterpret_cast<float*>(img + (K::OFF_PAR - K::OFF_B1));
  const int stride = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = t0; i < (K::SMEM - K::OFF_B1) / 4; i += stride) reinterpret_cast<uint32_t*>(img)[i] = 0u;
  __syncthreads();  // single-CTA launch: zero fill before the scatter below
  for (int i = t0; i < C * MC; i += stride) {
    const int ci = i / MC, j = i % MC;
    *reinterpret_cast<__nv_bfloat16*>(B1 + (ci / 8) * K::PB1 + j * 16 + (ci % 8) * 2) = a.w1[i];
  }
  for (int i = t0; i < 9 * MC * MC; i += stride) {
    const int tap = i / (MC * MC), r = i % (MC * MC), ci = r / MC, j = r % MC;
    *reinterpret_cast<__nv_bfloat16*>(B2 + tap * K::TAPB + (ci / 8) * K::PB2 + j * 16 + (ci % 8) * 2) = a.w2[i];
  }
  for (int i = t0; i < MC * C; i += stride) {
    const int j = i / C, co = i % C;
    *reinterpret_cast<__nv_bfloat16*>(B3 + (j / 8) * K::PB3 + co * 16 + (j % 8) * 2) = a.w3[i];
  }
  float* s1 = par;
  float* t1 = s1 + C;
  float* b3 = t1 + C;
  float* b1 = b3 + C;
  float* s2 = b1 + MC;
  float* t2 = s2 + MC;
  float* b2 = t2 + MC;
  float* s3 = b2 + MC;
  float* t3 = s3 + MC;
  for (int i = t0; i < C; i += stride) {
    s1[i] = a.s1[i];
    t1[i] = a.t1[i];
    b3[i] = bf(a.b3 + i);
  }
  for (int i = t0; i < MC; i += stride) {
    b1[i] = bf(a.b1 + i);
    s2[i] = a.s2[i];
    t2[i] = a.t2[i];
    b2[i] = bf(a.b2 + i);
    s3[i] = a.s3[i];
    t3[i] = a.t3[i];
  }
}

template <int C, int MC, int BS>
int pack(const TcArgs& a, void* img, cudaStream_t s) {
  unit_tc_pack_kernel<C, MC, BS><<<1, 1024, 0, s>>>(a, (uint8_t*)img);
  return launch_status("residual_unit_tc_pack");
}

template <int C, int MC, int BS>
size_t packed_bytes() {
  return (size_t)(Cfg<C, MC, BS>::SMEM - Cfg<C, MC, BS>::OFF_B1);
}

// CTAs per SM that are guaranteed co-resident (grid barriers depend on it).  The CUDA
// occupancy API reports 1 for these tcgen05 kernels although the hardware co-schedules
// more (verified with tools/coresidency_probe.py: 296 CTAs on 148 SMs entered within
// 1.1 us), so residency is computed from the real per-SM limits: registers, shared
// memory, threads, and TMEM columns (512 per SM).
template <typename KernT>
int resident_per_sm(KernT kern, int threads, int dyn_smem, int tmem_cols, int cap_bound) {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return 1;
  const int warps = (threads + 31) / 32;
  const int regs_per_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
  const int by_regs = 65536 / (regs_per_warp * warps);
  const int by_smem = (228 * 1024) / (dyn_smem + (int)fa.sharedSizeBytes + 1024);
  const int by_thr = 2048 / threads;
  const int by_tmem = 512 / tmem_cols;
  int r = by_regs;
  if (by_smem < r) r = by_smem;
  if (by_thr < r) r = by_thr;
  if (by_tmem < r) r = by_tmem;
  if (cap_bound < r) r = cap_bound;
  return r < 1 ? 1 : r;
}

template <int C, int MC, int BS>
int launch(const TcArgs& a, int cap, cudaStream_t s) {
  using K = Cfg<C, MC, BS>;
  auto kern = unit_tc_kernel<C, MC, BS>;
  static PerDeviceOnce attr;  // per instantiation and device
  attr([&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
  });
  int occ = resident_per_sm(kern, kThreads, K::SMEM, K::TALLOC, K::OCC);
  g_last_occ[0] = occ;
  {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess) {
      g_last_occ[2] = fa.numRegs;
      g_last_occ[3] = (int)fa.sharedSizeBytes;
      g_last_occ[4] = fa.maxDynamicSharedSizeBytes;
      g_last_occ[5] = K::SMEM;
      g_last_occ[6] = (int)fa.localSizeBytes;
    }
  }
  if (occ < 1) occ = 1;
  if (occ > K::OCC) occ = K::OCC;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(persistent_grid(cap, occ));  // <= co-resident capacity (grid barrier)
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = K::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = (debug_flags() & kDebugCooperative) ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kern, a);
  return launch_status("residual_unit_tcgen05");
}


// ---------------------------------------------------------------------------------------
// CTA-pair variant (thread-block cluster of 2, block size with exactly two 128-row M-tiles,
// e.g. 16x16): CTA rank r owns M-tile r of the block end to end — it stages only window
// pixels [128r, 128r+128), runs 1-tile GEMMs, and its epilogues cover 128 rows with two
// warps per TMEM lane quarter (column halves).  The 3x3 taps of tile 0 read A2 rows up to
// 128 + 2*BS + 1, which belong to tile 1: rank 1 pushes those rows into rank 0's A2 with
// DSMEM stores during epilogue 1, followed by one cluster barrier.  Per CTA this halves the
// window traffic, the smem-bandwidth-bound GEMM2 MMA stream and the epilogue rows.
template <int C, int MC, int BS>
struct PairCfg {
  using K = Cfg<C, MC, BS>;
  static_assert(K::NT1 == 2 && K::NT2 == 2, "pair variant needs two M-tiles");
  static constexpr int HALO_ROWS = 2 * BS + 2;
  static constexpr int R2 = (128 + HALO_ROWS + 7) / 8 * 8;
  static constexpr int P1 = 128 * 16 + 16;
  static constexpr int P2 = R2 * 16 + 16;
  static constexpr int P3 = 128 * 16 + 16;
  static constexpr int al(int v) { return (v + 127) / 128 * 128; }
  static constexpr int SZ_A1 = al((C / 8) * P1 > (MC / 8) * P3 ? (C / 8) * P1 : (MC / 8) * P3);
  static constexpr int OFF_A2 = SZ_A1;
  static constexpr int OFF_B1 = OFF_A2 + al((MC / 8) * P2);
  static constexpr int IMG = K::SMEM - K::OFF_B1;  // same packed image as the single-CTA kernel
  static constexpr int OFF_B2 = OFF_B1 + (K::OFF_B2 - K::OFF_B1);
  static constexpr int OFF_B3 = OFF_B1 + (K::OFF_B3 - K::OFF_B1);
  static constexpr int OFF_PAR = OFF_B1 + (K::OFF_PAR - K::OFF_B1);
  // raw x of this CTA's 128 window pixels plus (rank 0) the partner's first BS + 1 (the
  // residual of epilogue 3: output row o is window pixel o + BS + 1), 16-byte chunks
  // XOR-swizzled by pixel
  static constexpr int RAW_ROWS = 128 + BS + 1;
  static constexpr int OFF_RAW = OFF_B1 + IMG;
  static constexpr int SZ_RAW = al(RAW_ROWS * C * 2);
  static constexpr int RSW = (C / 8 < 8 ? C / 8 : 8) - 1;  // swizzle mask
  static constexpr int SMEM = OFF_RAW + SZ_RAW;
  static constexpr int COL1 = 0, COL2 = MC, COL3 = 2 * MC;
  static constexpr int TCOLS = 2 * MC + C;
  static constexpr int TALLOC = TCOLS <= 32 ? 32 : TCOLS <= 64 ? 64 : TCOLS <= 128 ? 128 : TCOLS <= 256 ? 256 : 512;
  static_assert(MC % 32 == 0 && C % 32 == 0, "column halves of 16-column chunks");
};

template <int C, int MC, int BS>
__global__ void __launch_bounds__(kThreads, 2) unit_tc_pair_kernel(TcArgs a) {
  using K = Cfg<C, MC, BS>;
  using PK = PairCfg<C, MC, BS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, wbar;
  __shared__ uint32_t tslot;
  uint8_t* A1 = smem;
  uint8_t* A2 = smem + PK::OFF_A2;
  uint8_t* A3 = smem;
  uint8_t* B1 = smem + PK::OFF_B1;
  uint8_t* B2 = smem + PK::OFF_B2;
  uint8_t* B3 = smem + PK::OFF_B3;
  uint4* RAW = reinterpret_cast<uint4*>(smem + PK::OFF_RAW);
  float* par = reinterpret_cast<float*>(smem + PK::OFF_PAR);
  float* s1 = par;
  float* t1 = s1 + C;
  float* b3 = t1 + C;
  float* b1 = b3 + C;
  float* s2 = b1 + MC;
  float* t2 = s2 + MC;
  float* b2 = t2 + MC;
  float* s3 = b2 + MC;
  float* t3 = s3 + MC;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, hf = warp >> 2;  // TMEM lane quarter, column half
  const Geo& g = a.g;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // "this CTA has started": the partner's first DSMEM write (epilogue 1) waits for it
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");

  trace(a.trace, 0);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&wbar, 1);
    tc::mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
    tc::mbar_expect_tx(&wbar, PK::IMG);
    tc::bulk_g2s(B1, a.packed, PK::IMG, &wbar);
  }
  __shared__ SlotSmem ss;
  const bool pretested = slot_pretest<C, BS>(a, ss);  // under the previous kernel's tail
  if (warp == 0) tc::tmem_alloc<PK::TALLOC>(&tslot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  uint32_t phase = 0;
  bool weights_ready = false;
  trace(a.trace, 1);
  tc::pdl_trigger();
  tc::pdl_wait();
  trace(a.trace, 16);
  int B = 0;
  const int32_t* idx = a.idx;
  unsigned tag = 0;
  const bool inplace = a.x == a.out;
  const bool fused = a.mask != nullptr;
  int n1 = 0, by1 = 0, bx1 = 0;
  bool have;
  if (fused) {  // mask -> blocks in this kernel (slot compaction), see slot_produce
    unsigned done_old = 0;
    tag = slot_produce<C, BS>(a, ss, pretested, done_old);
    idx = a.idx_out;
    have = slot_entry(a, tag, pair, n1, by1, bx1);
    slot_last_producer(a, tag, done_old);
  } else {
    B = ld_count(a.count, a.cap);
    have = pair < B;
    if (have) {
      n1 = __ldcg(idx + 3 * pair);
      by1 = __ldcg(idx + 3 * pair + 1);
      bx1 = __ldcg(idx + 3 * pair + 2);
    }
  }
  trace(a.trace, 2);
  const bool resident = !fused && B <= npairs;
  const __nv_bfloat16* rimsrc = nullptr;
  bool first_store = fused && inplace;  // slot_before_store still pending
  int known_B = -1;                     // block count, once slot_before_store has read it
  if (!fused && inplace && !resident) {  // streamed in place: snapshot every block's rim first
    const Rim r{BS, BS, 1};
    const int Pr = r.pixels();
    for (int blk = blockIdx.x; blk < B; blk += gridDim.x) {
      const int n = __ldcg(idx + 3 * blk), by = __ldcg(idx + 3 * blk + 1), bx = __ldcg(idx + 3 * blk + 2);
      const int ys = g.oy + by * g.sy, xs = g.ox + bx * g.sx;
      for (int i = tid; i < Pr * (C / 8); i += kThreads) {
        const int rp = i / (C / 8), k = i % (C / 8);
        int wy, wx;
        r.coord(rp, wy, wx);
        const int y = ys + wy, xx = xs + wx;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (y >= 0 && y < g.h && xx >= 0 && xx < g.w)
          v = *(reinterpret_cast<const uint4*>(a.x) + (((size_t)n * g.h + y) * g.w + xx) * (C / 8) + k);
        reinterpret_cast<uint4*>(a.rim_buf)[((size_t)blk * Pr + rp) * (C / 8) + k] = v;
      }
    }
    grid_barrier(a.gbar, gridDim.x);
    rimsrc = a.rim_buf;
  }
  if (!have) {  // idle pair
    tc::mbar_wait(&wbar, 0);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == 0) tc::tmem_free<PK::TALLOC>(tmem);
    trace(a.trace, 17);
    return;
  }
  const Rim rim{BS, BS, 1};
  const int P = rim.pixels();
  uint8_t* A2peer = rank > 0 ? cl.map_shared_rank(A2, rank - 1) : nullptr;

  int round = 0;
  for (int blk = pair;;) {
    const int n = n1, by = by1, bx = bx1;
    trace(a.trace, 18);
    const int ys = g.oy + by * g.sy, xs = g.ox + bx * g.sx;
    // ---- 1. stage my half of the window (pixels [128*rank, 128*rank + 128))
    constexpr int TOT = 128 * (C / 8);
    constexpr int ITEMS = TOT / kThreads;
    uint4 raw[ITEMS];
    if (rimsrc == nullptr) {  // every pixel from x (cheap addressing: frame base + y * w + x)
      const uint4* xf = reinterpret_cast<const uint4*>(a.x) + (size_t)n * g.h * g.w * (C / 8);
#pragma unroll
      for (int it = 0; it < ITEMS; ++it) {
        const int i = tid + it * kThreads;
        const int p = rank * 128 + i / (C / 8), k = i % (C / 8);
        const int y = ys + p / BS, xx = xs + p % BS;
        const bool ok = p < K::NPIX && (unsigned)y < (unsigned)g.h && (unsigned)xx < (unsigned)g.w;
        raw[it] = tc::ld_v4_pred(xf + (size_t)(ok ? y * g.w + xx : 0) * (C / 8) + k, ok);
      }
    } else {
#pragma unroll
      for (int it = 0; it < ITEMS; ++it) {
        const int i = tid + it * kThreads;
        const int pl = i / (C / 8), k = i % (C / 8);
        const int p = rank * 128 + pl;
        const int wy = p / BS, wx = p % BS;
        const int y = ys + wy, xx = xs + wx;
        const bool from_rim = !rim.interior(wy, wx);
        const bool inb = y >= 0 && y < g.h && xx >= 0 && xx < g.w;
        const uint4* src = from_rim
            ? reinterpret_cast<const uint4*>(rimsrc) + ((size_t)blk * P + rim.index(wy, wx)) * (C / 8) + k
            : reinterpret_cast<const uint4*>(a.x) + (((size_t)n * g.h + (inb ? y : 0)) * g.w + (inb ? xx : 0)) * (C / 8) + k;
        raw[it] = tc::ld_v4_pred(src, (p < K::NPIX) && (from_rim || inb));
      }
    }
    trace(a.trace, 3);
    if (rank == 0) prefetch_window<C, BS>(a, idx, tag, blk + npairs);
    if (inplace && resident) grid_arrive(a.gbar);
    trace(a.trace, 4);
    if (!weights_ready) {
      tc::mbar_wait(&wbar, 0);
      weights_ready = true;
    }
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const int i = tid + it * kThreads;
      const int pl = i / (C / 8), k = i % (C / 8);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[it]);
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        const int ch = k * 8 + 2 * e;
        const float v0 = fmaxf(__fadd_rn(__fmul_rn(f.x, s1[ch]), t1[ch]), 0.f);
        const float v1 = fmaxf(__fadd_rn(__fmul_rn(f.y, s1[ch + 1]), t1[ch + 1]), 0.f);
        o[e] = tc::pack_bf16(v0, v1);
      }
      *reinterpret_cast<uint4*>(A1 + k * PK::P1 + pl * 16) = make_uint4(o[0], o[1], o[2], o[3]);
      RAW[pl * (C / 8) + (k ^ (pl & PK::RSW))] = raw[it];
    }
    tc::fence_async_smem();
    __syncthreads();
    if (first_store) slot_staged(a, tag);  // window read (see slot_staged)
    trace(a.trace, 5);
    // ---- 2. GEMM1 (one tile)
    if (tid == 0) {
      tc::fence_after();
      constexpr uint32_t id1 = tc::idesc_bf16_f32(128, MC);
#pragma unroll
      for (int k = 0; k < C / 16; ++k)
        tc::mma_bf16(tmem + PK::COL1, tc::desc_add(tc::desc_kmajor_noswz(tc::smem_u32(A1), PK::P1, 128), 2 * k * PK::P1),
                     tc::desc_add(tc::desc_kmajor_noswz(tc::smem_u32(B1), K::PB1, 128), 2 * k * K::PB1), id1, k > 0);
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after();
    trace(a.trace, 6);
    // ---- 3. epilogue 1 -> A2 (local rows; rank>0 also feeds the previous tile's halo rows)
    if (round == 0) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // partner started
    trace(a.trace, 20);
    {
      const int j = q * 32 + lane;
      const int r = rank * 128 + j;
      const int wy = r / BS, wx = r % BS;
      const int y = ys + wy, xx = xs + wx;
      const bool valid = r < K::NPIX && y >= 0 && y < g.h && xx >= 0 && xx < g.w;
#pragma unroll
      for (int c0 = hf * (MC / 2); c0 < (hf + 1) * (MC / 2); c0 += 16) {
        float v[16];
        tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + PK::COL1 + c0, v);
        uint32_t o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float u0 = __bfloat162float(__float2bfloat16_rn(v[2 * e] + b1[c0 + 2 * e]));
          float u1 = __bfloat162float(__float2bfloat16_rn(v[2 * e + 1] + b1[c0 + 2 * e + 1]));
          u0 = fmaxf(__fadd_rn(__fmul_rn(u0, s2[c0 + 2 * e]), t2[c0 + 2 * e]), 0.f);
          u1 = fmaxf(__fadd_rn(__fmul_rn(u1, s2[c0 + 2 * e + 1]), t2[c0 + 2 * e + 1]), 0.f);
          o[e] = valid ? tc::pack_bf16(u0, u1) : 0u;
        }
        const uint4 lo = make_uint4(o[0], o[1], o[2], o[3]), hi = make_uint4(o[4], o[5], o[6], o[7]);
        *reinterpret_cast<uint4*>(A2 + (c0 / 8) * PK::P2 + j * 16) = lo;
        *reinterpret_cast<uint4*>(A2 + (c0 / 8 + 1) * PK::P2 + j * 16) = hi;
        if (rank > 0 && j < PK::HALO_ROWS) {
          *reinterpret_cast<uint4*>(A2peer + (c0 / 8) * PK::P2 + (128 + j) * 16) = lo;
          *reinterpret_cast<uint4*>(A2peer + (c0 / 8 + 1) * PK::P2 + (128 + j) * 16) = hi;
        }
      }
    }
    if (rank > 0) {  // my first BS + 1 raw pixels: the residuals of the partner's last rows
      uint4* peer = cl.map_shared_rank(RAW, rank - 1);
      for (int t = tid; t < (BS + 1) * (C / 8); t += kThreads) {
        const int pl = t / (C / 8), k = t % (C / 8);
        peer[(128 + pl) * (C / 8) + (k ^ ((128 + pl) & PK::RSW))] = RAW[pl * (C / 8) + (k ^ (pl & PK::RSW))];
      }
    }
    trace(a.trace, 21);
    tc::fence_before();
    asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
    cl.sync();  // A2 halo rows (and residual pixels) from the partner have landed
    tc::fence_async_smem();
    trace(a.trace, 7);
    // ---- 4. GEMM2: 9 row-shifted views of A2 (local rows 0 .. 127 + shift)
    if (tid == 0) {
      tc::fence_after();
      constexpr uint32_t id2 = tc::idesc_bf16_f32(128, MC);
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const int shift = (tap / 3) * BS + (tap % 3);
#pragma unroll
        for (int k = 0; k < MC / 16; ++k)
          tc::mma_bf16(tmem + PK::COL2,
                       tc::desc_add(tc::desc_kmajor_noswz(tc::smem_u32(A2), PK::P2, 128), 2 * k * PK::P2 + shift * 16),
                       tc::desc_add(tc::desc_kmajor_noswz(tc::smem_u32(B2), K::PB2, 128), tap * K::TAPB + 2 * k * K::PB2),
                       id2, (tap | k) > 0);
      }
      tc::mma_commit(&bar);
      trace(a.trace, 13);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after();
    trace(a.trace, 8);
    // ---- 5. epilogue 2 -> A3; prefetch this row's residual half
    const int j = q * 32 + lane;
    const int o_row = rank * 128 + j;
    const int oy = o_row / BS, ox = o_row % BS;
    const int Y = by * g.obh + oy, X = bx * g.obw + ox;
    const bool store = oy < BS - 2 && ox < BS - 2 && Y < g.oh && X < g.ow;
    uint4* op = reinterpret_cast<uint4*>(a.out) +
                (((size_t)n * g.oh + (store ? Y : 0)) * g.ow + (store ? X : 0)) * (C / 8) + hf * (C / 16);
    trace(a.trace, 22);
#pragma unroll
    for (int c0 = hf * (MC / 2); c0 < (hf + 1) * (MC / 2); c0 += 16) {
      float v[16];
      tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + PK::COL2 + c0, v);
      uint32_t o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float u0 = __bfloat162float(__float2bfloat16_rn(v[2 * e] + b2[c0 + 2 * e]));
        float u1 = __bfloat162float(__float2bfloat16_rn(v[2 * e + 1] + b2[c0 + 2 * e + 1]));
        u0 = fmaxf(__fadd_rn(__fmul_rn(u0, s3[c0 + 2 * e]), t3[c0 + 2 * e]), 0.f);
        u1 = fmaxf(__fadd_rn(__fmul_rn(u1, s3[c0 + 2 * e + 1]), t3[c0 + 2 * e + 1]), 0.f);
        o[e] = tc::pack_bf16(u0, u1);
      }
      *reinterpret_cast<uint4*>(A3 + (c0 / 8) * PK::P3 + j * 16) = make_uint4(o[0], o[1], o[2], o[3]);
      *reinterpret_cast<uint4*>(A3 + (c0 / 8 + 1) * PK::P3 + j * 16) = make_uint4(o[4], o[5], o[6], o[7]);
    }
    tc::fence_before();
    tc::fence_async_smem();
    __syncthreads();
    trace(a.trace, 9);
    // ---- 6. GEMM3
    if (tid == 0) {
      tc::fence_after();
      constexpr uint32_t id3 = tc::idesc_bf16_f32(128, C);
#pragma unroll
      for (int k = 0; k < MC / 16; ++k)
        tc::mma_bf16(tmem + PK::COL3, tc::desc_add(tc::desc_kmajor_noswz(tc::smem_u32(A3), PK::P3, 128), 2 * k * PK::P3),
                     tc::desc_add(tc::desc_kmajor_noswz(tc::smem_u32(B3), K::PB3, 128), 2 * k * K::PB3), id3, k > 0);
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after();
    trace(a.trace, 23);
    if (inplace && resident) grid_wait(a.gbar, 2u * (unsigned)B);
    if (first_store) {  // fused in place: neighbours staged / later rims snapshotted
      if (slot_before_store<C, BS>(a, tag, npairs, 2, known_B)) rimsrc = a.rim_buf;
      first_store = false;
    }
    trace(a.trace, 10);
    // ---- 7. epilogue 3: +b3 + residual (x at window pixel o_row + BS + 1, staged by this
    //      CTA or, for rank 0's last rows, pushed by the partner in epilogue 1), my column
    //      half of my rows
    const uint4* rsrc = RAW;
    const int rpl = o_row + BS + 1 - rank * 128;
    constexpr int EW = (C / 2) % 32 == 0 ? 32 : 16;  // columns per TMEM load (one wait each)
#pragma unroll
    for (int cc = 0; cc < C / 2; cc += EW) {
      float v[EW];
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + PK::COL3 + hf * (C / 2) + cc;
      if constexpr (EW == 32) tc::tmem_ld32(ta, v);
      else tc::tmem_ld16(ta, v);
      if (store) {
#pragma unroll
        for (int h = 0; h < EW / 16; ++h) {
          const int c0 = hf * (C / 2) + cc + 16 * h;
          const uint4 r0 = rsrc[rpl * (C / 8) + ((c0 / 8) ^ (rpl & PK::RSW))];
          const uint4 r1 = rsrc[rpl * (C / 8) + ((c0 / 8 + 1) ^ (rpl & PK::RSW))];
          const uint32_t xw[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
          uint32_t o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float2 xf = make_float2(__uint_as_float(xw[e] << 16), __uint_as_float(xw[e] & 0xffff0000u));
            const float u0 = __bfloat162float(__float2bfloat16_rn(v[16 * h + 2 * e] + b3[c0 + 2 * e]));
            const float u1 = __bfloat162float(__float2bfloat16_rn(v[16 * h + 2 * e + 1] + b3[c0 + 2 * e + 1]));
            o[e] = tc::pack_bf16(__fadd_rn(xf.x, u0), __fadd_rn(xf.y, u1));
          }
          op[(cc + 16 * h) / 8] = make_uint4(o[0], o[1], o[2], o[3]);
          op[(cc + 16 * h) / 8 + 1] = make_uint4(o[4], o[5], o[6], o[7]);
        }
      }
    }
    tc::fence_before();
    __syncthreads();
    trace(a.trace, 11);
    blk += npairs;
    bool next;
    if (fused) {
      next = !(known_B >= 0 && blk >= known_B) && slot_entry(a, tag, blk, n1, by1, bx1);
    } else {
      next = blk < B;
      if (next) {
        n1 = __ldcg(idx + 3 * blk);
        by1 = __ldcg(idx + 3 * blk + 1);
        bx1 = __ldcg(idx + 3 * blk + 2);
      }
    }
    if (!next) break;
    cl.sync();  // partner done with my A2 before it writes the next block's halo rows
    ++round;
  }
  tc::fence_after();
  if (warp == 0) tc::tmem_free<PK::TALLOC>(tmem);
  trace(a.trace, 17);
}

template <int C, int MC, int BS>
int launch_pair(const TcArgs& a, int cap, cudaStream_t s) {
  using PK = PairCfg<C, MC, BS>;
  auto kern = unit_tc_pair_kernel<C, MC, BS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PK::SMEM);
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = PK::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[3];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  at[2].id = cudaLaunchAttributeCooperative;
  at[2].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = (debug_flags() & kDebugCooperative) ? 3 : 2;
  const int per_sm = resident_per_sm(kern, kThreads, PK::SMEM, PK::TALLOC, 2);
  const int maxcl = sm_count() * per_sm / 2;
  g_last_occ[1] = maxcl;
  {
    int api_cl = -1;  // what the occupancy API believes (diagnostics: tools/coop_probe.py)
    cudaLaunchConfig_t q = cfg;
    q.gridDim = dim3(2);
    q.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&api_cl, kern, &q) != cudaSuccess) {
      cudaGetLastError();
      api_cl = -1;
    }
    g_last_occ[7] = api_cl;
  }
  long pairs = cap < maxcl ? cap : maxcl;  // all pairs co-resident (grid barriers)
  if (pairs < 1) pairs = 1;
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cudaLaunchKernelEx(&cfg, kern, a);
  return launch_status("residual_unit_tcgen05_pair");
}

#define SBN_UNIT_TC_CONFIGS(X) \
  X(64, 32, 16)                \
  X(64, 32, 8)                 \
  X(64, 64, 16)                \
  X(128, 64, 16)               \
  X(32, 16, 16)

}  // namespace

bool unit_tc_supported(int dtype, int c, int m, const Geo& g, int halo, int pre_act) {
  if (dtype != SBN_BF16 || halo != 1 || !pre_act || g.bh != g.bw) return false;
#define X(C_, M_, B_) if (c == C_ && m == M_ && g.bh == B_ && Cfg<C_, M_, B_>::SMEM <= max_smem_optin()) return true;
  SBN_UNIT_TC_CONFIGS(X)
#undef X
  return false;
}

size_t unit_tc_packed_bytes(int c, int m, const Geo& g) {
#define X(C_, M_, B_) if (c == C_ && m == M_ && g.bh == B_) return packed_bytes<C_, M_, B_>();
  SBN_UNIT_TC_CONFIGS(X)
#undef X
  return 0;
}

static TcArgs make_args(const void* x, void* out, const void* rim, const Geo& g,
                        const sbn_unit_params* p, const int32_t* idx, const int32_t* count, int cap) {
  TcArgs a;
  a.x = (const __nv_bfloat16*)x;
  a.out = (__nv_bfloat16*)out;
  a.rim = (const __nv_bfloat16*)rim;
  a.g = g;
  a.w1 = (const __nv_bfloat16*)p->w1; a.b1 = (const __nv_bfloat16*)p->b1;
  a.w2 = (const __nv_bfloat16*)p->w2; a.b2 = (const __nv_bfloat16*)p->b2;
  a.w3 = (const __nv_bfloat16*)p->w3; a.b3 = (const __nv_bfloat16*)p->b3;
  a.s1 = (const float*)p->bn1_scale; a.t1 = (const float*)p->bn1_shift;
  a.s2 = (const float*)p->bn2_scale; a.t2 = (const float*)p->bn2_shift;
  a.s3 = (const float*)p->bn3_scale; a.t3 = (const float*)p->bn3_shift;
  a.packed = (const uint8_t*)p->tc_packed;
  a.rim_buf = nullptr;
  a.gbar = nullptr;
  a.trace = trace_buffer();
  a.mask = nullptr;
  a.idx_out = nullptr;
  a.count_out = nullptr;
  a.cst = nullptr;
  a.etag = nullptr;
  a.sw = nullptr;
  a.early_mask = 0;
  a.idx = idx; a.count = count; a.cap = cap;
  return a;
}

int unit_tc_pack(const sbn_unit_params* p, int c, int m, const Geo& g, void* img, cudaStream_t s) {
  TcArgs a = make_args(nullptr, nullptr, nullptr, g, p, nullptr, nullptr, 0);
#define X(C_, M_, B_) if (c == C_ && m == M_ && g.bh == B_) return pack<C_, M_, B_>(a, img, s);
  SBN_UNIT_TC_CONFIGS(X)
#undef X
  set_error("no tcgen05 residual-unit instantiation for c=%d m=%d block=%d", c, m, g.bh);
  return SBN_ERR_UNSUPPORTED;
}

int unit_tc_launch(const void* x, void* out, void* rim_buf, unsigned int* gbar, int c, int m,
                   const Geo& g, const sbn_unit_params* p, const void* packed, const int32_t* idx,
                   const int32_t* count, int cap, cudaStream_t s, const uint8_t* mask,
                   int32_t* idx_out, int32_t* count_out, unsigned long long* cst,
                   unsigned long long* etag, unsigned int* slotw) {
  TcArgs a = make_args(x, out, nullptr, g, p, idx, count, cap);
  a.mask = mask;
  a.early_mask = !(debug_flags() & kDebugNoEarlyMask);
  a.idx_out = idx_out;
  a.count_out = count_out;
  a.cst = cst;
  a.etag = etag;
  // the slot words live in the same caller workspace as the tagged entries: if that
  // workspace is (re)allocated, epoch and entries restart together
  a.sw = slotw;
  a.packed = (const uint8_t*)packed;
  a.rim_buf = (__nv_bfloat16*)rim_buf;
  a.gbar = gbar;
  // The CTA pair halves a block's latency chain but also halves the number of blocks in
  // flight; it wins only when the candidate list is short (about one block per pair).
  if (!(debug_flags() & kDebugNoPair) && cap <= 4 * sm_count() * 2) {
    if (c == 64 && m == 32 && g.bh == 16) return launch_pair<64, 32, 16>(a, cap, s);
    if (c == 64 && m == 64 && g.bh == 16) return launch_pair<64, 64, 16>(a, cap, s);
    if (c == 128 && m == 64 && g.bh == 16) return launch_pair<128, 64, 16>(a, cap, s);
  }
#define X(C_, M_, B_) if (c == C_ && m == M_ && g.bh == B_) return launch<C_, M_, B_>(a, cap, s);
  SBN_UNIT_TC_CONFIGS(X)
#undef X
  set_error("no tcgen05 residual-unit instantiation for c=%d m=%d block=%d", c, m, g.bh);
  return SBN_ERR_UNSUPPORTED;
}

}  // namespace sbn

extern "C" int sbn_debug_last_occupancy(int which) { return sbn::g_last_occ[which & 7]; }
