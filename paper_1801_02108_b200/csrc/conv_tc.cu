// tcgen05 / TMEM fused sparse convolution (bf16 in/out, fp32 accumulate), 3x3 stride 1.
//
// Restates reference `sparse_conv2d` (`layers.py:27-47`): per active block, the
// gathered window (`blocks.py:57-74`) is convolved with a valid 3x3 conv
// (`ops.py:130-164`, pad (0, 0) on the block) and the (BS-2)^2 output window is written
// straight into the destination (`blocks.py:125-142`).  The block stack never exists
// in HBM.
//
// Implicit GEMM over the staged window (plane layout, tc_util.cuh): output row
// q = oy*BS + ox ("full width": ox >= BS-2 columns are computed and dropped), and tap
// (ky, kx) is the window viewed from row ky*BS + kx, so D[q, :] += A[q + shift, :] . W_tap.
//
// Warp roles (persistent CTA, 288 threads):
//   warp 8, lane 0   producer: streams the 9 per-tap weight images (COUT x CIN bf16,
//                    pre-packed) through a kStages-deep smem ring with cp.async.bulk,
//                    running ahead into the next block while the current one drains;
//   thread 0         MMA issuer: per tap, NT M-tiles x CIN/16 UMMAs (M=128, N=COUT);
//   warps 0-7        stage the window (zero-filled halo) and run the TMEM epilogue
//                    (+bias, bf16, clipped store).
#include "common.cuh"
#include "tc_util.cuh"
#include "tma_util.cuh"

#include <cstring>

namespace sbn {
namespace {

constexpr int kWorkers = 256;
constexpr int kThreads = kWorkers + 32;

template <int CIN, int COUT, int BS>
struct ConvCfg {
  static_assert(CIN % 16 == 0 && COUT % 16 == 0 && COUT <= 256, "channel constraints");
  static constexpr int NQ = (BS - 2) * BS;
  static constexpr int NT = (NQ + 127) / 128;
  static_assert(NT * COUT <= 512, "TMEM budget");
  static constexpr int R = (((NT * 128 + 2 * BS + 2) > BS * BS ? (NT * 128 + 2 * BS + 2) : BS * BS) + 7) / 8 * 8;
  static constexpr int PA = R * 16 + 16;          // window plane stride (padded)
  static constexpr int PW = COUT * 16;            // weight plane stride
  static constexpr int TAP = (CIN / 8) * PW;      // bytes per tap image
  static constexpr int al(int v) { return (v + 1023) / 1024 * 1024; }
  static constexpr int SZ_A = al((CIN / 8) * PA);
  static constexpr int STAGES = (SZ_A + 3 * TAP + COUT * 4 <= 220 * 1024) ? 3 : 2;
  static constexpr int OFF_W = SZ_A;
  static constexpr int OFF_BIAS = OFF_W + STAGES * TAP;
  static constexpr int SMEM = OFF_BIAS + COUT * 4;
  static constexpr int TCOLS = NT * COUT;
  static constexpr int TALLOC = TCOLS <= 32 ? 32 : TCOLS <= 64 ? 64 : TCOLS <= 128 ? 128 : TCOLS <= 256 ? 256 : 512;
};

struct ConvArgs {
  const __nv_bfloat16* x;
  __nv_bfloat16* out;
  Geo g;
  const uint8_t* wpk;   // 9 tap images
  const __nv_bfloat16* bias;  // nullable
  const int32_t* idx;
  const int32_t* count;
  int cap;
  unsigned long long* trace;  // diagnostics: per-CTA MMA-issuer wait totals (sbn_debug_set_trace)
  // mask-fused front end (double-buffered kernel only): when `mask` is set every CTA
  // reduces its share of the mask itself (conv_mask_local) and then either convolves its
  // own active blocks (gidx == nullptr), or publishes them into one global list
  // (conv_mask_global) that every CTA strides through as in list mode
  const uint8_t* mask;
  unsigned* sw;    // global list: [0] launch epoch, [4 + 4 * (tag & 1) + {0 claimed, 1 done}]
  int32_t* gidx;   // global list rows (cap x 3)
  int early_trigger;  // double-buffered kernel: griddepcontrol.launch_dependents after the prologue
};

// Mask reduction fused in front of the conv (reference `tiling.py:138-160`, MAX pool),
// without any grid-wide step: CTA c owns candidates c, c + G, c + 2G, ... (round-robin, so
// active regions spread evenly), tests each one's clipped input window (one warp per
// candidate, any-pixel by warp vote), and lists its own active blocks in shared memory.
// The conv then walks that local list.  Block order does not matter (disjoint outputs).
constexpr int kMaxLocal = 384;  // candidates per CTA (host falls back to reduce_mask above)

template <int NTHREADS, int BS>
__device__ int conv_mask_local(const ConvArgs& a, int32_t* s_idx) {
  const Geo& g = a.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = NTHREADS / 32, AREA = BS * BS, PL = (AREA + 31) / 32;  // pixels per lane
  __shared__ uint8_t s_flag[kMaxLocal];
  __shared__ int s_n;
  const int T = g.n * g.gy * g.gx, G = gridDim.x, gyx = g.gy * g.gx;
  const int nc = T > (int)blockIdx.x ? min((T - (int)blockIdx.x + G - 1) / G, kMaxLocal) : 0;
  for (int j = warp; j < nc; j += NW) {
    const int cand = (int)blockIdx.x + j * G;
    const int fr = cand / gyx, rr = cand - fr * gyx;
    const int y0 = g.oy + (rr / g.gx) * g.sy, x0 = g.ox + (rr % g.gx) * g.sx;
    uint32_t v[PL];  // predicated straight-line loads: all of the window's bytes in flight
#pragma unroll
    for (int u = 0; u < PL; ++u) {
      const int p = lane + 32 * u;
      const int y = y0 + p / BS, xx = x0 + p % BS;
      const bool ok = p < AREA && y >= 0 && y < g.h && xx >= 0 && xx < g.w;
      v[u] = tc::ld_u8_pred(a.mask + ((size_t)fr * g.h + (ok ? y : 0)) * g.w + (ok ? xx : 0), ok);
    }
    bool any = false;
#pragma unroll
    for (int u = 0; u < PL; ++u) any |= v[u] != 0;
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) s_flag[j] = any;
  }
  __syncthreads();
  if (warp == 0) {  // compact in candidate order
    int pos = 0;
    for (int c0 = 0; c0 < nc; c0 += 32) {
      const bool on = c0 + lane < nc && s_flag[c0 + lane];
      const unsigned bal = __ballot_sync(0xffffffffu, on);
      if (on) {
        const int q = pos + __popc(bal & ((1u << lane) - 1u));
        const int cand = (int)blockIdx.x + (c0 + lane) * G;
        const int fr = cand / gyx, rr = cand - fr * gyx;
        s_idx[3 * q] = fr;
        s_idx[3 * q + 1] = rr / g.gx;
        s_idx[3 * q + 2] = rr % g.gx;
      }
      pos += __popc(bal);
    }
    if (lane == 0) s_n = pos;
  }
  __syncthreads();
  return s_n;
}

// Global list from the per-CTA lists (few candidates per CTA, where per-CTA lists balance
// badly on structured masks): one atomic per CTA claims list slots, the rows are stored,
// and every CTA then waits until all G CTAs have published (the grid is at most one CTA
// per SM, so it is co-resident) and strides through the list like the ordered list mode —
// one launch instead of reduce_mask + conv, in an order that does not matter (disjoint
// outputs).  The counters of launch `tag` live in ring slot tag & 1; the last CTA to
// publish (every CTA has read the epoch by then) zeroes the other slot and bumps the epoch.
template <int NTHREADS, int BS>
__device__ int conv_mask_global(const ConvArgs& a, int32_t* s_idx) {
  __shared__ unsigned s_tag;
  __shared__ int s_base, s_B;
  if (threadIdx.x == 0) s_tag = *reinterpret_cast<volatile unsigned*>(a.sw) + 1u;
  const int nl = conv_mask_local<NTHREADS, BS>(a, s_idx);  // ends with __syncthreads
  const unsigned tag = s_tag;
  unsigned* ring = a.sw + 4 + 4 * (tag & 1u);
  if (threadIdx.x == 0) s_base = nl ? (int)atomicAdd(ring, (unsigned)nl) : 0;
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * nl; i += NTHREADS) a.gidx[3 * s_base + i] = s_idx[i];
  __syncthreads();
  if (threadIdx.x == 0) {
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
    s_B = (int)d;
  }
  __syncthreads();
  return s_B;
}

template <int CIN, int COUT, int BS>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(ConvArgs a) {
  using K = ConvCfg<CIN, COUT, BS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[K::STAGES], empty[K::STAGES], accb;
  __shared__ uint32_t tslot;
  uint8_t* A = smem;
  uint8_t* Wst = smem + K::OFF_W;
  float* bias = reinterpret_cast<float*>(smem + K::OFF_BIAS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Geo& g = a.g;

  if (tid == 0) {
    for (int s = 0; s < K::STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&accb, 1);
    tc::mbar_fence_init();
  }
  for (int i = tid; i < COUT; i += kThreads) bias[i] = a.bias ? __bfloat162float(a.bias[i]) : 0.f;
  if (warp == 0) tc::tmem_alloc<K::TALLOC>(&tslot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  tc::pdl_wait();
  const int B = ld_count(a.count, a.cap);

  if (warp == 8) {
    // ---------------- producer: weight taps through the ring
    if (lane == 0) {
      int it = 0;
      for (int blk = blockIdx.x; blk < B; blk += gridDim.x)
        for (int tap = 0; tap < 9; ++tap, ++it) {
          const int s = it % K::STAGES;
          tc::mbar_wait(&empty[s], ((it / K::STAGES) & 1) ^ 1);
          tc::mbar_expect_tx(&full[s], K::TAP);
          tc::bulk_g2s(Wst + s * K::TAP, a.wpk + (size_t)tap * K::TAP, K::TAP, &full[s]);
        }
    }
    __syncwarp();
  } else {
    // ---------------- workers (warps 0-7) + MMA issuer (thread 0)
    const int q = warp & 3, tpar = warp >> 2;
    int it = 0;
    uint32_t accphase = 0;
    for (int blk = blockIdx.x; blk < B; blk += gridDim.x) {
      const int n = __ldg(a.idx + 3 * blk), by = __ldg(a.idx + 3 * blk + 1), bx = __ldg(a.idx + 3 * blk + 2);
      const int ys = g.oy + by * g.sy, xs = g.ox + bx * g.sx;
      // stage the window (zero-filled halo): all loads in flight, then plane stores
      constexpr int TOT = BS * BS * (CIN / 8);
      constexpr int ITEMS = (TOT + kWorkers - 1) / kWorkers;
      constexpr int CH = ITEMS > 16 ? 16 : ITEMS;
#pragma unroll 1
      for (int base = 0; base < ITEMS; base += CH) {
        uint4 raw[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int i = tid + (base + j) * kWorkers;
          const int p = i / (CIN / 8), k = i % (CIN / 8);
          const int y = ys + p / BS, xx = xs + p % BS;
          raw[j] = make_uint4(0, 0, 0, 0);
          if (i < TOT && y >= 0 && y < g.h && xx >= 0 && xx < g.w)
            raw[j] = __ldg(reinterpret_cast<const uint4*>(a.x) + (((size_t)n * g.h + y) * g.w + xx) * (CIN / 8) + k);
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int i = tid + (base + j) * kWorkers;
          if (i < TOT) {
            const int p = i / (CIN / 8), k = i % (CIN / 8);
            *reinterpret_cast<uint4*>(A + k * K::PA + p * 16) = raw[j];
          }
        }
      }
      tc::fence_async_smem();
      tc::named_bar<1, kWorkers>();

      if (tid == 0) {
        tc::fence_after();
        constexpr uint32_t idesc = tc::idesc_bf16_f32(128, COUT);
        for (int tap = 0; tap < 9; ++tap, ++it) {
          const int s = it % K::STAGES;
          tc::mbar_wait(&full[s], (it / K::STAGES) & 1);
          tc::fence_after();
          const int shift = (tap / 3) * BS + (tap % 3);
          // one descriptor per operand and tap, immediate offsets per MMA (tc::desc_add)
          const uint64_t ad = tc::desc_kmajor_noswz(tc::smem_u32(A) + shift * 16, K::PA, 128);
          const uint64_t wd = tc::desc_kmajor_noswz(tc::smem_u32(Wst + s * K::TAP), K::PW, 128);
#pragma unroll
          for (int t = 0; t < K::NT; ++t)
#pragma unroll
            for (int k = 0; k < CIN / 16; ++k)
              tc::mma_bf16(tmem + t * COUT, tc::desc_add(ad, 2 * k * K::PA + t * 128 * 16),
                           tc::desc_add(wd, 2 * k * K::PW), idesc, (tap | k) > 0);
          tc::mma_commit(&empty[s]);  // frees the weight stage once these MMAs are done
        }
        tc::mma_commit(&accb);
      } else {
        it += 9;
      }
      tc::mbar_wait(&accb, accphase);
      accphase ^= 1;
      tc::fence_after();

      // epilogue: TMEM -> +bias -> bf16 -> clipped output window
      for (int t = tpar; t < K::NT; t += 2) {
        const int r = t * 128 + q * 32 + lane;
        const int oy = r / BS, ox = r % BS;
        const int Y = by * g.obh + oy, X = bx * g.obw + ox;
        const bool store = oy < g.obh && ox < g.obw && Y < g.oh && X < g.ow;
        uint4* op = reinterpret_cast<uint4*>(a.out) +
                    (((size_t)n * g.oh + (store ? Y : 0)) * g.ow + (store ? X : 0)) * (COUT / 8);
#pragma unroll 4
        for (int c0 = 0; c0 < COUT; c0 += 16) {
          float v[16];
          tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + t * COUT + c0, v);
          if (store) {
            uint32_t o[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = tc::pack_bf16(v[2 * e] + bias[c0 + 2 * e], v[2 * e + 1] + bias[c0 + 2 * e + 1]);
            op[c0 / 8] = make_uint4(o[0], o[1], o[2], o[3]);
            op[c0 / 8 + 1] = make_uint4(o[4], o[5], o[6], o[7]);
          }
        }
      }
      tc::fence_before();
      tc::named_bar<1, kWorkers>();
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_free<K::TALLOC>(tmem);
}

// HWIO (3, 3, CIN, COUT) -> 9 tap images, each CIN/8 planes x COUT rows x 16 B (single-CTA
// kernels), followed by the CTA-pair copy: per tap two halves (output channels
// [0, COUT/2) and [COUT/2, COUT)), each CIN/8 planes x COUT/2 rows x 16 B, so each CTA of a
// pair fetches its half with one contiguous bulk copy.
template <int CIN, int COUT>
__global__ void conv_tc_pack_kernel(const __nv_bfloat16* __restrict__ w, uint8_t* __restrict__ img) {
  const int total = 9 * CIN * COUT;
  constexpr size_t TAP = (size_t)(CIN / 8) * COUT * 16;
  constexpr int NH = COUT / 2;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int tap = i / (CIN * COUT), r = i % (CIN * COUT), ci = r / COUT, co = r % COUT;
    *reinterpret_cast<__nv_bfloat16*>(img + (size_t)tap * TAP + (ci / 8) * COUT * 16 + co * 16 + (ci % 8) * 2) = w[i];
    *reinterpret_cast<__nv_bfloat16*>(img + 9 * TAP + (size_t)tap * TAP + (size_t)(co / NH) * (TAP / 2) +
                                      (ci / 8) * NH * 16 + (co % NH) * 16 + (ci % 8) * 2) = w[i];
  }
}

template <int CIN, int COUT, int BS>
int launch_conv(const ConvArgs& a, int cap, cudaStream_t s) {
  using K = ConvCfg<CIN, COUT, BS>;
  auto kern = conv_tc_kernel<CIN, COUT, BS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(persistent_grid(cap, 1));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = K::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a);
  return launch_status("sparse_conv_tcgen05");
}


// ---------------------------------------------------------------------------------------
// Double-buffered variant: two window buffers and two TMEM accumulators so that, per CTA,
// the window load of block k+1 and the epilogue of block k-1 overlap the MMAs of block k.
// Roles (320 threads): warps 0-7 workers (stage windows, drain TMEM), warp 8 weight
// producer, warp 9 MMA issuer.  Handshakes are mbarriers:
//   win_full[b]  workers -> MMA   (256 arrivals: window b staged)
//   win_empty[b] MMA -> workers   (tcgen05.commit: MMAs reading window b done)
//   acc_full[b]  MMA -> workers   (tcgen05.commit: accumulator b complete)
//   acc_empty[b] workers -> MMA   (256 arrivals: accumulator b drained)
constexpr int kDbThreads = kWorkers + 64;

template <int CIN, int COUT, int BS>
struct DbCfg {
  using K = ConvCfg<CIN, COUT, BS>;
  static constexpr int al(int v) { return (v + 1023) / 1024 * 1024; }
  static constexpr int SZ_A = K::SZ_A;
  static constexpr int STAGES = (2 * SZ_A + 3 * K::TAP + COUT * 4 <= 222 * 1024) ? 3 : 2;
  static constexpr int OFF_W = 2 * SZ_A;
  static constexpr int OFF_BIAS = OFF_W + STAGES * K::TAP;
  static constexpr int SMEM = OFF_BIAS + COUT * 4;
  static constexpr int ACC = K::NT * COUT;  // TMEM columns per accumulator
  // small blocks share one M-tile: BPT windows stacked at BS*BS-row pitch (8x8 blocks: 2
  // per tile, 96 of 128 rows useful instead of 48).  A block's shifted views reach at most
  // 2*BS+2 rows past its own outputs, i.e. only into its neighbour's garbage columns.
  static constexpr int BPT = (K::NT == 1 && 2 * BS * BS <= 128) ? 128 / (BS * BS) : 1;
  static constexpr int TALLOC = 2 * ACC <= 32 ? 32 : 2 * ACC <= 64 ? 64 : 2 * ACC <= 128 ? 128 : 2 * ACC <= 256 ? 256 : 512;
  static_assert(2 * ACC <= 512, "two accumulators must fit TMEM");
};

template <int CIN, int COUT, int BS>
__global__ void __launch_bounds__(kDbThreads, 1) conv_tc_db_kernel(ConvArgs a) {
  using K = ConvCfg<CIN, COUT, BS>;
  using D = DbCfg<CIN, COUT, BS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[D::STAGES], empty[D::STAGES];
  __shared__ uint64_t win_full[2], win_empty[2], acc_full[2], acc_empty[2];
  __shared__ uint32_t tslot;
  uint8_t* Wst = smem + D::OFF_W;
  float* bias = reinterpret_cast<float*>(smem + D::OFF_BIAS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Geo& g = a.g;

  if (tid == 0) {
    for (int s = 0; s < D::STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&win_full[b], kWorkers);
      tc::mbar_init(&win_empty[b], 1);
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], kWorkers);
    }
    tc::mbar_fence_init();
  }
  for (int i = tid; i < COUT; i += kDbThreads) bias[i] = a.bias ? __bfloat162float(a.bias[i]) : 0.f;
  if (warp == 0) tc::tmem_alloc<D::TALLOC>(&tslot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  if (a.early_trigger) tc::pdl_trigger();  // the next launch may start its prologue
  tc::pdl_wait();
  __shared__ int32_t s_idx[3 * kMaxLocal];  // mask-fused mode: this CTA's own block list
  const bool global = a.mask != nullptr && a.gidx != nullptr;  // mask-fused, one global list
  const bool local = a.mask != nullptr && !global;             // mask-fused, per-CTA lists
  const int B = global ? conv_mask_global<kDbThreads, BS>(a, s_idx)
                       : local ? conv_mask_local<kDbThreads, BS>(a, s_idx) : ld_count(a.count, a.cap);
  const int32_t* lidx = local ? s_idx : global ? a.gidx : a.idx;  // (n, by, bx) rows
  const int jfirst = local ? 0 : (int)blockIdx.x, jstep = local ? 1 : (int)gridDim.x;
  // jobs: BPT consecutive blocks of the list.  Tail split (list mode, two M-tiles per
  // block): when B = q*G + R with 0 < 2R <= G, the last R blocks become 2R half-block jobs
  // (one M-tile each), so no CTA runs q+1 whole blocks while most run q (config 3 at 10 %,
  // 16x16: 304 blocks on 148 CTAs = 2.05 rounds -> 2.5 instead of 3 block-times).
  int NJ = (B + D::BPT - 1) / D::BPT, whole = NJ;
  if (K::NT == 2 && D::BPT == 1 && !local) {
    const int R = B % (int)gridDim.x;
    if (R > 0 && 2 * R <= (int)gridDim.x) {
      whole = B - R;
      NJ = whole + 2 * R;
    }
  }
  // first block of a job and the M-tiles it computes (bit t: tile t)
  auto job_blk = [&](int job) { return job < whole ? job * D::BPT : whole + ((job - whole) >> 1); };
  auto job_tiles = [&](int job) { return job < whole ? (1 << K::NT) - 1 : 1 << ((job - whole) & 1); };

  if (warp == 8) {
    // ---------------- producer: weight taps through the ring
    if (lane == 0) {
      int it = 0;
      for (int job = jfirst; job < NJ; job += jstep)
        for (int tap = 0; tap < 9; ++tap, ++it) {
          const int s = it % D::STAGES;
          tc::mbar_wait(&empty[s], ((it / D::STAGES) & 1) ^ 1);
          tc::mbar_expect_tx(&full[s], K::TAP);
          tc::bulk_g2s(Wst + s * K::TAP, a.wpk + (size_t)tap * K::TAP, K::TAP, &full[s]);
        }
    }
    __syncwarp();
  } else if (warp == 9) {
    // ---------------- MMA issuer
    if (lane == 0) {
      int it = 0, k = 0;
      constexpr uint32_t idesc = tc::idesc_bf16_f32(128, COUT);
      unsigned long long t_win = 0, t_acc = 0, t_w = 0, t0 = clock64();
      for (int job = jfirst; job < NJ; job += jstep, ++k) {
        const int b = k & 1;
        const uint32_t use = (uint32_t)(k >> 1);
        const unsigned long long c0 = clock64();
        tc::mbar_wait(&win_full[b], use & 1);
        const unsigned long long c1 = clock64();
        tc::mbar_wait(&acc_empty[b], (use & 1) ^ 1);
        t_win += c1 - c0;
        t_acc += clock64() - c1;
        tc::fence_after();
        const uint8_t* A = smem + b * D::SZ_A;
        const uint32_t acc = tmem + b * D::ACC;
        for (int tap = 0; tap < 9; ++tap, ++it) {
          const int s = it % D::STAGES;
          const unsigned long long c3 = clock64();
          tc::mbar_wait(&full[s], (it / D::STAGES) & 1);
          t_w += clock64() - c3;
          tc::fence_after();
          const int shift = (tap / 3) * BS + (tap % 3);
          // one descriptor per operand and tap, immediate offsets per MMA (tc::desc_add)
          const uint64_t ad = tc::desc_kmajor_noswz(tc::smem_u32(A) + shift * 16, K::PA, 128);
          const uint64_t wd = tc::desc_kmajor_noswz(tc::smem_u32(Wst + s * K::TAP), K::PW, 128);
          const int tm = job_tiles(job);
#pragma unroll
          for (int t = 0; t < K::NT; ++t)
#pragma unroll
            for (int kk = 0; kk < CIN / 16; ++kk)
              if (tm >> t & 1)
              tc::mma_bf16(acc + t * COUT, tc::desc_add(ad, 2 * kk * K::PA + t * 128 * 16),
                           tc::desc_add(wd, 2 * kk * K::PW), idesc, (tap | kk) > 0);
          tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&win_empty[b]);
        tc::mma_commit(&acc_full[b]);
      }
      if (a.trace) {
        unsigned long long* tb = a.trace + blockIdx.x * 8;
        tb[0] = clock64() - t0;
        tb[1] = t_win;
        tb[2] = t_acc;
        tb[3] = t_w;
        tb[4] = k;
      }
    }
    __syncwarp();
  } else {
    // ---------------- workers: stage window k, drain accumulator k-1
    const int q = warp & 3, tpar = warp >> 2;
    int pjob = 0;  // previous job (for its epilogue)
    int k = 0;
    auto epilogue = [&](int kk, int job) {
      const int b = kk & 1;
      tc::mbar_wait(&acc_full[b], (kk >> 1) & 1);
      tc::fence_after();
      const uint32_t acc = tmem + b * D::ACC;
      const int tm = job_tiles(job);
      for (int t = tpar; t < K::NT; t += 2) {
        if (!(tm >> t & 1)) continue;  // half-block job: the other M-tile is another CTA's
        int r = t * 128 + q * 32 + lane;
        int blk = job_blk(job);
        if (D::BPT > 1) {  // packed tile: this row belongs to block r / (BS*BS) of the job
          blk = job * D::BPT + r / (BS * BS);
          r %= BS * BS;
        }
        int n = 0, by = 0, bx = 0;
        if (blk < B) {
          n = lidx[3 * blk];
          by = lidx[3 * blk + 1];
          bx = lidx[3 * blk + 2];
        }
        const int oy = r / BS, ox = r % BS;
        const int Y = by * g.obh + oy, X = bx * g.obw + ox;
        const bool store = blk < B && oy < g.obh && ox < g.obw && Y < g.oh && X < g.ow;
        uint4* op = reinterpret_cast<uint4*>(a.out) +
                    (((size_t)n * g.oh + (store ? Y : 0)) * g.ow + (store ? X : 0)) * (COUT / 8);
#pragma unroll 4
        for (int c0 = 0; c0 < COUT; c0 += 16) {
          float v[16];
          tc::tmem_ld16(acc + ((uint32_t)(q * 32) << 16) + t * COUT + c0, v);
          if (store) {
            uint32_t o[8];
#pragma unroll
            for (int e = 0; e < 8; ++e)
              o[e] = tc::pack_bf16(v[2 * e] + bias[c0 + 2 * e], v[2 * e + 1] + bias[c0 + 2 * e + 1]);
            op[c0 / 8] = make_uint4(o[0], o[1], o[2], o[3]);
            op[c0 / 8 + 1] = make_uint4(o[4], o[5], o[6], o[7]);
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&acc_empty[b]);
    };
    for (int job = jfirst; job < NJ; job += jstep, ++k) {
      const int b = k & 1;
      tc::mbar_wait(&win_empty[b], ((k >> 1) & 1) ^ 1);
      uint8_t* A = smem + b * D::SZ_A;
      constexpr int PER = BS * BS * (CIN / 8);  // items per block window
      constexpr int TOT = D::BPT * PER;
      constexpr int ITEMS = (TOT + kWorkers - 1) / kWorkers;
      constexpr int CH = ITEMS > 16 ? 16 : ITEMS;
      // the job's block origins, loaded once (L2-coherent: the list may come from this launch)
      int jn[D::BPT], jy[D::BPT], jx[D::BPT];
#pragma unroll
      for (int jb = 0; jb < D::BPT; ++jb) {
        const int blk = job_blk(job) + jb;
        jn[jb] = 0, jy[jb] = -(1 << 20), jx[jb] = 0;  // missing block: every pixel out of image
        if (blk < B) {
          jn[jb] = lidx[3 * blk];
          jy[jb] = g.oy + lidx[3 * blk + 1] * g.sy;
          jx[jb] = g.ox + lidx[3 * blk + 2] * g.sx;
        }
      }
#pragma unroll 1
      for (int base = 0; base < ITEMS; base += CH) {
        uint4 raw[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int i = tid + (base + j) * kWorkers;
          const int jb = D::BPT > 1 ? min(i / PER, D::BPT - 1) : 0, ii = i - jb * PER;
          const int blk = job_blk(job) + jb;
          const int p = ii / (CIN / 8), kc = ii % (CIN / 8);
          const int n = jn[jb], ys = jy[jb], xs = jx[jb];
          const int y = ys + p / BS, xx = xs + p % BS;
          const bool ok = i < TOT && blk < B && (unsigned)y < (unsigned)g.h && (unsigned)xx < (unsigned)g.w;
          raw[j] = tc::ld_v4_pred(reinterpret_cast<const uint4*>(a.x) +
                                      (((size_t)n * g.h + (ok ? y : 0)) * g.w + (ok ? xx : 0)) * (CIN / 8) + kc,
                                  ok);
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int i = tid + (base + j) * kWorkers;
          if (i < TOT) {
            const int jb = i / PER, ii = i - jb * PER;
            const int p = jb * BS * BS + ii / (CIN / 8), kc = ii % (CIN / 8);
            *reinterpret_cast<uint4*>(A + kc * K::PA + p * 16) = raw[j];
          }
        }
      }
      tc::fence_async_smem();
      tc::mbar_arrive(&win_full[b]);
      if (k > 0) epilogue(k - 1, pjob);
      pjob = job;
    }
    if (k > 0) epilogue(k - 1, pjob);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_free<D::TALLOC>(tmem);
}

template <int CIN, int COUT, int BS>
int launch_conv_db(const ConvArgs& a_in, int cap, cudaStream_t s) {
  using D = DbCfg<CIN, COUT, BS>;
  ConvArgs a = a_in;
  a.early_trigger = !(debug_flags() & kDebugNoMaskPdl);
  auto kern = conv_tc_db_kernel<CIN, COUT, BS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, D::SMEM);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(persistent_grid((cap + D::BPT - 1) / D::BPT, 1));
  cfg.blockDim = dim3(kDbThreads);
  cfg.dynamicSmemBytes = D::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a);
  return launch_status("sparse_conv_tcgen05_db");
}

// ---------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2) for 16x16 blocks.  The single-CTA kernels issue
// 128 x COUT x 16 UMMAs whose A tile (4 KB) and B tile (COUT*32 B) both stream from shared
// memory (~120 B/clk at COUT = 128 against ~128 B/clk of bandwidth), and their 8 worker warps
// both stage windows and drain accumulators.  Here the block's two M-tiles (output rows
// q in [0, 128) and [128, 224)) are ONE M = 256 UMMA issued by rank 0 of a 2-CTA cluster:
//   * rank r holds window rows [8 r, 8 r + 11) — one 5-D TMA box (8 ch, 16 x, 11 y, C/8
//     planes, 1 frame) that lands directly in the K-major plane layout (plane stride
//     11*16*16 B), zero-filled outside the image (the gather's halo semantics);
//   * rank r holds output channels [r COUT/2, (r+1) COUT/2) of every tap (B is split along
//     N in cta_group::2), one contiguous bulk copy per tap from the pair copy of the packed
//     weights; per SM an MMA reads the A tile plus half of B;
//   * the worker warps only drain TMEM (+bias -> bf16 -> clipped store).
// Handshakes (rank 0 owns what its MMA issuer waits on):
//   full[s]      both weight halves of stage s landed (rank 1's TMA completes on it)  rank 0
//   empty[s]     MMAs reading stage s done (multicast commit)               both
//   win_full[b]  both window boxes landed (rank 1's TMA completes on it)    rank 0
//   win_empty[b] MMAs reading window b done (multicast commit)              both
//   acc_full[b]  accumulator b complete (multicast commit)                  both
//   acc_empty[b] 2 x 256 worker arrivals (rank 1's arrive remotely)          rank 0
constexpr int kPairThreads = kWorkers + 96;  // + weight loader, MMA / forwarder, window loader

template <int CIN, int COUT, int BS>
struct PairConvCfg {
  static_assert(BS == 16 && COUT % 32 == 0, "pair conv: two M-tiles per block, N/2 a multiple of 16");
  static constexpr int WROWS = 11;               // window rows per rank (128 + 2*BS + 2 pixels)
  static constexpr int RA = WROWS * BS;           // local A rows
  static constexpr int PA = RA * 16;              // plane stride = TMA box plane
  static constexpr int ABOX = (CIN / 8) * PA;     // bytes of one window box
  static constexpr int SZ_A = (ABOX + 1023) / 1024 * 1024;
  static constexpr int NH = COUT / 2;            // output channels (B rows) per CTA
  static constexpr int PWH = NH * 16;            // half-plane stride
  static constexpr int TAPH = (CIN / 8) * PWH;   // bytes of one tap's half
  static constexpr int TAP = (CIN / 8) * COUT * 16;  // one tap of the packed image
  static constexpr int STAGES = (2 * SZ_A + 8 * TAPH + COUT * 4 <= 222 * 1024) ? 8
                                : (2 * SZ_A + 6 * TAPH + COUT * 4 <= 222 * 1024) ? 6
                                : (2 * SZ_A + 3 * TAPH + COUT * 4 <= 222 * 1024) ? 3 : 2;
  static constexpr int WBOXR = TAPH / 128;  // weight half as a TMA box of 128-byte rows
  static constexpr int OFF_W = 2 * SZ_A;
  static constexpr int OFF_BIAS = OFF_W + STAGES * TAPH;
  static constexpr int SMEM = OFF_BIAS + COUT * 4;
  static constexpr int ACC = COUT;  // one 128-row tile per CTA
  static constexpr int TALLOC = 2 * ACC <= 32 ? 32 : 2 * ACC <= 64 ? 64 : 2 * ACC <= 128 ? 128 : 2 * ACC <= 256 ? 256 : 512;
};

struct __align__(64) PairConvArgs {
  CUtensorMap tmap;  // x as (8 ch, W, H, C/8 planes, N), box (8, 16, 11, C/8, 1)
  CUtensorMap wmap;  // pair copy of the packed weights as 128-byte rows, box = one tap half
  ConvArgs c;
  unsigned long long* trace;  // diagnostics: per-CTA issuer wait totals (sbn_debug_set_trace)
  int early_trigger;          // resident pair kernel: griddepcontrol.launch_dependents after the prologue
};

template <int CIN, int COUT, int BS>
__global__ void __launch_bounds__(kPairThreads, 1) conv_tc_pair_kernel(const __grid_constant__ PairConvArgs pa) {
  using P = PairConvCfg<CIN, COUT, BS>;
  const ConvArgs& a = pa.c;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[P::STAGES], empty[P::STAGES];
  __shared__ uint64_t win_full[2], win_empty[2], acc_full[2], acc_empty[2];
  __shared__ uint32_t tslot;
  uint8_t* Wst = smem + P::OFF_W;
  float* bias = reinterpret_cast<float*>(smem + P::OFF_BIAS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = tc::cluster_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const Geo& g = a.g;

  if (tid == 0) {
    for (int s = 0; s < P::STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&win_full[b], 1);
      tc::mbar_init(&win_empty[b], 1);
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], 2 * kWorkers);
    }
    tc::mbar_fence_init();
  }
  if (tid == 10 * 32) asm volatile("prefetch.tensormap [%0];" ::"l"(&pa.tmap) : "memory");
  if (tid == 8 * 32) asm volatile("prefetch.tensormap [%0];" ::"l"(&pa.wmap) : "memory");
  for (int i = tid; i < COUT; i += kPairThreads) bias[i] = a.bias ? __bfloat162float(a.bias[i]) : 0.f;
  if (warp == 0) tc::tmem_alloc_cg2<P::TALLOC>(&tslot);
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();  // both CTAs' barriers exist before any remote arrive / multicast commit
  tc::fence_after();
  const uint32_t tmem = tslot;
  tc::pdl_wait();
  const int B = ld_count(a.count, a.cap);

  if (warp == 8) {
    // ---------------- weight loader: my half (output channels) of every tap
    if (lane == 0) {
      int it = 0;
      for (int blk = pair; blk < B; blk += npairs)
        for (int tap = 0; tap < 9; ++tap, ++it) {
          const int s = it % P::STAGES;
          tc::mbar_wait(&empty[s], ((it / P::STAGES) & 1) ^ 1);
          const int row = (2 * tap + (int)rank) * P::WBOXR;  // my half of this tap
          if (rank == 0) {
            tc::mbar_expect_tx(&full[s], 2 * P::TAPH);
            tma_2d(Wst + s * P::TAPH, &pa.wmap, 0, row, &full[s]);
          } else {
            tma_2d_cg2(Wst + s * P::TAPH, &pa.wmap, 0, row, &full[s], 0);
          }
        }
    }
    __syncwarp();
  } else if (warp == 10) {
    // ---------------- window loader: my 11 window rows of every block, one TMA box
    if (lane == 0) {
      int k = 0;
      for (int blk = pair; blk < B; blk += npairs, ++k) {
        const int b = k & 1;
        const int n = __ldg(a.idx + 3 * blk), by = __ldg(a.idx + 3 * blk + 1), bx = __ldg(a.idx + 3 * blk + 2);
        const int ys = g.oy + by * g.sy + (int)rank * (P::WROWS - 3), xs = g.ox + bx * g.sx;
        tc::mbar_wait(&win_empty[b], ((k >> 1) & 1) ^ 1);
        if (rank == 0) {
          tc::mbar_expect_tx(&win_full[b], 2 * P::ABOX);
          tma_5d(smem + b * P::SZ_A, &pa.tmap, 0, xs, ys, 0, n, &win_full[b]);
        } else {
          tma_5d_cg2(smem + b * P::SZ_A, &pa.tmap, 0, xs, ys, 0, n, &win_full[b], 0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 9) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (rank 0): M = 256 over the pair
      int it = 0, k = 0;
      constexpr uint32_t idesc = tc::idesc_bf16_f32(256, COUT);
      unsigned long long t_win = 0, t_acc = 0, t_w = 0, t_iss = 0, t0 = clock64();
      for (int blk = pair; blk < B; blk += npairs, ++k) {
        const int b = k & 1;
        const uint32_t use = (uint32_t)(k >> 1);
        unsigned long long c0 = clock64();
        tc::mbar_wait(&win_full[b], use & 1);
        unsigned long long c1 = clock64();
        tc::mbar_wait(&acc_empty[b], (use & 1) ^ 1);
        unsigned long long c2 = clock64();
        t_win += c1 - c0;
        t_acc += c2 - c1;
        tc::fence_after();
        const uint8_t* A = smem + b * P::SZ_A;
        const uint32_t acc = tmem + b * P::ACC;
        for (int tap = 0; tap < 9; ++tap, ++it) {
          const int s = it % P::STAGES;
          unsigned long long c3 = clock64();
          tc::mbar_wait(&full[s], (it / P::STAGES) & 1);
          unsigned long long c4 = clock64();
          t_w += c4 - c3;
          tc::fence_after();
          const int shift = (tap / 3) * BS + (tap % 3);
          const uint32_t wbase = tc::smem_u32(Wst + s * P::TAPH);
#pragma unroll
          for (int kk = 0; kk < CIN / 16; ++kk)
            tc::mma_bf16_cg2(acc, tc::desc_kmajor_noswz(tc::smem_u32(A + 2 * kk * P::PA + shift * 16), P::PA, 128),
                             tc::desc_kmajor_noswz(wbase + 2 * kk * P::PWH, P::PWH, 128), idesc, (tap | kk) > 0);
          tc::mma_commit_mc(&empty[s], 3);
        }
        tc::mma_commit_mc(&win_empty[b], 3);
        tc::mma_commit_mc(&acc_full[b], 3);
      }
      if (pa.trace) {
        unsigned long long* tb = pa.trace + blockIdx.x * 8;
        tb[0] = clock64() - t0;
        tb[1] = t_win;
        tb[2] = t_acc;
        tb[3] = t_w;
        tb[4] = k;
      }
      (void)t_iss;
    }
    __syncwarp();
  } else {
    // ---------------- workers: drain my tile of each accumulator
    const int q = warp & 3, tpar = warp >> 2;
    int k = 0;
    for (int blk = pair; blk < B; blk += npairs, ++k) {
      const int n = __ldg(a.idx + 3 * blk), by = __ldg(a.idx + 3 * blk + 1), bx = __ldg(a.idx + 3 * blk + 2);
      const int b = k & 1;
      const int r = (int)rank * 128 + q * 32 + lane;
      const int oy = r / BS, ox = r % BS;
      const int Y = by * g.obh + oy, X = bx * g.obw + ox;
      const bool store = oy < g.obh && ox < g.obw && Y < g.oh && X < g.ow;
      uint4* op = reinterpret_cast<uint4*>(a.out) +
                  (((size_t)n * g.oh + (store ? Y : 0)) * g.ow + (store ? X : 0)) * (COUT / 8);
      tc::mbar_wait(&acc_full[b], (k >> 1) & 1);
      tc::fence_after();
      const uint32_t acc = tmem + b * P::ACC;
#pragma unroll
      for (int c0 = tpar * (COUT / 2); c0 < (tpar + 1) * (COUT / 2); c0 += 16) {
        float v[16];
        tc::tmem_ld16(acc + ((uint32_t)(q * 32) << 16) + c0, v);
        if (store) {
          uint32_t o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            o[e] = tc::pack_bf16(v[2 * e] + bias[c0 + 2 * e], v[2 * e + 1] + bias[c0 + 2 * e + 1]);
          op[c0 / 8] = make_uint4(o[0], o[1], o[2], o[3]);
          op[c0 / 8 + 1] = make_uint4(o[4], o[5], o[6], o[7]);
        }
      }
      tc::fence_before();
      if (rank == 0) tc::mbar_arrive(&acc_empty[b]);
      else tc::mbar_arrive_cluster(&acc_empty[b], 0);
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();  // the peer's MMAs / remote arrivals are done before TMEM is freed
  tc::fence_after();
  if (warp == 0) tc::tmem_free_cg2<P::TALLOC>(tmem);
}

template <int CIN, int COUT, int BS>
int launch_conv_pair(const ConvArgs& c, int cap, cudaStream_t s) {
  using P = PairConvCfg<CIN, COUT, BS>;
  PairConvArgs pa;
  memset(&pa, 0, sizeof(pa));
  pa.c = c;
  pa.trace = trace_buffer();
  const Geo& g = c.g;
  const uint64_t dims[5] = {8, (uint64_t)g.w, (uint64_t)g.h, (uint64_t)(CIN / 8), (uint64_t)g.n};
  const uint64_t str[4] = {(uint64_t)CIN * 2, (uint64_t)g.w * CIN * 2, 16, (uint64_t)g.h * g.w * CIN * 2};
  const uint32_t box[5] = {8, (uint32_t)BS, (uint32_t)P::WROWS, (uint32_t)(CIN / 8), 1};
  int st = encode_map(&pa.tmap, c.x, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st) return st;
  const uint64_t wdims[2] = {64, (uint64_t)18 * P::WBOXR};  // 18 tap halves of WBOXR 128-byte rows
  const uint64_t wstr[1] = {128};
  const uint32_t wbox[2] = {64, (uint32_t)P::WBOXR};
  st = encode_map(&pa.wmap, c.wpk + (size_t)9 * P::TAP, 2, wdims, wstr, wbox, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st) return st;
  auto kern = conv_tc_pair_kernel<CIN, COUT, BS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM);
  const int npairs = cap < sm_count() / 2 ? (cap < 1 ? 1 : cap) : sm_count() / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * npairs));
  cfg.blockDim = dim3(kPairThreads);
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
  return launch_status("sparse_conv_tcgen05_pair");
}

// ---------------------------------------------------------------------------------------
// CTA pair with RESIDENT weights (16x16 blocks, CIN = COUT = 128: config 3).  The
// single-CTA kernels stream all 9 weight taps (295 KB) through shared memory once per
// block, and at M = 128, N = 128 the MMA's own operand reads (4 KB A + 4 KB B per 64-cycle
// UMMA) already use the ~128 B/clk an SM's shared memory delivers, so the weight and window
// writes slow every MMA (~86 cycles issuing; tools/conv_pair_trace.py) and the weight stream
// costs ~25 B/clk per SM of L2 bandwidth on every SM at once.  Here, as in the streamed pair
// kernel above, a block's two M-tiles are ONE M = 256 cta_group::2 UMMA issued by rank 0 and
// each rank holds the output-channel half of B — but that half of ALL 9 taps (147 KB) stays
// resident for the whole launch (9 TMA boxes at start), and the window streams through a
// ring of KC-channel chunks (one 5-D TMA box per chunk and rank, 11 window rows) so the next
// block's chunks land while this block's MMAs run.  Per SM an UMMA reads 4 KB of A plus its
// 2 KB half of B (~96 B/clk) and the only other shared-memory writes are the window chunks.
// MMA order per block: chunk-major (for chunk: for tap: for k16), fp32 accumulation — a
// different rounding order from the single-CTA kernels (tap-major), so not bit-identical
// to them; parity against the fp32 oracle (test_gpu_parity.py).
// Block list: the reduce_mask list (list mode) or, mask-fused, the one-launch global list
// (conv_mask_global: every CTA tests its candidates, publishes, and waits for all CTAs —
// the grid is one CTA per SM, co-resident).
//   wres         both ranks' weight halves landed (rank 1's TMA completes on it)   rank 0
//   cfull[s]     both ranks' chunk boxes of stage s landed                       rank 0
//   cempty[s]    MMAs reading stage s done (multicast commit)                    both
//   acc_full[b]  accumulator b complete (multicast commit)                       both
//   acc_empty[b] 2 x 256 worker arrivals (rank 1's arrive remotely)              rank 0
template <int CIN, int COUT, int BS>
struct PairResCfg {
  static_assert(BS == 16 && COUT % 32 == 0 && CIN % 32 == 0, "resident pair conv");
  static constexpr int WROWS = 11;                 // window rows per rank
  static constexpr int PA = WROWS * BS * 16;       // plane stride (one 8-channel plane)
  static constexpr int KC = 32;                    // channels per window chunk
  static constexpr int KP = KC / 8;                // planes per chunk
  static constexpr int NCH = CIN / KC;             // chunks per block
  static constexpr int CHUNK = KP * PA;            // bytes of one chunk box (per rank)
  static constexpr int SZ_C = (CHUNK + 1023) / 1024 * 1024;
  static constexpr int NH = COUT / 2;
  static constexpr int PWH = NH * 16;
  static constexpr int TAPH = (CIN / 8) * PWH;      // one tap's half
  static constexpr int WBOXR = TAPH / 128;
  static constexpr int WCH = KP * PWH;             // one chunk's planes of one tap half
  static constexpr int WCHR = WCH / 128;           // ... as 128-byte rows (weight box)
  static constexpr int TAP = (CIN / 8) * COUT * 16;
  static constexpr int OFF_C = 9 * TAPH;           // resident weights first
  static constexpr int BUDGET = 220 * 1024;        // dynamic smem (static: mask-list arrays)
  static constexpr int STAGES = (BUDGET - OFF_C - COUT * 4) / SZ_C > 8 ? 8 : (BUDGET - OFF_C - COUT * 4) / SZ_C;
  static_assert(STAGES >= 2, "resident pair conv: ring does not fit");
  static constexpr int OFF_BIAS = OFF_C + STAGES * SZ_C;
  static constexpr int SMEM = OFF_BIAS + COUT * 4;
  static constexpr int ACC = COUT;
  static constexpr int TALLOC = 2 * ACC <= 32 ? 32 : 2 * ACC <= 64 ? 64 : 2 * ACC <= 128 ? 128 : 2 * ACC <= 256 ? 256 : 512;
};

template <int CIN, int COUT, int BS>
__global__ void __launch_bounds__(kPairThreads, 1) conv_tc_pair_res_kernel(const __grid_constant__ PairConvArgs pa) {
  using P = PairResCfg<CIN, COUT, BS>;
  const ConvArgs& a = pa.c;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t cfull[P::STAGES], cempty[P::STAGES];
  __shared__ uint64_t wres[P::NCH], acc_full[2], acc_empty[2];
  __shared__ uint32_t tslot;
  __shared__ int32_t s_idx[3 * kMaxLocal];  // mask-fused: this CTA's candidates before publishing
  uint8_t* W = smem;
  float* bias = reinterpret_cast<float*>(smem + P::OFF_BIAS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = tc::cluster_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const Geo& g = a.g;
  // diagnostics (tools/conv_res_timeline.py): %globaltimer phase stamps per CTA
  unsigned long long* tl = pa.trace ? pa.trace + 2048 * 8 + blockIdx.x * 8 : nullptr;
  if (tl && tid == 0) tl[0] = gtimer();

  if (tid == 0) {
    for (int s = 0; s < P::STAGES; ++s) {
      tc::mbar_init(&cfull[s], 1);
      tc::mbar_init(&cempty[s], 1);
    }
    for (int c = 0; c < P::NCH; ++c) tc::mbar_init(&wres[c], 1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], 2 * kWorkers);
    }
    tc::mbar_fence_init();
  }
  if (tid == 10 * 32) asm volatile("prefetch.tensormap [%0];" ::"l"(&pa.tmap) : "memory");
  if (tid == 8 * 32) asm volatile("prefetch.tensormap [%0];" ::"l"(&pa.wmap) : "memory");
  for (int i = tid; i < COUT; i += kPairThreads) bias[i] = a.bias ? __bfloat162float(a.bias[i]) : 0.f;
  if (warp == 0) tc::tmem_alloc_cg2<P::TALLOC>(&tslot);
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();  // both CTAs' barriers exist before any remote arrive / multicast commit
  tc::fence_after();
  const uint32_t tmem = tslot;
  // weight loader: my half of all 9 taps, once, chunk-major (the issuer starts on chunk 0
  // while the rest lands).  Issued before griddepcontrol.wait: the packed image does not
  // depend on the previous kernel (a reduce_mask launch triggers its dependents at entry, so
  // these copies overlap it), and mask-fused they also overlap the mask test.
  auto load_weights = [&]() {
    if (tid != 8 * 32) return;
    for (int c = 0; c < P::NCH; ++c) {
      if (rank == 0) tc::mbar_expect_tx(&wres[c], 2 * 9 * P::WCH);
      for (int tap = 0; tap < 9; ++tap) {
        const int row = (2 * tap + (int)rank) * P::WBOXR + c * P::WCHR;
        uint8_t* dst = W + tap * P::TAPH + c * P::WCH;
        if (rank == 0) tma_2d(dst, &pa.wmap, 0, row, &wres[c]);
        else tma_2d_cg2(dst, &pa.wmap, 0, row, &wres[c], 0);
      }
    }
  };
  load_weights();
  if (pa.early_trigger) tc::pdl_trigger();  // the next launch (e.g. reduce_mask) may start
  tc::pdl_wait();
  if (tl && tid == 0) tl[1] = gtimer();
  const bool global = a.mask != nullptr;
  const int B = global ? conv_mask_global<kPairThreads, BS>(a, s_idx) : ld_count(a.count, a.cap);
  const int nmine = B > pair ? (B - pair + npairs - 1) / npairs : 0;  // my pair's blocks
  // block k of my pair -> (frame, block row, block column)
  auto block_of = [&](int k, int& n, int& by, int& bx) {
    const int blk = pair + k * npairs;
    if (global) {  // rows written in this launch: coherent loads
      n = a.gidx[3 * blk];
      by = a.gidx[3 * blk + 1];
      bx = a.gidx[3 * blk + 2];
    } else {
      n = __ldg(a.idx + 3 * blk);
      by = __ldg(a.idx + 3 * blk + 1);
      bx = __ldg(a.idx + 3 * blk + 2);
    }
  };
  if (tl && tid == 0) {
    tl[2] = gtimer();
    tl[7] = B;
  }

  if (warp == 8) {
    // (the weight loader's copies were issued above)
  } else if (warp == 10) {
    // ---------------- window loader: my 11 rows of every block, KC channels per box
    if (lane == 0) {
      int it = 0;
      for (int kb = 0; kb < nmine; ++kb) {
        int n, by, bx;
        block_of(kb, n, by, bx);
        const int ys = g.oy + by * g.sy + (int)rank * (P::WROWS - 3), xs = g.ox + bx * g.sx;
        for (int c = 0; c < P::NCH; ++c, ++it) {
          const int s = it % P::STAGES;
          tc::mbar_wait(&cempty[s], ((it / P::STAGES) & 1) ^ 1);
          if (rank == 0) {
            tc::mbar_expect_tx(&cfull[s], 2 * P::CHUNK);
            tma_5d(smem + P::OFF_C + s * P::SZ_C, &pa.tmap, 0, xs, ys, c * P::KP, n, &cfull[s]);
          } else {
            tma_5d_cg2(smem + P::OFF_C + s * P::SZ_C, &pa.tmap, 0, xs, ys, c * P::KP, n, &cfull[s], 0);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 9) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (rank 0): M = 256 over the pair
      int it = 0, k = 0;
      constexpr uint32_t idesc = tc::idesc_bf16_f32(256, COUT);
      unsigned long long t_win = 0, t_acc = 0, t_w = 0, t0 = clock64();
      const uint64_t wd0 = tc::desc_kmajor_noswz(tc::smem_u32(W), P::PWH, 128);
      const uint64_t ad0 = tc::desc_kmajor_noswz(tc::smem_u32(smem + P::OFF_C), P::PA, 128);
      for (; k < nmine; ++k) {
        const int b = k & 1;
        unsigned long long c1 = clock64();
        tc::mbar_wait(&acc_empty[b], ((k >> 1) & 1) ^ 1);
        t_acc += clock64() - c1;
        tc::fence_after();
        const uint32_t acc = tmem + b * P::ACC;
        for (int c = 0; c < P::NCH; ++c, ++it) {
          const int s = it % P::STAGES;
          unsigned long long c3 = clock64();
          if (k == 0) tc::mbar_wait(&wres[c], 0);
          const unsigned long long c4 = clock64();
          t_w += c4 - c3;
          tc::mbar_wait(&cfull[s], (it / P::STAGES) & 1);
          t_win += clock64() - c4;
          if (tl && it == 0) tl[3] = gtimer();
          tc::fence_after();
          const uint64_t ad = tc::desc_add(ad0, s * P::SZ_C);
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const int shift = (tap / 3) * BS + (tap % 3);
#pragma unroll
            for (int kk = 0; kk < P::KP / 2; ++kk)
              tc::mma_bf16_cg2(acc, tc::desc_add(ad, 2 * kk * P::PA + shift * 16),
                               tc::desc_add(wd0, tap * P::TAPH + (c * P::KP + 2 * kk) * P::PWH), idesc,
                               (c | tap | kk) > 0);
          }
          tc::mma_commit_mc(&cempty[s], 3);
        }
        tc::mma_commit_mc(&acc_full[b], 3);
      }
      if (tl) tl[4] = gtimer();
      if (k == 0)  // no blocks: the weight copies must land before the CTAs exit
        for (int c = 0; c < P::NCH; ++c) tc::mbar_wait(&wres[c], 0);
      if (pa.trace) {
        unsigned long long* tb = pa.trace + blockIdx.x * 8;
        tb[0] = clock64() - t0;
        tb[1] = t_win;
        tb[2] = t_acc;
        tb[3] = t_w;
        tb[4] = k;
      }
    }
    __syncwarp();
  } else {
    // ---------------- workers: drain my tile of each accumulator
    const int q = warp & 3, tpar = warp >> 2;
    int k = 0;
    for (; k < nmine; ++k) {
      int n, by, bx;
      block_of(k, n, by, bx);
      const int b = k & 1;
      const int r = (int)rank * 128 + q * 32 + lane;
      const int oy = r / BS, ox = r % BS;
      const int Y = by * g.obh + oy, X = bx * g.obw + ox;
      const bool store = oy < g.obh && ox < g.obw && Y < g.oh && X < g.ow;
      uint4* op = reinterpret_cast<uint4*>(a.out) +
                  (((size_t)n * g.oh + (store ? Y : 0)) * g.ow + (store ? X : 0)) * (COUT / 8);
      tc::mbar_wait(&acc_full[b], (k >> 1) & 1);
      tc::fence_after();
      const uint32_t acc = tmem + b * P::ACC;
#pragma unroll
      for (int c0 = tpar * (COUT / 2); c0 < (tpar + 1) * (COUT / 2); c0 += 16) {
        float v[16];
        tc::tmem_ld16(acc + ((uint32_t)(q * 32) << 16) + c0, v);
        if (store) {
          uint32_t o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            o[e] = tc::pack_bf16(v[2 * e] + bias[c0 + 2 * e], v[2 * e + 1] + bias[c0 + 2 * e + 1]);
          op[c0 / 8] = make_uint4(o[0], o[1], o[2], o[3]);
          op[c0 / 8 + 1] = make_uint4(o[4], o[5], o[6], o[7]);
        }
      }
      tc::fence_before();
      if (rank == 0) tc::mbar_arrive(&acc_empty[b]);
      else tc::mbar_arrive_cluster(&acc_empty[b], 0);
    }
    if (tl && tid == 0) tl[5] = gtimer();
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();  // the peer's MMAs / remote arrivals / TMA completions are done before exit
  tc::fence_after();
  if (warp == 0) tc::tmem_free_cg2<P::TALLOC>(tmem);
  if (tl && tid == 0) tl[6] = gtimer();
}

// pairs the resident kernel may launch (2-CTA clusters of its size co-resident on this
// device; the mask-fused global list needs every CTA resident), cached per device
template <int CIN, int COUT, int BS>
int pair_res_max_pairs() {
  using P = PairResCfg<CIN, COUT, BS>;
  static int cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 0;
  if (cache[dev]) return cache[dev] > 0 ? cache[dev] : 0;
  auto kern = conv_tc_pair_res_kernel<CIN, COUT, BS>;
  int v = -1;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM) == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(kPairThreads);
    cfg.dynamicSmemBytes = P::SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) == cudaSuccess && nc > 0) v = nc < sm_count() / 2 ? nc : sm_count() / 2;
  }
  cudaGetLastError();
  cache[dev] = v;
  return v > 0 ? v : 0;
}

template <int CIN, int COUT, int BS>
int launch_conv_pair_res(const ConvArgs& c, int cap, cudaStream_t s) {
  using P = PairResCfg<CIN, COUT, BS>;
  const int maxp = pair_res_max_pairs<CIN, COUT, BS>();
  if (maxp <= 0) return SBN_ERR_UNSUPPORTED;
  if (c.mask && (cap + 2 * maxp - 1) / (2 * maxp) > kMaxLocal) return SBN_ERR_UNSUPPORTED;
  PairConvArgs pa;
  memset(&pa, 0, sizeof(pa));
  pa.c = c;
  pa.trace = trace_buffer();
  pa.early_trigger = !(debug_flags() & kDebugNoMaskPdl);
  const Geo& g = c.g;
  const uint64_t dims[5] = {8, (uint64_t)g.w, (uint64_t)g.h, (uint64_t)(CIN / 8), (uint64_t)g.n};
  const uint64_t str[4] = {(uint64_t)CIN * 2, (uint64_t)g.w * CIN * 2, 16, (uint64_t)g.h * g.w * CIN * 2};
  const uint32_t box[5] = {8, (uint32_t)BS, (uint32_t)P::WROWS, (uint32_t)P::KP, 1};
  int st = encode_map(&pa.tmap, c.x, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st) return st;
  const uint64_t wdims[2] = {64, (uint64_t)18 * P::WBOXR};  // 18 tap halves of WBOXR 128-byte rows
  const uint64_t wstr[1] = {128};
  const uint32_t wbox[2] = {64, (uint32_t)P::WCHR};
  st = encode_map(&pa.wmap, c.wpk + (size_t)9 * P::TAP, 2, wdims, wstr, wbox, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st) return st;
  auto kern = conv_tc_pair_res_kernel<CIN, COUT, BS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM);
  // mask-fused: every CTA tests candidates, so the full co-resident grid; list mode: no more
  // pairs than blocks
  const int npairs = c.mask ? maxp : (cap < maxp ? (cap < 1 ? 1 : cap) : maxp);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * npairs));
  cfg.blockDim = dim3(kPairThreads);
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
  return launch_status("sparse_conv_tcgen05_pair_res");
}

#define SBN_CONV_TC_CONFIGS(X) \
  X(128, 128, 16)              \
  X(128, 128, 8)               \
  X(64, 64, 16)                \
  X(64, 64, 8)                 \
  X(32, 32, 16)

}  // namespace

bool sparse_conv_tc_supported(int dtype, int cin, int cout, int kh, int kw, int sh, int sw,
                              const Geo& g) {
  if (dtype != SBN_BF16 || kh != 3 || kw != 3 || sh != 1 || sw != 1 || g.bh != g.bw) return false;
#define X(CI, CO, BS_) if (cin == CI && cout == CO && g.bh == BS_ && ConvCfg<CI, CO, BS_>::SMEM <= max_smem_optin()) return true;
  SBN_CONV_TC_CONFIGS(X)
#undef X
  return false;
}

size_t sparse_conv_tc_packed_bytes(int cin, int cout) { return (size_t)2 * 9 * cin * cout * 2; }  // + pair copy

int sparse_conv_tc_pack(const void* w, int cin, int cout, void* img, cudaStream_t s) {
#define X(CI, CO, BS_) if (cin == CI && cout == CO) { conv_tc_pack_kernel<CI, CO><<<64, 256, 0, s>>>((const __nv_bfloat16*)w, (uint8_t*)img); return launch_status("sparse_conv_tc_pack"); }
  SBN_CONV_TC_CONFIGS(X)
#undef X
  set_error("no tcgen05 conv instantiation for cin=%d cout=%d", cin, cout);
  return SBN_ERR_UNSUPPORTED;
}

// mask-fused launch: only the double-buffered kernel; returns SBN_ERR_UNSUPPORTED when that
// variant does not apply (the caller then reduces the mask separately)
int sparse_conv_tc_masked(const void* x, const uint8_t* mask, int cin, int cout, Geo g, const void* wpk,
                          const void* bias, int cap, void* dst, cudaStream_t s, unsigned* slotw, int32_t* gidx) {
  if (debug_flags() & (kDebugConvSingleBuffer | kDebugConvPair)) return SBN_ERR_UNSUPPORTED;
  // Per-CTA lists balance only statistically: with few candidates per CTA a structured
  // mask (e.g. a top-left rectangle) lands unevenly on the round-robin owners (measured,
  // config 3: 16x16 blocks, 20 candidates / CTA: 61 vs 36 us at 10 % against the ordered
  // reduce_mask + conv); 8x8 blocks, 106 / CTA: 40 vs 46 us.  So from kMinLocal candidates per
  // CTA the CTAs keep their own lists; below it they publish one global list in the same
  // launch (conv_mask_global: evenly striped like the ordered list, no reduce_mask launch).
  constexpr int kMinLocal = 64;
  const int per_cta = (cap + sm_count() - 1) / sm_count();
  if (per_cta > kMaxLocal || (per_cta < kMinLocal && (!slotw || !gidx || (debug_flags() & kDebugNoGlobalList))))
    return SBN_ERR_UNSUPPORTED;
  ConvArgs a;
  memset(&a, 0, sizeof(a));
  if (!(debug_flags() & (kDebugConvNoRes | kDebugNoGlobalList)) && slotw && gidx && g.bh == 16 && cin == 128 && cout == 128) {
    // Resident-weight CTA pair.  Default: reduce_mask (which triggers its PDL dependents at
    // entry) + the pair's list mode, whose prologue and 147 KB weight copies then overlap
    // the mask reduction — measured faster than the one-launch global list at every density
    // (config 3: 30.7 vs 31.5 us at 10 %, 200 vs 206 us at 100 %; tools/conv_res_ab.py).
    if (!(debug_flags() & kDebugConvResOneLaunch) && pair_res_max_pairs<128, 128, 16>() > 0)
      return SBN_ERR_UNSUPPORTED;
    // one launch: the mask test and the global list inside the pair kernel
    a.x = (const __nv_bfloat16*)x;
    a.out = (__nv_bfloat16*)dst;
    a.g = g;
    a.wpk = (const uint8_t*)wpk;
    a.bias = (const __nv_bfloat16*)bias;
    a.cap = cap;
    a.mask = mask;
    a.sw = slotw;
    a.gidx = gidx;
    const int st = launch_conv_pair_res<128, 128, 16>(a, cap, s);
    if (st != SBN_ERR_UNSUPPORTED) return st;
    memset(&a, 0, sizeof(a));
  }
  if (per_cta < kMinLocal) {
    a.sw = slotw;
    a.gidx = gidx;
  }
  a.x = (const __nv_bfloat16*)x;
  a.out = (__nv_bfloat16*)dst;
  a.g = g;
  a.wpk = (const uint8_t*)wpk;
  a.bias = (const __nv_bfloat16*)bias;
  a.cap = cap;
  a.trace = trace_buffer();
  a.mask = mask;
#define X(CI, CO, BS_) if (cin == CI && cout == CO && g.bh == BS_ && DbCfg<CI, CO, BS_>::SMEM <= max_smem_optin()) return launch_conv_db<CI, CO, BS_>(a, cap, s);
  SBN_CONV_TC_CONFIGS(X)
#undef X
  return SBN_ERR_UNSUPPORTED;
}

int sparse_conv_tc(const void* x, int cin, int cout, Geo g, const void* wpk, const void* bias,
                   const int32_t* idx, const int32_t* count, int cap, void* dst, cudaStream_t s) {
  ConvArgs a;
  memset(&a, 0, sizeof(a));
  a.x = (const __nv_bfloat16*)x;
  a.out = (__nv_bfloat16*)dst;
  a.g = g;
  a.wpk = (const uint8_t*)wpk;
  a.bias = (const __nv_bfloat16*)bias;
  a.idx = idx;
  a.count = count;
  a.cap = cap;
  a.trace = trace_buffer();
  // CTA-pair (cta_group::2) variant: opt-in (SBN_DEBUG_CONV_PAIR) — measured slower than the
  // double-buffered single-CTA kernel on config 3 (210 vs 175 us at 100 %, 37 vs 28 us at
  // 10 %): the M = 256 MMA still reads ~96 B/clk of smem per SM and the per-pair weight
  // stream (16 KB per tap per CTA) stalls the issuer 11 % of the time
  if ((debug_flags() & kDebugConvPair) && g.bh == 16) {
    if (cin == 128 && cout == 128) return launch_conv_pair<128, 128, 16>(a, cap, s);
    if (cin == 64 && cout == 64) return launch_conv_pair<64, 64, 16>(a, cap, s);
    if (cin == 32 && cout == 32) return launch_conv_pair<32, 32, 16>(a, cap, s);
  }
  if (!(debug_flags() & (kDebugConvSingleBuffer | kDebugConvNoRes)) && g.bh == 16 && cin == 128 && cout == 128) {
    const int st = launch_conv_pair_res<128, 128, 16>(a, cap, s);  // resident-weight CTA pair
    if (st != SBN_ERR_UNSUPPORTED) return st;
  }
  if (!(debug_flags() & kDebugConvSingleBuffer)) {
#define X(CI, CO, BS_) if (cin == CI && cout == CO && g.bh == BS_ && DbCfg<CI, CO, BS_>::SMEM <= max_smem_optin()) return launch_conv_db<CI, CO, BS_>(a, cap, s);
    SBN_CONV_TC_CONFIGS(X)
#undef X
  }
#define X(CI, CO, BS_) if (cin == CI && cout == CO && g.bh == BS_) return launch_conv<CI, CO, BS_>(a, cap, s);
  SBN_CONV_TC_CONFIGS(X)
#undef X
  set_error("no tcgen05 conv instantiation for cin=%d cout=%d block=%d", cin, cout, g.bh);
  return SBN_ERR_UNSUPPORTED;
}

}  // namespace sbn
