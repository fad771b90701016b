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
// Warp roles per persistent CTA (320 threads):
//   warps 0-3  A producers: per 128-row tile and K-chunk, load the rows (16-B vectors,
//              all in flight), apply the transform, store the K-major plane layout of
//              tc_util.cuh into an SA-deep ring
//   warps 4-7  epilogue: tcgen05.ld of the accumulator (TMEM lane quarter = warp % 4),
//              transform, vector stores; double-buffered accumulators when 2*N <= 512
//   warp 8     W producer: cp.async.bulk of pre-packed weight chunks through an SW ring
//   warp 9     MMA issuer (one thread): tcgen05.mma M=128, N<=256 per instruction
#include "unit.cuh"
#include "tc_util.cuh"

namespace sbn {
namespace {

constexpr int kAThreads = 128;
constexpr int kEThreads = 128;
constexpr int kWideThreads = kAThreads + kEThreads + 64;
constexpr int kMaxRows = 168;  // staged rows of a MID tile: 128 + 2*b + 2 (b <= 18)

enum { kIn = 1, kMid = 2, kOut = 3 };

template <int K, int N, int MODE>
struct WCfg {
  static constexpr int TAPS = MODE == kMid ? 9 : 1;
  static constexpr int KC = K <= 96 ? K : (K % 64 == 0 ? 64 : 32);
  static_assert(K % KC == 0 && KC % 16 == 0, "K chunking");
  static constexpr int NKC = K / KC;
  static constexpr int RA = MODE == kMid ? kMaxRows : 128;
  static constexpr int PA = RA * 16 + 16;  // A plane stride (16-B pad: conflict-free staging)
  static constexpr int ACH = (KC / 8) * PA;
  static constexpr int PW = N * 16;
  static constexpr int WCH = (KC / 8) * PW;
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
  static constexpr int BUDGET = 210 * 1024;
  static constexpr int SA = (4 * ACH + 2 * WCH + PARB <= BUDGET) ? 4 : (3 * ACH + 2 * WCH + PARB <= BUDGET) ? 3 : 2;
  static constexpr int SW = (SA * ACH + 4 * WCH + PARB <= BUDGET) ? 4 : (SA * ACH + 3 * WCH + PARB <= BUDGET) ? 3 : 2;
  static_assert(SA * ACH + SW * WCH + PARB <= BUDGET, "shared memory budget");
  static constexpr int OFF_W = SA * ACH;
  static constexpr int OFF_PAR = OFF_W + SW * WCH;
  static constexpr int SMEM = OFF_PAR + PARB;
  static constexpr int ITEMS = (RA * (KC / 8) + kAThreads - 1) / kAThreads;
  static constexpr int CHUNKS = NKC * TAPS;                       // weight chunks per tile
  static constexpr size_t WBYTES = (size_t)CHUNKS * WCH;          // packed weight bytes
};

struct WArgs {
  const __nv_bfloat16* src;  // IN: x    MID: S1    OUT: S2
  __nv_bfloat16* dst;        // IN: S1   MID: S2    OUT: out
  const uint8_t* wpk;        // this GEMM's packed weight chunks
  const float* par;          // this GEMM's parameter vectors
  Geo g;
  const int32_t* idx;
  const int32_t* count;
  int cap;
};

__device__ __forceinline__ void abar_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// rows of the GEMM for B active blocks of size b
template <int MODE>
__device__ __forceinline__ long total_rows(int B, int b) {
  return MODE == kOut ? (long)B * (b - 2) * (b - 2) : (long)B * b * b;
}

template <int K, int N, int MODE>
__global__ void __launch_bounds__(kWideThreads, 1) unit_wide_kernel(WArgs a) {
  using Q = WCfg<K, N, MODE>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t a_full[Q::SA], a_empty[Q::SA], w_full[Q::SW], w_empty[Q::SW];
  __shared__ uint64_t acc_full[Q::NACC], acc_empty[Q::NACC];
  __shared__ uint32_t tslot;
  __shared__ long long rowoff[Q::RA];
  uint8_t* Aring = smem;
  uint8_t* Wring = smem + Q::OFF_W;
  float* par = reinterpret_cast<float*>(smem + Q::OFF_PAR);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Geo& g = a.g;
  const int b = g.bh;

  if (tid == 0) {
    for (int s = 0; s < Q::SA; ++s) {
      tc::mbar_init(&a_full[s], kAThreads);
      tc::mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < Q::SW; ++s) {
      tc::mbar_init(&w_full[s], 1);
      tc::mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < Q::NACC; ++s) {
      tc::mbar_init(&acc_full[s], 1);
      tc::mbar_init(&acc_empty[s], kEThreads);
    }
    tc::mbar_fence_init();
  }
  for (int i = tid; i < Q::NPAR; i += kWideThreads) par[i] = a.par[i];
  if (warp == 0) tc::tmem_alloc<Q::TALLOC>(&tslot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  tc::pdl_trigger();
  tc::pdl_wait();  // the previous launch's S1 / S2 / x and the index list are visible
  const int B = ld_count(a.count, a.cap);
  const long TR = total_rows<MODE>(B, b);
  const int ntiles = (int)((TR + 127) / 128);

  if (warp < 4) {
    // ------------------------------------------------ A producers
    const int rows = MODE == kMid ? 128 + 2 * b + 2 : 128;
    const int bb = b * b;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      abar_sync();  // everyone is done with the previous tile's rowoff
      for (int r = tid; r < Q::RA; r += kAThreads) {
        const long gr = (long)tile * 128 + r;
        long long off = -1;
        if (r < rows && gr < TR) {
          if (MODE == kIn) {
            const int j = (int)(gr / bb), p = (int)(gr - (long)j * bb);
            const int n = __ldg(a.idx + 3 * j), by = __ldg(a.idx + 3 * j + 1), bx = __ldg(a.idx + 3 * j + 2);
            const int y = g.oy + by * g.sy + p / b, x = g.ox + bx * g.sx + p % b;
            if (y >= 0 && y < g.h && x >= 0 && x < g.w) off = (((long long)n * g.h + y) * g.w + x) * K;
          } else {
            off = gr * K;
          }
        }
        rowoff[r] = off;
      }
      abar_sync();
      for (int kc = 0; kc < Q::NKC; ++kc, ++it) {
        const int s = it % Q::SA;
        tc::mbar_wait(&a_empty[s], ((it / Q::SA) & 1) ^ 1);
        uint8_t* A = Aring + s * Q::ACH;
        uint4 raw[Q::ITEMS];
#pragma unroll
        for (int j = 0; j < Q::ITEMS; ++j) {
          const int i = tid + j * kAThreads;
          const int r = i / (Q::KC / 8), k8 = i % (Q::KC / 8);
          raw[j] = make_uint4(0, 0, 0, 0);
          if (r < Q::RA) {
            const long long off = rowoff[r];
            if (off >= 0) raw[j] = __ldg(reinterpret_cast<const uint4*>(a.src + off + kc * Q::KC) + k8);
          }
        }
#pragma unroll
        for (int j = 0; j < Q::ITEMS; ++j) {
          const int i = tid + j * kAThreads;
          const int r = i / (Q::KC / 8), k8 = i % (Q::KC / 8);
          if (r >= Q::RA) break;
          uint4 v = raw[j];
          if (MODE == kIn && rowoff[r] >= 0) {
            const float* s1 = par;
            const float* t1 = par + K;
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[j]);
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(h[e]);
              const int ch = kc * Q::KC + k8 * 8 + 2 * e;
              o[e] = tc::pack_bf16(fmaxf(__fadd_rn(__fmul_rn(f.x, s1[ch]), t1[ch]), 0.f),
                                   fmaxf(__fadd_rn(__fmul_rn(f.y, s1[ch + 1]), t1[ch + 1]), 0.f));
            }
            v = make_uint4(o[0], o[1], o[2], o[3]);
          }
          *reinterpret_cast<uint4*>(A + k8 * Q::PA + r * 16) = v;
        }
        tc::fence_async_smem();
        tc::mbar_arrive(&a_full[s]);
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------ epilogue
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const int bb = b * b, ob = b - 2;
    int k = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
      const int buf = Q::NACC == 2 ? (k & 1) : 0;
      const int use = Q::NACC == 2 ? (k >> 1) : k;
      const long gr = (long)tile * 128 + r;
      bool store = gr < TR;
      bool valid = true;  // IN: in-bounds pixel
      __nv_bfloat16* dp = nullptr;
      const __nv_bfloat16* xp = nullptr;
      if (store) {
        if (MODE == kIn) {
          const int j = (int)(gr / bb), p = (int)(gr - (long)j * bb);
          const int n = __ldg(a.idx + 3 * j), by = __ldg(a.idx + 3 * j + 1), bx = __ldg(a.idx + 3 * j + 2);
          const int y = g.oy + by * g.sy + p / b, x = g.ox + bx * g.sx + p % b;
          valid = y >= 0 && y < g.h && x >= 0 && x < g.w;
          (void)n;
          dp = a.dst + gr * N;
        } else if (MODE == kMid) {
          const int j = (int)(gr / bb), p = (int)(gr - (long)j * bb);
          const int oy = p / b, ox = p % b;
          store = oy < ob && ox < ob;
          dp = a.dst + ((long)j * ob * ob + oy * ob + ox) * N;
        } else {
          const int j = (int)(gr / (ob * ob)), p = (int)(gr - (long)j * ob * ob);
          const int oy = p / ob, ox = p % ob;
          const int n = __ldg(a.idx + 3 * j), by = __ldg(a.idx + 3 * j + 1), bx = __ldg(a.idx + 3 * j + 2);
          const int Y = by * g.obh + oy, X = bx * g.obw + ox;
          store = Y < g.oh && X < g.ow;
          dp = a.dst + (((long)n * g.oh + Y) * g.ow + X) * N;
          xp = dp;  // the residual: out holds x's values (clone or in place)
        }
      }
      tc::mbar_wait(&acc_full[buf], use & 1);
      tc::fence_after();
      const uint32_t acc = tmem + ((uint32_t)(qd * 32) << 16) + buf * N;
#pragma unroll 2
      for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        tc::tmem_ld16(acc + c0, v);
        if (!store) continue;
        uint32_t o[8];
        if (MODE == kOut) {
          const float* b3 = par;
          uint4 xr[2];
          xr[0] = reinterpret_cast<const uint4*>(xp + c0)[0];
          xr[1] = reinterpret_cast<const uint4*>(xp + c0)[1];
          const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(xr);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float2 xf = __bfloat1622float2(xh[e]);
            const float u0 = __bfloat162float(__float2bfloat16_rn(v[2 * e] + b3[c0 + 2 * e]));
            const float u1 = __bfloat162float(__float2bfloat16_rn(v[2 * e + 1] + b3[c0 + 2 * e + 1]));
            o[e] = tc::pack_bf16(__fadd_rn(xf.x, u0), __fadd_rn(xf.y, u1));
          }
        } else {
          // IN: +b1, bn2, relu, x valid      MID: +b2, bn3, relu
          const float* bi = MODE == kIn ? par + 2 * K : par;
          const float* sc = bi + N;
          const float* sh = sc + N;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            float u0 = __bfloat162float(__float2bfloat16_rn(v[2 * e] + bi[c0 + 2 * e]));
            float u1 = __bfloat162float(__float2bfloat16_rn(v[2 * e + 1] + bi[c0 + 2 * e + 1]));
            u0 = fmaxf(__fadd_rn(__fmul_rn(u0, sc[c0 + 2 * e]), sh[c0 + 2 * e]), 0.f);
            u1 = fmaxf(__fadd_rn(__fmul_rn(u1, sc[c0 + 2 * e + 1]), sh[c0 + 2 * e + 1]), 0.f);
            o[e] = valid ? tc::pack_bf16(u0, u1) : 0u;
          }
        }
        uint4* op = reinterpret_cast<uint4*>(dp + c0);
        op[0] = make_uint4(o[0], o[1], o[2], o[3]);
        op[1] = make_uint4(o[4], o[5], o[6], o[7]);
      }
      tc::fence_before();
      tc::mbar_arrive(&acc_empty[buf]);
    }
  } else if (warp == 8) {
    // ------------------------------------------------ W producer
    if (lane == 0) {
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int c = 0; c < Q::CHUNKS; ++c, ++it) {
          const int s = it % Q::SW;
          tc::mbar_wait(&w_empty[s], ((it / Q::SW) & 1) ^ 1);
          tc::mbar_expect_tx(&w_full[s], Q::WCH);
          tc::bulk_g2s(Wring + s * Q::WCH, a.wpk + (size_t)c * Q::WCH, Q::WCH, &w_full[s]);
        }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(128, Q::NS);
      int ait = 0, wit = 0, k = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
        const int buf = Q::NACC == 2 ? (k & 1) : 0;
        const int use = Q::NACC == 2 ? (k >> 1) : k;
        tc::mbar_wait(&acc_empty[buf], (use & 1) ^ 1);
        tc::fence_after();
        const uint32_t acc = tmem + buf * N;
        for (int kc = 0; kc < Q::NKC; ++kc, ++ait) {
          const int sa = ait % Q::SA;
          tc::mbar_wait(&a_full[sa], (ait / Q::SA) & 1);
          tc::fence_after();
          const uint32_t abase = tc::smem_u32(Aring + sa * Q::ACH);
          for (int tap = 0; tap < Q::TAPS; ++tap, ++wit) {
            const int sw = wit % Q::SW;
            tc::mbar_wait(&w_full[sw], (wit / Q::SW) & 1);
            tc::fence_after();
            const int shift = MODE == kMid ? (tap / 3) * b + (tap % 3) : 0;
            const uint32_t wbase = tc::smem_u32(Wring + sw * Q::WCH);
#pragma unroll
            for (int kk = 0; kk < Q::KC / 16; ++kk)
#pragma unroll
              for (int h = 0; h < Q::NSPLIT; ++h)
                tc::mma_bf16(acc + h * Q::NS,
                             tc::desc_kmajor_noswz(abase + 2 * kk * Q::PA + shift * 16, Q::PA, 128),
                             tc::desc_kmajor_noswz(wbase + 2 * kk * Q::PW + h * Q::NS * 16, Q::PW, 128),
                             idesc, (kc | tap | kk) > 0);
            tc::mma_commit(&w_empty[sw]);
          }
          tc::mma_commit(&a_empty[sa]);
        }
        tc::mma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_free<Q::TALLOC>(tmem);
}

// ---- packed image: [W1 chunks | W2 chunks | W3 chunks | params], regions 128-B aligned.
// A chunk c of a GEMM with K-chunk KC, N columns: KC/8 planes of N rows x 16 B,
// element (n, k) at (k/8)*N*16 + n*16 + (k%8)*2 — the kernel's B-operand layout.  MID
// chunks are ordered (kc, tap).
//   params (floats): IN  s1 t1 [c] b1 s2 t2 [m]   MID b2 s3 t3 [m]   OUT b3 [c]
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
  // W1 (1, 1, C, M): B[n = co][k = ci]
  for (int i = t0; i < C * M; i += stride) {
    const int ci = i / M, co = i % M;
    const int kc = ci / Q1::KC, k = ci % Q1::KC;
    *reinterpret_cast<__nv_bfloat16*>(img + L.w1 + (size_t)kc * Q1::WCH + (k / 8) * Q1::PW + co * 16 + (k % 8) * 2) = w1[i];
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
  for (int i = t0; i < C; i += stride) {
    p1[i] = ((const float*)p.bn1_scale)[i];
    p1[C + i] = ((const float*)p.bn1_shift)[i];
    p3[i] = bf(p.b3, i);
  }
  for (int i = t0; i < M; i += stride) {
    p1[2 * C + i] = bf(p.b1, i);
    p1[2 * C + M + i] = ((const float*)p.bn2_scale)[i];
    p1[2 * C + 2 * M + i] = ((const float*)p.bn2_shift)[i];
    p2[i] = bf(p.b2, i);
    p2[M + i] = ((const float*)p.bn3_scale)[i];
    p2[2 * M + i] = ((const float*)p.bn3_shift)[i];
  }
}

template <int K, int N, int MODE>
int launch_wide(const WArgs& a, long max_rows, cudaStream_t s, const char* what) {
  using Q = WCfg<K, N, MODE>;
  auto kern = unit_wide_kernel<K, N, MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Q::SMEM);
  const long tiles = (max_rows + 127) / 128;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(tiles < sm_count() ? (tiles < 1 ? 1 : tiles) : sm_count()));
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

template <int C, int M>
int run_wide(const void* x, void* out, const Geo& g, const uint8_t* img, const int32_t* idx,
             const int32_t* count, int cap, uint8_t* s1, uint8_t* s2, cudaStream_t s) {
  constexpr WLayout L = wide_layout<C, M>();
  const int b = g.bh;
  WArgs a;
  a.g = g;
  a.idx = idx;
  a.count = count;
  a.cap = cap;
  // IN: x windows -> S1
  a.src = (const __nv_bfloat16*)x;
  a.dst = (__nv_bfloat16*)s1;
  a.wpk = img + L.w1;
  a.par = (const float*)(img + L.p1);
  int st = launch_wide<C, M, kIn>(a, (long)cap * b * b, s, "residual_unit_wide_in");
  if (st) return st;
  // MID: S1 -> S2 (3x3 valid)
  a.src = (const __nv_bfloat16*)s1;
  a.dst = (__nv_bfloat16*)s2;
  a.wpk = img + L.w2;
  a.par = (const float*)(img + L.p2);
  st = launch_wide<M, M, kMid>(a, (long)cap * b * b, s, "residual_unit_wide_mid");
  if (st) return st;
  // OUT: S2 -> out (+ residual), in place or into the clone
  a.src = (const __nv_bfloat16*)s2;
  a.dst = (__nv_bfloat16*)out;
  a.wpk = img + L.w3;
  a.par = (const float*)(img + L.p3);
  return launch_wide<M, C, kOut>(a, (long)cap * (b - 2) * (b - 2), s, "residual_unit_wide_out");
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

size_t unit_wide_packed_bytes(int c, int m) {
#define X(C_, M_) if (c == C_ && m == M_) return wide_layout<C_, M_>().total;
  SBN_UNIT_WIDE_CONFIGS(X)
#undef X
  return 0;
}

size_t unit_wide_stack_bytes(int m, const Geo& g) {
  const size_t cap = (size_t)g.n * g.gy * g.gx;
  const size_t b = g.bh;
  const size_t s1 = (cap * b * b * m * 2 + 255) / 256 * 256;
  const size_t s2 = (cap * (b - 2) * (b - 2) * m * 2 + 255) / 256 * 256;
  return s1 + s2;
}

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
  const size_t b = g.bh;
  uint8_t* s2 = s1 + ((size_t)cap * b * b * m * 2 + 255) / 256 * 256;
#define X(C_, M_) \
  if (c == C_ && m == M_) return run_wide<C_, M_>(x, out, g, (const uint8_t*)packed, idx, count, cap, s1, s2, s);
  SBN_UNIT_WIDE_CONFIGS(X)
#undef X
  set_error("no wide tcgen05 unit instantiation for c=%d m=%d", c, m);
  return SBN_ERR_UNSUPPORTED;
}

}  // namespace sbn
