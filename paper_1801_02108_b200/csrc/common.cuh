// Shared helpers for the sbnet sm_100a kernels: dtype traits, status plumbing,
// device properties, geometry helpers.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <atomic>

#include "../../include/sbnet.h"

namespace sbn {

// ----------------------------------------------------------------- status / errors
void set_error(const char* fmt, ...);
void note_launch(int k = 1);

#define SBN_CHECK_ARG(cond, code, ...)            \
  do {                                            \
    if (!(cond)) {                                \
      ::sbn::set_error(__VA_ARGS__);              \
      return (code);                              \
    }                                             \
  } while (0)

inline int launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SBN_ERR_CUDA;
  }
  note_launch();
  return SBN_OK;
}

// Function attributes (max dynamic smem, carveout, cluster size) are per device: a call
// site sets them the first time it launches on each device.  Setting them twice is
// harmless, so two threads racing on the first launch both set them.
struct PerDeviceOnce {
  std::atomic<unsigned long long> done{0};
  template <typename F>
  void operator()(F&& set_attrs) {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long bit = 1ull << (d & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    set_attrs();
    done.fetch_or(bit, std::memory_order_release);
  }
};

int sm_count();           // SMs of the current device (cached)
int max_smem_optin();     // max dynamic smem per block (cached)

// ----------------------------------------------------------------- dtypes
template <typename T> struct Acc { using type = float; };
template <> struct Acc<double> { using type = double; };

__device__ __forceinline__ float to_acc(float v) { return v; }
__device__ __forceinline__ double to_acc(double v) { return v; }
__device__ __forceinline__ float to_acc(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_acc(float v);
template <> __device__ __forceinline__ float from_acc<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <typename T> __device__ __forceinline__ T from_acc(double v);
template <> __device__ __forceinline__ double from_acc<double>(double v) { return v; }

inline int dtype_size(int dtype) {
  switch (dtype) {
    case SBN_F32: return 4;
    case SBN_F64: return 8;
    case SBN_BF16: return 2;
    default: return 0;
  }
}

// ----------------------------------------------------------------- geometry
struct Geo {
  int n, h, w, bh, bw, sy, sx, oy, ox, gy, gx, obh, obw, oh, ow;
};

inline Geo to_geo(const sbn_geometry* g) {
  return Geo{g->n, g->h, g->w, g->bh, g->bw, g->sy, g->sx, g->oy, g->ox,
             g->gy, g->gx, g->obh, g->obw, g->oh, g->ow};
}

inline int check_geo(const sbn_geometry* g) {
  SBN_CHECK_ARG(g != nullptr, SBN_ERR_INVALID, "geometry is null");
  SBN_CHECK_ARG(g->n >= 0 && g->h > 0 && g->w > 0, SBN_ERR_SHAPE, "bad input dims n=%d h=%d w=%d",
                g->n, g->h, g->w);
  SBN_CHECK_ARG(g->bh > 0 && g->bw > 0 && g->sy > 0 && g->sx > 0, SBN_ERR_INVALID,
                "bad block/in_stride");
  SBN_CHECK_ARG(g->gy > 0 && g->gx > 0 && g->obh > 0 && g->obw > 0 && g->oh > 0 && g->ow > 0,
                SBN_ERR_INVALID, "bad grid/out geometry");
  SBN_CHECK_ARG(g->oy <= 0 && g->ox <= 0, SBN_ERR_INVALID, "grid origin must be <= 0");
  return SBN_OK;
}

// Persistent grid size for a per-block kernel: enough CTAs to fill the device
// `per_sm` deep, never more than the index-list capacity.
inline int persistent_grid(int cap, int per_sm) {
  long g = (long)sm_count() * per_sm;
  if (g > cap) g = cap;
  return g < 1 ? 1 : (int)g;
}

__device__ __forceinline__ int ld_count(const int32_t* count, int cap) {
  int c = __ldg(count);
  return c < cap ? c : cap;
}

// ---- optional phase tracing (diagnostics): kernels record %globaltimer at phase
// boundaries into trace[cta * kTraceSlots + phase] when a buffer has been set with
// sbn_debug_set_trace() (passed to kernels as an argument; null check otherwise).
constexpr int kTraceSlots = 32;
unsigned long long* trace_buffer();  // host side: current buffer or nullptr
int debug_flags();                   // host side: sbn_debug_set_flags()
enum { kDebugNoPair = 1, kDebugConvSingleBuffer = 2, kDebugForceWide = 4, kDebugForceFused = 8, kDebugConvTma = 16,
       kDebugConvPair = 32, kDebugCooperative = 64, kDebugNoGlobalList = 128,
       kDebugWideUnfused = 256, kDebugDenseSingle = 512, kDebugWideNoSplit = 1024, kDebugConvNoRes = 2048,
       kDebugNoEarlyMask = 4096,
       kDebugRowReduceMask = 8192,
       kDebugConvResOneLaunch = 16384,
       kDebugNoMaskPdl = 32768,
       kDebugTmaGlobalList = 65536 };
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace(unsigned long long* tb, int phase) {
  if (tb && threadIdx.x == 0) {
    tb[blockIdx.x * kTraceSlots + phase] = gtimer();
    if (phase == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tb[blockIdx.x * kTraceSlots + 15] = smid;
    }
  }
}

// Forward-progress guard for waits on OTHER CTAs of the same grid (grid barriers, the fused
// unit's list slots and in-place gate).  Such a wait completes only if every CTA it depends
// on is resident; the launchers size these grids to the co-resident capacity of an idle
// GPU, but concurrent work (other streams or processes, MPS clients) can keep part of a
// grid off the SMs.  Instead of hanging, a wait that exceeds kSpinTimeoutNs of %globaltimer
// prints where it stalled and traps: the launch fails with a CUDA error the caller sees at
// its next synchronisation.  Checked every 64 polls (a globaltimer read costs ~a poll).
#ifndef SBN_SPIN_TIMEOUT_NS
#define SBN_SPIN_TIMEOUT_NS 4000000000ull  // 4 s: >> any legitimate wait (us) or context timeslice (ms)
#endif
constexpr unsigned long long kSpinTimeoutNs = SBN_SPIN_TIMEOUT_NS;
enum SpinSite { kSpinGridBarrier = 1, kSpinGridWait = 2, kSpinSlotDone = 3, kSpinSlotStaged = 4, kSpinSlotEntry = 5 };

__device__ unsigned int g_spin_reported = 0u;

struct SpinGuard {
  unsigned long long t0 = 0;
  unsigned polls = 0;
  __device__ __forceinline__ void tick(int site) {
    if ((++polls & 63u) != 0) return;
    const unsigned long long t = gtimer();
    if (t0 == 0) {
      t0 = t;
    } else if (t - t0 > kSpinTimeoutNs) {
      if (atomicExch(&g_spin_reported, 1u) == 0u)  // one report per module load
        printf("sbnet: CTA %d of %d stalled %.1f s at spin site %d (grid not co-resident: concurrent work "
             "holds SMs); aborting the launch\n", (int)blockIdx.x, (int)gridDim.x, (double)(t - t0) * 1e-9, site);
      __trap();
    }
  }
};

// Grid-wide barrier among `expected` co-resident CTAs (caller guarantees residency).
// `bar` = two zero-initialised words in global memory; the last CTA to leave resets
// them, so the same words serve the next launch in the stream.
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int expected) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    SpinGuard sg;
    while (*reinterpret_cast<volatile unsigned int*>(bar) < expected) {
      __nanosleep(64);
      sg.tick(kSpinGridBarrier);
    }
    __threadfence();
    if (atomicAdd(bar + 1, 1u) == expected - 1) {
      bar[0] = 0u;
      bar[1] = 0u;
      __threadfence();
    }
  }
  __syncthreads();
}

// Split-phase grid barrier: arrive right after a CTA's last read of shared global data,
// wait right before its first conflicting write, so the wait overlaps the work between.
__device__ __forceinline__ void grid_arrive(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
  }
}
__device__ __forceinline__ void grid_wait(unsigned int* bar, unsigned int expected) {
  __syncthreads();
  if (threadIdx.x == 0) {
    SpinGuard sg;
    while (*reinterpret_cast<volatile unsigned int*>(bar) < expected) {
      __nanosleep(32);
      sg.tick(kSpinGridWait);
    }
    __threadfence();
    if (atomicAdd(bar + 1, 1u) == expected - 1) {
      bar[0] = 0u;
      bar[1] = 0u;
      __threadfence();
    }
  }
  __syncthreads();
}

}  // namespace sbn
