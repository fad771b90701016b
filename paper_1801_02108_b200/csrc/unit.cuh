// Residual-unit internals shared by the SIMT and tcgen05 paths.
#pragma once
#include "common.cuh"

namespace sbn {

// Halo rim of a unit window: the window pixels outside the block's own output
// (write) region.  For the unit geometry (stride 1, overlap 2*halo) the write region
// is exactly the window interior [halo, bh-halo) x [halo, bw-halo), so a fused
// in-place unit only races on the rim (its neighbours' interiors).  The rim is
// snapshotted before the fused kernel runs; interior pixels are read from x directly.
struct Rim {
  int bh, bw, halo;
  __host__ __device__ int pixels() const { return 2 * halo * bw + 2 * halo * (bh - 2 * halo); }
  __host__ __device__ void coord(int r, int& wy, int& wx) const {
    const int band = halo * bw;
    if (r < band) { wy = r / bw; wx = r - wy * bw; return; }
    r -= band;
    if (r < band) { const int q = r / bw; wy = bh - halo + q; wx = r - q * bw; return; }
    r -= band;
    const int side = 2 * halo;
    const int q = r / side, k = r - q * side;
    wy = halo + q;
    wx = k < halo ? k : bw - side + k;
  }
  __host__ __device__ bool interior(int wy, int wx) const {
    return wy >= halo && wy < bh - halo && wx >= halo && wx < bw - halo;
  }
  __host__ __device__ int index(int wy, int wx) const {
    const int band = halo * bw;
    if (wy < halo) return wy * bw + wx;
    if (wy >= bh - halo) return band + (wy - (bh - halo)) * bw + wx;
    const int side = 2 * halo;
    return 2 * band + (wy - halo) * side + (wx < halo ? wx : wx - (bw - side));
  }
};

// Snapshot the rims of all active blocks of x into rim (cap, P, c).
int unit_rim_snapshot(const void* x, int es, int c, const Geo& g, int halo, const int32_t* idx,
                      const int32_t* count, int cap, void* rim, cudaStream_t s);

template <typename A>
struct UnitFold {
  const A *s1, *t1, *s2, *t2, *s3, *t3;
};

// tcgen05 fast path (unit_tc.cu)
bool unit_tc_supported(int dtype, int c, int m, const Geo& g, int halo, int pre_act);
size_t unit_tc_packed_bytes(int c, int m, const Geo& g);
int unit_tc_pack(const sbn_unit_params* p, int c, int m, const Geo& g, void* img, cudaStream_t s);
int unit_tc_launch(const void* x, void* out, void* rim_buf, unsigned int* gbar, int c, int m,
                   const Geo& g, const sbn_unit_params* p, const void* packed, const int32_t* idx,
                   const int32_t* count, int cap, cudaStream_t s,
                   const uint8_t* mask = nullptr, int32_t* idx_out = nullptr,
                   int32_t* count_out = nullptr, unsigned long long* cst = nullptr,
                   unsigned long long* etag = nullptr, unsigned int* slotw = nullptr);
// wide tcgen05 path (unit_wide.cu): three chained implicit-GEMM launches over the stacked
// active windows, for channel counts whose weights do not fit one CTA's shared memory
bool unit_wide_supported(int dtype, int c, int m, const Geo& g, int halo, int pre_act);
size_t unit_wide_packed_bytes(int c, int m);
// the wide unit runs as ONE launch for this shape (16x16 blocks, buffers fit one CTA)
bool unit_wide_one_launch(int c, int m, const Geo& g);
size_t unit_wide_stack_bytes(int m, const Geo& g);
int unit_wide_pack(const sbn_unit_params* p, int c, int m, void* img, cudaStream_t s);
int unit_wide_launch(const void* x, void* out, int c, int m, const Geo& g, const void* packed,
                     const int32_t* idx, const int32_t* count, int cap, void* stacks, cudaStream_t s);
// epoch compaction handles up to this many mask candidates per CTA (else fused_compact)
constexpr int kEpochMaxPerHost = 1024;
constexpr int kEpochMaxCtas = 4096;

}  // namespace sbn
