// TMA tensor-map helpers shared by the TMA-fed kernels (unit_wide.cu, conv_dense_tc.cu).
#pragma once
#include "common.cuh"
#include "tc_util.cuh"

#include <cuda.h>  // CUtensorMap (TMA descriptors)

namespace sbn {

__device__ __forceinline__ void tma_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          tc::smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(tc::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_5d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
          tc::smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(tc::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_2d_cg2(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                           uint32_t rank) {
  uint32_t rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(tc::smem_u32(bar)), "r"(rank));
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          tc::smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(rb)
      : "memory");
}
// CTA-pair form: the box lands in THIS CTA's smem, completion is counted on the mbarrier at
// `bar`'s offset in CTA `rank` of the pair (the MMA issuer's barrier)
__device__ __forceinline__ void tma_5d_cg2(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                           uint64_t* bar, uint32_t rank) {
  uint32_t rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(tc::smem_u32(bar)), "r"(rank));
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
          tc::smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(rb)
      : "memory");
}
// CTA-pair form of tma_4d: lands in THIS CTA's smem, completes on the mbarrier at `bar`'s
// offset in CTA `rank` of the pair
__device__ __forceinline__ void tma_4d_cg2(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                           uint64_t* bar, uint32_t rank) {
  uint32_t rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(tc::smem_u32(bar)), "r"(rank));
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          tc::smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(rb)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          tc::smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(tc::smem_u32(bar))
      : "memory");
}


// TMA descriptor over a bf16 tensor: dims/strides innermost first (strides in bytes, for
// dims 1..rank-1), box in elements, out-of-bounds elements read as zero.
inline int encode_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
               const uint32_t* box, CUtensorMapSwizzle swz, const uint32_t* estride = nullptr) {
  // resolved through the runtime (no link-time libcuda dependency: the library must load
  // on GPU-less build hosts)
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;  // benign race: every thread resolves the same pointer
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return SBN_ERR_CUDA;
    }
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  uint32_t es[5] = {1, 1, 1, 1, 1};
  if (estride)
    for (int i = 0; i < rank; ++i) es[i] = estride[i];
  const CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base),
                                            dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                            swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SBN_ERR_CUDA;
  }
  return SBN_OK;
}

}  // namespace sbn
