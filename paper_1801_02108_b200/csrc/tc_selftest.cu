// Tensor-core self test: validates the plane-layout UMMA descriptors (row-shifted A
// views, padded plane stride) that the fused kernels rely on.
//   D[128 x 32] (fp32) = A[shift : shift+128, 0:32] @ B[0:32, 0:32]^T   (bf16 inputs)
#include "common.cuh"
#include "tc_util.cuh"

namespace sbn {
namespace {

constexpr int kK = 32, kN = 32;

__global__ void __launch_bounds__(128, 1)
umma_selftest_kernel(const __nv_bfloat16* __restrict__ a, const __nv_bfloat16* __restrict__ b,
                     int rows, int shift, int plane_pad, float* __restrict__ d) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int planeA = rows * 16 + plane_pad;
  uint8_t* sA = smem;
  uint8_t* sB = smem + ((planeA * (kK / 8) + 127) / 128) * 128;
  const int planeB = kN * 16;
  for (int i = threadIdx.x; i < rows * (kK / 8); i += blockDim.x) {
    const int r = i / (kK / 8), k = i % (kK / 8);
    *reinterpret_cast<uint4*>(sA + k * planeA + r * 16) =
        *reinterpret_cast<const uint4*>(a + (size_t)r * kK + k * 8);
  }
  for (int i = threadIdx.x; i < kN * (kK / 8); i += blockDim.x) {
    const int r = i / (kK / 8), k = i % (kK / 8);
    *reinterpret_cast<uint4*>(sB + k * planeB + r * 16) =
        *reinterpret_cast<const uint4*>(b + (size_t)r * kK + k * 8);
  }
  tc::fence_async_smem();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<32>(&tslot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = tc::idesc_bf16_f32(128, kN);
    for (int k = 0; k < kK / 16; ++k) {
      const uint64_t ad = tc::desc_kmajor_noswz(tc::smem_u32(sA + 2 * k * planeA + shift * 16), planeA, 128);
      const uint64_t bd = tc::desc_kmajor_noswz(tc::smem_u32(sB + 2 * k * planeB), planeB, 128);
      tc::mma_bf16(tmem, ad, bd, idesc, k > 0);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < kN; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    for (int j = 0; j < 16; ++j) d[row * kN + c0 + j] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free<32>(tmem);
}

}  // namespace
}  // namespace sbn

using namespace sbn;

extern "C" int sbn_selftest_umma(const void* a, const void* b, int rows, int shift, int plane_pad,
                                 float* d, sbn_stream_t stream) {
  SBN_CHECK_ARG(rows >= 128 + shift && rows % 8 == 0 && shift >= 0, SBN_ERR_INVALID,
                "rows must be >= 128 + shift and a multiple of 8");
  SBN_CHECK_ARG(plane_pad % 16 == 0, SBN_ERR_INVALID, "plane_pad must be a multiple of 16");
  const int planeA = rows * 16 + plane_pad;
  const size_t smem = ((planeA * 4 + 127) / 128) * 128 + kN * 16 * 4;
  cudaFuncSetAttribute(umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  umma_selftest_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)a, (const __nv_bfloat16*)b, rows, shift, plane_pad, d);
  return launch_status("selftest_umma");
}
