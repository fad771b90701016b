// UMMA issue-rate probe: cycles per tcgen05.mma (bf16, M=128, N in {64,128,256}, K=16,
// operands from shared memory) for the SWIZZLE_NONE "plane" K-major layout the row-shift
// kernels use vs the 128-byte-swizzled K-major layout TMA writes, with and without a
// one-row start offset (the row-shift trick).  One CTA per SM, back-to-back MMAs into one
// accumulator, timed with clock64 around issue + commit wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_1801_02108_b200/csrc -o tools/bin/umma_rate tools/umma_rate.cu
#include <cstdio>

#include <cuda_bf16.h>
#include <cstdint>
#include "tc_util.cuh"

using namespace sbn;

// MODE 0: noswz plane layout, 1: noswz + 1-row shift, 2: SW128, 3: SW128 + 8-row shift,
// 4: A SW64 (64-B rows, as the wide unit's IN / fused window chunks of 32 channels) x B plane layout,
// 5: A SW128 x B plane layout
template <int N, int MODE>
__global__ void __launch_bounds__(128, 1) rate_kernel(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* A = smem;                 // up to 64 KB
  uint8_t* B = smem + 64 * 1024;     // up to 64 KB
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&tslot);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = tc::idesc_bf16_f32(128, N);
    const uint32_t a0 = tc::smem_u32(A), b0 = tc::smem_u32(B);
    constexpr uint32_t PA = 200 * 16 + 16;  // plane stride (noswz): 200 rows
    constexpr uint32_t PB = N * 16;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 3;
      uint64_t ad, bd;
      if (MODE <= 1) {
        ad = tc::desc_kmajor_noswz(a0 + 2 * kk * PA + (MODE == 1 ? 16 * (1 + (i % 7)) : 0), PA, 128);
        bd = tc::desc_kmajor_noswz(b0 + 2 * kk * PB, PB, 128);
      } else if (MODE == 4) {
        ad = tc::desc_kmajor_swz(a0 + (kk & 1) * 32, 512, 4);
        bd = tc::desc_kmajor_noswz(b0 + 2 * kk * PB, PB, 128);
      } else if (MODE == 5) {
        ad = tc::desc_kmajor_swz(a0 + kk * 32, 1024, 2);
        bd = tc::desc_kmajor_noswz(b0 + 2 * kk * PB, PB, 128);
      } else {
        ad = tc::desc_kmajor_swz(a0 + kk * 32 + (MODE == 3 ? 1024 : 0), 1024, 2);
        bd = tc::desc_kmajor_swz(b0 + kk * 32, 1024, 2);
      }
      tc::mma_bf16(tmem, ad, bd, idesc, i > 0);
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (threadIdx.x < 32) tc::tmem_free<256>(tmem);
}

// CTA-pair (cta_group::2, M = 256) rate: rank 0 issues; A = 128 rows per CTA, B = N/2 rows per CTA.
// MODE 0: plane layout aligned, 1: plane layout + 1..7-row shift (the 3x3 tap views)
template <int N, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) rate_cg2_kernel(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* A = smem;
  uint8_t* B = smem + 64 * 1024;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  const uint32_t rank = tc::cluster_rank();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc_cg2<256>(&tslot);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0 && rank == 0) {
    constexpr uint32_t idesc = tc::idesc_bf16_f32(256, N);
    const uint32_t a0 = tc::smem_u32(A), b0 = tc::smem_u32(B);
    constexpr uint32_t PA = 200 * 16 + 16;
    constexpr uint32_t PB = (N / 2) * 16;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 3;
      const uint64_t ad = tc::desc_kmajor_noswz(a0 + 2 * kk * PA + (MODE == 1 ? 16 * (1 + (i % 7)) : 0), PA, 128);
      const uint64_t bd = tc::desc_kmajor_noswz(b0 + 2 * kk * PB, PB, 128);
      tc::mma_bf16_cg2(tmem, ad, bd, idesc, i > 0);
    }
    tc::mma_commit_mc(&bar, 3);
    tc::mbar_wait(&bar, 0);
    out[blockIdx.x / 2] = clock64() - t0;
  } else if (threadIdx.x == 0) {
    tc::mbar_wait(&bar, 0);
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after();
  if (threadIdx.x < 32) tc::tmem_free_cg2<256>(tmem);
}

template <int N, int MODE>
void run_cg2(const char* name, int nsm) {
  long long* d;
  cudaMalloc(&d, nsm * sizeof(long long));
  auto k = rate_cg2_kernel<N, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const int iters = 4096;
  k<<<nsm, 128, 128 * 1024>>>(d, iters);
  k<<<nsm, 128, 128 * 1024>>>(d, iters);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, nsm / 2 * sizeof(long long), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < nsm / 2; ++i) m += h[i];
  m /= nsm / 2;
  printf("cg2 M=256 %-24s N=%3d  %6.1f cyc/MMA  %s\n", name, N, m / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

template <int N, int MODE>
void run(const char* name, int nsm) {
  long long* d;
  cudaMalloc(&d, nsm * sizeof(long long));
  auto k = rate_kernel<N, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const int iters = 4096;
  k<<<nsm, 128, 128 * 1024>>>(d, iters);
  k<<<nsm, 128, 128 * 1024>>>(d, iters);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < nsm; ++i) m += h[i];
  m /= nsm;
  const double floor = 128.0 * N / 256.0;
  printf("%-34s N=%3d  %6.1f cyc/MMA  (floor %5.1f, %4.0f%%)  %s\n", name, N, m / iters, floor, 100 * floor / (m / iters),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int nsm = 148;
  run<128, 0>("noswz plane layout", nsm);
  run<128, 1>("noswz + row shift", nsm);
  run<128, 2>("SW128", nsm);
  run<128, 3>("SW128 + 8-row offset", nsm);
  run<64, 0>("noswz plane layout", nsm);
  run<64, 2>("SW128", nsm);
  run<256, 0>("noswz plane layout", nsm);
  run<256, 2>("SW128", nsm);
  run<48, 0>("noswz plane layout", nsm);
  run<48, 1>("noswz + row shift", nsm);
  run<96, 0>("noswz plane layout", nsm);
  run<96, 1>("noswz + row shift", nsm);
  run<64, 1>("noswz + row shift", nsm);
  run<32, 1>("noswz + row shift", nsm);
  run<32, 0>("noswz plane layout", nsm);
  run<32, 2>("SW128", nsm);
  run<48, 4>("A SW64 x B plane", nsm);
  run<48, 5>("A SW128 x B plane", nsm);
  run<96, 4>("A SW64 x B plane", nsm);
  run<96, 5>("A SW128 x B plane", nsm);
  run<32, 5>("A SW128 x B plane", nsm);
  run_cg2<96, 0>("plane aligned", nsm);
  run_cg2<96, 1>("plane + row shift", nsm);
  run_cg2<192, 0>("plane aligned", nsm);
  run_cg2<64, 1>("plane + row shift", nsm);
  run_cg2<128, 1>("plane + row shift", nsm);
  return 0;
}
