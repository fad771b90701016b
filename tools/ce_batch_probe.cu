// Copy-engine probe for the e2e host-frame path: can the active block windows of a
// config-2 frame (400x400x64 bf16, ~110 16x16 windows in, 14x14 interiors out) cross PCIe
// on the copy engines (cudaMemcpy3DBatchAsync: one 2-D op per window) faster than the
// SM zero-copy kernels?  Prints us/frame and GB/s for H2D alone, D2H alone, both on two
// streams, and the per-op cudaMemcpy2DAsync loop for comparison.
//   nvcc -O2 -o ce_batch_probe tools/ce_batch_probe.cu && ./ce_batch_probe [blocks]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::printf("%s failed: %s (line %d)\n", #x, cudaGetErrorString(e_), __LINE__); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

struct Win { int y, x, h, w; };

static cudaMemcpy3DBatchOp op2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t wbytes,
                               size_t rows) {
  cudaMemcpy3DBatchOp o{};
  o.src.type = cudaMemcpyOperandTypePointer;
  o.src.op.ptr.ptr = const_cast<void*>(src);
  o.src.op.ptr.rowLength = spitch;  // elements of 1 byte
  o.src.op.ptr.layerHeight = 0;
  o.dst.type = cudaMemcpyOperandTypePointer;
  o.dst.op.ptr.ptr = dst;
  o.dst.op.ptr.rowLength = dpitch;
  o.dst.op.ptr.layerHeight = 0;
  o.extent = make_cudaExtent(wbytes, rows, 1);
  o.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  o.flags = cudaMemcpyFlagPreferOverlapWithCompute;
  return o;
}

int main(int argc, char** argv) {
  const int H = 400, W = 400, C = 64, es = 2, B = argc > 1 ? std::atoi(argv[1]) : 110;
  const size_t pitch = (size_t)W * C * es, frame = (size_t)H * pitch;
  void *hin, *hout, *din;
  CK(cudaHostAlloc(&hin, frame, cudaHostAllocDefault));
  CK(cudaHostAlloc(&hout, frame, cudaHostAllocDefault));
  CK(cudaMalloc(&din, frame));
  std::vector<Win> in, out;
  std::srand(1);
  std::vector<int> used(29 * 29, 0);
  while ((int)in.size() < B) {
    const int c = std::rand() % (29 * 29);
    if (used[c]) continue;
    used[c] = 1;
    const int by = c / 29, bx = c % 29;
    int y0 = -1 + 14 * by, x0 = -1 + 14 * bx, y1 = y0 + 16, x1 = x0 + 16;
    y0 = y0 < 0 ? 0 : y0, x0 = x0 < 0 ? 0 : x0, y1 = y1 > H ? H : y1, x1 = x1 > W ? W : x1;
    in.push_back({y0, x0, y1 - y0, x1 - x0});
    int oy = 14 * by, ox = 14 * bx, oy1 = oy + 14 > H ? H : oy + 14, ox1 = ox + 14 > W ? W : ox + 14;
    out.push_back({oy, ox, oy1 - oy, ox1 - ox});
  }
  size_t bin = 0, bout = 0;
  std::vector<cudaMemcpy3DBatchOp> oi, oo;
  for (auto& w : in) {
    const size_t off = (size_t)w.y * pitch + (size_t)w.x * C * es;
    oi.push_back(op2d((char*)din + off, pitch, (char*)hin + off, pitch, (size_t)w.w * C * es, w.h));
    bin += (size_t)w.w * C * es * w.h;
  }
  for (auto& w : out) {
    const size_t off = (size_t)w.y * pitch + (size_t)w.x * C * es;
    oo.push_back(op2d((char*)hout + off, pitch, (char*)din + off, pitch, (size_t)w.w * C * es, w.h));
    bout += (size_t)w.w * C * es * w.h;
  }
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int N = 200;
  auto run = [&](const char* name, bool do_in, bool do_out, bool per_op) {
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0, s1));
      CK(cudaStreamWaitEvent(s2, e0, 0));
      for (int i = 0; i < N; ++i) {
        if (do_in) {
          if (per_op) {
            for (auto& w : in) {
              const size_t off = (size_t)w.y * pitch + (size_t)w.x * C * es;
              CK(cudaMemcpy2DAsync((char*)din + off, pitch, (char*)hin + off, pitch, (size_t)w.w * C * es, w.h,
                                   cudaMemcpyHostToDevice, s1));
            }
          } else {
            size_t fail = 0;
            CK(cudaMemcpy3DBatchAsync(oi.size(), oi.data(), &fail, 0, s1));
          }
        }
        if (do_out) {
          if (per_op) {
            for (auto& w : out) {
              const size_t off = (size_t)w.y * pitch + (size_t)w.x * C * es;
              CK(cudaMemcpy2DAsync((char*)hout + off, pitch, (char*)din + off, pitch, (size_t)w.w * C * es, w.h,
                                   cudaMemcpyDeviceToHost, s2));
            }
          } else {
            size_t fail = 0;
            CK(cudaMemcpy3DBatchAsync(oo.size(), oo.data(), &fail, 0, s2));
          }
        }
      }
      cudaEvent_t j;
      CK(cudaEventCreate(&j));
      CK(cudaEventRecord(j, s2));
      CK(cudaStreamWaitEvent(s1, j, 0));
      CK(cudaEventRecord(e1, s1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double us = ms * 1e3 / N;
      const double bytes = (do_in ? bin : 0) + (do_out ? bout : 0);
      if (rep == 1)
        std::printf("%-34s %8.1f us/frame  %7.1f GB/s  (%zu + %zu bytes)\n", name, us, bytes / us / 1e3,
                    do_in ? bin : (size_t)0, do_out ? bout : (size_t)0);
      CK(cudaEventDestroy(j));
    }
  };
  std::printf("blocks %d\n", B);
  run("batch3D H2D windows", true, false, false);
  run("batch3D D2H interiors", false, true, false);
  run("batch3D both (2 streams)", true, true, false);
  run("memcpy2D per op H2D", true, false, true);
  run("memcpy2D per op both", true, true, true);
  return 0;
}
