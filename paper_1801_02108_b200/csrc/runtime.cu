// Library runtime: error strings, device-property cache, launch accounting.
#include "common.cuh"

#include <atomic>
#include <mutex>

namespace sbn {
namespace {
unsigned long long* g_trace = nullptr;
thread_local char g_err[512] = "";
std::atomic<uint64_t> g_launches{0};
constexpr int kMaxDev = 64;
int g_sm[kMaxDev] = {0};
int g_smem[kMaxDev] = {0};
std::mutex g_mu;

int cur_dev() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDev) ? d : 0;
}
}  // namespace

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void note_launch(int k) { g_launches.fetch_add((uint64_t)k, std::memory_order_relaxed); }

int sm_count() {
  const int d = cur_dev();
  if (!g_sm[d]) {
    std::lock_guard<std::mutex> lk(g_mu);
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    g_sm[d] = v > 0 ? v : 1;
  }
  return g_sm[d];
}

int max_smem_optin() {
  const int d = cur_dev();
  if (!g_smem[d]) {
    std::lock_guard<std::mutex> lk(g_mu);
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
    g_smem[d] = v > 0 ? v : 48 * 1024;
  }
  return g_smem[d];
}

unsigned long long* trace_buffer() { return g_trace; }
static int g_flags = 0;
int debug_flags() { return g_flags; }

}  // namespace sbn

extern "C" int sbn_debug_set_flags(int flags) {
  const int old = sbn::g_flags;
  sbn::g_flags = flags;
  return old;
}

extern "C" int sbn_debug_set_trace(unsigned long long* buf) {
  sbn::g_trace = buf;
  return SBN_OK;
}

extern "C" const char* sbn_version(void) { return "sbnet-b200 0.1.0 (sm_100a)"; }
extern "C" const char* sbn_last_error(void) { return sbn::g_err; }
extern "C" uint64_t sbn_launch_count(void) { return sbn::g_launches.load(); }
extern "C" int sbn_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return v;
}
