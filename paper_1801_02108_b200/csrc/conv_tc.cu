// tcgen05 / TMEM fused sparse conv (bf16) — placeholder until the kernel lands.
#include "common.cuh"
namespace sbn {
bool sparse_conv_tc_supported(int, int, int, int, int, int, int, const Geo&) { return false; }
int sparse_conv_tc(const void*, int, int, Geo, const void*, const void*, const int32_t*,
                   const int32_t*, int, void*, cudaStream_t) {
  set_error("tcgen05 sparse conv not built");
  return SBN_ERR_UNSUPPORTED;
}
}  // namespace sbn
