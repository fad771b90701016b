// tcgen05 / TMEM fused residual unit (bf16) — placeholder until the kernel lands.
#include "unit.cuh"
namespace sbn {
bool unit_tc_supported(int, int, int, const Geo&, int, int) { return false; }
int unit_tc_launch(const void*, void*, const void*, int, int, const Geo&, const sbn_unit_params*,
                   const int32_t*, const int32_t*, int, cudaStream_t) {
  set_error("tcgen05 residual unit not built");
  return SBN_ERR_UNSUPPORTED;
}
}  // namespace sbn
