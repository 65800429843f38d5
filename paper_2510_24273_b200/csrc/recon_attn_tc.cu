// Fused tcgen05 reconstruct + RoPE + sparse attention (path T).  Placeholder
// until the kernel lands: reports itself unsupported so AUTO picks path S.
#include "recon_attn_tc.h"

namespace sals {
bool tc_supported(int, int, int, int) { return false; }
sals_status launch_recon_attn_tc(const TcArgs&, int, cudaStream_t) { return SALS_ERR_UNSUPPORTED; }
const char* tc_last_error() { return "tcgen05 path not built"; }
}  // namespace sals
