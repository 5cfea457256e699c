// tcgen05 jagged HSTU attention (placeholder).
#include "common.cuh"
#include "kernels.h"

namespace mtgr {
bool attn_tc_supported(int dh) { (void)dh; return false; }
mtgr_status_t attn_tc_fwd_launch(const AttnIO& a, cudaStream_t st) { (void)a; (void)st; return set_error(MTGR_E_UNSUPPORTED, "tc attention not built"); }
mtgr_status_t attn_tc_bwd_launch(const AttnIO& a, cudaStream_t st) { (void)a; (void)st; return set_error(MTGR_E_UNSUPPORTED, "tc attention not built"); }
}  // namespace mtgr
