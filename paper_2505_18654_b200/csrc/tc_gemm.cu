// tcgen05 bf16 GEMM (placeholder: routes to the SIMT kernel until the tensor-core kernel lands).
#include "common.cuh"
#include "kernels.h"

namespace mtgr {
size_t gemm_ws_bytes(int M, int N, int K, int epi, bool bf16) { (void)M; (void)N; (void)K; (void)epi; (void)bf16; return 0; }
mtgr_status_t gemm_bf16_launch(const GemmIO& g, int epi, void* ws, size_t ws_bytes, cudaStream_t st) {
  (void)ws; (void)ws_bytes;
  return gemm_simt_launch<__nv_bfloat16>(g, epi, st);
}
}  // namespace mtgr
