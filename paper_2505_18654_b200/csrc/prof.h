// Internal tracing hooks (see prof.cu).
#pragma once
#include <atomic>
#include <cuda_runtime.h>

namespace mtgr {

enum ProfKind {
  PROF_GLN_FWD = 0, PROF_GLN_BWD, PROF_GEMM_QKVU, PROF_GEMM_OUT, PROF_GEMM_DGRAD,
  PROF_GEMM_WGRAD, PROF_ATTN_DIAG, PROF_ATTN_FWD, PROF_ATTN_DV, PROF_ATTN_DK, PROF_ATTN_DQ,
  PROF_COLSUM, PROF_OTHER, PROF_HEAD, PROF_TOKEN, PROF_EMBED, PROF_ATTN_SC,
  PROF_ATTN_DK_FUSED, PROF_ATTN_KV, PROF_ATTN_DRAB, PROF_NKINDS
};

void count_launch();

class ProfScope {
 public:
  ProfScope(int kind, cudaStream_t st);
  ~ProfScope();

 private:
  int kind_;
  cudaStream_t st_;
  bool on_;
  bool nv_ = false;  // an NVTX range was pushed (MTGR_NVTX=1)
  cudaEvent_t a_{}, b_{};
};

}  // namespace mtgr
