// Internal launcher declarations of libmtgr (not part of the public ABI).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/mtgr.h"

namespace mtgr {

// ------------------------------------------------------------------ GLN
enum { GLNB_PLAIN = 0, GLNB_GATE = 1, GLNB_RESID = 2 };
struct GlnBwdIO {
  const void* dy; const void* x; const float* mean; const float* rstd; const float* gamma;
  const uint8_t* gid; void* dx; int ntok, d, G;
  const void* o; const void* u; const void* pre_u; int64_t ld_a; void* dpu; int64_t ld_dp;
  const void* dz;
  float* dcol;  // optional fused column sum (red.add): sum_t dz (RESID) or sum_t dp_U (GATE)
  int pre_dsilu;  // pre_u already holds silu'(p_U) (the layer's saved form)
};
size_t gln_bwd_ws_bytes(int ntok, int d, int G);
template <class T>
mtgr_status_t gln_fwd_launch(const T* x, const uint8_t* gid, const float* gamma,
                             const float* beta, T* y, float* mean, float* rstd, int ntok, int d,
                             float eps, cudaStream_t st, const T* gate = nullptr,
                             int64_t ld_gate = 0);
template <class T>
mtgr_status_t gln_bwd_launch(const GlnBwdIO& io, int mode, float* part, float* dgamma,
                             float* dbeta, int accumulate, cudaStream_t st);

// ------------------------------------------------------------------ GEMM
enum { EPI_STORE = 0, EPI_QKVU = 1, EPI_RESID = 2, EPI_F32 = 3 };
struct GemmIO {
  int M, N, K;
  const void* A; int64_t lda; int a_kmajor;
  const void* B; int64_t ldb; int b_kmajor;
  void* C; int64_t ldc;        // EPI_F32: float
  void* C2;                    // EPI_QKVU: activated output (same ld as C)
  const float* bias;           // [N] or NULL
  const void* R; int64_t ldr;  // EPI_RESID residual
  int accumulate;              // EPI_F32
  int silu;                    // EPI_QKVU: 1 = C2 = silu(C), 0 = C2 = C
  int c_dsilu;                 // EPI_QKVU with silu: C receives silu'(pre) instead of pre
};
template <class T>
mtgr_status_t gemm_simt_launch(const GemmIO& g, int epi, cudaStream_t st);
size_t gemm_ws_bytes(int M, int N, int K, int epi, bool bf16);
mtgr_status_t gemm_bf16_launch(const GemmIO& g, int epi, void* ws, size_t ws_bytes,
                               cudaStream_t st);

// ------------------------------------------------------------------ attention
struct AttnIO {
  mtgr_jagged_t jag;
  int causal;                  // mask mode MTGR_MASK_CAUSAL: m_ij = [j <= i] (else dynamic)
  int full;                    // mask mode MTGR_MASK_FULL: m_ij = [j < ns + nr] or [i == j]
  int H, dh, d, nb;            // heads, head dim, d_model, rab buckets (0 = off)
  const void* q; const void* k; const void* v; int64_t ld;
  const void* u;               // gate or NULL
  void* o; void* y;            // fwd outputs [T][d]
  const void* dO;              // bwd input [T][d]
  const void* pre; int64_t ld_pre;  // silu' source (points at Q block) or NULL
  int pre_dsilu;               // pre already holds silu'(p) (the layer's saved form)
  void* dq; void* dk; void* dv; int64_t ld_out;
  const float* diag_a;         // [T][H]  nu*silu(s_ii) for non-static tokens, 0 otherwise
  const float* diag_ds;        // [T][H]  nu*silu'(s_ii)*(dO_i . v_i)
  const float* rab_w; float* drab;
  int diag_cand_only;          // diagonal scalars only for candidate rows (>= ns + nr)
  float* dbias;                // optional: column sums of the (bwd) outputs, red.add into
                               // dbias[col] for the Q|K|V blocks (tensor-core path only)
  void* mm_ws; size_t mm_ws_bytes;  // stored-score backward scratch (attn_store_ws_bytes), or NULL
  int* ctr;                    // >= 8 device ints of workspace: the tensor-core work-queue counters
};
// scratch of the stored-score tensor-core backward for this batch (0: recompute path)
size_t attn_store_ws_bytes(const mtgr_jagged_t& j, int H);
size_t attn_kv_ws_bytes(const mtgr_jagged_t& j, int H);  // coupling workspace of attn_kv_launch
size_t attn_ws_bytes(int ntok, int H);
template <class T>
mtgr_status_t attn_diag_launch(const AttnIO& a, bool bwd, float* diag_a, float* diag_ds,
                               cudaStream_t st);
template <class T>
mtgr_status_t attn_simt_fwd_launch(const AttnIO& a, cudaStream_t st);
template <class T>
mtgr_status_t attn_simt_bwd_launch(const AttnIO& a, cudaStream_t st);
mtgr_status_t attn_tc_fwd_launch(const AttnIO& a, cudaStream_t st);
mtgr_status_t attn_tc_bwd_launch(const AttnIO& a, cudaStream_t st);
bool attn_tc_supported(int dh);

// ------------------------------------------------------------------ misc
template <class T>
mtgr_status_t colsum_launch(const T* X, int64_t ld, int ntok, int n, float* out, float* part,
                            int accumulate, cudaStream_t st);
size_t colsum_ws_bytes(int ntok, int n);
mtgr_status_t scale_launch(float* g, int64_t n, float s, cudaStream_t st);
template <class T>
mtgr_status_t mul_launch(const T* a, const T* b, T* y, int64_t n, cudaStream_t st);  // y = a (.) b
mtgr_status_t gate_mul_launch(const void* o, int64_t ldo, const void* u, int64_t ldu, void* y,
                              int64_t ldy, int ntok, int d, cudaStream_t st);
mtgr_status_t mask_dense_launch(const mtgr_jagged_t& j, int user, uint8_t* out, cudaStream_t st);
mtgr_status_t validate_launch(const mtgr_jagged_t& j, int G, cudaStream_t st);

}  // namespace mtgr

#include <cuda.h>
namespace mtgr {
// 2-D bf16 TMA descriptor: `inner` contiguous elements x `outer` rows (row stride ld_elems),
// box {box_inner, box_outer}, SWIZZLE_128B, zero fill out of bounds.
mtgr_status_t make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                             uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer);
}  // namespace mtgr
