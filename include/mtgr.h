/*
 * mtgr.h — C ABI of the B200-native MTGR hot path (libmtgr.so).
 *
 * MTGR: Industrial-Scale Generative Recommendation Framework in Meituan
 * (arXiv 2505.18654).  Citations "P:n" are lines of the paper's LaTeX source
 * (PAPER.md); readings "R#n" are listed in DESIGN.md §2.
 *
 * What is computed: one HSTU encoder layer over user-level-compressed jagged
 * sequences (Eq.3-6), forward and backward, plus the dynamic-BS
 * load balancer and jagged batch builder of §5.
 *
 * Conventions (all entry points):
 *  - Device pointers are caller-owned CUDA device memory; host pointers are
 *    marked "host".  The library never allocates or frees caller memory; GPU
 *    scratch comes from a caller workspace sized by the *_bytes queries.
 *  - Tensors are row-major, token-major: a [T][d] tensor has element (t, c)
 *    at t*ld + c (ld = d unless an ld argument is given).  Token t belongs to
 *    user u iff offsets[u] <= t < offsets[u+1]; within a user the layout is
 *    [static = profile U | lifelong S (n_static) | real-time R (n_rt) |
 *     candidates (n_cand)]  (Eq.3; Eq.4).
 *  - dtype selects the storage type of activations and W1/W2: MTGR_BF16
 *    (tcgen05 tensor-core path, fp32 accumulation) or MTGR_F32 (fp32 SIMT
 *    path, no TF32).  Norm parameters, biases, statistics and all gradients
 *    of parameters are fp32.
 *  - GPU calls are stream-ordered and asynchronous on `stream`; they are
 *    thread-safe across streams.  Host-visible argument checks are
 *    synchronous and return a status; nothing aborts.  Asynchronous CUDA
 *    faults surface as MTGR_E_CUDA at a later call.  mtgr_last_error()
 *    returns a thread-local message for the last failing call.
 *
 * Environment switches (read once per process; in the default build none
 * changes results beyond the floating-point summation order; defaults are the
 * measured-fastest):
 *  - MTGR_ATTN_BWD=kv|stored|fused_dk   bf16 attention backward: the coupled
 *    dK/dV kernel + dQ GEMM (default), the stored-score kernels, or the DK
 *    kernel that writes the scores.  MTGR_ATTN_RECOMPUTE=1 forces the
 *    recompute kernels (otherwise used only when the score scratch would
 *    exceed 48 GB).  MTGR_ATTN_FUSED_DK=0|1: round-1 spelling of the choice.
 *  - MTGR_ROW_CP=0, MTGR_SC_CP=0   row operands into TMEM through registers
 *    instead of tcgen05.cp (A/B only).
 *  - MTGR_KV_NG=n (ring depth, power of two <= 32), MTGR_KV_SLEEP=ns (sync
 *    thread poll period): coupled-kernel tuning knobs.
 *  - MTGR_NVTX=1   an NVTX range around every instrumented kernel launch.
 *  - MTGR_ATTN_TRACE=1, MTGR_KV_TRACE=1 (trace builds), MTGR_KV_DEBUG=bits
 *    (debug builds only: the timing experiments drop work): clock-stamp /
 *    timing-experiment hooks; they synchronise the stream and are not for
 *    production use.
 */
#ifndef MTGR_H_
#define MTGR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* mtgr_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  MTGR_OK = 0,
  MTGR_E_ARG = 1,         /* null pointer / invalid scalar argument                        */
  MTGR_E_SHAPE = 2,       /* d_model % n_heads != 0, sizes inconsistent                    */
  MTGR_E_LAYOUT = 3,      /* pointer or leading dimension not 16-byte aligned              */
  MTGR_E_DTYPE = 4,       /* unknown dtype                                                 */
  MTGR_E_WORKSPACE = 5,   /* workspace / saved buffer smaller than the query says          */
  MTGR_E_BUDGET = 6,      /* a user's cost exceeds the per-rank cap (balancer)             */
  MTGR_E_UNSUPPORTED = 7, /* valid but not implemented (e.g. head dim on the bf16 path)    */
  MTGR_E_CUDA = 8,        /* CUDA launch/runtime error                                     */
  MTGR_E_INVALID = 9      /* mtgr_validate_jagged found inconsistent device metadata       */
} mtgr_status_t;

typedef enum { MTGR_F32 = 0, MTGR_BF16 = 1 } mtgr_dtype_t;

/* Jagged batch metadata.  All pointers are DEVICE memory except where noted. */
typedef struct {
  int32_t num_users;     /* B >= 0 (host scalar)                                             */
  int32_t total_tokens;  /* T = offsets[B] (host scalar)                                     */
  int32_t max_len;       /* >= max_u L_u (host scalar; sizes the launch grids)               */
  const int32_t* offsets;  /* [B+1], offsets[0] = 0, nondecreasing, offsets[B] = T           */
  const int32_t* n_static; /* [B] static tokens n_U + n_S ("static sequence")           */
  const int32_t* n_rt;     /* [B] real-time tokens n_r ("dynamic")                      */
  const int32_t* n_cand;   /* [B] candidates K; n_static + n_rt + n_cand == L_u               */
  const uint8_t* group_id; /* [T] GLN group of each token, < num_groups               */
  const int64_t* ts;       /* [T] seconds; read for real-time and candidate tokens (P:325-337,
                              R#10, R#11); may be NULL iff every n_rt == 0 and rab is off    */
  const float* inv_norm;   /* [B] or NULL.  NULL: 1/N = 1/L_u exactly as Eq.5 (R#3).
                              Non-NULL: caller-fixed normaliser (enables the
                              candidate-removal invariant).                         */
} mtgr_jagged_t;

/* Layer configuration (Table 2; R#5, R#14). */
typedef struct {
  int32_t d_model;     /* d                                                                  */
  int32_t n_heads;     /* H; d_h = d / H                                                     */
  int32_t num_groups;  /* G GLN groups (default 4: profile, lifelong, real-time, candidate)  */
  int32_t rab_buckets; /* 0 = off (Eq.5 exactly).  >0: optional relative-time bias R#4:
                          s_ij += rab_w[h][min(NB-1, floor(log2(max(|ts_i-ts_j|,1))))]        */
  float eps;           /* LayerNorm epsilon (1e-6, R#14)                                     */
  int32_t qkvu_silu;   /* 1: Q,K,V,U = SiLU(X~ W1^T + b1) (R#5); 0: linear                   */
  int32_t mask_mode;   /* MTGR_MASK_DYNAMIC (0): MTGR's dynamic mask (R#8-R#12).
                          MTGR_MASK_CAUSAL (1): the plain causal mask over the packed order,
                          m_ij = [j <= i] (HSTU's) -- the "w/o dynamic mask"
                          ablation of Table 4, read as causal.
                          MTGR_MASK_FULL (2): the same ablation read as full attention
                          (SPEC S:345): m_ij = [j < n_static + n_rt] or [i == j]
                          (every static and real-time token visible to every token,
                          candidates only to themselves).  Other values: MTGR_E_ARG.        */
  int32_t post_mlp_layers; /* "another MLP" above the gate: 0 or 1 = one Linear
                              d->d + b2 (R#6); 2 = Linear(W2,b2) -> SiLU -> Linear(W3,b3)
                              (S:354 reading; the f3 variant).  Other values: MTGR_E_ARG.   */
} mtgr_layer_cfg_t;
enum { MTGR_MASK_DYNAMIC = 0, MTGR_MASK_CAUSAL = 1, MTGR_MASK_FULL = 2 };

/* Parameters of one layer.  W1/W2 have the activation dtype; everything else fp32. */
typedef struct {
  const void* w1;      /* [4d][d]  rows: Q (0..d-1), K, V, U; head h = rows h*d_h.. of each  */
  const float* b1;     /* [4d]                                                               */
  const void* w2;      /* [d][d]   post-gate "MLP" = one Linear (R#6)                         */
  const float* b2;     /* [d]                                                                */
  const float* gamma1; /* [G][d]   GLN1                                               */
  const float* beta1;  /* [G][d]                                                             */
  const float* gamma2; /* [G][d]   GLN2 (Eq.6, R#7)                                    */
  const float* beta2;  /* [G][d]                                                             */
  const float* rab_w;  /* [H][NB] or NULL when rab_buckets == 0                               */
  const void* w3;      /* [d][d] second post-gate Linear (post_mlp_layers == 2), else unused  */
  const float* b3;     /* [d]                                                                */
} mtgr_layer_params_t;

/* Parameter gradients, all fp32, same shapes as mtgr_layer_params_t.  They are SUMS over the
 * batch's tokens (dividing by the global user count is the aggregation step, R#20). */
typedef struct {
  float* w1; float* b1; float* w2; float* b2;
  float* gamma1; float* beta1; float* gamma2; float* beta2;
  float* rab_w; /* may be NULL when rab is off */
  float* w3; float* b3; /* post_mlp_layers == 2 only */
} mtgr_layer_grads_t;

/* ---------------------------------------------------------------- library info */
const char* mtgr_status_str(mtgr_status_t s);
const char* mtgr_last_error(void); /* thread-local message of the last failing call */
int32_t mtgr_version(void);        /* MAJOR*10000 + MINOR*100 + PATCH */

/* ---------------------------------------------------------------- host integer artefacts */

/* Jagged batch builder (user-level sample aggregation, Eq.3; tokens Eq.4).
 * host: seg4 [n][4] = (n_U, n_S, n_r, K) per user of the global batch; users [m] indices into
 * seg4 in the order they are packed (NULL = 0..n-1, m = n).
 * host outputs: offsets [m+1] (exclusive prefix sum of L_u), n_static/n_rt/n_cand [m],
 * group_id [T] (0 = U, 1 = S, 2 = R, 3 = candidate; may be NULL).  Bit-exact with the oracle.
 * Errors: E_ARG (null / negative lengths / index out of range / int32 overflow of T). */
mtgr_status_t mtgr_build_jagged(const int32_t* seg4, int32_t n, const int32_t* users, int32_t m,
                                int32_t* offsets, int32_t* n_static, int32_t* n_rt,
                                int32_t* n_cand, uint8_t* group_id);

/* Dynamic-BS load balancer (R#19): LPT over per-user costs.
 * host: cost [n] (e.g. L_u); world >= 1; cap <= 0 disables the budget check.
 * Users are taken in (cost desc, index asc) order, each placed on the rank with
 * (load asc, rank asc).  host outputs: rank_of [n], load [world].  Bit-exact with the oracle.
 * Errors: E_ARG; E_BUDGET if some cost > cap. */
mtgr_status_t mtgr_balance_lpt(const int64_t* cost, int32_t n, int32_t world, int64_t cap,
                               int32_t* rank_of, int64_t* load);

/* ---------------------------------------------------------------- device checks / exports */

/* Checks device metadata (offsets monotone and ending at T, n_static+n_rt+n_cand == L_u,
 * group_id < num_groups, L_u <= max_len).  Synchronises `stream`.  E_INVALID on failure. */
mtgr_status_t mtgr_validate_jagged(const mtgr_jagged_t* jag, int32_t num_groups,
                                   mtgr_stream_t stream);

/* Dense export of the exact device mask predicate of user `user` (tests, Fig.2(c) P:274,
 * P:335-338): out[i*L_u + j] = 1 iff token i reads token j.  out: device [L_u*L_u] u8, where
 * L_u must be <= max_len.  Reading of the rules: R#8-R#12. */
mtgr_status_t mtgr_mask_dense(const mtgr_jagged_t* jag, int32_t user, uint8_t* out,
                              mtgr_stream_t stream);

/* ---------------------------------------------------------------- Group-Layer Norm */

/* y = gamma[g_t] * (x_t - mean_t) * rstd_t + beta[g_t], rstd = 1/sqrt(var + eps) (biased var).
 * x, y: [T][d] dtype; gamma, beta: [G][d] fp32; mean, rstd: [T] fp32 (may be NULL).
 * d <= 1024 and d % 8 == 0. */
mtgr_status_t mtgr_gln_fwd(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                           mtgr_dtype_t dtype, const void* x, const float* gamma,
                           const float* beta, void* y, float* mean, float* rstd,
                           mtgr_stream_t stream);

/* Backward of mtgr_gln_fwd.  dy, x, dx: [T][d] dtype; mean, rstd from the forward;
 * dgamma, dbeta: [G][d] fp32, OVERWRITTEN with sums over tokens of each group.
 * Workspace: mtgr_gln_bwd_workspace_bytes(). */
size_t mtgr_gln_bwd_workspace_bytes(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag);
mtgr_status_t mtgr_gln_bwd(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                           mtgr_dtype_t dtype, const void* dy, const void* x,
                           const float* mean, const float* rstd, const float* gamma,
                           void* dx, float* dgamma, float* dbeta, void* ws, size_t ws_bytes,
                           mtgr_stream_t stream);

/* ---------------------------------------------------------------- HSTU attention (Eq.5) */

/* Per user u, head h (d_h = d/H), tokens i, j of u:
 *   s_ij = q_i . k_j (+ rab),  A_ij = silu(s_ij) * m_ij / N_u,  o_i = sum_j A_ij v_j
 * with m the dynamic mask (R#8-R#12) and 1/N_u = inv_norm[u] or 1/L_u (R#3).
 * q, k, v, u: [T] rows with leading dimension ld elements (ld % 8 == 0, 16-byte aligned
 * pointers); head h occupies columns [h*d_h, (h+1)*d_h).  o, y: [T][d] (ld d).
 * u == NULL: no gate, y ignored.  Otherwise y = o (.) u (Eq.6 gate).
 * bf16 path: the tcgen05 kernels only, d_h = 256 (Table 2's 512/2 and 768/3), rab
 * on or off (the bias is added to the fp32 scores in TMEM before SiLU); any other bf16 head dim
 * returns MTGR_E_UNSUPPORTED before launching anything (there is no fallback).  fp32 path: SIMT
 * kernels, d_h a multiple of 8 up to 256.
 * Workspace: mtgr_attn_workspace_bytes(). */
size_t mtgr_attn_workspace_bytes(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                 mtgr_dtype_t dtype);
mtgr_status_t mtgr_hstu_attn_fwd(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                 mtgr_dtype_t dtype, const void* q, const void* k,
                                 const void* v, int64_t ld, const void* u,
                                 const float* rab_w, void* o, void* y, void* ws,
                                 size_t ws_bytes, mtgr_stream_t stream);

/* Backward of mtgr_hstu_attn_fwd w.r.t. q, k, v given the PRE-gate dO ([T][d]).
 * dq, dk, dv: rows with leading dimension ld_out.  When silu_pre != NULL (rows with leading
 * dimension ld, same layout as q|k|v), the outputs are multiplied by silu'(pre) of the matching
 * Q/K/V column block (fusing the QKV activation backward, R#5): pre points at the Q block.
 * drab_w: [H][NB] fp32 overwritten, or NULL. */
mtgr_status_t mtgr_hstu_attn_bwd(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                 mtgr_dtype_t dtype, const void* dO, const void* q,
                                 const void* k, const void* v, int64_t ld,
                                 const float* rab_w, const void* silu_pre, void* dq, void* dk,
                                 void* dv, int64_t ld_out, float* drab_w, void* ws,
                                 size_t ws_bytes, mtgr_stream_t stream);

/* ---------------------------------------------------------------- full layer (Eq.5-6) */

/* Forward: X~ = GLN1(x); p = X~ W1^T + b1; [q|k|v|u] = silu(p); o = attn(q,k,v);
 * y = o (.) u; Y~ = GLN2(y); z = Y~ W2^T + b2 + x.
 * x, z: [T][d] dtype (may not alias).  saved: opaque buffer of mtgr_layer_saved_bytes() bytes
 * that the backward reads, or NULL for inference.  ws: at least
 * mtgr_layer_fwd_workspace_bytes(cfg, jag, dtype, saved == NULL) bytes (the forward's own
 * scratch; mtgr_layer_workspace_bytes() covers the forward and the backward, so one workspace
 * serves a training step).  Both depend on num_users and max_len as well as total_tokens. */
size_t mtgr_layer_saved_bytes(const mtgr_layer_cfg_t* cfg, int32_t total_tokens,
                              mtgr_dtype_t dtype);
size_t mtgr_layer_workspace_bytes(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                  mtgr_dtype_t dtype);
size_t mtgr_layer_fwd_workspace_bytes(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                      mtgr_dtype_t dtype, int32_t inference);
mtgr_status_t mtgr_hstu_layer_fwd(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                  mtgr_dtype_t dtype, const mtgr_layer_params_t* params,
                                  const void* x, void* z, void* saved, void* ws,
                                  size_t ws_bytes, mtgr_stream_t stream);

/* Backward: given dz [T][d] and the forward's x and saved buffer, writes dx [T][d] and the
 * parameter gradients (sums over tokens).  accumulate = 0 overwrites grads, 1 adds to them. */
mtgr_status_t mtgr_hstu_layer_bwd(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                  mtgr_dtype_t dtype, const mtgr_layer_params_t* params,
                                  const void* x, const void* saved, const void* dz, void* dx,
                                  const mtgr_layer_grads_t* grads, int32_t accumulate,
                                  void* ws, size_t ws_bytes, mtgr_stream_t stream);

/* ---------------------------------------------------------------- aggregation */

/* g[i] *= scale for n fp32 elements (the 1/B_global step after the all-reduce-sum, R#20). */
mtgr_status_t mtgr_scale_f32(float* g, int64_t n, float scale, mtgr_stream_t stream);

/* ---------------------------------------------------------------- utility GEMM */

/* C = A * B^T (+ epilogue) on the layer's GEMM kernels, exposed for unit tests and tools.
 * A: element (m,k) at a_kmajor ? A[m*lda+k] : A[k*lda+m]; B: (n,k) at b_kmajor ? B[n*ldb+k]
 * : B[k*ldb+n].  C fp32 [M][ldc] when c_f32, else dtype.  bias: [N] fp32 or NULL.
 * accumulate: C += result (fp32 C only). */
mtgr_status_t mtgr_gemm(mtgr_dtype_t dtype, int32_t M, int32_t N, int32_t K, const void* A,
                        int64_t lda, int32_t a_kmajor, const void* B, int64_t ldb,
                        int32_t b_kmajor, void* C, int64_t ldc, int32_t c_f32,
                        const float* bias, int32_t accumulate, void* ws, size_t ws_bytes,
                        mtgr_stream_t stream);
size_t mtgr_gemm_workspace_bytes(mtgr_dtype_t dtype, int32_t M, int32_t N, int32_t K,
                                 int32_t c_f32);

/* ---------------------------------------------------------------- candidate head */

/* Candidate logit head + two-task loss: "the representation of the tokens of candidates are
 * used for logit via another MLP module" (Fig.2(a) caption), tasks CTR and CTCVR.
 * Reading R#21: per candidate row c of the encoder output Z,
 *   h = SiLU(W_a z_c + b_a) (d_hidden),  [l_ctr, l_ctcvr] = W_b h + b_b,
 *   loss[0] = sum_c BCE(l_ctr, click_c),  loss[1] = sum_c BCE(l_ctcvr, click_c AND purchase_c),
 * with BCE(l, y) = softplus(l) - y l.  Losses and gradients are SUMS over the batch's candidates
 * (the 1/B_global scaling is the aggregation step, R#20). */
typedef struct {
  int32_t d_model;   /* d                                                                     */
  int32_t d_hidden;  /* hidden width (d/2); multiple of 8, <= 1024                      */
} mtgr_head_cfg_t;
typedef struct {
  const void* w_a;   /* [d_hidden][d] activation dtype                                        */
  const float* b_a;  /* [d_hidden]                                                             */
  const float* w_b;  /* [2][d_hidden] fp32 (row 0: CTR, row 1: CTCVR)                          */
  const float* b_b;  /* [2]                                                                    */
} mtgr_head_params_t;
typedef struct { float* w_a; float* b_a; float* w_b; float* b_b; } mtgr_head_grads_t; /* fp32 */

size_t mtgr_head_workspace_bytes(const mtgr_head_cfg_t* cfg, const mtgr_jagged_t* jag,
                                 int32_t total_candidates, mtgr_dtype_t dtype);
/* One forward (+ backward) of the head over the jagged batch (DEVICE pointers, stream-ordered).
 *   total_candidates: host-known sum of n_cand (the compact candidate count K).
 *   z:      [T][d] encoder output (dtype); only candidate rows [n_s+n_r, L_u) are read.
 *   labels: [T] uint8, bit 0 = click, bit 1 = purchase; only candidate rows are read.
 *   logits: [K][2] fp32 in candidate order (user-major), or NULL.
 *   loss:   [2] fp32 sums (CTR, CTCVR), or NULL.
 *   dz:     [T][d] (dtype) d(loss[0] + loss[1]) / dz, zero on non-candidate rows; NULL = forward
 *           only (grads ignored).  grads: overwritten fp32 sums.
 * Errors: MTGR_E_ARG (null pointers, K > T), MTGR_E_UNSUPPORTED (dims), MTGR_E_LAYOUT (z / dz not
 * 16-byte aligned), MTGR_E_WORKSPACE.  Deterministic (fixed-order reductions). */
mtgr_status_t mtgr_head_fwd_bwd(const mtgr_head_cfg_t* cfg, const mtgr_jagged_t* jag,
                                int32_t total_candidates, mtgr_dtype_t dtype,
                                const mtgr_head_params_t* params, const void* z,
                                const uint8_t* labels, float* logits, float* loss, void* dz,
                                const mtgr_head_grads_t* grads, void* ws, size_t ws_bytes,
                                mtgr_stream_t stream);

/* ---------------------------------------------------------------- token construction */

/* Eq.4: U tokens are the given d-wide feature embeddings ("each feature is
 * naturally converted to individual token"); every S / R / candidate item token is
 * MLP(Concat(Emb)) of its concatenated feature embeddings.  Reading R#23: one MLP
 * per item type, Linear(k_t -> d) -> SiLU -> Linear(d -> d).  Features are packed per type in
 * user-major order; X rows follow the jagged layout [U | S | R | candidates] of each user. */
typedef struct {
  int32_t d_model;             /* d                                                          */
  int32_t k_s, k_r, k_c;       /* concatenated feature widths of S, R and candidate items   */
} mtgr_token_cfg_t;            /* (all multiples of 8)                                       */
typedef struct {
  const void* w1;  /* [d][k] activation dtype */  const float* b1;  /* [d] */
  const void* w2;  /* [d][d] activation dtype */  const float* b2;  /* [d] */
} mtgr_mlp_params_t;
typedef struct { float* w1; float* b1; float* w2; float* b2; } mtgr_mlp_grads_t; /* fp32 sums */
typedef struct { mtgr_mlp_params_t s, r, c; } mtgr_token_params_t;
typedef struct { mtgr_mlp_grads_t s, r, c; } mtgr_token_grads_t;

/* n_tot: HOST int32[4] = total U, S, R, candidate tokens of the batch (sum == total_tokens). */
size_t mtgr_token_saved_bytes(const mtgr_token_cfg_t* cfg, const int32_t* n_tot, mtgr_dtype_t dtype);
size_t mtgr_token_workspace_bytes(const mtgr_token_cfg_t* cfg, const mtgr_jagged_t* jag,
                                  const int32_t* n_tot, mtgr_dtype_t dtype);
/* X [T][d] <- tokens.  n_user: DEVICE int32 [B] profile tokens per user (the U part of
 * n_static; n_static - n_user are the S tokens).  feat_u [n_U][d], feat_s [n_S][k_s],
 * feat_r [n_R][k_r], feat_c [n_C][k_c] (dtype, device; NULL allowed for an empty type).
 * saved: mtgr_token_saved_bytes, written here and read by the backward.
 * Errors: MTGR_E_ARG (null pointers, n_tot inconsistent with total_tokens), MTGR_E_UNSUPPORTED
 * (widths), MTGR_E_LAYOUT (alignment), MTGR_E_WORKSPACE. */
mtgr_status_t mtgr_token_fwd(const mtgr_token_cfg_t* cfg, const mtgr_jagged_t* jag,
                             const int32_t* n_user, const int32_t* n_tot, mtgr_dtype_t dtype,
                             const mtgr_token_params_t* params, const void* feat_u,
                             const void* feat_s, const void* feat_r, const void* feat_c, void* x,
                             void* saved, void* ws, size_t ws_bytes, mtgr_stream_t stream);
/* Given dX [T][d]: parameter gradients (overwritten fp32 sums) and, when non-NULL, the feature
 * gradients dfeat_* (same shapes as the features; for the embedding tables). */
mtgr_status_t mtgr_token_bwd(const mtgr_token_cfg_t* cfg, const mtgr_jagged_t* jag,
                             const int32_t* n_user, const int32_t* n_tot, mtgr_dtype_t dtype,
                             const mtgr_token_params_t* params, const void* feat_s,
                             const void* feat_r, const void* feat_c, const void* saved,
                             const void* dx, void* dfeat_u, void* dfeat_s, void* dfeat_r,
                             void* dfeat_c, const mtgr_token_grads_t* grads, void* ws,
                             size_t ws_bytes, mtgr_stream_t stream);

/* ---------------------------------------------------------------- hash embedding */

/* Dynamic hash embedding table: a decoupled KEY structure (open addressing, linear
 * probing over cap_k = 2^m buckets of (int64 key, int32 value slot)) and VALUE structure (rows
 * [cap_v][dim] fp32 plus per-slot access counter, last-access timestamp and owning key for
 * eviction).  A missing key gets a value slot (recycled by eviction first, else fresh) whose row
 * is initialised to init_scale * U(-1, 1) from a counter-based hash of (seed, key, column).
 * Expansion replicates only the key structure (mtgr_hash_expand).  Keys INT64_MIN and
 * INT64_MIN+1 are reserved.  All buffers are caller-owned DEVICE memory; every call is
 * stream-ordered (no two calls on one table may run concurrently). */
typedef struct {
  int64_t* keys;       /* [cap_k] key structure                                               */
  int32_t* slots;      /* [cap_k] value slot of each bucket (-1 empty / being published)     */
  int64_t cap_k;       /* power of two; keep the load factor below ~0.7                      */
  float* values;       /* [cap_v][dim] value structure                                        */
  uint32_t* counter;   /* [cap_v] accesses since insertion                                    */
  int64_t* ts;         /* [cap_v] last access time (caller's clock)                           */
  int64_t* slot_key;   /* [cap_v] key owning the slot                                         */
  int64_t cap_v;
  int32_t dim;
  int32_t* alloc;      /* [3]: fresh-slot bump pointer, free-stack size, failed inserts (full) */
  int32_t* free_stack; /* [cap_v] slots returned by eviction                                  */
  uint64_t seed;
  float init_scale;
} mtgr_hash_table_t;

mtgr_status_t mtgr_hash_init(const mtgr_hash_table_t* t, mtgr_stream_t stream);
/* slots[i] = value slot of ids[i]; missing keys are inserted when `insert` (else -1).  -2: the
 * value structure was full (counted in alloc[2]).  Touches counter / ts (= now). */
mtgr_status_t mtgr_hash_find_or_insert(const mtgr_hash_table_t* t, const int64_t* ids, int32_t n,
                                       int64_t now, int32_t insert, int32_t* slots,
                                       mtgr_stream_t stream);
/* out[i][:] = values[slots[i]] (zeros for a negative slot), in dtype. */
mtgr_status_t mtgr_hash_gather(const mtgr_hash_table_t* t, const int32_t* slots, int32_t n,
                               mtgr_dtype_t dtype, void* out, mtgr_stream_t stream);
/* values[slots[i]] -= lr * grads[i] (duplicate slots accumulate). */
mtgr_status_t mtgr_hash_sgd(const mtgr_hash_table_t* t, const int32_t* slots, int32_t n,
                            mtgr_dtype_t dtype, const void* grads, float lr, mtgr_stream_t stream);
/* Evict every key whose last access is < ts_before: bucket -> tombstone, slot -> free stack. */
mtgr_status_t mtgr_hash_evict(const mtgr_hash_table_t* t, int64_t ts_before, mtgr_stream_t stream);
/* Re-insert the live (key, slot) pairs into a new key structure of new_cap_k buckets (the value
 * structure is shared, untouched); the caller then points the table at new_keys / new_slots. */
mtgr_status_t mtgr_hash_expand(const mtgr_hash_table_t* t, int64_t* new_keys, int32_t* new_slots,
                               int64_t new_cap_k, mtgr_stream_t stream);

/* ID unique ("two-stage ID unique"): uniq[0..count) = the distinct ids (order
 * unspecified), inverse[i] = position of ids[i] in uniq; count is a DEVICE int32. */
size_t mtgr_unique_workspace_bytes(int32_t n);
mtgr_status_t mtgr_unique(const int64_t* ids, int32_t n, int64_t* uniq, int32_t* inverse,
                          int32_t* count, void* ws, size_t ws_bytes, mtgr_stream_t stream);
/* out[inverse[i]][:] += g[i][:] over i < n; out [n_out][dim] fp32 is zeroed first. */
mtgr_status_t mtgr_segment_sum(mtgr_dtype_t dtype, const void* g, const int32_t* inverse, int32_t n,
                               int32_t dim, float* out, int32_t n_out, mtgr_stream_t stream);
/* out[i][:] = src[idx[i]][:]. */
mtgr_status_t mtgr_take_rows(mtgr_dtype_t dtype, const void* src, const int32_t* idx, int32_t n,
                             int32_t dim, void* out, mtgr_stream_t stream);
/* out[idx[i]][:] = src[i][:] (idx injective). */
mtgr_status_t mtgr_put_rows(mtgr_dtype_t dtype, const void* src, const int32_t* idx, int32_t n,
                            int32_t dim, void* out, mtgr_stream_t stream);
/* All-to-all packing: dest[i] = owner rank of ids[i] (hash(ids[i] ^ salt) % world), counts[r] =
 * ids owned by r, send = ids grouped by owner (rank-major; order within a rank unspecified),
 * pos[i] = position of ids[i] in send.  starts_ws: DEVICE int32 [2*world] scratch. */
mtgr_status_t mtgr_partition_ids(const int64_t* ids, int32_t n, int32_t world, uint64_t salt,
                                 int32_t* counts, int32_t* dest, int32_t* starts_ws, int64_t* send,
                                 int32_t* pos, mtgr_stream_t stream);

/* ---------------------------------------------------------------- tracing */

/* Number of CUDA kernels libmtgr has launched in this process (all streams). */
int64_t mtgr_launch_count(void);
/* Per-kernel-kind CUDA-event timing: when enabled, each instrumented launch records an event
 * pair on its own stream.  query() synchronises on the recorded events and returns the number
 * of launches and the summed device time (ms) of `kind` since the last reset. */
void mtgr_prof_enable(int32_t on);
void mtgr_prof_reset(void);
int32_t mtgr_prof_num_kinds(void);
const char* mtgr_prof_kind_name(int32_t kind);
mtgr_status_t mtgr_prof_query(int32_t kind, int64_t* launches, double* total_ms);

#ifdef __cplusplus
}
#endif
#endif /* MTGR_H_ */
