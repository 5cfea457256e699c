// C ABI of libmtgr (include/mtgr.h): argument checks, workspace carving and the orchestration
// of the HSTU layer forward / backward (Eq.5-6) on the caller's stream.
#include <algorithm>
#include <cstdarg>
#include <type_traits>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace mtgr {

static thread_local char g_err[512] = "";

mtgr_status_t set_error(mtgr_status_t s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

mtgr_status_t check_launch(const char* what) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(MTGR_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return MTGR_OK;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  return cache[dev];
}

// ------------------------------------------------------------------ checks
static mtgr_status_t check_cfg(const mtgr_layer_cfg_t* c) {
  MTGR_CHECK(c, MTGR_E_ARG, "cfg is NULL");
  MTGR_CHECK(c->d_model > 0 && c->n_heads > 0 && c->num_groups > 0 && c->num_groups <= 256,
             MTGR_E_ARG, "cfg: d_model, n_heads, num_groups must be positive (num_groups <= 256)");
  MTGR_CHECK(c->d_model % c->n_heads == 0, MTGR_E_SHAPE, "d_model %% n_heads != 0 (S:309)");
  MTGR_CHECK(c->d_model % 8 == 0 && c->d_model <= 1024, MTGR_E_UNSUPPORTED,
             "d_model must be a multiple of 8 and <= 1024");
  const int dh = c->d_model / c->n_heads;
  MTGR_CHECK(dh % 8 == 0 && dh <= 256, MTGR_E_UNSUPPORTED, "head dim %d must be a multiple of 8, <= 256", dh);
  MTGR_CHECK(c->rab_buckets >= 0 && c->rab_buckets <= 64, MTGR_E_ARG, "rab_buckets must be in [0, 64]");
  MTGR_CHECK(c->eps > 0.f, MTGR_E_ARG, "eps must be positive");
  MTGR_CHECK(c->mask_mode == MTGR_MASK_DYNAMIC || c->mask_mode == MTGR_MASK_CAUSAL ||
                 c->mask_mode == MTGR_MASK_FULL,
             MTGR_E_ARG, "mask_mode must be MTGR_MASK_DYNAMIC, MTGR_MASK_CAUSAL or MTGR_MASK_FULL");
  MTGR_CHECK(c->post_mlp_layers >= 0 && c->post_mlp_layers <= 2, MTGR_E_ARG, "post_mlp_layers must be 0, 1 or 2");
  return MTGR_OK;
}

static mtgr_status_t check_jag(const mtgr_jagged_t* j, bool need_groups) {
  MTGR_CHECK(j, MTGR_E_ARG, "jagged metadata is NULL");
  MTGR_CHECK(j->num_users >= 0 && j->total_tokens >= 0 && j->max_len >= 0, MTGR_E_ARG,
             "negative jagged sizes");
  if (j->num_users > 0) {
    MTGR_CHECK(j->offsets && j->n_static && j->n_rt && j->n_cand, MTGR_E_ARG,
               "jagged: offsets / n_static / n_rt / n_cand must be non-NULL");
  }
  if (need_groups && j->total_tokens > 0) MTGR_CHECK(j->group_id, MTGR_E_ARG, "group_id is NULL");
  return MTGR_OK;
}

static mtgr_status_t check_dtype(mtgr_dtype_t d) {
  MTGR_CHECK(d == MTGR_F32 || d == MTGR_BF16, MTGR_E_DTYPE, "unknown dtype %d", (int)d);
  return MTGR_OK;
}
static size_t esize(mtgr_dtype_t d) { return d == MTGR_BF16 ? 2 : 4; }

// ------------------------------------------------------------------ saved-buffer layout
struct SavedLayout {
  size_t xt, p, a, o, yt, mu1, r1, mu2, r2, h, hds, total;
};
// post2: the 2-layer post-gate MLP also saves its hidden activation and SiLU' (R#6 variant)
static SavedLayout saved_layout(int d, int ntok, size_t es, bool post2 = false) {
  SavedLayout s;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
  const size_t T = (size_t)ntok;
  s.xt = take(T * d * es);
  s.p = take(T * 4 * d * es);
  s.a = take(T * 4 * d * es);
  s.o = take(T * d * es);
  s.yt = take(T * d * es);
  s.mu1 = take(T * 4);
  s.r1 = take(T * 4);
  s.mu2 = take(T * 4);
  s.r2 = take(T * 4);
  s.h = post2 ? take(T * d * es) : 0;
  s.hds = post2 ? take(T * d * es) : 0;
  s.total = off;
  return s;
}

// diag_a [T][H] | diag_ds [T][H] | 64 work-queue counters (public attention calls; the layer
// calls carve the same pieces from their own workspace)
size_t attn_ws_bytes(int ntok, int H) { return 2 * align_up((size_t)ntok * H * sizeof(float), 256) + 256; }
static size_t attn_diag_half(int ntok, int H) { return align_up((size_t)ntok * H * sizeof(float), 256); }

static bool tc_attn_path(const mtgr_layer_cfg_t* c, mtgr_dtype_t dt) {
  return dt == MTGR_BF16 && c->n_heads > 0 && attn_tc_supported(c->d_model / c->n_heads);
}

// bf16 attention = the tcgen05 kernels only: head dim 256 (every MTGR config, Table 2);
// the optional rab term (R#4) is added inside them (RAB instantiations)
static mtgr_status_t check_attn_dtype(const mtgr_layer_cfg_t* c, mtgr_dtype_t dt) {
  if (dt != MTGR_BF16) return MTGR_OK;
  MTGR_CHECK(attn_tc_supported(c->d_model / c->n_heads), MTGR_E_UNSUPPORTED,
             "bf16 attention: head dim %d unsupported (the tensor-core kernels need d_h = 256)",
             c->d_model / c->n_heads);
  return MTGR_OK;
}

static size_t bwd_ws_bytes(const mtgr_layer_cfg_t* c, const mtgr_jagged_t* j, mtgr_dtype_t dt) {
  const int ntok = j->total_tokens;
  const size_t es = esize(dt), T = ntok;
  const int d = c->d_model;
  size_t b = 0;
  b += align_up(T * d * es, 256);       // dY~ then dX~
  b += align_up(T * d * es, 256);       // dO
  b += align_up(T * 4 * d * es, 256);   // dp = [dq|dk|dv|du] * silu'(p)
  b += attn_ws_bytes(ntok, c->n_heads);
  size_t g = gln_bwd_ws_bytes(ntok, d, c->num_groups);
  size_t cs = colsum_ws_bytes(ntok, 4 * d);
  size_t gm = std::max(gemm_ws_bytes(4 * d, d, ntok, EPI_F32, dt == MTGR_BF16),
                       gemm_ws_bytes(ntok, d, 4 * d, EPI_STORE, dt == MTGR_BF16));
  const size_t mm = tc_attn_path(c, dt) ? attn_store_ws_bytes(*j, c->n_heads) : 0;
  b += std::max(std::max(std::max(g, cs), gm), mm);
  return b;
}

static size_t fwd_ws_bytes(const mtgr_layer_cfg_t* c, int ntok, mtgr_dtype_t dt, bool inference) {
  size_t b = attn_ws_bytes(ntok, c->n_heads);
  b += std::max(gemm_ws_bytes(ntok, 4 * c->d_model, c->d_model, EPI_QKVU, dt == MTGR_BF16),
                gemm_ws_bytes(ntok, c->d_model, c->d_model, EPI_RESID, dt == MTGR_BF16));
  if (inference) b += saved_layout(c->d_model, ntok, esize(dt), c->post_mlp_layers == 2).total;
  return b;
}

// ------------------------------------------------------------------ dispatch helpers
template <class T>
static mtgr_status_t run_gemm(const GemmIO& g, int epi, void* ws, size_t wsb, cudaStream_t st) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) return gemm_bf16_launch(g, epi, ws, wsb, st);
  else return gemm_simt_launch<float>(g, epi, st);
}

// The bf16 attention runs only on the tensor-core kernels (d_h = 256); the SIMT kernels
// are the fp32 parity path.  There is no dispatch between them: check_attn_dtype rejects every
// other bf16 configuration with MTGR_E_UNSUPPORTED before anything is launched.
template <class T>
static mtgr_status_t run_attn_fwd(const AttnIO& a, float* diag, cudaStream_t st) {
  constexpr bool tc = std::is_same<T, __nv_bfloat16>::value;
  AttnIO b = a;
  b.diag_cand_only = tc;  // the tensor-core path adds real-time diagonals inside its tile loop
  // causal: every diagonal entry is inside the key range of the tile loops (no diagonal terms)
  if (!a.causal) MTGR_TRY(attn_diag_launch<T>(b, false, diag, nullptr, st));
  b.diag_a = diag;
  if constexpr (tc) return attn_tc_fwd_launch(b, st);
  else return attn_simt_fwd_launch<float>(b, st);
}

template <class T>
static mtgr_status_t run_attn_bwd(const AttnIO& a, float* diag_a, float* diag_ds, cudaStream_t st) {
  constexpr bool tc = std::is_same<T, __nv_bfloat16>::value;
  AttnIO b = a;
  b.diag_cand_only = tc;
  if (!a.causal) MTGR_TRY(attn_diag_launch<T>(b, true, diag_a, diag_ds, st));
  b.diag_a = diag_a;
  b.diag_ds = diag_ds;
  if constexpr (tc) return attn_tc_bwd_launch(b, st);
  else return attn_simt_bwd_launch<float>(b, st);
}

// ------------------------------------------------------------------ layer forward
template <class T>
static mtgr_status_t layer_fwd_t(const mtgr_layer_cfg_t* c, const mtgr_jagged_t* j,
                                 const mtgr_layer_params_t* P, const T* x, T* z, char* saved,
                                 char* ws, size_t wsb, cudaStream_t st) {
  const int d = c->d_model, ntok = j->total_tokens;
  const bool post2 = c->post_mlp_layers == 2;
  SavedLayout L = saved_layout(d, ntok, sizeof(T), post2);
  Carve cw(ws, wsb);
  char* sv = saved;
  if (!sv) sv = cw.take<char>(L.total);
  float* diag = cw.take<float>((size_t)ntok * c->n_heads);
  int* ctr = cw.take<int>(64);
  size_t gws_bytes = cw.cap > cw.used ? cw.cap - align_up(cw.used, 256) : 0;
  void* gws = cw.take<char>(0);
  T* xt = (T*)(sv + L.xt); T* p = (T*)(sv + L.p); T* a = (T*)(sv + L.a);
  T* o = (T*)(sv + L.o); T* yt = (T*)(sv + L.yt);
  float* mu1 = (float*)(sv + L.mu1); float* r1 = (float*)(sv + L.r1);
  float* mu2 = (float*)(sv + L.mu2); float* r2 = (float*)(sv + L.r2);
  if (ntok == 0) return MTGR_OK;
  // X~ = GroupLN(X)
  MTGR_TRY(gln_fwd_launch<T>(x, j->group_id, P->gamma1, P->beta1, xt, mu1, r1, ntok, d, c->eps, st));
  // p = X~ W1^T + b1; [Q|K|V|U] = silu(p)  (R#5)
  GemmIO g{};
  g.M = ntok; g.N = 4 * d; g.K = d;
  g.A = xt; g.lda = d; g.a_kmajor = 1;
  g.B = P->w1; g.ldb = d; g.b_kmajor = 1;
  g.C = p; g.ldc = 4 * d; g.C2 = a; g.bias = P->b1; g.silu = c->qkvu_silu;
  g.c_dsilu = 1;  // the backward needs only silu'(p): saved in p's place
  MTGR_TRY(run_gemm<T>(g, EPI_QKVU, gws, gws_bytes, st));
  // O = silu(Q K^T)/N (.) M V  (Eq.5); the gate Y = O (.) U (Eq.6) is formed inside GLN2
  AttnIO at{};
  at.jag = *j; at.causal = c->mask_mode == MTGR_MASK_CAUSAL; at.full = c->mask_mode == MTGR_MASK_FULL; at.H = c->n_heads; at.dh = d / c->n_heads; at.d = d; at.nb = c->rab_buckets;
  at.q = a; at.k = a + d; at.v = a + 2 * d; at.ld = 4 * d;
  at.o = o; at.u = nullptr; at.y = nullptr; at.rab_w = P->rab_w;  // gate folded into GLN2
  at.ctr = ctr;
  MTGR_TRY(run_attn_fwd<T>(at, diag, st));
  // Y~ = GroupLN2(O (.) U)  (Eq.6)
  MTGR_TRY(gln_fwd_launch<T>(o, j->group_id, P->gamma2, P->beta2, yt, mu2, r2, ntok, d, c->eps, st,
                             a + 3 * d, 4 * d));
  if (post2) {  // H = silu(Y~ W2^T + b2) (and SiLU'), Z = H W3^T + b3 + X  (R#6 variant)
    T* hh = (T*)(sv + L.h); T* hds = (T*)(sv + L.hds);
    GemmIO h1{};
    h1.M = ntok; h1.N = d; h1.K = d;
    h1.A = yt; h1.lda = d; h1.a_kmajor = 1;
    h1.B = P->w2; h1.ldb = d; h1.b_kmajor = 1;
    h1.C = hds; h1.ldc = d; h1.C2 = hh; h1.bias = P->b2; h1.silu = 1; h1.c_dsilu = 1;
    MTGR_TRY(run_gemm<T>(h1, EPI_QKVU, gws, gws_bytes, st));
    GemmIO h2{};
    h2.M = ntok; h2.N = d; h2.K = d;
    h2.A = hh; h2.lda = d; h2.a_kmajor = 1;
    h2.B = P->w3; h2.ldb = d; h2.b_kmajor = 1;
    h2.C = z; h2.ldc = d; h2.bias = P->b3; h2.R = x; h2.ldr = d;
    return run_gemm<T>(h2, EPI_RESID, gws, gws_bytes, st);
  }
  // Z = Y~ W2^T + b2 + X  (Eq.6)
  GemmIO h{};
  h.M = ntok; h.N = d; h.K = d;
  h.A = yt; h.lda = d; h.a_kmajor = 1;
  h.B = P->w2; h.ldb = d; h.b_kmajor = 1;
  h.C = z; h.ldc = d; h.bias = P->b2; h.R = x; h.ldr = d;
  return run_gemm<T>(h, EPI_RESID, gws, gws_bytes, st);
}

// ------------------------------------------------------------------ layer backward
template <class T>
static mtgr_status_t layer_bwd_t(const mtgr_layer_cfg_t* c, const mtgr_jagged_t* j,
                                 const mtgr_layer_params_t* P, const T* x, const char* sv,
                                 const T* dz, T* dx, const mtgr_layer_grads_t* G, int acc,
                                 char* ws, size_t wsb, cudaStream_t st) {
  const int d = c->d_model, ntok = j->total_tokens, H = c->n_heads;
  const bool post2 = c->post_mlp_layers == 2;
  SavedLayout L = saved_layout(d, ntok, sizeof(T), post2);
  const T* xt = (const T*)(sv + L.xt); const T* p = (const T*)(sv + L.p);
  const T* a = (const T*)(sv + L.a); const T* o = (const T*)(sv + L.o);
  const T* yt = (const T*)(sv + L.yt);
  const float* mu1 = (const float*)(sv + L.mu1); const float* r1 = (const float*)(sv + L.r1);
  const float* mu2 = (const float*)(sv + L.mu2); const float* r2 = (const float*)(sv + L.r2);
  Carve cw(ws, wsb);
  T* buf = cw.take<T>((size_t)ntok * d);     // dY~, later dX~
  T* dO = cw.take<T>((size_t)ntok * d);
  T* dp = cw.take<T>((size_t)ntok * 4 * d);
  float* diag_a = cw.take<float>((size_t)ntok * H);
  float* diag_ds = cw.take<float>((size_t)ntok * H);
  int* ctr = cw.take<int>(64);
  void* scratch = cw.take<char>(0);
  size_t scratch_bytes = cw.cap > cw.used ? cw.cap - align_up(cw.used, 256) : 0;
  if (c->rab_buckets > 0 && G->rab_w && !acc)
    cudaMemsetAsync(G->rab_w, 0, sizeof(float) * H * c->rab_buckets, st);
  // bias gradients are accumulated by the producing kernels (red.add): start from zero
  if (!acc && ntok > 0) {
    cudaMemsetAsync(G->b1, 0, sizeof(float) * 4 * d, st);
    cudaMemsetAsync(G->b2, 0, sizeof(float) * d, st);
    if (post2) cudaMemsetAsync(G->b3, 0, sizeof(float) * d, st);
  }
  constexpr bool tc_attn = std::is_same<T, __nv_bfloat16>::value;  // check_attn_dtype
  if (ntok == 0) {
    // gradients of an empty batch are zero
    if (!acc) {
      cudaMemsetAsync(G->w1, 0, sizeof(float) * 4 * d * d, st);
      cudaMemsetAsync(G->b1, 0, sizeof(float) * 4 * d, st);
      cudaMemsetAsync(G->w2, 0, sizeof(float) * d * d, st);
      cudaMemsetAsync(G->b2, 0, sizeof(float) * d, st);
      if (post2) {
        cudaMemsetAsync(G->w3, 0, sizeof(float) * d * d, st);
        cudaMemsetAsync(G->b3, 0, sizeof(float) * d, st);
      }
      for (float* q : {G->gamma1, G->beta1, G->gamma2, G->beta2})
        cudaMemsetAsync(q, 0, sizeof(float) * c->num_groups * d, st);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? MTGR_OK : set_error(MTGR_E_CUDA, "layer_bwd: %s", cudaGetErrorString(e));
  }
  if (post2) {
    // Z = H W3^T + b3 + X, H = silu(Y~ W2^T + b2):  dW3 = dZ^T H, db3 = sum dZ (GLN1 backward),
    // dPre = (dZ W3) (.) silu', dW2 = dPre^T Y~, db2 = sum dPre, dY~ = dPre W2.  dPre lives in
    // the dO buffer until the GLN2 backward overwrites it.
    const T* hh = (const T*)(sv + L.h); const T* hds = (const T*)(sv + L.hds);
    GemmIO g3{};
    g3.M = d; g3.N = d; g3.K = ntok;
    g3.A = dz; g3.lda = d; g3.a_kmajor = 0;
    g3.B = hh; g3.ldb = d; g3.b_kmajor = 0;
    g3.C = G->w3; g3.ldc = d; g3.accumulate = acc;
    MTGR_TRY(run_gemm<T>(g3, EPI_F32, scratch, scratch_bytes, st));
    GemmIO h3{};
    h3.M = ntok; h3.N = d; h3.K = d;
    h3.A = dz; h3.lda = d; h3.a_kmajor = 1;
    h3.B = P->w3; h3.ldb = d; h3.b_kmajor = 0;
    h3.C = dO; h3.ldc = d;
    MTGR_TRY(run_gemm<T>(h3, EPI_STORE, scratch, scratch_bytes, st));
    MTGR_TRY(mul_launch<T>(dO, hds, dO, (int64_t)ntok * d, st));
    GemmIO g2{};
    g2.M = d; g2.N = d; g2.K = ntok;
    g2.A = dO; g2.lda = d; g2.a_kmajor = 0;
    g2.B = yt; g2.ldb = d; g2.b_kmajor = 0;
    g2.C = G->w2; g2.ldc = d; g2.accumulate = acc;
    MTGR_TRY(run_gemm<T>(g2, EPI_F32, scratch, scratch_bytes, st));
    MTGR_TRY(colsum_launch<T>(dO, d, ntok, d, G->b2, (float*)scratch, 1, st));
    GemmIO h2{};
    h2.M = ntok; h2.N = d; h2.K = d;
    h2.A = dO; h2.lda = d; h2.a_kmajor = 1;
    h2.B = P->w2; h2.ldb = d; h2.b_kmajor = 0;
    h2.C = buf; h2.ldc = d;
    MTGR_TRY(run_gemm<T>(h2, EPI_STORE, scratch, scratch_bytes, st));
  } else {
  // dW2 = dZ^T Y~, db2 = sum dZ, dY~ = dZ W2
  GemmIO g{};
  g.M = d; g.N = d; g.K = ntok;
  g.A = dz; g.lda = d; g.a_kmajor = 0;
  g.B = yt; g.ldb = d; g.b_kmajor = 0;
  g.C = G->w2; g.ldc = d; g.accumulate = acc;
  MTGR_TRY(run_gemm<T>(g, EPI_F32, scratch, scratch_bytes, st));
  GemmIO h{};
  h.M = ntok; h.N = d; h.K = d;
  h.A = dz; h.lda = d; h.a_kmajor = 1;
  h.B = P->w2; h.ldb = d; h.b_kmajor = 0;
  h.C = buf; h.ldc = d;
  MTGR_TRY(run_gemm<T>(h, EPI_STORE, scratch, scratch_bytes, st));
  }
  // GLN2 backward fused with the gate: dO = dY (.) U, dp_U = dY (.) O (.) silu'(p_U)
  GlnBwdIO gi{};
  gi.dy = buf; gi.x = nullptr;  // norm input x = O (.) U, recomputed from o and u
  gi.mean = mu2; gi.rstd = r2; gi.gamma = P->gamma2; gi.gid = j->group_id;
  gi.dx = dO; gi.ntok = ntok; gi.d = d; gi.G = c->num_groups;
  gi.o = o; gi.u = a + 3 * d; gi.pre_u = c->qkvu_silu ? p + 3 * d : nullptr; gi.pre_dsilu = 1; gi.ld_a = 4 * d;
  gi.dpu = dp + 3 * d; gi.ld_dp = 4 * d; gi.dcol = G->b1 + 3 * d;  // db1 of the U block
  MTGR_TRY(gln_bwd_launch<T>(gi, GLNB_GATE, (float*)scratch, G->gamma2, G->beta2, acc, st));
  // attention backward (+ silu' of Q, K, V) into dp[:, 0:3d]
  AttnIO at{};
  at.jag = *j; at.causal = c->mask_mode == MTGR_MASK_CAUSAL; at.full = c->mask_mode == MTGR_MASK_FULL; at.H = H; at.dh = d / H; at.d = d; at.nb = c->rab_buckets;
  at.q = a; at.k = a + d; at.v = a + 2 * d; at.ld = 4 * d;
  at.dO = dO; at.pre = c->qkvu_silu ? p : nullptr; at.ld_pre = 4 * d; at.pre_dsilu = 1;
  at.dq = dp; at.dk = dp + d; at.dv = dp + 2 * d; at.ld_out = 4 * d;
  at.rab_w = P->rab_w; at.drab = c->rab_buckets > 0 ? G->rab_w : nullptr;
  at.dbias = tc_attn ? G->b1 : nullptr;  // db1 of the Q|K|V blocks fused into the epilogues
  at.mm_ws = scratch; at.mm_ws_bytes = scratch_bytes;  // stored scores (free until the wgrad GEMM)
  at.ctr = ctr;
  MTGR_TRY(run_attn_bwd<T>(at, diag_a, diag_ds, st));
  if (!tc_attn) MTGR_TRY(colsum_launch<T>(dp, 4 * d, ntok, 3 * d, G->b1, (float*)scratch, 1, st));
  // dW1 = dp^T X~, db1 = sum dp, dX~ = dp W1
  GemmIO k{};
  k.M = 4 * d; k.N = d; k.K = ntok;
  k.A = dp; k.lda = 4 * d; k.a_kmajor = 0;
  k.B = xt; k.ldb = d; k.b_kmajor = 0;
  k.C = G->w1; k.ldc = d; k.accumulate = acc;
  MTGR_TRY(run_gemm<T>(k, EPI_F32, scratch, scratch_bytes, st));
  GemmIO m{};
  m.M = ntok; m.N = d; m.K = 4 * d;
  m.A = dp; m.lda = 4 * d; m.a_kmajor = 1;
  m.B = P->w1; m.ldb = d; m.b_kmajor = 0;
  m.C = buf; m.ldc = d;
  MTGR_TRY(run_gemm<T>(m, EPI_STORE, scratch, scratch_bytes, st));
  // GLN1 backward + residual: dX = GLN1_bwd(dX~) + dZ
  GlnBwdIO gj{};
  gj.dy = buf; gj.x = x; gj.mean = mu1; gj.rstd = r1; gj.gamma = P->gamma1; gj.gid = j->group_id;
  gj.dx = dx; gj.ntok = ntok; gj.d = d; gj.G = c->num_groups; gj.dz = dz;
  gj.dcol = post2 ? G->b3 : G->b2;  // the last bias: sum_t dZ fused into the GLN1 backward
  return gln_bwd_launch<T>(gj, GLNB_RESID, (float*)scratch, G->gamma1, G->beta1, acc, st);
}

}  // namespace mtgr

using namespace mtgr;

// ================================================================== exported ABI
MTGR_API const char* mtgr_status_str(mtgr_status_t s) {
  switch (s) {
    case MTGR_OK: return "MTGR_OK";
    case MTGR_E_ARG: return "MTGR_E_ARG";
    case MTGR_E_SHAPE: return "MTGR_E_SHAPE";
    case MTGR_E_LAYOUT: return "MTGR_E_LAYOUT";
    case MTGR_E_DTYPE: return "MTGR_E_DTYPE";
    case MTGR_E_WORKSPACE: return "MTGR_E_WORKSPACE";
    case MTGR_E_BUDGET: return "MTGR_E_BUDGET";
    case MTGR_E_UNSUPPORTED: return "MTGR_E_UNSUPPORTED";
    case MTGR_E_CUDA: return "MTGR_E_CUDA";
    case MTGR_E_INVALID: return "MTGR_E_INVALID";
  }
  return "MTGR_E_?";
}

MTGR_API const char* mtgr_last_error(void) { return g_err; }
MTGR_API int32_t mtgr_version(void) { return 100; }

MTGR_API mtgr_status_t mtgr_validate_jagged(const mtgr_jagged_t* jag, int32_t num_groups,
                                            mtgr_stream_t stream) {
  MTGR_TRY(check_jag(jag, true));
  if (jag->num_users == 0) return MTGR_OK;
  return validate_launch(*jag, num_groups, (cudaStream_t)stream);
}

MTGR_API mtgr_status_t mtgr_mask_dense(const mtgr_jagged_t* jag, int32_t user, uint8_t* out,
                                       mtgr_stream_t stream) {
  MTGR_TRY(check_jag(jag, false));
  MTGR_CHECK(out, MTGR_E_ARG, "out is NULL");
  MTGR_CHECK(user >= 0 && user < jag->num_users, MTGR_E_ARG, "user %d out of range", user);
  return mask_dense_launch(*jag, user, out, (cudaStream_t)stream);
}

MTGR_API mtgr_status_t mtgr_gln_fwd(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                    mtgr_dtype_t dtype, const void* x, const float* gamma,
                                    const float* beta, void* y, float* mean, float* rstd,
                                    mtgr_stream_t stream) {
  MTGR_TRY(check_cfg(cfg));
  MTGR_TRY(check_jag(jag, true));
  MTGR_TRY(check_dtype(dtype));
  if (jag->total_tokens == 0) return MTGR_OK;
  MTGR_CHECK(x && gamma && beta && y, MTGR_E_ARG, "gln_fwd: null pointer");
  MTGR_CHECK(aligned16(x) && aligned16(y) && aligned16(gamma) && aligned16(beta), MTGR_E_LAYOUT,
             "gln_fwd: pointers must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == MTGR_BF16)
    return gln_fwd_launch<__nv_bfloat16>((const __nv_bfloat16*)x, jag->group_id, gamma, beta,
                                         (__nv_bfloat16*)y, mean, rstd, jag->total_tokens,
                                         cfg->d_model, cfg->eps, st);
  return gln_fwd_launch<float>((const float*)x, jag->group_id, gamma, beta, (float*)y, mean, rstd,
                               jag->total_tokens, cfg->d_model, cfg->eps, st);
}

MTGR_API size_t mtgr_gln_bwd_workspace_bytes(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag) {
  if (!cfg || !jag) return 0;
  return gln_bwd_ws_bytes(jag->total_tokens, cfg->d_model, cfg->num_groups);
}

MTGR_API mtgr_status_t mtgr_gln_bwd(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                    mtgr_dtype_t dtype, const void* dy, const void* x,
                                    const float* mean, const float* rstd, const float* gamma,
                                    void* dx, float* dgamma, float* dbeta, void* ws,
                                    size_t ws_bytes, mtgr_stream_t stream) {
  MTGR_TRY(check_cfg(cfg));
  MTGR_TRY(check_jag(jag, true));
  MTGR_TRY(check_dtype(dtype));
  MTGR_CHECK(dgamma && dbeta && ws, MTGR_E_ARG, "gln_bwd: null pointer");
  MTGR_CHECK(ws_bytes >= mtgr_gln_bwd_workspace_bytes(cfg, jag), MTGR_E_WORKSPACE,
             "gln_bwd: workspace too small");
  if (jag->total_tokens > 0) {
    MTGR_CHECK(dy && x && mean && rstd && gamma && dx, MTGR_E_ARG, "gln_bwd: null pointer");
    MTGR_CHECK(aligned16(dy) && aligned16(x) && aligned16(dx) && aligned16(gamma), MTGR_E_LAYOUT,
               "gln_bwd: pointers must be 16-byte aligned");
  }
  GlnBwdIO io{};
  io.dy = dy; io.x = x; io.mean = mean; io.rstd = rstd; io.gamma = gamma; io.gid = jag->group_id;
  io.dx = dx; io.ntok = jag->total_tokens; io.d = cfg->d_model; io.G = cfg->num_groups;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == MTGR_BF16)
    return gln_bwd_launch<__nv_bfloat16>(io, GLNB_PLAIN, (float*)ws, dgamma, dbeta, 0, st);
  return gln_bwd_launch<float>(io, GLNB_PLAIN, (float*)ws, dgamma, dbeta, 0, st);
}

MTGR_API size_t mtgr_attn_workspace_bytes(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                          mtgr_dtype_t dtype) {
  if (!cfg || !jag) return 0;
  const size_t mm = (cfg->n_heads > 0 && tc_attn_path(cfg, dtype)) ? attn_store_ws_bytes(*jag, cfg->n_heads) : 0;
  return attn_ws_bytes(jag->total_tokens, cfg->n_heads) + mm;
}

static mtgr_status_t attn_common_checks(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                        mtgr_dtype_t dtype, int64_t ld, const float* rab_w,
                                        size_t ws_bytes) {
  MTGR_TRY(check_cfg(cfg));
  MTGR_TRY(check_jag(jag, false));
  MTGR_TRY(check_dtype(dtype));
  MTGR_TRY(check_attn_dtype(cfg, dtype));
  MTGR_CHECK(ld >= cfg->d_model && ld % 8 == 0, MTGR_E_LAYOUT, "ld must be >= d_model and a multiple of 8");
  MTGR_CHECK(cfg->rab_buckets == 0 || rab_w, MTGR_E_ARG, "rab on but rab_w is NULL");
  MTGR_CHECK(ws_bytes >= mtgr_attn_workspace_bytes(cfg, jag, dtype), MTGR_E_WORKSPACE,
             "attention workspace too small");
  return MTGR_OK;
}

MTGR_API mtgr_status_t mtgr_hstu_attn_fwd(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                          mtgr_dtype_t dtype, const void* q, const void* k,
                                          const void* v, int64_t ld, const void* u,
                                          const float* rab_w, void* o, void* y, void* ws,
                                          size_t ws_bytes, mtgr_stream_t stream) {
  MTGR_TRY(attn_common_checks(cfg, jag, dtype, ld, rab_w, ws_bytes));
  if (jag->total_tokens == 0) return MTGR_OK;
  MTGR_CHECK(q && k && v && o && ws && (!u || y), MTGR_E_ARG, "attn_fwd: null pointer");
  MTGR_CHECK(aligned16(q) && aligned16(k) && aligned16(v) && aligned16(o) && (!u || aligned16(u)),
             MTGR_E_LAYOUT, "attn_fwd: pointers must be 16-byte aligned");
  AttnIO at{};
  at.jag = *jag; at.causal = cfg->mask_mode == MTGR_MASK_CAUSAL; at.full = cfg->mask_mode == MTGR_MASK_FULL; at.H = cfg->n_heads; at.dh = cfg->d_model / cfg->n_heads; at.d = cfg->d_model;
  at.nb = cfg->rab_buckets; at.q = q; at.k = k; at.v = v; at.ld = ld; at.u = u; at.o = o; at.y = y;
  at.rab_w = rab_w;
  at.ctr = (int*)((char*)ws + 2 * attn_diag_half(jag->total_tokens, cfg->n_heads));
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == MTGR_BF16) return run_attn_fwd<__nv_bfloat16>(at, (float*)ws, st);
  return run_attn_fwd<float>(at, (float*)ws, st);
}

MTGR_API mtgr_status_t mtgr_hstu_attn_bwd(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                          mtgr_dtype_t dtype, const void* dO, const void* q,
                                          const void* k, const void* v, int64_t ld,
                                          const float* rab_w, const void* silu_pre, void* dq,
                                          void* dk, void* dv, int64_t ld_out, float* drab_w,
                                          void* ws, size_t ws_bytes, mtgr_stream_t stream) {
  MTGR_TRY(attn_common_checks(cfg, jag, dtype, ld, rab_w, ws_bytes));
  MTGR_CHECK(ld_out >= cfg->d_model && ld_out % 8 == 0, MTGR_E_LAYOUT, "ld_out invalid");
  cudaStream_t st = (cudaStream_t)stream;
  if (cfg->rab_buckets > 0 && drab_w)
    cudaMemsetAsync(drab_w, 0, sizeof(float) * cfg->n_heads * cfg->rab_buckets, st);
  if (jag->total_tokens == 0) return MTGR_OK;
  MTGR_CHECK(dO && q && k && v && dq && dk && dv && ws, MTGR_E_ARG, "attn_bwd: null pointer");
  MTGR_CHECK(aligned16(dO) && aligned16(q) && aligned16(k) && aligned16(v) && aligned16(dq) &&
                 aligned16(dk) && aligned16(dv),
             MTGR_E_LAYOUT, "attn_bwd: pointers must be 16-byte aligned");
  const size_t half = attn_diag_half(jag->total_tokens, cfg->n_heads);
  AttnIO at{};
  at.jag = *jag; at.causal = cfg->mask_mode == MTGR_MASK_CAUSAL; at.full = cfg->mask_mode == MTGR_MASK_FULL; at.H = cfg->n_heads; at.dh = cfg->d_model / cfg->n_heads; at.d = cfg->d_model;
  at.nb = cfg->rab_buckets; at.q = q; at.k = k; at.v = v; at.ld = ld; at.dO = dO;
  at.pre = silu_pre; at.ld_pre = ld; at.dq = dq; at.dk = dk; at.dv = dv; at.ld_out = ld_out;
  at.rab_w = rab_w; at.drab = drab_w;
  float* da = (float*)ws;
  float* dd = (float*)((char*)ws + half);
  at.ctr = (int*)((char*)ws + 2 * half);
  at.mm_ws = (char*)ws + 2 * half + 256;
  at.mm_ws_bytes = ws_bytes > 2 * half + 256 ? ws_bytes - 2 * half - 256 : 0;
  if (dtype == MTGR_BF16) return run_attn_bwd<__nv_bfloat16>(at, da, dd, st);
  return run_attn_bwd<float>(at, da, dd, st);
}

MTGR_API size_t mtgr_layer_saved_bytes(const mtgr_layer_cfg_t* cfg, int32_t total_tokens,
                                       mtgr_dtype_t dtype) {
  if (!cfg || total_tokens < 0) return 0;
  return saved_layout(cfg->d_model, total_tokens, esize(dtype), cfg->post_mlp_layers == 2).total;
}

MTGR_API size_t mtgr_layer_workspace_bytes(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                           mtgr_dtype_t dtype) {
  if (!cfg || !jag) return 0;
  return std::max(fwd_ws_bytes(cfg, jag->total_tokens, dtype, true),
                  bwd_ws_bytes(cfg, jag, dtype)) + 4096;
}

MTGR_API size_t mtgr_layer_fwd_workspace_bytes(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                               mtgr_dtype_t dtype, int32_t inference) {
  if (!cfg || !jag) return 0;
  return fwd_ws_bytes(cfg, jag->total_tokens, dtype, inference != 0) + 4096;
}

static mtgr_status_t check_params(const mtgr_layer_cfg_t* cfg, const mtgr_layer_params_t* P) {
  MTGR_CHECK(P, MTGR_E_ARG, "params is NULL");
  MTGR_CHECK(P->w1 && P->b1 && P->w2 && P->b2 && P->gamma1 && P->beta1 && P->gamma2 && P->beta2,
             MTGR_E_ARG, "params: null pointer");
  MTGR_CHECK(cfg->rab_buckets == 0 || P->rab_w, MTGR_E_ARG, "params: rab on but rab_w NULL");
  MTGR_CHECK(aligned16(P->w1) && aligned16(P->w2) && aligned16(P->gamma1) && aligned16(P->beta1) &&
                 aligned16(P->gamma2) && aligned16(P->beta2),
             MTGR_E_LAYOUT, "params must be 16-byte aligned");
  return MTGR_OK;
}

MTGR_API mtgr_status_t mtgr_hstu_layer_fwd(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                           mtgr_dtype_t dtype, const mtgr_layer_params_t* params,
                                           const void* x, void* z, void* saved, void* ws,
                                           size_t ws_bytes, mtgr_stream_t stream) {
  MTGR_TRY(check_cfg(cfg));
  MTGR_TRY(check_jag(jag, true));
  MTGR_TRY(check_dtype(dtype));
  MTGR_TRY(check_attn_dtype(cfg, dtype));
  MTGR_TRY(check_params(cfg, params));
  {
    const size_t need = mtgr_layer_fwd_workspace_bytes(cfg, jag, dtype, saved == nullptr);
    MTGR_CHECK(ws_bytes >= need, MTGR_E_WORKSPACE, "layer forward workspace too small (%zu < %zu)", ws_bytes, need);
  }
  if (jag->total_tokens == 0) return MTGR_OK;
  MTGR_CHECK(x && z && ws, MTGR_E_ARG, "layer_fwd: null pointer");
  MTGR_CHECK(x != z, MTGR_E_ARG, "layer_fwd: x and z must not alias");
  MTGR_CHECK(aligned16(x) && aligned16(z) && aligned16(ws) && (!saved || aligned16(saved)),
             MTGR_E_LAYOUT, "layer_fwd: pointers must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == MTGR_BF16)
    return layer_fwd_t<__nv_bfloat16>(cfg, jag, params, (const __nv_bfloat16*)x,
                                      (__nv_bfloat16*)z, (char*)saved, (char*)ws, ws_bytes, st);
  return layer_fwd_t<float>(cfg, jag, params, (const float*)x, (float*)z, (char*)saved,
                            (char*)ws, ws_bytes, st);
}

MTGR_API mtgr_status_t mtgr_hstu_layer_bwd(const mtgr_layer_cfg_t* cfg, const mtgr_jagged_t* jag,
                                           mtgr_dtype_t dtype, const mtgr_layer_params_t* params,
                                           const void* x, const void* saved, const void* dz,
                                           void* dx, const mtgr_layer_grads_t* grads,
                                           int32_t accumulate, void* ws, size_t ws_bytes,
                                           mtgr_stream_t stream) {
  MTGR_TRY(check_cfg(cfg));
  MTGR_TRY(check_jag(jag, true));
  MTGR_TRY(check_dtype(dtype));
  MTGR_TRY(check_attn_dtype(cfg, dtype));
  MTGR_TRY(check_params(cfg, params));
  MTGR_CHECK(grads && grads->w1 && grads->b1 && grads->w2 && grads->b2 && grads->gamma1 &&
                 grads->beta1 && grads->gamma2 && grads->beta2,
             MTGR_E_ARG, "grads: null pointer");
  MTGR_CHECK(ws_bytes >= mtgr_layer_workspace_bytes(cfg, jag, dtype), MTGR_E_WORKSPACE,
             "layer workspace too small");
  MTGR_CHECK(ws, MTGR_E_ARG, "layer_bwd: ws is NULL");
  if (jag->total_tokens > 0) {
    MTGR_CHECK(x && saved && dz && dx, MTGR_E_ARG, "layer_bwd: null pointer");
    MTGR_CHECK(aligned16(x) && aligned16(saved) && aligned16(dz) && aligned16(dx), MTGR_E_LAYOUT,
               "layer_bwd: pointers must be 16-byte aligned");
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == MTGR_BF16)
    return layer_bwd_t<__nv_bfloat16>(cfg, jag, params, (const __nv_bfloat16*)x,
                                      (const char*)saved, (const __nv_bfloat16*)dz,
                                      (__nv_bfloat16*)dx, grads, accumulate, (char*)ws, ws_bytes, st);
  return layer_bwd_t<float>(cfg, jag, params, (const float*)x, (const char*)saved,
                            (const float*)dz, (float*)dx, grads, accumulate, (char*)ws, ws_bytes, st);
}

MTGR_API mtgr_status_t mtgr_scale_f32(float* g, int64_t n, float scale, mtgr_stream_t stream) {
  MTGR_CHECK(n >= 0 && (g || n == 0), MTGR_E_ARG, "scale: invalid arguments");
  return scale_launch(g, n, scale, (cudaStream_t)stream);
}

MTGR_API size_t mtgr_gemm_workspace_bytes(mtgr_dtype_t dtype, int32_t M, int32_t N, int32_t K,
                                          int32_t c_f32) {
  return gemm_ws_bytes(M, N, K, c_f32 ? EPI_F32 : EPI_STORE, dtype == MTGR_BF16);
}

MTGR_API mtgr_status_t mtgr_gemm(mtgr_dtype_t dtype, int32_t M, int32_t N, int32_t K, const void* A,
                                 int64_t lda, int32_t a_kmajor, const void* B, int64_t ldb,
                                 int32_t b_kmajor, void* C, int64_t ldc, int32_t c_f32,
                                 const float* bias, int32_t accumulate, void* ws, size_t ws_bytes,
                                 mtgr_stream_t stream) {
  MTGR_TRY(check_dtype(dtype));
  MTGR_CHECK(M >= 0 && N >= 0 && K >= 0, MTGR_E_ARG, "gemm: negative size");
  if (M == 0 || N == 0) return MTGR_OK;
  MTGR_CHECK(A && B && C, MTGR_E_ARG, "gemm: null pointer");
  MTGR_CHECK(ws_bytes >= mtgr_gemm_workspace_bytes(dtype, M, N, K, c_f32), MTGR_E_WORKSPACE,
             "gemm: workspace too small");
  MTGR_CHECK(!accumulate || c_f32, MTGR_E_ARG, "gemm: accumulate needs an fp32 C");
  GemmIO g{};
  g.M = M; g.N = N; g.K = K; g.A = A; g.lda = lda; g.a_kmajor = a_kmajor; g.B = B; g.ldb = ldb;
  g.b_kmajor = b_kmajor; g.C = C; g.ldc = ldc; g.bias = bias; g.accumulate = accumulate;
  cudaStream_t st = (cudaStream_t)stream;
  const int epi = c_f32 ? EPI_F32 : EPI_STORE;
  if (dtype == MTGR_BF16) return gemm_bf16_launch(g, epi, ws, ws_bytes, st);
  return gemm_simt_launch<float>(g, epi, st);
}
