// Token construction of Eq.4: the step before the encoder.
//
//   U:  "each feature is naturally converted to individual token with dimension ...
//        Feat_U in R^{N_U x d}"                      -> U rows of X are the given embeddings
//   S:  "Features in S is firstly embedded and concatenated, then a MLP module is adopted for
//        dimension unification", Feat_S_i = MLP(Concat(Emb_s))
//   R:  the real-time items, "similar"
//   C:  "each item I in candidates ... converted to the unified dimension by another MLP",
//        MLP(Concat(Emb_C_i, Emb_I_i))
//   X = Concat([Feat_U, Feat_S, Feat_R, Feat_I]) per user                     (Eq.4)
// Reading R#23: one MLP per item type (S, R, candidates), each
// Linear(k_t -> d) -> SiLU -> Linear(d -> d); inputs are the concatenated feature embeddings
// of each token (k_t wide, from the embedding tables of f4 -- synthetic here), packed per type
// in user-major order.
//
// Forward per type: GEMM (bias + SiLU epilogue, also writing SiLU'), GEMM (+bias), scatter into
// the type's rows of X.  Backward: gather of the type's rows of dX, wgrad / dgrad GEMMs, the
// SiLU' product, bias column sums; optional input gradients (for the embedding tables).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace mtgr {
namespace {

enum { TU = 0, TS = 1, TR = 2, TC = 3 };

__device__ __forceinline__ void type_span(const mtgr_jagged_t& j, const int* n_user, int t, int u,
                                          int& start, int& count) {
  const int nu = n_user[u], ns = j.n_static[u], nr = j.n_rt[u], nc = j.n_cand[u];
  switch (t) {
    case TU: start = 0; count = nu; break;
    case TS: start = nu; count = ns - nu; break;
    case TR: start = ns; count = nr; break;
    default: start = ns + nr; count = nc; break;
  }
}

// toff[t][u] = compact row of user u's first type-t token (exclusive prefix sums); block t
__global__ void token_scan_kernel(mtgr_jagged_t j, const int* n_user, int* toff) {
  __shared__ int wsum[32];
  __shared__ int carry;
  const int t = blockIdx.x;
  int* out = toff + (size_t)t * (j.num_users + 1);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < j.num_users; base += 1024) {
    const int u = base + threadIdx.x;
    int x = 0;
    if (u < j.num_users) { int s; type_span(j, n_user, t, u, s, x); }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      int w = wsum[threadIdx.x];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= o) w += y;
      }
      wsum[threadIdx.x] = w;
    }
    __syncthreads();
    const int incl = carry + x + ((threadIdx.x >> 5) > 0 ? wsum[(threadIdx.x >> 5) - 1] : 0);
    if (u < j.num_users) out[u + 1] = incl;
    if (base == 0 && threadIdx.x == 0) out[0] = 0;
    __syncthreads();
    if (threadIdx.x == 1023) carry = incl;
    __syncthreads();
  }
}

// block per user: the type-t rows of X <-> the compact rows (16-byte moves)
template <class T>
__global__ void token_move_kernel(mtgr_jagged_t j, const int* __restrict__ n_user,
                                  const int* __restrict__ toff, int t, T* __restrict__ x,
                                  T* __restrict__ c, int d, int to_x) {
  const int u = blockIdx.x;
  int start, count;
  type_span(j, n_user, t, u, start, count);
  const int64_t xr = (int64_t)j.offsets[u] + start;
  const int64_t cr = toff[(size_t)t * (j.num_users + 1) + u];
  const int vec = d * (int)sizeof(T) / 16;
  for (int e = threadIdx.x; e < count * vec; e += blockDim.x) {
    const int r = e / vec, k = e % vec;
    uint4* xp = reinterpret_cast<uint4*>(x + (xr + r) * d) + k;
    uint4* cp = reinterpret_cast<uint4*>(c + (cr + r) * d) + k;
    if (to_x) *xp = *cp; else *cp = *xp;
  }
}

// y = a (.) b elementwise over n contiguous values (in place allowed)
template <class T>
__global__ void token_mul_kernel(const T* a, const T* b, T* y, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    y[e] = from_f<T>(to_f(a[e]) * to_f(b[e]));
}

struct TokLayout {
  size_t toff, y, dh, scratch, total;
};

int max_items(const int32_t n_tot[4]) { return std::max(std::max(n_tot[1], n_tot[2]), n_tot[3]); }
int kdim(const mtgr_token_cfg_t* c, int t) { return t == TS ? c->k_s : t == TR ? c->k_r : c->k_c; }

TokLayout tok_layout(const mtgr_token_cfg_t* c, int B, const int32_t n_tot[4], size_t es, bool bf16) {
  TokLayout l{};
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
  const int nmax = max_items(n_tot), d = c->d_model;
  l.toff = take((size_t)4 * (B + 1) * 4);
  l.y = take((size_t)nmax * d * es);
  l.dh = take((size_t)nmax * d * es);
  size_t g = 0;
  for (int t = TS; t <= TC; ++t) {
    g = std::max(g, gemm_ws_bytes(d, d, n_tot[t], EPI_F32, bf16));
    g = std::max(g, gemm_ws_bytes(d, kdim(c, t), n_tot[t], EPI_F32, bf16));
    g = std::max(g, colsum_ws_bytes(n_tot[t], d));
  }
  l.scratch = take(g);
  l.total = off;
  return l;
}

// saved: per type t in S, R, C: H_t and SiLU'(pre_t), [n_t][d] each
size_t saved_off(const mtgr_token_cfg_t* c, const int32_t n_tot[4], size_t es, int t, int which) {
  size_t off = 0;
  for (int s = TS; s <= TC; ++s)
    for (int w = 0; w < 2; ++w) {
      if (s == t && w == which) return off;
      off += align_up((size_t)n_tot[s] * c->d_model * es, 256);
    }
  return off;
}

template <class T>
mtgr_status_t gemm_t(const GemmIO& g, int epi, void* ws, size_t wsb, cudaStream_t st) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) return gemm_bf16_launch(g, epi, ws, wsb, st);
  else return gemm_simt_launch<float>(g, epi, st);
}

const mtgr_mlp_params_t& mlp_of(const mtgr_token_params_t* P, int t) {
  return t == TS ? P->s : t == TR ? P->r : P->c;
}
const mtgr_mlp_grads_t& mlpg_of(const mtgr_token_grads_t* G, int t) {
  return t == TS ? G->s : t == TR ? G->r : G->c;
}

template <class T>
mtgr_status_t token_fwd_t(const mtgr_token_cfg_t* c, const mtgr_jagged_t* j, const int* n_user,
                          const int32_t n_tot[4], const mtgr_token_params_t* P, const T* const feat[4],
                          T* x, char* saved, char* ws, cudaStream_t st) {
  const int d = c->d_model, B = j->num_users;
  const bool bf16 = std::is_same<T, __nv_bfloat16>::value;
  const TokLayout l = tok_layout(c, B, n_tot, sizeof(T), bf16);
  int* toff = (int*)(ws + l.toff);
  T* y = (T*)(ws + l.y);
  void* scratch = ws + l.scratch;
  const size_t sb = l.total - l.scratch;
  {
    ProfScope ps(PROF_TOKEN, st);
    token_scan_kernel<<<4, 1024, 0, st>>>(*j, n_user, toff);
    MTGR_TRY(check_launch("token_scan"));
    if (n_tot[TU] > 0) {
      token_move_kernel<T><<<B, 256, 0, st>>>(*j, n_user, toff, TU, x, const_cast<T*>(feat[TU]), d, 1);
      MTGR_TRY(check_launch("token_move"));
    }
  }
  for (int t = TS; t <= TC; ++t) {
    if (n_tot[t] == 0) continue;
    const mtgr_mlp_params_t& p = mlp_of(P, t);
    T* h = (T*)(saved + saved_off(c, n_tot, sizeof(T), t, 0));
    T* hds = (T*)(saved + saved_off(c, n_tot, sizeof(T), t, 1));
    GemmIO g{};  // H = silu(F W1^T + b1), Hds = silu'(.)
    g.M = n_tot[t]; g.N = d; g.K = kdim(c, t);
    g.A = feat[t]; g.lda = kdim(c, t); g.a_kmajor = 1;
    g.B = p.w1; g.ldb = kdim(c, t); g.b_kmajor = 1;
    g.C = hds; g.ldc = d; g.C2 = h; g.bias = p.b1; g.silu = 1; g.c_dsilu = 1;
    MTGR_TRY(gemm_t<T>(g, EPI_QKVU, scratch, sb, st));
    GemmIO o{};  // Y = H W2^T + b2
    o.M = n_tot[t]; o.N = d; o.K = d;
    o.A = h; o.lda = d; o.a_kmajor = 1;
    o.B = p.w2; o.ldb = d; o.b_kmajor = 1;
    o.C = y; o.ldc = d; o.bias = p.b2;
    MTGR_TRY(gemm_t<T>(o, EPI_STORE, scratch, sb, st));
    ProfScope ps(PROF_TOKEN, st);
    token_move_kernel<T><<<B, 256, 0, st>>>(*j, n_user, toff, t, x, y, d, 1);
    MTGR_TRY(check_launch("token_move"));
  }
  return MTGR_OK;
}

template <class T>
mtgr_status_t token_bwd_t(const mtgr_token_cfg_t* c, const mtgr_jagged_t* j, const int* n_user,
                          const int32_t n_tot[4], const mtgr_token_params_t* P, const T* const feat[4],
                          const char* saved, const T* dx, T* const dfeat[4], const mtgr_token_grads_t* G,
                          char* ws, cudaStream_t st) {
  const int d = c->d_model, B = j->num_users;
  const bool bf16 = std::is_same<T, __nv_bfloat16>::value;
  const TokLayout l = tok_layout(c, B, n_tot, sizeof(T), bf16);
  int* toff = (int*)(ws + l.toff);
  T* dy = (T*)(ws + l.y);
  T* dh = (T*)(ws + l.dh);
  void* scratch = ws + l.scratch;
  const size_t sb = l.total - l.scratch;
  {
    ProfScope ps(PROF_TOKEN, st);
    token_scan_kernel<<<4, 1024, 0, st>>>(*j, n_user, toff);
    MTGR_TRY(check_launch("token_scan"));
    if (n_tot[TU] > 0 && dfeat[TU]) {
      token_move_kernel<T><<<B, 256, 0, st>>>(*j, n_user, toff, TU, const_cast<T*>(dx), dfeat[TU], d, 0);
      MTGR_TRY(check_launch("token_move"));
    }
  }
  for (int t = TS; t <= TC; ++t) {
    const mtgr_mlp_params_t& p = mlp_of(P, t);
    const mtgr_mlp_grads_t& g = mlpg_of(G, t);
    const int k = kdim(c, t), n = n_tot[t];
    if (n == 0) {  // no tokens of this type: zero gradients
      cudaMemsetAsync(g.w1, 0, sizeof(float) * d * k, st);
      cudaMemsetAsync(g.b1, 0, sizeof(float) * d, st);
      cudaMemsetAsync(g.w2, 0, sizeof(float) * d * d, st);
      cudaMemsetAsync(g.b2, 0, sizeof(float) * d, st);
      continue;
    }
    const T* h = (const T*)(saved + saved_off(c, n_tot, sizeof(T), t, 0));
    const T* hds = (const T*)(saved + saved_off(c, n_tot, sizeof(T), t, 1));
    {
      ProfScope ps(PROF_TOKEN, st);
      token_move_kernel<T><<<B, 256, 0, st>>>(*j, n_user, toff, t, const_cast<T*>(dx), dy, d, 0);
      MTGR_TRY(check_launch("token_move"));
    }
    GemmIO w2{};  // dW2 = dY^T H
    w2.M = d; w2.N = d; w2.K = n;
    w2.A = dy; w2.lda = d; w2.a_kmajor = 0;
    w2.B = h; w2.ldb = d; w2.b_kmajor = 0;
    w2.C = g.w2; w2.ldc = d;
    MTGR_TRY(gemm_t<T>(w2, EPI_F32, scratch, sb, st));
    MTGR_TRY(colsum_launch<T>(dy, d, n, d, g.b2, (float*)scratch, 0, st));
    GemmIO a{};  // dH = dY W2, then dPre = dH (.) silu'(pre)
    a.M = n; a.N = d; a.K = d;
    a.A = dy; a.lda = d; a.a_kmajor = 1;
    a.B = p.w2; a.ldb = d; a.b_kmajor = 0;
    a.C = dh; a.ldc = d;
    MTGR_TRY(gemm_t<T>(a, EPI_STORE, scratch, sb, st));
    {
      ProfScope ps(PROF_TOKEN, st);
      const int64_t ne = (int64_t)n * d;
      token_mul_kernel<T><<<(int)std::min<int64_t>(ceil_div64(ne, 256), 1184), 256, 0, st>>>(dh, hds, dh, ne);
      MTGR_TRY(check_launch("token_mul"));
    }
    GemmIO w1{};  // dW1 = dPre^T F
    w1.M = d; w1.N = k; w1.K = n;
    w1.A = dh; w1.lda = d; w1.a_kmajor = 0;
    w1.B = feat[t]; w1.ldb = k; w1.b_kmajor = 0;
    w1.C = g.w1; w1.ldc = k;
    MTGR_TRY(gemm_t<T>(w1, EPI_F32, scratch, sb, st));
    MTGR_TRY(colsum_launch<T>(dh, d, n, d, g.b1, (float*)scratch, 0, st));
    if (dfeat[t]) {  // dF = dPre W1 (for the embedding tables)
      GemmIO f{};
      f.M = n; f.N = k; f.K = d;
      f.A = dh; f.lda = d; f.a_kmajor = 1;
      f.B = p.w1; f.ldb = k; f.b_kmajor = 0;
      f.C = dfeat[t]; f.ldc = k;
      MTGR_TRY(gemm_t<T>(f, EPI_STORE, scratch, sb, st));
    }
  }
  return MTGR_OK;
}

mtgr_status_t check_tok(const mtgr_token_cfg_t* c, const mtgr_jagged_t* j, const int32_t* n_user,
                        const int32_t* n_tot, mtgr_dtype_t dt) {
  MTGR_CHECK(c && j && n_tot, MTGR_E_ARG, "token: null cfg / jagged / n_tot");
  MTGR_CHECK(dt == MTGR_F32 || dt == MTGR_BF16, MTGR_E_DTYPE, "token: dtype must be MTGR_F32 or MTGR_BF16");
  MTGR_CHECK(c->d_model > 0 && c->d_model % 8 == 0 && c->k_s > 0 && c->k_s % 8 == 0 && c->k_r > 0 &&
                 c->k_r % 8 == 0 && c->k_c > 0 && c->k_c % 8 == 0,
             MTGR_E_UNSUPPORTED, "token: d_model and the feature widths must be positive multiples of 8");
  MTGR_CHECK(j->num_users >= 0 && j->total_tokens >= 0, MTGR_E_ARG, "token: bad jagged sizes");
  int64_t sum = 0;
  for (int t = 0; t < 4; ++t) {
    MTGR_CHECK(n_tot[t] >= 0, MTGR_E_ARG, "token: negative n_tot");
    sum += n_tot[t];
  }
  MTGR_CHECK(sum == j->total_tokens, MTGR_E_ARG, "token: n_tot must sum to total_tokens (%lld != %d)",
             (long long)sum, j->total_tokens);
  MTGR_CHECK(j->num_users == 0 || (n_user && j->offsets && j->n_static && j->n_rt && j->n_cand),
             MTGR_E_ARG, "token: jagged metadata or n_user is NULL");
  return MTGR_OK;
}

}  // namespace
}  // namespace mtgr

using namespace mtgr;

MTGR_API size_t mtgr_token_saved_bytes(const mtgr_token_cfg_t* cfg, const int32_t* n_tot, mtgr_dtype_t dtype) {
  if (!cfg || !n_tot) return 0;
  return saved_off(cfg, n_tot, dtype == MTGR_BF16 ? 2 : 4, 4, 0);  // past the last buffer
}

MTGR_API size_t mtgr_token_workspace_bytes(const mtgr_token_cfg_t* cfg, const mtgr_jagged_t* jag,
                                           const int32_t* n_tot, mtgr_dtype_t dtype) {
  if (!cfg || !jag || !n_tot) return 0;
  return tok_layout(cfg, jag->num_users, n_tot, dtype == MTGR_BF16 ? 2 : 4, dtype == MTGR_BF16).total + 256;
}

MTGR_API mtgr_status_t mtgr_token_fwd(const mtgr_token_cfg_t* cfg, const mtgr_jagged_t* jag,
                                      const int32_t* n_user, const int32_t* n_tot, mtgr_dtype_t dtype,
                                      const mtgr_token_params_t* params, const void* feat_u,
                                      const void* feat_s, const void* feat_r, const void* feat_c,
                                      void* x, void* saved, void* ws, size_t ws_bytes,
                                      mtgr_stream_t stream) {
  MTGR_TRY(check_tok(cfg, jag, n_user, n_tot, dtype));
  MTGR_CHECK(ws_bytes >= mtgr_token_workspace_bytes(cfg, jag, n_tot, dtype), MTGR_E_WORKSPACE,
             "token_fwd: workspace too small");
  if (jag->total_tokens == 0) return MTGR_OK;
  MTGR_CHECK(params && x && saved && ws, MTGR_E_ARG, "token_fwd: null pointer");
  const void* f[4] = {feat_u, feat_s, feat_r, feat_c};
  for (int t = 0; t < 4; ++t) {
    MTGR_CHECK(n_tot[t] == 0 || f[t], MTGR_E_ARG, "token_fwd: features of a non-empty type are NULL");
    MTGR_CHECK(!f[t] || aligned16(f[t]), MTGR_E_LAYOUT, "token_fwd: features must be 16-byte aligned");
  }
  MTGR_CHECK(aligned16(x) && aligned16(saved), MTGR_E_LAYOUT, "token_fwd: x / saved must be 16-byte aligned");
  char* w = (char*)ws + ((256 - (reinterpret_cast<uintptr_t>(ws) & 255)) & 255);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == MTGR_BF16) {
    typedef __nv_bfloat16 bf;
    const bf* ff[4] = {(const bf*)feat_u, (const bf*)feat_s, (const bf*)feat_r, (const bf*)feat_c};
    return token_fwd_t<bf>(cfg, jag, n_user, n_tot, params, ff, (bf*)x, (char*)saved, w, st);
  }
  const float* ff[4] = {(const float*)feat_u, (const float*)feat_s, (const float*)feat_r, (const float*)feat_c};
  return token_fwd_t<float>(cfg, jag, n_user, n_tot, params, ff, (float*)x, (char*)saved, w, st);
}

MTGR_API mtgr_status_t mtgr_token_bwd(const mtgr_token_cfg_t* cfg, const mtgr_jagged_t* jag,
                                      const int32_t* n_user, const int32_t* n_tot, mtgr_dtype_t dtype,
                                      const mtgr_token_params_t* params, const void* feat_s,
                                      const void* feat_r, const void* feat_c, const void* saved,
                                      const void* dx, void* dfeat_u, void* dfeat_s, void* dfeat_r,
                                      void* dfeat_c, const mtgr_token_grads_t* grads, void* ws,
                                      size_t ws_bytes, mtgr_stream_t stream) {
  MTGR_TRY(check_tok(cfg, jag, n_user, n_tot, dtype));
  MTGR_CHECK(ws_bytes >= mtgr_token_workspace_bytes(cfg, jag, n_tot, dtype), MTGR_E_WORKSPACE,
             "token_bwd: workspace too small");
  MTGR_CHECK(params && grads && ws, MTGR_E_ARG, "token_bwd: null pointer");
  MTGR_CHECK(jag->total_tokens == 0 || (dx && saved), MTGR_E_ARG, "token_bwd: null dx / saved");
  const void* f[4] = {nullptr, feat_s, feat_r, feat_c};
  for (int t = 1; t < 4; ++t)
    MTGR_CHECK(n_tot[t] == 0 || f[t], MTGR_E_ARG, "token_bwd: features of a non-empty type are NULL");
  char* w = (char*)ws + ((256 - (reinterpret_cast<uintptr_t>(ws) & 255)) & 255);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == MTGR_BF16) {
    typedef __nv_bfloat16 bf;
    const bf* ff[4] = {nullptr, (const bf*)feat_s, (const bf*)feat_r, (const bf*)feat_c};
    bf* df[4] = {(bf*)dfeat_u, (bf*)dfeat_s, (bf*)dfeat_r, (bf*)dfeat_c};
    return token_bwd_t<bf>(cfg, jag, n_user, n_tot, params, ff, (const char*)saved, (const bf*)dx, df,
                           grads, w, st);
  }
  const float* ff[4] = {nullptr, (const float*)feat_s, (const float*)feat_r, (const float*)feat_c};
  float* df[4] = {(float*)dfeat_u, (float*)dfeat_s, (float*)dfeat_r, (float*)dfeat_c};
  return token_bwd_t<float>(cfg, jag, n_user, n_tot, params, ff, (const char*)saved, (const float*)dx, df,
                            grads, w, st);
}
