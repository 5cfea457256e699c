// Candidate logit head and the two-task BCE loss: the step after the encoder.
//
//   "The representation of the tokens of candidates are used for logit via another MLP module"
//   (Fig.2(a) caption); two tasks, CTR and CTCVR.  Reading R#21:
//   the MLP is d -> d_hidden (SiLU) -> 2 (S:358 sizes d_hidden = d/2), one logit per task; the
//   loss is the sum over candidates of BCE-with-logits of click (CTR) and click AND purchase
//   (CTCVR) -- sums, like the layer gradients, so the 1/B scaling stays the aggregation step.
//
// Data path (one call = forward + backward of the head):
//   gather   candidate rows of Z -> Xc [K][d] (user-major), labels -> yc [K]     (head_gather)
//   GEMM     Hds = silu'(Xc Wa^T + ba), H = silu(.)   [K][dh]       (tcgen05 GEMM, QKVU epilogue)
//   rows     l = H Wb^T + bb, BCE, dl = sigmoid(l) - y, dP = (dl Wb) (.) Hds,
//            block partials of dWb, dbb, loss                         (head_logits, warp per row)
//   finish   fixed-order sums of the partials (deterministic)         (head_finish)
//   GEMMs    dWa = dP^T Xc, dXc = dP Wa; dba = column sums of dP
//   scatter  dZ = 0 except candidate rows = dXc                       (head_scatter)
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace mtgr {

namespace {

constexpr int HEAD_WARPS = 8;
constexpr int HEAD_MAX_BLOCKS = 296;
constexpr int HEAD_MAX_DH = 1024;

// coff[u] = sum_{v<u} n_cand[v] (one block, chunks of 1024 users)
__global__ void head_scan_kernel(mtgr_jagged_t j, int* coff) {
  __shared__ int wsum[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < j.num_users; base += 1024) {
    const int u = base + threadIdx.x;
    int x = u < j.num_users ? j.n_cand[u] : 0;
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
    if (u < j.num_users) coff[u + 1] = incl;
    if (base == 0 && threadIdx.x == 0) coff[0] = 0;
    __syncthreads();
    if (threadIdx.x == 1023) carry = incl;
    __syncthreads();
  }
}

// block per user: candidate rows [ns+nr, L) of Z -> Xc[coff[u] ..], labels -> yc (16-byte moves)
template <class T>
__global__ void head_gather_kernel(mtgr_jagged_t j, const int* __restrict__ coff, const T* __restrict__ z,
                                   int d, const uint8_t* __restrict__ labels, T* __restrict__ xc,
                                   uint8_t* __restrict__ yc) {
  const UserSpan us = load_user(j, blockIdx.x);
  const int c0 = us.ns + us.nr, nc = us.L - c0;
  const int dst0 = coff[blockIdx.x];
  const int vec = d * (int)sizeof(T) / 16;  // 16-byte pieces per row
  for (int e = threadIdx.x; e < nc * vec; e += blockDim.x) {
    const int r = e / vec, c = e % vec;
    reinterpret_cast<uint4*>(xc + (int64_t)(dst0 + r) * d)[c] =
        reinterpret_cast<const uint4*>(z + (int64_t)(us.off + c0 + r) * d)[c];
  }
  for (int r = threadIdx.x; r < nc; r += blockDim.x) yc[dst0 + r] = labels[us.off + c0 + r];
}

// warp per candidate row: logits, BCE terms, dl, dP = (dl Wb) (.) silu'(pre); per-block partials
// of dWb [2][dh], dbb [2] and the two loss sums (rows of a block in a fixed order)
template <class T>
__global__ void __launch_bounds__(32 * HEAD_WARPS)
    head_logits_kernel(int K, int dh, const T* __restrict__ hact, const T* __restrict__ hds,
                       const float* __restrict__ wb, const float* __restrict__ bb,
                       const uint8_t* __restrict__ yc, float* __restrict__ logits, T* __restrict__ dp,
                       float* __restrict__ part, int want_grad) {
  extern __shared__ float sred[];  // [HEAD_WARPS][2 * dh + 4]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stride = 2 * dh + 4;
  float* mine = sred + warp * stride;
  for (int c = lane; c < stride; c += 32) mine[c] = 0.f;
  __syncwarp();
  const float b0 = bb[0], b1 = bb[1];
  for (int r = blockIdx.x * HEAD_WARPS + warp; r < K; r += gridDim.x * HEAD_WARPS) {
    const T* h = hact + (int64_t)r * dh;
    float s0 = 0.f, s1 = 0.f;
    for (int c = lane; c < dh; c += 32) {
      const float hv = to_f(h[c]);
      s0 = fmaf(hv, wb[c], s0);
      s1 = fmaf(hv, wb[dh + c], s1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    const float l0 = s0 + b0, l1 = s1 + b1;
    const uint8_t y = yc[r];
    const float y0 = (y & 1u) ? 1.f : 0.f;                 // click
    const float y1 = ((y & 3u) == 3u) ? 1.f : 0.f;         // click and purchase
    // BCE with logits, stable: max(l, 0) - l y + log1p(exp(-|l|))
    const float e0 = fmaxf(l0, 0.f) - l0 * y0 + log1pf(expf(-fabsf(l0)));
    const float e1 = fmaxf(l1, 0.f) - l1 * y1 + log1pf(expf(-fabsf(l1)));
    const float g0 = 1.f / (1.f + expf(-l0)) - y0;
    const float g1 = 1.f / (1.f + expf(-l1)) - y1;
    if (lane == 0) {
      if (logits) { logits[2 * (int64_t)r] = l0; logits[2 * (int64_t)r + 1] = l1; }
      mine[2 * dh] += e0; mine[2 * dh + 1] += e1;
      mine[2 * dh + 2] += g0; mine[2 * dh + 3] += g1;
    }
    if (want_grad) {
      const T* sd = hds + (int64_t)r * dh;
      T* o = dp + (int64_t)r * dh;
      for (int c = lane; c < dh; c += 32) {
        const float hv = to_f(h[c]);
        mine[c] = fmaf(g0, hv, mine[c]);
        mine[dh + c] = fmaf(g1, hv, mine[dh + c]);
        o[c] = from_f<T>(fmaf(g0, wb[c], g1 * wb[dh + c]) * to_f(sd[c]));
      }
    }
    __syncwarp();
  }
  __syncthreads();
  for (int c = threadIdx.x; c < stride; c += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < HEAD_WARPS; ++w) s += sred[w * stride + c];
    part[(int64_t)blockIdx.x * stride + c] = s;
  }
}

// fixed-order reduction of the block partials: loss[2], dWb [2][dh], dbb [2]
__global__ void head_finish_kernel(const float* __restrict__ part, int nblk, int dh, float* loss,
                                   float* dwb, float* dbb) {
  const int stride = 2 * dh + 4;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < stride; c += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * stride + c];
    if (c < 2 * dh) { if (dwb) dwb[c] = s; }
    else if (c < 2 * dh + 2) { if (loss) loss[c - 2 * dh] = s; }
    else if (dbb) dbb[c - 2 * dh - 2] = s;
  }
}

// block per user: dZ candidate rows <- dXc (the other rows were zeroed)
template <class T>
__global__ void head_scatter_kernel(mtgr_jagged_t j, const int* __restrict__ coff, const T* __restrict__ dxc,
                                    int d, T* __restrict__ dz) {
  const UserSpan us = load_user(j, blockIdx.x);
  const int c0 = us.ns + us.nr, nc = us.L - c0;
  const int src0 = coff[blockIdx.x];
  const int vec = d * (int)sizeof(T) / 16;
  for (int e = threadIdx.x; e < nc * vec; e += blockDim.x) {
    const int r = e / vec, c = e % vec;
    reinterpret_cast<uint4*>(dz + (int64_t)(us.off + c0 + r) * d)[c] =
        reinterpret_cast<const uint4*>(dxc + (int64_t)(src0 + r) * d)[c];
  }
}

struct HeadLayout {
  size_t coff, xc, yc, hds, hact, dp, dxc, part, scratch, total;
  int nblk;
};

HeadLayout head_layout(const mtgr_head_cfg_t* c, int K, int B, size_t es, bool bf16) {
  HeadLayout l{};
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
  l.nblk = std::max(1, std::min(HEAD_MAX_BLOCKS, ceil_div(std::max(K, 1), HEAD_WARPS)));
  l.coff = take((size_t)(B + 1) * 4);
  l.xc = take((size_t)K * c->d_model * es);
  l.yc = take((size_t)K);
  l.hds = take((size_t)K * c->d_hidden * es);
  l.hact = take((size_t)K * c->d_hidden * es);
  l.dp = take((size_t)K * c->d_hidden * es);
  l.dxc = take((size_t)K * c->d_model * es);
  l.part = take((size_t)l.nblk * (2 * c->d_hidden + 4) * 4);
  const size_t g = std::max(gemm_ws_bytes(c->d_hidden, c->d_model, K, EPI_F32, bf16),
                            colsum_ws_bytes(K, c->d_hidden));
  l.scratch = take(g);
  l.total = off;
  return l;
}

template <class T>
mtgr_status_t gemm_any(const GemmIO& g, int epi, void* ws, size_t wsb, cudaStream_t st) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) return gemm_bf16_launch(g, epi, ws, wsb, st);
  else return gemm_simt_launch<float>(g, epi, st);
}

template <class T>
mtgr_status_t head_run(const mtgr_head_cfg_t* c, const mtgr_jagged_t* j, int K,
                       const mtgr_head_params_t* P, const T* z, const uint8_t* labels, float* logits,
                       float* loss, T* dz, const mtgr_head_grads_t* G, char* ws, cudaStream_t st) {
  const int d = c->d_model, dh = c->d_hidden, B = j->num_users;
  const bool bf16 = std::is_same<T, __nv_bfloat16>::value;
  const HeadLayout l = head_layout(c, K, B, sizeof(T), bf16);
  int* coff = (int*)(ws + l.coff);
  T* xc = (T*)(ws + l.xc);
  uint8_t* yc = (uint8_t*)(ws + l.yc);
  T* hds = (T*)(ws + l.hds);
  T* hact = (T*)(ws + l.hact);
  T* dp = (T*)(ws + l.dp);
  T* dxc = (T*)(ws + l.dxc);
  float* part = (float*)(ws + l.part);
  void* scratch = ws + l.scratch;
  const size_t scratch_bytes = l.total - l.scratch;
  const bool grad = dz != nullptr;
  if (grad && j->total_tokens > 0) cudaMemsetAsync(dz, 0, (size_t)j->total_tokens * d * sizeof(T), st);
  if (K == 0) {  // no candidates: zero loss and gradients
    if (loss) cudaMemsetAsync(loss, 0, 2 * sizeof(float), st);
    if (grad) {
      cudaMemsetAsync(G->w_a, 0, sizeof(float) * dh * d, st);
      cudaMemsetAsync(G->b_a, 0, sizeof(float) * dh, st);
      cudaMemsetAsync(G->w_b, 0, sizeof(float) * 2 * dh, st);
      cudaMemsetAsync(G->b_b, 0, sizeof(float) * 2, st);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? MTGR_OK : set_error(MTGR_E_CUDA, "head: %s", cudaGetErrorString(e));
  }
  {
    ProfScope ps(PROF_HEAD, st);
    head_scan_kernel<<<1, 1024, 0, st>>>(*j, coff);
    MTGR_TRY(check_launch("head_scan"));
    head_gather_kernel<T><<<B, 256, 0, st>>>(*j, coff, z, d, labels, xc, yc);
    MTGR_TRY(check_launch("head_gather"));
  }
  // H = silu(Xc Wa^T + ba), Hds = silu'(Xc Wa^T + ba)
  GemmIO g{};
  g.M = K; g.N = dh; g.K = d;
  g.A = xc; g.lda = d; g.a_kmajor = 1;
  g.B = P->w_a; g.ldb = d; g.b_kmajor = 1;
  g.C = hds; g.ldc = dh; g.C2 = hact; g.bias = P->b_a; g.silu = 1; g.c_dsilu = 1;
  MTGR_TRY(gemm_any<T>(g, EPI_QKVU, scratch, scratch_bytes, st));
  {
    ProfScope ps(PROF_HEAD, st);
    const size_t smem = (size_t)HEAD_WARPS * (2 * dh + 4) * sizeof(float);
    cudaFuncSetAttribute(head_logits_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    head_logits_kernel<T><<<l.nblk, 32 * HEAD_WARPS, smem, st>>>(K, dh, hact, hds, P->w_b, P->b_b, yc,
                                                                   logits, dp, part, grad ? 1 : 0);
    MTGR_TRY(check_launch("head_logits"));
    head_finish_kernel<<<ceil_div(2 * dh + 4, 256), 256, 0, st>>>(part, l.nblk, dh, loss,
                                                                    grad ? G->w_b : nullptr,
                                                                    grad ? G->b_b : nullptr);
    MTGR_TRY(check_launch("head_finish"));
  }
  if (!grad) return MTGR_OK;
  // dWa = dP^T Xc, dba = sum dP, dXc = dP Wa
  GemmIO w{};
  w.M = dh; w.N = d; w.K = K;
  w.A = dp; w.lda = dh; w.a_kmajor = 0;
  w.B = xc; w.ldb = d; w.b_kmajor = 0;
  w.C = G->w_a; w.ldc = d; w.accumulate = 0;
  MTGR_TRY(gemm_any<T>(w, EPI_F32, scratch, scratch_bytes, st));
  MTGR_TRY(colsum_launch<T>(dp, dh, K, dh, G->b_a, (float*)scratch, 0, st));
  GemmIO x{};
  x.M = K; x.N = d; x.K = dh;
  x.A = dp; x.lda = dh; x.a_kmajor = 1;
  x.B = P->w_a; x.ldb = d; x.b_kmajor = 0;
  x.C = dxc; x.ldc = d;
  MTGR_TRY(gemm_any<T>(x, EPI_STORE, scratch, scratch_bytes, st));
  ProfScope ps(PROF_HEAD, st);
  head_scatter_kernel<T><<<B, 256, 0, st>>>(*j, coff, dxc, d, dz);
  return check_launch("head_scatter");
}

mtgr_status_t check_head_cfg(const mtgr_head_cfg_t* c) {
  MTGR_CHECK(c, MTGR_E_ARG, "head cfg is NULL");
  MTGR_CHECK(c->d_model > 0 && c->d_model % 8 == 0 && c->d_hidden > 0 && c->d_hidden % 8 == 0 &&
                 c->d_hidden <= HEAD_MAX_DH,
             MTGR_E_UNSUPPORTED, "head: d_model and d_hidden must be positive multiples of 8 (d_hidden <= %d)",
             HEAD_MAX_DH);
  return MTGR_OK;
}

}  // namespace

}  // namespace mtgr

using namespace mtgr;

MTGR_API size_t mtgr_head_workspace_bytes(const mtgr_head_cfg_t* cfg, const mtgr_jagged_t* jag,
                                          int32_t total_candidates, mtgr_dtype_t dtype) {
  if (!cfg || !jag || total_candidates < 0) return 0;
  const size_t es = dtype == MTGR_BF16 ? 2 : 4;
  return head_layout(cfg, total_candidates, jag->num_users, es, dtype == MTGR_BF16).total + 256;
}

MTGR_API mtgr_status_t mtgr_head_fwd_bwd(const mtgr_head_cfg_t* cfg, const mtgr_jagged_t* jag,
                                         int32_t total_candidates, mtgr_dtype_t dtype,
                                         const mtgr_head_params_t* params, const void* z,
                                         const uint8_t* labels, float* logits, float* loss, void* dz,
                                         const mtgr_head_grads_t* grads, void* ws, size_t ws_bytes,
                                         mtgr_stream_t stream) {
  MTGR_TRY(check_head_cfg(cfg));
  MTGR_CHECK(jag && params, MTGR_E_ARG, "head: null jagged batch or params");
  MTGR_CHECK(dtype == MTGR_F32 || dtype == MTGR_BF16, MTGR_E_DTYPE, "head: dtype must be MTGR_F32 or MTGR_BF16");
  MTGR_CHECK(jag->num_users >= 0 && jag->total_tokens >= 0 && total_candidates >= 0 &&
                 total_candidates <= jag->total_tokens,
             MTGR_E_ARG, "head: bad sizes");
  MTGR_CHECK(ws_bytes >= mtgr_head_workspace_bytes(cfg, jag, total_candidates, dtype), MTGR_E_WORKSPACE,
             "head: workspace too small");
  if (jag->num_users == 0 && total_candidates == 0 && loss == nullptr && dz == nullptr) return MTGR_OK;
  MTGR_CHECK(jag->num_users == 0 || (jag->offsets && jag->n_static && jag->n_rt && jag->n_cand),
             MTGR_E_ARG, "head: jagged metadata is NULL");
  MTGR_CHECK(total_candidates == 0 || (z && labels && params->w_a && params->b_a && params->w_b && params->b_b && ws),
             MTGR_E_ARG, "head: null pointer");
  MTGR_CHECK(!dz || (grads && grads->w_a && grads->b_a && grads->w_b && grads->b_b), MTGR_E_ARG,
             "head: gradients requested but grads is NULL");
  MTGR_CHECK(!z || aligned16(z), MTGR_E_LAYOUT, "head: z must be 16-byte aligned");
  MTGR_CHECK(!dz || aligned16(dz), MTGR_E_LAYOUT, "head: dz must be 16-byte aligned");
  char* w = (char*)ws;
  if (w) w += (256 - (reinterpret_cast<uintptr_t>(w) & 255)) & 255;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == MTGR_BF16)
    return head_run<__nv_bfloat16>(cfg, jag, total_candidates, params, (const __nv_bfloat16*)z, labels,
                                   logits, loss, (__nv_bfloat16*)dz, grads, w, st);
  return head_run<float>(cfg, jag, total_candidates, params, (const float*)z, labels, logits, loss,
                         (float*)dz, grads, w, st);
}
