// FP32-arithmetic SIMT kernels: the <= 1e-4 parity path of the layer (SURVEY §7 hard part 6:
// TF32 tensor cores cannot meet 1e-4, so fp32 FFMA).  Templated on the storage type, so they
// also run the bf16 layer for head dims the tensor-core kernels do not cover.
//
//  * gemm_simt:  C = A B^T (+ epilogue) with either operand K- or MN-major.
//  * attention fwd / bwd (Eq.5) per (user, head, 32-row tile): exact mask predicate
//    in registers (R#8-R#12), keys restricted to [0, n_static + n_rt) (candidate columns are
//    visible only to themselves, rule 3 P:338, and enter through the diagonal term).
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace mtgr {

// ------------------------------------------------------------------ GEMM
constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;

template <class T, int EPI>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmIO g) {
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  const T* A = (const T*)g.A;
  const T* B = (const T*)g.B;
  const int m0 = blockIdx.y * SG_BM, n0 = blockIdx.x * SG_BN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += SG_BK) {
    for (int e = threadIdx.x; e < SG_BM * SG_BK; e += 256) {
      int mm, kk;
      if (g.a_kmajor) { mm = e / SG_BK; kk = e % SG_BK; } else { kk = e / SG_BM; mm = e % SG_BM; }
      int m = m0 + mm, k = k0 + kk;
      float v = 0.f;
      if (m < g.M && k < g.K) v = to_f(g.a_kmajor ? A[(int64_t)m * g.lda + k] : A[(int64_t)k * g.lda + m]);
      As[kk][mm] = v;
    }
    for (int e = threadIdx.x; e < SG_BN * SG_BK; e += 256) {
      int nn, kk;
      if (g.b_kmajor) { nn = e / SG_BK; kk = e % SG_BK; } else { kk = e / SG_BN; nn = e % SG_BN; }
      int n = n0 + nn, k = k0 + kk;
      float v = 0.f;
      if (n < g.N && k < g.K) v = to_f(g.b_kmajor ? B[(int64_t)n * g.ldb + k] : B[(int64_t)k * g.ldb + n]);
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty * 4 + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n >= g.N) continue;
      float v = acc[i][j] + (g.bias ? g.bias[n] : 0.f);
      if (EPI == EPI_F32) {
        float* C = (float*)g.C + (int64_t)m * g.ldc + n;
        *C = g.accumulate ? *C + v : v;
      } else if (EPI == EPI_QKVU) {
        ((T*)g.C)[(int64_t)m * g.ldc + n] = from_f<T>(g.silu && g.c_dsilu ? dsilu_f(v) : v);
        ((T*)g.C2)[(int64_t)m * g.ldc + n] = from_f<T>(g.silu ? silu_f(v) : v);
      } else if (EPI == EPI_RESID) {
        v += to_f(((const T*)g.R)[(int64_t)m * g.ldr + n]);
        ((T*)g.C)[(int64_t)m * g.ldc + n] = from_f<T>(v);
      } else {
        ((T*)g.C)[(int64_t)m * g.ldc + n] = from_f<T>(v);
      }
    }
  }
}

template <class T>
mtgr_status_t gemm_simt_launch(const GemmIO& g, int epi, cudaStream_t st) {
  if (g.M == 0 || g.N == 0) return MTGR_OK;
  ProfScope ps(epi == EPI_QKVU ? PROF_GEMM_QKVU : epi == EPI_RESID ? PROF_GEMM_OUT
               : epi == EPI_STORE ? PROF_GEMM_DGRAD : PROF_GEMM_WGRAD, st);
  dim3 grid(ceil_div(g.N, SG_BN), ceil_div(g.M, SG_BM));
  switch (epi) {
    case EPI_STORE: gemm_simt_kernel<T, EPI_STORE><<<grid, 256, 0, st>>>(g); break;
    case EPI_QKVU: gemm_simt_kernel<T, EPI_QKVU><<<grid, 256, 0, st>>>(g); break;
    case EPI_RESID: gemm_simt_kernel<T, EPI_RESID><<<grid, 256, 0, st>>>(g); break;
    default: gemm_simt_kernel<T, EPI_F32><<<grid, 256, 0, st>>>(g); break;
  }
  return check_launch("gemm_simt");
}
template mtgr_status_t gemm_simt_launch<float>(const GemmIO&, int, cudaStream_t);
template mtgr_status_t gemm_simt_launch<__nv_bfloat16>(const GemmIO&, int, cudaStream_t);

// ------------------------------------------------------------------ attention helpers
constexpr int SA_B = 32;  // rows per tile (queries or keys)

// diagonal terms of non-static tokens (R#9): a_ii = nu*silu(s_ii), ds_ii = nu*silu'(s_ii)*(dO_i.v_i)
// with s_ii = q_i.k_i (+ rab_w[h][0], the bucket of |dt| = 0).  One warp per token.
template <class T>
__device__ __forceinline__ void ld8f(const T* p, float* v) {
  if constexpr (std::is_same<T, float>::value) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
    const uint4 a = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x; v[2 * i + 1] = f.y;
    }
  }
}

// one block per user, one warp per NON-STATIC token of that user (static tokens have no diagonal
// term: their self-visibility is inside the static block, R#8/R#9); lane c handles 8-element
// chunks c, c+32, ... of each head (16-byte loads).  Entries of static tokens are never read.
template <class T>
__global__ void __launch_bounds__(256) attn_diag_kernel(AttnIO a, int bwd, float* __restrict__ diag_a,
                                                        float* __restrict__ diag_ds) {
  const int lane = threadIdx.x & 31;
  const UserSpan us = load_user(a.jag, blockIdx.y);
  const T* q = (const T*)a.q; const T* k = (const T*)a.k; const T* v = (const T*)a.v;
  const T* dO = (const T*)a.dO;
  const int nch = a.dh >> 3;
  const int first = a.diag_cand_only ? us.ns + us.nr : us.ns;
  // grid (row blocks, users): a single long request still spreads over many SMs
  const int wpb = blockDim.x >> 5;
  for (int li = first + blockIdx.x * wpb + (threadIdx.x >> 5); li < us.L; li += gridDim.x * wpb) {
    const int64_t t = us.off + li;
    for (int h = 0; h < a.H; ++h) {
      float s = 0.f, pv = 0.f;
      for (int c = lane; c < nch; c += 32) {
        const int64_t col = (int64_t)h * a.dh + c * 8;
        float qa[8], ka[8];
        ld8f(q + t * a.ld + col, qa);
        ld8f(k + t * a.ld + col, ka);
#pragma unroll
        for (int e = 0; e < 8; ++e) s = fmaf(qa[e], ka[e], s);
        if (bwd) {
          float da[8], va[8];
          ld8f(dO + t * a.d + col, da);
          ld8f(v + t * a.ld + col, va);
#pragma unroll
          for (int e = 0; e < 8; ++e) pv = fmaf(da[e], va[e], pv);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        pv += __shfl_xor_sync(0xffffffffu, pv, o);
      }
      if (a.nb > 0) s += a.rab_w[h * a.nb + 0];
      if (lane == 0) {
        diag_a[t * a.H + h] = us.nu * silu_f(s);
        if (bwd) {
          const float ds = us.nu * dsilu_f(s) * pv;
          diag_ds[t * a.H + h] = ds;
          if (a.nb > 0 && a.drab) atomicAdd(&a.drab[h * a.nb + 0], ds);
        }
      }
    }
  }
}

template <class T>
mtgr_status_t attn_diag_launch(const AttnIO& a, bool bwd, float* diag_a, float* diag_ds,
                               cudaStream_t st) {
  if (a.jag.total_tokens == 0 || a.jag.num_users == 0) return MTGR_OK;
  ProfScope ps(PROF_ATTN_DIAG, st);
  // one warp per token; enough row blocks per user that ~4 waves cover the batch
  const int users = a.jag.num_users;
  int rb = std::max(1, std::min(ceil_div(a.jag.max_len, 8), ceil_div(4 * num_sms(), users)));
  attn_diag_kernel<T><<<dim3(rb, users), 256, 0, st>>>(a, bwd ? 1 : 0, diag_a, diag_ds);
  return check_launch("attn_diag");
}
template mtgr_status_t attn_diag_launch<float>(const AttnIO&, bool, float*, float*, cudaStream_t);
template mtgr_status_t attn_diag_launch<__nv_bfloat16>(const AttnIO&, bool, float*, float*,
                                                       cudaStream_t);

template <class T>
__device__ __forceinline__ void load_rows(float* dst, const T* src, int64_t ld, int row0,
                                          int nrows_valid, int dh) {
  for (int e = threadIdx.x; e < SA_B * dh; e += blockDim.x) {
    int r = e / dh, c = e % dh;
    dst[r * dh + c] = r < nrows_valid ? to_f(src[(int64_t)(row0 + r) * ld + c]) : 0.f;
  }
}

// forward: block (q tile, head, user).  thread = (row r = tid/8, column group cg = tid%8)
template <class T>
__global__ void __launch_bounds__(256) attn_simt_fwd_kernel(AttnIO a) {
  extern __shared__ float sm[];
  const int dh = a.dh;
  float* Qs = sm;
  float* Ks = Qs + SA_B * dh;
  float* Vs = Ks + SA_B * dh;
  float* Ps = Vs + SA_B * dh;  // [SA_B][SA_B+1]
  long long* tsk = (long long*)(Ps + SA_B * (SA_B + 1));
  const int u = blockIdx.z, h = blockIdx.y;
  UserSpan us = load_user(a.jag, u);
  const int i0 = blockIdx.x * SA_B;
  if (i0 >= us.L) return;
  const int nq = min(SA_B, us.L - i0);
  const int kv_end = a.causal ? min(us.L, i0 + nq)
                              : ((a.full || i0 + nq > us.ns) ? us.ns + us.nr : us.ns);
  const int r = threadIdx.x / 8, cg = threadIdx.x % 8;
  const int i = i0 + r;
  const int64_t col0 = (int64_t)h * dh;
  const T* q = (const T*)a.q + col0; const T* k = (const T*)a.k + col0;
  const T* v = (const T*)a.v + col0;
  const long long ts_i = (i < us.L && a.jag.ts) ? a.jag.ts[us.off + i] : 0;
  load_rows(Qs, q, a.ld, us.off + i0, nq, dh);
  float acc[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) acc[c] = 0.f;
  const int ncol = dh / 8;  // columns per thread (<= 32)
  for (int j0 = 0; j0 < kv_end; j0 += SA_B) {
    const int nk = min(SA_B, kv_end - j0);
    __syncthreads();
    load_rows(Ks, k, a.ld, us.off + j0, nk, dh);
    load_rows(Vs, v, a.ld, us.off + j0, nk, dh);
    if (threadIdx.x < SA_B)
      tsk[threadIdx.x] = (threadIdx.x < nk && a.jag.ts) ? a.jag.ts[us.off + j0 + threadIdx.x] : 0;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int jj = cg + 8 * e;
      int j = j0 + jj;
      float s = 0.f;
      for (int c = 0; c < dh; ++c) s = fmaf(Qs[r * dh + c], Ks[jj * dh + c], s);
      bool vis = i < us.L && jj < nk &&
                 (a.causal ? j <= i
                           : (a.full ? visible_offdiag_full(i, j, us.ns, us.nr)
                                     : visible_offdiag(i, j, us.ns, ts_i, tsk[jj])));
      if (a.nb > 0) s += a.rab_w[h * a.nb + rab_bucket(ts_i - tsk[jj], a.nb)];
      Ps[r * (SA_B + 1) + jj] = vis ? silu_f(s) : 0.f;
    }
    __syncthreads();
    for (int jj = 0; jj < nk; ++jj) {
      float p = Ps[r * (SA_B + 1) + jj];
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c < ncol) acc[c] = fmaf(p, Vs[jj * dh + cg + 8 * c], acc[c]);
    }
  }
  if (i >= us.L) return;
  const int64_t t = us.off + i;
  const float da = (!a.causal && i >= us.ns) ? a.diag_a[t * a.H + h] : 0.f;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    if (c >= ncol) break;
    int cc = cg + 8 * c;
    float o = us.nu * acc[c] + da * to_f(v[t * a.ld + cc]);
    ((T*)a.o)[t * a.d + col0 + cc] = from_f<T>(o);
    if (a.u) ((T*)a.y)[t * a.d + col0 + cc] = from_f<T>(o * to_f(((const T*)a.u)[t * a.ld + col0 + cc]));
  }
}

// dK / dV: block (key tile j, head, user); loops over query tiles.
template <class T>
__global__ void __launch_bounds__(256) attn_simt_dkv_kernel(AttnIO a) {
  extern __shared__ float sm[];
  const int dh = a.dh;
  float* Ks = sm;
  float* Vs = Ks + SA_B * dh;
  float* Qs = Vs + SA_B * dh;
  float* Ds = Qs + SA_B * dh;        // dO rows
  float* Pt = Ds + SA_B * dh;        // [key][query]
  float* St = Pt + SA_B * (SA_B + 1);
  long long* tsq = (long long*)(St + SA_B * (SA_B + 1));
  float* rab_acc = (float*)(tsq + SA_B);  // [nb]
  const int u = blockIdx.z, h = blockIdx.y;
  UserSpan us = load_user(a.jag, u);
  const int j0 = blockIdx.x * SA_B;
  if (j0 >= us.L) return;
  const int nk = min(SA_B, us.L - j0);
  // dynamic: candidate keys only ever meet the diagonal; causal: every key up to the end
  const int key_end = a.causal ? us.L : us.ns + us.nr;
  const int r = threadIdx.x / 8, cg = threadIdx.x % 8;
  const int j = j0 + r;
  const int64_t col0 = (int64_t)h * dh;
  const T* q = (const T*)a.q + col0; const T* k = (const T*)a.k + col0;
  const T* v = (const T*)a.v + col0; const T* dO = (const T*)a.dO + col0;
  for (int e = threadIdx.x; e < a.nb; e += blockDim.x) rab_acc[e] = 0.f;
  const long long ts_j = (j < us.L && a.jag.ts) ? a.jag.ts[us.off + j] : 0;
  load_rows(Ks, k, a.ld, us.off + j0, nk, dh);
  load_rows(Vs, v, a.ld, us.off + j0, nk, dh);
  float accv[32], acck[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) accv[c] = acck[c] = 0.f;
  const int ncol = dh / 8;
  const int q_begin = a.causal ? j0 : ((a.full || j0 < us.ns) ? 0 : us.ns);
  const int q_end = (j0 < key_end) ? us.L : 0;
  for (int i0 = q_begin; i0 < q_end; i0 += SA_B) {
    const int nq = min(SA_B, us.L - i0);
    __syncthreads();
    load_rows(Qs, q, a.ld, us.off + i0, nq, dh);
    load_rows(Ds, dO, a.d, us.off + i0, nq, dh);
    if (threadIdx.x < SA_B)
      tsq[threadIdx.x] = (threadIdx.x < nq && a.jag.ts) ? a.jag.ts[us.off + i0 + threadIdx.x] : 0;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int ii = cg + 8 * e;
      int i = i0 + ii;
      float s = 0.f, dp = 0.f;
      for (int c = 0; c < dh; ++c) {
        s = fmaf(Qs[ii * dh + c], Ks[r * dh + c], s);
        dp = fmaf(Ds[ii * dh + c], Vs[r * dh + c], dp);
      }
      bool vis = ii < nq && j < key_end &&
                 (a.causal ? i >= j
                           : (a.full ? visible_offdiag_full(i, j, us.ns, us.nr)
                                     : visible_offdiag(i, j, us.ns, tsq[ii], ts_j)));
      int bk = 0;
      if (a.nb > 0) { bk = rab_bucket(tsq[ii] - ts_j, a.nb); s += a.rab_w[h * a.nb + bk]; }
      float ds = vis ? dp * dsilu_f(s) : 0.f;
      Pt[r * (SA_B + 1) + ii] = vis ? silu_f(s) : 0.f;
      St[r * (SA_B + 1) + ii] = ds;
      if (a.nb > 0 && a.drab && vis) atomicAdd(&rab_acc[bk], ds);
    }
    __syncthreads();
    for (int ii = 0; ii < nq; ++ii) {
      float p = Pt[r * (SA_B + 1) + ii], ds = St[r * (SA_B + 1) + ii];
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c < ncol) {
          accv[c] = fmaf(p, Ds[ii * dh + cg + 8 * c], accv[c]);
          acck[c] = fmaf(ds, Qs[ii * dh + cg + 8 * c], acck[c]);
        }
    }
  }
  __syncthreads();
  if (a.nb > 0 && a.drab)
    for (int e = threadIdx.x; e < a.nb; e += blockDim.x)
      if (rab_acc[e] != 0.f) atomicAdd(&a.drab[h * a.nb + e], us.nu * rab_acc[e]);
  if (j >= us.L) return;
  const int64_t t = us.off + j;
  const float da = (!a.causal && j >= us.ns) ? a.diag_a[t * a.H + h] : 0.f;
  const float dd = (!a.causal && j >= us.ns) ? a.diag_ds[t * a.H + h] : 0.f;
  const T* pre = (const T*)a.pre;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    if (c >= ncol) break;
    int cc = cg + 8 * c;
    float gv = us.nu * accv[c] + da * to_f(dO[t * a.d + cc]);
    float gk = us.nu * acck[c] + dd * to_f(q[t * a.ld + cc]);
    if (pre) {
      const float pk = to_f(pre[t * a.ld_pre + (int64_t)a.d + col0 + cc]);
      const float pv = to_f(pre[t * a.ld_pre + 2 * (int64_t)a.d + col0 + cc]);
      gk *= a.pre_dsilu ? pk : dsilu_f(pk);
      gv *= a.pre_dsilu ? pv : dsilu_f(pv);
    }
    ((T*)a.dk)[t * a.ld_out + col0 + cc] = from_f<T>(gk);
    ((T*)a.dv)[t * a.ld_out + col0 + cc] = from_f<T>(gv);
  }
}

// dQ: block (query tile, head, user); loops over key tiles.
template <class T>
__global__ void __launch_bounds__(256) attn_simt_dq_kernel(AttnIO a) {
  extern __shared__ float sm[];
  const int dh = a.dh;
  float* Qs = sm;
  float* Ds = Qs + SA_B * dh;
  float* Ks = Ds + SA_B * dh;
  float* Vs = Ks + SA_B * dh;
  float* Ss = Vs + SA_B * dh;  // dS [query][key]
  long long* tsk = (long long*)(Ss + SA_B * (SA_B + 1));
  const int u = blockIdx.z, h = blockIdx.y;
  UserSpan us = load_user(a.jag, u);
  const int i0 = blockIdx.x * SA_B;
  if (i0 >= us.L) return;
  const int nq = min(SA_B, us.L - i0);
  const int kv_end = a.causal ? min(us.L, i0 + nq)
                              : ((a.full || i0 + nq > us.ns) ? us.ns + us.nr : us.ns);
  const int r = threadIdx.x / 8, cg = threadIdx.x % 8;
  const int i = i0 + r;
  const int64_t col0 = (int64_t)h * dh;
  const T* q = (const T*)a.q + col0; const T* k = (const T*)a.k + col0;
  const T* v = (const T*)a.v + col0; const T* dO = (const T*)a.dO + col0;
  const long long ts_i = (i < us.L && a.jag.ts) ? a.jag.ts[us.off + i] : 0;
  load_rows(Qs, q, a.ld, us.off + i0, nq, dh);
  load_rows(Ds, dO, a.d, us.off + i0, nq, dh);
  float acc[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) acc[c] = 0.f;
  const int ncol = dh / 8;
  for (int j0 = 0; j0 < kv_end; j0 += SA_B) {
    const int nk = min(SA_B, kv_end - j0);
    __syncthreads();
    load_rows(Ks, k, a.ld, us.off + j0, nk, dh);
    load_rows(Vs, v, a.ld, us.off + j0, nk, dh);
    if (threadIdx.x < SA_B)
      tsk[threadIdx.x] = (threadIdx.x < nk && a.jag.ts) ? a.jag.ts[us.off + j0 + threadIdx.x] : 0;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int jj = cg + 8 * e;
      int j = j0 + jj;
      float s = 0.f, dp = 0.f;
      for (int c = 0; c < dh; ++c) {
        s = fmaf(Qs[r * dh + c], Ks[jj * dh + c], s);
        dp = fmaf(Ds[r * dh + c], Vs[jj * dh + c], dp);
      }
      bool vis = i < us.L && jj < nk &&
                 (a.causal ? j <= i
                           : (a.full ? visible_offdiag_full(i, j, us.ns, us.nr)
                                     : visible_offdiag(i, j, us.ns, ts_i, tsk[jj])));
      if (a.nb > 0) s += a.rab_w[h * a.nb + rab_bucket(ts_i - tsk[jj], a.nb)];
      Ss[r * (SA_B + 1) + jj] = vis ? dp * dsilu_f(s) : 0.f;
    }
    __syncthreads();
    for (int jj = 0; jj < nk; ++jj) {
      float ds = Ss[r * (SA_B + 1) + jj];
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c < ncol) acc[c] = fmaf(ds, Ks[jj * dh + cg + 8 * c], acc[c]);
    }
  }
  if (i >= us.L) return;
  const int64_t t = us.off + i;
  const float dd = (!a.causal && i >= us.ns) ? a.diag_ds[t * a.H + h] : 0.f;
  const T* pre = (const T*)a.pre;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    if (c >= ncol) break;
    int cc = cg + 8 * c;
    float g = us.nu * acc[c] + dd * to_f(k[t * a.ld + cc]);
    if (pre) {
      const float pq = to_f(pre[t * a.ld_pre + col0 + cc]);
      g *= a.pre_dsilu ? pq : dsilu_f(pq);
    }
    ((T*)a.dq)[t * a.ld_out + col0 + cc] = from_f<T>(g);
  }
}

template <class T>
mtgr_status_t attn_simt_fwd_launch(const AttnIO& a, cudaStream_t st) {
  if (a.jag.num_users == 0 || a.jag.max_len == 0) return MTGR_OK;
  dim3 grid(ceil_div(a.jag.max_len, SA_B), a.H, a.jag.num_users);
  ProfScope ps(PROF_ATTN_FWD, st);
  size_t smem = (3 * SA_B * a.dh + SA_B * (SA_B + 1)) * sizeof(float) + SA_B * sizeof(long long);
  cudaFuncSetAttribute(attn_simt_fwd_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  attn_simt_fwd_kernel<T><<<grid, 256, smem, st>>>(a);
  return check_launch("attn_simt_fwd");
}

template <class T>
mtgr_status_t attn_simt_bwd_launch(const AttnIO& a, cudaStream_t st) {
  if (a.jag.num_users == 0 || a.jag.max_len == 0) return MTGR_OK;
  dim3 grid(ceil_div(a.jag.max_len, SA_B), a.H, a.jag.num_users);
  size_t smem_kv = (4 * SA_B * a.dh + 2 * SA_B * (SA_B + 1)) * sizeof(float) +
                   SA_B * sizeof(long long) + (size_t)(a.nb > 0 ? a.nb : 1) * sizeof(float);
  {
    ProfScope ps(PROF_ATTN_DV, st);
    cudaFuncSetAttribute(attn_simt_dkv_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_kv);
    attn_simt_dkv_kernel<T><<<grid, 256, smem_kv, st>>>(a);
    MTGR_TRY(check_launch("attn_simt_dkv"));
  }
  ProfScope ps(PROF_ATTN_DQ, st);
  size_t smem_q = (4 * SA_B * a.dh + SA_B * (SA_B + 1)) * sizeof(float) + SA_B * sizeof(long long);
  cudaFuncSetAttribute(attn_simt_dq_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_q);
  attn_simt_dq_kernel<T><<<grid, 256, smem_q, st>>>(a);
  return check_launch("attn_simt_dq");
}

template mtgr_status_t attn_simt_fwd_launch<float>(const AttnIO&, cudaStream_t);
template mtgr_status_t attn_simt_bwd_launch<float>(const AttnIO&, cudaStream_t);

}  // namespace mtgr
