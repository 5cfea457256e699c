#include <algorithm>
// Small HBM-bound kernels: bias-gradient column sums, gradient scaling (P:360 aggregation),
// the dense mask export and the jagged metadata validator.
#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace mtgr {

// ------------------------------------------------------------------ column sums (db = sum_t dY)
constexpr int CS_ROWS = 128;  // tokens per partial

__device__ __forceinline__ void cs_load8(const float* p, float* v) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void cs_load8(const __nv_bfloat16* p, float* v) {
  const uint4 a = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x; v[2 * i + 1] = f.y;
  }
}

// thread = 8 consecutive columns (16-byte loads), block.y = CS_ROWS tokens
template <class T>
__global__ void __launch_bounds__(256) colsum_part_kernel(const T* __restrict__ X, int64_t ld,
                                                          int ntok, int n, float* __restrict__ part) {
  const int c0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c0 >= n) return;
  const int r0 = blockIdx.y * CS_ROWS, r1 = min(ntok, r0 + CS_ROWS);
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
  for (int r = r0; r < r1; ++r) {
    float v[8];
    cs_load8(X + (int64_t)r * ld + c0, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) s[e] += v[e];
  }
  float* dst = part + (int64_t)blockIdx.y * n + c0;
  reinterpret_cast<float4*>(dst)[0] = make_float4(s[0], s[1], s[2], s[3]);
  reinterpret_cast<float4*>(dst)[1] = make_float4(s[4], s[5], s[6], s[7]);
}

// fixed-order two-level sum of the partials (deterministic)
__global__ void __launch_bounds__(256) colsum_reduce_kernel(const float* __restrict__ part,
                                                            int nparts, int n,
                                                            float* __restrict__ out, int accumulate) {
  __shared__ float red[8][33];
  const int col = blockIdx.x * 32 + (threadIdx.x & 31);
  const int rg = threadIdx.x >> 5;
  float s = 0.f;
  if (col < n)
    for (int p = rg; p < nparts; p += 8) s += part[(int64_t)p * n + col];
  red[rg][threadIdx.x & 31] = s;
  __syncthreads();
  if (rg == 0 && col < n) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][threadIdx.x];
    out[col] = accumulate ? out[col] + t : t;
  }
}

size_t colsum_ws_bytes(int ntok, int n) {
  return align_up((size_t)ceil_div(ntok > 0 ? ntok : 1, CS_ROWS) * n * sizeof(float), 256);
}

template <class T>
mtgr_status_t colsum_launch(const T* X, int64_t ld, int ntok, int n, float* out, float* part,
                            int accumulate, cudaStream_t st) {
  ProfScope ps(PROF_COLSUM, st);
  MTGR_CHECK(n % 8 == 0 && ld % 8 == 0, MTGR_E_LAYOUT, "colsum: n and ld must be multiples of 8");
  int nparts = ntok > 0 ? ceil_div(ntok, CS_ROWS) : 0;
  if (nparts > 0) {
    colsum_part_kernel<T><<<dim3(ceil_div(n, 8 * 256), nparts), 256, 0, st>>>(X, ld, ntok, n, part);
    MTGR_TRY(check_launch("colsum_part"));
  }
  colsum_reduce_kernel<<<ceil_div(n, 32), 256, 0, st>>>(part, nparts, n, out, accumulate);
  return check_launch("colsum_reduce");
}
template mtgr_status_t colsum_launch<float>(const float*, int64_t, int, int, float*, float*, int,
                                            cudaStream_t);
template mtgr_status_t colsum_launch<__nv_bfloat16>(const __nv_bfloat16*, int64_t, int, int,
                                                    float*, float*, int, cudaStream_t);

// ------------------------------------------------------------------ scale
__global__ void scale_kernel(float* g, int64_t n, float s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    g[i] *= s;
}
mtgr_status_t scale_launch(float* g, int64_t n, float s, cudaStream_t st) {
  if (n == 0) return MTGR_OK;
  int64_t nb64 = ceil_div64(n, 256); int blocks = (int)(nb64 < 4 * num_sms() ? nb64 : 4 * num_sms());
  scale_kernel<<<blocks, 256, 0, st>>>(g, n, s);
  return check_launch("scale");
}

// ------------------------------------------------------------------ gate: y = o (.) u (bf16)
// (Eq.6 gate for the public attention call; the layer folds it into the GLN2 load instead)
__global__ void gate_mul_kernel(const __nv_bfloat16* o, int64_t ldo, const __nv_bfloat16* u,
                                int64_t ldu, __nv_bfloat16* y, int64_t ldy, int ntok, int d) {
  const int nv = d >> 3;
  const int64_t n = (int64_t)ntok * nv;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / nv;
    const int c = (int)(e % nv) * 8;
    const uint4 ow = *reinterpret_cast<const uint4*>(o + t * ldo + c);
    const uint4 uw = *reinterpret_cast<const uint4*>(u + t * ldu + c);
    const __nv_bfloat162* oh = reinterpret_cast<const __nv_bfloat162*>(&ow);
    const __nv_bfloat162* uh = reinterpret_cast<const __nv_bfloat162*>(&uw);
    uint4 yw;
    __nv_bfloat162* yh = reinterpret_cast<__nv_bfloat162*>(&yw);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 a = __bfloat1622float2(oh[k]), b = __bfloat1622float2(uh[k]);
      yh[k] = __floats2bfloat162_rn(a.x * b.x, a.y * b.y);
    }
    *reinterpret_cast<uint4*>(y + t * ldy + c) = yw;
  }
}
mtgr_status_t gate_mul_launch(const void* o, int64_t ldo, const void* u, int64_t ldu, void* y,
                              int64_t ldy, int ntok, int d, cudaStream_t st) {
  const int64_t n = (int64_t)ntok * (d >> 3);
  if (n == 0) return MTGR_OK;
  int64_t nb64 = ceil_div64(n, 256); int blocks = (int)(nb64 < 8 * num_sms() ? nb64 : 8 * num_sms());
  gate_mul_kernel<<<blocks, 256, 0, st>>>((const __nv_bfloat16*)o, ldo, (const __nv_bfloat16*)u, ldu,
                                          (__nv_bfloat16*)y, ldy, ntok, d);
  return check_launch("gate_mul");
}

// ------------------------------------------------------------------ elementwise product
template <class T>
__global__ void mul_kernel(const T* a, const T* b, T* y, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    y[e] = from_f<T>(to_f(a[e]) * to_f(b[e]));
}
template <class T>
mtgr_status_t mul_launch(const T* a, const T* b, T* y, int64_t n, cudaStream_t st) {
  if (n == 0) return MTGR_OK;
  const int blocks = (int)std::min<int64_t>(ceil_div64(n, 256), 8 * num_sms());
  mul_kernel<T><<<blocks, 256, 0, st>>>(a, b, y, n);
  return check_launch("mul");
}
template mtgr_status_t mul_launch<float>(const float*, const float*, float*, int64_t, cudaStream_t);
template mtgr_status_t mul_launch<__nv_bfloat16>(const __nv_bfloat16*, const __nv_bfloat16*, __nv_bfloat16*,
                                                 int64_t, cudaStream_t);

// ------------------------------------------------------------------ dense mask export
// The exact composition the attention kernels use: the off-diagonal predicate on the key range
// [0, n_static + n_rt) plus the diagonal of non-static rows (R#8-R#12).
__global__ void mask_dense_kernel(mtgr_jagged_t j, int user, uint8_t* out) {
  UserSpan us = load_user(j, user);
  const int64_t n = (int64_t)us.L * us.L;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int r = (int)(e / us.L), c = (int)(e % us.L);
    long long tr = j.ts ? j.ts[us.off + r] : 0, tc = j.ts ? j.ts[us.off + c] : 0;
    bool v = (c < us.ns + us.nr && visible_offdiag(r, c, us.ns, tr, tc)) || (r >= us.ns && r == c);
    out[e] = v ? 1 : 0;
  }
}
mtgr_status_t mask_dense_launch(const mtgr_jagged_t& j, int user, uint8_t* out, cudaStream_t st) {
  int blocks = 2 * num_sms();
  mask_dense_kernel<<<blocks, 256, 0, st>>>(j, user, out);
  return check_launch("mask_dense");
}

// ------------------------------------------------------------------ validation
__device__ int g_validate_flag;
__global__ void validate_kernel(mtgr_jagged_t j, int G) {
  int bad = 0;
  const int B = j.num_users;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (j.offsets[0] != 0) bad |= 1;
    if (j.offsets[B] != j.total_tokens) bad |= 2;
  }
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < B; u += gridDim.x * blockDim.x) {
    int L = j.offsets[u + 1] - j.offsets[u];
    if (L < 0) bad |= 4;
    if (L > j.max_len) bad |= 8;
    if (j.n_static[u] < 0 || j.n_rt[u] < 0 || j.n_cand[u] < 0) bad |= 16;
    if (j.n_static[u] + j.n_rt[u] + j.n_cand[u] != L) bad |= 32;
    if (j.n_rt[u] > 0 && !j.ts) bad |= 64;
  }
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < j.total_tokens; t += gridDim.x * blockDim.x)
    if (j.group_id && j.group_id[t] >= G) bad |= 128;
  if (bad) atomicOr(&g_validate_flag, bad);
}
mtgr_status_t validate_launch(const mtgr_jagged_t& j, int G, cudaStream_t st) {
  int zero = 0, flag = 0;
  cudaMemcpyToSymbolAsync(g_validate_flag, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, st);
  validate_kernel<<<num_sms(), 256, 0, st>>>(j, G);
  MTGR_TRY(check_launch("validate"));
  cudaMemcpyFromSymbolAsync(&flag, g_validate_flag, sizeof(int), 0, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return set_error(MTGR_E_CUDA, "validate: %s", cudaGetErrorString(e));
  if (flag) return set_error(MTGR_E_INVALID, "mtgr_validate_jagged: metadata check failed (flags 0x%x)", flag);
  return MTGR_OK;
}

}  // namespace mtgr
