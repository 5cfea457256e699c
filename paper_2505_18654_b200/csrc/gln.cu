// Group-Layer Norm forward / backward (Eq.6; readings R#13, R#14).
//
// HBM-bound: one warp per token, 16-byte vector loads (8 elements per lane per chunk),
// warp-shuffle reductions, statistics kept in registers.  The backward optionally fuses
//  * MODE_GATE: the gate backward of Eq.6 (dO = dY (.) U, dU = dY (.) O) and the SiLU'
//    of the U projection (R#5), writing dO and dp_U directly, and
//  * MODE_RESID: the residual of Eq.6 (dx = GLN1_bwd(dX~) + dZ).
// Parameter gradients are per-block partial sums (smem) reduced in block order by a second
// kernel.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"
#include "sm100.cuh"

namespace mtgr {

__device__ __forceinline__ void load8(const float* p, float* v) {
  float4 a = reinterpret_cast<const float4*>(p)[0];
  float4 b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* v) {
  uint4 a = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x; v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void store8(float* p, const float* v) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float* v) {
  uint4 a;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = a;
}

// raw (still packed) 8-element vectors: 16 B for bf16, 32 B for fp32; unpacked only when used
template <class T> struct Raw8;
template <> struct Raw8<__nv_bfloat16> { uint4 v; };
template <> struct Raw8<float> { float4 a, b; };
__device__ __forceinline__ void rload(const __nv_bfloat16* p, Raw8<__nv_bfloat16>& r) {
  r.v = *reinterpret_cast<const uint4*>(p);
}
__device__ __forceinline__ void rload(const float* p, Raw8<float>& r) {
  r.a = reinterpret_cast<const float4*>(p)[0];
  r.b = reinterpret_cast<const float4*>(p)[1];
}
__device__ __forceinline__ void unpack(const Raw8<__nv_bfloat16>& r, float* v) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r.v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x; v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void unpack(const Raw8<float>& r, float* v) {
  v[0] = r.a.x; v[1] = r.a.y; v[2] = r.a.z; v[3] = r.a.w; v[4] = r.b.x; v[5] = r.b.y; v[6] = r.b.z; v[7] = r.b.w;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp per token over a CONTIGUOUS token range per warp (tokens of a group are contiguous
// within a user, so gamma / beta of the current group are reloaded only on a group change: the
// per-token traffic is the token's own rows, not 2d fp32 parameters through L1).  Software
// pipelined: the next token's rows (and group id) are in flight while this one is reduced,
// normalised and stored.  The current group's gamma / beta live in a per-warp shared-memory slot
// (each lane reads back only the chunks it wrote, float4-interleaved: conflict-free) instead of
// 16 registers per chunk, so the kernel fits MINB 256-thread blocks per SM: the resident warps,
// each with two tokens in flight, are what keeps enough bytes in flight for HBM.
template <class T, int NC, bool GATE> constexpr int gln_fwd_minb() {
  return sizeof(T) == 2 ? (NC <= 2 ? (GATE ? 2 : 3) : (NC == 3 ? 2 : 1)) : (NC <= 1 ? 3 : (NC == 2 ? 2 : 1));
}
template <int NC> constexpr int gln_fwd_smem() { return 8 * NC * 2 * 2 * 32 * 16; }  // 8 warps

template <class T, int NC, bool GATE>
__global__ void __launch_bounds__(256, gln_fwd_minb<T, NC, GATE>()) gln_fwd_kernel(const T* __restrict__ x,
                                                      const uint8_t* __restrict__ gid,
                                                      const float* __restrict__ gamma,
                                                      const float* __restrict__ beta,
                                                      T* __restrict__ y, float* __restrict__ mean,
                                                      float* __restrict__ rstd, int ntok, int d,
                                                      float eps, const T* __restrict__ gate,
                                                      int64_t ld_gate, int tok_per_warp) {
  extern __shared__ float4 gln_sp[];
  const int lane = threadIdx.x & 31;
  const int nch = d >> 3;
  const float inv_d = 1.0f / (float)d;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  // this warp's slot: [k][gamma lo, gamma hi, beta lo, beta hi][lane] float4
  float4* gb = gln_sp + (threadIdx.x >> 5) * (NC * 4 * 32) + lane;
  const int t_begin = w * tok_per_warp;
  const int t_end = min(ntok, t_begin + tok_per_warp);
  Raw8<T> cx[NC], nx[NC];
  Raw8<T> cg[GATE ? NC : 1], ng[GATE ? NC : 1];
  auto issue = [&](int tt, Raw8<T>* xa, Raw8<T>* ga) {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = lane + 32 * k;
      if (c < nch) {
        rload(x + (int64_t)tt * d + c * 8, xa[k]);
        if constexpr (GATE) rload(gate + (int64_t)tt * ld_gate + c * 8, ga[k]);
      }
    }
  };
  int g_loaded = -1;
  int t = t_begin;
  int g_cur = 0;
  if (t < t_end) { issue(t, cx, cg); g_cur = gid[t]; }
  for (; t < t_end; ++t) {
    const int tn = t + 1;
    int g_next = 0;
    if (tn < t_end) { issue(tn, nx, ng); g_next = gid[tn]; }
    if (g_cur != g_loaded) {  // group change: this group's affine parameters into the slot
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const int c = lane + 32 * k;
        if (c < nch) {
          const float4* gp = reinterpret_cast<const float4*>(gamma + (int64_t)g_cur * d + c * 8);
          const float4* bp = reinterpret_cast<const float4*>(beta + (int64_t)g_cur * d + c * 8);
          gb[(k * 4 + 0) * 32] = gp[0]; gb[(k * 4 + 1) * 32] = gp[1];
          gb[(k * 4 + 2) * 32] = bp[0]; gb[(k * 4 + 3) * 32] = bp[1];
        }
      }
      g_loaded = g_cur;
    }
    float v[NC][8];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      int c = lane + 32 * k;
      if (c < nch) {
        unpack(cx[k], v[k]);
        if constexpr (GATE) {  // input = x (.) gate (Eq.6 gate folded into the norm's load)
          float gv[8];
          unpack(cg[k], gv);
#pragma unroll
          for (int e = 0; e < 8; ++e) v[k][e] *= gv[e];
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) s += v[k][e];
      }
    }
    const float mu = warp_sum(s) * inv_d;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k)
      if (lane + 32 * k < nch) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float dlt = v[k][e] - mu;
          q += dlt * dlt;
        }
      }
    const float var = warp_sum(q) * inv_d;
    const float r = 1.0f / sqrtf(var + eps);
    T* yr = y + (int64_t)t * d;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      int c = lane + 32 * k;
      if (c < nch) {
        const float4 g0 = gb[(k * 4 + 0) * 32], g1 = gb[(k * 4 + 1) * 32];
        const float4 b0 = gb[(k * 4 + 2) * 32], b1 = gb[(k * 4 + 3) * 32];
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = gg[e] * ((v[k][e] - mu) * r) + bb[e];
        store8(yr + c * 8, o);
      }
    }
    if (lane == 0) {
      if (mean) mean[t] = mu;
      if (rstd) rstd[t] = r;
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      cx[k] = nx[k];
      if constexpr (GATE) cg[k] = ng[k];
    }
    g_cur = g_next;
  }
}

enum { GLN_PLAIN = 0, GLN_GATE = 1, GLN_RESID = 2 };

template <class T>
struct GlnBwdArgs {
  const T* dy;
  const T* x;
  const float* mean;
  const float* rstd;
  const float* gamma;
  const uint8_t* gid;
  T* dx;          // GLN_GATE: dO
  float* part;    // [G][2][d] fp32 accumulators (zeroed by the launcher)
  int ntok, d, G, tok_per_warp;
  // GLN_GATE
  const T* o;     // [T][d]
  const T* u;     // rows ld_a
  const T* pre_u; // rows ld_a (pre-activation of U) or NULL (linear)
  int pre_dsilu;  // pre_u holds silu'(p_U) already
  int64_t ld_a;
  T* dpu;         // rows ld_dp
  int64_t ld_dp;
  // GLN_RESID
  const T* dz;
  float* dcol;    // [d] column-sum accumulator (red.add): sum of dz (RESID) / dp_U (GATE), or NULL
};

constexpr int GLNB_WARPS = 4;

// One warp per token, a contiguous token range per warp.  All of a token's loads are issued
// before any reduction (memory-level parallelism); the parameter-gradient contributions
// dgamma[g] += dy*xhat, dbeta[g] += dy are accumulated in registers while the group id stays
// the same (tokens of a group are contiguous within a user) and flushed to the block's smem
// accumulator [G][2][d] on a group change; block partials go to global with red.add.
template <class T, int MODE, int NC>
__global__ void __launch_bounds__(32 * GLNB_WARPS, (NC <= 2 ? (MODE == GLN_GATE ? 3 : 4) : 2)) gln_bwd_kernel(GlnBwdArgs<T> a) {
  extern __shared__ float sacc[];  // [G][2][d] (+ [d] column sums)
  const int d = a.d, G = a.G;
  const bool csum = MODE != GLN_PLAIN && a.dcol != nullptr;
  for (int i = threadIdx.x; i < G * 2 * d + d; i += blockDim.x) sacc[i] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nch = d >> 3;
  const float inv_d = 1.0f / (float)d;
  const int w_begin = (blockIdx.x * GLNB_WARPS + warp) * a.tok_per_warp;
  const int w_end = min(a.ntok, w_begin + a.tok_per_warp);
  float pg[NC][8], pb[NC][8], pc[NC][8];
#pragma unroll
  for (int k = 0; k < NC; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) pg[k][e] = pb[k][e] = pc[k][e] = 0.f;
  int cur_g = w_begin < w_end ? a.gid[w_begin] : 0;
  auto flush = [&]() {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = lane + 32 * k;
      if (c < nch) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          atomicAdd(&sacc[(cur_g * 2 + 0) * d + c * 8 + e], pg[k][e]);
          atomicAdd(&sacc[(cur_g * 2 + 1) * d + c * 8 + e], pb[k][e]);
          pg[k][e] = pb[k][e] = 0.f;
        }
      }
    }
  };
#pragma unroll 1
  for (int t = w_begin; t < w_end; ++t) {
    const int g = a.gid[t];
    const float mu = a.mean[t], r = a.rstd[t];
    Raw8<T> xr[NC], dyr[NC], e1r[NC], e2r[NC], e3r[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = lane + 32 * k;
      if (c < nch) {
        if (MODE != GLN_GATE || a.x != nullptr) rload(a.x + (int64_t)t * d + c * 8, xr[k]);
        rload(a.dy + (int64_t)t * d + c * 8, dyr[k]);
        if (MODE == GLN_RESID) rload(a.dz + (int64_t)t * d + c * 8, e1r[k]);
        if (MODE == GLN_GATE) {
          rload(a.u + (int64_t)t * a.ld_a + c * 8, e1r[k]);
          rload(a.o + (int64_t)t * d + c * 8, e2r[k]);
          if (a.pre_u) rload(a.pre_u + (int64_t)t * a.ld_a + c * 8, e3r[k]);
        }
      }
    }
    if (g != cur_g) {
      flush();
      cur_g = g;
    }
    const float* gr = a.gamma + (int64_t)g * d;
    // gated norm input (x == NULL): x = o (.) u, recomputed exactly as the forward formed it
    auto x_of = [&](int k, float* xv) {
      if (MODE == GLN_GATE && a.x == nullptr) {
        float uu[8], oo[8];
        unpack(e1r[k], uu);
        unpack(e2r[k], oo);
#pragma unroll
        for (int e = 0; e < 8; ++e) xv[e] = oo[e] * uu[e];
      } else {
        unpack(xr[k], xv);
      }
    };
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = lane + 32 * k;
      if (c < nch) {
        float xv[8], dyv[8], gg[8];
        x_of(k, xv);
        unpack(dyr[k], dyv);
        load8(gr + c * 8, gg);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float xh = (xv[e] - mu) * r;
          const float dxh = dyv[e] * gg[e];
          pg[k][e] = fmaf(dyv[e], xh, pg[k][e]);
          pb[k][e] += dyv[e];
          s1 += dxh;
          s2 = fmaf(dxh, xh, s2);
        }
      }
    }
    const float m1 = warp_sum(s1) * inv_d, m2 = warp_sum(s2) * inv_d;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = lane + 32 * k;
      if (c < nch) {
        float xv[8], dyv[8], gg[8], o[8];
        x_of(k, xv);
        unpack(dyr[k], dyv);
        load8(gr + c * 8, gg);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = r * (dyv[e] * gg[e] - m1 - (xv[e] - mu) * r * m2);
        if (MODE == GLN_RESID) {
          float z[8];
          unpack(e1r[k], z);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            o[e] += z[e];
            pc[k][e] += z[e];
          }
          store8(a.dx + (int64_t)t * d + c * 8, o);
        } else if (MODE == GLN_GATE) {
          // o[] = dY; dO = dY * U;  dp_U = dY * O * silu'(p_U)
          float uu[8], oo[8], dO[8], du[8];
          unpack(e1r[k], uu);
          unpack(e2r[k], oo);
          float pp[8];
          if (a.pre_u) unpack(e3r[k], pp);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            dO[e] = o[e] * uu[e];
            du[e] = o[e] * oo[e];
            if (a.pre_u) du[e] *= a.pre_dsilu ? pp[e] : dsilu_f(pp[e]);
            pc[k][e] += du[e];
          }
          store8(a.dx + (int64_t)t * d + c * 8, dO);
          store8(a.dpu + (int64_t)t * a.ld_dp + c * 8, du);
        } else {
          store8(a.dx + (int64_t)t * d + c * 8, o);
        }
      }
    }
  }
  if (w_begin < w_end) flush();
  if (csum) {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = lane + 32 * k;
      if (c < nch)
#pragma unroll
        for (int e = 0; e < 8; ++e) atomicAdd(&sacc[G * 2 * d + c * 8 + e], pc[k][e]);
    }
  }
  __syncthreads();
  if (csum)
    for (int i = threadIdx.x; i < d; i += blockDim.x) atomicAdd(a.dcol + i, sacc[G * 2 * d + i]);
  // block partial -> global accumulators [G][2][d] (red.global.add; order not deterministic)
  for (int i = threadIdx.x; i < G * 2 * d; i += blockDim.x) {
    const float v = sacc[i];
    if (v != 0.f) atomicAdd(a.part + i, v);
  }
}

// ---- bf16 backward, bulk-copy pipelined.  The same arithmetic as gln_bwd_kernel, but a
// token's input rows (dy, x | o, u, pre | dz: 1-D contiguous rows) are streamed into a per-warp
// shared-memory ring by cp.async.bulk, S tokens ahead, so the bytes in flight per SM no longer
// depend on registers (the register version keeps ~12 warps x 4 KB in flight, ~45% of HBM
// bandwidth).  One warp per token, a contiguous token range per warp, 16-byte lanes.
struct GlnRing {
  int S;          // stages per warp
  int nrows;      // input rows per token
  int r_x, r_dz, r_o, r_u, r_pre;  // row slot of each input (-1 absent); dy is slot 0
  uint32_t stage_bytes;
  uint32_t ring_off;  // byte offset of the first warp's ring in dynamic smem
};

// packed fp32 pairs (sm_100 FFMA2 / FMUL2 / FADD2) and bf16 pair conversions for the bulk backward
__device__ __forceinline__ unsigned long long p2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2p(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 p2fma(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(p2u(a)), "l"(p2u(b)), "l"(p2u(c)));
  return u2p(d);
}
__device__ __forceinline__ float2 p2mul(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(p2u(a)), "l"(p2u(b)));
  return u2p(d);
}
__device__ __forceinline__ float2 p2add(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(p2u(a)), "l"(p2u(b)));
  return u2p(d);
}
__device__ __forceinline__ float2 bf2_to_f2(uint32_t w) {  // (lo, hi) bf16 -> fp32: shifts only
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
__device__ __forceinline__ void store8p(__nv_bfloat16* p, const float2* v) {
  uint4 a;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __float22bfloat162_rn(v[i]);
  *reinterpret_cast<uint4*>(p) = a;
}

template <int MODE, int NC>
__global__ void __launch_bounds__(512, 1) gln_bwd_bulk_kernel(GlnBwdArgs<__nv_bfloat16> a, GlnRing R) {
  using namespace sm100;
  typedef __nv_bfloat16 bf;
  extern __shared__ __align__(128) uint8_t gsm[];
  float* sacc = reinterpret_cast<float*>(gsm);  // [G][2][d] (+ [d] column sums)
  const int d = a.d, G = a.G;
  const int nwarps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = gsm + R.ring_off + (size_t)warp * R.S * R.stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(gsm + R.ring_off + (size_t)nwarps * R.S * R.stage_bytes) + warp * R.S;
  const bool csum = MODE != GLN_PLAIN && a.dcol != nullptr;
  for (int i = threadIdx.x; i < G * 2 * d + d; i += blockDim.x) sacc[i] = 0.f;
  float* sgam = sacc + G * 2 * d + d;  // gamma [G][d], staged once per block
  for (int i = threadIdx.x; i < G * d; i += blockDim.x) sgam[i] = a.gamma[i];
  if (lane == 0) {
    for (int s = 0; s < R.S; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int nch = d >> 3;
  const float inv_d = 1.0f / (float)d;
  const int w_begin = (blockIdx.x * nwarps + warp) * a.tok_per_warp;
  const int w_end = min(a.ntok, w_begin + a.tok_per_warp);
  const uint32_t row_bytes = (uint32_t)d * 2;
  auto issue = [&](int t, int s) {  // lane 0: all input rows of token t -> stage s
    uint8_t* st = ring + (size_t)s * R.stage_bytes;
    mbar_expect_tx(&bars[s], R.nrows * row_bytes);
    bulk_load(st, a.dy + (int64_t)t * d, row_bytes, &bars[s]);
    if (R.r_x >= 0) bulk_load(st + R.r_x * row_bytes, a.x + (int64_t)t * d, row_bytes, &bars[s]);
    if (R.r_dz >= 0) bulk_load(st + R.r_dz * row_bytes, a.dz + (int64_t)t * d, row_bytes, &bars[s]);
    if (R.r_o >= 0) bulk_load(st + R.r_o * row_bytes, a.o + (int64_t)t * d, row_bytes, &bars[s]);
    if (R.r_u >= 0) bulk_load(st + R.r_u * row_bytes, a.u + (int64_t)t * a.ld_a, row_bytes, &bars[s]);
    if (R.r_pre >= 0) bulk_load(st + R.r_pre * row_bytes, a.pre_u + (int64_t)t * a.ld_a, row_bytes, &bars[s]);
  };
  if (lane == 0)
    for (int s = 0; s < R.S && w_begin + s < w_end; ++s) issue(w_begin + s, s);
  // packed fp32 pairs (FFMA2 / FMUL2 / FADD2): the per-token math in half the issue slots
  float2 pg[NC][4], pb[NC][4], pc[NC][4];
#pragma unroll
  for (int k = 0; k < NC; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) pg[k][e] = pb[k][e] = pc[k][e] = make_float2(0.f, 0.f);
  int cur_g = w_begin < w_end ? a.gid[w_begin] : 0;
  auto flush = [&]() {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = lane + 32 * k;
      if (c < nch) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          atomicAdd(&sacc[(cur_g * 2 + 0) * d + c * 8 + 2 * e], pg[k][e].x);
          atomicAdd(&sacc[(cur_g * 2 + 0) * d + c * 8 + 2 * e + 1], pg[k][e].y);
          atomicAdd(&sacc[(cur_g * 2 + 1) * d + c * 8 + 2 * e], pb[k][e].x);
          atomicAdd(&sacc[(cur_g * 2 + 1) * d + c * 8 + 2 * e + 1], pb[k][e].y);
          pg[k][e] = pb[k][e] = make_float2(0.f, 0.f);
        }
      }
    }
  };
  // per-token scalars one token ahead (their latency hides behind the current token)
  int g_n = 0; float mu_n = 0.f, r_n = 0.f;
  if (w_begin < w_end) { g_n = a.gid[w_begin]; mu_n = a.mean[w_begin]; r_n = a.rstd[w_begin]; }
#pragma unroll 1
  for (int t = w_begin, i = 0; t < w_end; ++t, ++i) {
    const int s = i % R.S;
    const int g = g_n;
    const float mu = mu_n, r = r_n;
    if (t + 1 < w_end) { g_n = a.gid[t + 1]; mu_n = a.mean[t + 1]; r_n = a.rstd[t + 1]; }
    mbar_wait(&bars[s], (i / R.S) & 1);
    const uint8_t* st = ring + (size_t)s * R.stage_bytes;
    auto row8 = [&](int slot, int c, float2* v) {  // 8 elements of an input row (16-byte lane)
      uint32_t w0, w1, w2, w3;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                   : "r"(smem_u32(st + slot * row_bytes + c * 16)));
      v[0] = bf2_to_f2(w0); v[1] = bf2_to_f2(w1); v[2] = bf2_to_f2(w2); v[3] = bf2_to_f2(w3);
    };
    auto gam = [&](const float* gr, float2* v) {
      const float4 g0 = reinterpret_cast<const float4*>(gr)[0], g1 = reinterpret_cast<const float4*>(gr)[1];
      v[0] = make_float2(g0.x, g0.y); v[1] = make_float2(g0.z, g0.w);
      v[2] = make_float2(g1.x, g1.y); v[3] = make_float2(g1.z, g1.w);
    };
    if (g != cur_g) {
      flush();
      cur_g = g;
    }
    const float* gr = sgam + g * d;
    const float2 r2 = make_float2(r, r), nmur2 = make_float2(-mu * r, -mu * r);
    float2 s1 = make_float2(0.f, 0.f), s2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = lane + 32 * k;
      if (c < nch) {
        float2 xv[4], dyv[4], gg[4];
        if (MODE == GLN_GATE && R.r_x < 0) {  // gated norm input x = o (.) u
          float2 uu[4];
          row8(R.r_u, c, uu);
          row8(R.r_o, c, xv);
#pragma unroll
          for (int e = 0; e < 4; ++e) xv[e] = p2mul(xv[e], uu[e]);
        } else {
          row8(R.r_x, c, xv);
        }
        row8(0, c, dyv);
        gam(gr + c * 8, gg);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 xh = p2fma(xv[e], r2, nmur2);
          const float2 dxh = p2mul(dyv[e], gg[e]);
          pg[k][e] = p2fma(dyv[e], xh, pg[k][e]);
          pb[k][e] = p2add(pb[k][e], dyv[e]);
          s1 = p2add(s1, dxh);
          s2 = p2fma(dxh, xh, s2);
        }
      }
    }
    const float m1 = warp_sum(s1.x + s1.y) * inv_d, m2 = warp_sum(s2.x + s2.y) * inv_d;
    const float2 nm1 = make_float2(-m1, -m1), nm2 = make_float2(-m2, -m2);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = lane + 32 * k;
      if (c < nch) {
        float2 xv[4], dyv[4], gg[4], o[4], uu[4], oo[4];
        if (MODE == GLN_GATE) {
          row8(R.r_u, c, uu);
          row8(R.r_o, c, oo);
        }
        if (MODE == GLN_GATE && R.r_x < 0) {  // x = o (.) u, keeping o and u for the gate
#pragma unroll
          for (int e = 0; e < 4; ++e) xv[e] = p2mul(oo[e], uu[e]);
        } else {
          row8(R.r_x, c, xv);
        }
        row8(0, c, dyv);
        gam(gr + c * 8, gg);
        // dx = r (dy g - m1 - xhat m2)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 xh = p2fma(xv[e], r2, nmur2);
          o[e] = p2mul(p2fma(xh, nm2, p2fma(dyv[e], gg[e], nm1)), r2);
        }
        if (MODE == GLN_RESID) {
          float2 z[4];
          row8(R.r_dz, c, z);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            o[e] = p2add(o[e], z[e]);
            pc[k][e] = p2add(pc[k][e], z[e]);
          }
          store8p(a.dx + (int64_t)t * d + c * 8, o);
        } else if (MODE == GLN_GATE) {
          // o[] = dY; dO = dY * U;  dp_U = dY * O * silu'(p_U)
          float2 dO[4], du[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            dO[e] = p2mul(o[e], uu[e]);
            du[e] = p2mul(o[e], oo[e]);
          }
          if (R.r_pre >= 0) {
            float2 pp[4];
            row8(R.r_pre, c, pp);
            if (a.pre_dsilu) {
#pragma unroll
              for (int e = 0; e < 4; ++e) du[e] = p2mul(du[e], pp[e]);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) du[e] = make_float2(du[e].x * dsilu_f(pp[e].x), du[e].y * dsilu_f(pp[e].y));
            }
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) pc[k][e] = p2add(pc[k][e], du[e]);
          store8p(a.dx + (int64_t)t * d + c * 8, dO);
          store8p(a.dpu + (int64_t)t * a.ld_dp + c * 8, du);
        } else {
          store8p(a.dx + (int64_t)t * d + c * 8, o);
        }
      }
    }
    __syncwarp();  // every lane has consumed stage s
    if (lane == 0 && t + R.S < w_end) issue(t + R.S, s);
  }
  if (w_begin < w_end) flush();
  if (csum) {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int c = lane + 32 * k;
      if (c < nch)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          atomicAdd(&sacc[G * 2 * d + c * 8 + 2 * e], pc[k][e].x);
          atomicAdd(&sacc[G * 2 * d + c * 8 + 2 * e + 1], pc[k][e].y);
        }
    }
  }
  __syncthreads();
  if (csum)
    for (int i = threadIdx.x; i < d; i += blockDim.x) atomicAdd(a.dcol + i, sacc[G * 2 * d + i]);
  for (int i = threadIdx.x; i < G * 2 * d; i += blockDim.x) {
    const float v = sacc[i];
    if (v != 0.f) atomicAdd(a.part + i, v);
  }
}

// dgamma/dbeta (+)= accumulators
__global__ void gln_param_finish_kernel(const float* __restrict__ acc, int G, int d,
                                        float* __restrict__ dgamma, float* __restrict__ dbeta,
                                        int accumulate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G * 2 * d) return;
  const int g = i / (2 * d), w = (i / d) & 1, c = i % d;
  float* out = (w == 0 ? dgamma : dbeta) + g * d + c;
  *out = accumulate ? *out + acc[i] : acc[i];
}

// ------------------------------------------------------------------ host launchers

static int gln_nc(int d) { return (d + 255) / 256; }  // 8-element chunks per lane

static int gln_bwd_tok_per_warp(int ntok) {
  const int warps_wanted = 16 * num_sms() * GLNB_WARPS;  // ~16 blocks per SM worth of work
  int tpw = ceil_div(ntok > 0 ? ntok : 1, warps_wanted);
  return std::max(tpw, 32);
}
static int gln_bwd_blocks(int ntok) {
  return ceil_div(ceil_div(ntok > 0 ? ntok : 1, gln_bwd_tok_per_warp(ntok)), GLNB_WARPS);
}

size_t gln_bwd_ws_bytes(int ntok, int d, int G) {
  (void)ntok;
  return align_up((size_t)G * 2 * d * sizeof(float), 256);
}

template <class T, int NC>
static void gln_fwd_go(const T* x, const uint8_t* gid, const float* gamma, const float* beta, T* y,
                       float* mean, float* rstd, int ntok, int d, float eps, const T* gate,
                       int64_t ld_gate, cudaStream_t st) {
  // MINB resident 256-thread blocks per SM, each warp a contiguous run of tokens
  constexpr int smem = gln_fwd_smem<NC>();
  const int minb = gate != nullptr ? gln_fwd_minb<T, NC, true>() : gln_fwd_minb<T, NC, false>();
  const int warps = 8 * minb * num_sms();
  const int tpw = std::max(1, ceil_div(ntok, warps));
  const int blocks = ceil_div(ceil_div(ntok, tpw), 8);
  auto kern = gate != nullptr ? gln_fwd_kernel<T, NC, true> : gln_fwd_kernel<T, NC, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<blocks, 256, smem, st>>>(x, gid, gamma, beta, y, mean, rstd, ntok, d, eps, gate, ld_gate, tpw);
}

template <class T>
mtgr_status_t gln_fwd_launch(const T* x, const uint8_t* gid, const float* gamma,
                             const float* beta, T* y, float* mean, float* rstd, int ntok, int d,
                             float eps, cudaStream_t st, const T* gate, int64_t ld_gate) {
  if (ntok == 0) return MTGR_OK;
  ProfScope ps(PROF_GLN_FWD, st);
  switch (gln_nc(d)) {
    case 1: gln_fwd_go<T, 1>(x, gid, gamma, beta, y, mean, rstd, ntok, d, eps, gate, ld_gate, st); break;
    case 2: gln_fwd_go<T, 2>(x, gid, gamma, beta, y, mean, rstd, ntok, d, eps, gate, ld_gate, st); break;
    case 3: gln_fwd_go<T, 3>(x, gid, gamma, beta, y, mean, rstd, ntok, d, eps, gate, ld_gate, st); break;
    default: gln_fwd_go<T, 4>(x, gid, gamma, beta, y, mean, rstd, ntok, d, eps, gate, ld_gate, st); break;
  }
  return check_launch("gln_fwd");
}

template <class T, int MODE, int NC>
static void gln_bwd_go(const GlnBwdArgs<T>& a, int nb, size_t smem, cudaStream_t st) {
  cudaFuncSetAttribute(gln_bwd_kernel<T, MODE, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gln_bwd_kernel<T, MODE, NC><<<nb, 32 * GLNB_WARPS, smem, st>>>(a);
}

template <class T, int MODE>
static void gln_bwd_mode(const GlnBwdArgs<T>& a, int nb, size_t smem, cudaStream_t st) {
  switch (gln_nc(a.d)) {
    case 1: gln_bwd_go<T, MODE, 1>(a, nb, smem, st); break;
    case 2: gln_bwd_go<T, MODE, 2>(a, nb, smem, st); break;
    case 3: gln_bwd_go<T, MODE, 3>(a, nb, smem, st); break;
    default: gln_bwd_go<T, MODE, 4>(a, nb, smem, st); break;
  }
}

template <int MODE, int NC>
static void gln_bwd_bulk_go(const GlnBwdArgs<__nv_bfloat16>& a, const GlnRing& R, int blocks,
                            int threads, size_t smem, cudaStream_t st) {
  cudaFuncSetAttribute(gln_bwd_bulk_kernel<MODE, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gln_bwd_bulk_kernel<MODE, NC><<<blocks, threads, smem, st>>>(a, R);
}
template <int MODE>
static void gln_bwd_bulk_mode(const GlnBwdArgs<__nv_bfloat16>& a, const GlnRing& R, int blocks,
                              int threads, size_t smem, cudaStream_t st) {
  switch (gln_nc(a.d)) {
    case 1: gln_bwd_bulk_go<MODE, 1>(a, R, blocks, threads, smem, st); break;
    case 2: gln_bwd_bulk_go<MODE, 2>(a, R, blocks, threads, smem, st); break;
    case 3: gln_bwd_bulk_go<MODE, 3>(a, R, blocks, threads, smem, st); break;
    default: gln_bwd_bulk_go<MODE, 4>(a, R, blocks, threads, smem, st); break;
  }
}
static mtgr_status_t gln_bwd_bulk_launch(GlnBwdArgs<__nv_bfloat16> a, int mode, cudaStream_t st) {
  GlnRing R{};
  int n = 1;
  auto slot = [&](bool present) { return present ? n++ : -1; };
  R.r_x = slot(mode != GLN_GATE || a.x != nullptr);
  R.r_dz = slot(mode == GLN_RESID);
  R.r_o = slot(mode == GLN_GATE);
  R.r_u = slot(mode == GLN_GATE);
  R.r_pre = slot(mode == GLN_GATE && a.pre_u != nullptr);
  R.nrows = n;
  R.stage_bytes = (uint32_t)(n * a.d * 2);
  const size_t acc_bytes = align_up(((size_t)a.G * 3 * a.d + a.d) * sizeof(float), 128);  // + gamma
  R.ring_off = (uint32_t)acc_bytes;
  const size_t budget = 226 * 1024;  // of the 227 KB opt-in: 16 warps for the 4-row GLN2 stages at d = 512
  // three stages per warp while that still fits 14 warps per SM, else two (d = 768: 10 -> 15 warps)
  R.S = 3;
  if ((budget - acc_bytes) / ((size_t)3 * R.stage_bytes + 24) < 14) R.S = 2;
  int warps = (int)((budget - acc_bytes) / ((size_t)R.S * R.stage_bytes + R.S * 8));
  warps = std::max(1, std::min(16, warps));
  const int threads = 32 * warps;
  const size_t smem = acc_bytes + (size_t)warps * R.S * R.stage_bytes + (size_t)warps * R.S * 8;
  const int blocks = num_sms();
  a.tok_per_warp = ceil_div(a.ntok, blocks * warps);
  if (mode == GLN_GATE) gln_bwd_bulk_mode<GLN_GATE>(a, R, blocks, threads, smem, st);
  else if (mode == GLN_RESID) gln_bwd_bulk_mode<GLN_RESID>(a, R, blocks, threads, smem, st);
  else gln_bwd_bulk_mode<GLN_PLAIN>(a, R, blocks, threads, smem, st);
  return check_launch("gln_bwd_bulk");
}

template <class T>
mtgr_status_t gln_bwd_launch(const GlnBwdIO& io, int mode, float* part, float* dgamma,
                             float* dbeta, int accumulate, cudaStream_t st) {
  ProfScope ps(PROF_GLN_BWD, st);
  GlnBwdArgs<T> a{};
  a.dy = (const T*)io.dy; a.x = (const T*)io.x; a.mean = io.mean; a.rstd = io.rstd;
  a.gamma = io.gamma; a.gid = io.gid; a.dx = (T*)io.dx; a.part = part;
  a.ntok = io.ntok; a.d = io.d; a.G = io.G;
  a.o = (const T*)io.o; a.u = (const T*)io.u; a.pre_u = (const T*)io.pre_u; a.pre_dsilu = io.pre_dsilu; a.ld_a = io.ld_a;
  a.dpu = (T*)io.dpu; a.ld_dp = io.ld_dp; a.dz = (const T*)io.dz; a.dcol = io.dcol;
  a.tok_per_warp = gln_bwd_tok_per_warp(io.ntok);
  int nb = io.ntok > 0 ? gln_bwd_blocks(io.ntok) : 0;
  size_t smem = ((size_t)io.G * 2 * io.d + io.d) * sizeof(float);
  cudaMemsetAsync(part, 0, (size_t)io.G * 2 * io.d * sizeof(float), st);
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (io.ntok > 0 && gln_nc(io.d) <= 4) {
      MTGR_TRY(gln_bwd_bulk_launch(a, mode, st));
      nb = 0;
    }
  }
  if (nb > 0) {
    if (mode == GLN_GATE) gln_bwd_mode<T, GLN_GATE>(a, nb, smem, st);
    else if (mode == GLN_RESID) gln_bwd_mode<T, GLN_RESID>(a, nb, smem, st);
    else gln_bwd_mode<T, GLN_PLAIN>(a, nb, smem, st);
    MTGR_TRY(check_launch("gln_bwd"));
  }
  int n = io.G * 2 * io.d;
  gln_param_finish_kernel<<<ceil_div(n, 256), 256, 0, st>>>(part, io.G, io.d, dgamma, dbeta,
                                                            accumulate);
  return check_launch("gln_param_finish");
}

template mtgr_status_t gln_fwd_launch<float>(const float*, const uint8_t*, const float*,
                                             const float*, float*, float*, float*, int, int,
                                             float, cudaStream_t, const float*, int64_t);
template mtgr_status_t gln_fwd_launch<__nv_bfloat16>(const __nv_bfloat16*, const uint8_t*,
                                                     const float*, const float*, __nv_bfloat16*,
                                                     float*, float*, int, int, float,
                                                     cudaStream_t, const __nv_bfloat16*, int64_t);
template mtgr_status_t gln_bwd_launch<float>(const GlnBwdIO&, int, float*, float*, float*, int,
                                             cudaStream_t);
template mtgr_status_t gln_bwd_launch<__nv_bfloat16>(const GlnBwdIO&, int, float*, float*,
                                                     float*, int, cudaStream_t);

}  // namespace mtgr
