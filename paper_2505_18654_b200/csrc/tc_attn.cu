// tcgen05 jagged HSTU attention, forward and backward (Eq.5, dynamic mask
// P:323-346), head dim 256 (every MTGR config of Table 2: 512/2, 768/3).
//
// One CTA = (128-row tile, head, user); rows never cross users.  Four modes share one kernel:
//
//   mode | rows (R1, in TMEM) | R2 (smem) | column tile C1 | C2 / X     | T tile          | acc
//   FWD  | Q                  |  -        | K (64 keys)    | X = V      | P  = silu(S)*m  | O
//   DV   | K                  |  -        | Q (64 queries) | X = dO     | P^T             | dV
//   DQ   | Q                  | dO        | K              | C2 = V     | dS = dP*silu'(S)*m | dQ (X = C1)
//   DK   | K                  | V         | Q              | C2 = dO    | dS^T            | dK (X = C1)
//
// Per column tile:  S = R1 C1^T (tcgen05.mma, A from TMEM, B = C1 K-major smem, M=128 N=64
// K=256) [and dP = R2 C2^T, SS];  4 "softmax" warps tcgen05.ld S (and dP), apply the mask
// predicate in registers and SiLU / SiLU' (tanh.approx), write the bf16 T tile into a
// SWIZZLE_128B smem buffer;  acc += T X (M=128 N=256 K=64, B = X MN-major — the same
// TMA-loaded tile read with an MN-major descriptor).  The 1/N factor, the diagonal term of
// non-static tokens (R#9: candidates and real-time tokens see themselves), the gate
// (FWD: y = o*u) and the QKV activation backward (silu'(p)) are fused into the epilogue.
// Keys of a query tile are restricted to [0, n_static + n_rt) (candidate keys are visible only
// to themselves, rule 3 P:338) and to [0, n_static) when every row of the tile is static
// (R#8), so fully masked tiles are never loaded.
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator,
// w4-w11 softmax/epilogue (two warps per TMEM lane quadrant, thread = row = TMEM lane).  TMEM: R1 [0,128) (bf16 pairs),
// acc [128,384), S buffers [384,512).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"
#include "sm100.cuh"

namespace mtgr {
namespace tca {

constexpr int DH = 256;
constexpr int BR = 128;                 // rows per CTA
constexpr int BC = 64;                  // columns per iterated tile
constexpr int CT_BYTES = BC * DH * 2;   // 32 KB: 4 boxes {64 dh, 64 rows}
constexpr int R2_BYTES = BR * DH * 2;   // 64 KB: 4 boxes {64 dh, 128 rows}
constexpr int T_BYTES = BR * BC * 2;    // 16 KB
constexpr int OFF_T = 192 * 1024;
constexpr int OFF_TS = OFF_T + 2 * T_BYTES;
constexpr int OFF_BAR = OFF_TS + 2 * BC * 8;
constexpr int SMEM_BYTES = OFF_BAR + 256 + 1024;
constexpr uint32_t COL_R1 = 0, COL_ACC = 128, COL_S = 384;

enum { FWD = 0, DV = 1, DQ = 2, DK = 3 };

struct Args {
  mtgr_jagged_t jag;
  int H, d;
  const __nv_bfloat16* r1; int64_t ld_r1;   // row operand 1 (block start)
  const __nv_bfloat16* e; int64_t ld_e;     // epilogue diagonal vector
  const __nv_bfloat16* u; int64_t ld_u;     // FWD gate
  const __nv_bfloat16* pre; int64_t ld_pre; // silu' source block or NULL
  __nv_bfloat16* out; int64_t ld_out;
  __nv_bfloat16* out2;                      // FWD y (ld_out)
  const float* diag;                        // [T][H]
  long long* dbg;                           // debug timestamps (MTGR_ATTN_TRACE) or NULL
};

// debug tracing of one CTA (MTGR_ATTN_TRACE=1): slot layout [role][event][tile]
#define DBG_ON (a.dbg != nullptr && blockIdx.x == 2 && blockIdx.y == 0 && blockIdx.z == 0)
#define DBG(slot) do { if (DBG_ON) a.dbg[(slot)] = clock64(); } while (0)

__device__ __forceinline__ float silu_fast(float s) {
  const float h = 0.5f * s;
  return fmaf(h, sm100::tanh_approx(h), h);
}
__device__ __forceinline__ float dsilu_fast(float s) {
  const float sg = fmaf(0.5f, sm100::tanh_approx(0.5f * s), 0.5f);
  return fmaf(s * sg, 1.0f - sg, sg);
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int MODE>
__global__ void __launch_bounds__(384, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmC1, const __grid_constant__ CUtensorMap tmC2,
                   const __grid_constant__ CUtensorMap tmR2, Args a) {
  using namespace sm100;
  constexpr bool TWO = (MODE == DQ || MODE == DK);
  constexpr bool TRANS = (MODE == DV || MODE == DK);
  constexpr int STAGES = TWO ? 2 : 3;
  constexpr int STAGE_BYTES = 2 * CT_BYTES;

  const int u = blockIdx.z, h = blockIdx.y, r0 = blockIdx.x * BR;
  const UserSpan us = load_user(a.jag, u);
  if (r0 >= us.L) return;
  const int kv_end = us.ns + us.nr;
  int c_begin = 0, c_end = 0;
  if (!TRANS) {
    c_end = (min(BR, us.L - r0) + r0 > us.ns) ? kv_end : us.ns;
  } else if (r0 < kv_end) {
    c_begin = (r0 < us.ns) ? 0 : us.ns;
    c_end = us.L;
  }
  const int ntiles = c_end > c_begin ? (c_end - c_begin + BC - 1) / BC : 0;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sR2 = smem;                              // TWO only (64 KB)
  uint8_t* sStage = smem + (TWO ? R2_BYTES : 0);    // STAGES x 64 KB
  uint8_t* sT = smem + OFF_T;                       // 2 x 16 KB
  long long* sTs = reinterpret_cast<long long*>(smem + OFF_TS);  // [2][64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* kv_full = bars;            // [3]
  uint64_t* kv_empty = bars + 3;       // [3]
  uint64_t* s_full = bars + 6;         // [2]
  uint64_t* s_free = bars + 8;         // [2]
  uint64_t* t_full = bars + 10;        // [2]
  uint64_t* t_free = bars + 12;        // [2]
  uint64_t* r1_ready = bars + 14;
  uint64_t* r2_full = bars + 15;
  uint64_t* o_full = bars + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) DBG(10 * 64 + 4);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmC1);
    tma_prefetch(&tmC2);
    if (TWO) tma_prefetch(&tmR2);
    for (int s = 0; s < 3; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1); mbar_init(&s_free[b], 256);
      mbar_init(&t_full[b], 256); mbar_init(&t_free[b], 1);
    }
    mbar_init(r1_ready, 256);
    mbar_init(r2_full, 1);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int hcol = h * DH;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0 && ntiles > 0) {
      if (TWO) {
        mbar_expect_tx(r2_full, R2_BYTES);
#pragma unroll
        for (int c = 0; c < 4; ++c) tma_load_2d(sR2 + c * (R2_BYTES / 4), &tmR2, r2_full, hcol + c * 64, us.off + r0);
      }
      for (int t = 0; t < ntiles; ++t) {
        const int stage = t % STAGES;
        mbar_wait(&kv_empty[stage], ((t / STAGES) & 1) ^ 1);
        mbar_expect_tx(&kv_full[stage], STAGE_BYTES);
        const int row = us.off + c_begin + t * BC;
        uint8_t* c1 = sStage + stage * STAGE_BYTES;
#pragma unroll
        for (int c = 0; c < 4; ++c) tma_load_2d(c1 + c * (CT_BYTES / 4), &tmC1, &kv_full[stage], hcol + c * 64, row);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          tma_load_2d(c1 + CT_BYTES + c * (CT_BYTES / 4), &tmC2, &kv_full[stage], hcol + c * 64, row);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      if (ntiles == 0) {
        mbar_arrive(o_full);
      } else {
        constexpr uint32_t idesc_s = idesc_bf16_f32(BR, BC, 0, 0);
        constexpr uint32_t idesc_acc = idesc_bf16_f32(BR, DH, 0, 1);
        mbar_wait(r1_ready, 0);
        if (TWO) mbar_wait(r2_full, 0);
        tc_fence_after();
        const uint32_t t_base = smem_u32(sT);
        const uint32_t r2_base = smem_u32(sR2);
        for (int t = 0; t <= ntiles; ++t) {
          if (t < ntiles) {
            const int stage = t % STAGES;
            if (t < 64) DBG(0 * 64 + t);
            mbar_wait(&kv_full[stage], (t / STAGES) & 1);
            if (t < 64) DBG(1 * 64 + t);
            const int sb = TWO ? 0 : (t & 1);
            const int use = TWO ? t : (t >> 1);
            mbar_wait(&s_free[sb], (use & 1) ^ 1);
            if (t < 64) DBG(2 * 64 + t);
            tc_fence_after();
            const uint32_t c1 = smem_u32(sStage + stage * STAGE_BYTES);
            const uint32_t s_col = tmem + COL_S + sb * BC;
#pragma unroll
            for (int k = 0; k < DH / 16; ++k)
              mma_bf16_ts(s_col, tmem + COL_R1 + k * 8,
                          desc_sw128(c1 + (k >> 2) * (CT_BYTES / 4) + (k & 3) * 32, 16, 1024), idesc_s,
                          k > 0);
            if (TWO) {
              const uint32_t c2 = c1 + CT_BYTES;
#pragma unroll
              for (int k = 0; k < DH / 16; ++k)
                mma_bf16_ss(tmem + COL_S + BC,
                            desc_sw128(r2_base + (k >> 2) * (R2_BYTES / 4) + (k & 3) * 32, 16, 1024),
                            desc_sw128(c2 + (k >> 2) * (CT_BYTES / 4) + (k & 3) * 32, 16, 1024),
                            idesc_s, k > 0);
            }
            mma_commit(&s_full[sb]);
          }
          if (t >= 1) {
            const int tp = t - 1, tb = tp & 1, sp = tp % STAGES;
            if (tp < 64) DBG(3 * 64 + tp);
            mbar_wait(&t_full[tb], (tp >> 1) & 1);
            if (tp < 64) DBG(4 * 64 + tp);
            tc_fence_after();
            const uint32_t x = smem_u32(sStage + sp * STAGE_BYTES) + (TWO ? 0 : CT_BYTES);
#pragma unroll
            for (int k = 0; k < BC / 16; ++k)
              mma_bf16_ss(tmem + COL_ACC, desc_sw128(t_base + tb * T_BYTES + k * 32, 16, 1024),
                          desc_sw128(x + k * 2048, CT_BYTES / 4, 1024), idesc_acc, (tp > 0 || k > 0));
            mma_commit(&t_free[tb]);
            mma_commit(&kv_empty[sp]);
          }
        }
        mma_commit(o_full);
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax + epilogue
    // 8 warps: quadrant q = warp % 4 owns TMEM lanes (rows) q*32..q*32+31; half = which 32 of the
    // 64 tile columns (and which 128 of the 256 accumulator columns) the warp handles.
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int row = q * 32 + lane;
    const int my = r0 + row;                 // user-local index of this thread's row
    const int64_t g = (int64_t)us.off + my;  // global token index
    const int T = a.jag.total_tokens;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    // R1 row (this warp's 128 head-dim columns) -> TMEM as bf16 pairs
#pragma unroll 1
    for (int cc = 0; cc < 2; ++cc) {
      uint32_t w[32];
      if (g < T) {
        const uint4* src = reinterpret_cast<const uint4*>(a.r1 + g * a.ld_r1 + hcol + half * 128 + cc * 64);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint4 v = __ldg(src + i);
          w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) w[i] = 0u;
      }
      tmem_st32(tmem + COL_R1 + half * 64 + cc * 32 + lane_off, w);
    }
    tmem_st_wait();
    tc_fence_before();
    mbar_arrive(r1_ready);
    if (warp == 4 && lane == 0) DBG(10 * 64 + 3);

    const long long my_ts = (my < us.L && a.jag.ts) ? a.jag.ts[g] : 0;
    const bool need_ts_rows = TRANS && (r0 + BR > us.ns) && (r0 < kv_end);
    const int j_half = half * 32;
#pragma unroll 1
    for (int t = 0; t < ntiles; ++t) {
      const int c0 = c_begin + t * BC;
      const bool need_ts = TRANS ? need_ts_rows : (c0 + BC > us.ns && c0 < kv_end);
      long long* tsb = sTs;
      if (need_ts) {  // uniform over the 8 softmax warps
        const int i = threadIdx.x - 128;
        named_bar_sync(1, 256);  // everyone is done reading the previous tile's times
        if (i < BC) tsb[i] = (c0 + i < us.L && a.jag.ts) ? a.jag.ts[us.off + c0 + i] : 0;
        named_bar_sync(1, 256);
      }
      const int sb = TWO ? 0 : (t & 1);
      const int use = TWO ? t : (t >> 1);
      const bool dbgt = warp == 4 && lane == 0 && t < 64;
      if (dbgt) DBG(5 * 64 + t);
      mbar_wait(&s_full[sb], use & 1);
      if (dbgt) DBG(6 * 64 + t);
      tc_fence_after();
      uint32_t s[32];
      uint32_t dp[TWO ? 32 : 1];
      tmem_ld32(tmem + COL_S + sb * BC + j_half + lane_off, s);
      if constexpr (TWO) {
        uint32_t (&d0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&dp[0]);
        tmem_ld32(tmem + COL_S + BC + j_half + lane_off, d0);
      }
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&s_free[sb]);
      // visibility of this warp's 32 columns for this row (dynamic mask, R#8-R#12)
      const int cb = c0 + j_half;
      uint32_t vis;
      if (!TRANS) {
        if (cb + 32 <= us.ns) {
          vis = 0xffffffffu;
        } else {
          vis = 0;
          const bool rs = my < us.ns;
#pragma unroll 8
          for (int jj = 0; jj < 32; ++jj) {
            const int j = cb + jj;
            const bool v = j < kv_end && (j < us.ns || (!rs && tsb[j_half + jj] < my_ts));
            vis |= (uint32_t)v << jj;
          }
        }
      } else {
        if (my < us.ns) {
          const int nvalid = us.L - cb;
          vis = nvalid >= 32 ? 0xffffffffu : (nvalid <= 0 ? 0u : ((1u << nvalid) - 1u));
        } else if (my < kv_end) {
          vis = 0;
#pragma unroll 8
          for (int jj = 0; jj < 32; ++jj) {
            const int i = cb + jj;
            const bool v = i < us.L && i >= us.ns && my_ts < tsb[j_half + jj];
            vis |= (uint32_t)v << jj;
          }
        } else {
          vis = 0;
        }
      }
      // T values -> bf16 -> swizzled smem (row = 128 B, 16-byte chunk c at c ^ (row & 7))
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        const float s0 = __uint_as_float(s[e]), s1 = __uint_as_float(s[e + 1]);
        float v0, v1;
        if constexpr (TWO) {
          v0 = __uint_as_float(dp[e]) * dsilu_fast(s0);
          v1 = __uint_as_float(dp[e + 1]) * dsilu_fast(s1);
        } else {
          v0 = silu_fast(s0);
          v1 = silu_fast(s1);
        }
        if (vis != 0xffffffffu) {
          v0 = ((vis >> e) & 1u) ? v0 : 0.f;
          v1 = ((vis >> (e + 1)) & 1u) ? v1 : 0.f;
        }
        pk[e >> 1] = pack2(v0, v1);
      }
      const int tb = t & 1;
      if (dbgt) DBG(7 * 64 + t);
      mbar_wait(&t_free[tb], ((t >> 1) & 1) ^ 1);
      if (dbgt) DBG(8 * 64 + t);
      uint8_t* trow = sT + tb * T_BYTES + row * 128;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int chunk = half * 4 + c;
        *reinterpret_cast<uint4*>(trow + ((chunk ^ (row & 7)) << 4)) =
            make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(&t_full[tb]);
      if (dbgt) DBG(9 * 64 + t);
    }

    // ---------------------------------------------------------------- epilogue
    if (warp == 4 && lane == 0) DBG(10 * 64 + 0);
    mbar_wait(o_full, 0);
    if (warp == 4 && lane == 0) DBG(10 * 64 + 1);
    tc_fence_after();
    const bool row_ok = my < us.L;
    const float dg = row_ok ? a.diag[g * a.H + h] : 0.f;
#pragma unroll 1
    for (int cc = 0; cc < 4; ++cc) {
      const int acol = half * 128 + cc * 32;
      uint32_t r[32];
      if (ntiles > 0) {
        tmem_ld32(tmem + COL_ACC + acol + lane_off, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = 0u;
      }
      if (!row_ok) continue;
      const int col = hcol + acol;
      float v[32];
      const uint4* ep = reinterpret_cast<const uint4*>(a.e + g * a.ld_e + col);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 w = __ldg(ep + i);
        const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float2 f = __bfloat1622float2(hh[k]);
          v[8 * i + 2 * k] = fmaf(us.nu, __uint_as_float(r[8 * i + 2 * k]), dg * f.x);
          v[8 * i + 2 * k + 1] = fmaf(us.nu, __uint_as_float(r[8 * i + 2 * k + 1]), dg * f.y);
        }
      }
      uint4* op = reinterpret_cast<uint4*>(a.out + g * a.ld_out + col);
      if (MODE == FWD) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          op[i] = make_uint4(pack2(v[8 * i], v[8 * i + 1]), pack2(v[8 * i + 2], v[8 * i + 3]),
                             pack2(v[8 * i + 4], v[8 * i + 5]), pack2(v[8 * i + 6], v[8 * i + 7]));
        const uint4* up = reinterpret_cast<const uint4*>(a.u + g * a.ld_u + col);
        uint4* yp = reinterpret_cast<uint4*>(a.out2 + g * a.ld_out + col);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint4 w = __ldg(up + i);
          const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&w);
          float y[8];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            float2 f = __bfloat1622float2(hh[k]);
            y[2 * k] = v[8 * i + 2 * k] * f.x;
            y[2 * k + 1] = v[8 * i + 2 * k + 1] * f.y;
          }
          yp[i] = make_uint4(pack2(y[0], y[1]), pack2(y[2], y[3]), pack2(y[4], y[5]), pack2(y[6], y[7]));
        }
      } else {
        if (a.pre) {
          const uint4* pp = reinterpret_cast<const uint4*>(a.pre + g * a.ld_pre + col);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            uint4 w = __ldg(pp + i);
            const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              float2 f = __bfloat1622float2(hh[k]);
              v[8 * i + 2 * k] *= dsilu_f(f.x);
              v[8 * i + 2 * k + 1] *= dsilu_f(f.y);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          op[i] = make_uint4(pack2(v[8 * i], v[8 * i + 1]), pack2(v[8 * i + 2], v[8 * i + 3]),
                             pack2(v[8 * i + 4], v[8 * i + 5]), pack2(v[8 * i + 6], v[8 * i + 7]));
      }
    }
  }
  if (warp == 4 && lane == 0) DBG(10 * 64 + 2);
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int MODE>
static mtgr_status_t launch_mode(const AttnIO& io, const void* c1, int64_t ld_c1, const void* c2,
                                 int64_t ld_c2, const void* r2, int64_t ld_r2, const Args& args,
                                 cudaStream_t st) {
  const int T = io.jag.total_tokens, d = io.d;
  CUtensorMap m1, m2, m3;
  MTGR_TRY(make_tmap_bf16(&m1, c1, d, T, ld_c1, 64, BC));
  MTGR_TRY(make_tmap_bf16(&m2, c2, d, T, ld_c2, 64, BC));
  if (r2) MTGR_TRY(make_tmap_bf16(&m3, r2, d, T, ld_r2, 64, BR));
  else m3 = m1;
  dim3 grid(ceil_div(io.jag.max_len, BR), io.H, io.jag.num_users);
  ProfScope ps(MODE == FWD ? PROF_ATTN_FWD : MODE == DV ? PROF_ATTN_DV : MODE == DK ? PROF_ATTN_DK : PROF_ATTN_DQ, st);
  cudaFuncSetAttribute(attn_tc_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  static const bool trace = getenv("MTGR_ATTN_TRACE") != nullptr;
  Args a2 = args;
  if (trace) {  // debug only: time-stamp one CTA's pipeline events
    cudaMalloc(&a2.dbg, 11 * 64 * sizeof(long long));
    cudaMemsetAsync(a2.dbg, 0, 11 * 64 * sizeof(long long), st);
  }
  attn_tc_kernel<MODE><<<grid, 384, SMEM_BYTES, st>>>(m1, m2, m3, a2);
  if (trace) {
    long long h[11 * 64];
    cudaMemcpyAsync(h, a2.dbg, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(a2.dbg);
    fprintf(stderr, "ATTN_TRACE mode=%d", MODE);
    for (int i = 0; i < 11 * 64; ++i) fprintf(stderr, " %lld", h[i]);
    fprintf(stderr, "\n");
  }
  return check_launch("attn_tc");
}

}  // namespace tca

bool attn_tc_supported(int dh) { return dh == tca::DH; }

mtgr_status_t attn_tc_fwd_launch(const AttnIO& io, cudaStream_t st) {
  using namespace tca;
  if (io.jag.num_users == 0 || io.jag.max_len == 0 || io.jag.total_tokens == 0) return MTGR_OK;
  MTGR_CHECK(io.u && io.y, MTGR_E_UNSUPPORTED, "tc attention forward needs the gate (u, y)");
  typedef __nv_bfloat16 bf;
  Args a{};
  a.jag = io.jag; a.H = io.H; a.d = io.d;
  a.r1 = (const bf*)io.q; a.ld_r1 = io.ld;
  a.e = (const bf*)io.v; a.ld_e = io.ld;
  a.u = (const bf*)io.u; a.ld_u = io.ld;
  a.out = (bf*)io.o; a.out2 = (bf*)io.y; a.ld_out = io.d;
  a.diag = io.diag_a;
  return launch_mode<FWD>(io, io.k, io.ld, io.v, io.ld, nullptr, 0, a, st);
}

mtgr_status_t attn_tc_bwd_launch(const AttnIO& io, cudaStream_t st) {
  using namespace tca;
  if (io.jag.num_users == 0 || io.jag.max_len == 0 || io.jag.total_tokens == 0) return MTGR_OK;
  typedef __nv_bfloat16 bf;
  const bf* pre = (const bf*)io.pre;
  {  // dV = nu P^T dO (+ diag a_jj dO_j), * silu'(p_V)
    Args a{};
    a.jag = io.jag; a.H = io.H; a.d = io.d;
    a.r1 = (const bf*)io.k; a.ld_r1 = io.ld;
    a.e = (const bf*)io.dO; a.ld_e = io.d;
    a.pre = pre ? pre + 2 * (int64_t)io.d : nullptr; a.ld_pre = io.ld_pre;
    a.out = (bf*)io.dv; a.ld_out = io.ld_out;
    a.diag = io.diag_a;
    MTGR_TRY(launch_mode<DV>(io, io.q, io.ld, io.dO, io.d, nullptr, 0, a, st));
  }
  {  // dK = nu dS^T Q (+ diag ds_jj q_j), * silu'(p_K)
    Args a{};
    a.jag = io.jag; a.H = io.H; a.d = io.d;
    a.r1 = (const bf*)io.k; a.ld_r1 = io.ld;
    a.e = (const bf*)io.q; a.ld_e = io.ld;
    a.pre = pre ? pre + (int64_t)io.d : nullptr; a.ld_pre = io.ld_pre;
    a.out = (bf*)io.dk; a.ld_out = io.ld_out;
    a.diag = io.diag_ds;
    MTGR_TRY(launch_mode<DK>(io, io.q, io.ld, io.dO, io.d, io.v, io.ld, a, st));
  }
  {  // dQ = nu dS K (+ diag ds_ii k_i), * silu'(p_Q)
    Args a{};
    a.jag = io.jag; a.H = io.H; a.d = io.d;
    a.r1 = (const bf*)io.q; a.ld_r1 = io.ld;
    a.e = (const bf*)io.k; a.ld_e = io.ld;
    a.pre = pre; a.ld_pre = io.ld_pre;
    a.out = (bf*)io.dq; a.ld_out = io.ld_out;
    a.diag = io.diag_ds;
    MTGR_TRY(launch_mode<DQ>(io, io.k, io.ld, io.v, io.ld, io.dO, io.d, a, st));
  }
  return MTGR_OK;
}

}  // namespace mtgr
