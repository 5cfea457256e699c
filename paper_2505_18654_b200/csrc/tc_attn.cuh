// Shared pieces of the tcgen05 jagged attention kernels (tc_attn.cu: forward, recompute and
// stored-score backward; tc_attn_kv.cu: the coupled dK/dV backward): tile constants, kernel
// arguments, the SiLU forms, and the work-item decode (rows never cross users; key / query
// ranges from the dynamic mask).
#pragma once
#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"
#include <cuda_fp16.h>

namespace mtgr {
namespace tca {

constexpr int DH = 256;
constexpr int BR = 128;                 // rows per CTA
constexpr int BC = 64;                  // columns per iterated tile
constexpr int KB = 1024;
constexpr int RT_BYTES = BR * DH * 2;   // 64 KB: 4 boxes {64 dh, 128 rows}
// key timestamps of the current tile (int64 x 64) and the barriers: after the epilogue tile
// (!TWO) / after the dbias scratch [208,216) KB (TWO)
constexpr int off_ts(bool two) { return (two ? 216 : 224) * KB; }
constexpr int off_bar(bool two) { return off_ts(two) + BC * 8; }
// after the barriers: the item's rab weights rab_w[h][0, nb) and the drab bins (fp32 x 64 each)
constexpr int off_rab(bool two) { return off_bar(two) + 512; }
constexpr int off_racc(bool two) { return off_rab(two) + 256; }
constexpr int SMEM_BYTES = off_racc(false) + 256 + 1024;
constexpr int NSM = 8;  // softmax/epilogue warps

enum { FWD = 0, DV = 1, DQ = 2, DK = 3 };

struct Args {
  mtgr_jagged_t jag;
  int H, d;
  int pmax, nitems;                         // row pairs per user (max), work items B*pmax*H
  int* ctr;                                 // work-queue counter (zeroed before the launch)
  __nv_bfloat16* out; int64_t ld_out;
  const __nv_bfloat16* e; int64_t ld_e;     // diagonal-term rows (E) of the epilogue
  const __nv_bfloat16* uu; int64_t ld_u;    // gate (FWD) / SiLU' source (bwd) rows, or NULL
  const float* diag;                        // [T][H]
  int pre_dsilu;                            // the pre rows hold silu'(p) already
  float* dbias;                             // bwd: red.add column sums of the outputs, or NULL
  long long* dbg;                           // debug timestamps (MTGR_ATTN_TRACE) or NULL
  // stored-score backward (DK writes P^T and dS^T, the DV / DQ products read them back):
  // matrices [H][st_rows][st_pitch] bf16, row = koff[u] + key (user-local), column = query
  __nv_bfloat16* st_p;                      // P^T  = silu(S^T) * m      (DK writes, or NULL)
  __nv_bfloat16* st_ds;                     // dS^T = dP^T silu'(S^T) m  (DK writes, or NULL)
  int64_t st_pitch, st_rows;
  const int* koff;                          // [B+1] padded key-row offsets (multiples of 256)
  int causal;                               // MTGR_MASK_CAUSAL: m_ij = [j <= i]
  int full;                                 // MTGR_MASK_FULL: m_ij = [j < ns + nr] or [i == j]
  int sc_cp;                                // score kernel: row operands via tcgen05.cp
  int row_cp;                               // FWD / DV: row operand via tcgen05.cp
  int c_align;                              // TRANS items of real-time keys start their query
                                            // range at the 256-aligned pair holding n_static
  // relative-attention bias (R#4; kernels instantiated with RAB): s_ij += rab_w[h][bucket(ts_i -
  // ts_j)]; drab (DQ only, the recompute backward) accumulates nu * dS per bucket
  const float* rab_w; float* drab; int nb;
};

// debug tracing (MTGR_ATTN_TRACE=1) of the CTA pair of cluster 1: slot layout [event][item]
// per CTA, events: 0 item start, 1 tiles done, 2 next R1 copied, 3 o_full, 4 epilogue done
// (softmax warp 4); 5 first S issued, 6 last acc issued (MMA warp); 7 R1 load issued, 8 last C1
// load issued (producer); 9 ntiles (value); 10*64 = time base after the start-up cluster barrier
#define DBG_ON (a.dbg != nullptr && (blockIdx.x >> 1) == 1)
#define DBGV(ev, i, val) do { if (DBG_ON && (i) < 64) a.dbg[(blockIdx.x & 1) * 20 * 64 + (ev) * 64 + (i)] = (val); } while (0)
#define DBG(ev, i) DBGV(ev, i, clock64())

// rab bucket (R#4): min(nb - 1, floor(log2(max(|dt|, 1)))); nb1 = nb - 1 (0 and 1 both map to
// bucket 0).  Default: one round-toward-zero int64 -> fp32 conversion (MTGR_RAB_BKT=1: integer
// |dt| | 1 and a 64-bit count of leading zeros)
#ifndef MTGR_RAB_BKT
#define MTGR_RAB_BKT 3
#endif
__device__ __forceinline__ int rab_bkt(long long dt, int nb1) {
#if MTGR_RAB_BKT == 1  // integer form (A/B: 1.15x slower FWD, 1.12x kv at small with NB = 16)
  const unsigned long long x = (unsigned long long)(dt < 0 ? -dt : dt) | 1ull;
  return min(63 - __clzll((long long)x), nb1);
#else
  // round-toward-zero conversion never crosses up to the next power of two: the exponent of
  // rz(|dt|) is floor(log2 |dt|) exactly; dt = 0 gives exponent field 0 (clamped to bucket 0)
  const int e = (int)((__float_as_uint(__ll2float_rz(dt)) >> 23) & 0xffu) - 127;
  return min(max(e, 0), nb1);
#endif
}
// s[e] += w[bucket(ts_row - ts_col[e])] for n score values of one row (fp32 bit patterns)
template <int N>
__device__ __forceinline__ void add_rab(uint32_t* s, long long ts_row, const long long* ts_col,
                                        const float* w, int nb1) {
#pragma unroll
  for (int e = 0; e < N; ++e)
    s[e] = __float_as_uint(__uint_as_float(s[e]) + w[rab_bkt(ts_row - ts_col[e], nb1)]);
}

__device__ __forceinline__ float silu_fast(float s) {
  const float h = 0.5f * s;
  return fmaf(h, sm100::tanh_approx(h), h);
}
__device__ __forceinline__ float dsilu_fast(float s) {
  const float sg = fmaf(0.5f, sm100::tanh_approx(0.5f * s), 0.5f);
  return fmaf(s * sg, 1.0f - sg, sg);
}
// packed fp32 pairs (FFMA2 / FMUL2 / FADD2 on sm_100): half the issue slots of scalar math
__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(d);
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(d);
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(d);
}
// sigma(s) = 0.5 + 0.5 tanh(s/2) for a pair (two MUFU.TANH; the f16x2 / bf16x2 forms split into
// two MUFU ops on sm_100 as well, plus conversions)
__device__ __forceinline__ float2 sigmoid2_fast(float2 s) {
  const float2 h = f2mul(s, make_float2(0.5f, 0.5f));
  const float2 tf = make_float2(sm100::tanh_approx(h.x), sm100::tanh_approx(h.y));
  return f2fma(tf, make_float2(0.5f, 0.5f), make_float2(0.5f, 0.5f));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// 16-byte chunk j (0..7) of row r inside a SWIZZLE_128B box of 128-byte rows
__device__ __forceinline__ uint32_t sw128(int r, int j) { return r * 128 + ((j ^ (r & 7)) << 4); }

// One work item = (user u, row pair p, head h): rows [p*256, p*256+256) of user u, 128 per CTA.
struct Item {
  UserSpan us;
  int u, h, hcol, pr0, r0, kv_end, c_begin, ntiles;
  bool need_e;  // some rows of this CTA are candidates (diagonal terms outside the key range)
};

template <bool TRANS>
__device__ __forceinline__ bool decode_item(const Args& a, int k, uint32_t crank, Item& it) {
  it.h = k % a.H;
  const int rest = k / a.H;
  const int p = rest % a.pmax;
  it.u = rest / a.pmax;
  it.us = load_user(a.jag, it.u);
  it.pr0 = p * 2 * BR;
  if (it.pr0 >= it.us.L) return false;
  it.r0 = it.pr0 + (int)crank * BR;
  it.hcol = it.h * DH;
  // keys that can be visible to some row (beyond them only the candidates' own diagonal):
  // dynamic mask [0, ns + nr); causal mask every key
  it.kv_end = a.causal ? it.us.L : it.us.ns + it.us.nr;
  const int pair_end = min(it.us.L, it.pr0 + 2 * BR);
  int c_end = 0;
  it.c_begin = 0;
  if (a.causal) {  // keys [0, pair_end) of a query pair; queries [pr0, L) of a key pair
    if (!TRANS) c_end = pair_end;
    else { it.c_begin = it.pr0; c_end = it.us.L; }
  } else if (a.full) {  // keys [0, ns + nr) for every query (candidate keys: their diagonal only)
    if (!TRANS) c_end = it.kv_end;
    else if (it.pr0 < it.kv_end) c_end = it.us.L;
  } else if (!TRANS) {
    c_end = (pair_end > it.us.ns) ? it.kv_end : it.us.ns;
  } else if (it.pr0 < it.kv_end) {
    // keys that only non-static queries read.  With c_align the range starts at the query pair
    // holding n_static, so that every query pair that reads these keys finds them stored (its
    // static rows read masked zeros)
    it.c_begin = (it.pr0 < it.us.ns) ? 0 : (a.c_align ? (it.us.ns / (2 * BR)) * (2 * BR) : it.us.ns);
    c_end = it.us.L;
  }
  it.ntiles = c_end > it.c_begin ? (c_end - it.c_begin + BC - 1) / BC : 0;
  it.need_e = it.r0 + BR > it.kv_end && it.r0 < it.us.L;
  return true;
}

}  // namespace tca

// tc_attn_kv.cu: the coupled dK / dV backward (X pairs: S^T, P^T, dV; Y pairs: dP^T, dS^T, dK and
// the stored dS^T rows of the dQ GEMM).  ax / ay: per-role arguments (jag, H, d, koff; ay also
// st_ds / st_pitch / st_rows); sync_ws: attn_kv_ws_bytes() bytes
mtgr_status_t attn_kv_launch(const AttnIO& io, const tca::Args& ax, const tca::Args& ay, void* sync_ws,
                             cudaStream_t st);
}  // namespace mtgr
