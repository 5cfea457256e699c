// tcgen05 jagged HSTU attention, forward and backward (Eq.5, dynamic mask
// P:323-346), head dim 256 (every MTGR config of Table 2: 512/2, 768/3).
//
// One CTA = (128-row tile, head, user); rows never cross users.  Four modes share one kernel:
//
//   mode | rows (R1, in TMEM) | R2 (smem) | column tile C1 | X (acc B)  | T tile            | acc
//   FWD  | Q                  |  -        | K (64 keys)    | V          | P  = silu(S)*m    | O
//   DV   | K                  |  -        | Q (64 queries) | dO         | P^T               | dV
//   DQ   | Q                  | dO        | K              | K  (= C1)  | dS = dP*silu'(S)*m| dQ
//   DK   | K                  | V         | Q              | Q  (= C1)  | dS^T              | dK
//   (DQ/DK also stream C2 = V / dO for dP = R2 C2^T.)
//
// Per column tile:  S = R1 C1^T (tcgen05.mma SS: A = R1 resident in smem, B = C1 K-major,
// M=128 N=64 K=256) [and dP = R2 C2^T];  8 "softmax" warps tcgen05.ld S (and dP), apply the
// mask predicate in registers and SiLU / SiLU' (tanh.approx), and tcgen05.st the bf16 T tile
// into TMEM;  acc += T X (A = T from TMEM, B = X MN-major — the same TMA-loaded tile read with
// an MN-major descriptor, M=128 N=256 K=64).  (Measured: with A from TMEM an N=64 MMA is bound
// by the TMEM A-operand read, ~70 cycles instead of 32, so the N=64 score MMAs read A from smem
// and only the N=256 accumulate MMAs read A from TMEM.)
// The 1/N factor, the diagonal term of non-static tokens (R#9: candidates and real-time tokens
// see themselves), the gate (FWD: y = o*u) and the QKV activation backward (silu'(p)) are fused
// into the epilogue, which stages E/U tiles and the outputs in shared memory (TMA in, coalesced
// row stores out).  Keys of a query tile are restricted to [0, n_static + n_rt) (candidate keys
// are visible only to themselves, rule 3 P:338) and to [0, n_static) when every row of the tile
// is static (R#8), so fully masked tiles are never loaded.
//
// Warp roles (384 threads): w0 TMA producer (R1, R2, C1, E, U), w1 MMA issuer, w2 TMEM allocator,
// w3 TMA producer (X or C2), w4-w11 softmax/epilogue (two warps per TMEM lane quadrant,
// thread = row = TMEM lane).  TMEM: acc [0,256), S [256,384) (two buffers, or S and dP),
// T [384,448) (two buffers of bf16 pairs).
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
constexpr int KB = 1024;
constexpr int RT_BYTES = BR * DH * 2;   // 64 KB: 4 boxes {64 dh, 128 rows}
constexpr int T_BYTES = BR * BC * 2;    // 16 KB
constexpr int OFF_T = 192 * KB;
constexpr int OFF_TS = OFF_T + 2 * T_BYTES;
constexpr int OFF_BAR = OFF_TS + BC * 8;
constexpr int SMEM_BYTES = OFF_BAR + 512 + 1024;
constexpr int NSM = 8;  // softmax/epilogue warps

enum { FWD = 0, DV = 1, DQ = 2, DK = 3 };

struct Args {
  mtgr_jagged_t jag;
  int H, d;
  __nv_bfloat16* out; int64_t ld_out;
  __nv_bfloat16* out2;                      // FWD y (ld_out)
  const float* diag;                        // [T][H]
  int has_u;                                // U / pre tile present
  int pre_dsilu;                            // the pre tile holds silu'(p) already
  float* dbias;                             // bwd: red.add column sums of the outputs, or NULL
  long long* dbg;                           // debug timestamps (MTGR_ATTN_TRACE) or NULL
};

// debug tracing of one CTA (MTGR_ATTN_TRACE=1): slot layout [event][tile]
// (the CTA pair (2,0,0) / (3,0,0); slot 10*64+10 = after the start-up cluster barrier, the
// common time base of the two SMs' clocks)
#define DBG_ON (a.dbg != nullptr && (blockIdx.x == 2 || blockIdx.x == 3) && blockIdx.y == 0 && blockIdx.z == 0)
#define DBG(slot) do { if (DBG_ON) a.dbg[(blockIdx.x - 2) * 11 * 64 + (slot)] = clock64(); } while (0)

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
// 16-byte chunk j (0..7) of row r inside a SWIZZLE_128B box of 128-byte rows
__device__ __forceinline__ uint32_t sw128(int r, int j) { return r * 128 + ((j ^ (r & 7)) << 4); }

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmC1, const __grid_constant__ CUtensorMap tmC2,
                   const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmR1,
                   const __grid_constant__ CUtensorMap tmR2, const __grid_constant__ CUtensorMap tmE,
                   const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmO,
                   const __grid_constant__ CUtensorMap tmO2, Args a) {
  using namespace sm100;
  constexpr bool TWO = (MODE == DQ || MODE == DK);
  constexpr bool TRANS = (MODE == DV || MODE == DK);
  // A CTA pair (cluster of 2) owns two consecutive 128-row tiles of one (user, head) and runs
  // every MMA as tcgen05.mma.cta_group::2 with M = 256: each CTA keeps its own 128 rows of the
  // A operands and receives only HALF of every column tile — the score MMA's B operand is split
  // by columns (32 of the 64), the accumulate MMA's B operand by head dim (128 of the 256) — so
  // per-SM operand traffic is halved.  The leader CTA issues the MMAs; both CTAs run the softmax
  // and epilogue warps on their own rows.
  // smem (KB):     !TWO (FWD, DV)                        TWO (DQ, DK)
  //   [0,48)      C1 ring: 3 x 16 (32 cols x 256 dh)    R1 (S A operand, SS)   [0,64) -> E
  //   [48,96)     X ring:  3 x 16 (64 cols x 128 dh)    R2 dh 128..255 [64,96) (staging of
  //                                                     R2 dh 0..127 first) -> U 0,1
  //   [96,160)    R1 staging -> U                       C1 ring 3 x 16 [96,144)
  //   [160,224)   E (prefetched at start)               C2 ring 2 x 16 [144,176) -> U 2,3
  //                                                     X ring 2 x 16 [176,208)
  // TMEM:  !TWO: R1 [0,128) (TS A), acc [128,384), S [384,448), P [448,512)
  //         TWO: acc [0,256), S [256,320), dP [320,384), P [384,448), R2 dh 0..127 [448,512)
  constexpr int C1_BYTES = 32 * DH * 2;        // 16 KB: 4 boxes {64 dh, 32 cols}
  constexpr int X_BYTES = BC * (DH / 2) * 2;   // 16 KB: 2 boxes {64 dh, 64 cols}
  constexpr int NC1 = 3;
  constexpr int NC2 = 2;
  constexpr int NX = TWO ? 2 : 3;
  constexpr int OFF_C1 = TWO ? 96 * KB : 0;
  constexpr int OFF_C2 = 144 * KB;
  constexpr int OFF_X = TWO ? 176 * KB : 48 * KB;
  constexpr int OFF_R1 = 0, OFF_R2B = 64 * KB;
  constexpr int OFF_R1STAGE = 96 * KB;
  constexpr int OFF_E = TWO ? 0 : 160 * KB;
  constexpr uint32_t T_R1 = 0;
  constexpr uint32_t T_ACC = TWO ? 0 : 128;
  constexpr uint32_t T_S = TWO ? 256 : 384;
  constexpr uint32_t T_DP = 320;
  constexpr uint32_t T_P = TWO ? 384 : 448;
  constexpr uint32_t T_R2A = 448;

  const int u = blockIdx.z, h = blockIdx.y, r0 = blockIdx.x * BR;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const UserSpan us = load_user(a.jag, u);
  const int pr0 = (blockIdx.x & ~1) * BR;
  if (pr0 >= us.L) return;  // uniform over the cluster
  const int pair_end = min(us.L, pr0 + 2 * BR);
  const int kv_end = us.ns + us.nr;
  int c_begin = 0, c_end = 0;
  if (!TRANS) {
    c_end = (pair_end > us.ns) ? kv_end : us.ns;
  } else if (pr0 < kv_end) {
    c_begin = (pr0 < us.ns) ? 0 : us.ns;
    c_end = us.L;
  }
  const int ntiles = c_end > c_begin ? (c_end - c_begin + BC - 1) / BC : 0;
  const bool need_e = r0 + BR > us.ns;  // only tiles with non-static rows have diagonal terms

  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base, derived by indexing the shared array so the compiler keeps the shared
  // address space (LDS/STS rather than generic LD/ST for every staged access)
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  long long* sTs = reinterpret_cast<long long*>(smem + OFF_TS);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* c1_full = bars;           // [3] leader
  uint64_t* c1_empty = bars + 3;      // [3]
  uint64_t* x_full = bars + 6;        // [3] leader
  uint64_t* x_empty = bars + 9;       // [3]
  uint64_t* c2_full = bars + 12;      // [2] leader
  uint64_t* c2_empty = bars + 14;     // [2]
  uint64_t* s_full = bars + 16;
  uint64_t* s_free = bars + 17;       // leader, both CTAs' softmax threads
  uint64_t* t_full = bars + 18;       // [2] leader, both CTAs
  uint64_t* t_free = bars + 20;       // [2]
  uint64_t* r1_full = bars + 22;
  uint64_t* r1_done = bars + 23;      // leader, both CTAs (R1 in TMEM)
  uint64_t* r1_copied = bars + 24;    // own (staging area reusable)
  uint64_t* r2a_full = bars + 25;
  uint64_t* r2a_done = bars + 26;     // leader, both CTAs
  uint64_t* r2a_copied = bars + 27;   // own
  uint64_t* r2_full = bars + 28;      // leader: R2B of both CTAs (SS A operand)
  uint64_t* r1s_full = bars + 29;     // leader: R1 of both CTAs (TWO: SS A operand)
  uint64_t* e_full = bars + 30;
  uint64_t* u_full = bars + 31;
  uint64_t* o_full = bars + 32;
  uint64_t* sc_done = bars + 33;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 34);
  auto u_box = [&](int b) -> uint8_t* {  // smem of U box b (16 KB each)
    if (TWO) return b < 2 ? smem + 64 * KB + b * (RT_BYTES / 4) : smem + OFF_C2 + (b - 2) * (RT_BYTES / 4);
    return smem + OFF_R1STAGE + b * (RT_BYTES / 4);
  };
  auto arrive_leader = [&](uint64_t* bar) {  // one arrival per warp (whole warp calls)
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      if (leader) mbar_arrive(bar);
      else mbar_arrive_cluster(bar, 0);
    }
  };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) DBG(10 * 64 + 4);
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < 3; ++s) {
      mbar_init(&c1_full[s], 1); mbar_init(&c1_empty[s], 1);
      mbar_init(&x_full[s], 1); mbar_init(&x_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&c2_full[s], 1); mbar_init(&c2_empty[s], 1);
      mbar_init(&t_full[s], 2 * NSM); mbar_init(&t_free[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 2 * NSM);
    mbar_init(r1_full, 1);
    mbar_init(r1_done, 2 * NSM);
    mbar_init(r1_copied, 32 * NSM);
    mbar_init(r2a_full, 1);
    mbar_init(r2a_done, 2 * NSM);
    mbar_init(r2a_copied, 32 * NSM);
    mbar_init(r2_full, 1);
    mbar_init(r1s_full, 1);
    mbar_init(e_full, 1);
    mbar_init(u_full, 1);
    mbar_init(o_full, 1);
    mbar_init(sc_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated in both
  tc_fence_after();
  if (threadIdx.x == 0) DBG(10 * 64 + 10);
  const uint32_t tmem = *tmem_slot;
  const int hcol = h * DH;
  const int row0 = us.off + r0;  // global row of this CTA's first row

  if (warp == 0) {
    // ---------------------------------------------------------------- producer A: R1 / R2, C1, E (, U)
    if (lane == 0) {
      if (ntiles > 0) {
        if (!TWO) {
          mbar_expect_tx(r1_full, RT_BYTES);
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_2d(smem + OFF_R1STAGE + c * (RT_BYTES / 4), &tmR1, r1_full, hcol + c * 64, row0);
        } else {
          // R1 (SS A operand of S): both CTAs' bytes complete on the leader's r1s_full
          if (leader) mbar_expect_tx(r1s_full, 2 * RT_BYTES);
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_2d_2sm(smem + OFF_R1 + c * (RT_BYTES / 4), &tmR1, r1s_full, hcol + c * 64, row0);
          // R2 head-dim 0..127 -> staging (then TMEM via the softmax warps)
          mbar_expect_tx(r2a_full, RT_BYTES / 2);
#pragma unroll
          for (int c = 0; c < 2; ++c) tma_load_2d(smem + OFF_R2B + c * (RT_BYTES / 4), &tmR2, r2a_full, hcol + c * 64, row0);
        }
        for (int t = 0; t < ntiles; ++t) {
          if (TWO && t == NC1) {
            mbar_wait(r2a_copied, 0);
            if (leader) mbar_expect_tx(r2_full, RT_BYTES);
#pragma unroll
            for (int c = 2; c < 4; ++c) tma_load_2d_2sm(smem + OFF_R2B + (c - 2) * (RT_BYTES / 4), &tmR2, r2_full, hcol + c * 64, row0);
          }
          const int slot = t % NC1;
          mbar_wait(&c1_empty[slot], ((t / NC1) & 1) ^ 1);
          if (leader) mbar_expect_tx(&c1_full[slot], 2 * C1_BYTES);
          const int row = us.off + c_begin + t * BC + 32 * crank;  // this CTA's 32 columns
          uint8_t* dst = smem + OFF_C1 + slot * C1_BYTES;
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_2d_2sm(dst + c * (C1_BYTES / 4), &tmC1, &c1_full[slot], hcol + c * 64, row);
        }
        if (TWO && ntiles <= NC1) {
          mbar_wait(r2a_copied, 0);
          if (leader) mbar_expect_tx(r2_full, RT_BYTES);
#pragma unroll
          for (int c = 2; c < 4; ++c) tma_load_2d_2sm(smem + OFF_R2B + (c - 2) * (RT_BYTES / 4), &tmR2, r2_full, hcol + c * 64, row0);
        }
        if (TWO) mbar_wait(sc_done, 0);  // R1 / R2B / C2 regions are free from here on
      }
      if (!TWO && need_e) {  // private region, needed only by the epilogue: behind the C1 ring
        mbar_expect_tx(e_full, RT_BYTES);
#pragma unroll
        for (int c = 0; c < 4; ++c) tma_load_2d(smem + OFF_E + c * (RT_BYTES / 4), &tmE, e_full, hcol + c * 64, row0);
      }
      if (TWO) {
        if (need_e) {
          mbar_expect_tx(e_full, RT_BYTES);
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_2d(smem + OFF_E + c * (RT_BYTES / 4), &tmE, e_full, hcol + c * 64, row0);
        }
        if (a.has_u) {
          mbar_expect_tx(u_full, RT_BYTES);
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_2d(u_box(c), &tmU, u_full, hcol + c * 64, row0);
        }
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- producer B: X (, U) | C2
    if (lane == 0) {
      auto load_u = [&]() {  // !TWO: U replaces the R1 staging area
        if (!TWO && a.has_u) {
          if (ntiles > 0) mbar_wait(r1_copied, 0);
          mbar_expect_tx(u_full, RT_BYTES);
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_2d(u_box(c), &tmU, u_full, hcol + c * 64, row0);
        }
      };
      for (int t = 0; t < ntiles; ++t) {
        if (TWO) {
          const int slot = t % NC2;
          mbar_wait(&c2_empty[slot], ((t / NC2) & 1) ^ 1);
          if (leader) mbar_expect_tx(&c2_full[slot], 2 * C1_BYTES);
          const int row = us.off + c_begin + t * BC + 32 * crank;
          uint8_t* dst = smem + OFF_C2 + slot * C1_BYTES;
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_2d_2sm(dst + c * (C1_BYTES / 4), &tmC2, &c2_full[slot], hcol + c * 64, row);
        } else {
          const int slot = t % NX;
          mbar_wait(&x_empty[slot], ((t / NX) & 1) ^ 1);
          if (leader) mbar_expect_tx(&x_full[slot], 2 * X_BYTES);
          const int row = us.off + c_begin + t * BC;
          uint8_t* dst = smem + OFF_X + slot * X_BYTES;
#pragma unroll
          for (int c = 0; c < 2; ++c)  // this CTA's half of the head dim
            tma_load_2d_2sm(dst + c * (X_BYTES / 2), &tmX, &x_full[slot], hcol + (2 * crank + c) * 64, row);
        }
      }
      load_u();
    }
  } else if (warp == 2) {
    // ---------------------------------------------------------------- producer C (TWO): X
    if (TWO && lane == 0) {
      for (int t = 0; t < ntiles; ++t) {
        const int slot = t % NX;
        mbar_wait(&x_empty[slot], ((t / NX) & 1) ^ 1);
        if (leader) mbar_expect_tx(&x_full[slot], 2 * X_BYTES);
        const int row = us.off + c_begin + t * BC;
        uint8_t* dst = smem + OFF_X + slot * X_BYTES;
#pragma unroll
        for (int c = 0; c < 2; ++c)
          tma_load_2d_2sm(dst + c * (X_BYTES / 2), &tmX, &x_full[slot], hcol + (2 * crank + c) * 64, row);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA)
    // The whole warp walks the schedule so every operand is warp-uniform; one lane issues.
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const int nt = __shfl_sync(0xffffffffu, ntiles, 0);
    if (leader && nt == 0) {
      if (elect_one()) mbar_arrive(o_full);
      __syncwarp();
    }
    if (!leader && nt == 0) {
      if (lane == 0) mbar_arrive(o_full);
    }
    if (leader && nt > 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(2 * BR, BC, 0, 0);
      constexpr uint32_t idesc_acc = idesc_bf16_f32(2 * BR, DH, 0, 1);
      const uint32_t r1_base = smem_u32(smem + OFF_R1);
      const uint32_t r2b_base = smem_u32(smem + OFF_R2B);
      const uint32_t c1_base = smem_u32(smem + OFF_C1);
      const uint32_t c2_base = smem_u32(smem + OFF_C2);
      const uint32_t x_base = smem_u32(smem + OFF_X);
      if (TWO) {
        mbar_wait(r1s_full, 0);
        mbar_wait(r2a_done, 0);
        mbar_wait(r2_full, 0);
      } else {
        mbar_wait(r1_done, 0);  // R1 of both CTAs copied into TMEM
      }
      // acc += P_j X_j  (A = P from each CTA's TMEM, B = X: each CTA's half of the head dim)
      auto acc = [&](int j) {
        const int tb = j & 1;
        if (j < 64 && lane == 0) DBG(3 * 64 + j);
        mbar_wait(&t_full[tb], (j >> 1) & 1);
        if (j < 64 && lane == 0) DBG(4 * 64 + j);
        mbar_wait(&x_full[j % NX], (j / NX) & 1);
        const uint32_t x = x_base + (j % NX) * X_BYTES;
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BC / 16; ++k)
            mma_bf16_ts_2sm(tm + T_ACC, tm + T_P + tb * 32 + k * 8,
                            desc_sw128(x + k * 2048, X_BYTES / 2, 1024), idesc_acc, (j > 0 || k > 0));
          mma_commit_2sm_mc(&t_free[tb], 0x3);
          mma_commit_2sm_mc(&x_empty[j % NX], 0x3);
        }
        __syncwarp();
      };
      for (int t = 0; t < nt; ++t) {
        if (t < 64 && lane == 0) DBG(0 * 64 + t);
        mbar_wait(&c1_full[t % NC1], (t / NC1) & 1);
        if (TWO) mbar_wait(&c2_full[t % NC2], (t / NC2) & 1);
        if (t < 64 && lane == 0) DBG(1 * 64 + t);
        mbar_wait(s_free, (t & 1) ^ 1);  // single S (and dP) buffer, released on tcgen05.ld
        if (t < 64 && lane == 0) DBG(2 * 64 + t);
        tc_fence_after();
        const uint32_t c1 = c1_base + (t % NC1) * C1_BYTES;
        const uint32_t c2 = c2_base + (t % NC2) * C1_BYTES;
        if (elect_one()) {
          if (TWO) {
            // dP = R2 C2^T (head dim 0..127 of R2 from TMEM, 128..255 from smem), then S = R1 C1^T
#pragma unroll
            for (int k = 0; k < DH / 16; ++k) {
              const uint64_t bd = desc_sw128(c2 + (k >> 2) * (C1_BYTES / 4) + (k & 3) * 32, 16, 1024);
              if (k < 8)
                mma_bf16_ts_2sm(tm + T_DP, tm + T_R2A + k * 8, bd, idesc_s, k > 0);
              else
                mma_bf16_ss_2sm(tm + T_DP, desc_sw128(r2b_base + ((k >> 2) - 2) * (RT_BYTES / 4) + (k & 3) * 32, 16, 1024),
                                bd, idesc_s, 1);
            }
            mma_commit_2sm_mc(&c2_empty[t % NC2], 0x3);
#pragma unroll
            for (int k = 0; k < DH / 16; ++k)
              mma_bf16_ss_2sm(tm + T_S, desc_sw128(r1_base + (k >> 2) * (RT_BYTES / 4) + (k & 3) * 32, 16, 1024),
                              desc_sw128(c1 + (k >> 2) * (C1_BYTES / 4) + (k & 3) * 32, 16, 1024), idesc_s, k > 0);
          } else {
#pragma unroll
            for (int k = 0; k < DH / 16; ++k)
              mma_bf16_ts_2sm(tm + T_S, tm + T_R1 + k * 8,
                              desc_sw128(c1 + (k >> 2) * (C1_BYTES / 4) + (k & 3) * 32, 16, 1024), idesc_s, k > 0);
          }
          mma_commit_2sm_mc(s_full, 0x3);
          mma_commit_2sm_mc(&c1_empty[t % NC1], 0x3);
          if (t + 1 == nt) mma_commit_2sm_mc(sc_done, 0x3);
        }
        __syncwarp();
        if (t >= 1) acc(t - 1);
      }
      acc(nt - 1);
      if (elect_one()) mma_commit_2sm_mc(o_full, 0x3);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax + epilogue
    // quadrant q = warp % 4 owns TMEM lanes (this CTA's rows) q*32..q*32+31; half = which 32 of
    // the 64 tile columns (and which 128 of the 256 head-dim columns) the warp handles.
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int row = q * 32 + lane;
    const int my = r0 + row;                 // user-local index of this thread's row
    const int64_t g = (int64_t)row0 + row;   // global token index
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    if (ntiles > 0) {
      // row operand -> TMEM (bf16 pairs): !TWO: R1 (this warp's 128 head-dim columns),
      // TWO: R2 head-dim 0..127 (this warp's 64)
      mbar_wait(TWO ? r2a_full : r1_full, 0);
#pragma unroll 1
      for (int cc = 0; cc < (TWO ? 1 : 2); ++cc) {
        const uint8_t* box = TWO ? smem + OFF_R2B + half * (RT_BYTES / 4)
                                 : smem + OFF_R1STAGE + (half * 2 + cc) * (RT_BYTES / 4);
        uint32_t w[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 v = *reinterpret_cast<const uint4*>(box + sw128(row, j));
          w[4 * j] = v.x; w[4 * j + 1] = v.y; w[4 * j + 2] = v.z; w[4 * j + 3] = v.w;
        }
        tmem_st32(tmem + (TWO ? T_R2A + half * 32 : T_R1 + half * 64 + cc * 32) + lane_off, w);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(TWO ? r2a_copied : r1_copied);
      arrive_leader(TWO ? r2a_done : r1_done);
    }
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
        named_bar_sync(1, 32 * NSM);  // everyone is done reading the previous tile's times
        if (i < BC) tsb[i] = (c0 + i < us.L && a.jag.ts) ? a.jag.ts[us.off + c0 + i] : 0;
        named_bar_sync(1, 32 * NSM);
      }
      const bool dbgt = warp == 4 && lane == 0 && t < 64;
      if (dbgt) DBG(5 * 64 + t);
      mbar_wait(s_full, t & 1);
      if (dbgt) DBG(6 * 64 + t);
      tc_fence_after();
      uint32_t s[32];
      uint32_t dp[TWO ? 32 : 1];
      tmem_ld32(tmem + T_S + j_half + lane_off, s);
      if constexpr (TWO) {
        uint32_t (&d0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&dp[0]);
        tmem_ld32(tmem + T_DP + j_half + lane_off, d0);
      }
      tmem_ld_wait();
      tc_fence_before();
      arrive_leader(s_free);
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
      // P (T) values -> bf16 pairs -> TMEM P buffer (A operand of the accumulate MMA)
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
      tc_fence_after();
      tmem_st16(tmem + T_P + tb * 32 + half * 16 + lane_off, pk);
      tmem_st_wait();
      tc_fence_before();
      arrive_leader(&t_full[tb]);
      if (dbgt) DBG(9 * 64 + t);
    }

    // ---------------------------------------------------------------- epilogue
    // Warp (q, half) owns rows q*32..q*32+31 and head-dim columns half*128..half*128+127: four
    // 32-column chunks, the TMEM load of chunk cc+1 in flight while chunk cc is processed; each
    // finished 64-column box (cc = 1, 3) is stored by the warp right away (TMA for a full 32-row
    // chunk, row stores for the ragged last one), so the HBM writes overlap the rest.
    if (warp == 4 && lane == 0) DBG(10 * 64 + 0);
    mbar_wait(o_full, 0);
    if (warp == 4 && lane == 0) DBG(10 * 64 + 1);
    tc_fence_after();
    if (need_e) mbar_wait(e_full, 0);
    if (warp == 4 && lane == 0) DBG(10 * 64 + 5);
    if (a.has_u) mbar_wait(u_full, 0);
    if (warp == 4 && lane == 0) DBG(10 * 64 + 6);
    const bool row_ok = my < us.L;
    const float dg = (row_ok && my >= us.ns) ? a.diag[g * a.H + h] : 0.f;  // static rows: none
    uint8_t* sE = smem + OFF_E;
    if (warp == 4 && lane == 0) DBG(10 * 64 + 11);
    const int nrows = min(BR, us.L - r0);
    const bool full_chunk = q * 32 + 32 <= nrows;
    uint32_t r[2][32];
    if (ntiles > 0) tmem_ld32(tmem + T_ACC + half * 128 + lane_off, r[0]);
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const int acol = half * 128 + cc * 32;  // head-dim column of this chunk
      uint32_t (&rc)[32] = r[cc & 1];
      if (ntiles > 0) {
        tmem_ld_wait();
        if (cc < 3) tmem_ld32(tmem + T_ACC + acol + 32 + lane_off, r[(cc + 1) & 1]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) rc[i] = 0u;
      }
      const int bx = acol >> 6, j0 = (acol & 63) >> 3;
      uint8_t* ebox = sE + bx * (RT_BYTES / 4);
      uint8_t* ubox = u_box(bx);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t off = sw128(row, j0 + i);
        uint4 w = need_e ? *reinterpret_cast<const uint4*>(ebox + off) : make_uint4(0u, 0u, 0u, 0u);
        const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&w);
        float v[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(hh[k]);
          v[2 * k] = fmaf(us.nu, __uint_as_float(rc[8 * i + 2 * k]), dg * f.x);
          v[2 * k + 1] = fmaf(us.nu, __uint_as_float(rc[8 * i + 2 * k + 1]), dg * f.y);
        }
        if (MODE == FWD) {
          const uint4 uw = *reinterpret_cast<const uint4*>(ubox + off);
          const __nv_bfloat162* uh = reinterpret_cast<const __nv_bfloat162*>(&uw);
          float y[8];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 f = __bfloat1622float2(uh[k]);
            y[2 * k] = v[2 * k] * f.x;
            y[2 * k + 1] = v[2 * k + 1] * f.y;
          }
          *reinterpret_cast<uint4*>(ubox + off) =
              make_uint4(pack2(y[0], y[1]), pack2(y[2], y[3]), pack2(y[4], y[5]), pack2(y[6], y[7]));
        } else if (a.has_u) {
          const uint4 pw = *reinterpret_cast<const uint4*>(ubox + off);
          const __nv_bfloat162* ph = reinterpret_cast<const __nv_bfloat162*>(&pw);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 f = __bfloat1622float2(ph[k]);
            v[2 * k] *= a.pre_dsilu ? f.x : dsilu_fast(f.x);
            v[2 * k + 1] *= a.pre_dsilu ? f.y : dsilu_fast(f.y);
          }
        }
        *reinterpret_cast<uint4*>(ebox + off) =
            make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7]));
      }
      if (warp == 4 && lane == 0) DBG(10 * 64 + 12 + cc);
      if (cc & 1) {  // box bx of this warp's 32 rows is complete: store it
        if (full_chunk) {
          fence_proxy_async_smem();  // the bulk store reads what the generic proxy wrote
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmO, ebox + q * 32 * 128, hcol + bx * 64, row0 + q * 32);
            if (MODE == FWD) tma_store_2d(&tmO2, ubox + q * 32 * 128, hcol + bx * 64, row0 + q * 32);
            tma_store_commit();
          }
        } else {
          __syncwarp();
          // rows of the next user must not be touched: 4 rows x 8 16-byte pieces per pass
          for (int rr = q * 32 + (lane >> 3); rr < nrows; rr += 4) {
            const uint32_t off = sw128(rr, lane & 7);
            const int64_t go = (int64_t)(row0 + rr) * a.ld_out + hcol + bx * 64 + (lane & 7) * 8;
            *reinterpret_cast<uint4*>(a.out + go) = *reinterpret_cast<const uint4*>(ebox + off);
            if (MODE == FWD) *reinterpret_cast<uint4*>(a.out2 + go) = *reinterpret_cast<const uint4*>(ubox + off);
          }
        }
      }
    }
    if (warp == 4 && lane == 0) DBG(10 * 64 + 7);
    if (MODE != FWD && a.dbias != nullptr) {
      // bias gradient of this projection block: column sums over the tile's rows (fused, so
      // the layer never re-reads dp for it); [8 warps][256 columns] partials in free smem
      named_bar_sync(1, 32 * NSM);  // every warp's output rows are in smem
      if (warp == 4 && lane == 0) DBG(10 * 64 + 8);
      const int sw = warp - 4;
      const int bx = lane >> 3, jj = lane & 7;
      float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int rr = sw; rr < nrows; rr += NSM) {
        const uint4 w = *reinterpret_cast<const uint4*>(sE + bx * (RT_BYTES / 4) + sw128(rr, jj));
        const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(hh[k]);
          cs[2 * k] += f.x;
          cs[2 * k + 1] += f.y;
        }
      }
      float* red = reinterpret_cast<float*>(smem + OFF_C1);  // C1 ring is free by now
#pragma unroll
      for (int e = 0; e < 8; ++e) red[sw * DH + lane * 8 + e] = cs[e];
      named_bar_sync(1, 32 * NSM);
      const int col = threadIdx.x - 128;
      float sum = 0.f;
#pragma unroll
      for (int w2 = 0; w2 < NSM; ++w2) sum += red[w2 * DH + col];
      if (sum != 0.f) atomicAdd(a.dbias + hcol + col, sum);
    }
    if (lane == 0) tma_store_wait_read<0>();  // smem must outlive the bulk stores' reads
    if (warp == 4 && lane == 0) DBG(10 * 64 + 9);
  }
  if (warp == 4 && lane == 0) DBG(10 * 64 + 2);
  tc_fence_before();
  cluster_sync();  // no CTA leaves while its peer may still signal its barriers
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<512>(tmem);
  }
}

struct Maps {
  CUtensorMap c1, c2, x, r1, r2, e, u, o, o2;
};

template <int MODE>
static mtgr_status_t launch_mode(const AttnIO& io, const void* c1, int64_t ld_c1, const void* x,
                                 int64_t ld_x, const void* r1, int64_t ld_r1, const void* r2,
                                 int64_t ld_r2, const void* e, int64_t ld_e, const void* uu,
                                 int64_t ld_u, const Args& args, cudaStream_t st) {
  const int T = io.jag.total_tokens, d = io.d;
  Maps m;
  constexpr bool TWO = (MODE == DQ || MODE == DK);
  // column operands: each CTA of a pair loads half of every tile (32 columns of C1 / C2,
  // 128 head-dim columns of X); for DQ / DK, X is the C1 tensor and `x` is C2
  MTGR_TRY(make_tmap_bf16(&m.c1, c1, d, T, ld_c1, 64, BC / 2));
  if (TWO) {
    MTGR_TRY(make_tmap_bf16(&m.c2, x, d, T, ld_x, 64, BC / 2));
    MTGR_TRY(make_tmap_bf16(&m.x, c1, d, T, ld_c1, 64, BC));
  } else {
    MTGR_TRY(make_tmap_bf16(&m.x, x, d, T, ld_x, 64, BC));
    m.c2 = m.c1;
  }
  MTGR_TRY(make_tmap_bf16(&m.r1, r1, d, T, ld_r1, 64, BR));
  if (r2) MTGR_TRY(make_tmap_bf16(&m.r2, r2, d, T, ld_r2, 64, BR)); else m.r2 = m.r1;
  MTGR_TRY(make_tmap_bf16(&m.e, e, d, T, ld_e, 64, BR));
  if (uu) MTGR_TRY(make_tmap_bf16(&m.u, uu, d, T, ld_u, 64, BR)); else m.u = m.e;
  MTGR_TRY(make_tmap_bf16(&m.o, args.out, d, T, args.ld_out, 64, 32));
  if (args.out2) MTGR_TRY(make_tmap_bf16(&m.o2, args.out2, d, T, args.ld_out, 64, 32)); else m.o2 = m.o;
  Args a2 = args;
  a2.has_u = uu != nullptr;
  a2.pre_dsilu = io.pre_dsilu;
  dim3 grid(2 * ceil_div(io.jag.max_len, 2 * BR), io.H, io.jag.num_users);  // cluster pairs
  ProfScope ps(MODE == FWD ? PROF_ATTN_FWD : MODE == DV ? PROF_ATTN_DV : MODE == DK ? PROF_ATTN_DK : PROF_ATTN_DQ, st);
  cudaFuncSetAttribute(attn_tc_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  static const bool trace = getenv("MTGR_ATTN_TRACE") != nullptr;
  if (trace) {  // debug only: time-stamp one CTA's pipeline events
    cudaMalloc(&a2.dbg, 2 * 11 * 64 * sizeof(long long));
    cudaMemsetAsync(a2.dbg, 0, 2 * 11 * 64 * sizeof(long long), st);
  }
  attn_tc_kernel<MODE><<<grid, 384, SMEM_BYTES, st>>>(m.c1, m.c2, m.x, m.r1, m.r2, m.e, m.u, m.o, m.o2, a2);
  if (trace) {
    long long hb[2 * 11 * 64];
    cudaMemcpyAsync(hb, a2.dbg, sizeof(hb), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(a2.dbg);
    fprintf(stderr, "ATTN_TRACE mode=%d", MODE);
    for (int i = 0; i < 2 * 11 * 64; ++i) fprintf(stderr, " %lld", hb[i]);
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
  MTGR_CHECK(io.d % 8 == 0, MTGR_E_LAYOUT, "d_model must be a multiple of 8");
  Args a{};
  a.jag = io.jag; a.H = io.H; a.d = io.d;
  a.out = (__nv_bfloat16*)io.o; a.out2 = (__nv_bfloat16*)io.y; a.ld_out = io.d;
  a.diag = io.diag_a;
  // C1 = K, X = V, R1 = Q, E = V, U = U
  return launch_mode<FWD>(io, io.k, io.ld, io.v, io.ld, io.q, io.ld, nullptr, 0, io.v, io.ld, io.u,
                          io.ld, a, st);
}

mtgr_status_t attn_tc_bwd_launch(const AttnIO& io, cudaStream_t st) {
  using namespace tca;
  if (io.jag.num_users == 0 || io.jag.max_len == 0 || io.jag.total_tokens == 0) return MTGR_OK;
  typedef __nv_bfloat16 bf;
  const bf* pre = (const bf*)io.pre;
  const int64_t D = io.d;
  {  // dV = nu P^T dO (+ diag a_jj dO_j), * silu'(p_V): C1 = Q, X = dO, R1 = K, E = dO, U = p_V
    Args a{};
    a.jag = io.jag; a.H = io.H; a.d = io.d;
    a.out = (bf*)io.dv; a.ld_out = io.ld_out; a.diag = io.diag_a;
    a.dbias = io.dbias ? io.dbias + 2 * D : nullptr;
    MTGR_TRY(launch_mode<DV>(io, io.q, io.ld, io.dO, D, io.k, io.ld, nullptr, 0, io.dO, D,
                             pre ? pre + 2 * D : nullptr, io.ld_pre, a, st));
  }
  {  // dK = nu dS^T Q (+ diag ds_jj q_j), * silu'(p_K): C1 = Q, C2 = dO, R1 = K, R2 = V, E = Q
    Args a{};
    a.jag = io.jag; a.H = io.H; a.d = io.d;
    a.out = (bf*)io.dk; a.ld_out = io.ld_out; a.diag = io.diag_ds;
    a.dbias = io.dbias ? io.dbias + D : nullptr;
    MTGR_TRY(launch_mode<DK>(io, io.q, io.ld, io.dO, D, io.k, io.ld, io.v, io.ld, io.q, io.ld,
                             pre ? pre + D : nullptr, io.ld_pre, a, st));
  }
  {  // dQ = nu dS K (+ diag ds_ii k_i), * silu'(p_Q): C1 = K, C2 = V, R1 = Q, R2 = dO, E = K
    Args a{};
    a.jag = io.jag; a.H = io.H; a.d = io.d;
    a.out = (bf*)io.dq; a.ld_out = io.ld_out; a.diag = io.diag_ds;
    a.dbias = io.dbias;
    MTGR_TRY(launch_mode<DQ>(io, io.k, io.ld, io.v, io.ld, io.q, io.ld, io.dO, D, io.k, io.ld, pre,
                             io.ld_pre, a, st));
  }
  return MTGR_OK;
}

}  // namespace mtgr
