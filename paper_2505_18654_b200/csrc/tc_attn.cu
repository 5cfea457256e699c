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
// Per column tile:  S = R1 C1^T (tcgen05.mma, M=256 on the CTA pair, N=64, K=256; A = R1 from
// TMEM for FWD/DV, from smem for DQ/DK; B = C1 K-major) [and dP = R2 C2^T];  8 "softmax" warps
// tcgen05.ld S (and dP), apply the mask predicate in registers and SiLU / SiLU' (tanh.approx),
// and tcgen05.st the bf16 T tile into TMEM;  acc += T X (A = T from TMEM, B = X MN-major — the
// same TMA-loaded tile read with an MN-major descriptor, N=256, K=64).  (Measured on B200,
// tools/microbench/mma_rate.cu: SS N=64 is smem-bound at ~48 cycles per K=16 step, TS runs at
// the ideal for every N, so the score MMAs read A from TMEM where TMEM has room.)
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
// T [384,448) (two buffers of bf16 pairs).  (The exact layouts per mode are in the kernel;
// FWD/DV stage their row operand through warp 2 and move it into TMEM with tcgen05.cp from the
// MMA warp, right behind the previous item's MMAs.)
//
// The default backward is the stored-score path (attn_tc_bwd_launch): attn_sc_kernel computes
// S^T and dP^T per (key pair, head) and writes P^T and dS^T (bf16) into padded per-user key
// blocks; attn_mm_kernel then forms dV = nu P^T dO, dK = nu dS^T Q and dQ = nu dS K as jagged
// GEMMs (double-buffered TMEM accumulator, the same epilogue).  For long users (mean >= 2048
// tokens) the DK mode above writes the scores while forming dK (fewer item transitions); the
// recompute kernels (DV, DK, DQ modes) remain for batches whose score scratch would not fit.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"
#include "sm100.cuh"
#include "tc_attn.cuh"

namespace mtgr {
namespace tca {

template <int MODE, bool RAB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmC1, const __grid_constant__ CUtensorMap tmC2,
                   const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmR1,
                   const __grid_constant__ CUtensorMap tmR2, const __grid_constant__ CUtensorMap tmE,
                   const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmO,
                   Args a) {
  using namespace sm100;
  constexpr bool TWO = (MODE == DQ || MODE == DK);
  constexpr bool TRANS = (MODE == DV || MODE == DK);
  // Persistent CTA pairs (clusters of 2): pair c walks the work items c, c + #pairs, ...  Within
  // an item every MMA is a tcgen05.mma.cta_group::2 with M = 256: each CTA keeps its own 128 rows
  // of the A operands and receives only HALF of every column tile (the score MMA's B operand is
  // split by columns, 32 of 64; the accumulate MMA's B operand by head dim, 128 of 256), so the
  // per-SM operand traffic is halved.  The leader CTA issues the MMAs; both CTAs run softmax and
  // epilogue warps on their own rows.  Item boundaries overlap: the producers stream the next
  // item's operands as soon as ring slots free up, and the softmax warps move the next item's
  // row operand into TMEM before running the current item's epilogue, so the tensor pipe starts
  // the next item while the epilogue (which reads E/U rows straight from L2 and writes the
  // outputs from registers) drains the accumulator.
  // smem (KB):     !TWO (FWD, DV)                        TWO (DQ, DK)
  //   [0,48)      C1 ring: 3 x 16 (32 cols x 256 dh)    R1 (S A operand, SS) [0,64)
  //   [48,96)     X ring:  3 x 16 (64 cols x 128 dh)
  //   [96,160)    R1 staging                            R2 dh 128..255 [64,96) (staging of
  //   [160,224)   epilogue tile                           R2 dh 0..127 first)
  //                                                     C1 ring 3 x 16 [96,144) \ epilogue
  //                                                     C2 ring 2 x 16 [144,176) / tile [96,160)
  //                                                     X ring 2 x 16 [176,208)
  //   [224,224.5) key timestamps; barriers
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
  // epilogue tile (4 SW128 boxes of 128 rows x 64 head-dim columns): the SiLU' source (bwd)
  // arrives here by TMA and the outputs are formed in place and leave by TMA stores.  !TWO: a
  // dedicated region; TWO: the C1 ring plus the first C2 slot, free once the item's score MMAs
  // are done (the next item's column tiles are loaded after the epilogue released it, its row
  // operands before)
  constexpr int OFF_EPI = TWO ? 96 * KB : 160 * KB;
  constexpr uint32_t T_R1 = 0;
  constexpr uint32_t T_ACC = TWO ? 0 : 128;
  constexpr uint32_t T_S = TWO ? 256 : 384;
  constexpr uint32_t T_DP = 320;
  constexpr uint32_t T_P = TWO ? 384 : 448;
  constexpr uint32_t T_R2A = 448;

  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;

  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base, derived by indexing the shared array so the compiler keeps the shared
  // address space (LDS/STS rather than generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  long long* sTs = reinterpret_cast<long long*>(smem + off_ts(TWO));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + off_bar(TWO));
  float* sRab = reinterpret_cast<float*>(smem + off_rab(TWO));    // RAB: rab_w[h][0, nb)
  float* sRacc = reinterpret_cast<float*>(smem + off_racc(TWO));  // RAB, DQ: drab bins of the item
  uint64_t* c1_full = bars;           // [3] leader
  uint64_t* c1_empty = bars + 3;      // [3]
  uint64_t* x_full = bars + 6;        // [3] leader
  uint64_t* x_empty = bars + 9;       // [3]
  uint64_t* c2_full = bars + 12;      // [2] leader
  uint64_t* c2_empty = bars + 14;     // [2]
  // !TWO: the score tile is double-buffered (S[b] = T_S + 64 b) and the P tile written in place,
  // so s_full is [2] (bars 16 and 44) and neither s_free nor t_free is used; TWO: single S / dP
  uint64_t* s_full = bars + 16;
  uint64_t* s_free = bars + 17;       // leader, both CTAs' softmax warps (TWO)
  uint64_t* s_full1 = bars + 46;      // !TWO: score tile 1 (after q_item [43, 45))
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
  uint64_t* o_full = bars + 30;
  uint64_t* sc_done = bars + 31;
  uint64_t* q_full = bars + 32;       // [4] work queue: item index published (own)
  uint64_t* q_empty = bars + 36;      // [4] leader: every consumer of both CTAs has read it
  uint64_t* eu_full = bars + 40;      // epilogue SiLU' source tile landed (own)
  uint64_t* epi_free = bars + 41;     // epilogue tile free again (own; 8 softmax warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 42);
  int* q_item = reinterpret_cast<int*>(bars + 43);  // [4]
  auto arrive_leader = [&](uint64_t* bar) {  // one arrival per warp (whole warp calls)
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      if (leader) mbar_arrive(bar);
      else mbar_arrive_cluster(bar, 0);
    }
  };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
    mbar_init(s_full1, 1);
    mbar_init(s_free, 2 * NSM);
    mbar_init(r1_full, 1);
    mbar_init(r1_done, 2 * NSM);
    mbar_init(r1_copied, (!TWO && a.row_cp) ? 1 : NSM);  // tcgen05.cp: one commit arrival
    mbar_init(r2a_full, 1);
    mbar_init(r2a_done, 2 * NSM);
    mbar_init(r2a_copied, NSM);
    mbar_init(r2_full, 1);
    mbar_init(r1s_full, 1);
    mbar_init(o_full, 1);
    mbar_init(sc_done, 1);
    mbar_init(eu_full, 1);
    mbar_init(epi_free, NSM);
    for (int s = 0; s < 4; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 2 * (NSM + 3));  // per CTA: B, C / epilogue loader, 8 softmax, MMA | A
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated in both
  tc_fence_after();
  if (threadIdx.x == 0) DBGV(10, 0, clock64());
  const uint32_t tmem = *tmem_slot;

  // ---- dynamic work queue: the leader's producer thread claims items (global atomic counter,
  // empty pairs skipped) and publishes them, in order, to both CTAs; every role of both CTAs
  // reads entry n, n+1, ... and releases it on the leader.  Consumers per CTA: producer B,
  // (TWO) producer C, 8 softmax warps, and the MMA warp (leader) / producer A (peer).
  auto q_read = [&](int n) -> int {
    mbar_wait_cluster(&q_full[n & 3], (n >> 2) & 1);
    return *reinterpret_cast<volatile int*>(&q_item[n & 3]);
  };
  auto q_release = [&](int n) {  // one thread per consuming warp
    if (leader) mbar_arrive(&q_empty[n & 3]);
    else mbar_arrive_cluster(&q_empty[n & 3], 0);
  };
  auto q_push = [&](int n) -> int {  // leader producer thread
    if (n >= 4) mbar_wait(&q_empty[n & 3], ((n >> 2) & 1) ^ 1);
    int k;
    for (;;) {
      k = atomicAdd(a.ctr, 1);
      if (k >= a.nitems) { k = -1; break; }
      const int rest = k / a.H;
      const int u = rest / a.pmax, p = rest % a.pmax;
      if (p * 2 * BR < a.jag.offsets[u + 1] - a.jag.offsets[u]) break;  // non-empty pair
    }
    q_item[n & 3] = k;
    st_cluster_u32(reinterpret_cast<uint32_t*>(&q_item[n & 3]), 1, (uint32_t)k);
    mbar_arrive(&q_full[n & 3]);
    mbar_arrive_cluster_release(&q_full[n & 3], 1);
    return k;
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- producer A: R1 / R2, C1
    if (lane == 0) {
      int gt = 0, mi = 0, idx = 0;
      // the leader publishes one item ahead, so every role (the row-operand loader, the softmax
      // warps' end-of-loop peek) learns the next item before this item's column tiles are issued
      int k_next = leader ? q_push(0) : 0;
      for (int n = 0;; ++n) {
        int k;
        if (leader) {
          k = k_next;
          if (k >= 0) k_next = q_push(n + 1);
        } else {
          k = q_read(n);
          q_release(n);
        }
        if (k < 0) break;
        Item it;
        decode_item<TRANS>(a, k, crank, it);
        const int row0 = it.us.off + it.r0;
        auto load_u = [&]() {  // SiLU' source tile of the epilogue (bwd modes)
          if (a.uu != nullptr) {
            mbar_expect_tx(eu_full, RT_BYTES);
#pragma unroll
            for (int c = 0; c < 4; ++c) tma_load_2d(smem + OFF_EPI + c * (RT_BYTES / 4), &tmU, eu_full, it.hcol + c * 64, row0);
          }
        };
        auto wait_epi = [&]() { if (idx > 0) mbar_wait(epi_free, (idx - 1) & 1); };
        if (it.ntiles > 0) {
          // (!TWO: the row operand is staged by warp 2, ahead of this item's column tiles)
          // TWO: the row operands are loaded as soon as the previous item's score MMAs are done
          // (they overlap its epilogue); the column ring doubles as that epilogue's tile, so the
          // column tiles wait for the epilogue to release it
          if (TWO) {
            if (mi > 0) mbar_wait(sc_done, (mi - 1) & 1);
            if (leader) mbar_expect_tx(r1s_full, 2 * RT_BYTES);
#pragma unroll
            for (int c = 0; c < 4; ++c) tma_load_2d_2sm(smem + OFF_R1 + c * (RT_BYTES / 4), &tmR1, r1s_full, it.hcol + c * 64, row0);
            mbar_expect_tx(r2a_full, RT_BYTES / 2);  // R2 head-dim 0..127 -> staging (then TMEM)
#pragma unroll
            for (int c = 0; c < 2; ++c) tma_load_2d(smem + OFF_R2B + c * (RT_BYTES / 4), &tmR2, r2a_full, it.hcol + c * 64, row0);
            DBG(7, idx);
            wait_epi();
          }
          auto head = [&]() {  // TWO: R2 head-dim 128..255 once the staging was copied out
            mbar_wait(r2a_copied, mi & 1);
            if (leader) mbar_expect_tx(r2_full, RT_BYTES);
#pragma unroll
            for (int c = 2; c < 4; ++c) tma_load_2d_2sm(smem + OFF_R2B + (c - 2) * (RT_BYTES / 4), &tmR2, r2_full, it.hcol + c * 64, row0);
          };
          const int npre = min(NC1, it.ntiles);
          for (int t = 0; t < it.ntiles; ++t, ++gt) {
            if (TWO && t == npre) head();
            const int slot = gt % NC1;
            mbar_wait(&c1_empty[slot], ((gt / NC1) & 1) ^ 1);
            if (leader) mbar_expect_tx(&c1_full[slot], 2 * C1_BYTES);
            const int row = it.us.off + it.c_begin + t * BC + 32 * crank;  // this CTA's 32 columns
            uint8_t* dst = smem + OFF_C1 + slot * C1_BYTES;
#pragma unroll
            for (int c = 0; c < 4; ++c) tma_load_2d_2sm(dst + c * (C1_BYTES / 4), &tmC1, &c1_full[slot], it.hcol + c * 64, row);
          }
          if (TWO && npre == it.ntiles) head();
          DBG(8, idx);
          if (TWO) {  // the column ring becomes the epilogue tile once the score MMAs are done
            mbar_wait(sc_done, mi & 1);
            load_u();
          }
          ++mi;
        } else if (TWO) {
          wait_epi();
          load_u();
        }
        ++idx;
      }
    }
  } else if (!TWO && warp == 2) {
    // ---------------------------------------------------------------- !TWO: row operand + epilogue
    // tile loader.  The next item's row operand is staged as soon as the softmax warps copied the
    // previous one into TMEM, independently of the column-tile producer (which reaches the next
    // item only after issuing this item's last tiles), so it has landed when the softmax warps
    // move it into TMEM at the end of this item's tile loop
    if (lane == 0) {
      int idx = 0, mi = 0;
      for (int n = 0;; ++n) {
        const int k = q_read(n);
        q_release(n);
        if (k < 0) break;
        Item it;
        decode_item<TRANS>(a, k, crank, it);
        if (it.ntiles > 0) {
          if (mi > 0) mbar_wait(r1_copied, (mi - 1) & 1);  // staging free again
          if (a.row_cp) {  // both CTAs' rows on the leader's barrier: the MMA warp copies them
            if (leader) mbar_expect_tx(r1_full, 2 * RT_BYTES);
#pragma unroll
            for (int c = 0; c < 4; ++c)
              tma_load_2d_2sm(smem + OFF_R1STAGE + c * (RT_BYTES / 4), &tmR1, r1_full, it.hcol + c * 64,
                              it.us.off + it.r0);
          } else {
            mbar_expect_tx(r1_full, RT_BYTES);
#pragma unroll
            for (int c = 0; c < 4; ++c)
              tma_load_2d(smem + OFF_R1STAGE + c * (RT_BYTES / 4), &tmR1, r1_full, it.hcol + c * 64, it.us.off + it.r0);
          }
          ++mi;
        }
        if (a.uu != nullptr) {
          if (idx > 0) mbar_wait(epi_free, (idx - 1) & 1);
          mbar_expect_tx(eu_full, RT_BYTES);
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_2d(smem + OFF_EPI + c * (RT_BYTES / 4), &tmU, eu_full, it.hcol + c * 64, it.us.off + it.r0);
        }
        ++idx;
      }
    }
  } else if (warp == 3 || (TWO && warp == 2)) {
    // ---------------------------------------------------------------- producers B (X | C2), C (TWO: X)
    if (lane == 0) {
      const bool load_x = !TWO || warp == 2;
      int gt = 0, idx = 0;
      for (int n = 0;; ++n) {
        const int k = q_read(n);
        q_release(n);
        if (k < 0) break;
        Item it;
        decode_item<TRANS>(a, k, crank, it);
        // TWO: the C2 ring's first slot is part of the previous item's epilogue tile.  Wait for
        // every item, tiles or not: parity waits must not skip a phase (a skipped one lets the
        // wait for phase i pass while phase i-1 is still pending)
        if (TWO && !load_x && idx > 0) mbar_wait(epi_free, (idx - 1) & 1);
        ++idx;
        for (int t = 0; t < it.ntiles; ++t, ++gt) {
          if (!load_x) {
            const int slot = gt % NC2;
            mbar_wait(&c2_empty[slot], ((gt / NC2) & 1) ^ 1);
            if (leader) mbar_expect_tx(&c2_full[slot], 2 * C1_BYTES);
            const int row = it.us.off + it.c_begin + t * BC + 32 * crank;
            uint8_t* dst = smem + OFF_C2 + slot * C1_BYTES;
#pragma unroll
            for (int c = 0; c < 4; ++c) tma_load_2d_2sm(dst + c * (C1_BYTES / 4), &tmC2, &c2_full[slot], it.hcol + c * 64, row);
          } else {
            const int slot = gt % NX;
            mbar_wait(&x_empty[slot], ((gt / NX) & 1) ^ 1);
            if (leader) mbar_expect_tx(&x_full[slot], 2 * X_BYTES);
            const int row = it.us.off + it.c_begin + t * BC;
            uint8_t* dst = smem + OFF_X + slot * X_BYTES;
#pragma unroll
            for (int c = 0; c < 2; ++c)  // this CTA's half of the head dim
              tma_load_2d_2sm(dst + c * (X_BYTES / 2), &tmX, &x_full[slot], it.hcol + (2 * crank + c) * 64, row);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA)
    // The whole warp walks the schedule so every operand is warp-uniform; one lane issues.
    if (leader) {
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      constexpr uint32_t idesc_s = idesc_bf16_f32(2 * BR, BC, 0, 0);
      constexpr uint32_t idesc_acc = idesc_bf16_f32(2 * BR, DH, 0, 1);
      const uint32_t r1_base = smem_u32(smem + OFF_R1);
      const uint32_t r2b_base = smem_u32(smem + OFF_R2B);
      const uint32_t c1_base = smem_u32(smem + OFF_C1);
      const uint32_t c2_base = smem_u32(smem + OFF_C2);
      const uint32_t x_base = smem_u32(smem + OFF_X);
      int gt = 0, mi = 0, idx = 0;
      int cp_done = 0;  // !TWO with row_cp: items whose row operand has been copied into TMEM
      const uint32_t r1s_base = smem_u32(smem + OFF_R1STAGE);
      // R1 staging (both CTAs) -> TMEM by tcgen05.cp, ordered after the MMAs issued so far; the
      // commit frees the staging for the loader
      auto copy_r1 = [&]() {
        mbar_wait(r1_full, cp_done & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk)
            tmem_cp_128x256b_2sm(tm + T_R1 + kk * 8,
                                 desc_sw128(r1s_base + (kk >> 2) * (RT_BYTES / 4) + (kk & 3) * 32, 16, 1024));
          mma_commit_2sm_mc(r1_copied, 0x3);
        }
        __syncwarp();
        ++cp_done;
      };
      for (int n = 0;; ++n) {
        const int k = q_read(n);
        if (lane == 0) q_release(n);
        if (k < 0) break;
        Item it;
        decode_item<TRANS>(a, k, crank, it);
        const int nt = it.ntiles;
        if (lane == 0) DBGV(9, idx, nt);
        if (nt == 0) { ++idx; continue; }
        if (TWO) {
          mbar_wait(r1s_full, mi & 1);
          mbar_wait(r2a_done, mi & 1);
          mbar_wait(r2_full, mi & 1);
        } else if (a.row_cp) {
          if (cp_done == mi) copy_r1();  // not prefetched at the end of the previous item
        } else {
          mbar_wait(r1_done, mi & 1);  // R1 of both CTAs copied into TMEM
        }
        // acc += P_j X_j  (A = P from each CTA's TMEM, B = X: each CTA's half of the head dim)
        auto acc = [&](int j, int g) {
          const int tb = g & 1;
          mbar_wait(&t_full[tb], (g >> 1) & 1);
          mbar_wait(&x_full[g % NX], (g / NX) & 1);
          const uint32_t x = x_base + (g % NX) * X_BYTES;
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BC / 16; ++kk)
              mma_bf16_ts_2sm(tm + T_ACC, TWO ? tm + T_P + tb * 32 + kk * 8
                                                : tm + T_S + 64 * tb + (kk >> 1) * 32 + (kk & 1) * 8,
                              desc_sw128(x + kk * 2048, X_BYTES / 2, 1024), idesc_acc, (j > 0 || kk > 0));
            if (TWO) mma_commit_2sm_mc(&t_free[tb], 0x3);
            mma_commit_2sm_mc(&x_empty[g % NX], 0x3);
          }
          __syncwarp();
        };
        for (int t = 0; t < nt; ++t) {
          const int g = gt + t;
          mbar_wait(&c1_full[g % NC1], (g / NC1) & 1);
          if (TWO) mbar_wait(&c2_full[g % NC2], (g / NC2) & 1);
          // TWO: single S (and dP) buffer, released on tcgen05.ld; !TWO: score tile (g & 1) was
          // last read by the accumulate MMA of tile g - 2, issued (in order) before this one
          if (TWO) mbar_wait(s_free, (g & 1) ^ 1);
          tc_fence_after();
          const uint32_t c1 = c1_base + (g % NC1) * C1_BYTES;
          const uint32_t c2 = c2_base + (g % NC2) * C1_BYTES;
          if (elect_one()) {
            if (TWO) {
              // dP = R2 C2^T (head dim 0..127 of R2 from TMEM, 128..255 from smem), then S = R1 C1^T
#pragma unroll
              for (int kk = 0; kk < DH / 16; ++kk) {
                const uint64_t bd = desc_sw128(c2 + (kk >> 2) * (C1_BYTES / 4) + (kk & 3) * 32, 16, 1024);
                if (kk < 8)
                  mma_bf16_ts_2sm(tm + T_DP, tm + T_R2A + kk * 8, bd, idesc_s, kk > 0);
                else
                  mma_bf16_ss_2sm(tm + T_DP, desc_sw128(r2b_base + ((kk >> 2) - 2) * (RT_BYTES / 4) + (kk & 3) * 32, 16, 1024),
                                  bd, idesc_s, 1);
              }
              mma_commit_2sm_mc(&c2_empty[g % NC2], 0x3);
#pragma unroll
              for (int kk = 0; kk < DH / 16; ++kk)
                mma_bf16_ss_2sm(tm + T_S, desc_sw128(r1_base + (kk >> 2) * (RT_BYTES / 4) + (kk & 3) * 32, 16, 1024),
                                desc_sw128(c1 + (kk >> 2) * (C1_BYTES / 4) + (kk & 3) * 32, 16, 1024), idesc_s, kk > 0);
            } else {
#pragma unroll
              for (int kk = 0; kk < DH / 16; ++kk)
                mma_bf16_ts_2sm(tm + T_S + 64 * (g & 1), tm + T_R1 + kk * 8,
                                desc_sw128(c1 + (kk >> 2) * (C1_BYTES / 4) + (kk & 3) * 32, 16, 1024), idesc_s, kk > 0);
            }
            mma_commit_2sm_mc((TWO || (g & 1) == 0) ? s_full : s_full1, 0x3);
            mma_commit_2sm_mc(&c1_empty[g % NC1], 0x3);
            if (TWO && t + 1 == nt) mma_commit_2sm_mc(sc_done, 0x3);
          }
          __syncwarp();
          if (t == 0 && lane == 0) DBG(5, idx);
          if (t >= 1) acc(t - 1, g - 1);
        }
        acc(nt - 1, gt + nt - 1);
        if (elect_one()) mma_commit_2sm_mc(o_full, 0x3);
        __syncwarp();
        if (!TWO && a.row_cp) {  // the next item's row operand, right behind this item's MMAs
          const int k2 = q_read(n + 1);  // peek (released when it is processed)
          Item nx;
          if (k2 >= 0 && decode_item<TRANS>(a, k2, crank, nx) && nx.ntiles > 0) copy_r1();
        }
        if (lane == 0) DBG(6, idx);
        gt += nt;
        ++mi;
        ++idx;
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax + epilogue
    // quadrant q = warp % 4 owns TMEM lanes (this CTA's rows) q*32..q*32+31; half = which 32 of
    // the 64 tile columns (and which 128 of the 256 head-dim columns) the warp handles.
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int j_half = half * 32;
    const bool dbgw = warp == 4 && lane == 0;
    const bool store_scores = MODE == DK && a.st_ds != nullptr;  // uniform
    constexpr int PPN = 16;  // P^T words (stored-score DK; dead in the other modes)
    int gt = 0;      // global tile counter
    int mi = 0;      // items with tiles, in order
    int copied = 0;  // R1 (R2A) copies issued so far (the row operand of mma-item `copied - 1`)
    // row operand -> TMEM (bf16 pairs): !TWO: R1 (this warp's 128 head-dim columns),
    // TWO: R2 head-dim 0..127 (this warp's 64); phase = index of the mma-item
    auto copy_rows = [&]() {
      const int ph = copied & 1;
      mbar_wait(TWO ? r2a_full : r1_full, ph);
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
      __syncwarp();
      if (lane == 0) mbar_arrive(TWO ? r2a_copied : r1_copied);  // one arrival per warp
      arrive_leader(TWO ? r2a_done : r1_done);
      ++copied;
    };
    int idx = 0;
    // RAB, DQ recompute backward: drab bins.  Each thread sums its dS run by run (a run = equal
    // buckets along its row; the time gaps change bucket rarely), a finished run goes into the
    // CTA's shared bins, and the bins leave (x nu) to drab at the end of every item
    const bool acc_drab = RAB && MODE == DQ && a.drab != nullptr;  // uniform
    int rb = 0;
    float racc = 0.f;
    if (acc_drab && threadIdx.x - 128 < 64) sRacc[threadIdx.x - 128] = 0.f;  // ordered by tile 0's barriers
    for (int n = 0;; ++n) {
      const int k = q_read(n);
      __syncwarp();
      if (lane == 0) q_release(n);
      if (k < 0) break;
      Item it;
      decode_item<TRANS>(a, k, crank, it);
      const UserSpan& us = it.us;
      const int my = it.r0 + row;                    // user-local index of this thread's row
      const int64_t g = (int64_t)us.off + my;        // global token index
      if (dbgw) DBG(0, idx);
      // the candidate-row diagonal scalar of the epilogue, loaded now: its latency hides behind the tiles
      const float dg_pre = (my < us.L && my >= it.kv_end) ? a.diag[g * a.H + it.h] : 0.f;
      if (it.ntiles > 0) {
        if (copied == mi && !(!TWO && a.row_cp)) copy_rows();  // not prefetched by the previous item
        const long long my_ts = (my < us.L && a.jag.ts) ? a.jag.ts[g] : 0;
        // stored-score row of this key (DK): [h][koff[u] + my][query]
        const int64_t st_row = store_scores ? ((int64_t)it.h * a.st_rows + a.koff[it.u] + my) * a.st_pitch : 0;
        const bool need_ts_rows = TRANS && !a.causal && !a.full && (it.r0 + BR > us.ns) && (it.r0 < it.kv_end);
#pragma unroll 1
        for (int t = 0; t < it.ntiles; ++t, ++gt) {
          const int c0 = it.c_begin + t * BC;
          const bool need_ts = RAB || (TRANS ? need_ts_rows : (!a.causal && !a.full && c0 + BC > us.ns && c0 < it.kv_end));
          long long* tsb = sTs;
          if (need_ts) {  // uniform over the 8 softmax warps
            const int i = threadIdx.x - 128;
            named_bar_sync(1, 32 * NSM);  // everyone is done reading the previous tile's times
            if (i < BC) tsb[i] = (c0 + i < us.L && a.jag.ts) ? a.jag.ts[us.off + c0 + i] : 0;
            if (RAB && t == 0 && i >= BC && i < BC + a.nb) sRab[i - BC] = a.rab_w[it.h * a.nb + i - BC];
            named_bar_sync(1, 32 * NSM);
          }
          const uint32_t t_s = TWO ? T_S : T_S + 64 * (gt & 1);
          if (TWO) mbar_wait(s_full, gt & 1);
          else mbar_wait((gt & 1) ? s_full1 : s_full, (gt >> 1) & 1);
          tc_fence_after();
          uint32_t s[32];
          uint32_t dp[TWO ? 32 : 1];
          tmem_ld32(tmem + t_s + j_half + lane_off, s);
          if constexpr (TWO) {
            uint32_t (&d0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&dp[0]);
            tmem_ld32(tmem + T_DP + j_half + lane_off, d0);
          }
          tmem_ld_wait();
          if (TWO) {
            tc_fence_before();
            arrive_leader(s_free);
          }
          if constexpr (RAB) add_rab<32>(s, my_ts, tsb + j_half, sRab, a.nb - 1);  // s_ij + rab (R#4)
          // visibility of this warp's 32 columns for this row (dynamic mask, R#8-R#12)
          const int cb = c0 + j_half;
          uint32_t vis;
          if (a.causal) {
            // causal (uniform branch): row i reads keys j <= i (rows are readers for !TRANS,
            // keys for TRANS, whose columns are the queries i >= j, i < L)
            const int lo = TRANS ? min(max(my - cb, 0), 32) : 0;
            const int hi = TRANS ? min(max(us.L - cb, 0), 32) : min(max(my - cb + 1, 0), 32);
            const uint32_t below_hi = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
            const uint32_t below_lo = lo >= 32 ? 0xffffffffu : ((1u << lo) - 1u);
            vis = (my < us.L) ? (below_hi & ~below_lo) : 0u;
          } else if (a.full) {
            // full mask (Table 4 "w/o dynamic mask" read as full attention): static
            // and real-time keys [0, kv_end) visible to every query; candidates: diagonal only
            if (!TRANS) {
              const int n_kv = min(max(it.kv_end - cb, 0), 32);
              vis = n_kv >= 32 ? 0xffffffffu : ((1u << n_kv) - 1u);
            } else {
              const int nvalid = us.L - cb;
              vis = (my >= it.kv_end || nvalid <= 0) ? 0u : (nvalid >= 32 ? 0xffffffffu : ((1u << nvalid) - 1u));
            }
          } else if (!TRANS) {
            // static columns [0, ns) are visible to every row; real-time columns [ns, kv_end)
            // only to non-static rows with an earlier timestamp (diagonal: epilogue)
            const int n_stat = min(max(us.ns - cb, 0), 32);
            vis = n_stat >= 32 ? 0xffffffffu : ((1u << n_stat) - 1u);
            if (my >= us.ns) {
              const int n_kv = min(max(it.kv_end - cb, 0), 32);
              for (int jj = n_stat; jj < n_kv; ++jj) vis |= (uint32_t)(tsb[j_half + jj] < my_ts) << jj;
              const int jd = my - cb;  // the row's own column (real-time rows: R#9)
              if (my < it.kv_end && jd >= 0 && jd < 32) vis |= 1u << jd;
            }
          } else {
            if (my < us.ns) {
              const int nvalid = us.L - cb;
              vis = nvalid >= 32 ? 0xffffffffu : (nvalid <= 0 ? 0u : ((1u << nvalid) - 1u));
            } else if (my < it.kv_end) {
              vis = 0;
              const int lo = min(max(us.ns - cb, 0), 32), hi = min(max(us.L - cb, 0), 32);
              for (int jj = lo; jj < hi; ++jj) vis |= (uint32_t)(my_ts < tsb[j_half + jj]) << jj;
              const int jd = my - cb;  // the key's own query column (real-time rows: R#9)
              if (jd >= 0 && jd < 32) vis |= 1u << jd;
            } else {
              vis = 0;
            }
          }
          // P (T) values -> bf16 pairs -> TMEM P buffer (A operand of the accumulate MMA)
          uint32_t pk[16];
          uint32_t pp[PPN];
          if (store_scores) {
            // DK with stored scores: dS^T for the MMA and the store, P^T for the store only
            // (silu and silu' share sigma(s) = 0.5 + 0.5 tanh(s/2))
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              const float s0 = __uint_as_float(s[e]), s1 = __uint_as_float(s[e + 1]);
              const float g0 = fmaf(0.5f, sm100::tanh_approx(0.5f * s0), 0.5f);
              const float g1 = fmaf(0.5f, sm100::tanh_approx(0.5f * s1), 0.5f);
              float p0 = s0 * g0, p1 = s1 * g1;
              float v0 = __uint_as_float(dp[e]) * fmaf(p0, 1.0f - g0, g0);
              float v1 = __uint_as_float(dp[e + 1]) * fmaf(p1, 1.0f - g1, g1);
              {  // selects, no branch (masked entries are exact zeros, R#2)
                const bool m0 = (vis >> e) & 1u, m1 = (vis >> (e + 1)) & 1u;
                v0 = m0 ? v0 : 0.f; p0 = m0 ? p0 : 0.f;
                v1 = m1 ? v1 : 0.f; p1 = m1 ? p1 : 0.f;
              }
              pk[e >> 1] = pack2(v0, v1);
              pp[(e >> 1) % PPN] = pack2(p0, p1);
            }
          } else {
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
            v0 = ((vis >> e) & 1u) ? v0 : 0.f;  // selects, no branch (masked: exact zeros, R#2)
            v1 = ((vis >> (e + 1)) & 1u) ? v1 : 0.f;
            pk[e >> 1] = pack2(v0, v1);
            if (acc_drab && my < us.L) {  // dS (before nu) of the two entries into this row's bucket runs
              // (rows past L are the pair's padding: their values are discarded, never summed)
#pragma unroll
              for (int h2 = 0; h2 < 2; ++h2) {
                const int bk = rab_bkt(my_ts - tsb[j_half + e + h2], a.nb - 1);
                if (bk != rb) {
                  if (racc != 0.f) atomicAdd(&sRacc[rb], racc);
                  rb = bk;
                  racc = 0.f;
                }
                racc += h2 ? v1 : v0;
              }
            }
          }
          }
          const int tb = gt & 1;
          if (TWO) {
            mbar_wait(&t_free[tb], ((gt >> 1) & 1) ^ 1);
            tc_fence_after();
          }
          // !TWO: in place, into this warp's own 32 columns of the score tile it just read
          tmem_st16(tmem + (TWO ? T_P + tb * 32 + half * 16 : t_s + j_half) + lane_off, pk);
          tmem_st_wait();
          tc_fence_before();
          arrive_leader(&t_full[tb]);
          if (store_scores) {
            // this row's 32 query columns are 64 contiguous bytes per matrix.  Lane pairs swap
            // halves so that each 256-bit store instruction writes 16 whole 64-byte row pieces
            // (lanes 2k, 2k+1: row 2k, then row 2k+1) instead of 32 scattered 16-byte pieces
            const int b = lane & 1;
            auto put = [&](__nv_bfloat16* base, const uint32_t* w) {
              U8 own, oth;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                own.v[i] = b ? w[8 + i] : w[i];  // selects, not dynamic register indexing
                oth.v[i] = __shfl_xor_sync(0xffffffffu, b ? w[i] : w[8 + i], 1);
              }
              __nv_bfloat16* p0 = base + st_row + cb + 16 * b;
              stg256(p0 - (int64_t)b * a.st_pitch, b ? oth : own);        // row (lane & ~1)
              stg256(p0 + (int64_t)(1 - b) * a.st_pitch, b ? own : oth);  // row (lane | 1)
            };
            put(a.st_ds, pk);
            put(a.st_p, pp);
          }
        }
        if (dbgw) DBG(1, idx);
        if (acc_drab) {  // the item's bins (x nu: ds carries the user's 1/N, R#5) -> drab[h]
          if (racc != 0.f) atomicAdd(&sRacc[rb], racc);
          racc = 0.f;
          named_bar_sync(1, 32 * NSM);
          const int i = threadIdx.x - 128;
          if (i < a.nb) {
            const float v = sRacc[i];
            if (v != 0.f) atomicAdd(&a.drab[it.h * a.nb + i], us.nu * v);
            sRacc[i] = 0.f;  // the next item's first atomics follow its tile 0 barriers
          }
        }
        // !TWO: every S MMA of this item has completed: hand the next item's row operand (already
        // in the staging area) to the tensor pipe before draining this item's accumulator.
        // (TWO: the next item's rows are loaded only after this epilogue frees the region.)
        if (!TWO && !a.row_cp) {
          const int k2 = q_read(n + 1);  // peek (released when it is processed)
          Item nx;
          if (k2 >= 0 && decode_item<TRANS>(a, k2, crank, nx) && nx.ntiles > 0) copy_rows();
        }
        if (dbgw) DBG(2, idx);
        mbar_wait(o_full, mi & 1);
        tc_fence_after();
        ++mi;
      }
      if (dbgw) DBG(3, idx);

      // ---------------------------------------------------------------- epilogue
      // Warp (q, half): rows q*32.., head-dim columns half*128.. in four 32-column chunks, the
      // TMEM load of chunk cc+1 in flight while chunk cc is processed.  The SiLU' source (bwd)
      // is in the epilogue tile (TMA); the outputs are formed in place and each finished
      // 64-column box of the warp's 32 rows leaves by a TMA store (row stores for a ragged last
      // chunk).  Candidate rows add their diagonal term from E (global; R#9).
      const bool row_ok = my < us.L;
      // the diagonal of real-time rows is inside the iterated key range (added in the loop);
      // candidate rows' own column lies outside it: their diagonal term is added here
      const bool has_e = row_ok && my >= it.kv_end;
      const float dg = dg_pre;
      const __nv_bfloat16* erow = a.e + g * a.ld_e + it.hcol + half * 128;
      const int nrows = min(BR, us.L - it.r0);
      const bool full_chunk = q * 32 + 32 <= nrows;
      const int row0 = us.off + it.r0;
      uint8_t* epi = smem + OFF_EPI;
      // FWD has no SiLU' source: compile the element loop without it
      const bool use_u = MODE != FWD && a.uu != nullptr;
      const bool pre_ds = a.pre_dsilu != 0;
      const bool any_e = __any_sync(0xffffffffu, has_e);  // warp-uniform: skip the E loads
      if (a.uu != nullptr) mbar_wait(eu_full, idx & 1);
      const bool do_bias = MODE != FWD && a.dbias != nullptr;
      uint32_t r[2][32];
      if (it.ntiles > 0) tmem_ld32(tmem + T_ACC + half * 128 + lane_off, r[0]);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int acol = half * 128 + cc * 32;  // head-dim column of this chunk
        uint32_t (&rc)[32] = r[cc & 1];
        if (it.ntiles > 0) {
          tmem_ld_wait();
          if (cc < 3) tmem_ld32(tmem + T_ACC + acol + 32 + lane_off, r[(cc + 1) & 1]);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) rc[i] = 0u;
        }
        const int bx = acol >> 6, j0 = (acol & 63) >> 3;
        uint8_t* box = epi + bx * (RT_BYTES / 4);
        float v[32];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t off = sw128(row, j0 + i);
          uint4 ew = make_uint4(0u, 0u, 0u, 0u);
          if (any_e && has_e) ew = __ldg(reinterpret_cast<const uint4*>(erow + cc * 32 + 8 * i));
          uint4 uw = make_uint4(0u, 0u, 0u, 0u);
          if (use_u) uw = *reinterpret_cast<const uint4*>(box + off);
          const __nv_bfloat162* eh = reinterpret_cast<const __nv_bfloat162*>(&ew);
          const __nv_bfloat162* uh = reinterpret_cast<const __nv_bfloat162*>(&uw);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const float2 fe = __bfloat1622float2(eh[kk]);
            float x0 = fmaf(us.nu, __uint_as_float(rc[8 * i + 2 * kk]), dg * fe.x);
            float x1 = fmaf(us.nu, __uint_as_float(rc[8 * i + 2 * kk + 1]), dg * fe.y);
            if (use_u) {
              const float2 fu = __bfloat1622float2(uh[kk]);
              x0 *= pre_ds ? fu.x : dsilu_fast(fu.x);
              x1 *= pre_ds ? fu.y : dsilu_fast(fu.y);
            }
            v[8 * i + 2 * kk] = x0;
            v[8 * i + 2 * kk + 1] = x1;
          }
          *reinterpret_cast<uint4*>(box + off) =
              make_uint4(pack2(v[8 * i], v[8 * i + 1]), pack2(v[8 * i + 2], v[8 * i + 3]),
                         pack2(v[8 * i + 4], v[8 * i + 5]), pack2(v[8 * i + 6], v[8 * i + 7]));
        }
        if (cc & 1) {  // box bx of this warp's 32 rows is complete: store it
          if (full_chunk) {
            fence_proxy_async_smem();  // the bulk store reads what the generic proxy wrote
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmO, box + q * 32 * 128, it.hcol + bx * 64, row0 + q * 32);
              tma_store_commit();
            }
          } else {
            __syncwarp();
            // rows of the next user must not be touched: 4 rows x 8 16-byte pieces per pass
            for (int rr = q * 32 + (lane >> 3); rr < nrows; rr += 4) {
              const int64_t go = (int64_t)(row0 + rr) * a.ld_out + it.hcol + bx * 64 + (lane & 7) * 8;
              *reinterpret_cast<uint4*>(a.out + go) = *reinterpret_cast<const uint4*>(box + sw128(rr, lane & 7));
            }
          }
        }
        if (dbgw) DBG(11 + cc, idx);
      }
      if constexpr (TWO) {
       if (do_bias) {
        // bias gradient of this projection block: column sums of the tile's (stored) outputs,
        // read back from the epilogue tile: warp sw sums rows sw, sw+8, ..., lane = 8 columns;
        // the [8 warps][256 columns] partials go through the scratch after the rings
        named_bar_sync(1, 32 * NSM);  // every warp's outputs are in the tile
        const int sw = warp - 4, bx = lane >> 3, jj = lane & 7;
        float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const uint8_t* cbox = epi + bx * (RT_BYTES / 4);
        for (int rr = sw; rr < nrows; rr += NSM) {
          const uint4 w = *reinterpret_cast<const uint4*>(cbox + sw128(rr, jj));
          const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            const float2 f = __bfloat1622float2(hh[k2]);
            cs[2 * k2] += f.x;
            cs[2 * k2 + 1] += f.y;
          }
        }
        float* red = reinterpret_cast<float*>(smem + 208 * KB);
#pragma unroll
        for (int e = 0; e < 8; ++e) red[sw * DH + lane * 8 + e] = cs[e];
        named_bar_sync(1, 32 * NSM);
        const int col = threadIdx.x - 128;
        float sum = 0.f;
#pragma unroll
        for (int w2 = 0; w2 < NSM; ++w2) sum += red[w2 * DH + col];
        if (sum != 0.f) atomicAdd(a.dbias + it.hcol + col, sum);
        named_bar_sync(1, 32 * NSM);  // scratch reusable
       }
      } else if (do_bias) {
        // (!TWO has no room for the scratch) warp sw owns columns sw*32.., lane = one column
        named_bar_sync(1, 32 * NSM);  // every warp's outputs are in the tile
        const int col = (warp - 4) * 32 + lane;
        const uint8_t* cbox = epi + (col >> 6) * (RT_BYTES / 4);
        const int cj = (col & 63) >> 3, ce = (col & 7) * 2;
        float ps[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // 8 independent chains
        int rr = 0;
        for (; rr + 8 <= nrows; rr += 8) {
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2)
            ps[k2] += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(cbox + sw128(rr + k2, cj) + ce));
        }
        for (; rr < nrows; ++rr)
          ps[0] += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(cbox + sw128(rr, cj) + ce));
        const float sum = ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
        if (sum != 0.f) atomicAdd(a.dbias + it.hcol + col, sum);
      }
      // the epilogue tile may be refilled once this warp's bulk stores have read it
      if (lane == 0) tma_store_wait_read<0>();
      __syncwarp();
      if (lane == 0) mbar_arrive(epi_free);
      if (dbgw) DBG(4, idx);
      if (dbgw) DBG(15, idx);
      ++idx;
    }
  }
  tc_fence_before();
  cluster_sync();  // no CTA leaves while its peer may still signal its barriers
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<512>(tmem);
  }
}

// ---------------------------------------------------------------------------------------------
// Score kernel of the stored-score backward.  Per (key pair, head) item: S^T = K Q^T and
// dP^T = V dO^T tile by tile, both row operands in TMEM (TS MMAs, M=256 on CTA pairs, N=64 query
// columns, K=256), and the softmax warps write P^T = silu(S^T) m and dS^T = dP^T silu'(S^T) m
// into the stored-score matrices.  No accumulator and no epilogue: dK, dV and dQ are the three
// stored-score GEMMs (attn_mm_kernel).  Warp roles: w0 producer (Q tiles), w3 producer (dO
// tiles), w2 TMEM allocator + row loader (K, V of the next item into the staging as soon as the
// previous rows are in TMEM), w1 MMA issuer (leader), w4-w11 softmax.
// smem: R1 (K) staging [0,64) KB, R2 (V) staging [64,128), Q ring 3 x 16 [128,176), dO ring
// 3 x 16 [176,224), query timestamps, barriers.  TMEM: R1 [0,128), R2 [128,256), S/dP double
// buffered [256,512).
constexpr int SC_OFF_R1 = 0, SC_OFF_R2 = 64 * KB, SC_OFF_C1 = 128 * KB, SC_OFF_C2 = 176 * KB;
constexpr int SC_OFF_TS = 224 * KB;
constexpr int SC_OFF_BAR = SC_OFF_TS + BC * 8;
constexpr int SC_SMEM_BYTES = SMEM_BYTES;  // the rab weights at off_rab(false) as in FWD / DV
constexpr int SC_NC = 3;

template <bool RAB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    attn_sc_kernel(const __grid_constant__ CUtensorMap tmC1, const __grid_constant__ CUtensorMap tmC2,
                   const __grid_constant__ CUtensorMap tmR1, const __grid_constant__ CUtensorMap tmR2, Args a) {
  using namespace sm100;
  constexpr bool TRANS = true;
  constexpr int C1_BYTES = 32 * DH * 2;  // 16 KB: 4 boxes {64 dh, 32 cols}
  constexpr uint32_t T_R1 = 0, T_R2 = 128, T_S0 = 256;  // S[b] = T_S0 + 128 b, dP[b] = S[b] + 64
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  long long* sTs = reinterpret_cast<long long*>(smem + SC_OFF_TS);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SC_OFF_BAR);
  float* sRab = reinterpret_cast<float*>(smem + off_rab(false));  // RAB: rab_w[h][0, nb)
  uint64_t* c1_full = bars;        // [3] leader
  uint64_t* c1_empty = bars + 3;   // [3]
  uint64_t* c2_full = bars + 6;    // [3] leader
  uint64_t* c2_empty = bars + 9;   // [3]
  uint64_t* s_full = bars + 12;    // [2]
  uint64_t* s_free = bars + 14;    // [2] leader, both CTAs' softmax warps
  uint64_t* r_full = bars + 16;    // own: R1 + R2 staging landed
  uint64_t* r_copied = bars + 17;  // own: staging copied into TMEM (8 softmax warps)
  uint64_t* r_done = bars + 18;    // leader: both CTAs' rows in TMEM
  uint64_t* r_free = bars + 19;    // every MMA of the item done (TMEM rows reusable)
  uint64_t* q_full = bars + 20;    // [4]
  uint64_t* q_empty = bars + 24;   // [4] leader
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 28);
  int* q_item = reinterpret_cast<int*>(bars + 29);  // [4]
  auto arrive_leader = [&](uint64_t* bar) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      if (leader) mbar_arrive(bar);
      else mbar_arrive_cluster(bar, 0);
    }
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < SC_NC; ++s) {
      mbar_init(&c1_full[s], 1); mbar_init(&c1_empty[s], 1);
      mbar_init(&c2_full[s], 1); mbar_init(&c2_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) { mbar_init(&s_full[s], 1); mbar_init(&s_free[s], 2 * NSM); }
    mbar_init(r_full, 1);
    mbar_init(r_copied, a.sc_cp ? 1 : NSM);  // tcgen05.cp: one commit arrival
    mbar_init(r_done, 2 * NSM);
    mbar_init(r_free, 1);
    for (int s = 0; s < 4; ++s) {
      mbar_init(&q_full[s], 1);
      // per CTA: 8 softmax warps, producer B, row loader, MMA | producer A
      mbar_init(&q_empty[s], 2 * (NSM + 3));
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto q_read = [&](int n) -> int {
    mbar_wait_cluster(&q_full[n & 3], (n >> 2) & 1);
    return *reinterpret_cast<volatile int*>(&q_item[n & 3]);
  };
  auto q_release = [&](int n) {
    if (leader) mbar_arrive(&q_empty[n & 3]);
    else mbar_arrive_cluster(&q_empty[n & 3], 0);
  };
  auto q_push = [&](int n) -> int {
    if (n >= 4) mbar_wait(&q_empty[n & 3], ((n >> 2) & 1) ^ 1);
    int k;
    for (;;) {
      k = atomicAdd(a.ctr, 1);
      if (k >= a.nitems) { k = -1; break; }
      const int rest = k / a.H;
      const int u = rest / a.pmax, p = rest % a.pmax;
      const int L = a.jag.offsets[u + 1] - a.jag.offsets[u];
      // items with query tiles only: key pairs below kv_end (dynamic) / below L (causal)
      const int kv = a.causal ? L : a.jag.n_static[u] + a.jag.n_rt[u];
      if (p * 2 * BR < kv) break;
    }
    q_item[n & 3] = k;
    st_cluster_u32(reinterpret_cast<uint32_t*>(&q_item[n & 3]), 1, (uint32_t)k);
    mbar_arrive(&q_full[n & 3]);
    mbar_arrive_cluster_release(&q_full[n & 3], 1);
    return k;
  };

  if (warp == 2) {
    // ---------------------------------------------------------------- row loader: K, V rows of the
    // next item into the staging as soon as the softmax warps copied the previous ones to TMEM
    if (lane == 0) {
      int mi = 0;
      for (int n = 0;; ++n) {
        const int k = q_read(n);
        q_release(n);
        if (k < 0) break;
        Item it;
        decode_item<true>(a, k, crank, it);
        if (it.ntiles == 0) continue;
        const int row0 = it.us.off + it.r0;
        if (mi > 0) mbar_wait(r_copied, (mi - 1) & 1);
        if (a.sc_cp) {  // both CTAs' rows land on the leader's barrier (the MMA warp copies them)
          if (leader) mbar_expect_tx(r_full, 2 * 2 * RT_BYTES);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            tma_load_2d_2sm(smem + SC_OFF_R1 + c * (RT_BYTES / 4), &tmR1, r_full, it.hcol + c * 64, row0);
            tma_load_2d_2sm(smem + SC_OFF_R2 + c * (RT_BYTES / 4), &tmR2, r_full, it.hcol + c * 64, row0);
          }
        } else {
          mbar_expect_tx(r_full, 2 * RT_BYTES);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            tma_load_2d(smem + SC_OFF_R1 + c * (RT_BYTES / 4), &tmR1, r_full, it.hcol + c * 64, row0);
            tma_load_2d(smem + SC_OFF_R2 + c * (RT_BYTES / 4), &tmR2, r_full, it.hcol + c * 64, row0);
          }
        }
        ++mi;
      }
    }
  } else if (warp == 0 || warp == 3) {
    // ---------------------------------------------------------------- producers
    if (lane == 0) {
      const bool pa = warp == 0;
      int gt = 0;
      for (int n = 0;; ++n) {
        int k;
        if (pa && leader) {
          k = q_push(n);
        } else {
          k = q_read(n);
          q_release(n);
        }
        if (k < 0) break;
        Item it;
        decode_item<TRANS>(a, k, crank, it);
        if (it.ntiles == 0) continue;
        const CUtensorMap* tm = pa ? &tmC1 : &tmC2;
        uint64_t* full = pa ? c1_full : c2_full;
        uint64_t* empty = pa ? c1_empty : c2_empty;
        uint8_t* ring = smem + (pa ? SC_OFF_C1 : SC_OFF_C2);
        for (int t = 0; t < it.ntiles; ++t, ++gt) {
          const int slot = gt % SC_NC;
          mbar_wait(&empty[slot], ((gt / SC_NC) & 1) ^ 1);
          if (leader) mbar_expect_tx(&full[slot], 2 * C1_BYTES);
          const int row = it.us.off + it.c_begin + t * BC + 32 * crank;  // this CTA's 32 columns
          uint8_t* dst = ring + slot * C1_BYTES;
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_2d_2sm(dst + c * (C1_BYTES / 4), tm, &full[slot], it.hcol + c * 64, row);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA)
    if (leader) {
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      constexpr uint32_t idesc_s = idesc_bf16_f32(2 * BR, BC, 0, 0);
      const uint32_t c1_base = smem_u32(smem + SC_OFF_C1), c2_base = smem_u32(smem + SC_OFF_C2);
      int gt = 0, mi = 0;
      for (int n = 0;; ++n) {
        const int k = q_read(n);
        if (lane == 0) q_release(n);
        if (k < 0) break;
        Item it;
        decode_item<TRANS>(a, k, crank, it);
        if (it.ntiles == 0) continue;
        if (a.sc_cp) {
          // K and V rows of both CTAs: staging -> TMEM by tcgen05.cp (ordered after the previous
          // item's MMAs, before this item's); the commit frees the staging for the loaders
          mbar_wait(r_full, mi & 1);
          tc_fence_after();
          const uint32_t r1b = smem_u32(smem + SC_OFF_R1), r2b = smem_u32(smem + SC_OFF_R2);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk) {
              const uint32_t so = (kk >> 2) * (RT_BYTES / 4) + (kk & 3) * 32;
              tmem_cp_128x256b_2sm(tm + T_R1 + kk * 8, desc_sw128(r1b + so, 16, 1024));
              tmem_cp_128x256b_2sm(tm + T_R2 + kk * 8, desc_sw128(r2b + so, 16, 1024));
            }
            mma_commit_2sm_mc(r_copied, 0x3);
          }
          __syncwarp();
        } else {
          mbar_wait(r_done, mi & 1);  // both CTAs' K and V rows in TMEM
        }
        for (int t = 0; t < it.ntiles; ++t, ++gt) {
          const int slot = gt % SC_NC, b = gt & 1;
          mbar_wait(&c1_full[slot], (gt / SC_NC) & 1);
          mbar_wait(&c2_full[slot], (gt / SC_NC) & 1);
          mbar_wait(&s_free[b], ((gt >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t c1 = c1_base + slot * C1_BYTES, c2 = c2_base + slot * C1_BYTES;
          const uint32_t ts = tm + T_S0 + 128 * b;
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk)  // dP^T = V dO^T
              mma_bf16_ts_2sm(ts + 64, tm + T_R2 + kk * 8,
                              desc_sw128(c2 + (kk >> 2) * (C1_BYTES / 4) + (kk & 3) * 32, 16, 1024), idesc_s, kk > 0);
            mma_commit_2sm_mc(&c2_empty[slot], 0x3);
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk)  // S^T = K Q^T
              mma_bf16_ts_2sm(ts, tm + T_R1 + kk * 8,
                              desc_sw128(c1 + (kk >> 2) * (C1_BYTES / 4) + (kk & 3) * 32, 16, 1024), idesc_s, kk > 0);
            mma_commit_2sm_mc(&c1_empty[slot], 0x3);
            mma_commit_2sm_mc(&s_full[b], 0x3);
            if (t + 1 == it.ntiles) mma_commit_2sm_mc(r_free, 0x3);
          }
          __syncwarp();
        }
        ++mi;
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax + stores
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int j_half = half * 32;
    int gt = 0, mi = 0;
    for (int n = 0;; ++n) {
      const int k = q_read(n);
      __syncwarp();
      if (lane == 0) q_release(n);
      if (k < 0) break;
      Item it;
      decode_item<TRANS>(a, k, crank, it);
      if (it.ntiles == 0) continue;
      const UserSpan& us = it.us;
      const int my = it.r0 + row;  // this thread's key (user-local)
      // K and V rows of this item into TMEM (this warp: rows q*32.., head dims half*128..);
      // with tcgen05.cp the MMA warp does it
      if (!a.sc_cp) {
      if (mi > 0) mbar_wait(r_free, (mi - 1) & 1);
      mbar_wait(r_full, mi & 1);
      tc_fence_after();
#pragma unroll 1
      for (int op = 0; op < 2; ++op)
#pragma unroll 1
        for (int cc = 0; cc < 2; ++cc) {
          const uint8_t* box = smem + (op ? SC_OFF_R2 : SC_OFF_R1) + (half * 2 + cc) * (RT_BYTES / 4);
          uint32_t w[32];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 v = *reinterpret_cast<const uint4*>(box + sw128(row, j));
            w[4 * j] = v.x; w[4 * j + 1] = v.y; w[4 * j + 2] = v.z; w[4 * j + 3] = v.w;
          }
          tmem_st32(tmem + (op ? T_R2 : T_R1) + half * 64 + cc * 32 + lane_off, w);
        }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(r_copied);
      arrive_leader(r_done);
      }
      const long long my_ts = (my < us.L && a.jag.ts) ? a.jag.ts[(int64_t)us.off + my] : 0;
      const bool need_ts = RAB || (!a.causal && !a.full && (it.r0 + BR > us.ns) && (it.r0 < it.kv_end));  // uniform
      const int64_t st_row = ((int64_t)it.h * a.st_rows + a.koff[it.u] + my) * a.st_pitch;
#pragma unroll 1
      for (int t = 0; t < it.ntiles; ++t, ++gt) {
        const int c0 = it.c_begin + t * BC;
        const int b = gt & 1;
        if (need_ts) {
          const int i = threadIdx.x - 128;
          named_bar_sync(1, 32 * NSM);
          if (i < BC) sTs[i] = (c0 + i < us.L && a.jag.ts) ? a.jag.ts[us.off + c0 + i] : 0;
          if (RAB && t == 0 && i >= BC && i < BC + a.nb) sRab[i - BC] = a.rab_w[it.h * a.nb + i - BC];
          named_bar_sync(1, 32 * NSM);
        }
        mbar_wait(&s_full[b], (gt >> 1) & 1);
        tc_fence_after();
        uint32_t s[32], dp[32];
        tmem_ld32(tmem + T_S0 + 128 * b + j_half + lane_off, s);
        tmem_ld32(tmem + T_S0 + 128 * b + 64 + j_half + lane_off, dp);
        tmem_ld_wait();
        tc_fence_before();
        arrive_leader(&s_free[b]);
        if constexpr (RAB) add_rab<32>(s, my_ts, sTs + j_half, sRab, a.nb - 1);  // s_ij + rab (R#4)
        const int cb = c0 + j_half;  // this warp's 32 query columns
        uint32_t vis;
        if (a.causal) {  // queries i >= key j, i < L
          const int lo = min(max(my - cb, 0), 32), hi = min(max(us.L - cb, 0), 32);
          const uint32_t below_hi = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
          const uint32_t below_lo = lo >= 32 ? 0xffffffffu : ((1u << lo) - 1u);
          vis = (my < us.L) ? (below_hi & ~below_lo) : 0u;
        } else if (my < us.ns || (a.full && my < it.kv_end)) {  // every query of the user
          const int nvalid = us.L - cb;
          vis = nvalid >= 32 ? 0xffffffffu : (nvalid <= 0 ? 0u : ((1u << nvalid) - 1u));
        } else if (my < it.kv_end) {  // real-time keys: later non-static queries, and itself
          vis = 0;
          const int lo = min(max(us.ns - cb, 0), 32), hi = min(max(us.L - cb, 0), 32);
          for (int jj = lo; jj < hi; ++jj) vis |= (uint32_t)(my_ts < sTs[j_half + jj]) << jj;
          const int jd = my - cb;
          if (jd >= 0 && jd < 32) vis |= 1u << jd;
        } else {
          vis = 0;
        }
        uint32_t pk[16], pp[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float s0 = __uint_as_float(s[e]), s1 = __uint_as_float(s[e + 1]);
          const float g0 = fmaf(0.5f, sm100::tanh_approx(0.5f * s0), 0.5f);
          const float g1 = fmaf(0.5f, sm100::tanh_approx(0.5f * s1), 0.5f);
          float p0 = s0 * g0, p1 = s1 * g1;
          float v0 = __uint_as_float(dp[e]) * fmaf(p0, 1.0f - g0, g0);
          float v1 = __uint_as_float(dp[e + 1]) * fmaf(p1, 1.0f - g1, g1);
          {  // selects, no branch (masked entries are exact zeros, R#2)
            const bool m0 = (vis >> e) & 1u, m1 = (vis >> (e + 1)) & 1u;
            v0 = m0 ? v0 : 0.f; p0 = m0 ? p0 : 0.f;
            v1 = m1 ? v1 : 0.f; p1 = m1 ? p1 : 0.f;
          }
          pk[e >> 1] = pack2(v0, v1);
          pp[e >> 1] = pack2(p0, p1);
        }
        // 64 contiguous bytes per row and matrix; lane pairs swap halves so one 256-bit store
        // writes 16 whole row pieces
        const int bb = lane & 1;
        auto put = [&](__nv_bfloat16* base, const uint32_t* w) {
          U8 own, oth;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            own.v[i] = bb ? w[8 + i] : w[i];
            oth.v[i] = __shfl_xor_sync(0xffffffffu, bb ? w[i] : w[8 + i], 1);
          }
          __nv_bfloat16* p0 = base + st_row + cb + 16 * bb;
          stg256(p0 - (int64_t)bb * a.st_pitch, bb ? oth : own);
          stg256(p0 + (int64_t)(1 - bb) * a.st_pitch, bb ? own : oth);
        };
        put(a.st_ds, pk);
        put(a.st_p, pp);
      }
      ++mi;
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<512>(tmem);
  }
}

// ---------------------------------------------------------------------------------------------
// Stored-score backward products (the DK kernel wrote P^T and dS^T of every visible key row):
//
//   MM_DV: dV_j = nu sum_i P^T_ji dO_i   rows = keys    A = P^T  (K-major: queries contiguous)
//   MM_DQ: dQ_i = nu sum_j dS^T_ji K_j   rows = queries A = dS^T (MN-major: queries contiguous)
//
// plus the candidate diagonal term, silu'(p) and the bias-gradient column sums in the same
// epilogue as the attention kernel.  These are plain jagged GEMMs (M = 256 rows per CTA pair,
// N = 256 head dims, K = 64 per tile): both operands come from smem by TMA (B = dO / K rows,
// each CTA loads half of the head dim), and the accumulator is double-buffered in TMEM
// (2 x 256 columns) so an item's epilogue overlaps the next item's MMAs.  The work items, key /
// query ranges and the dynamic work queue are those of the attention kernel, so every tile read
// here was written by the DK kernel (rows of a user's padded key block, see attn_koff_kernel).
// Warp roles (384 threads): w0 TMA producer (A, B), w1 MMA issuer (leader CTA), w2 TMEM
// allocator + SiLU' tile loader, w3 idle, w4-w11 epilogue.
enum { MM_DV = 0, MM_DQ = 1 };
constexpr int MM_STAGES = 4;
constexpr int MM_A_BYTES = BR * BC * 2;             // 16 KB
constexpr int MM_B_BYTES = BC * (DH / 2) * 2;       // 16 KB (this CTA's half of the head dim)
constexpr int MM_STAGE_BYTES = MM_A_BYTES + MM_B_BYTES;
constexpr int MM_OFF_EPI = MM_STAGES * MM_STAGE_BYTES;  // 128 KB
constexpr int MM_OFF_RED = MM_OFF_EPI + RT_BYTES;       // 192 KB: dbias partials [8][256] fp32
constexpr int MM_OFF_BAR = MM_OFF_RED + NSM * DH * 4;   // 200 KB
constexpr int MM_SMEM_BYTES = MM_OFF_BAR + 512 + 1024;

template <int M2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    attn_mm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmO,
                   Args a) {
  using namespace sm100;
  constexpr bool TRANS = (M2 == MM_DV);
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + MM_OFF_BAR);
  uint64_t* full = bars;              // [4] leader
  uint64_t* empty = bars + 4;         // [4]
  uint64_t* tfull = bars + 8;         // [2] (multicast commit)
  uint64_t* tempty = bars + 10;       // [2] leader, both CTAs' epilogue warps
  uint64_t* eu_full = bars + 12;      // own
  uint64_t* epi_free = bars + 13;     // own
  uint64_t* q_full = bars + 14;       // [4]
  uint64_t* q_empty = bars + 18;      // [4] leader
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);
  int* q_item = reinterpret_cast<int*>(bars + 23);  // [4]
  auto arrive_leader = [&](uint64_t* bar) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      if (leader) mbar_arrive(bar);
      else mbar_arrive_cluster(bar, 0);
    }
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < MM_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * NSM); }
    mbar_init(eu_full, 1);
    mbar_init(epi_free, NSM);
    for (int s = 0; s < 4; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 2 * (NSM + 2));  // per CTA: 8 epilogue warps, U loader, MMA | producer
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto q_read = [&](int n) -> int {
    mbar_wait_cluster(&q_full[n & 3], (n >> 2) & 1);
    return *reinterpret_cast<volatile int*>(&q_item[n & 3]);
  };
  auto q_release = [&](int n) {
    if (leader) mbar_arrive(&q_empty[n & 3]);
    else mbar_arrive_cluster(&q_empty[n & 3], 0);
  };
  auto q_push = [&](int n) -> int {
    if (n >= 4) mbar_wait(&q_empty[n & 3], ((n >> 2) & 1) ^ 1);
    int k;
    for (;;) {
      k = atomicAdd(a.ctr, 1);
      if (k >= a.nitems) { k = -1; break; }
      const int rest = k / a.H;
      const int u = rest / a.pmax, p = rest % a.pmax;
      if (p * 2 * BR < a.jag.offsets[u + 1] - a.jag.offsets[u]) break;
    }
    q_item[n & 3] = k;
    st_cluster_u32(reinterpret_cast<uint32_t*>(&q_item[n & 3]), 1, (uint32_t)k);
    mbar_arrive(&q_full[n & 3]);
    mbar_arrive_cluster_release(&q_full[n & 3], 1);
    return k;
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- producer: A and B tiles
    if (lane == 0) {
      int gt = 0;
      for (int n = 0;; ++n) {
        int k;
        if (leader) {
          k = q_push(n);
        } else {
          k = q_read(n);
          q_release(n);
        }
        if (k < 0) break;
        Item it;
        decode_item<TRANS>(a, k, crank, it);
        const int64_t krow = (int64_t)it.h * a.st_rows + a.koff[it.u];  // user's key block
        for (int t = 0; t < it.ntiles; ++t, ++gt) {
          const int slot = gt % MM_STAGES;
          mbar_wait(&empty[slot], ((gt / MM_STAGES) & 1) ^ 1);
          // DQ: 64-query boxes wholly past the user's last query are not loaded (their D rows are
          // never stored; MMA rows are independent), e.g. 3 of the 4 boxes of a last pair holding
          // 6 queries.  The leader expects the bytes both CTAs actually load.
          int nbox = 4;
          if (M2 == MM_DQ) nbox = (it.pr0 < it.us.L) + (it.pr0 + 64 < it.us.L) + (it.pr0 + 128 < it.us.L) + (it.pr0 + 192 < it.us.L);
          if (leader) mbar_expect_tx(&full[slot], 2 * MM_B_BYTES + (M2 == MM_DQ ? nbox * (MM_A_BYTES / 2) : 2 * MM_A_BYTES));
          uint8_t* sa = smem + slot * MM_STAGE_BYTES;
          uint8_t* sb = sa + MM_A_BYTES;
          const int c0 = it.c_begin + t * BC;
          if (M2 == MM_DV) {  // P^T rows = this CTA's 128 keys, 64 query columns (K-major)
            tma_load_2d_2sm(sa, &tmA, &full[slot], c0, (int)(krow + it.r0));
          } else {            // dS^T rows = 64 keys, this CTA's 128 query columns (MN-major)
#pragma unroll
            for (int c = 0; c < 2; ++c)
              if (it.r0 + c * 64 < it.us.L)
                tma_load_2d_2sm(sa + c * (MM_A_BYTES / 2), &tmA, &full[slot], it.r0 + c * 64, (int)(krow + c0));
          }
#pragma unroll
          for (int c = 0; c < 2; ++c)  // B: 64 rows (dO for DV, K for DQ), this CTA's 128 head dims
            tma_load_2d_2sm(sb + c * (MM_B_BYTES / 2), &tmB, &full[slot], it.hcol + (2 * crank + c) * 64,
                            it.us.off + c0);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA)
    if (leader) {
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      constexpr uint32_t idesc = idesc_bf16_f32(2 * BR, DH, M2 == MM_DQ ? 1 : 0, 1);
      const uint32_t base = smem_u32(smem);
      int gt = 0, mi = 0;
      for (int n = 0;; ++n) {
        const int k = q_read(n);
        if (lane == 0) q_release(n);
        if (k < 0) break;
        Item it;
        decode_item<TRANS>(a, k, crank, it);
        if (it.ntiles == 0) continue;
        const int buf = mi & 1;
        mbar_wait(&tempty[buf], ((mi >> 1) & 1) ^ 1);
        tc_fence_after();
        for (int t = 0; t < it.ntiles; ++t, ++gt) {
          const int slot = gt % MM_STAGES;
          mbar_wait(&full[slot], (gt / MM_STAGES) & 1);
          tc_fence_after();
          const uint32_t sa = base + slot * MM_STAGE_BYTES, sb = sa + MM_A_BYTES;
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BC / 16; ++kk) {
              const uint64_t ad = M2 == MM_DQ ? desc_sw128(sa + kk * 2048, MM_A_BYTES / 2, 1024)
                                              : desc_sw128(sa + kk * 32, 16, 1024);
              mma_bf16_ss_2sm(tm + buf * DH, ad, desc_sw128(sb + kk * 2048, MM_B_BYTES / 2, 1024), idesc,
                              (t > 0 || kk > 0) ? 1u : 0u);
            }
            mma_commit_2sm_mc(&empty[slot], 0x3);
            if (t + 1 == it.ntiles) mma_commit_2sm_mc(&tfull[buf], 0x3);
          }
          __syncwarp();
        }
        ++mi;
      }
    }
  } else if (warp == 2) {
    // ---------------------------------------------------------------- SiLU' source tile loader
    if (lane == 0) {
      int idx = 0;
      for (int n = 0;; ++n) {
        const int k = q_read(n);
        q_release(n);
        if (k < 0) break;
        Item it;
        decode_item<TRANS>(a, k, crank, it);
        if (a.uu != nullptr) {
          if (idx > 0) mbar_wait(epi_free, (idx - 1) & 1);
          mbar_expect_tx(eu_full, RT_BYTES);
#pragma unroll
          for (int c = 0; c < 4; ++c)
            tma_load_2d(smem + MM_OFF_EPI + c * (RT_BYTES / 4), &tmU, eu_full, it.hcol + c * 64, it.us.off + it.r0);
        }
        ++idx;
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int mi = 0, idx = 0;
    for (int n = 0;; ++n) {
      const int k = q_read(n);
      __syncwarp();
      if (lane == 0) q_release(n);
      if (k < 0) break;
      Item it;
      decode_item<TRANS>(a, k, crank, it);
      const UserSpan& us = it.us;
      const int my = it.r0 + row;
      const int64_t g = (int64_t)us.off + my;
      const bool has_acc = it.ntiles > 0;
      const int buf = mi & 1;
      if (has_acc) {
        mbar_wait(&tfull[buf], (mi >> 1) & 1);
        tc_fence_after();
      }
      const uint32_t tacc = tmem + buf * DH + half * 128 + lane_off;
      const bool row_ok = my < us.L;
      const bool has_e = row_ok && my >= it.kv_end;  // candidate rows: diagonal term (R#9)
      const float dg = has_e ? a.diag[g * a.H + it.h] : 0.f;
      const __nv_bfloat16* erow = a.e + g * a.ld_e + it.hcol + half * 128;
      const int nrows = min(BR, us.L - it.r0);
      const bool full_chunk = q * 32 + 32 <= nrows;
      const int row0 = us.off + it.r0;
      uint8_t* epi = smem + MM_OFF_EPI;
      if (a.uu != nullptr) mbar_wait(eu_full, idx & 1);
      uint32_t r[2][32];
      if (has_acc) tmem_ld32(tacc, r[0]);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int acol = half * 128 + cc * 32;
        uint32_t (&rc)[32] = r[cc & 1];
        if (has_acc) {
          tmem_ld_wait();
          if (cc < 3) {
            tmem_ld32(tacc + (cc + 1) * 32, r[(cc + 1) & 1]);
          } else {  // the whole accumulator is in registers: the next item may overwrite it
            tc_fence_before();
            arrive_leader(&tempty[buf]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) rc[i] = 0u;
        }
        const int bx = acol >> 6, j0 = (acol & 63) >> 3;
        uint8_t* box = epi + bx * (RT_BYTES / 4);
        float v[32];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t off = sw128(row, j0 + i);
          uint4 ew = make_uint4(0u, 0u, 0u, 0u);
          if (has_e) ew = __ldg(reinterpret_cast<const uint4*>(erow + cc * 32 + 8 * i));
          uint4 uw = make_uint4(0u, 0u, 0u, 0u);
          if (a.uu != nullptr) uw = *reinterpret_cast<const uint4*>(box + off);
          const __nv_bfloat162* eh = reinterpret_cast<const __nv_bfloat162*>(&ew);
          const __nv_bfloat162* uh = reinterpret_cast<const __nv_bfloat162*>(&uw);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const float2 fe = __bfloat1622float2(eh[kk]);
            float x0 = fmaf(us.nu, __uint_as_float(rc[8 * i + 2 * kk]), dg * fe.x);
            float x1 = fmaf(us.nu, __uint_as_float(rc[8 * i + 2 * kk + 1]), dg * fe.y);
            if (a.uu != nullptr) {
              const float2 fu = __bfloat1622float2(uh[kk]);
              x0 *= a.pre_dsilu ? fu.x : dsilu_fast(fu.x);
              x1 *= a.pre_dsilu ? fu.y : dsilu_fast(fu.y);
            }
            v[8 * i + 2 * kk] = x0;
            v[8 * i + 2 * kk + 1] = x1;
          }
          *reinterpret_cast<uint4*>(box + off) =
              make_uint4(pack2(v[8 * i], v[8 * i + 1]), pack2(v[8 * i + 2], v[8 * i + 3]),
                         pack2(v[8 * i + 4], v[8 * i + 5]), pack2(v[8 * i + 6], v[8 * i + 7]));
        }
        if (cc & 1) {
          if (full_chunk) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmO, box + q * 32 * 128, it.hcol + bx * 64, row0 + q * 32);
              tma_store_commit();
            }
          } else {
            __syncwarp();
            for (int rr = q * 32 + (lane >> 3); rr < nrows; rr += 4) {
              const int64_t go = (int64_t)(row0 + rr) * a.ld_out + it.hcol + bx * 64 + (lane & 7) * 8;
              *reinterpret_cast<uint4*>(a.out + go) = *reinterpret_cast<const uint4*>(box + sw128(rr, lane & 7));
            }
          }
        }
      }
      if (has_acc) ++mi;
      if (a.dbias != nullptr) {
        // bias gradient: column sums of the stored outputs, read back from the epilogue tile
        named_bar_sync(1, 32 * NSM);
        const int sw = warp - 4, bx = lane >> 3, jj = lane & 7;
        float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const uint8_t* cbox = epi + bx * (RT_BYTES / 4);
        for (int rr = sw; rr < nrows; rr += NSM) {
          const uint4 w = *reinterpret_cast<const uint4*>(cbox + sw128(rr, jj));
          const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            const float2 f = __bfloat1622float2(hh[k2]);
            cs[2 * k2] += f.x;
            cs[2 * k2 + 1] += f.y;
          }
        }
        float* red = reinterpret_cast<float*>(smem + MM_OFF_RED);
#pragma unroll
        for (int e = 0; e < 8; ++e) red[sw * DH + lane * 8 + e] = cs[e];
        named_bar_sync(1, 32 * NSM);
        const int col = threadIdx.x - 128;
        float sum = 0.f;
#pragma unroll
        for (int w2 = 0; w2 < NSM; ++w2) sum += red[w2 * DH + col];
        if (sum != 0.f) atomicAdd(a.dbias + it.hcol + col, sum);
        named_bar_sync(1, 32 * NSM);
      }
      if (lane == 0) tma_store_wait_read<0>();
      __syncwarp();
      if (lane == 0) mbar_arrive(epi_free);
      ++idx;
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<512>(tmem);
  }
}

// Padded key-row offsets of the stored scores: user u owns rows [koff[u], koff[u+1]) of every
// head's slab, koff[u+1] - koff[u] = 256 * ceil((n_static + n_rt) / 256) (the key pairs the DK
// kernel visits; causal: 256 * ceil(L / 256)).  One block, sequential over chunks of 1024 users.
__global__ void attn_koff_kernel(mtgr_jagged_t j, int causal, int* koff) {
  __shared__ int wsum[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < j.num_users; base += 1024) {
    const int u = base + threadIdx.x;
    const int kv = u < j.num_users ? (causal ? j.offsets[u + 1] - j.offsets[u] : j.n_static[u] + j.n_rt[u]) : 0;
    const int v = ((kv + 2 * BR - 1) / (2 * BR)) * (2 * BR);
    int x = v;  // inclusive warp scan
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
    if (u < j.num_users) koff[u + 1] = incl;
    if (base == 0 && threadIdx.x == 0) koff[0] = 0;
    __syncthreads();
    if (threadIdx.x == 1023) carry = incl;
    __syncthreads();
  }
}

// drab[h][b] = sum over visible (i, j) with bucket(ts_i - ts_j) = b of ds_ij (R#4; the
// oracle's attn_bwd_user), read back from the stored dS^T of the kv / stored-score backward.
// A block owns 64 consecutive padded key rows [koff[u] + 64c, +64) of one head (a user's block
// of rows is a multiple of 256, so a chunk never spans two users; one search for u per block,
// the user's timestamps staged in shared memory), each warp 8 of them: the key's visible query
// range [lo, L) in lane-interleaved bf16 pairs (coalesced; 8 pairs in flight), summed run by run (equal buckets: the time gaps along a row change
// bucket rarely) and each finished run (x nu, the user's 1/N in ds) into the block's shared bins,
// which leave to drab at the end.  Candidate keys have no off-diagonal entries (their diagonal
// terms come from the diagonal kernel).
constexpr int DRAB_TS_CAP = 8192;  // query chunk whose timestamps are staged in smem

__global__ void __launch_bounds__(256) attn_drab_kernel(mtgr_jagged_t j, int causal, int full, int nb,
                                                        const int* koff, const __nv_bfloat16* ds,
                                                        int64_t pitch, int64_t rows, float* drab) {
  // dynamic smem: the chunk's timestamps [min(max_len, CAP)], then per-lane private bins
  // [8 warps][nb][32 lanes] (conflict-free, no atomics: a lane adds a finished run to its own)
  extern __shared__ int64_t s_ts[];
  __shared__ int s_u;
  const int h = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row0 = blockIdx.x * 64;
  if (threadIdx.x == 0) {
    int u = -1;
    if (row0 < koff[j.num_users]) {  // the user whose padded rows hold row0
      int lo_u = 0, hi_u = j.num_users - 1;
      while (lo_u < hi_u) {
        const int mid = (lo_u + hi_u + 1) >> 1;
        if (koff[mid] <= row0) lo_u = mid; else hi_u = mid - 1;
      }
      u = lo_u;
    }
    s_u = u;
  }
  __syncthreads();
  const int u = s_u;
  if (u < 0) return;  // uniform: padded rows past the last user
  const UserSpan us = load_user(j, u);
  const int cap = min(max(j.max_len, 1), DRAB_TS_CAP);
  float* bins = reinterpret_cast<float*>(s_ts + cap);
  float* mine = bins + warp * nb * 32 + lane;  // bins of this lane: mine[b * 32]
  for (int b = 0; b < nb; ++b) mine[b * 32] = 0.f;
  const int64_t* tsg = j.ts + us.off;  // ts may be NULL: every timestamp 0
  const int kv_end = causal ? us.L : us.ns + us.nr;
  for (int c0 = 0; c0 < us.L; c0 += DRAB_TS_CAP) {  // query chunks (one up to CAP tokens)
    const int c1 = min(us.L, c0 + DRAB_TS_CAP);
    __syncthreads();
    for (int i = c0 + threadIdx.x; i < c1; i += 256) s_ts[i - c0] = j.ts ? tsg[i] : 0;
    __syncthreads();
    for (int r = 0; r < 8; ++r) {
      const int kj = row0 - koff[u] + warp * 8 + r;  // key (user-local)
      if (kj >= kv_end) break;
      const int64_t ts_j = j.ts ? tsg[kj] : 0;
      // visible queries of key kj: causal i >= kj; full / static keys every i; real-time keys
      // i == kj or (i >= ns and ts_j < ts_i)
      const int lo = causal ? kj : ((full || kj < us.ns) ? 0 : us.ns);
      const bool all_vis = causal || full || kj < us.ns;  // uniform
      const int qa = max(lo, c0);
      const __nv_bfloat16* row = ds + ((int64_t)h * rows + row0 + warp * 8 + r) * pitch;
      int rb = 0;
      float racc = 0.f;
      // lane-interleaved query pairs (coalesced dS^T and timestamp reads), 8 pairs in flight;
      // a run of equal buckets is summed in a register and added to the lane's bin when it ends
      for (int i0 = (qa & ~1) + 2 * lane; i0 < c1; i0 += 512) {
        __nv_bfloat162 w[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int i = i0 + 64 * e;
          w[e] = i < c1 ? *reinterpret_cast<const __nv_bfloat162*>(row + i) : __nv_bfloat162{};
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int i = i0 + 64 * e;
          const float2 f = __bfloat1622float2(w[e]);
          const longlong2 t2 = *reinterpret_cast<const longlong2*>(s_ts + ((min(i, c1 - 1) - c0) & ~1));  // pair (i, i+1)
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int ii = i + h2;
            const int64_t ts_i = h2 ? t2.y : t2.x;
            const bool ok = ii >= qa && ii < c1 && (all_vis || ii == kj || (ii >= us.ns && ts_j < ts_i));
            const int bk = rab_bkt(ts_i - ts_j, nb - 1);
            const bool brk = ok && bk != rb;
            if (brk) {  // predicated, not atomic: the lane's own bin
              mine[rb * 32] += racc;
              rb = bk;
              racc = 0.f;
            }
            racc += ok ? (h2 ? f.y : f.x) : 0.f;
          }
        }
      }
      mine[rb * 32] += racc;
    }
  }
  __syncthreads();
  for (int b = threadIdx.x >> 5; b < nb; b += 8) {  // warp per bucket: 8 x 32 lane bins
    float v = 0.f;
    for (int w2 = 0; w2 < 8; ++w2) v += bins[(w2 * nb + b) * 32 + lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && v != 0.f) atomicAdd(&drab[h * nb + b], us.nu * v);  // x nu (R#5's 1/N in ds)
  }
}

static mtgr_status_t launch_drab(const AttnIO& io, const int* koff, const __nv_bfloat16* ds, int64_t pitch,
                                 int64_t rows, cudaStream_t st) {
  if (io.nb <= 0 || io.drab == nullptr || io.rab_w == nullptr) return MTGR_OK;
  ProfScope ps(PROF_ATTN_DRAB, st);
  // padded rows koff[B] <= rows (= T + 256 B); chunks past koff[B] exit at once
  dim3 grid((unsigned)ceil_div64(rows, 64), io.H);
  const int smem = std::min(std::max(io.jag.max_len, 1), DRAB_TS_CAP) * 8 + 8 * io.nb * 32 * 4;
  cudaFuncSetAttribute(attn_drab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  attn_drab_kernel<<<grid, 256, smem, st>>>(io.jag, io.causal, io.full, io.nb, koff, ds, pitch, rows, io.drab);
  return check_launch("attn_drab");
}

static int num_sms_cached() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct Maps {
  CUtensorMap c1, c2, x, r1, r2, e, u, o;
};

template <int MODE>
static mtgr_status_t launch_mode(const AttnIO& io, const void* c1, int64_t ld_c1, const void* x,
                                 int64_t ld_x, const void* r1, int64_t ld_r1, const void* r2,
                                 int64_t ld_r2, const void* e, int64_t ld_e, const void* uu,
                                 int64_t ld_u, const Args& args, cudaStream_t st) {
  const int T = io.jag.total_tokens, d = io.d;
  constexpr bool TWO = (MODE == DQ || MODE == DK);
  Maps m;
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
  Args a2 = args;
  a2.causal = io.causal;
  a2.full = io.full;
  a2.nb = io.nb > 0 && io.rab_w != nullptr ? io.nb : 0;
  a2.rab_w = io.rab_w;
  // row operand into TMEM by tcgen05.cp from the MMA warp (default) or through the softmax
  // warps' registers (MTGR_ROW_CP=0)
  { const char* x = getenv("MTGR_ROW_CP"); a2.row_cp = !(x != nullptr && x[0] == '0'); }
  a2.e = (const __nv_bfloat16*)e; a2.ld_e = ld_e;
  a2.uu = (const __nv_bfloat16*)uu; a2.ld_u = ld_u;
  a2.pre_dsilu = io.pre_dsilu;
  a2.pmax = ceil_div(io.jag.max_len, 2 * BR);
  a2.nitems = io.jag.num_users * a2.pmax * io.H;
  MTGR_CHECK(io.ctr != nullptr, MTGR_E_ARG, "attention: work-queue counters (workspace) missing");
  a2.ctr = io.ctr + MODE;  // per-call counters in the caller's workspace (stream-safe)
  cudaMemsetAsync(a2.ctr, 0, sizeof(int), st);
  const int pairs = std::max(1, std::min(num_sms_cached() / 2, a2.nitems));
  dim3 grid(2 * pairs, 1, 1);  // persistent CTA pairs
  ProfScope ps(MODE == FWD ? PROF_ATTN_FWD : MODE == DV ? PROF_ATTN_DV : MODE == DK ? PROF_ATTN_DK_FUSED : PROF_ATTN_DQ, st);
  // rab on: the instantiation that adds the bias (and reads the timestamps of every tile)
  auto kern = a2.nb > 0 ? attn_tc_kernel<MODE, true> : attn_tc_kernel<MODE, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  static const bool trace = getenv("MTGR_ATTN_TRACE") != nullptr;
  if (trace) {  // debug only: time-stamp one CTA pair's pipeline events
    cudaMalloc(&a2.dbg, 2 * 20 * 64 * sizeof(long long));
    cudaMemsetAsync(a2.dbg, 0, 2 * 20 * 64 * sizeof(long long), st);
  }
  kern<<<grid, 384, SMEM_BYTES, st>>>(m.c1, m.c2, m.x, m.r1, m.r2, m.e, m.u, m.o, a2);
  if (trace) {
    long long hb[2 * 20 * 64];
    cudaMemcpyAsync(hb, a2.dbg, sizeof(hb), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(a2.dbg);
    fprintf(stderr, "ATTN_TRACE mode=%d", MODE);
    for (int i = 0; i < 2 * 20 * 64; ++i) fprintf(stderr, " %lld", hb[i]);
    fprintf(stderr, "\n");
  }
  return check_launch("attn_tc");
}

// Stored-score scratch: koff [B+1] int32, then P^T and dS^T, each [H][rows][pitch] bf16 with
// rows = T + 256 B (>= sum_u 256 ceil(kv_u / 256)) and pitch = 256 ceil(max_len / 256).
struct MmLayout {
  int64_t pitch = 0, rows = 0;
  size_t koff = 0, p = 0, ds = 0, total = 0;
};
static MmLayout mm_layout(const mtgr_jagged_t& j, int H) {
  MmLayout l;
  l.pitch = (int64_t)ceil_div(std::max(j.max_len, 1), 2 * BR) * 2 * BR;
  l.rows = (int64_t)j.total_tokens + (int64_t)2 * BR * j.num_users;
  const size_t mat = (size_t)H * l.rows * l.pitch * 2;
  l.koff = 0;
  l.p = ((size_t)(j.num_users + 1) * 4 + 1023) / 1024 * 1024;
  l.ds = l.p + (mat + 1023) / 1024 * 1024;
  l.total = l.ds + (mat + 1023) / 1024 * 1024;
  return l;
}

template <int M2>
static mtgr_status_t launch_mm(const AttnIO& io, const void* amat, const void* b, int64_t ld_b,
                               const void* e, int64_t ld_e, const void* uu, int64_t ld_u,
                               const MmLayout& l, const Args& args, int prof, cudaStream_t st) {
  const int T = io.jag.total_tokens, d = io.d;
  CUtensorMap ta, tb, tu, to;
  MTGR_TRY(make_tmap_bf16(&ta, amat, (uint64_t)l.pitch, (uint64_t)io.H * l.rows, (uint64_t)l.pitch, 64,
                          M2 == MM_DV ? BR : BC));
  MTGR_TRY(make_tmap_bf16(&tb, b, d, T, ld_b, 64, BC));
  if (uu) MTGR_TRY(make_tmap_bf16(&tu, uu, d, T, ld_u, 64, BR)); else tu = tb;
  MTGR_TRY(make_tmap_bf16(&to, args.out, d, T, args.ld_out, 64, 32));
  Args a2 = args;
  a2.causal = io.causal;
  a2.full = io.full;
  // row operand into TMEM by tcgen05.cp from the MMA warp (default) or through the softmax
  // warps' registers (MTGR_ROW_CP=0)
  { const char* x = getenv("MTGR_ROW_CP"); a2.row_cp = !(x != nullptr && x[0] == '0'); }
  a2.e = (const __nv_bfloat16*)e; a2.ld_e = ld_e;
  a2.uu = (const __nv_bfloat16*)uu; a2.ld_u = ld_u;
  a2.pre_dsilu = io.pre_dsilu;
  a2.pmax = ceil_div(io.jag.max_len, 2 * BR);
  a2.nitems = io.jag.num_users * a2.pmax * io.H;
  a2.st_pitch = l.pitch; a2.st_rows = l.rows;
  a2.c_align = 1;
  MTGR_CHECK(io.ctr != nullptr, MTGR_E_ARG, "attention: work-queue counters (workspace) missing");
  a2.ctr = io.ctr + 4 + M2;
  cudaMemsetAsync(a2.ctr, 0, sizeof(int), st);
  const int pairs = std::max(1, std::min(num_sms_cached() / 2, a2.nitems));
  ProfScope ps(prof, st);
  cudaFuncSetAttribute(attn_mm_kernel<M2>, cudaFuncAttributeMaxDynamicSharedMemorySize, MM_SMEM_BYTES);
  attn_mm_kernel<M2><<<2 * pairs, 384, MM_SMEM_BYTES, st>>>(ta, tb, tu, to, a2);
  return check_launch("attn_mm");
}

static mtgr_status_t launch_sc(const AttnIO& io, const MmLayout& l, const Args& args, cudaStream_t st) {
  const int T = io.jag.total_tokens, d = io.d;
  CUtensorMap tc1, tc2, tr1, tr2;
  MTGR_TRY(make_tmap_bf16(&tc1, io.q, d, T, io.ld, 64, BC / 2));   // Q columns (32 per CTA)
  MTGR_TRY(make_tmap_bf16(&tc2, io.dO, d, T, io.d, 64, BC / 2));  // dO columns
  MTGR_TRY(make_tmap_bf16(&tr1, io.k, d, T, io.ld, 64, BR));      // K rows
  MTGR_TRY(make_tmap_bf16(&tr2, io.v, d, T, io.ld, 64, BR));      // V rows
  Args a2 = args;
  a2.causal = io.causal;
  a2.full = io.full;
  a2.pmax = ceil_div(io.jag.max_len, 2 * BR);
  a2.nitems = io.jag.num_users * a2.pmax * io.H;
  a2.st_pitch = l.pitch; a2.st_rows = l.rows;
  a2.c_align = 1;
  a2.nb = io.nb > 0 && io.rab_w != nullptr ? io.nb : 0;
  a2.rab_w = io.rab_w;
  { const char* x = getenv("MTGR_SC_CP"); a2.sc_cp = !(x != nullptr && x[0] == '0'); }  // as MTGR_ROW_CP
  MTGR_CHECK(io.ctr != nullptr, MTGR_E_ARG, "attention: work-queue counters (workspace) missing");
  a2.ctr = io.ctr + 6;
  cudaMemsetAsync(a2.ctr, 0, sizeof(int), st);
  const int pairs = std::max(1, std::min(num_sms_cached() / 2, a2.nitems));
  ProfScope ps(PROF_ATTN_SC, st);
  auto kern = a2.nb > 0 ? attn_sc_kernel<true> : attn_sc_kernel<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SC_SMEM_BYTES);
  kern<<<2 * pairs, 384, SC_SMEM_BYTES, st>>>(tc1, tc2, tr1, tr2, a2);
  return check_launch("attn_sc");
}

// Coupled dK/dV backward (tc_attn_kv.cu): koff [B+1], the stored dS^T matrix [H][rows][pitch]
// of the dQ GEMM, then the coupling workspace (tickets, flags, item lists, G rings)
struct KvLayout {
  size_t koff = 0, ds = 0, sync = 0, total = 0;
};
static KvLayout kv_layout(const mtgr_jagged_t& j, int H) {
  const MmLayout m = mm_layout(j, H);
  KvLayout l;
  l.ds = m.p;  // same koff / matrix geometry as the stored-score path
  l.sync = l.ds + (m.ds - m.p);
  l.total = l.sync + align_up(attn_kv_ws_bytes(j, H), 1024);
  return l;
}

}  // namespace tca

bool attn_tc_supported(int dh) { return dh == tca::DH; }

size_t attn_store_ws_bytes(const mtgr_jagged_t& j, int H) {
  if (j.num_users == 0 || j.total_tokens == 0) return 0;
  const char* env = getenv("MTGR_ATTN_RECOMPUTE");  // tests / A-B: force the recompute kernels
  if (env != nullptr && env[0] == '1') return 0;
  const size_t b = std::max(tca::mm_layout(j, H).total, tca::kv_layout(j, H).total);
  // beyond this the backward recomputes the scores in the DV / DQ kernels instead
  return b <= ((size_t)48 << 30) ? b : 0;
}

mtgr_status_t attn_tc_fwd_launch(const AttnIO& io, cudaStream_t st) {
  using namespace tca;
  if (io.jag.num_users == 0 || io.jag.max_len == 0 || io.jag.total_tokens == 0) return MTGR_OK;
  MTGR_CHECK(!io.u || io.y, MTGR_E_ARG, "attention forward: gate without y output");
  MTGR_CHECK(io.d % 8 == 0, MTGR_E_LAYOUT, "d_model must be a multiple of 8");
  Args a{};
  a.jag = io.jag; a.H = io.H; a.d = io.d;
  a.out = (__nv_bfloat16*)io.o; a.ld_out = io.d;
  a.diag = io.diag_a;
  // C1 = K, X = V, R1 = Q, E = V; the gate (if any) is a separate elementwise pass
  MTGR_TRY(launch_mode<FWD>(io, io.k, io.ld, io.v, io.ld, io.q, io.ld, nullptr, 0, io.v, io.ld,
                            nullptr, 0, a, st));
  if (io.u) MTGR_TRY(gate_mul_launch(io.o, io.d, io.u, io.ld, io.y, io.d, io.jag.total_tokens, io.d, st));
  return MTGR_OK;
}

mtgr_status_t attn_tc_bwd_launch(const AttnIO& io, cudaStream_t st) {
  using namespace tca;
  if (io.jag.num_users == 0 || io.jag.max_len == 0 || io.jag.total_tokens == 0) return MTGR_OK;
  typedef __nv_bfloat16 bf;
  const bf* pre = (const bf*)io.pre;
  const int64_t D = io.d;
  const size_t need = attn_store_ws_bytes(io.jag, io.H);
  if (need > 0 && io.mm_ws != nullptr && io.mm_ws_bytes >= need) {
    // stored-score backward: DK computes S^T, dP^T once and writes P^T and dS^T; dV and dQ are
    // then plain jagged GEMMs over them (no recomputation of S and dP)
    const MmLayout l = mm_layout(io.jag, io.H);
    char* ws = (char*)io.mm_ws;
    int* koff = (int*)(ws + l.koff);
    bf* sp = (bf*)(ws + l.p);
    bf* sds = (bf*)(ws + l.ds);
    attn_koff_kernel<<<1, 1024, 0, st>>>(io.jag, io.causal, koff);
    MTGR_TRY(check_launch("attn_koff"));
    // Which backward: MTGR_ATTN_BWD = kv (default: the coupled dK/dV kernel writes dS^T, then the
    // dQ GEMM), stored (score kernel writes P^T and dS^T, then dK / dV / dQ GEMMs) or fused_dk
    // (the DK kernel writes both while forming dK).  MTGR_ATTN_FUSED_DK=1 / =0 (round 1) still
    // selects fused_dk / stored.
    const char* benv = getenv("MTGR_ATTN_BWD");
    const char* fenv = getenv("MTGR_ATTN_FUSED_DK");
    int path = 0;  // 0 kv, 1 stored, 2 fused_dk
    if (benv != nullptr) path = benv[0] == 's' ? 1 : (benv[0] == 'f' ? 2 : 0);
    else if (fenv != nullptr) path = fenv[0] == '1' ? 2 : 1;
    if (path == 0) {
      const KvLayout kl = kv_layout(io.jag, io.H);
      bf* kds = (bf*)(ws + kl.ds);
      Args ax{}, ay{};
      for (Args* p : {&ax, &ay}) { p->jag = io.jag; p->H = io.H; p->d = io.d; p->koff = koff; }
      ay.st_ds = kds; ay.st_pitch = l.pitch; ay.st_rows = l.rows;
      MTGR_TRY(attn_kv_launch(io, ax, ay, ws + kl.sync, st));
      Args a{};
      a.jag = io.jag; a.H = io.H; a.d = io.d;
      a.out = (bf*)io.dq; a.ld_out = io.ld_out; a.diag = io.diag_ds;
      a.dbias = io.dbias;
      a.koff = koff;
      MTGR_TRY(launch_mm<MM_DQ>(io, kds, io.k, io.ld, io.k, io.ld, pre, io.ld_pre, l, a, PROF_ATTN_DQ, st));
      return launch_drab(io, koff, kds, l.pitch, l.rows, st);
    }
    if (path == 2) {  // dK = nu dS^T Q (+ diag), * silu'(p_K); also stores P^T, dS^T
      Args a{};
      a.jag = io.jag; a.H = io.H; a.d = io.d;
      a.out = (bf*)io.dk; a.ld_out = io.ld_out; a.diag = io.diag_ds;
      a.dbias = io.dbias ? io.dbias + D : nullptr;
      a.st_p = sp; a.st_ds = sds; a.st_pitch = l.pitch; a.st_rows = l.rows; a.koff = koff;
      a.c_align = 1;
      MTGR_TRY(launch_mode<DK>(io, io.q, io.ld, io.dO, D, io.k, io.ld, io.v, io.ld, io.q, io.ld,
                               pre ? pre + D : nullptr, io.ld_pre, a, st));
    } else {
      {  // scores: S^T, dP^T -> P^T, dS^T
        Args a{};
        a.jag = io.jag; a.H = io.H; a.d = io.d;
        a.st_p = sp; a.st_ds = sds; a.koff = koff;
        MTGR_TRY(launch_sc(io, l, a, st));
      }
      {  // dK = nu dS^T Q (+ diag ds_jj q_j), * silu'(p_K)
        Args a{};
        a.jag = io.jag; a.H = io.H; a.d = io.d;
        a.out = (bf*)io.dk; a.ld_out = io.ld_out; a.diag = io.diag_ds;
        a.dbias = io.dbias ? io.dbias + D : nullptr;
        a.koff = koff;
        MTGR_TRY(launch_mm<MM_DV>(io, sds, io.q, io.ld, io.q, io.ld, pre ? pre + D : nullptr, io.ld_pre, l, a,
                                  PROF_ATTN_DK, st));
      }
    }
    {  // dV = nu P^T dO (+ diag a_jj dO_j), * silu'(p_V)
      Args a{};
      a.jag = io.jag; a.H = io.H; a.d = io.d;
      a.out = (bf*)io.dv; a.ld_out = io.ld_out; a.diag = io.diag_a;
      a.dbias = io.dbias ? io.dbias + 2 * D : nullptr;
      a.koff = koff;
      MTGR_TRY(launch_mm<MM_DV>(io, sp, io.dO, D, io.dO, D, pre ? pre + 2 * D : nullptr, io.ld_pre, l, a,
                                PROF_ATTN_DV, st));
    }
    {  // dQ = nu dS K (+ diag ds_ii k_i), * silu'(p_Q)
      Args a{};
      a.jag = io.jag; a.H = io.H; a.d = io.d;
      a.out = (bf*)io.dq; a.ld_out = io.ld_out; a.diag = io.diag_ds;
      a.dbias = io.dbias;
      a.koff = koff;
      MTGR_TRY(launch_mm<MM_DQ>(io, sds, io.k, io.ld, io.k, io.ld, pre, io.ld_pre, l, a, PROF_ATTN_DQ, st));
    }
    return launch_drab(io, koff, sds, l.pitch, l.rows, st);
  }
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
    a.drab = io.nb > 0 ? io.drab : nullptr;  // drab summed inside the DQ kernel (no stored dS)
    MTGR_TRY(launch_mode<DQ>(io, io.k, io.ld, io.v, io.ld, io.q, io.ld, io.dO, D, io.k, io.ld, pre,
                             io.ld_pre, a, st));
  }
  return MTGR_OK;
}

}  // namespace mtgr
