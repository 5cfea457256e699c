// Coupled dK / dV backward of the jagged HSTU attention (Eq.5, dynamic mask
// P:323-346): the S^T / dP^T / dV / dK products of one key pair in ONE launch, without storing
// P^T and without a dV or dK GEMM over stored scores.
//
// Why two kinds of CTA pair.  With d_h = 256 the dK and dV accumulators of one CTA's 128 key
// rows take 256 TMEM columns each, so one CTA (or CTA pair) cannot hold both plus the score
// tiles.  Here the persistent CTA pairs come in COUPLES: an X pair and a Y pair process the same
// work items (256-key pair, head) in the same order, each keeping the FWD/DV kernel's TMEM plan
// (row operand 128 + accumulator 256 + score tile 64 + T tile 64 columns) and every MMA on CTA
// pairs (cta_group::2, M = 256, B split across the pair):
//
//   role | row operand (TMEM) | column tile C1 | X (acc B) | score MMA      | T tile                 | acc
//   X    | K                  | Q (64 queries) | dO        | S^T = K Q^T    | P^T = silu(S^T) m      | dV
//   Y    | V                  | dO             | Q         | dP^T = V dO^T  | dS^T = dP^T (.) G      | dK
//
// X's softmax warps also form G = silu'(S^T) m (the only thing Y needs from S) and hand it to
// Y's CTA of the same rank through an L2-resident ring (fp16, NG tiles per CTA; written and read
// at the same thread -> row mapping, 512-byte coalesced pieces per warp).  Y stores dS^T (bf16)
// for the dQ GEMM (attn_mm_kernel<MM_DQ>), exactly the layout the stored-score path uses.
//
// Coupling.  Each cluster takes a ticket when it starts (atomic counter): even = X of couple
// ticket/2, odd = its Y, so couples form in start order and a running X always gets a partner
// once SMs free up.  X's leader producer claims items from the work queue and publishes them
// (release) to its couple's item list; Y's leader producer reads them (acquire).  Per tile, X's
// softmax warps write their G pieces and bump a shared-memory counter; X's sync thread
// publishes the minimum over the 8 warps with a gpu-scope release (one fence per tile, off the
// softmax warps' path), and mirrors Y's consumed count back into shared memory, which gates the
// reuse of a ring slot.  Y's softmax warps poll the published count (acquire) and read G with
// L1-bypassing loads; Y's sync warp publishes how many tiles all 8 warps have consumed (the G
// values were used, so those loads have retired, before the counter moves).
//
// Warp roles (384 threads): w0 TMA producer (C1), w1 MMA issuer (leader CTA), w2 TMEM allocator
// with lane 0 the row-operand / epilogue-tile loader (once per item) and lane 1 the sync thread
// (independent thread scheduling: the two lanes run their own loops), w3 TMA producer (X),
// w4-w11 softmax + epilogue.
// smem and TMEM layouts are those of the FWD/DV modes of attn_tc_kernel (tc_attn.cu).
#include <algorithm>
#include <climits>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"
#include "sm100.cuh"
#include "tc_attn.cuh"

namespace mtgr {
namespace tca {

#ifndef KV_NS
#define KV_NS 2
#endif
// timing experiments only (`make EXTRA=-DMTGR_KV_DEBUG_BUILD`, then MTGR_KV_DEBUG=bits; results
// are wrong when set): 1 Y does not wait for G, 2 X writes no G, 4 Y stores no dS^T, 8 X ignores
// ring reuse, 16 X skips the softmax math.  Compiled out otherwise (the branches cost registers)
#ifdef MTGR_KV_DEBUG_BUILD
#define KV_DBG(bit) (ks.dbg & (bit))
#else
#define KV_DBG(bit) false
#endif
constexpr int KV_NG_MAX = 32;       // G ring depth (tiles) per CTA: ks.ng <= this (MTGR_KV_NG)
constexpr int KV_THREADS = 384;     // 12 warps (13 would round the register budget to 16 warps')
constexpr int KV_EXIT = 1 << 30;    // per-warp counter flag: the warp has left its item loop
constexpr int KV_FLAG_STRIDE = 32;  // ints per couple in the flag block (own 128-byte line)
constexpr int KV_SMEM_BYTES = SMEM_BYTES;

struct KvSync {
  int* role_ctr;   // cluster tickets (zeroed before the launch)
  int* flags;      // [ncouples][32]: [0] items published, [1+r] G tiles published by X CTA r,
                   // [3+r] G tiles consumed by Y CTA r (zeroed before the launch)
  int* items;      // [ncouples][item_cap] work items in X's claim order, -1 = end
  uint4* gbuf;     // [ncouples][2][KV_NG][8 warps][4 chunks][32 lanes] fp16 G pieces
  int ncouples, item_cap;
  long long* trace;  // MTGR_KV_TRACE: [role][10 events][1024] globaltimer stamps of couple 0, rank 0
  int ng;          // G ring depth in tiles
  int sleep_ns;    // sync thread poll period (MTGR_KV_SLEEP)
  int dbg;         // MTGR_KV_DEBUG (timing experiments only; results are wrong when set): 1 Y does
                   // not wait for G, 2 X writes no G, 4 Y stores no dS^T, 8 X ignores ring reuse
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release_cta_smem(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(sm100::smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta_smem(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(sm100::smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// trace events (MTGR_KV_TRACE): per item 0 start, 1 tiles done, 2 o_full, 3 epilogue done,
// 4 ntiles, 5 first S issued, 6 last acc issued; per tile 7 s_full passed, 8 t_full arrived,
// 9 S issued, 10 C1 load issued, 11 X load issued, 12 MMA saw c1_full, 13 MMA saw x_full
// (compiled in only with -DMTGR_KV_TRACE_BUILD, `make TRACE=1`: the stamps cost registers)
#ifdef MTGR_KV_TRACE_BUILD
#define KV_TR(ev, i, v) do { if (tr != nullptr && (i) < 1024) tr[(ev) * 1024 + (i)] = (v); } while (0)
#else
#define KV_TR(ev, i, v) do { } while (0)
#endif

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <bool RAB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(KV_THREADS, 1)
    attn_kv_kernel(const __grid_constant__ CUtensorMap xC1, const __grid_constant__ CUtensorMap xX,
                   const __grid_constant__ CUtensorMap xR1, const __grid_constant__ CUtensorMap xU,
                   const __grid_constant__ CUtensorMap xO, const __grid_constant__ CUtensorMap yC1,
                   const __grid_constant__ CUtensorMap yX, const __grid_constant__ CUtensorMap yR1,
                   const __grid_constant__ CUtensorMap yU, const __grid_constant__ CUtensorMap yO,
                   const __grid_constant__ Args ax, const __grid_constant__ Args ay,
                   const __grid_constant__ KvSync ks) {
  using namespace sm100;
  constexpr bool TRANS = true;
  constexpr int C1_BYTES = 32 * DH * 2;        // 16 KB: 4 boxes {64 dh, 32 cols}
  constexpr int X_BYTES = BC * (DH / 2) * 2;   // 16 KB: 2 boxes {64 dh, 64 cols}
  constexpr int NC1 = 3, NX = 3;
  // smem: C1 ring, X ring, the row operand's head dims 0..127 staged for tcgen05.cp [96,128) KB,
  // its head dims 128..255 resident for the item as the SS half of the score MMA [128,160) KB,
  // the epilogue tile [160,224) KB
  constexpr int OFF_C1 = 0, OFF_X = 48 * KB, OFF_R1STAGE = 96 * KB, OFF_R1U = 128 * KB, OFF_EPI = 160 * KB;
  // KV_NS score tiles in flight.  2 (default): the whole row operand in TMEM (TS score MMA);
  // 3: head dims 128..255 of the row operand resident in smem as the SS half of the score MMA,
  // freeing 64 TMEM columns for a third tile (measured ~3 % slower at `small`: the SS half is
  // shared-memory bound, and the two-tile chain is not what limits the loop)
  constexpr int NS = KV_NS;
  constexpr bool SPLIT_R1 = NS == 3;
  // TMEM: row operand [0,128), accumulator [128,384), score tiles S[b] = [384 + 64b, +64), b = tile & 1;
  // the bf16 T tile is written in place: warp half h's 32 values into columns [32h, 32h + 16) of
  // its own S[b] half, so the next tile's score MMA never waits for the softmax
  // TMEM: row operand head dims 0..127 [0,64), accumulator [64,320), score tiles S[b] =
  // [320 + 64b, +64), b = tile % 3 (triple-buffered: the score MMA runs two tiles ahead of the
  // softmax)
  constexpr uint32_t T_R1 = 0, T_ACC = SPLIT_R1 ? 64 : 128, T_S = SPLIT_R1 ? 320 : 384;

  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  long long* sTs = reinterpret_cast<long long*>(smem + off_ts(false));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + off_bar(false));
  float* sRab = reinterpret_cast<float*>(smem + off_rab(false));  // RAB (X): rab_w[h][0, nb)
  uint64_t* c1_full = bars;           // [3] leader
  uint64_t* c1_empty = bars + 3;      // [3]
  uint64_t* x_full = bars + 6;        // [3] leader
  uint64_t* x_empty = bars + 9;       // [3]
  uint64_t* s_full = bars + 12;       // [3] score tile b complete (multicast commit)
  uint64_t* t_full = bars + 16;       // [NS][2] leader: T tile b, warp half w written (both CTAs)
  uint64_t* r1_full = bars + 22;      // leader: both CTAs' row operand (dh 0..127) staged
  uint64_t* r1_copied = bars + 24;    // own (tcgen05.cp done: staging reusable)
  uint64_t* r1u_full = bars + 25;     // leader: both CTAs' row operand dh 128..255 resident
  uint64_t* r1u_free = bars + 26;     // own (multicast): the item's last score MMA is done
  uint64_t* o_full = bars + 30;
  uint64_t* q_full = bars + 32;       // [4] work queue: item index published (own)
  uint64_t* q_empty = bars + 36;      // [4] leader: every consumer of both CTAs has read it
  uint64_t* eu_full = bars + 40;      // epilogue SiLU' source tile landed (own)
  uint64_t* epi_free = bars + 41;     // epilogue tile free again (own; 8 softmax warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 42);
  int* q_item = reinterpret_cast<int*>(bars + 43);       // [4]
  int* ticket = reinterpret_cast<int*>(bars + 46);       // this cluster's ticket
  int* cons_ok = ticket + 1;                             // X: Y's consumed count (mirror)
  int* wcnt = ticket + 2;                                // [8] X: tiles written / Y: consumed
  int* gready = ticket + 10;                             // Y: G tiles published by X (mirror)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto arrive_leader = [&](uint64_t* bar) {  // one arrival per warp (whole warp calls)
    __syncwarp();
    if (lane == 0) {
      if (leader) mbar_arrive(bar);
      else mbar_arrive_cluster(bar, 0);
    }
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < 3; ++s) {
      mbar_init(&c1_full[s], 1); mbar_init(&c1_empty[s], 1);
      mbar_init(&x_full[s], 1); mbar_init(&x_empty[s], 1);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&t_full[2 * s], NSM); mbar_init(&t_full[2 * s + 1], NSM); mbar_init(&s_full[s], 1);
    }
    mbar_init(r1_full, 1);
    mbar_init(r1_copied, 1);
    mbar_init(r1u_full, 1);
    mbar_init(r1u_free, 1);
    mbar_init(o_full, 1);
    mbar_init(eu_full, 1);
    mbar_init(epi_free, NSM);
    for (int s = 0; s < 4; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 2 * (NSM + 3));  // per CTA: X producer, row loader, 8 softmax, MMA | C1 producer
    }
    *cons_ok = 0;
    *gready = 0;
    for (int w = 0; w < NSM; ++w) wcnt[w] = 0;
    if (leader) {  // role ticket, shared with the peer before the cluster barrier
      const int t = atomicAdd(ks.role_ctr, 1);
      *ticket = t;
      st_cluster_u32(reinterpret_cast<uint32_t*>(ticket), 1, (uint32_t)t);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int tk = *reinterpret_cast<volatile int*>(ticket);
  const int role = tk & 1;        // 0: X (S^T, P^T, dV, writes G), 1: Y (dP^T, dS^T, dK)
  const int couple = tk >> 1;
  const Args& a = role ? ay : ax;
  const CUtensorMap* mC1 = role ? &yC1 : &xC1;
  const CUtensorMap* mX = role ? &yX : &xX;
  const CUtensorMap* mR1 = role ? &yR1 : &xR1;
  const CUtensorMap* mU = role ? &yU : &xU;
  const CUtensorMap* mO = role ? &yO : &xO;
  int* cflags = ks.flags + (size_t)couple * KV_FLAG_STRIDE;
  int* items = ks.items + (size_t)couple * ks.item_cap;
  // this CTA's G ring: [KV_NG slots][8 warps][4 chunks][32 lanes] x 16 B
  uint4* gring = ks.gbuf + (size_t)(couple * 2 + (int)crank) * KV_NG_MAX * NSM * 128;
  long long* tr = (ks.trace != nullptr && couple == 0) ? ks.trace + ((size_t)role * 2 + crank) * 26 * 1024 : nullptr;
  (void)tr;  // used by the KV_TR stamps of trace builds only

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
    if (role == 0) {  // X: claim from the work queue (key pairs with query tiles) and publish
      for (;;) {
        k = atomicAdd(a.ctr, 1);
        if (k >= a.nitems) { k = -1; break; }
        const int rest = k / a.H;
        const int u = rest / a.pmax, p = rest % a.pmax;
        if (p * 2 * BR < a.jag.offsets[u + 1] - a.jag.offsets[u]) break;  // non-empty pair
      }
      items[n] = k;
      st_release_gpu(&cflags[0], n + 1);
    } else {  // Y: X's items in X's order
      while (ld_acquire_gpu(&cflags[0]) < n + 1) __nanosleep(128);
      k = __ldcg(&items[n]);
    }
    q_item[n & 3] = k;
    st_cluster_u32(reinterpret_cast<uint32_t*>(&q_item[n & 3]), 1, (uint32_t)k);
    mbar_arrive(&q_full[n & 3]);
    mbar_arrive_cluster_release(&q_full[n & 3], 1);
    return k;
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- producer: C1 column tiles
    if (lane == 0) {
      int gt = 0;
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
        for (int t = 0; t < it.ntiles; ++t, ++gt) {
          const int slot = gt % NC1;
          mbar_wait(&c1_empty[slot], ((gt / NC1) & 1) ^ 1);
          if (leader) mbar_expect_tx(&c1_full[slot], 2 * C1_BYTES);
          KV_TR(10, gt, gtimer());
          const int row = it.us.off + it.c_begin + t * BC + 32 * crank;  // this CTA's 32 columns
          uint8_t* dst = smem + OFF_C1 + slot * C1_BYTES;
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_2d_2sm(dst + c * (C1_BYTES / 4), mC1, &c1_full[slot], it.hcol + c * 64, row);
        }
      }
    }
  } else if (warp == 2 && lane == 1) {
    // ---------------------------------------------------------------- sync thread
    int done = 0;   // X: tiles published / Y: tiles reported consumed
    int seen = 0;   // Y: X's published count mirrored into shared memory
    for (;;) {
      int mn = INT_MAX;
      bool all_exit = true;
#pragma unroll
      for (int w = 0; w < NSM; ++w) {
        const int v = ld_acquire_cta_smem(&wcnt[w]);
        all_exit = all_exit && (v & KV_EXIT);
        mn = min(mn, v & ~KV_EXIT);
      }
      if (mn > done) {
        if (role == 0) {
          // the 8 warps' G stores (observed through the acquire above) before the count
          fence_acq_rel_gpu();
          st_relaxed_gpu(&cflags[1 + crank], mn);
        } else {
          // the G values of these tiles were consumed (their loads retired) before the warps
          // bumped their counters
          st_relaxed_gpu(&cflags[3 + crank], mn);
        }
        done = mn;
      }
      if (role == 0) {
        *reinterpret_cast<volatile int*>(cons_ok) = ld_relaxed_gpu(&cflags[3 + crank]);
      } else {
        // X's release -> this acquire -> the release below -> the softmax warps' acquire (smem)
        const int p = ld_acquire_gpu(&cflags[1 + crank]);
        if (p > seen) { st_release_cta_smem(gready, p); seen = p; }
      }
      if (all_exit) break;
      // the thread shares an SM sub-partition with two softmax warps: poll sparingly
      __nanosleep(ks.sleep_ns);
    }
  } else if (warp == 2) {
    // ---------------------------------------------------------------- row operand + epilogue tile
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
          constexpr int NSTAGED = SPLIT_R1 ? 2 : 4;  // 64-column boxes staged for TMEM
          if (leader) mbar_expect_tx(r1_full, NSTAGED * (RT_BYTES / 2));
#pragma unroll
          for (int c = 0; c < NSTAGED; ++c)  // head dims -> staging (then TMEM)
            tma_load_2d_2sm(smem + OFF_R1STAGE + c * (RT_BYTES / 4), mR1, r1_full, it.hcol + c * 64, it.us.off + it.r0);
          if constexpr (SPLIT_R1) {
            if (mi > 0) mbar_wait(r1u_free, (mi - 1) & 1);  // the previous item's score MMAs are done
            if (leader) mbar_expect_tx(r1u_full, RT_BYTES);
#pragma unroll
            for (int c = 2; c < 4; ++c)  // head dims 128..255 -> resident (SS half of the score MMA)
              tma_load_2d_2sm(smem + OFF_R1U + (c - 2) * (RT_BYTES / 4), mR1, r1u_full, it.hcol + c * 64, it.us.off + it.r0);
          }
          ++mi;
        }
        if (a.uu != nullptr) {
          if (idx > 0) mbar_wait(epi_free, (idx - 1) & 1);
          mbar_expect_tx(eu_full, RT_BYTES);
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_2d(smem + OFF_EPI + c * (RT_BYTES / 4), mU, eu_full, it.hcol + c * 64, it.us.off + it.r0);
        }
        ++idx;
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- producer: X tiles
    if (lane == 0) {
      int gt = 0;
      for (int n = 0;; ++n) {
        const int k = q_read(n);
        q_release(n);
        if (k < 0) break;
        Item it;
        decode_item<TRANS>(a, k, crank, it);
        for (int t = 0; t < it.ntiles; ++t, ++gt) {
          const int slot = gt % NX;
          mbar_wait(&x_empty[slot], ((gt / NX) & 1) ^ 1);
          if (leader) mbar_expect_tx(&x_full[slot], 2 * X_BYTES);
          KV_TR(11, gt, gtimer());
          const int row = it.us.off + it.c_begin + t * BC;
          uint8_t* dst = smem + OFF_X + slot * X_BYTES;
#pragma unroll
          for (int c = 0; c < 2; ++c)  // this CTA's half of the head dim
            tma_load_2d_2sm(dst + c * (X_BYTES / 2), mX, &x_full[slot], it.hcol + (2 * crank + c) * 64, row);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA)
    if (leader) {
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      constexpr uint32_t idesc_s = idesc_bf16_f32(2 * BR, BC, 0, 0);
      constexpr uint32_t idesc_acc = idesc_bf16_f32(2 * BR, DH, 0, 1);
      const uint32_t c1_base = smem_u32(smem + OFF_C1);
      const uint32_t x_base = smem_u32(smem + OFF_X);
      const uint32_t r1s_base = smem_u32(smem + OFF_R1STAGE);
      int gt = 0, mi = 0, cp_done = 0;
      // row-operand staging (both CTAs) -> TMEM by tcgen05.cp, ordered after the MMAs issued so
      // far; the commit frees the staging for the loader
      auto copy_r1 = [&]() {
        mbar_wait(r1_full, cp_done & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < (SPLIT_R1 ? DH / 32 : DH / 16); ++kk)  // the TMEM-resident head dims
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
        if (nt == 0) continue;
        if (cp_done == mi) copy_r1();  // not prefetched at the end of the previous item
        const int item_n = n;
        (void)item_n;  // trace builds only
        if constexpr (SPLIT_R1) mbar_wait(r1u_full, mi & 1);  // head dims 128..255 of the rows in smem
        const uint32_t r1u_base = smem_u32(smem + OFF_R1U);
        // acc += T_j X_j  (A = T from each CTA's TMEM, B = X: each CTA's half of the head dim)
        // per warp half w (queries 32 w.., K chunks 2w, 2w + 1): its MMAs go as soon as the 8
        // warps of that half (both CTAs) have written their T columns, not after all 16
        auto acc = [&](int j, int g) {
          const int tb = g % NS;
          mbar_wait(&x_full[g % NX], (g / NX) & 1);
          const uint32_t x = x_base + (g % NX) * X_BYTES;
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            mbar_wait(&t_full[2 * tb + w], (g / NS) & 1);
            if (lane == 0 && w == 1) KV_TR(13, g, gtimer());
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int kk = 2 * w; kk < 2 * w + 2; ++kk)
                mma_bf16_ts_2sm(tm + T_ACC, tm + T_S + 64 * tb + (kk >> 1) * 32 + (kk & 1) * 8,
                                desc_sw128(x + kk * 2048, X_BYTES / 2, 1024), idesc_acc, (j > 0 || kk > 0));
              if (w == 1) mma_commit_2sm_mc(&x_empty[g % NX], 0x3);
            }
            __syncwarp();
          }
        };
        // score tile g: head dims 0..127 with A from TMEM, 128..255 with A from smem.  Its buffer
        // (g % 3) was last read by the T MMA of tile g - 3, issued (in order) before this one
        auto score = [&](int t) {
          const int g = gt + t;
          mbar_wait(&c1_full[g % NC1], (g / NC1) & 1);
          if (lane == 0) KV_TR(12, g, gtimer());
          tc_fence_after();
          const uint32_t c1 = c1_base + (g % NC1) * C1_BYTES;
          const uint32_t ts = tm + T_S + 64 * (g % NS);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk) {
              const uint64_t bd = desc_sw128(c1 + (kk >> 2) * (C1_BYTES / 4) + (kk & 3) * 32, 16, 1024);
              if (!SPLIT_R1 || kk < 8)
                mma_bf16_ts_2sm(ts, tm + T_R1 + kk * 8, bd, idesc_s, kk > 0);
              else
                mma_bf16_ss_2sm(ts, desc_sw128(r1u_base + ((kk >> 2) - 2) * (RT_BYTES / 4) + (kk & 3) * 32, 16, 1024),
                                bd, idesc_s, 1);
            }
            mma_commit_2sm_mc(&s_full[g % NS], 0x3);
            mma_commit_2sm_mc(&c1_empty[g % NC1], 0x3);
            if (SPLIT_R1 && t + 1 == nt) mma_commit_2sm_mc(r1u_free, 0x3);  // the resident half may go
          }
          __syncwarp();
          if (lane == 0) { const long long tt = gtimer(); KV_TR(9, g, tt); if (t == 0) KV_TR(5, item_n, tt); }
        };
        // score MMAs run NS - 1 tiles ahead of the T MMAs: a score tile's buffer was last read
        // by the T MMA of tile g - NS, issued (in order) in an earlier iteration
        for (int t = 0; t < NS - 1 && t < nt; ++t) score(t);
        for (int t = 0; t < nt; ++t) {
          if (t + NS - 1 < nt) score(t + NS - 1);
          acc(t, gt + t);
        }
        if (elect_one()) mma_commit_2sm_mc(o_full, 0x3);
        __syncwarp();
        if (lane == 0) KV_TR(6, item_n, gtimer());
        {  // the next item's row operand, right behind this item's MMAs
          const int k2 = q_read(n + 1);  // peek (released when it is processed)
          Item nx;
          if (k2 >= 0 && decode_item<TRANS>(a, k2, crank, nx) && nx.ntiles > 0) copy_r1();
        }
        gt += nt;
        ++mi;
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax + epilogue
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int sw = warp - 4;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int j_half = half * 32;
    int gt = 0, mi = 0, idx = 0;
    int ready = 0;  // Y: G tiles known published
    uint4 gpre[4];  // Y: the next tile's G piece, prefetched
    int gpre_t = -1;
    for (int n = 0;; ++n) {
      const int k = q_read(n);
      __syncwarp();
      if (lane == 0) q_release(n);
      if (k < 0) break;
      Item it;
      decode_item<TRANS>(a, k, crank, it);
      const UserSpan& us = it.us;
      const int my = it.r0 + row;                    // this thread's key (user-local)
      const int64_t g = (int64_t)us.off + my;        // global token index
      const bool trw = warp == 4 && lane == 0;
      if (trw) { KV_TR(0, n, gtimer()); KV_TR(4, n, it.ntiles); }
      // the candidate-row diagonal scalar of the epilogue, loaded now: its latency hides behind the tiles
      const float dg_pre = (my < us.L && my >= it.kv_end) ? a.diag[g * a.H + it.h] : 0.f;
      if (it.ntiles > 0) {
        const long long my_ts = (role == 0 && my < us.L && a.jag.ts) ? a.jag.ts[g] : 0;
        // stored dS^T row of this key (Y): [h][koff[u] + my][query]
        const int64_t st_row = role ? ((int64_t)it.h * a.st_rows + a.koff[it.u] + my) * a.st_pitch : 0;
        const bool need_ts = role == 0 && (RAB || (!a.causal && a.full == 0 && (it.r0 + BR > us.ns) && (it.r0 < it.kv_end)));
#pragma unroll 1
        for (int t = 0; t < it.ntiles; ++t, ++gt) {
          const int c0 = it.c_begin + t * BC;
          const int cb = c0 + j_half;  // this warp's 32 query columns
          uint4* gp = gring + ((size_t)(gt & (ks.ng - 1)) * NSM + sw) * 128;  // this warp's G piece
          uint32_t pk[16];
          if (role == 0) {
            // ---------------- X: P^T = silu(S^T) m for the dV MMA, G = silu'(S^T) m for Y
            if (need_ts) {  // query timestamps of this tile (uniform over the 8 softmax warps)
              const int i = threadIdx.x - 128;
              named_bar_sync(1, 32 * NSM);
              if (i < BC) sTs[i] = (c0 + i < us.L && a.jag.ts) ? a.jag.ts[us.off + c0 + i] : 0;
              if (RAB && t == 0 && i >= BC && i < BC + a.nb) sRab[i - BC] = a.rab_w[it.h * a.nb + i - BC];
              named_bar_sync(1, 32 * NSM);
            }
            const int tb = gt % NS;
            mbar_wait(&s_full[tb], (gt / NS) & 1);
            if (trw) KV_TR(7, gt, gtimer());
            tc_fence_after();
            // the 32 columns in two halves: the second TMEM load is in flight while the first
            // half's SiLU / SiLU' are formed
            uint32_t sa[16], sb[16];
            tmem_ld16(tmem + T_S + 64 * tb + j_half + lane_off, sa);
            tmem_ld_wait();
            tmem_ld16(tmem + T_S + 64 * tb + j_half + 16 + lane_off, sb);
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
            uint32_t gw[16];
            const bool all_vis = vis == 0xffffffffu;
            auto half16 = [&](const uint32_t* sv, int e0) {
#pragma unroll
              for (int e = 0; e < 16; e += 2) {
                const float2 x = make_float2(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1]));
                // silu and silu' share sigma(s): p = s sigma, g = sigma + p (1 - sigma)
                const float2 sg = sigmoid2_fast(x);
                float2 p2 = f2mul(x, sg);
                float2 d2 = f2fma(p2, f2add(make_float2(1.f, 1.f), make_float2(-sg.x, -sg.y)), sg);
                if (!all_vis) {  // selects, no branch per element (masked entries exact zeros, R#2)
                  const bool m0 = (vis >> (e0 + e)) & 1u, m1 = (vis >> (e0 + e + 1)) & 1u;
                  p2.x = m0 ? p2.x : 0.f; d2.x = m0 ? d2.x : 0.f;
                  p2.y = m1 ? p2.y : 0.f; d2.y = m1 ? d2.y : 0.f;
                }
                pk[(e0 + e) >> 1] = pack2(p2.x, p2.y);
                gw[(e0 + e) >> 1] = pack_h2(d2.x, d2.y);
              }
            };
            if (KV_DBG(16)) {  // timing experiment: no softmax math
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 16; ++e) { pk[e] = sa[e]; gw[e] = sb[e]; }
            } else {
              if constexpr (RAB) add_rab<16>(sa, my_ts, sTs + j_half, sRab, a.nb - 1);  // s + rab (R#4)
              half16(sa, 0);
              tmem_ld_wait();
              if constexpr (RAB) add_rab<16>(sb, my_ts, sTs + j_half + 16, sRab, a.nb - 1);
              half16(sb, 16);
            }
            tmem_st16(tmem + T_S + 64 * tb + j_half + lane_off, pk);  // in place (this warp's S)
            tmem_st_wait();
            tc_fence_before();
            arrive_leader(&t_full[2 * tb + half]);
            if (trw) KV_TR(8, gt, gtimer());
            if (lane == 0) KV_TR(18 + sw, gt, gtimer());
            // publish the PREVIOUS tile's G piece: its stores were issued a tile ago, so this
            // release (which waits for them) does not stall; this tile's follow below
            __syncwarp();
            if (lane == 0 && t > 0) st_release_cta_smem(&wcnt[sw], gt);
            // G piece -> ring slot gt % NG (free once Y consumed tile gt - NG)
            if (gt >= ks.ng && !KV_DBG(8))
              while (*reinterpret_cast<volatile int*>(cons_ok) < gt - ks.ng + 1) __nanosleep(32);
            if (!KV_DBG(2)) {
#pragma unroll
              for (int c = 0; c < 4; ++c)  // L2 evict-last: Y reads the piece back within a few tiles
                stg128_hint(&gp[c * 32 + lane], make_uint4(gw[4 * c], gw[4 * c + 1], gw[4 * c + 2], gw[4 * c + 3]),
                            l2_policy_evict_last());
            }
            if (t + 1 == it.ntiles) {  // the item's last tile: publish now (before the epilogue)
              __syncwarp();
              if (lane == 0) st_release_cta_smem(&wcnt[sw], gt + 1);
            }
          } else {
            // ---------------- Y: dS^T = dP^T (.) G for the dK MMA and the dQ GEMM
            if (ready < gt + 1 && !KV_DBG(1)) {  // X's count, mirrored by the sync thread
              int v;
              while ((v = ld_acquire_cta_smem(gready)) < gt + 1) __nanosleep(32);
              ready = v;
            }
            uint4 gv[4];
            if (gpre_t == gt) {  // prefetched during the previous tile
#pragma unroll
              for (int c = 0; c < 4; ++c) gv[c] = gpre[c];
            } else {
#pragma unroll
              for (int c = 0; c < 4; ++c) gv[c] = __ldcg(&gp[c * 32 + lane]);  // L2 (never a stale L1 line)
            }
            const int tb = gt % NS;
            mbar_wait(&s_full[tb], (gt / NS) & 1);
            if (trw) KV_TR(7, gt, gtimer());
            tc_fence_after();
            uint32_t dp[32];
            tmem_ld32(tmem + T_S + 64 * tb + j_half + lane_off, dp);
            tmem_ld_wait();
            const uint32_t* gw = reinterpret_cast<const uint32_t*>(gv);
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              __half2 h = *reinterpret_cast<const __half2*>(&gw[e >> 1]);
              const float2 ds = f2mul(make_float2(__uint_as_float(dp[e]), __uint_as_float(dp[e + 1])), __half22float2(h));
              pk[e >> 1] = pack2(ds.x, ds.y);
            }
            tmem_st16(tmem + T_S + 64 * tb + j_half + lane_off, pk);  // in place (this warp's S)
            tmem_st_wait();
            tc_fence_before();
            arrive_leader(&t_full[2 * tb + half]);
            if (trw) KV_TR(8, gt, gtimer());
            if (lane == 0) KV_TR(18 + sw, gt, gtimer());
            // this tile's G is consumed
            __syncwarp();
            if (lane == 0) *reinterpret_cast<volatile int*>(&wcnt[sw]) = gt + 1;
            // dS^T (bf16) of this row's 32 query columns: 64 contiguous bytes; lane pairs swap
            // halves so that one 256-bit store writes 16 whole 64-byte row pieces
            const int b = lane & 1;
            U8 own, oth;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              own.v[i] = b ? pk[8 + i] : pk[i];
              oth.v[i] = __shfl_xor_sync(0xffffffffu, b ? pk[i] : pk[8 + i], 1);
            }
            __nv_bfloat16* p0 = a.st_ds + st_row + cb + 16 * b;
            if (!KV_DBG(4)) {
              // streaming stores: dS^T is read back by the dQ GEMM only after the whole kernel
              stg256_cs(p0 - (int64_t)b * a.st_pitch, b ? oth : own);
              stg256_cs(p0 + (int64_t)(1 - b) * a.st_pitch, b ? own : oth);
            }
            // prefetch the next tile's G when it is already published (its L2 latency then hides
            // behind this tile's tail and the next score wait)
            if (t + 1 < it.ntiles && !KV_DBG(1)) {
              if (ready < gt + 2) ready = ld_acquire_cta_smem(gready);
              if (ready >= gt + 2) {
                const uint4* gn = gring + ((size_t)((gt + 1) & (ks.ng - 1)) * NSM + sw) * 128;
#pragma unroll
                for (int c = 0; c < 4; ++c) gpre[c] = __ldcg(&gn[c * 32 + lane]);
                gpre_t = gt + 1;
              }
            }
          }
        }
        if (trw) KV_TR(1, n, gtimer());
        mbar_wait(o_full, mi & 1);
        if (trw) KV_TR(2, n, gtimer());
        tc_fence_after();
        ++mi;
      }

      // ---------------------------------------------------------------- epilogue
      // (as attn_tc_kernel's DV / DK modes) warp (q, half): rows q*32.., head-dim columns
      // half*128.. in four 32-column chunks; 1/N, the candidate-key diagonal term from E, the
      // SiLU' of the projection from the TMA-staged tile; outputs formed in place and stored by TMA
      const bool row_ok = my < us.L;
      const bool has_e = row_ok && my >= it.kv_end;
      const float dg = dg_pre;
      const __nv_bfloat16* erow = a.e + g * a.ld_e + it.hcol + half * 128;
      const int nrows = min(BR, us.L - it.r0);
      const bool full_chunk = q * 32 + 32 <= nrows;
      const int row0 = us.off + it.r0;
      uint8_t* epi = smem + OFF_EPI;
      const bool use_u = a.uu != nullptr;
      const bool pre_ds = a.pre_dsilu != 0;
      const bool any_e = __any_sync(0xffffffffu, has_e);
      if (use_u) mbar_wait(eu_full, idx & 1);
      if (trw) KV_TR(14, n, gtimer());
      uint32_t r[2][32];
      if (it.ntiles > 0) tmem_ld32(tmem + T_ACC + half * 128 + lane_off, r[0]);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int acol = half * 128 + cc * 32;
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
        // one copy of the element loop per epilogue form (uniform branch outside the loop):
        // 0 no SiLU' source, 1 the saved silu'(p), 2 pre-activations (silu' formed here)
        auto elems = [&](auto form) {
          constexpr int F = decltype(form)::value;
          const float2 nu2 = make_float2(us.nu, us.nu), dg2 = make_float2(dg, dg);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t off = sw128(row, j0 + i);
            uint4 ew = make_uint4(0u, 0u, 0u, 0u);
            if (any_e && has_e) ew = __ldg(reinterpret_cast<const uint4*>(erow + cc * 32 + 8 * i));
            uint4 uw = make_uint4(0u, 0u, 0u, 0u);
            if (F != 0) uw = *reinterpret_cast<const uint4*>(box + off);
            const __nv_bfloat162* eh = reinterpret_cast<const __nv_bfloat162*>(&ew);
            const __nv_bfloat162* uh = reinterpret_cast<const __nv_bfloat162*>(&uw);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              float2 x = f2mul(nu2, make_float2(__uint_as_float(rc[8 * i + 2 * kk]), __uint_as_float(rc[8 * i + 2 * kk + 1])));
              if (any_e) x = f2fma(dg2, __bfloat1622float2(eh[kk]), x);
              if constexpr (F == 1) x = f2mul(x, __bfloat1622float2(uh[kk]));
              if constexpr (F == 2) {
                const float2 fu = __bfloat1622float2(uh[kk]);
                x = f2mul(x, make_float2(dsilu_fast(fu.x), dsilu_fast(fu.y)));
              }
              v[8 * i + 2 * kk] = x.x;
              v[8 * i + 2 * kk + 1] = x.y;
            }
            *reinterpret_cast<uint4*>(box + off) =
                make_uint4(pack2(v[8 * i], v[8 * i + 1]), pack2(v[8 * i + 2], v[8 * i + 3]),
                           pack2(v[8 * i + 4], v[8 * i + 5]), pack2(v[8 * i + 6], v[8 * i + 7]));
          }
        };
        if (!use_u) elems(std::integral_constant<int, 0>{});
        else if (pre_ds) elems(std::integral_constant<int, 1>{});
        else elems(std::integral_constant<int, 2>{});
        if (a.dbias != nullptr) {
          // bias gradient of this projection block: column sums over the item's rows.  The 32
          // columns of the chunk are summed over the warp's 32 rows by a butterfly
          // reduce-scatter (lane l ends with column l), then one red.add per lane.  (Reading the
          // column pairs back from the bf16 tile instead was 2x slower: measured.)
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = row_ok ? v[i] : 0.f;
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < o; ++i) {
              const float send = up ? v[i] : v[i + o];
              const float keep = up ? v[i + o] : v[i];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
          if (v[0] != 0.f) atomicAdd(a.dbias + it.hcol + acol + lane, v[0]);
        }
        if (trw && cc == 1) KV_TR(15, n, gtimer());
        if (cc & 1) {  // box bx of this warp's 32 rows is complete: store it
          if (full_chunk) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(mO, box + q * 32 * 128, it.hcol + bx * 64, row0 + q * 32);
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
      if (trw) KV_TR(16, n, gtimer());
      if (lane == 0) tma_store_wait_read<0>();
      __syncwarp();
      if (lane == 0) mbar_arrive(epi_free);
      if (trw) KV_TR(3, n, gtimer());
      ++idx;
    }
    // leave the item loop: the sync thread stops once every warp has (X: after publishing the
    // last tiles)
    __syncwarp();
    if (lane == 0) {
      if (role == 0) st_release_cta_smem(&wcnt[sw], gt | KV_EXIT);
      else *reinterpret_cast<volatile int*>(&wcnt[sw]) = gt | KV_EXIT;
    }
  }
  tc_fence_before();
  cluster_sync();  // no CTA leaves while its peer may still signal its barriers
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<512>(tmem);
  }
}

// workspace of the coupled kernel: tickets + flags (zeroed per launch), item lists, G rings
size_t kv_sync_bytes(int ncouples, int item_cap) {
  return align_up(256 + (size_t)ncouples * KV_FLAG_STRIDE * 4, 256) +
         align_up((size_t)ncouples * item_cap * 4, 256) +
         (size_t)ncouples * 2 * KV_NG_MAX * NSM * 128 * sizeof(uint4);
}

static int kv_couples() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (n <= 0) n = 148;
  return std::max(1, n / 4);  // clusters of 2, couples of 2 clusters
}

}  // namespace tca

size_t attn_kv_ws_bytes(const mtgr_jagged_t& j, int H) {
  using namespace tca;
  const int pmax = ceil_div(std::max(j.max_len, 1), 2 * BR);
  const int item_cap = j.num_users * pmax * H + 8;
  return kv_sync_bytes(kv_couples(), item_cap);
}

// dK and dV of the tensor-core backward (no dQ): X pairs write dV, Y pairs dK and the stored
// dS^T rows (l.ds layout of the stored-score path) the dQ GEMM reads
mtgr_status_t attn_kv_launch(const AttnIO& io, const tca::Args& ax_in, const tca::Args& ay_in, void* sync_ws,
                             cudaStream_t st) {
  using namespace tca;
  const int T = io.jag.total_tokens, d = io.d;
  const int64_t D = io.d;
  typedef __nv_bfloat16 bf;
  const bf* pre = (const bf*)io.pre;
  CUtensorMap xc1, xx, xr1, xu, xo, yc1, yx, yr1, yu, yo;
  // X: C1 = Q columns (32 per CTA), X = dO (64 rows, d_h halves), R1 = K rows, U = p_V, O = dV
  MTGR_TRY(make_tmap_bf16(&xc1, io.q, d, T, io.ld, 64, BC / 2));
  MTGR_TRY(make_tmap_bf16(&xx, io.dO, d, T, D, 64, BC));
  MTGR_TRY(make_tmap_bf16(&xr1, io.k, d, T, io.ld, 64, BR));
  if (pre) MTGR_TRY(make_tmap_bf16(&xu, pre + 2 * D, d, T, io.ld_pre, 64, BR)); else xu = xr1;
  MTGR_TRY(make_tmap_bf16(&xo, io.dv, d, T, io.ld_out, 64, 32));
  // Y: C1 = dO columns, X = Q, R1 = V rows, U = p_K, O = dK
  MTGR_TRY(make_tmap_bf16(&yc1, io.dO, d, T, D, 64, BC / 2));
  MTGR_TRY(make_tmap_bf16(&yx, io.q, d, T, io.ld, 64, BC));
  MTGR_TRY(make_tmap_bf16(&yr1, io.v, d, T, io.ld, 64, BR));
  if (pre) MTGR_TRY(make_tmap_bf16(&yu, pre + D, d, T, io.ld_pre, 64, BR)); else yu = yr1;
  MTGR_TRY(make_tmap_bf16(&yo, io.dk, d, T, io.ld_out, 64, 32));
  Args ax = ax_in, ay = ay_in;
  for (Args* p : {&ax, &ay}) {
    p->causal = io.causal;
    p->full = io.full;
    p->pre_dsilu = io.pre_dsilu;
    p->pmax = ceil_div(io.jag.max_len, 2 * BR);
    p->nitems = io.jag.num_users * p->pmax * io.H;
    p->c_align = 1;
    p->ld_out = io.ld_out;
  }
  ax.out = (bf*)io.dv; ax.e = (const bf*)io.dO; ax.ld_e = D; ax.diag = io.diag_a;
  ax.uu = pre ? pre + 2 * D : nullptr; ax.ld_u = io.ld_pre;
  ax.dbias = io.dbias ? io.dbias + 2 * D : nullptr;
  ay.out = (bf*)io.dk; ay.e = (const bf*)io.q; ay.ld_e = io.ld; ay.diag = io.diag_ds;
  ay.uu = pre ? pre + D : nullptr; ay.ld_u = io.ld_pre;
  ay.dbias = io.dbias ? io.dbias + D : nullptr;
  MTGR_CHECK(io.ctr != nullptr, MTGR_E_ARG, "attention: work-queue counters (workspace) missing");
  ax.ctr = ay.ctr = io.ctr + 7;
  const int nc = kv_couples();
  const int item_cap = ax.nitems + 8;
  KvSync ks{};
  char* w = (char*)sync_ws;
  const size_t flag_bytes = align_up(256 + (size_t)nc * KV_FLAG_STRIDE * 4, 256);
  ks.role_ctr = (int*)w;
  ks.flags = (int*)(w + 256);
  ks.items = (int*)(w + flag_bytes);
  ks.gbuf = (uint4*)(w + flag_bytes + align_up((size_t)nc * item_cap * 4, 256));
  ks.ncouples = nc;
  ks.item_cap = item_cap;
  { const char* e = getenv("MTGR_KV_DEBUG"); ks.dbg = e ? atoi(e) : 0; }
  { const char* e = getenv("MTGR_KV_SLEEP"); ks.sleep_ns = e ? std::max(0, atoi(e)) : 256; }
  {  // a power of two (slot = tile & (ng - 1))
    const char* e = getenv("MTGR_KV_NG");
    int ng = e ? std::max(2, std::min(KV_NG_MAX, atoi(e))) : 16;
    while (ng & (ng - 1)) ng &= ng - 1;
    ks.ng = ng;
  }
  static const bool trace = getenv("MTGR_KV_TRACE") != nullptr;
  const size_t trn = 2 * 2 * 26 * 1024;
  if (trace) {  // debug only
    cudaMalloc(&ks.trace, trn * sizeof(long long));
    cudaMemsetAsync(ks.trace, 0, trn * sizeof(long long), st);
  }
  cudaMemsetAsync(w, 0, flag_bytes, st);
  cudaMemsetAsync(ax.ctr, 0, sizeof(int), st);
  // rab on (X role adds the bias; drab: attn_drab_kernel over the stored dS^T afterwards)
  ax.nb = io.nb > 0 && io.rab_w != nullptr ? io.nb : 0;
  ax.rab_w = io.rab_w;
  ProfScope ps(PROF_ATTN_KV, st);
  auto kern = ax.nb > 0 ? attn_kv_kernel<true> : attn_kv_kernel<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, KV_SMEM_BYTES);
  kern<<<4 * nc, KV_THREADS, KV_SMEM_BYTES, st>>>(xc1, xx, xr1, xu, xo, yc1, yx, yr1, yu, yo, ax, ay, ks);
  if (trace) {
    std::vector<long long> hb(trn);
    cudaMemcpyAsync(hb.data(), ks.trace, trn * sizeof(long long), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(ks.trace);
    fprintf(stderr, "KV_TRACE");
    for (size_t i = 0; i < trn; ++i) fprintf(stderr, " %lld", hb[i]);
    fprintf(stderr, "\n");
  }
  return check_launch("attn_kv");
}

}  // namespace mtgr
