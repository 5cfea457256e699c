// tcgen05 bf16 GEMM for the layer's dense contractions (PAPER.md P:313 QKVU projection,
// Eq.6 output "MLP", and their backward): C[M][N] = A[M][K] * B[N][K]^T, fp32 accumulation
// in TMEM.
//
// Persistent, warp-specialised; the layer GEMMs run on CTA pairs (cta_group::2, clusters of 2):
//   warp 0 : TMA producer  (4-stage ring: this CTA's 128x64 rows of A + its half, 128x64, of the
//            256x64 B tile, SWIZZLE_128B, 2-SM TMA onto the leader's barriers)
//   warp 1 : MMA issuer    (leader CTA, one elected thread, tcgen05.mma.cta_group::2 M=256
//            N=256 K=16: each CTA's 128 rows of A against the whole B tile, B read half from
//            each CTA's shared memory)
//   warp 2 : TMEM allocator (512 columns = two 128x256 fp32 accumulators per CTA,
//            double-buffered so an epilogue overlaps the next tile's MMAs)
//   warps 4-11: epilogue   (two per TMEM lane quadrant: tcgen05.ld 32x32b -> registers -> fused
//            epilogue -> SW128 staging -> TMA store)
// (Geo<1, ...> is the one-CTA cta_group::1 M=128 variant, compiled in by CG_USE = 1.)
// Either operand may be K-major or MN-major (the weight-gradient and data-gradient GEMMs read
// activations [T][n] as MN-major operands directly — no transposes).  Small output grids
// (weight gradients, K = T) are split along K with a deterministic second-pass reduction.
// Fused epilogues: +bias and SiLU with both pre/post-activation stores (QKVU, R#5);
// +bias +residual (Eq.6); fp32 (partial) stores for weight gradients.
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"
#include "sm100.cuh"

namespace mtgr {
namespace tcg {

constexpr int BM = 128, BN = 256, BK = 64;  // BM = rows per CTA; a CTA pair covers 256 rows
constexpr int A_BYTES = BM * BK * 2;
constexpr int NUM_EPI_WARPS = 8;                     // 2 per TMEM lane quadrant
constexpr int CHUNK_BYTES = 32 * 128;                // one [32 rows][64 bf16] SW128 staging tile
constexpr int NTHREADS = 128 + 32 * NUM_EPI_WARPS;

// per-cta_group geometry: CG = 1 (one CTA, M=128 MMA) or 2 (CTA pair, M=256 MMA; each CTA holds
// its 128 rows of A and half of the 256 B rows, so per-SM operand traffic halves)
// Each epilogue warp double-buffers its staging tile, so the bulk store of one 64-column chunk
// drains while the next chunk is formed (QKVU, two outputs per chunk, keeps one buffer pair: its
// shared memory goes to a fourth pipeline stage instead, which measured faster).
template <int CG, int EPI>
struct Geo {
  static constexpr int B_ROWS = BN / CG;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int NOUT = EPI == 1 ? 2 : 1;  // EPI_QKVU writes C and C2
  static constexpr int BUF_BYTES = NOUT * CHUNK_BYTES;
  static constexpr int NBUF = NOUT == 2 ? 1 : 2;
  static constexpr int STG_BYTES = NBUF * BUF_BYTES;
  static constexpr int STAGES = CG == 2 ? 4 : 3;
  static constexpr int OFF_STG = STAGES * STAGE_BYTES;
  static constexpr int OFF_BAR = OFF_STG + NUM_EPI_WARPS * STG_BYTES;
  static constexpr int SMEM_BYTES = OFF_BAR + 512 + 1024;
};

struct Params {
  int M, N, K;
  int num_m, num_n, num_splits, kb_per_split, num_kb;
  int a_mn, b_mn;
  void* C;
  int64_t ldc;
  const float* bias;
  float* part;  // split-K partials [splits][M][N]
  int accumulate;
  int silu;
  int c_dsilu;  // QKVU with silu: C = silu'(pre) instead of pre
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float silu_tanh(float x) {
  const float h = 0.5f * x;
  return fmaf(h, sm100::tanh_approx(h), h);
}

// Epilogue layout: epilogue warp ew (warps 4..11) owns TMEM lane quadrant q = warp % 4 (rows
// q*32..q*32+31 of the CTA's 128 rows) and column half ew / 4; it drains two 64-column chunks
// per tile: tcgen05.ld -> fused math -> bf16 into a SWIZZLE_128B smem staging tile [32][64] ->
// TMA store (bulk group).  The residual tile is TMA-loaded into the same staging buffer.
template <int EPI, int CG>
__global__ void __launch_bounds__(NTHREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
                   const __grid_constant__ CUtensorMap tmR, Params p) {
  using namespace sm100;
  using G = Geo<CG, EPI>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base, derived by indexing the shared array so the compiler keeps the shared
  // address space (LDS/STS rather than generic LD/ST for every staged access)
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + G::STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  uint64_t* empty = full + G::STAGES;
  uint64_t* tfull = empty + G::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;  // [NUM_EPI_WARPS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + NUM_EPI_WARPS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int cta_id = blockIdx.x / CG, ncta = gridDim.x / CG;  // cluster-level work distribution
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (EPI != EPI_F32) tma_prefetch(&tmC);
    if (EPI == EPI_QKVU) tma_prefetch(&tmC2);
    if (EPI == EPI_RESID) tma_prefetch(&tmR);
    for (int s = 0; s < G::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], CG * 32 * NUM_EPI_WARPS);  // the leader collects both CTAs' epilogues
    }
    for (int w = 0; w < NUM_EPI_WARPS; ++w) mbar_init(&rbar[w], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    if (CG == 2) tmem_alloc_2sm<512>(tmem_slot);
    else tmem_alloc<512>(tmem_slot);
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = p.num_m * p.num_n * p.num_splits;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int item = cta_id; item < total; item += ncta) {
        const int nb = item % p.num_n, rest = item / p.num_n;
        const int mb = rest % p.num_m, sp = rest / p.num_m;
        const int kb0 = sp * p.kb_per_split, kb1 = min(p.num_kb, kb0 + p.kb_per_split);
        const int m0 = mb * BM * CG + rank * BM;
        const int n0 = nb * BN + rank * G::B_ROWS;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full[stage], CG * G::STAGE_BYTES);
          const int k = kb * BK;
          uint8_t* a_dst = sA + stage * A_BYTES;
          uint8_t* b_dst = sB + stage * G::B_BYTES;
          auto load = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
            if (CG == 2) tma_load_2d_2sm(dst, m, &full[stage], c0, c1);
            else tma_load_2d(dst, m, &full[stage], c0, c1);
          };
          if (!p.a_mn) {
            load(a_dst, &tmA, k, m0);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) load(a_dst + c * 8192, &tmA, m0 + c * 64, k);
          }
          if (!p.b_mn) {
            load(b_dst, &tmB, k, n0);
          } else {
#pragma unroll
            for (int c = 0; c < G::B_ROWS / 64; ++c) load(b_dst + c * 8192, &tmB, n0 + c * 64, k);
          }
          if (++stage == G::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // the whole warp walks the schedule (warp-uniform operands); one elected lane of the leader
    // CTA issues (cta_group::2: one MMA covers both CTAs' rows)
    if (leader) {
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const int a_mn = __shfl_sync(0xffffffffu, p.a_mn, 0), b_mn = __shfl_sync(0xffffffffu, p.b_mn, 0);
      const uint32_t idesc = idesc_bf16_f32(BM * CG, BN, a_mn, b_mn);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int item = cta_id; item < total; item += ncta, ++it) {
        const int sp = item / (p.num_n * p.num_m);
        const int kb0 = sp * p.kb_per_split, kb1 = min(p.num_kb, kb0 + p.kb_per_split);
        const int buf = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[buf], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tm + buf * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * G::B_BYTES);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = a_mn ? desc_sw128(a_base + k * 2048, 8192, 1024)
                                       : desc_sw128(a_base + k * 32, 16, 1024);
              const uint64_t bd = b_mn ? desc_sw128(b_base + k * 2048, 8192, 1024)
                                       : desc_sw128(b_base + k * 32, 16, 1024);
              if (CG == 2) mma_bf16_ss_2sm(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
              else mma_bf16_ss(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            }
            if (CG == 2) mma_commit_2sm_mc(&empty[stage], 0x3);
            else mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == G::STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) {
          if (CG == 2) mma_commit_2sm_mc(&tfull[buf], 0x3);
          else mma_commit(&tfull[buf]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int q = warp & 3;
    const int hf = ew >> 2;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    uint8_t* stg_base = smem + G::OFF_STG + ew * G::STG_BYTES;
    uint32_t rphase = 0;
    int nchunk = 0;  // chunks staged by this warp (buffer = nchunk & 1)
    int it = 0;
    for (int item = cta_id; item < total; item += ncta, ++it) {
      const int nb = item % p.num_n, rest = item / p.num_n;
      const int mb = rest % p.num_m, sp = rest / p.num_m;
      const int buf = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[buf], acc_phase);
      tc_fence_after();
      const int m0 = mb * BM * CG + rank * BM + q * 32;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        const int col = hf * 128 + c * 64;
        const int n0 = nb * BN + col;
        uint32_t r0[32], r1[32];
        tmem_ld32(tmem + buf * BN + col + lane_off, r0);
        tmem_ld32(tmem + buf * BN + col + 32 + lane_off, r1);
        tmem_ld_wait();
        if (c == 1) {
          tc_fence_before();
          if (CG == 2 && !leader) mbar_arrive_cluster(&tempty[buf], 0);
          else mbar_arrive(&tempty[buf]);
        }
        if (n0 >= p.N || m0 >= p.M) continue;  // warp-uniform
        float v[64];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          v[e] = __uint_as_float(r0[e]);
          v[32 + e] = __uint_as_float(r1[e]);
        }
        if (EPI == EPI_F32) {
          const int m = m0 + lane;
          if (m < p.M) {
            float* dst;
            bool acc = false;
            if (p.num_splits > 1) {
              dst = p.part + ((int64_t)sp * p.M + m) * p.N + n0;
            } else {
              dst = (float*)p.C + (int64_t)m * p.ldc + n0;
              acc = p.accumulate;
            }
            if (n0 + 64 <= p.N) {
#pragma unroll
              for (int e = 0; e < 64; e += 4) {
                float4 o = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
                if (acc) {
                  const float4 old = *reinterpret_cast<const float4*>(dst + e);
                  o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
                }
                *reinterpret_cast<float4*>(dst + e) = o;
              }
            } else {
#pragma unroll
              for (int e = 0; e < 64; ++e)
                if (n0 + e < p.N) dst[e] = acc ? dst[e] + v[e] : v[e];
            }
          }
          continue;
        }
        if (p.bias) {
          if (n0 + 64 <= p.N) {
            const float4* b4 = reinterpret_cast<const float4*>(p.bias + n0);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float4 b = __ldg(b4 + e);
              v[4 * e] += b.x; v[4 * e + 1] += b.y; v[4 * e + 2] += b.z; v[4 * e + 3] += b.w;
            }
          } else {
#pragma unroll
            for (int e = 0; e < 64; ++e) v[e] += (n0 + e < p.N) ? __ldg(p.bias + n0 + e) : 0.f;
          }
        }
        // the bulk store issued from this buffer two chunks ago must have finished reading it
        uint8_t* stg = stg_base + (G::NBUF == 2 ? (nchunk & 1) : 0) * G::BUF_BYTES;
        uint8_t* srow = stg + lane * 128;
        ++nchunk;
        if (lane == 0) {
          if (G::NBUF == 2) tma_store_wait_read<1>();
          else tma_store_wait_read<0>();
        }
        __syncwarp();
        if (EPI == EPI_RESID) {
          if (lane == 0) {
            mbar_expect_tx(&rbar[ew], 32 * 128);
            tma_load_2d(stg, &tmR, &rbar[ew], n0, m0);
          }
          mbar_wait(&rbar[ew], rphase);
          rphase ^= 1;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 w = *reinterpret_cast<const uint4*>(srow + ((j ^ (lane & 7)) << 4));
            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 f = __bfloat1622float2(h2[k]);
              v[8 * j + 2 * k] += f.x;
              v[8 * j + 2 * k + 1] += f.y;
            }
          }
        }
        if (EPI == EPI_QKVU && p.silu && p.c_dsilu) {
          // C2 = silu(p), C = silu'(p) = sg + silu(p) (1 - sg): one tanh per element for both
          uint8_t* srow2 = srow + 32 * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float a[8], ds[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float x = v[8 * j + k];
              const float sg = fmaf(0.5f, sm100::tanh_approx(0.5f * x), 0.5f);
              a[k] = x * sg;
              ds[k] = fmaf(a[k], 1.0f - sg, sg);
            }
            *reinterpret_cast<uint4*>(srow + ((j ^ (lane & 7)) << 4)) =
                make_uint4(pack_bf16(ds[0], ds[1]), pack_bf16(ds[2], ds[3]), pack_bf16(ds[4], ds[5]), pack_bf16(ds[6], ds[7]));
            *reinterpret_cast<uint4*>(srow2 + ((j ^ (lane & 7)) << 4)) =
                make_uint4(pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]), pack_bf16(a[6], a[7]));
          }
        } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 w = make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                                     pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
          *reinterpret_cast<uint4*>(srow + ((j ^ (lane & 7)) << 4)) = w;
        }
        if (EPI == EPI_QKVU) {
          uint8_t* srow2 = srow + 32 * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float a[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = p.silu ? silu_tanh(v[8 * j + k]) : v[8 * j + k];
            const uint4 w = make_uint4(pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]),
                                       pack_bf16(a[4], a[5]), pack_bf16(a[6], a[7]));
            *reinterpret_cast<uint4*>(srow2 + ((j ^ (lane & 7)) << 4)) = w;
          }
        }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmC, stg, n0, m0);
          if (EPI == EPI_QKVU) tma_store_2d(&tmC2, stg + 32 * 128, n0, m0);
          tma_store_commit();
        }
      }
    }
    if (lane == 0) tma_store_wait<0>();
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_2sm<512>(tmem);
    else tmem_dealloc<512>(tmem);
  }
}

// C (+)= sum over splits of the partials (fixed order: deterministic)
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int splits, int M, int N,
                                     float* __restrict__ C, int64_t ldc, int accumulate) {
  const int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += part[(int64_t)k * total + i];
    const int64_t m = i / N, n = i % N;
    float* c = C + m * ldc + n;
    *c = accumulate ? *c + s : s;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

struct Split {
  int splits, kb_per_split;
};
constexpr int CG_USE = 2;  // the layer GEMMs run on CTA pairs (cta_group::2)

static Split choose_split(int M, int N, int K, int epi) {
  const int num_kb = ceil_div(K, BK);
  const int tiles = ceil_div(M, BM * CG_USE) * ceil_div(N, BN);  // pair tiles
  const int units = num_sms() / CG_USE;
  Split s{1, num_kb};
  if (epi == EPI_F32 && tiles < units && num_kb > 1) {
    // the persistent grid walks tiles x splits work items in rounds of `units` CTA pairs: pick
    // the split count whose item count fills the last round best (fewest splits on ties), from
    // one to four rounds' worth -- e.g. dW1 of `small` (16 tiles): 9 splits = 144 items over 74
    // pairs (97%), where 10 splits left a third round mostly idle
    const int lo = ceil_div(units, tiles);
    double best = -1.0;
    for (int want = lo; want <= 4 * lo && want <= num_kb; ++want) {
      const int kbs = ceil_div(num_kb, want);
      const int sp = ceil_div(num_kb, kbs);
      const int items = tiles * sp;
      const double eff = (double)items / ((double)units * ceil_div(items, units));
      if (eff > best + 1e-9) {
        best = eff;
        s.kb_per_split = kbs;
        s.splits = sp;
      }
    }
  }
  return s;
}

}  // namespace tcg

mtgr_status_t make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                             uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer) {
  auto fn = tcg::encode_fn();
  if (!fn) return set_error(MTGR_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(MTGR_E_CUDA, "cuTensorMapEncodeTiled failed (%d): inner %llu outer %llu ld %llu",
                     (int)r, (unsigned long long)inner, (unsigned long long)outer,
                     (unsigned long long)ld_elems);
  return MTGR_OK;
}

size_t gemm_ws_bytes(int M, int N, int K, int epi, bool bf16) {
  if (!bf16 || epi != EPI_F32) return 0;
  tcg::Split s = tcg::choose_split(M, N, K, epi);
  return s.splits > 1 ? align_up((size_t)s.splits * M * N * sizeof(float), 256) : 0;
}

mtgr_status_t gemm_bf16_launch(const GemmIO& g, int epi, void* ws, size_t ws_bytes,
                               cudaStream_t st) {
  using namespace tcg;
  if (g.M == 0 || g.N == 0) return MTGR_OK;
  if (g.K == 0) return gemm_simt_launch<__nv_bfloat16>(g, epi, st);  // bias / zero only
  MTGR_CHECK(g.lda % 8 == 0 && g.ldb % 8 == 0 && aligned16(g.A) && aligned16(g.B), MTGR_E_LAYOUT,
             "tc gemm: operands need 16-byte aligned rows (ld %% 8 == 0)");
  MTGR_CHECK(g.ldc % 8 == 0 && aligned16(g.C) && (!g.C2 || aligned16(g.C2)) &&
                 (!g.R || (g.ldr % 8 == 0 && aligned16(g.R))) && (!g.bias || aligned16(g.bias)),
             MTGR_E_LAYOUT, "tc gemm: outputs need 16-byte aligned rows");
  constexpr int CG = CG_USE;
  using Gm = Geo<CG, EPI_QKVU>;  // the largest footprint
  CUtensorMap ta, tb;
  if (g.a_kmajor) MTGR_TRY(make_tmap_bf16(&ta, g.A, g.K, g.M, g.lda, 64, BM));
  else MTGR_TRY(make_tmap_bf16(&ta, g.A, g.M, g.K, g.lda, 64, 64));
  if (g.b_kmajor) MTGR_TRY(make_tmap_bf16(&tb, g.B, g.K, g.N, g.ldb, 64, Gm::B_ROWS));
  else MTGR_TRY(make_tmap_bf16(&tb, g.B, g.N, g.K, g.ldb, 64, 64));
  CUtensorMap tc = ta, tc2 = ta, tr = ta;
  if (epi != EPI_F32) MTGR_TRY(make_tmap_bf16(&tc, g.C, g.N, g.M, g.ldc, 64, 32));
  if (epi == EPI_QKVU) MTGR_TRY(make_tmap_bf16(&tc2, g.C2, g.N, g.M, g.ldc, 64, 32));
  if (epi == EPI_RESID) MTGR_TRY(make_tmap_bf16(&tr, g.R, g.N, g.M, g.ldr, 64, 32));
  Params p{};
  p.M = g.M; p.N = g.N; p.K = g.K;
  p.num_m = ceil_div(g.M, BM * CG); p.num_n = ceil_div(g.N, BN); p.num_kb = ceil_div(g.K, BK);
  Split s = choose_split(g.M, g.N, g.K, epi);
  p.num_splits = s.splits; p.kb_per_split = s.kb_per_split;
  p.a_mn = g.a_kmajor ? 0 : 1; p.b_mn = g.b_kmajor ? 0 : 1;
  p.C = g.C; p.ldc = g.ldc; p.bias = g.bias;
  p.accumulate = g.accumulate; p.silu = g.silu; p.c_dsilu = g.c_dsilu;
  if (epi == EPI_F32 && s.splits > 1) {
    MTGR_CHECK(ws && ws_bytes >= gemm_ws_bytes(g.M, g.N, g.K, epi, true), MTGR_E_WORKSPACE,
               "tc gemm: split-K workspace too small");
    p.part = (float*)ws;
  }
  const int total = p.num_m * p.num_n * p.num_splits;
  const int grid = CG * std::min(total, num_sms() / CG);
  ProfScope ps(epi == EPI_QKVU ? PROF_GEMM_QKVU : epi == EPI_RESID ? PROF_GEMM_OUT
               : epi == EPI_STORE ? PROF_GEMM_DGRAD : PROF_GEMM_WGRAD, st);
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Gm::SMEM_BYTES);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = Gm::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, tc2, tr, p);
  };
  switch (epi) {
    case EPI_STORE: launch(gemm_tc_kernel<EPI_STORE, CG>); break;
    case EPI_QKVU: launch(gemm_tc_kernel<EPI_QKVU, CG>); break;
    case EPI_RESID: launch(gemm_tc_kernel<EPI_RESID, CG>); break;
    default: launch(gemm_tc_kernel<EPI_F32, CG>); break;
  }
  MTGR_TRY(check_launch("gemm_tc"));
  if (epi == EPI_F32 && s.splits > 1) {
    const int64_t tot = (int64_t)g.M * g.N;
    const int blocks = (int)std::min<int64_t>(ceil_div64(tot, 256), 8 * num_sms());
    splitk_reduce_kernel<<<blocks, 256, 0, st>>>(p.part, s.splits, g.M, g.N, (float*)g.C, g.ldc,
                                                 g.accumulate);
    MTGR_TRY(check_launch("splitk_reduce"));
  }
  return MTGR_OK;
}

}  // namespace mtgr
