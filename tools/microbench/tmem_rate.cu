// TMEM read (tcgen05.ld) throughput per SM on B200: one CTA per SM, NW warps (NW/4 per lane
// quadrant) each reading its share of the 512 allocated columns with .32x32b.xN loads, N = 16,
// 32 or 64 columns per instruction; two loads in flight per wait.  Reports bytes per cycle per SM.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2505_18654_b200/csrc/sm100.cuh"

using namespace mtgr::sm100;

template <int N>
__device__ __forceinline__ void ldN(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ldN<16>(uint32_t t, uint32_t* r) { tmem_ld16(t, *reinterpret_cast<uint32_t(*)[16]>(r)); }
template <>
__device__ __forceinline__ void ldN<32>(uint32_t t, uint32_t* r) { tmem_ld32(t, *reinterpret_cast<uint32_t(*)[32]>(r)); }
template <>
__device__ __forceinline__ void ldN<64>(uint32_t t, uint32_t* r) {
  tmem_ld32(t, *reinterpret_cast<uint32_t(*)[32]>(r));
  tmem_ld32(t + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
}

// one tcgen05.ld of 64 columns
__device__ __forceinline__ void ld64(uint32_t t, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(t));
}

// W = width per instruction (16, 32, 64), K = loads in flight per wait
template <int W, int K, int NW>
__global__ void __launch_bounds__(32 * NW, 1) k(int iters, long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  const int q = warp & 3, part = warp >> 2, nparts = NW / 4;
  const int cols = 512 / nparts;
  const uint32_t base = tm + ((uint32_t)(q * 32) << 16) + part * cols;
  uint32_t r[K][W];
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int c = 0; c < cols; c += K * W) {
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (W == 16) tmem_ld16(base + c + j * W, *reinterpret_cast<uint32_t(*)[16]>(r[j]));
        else if (W == 32) tmem_ld32(base + c + j * W, *reinterpret_cast<uint32_t(*)[32]>(r[j]));
        else ld64(base + c + j * W, r[j]);
      }
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < K; ++j) acc += r[j][0] ^ r[j][W - 1] ^ r[j][W / 2];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

template <int W, int K, int NW>
void run(long long* cyc, uint32_t* sink) {
  const int iters = 200;
  k<W, K, NW><<<148, 32 * NW>>>(iters, cyc, sink);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double bytes = 128.0 * 512 * 4 * iters;
  printf("x%-3d in-flight %d warps %2d: %.1f B/clk/SM (%s)\n", W, K, NW, bytes / avg, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* cyc; uint32_t* sink;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaMalloc(&sink, 148 * 1024 * sizeof(uint32_t));
  for (int rep = 0; rep < 2; ++rep) {
    run<16, 1, 8>(cyc, sink); run<16, 2, 8>(cyc, sink); run<16, 8, 8>(cyc, sink);
    run<32, 1, 8>(cyc, sink); run<32, 2, 8>(cyc, sink); run<32, 4, 8>(cyc, sink);
    run<64, 1, 8>(cyc, sink); run<64, 2, 8>(cyc, sink);
  }
  return 0;
}
