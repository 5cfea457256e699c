// Microbenchmark: issue rate / throughput of tcgen05.mma kind::f16 (M=128, K=16) for SS and
// TS (A from TMEM) operands and several N, one CTA per SM.  Prints cycles per instruction.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2505_18654_b200/csrc/sm100.cuh"
using namespace mtgr::sm100;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) bench(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = __shfl_sync(0xffffffffu, slot, 0);
  if (threadIdx.x < 32) {
    const uint32_t a = smem_u32(base), b = smem_u32(base + 32 * 1024);
    constexpr uint32_t idesc = idesc_bf16_f32(128, N, 0, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          if (TS) mma_bf16_ts(tm + 256, tm + 0 + (k & 7) * 8, desc_sw128(b + (k & 3) * 32, 16, 1024), idesc, 1);
          else mma_bf16_ss(tm + 256, desc_sw128(a + (k & 3) * 32, 16, 1024), desc_sw128(b + (k & 3) * 32, 16, 1024), idesc, 1);
        }
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tm);
}

template <int N, bool TS>
void run(const char* name, int grid) {
  long long* d; cudaMalloc(&d, grid * sizeof(long long));
  int iters = 200;
  cudaFuncSetAttribute(bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  bench<N, TS><<<grid, 128, 66 * 1024>>>(d, 10);
  bench<N, TS><<<grid, 128, 66 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  double per = mx / (iters * 16.0);
  double ideal = 128.0 * N / 256.0;
  printf("%-10s grid %3d: %7.1f cycles/instr (ideal %5.1f, %5.1f%%) %s\n", name, grid, per, ideal, 100 * ideal / per, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int g : {1, 148}) {
    run<64, false>("SS N=64", g);
    run<128, false>("SS N=128", g);
    run<256, false>("SS N=256", g);
    run<64, true>("TS N=64", g);
    run<128, true>("TS N=128", g);
    run<256, true>("TS N=256", g);
  }
  return 0;
}
