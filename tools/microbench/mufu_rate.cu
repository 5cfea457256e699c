// MUFU.TANH / MUFU.EX2 throughput per SM on B200: 4 blocks x 256 threads on one SM-resident
// grid (148 blocks per kernel -> one per SM), 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters, long long* cyc) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = 0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(v[i]));
      else if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      else asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(v[i]));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  for (int threads : {256, 512, 1024}) {
    for (int op = 0; op < 3; ++op) {
      auto f = op == 0 ? k<0> : op == 1 ? k<1> : k<2>;
      f<<<148, threads>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double ops = (double)threads * iters * 8;
      printf("threads %4d op %s: %.2f lane-ops/clk/SM\n", threads, op == 0 ? "tanh" : op == 1 ? "ex2 " : "ffma",
             ops / (double)h[0]);
    }
  }
  return 0;
}
