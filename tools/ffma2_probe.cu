// ffma2_probe.cu -- issue rate of FFMA vs FFMA2 (fma.rn.f32x2) per SMSP on sm_100a.
// One CTA of W warps on one SM; each thread runs 8 independent accumulator chains for
// ITER iterations; clock64 around the loop.  Prints cycles per warp-instruction per SMSP.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITER = 4096;
template <bool PAIR>
__global__ void k(float* out, long long* cyc, float a0, float b0) {
  float2 acc[8];
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(threadIdx.x + i, i);
  const float2 a = make_float2(a0, a0 + 1.f), b = make_float2(b0, b0 - 1.f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (PAIR) {
        acc[i] = __ffma2_rn(a, b, acc[i]);
      } else {
        acc[i].x = fmaf(a.x, b.x, acc[i].x);
        acc[i].y = fmaf(a.y, b.y, acc[i].y);
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 4096 * 4); cudaMalloc(&cyc, 64);
  for (int warps : {1, 2, 4, 8, 16}) {
    for (int pair = 0; pair < 2; ++pair) {
      long long c = 0;
      for (int rep = 0; rep < 3; ++rep) {
        if (pair) k<true><<<1, 32 * warps>>>(out, cyc, 1.0001f, 0.9999f);
        else k<false><<<1, 32 * warps>>>(out, cyc, 1.0001f, 0.9999f);
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      }
      const double fma_per_thread = 16.0 * ITER;  // scalar FMAs per thread
      const int wps = warps < 4 ? 1 : warps / 4;  // warps per SMSP
      const double instr = (pair ? 8.0 : 16.0) * ITER * wps;
      printf("warps=%2d %s: %lld cycles, %.2f cycles/warp-instr/SMSP, %.1f FMA/clk/SM\n", warps,
             pair ? "FFMA2" : "FFMA ", c, c / instr, fma_per_thread * 32 * warps / c);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
