// tput_probe.cu -- FFMA issue throughput per SM (3-register form, weights in registers).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void k(const float* __restrict__ in, float* out, long long* cyc) {
  float w[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) w[i] = in[i * blockDim.x + threadIdx.x];
  float x0 = in[threadIdx.x] + 1.f, x1 = x0 * 0.5f;
  float a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0, a7 = 0;
  __syncthreads();
  long long c0 = clock64();
  for (int it = 0; it < N; ++it) {
#pragma unroll
    for (int q = 0; q < 32; q += 8) {
      a0 = fmaf(w[q], x0, a0); a1 = fmaf(w[q + 1], x1, a1); a2 = fmaf(w[q + 2], x0, a2); a3 = fmaf(w[q + 3], x1, a3);
      a4 = fmaf(w[q + 4], x0, a4); a5 = fmaf(w[q + 5], x1, a5); a6 = fmaf(w[q + 6], x0, a6); a7 = fmaf(w[q + 7], x1, a7);
    }
    x0 += 1e-7f;
  }
  long long c1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  float *in, *out; long long* cyc;
  cudaMalloc(&in, 1 << 20); cudaMalloc(&out, 1 << 16); cudaMalloc(&cyc, 8);
  cudaMemset(in, 0, 1 << 20);
  for (int th : {128, 256, 512, 1024}) {
    k<<<1, th>>>(in, out, cyc); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double ffma = (double)N * 32 * th;
    printf("threads=%d  FFMA/cycle/SM = %.1f\n", th, ffma / h);
  }
}
