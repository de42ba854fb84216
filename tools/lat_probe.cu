// lat_probe.cu -- dependent-chain latencies (cycles) of the primitives on the batch-1 critical path.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1702_07825_b200/csrc/ptx.cuh"
using namespace dvw;
constexpr int N = 1024;

__global__ void k(float* out, long long* cyc, int nwarps_bar) {
  __shared__ __align__(16) float sm[1024];
  const int t = threadIdx.x;
  for (int i = t; i < 1024; i += blockDim.x) sm[i] = (i * 7 % 1024) * 1.0f;
  __syncthreads();
  float v = t * 1e-3f;
  long long c0, c1;
  // 1 FFMA chain
  c0 = clock64(); for (int i = 0; i < N; ++i) v = fmaf(v, 1.0000001f, 1e-7f); c1 = clock64(); if (t == 0) cyc[0] = c1 - c0;
  // 2 SHFL chain
  c0 = clock64(); for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1); c1 = clock64(); if (t == 0) cyc[1] = c1 - c0;
  // 3 SHFL+FADD chain (reduction step)
  c0 = clock64(); for (int i = 0; i < N; ++i) v += __shfl_xor_sync(0xffffffffu, v, 1); c1 = clock64(); if (t == 0) cyc[2] = c1 - c0;
  // 4 LDS chain (pointer chase)
  int idx = t & 1023;
  c0 = clock64(); for (int i = 0; i < N; ++i) idx = (int)sm[idx]; c1 = clock64(); if (t == 0) cyc[3] = c1 - c0;
  v += idx;
  // 5 MUFU ex2 chain
  c0 = clock64(); for (int i = 0; i < N; ++i) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v)); v = r * 1e-30f; } c1 = clock64(); if (t == 0) cyc[4] = c1 - c0;
  // 6 accurate tanhf chain
  c0 = clock64(); for (int i = 0; i < N; ++i) v = tanhf(v + 0.3f); c1 = clock64(); if (t == 0) cyc[5] = c1 - c0;
  // 7 accurate expf + IEEE div chain (sigmoid)
  c0 = clock64(); for (int i = 0; i < N; ++i) v = 1.0f / (1.0f + expf(-v)); c1 = clock64(); if (t == 0) cyc[6] = c1 - c0;
  // 8 bar.sync among all threads, STS -> BAR -> LDS round trip
  c0 = clock64();
  for (int i = 0; i < N; ++i) {
    if ((t & 31) == 0) sm[(t >> 5) + 32 * (i & 1)] = v;
    asm volatile("bar.sync 1, %0;" :: "r"((int)blockDim.x) : "memory");
    v = sm[((t >> 5) + 1) % (blockDim.x >> 5) + 32 * (i & 1)] * 0.5f;
  }
  c1 = clock64(); if (t == 0) cyc[7] = c1 - c0;
  // 9 bare bar.sync
  c0 = clock64(); for (int i = 0; i < N; ++i) asm volatile("bar.sync 1, %0;" :: "r"((int)blockDim.x) : "memory"); c1 = clock64(); if (t == 0) cyc[8] = c1 - c0;
  // 10 tanh.approx chain
  c0 = clock64(); for (int i = 0; i < N; ++i) { float r; asm volatile("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(v)); v = r + 0.1f; } c1 = clock64(); if (t == 0) cyc[9] = c1 - c0;
  // 11 rcp.approx chain
  c0 = clock64(); for (int i = 0; i < N; ++i) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v)); v = r + 1.0f; } c1 = clock64(); if (t == 0) cyc[10] = c1 - c0;
  out[t] = v;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 4096 * 4); cudaMalloc(&cyc, 16 * 8);
  const char* names[] = {"FFMA", "SHFL", "SHFL+FADD", "LDS chase", "MUFU.EX2+FMUL", "tanhf(+FADD)", "sigmoid expf+div", "STS-BAR-LDS", "BAR.SYNC", "tanh.approx+FADD", "rcp.approx+FADD"};
  for (int th : {32, 256, 384}) {
    k<<<1, th>>>(out, cyc, th / 32);
    cudaDeviceSynchronize();
    long long h[16]; cudaMemcpy(h, cyc, 11 * 8, cudaMemcpyDeviceToHost);
    printf("threads=%d:", th);
    for (int i = 0; i < 11; ++i) printf("  %s=%.1f", names[i], (double)h[i] / N);
    printf("\n");
  }
  return 0;
}
