// layer_probe2.cu -- alternative chain-layer mapping: warpgroup 0 owns W_cur (one full row per
// thread, tanh/sigmoid partner rows 16 lanes apart), warpgroup 1 owns W_res (half rows),
// producer/consumer named barriers (bar.arrive / bar.sync) between them.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1702_07825_b200/csrc/ptx.cuh"
using namespace dvw;
constexpr int R = 64, LPC = 3, kThreads = 384;

__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" :: "r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ float gate_fast(float ah, float ag) {
  float e2, eg, r1, r2;
  const float a1 = 2.8853900817779268f * ah, a2 = -1.4426950408889634f * ag;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e2) : "f"(a1));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(eg) : "f"(a2));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(e2 + 1.0f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(eg + 1.0f));
  return fmaf(-2.0f, r1, 1.0f) * r2;
}

template <int VAR>
__global__ void __launch_bounds__(kThreads, 1) probe(const float* wts, int iters, float* out, long long* cyc) {
  __shared__ __align__(16) float xs[LPC + 1][R];
  __shared__ __align__(16) float hs[LPC][R];
  __shared__ __align__(16) float pre[LPC][2 * R];
  const int t = threadIdx.x;
  if (t < R) xs[0][t] = 0.01f * t;
  for (int i = t; i < LPC * 2 * R; i += kThreads) (&pre[0][0])[i] = 0.001f * i;
  __syncthreads();
  if (t >= 256) { ptx::setmaxnreg_dec<40>(); return; }
  if (t < 128) {
    ptx::setmaxnreg_inc<232>();
    // WG0: W_cur. lane l<16: tanh row 16w+l ; l>=16: sigmoid row 64+16w+l-16
    const int w = t >> 5, l = t & 31;
    const int row = (l < 16) ? (16 * w + l) : (64 + 16 * w + (l - 16));
    const int hi = 16 * w + (l & 15);
    float wc[LPC][64];
#pragma unroll
    for (int jl = 0; jl < LPC; ++jl)
#pragma unroll
      for (int q = 0; q < 64; ++q) wc[jl][q] = wts[(jl * 64 + q) * 128 + t];
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int jl = 0; jl < LPC; ++jl) {
        if (jl > 0 || it > 0) ptx::bar_sync(2, 256);  // x of this layer ready
        const float* xin = xs[jl];
        const float pv = pre[jl][row];
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
        for (int q = 0; q < 64; q += 4) {
          const float4 v = *reinterpret_cast<const float4*>(xin + q);
          a0 = fmaf(wc[jl][q], v.x, a0);
          a1 = fmaf(wc[jl][q + 1], v.y, a1);
          a2 = fmaf(wc[jl][q + 2], v.z, a2);
          a3 = fmaf(wc[jl][q + 3], v.w, a3);
        }
        const float a = ((a0 + a1) + (a2 + a3)) + pv;
        const float other = __shfl_xor_sync(0xffffffffu, a, 16);
        if (l < 16) hs[jl][hi] = (VAR == 1) ? gate_fast(a, other) : (tanhf(a) * (1.0f / (1.0f + expf(-other))));
        bar_arrive(1, 256);  // h of this layer ready
      }
    }
    long long t1 = clock64();
    if (t == 0) cyc[0] = t1 - t0;
  } else {
    ptx::setmaxnreg_inc<232>();
    // WG1: W_res. thread t' : row t'>>1, half t'&1 (32 columns)
    const int tp = t - 128, row = tp >> 1, half = tp & 1;
    float wr[LPC][32];
#pragma unroll
    for (int jl = 0; jl < LPC; ++jl)
#pragma unroll
      for (int q = 0; q < 32; ++q) wr[jl][q] = wts[(3 * 64 + jl * 32 + q) * 128 + tp];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int jl = 0; jl < LPC; ++jl) {
        const float xi = xs[jl][row];
        ptx::bar_sync(1, 256);  // wait h
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int q = 0; q < 32; q += 4) {
          const float4 v = *reinterpret_cast<const float4*>(&hs[jl][32 * half + q]);
          a0 = fmaf(wr[jl][q], v.x, a0);
          a1 = fmaf(wr[jl][q + 1], v.y, a1);
          a0 = fmaf(wr[jl][q + 2], v.z, a0);
          a1 = fmaf(wr[jl][q + 3], v.w, a1);
        }
        float rr = a0 + a1;
        rr += __shfl_xor_sync(0xffffffffu, rr, 1);
        const float xn = xi + rr * 0.5f;
        if (half == 0) {
          if (jl + 1 < LPC) xs[jl + 1][row] = xn;
          else xs[0][row] = xn * 0.5f;
        }
        bar_arrive(2, 256);  // x of next layer ready
      }
    }
  }
  if (t < R) out[t] = xs[0][t];
}

template <int V>
void run(const char* name, const float* w, float* out, long long* cyc) {
  const int iters = 2000;
  probe<V><<<1, kThreads>>>(w, iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-30s err=%s cycles/layer=%.1f\n", name, cudaGetErrorString(e), (double)h / iters / LPC);
}

int main() {
  float *w, *out; long long* cyc;
  cudaMalloc(&w, sizeof(float) * 8 * 64 * 128); cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  cudaMemset(w, 0, sizeof(float) * 8 * 64 * 128);
  run<0>("v2 split WGs, accurate gate", w, out, cyc);
  run<1>("v2 split WGs, mufu gate", w, out, cyc);
  return 0;
}
