// layer_probe.cu -- cycles per chain layer on one SM, no cluster traffic.
// Variants: aux warps (a) exit immediately, (b) spin on an mbarrier that never
// completes (as in the cluster kernel between samples), (c) nanosleep-poll it.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1702_07825_b200/csrc/dvw_internal.cuh"
#include "../paper_1702_07825_b200/csrc/ptx.cuh"
using namespace dvw;

constexpr int R = 64, LPC = 4, kMain = 256, kThreads = 384;

template <int AUX, bool FASTGATE>
__global__ void __launch_bounds__(kThreads, 1) probe(const float* wts, int iters, float* out, long long* cyc) {
  __shared__ __align__(16) float xs[LPC + 1][R];
  __shared__ __align__(16) float hs[R];
  __shared__ __align__(16) float pre[LPC][2 * R];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int stop;
  const int t = threadIdx.x;
  if (t == 0) { ptx::mbar_init(ptx::smem_u32(&bar), 1); stop = 0; }
  if (t < R) xs[0][t] = 0.01f * t;
  for (int i = t; i < LPC * 2 * R; i += kThreads) (&pre[0][0])[i] = 0.001f * i;
  __syncthreads();
  if (t >= kMain) {
    ptx::setmaxnreg_dec<40>();
    if (AUX == 1) { while (!ptx::mbar_try_wait(ptx::smem_u32(&bar), 0)) { if (*(volatile int*)&stop) break; } }
    if (AUX == 2) { while (!*(volatile int*)&stop) __nanosleep(500); }
    return;
  }
  ptx::setmaxnreg_inc<232>();
  const int pr = t >> 2, ch = t & 3;
  float wc[LPC][32], wr[LPC][16];
#pragma unroll
  for (int jl = 0; jl < LPC; ++jl) {
#pragma unroll
    for (int q = 0; q < 32; ++q) wc[jl][q] = wts[(jl * 48 + q) * kMain + t];
#pragma unroll
    for (int q = 0; q < 16; ++q) wr[jl][q] = wts[(jl * 48 + 32 + q) * kMain + t];
  }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int jl = 0; jl < LPC; ++jl) {
      const float* xin = xs[jl];
      float xv[16];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4 v = *reinterpret_cast<const float4*>(xin + ch * 16 + 4 * k);
        xv[4 * k] = v.x; xv[4 * k + 1] = v.y; xv[4 * k + 2] = v.z; xv[4 * k + 3] = v.w;
      }
      const float ph = pre[jl][pr], pg = pre[jl][R + pr];
      const float xi = xin[pr];
      float h0 = 0.f, h1 = 0.f, g0 = 0.f, g1 = 0.f;
#pragma unroll
      for (int q = 0; q < 16; q += 2) {
        h0 = fmaf(wc[jl][q], xv[q], h0);
        g0 = fmaf(wc[jl][16 + q], xv[q], g0);
        h1 = fmaf(wc[jl][q + 1], xv[q + 1], h1);
        g1 = fmaf(wc[jl][16 + q + 1], xv[q + 1], g1);
      }
      float ah = h0 + h1, ag = g0 + g1;
      ah += __shfl_xor_sync(0xffffffffu, ah, 1);
      ag += __shfl_xor_sync(0xffffffffu, ag, 1);
      ah += __shfl_xor_sync(0xffffffffu, ah, 2);
      ag += __shfl_xor_sync(0xffffffffu, ag, 2);
      float hv;
      if (FASTGATE) {
        const float e2 = exp2f(2.8853900817779268f * (ah + ph));
        const float eg = exp2f(-1.4426950408889634f * (ag + pg));
        hv = (1.0f - 2.0f * __frcp_rn(e2 + 1.0f)) * __frcp_rn(1.0f + eg);
      } else {
        hv = gate(ah + ph, ag + pg);
      }
      if (ch == 0) hs[pr] = hv;
      ptx::bar_sync(1, kMain);
      float hvv[16];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4 v = *reinterpret_cast<const float4*>(hs + ch * 16 + 4 * k);
        hvv[4 * k] = v.x; hvv[4 * k + 1] = v.y; hvv[4 * k + 2] = v.z; hvv[4 * k + 3] = v.w;
      }
      float r0 = 0.f, r1 = 0.f;
#pragma unroll
      for (int q = 0; q < 16; q += 2) {
        r0 = fmaf(wr[jl][q], hvv[q], r0);
        r1 = fmaf(wr[jl][q + 1], hvv[q + 1], r1);
      }
      float rr = r0 + r1;
      rr += __shfl_xor_sync(0xffffffffu, rr, 1);
      rr += __shfl_xor_sync(0xffffffffu, rr, 2);
      const float xn = xi + rr * 0.5f;
      if (ch == 0) xs[jl + 1][pr] = xn;
      ptx::bar_sync(1, kMain);
    }
    if (t < R) xs[0][t] = xs[LPC][t] * 0.5f;
    ptx::bar_sync(1, kMain);
  }
  long long t1 = clock64();
  if (t == 0) { cyc[0] = t1 - t0; stop = 1; }
  if (t < R) out[t] = xs[0][t];
}

template <int AUX, bool FG>
void run(const char* name, const float* w, float* out, long long* cyc) {
  const int iters = 2000;
  probe<AUX, FG><<<1, kThreads>>>(w, iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-28s err=%s cycles/layer=%.1f\n", name, cudaGetErrorString(e), (double)h / iters / LPC);
}

int main() {
  float *w, *out; long long* cyc;
  cudaMalloc(&w, sizeof(float) * LPC * 48 * kMain); cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
  cudaMemset(w, 0, sizeof(float) * LPC * 48 * kMain);
  for (int rep = 0; rep < 2; ++rep) {
    run<0, false>("aux exit, accurate gate", w, out, cyc);
    run<1, false>("aux try_wait spin, accurate", w, out, cyc);
    run<2, false>("aux nanosleep, accurate", w, out, cyc);
    run<0, true>("aux exit, fast gate", w, out, cyc);
    run<1, true>("aux try_wait spin, fast", w, out, cyc);
  }
  return 0;
}
