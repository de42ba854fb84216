// layer_probe.cu -- cycles per chain layer on one SM, no cluster traffic.
// Variants: aux warps (a) exit immediately, (b) spin on an mbarrier that never
// completes (as in the cluster kernel between samples), (c) nanosleep-poll it.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1702_07825_b200/csrc/dvw_internal.cuh"
#include "../paper_1702_07825_b200/csrc/ptx.cuh"
using namespace dvw;

constexpr int R = 64, LPC = 4, kMain = 256, kThreads = 384;

template <int AUX, int GATE, int FL>
__global__ void __launch_bounds__(kThreads, 1) probe(const float* wts, int iters, float* out, long long* cyc) {
  long long ph_acc[6] = {0, 0, 0, 0, 0, 0};
  long long tp = 0;
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
      if (FL & 4) tp = clock64();
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
      if (!(FL & 1)) {
        ah += __shfl_xor_sync(0xffffffffu, ah, 1);
        ag += __shfl_xor_sync(0xffffffffu, ag, 1);
        ah += __shfl_xor_sync(0xffffffffu, ah, 2);
        ag += __shfl_xor_sync(0xffffffffu, ag, 2);
      }
      float hv;
      if (GATE == 1) {
        float e2, eg, r1, r2;
        const float a1 = 2.8853900817779268f * (ah + ph), a2 = -1.4426950408889634f * (ag + pg);
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e2) : "f"(a1));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(eg) : "f"(a2));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(e2 + 1.0f));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(eg + 1.0f));
        hv = fmaf(-2.0f, r1, 1.0f) * r2;
      } else if (GATE == 2) {
        hv = (ah + ph) * (ag + pg);
      } else {
        hv = gate(ah + ph, ag + pg);
      }
      if (FL & 4) { long long c = clock64(); ph_acc[0] += c - tp; tp = c; }
      if (ch == 0) hs[pr] = hv;
      ptx::bar_sync(1, kMain);
      if (FL & 4) { long long c = clock64(); ph_acc[1] += c - tp; tp = c; }
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
      if (!(FL & 1)) {
        rr += __shfl_xor_sync(0xffffffffu, rr, 1);
        rr += __shfl_xor_sync(0xffffffffu, rr, 2);
      }
      const float xn = xi + rr * 0.5f;
      if (FL & 4) { long long c = clock64(); ph_acc[2] += c - tp; tp = c; }
      if (ch == 0) xs[jl + 1][pr] = xn;
      if (!(FL & 2)) ptx::bar_sync(1, kMain);
      if (FL & 4) { long long c = clock64(); ph_acc[3] += c - tp; tp = c; }
    }
    if (t < R) xs[0][t] = xs[LPC][t] * 0.5f;
    ptx::bar_sync(1, kMain);
  }
  long long t1 = clock64();
  if (t == 0) { cyc[0] = t1 - t0; stop = 1; for (int i = 0; i < 4; ++i) cyc[1 + i] = ph_acc[i]; }
  if (t < R) out[t] = xs[0][t];
}

template <int AUX, int G, int FL>
void run(const char* name, const float* w, float* out, long long* cyc) {
  const int iters = 2000;
  probe<AUX, G, FL><<<1, kThreads>>>(w, iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[5] = {0}; cudaMemcpy(h, cyc, 40, cudaMemcpyDeviceToHost);
  const double L = (double)iters * LPC;
  printf("%-28s err=%s cycles/layer=%.1f  phases: gemv1+gate=%.0f bar1=%.0f gemv2=%.0f bar2=%.0f\n", name, cudaGetErrorString(e), (double)h[0] / L, h[1] / L, h[2] / L, h[3] / L, h[4] / L);
}

int main() {
  float *w, *out; long long* cyc;
  cudaMalloc(&w, sizeof(float) * LPC * 48 * kMain); cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  cudaMemset(w, 0, sizeof(float) * LPC * 48 * kMain);
  run<0, 0, 4>("accurate gate, phase clocks", w, out, cyc);
  run<0, 1, 4>("mufu gate, phase clocks", w, out, cyc);
  run<0, 0, 0>("accurate gate (baseline)", w, out, cyc);
  run<0, 1, 0>("mufu gate", w, out, cyc);
  run<0, 2, 0>("no gate", w, out, cyc);
  run<0, 0, 1>("accurate, no shuffles", w, out, cyc);
  run<0, 0, 2>("accurate, no 2nd barrier", w, out, cyc);
  run<0, 2, 3>("no gate/shfl/2nd bar", w, out, cyc);
  run<1, 1, 0>("mufu gate, aux spin", w, out, cyc);
  return 0;
}
