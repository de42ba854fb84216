// layer_probe3.cu -- the v3 chain layer (register tiles + transposing reductions) on one SM,
// no cluster traffic: cycles per layer, split into the A phase (W_cur + gate) and B phase.
#include <cstdio>
#include "../paper_1702_07825_b200/csrc/kernel_cluster.cu"
namespace dvw {
namespace {
template <int VAR>
__global__ void __launch_bounds__(kThreads, 1) probe3(const float* wts, int iters, float* out, long long* cyc) {
  __shared__ __align__(16) float xs[LPC + 1][kHLen];
  __shared__ __align__(16) float hs[LPC][kHLen];
  __shared__ __align__(16) float pre[LPC][2 * R];
  const int t = threadIdx.x;
  if (t < kHLen) xs[0][t] = 0.01f * t;
  for (int i = t; i < LPC * 2 * R; i += kThreads) (&pre[0][0])[i] = 0.001f * i;
  __syncthreads();
  if (t < kAux) { ptx::setmaxnreg_dec<kAuxRegs>(); return; }
  ptx::setmaxnreg_inc<kMainRegs>();
  long long accA = 0, accB = 0;
  if (t < kAux + 128) {
    const int a = t - kAux, g = a >> 2, cc = a & 3;
    const int hrow = g + ((cc & 2) ? 32 : 0);
    const bool writer = (cc & 1) == 0;
    float wc[LPC][64];
#pragma unroll
    for (int jl = 0; jl < LPC; ++jl)
#pragma unroll
      for (int q = 0; q < 64; ++q) wc[jl][q] = wts[(jl * 64 + q) * 128 + a];
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int jl = 0; jl < LPC; ++jl) {
        if (jl > 0 || it > 0) ptx::bar_sync(kBarX, kMain);
        long long c0 = clock64();
        const float ph = pre[jl][hrow], pg = pre[jl][R + hrow];
        float v[4];
        tile_dot<4, 16>(wc[jl], &xs[jl][20 * cc], v);
        xpose_level<4>(v, cc, 2);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        v[1] += __shfl_xor_sync(0xffffffffu, v[1], 1);
        const float hv = (VAR == 1) ? (v[0] + ph) * (v[1] + pg) : gate_fast(v[0] + ph, v[1] + pg);
        if (writer) hs[jl][pad16(hrow)] = hv;
        bar_arrive(kBarH, kMain);
        accA += clock64() - c0;
      }
    }
    long long t1 = clock64();
    if (a == 0) { cyc[0] = t1 - t0; cyc[1] = accA; }
  } else {
    const int b = t - kAux - 128, g = b >> 2, cc = b & 3;
    const int row = g + ((cc & 2) ? 32 : 0);
    const bool writer = (cc & 1) == 0;
    float wr[LPC][32];
#pragma unroll
    for (int jl = 0; jl < LPC; ++jl)
#pragma unroll
      for (int q = 0; q < 32; ++q) wr[jl][q] = wts[(LPC * 64 + jl * 32 + q) * 128 + b];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int jl = 0; jl < LPC; ++jl) {
        ptx::bar_sync(kBarH, kMain);
        long long c0 = clock64();
        const float xi = xs[jl][pad16(row)];
        float v[2];
        tile_dot<2, 16>(wr[jl], &hs[jl][20 * cc], v);
        xpose_level<2>(v, cc, 2);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        const float xn = xi + v[0] * 0.5f;
        if (writer) xs[(jl + 1) % (LPC + 1) == LPC ? 0 : jl + 1][pad16(row)] = xn * 0.9f;
        accB += clock64() - c0;
        bar_arrive(kBarX, kMain);
      }
    }
    if (b == 0) cyc[2] = accB;
  }
  if (t == kAux) out[0] = xs[0][1];
}
}  // namespace
}  // namespace dvw

int main() {
  float *w, *out; long long* cyc;
  cudaMalloc(&w, sizeof(float) * 8 * 64 * 128); cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  cudaMemset(w, 0, sizeof(float) * 8 * 64 * 128);
  const int iters = 2000;
  for (int v = 0; v < 2; ++v) {
    if (v == 0) dvw::probe3<0><<<1, dvw::kThreads>>>(w, iters, out, cyc);
    else dvw::probe3<1><<<1, dvw::kThreads>>>(w, iters, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[3]; cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
    const double L = (double)iters * dvw::LPC;
    printf("%s err=%s cycles/layer=%.1f  A-phase=%.1f  B-phase=%.1f\n", v ? "no gate  " : "mufu gate",
           cudaGetErrorString(e), h[0] / L, h[1] / L, h[2] / L);
  }
  return 0;
}
