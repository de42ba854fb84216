// sampler_probe.cu -- cycles of the one-warp inverse-CDF sampler (sample_warp) and of its pieces.
#include <cstdio>
#include "../paper_1702_07825_b200/csrc/kernel_cluster.cu"
namespace dvw {
namespace {
__global__ void sp(float* out, long long* cyc, int iters) {
  __shared__ __align__(16) float lg[256];
  const int lane = threadIdx.x;
  for (int i = lane; i < 256; i += 32) lg[i] = 0.01f * ((i * 37) % 101);
  __syncwarp();
  int acc = 0;
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float u = (it % 997) / 997.0f;
    acc += sample_warp(lg, u, lane);
    lg[it & 255] += 1e-3f;
    __syncwarp();
  }
  long long c1 = clock64();
  // fp64 dependent add chain
  double d = lane;
  long long c2 = clock64();
  for (int it = 0; it < 1024; ++it) d = d + 1.000001;
  long long c3 = clock64();
  if (lane == 0) { cyc[0] = c1 - c0; cyc[1] = c3 - c2; }
  out[lane] = acc + (float)d;
}
}  // namespace
}  // namespace dvw
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 16);
  dvw::sp<<<1, 32>>>(o, c, 1000); cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("sample_warp: %.1f cycles/call   DADD latency: %.1f cycles\n", h[0] / 1000.0, h[1] / 1024.0);
}
