// lds_probe.cu -- shared-memory load throughput for the access shapes used by the kernels.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 256;
template <int MODE>
__global__ void k(float* out, long long* cyc) {
  __shared__ __align__(16) float sm[4096];
  const int t = threadIdx.x, l = t & 31;
  for (int i = t; i < 4096; i += blockDim.x) sm[i] = i * 1e-3f;
  __syncthreads();
  float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  long long c0 = clock64();
#pragma unroll 1
  for (int it = 0; it < N; ++it) {
    const int base = (it & 7) * 64;
#pragma unroll
    for (int q = 0; q < 64; q += 4) {
      float4 x;
      if (MODE == 0) x = *reinterpret_cast<const float4*>(&sm[base + q]);                      // broadcast LDS.128
      if (MODE == 1) x = *reinterpret_cast<const float4*>(&sm[base + q + 4 * (l & 7) * 0 + 256 * (l & 3)]);  // 4 distinct, same banks
      if (MODE == 2) x = *reinterpret_cast<const float4*>(&sm[(base + q + 68 * (l & 3)) & 4095]); // 4 distinct, padded
      if (MODE == 3) { x.x = sm[base + q]; x.y = sm[base + q + 1]; x.z = sm[base + q + 2]; x.w = sm[base + q + 3]; }  // LDS.32 broadcast
      if (MODE == 4) x = *reinterpret_cast<const float4*>(&sm[(base * 4 + 4 * l + q * 32) & 4095]); // 32 distinct consecutive
      a0 += x.x; a1 += x.y; a2 += x.z; a3 += x.w;
    }
  }
  long long c1 = clock64();
  if (t == 0) cyc[0] = c1 - c0;
  out[t] = a0 + a1 + a2 + a3;
}
template <int M>
void run(const char* name, int th, float* o, long long* c) {
  k<M><<<1, th>>>(o, c); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double loads = (double)N * 16 * (th / 32);
  printf("%-36s warps=%2d  cycles per warp-LDS.128 (SM-wide) = %.2f\n", name, th / 32, (double)h / loads);
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 1 << 16); cudaMalloc(&c, 8);
  for (int th : {128, 256}) {
    run<0>("LDS.128 broadcast", th, o, c);
    run<1>("LDS.128 4 addrs, same banks", th, o, c);
    run<2>("LDS.128 4 addrs, padded", th, o, c);
    run<3>("4x LDS.32 broadcast", th, o, c);
    run<4>("LDS.128 32 consecutive", th, o, c);
  }
}
