// tmem_bw_probe.cu -- TMEM -> register bandwidth when several warps per SM sub-partition load
// at once (the cluster kernel's A, B, C warpgroups each pull a weight tile every layer).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bw_probe tools/tmem_bw_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// every warp: `iters` times { load NC columns of its lane quarter; wait }.
template <int NC>
__global__ void __launch_bounds__(512, 1) bw(float* out, long long* cyc, int iters, int active_warps) {
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t my = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  float acc = 0.f;
  __syncthreads();
  long long c0 = clock64();
  if (warp < active_warps) {
    uint32_t r[NC];
    for (int it = 0; it < iters; ++it) {
      const uint32_t col = (uint32_t)((warp >> 2) * 128 + (it & 1) * 64) & 511u;
#pragma unroll
      for (int i = 0; i < NC; i += 16) ld16(my + col + i, r + i);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += __uint_as_float(r[0]) + __uint_as_float(r[NC - 1]);
    }
  }
  __syncthreads();
  long long c1 = clock64();
  if (t == 0) cyc[0] = c1 - c0;
  out[t] = acc;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  float* o;
  long long* c;
  cudaMalloc(&o, 512 * 4);
  cudaMalloc(&c, 16);
  const int iters = 2000;
  for (int aw : {1, 4, 8, 12, 16}) {
    long long h = 0;
    bw<64><<<1, 512>>>(o, c, iters, aw);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / iters;
    const double bytes = (double)aw * 32 * 64 * 4;  // per iteration, all warps
    printf("x64 active warps %2d: %7.1f cycles/iter  -> %6.1f B/cycle per SM (%s)\n", aw, per, bytes / per,
           cudaGetErrorString(e));
  }
  for (int aw : {1, 4, 12}) {
    long long h = 0;
    bw<32><<<1, 512>>>(o, c, iters, aw);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / iters;
    printf("x32 active warps %2d: %7.1f cycles/iter  -> %6.1f B/cycle per SM\n", aw, per, aw * 32 * 32 * 4 / per);
  }
  return 0;
}
