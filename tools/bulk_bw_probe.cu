// bulk_bw_probe.cu -- L2 -> shared-memory ingress of one SM through a ring of cp.async.bulk
// stages (the batched kernel's staging pattern), vs stage size, ring depth and active SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulk_bw_probe tools/bulk_bw_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory");
}
__device__ __forceinline__ void arm(uint32_t b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(tx) : "memory");
}
__device__ __forceinline__ bool test_wait(uint32_t b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok)
               : "r"(b), "r"(par)
               : "memory");
  return ok;
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// lane 0 of warps 0..np-1 produce (stage st is produced by warp st % np, split into `pieces`
// copies), thread 32*np consumes (waits full, marks the stage free by a plain flag)
__global__ void __launch_bounds__(288, 1) probe(const char* src, size_t src_bytes, int stage_bytes, int stages,
                                                int chunks, long long* cyc, int np, int pieces) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  volatile int* freed = reinterpret_cast<volatile int*>(sm + 64);
  unsigned char* buf = sm + 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(smem_u32(&full[s]), 1);
    freed[0] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long t0 = clock64();
  const size_t per = (size_t)stage_bytes;
  const size_t off0 = ((size_t)blockIdx.x * 7919 * per) % (src_bytes - per);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && w < np) {
    for (int c = w; c < chunks; c += np) {
      const int st = c % stages;
      while (c - freed[0] >= stages) {
      }
      const uint32_t b = smem_u32(&full[st]);
      arm(b, stage_bytes);
      const size_t off = ((off0 + (size_t)c * per) % (src_bytes - per)) & ~size_t(15);
      const int pb = stage_bytes / pieces;
      for (int q = 0; q < pieces; ++q)
        bulk(smem_u32(buf + (size_t)st * per + q * pb), src + off + q * pb, pb, b);
    }
  } else if (threadIdx.x == 32 * np) {
    for (int c = 0; c < chunks; ++c) {
      const int st = c % stages;
      while (!test_wait(smem_u32(&full[st]), (c / stages) & 1)) {
      }
      freed[0] = c + 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  const size_t src_bytes = 32u << 20;  // L2-resident
  char* src;
  long long* cyc;
  cudaMalloc(&src, src_bytes);
  cudaMemset(src, 1, src_bytes);
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ghz = 1.965;
  struct Cfg { int bytes, stages, ctas, np, pieces; };
  const Cfg cfgs[] = {{49152, 4, 1, 1, 1},  {49152, 4, 1, 1, 3},  {49152, 4, 1, 4, 1},  {49152, 4, 1, 4, 3},
                      {16384, 8, 1, 8, 1},  {16384, 8, 1, 1, 1},  {49152, 4, 32, 4, 1}, {49152, 4, 32, 4, 3},
                      {49152, 4, 1, 1, 12}, {49152, 4, 1, 4, 12}, {8192, 16, 1, 8, 1}, {8192, 24, 1, 8, 1}};
  for (const Cfg& c : cfgs) {
    const int chunks = 400;
    probe<<<c.ctas, 288, 128 + c.bytes * c.stages>>>(src, src_bytes, c.bytes, c.stages, chunks, cyc, c.np, c.pieces);
    probe<<<c.ctas, 288, 128 + c.bytes * c.stages>>>(src, src_bytes, c.bytes, c.stages, chunks, cyc, c.np, c.pieces);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, c.ctas * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < c.ctas; ++i) mx = h[i] > mx ? h[i] : mx;
    const double us = mx / (ghz * 1e3);
    const double gbs = (double)c.bytes * chunks / (us * 1e-6) / 1e9;
    printf("stage %6d B x %2d stages, %3d SMs, %d producer warps, %2d copies/stage: %7.1f GB/s per SM  %s\n", c.bytes,
           c.stages, c.ctas, c.np, c.pieces, gbs, cudaGetErrorString(e));
  }
  return 0;
}
