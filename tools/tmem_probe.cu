// tmem_probe.cu -- tensor memory as a weight store: latency/throughput of tcgen05.ld
// (32x32b.x64: each thread gets 64 consecutive 32-bit columns of its lane) into registers.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define LD64(taddr, r) asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];" \
  : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]), \
    "=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]), \
    "=r"(r[32]),"=r"(r[33]),"=r"(r[34]),"=r"(r[35]),"=r"(r[36]),"=r"(r[37]),"=r"(r[38]),"=r"(r[39]),"=r"(r[40]),"=r"(r[41]),"=r"(r[42]),"=r"(r[43]),"=r"(r[44]),"=r"(r[45]),"=r"(r[46]),"=r"(r[47]), \
    "=r"(r[48]),"=r"(r[49]),"=r"(r[50]),"=r"(r[51]),"=r"(r[52]),"=r"(r[53]),"=r"(r[54]),"=r"(r[55]),"=r"(r[56]),"=r"(r[57]),"=r"(r[58]),"=r"(r[59]),"=r"(r[60]),"=r"(r[61]),"=r"(r[62]),"=r"(r[63]) : "r"(taddr))

template <int NW>
__global__ void __launch_bounds__(128, 1) tm(float* out, long long* cyc, int iters) {
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tbase;
  // lane field = bits 31:16, column = bits 15:0; warp w owns lanes 32w..32w+31
  const uint32_t my = base + ((uint32_t)(32 * warp) << 16);
  // fill: tcgen05.st 32x32b.x1 per column
  for (int c = 0; c < 512; ++c) {
    uint32_t v = __float_as_uint(1.0f + 1e-3f * (t + c));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(my + c), "r"(v));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  __syncthreads();
  float acc = 0.f;
  long long best = 0;
  if (warp < NW) {
    uint32_t r[64];
    // latency: dependent chain ld -> wait -> use
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t col = (uint32_t)((it * 64 + (int)acc * 0) & 511) & ~63u;
      LD64(my + col, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 64; ++i) acc = fmaf(__uint_as_float(r[i]), 1.0f, acc);
    }
    long long c1 = clock64();
    best = c1 - c0;
  }
  if (t == 0) cyc[0] = best;
  // throughput: 4 loads in flight, no dependency
  long long c2 = clock64();
  if (warp < NW) {
    uint32_t r0[64], r1[64];
    for (int it = 0; it < iters; ++it) {
      LD64(my + 0, r0);
      LD64(my + 64, r1);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += __uint_as_float(r0[it & 63]) + __uint_as_float(r1[(it + 5) & 63]);
    }
  }
  long long c3 = clock64();
  if (t == 0) cyc[1] = c3 - c2;
  out[t] = acc;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(base));
}

int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 16);
  const int iters = 1000;
  tm<1><<<1, 128>>>(o, c, iters); cudaError_t e = cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("1 warp : err=%s  ld(64 cols)+wait+64 FFMA chain = %.1f cycles/iter ; 2 loads (512 B/thread) per wait = %.1f cycles/iter\n", cudaGetErrorString(e), (double)h[0]/iters, (double)h[1]/iters);
  tm<4><<<1, 128>>>(o, c, iters); e = cudaDeviceSynchronize();
  cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("4 warps: err=%s  ld(64 cols)+wait+64 FFMA chain = %.1f cycles/iter ; 2 loads per wait = %.1f cycles/iter\n", cudaGetErrorString(e), (double)h[0]/iters, (double)h[1]/iters);
}
