// dsmem_tag_probe.cu -- one-way latency of a DSMEM hand-off between two CTAs of a cluster:
//   A: st.async.b32 + mbarrier complete_tx, receiver mbarrier.try_wait (the cluster kernel's hand-off)
//   B: st.relaxed.cluster.shared::cluster.b64 of {value, tag}, receiver spins ld.relaxed.cluster
//   C: as B, receiver spins ld.volatile.shared
// Ping-pong of ITER round trips between lane 0 of CTA 0 and CTA 1; cycles / (2 ITER).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int ITER = 4000;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank)); return r;
}
__device__ __forceinline__ uint32_t cluster_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <int V>
__global__ void __cluster_dims__(2, 1, 1) k(long long* out) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t box;
  const uint32_t me = cluster_rank(), peer = me ^ 1;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    box = 0xffffffffull << 32;
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cluster_sync();
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t rbar = mapa(smem_u32(&bar), peer), rbox = mapa(smem_u32(&box), peer);
    t0 = clock64();
    for (int i = 0; i < ITER; ++i) {
      const bool send_first = (me == 0);
      for (int step = 0; step < 2; ++step) {
        const bool do_send = (step == 0) == send_first;
        if (do_send) {
          if (V == 0) {
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
                         :: "r"(rbox), "r"(i), "r"(rbar) : "memory");
          } else {
            const uint64_t v = ((uint64_t)i << 32) | 0x3f800000u;
            asm volatile("st.relaxed.cluster.shared::cluster.b64 [%0], %1;" :: "r"(rbox), "l"(v) : "memory");
          }
        } else {
          if (V == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], 4;" :: "r"(smem_u32(&bar)) : "memory");
            uint32_t ok = 0;
            while (!ok)
              asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                           : "=r"(ok) : "r"(smem_u32(&bar)), "r"((uint32_t)(i & 1)) : "memory");
          } else {
            uint64_t v;
            do {
              if (V == 1) asm volatile("ld.relaxed.cluster.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"(smem_u32(&box)) : "memory");
              else asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(v) : "r"(smem_u32(&box)) : "memory");
            } while ((uint32_t)(v >> 32) != (uint32_t)i);
          }
        }
      }
    }
    t1 = clock64();
    if (me == 0) out[V] = t1 - t0;
  }
  cluster_sync();
}
int main() {
  long long* out; cudaMalloc(&out, 64); cudaMemset(out, 0, 64);
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<2, 32>>>(out); k<1><<<2, 32>>>(out); k<2><<<2, 32>>>(out);
    cudaDeviceSynchronize();
  }
  long long h[3]; cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
  const char* nm[3] = {"st.async+mbarrier", "st.relaxed.cluster b64 tag + ld.relaxed.cluster spin", "tag + ld.volatile spin"};
  for (int v = 0; v < 3; ++v) printf("%-55s one-way %.1f cycles\n", nm[v], h[v] / (2.0 * ITER));
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
