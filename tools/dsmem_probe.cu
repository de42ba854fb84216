// dsmem_probe.cu -- one-way hand-off latency between two cluster CTAs for the message shapes
// the cluster kernel uses: 64 x st.async.b32, 16 x st.async.v4, 1 x cp.async.bulk (256 B),
// and a 4-destination fan-out (4 x 256 B) with each shape.  Ping-pong, cycles per round trip / 2.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1702_07825_b200/csrc/ptx.cuh"
using namespace dvw;

__device__ __forceinline__ void bulk_s2s(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes, uint32_t rbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst_cluster), "r"(src_cta), "r"(bytes), "r"(rbar) : "memory");
}

template <int MODE, int FAN>
__global__ void __cluster_dims__(5, 1, 1) pp(int iters, long long* out, float* sink) {
  __shared__ __align__(128) float buf[4][64];   // receive slots (one per potential sender slot)
  __shared__ __align__(128) float stage[64];
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  const uint32_t rank = ptx::cluster_rank();
  if (t == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_mbar_init();
    ptx::mbar_arm(ptx::smem_u32(&bar), rank == 0 ? 64 * 4 * FAN : 64 * 4);
  }
  if (t < 64) stage[t] = t;
  __syncthreads();
  ptx::cluster_sync();
  long long t0 = clock64();
  // rank 0 sends to ranks 1..FAN; each of them answers rank 0 (into slot rank-1)
  for (int i = 0; i < iters; ++i) {
    const bool sender = (rank == 0);
    if (!sender) {
      if (rank > FAN) break;
      while (!ptx::mbar_try_wait(ptx::smem_u32(&bar), i & 1)) {}
      if (t == 0) ptx::mbar_arm(ptx::smem_u32(&bar), 64 * 4);
    }
    if (rank <= FAN) {
      const int ndst = sender ? FAN : 1;
      for (int d = 0; d < ndst; ++d) {
        const uint32_t dst = sender ? (uint32_t)(d + 1) : 0u;
        const int slot = sender ? 0 : (int)rank - 1;
        const uint32_t rb = ptx::mapa(ptx::smem_u32(&bar), dst);
        if (MODE == 0) { if (t < 64) ptx::st_async(ptx::mapa(ptx::smem_u32(&buf[slot][t]), dst), stage[t], rb); }
        else if (MODE == 1) { if (t < 16) ptx::st_async4(ptx::mapa(ptx::smem_u32(&buf[slot][4 * t]), dst), *reinterpret_cast<float4*>(&stage[4 * t]), rb); }
        else { if (t == 0) bulk_s2s(ptx::mapa(ptx::smem_u32(&buf[slot][0]), dst), ptx::smem_u32(stage), 256, rb); }
      }
    }
    if (sender) {
      while (!ptx::mbar_try_wait(ptx::smem_u32(&bar), i & 1)) {}
      if (t == 0) ptx::mbar_arm(ptx::smem_u32(&bar), 64 * 4 * FAN);
    }
  }
  long long t1 = clock64();
  if (t == 0 && rank == 0) out[0] = t1 - t0;
  sink[rank * 64 + (t & 63)] = buf[0][t & 63];
  __syncwarp();
  ptx::cluster_sync();
}

template <int MODE, int FAN>
void run(const char* name, long long* d, float* s) {
  const int iters = 10000;
  pp<MODE, FAN><<<5, 128>>>(iters, d, s);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-34s err=%s one-way (rt/2) = %.1f cycles\n", name, cudaGetErrorString(e), (double)h / iters / 2);
}

int main() {
  long long* d; float* s;
  cudaMalloc(&d, 8); cudaMalloc(&s, 1 << 14);
  run<0, 1>("64 x st.async.b32, fan 1", d, s);
  run<1, 1>("16 x st.async.v4, fan 1", d, s);
  run<2, 1>("1 x cp.async.bulk 256B, fan 1", d, s);
  run<0, 4>("64 x st.async.b32, fan 4", d, s);
  run<1, 4>("16 x st.async.v4, fan 4", d, s);
  run<2, 4>("1 x cp.async.bulk 256B, fan 4", d, s);
  return 0;
}
