// ptx_probe.cu -- microbenchmark / sanity check of the DSMEM hand-off primitives
// used by the cluster kernel: st.async + remote mbarrier complete_tx, re-arming,
// ping-pong latency between two CTAs of a cluster.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1702_07825_b200/csrc/ptx.cuh"
using namespace dvw;

__global__ void __cluster_dims__(2, 1, 1) pingpong(int iters, int nthr_send, unsigned long long* out, float* sink) {
  __shared__ __align__(16) float buf[64];
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  const uint32_t rank = ptx::cluster_rank();
  if (t == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_mbar_init();
    ptx::mbar_arm(ptx::smem_u32(&bar), 64 * 4);
  }
  __syncthreads();
  ptx::cluster_sync();
  const uint32_t peer = rank ^ 1;
  const uint32_t rbuf = ptx::mapa(ptx::smem_u32(&buf[t]), peer);
  const uint32_t rbar = ptx::mapa(ptx::smem_u32(&bar), peer);
  unsigned long long t0 = clock64();
  float v = (float)t;
  for (int i = 0; i < iters; ++i) {
    if (rank == 0 || i > 0) {
      if (rank == 1) {
        // wait for phase i-1... handled below
      }
    }
    if (rank == 0) {
      ptx::st_async(rbuf, v, rbar);
      while (!ptx::mbar_try_wait(ptx::smem_u32(&bar), i & 1)) {}
      if (t == 0) ptx::mbar_arm(ptx::smem_u32(&bar), 64 * 4);
      v = buf[t] + 1.0f;
    } else {
      while (!ptx::mbar_try_wait(ptx::smem_u32(&bar), i & 1)) {}
      if (t == 0) ptx::mbar_arm(ptx::smem_u32(&bar), 64 * 4);
      v = buf[t] + 1.0f;
      ptx::st_async(rbuf, v, rbar);
    }
  }
  unsigned long long t1 = clock64();
  if (t == 0 && rank == 0) out[0] = t1 - t0;
  sink[rank * 64 + t] = v;
  __syncwarp();
  ptx::cluster_sync();
}

int main() {
  unsigned long long* d_out; float* sink;
  cudaMalloc(&d_out, 8); cudaMalloc(&sink, 4096);
  for (int iters : {1, 10, 1000, 100000}) {
    pingpong<<<2, 64>>>(iters, 64, d_out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0; cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
    float hs[128]; cudaMemcpy(hs, sink, 512, cudaMemcpyDeviceToHost);
    printf("iters=%d err=%s cycles/roundtrip=%.1f sink0=%.0f sink1=%.0f\n", iters, cudaGetErrorString(e), (double)h / iters, hs[0], hs[64]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
