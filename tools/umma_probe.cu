// umma_probe.cu -- validate the tcgen05.mma kind::tf32 operand layout used by the batched
// kernel: D[128 x N] = A[128 x K] * B[N x K]^T with both operands K-major, no swizzle,
// staged by 1-D bulk copies from global memory already in the canonical core-matrix
// order [K/4][rows][4].  Checks 1xTF32 and the 3-pass split (hi*hi + hi*lo + lo*hi)
// against an fp64 host product, and times a chain of MMAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_probe tools/umma_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int M, int N, int K>
__global__ void k_probe(const float* A, const float* Alo, const float* B, const float* Blo, float* D, int mode,
                        int swap, int reps, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sA = (float*)sm;
  float* sAl = sA + M * K;
  float* sB = sAl + M * K;
  float* sBl = sB + N * K;
  __shared__ uint64_t bar_ld, bar_mma;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_ld)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_mma)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (t == 0) {
    const uint32_t bytes = 4u * (2 * M * K + 2 * N * K);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar_ld)), "r"(bytes));
    auto cp = [&](void* dst, const float* src, uint32_t nb) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(dst)),
                   "l"(src), "r"(nb), "r"(su32(&bar_ld))
                   : "memory");
    };
    cp(sA, A, 4 * M * K);
    cp(sAl, Alo, 4 * M * K);
    cp(sB, B, 4 * N * K);
    cp(sBl, Blo, 4 * N * K);
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok)
                   : "r"(su32(&bar_ld)));
  }
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  const uint32_t lboA = swap ? 128 : M * 16, sboA = swap ? M * 16 : 128;
  const uint32_t lboB = swap ? 128 : N * 16, sboB = swap ? N * 16 : 128;
  long long c0 = 0, c1 = 0;
  if (t == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    c0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
      for (int k = 0; k < K / 8; ++k) {
        const uint32_t offA = k * 2 * M * 16, offB = k * 2 * N * 16;
        const uint32_t acc = (k > 0) ? 1u : 0u;
        mma_tf32(tbase, make_desc(su32(sA) + offA, lboA, sboA), make_desc(su32(sB) + offB, lboB, sboB), idesc, acc);
        if (mode == 3) {
          mma_tf32(tbase, make_desc(su32(sA) + offA, lboA, sboA), make_desc(su32(sBl) + offB, lboB, sboB), idesc, 1);
          mma_tf32(tbase, make_desc(su32(sAl) + offA, lboA, sboA), make_desc(su32(sB) + offB, lboB, sboB), idesc, 1);
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar_mma))
                 : "memory");
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok)
                   : "r"(su32(&bar_mma)));
  }
  if (t == 0) {
    c1 = clock64();
    cycles[0] = c1 - c0;
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int w = t >> 5;
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    const uint32_t ta = tbase + ((uint32_t)(32 * w) << 16) + c;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 16; ++i) D[t * N + c + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
}

static float tf32_trunc(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

// canonical K-major: element (row, k) at ((k/4) * rows + row) * 4 + k%4
static void canon(const std::vector<float>& X, int rows, int K, std::vector<float>& out) {
  out.assign((size_t)rows * K, 0.f);
  for (int i = 0; i < rows; ++i)
    for (int k = 0; k < K; ++k) out[((size_t)(k / 4) * rows + i) * 4 + k % 4] = X[(size_t)i * K + k];
}

template <int M, int N, int K>
static void run(int mode, int swap, int reps) {
  std::vector<float> A(M * K), B(N * K);
  srand(1);
  for (auto& v : A) v = (float)rand() / RAND_MAX - 0.5f;
  for (auto& v : B) v = (float)rand() / RAND_MAX - 0.5f;
  std::vector<float> Ah(M * K), Al(M * K), Bh(N * K), Bl(N * K);
  for (int i = 0; i < M * K; ++i) { Ah[i] = A[i]; Al[i] = A[i] - tf32_trunc(A[i]); }
  for (int i = 0; i < N * K; ++i) { Bh[i] = B[i]; Bl[i] = B[i] - tf32_trunc(B[i]); }
  std::vector<float> cA, cAl, cB, cBl;
  canon(Ah, M, K, cA); canon(Al, M, K, cAl); canon(Bh, N, K, cB); canon(Bl, N, K, cBl);
  float *dA, *dAl, *dB, *dBl, *dD;
  long long* dc;
  cudaMalloc(&dA, 4 * M * K); cudaMalloc(&dAl, 4 * M * K); cudaMalloc(&dB, 4 * N * K); cudaMalloc(&dBl, 4 * N * K);
  cudaMalloc(&dD, 4 * M * N); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, cA.data(), 4 * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dAl, cAl.data(), 4 * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, cB.data(), 4 * N * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dBl, cBl.data(), 4 * N * K, cudaMemcpyHostToDevice);
  const int smem = 4 * (2 * M * K + 2 * N * K);
  cudaFuncSetAttribute(k_probe<M, N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_probe<M, N, K><<<1, 128, smem>>>(dA, dAl, dB, dBl, dD, mode, swap, reps, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("M%d N%d K%d mode %d swap %d: %s\n", M, N, K, mode, swap, cudaGetErrorString(e)); exit(1); }
  std::vector<float> D(M * N);
  long long cyc;
  cudaMemcpy(D.data(), dD, 4 * M * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  double maxrel = 0, maxabs = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double ref = 0, mag = 0;
      for (int k = 0; k < K; ++k) { ref += (double)A[i * K + k] * B[j * K + k]; mag += fabs((double)A[i * K + k] * B[j * K + k]); }
      const double err = fabs(D[i * N + j] - ref);
      maxabs = fmax(maxabs, err);
      maxrel = fmax(maxrel, err / mag);
    }
  printf("M%d N%d K%d mode %dxTF32 swap %d: max|err| %.3e  max err/sum|ab| %.3e  D[0]=%f  cycles(%d reps, %d mma) %lld\n", M, N,
         K, mode, swap, maxabs, maxrel, D[0], reps, reps * (K / 8) * mode, cyc);
  cudaFree(dA); cudaFree(dAl); cudaFree(dB); cudaFree(dBl); cudaFree(dD); cudaFree(dc);
}

int main() {
  run<128, 32, 64>(1, 0, 1);
  run<128, 32, 64>(1, 1, 1);
  run<128, 32, 64>(3, 0, 1);
  run<128, 16, 64>(3, 0, 1);
  run<128, 64, 64>(3, 0, 1);
  run<128, 256, 64>(3, 0, 1);
  run<128, 32, 128>(3, 0, 1);
  // timing: chains of MMAs
  run<128, 16, 64>(3, 0, 16);
  run<128, 32, 64>(3, 0, 16);
  run<128, 64, 64>(3, 0, 16);
  run<128, 128, 64>(3, 0, 16);
  run<128, 256, 64>(3, 0, 16);
  return 0;
}
