// umma_probe.cu -- tcgen05.mma kind::i8 issue/throughput probe on sm_100a:
// M=128 x N x K=32 MMAs from shared memory, one CTA per SM.  Variants:
// consecutive MMAs into the SAME accumulator (a K-chain, as in a GEMM tile)
// or alternating between NACC accumulators.  Prints MACs/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I.. -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1603_06757_b200/csrc/bz_umma.cuh"

template <int N, int NACC, int CHAIN>
__global__ void __launch_bounds__(128, 1) probe(int iters, long long* clk) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5;
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    bz::mbar_init(bar_s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  bz::tc_fence_before();
  __syncthreads();
  bz::tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint64_t ad = bz::umma_desc(base, 128, 1280);
    const uint64_t bd = bz::umma_desc(base + 20480, 128, 1280);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int chain = i % CHAIN;          // position in a K-chain
      const int acc = (i / CHAIN) % NACC;   // which accumulator
      bz::umma_i8(tmem + (uint32_t)(acc * N), ad + 16u * chain, bd + 16u * chain, idesc,
                  chain > 0 ? 1u : 0u);
    }
    bz::umma_commit(bar_s);
    bz::mbar_wait(bar_s, 0);
    clk[blockIdx.x] = clock64() - t0;
  }
  bz::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    bz::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int N, int NACC, int CHAIN>
void run(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* clk; cudaMalloc(&clk, sizeof(long long) * sms);
  const size_t smem = 64 * 1024;
  cudaFuncSetAttribute(probe<N, NACC, CHAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) probe<N, NACC, CHAIN><<<sms, 128, smem>>>(iters, clk);
  cudaDeviceSynchronize();
  long long h[256]; cudaMemcpy(h, clk, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-28s N=%3d: %6.0f MACs/clk/SM  (%s)\n", name, N,
         (double)iters * 128 * N * 32 / mx, cudaGetErrorString(cudaGetLastError()));
  cudaFree(clk);
}

int main() {
  run<256, 2, 1>("alternate 2 acc, no chain");
  run<256, 1, 5>("1 acc, K-chain of 5");
  run<256, 2, 5>("2 acc, K-chains of 5");
  run<128, 4, 5>("4 acc, K-chains of 5");
  run<128, 1, 5>("1 acc, K-chain of 5");
  run<256, 1, 1000000>("1 acc, endless chain");
  return 0;
}
