// issue_probe.cu -- how does the single MMA-issuing thread interact with the
// tensor pipe?  One CTA per SM; thread 0 issues K5-shaped MMAs
// (kind::mxf4 M=128 N=240 K=64, unit scales) and timestamps every issue.
//   A: 24 back-to-back MMAs into one accumulator (K-chain)
//   B: same, with a tcgen05.commit after every MMA
//   C: an idle gap of G clocks between consecutive MMAs: total time vs G
//      shows how much work the pipe queues ahead of the issuing thread
//   D: cost of an already-complete mbarrier try_wait by 1 lane / 32 lanes
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o issue_probe issue_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1603_06757_b200/csrc/bz_umma.cuh"

using namespace bz;

__device__ __forceinline__ void spin(long long g) {
  const long long t = clock64();
  while (clock64() - t < g) {
  }
}

__global__ void __launch_bounds__(128, 1) probe(int mode, int gap, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5;
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&bar[0]);
  const uint32_t bar2 = (uint32_t)__cvta_generic_to_shared(&bar[1]);
  if (threadIdx.x == 0) {
    mbar_init(bar_s, 1);
    mbar_init(bar2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  for (int c = 0; c < 512 - kSfCol; c += 8)
    tmem_st8(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(kSfCol + c), 0x7F7F7F7Fu);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  const uint64_t ad = umma_desc(base, 128, 256), bd = umma_desc(base + 16384, 128, 256);
  long long* o = out + blockIdx.x * 64;
  if ((mode <= 2 || mode == 4) && threadIdx.x == 0) {
    const int n = 24;
    long long t[n + 1];
    t[0] = clock64();
    for (int i = 0; i < n; ++i) {
      if ((mode == 2 || mode == 4) && i) spin(gap);
      if (mode == 4)  // alternate between two independent accumulators
        umma_mxf4(tmem + (uint32_t)((i & 1) * kUmmaN4), ad, bd, kMxf4Idesc, i >= 2 ? 1u : 0u,
                  tmem + kSfCol, tmem + kSfCol + 8);
      else
        umma_mxf4(tmem, ad, bd, kMxf4Idesc, i ? 1u : 0u, tmem + kSfCol, tmem + kSfCol + 8);
      if (mode == 1) umma_commit(bar2);
      t[i + 1] = clock64();
    }
    umma_commit(bar_s);
    mbar_wait(bar_s, 0);
    const long long te = clock64();
    for (int i = 0; i <= n; ++i) o[i] = t[i] - t[0];
    o[n + 1] = te - t[0];
  }
  if (mode == 5 && (warp == 0 || warp == 1) && (threadIdx.x & 31) == 0) {
    // two issuing threads (warps 0 and 1), 12 MMAs each into their own
    // accumulator, gap G between consecutive MMAs of the same thread
    const long long t0 = clock64();
    for (int i = 0; i < 12; ++i) {
      if (i) spin(gap);
      umma_mxf4(tmem + (uint32_t)(warp * kUmmaN4), ad, bd, kMxf4Idesc, i ? 1u : 0u,
                tmem + kSfCol, tmem + kSfCol + 8);
    }
    umma_commit(warp ? bar2 : bar_s);
    mbar_wait(warp ? bar2 : bar_s, 0);
    o[warp] = clock64() - t0;
  }
  if (mode == 6 && threadIdx.x == 0) {
    // commit latency: (a) no MMA pending, (b) after one MMA, (c) after 3 chained
    uint32_t ph = 0;
    for (int rep = 0; rep < 3; ++rep) {
      long long t0 = clock64();
      umma_commit(bar_s);
      mbar_wait(bar_s, ph); ph ^= 1;
      o[3 * rep + 0] = clock64() - t0;
      t0 = clock64();
      umma_mxf4(tmem, ad, bd, kMxf4Idesc, 0u, tmem + kSfCol, tmem + kSfCol + 8);
      const long long ti = clock64();
      umma_commit(bar_s);
      mbar_wait(bar_s, ph); ph ^= 1;
      o[3 * rep + 1] = clock64() - t0;
      o[20 + rep] = ti - t0;
      t0 = clock64();
      for (int i = 0; i < 3; ++i)
        umma_mxf4(tmem, ad, bd, kMxf4Idesc, i ? 1u : 0u, tmem + kSfCol, tmem + kSfCol + 8);
      umma_commit(bar_s);
      mbar_wait(bar_s, ph); ph ^= 1;
      o[3 * rep + 2] = clock64() - t0;
    }
  }
  if (mode == 3 && warp == 0) {
    // already-complete barrier: phase 0 completed by one arrive
    if (threadIdx.x == 0) mbar_arrive(bar2);
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < 64; ++i) mbar_wait_fast(bar2, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      o[0] = (t1 - t0) / 64;
      t0 = clock64();
      for (int i = 0; i < 64; ++i) mbar_wait_fast(bar2, 0);
      t1 = clock64();
      o[1] = (t1 - t0) / 64;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 64 * sms);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  std::vector<long long> h(64 * sms);
  auto run = [&](int mode, int gap) {
    cudaMemset(d, 0, sizeof(long long) * 64 * sms);
    probe<<<sms, 128, 64 * 1024>>>(mode, gap, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h.data(), d, sizeof(long long) * 64 * sms, cudaMemcpyDeviceToHost);
    return e;
  };
  for (int mode = 0; mode < 2; ++mode) {
    cudaError_t e = run(mode, 0);
    printf("mode %c (%s): issue times", mode ? 'B' : 'A', cudaGetErrorString(e));
    for (int i = 1; i <= 24; ++i) printf(" %lld", h[i]);
    printf(" | done %lld\n", h[25]);
  }
  for (int gap : {0, 32, 64, 96, 128, 160, 192, 256, 384}) {
    cudaError_t e = run(2, gap);
    printf("mode C gap %3d: total %6lld clk for 24 MMAs (%.1f per MMA)  last issue %lld (%s)\n", gap,
           h[25], h[25] / 24.0, h[24], cudaGetErrorString(e));
  }
  for (int gap : {0, 64, 128, 192, 256}) {
    cudaError_t e = run(4, gap);
    printf("mode E (2 accumulators) gap %3d: total %6lld clk for 24 MMAs (%.1f per MMA) issues", gap,
           h[25], h[25] / 24.0);
    for (int i = 1; i <= 8; ++i) printf(" %lld", h[i]);
    printf(" (%s)\n", cudaGetErrorString(e));
  }
  for (int gap : {0, 64, 128, 192, 256}) {
    cudaError_t e = run(5, gap);
    printf("mode F (2 issuing warps x 12) gap %3d: %6lld / %6lld clk (%.1f per MMA) (%s)\n", gap,
           h[0], h[1], (h[0] > h[1] ? h[0] : h[1]) / 24.0, cudaGetErrorString(e));
  }
  {
    cudaError_t e = run(6, 0);
    printf("mode G: commit->wait: none %lld / 1 MMA %lld (issue returned at %lld) / 3 MMAs %lld clk;"
           " rep2: %lld %lld %lld (%s)\n", h[6], h[7], h[22], h[8], h[3], h[4], h[5],
           cudaGetErrorString(e));
  }
  cudaError_t e = run(3, 0);
  printf("mode D: satisfied try_wait 32 lanes %lld clk, 1 lane %lld clk (%s)\n", h[0], h[1],
         cudaGetErrorString(e));
  return 0;
}
