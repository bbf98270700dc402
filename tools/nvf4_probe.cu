// nvf4_probe.cu -- what bounds a K5q / K5f tile?
//
//  1. tcgen05.mma rate, M = 128 x N = 240 x K = 64 back to back from shared
//     memory: kind::mxf4 (block32, the roofline probe), kind::mxf4nvf4
//     (block16, what K5q / K5f issue), and mxf4nvf4 with every third MMA's B
//     descriptor stepping N / 8 row groups between its two K chunks (K5f's
//     tail fold);
//  2. tcgen05.ld rate: R reader warps (warp w: lane quarter w % 4, column
//     slice w / 4) each load 60 columns packed (.pack::16b, 30 registers) or
//     unpacked per wait, as the epilogue does, alone and under the MMAs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvf4_probe nvf4_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1603_06757_b200/csrc/bz_umma.cuh"

using namespace bz;

constexpr int N = 240;

// KIND 0: mxf4 block32; 1: nvf4 block16; 2: nvf4, third MMA folded
template <int KIND>
__global__ void __launch_bounds__(32 * 17, 1) probe(int iters, int readers, int packed, int alu,
                                                    long long* clk) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ uint32_t s_tmem;
  __shared__ volatile int s_done;
  const int warp = threadIdx.x >> 5;
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    s_done = 0;
    mbar_init(bar_s, 1);
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
  if (warp < 4) {
    for (int c = 0; c < 512 - kSfCol; c += 8)
      tmem_st8(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(kSfCol + c),
               KIND == 0 ? 0x7F7F7F7Fu : 0x38383838u);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  if (threadIdx.x == 0) {
    // A: 128 rows x 4 chunks; B: 480 rows x 3 chunks (a K5f stage)
    const uint64_t ad = umma_desc(base, 128, 4 * 128);
    const uint64_t bd = umma_desc(base + 8192, 128, 3 * 128);
    const uint64_t bf = umma_desc(base + 8192 + 256, (N / 8) * 3 * 128, 3 * 128);
    const uint32_t id32 = mxf4_idesc(N), id16 = mxf4_idesc(N) & ~(1u << 23);
    const uint32_t sf = tmem + kSfCol;
    const long long t0 = clock64();
    if (iters < 0) {
      while (clock64() - t0 < -(long long)iters) {
      }
    } else {
      for (int i = 0; i < iters; ++i) {
        const uint32_t d = tmem + (uint32_t)((i & 1) * N);
        if (KIND == 0) {
          umma_mxf4(d, ad, bd, id32, 0u, sf, sf);
          umma_mxf4(d, ad, bd + (N / 8) * 24, id32, 1u, sf, sf);
          umma_mxf4(d, ad + 16u, bd + 16u, id32, 1u, sf, sf);
        } else {
          umma_nvf4(d, ad, bd, id16, 0u, sf, sf);
          umma_nvf4(d, ad, bd + (N / 8) * 24, id16, 1u, sf, sf);
          umma_nvf4(d, ad + 16u, KIND == 2 ? bf : bd + 16u, id16, 1u, sf, sf);
        }
      }
    }
    umma_commit(bar_s);
    mbar_wait(bar_s, 0);
    clk[2 * blockIdx.x] = clock64() - t0;
    s_done = 1;
  } else if (warp >= 1 && warp <= readers) {
    const int w = warp - 1;
    // columns of accumulator region [0, 480): the MMAs write there too (the
    // values are irrelevant), so reads and writes share the TMEM ports as in
    // the kernel
    const uint32_t tq = tmem + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)(60 * ((w >> 2) & 3)) +
                        (uint32_t)(240 * ((w >> 4) & 1));
    long long loads = 0;
    uint32_t acc = 0xFFFFFFFFu;
    if (packed && alu == 3) {
      // software-pipelined halves: the 32-column half A and the 28-column
      // half B alternate, each load in flight while the other half's
      // add + AND pass runs
      uint32_t va[16], vb[14];
      uint32_t k = (uint32_t)clock64() & 0xFF;
      tmem_ld_cols_p<32>(tq, va);
      while (!s_done) {
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("" : "+r"(va[j]));
        tmem_ld_cols_p<28>(tq + 32, vb);
#pragma unroll
        for (int j = 0; j + 1 < 16; j += 2) acc &= (k * 0x10001u + va[j]) & (k * 0x10001u + va[j + 1]);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 14; ++j) asm volatile("" : "+r"(vb[j]));
        tmem_ld_cols_p<32>(tq, va);
#pragma unroll
        for (int j = 0; j + 1 < 14; j += 2) acc &= (k * 0x10001u + vb[j]) & (k * 0x10001u + vb[j + 1]);
        ++loads;
      }
      tmem_ld_wait();
    }
    while (!s_done) {
      if (packed) {
        uint32_t v[30];
        tmem_ld_cols_p<60>(tq, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 30; ++j) asm volatile("" : "+r"(v[j]));
        if (alu == 1) {
#pragma unroll
          for (int j = 0; j + 1 < 30; j += 2) acc &= v[j] & v[j + 1];
        } else if (alu == 2) {
          uint32_t k = (uint32_t)loads;
          asm volatile("" : "+r"(k));
#pragma unroll
          for (int j = 0; j + 1 < 30; j += 2) acc &= (v[j] + k) & (v[j + 1] + k);
        } else {
          acc &= v[0];
        }
      } else {
        uint32_t v[60];
        tmem_ld_cols<60>(tq, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 60; ++j) asm volatile("" : "+r"(v[j]));
        if (alu) {
#pragma unroll
          for (int j = 0; j + 1 < 60; j += 2) acc &= v[j] & v[j + 1];
        } else {
          acc &= v[0];
        }
      }
      ++loads;
    }
    if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long*)&clk[2 * blockIdx.x + 1], loads);
    if (acc == 0x12345678u) clk[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int KIND>
void run(int readers, int packed, int alu, int iters = 4000) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* clk;
  cudaMalloc(&clk, sizeof(long long) * 2 * sms);
  const int smem = 64 * 1024;
  cudaFuncSetAttribute(probe<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(clk, 0, sizeof(long long) * 2 * sms);
    probe<KIND><<<sms, 32 * 17, smem>>>(iters, readers, packed, alu, clk);
  }
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(2 * sms);
  cudaMemcpy(h.data(), clk, sizeof(long long) * 2 * sms, cudaMemcpyDeviceToHost);
  long long mx = 0, loads = 0;
  for (int i = 0; i < sms; ++i) {
    mx = h[2 * i] > mx ? h[2 * i] : mx;
    loads += h[2 * i + 1];
  }
  const char* names[] = {"mxf4 b32", "nvf4 b16", "nvf4 fold"};
  printf("%-9s readers=%2d packed=%d alu=%d: %6.1f clk per MMA, %6.1f clk per 3-MMA tile; "
         "tcgen05.ld %6.1f columns/clk/SM = one 128 x 240 tile per %6.1f clk (%s)\n",
         iters < 0 ? "no MMAs" : names[KIND], readers, packed, alu,
         iters < 0 ? 0.0 : (double)mx / iters / 3, iters < 0 ? 0.0 : (double)mx / iters,
         (double)loads * 60 * 32 / sms / mx,
         loads ? 128.0 * 240.0 / ((double)loads * 60 * 32 / sms / mx) : 0.0, cudaGetErrorString(e));
  cudaFree(clk);
}

int main() {
  run<0>(0, 1, 0);
  run<1>(0, 1, 0);
  run<2>(0, 1, 0);
  for (int packed = 1; packed >= 0; --packed)
    for (int alu = packed ? 1 : 2; alu <= (packed ? 2 : 1); ++alu) {
      run<1>(16, packed, alu, -2000000);
      run<2>(16, packed, alu);
    }
  run<1>(16, 1, 3, -2000000);
  run<2>(16, 1, 3);
  return 0;
}
