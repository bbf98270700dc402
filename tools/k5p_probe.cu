// k5p_probe.cu -- back-to-back tcgen05.mma kind::mxf4 throughput for the
// K5p issue pattern (one thread, no epilogue, no loads), to separate the
// tensor pipe's own rate from the kernel's hand-offs.
//
// Variants (one CTA per SM, 148 CTAs, clocks per MMA):
//   0  probe baseline: same A/B, SBO 256, alternating accumulators
//   1  K5p tile: 4 MMAs per tile into one accumulator (part 0 / part 1 of a
//      480-row B stage, B SBO 512, A SBO 640, LBO 256 on the last), stages
//      rotate over 5 B buffers, A over 4 buffers, accumulators alternate
//   2  variant 1 without the LBO-256 MMA
//   3  variant 1 with one B stage only
//   4  variant 1 with 16 warps streaming tcgen05.ld (60 columns, unpacked)
//      from the other accumulator meanwhile
//   5  variant 1 with one commit per tile to an mbarrier (no waits)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/k5p_probe tools/k5p_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1603_06757_b200/csrc/bz_umma.cuh"

using namespace bz;

constexpr int kN = 240, kCB = 4, kCA = 5, kStages = 5, kABufs = 4;
constexpr uint32_t kTB = 2 * kN * kCB * 16;   // 30 KB
constexpr uint32_t kTA = 128 * kCA * 16;      // 10 KB

__global__ void __launch_bounds__(544, 1) probe(int variant, int tiles, long long* clk) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ uint32_t s_tmem;
  __shared__ volatile int s_stop;
  const int warp = threadIdx.x >> 5;
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    mbar_init(bar_s, 1);
    mbar_init(bar_s + 8, 1);
    s_stop = 0;
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
    for (int c = 0; c < 32; c += 8)
      tmem_st8(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(kSfCol + c),
               kSfCol + c == kSfColMagic ? 0x8F8F8F8Fu : 0x7F7F7F7Fu);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  // operands: zeros are fine for timing
  for (uint32_t i = threadIdx.x; i < (kStages * kTB + kABufs * kTA) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t sB = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sA = sB + kStages * kTB;
  const uint32_t idesc = mxf4_idesc(kN);
  const uint32_t sfa = tmem + kSfCol, sfb = tmem + kSfCol + 8, sfm = tmem + kSfColMagic;
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    if (variant == 0) {
      const uint64_t ad = umma_desc(sA, 128, 256), bd = umma_desc(sB, 128, 256);
      for (int i = 0; i < 4 * tiles; ++i)
        umma_mxf4(tmem + (uint32_t)((i & 1) * kN), ad, bd, idesc, (i & 2) ? 1u : 0u, sfa, sfb);
    } else {
      const uint64_t a0 = umma_desc(sA, 128, kCA * 128), b0 = umma_desc(sB, 128, kCB * 128);
      for (int t = 0; t < tiles; ++t) {
        const int stg = variant == 3 ? 0 : t % kStages, ab = (t / 3) % kABufs;
        const uint64_t bd = b0 + (uint64_t)(stg * (kTB >> 4));
        const uint64_t ad = a0 + (uint64_t)(ab * (kTA >> 4));
        const uint32_t d = tmem + (uint32_t)((t & 1) * kN);
        for (int q = 0; q < 2; ++q) {
          const uint64_t bq = bd + (uint64_t)(q * (kN / 8) * kCB * 8);
          for (int kb = 0; kb < 2; ++kb)
            if (variant == 6)
              umma_nvf4(d, ad + 16u * kb + (kb == 1 ? (uint64_t)(8 * q) << 16 : 0ull),
                        bq + 16u * kb, idesc & ~(1u << 23), (q | kb) ? 1u : 0u, sfa, q ? sfm : sfb);
            else
              umma_mxf4(d, ad + 16u * kb + ((variant != 2 && kb == 1) ? (uint64_t)(8 * q) << 16 : 0ull),
                        bq + 16u * kb, idesc, (q | kb) ? 1u : 0u, sfa, q ? sfm : sfb);
        }
        if (variant == 5) umma_commit(bar_s + 8);
      }
    }
    umma_commit(bar_s);
    mbar_wait(bar_s, 0);
    clk[blockIdx.x] = clock64() - t0;
    s_stop = 1;
  } else if (variant == 4 && warp >= 1 && warp <= 16) {
    // epilogue-like TMEM traffic: 16 warps x 60 columns, unpacked
    const int e = warp - 1, quarter = e & 3, sl = e >> 2;
    uint32_t sink = 0;
    for (int it = 0; !s_stop; ++it) {
      uint32_t v[60];
      tmem_ld_cols<60>(tmem + ((uint32_t)(32 * quarter) << 16) + (uint32_t)((it & 1) * kN + 60 * sl), v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 60; ++i) sink ^= v[i];
    }
    if (sink == 0x12345678u) clk[1000 + blockIdx.x] = sink;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}


// Pipeline probe: one issuer thread (warp 0) and 16 epilogue warps hand
// accumulators back and forth through mbarriers exactly like K5p (ACC
// buffers, commit -> accfull, 16 arrivals -> accempty).  mode bits:
//   1  epilogue loads its 60 columns (unpacked) before releasing
//   2  ... packed (.pack::16b, 30 registers)
//   4  SPLIT: each tile's accumulator is two halves of N/2 columns with
//      their own barriers; the MMAs of half h only wait for half h
//   8  the epilogue releases, then does 30 VIMNMX3 on what it loaded
//  16  one issuer warp per accumulator buffer (else warp 0 issues all)
//  32 / 64  8 / 4 epilogue warps instead of 16
// 128  epilogue waits with the tight PTX loop
// 256  no epilogue hand-off at all (issue-only timing)
// 512  no tcgen05 fences around the hand-off
// 1024 one waiting warp per lane quarter, named barriers for the rest
//
// Measured (B200): the MMA pattern alone and two issuers without hand-off
// run at 480 clk per tile (peak); one issuer 559; the hand-off with 16
// epilogue warps ~570-720 (run to run), 4 warps ~565; fences cost nothing;
// named-barrier leaders and more, smaller buffers are slower.
constexpr int kPipeWarps = 20;  // up to 3 issuers (mode 16) + 16 epilogue warps
__global__ void __launch_bounds__(32 * kPipeWarps, 1) pipe_probe(int mode, int acc_bufs, int tiles,
                                                              long long* clk) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bars[32];
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bars);
  const bool split = mode & 4;
  const int parts = split ? 2 : 1;
  const int N = (480 / acc_bufs) & ~15;
  auto accfull = [&](int i) { return bar_s + 8u * i; };
  auto accempty = [&](int i) { return bar_s + 8u * (16 + i); };
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) {
      mbar_init(accfull(i), 1);
      mbar_init(accempty(i), (mode & 1024) ? 4 : ((mode & 64) ? 4 : (mode & 32) ? 8 : 16) / (split ? 2 : 1));
    }
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
  if (warp >= 1 && warp <= 4) {
    for (int c = 0; c < 32; c += 8)
      tmem_st8(tmem + ((uint32_t)(32 * (warp - 1)) << 16) + (uint32_t)(kSfCol + c),
               kSfCol + c == kSfColMagic ? 0x8F8F8F8Fu : 0x7F7F7F7Fu);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  for (uint32_t i = threadIdx.x; i < (kStages * kTB + kABufs * kTA) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t sB = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sA = sB + kStages * kTB;
  const uint32_t sfa = tmem + kSfCol, sfb = tmem + kSfCol + 8, sfm = tmem + kSfColMagic;
  long long t0 = clock64();
  // mode 16: one issuer warp per accumulator buffer (warp b issues tiles
  // t % acc_bufs == b), like the kernel; else warp 0 issues every tile
  const int nis = (mode & 16) ? acc_bufs : 1;
  const int e0 = 3;  // first epilogue warp
  if (warp < nis) {
    const uint32_t idesc = mxf4_idesc(N / parts);
    const uint64_t a0 = umma_desc(sA, 128, kCA * 128), b0 = umma_desc(sB, 128, kCB * 128);
    for (int t = warp; t < tiles; t += nis) {
      const int buf = t % acc_bufs;
      const int stg = t % kStages, ab = (t / 3) % kABufs;
      const uint64_t bd = b0 + (uint64_t)(stg * (kTB >> 4));
      const uint64_t ad = a0 + (uint64_t)(ab * (kTA >> 4));
      for (int h = 0; h < parts; ++h) {
        const int hb = buf * parts + h;
        if (!(mode & 256)) mbar_wait_fast(accempty(hb), ((t / acc_bufs) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(buf * N + h * (N / parts));
        if (elect_one()) {
          for (int q = 0; q < 2; ++q) {
            const uint64_t bq = bd + (uint64_t)(q * (kN / 8) * kCB * 8) +
                                (uint64_t)(h * (N / parts / 8) * kCB * 8);
            for (int kb = 0; kb < 2; ++kb)
              umma_mxf4(d, ad + 16u * kb + (kb == 1 ? (uint64_t)(8 * q) << 16 : 0ull),
                        bq + 16u * kb, idesc, (q | kb) ? 1u : 0u, sfa, q ? sfm : sfb);
          }
          umma_commit(accfull(hb));
        }
        __syncwarp();
      }
    }
  } else if (warp >= e0 && warp < e0 + ((mode & 64) ? 4 : (mode & 32) ? 8 : 16)) {
    const int e = warp - e0, quarter = e & 3, sl = e >> 2;   // 4 column slices
    const int cols = N / 4;                                 // per warp
    const int h = split ? sl / 2 : 0;
    uint32_t sink = 0x7fff7fffu;
    for (int t = 0; t < tiles; ++t) {
      const int buf = t % acc_bufs;
      const int hb = buf * parts + h;
      if (mode & 256) break;  // mode 256: no epilogue at all (issue-only timing)
      // mode 1024: one warp per lane quarter waits on the mbarrier and
      // releases the quarter's other warps through a named barrier
      const bool lead = !(mode & 1024) || e < 4;
      if (lead) {
        if (mode & 128) mbar_wait_fast(accfull(hb), (t / acc_bufs) & 1);
        else mbar_wait(accfull(hb), (t / acc_bufs) & 1);
      }
      if (mode & 1024) asm volatile("bar.sync %0, 128;" ::"r"(1 + quarter) : "memory");
      if (!(mode & 512)) tc_fence_after();
      const uint32_t tb = tmem + ((uint32_t)(32 * quarter) << 16) + (uint32_t)(buf * N + cols * sl);
      uint32_t v[64];
      if (mode & 1) {
        tmem_ld_cols<60>(tb, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 60; i += 4) tmem_regs4_after_wait(v + i);
      } else if (mode & 2) {
        tmem_ld_cols_p<60>(tb, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 28; i += 4) tmem_regs4_after_wait(v + i);
        tmem_regs4_after_wait(v + 26);
      }
      if (!(mode & 512)) tc_fence_before();
      __syncwarp();
      if (mode & 1024) {
        asm volatile("bar.sync %0, 128;" ::"r"(1 + quarter) : "memory");
        if (e < 4 && lane == 0) mbar_arrive(accempty(hb));
      } else if (lane == 0) {
        mbar_arrive(accempty(hb));
      }
      if (mode & 8) {
#pragma unroll
        for (int i = 0; i + 1 < 60; i += 2) sink = __vimin3_s16x2(sink, v[i], v[i + 1]);
      }
    }
    if (sink == 0x12345u) clk[2000] = sink;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) clk[blockIdx.x] = clock64() - t0;
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int main() {
  const size_t smem = kStages * kTB + kABufs * kTA;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long* d;
  cudaMalloc(&d, 2048 * sizeof(long long));
  const int tiles = 4000;
  for (int v = 0; v <= 6; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      probe<<<148, 544, smem>>>(v, tiles, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("variant %d: %s\n", v, cudaGetErrorString(e)); return 1; }
    }
    std::vector<long long> h(148);
    cudaMemcpy(h.data(), d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0;
    for (long long x : h) s += x;
    s /= 148;
    const double per_mma = s / (4.0 * tiles);
    printf("variant %d: %.1f clk per MMA (ideal 120), %.0f MACs/clk/SM\n", v, per_mma,
           128.0 * kN * 64 / per_mma);
  }
  cudaFuncSetAttribute(pipe_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // {mode, buffers}: see the mode bits above pipe_probe
  const int cfgs[][2] = {{0, 2},   {16, 2},  {17, 2},  {18, 2}, {25, 2}, {80, 2},
                         {272, 2}, {256, 2}, {528, 2}, {1040, 2}, {16, 3}, {272, 3}};
  for (auto& c : cfgs) {
    for (int rep = 0; rep < 2; ++rep) {
      pipe_probe<<<148, 32 * kPipeWarps, smem>>>(c[0], c[1], tiles, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("pipe %d/%d: %s\n", c[0], c[1], cudaGetErrorString(e)); return 1; }
    }
    std::vector<long long> h(148);
    cudaMemcpy(h.data(), d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0;
    for (long long x : h) s += x;
    s /= 148;
    const int N = (480 / c[1]) & ~15;
    printf("pipe mode %2d bufs %d (N %d): %.0f clk per tile, MMA-ideal %d, %.2f of peak\n", c[0], c[1], N,
           s / tiles, 2 * N, 2.0 * N / (s / tiles));
  }
  return 0;
}
