// mxf4_probe.cu -- can the BZ weight GEMM run on the fp4 tensor path?
//
// A = +-1 prefix rows, B = 0/1 triple rows, both exactly representable in
// e2m1; with every block scale = 1.0 (ue8m0 0x7F) tcgen05.mma kind::mxf4
// computes the same integer dot products as kind::i8, in fp32 (exact below
// 2^24), at twice the MAC rate and from half the operand bytes.
//
//  1. correctness: one M=128 x N x K=160 product as K=64 + K=96 MMAs,
//     checked against the host;
//  2. throughput: back-to-back MMAs per SM (kind::i8 K=32 and kind::mxf4
//     K=64 / K=96), optionally with 8 warps streaming tcgen05.ld from TMEM
//     meanwhile (the epilogue's load on the accumulator port).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mxf4_probe mxf4_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1603_06757_b200/csrc/bz_umma.cuh"

using namespace bz;

__device__ __forceinline__ void mma_mxf4(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc,
                                         uint32_t acc, uint32_t sfa, uint32_t sfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
      ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb)
      : "memory");
}

__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N, int k96) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) |
         ((uint32_t)(M >> 4) << 24) | ((uint32_t)k96 << 31);
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}


__device__ void alloc512(uint32_t* s_tmem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(s_tmem)),
               "r"(512));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ void dealloc512(uint32_t tmem) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
// every warp of the first four fills its lane quarter of columns [kSfCol, +32)
__device__ void fill_sf(uint32_t tmem) {
  const int warp = threadIdx.x >> 5;
  if (warp < 4) {
    for (int c = 0; c < 32; c += 8)
      tmem_st8(tmem + ((uint32_t)(32 * warp) << 16) + kSfCol + c, 0x7F7F7F7Fu);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
}

// ---- 1. correctness: D[128][N] = A[128][160] . B[N][160]^T
// gA / gB: operand tiles already in the K-major no-swizzle core-matrix
// layout (16-byte chunks of 32 e2m1, 5 chunks per row)
template <int N>
__global__ void __launch_bounds__(128, 1) check(const uint8_t* gA, const uint8_t* gB, float* gD, int mode) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ uint32_t s_tmem;
  constexpr int TA = 128 * 80, TB = N * 80;
  for (int i = threadIdx.x; i < (TA + TB) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] =
        i < TA / 16 ? reinterpret_cast<const uint4*>(gA)[i]
                    : reinterpret_cast<const uint4*>(gB)[i - TA / 16];
  fence_proxy_async();
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    mbar_init(bar_s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) alloc512(&s_tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  fill_sf(tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  if (threadIdx.x == 0) {
    const uint64_t ad = umma_desc(base, 128, 640), bd = umma_desc(base + TA, 128, 640);
    if (mode == 2) {
      mma_mxf4(tmem, ad, bd, idesc_mxf4(128, N, 1), 0u, tmem + kSfCol, tmem + kSfCol + 8);
    } else {
      mma_mxf4(tmem, ad, bd, idesc_mxf4(128, N, 0), 0u, tmem + kSfCol, tmem + kSfCol + 8);
      if (mode == 0)
        mma_mxf4(tmem, ad + 16u, bd + 16u, idesc_mxf4(128, N, 1), 1u, tmem + kSfCol,
                 tmem + kSfCol + 8);
    }
    umma_commit(bar_s);
    mbar_wait(bar_s, 0);
  }
  __syncthreads();
  tc_fence_after();
  const int warp = threadIdx.x >> 5, r = threadIdx.x;
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    tmem_ld8(tmem + ((uint32_t)(32 * warp) << 16) + c, v);
    tmem_ld_wait();
    for (int j = 0; j < 8; ++j) gD[r * N + c + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    dealloc512(tmem);
  }
}

// ---- 2. throughput: warp 0 issues `iters` MMA pairs; warps 1..8 optionally
// stream tcgen05.ld over columns [256, 480) while it runs
template <int KIND, int N>
__global__ void __launch_bounds__(32 * 17, 1) thr(int iters, int readers, int packed, long long* clk) {
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
  if (warp == 0) alloc512(&s_tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  fill_sf(tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    if (iters < 0) {  // no MMAs: readers alone for -iters clocks
      while (clock64() - t0 < -(long long)iters) {
      }
    } else if (KIND == 0) {  // kind::i8, K-chains of 5 x K=32 (K=160)
      const uint64_t ad = umma_desc(base, 128, 1280), bd = umma_desc(base + 20480, 128, 1280);
      for (int i = 0; i < iters; ++i)
        for (int kb = 0; kb < 5; ++kb)
          umma_i8(tmem, ad + 16u * kb, bd + 16u * kb, idesc_i8(128, N), kb ? 1u : 0u);
    } else {  // kind::mxf4, 3 x K=64 chains into accumulator 0 (K=192)
      const uint64_t ad = umma_desc(base, 128, 768), bd = umma_desc(base + 12288, 128, 768);
      for (int i = 0; i < iters; ++i) {
        mma_mxf4(tmem, ad, bd, idesc_mxf4(128, N, 0), 0u, tmem + kSfCol, tmem + kSfCol + 8);
        mma_mxf4(tmem, ad + 16u, bd + 16u, idesc_mxf4(128, N, 0), 1u, tmem + kSfCol,
                 tmem + kSfCol + 8);
        mma_mxf4(tmem, ad + 32u, bd + 32u, idesc_mxf4(128, N, 0), 1u, tmem + kSfCol,
                 tmem + kSfCol + 8);
      }
    }
    umma_commit(bar_s);
    mbar_wait(bar_s, 0);
    clk[2 * blockIdx.x] = clock64() - t0;
    s_done = 1;
  } else if (warp >= 1 && warp <= readers) {
    // tcgen05.ld streaming: each reader warp covers its lane quarter
    const uint32_t tq = tmem + ((uint32_t)(32 * (warp & 3)) << 16);  // warp % 4 = lane quarter
    long long loads = 0;
    uint32_t acc = 0;
    // reader warp w: lane quarter w % 4, 64 columns at 240 + 32 * ((w / 4) % 4)
    // (inside accumulator 1, which the MMAs do not touch), 4 loads per wait
    while (!s_done) {
      uint32_t v[64];
      if (packed) {
        // 4 x (32 columns as 16 packed registers): 128 columns per wait
        tmem_ld16p(tq + 240 + 32 * (((warp - 1) / 4) % 4), v);
        tmem_ld16p(tq + 272 + 32 * (((warp - 1) / 4) % 4), v + 16);
        tmem_ld16p(tq + 240 + 32 * (((warp - 1) / 4) % 4) + 8, v + 32);
        tmem_ld16p(tq + 272 + 32 * (((warp - 1) / 4) % 4) + 8, v + 48);
        tmem_ld_wait();
        for (int j = 0; j < 64; ++j) acc ^= v[j];
        loads += 4;
      } else {
        tmem_ld16(tq + 240 + 32 * (((warp - 1) / 4) % 4), v);
        tmem_ld16(tq + 256 + 32 * (((warp - 1) / 4) % 4), v + 16);
        tmem_ld16(tq + 240 + 32 * (((warp - 1) / 4) % 4) + 8, v + 32);
        tmem_ld16(tq + 256 + 32 * (((warp - 1) / 4) % 4) + 8, v + 48);
        tmem_ld_wait();
        for (int j = 0; j < 64; ++j) acc ^= v[j];
        loads += 2;  // 64 columns = two 32-column units
      }
    }
    if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long*)&clk[2 * blockIdx.x + 1], loads);
    if (acc == 0x12345678u) clk[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    dealloc512(tmem);
  }
}

static uint8_t e2m1(int v) { return v == 0 ? 0x0 : (v > 0 ? 0x2 : 0xA); }

// element (row, kk) of a K-major no-swizzle tile of 5 chunks per row
static void put(std::vector<uint8_t>& t, int row, int kk, uint8_t nib) {
  const int chunk = kk / 32, byte = (kk % 32) / 2;
  const size_t off = (size_t)(row >> 3) * 640 + chunk * 128 + (row & 7) * 16 + byte;
  t[off] |= (kk & 1) ? (uint8_t)(nib << 4) : nib;
}

template <int N>
bool run_check() {
  const int K = 160;
  std::vector<int> A(128 * K), B(N * K);
  srand(7);
  for (auto& x : A) x = (rand() & 1) ? 1 : -1;
  for (auto& x : B) x = rand() & 1;
  std::vector<uint8_t> tA(128 * 80, 0), tB(N * 80, 0);
  for (int r = 0; r < 128; ++r)
    for (int kk = 0; kk < K; ++kk) put(tA, r, kk, e2m1(A[r * K + kk]));
  for (int r = 0; r < N; ++r)
    for (int kk = 0; kk < K; ++kk) put(tB, r, kk, e2m1(B[r * K + kk]));
  uint8_t *dA, *dB;
  float* dD;
  cudaMalloc(&dA, tA.size());
  cudaMalloc(&dB, tB.size());
  cudaMalloc(&dD, sizeof(float) * 128 * N);
  cudaMemcpy(dA, tA.data(), tA.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, tB.data(), tB.size(), cudaMemcpyHostToDevice);
  const int smem = 128 * 80 + N * 80;
  cudaFuncSetAttribute(check<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<float> D(128 * N);
  cudaError_t e = cudaSuccess;
  for (int mode = 2; mode >= 0; --mode) {
    check<N><<<1, 128, smem>>>(dA, dB, dD, mode);
    e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, sizeof(float) * D.size(), cudaMemcpyDeviceToHost);
    char name[128];
    snprintf(name, sizeof name, "gpurun_out/mxf4_D_N%d_mode%d.bin", N, mode);
    FILE* f = fopen(name, "wb");
    if (f) { fwrite(D.data(), sizeof(float), D.size(), f); fclose(f); }
  }
  {
    char name[128];
    snprintf(name, sizeof name, "gpurun_out/mxf4_AB_N%d.bin", N);
    FILE* f = fopen(name, "wb");
    if (f) { fwrite(A.data(), sizeof(int), A.size(), f); fwrite(B.data(), sizeof(int), B.size(), f); fclose(f); }
  }
  int bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < N; ++c) {
      int s = 0;
      for (int kk = 0; kk < K; ++kk) s += A[r * K + kk] * B[c * K + kk];
      if (D[r * N + c] != (float)s) {
        if (bad < 5) printf("  mismatch r=%d c=%d got %f want %d\n", r, c, D[r * N + c], s);
        ++bad;
      }
    }
  printf("check mxf4 M=128 N=%d K=64+96: %s (%d mismatches, %s)\n", N, bad ? "FAIL" : "ok", bad,
         cudaGetErrorString(e));
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return bad == 0;
}

template <int KIND, int N>
void run_thr(int readers, int packed = 0, int iters_arg = 4000) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* clk;
  cudaMalloc(&clk, sizeof(long long) * 2 * sms);
  const int smem = 64 * 1024, iters = iters_arg;
  cudaFuncSetAttribute(thr<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(clk, 0, sizeof(long long) * 2 * sms);
    thr<KIND, N><<<sms, 32 * 17, smem>>>(iters, readers, packed, clk);
  }
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(2 * sms);
  cudaMemcpy(h.data(), clk, sizeof(long long) * 2 * sms, cudaMemcpyDeviceToHost);
  long long mx = 0, loads = 0;
  for (int i = 0; i < sms; ++i) {
    mx = h[2 * i] > mx ? h[2 * i] : mx;
    loads += h[2 * i + 1];
  }
  const double macs = iters < 0 ? 0.0 : (double)iters * 128 * N * (KIND ? 192 : 160);
  printf("%s N=%d readers=%d packed=%d: %7.0f MACs/clk/SM, %6.1f clk per K=160 tile, tcgen05.ld %6.0f B/clk/SM (%s)\n",
         KIND ? "mxf4" : "i8  ", N, readers, packed, macs / mx, (double)mx / iters,
         (double)loads * 32 * 32 * 4 / sms / mx, cudaGetErrorString(e));
  cudaFree(clk);
}

int main() {
  run_check<256>();
  run_check<240>();
  for (int readers : {0, 8, 16}) run_thr<1, 240>(readers, 0);
  for (int readers : {8, 16}) run_thr<1, 240>(readers, 1);
  for (int packed : {0, 1}) run_thr<1, 240>(16, packed, -2000000);
  return 0;
}
