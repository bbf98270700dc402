// sf_probe.cu -- which byte of a TMEM scale-factor column scales which
// 32-element K block of a tcgen05.mma kind::mxf4 (block32, K = 64)?
// A and B hold 1.0 at element 0 of each of the two K chunks; the scale
// columns hold bytes (2^0, 2^1, 2^2, 2^3) on one operand, 1.0 on the other,
// so D = s[b0] + s[b1] names the bytes used.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sf_probe sf_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1603_06757_b200/csrc/bz_umma.cuh"

using namespace bz;

__global__ void __launch_bounds__(128, 1) probe(int which, float* out) {
  __shared__ __align__(1024) unsigned char sm[2 * 2 * 16 * 128];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5;
  // A: 128 rows x 2 chunks, B: 128 rows x 2 chunks, K-major no swizzle
  for (int i = threadIdx.x; i < (int)sizeof(sm) / 16; i += blockDim.x) {
    const int op = i / 256, rem = i % 256;          // 256 x 16 B per operand
    const int chunk = (rem / 8) % 2;
    uint4 z = make_uint4(0, 0, 0, 0);
    // element 0 of every row: A = 1.0 in chunk 0, 2.0 in chunk 1; B = 1.0
    z.x = (op == 0 && chunk == 1) ? 0x4u : 0x2u;
    reinterpret_cast<uint4*>(sm)[i] = z;
  }
  fence_proxy_async();
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
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
  // SF columns 480.. (A) and 488.. (B): the probed operand gets bytes
  // 0x7F, 0x80, 0x81, 0x82 (1, 2, 4, 8), the other all 0x7F
  const uint32_t pat = 0x82817F7Fu + 0x00000100u;  // bytes: 7F 80 81 82
  for (int c = 0; c < 32; c += 8) {
    const uint32_t col = 480 + c;
    const bool probed = (which == 0) ? (col < 488) : (col >= 488 && col < 496);
    tmem_st8(tmem + ((uint32_t)(32 * warp) << 16) + col, probed ? pat : 0x7F7F7F7Fu);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    const uint64_t ad = umma_desc(base, 128, 256), bd = umma_desc(base + 4096, 128, 256);
    umma_mxf4(tmem, ad, bd, mxf4_idesc(128), 0u, tmem + 480, tmem + 488);
    umma_commit(bar_s);
    mbar_wait(bar_s, 0);
  }
  __syncthreads();
  tc_fence_after();
  uint32_t v[8];
  tmem_ld8(tmem + ((uint32_t)(32 * warp) << 16), *reinterpret_cast<uint32_t(*)[8]>(v));
  tmem_ld_wait();
  if (threadIdx.x == 0 || threadIdx.x == 77) {
    out[(threadIdx.x ? 8 : 0) + 0] = __uint_as_float(v[0]);
    out[(threadIdx.x ? 8 : 0) + 1] = __uint_as_float(v[5]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 64);
  for (int which = 0; which < 2; ++which) {
    cudaMemset(d, 0, 64);
    probe<<<1, 128>>>(which, d);
    cudaError_t e = cudaDeviceSynchronize();
    float h[16];
    cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("%s scales bytes (1,2,4,8): D[0][0]=%g D[0][5]=%g D[77][0]=%g D[77][5]=%g (%s)\n",
           which ? "B" : "A", h[0], h[1], h[8], h[9], cudaGetErrorString(e));
  }
  return 0;
}
