// tmem_probe.cu -- tcgen05.ld (TMEM -> registers) throughput on sm_100a:
// NW warps per CTA (one CTA per SM) each load `batch` x (32 lanes x 32
// columns x 4 B) per wait, many times.  Prints bytes per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_probe tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void ld16p(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

template <int BATCH, bool PACK>
__global__ void probe(int iters, long long* clk, int* sink) {
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16);
  int acc = 0;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (PACK) {
      uint32_t v[BATCH][16];
#pragma unroll
      for (int b = 0; b < BATCH; ++b) ld16p(tm + ((32 * (b + i + warp)) & 511), v[b]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int b = 0; b < BATCH; ++b) acc += (int)(v[b][0] ^ v[b][15]);
    } else {
      uint32_t v[BATCH][32];
#pragma unroll
      for (int b = 0; b < BATCH; ++b) ld32(tm + ((32 * (b + i + warp)) & 511), v[b]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int b = 0; b < BATCH; ++b) acc += (int)(v[b][0] ^ v[b][31]);
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512));
  }
}

template <int BATCH, bool PACK>
void run(int nw) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* clk; int* sink;
  cudaMalloc(&clk, sizeof(long long) * sms);
  cudaMalloc(&sink, sizeof(int) * sms * 32 * nw);
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) probe<BATCH, PACK><<<sms, 32 * nw>>>(iters, clk, sink);
  cudaDeviceSynchronize();
  long long h[256]; cudaMemcpy(h, clk, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes = (double)iters * BATCH * 32 * 32 * 4 * nw;  // TMEM bytes per CTA
  printf("warps=%2d batch=%d pack=%d: %.1f TMEM bytes/clk/SM  (%s)\n", nw, BATCH, (int)PACK,
         bytes / mx, cudaGetErrorString(cudaGetLastError()));
  cudaFree(clk); cudaFree(sink);
}

int main() {
  for (int nw : {4, 8, 16}) {
    run<1, false>(nw); run<2, false>(nw); run<4, false>(nw);
    run<2, true>(nw); run<4, true>(nw);
  }
  return 0;
}
