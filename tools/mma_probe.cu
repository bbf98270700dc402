// mma_probe.cu -- measures legacy warp-level MMA throughput on sm_100a
// (IMMA s8, HMMA f16/f16, e4m3 mma.sync) against POPC, to decide whether
// the weight computation w(P^S) = w(P) + sum_j (1-2P_j) S_j belongs on the
// tensor pipes.  Standalone: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o mma_probe mma_probe.cu && ./mma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 4
__global__ void k_imma(int* out, int iters, long long* clk) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * (i + 3);
  b[0] = threadIdx.x * 11; b[1] = threadIdx.x * 13;
  int c[CH][4] = {};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ch = 0; ch < CH; ++ch)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[ch][0]), "+r"(c[ch][1]), "+r"(c[ch][2]), "+r"(c[ch][3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  long long t1 = clock64();
  int s = 0;
  for (int ch = 0; ch < CH; ++ch) s += c[ch][0] + c[ch][1] + c[ch][2] + c[ch][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void k_hmma(int* out, int iters, long long* clk) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u;
  b[0] = 0x3c003c00u; b[1] = 0x3c003c00u;
  uint32_t c[CH][2] = {};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ch = 0; ch < CH; ++ch)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};"
        : "+r"(c[ch][0]), "+r"(c[ch][1])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  long long t1 = clock64();
  int s = 0;
  for (int ch = 0; ch < CH; ++ch) s += c[ch][0] + c[ch][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void k_qmma(int* out, int iters, long long* clk) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x38383838u;
  b[0] = 0x38383838u; b[1] = 0x38383838u;
  uint32_t c[CH][2] = {};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ch = 0; ch < CH; ++ch)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.f16.e4m3.e4m3.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};"
        : "+r"(c[ch][0]), "+r"(c[ch][1])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  long long t1 = clock64();
  int s = 0;
  for (int ch = 0; ch < CH; ++ch) s += c[ch][0] + c[ch][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <typename F>
void run(const char* name, F kern, double macs_per_mma, int warps_per_block, int blocks_per_sm) {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int blocks = sms * blocks_per_sm, threads = 32 * warps_per_block, iters = 4096;
  int* out; long long* clk;
  cudaMalloc(&out, sizeof(int) * blocks * threads);
  cudaMalloc(&clk, sizeof(long long) * blocks);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks];
  cudaMemcpy(h, clk, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
  double mmas = (double)blocks * warps_per_block * iters * CH;
  double macs = mmas * macs_per_mma;
  printf("%-6s warps/SM=%3d  %.3f ms  %.1f MACs/clk/SM  %.1f TMAC/s  (%.0f MHz)  err=%s\n", name,
         warps_per_block * blocks_per_sm, ms, macs / (sms * (double)mx), macs / (ms * 1e-3) / 1e12,
         mx / (ms * 1e-3) / 1e6, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(clk); delete[] h;
}

int main() {
  for (int w : {4, 8, 16}) {
    run("imma", k_imma, 16.0 * 8 * 32, w, 1);
    run("hmma", k_hmma, 16.0 * 8 * 16, w, 1);
    run("qmma", k_qmma, 16.0 * 8 * 32, w, 1);
  }
  return 0;
}
