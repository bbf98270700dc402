// tmem_ld_probe.cu -- cost model of tcgen05.ld (TMEM -> registers) on
// sm_100a: NW warps per CTA (one CTA per SM), each loop issues L loads of
// 32x32b.xX (optionally .pack::16b) then one tcgen05.wait::ld.  Prints TMEM
// columns x 4 B delivered per clock per SM, to pick the epilogue's load
// shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld_probe tmem_ld_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1603_06757_b200/csrc/bz_umma.cuh"

using namespace bz;

__device__ __forceinline__ void ld64(uint32_t taddr, uint32_t* v) {
  tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(v));
  tmem_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
}
__device__ __forceinline__ void ld64x(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,"
      "%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,"
      "%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]),
        "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]),
        "=r"(v[38]), "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]),
        "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]),
        "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]),
        "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]),
        "=r"(v[62]), "=r"(v[63])
      : "r"(taddr));
}

// MODE: 0 = 4 x x16, 1 = 2 x x32, 2 = 1 x x64, 3 = 4 x x16.pack (128 cols),
//       4 = 2 x x32 via x16.pack pairs (64 cols as 32 regs)
template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(int iters, long long* clk, int* sink) {
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 64 * ((warp >> 2) & 3);
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t v[64];
    if (MODE == 0) {
      tmem_ld16(tm, v); tmem_ld16(tm + 16, v + 16); tmem_ld16(tm + 32, v + 32); tmem_ld16(tm + 48, v + 48);
    } else if (MODE == 1) {
      ld64(tm, v);
    } else if (MODE == 2) {
      ld64x(tm, v);
    } else if (MODE == 3) {
      tmem_ld16p(tm, v); tmem_ld16p(tm + 32, v + 16);
      tmem_ld16p(tm + 64, v + 32); tmem_ld16p(tm + 96, v + 48);
    } else {
      tmem_ld16p(tm, v); tmem_ld16p(tm + 32, v + 16);
    }
    tmem_ld_wait();
    const int nreg = MODE == 4 ? 32 : 64;
    for (int j = 0; j < nreg; ++j) acc ^= v[j];
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = (int)acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512));
  }
}

template <int MODE>
void run(int nw, const char* name) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* clk;
  int* sink;
  cudaMalloc(&clk, sizeof(long long) * sms);
  cudaMalloc(&sink, sizeof(int) * sms * 1024);
  const int iters = 2048;
  for (int rep = 0; rep < 2; ++rep) probe<MODE><<<sms, 32 * nw>>>(iters, clk, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, clk, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const int cols = MODE == 3 ? 128 : 64;
  printf("%-26s warps=%2d: %6.0f column-bytes/clk/SM, %5.1f clk per load round (%s)\n", name, nw,
         (double)iters * nw * 32 * cols * 4 / mx, (double)mx / iters, cudaGetErrorString(e));
  cudaFree(clk);
  cudaFree(sink);
}

int main() {
  for (int nw : {4, 8, 16}) {
    run<0>(nw, "4 x x16 (64 cols)");
    run<1>(nw, "2 x x32 (64 cols)");
    run<2>(nw, "1 x x64 (64 cols)");
    run<3>(nw, "4 x x16.pack16 (128 cols)");
    run<4>(nw, "2 x x16.pack16 (64 cols)");
  }
  return 0;
}
