// bz_brute.cuh -- K6: GPU brute-force minimum distance,
// the independent check of brute_force_distance (m/engine.py:223-237): all
// 2^k - 1 nonzero messages of one generator matrix in Gray-code order, one
// row XOR per codeword.  Message index i in [1, 2^k) maps to gray(i) =
// i ^ (i >> 1); consecutive Gray codes differ in bit ctz(i), so a thread that
// owns the index range [s, s + L) unranks gray(s) once (XOR of its set rows)
// and then steps with one row XOR, W POPC and one min per codeword.
// Persistent grid, ranges drawn from a global atomic cursor.
#pragma once

#include "bz_kernels.cuh"

namespace bz {

constexpr int kBruteMaxK = 48;
constexpr int kBruteSpan = 1 << 12;  // messages per thread range

template <int W>
__global__ void __launch_bounds__(256)
k6_brute(const uint32_t* __restrict__ rows, int k, unsigned long long nranges,
         unsigned long long* __restrict__ counter, int* __restrict__ best_out) {
  constexpr int WP = padded_words(W);
  __shared__ uint32_t srow[kBruteMaxK * WP];
  for (int i = threadIdx.x; i < k * WP; i += blockDim.x) srow[i] = rows[i];
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  int best = INT_MAX;
  const unsigned long long total = 1ull << k;
  while (true) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(counter, 32ull);
    c = __shfl_sync(FULL, c, 0) + (unsigned long long)lane;
    if (__all_sync(FULL, c >= nranges)) break;
    if (c < nranges) {
      const unsigned long long s = c * (unsigned long long)kBruteSpan;
      unsigned long long e = s + kBruteSpan;
      if (e > total) e = total;
      // codeword of gray(s)
      uint32_t acc[W];
#pragma unroll
      for (int j = 0; j < W; ++j) acc[j] = 0u;
      const unsigned long long gs = s ^ (s >> 1);
      for (int b = 0; b < k; ++b)
        if ((gs >> b) & 1ull)
#pragma unroll
          for (int j = 0; j < W; ++j) acc[j] ^= srow[b * WP + j];
      if (s > 0) {
        int w = 0;
#pragma unroll
        for (int j = 0; j < W; ++j) w += __popc(acc[j]);
        best = min(best, w);
      }
      for (unsigned long long i = s + 1; i < e; ++i) {
        const int b = __ffsll((long long)i) - 1;
        int w = 0;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          acc[j] ^= srow[b * WP + j];
          w += __popc(acc[j]);
        }
        best = min(best, w);
      }
    }
  }
  const int wbest = __reduce_min_sync(FULL, best);
  if (lane == 0 && wbest < INT_MAX) atomicMin(best_out, wbest);
}

}  // namespace bz
