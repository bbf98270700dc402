// bz_tc.cuh -- K2: the round on the tensor pipe (legacy warp-level IMMA,
// mma.sync.m16n8k32 s8 x s8 -> s32, native on sm_100a).
//
// The weight of a codeword P ^ S over GF(2) is an integer dot product:
//     w(P ^ S) = w(P) + sum_j (1 - 2 P_j) * S_j ,
// so with the prefix P encoded as +-1 bytes (A operand, 16 rows per m-tile)
// and the suffix sum S encoded as 0/1 bytes (B operand, 8 columns per
// n-tile), one IMMA chain over the n columns (K = 32 per instruction) with
// the accumulator initialised to w(P) yields the exact weights of 16 x 8
// codewords.  Every weight is exact (|values| <= 256 in s32).
//
// Work decomposition (same chunk/lane plan as K1, suffix depth D = 3):
//   combination = prefix {(g-4)-subset of [0, ell)} + ell  (lane-owned
//   walker, one prefix per lane per step)  +  suffix e1 < e2 < e3 in (ell, k).
//   The 32 lanes' current prefixes form the A operand (two m16 tiles); the
//   warp walks e1 < e2 uniformly, forms the fragment of R[e1] ^ R[e2] in
//   registers, and streams e3 in n8 tiles through ldmatrix from a 0/1 byte
//   image of the rows in shared memory; B = ldmatrix ^ (R[e1]^R[e2]).
//   Tail columns (e3 >= k) read a zero row and are masked in the epilogue;
//   lanes without a prefix duplicate a valid one (harmless for a minimum).
#pragma once

#include "bz_kernels.cuh"

namespace bz {

// Byte stride of one row of the 0/1 image: 32 bytes per 32-column block plus
// 16, so 8 consecutive rows hit 8 distinct 16-byte bank groups (ldmatrix is
// conflict-free).
__host__ __device__ constexpr int tc_stride(int w) { return 32 * w + 16; }
constexpr int kTcPadRows = 8;  // zero rows after the k rows of each Gamma

// +-1 bytes of the 4 bits of `word` at `shift`: bit 0 -> 0x01, bit 1 -> 0xff.
__device__ __forceinline__ uint32_t pm1_nibble(uint32_t word, int shift) {
  const uint32_t x = (word >> shift) & 0xFu;
  const uint32_t m = (x * 0x00204081u) & 0x01010101u;
  return m * 0xFEu + 0x01010101u;
}

__device__ __forceinline__ void imma16832(int (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                          uint32_t b1, const int (&c)[4]) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%10,%11,%12,%13};"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(c[0]), "r"(c[1]),
        "r"(c[2]), "r"(c[3]));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void ldsm_x2(uint32_t& r0, uint32_t& r1, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(addr));
}

template <int W>
__host__ __device__ inline size_t tc_smem_bytes(int m, int k, int ngroups) {
  size_t base = (smem_base_bytes<W>(m, k, ngroups) + 15) & ~size_t(15);
  return base + (size_t)m * (k + kTcPadRows) * tc_stride(W);
}

template <int W>
__global__ void __launch_bounds__(256)
k2_round_mma(const RoundArgs a, const uint8_t* __restrict__ tbl) {
  constexpr int TS = tc_stride(W);
  constexpr int WP = padded_words(W);
  extern __shared__ __align__(16) unsigned char smem[];
  // 0/1 byte image first (its copy overlaps the staging below)
  const size_t tbase = (smem_base_bytes<W>(a.m, a.k, a.ngroups) + 15) & ~size_t(15);
  unsigned char* stbl = smem + tbase;
  {
    const int n16 = a.m * (a.k + kTcPadRows) * TS / 16;
    const uint4* src = reinterpret_cast<const uint4*>(tbl);
    uint4* dst = reinterpret_cast<uint4*>(stbl);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
  }
  uint32_t *srows, *spx;
  Group* sgroups;
  stage<W>(a, srows, spx, sgroups, smem);  // ends with __syncthreads

  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int gid = lane >> 2, t0 = lane & 3;
  const int k = a.k, q = a.g - 4;
  volatile int* vbound = a.bound;
  const uint32_t stbl_s = (uint32_t)__cvta_generic_to_shared(stbl);
  // this lane's ldmatrix row offset inside an 8-row tile and its 16-byte half
  const int ld_row = lane & 7;
  const int ld_off = (lane >> 4) * 32 + ((lane >> 3) & 1) * 16;

  while (true) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(a.counter, 1ull);
    c = __shfl_sync(FULL, c, 0);
    const unsigned long long chunk = c * (unsigned long long)a.nshards + a.shard;
    if (chunk >= a.nchunks) break;
    if (vbound[0] <= a.lower_prev) break;

    const ChunkView v = open_chunk(sgroups, a.ngroups, chunk, lane);
    const long long maxcnt = __shfl_sync(FULL, v.cnt, 0);
    const unsigned long long first0 = __shfl_sync(FULL, v.first, 0);
    const uint32_t* R = srows + v.gr.gamma * k * WP;
    const uint32_t* PX = spx + v.gr.gamma * (k + 1) * px_stride(W);
    const uint32_t tg = stbl_s + (uint32_t)(v.gr.gamma * (k + kTcPadRows) * TS);
    const unsigned char* tgp = stbl + v.gr.gamma * (k + kTcPadRows) * TS;
    const int e0 = v.gr.ell + 1;

    // lanes without prefixes duplicate lane 0's first prefix
    Walker<W> wk;
    wk.init(v.cnt > 0 ? v.first : first0, q, v.gr.ell, R, a.binom);

    int best = INT_MAX;
    for (long long p = 0; p < maxcnt; ++p) {
      // ---- A operand: the 32 lanes' prefixes as +-1 bytes; C init = w(P)
      int wt = 0;
#pragma unroll
      for (int j = 0; j < W; ++j) wt += __popc(wk.acc[j]);
      uint32_t A[2][W][4];
      int C0[4], C1[4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int r0 = gid + 16 * mt, r1 = r0 + 8;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const uint32_t w0 = __shfl_sync(FULL, wk.acc[j], r0);
          const uint32_t w1 = __shfl_sync(FULL, wk.acc[j], r1);
          A[mt][j][0] = pm1_nibble(w0, 4 * t0);
          A[mt][j][1] = pm1_nibble(w1, 4 * t0);
          A[mt][j][2] = pm1_nibble(w0, 16 + 4 * t0);
          A[mt][j][3] = pm1_nibble(w1, 16 + 4 * t0);
        }
        const int c0 = __shfl_sync(FULL, wt, r0), c1 = __shfl_sync(FULL, wt, r1);
        if (mt == 0) { C0[0] = C0[1] = c0; C0[2] = C0[3] = c1; }
        else         { C1[0] = C1[1] = c0; C1[2] = C1[3] = c1; }
      }

      // ---- suffixes e1 < e2 < e3 above ell
#pragma unroll 1
      for (int e1 = e0; e1 < k - 2; ++e1) {
        uint32_t f1[W][2];
        const unsigned char* p1 = tgp + e1 * TS + 4 * t0;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          f1[j][0] = *reinterpret_cast<const uint32_t*>(p1 + 32 * j);
          f1[j][1] = *reinterpret_cast<const uint32_t*>(p1 + 32 * j + 16);
        }
#pragma unroll 1
        for (int e2 = e1 + 1; e2 < k - 1; ++e2) {
          uint32_t f12[W][2];
          const unsigned char* p2 = tgp + e2 * TS + 4 * t0;
#pragma unroll
          for (int j = 0; j < W; ++j) {
            f12[j][0] = f1[j][0] ^ *reinterpret_cast<const uint32_t*>(p2 + 32 * j);
            f12[j][1] = f1[j][1] ^ *reinterpret_cast<const uint32_t*>(p2 + 32 * j + 16);
          }
#pragma unroll 1
          for (int e3 = e2 + 1; e3 < k; e3 += 8) {
            const int row = min(e3 + ld_row, k);  // row k is all zero
            const uint32_t addr = tg + (uint32_t)(row * TS + ld_off);
            uint32_t B[W][2];
#pragma unroll
            for (int j = 0; j + 1 < W; j += 2) {
              uint32_t r[4];
              ldsm_x4(r, addr + 32 * j);
              B[j][0] = r[0] ^ f12[j][0];
              B[j][1] = r[1] ^ f12[j][1];
              B[j + 1][0] = r[2] ^ f12[j + 1][0];
              B[j + 1][1] = r[3] ^ f12[j + 1][1];
            }
            if constexpr (W & 1) {
              uint32_t r0, r1;
              ldsm_x2(r0, r1, addr + 32 * (W - 1));
              B[W - 1][0] = r0 ^ f12[W - 1][0];
              B[W - 1][1] = r1 ^ f12[W - 1][1];
            }
            int d0[4], d1[4];
            imma16832(d0, A[0][0], B[0][0], B[0][1], C0);
            imma16832(d1, A[1][0], B[0][0], B[0][1], C1);
#pragma unroll
            for (int j = 1; j < W; ++j) {
              imma16832(d0, A[0][j], B[j][0], B[j][1], d0);
              imma16832(d1, A[1][j], B[j][0], B[j][1], d1);
            }
            if (e3 + 8 <= k) {
              best = min(best, min(min(min(d0[0], d0[1]), min(d0[2], d0[3])),
                                   min(min(d1[0], d1[1]), min(d1[2], d1[3]))));
            } else {
              const int col = e3 + 2 * t0;
              const int m0 = col < k ? 0 : 0x3fffffff;
              const int m1 = col + 1 < k ? 0 : 0x3fffffff;
              best = min(best, min(min(d0[0] + m0, d0[1] + m1), min(d0[2] + m0, d0[3] + m1)));
              best = min(best, min(min(d1[0] + m0, d1[1] + m1), min(d1[2] + m0, d1[3] + m1)));
            }
          }
        }
      }
      if (p + 1 < v.cnt) wk.step(PX);
    }

    const int wbest = __reduce_min_sync(FULL, best);
    const unsigned tot = __reduce_add_sync(FULL, (unsigned)v.cnt);
    if (lane == 0) {
      if (wbest < vbound[1 + v.gr.gamma]) atomicMin(a.bound + 1 + v.gr.gamma, wbest);
      if (wbest < vbound[0]) atomicMin(a.bound, wbest);
      const unsigned long long t = (unsigned long long)(k - e0);
      atomicAdd(a.combos + v.gr.gamma,
                (unsigned long long)tot * (t * (t - 1) * (t - 2) / 6));
    }
  }
}

}  // namespace bz
