// bz_tc.cuh -- K3: the round as a GEMM on the tensor pipe (legacy
// warp-level IMMA, mma.sync.m16n8k32 s8 x s8 -> s32, native on sm_100a).
//
// The weight of a codeword P ^ S over GF(2) is an integer dot product:
//     w(P ^ S) = w(P) + sum_j (1 - 2 P_j) * S_j ,
// so with the prefix P encoded as +-1 bytes (A operand, 16 rows per m-tile)
// and the suffix sum S encoded as 0/1 bytes (B operand, 8 columns per
// n-tile), one IMMA chain over the n columns (K = 32 per instruction)
// started from the accumulator w(P) yields the exact weights of 16 x 8
// codewords (|values| <= 256: exact in s32).
//
// Decomposition (suffix depth D = 3, g >= 4): a g-combination is
//   prefix = {(g-4)-subset of [0, ell)} + ell      (A side, lane walkers)
//   suffix = {e1 < e2 < e3} with e1 > ell          (B side, a table row)
// For each Gamma the device holds the TRIPLE TABLE: every 3-subset of the
// rows as a 0/1 byte row, ordered by smallest element descending, so the
// suffixes valid for ell -- all triples above ell -- are exactly its first
// C(k-1-ell, 3) rows.  A (Gamma, ell) group is then a dense GEMM
//   [C(ell, g-4) prefixes] x [C(k-1-ell, 3) triples] x [n columns]
// with a min-reduction epilogue.  A block (8 warps = 256 prefixes, one per
// lane) streams that slice of the table from L2 through shared memory in
// double-buffered cp.async tiles of 64 triples; every warp multiplies its
// two m16 tiles of prefixes against each n8 sub-tile (ldmatrix, no ALU work
// on the B side), so the inner loop is 3 ldmatrix + 2W IMMA + 8 min.
#pragma once

#include "bz_kernels.cuh"

namespace bz {

// Byte stride of one row of a 0/1 table: 32 bytes per 32-column block plus
// 16, so 8 consecutive rows hit 8 distinct 16-byte bank groups (ldmatrix is
// conflict-free).
__host__ __device__ constexpr int tc_stride(int w) { return 32 * w + 16; }
constexpr int kTileRows = 64;    // triples per cp.async tile
constexpr int kTcThreads = 256;  // 8 warps, one prefix per lane

// +-1 bytes of the 4 bits of `word` at `shift`: bit 0 -> 0x01, bit 1 -> 0xff.
__device__ __forceinline__ uint32_t pm1_nibble(uint32_t word, int shift) {
  const uint32_t x = (word >> shift) & 0xFu;
  const uint32_t m = (x * 0x00204081u) & 0x01010101u;
  return m * 0xFEu + 0x01010101u;
}

// 0/1 bytes of the 4 bits of `word` at `shift`.
__device__ __forceinline__ uint32_t bit_nibble(uint32_t word, int shift) {
  return (((word >> shift) & 0xFu) * 0x00204081u) & 0x01010101u;
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

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;"); }

// ---------------------------------------------------------------------------
// Triple table: row index of {a < b < c} = C(k-1-a, 3) + (lex rank of (b, c)
// among the pairs of (a, k)).  Built on the device at load time; one block
// per (Gamma, a), threads over (pair, 32-column word).
template <int W>
__global__ void k_build_triples(const uint32_t* __restrict__ rows, uint8_t* __restrict__ trip,
                                int k, size_t gamma_stride_rows) {
  constexpr int WP = padded_words(W);
  constexpr int TS = tc_stride(W);
  const int j = blockIdx.y, a = blockIdx.x;
  if (a > k - 3) return;
  const uint32_t* R = rows + (size_t)j * k * WP;
  const long long base = (long long)(k - 1 - a) * (k - 2 - a) * (k - 3 - a) / 6;
  const int span = k - 1 - a;  // candidates for b, c
  const int npairs = span * (span - 1) / 2;
  uint8_t* out = trip + (size_t)j * gamma_stride_rows * TS;
  for (int t = threadIdx.x; t < npairs * W; t += blockDim.x) {
    const int pi = t / W, w = t - pi * W;
    // lex pair index pi -> (b, c) over (a, k)
    int b = a + 1, rem = pi;
    while (rem >= k - 1 - b) { rem -= k - 1 - b; ++b; }
    const int c = b + 1 + rem;
    const uint32_t v = R[a * WP + w] ^ R[b * WP + w] ^ R[c * WP + w];
    uint32_t* dst = reinterpret_cast<uint32_t*>(out + (size_t)(base + pi) * TS + 32 * w);
#pragma unroll
    for (int s = 0; s < 8; ++s) dst[s] = bit_nibble(v, 4 * s);
  }
}

template <int W>
__host__ __device__ inline size_t k3_smem_bytes(int m, int k, int ngroups) {
  const size_t base = (smem_base_bytes<W>(m, k, ngroups) + 127) & ~size_t(127);
  return base + 2 * (size_t)kTileRows * tc_stride(W) + 16;
}

template <int W>
__global__ void __launch_bounds__(kTcThreads, 2)
k3_round_gemm(const RoundArgs a, const uint8_t* __restrict__ trip, size_t gamma_stride_rows) {
  constexpr int TS = tc_stride(W);
  constexpr int WP = padded_words(W);
  constexpr int TILE_BYTES = kTileRows * TS;
  constexpr int N16 = TILE_BYTES / 16;
  extern __shared__ __align__(128) unsigned char smem[];
  const size_t bbase = (smem_base_bytes<W>(a.m, a.k, a.ngroups) + 127) & ~size_t(127);
  unsigned char* sbuf = smem + bbase;                      // 2 tiles
  int* sctl = reinterpret_cast<int*>(sbuf + 2 * TILE_BYTES);  // chunk broadcast
  uint32_t *srows, *spx;
  Group* sgroups;
  stage<W>(a, srows, spx, sgroups, smem);  // ends with __syncthreads
  const unsigned long long* sbinom = smem_binom<W>(smem, a);
  if (a.chain && threadIdx.x == 0 && blockIdx.x == 0) {
    // batched round: start from the U the previous round ended with (one
    // thread of the grid: atomics on one address serialise; blocks that read
    // the bound before it lands just see the looser start value)
    const int u = ((volatile const int*)a.chain)[0];
    for (int j = 0; j <= a.m; ++j) atomicMin(a.bound + j, u);
  }

  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int gid = lane >> 2, t0 = lane & 3;
  const int k = a.k, q = a.g - 4;
  volatile int* vbound = a.bound;
  const uint32_t sbuf_s = (uint32_t)__cvta_generic_to_shared(sbuf);
  // this lane's ldmatrix row inside an 8-row sub-tile and its 16-byte half
  const uint32_t ld_off = (uint32_t)((lane & 7) * TS + (lane >> 4) * 32 + ((lane >> 3) & 1) * 16);

  while (true) {
    if (tid == 0) {
      const unsigned long long c = atomicAdd(a.counter, 1ull);
      const unsigned long long chunk = c * (unsigned long long)a.nshards + a.shard;
      const bool stop = chunk >= a.nchunks || (a.exit_own && vbound[0] <= a.lower_prev);
      sctl[0] = stop ? -1 : find_group(sgroups, a.ngroups, chunk);
      reinterpret_cast<unsigned long long*>(sctl)[1] = chunk;
    }
    __syncthreads();
    const int gi = sctl[0];
    const unsigned long long chunk = reinterpret_cast<unsigned long long*>(sctl)[1];
    __syncthreads();
    if (gi < 0) break;

    const Group gr = sgroups[gi];
    const unsigned long long local = chunk - gr.chunk_begin;
    const unsigned long long pb = local / (unsigned long long)gr.ntb;
    const int tb = (int)(local - pb * (unsigned long long)gr.ntb);
    const unsigned long long bfirst = pb * (unsigned long long)kTcThreads * gr.ppl;
    const unsigned long long first = bfirst + (unsigned long long)tid * gr.ppl;
    long long cnt = 0;
    if (first < gr.nprefix) {
      const unsigned long long left = gr.nprefix - first;
      cnt = left < (unsigned long long)gr.ppl ? (long long)left : gr.ppl;
    }
    const unsigned long long bleft = gr.nprefix - bfirst;
    const long long maxcnt = bleft < (unsigned long long)gr.ppl ? (long long)bleft : gr.ppl;
    const uint32_t* R = srows + gr.gamma * k * WP;
    const uint32_t* PX = spx + gr.gamma * (k + 1) * px_stride(W);
    const int e0 = gr.ell + 1;
    const long long t = k - e0;
    const int slice = (int)(t * (t - 1) * (t - 2) / 6);  // triples above ell
    const int ntiles = (slice + kTileRows - 1) / kTileRows;
    const int tile_lo = tb * gr.tpc;
    const int tile_hi = min(ntiles, tile_lo + gr.tpc);
    const int nt = tile_hi - tile_lo;  // tiles per prefix step
    const uint8_t* tsrc = trip + (size_t)gr.gamma * gamma_stride_rows * TS;

    // lanes without prefixes duplicate the block's first prefix
    Walker<W> wk;
    wk.init(cnt > 0 ? first : bfirst, q, gr.ell, R, a.binom, sbinom);

    auto load_tile = [&](int tile, int buf) {
      const uint8_t* src = tsrc + (size_t)tile * TILE_BYTES;
      const uint32_t dst = sbuf_s + (uint32_t)(buf * TILE_BYTES);
      for (int i = tid; i < N16; i += kTcThreads) cp_async16(dst + 16 * i, src + 16 * i);
      cp_async_commit();
    };

    int best = INT_MAX;
    uint32_t A[2][W][4];
    int wrow[4];  // prefix weights of this thread's rows g, g+8, g+16, g+24
    // one tile per step: it stays resident for every prefix step
    const bool resident = nt == 1;
    long long s = 0;  // flat (prefix step, tile) index: buffer = s & 1
    const long long nsteps = maxcnt * nt;
    load_tile(tile_lo, 0);
    if (resident) {
      cp_async_wait0();
      __syncthreads();
    }
    for (long long p = 0; p < maxcnt; ++p) {
      if (p > 0 && p < cnt) wk.step(PX);  // exhausted lanes keep a duplicate
      // ---- A operand (+-1 prefix bytes) and C init (prefix weight)
      int wt = 0;
#pragma unroll
      for (int j = 0; j < W; ++j) wt += __popc(wk.acc[j]);
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
        wrow[2 * mt] = __shfl_sync(FULL, wt, r0);
        wrow[2 * mt + 1] = __shfl_sync(FULL, wt, r1);
      }
      // running minima of sum_j (1 - 2 P_j) S_j per row; w(P) is added once
      // per prefix step (min over columns commutes with the row constant)
      int rmin[4] = {INT_MAX / 2, INT_MAX / 2, INT_MAX / 2, INT_MAX / 2};

      for (int tile = tile_lo; tile < tile_hi; ++tile, ++s) {
        if (!resident) {
          // prefetch the next tile into the other buffer (freed by the sync
          // at the end of the previous step), then wait for this one
          if (s + 1 < nsteps) {
            load_tile(tile + 1 < tile_hi ? tile + 1 : tile_lo, (int)((s + 1) & 1));
            cp_async_wait1();
          } else {
            cp_async_wait0();
          }
          __syncthreads();
        }

        // ---- 8 n8 sub-tiles of this 64-triple tile
        const uint32_t tbuf = sbuf_s + (uint32_t)((resident ? 0 : (s & 1)) * TILE_BYTES) + ld_off;
        const int col0 = tile * kTileRows;
#pragma unroll 2
        for (int sub = 0; sub < kTileRows / 8; ++sub) {
          if (col0 + 8 * sub >= slice) break;
          const uint32_t addr = tbuf + (uint32_t)(sub * 8 * TS);
          uint32_t B[W][2];
#pragma unroll
          for (int j = 0; j + 1 < W; j += 2) {
            uint32_t r[4];
            ldsm_x4(r, addr + 32 * j);
            B[j][0] = r[0]; B[j][1] = r[1]; B[j + 1][0] = r[2]; B[j + 1][1] = r[3];
          }
          if constexpr (W & 1) ldsm_x2(B[W - 1][0], B[W - 1][1], addr + 32 * (W - 1));
          // two independent K-chains per m-tile (words [0, H) and [H, W))
          constexpr int H = (W + 1) / 2;
          const int zero4[4] = {0, 0, 0, 0};
          int d0[4], d1[4], e0v[4], e1v[4];
          imma16832(d0, A[0][0], B[0][0], B[0][1], zero4);
          imma16832(d1, A[1][0], B[0][0], B[0][1], zero4);
          if constexpr (W > 1) {
            imma16832(e0v, A[0][H], B[H][0], B[H][1], zero4);
            imma16832(e1v, A[1][H], B[H][0], B[H][1], zero4);
          }
#pragma unroll
          for (int j = 1; j < H; ++j) {
            imma16832(d0, A[0][j], B[j][0], B[j][1], d0);
            imma16832(d1, A[1][j], B[j][0], B[j][1], d1);
          }
#pragma unroll
          for (int j = H + 1; j < W; ++j) {
            imma16832(e0v, A[0][j], B[j][0], B[j][1], e0v);
            imma16832(e1v, A[1][j], B[j][0], B[j][1], e1v);
          }
          if constexpr (W == 1) {
#pragma unroll
            for (int i = 0; i < 4; ++i) { e0v[i] = 0; e1v[i] = 0; }
          }
          // c0,c1: row g (cols 2t0, 2t0+1); c2,c3: row g+8
          if (col0 + 8 * sub + 8 <= slice) {
            rmin[0] = min(rmin[0], min(d0[0] + e0v[0], d0[1] + e0v[1]));
            rmin[1] = min(rmin[1], min(d0[2] + e0v[2], d0[3] + e0v[3]));
            rmin[2] = min(rmin[2], min(d1[0] + e1v[0], d1[1] + e1v[1]));
            rmin[3] = min(rmin[3], min(d1[2] + e1v[2], d1[3] + e1v[3]));
          } else {
            const int col = col0 + 8 * sub + 2 * t0;
            const int m0 = col < slice ? 0 : 0x3fffffff;
            const int m1 = col + 1 < slice ? 0 : 0x3fffffff;
            rmin[0] = min(rmin[0], min(d0[0] + e0v[0] + m0, d0[1] + e0v[1] + m1));
            rmin[1] = min(rmin[1], min(d0[2] + e0v[2] + m0, d0[3] + e0v[3] + m1));
            rmin[2] = min(rmin[2], min(d1[0] + e1v[0] + m0, d1[1] + e1v[1] + m1));
            rmin[3] = min(rmin[3], min(d1[2] + e1v[2] + m0, d1[3] + e1v[3] + m1));
          }
        }
        if (!resident) __syncthreads();  // buffer (s & 1) is refilled at step s + 1
      }
      best = min(best, min(min(rmin[0] + wrow[0], rmin[1] + wrow[1]),
                           min(rmin[2] + wrow[2], rmin[3] + wrow[3])));
    }
    if (resident) __syncthreads();  // the next chunk reloads buffer 0

    // visited combinations: this chunk's prefixes x its triples
    const long long col_lo = (long long)tile_lo * kTileRows;
    const long long col_hi = min((long long)tile_hi * kTileRows, (long long)slice);
    const unsigned long long ncols = (unsigned long long)(col_hi - col_lo);
    int wbest = __reduce_min_sync(FULL, best);
    if (wbest < INT_MAX / 2) wbest += gamma_woff(a, gr.gamma);
    const unsigned tot = __reduce_add_sync(FULL, (unsigned)cnt);
    if (lane == 0) {
      if (wbest < vbound[1 + gr.gamma]) atomicMin(a.bound + 1 + gr.gamma, wbest);
      if (wbest < vbound[0]) atomicMin(a.bound, wbest);
      if (tot) atomicAdd(a.combos + gr.gamma, (unsigned long long)tot * ncols);
    }
  }
}

}  // namespace bz
