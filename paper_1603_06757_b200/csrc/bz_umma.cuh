// bz_umma.cuh -- K4: the round as an integer GEMM on the Blackwell 5th-gen
// tensor cores (tcgen05.mma kind::i8, accumulators in TMEM).
//
// Same algebra as K3 (bz_tc.cuh): w(P ^ S) = w(P) + sum_j (1 - 2 P_j) S_j,
// prefixes P as +-1 bytes (A, M = 128 rows), triples S as 0/1 bytes (B,
// N = 256 columns), K = the 32*W padded code columns (W MMAs of K = 32).
// A (Gamma, ell) group is the GEMM [C(ell,g-4) prefixes] x [C(k-1-ell,3)
// triples]; D[r][c] + w(P_r) is the weight of codeword (prefix r, triple c)
// and only its minimum is kept.
//
// One CTA per SM (persistent, static chunk striding), warp-specialised:
//   warps 0-3  producer + epilogue: thread r owns prefix row r of the tile.
//              It walks its prefixes (colex walker), writes its A row (+-1
//              bytes, UMMA K-major core-matrix layout) into one of two A
//              buffers, and later reads its row of the accumulator from TMEM
//              (tcgen05.ld 32x32b, warp w <-> TMEM lanes 32w..32w+31) and
//              min-reduces it.
//   warp 4     TMEM allocator + MMA issuer (one thread): per tile W x
//              tcgen05.mma into one of two 256-column accumulators, then
//              tcgen05.commit to the barriers that free the B stage and
//              publish the accumulator.
//   warp 5     loader (one thread): 1-D TMA bulk copies (cp.async.bulk) of
//              contiguous triple-table tiles into a ring of B stages.
// All synchronisation is mbarrier-based; every role walks the same chunk
// sequence, so the pipeline counters agree without extra signalling.
//
// Triple table (device-built at load time): all C(k,3) row triples in the
// K3 order (smallest element descending, then lex), stored directly in the
// UMMA SWIZZLE_NONE K-major canonical layout -- 8-row x 16-byte core
// matrices, the 2W 16-byte K chunks of an 8-row group contiguous -- so a
// 256-row tile is one contiguous byte range and the TMA copy lands it in
// exactly the layout the smem descriptor describes.
#pragma once

#include "bz_tc.cuh"

namespace bz {

constexpr int kUmmaM = 128;       // prefixes per A tile = producer threads
#ifndef BZ_K4_N
#define BZ_K4_N 256
#endif
#ifndef BZ_K4_MA
#define BZ_K4_MA 1
#endif
#ifndef BZ_K4_HOLDBACK
#define BZ_K4_HOLDBACK 0
#endif
constexpr bool kHoldBack = BZ_K4_HOLDBACK != 0;  // last MMA of a tile waits for the next tile's barriers
constexpr int kUmmaN = BZ_K4_N;   // triples per B tile
constexpr int kUmmaMA = BZ_K4_MA; // A tiles (consecutive prefix steps) per B tile
// warp roles: [0, E) epilogue (TMEM lane quarter = warp % 4, column slice
// = warp / 4), E MMA issuer + TMEM owner, E+1 TMA loader, E+2..E+5 producers
#ifndef BZ_K4_EPI_WARPS
#define BZ_K4_EPI_WARPS 8
#endif
constexpr int kK4EpiWarps = BZ_K4_EPI_WARPS;
constexpr int kK4EpiCols = kUmmaN / (kK4EpiWarps / 4);  // columns per epilogue warp and A tile
constexpr int kK4MmaWarp = kK4EpiWarps;
constexpr int kK4LoadWarp = kK4EpiWarps + 1;
constexpr int kK4ProdWarp0 = kK4EpiWarps + 2;
constexpr int kK4Threads = 32 * (kK4EpiWarps + 6);
constexpr int kTmemCols = 512;    // kAccBufs buffers x kUmmaMA accumulators x kUmmaN columns
constexpr int kAccBufs = kTmemCols / (kUmmaMA * kUmmaN);  // accumulator ring depth
constexpr int kMaxStages = 4;
constexpr int kChunkQ = 4;         // depth of the loader -> roles chunk queue
constexpr int kBarSlots = 4 + 2 * kMaxStages + 2 * kAccBufs + 2 * kChunkQ;
#ifndef BZ_K4_TMA_PIECES
#define BZ_K4_TMA_PIECES 1
#endif
constexpr int kTmaPieces = BZ_K4_TMA_PIECES;  // parallel bulk copies per B tile

__host__ __device__ constexpr int umma_tile_bytes_b(int w) { return kUmmaN * 32 * w; }
__host__ __device__ constexpr int umma_tile_bytes_a(int w) { return kUmmaM * 32 * w; }
// B-tile ring depth (shared memory: S x 8 KB x W plus 2 A tiles)
__host__ __device__ constexpr int umma_stages(int w) { return w <= 5 ? 4 : (w <= 6 ? 3 : 2); }

// byte offset of (row, 16-byte chunk kc) in a K-major no-swizzle UMMA tile
__host__ __device__ constexpr uint32_t umma_off(int row, int kc, int w) {
  return (uint32_t)((row >> 3) * (2 * w * 128) + kc * 128 + (row & 7) * 16);
}

// tcgen05 shared-memory matrix descriptor, SWIZZLE_NONE, K-major:
// LBO = distance between the two 16-byte K chunks of one MMA (128 B here),
// SBO = distance between 8-row core-matrix groups (2W * 128 B).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

// instruction descriptor: D = s32, A = s8, B = s8, both K-major, N, M
constexpr uint32_t kUmmaIdesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                ((uint32_t)(kUmmaN >> 3) << 17) |
                                ((uint32_t)(kUmmaM >> 4) << 24);

// ---- mbarrier / TMA / tcgen05 primitives
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
          bar),
      "r"(bytes)
      : "memory");
}
// wait for the phase of parity `parity` to complete; traps instead of
// hanging forever if the pipeline is ever wedged
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (unsigned long long spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (spin > (1ull << 26)) __trap();
  }
}
// Tight wait (loop inside PTX; labels are local to the braces): used on the
// MMA-issuing warp, where every cycle of handshake latency idles the pipe.
__device__ __forceinline__ void mbar_wait_fast(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tma_load_1d(uint32_t dst, const void* src, uint32_t bytes,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
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
// 32 columns of s32 accumulators as 16 registers of two s16 each (the low
// halves of adjacent columns; |values| <= 256 so nothing is lost)
__device__ __forceinline__ void tmem_ld16p(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
      "%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_regs16_after_wait(uint32_t* v) {
  asm volatile(""
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
               :
               : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// Ties 32 loaded registers to a point after tcgen05.wait::ld, so no use of
// them can be scheduled before the wait.
__device__ __forceinline__ void tmem_regs_after_wait(uint32_t* v) {
  asm volatile(""
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]),
                 "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                 "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]),
                 "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
}

// ---------------------------------------------------------------------------
// Triple table in UMMA layout: one block per (Gamma, a).
template <int W>
__global__ void k_build_triples_umma(const uint32_t* __restrict__ rows,
                                     uint8_t* __restrict__ trip, int k,
                                     size_t gamma_stride_rows) {
  constexpr int WP = padded_words(W);
  const int j = blockIdx.y, a = blockIdx.x;
  if (a > k - 3) return;
  const uint32_t* R = rows + (size_t)j * k * WP;
  const long long base = (long long)(k - 1 - a) * (k - 2 - a) * (k - 3 - a) / 6;
  const int span = k - 1 - a;
  const int npairs = span * (span - 1) / 2;
  uint8_t* out = trip + (size_t)j * gamma_stride_rows * 32 * W;
  for (int t = threadIdx.x; t < npairs * W; t += blockDim.x) {
    const int pi = t / W, w = t - pi * W;
    int b = a + 1, rem = pi;
    while (rem >= k - 1 - b) { rem -= k - 1 - b; ++b; }
    const int c = b + 1 + rem;
    const uint32_t v = R[a * WP + w] ^ R[b * WP + w] ^ R[c * WP + w];
    const long long row = base + pi;
    // 32 bytes of word w = K chunks 2w and 2w+1 of this row
    uint8_t* tile = out + (size_t)(row >> 3) * (2 * W * 128);
    uint4 lo, hi;
    lo.x = bit_nibble(v, 0);  lo.y = bit_nibble(v, 4);  lo.z = bit_nibble(v, 8);  lo.w = bit_nibble(v, 12);
    hi.x = bit_nibble(v, 16); hi.y = bit_nibble(v, 20); hi.z = bit_nibble(v, 24); hi.w = bit_nibble(v, 28);
    *reinterpret_cast<uint4*>(tile + (2 * w) * 128 + (row & 7) * 16) = lo;
    *reinterpret_cast<uint4*>(tile + (2 * w + 1) * 128 + (row & 7) * 16) = hi;
  }
}

template <int W>
__host__ __device__ inline size_t k4_smem_bytes(int m, int k, int ngroups) {
  size_t off = (smem_base_bytes<W>(m, k, ngroups) + 1023) & ~size_t(1023);
  off += (size_t)umma_stages(W) * umma_tile_bytes_b(W);
  off += 2 * (size_t)kUmmaMA * umma_tile_bytes_a(W);
  off += kBarSlots * 8 + 16;     // barriers + TMEM base
  off += 2 * kUmmaMA * kUmmaM * sizeof(int);  // prefix weights of the A buffers
  off += kChunkQ * sizeof(long long) + 16;    // chunk queue
  return off;
}

// Decoded chunk: identical on every role.
struct K4Chunk {
  Group gr;
  unsigned long long bfirst;
  long long maxcnt;
  int slice, tile_lo, tile_hi;
};

__device__ __forceinline__ K4Chunk k4_decode(const Group* sg, int ngroups,
                                             unsigned long long chunk, int k) {
  K4Chunk c;
  c.gr = sg[find_group(sg, ngroups, chunk)];
  const unsigned long long local = chunk - c.gr.chunk_begin;
  const unsigned long long pb = local / (unsigned long long)c.gr.ntb;
  const int tb = (int)(local - pb * (unsigned long long)c.gr.ntb);
  c.bfirst = pb * (unsigned long long)kUmmaM * c.gr.ppl;
  const unsigned long long bleft = c.gr.nprefix - c.bfirst;
  c.maxcnt = bleft < (unsigned long long)c.gr.ppl ? (long long)bleft : c.gr.ppl;
  const long long t = k - 1 - c.gr.ell;
  c.slice = (int)(t * (t - 1) * (t - 2) / 6);
  const int ntiles = (c.slice + kUmmaN - 1) / kUmmaN;
  c.tile_lo = tb * c.gr.tpc;
  c.tile_hi = min(ntiles, c.tile_lo + c.gr.tpc);
  return c;
}

template <int W>
__global__ void __launch_bounds__(kK4Threads, 1)
k4_round_umma(const RoundArgs a, const uint8_t* __restrict__ trip, size_t gamma_stride_rows) {
  constexpr int WP = padded_words(W);
  constexpr int S = umma_stages(W);
  constexpr uint32_t TB = umma_tile_bytes_b(W);
  constexpr uint32_t TA = umma_tile_bytes_a(W);
  extern __shared__ __align__(128) unsigned char smem[];
  const size_t base = (smem_base_bytes<W>(a.m, a.k, a.ngroups) + 1023) & ~size_t(1023);
  unsigned char* sB = smem + base;
  unsigned char* sA = sB + S * TB;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sA + 2 * kUmmaMA * TA);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + kBarSlots);
  int* s_wt = reinterpret_cast<int*>(s_tmem + 4);  // [2][kUmmaMA][kUmmaM] prefix weights
  volatile long long* s_q = reinterpret_cast<volatile long long*>(
      (reinterpret_cast<uintptr_t>(s_wt + 2 * kUmmaMA * kUmmaM) + 15) & ~uintptr_t(15));
  const uint32_t sB_s = (uint32_t)__cvta_generic_to_shared(sB);
  const uint32_t sA_s = (uint32_t)__cvta_generic_to_shared(sA);
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bars);
  // Rings: B stages (loader -> MMA: bfull; MMA commit -> loader: bempty),
  // accumulators (MMA commit -> epilogue: accfull; epilogue -> MMA:
  // accempty), A buffers (producers -> MMA, epilogue: afull; MMA commit +
  // epilogue -> producers: aempty).
  auto afull = [&](int i) { return bar_s + 8u * (0 + i); };
  auto aempty = [&](int i) { return bar_s + 8u * (2 + i); };
  auto bfull = [&](int i) { return bar_s + 8u * (4 + i); };
  auto bempty = [&](int i) { return bar_s + 8u * (4 + kMaxStages + i); };
  auto accfull = [&](int i) { return bar_s + 8u * (4 + 2 * kMaxStages + i); };
  auto accempty = [&](int i) { return bar_s + 8u * (4 + 2 * kMaxStages + kAccBufs + i); };
  // chunk queue: the loader draws chunks from the round's global counter
  // (dynamic balance across CTAs) and publishes them to every other role
  auto qfull = [&](int i) { return bar_s + 8u * (4 + 2 * kMaxStages + 2 * kAccBufs + i); };
  auto qempty = [&](int i) {
    return bar_s + 8u * (4 + 2 * kMaxStages + 2 * kAccBufs + kChunkQ + i);
  };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(bfull(i), 1); mbar_init(bempty(i), 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(afull(i), kUmmaM);               // every producer thread
      mbar_init(aempty(i), 1 + kK4EpiWarps);     // MMA commit + each epilogue warp
    }
    for (int i = 0; i < kAccBufs; ++i) {
      mbar_init(accfull(i), 1);                  // MMA commit
      mbar_init(accempty(i), kK4EpiWarps);       // each epilogue warp
    }
    for (int i = 0; i < kChunkQ; ++i) {
      mbar_init(qfull(i), 1);                    // loader
      mbar_init(qempty(i), kK4EpiWarps + 5);     // epilogue, producer and MMA warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async();
  }
  if (warp == kK4MmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(s_tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  uint32_t *srows, *spx;
  Group* sgroups;
  tc_fence_before();
  stage<W>(a, srows, spx, sgroups, smem);  // ends with __syncthreads
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const int k = a.k, q = a.g - 4;
  const unsigned FULL = 0xffffffffu;

  if (warp < kK4EpiWarps) {
    // ================= epilogue: warp e reads TMEM lanes 32(e%4).. (rows),
    // columns [kK4EpiCols*(e/4), +kK4EpiCols) of each accumulator
    const int quarter = warp & 3, slice_id = warp >> 2;
    const int r = 32 * quarter + lane;
    uint32_t grp = 0, tcount = 0;
    for (uint32_t qi = 0;; ++qi) {
      const int qs = qi % kChunkQ;
      mbar_wait(qfull(qs), (qi / kChunkQ) & 1);
      const long long qchunk = s_q[qs];
      __syncwarp();
      if (lane == 0) mbar_arrive(qempty(qs));
      if (qchunk < 0) break;
      const unsigned long long chunk = (unsigned long long)qchunk;
      const K4Chunk c = k4_decode(sgroups, a.ngroups, chunk, k);
      int best = INT_MAX;
      for (long long p = 0; p < c.maxcnt; p += kUmmaMA, ++grp) {
        const int ab = grp & 1;
        mbar_wait(afull(ab), (grp >> 1) & 1);
        int wt[kUmmaMA];
#pragma unroll
        for (int j = 0; j < kUmmaMA; ++j) wt[j] = s_wt[(ab * kUmmaMA + j) * kUmmaM + r];
        __syncwarp();
        if (lane == 0) mbar_arrive(aempty(ab));
        int rmin[kUmmaMA];
#pragma unroll
        for (int j = 0; j < kUmmaMA; ++j) rmin[j] = INT_MAX / 2;
        for (int t = c.tile_lo; t < c.tile_hi; ++t, ++tcount) {
          const int buf = tcount % kAccBufs;
          mbar_wait(accfull(buf), (tcount / kAccBufs) & 1);
          tc_fence_after();
          if (a.trace && blockIdx.x == 0 && warp == 0 && lane == 0 && tcount < 256)
            a.trace[2 * 256 + tcount] = clock64();
          if (a.trace && blockIdx.x == 0 && warp == kK4EpiWarps - 1 && lane == 0 && tcount < 256)
            a.trace[7 * 256 + tcount] = clock64();
          const int lim = min(kUmmaN, c.slice - t * kUmmaN) - kK4EpiCols * slice_id;
          const uint32_t tb = tmem + ((uint32_t)(32 * quarter) << 16) +
                              (uint32_t)(buf * kUmmaMA * kUmmaN + kK4EpiCols * slice_id);
          // kK4EpiCols columns as packed s16 pairs: 3-input SIMD minima
          constexpr int NP = kK4EpiCols / 2;
          uint32_t v[kUmmaMA][NP];
          if (a.debug & 1) {
            __syncwarp();
            if (lane == 0) mbar_arrive(accempty(buf));
            continue;
          }
#pragma unroll
          for (int j = 0; j < kUmmaMA; ++j)
#pragma unroll
            for (int cc = 0; cc < kK4EpiCols / 32; ++cc)
              tmem_ld16p(tb + j * kUmmaN + 32 * cc, &v[j][16 * cc]);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < kUmmaMA; ++j)
#pragma unroll
            for (int cc = 0; cc < kK4EpiCols / 32; ++cc) tmem_regs16_after_wait(&v[j][16 * cc]);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(accempty(buf));  // accumulators are in registers
          if (a.trace && blockIdx.x == 0 && warp == 0 && lane == 0 && tcount < 256)
            a.trace[3 * 256 + tcount] = clock64();
#pragma unroll
          for (int j = 0; j < kUmmaMA; ++j) {
            if (lim < kK4EpiCols) {
#pragma unroll
              for (int i = 0; i < NP; ++i) {
                if (2 * i >= lim) v[j][i] = (v[j][i] & 0xffff0000u) | 0x00007fffu;
                if (2 * i + 1 >= lim) v[j][i] = (v[j][i] & 0x0000ffffu) | 0x7fff0000u;
              }
            }
            // packed s16 pairs: 3-input SIMD minima down to one register
            uint32_t m = __vimin3_s16x2(v[j][0], v[j][1], v[j][2]);
#pragma unroll
            for (int i = 3; i + 1 < NP; i += 2) m = __vimin3_s16x2(m, v[j][i], v[j][i + 1]);
            if (NP % 2 == 0) m = __vmins2(m, v[j][NP - 1]);
            const int lo = (int)(short)(m & 0xffffu), hi = (int)(short)(m >> 16);
            rmin[j] = min(rmin[j], min(lo, hi));
          }
        }
#pragma unroll
        for (int j = 0; j < kUmmaMA; ++j) best = min(best, rmin[j] + wt[j]);
      }
      const int wbest = __reduce_min_sync(FULL, best);
      if (lane == 0) {
        volatile int* vb = a.bound;
        if (wbest < vb[1 + c.gr.gamma]) atomicMin(a.bound + 1 + c.gr.gamma, wbest);
        if (wbest < vb[0]) atomicMin(a.bound, wbest);
      }
    }
  } else if (warp >= kK4ProdWarp0) {
    // ================= producers: thread r walks prefix row r
    const int r = tid - 32 * kK4ProdWarp0;
    uint32_t grp = 0;
    for (uint32_t qi = 0;; ++qi) {
      const int qs = qi % kChunkQ;
      mbar_wait(qfull(qs), (qi / kChunkQ) & 1);
      const long long qchunk = s_q[qs];
      __syncwarp();
      if (lane == 0) mbar_arrive(qempty(qs));
      if (qchunk < 0) break;
      const unsigned long long chunk = (unsigned long long)qchunk;
      const K4Chunk c = k4_decode(sgroups, a.ngroups, chunk, k);
      const unsigned long long first = c.bfirst + (unsigned long long)r * c.gr.ppl;
      long long cnt = 0;
      if (first < c.gr.nprefix) {
        const unsigned long long left = c.gr.nprefix - first;
        cnt = left < (unsigned long long)c.gr.ppl ? (long long)left : c.gr.ppl;
      }
      const uint32_t* R = srows + c.gr.gamma * k * WP;
      const uint32_t* PX = spx + c.gr.gamma * (k + 1) * px_stride(W);
      Walker<W> wk;
      // rows without prefixes duplicate the block's first prefix
      wk.init(cnt > 0 ? first : c.bfirst, q, c.gr.ell, R, a.binom);
      for (long long p = 0; p < c.maxcnt; p += kUmmaMA, ++grp) {
        const int ab = grp & 1;
        mbar_wait(aempty(ab), ((grp >> 1) & 1) ^ 1);
#pragma unroll 1
        for (int j = 0; j < kUmmaMA; ++j) {
          // step j of the group; past this row's range the last prefix repeats
          if (p + j > 0 && p + j < cnt) wk.step(PX);
          unsigned char* dst = sA + (ab * kUmmaMA + j) * TA;
          int wt = 0;
#pragma unroll
          for (int jj = 0; jj < W; ++jj) {
            uint4 lo, hi;
            const uint32_t v = wk.acc[jj];
            wt += __popc(v);
            lo.x = pm1_nibble(v, 0);  lo.y = pm1_nibble(v, 4);
            lo.z = pm1_nibble(v, 8);  lo.w = pm1_nibble(v, 12);
            hi.x = pm1_nibble(v, 16); hi.y = pm1_nibble(v, 20);
            hi.z = pm1_nibble(v, 24); hi.w = pm1_nibble(v, 28);
            *reinterpret_cast<uint4*>(dst + umma_off(r, 2 * jj, W)) = lo;
            *reinterpret_cast<uint4*>(dst + umma_off(r, 2 * jj + 1, W)) = hi;
          }
          s_wt[(ab * kUmmaMA + j) * kUmmaM + r] = wt;
        }
        fence_proxy_async();  // generic-proxy writes -> tensor-core reads
        mbar_arrive(afull(ab));
      }
      // visited combinations of this chunk
      const unsigned tot = __reduce_add_sync(FULL, (unsigned)cnt);
      if (lane == 0 && tot) {
        const long long cols = min((long long)c.tile_hi * kUmmaN, (long long)c.slice) -
                               (long long)c.tile_lo * kUmmaN;
        atomicAdd(a.combos + c.gr.gamma, (unsigned long long)tot * (unsigned long long)cols);
      }
    }
  } else if (warp == kK4MmaWarp) {
    // ================= MMA issuer
    // tcgen05.mma issue blocks while the tensor pipe is busy, so the waits
    // for tile t+1 are placed *before* the last MMA of tile t: the pipe then
    // still holds queued work while this thread does its barrier handshakes.
    // the whole warp runs the loop (warp-uniform values stay in uniform
    // registers); one elected lane issues the MMAs and commits
    {
      const uint64_t a_desc0 = umma_desc(sA_s, 128, 2 * W * 128);
      const uint64_t b_desc0 = umma_desc(sB_s, 128, 2 * W * 128);
      uint32_t grp = 0, tcount = 0, bcount = 0;
      // the held-back last MMA of the previous tile and its commits
      bool pend = false;
      uint32_t pd = 0, pstg = 0, pbuf = 0, pab = 0;
      uint64_t pad = 0, pbd = 0;
      bool pend_group_end = false;
      auto flush = [&]() {
        if (!pend) return;
        if (elect_one()) {
          if (!(a.debug & 4)) umma_i8(pd, pad, pbd, kUmmaIdesc, W > 1 ? 1u : 0u);
          umma_commit(bempty(pstg));
          umma_commit(accfull(pbuf));
          if (pend_group_end) umma_commit(aempty(pab));
        }
        __syncwarp();
        pend = false;
      };
      for (uint32_t qi = 0;; ++qi) {
        const int qs = qi % kChunkQ;
        mbar_wait_fast(qfull(qs), (qi / kChunkQ) & 1);
        const long long qchunk = s_q[qs];
        __syncwarp();
        if (lane == 0) mbar_arrive(qempty(qs));
        if (qchunk < 0) break;
        const unsigned long long chunk = (unsigned long long)qchunk;
        const K4Chunk c = k4_decode(sgroups, a.ngroups, chunk, k);
        for (long long p = 0; p < c.maxcnt; p += kUmmaMA, ++grp) {
          const int ab = grp & 1;
          mbar_wait_fast(afull(ab), (grp >> 1) & 1);
          for (int t = c.tile_lo; t < c.tile_hi; ++t, ++tcount, ++bcount) {
            const int stg = bcount % S;
            const int buf = tcount % kAccBufs;
            if (a.trace && blockIdx.x == 0 && lane == 0 && tcount < 256)
              a.trace[5 * 256 + tcount] = clock64();
            mbar_wait_fast(accempty(buf), ((tcount / kAccBufs) & 1) ^ 1);
            if (a.trace && blockIdx.x == 0 && lane == 0 && tcount < 256)
              a.trace[6 * 256 + tcount] = clock64();
            mbar_wait_fast(bfull(stg), (bcount / S) & 1);
            tc_fence_after();
            flush();  // previous tile's last MMA + commits
            if (a.trace && blockIdx.x == 0 && lane == 0 && tcount < 256)
              a.trace[1 * 256 + tcount] = clock64();
            // K step kb advances both start addresses by 256 B (16 in the
            // 16-byte-granular address field)
            const uint64_t bd0 = b_desc0 + (uint64_t)(stg * (TB >> 4));
            if (!(a.debug & 4)) {
              if (elect_one()) {
#pragma unroll
                for (int j = 0; j < kUmmaMA; ++j) {
                  const uint32_t dj = tmem + (uint32_t)((buf * kUmmaMA + j) * kUmmaN);
                  const uint64_t adj = a_desc0 + (uint64_t)((ab * kUmmaMA + j) * (TA >> 4));
#pragma unroll
                  for (int kb = 0; kb < W; ++kb) {
                    if (kHoldBack && j == kUmmaMA - 1 && kb == W - 1) break;  // held back
                    umma_i8(dj, adj + 16u * kb, bd0 + 16u * kb, kUmmaIdesc, kb > 0 ? 1u : 0u);
                  }
                }
              }
              __syncwarp();
            }
            const uint32_t d = tmem + (uint32_t)((buf * kUmmaMA + kUmmaMA - 1) * kUmmaN);
            const uint64_t ad0 = a_desc0 + (uint64_t)((ab * kUmmaMA + kUmmaMA - 1) * (TA >> 4));
            pend = true;
            if (!kHoldBack) {  // everything issued: commit right away
              if (elect_one()) {
                umma_commit(bempty(stg));
                umma_commit(accfull(buf));
                if (t + 1 == c.tile_hi) umma_commit(aempty(ab));
              }
              __syncwarp();
              pend = false;
            }
            pd = d;
            pad = ad0 + 16u * (W - 1);
            pbd = bd0 + 16u * (W - 1);
            pstg = stg;
            pbuf = buf;
            pab = ab;
            pend_group_end = (t + 1 == c.tile_hi);
            if (a.trace && blockIdx.x == 0 && lane == 0 && tcount < 256)
              a.trace[4 * 256 + tcount] = clock64();
          }
        }
      }
      flush();
    }
    __syncwarp();
  } else {
    // ================= loader: TMA bulk copies of triple tiles
    if (lane == 0) {
      uint32_t bcount = 0;
      volatile int* vb = a.bound;
      for (uint32_t qi = 0;; ++qi) {
        const int qs = qi % kChunkQ;
        mbar_wait(qempty(qs), ((qi / kChunkQ) & 1) ^ 1);
        // next chunk of this shard, or -1 (done, or U reached L_prev)
        const unsigned long long cidx = atomicAdd(a.counter, 1ull);
        const unsigned long long ch = cidx * (unsigned long long)a.nshards + a.shard;
        const long long qchunk = (ch < a.nchunks && vb[0] > a.lower_prev) ? (long long)ch : -1;
        s_q[qs] = qchunk;
        mbar_arrive(qfull(qs));
        if (qchunk < 0) break;
        const unsigned long long chunk = (unsigned long long)qchunk;
        const K4Chunk c = k4_decode(sgroups, a.ngroups, chunk, k);
        const uint8_t* tsrc = trip + (size_t)c.gr.gamma * gamma_stride_rows * 32 * W;
        for (long long p = 0; p < c.maxcnt; p += kUmmaMA) {
          for (int t = c.tile_lo; t < c.tile_hi; ++t, ++bcount) {
            const int stg = bcount % S;
            mbar_wait(bempty(stg), ((bcount / S) & 1) ^ 1);
            if (a.trace && blockIdx.x == 0 && bcount < 256) a.trace[0 * 256 + bcount] = clock64();
            // only the rows this tile needs (8-row granularity); the rest of
            // the stage keeps stale rows whose columns the epilogue masks
            const int valid = min(kUmmaN, c.slice - t * kUmmaN);
            const uint32_t bytes = (uint32_t)((valid + 7) / 8) * (2 * W * 128);
            if (a.debug & 2) {
              mbar_arrive(bfull(stg));
            } else {
              mbar_arrive_tx(bfull(stg), bytes);
              // a few bulk copies in flight per tile (one per 8-row groups
              // slice) keep more of the L2->SMEM path busy
              const uint32_t groups8 = (uint32_t)((valid + 7) / 8);
              const uint32_t per = (groups8 + kTmaPieces - 1) / kTmaPieces;
              for (uint32_t g0 = 0; g0 < groups8; g0 += per) {
                const uint32_t gn = min(per, groups8 - g0);
                const uint32_t off = g0 * (2 * W * 128);
                tma_load_1d(sB_s + stg * TB + off, tsrc + (size_t)t * TB + off,
                            gn * (2 * W * 128), bfull(stg));
              }
            }
          }
        }
      }
    }
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kK4MmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// tcgen05 kind::i8 throughput probe (roofline denominator of K4): one CTA per
// SM issues `iters` back-to-back M=128 x N x K=32 MMAs from shared memory
// into TMEM (operand contents are irrelevant), then waits for completion.
template <int N>
__global__ void __launch_bounds__(128, 1) peak_umma_i8(int iters, long long* clk) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5;
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
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint64_t ad = umma_desc(base, 128, 256);
    const uint64_t bd = umma_desc(base + 128 * 32, 128, 256);
    t0 = clock64();
    for (int i = 0; i < iters; ++i)
      umma_i8(tmem + (uint32_t)((i & 1) * N), ad, bd, idesc, (i & 2) ? 1u : 0u);
    umma_commit(bar_s);
    mbar_wait(bar_s, 0);
    t1 = clock64();
    clk[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace bz
