// bz_umma.cuh -- K4 / K5: the round as a GEMM on the Blackwell 5th-gen
// tensor cores (tcgen05.mma, accumulators in TMEM).
//
// Same algebra as K3 (bz_tc.cuh): w(P ^ S) = w(P) + sum_j (1 - 2 P_j) S_j,
// prefixes P as +-1 (A, M = 128 rows), suffixes S as 0/1 (B, N columns), K =
// the padded stored code columns.  A (Gamma, ell, D) group is the GEMM
// [C(ell, g-1-D) prefixes] x [its suffix slice]; D[r][c] + w(P_r) is the
// weight of codeword (prefix r, suffix c) and only its minimum is kept.
//
//   K4  kind::i8: s8 operands (32 K per byte-pair chunk), N = 256, s32
//       accumulators read back as packed s16 pairs.  W MMAs of K = 32.
//       Triple table only (depth 3).
//   K5  kind::mxf4 with unit block scales: +-1 and 0/1 are exact e2m1
//       values, so the products and their fp32 sums are the same integers,
//       at twice the i8 MAC rate from half the operand bytes.  N = 240
//       (2 x 240 accumulator columns + 32 scale-factor columns fill TMEM),
//       ceil(W/2) MMAs of K = 64; suffix tables of depth 3, 4 and 5 (host
//       level plan).  The accumulators start at 1.5 * 2^23 (on the K padding
//       chunk for odd W, else one extra MMA), so their low 16 bits are the
//       integer result and the epilogue reads packed s16 pairs.
//
// One persistent CTA per SM, warp-specialised, every hand-off an mbarrier
// (K4Roles):
//   warps [0, E)        epilogue: warp e reads TMEM lanes 32(e%4).. (its
//                       prefix rows) of one column slice of each accumulator
//                       (tcgen05.ld), releases the buffer, min-reduces.
//   warps E, E+1        MMA issuers (one elected lane each): issuer b owns
//                       accumulator b and issues every other tile, then
//                       tcgen05.commit to the barriers that free the B stage,
//                       publish the accumulator and free the A tile.  Two
//                       issuers hide each other's handshakes (a tcgen05.mma
//                       issue stalls while the pipe is busy).
//   warp E+2            loader: draws chunks from the round's global counter,
//                       publishes them to the other roles through a small
//                       smem queue, and streams each chunk's suffix tiles
//                       with 1-D TMA bulk copies into a ring of B stages.
//   warps E+3 .. E+6    producers: thread r walks prefix row r (colex
//                       walker) and writes its A row into an A ring.
//
// Suffix tables (device-built on first use): every D-subset of the rows
// above a floor, smallest element descending, stored directly in the UMMA
// SWIZZLE_NONE K-major canonical layout -- 8-row x 16-byte core matrices,
// the K chunks of an 8-row group contiguous -- so a tile is one contiguous
// byte range and the TMA copy lands it in exactly the layout the smem
// descriptor describes.
#pragma once

#include <type_traits>

#include "bz_tc.cuh"

namespace bz {

constexpr int kUmmaM = 128;       // prefixes per A tile = producer threads
#ifndef BZ_K4_N
#define BZ_K4_N 256
#endif
#ifndef BZ_K4_MA
#define BZ_K4_MA 1
#endif
#ifndef BZ_K4_EPI_WARPS
#define BZ_K4_EPI_WARPS 8
#endif
#ifndef BZ_K5_EPI_WARPS
#define BZ_K5_EPI_WARPS 8
#endif
#ifndef BZ_K5_BUFS
#define BZ_K5_BUFS 2
#endif
#ifndef BZ_K5_SPLIT
#define BZ_K5_SPLIT 1
#endif
#ifndef BZ_K5Q_SPLIT
#define BZ_K5Q_SPLIT 1  // K5q: accumulator column halves with their own barriers
#endif
#ifndef BZ_K5_LEAN
#define BZ_K5_LEAN 1  // K5q / K5f epilogue: the lean tile loop (0: the general one)
#endif
#ifndef BZ_GBOUND_THR
#define BZ_GBOUND_THR 1  // K5q / K5w thresholds also follow the other ranks' minima
#endif
#ifndef BZ_K5_LD64
#define BZ_K5_LD64 1  // lean epilogue: one 64-column packed load per tile
#endif
#ifndef BZ_K5F_SPLIT
#define BZ_K5F_SPLIT 1  // K5f: accumulator column halves with their own barriers
#endif
#ifndef BZ_K5_EPI_GROUPS
#define BZ_K5_EPI_GROUPS 1
#endif
#ifndef BZ_K5_NOFENCE
#define BZ_K5_NOFENCE 0  // timing experiment only: drops the per-tile tcgen05 fences
#endif
#ifndef BZ_K5_EVEN_F32
#define BZ_K5_EVEN_F32 0  // K5, even W: f32 accumulators instead of the offset MMA
#endif
#ifndef BZ_K5_MAGIC
#define BZ_K5_MAGIC 1
#endif
// K5p geometry: accumulator buffers (= MMA issuer warps; N = 480 / BUFS
// columns each) and epilogue warps
#ifndef BZ_K5P_BUFS
#define BZ_K5P_BUFS 2
#endif
#ifndef BZ_K5P_EPI_WARPS
#define BZ_K5P_EPI_WARPS 16
#endif
#ifndef BZ_K5P_EPI_GROUPS
#define BZ_K5P_EPI_GROUPS 1  // K5q: epilogue groups taking alternate tiles
#endif
// K5 accumulators start at 1.5 * 2^23 (one extra MMA per part from two tiny
// constant operands): the fp32 sum then carries the integer dot product in
// its low 16 bits, so the epilogue reads them with .pack::16b (half the
// register traffic) and reduces packed s16 pairs, like K4.
// For odd W the offset rides on the zero K padding chunk instead: the last
// real MMA's padding block gets A = 1.5, B = 1.0 (every table row carries
// the extra chunk) and an A scale of 2^23 for that block only, so no extra
// MMA is issued.
constexpr bool kK5Magic = BZ_K5_MAGIC != 0;
constexpr int kSfColMagic = 496;  // ue8m0 2^23 scale columns of the magic MMA
constexpr int kSfColPad = 504;    // A scales (1, 2^23): block 0 = chunk W-1, block 1 = pad
constexpr uint32_t kMagicBytes = 512;  // A and B magic operands (K = 64, SBO = 0)
constexpr int kUmmaN = BZ_K4_N;   // K4 triples per B tile
constexpr int kUmmaMA = BZ_K4_MA; // K4 A tiles (consecutive prefix steps) per B tile
constexpr int kTmemCols = 512;    // accumulators (+ K5 scale factors)
constexpr int kSfCol = 480;       // K5 scale-factor columns [480, 512)
constexpr int kUmmaN4 = kSfCol / BZ_K5_BUFS;  // K5 triples per B tile (240 / 120)
constexpr int kUmmaN4P = (kSfCol / BZ_K5P_BUFS) & ~15;  // K5p/K5q accumulator columns per tile
constexpr int kMaxStages = 8;
constexpr int kMaxAcc = 8;
constexpr int kMaxABuf = 4;
constexpr int kChunkQ = 4;         // depth of the loader -> roles chunk queue
constexpr int kBndCache = 64;       // K5q: per-CTA cache of the per-Gamma bounds (bnd_publish)
constexpr int kBndPerRound = kBndCache / 4;  // ... for Gammas < 16 of each fused round
constexpr int kBarSlots = 2 * kMaxABuf + 2 * kMaxStages + 2 * kMaxAcc + 2 * kChunkQ;

// Warp roles of K4 (F4 = false) / K5 (F4 = true):
//   [0, E)            epilogue
//   [E, E + ACC)      MMA issuers: warp E + b owns accumulator buffer b and
//                     issues every tile t with t % ACC == b (a second issuer
//                     hides one issuer's barrier handshakes behind the other's
//                     MMAs: tcgen05.mma issue stalls while the pipe is busy)
//   E + ACC           loader
//   E + ACC + 1 .. 4  producers (thread r <-> prefix row r)
template <bool F4, int CW = 1>
struct K4Roles {
  static constexpr int E = CW > 1 ? BZ_K5P_EPI_WARPS : (F4 ? BZ_K5_EPI_WARPS : BZ_K4_EPI_WARPS);
  static constexpr int ACC = CW > 1 ? BZ_K5P_BUFS : (F4 ? BZ_K5_BUFS : kTmemCols / (kUmmaMA * kUmmaN));
  static constexpr int MMA0 = E;
  static constexpr int LOAD = E + ACC;
  static constexpr int PROD0 = E + ACC + 1;
  static constexpr int THREADS = 32 * (E + ACC + 5);
  // column parts of each accumulator with their own full/empty barriers:
  // the epilogue drains part 0 while the MMAs of part 1 still run, and the
  // next tile's part-0 MMAs start as soon as part 0 is drained
  static constexpr int SPLIT =
      CW == 4 ? BZ_K5Q_SPLIT : CW == 6 ? BZ_K5F_SPLIT : (CW > 1 ? 1 : (F4 ? BZ_K5_SPLIT : 1));
  // epilogue groups: group q drains the tiles t with t % EGRP == q (each
  // group covers the whole accumulator), so a group has EGRP tile periods
  // for its loads and reductions while the other groups take the tiles in
  // between
  static constexpr int EGRP = CW == 4 ? BZ_K5P_EPI_GROUPS : (CW > 1 ? 1 : (F4 ? BZ_K5_EPI_GROUPS : 1));
  static constexpr int EW = E / EGRP;  // warps per group
  static_assert(E % 4 == 0 && ACC * SPLIT <= kMaxAcc && EW % 4 == 0 && (EW / 4) % SPLIT == 0 &&
                    ACC % EGRP == 0,
                "roles");
};

template <bool F4, int CW = 1> __host__ __device__ constexpr int k4_n() {
  return CW > 1 ? kUmmaN4P : (F4 ? kUmmaN4 : kUmmaN);
}
// bytes per table (B) row: K4 one byte per column, K5 one nibble
// K5 with the padding-chunk offset (odd W): tables carry the pad chunk
__host__ __device__ constexpr bool k5_padmagic(int w) { return kK5Magic && (w & 1); }
// (K5f, form 6: W chunks, the last one half data, half offset pattern)
template <bool F4> __host__ __device__ constexpr int k4_row_bytes(int w, int cw = 1) {
  return F4 ? 16 * (cw != 6 && k5_padmagic(w) ? w + 1 : w) : 32 * w;
}
// 16-byte K chunks per A row (K5 pads to whole K = 64 MMAs; K5p / K5t with
// CW codewords per accumulator column carry CW offset chunks after the W
// data chunks)
// codewords per accumulator column of kernel form CW (1 = K5, 2 = K5p,
// 3 = K5t, 4 = K5q: two codewords as bytes, 5 = K5w: two codewords as 11-bit
// fields, for wide rows, 6 = K5f: K5q's bytes from folded MMAs, see k5f_ok)
__host__ __device__ constexpr int k5_ncw(int cw) { return (cw >= 4 && cw <= 6) ? 2 : cw; }
// K5w A row: the data chunks padded to whole K = 64 MMAs (a zero chunk for
// odd W meets the table's offset chunk), then the offset chunks R, Ca, Cb
__host__ __device__ constexpr int k5w_data_chunks(int w) { return 2 * ((w + 1) / 2); }
template <bool F4, int CW = 1> __host__ __device__ constexpr int k4_a_chunks(int w) {
  return CW == 5 ? k5w_data_chunks(w) + 3
         : CW == 6 ? w + 1  // K5f: W - 1 whole chunks, then the tail chunk once per part
                   : (CW > 1 ? w + k5_ncw(CW) : (F4 ? 2 * ((w + 1) / 2) : 2 * w));
}
// MMAs per tile (per half for K5p)
template <bool F4> __host__ __device__ constexpr int k4_passes(int w) { return k4_a_chunks<F4>(w) / 2; }
// table rows per B tile: K5p pairs two rows per accumulator column
template <bool F4, int CW = 1> __host__ __device__ constexpr int k4_tile_rows() {
  return k5_ncw(CW) * k4_n<F4, CW>();
}
template <bool F4, int CW = 1> __host__ __device__ constexpr uint32_t k4_tile_b(int w) {
  return (uint32_t)(k4_tile_rows<F4, CW>() * k4_row_bytes<F4>(w, CW));
}
template <bool F4, int CW = 1> __host__ __device__ constexpr uint32_t k4_tile_a(int w) {
  return (uint32_t)(kUmmaM * 16 * k4_a_chunks<F4, CW>(w));
}
// A-tile ring depth (producers run that many prefix steps ahead; K5w's wide
// A rows and B tiles leave room for two)
#ifndef BZ_K5W_ABUFS
#define BZ_K5W_ABUFS 2
#endif
#ifndef BZ_K5W_STAGE_BYTES
#define BZ_K5W_STAGE_BYTES 140000
#endif
template <bool F4, int CW = 1> __host__ __device__ constexpr int k4_abufs(int w) {
  return CW == 5 ? BZ_K5W_ABUFS : (F4 && w <= 6 ? 4 : 2);
}
// B-tile ring depth: K5 ~136 KB of stages, K4 4 x 40 KB at W = 5
#ifndef BZ_K5P_STAGE_BYTES
#define BZ_K5P_STAGE_BYTES 160000
#endif
template <bool F4, int CW = 1> __host__ __device__ constexpr int k4_stages(int w) {
  if (CW == 5) {
    const int s = BZ_K5W_STAGE_BYTES / (int)k4_tile_b<true, CW>(w);
    return s < 2 ? 2 : (s > kMaxStages ? kMaxStages : s);
  }
  return F4 ? ((CW > 1 ? BZ_K5P_STAGE_BYTES : 136000) / (int)k4_tile_b<true, CW>(w) < kMaxStages
                   ? (CW > 1 ? BZ_K5P_STAGE_BYTES : 136000) / (int)k4_tile_b<true, CW>(w)
                   : kMaxStages)
            : (w <= 5 ? 4 : (w <= 6 ? 3 : 2));
}

// byte offset of (row, 16-byte chunk kc) in a K-major no-swizzle tile of
// `chunks` chunks per row
__host__ __device__ constexpr uint32_t umma_off_c(int row, int kc, int chunks) {
  return (uint32_t)((row >> 3) * (chunks * 128) + kc * 128 + (row & 7) * 16);
}

// K5 operand encoding of one 32-bit code word into 16 bytes = 32 e2m1
// nibbles, as 4 words: nibble q of word j holds bit 4q + j (a fixed K
// permutation, the same on both operands, so dot products are unchanged).
// B: 0 / 1.0 (0x2); A: +1.0 (0x2) for a 0 bit, -1.0 (0xA) for a 1 bit.
__host__ __device__ __forceinline__ uint4 e2m1_bits01(uint32_t v) {
  return make_uint4((v << 1) & 0x22222222u, v & 0x22222222u, (v >> 1) & 0x22222222u,
                    (v >> 2) & 0x22222222u);
}
__host__ __device__ __forceinline__ uint4 e2m1_pm1(uint32_t v) {
  return make_uint4(((v << 3) & 0x88888888u) | 0x22222222u, ((v << 2) & 0x88888888u) | 0x22222222u,
                    ((v << 1) & 0x88888888u) | 0x22222222u, (v & 0x88888888u) | 0x22222222u);
}

// K5 table offset chunk (the extra K chunk of every table row for odd W):
// in each 16-element block (bytes 0..7 / 8..15) elements 0..7 = 4.0 and
// 8..15 = 1.0.  The A side picks what it adds with its own offset chunk:
// K5 1.5 at element 8 (block scale 2^23), K5p / K5t pad_chunk(T, 0) = T,
// K5q pad_chunk(X, 128) with per-block scales.
__host__ __device__ __forceinline__ uint4 k5_table_offset_chunk() {
  return make_uint4(0x66666666u, 0x22222222u, 0x66666666u, 0x22222222u);
}
// v (0 <= v <= 46, or 48) as 8 e2m1 nibbles: 6.0s, then the remainder
__host__ __device__ __forceinline__ uint32_t e2m1_sum8(int v) {
  // e2m1 nibble of 0, 1, 2, 3, 4, 4 (+ 1.0 on the next nibble for 5)
  constexpr uint32_t kSmall = 0x665420u;
  const int n6 = v / 6, rem = v - 6 * n6;
  uint32_t x = n6 ? (0x77777777u >> (32 - 4 * n6)) : 0u;
  if (n6 < 8) x |= ((kSmall >> (4 * rem)) & 0xFu) << (4 * n6);
  if (rem == 5) x |= 0x2u << (4 * n6 + 4);
  return x;
}
// one 16-element A block whose dot product with a table offset block is T
// (0 <= T <= 238): 6.0s on the 4.0 elements (24 each), the rest on the 1.0s
__host__ __device__ __forceinline__ unsigned long long e2m1_block(int T) {
  const int k = min(8, T / 24);
  const uint32_t lo = k ? (0x77777777u >> (32 - 4 * k)) : 0u;
  return (unsigned long long)lo | ((unsigned long long)e2m1_sum8(T - 24 * k) << 32);
}
// K5q: the prefix weight may exceed the threshold by at most this much, so
// the A offset x = wt + 128 - thr stays <= 238 (e2m1_block's exact range)
constexpr int kQMaxSpan = 110;
// K5q producer threshold for a prefix of stored weight wt (0..128) against a
// bound rel = the Gamma's bound less its weight offset (<= the Gamma's
// stored columns <= 128: run_batch caps every Gamma's start bound there):
// codewords of stored weight < thr have bit 7 of their byte clear.
// thr in [1, 128] keeps every byte field wt(P^S) + 128 - thr in [0, 255]
// for stored weights 0..128 (a threshold of 1 under a bound <= 0 only flags
// weight-0 codewords, which the exact path then finds are not below it);
// thr >= wt - kQMaxSpan keeps the offset x = wt + 128 - thr <= 238.
__host__ __device__ __forceinline__ int k5q_threshold(int wt, int rel) {
  return max(wt - kQMaxSpan, max(1, min(128, rel)));
}
// A offset chunk: T0 on block 0, T1 on block 1
__host__ __device__ __forceinline__ uint4 pad_chunk(int T0, int T1) {
  const unsigned long long b0 = e2m1_block(T0), b1 = T1 ? e2m1_block(T1) : 0ull;
  return make_uint4((uint32_t)b0, (uint32_t)(b0 >> 32), (uint32_t)b1, (uint32_t)(b1 >> 32));
}
__host__ __device__ __forceinline__ uint4 k5p_offset_chunk(int T) { return pad_chunk(T, 0); }

// K5f (form 6): K5q's byte fields from fewer MMAs, for odd W whose last
// stored word holds at most 16 columns (stored columns <= 32 (W - 1) + 16:
// config 5's 80).  The last K chunk of a row is then half free: its 16 data
// columns move to block 0 (k5f_spread + the usual nibble order) and block 1
// carries offsets, so both parts' tails fit ONE K = 64 MMA whose B descriptor
// steps from table row c to row N + c (LBO = (N / 8) SBO):
//   table row, last chunk   [ data16 | offset pattern (8 x 4.0, 8 x 1.0) ]
//   A row, chunk W - 1 (ta) [ data16 | 4.0 on the pattern's 4.0s: 128    ]
//   A row, chunk W     (tb) [ data16 | e2m1_block(X), X = wt + 128 - thr ]
//   ue4m3 block scales      A (1, 256, 1, 1) x B (1, 256, 256, 256)
//   = d_a(tail) + 2^23 + 256 d_b(tail) + 256 X.
// With the whole chunks' MMAs (part b with B scale 256) an accumulator is
// 2^23 + d_a + 256 x_b, d = w(P ^ S) - w(P), x = w(P ^ S) + 128 - thr: part
// b's byte is K5q's, part a's lacks its X -- three offset classes (X, 256 X,
// 2^23) do not fit the two free blocks -- and the epilogue adds X to both
// 16-bit halves of every packed register (one IADD per four codewords), after
// which the registers equal K5q's bit for bit.  thr <= 127 keeps x_b >= 1, so
// a half d_a + 256 x_b is never negative and the add never carries across
// halves.  MMAs per tile at W = 3: 3 (96 MACs per codeword) against K5q's 4,
// table rows 48 B against 64.
__host__ __device__ constexpr bool k5f_ok(int w, int n_eff) {
  return (w == 1 || w == 3) && n_eff <= 32 * (w - 1) + 16;
}
// bit pair i (bits 2i, 2i + 1) of the low 16 bits -> bits 4i, 4i + 1: the
// elements e2m1_bits01 / e2m1_pm1 put into words x and y (block 0)
__host__ __device__ __forceinline__ uint32_t k5f_spread(uint32_t v) {
  v = (v | (v << 8)) & 0x00FF00FFu;
  v = (v | (v << 4)) & 0x0F0F0F0Fu;
  return (v | (v << 2)) & 0x33333333u;
}
__host__ __device__ __forceinline__ int k5f_threshold(int wt, int rel) {
  return max(wt - kQMaxSpan, max(1, min(127, rel)));
}
// table row, last chunk (tail word v: its low 16 bits are columns)
__host__ __device__ __forceinline__ uint4 k5f_table_tail(uint32_t v) {
  const uint4 d = e2m1_bits01(k5f_spread(v));
  return make_uint4(d.x, d.y, 0x66666666u, 0x22222222u);
}
// A row, chunks ta (part 0) and tb (part 1) of tail word v and offset x
__host__ __device__ __forceinline__ uint4 k5f_a_tail(uint32_t v, int part, int x) {
  const uint4 d = e2m1_pm1(k5f_spread(v));
  if (part == 0) return make_uint4(d.x, d.y, 0x66666666u, 0u);
  const unsigned long long b = e2m1_block(x);
  return make_uint4(d.x, d.y, (uint32_t)b, (uint32_t)(b >> 32));
}

// K5w (wide rows, two codewords per accumulator column as 11-bit fields):
//   acc = 2^23 + x_a + 2^11 x_b,  x = w(P ^ S) + 1024 - thr  in [0, 2047],
// so a codeword can lower the bound iff bit 10 of its field is clear.  Part b
// (table rows N + c) runs with B scale 2^11; each part's offset MMA adds
// R = w(P) - thr from the A chunk R (against the table-offset pattern: 16
// elements of 4.0, 16 of 1.0) and a constant from chunk Ca (part a: 5 x
// 2^21) or Cb (part b: 1 x 2^10) against B = (1.0, 1.0, 0, ...), ue8m0
// block scales (1, 2^21) / (2^11, 2^10): the constants sum to 2^23 + 1024 +
// 2^11 * 1024.  Every product and partial sum is an integer below 2^24.
constexpr int kWMaxSpan = 450;  // |R| <= 450: 4 * S4 + S1 with S4, S1 <= 90
// producer threshold for a prefix of stored weight wt (<= 256) against a
// bound rel (<= stored columns + g <= 384): raised to wt - kWMaxSpan at most
// (only more tiles take the exact path), never lowered below rel
__host__ __device__ __forceinline__ int k5w_threshold(int wt, int rel) {
  return max(wt - kWMaxSpan, max(1, min(384, rel)));
}
// 16 e2m1 elements (two words of 8) summing to S (0 <= S <= 90)
__host__ __device__ __forceinline__ void e2m1_sum16(int S, uint32_t& w0, uint32_t& w1) {
  const int a = S < 46 ? S : 46;
  w0 = e2m1_sum8(a);
  w1 = e2m1_sum8(S - a);
}
// chunk R: R = 4 * S4 + S1 (sign on every nibble), S4 on the elements facing
// the pattern's 4.0s (words 0, 2), S1 on its 1.0s (words 1, 3)
__host__ __device__ __forceinline__ uint4 k5w_r_chunk(int R) {
  const int A = R < 0 ? -R : R;
  const int S4 = min(A / 4, 90), S1 = A - 4 * S4;
  uint4 c;
  e2m1_sum16(S4, c.x, c.z);
  e2m1_sum16(S1, c.y, c.w);
  if (R < 0) {
    c.x |= 0x88888888u; c.y |= 0x88888888u; c.z |= 0x88888888u; c.w |= 0x88888888u;
  }
  return c;
}
// chunks Ca (4.0, 1.0 against B's 1.0, 1.0: 5) and Cb (1.0: 1)
__host__ __device__ __forceinline__ uint4 k5w_const_chunk(int part) {
  return make_uint4(part == 0 ? 0x26u : 0x02u, 0u, 0u, 0u);
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
// block-scaled: A = B = e2m1 (format 1), K-major, N, scale type ue8m0
// (bit 23), M, K = 64 (bit 31 clear), scale-factor ids 0
__host__ __device__ constexpr uint32_t mxf4_idesc(int n) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) |
         ((uint32_t)(kUmmaM >> 4) << 24);
}
constexpr uint32_t kMxf4Idesc = mxf4_idesc(kUmmaN4);

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
// Sleeping wait: try_wait with a suspend-time hint, so a warp that waits
// long (producers between chunks, the loader behind a full ring) sleeps in
// the barrier instead of spinning through issue slots and ALU ops.
#ifndef BZ_K5_SLEEPMASK
#define BZ_K5_SLEEPMASK 37  // non-critical waits sleep (chunk queue, A ring, loader)
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  for (uint32_t spin = 0;; ++spin) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(20000u)
        : "memory");
    if (done) return;
    if (spin > (1u << 20)) __trap();
  }
}
template <int BIT>
__device__ __forceinline__ void mbar_wait_sel(uint32_t bar, uint32_t parity) {
  if constexpr ((BZ_K5_SLEEPMASK & BIT) != 0) mbar_wait_sleep(bar, parity);
  else mbar_wait(bar, parity);
}
template <int BIT>
__device__ __forceinline__ void mbar_wait_fast_sel(uint32_t bar, uint32_t parity);

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
template <int BIT>
__device__ __forceinline__ void mbar_wait_fast_sel(uint32_t bar, uint32_t parity) {
  if constexpr ((BZ_K5_SLEEPMASK & BIT) != 0) mbar_wait_sleep(bar, parity);
  else mbar_wait_fast(bar, parity);
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
// D (f32) [+]= A . B with per-32-K block scales read from TMEM (sfa, sfb)
__device__ __forceinline__ void umma_mxf4(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate, uint32_t sfa,
                                          uint32_t sfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], "
      "p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
      : "memory");
}
// kind::mxf4nvf4: e2m1 operands, ue4m3 scales per 16-element block
__device__ __forceinline__ void umma_nvf4(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate, uint32_t sfa,
                                          uint32_t sfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], "
      "p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
      : "memory");
}
__device__ __forceinline__ float fmin3f(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(v)
      : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_regs4_after_wait(uint32_t* v) {
  asm volatile("" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]) : : "memory");
}
__device__ __forceinline__ void tmem_regs8_after_wait(uint32_t* v) {
  asm volatile(""
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7])
               :
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
// 64 columns as 32 registers in ONE load (the K5q / K5f lean epilogue reads
// its 60 columns with it: ptxas cannot slide arithmetic on the first
// registers between the pieces of a split load and reuse their registers for
// the later pieces, which is what delayed K5f's last loads and its release)
__device__ __forceinline__ void tmem_ld32p(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
      "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
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

// C consecutive 32-bit columns of this warp's 32 TMEM lanes as packed
// 16-bit pairs (low halves) into v[0, C/2) (C a multiple of 4, at most 128)
__device__ __forceinline__ void tmem_ld8p(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld4p(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.pack::16b.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld2p(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.pack::16b.b32 {%0,%1}, [%2];"
               : "=r"(v[0]), "=r"(v[1])
               : "r"(taddr));
}
template <int C>
__device__ __forceinline__ void tmem_ld_cols_p(uint32_t taddr, uint32_t* v) {
  if constexpr (C >= 32) {
    tmem_ld16p(taddr, v);
    tmem_ld_cols_p<C - 32>(taddr + 32, v + 16);
  } else if constexpr (C >= 16) {
    tmem_ld8p(taddr, v);
    tmem_ld_cols_p<C - 16>(taddr + 16, v + 8);
  } else if constexpr (C >= 8) {
    tmem_ld4p(taddr, v);
    tmem_ld_cols_p<C - 8>(taddr + 8, v + 4);
  } else if constexpr (C >= 4) {
    tmem_ld2p(taddr, v);
  }
}

// C consecutive 32-bit columns of this warp's 32 TMEM lanes into v[0, C)
// (C a multiple of 4, at most 128): x32 / x16 / x8 / x4 loads, no wait.
template <int C>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t* v) {
  if constexpr (C >= 32) {
    tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(v));
    tmem_ld_cols<C - 32>(taddr + 32, v + 32);
  } else if constexpr (C >= 16) {
    tmem_ld16(taddr, v);
    tmem_ld_cols<C - 16>(taddr + 16, v + 16);
  } else if constexpr (C >= 8) {
    tmem_ld8(taddr, *reinterpret_cast<uint32_t(*)[8]>(v));
    tmem_ld_cols<C - 8>(taddr + 8, v + 8);
  } else if constexpr (C >= 4) {
    tmem_ld4(taddr, v);
  }
}

// Consecutive rounds of one bz_rounds call on the same tensor-core kernel in
// ONE launch (K5q rounds g = 5..8 of config 5): the rows, prefix table and
// binomials are staged once, the rounds' plans side by side, and the rounds'
// chunk spaces concatenated into one cursor (round 0's counter), so the
// persistent CTAs run the rounds back to back without a launch, prologue or
// tail between them.  A queue entry carries its round in bits 56..63.
constexpr int kK5MaxFused = 4;
struct K5Batch {
  RoundArgs a[kK5MaxFused];
  unsigned long long cend[kK5MaxFused];  // this shard's chunks of rounds <= r, cumulative
  int goff[kK5MaxFused];                 // round r's first group in the staged plans
  int count;
};
constexpr int kQRoundShift = 56;

// Suffix tables of one round: level D = 3 + i at t[i], stride_rows[i] rows
// per Gamma (K4 uses t[0] only).
struct K4Tables {
  const uint8_t* t[3];
  unsigned long long stride_rows[3];
};

// K5 suffix table of level D: every D-subset of rows [floor, k), smallest
// element a descending (so the subsets with smallest element >= f are the
// first C(k - f, D) rows), then the other D - 1 elements lex.  One thread per
// table row (grid.y = Gamma); rows stored as e2m1 0 / 1.0 nibbles in the
// UMMA K-major no-swizzle layout (+ the offset chunk for odd W).
#ifndef BZ_BUILD_ROWS
#define BZ_BUILD_ROWS 2
#endif
constexpr int kBuildRows = BZ_BUILD_ROWS;  // suffix-table rows per builder thread (divides 8)

template <int W, int FORM = 1>
__global__ void k_build_subsets_mxf4(const uint32_t* __restrict__ rows,
                                     uint8_t* __restrict__ out, int k, int D,
                                     unsigned long long nrows, size_t gamma_stride_rows,
                                     const unsigned long long* __restrict__ binom) {
  constexpr int WP = padded_words(W);
  constexpr int C = k4_row_bytes<true>(W, FORM) / 16;  // chunks per row (+ offset chunk)
  constexpr bool FD = FORM == 6;  // K5f rows: the last chunk half data, half offset pattern
  // binomials C(x, 0..5) for x <= k in shared memory (the one unrank per
  // thread is a binary search over them)
  __shared__ unsigned long long sbt[kBinomDim * 6];
  for (int i = threadIdx.x; i < (k + 1) * 6; i += blockDim.x)
    sbt[i] = binom[(i / 6) * kBinomDim + (i % 6)];
  __syncthreads();
  auto B = [&](int x, int q) { return sbt[x * 6 + q]; };
  // kBuildRows consecutive rows per thread: it unranks the first once and
  // steps to the others with the table order's successor (the unrank's
  // binary searches were the builder's cost)
  const unsigned long long row0 =
      ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) * (unsigned long long)kBuildRows;
  if (row0 >= gamma_stride_rows) return;
  const int j = blockIdx.y;
  uint8_t* grp = out + (size_t)j * gamma_stride_rows * (16 * C);
  const uint32_t* R = rows + (size_t)j * k * WP;
  int e[5];  // the subset, e[0] = smallest element a, e[1..D-1] ascending
  if (row0 < nrows) {
    // smallest element a: rows of a start at C(k-1-a, D); x = k-1-a is the
    // largest x <= k-1 with C(x, D) <= row (C(D-1, D) = 0)
    int lo = D - 1, hi = k - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (B(mid, D) <= row0) lo = mid; else hi = mid - 1;
    }
    e[0] = k - 1 - lo;
    unsigned long long r = row0 - B(lo, D);
    // lex unrank of r among the (D-1)-subsets of [a+1, k)
    int at = e[0] + 1;
    for (int i = D - 1; i >= 1; --i) {
      const unsigned long long T = B(k - at, i) - r;
      int l2 = at, h2 = k - i;
      while (l2 < h2) {
        const int mid = (l2 + h2) >> 1;
        if (B(k - 1 - mid, i) < T) h2 = mid; else l2 = mid + 1;
      }
      r = r - B(k - at, i) + B(k - l2, i);
      e[D - i] = l2;
      at = l2 + 1;
    }
  }
  for (int q = 0; q < kBuildRows; ++q) {
    const unsigned long long row = row0 + (unsigned long long)q;
    uint8_t* dst = grp + (size_t)(row >> 3) * (8 * 16 * C) + (row & 7) * 16;
    if (row >= nrows) {
      // tail rows (read by whole-tile copies, their columns masked): the
      // empty subset, so every column a K5p/K5q tile pairs stays in range
#pragma unroll
      for (int w = 0; w < W; ++w) *reinterpret_cast<uint4*>(dst + w * 128) = make_uint4(0u, 0u, 0u, 0u);
      if constexpr (C > W) *reinterpret_cast<uint4*>(dst + W * 128) = k5_table_offset_chunk();
      if constexpr (FD) *reinterpret_cast<uint4*>(dst + (W - 1) * 128) = k5f_table_tail(0u);
      continue;
    }
    uint32_t v[W];
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] = R[e[0] * WP + w];
    for (int i = 1; i < D; ++i)
#pragma unroll
      for (int w = 0; w < W; ++w) v[w] ^= R[e[i] * WP + w];
#pragma unroll
    for (int w = 0; w < (FD ? W - 1 : W); ++w)
      *reinterpret_cast<uint4*>(dst + w * 128) = e2m1_bits01(v[w]);
    if constexpr (FD) *reinterpret_cast<uint4*>(dst + (W - 1) * 128) = k5f_table_tail(v[W - 1]);
    if constexpr (C > W)  // offset chunk
      *reinterpret_cast<uint4*>(dst + W * 128) = k5_table_offset_chunk();
    // successor in table order: the next (D-1)-subset of [a+1, k) in lex
    // order, or (after the last one) a - 1 with its first subset
    int i = D - 1;
    while (i >= 1 && e[i] == k - D + i) --i;
    if (i >= 1) {
      ++e[i];
      for (int t = i + 1; t < D; ++t) e[t] = e[t - 1] + 1;
    } else {
      --e[0];
      for (int t = 1; t < D; ++t) e[t] = e[0] + t;
    }
  }
}

// ---------------------------------------------------------------------------
// K4 triple table, one block per (Gamma, a): 0/1 bytes (kind::i8), 2W
// 16-byte K chunks per row.  (K5's tables come from k_build_subsets_mxf4.)
template <int W>
__global__ void k_build_triples_umma(const uint32_t* __restrict__ rows,
                                     uint8_t* __restrict__ trip, int k,
                                     size_t gamma_stride_rows) {
  constexpr int WP = padded_words(W);
  constexpr int RB = k4_row_bytes<false>(W);  // bytes per table row
  const int j = blockIdx.y, a = blockIdx.x;
  if (a > k - 3) return;
  const uint32_t* R = rows + (size_t)j * k * WP;
  const long long base = (long long)(k - 1 - a) * (k - 2 - a) * (k - 3 - a) / 6;
  const int span = k - 1 - a;
  const int npairs = span * (span - 1) / 2;
  uint8_t* out = trip + (size_t)j * gamma_stride_rows * RB;
  for (int t = threadIdx.x; t < npairs * W; t += blockDim.x) {
    const int pi = t / W, w = t - pi * W;
    int b = a + 1, rem = pi;
    while (rem >= k - 1 - b) { rem -= k - 1 - b; ++b; }
    const int c = b + 1 + rem;
    const uint32_t v = R[a * WP + w] ^ R[b * WP + w] ^ R[c * WP + w];
    const long long row = base + pi;
    uint8_t* grp = out + (size_t)(row >> 3) * (8 * RB);
    // 32 bytes of word w = K chunks 2w and 2w+1 of this row
    uint4 lo, hi;
    lo.x = bit_nibble(v, 0);  lo.y = bit_nibble(v, 4);  lo.z = bit_nibble(v, 8);  lo.w = bit_nibble(v, 12);
    hi.x = bit_nibble(v, 16); hi.y = bit_nibble(v, 20); hi.z = bit_nibble(v, 24); hi.w = bit_nibble(v, 28);
    *reinterpret_cast<uint4*>(grp + (2 * w) * 128 + (row & 7) * 16) = lo;
    *reinterpret_cast<uint4*>(grp + (2 * w + 1) * 128 + (row & 7) * 16) = hi;
  }
}

template <int W, bool F4, int CW = 1>
__host__ __device__ inline size_t k4_smem_bytes(int m, int k, int ngroups) {
  size_t off = (smem_base_bytes<W>(m, k, ngroups) + 1023) & ~size_t(1023);
  off += (size_t)k4_stages<F4, CW>(W) * k4_tile_b<F4, CW>(W);
  off += (size_t)k4_abufs<F4, CW>(W) * kUmmaMA * k4_tile_a<F4, CW>(W);
  off += F4 ? kMagicBytes : 0;   // K5 magic operands
  off += kBarSlots * 8 + 16;     // barriers + TMEM base
  off += k4_abufs<F4, CW>(W) * kUmmaMA * kUmmaM * sizeof(int);  // prefix weights of the A buffers
  off += kChunkQ * sizeof(long long) + 16;    // chunk queue
  off += kBndCache * sizeof(int);              // K5q bound cache
  return off;
}

// debug timeline (BZ_K4_DEBUG & 8): block 0, tiles [trace_from, +256)
// (BZ_K4_TRACE_ELL = L >= 0 instead traces from the first chunk with ell >= L;
// every role tracks that tile offset in `toff`)
constexpr uint32_t kNoTrace = 0xF0000000u;
__device__ __forceinline__ uint32_t k4_trace_off(const RoundArgs& a) {
  return a.trace_ell >= 0 ? kNoTrace : (uint32_t)a.trace_from;
}
__device__ __forceinline__ void k4_trace_chunk(const RoundArgs& a, uint32_t& toff, int ell,
                                               uint32_t tile) {
  if (a.trace_ell >= 0 && toff == kNoTrace && ell >= a.trace_ell) toff = tile;
}
#ifndef BZ_K4_TRACE
#define BZ_K4_TRACE 0  // build with -DBZ_K4_TRACE=1 for the BZ_K4_DEBUG & 8 timeline
#endif
#ifndef BZ_K4_TRACE_WARP
#define BZ_K4_TRACE_WARP -1  // second traced epilogue warp (slots 7, 14); default the last
#endif
__device__ __forceinline__ void k4_trace(const RoundArgs& a, int slot, uint32_t tile,
                                         uint32_t toff) {
  if (!BZ_K4_TRACE || !a.trace || blockIdx.x != 0) return;
  const uint32_t i = tile - toff;
  if (i < 256) a.trace[slot * 256 + i] = clock64();
}

// debug per-chunk timeline (BZ_K4_DEBUG & 32): per block, the first 64
// chunks as {chunk, dequeued (clock64), done (clock64), done (globaltimer)}
__device__ __forceinline__ long long* k4_ctrace(const RoundArgs& a, uint32_t qi) {
  return (a.ctrace && qi < 63) ? a.ctrace + ((size_t)blockIdx.x * 64 + qi) * 4 : nullptr;
}
// K5q: a per-CTA cache of the per-Gamma bound words (Gammas < kBndCache).
// It only ever holds a value read from the global word or one this CTA
// published to it, and the global words only decrease, so the cache is never
// below its global word: a candidate not below the cache cannot lower the
// global bound, and the epilogue skips the global atomics for it.
__device__ __forceinline__ int bnd_cache_read(const int* s_bnd, int round, int gamma) {
  return gamma < kBndPerRound ? ((const volatile int*)s_bnd)[round * kBndPerRound + gamma] : INT_MAX;
}
__device__ __forceinline__ void bnd_publish(int* s_bnd, const RoundArgs& a, int round, int gamma,
                                            int w) {
  if (gamma < kBndPerRound && atomicMin(s_bnd + round * kBndPerRound + gamma, w) <= w) return;
  atomicMin(a.bound + 1 + gamma, w);
  atomicMin(a.bound, w);
  gbound_publish(a, w);
}

__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Decoded chunk: identical on every role.
struct K4Chunk {
  Group gr;
  unsigned long long bfirst;
  long long maxcnt;
  int slice, tile_lo, tile_hi;
};

template <int N>
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
  c.slice = c.gr.slice;
  const int ntiles = (c.slice + N - 1) / N;
  c.tile_lo = tb * c.gr.tpc;
  c.tile_hi = min(ntiles, c.tile_lo + c.gr.tpc);
  return c;
}

// K5w epilogue: H columns c0.. of 2^23 + x_a + 2^11 x_b (11-bit fields);
// columns past the valid part-a (la) / part-b (lb) range get bit 10 / 21
// set.  Returns the smallest field below lx (lx if none).  The common case
// -- every column in range, every field at or above the threshold -- is one
// 3-input AND per two columns and one test; masking and the exact scan only
// run on the slice's last tile / when some threshold bit is clear.
template <int H>
__device__ __forceinline__ int k5w_scan(uint32_t* v, int c0, int la, int lb, int lx) {
  constexpr uint32_t kFlags = (1u << 10) | (1u << 21);
  if (lb < c0 + H) {  // uniform: some column of this slice is past a range
#pragma unroll
    for (int i = 0; i < H; ++i) {
      if (c0 + i >= la) v[i] |= 1u << 10;
      if (c0 + i >= lb) v[i] |= 1u << 21;
    }
  }
  uint32_t acc = 0xFFFFFFFFu;
#pragma unroll
  for (int i = 0; i + 1 < H; i += 2) acc &= v[i] & v[i + 1];
  if (H & 1) acc &= v[H - 1];
  if (__builtin_expect(!((~acc) & kFlags), 1)) return lx;
  int mn = lx;
#pragma unroll
  for (int i = 0; i < H; ++i)
    mn = min(mn, min((int)(v[i] & 0x7FFu), (int)((v[i] >> 11) & 0x7FFu)));
  return mn;
}

// K5f epilogue: NPH packed registers = 2 NPH accumulator columns (low 16 bits
// each: d_a + 256 x_b) of one row.  Adds the row offset X to both halves of
// every register (x * 0x10001 + v: one IMAD on the FMA pipe, which the rest of
// the epilogue leaves idle, interleaved with the AND pass on the ALU pipe),
// after which the registers are K5q's: bytes x = w + 128 - thr, and a
// codeword can lower the bound iff bit 7 of its byte is clear.  Columns at or
// past la (part a) / lb (part b), relative to the first, are masked.  Returns
// the smallest byte below lx (and lowers lx to it), else INT_MAX.
template <int NPH, bool ADD = true>
__device__ __forceinline__ int k5f_scan(uint32_t* v, uint32_t xoff, int la, int lb, int& lx) {
  static_assert(NPH % 2 == 0, "register pairs");
  uint32_t acc = 0xFFFFFFFFu;
#pragma unroll
  for (int i = 0; i < NPH; i += 2) {
    if constexpr (ADD) {  // (K5q's registers carry X already)
      v[i] += xoff * 0x00010001u;
      v[i + 1] += xoff * 0x00010001u;
    }
    acc &= v[i] & v[i + 1];
  }
  if (lb < 2 * NPH) {  // uniform: a slice's last tile
#pragma unroll
    for (int i = 0; i < NPH; ++i) {
      if (2 * i >= la) v[i] |= 0x000000FFu;
      if (2 * i >= lb) v[i] |= 0x0000FF00u;
      if (2 * i + 1 >= la) v[i] |= 0x00FF0000u;
      if (2 * i + 1 >= lb) v[i] |= 0xFF000000u;
    }
    acc = 0xFFFFFFFFu;
#pragma unroll
    for (int i = 0; i < NPH; i += 2) acc &= v[i] & v[i + 1];
  }
  if (__builtin_expect(!((~acc) & 0x80808080u), 1)) return INT_MAX;
  // some byte is below the producer's threshold; below this row's own
  // minimum so far?  ((x - lx * 0x01010101) & ~x has bit 7 of the lowest
  // such byte set, lx <= 128)
  const uint32_t kx = (uint32_t)lx * 0x01010101u;
  uint32_t h = 0;
#pragma unroll
  for (int i = 0; i < NPH; ++i) h |= (v[i] - kx) & ~v[i];
  if (!(h & 0x80808080u)) return INT_MAX;
  int mn = lx;
#pragma unroll
  for (int i = 0; i < NPH; ++i)
#pragma unroll
    for (int b = 0; b < 4; ++b) mn = min(mn, (int)((v[i] >> (8 * b)) & 0xFFu));
  lx = mn;
  return mn;
}

// K4 (F4 = false, tcgen05.mma kind::i8) and K5 (F4 = true, kind::mxf4 with
// unit block scales): one persistent CTA per SM, warp-specialised (see the
// file comment).  The two differ only in operand encoding, MMA kind,
// accumulator type (s32 read as packed s16 / f32) and tile geometry.
template <int W, bool F4, int CW>
__global__ void __launch_bounds__(K4Roles<F4, CW>::THREADS, 1)
k4_round_umma(const K5Batch bt, const K4Tables tabs) {
  // round 0's arguments: everything the fused rounds share (rows, prefix
  // table, m, k, n, binomials, the chunk cursor, debug and trace switches)
  const RoundArgs& a = bt.a[0];
  constexpr bool PR = CW > 1;  // K5p (CW = 2) / K5t (CW = 3) / K5q (CW = 4)
  constexpr bool FD = CW == 6;  // K5f: K5q's bytes from folded MMAs (k5f_ok)
  constexpr bool Q = CW == 4 || FD;  // K5q: two codewords as bytes, block16 scales
  constexpr bool WQ = CW == 5;  // K5w: two codewords as 11-bit fields (wide rows)
  constexpr bool QQ = Q || WQ;  // threshold-offset forms (bit test, bound cache)
  constexpr int NC = k5_ncw(CW);  // codewords per accumulator column
  static_assert(!F4 || kUmmaMA == 1, "K5 runs one A tile per B tile");
  static_assert(CW >= 1 && CW <= 6, "kernel form");
  // offset accumulators (packed s16 epilogue) for this instantiation
  constexpr bool MG = kK5Magic && (CW > 1 || (W & 1) || !BZ_K5_EVEN_F32);
  static_assert(!PR || (F4 && kK5Magic && (Q || BZ_K5_SPLIT == 1) &&
                        (WQ ? W >= 2 : (((W & 1) || CW == 4) && W <= (CW == 4 ? 4 : 3) &&
                                        (CW == 4 || BZ_K5_EPI_GROUPS == 1)))),
                "K5p/K5t: odd W <= 3, K5q: W <= 4 (stored weights <= 127 fit the fields)");
  constexpr int N = k4_n<F4, CW>();
  constexpr int TR = k4_tile_rows<F4, CW>();  // table rows per B tile
  constexpr int S = k4_stages<F4, CW>(W);
  constexpr int P = k4_passes<F4>(W);        // MMAs per tile (K5p: per half)
  constexpr int CA = k4_a_chunks<F4, CW>(W); // 16-byte K chunks per A row
  constexpr int CB = k4_row_bytes<F4>(W, CW) / 16;  // ... per B row
  constexpr uint32_t TB = k4_tile_b<F4, CW>(W);
  constexpr uint32_t TA = k4_tile_a<F4, CW>(W);
  using RL = K4Roles<F4, CW>;
  constexpr int ACC = RL::ACC;
  constexpr int E = RL::E;
  constexpr int TW = (BZ_K4_TRACE_WARP >= 0 && BZ_K4_TRACE_WARP < E) ? BZ_K4_TRACE_WARP : E - 1;
  constexpr int EGRP = RL::EGRP;
  constexpr int EC = N / (RL::EW / 4);  // columns per epilogue warp and A tile
  constexpr int SPLIT = RL::SPLIT;
  constexpr int NH = N / SPLIT;  // accumulator columns per part
  static_assert(NH % 8 == 0, "parts are whole 8-row groups of the B tile");
  // K5q: kind::mxf4nvf4 with ue4m3 block16 scales (scale-format bit 23 clear)
  constexpr uint32_t IDESC =
      F4 ? (Q ? mxf4_idesc(NH) & ~(1u << 23) : mxf4_idesc(NH)) : kUmmaIdesc;
  static_assert(S <= kMaxStages, "barrier slots");
  static_assert(EC * (RL::EW / 4) == N && (F4 ? EC % 4 == 0 && EC <= 128 : EC % 32 == 0),
                "epilogue");
  extern __shared__ __align__(128) unsigned char smem[];
  const size_t base = (smem_base_bytes<W>(a.m, a.k, staged_groups(a)) + 1023) & ~size_t(1023);
  unsigned char* sB = smem + base;
  unsigned char* sA = sB + S * TB;
  constexpr int NA = k4_abufs<F4, CW>(W);
  unsigned char* sMagic = sA + NA * kUmmaMA * TA;  // K5: A, B magic core matrices
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(sMagic + (F4 ? kMagicBytes : 0));
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + kBarSlots);
  int* s_wt = reinterpret_cast<int*>(s_tmem + 4);  // [2][kUmmaMA][kUmmaM] prefix weights
  volatile long long* s_q = reinterpret_cast<volatile long long*>(
      (reinterpret_cast<uintptr_t>(s_wt + NA * kUmmaMA * kUmmaM) + 15) & ~uintptr_t(15));
  int* s_bnd = const_cast<int*>(reinterpret_cast<volatile int*>(s_q + kChunkQ));  // [kBndCache]
  const uint32_t sB_s = (uint32_t)__cvta_generic_to_shared(sB);
  const uint32_t sA_s = (uint32_t)__cvta_generic_to_shared(sA);
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bars);
  // Rings: B stages (loader -> MMA: bfull; MMA commit -> loader: bempty),
  // accumulators (MMA commit -> epilogue: accfull; epilogue -> MMA:
  // accempty), A buffers (producers -> MMA, epilogue: afull; MMA commit +
  // epilogue -> producers: aempty).
  constexpr uint32_t B0 = 2 * kMaxABuf;  // first B-stage barrier slot
  auto afull = [&](int i) { return bar_s + 8u * (0 + i); };
  auto aempty = [&](int i) { return bar_s + 8u * (kMaxABuf + i); };
  auto bfull = [&](int i) { return bar_s + 8u * (B0 + i); };
  auto bempty = [&](int i) { return bar_s + 8u * (B0 + kMaxStages + i); };
  auto accfull = [&](int i) { return bar_s + 8u * (B0 + 2 * kMaxStages + i); };
  auto accempty = [&](int i) { return bar_s + 8u * (B0 + 2 * kMaxStages + kMaxAcc + i); };
  // chunk queue: the loader draws chunks from the round's global counter
  // (dynamic balance across CTAs) and publishes them to every other role
  auto qfull = [&](int i) { return bar_s + 8u * (B0 + 2 * kMaxStages + 2 * kMaxAcc + i); };
  auto qempty = [&](int i) {
    return bar_s + 8u * (B0 + 2 * kMaxStages + 2 * kMaxAcc + kChunkQ + i);
  };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(bfull(i), 1); mbar_init(bempty(i), 1); }
    for (int i = 0; i < NA; ++i) {
      mbar_init(afull(i), 4);                    // each producer warp
      mbar_init(aempty(i), ACC + E);             // each MMA warp's commit + epilogue warp
    }
    for (int i = 0; i < ACC * SPLIT; ++i) {
      mbar_init(accfull(i), 1);                  // MMA commit
      mbar_init(accempty(i), RL::EW / SPLIT);    // each epilogue warp of the part
    }
    for (int i = 0; i < kChunkQ; ++i) {
      mbar_init(qfull(i), 1);                    // loader
      mbar_init(qempty(i), E + ACC + 4);         // epilogue, MMA and producer warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async();
  }
  if (warp == RL::MMA0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(s_tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // the next round's kernel (programmatic dependent launch) may start its
  // CTAs as this kernel's CTAs exit: rounds are independent
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // per-block lifetime (BZ_K4_DEBUG & 32): slot 63 = {entry, prologue done,
  // exit} in globaltimer ns
  long long* const life = a.ctrace ? a.ctrace + ((size_t)blockIdx.x * 64 + 63) * 4 : nullptr;
  if (life && tid == 0) life[0] = global_ns();
  uint32_t *srows, *spx;
  Group* sgroups;
  tc_fence_before();
  stage<W>(a, srows, spx, sgroups, smem);  // ends with __syncthreads
  const unsigned long long* sbinom = smem_binom<W>(smem, a);
  // the other fused rounds' plans after round 0's (made visible by the
  // __syncthreads below)
  for (int rr = 1; rr < bt.count; ++rr)
    if (!a.groups_global) stage_groups(bt.a[rr], sgroups + bt.goff[rr]);
  // round rr's plan: staged, or in global memory
  auto plan_of = [&](int rr) -> const Group* {
    return a.groups_global ? bt.a[rr].groups : sgroups + bt.goff[rr];
  };
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  // a batched round starts from the U its predecessor ended with (the
  // running U the reference clips with, m/engine.py:209-211): chained on this
  // device and/or through the shared mirror (round_start)
  for (int rr = 0; rr < bt.count; ++rr) round_start(bt.a[rr]);
  if constexpr (F4) {
    // unit block scales (ue8m0 0x7F = 2^0) in TMEM columns [kSfCol, 512);
    // the zero K-padding chunk of both A buffers (odd W)
    if (warp < 4) {
      for (int c = 0; c < 512 - kSfCol; c += 8)
        tmem_st8(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(kSfCol + c),
                 WQ ? (c == 0 ? 0x7F7F7F7Fu                             // ue8m0 1
                       : c == 8 ? 0x8A8A8A8Au                           // 2^11: part b
                       : kSfCol + c == kSfColMagic ? 0x7F7F947Fu        // (1, 2^21): part a offset
                                                   : 0x7F7F898Au)       // (2^11, 2^10): part b
                 : FD ? (kSfCol + c == kSfColMagic ? 0x78787878u  // ue4m3 256: part b
                       : kSfCol + c == kSfColPad ? 0x38387838u   // A tail: (1, 256, 1, 1)
                       : c == 8 ? 0x78787838u                    // B tail: (1, 256, 256, 256)
                                : 0x38383838u)                   // ue4m3 1.0
                 : Q ? (kSfCol + c == kSfColMagic ? 0x78787878u   // ue4m3 256: half b
                      : kSfCol + c == kSfColPad ? 0x78383838u  // A: 256 on block 3
                                                : 0x38383838u) // ue4m3 1.0
                 : kSfCol + c == kSfColMagic
                     ? (PR ? 0x8F8F8F8Fu : 0x96969696u)                       // 2^16 | 2^23
                     : (kSfCol + c == kSfColPad ? (CW == 3 ? 0x87878787u      // 2^8
                                                           : 0x7F7F967Fu)
                                                : 0x7F7F7F7Fu));
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    if (MG && tid < (int)kMagicBytes / 16) {
      // two K-chunks x 8 rows x 16 B per operand (SBO = 0: every 8-row group
      // reads these rows)
      const int op = tid / 16, row16 = tid % 16;  // row16 < 8: chunk 0
      uint4 z = make_uint4(0, 0, 0, 0);
      if constexpr (WQ) {
        // K5w: B of both parts' offset MMAs (op 1) = [offset pattern,
        // (1.0, 1.0, 0, ...)] against A chunks (R, Ca) / (R, Cb)
        if (op == 1) z = row16 < 8 ? k5_table_offset_chunk() : make_uint4(0x22u, 0u, 0u, 0u);
      } else if constexpr (Q) {
        // K5q, even W: the B side of the offset MMAs (the tables carry no
        // offset chunk): op 0 = [offset pattern, 0] (part a), op 1 =
        // [0, offset pattern] (part b), against A chunks (pad_a, pad_b)
        if ((row16 < 8) == (op == 0)) z = k5_table_offset_chunk();
      } else {
        // element 0 of every row: A = 1.5 (0x3), B = 1.0 (0x2); scaled by
        // 2^23 the product is the 1.5 * 2^23 the accumulators start from
        if (row16 < 8) z.x = op == 0 ? 0x3u : 0x2u;
      }
      *reinterpret_cast<uint4*>(sMagic + op * 256 + row16 * 16) = z;
      fence_proxy_async();
    }
    if constexpr (QQ)
      if (tid < kBndCache) {
        const int rr = tid / kBndPerRound, j = tid % kBndPerRound;
        s_bnd[tid] = rr < bt.count && j < a.m ? ((volatile int*)bt.a[rr].bound)[1 + j] : INT_MAX;
      }
    if (WQ && warp >= RL::PROD0) {
      // K5w: the constant A chunks of both A buffers -- zero padding (odd
      // W: it meets the table's offset chunk), Ca, Cb
      const int r = tid - 32 * RL::PROD0;
      constexpr int WD = k5w_data_chunks(W);
      for (int ab = 0; ab < NA; ++ab) {
        unsigned char* row = sA + ab * TA;
        if (WD > W) *reinterpret_cast<uint4*>(row + umma_off_c(r, W, CA)) = make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(row + umma_off_c(r, WD + 1, CA)) = k5w_const_chunk(0);
        *reinterpret_cast<uint4*>(row + umma_off_c(r, WD + 2, CA)) = k5w_const_chunk(1);
      }
      fence_proxy_async();
    }
    if (!PR && CA > W && warp >= RL::PROD0) {
      // the A padding chunk: zero, or 1.5 at element 8 (padding-chunk offset)
      const int r = tid - 32 * RL::PROD0;
      for (int ab = 0; ab < NA; ++ab)
        *reinterpret_cast<uint4*>(sA + ab * TA + umma_off_c(r, W, CA)) =
            make_uint4(0u, k5_padmagic(W) ? 0x3u : 0u, 0u, 0u);  // 1.5 at element 8
      fence_proxy_async();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  const int k = a.k;
  const unsigned FULL = 0xffffffffu;
  if (life && tid == 0) life[1] = global_ns();

  if (warp < E) {
    // ================= epilogue: warp e reads TMEM lanes 32(e%4).. (rows),
    // columns [EC*(e/4), +EC) of each accumulator
    const int egroup = warp / RL::EW;  // this warp drains tiles t % EGRP == egroup
    const int quarter = warp & 3, slice_id = (warp % RL::EW) >> 2;
    const int part = slice_id / ((RL::EW / 4) / SPLIT);  // accumulator part this warp drains
    const int r = 32 * quarter + lane;
    uint32_t grp = 0, tcount = 0, toff = k4_trace_off(a);
    for (uint32_t qi = 0;; ++qi) {
      const int qs = qi % kChunkQ;
      mbar_wait_sel<1>(qfull(qs), (qi / kChunkQ) & 1);
      const long long qchunk = s_q[qs];
      __syncwarp();
      if (lane == 0) mbar_arrive(qempty(qs));
      if (qchunk < 0) break;
      const int rr = (int)((unsigned long long)qchunk >> kQRoundShift);
      const RoundArgs& ar = bt.a[rr];
      const unsigned long long chunk = (unsigned long long)qchunk & ((1ull << kQRoundShift) - 1);
      const K4Chunk c = k4_decode<TR>(plan_of(rr), ar.ngroups, chunk, k);
      k4_trace_chunk(a, toff, c.gr.ell, tcount);
      int best = INT_MAX;
      // K5t: stored weights below thr can lower this Gamma's bound
      int thr = 127;
      if constexpr (CW == 3)
        thr = max(0, min(127, ((volatile int*)ar.bound)[1 + c.gr.gamma] - gamma_woff(ar, c.gr.gamma)));
      for (long long p = 0; p < c.maxcnt; p += kUmmaMA, ++grp) {
        const int ab = grp % NA;
        mbar_wait_sel<1>(afull(ab), (grp / NA) & 1);
        int wt[kUmmaMA];
#pragma unroll
        for (int j = 0; j < kUmmaMA; ++j) wt[j] = s_wt[(ab * kUmmaMA + j) * kUmmaM + r];
        __syncwarp();
        if (lane == 0) mbar_arrive(aempty(ab));
        int rmin[kUmmaMA];
#pragma unroll
        for (int j = 0; j < kUmmaMA; ++j) rmin[j] = INT_MAX / 2;
        float fmin_acc = __int_as_float(0x7f800000);  // K5: +inf
        int lx = 128;  // K5q: this row's bytes below lx can still lower its minimum
        int lx1024 = 1024;  // K5w: this row's fields below lx1024 can still lower it
        // K5q / K5f: the step's tiles in a lean loop -- the tile loop below
        // with the debug switches, trace points and per-tile address
        // arithmetic hoisted and the two accumulator buffers unrolled (the
        // epilogue warps of a scheduler share its issue slots, and per-tile
        // bookkeeping was most of what they issued)
        bool lean = false;
        if constexpr (Q && SPLIT == 1 && EGRP == 1 && ACC == 2 && kUmmaMA == 1 && !BZ_K4_TRACE &&
                      BZ_K5_LEAN) {
          if (!a.debug) {
            lean = true;
            constexpr int NP = EC / 2;
            const uint32_t tq = tmem + ((uint32_t)(32 * quarter) << 16) + (uint32_t)(EC * slice_id);
            const bool l0 = lane == 0;
            const int thr = FD ? (wt[0] & 0xFFFF) : wt[0];
            const uint32_t xoff = FD ? (uint32_t)(wt[0] >> 16) : 0u;
            int la = c.slice - c.tile_lo * TR - EC * slice_id;  // part-a columns < la valid
            auto tile = [&](auto bufc) {
              constexpr int BUF = decltype(bufc)::value;
              mbar_wait_fast(accfull(BUF), (tcount >> 1) & 1);
              tc_fence_after();
              uint32_t v[BZ_K5_LD64 && EC > 32 ? 32 : NP];
              // (a 60-column slice read as 64: the 4 extra columns -- the next
              // buffer's or the scale factors' -- land in v[30], v[31], unused)
              if constexpr (BZ_K5_LD64 && EC > 32) tmem_ld32p(tq + (uint32_t)(BUF * N), v);
              else tmem_ld_cols_p<EC>(tq + (uint32_t)(BUF * N), v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i + 1 < NP; i += 2) asm volatile("" : "+r"(v[i]), "+r"(v[i + 1]) : : "memory");
              tc_fence_before();
              __syncwarp();
              if (l0) mbar_arrive(accempty(BUF));  // the accumulator is in registers
              const int mn = k5f_scan<NP, FD>(v, xoff, la, la - N, lx);
              if (mn != INT_MAX) {
                const int w = mn - 128 + thr;
                rmin[0] = min(rmin[0], w);
                const int w2 = w + gamma_woff(ar, c.gr.gamma);
                // publish at once (the producers' next thresholds tighten),
                // only below the CTA's cached bound
                if (w2 < bnd_cache_read(s_bnd, rr, c.gr.gamma)) bnd_publish(s_bnd, ar, rr, c.gr.gamma, w2);
              }
              ++tcount;
              la -= TR;
            };
            int nt = c.tile_hi - c.tile_lo;
            if (nt > 0 && (tcount & 1)) {
              tile(std::integral_constant<int, 1>{});
              --nt;
            }
            for (; nt >= 2; nt -= 2) {
              tile(std::integral_constant<int, 0>{});
              tile(std::integral_constant<int, 1>{});
            }
            if (nt) tile(std::integral_constant<int, 0>{});
          }
        }
        if (!lean)
        for (int t = c.tile_lo; t < c.tile_hi; ++t, ++tcount) {
          if (EGRP > 1 && (int)(tcount % EGRP) != egroup) continue;
          const int buf = tcount % ACC;
          const int hb = buf * SPLIT + part;
          if (warp == 0 && lane == 0) k4_trace(a, 8, tcount, toff);
          mbar_wait_sel<2>(accfull(hb), (tcount / ACC) & 1);
          if (warp == 0 && lane == 0) k4_trace(a, 9, tcount, toff);
          if (!BZ_K5_NOFENCE) tc_fence_after();
          if (warp == 0 && lane == 0) k4_trace(a, 2, tcount, toff);
          if (warp == TW && lane == 0) k4_trace(a, 7, tcount, toff);
          const int lim = min(N, c.slice - t * TR) - EC * slice_id;
          const uint32_t tb = tmem + ((uint32_t)(32 * quarter) << 16) +
                              (uint32_t)(buf * kUmmaMA * N + EC * slice_id);
          if (a.debug & 1) {
            __syncwarp();
            if (lane == 0) mbar_arrive(accempty(hb));
            continue;
          }
          if constexpr (Q) {
            // K5q: every column holds 2^23 + x_a + 2^8 x_b, x = wt + 128 -
            // thr (thr = wt[0], the producer's threshold for this row): the
            // low 16 bits of two columns are four bytes per register, and a
            // codeword can lower the bound iff its byte has bit 7 clear.
            // One 3-input AND per two registers; exact minima only then.
            constexpr int NP = EC / 2;
            const int la = c.slice - t * TR - EC * slice_id;  // half-a columns < la valid
            uint32_t v[NP];
            tmem_ld_cols_p<EC>(tb, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i + 1 < NP; i += 2) asm volatile("" : "+r"(v[i]), "+r"(v[i + 1]) : : "memory");
            if (NP % 2) asm volatile("" : "+r"(v[NP - 1]) : : "memory");
            if (warp == 0 && lane == 0) k4_trace(a, 10, tcount, toff);
            if (!BZ_K5_NOFENCE) tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(accempty(hb));  // accumulators are in registers
            if (warp == 0 && lane == 0) k4_trace(a, 11, tcount, toff);
            if (warp == TW && lane == 0) k4_trace(a, 14, tcount, toff);
            if (a.debug & 64) continue;  // timing experiment: loads only
            if constexpr (FD) {
              const int mn = k5f_scan<NP>(v, (uint32_t)(wt[0] >> 16), la, la - N, lx);
              if (mn != INT_MAX) {
                const int w = mn - 128 + (wt[0] & 0xFFFF);
                rmin[0] = min(rmin[0], w);
                const int w2 = w + gamma_woff(ar, c.gr.gamma);
                if (w2 < bnd_cache_read(s_bnd, rr, c.gr.gamma)) bnd_publish(s_bnd, ar, rr, c.gr.gamma, w2);
              }
              continue;
            }
            if (la - N < EC) {
#pragma unroll
              for (int i = 0; i < NP; ++i) {
                if (2 * i >= la) v[i] |= 0x000000FFu;
                if (2 * i >= la - N) v[i] |= 0x0000FF00u;
                if (2 * i + 1 >= la) v[i] |= 0x00FF0000u;
                if (2 * i + 1 >= la - N) v[i] |= 0xFF000000u;
              }
            }
            uint32_t acc = 0xFFFFFFFFu;
#pragma unroll
            for (int i = 0; i + 1 < NP; i += 2) acc &= v[i] & v[i + 1];
            if (NP % 2) acc &= v[NP - 1];
            int wg = INT_MAX;  // this row's new minimum below the CTA's bound, if any
            if ((~acc) & 0x80808080u) {
              // some byte is below the producer's threshold; below this
              // row's own minimum so far?  (x - lx*0x01010101) & ~x has bit
              // 7 of the lowest such byte set, lx <= 128)
              const uint32_t kx = (uint32_t)lx * 0x01010101u;
              uint32_t h = 0;
#pragma unroll
              for (int i = 0; i < NP; ++i) h |= (v[i] - kx) & ~v[i];
              if (h & 0x80808080u) {
                int mn = lx;
#pragma unroll
                for (int i = 0; i < NP; ++i)
#pragma unroll
                  for (int b = 0; b < 4; ++b) mn = min(mn, (int)((v[i] >> (8 * b)) & 0xFFu));
                lx = mn;
                const int w = mn - 128 + wt[0];
                rmin[0] = min(rmin[0], w);
                const int w2 = w + gamma_woff(ar, c.gr.gamma);
                if (w2 < bnd_cache_read(s_bnd, rr, c.gr.gamma)) wg = w2;
              }
            }
            // publish at once, so the producers' next thresholds tighten --
            // only below the CTA's cached bound: under a loose bound every row
            // of every SM would otherwise send global atomics to the same two
            // words each tile (config 4: 105 -> 48 us).  (A warp-level
            // reduction first measured 4 % slower on config 5's g = 8.)
            if (wg != INT_MAX) bnd_publish(s_bnd, ar, rr, c.gr.gamma, wg);
          } else if constexpr (WQ) {
            // K5w: every column holds 2^23 + x_a + 2^11 x_b, x = w + 1024 -
            // thr (thr = wt[0]): a codeword can lower the bound iff bit 10 of
            // its field is clear.  Two loads (register budget), each tested
            // before the next; the buffer is released after the second.
            constexpr int H0 = EC > 32 ? 32 : EC, H1 = EC - H0;
            static_assert(H0 % 4 == 0 && H1 % 4 == 0, "K5w epilogue phases");
            const int la = c.slice - t * TR - EC * slice_id;  // part-a columns < la valid
            uint32_t v[H0];
            tmem_ld_cols<H0>(tb, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < H0; i += 4) tmem_regs4_after_wait(v + i);
            int mn = k5w_scan<H0>(v, 0, la, la - N, lx1024);
            if constexpr (H1 > 0) {
              tmem_ld_cols<H1>(tb + H0, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < H1; i += 4) tmem_regs4_after_wait(v + i);
            }
            if (!BZ_K5_NOFENCE) tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(accempty(hb));  // accumulators are in registers
            if constexpr (H1 > 0) mn = k5w_scan<H1>(v, H0, la, la - N, mn);
            if (mn < lx1024) {
              lx1024 = mn;
              const int w = mn - 1024 + wt[0];
              rmin[0] = min(rmin[0], w);
              const int w2 = w + gamma_woff(ar, c.gr.gamma);
              if (w2 < bnd_cache_read(s_bnd, rr, c.gr.gamma)) bnd_publish(s_bnd, ar, rr, c.gr.gamma, w2);
            }
          } else if constexpr (CW == 3) {
            // K5t: every column holds three codewords, 2^23 + wt_a + 2^8 wt_b
            // + 2^16 wt_c: bytes 0..2 are stored weights <= 96, byte 3 the
            // exponent.  A SWAR test finds whether any byte is below this
            // row's threshold thr (x - thr*0x010101 borrows into bit 7 of the
            // lowest such byte; no byte exceeds 127); only then are the
            // exact minima taken (rare once the bound has settled).
            const int la = c.slice - t * TR - EC * slice_id;  // part-0 columns < la valid
            uint32_t v[EC];
            tmem_ld_cols<EC>(tb, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < EC; i += 4) tmem_regs4_after_wait(v + i);
            if (!BZ_K5_NOFENCE) tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(accempty(hb));  // accumulators are in registers
            if (la - 2 * N < EC) {
#pragma unroll
              for (int i = 0; i < EC; ++i)
#pragma unroll
                for (int q = 0; q < 3; ++q)
                  if (i >= la - q * N) v[i] |= 0x7Fu << (8 * q);  // 127: never below thr
            }
            const uint32_t kthr = (uint32_t)thr * 0x00010101u;
            uint32_t acc = 0;
#pragma unroll
            for (int i = 0; i + 1 < EC; i += 2) acc |= (v[i] - kthr) | (v[i + 1] - kthr);
            if (EC & 1) acc |= v[EC - 1] - kthr;
            if (acc & 0x00808080u) {
              int mn = INT_MAX / 2;
#pragma unroll
              for (int i = 0; i < EC; ++i)
                mn = min(mn, min((int)(v[i] & 0x7Fu),
                                 min((int)((v[i] >> 8) & 0x7Fu), (int)((v[i] >> 16) & 0x7Fu))));
              rmin[0] = min(rmin[0], mn);
              thr = min(thr, mn);
            }
          } else if constexpr (PR) {
            // K5p: every column holds two codewords, 2^23 + wt_a + 2^16 wt_b
            // (stored weights <= 96): bits 0..15 = wt_a, bits 16..31 =
            // 0x4B00 + wt_b, so one s16x2 minimum serves both.  Two loads of
            // EC/2 columns (register budget), then the buffer is released.
            constexpr int NPH = EC > 64 ? 2 : 1;
            constexpr int H = EC / NPH;
            static_assert(H * NPH == EC && H % 4 == 0, "K5p epilogue phases");
            const int la = c.slice - t * TR - EC * slice_id;  // half-a columns < la valid
            const int lb = la - N;                             // half-b columns < lb valid
            uint32_t m0 = 0x7FFF7FFFu, m1 = 0x7FFF7FFFu;
#pragma unroll
            for (int hh = 0; hh < NPH; ++hh) {
              uint32_t v[H];
              tmem_ld_cols<H>(tb + hh * H, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < H; i += 4) tmem_regs4_after_wait(v + i);
              if (hh == NPH - 1) {
                if (!BZ_K5_NOFENCE) tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(accempty(hb));  // accumulators are in registers
              }
              if (a.debug & 64) continue;  // timing experiment: loads only
              if (lb < EC) {
#pragma unroll
                for (int i = 0; i < H; ++i) {
                  if (hh * H + i >= la) v[i] = (v[i] & 0xffff0000u) | 0x00007fffu;
                  if (hh * H + i >= lb) v[i] = (v[i] & 0x0000ffffu) | 0x7fff0000u;
                }
              }
#pragma unroll
              for (int i = 0; i + 3 < H; i += 4) {
                m0 = __vimin3_s16x2(m0, v[i], v[i + 1]);
                m1 = __vimin3_s16x2(m1, v[i + 2], v[i + 3]);
              }
#pragma unroll
              for (int i = (H / 4) * 4; i < H; ++i) m0 = __vmins2(m0, v[i]);
            }
            const uint32_t m = __vmins2(m0, m1);
            const int lo = (int)(m & 0xffffu), hi = (int)(m >> 16) - 0x4B00;
            rmin[0] = min(rmin[0], min(lo, hi));
          } else if constexpr (F4 && MG) {
            // EC accumulators as packed s16 pairs (low halves of 1.5*2^23 + D)
            constexpr int NP = EC / 2;
            uint32_t v[NP];
            tmem_ld_cols_p<EC>(tb, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i + 1 < NP; i += 2) {
              asm volatile("" : "+r"(v[i]), "+r"(v[i + 1]) : : "memory");
            }
            if (NP % 2) asm volatile("" : "+r"(v[NP - 1]) : : "memory");
            if (warp == 0 && lane == 0) k4_trace(a, 10, tcount, toff);
            if (!BZ_K5_NOFENCE) tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(accempty(hb));  // accumulators are in registers
            if (warp == 0 && lane == 0) k4_trace(a, 11, tcount, toff);
            if (warp == TW && lane == 0) k4_trace(a, 14, tcount, toff);
            if (lim < EC) {
#pragma unroll
              for (int i = 0; i < NP; ++i) {
                if (2 * i >= lim) v[i] = (v[i] & 0xffff0000u) | 0x00007fffu;
                if (2 * i + 1 >= lim) v[i] = (v[i] & 0x0000ffffu) | 0x7fff0000u;
              }
            }
            // two independent 3-input SIMD chains
            uint32_t m0 = __vimin3_s16x2(v[0], v[1], v[2]);
            uint32_t m1 = NP > 5 ? __vimin3_s16x2(v[3], v[4], v[5]) : v[0];
#pragma unroll
            for (int i = 6; i + 3 < NP; i += 4) {
              m0 = __vimin3_s16x2(m0, v[i], v[i + 1]);
              m1 = __vimin3_s16x2(m1, v[i + 2], v[i + 3]);
            }
#pragma unroll
            for (int i = 6 + ((NP - 6) / 4) * 4; i < NP; ++i) m0 = __vmins2(m0, v[i]);
            const uint32_t m = __vmins2(m0, m1);
            const int lo = (int)(short)(m & 0xffffu), hi = (int)(short)(m >> 16);
            rmin[0] = min(rmin[0], min(lo, hi));
          } else if constexpr (F4) {
            // EC f32 accumulators: every load, one wait, release the buffer,
            // then 3-input float minima
            uint32_t v[EC];
            tmem_ld_cols<EC>(tb, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < EC; i += 4) tmem_regs4_after_wait(v + i);
            if (warp == 0 && lane == 0) k4_trace(a, 10, tcount, toff);
            if (!BZ_K5_NOFENCE) tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(accempty(hb));  // accumulators are in registers
            if (warp == 0 && lane == 0) k4_trace(a, 11, tcount, toff);
            if (warp == TW && lane == 0) k4_trace(a, 14, tcount, toff);
            if (lim < EC) {
#pragma unroll
              for (int i = 0; i < EC; ++i)
                if (i >= lim) v[i] = 0x7f800000u;
            }
            // four independent 3-input chains, then combine
            float m0 = fmin_acc, m1 = __uint_as_float(v[0]), m2 = __uint_as_float(v[1]),
                  m3 = __uint_as_float(v[2]);
#pragma unroll
            for (int i = 3; i + 7 < EC; i += 8) {
              m0 = fmin3f(m0, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
              m1 = fmin3f(m1, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
              m2 = fmin3f(m2, __uint_as_float(v[i + 4]), __uint_as_float(v[i + 5]));
              m3 = fmin3f(m3, __uint_as_float(v[i + 6]), __uint_as_float(v[i + 7]));
            }
#pragma unroll
            for (int i = 3 + ((EC - 3) / 8) * 8; i < EC; ++i) m0 = fminf(m0, __uint_as_float(v[i]));
            fmin_acc = fmin3f(fminf(m0, m1), m2, m3);
          } else {
            // EC columns as packed s16 pairs: 3-input SIMD minima
            constexpr int NP = EC / 2;
            uint32_t v[kUmmaMA][NP];
#pragma unroll
            for (int j = 0; j < kUmmaMA; ++j)
#pragma unroll
              for (int cc = 0; cc < EC / 32; ++cc)
                tmem_ld16p(tb + j * N + 32 * cc, &v[j][16 * cc]);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < kUmmaMA; ++j)
#pragma unroll
              for (int cc = 0; cc < EC / 32; ++cc) tmem_regs16_after_wait(&v[j][16 * cc]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(accempty(hb));  // accumulators are in registers
#pragma unroll
            for (int j = 0; j < kUmmaMA; ++j) {
              if (lim < EC) {
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                  if (2 * i >= lim) v[j][i] = (v[j][i] & 0xffff0000u) | 0x00007fffu;
                  if (2 * i + 1 >= lim) v[j][i] = (v[j][i] & 0x0000ffffu) | 0x7fff0000u;
                }
              }
              uint32_t m = __vimin3_s16x2(v[j][0], v[j][1], v[j][2]);
#pragma unroll
              for (int i = 3; i + 1 < NP; i += 2) m = __vimin3_s16x2(m, v[j][i], v[j][i + 1]);
              if (NP % 2 == 0) m = __vmins2(m, v[j][NP - 1]);
              const int lo = (int)(short)(m & 0xffffu), hi = (int)(short)(m >> 16);
              rmin[j] = min(rmin[j], min(lo, hi));
            }
          }
          if (warp == 0 && lane == 0) k4_trace(a, 3, tcount, toff);
        }
        if constexpr (F4 && !MG) {
          // |D| <= n, so a finite minimum converts exactly; +inf (every
          // column of this slice masked) stays out of the way
          if (fmin_acc < 1.0e6f) rmin[0] = (int)fmin_acc;
        }
        // K5p minima are whole stored weights (the prefix weight rode on the
        // offset chunks)
#pragma unroll
        for (int j = 0; j < kUmmaMA; ++j) best = min(best, rmin[j] + (PR ? 0 : wt[j]));
      }
      const int wbest = __reduce_min_sync(FULL, best);
      if (lane == 0) {
        if (wbest < INT_MAX / 2) {
          // fire-and-forget reductions (RED.MIN): no load round trip stalls
          // the epilogue at a chunk boundary
          const int wb = wbest + gamma_woff(ar, c.gr.gamma);
          atomicMin(ar.bound + 1 + c.gr.gamma, wb);
          atomicMin(ar.bound, wb);
          gbound_publish(ar, wb);
          if constexpr (QQ)
            if (c.gr.gamma < kBndPerRound) atomicMin(s_bnd + rr * kBndPerRound + c.gr.gamma, wb);
        }

        long long* ct = k4_ctrace(a, qi);
        if (ct && warp == 0) { ct[2] = clock64(); ct[3] = global_ns(); }
      }
    }
  } else if (warp >= RL::PROD0) {
    // ================= producers: thread r walks prefix row r
    const int r = tid - 32 * RL::PROD0;
    uint32_t grp = 0;
    for (uint32_t qi = 0;; ++qi) {
      const int qs = qi % kChunkQ;
      mbar_wait_sel<4>(qfull(qs), (qi / kChunkQ) & 1);
      const long long qchunk = s_q[qs];
      __syncwarp();
      if (lane == 0) mbar_arrive(qempty(qs));
      if (qchunk < 0) break;
      const int rr = (int)((unsigned long long)qchunk >> kQRoundShift);
      const RoundArgs& ar = bt.a[rr];
      const unsigned long long chunk = (unsigned long long)qchunk & ((1ull << kQRoundShift) - 1);
      const K4Chunk c = k4_decode<TR>(plan_of(rr), ar.ngroups, chunk, k);
      const unsigned long long first = c.bfirst + (unsigned long long)r * c.gr.ppl;
      long long cnt = 0;
      if (first < c.gr.nprefix) {
        const unsigned long long left = c.gr.nprefix - first;
        cnt = left < (unsigned long long)c.gr.ppl ? (long long)left : c.gr.ppl;
      }
      const uint32_t* R = srows + c.gr.gamma * k * padded_words(W);
      const uint32_t* PX = spx + c.gr.gamma * (k + 1) * px_stride(W);
      Walker<W> wk;
      // rows without prefixes duplicate the block's first prefix
      // (a merged group, sl == 0: (g - D)-subsets of [0, ell + 1), no fixed row)
      const bool merged = c.gr.sl == 0;
      wk.init(cnt > 0 ? first : c.bfirst, ar.g - 1 - c.gr.depth + (merged ? 1 : 0),
              c.gr.ell + (merged ? 1 : 0), R, a.binom, sbinom, !merged);
      // walker row additions of this row's valid prefixes (counters)
      unsigned long long wadd = cnt > 0 ? (unsigned long long)max(ar.g - 1 - c.gr.depth, 0) : 0ull;
      for (long long p = 0; p < c.maxcnt; p += kUmmaMA, ++grp) {
        const int ab = grp % NA;
        mbar_wait_sel<4>(aempty(ab), ((grp / NA) & 1) ^ 1);
#pragma unroll 1
        for (int j = 0; j < kUmmaMA; ++j) {
          // step j of the group; past this row's range the last prefix repeats
          if (p + j > 0 && p + j < cnt) wadd += (unsigned long long)wk.step(PX);
          unsigned char* dst = sA + (ab * kUmmaMA + j) * TA;
          int wt = 0;
          if (a.debug & 16) continue;  // timing experiment: no A rows
#pragma unroll
          for (int jj = 0; jj < W; ++jj) {
            const uint32_t v = wk.acc[jj];
            wt += __popc(v);
            if constexpr (FD) {
              // (the tail word's chunks ta / tb follow with the offsets)
              if (jj < W - 1) *reinterpret_cast<uint4*>(dst + umma_off_c(r, jj, CA)) = e2m1_pm1(v);
            } else if constexpr (F4) {
              // e2m1 +1 (0x2) for a 0 bit, -1 (0xA) for a 1 bit
              *reinterpret_cast<uint4*>(dst + umma_off_c(r, jj, CA)) = e2m1_pm1(v);
            } else {
              uint4 lo, hi;
              lo.x = pm1_nibble(v, 0);  lo.y = pm1_nibble(v, 4);
              lo.z = pm1_nibble(v, 8);  lo.w = pm1_nibble(v, 12);
              hi.x = pm1_nibble(v, 16); hi.y = pm1_nibble(v, 20);
              hi.z = pm1_nibble(v, 24); hi.w = pm1_nibble(v, 28);
              *reinterpret_cast<uint4*>(dst + umma_off_c(r, 2 * jj, CA)) = lo;
              *reinterpret_cast<uint4*>(dst + umma_off_c(r, 2 * jj + 1, CA)) = hi;
            }
          }
          if constexpr (Q) {
            // K5q: both fields read x = wt + 128 - thr (thr: this Gamma's
            // bound less the weight offset, as this thread sees it now), so
            // a codeword can lower the bound iff bit 7 of its byte is clear;
            // block 1 of the second chunk (scale 2^16) is the 2^23 offset.
            // Range (k5q_threshold): thr in [1, 128] keeps every field a
            // byte, thr >= wt - kQMaxSpan keeps the offset x <= 238, the
            // largest sum an A offset block encodes exactly (e2m1_block).
            // A threshold raised above the bound only sends more tiles down
            // the exact path.
            // The bound: this Gamma's word and this CTA's cache of it, and in
            // a fused launch the running minima of the earlier rounds (they
            // ran first, and the host's U will not exceed them; without them
            // a round would start from its loose start bound and send its
            // first tiles down the exact path).
            int ub = min(((volatile int*)ar.bound)[1 + c.gr.gamma], bnd_cache_read(s_bnd, rr, c.gr.gamma));
            for (int q = 0; q < rr; ++q) ub = min(ub, ((volatile const int*)bt.a[q].bound)[0]);
            if constexpr (FD) {
              // K5f: the tail word once per part, ta with the 2^23 block, tb
              // with X; the epilogue adds X to part a's bytes (thr | X << 16)
              const int thr = k5f_threshold(wt, ub - gamma_woff(ar, c.gr.gamma));
              const int x = wt + 128 - thr;
              *reinterpret_cast<uint4*>(dst + umma_off_c(r, W - 1, CA)) = k5f_a_tail(wk.acc[W - 1], 0, x);
              *reinterpret_cast<uint4*>(dst + umma_off_c(r, W, CA)) = k5f_a_tail(wk.acc[W - 1], 1, x);
              wt = thr | (x << 16);
            } else {
            const int thr = k5q_threshold(wt, ub - gamma_woff(ar, c.gr.gamma));
            const int x = wt + 128 - thr;
            *reinterpret_cast<uint4*>(dst + umma_off_c(r, W, CA)) = pad_chunk(x, 0);
            *reinterpret_cast<uint4*>(dst + umma_off_c(r, W + 1, CA)) = pad_chunk(x, 128);
            wt = thr;  // the epilogue needs thr to turn a byte back into a weight
            }
          } else if constexpr (WQ) {
            // K5w: chunk R = w(P) - thr, so both 11-bit fields read
            // x = w(P ^ S) + 1024 - thr (k5w_threshold keeps |R| <= 450)
            int ub = min(((volatile int*)ar.bound)[1 + c.gr.gamma], bnd_cache_read(s_bnd, rr, c.gr.gamma));
            for (int q = 0; q < rr; ++q) ub = min(ub, ((volatile const int*)bt.a[q].bound)[0]);
            const int thr = k5w_threshold(wt, ub - gamma_woff(ar, c.gr.gamma));
            *reinterpret_cast<uint4*>(dst + umma_off_c(r, k5w_data_chunks(W), CA)) = k5w_r_chunk(wt - thr);
            wt = thr;  // the epilogue turns a field back into a weight with it
          } else if constexpr (PR) {
            // offset chunks: w(P) for every part (so each field is a whole
            // stored weight), + 128 on the last (its scale 2^16 makes that the
            // 2^23 offset)
#pragma unroll
            for (int q = 0; q < CW; ++q)
              *reinterpret_cast<uint4*>(dst + umma_off_c(r, W + q, CA)) =
                  k5p_offset_chunk(q == CW - 1 ? wt + 128 : wt);
          }
          s_wt[(ab * kUmmaMA + j) * kUmmaM + r] = wt;
        }
        fence_proxy_async();  // generic-proxy writes -> tensor-core reads
        __syncwarp();
        if (lane == 0) mbar_arrive(afull(ab));
      }
      // visited combinations of this chunk
      const unsigned tot = __reduce_add_sync(FULL, (unsigned)cnt);
      const long long cols = min((long long)c.tile_hi * TR, (long long)c.slice) -
                             (long long)c.tile_lo * TR;
      if (lane == 0 && tot)
        atomicAdd(ar.combos + c.gr.gamma, (unsigned long long)tot * (unsigned long long)cols);
      if (ar.adds) {
        // one tensor-core addition per codeword (the prefix sum combined
        // with a stored suffix row), plus the walkers' prefix-XOR rows; the
        // walkers read one table row per addition and R[ell] per init (the
        // loader counts the stored rows it streams)
        const unsigned long long wsum = warp_sum_u64(wadd);
        const unsigned long long winit = (unsigned long long)__popc(__ballot_sync(FULL, cnt > 0));
        if (lane == 0) {
          atomicAdd(ar.adds + c.gr.gamma, wsum + (unsigned long long)tot * (unsigned long long)cols);
          atomicAdd(ar.accs + c.gr.gamma, wsum + winit);
        }
      }
    }
  } else if (warp < RL::LOAD) {
    // ================= MMA issuers: warp MMA0 + mb owns accumulator buffer
    // mb.  The whole warp runs the loop (warp-uniform values stay in uniform
    // registers); one elected lane issues the MMAs and commits.
    const int mb = warp - RL::MMA0;
    {
      const uint64_t a_desc0 = umma_desc(sA_s, 128, CA * 128);
      const uint64_t b_desc0 = umma_desc(sB_s, 128, CB * 128);
      const uint64_t b_fold0 = umma_desc(sB_s, (N / 8) * CB * 128, CB * 128);  // K5f tail fold
      (void)b_fold0;
      const uint32_t sfa = tmem + kSfCol, sfb = tmem + kSfCol + 8, sfm = tmem + kSfColMagic;
      const uint32_t sfp = tmem + kSfColPad;
      // magic operands: one core matrix per K chunk, SBO = 0 (every 8-row
      // group reads the same 8 rows)
      const uint32_t sM = (uint32_t)__cvta_generic_to_shared(sMagic);
      const uint64_t magic_a = umma_desc(sM, 128, 0), magic_b = umma_desc(sM + 256, 128, 0);
      const uint32_t dbase = tmem + (uint32_t)(mb * kUmmaMA * N);
      uint32_t grp = 0, tcount = 0, toff = k4_trace_off(a);
      for (uint32_t qi = 0;; ++qi) {
        const int qs = qi % kChunkQ;
        mbar_wait_fast_sel<8>(qfull(qs), (qi / kChunkQ) & 1);
        const long long qchunk = s_q[qs];
        __syncwarp();
        if (lane == 0) mbar_arrive(qempty(qs));
        if (qchunk < 0) break;
        const int rr = (int)((unsigned long long)qchunk >> kQRoundShift);
        const RoundArgs& ar = bt.a[rr];
        const unsigned long long chunk = (unsigned long long)qchunk & ((1ull << kQRoundShift) - 1);
        const K4Chunk c = k4_decode<TR>(plan_of(rr), ar.ngroups, chunk, k);
        k4_trace_chunk(a, toff, c.gr.ell, tcount);
        const int ntile = c.tile_hi - c.tile_lo;
        // Multi-GPU: any rank's running minimum of this round (the shared
        // mirror) tightens this CTA's cached bounds, so the producers'
        // thresholds follow the whole job's U, not just this rank's finds.
        // One peer load per chunk and CTA, issued here by the first issuer's
        // lane 0 and consumed at the chunk's end, so nothing waits for it
        // (polled by the loader before each chunk it cost a shard 27 us of
        // 460; held in the epilogue's registers across its tile loop, 9 us).
        // A minimum found here at or above the mirror's is then not published
        // -- the rank that holds the lower one reports it, and the fold over
        // ranks is a min (the same clip the earlier fused rounds' minima
        // apply).
        unsigned long long graw = ~0ull;
        if constexpr (QQ && BZ_GBOUND_THR)
          if (mb == 0 && lane == 0 && ar.gbound) graw = ((volatile unsigned long long*)ar.gbound)[ar.g];
        for (long long p = 0; p < c.maxcnt; p += kUmmaMA, ++grp) {
          const int ab = grp % NA;
          // first tile of this step that falls to this issuer
          // (every issuer waits for every step, so no issuer's arrivals run
          // ahead into a later phase of the A-buffer barriers)
          const int t0 = (int)((mb - (int)(tcount % ACC) + ACC) % ACC);
          mbar_wait_fast_sel<8>(afull(ab), (grp / NA) & 1);
          for (int i = t0; i < ntile; i += ACC) {
            const uint32_t tc = tcount + (uint32_t)i;  // global tile number
            const int stg = (int)(tc % S);
            // the B stage is normally long loaded: wait for it first, so the
            // accumulator hand-back (the critical loop) is the last wait
            // before the MMAs
            if (lane == 0) k4_trace(a, 5, tc, toff);
            mbar_wait_fast_sel<16>(bfull(stg), (tc / S) & 1);
            if (lane == 0) k4_trace(a, 6, tc, toff);
            const int valid = min(N, c.slice - (c.tile_lo + i) * TR);
#pragma unroll
            for (int h = 0; h < SPLIT; ++h) {
              if (!(a.debug & 128))  // timing experiment: MMAs never wait for the epilogue
                mbar_wait_fast_sel<16>(accempty(mb * SPLIT + h), ((tc / ACC) & 1) ^ 1);
              if (lane == 0 && h == 1) k4_trace(a, 13, tc, toff);
              if (!BZ_K5_NOFENCE) tc_fence_after();
              if (lane == 0 && h == 0) k4_trace(a, 1, tc, toff);
              // pass kb advances both start addresses by 32 bytes of K per
              // row = two core matrices = 256 B (16 in the 16-byte-granular
              // address field); part h starts NH/8 row groups into the tile
              const uint64_t bd0 =
                  b_desc0 + (uint64_t)(stg * (TB >> 4)) + (uint64_t)(h * (NH / 8) * CB * 8);
              if (elect_one()) {
                // a part holding no valid suffix is only committed (its
                // columns are masked anyway)
                if (PR && !(a.debug & 4)) {
                  // K5p / K5t: part q of the column (table rows [qN, (q+1)N)
                  // of the stage) with B scale 2^(8q) (K5t) / 2^(16q) (K5p);
                  // its last MMA reads A chunks W-1 and W+q (LBO (q+1)*128 B)
                  // so it meets offset chunk q
                  const uint32_t dj = dbase + (uint32_t)(h * NH);
                  const uint64_t adj = a_desc0 + (uint64_t)(ab * (TA >> 4));
                  if constexpr (WQ) {
                    // K5w: per part the data MMAs (part b with B scale 2^11),
                    // then one offset MMA of A chunks (R, Ca) / (R, Cb) (LBO
                    // 128 / 256 B) against the constant B operand
                    constexpr int WD = k5w_data_chunks(W);
                    const uint32_t sf1 = tmem + kSfCol, sf11 = tmem + kSfCol + 8;
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                      const uint64_t bdq = bd0 + (uint64_t)(q * (N / 8) * CB * 8);
#pragma unroll
                      for (int kb = 0; kb < WD / 2; ++kb)
                        umma_mxf4(dj, adj + 16u * kb, bdq + 16u * kb, IDESC, (q | kb) ? 1u : 0u,
                                  sf1, q ? sf11 : sf1);
                      umma_mxf4(dj, adj + 8u * WD + ((uint64_t)(8 * q) << 16), magic_b, IDESC, 1u,
                                q ? sfp : sfm, sf1);
                    }
                  } else if constexpr (FD) {
                    // K5f: the whole chunks per part (part b with B scale
                    // 256), then both parts' tails in one MMA: A chunks (ta,
                    // tb), B the last chunk of table rows c and N + c (LBO =
                    // N / 8 row groups)
                    constexpr int F2 = (W - 1) / 2;
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                      const uint64_t bdq = bd0 + (uint64_t)(q * (N / 8) * CB * 8);
#pragma unroll
                      for (int kb = 0; kb < F2; ++kb)
                        umma_nvf4(dj, adj + 16u * kb, bdq + 16u * kb, IDESC, (q | kb) ? 1u : 0u,
                                  sfa, q ? sfm : sfa);
                    }
                    const uint64_t bfold = b_fold0 + (uint64_t)(stg * (TB >> 4)) + 8u * (W - 1) +
                                           (uint64_t)(h * (NH / 8) * CB * 8);
                    umma_nvf4(dj, adj + 8u * (W - 1), bfold, IDESC, F2 ? 1u : 0u, sfp, sfb);
                  } else if constexpr (Q && !(W & 1)) {
                    // K5q, even W: W/2 data MMAs per part, then one offset MMA
                    // of A chunks (pad_a, pad_b) against a constant B
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                      const uint64_t bdq = bd0 + (uint64_t)(q * (N / 8) * CB * 8);
#pragma unroll
                      for (int kb = 0; kb < W / 2; ++kb)
                        umma_nvf4(dj, adj + 16u * kb, bdq + 16u * kb, IDESC, (q | kb) ? 1u : 0u,
                                  sfa, q ? sfm : sfb);
                      umma_nvf4(dj, adj + 16u * (W / 2), q ? magic_b : magic_a, IDESC, 1u,
                                q ? sfp : sfa, q ? sfm : sfb);
                    }
                  } else
#pragma unroll
                  for (int q = 0; q < NC; ++q) {
                    const uint64_t bdq = bd0 + (uint64_t)(q * (N / 8) * CB * 8);
                    const uint32_t sfq = q == 0 ? sfb : (CW == 3 && q == 1 ? sfp : sfm);
#pragma unroll
                    for (int kb = 0; kb < P; ++kb) {
                      const uint64_t ad = adj + 16u * kb + (kb == P - 1 ? (uint64_t)(8 * q) << 16 : 0ull);
                      if constexpr (Q)  // K5q: A scale 256 on the offset block of the last MMA
                        umma_nvf4(dj, ad, bdq + 16u * kb, IDESC, (q | kb) ? 1u : 0u,
                                  (q == 1 && kb == P - 1) ? sfp : sfa, sfq);
                      else
                        umma_mxf4(dj, ad, bdq + 16u * kb, IDESC, (q | kb) ? 1u : 0u, sfa, sfq);
                    }
                  }
                } else if (!(a.debug & 4) && valid > h * NH) {
#pragma unroll
                  for (int j = 0; j < kUmmaMA; ++j) {
                    const uint32_t dj = dbase + (uint32_t)(j * N + h * NH);
                    const uint64_t adj = a_desc0 + (uint64_t)((ab * kUmmaMA + j) * (TA >> 4));
                    constexpr bool kExtra = F4 && MG && !k5_padmagic(W);
                    if constexpr (kExtra) umma_mxf4(dj, magic_a, magic_b, IDESC, 0u, sfm, sfb);
#pragma unroll
                    for (int kb = 0; kb < P; ++kb) {
                      if constexpr (F4)
                        umma_mxf4(dj, adj + 16u * kb, bd0 + 16u * kb, IDESC,
                                  (kb > 0 || kExtra) ? 1u : 0u,
                                  (k5_padmagic(W) && kb == P - 1) ? sfp : sfa, sfb);
                      else
                        umma_i8(dj, adj + 16u * kb, bd0 + 16u * kb, IDESC, kb > 0 ? 1u : 0u);
                    }
                  }
                }
                umma_commit(accfull(mb * SPLIT + h));
                if (h == SPLIT - 1) umma_commit(bempty(stg));
              }
              __syncwarp();
              if (lane == 0 && h == 0) k4_trace(a, 12, tc, toff);
            }
            if (lane == 0) k4_trace(a, 4, tc, toff);
          }
          // the A buffer is free once every issuer's MMAs on it completed
          if (elect_one()) umma_commit(aempty(ab));
          __syncwarp();
          tcount += (uint32_t)ntile;
        }
        if constexpr (QQ && BZ_GBOUND_THR)
          if (ar.gbound && (graw >> 32) == (ar.gtag >> 32)) {  // this run's word (cf. gbound_read)
            const int sv = (int)(unsigned)(graw & 0xffffffffull);
            for (int j = 0; j < ar.m && j < kBndPerRound; ++j)
              atomicMin(s_bnd + rr * kBndPerRound + j, sv);
          }
      }
    }
    __syncwarp();
  } else {
    // ================= loader: TMA bulk copies of triple tiles, and the
    // chunk queue.  Chunks are published up to kChunkQ ahead of the one
    // being loaded (non-blocking between tiles), so the producers' walker
    // unrank and first A rows of the next chunk overlap this chunk's tiles
    // instead of waiting for its last TMA.
    if (lane == 0) {
      uint32_t bcount = 0, toff = k4_trace_off(a);
      volatile int* vb = a.bound;
      uint32_t qpub = 0;   // chunk entries published
      bool qdone = false;  // the -1 entry is out
      // publish queue entries while slots are free (blocking for the first
      // one when `block`); never more than kChunkQ ahead of entry `qload`
      auto publish = [&](uint32_t qload, bool block) {
        while (!qdone && qpub < qload + kChunkQ) {
          const int qs = qpub % kChunkQ;
          const uint32_t par = ((qpub / kChunkQ) & 1) ^ 1;
          if (block) {
            mbar_wait_sel<32>(qempty(qs), par);
            block = false;
          } else {
            uint32_t ok;
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(qempty(qs)), "r"(par)
                : "memory");
            if (!ok) return;
          }
          // next chunk of this shard, or -1 (done, or U reached L_prev)
          // (the fused rounds' chunk spaces one after the other on round
          // 0's cursor; round_done: this round's or the previous round's
          // running minimum -- local, chained, or any rank's through the
          // shared mirror -- already meets L_prev, so the run has ended at
          // or before this round and every later round is void too)
          const unsigned long long cidx = atomicAdd(a.counter, 1ull);
          int rq = 0;
          while (rq + 1 < bt.count && cidx >= bt.cend[rq]) ++rq;
          const RoundArgs& aq = bt.a[rq];
          const unsigned long long local = cidx - (rq > 0 ? bt.cend[rq - 1] : 0ull);
          const unsigned long long ch = local * (unsigned long long)aq.nshards + aq.shard;
          (void)vb;
          const long long qchunk = (cidx < bt.cend[bt.count - 1] && ch < aq.nchunks && !round_done(aq))
                                       ? (long long)(((unsigned long long)rq << kQRoundShift) | ch)
                                       : -1;
          s_q[qs] = qchunk;
          long long* ct = k4_ctrace(a, qpub);
          if (ct) { ct[0] = qchunk; ct[1] = clock64(); }
          mbar_arrive(qfull(qs));
          ++qpub;
          if (qchunk < 0) qdone = true;
        }
      };
      for (uint32_t qload = 0;; ++qload) {
        publish(qload, qload == qpub);
        const long long qchunk = s_q[qload % kChunkQ];
        if (qchunk < 0) break;
        const int rr = (int)((unsigned long long)qchunk >> kQRoundShift);
        const RoundArgs& ar = bt.a[rr];
        const unsigned long long chunk = (unsigned long long)qchunk & ((1ull << kQRoundShift) - 1);
        const K4Chunk c = k4_decode<TR>(plan_of(rr), ar.ngroups, chunk, k);
        k4_trace_chunk(a, toff, c.gr.ell, bcount);
        if (ar.accs) {
          // stored suffix rows streamed into shared memory: every tile of
          // the chunk once per prefix step, each shared by up to 128 prefixes
          const long long cols = min((long long)c.tile_hi * TR, (long long)c.slice) -
                                 (long long)c.tile_lo * TR;
          atomicAdd(ar.accs + c.gr.gamma, (unsigned long long)c.maxcnt * (unsigned long long)cols);
        }
        const int lvl = c.gr.depth - 3;  // suffix table of this group's level
        const uint8_t* tsrc =
            tabs.t[lvl] + (size_t)c.gr.gamma * tabs.stride_rows[lvl] * (CB * 16);
        for (long long p = 0; p < c.maxcnt; p += kUmmaMA) {
          for (int t = c.tile_lo; t < c.tile_hi; ++t, ++bcount) {
            const int stg = bcount % S;
            mbar_wait_sel<32>(bempty(stg), ((bcount / S) & 1) ^ 1);
            k4_trace(a, 0, bcount, toff);
            // only the rows this tile needs (8-row granularity); the rest of
            // the stage keeps stale rows whose columns the epilogue masks
            // (K5p/K5q/K5t: always the whole tile -- every part of a column
            // must hold in-range table rows, which the empty-subset tail
            // provides)
            const int valid = min(TR, c.slice - t * TR);
            const uint32_t bytes = PR ? TB : (uint32_t)((valid + 7) / 8) * (CB * 128);
            if (a.debug & 2) {
              mbar_arrive(bfull(stg));
            } else {
              mbar_arrive_tx(bfull(stg), bytes);
              tma_load_1d(sB_s + stg * TB, tsrc + (size_t)t * TB, bytes, bfull(stg));
              k4_trace(a, 15, bcount, toff);
            }
            publish(qload + 1, false);
          }
        }
      }
    }
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (life && tid == 0) life[2] = global_ns();
  if (warp == RL::MMA0) {
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

// tcgen05 kind::mxf4 throughput probe (roofline denominator of K5): one CTA
// per SM issues `iters` back-to-back M=128 x N=240 x K=64 block-scaled MMAs
// (unit scales in TMEM) alternating between the two accumulators.
__global__ void __launch_bounds__(128, 1) peak_umma_mxf4(int iters, long long* clk) {
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
  for (int c = 0; c < 512 - kSfCol; c += 8)
    tmem_st8(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(kSfCol + c), 0x7F7F7F7Fu);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  if (threadIdx.x == 0) {
    const uint64_t ad = umma_desc(base, 128, 256);
    const uint64_t bd = umma_desc(base + 128 * 32, 128, 256);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
      umma_mxf4(tmem + (uint32_t)((i & 1) * kUmmaN4), ad, bd, kMxf4Idesc, (i & 2) ? 1u : 0u,
                tmem + kSfCol, tmem + kSfCol + 8);
    umma_commit(bar_s);
    mbar_wait(bar_s, 0);
    clk[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace bz
