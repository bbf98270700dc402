// bz_kernels.cuh -- sm_100a enumeration kernels for the Brouwer-Zimmermann
// minimum-distance round (the hot path of arXiv 1603.06757's mindist
// package, pkg/src/mindist/enumeration.py:76-444).
//
// Work decomposition:
//   A g-combination {c_1 < ... < c_g} of the k rows of Gamma_j is split into
//   a prefix {c_1..c_{g-1}} with last element ell = c_{g-1} and a suffix
//   element e = c_g in (ell, k).  Prefixes with the same ell form a *group*:
//   they are the (g-2)-subsets of [0, ell) plus ell itself, C(ell, g-2) of
//   them, each extended by the same k-1-ell suffix rows.  A warp takes a
//   chunk of one group; each lane owns a contiguous colex range of its
//   prefixes, keeps the prefix XOR in registers and steps through its range
//   with Gosper's successor (three prefix-XOR-table rows per step, branch
//   free).  All lanes then run the SAME suffix loop e = ell+1 .. k-1, so
//   row e is one broadcast shared-memory read reused by 32 lanes and there
//   is no divergence in the hot loop:
//        w = sum_j popc(acc[j] ^ row_e[j]);   best = min(best, w)
//   (W LOP3 + W POPC + IADD3s + one IMNMX per codeword).
//   This is the warp-scale form of the paper's "saved additions" and
//   "unrolling" ideas: every codeword costs
//   one row XOR per word, and every row access is shared by 32 codewords.
//
// Scheduling: chunks are handed out dynamically through one global 64-bit
// counter (the GPU analogue of the reference's locked unit cursor,
// enumeration.py:413-423).  Multi-GPU shards take every nshards-th chunk.
//
// Early exit: the running round minimum lives in bound[0]; a warp stops
// taking chunks once bound[0] <= lower_prev (the only exit that keeps the
// reference's bounds trace bit-exact, SURVEY.md 8(a) invariant 5).
#pragma once

#include <cstdint>
#include <climits>

namespace bz {

constexpr int kMaxK = 128;
constexpr int kMaxW = 8;
constexpr int kBinomDim = kMaxK + 1;  // C(p, q) for 0 <= p, q <= 128

struct Group {
  unsigned long long chunk_begin;  // first global chunk index of the group
  unsigned long long nprefix;      // C(ell, g-1-D) prefixes in the group
  int gamma;                       // matrix index
  int ell;                         // last prefix element (-1 when g == 1)
  int ppl;                         // prefixes per lane per chunk
  int depth;                       // suffix depth D (1, 2 or 3; K5 levels 3..5)
  int tpc;                         // D = 3: suffix tiles per chunk
  int ntb;                         // D = 3: tile blocks per prefix block
  int lanes;                       // prefixes walked in parallel per chunk
  int tile_rows;                   // D >= 3: suffixes per table tile
  int slice;                       // suffixes per prefix: C(k - sfloor, D)
  int sfloor;                      // smallest suffix row: max(ell + 1, level floor)
  int sl;                          // K1: suffix lanes per prefix block (1, 2, .., 32);
                                   // K5 family: 1, or 0 for a merged group -- its
                                   // prefixes are the (g - D)-subsets of [0, ell + 1),
                                   // nprefix = C(ell + 1, g - D), no fixed last row
};

struct RoundArgs {
  const uint32_t* rows;        // m * k * WP words (padded rows)
  const uint32_t* px;          // m * (k+1) * WP prefix-XOR table
  const Group* groups;         // ngroups, sorted by chunk_begin
  const unsigned long long* binom;  // kBinomDim^2 saturating binomials
  int* bound;                  // [0] round minimum, [1+j] per-Gamma minimum
  unsigned long long* combos;  // per-Gamma visited combinations
  // per-Gamma row-level operation counters (null: not counted), the
  // device analogue of the reference's (m/enumeration.py:19-24):
  // adds = full-row additions (XORs, and the tensor-core dot products that
  // combine a prefix sum with a stored row), accs = rows brought into the
  // working set (table rows a warp / CTA loads once for all its codewords)
  unsigned long long* adds;
  unsigned long long* accs;
  unsigned long long* counter; // dynamic chunk cursor
  unsigned long long* hist;    // n+1 bins (histogram kernel only)
  unsigned long long nchunks;  // chunks of the whole round (all shards)
  int ngroups;
  int m, k, g, n;
  int shard, nshards;
  int lower_prev;              // the run's lower bound before this round (L_prev)
  int exit_own;                // 1: stop once this round's own minimum meets L_prev
                               // (in-round early exit, bz_set_early_exit); the
                               // previous round's U meeting it (the run ended:
                               // a batched round past termination) always stops
  unsigned long long elide;    // bit j: Gamma j's identity columns were dropped at load
                               // time, so its codeword weights get + g (see bz_load_gammas)
  int debug;                   // K4 timing experiments only (see BZ_K4_DEBUG)
  long long* trace;            // K4 debug timeline (BZ_K4_DEBUG & 8), else null
  int trace_from;              // first traced tile (BZ_K4_TRACE_FROM)
  int trace_ell;               // or: from the first chunk with ell >= this (BZ_K4_TRACE_ELL)
  long long* ctrace;           // K4/K5 per-chunk timeline (BZ_K4_DEBUG & 32), else null
  const int* chain;            // batched rounds: the previous round's bounds (its U
                               // after the round tightens this round's start), or null
  int sgroups_cap;             // shared-memory room for this many groups (fused K1
                               // launches stage several plans in turn), 0 = ngroups
  int groups_global;           // 1: the plan is too large to stage in shared memory
                               // (many groups at large k); read it from global
                               // memory (L2-resident) instead
  // Multi-GPU: the running minimum of every round g across all ranks, one
  // 64-bit word per g in one rank's device memory, mapped into every rank
  // (CUDA IPC over NVLink) -- kernels RED.MIN their chunk minima into it and
  // read it for the early exits, so a rank stops as soon as ANY rank has
  // met the bound.  Words carry the run's tag in their high half (newer
  // runs have smaller tags and win the min; stale words read as empty).
  // Null on a single device.
  unsigned long long* gbound;
  unsigned long long gtag;     // (0xffffffff - epoch) << 32
};

// shared-bound helpers (no-ops without a mapped mirror)
__device__ __forceinline__ int gbound_read(const RoundArgs& a, int g) {
  if (!a.gbound || g < 1) return INT_MAX;
  const unsigned long long v = ((volatile unsigned long long*)a.gbound)[g];
  return (v >> 32) == (a.gtag >> 32) ? (int)(unsigned)(v & 0xffffffffull) : INT_MAX;
}
__device__ __forceinline__ void gbound_publish(const RoundArgs& a, int w) {
  if (a.gbound && w >= 0) atomicMin(a.gbound + a.g, a.gtag | (unsigned long long)(unsigned)w);
}
// Round start (one thread of the grid): the running U the previous round
// ended with -- chained on this device, or any rank's through the shared
// mirror -- clips this round's bounds, and the mirror word of this round
// inherits the previous one, so it carries the global running U after
// round g (what the next round's termination test needs).
__device__ __forceinline__ void round_start(const RoundArgs& a) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int u = INT_MAX;
  if (a.chain) u = ((volatile const int*)a.chain)[0];
  const int v = gbound_read(a, a.g - 1);
  if (v < u) u = v;
  if (u == INT_MAX) return;
  for (int j = 0; j <= a.m; ++j) atomicMin(a.bound + j, u);
  if (v < INT_MAX) gbound_publish(a, v);
}

// a round may stop taking work: the previous round's running U (chain /
// shared mirror) already meets L_prev -- the run has terminated and this
// batched round's result will be discarded -- or, with the in-round early
// exit on, this round's own running minimum (or any rank's) meets it, so
// the round's result is exactly L_prev
__device__ __forceinline__ bool round_done(const RoundArgs& a) {
  if (a.exit_own && ((volatile const int*)a.bound)[0] <= a.lower_prev) return true;
  if (a.chain && ((volatile const int*)a.chain)[0] <= a.lower_prev) return true;
  if (a.gbound && ((a.exit_own && gbound_read(a, a.g) <= a.lower_prev) ||
                   gbound_read(a, a.g - 1) <= a.lower_prev))
    return true;
  return false;
}

__host__ __device__ constexpr int padded_words(int w) {
  return w <= 1 ? 1 : (w <= 2 ? 2 : (w <= 4 ? 4 : 8));
}

// Prefix-XOR rows are read at lane-divergent indices; an odd row stride in
// shared memory spreads them over distinct banks (scalar LDS per word).
__host__ __device__ constexpr int px_stride(int w) { return (w & 1) ? w : w + 1; }

// 128-bit subset mask over row indices [0, 128).
struct Mask {
  unsigned long long lo, hi;
};

__device__ __forceinline__ int mask_ctz(const Mask& x) {
  return x.lo ? __ffsll((long long)x.lo) - 1 : 64 + __ffsll((long long)x.hi) - 1;
}

__device__ __forceinline__ int mask_popc(const Mask& x) {
  return __popcll(x.lo) + __popcll(x.hi);
}

__device__ __forceinline__ Mask mask_shr(const Mask& x, int s) {
  Mask r;
  if (s >= 128) {
    r.lo = r.hi = 0;
  } else if (s >= 64) {
    r.lo = x.hi >> (s - 64);
    r.hi = 0;
  } else if (s == 0) {
    r = x;
  } else {
    r.lo = (x.lo >> s) | (x.hi << (64 - s));
    r.hi = x.hi >> s;
  }
  return r;
}

// Colex successor of a q-subset (Gosper's hack on 128 bits).  Returns the
// three prefix-XOR-table indices whose rows XOR to the change of the
// subset's row sum: the low run [s, s+L) is removed, bit s+L and the bits
// [0, L-1) are added, so  delta = PX[s] ^ PX[s+L+1] ^ PX[L-1].
__device__ __forceinline__ void colex_next(Mask& x, int& i0, int& i1, int& i2) {
  const int s = mask_ctz(x);
  Mask u;
  u.lo = s < 64 ? (1ull << s) : 0ull;
  u.hi = s < 64 ? 0ull : (1ull << (s - 64));
  Mask v;
  v.lo = x.lo + u.lo;
  v.hi = x.hi + u.hi + (v.lo < x.lo ? 1ull : 0ull);
  Mask d;
  d.lo = v.lo ^ x.lo;
  d.hi = v.hi ^ x.hi;
  const int l1 = mask_popc(d);  // run length + 1
  Mask t = mask_shr(d, s + 2);
  x.lo = v.lo | t.lo;
  x.hi = v.hi | t.hi;
  i0 = s;
  i1 = s + l1;
  i2 = l1 - 2;
}

// Colex unrank of rank r among the q-subsets of [0, ell).
// Shared-memory copy of C(c, i) for c < 128, i <= kSBinomQ (row-major,
// kSBinomQ + 1 per row): walker unranks read it instead of the 133 KB global
// table, whose L2 round trips made a chunk start cost microseconds.
constexpr int kSBinomQ = 8;
constexpr int kSBinomBytes = kMaxK * (kSBinomQ + 1) * 8;

__device__ __forceinline__ Mask colex_unrank(unsigned long long r, int q, int ell,
                                             const unsigned long long* __restrict__ binom,
                                             const unsigned long long* sb) {
  Mask x{0ull, 0ull};
  int c = ell - 1;
  if (q <= kSBinomQ) {
    // element i: the largest c' <= c with C(c', i) <= r (binary search;
    // C(i - 1, i) = 0 bounds it below)
    for (int i = q; i >= 1; --i) {
      int lo = i - 1, hi = c;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sb[mid * (kSBinomQ + 1) + i] <= r) lo = mid; else hi = mid - 1;
      }
      c = lo;
      r -= sb[c * (kSBinomQ + 1) + i];
      if (c < 64) x.lo |= 1ull << c; else x.hi |= 1ull << (c - 64);
      --c;
    }
    return x;
  }
  for (int i = q; i >= 1; --i) {
    while (__ldg(binom + c * kBinomDim + i) > r) --c;
    r -= __ldg(binom + c * kBinomDim + i);
    if (c < 64) x.lo |= 1ull << c; else x.hi |= 1ull << (c - 64);
    --c;
  }
  return x;
}

template <int W>
__device__ __forceinline__ void load_row(uint32_t (&r)[W], const uint32_t* p) {
  constexpr int WP = padded_words(W);
  if constexpr (W == 5 || W == 6 || W == 7) {
    const uint4 v = reinterpret_cast<const uint4*>(p)[0];
    r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
    if constexpr (W == 5) {
      r[4 % W] = p[4];
    } else {
      const uint2 u = reinterpret_cast<const uint2*>(p)[2];
      r[4 % W] = u.x; r[5 % W] = u.y;
      if constexpr (W == 7) r[6 % W] = p[6];
    }
  } else if constexpr (WP >= 4) {
#pragma unroll
    for (int j = 0; j < WP / 4; ++j) {
      const uint4 v = reinterpret_cast<const uint4*>(p)[j];
      if (4 * j + 0 < W) r[(4 * j + 0) % W] = v.x;
      if (4 * j + 1 < W) r[(4 * j + 1) % W] = v.y;
      if (4 * j + 2 < W) r[(4 * j + 2) % W] = v.z;
      if (4 * j + 3 < W) r[(4 * j + 3) % W] = v.w;
    }
  } else if constexpr (WP == 2) {
    const uint2 v = reinterpret_cast<const uint2*>(p)[0];
    r[0] = v.x;
    if (W > 1) r[W > 1 ? 1 : 0] = v.y;
  } else {
    r[0] = p[0];
  }
}

template <int W>
__device__ __forceinline__ void xor_row(uint32_t (&acc)[W], const uint32_t* p) {
  uint32_t r[W];
  load_row<W>(r, p);
#pragma unroll
  for (int j = 0; j < W; ++j) acc[j] ^= r[j];
}

template <int W>
__device__ __forceinline__ int weight_xor(const uint32_t (&acc)[W], const uint32_t (&r)[W]) {
  int w = 0;
#pragma unroll
  for (int j = 0; j < W; ++j) w += __popc(acc[j] ^ r[j]);
  return w;
}

template <int W>
__device__ __forceinline__ void xor_px(uint32_t (&acc)[W], const uint32_t* px, int i) {
  constexpr int PS = px_stride(W);
#pragma unroll
  for (int j = 0; j < W; ++j) acc[j] ^= px[i * PS + j];
}

// One lane-private walker over consecutive colex ranks of the (g-2)-subsets
// of [0, ell): subset mask + XOR of its rows and of row ell.
template <int W>
struct Walker {
  Mask x;
  uint32_t acc[W];

  // The prefix of colex rank `rank`: a q-subset of [0, ell) plus row ell --
  // or, for a merged group (fixed = false: every prefix whose last element is
  // below a level's floor shares one suffix slice, and those prefixes are
  // consecutive in colex order), a q-subset of [0, ell) alone.
  __device__ __forceinline__ void init(unsigned long long rank, int q, int ell,
                                       const uint32_t* R, const unsigned long long* binom,
                                       const unsigned long long* sb, bool fixed = true) {
    constexpr int WP = padded_words(W);
#pragma unroll
    for (int j = 0; j < W; ++j) acc[j] = 0u;
    x = Mask{0ull, 0ull};
    if (ell < 0) return;
    if (fixed) xor_row<W>(acc, R + ell * WP);
    if (q > 0) {
      x = colex_unrank(rank, q, ell, binom, sb);
      Mask y = x;
      while (y.lo | y.hi) {
        const int b = mask_ctz(y);
        xor_row<W>(acc, R + b * WP);
        if (b < 64) y.lo &= y.lo - 1; else y.hi &= y.hi - 1;
      }
    }
  }

  // colex successor; PX[0] = 0, so the third row only matters for runs > 1.
  // Returns the prefix-XOR rows it added (2 or 3).
  __device__ __forceinline__ int step(const uint32_t* PX) {
    int i0, i1, i2;
    colex_next(x, i0, i1, i2);
    xor_px<W>(acc, PX, i0);
    xor_px<W>(acc, PX, i1);
    if (i2 > 0) xor_px<W>(acc, PX, i2);
    return i2 > 0 ? 3 : 2;
  }
};

// 64-bit sum over the warp (all lanes active)
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Weight of the dropped identity columns of Gamma j: every chosen row has
// exactly one of them set.
__device__ __forceinline__ int gamma_woff(const RoundArgs& a, int gamma) {
  return (gamma < 64 && ((a.elide >> gamma) & 1ull)) ? a.g : 0;
}

// Locate the group owning `chunk` (groups sorted by chunk_begin).
__device__ __forceinline__ int find_group(const Group* sg, int ngroups,
                                          unsigned long long chunk) {
  int lo = 0, hi = ngroups - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sg[mid].chunk_begin <= chunk) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Shared-memory layout: rows | px | groups  (+ per-thread u16 histogram)
template <int W>
__host__ __device__ inline size_t smem_base_bytes(int m, int k, int ngroups) {
  constexpr int WP = padded_words(W);
  constexpr int PS = px_stride(W);
  size_t words = (size_t)m * k * WP + (size_t)m * (k + 1) * PS;
  size_t bytes = words * 4;
  bytes = (bytes + 15) & ~size_t(15);
  bytes += (size_t)ngroups * sizeof(Group);
  bytes = (bytes + 15) & ~size_t(15);
  return bytes + kSBinomBytes;  // the small binomial table (colex_unrank)
}

// groups held in shared memory (0 when the plan is read from global memory)
__host__ __device__ inline int staged_groups(const RoundArgs& a) {
  return a.groups_global ? 0 : (a.ngroups > a.sgroups_cap ? a.ngroups : a.sgroups_cap);
}

// the small binomial table at the end of the staged region
template <int W>
__device__ __forceinline__ unsigned long long* smem_binom(unsigned char* smem, const RoundArgs& a) {
  return reinterpret_cast<unsigned long long*>(
      smem + smem_base_bytes<W>(a.m, a.k, staged_groups(a)) - kSBinomBytes);
}

// dst[i] = load(i) for i < n, block-strided, 8 loads in flight per thread
template <typename Load, typename T>
__device__ __forceinline__ void stage_copy(int n, Load&& load, T* dst) {
  constexpr int U = 8;
  for (int base = threadIdx.x; base < n; base += U * blockDim.x) {
    T t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * (int)blockDim.x;
      if (i < n) t[u] = load(i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * (int)blockDim.x;
      if (i < n) dst[i] = t[u];
    }
  }
}

// the round's work plan into shared memory
__device__ __forceinline__ void stage_groups(const RoundArgs& a, Group* sgroups) {
  const uint32_t* gsrc = reinterpret_cast<const uint32_t*>(a.groups);
  stage_copy(a.ngroups * (int)(sizeof(Group) / 4), [&](int i) { return gsrc[i]; },
             reinterpret_cast<uint32_t*>(sgroups));
}

template <int W>
__device__ __forceinline__ void stage(const RoundArgs& a, uint32_t*& srows,
                                      uint32_t*& spx, Group*& sgroups,
                                      unsigned char* smem) {
  constexpr int WP = padded_words(W);
  constexpr int PS = px_stride(W);
  const int nrow_words = a.m * a.k * WP;
  const int npx_rows = a.m * (a.k + 1);
  const int npx_words = npx_rows * PS;
  srows = reinterpret_cast<uint32_t*>(smem);
  spx = srows + nrow_words;
  size_t off = ((size_t)(nrow_words + npx_words) * 4 + 15) & ~size_t(15);
  sgroups = reinterpret_cast<Group*>(smem + off);
  // every copy issues 8 predicated loads per thread before its stores: a
  // load-store chain (what a bounds-checked unrolled loop compiles to) pays
  // one L2 round trip per element and made short launches' prologues cost
  // microseconds
  stage_copy(nrow_words, [&](int i) { return a.rows[i]; }, srows);
  stage_copy(npx_words, [&](int i) {
    const int r = i / PS, j = i - r * PS;
    return j < W ? a.px[r * WP + j] : 0u;
  }, spx);
  if (a.groups_global)
    sgroups = const_cast<Group*>(a.groups);
  else
    stage_groups(a, sgroups);
  unsigned long long* sb = smem_binom<W>(smem, a);
  stage_copy(kMaxK * (kSBinomQ + 1), [&](int i) {
    const int c = i / (kSBinomQ + 1), j = i - c * (kSBinomQ + 1);
    return a.binom[c * kBinomDim + j];
  }, sb);
  __syncthreads();
}

// Suffix enumeration of one prefix (row sum `acc`, last element ell):
//   D = 1: codewords acc ^ R[e]           for ell < e < k
//   D = 2: codewords acc ^ R[e1] ^ R[e2]  for ell < e1 < e2 < k
// Two prefixes (walkers A and B) share every broadcast row load.  `visit`
// receives the weight of each codeword of A and of B.
template <int W, int D, typename Visit>
__device__ __forceinline__ void suffix_pair(const uint32_t (&a)[W], const uint32_t (&b)[W],
                                            const uint32_t* R, int e0, int k, int s0, int ss,
                                            Visit&& visit) {
  constexpr int WP = padded_words(W);
  // this lane's share of the first suffix row: e0 + s0, e0 + s0 + ss, ...
  // (ss = the group's suffix lanes; 1: every row)
  if constexpr (D == 1) {
    const uint32_t* re = R + (e0 + s0) * WP;
#pragma unroll 2
    for (int e = e0 + s0; e < k; e += ss, re += ss * WP) {
      uint32_t r0[W];
      load_row<W>(r0, re);
      visit(weight_xor<W>(a, r0), weight_xor<W>(b, r0));
    }
  } else {
    const uint32_t* r1p = R + (e0 + s0) * WP;
#pragma unroll 1
    for (int e1 = e0 + s0; e1 < k - 1; e1 += ss, r1p += ss * WP) {
      uint32_t r1[W], a1[W], b1[W];
      load_row<W>(r1, r1p);
#pragma unroll
      for (int j = 0; j < W; ++j) {
        a1[j] = a[j] ^ r1[j];
        b1[j] = b[j] ^ r1[j];
      }
      const uint32_t* re = r1p + WP;
#pragma unroll 2
      for (int e2 = e1 + 1; e2 < k; ++e2, re += WP) {
        uint32_t r0[W];
        load_row<W>(r0, re);
        visit(weight_xor<W>(a1, r0), weight_xor<W>(b1, r0));
      }
    }
  }
}

template <int D>
__device__ __forceinline__ unsigned long long suffix_count(int k, int e0) {
  const unsigned long long t = (unsigned long long)(k - e0);
  return D == 1 ? t : t * (t - 1) / 2;
}

// A lane's share of one prefix's suffixes (first row e0 + s0, stride ss):
// codewords, and for D = 2 the partial sums prefix ^ R[e1] it forms
template <int D>
__device__ __forceinline__ void lane_suffixes(int k, int e0, int s0, int ss,
                                              unsigned long long& words,
                                              unsigned long long& partial) {
  const int f = e0 + s0;
  const int last = D == 1 ? k : k - 1;  // first-row values below `last`
  const long long t = f < last ? (last - f + ss - 1) / ss : 0;
  if (D == 1) {
    words = (unsigned long long)t;
    partial = 0ull;
  } else {
    // sum over j < t of (k - 1 - (f + j ss))
    words = (unsigned long long)(t * (long long)(k - 1 - f) - (long long)ss * t * (t - 1) / 2);
    partial = (unsigned long long)t;
  }
}

// Shared prologue of a chunk: the lane's prefix range [first, first+cnt).
struct ChunkView {
  Group gr;
  unsigned long long first;
  long long cnt;
  int s0;  // this lane's first suffix offset (stride gr.sl)
};

// K1 lanes: 32 / sl prefix blocks of ppl colex ranks (block-major) x sl
// suffix lanes sharing each block (lane = block * sl + s0)
__device__ __forceinline__ ChunkView open_chunk(const Group* sg, int ngroups,
                                                unsigned long long chunk, int lane) {
  ChunkView v;
  v.gr = sg[find_group(sg, ngroups, chunk)];
  const unsigned long long local = chunk - v.gr.chunk_begin;
  const int sl = v.gr.sl;
  v.s0 = lane & (sl - 1);
  v.first = (local * (unsigned long long)(32 / sl) + (unsigned long long)(lane / sl)) *
            (unsigned long long)v.gr.ppl;
  v.cnt = 0;
  if (v.first < v.gr.nprefix) {
    const unsigned long long left = v.gr.nprefix - v.first;
    v.cnt = left < (unsigned long long)v.gr.ppl ? (long long)left : v.gr.ppl;
  }
  return v;
}

// ---------------------------------------------------------------------------
// K1: minimum-weight enumeration of one round (all Gammas, one shard).
// Each lane runs two walkers over the two halves of its prefix range so that
// every broadcast row load feeds two codewords (and two independent
// XOR/POPC chains).  When the range is odd the second walker duplicates the
// first on the last step -- harmless for a minimum.
// One chunk (a warp's share of the plan) of round a.
// Per-block tallies of one round in shared memory: a chunk's counts and
// minimum go here with shared-memory atomics and reach the round's global
// words once per block (k1_tally_flush) -- thousands of short chunks of a
// small round otherwise queue that many atomics on the same few L2 words.
// A chunk minimum below the block's best so far is still published at once.
constexpr int kTallyM = 16;  // Gammas tallied per block (more: per-chunk atomics)
struct K1Tally {
  unsigned long long combos[kTallyM], adds[kTallyM], accs[kTallyM];
  int best[kTallyM];
};

__device__ __forceinline__ void k1_tally_init(K1Tally* t, int count) {
  for (int i = threadIdx.x; i < count * kTallyM; i += blockDim.x) {
    K1Tally& u = t[i / kTallyM];
    const int j = i % kTallyM;
    u.combos[j] = u.adds[j] = u.accs[j] = 0ull;
    u.best[j] = INT_MAX;
  }
}

// after a __syncthreads that follows every chunk of the block
__device__ __forceinline__ void k1_tally_flush(const RoundArgs& a, const K1Tally& t) {
  const int m = min(a.m, kTallyM);
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    if (t.combos[j]) atomicAdd(a.combos + j, t.combos[j]);
    if (a.adds && t.adds[j]) atomicAdd(a.adds + j, t.adds[j]);
    if (a.accs && t.accs[j]) atomicAdd(a.accs + j, t.accs[j]);
  }
}

template <int W, int D>
__device__ __forceinline__ void k1_chunk(const RoundArgs& a, unsigned long long chunk,
                                         const uint32_t* srows, const uint32_t* spx,
                                         const Group* sgroups, const unsigned long long* sbinom,
                                         K1Tally* tally) {
  constexpr int WP = padded_words(W);
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int k = a.k, q = a.g - 1 - D;

  {
    const ChunkView v = open_chunk(sgroups, a.ngroups, chunk, lane);
    const long long ca = (v.cnt + 1) >> 1;  // walker A: [first, first+ca)
    const long long cb = v.cnt - ca;        // walker B: [first+ca, first+cnt)
    const long long maxca = __shfl_sync(FULL, ca, 0);
    const uint32_t* R = srows + v.gr.gamma * k * WP;
    const uint32_t* PX = spx + v.gr.gamma * (k + 1) * px_stride(W);
    const int e0 = v.gr.ell + 1;

    Walker<W> A, B;
    if (v.cnt > 0) A.init(v.first, q, v.gr.ell, R, a.binom, sbinom);
    if (cb > 0) B.init(v.first + ca, q, v.gr.ell, R, a.binom, sbinom);
    // walker row additions: an init folds R[ell] and q more rows (q
    // additions), a step adds 2 or 3 prefix-XOR rows
    const int ninit = (v.cnt > 0) + (cb > 0);
    unsigned long long wadd = (unsigned long long)ninit * (unsigned long long)max(q, 0);

    int best = INT_MAX;
    for (long long p = 0; p < maxca; ++p) {
      if (p < ca) {
        if (p >= cb) {
#pragma unroll
          for (int j = 0; j < W; ++j) B.acc[j] = A.acc[j];
        }
        int pa = INT_MAX, pb = INT_MAX;
        suffix_pair<W, D>(A.acc, B.acc, R, e0, k, v.s0, v.gr.sl, [&](int wa, int wb) {
          pa = min(pa, wa);
          pb = min(pb, wb);
        });
        best = min(best, min(pa, pb));
        if (p + 1 < ca) wadd += (unsigned long long)A.step(PX);
        if (p + 1 < cb) wadd += (unsigned long long)B.step(PX);
      }
    }

    // chunk epilogue: warp min -> per-Gamma and round minima (fire-and-
    // forget reductions); combos count
    int wbest = __reduce_min_sync(FULL, best);
    if (wbest != INT_MAX) wbest += gamma_woff(a, v.gr.gamma);
    unsigned long long lw, lp;  // this lane's codewords / partial sums per prefix
    lane_suffixes<D>(k, e0, v.s0, v.gr.sl, lw, lp);
    const unsigned tot = __reduce_add_sync(FULL, (unsigned)((unsigned long long)v.cnt * lw));
    const bool tallied = v.gr.gamma < kTallyM;
    if (lane == 0) {
      if (wbest != INT_MAX && (!tallied || wbest < tally->best[v.gr.gamma])) {
        if (tallied) atomicMin(tally->best + v.gr.gamma, wbest);
        atomicMin(a.bound + 1 + v.gr.gamma, wbest);
        atomicMin(a.bound, wbest);
        gbound_publish(a, wbest);
      }
      if (tallied) atomicAdd(tally->combos + v.gr.gamma, (unsigned long long)tot);
      else atomicAdd(a.combos + v.gr.gamma, (unsigned long long)tot);
    }
    if (a.adds) {
      // every codeword is one row addition (prefix sum ^ its last suffix
      // row); D = 2 adds the partial sum prefix ^ R[e1] once per e1.  A
      // suffix row is loaded once per walker-pair step for the whole warp
      // (sl > 1: each by the suffix lanes owning it); the walkers read one
      // table row per addition plus R[ell] per init -- counted once per
      // prefix block (its other suffix lanes repeat the same prefix sums)
      const unsigned long long per_prefix =
          suffix_count<D>(k, e0) + (D == 2 ? (unsigned long long)max(0, k - 1 - e0) : 0ull);
      if (v.s0 != 0) wadd = 0ull;
      const unsigned long long adds = warp_sum_u64(wadd + (unsigned long long)v.cnt * (lw + lp));
      const unsigned long long accs = warp_sum_u64(wadd + (v.s0 == 0 ? (unsigned long long)ninit : 0ull)) +
                                      (unsigned long long)maxca * per_prefix;
      if (lane == 0) {
        if (tallied) {
          atomicAdd(tally->adds + v.gr.gamma, adds);
          atomicAdd(tally->accs + v.gr.gamma, accs);
        } else {
          atomicAdd(a.adds + v.gr.gamma, adds);
          atomicAdd(a.accs + v.gr.gamma, accs);
        }
      }
    }
  }
}

// This shard's chunks: warp w first takes chunk w (no atomic), then, when
// the grid has fewer warps than chunks, draws the rest from an atomic
// cursor (uneven prefix walks balance themselves).  A small round's warps
// each run one chunk and never touch the cursor.
template <bool kMayStop = true, typename Body>
__device__ __forceinline__ void deal_chunks(const RoundArgs& a, Body&& body) {
  const unsigned long long nw = (unsigned long long)gridDim.x * (blockDim.x >> 5);
  const unsigned long long mine =
      a.nchunks > (unsigned long long)a.shard
          ? (a.nchunks - a.shard + a.nshards - 1) / a.nshards : 0ull;
  unsigned long long c = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  while (c < mine) {
    if (kMayStop && round_done(a)) break;
    body(c * (unsigned long long)a.nshards + a.shard);
    if (nw >= mine) break;
    unsigned long long nx = 0;
    if ((threadIdx.x & 31) == 0) nx = atomicAdd(a.counter, 1ull);
    c = nw + __shfl_sync(0xffffffffu, nx, 0);
  }
}

template <int W, int D>
__global__ void __launch_bounds__(256)
k1_round_min(const RoundArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ K1Tally tally;
  uint32_t *srows, *spx;
  Group* sgroups;
  k1_tally_init(&tally, 1);
  stage<W>(a, srows, spx, sgroups, smem);  // ends with __syncthreads
  const unsigned long long* sbinom = smem_binom<W>(smem, a);
  // batched round: start from the U the previous round ended with (one
  // thread of the grid: atomics on one address serialise; blocks that read
  // the bound before it lands just see the looser start value)
  round_start(a);
  deal_chunks(a, [&](unsigned long long chunk) {
    k1_chunk<W, D>(a, chunk, srows, spx, sgroups, sbinom, &tally);
  });
  __syncthreads();
  k1_tally_flush(a, tally);
}

// Several small rounds (same family, same suffix depth) in one launch: the
// rows, prefix table and binomials are staged once, every round's work plan
// side by side, and the rounds' chunks form one space dealt round-robin by
// global warp index (about one chunk per warp: a returning atomic cursor per
// warp and round was this kernel's main stall), so the rounds run
// concurrently.  (No device-side U chain between them: bz_rounds clips each
// round's minima to its predecessor's U on the host, which gives the same
// results.)
constexpr int kK1MaxFused = 4;
constexpr int kK1FusedGroupBytes = 64 * 1024;  // shared-memory budget for the plans
struct K1Batch {
  RoundArgs a[kK1MaxFused];
  int count;
};

template <int W, int D>
__global__ void __launch_bounds__(256) k1_rounds(const K1Batch b) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ K1Tally tally[kK1MaxFused];
  uint32_t *srows, *spx;
  Group* sgroups;
  k1_tally_init(tally, b.count);
  stage<W>(b.a[0], srows, spx, sgroups, smem);  // round 0's plan at sgroups
  const unsigned long long* sbinom = smem_binom<W>(smem, b.a[0]);
  int goff[kK1MaxFused];
  unsigned long long cend[kK1MaxFused];  // this shard's chunks of rounds <= r
  unsigned long long total = 0;
  int go = 0;
#pragma unroll
  for (int r = 0; r < kK1MaxFused; ++r) {
    if (r < b.count) {
      const RoundArgs& a = b.a[r];
      goff[r] = go;
      if (r > 0) stage_groups(a, sgroups + go);
      go += a.ngroups;
      const unsigned long long mine =
          a.nchunks > (unsigned long long)a.shard
              ? (a.nchunks - a.shard + a.nshards - 1) / a.nshards : 0ull;
      total += mine;
      cend[r] = total;
      if (a.gbound) round_start(a);
    }
  }
  __syncthreads();
  // the next round kernel (a programmatic dependent) may take SMs as these
  // blocks retire
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const unsigned long long nwarps = (unsigned long long)gridDim.x * (blockDim.x >> 5);
  for (unsigned long long c = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
       c < total; c += nwarps) {
    int r = 0;
#pragma unroll
    for (int i = 0; i + 1 < kK1MaxFused; ++i)
      if (i + 1 < b.count && c >= cend[i]) r = i + 1;
    const RoundArgs& a = b.a[r];
    const unsigned long long local = c - (r > 0 ? cend[r - 1] : 0ull);
    if (round_done(a)) continue;
    k1_chunk<W, D>(a, local * a.nshards + a.shard, srows, spx, sgroups + goff[r], sbinom,
                   tally + r);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kK1MaxFused; ++r)
    if (r < b.count) k1_tally_flush(b.a[r], tally[r]);
}

// ---------------------------------------------------------------------------
// Bound seed for the threshold kernels (K5q / K5w).  Their producers write
// each prefix row against the Gamma's bound as it stands, and every
// codeword under that threshold takes the exact path in the epilogue; a pass
// that starts with no bound at all (bz_enumerate, config 4) would send its
// first prefix steps on every SM down that path.  Before such a pass, every
// thread weighs a few pseudo-random g-combinations of the pass (colex
// unrank of a hashed rank) and lowers the bounds with their weights -- true
// codeword weights of this pass, so the result stays min(start, true
// minimum) exactly; only the thresholds get tight from the first tile on.
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

constexpr int kSeedMaxG = 16;  // deeper rounds always start from a bound

template <int W>
__global__ void __launch_bounds__(128) k_seed_bound(const RoundArgs a, int gamma_only, int samples) {
  constexpr int WP = padded_words(W);
  // C(c, q) for c <= k, q <= g and the Gamma's rows in shared memory: the
  // unrank's binary searches would otherwise wait on L2 at every step
  __shared__ unsigned long long sb[kBinomDim * (kSeedMaxG + 1)];
  __shared__ __align__(16) uint32_t sr[kMaxK * kMaxW];
  const int k = a.k, g = a.g;
  for (int i = threadIdx.x; i < (k + 1) * (g + 1); i += blockDim.x)
    sb[i] = a.binom[(i / (g + 1)) * kBinomDim + i % (g + 1)];
  const int j0 = gamma_only < 0 ? 0 : gamma_only, j1 = gamma_only < 0 ? a.m : gamma_only + 1;
  const unsigned long long total = a.binom[k * kBinomDim + g];
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (int j = j0; j < j1; ++j) {
    __syncthreads();
    for (int i = threadIdx.x; i < k * WP; i += blockDim.x) sr[i] = a.rows[(size_t)j * k * WP + i];
    __syncthreads();
    int best = INT_MAX;
    for (int i = 0; i < samples; ++i) {
      unsigned long long r = mix64(tid * 0x100000001B3ull + (unsigned long long)i * 7919 + j) % total;
      uint32_t acc[W];
#pragma unroll
      for (int w = 0; w < W; ++w) acc[w] = 0u;
      int hi = k - 1;
      for (int q = g; q >= 1; --q) {
        // colex unrank: the largest c <= hi with C(c, q) <= r (C(q-1, q) = 0)
        int lo = q - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (sb[mid * (g + 1) + q] <= r) lo = mid; else hi = mid - 1;
        }
        r -= sb[lo * (g + 1) + q];
        xor_row<W>(acc, sr + lo * WP);
        hi = lo - 1;
      }
      int wt = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) wt += __popc(acc[w]);
      best = min(best, wt);
    }
    best = __reduce_min_sync(0xffffffffu, best);
    if ((threadIdx.x & 31) == 0) {
      const int wg = best + gamma_woff(a, j);
      atomicMin(a.bound + 1 + j, wg);
      if (gamma_only < 0) atomicMin(a.bound, wg);
    }
  }
}

// ---------------------------------------------------------------------------
// K1h: weight histogram of one (Gamma, g) pass.  Each thread owns a private
// 16-bit counter per bin of a WINDOW of kK1hWindow weights in shared memory,
// flushed into a block-wide u32 histogram (all bins) before it can overflow,
// and finally into the global u64 bins; a weight outside the window goes to
// the block histogram directly.  The window is centred on the weight a sum of
// g rows of this density would have if the rows were random
// (n/2 (1 - (1 - 2p)^g), p from the staged rows), computed alike by every
// block; it only steers which path a codeword takes -- any placement gives
// the same bins -- and on the codes of BASELINE's configs a codeword leaves
// it about once in 1e7.  64 instead of n + 1 private bins per thread is what
// lets 4 blocks (32 warps) share an SM instead of 2.
// Layout [bin][slot]: warps 2j and 2j + 1 own the low and high halves of the
// same 32 words, so a warp's 32 lanes touch 32 distinct banks for any bin
// pattern (adjacent threads sharing a word made every access a 2-way
// conflict); a count is a 16-bit load / add / store (one shared-memory atomic
// on the word, +1 or +65536, measured slower: 158 against 128 us on config 4:
// shared atomics issue at a fraction of the load / store rate).  The round's
// minimum is the lowest
// occupied bin, read off the block histogram at the end instead of a min per
// codeword.  Same two-walker structure as K1; on an odd range the second
// walker's last step is masked.
constexpr int kK1hWindow = 64;
constexpr int kK1hMinThreads = 64;  // two warps share a word
// bins of a block's shared histogram: stored weights 0 .. min(n, 32 W)
template <int W> __host__ __device__ constexpr int k1h_bins(int n) {
  return (n < 32 * W ? n : 32 * W) + 1;
}
__host__ __device__ constexpr int k1h_window(int nbins) {
  return nbins < kK1hWindow ? nbins : kK1hWindow;
}
template <int W, int D>
__global__ void __launch_bounds__(256)
k1h_histogram(const RoundArgs a) {
  constexpr int WP = padded_words(W);
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned int s_pop;
  uint32_t *srows, *spx;
  Group* sgroups;
  const int nbins = k1h_bins<W>(a.n);
  const int win = k1h_window(nbins);
  const int tid = threadIdx.x;
  const int bd = blockDim.x;
  size_t base = smem_base_bytes<W>(a.m, a.k, staged_groups(a));
  base = (base + 15) & ~size_t(15);
  unsigned int* bhist = reinterpret_cast<unsigned int*>(smem + base);
  unsigned int* th32 = bhist + ((nbins + 3) & ~3);
  unsigned short* th = reinterpret_cast<unsigned short*>(th32);
  if (tid == 0) s_pop = 0u;
  for (int i = tid; i < nbins; i += bd) bhist[i] = 0u;
  for (int i = tid; i < (win + 1) * (bd >> 1); i += bd) th32[i] = 0u;  // + the trash row
  stage<W>(a, srows, spx, sgroups, smem);  // ends with __syncthreads
  const unsigned long long* sbinom = smem_binom<W>(smem, a);

  const unsigned FULL = 0xffffffffu;
  const int lane = tid & 31;
  const int k = a.k, q = a.g - 1 - D;
  unsigned int since_flush = 0;
  // this thread's half-word of a bin row (see the layout above)
  const int wrp = tid >> 5;
  unsigned short* const mine = th + 64 * (wrp >> 1) + 2 * lane + (wrp & 1);
  // window start: the expected weight of a sum of g of this Gamma's rows
  int lo = 0;
  if (nbins > win) {
    const int gam = a.ngroups > 0 ? sgroups[0].gamma : 0;
    const uint32_t* R0 = srows + gam * k * WP;
    unsigned int pc = 0;
    for (int i = tid; i < k * WP; i += bd) pc += __popc(R0[i]);
    pc = __reduce_add_sync(FULL, pc);
    if (lane == 0 && pc) atomicAdd(&s_pop, pc);
    __syncthreads();
    const int ncols = max(1, min(a.n - (((a.elide >> gam) & 1ull) ? k : 0), 32 * W));
    const float dens = fminf(1.0f, (float)s_pop / ((float)k * (float)ncols));
    const float c = 0.5f * (float)ncols * (1.0f - powf(1.0f - 2.0f * dens, (float)a.g));
    lo = max(0, min(nbins - win, (int)(c + 0.5f) - win / 2));
  }

  auto flush = [&]() {
    for (int b = 0; b < win; ++b) {
      const unsigned int v = mine[b * bd];
      if (v) {
        atomicAdd(bhist + lo + b, v);
        mine[b * bd] = 0;
      }
    }
    since_flush = 0;
  };
  // The hot loop is branch-free: a weight outside the window (and the
  // masked second walker) counts into a trash row, oow keeps the step's
  // largest window offset, and a step that saw one outside is walked again
  // for just those codewords (rare).
  const unsigned int uwin = (unsigned int)win;
  auto count2 = [&](int wa, int wb, unsigned int notb, unsigned int& oow) {
    const unsigned int da = (unsigned int)(wa - lo), db = (unsigned int)(wb - lo);
    oow = max(oow, max(da, db));
    unsigned short* ha = mine + min(da, uwin) * (unsigned int)bd;
    *ha = (unsigned short)(*ha + 1);
    unsigned short* hb = mine + min(db | notb, uwin) * (unsigned int)bd;
    *hb = (unsigned short)(*hb + 1);
  };

  unsigned long long wcombos = 0;  // this warp's combinations (one atomic at the end)
  deal_chunks<false>(a, [&](unsigned long long chunk) {  // every combination
    const ChunkView v = open_chunk(sgroups, a.ngroups, chunk, lane);
    const long long ca = (v.cnt + 1) >> 1;
    const long long cb = v.cnt - ca;
    const long long maxca = __shfl_sync(FULL, ca, 0);
    const uint32_t* R = srows + v.gr.gamma * k * WP;
    const uint32_t* PX = spx + v.gr.gamma * (k + 1) * px_stride(W);
    const int e0 = v.gr.ell + 1;
    unsigned long long lw, lp;  // this lane's codewords per prefix
    lane_suffixes<D>(k, e0, v.s0, v.gr.sl, lw, lp);
    const unsigned chunk_work = (unsigned)((unsigned long long)v.cnt * lw);
    if (since_flush + chunk_work > 65535u) flush();
    since_flush += chunk_work;

    Walker<W> A, B;
    if (v.cnt > 0) A.init(v.first, q, v.gr.ell, R, a.binom, sbinom);
    if (cb > 0) B.init(v.first + ca, q, v.gr.ell, R, a.binom, sbinom);
    for (long long p = 0; p < maxca; ++p) {
      if (p < ca) {
        const bool with_b = p < cb;
        const unsigned int notb = with_b ? 0u : 0xFFFFFFFFu;
        unsigned int oow = 0u;
        suffix_pair<W, D>(A.acc, B.acc, R, e0, k, v.s0, v.gr.sl,
                          [&](int wa, int wb) { count2(wa, wb, notb, oow); });
        if (oow >= uwin)
          suffix_pair<W, D>(A.acc, B.acc, R, e0, k, v.s0, v.gr.sl, [&](int wa, int wb) {
            if ((unsigned int)(wa - lo) >= uwin) atomicAdd(bhist + wa, 1u);
            if (with_b && (unsigned int)(wb - lo) >= uwin) atomicAdd(bhist + wb, 1u);
          });
        if (p + 1 < ca) A.step(PX);
        if (p + 1 < cb) B.step(PX);
      }
    }
    wcombos += __reduce_add_sync(FULL, chunk_work);
  });
  flush();
  // the pass is one Gamma
  if (lane == 0 && wcombos && a.ngroups > 0) atomicAdd(a.combos + sgroups[0].gamma, wcombos);
  // the pass is one Gamma (all groups share it): shift by its dropped
  // identity weight
  const int off = a.ngroups > 0 ? gamma_woff(a, sgroups[0].gamma) : 0;
  __syncthreads();
  int best = INT_MAX;  // the lowest occupied bin
  for (int b = tid; b < nbins && b + off <= a.n; b += bd)
    if (bhist[b]) {
      atomicAdd(a.hist + b + off, (unsigned long long)bhist[b]);
      best = min(best, b);
    }
  const int wbest = __reduce_min_sync(FULL, best);
  if (lane == 0 && wbest < INT_MAX) atomicMin(a.bound, wbest + off);
}

// ---------------------------------------------------------------------------
// Integer-pipe microbenchmarks (roofline denominators).
__global__ void peak_popc(uint32_t* out, uint32_t seed, int iters, long long* clk) {
  uint32_t y0 = seed ^ threadIdx.x, y1 = y0 * 3u, y2 = y0 * 5u, y3 = y0 * 7u;
  uint32_t y4 = y0 * 11u, y5 = y0 * 13u, y6 = y0 * 17u, y7 = y0 * 19u;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      asm volatile("popc.b32 %0, %0;" : "+r"(y0));
      asm volatile("popc.b32 %0, %0;" : "+r"(y1));
      asm volatile("popc.b32 %0, %0;" : "+r"(y2));
      asm volatile("popc.b32 %0, %0;" : "+r"(y3));
      asm volatile("popc.b32 %0, %0;" : "+r"(y4));
      asm volatile("popc.b32 %0, %0;" : "+r"(y5));
      asm volatile("popc.b32 %0, %0;" : "+r"(y6));
      asm volatile("popc.b32 %0, %0;" : "+r"(y7));
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = y0 + y1 + y2 + y3 + y4 + y5 + y6 + y7;
}

__global__ void peak_lop3(uint32_t* out, uint32_t seed, int iters, long long* clk) {
  uint32_t y0 = seed ^ threadIdx.x, y1 = y0 * 3u, y2 = y0 * 5u, y3 = y0 * 7u;
  uint32_t y4 = y0 * 11u, y5 = y0 * 13u, y6 = y0 * 17u, y7 = y0 * 19u;
  const uint32_t a = seed * 0x9e3779b9u, b = seed * 0x85ebca6bu;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y0) : "r"(a), "r"(b));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y1) : "r"(a), "r"(b));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y2) : "r"(a), "r"(b));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y3) : "r"(a), "r"(b));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y4) : "r"(a), "r"(b));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y5) : "r"(a), "r"(b));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y6) : "r"(a), "r"(b));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y7) : "r"(a), "r"(b));
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = y0 + y1 + y2 + y3 + y4 + y5 + y6 + y7;
}

// Legacy warp-level IMMA (mma.sync m16n8k32 s8) throughput: 4 independent
// accumulator chains per warp -- the denominator of K3's tensor roofline.
__global__ void peak_imma(int* out, uint32_t seed, int iters, long long* clk) {
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
  uint32_t b0 = a0 * 11u, b1 = a0 * 13u;
  int c[4][4] = {};
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int ch = 0; ch < 4; ++ch)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[ch][0]), "+r"(c[ch][1]), "+r"(c[ch][2]), "+r"(c[ch][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  int s = 0;
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) s += c[ch][0] + c[ch][1] + c[ch][2] + c[ch][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Synthetic codeword loop: register-resident rows, W words, 4 codewords per
// iteration -- the best the XOR+POPC+min recipe can do on this chip.
template <int W>
__global__ void peak_codeword(int* out, uint32_t seed, int iters, long long* clk) {
  uint32_t acc[W], r0[W], r1[W], r2[W], r3[W];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    acc[j] = seed * (j + 1) ^ threadIdx.x;
    r0[j] = acc[j] * 3u; r1[j] = acc[j] * 5u; r2[j] = acc[j] * 7u; r3[j] = acc[j] * 9u;
  }
  int best = INT_MAX;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int w0 = weight_xor<W>(acc, r0);
    const int w1 = weight_xor<W>(acc, r1);
    const int w2 = weight_xor<W>(acc, r2);
    const int w3 = weight_xor<W>(acc, r3);
    best = min(best, min(min(w0, w1), min(w2, w3)));
#pragma unroll
    for (int j = 0; j < W; ++j) acc[j] += 0x9e3779b9u;  // keep iterations distinct
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = best;
}

}  // namespace bz
