/*
 * bz.h -- C ABI of the B200 Brouwer-Zimmermann enumeration core.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `mindist` (arXiv 1603.06757): for one generator count g it visits every
 * g-row combination of every systematic information-set matrix Gamma_j,
 * XORs the bit-packed rows, popcounts the codeword and min-reduces it.
 *
 * Reference interfaces replaced (paths relative to the reference's
 * pkg/src/mindist/):
 *   bz_round      <- engine.py:208-211  the per-round loop
 *                      `for idx, gamma in enumerate(gs.gammas):
 *                           res = runner.run(idx, gamma, g, U)`
 *                    i.e. _Runner.run (engine.py:136-150) dispatching to
 *                    enumerate_basic/optimized/stack (enumeration.py:76,96,128)
 *                    or enumerate_saved/_unrolled/_parallel
 *                    (enumeration.py:305,351,385), each returning an
 *                    EnumerationResult (enumeration.py:43-50) whose
 *                    min_weight is clipped to ubound (enumeration.py:60-64).
 *   bz_enumerate  <- one (Gamma, g) pass: enumerate_*(gamma, g, ubound)
 *                    (enumeration.py:76-93) -> (min_weight, combinations).
 *   bz_histogram  <- no reference counterpart (the reference keeps only the
 *                    minimum); weight histogram of one (Gamma, g) pass, used
 *                    as the bit-exact checksum of BASELINE.json config 4.
 *   bz_load_gammas<- the packed row layout of BitMatrix.to_numpy()
 *                    (gf2.py:74-79, word_width 64): little-endian words,
 *                    bit j of the row = column j, zero padding past n-1.
 *
 * Conventions: plain C types only; every pointer is caller-owned host
 * memory and is not retained past the call.  Calls on one context are not
 * thread-safe (serialise them; the reference driver is single-threaded,
 * SPEC.md:394).  Status codes map onto the reference's MindistError
 * hierarchy (errors.py:6-71) in the Python wrapper.  There is no CPU
 * fallback: without a usable sm_100 device bz_create fails with
 * BZ_ERR_NO_DEVICE.
 */
#ifndef BZ_H_
#define BZ_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BZ_ABI_VERSION 16

/* limits of the device kernels */
#define BZ_MAX_K 128 /* rows per Gamma (prefix masks are 128-bit)      */
#define BZ_MAX_N 384 /* columns of the uploaded rows (k + 256 at most)   */
#define BZ_MAX_N_STORED 256 /* columns a Gamma keeps on the device after
                               identity-column elision: 8 x 32-bit words  */

/* status codes */
#define BZ_OK 0
#define BZ_ERR_INVALID_ARITY 1      /* g outside 1..k        -> InvalidArity      */
#define BZ_ERR_INVALID_DIMENSIONS 2 /* bad m/k/n/padding     -> InvalidDimensions */
#define BZ_ERR_TOO_LARGE 3          /* k>128, n>384, >256 stored columns, C(k,g) >= 2^62 -> TooLarge  */
#define BZ_ERR_CUDA 4               /* CUDA runtime failure                      */
#define BZ_ERR_NO_DEVICE 5          /* no sm_100 device visible                  */
#define BZ_ERR_STATE 6              /* no Gamma loaded / bad gamma index         */
#define BZ_ERR_ARGUMENT 7           /* null pointer, bad shard                   */

/* enumeration engines (bz_set_engine) */
#define BZ_ENGINE_AUTO 0 /* K5q (stored weights <= 128) or K5 for g >= 4   */
#define BZ_ENGINE_POPC 1 /* K1 only: XOR + POPC on the integer pipes       */
/* 2, 3, 5, 6: round-1 comparison kernels, built only with
 * -DBZ_LEGACY_KERNELS=1 (bz_set_engine fails with BZ_ERR_ARGUMENT otherwise) */
#define BZ_ENGINE_IMMA 2 /* K3 (legacy warp-level IMMA) for g >= 4        */
#define BZ_ENGINE_UMMA 3 /* K4 (tcgen05.mma kind::i8, TMEM) for g >= 4     */
#define BZ_ENGINE_MXF4 4 /* K5 (tcgen05.mma kind::mxf4, unit scales) g >= 4 */
#define BZ_ENGINE_MXF4P 5 /* K5p: K5 with two codewords per accumulator     \
                             column (stored words W = 1 or 3; else K5)     */
#define BZ_ENGINE_MXF4T 6 /* K5t: three codewords per column (W = 1, 3)     */
#define BZ_ENGINE_MXF4Q 7 /* K5q: two codewords as bytes (mxf4nvf4; W <= 4,
                             stored columns <= 128; else K5)              */
#define BZ_ENGINE_MXF4W 8 /* K5w: two codewords as 11-bit fields (mxf4,
                             ue8m0 scales; any W >= 2, rows wider than
                             K5q's 128 stored columns; W = 1 runs K5).
                             On request: measured no faster than K5 on the
                             section-6 codes      */
#define BZ_ENGINE_MXF4F 9 /* K5f: K5q's byte fields from folded MMAs (odd
                             W <= 3 whose last stored word holds <= 16
                             columns, e.g. config 5's 80: 3 MMAs per tile
                             instead of 4); else as BZ_ENGINE_MXF4Q.  On
                             request: measured no faster than K5q (1.97
                             against 1.92 ms on config 5's g = 8 round)  */

typedef struct bz_ctx bz_ctx;

/* Library / ABI version (BZ_ABI_VERSION). */
int bz_abi_version(void);

/* Number of visible CUDA devices (0 when none); never fails. */
int bz_device_count(void);

/* Create a context on CUDA device `device` (one process per GPU). */
int bz_create(int device, bz_ctx **out);

/* Destroy a context and free its device memory; NULL is ignored. */
void bz_destroy(bz_ctx *ctx);

/* Human-readable description of the last error on ctx (never NULL). */
const char *bz_last_error(const bz_ctx *ctx);

/* GPU brute force (brute_force_distance, m/engine.py:223-237): the minimum
 * weight over all 2^k - 1 nonzero messages of the k x n generator `rows`
 * (ceil(n/64) u64 words per row, bit j = column j), Gray-code order, one
 * row XOR per codeword.  k <= min(max_k, 48) else BZ_ERR_TOO_LARGE.
 * Zero-weight codewords (rank-deficient G) give 0, as in the reference;
 * *out_codewords = 2^k - 1. */
int bz_brute_force(bz_ctx *ctx, const uint64_t *rows, int k, int n, int max_k,
                   int32_t *out_distance, uint64_t *out_codewords);

/* Host-only Gauss-Jordan (reduce_on_columns, m/gf2.py:133-161): reduce the
 * k x n matrix `rows` (row-major, ceil(n/64) u64 words per row, bit j =
 * column j) in place, taking pivots from `cols` in the given order (leftmost
 * available row, swapped to the top, eliminated from every other row).
 * Writes the pivot columns to out_pivots (capacity k, may be NULL) and the
 * rank to *out_rank.  Needs no device. */
int bz_reduce_on_columns(uint64_t *rows, int k, int n, const int32_t *cols, int ncols,
                         int32_t *out_pivots, int *out_rank);

/* Host only: the information-set family of build_gamma_set
 * (m/gf2.py:168-199) in one call.  Greedy Gauss-Jordan on the still-unused
 * columns (leftmost first), each pass continuing from the previous reduced
 * matrix; full-rank passes append Gamma_j, the first deficient pass with
 * rank > 0 is the remainder.  rows: k x ceil(n/64) words of G.  out_rows:
 * m_max x k x ceil(n/64), out_pivots: m_max x k, out_ranks: m_max.  *out_m =
 * 0 with out_ranks[0] = rank means G itself is rank deficient. */
int bz_gamma_family(const uint64_t *rows, int k, int n, int m_max, uint64_t *out_rows,
                    int32_t *out_pivots, int32_t *out_ranks, int *out_m);

/* Multi-GPU shared bound (one process per GPU).  Rank 0 allocates the
 * mirror and exports a 64-byte CUDA IPC handle (bz_shared_bound_export),
 * every rank opens it (rank 0 with handle = NULL, i.e. its own array), and
 * before each minimum-distance run every rank sets the same epoch.  Round
 * kernels then RED.MIN their chunk minima into the mirror over NVLink and
 * stop taking work as soon as any rank's running minimum meets L_prev, so
 * a batch of rounds can run ahead of termination on every rank.  Results
 * are still each rank's own shard (combine them as before). */
int bz_shared_bound_export(bz_ctx *ctx, void *out_handle /* 64 bytes */);
int bz_shared_bound_open(bz_ctx *ctx, const void *handle /* NULL: own */);
int bz_shared_bound_epoch(bz_ctx *ctx, uint32_t epoch);
/* The shared running minimum of round g in the current epoch (INT32_MAX if
 * none yet), read through this rank's mapping (diagnostics, tests). */
int bz_shared_bound_read(bz_ctx *ctx, int g, int32_t *out);
int bz_shared_bound_close(bz_ctx *ctx);

/* Identity-column elision (default on; applies from the next
 * bz_load_gammas): a Gamma with one unit column per row is stored without
 * those k columns and its weights get + g, which is exact because each
 * chosen row carries exactly one of them.  That covers every Gamma from
 * build_gamma_set (m/gf2.py:133-199), the rank-deficient remainder too: it
 * spans the row space of G and keeps the earlier passes' pivots as unit
 * columns.  The test is made per Gamma at load time (bz_elided reports it).
 * Results are identical either way. */
int bz_set_elision(bz_ctx *ctx, int on);

/* In-round early exit (default off): a round stops taking work once its
 * running minimum meets lower_prev.  Results and the bounds trace are the
 * same either way; only the `combinations` counts of such rounds drop below
 * the reference's m*C(k,g).  Batched rounds past termination (the previous
 * round's U already <= lower_prev) stop at once in both modes; the caller
 * discards them. */
int bz_set_early_exit(bz_ctx *ctx, int on);

/* Bit j set: Gamma j of the loaded family was stored with its identity
 * columns dropped. */
int bz_elided(bz_ctx *ctx, uint64_t *out_mask);

/* Select the enumeration engine for later calls (BZ_ENGINE_*).  Results
 * are identical; only the kernel and the work plan differ. */
int bz_set_engine(bz_ctx *ctx, int engine);

/* Upload the m systematic matrices of one generator: `rows` holds
 * m*k*ceil(n/64) little-endian uint64 words, matrix-major then row-major
 * (bit j of a row = column j; bits past n-1 must be zero).  Replaces any
 * previously loaded family. */
int bz_load_gammas(bz_ctx *ctx, const uint64_t *rows, int m, int k, int n);

/* One Brouwer-Zimmermann round: enumerate every g-combination of every
 * loaded Gamma_j and report, per Gamma, min(true minimum weight, upper)
 * in out_min[j] and the number of combinations visited in out_combos[j].
 *
 * lower_prev is the certified lower bound before this round.  With the
 * in-round early exit on (bz_set_early_exit) the kernel stops once the
 * running minimum reaches lower_prev (the round's result is then exactly
 * lower_prev, as in the reference trace, but fewer combinations are
 * visited); off (the default) every combination is visited, as the
 * reference does.
 *
 * shard/nshards split the round's work into nshards disjoint parts (one
 * per GPU/process); nshards = 1 is the whole round.  Results of the shards
 * combine by min (out_min) and sum (out_combos). */
int bz_round(bz_ctx *ctx, int g, int lower_prev, int upper, int shard,
             int nshards, int32_t *out_min, uint64_t *out_combos);

/* Rounds g0 .. g0+count-1 in one call: planned together, launched back to
 * back, one synchronisation -- for the short early rounds, where launch and
 * synchronisation latency dominate.  lower_prev[i] is round g0+i's early
 * exit threshold.  Round g0 starts from `upper`, each later round from the
 * U its predecessor ended with (min of `upper` and that round's minima) --
 * the running U the reference clips with (m/engine.py:209-211); the caller
 * folds the rounds into its bounds in order and discards rounds past
 * termination (those exit at once: their start U is already <= lower_prev).
 * out_min / out_combos hold count x m values, round-major. */
int bz_rounds(bz_ctx *ctx, int g0, int count, const int32_t *lower_prev, int upper,
              int shard, int nshards, int32_t *out_min, uint64_t *out_combos);

/* The Algorithm-1 loop itself (m/engine.py:204-217, one rank), one device
 * call per bz_advance: from st = (g, L, U) it takes the next rounds whose
 * m*C(k, g') total fits batch_budget (at least one; batch_budget <= 0: one
 * round per call), not past min(k, max_g) and not past the first round g'
 * with L(g'-1) >= min(U, u_rows) (u_rows: the weight of the lightest row of
 * any Gamma, an upper bound on U once round 1 is in), runs them as
 * bz_rounds does, and folds them in order: U = min(U, every Gamma's
 * minimum), L = (m_arg-1)(g'+1) + max(0, g'+1-k+km_arg)
 * (lower_bound_update, engine.py:97-103), one record (g', L, U, counters
 * summed over the Gammas, device ms) per round -- rounds past termination
 * are discarded.  st->status: BZ_LOOP_RUNNING while the loop goes on,
 * BZ_LOOP_DONE once L >= U or g > k (exact), BZ_LOOP_MAX_G when it would
 * continue past max_g (upper bound only).  Writes at most `cap` records. */
#define BZ_LOOP_RUNNING 0
#define BZ_LOOP_DONE 1
#define BZ_LOOP_MAX_G 2
typedef struct {
  int32_t g, L, U;   /* in/out: the next round and the bounds before it */
  int32_t g_reached; /* out: last round folded in                       */
  int32_t status;    /* in/out: BZ_LOOP_*                                */
} bz_loop_state;
typedef struct {
  int32_t g, L, U;   /* the trace entry (g, L, U) after round g          */
  int32_t pad;
  uint64_t combinations, row_additions, row_accesses;
  float kernel_ms;
  int32_t pad2;
} bz_round_record;
int bz_advance(bz_ctx *ctx, int m_arg, int km_arg, int max_g, int u_rows, int64_t batch_budget,
               bz_loop_state *st, bz_round_record *out, int cap, int *n_out);

/* One (Gamma_gamma, g) pass without early exit; out_min is the unclipped
 * minimum weight (INT32_MAX when the shard is empty). */
int bz_enumerate(bz_ctx *ctx, int gamma, int g, int shard, int nshards,
                 int32_t *out_min, uint64_t *out_combos);

/* Row-level operation counters of the last bz_round / bz_rounds /
 * bz_enumerate call (count <= its rounds; count x m values, round-major; for
 * bz_enumerate only the enumerated Gamma's entries are non-zero) -- the
 * device analogue of the reference's EnumerationResult.row_additions /
 * row_accesses (m/enumeration.py:19-24, :254-302):
 *   out_adds: full-row additions performed for the visited combinations --
 *     one per codeword (its prefix sum combined with its last stored row:
 *     a XOR in K1, the tensor-core dot product in K5/K5q), K1's D = 2
 *     partial sums (prefix ^ R[e1], once per e1), and the prefix walkers'
 *     updates (q rows per colex unrank, 2 or 3 prefix-XOR rows per step;
 *     once per K1 prefix block, not per suffix lane repeating them);
 *   out_accs: rows brought into the working set -- every stored suffix row
 *     a warp (K1) or CTA (K5/K5q: shared memory, up to 128 prefixes per
 *     load) loads per prefix step, plus the table rows the walkers read.
 * Suffix-table construction is not included (cf. store_build_additions).
 * bz_plan + the oracle's chunk walk reproduce both exactly. */
int bz_counters(bz_ctx *ctx, int count, uint64_t *out_adds, uint64_t *out_accs);

/* Weight histogram of one (Gamma_gamma, g) pass: out_hist[w] (n+1 bins)
 * counts the g-combinations whose codeword has weight w. */
int bz_histogram(bz_ctx *ctx, int gamma, int g, int shard, int nshards,
                 uint64_t *out_hist, int32_t *out_min, uint64_t *out_combos);

/* Host-only: the work plan bz_round uses for (m, k, g, nshards), for inspection and
 * for the CPU tests of the sharding logic.  Writes *out_ngroups groups of 12
 * int64 each -- chunk_begin, nprefix, gamma, ell, prefixes_per_lane,
 * combinations, depth, lanes_per_chunk, suffixes_per_chunk, suffix_blocks,
 * suffix_floor, suffix_lanes -- into out (capacity `cap` groups; out may be
 * NULL to query the count) and the round's chunk count into *out_nchunks.
 * Chunk c of the round belongs to shard c % nshards.  Within group (gamma,
 * ell, depth), local chunk index c_local = pb * suffix_blocks + sb: prefix
 * block l (0 <= l < lanes = lanes_per_chunk / suffix_lanes; lanes_per_chunk
 * is 32 for a warp of K1, 256 for a block of K3, 128 for K4 / K5, and
 * suffix_lanes > 1 only in K1, whose lanes l*suffix_lanes + s share block l
 * and take its first suffix rows suffix_floor + s, + 2 suffix_lanes, ...)
 * walks the colex ranks [(pb*lanes + l)*ppl, +ppl) of the
 * (g-1-depth)-subsets of [0, ell), each extended by ell and then by every
 * depth-subset of the suffix rows [suffix_floor, k) -- for depth >= 3 only
 * those with index in [sb*S, (sb+1)*S) of the table order (smallest element
 * descending, then the rest lex), S = suffixes_per_chunk.  suffix_floor is
 * ell + 1 except in K5's deeper levels (depth 4, 5), which take the
 * combinations whose top `depth` elements all lie in rows >= a level floor.
 * In those levels every prefix whose last element is below the floor has the
 * same suffix slice, and they are consecutive in colex order, so they form
 * ONE group, marked suffix_lanes = 0 (ABI 16): its ell is the last such
 * element, nprefix = C(ell + 1, g - depth), and a lane walks the colex ranks
 * of the (g-depth)-subsets of [0, ell + 1) with no fixed last row.
 * depth = 3..5 (K5) or 3 (K3, K4) for g >= 4 unless engine ==
 * BZ_ENGINE_POPC, else 2 for g >= 4, else 1 (g = 1: ell = -1, empty
 * prefix). */
int bz_plan(int m, int k, int g, int engine, int nshards, int64_t *out, int cap,
            int *out_ngroups, uint64_t *out_nchunks);

/* Device timing on the context's stream: bz_timer_start records a CUDA
 * event, bz_timer_stop records a second one, synchronises and returns the
 * elapsed milliseconds. */
int bz_timer_start(bz_ctx *ctx);
int bz_timer_stop(bz_ctx *ctx, float *ms);

/* Device time (ms) of the enumeration kernel of the last bz_round /
 * bz_enumerate / bz_histogram call, from CUDA events around that launch. */
int bz_last_kernel_ms(bz_ctx *ctx, float *ms);

/* Per-round device time (ms) of the last bz_round / bz_rounds call, count
 * <= rounds of that call.  The largest round of a batch is bracketed by CUDA
 * events; the other rounds (launched as programmatic dependents, so their
 * kernels overlap) share the rest of the batch time by combination count. */
int bz_round_ms(bz_ctx *ctx, float *out_ms, int count);

/* Number of kernels this context has launched so far. */
int bz_launch_count(bz_ctx *ctx, uint64_t *out);

/* Integer-pipe microbenchmark on the context's device (roofline
 * denominators): out[0] = POPC per second (whole GPU), out[1] = LOP3 per
 * second, out[2] = SM clock in MHz during the run, out[3] = SM count,
 * out[4] = POPC per clock per SM, out[5] = LOP3 per clock per SM,
 * out[6] = codewords/s of a synthetic W-word XOR+POPC+min loop (w_words
 * selects W, 1..8), out[7] = its codewords per clock per SM, out[8] = s8
 * IMMA (mma.sync m16n8k32) multiply-accumulates per second, out[9] = IMMA
 * MACs per clock per SM, out[10] = tcgen05.mma kind::i8 (M=128, N=256,
 * K=32, operands in shared memory, one CTA per SM) MACs per second,
 * out[11] = its MACs per clock per SM, out[12] = tcgen05.mma kind::mxf4
 * (M=128, N=240, K=64, unit block scales) MACs per second, out[13] = its
 * MACs per clock per SM.  `out` must hold 14 doubles. */
int bz_measure_int_peaks(bz_ctx *ctx, int w_words, double *out);

/* Host-only self-check of the K5q and K5w offset encodings (no device
 * needed): the producers' thresholds and e2m1 offset chunks over every
 * prefix weight (K5q 0..128, bound -4..128; K5w 0..256, bound -4..400) must
 * stay in range and dot to their integers exactly.  Returns the number of
 * failures (0 = ok); the first failing (prefix weight, bound) goes to
 * out_bad[0..1] (may be NULL; K5w bounds are reported + 1000). */
int bz_k5q_selftest(int32_t *out_bad);

#ifdef __cplusplus
}
#endif

#endif /* BZ_H_ */
