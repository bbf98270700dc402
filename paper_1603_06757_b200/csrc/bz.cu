// bz.cu -- context management, round planning and the C ABI (include/bz.h)
// for the B200 Brouwer-Zimmermann enumeration core.
//
// One context owns one CUDA device and one stream.  bz_load_gammas uploads
// the padded 32-bit row image of every Gamma_j plus its prefix-XOR table
// once per minimum-distance run; each bz_round then costs one small H2D of
// the round's group table, one kernel launch and one D2H of m+1 minima and
// m counters -- the host-side work that the reference does per round in
// engine.py:204-217 stays in Python above this library.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/bz.h"
#include "bz_kernels.cuh"
// Comparison kernels of the round-1 evolution (K3 legacy mma.sync IMMA, K4
// tcgen05 kind::i8, K5p / K5t packed variants) are not part of the product
// library; build with -DBZ_LEGACY_KERNELS=1 (tools/build_legacy.sh) to get
// them back for A/B measurements.
#ifndef BZ_LEGACY_KERNELS
#define BZ_LEGACY_KERNELS 0
#endif
#include "bz_tc.cuh"  // K3 is only instantiated with BZ_LEGACY_KERNELS
#include "bz_umma.cuh"
#include "bz_brute.cuh"

using bz::Group;
using bz::RoundArgs;

struct bz_ctx {
  int device = -1;
  int last_count = 0;  // rounds of the last run_batch (bz_counters)
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;      // user timer
  cudaEvent_t ev_k0 = nullptr, ev_k1 = nullptr;    // last kernel
  std::string err;
  uint64_t launches = 0;
  float last_kernel_ms = 0.f;
  std::vector<cudaEvent_t> ev_round;  // one per launch boundary of the last batch
  std::vector<float> round_ms;        // per-round device ms of the last batch
  bool pdl_next = false;              // the next round launch may overlap the previous one
  // multi-GPU shared bound mirror (bz_shared_bound_*): this rank's own array
  // (allocated on export), the array the kernels use (the owner's, mapped
  // over CUDA IPC, or this rank's own), and the run tag
  unsigned long long* d_gbound_own = nullptr;
  unsigned long long* d_gbound = nullptr;
  bool gbound_ipc = false;
  unsigned long long gtag = 0;

  // loaded family
  int m = 0, k = 0, n = 0, w32 = 0, wp = 0, n_eff = 0;
  std::vector<int> n_stored;         // columns each Gamma keeps on the device
  int engine = BZ_ENGINE_AUTO;
  int elision = 1;                   // bz_set_elision (applies at the next load)
  int early_exit = 0;                // bz_set_early_exit: in-round exit at lower_prev
  unsigned long long elide_mask = 0; // Gammas loaded with identity columns dropped
  uint32_t* d_rows = nullptr;   // m*k*wp
  uint8_t* d_trip = nullptr;    // K3 triple tables: m x trip_rows rows of 0/1 bytes
  size_t trip_rows = 0;         // rows per Gamma (C(k,3) + one tile of padding)
  uint8_t* d_trip4 = nullptr;   // K4 triple tables (UMMA core-matrix layout, s8)
  size_t trip4_rows = 0;        // rows per Gamma (C(k,3) rounded up to a tile, + a tile)
  // K5 suffix tables, level D = 3 + i (UMMA core-matrix layout, e2m1):
  // all D-subsets of rows >= lvl_floor[i] (-1: not built), lvl_rows[i] rows
  // per Gamma
  uint8_t* d_lvl[3] = {nullptr, nullptr, nullptr};
  size_t lvl_cap[3] = {0, 0, 0};
  size_t lvl_rows[3] = {0, 0, 0};
  int lvl_floor[3] = {-1, -1, -1};
  int lvl_form = 1;                  // row format the level tables were built in (ensure_level)
  // grow-only capacities (bytes) so repeated loads do not reallocate
  size_t rows_cap = 0, px_cap = 0, trip_cap = 0, trip4_cap = 0;
  // tables are built on first use
  bool trip_built = false, trip4_built = false;
  uint32_t* d_px = nullptr;     // m*(k+1)*wp
  unsigned long long* d_binom = nullptr;
  // per-round scratch
  // per-round I/O slots (io_layout): one H2D and one D2H per batch
  unsigned char* d_io = nullptr;
  unsigned char* h_io = nullptr;  // pinned mirror
  size_t io_cap = 0;
  unsigned char* h_stage = nullptr;  // pinned staging of the row images (bz_load_gammas)
  size_t stage_cap = 0;
  cudaEvent_t ev_load = nullptr;     // the last staging upload
  bool ev_load_pending = false;
  // suffix tables are built on a side stream, overlapping the small rounds'
  // K1 launch; the first tensor-core launch waits for them
  cudaStream_t side = nullptr;
  cudaEvent_t ev_main = nullptr, ev_side = nullptr;
  bool side_pending = false;
  // the plan keys and offsets of the last batch whose group tables are in
  // h_io and d_io: an identical round (same key, same offset) is neither
  // copied nor uploaded again
  std::vector<std::pair<std::string, size_t>> io_plans;
  unsigned long long* d_hist = nullptr;    // BZ_MAX_N + 1
  // pinned histogram staging
  unsigned long long* h_hist = nullptr;
};

namespace {

// Codewords per lane per chunk: aim for ~40k chunks per round (dynamic
// balance over 148 SMs x 32 warps), within [32, 4096].  Depends only on the
// problem size, so every process computes the same plan.
constexpr long long kChunksTarget = 40000;
constexpr long long kLaneMin = 32, kLaneMax = 4096;
constexpr int kPlanCols = 12;  // int64 columns per group in bz_plan

int fail(bz_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess)                                                    \
      return fail(ctx, BZ_ERR_CUDA, "%s failed: %s", #call,                   \
                  cudaGetErrorString(e_));                                    \
  } while (0)

// saturating binomial on the host
unsigned long long binom_sat(int p, int q) {
  if (q < 0 || p < 0 || q > p) return 0ull;
  q = std::min(q, p - q);
  unsigned __int128 r = 1;
  for (int i = 1; i <= q; ++i) {
    r = r * (unsigned)(p - q + i) / (unsigned)i;
    if (r > (unsigned __int128)~0ull) return ~0ull;
  }
  return (unsigned long long)r;
}

// grow-only device buffer
cudaError_t grow(bz_ctx*, void** p, size_t* cap, size_t bytes) {
  if (bytes <= *cap && *p) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc(p, std::max<size_t>(bytes, 256));
  if (e == cudaSuccess) *cap = std::max<size_t>(bytes, 256);
  return e;
}

// Per-round I/O slot: [counter u64][combos m x u64][bound (m+1) x int32]
// [pad][groups].  A batch of rounds uses consecutive slots; the whole block
// goes to the device in one copy and comes back in one copy.
struct IoSlot {
  size_t off_combos, off_adds, off_accs, off_bound, off_groups, size;
};

// I/O image of a batch of rounds: first every round's result record
// {cursor, combos[m], adds[m], accs[m], bound[m+1]} (off_groups bytes each, contiguous: the
// only part read back), then each round's plan at a variable offset
// (ctx->gbase[i]; only the used groups travel host -> device).
IoSlot io_layout(int m, int k) {
  IoSlot l;
  l.off_combos = 8;
  l.off_adds = l.off_combos + 8 * (size_t)m;
  l.off_accs = l.off_adds + 8 * (size_t)m;
  l.off_bound = l.off_accs + 8 * (size_t)m;
  l.off_groups = (l.off_bound + 4 * (size_t)(m + 1) + 15) & ~size_t(15);  // record size
  const size_t max_groups = (size_t)m * (size_t)(3 * k + 6) + 1;  // K5: up to 3 levels
  l.size = (l.off_groups + sizeof(Group) * max_groups + 255) & ~size_t(255);  // worst case
  return l;
}

int ensure_io(bz_ctx* ctx, int nslots) {
  const IoSlot l = io_layout(ctx->m, ctx->k);
  const size_t total = l.size * (size_t)std::max(nslots, 1) + 256;
  if (total > ctx->io_cap) {
    if (ctx->d_io) cudaFree(ctx->d_io);
    if (ctx->h_io) cudaFreeHost(ctx->h_io);
    ctx->d_io = ctx->h_io = nullptr;
    ctx->io_cap = 0;
    ctx->io_plans.clear();
    const size_t cap = std::max<size_t>(total, 64 * 1024);
    CK(cudaMalloc(&ctx->d_io, cap));
    CK(cudaMallocHost(&ctx->h_io, cap));
    ctx->io_cap = cap;
  }
  return BZ_OK;
}

// host / device views of slot i
// result record of round i (off < l.off_groups)
template <typename T>
T* slot_ptr(unsigned char* base, const IoSlot& l, int i, size_t off) {
  return reinterpret_cast<T*>(base + l.off_groups * (size_t)i + off);
}

// Work plan of one round (host only): one Group per (Gamma, ell) with its
// chunk range.  gamma_only < 0: all m Gammas.
// Shape of a pass: suffix depth D, prefixes walked in parallel per chunk,
// triples per tile.  K4 (tcgen05) and K3 (legacy IMMA) take D = 3 for
// g >= 4; K1 (POPC) takes D = 2 for g >= 4, else 1.  Histograms run on K1.
struct PlanShape {
  int depth, lanes, tile_rows, kernel;  // kernel: 1 = K1, 3 = K3, 4 = K4, 5 = K5, 6 = K5p,
                                        // 7 = K5t, 8 = K5q, 9 = K5w, 10 = K5f
};

// K5p (two codewords per accumulator column) needs odd W <= 3 stored words
bool k5p_ok(int w32) { return w32 == 1 || w32 == 3; }

// w32: stored words of the loaded family (0 = unknown, host-only plans):
// AUTO takes K5q where it applies (odd W <= 3), else K5
double binom_d(int p, int q);

// AUTO keeps K1 (D = 1) for rounds this small: their tensor-core groups
// hold few prefixes (g = 4: one per group), so a K5 launch is all fixed
// latency (~40 us warm on B200; K1 runs cfg5's g = 4 in 32 us)
// K4 / K5 chunk size: ~kK5ChunksPerCta chunks per persistent CTA, and at
// least kK5LaneMin prefixes x suffix rows per lane (a chunk costs a walker
// unrank per producer thread).  Swept on config 5 (tools/_lm.sh): 16 / 4096
// -> 11 / 8192 takes ~1 % off a run (g = 5..7 launches; g = 8 unchanged).
constexpr long long kK5ChunksPerCta = 11;
constexpr long long kK5LaneMin = 8192;
#ifndef BZ_AUTO_K1_COMBOS
#define BZ_AUTO_K1_COMBOS 1e7
#endif
constexpr double kAutoK1Combos = BZ_AUTO_K1_COMBOS;
// sharded calls: rounds below this many combinations x (nshards - 1) run
// whole on one rank (run_batch).  Only the trivial rounds: a batch's K1 rounds
// share one launch and its tensor-core rounds another, so splitting a small
// round adds no launch to any rank, while a rank that owned g = 5 or g = 6
// whole was the slowest of the job (config 5 as shard s of 8 on one GPU,
// slowest shard: 6e8 0.54 ms, 1e8 0.52, 1e7 .. 0 0.45-0.46 ms;
// tools/_own_sweep.sh)
constexpr double kOwnWholeCombos = 1e5;

// K5q: stored weights <= 128 (byte fields x = w + 128 - thr, thr in [1, 128];
// every Gamma's start bound is capped at its stored columns + offset), W <= 4
bool k5q_ok(int w32, int n_eff) { return w32 >= 1 && w32 <= 4 && n_eff <= 128; }

PlanShape pass_shape(int engine, int g, bool hist, int w32 = 0, int m = 0, int k = 0,
                     int n_eff = 0) {
  if (!hist && g >= 4 && engine == BZ_ENGINE_AUTO && m > 0 &&
      binom_d(k, g) * m <= kAutoK1Combos)
    return {1, 32, 0, 1};  // D = 1: many short prefixes keep every warp busy
  if (!hist && g >= 4) {
    if (engine == BZ_ENGINE_IMMA) return {3, bz::kTcThreads, bz::kTileRows, 3};
    if (engine == BZ_ENGINE_UMMA) return {3, bz::kUmmaM, bz::kUmmaN, 4};
    const bool packed_ok = w32 == 0 || k5p_ok(w32);
    if (engine == BZ_ENGINE_MXF4T && packed_ok) return {3, bz::kUmmaM, bz::k4_tile_rows<true, 3>(), 7};
    const bool q_ok = w32 == 0 || k5q_ok(w32, n_eff);
    // K5f: K5q's fields from folded MMAs (3 instead of 4 per tile at W = 3)
    // where the last stored word is at most half used (bz::k5f_ok); a
    // host-only plan (w32 = 0) has K5q's shape either way.  On request only:
    // config 5's g = 8 round measured 1.97 ms against K5q's 1.92 ms -- the
    // release chain of an accumulator buffer bounds both, and K5f adds an
    // IMAD per register to the epilogue (K5q)
    if (engine == BZ_ENGINE_MXF4F && w32 != 0 && bz::k5f_ok(w32, n_eff))
      return {3, bz::kUmmaM, bz::k4_tile_rows<true, 6>(), 10};
    if ((engine == BZ_ENGINE_MXF4Q || engine == BZ_ENGINE_MXF4F || engine == BZ_ENGINE_AUTO) && q_ok)
      return {3, bz::kUmmaM, bz::k4_tile_rows<true, 4>(), 8};  // K5q
    // K5w (two codewords per column as 11-bit fields) on request only: on
    // the wide section-6 codes it measured no faster than K5 (C1 round 12:
    // 70.0 vs 64.2 ms, tools/s6_rates.py) -- their rounds are bound by the
    // per-prefix-step cost (~13 tiles per step), and 480-row tiles fit
    // their suffix slices worse (tile efficiency 0.89 vs 0.94)
    if (engine == BZ_ENGINE_MXF4W && w32 != 1)
      return {3, bz::kUmmaM, bz::k4_tile_rows<true, 5>(), 9};
    if (engine == BZ_ENGINE_MXF4P && packed_ok) return {3, bz::kUmmaM, bz::k4_tile_rows<true, 2>(), 6};
    if (engine == BZ_ENGINE_AUTO || engine == BZ_ENGINE_MXF4 || engine == BZ_ENGINE_MXF4P ||
        engine == BZ_ENGINE_MXF4T || engine == BZ_ENGINE_MXF4Q || engine == BZ_ENGINE_MXF4F)
      return {3, bz::kUmmaM, bz::kUmmaN4, 5};
  }
  // D = 2 needs enough (g-3)-prefixes per group to fill a warp; at g = 3
  // every group would hold one prefix, so g <= 3 keeps D = 1
  return {g >= 4 ? 2 : 1, 32, 0, 1};
}

// K5 suffix levels.  Level D (3..5) owns the combinations whose top D
// elements all lie in rows >= floor[D] and whose (D+1)-th largest element
// ell is below floor[D+1]; its groups are (ell, D) with prefixes = the
// (g-1-D)-subsets of [0, ell) plus ell, and suffixes = the D-subsets of
// rows >= max(ell + 1, floor[D]) -- a prefix of that level's table (all
// D-subsets of rows >= floor[D], smallest element descending).  Deeper
// levels turn the many one-tile prefix steps of the small slices near
// ell = k - 4 into few steps over large slices; the floors are chosen by a
// cost model fitted to K5 (clocks per tile and per prefix step), with every
// table capped at kLevelRowCap rows per Gamma.
constexpr int kMaxLevel = 5;
constexpr unsigned long long kLevelRowCap = 1ull << 20;

struct Levels {
  int dmax = 3;                  // deepest level (3: plain triples)
  int floor[kMaxLevel + 2] = {}; // floor[D] for D in 3..dmax; floor[dmax+1] = k
};

// C(p, q) as double for 0 <= p, q <= BZ_MAX_K (cost model only)
double binom_d(int p, int q) {
  static const std::vector<double> t = [] {
    std::vector<double> v((BZ_MAX_K + 1) * (BZ_MAX_K + 1), 0.0);
    for (int a = 0; a <= BZ_MAX_K; ++a) {
      v[a * (BZ_MAX_K + 1)] = 1.0;
      for (int b = 1; b <= a; ++b)
        v[a * (BZ_MAX_K + 1) + b] = v[(a - 1) * (BZ_MAX_K + 1) + b - 1] +
                                    (b <= a - 1 ? v[(a - 1) * (BZ_MAX_K + 1) + b] : 0.0);
    }
    return v;
  }();
  if (p < 0 || q < 0 || q > p || p > BZ_MAX_K) return 0.0;
  return t[p * (BZ_MAX_K + 1) + q];
}

// (BZ_K5_MERGE=0: one group per ell, as before -- for A/B runs)
static bool merge_groups() {
  const char* e = getenv("BZ_K5_MERGE");
  return !e || atoi(e) != 0;
}

double k5_cost(int k, int g, const Levels& lv, int tile_rows) {
  // K5 clocks per tile / per prefix step (cfg5, B200); K5p/K5q tiles hold
  // twice the rows
  const bool pair = tile_rows > bz::kUmmaN4;
  // (K5q measured: ~625 clocks per tile in steady state; a prefix step --
  // walker step, A rows, the first tile's latency -- weighed ~3500 when every
  // ell was its own group.  The model still counts one group per ell while
  // build_plan merges the ells below a floor, and with merged plans a heavier
  // step weight finds better floors: swept 1500 .. 40000 on config 5, batch
  // 2.32 / 2.28 (3500) / 2.27 (8000) / 2.256 (12000 .. 20000) / 2.30 ms)
  double kTile = pair ? 650.0 : 727.0, kStep = pair ? 16000.0 : 1271.0;
  if (const char* env = getenv("BZ_K5_COST")) sscanf(env, "%lf,%lf", &kTile, &kStep);
  double cost = 0;
  for (int D = 3; D <= lv.dmax; ++D) {
    const int hi = std::min(lv.floor[D + 1] - 1, k - 1 - D);
    // (per ell, although build_plan merges the prefixes below a level's
    // floor into one group: floors chosen with the merged groups' fewer
    // steps counted -- (23, 42) instead of (26, 52) for config 5's g = 8 --
    // measured slower, 1.94 against 1.91 ms; the step weight was fitted to
    // the unmerged plans)
    for (int ell = g - 1 - D; ell <= hi; ++ell) {
      const double np = binom_d(ell, g - 1 - D);
      const int f = std::max(ell + 1, lv.floor[D]);
      const double slice = binom_d(k - f, D);
      if (np == 0 || slice == 0) continue;
      const double steps = std::ceil(np / bz::kUmmaM);
      cost += steps * (std::ceil(slice / tile_rows) * kTile + kStep);
    }
  }
  return cost;
}

Levels k5_levels_search(int k, int g, int tile_rows);

// memoised per (k, g, tile rows, BZ_K5_FLOORS): the search costs
// milliseconds and every round's plan (every process the same) asks for it
Levels k5_levels(int k, int g, int tile_rows) {
  static std::mutex mu;
  static std::map<std::string, Levels> memo;
  const char* env = getenv("BZ_K5_FLOORS");
  const char* cost = getenv("BZ_K5_COST");
  const std::string key = std::to_string(k) + "/" + std::to_string(g) + "/" +
                          std::to_string(tile_rows) + "/" + (env ? env : "") + "/" +
                          (cost ? cost : "");
  std::lock_guard<std::mutex> lock(mu);
  auto it = memo.find(key);
  if (it != memo.end()) return it->second;
  const Levels lv = k5_levels_search(k, g, tile_rows);
  memo.emplace(key, lv);
  return lv;
}

Levels k5_levels_search(int k, int g, int tile_rows) {
  Levels best;
  best.floor[3] = 0;
  best.floor[4] = k;
  if (g < 5) return best;  // a level-D prefix needs g - 1 - D >= 0
  if (const char* env = getenv("BZ_K5_FLOORS")) {
    // test hook: force the level floors "t1[,t2]" (clamped to valid ranges)
    int t1 = k, t2 = k;
    if (sscanf(env, "%d,%d", &t1, &t2) >= 1 && t1 >= 0 && t1 <= k - 4) {
      best.dmax = 4;
      best.floor[4] = t1;
      best.floor[5] = k;
      if (g >= 6 && t2 > t1 && t2 <= k - 5) {
        best.dmax = 5;
        best.floor[5] = t2;
        best.floor[6] = k;
      }
    }
    return best;
  }
  double best_cost = k5_cost(k, g, best, tile_rows);
  // one extra level (D = 4), then optionally D = 5 above it
  for (int t1 = 1; t1 <= k - 4; ++t1) {
    if (binom_sat(k - t1, 4) > kLevelRowCap) continue;
    Levels lv;
    lv.dmax = 4;
    lv.floor[3] = 0;
    lv.floor[4] = t1;
    lv.floor[5] = k;
    const double c4 = k5_cost(k, g, lv, tile_rows);
    if (c4 < best_cost) { best_cost = c4; best = lv; }
    if (g < 6) continue;
    for (int t2 = t1 + 1; t2 <= k - 5; ++t2) {
      if (binom_sat(k - t2, 5) > kLevelRowCap) continue;
      Levels l5 = lv;
      l5.dmax = 5;
      l5.floor[5] = t2;
      l5.floor[6] = k;
      const double c5 = k5_cost(k, g, l5, tile_rows);
      if (c5 < best_cost) { best_cost = c5; best = l5; }
    }
  }
  return best;
}

int build_plan(bz_ctx* ctx, int m, int k, int g, int gamma_only, PlanShape shape, int nshards,
               std::vector<Group>& gs, unsigned long long* out_nchunks) {
  gs.clear();
  unsigned long long chunk = 0;
  const int j0 = gamma_only < 0 ? 0 : gamma_only;
  const int j1 = gamma_only < 0 ? m : gamma_only + 1;
  const unsigned long long total = binom_sat(k, g) * (unsigned long long)(j1 - j0);
  long long lane_target = (long long)(total / (32ull * kChunksTarget));
  lane_target = std::min(kLaneMax, std::max(kLaneMin, lane_target));
  if (shape.kernel >= 4) {
    // K4 / K5: one persistent CTA per SM walks ~kK5ChunksPerCta chunks; a
    // chunk costs a walker unrank per producer thread, so chunks are large
    lane_target = (long long)(total / ((unsigned long long)shape.lanes * 148ull *
                                       (unsigned long long)kK5ChunksPerCta *
                                       (unsigned long long)std::max(1, nshards)));
    long long lane_min = kK5LaneMin;
    if (const char* lm = getenv("BZ_K5_LANE_MIN")) lane_min = atoll(lm);
    lane_target = std::min(1ll << 20, std::max(lane_min, lane_target));
    if (const char* sc = getenv("BZ_K5_CHUNK_SCALE")) lane_target = (long long)(lane_target * atof(sc));
  }
  // suffix levels: K5 may split the round over depths 3..5, every other
  // kernel runs one depth with floor ell + 1
  Levels lv;
  lv.dmax = shape.depth;
  lv.floor[shape.depth] = 0;
  lv.floor[shape.depth + 1] = k;
  if (shape.kernel >= 5) lv = k5_levels(k, g, shape.tile_rows);
  const int dmin = shape.depth;
  // K4/K5: the round's last ~15 % of combinations (in chunk order, which is
  // the order the CTAs draw them in) go in chunks 8x finer, so the SMs
  // finish together instead of waiting on a few large last chunks
  const unsigned long long fine_from = total - total / 7;
  unsigned long long done = 0;
  for (int j = j0; j < j1; ++j) {
    for (int depth = dmin; depth <= lv.dmax; ++depth) {
      const int ell_lo = g == 1 ? -1 : g - 1 - depth;
      const int ell_hi = g == 1 ? -1 : std::min(k - 1 - depth, lv.floor[depth + 1] - 1);
      // K5 family, levels above the first: every prefix whose last element
      // is below the level's floor has the same suffix slice [floor, k), and
      // those prefixes -- (g - D)-subsets of [0, bound) -- are consecutive
      // in colex order, so they form ONE group (sl = 0) instead of one per
      // ell: a group's last prefix step is partly empty, and the deep levels
      // have few prefixes per ell and thousands of tiles per step (config 5:
      // 7.7 % fewer tiles at g = 7, 2.7 % at g = 8, 0.9 % at g = 9).
      int merged_to = ell_lo - 1;  // last ell folded into the merged group
      if (shape.kernel >= 5 && g > 1 && depth > dmin && lv.floor[depth] - 1 > ell_lo && merge_groups())
        merged_to = std::min(ell_hi, lv.floor[depth] - 1);
      for (int ell = std::max(ell_lo, merged_to); ell <= ell_hi; ++ell) {
        const bool merged = ell == merged_to;
        const unsigned long long np = g == 1    ? 1ull
                                      : merged ? binom_sat(ell + 1, g - depth)
                                               : binom_sat(ell, g - 1 - depth);
        if (np == 0) continue;
        if (np >= (1ull << 62))
          return fail(ctx, BZ_ERR_TOO_LARGE, "C(%d,%d) prefixes exceed 2^62", ell, g - 1 - depth);
        const int sfloor = std::max(ell + 1, lv.floor[depth]);
        const long long work = (long long)binom_sat(k - sfloor, depth);
        if (work == 0) continue;
        const bool tiled = depth >= 3;
        const long long lt =
            (shape.kernel >= 4 && done >= fine_from) ? std::max(4096ll, lane_target / 8) : lane_target;
        done += np * (unsigned long long)work;
        // D >= 3: every prefix step also rebuilds the A operand and streams
        // at least one whole tile, which bounds chunk duration for the tiny
        // slices near ell = k - 4
        const long long step_cost =
            tiled ? std::max(work, (long long)shape.tile_rows) + 256 : work;
        // K1: the warp's 32 lanes are 32/sl prefix blocks x sl suffix lanes
        // (each takes every sl-th first suffix row).  A group with fewer
        // than 64 prefixes would leave lanes idle while others walk every
        // suffix (g = 1: one lane walked all k rows at ~125 clocks each), so
        // its suffixes are spread over the idle lanes.  (Spreading larger
        // groups too, for more and shorter chunks, measured slower: a
        // chunk's fixed cost -- group lookup, walker unrank -- is several
        // thousand clocks, config 5's fused g <= 4 went 25 -> 28 us.)
        long long sl = 1;
        if (!tiled) {
          const long long first_rows = depth == 1 ? k - sfloor : k - 1 - sfloor;
          while (sl < 32 && 2 * sl <= first_rows && 32 / sl > (long long)((np + 1) / 2))
            sl *= 2;
          // D = 2: a prefix carries up to C(k - 1, 2) codewords, so two of
          // them can be a chunk thousands of times longer than the round's
          // average -- the SMs holding those finish last (config 4's
          // histogram: SMs active 59 % of the launch).  Spread such
          // prefixes' first suffix rows over lanes until a lane's share is
          // near an even split of the round over 16 warps per SM (swept
          // 2..512, and again 16..128 with K1h at 32 warps per SM: flat to
          // 32, slower beyond: config-4 histogram 191 -> 127 us, its K1 minimum 156 ->
          // 101 us, config 5's g = 5 on K1 184 -> 65 us).
          if (depth == 2) {
            const long long even = (long long)(total / (32ull * 148ull * 16ull));
            const long long lt_w = std::max(lane_target, even);
            while (sl < 32 && 2 * sl <= first_rows && 2 * work / sl > lt_w) sl *= 2;
          }
        }
        const long long lanes_ll = tiled ? shape.lanes : 32 / sl;
        const long long spread = (long long)((np + lanes_ll - 1) / lanes_ll);
        long long ppl = std::max(1ll, lt * sl / std::max(1ll, step_cost));
        // K1 lanes walk their range with two walkers (halves): a lane with a
        // single prefix runs its second walker on a duplicate, so give every
        // lane two prefixes where the group has them (config 4: 2x the work)
        if (!tiled) ppl = std::max(ppl, 2ll);
        // one-element prefix tails (g - 1 - D <= 1): a fresh init is one row,
        // cheaper than a colex step (two), so walkers take one prefix each
        if (!tiled && g - 1 - depth <= 1) ppl = 2;
        ppl = std::min(ppl, std::max(1ll, spread));
        // D >= 3: a chunk is lanes prefixes x ppl steps x tpc tiles; a slice
        // too large for one chunk is split into tile blocks
        const long long trows = tiled ? shape.tile_rows : 1;
        long long ntiles = (work + trows - 1) / trows;
        long long tpc = ntiles;
        if (tiled && work > lt) tpc = std::max(1ll, lt / trows);
        const long long ntb = tiled ? (ntiles + tpc - 1) / tpc : 1;
        Group gr{};
        gr.chunk_begin = chunk;
        gr.nprefix = np;
        gr.gamma = j;
        gr.ell = ell;
        gr.ppl = (int)ppl;
        gr.depth = depth;
        gr.tpc = (int)tpc;
        gr.ntb = (int)ntb;
        gr.lanes = shape.lanes;
        gr.tile_rows = shape.tile_rows;
        gr.slice = (int)work;
        gr.sfloor = sfloor;
        gr.sl = merged ? 0 : (int)sl;
        const unsigned long long per_chunk = (unsigned long long)lanes_ll * (unsigned long long)ppl;
        chunk += (np + per_chunk - 1) / per_chunk * (unsigned long long)ntb;
        gs.push_back(gr);
      }
    }
  }
  *out_nchunks = chunk;
  return BZ_OK;
}

// Build the round's group table into I/O slot `slot` (host side).
// A plan depends only on (m, k, g, Gamma filter, kernel shape, shard count)
// and the planning knobs, never on the matrices, so plans are memoised per
// process: a repeated run (same dimensions) copies its group tables instead
// of re-planning every round before the first launch.
// the planning knobs (test and tuning hooks), read once per batch
struct PlanKnobs {
  const char *floors, *scale, *cost, *lmin, *merge;
  PlanKnobs()
      : floors(getenv("BZ_K5_FLOORS")), scale(getenv("BZ_K5_CHUNK_SCALE")),
        cost(getenv("BZ_K5_COST")), lmin(getenv("BZ_K5_LANE_MIN")),
        merge(getenv("BZ_K5_MERGE")) {}
};

int plan_round(bz_ctx* ctx, int g, int gamma_only, PlanShape shape, int nshards, size_t goff,
               int* out_ngroups, unsigned long long* out_nchunks, int slot, bool* out_fresh,
               const PlanKnobs& kn) {
  struct Plan {
    std::vector<Group> groups;
    unsigned long long nchunks;
  };
  static std::mutex mu;
  static std::map<std::string, Plan> memo;
  const char *floors = kn.floors, *scale = kn.scale, *cost = kn.cost, *lmin = kn.lmin;
  char key[384];
  snprintf(key, sizeof key, "%d/%d/%d/%d/%d/%d/%d/%d/%d/%s/%s/%s/%s/%s", ctx->m, ctx->k, g, gamma_only,
           shape.kernel, shape.depth, shape.lanes, shape.tile_rows, nshards, floors ? floors : "",
           scale ? scale : "", cost ? cost : "", lmin ? lmin : "", kn.merge ? kn.merge : "");
  const IoSlot l = io_layout(ctx->m, ctx->k);
  std::lock_guard<std::mutex> lock(mu);
  auto it = memo.find(key);
  if (it == memo.end()) {
    Plan p;
    int rc = build_plan(ctx, ctx->m, ctx->k, g, gamma_only, shape, nshards, p.groups, &p.nchunks);
    if (rc) return rc;
    if (memo.size() > 4096) memo.clear();
    it = memo.emplace(key, std::move(p)).first;
  }
  (void)l;
  // already in place from the last batch (host image and device copy)?
  const bool same = slot < (int)ctx->io_plans.size() && ctx->io_plans[slot].first == key &&
                    ctx->io_plans[slot].second == goff;
  if (!same) {
    std::memcpy(ctx->h_io + goff, it->second.groups.data(), it->second.groups.size() * sizeof(Group));
    if ((int)ctx->io_plans.size() <= slot) ctx->io_plans.resize(slot + 1);
    ctx->io_plans[slot] = {key, goff};
  }
  *out_fresh = !same;
  *out_ngroups = (int)it->second.groups.size();
  *out_nchunks = it->second.nchunks;
  return BZ_OK;
}

int check_g(bz_ctx* ctx, int g) {
  if (!ctx->d_rows) return fail(ctx, BZ_ERR_STATE, "no Gamma family loaded");
  if (g < 1 || g > ctx->k)
    return fail(ctx, BZ_ERR_INVALID_ARITY, "g=%d not in 1..%d", g, ctx->k);
  if (binom_sat(ctx->k, g) >= (1ull << 62))
    return fail(ctx, BZ_ERR_TOO_LARGE, "C(%d,%d) >= 2^62 combinations", ctx->k, g);
  return BZ_OK;
}

// Host-side launch preparation, memoised: the dynamic shared memory limit
// is raised once per kernel and the occupancy query runs once per (device,
// kernel, block size, shared memory).  Uncached they cost more host time per
// launch than a small round's kernel runs, which left the stream idle
// between the batched early rounds.
int prep_launch(bz_ctx* ctx, const void* fn, int threads, size_t smem, int* per_sm) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*>, size_t> attr;
  static std::map<std::tuple<int, const void*, int, size_t>, int> occ;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = attr[{ctx->device, fn}];
  if (smem > have) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    have = smem;
  }
  const auto key = std::make_tuple(ctx->device, fn, threads, smem);
  auto it = occ.find(key);
  if (it == occ.end()) {
    int n = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem));
    it = occ.emplace(key, n).first;
  }
  *per_sm = it->second;
  return BZ_OK;
}

// largest dynamic shared memory per block (sm_100: 227 KB)
constexpr size_t kMaxSmem = 232448;

template <int W, int D>
int launch_wd(bz_ctx* ctx, const RoundArgs& a0, bool hist) {
  RoundArgs a = a0;
  size_t smem = bz::smem_base_bytes<W>(a.m, a.k, a.ngroups);
  if (smem + (hist ? (size_t)bz::k1h_bins<W>(a.n) * 4 + (size_t)(bz::kK1hWindow + 1) * 2 * bz::kK1hMinThreads + 32 : 0) > kMaxSmem) {
    a.groups_global = 1;  // a plan too large to stage: read from global memory
    smem = bz::smem_base_bytes<W>(a.m, a.k, 0);
  }
  int threads = 256;
  if (hist) {
    // bins for the stored weights only (at most 32 W stored columns: the
    // dropped identity weight is added when the block's bins are flushed)
    const size_t nbins = (size_t)bz::k1h_bins<W>(a.n);
    smem = ((smem + 15) & ~size_t(15)) + ((nbins + 3) & ~size_t(3)) * 4;
    // per-thread 16-bit counters over the window
    int dev_max = 0;
    CK(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    const size_t win = (size_t)bz::k1h_window((int)nbins);
    while (threads > bz::kK1hMinThreads && smem + (win + 1) * threads * 2 > (size_t)dev_max / 2)
      threads /= 2;
    smem += (win + 1) * threads * 2;  // + the trash row
  }
  int per_sm = 0;
  const void* fn = hist ? (const void*)bz::k1h_histogram<W, D> : (const void*)bz::k1_round_min<W, D>;
  int rc = prep_launch(ctx, fn, threads, smem, &per_sm);
  if (rc) return rc;
  if (per_sm < 1) return fail(ctx, BZ_ERR_TOO_LARGE, "kernel does not fit on an SM (smem %zu)", smem);
  // persistent grid: one wave, but no more warps than chunks need
  unsigned long long warps_needed = (a.nchunks + a.nshards - 1) / a.nshards;
  long long blocks = (long long)per_sm * ctx->sm_count;
  long long need = (long long)((warps_needed + (threads / 32) - 1) / (threads / 32));
  blocks = std::max(1ll, std::min(blocks, need));
  if (hist)
    bz::k1h_histogram<W, D><<<(unsigned)blocks, threads, smem, ctx->stream>>>(a);
  else
    bz::k1_round_min<W, D><<<(unsigned)blocks, threads, smem, ctx->stream>>>(a);
  CK(cudaGetLastError());
  ctx->launches += 1;
  return BZ_OK;
}

// Consecutive K1 rounds of one batch in one launch (k1_rounds).
template <int W, int D>
int launch_k1_fused(bz_ctx* ctx, const RoundArgs* as, int count) {
  bz::K1Batch b{};
  int cap = 0;
  unsigned long long warps = 0;
  for (int i = 0; i < count; ++i) {  // the plans side by side, one chunk space
    cap += as[i].ngroups;
    if (as[i].nchunks > (unsigned long long)as[i].shard)
      warps += (as[i].nchunks - as[i].shard + as[i].nshards - 1) / as[i].nshards;
  }
  for (int i = 0; i < count; ++i) {
    b.a[i] = as[i];
    b.a[i].sgroups_cap = cap;
    b.a[i].chain = nullptr;
  }
  b.count = count;
  const size_t smem = bz::smem_base_bytes<W>(as[0].m, as[0].k, cap);
  const int threads = 256;
  int per_sm = 0;
  int rc = prep_launch(ctx, (const void*)bz::k1_rounds<W, D>, threads, smem, &per_sm);
  if (rc) return rc;
  if (per_sm < 1) return fail(ctx, BZ_ERR_TOO_LARGE, "kernel does not fit on an SM (smem %zu)", smem);
  long long blocks = (long long)per_sm * ctx->sm_count;
  blocks = std::max(1ll, std::min(blocks, (long long)((warps + 7) / 8)));
  bz::k1_rounds<W, D><<<(unsigned)blocks, threads, smem, ctx->stream>>>(b);
  CK(cudaGetLastError());
  ctx->launches += 1;
  return BZ_OK;
}

template <int W>
int launch_fused_w(bz_ctx* ctx, const RoundArgs* as, int count, int depth) {
  return depth == 2 ? launch_k1_fused<W, 2>(ctx, as, count) : launch_k1_fused<W, 1>(ctx, as, count);
}

int launch_fused(bz_ctx* ctx, const RoundArgs* as, int count, int depth) {
  switch (ctx->w32) {
    case 1: return launch_fused_w<1>(ctx, as, count, depth);
    case 2: return launch_fused_w<2>(ctx, as, count, depth);
    case 3: return launch_fused_w<3>(ctx, as, count, depth);
    case 4: return launch_fused_w<4>(ctx, as, count, depth);
    case 5: return launch_fused_w<5>(ctx, as, count, depth);
    case 6: return launch_fused_w<6>(ctx, as, count, depth);
    case 7: return launch_fused_w<7>(ctx, as, count, depth);
    case 8: return launch_fused_w<8>(ctx, as, count, depth);
    default: return fail(ctx, BZ_ERR_TOO_LARGE, "unsupported word count %d", ctx->w32);
  }
}

#if BZ_LEGACY_KERNELS
template <int W>
int launch_tc(bz_ctx* ctx, const RoundArgs& a) {
  const size_t smem = bz::k3_smem_bytes<W>(a.m, a.k, a.ngroups);
  const int threads = bz::kTcThreads;
  int per_sm = 0;
  int rc = prep_launch(ctx, (const void*)bz::k3_round_gemm<W>, threads, smem, &per_sm);
  if (rc) return rc;
  if (per_sm < 1) return fail(ctx, BZ_ERR_TOO_LARGE, "K3 does not fit on an SM (smem %zu)", smem);
  const unsigned long long blocks_needed = (a.nchunks + a.nshards - 1) / a.nshards;
  long long blocks = (long long)per_sm * ctx->sm_count;
  blocks = std::max(1ll, std::min(blocks, (long long)blocks_needed));
  bz::k3_round_gemm<W><<<(unsigned)blocks, threads, smem, ctx->stream>>>(a, ctx->d_trip,
                                                                         ctx->trip_rows);
  CK(cudaGetLastError());
  ctx->launches += 1;
  return BZ_OK;
}

#endif

// One tensor-core launch of `count` consecutive rounds (K5Batch): their
// plans staged side by side (or all read from global memory when they do not
// fit), their chunk spaces concatenated on round 0's cursor.
template <int W, bool F4, int CW = 1>
int launch_umma(bz_ctx* ctx, const RoundArgs* as, int count) {
  bz::K5Batch bt{};
  int total_groups = 0;
  unsigned long long mine_total = 0;
  for (int i = 0; i < count; ++i) {
    bt.a[i] = as[i];
    bt.goff[i] = total_groups;
    total_groups += as[i].ngroups;
    const RoundArgs& r = as[i];
    mine_total += r.nchunks > (unsigned long long)r.shard
                      ? (r.nchunks - r.shard + r.nshards - 1) / r.nshards : 0ull;
    bt.cend[i] = mine_total;
  }
  bt.count = count;
  for (int i = 0; i < count; ++i) {
    bt.a[i].sgroups_cap = total_groups;
    bt.a[i].trace = as[count - 1].trace;
    bt.a[i].ctrace = as[count - 1].ctrace;
  }
  RoundArgs& a = bt.a[0];
  size_t smem = bz::k4_smem_bytes<W, F4, CW>(a.m, a.k, total_groups);
  if (smem > kMaxSmem) {
    // plans too large to stage: read from global memory
    for (int i = 0; i < count; ++i) bt.a[i].groups_global = 1;
    smem = bz::k4_smem_bytes<W, F4, CW>(a.m, a.k, 0);
  }
  if (smem > kMaxSmem)
    return fail(ctx, BZ_ERR_TOO_LARGE, "K%d does not fit on an SM (smem %zu)", F4 ? 5 : 4, smem);
  {
    static std::mutex mu;
    static std::map<int, size_t> have;  // per device: the attribute is per function
    std::lock_guard<std::mutex> lock(mu);
    if (smem > have[ctx->device]) {
      CK(cudaFuncSetAttribute(bz::k4_round_umma<W, F4, CW>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      have[ctx->device] = smem;
    }
  }
  long long blocks = std::max(1ll, std::min((long long)ctx->sm_count, (long long)mine_total));
  bz::K4Tables tabs{};
  if (F4) {
    for (int i = 0; i < 3; ++i) {
      tabs.t[i] = ctx->d_lvl[i];
      tabs.stride_rows[i] = ctx->lvl_rows[i];
    }
  } else {
    tabs.t[0] = ctx->d_trip4;
    tabs.stride_rows[0] = ctx->trip4_rows;
  }
  // programmatic dependent launch after another round kernel: this
  // launch's CTAs take SMs as the previous round's CTAs exit (the rounds
  // are independent; the optional U chain tolerates an early read)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(bz::K4Roles<F4, CW>::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx->pdl_next ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, bz::k4_round_umma<W, F4, CW>, bt, tabs));
  ctx->launches += 1;
  return BZ_OK;
}

#if BZ_LEGACY_KERNELS
template <int W>
int build_triples_w(bz_ctx* ctx, int which) {
  dim3 grid(ctx->k, ctx->m);
  if (which == 3) {
    bz::k_build_triples<W><<<grid, 256, 0, ctx->stream>>>(ctx->d_rows, ctx->d_trip, ctx->k,
                                                          ctx->trip_rows);
  } else {
    bz::k_build_triples_umma<W><<<grid, 256, 0, ctx->stream>>>(
        ctx->d_rows, ctx->d_trip4, ctx->k, ctx->trip4_rows);
  }
  CK(cudaGetLastError());
  ctx->launches += 1;
  return BZ_OK;
}

#endif

template <int W, int FORM = 1>
int build_level_w(bz_ctx* ctx, int D, int floor) {
  const unsigned long long n = binom_sat(ctx->k - floor, D);
  // every row of the Gamma's stride: the subsets, then the empty-subset tail
  // kBuildRows rows per thread (k_build_subsets_mxf4)
  dim3 grid((unsigned)((ctx->lvl_rows[D - 3] / bz::kBuildRows + 127) / 128), ctx->m);
  if (!ctx->side_pending) {
    // the side stream starts after everything enqueued so far (the rows)
    CK(cudaEventRecord(ctx->ev_main, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_main, 0));
    ctx->side_pending = true;
  }
  bz::k_build_subsets_mxf4<W, FORM><<<grid, 128, 0, ctx->side>>>(
      ctx->d_rows, ctx->d_lvl[D - 3], ctx->k, D, n, ctx->lvl_rows[D - 3], ctx->d_binom);
  CK(cudaGetLastError());
  ctx->launches += 1;
  return BZ_OK;
}

// K5 suffix table of level D covering every D-subset of rows >= floor
// (grow-only: a table built for a lower floor already holds these subsets
// as its first rows).  Not zero-filled: padding rows are only ever read into
// columns the kernel masks.
// form: the row format -- 6 for K5f (the last chunk half data, half offset
// pattern), else 1 (K5 / K5q / K5w rows); tables of another format are
// rebuilt.
int ensure_level(bz_ctx* ctx, int D, int floor, int form) {
  const int i = D - 3;
  if (ctx->lvl_form != form) {
    for (int q = 0; q < 3; ++q) ctx->lvl_floor[q] = -1;
    ctx->lvl_form = form;
  }
  if (ctx->lvl_floor[i] >= 0 && ctx->lvl_floor[i] <= floor) return BZ_OK;
  if (ctx->k - floor < D) return BZ_OK;  // no subsets: nothing reads it
  const size_t n = (size_t)binom_sat(ctx->k - floor, D);
  // whole K5t tiles (three accumulator widths; also covers K5p's two) plus
  // one tile of slack
  const size_t N = bz::k4_tile_rows<true, 3>();
  ctx->lvl_rows[i] = (n + N - 1) / N * N + N;
  const size_t row_bytes = (size_t)bz::k4_row_bytes<true>(ctx->w32, form);
  const size_t bytes = (size_t)ctx->m * ctx->lvl_rows[i] * row_bytes;
  CK(grow(ctx, (void**)&ctx->d_lvl[i], &ctx->lvl_cap[i], bytes));
  int rc;
  switch (ctx->w32) {
    case 1: rc = form == 6 ? build_level_w<1, 6>(ctx, D, floor) : build_level_w<1>(ctx, D, floor); break;
    case 2: rc = build_level_w<2>(ctx, D, floor); break;
    case 3: rc = form == 6 ? build_level_w<3, 6>(ctx, D, floor) : build_level_w<3>(ctx, D, floor); break;
    case 4: rc = build_level_w<4>(ctx, D, floor); break;
    case 5: rc = build_level_w<5>(ctx, D, floor); break;
    case 6: rc = build_level_w<6>(ctx, D, floor); break;
    case 7: rc = build_level_w<7>(ctx, D, floor); break;
    case 8: rc = build_level_w<8>(ctx, D, floor); break;
    default: return fail(ctx, BZ_ERR_TOO_LARGE, "unsupported word count %d", ctx->w32);
  }
  if (rc) return rc;
  ctx->lvl_floor[i] = floor;
  return BZ_OK;
}

#if BZ_LEGACY_KERNELS
// Build (once per loaded family) the triple table kernel `which` (3: K3
// layout, 4: K4 s8 UMMA layout) reads.  Tables are not zero-filled: padding
// rows are only ever read into columns the kernels mask.
int ensure_triples(bz_ctx* ctx, int which) {
  bool& built = which == 3 ? ctx->trip_built : ctx->trip4_built;
  if (built) return BZ_OK;
  if (ctx->k < 4) return fail(ctx, BZ_ERR_STATE, "triple tables need k >= 4");
  const size_t bytes = which == 3
                           ? (size_t)ctx->m * ctx->trip_rows * bz::tc_stride(ctx->w32)
                           : (size_t)ctx->m * ctx->trip4_rows * 32 * ctx->w32;
  if (which == 3)
    CK(grow(ctx, (void**)&ctx->d_trip, &ctx->trip_cap, bytes));
  else
    CK(grow(ctx, (void**)&ctx->d_trip4, &ctx->trip4_cap, bytes));
  int rc;
  switch (ctx->w32) {
    case 1: rc = build_triples_w<1>(ctx, which); break;
    case 2: rc = build_triples_w<2>(ctx, which); break;
    case 3: rc = build_triples_w<3>(ctx, which); break;
    case 4: rc = build_triples_w<4>(ctx, which); break;
    case 5: rc = build_triples_w<5>(ctx, which); break;
    case 6: rc = build_triples_w<6>(ctx, which); break;
    case 7: rc = build_triples_w<7>(ctx, which); break;
    case 8: rc = build_triples_w<8>(ctx, which); break;
    default: return fail(ctx, BZ_ERR_TOO_LARGE, "unsupported word count %d", ctx->w32);
  }
  if (rc) return rc;
  built = true;
  return BZ_OK;
}

#else
int ensure_triples(bz_ctx* ctx, int) {
  return fail(ctx, BZ_ERR_STATE, "K3/K4 not built (BZ_LEGACY_KERNELS=0)");
}
#endif

template <int W>
int launch_seed_w(bz_ctx* ctx, const RoundArgs& a, int gamma_only) {
  if (a.g > bz::kSeedMaxG) return BZ_OK;
  bz::k_seed_bound<W><<<(unsigned)ctx->sm_count, 128, 0, ctx->stream>>>(a, gamma_only, 1);
  CK(cudaGetLastError());
  ctx->launches += 1;
  return BZ_OK;
}

int launch_seed(bz_ctx* ctx, const RoundArgs& a, int gamma_only) {
  switch (ctx->w32) {
    case 1: return launch_seed_w<1>(ctx, a, gamma_only);
    case 2: return launch_seed_w<2>(ctx, a, gamma_only);
    case 3: return launch_seed_w<3>(ctx, a, gamma_only);
    case 4: return launch_seed_w<4>(ctx, a, gamma_only);
    case 5: return launch_seed_w<5>(ctx, a, gamma_only);
    case 6: return launch_seed_w<6>(ctx, a, gamma_only);
    case 7: return launch_seed_w<7>(ctx, a, gamma_only);
    case 8: return launch_seed_w<8>(ctx, a, gamma_only);
    default: return fail(ctx, BZ_ERR_TOO_LARGE, "unsupported word count %d", ctx->w32);
  }
}

// `count` consecutive rounds of the same tensor-core shape in one launch
// (count = 1 for every other kernel)
template <int W>
int launch_w(bz_ctx* ctx, const RoundArgs* as, int count, bool hist, const PlanShape& shape) {
  const RoundArgs& a = as[0];
#if BZ_LEGACY_KERNELS
  if constexpr (W == 1 || W == 3) {
    if (shape.kernel == 6) return launch_umma<W, true, 2>(ctx, as, count);
    if (shape.kernel == 7) return launch_umma<W, true, 3>(ctx, as, count);
  }
  if (shape.kernel == 4) return launch_umma<W, false>(ctx, as, count);
  if (shape.kernel == 3) return launch_tc<W>(ctx, a);
#endif
  if constexpr (W <= 4)
    if (shape.kernel == 8) return launch_umma<W, true, 4>(ctx, as, count);
  if constexpr (W >= 2)
    if (shape.kernel == 9) return launch_umma<W, true, 5>(ctx, as, count);
  if constexpr (W == 1 || W == 3)
    if (shape.kernel == 10) return launch_umma<W, true, 6>(ctx, as, count);
  if (shape.kernel >= 3 && shape.kernel != 5)
    return fail(ctx, BZ_ERR_STATE, "kernel %d not available at W = %d", shape.kernel, W);
  if (shape.kernel == 5) return launch_umma<W, true>(ctx, as, count);
  return shape.depth == 2 ? launch_wd<W, 2>(ctx, a, hist) : launch_wd<W, 1>(ctx, a, hist);
}

int launch(bz_ctx* ctx, const RoundArgs* as, int count, bool hist, const PlanShape& depth) {
  switch (ctx->w32) {
    case 1: return launch_w<1>(ctx, as, count, hist, depth);
    case 2: return launch_w<2>(ctx, as, count, hist, depth);
    case 3: return launch_w<3>(ctx, as, count, hist, depth);
    case 4: return launch_w<4>(ctx, as, count, hist, depth);
    case 5: return launch_w<5>(ctx, as, count, hist, depth);
    case 6: return launch_w<6>(ctx, as, count, hist, depth);
    case 7: return launch_w<7>(ctx, as, count, hist, depth);
    case 8: return launch_w<8>(ctx, as, count, hist, depth);
    default: return fail(ctx, BZ_ERR_TOO_LARGE, "unsupported word count %d", ctx->w32);
  }
}

// Shared body of bz_round / bz_rounds / bz_enumerate / bz_histogram: rounds
// g0 .. g0+count-1 (each over all Gammas, or only `gamma_only`) planned on
// the host, one H2D of their I/O slots, the launches back to back on the
// stream, one D2H, one synchronisation.  lower_prev[i] is round i's early
// exit threshold; every round starts from the same `upper`.
int run_batch(bz_ctx* ctx, int g0, int count, int gamma_only, const int* lower_prev,
              int upper, int shard, int nshards, bool hist) {
  if (nshards < 1 || shard < 0 || shard >= nshards)
    return fail(ctx, BZ_ERR_ARGUMENT, "bad shard %d of %d", shard, nshards);
  if (count < 1 || (hist && count != 1)) return fail(ctx, BZ_ERR_ARGUMENT, "bad count %d", count);
  for (int i = 0; i < count; ++i) {
    int rc = check_g(ctx, g0 + i);
    if (rc) return rc;
  }
  int rc = ensure_io(ctx, count);
  if (rc) return rc;
  const IoSlot l = io_layout(ctx->m, ctx->k);
  const int m = ctx->m;
  struct Pending {
    RoundArgs a;
    PlanShape shape;
    bool run;
    bool seed;  // a threshold kernel starting with no bound: seed it first
  };
  std::vector<Pending> todo(count);
  long long* trace = nullptr;
  long long* ctrace = nullptr;
  int debug = 0;
  {
    // timing experiments on K4 (results are NOT valid when set): bit 0 skips
    // the epilogue's TMEM reads, bit 1 the TMA tile loads, bit 2 the MMAs,
    // bit 3 records a per-tile timeline of block 0, bit 4 skips the producers' A rows, bit 5 records per-chunk times
    const char* dbg = getenv("BZ_K4_DEBUG");
    debug = dbg ? atoi(dbg) : 0;
    if (debug & 8) {
      static long long* d_trace = nullptr;
      if (!d_trace) CK(cudaMalloc(&d_trace, 16 * 256 * sizeof(long long)));
      CK(cudaMemsetAsync(d_trace, 0, 16 * 256 * sizeof(long long), ctx->stream));
      trace = d_trace;
    }
    if (debug & 32) {
      static long long* d_ct = nullptr;
      if (!d_ct) CK(cudaMalloc(&d_ct, 1024 * 64 * 4 * sizeof(long long)));
      CK(cudaMemsetAsync(d_ct, 0xff, 1024 * 64 * 4 * sizeof(long long), ctx->stream));
      ctrace = d_ct;
    }
  }
  // Sharded calls: a round too small to be worth splitting (a few hundred
  // thousand combinations: kOwnWholeCombos) is run
  // whole by one rank, round-robin over such rounds; the other ranks
  // report nothing for it (upper / 0), which the exchange's min / sum
  // absorbs.  Every rank decides alike from (m, k, g, nshards).
  std::vector<int> owner(count, -1);
  if (nshards > 1 && !hist) {
    int owned = 0;
    double own_whole = kOwnWholeCombos;
    if (const char* e = getenv("BZ_OWN_WHOLE")) own_whole = atof(e);  // (experiments; alike on every rank)
    const double mult = gamma_only < 0 ? (double)m : 1.0;
    for (int i = 0; i < count; ++i)
      if (mult * binom_d(ctx->k, g0 + i) < own_whole * (nshards - 1))
        owner[i] = owned++ % nshards;
  }
  const auto t_plan0 = std::chrono::steady_clock::now();
  // plans follow the result records; goff = where round i's groups go
  size_t goff = ((size_t)count * l.off_groups + 255) & ~size_t(255);
  size_t first_fresh = SIZE_MAX;  // first group table this batch has to upload
  const PlanKnobs knobs;
  int trace_from = 0, trace_ell = -1;
  int lvl_lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX};  // lowest floor per level (D = 3..5)
  int lvl_form = 1;                                   // row format of the batch's tables
  if (debug) {
    if (const char* e = getenv("BZ_K4_TRACE_FROM")) trace_from = atoi(e);
    if (const char* e = getenv("BZ_K4_TRACE_ELL")) trace_ell = atoi(e);
  }
  for (int i = 0; i < count; ++i) {
    const int g = g0 + i;
    const PlanShape shape = pass_shape(ctx->engine, g, hist, ctx->w32, ctx->m, ctx->k, ctx->n_eff);
    if (shape.kernel == 3 || shape.kernel == 4) {
      rc = ensure_triples(ctx, shape.kernel);
      if (rc) return rc;
    }
    int ngroups = 0;
    unsigned long long nchunks = 0;
    const size_t gthis = goff;
    const int r_shard = owner[i] >= 0 ? 0 : shard, r_nshards = owner[i] >= 0 ? 1 : nshards;
    bool fresh = true;
    rc = plan_round(ctx, g, gamma_only, shape, r_nshards, gthis, &ngroups, &nchunks, i, &fresh,
                    knobs);
    if (rc) return rc;
    if (fresh && first_fresh == SIZE_MAX) first_fresh = gthis;
    if (shape.kernel >= 5) {
      // the suffix tables this round's levels read
      const Group* gp = reinterpret_cast<const Group*>(ctx->h_io + gthis);
      for (int q = 0; q < ngroups; ++q)
        lvl_lo[gp[q].depth - 3] = std::min(lvl_lo[gp[q].depth - 3], gp[q].sfloor);
      if (shape.kernel == 10) lvl_form = 6;
    }
    *slot_ptr<unsigned long long>(ctx->h_io, l, i, 0) = 0ull;
    unsigned long long* hc = slot_ptr<unsigned long long>(ctx->h_io, l, i, l.off_combos);
    int* hb = slot_ptr<int>(ctx->h_io, l, i, l.off_bound);
    for (int j = 0; j < 3 * m; ++j) hc[j] = 0ull;  // combos, adds, accs
    for (int j = 0; j <= m; ++j) hb[j] = upper;  // per-Gamma caps below, once `run` is known
    RoundArgs& a = todo[i].a;
    a = RoundArgs{};
    a.rows = ctx->d_rows;
    a.px = ctx->d_px;
    a.groups = reinterpret_cast<const Group*>(ctx->d_io + gthis);
    a.binom = ctx->d_binom;
    a.bound = slot_ptr<int>(ctx->d_io, l, i, l.off_bound);
    a.combos = slot_ptr<unsigned long long>(ctx->d_io, l, i, l.off_combos);
    a.adds = hist ? nullptr : slot_ptr<unsigned long long>(ctx->d_io, l, i, l.off_adds);
    a.accs = hist ? nullptr : slot_ptr<unsigned long long>(ctx->d_io, l, i, l.off_accs);
    a.counter = slot_ptr<unsigned long long>(ctx->d_io, l, i, 0);
    a.hist = ctx->d_hist;
    a.nchunks = nchunks;
    a.ngroups = ngroups;
    a.m = m;
    a.k = ctx->k;
    a.g = g;
    a.n = ctx->n;
    a.shard = r_shard;
    a.nshards = r_nshards;
    a.lower_prev = lower_prev ? lower_prev[i] : 0;
    a.exit_own = ctx->early_exit;
    a.elide = ctx->elide_mask;
    a.debug = debug;
    a.trace = (i == count - 1) ? trace : nullptr;
    a.trace_from = trace_from;
    a.ctrace = (i == count - 1) ? ctrace : nullptr;
    a.trace_ell = trace_ell;
    a.chain = i > 0 ? todo[i - 1].a.bound : nullptr;
    a.gbound = gamma_only < 0 ? ctx->d_gbound : nullptr;  // whole rounds only
    a.gtag = ctx->gtag;
    todo[i].shape = shape;
    todo[i].run = nchunks > 0 && (unsigned long long)r_shard < nchunks &&
                  (owner[i] < 0 || owner[i] == shard);
    if (todo[i].run && !hist) {
      // no codeword of Gamma j weighs more than its stored columns plus the
      // elided g, so a shard that visits any of its combinations reports
      // min(upper, true minimum) exactly when its bound starts at that cap --
      // which keeps K5q's threshold inside its byte fields (k5q_threshold)
      bool loose = shape.kernel == 8 || shape.kernel == 9 || shape.kernel == 10;
      for (int j = 0; j < m; ++j)
        if (gamma_only < 0 || gamma_only == j) {
          const long long cap =
              (long long)ctx->n_stored[j] + (((ctx->elide_mask >> j) & 1ull) ? g : 0);
          if (cap < hb[1 + j]) hb[1 + j] = (int)cap;
          else loose = false;  // the caller's bound already says something
        }
      todo[i].seed = loose && !debug;
    }
    goff = (gthis + (size_t)ngroups * sizeof(Group) + 255) & ~size_t(255);
  }
  // entries past this batch describe memory it may have overwritten
  ctx->io_plans.resize(count);
  // every suffix table once, at the lowest floor any round of the batch
  // reads (a table for a lower floor holds a higher floor's rows as its
  // first rows): rounds g = 5, 6, 7 ... lower the D = 4, 5 floors in turn,
  // and building per round rebuilt each table up to three times
  for (int D = 3; D <= 5; ++D)
    if (lvl_lo[D - 3] != INT32_MAX) {
      rc = ensure_level(ctx, D, D == 3 ? 0 : lvl_lo[D - 3], lvl_form);
      if (rc) return rc;
    }
  const auto t_plan1 = std::chrono::steady_clock::now();
  if (hist)
    CK(cudaMemsetAsync(ctx->d_hist, 0, sizeof(unsigned long long) * (ctx->n + 1), ctx->stream));
  // the used image only: the result records, and the group tables from the
  // first one that is not already on the device (a repeated run of the same
  // shape uploads its records alone)
  CK(cudaMemcpyAsync(ctx->d_io, ctx->h_io, (size_t)count * l.off_groups, cudaMemcpyHostToDevice,
                     ctx->stream));
  if (first_fresh != SIZE_MAX)
    CK(cudaMemcpyAsync(ctx->d_io + first_fresh, ctx->h_io + first_fresh, goff - first_fresh,
                       cudaMemcpyHostToDevice, ctx->stream));
  while ((int)ctx->ev_round.size() < count + 1) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ctx->ev_round.push_back(e);
  }
  // Launch order: back to back on one stream; a round kernel that follows
  // another round kernel is launched as a programmatic dependent (it fills
  // SMs as the previous one drains).  Only the largest round of the batch
  // is bracketed by events (an event between two kernels would serialise
  // them): its device time is measured, the others share the remainder by
  // combination count.
  int big = 0;
  for (int i = 1; i < count; ++i)
    if (todo[i].run && todo[i].a.g >= todo[big].a.g) big = i;
  CK(cudaEventRecord(ctx->ev_k0, ctx->stream));
  bool prev_round = false;
  const bool timed = count > 1;
  // the launch holding the largest round is bracketed by events: rounds
  // [big_lo, big_hi)
  int big_lo = big, big_hi = big + 1;
  for (int i = 0; i < count; ++i) {
    if (!todo[i].run) continue;
    // consecutive small K1 rounds of the same depth share one launch, and so
    // do consecutive rounds on the same tensor-core kernel (K5 / K5q: one
    // persistent launch runs them back to back, no launch, prologue or tail
    // between them)
    int f = 1;
    size_t fused_groups = (size_t)todo[i].a.ngroups;
    const int kern = todo[i].shape.kernel;
    const bool tensor = kern == 5 || kern == 8 || kern == 9 || kern == 10;
    while (!hist && !debug && i + f < count && todo[i + f].run &&
           todo[i + f].shape.kernel == kern &&
           ((kern == 1 && f < bz::kK1MaxFused && todo[i + f].shape.depth == todo[i].shape.depth &&
             i + f != big &&
             (fused_groups + todo[i + f].a.ngroups) * sizeof(bz::Group) <=
                 (size_t)bz::kK1FusedGroupBytes) ||
            (tensor && f < bz::kK5MaxFused))) {
      fused_groups += todo[i + f].a.ngroups;
      ++f;
    }
    const bool has_big = timed && i <= big && big < i + f;
    if (has_big) {
      CK(cudaEventRecord(ctx->ev_round[0], ctx->stream));
      prev_round = false;
      big_lo = i;
      big_hi = i + f;
    }
    if (todo[i].seed && !hist) {
      // a threshold kernel (K5q / K5w) with no bound to start from: a
      // sample of the pass lowers it first (k_seed_bound)
      rc = launch_seed(ctx, todo[i].a, gamma_only);
      if (rc) return rc;
      prev_round = false;
    }
    if (ctx->side_pending && (kern >= 3 || todo[i].seed)) {
      // the suffix tables this launch reads were built on the side stream
      CK(cudaEventRecord(ctx->ev_side, ctx->side));
      CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_side, 0));
      ctx->side_pending = false;
    }
    ctx->pdl_next = prev_round && !debug;
    std::vector<RoundArgs> as;
    for (int q = 0; q < f; ++q) as.push_back(todo[i + q].a);
    if (f > 1 && kern == 1)
      rc = launch_fused(ctx, as.data(), f, todo[i].shape.depth);
    else
      rc = launch(ctx, as.data(), f, hist, todo[i].shape);
    ctx->pdl_next = false;
    if (rc) return rc;
    prev_round = true;
    if (has_big) {
      CK(cudaEventRecord(ctx->ev_round[1], ctx->stream));
      prev_round = false;
    }
    i += f - 1;
  }
  if (ctx->side_pending) {  // tables built but not read by this batch: still join
    CK(cudaEventRecord(ctx->ev_side, ctx->side));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_side, 0));
    ctx->side_pending = false;
  }
  CK(cudaEventRecord(ctx->ev_k1, ctx->stream));
  const auto t_launch1 = std::chrono::steady_clock::now();
  // the result records only
  CK(cudaMemcpyAsync(ctx->h_io, ctx->d_io, l.off_groups * (size_t)count,
                     cudaMemcpyDeviceToHost, ctx->stream));
  if (hist)
    CK(cudaMemcpyAsync(ctx->h_hist, ctx->d_hist, sizeof(unsigned long long) * (ctx->n + 1),
                       cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (getenv("BZ_HOST_TIMING")) {
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    fprintf(stderr, "run_batch g0=%d count=%d: plan %.1f us, launches %.1f us, wait %.1f us\n", g0,
            count, us(t_plan0, t_plan1), us(t_plan1, t_launch1),
            us(t_launch1, std::chrono::steady_clock::now()));
  }
  CK(cudaEventElapsedTime(&ctx->last_kernel_ms, ctx->ev_k0, ctx->ev_k1));
  ctx->last_count = hist ? 0 : count;
  ctx->round_ms.assign(count, 0.f);
  if (count == 1) {
    ctx->round_ms[0] = ctx->last_kernel_ms;
  } else {
    // the bracketed launch's time over its rounds, the rest of the batch
    // time over the other rounds, by combination count
    float big_ms = 0.f;
    CK(cudaEventElapsedTime(&big_ms, ctx->ev_round[0], ctx->ev_round[1]));
    double in_big = 0, rest = 0;
    for (int i = 0; i < count; ++i)
      if (todo[i].run) (i >= big_lo && i < big_hi ? in_big : rest) += binom_d(ctx->k, todo[i].a.g);
    for (int i = 0; i < count; ++i) {
      if (!todo[i].run) continue;
      const double share = binom_d(ctx->k, todo[i].a.g);
      if (i >= big_lo && i < big_hi)
        ctx->round_ms[i] = in_big > 0 ? (float)(big_ms * share / in_big) : 0.f;
      else if (rest > 0)
        ctx->round_ms[i] = (float)((ctx->last_kernel_ms - big_ms) * share / rest);
    }
  }
  if (ctrace) {
    // BZ_K4_DEBUG & 32: per-chunk timeline to $BZ_K4_CTRACE (raw int64)
    std::vector<long long> h(1024 * 64 * 4);
    CK(cudaMemcpy(h.data(), ctrace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    const char* path = getenv("BZ_K4_CTRACE");
    if (FILE* f = fopen(path ? path : "bz_ctrace.bin", "wb")) {
      fwrite(h.data(), sizeof(long long), h.size(), f);
      fclose(f);
    }
  }
  if (trace) {
    // 16 timeline slots x 256 tiles (clock64 of block 0) to $BZ_K4_TRACE_OUT
    std::vector<long long> h(16 * 256);
    CK(cudaMemcpy(h.data(), trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    const char* path = getenv("BZ_K4_TRACE_OUT");
    if (FILE* f = fopen(path ? path : "bz_trace.bin", "wb")) {
      fwrite(h.data(), sizeof(long long), h.size(), f);
      fclose(f);
    }
  }
  return BZ_OK;
}

// results of slot i after run_batch
const int* slot_bound(bz_ctx* ctx, int i) {
  const IoSlot l = io_layout(ctx->m, ctx->k);
  return slot_ptr<int>(ctx->h_io, l, i, l.off_bound);
}
const unsigned long long* slot_combos(bz_ctx* ctx, int i) {
  const IoSlot l = io_layout(ctx->m, ctx->k);
  return slot_ptr<unsigned long long>(ctx->h_io, l, i, l.off_combos);
}
const unsigned long long* slot_adds(bz_ctx* ctx, int i) {
  const IoSlot l = io_layout(ctx->m, ctx->k);
  return slot_ptr<unsigned long long>(ctx->h_io, l, i, l.off_adds);
}
const unsigned long long* slot_accs(bz_ctx* ctx, int i) {
  const IoSlot l = io_layout(ctx->m, ctx->k);
  return slot_ptr<unsigned long long>(ctx->h_io, l, i, l.off_accs);
}

}  // namespace

namespace {
template <int W>
int launch_brute(bz_ctx* ctx, const uint32_t* d_rows, int k, unsigned long long nranges,
                 unsigned long long* d_counter, int* d_best) {
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bz::k6_brute<W>, 256, 0));
  const unsigned long long want = (nranges + 255) / 256;
  const long long blocks =
      std::max(1ll, std::min((long long)std::max(per_sm, 1) * ctx->sm_count, (long long)want));
  bz::k6_brute<W><<<(unsigned)blocks, 256, 0, ctx->stream>>>(d_rows, k, nranges, d_counter,
                                                             d_best);
  CK(cudaGetLastError());
  ctx->launches += 1;
  return BZ_OK;
}
}  // namespace

extern "C" {

int bz_abi_version(void) { return BZ_ABI_VERSION; }

int bz_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int bz_create(int device, bz_ctx** out) {
  if (!out) return BZ_ERR_ARGUMENT;
  *out = nullptr;
  bz_ctx* ctx = new bz_ctx();
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0 || device < 0 || device >= n) {
    cudaGetLastError();
    *out = ctx;  // carries the error text
    return fail(ctx, BZ_ERR_NO_DEVICE, "no CUDA device %d (count %d: %s)", device, n,
                e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  }
  ctx->device = device;
  *out = ctx;
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(ctx, BZ_ERR_NO_DEVICE, "device %d is sm_%d%d, this library is built for sm_100a",
                device, prop.major, prop.minor);
  ctx->sm_count = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  CK(cudaEventCreate(&ctx->ev_a));
  CK(cudaEventCreate(&ctx->ev_b));
  CK(cudaEventCreate(&ctx->ev_k0));
  CK(cudaEventCreate(&ctx->ev_k1));
  CK(cudaEventCreateWithFlags(&ctx->ev_load, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ctx->ev_main, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_side, cudaEventDisableTiming));
  // binomial table, saturating at UINT64_MAX
  std::vector<unsigned long long> tab(bz::kBinomDim * bz::kBinomDim);
  for (int p = 0; p < bz::kBinomDim; ++p)
    for (int q = 0; q < bz::kBinomDim; ++q) tab[p * bz::kBinomDim + q] = binom_sat(p, q);
  CK(cudaMalloc(&ctx->d_binom, tab.size() * sizeof(unsigned long long)));
  CK(cudaMemcpy(ctx->d_binom, tab.data(), tab.size() * sizeof(unsigned long long),
                cudaMemcpyHostToDevice));
  CK(cudaMalloc(&ctx->d_hist, sizeof(unsigned long long) * (BZ_MAX_N + 1)));
  CK(cudaMallocHost(&ctx->h_hist, sizeof(unsigned long long) * (BZ_MAX_N + 1)));
  ctx->err.clear();
  return BZ_OK;
}

void bz_destroy(bz_ctx* ctx) {
  if (!ctx) return;
  if (ctx->device >= 0) {
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->d_rows);
    cudaFree(ctx->d_px);
    cudaFree(ctx->d_trip);
    cudaFree(ctx->d_trip4);
    for (int i = 0; i < 3; ++i) cudaFree(ctx->d_lvl[i]);
    cudaFree(ctx->d_binom);
    cudaFree(ctx->d_io);
    cudaFree(ctx->d_hist);
    if (ctx->h_io) cudaFreeHost(ctx->h_io);
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    if (ctx->ev_load) cudaEventDestroy(ctx->ev_load);
    if (ctx->side) {
      cudaStreamSynchronize(ctx->side);
      cudaStreamDestroy(ctx->side);
    }
    if (ctx->ev_main) cudaEventDestroy(ctx->ev_main);
    if (ctx->ev_side) cudaEventDestroy(ctx->ev_side);
    if (ctx->h_hist) cudaFreeHost(ctx->h_hist);
    if (ctx->ev_a) cudaEventDestroy(ctx->ev_a);
    if (ctx->ev_b) cudaEventDestroy(ctx->ev_b);
    if (ctx->gbound_ipc && ctx->d_gbound) cudaIpcCloseMemHandle(ctx->d_gbound);
    cudaFree(ctx->d_gbound_own);
    if (ctx->ev_k0) cudaEventDestroy(ctx->ev_k0);
    for (cudaEvent_t e : ctx->ev_round) cudaEventDestroy(e);
    if (ctx->ev_k1) cudaEventDestroy(ctx->ev_k1);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
  }
  delete ctx;
}

const char* bz_last_error(const bz_ctx* ctx) {
  if (!ctx) return "null context";
  return ctx->err.c_str();
}

int bz_load_gammas(bz_ctx* ctx, const uint64_t* rows, int m, int k, int n) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  if (ctx->device < 0) return fail(ctx, BZ_ERR_NO_DEVICE, "context has no device");
  if (!rows) return fail(ctx, BZ_ERR_ARGUMENT, "rows is NULL");
  if (m < 1 || k < 1 || n < 1)
    return fail(ctx, BZ_ERR_INVALID_DIMENSIONS, "need m, k, n >= 1 (got %d, %d, %d)", m, k, n);
  if (k > BZ_MAX_K) return fail(ctx, BZ_ERR_TOO_LARGE, "k=%d exceeds %d", k, BZ_MAX_K);
  if (n > BZ_MAX_N) return fail(ctx, BZ_ERR_TOO_LARGE, "n=%d exceeds %d", n, BZ_MAX_N);
  CK(cudaSetDevice(ctx->device));
  const int w64 = (n + 63) / 64;
  // validate padding
  for (int j = 0; j < m; ++j)
    for (int r = 0; r < k; ++r) {
      const uint64_t* src = rows + ((size_t)j * k + r) * w64;
      const int keep = n - 64 * (w64 - 1);
      const uint64_t mask = keep >= 64 ? ~0ull : ((1ull << keep) - 1ull);
      if (src[w64 - 1] & ~mask)
        return fail(ctx, BZ_ERR_INVALID_DIMENSIONS,
                    "Gamma %d row %d has bits outside columns 0..%d", j, r, n - 1);
    }
  auto row_of = [&](int j, int r) { return rows + ((size_t)j * k + r) * w64; };
  // Identity-column elision: a Gamma with one unit column per row (every
  // full-rank information set, m/gf2.py:133-199) has exactly one 1 of those
  // columns in each chosen row, so the weight of any g-combination is
  // g + the weight of its other n - k columns.  Those columns are dropped
  // here and the kernels add g back (RoundArgs::elide).  Word-level: set
  // bits are visited with ctz, kept columns gathered by rank.
  std::vector<std::vector<uint64_t>> keep(m, std::vector<uint64_t>(w64, 0ull));
  unsigned long long elide = 0;
  int n_eff = 1;
  std::vector<int> n_stored(m, 0);
  for (int j = 0; j < m; ++j) {
    std::vector<uint64_t>& km = keep[j];
    for (int w = 0; w < w64; ++w) {
      const int bits = std::min(64, n - 64 * w);
      km[w] = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
    }
    bool ok = ctx->elision && m <= 64 && k < n;
    std::vector<int> ones(n, 0);
    for (int r = 0; ok && r < k; ++r)
      for (int w = 0; w < w64; ++w)
        for (uint64_t x = row_of(j, r)[w]; x; x &= x - 1) ++ones[64 * w + __builtin_ctzll(x)];
    std::vector<uint64_t> drop(w64, 0ull);
    for (int r = 0; ok && r < k; ++r) {
      int unit = -1;
      for (int w = 0; w < w64 && unit < 0; ++w)
        for (uint64_t x = row_of(j, r)[w]; x && unit < 0; x &= x - 1) {
          const int c = 64 * w + __builtin_ctzll(x);
          if (ones[c] == 1) unit = c;
        }
      if (unit < 0) ok = false; else drop[unit >> 6] |= 1ull << (unit & 63);
    }
    if (ok) {
      for (int w = 0; w < w64; ++w) km[w] &= ~drop[w];
      elide |= 1ull << j;
    }
    int cnt = 0;
    for (int w = 0; w < w64; ++w) cnt += __builtin_popcountll(km[w]);
    n_eff = std::max(n_eff, cnt);
    n_stored[j] = cnt;
  }
  if (n_eff > BZ_MAX_N_STORED)
    return fail(ctx, BZ_ERR_TOO_LARGE,
                "a Gamma keeps %d columns on the device (limit %d; identity columns of a "
                "systematic Gamma are not stored)", n_eff, BZ_MAX_N_STORED);
  const int w32 = (n_eff + 31) / 32;
  const int wp = bz::padded_words(w32);
  // repack the kept columns to padded 32-bit rows, build prefix-XOR tables
  std::vector<uint32_t> img((size_t)m * k * wp, 0u);
  std::vector<uint32_t> px((size_t)m * (k + 1) * wp, 0u);
  for (int j = 0; j < m; ++j) {
    // kept columns below word w: the gathered index base of word w
    std::vector<int> base(w64 + 1, 0);
    for (int w = 0; w < w64; ++w) base[w + 1] = base[w] + __builtin_popcountll(keep[j][w]);
    for (int r = 0; r < k; ++r) {
      uint32_t* dst = img.data() + ((size_t)j * k + r) * wp;
      for (int w = 0; w < w64; ++w) {
        const uint64_t km = keep[j][w];
        for (uint64_t x = row_of(j, r)[w] & km; x; x &= x - 1) {
          const int b = __builtin_ctzll(x);
          const int i = base[w] + __builtin_popcountll(km & ((1ull << b) - 1ull));
          dst[i >> 5] |= 1u << (i & 31);
        }
      }
    }
    for (int r = 0; r < k; ++r)
      for (int w = 0; w < wp; ++w)
        px[((size_t)j * (k + 1) + r + 1) * wp + w] =
            px[((size_t)j * (k + 1) + r) * wp + w] ^ img[((size_t)j * k + r) * wp + w];
  }
  CK(grow(ctx, (void**)&ctx->d_rows, &ctx->rows_cap, img.size() * 4));
  CK(grow(ctx, (void**)&ctx->d_px, &ctx->px_cap, px.size() * 4));
  // one asynchronous H2D from a pinned staging buffer (no stream
  // synchronisation: the rounds that read the rows follow on the stream;
  // the staging buffer is reused only once the previous upload has landed)
  const size_t stage_bytes = (img.size() + px.size()) * 4;
  if (ctx->ev_load_pending) {
    CK(cudaEventSynchronize(ctx->ev_load));
    ctx->ev_load_pending = false;
  }
  if (stage_bytes > ctx->stage_cap) {
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    ctx->h_stage = nullptr;
    ctx->stage_cap = 0;
    CK(cudaMallocHost(&ctx->h_stage, stage_bytes));
    ctx->stage_cap = stage_bytes;
  }
  std::memcpy(ctx->h_stage, img.data(), img.size() * 4);
  std::memcpy(ctx->h_stage + img.size() * 4, px.data(), px.size() * 4);
  CK(cudaMemcpyAsync(ctx->d_rows, ctx->h_stage, img.size() * 4, cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_px, ctx->h_stage + img.size() * 4, px.size() * 4,
                     cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaEventRecord(ctx->ev_load, ctx->stream));
  ctx->ev_load_pending = true;
  // triple tables (K3, K4) are sized here and built lazily by the first
  // round that needs them
  ctx->trip_built = ctx->trip4_built = false;
  ctx->trip_rows = ctx->trip4_rows = 0;
  for (int i = 0; i < 3; ++i) ctx->lvl_floor[i] = -1;
  if (k >= 4) {
    const size_t n3 = (size_t)k * (k - 1) * (k - 2) / 6;
    ctx->trip_rows = n3 + bz::kTileRows;
    ctx->trip4_rows = (n3 + bz::kUmmaN - 1) / bz::kUmmaN * bz::kUmmaN + bz::kUmmaN;
  }

  ctx->m = m;
  ctx->k = k;
  ctx->n = n;
  ctx->w32 = w32;
  ctx->wp = wp;
  ctx->n_eff = n_eff;
  ctx->n_stored = n_stored;
  ctx->elide_mask = elide;
  return BZ_OK;
}

int bz_round(bz_ctx* ctx, int g, int lower_prev, int upper, int shard, int nshards,
             int32_t* out_min, uint64_t* out_combos) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  if (!out_min || !out_combos) return fail(ctx, BZ_ERR_ARGUMENT, "null output");
  if (ctx->device < 0) return fail(ctx, BZ_ERR_NO_DEVICE, "context has no device");
  CK(cudaSetDevice(ctx->device));
  int rc = run_batch(ctx, g, 1, -1, &lower_prev, upper, shard, nshards, false);
  if (rc) return rc;
  for (int j = 0; j < ctx->m; ++j) {
    out_min[j] = std::min(slot_bound(ctx, 0)[1 + j], upper);
    out_combos[j] = slot_combos(ctx, 0)[j];
  }
  return BZ_OK;
}

int bz_rounds(bz_ctx* ctx, int g0, int count, const int32_t* lower_prev, int upper,
              int shard, int nshards, int32_t* out_min, uint64_t* out_combos) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  if (!out_min || !out_combos || !lower_prev) return fail(ctx, BZ_ERR_ARGUMENT, "null argument");
  if (ctx->device < 0) return fail(ctx, BZ_ERR_NO_DEVICE, "context has no device");
  CK(cudaSetDevice(ctx->device));
  std::vector<int> lp(lower_prev, lower_prev + std::max(count, 0));
  int rc = run_batch(ctx, g0, count, -1, lp.data(), upper, shard, nshards, false);
  if (rc) return rc;
  // round i reports its minima clipped to the U round i-1 ended with (the
  // device chain already starts it there; rounds fused into one launch are
  // clipped here)
  int U = upper;
  for (int i = 0; i < count; ++i) {
    const int Ui = U;
    for (int j = 0; j < ctx->m; ++j) {
      const int v = std::min(slot_bound(ctx, i)[1 + j], Ui);
      out_min[(size_t)i * ctx->m + j] = v;
      out_combos[(size_t)i * ctx->m + j] = slot_combos(ctx, i)[j];
      U = std::min(U, v);
    }
  }
  return BZ_OK;
}

// The Algorithm-1 loop (m/engine.py:204-217) one device call at a time: the
// batch rule and the fold of engine.py run_rounds, natively (see bz.h).
int bz_advance(bz_ctx* ctx, int m_arg, int km_arg, int max_g, int u_rows, int64_t batch_budget,
               bz_loop_state* st, bz_round_record* out, int cap, int* n_out) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  if (!st || !n_out || (!out && cap > 0)) return fail(ctx, BZ_ERR_ARGUMENT, "null argument");
  *n_out = 0;
  if (ctx->device < 0) return fail(ctx, BZ_ERR_NO_DEVICE, "context has no device");
  if (!ctx->d_rows) return fail(ctx, BZ_ERR_STATE, "no Gamma family loaded");
  const int k = ctx->k, m = ctx->m;
  // lower_bound_update (engine.py:97-103)
  auto lower = [&](int gg) { return (m_arg - 1) * (gg + 1) + std::max(0, gg + 1 - k + km_arg); };
  auto settle = [&]() {
    if (!(st->g <= k && st->L < st->U)) st->status = BZ_LOOP_DONE;
    else if (st->g > max_g) st->status = BZ_LOOP_MAX_G;
  };
  settle();
  if (st->status != BZ_LOOP_RUNNING) return BZ_OK;
  if (cap < 1) return fail(ctx, BZ_ERR_ARGUMENT, "no room for a round record");
  CK(cudaSetDevice(ctx->device));
  // the batch: the next rounds whose combinations fit the budget, not past
  // max_g, not past the round where the loop must stop (L(g-1) >= U, and U
  // never exceeds the lightest row once round 1 is in) -- engine.py's rule
  const int g = st->g;
  const int top = std::min(k, max_g);
  const int u_cap = std::min(st->U, u_rows);
  int count = 0;
  double total = 0;
  while (g + count <= top && count < cap && (count == 0 || lower(g + count - 1) < u_cap)) {
    const double c = (double)m * binom_d(k, g + count);
    if (batch_budget > 0 && total + c > (double)batch_budget) break;
    total += c;
    ++count;
  }
  if (batch_budget <= 0 || count < 1) count = 1;
  std::vector<int> lp(count);
  lp[0] = st->L;
  for (int i = 1; i < count; ++i) lp[i] = lower(g + i - 1);
  int rc = run_batch(ctx, g, count, -1, lp.data(), st->U, 0, 1, false);
  if (rc) return rc;
  // fold the rounds in order (engine.py:209-216); rounds past termination
  // are discarded, their counters too
  int n = 0;
  for (int i = 0; i < count; ++i) {
    if (i > 0) {
      settle();
      if (st->status != BZ_LOOP_RUNNING) break;
    }
    const int gi = g + i;
    bz_round_record& r = out[n++];
    r = bz_round_record{};
    int U = st->U;
    for (int j = 0; j < m; ++j) {
      U = std::min(U, slot_bound(ctx, i)[1 + j]);
      r.combinations += slot_combos(ctx, i)[j];
      r.row_additions += slot_adds(ctx, i)[j];
      r.row_accesses += slot_accs(ctx, i)[j];
    }
    r.kernel_ms = i < (int)ctx->round_ms.size() ? ctx->round_ms[i] : 0.f;
    st->U = U;
    st->L = lower(gi);
    st->g_reached = gi;
    st->g = gi + 1;
    r.g = gi;
    r.L = st->L;
    r.U = st->U;
  }
  *n_out = n;
  settle();
  return BZ_OK;
}

int bz_enumerate(bz_ctx* ctx, int gamma, int g, int shard, int nshards, int32_t* out_min,
                 uint64_t* out_combos) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  if (!out_min || !out_combos) return fail(ctx, BZ_ERR_ARGUMENT, "null output");
  if (ctx->device < 0) return fail(ctx, BZ_ERR_NO_DEVICE, "context has no device");
  if (gamma < 0 || gamma >= ctx->m)
    return fail(ctx, BZ_ERR_STATE, "gamma %d not in 0..%d", gamma, ctx->m - 1);
  CK(cudaSetDevice(ctx->device));
  const int zero = 0;
  int rc = run_batch(ctx, g, 1, gamma, &zero, INT32_MAX, shard, nshards, false);
  if (rc) return rc;
  *out_min = slot_bound(ctx, 0)[1 + gamma];
  *out_combos = slot_combos(ctx, 0)[gamma];
  return BZ_OK;
}

int bz_counters(bz_ctx* ctx, int count, uint64_t* out_adds, uint64_t* out_accs) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  if (!out_adds || !out_accs) return fail(ctx, BZ_ERR_ARGUMENT, "null output");
  if (count < 1 || count > ctx->last_count)
    return fail(ctx, BZ_ERR_ARGUMENT, "count %d not in 1..%d (rounds of the last call)", count,
                ctx->last_count);
  for (int i = 0; i < count; ++i)
    for (int j = 0; j < ctx->m; ++j) {
      out_adds[(size_t)i * ctx->m + j] = slot_adds(ctx, i)[j];
      out_accs[(size_t)i * ctx->m + j] = slot_accs(ctx, i)[j];
    }
  return BZ_OK;
}

int bz_histogram(bz_ctx* ctx, int gamma, int g, int shard, int nshards, uint64_t* out_hist,
                 int32_t* out_min, uint64_t* out_combos) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  if (!out_hist || !out_min || !out_combos) return fail(ctx, BZ_ERR_ARGUMENT, "null output");
  if (ctx->device < 0) return fail(ctx, BZ_ERR_NO_DEVICE, "context has no device");
  if (gamma < 0 || gamma >= ctx->m)
    return fail(ctx, BZ_ERR_STATE, "gamma %d not in 0..%d", gamma, ctx->m - 1);
  CK(cudaSetDevice(ctx->device));
  const int zero = 0;
  int rc = run_batch(ctx, g, 1, gamma, &zero, INT32_MAX, shard, nshards, true);
  if (rc) return rc;
  for (int b = 0; b <= ctx->n; ++b) out_hist[b] = ctx->h_hist[b];
  *out_min = slot_bound(ctx, 0)[0];
  *out_combos = slot_combos(ctx, 0)[gamma];
  return BZ_OK;
}


int bz_brute_force(bz_ctx* ctx, const uint64_t* rows, int k, int n, int max_k,
                   int32_t* out_distance, uint64_t* out_codewords) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  if (ctx->device < 0) return fail(ctx, BZ_ERR_NO_DEVICE, "context has no device");
  if (!rows || !out_distance) return fail(ctx, BZ_ERR_ARGUMENT, "null argument");
  if (k < 1 || n < 1) return fail(ctx, BZ_ERR_INVALID_DIMENSIONS, "need k, n >= 1");
  if (n > BZ_MAX_N_STORED)
    return fail(ctx, BZ_ERR_TOO_LARGE, "brute force: n=%d exceeds %d", n, BZ_MAX_N_STORED);
  const int cap = std::min(max_k, bz::kBruteMaxK);
  if (k > cap)
    return fail(ctx, BZ_ERR_TOO_LARGE, "brute force limited to k <= %d (got %d)", cap, k);
  CK(cudaSetDevice(ctx->device));
  const int w64 = (n + 63) / 64, w32 = (n + 31) / 32, wp = bz::padded_words(w32);
  std::vector<uint32_t> img((size_t)k * wp, 0u);
  for (int r = 0; r < k; ++r)
    for (int w = 0; w < w64; ++w) {
      const uint64_t v = rows[(size_t)r * w64 + w];
      if (2 * w < w32) img[(size_t)r * wp + 2 * w] = (uint32_t)v;
      if (2 * w + 1 < w32) img[(size_t)r * wp + 2 * w + 1] = (uint32_t)(v >> 32);
    }
  const size_t bytes = img.size() * 4 + 16;
  unsigned char* d = nullptr;
  CK(cudaMallocAsync((void**)&d, bytes, ctx->stream));
  unsigned long long* d_counter = reinterpret_cast<unsigned long long*>(d);
  int* d_best = reinterpret_cast<int*>(d + 8);
  uint32_t* d_rows = reinterpret_cast<uint32_t*>(d + 16);
  const int init[2] = {0, INT32_MAX};
  CK(cudaMemsetAsync(d_counter, 0, 8, ctx->stream));
  CK(cudaMemcpyAsync(d_best, &init[1], 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(d_rows, img.data(), img.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  const unsigned long long total = 1ull << k;
  const unsigned long long nranges = (total + bz::kBruteSpan - 1) / bz::kBruteSpan;
  CK(cudaEventRecord(ctx->ev_k0, ctx->stream));
  int rc;
  switch (w32) {
    case 1: rc = launch_brute<1>(ctx, d_rows, k, nranges, d_counter, d_best); break;
    case 2: rc = launch_brute<2>(ctx, d_rows, k, nranges, d_counter, d_best); break;
    case 3: rc = launch_brute<3>(ctx, d_rows, k, nranges, d_counter, d_best); break;
    case 4: rc = launch_brute<4>(ctx, d_rows, k, nranges, d_counter, d_best); break;
    case 5: rc = launch_brute<5>(ctx, d_rows, k, nranges, d_counter, d_best); break;
    case 6: rc = launch_brute<6>(ctx, d_rows, k, nranges, d_counter, d_best); break;
    case 7: rc = launch_brute<7>(ctx, d_rows, k, nranges, d_counter, d_best); break;
    default: rc = launch_brute<8>(ctx, d_rows, k, nranges, d_counter, d_best); break;
  }
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev_k1, ctx->stream));
  int best = 0;
  CK(cudaMemcpyAsync(&best, d_best, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaFreeAsync(d, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaEventElapsedTime(&ctx->last_kernel_ms, ctx->ev_k0, ctx->ev_k1));
  *out_distance = best;  // INT32_MAX: every message maps to the zero word
  if (out_codewords) *out_codewords = total - 1;
  return BZ_OK;
}

int bz_reduce_on_columns(uint64_t* rows, int k, int n, const int32_t* cols, int ncols,
                         int32_t* out_pivots, int* out_rank) {
  if (!rows || !out_rank || (ncols > 0 && !cols)) return BZ_ERR_ARGUMENT;
  if (k < 1 || n < 1 || k > 4096 || n > 65536) return BZ_ERR_INVALID_DIMENSIONS;
  const int w = (n + 63) / 64;
  std::vector<uint64_t> tmp(w);
  int top = 0;
  for (int i = 0; i < ncols && top < k; ++i) {
    const int col = cols[i];
    if (col < 0 || col >= n) return BZ_ERR_INVALID_DIMENSIONS;
    const int cw = col >> 6;
    const uint64_t cb = 1ull << (col & 63);
    int hit = -1;
    for (int r = top; r < k; ++r)
      if (rows[(size_t)r * w + cw] & cb) { hit = r; break; }
    if (hit < 0) continue;
    if (hit != top)
      for (int x = 0; x < w; ++x) std::swap(rows[(size_t)hit * w + x], rows[(size_t)top * w + x]);
    // eliminate the pivot column from every other row, branch-free (the
    // data-dependent branch mispredicted on half the rows: this loop was
    // most of the Gamma family's host time)
    const uint64_t* pr = rows + (size_t)top * w;
    const int sh = col & 63;
    if (w <= 8) {
      uint64_t p8[8];
      for (int x = 0; x < w; ++x) p8[x] = pr[x];
      for (int r = 0; r < k; ++r) {
        uint64_t* rr = rows + (size_t)r * w;
        const uint64_t mask = (r == top) ? 0ull : (0ull - ((rr[cw] >> sh) & 1ull));
        for (int x = 0; x < w; ++x) rr[x] ^= p8[x] & mask;
      }
    } else {
      for (int r = 0; r < k; ++r)
        if (r != top && (rows[(size_t)r * w + cw] & cb))
          for (int x = 0; x < w; ++x) rows[(size_t)r * w + x] ^= pr[x];
    }
    if (out_pivots) out_pivots[top] = col;
    ++top;
  }
  *out_rank = top;
  return BZ_OK;
}

int bz_gamma_family(const uint64_t* rows, int k, int n, int m_max, uint64_t* out_rows,
                    int32_t* out_pivots, int32_t* out_ranks, int* out_m) {
  if (!rows || !out_rows || !out_pivots || !out_ranks || !out_m || m_max < 1)
    return BZ_ERR_ARGUMENT;
  if (k < 1 || n < 1 || k > 4096 || n > 65536) return BZ_ERR_INVALID_DIMENSIONS;
  const int w = (n + 63) / 64;
  const size_t img = (size_t)k * w;
  std::vector<uint64_t> cur(rows, rows + img);
  std::vector<char> used(n, 0);
  std::vector<int32_t> free_cols, piv(k);
  int nused = 0, m = 0;
  *out_m = 0;
  while (nused < n) {
    free_cols.clear();
    for (int c = 0; c < n; ++c)
      if (!used[c]) free_cols.push_back(c);
    int rank = 0;
    int rc = bz_reduce_on_columns(cur.data(), k, n, free_cols.data(), (int)free_cols.size(),
                                  piv.data(), &rank);
    if (rc) return rc;
    if (m == 0 && rank < k) {  // G itself is rank deficient
      out_ranks[0] = rank;
      return BZ_OK;
    }
    if (rank == 0) break;
    if (m >= m_max) return BZ_ERR_ARGUMENT;
    std::copy(cur.begin(), cur.end(), out_rows + (size_t)m * img);
    std::copy(piv.begin(), piv.begin() + rank, out_pivots + (size_t)m * k);
    out_ranks[m++] = rank;
    if (rank < k) break;  // the first deficient pass is the remainder Gamma_m
    for (int i = 0; i < rank; ++i) used[piv[i]] = 1;
    nused += rank;
  }
  *out_m = m;
  return BZ_OK;
}

// ---- multi-GPU shared bound mirror
constexpr int kGBoundWords = BZ_MAX_K + 2;  // one word per round g (1..k)

int bz_shared_bound_export(bz_ctx* ctx, void* out_handle) {
  if (!ctx || !out_handle) return BZ_ERR_ARGUMENT;
  if (ctx->device < 0) return fail(ctx, BZ_ERR_NO_DEVICE, "context has no device");
  CK(cudaSetDevice(ctx->device));
  if (!ctx->d_gbound_own) {
    CK(cudaMalloc(&ctx->d_gbound_own, kGBoundWords * sizeof(unsigned long long)));
    // all ones: tag 0xffffffff (older than every run) = empty
    CK(cudaMemset(ctx->d_gbound_own, 0xff, kGBoundWords * sizeof(unsigned long long)));
  }
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, ctx->d_gbound_own));
  std::memcpy(out_handle, &h, sizeof h);
  return BZ_OK;
}

int bz_shared_bound_open(bz_ctx* ctx, const void* handle) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  if (ctx->device < 0) return fail(ctx, BZ_ERR_NO_DEVICE, "context has no device");
  CK(cudaSetDevice(ctx->device));
  if (ctx->gbound_ipc && ctx->d_gbound) {
    cudaIpcCloseMemHandle(ctx->d_gbound);
    ctx->gbound_ipc = false;
  }
  ctx->d_gbound = nullptr;
  if (!handle) {  // the owner: its own array
    if (!ctx->d_gbound_own)
      return fail(ctx, BZ_ERR_STATE, "bz_shared_bound_export first");
    ctx->d_gbound = ctx->d_gbound_own;
    return BZ_OK;
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  void* p = nullptr;
  CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  ctx->d_gbound = static_cast<unsigned long long*>(p);
  ctx->gbound_ipc = true;
  return BZ_OK;
}

int bz_shared_bound_epoch(bz_ctx* ctx, uint32_t epoch) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  ctx->gtag = (unsigned long long)(0xffffffffu - epoch) << 32;
  return BZ_OK;
}

int bz_shared_bound_read(bz_ctx* ctx, int g, int32_t* out) {
  if (!ctx || !out) return BZ_ERR_ARGUMENT;
  if (!ctx->d_gbound) return fail(ctx, BZ_ERR_STATE, "no shared bound mapped");
  if (g < 1 || g >= kGBoundWords) return fail(ctx, BZ_ERR_ARGUMENT, "g=%d out of range", g);
  CK(cudaSetDevice(ctx->device));
  unsigned long long v = 0;
  CK(cudaMemcpy(&v, ctx->d_gbound + g, sizeof v, cudaMemcpyDeviceToHost));
  *out = (v >> 32) == (ctx->gtag >> 32) ? (int32_t)(v & 0xffffffffull) : INT32_MAX;
  return BZ_OK;
}

int bz_shared_bound_close(bz_ctx* ctx) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  if (ctx->device >= 0) cudaSetDevice(ctx->device);
  if (ctx->gbound_ipc && ctx->d_gbound) cudaIpcCloseMemHandle(ctx->d_gbound);
  ctx->gbound_ipc = false;
  ctx->d_gbound = nullptr;
  return BZ_OK;
}

int bz_set_elision(bz_ctx* ctx, int on) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  ctx->elision = on ? 1 : 0;
  return BZ_OK;
}

int bz_set_early_exit(bz_ctx* ctx, int on) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  ctx->early_exit = on ? 1 : 0;
  return BZ_OK;
}

int bz_elided(bz_ctx* ctx, uint64_t* out_mask) {
  if (!ctx || !out_mask) return BZ_ERR_ARGUMENT;
  *out_mask = ctx->elide_mask;
  return BZ_OK;
}

int bz_set_engine(bz_ctx* ctx, int engine) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  if (engine < BZ_ENGINE_AUTO || engine > BZ_ENGINE_MXF4F)
    return fail(ctx, BZ_ERR_ARGUMENT, "unknown engine %d", engine);
  if (!BZ_LEGACY_KERNELS && (engine == BZ_ENGINE_IMMA || engine == BZ_ENGINE_UMMA ||
                             engine == BZ_ENGINE_MXF4P || engine == BZ_ENGINE_MXF4T))
    return fail(ctx, BZ_ERR_ARGUMENT,
                "engine %d is a comparison kernel not built into this library "
                "(rebuild with -DBZ_LEGACY_KERNELS=1)", engine);
  ctx->engine = engine;
  return BZ_OK;
}

int bz_plan(int m, int k, int g, int engine, int nshards, int64_t* out, int cap,
            int* out_ngroups, uint64_t* out_nchunks) {
  if (!out_ngroups || !out_nchunks) return BZ_ERR_ARGUMENT;
  if (m < 1 || k < 1) return BZ_ERR_INVALID_DIMENSIONS;
  if (k > BZ_MAX_K) return BZ_ERR_TOO_LARGE;
  if (g < 1 || g > k) return BZ_ERR_INVALID_ARITY;
  if (binom_sat(k, g) >= (1ull << 62)) return BZ_ERR_TOO_LARGE;
  std::vector<Group> gs;
  unsigned long long nchunks = 0;
  if (engine < BZ_ENGINE_AUTO || engine > BZ_ENGINE_MXF4F) return BZ_ERR_ARGUMENT;
  if (nshards < 1) return BZ_ERR_ARGUMENT;
  int rc = build_plan(nullptr, m, k, g, -1, pass_shape(engine, g, false), nshards, gs, &nchunks);
  if (rc) return rc;
  *out_ngroups = (int)gs.size();
  *out_nchunks = nchunks;
  if (out) {
    if ((int)gs.size() > cap) return BZ_ERR_ARGUMENT;
    for (size_t i = 0; i < gs.size(); ++i) {
      int64_t* o = out + (size_t)kPlanCols * i;
      o[0] = (int64_t)gs[i].chunk_begin;
      o[1] = (int64_t)gs[i].nprefix;
      o[2] = gs[i].gamma;
      o[3] = gs[i].ell;
      o[4] = gs[i].ppl;
      o[5] = (int64_t)gs[i].nprefix * (int64_t)gs[i].slice;
      o[6] = gs[i].depth;
      o[7] = gs[i].lanes;
      o[8] = gs[i].depth >= 3 ? (int64_t)gs[i].tpc * gs[i].tile_rows : 0;
      o[9] = gs[i].ntb;
      o[10] = gs[i].sfloor;
      o[11] = gs[i].sl;
    }
  }
  return BZ_OK;
}

int bz_timer_start(bz_ctx* ctx) {
  if (!ctx) return BZ_ERR_ARGUMENT;
  if (ctx->device < 0) return fail(ctx, BZ_ERR_NO_DEVICE, "context has no device");
  CK(cudaSetDevice(ctx->device));
  CK(cudaEventRecord(ctx->ev_a, ctx->stream));
  return BZ_OK;
}

int bz_timer_stop(bz_ctx* ctx, float* ms) {
  if (!ctx || !ms) return BZ_ERR_ARGUMENT;
  if (ctx->device < 0) return fail(ctx, BZ_ERR_NO_DEVICE, "context has no device");
  CK(cudaSetDevice(ctx->device));
  CK(cudaEventRecord(ctx->ev_b, ctx->stream));
  CK(cudaEventSynchronize(ctx->ev_b));
  CK(cudaEventElapsedTime(ms, ctx->ev_a, ctx->ev_b));
  return BZ_OK;
}

int bz_round_ms(bz_ctx* ctx, float* out_ms, int count) {
  if (!ctx || !out_ms || count < 0) return BZ_ERR_ARGUMENT;
  if (count > (int)ctx->round_ms.size())
    return fail(ctx, BZ_ERR_ARGUMENT, "%d rounds requested, last call ran %zu", count,
                ctx->round_ms.size());
  for (int i = 0; i < count; ++i) out_ms[i] = ctx->round_ms[i];
  return BZ_OK;
}

int bz_last_kernel_ms(bz_ctx* ctx, float* ms) {
  if (!ctx || !ms) return BZ_ERR_ARGUMENT;
  *ms = ctx->last_kernel_ms;
  return BZ_OK;
}

int bz_launch_count(bz_ctx* ctx, uint64_t* out) {
  if (!ctx || !out) return BZ_ERR_ARGUMENT;
  *out = ctx->launches;
  return BZ_OK;
}

// Host check of the K5q offset encoding (no device needed): every A offset
// block the producer can emit, dotted with the table's offset block, must
// give back its integer exactly.  Walks every (prefix stored weight wt,
// bound) pair the producer can see -- wt in [0, 128], the Gamma's bound
// less its weight offset in [-4, 128] (run_batch caps it at the stored
// columns) -- through the kernel's own
// k5q_threshold / pad_chunk, and checks thr in [1, 128], x in [0, 238],
// dot(pad_chunk(x, 0)) = x and dot(pad_chunk(x, 128)) = x + 128 (block 1
// of the second chunk: the 2^23 offset at scale 2^16).  Returns the number
// of failures; the first failing (wt, rel) goes to out_bad[0..1].
static double e2m1_value(uint32_t nib) {
  static const double mag[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
  return (nib & 8u) ? -mag[nib & 7u] : mag[nib & 7u];
}
static double e2m1_dot16(uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
  double s = 0;
  for (int q = 0; q < 8; ++q) {
    s += e2m1_value((a0 >> (4 * q)) & 0xFu) * e2m1_value((b0 >> (4 * q)) & 0xFu);
    s += e2m1_value((a1 >> (4 * q)) & 0xFu) * e2m1_value((b1 >> (4 * q)) & 0xFu);
  }
  return s;
}

int bz_k5q_selftest(int32_t* out_bad) {
  const uint4 tb = bz::k5_table_offset_chunk();
  int bad = 0;
  auto note = [&](int wt, int rel) {
    if (!bad++ && out_bad) {
      out_bad[0] = wt;
      out_bad[1] = rel;
    }
  };
  for (int T = 0; T <= bz::kQMaxSpan + 128; ++T) {
    const unsigned long long b = bz::e2m1_block(T);
    if (e2m1_dot16((uint32_t)b, (uint32_t)(b >> 32), tb.x, tb.y) != (double)T) note(-1, T);
  }
  for (int wt = 0; wt <= 128; ++wt)
    for (int rel = -4; rel <= 128; ++rel) {
      const int thr = bz::k5q_threshold(wt, rel);
      const int x = wt + 128 - thr;
      // exactness: every stored weight below rel must be flagged (w < thr),
      // and every field w + 128 - thr of a stored weight w in [0, 128] must
      // stay a byte
      const bool range_ok = thr >= 1 && thr <= 128 && x >= 0 && x <= bz::kQMaxSpan + 128 &&
                            thr >= rel && 128 + 128 - thr <= 255;
      const uint4 pa = bz::pad_chunk(x, 0), pb = bz::pad_chunk(x, 128);
      const bool enc_ok = e2m1_dot16(pa.x, pa.y, tb.x, tb.y) == (double)x &&
                          e2m1_dot16(pa.z, pa.w, tb.z, tb.w) == 0.0 &&
                          e2m1_dot16(pb.x, pb.y, tb.x, tb.y) == (double)x &&
                          e2m1_dot16(pb.z, pb.w, tb.z, tb.w) == 128.0;
      if (!range_ok || !enc_ok) note(wt, rel);
    }
  // K5w: R = wt - thr against the offset pattern, the constant chunks, and
  // the 11-bit field range x = w + 1024 - thr for stored weights 0..256
  for (int R = -bz::kWMaxSpan; R <= bz::kWMaxSpan; ++R) {
    const uint4 c = bz::k5w_r_chunk(R);
    if (e2m1_dot16(c.x, c.y, tb.x, tb.y) + e2m1_dot16(c.z, c.w, tb.z, tb.w) != (double)R)
      note(-2, R);
  }
  const uint4 ca = bz::k5w_const_chunk(0), cb = bz::k5w_const_chunk(1);
  if (e2m1_dot16(ca.x, ca.y, 0x22u, 0u) != 5.0 || e2m1_dot16(cb.x, cb.y, 0x22u, 0u) != 1.0)
    note(-3, 0);
  static_assert(5ll * (1ll << 21) + (1ll << 10) == (1ll << 23) + 1024 + 2048ll * 1024,
                "K5w offset constants");
  for (int wt = 0; wt <= 256; ++wt)
    for (int rel = -4; rel <= 400; ++rel) {
      const int thr = bz::k5w_threshold(wt, rel);
      const bool ok = thr >= 1 && thr >= std::min(rel, 257) && wt - thr >= -bz::kWMaxSpan &&
                      wt - thr <= bz::kWMaxSpan && 0 + 1024 - thr >= 0 && 256 + 1024 - thr <= 2047;
      if (!ok) note(wt, 1000 + rel);
    }
  return bad;
}

int bz_measure_int_peaks(bz_ctx* ctx, int w_words, double* out) {
  if (!ctx || !out) return BZ_ERR_ARGUMENT;
  if (ctx->device < 0) return fail(ctx, BZ_ERR_NO_DEVICE, "context has no device");
  if (w_words < 1 || w_words > 8) return fail(ctx, BZ_ERR_ARGUMENT, "w_words=%d", w_words);
  CK(cudaSetDevice(ctx->device));
  const int threads = 256, per_sm = 4;  // 32 warps/SM, one wave
  const int blocks = ctx->sm_count * per_sm;
  uint32_t* d_out = nullptr;
  long long* d_clk = nullptr;
  CK(cudaMalloc(&d_out, sizeof(uint32_t) * blocks * threads));
  CK(cudaMalloc(&d_clk, sizeof(long long) * blocks));
  std::vector<long long> clk(blocks);
  auto run = [&](int which, int iters, double* ops_per_s, double* ops_per_clk_sm,
                 double* mhz) -> int {
    for (int rep = 0; rep < 2; ++rep) {  // first pass warms up clocks
      CK(cudaEventRecord(ctx->ev_a, ctx->stream));
      if (which == 3)
        bz::peak_imma<<<blocks, threads, 0, ctx->stream>>>(reinterpret_cast<int*>(d_out), 9u,
                                                           iters, d_clk);
      else if (which == 0)
        bz::peak_popc<<<blocks, threads, 0, ctx->stream>>>(d_out, 12345u, iters, d_clk);
      else if (which == 1)
        bz::peak_lop3<<<blocks, threads, 0, ctx->stream>>>(d_out, 12345u, iters, d_clk);
      else {
        int* o = reinterpret_cast<int*>(d_out);
        switch (w_words) {
          case 1: bz::peak_codeword<1><<<blocks, threads, 0, ctx->stream>>>(o, 7u, iters, d_clk); break;
          case 2: bz::peak_codeword<2><<<blocks, threads, 0, ctx->stream>>>(o, 7u, iters, d_clk); break;
          case 3: bz::peak_codeword<3><<<blocks, threads, 0, ctx->stream>>>(o, 7u, iters, d_clk); break;
          case 4: bz::peak_codeword<4><<<blocks, threads, 0, ctx->stream>>>(o, 7u, iters, d_clk); break;
          case 5: bz::peak_codeword<5><<<blocks, threads, 0, ctx->stream>>>(o, 7u, iters, d_clk); break;
          case 6: bz::peak_codeword<6><<<blocks, threads, 0, ctx->stream>>>(o, 7u, iters, d_clk); break;
          case 7: bz::peak_codeword<7><<<blocks, threads, 0, ctx->stream>>>(o, 7u, iters, d_clk); break;
          default: bz::peak_codeword<8><<<blocks, threads, 0, ctx->stream>>>(o, 7u, iters, d_clk); break;
        }
      }
      CK(cudaGetLastError());
      CK(cudaEventRecord(ctx->ev_b, ctx->stream));
      ctx->launches += 1;
      CK(cudaEventSynchronize(ctx->ev_b));
    }
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev_a, ctx->ev_b));
    CK(cudaMemcpy(clk.data(), d_clk, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
    double max_clk = 0;
    for (long long c : clk) max_clk = std::max(max_clk, (double)c);
    // ops per thread: codewords (2), MACs (3: 4 chains x 16*8*32 MACs per
    // warp-level MMA = 128 per lane), or single instructions (0, 1)
    const double per_thread = which == 2 ? 4.0 * iters
                            : which == 3 ? 4.0 * 128.0 * iters : 128.0 * iters;
    const double total = per_thread * threads * blocks;
    *ops_per_s = total / (ms * 1e-3);
    // per clock per SM: blocks resident concurrently (per_sm per SM)
    *ops_per_clk_sm = total / ((double)ctx->sm_count * max_clk);
    *mhz = max_clk / (ms * 1e-3) / 1e6;
    return BZ_OK;
  };
  // tcgen05 kind::i8 M=128 x N=256 x K=32 (f4 = false) or kind::mxf4
  // M=128 x N=240 x K=64 (f4 = true) from shared memory, one CTA per SM
  auto run_umma = [&](bool f4, double* macs_per_s, double* macs_per_clk_sm) -> int {
    const int iters = 20000;
    const size_t smem = 128 * 32 + 256 * 32 + 1024;
    if (f4)
      CK(cudaFuncSetAttribute(bz::peak_umma_mxf4, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem));
    else
      CK(cudaFuncSetAttribute(bz::peak_umma_i8<256>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaEventRecord(ctx->ev_a, ctx->stream));
      if (f4)
        bz::peak_umma_mxf4<<<ctx->sm_count, 128, smem, ctx->stream>>>(iters, d_clk);
      else
        bz::peak_umma_i8<256><<<ctx->sm_count, 128, smem, ctx->stream>>>(iters, d_clk);
      CK(cudaGetLastError());
      CK(cudaEventRecord(ctx->ev_b, ctx->stream));
      ctx->launches += 1;
      CK(cudaEventSynchronize(ctx->ev_b));
    }
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev_a, ctx->ev_b));
    CK(cudaMemcpy(clk.data(), d_clk, sizeof(long long) * ctx->sm_count, cudaMemcpyDeviceToHost));
    double max_clk = 0;
    for (int i = 0; i < ctx->sm_count; ++i) max_clk = std::max(max_clk, (double)clk[i]);
    const double per_mma = f4 ? 128.0 * bz::kUmmaN4 * 64.0 : 128.0 * 256.0 * 32.0;
    const double macs = (double)iters * per_mma * ctx->sm_count;
    *macs_per_s = macs / (ms * 1e-3);
    *macs_per_clk_sm = macs / ((double)ctx->sm_count * max_clk);
    return BZ_OK;
  };
  double umma_s = 0, umma_clk = 0, mxf4_s = 0, mxf4_clk = 0;
  double popc_s, popc_clk, lop_s, lop_clk, cw_s, cw_clk, mma_s, mma_clk, mhz0, mhz1, mhz2, mhz3;
  int rc = run(0, 2048, &popc_s, &popc_clk, &mhz0);
  if (!rc) rc = run(1, 2048, &lop_s, &lop_clk, &mhz1);
  if (!rc) rc = run(2, 16384, &cw_s, &cw_clk, &mhz2);
  if (!rc) rc = run(3, 4096, &mma_s, &mma_clk, &mhz3);
  if (!rc) rc = run_umma(false, &umma_s, &umma_clk);
  if (!rc) rc = run_umma(true, &mxf4_s, &mxf4_clk);
  cudaFree(d_out);
  cudaFree(d_clk);
  if (rc) return rc;
  out[0] = popc_s;
  out[1] = lop_s;
  out[2] = mhz0;
  out[3] = ctx->sm_count;
  out[4] = popc_clk;
  out[5] = lop_clk;
  out[6] = cw_s;
  out[7] = cw_clk;
  out[8] = mma_s;
  out[9] = mma_clk;
  out[10] = umma_s;
  out[11] = umma_clk;
  out[12] = mxf4_s;
  out[13] = mxf4_clk;
  return BZ_OK;
}

}  // extern "C"
