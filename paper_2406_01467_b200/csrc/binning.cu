// binning.cu — stage 2 (K2) of the RaDe-GS rasterizer, sm_100a, hand-written (no library sort).
//
// The depth sort of PAPER:422 per tile, as a two-stage stable LSD radix sort whose result is
// bit-identical to one stable sort of 64-bit keys (tile << 32 | float_bits(z_c)) over the
// (Gaussian, tile) pairs emitted in id order (reading S7):
//
//   K2h  histograms: one pass over the N depth keys (id order) builds the four 8-bit digit
//        histograms of the visible keys and two difference arrays over the tile columns and
//        rows — a rect [x0, x1) × [y0, y1) adds h = y1 − y0 at x0 and −h at x1 (and w = x1 − x0
//        at y0, −w at y1), so their prefix sums are the number of duplicates per tile column
//        and per tile row: the digit histograms of every tile pass, without the duplicates
//   K2a  depth sort: 4 onesweep passes (8-bit digits) of (float_bits(z_c), id). The first pass
//        reads the N keys in id order and keeps only the visible ones (culled keys are
//        0xFFFFFFFF and are never read downstream), so passes 2-4 move n_vis pairs. Order
//        (z_c, id): z_c > znear > 0, so the IEEE bit pattern orders like the value
//   K2b  inclusive scan of tiles_touched gathered in that order → offsets (single pass,
//        decoupled look-back)
//   K2c  duplicate + first tile pass, fused: each 4096-output block emits (tile, id) for its
//        outputs (load-balanced over outputs, as K2's generator) and ranks them by the first
//        tile digit right away, so the unsorted duplicates never reach HBM
//   K2d  remaining tile passes: the tile key is packed as (ty << 16 | tx) and sorted tx digits
//        first, then ty digits — the same order as ty·tiles_x + tx, so within a tile the
//        (z_c, id) order of K2a is preserved; the last pass writes ty·tiles_x + tx. At 8×8
//        tiles up to 2048×2048 px this is 2 passes (tx, ty ≤ 256)
//   K2e  ranges[tile] = [first, last) in the sorted list
//
// Every onesweep pass: 512 threads × 8 items per block (4096), items warp-striped so a
// warp ranks them stably (8 ballots per item); per-warp digit counters → warp offsets →
// block-local sorted layout in shared memory; the block's per-digit counts published to and
// prefixed by a decoupled look-back over the blocks (one thread per digit, a window of
// predecessors per round trip; status words carry an epoch tag, so no zeroing between
// passes); then coalesced runs per digit to HBM. A pass is a chain of dependent L2/HBM round
// trips per block (items, look-back, scatter), so everything a block can know beforehand is
// precomputed: the digit bases of every pass (the last K2h block scans the histograms) and,
// for K2c, the first Gaussian of every output block (written by K2b). Integer work: checked
// bit-exactly against the oracle's global (z_key, id) order restricted per tile and a CPU
// stable sort.
#include "rade_internal.cuh"

#include <atomic>
#include <mutex>

namespace rade {
namespace {

#ifndef RD_SORT_THREADS
#define RD_SORT_THREADS 512
#endif
#ifndef RD_RANK_MATCH
#define RD_RANK_MATCH 0  // 1: __match_any_sync ranking instead of the 8 ballots
#endif
constexpr int kST = RD_SORT_THREADS;  // threads per sort block
constexpr int kSI = 8;            // items per thread
constexpr int kSTile = kST * kSI; // items per block
constexpr int kRadix = 256;
constexpr int kMaxTileAxis = 2048;  // difference-array entries per axis (tiles per axis ≤ 2047)
#ifndef RD_LOOKWIN
#define RD_LOOKWIN 8
#endif
constexpr int kLookWin = RD_LOOKWIN;  // look-back predecessors read per round trip
#ifndef RD_SORT_MINB
#define RD_SORT_MINB (1024 / RD_SORT_THREADS)  // ≤ 64 registers: 32 warps per SM
#endif
#ifndef RD_HIST_BPS
#define RD_HIST_BPS 2   // K2h blocks per SM (each flushes its histograms with global atomics)
#endif

__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// status word: (tag << 32) | value, tag = 4·epoch + 1 (block aggregate) or + 2 (inclusive
// prefix); any tag from an earlier epoch is < 4·epoch, i.e. "not yet published"
__device__ __forceinline__ unsigned long long pack_status(uint32_t epoch, uint32_t flag, uint32_t v) {
  return ((unsigned long long)(4u * epoch + flag) << 32) | v;
}
// Exclusive prefix of `mine` over the blocks before b for one counter: publishes the
// aggregate, walks back summing aggregates until an inclusive prefix, publishes the inclusive.
__device__ __forceinline__ uint32_t lookback(unsigned long long* status, int stride, int b, uint32_t epoch,
                                             uint32_t mine) {
  if (b == 0) {
    st_status(status, pack_status(epoch, 2u, mine));
    return 0u;
  }
  st_status(status + (size_t)b * stride, pack_status(epoch, 1u, mine));
  const uint32_t agg = 4u * epoch + 1u, inc = 4u * epoch + 2u;
  uint32_t excl = 0u;
  // a window of kLookWin predecessors per round trip (independent loads; across the block's
  // digit threads each row is one contiguous 2-KB read): blocks that start together walk back
  // ~b/2 predecessors before they meet an inclusive prefix, so one load per step would make
  // the first wave's latency hundreds of L2 round trips
  int p = b - 1;
  for (;;) {
    unsigned long long s[kLookWin];
#pragma unroll
    for (int k = 0; k < kLookWin; ++k) s[k] = p - k >= 0 ? ld_status(status + (size_t)(p - k) * stride) : 0ull;
    int used = 0;
    bool done = false;
#pragma unroll
    for (int k = 0; k < kLookWin; ++k) {
      if (!done && used == k) {
        const uint32_t tag = (uint32_t)(s[k] >> 32);
        if (tag >= agg) {  // published (block 0 always publishes an inclusive prefix)
          excl += (uint32_t)s[k];
          done = tag == inc;
          ++used;
        }
      }
    }
    if (done) break;
    p -= used;  // a not-yet-published entry: reload the window from it
  }
  st_status(status + (size_t)b * stride, pack_status(epoch, 2u, excl + mine));
  return excl;
}

// The same for a single counter, walked by a whole warp (all 32 lanes call it): lane i reads
// predecessor b − 1 − i, so one round trip covers 32 blocks (a single-word scan's blocks are
// all resident at once and would otherwise walk ~b/2 predecessors 8 per round trip). Returns
// the exclusive prefix on every lane.
__device__ __forceinline__ uint32_t lookback_warp(unsigned long long* status, int b, uint32_t epoch,
                                                  uint32_t mine) {
  const int lane = (int)(threadIdx.x & 31);
  if (b == 0) {
    if (lane == 0) st_status(status, pack_status(epoch, 2u, mine));
    return 0u;
  }
  if (lane == 0) st_status(status + b, pack_status(epoch, 1u, mine));
  const uint32_t agg = 4u * epoch + 1u, inc = 4u * epoch + 2u;
  uint32_t excl = 0u;
  int p = b - 1;
  for (;;) {
    const int q = p - lane;
    const unsigned long long st = q >= 0 ? ld_status(status + q) : 0ull;
    const uint32_t tag = (uint32_t)(st >> 32);
    const bool ready = q < 0 || tag >= agg, is_inc = q >= 0 && tag == inc;
    const unsigned nr = __ballot_sync(0xffffffffu, !ready), ic = __ballot_sync(0xffffffffu, is_inc);
    const int first_nr = nr ? __ffs(nr) - 1 : 32, first_inc = ic ? __ffs(ic) - 1 : 32;
    if (first_inc < first_nr) {  // lanes 0..first_inc: aggregates then an inclusive prefix
      excl += __reduce_add_sync(0xffffffffu, lane <= first_inc ? (uint32_t)st : 0u);
      break;
    }
    excl += __reduce_add_sync(0xffffffffu, lane < first_nr ? (uint32_t)st : 0u);  // the ready aggregates
    p -= first_nr;  // restart at the first one not yet published
  }
  if (lane == 0) st_status(status + b, pack_status(epoch, 2u, excl + mine));
  return excl;
}

// Exclusive scan over the block's NT threads (one value each); *total = the sum.
template <int NT = kST>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* s_warp, uint32_t* total) {
  const int lane = (int)(threadIdx.x & 31), warp = (int)(threadIdx.x >> 5);
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  uint32_t wpre = 0u, tot = 0u;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) {
    const uint32_t v = s_warp[w];
    wpre += w < warp ? v : 0u;
    tot += v;
  }
  *total = tot;
  __syncthreads();  // s_warp reusable
  return wpre + inc - x;
}

// The tile passes on the packed key (ty << 16 | tx): tx low digit [, tx high digit], ty low
// digit [, ty high digit] — 8-bit digits of one axis each, so their histograms follow from the
// axis difference arrays.
struct TilePass {
  int axis;    // 0: tx, 1: ty
  int dshift;  // digit = (coordinate >> dshift) & 255
};
__host__ __device__ __forceinline__ int tile_pass_list(int tiles_x, int tiles_y, TilePass* tp) {
  int np = 0;
  tp[np++] = TilePass{0, 0};
  if (tiles_x > 256) tp[np++] = TilePass{0, 8};
  tp[np++] = TilePass{1, 0};
  if (tiles_y > 256) tp[np++] = TilePass{1, 8};
  return np;
}
constexpr int kBaseStride = kRadix + 1;  // bases of one pass: 256 exclusive digit starts + the total

// ------------------------------------------------------------------------------- K2h
// Depth digit histograms of the visible keys (digits aggregated per warp with
// __match_any_sync: the high digits of nearby depths coincide) and the tile difference arrays;
// the last block to finish turns them into the digit bases of every pass (bases[pass][257]:
// depth passes 0-3, then the tile passes).
constexpr int kHistThreads = 512;
__global__ void __launch_bounds__(kHistThreads) k_bin_hist(int64_t n, const uint32_t* __restrict__ dkey,
                                                           const uint2* __restrict__ rect, int tiles_x, int tiles_y,
                                                           uint32_t* __restrict__ hist, int* __restrict__ diff_x,
                                                           int* __restrict__ diff_y, uint32_t* __restrict__ cnt,
                                                           uint32_t* __restrict__ bases,
                                                           volatile uint32_t* __restrict__ host_counts) {
  uint32_t* done = cnt + 3;
  __shared__ uint32_t sh[4][kRadix];
  __shared__ int sx[kMaxTileAxis], sy[kMaxTileAxis];
  __shared__ uint32_t s_warp[kHistThreads / 32];
  __shared__ uint32_t s_bins[kRadix];
  __shared__ bool s_last;
  __shared__ uint32_t s_m;
  const int tid = (int)threadIdx.x;
  if (tid == 0) s_m = 0u;
  for (int k = tid; k < 4 * kRadix; k += kHistThreads) (&sh[0][0])[k] = 0u;
  for (int k = tid; k < kMaxTileAxis; k += kHistThreads) sx[k] = sy[k] = 0;
  __syncthreads();
  const int lane = tid & 31;
  uint32_t mdup = 0u;  // this thread's duplicates (tiles touched)
  const int64_t stride = (int64_t)gridDim.x * kHistThreads;
  const int64_t rounds = (n + stride - 1) / stride;  // warp-uniform trip count (match_any below)
#ifndef RD_HIST_U
#define RD_HIST_U 4  // rounds whose key and rect loads are issued together (one round trip per U)
#endif
  for (int64_t r0 = 0; r0 < rounds; r0 += RD_HIST_U) {
    uint32_t kk[RD_HIST_U];
    uint2 qq[RD_HIST_U];
#pragma unroll
    for (int u = 0; u < RD_HIST_U; ++u) {  // loads first (rect unconditionally: no key → rect chain)
      const int64_t i = (r0 + u) * stride + (int64_t)blockIdx.x * kHistThreads + tid;
      kk[u] = i < n ? dkey[i] : 0xffffffffu;
      qq[u] = i < n ? rect[i] : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < RD_HIST_U; ++u) {
    if (r0 + u >= rounds) break;  // warp-uniform
    const uint32_t k = kk[u];
    const bool vis = k != 0xffffffffu;
    const uint2 q = qq[u];
    if (vis) {  // the low digits of nearby depths differ: plain shared atomics
      atomicAdd(&sh[0][k & 255u], 1u);
      atomicAdd(&sh[1][(k >> 8) & 255u], 1u);
    }
#pragma unroll
    for (int p = 2; p < 4; ++p) {  // the high ones mostly coincide: one atomic per distinct digit
      const uint32_t d = vis ? (k >> (8 * p)) & 255u : 256u;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      if (vis && (peers & ((1u << lane) - 1u)) == 0u) atomicAdd(&sh[p][d], (uint32_t)__popc(peers));
    }
    if (vis) {
      const int x0 = (int)(q.x & 0xffffu), y0 = (int)(q.x >> 16), x1 = (int)(q.y & 0xffffu), y1 = (int)(q.y >> 16);
      RD_CHECK(x0 < x1 && x1 <= tiles_x && y0 < y1 && y1 <= tiles_y);
      atomicAdd(&sx[x0], y1 - y0);
      atomicSub(&sx[x1], y1 - y0);
      atomicAdd(&sy[y0], x1 - x0);
      atomicSub(&sy[y1], x1 - x0);
      mdup += (uint32_t)((x1 - x0) * (y1 - y0));
    }
    }
  }
  mdup = __reduce_add_sync(0xffffffffu, mdup);
  if (lane == 0 && mdup) atomicAdd(&s_m, mdup);
  __syncthreads();
  if (tid == 0 && s_m) atomicAdd(cnt + 2, s_m);  // M
  for (int k = tid; k < 4 * kRadix; k += kHistThreads) {
    const uint32_t v = (&sh[0][0])[k];
    if (v) atomicAdd(hist + k, v);
  }
  for (int k = tid; k <= tiles_x; k += kHistThreads)
    if (sx[k]) atomicAdd(diff_x + k, sx[k]);
  for (int k = tid; k <= tiles_y; k += kHistThreads)
    if (sy[k]) atomicAdd(diff_y + k, sy[k]);

  // the last block: digit bases of every pass
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) {  // K1's visible / big counts and M, to mapped pinned host memory (the host
    host_counts[0] = __ldcg(cnt);  // reads them once this kernel's completion event fires)
    host_counts[1] = __ldcg(cnt + 1);
    host_counts[2] = __ldcg(cnt + 2);
  }
  uint32_t tot;
  for (int p = 0; p < 4; ++p) {
    const uint32_t c = tid < kRadix ? __ldcg(hist + kRadix * p + tid) : 0u;
    const uint32_t e = block_excl_scan<kHistThreads>(c, s_warp, &tot);
    if (tid < kRadix) bases[kBaseStride * p + tid] = e;
    if (tid == 0) bases[kBaseStride * p + kRadix] = tot;
  }
  // per-axis duplicate counts (prefix sums of the difference arrays) into sx / sy: thread t owns
  // entries [4t, 4t + 4) of the ≤ 2048
  for (int axis = 0; axis < 2; ++axis) {
    const int len = axis == 0 ? tiles_x : tiles_y;
    const int* diff = axis == 0 ? diff_x : diff_y;
    int* h = axis == 0 ? sx : sy;
    int v[4], sum = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int e = 4 * tid + j;
      v[j] = e < len ? __ldcg(diff + e) : 0;
      sum += v[j];
    }
    int run = (int)block_excl_scan<kHistThreads>((uint32_t)sum, s_warp, &tot);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      run += v[j];
      h[4 * tid + j] = 4 * tid + j < len ? run : 0;
    }
  }
  __syncthreads();
  TilePass tp[4];
  const int np = tile_pass_list(tiles_x, tiles_y, tp);
  for (int p = 0; p < np; ++p) {
    if (tid < kRadix) s_bins[tid] = 0u;
    __syncthreads();
    const int* h = tp[p].axis == 0 ? sx : sy;
    const int len = tp[p].axis == 0 ? tiles_x : tiles_y;
    for (int e = tid; e < len; e += kHistThreads)
      if (h[e] > 0) atomicAdd(&s_bins[(e >> tp[p].dshift) & 255], (uint32_t)h[e]);
    __syncthreads();
    const uint32_t c = tid < kRadix ? s_bins[tid] : 0u;
    const uint32_t e = block_excl_scan<kHistThreads>(c, s_warp, &tot);
    if (tid < kRadix) bases[kBaseStride * (4 + p) + tid] = e;
    if (tid == 0) bases[kBaseStride * (4 + p) + kRadix] = tot;
  }
  if (tid == 0) *done = 0u;  // for the next view
}

// ------------------------------------------------------------------------------- onesweep
enum PassMode { kDepthFirst = 0, kDepth = 1, kTileGen = 2, kTile = 3 };

struct PassArgs {
  const uint32_t* __restrict__ keys_in;  // kDepthFirst: the N keys in id order; kDepth/kTile: pass input
  const uint32_t* __restrict__ vals_in;
  uint32_t* __restrict__ keys_out;
  uint32_t* __restrict__ vals_out;
  int64_t n;   // items: kDepthFirst N Gaussians, kDepth n_vis, kTileGen/kTile M
  const uint32_t* n_dev;  // if set, the item count is read here (kDepth: K1's visible count)
  int shift;   // digit = (key >> shift) & 255
  const uint32_t* __restrict__ bases;  // this pass's 256 digit bases + total (K2h)
  int last, tiles_x;                   // kTile: the last pass writes ty·tiles_x + tx
  // kTileGen: the generator's inputs (K2b offsets over the depth-sorted visible ids, K2b's
  // first Gaussian of each output block)
  const uint32_t* __restrict__ offsets;
  const uint32_t* __restrict__ sorted_ids;
  const uint2* __restrict__ rect;  // in depth order (K2b's rect_s)
  const uint32_t* __restrict__ bstart;
  int64_t n_gauss;  // entries of offsets / sorted_ids (RD_CHECKS)
  unsigned long long* status;
  uint32_t epoch;
  int match;  // rank with __match_any_sync (passes whose digits repeat within a warp)
};

struct GenSmem {  // kTileGen: the block's Gaussians (≤ 2049: every visible one touches ≥ 1 tile)
  uint32_t end[kSTile + 2];
  uint32_t id[kSTile + 1];
  uint2 rect[kSTile + 1];
};
struct PassSmem {
  uint2 kv[kSTile];  // (key, value) pairs: one 8-B access per item
  uint32_t cnt[kST / 32][kRadix];  // per-warp digit counts → warp offsets within the block's digit run
};
union SortSmem {
  GenSmem gen;
  PassSmem pass;
};

// K2c generator: the block's Gaussians are [bstart[b], bstart[b + 1]] (K2b: the owners of its
// first output and of the next block's first output). Thread t produces outputs o0 + 8t ..
// o0 + 8t + 7 (one binary search for the first one's owner in the staged Gaussians, then a
// walk: the owner advances by at most one per output, the tile steps row-major over its
// rect) as packed (ty << 16 | tx) keys.
__device__ __forceinline__ void generate_dups(const PassArgs& a, GenSmem& g, int b, uint32_t o0, uint32_t o1,
                                              uint32_t (&key)[kSI], uint32_t (&val)[kSI]) {
  const uint32_t g0 = a.bstart[b];
  const int ng = (int)(a.bstart[b + 1] - g0) + 1;
  RD_CHECK(ng >= 1 && ng <= kSTile + 1 && (int64_t)g0 + ng <= a.n_gauss);
  if (threadIdx.x == 0) g.end[0] = g0 == 0 ? 0u : a.offsets[g0 - 1];
  for (int k = threadIdx.x; k < ng; k += kST) {
    g.end[k + 1] = a.offsets[g0 + k];
    const uint32_t id = a.sorted_ids[g0 + k];
    g.id[k] = id;
    g.rect[k] = a.rect[g0 + k];  // K2b's depth-ordered copy
  }
  __syncthreads();
  const uint32_t o = o0 + (uint32_t)threadIdx.x * kSI;
#pragma unroll
  for (int j = 0; j < kSI; ++j) key[j] = val[j] = 0u;
  if (o >= o1) return;
  int lo = 0, hi = ng - 1;  // owner k: end[k] <= o < end[k + 1]
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (g.end[mid] <= o) lo = mid; else hi = mid - 1;
  }
  int k = lo;
  uint2 r = g.rect[k];
  uint32_t x0 = r.x & 0xffffu, x1 = r.y & 0xffffu;
  const uint32_t li = o - g.end[k], w = x1 - x0;
  uint32_t ty = (r.x >> 16) + li / w, tx = x0 + li % w;
#pragma unroll
  for (int j = 0; j < kSI; ++j) {
    const uint32_t oj = o + (uint32_t)j;
    if (oj < o1) {
      if (oj >= g.end[k + 1]) {  // the next Gaussian starts here, at its rect's first tile
        ++k;
        r = g.rect[k];
        x0 = r.x & 0xffffu;
        x1 = r.y & 0xffffu;
        tx = x0;
        ty = r.x >> 16;
      }
      key[j] = (ty << 16) | tx;
      val[j] = g.id[k];
      if (++tx == x1) {
        tx = x0;
        ++ty;
      }
    }
  }
}

// One LSD pass. Blocks are processed in blockIdx order (the dispatch order of a 1-D grid, as
// every single-pass look-back scan assumes), so a block's predecessors are resident or done.
#ifdef RD_BIN_TRACE  // development: per-block phase timestamps of the last tile pass
__device__ unsigned long long g_bin_trace[8192][6];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define RD_TRACE(k) if (MODE == kTile && threadIdx.x == 0 && blockIdx.x < 8192) g_bin_trace[blockIdx.x][k] = gtimer();
#else
#define RD_TRACE(k)
#endif

template <int MODE>
__global__ void __launch_bounds__(kST, RD_SORT_MINB) k_onesweep(PassArgs a) {
  extern __shared__ __align__(16) unsigned char dsmem[];  // SortSmem (> 48 KB at 512 threads)
  SortSmem& sm = *reinterpret_cast<SortSmem*>(dsmem);
  __shared__ uint32_t s_gbase[kRadix + 1];  // the pass's digit bases (K2h) + total
  __shared__ uint32_t s_dst[kRadix];        // global position of the block's first item of digit d − lstart
  __shared__ uint32_t s_warp[kST / 32];
  __shared__ uint32_t s_cnt;
  const int tid = (int)threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = (int)blockIdx.x;
  const int64_t n = a.n_dev ? (int64_t)*a.n_dev : a.n;
  const int64_t base = (int64_t)b * kSTile;
  if (base >= n) return;  // the grid is sized for an upper bound; later blocks are empty too
  RD_TRACE(0)

  // this block's items, warp-striped: warp w, lane l, item j ↔ position base + 256w + 32j + l
  uint32_t key[kSI], val[kSI];
  bool ok[kSI];
  if constexpr (MODE != kTileGen) {  // loads first: their latency overlaps the set-up below
    const uint32_t p0 = (uint32_t)base + (uint32_t)(warp * 256 + lane), nn = (uint32_t)n;  // < 2^31
#pragma unroll
    for (int j = 0; j < kSI; ++j) {
      const uint32_t p = p0 + (uint32_t)(j * 32);
      ok[j] = p < nn;
      key[j] = ok[j] ? a.keys_in[p] : 0u;
      if constexpr (MODE == kDepthFirst) {
        val[j] = p;
      } else {
        val[j] = ok[j] ? a.vals_in[p] : 0u;
      }
    }
  }
  if (tid <= kRadix) s_gbase[tid] = a.bases[tid];
  if constexpr (MODE == kTileGen) {
    const uint32_t o0 = (uint32_t)base, o1 = (uint32_t)(n < base + kSTile ? n : base + kSTile);
    uint32_t gk[kSI], gv[kSI];
    generate_dups(a, sm.gen, b, o0, o1, gk, gv);
    __syncthreads();  // the staged Gaussians are dead: the same shared memory takes the transpose
    uint4* kk = reinterpret_cast<uint4*>(sm.pass.kv + tid * kSI);
    kk[0] = make_uint4(gk[0], gv[0], gk[1], gv[1]);
    kk[1] = make_uint4(gk[2], gv[2], gk[3], gv[3]);
    kk[2] = make_uint4(gk[4], gv[4], gk[5], gv[5]);
    kk[3] = make_uint4(gk[6], gv[6], gk[7], gv[7]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSI; ++j) {
      const int p = warp * 256 + j * 32 + lane;
      ok[j] = (uint32_t)base + (uint32_t)p < (uint32_t)n;
      const uint2 q = sm.pass.kv[p];
      key[j] = q.x;
      val[j] = q.y;
    }
    __syncthreads();  // every lane has read its transposed items
  }
  if constexpr (MODE == kDepthFirst) {
#pragma unroll
    for (int j = 0; j < kSI; ++j) ok[j] = ok[j] && key[j] != 0xffffffffu;  // culled / off screen: dropped
  }
  for (int k = tid; k < (kST / 32) * kRadix; k += kST) (&sm.pass.cnt[0][0])[k] = 0u;
  __syncthreads();
  RD_TRACE(1)

  // stable rank within the warp: items in (j, lane) order = position order; the lanes holding
  // the same digit found by 8 ballots (constant cost, unlike __match_any_sync, whose cost grows
  // with the number of distinct digits in the warp — the tile digits of consecutive duplicates
  // are mostly distinct)
  uint32_t rank[kSI];
  const unsigned below = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kSI; ++j) {
    const uint32_t d = (key[j] >> a.shift) & 255u;
    unsigned peers;
    if (RD_RANK_MATCH || a.match) {  // warp-uniform
      peers = __match_any_sync(0xffffffffu, ok[j] ? d : 256u);
    } else {
      peers = __ballot_sync(0xffffffffu, ok[j]);
#pragma unroll
      for (int bit = 0; bit < 8; ++bit) {  // m = all ones where this lane's digit has the bit
        const unsigned m = (unsigned)((int)(d << (31 - bit)) >> 31);
        peers &= ~(__ballot_sync(0xffffffffu, (int)m < 0) ^ m);
      }
    }
    uint32_t c = 0u;
    if (ok[j]) c = sm.pass.cnt[warp][d];
    __syncwarp();
    rank[j] = c + (uint32_t)__popc(peers & below);
    if (ok[j] && (peers & below) == 0u) sm.pass.cnt[warp][d] = c + (uint32_t)__popc(peers);
    __syncwarp();
  }
  __syncthreads();

  RD_TRACE(2)
  // per digit (thread d < 256): warp offsets, the block's count, its sorted-layout start,
  // look-back
  {
    const int d = tid;
    uint32_t run = 0u;
    if (d < kRadix) {
#pragma unroll
      for (int w = 0; w < kST / 32; ++w) {
        const uint32_t c = sm.pass.cnt[w][d];
        sm.pass.cnt[w][d] = run;
        run += c;
      }
    }
    uint32_t btot;
    const uint32_t ls = block_excl_scan(run, s_warp, &btot);
    if (d == 0) s_cnt = btot;
    if (d < kRadix) {
#pragma unroll
      for (int w = 0; w < kST / 32; ++w) sm.pass.cnt[w][d] += ls;  // warp offsets → block positions
      uint32_t excl = 0u;
      if (s_gbase[d + 1] != s_gbase[d])  // digits no item of the pass has are never looked up
        excl = lookback(a.status + d, kRadix, b, a.epoch, run);
      s_dst[d] = s_gbase[d] + excl - ls;
    }
  }
  __syncthreads();
  RD_TRACE(3)
  // block-local sorted layout, then coalesced runs per digit
#pragma unroll
  for (int j = 0; j < kSI; ++j) {
    if (ok[j]) {
      const uint32_t d = (key[j] >> a.shift) & 255u;
      const uint32_t p = sm.pass.cnt[warp][d] + rank[j];  // (the digit's block start included)
      RD_CHECK(p < (uint32_t)kSTile);
      sm.pass.kv[p] = make_uint2(key[j], val[j]);
    }
  }
  __syncthreads();
  const int cnt = (int)s_cnt;
  for (int i = tid; i < cnt; i += kST) {
    const uint2 q = sm.pass.kv[i];
    const uint32_t k = q.x;
    const uint32_t dst = s_dst[(k >> a.shift) & 255u] + (uint32_t)i;
    RD_CHECK(dst < s_gbase[kRadix]);
    uint32_t out = k;
    if constexpr (MODE == kTile || MODE == kTileGen)
      if (a.last) out = (k >> 16) * (uint32_t)a.tiles_x + (k & 0xffffu);
    a.keys_out[dst] = out;
    a.vals_out[dst] = q.y;
  }
  RD_TRACE(4)
}

// ------------------------------------------------------------------------------- K2b
// offsets[p] = Σ_{q ≤ p} tiles_touched[ids[q]]: thread t sums items 8t..8t+7 of its block,
// block scan, one look-back word per block. The count of a Gaussian is its rect's area, so the
// scan gathers the rect (8 B) and also writes it in depth order (rect_s), which K2c then reads
// coalesced alongside the offsets instead of gathering it by id behind them. Each Gaussian
// also records itself as the first Gaussian of the K2c output blocks whose first output it
// owns: bstart[ob] = p for every ob·4096 in [offset_before, offset), and bstart[out_blocks] =
// n − 1.
__global__ void __launch_bounds__(kST) k_scan(const uint32_t* __restrict__ n_dev, const uint32_t* __restrict__ ids,
                                              const uint2* __restrict__ rect, uint2* __restrict__ rect_s,
                                              uint32_t* __restrict__ offsets, uint32_t* __restrict__ bstart,
                                              uint32_t out_blocks, unsigned long long* status, uint32_t epoch) {
  __shared__ uint32_t s_warp[kST / 32];
  __shared__ uint32_t s_excl;
  const int b = (int)blockIdx.x;
  const int64_t n = (int64_t)*n_dev;
  if ((int64_t)b * kSTile >= n) return;  // grid sized for N
  const int64_t p0 = (int64_t)b * kSTile + (int64_t)threadIdx.x * kSI;
  uint32_t v[kSI], t[kSI];
  uint2 r[kSI];
  if (p0 + kSI <= n) {
    const uint4 q0 = *reinterpret_cast<const uint4*>(ids + p0);
    const uint4 q1 = *reinterpret_cast<const uint4*>(ids + p0 + 4);
    r[0] = rect[q0.x]; r[1] = rect[q0.y]; r[2] = rect[q0.z]; r[3] = rect[q0.w];
    r[4] = rect[q1.x]; r[5] = rect[q1.y]; r[6] = rect[q1.z]; r[7] = rect[q1.w];
    uint4* o = reinterpret_cast<uint4*>(rect_s + p0);
#pragma unroll
    for (int j = 0; j < kSI; j += 2) o[j / 2] = make_uint4(r[j].x, r[j].y, r[j + 1].x, r[j + 1].y);
  } else {
#pragma unroll
    for (int j = 0; j < kSI; ++j) {
      r[j] = p0 + j < n ? rect[ids[p0 + j]] : make_uint2(0u, 0u);
      if (p0 + j < n) rect_s[p0 + j] = r[j];
    }
  }
#pragma unroll
  for (int j = 0; j < kSI; ++j)  // tiles touched = rect area (0 past the end)
    v[j] = ((r[j].y & 0xffffu) - (r[j].x & 0xffffu)) * ((r[j].y >> 16) - (r[j].x >> 16));
  uint32_t s = 0u;
#pragma unroll
  for (int j = 0; j < kSI; ++j) {
    t[j] = v[j];
    s += v[j];
    v[j] = s;
  }
  uint32_t btot;
  const uint32_t te = block_excl_scan(s, s_warp, &btot);
  if (threadIdx.x < 32) {
    const uint32_t x = lookback_warp(status, b, epoch, btot);
    if (threadIdx.x == 0) s_excl = x;
  }
  __syncthreads();
  const uint32_t e = s_excl + te;
  if (p0 + kSI <= n) {
    uint4* o = reinterpret_cast<uint4*>(offsets + p0);
    o[0] = make_uint4(e + v[0], e + v[1], e + v[2], e + v[3]);
    o[1] = make_uint4(e + v[4], e + v[5], e + v[6], e + v[7]);
  } else {
#pragma unroll
    for (int j = 0; j < kSI; ++j)
      if (p0 + j < n) offsets[p0 + j] = e + v[j];
  }
#pragma unroll
  for (int j = 0; j < kSI; ++j) {
    if (p0 + j < n) {
      const uint32_t hi = e + v[j], lo = hi - t[j];  // this Gaussian's outputs [lo, hi)
      for (uint32_t ob = (lo + kSTile - 1) / kSTile; ob * (uint32_t)kSTile < hi; ++ob) {
        RD_CHECK(ob < out_blocks);
        bstart[ob] = (uint32_t)(p0 + j);
      }
      if (p0 + j == n - 1) bstart[out_blocks] = (uint32_t)(p0 + j);
    }
  }
}

// Plain exclusive scan of a u32 array (marching cubes' per-cell triangle counts, NEXT-4):
// thread t scans items 8t..8t+7 of its block, block scan, one look-back word per block.
__global__ void __launch_bounds__(kST) k_scan_excl(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                   int64_t n, unsigned long long* status, uint32_t epoch) {
  __shared__ uint32_t s_warp[kST / 32];
  __shared__ uint32_t s_excl;
  const int b = (int)blockIdx.x;
  const int64_t p0 = (int64_t)b * kSTile + (int64_t)threadIdx.x * kSI;
  uint32_t v[kSI];
  if (p0 + kSI <= n) {
    const uint4 q0 = *reinterpret_cast<const uint4*>(in + p0);
    const uint4 q1 = *reinterpret_cast<const uint4*>(in + p0 + 4);
    v[0] = q0.x; v[1] = q0.y; v[2] = q0.z; v[3] = q0.w;
    v[4] = q1.x; v[5] = q1.y; v[6] = q1.z; v[7] = q1.w;
  } else {
#pragma unroll
    for (int j = 0; j < kSI; ++j) v[j] = p0 + j < n ? in[p0 + j] : 0u;
  }
  uint32_t s = 0u;
#pragma unroll
  for (int j = 0; j < kSI; ++j) {
    const uint32_t x = v[j];
    v[j] = s;  // exclusive
    s += x;
  }
  uint32_t btot;
  const uint32_t te = block_excl_scan(s, s_warp, &btot);
  if (threadIdx.x < 32) {
    const uint32_t x = lookback_warp(status, b, epoch, btot);
    if (threadIdx.x == 0) s_excl = x;
  }
  __syncthreads();
  const uint32_t e = s_excl + te;
  if (p0 + kSI <= n) {
    uint4* o = reinterpret_cast<uint4*>(out + p0);
    o[0] = make_uint4(e + v[0], e + v[1], e + v[2], e + v[3]);
    o[1] = make_uint4(e + v[4], e + v[5], e + v[6], e + v[7]);
  } else {
#pragma unroll
    for (int j = 0; j < kSI; ++j)
      if (p0 + j < n) out[p0 + j] = e + v[j];
  }
}

// ------------------------------------------------------------------------------- K2e
// 8 consecutive sorted keys per thread (two 16-B loads) + the next one; a boundary between
// positions k and k+1 closes tile keys[k] and opens tile keys[k+1].
__global__ void __launch_bounds__(256) k_ranges(const uint32_t* __restrict__ keys, int64_t m,
                                                 uint2* __restrict__ ranges) {
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (b >= m) return;
  uint32_t k[9];
  if (b + 8 <= m) {
    const uint4 q0 = *reinterpret_cast<const uint4*>(keys + b);
    const uint4 q1 = *reinterpret_cast<const uint4*>(keys + b + 4);
    k[0] = q0.x; k[1] = q0.y; k[2] = q0.z; k[3] = q0.w;
    k[4] = q1.x; k[5] = q1.y; k[6] = q1.z; k[7] = q1.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) k[j] = b + j < m ? keys[b + j] : 0xffffffffu;
  }
  k[8] = b + 8 < m ? keys[b + 8] : 0xffffffffu;
  if (b == 0) ranges[k[0]].x = 0u;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t p = b + j;
    if (p < m && k[j] != k[j + 1]) {
      ranges[k[j]].y = (uint32_t)(p + 1);
      if (p + 1 < m) ranges[k[j + 1]].x = (uint32_t)(p + 1);
    }
  }
}

__global__ void __launch_bounds__(256) k_keys64(const uint32_t* __restrict__ tiles, const uint32_t* __restrict__ ids,
                                                 const Record* __restrict__ rec, int64_t m,
                                                 uint64_t* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  out[k] = ((uint64_t)tiles[k] << 32) | (uint64_t)__float_as_uint(rec[ids[k]].r3.x);
}

unsigned blocks_of(int64_t n) { return (unsigned)((n + kSTile - 1) / kSTile); }

}  // namespace

size_t bin_status_words(int64_t n_items) { return (size_t)(blocks_of(n_items) + 1) * kRadix; }
size_t scan_status_words(int64_t n) { return (size_t)blocks_of(n) + 1; }
size_t bin_bstart_words(int64_t m) { return (size_t)blocks_of(m) + 2; }
int bin_max_tiles_per_axis() { return kMaxTileAxis - 1; }
int bin_bases_words() { return 8 * kBaseStride; }

constexpr int kSortSmem = (int)sizeof(SortSmem);
template <int MODE>
static void sort_attrs() {
  cudaFuncSetAttribute(k_onesweep<MODE>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_onesweep<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSortSmem);
}
static void set_carveout_once() {  // views are binned from several host threads at once
  static std::once_flag once;
  std::call_once(once, [] {
    sort_attrs<kDepthFirst>();
    sort_attrs<kDepth>();
    sort_attrs<kTileGen>();
    sort_attrs<kTile>();
  });
}

void launch_bin_hist(int64_t n, const uint32_t* dkey, const uint2* rect, int tiles_x, int tiles_y, uint32_t* cnt,
                     uint32_t* bases, uint32_t* host_counts, cudaStream_t s) {
  uint32_t* hist = cnt + kBinCntHist;
  int* diff_x = (int*)(cnt + kBinCntDiff);
  int* diff_y = diff_x + (tiles_x + 1);
  if (n == 0) return;
  static std::atomic<int> sms_cache{0};
  int sms = sms_cache.load();
  if (sms == 0) {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms_cache.store(v);
    sms = v;
  }
  const int64_t want = (n + kHistThreads - 1) / kHistThreads;
  const unsigned grid = (unsigned)(want < RD_HIST_BPS * sms ? want : RD_HIST_BPS * sms);
  k_bin_hist<<<grid, kHistThreads, 0, s>>>(n, dkey, rect, tiles_x, tiles_y, hist, diff_x, diff_y, cnt, bases,
                                           host_counts);
}

// Pass p (0..3) of the depth sort: pass 0 reads the N keys in id order (ids implicit) and
// writes buffer 1, then 1 → 0 → 1 → 0, so the result is in buffer 0. Passes 1-3 read the
// visible count from n_vis_dev (grid sized for N: no host sync before them).
void launch_depth_pass(int p, const uint32_t* dkey_id_order, int64_t n, const uint32_t* n_vis_dev,
                       const uint32_t* bases, uint32_t* const kb[2], uint32_t* const vb[2], BinSort& bs,
                       cudaStream_t s) {
  if (n == 0) return;
  set_carveout_once();
  const int out = p % 2 == 0 ? 1 : 0;
  PassArgs a{};
  a.keys_in = p == 0 ? dkey_id_order : kb[out ^ 1];
  a.vals_in = p == 0 ? nullptr : vb[out ^ 1];
  a.keys_out = kb[out];
  a.vals_out = vb[out];
  a.n = n;
  a.n_dev = p == 0 ? nullptr : n_vis_dev;
  a.shift = 8 * p;
  a.bases = bases + kBaseStride * p;
  a.status = bs.status;
  a.epoch = ++bs.epoch;
#ifndef RD_MATCH_DEPTH
#define RD_MATCH_DEPTH 8  // bit p: depth pass p ranks with __match_any_sync (pass 3: the top byte — sign and
                           // 7 exponent bits — takes few values per warp; 2 and the tile passes: slower)
#endif
  a.match = (RD_MATCH_DEPTH >> p) & 1;
  if (p == 0)
    k_onesweep<kDepthFirst><<<blocks_of(n), kST, kSortSmem, s>>>(a);
  else
    k_onesweep<kDepth><<<blocks_of(n), kST, kSortSmem, s>>>(a);
}

void launch_scan(const uint32_t* sorted_ids, const uint2* rect, uint2* rect_s, uint32_t* offsets, int64_t n_max,
                 const uint32_t* n_dev, uint32_t* bstart, int64_t m, BinSort& bs, cudaStream_t s) {
  if (n_max == 0) return;
  k_scan<<<blocks_of(n_max), kST, 0, s>>>(n_dev, sorted_ids, rect, rect_s, offsets, bstart, blocks_of(m), bs.status,
                                          ++bs.epoch);
}

int tile_sort_passes(int tiles_x, int tiles_y) {
  TilePass tp[4];
  return tile_pass_list(tiles_x, tiles_y, tp);
}

// Tile pass p writes buffer p % 2; pass 0 generates the duplicates (K2c) from the scan.
void launch_tile_pass(int p, int64_t m, int64_t n_gauss, const uint32_t* offsets, const uint32_t* sorted_ids,
                      const uint2* rect, const uint32_t* bstart, int tiles_x, int tiles_y, const uint32_t* bases,
                      uint32_t* const kb[2], uint32_t* const vb[2], BinSort& bs, cudaStream_t s) {
  if (m == 0) return;
  set_carveout_once();
  TilePass tp[4];
  const int np = tile_pass_list(tiles_x, tiles_y, tp);
  const int out = p % 2;
  PassArgs a{};
  a.keys_in = p == 0 ? nullptr : kb[out ^ 1];
  a.vals_in = p == 0 ? nullptr : vb[out ^ 1];
  a.keys_out = kb[out];
  a.vals_out = vb[out];
  a.n = m;
  a.shift = 16 * tp[p].axis + tp[p].dshift;
  a.bases = bases + kBaseStride * (4 + p);
  a.last = p == np - 1 ? 1 : 0;
  a.tiles_x = tiles_x;
  a.offsets = offsets;
  a.sorted_ids = sorted_ids;
  a.rect = rect;
  a.bstart = bstart;
  a.n_gauss = n_gauss;
  a.status = bs.status;
  a.epoch = ++bs.epoch;
#ifndef RD_MATCH_TILE
#define RD_MATCH_TILE 0  // bit p: tile pass p ranks with __match_any_sync
#endif
  a.match = (RD_MATCH_TILE >> p) & 1;
  if (p == 0)
    k_onesweep<kTileGen><<<blocks_of(m), kST, kSortSmem, s>>>(a);
  else
    k_onesweep<kTile><<<blocks_of(m), kST, kSortSmem, s>>>(a);
}

void launch_scan_excl_u32(const uint32_t* in, uint32_t* out, int64_t n, BinSort& bs, cudaStream_t s) {
  if (n == 0) return;
  k_scan_excl<<<blocks_of(n), kST, 0, s>>>(in, out, n, bs.status, ++bs.epoch);
}

void launch_ranges(const uint32_t* keys, int64_t m, int n_tiles, uint2* ranges, cudaStream_t s) {
  cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)n_tiles, s);
  if (m == 0) return;
  const int threads = 256;
  const int64_t items = (m + 7) / 8;
  k_ranges<<<(unsigned)((items + threads - 1) / threads), threads, 0, s>>>(keys, m, ranges);
}

void launch_keys64(const uint32_t* tiles, const uint32_t* ids, const Record* rec, int64_t m, uint64_t* out,
                   cudaStream_t s) {
  if (m == 0) return;
  const int threads = 256;
  k_keys64<<<(unsigned)((m + threads - 1) / threads), threads, 0, s>>>(tiles, ids, rec, m, out);
}

}  // namespace rade

#ifdef RD_BIN_TRACE
extern "C" int rd_debug_bin_trace(unsigned long long* host, int nblocks) {
  return (int)cudaMemcpyFromSymbol(host, rade::g_bin_trace, sizeof(unsigned long long) * 6 * (size_t)nblocks);
}
#endif
