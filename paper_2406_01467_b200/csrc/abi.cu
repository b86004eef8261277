// abi.cu — the C ABI of include/rade.h: argument validation, the per-view stage machine,
// capacity-cached scratch buffers (caller allocator or cudaMallocAsync), optional per-kernel
// CUDA-event profiling, and the launch sequence of the five stages. Host code only;
// kernels live in preprocess.cu, binning.cu and render.cu.
#include "../../include/rade.h"
#include "rade_internal.cuh"

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <vector>

using namespace rade;

namespace {

thread_local std::string g_err;

rd_status fail(rd_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
rd_status fail(rd_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define RD_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return fail(RD_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

// RADE_SYNC_CHECK=1 in the environment synchronises after every launch so a device fault
// is attributed to the kernel that raised it (debugging only).
bool sync_check() {
  static const bool on = [] {
    const char* e = getenv("RADE_SYNC_CHECK");
    return e && e[0] == '1';
  }();
  return on;
}

#define RD_CHECK_LAUNCH(what)                                                                       \
  do {                                                                                              \
    cudaError_t e_ = cudaGetLastError();                                                            \
    if (e_ == cudaSuccess && sync_check()) e_ = cudaDeviceSynchronize();                            \
    if (e_ != cudaSuccess) return fail(RD_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e_)); \
  } while (0)

struct Buf {
  void* ptr = nullptr;
  size_t cap = 0;
};

enum Kernel { K_PRE = 0, K_DSORT, K_SCAN, K_DUP, K_TSORT, K_RANGES, K_FWD, K_BWD, K_PREBWD };

}  // namespace

struct rd_view {
  rd_alloc_fn alloc = nullptr;
  rd_free_fn free_fn = nullptr;
  void* ctx = nullptr;
  int stage = 0;
  int64_t n = 0;
  int sh_coeffs = 0;
  DevCam cam{};
  DevOpt opt{};
  int tiles_x = 0, tiles_y = 0;
  int key_bits = 0;   // 32 + tile_bits: the equivalent one-pass 64-bit key width
  int tile_bits = 0;
  int64_t M = 0;
  int tsel = 0;  // buffer (0/1) holding the sorted tile keys and ids
  bool binned = false;  // rd_bin ran since the last rd_preprocess
  int64_t n_vis = 0, n_big = 0;
  bool g2d_dirty = false;  // the G2D rows hold a previous rd_blend_bwd's sums (K1 zeroes them)
  bool dist_fwd = false;   // the last forward produced the distortion map and its K4 state
  Buf dist_d0, dist_D1;
  uint32_t* host_M = nullptr;  // mapped pinned: [0] visible, [1] big, [2] M, written by K2h
  uint32_t* host_M_dev = nullptr;  // its device alias
  cudaEvent_t m_ready = nullptr;  // recorded after K2h, waited on by rd_bin (the path's one sync)
  BinSort bs{nullptr, 0u};  // K2's look-back state (binning.cu)
  Buf rec, rect, rect_s, touched, offsets, dkey0, dkey1, didx0, didx1, vis, big, bincnt, status, bstart;
  Buf tkeys0, tkeys1, vals0, vals1;
  Buf ranges;
  Buf T_final, n_contrib, median_pos;
  Buf g2d;
  Buf bmask;  // K3 → K4 blend mask (tile 8)
  Buf tile_order;  // K3/K4 launch order (longest lists first)
  // profiling
  bool prof = false;
  cudaStream_t last_stream = nullptr;
  struct Ev {
    cudaEvent_t a, b;
    int k;
  };
  std::vector<Ev> pending;
  std::vector<cudaEvent_t> pool;
  Buf counters;
  double acc_ms[RD_NUM_KERNELS] = {0};
  int64_t acc_launch[RD_NUM_KERNELS] = {0};
  int64_t acc_M = 0, acc_views = 0;
  cudaEvent_t cur_a = nullptr;

  rd_status ensure(Buf& b, size_t bytes, cudaStream_t s) {
    if (bytes == 0) bytes = 16;
    if (b.cap >= bytes) return RD_OK;
    release(b, s);
    size_t want = bytes + bytes / 4 + 256;
    void* p = nullptr;
    if (alloc) {
      p = alloc(want, ctx);
      if (!p) return fail(RD_ERR_ALLOC, "allocator callback failed for %zu bytes", want);
    } else {
      cudaError_t e = cudaMallocAsync(&p, want, s);
      if (e != cudaSuccess) return fail(RD_ERR_ALLOC, "cudaMallocAsync(%zu): %s", want, cudaGetErrorString(e));
    }
    b.ptr = p;
    b.cap = want;
    return RD_OK;
  }
  void release(Buf& b, cudaStream_t s) {
    if (!b.ptr) return;
    if (free_fn)
      free_fn(b.ptr, ctx);
    else
      cudaFreeAsync(b.ptr, s);
    b.ptr = nullptr;
    b.cap = 0;
  }
  cudaEvent_t get_event() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  void begin(cudaStream_t s) {
    last_stream = s;
    if (!prof) return;
    cur_a = get_event();
    cudaEventRecord(cur_a, s);
  }
  void end(int k, cudaStream_t s) {
    if (!prof) return;
    cudaEvent_t b = get_event();
    cudaEventRecord(b, s);
    pending.push_back(Ev{cur_a, b, k});
  }
  Counter* ctr() { return prof ? (Counter*)counters.ptr : nullptr; }
  DevBounds bounds() const {
    return DevBounds{n, M, (int64_t)(bmask.cap / sizeof(uint32_t)), (int64_t)tiles_x * tiles_y};
  }
  void resolve() {
    for (const Ev& e : pending) {
      float ms = 0.f;
      cudaEventSynchronize(e.b);
      cudaEventElapsedTime(&ms, e.a, e.b);
      acc_ms[e.k] += ms;
      acc_launch[e.k] += 1;
      pool.push_back(e.a);
      pool.push_back(e.b);
    }
    pending.clear();
  }
  void reset_acc() {
    resolve();
    for (int k = 0; k < RD_NUM_KERNELS; ++k) {
      acc_ms[k] = 0.0;
      acc_launch[k] = 0;
    }
    acc_M = acc_views = 0;
    if (counters.ptr) cudaMemsetAsync(counters.ptr, 0, kNumCounters * sizeof(Counter), last_stream);
  }
};

#define RD_ENSURE(buf, bytes, s)              \
  do {                                        \
    rd_status st_ = v->ensure(buf, bytes, s); \
    if (st_ != RD_OK) return st_;             \
  } while (0)

// K2's look-back status words for up to n_items per pass; zeroed when (re)allocated (every
// later pass tags its words with a fresh epoch, so they are never cleared again)
#define RD_ENSURE_STATUS(v, n_items, s)                                                   \
  do {                                                                                   \
    const size_t bytes_ = bin_status_words(n_items) * sizeof(unsigned long long);        \
    if ((v)->status.cap < bytes_) {                                                       \
      RD_ENSURE((v)->status, bytes_, s);                                                  \
      RD_CUDA(cudaMemsetAsync((v)->status.ptr, 0, (v)->status.cap, s));                   \
      (v)->bs.status = (unsigned long long*)(v)->status.ptr;                              \
    }                                                                                    \
  } while (0)

extern "C" {

const char* rd_last_error(void) { return g_err.c_str(); }

const char* rd_version(void) { return "rade-b200 0.1 (sm_100a)"; }

rd_status rd_options_default(rd_options* opt) {
  if (!opt) return fail(RD_ERR_INVALID_ARGUMENT, "opt is NULL");
  opt->tile = 16;
  opt->alpha_min = 1.f / 255.f;
  opt->alpha_max = 0.99f;
  opt->T_min = 1e-4f;
  opt->median_T = 0.5f;
  opt->dilation = 0.3f;
  opt->bg[0] = opt->bg[1] = opt->bg[2] = 0.f;
  opt->sh_degree = 3;
  opt->guard_band = 0.f;  // reading S6b off
  return RD_OK;
}

rd_status rd_view_create(rd_view** view, rd_alloc_fn alloc, rd_free_fn free_fn, void* ctx) {
  g_err.clear();
  if (!view) return fail(RD_ERR_INVALID_ARGUMENT, "view is NULL");
  if ((alloc == nullptr) != (free_fn == nullptr))
    return fail(RD_ERR_INVALID_ARGUMENT, "alloc and free_fn must both be given or both be NULL");
  rd_view* v = new (std::nothrow) rd_view();
  if (!v) return fail(RD_ERR_ALLOC, "out of host memory");
  v->alloc = alloc;
  v->free_fn = free_fn;
  v->ctx = ctx;
  *view = v;  // no CUDA call here: the pinned M slot is allocated by the first rd_bin
  return RD_OK;
}

rd_status rd_view_destroy(rd_view* v) {
  if (!v) return fail(RD_ERR_INVALID_ARGUMENT, "view is NULL");
  Buf* all[] = {&v->rec,    &v->rect,   &v->touched, &v->offsets, &v->dkey0,   &v->dkey1,     &v->didx0,
                &v->didx1,  &v->status, &v->tkeys0,  &v->tkeys1,  &v->vals0,   &v->vals1,     &v->ranges,
                &v->T_final, &v->n_contrib, &v->median_pos, &v->g2d, &v->counters, &v->bmask, &v->tile_order, &v->vis, &v->big, &v->bincnt, &v->bstart, &v->rect_s, &v->dist_d0, &v->dist_D1};
  if (v->stage > 0 || v->prof) cudaStreamSynchronize(v->last_stream);
  v->resolve();
  for (cudaEvent_t e : v->pool) cudaEventDestroy(e);
  for (Buf* b : all) v->release(*b, v->last_stream);
  if (v->host_M) cudaFreeHost(v->host_M);
  if (v->m_ready) cudaEventDestroy(v->m_ready);
  delete v;
  return RD_OK;
}

static bool in01(float x) { return x > 0.f && x < 1.f && std::isfinite(x); }

static rd_status preprocess_setup(rd_view* v, const rd_gaussians* g, const rd_camera* cam, const rd_options* opt,
                                 cudaStream_t s) {
  g_err.clear();
  if (!v || !g || !cam || !opt) return fail(RD_ERR_INVALID_ARGUMENT, "NULL view/gaussians/camera/options");
  if (g->n < 0) return fail(RD_ERR_INVALID_ARGUMENT, "n < 0");
  if (g->n > 0x7fffffffLL) return fail(RD_ERR_INVALID_ARGUMENT, "n >= 2^31 not supported");
  if (g->n > 0 && (!g->means || !g->scales || !g->rotations || !g->opacities || !g->sh))
    return fail(RD_ERR_INVALID_ARGUMENT, "NULL Gaussian array");
  if (((uintptr_t)g->rotations & 15u) != 0) return fail(RD_ERR_INVALID_ARGUMENT, "rotations not 16-byte aligned");
  if ((g->sh_coeffs * 3) % 4 == 0 && ((uintptr_t)g->sh & 15u) != 0)
    return fail(RD_ERR_INVALID_ARGUMENT, "sh not 16-byte aligned");
  if (cam->width <= 0 || cam->height <= 0) return fail(RD_ERR_INVALID_ARGUMENT, "width/height must be > 0");
  if (!(cam->fx > 0.f && cam->fy > 0.f) || !std::isfinite(cam->fx) || !std::isfinite(cam->fy))
    return fail(RD_ERR_INVALID_ARGUMENT, "fx, fy must be finite and > 0");
  if (!(cam->znear > 0.f)) return fail(RD_ERR_INVALID_ARGUMENT, "znear must be > 0");
  if (opt->tile != 8 && opt->tile != 16 && opt->tile != 32)
    return fail(RD_ERR_INVALID_ARGUMENT, "tile must be 8, 16 or 32");
  if (!in01(opt->alpha_min) || !in01(opt->alpha_max) || !in01(opt->T_min) || !in01(opt->median_T))
    return fail(RD_ERR_INVALID_ARGUMENT, "alpha_min, alpha_max, T_min, median_T must lie in (0, 1)");
  if (!(opt->alpha_min < opt->alpha_max)) return fail(RD_ERR_INVALID_ARGUMENT, "alpha_min must be < alpha_max");
  if (!(opt->dilation >= 0.f) || !std::isfinite(opt->dilation))
    return fail(RD_ERR_INVALID_ARGUMENT, "dilation must be finite and >= 0");
  if (opt->sh_degree < 0 || opt->sh_degree > 3) return fail(RD_ERR_INVALID_ARGUMENT, "sh_degree must be 0..3");
  if (!(opt->guard_band >= 0.f) || !std::isfinite(opt->guard_band))
    return fail(RD_ERR_INVALID_ARGUMENT, "guard_band must be finite and >= 0 (0 = off)");
  const int need = (opt->sh_degree + 1) * (opt->sh_degree + 1);
  if (g->sh_coeffs < need || g->sh_coeffs > 16)
    return fail(RD_ERR_INVALID_ARGUMENT, "sh_coeffs=%d incompatible with sh_degree=%d", g->sh_coeffs,
                opt->sh_degree);
  const int tiles_x = (cam->width + opt->tile - 1) / opt->tile;
  const int tiles_y = (cam->height + opt->tile - 1) / opt->tile;
  if (tiles_x > bin_max_tiles_per_axis() || tiles_y > bin_max_tiles_per_axis())
    return fail(RD_ERR_INVALID_ARGUMENT, "image too large: more than %d tiles per axis", bin_max_tiles_per_axis());

  v->n = g->n;
  v->sh_coeffs = g->sh_coeffs;
  DevCam& c = v->cam;
  c.fx = cam->fx; c.fy = cam->fy; c.cx = cam->cx; c.cy = cam->cy;
  c.W = cam->width; c.H = cam->height;
  for (int k = 0; k < 9; ++k) c.R[k] = cam->R[k];
  for (int k = 0; k < 3; ++k) c.t[k] = cam->t[k];
  c.znear = cam->znear;
  const double gb = (double)opt->guard_band;  // reading S6b: off at 0
  c.guard = gb > 0.0 ? 1 : 0;
  c.gu0 = (float)(-gb * cam->width - (double)cam->cx);
  c.gu1 = (float)((1.0 + gb) * cam->width - (double)cam->cx);
  c.gv0 = (float)(-gb * cam->height - (double)cam->cy);
  c.gv1 = (float)((1.0 + gb) * cam->height - (double)cam->cy);
  for (int i = 0; i < 3; ++i) {
    double acc = 0.0;
    for (int k = 0; k < 3; ++k) acc -= (double)cam->R[3 * k + i] * (double)cam->t[k];
    c.campos[i] = (float)acc;
  }
  DevOpt& o = v->opt;
  o.tile = opt->tile;
  o.alpha_min = opt->alpha_min; o.alpha_max = opt->alpha_max; o.T_min = opt->T_min;
  o.median_T = opt->median_T; o.dilation = opt->dilation;
  for (int k = 0; k < 3; ++k) o.bg[k] = opt->bg[k];
  o.sh_degree = opt->sh_degree;
  o.ln_alpha_min = logf(opt->alpha_min);
  o.log2_alpha_min = log2f(opt->alpha_min);
  v->tiles_x = tiles_x;
  v->tiles_y = tiles_y;
  int bits = 1;
  while ((1LL << bits) < (long long)tiles_x * tiles_y) ++bits;
  v->tile_bits = bits;
  v->key_bits = 32 + bits;

  const size_t n = (size_t)g->n;
  RD_ENSURE(v->rec, n * sizeof(Record), s);
  RD_ENSURE(v->rect, n * sizeof(uint2), s);
  RD_ENSURE(v->rect_s, n * sizeof(uint2), s);
  RD_ENSURE(v->touched, n * sizeof(uint32_t), s);
  RD_ENSURE(v->offsets, n * sizeof(uint32_t), s);
  RD_ENSURE(v->dkey0, n * sizeof(uint32_t), s);
  RD_ENSURE(v->dkey1, n * sizeof(uint32_t), s);
  RD_ENSURE(v->didx0, n * sizeof(uint32_t), s);
  RD_ENSURE(v->didx1, n * sizeof(uint32_t), s);
  RD_ENSURE(v->vis, n * sizeof(uint32_t), s);
  RD_ENSURE(v->big, n * sizeof(uint32_t), s);
  const size_t cnt_words = (size_t)kBinCntDiff + (size_t)(tiles_x + 1) + (size_t)(tiles_y + 1) + (size_t)bin_bases_words();
  RD_ENSURE(v->bincnt, cnt_words * sizeof(uint32_t), s);
  RD_ENSURE(v->g2d, n * sizeof(G2D), s);
  if (!v->host_M) {
    RD_CUDA(cudaHostAlloc((void**)&v->host_M, 4 * sizeof(uint32_t), cudaHostAllocMapped));
    RD_CUDA(cudaHostGetDevicePointer((void**)&v->host_M_dev, v->host_M, 0));
  }
  if (!v->m_ready) RD_CUDA(cudaEventCreateWithFlags(&v->m_ready, cudaEventDisableTiming));

  return RD_OK;
}

// After K1 (one view or a round): the view's state.
static void preprocess_done(rd_view* v) {
  v->stage = 1;
  v->binned = false;
  v->M = 0;
  v->n_vis = v->n_big = 0;
  v->g2d_dirty = false;
}

rd_status rd_preprocess(rd_view* v, const rd_gaussians* g, const rd_camera* cam, const rd_options* opt,
                        rd_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  rd_status st = preprocess_setup(v, g, cam, opt, s);
  if (st != RD_OK) return st;
  const DevCam& c = v->cam;
  const DevOpt& o = v->opt;
  DevGauss dg{g->n, g->sh_coeffs, g->means, g->scales, g->rotations, g->opacities, g->sh, g->filter3d};
  v->begin(s);  // K1 timing includes the zeroing of its counters
  RD_CUDA(cudaMemsetAsync(v->bincnt.ptr, 0, kBinCntHist * sizeof(uint32_t), s));
  launch_preprocess_fwd(dg, c, o, v->tiles_x, (Record*)v->rec.ptr, (uint2*)v->rect.ptr, (uint32_t*)v->touched.ptr,
                        (uint32_t*)v->dkey0.ptr, (uint32_t*)v->bincnt.ptr, (uint32_t*)v->vis.ptr,
                        (uint32_t*)v->big.ptr, (G2D*)v->g2d.ptr, v->ctr(), s);
  RD_CHECK_LAUNCH("preprocess_fwd");
  v->end(K_PRE, s);
  preprocess_done(v);
  return RD_OK;
}

rd_status rd_preprocess_views(rd_view* const* views, int32_t n_views, const rd_gaussians* g, const rd_camera* cams,
                              const rd_options* opt, rd_stream stream) {
  g_err.clear();
  if (!views || !cams) return fail(RD_ERR_INVALID_ARGUMENT, "NULL views / cameras");
  if (n_views < 1 || n_views > kMaxBatchViews)
    return fail(RD_ERR_INVALID_ARGUMENT, "n_views must be 1..%d", kMaxBatchViews);
  for (int k = 0; k < n_views; ++k) {
    if (!views[k]) return fail(RD_ERR_INVALID_ARGUMENT, "views[%d] is NULL", k);
    for (int j = 0; j < k; ++j)
      if (views[j] == views[k]) return fail(RD_ERR_INVALID_ARGUMENT, "views[%d] repeats views[%d]", k, j);
  }
  cudaStream_t s = (cudaStream_t)stream;
  K1Views kv{};
  kv.nv = n_views;
  for (int k = 0; k < n_views; ++k) {
    rd_view* v = views[k];
    rd_status st = preprocess_setup(v, g, &cams[k], opt, s);
    if (st != RD_OK) return st;
    RD_CUDA(cudaMemsetAsync(v->bincnt.ptr, 0, kBinCntHist * sizeof(uint32_t), s));
    kv.v[k] = K1Out{v->cam, (Record*)v->rec.ptr, (uint2*)v->rect.ptr, (uint32_t*)v->touched.ptr,
                    (uint32_t*)v->dkey0.ptr, (uint32_t*)v->bincnt.ptr, (uint32_t*)v->vis.ptr, (uint32_t*)v->big.ptr,
                    (G2D*)v->g2d.ptr, v->ctr()};
  }
  DevGauss dg{g->n, g->sh_coeffs, g->means, g->scales, g->rotations, g->opacities, g->sh, g->filter3d};
  rd_view* v0 = views[0];
  v0->begin(s);  // timed on views[0] (one K1 launch for the round)
  launch_preprocess_fwd_views(dg, v0->opt, kv, s);
  RD_CHECK_LAUNCH("preprocess_fwd_views");
  v0->end(K_PRE, s);
  for (int k = 0; k < n_views; ++k) {
    views[k]->last_stream = s;
    preprocess_done(views[k]);
  }
  return RD_OK;
}

rd_status rd_bin(rd_view* v, int64_t* n_duplicates_out, rd_stream stream) {
  g_err.clear();
  if (!v) return fail(RD_ERR_INVALID_ARGUMENT, "view is NULL");
  if (v->stage < 1) return fail(RD_ERR_STATE, "rd_bin before rd_preprocess");
  if (v->binned) {  // already binned since the last rd_preprocess: the sorted lists stand (the depth
    if (n_duplicates_out) *n_duplicates_out = v->M;  // passes consumed K1's id-order keys)
    return RD_OK;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = v->n;
  const int n_tiles = v->tiles_x * v->tiles_y;
  uint32_t* cnt = (uint32_t*)v->bincnt.ptr;
  uint32_t* hist = cnt + kBinCntHist;
  int* diff_x = (int*)(cnt + kBinCntDiff);
  int* diff_y = diff_x + (v->tiles_x + 1);
  uint32_t* bases = (uint32_t*)(diff_y + (v->tiles_y + 1));
  uint32_t* const dk[2] = {(uint32_t*)v->dkey0.ptr, (uint32_t*)v->dkey1.ptr};
  uint32_t* const di[2] = {(uint32_t*)v->didx0.ptr, (uint32_t*)v->didx1.ptr};
  const uint32_t* sorted_ids = di[0];  // depth pass 3 writes buffer 0
  int64_t M = 0;
  if (n > 0) {
    // K2h and the depth passes are sized on the device (K1's visible count), so they are queued
    // before the host waits for the counts K2h writes (the one sync of the path)
    RD_ENSURE_STATUS(v, n, s);
    v->begin(s);  // the depth sort's time includes K2h and the zeroing of its histograms
    RD_CUDA(cudaMemsetAsync(hist, 0, (kBinCntDiff - kBinCntHist + v->tiles_x + v->tiles_y + 2) * sizeof(uint32_t), s));
    launch_bin_hist(n, dk[0], (const uint2*)v->rect.ptr, v->tiles_x, v->tiles_y, cnt, bases, v->host_M_dev, s);
    RD_CHECK_LAUNCH("bin_hist");
    RD_CUDA(cudaEventRecord(v->m_ready, s));  // K2h has written the counts to host_M
    for (int p = 0; p < 4; ++p) {
      launch_depth_pass(p, dk[0], n, cnt, bases, dk, di, v->bs, s);
      RD_CHECK_LAUNCH("depth_sort");
    }
    v->end(K_DSORT, s);
    RD_CUDA(cudaEventSynchronize(v->m_ready));
    v->n_vis = (int64_t)v->host_M[0];
    v->n_big = (int64_t)v->host_M[1];
    M = (int64_t)v->host_M[2];
    if (M > 0x7fffffffLL) return fail(RD_ERR_INVALID_ARGUMENT, "M = %lld duplicates >= 2^31", (long long)M);
    RD_ENSURE(v->bstart, bin_bstart_words(M) * sizeof(uint32_t), s);
    v->begin(s);
    launch_scan(sorted_ids, (const uint2*)v->rect.ptr, (uint2*)v->rect_s.ptr, (uint32_t*)v->offsets.ptr, n, cnt,
                (uint32_t*)v->bstart.ptr, M, v->bs, s);
    RD_CHECK_LAUNCH("scan");
    v->end(K_SCAN, s);
  }
  RD_ENSURE(v->tkeys0, (size_t)M * sizeof(uint32_t), s);
  RD_ENSURE(v->tkeys1, (size_t)M * sizeof(uint32_t), s);
  RD_ENSURE(v->vals0, (size_t)M * sizeof(uint32_t), s);
  RD_ENSURE(v->vals1, (size_t)M * sizeof(uint32_t), s);
  RD_ENSURE(v->ranges, (size_t)n_tiles * sizeof(uint2), s);
  v->tsel = 0;
  if (M > 0) {
    RD_ENSURE_STATUS(v, M, s);
    uint32_t* const tk[2] = {(uint32_t*)v->tkeys0.ptr, (uint32_t*)v->tkeys1.ptr};
    uint32_t* const tv[2] = {(uint32_t*)v->vals0.ptr, (uint32_t*)v->vals1.ptr};
    const int np = tile_sort_passes(v->tiles_x, v->tiles_y);
    for (int p = 0; p < np; ++p) {
      v->begin(s);
      launch_tile_pass(p, M, v->n_vis, (const uint32_t*)v->offsets.ptr, sorted_ids, (const uint2*)v->rect_s.ptr,
                       (const uint32_t*)v->bstart.ptr, v->tiles_x, v->tiles_y, bases, tk, tv, v->bs, s);
      RD_CHECK_LAUNCH(p == 0 ? "duplicate" : "tile_sort");
      if (p == 0) {
        v->end(K_DUP, s);  // K2c: the duplicates generated and ranked by their first tile digit
      } else {
        v->end(K_TSORT, s);
      }
    }
    v->tsel = (np - 1) % 2;
  }
  const uint32_t* keys = (const uint32_t*)(v->tsel ? v->tkeys1.ptr : v->tkeys0.ptr);
  v->begin(s);
  launch_ranges(keys, M, n_tiles, (uint2*)v->ranges.ptr, s);
  RD_CHECK_LAUNCH("ranges");
  v->end(K_RANGES, s);
  v->M = M;
  v->acc_M += M;
  v->stage = 2;
  v->binned = true;
  if (n_duplicates_out) *n_duplicates_out = M;
  return RD_OK;
}

rd_status rd_render_fwd_ex(rd_view* v, const rd_fwd_maps* maps, rd_stream stream) {
  g_err.clear();
  if (!v || !maps) return fail(RD_ERR_INVALID_ARGUMENT, "view / maps is NULL");
  if (v->stage < 2) return fail(RD_ERR_STATE, "rd_render_fwd before rd_bin");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t HW = (size_t)v->cam.W * v->cam.H;
  RD_ENSURE(v->T_final, HW * sizeof(float), s);
  RD_ENSURE(v->n_contrib, HW * sizeof(int32_t), s);
  RD_ENSURE(v->median_pos, HW * sizeof(int32_t), s);
  RD_ENSURE(v->bmask, blend_mask_words(v->M, v->tiles_x * v->tiles_y) * sizeof(uint32_t), s);
  RD_ENSURE(v->tile_order, (size_t)v->tiles_x * v->tiles_y * sizeof(uint32_t), s);
  DistIO dio{nullptr, nullptr, nullptr, nullptr};
  v->dist_fwd = maps->distortion != nullptr;
  if (v->dist_fwd) {
    RD_ENSURE(v->dist_d0, HW * sizeof(float), s);
    RD_ENSURE(v->dist_D1, HW * sizeof(float), s);
    dio = DistIO{maps->distortion, (float*)v->dist_d0.ptr, (float*)v->dist_D1.ptr, nullptr};
  }
  const uint32_t* ids = (const uint32_t*)(v->tsel ? v->vals1.ptr : v->vals0.ptr);
  v->begin(s);
  launch_render_fwd(v->cam, v->opt, v->tiles_x, v->tiles_y, (const uint2*)v->ranges.ptr, ids,
                    (const Record*)v->rec.ptr, maps->color, maps->depth, maps->normal, maps->alpha,
                    (float*)v->T_final.ptr, (int32_t*)v->n_contrib.ptr, (int32_t*)v->median_pos.ptr, dio,
                    (uint32_t*)v->bmask.ptr, (uint32_t*)v->tile_order.ptr, v->ctr(), v->bounds(), s);
  RD_CHECK_LAUNCH("render_fwd");
  v->end(K_FWD, s);
  v->acc_views += 1;
  v->stage = 3;
  return RD_OK;
}

rd_status rd_render_fwd(rd_view* v, float* color, float* depth, float* normal, float* alpha, rd_stream stream) {
  const rd_fwd_maps maps{color, depth, normal, alpha, nullptr};
  return rd_render_fwd_ex(v, &maps, stream);
}

rd_status rd_blend_bwd(rd_view* v, const float* dL_dcolor, const float* dL_ddepth, const float* dL_dnormal,
                       const float* dL_dalpha, rd_stream stream) {
  const rd_bwd_cotangents cot{dL_dcolor, dL_ddepth, dL_dnormal, dL_dalpha, nullptr};
  return rd_blend_bwd_ex(v, &cot, stream);
}

rd_status rd_blend_bwd_ex(rd_view* v, const rd_bwd_cotangents* cot, rd_stream stream) {
  g_err.clear();
  if (!v || !cot) return fail(RD_ERR_INVALID_ARGUMENT, "view / cotangents is NULL");
  if (v->stage < 3) return fail(RD_ERR_STATE, "rd_blend_bwd before rd_render_fwd");
  if (cot->dL_ddistortion && !v->dist_fwd)
    return fail(RD_ERR_STATE, "distortion cotangent given, but the forward produced no distortion map");
  const float* dL_dcolor = cot->dL_dcolor;
  const float* dL_ddepth = cot->dL_ddepth;
  const float* dL_dnormal = cot->dL_dnormal;
  const float* dL_dalpha = cot->dL_dalpha;
  DistIO dio{nullptr, nullptr, nullptr, nullptr};
  if (cot->dL_ddistortion) dio = DistIO{nullptr, (float*)v->dist_d0.ptr, (float*)v->dist_D1.ptr, cot->dL_ddistortion};
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t* ids = (const uint32_t*)(v->tsel ? v->vals1.ptr : v->vals0.ptr);
  v->begin(s);
  if (v->g2d_dirty && v->n > 0)  // another backward after the same rd_preprocess: re-zero the rows
    RD_CUDA(cudaMemsetAsync(v->g2d.ptr, 0, (size_t)v->n * sizeof(G2D), s));
  v->g2d_dirty = true;
  launch_render_bwd(v->cam, v->opt, v->tiles_x, v->tiles_y, (const uint2*)v->ranges.ptr, ids,
                    (const Record*)v->rec.ptr, (const float*)v->T_final.ptr, (const int32_t*)v->n_contrib.ptr,
                    (const int32_t*)v->median_pos.ptr, dL_dcolor, dL_ddepth, dL_dnormal, dL_dalpha, dio,
                    (const uint32_t*)v->bmask.ptr, (const uint32_t*)v->tile_order.ptr, (G2D*)v->g2d.ptr, v->ctr(),
                    v->bounds(), s);
  RD_CHECK_LAUNCH("render_bwd");
  v->end(K_BWD, s);
  v->stage = 4;
  return RD_OK;
}

static rd_status preprocess_bwd_parts(rd_view* v, const rd_gaussians* g, const rd_grads* grads, rd_stream stream,
                                      int parts) {
  g_err.clear();
  if (!v || !g || !grads) return fail(RD_ERR_INVALID_ARGUMENT, "NULL view/gaussians/grads");
  if (v->stage < 4) return fail(RD_ERR_STATE, "rd_preprocess_bwd before rd_blend_bwd");
  if (g->n != v->n || g->sh_coeffs != v->sh_coeffs)
    return fail(RD_ERR_INVALID_ARGUMENT, "Gaussians differ from those given to rd_preprocess");
  if (g->n > 0 && (!g->means || !g->scales || !g->rotations || !g->opacities || !g->sh))
    return fail(RD_ERR_INVALID_ARGUMENT, "NULL Gaussian array");
  if (g->n > 0 && (!grads->means || !grads->scales || !grads->rotations || !grads->opacities || !grads->sh))
    return fail(RD_ERR_INVALID_ARGUMENT, "NULL gradient array");
  if ((((uintptr_t)g->rotations | (uintptr_t)grads->rotations) & 15u) != 0)
    return fail(RD_ERR_INVALID_ARGUMENT, "rotations / their gradients not 16-byte aligned");
  if ((g->sh_coeffs * 3) % 4 == 0 && (((uintptr_t)g->sh | (uintptr_t)grads->sh) & 15u) != 0)
    return fail(RD_ERR_INVALID_ARGUMENT, "sh / its gradient not 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  DevGauss dg{g->n, g->sh_coeffs, g->means, g->scales, g->rotations, g->opacities, g->sh, g->filter3d};
  DevGrads dgr{grads->means, grads->scales, grads->rotations, grads->opacities, grads->sh, grads->means2d};
  v->begin(s);
  launch_preprocess_bwd(dg, v->cam, v->opt, (const uint32_t*)v->touched.ptr, (const uint32_t*)v->vis.ptr, v->n_vis,
                        (const uint32_t*)v->big.ptr, v->n_big, (const G2D*)v->g2d.ptr, dgr, s, parts);
  RD_CHECK_LAUNCH("preprocess_bwd");
  v->end(K_PREBWD, s);
  return RD_OK;
}

rd_status rd_preprocess_bwd(rd_view* v, const rd_gaussians* g, const rd_grads* grads, rd_stream stream) {
  return preprocess_bwd_parts(v, g, grads, stream, kK5All);
}

rd_status rd_preprocess_bwd_geometry(rd_view* v, const rd_gaussians* g, const rd_grads* grads, rd_stream stream) {
  return preprocess_bwd_parts(v, g, grads, stream, kK5Geometry);
}

static rd_status preprocess_bwd_views_parts(rd_view* const* views, int32_t n_views, const rd_gaussians* g,
                                            const rd_grads* grads, rd_stream stream, int parts) {
  g_err.clear();
  if (!views || !g || !grads) return fail(RD_ERR_INVALID_ARGUMENT, "NULL views/gaussians/grads");
  if (n_views < 1 || n_views > kMaxBatchViews)
    return fail(RD_ERR_INVALID_ARGUMENT, "n_views must be 1..%d", kMaxBatchViews);
  if (g->n > 0 && (!g->means || !g->scales || !g->rotations || !g->opacities || !g->sh))
    return fail(RD_ERR_INVALID_ARGUMENT, "NULL Gaussian array");
  if (g->n > 0 && (!grads->means || !grads->scales || !grads->rotations || !grads->opacities || !grads->sh))
    return fail(RD_ERR_INVALID_ARGUMENT, "NULL gradient array");
  if ((((uintptr_t)g->rotations | (uintptr_t)grads->rotations) & 15u) != 0)
    return fail(RD_ERR_INVALID_ARGUMENT, "rotations / their gradients not 16-byte aligned");
  if ((g->sh_coeffs * 3) % 4 == 0 && (((uintptr_t)g->sh | (uintptr_t)grads->sh) & 15u) != 0)
    return fail(RD_ERR_INVALID_ARGUMENT, "sh / its gradient not 16-byte aligned");
  DevCam cams[kMaxBatchViews];
  const uint32_t* touched[kMaxBatchViews];
  const G2D* g2d[kMaxBatchViews];
  const uint32_t* big[kMaxBatchViews];
  int64_t n_big[kMaxBatchViews];
  const uint32_t* vis[kMaxBatchViews];
  int64_t n_vis[kMaxBatchViews];
  for (int k = 0; k < n_views; ++k) {
    const rd_view* v = views[k];
    if (!v) return fail(RD_ERR_INVALID_ARGUMENT, "views[%d] is NULL", k);
    if (v->stage < 4) return fail(RD_ERR_STATE, "views[%d]: rd_preprocess_bwd_views before rd_blend_bwd", k);
    if (g->n != v->n || g->sh_coeffs != v->sh_coeffs)
      return fail(RD_ERR_INVALID_ARGUMENT, "views[%d]: Gaussians differ from those given to rd_preprocess", k);
    if (std::memcmp(&v->opt, &views[0]->opt, sizeof(DevOpt)) != 0)
      return fail(RD_ERR_INVALID_ARGUMENT, "views[%d]: options differ from views[0]'s", k);
    for (int j = 0; j < k; ++j)
      if (views[j] == v) return fail(RD_ERR_INVALID_ARGUMENT, "views[%d] repeats views[%d]", k, j);
    cams[k] = v->cam;
    touched[k] = (const uint32_t*)v->touched.ptr;
    g2d[k] = (const G2D*)v->g2d.ptr;
    big[k] = (const uint32_t*)v->big.ptr;
    n_big[k] = v->n_big;
    vis[k] = (const uint32_t*)v->vis.ptr;
    n_vis[k] = v->n_vis;
  }
  cudaStream_t s = (cudaStream_t)stream;
  DevGauss dg{g->n, g->sh_coeffs, g->means, g->scales, g->rotations, g->opacities, g->sh, g->filter3d};
  DevGrads dgr{grads->means, grads->scales, grads->rotations, grads->opacities, grads->sh, grads->means2d};
  rd_view* v0 = views[0];
  v0->begin(s);  // timed on views[0] (K_PREBWD, one launch for the batch)
  launch_preprocess_bwd_views(dg, v0->opt, n_views, cams, touched, g2d, vis, n_vis, big, n_big, dgr, v0->ctr(), s,
                              parts);
  RD_CHECK_LAUNCH("preprocess_bwd_views");
  v0->end(K_PREBWD, s);
  return RD_OK;
}

rd_status rd_preprocess_bwd_views(rd_view* const* views, int32_t n_views, const rd_gaussians* g, const rd_grads* grads,
                                  rd_stream stream) {
  return preprocess_bwd_views_parts(views, n_views, g, grads, stream, kK5All);
}

rd_status rd_preprocess_bwd_views_sh(rd_view* const* views, int32_t n_views, const rd_gaussians* g,
                                     const rd_grads* grads, rd_stream stream) {
  return preprocess_bwd_views_parts(views, n_views, g, grads, stream, kK5Sh);
}

rd_status rd_preprocess_bwd_views_ex(rd_view* const* views, int32_t n_views, const rd_gaussians* g,
                                     const rd_grads* grads, uint32_t flags, rd_stream stream) {
  g_err.clear();
  if (flags & ~(uint32_t)(RD_K5_SH_ONLY | RD_K5_GEOMETRY_ONLY | RD_K5_SET_SH))
    return fail(RD_ERR_INVALID_ARGUMENT, "unknown flags 0x%x", flags);
  if ((flags & RD_K5_SH_ONLY) && (flags & RD_K5_GEOMETRY_ONLY))
    return fail(RD_ERR_INVALID_ARGUMENT, "RD_K5_SH_ONLY and RD_K5_GEOMETRY_ONLY exclude each other");
  if ((flags & RD_K5_SET_SH) && (flags & RD_K5_GEOMETRY_ONLY))
    return fail(RD_ERR_INVALID_ARGUMENT, "RD_K5_SET_SH needs the SH part");
  if ((flags & RD_K5_SET_SH) && g && (g->sh_coeffs * 3) % 4 != 0)
    return fail(RD_ERR_INVALID_ARGUMENT, "RD_K5_SET_SH needs SH rows of a multiple of 4 floats");
  int parts = (flags & RD_K5_SH_ONLY) ? kK5Sh : (flags & RD_K5_GEOMETRY_ONLY) ? kK5Geometry : kK5All;
  if (flags & RD_K5_SET_SH) parts |= kK5ShSet;
  return preprocess_bwd_views_parts(views, n_views, g, grads, stream, parts);
}

rd_status rd_render_bwd(rd_view* v, const rd_gaussians* g, const float* dL_dcolor, const float* dL_ddepth,
                        const float* dL_dnormal, const float* dL_dalpha, const rd_grads* grads, rd_stream stream) {
  g_err.clear();
  if (!v || !g || !grads) return fail(RD_ERR_INVALID_ARGUMENT, "NULL view/gaussians/grads");
  if (v->stage < 3) return fail(RD_ERR_STATE, "rd_render_bwd before rd_render_fwd");
  if (g->n != v->n || g->sh_coeffs != v->sh_coeffs)
    return fail(RD_ERR_INVALID_ARGUMENT, "Gaussians differ from those given to rd_preprocess");
  if (g->n > 0 && (!g->means || !g->scales || !g->rotations || !g->opacities || !g->sh))
    return fail(RD_ERR_INVALID_ARGUMENT, "NULL Gaussian array");
  if (g->n > 0 && (!grads->means || !grads->scales || !grads->rotations || !grads->opacities || !grads->sh))
    return fail(RD_ERR_INVALID_ARGUMENT, "NULL gradient array");
  rd_status st = rd_blend_bwd(v, dL_dcolor, dL_ddepth, dL_dnormal, dL_dalpha, stream);
  if (st != RD_OK) return st;
  return rd_preprocess_bwd(v, g, grads, stream);
}

rd_status rd_normal_consistency(const rd_camera* cam, const float* depth, const float* alpha, const float* normal,
                                float* consistency, float* depth_normal, rd_stream stream) {
  g_err.clear();
  if (!cam || !depth) return fail(RD_ERR_INVALID_ARGUMENT, "NULL camera / depth");
  if (consistency && (!alpha || !normal)) return fail(RD_ERR_INVALID_ARGUMENT, "consistency needs alpha and normal");
  if (cam->width < 0 || cam->height < 0) return fail(RD_ERR_INVALID_ARGUMENT, "negative image size");
  if (!(cam->fx > 0.f && cam->fy > 0.f)) return fail(RD_ERR_INVALID_ARGUMENT, "fx, fy must be > 0");
  launch_normal_consistency(cam->fx, cam->fy, cam->cx, cam->cy, cam->width, cam->height, depth, alpha, normal,
                            consistency, depth_normal, (cudaStream_t)stream);
  RD_CHECK_LAUNCH("normal_consistency");
  return RD_OK;
}

rd_status rd_normal_consistency_bwd(const rd_camera* cam, const float* depth, const float* normal,
                                    const float* dL_dconsistency, float* dL_ddepth, float* dL_dalpha,
                                    float* dL_dnormal, rd_stream stream) {
  g_err.clear();
  if (!cam || !depth || !normal || !dL_dconsistency)
    return fail(RD_ERR_INVALID_ARGUMENT, "NULL camera / depth / normal / dL_dconsistency");
  if (cam->width < 0 || cam->height < 0) return fail(RD_ERR_INVALID_ARGUMENT, "negative image size");
  if (!(cam->fx > 0.f && cam->fy > 0.f)) return fail(RD_ERR_INVALID_ARGUMENT, "fx, fy must be > 0");
  launch_normal_consistency_bwd(cam->fx, cam->fy, cam->cx, cam->cy, cam->width, cam->height, depth, normal,
                                dL_dconsistency, dL_ddepth, dL_dalpha, dL_dnormal, (cudaStream_t)stream);
  RD_CHECK_LAUNCH("normal_consistency_bwd");
  return RD_OK;
}

rd_status rd_tsdf_integrate(const rd_tsdf* vol, const float* depths, const rd_camera* cams, int32_t n_views,
                            rd_stream stream) {
  g_err.clear();
  if (!vol || (n_views > 0 && (!depths || !cams))) return fail(RD_ERR_INVALID_ARGUMENT, "NULL volume/depths/cams");
  if (n_views < 0) return fail(RD_ERR_INVALID_ARGUMENT, "n_views < 0");
  if (vol->dims[0] < 0 || vol->dims[1] < 0 || vol->dims[2] < 0) return fail(RD_ERR_INVALID_ARGUMENT, "negative dims");
  if ((int64_t)vol->dims[0] * vol->dims[1] * vol->dims[2] > 0 && (!vol->tsdf || !vol->weight))
    return fail(RD_ERR_INVALID_ARGUMENT, "NULL tsdf/weight");
  if (!(vol->voxel_size > 0.f) || !(vol->truncation > 0.f))
    return fail(RD_ERR_INVALID_ARGUMENT, "voxel_size and truncation must be > 0");
  const int W = n_views > 0 ? cams[0].width : 0, H = n_views > 0 ? cams[0].height : 0;
  for (int v = 0; v < n_views; ++v) {
    if (cams[v].width != W || cams[v].height != H)
      return fail(RD_ERR_INVALID_ARGUMENT, "all cameras must have the same width/height");
    if (!(cams[v].fx > 0.f && cams[v].fy > 0.f)) return fail(RD_ERR_INVALID_ARGUMENT, "fx, fy must be > 0");
  }
  const int per = tsdf_views_per_launch();
  std::vector<float> rows(17 * (size_t)per);
  for (int v0 = 0; v0 < n_views; v0 += per) {
    const int nv = std::min(per, n_views - v0);
    for (int k = 0; k < nv; ++k) {
      const rd_camera& c = cams[v0 + k];
      float* r = rows.data() + 17 * k;
      for (int j = 0; j < 9; ++j) r[j] = c.R[j];
      for (int j = 0; j < 3; ++j) r[9 + j] = c.t[j];
      r[12] = c.fx; r[13] = c.fy; r[14] = c.cx; r[15] = c.cy; r[16] = c.znear;
    }
    launch_tsdf_integrate(rows.data(), nv, depths + (size_t)v0 * W * H, W, H, vol->origin, vol->voxel_size,
                          vol->truncation, vol->max_depth, vol->dims, vol->tsdf, vol->weight, (cudaStream_t)stream);
    RD_CHECK_LAUNCH("tsdf_integrate");
  }
  return RD_OK;
}

rd_status rd_marching_cubes(const rd_tsdf* vol, float iso, float* triangles, int64_t capacity, int64_t* n_triangles,
                            rd_stream stream) {
  g_err.clear();
  if (!vol || !n_triangles) return fail(RD_ERR_INVALID_ARGUMENT, "NULL volume/n_triangles");
  if (vol->dims[0] < 0 || vol->dims[1] < 0 || vol->dims[2] < 0) return fail(RD_ERR_INVALID_ARGUMENT, "negative dims");
  if ((int64_t)vol->dims[0] * vol->dims[1] * vol->dims[2] > 0 && (!vol->tsdf || !vol->weight))
    return fail(RD_ERR_INVALID_ARGUMENT, "NULL tsdf/weight");
  if (!(vol->voxel_size > 0.f)) return fail(RD_ERR_INVALID_ARGUMENT, "voxel_size must be > 0");
  if (capacity < 0) return fail(RD_ERR_INVALID_ARGUMENT, "capacity < 0");
  const cudaError_t e = launch_marching_cubes(vol->origin, vol->voxel_size, vol->dims, vol->tsdf, vol->weight, iso,
                                              triangles, capacity, n_triangles, (cudaStream_t)stream);
  if (e == cudaErrorInvalidValue) return fail(RD_ERR_INVALID_ARGUMENT, "volume has more than 2^31 cells");
  if (e == cudaErrorMemoryAllocation) return fail(RD_ERR_ALLOC, "marching_cubes temporaries");
  if (e != cudaSuccess) return fail(RD_ERR_CUDA, "marching_cubes: %s", cudaGetErrorString(e));
  return RD_OK;
}

rd_status rd_set_profiling(rd_view* v, int32_t enabled) {
  if (!v) return fail(RD_ERR_INVALID_ARGUMENT, "view is NULL");
  if (enabled) {
    rd_status st = v->ensure(v->counters, kNumCounters * sizeof(Counter), v->last_stream);
    if (st != RD_OK) return st;
  }
  v->prof = enabled != 0;
  v->reset_acc();
  if (cudaGetLastError() != cudaSuccess) return fail(RD_ERR_CUDA, "rd_set_profiling: CUDA error");
  return RD_OK;
}

rd_status rd_get_timings(rd_view* v, rd_timings* out, int32_t reset) {
  if (!v || !out) return fail(RD_ERR_INVALID_ARGUMENT, "NULL view/out");
  v->resolve();
  std::memset(out, 0, sizeof(*out));
  for (int k = 0; k < RD_NUM_KERNELS; ++k) {
    out->ms[k] = v->acc_ms[k];
    out->launches[k] = v->acc_launch[k];
  }
  out->n_duplicates = v->acc_M;
  out->views = v->acc_views;
  if (v->counters.ptr) {
    Counter h[kNumCounters] = {0};
    RD_CUDA(cudaMemcpyAsync(h, v->counters.ptr, sizeof(h), cudaMemcpyDeviceToHost, v->last_stream));
    RD_CUDA(cudaStreamSynchronize(v->last_stream));
    out->pairs_evaluated_fwd = (int64_t)h[0];
    out->pairs_blended_fwd = (int64_t)h[1];
    out->pairs_evaluated_bwd = (int64_t)h[2];
    out->n_visible = (int64_t)h[3];
    out->n_visible_union = (int64_t)h[4];
    out->pairs_issued_fwd = (int64_t)h[kIssuedCounter];
    for (int k = 0; k < 6; ++k)
      for (int b = 0; b < kCullSlots; ++b) out->n_culled[k] += (int64_t)h[kCullCounter0 + k * kCullSlots + b];
  }
  if (reset) v->reset_acc();
  return RD_OK;
}

rd_status rd_view_stats(const rd_view* v, rd_stats* out) {
  if (!v || !out) return fail(RD_ERR_INVALID_ARGUMENT, "NULL view/out");
  out->n = v->n;
  out->n_duplicates = v->M;
  out->tiles_x = v->tiles_x;
  out->tiles_y = v->tiles_y;
  out->width = v->cam.W;
  out->height = v->cam.H;
  out->stage = v->stage;
  out->key_bits = v->key_bits;
  out->n_visible = v->n_vis;
  out->n_big = v->n_big;
  return RD_OK;
}

rd_status rd_debug_binning(const rd_view* v, uint64_t* keys, uint32_t* ids, uint32_t* ranges, rd_stream stream) {
  if (!v) return fail(RD_ERR_INVALID_ARGUMENT, "view is NULL");
  if (v->stage < 2) return fail(RD_ERR_STATE, "rd_debug_binning before rd_bin");
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t* tk = (const uint32_t*)(v->tsel ? v->tkeys1.ptr : v->tkeys0.ptr);
  const uint32_t* iv = (const uint32_t*)(v->tsel ? v->vals1.ptr : v->vals0.ptr);
  if (keys && v->M) {
    launch_keys64(tk, iv, (const Record*)v->rec.ptr, v->M, keys, s);
    RD_CHECK_LAUNCH("keys64");
  }
  if (ids && v->M) RD_CUDA(cudaMemcpyAsync(ids, iv, (size_t)v->M * 4, cudaMemcpyDeviceToDevice, s));
  if (ranges)
    RD_CUDA(cudaMemcpyAsync(ranges, v->ranges.ptr, (size_t)v->tiles_x * v->tiles_y * 8, cudaMemcpyDeviceToDevice, s));
  return RD_OK;
}

rd_status rd_debug_preprocess(const rd_view* v, float* records, uint32_t* rects, uint32_t* tiles_touched,
                              rd_stream stream) {
  if (!v) return fail(RD_ERR_INVALID_ARGUMENT, "view is NULL");
  if (v->stage < 1) return fail(RD_ERR_STATE, "rd_debug_preprocess before rd_preprocess");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t n = (size_t)v->n;
  if (n == 0) return RD_OK;
  if (records) RD_CUDA(cudaMemcpyAsync(records, v->rec.ptr, n * sizeof(Record), cudaMemcpyDeviceToDevice, s));
  if (rects) RD_CUDA(cudaMemcpyAsync(rects, v->rect.ptr, n * sizeof(uint2), cudaMemcpyDeviceToDevice, s));
  if (tiles_touched) RD_CUDA(cudaMemcpyAsync(tiles_touched, v->touched.ptr, n * 4, cudaMemcpyDeviceToDevice, s));
  return RD_OK;
}

rd_status rd_debug_pixel_state(const rd_view* v, float* T_final, int32_t* n_contrib, int32_t* median_pos,
                               rd_stream stream) {
  if (!v) return fail(RD_ERR_INVALID_ARGUMENT, "view is NULL");
  if (v->stage < 3) return fail(RD_ERR_STATE, "rd_debug_pixel_state before rd_render_fwd");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t HW = (size_t)v->cam.W * v->cam.H;
  if (T_final) RD_CUDA(cudaMemcpyAsync(T_final, v->T_final.ptr, HW * 4, cudaMemcpyDeviceToDevice, s));
  if (n_contrib) RD_CUDA(cudaMemcpyAsync(n_contrib, v->n_contrib.ptr, HW * 4, cudaMemcpyDeviceToDevice, s));
  if (median_pos) RD_CUDA(cudaMemcpyAsync(median_pos, v->median_pos.ptr, HW * 4, cudaMemcpyDeviceToDevice, s));
  return RD_OK;
}

rd_status rd_debug_grads2d(const rd_view* v, float* grads2d, rd_stream stream) {
  if (!v || !grads2d) return fail(RD_ERR_INVALID_ARGUMENT, "NULL view/grads2d");
  if (!v->g2d.ptr) return fail(RD_ERR_STATE, "rd_debug_grads2d before rd_render_bwd");
  cudaStream_t s = (cudaStream_t)stream;
  launch_g2d_to_f32((const G2D*)v->g2d.ptr, v->n, grads2d, s);
  RD_CHECK_LAUNCH("g2d_to_f32");
  return RD_OK;
}

}  // extern "C"
