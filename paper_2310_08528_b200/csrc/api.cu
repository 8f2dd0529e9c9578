// C ABI of libfgs.so (include/fgs.h): argument validation, workspace layout, frame batching.
// Everything here is host code; the arithmetic of the method lives in deform.cu / render.cu.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "fgs_internal.cuh"

namespace fgs {
namespace {

thread_local std::string g_err = "ok";

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(FGS_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
bool aligned4(const void* p) { return ((uintptr_t)p & 3u) == 0; }

#define FGS_CHECK(cond, msg) \
  do {                       \
    if (!(cond)) return fail(FGS_E_INVALID, msg); \
  } while (0)

int check_gaussians(const fgs_gaussians* g) {
  FGS_CHECK(g, "gaussians is NULL");
  FGS_CHECK(g->n >= 0 && g->n < (int64_t)1 << 31, "gaussians.n out of range [0, 2^31)");
  FGS_CHECK(g->sh_degree >= 0 && g->sh_degree <= 3, "sh_degree must be in [0,3]");
  if (g->n == 0) return FGS_OK;
  FGS_CHECK(g->means && g->log_scales && g->quats && g->opacity_logits && g->sh, "null Gaussian array");
  FGS_CHECK(aligned4(g->means) && aligned4(g->log_scales) && aligned16(g->quats) &&
                aligned4(g->opacity_logits) && aligned16(g->sh),
            "Gaussian arrays misaligned (quats, sh: 16 B; means, log_scales, opacity: 4 B)");
  return FGS_OK;
}

int check_field(const fgs_hexplanes* h, const fgs_mlp* m) {
  FGS_CHECK(h && m, "hexplanes/mlp is NULL");
  FGS_CHECK(h->n_scales >= 1 && h->n_scales <= FGS_MAX_SCALES, "n_scales must be in [1,4]");
  FGS_CHECK(h->feat == 8 || h->feat == 16 || h->feat == 32, "feat must be 8, 16 or 32");
  FGS_CHECK(h->t_res >= 2, "t_res must be >= 2");
  for (int l = 0; l < h->n_scales; ++l) {
    FGS_CHECK(h->res[l] >= 2 && h->res[l] <= 4096, "res[l] must be in [2,4096]");
    for (int p = 0; p < FGS_PLANES; ++p)
      FGS_CHECK(h->planes[l][p] && aligned16(h->planes[l][p]), "plane pointer NULL or misaligned");
  }
  for (int a = 0; a < 3; ++a)
    FGS_CHECK(isfinite(h->bmin[a]) && isfinite(h->bmax[a]) && h->bmax[a] > h->bmin[a], "bad AABB");
  FGS_CHECK(m->in_dim == h->feat * h->n_scales, "mlp.in_dim != feat * n_scales");
  FGS_CHECK(m->in_dim <= 64, "in_dim must be <= 64");
  FGS_CHECK(m->width == 32 || m->width == 64 || m->width == 128, "mlp.width must be 32, 64 or 128");
  FGS_CHECK(m->w_d && m->b_d && m->w_x && m->b_x && m->w_r && m->b_r && m->w_s && m->b_s, "null MLP array");
  FGS_CHECK((m->w_c == nullptr) == (m->b_c == nullptr), "phi_C needs both w_c and b_c");
  FGS_CHECK((m->w_a == nullptr) == (m->b_a == nullptr), "phi_alpha needs both w_a and b_a");
  FGS_CHECK(aligned16(m->w_d), "w_d must be 16-byte aligned");
  return FGS_OK;
}

int check_deformed(const fgs_deformed* d, int64_t n, int sh_degree, bool writable) {
  FGS_CHECK(d, "deformed is NULL");
  FGS_CHECK(d->n == n, "deformed.n != gaussians.n");
  FGS_CHECK(d->sh_degree == sh_degree, "deformed.sh_degree mismatch");
  if (n == 0) return FGS_OK;
  FGS_CHECK(d->means && d->log_scales && d->quats, "null deformed output array");
  FGS_CHECK(aligned4(d->means) && aligned4(d->log_scales) && aligned16(d->quats),
            "deformed arrays misaligned (quats: 16 B; means, log_scales: 4 B)");
  if (!writable) {
    FGS_CHECK(d->opacity_logits && d->sh, "null deformed opacity/sh");
    FGS_CHECK(aligned4(d->opacity_logits) && aligned16(d->sh), "deformed opacity/sh misaligned");
  }
  return FGS_OK;
}

int check_camera(const fgs_camera* c) {
  FGS_CHECK(c, "camera is NULL");
  FGS_CHECK(c->width > 0 && c->height > 0 && c->width <= 16384 && c->height <= 16384, "bad image size");
  FGS_CHECK(isfinite(c->fx) && isfinite(c->fy) && c->fx > 0 && c->fy > 0, "bad focal length");
  return FGS_OK;
}

void fill_deform(DeformBatch& p, const fgs_gaussians* g, const fgs_hexplanes* h, const fgs_mlp* m) {
  memset(&p, 0, sizeof(p));
  p.means = g->means; p.log_scales = g->log_scales; p.quats = g->quats;
  p.n_scales = h->n_scales; p.feat = h->feat; p.t_res = h->t_res;
  for (int l = 0; l < FGS_MAX_SCALES; ++l) {
    p.res[l] = h->res[l];
    for (int q = 0; q < FGS_PLANES; ++q) p.planes[l][q] = l < h->n_scales ? h->planes[l][q] : nullptr;
  }
  for (int a = 0; a < 3; ++a) { p.bmin[a] = h->bmin[a]; p.ext[a] = h->bmax[a] - h->bmin[a]; }
  p.in_dim = m->in_dim; p.width = m->width;
  p.w_d = m->w_d; p.b_d = m->b_d; p.w_x = m->w_x; p.b_x = m->b_x;
  p.w_r = m->w_r; p.b_r = m->b_r; p.w_s = m->w_s; p.b_s = m->b_s;
  p.w_c = m->w_c; p.b_c = m->b_c; p.w_a = m->w_a; p.b_a = m->b_a;
  p.n_c = m->w_c ? 3 * (g->sh_degree + 1) * (g->sh_degree + 1) : 0;
  p.sh_in = g->sh; p.opac_in = g->opacity_logits;
  p.n_peer = 1;                          // one replica at offset 0 (memset)
}


int deform_impl(const fgs_gaussians* g, const fgs_hexplanes* h, const fgs_mlp* m, const float* ts, int n_t,
                int64_t begin, int64_t end, fgs_deformed* outs, cudaStream_t s, const int64_t* peer_off = nullptr,
                int n_peers = 0) {
  int rc;
  if ((rc = check_gaussians(g)) != FGS_OK) return rc;
  if ((rc = check_field(h, m)) != FGS_OK) return rc;
  FGS_CHECK(ts && outs && n_t >= 0, "null times/outputs");
  FGS_CHECK(begin >= 0 && begin <= end && end <= g->n, "begin/end out of range");
  const bool heads_c = m->w_c != nullptr, heads_a = m->w_a != nullptr;
  for (int f = 0; f < n_t; ++f) {
    FGS_CHECK(isfinite(ts[f]) && ts[f] >= 0.f && ts[f] <= 1.f, "t must be finite and in [0,1]");
    if ((rc = check_deformed(&outs[f], g->n, g->sh_degree, true)) != FGS_OK) return rc;
    if (g->n > 0 && heads_c)
      FGS_CHECK(outs[f].sh && aligned16(outs[f].sh) && outs[f].sh != g->sh,
                "phi_C: deformed.sh must be a caller buffer (16-byte aligned), not the canonical SH");
    if (g->n > 0 && heads_a)
      FGS_CHECK(outs[f].opacity_logits && aligned4(outs[f].opacity_logits) && outs[f].opacity_logits != g->opacity_logits,
                "phi_alpha: deformed.opacity_logits must be a caller buffer, not the canonical array");
  }
  if (end == begin || n_t == 0) return FGS_OK;
  DeformBatch p;
  fill_deform(p, g, h, m);
  p.begin = begin; p.end = end;
  // every field check_field accepts fits the warp-specialised kernel (feat 8..32, in_dim <= 64, W <= 128)
  if (!deform_tc3_supported(p)) return fail(FGS_E_NOTIMPL, "field does not fit the deform kernel's TMEM plan");
  if (peer_off) {
    FGS_CHECK(n_peers >= 1 && n_peers <= kMaxPeers, "n_peers must be in [1, 8]");
    FGS_CHECK(!heads_c && !heads_a, "peer replicas: only means / log_scales / quats (no phi_C / phi_alpha)");
    for (int q = 0; q < n_peers; ++q) FGS_CHECK(peer_off[q] % 4 == 0, "peer offsets must be multiples of 4 bytes");
    p.n_peer = n_peers;
    for (int q = 0; q < n_peers; ++q) p.peer_off[q] = peer_off[q];
  }
  for (int f0 = 0; f0 < n_t; f0 += kMaxFrames) {
    p.n_t = std::min(kMaxFrames, n_t - f0);
    for (int f = 0; f < p.n_t; ++f) {
      p.t[f] = ts[f0 + f];
      p.out_means[f] = outs[f0 + f].means;
      p.out_log_scales[f] = outs[f0 + f].log_scales;
      p.out_quats[f] = outs[f0 + f].quats;
      p.out_sh[f] = outs[f0 + f].sh;
      p.out_opacity[f] = outs[f0 + f].opacity_logits;
    }
    cudaError_t e = launch_deform_tc3(p, s);
    if (e != cudaSuccess) return cuda_fail(e, "deform launch");
  }
  return FGS_OK;
}

__global__ void fill_bg_kernel(float* img, int w, int h, float r, float g, float b, float* fT, uint32_t* nc,
                               uint32_t* ne) {
  const size_t hw = (size_t)w * h;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < hw; i += (size_t)gridDim.x * blockDim.x) {
    img[i] = r; img[hw + i] = g; img[2 * hw + i] = b;
    if (fT) fT[i] = 1.f;
    if (nc) nc[i] = 0;
    if (ne) ne[i] = 0;
  }
}

int render_impl(const fgs_camera* cams, const fgs_deformed* defs, float* const* images, int n_frames, void* ws,
                size_t ws_bytes, const fgs_render_aux* aux, cudaStream_t s) {
  FGS_CHECK(cams && defs && images && n_frames >= 0, "null camera/deformed/image arrays");
  if (n_frames == 0) return FGS_OK;
  int rc;
  for (int f = 0; f < n_frames; ++f) {
    if ((rc = check_camera(&cams[f])) != FGS_OK) return rc;
    FGS_CHECK(cams[f].width == cams[0].width && cams[f].height == cams[0].height,
              "all frames of a batch must share width/height");
    if ((rc = check_deformed(&defs[f], defs[0].n, defs[0].sh_degree, false)) != FGS_OK) return rc;
    FGS_CHECK(images[f] && aligned16(images[f]), "image pointer NULL or misaligned");
  }
  FGS_CHECK(defs[0].n >= 0 && defs[0].n < ((int64_t)1 << 31), "n out of range");
  FGS_CHECK(defs[0].sh_degree >= 0 && defs[0].sh_degree <= 3, "sh_degree must be in [0,3]");
  const int W = cams[0].width, H = cams[0].height;
  const int64_t n = defs[0].n;
  FGS_CHECK(ws && aligned16(ws), "workspace NULL or misaligned");
  const size_t per = (ws_bytes / (size_t)n_frames) & ~(size_t)255;
  const int64_t cap = capacity_for(n, W, H, per);
  FGS_CHECK(cap > 0 || n == 0, "workspace too small (see fgs_render_workspace_bytes)");
  if (n == 0) {
    for (int f = 0; f < n_frames; ++f) {
      fill_bg_kernel<<<64, 256, 0, s>>>(images[f], W, H, cams[f].bg[0], cams[f].bg[1], cams[f].bg[2],
                                        aux ? aux->final_T : nullptr, aux ? aux->n_contrib : nullptr,
                                        aux ? aux->n_evaluated : nullptr);
      // counters of an empty frame: zero instances, no overflow
      cudaMemsetAsync((char*)ws + (size_t)f * per, 0, 64, s);
    }
    if (aux && aux->n_instances) cudaMemsetAsync(aux->n_instances, 0, 4, s);
    if (aux && aux->ranges) cudaMemsetAsync(aux->ranges, 0, sizeof(uint32_t) * 2 * ((W + 15) / 16) * ((H + 15) / 16), s);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FGS_OK : cuda_fail(e, "background fill");
  }
  RenderBatch local;
  memset(&local, 0, sizeof(local));
  local.L = make_layout(n, W, H, cap);
  local.n = n;
  local.sh_degree = defs[0].sh_degree;
  local.width = W; local.height = H;
  local.gx = local.L.gx; local.gy = local.L.gy; local.ntiles = local.L.ntiles;
  local.sort_cap = tile_sort_cap();
  local.cull = blend_cull();
  local.agg_tiles = agg_tiles();
  local.radix_mode = local.L.ntiles <= kRxMaxTiles ? radix_mode() : 0;
  local.radix_min_list = radix_min_list();
  local.long_sort = long_sort();
  local.tile_cull = tile_cull();
  if (local.tile_cull) local.radix_mode = 0;   // the radix path emits whole rects
  local.debug = aux != nullptr;
  local.blend_work = aux ? (unsigned long long*)aux->blend_work : nullptr;
  local.ws_stride = per;
  for (int f0 = 0; f0 < n_frames; f0 += kMaxFrames) {
    local.n_frames = std::min(kMaxFrames, n_frames - f0);
    local.ws = (char*)ws + (size_t)f0 * per;
    for (int f = 0; f < local.n_frames; ++f) {
      const fgs_camera& c = cams[f0 + f];
      FrameCam& fc = local.cam[f];
      memcpy(fc.R, c.R, sizeof(fc.R));
      memcpy(fc.t, c.t, sizeof(fc.t));
      fc.fx = c.fx; fc.fy = c.fy; fc.cx = c.cx; fc.cy = c.cy;
      memcpy(fc.bg, c.bg, sizeof(fc.bg));
      const fgs_deformed& d = defs[f0 + f];
      local.means[f] = d.means; local.log_scales[f] = d.log_scales; local.quats[f] = d.quats;
      local.opacity[f] = d.opacity_logits; local.sh[f] = d.sh;
      local.image[f] = images[f0 + f];
      local.final_T[f] = (aux && f0 + f == 0) ? aux->final_T : nullptr;
      local.n_contrib[f] = (aux && f0 + f == 0) ? aux->n_contrib : nullptr;
      local.n_eval[f] = (aux && f0 + f == 0) ? aux->n_evaluated : nullptr;
    }
    cudaError_t e = launch_render(local, s);
    if (e != cudaSuccess) return cuda_fail(e, "render launch");
    if (aux && f0 == 0) {
      e = launch_debug_copy(local, *aux, s);
      if (e != cudaSuccess) return cuda_fail(e, "debug copy");
    }
  }
  return FGS_OK;
}

struct ProfRec { int stage; cudaEvent_t a, b; };
struct Profiler {
  std::mutex mu;
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<ProfRec> pending;
  cudaEvent_t open[FGS_N_STAGES] = {};
  double ms[FGS_N_STAGES] = {};
  int64_t count[FGS_N_STAGES] = {};
  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};
Profiler& prof() { static Profiler p; return p; }
std::atomic<int64_t> g_launches{0};

}  // namespace

void prof_mark(int stage, bool begin, cudaStream_t s) {
  Profiler& P = prof();
  if (!P.on || stage < 0 || stage >= FGS_N_STAGES) return;
  std::lock_guard<std::mutex> lk(P.mu);
  cudaEvent_t e = P.get();
  cudaEventRecord(e, s);
  if (begin) {
    P.open[stage] = e;
  } else if (P.open[stage]) {
    P.pending.push_back({stage, P.open[stage], e});
    P.open[stage] = nullptr;
  }
}

void note_launches(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

WsLayout make_layout(int64_t n, int width, int height, int64_t cap) {
  WsLayout L;
  L.n = n; L.cap = cap; L.width = width; L.height = height;
  L.gx = (width + kTile - 1) / kTile;
  L.gy = (height + kTile - 1) / kTile;
  L.ntiles = L.gx * L.gy;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = align256(o + bytes); return at; };
  const size_t nn = (size_t)std::max<int64_t>(n, 1);
  const size_t cc = (size_t)std::max<int64_t>(cap, 1);
  const size_t nt = (size_t)L.ntiles;
  L.cnt = take(64);
  L.keys = take(4 * nn);
  L.tt = take(4 * nn);
  L.rect = take(8 * nn);
  L.rec = take(48 * nn);
  L.radii = take(4 * nn);
  L.tile_count = take(4 * nt);
  L.cursor = take(4 * nt);
  L.ranges = take(8 * nt);
  L.long_list = take(4 * nt);
  L.order = take(4 * nt);
  L.inst = take(8 * cc);
  L.inst2 = take(8 * cc);
  L.rx_blocks = (int)((std::max<int64_t>(std::max<int64_t>(n, cap), 1) + kRxItems - 1) / kRxItems);
  L.rx_hist = take(4 * 256 * (size_t)L.rx_blocks);
  L.rx_dtot = take(4 * 256);
  L.rx_bsum = take(4 * (size_t)((std::max<int64_t>(n, 1) + kRxItems - 1) / kRxItems));
  L.tmask = take(8 * nn);
  L.total = o;
  return L;
}

int64_t capacity_for(int64_t n, int width, int height, size_t bytes) {
  // total(cap) is non-decreasing in cap: binary search the largest cap that fits.
  if (make_layout(n, width, height, 1).total > bytes) return 0;
  int64_t lo = 1, hi = (int64_t)(bytes / 16) + 1;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo + 1) / 2;
    if (make_layout(n, width, height, mid).total <= bytes) lo = mid; else hi = mid - 1;
  }
  return std::min<int64_t>(lo, (int64_t)0xFFFFFFF0);
}

namespace {
std::atomic<int> g_tile_sort_cap{kBlendSortMax};
std::atomic<int> g_blend_cull{1};
std::atomic<int> g_agg_tiles{kAggTilesMax};
std::atomic<int> g_radix_mode{0};
std::atomic<int> g_radix_min_list{kRadixMinListDefault};
std::atomic<int> g_long_sort{1};
std::atomic<int> g_tile_cull{0};
}
int tile_sort_cap() { return g_tile_sort_cap.load(std::memory_order_relaxed); }
int blend_cull() { return g_blend_cull.load(std::memory_order_relaxed); }
int agg_tiles() { return g_agg_tiles.load(std::memory_order_relaxed); }
int radix_mode() { return g_radix_mode.load(std::memory_order_relaxed); }
int radix_min_list() { return g_radix_min_list.load(std::memory_order_relaxed); }
int long_sort() { return g_long_sort.load(std::memory_order_relaxed); }
int tile_cull() { return g_tile_cull.load(std::memory_order_relaxed); }

}  // namespace fgs

using namespace fgs;

extern "C" {

int fgs_deform(const fgs_gaussians* g, const fgs_hexplanes* field, const fgs_mlp* mlp, float t,
               fgs_deformed* out, fgs_stream_t stream) {
  if (!g) return fail(FGS_E_INVALID, "gaussians is NULL");
  return deform_impl(g, field, mlp, &t, 1, 0, g->n, out, (cudaStream_t)stream);
}

int fgs_deform_range(const fgs_gaussians* g, const fgs_hexplanes* field, const fgs_mlp* mlp, float t,
                     int64_t begin, int64_t end, fgs_deformed* out, fgs_stream_t stream) {
  return deform_impl(g, field, mlp, &t, 1, begin, end, out, (cudaStream_t)stream);
}

int fgs_deform_range_peers(const fgs_gaussians* g, const fgs_hexplanes* field, const fgs_mlp* mlp, float t,
                           int64_t begin, int64_t end, fgs_deformed* out, const int64_t* peer_offsets,
                           int32_t n_peers, fgs_stream_t stream) {
  if (!peer_offsets) return fail(FGS_E_INVALID, "peer_offsets is NULL");
  return deform_impl(g, field, mlp, &t, 1, begin, end, out, (cudaStream_t)stream, peer_offsets, n_peers);
}

int fgs_deform_batch(const fgs_gaussians* g, const fgs_hexplanes* field, const fgs_mlp* mlp, const float* ts,
                     int32_t n_t, fgs_deformed* outs, fgs_stream_t stream) {
  if (!g) return fail(FGS_E_INVALID, "gaussians is NULL");
  return deform_impl(g, field, mlp, ts, n_t, 0, g->n, outs, (cudaStream_t)stream);
}

size_t fgs_render_workspace_bytes(int64_t n, int32_t width, int32_t height, int64_t max_instances) {
  if (n < 0 || width <= 0 || height <= 0 || max_instances < 1) return 0;
  return make_layout(n, width, height, max_instances).total;
}

int fgs_render(const fgs_camera* cam, const fgs_deformed* g, float* image, void* ws, size_t ws_bytes,
               fgs_stream_t stream) {
  return render_impl(cam, g, &image, 1, ws, ws_bytes, nullptr, (cudaStream_t)stream);
}

int fgs_render_batch(const fgs_camera* cams, const fgs_deformed* defs, float* const* images, int32_t n_frames,
                     void* ws, size_t ws_bytes, fgs_stream_t stream) {
  return render_impl(cams, defs, images, n_frames, ws, ws_bytes, nullptr, (cudaStream_t)stream);
}

int fgs_render_debug(const fgs_camera* cam, const fgs_deformed* g, float* image, void* ws, size_t ws_bytes,
                     const fgs_render_aux* aux, fgs_stream_t stream) {
  if (!aux) return fail(FGS_E_INVALID, "aux is NULL");
  return render_impl(cam, g, &image, 1, ws, ws_bytes, aux, (cudaStream_t)stream);
}

int fgs_render_status(const void* ws, size_t ws_bytes, int32_t n_frames, fgs_stream_t stream) {
  if (!ws || n_frames <= 0) return fail(FGS_E_INVALID, "bad workspace/n_frames");
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "stream sync");
  const size_t per = (ws_bytes / (size_t)n_frames) & ~(size_t)255;
  for (int f = 0; f < n_frames; ++f) {
    uint32_t flag = 0;
    e = cudaMemcpy(&flag, (const char*)ws + (size_t)f * per + 8, 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "status read");
    if (flag) return fail(FGS_E_CAPACITY, "instance capacity overflow in frame " + std::to_string(f));
  }
  return FGS_OK;
}

namespace fgs {
namespace {
// Deform the distinct times of a frame batch once each (frames sharing a time — several views of one
// instant — share its G'); fills `render_defs` with the deformed set each frame renders.
int frames_deform(const fgs_gaussians* g, const fgs_hexplanes* h, const fgs_mlp* m, const float* ts, int F,
                  fgs_deformed* defs, cudaStream_t s, std::vector<fgs_deformed>& render_defs) {
  FGS_CHECK(ts && defs && F >= 0, "null times/outputs");
  int rc;
  for (int f = 0; f < F; ++f)
    if ((rc = check_deformed(&defs[f], g->n, g->sh_degree, true)) != FGS_OK) return rc;
  std::vector<float> ut;
  std::vector<fgs_deformed> uo;
  std::vector<int> map(F);
  for (int f = 0; f < F; ++f) {
    int j = 0;
    while (j < (int)ut.size() && memcmp(&ut[j], &ts[f], sizeof(float)) != 0) ++j;
    if (j == (int)ut.size()) { ut.push_back(ts[f]); uo.push_back(defs[f]); }
    map[f] = j;
  }
  rc = deform_impl(g, h, m, ut.data(), (int)ut.size(), 0, g->n, uo.data(), s);
  if (rc != FGS_OK) return rc;
  render_defs.resize(F);
  for (int f = 0; f < F; ++f) render_defs[f] = uo[map[f]];
  return FGS_OK;
}
}  // namespace
}  // namespace fgs

int fgs_frames(const fgs_gaussians* g, const fgs_hexplanes* field, const fgs_mlp* mlp, const float* ts,
               const fgs_camera* cams, int32_t n_frames, fgs_deformed* defs_scratch, float* const* images,
               void* ws, size_t ws_bytes, fgs_stream_t stream) {
  if (!g) return fail(FGS_E_INVALID, "gaussians is NULL");
  std::vector<fgs_deformed> rd;
  int rc = frames_deform(g, field, mlp, ts, n_frames, defs_scratch, (cudaStream_t)stream, rd);
  if (rc != FGS_OK) return rc;
  return render_impl(cams, rd.data(), images, n_frames, ws, ws_bytes, nullptr, (cudaStream_t)stream);
}

int fgs_profile_enable(int enable) {
  Profiler& P = prof();
  std::lock_guard<std::mutex> lk(P.mu);
  P.on = enable != 0;
  return FGS_OK;
}

int fgs_profile_read(double* ms, int64_t* launches) {
  Profiler& P = prof();
  std::lock_guard<std::mutex> lk(P.mu);
  for (const ProfRec& r : P.pending) {
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return cuda_fail(e, "profile event sync");
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    P.ms[r.stage] += t;
    P.count[r.stage] += 1;
    P.pool.push_back(r.a);
    P.pool.push_back(r.b);
  }
  P.pending.clear();
  for (int i = 0; i < FGS_N_STAGES; ++i) {
    if (ms) ms[i] = P.ms[i];
    if (launches) launches[i] = P.count[i];
    P.ms[i] = 0.0;
    P.count[i] = 0;
  }
  return FGS_OK;
}

int64_t fgs_launch_count(void) { return g_launches.load(); }

int fgs_set_tuning(int32_t key, int64_t value) {
  switch (key) {
    case FGS_TUNE_TILE_SORT_CAP:
      FGS_CHECK(value >= 1 && value <= kBlendSortMax, "tile sort cap must be in [1, 1024]");
      g_tile_sort_cap.store((int)value);
      return FGS_OK;
    case FGS_TUNE_BLEND_CULL:
      FGS_CHECK(value == 0 || value == 1, "blend cull must be 0 or 1");
      g_blend_cull.store((int)value);
      return FGS_OK;
    case FGS_TUNE_AGG_TILES:
      FGS_CHECK(value >= 1 && value <= kAggTilesMax, "aggregation limit must be in [1, 4096]");
      g_agg_tiles.store((int)value);
      return FGS_OK;
    case FGS_TUNE_RADIX:
      FGS_CHECK(value >= 0 && value <= 2, "radix mode must be 0, 1 or 2");
      g_radix_mode.store((int)value);
      return FGS_OK;
    case FGS_TUNE_RADIX_MIN_LIST:
      FGS_CHECK(value >= 1 && value <= (1 << 20), "radix threshold must be in [1, 2^20]");
      g_radix_min_list.store((int)value);
      return FGS_OK;
    case FGS_TUNE_LONG_SORT:
      FGS_CHECK(value == 0 || value == 1, "long sort mode must be 0 or 1");
      g_long_sort.store((int)value);
      return FGS_OK;
    case FGS_TUNE_TILE_CULL:
      FGS_CHECK(value == 0 || value == 1, "tile cull must be 0 or 1");
      g_tile_cull.store((int)value);
      return FGS_OK;
    default:
      return fail(FGS_E_INVALID, "unknown tuning key");
  }
}

int64_t fgs_get_tuning(int32_t key) {
  if (key == FGS_TUNE_TILE_SORT_CAP) return tile_sort_cap();
  if (key == FGS_TUNE_BLEND_CULL) return blend_cull();
  if (key == FGS_TUNE_AGG_TILES) return agg_tiles();
  if (key == FGS_TUNE_RADIX) return radix_mode();
  if (key == FGS_TUNE_RADIX_MIN_LIST) return radix_min_list();
  if (key == FGS_TUNE_LONG_SORT) return long_sort();
  if (key == FGS_TUNE_TILE_CULL) return tile_cull();
  return -1;
}

// ---- end to end with host buffers -------------------------------------------------------------
namespace {
struct HostLayout {
  size_t means, log_scales, quats, opac, sh, planes[FGS_MAX_SCALES][FGS_PLANES], mlp[12], defs, images, render;
  size_t plane_bytes[FGS_MAX_SCALES][FGS_PLANES], mlp_bytes[12];
  size_t per_def, def_sh, def_opac, per_img, per_render, total;
};
HostLayout host_layout(const fgs_gaussians* g, const fgs_hexplanes* h, const fgs_mlp* m, int F, int W, int H,
                       int64_t cap) {
  HostLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = align256(o + bytes); return at; };
  const size_t n = (size_t)g->n, K = (size_t)(g->sh_degree + 1) * (g->sh_degree + 1);
  L.means = take(12 * n); L.log_scales = take(12 * n); L.quats = take(16 * n); L.opac = take(4 * n);
  L.sh = take(12 * K * n);
  for (int l = 0; l < h->n_scales; ++l)
    for (int p = 0; p < FGS_PLANES; ++p) {
      const size_t nb = p < 3 ? (size_t)h->res[l] : (size_t)h->t_res;
      L.plane_bytes[l][p] = nb * (size_t)h->res[l] * (size_t)h->feat * 4;
      L.planes[l][p] = take(L.plane_bytes[l][p]);
    }
  const size_t Wd = (size_t)m->width, In = (size_t)m->in_dim;
  const size_t hc = m->w_c ? 3 * K : 0, ha = m->w_a ? 1 : 0;
  const size_t mb[12] = {Wd * In * 4, Wd * 4, 3 * Wd * 4, 12, 4 * Wd * 4, 16, 3 * Wd * 4, 12,
                         hc * Wd * 4, hc * 4, ha * Wd * 4, ha * 4};
  for (int i = 0; i < 12; ++i) { L.mlp_bytes[i] = mb[i]; L.mlp[i] = take(mb[i]); }
  // per frame: X', s', r' and, with the P:1232 decoders, the deformed SH / opacity
  L.def_sh = align256(12 * n) * 2 + align256(16 * n);
  L.def_opac = L.def_sh + (hc ? align256(4 * hc * n) : 0);
  L.per_def = L.def_opac + (ha ? align256(4 * n) : 0);
  L.defs = take(L.per_def * (size_t)F);
  L.per_img = align256((size_t)3 * W * H * 4);
  L.images = take(L.per_img * (size_t)F);
  L.per_render = make_layout(g->n, W, H, cap).total;
  L.render = take(L.per_render * (size_t)F);
  L.total = o;
  return L;
}
}  // namespace

namespace {
constexpr int kHostChunkFrames = 4;
// Side streams + events of ONE fgs_frames_host call (`up`: the SH upload, `copy`: the image downloads —
// two streams, so that when calls on different caller streams are in flight together the upload of one
// never queues behind the downloads of another).  Calls take a set from a per-device free list for
// the duration of their enqueue and give it back before returning, so concurrent calls (distinct
// workspaces, any threads) never share a stream or an event while enqueueing.  Re-recording an event
// after the set is returned does not affect the waits already enqueued on it (a wait captures the
// event's state at enqueue time), so a set is reusable as soon as its call has returned.
struct CopySet {
  int dev = -1;
  cudaStream_t copy = nullptr, up = nullptr;
  cudaEvent_t done = nullptr, fork = nullptr, sh_done = nullptr;
  std::vector<cudaEvent_t> evs;
  cudaError_t event(int i, cudaEvent_t* out) {
    while ((int)evs.size() <= i) {
      cudaEvent_t e = nullptr;
      const cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      if (r != cudaSuccess) return r;
      evs.push_back(e);
    }
    *out = evs[i];
    return cudaSuccess;
  }
};
struct CopyPool {
  std::mutex mu;
  std::vector<CopySet*> free;    // sets of any device; a call takes one of its current device
};
CopyPool& copy_pool() { static CopyPool p; return p; }   // sets live for the process (never freed)

cudaError_t acquire_copy_set(CopySet** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  CopyPool& P = copy_pool();
  {
    std::lock_guard<std::mutex> lk(P.mu);
    for (size_t i = 0; i < P.free.size(); ++i)
      if (P.free[i]->dev == dev) {
        *out = P.free[i];
        P.free.erase(P.free.begin() + (ptrdiff_t)i);
        return cudaSuccess;
      }
  }
  CopySet* c = new CopySet();
  c->dev = dev;
  e = cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->up, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->sh_done, cudaEventDisableTiming);
  if (e != cudaSuccess) return e;   // (leaks the partial set; only on a failing device)
  *out = c;
  return cudaSuccess;
}
void release_copy_set(CopySet* c) {
  CopyPool& P = copy_pool();
  std::lock_guard<std::mutex> lk(P.mu);
  P.free.push_back(c);
}
// RAII: the set goes back to the pool on every return path of fgs_frames_host
struct CopySetLease {
  CopySet* c = nullptr;
  ~CopySetLease() { if (c) release_copy_set(c); }
};
}  // namespace

size_t fgs_frames_host_workspace_bytes(const fgs_gaussians* g, const fgs_hexplanes* field, const fgs_mlp* mlp,
                                       int32_t n_frames, int32_t width, int32_t height, int64_t max_instances) {
  if (!g || !field || !mlp || n_frames <= 0 || width <= 0 || height <= 0 || max_instances < 1) return 0;
  if (g->n < 0 || field->n_scales < 1 || field->n_scales > FGS_MAX_SCALES) return 0;
  return host_layout(g, field, mlp, n_frames, width, height, max_instances).total;
}

int fgs_frames_host(const fgs_gaussians* gh, const fgs_hexplanes* hh, const fgs_mlp* mh, const float* ts,
                    const fgs_camera* cams, int32_t F, float* const* images_host, void* dev_ws,
                    size_t dev_ws_bytes, fgs_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  FGS_CHECK(gh && hh && mh && ts && cams && images_host && dev_ws && F > 0, "null argument");
  int rc;
  if ((rc = check_gaussians(gh)) != FGS_OK) return rc;
  if ((rc = check_field(hh, mh)) != FGS_OK) return rc;
  if ((rc = check_camera(&cams[0])) != FGS_OK) return rc;
  for (int f = 0; f < F; ++f) FGS_CHECK(images_host[f], "null host image");
  const int W = cams[0].width, H = cams[0].height;
  const HostLayout L0 = host_layout(gh, hh, mh, F, W, H, 1);
  FGS_CHECK(dev_ws_bytes >= L0.total, "device workspace too small");
  const size_t fixed = L0.total - L0.per_render * (size_t)F;
  const int64_t cap = capacity_for(gh->n, W, H, ((dev_ws_bytes - fixed) / (size_t)F) & ~(size_t)255);
  FGS_CHECK(cap > 0, "device workspace too small");
  const HostLayout L = host_layout(gh, hh, mh, F, W, H, cap);
  char* d = (char*)dev_ws;
  const size_t n = (size_t)gh->n, K = (size_t)(gh->sh_degree + 1) * (gh->sh_degree + 1);
  CopySetLease lease;
  {
    const cudaError_t ce = acquire_copy_set(&lease.c);
    if (ce != cudaSuccess) return cuda_fail(ce, "copy stream setup");
  }
  CopySet& cs = *lease.c;
  auto h2d = [&](size_t off, const void* src, size_t bytes) {
    return bytes ? cudaMemcpyAsync(d + off, src, bytes, cudaMemcpyHostToDevice, s) : cudaSuccess;
  };
  cudaError_t e = cudaSuccess;
  // The SH coefficients (the bulk of the model, needed only from preprocess on) are uploaded on the
  // side stream while the deformation runs, unless phi_C reads them in the deform.  They are queued
  // AFTER the deformation's inputs so the two uploads do not share the link: the deformation starts
  // once its ~14 MB (D) are on the device, and the SH upload hides behind it.
  const bool sh_side = n && !mh->w_c;
  if (n) {
    e = h2d(L.means, gh->means, 12 * n);
    if (e == cudaSuccess) e = h2d(L.log_scales, gh->log_scales, 12 * n);
    if (e == cudaSuccess) e = h2d(L.quats, gh->quats, 16 * n);
    if (e == cudaSuccess) e = h2d(L.opac, gh->opacity_logits, 4 * n);
    if (e == cudaSuccess && !sh_side) e = h2d(L.sh, gh->sh, 12 * K * n);
  }
  fgs_hexplanes hd = *hh;
  for (int l = 0; l < hh->n_scales && e == cudaSuccess; ++l)
    for (int p = 0; p < FGS_PLANES && e == cudaSuccess; ++p) {
      e = h2d(L.planes[l][p], hh->planes[l][p], L.plane_bytes[l][p]);
      hd.planes[l][p] = (const float*)(d + L.planes[l][p]);
    }
  fgs_mlp md = *mh;
  const float* srcs[12] = {mh->w_d, mh->b_d, mh->w_x, mh->b_x, mh->w_r, mh->b_r, mh->w_s, mh->b_s,
                           mh->w_c, mh->b_c, mh->w_a, mh->b_a};
  const float** dsts[12] = {&md.w_d, &md.b_d, &md.w_x, &md.b_x, &md.w_r, &md.b_r, &md.w_s, &md.b_s,
                            &md.w_c, &md.b_c, &md.w_a, &md.b_a};
  for (int i = 0; i < 12 && e == cudaSuccess; ++i) {
    if (!srcs[i]) { *dsts[i] = nullptr; continue; }
    e = h2d(L.mlp[i], srcs[i], L.mlp_bytes[i]);
    *dsts[i] = (const float*)(d + L.mlp[i]);
  }
  if (e != cudaSuccess) return cuda_fail(e, "host->device copy");
  if (sh_side) {
    if ((e = cudaEventRecord(cs.fork, s)) != cudaSuccess) return cuda_fail(e, "event record");
    if ((e = cudaStreamWaitEvent(cs.up, cs.fork, 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
    if ((e = cudaMemcpyAsync(d + L.sh, gh->sh, 12 * K * n, cudaMemcpyHostToDevice, cs.up)) != cudaSuccess)
      return cuda_fail(e, "host->device copy");
    if ((e = cudaEventRecord(cs.sh_done, cs.up)) != cudaSuccess) return cuda_fail(e, "event record");
  }
  fgs_gaussians gd = *gh;
  gd.means = (const float*)(d + L.means); gd.log_scales = (const float*)(d + L.log_scales);
  gd.quats = (const float*)(d + L.quats); gd.opacity_logits = (const float*)(d + L.opac);
  gd.sh = (const float*)(d + L.sh);
  std::vector<fgs_deformed> defs(F);
  std::vector<float*> imgs(F);
  for (int f = 0; f < F; ++f) {
    char* base = d + L.defs + (size_t)f * L.per_def;
    defs[f].n = gh->n; defs[f].sh_degree = gh->sh_degree;
    defs[f].means = (float*)base;
    defs[f].log_scales = (float*)(base + align256(12 * n));
    defs[f].quats = (float*)(base + 2 * align256(12 * n));
    defs[f].opacity_logits = mh->w_a ? (float*)(base + L.def_opac) : const_cast<float*>(gd.opacity_logits);
    defs[f].sh = mh->w_c ? (float*)(base + L.def_sh) : const_cast<float*>(gd.sh);
    imgs[f] = (float*)(d + L.images + (size_t)f * L.per_img);
  }
  // Deform all frames in one launch (the spatial-plane work is shared across times), then render in
  // growing chunks; the device->host copy of chunk c runs on the side stream while chunk c+1 renders.
  std::vector<fgs_deformed> rdefs;
  rc = frames_deform(&gd, &hd, &md, ts, F, defs.data(), s, rdefs);
  if (rc != FGS_OK) return rc;
  if (sh_side && (e = cudaStreamWaitEvent(s, cs.sh_done, 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
  // chunks of 1, 2, 4, 4, ... frames: the first image leaves the device as early as possible
  int ci = 0;
  for (int f0 = 0, chunk = 1; f0 < F; f0 += chunk, chunk = std::min(2 * chunk, kHostChunkFrames), ++ci) {
    const int nf = std::min(chunk, F - f0);
    rc = render_impl(cams + f0, rdefs.data() + f0, imgs.data() + f0, nf, d + L.render + (size_t)f0 * L.per_render,
                     L.per_render * (size_t)nf, nullptr, s);
    if (rc != FGS_OK) return rc;
    cudaEvent_t ev = nullptr;
    if ((e = cs.event(ci, &ev)) != cudaSuccess) return cuda_fail(e, "event create");
    if ((e = cudaEventRecord(ev, s)) != cudaSuccess) return cuda_fail(e, "event record");
    if ((e = cudaStreamWaitEvent(cs.copy, ev, 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
    for (int f = f0; f < f0 + nf; ++f) {
      e = cudaMemcpyAsync(images_host[f], imgs[f], (size_t)3 * W * H * 4, cudaMemcpyDeviceToHost, cs.copy);
      if (e != cudaSuccess) return cuda_fail(e, "device->host copy");
    }
  }
  // the caller's stream covers the copies: it waits for the side stream's last copy
  if ((e = cudaEventRecord(cs.done, cs.copy)) != cudaSuccess) return cuda_fail(e, "event record");
  if ((e = cudaStreamWaitEvent(s, cs.done, 0)) != cudaSuccess) return cuda_fail(e, "stream wait");
  return FGS_OK;
}

int fgs_frames_host_status(const fgs_gaussians* gh, const fgs_hexplanes* hh, const fgs_mlp* mh,
                           const fgs_camera* cams, int32_t F, const void* dev_ws, size_t dev_ws_bytes,
                           fgs_stream_t stream) {
  FGS_CHECK(gh && hh && mh && cams && dev_ws && F > 0, "null argument");
  int rc;
  if ((rc = check_gaussians(gh)) != FGS_OK) return rc;
  if ((rc = check_field(hh, mh)) != FGS_OK) return rc;
  if ((rc = check_camera(&cams[0])) != FGS_OK) return rc;
  const int W = cams[0].width, H = cams[0].height;
  // the same layout fgs_frames_host derived from these arguments
  const HostLayout L0 = host_layout(gh, hh, mh, F, W, H, 1);
  FGS_CHECK(dev_ws_bytes >= L0.total, "device workspace too small");
  const size_t fixed = L0.total - L0.per_render * (size_t)F;
  const int64_t cap = capacity_for(gh->n, W, H, ((dev_ws_bytes - fixed) / (size_t)F) & ~(size_t)255);
  FGS_CHECK(cap > 0, "device workspace too small");
  const HostLayout L = host_layout(gh, hh, mh, F, W, H, cap);
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "stream sync");
  if (gh->n == 0) return FGS_OK;
  for (int f = 0; f < F; ++f) {
    uint32_t flag = 0;
    e = cudaMemcpy(&flag, (const char*)dev_ws + L.render + (size_t)f * L.per_render + 8, 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "status read");
    if (flag) return fail(FGS_E_CAPACITY, "instance capacity overflow in frame " + std::to_string(f));
  }
  return FGS_OK;
}

// ---- training side ----------------------------------------------------------------------------
int fgs_l1_loss(const float* image, const float* target, int32_t width, int32_t height, float* dL_dimage,
                double* partials, float* loss, fgs_stream_t stream) {
  FGS_CHECK(image && target && partials && loss, "null argument");
  FGS_CHECK(width > 0 && height > 0, "bad image size");
  const cudaError_t e = launch_l1(image, target, (int64_t)3 * width * height, dL_dimage, partials, loss,
                                  (cudaStream_t)stream);
  return e == cudaSuccess ? FGS_OK : cuda_fail(e, "l1 loss");
}

int fgs_tv_loss(const fgs_hexplanes* h, float weight, fgs_field_grads* grads, double* partials, float* loss,
                fgs_stream_t stream) {
  FGS_CHECK(h && partials && loss, "null argument");
  FGS_CHECK(h->n_scales >= 1 && h->n_scales <= FGS_MAX_SCALES, "n_scales must be in [1,4]");
  FGS_CHECK(h->feat >= 1 && h->t_res >= 2 && isfinite(weight), "bad field / weight");
  TvArgs a;
  memset(&a, 0, sizeof(a));
  a.feat = h->feat;
  a.weight = weight;
  a.partials = partials;
  a.loss = loss;
  for (int l = 0; l < h->n_scales; ++l) {
    FGS_CHECK(h->res[l] >= 2, "res[l] must be >= 2");
    for (int q = 0; q < FGS_PLANES; ++q) {
      FGS_CHECK(h->planes[l][q], "null plane");
      const int k = a.n_planes++;
      a.planes[k] = h->planes[l][q];
      a.na[k] = h->res[l];
      a.nb[k] = q < 3 ? h->res[l] : h->t_res;
      a.grads[k] = grads ? grads->planes[l][q] : nullptr;
    }
  }
  const cudaError_t e = launch_tv(a, (cudaStream_t)stream);
  return e == cudaSuccess ? FGS_OK : cuda_fail(e, "tv loss");
}

size_t fgs_render_backward_scratch_bytes(int64_t n) {
  return n < 0 ? 0 : (size_t)std::max<int64_t>(n, 1) * 9 * sizeof(unsigned long long);
}

int fgs_render_backward(const fgs_camera* cam, const fgs_deformed* g, const float* image, const float* dL_dimage,
                        const void* ws, size_t ws_bytes, void* scratch, size_t scratch_bytes,
                        const fgs_gaussian_grads* dg, fgs_stream_t stream) {
  int rc;
  if ((rc = check_camera(cam)) != FGS_OK) return rc;
  if ((rc = check_deformed(g, g ? g->n : 0, g ? g->sh_degree : 0, false)) != FGS_OK) return rc;
  FGS_CHECK(g->n >= 0 && g->n < ((int64_t)1 << 31) && g->sh_degree >= 0 && g->sh_degree <= 3, "bad deformed set");
  FGS_CHECK(image && dL_dimage && ws && scratch && dg, "null argument");
  FGS_CHECK(scratch_bytes >= fgs_render_backward_scratch_bytes(g->n), "scratch too small");
  const int64_t n = g->n;
  if (n == 0) return FGS_OK;
  FGS_CHECK(dg->means && dg->log_scales && dg->quats && dg->opacity_logits && dg->sh, "null gradient array");
  const int W = cam->width, H = cam->height;
  const size_t per = ws_bytes & ~(size_t)255;
  const int64_t cap = capacity_for(n, W, H, per);
  FGS_CHECK(cap > 0, "workspace too small (see fgs_render_workspace_bytes)");
  RenderBatch b;
  memset(&b, 0, sizeof(b));
  b.L = make_layout(n, W, H, cap);
  b.n = n; b.n_frames = 1; b.sh_degree = g->sh_degree;
  b.width = W; b.height = H; b.gx = b.L.gx; b.gy = b.L.gy; b.ntiles = b.L.ntiles;
  b.ws = (char*)const_cast<void*>(ws); b.ws_stride = per;
  FrameCam& fc = b.cam[0];
  memcpy(fc.R, cam->R, sizeof(fc.R)); memcpy(fc.t, cam->t, sizeof(fc.t));
  fc.fx = cam->fx; fc.fy = cam->fy; fc.cx = cam->cx; fc.cy = cam->cy;
  memcpy(fc.bg, cam->bg, sizeof(fc.bg));
  b.means[0] = g->means; b.log_scales[0] = g->log_scales; b.quats[0] = g->quats;
  b.opacity[0] = g->opacity_logits; b.sh[0] = g->sh;
  const cudaError_t e = launch_render_backward(b, image, dL_dimage, (unsigned long long*)scratch, dg->means,
                                               dg->log_scales, dg->quats, dg->opacity_logits, dg->sh,
                                               (cudaStream_t)stream);
  return e == cudaSuccess ? FGS_OK : cuda_fail(e, "render backward");
}

size_t fgs_deform_backward_scratch_bytes(const fgs_hexplanes* field, const fgs_mlp* mlp) {
  if (!field || !mlp || field->n_scales < 1 || field->n_scales > FGS_MAX_SCALES) return 0;
  DeformBatch p;
  memset(&p, 0, sizeof(p));
  p.n_scales = field->n_scales; p.feat = field->feat; p.t_res = field->t_res;
  for (int l = 0; l < field->n_scales; ++l) p.res[l] = field->res[l];
  p.width = mlp->width; p.in_dim = mlp->in_dim;
  p.w_c = mlp->w_c; p.w_a = mlp->w_a;
  p.n_c = mlp->w_c ? 3 * 16 : 0;     // sized for SH degree 3 (the largest K); exact for lower degrees
  return deform_backward_acc_elems(p) * sizeof(unsigned long long);
}

int fgs_deform_backward(const fgs_gaussians* g, const fgs_hexplanes* h, const fgs_mlp* m, float t,
                        const fgs_gaussian_grads* dd, const fgs_gaussian_grads* dc, const fgs_field_grads* df,
                        void* scratch, size_t scratch_bytes, fgs_stream_t stream) {
  int rc;
  if ((rc = check_gaussians(g)) != FGS_OK) return rc;
  if ((rc = check_field(h, m)) != FGS_OK) return rc;
  FGS_CHECK(isfinite(t) && t >= 0.f && t <= 1.f, "t must be finite and in [0,1]");
  FGS_CHECK(dd && dc && df && scratch, "null argument");
  FGS_CHECK(scratch_bytes >= fgs_deform_backward_scratch_bytes(h, m), "scratch too small");
  for (int l = 0; l < h->n_scales; ++l)
    for (int q = 0; q < FGS_PLANES; ++q) FGS_CHECK(df->planes[l][q], "null plane gradient");
  FGS_CHECK(df->w_d && df->b_d && df->w_x && df->b_x && df->w_r && df->b_r && df->w_s && df->b_s,
            "null MLP gradient");
  if (m->w_c) FGS_CHECK(df->w_c && df->b_c, "phi_C: null w_c / b_c gradient");
  if (m->w_a) FGS_CHECK(df->w_a && df->b_a, "phi_alpha: null w_a / b_a gradient");
  if (g->n > 0) {
    FGS_CHECK(dd->means && dd->log_scales && dd->quats && dc->means && dc->log_scales && dc->quats,
              "null per-Gaussian gradient");
    if (m->w_c) FGS_CHECK(dd->sh && dc->sh, "phi_C: null SH gradient (d_deformed.sh in, d_canonical.sh out)");
    if (m->w_a) FGS_CHECK(dd->opacity_logits && dc->opacity_logits, "phi_alpha: null opacity gradient");
  }
  DeformBatch p;
  fill_deform(p, g, h, m);
  p.begin = 0; p.end = g->n; p.n_t = 1; p.t[0] = t;
  float* pg[FGS_MAX_SCALES * FGS_PLANES] = {};
  for (int l = 0; l < h->n_scales; ++l)
    for (int q = 0; q < FGS_PLANES; ++q) pg[l * FGS_PLANES + q] = df->planes[l][q];
  float* mg[12] = {df->w_d, df->b_d, df->w_x, df->b_x, df->w_r, df->b_r, df->w_s, df->b_s,
                   df->w_c, df->b_c, df->w_a, df->b_a};
  const cudaError_t e = launch_deform_backward(p, dd->means, dd->log_scales, dd->quats, m->w_c ? dd->sh : nullptr,
                                               m->w_a ? dd->opacity_logits : nullptr, dc->means, dc->log_scales,
                                               dc->quats, m->w_c ? dc->sh : nullptr,
                                               m->w_a ? dc->opacity_logits : nullptr, (unsigned long long*)scratch, pg,
                                               mg, (cudaStream_t)stream);
  return e == cudaSuccess ? FGS_OK : cuda_fail(e, "deform backward");
}

int fgs_adam_step(float* param, const float* grad, float* m, float* v, int64_t n, float lr, float beta1,
                  float beta2, float eps, int32_t step, fgs_stream_t stream) {
  FGS_CHECK(n >= 0, "n must be >= 0");
  if (n == 0) return FGS_OK;
  FGS_CHECK(param && grad && m && v, "null argument");
  FGS_CHECK(step >= 1, "step counts from 1");
  FGS_CHECK(isfinite(lr) && beta1 >= 0.f && beta1 < 1.f && beta2 >= 0.f && beta2 < 1.f && eps > 0.f,
            "bad Adam hyper-parameters");
  const cudaError_t e = launch_adam(param, grad, m, v, n, lr, beta1, beta2, eps, step, (cudaStream_t)stream);
  return e == cudaSuccess ? FGS_OK : cuda_fail(e, "adam");
}

const char* fgs_last_error(void) { return g_err.c_str(); }


const char* fgs_version(void) { return "fgs 0.1 (4D-GS forward, sm_100a)"; }

}  // extern "C"
