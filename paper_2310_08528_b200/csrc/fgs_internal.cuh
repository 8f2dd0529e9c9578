// Internal declarations shared by the sm_100a kernels of libfgs.so (never by the oracle).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fgs.h"

// Checked build (libfgs_checked.so, build.py --checked): device-side bounds / invariant assertions on
// the shared-memory, TMEM and workspace indices of every kernel, and a watchdog on every mbarrier wait.
// A failed check prints its condition and traps (the launch fails with an error the tests see).  The
// normal build compiles every FGS_DCHECK to nothing.  (compute-sanitizer is closed on the GPU pool this
// was developed on; this is its stand-in — DESIGN.md §6.)
#ifdef FGS_CHECKED
#include <stdio.h>
#define FGS_DCHECK(cond)                                                                               \
  do {                                                                                                 \
    if (!(cond)) {                                                                                     \
      printf("FGS_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x,   \
             (int)threadIdx.x, #cond);                                                                 \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define FGS_DCHECK(cond) ((void)0)
#endif

namespace fgs {

constexpr int kTile = FGS_TILE;              // 16x16 pixel tiles ([3dgs] rasterizer, reading R8)
constexpr int kMaxFrames = 32;               // frames per launch (kernel-parameter table)
constexpr int kMaxPeers = 8;                 // replicas of the deform outputs (fgs_deform_range_peers)
constexpr int kScanThreads = 1024;           // tile-count scan CTA (one per frame)
constexpr int kBlendThreads = 128;           // blend CTA: 4 warps x 8x8 pixel boxes of a 16x16 tile
constexpr int kBlendSortMax = 1024;          // longest tile list one warp sorts (tile_sort_kernel); longer: long_sort_kernel
constexpr int kLargeSortThreads = 256;       // CTA sort of lists longer than the warp-sort cap
constexpr int kRxItems = 4096;               // items per block of the radix binning passes (radix.cu)
constexpr int kRxMaxTiles = 65536;           // tile ids the two 8-bit tile passes cover

// Per-frame workspace layout (all offsets in bytes from the frame's slice, 256-B aligned).
struct WsLayout {
  int64_t n = 0, cap = 0;
  int width = 0, height = 0, gx = 0, gy = 0, ntiles = 0;
  size_t cnt = 0;            // uint32[16]: 0 n, 1 M clamped to cap, 2 overflow flag, 3 M raw, 4 long lists,
                             // 5 (frame 0) long-list claim counter of the batch, 6 / 7 CTAs of
                             // preprocess / duplicate that took the direct-atomics binning path,
                             // 8 the frame takes the radix binning path (radix.cu)
  size_t keys = 0;           // uint32[n] depth key (IEEE bits of fp32 view depth), gid order
  size_t tt = 0;             // uint32[n] tiles_touched
  size_t rect = 0;           // uint2[n]  (x0 | y0<<16, x1 | y1<<16)
  size_t rec = 0;            // float4[n][3] blend records
  size_t radii = 0;          // int32[n]
  size_t tile_count = 0;     // uint32[ntiles] instances per tile (atomics in preprocess)
  size_t cursor = 0;         // uint32[ntiles] scatter cursors
  size_t ranges = 0;         // uint2[ntiles]  [start, end) of each tile's list (clamped to cap)
  size_t long_list = 0;      // uint32[ntiles] tiles whose lists exceed the warp-sort cap (count in cnt[4])
  size_t order = 0;          // uint32[ntiles] tiles by descending list length (blend dispatch order)
  size_t inst = 0;           // uint64[cap] instances (depth_key << 32 | gid), bucketed by tile
  size_t inst2 = 0;          // uint64[cap] scratch of the long-list sort / the radix passes
  int rx_blocks = 0;         // blocks of kRxItems over max(n, cap): the radix histogram stride
  size_t rx_hist = 0;        // uint32[256][rx_blocks] per-block digit counts -> offsets (radix.cu)
  size_t rx_dtot = 0;        // uint32[256] digit totals of a pass
  size_t rx_bsum = 0;        // uint32[ceil(n / kRxItems)] tiles_touched sums of depth-ordered blocks
  size_t tmask = 0;          // uint64[n] tiles of the rect (row-major bit (ty - y0) * w + tx - x0) a Gaussian
                             // stays listed on (FGS_TUNE_TILE_CULL = 1; rects of at most 64 tiles)
  size_t total = 0;
};

WsLayout make_layout(int64_t n, int width, int height, int64_t cap);
// Largest capacity whose layout fits in `bytes` (0 if none).
int64_t capacity_for(int64_t n, int width, int height, size_t bytes);

// Frame batch table passed by value to the render kernels.
struct FrameCam {
  float R[9], t[3];
  float fx, fy, cx, cy;
  float bg[3];
};
struct RenderBatch {
  int n_frames;
  int64_t n;
  int sh_degree;
  int width, height, gx, gy, ntiles;
  int sort_cap;              // lists longer than this are sorted by the global-memory path
  int debug;                 // 1: blend writes each tile's sorted list back (fgs_render_debug)
  int cull;                  // 1: per-warp ellipse cull in the blend (FGS_TUNE_BLEND_CULL), 0: none
  int agg_tiles;             // CTA binning aggregation limit in tiles (FGS_TUNE_AGG_TILES, <= 4096)
  int radix_mode;            // FGS_TUNE_RADIX: 0 per-tile sorts only, 1 auto, 2 radix path for every frame
  int radix_min_list;        // auto: a frame takes the radix path when M >= radix_min_list x tiles
  int long_sort;             // FGS_TUNE_LONG_SORT: 1 bucket pass for long lists, 0 networks + merges
  int tile_cull;             // FGS_TUNE_TILE_CULL: 1 = non-contributing (tile, Gaussian) pairs left out of the lists
  char* ws;                  // frame f slice = ws + f * ws_stride
  size_t ws_stride;
  WsLayout L;
  FrameCam cam[kMaxFrames];
  const float* means[kMaxFrames];
  const float* log_scales[kMaxFrames];
  const float* quats[kMaxFrames];
  const float* opacity[kMaxFrames];
  const float* sh[kMaxFrames];
  float* image[kMaxFrames];
  float* final_T[kMaxFrames];      // optional
  uint32_t* n_contrib[kMaxFrames]; // optional
  uint32_t* n_eval[kMaxFrames];    // optional
  unsigned long long* blend_work;  // optional [2], frame 0 of a debug render
};

// Deformation launch (times batched over frames of the same model).
struct DeformBatch {
  int n_t;
  int64_t begin, end;        // Gaussian range
  const float* means;
  const float* log_scales;
  const float* quats;
  int n_scales, feat, t_res;
  int res[FGS_MAX_SCALES];
  float bmin[3], ext[3];
  const float* planes[FGS_MAX_SCALES][FGS_PLANES];
  int in_dim, width;
  const float *w_d, *b_d, *w_x, *b_x, *w_r, *b_r, *w_s, *b_s;
  const float *w_c, *b_c, *w_a, *b_a;   // optional colour / opacity decoders
  int n_c;                              // 3K when phi_C is present, else 0
  const float* sh_in;                   // canonical SH [n][K][3] and opacity logits [n]
  const float* opac_in;
  float t[kMaxFrames];
  float* out_means[kMaxFrames];
  float* out_log_scales[kMaxFrames];
  float* out_quats[kMaxFrames];
  float* out_sh[kMaxFrames];            // written when phi_C is present
  float* out_opacity[kMaxFrames];       // written when phi_alpha is present
  // means / log_scales / quats are stored n_peer times, replica q at byte offset peer_off[q] from the
  // out_* address (1 replica at offset 0 by default; §8(e2) fused: every rank's gather buffer)
  int n_peer;
  int64_t peer_off[kMaxPeers];
};

// Kernel launchers (return cudaError_t of the launch).
cudaError_t launch_deform_tc3(const DeformBatch& p, cudaStream_t s);  // warp-specialised v3 (deform_tc3.cu)
bool deform_tc3_supported(const DeformBatch& p);
cudaError_t launch_render(const RenderBatch& b, cudaStream_t s);
cudaError_t launch_radix_bin(const RenderBatch& b, cudaStream_t s);
cudaError_t launch_debug_copy(const RenderBatch& b, const fgs_render_aux& aux, cudaStream_t s);

// Training side (backward.cu): losses and gradients (§4.3).
constexpr int kLossPartials = FGS_LOSS_PARTIALS;  // fp64 block partials of a loss (caller scratch)
constexpr int kMaxTvPlanes = FGS_MAX_SCALES * FGS_PLANES;
struct TvArgs {
  int n_planes, feat;
  const float* planes[kMaxTvPlanes];
  int na[kMaxTvPlanes], nb[kMaxTvPlanes];
  int64_t off[kMaxTvPlanes + 1];   // element offsets of the planes in the concatenated index (launch_tv)
  float* grads[kMaxTvPlanes];      // may be NULL (loss only)
  float weight;
  double* partials;
  float* loss;
};
cudaError_t launch_l1(const float* img, const float* tgt, int64_t count, float* grad, double* partials, float* loss,
                      cudaStream_t s);
cudaError_t launch_tv(const TvArgs& a, cudaStream_t s);
cudaError_t launch_render_backward(const RenderBatch& b, const float* image, const float* dimg,
                                   unsigned long long* acc, float* d_means, float* d_log_scales, float* d_quats,
                                   float* d_opacity, float* d_sh, cudaStream_t s);
size_t deform_backward_acc_elems(const DeformBatch& p);
cudaError_t launch_adam(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                        float eps, int32_t t, cudaStream_t s);
cudaError_t launch_deform_backward(const DeformBatch& p, const float* dm, const float* dls, const float* dq,
                                   const float* dsh, const float* dop, float* om, float* ols, float* oq, float* osh,
                                   float* oop, unsigned long long* acc, float* const* plane_grads,
                                   float* const* mlp_grads, cudaStream_t s);

// Tuning knobs (api.cu, fgs_set_tuning).
int tile_sort_cap();
int blend_cull();
int agg_tiles();
int radix_mode();
int radix_min_list();
int long_sort();
int tile_cull();
constexpr int kAggTilesMax = 4096;           // shared histogram of the CTA binning aggregation
constexpr int kRadixMinListDefault = 768;    // FGS_TUNE_RADIX_MIN_LIST default (mean list length)

// Profiling / launch accounting (api.cu).
void prof_mark(int stage, bool begin, cudaStream_t s);
void note_launches(int64_t k);

// Packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2 / FMUL2, two fp32 lanes per instruction, each lane
// rounded exactly as the scalar fmaf / + / * — bit-equal results).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rc, rd;\n"
      "mov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nmov.b64 rc, {%6, %7};\n"
      "fma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rd;\n"
      "mov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\n"
      "add.rn.f32x2 rd, ra, rb;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rd;\n"
      "mov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\n"
      "mul.rn.f32x2 rd, ra, rb;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

// Conservative ellipse-vs-box cull (the blend, render.cu, and the backward's re-walk, backward.cu, cull
// with this same test): bit k set if the Gaussian's alpha may reach 1/255 somewhere in sub-box k (rows
// y0 + 4k .. y0 + 4k + 3 of the warp's 8-wide column [xl, xh], offsets d = pixel - mean), i.e. if the
// minimum of the PSD quadratic q2(d) = qa dx^2 + qb dx dy + qc dy^2 over the box is <= thr.
// The minimum of a convex quadratic over a box lies at d = 0 if the box holds 0, else on a face whose
// half-space excludes 0 (KKT): at most the x-face ex (xl if xl > 0, xh if xh < 0) and the y-face ey.  On
// each face the 1-D minimiser (ratios kx = -qb / 2qa, ky = -qb / 2qc) is clamped to the face.  Branch
// free: both face candidates are always evaluated — with ex = 0 (resp. ey = 0) the "face" is the line
// x = 0 (y = 0) through the box, whose clamped point is still a point of the box, so the minimum of the
// two candidates is exactly the box minimum in every case (0 when the box holds the origin).
template <int NP>
__device__ __forceinline__ void subboxes_reach(float qa, float qb, float qc, float thr, float xl, float xh, float y0,
                                               bool (&reach)[NP]) {
  const float kx = __fdividef(-qb, 2.f * qa), ky = __fdividef(-qb, 2.f * qc);
  const float ex = fmaxf(xl, fminf(xh, 0.f));     // xl if xl > 0, xh if xh < 0, else 0
  const float kyex = ky * ex;
  const float a0 = qa * ex * ex, b0 = qb * ex;     // q2(ex, y) = a0 + y (b0 + qc y)
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const float yl = y0 + 4.f * k, yh = yl + 3.f;
    const float ey = fmaxf(yl, fminf(yh, 0.f));
    const float yy = fminf(fmaxf(kyex, yl), yh);
    const float qx = fmaf(yy, fmaf(qc, yy, b0), a0);
    const float xx = fminf(fmaxf(kx * ey, xl), xh);
    const float qy = fmaf(xx, fmaf(qa, xx, qb * ey), qc * ey * ey);
    reach[k] = fminf(qx, qy) <= thr;
  }
}
template <int NP>
__device__ __forceinline__ uint32_t subboxes_may_reach(float qa, float qb, float qc, float thr, float xl, float xh,
                                                       float y0) {
  bool r[NP];
  subboxes_reach<NP>(qa, qb, qc, thr, xl, xh, y0, r);
  uint32_t need = 0;
#pragma unroll
  for (int k = 0; k < NP; ++k) need |= r[k] ? 1u << k : 0u;
  return need;
}

template <typename T>
__host__ __device__ inline T* ws_ptr(char* base, size_t stride, int f, size_t off) {
  return reinterpret_cast<T*>(base + (size_t)f * stride + off);
}

}  // namespace fgs
