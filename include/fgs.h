/*
 * fgs.h — C ABI of the B200-native 4D Gaussian Splatting forward path
 *         (arXiv 2310.08528, "4D Gaussian Splatting for Real-Time Dynamic Scene Rendering").
 *
 * The two calls of the paper's problem statement (§4.1):
 *     G' = G + F(G, t)      ->  fgs_deform   (Gaussian deformation field, §4.2)
 *     I  = S(M, G')         ->  fgs_render   (differentiable splatting of [3dgs], §3.1)
 * plus their frame-batched, range (sharded) and debug variants.  Citations: P:n = PAPER.md line n.
 *
 * Conventions (all entry points):
 *  - Every array pointer inside the structs and every image/workspace pointer is a DEVICE pointer
 *    (cudaMalloc / torch CUDA tensor), fp32 unless stated, C-contiguous, 16-byte aligned — except
 *    means, log_scales and opacity_logits, which need only 4-byte alignment, so that a struct may
 *    view a row range of a larger array (composition of several models into one G').  Struct
 *    and struct-array arguments themselves (and `ts`) live in HOST memory and are read before the
 *    call returns.  `stream` is a cudaStream_t (0 = legacy default stream).
 *  - Ownership: the caller owns every buffer; the library never allocates device memory on these
 *    paths and keeps no pointer after the call returns (kernels enqueued on `stream` use them).
 *  - Asynchrony: calls validate arguments synchronously, then enqueue kernels and return.  No call
 *    except fgs_render_status synchronises.  All calls are CUDA-graph capturable.
 *  - Errors: an int code, never an exception.  FGS_E_INVALID for bad arguments (null pointers,
 *    n < 0, sh_degree outside [0,3], width/height <= 0, res/t_res < 2, n_scales outside [1,4],
 *    feat not in {8,16,32}, in_dim != feat*n_scales, in_dim > 64, width not in {32,64,128},
 *    t not finite or outside [0,1], misaligned pointers, begin/end out of range, workspace too
 *    small).  FGS_E_CUDA when a launch fails (message in fgs_last_error()).  Instance-capacity
 *    overflow is data dependent and reported by fgs_render_status as FGS_E_CAPACITY.
 *  - Data-dependent degeneracies are not validated: NaN or zero quaternions make a Gaussian
 *    culled (its projected determinant is NaN), never a crash.
 *  - Reentrant for distinct workspaces, from any number of host threads; the only global state is the
 *    tuning knobs below, the profiler, and fgs_frames_host's pool of copy streams / events (each call
 *    holds its own set while it enqueues).
 */
#ifndef FGS_H
#define FGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fgs_stream_t; /* == cudaStream_t */

enum {
  FGS_OK = 0,
  FGS_E_INVALID = -1,
  FGS_E_CUDA = -2,
  FGS_E_CAPACITY = -3,
  FGS_E_NOTIMPL = -4
};
enum { FGS_MAX_SCALES = 4, FGS_PLANES = 6, FGS_TILE = 16 };

/* Canonical 3D Gaussians G = {X, r, s, sigma, C}. */
typedef struct {
  int64_t n;                    /* number of Gaussians (>= 0) */
  int32_t sh_degree;            /* 0..3; K = (deg+1)^2 SH functions ("k nums of SH functions") */
  const float* means;           /* [n][3]  X (world)                                              */
  const float* log_scales;      /* [n][3]  log s; s = exp(.)                                      */
  const float* quats;           /* [n][4]  r, raw quaternion (w,x,y,z); normalised at render      */
  const float* opacity_logits;  /* [n]     sigma = sigmoid(.)                                     */
  const float* sh;              /* [n][K][3] SH coefficients, k = l^2 + l + m                     */
} fgs_gaussians;

/* Multi-resolution HexPlane R_l(i,j) (Eq. 7).  Plane order
 * (x,y),(x,z),(y,z),(x,t),(y,t),(z,t); plane (a,b) of scale l is [n_b][n_a][feat] with
 * n_x = n_y = n_z = res[l] and n_t = t_res (same at every scale).  A mean maps to the grid by
 * u = clamp((X - bmin)/(bmax - bmin), 0, 1); knot k of an axis of n knots sits at u = k/(n-1). */
typedef struct {
  int32_t n_scales;             /* L, 1..4                                                        */
  int32_t feat;                 /* h: 8, 16 or 32                                                 */
  int32_t t_res;                /* temporal knots, >= 2                                           */
  int32_t res[FGS_MAX_SCALES];  /* spatial knots per scale, >= 2                                  */
  float bmin[3], bmax[3];       /* world AABB of the field (bmax > bmin)                          */
  const float* planes[FGS_MAX_SCALES][FGS_PLANES];
} fgs_hexplanes;

/* phi_d (one Linear + ReLU) and the heads phi_x, phi_r, phi_s (one Linear each).
 * Row-major [out][in] (PyTorch Linear layout).  Optional: the colour and opacity decoders phi_C,
 * phi_alpha of P:1232 ("Color and Opacity's Deformation"): dC = phi_C(f_d) over all K x 3 SH
 * coefficients (output o = 3k + channel, the SH layout), dalpha = phi_alpha(f_d) on the opacity logit;
 * NULL weights = no such head.  With either head, fgs_deform writes the deformed SH / opacity into the
 * fgs_deformed arrays (which must then be caller buffers, not the canonical arrays); the field must fit
 * the warp-specialised deform kernel (else FGS_E_NOTIMPL). */
typedef struct {
  int32_t in_dim;               /* = feat * n_scales (<= 64)                                      */
  int32_t width;                /* hidden width W of phi_d: 32, 64 or 128                         */
  const float *w_d, *b_d;       /* [W][in_dim], [W]                                               */
  const float *w_x, *b_x;       /* [3][W], [3]                                                    */
  const float *w_r, *b_r;       /* [4][W], [4]                                                    */
  const float *w_s, *b_s;       /* [3][W], [3]                                                    */
  const float *w_c, *b_c;       /* optional phi_C: [3K][W], [3K]  (K = (sh_degree+1)^2)           */
  const float *w_a, *b_a;       /* optional phi_alpha: [1][W], [1]                                 */
} fgs_mlp;

/* Deformed Gaussians G' = {X', s', r', sigma, C}.  fgs_deform writes means, log_scales and
 * quats (raw: X + dX, log s + ds, r + dr); opacity and SH alias the canonical arrays, unless the
 * MLP has phi_alpha / phi_C, in which case fgs_deform writes logit + dalpha / C + dC there. */
typedef struct {
  int64_t n;
  int32_t sh_degree;
  float* means;                 /* [n][3] */
  float* log_scales;            /* [n][3] */
  float* quats;                 /* [n][4] */
  float* opacity_logits;        /* [n]       canonical alias, or written (phi_alpha)               */
  float* sh;                    /* [n][K][3] canonical alias, or written (phi_C)                   */
} fgs_deformed;

/* View matrix M = [R, T] + pinhole intrinsics.  World->camera, row-major, OpenCV axes
 * (x right, y down, z forward); pixel (px,py) is evaluated at continuous (px,py).  Host struct. */
typedef struct {
  float R[9];
  float t[3];
  float fx, fy, cx, cy;
  int32_t width, height;        /* > 0, <= 16384                                                  */
  float bg[3];                  /* background colour added as T_final * bg                        */
} fgs_camera;

/* Optional device outputs of fgs_render_debug; any pointer may be NULL. */
typedef struct {
  int32_t* radii;               /* [n]          integer pixel radius, 0 if culled                 */
  int32_t* rect;                /* [n][4]       tile rect x0,y0,x1,y1 ([x0,x1) x [y0,y1)), 0s if culled */
  float* mean2d;                /* [n][2]       projected mean                                    */
  uint32_t* depth_key;          /* [n]          IEEE bits of fp32 view-space depth, 0 if culled   */
  uint32_t* tiles_touched;      /* [n]                                                            */
  uint32_t* n_instances;        /* [1]          M (un-clamped)                                    */
  uint32_t* sorted_tile;        /* [max_instances] tile id of each sorted instance                */
  uint32_t* sorted_gid;         /* [max_instances] Gaussian index of each sorted instance         */
  uint32_t* ranges;             /* [tiles][2]   [start,end) of each tile's list                   */
  float* final_T;               /* [H][W]       final transmittance                               */
  uint32_t* n_contrib;          /* [H][W]       number of composited Gaussians                    */
  uint32_t* n_evaluated;        /* [H][W]       list entries evaluated before the pixel terminated */
  uint64_t* blend_work;         /* [2] (accumulated, caller zeroes): [0] (warp, Gaussian) pairs the
                                 * blend evaluated after its per-warp cull, [1] pairs it tested; a warp
                                 * covers 64 pixels, so [0] * 64 bounds the pixel evaluations           */
  uint32_t* binning_direct;     /* [2]          CTAs of the per-tile counting [0] and of the key
                                 * duplication [1] whose Gaussians' rect union exceeded the shared
                                 * aggregation box (FGS_TUNE_AGG_TILES) and went to direct global atomics */
  uint32_t* long_sort_paths;    /* [3]          lists longer than the warp-sort cap sorted by the bucket
                                 * pass with its scratch in shared memory [0] / in the inst2 scratch [1],
                                 * and by the networks + merges (a bucket over kBucketMax: skewed depths) [2] */
} fgs_render_aux;

/* ---- deformation field F --------------------------------------------------
 * For every Gaussian i and time t in [0,1]: f_h = concat_l prod_planes bilinear(R_l(i,j)) at
 * (X_i, t) (Eq. 7); f_d = ReLU(W_d f_h + b_d); (X', r', s') = (X, r, s) + heads(f_d). */
int fgs_deform(const fgs_gaussians* g, const fgs_hexplanes* field, const fgs_mlp* mlp, float t,
               fgs_deformed* out, fgs_stream_t stream);
/* Only Gaussians [begin, end) are written (the rest of `out` untouched): the shard of §8(e2).
 * Results are bit-identical to the same rows of fgs_deform. */
int fgs_deform_range(const fgs_gaussians* g, const fgs_hexplanes* field, const fgs_mlp* mlp, float t,
                     int64_t begin, int64_t end, fgs_deformed* out, fgs_stream_t stream);
/* §8(e2) fused deform + gather: as fgs_deform_range, but means / log_scales / quats of rows
 * [begin, end) are stored n_peers times, replica q at byte offset peer_offsets[q] from the `out`
 * address (peer_offsets: HOST array of int64, multiples of 4; 1 <= n_peers <= 8).  With the
 * symmetric-memory gather buffers of a process group (offset q = buffer_ptrs[q] - buffer_ptrs[rank])
 * the deform epilogue itself writes every rank's copy — over NVLink, tile by tile, overlapped with
 * the deformation — and no separate all-gather pass is needed; the caller orders the ranks with a
 * stream-ordered barrier before rendering.  Every replica must lie in caller-owned memory the device
 * can write (peer access).  Not with phi_C / phi_alpha.  Results are bit-identical to
 * fgs_deform_range in every replica. */
int fgs_deform_range_peers(const fgs_gaussians* g, const fgs_hexplanes* field, const fgs_mlp* mlp, float t,
                           int64_t begin, int64_t end, fgs_deformed* out, const int64_t* peer_offsets,
                           int32_t n_peers, fgs_stream_t stream);
/* n_t times ts[0..n_t) (HOST array) into outs[0..n_t) (HOST array of structs) in one pass that
 * shares the spatial-plane work across times.  Bit-identical to n_t calls of fgs_deform. */
int fgs_deform_batch(const fgs_gaussians* g, const fgs_hexplanes* field, const fgs_mlp* mlp,
                     const float* ts, int32_t n_t, fgs_deformed* outs, fgs_stream_t stream);

/* ---- splatting S (§3.1, [3dgs] rasterizer P:728) ----------------------------
 * Device workspace bytes for ONE frame of n Gaussians at width x height with room for
 * max_instances (tile, Gaussian) instances; a batch of F frames needs F times this. */
size_t fgs_render_workspace_bytes(int64_t n, int32_t width, int32_t height, int64_t max_instances);
/* Renders image [3][height][width] fp32 (CHW, no final clamp).  ws/ws_bytes: device workspace;
 * the instance capacity is the largest max_instances whose workspace fits in ws_bytes. */
int fgs_render(const fgs_camera* cam, const fgs_deformed* g, float* image, void* ws, size_t ws_bytes,
               fgs_stream_t stream);
/* n_frames frames (all cameras must share width/height); cams, defs and images are HOST arrays,
 * images[f] a DEVICE pointer.  ws holds n_frames equal per-frame slices of ws_bytes/n_frames. */
int fgs_render_batch(const fgs_camera* cams, const fgs_deformed* defs, float* const* images,
                     int32_t n_frames, void* ws, size_t ws_bytes, fgs_stream_t stream);
/* fgs_render plus the intermediate results in `aux` (debugging and parity tests). */
int fgs_render_debug(const fgs_camera* cam, const fgs_deformed* g, float* image, void* ws,
                     size_t ws_bytes, const fgs_render_aux* aux, fgs_stream_t stream);
/* Synchronises `stream`; FGS_E_CAPACITY if any frame of the last render into `ws` overflowed its
 * instance capacity (its image is then invalid), else FGS_OK.  n_frames = frames in ws. */
int fgs_render_status(const void* ws, size_t ws_bytes, int32_t n_frames, fgs_stream_t stream);

/* ---- whole frames (deform + render), the step bench.py times --------------------------------
 * Frame f deforms G at ts[f] into defs_scratch[f] (device buffers owned by the caller) and renders
 * it with cams[f] into images[f].  Device pointers everywhere except the host arrays.  Frames whose
 * ts are bitwise equal (several views of one instant) share one deformation: only the first such
 * frame's defs_scratch is written and all of them render from it. */
int fgs_frames(const fgs_gaussians* g, const fgs_hexplanes* field, const fgs_mlp* mlp,
               const float* ts, const fgs_camera* cams, int32_t n_frames, fgs_deformed* defs_scratch,
               float* const* images, void* ws, size_t ws_bytes, fgs_stream_t stream);

/* ---- end to end with HOST buffers (what e2e in bench.py times) ---------------------------------
 * Same as fgs_frames, but every array pointer in g_host / field_host / mlp_host and images_host[f]
 * is a HOST pointer (pinned memory gives asynchronous copies).  The call enqueues the host->device
 * copies of the model into `dev_ws`, the deform + render of all frames, and the device->host copies
 * of the images, all on `stream`; the images are valid after the stream synchronises.
 * dev_ws: device memory of at least fgs_frames_host_workspace_bytes(...) bytes. */
size_t fgs_frames_host_workspace_bytes(const fgs_gaussians* g_host, const fgs_hexplanes* field_host,
                                       const fgs_mlp* mlp_host, int32_t n_frames, int32_t width,
                                       int32_t height, int64_t max_instances);
int fgs_frames_host(const fgs_gaussians* g_host, const fgs_hexplanes* field_host, const fgs_mlp* mlp_host,
                    const float* ts, const fgs_camera* cams, int32_t n_frames, float* const* images_host,
                    void* dev_ws, size_t dev_ws_bytes, fgs_stream_t stream);
/* The instance-capacity check of a fgs_frames_host call (its renders live inside dev_ws): pass the same
 * g_host / field_host / mlp_host / cams / n_frames / dev_ws / dev_ws_bytes.  Synchronises `stream`;
 * FGS_E_CAPACITY if any frame overflowed (its host image is then invalid), else FGS_OK. */
int fgs_frames_host_status(const fgs_gaussians* g_host, const fgs_hexplanes* field_host, const fgs_mlp* mlp_host,
                           const fgs_camera* cams, int32_t n_frames, const void* dev_ws, size_t dev_ws_bytes,
                           fgs_stream_t stream);

/* ---- training side: loss and gradients (§4.3 P:828-833 "L = |I^ - I| + L_tv") ----------
 * The backward of the frame: L1 image loss and grid total variation, then dL/dI^ back through the
 * splatting (the [3dgs] "differentiable" rasterizer) to the deformed Gaussians, and back through
 * the deformation field (Eq. 7, phi_d, heads) to the canonical Gaussians, the planes and the MLP.
 * Discontinuous decisions (culls, tile lists, depth order, alpha skip / stop, 0.99 clamp, colour
 * clamp, ReLU, AABB clamp, knot indices) are held fixed, as in [3dgs].  Gradients are accumulated in
 * 2^-40 fixed point with integer atomics: every result is bit-identical from run to run.
 * Readings B1-B4: L1 = mean over 3 H W of |I^ - I|; L_tv = pooled mean of squared
 * differences of adjacent entries of all planes, channels and both grid directions; L = L1 + w L_tv. */
enum { FGS_LOSS_PARTIALS = 1024 };  /* fp64 scratch entries of a loss call (one per block)            */
typedef struct {                    /* dL/d per-Gaussian arrays (device, fp32, layouts as fgs_gaussians) */
  float* means;                     /* [n][3] */
  float* log_scales;                /* [n][3] */
  float* quats;                     /* [n][4] */
  float* opacity_logits;            /* [n]    */
  float* sh;                        /* [n][K][3] */
} fgs_gaussian_grads;
typedef struct {                    /* dL/d field + MLP (device, fp32, layouts as fgs_hexplanes / fgs_mlp) */
  float* planes[FGS_MAX_SCALES][FGS_PLANES];
  float *w_d, *b_d, *w_x, *b_x, *w_r, *b_r, *w_s, *b_s;
  float *w_c, *b_c, *w_a, *b_a;     /* the P:1232 decoders' gradients (needed only when the MLP has them) */
} fgs_field_grads;
/* loss[0] = mean |image - target| over [3][H][W] (B2); dL_dimage (may be NULL) = sign(image - target) /
 * (3 H W), 0 where equal.  partials: device double[FGS_LOSS_PARTIALS] scratch. */
int fgs_l1_loss(const float* image, const float* target, int32_t width, int32_t height, float* dL_dimage,
                double* partials, float* loss, fgs_stream_t stream);
/* loss[0] = weight * L_tv(field) (B1); grads->planes[l][p] (if grads != NULL) += weight * dL_tv/dplane. */
int fgs_tv_loss(const fgs_hexplanes* field, float weight, fgs_field_grads* grads, double* partials, float* loss,
                fgs_stream_t stream);
/* Splat backward for ONE frame: cam, g and the workspace ws must be those of the fgs_render call that
 * produced `image` (the sorted lists and records are read from ws, which must be unchanged since); for
 * frame f of an fgs_render_batch / fgs_frames call pass that frame's slice: ws + f * per, per bytes, with
 * per = (ws_bytes / n_frames) rounded down to a multiple of 256.
 * Accumulation is in 2^-40 fixed point (64-bit integer atomics): every per-Gaussian and per-weight sum
 * must stay within +-8.4e6 (ample for the mean-reduced losses above; scale a sum-reduced loss down).
 * Writes (overwrites) dg->means, log_scales, quats (raw), opacity_logits and sh for all n Gaussians
 * (0 for culled ones).  scratch: device memory of fgs_render_backward_scratch_bytes(n) bytes. */
size_t fgs_render_backward_scratch_bytes(int64_t n);
int fgs_render_backward(const fgs_camera* cam, const fgs_deformed* g, const float* image, const float* dL_dimage,
                        const void* ws, size_t ws_bytes, void* scratch, size_t scratch_bytes,
                        const fgs_gaussian_grads* dg, fgs_stream_t stream);
/* Deformation backward at time t: given dL/dG' (d_deformed: means, log_scales, quats; with the P:1232
 * decoders also sh and/or opacity_logits — the render backward's gradients of the deformed SH / logits),
 * writes dL/dG for the canonical means (additive path + the query-position path u(X)), log_scales and
 * quats into d_canonical (and, with the decoders, sh / opacity_logits: the decoders add to them, so their
 * gradient passes through; without them d_canonical's sh / opacity_logits are untouched — use the render
 * backward's directly), and ADDS dL/d planes and MLP weights (incl. w_c, b_c, w_a, b_a) into d_field.
 * scratch: device memory of fgs_deform_backward_scratch_bytes(field, mlp) bytes. */
size_t fgs_deform_backward_scratch_bytes(const fgs_hexplanes* field, const fgs_mlp* mlp);
int fgs_deform_backward(const fgs_gaussians* g, const fgs_hexplanes* field, const fgs_mlp* mlp, float t,
                        const fgs_gaussian_grads* d_deformed, const fgs_gaussian_grads* d_canonical,
                        const fgs_field_grads* d_field, void* scratch, size_t scratch_bytes, fgs_stream_t stream);

/* One Adam step over n parameters (elementwise, the optimiser [3dgs] and the paper
 * train with): m = b1 m + (1 - b1) g; v = b2 v + (1 - b2) g^2; p -= lr (m / (1 - b1^step)) /
 * (sqrt(v / (1 - b2^step)) + eps) (reading A1).  param / m / v updated in place, grad read; step >= 1.
 * Apply it to every gradient tensor of fgs_gaussian_grads / fgs_field_grads with its own moments. */
int fgs_adam_step(float* param, const float* grad, float* m, float* v, int64_t n, float lr, float beta1,
                  float beta2, float eps, int32_t step, fgs_stream_t stream);

/* ---- profiling -------------------------------------------------------------------------------
 * When enabled, the library records a CUDA event pair around every stage it launches, on the
 * stream of the call.  fgs_profile_read synchronises those events and writes the accumulated
 * milliseconds and launch counts per stage into ms[FGS_N_STAGES] / launches[FGS_N_STAGES]
 * (either may be NULL), then resets them.  Not thread-safe (one profiling client at a time). */
enum {
  FGS_STAGE_DEFORM = 0,         /* HexPlane sampling + phi_d + heads (a1-a3)                        */
  FGS_STAGE_PREPROCESS,         /* counter clear + preprocess incl. per-tile instance counts (a4)   */
  FGS_STAGE_TILE_SCAN,          /* scan of the tile counts -> ranges (a7)                           */
  FGS_STAGE_DUPLICATE,          /* key duplication into tile buckets (a5)                           */
  FGS_STAGE_TILE_SORT,          /* per-tile (depth, index) sort: warp sorts + long-list CTA sort (a6) */
  FGS_STAGE_BLEND,              /* front-to-back alpha blending of the sorted lists (a8, Eq. 4)     */
  FGS_N_STAGES
};
int fgs_profile_enable(int enable);
int fgs_profile_read(double* ms, int64_t* launches);
/* Number of kernels this library has launched since it was loaded (all threads). */
int64_t fgs_launch_count(void);

/* ---- tuning (process-global; change only while no call of this library is enqueueing) --------
 * FGS_TUNE_TILE_SORT_CAP: tile lists of at most this many instances are sorted by (depth, index) by
 * one warp (registers + shared memory); longer lists by the persistent long-list CTA sort (see
 * FGS_TUNE_LONG_SORT).  Both run in FGS_STAGE_TILE_SORT.
 * Range [1, 1024], default 1024.  Results are identical for every value (tests lower it to exercise
 * the long-list path).  fgs_set_tuning returns FGS_E_INVALID for an unknown key or a value out of
 * range; fgs_get_tuning returns -1 for an unknown key.
 * FGS_TUNE_BLEND_CULL: 1 (default) = the blend skips, per warp, the Gaussians whose alpha is below
 * 1/255 on a whole 8x4 pixel sub-box (conservative ellipse-vs-box bound); 0 = every list entry is
 * evaluated on every live pixel.  Images, final T and contributor counts are identical (tests check it
 * on whole full-size frames).
 * FGS_TUNE_AGG_TILES: the per-tile counting and key duplication aggregate a CTA's per-tile atomics in
 * shared memory when the CTA's rect union holds at most this many tiles, else use direct global
 * atomics.  Range [1, 4096], default 4096.  Results are identical for every value (tests lower it to
 * force the direct path; fgs_render_aux.binning_direct counts the CTAs that took it).
 * FGS_TUNE_RADIX: how a frame's tile lists are put in (tile, depth, index) order.  0 (default) = per-tile sorts
 * (the warp and long-list sorts above); 2 = the radix binning path for every frame: a stable LSD radix
 * sort of the Gaussians by depth key, emission of the instances in that order, and stable radix passes on
 * the tile id (images of up to 65536 tiles); 1 = the radix path for frames whose mean list length
 * M / tiles reaches FGS_TUNE_RADIX_MIN_LIST (default 768; range [1, 2^20]), the per-tile sorts for the
 * others.  Default 0 (the per-tile sorts were faster at every measured N).  The order, hence every image,
 * is identical whichever path a frame takes.
 * FGS_TUNE_LONG_SORT: how the long-list CTA sort orders a list.  1 (default) = one bucket pass: the
 * instances bucketed by the top 11 bits of their depth key relative to the list's minimum, each then
 * placed at its bucket's start + the number of its bucket's instances below it (a list with a bucket of
 * more than 64 instances falls back to 0); 0 = CTA bitonic networks on 4096-instance segments + merge
 * levels.  The order is identical either way (fgs_render_aux.long_sort_paths counts which ran).
 * FGS_TUNE_TILE_CULL: 0 (default) = a tile's list holds every kept Gaussian whose [3dgs] rect covers the
 * tile (the oracle's lists, bit for bit); 1 = a Gaussian whose rect holds at most 64 tiles is left
 * out of the list of a tile on which its alpha provably stays below 1/255 at every pixel (the ellipse where
 * its Eq. 1 exponent reaches the blend's own threshold, margin included, does not meet the tile's 16x16
 * pixel box: one x-interval of the ellipse per tile row, widened by 0.01 px): the
 * lists are then ordered subsequences of the [3dgs] lists that keep every contributing entry, and images,
 * final T and contributor counts are identical (tests check both on whole full-size frames);
 * fgs_render_aux.tiles_touched counts the remaining tiles, n_instances the remaining entries.  With 1
 * the per-tile sorts are used for every frame (FGS_TUNE_RADIX is ignored).
 * (Key 1 is retired: there is a single deformation kernel.) */
enum { FGS_TUNE_TILE_SORT_CAP = 0, FGS_TUNE_BLEND_CULL = 2, FGS_TUNE_AGG_TILES = 3, FGS_TUNE_RADIX = 4,
       FGS_TUNE_RADIX_MIN_LIST = 5, FGS_TUNE_LONG_SORT = 6, FGS_TUNE_TILE_CULL = 7 };
int fgs_set_tuning(int32_t key, int64_t value);
int64_t fgs_get_tuning(int32_t key);

/* Message of the last non-OK return on this thread (static storage, never NULL). */
const char* fgs_last_error(void);
/* Library version string and the compute capability it was built for ("sm_100a"). */
const char* fgs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FGS_H */
