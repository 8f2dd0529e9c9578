// Tile-based splatting S(M, G') on sm_100a — PAPER.md §3.1 with the [3dgs] rasterizer
// conventions the paper renders with; readings R1-R20 in DESIGN.md.
//
// Per frame (the frames of a batch share every launch, blockIdx.y = frame):
//   clear        zero the per-tile instance counters.
//   preprocess   Eq. 2 covariance, Eq. 3 EWA projection, conic, radius, tile rect, depth key, SH
//                colour; every kept Gaussian adds 1 to the counter of each tile of its rect (RED).
//                Decision geometry (depth key, radius, rect) in fp64 with the oracle's fixed
//                summation order, so the integer work is bit-exact against the fp64 oracle.
//   tile scan    exclusive scan of the tile counters -> per-tile ranges [start, end),
//                scatter cursors, M and the capacity-overflow flag.
//   duplicate    each kept Gaussian writes one 64-bit instance (depth_key << 32 | gid) into every
//                tile bucket of its rect, at an atomically claimed slot.  The order
//                inside a bucket is arbitrary here; the sort below makes it unique.
//   tile sort    (a6) every tile's list sorted ascending by (depth key, gid): lists of up to
//                sort_cap instances by one warp (tile_sort_kernel: register bitonic networks on 32-bit
//                depth-prefix words + merge path), longer lists by long_sort_kernel (shared-memory
//                segments + merge-path merges in global memory).
//                Result: the [3dgs] (tile, depth, index) order (reading R14), without global passes.
//   blend        Eq. 4 front to back per pixel; 16x16 tile per CTA.
#include <cuda_runtime.h>
#include <math.h>

#include <limits.h>

#include <algorithm>

#include "fgs_internal.cuh"

namespace fgs {

namespace {

constexpr float kNear = 0.2f;               // R6
constexpr float kAlphaMin = 1.0f / 255.0f;  // R9
constexpr float kTMin = 1e-4f;              // R9
constexpr float kAlphaMax = 0.99f;          // R9
constexpr double kDilation = 0.3;           // R5
constexpr double kLambdaFloor = 0.1;        // R7
constexpr double kFovClamp = 1.3;           // R4
constexpr double kLog2e = 1.4426950408889634;

// Real SH constants (CS phase, [3dgs] table; reading R10).
constexpr float SH_C0 = 0.28209479177387814f;
constexpr float SH_C1 = 0.4886025119029199f;
constexpr float SH_C2_0 = 1.0925484305920792f, SH_C2_1 = -1.0925484305920792f,
                SH_C2_2 = 0.31539156525252005f, SH_C2_3 = -1.0925484305920792f,
                SH_C2_4 = 0.5462742152960396f;
constexpr float SH_C3_0 = -0.5900435899266435f, SH_C3_1 = 2.890611442640554f,
                SH_C3_2 = -0.4570457994644658f, SH_C3_3 = 0.3731763325901154f,
                SH_C3_4 = -0.4570457994644658f, SH_C3_5 = 1.445305721320277f,
                SH_C3_6 = -0.5900435899266435f;

__device__ __forceinline__ uint32_t* cnt_ptr(const RenderBatch& b, int f) {
  return ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.cnt);
}

// ------------------------------------------------------------------------------ clear
__global__ void clear_kernel(const __grid_constant__ RenderBatch b) {
  const int f = blockIdx.y;
  uint32_t* tc = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.tile_count);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < b.ntiles; t += gridDim.x * blockDim.x) tc[t] = 0;
  if (blockIdx.x == 0 && threadIdx.x < 16) cnt_ptr(b, f)[threadIdx.x] = threadIdx.x == 0 ? (uint32_t)b.n : 0u;
}

// ------------------------------------------------------------------------------ preprocess
// SH coefficients of Gaussian i ([K][3] fp32) -> colour (step 12).  DEG is the SH degree.
template <int DEG>
__device__ __forceinline__ void sh_colour(const float* __restrict__ sh, float X, float Y, float Z, float col[3]) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  float c[3 * K];
  if constexpr ((3 * K) % 4 == 0) {            // 16-B aligned rows (K = 4, 16): vector loads
#pragma unroll
    for (int q = 0; q < 3 * K / 4; ++q) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(sh) + q);
      c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 3 * K; ++q) c[q] = __ldg(sh + q);
  }
  float basis[K];
  basis[0] = SH_C0;
  if constexpr (DEG >= 1) { basis[1] = -SH_C1 * Y; basis[2] = SH_C1 * Z; basis[3] = -SH_C1 * X; }
  if constexpr (DEG >= 2) {
    const float xx = X * X, yy = Y * Y, zz = Z * Z;
    basis[4] = SH_C2_0 * X * Y;
    basis[5] = SH_C2_1 * Y * Z;
    basis[6] = SH_C2_2 * (2.f * zz - xx - yy);
    basis[7] = SH_C2_3 * X * Z;
    basis[8] = SH_C2_4 * (xx - yy);
    if constexpr (DEG >= 3) {
      basis[9] = SH_C3_0 * Y * (3.f * xx - yy);
      basis[10] = SH_C3_1 * X * Y * Z;
      basis[11] = SH_C3_2 * Y * (4.f * zz - xx - yy);
      basis[12] = SH_C3_3 * Z * (2.f * zz - 3.f * xx - 3.f * yy);
      basis[13] = SH_C3_4 * X * (4.f * zz - xx - yy);
      basis[14] = SH_C3_5 * Z * (xx - yy);
      basis[15] = SH_C3_6 * X * (xx - 3.f * yy);
    }
  }
  col[0] = col[1] = col[2] = 0.5f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    col[0] = fmaf(basis[k], c[3 * k + 0], col[0]);
    col[1] = fmaf(basis[k], c[3 * k + 1], col[1]);
    col[2] = fmaf(basis[k], c[3 * k + 2], col[2]);
  }
}

// CTA-level aggregation of per-tile atomics.  The CTA's kept Gaussians are bounded by the tile box
// [bx0,bx1) x [by0,by1); when it holds at most b.agg_tiles (<= kAggTilesMax) tiles (spatially ordered models: a CTA's
// Gaussians are neighbours), per-tile sums are formed in shared memory and each touched tile gets one
// global atomic; otherwise every instance goes to global memory directly.
struct AggBox {
  int x0, y0, x1, y1;
};

__device__ __forceinline__ AggBox cta_rect_union(bool kept, int x0, int y0, int x1, int y1, int* sbox) {
  if (threadIdx.x == 0) { sbox[0] = INT_MAX; sbox[1] = INT_MAX; sbox[2] = INT_MIN; sbox[3] = INT_MIN; }
  __syncthreads();
  if (kept) {
    atomicMin(sbox + 0, x0); atomicMin(sbox + 1, y0);
    atomicMax(sbox + 2, x1); atomicMax(sbox + 3, y1);
  }
  __syncthreads();
  AggBox r{sbox[0], sbox[1], sbox[2], sbox[3]};
  __syncthreads();
  return r;
}

// `limit` = b.agg_tiles (<= kAggTilesMax; FGS_TUNE_AGG_TILES lowers it so tests can force the direct path)
__device__ __forceinline__ bool agg_fits(const AggBox& r, int limit) {
  return r.x1 > r.x0 && (int64_t)(r.x1 - r.x0) * (r.y1 - r.y0) <= limit;
}

// The tiles (tx, ty) of a rect a Gaussian is listed on, in row-major order.  CULL: the set bits of tmask
// (bit (ty - y0) * w + tx - x0) for rects of at most 64 tiles; every tile otherwise.
template <bool CULL, typename Fn>
__device__ __forceinline__ void for_each_tile(int x0, int y0, int x1, int y1, unsigned long long tmask, Fn&& fn) {
  const int w = x1 - x0;
  if (!CULL || w * (y1 - y0) > 64) {
    for (int ty = y0; ty < y1; ++ty)
      for (int tx = x0; tx < x1; ++tx) fn(tx, ty);
  } else {
    const unsigned long long wm = w >= 64 ? ~0ull : (1ull << w) - 1ull;
    int sh = 0;
    for (int ty = y0; ty < y1; ++ty, sh += w) {
      unsigned long long rm = (tmask >> sh) & wm;
      while (rm) {
        const int rx = __ffsll((long long)rm) - 1;
        rm &= rm - 1ull;
        fn(x0 + rx, ty);
      }
    }
  }
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Per-tile instance counts of a CTA's Gaussians: aggregated in shared memory over the CTA's
// rect union when it holds at most agg_tiles tiles (one global atomic per touched tile), else direct
// global atomics (cnt67[0] counts the CTAs that took that path: fgs_render_aux.binning_direct[0]).
// CULL: only the tiles of tmask (FGS_TUNE_TILE_CULL).  Called by every thread of the CTA.
template <bool CULL>
__device__ __forceinline__ void count_tiles(bool keep, int x0, int y0, int x1, int y1, unsigned long long tmask,
                                            uint32_t* tile_count, int gx, int gy, int agg_tiles, uint32_t* cnt67,
                                            int* sbox, uint32_t* scount) {
  const AggBox box = cta_rect_union(keep, x0, y0, x1, y1, sbox);
  if (agg_fits(box, agg_tiles)) {
    const int bw = box.x1 - box.x0, area = bw * (box.y1 - box.y0);
    FGS_DCHECK(area <= kAggTilesMax && box.x0 >= 0 && box.y0 >= 0 && box.x1 <= gx && box.y1 <= gy);
    for (int q = threadIdx.x; q < area; q += blockDim.x) scount[q] = 0;
    __syncthreads();
    if (keep)
      for_each_tile<CULL>(x0, y0, x1, y1, tmask,
                          [&](int tx, int ty) { atomicAdd(scount + (ty - box.y0) * bw + (tx - box.x0), 1u); });
    __syncthreads();
    for (int q = threadIdx.x; q < area; q += blockDim.x)
      if (scount[q]) atomicAdd(tile_count + (box.y0 + q / bw) * gx + box.x0 + q % bw, scount[q]);
  } else {
    if (threadIdx.x == 0 && box.x1 > box.x0) atomicAdd(cnt67, 1u);
    if (keep)
      for_each_tile<CULL>(x0, y0, x1, y1, tmask, [&](int tx, int ty) { atomicAdd(tile_count + ty * gx + tx, 1u); });
  }
}

template <int DEG, bool CULL>
__global__ void __launch_bounds__(256, 4) preprocess_kernel(const __grid_constant__ RenderBatch b) {
  // frame-minor CTA order: the F CTAs of one Gaussian block are adjacent in launch order, so its SH
  // (192 B per Gaussian at degree 3, frame-invariant) come from HBM once and from L2 for the other frames
  const int f = (int)(blockIdx.x % (unsigned)b.n_frames);
  const int64_t i0 = (int64_t)(blockIdx.x / (unsigned)b.n_frames) * blockDim.x + threadIdx.x;
  const bool valid = i0 < b.n;
  const int64_t i = valid ? i0 : b.n - 1;     // out-of-range threads mirror the last Gaussian, write nothing
  uint32_t* keys = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.keys);
  uint32_t* tt = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.tt);
  uint2* rect = ws_ptr<uint2>(b.ws, b.ws_stride, f, b.L.rect);
  int32_t* radii = ws_ptr<int32_t>(b.ws, b.ws_stride, f, b.L.radii);
  float4* rec = ws_ptr<float4>(b.ws, b.ws_stride, f, b.L.rec);
  uint32_t* tile_count = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.tile_count);
  const FrameCam& c = b.cam[f];

  // ---- step 3: p = R X + t with the oracle's summation order (products exact in fp64) ----
  const float* Xp = b.means[f] + 3 * i;
  const double x = Xp[0], y = Xp[1], z = Xp[2];
  const double px = ((((double)c.R[0] * x) + (double)c.R[1] * y) + (double)c.R[2] * z) + (double)c.t[0];
  const double py = ((((double)c.R[3] * x) + (double)c.R[4] * y) + (double)c.R[5] * z) + (double)c.t[1];
  const double pz = ((((double)c.R[6] * x) + (double)c.R[7] * y) + (double)c.R[8] * z) + (double)c.t[2];
  bool keep = pz > (double)kNear;
  // ---- steps 1-2: activation and Sigma = R S S^T R^T (Eq. 2) ----
  const float* ls = b.log_scales[f] + 3 * i;
  const double s0 = exp((double)ls[0]), s1 = exp((double)ls[1]), s2 = exp((double)ls[2]);
  const float4 qv = *reinterpret_cast<const float4*>(b.quats[f] + 4 * i);
  double qw = qv.x, qx = qv.y, qy = qv.z, qz = qv.w;
  const double qinv = 1.0 / sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  qw *= qinv; qx *= qinv; qy *= qinv; qz *= qinv;
  const double r00 = 1 - 2 * (qy * qy + qz * qz), r01 = 2 * (qx * qy - qw * qz), r02 = 2 * (qx * qz + qw * qy);
  const double r10 = 2 * (qx * qy + qw * qz), r11 = 1 - 2 * (qx * qx + qz * qz), r12 = 2 * (qy * qz - qw * qx);
  const double r20 = 2 * (qx * qz - qw * qy), r21 = 2 * (qy * qz + qw * qx), r22 = 1 - 2 * (qx * qx + qy * qy);
  const double m00 = r00 * s0, m01 = r01 * s1, m02 = r02 * s2;
  const double m10 = r10 * s0, m11 = r11 * s1, m12 = r12 * s2;
  const double m20 = r20 * s0, m21 = r21 * s1, m22 = r22 * s2;
  const double S00 = m00 * m00 + m01 * m01 + m02 * m02;
  const double S01 = m00 * m10 + m01 * m11 + m02 * m12;
  const double S02 = m00 * m20 + m01 * m21 + m02 * m22;
  const double S11 = m10 * m10 + m11 * m11 + m12 * m12;
  const double S12 = m10 * m20 + m11 * m21 + m12 * m22;
  const double S22 = m20 * m20 + m21 * m21 + m22 * m22;
  // ---- steps 4-6: J (x/z, y/z clamped, R4), Sigma2 = J W Sigma W^T J^T + 0.3 I (Eq. 3) ----
  // (one fp64 reciprocal of z; a reordering at the 1e-16 level, far inside the 1e-5 px decision band)
  const double fx = c.fx, fy = c.fy;
  const double iz = 1.0 / pz;
  const double limx = kFovClamp * ((double)b.width / (2.0 * fx));
  const double limy = kFovClamp * ((double)b.height / (2.0 * fy));
  const double xt = fmin(limx, fmax(-limx, px * iz)) * pz;
  const double yt = fmin(limy, fmax(-limy, py * iz)) * pz;
  const double j00 = fx * iz, j02 = -fx * xt * (iz * iz);
  const double j11 = fy * iz, j12 = -fy * yt * (iz * iz);
  const double W00 = c.R[0], W01 = c.R[1], W02 = c.R[2];
  const double W10 = c.R[3], W11 = c.R[4], W12 = c.R[5];
  const double W20 = c.R[6], W21 = c.R[7], W22 = c.R[8];
  const double t00 = j00 * W00 + j02 * W20, t01 = j00 * W01 + j02 * W21, t02 = j00 * W02 + j02 * W22;
  const double t10 = j11 * W10 + j12 * W20, t11 = j11 * W11 + j12 * W21, t12 = j11 * W12 + j12 * W22;
  const double u0 = t00 * S00 + t01 * S01 + t02 * S02;
  const double u1 = t00 * S01 + t01 * S11 + t02 * S12;
  const double u2 = t00 * S02 + t01 * S12 + t02 * S22;
  const double v0 = t10 * S00 + t11 * S01 + t12 * S02;
  const double v1 = t10 * S01 + t11 * S11 + t12 * S12;
  const double v2 = t10 * S02 + t11 * S12 + t12 * S22;
  const double a = u0 * t00 + u1 * t01 + u2 * t02 + kDilation;
  const double bb = u0 * t10 + u1 * t11 + u2 * t12;
  const double cc = v0 * t10 + v1 * t11 + v2 * t12 + kDilation;
  // ---- step 7: det, conic (Eq. 1 inverse) ----
  const double det = a * cc - bb * bb;
  keep = keep && (det > 0.0);
  // ---- step 8: radius ----
  const double mid = 0.5 * (a + cc);
  const double disc = sqrt(fmax(kLambdaFloor, mid * mid - det));
  const double lam1 = mid + disc;
  const double rad = ceil(3.0 * sqrt(lam1));
  // ---- step 9: mean2d ----
  const double mx = fx * px * iz + (double)c.cx;
  const double my = fy * py * iz + (double)c.cy;
  // ---- step 10: tile rect ([3dgs] truncating rule, R8) ----
  int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
  if (keep) {
    const double gxd = b.gx, gyd = b.gy;
    x0 = (int)fmin(gxd, fmax(0.0, trunc((mx - rad) / kTile)));
    y0 = (int)fmin(gyd, fmax(0.0, trunc((my - rad) / kTile)));
    x1 = (int)fmin(gxd, fmax(0.0, trunc((mx + rad + (kTile - 1)) / kTile)));
    y1 = (int)fmin(gyd, fmax(0.0, trunc((my + rad + (kTile - 1)) / kTile)));
    keep = (x1 - x0) * (y1 - y0) > 0;
  }
  keep = keep && valid;
  // ---- FGS_TUNE_TILE_CULL: the tiles of the rect on which the Gaussian stays listed ----
  // Bit (ty - y0) * w + (tx - x0) of tmask; all ones without the cull or for rects over 64 tiles.  A
  // tile is dropped only if the minimum over its 16x16 pixel box of q2(d) = qa dx^2 + qb dx dy + qc dy^2
  // (d = pixel - mean) exceeds the blend's threshold thr_keep (below: log2(255 o) plus the margin that
  // covers fp32 evaluation): then every pixel of the tile has alpha < 1/255 in the blend (the blend's
  // sub-box cull applies the same bound to sub-boxes of the tile).
  unsigned long long tmask = ~0ull;
  int ntl = (x1 - x0) * (y1 - y0);
  // blend threshold: q2 = -p2 >= 0; alpha >= 1/255 needs q2 <= log2(255 o).  The margin covers the fp32
  // evaluation of q2 in the blend and in the cull tests, whose relative error grows with the conic's
  // condition number kappa = lambda_max / lambda_min of Sigma2.  (Computed here with the tile cull, which
  // needs it; after the counts otherwise, where fewer values are live.)
  float opac = 0.f, thr_keep = 0.f;
  double idet = 0.0;
  auto blend_threshold = [&]() {
    opac = 1.f / (1.f + __expf(-b.opacity[f][i]));
    idet = kLog2e / det;
    const float root = (float)sqrt(fmax(0.0, mid * mid - det));
    const float lam_max = (float)mid + root, lam_min = fmaxf((float)mid - root, 1e-30f);
    const float thr2 = __log2f(255.f * opac);
    thr_keep = thr2 + (fabsf(thr2) + 1.f) * (2e-3f + 4e-6f * (lam_max / lam_min));
  };
  if (CULL && keep) {
    blend_threshold();
    if (ntl <= 64) {
      // One x-interval per tile ROW: the ellipse E = {q2 <= thr_keep} is, in pixel offsets d = pixel - mean,
      // {d^T Sigma2^-1 d <= T} with T = 2 thr_keep / log2(e).  E meets the strip y in [yl, yh] of a tile row
      // in a convex set whose x-projection is [X_lo, X_hi]: x_hi(y) = (b/c) y + sqrt((T - y^2/c) det/c)
      // (Sigma2 = [[a, b], [b, c]]) is concave with its maximum at the ordinate y_r = (b/a) sqrt(T a) of
      // E's rightmost point, so X_hi = x_hi(clamp(y_r, yl, yh)) and, by symmetry, X_lo = x_lo(clamp(-y_r,
      // yl, yh)).  A tile of the row (it spans the strip's whole height) meets E iff its x-range meets
      // [X_lo, X_hi]: the listed tiles of a row are one contiguous run of mask bits.  Coefficients from
      // the fp64 covariance rounded to fp32 (no cancellation: det is formed in fp64); strip and interval are
      // widened by 0.01 px (+ 1e-5 relative), which covers the fp32 mean (ulp 0.002 px at 16384) and the
      // approximate square roots, on top of thr_keep's margin.
      tmask = 0ull;
      const float Tq = thr_keep * (float)(2.0 / kLog2e);
      if (Tq > 0.f) {
        const float fa = (float)a, fb = (float)bb, fc = (float)cc, fmx = (float)mx, fmy = (float)my;
        const float inv_c = __frcp_rn(fc), r_bc = fb * inv_c, s_c = (float)det * inv_c;
        const float ymax = sqrt_approx(Tq * fc) * 1.00001f + 1e-2f;
        const float y_r = fb * __frcp_rn(fa) * sqrt_approx(Tq * fa);
        const int w = x1 - x0;
        float yl = (float)(y0 * kTile) - fmy - 1e-2f;          // strip widened by 0.01 px (fp32 mean2d)
        for (int ty = y0, sh = 0; ty < y1; ++ty, sh += w, yl += (float)kTile) {
          const float yh = yl + ((float)(kTile - 1) + 2e-2f);
          if (yl > ymax || yh < -ymax) continue;
          const float ya = fminf(fmaxf(y_r, yl), yh), yb = fminf(fmaxf(-y_r, yl), yh);
          float X_hi = fmaf(r_bc, ya, sqrt_approx(fmaxf(0.f, fmaf(-ya * ya, inv_c, Tq)) * s_c));
          float X_lo = fmaf(r_bc, yb, -sqrt_approx(fmaxf(0.f, fmaf(-yb * yb, inv_c, Tq)) * s_c));
          X_hi += 1e-2f + 1e-5f * fabsf(X_hi);
          X_lo -= 1e-2f + 1e-5f * fabsf(X_lo);
          const int ta = max(x0, __float2int_ru((X_lo + fmx - (float)(kTile - 1)) * (1.f / kTile)));
          const int tb = min(x1 - 1, __float2int_rd((X_hi + fmx) * (1.f / kTile)));
          if (tb >= ta) {
            const int nrun = tb - ta + 1;
            const unsigned long long run = nrun >= 64 ? ~0ull : (1ull << nrun) - 1ull;
            tmask |= run << (sh + ta - x0);
          }
        }
      }
      ntl = __popcll(tmask);
    }
  }
  // ---- instance counts per tile (the bucket sizes of the duplication) ----
  __shared__ int sbox[4];
  __shared__ uint32_t scount[kAggTilesMax];
  uint32_t* cnt67 = cnt_ptr(b, f) + 6;
  count_tiles<CULL>(keep, x0, y0, x1, y1, tmask, tile_count, b.gx, b.gy, b.agg_tiles, cnt67, sbox, scount);
  if (!valid) return;
  if (!keep) {
    keys[i] = 0u;
    tt[i] = 0;
    rect[i] = make_uint2(0, 0);
    radii[i] = 0;
    return;
  }
  // ---- step 11: depth key = bits of fp32(p.z) (> 0.2 so unsigned order = depth order) ----
  keys[i] = __float_as_uint((float)pz);
  tt[i] = (uint32_t)ntl;      // tiles the Gaussian is listed on (the whole rect without the tile cull)
  if (CULL) ws_ptr<unsigned long long>(b.ws, b.ws_stride, f, b.L.tmask)[i] = tmask;
  rect[i] = make_uint2((uint32_t)x0 | ((uint32_t)y0 << 16), (uint32_t)x1 | ((uint32_t)y1 << 16));
  radii[i] = (int32_t)rad;
  // ---- step 12: SH colour at d = normalize(X - campos), campos = -R^T t (R10, R11) ----
  // (colour is not a decision: fp32 direction)
  const float cxw = -(c.R[0] * c.t[0] + c.R[3] * c.t[1] + c.R[6] * c.t[2]);
  const float cyw = -(c.R[1] * c.t[0] + c.R[4] * c.t[1] + c.R[7] * c.t[2]);
  const float czw = -(c.R[2] * c.t[0] + c.R[5] * c.t[1] + c.R[8] * c.t[2]);
  const float dx = (float)x - cxw, dy = (float)y - cyw, dz = (float)z - czw;
  const float dn = rsqrtf(dx * dx + dy * dy + dz * dz);
  float col[3];
  sh_colour<DEG>(b.sh[f] + (size_t)i * (DEG + 1) * (DEG + 1) * 3, dx * dn, dy * dn, dz * dn, col);
  // ---- blend record: mean2d as hi/lo fp32 pairs, conic pre-scaled to the log2 domain ----
  //   p2 = a2 dx^2 + b2 dx dy + c2 dy^2 = power * log2(e);  alpha = min(0.99, 2^(p2 + log2 o))
  const float mxh = (float)mx, myh = (float)my;
  const float mxl = (float)(mx - (double)mxh), myl = (float)(my - (double)myh);
  if (!CULL) blend_threshold();
  rec[3 * i + 0] = make_float4(mxh, myh, (float)(-0.5 * cc * idet), (float)(bb * idet));
  rec[3 * i + 1] = make_float4((float)(-0.5 * a * idet), __log2f(opac), fmaxf(col[0], 0.f), fmaxf(col[1], 0.f));
  rec[3 * i + 2] = make_float4(fmaxf(col[2], 0.f), mxl, myl, thr_keep);
}

// ------------------------------------------------------------------------------ tile scan (a7)
constexpr int kOrderBuckets = 1024;     // list-length buckets of the blend dispatch order
// Block-wide exclusive scan of one value per thread; returns the block total.
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t& excl, uint32_t* sw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sw[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < NT / 32 ? sw[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) sw[lane] = w;
  }
  __syncthreads();
  const uint32_t warp_off = warp > 0 ? sw[warp - 1] : 0;
  const uint32_t total = sw[NT / 32 - 1];
  excl = warp_off + x - v;
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kScanThreads) tile_scan_kernel(const __grid_constant__ RenderBatch b) {
  const int f = blockIdx.x;
  const uint32_t* tc = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.tile_count);
  uint32_t* cursor = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.cursor);
  uint2* ranges = ws_ptr<uint2>(b.ws, b.ws_stride, f, b.L.ranges);
  uint32_t* cnt = cnt_ptr(b, f);
  const int nt = b.ntiles;
  const int chunk = (nt + kScanThreads - 1) / kScanThreads;
  const int beg = min(nt, (int)threadIdx.x * chunk), end = min(nt, beg + chunk);
  uint64_t s = 0;
  for (int t = beg; t < end; ++t) s += tc[t];
  __shared__ uint32_t sw[32];
  uint32_t excl;
  // the total can exceed 2^32 only far past any capacity; saturate (overflow flag below)
  const uint32_t total = block_exclusive_scan<kScanThreads>((uint32_t)(s < 0xFFFFFFFFull ? s : 0xFFFFFFFFull), excl, sw);
  const uint64_t cap = (uint64_t)b.L.cap;
  uint64_t run = excl;
  for (int t = beg; t < end; ++t) {
    const uint64_t e = run + tc[t];
    cursor[t] = (uint32_t)(run < 0xFFFFFFFFull ? run : 0xFFFFFFFFull);
    ranges[t] = make_uint2((uint32_t)(run < cap ? run : cap), (uint32_t)(e < cap ? e : cap));
    run = e;
  }
  if (threadIdx.x == 0) {
    cnt[3] = total;
    cnt[1] = (uint32_t)((uint64_t)total < cap ? (uint64_t)total : cap);
    cnt[2] = (uint64_t)total > cap ? 1u : 0u;
    // binning path of this frame (radix.cu): the radix passes when the lists are long on average
    cnt[8] = (b.radix_mode == 2 || (b.radix_mode == 1 && (uint64_t)total >= (uint64_t)b.radix_min_list * (uint64_t)nt))
                 ? 1u : 0u;
  }
  // Blend dispatch order: the frame's tiles by descending list length (counting sort on the length,
  // capped), so the longest tiles start first and the grid does not end on a long tile — the blend
  // grid runs (rank-major, frame-minor) through it.  Order within a length bucket is arbitrary: every
  // tile is blended independently, so the images do not depend on it.
  __shared__ uint32_t hist[kOrderBuckets];
  for (int i = threadIdx.x; i < kOrderBuckets; i += kScanThreads) hist[i] = 0u;
  __syncthreads();
  for (int t = beg; t < end; ++t) {
    const uint32_t len = tc[t];
    atomicAdd(hist + (kOrderBuckets - 1 - (int)min(len, (uint32_t)(kOrderBuckets - 1))), 1u);
  }
  __syncthreads();
  static_assert(kOrderBuckets == kScanThreads, "one bucket per thread");
  uint32_t bexcl;
  const uint32_t hb = hist[threadIdx.x];
  block_exclusive_scan<kScanThreads>(hb, bexcl, sw);
  __syncthreads();
  hist[threadIdx.x] = bexcl;
  __syncthreads();
  uint32_t* order = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.order);
  for (int t = beg; t < end; ++t) {
    const uint32_t len = tc[t];
    const uint32_t pos = atomicAdd(hist + (kOrderBuckets - 1 - (int)min(len, (uint32_t)(kOrderBuckets - 1))), 1u);
    FGS_DCHECK(pos < (uint32_t)nt);
    order[pos] = (uint32_t)t;
  }
}

// ------------------------------------------------------------------------------ duplicate (a5)
// Key duplication of a CTA's Gaussians: one global cursor claim per touched tile for the
// whole CTA with the slots handed out in shared memory, or direct global atomics when the CTA's rect
// union exceeds agg_tiles (cnt7 counts those CTAs: fgs_render_aux.binning_direct[1]).  CULL: only the
// tiles of tmask (FGS_TUNE_TILE_CULL; the same mask preprocess counted with).
template <bool CULL>
__device__ __forceinline__ void emit_instances(bool keep, int x0, int y0, int x1, int y1, unsigned long long tmask,
                                               unsigned long long v, uint32_t* cursor, unsigned long long* inst,
                                               uint64_t cap, int gx, int gy, int agg_tiles, uint32_t* cnt7,
                                               int* sbox, uint32_t* sbase) {
  const AggBox box = cta_rect_union(keep, x0, y0, x1, y1, sbox);
  if (agg_fits(box, agg_tiles)) {
    const int bw = box.x1 - box.x0, area = bw * (box.y1 - box.y0);
    FGS_DCHECK(area <= kAggTilesMax && box.x0 >= 0 && box.y0 >= 0 && box.x1 <= gx && box.y1 <= gy);
    for (int q = threadIdx.x; q < area; q += blockDim.x) sbase[q] = 0;
    __syncthreads();
    if (keep)
      for_each_tile<CULL>(x0, y0, x1, y1, tmask,
                          [&](int tx, int ty) { atomicAdd(sbase + (ty - box.y0) * bw + (tx - box.x0), 1u); });
    __syncthreads();
    for (int q = threadIdx.x; q < area; q += blockDim.x)
      if (sbase[q]) sbase[q] = atomicAdd(cursor + (box.y0 + q / bw) * gx + box.x0 + q % bw, sbase[q]);
    __syncthreads();
    if (keep)
      for_each_tile<CULL>(x0, y0, x1, y1, tmask, [&](int tx, int ty) {
        const uint32_t pos = atomicAdd(sbase + (ty - box.y0) * bw + (tx - box.x0), 1u);
        if (pos < cap) inst[pos] = v;
      });
  } else {
    if (threadIdx.x == 0 && box.x1 > box.x0) atomicAdd(cnt7, 1u);
    if (keep)
      for_each_tile<CULL>(x0, y0, x1, y1, tmask, [&](int tx, int ty) {
        const uint32_t pos = atomicAdd(cursor + ty * gx + tx, 1u);
        if (pos < cap) inst[pos] = v;
      });
  }
}

__global__ void __launch_bounds__(256) duplicate_kernel(const __grid_constant__ RenderBatch b) {
  const int f = blockIdx.y;
  if (cnt_ptr(b, f)[8]) return;                 // the radix path emits this frame's instances (radix.cu)
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < b.n;
  const uint32_t* tt = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.tt);
  const bool keep = valid && tt[i] != 0;
  uint32_t key = 0;
  uint2 r = make_uint2(0, 0);
  if (keep) {
    key = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.keys)[i];
    r = ws_ptr<uint2>(b.ws, b.ws_stride, f, b.L.rect)[i];
  }
  uint32_t* cursor = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.cursor);
  unsigned long long* inst = ws_ptr<unsigned long long>(b.ws, b.ws_stride, f, b.L.inst);
  const int x0 = r.x & 0xFFFF, y0 = r.x >> 16, x1 = r.y & 0xFFFF, y1 = r.y >> 16;
  const uint64_t cap = (uint64_t)b.L.cap;
  const unsigned long long v = ((unsigned long long)key << 32) | (uint32_t)i;
  __shared__ int sbox[4];
  __shared__ uint32_t sbase[kAggTilesMax];
  if (b.tile_cull) {
    const unsigned long long tmask = keep ? ws_ptr<unsigned long long>(b.ws, b.ws_stride, f, b.L.tmask)[i] : 0ull;
    emit_instances<true>(keep, x0, y0, x1, y1, tmask, v, cursor, inst, cap, b.gx, b.gy, b.agg_tiles,
                         cnt_ptr(b, f) + 7, sbox, sbase);
  } else {
    emit_instances<false>(keep, x0, y0, x1, y1, ~0ull, v, cursor, inst, cap, b.gx, b.gy, b.agg_tiles,
                          cnt_ptr(b, f) + 7, sbox, sbase);
  }
}

// ------------------------------------------------------------------------------ tile sort (a6)
__device__ __forceinline__ int pow2_at_least(int v) {
  int p = 2;
  while (p < v) p <<= 1;
  return p;
}

// Lists of 2..sort_cap instances: one warp per tile sorts the list in registers — a bitonic network
// over N2 = 32 R keys in the blocked layout (key e = R lane + r in register r of lane `lane`), so that
// partners at distance j < R are compare-exchanged inside a thread and those at j >= R are exchanged
// with shuffles (lane ^ j/R) — and writes it back in place.  Longer lists are queued for
// long_sort_kernel.
//
// The network runs on 32-bit words, not on the 64-bit (depth_key << 32 | gid) instances: word e =
// ((depth_key - min) >> s) << log2(N2) | e, the list's depth keys relative to its minimum, shifted
// right by the s bits that do not fit next to the slot index e.  The map from depth key to prefix is
// monotone, so the words order the list by (depth key, gid) except inside groups of equal prefix,
// whose members come out in slot order; each sorted word's slot then fetches its 64-bit instance, and
// only when two neighbours share a prefix (an exact depth tie, or s > 0 and a near one) does an
// odd-even transposition over the written list put every such group in (depth key, gid) order.
// Half the registers, shuffles and compare instructions of the 64-bit network.
__device__ __forceinline__ void cmp_swap(uint32_t& a, uint32_t& c, bool up) {
  const bool sw = (a > c) == up;
  const uint32_t lo = sw ? c : a, hi = sw ? a : c;
  a = lo;
  c = hi;
}

// Bitonic network over the 32 R words of a warp in the blocked layout (word e = R lane + r in
// register r): thread-local stages for partner distances j < R, shuffles (lane ^ j/R) beyond.
template <int R>
__device__ __forceinline__ void warp_sort_words(uint32_t (&v)[R], int lane) {
  constexpr int N2 = 32 * R;
  // k < R: every stage is thread-local and every direction a compile-time function of r
#pragma unroll
  for (int k = 2; k < R; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if ((r & j) == 0) cmp_swap(v[r], v[r | j], (r & k) == 0);
    }
  }
  // k >= R: bit k of e = R lane + r comes from the lane, so the direction is one value per lane
#pragma unroll 1
  for (int k = R; k <= N2; k <<= 1) {
    if (k < 2) continue;
    const bool up = ((R * lane) & k) == 0;
#pragma unroll 1
    for (int j = k >> 1; j >= R; j >>= 1) {
      const int jl = j / R;                          // partner lane distance
      const bool keep_min = ((lane & jl) == 0) == up;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], jl);
        const bool lt = v[r] < o;
        v[r] = (lt == keep_min) ? v[r] : o;
      }
    }
    // j < R: the remaining stages of this k are thread-local (compile-time j)
#pragma unroll
    for (int j = R >> 1; j > 0; j >>= 1) {
      if (j < k) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if ((r & j) == 0) cmp_swap(v[r], v[r | j], up);
      }
    }
  }
}

template <int R>
__device__ __noinline__ void warp_sort_tile(const unsigned long long* src, unsigned long long* dst, int L,
                                            int lane) {
  constexpr int N2 = 32 * R;
  constexpr int LB = R == 1 ? 5 : R == 2 ? 6 : R == 4 ? 7 : R == 8 ? 8 : 9;   // log2(N2)
  FGS_DCHECK(L >= 1 && L <= N2);
  static_assert((1 << LB) == N2, "slot bits");
  uint32_t hk[R];
  uint32_t mn = 0xFFFFFFFFu, mx = 0u;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = R * lane + r;
    hk[r] = e < L ? (uint32_t)(src[e] >> 32) : 0u;
    if (e < L) { mn = min(mn, hk[r]); mx = max(mx, hk[r]); }
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  const uint32_t range = mx - mn;                       // L >= 1: mn <= mx
  const int s = max(0, (32 - __clz(range)) - (32 - LB));
  uint32_t v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = R * lane + r;
    v[r] = e < L ? (((hk[r] - mn) >> s) << LB) | (uint32_t)e : 0xFFFFFFFFu;
  }
  warp_sort_words<R>(v, lane);
  // slots -> instances (all fetched before any write: src may alias dst), then prefix ties
  unsigned long long out[R];
  bool tie = false;
  const uint32_t next0 = __shfl_down_sync(0xffffffffu, v[0], 1);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = R * lane + r;
    FGS_DCHECK(e >= L || (int)(v[r] & (uint32_t)(N2 - 1)) < L);
    out[r] = e < L ? src[v[r] & (uint32_t)(N2 - 1)] : 0ull;
    const uint32_t nx = r + 1 < R ? v[r + 1 < R ? r + 1 : r] : next0;
    if (e + 1 < L && (v[r] >> LB) == (nx >> LB)) tie = true;
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = R * lane + r;
    if (e < L) dst[e] = out[r];
  }
  if (__any_sync(0xffffffffu, tie)) {
    // odd-even transposition restricted to neighbours of equal prefix, until no swap (rare: ties)
    __syncwarp();
    for (;;) {
      bool swapped = false;
#pragma unroll 1
      for (int ph = 0; ph < 2; ++ph) {
        for (int e = 2 * lane + ph; e + 1 < L; e += 64) {
          const unsigned long long x = dst[e], y = dst[e + 1];
          if (((((uint32_t)(x >> 32) - mn) >> s) == (((uint32_t)(y >> 32) - mn) >> s)) && x > y) {
            dst[e] = y;
            dst[e + 1] = x;
            swapped = true;
          }
        }
        __syncwarp();
      }
      if (!__any_sync(0xffffffffu, swapped)) break;
    }
  }
}

// Sorts L <= 256 keys src[0..L) -> dst[0..L) with the smallest register network that holds them.
__device__ __forceinline__ void warp_sort_upto256(const unsigned long long* src, unsigned long long* dst, int L,
                                                  int lane) {
  if (L <= 32) warp_sort_tile<1>(src, dst, L, lane);
  else if (L <= 64) warp_sort_tile<2>(src, dst, L, lane);
  else if (L <= 128) warp_sort_tile<4>(src, dst, L, lane);
  else warp_sort_tile<8>(src, dst, L, lane);
}

// Warp-cooperative merge of sorted runs a[0..na) and b[0..nb) (shared memory) into out[0..na+nb):
// lane l produces a contiguous slice of the output, found by a merge-path binary search (keys are
// unique, so the split is exact).
__device__ __forceinline__ void warp_merge(const unsigned long long* a, int na, const unsigned long long* bq,
                                           int nb, unsigned long long* out, int lane) {
  const int n = na + nb;
  const int per = (n + 31) >> 5;
  const int d0 = min(n, lane * per), d1 = min(n, d0 + per);
  int lo = max(0, d0 - nb), hi = min(d0, na);
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (a[m] < bq[d0 - 1 - m]) lo = m + 1; else hi = m;
  }
  int ia = lo, ib = d0 - lo;
  unsigned long long va = ia < na ? a[ia] : ~0ull, vb = ib < nb ? bq[ib] : ~0ull;
  for (int d = d0; d < d1; ++d) {
    const bool ta = va < vb;
    out[d] = ta ? va : vb;
    if (ta) { ++ia; va = ia < na ? a[ia] : ~0ull; }
    else { ++ib; vb = ib < nb ? bq[ib] : ~0ull; }
  }
}

// One warp per tile.  Lists of up to 256 keys are sorted by one register network; longer ones (up to
// sort_cap <= 1024) as two runs sorted in registers into the warp's shared buffer (256-key runs up to
// 512, 512-key runs beyond: one merge level either way) and merged by merge path straight into the
// list.  Longer lists are queued for long_sort_kernel.
#ifndef FGS_TILE_SORT_WARPS
#define FGS_TILE_SORT_WARPS 2
#endif
constexpr int kTileSortWarps = FGS_TILE_SORT_WARPS;
// A warp's list (129..1024 instances) sorted by ONE bucket pass, the warp-level form of long_sort_bucket
// below: the 64-bit instances (depth_key << 32 | gid) are all distinct, so with the monotone map
// bucket(x) = (depth_key - list min) >> shift (512 buckets) an instance's final position is its bucket's
// start + the number of its bucket's instances below it.  Passes over the list (global reads, L1-resident
// after the first): depth range, bucket counts (shared-memory atomics), a warp scan of the 512 counts
// (16 per lane; counters padded by 4 words per 16 so the lanes' 16-B loads do not conflict), a scatter
// into the warp's shared buffer S in bucket order, and the rank within the bucket (<= kWBucketMax
// comparisons) writing the list in place.  ~40 instructions per instance + ~110 per list against the
// O(L log^2 L) register networks (D: ~220 per instance at the mean list of 240).  Returns false, the
// list untouched, when a bucket holds more than kWBucketMax instances (skewed depths, exact ties): the
// caller then sorts by the networks.
constexpr int kWSortBits = 9, kWSortBuckets = 1 << kWSortBits;
constexpr int kWSortCntWords = kWSortBuckets + kWSortBuckets / 4;     // 4 pad words per 16 counters
#ifndef FGS_WBUCKET_MAX
#define FGS_WBUCKET_MAX 32
#endif
constexpr uint32_t kWBucketMax = FGS_WBUCKET_MAX;
#ifndef FGS_WSORT_MIN
#define FGS_WSORT_MIN 128
#endif
constexpr int kWSortMin = FGS_WSORT_MIN;              // shorter lists stay on the register networks
__device__ __forceinline__ int wcnt_idx(uint32_t i) { return (int)(i + ((i >> 4) << 2)); }
__device__ __forceinline__ bool warp_sort_bucket(unsigned long long* inst, int L, int lane, unsigned long long* S,
                                                 uint32_t* cnt) {
  uint32_t mn = 0xFFFFFFFFu, mx = 0u;
  for (int q = lane; q < L; q += 32) {
    const uint32_t h = (uint32_t)(inst[q] >> 32);
    mn = min(mn, h);
    mx = max(mx, h);
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  const int shift = max(0, (32 - __clz(mx - mn)) - kWSortBits);
  for (int k = lane; k < kWSortCntWords / 4; k += 32) reinterpret_cast<uint4*>(cnt)[k] = make_uint4(0u, 0u, 0u, 0u);
  __syncwarp();
  for (int q = lane; q < L; q += 32)
    atomicAdd(&cnt[wcnt_idx(((uint32_t)(inst[q] >> 32) - mn) >> shift)], 1u);
  __syncwarp();
  // lane owns buckets [16 lane, 16 lane + 16) = words [20 lane, 20 lane + 16)
  uint4* cp = reinterpret_cast<uint4*>(cnt + 20 * lane);
  uint32_t c[16], tot = 0;
  bool big = false;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint4 v = cp[k];
    c[4 * k + 0] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    tot += c[i];
    big |= c[i] > kWBucketMax;
  }
  if (__any_sync(0xffffffffu, big)) return false;
  uint32_t run = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, run, o);
    if (lane >= o) run += y;
  }
  run -= tot;                                        // exclusive
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t s0 = run;
    run += c[i];
    c[i] = s0;                                       // bucket start; the scatter's cursor
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) cp[k] = make_uint4(c[4 * k + 0], c[4 * k + 1], c[4 * k + 2], c[4 * k + 3]);
  __syncwarp();
  for (int q = lane; q < L; q += 32) {
    const unsigned long long x = inst[q];
    const uint32_t pos = atomicAdd(&cnt[wcnt_idx(((uint32_t)(x >> 32) - mn) >> shift)], 1u);
    FGS_DCHECK(pos < (uint32_t)L);
    S[pos] = x;
  }
  __syncwarp();                                      // cnt[k] is now the END of bucket k
  for (int q = lane; q < L; q += 32) {
    const unsigned long long x = S[q];
    const uint32_t bk = ((uint32_t)(x >> 32) - mn) >> shift;
    const uint32_t st = bk ? cnt[wcnt_idx(bk - 1)] : 0u, en = cnt[wcnt_idx(bk)];
    FGS_DCHECK(st <= (uint32_t)q && (uint32_t)q < en && en - st <= kWBucketMax && en <= (uint32_t)L);
    uint32_t r = st;
    for (uint32_t k = st; k < en; ++k) r += S[k] < x;
    inst[r] = x;
  }
  return true;
}

__global__ void __launch_bounds__(32 * kTileSortWarps) tile_sort_kernel(const __grid_constant__ RenderBatch b) {
  // 1-D grid over (rank group, frame), frame-minor, tiles in descending list length (as the blend)
  const int f = (int)(blockIdx.x % (unsigned)b.n_frames);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)(blockIdx.x / (unsigned)b.n_frames) * kTileSortWarps + warp;
  if (rank >= b.ntiles) return;                 // no CTA-wide barriers below
  if (cnt_ptr(b, f)[8]) return;                 // radix path: the lists are already in order
  const int tile = (int)ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.order)[rank];
  FGS_DCHECK(tile >= 0 && tile < b.ntiles);
  const uint2 rg = ws_ptr<uint2>(b.ws, b.ws_stride, f, b.L.ranges)[tile];
  const int L = (int)(rg.y - rg.x);
  FGS_DCHECK(rg.x <= rg.y && (int64_t)rg.y <= b.L.cap);
  if (L <= 1) return;
  if (L > b.sort_cap) {
    if (lane == 0) {
      const uint32_t w = atomicAdd(cnt_ptr(b, f) + 4, 1u);
      ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.long_list)[w] = (uint32_t)tile;
    }
    return;
  }
  unsigned long long* inst = ws_ptr<unsigned long long>(b.ws, b.ws_stride, f, b.L.inst) + rg.x;
  __shared__ unsigned long long buf[kTileSortWarps][kBlendSortMax];
  __shared__ __align__(16) uint32_t wcnt[kTileSortWarps][kWSortCntWords];
  // lists over kWSortMin instances: one bucket pass (FGS_TUNE_LONG_SORT = 1, the default); the register
  // networks below for shorter lists, skewed depth distributions, or FGS_TUNE_LONG_SORT = 0
  if (b.long_sort && L > kWSortMin) {
    if (warp_sort_bucket(inst, L, lane, buf[warp], wcnt[warp])) return;
    __syncwarp();
  }
  if (L <= 256) {
    warp_sort_upto256(inst, inst, L, lane);
    return;
  }
  // two runs sorted in registers into the warp's shared buffer (256 + up to 256, or 512 + up to 512,
  // each by the smallest network that holds it), one merge-path merge into the list
  unsigned long long* A = buf[warp];
  FGS_DCHECK(L <= kBlendSortMax);
  const int h = L <= 512 ? 256 : 512;
  if (h == 256) warp_sort_upto256(inst, A, 256, lane);
  else warp_sort_tile<16>(inst, A, 512, lane);
  if (L - h <= 256) warp_sort_upto256(inst + h, A + h, L - h, lane);
  else warp_sort_tile<16>(inst + h, A + h, L - h, lane);
  __syncwarp();
  warp_merge(A, h, A + h, L - h, inst, lane);
}

// Lists longer than b.sort_cap: one CTA (8 warps) per list, persistent over the frame's worklist.
// Up to kCtaSortMax keys: runs of 256 sorted in registers by the warps, then merge-path levels over
// all 256 threads, ping-ponging between two shared buffers.  Longer lists: segments of kCtaSortMax
// sorted that way in place, then merge-path levels in global memory through the inst2 scratch.
constexpr int kCtaSortMax = 4096;
constexpr size_t kLongSortSmem = 2 * kCtaSortMax * sizeof(unsigned long long);   // 64 KB dynamic

template <typename K>
__device__ __forceinline__ void block_merge(const K* a, int na, const K* bq, int nb, K* out, int t, int nt) {
  const int n = na + nb;
  const int per = (n + nt - 1) / nt;
  const int d0 = min(n, t * per), d1 = min(n, d0 + per);
  if (d0 >= d1) return;
  int lo = max(0, d0 - nb), hi = min(d0, na);
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (a[m] < bq[d0 - 1 - m]) lo = m + 1; else hi = m;
  }
  int ia = lo, ib = d0 - lo;
  const K kmax = (K)~(K)0;
  K va = ia < na ? a[ia] : kmax, vb = ib < nb ? bq[ib] : kmax;
  for (int d = d0; d < d1; ++d) {
    const bool ta = va < vb;
    out[d] = ta ? va : vb;
    if (ta) { ++ia; va = ia < na ? a[ia] : kmax; }
    else { ++ib; vb = ib < nb ? bq[ib] : kmax; }
  }
}

// CTA-wide bitonic network over the NT R words of the CTA in the blocked layout (word e = R t + r in
// register r of thread t), ascending: thread-local stages for partner distances j < R, warp shuffles for
// partner threads in the same warp (j / R < 32), a shared-memory exchange (transposed: conflict-free) for
// partners in other warps.  The CTA analogue of warp_sort_words.
template <int R>
__device__ __forceinline__ void cta_bitonic_words(uint32_t (&v)[R], uint32_t* xbuf) {
  constexpr int NT = kLargeSortThreads;
  constexpr int N2 = NT * R;
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 2; k < R; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if ((r & j) == 0) cmp_swap(v[r], v[r | j], (r & k) == 0);
    }
  }
#pragma unroll 1
  for (int k = R; k <= N2; k <<= 1) {
    if (k < 2) continue;
    const bool up = ((R * t) & k) == 0;
#pragma unroll 1
    for (int j = k >> 1; j >= R; j >>= 1) {
      const int jt = j / R;                          // partner thread distance
      const bool keep_min = ((t & jt) == 0) == up;
      if (jt < 32) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], jt);
          v[r] = ((v[r] < o) == keep_min) ? v[r] : o;
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) xbuf[r * NT + t] = v[r];
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t o = xbuf[r * NT + (t ^ jt)];
          v[r] = ((v[r] < o) == keep_min) ? v[r] : o;
        }
        __syncthreads();
      }
    }
#pragma unroll
    for (int j = R >> 1; j > 0; j >>= 1) {
      if (j < k) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if ((r & j) == 0) cmp_swap(v[r], v[r | j], up);
      }
    }
  }
}

// words[0..L) (smem) sorted ascending in place by one CTA bitonic network of the smallest power of two
// >= L (pads 0xFFFFFFFF sort last)
template <int R>
__device__ __forceinline__ void cta_sort_words_bitonic(uint32_t* words, int L, uint32_t* xbuf) {
  uint32_t v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = R * threadIdx.x + r;
    v[r] = e < L ? words[e] : 0xFFFFFFFFu;
  }
  __syncthreads();
  cta_bitonic_words<R>(v, xbuf);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = R * threadIdx.x + r;
    if (e < L) words[e] = v[r];
  }
  __syncthreads();
}

// Sorts src[0..L) (L <= kCtaSortMax) into dst[0..L) (may alias src) with the whole CTA, on 32-bit
// words as the warp sorts: prefix of the depth key relative to the segment minimum (shifted right by
// the range bits that do not fit beside 12 slot bits) | slot.  One CTA bitonic network (registers,
// shuffles, shared-memory exchanges) over the next power of two of L words — round 2: replaced warp runs
// + merge-path levels (N = 1M tile sort 171 -> 154, 3M 748 -> 674 us per frame, unchanged below) — then
// neighbours of equal prefix are put in (depth key, gid) order and each word's slot fetches its
// instance for the output.  The segment is read from global memory once.  sm: kLongSortSmem.
__device__ void cta_sort_words(const unsigned long long* src, unsigned long long* dst, int L, unsigned long long* sm) {
  static_assert(kCtaSortMax == 4096, "12 slot bits");
  constexpr int SB = 12;
  constexpr int NT = kLargeSortThreads;
  uint32_t* wA = reinterpret_cast<uint32_t*>(sm);
  uint32_t* wB = wA + kCtaSortMax;
  FGS_DCHECK(L >= 1 && L <= kCtaSortMax);
  unsigned long long* stage = sm + kCtaSortMax;
  __shared__ uint32_t s_mn, s_mx;
  const int lane = threadIdx.x & 31;
  // the segment is read from global memory ONCE, into the stage; everything after works in shared memory
  uint32_t mn = 0xFFFFFFFFu, mx = 0u;
  for (int q = threadIdx.x; q < L; q += NT) {
    const unsigned long long x = src[q];
    stage[q] = x;
    const uint32_t h = (uint32_t)(x >> 32);
    mn = min(mn, h);
    mx = max(mx, h);
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (threadIdx.x == 0) { s_mn = 0xFFFFFFFFu; s_mx = 0u; }
  __syncthreads();
  if (lane == 0) { atomicMin(&s_mn, mn); atomicMax(&s_mx, mx); }
  __syncthreads();
  mn = s_mn;
  mx = s_mx;
  const int s = max(0, (32 - __clz(mx - mn)) - (32 - SB));
  for (int q = threadIdx.x; q < L; q += NT)
    wA[q] = (((((uint32_t)(stage[q] >> 32)) - mn) >> s) << SB) | (uint32_t)q;
  __syncthreads();
  if (L <= 1024) cta_sort_words_bitonic<4>(wA, L, wB);
  else if (L <= 2048) cta_sort_words_bitonic<8>(wA, L, wB);
  else cta_sort_words_bitonic<16>(wA, L, wB);
  // neighbours of equal prefix (exact depth ties, or near ones when s > 0) put in (depth key, gid) order:
  // an odd-even transposition on the WORDS comparing the instances their slots point to (skipped by a
  // vote when there are none)
  constexpr uint32_t kSlot = (1u << SB) - 1u;
  bool tie = false;
  for (int q = threadIdx.x; q + 1 < L; q += NT)
    if ((wA[q] >> SB) == (wA[q + 1] >> SB)) tie = true;
  if (__syncthreads_or(tie)) {
    for (;;) {
      bool swapped = false;
      for (int ph = 0; ph < 2; ++ph) {
        for (int e = 2 * threadIdx.x + ph; e + 1 < L; e += 2 * NT) {
          const uint32_t x = wA[e], y = wA[e + 1];
          if ((x >> SB) == (y >> SB) && stage[x & kSlot] > stage[y & kSlot]) {
            wA[e] = y;
            wA[e + 1] = x;
            swapped = true;
          }
        }
        __syncthreads();
      }
      if (!__syncthreads_or(swapped)) break;
    }
  }
  for (int q = threadIdx.x; q < L; q += NT) {
    FGS_DCHECK((int)(wA[q] & kSlot) < L);
    dst[q] = stage[wA[q] & kSlot];
  }
  __syncthreads();
}

// A whole long list A[0..L) sorted in place by ONE bucket pass: the 64-bit instances (depth_key << 32 |
// gid) are all distinct, so bucketing them by the top kSortBucketBits of (depth_key - list min) — a
// monotone map — and placing each at its bucket's start + the number of its bucket's instances below it
// gives exactly the ascending (depth, gid) order, with no merge levels and no tie fixup.  Passes: the
// depth range (one read), bucket counts (shared-memory atomics), an exclusive scan, a scatter into the
// buckets in any order (into shared memory when L <= kLongSortSmem / 8, else the inst2 scratch), and the
// per-instance rank within its bucket (<= kBucketMax comparisons) writing A in final order (nearly
// coalesced: a bucket's instances land in its own range).  Returns false, A untouched, when a bucket holds
// more than kBucketMax instances (a skewed depth distribution; the caller sorts by the networks then).
// About 45 instructions per instance against ~150+ for the word network at 4096 (round 2).
constexpr int kSortBuckets = 2048;
constexpr int kSortBucketBits = 11;
constexpr uint32_t kBucketMax = 64;
__device__ bool long_sort_bucket(unsigned long long* A, unsigned long long* B, int L, unsigned long long* sm,
                                 uint32_t* paths) {
  constexpr int NT = kLargeSortThreads;
  constexpr int PER = kSortBuckets / NT;
  static_assert(kSortBuckets % NT == 0, "layout");
  __shared__ uint32_t cnt[kSortBuckets];
  __shared__ uint32_t s_scan[NT / 32];
  __shared__ uint32_t s_mn, s_mx, s_big;
  const int lane = threadIdx.x & 31;
  uint32_t mn = 0xFFFFFFFFu, mx = 0u;
  for (int q = threadIdx.x; q < L; q += NT) {
    const uint32_t h = (uint32_t)(A[q] >> 32);
    mn = min(mn, h);
    mx = max(mx, h);
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  for (int i = threadIdx.x; i < kSortBuckets; i += NT) cnt[i] = 0;
  if (threadIdx.x == 0) { s_mn = 0xFFFFFFFFu; s_mx = 0u; s_big = 0u; }
  __syncthreads();
  if (lane == 0) { atomicMin(&s_mn, mn); atomicMax(&s_mx, mx); }
  __syncthreads();
  mn = s_mn;
  const int shift = max(0, (32 - __clz(s_mx - mn)) - kSortBucketBits);
  for (int q = threadIdx.x; q < L; q += NT) atomicAdd(&cnt[((uint32_t)(A[q] >> 32) - mn) >> shift], 1u);
  __syncthreads();
  uint32_t c[PER], tot = 0;
  bool big = false;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    c[i] = cnt[PER * threadIdx.x + i];
    tot += c[i];
    big |= c[i] > kBucketMax;
  }
  uint32_t run;
  block_exclusive_scan<NT>(tot, run, s_scan);      // (ends with a barrier)
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    cnt[PER * threadIdx.x + i] = run;              // bucket start; the scatter's cursor
    run += c[i];
  }
  if (big) s_big = 1u;
  __syncthreads();
  if (s_big) return false;                         // CTA-uniform
  const bool in_smem = L <= (int)(kLongSortSmem / sizeof(unsigned long long));
  unsigned long long* tmp = in_smem ? sm : B;
  if (threadIdx.x == 0) atomicAdd(paths + (in_smem ? 0 : 1), 1u);   // debug evidence (long_sort_paths)
  for (int q = threadIdx.x; q < L; q += NT) {
    const unsigned long long x = A[q];
    tmp[atomicAdd(&cnt[((uint32_t)(x >> 32) - mn) >> shift], 1u)] = x;
  }
  __syncthreads();                                 // cnt[k] is now the END of bucket k
  for (int q = threadIdx.x; q < L; q += NT) {
    const unsigned long long x = tmp[q];
    const uint32_t bk = ((uint32_t)(x >> 32) - mn) >> shift;
    const uint32_t st = bk ? cnt[bk - 1] : 0u, en = cnt[bk];
    FGS_DCHECK(st <= (uint32_t)q && (uint32_t)q < en && en - st <= kBucketMax);
    uint32_t r = st;
    for (uint32_t k = st; k < en; ++k) r += tmp[k] < x;
    A[r] = x;
  }
  __syncthreads();
  return true;
}

__device__ void long_sort_one(const RenderBatch& b, int f, int tile, unsigned long long* sm) {
  const uint2 rg = ws_ptr<uint2>(b.ws, b.ws_stride, f, b.L.ranges)[tile];
  const int L = (int)(rg.y - rg.x);
  unsigned long long* A = ws_ptr<unsigned long long>(b.ws, b.ws_stride, f, b.L.inst) + rg.x;
  unsigned long long* B = ws_ptr<unsigned long long>(b.ws, b.ws_stride, f, b.L.inst2) + rg.x;
  uint32_t* paths = cnt_ptr(b, f) + 9;             // cnt[9..11]: fgs_render_aux.long_sort_paths
  if (b.long_sort && long_sort_bucket(A, B, L, sm, paths)) return;
  if (threadIdx.x == 0) atomicAdd(paths + 2, 1u);
  for (int c0 = 0; c0 < L; c0 += kCtaSortMax) {
    const int l = min(kCtaSortMax, L - c0);
    cta_sort_words(A + c0, A + c0, l, sm);
  }
  if (L > kCtaSortMax && L <= 2 * kCtaSortMax) {
    // two sorted segments: both back into shared memory and one merge-path merge straight into the
    // list (the merge reads shared memory, not dependent L2 loads as the global levels below)
    const int L1 = L - kCtaSortMax;
    for (int q = threadIdx.x; q < L; q += kLargeSortThreads) sm[q] = A[q];
    __syncthreads();
    block_merge(sm, kCtaSortMax, sm + kCtaSortMax, L1, A, threadIdx.x, kLargeSortThreads);
    __syncthreads();
    return;
  }
  unsigned long long* src = A;
  unsigned long long* dst = B;
  for (int w = kCtaSortMax; w < L; w <<= 1) {
    for (int s0 = 0; s0 < L; s0 += 2 * w) {
      const int na = min(w, L - s0), nb = max(0, min(w, L - s0 - w));
      block_merge(src + s0, na, src + s0 + na, nb, dst + s0, threadIdx.x, kLargeSortThreads);
    }
    __syncthreads();
    unsigned long long* t = src; src = dst; dst = t;
  }
  if (src != A) {
    for (int q = threadIdx.x; q < L; q += kLargeSortThreads) A[q] = src[q];
    __syncthreads();
  }
}

// Persistent CTAs share ONE queue over the long lists of all frames of the batch (frame 0's cnt[5] is
// the claim counter, zeroed by clear_kernel), so frames with many long lists do not leave the CTAs of
// frames with few idle; within a frame the worklist is roughly longest-first (tile_sort_kernel runs
// the tiles in descending length order).
__global__ void __launch_bounds__(kLargeSortThreads) long_sort_kernel(const __grid_constant__ RenderBatch b) {
  extern __shared__ unsigned long long long_sm[];
  __shared__ uint32_t s_item;
  uint32_t* claim = cnt_ptr(b, 0) + 5;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(claim, 1u);
    __syncthreads();
    uint32_t w = s_item;
    __syncthreads();
    int f = 0;
    for (; f < b.n_frames; ++f) {
      const uint32_t n_long = cnt_ptr(b, f)[4];
      if (w < n_long) break;
      w -= n_long;
    }
    if (f == b.n_frames) return;                    // CTA-uniform
    FGS_DCHECK(w < (uint32_t)b.ntiles);
    long_sort_one(b, f, (int)ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.long_list)[w], long_sm);
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ blend (Eq. 4)
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// thr: the exponent threshold of the alpha >= 1/255 test while the pixel is live, +inf once it has
// stopped (or lies outside the image) — one compare then covers both "live" and "alpha >= 1/255"
// (no separate done flag to test and update per evaluation)
struct PixelState {
  float2 c01;                // red, green: one packed FFMA2 per step
  float T, c2, thr;
  uint32_t ncon, nev;
  __device__ __forceinline__ bool done() const { return thr == __int_as_float(0x7f800000); }
};

// Eq. 4 for one pixel and one Gaussian; e = p2 + log2(o) with p2 = power * log2(e) (R9: skip if
// power > 0 or alpha < 1/255; stop, without adding it, when T (1 - alpha) < 1e-4).
//  * power > 0 cannot happen for a kept Gaussian: det > 0 and a > 0 make the conic positive definite,
//    so power <= 0 exactly (p2 > 0 could only come from fp32 rounding at power ~ 0, where the fp64
//    oracle includes the Gaussian too) — no test.
//  * alpha >= 1/255 is decided on the exponent, e >= log2(1/255) (min(0.99, .) cannot take alpha
//    below 1/255), which takes the decision off the ex2 latency; the two forms differ only within the
//    ex2.approx error of the threshold, inside the parity band of reading P1.
constexpr float kLog2AlphaMin = -7.9943534368588578f;   // log2(1/255)
template <bool DBG>
__device__ __forceinline__ void blend_step(PixelState& s, float e, float lo, float r, float g, float bch,
                                           uint32_t pos) {
  (void)lo;
  const float alpha = fminf(kAlphaMax, ex2_approx(e));
  const bool ok = e >= s.thr;              // live and alpha >= 1/255 (s.thr = kLog2AlphaMin or +inf)
  const float test_T = fmaf(-alpha, s.T, s.T);
  const bool stop = ok && test_T < kTMin;
  if (ok && !stop) {
    const float w = alpha * s.T;
    s.c01 = ffma2(make_float2(r, g), make_float2(w, w), s.c01);   // FFMA2, bit-equal to 2 x fmaf
    s.c2 = fmaf(bch, w, s.c2);
    s.T = test_T;
    if (DBG) s.ncon += 1u;
  }
  s.thr = stop ? __int_as_float(0x7f800000) : s.thr;
  if (DBG && stop) s.nev = pos;
}

// Conservative ellipse-vs-box cull: a half-box is skipped only if q2(d) = qa dx^2 + qb dx dy + qc dy^2
// (the negated log2-domain exponent, PSD) exceeds thr over the whole box of offsets d = pixel - mean.
// The minimum of a convex quadratic over a box that does not contain its minimiser d = 0 lies on a
// face whose half-space excludes 0 (KKT), so at most one x-face and one y-face are candidates; on
// each the 1-D minimiser is clamped to the face.  An inexact minimiser only raises the computed value
// by qc delta^2 (quadratic in its error), far inside thr's margin.
// face_min / subboxes_may_reach (fgs_internal.cuh): shared with the backward re-walk (backward.cu).

// NP pixels per lane: warp w of the tile's NW = 64/NP... warps owns a column block; lane l owns pixel
// (x, y + 4k), k < NP, of that block (x = l & 7, y = l >> 3).  Sub-box k = rows [4k, 4k+4) of the block.
constexpr int kBlendPix = 4;                         // pixels per lane
constexpr int kBlendBatch = 128;                     // records staged per batch (6 KB of smem)
constexpr int kBlendWarps = 256 / (32 * kBlendPix);  // warps per 16x16 tile (2)

#ifndef FGS_BLEND_MIN_CTAS
#define FGS_BLEND_MIN_CTAS 24   // 40 registers (sweep: DESIGN 7b / 7c)
#endif
template <bool DBG>
__global__ void __launch_bounds__(32 * kBlendWarps, FGS_BLEND_MIN_CTAS) blend_kernel(const __grid_constant__ RenderBatch b) {
  // One CTA (kBlendWarps warps) per 16x16 tile.  Warp w owns the 8-wide column block x in [8w, 8w+8)
  // of all 16 rows; lane l owns the kBlendPix pixels (8w + (l&7), (l>>3) + 4k).  The tile's list (sorted
  // by (depth, gid)) is walked in batches of kBlendBatch records staged in smem; per 32 Gaussians each lane tests
  // one against the exact ellipse bound over the warp's kBlendPix 8x4 sub-boxes, and the warp
  // evaluates, in list order, each Gaussian on the sub-boxes it can reach (warp-uniform branches), so
  // the per-Gaussian loads and dx terms are shared by up to kBlendPix pixels per lane.
  constexpr int NT = 32 * kBlendWarps;
  // 1-D grid over (rank, frame), frame-minor: the tiles of every frame in descending list length
  // (tile_scan_kernel), so the longest lists of all frames are dispatched first
  const int f = (int)(blockIdx.x % (unsigned)b.n_frames);
  const int rank = (int)(blockIdx.x / (unsigned)b.n_frames);
  const int tile = (int)ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.order)[rank];
  const int tx = tile % b.gx, ty = tile / b.gx;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int bx0 = warp * 8;                                       // column block origin, tile-relative
  const int lxi = bx0 + (lane & 7), lyi = lane >> 3;
  const int pxi = tx * kTile + lxi, py0 = ty * kTile + lyi;
  const uint2 rg = ws_ptr<uint2>(b.ws, b.ws_stride, f, b.L.ranges)[tile];
  const int L = (int)(rg.y - rg.x);
  const unsigned long long* inst = ws_ptr<unsigned long long>(b.ws, b.ws_stride, f, b.L.inst) + rg.x;
  const float4* rec = ws_ptr<float4>(b.ws, b.ws_stride, f, b.L.rec);
  // staged records, one 48-B struct per list entry so one address serves all three loads
  struct __align__(16) SRec { float4 a, q; float2 c; float2 pad; };
  constexpr int BATCH = kBlendBatch;
  __shared__ SRec srec[BATCH];
  const float tx0 = (float)(tx * kTile), ty0 = (float)(ty * kTile);
  const float lx = (float)lxi, ly = (float)lyi;
  const float2 nl = make_float2(-lx, -ly);   // a - l == a + (-l) exactly
  const float bxl = (float)bx0, bxh = (float)(bx0 + 7);
  uint32_t n_tested = 0, n_evald = 0;    // DBG: per-warp cull statistics (sub-box evaluations)
  PixelState P[kBlendPix];
#pragma unroll
  for (int k = 0; k < kBlendPix; ++k) {
    const bool in = pxi < b.width && py0 + 4 * k < b.height;
    P[k] = PixelState{make_float2(0.f, 0.f), 1.f, 0.f, in ? kLog2AlphaMin : __int_as_float(0x7f800000), 0u, (uint32_t)L};
  }
  auto all_done = [&]() {
    bool d = true;
#pragma unroll
    for (int k = 0; k < kBlendPix; ++k) d = d && P[k].done();
    return d;
  };
  for (int start = 0; start < L; start += BATCH) {
    if (__syncthreads_count(all_done()) == NT) break;
#pragma unroll
    for (int k = 0; k < BATCH / NT; ++k) {
      const int idx = start + threadIdx.x + NT * k;
      if (idx < L) {
        const uint32_t g = (uint32_t)inst[idx];
        FGS_DCHECK((int64_t)g < b.n && (int64_t)rg.x + idx < b.L.cap);
        float4 a = rec[3 * g + 0];
        const float4 c = rec[3 * g + 2];
        a.x = (a.x - tx0) + c.y;      // tile-relative mean: exact hi difference + lo part
        a.y = (a.y - ty0) + c.z;
        SRec& d = srec[threadIdx.x + NT * k];
        d.a = a;
        d.q = rec[3 * g + 1];
        d.c = make_float2(c.x, c.w);
      }
    }
    __syncthreads();
    const int cnt = min(BATCH, L - start);
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      uint32_t live = 0;
#pragma unroll
      for (int k = 0; k < kBlendPix; ++k)
        if (__any_sync(0xffffffffu, !P[k].done())) live |= 1u << k;
      if (!live) break;
      const int jt = c0 + lane;
      bool reach[kBlendPix];
#pragma unroll
      for (int k = 0; k < kBlendPix; ++k) reach[k] = jt < cnt;
      if (jt < cnt && b.cull) {
        // b.cull = 0 (FGS_TUNE_BLEND_CULL): every Gaussian on every live sub-box — the unculled Eq. 4
        // loop, which the culled one must equal bit for bit
        const float4 a = srec[jt].a;
        subboxes_reach<kBlendPix>(-a.z, -a.w, -srec[jt].q.x, srec[jt].c.y, bxl - a.x, bxh - a.x, -a.y, reach);
      }
      // sub-box masks straight from the per-lane predicates; a stopped sub-box (not live) gets none
      uint32_t mk[kBlendPix];
#pragma unroll
      for (int k = 0; k < kBlendPix; ++k) mk[k] = __ballot_sync(0xffffffffu, reach[k]) & (0u - ((live >> k) & 1u));
      // walked from the most significant bit of the bit-reversed masks (= list order): the next
      // Gaussian is one FLO (bfind), its bit one shift, clearing it one XOR
      uint32_t m = 0;
#pragma unroll
      for (int k = 0; k < kBlendPix; ++k) {
        m |= mk[k];
        mk[k] = __brev(mk[k]);
      }
      m = __brev(m);
      if (DBG) {
        n_tested += (uint32_t)min(32, cnt - c0);
#pragma unroll
        for (int k = 0; k < kBlendPix; ++k) n_evald += __popc(mk[k]);
      }
      // record of bit h = list entry c0 + 31 - h: one multiply-add from the chunk's last record
      const char* rlast = reinterpret_cast<const char*>(&srec[c0 + 31]);
      while (m) {
        int h;                                 // bit index of m's most significant set bit (FLO)
        asm("bfind.u32 %0, %1;" : "=r"(h) : "r"(m));
        const uint32_t hb = 1u << h;
        m ^= hb;
        const SRec& rj = *reinterpret_cast<const SRec*>(rlast - h * (int)sizeof(SRec));
        const float4 a = rj.a, q = rj.q;
        const float bch = rj.c.x;
        // packed pairs (each half rounded as its scalar op): (dx, dy0) = mean - pixel, (a2 dx, b2 dx)
        const float2 d0 = fadd2(make_float2(a.x, a.y), nl);
        const float dx = d0.x, dy0 = d0.y;
        const float2 abdx = fmul2(make_float2(a.z, a.w), make_float2(dx, dx));
        const float bdx = abdx.y;                                // b2 dx, shared by the lane's pixels
        const float base = fmaf(abdx.x, dx, q.y);                // a2 dx^2 + log2(o)
        const uint32_t pos = (uint32_t)(start + c0 + 31 - h + 1);
#pragma unroll
        for (int k = 0; k < kBlendPix; ++k) {
          if (mk[k] & hb) {
            const float dy = dy0 - 4.f * k;
            const float e = fmaf(dy, fmaf(q.x, dy, bdx), base);
            blend_step<DBG>(P[k], e, q.y, q.z, q.w, bch, pos);
          }
        }
      }
    }
    __syncthreads();
  }
  if (DBG && b.blend_work && f == 0 && lane == 0) {
    atomicAdd(b.blend_work, (unsigned long long)n_evald);
    atomicAdd(b.blend_work + 1, (unsigned long long)n_tested);
  }
  const size_t hw = (size_t)b.width * b.height;
  float* img = b.image[f];
  const FrameCam& cm = b.cam[f];
#pragma unroll
  for (int k = 0; k < kBlendPix; ++k) {
    const PixelState& s = P[k];
    const int py = py0 + 4 * k;
    if (!(pxi < b.width && py < b.height)) continue;
    const size_t pix = (size_t)py * b.width + pxi;
    img[pix] = s.c01.x + s.T * cm.bg[0];
    img[hw + pix] = s.c01.y + s.T * cm.bg[1];
    img[2 * hw + pix] = s.c2 + s.T * cm.bg[2];
    if (DBG) {
      if (b.final_T[f]) b.final_T[f][pix] = s.T;
      if (b.n_contrib[f]) b.n_contrib[f][pix] = s.ncon;
      if (b.n_eval[f]) b.n_eval[f][pix] = s.nev;
    }
  }
}

int num_sms_current() {   // SM count of the calling thread's current device (cheap attribute query)
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

}  // namespace

cudaError_t launch_render(const RenderBatch& b, cudaStream_t s) {
  const int F = b.n_frames;
  const int64_t n = b.n;
  const unsigned nb = (unsigned)std::max<int64_t>(1, (n + 255) / 256);
  prof_mark(FGS_STAGE_PREPROCESS, true, s);
  clear_kernel<<<dim3((unsigned)std::min(64, (b.ntiles + 255) / 256), F), 256, 0, s>>>(b);
  const dim3 pre_grid((unsigned)(nb * (unsigned)F));   // 1-D, frame-minor (see preprocess_kernel)
  if (b.tile_cull) {
    switch (b.sh_degree) {
      case 0: preprocess_kernel<0, true><<<pre_grid, 256, 0, s>>>(b); break;
      case 1: preprocess_kernel<1, true><<<pre_grid, 256, 0, s>>>(b); break;
      case 2: preprocess_kernel<2, true><<<pre_grid, 256, 0, s>>>(b); break;
      default: preprocess_kernel<3, true><<<pre_grid, 256, 0, s>>>(b); break;
    }
  } else {
    switch (b.sh_degree) {
      case 0: preprocess_kernel<0, false><<<pre_grid, 256, 0, s>>>(b); break;
      case 1: preprocess_kernel<1, false><<<pre_grid, 256, 0, s>>>(b); break;
      case 2: preprocess_kernel<2, false><<<pre_grid, 256, 0, s>>>(b); break;
      default: preprocess_kernel<3, false><<<pre_grid, 256, 0, s>>>(b); break;
    }
  }
  note_launches(2);
  prof_mark(FGS_STAGE_PREPROCESS, false, s);
  prof_mark(FGS_STAGE_TILE_SCAN, true, s);
  tile_scan_kernel<<<F, kScanThreads, 0, s>>>(b);
  note_launches(1);
  prof_mark(FGS_STAGE_TILE_SCAN, false, s);
  prof_mark(FGS_STAGE_DUPLICATE, true, s);
  duplicate_kernel<<<dim3(nb, F), 256, 0, s>>>(b);
  note_launches(1);
  prof_mark(FGS_STAGE_DUPLICATE, false, s);
  prof_mark(FGS_STAGE_TILE_SORT, true, s);
  // radix binning path (radix.cu) for the frames tile_scan selected (it emits their instances, so on
  // those frames the stage holds the key duplication too); launched only when some frame may take it:
  // always (mode 2), or in auto mode when there are at least 64 Gaussians per tile (a mean list of
  // radix_min_list needs ~radix_min_list / 6 Gaussians per tile at the configs' ~6 tiles per Gaussian)
  if (b.radix_mode == 2 || (b.radix_mode == 1 && b.n >= (int64_t)64 * b.ntiles)) {
    const cudaError_t e = launch_radix_bin(b, s);
    if (e != cudaSuccess) return e;
  }
  tile_sort_kernel<<<(unsigned)(F * ((b.ntiles + kTileSortWarps - 1) / kTileSortWarps)), 32 * kTileSortWarps, 0, s>>>(b);
  // long lists: persistent CTAs (3 per SM over the batch) walk each frame's worklist (usually empty)
  // (per call: the attribute is per device, and the calling thread's current device may change)
  const cudaError_t attr = cudaFuncSetAttribute(long_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)kLongSortSmem);
  if (attr != cudaSuccess) return attr;
  long_sort_kernel<<<(unsigned)(3 * num_sms_current()), kLargeSortThreads,
                     kLongSortSmem, s>>>(b);
  note_launches(2);
  prof_mark(FGS_STAGE_TILE_SORT, false, s);
  prof_mark(FGS_STAGE_BLEND, true, s);
  const bool dbg = b.final_T[0] || b.n_contrib[0] || b.n_eval[0] || b.debug;
  if (dbg)
    blend_kernel<true><<<(unsigned)(F * b.ntiles), 32 * kBlendWarps, 0, s>>>(b);
  else
    blend_kernel<false><<<(unsigned)(F * b.ntiles), 32 * kBlendWarps, 0, s>>>(b);
  note_launches(1);
  prof_mark(FGS_STAGE_BLEND, false, s);
  return cudaGetLastError();
}

// Debug outputs: copy the per-frame intermediates of frame 0 into caller buffers (after a DBG blend,
// which writes every tile's sorted list back to the instance array).
__global__ void debug_copy_kernel(const __grid_constant__ RenderBatch b, fgs_render_aux aux) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t* cnt = cnt_ptr(b, 0);
  const uint32_t* tt = ws_ptr<uint32_t>(b.ws, b.ws_stride, 0, b.L.tt);
  const uint2* rect = ws_ptr<uint2>(b.ws, b.ws_stride, 0, b.L.rect);
  const int32_t* radii = ws_ptr<int32_t>(b.ws, b.ws_stride, 0, b.L.radii);
  const uint32_t* keys = ws_ptr<uint32_t>(b.ws, b.ws_stride, 0, b.L.keys);
  const float4* rec = ws_ptr<float4>(b.ws, b.ws_stride, 0, b.L.rec);
  const uint2* ranges = ws_ptr<uint2>(b.ws, b.ws_stride, 0, b.L.ranges);
  const unsigned long long* inst = ws_ptr<unsigned long long>(b.ws, b.ws_stride, 0, b.L.inst);
  if (i < b.n) {
    const bool kept = radii[i] != 0;       // (not tt: the tile cull may leave a kept Gaussian on no tile)
    if (aux.radii) aux.radii[i] = radii[i];
    if (aux.tiles_touched) aux.tiles_touched[i] = tt[i];
    if (aux.depth_key) aux.depth_key[i] = kept ? keys[i] : 0u;
    if (aux.rect) {
      const uint2 r = rect[i];
      aux.rect[4 * i + 0] = (int32_t)(r.x & 0xFFFF);
      aux.rect[4 * i + 1] = (int32_t)(r.x >> 16);
      aux.rect[4 * i + 2] = (int32_t)(r.y & 0xFFFF);
      aux.rect[4 * i + 3] = (int32_t)(r.y >> 16);
    }
    if (aux.mean2d) {
      const float4 a = rec[3 * i], c = rec[3 * i + 2];
      aux.mean2d[2 * i + 0] = kept ? a.x + c.y : 0.f;
      aux.mean2d[2 * i + 1] = kept ? a.y + c.z : 0.f;
    }
  }
  const uint32_t M = cnt[1];
  if (i < (int64_t)M && aux.sorted_gid) aux.sorted_gid[i] = (uint32_t)inst[i];
  if (i < b.ntiles) {
    const uint2 r = ranges[i];
    if (aux.ranges) {
      aux.ranges[2 * i] = r.x;
      aux.ranges[2 * i + 1] = r.y;
    }
    if (aux.sorted_tile)
      for (uint32_t p = r.x; p < r.y; ++p) aux.sorted_tile[p] = (uint32_t)i;
  }
  if (i == 0 && aux.n_instances) aux.n_instances[0] = cnt[3];
  if (i == 0 && aux.binning_direct) {
    aux.binning_direct[0] = cnt[6];
    aux.binning_direct[1] = cnt[7];
  }
  if (i == 0 && aux.long_sort_paths) {
    for (int k = 0; k < 3; ++k) aux.long_sort_paths[k] = cnt[9 + k];
  }
}

cudaError_t launch_debug_copy(const RenderBatch& b, const fgs_render_aux& aux, cudaStream_t s) {
  const int64_t m = std::max<int64_t>(std::max<int64_t>(b.n, b.L.cap), b.ntiles);
  debug_copy_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(b, aux);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace fgs
