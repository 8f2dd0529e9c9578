// Tile-based splatting S(M, G') on sm_100a — PAPER.md §3.1 with the [3dgs]
// rasterizer conventions the paper renders with; readings R1-R20 in DESIGN.md.
//
// Per frame (frames of a batch run in the same launches, blockIdx.y = frame):
//   preprocess   Eq. 2 covariance, Eq. 3 EWA projection, conic, radius, tile rect, depth key,
//                SH colour.  Decision geometry (everything that yields an integer: depth key,
//                radius, rect) in fp64 with the oracle's fixed summation order for the depth.
//   depth sort   stable LSD radix sort (4 x 8-bit digits) of the N depth keys, values = index.
//   offsets      exclusive scan of tiles_touched in depth order -> instance offsets, M.
//   duplicate    each kept Gaussian emits (tile, index) for every tile of its rect, in depth order.
//   tile sort    stable LSD radix sort of the instances by tile id (<= 8-bit digits).  Because the
//                input is already in (depth, index) order, the result is sorted by
//                (tile, depth, index) — the [3dgs] 64-bit key order, reading R14.
//   ranges       per-tile [start, end) by boundary detection on the sorted tile ids.
//   blend        Eq. 4 front-to-back per pixel, 16x16 CTA per tile, records staged in smem.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "fgs_internal.cuh"

namespace fgs {

namespace {

constexpr float kNear = 0.2f;             // R6
constexpr float kAlphaMin = 1.0f / 255.0f;  // R9
constexpr float kTMin = 1e-4f;            // R9
constexpr float kAlphaMax = 0.99f;        // R9
constexpr double kDilation = 0.3;         // R5
constexpr double kLambdaFloor = 0.1;      // R7
constexpr double kFovClamp = 1.3;         // R4

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

// ------------------------------------------------------------------------------ preprocess
__global__ void __launch_bounds__(256) preprocess_kernel(const __grid_constant__ RenderBatch b) {
  const int f = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t* cnt = cnt_ptr(b, f);
  if (i == 0) { cnt[0] = (uint32_t)b.n; cnt[1] = 0; cnt[2] = 0; cnt[3] = 0; }
  if (i >= b.n) return;
  uint32_t* keys = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.keys0);
  uint32_t* vals = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.vals0);
  uint32_t* tt = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.tt);
  uint2* rect = ws_ptr<uint2>(b.ws, b.ws_stride, f, b.L.rect);
  int32_t* radii = ws_ptr<int32_t>(b.ws, b.ws_stride, f, b.L.radii);
  float4* rec = ws_ptr<float4>(b.ws, b.ws_stride, f, b.L.rec);
  const FrameCam& c = b.cam[f];

  vals[i] = (uint32_t)i;
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
  const float* qp = b.quats[f] + 4 * i;
  double qw = qp[0], qx = qp[1], qy = qp[2], qz = qp[3];
  const double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  qw /= qn; qx /= qn; qy /= qn; qz /= qn;
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
  const double fx = c.fx, fy = c.fy;
  const double limx = kFovClamp * ((double)b.width / (2.0 * fx));
  const double limy = kFovClamp * ((double)b.height / (2.0 * fy));
  const double xt = fmin(limx, fmax(-limx, px / pz)) * pz;
  const double yt = fmin(limy, fmax(-limy, py / pz)) * pz;
  const double j00 = fx / pz, j02 = -fx * xt / (pz * pz);
  const double j11 = fy / pz, j12 = -fy * yt / (pz * pz);
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
  const double lam1 = mid + sqrt(fmax(kLambdaFloor, mid * mid - det));
  const double rad = ceil(3.0 * sqrt(lam1));
  // ---- step 9: mean2d ----
  const double mx = fx * px / pz + (double)c.cx;
  const double my = fy * py / pz + (double)c.cy;
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
  if (!keep) {
    keys[i] = 0xFFFFFFFFu;
    tt[i] = 0;
    rect[i] = make_uint2(0, 0);
    radii[i] = 0;
    return;
  }
  // ---- step 11: depth key = bits of fp32(p.z) (> 0.2 so unsigned order = depth order) ----
  keys[i] = __float_as_uint((float)pz);
  tt[i] = (uint32_t)((x1 - x0) * (y1 - y0));
  rect[i] = make_uint2((uint32_t)x0 | ((uint32_t)y0 << 16), (uint32_t)x1 | ((uint32_t)y1 << 16));
  radii[i] = (int32_t)rad;
  // ---- step 12: SH colour at d = normalize(X - campos), campos = -R^T t (R10, R11) ----
  const double cxw = -((double)c.R[0] * c.t[0] + (double)c.R[3] * c.t[1] + (double)c.R[6] * c.t[2]);
  const double cyw = -((double)c.R[1] * c.t[0] + (double)c.R[4] * c.t[1] + (double)c.R[7] * c.t[2]);
  const double czw = -((double)c.R[2] * c.t[0] + (double)c.R[5] * c.t[1] + (double)c.R[8] * c.t[2]);
  double dx = x - cxw, dy = y - cyw, dz = z - czw;
  const double dn = sqrt(dx * dx + dy * dy + dz * dz);
  const float X = (float)(dx / dn), Y = (float)(dy / dn), Z = (float)(dz / dn);
  const int deg = b.sh_degree;
  const int K = (deg + 1) * (deg + 1);
  const float* sh = b.sh[f] + (size_t)i * K * 3;
  float basis[16];
  basis[0] = SH_C0;
  if (deg >= 1) { basis[1] = -SH_C1 * Y; basis[2] = SH_C1 * Z; basis[3] = -SH_C1 * X; }
  if (deg >= 2) {
    const float xx = X * X, yy = Y * Y, zz = Z * Z;
    basis[4] = SH_C2_0 * X * Y;
    basis[5] = SH_C2_1 * Y * Z;
    basis[6] = SH_C2_2 * (2.f * zz - xx - yy);
    basis[7] = SH_C2_3 * X * Z;
    basis[8] = SH_C2_4 * (xx - yy);
    if (deg >= 3) {
      basis[9] = SH_C3_0 * Y * (3.f * xx - yy);
      basis[10] = SH_C3_1 * X * Y * Z;
      basis[11] = SH_C3_2 * Y * (4.f * zz - xx - yy);
      basis[12] = SH_C3_3 * Z * (2.f * zz - 3.f * xx - 3.f * yy);
      basis[13] = SH_C3_4 * X * (4.f * zz - xx - yy);
      basis[14] = SH_C3_5 * Z * (xx - yy);
      basis[15] = SH_C3_6 * X * (xx - 3.f * yy);
    }
  }
  float col[3] = {0.5f, 0.5f, 0.5f};
  for (int k = 0; k < K; ++k) {
    col[0] = fmaf(basis[k], __ldg(sh + 3 * k + 0), col[0]);
    col[1] = fmaf(basis[k], __ldg(sh + 3 * k + 1), col[1]);
    col[2] = fmaf(basis[k], __ldg(sh + 3 * k + 2), col[2]);
  }
  // ---- blend record: mean2d as hi/lo fp32 pairs, conic pre-scaled to the log2 domain ----
  //   p2 = A' dx^2 + B' dx dy + C' dy^2 = power * log2(e);  alpha = min(0.99, 2^(p2 + log2 o))
  const float mxh = (float)mx, myh = (float)my;
  const float mxl = (float)(mx - (double)mxh), myl = (float)(my - (double)myh);
  const double opac = 1.0 / (1.0 + exp(-(double)b.opacity[f][i]));
  const double L2E = 1.4426950408889634;
  rec[3 * i + 0] = make_float4(mxh, myh, (float)(-0.5 * L2E * cc / det), (float)(L2E * bb / det));
  rec[3 * i + 1] = make_float4((float)(-0.5 * L2E * a / det), (float)log2(opac), fmaxf(col[0], 0.f),
                               fmaxf(col[1], 0.f));
  // Conservative per-Gaussian cull radius^2 for the blend's warp-box test: for any pixel at distance
  // d from the mean, alpha <= o exp(-d^2 / (2 lambda_max(Sigma2))), so alpha < 1/255 (skipped anyway)
  // whenever d^2 > 2 lambda_max (ln(255 o) + 0.01); margins cover fp32 evaluation error.
  const double lam_max = mid + sqrt(fmax(0.0, mid * mid - det));
  const double r2 = (2.0 * log(255.0 * opac) + 0.02) * lam_max * (1.0 + 1e-4) + 1e-3;
  rec[3 * i + 2] = make_float4(fmaxf(col[2], 0.f), mxl, myl, (float)r2);
}

// ------------------------------------------------------------------------------ radix sort
struct SortArgs {
  char* ws;
  size_t stride;
  size_t cnt;       // counter block offset
  int cnt_idx;      // which counter holds the item count
  size_t kin, vin, kout, vout, hist;
  int shift, bits;
};

__device__ __forceinline__ uint32_t sort_count(const SortArgs& a, int f) {
  return ws_ptr<uint32_t>(a.ws, a.stride, f, a.cnt)[a.cnt_idx];
}

__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(const __grid_constant__ SortArgs a) {
  const int f = blockIdx.y;
  const uint32_t count = sort_count(a, f);
  const uint32_t ntl = (count + kSortTile - 1) / kSortTile;
  const uint32_t* keys = ws_ptr<uint32_t>(a.ws, a.stride, f, a.kin);
  uint32_t* hist = ws_ptr<uint32_t>(a.ws, a.stride, f, a.hist);
  const int radix = 1 << a.bits;
  const uint32_t mask = radix - 1;
  __shared__ uint32_t h[256];
  for (uint32_t tile = blockIdx.x; tile < ntl; tile += gridDim.x) {
    for (int d = threadIdx.x; d < radix; d += kSortThreads) h[d] = 0;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kSortItems; ++it) {
      const uint32_t idx = tile * kSortTile + it * kSortThreads + threadIdx.x;
      if (idx < count) atomicAdd(&h[(keys[idx] >> a.shift) & mask], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < radix; d += kSortThreads) hist[(size_t)d * ntl + tile] = h[d];
    __syncthreads();
  }
}

// Block-wide exclusive scan of one value per thread (1024 threads); returns the block total.
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

__global__ void __launch_bounds__(1024) radix_scan_kernel(const __grid_constant__ SortArgs a) {
  const int f = blockIdx.x;
  const uint32_t count = sort_count(a, f);
  const uint32_t ntl = (count + kSortTile - 1) / kSortTile;
  uint32_t* hist = ws_ptr<uint32_t>(a.ws, a.stride, f, a.hist);
  const uint32_t total = (uint32_t)(1 << a.bits) * ntl;
  const uint32_t chunk = (total + 1023) / 1024;
  const uint32_t beg = min(total, threadIdx.x * chunk), end = min(total, beg + chunk);
  uint32_t s = 0;
  for (uint32_t k = beg; k < end; ++k) s += hist[k];
  __shared__ uint32_t sw[32];
  uint32_t excl;
  block_exclusive_scan<1024>(s, excl, sw);
  for (uint32_t k = beg; k < end; ++k) {
    const uint32_t v = hist[k];
    hist[k] = excl;
    excl += v;
  }
}

__global__ void __launch_bounds__(kSortThreads) radix_scatter_kernel(const __grid_constant__ SortArgs a) {
  const int f = blockIdx.y;
  const uint32_t count = sort_count(a, f);
  const uint32_t ntl = (count + kSortTile - 1) / kSortTile;
  const uint32_t* kin = ws_ptr<uint32_t>(a.ws, a.stride, f, a.kin);
  const uint32_t* vin = ws_ptr<uint32_t>(a.ws, a.stride, f, a.vin);
  uint32_t* kout = ws_ptr<uint32_t>(a.ws, a.stride, f, a.kout);
  uint32_t* vout = ws_ptr<uint32_t>(a.ws, a.stride, f, a.vout);
  const uint32_t* hist = ws_ptr<uint32_t>(a.ws, a.stride, f, a.hist);
  const int radix = 1 << a.bits;
  const uint32_t mask = radix - 1;
  constexpr int NW = kSortThreads / 32;
  __shared__ uint32_t wc[NW][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t tile = blockIdx.x; tile < ntl; tile += gridDim.x) {
    for (int d = threadIdx.x; d < NW * 256; d += kSortThreads) (&wc[0][0])[d] = 0;
    __syncthreads();
    uint32_t k[kSortItems], v[kSortItems], rank[kSortItems];
    // Warp `warp` owns the contiguous chunk [warp*256, warp*256+256) of the tile, in rounds of 32,
    // so ranks are stable (input order) within the warp; warps are combined in order below.
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
      const uint32_t idx = tile * kSortTile + warp * (32 * kSortItems) + r * 32 + lane;
      const bool valid = idx < count;
      const uint32_t vm = __ballot_sync(0xffffffffu, valid);
      uint32_t d = 0, peers = 0;
      if (valid) {
        k[r] = kin[idx];
        v[r] = vin[idx];
        d = (k[r] >> a.shift) & mask;
        peers = __match_any_sync(vm, d);
        rank[r] = wc[warp][d] + __popc(peers & lt);
      }
      __syncwarp();
      if (valid && (__ffs(peers) - 1) == lane) wc[warp][d] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    for (int d = threadIdx.x; d < radix; d += kSortThreads) {
      uint32_t run = hist[(size_t)d * ntl + tile];
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const uint32_t c = wc[w][d];
        wc[w][d] = run;
        run += c;
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
      const uint32_t idx = tile * kSortTile + warp * (32 * kSortItems) + r * 32 + lane;
      if (idx < count) {
        const uint32_t pos = wc[warp][(k[r] >> a.shift) & mask] + rank[r];
        kout[pos] = k[r];
        vout[pos] = v[r];
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ instance offsets
// Exclusive scan over depth order of tiles_touched[vals[p]] (3 phases).
__global__ void __launch_bounds__(kScanThreads) offsets_reduce_kernel(const __grid_constant__ RenderBatch b) {
  const int f = blockIdx.y;
  const int64_t n = b.n;
  const int64_t nt = (n + kScanTile - 1) / kScanTile;
  const uint32_t* vals = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.vals0);
  const uint32_t* tt = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.tt);
  uint32_t* part = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.partial);
  __shared__ uint32_t sw[32];
  for (int64_t tile = blockIdx.x; tile < nt; tile += gridDim.x) {
    uint32_t s = 0;
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
      const int64_t p = tile * kScanTile + it * kScanThreads + threadIdx.x;
      if (p < n) s += tt[vals[p]];
    }
    uint32_t excl;
    const uint32_t tot = block_exclusive_scan<kScanThreads>(s, excl, sw);
    if (threadIdx.x == 0) part[tile] = tot;
  }
}

__global__ void __launch_bounds__(1024) offsets_partials_kernel(const __grid_constant__ RenderBatch b) {
  const int f = blockIdx.x;
  const int64_t nt = (b.n + kScanTile - 1) / kScanTile;
  uint32_t* part = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.partial);
  uint32_t* cnt = cnt_ptr(b, f);
  const uint32_t chunk = (uint32_t)((nt + 1023) / 1024);
  const uint32_t beg = (uint32_t)min((int64_t)threadIdx.x * chunk, nt);
  const uint32_t end = (uint32_t)min((int64_t)beg + chunk, nt);
  unsigned long long s = 0;
  for (uint32_t k = beg; k < end; ++k) s += part[k];
  __shared__ uint32_t sw[32];
  uint32_t excl;
  const uint32_t total = block_exclusive_scan<1024>((uint32_t)s, excl, sw);
  for (uint32_t k = beg; k < end; ++k) {
    const uint32_t v = part[k];
    part[k] = excl;
    excl += v;
  }
  if (threadIdx.x == 0) {
    const uint64_t cap = (uint64_t)b.L.cap;
    cnt[3] = total;
    cnt[1] = (uint32_t)min((uint64_t)total, cap);
    cnt[2] = (uint64_t)total > cap ? 1u : 0u;
  }
}

__global__ void __launch_bounds__(kScanThreads) offsets_downsweep_kernel(const __grid_constant__ RenderBatch b) {
  const int f = blockIdx.y;
  const int64_t n = b.n;
  const int64_t nt = (n + kScanTile - 1) / kScanTile;
  const uint32_t* vals = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.vals0);
  const uint32_t* tt = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.tt);
  const uint32_t* part = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.partial);
  uint32_t* offs = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.offs);
  __shared__ uint32_t sw[32];
  for (int64_t tile = blockIdx.x; tile < nt; tile += gridDim.x) {
    // thread owns kScanItems consecutive items
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
      const int64_t p = tile * kScanTile + (int64_t)threadIdx.x * kScanItems + it;
      v[it] = p < n ? tt[vals[p]] : 0u;
      s += v[it];
    }
    uint32_t excl;
    block_exclusive_scan<kScanThreads>(s, excl, sw);
    excl += part[tile];
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
      const int64_t p = tile * kScanTile + (int64_t)threadIdx.x * kScanItems + it;
      if (p < n) offs[p] = excl;
      excl += v[it];
    }
  }
}

// ------------------------------------------------------------------------------ duplicate
__global__ void __launch_bounds__(256) duplicate_kernel(const __grid_constant__ RenderBatch b) {
  const int f = blockIdx.y;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= b.n) return;
  const uint32_t* vals = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.vals0);
  const uint32_t* tt = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.tt);
  const uint2* rect = ws_ptr<uint2>(b.ws, b.ws_stride, f, b.L.rect);
  const uint32_t* offs = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.offs);
  uint32_t* ikey = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.ikey0);
  uint32_t* ival = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.ival0);
  const uint32_t gid = vals[p];
  if (tt[gid] == 0) return;
  const uint2 r = rect[gid];
  const uint32_t x0 = r.x & 0xFFFF, y0 = r.x >> 16, x1 = r.y & 0xFFFF, y1 = r.y >> 16;
  const uint64_t cap = (uint64_t)b.L.cap;
  uint64_t o = offs[p];
  for (uint32_t ty = y0; ty < y1; ++ty)
    for (uint32_t tx = x0; tx < x1; ++tx, ++o)
      if (o < cap) { ikey[o] = ty * (uint32_t)b.gx + tx; ival[o] = gid; }
}

// ------------------------------------------------------------------------------ tile ranges
__global__ void ranges_clear_kernel(const __grid_constant__ RenderBatch b) {
  const int f = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < b.ntiles) ws_ptr<uint2>(b.ws, b.ws_stride, f, b.L.ranges)[t] = make_uint2(0, 0);
}

__global__ void ranges_kernel(const __grid_constant__ RenderBatch b, size_t keys_off) {
  const int f = blockIdx.y;
  const uint32_t M = cnt_ptr(b, f)[1];
  const uint32_t* keys = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, keys_off);
  uint2* ranges = ws_ptr<uint2>(b.ws, b.ws_stride, f, b.L.ranges);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    const uint32_t t = keys[i];
    if (i == 0 || keys[i - 1] != t) ranges[t].x = i;
    if (i == M - 1 || keys[i + 1] != t) ranges[t].y = i + 1;
  }
}

// ------------------------------------------------------------------------------ blend (Eq. 4)
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Eq. 4 for one pixel and one Gaussian, branch-free (the warp stays converged).
// p2 = power * log2(e); the Gaussian is skipped if p2 > 0 or alpha < 1/255 (R9); the pixel stops
// (without adding the Gaussian) when T (1 - alpha) < 1e-4 (R9).
struct PixelState {
  float T, c0, c1, c2;
  bool done;
  uint32_t ncon, nev;
};

__device__ __forceinline__ void blend_step(PixelState& s, float p2, float lo, float r, float g, float bch,
                                           uint32_t pos) {
  const float alpha = fminf(kAlphaMax, ex2_approx(p2 + lo));
  const bool ok = !s.done && !(p2 > 0.f) && !(alpha < kAlphaMin);
  const float test_T = s.T * (1.f - alpha);
  const bool stop = ok && test_T < kTMin;
  const bool add = ok && !stop;
  if (stop) { s.done = true; s.nev = pos; }
  const float w = add ? alpha * s.T : 0.f;
  s.c0 = fmaf(r, w, s.c0);
  s.c1 = fmaf(g, w, s.c1);
  s.c2 = fmaf(bch, w, s.c2);
  s.T = add ? test_T : s.T;
  s.ncon += add ? 1u : 0u;
}

template <bool DBG>
__global__ void __launch_bounds__(128) blend_kernel(const __grid_constant__ RenderBatch b, size_t vals_off) {
  // One CTA (4 warps) per 16x16 tile.  Warp w owns the 8x8 pixel box ((w&1)*8, (w>>1)*8); each lane
  // two pixels (x, y) and (x, y+4).  Per batch of 256 Gaussians (smem), each warp tests 32 Gaussians
  // at a time against a conservative alpha bound over its box (lane-parallel + ballot) and then
  // evaluates only the survivors for its 64 pixels, in list order.
  const int f = blockIdx.y;
  const int tile = blockIdx.x;
  const int tx = tile % b.gx, ty = tile / b.gx;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int bx0 = (warp & 1) * 8, by0 = (warp >> 1) * 8;          // box origin, tile-relative
  const int lxi = bx0 + (lane & 7), lyi = by0 + (lane >> 3);
  const int pxi = tx * kTile + lxi, pyA = ty * kTile + lyi, pyB = pyA + 4;
  const bool inA = pxi < b.width && pyA < b.height;
  const bool inB = pxi < b.width && pyB < b.height;
  const uint2 rg = ws_ptr<uint2>(b.ws, b.ws_stride, f, b.L.ranges)[tile];
  const uint32_t* gids = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, vals_off);
  const float4* rec = ws_ptr<float4>(b.ws, b.ws_stride, f, b.L.rec);
  __shared__ float4 s0[256], s1[256];
  __shared__ float2 s2[256];
  const float tx0 = (float)(tx * kTile), ty0 = (float)(ty * kTile);
  const float lx = (float)lxi, ly = (float)lyi;
  const float bxl = (float)bx0, bxh = (float)(bx0 + 7), byl = (float)by0, byh = (float)(by0 + 7);
  PixelState A{1.f, 0.f, 0.f, 0.f, !inA, 0u, rg.y - rg.x};
  PixelState B{1.f, 0.f, 0.f, 0.f, !inB, 0u, rg.y - rg.x};
  for (uint32_t start = rg.x; start < rg.y; start += 256) {
    if (__syncthreads_count(A.done && B.done) == 128) break;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t idx = start + threadIdx.x + 128 * k;
      if (idx < rg.y) {
        const uint32_t g = gids[idx];
        float4 a = rec[3 * g + 0];
        const float4 c = rec[3 * g + 2];
        a.x = (a.x - tx0) + c.y;      // tile-relative mean: exact hi difference + lo part
        a.y = (a.y - ty0) + c.z;
        s0[threadIdx.x + 128 * k] = a;
        s1[threadIdx.x + 128 * k] = rec[3 * g + 1];
        s2[threadIdx.x + 128 * k] = make_float2(c.x, c.w);
      }
    }
    __syncthreads();
    const int cnt = (int)min(256u, rg.y - start);
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      if (__all_sync(0xffffffffu, A.done && B.done)) break;
      const int jt = c0 + lane;
      bool need = false;
      if (jt < cnt) {
        const float4 a = s0[jt];
        const float ddx = fmaxf(fmaxf(bxl - a.x, a.x - bxh), 0.f);
        const float ddy = fmaxf(fmaxf(byl - a.y, a.y - byh), 0.f);
        need = ddx * ddx + ddy * ddy <= s2[jt].y;
      }
      uint32_t m = __ballot_sync(0xffffffffu, need);
      while (m) {
        const int j = c0 + __ffs(m) - 1;
        m &= m - 1;
        const float4 a = s0[j], q = s1[j];
        const float bch = s2[j].x;
        const float dx = a.x - lx;
        const float dyA = a.y - ly, dyB = dyA - 4.f;
        const float adx = a.z * dx;                         // A' dx, shared by both pixels
        const float pA = fmaf(dx, fmaf(a.w, dyA, adx), q.x * dyA * dyA);
        const float pB = fmaf(dx, fmaf(a.w, dyB, adx), q.x * dyB * dyB);
        const uint32_t pos = start + j - rg.x + 1;
        blend_step(A, pA, q.y, q.z, q.w, bch, pos);
        blend_step(B, pB, q.y, q.z, q.w, bch, pos);
      }
    }
    __syncthreads();
  }
  const size_t hw = (size_t)b.width * b.height;
  float* img = b.image[f];
  const FrameCam& cm = b.cam[f];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const PixelState& s = k ? B : A;
    const bool in = k ? inB : inA;
    if (!in) continue;
    const size_t pix = (size_t)(k ? pyB : pyA) * b.width + pxi;
    img[pix] = s.c0 + s.T * cm.bg[0];
    img[hw + pix] = s.c1 + s.T * cm.bg[1];
    img[2 * hw + pix] = s.c2 + s.T * cm.bg[2];
    if (DBG) {
      if (b.final_T[f]) b.final_T[f][pix] = s.T;
      if (b.n_contrib[f]) b.n_contrib[f][pix] = s.ncon;
      if (b.n_eval[f]) b.n_eval[f][pix] = s.nev;
    }
  }
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

cudaError_t run_sort(SortArgs a, int n_frames, int64_t max_items, int key_bits, bool& swapped,
                     cudaStream_t s) {
  // key_bits total bits, split into passes of <= 8 bits; ping-pong kin <-> kout.
  swapped = false;
  if (key_bits <= 0) return cudaSuccess;
  const int passes = (key_bits + 7) / 8;
  const int base = key_bits / passes, extra = key_bits % passes;
  const int64_t tiles = (max_items + kSortTile - 1) / kSortTile;
  int64_t gx = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)num_sms() * 8 / std::max(1, n_frames) + 1));
  dim3 grid((unsigned)gx, n_frames);
  int shift = 0;
  for (int p = 0; p < passes; ++p) {
    a.shift = shift;
    a.bits = base + (p < extra ? 1 : 0);
    shift += a.bits;
    radix_hist_kernel<<<grid, kSortThreads, 0, s>>>(a);
    radix_scan_kernel<<<n_frames, 1024, 0, s>>>(a);
    radix_scatter_kernel<<<grid, kSortThreads, 0, s>>>(a);
    note_launches(3);
    std::swap(a.kin, a.kout);
    std::swap(a.vin, a.vout);
    swapped = !swapped;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_render(const RenderBatch& b, cudaStream_t s) {
  const int F = b.n_frames;
  const int64_t n = b.n;
  const unsigned nb = (unsigned)std::max<int64_t>(1, (n + 255) / 256);
  prof_mark(FGS_STAGE_PREPROCESS, true, s);
  preprocess_kernel<<<dim3(nb, F), 256, 0, s>>>(b);
  note_launches(1);
  prof_mark(FGS_STAGE_PREPROCESS, false, s);
  // depth sort: 32-bit keys, values = index (stable -> ties by index)
  SortArgs a{};
  a.ws = b.ws; a.stride = b.ws_stride; a.cnt = b.L.cnt; a.cnt_idx = 0; a.hist = b.L.hist;
  a.kin = b.L.keys0; a.vin = b.L.vals0; a.kout = b.L.keys1; a.vout = b.L.vals1;
  bool sw = false;
  prof_mark(FGS_STAGE_DEPTH_SORT, true, s);
  cudaError_t e = run_sort(a, F, n, 32, sw, s);
  prof_mark(FGS_STAGE_DEPTH_SORT, false, s);
  if (e != cudaSuccess) return e;
  // (4 passes -> result back in keys0/vals0)
  const int64_t nt = std::max<int64_t>(1, (n + kScanTile - 1) / kScanTile);
  const unsigned sg = (unsigned)std::min<int64_t>(nt, (int64_t)num_sms() * 4 / F + 1);
  prof_mark(FGS_STAGE_OFFSETS, true, s);
  offsets_reduce_kernel<<<dim3(sg, F), kScanThreads, 0, s>>>(b);
  offsets_partials_kernel<<<F, 1024, 0, s>>>(b);
  offsets_downsweep_kernel<<<dim3(sg, F), kScanThreads, 0, s>>>(b);
  note_launches(3);
  prof_mark(FGS_STAGE_OFFSETS, false, s);
  prof_mark(FGS_STAGE_DUPLICATE, true, s);
  duplicate_kernel<<<dim3(nb, F), 256, 0, s>>>(b);
  note_launches(1);
  prof_mark(FGS_STAGE_DUPLICATE, false, s);
  // tile sort: ceil(log2(ntiles)) bits
  int tbits = 0;
  while ((1 << tbits) < b.ntiles) ++tbits;
  SortArgs t{};
  t.ws = b.ws; t.stride = b.ws_stride; t.cnt = b.L.cnt; t.cnt_idx = 1; t.hist = b.L.hist;
  t.kin = b.L.ikey0; t.vin = b.L.ival0; t.kout = b.L.ikey1; t.vout = b.L.ival1;
  prof_mark(FGS_STAGE_TILE_SORT, true, s);
  e = run_sort(t, F, b.L.cap, tbits, sw, s);
  prof_mark(FGS_STAGE_TILE_SORT, false, s);
  if (e != cudaSuccess) return e;
  const size_t kfin = sw ? b.L.ikey1 : b.L.ikey0;
  const size_t vfin = sw ? b.L.ival1 : b.L.ival0;
  prof_mark(FGS_STAGE_RANGES, true, s);
  ranges_clear_kernel<<<dim3((b.ntiles + 255) / 256, F), 256, 0, s>>>(b);
  const unsigned rg = (unsigned)std::max<int64_t>(1, std::min<int64_t>((b.L.cap + 255) / 256, (int64_t)num_sms() * 8 / F + 1));
  ranges_kernel<<<dim3(rg, F), 256, 0, s>>>(b, kfin);
  note_launches(2);
  prof_mark(FGS_STAGE_RANGES, false, s);
  prof_mark(FGS_STAGE_BLEND, true, s);
  const bool dbg = b.final_T[0] || b.n_contrib[0] || b.n_eval[0];
  if (dbg)
    blend_kernel<true><<<dim3(b.ntiles, F), 128, 0, s>>>(b, vfin);
  else
    blend_kernel<false><<<dim3(b.ntiles, F), 128, 0, s>>>(b, vfin);
  note_launches(1);
  prof_mark(FGS_STAGE_BLEND, false, s);
  return cudaGetLastError();
}

// Debug outputs: copy the per-frame intermediates of frame 0 into caller buffers.
__global__ void debug_copy_kernel(const __grid_constant__ RenderBatch b, fgs_render_aux aux, size_t kfin,
                                  size_t vfin) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t* cnt = cnt_ptr(b, 0);
  const uint32_t* tt = ws_ptr<uint32_t>(b.ws, b.ws_stride, 0, b.L.tt);
  const uint2* rect = ws_ptr<uint2>(b.ws, b.ws_stride, 0, b.L.rect);
  const int32_t* radii = ws_ptr<int32_t>(b.ws, b.ws_stride, 0, b.L.radii);
  const float4* rec = ws_ptr<float4>(b.ws, b.ws_stride, 0, b.L.rec);
  if (i < b.n) {
    // depth keys are permuted by the sort; recompute key from the record of kept Gaussians via
    // the sorted arrays below instead.  Here: per-Gaussian outputs.
    const bool kept = tt[i] != 0;
    if (aux.radii) aux.radii[i] = radii[i];
    if (aux.tiles_touched) aux.tiles_touched[i] = tt[i];
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
  // depth keys: scatter from the depth-sorted arrays (keys0/vals0 after 4 passes)
  if (aux.depth_key && i < b.n) {
    const uint32_t* k = ws_ptr<uint32_t>(b.ws, b.ws_stride, 0, b.L.keys0);
    const uint32_t* v = ws_ptr<uint32_t>(b.ws, b.ws_stride, 0, b.L.vals0);
    const uint32_t key = k[i];
    aux.depth_key[v[i]] = key == 0xFFFFFFFFu ? 0u : key;
  }
  const uint32_t M = cnt[1];
  if (i < (int64_t)M) {
    if (aux.sorted_tile) aux.sorted_tile[i] = ws_ptr<uint32_t>(b.ws, b.ws_stride, 0, kfin)[i];
    if (aux.sorted_gid) aux.sorted_gid[i] = ws_ptr<uint32_t>(b.ws, b.ws_stride, 0, vfin)[i];
  }
  if (i < b.ntiles && aux.ranges) {
    const uint2 r = ws_ptr<uint2>(b.ws, b.ws_stride, 0, b.L.ranges)[i];
    aux.ranges[2 * i] = r.x;
    aux.ranges[2 * i + 1] = r.y;
  }
  if (i == 0 && aux.n_instances) aux.n_instances[0] = cnt[3];
}

cudaError_t launch_debug_copy(const RenderBatch& b, const fgs_render_aux& aux, cudaStream_t s) {
  int tbits = 0;
  while ((1 << tbits) < b.ntiles) ++tbits;
  const int passes = tbits > 0 ? (tbits + 7) / 8 : 0;
  const bool sw = passes & 1;
  const size_t kfin = sw ? b.L.ikey1 : b.L.ikey0;
  const size_t vfin = sw ? b.L.ival1 : b.L.ival0;
  const int64_t m = std::max<int64_t>(std::max<int64_t>(b.n, b.L.cap), b.ntiles);
  debug_copy_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(b, aux, kfin, vfin);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace fgs
