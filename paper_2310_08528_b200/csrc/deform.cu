// Gaussian deformation field F(G, t) = D(H(G, t)) on sm_100a — PAPER.md §4.2.
//
//   f_h = concat_l  prod_{(i,j)} bilinear(R_l(i,j))(mu, t)     Eq. 7
//   f_d = ReLU(W_d f_h + b_d)                                   phi_d
//   (dX, dr, ds) = (W_x, W_r, W_s) f_d + b                      heads
//   (X', r', s') = (X + dX, r + dr, s + ds)                     P:800 (raw space)
//
// One persistent kernel (grid = resident CTAs) loops over tiles of 64 Gaussians.  Per tile the
// three spatial planes (xy, xz, yz) are sampled ONCE and their product is kept in shared memory;
// then for every time t of the batch only the three temporal planes are sampled, multiplied in,
// and phi_d + heads run on the tile.  Plane corners are channel-last, so one Gaussian's corner is
// `feat` contiguous floats read as float4 by feat/4 lanes (coalesced 128-B rows).
#include <cuda_runtime.h>

#include "fgs_internal.cuh"

namespace fgs {

namespace {

constexpr int kTG = 64;            // Gaussians per tile
constexpr int kDeformThreads = 128;
constexpr int kMaxIn = 64;
constexpr int kRow = kMaxIn + 1;   // smem row stride of S / F (bank-conflict padding)

__device__ __forceinline__ float4 f4mul(float4 a, float4 b) {
  return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
}

// Bilinear "interp ... 4 vertices" of a channel-last plane [nb][na][FEAT] at grid
// coordinates (ua, ub) in [0,1]; returns channels [4*c4, 4*c4+4).  Knot k at u = k/(n-1).
template <int FEAT>
__device__ __forceinline__ float4 bilerp4(const float* __restrict__ P, int na, int nb, float ua,
                                          float ub, int c4) {
  const float ga = ua * (float)(na - 1);
  const float gb = ub * (float)(nb - 1);
  const int i0 = min((int)floorf(ga), na - 2);
  const int j0 = min((int)floorf(gb), nb - 2);
  const float fa = ga - (float)i0;
  const float fb = gb - (float)j0;
  const float4* row0 = reinterpret_cast<const float4*>(P + ((size_t)j0 * na + i0) * FEAT) + c4;
  const float4* row1 = reinterpret_cast<const float4*>(P + ((size_t)(j0 + 1) * na + i0) * FEAT) + c4;
  const float4 v00 = __ldg(row0);
  const float4 v01 = __ldg(row0 + FEAT / 4);
  const float4 v10 = __ldg(row1);
  const float4 v11 = __ldg(row1 + FEAT / 4);
  const float w00 = (1.f - fa) * (1.f - fb), w01 = fa * (1.f - fb);
  const float w10 = (1.f - fa) * fb, w11 = fa * fb;
  float4 r;
  r.x = w00 * v00.x + w01 * v01.x + w10 * v10.x + w11 * v11.x;
  r.y = w00 * v00.y + w01 * v01.y + w10 * v10.y + w11 * v11.y;
  r.z = w00 * v00.z + w01 * v01.z + w10 * v10.z + w11 * v11.z;
  r.w = w00 * v00.w + w01 * v01.w + w10 * v10.w + w11 * v11.w;
  return r;
}

template <int FEAT, int WIDTH>
__global__ void __launch_bounds__(kDeformThreads)
deform_kernel(const __grid_constant__ DeformBatch p) {
  constexpr int LPG = FEAT / 4;            // lanes per Gaussian (one float4 of channels each)
  constexpr int GPW = 32 / LPG;            // Gaussians per warp pass
  constexpr int NW = kDeformThreads / 32;
  constexpr int OPT = WIDTH / 8;           // hidden outputs per thread in phi_d
  const int IN = p.in_dim;
  const int NS = p.n_scales;

  extern __shared__ __align__(16) float smem[];
  float* WdT = smem;                                  // [IN][WIDTH]  (W_d transposed)
  float* bd = WdT + kMaxIn * WIDTH;                   // [WIDTH]
  float* Wh = bd + WIDTH;                             // [10][WIDTH]  rows: x(3) r(4) s(3)
  float* bh = Wh + 10 * WIDTH;                        // [16]
  float* S = bh + 16;                                 // [kTG][kRow] spatial product
  float* F = S + kTG * kRow;                          // [kTG][kRow] f_h
  float* Hd = F + kTG * kRow;                         // [kTG][WIDTH+1] f_d
  float* U = Hd + kTG * (WIDTH + 1);                  // [kTG][4] grid coords

  const int tid = threadIdx.x;
  for (int i = tid; i < IN * WIDTH; i += kDeformThreads) {
    const int o = i / IN, k = i - o * IN;
    WdT[k * WIDTH + o] = p.w_d[i];
  }
  for (int i = tid; i < WIDTH; i += kDeformThreads) bd[i] = p.b_d[i];
  for (int i = tid; i < 3 * WIDTH; i += kDeformThreads) Wh[i] = p.w_x[i];
  for (int i = tid; i < 4 * WIDTH; i += kDeformThreads) Wh[3 * WIDTH + i] = p.w_r[i];
  for (int i = tid; i < 3 * WIDTH; i += kDeformThreads) Wh[7 * WIDTH + i] = p.w_s[i];
  if (tid < 3) bh[tid] = p.b_x[tid];
  if (tid < 4) bh[3 + tid] = p.b_r[tid];
  if (tid < 3) bh[7 + tid] = p.b_s[tid];
  __syncthreads();

  const int warp = tid >> 5, lane = tid & 31;
  const int c4 = lane % LPG;
  const int64_t count = p.end - p.begin;
  const int64_t n_tiles = (count + kTG - 1) / kTG;

  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t g0 = p.begin + tile * kTG;
    // ---- phase A: grid coords + spatial planes (xy, xz, yz), shared by all times ----
    for (int gi = warp * GPW + lane / LPG; gi < kTG; gi += NW * GPW) {
      const int64_t g = g0 + gi;
      if (g >= p.end) continue;
      float u[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const float m = __ldg(p.means + g * 3 + a);
        u[a] = fminf(fmaxf((m - p.bmin[a]) / p.ext[a], 0.f), 1.f);
      }
      if (c4 == 0) { U[gi * 4 + 0] = u[0]; U[gi * 4 + 1] = u[1]; U[gi * 4 + 2] = u[2]; }
      for (int l = 0; l < NS; ++l) {
        const int R = p.res[l];
        float4 v = bilerp4<FEAT>(p.planes[l][0], R, R, u[0], u[1], c4);
        v = f4mul(v, bilerp4<FEAT>(p.planes[l][1], R, R, u[0], u[2], c4));
        v = f4mul(v, bilerp4<FEAT>(p.planes[l][2], R, R, u[1], u[2], c4));
        float* dst = S + gi * kRow + l * FEAT + 4 * c4;
        dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
      }
    }
    __syncthreads();

    for (int f = 0; f < p.n_t; ++f) {
      const float t = p.t[f];
      // ---- phase B: temporal planes (xt, yt, zt) at t; f_h = spatial * temporal ----
      for (int gi = warp * GPW + lane / LPG; gi < kTG; gi += NW * GPW) {
        if (g0 + gi >= p.end) continue;
        const float ux = U[gi * 4 + 0], uy = U[gi * 4 + 1], uz = U[gi * 4 + 2];
        for (int l = 0; l < NS; ++l) {
          const int R = p.res[l];
          float4 v = bilerp4<FEAT>(p.planes[l][3], R, p.t_res, ux, t, c4);
          v = f4mul(v, bilerp4<FEAT>(p.planes[l][4], R, p.t_res, uy, t, c4));
          v = f4mul(v, bilerp4<FEAT>(p.planes[l][5], R, p.t_res, uz, t, c4));
          const float* src = S + gi * kRow + l * FEAT + 4 * c4;
          float* dst = F + gi * kRow + l * FEAT + 4 * c4;
          dst[0] = src[0] * v.x; dst[1] = src[1] * v.y; dst[2] = src[2] * v.z; dst[3] = src[3] * v.w;
        }
      }
      __syncthreads();
      // ---- phase C: f_d = ReLU(W_d f_h + b_d), register tile 4 Gaussians x OPT outputs ----
      {
        const int gq = tid & 15;          // Gaussians gq, gq+16, gq+32, gq+48
        const int oq = tid >> 4;          // outputs [oq*OPT, oq*OPT+OPT)
        float acc[4][OPT];
#pragma unroll
        for (int o = 0; o < OPT; ++o) {
          const float b = bd[oq * OPT + o];
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[j][o] = b;
        }
        for (int k = 0; k < IN; ++k) {
          float fa[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) fa[j] = F[(gq + 16 * j) * kRow + k];
          const float4* w4 = reinterpret_cast<const float4*>(WdT + k * WIDTH + oq * OPT);
#pragma unroll
          for (int o4 = 0; o4 < OPT / 4; ++o4) {
            const float4 w = w4[o4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              acc[j][o4 * 4 + 0] = fmaf(fa[j], w.x, acc[j][o4 * 4 + 0]);
              acc[j][o4 * 4 + 1] = fmaf(fa[j], w.y, acc[j][o4 * 4 + 1]);
              acc[j][o4 * 4 + 2] = fmaf(fa[j], w.z, acc[j][o4 * 4 + 2]);
              acc[j][o4 * 4 + 3] = fmaf(fa[j], w.w, acc[j][o4 * 4 + 3]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int o = 0; o < OPT; ++o)
            Hd[(gq + 16 * j) * (WIDTH + 1) + oq * OPT + o] = fmaxf(acc[j][o], 0.f);
      }
      __syncthreads();
      // ---- phase D: heads + additive update, 5 outputs per thread ----
      {
        const int gi = tid & 63;
        const int half = tid >> 6;
        const int64_t g = g0 + gi;
        float acc[5];
#pragma unroll
        for (int o = 0; o < 5; ++o) acc[o] = bh[half * 5 + o];
        const float* h = Hd + gi * (WIDTH + 1);
        for (int k = 0; k < WIDTH; ++k) {
          const float hv = h[k];
#pragma unroll
          for (int o = 0; o < 5; ++o) acc[o] = fmaf(hv, Wh[(half * 5 + o) * WIDTH + k], acc[o]);
        }
        if (g < p.end) {
#pragma unroll
          for (int o = 0; o < 5; ++o) {
            const int c = half * 5 + o;     // 0-2 dX, 3-6 dr, 7-9 ds
            if (c < 3) {
              p.out_means[f][g * 3 + c] = __ldg(p.means + g * 3 + c) + acc[o];
            } else if (c < 7) {
              p.out_quats[f][g * 4 + (c - 3)] = __ldg(p.quats + g * 4 + (c - 3)) + acc[o];
            } else {
              p.out_log_scales[f][g * 3 + (c - 7)] = __ldg(p.log_scales + g * 3 + (c - 7)) + acc[o];
            }
          }
        }
      }
      __syncthreads();
    }
  }
}

template <int FEAT, int WIDTH>
cudaError_t launch_t(const DeformBatch& p, cudaStream_t s) {
  const size_t smem = sizeof(float) * (size_t)(kMaxIn * WIDTH + WIDTH + 10 * WIDTH + 16 + 2 * kTG * kRow +
                                               kTG * (WIDTH + 1) + kTG * 4);
  auto kern = deform_kernel<FEAT, WIDTH>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDeformThreads, smem);
  const int64_t tiles = (p.end - p.begin + kTG - 1) / kTG;
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > tiles) grid = tiles;
  if (grid < 1) return cudaSuccess;
  prof_mark(FGS_STAGE_DEFORM, true, s);
  kern<<<(unsigned)grid, kDeformThreads, smem, s>>>(p);
  note_launches(1);
  prof_mark(FGS_STAGE_DEFORM, false, s);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_deform(const DeformBatch& p, cudaStream_t s) {
  if (p.end <= p.begin || p.n_t <= 0) return cudaSuccess;
#define FGS_DISPATCH_W(FEAT)                                       \
  switch (p.width) {                                               \
    case 32: return launch_t<FEAT, 32>(p, s);                      \
    case 64: return launch_t<FEAT, 64>(p, s);                      \
    case 128: return launch_t<FEAT, 128>(p, s);                    \
    default: return cudaErrorInvalidValue;                         \
  }
  switch (p.feat) {
    case 4: FGS_DISPATCH_W(4)
    case 8: FGS_DISPATCH_W(8)
    case 16: FGS_DISPATCH_W(16)
    case 32: FGS_DISPATCH_W(32)
    default: return cudaErrorInvalidValue;
  }
#undef FGS_DISPATCH_W
}

}  // namespace fgs
