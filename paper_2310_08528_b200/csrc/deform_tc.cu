// Gaussian deformation field on the 5th-gen tensor cores (tcgen05, TMEM) — PAPER.md §4.2.
//
// Same computation as deform.cu (Eq. 7 HexPlane sampling, phi_d, heads, additive update), but the
// dense layer phi_d — the one real contraction on the path, f_h[128 x K] . W_d^T[K x W] per tile of
// 128 Gaussians — runs as tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=W, K=8 per instruction)
// with the fp32 accumulator in TMEM.  fp32 accuracy is kept with the 3xTF32 split
// (A_hi B_hi + A_hi B_lo + A_lo B_hi), because the stress parity set (heads N(0,1)) needs
// <= 1e-4 on |Delta| ~ 1 and a single TF32 pass gives ~5e-4.
//
// CTA = 256 threads (8 warps), persistent over tiles of 128 Gaussians:
//   per tile   : every thread owns up to 8 (Gaussian, scale, channel-quad) items; the spatial planes
//                (xy, xz, yz) are sampled once and their product kept in registers for all times;
//   per time t : temporal planes (xt, yt, zt) sampled, f_h = S * T_t split hi/lo into the UMMA
//                K-major core-matrix layout in smem; one elected thread issues 3 x K/8 MMAs and
//                commits to an mbarrier; epilogue warps (warp w reads TMEM lanes 32(w%4).., columns
//                half w/4) apply bias + ReLU, the 10 head dot products, the additive update.
#include <cuda_runtime.h>

#include "fgs_internal.cuh"
#include "tc.cuh"

namespace fgs {

namespace {

constexpr int kM = 128;          // Gaussians per tile (UMMA M, TMEM lanes)
constexpr int kThreads = 256;
constexpr int kMaxItems = 8;     // (Gaussian, quad) items per thread: 128 * (64/4) / 256

template <int FEAT>
__device__ __forceinline__ float4 bilerp4(const float* __restrict__ P, int na, int nb, float ua, float ub,
                                          int c4) {
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

__device__ __forceinline__ float4 f4mul(float4 a, float4 b) {
  return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
}

// byte offset of element (row, k) in a K-major SWIZZLE_NONE operand with `rows` rows
__device__ __forceinline__ uint32_t core_off(int row, int k, int rows) {
  return (uint32_t)((((k >> 2) * (rows >> 3) + (row >> 3)) << 7) + ((row & 7) << 4) + ((k & 3) << 2));
}

template <int WIDTH>
struct TcSmem {
  static constexpr int A_BYTES = 64 * kM * 4;          // K (<= 64) x 128 rows, fp32
  static constexpr int B_BYTES = 64 * WIDTH * 4;
  static constexpr int OFF_AHI = 0;
  static constexpr int OFF_ALO = OFF_AHI + A_BYTES;
  static constexpr int OFF_BHI = OFF_ALO + A_BYTES;
  static constexpr int OFF_BLO = OFF_BHI + B_BYTES;
  static constexpr int OFF_WH = OFF_BLO + B_BYTES;          // [10][WIDTH]
  static constexpr int OFF_BD = OFF_WH + 10 * WIDTH * 4;    // [WIDTH]
  static constexpr int OFF_BH = OFF_BD + WIDTH * 4;         // [16]
  static constexpr int OFF_PART = OFF_BH + 16 * 4;          // [kM][11]
  static constexpr int OFF_BAR = OFF_PART + kM * 11 * 4;    // mbarrier (8 B) + tmem base (4 B)
  static constexpr int TOTAL = OFF_BAR + 16;
};

template <int FEAT, int WIDTH>
__global__ void __launch_bounds__(kThreads, 1) deform_tc_kernel(const __grid_constant__ DeformBatch p) {
  using SM = TcSmem<WIDTH>;
  constexpr int LPG = FEAT / 4;
  constexpr uint32_t NCOLS = WIDTH < 32 ? 32 : WIDTH;
  constexpr uint32_t IDESC = tc::idesc_tf32(kM, WIDTH);
  const int NS = p.n_scales;
  const int IN = p.in_dim;
  const int KP = (IN + 7) & ~7;            // K padded to the MMA K step
  const int NQ = IN / 4;                   // channel quads per Gaussian
  const int items = kM * NQ;

  extern __shared__ __align__(128) unsigned char smem[];
  float* Wh = reinterpret_cast<float*>(smem + SM::OFF_WH);
  float* bd = reinterpret_cast<float*>(smem + SM::OFF_BD);
  float* bh = reinterpret_cast<float*>(smem + SM::OFF_BH);
  float* part = reinterpret_cast<float*>(smem + SM::OFF_PART);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::OFF_BAR + 8);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- one-time setup: W_d split into B_hi/B_lo (K-major core layout), heads, TMEM, mbarrier ----
  for (int i = tid; i < WIDTH * KP; i += kThreads) {
    const int n = i / KP, k = i - n * KP;
    const float w = k < IN ? p.w_d[n * IN + k] : 0.f;
    float hi, lo;
    tc::tf32_split(w, hi, lo);
    const uint32_t o = core_off(n, k, WIDTH);
    *reinterpret_cast<float*>(smem + SM::OFF_BHI + o) = hi;
    *reinterpret_cast<float*>(smem + SM::OFF_BLO + o) = lo;
  }
  for (int i = tid; i < kM * (KP - IN); i += kThreads) {     // zero the padded K columns of A
    const int r = i / (KP - IN), k = IN + i % (KP - IN);
    *reinterpret_cast<float*>(smem + SM::OFF_AHI + core_off(r, k, kM)) = 0.f;
    *reinterpret_cast<float*>(smem + SM::OFF_ALO + core_off(r, k, kM)) = 0.f;
  }
  for (int i = tid; i < 3 * WIDTH; i += kThreads) Wh[i] = p.w_x[i];
  for (int i = tid; i < 4 * WIDTH; i += kThreads) Wh[3 * WIDTH + i] = p.w_r[i];
  for (int i = tid; i < 3 * WIDTH; i += kThreads) Wh[7 * WIDTH + i] = p.w_s[i];
  for (int i = tid; i < WIDTH; i += kThreads) bd[i] = p.b_d[i];
  if (tid < 3) bh[tid] = p.b_x[tid];
  if (tid < 4) bh[3 + tid] = p.b_r[tid];
  if (tid < 3) bh[7 + tid] = p.b_s[tid];
  if (tid == 0) {
    tc::mbar_init(bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, NCOLS);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  uint32_t phase = 0;

  const uint32_t a_hi = tc::smem_u32(smem + SM::OFF_AHI), a_lo = tc::smem_u32(smem + SM::OFF_ALO);
  const uint32_t b_hi = tc::smem_u32(smem + SM::OFF_BHI), b_lo = tc::smem_u32(smem + SM::OFF_BLO);

  const int64_t count = p.end - p.begin;
  const int64_t n_tiles = (count + kM - 1) / kM;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t g0 = p.begin + tile * kM;
    // ---- per tile: grid coordinates and the spatial-plane product of every owned item ----
    float u[kMaxItems][3];
    float4 S[kMaxItems];
#pragma unroll
    for (int j = 0; j < kMaxItems; ++j) {
      const int item = j * kThreads + tid;
      S[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      u[j][0] = u[j][1] = u[j][2] = 0.f;
      if (item < items) {
        const int row = item / NQ, q = item - row * NQ;
        const int64_t g = g0 + row;
        if (g < p.end) {
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const float m = __ldg(p.means + g * 3 + a);
            u[j][a] = fminf(fmaxf((m - p.bmin[a]) / p.ext[a], 0.f), 1.f);
          }
          const int l = q / LPG, c4 = q - l * LPG;
          const int R = p.res[l];
          float4 v = bilerp4<FEAT>(p.planes[l][0], R, R, u[j][0], u[j][1], c4);
          v = f4mul(v, bilerp4<FEAT>(p.planes[l][1], R, R, u[j][0], u[j][2], c4));
          S[j] = f4mul(v, bilerp4<FEAT>(p.planes[l][2], R, R, u[j][1], u[j][2], c4));
        }
      }
    }
    for (int f = 0; f < p.n_t; ++f) {
      const float t = p.t[f];
      // ---- temporal planes at t; f_h = S * T split hi/lo into the A operand ----
#pragma unroll
      for (int j = 0; j < kMaxItems; ++j) {
        const int item = j * kThreads + tid;
        if (item < items) {
          const int row = item / NQ, q = item - row * NQ;
          const int l = q / LPG, c4 = q - l * LPG;
          float4 fh = make_float4(0.f, 0.f, 0.f, 0.f);
          if (g0 + row < p.end) {
            const int R = p.res[l];
            float4 v = bilerp4<FEAT>(p.planes[l][3], R, p.t_res, u[j][0], t, c4);
            v = f4mul(v, bilerp4<FEAT>(p.planes[l][4], R, p.t_res, u[j][1], t, c4));
            v = f4mul(v, bilerp4<FEAT>(p.planes[l][5], R, p.t_res, u[j][2], t, c4));
            fh = f4mul(S[j], v);
          }
          float4 hi, lo;
          tc::tf32_split(fh.x, hi.x, lo.x);
          tc::tf32_split(fh.y, hi.y, lo.y);
          tc::tf32_split(fh.z, hi.z, lo.z);
          tc::tf32_split(fh.w, hi.w, lo.w);
          const uint32_t o = core_off(row, 4 * q, kM);
          *reinterpret_cast<float4*>(smem + SM::OFF_AHI + o) = hi;
          *reinterpret_cast<float4*>(smem + SM::OFF_ALO + o) = lo;
        }
      }
      tc::fence_async_smem();
      tc::fence_before_sync();
      __syncthreads();
      // ---- phi_d on the tensor core: D[128 x W] = f_h . W_d^T (3xTF32), single issuing thread ----
      if (tid == 0) {
        tc::fence_after_sync();
        uint32_t acc = 0;
        for (int s = 0; s < KP / 8; ++s) {
          const uint32_t ao = (uint32_t)s * (2 * (kM / 8) * 128), bo = (uint32_t)s * (2 * (WIDTH / 8) * 128);
          const uint64_t dah = tc::smem_desc(a_hi + ao, (kM / 8) * 128, 128);
          const uint64_t dal = tc::smem_desc(a_lo + ao, (kM / 8) * 128, 128);
          const uint64_t dbh = tc::smem_desc(b_hi + bo, (WIDTH / 8) * 128, 128);
          const uint64_t dbl = tc::smem_desc(b_lo + bo, (WIDTH / 8) * 128, 128);
          tc::mma_tf32(tmem, dal, dbh, IDESC, acc);   // small terms first
          tc::mma_tf32(tmem, dah, dbl, IDESC, 1);
          tc::mma_tf32(tmem, dah, dbh, IDESC, 1);
          acc = 1;
        }
        tc::mma_commit(bar);
      }
      tc::mbar_wait(bar, phase);
      phase ^= 1u;
      tc::fence_after_sync();
      // ---- epilogue: warp w -> rows 32(w%4)+lane, hidden columns [h W/2, (h+1) W/2), h = w/4 ----
      const int quarter = warp & 3, half = warp >> 2;
      const int row = quarter * 32 + lane;
      float ho[10];
#pragma unroll
      for (int o = 0; o < 10; ++o) ho[o] = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < WIDTH / 2; c0 += 16) {
        const int col = half * (WIDTH / 2) + c0;
        float v[16];
        tc::tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)col, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float fd = fmaxf(v[i] + bd[col + i], 0.f);      // f_d = ReLU(W_d f_h + b_d)
#pragma unroll
          for (int o = 0; o < 10; ++o) ho[o] = fmaf(fd, Wh[o * WIDTH + col + i], ho[o]);
        }
      }
      if (half == 1) {
#pragma unroll
        for (int o = 0; o < 10; ++o) part[row * 11 + o] = ho[o];
      }
      tc::fence_before_sync();
      __syncthreads();
      if (half == 0) {
        const int64_t g = g0 + row;
        if (g < p.end) {
#pragma unroll
          for (int o = 0; o < 10; ++o) ho[o] += part[row * 11 + o] + bh[o];
#pragma unroll
          for (int c = 0; c < 3; ++c) p.out_means[f][g * 3 + c] = __ldg(p.means + g * 3 + c) + ho[c];
#pragma unroll
          for (int c = 0; c < 4; ++c) p.out_quats[f][g * 4 + c] = __ldg(p.quats + g * 4 + c) + ho[3 + c];
#pragma unroll
          for (int c = 0; c < 3; ++c)
            p.out_log_scales[f][g * 3 + c] = __ldg(p.log_scales + g * 3 + c) + ho[7 + c];
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, NCOLS);
  }
}

template <int FEAT, int WIDTH>
cudaError_t launch_tc_t(const DeformBatch& p, cudaStream_t s) {
  using SM = TcSmem<WIDTH>;
  auto kern = deform_tc_kernel<FEAT, WIDTH>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::TOTAL);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, SM::TOTAL);
  const int64_t tiles = (p.end - p.begin + kM - 1) / kM;
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > tiles) grid = tiles;
  if (grid < 1) return cudaSuccess;
  prof_mark(FGS_STAGE_DEFORM, true, s);
  kern<<<(unsigned)grid, kThreads, SM::TOTAL, s>>>(p);
  note_launches(1);
  prof_mark(FGS_STAGE_DEFORM, false, s);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_deform_tc(const DeformBatch& p, cudaStream_t s) {
  if (p.end <= p.begin || p.n_t <= 0) return cudaSuccess;
#define FGS_DISPATCH_W(FEAT)                          \
  switch (p.width) {                                  \
    case 32: return launch_tc_t<FEAT, 32>(p, s);      \
    case 64: return launch_tc_t<FEAT, 64>(p, s);      \
    case 128: return launch_tc_t<FEAT, 128>(p, s);    \
    default: return cudaErrorInvalidValue;            \
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
