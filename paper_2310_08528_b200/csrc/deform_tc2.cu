// Gaussian deformation field, v2: TMEM-resident operands, frame-outer schedule (sm_100a).
// PAPER.md §4.2: Eq. 7 HexPlane query, phi_d, heads, additive update.
//
// Schedule per CTA (persistent, 8 warps, 1 CTA/SM), over a contiguous range of 128-Gaussian tiles
// processed in groups of G tiles:
//   group prologue : the spatial-plane product S = xy . xz . yz of every (Gaussian, feature) of the
//                    group is sampled once and parked in TENSOR MEMORY (IN columns per tile);
//   per time t     : the three temporal planes are collapsed to 1-D "lines" at t (time lerp) in
//                    shared memory, once per CTA;  then per tile: f_h = S . lerp(line_x) .
//                    lerp(line_y) . lerp(line_z) (smem lookups), split hi/lo and stored straight to
//                    TMEM as the A operand; one thread issues 3 x K/8 tcgen05.mma.kind::tf32 with A
//                    from TMEM and B = W_d (hi/lo) from smem; the epilogue reads D from TMEM, applies
//                    bias + ReLU, the 10 head dot products and the additive update.
// Thread (warp w, lane i) owns TMEM lane / tile row r = 32 (w%4) + i and, for every scale, the
// feature half h = w/4 — the tcgen05.ld/st lane-quarter rule maps one row to one thread.
// Used when the lines of all scales fit in shared memory (D-NeRF/HyperNeRF/Neu3D configs);
// otherwise deform_tc.cu (v1) runs.
#include <cuda_runtime.h>

#include "fgs_internal.cuh"
#include "tc.cuh"

namespace fgs {

namespace {

constexpr int kM = 128;
constexpr int kTmemCols = 512;
constexpr int kMaxG = 16;
constexpr int kMaxLineFloats = 3 * 192 * 32;   // 72 KB: 3 planes x (64 + 128) knots x h 32

__device__ __forceinline__ uint32_t core_off(int row, int k, int rows) {
  return (uint32_t)((((k >> 2) * (rows >> 3) + (row >> 3)) << 7) + ((row & 7) << 4) + ((k & 3) << 2));
}

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
  const float4 v00 = __ldg(row0), v01 = __ldg(row0 + FEAT / 4);
  const float4 v10 = __ldg(row1), v11 = __ldg(row1 + FEAT / 4);
  const float w00 = (1.f - fa) * (1.f - fb), w01 = fa * (1.f - fb);
  const float w10 = (1.f - fa) * fb, w11 = fa * fb;
  float4 r;
  r.x = w00 * v00.x + w01 * v01.x + w10 * v10.x + w11 * v11.x;
  r.y = w00 * v00.y + w01 * v01.y + w10 * v10.y + w11 * v11.y;
  r.z = w00 * v00.z + w01 * v01.z + w10 * v10.z + w11 * v11.z;
  r.w = w00 * v00.w + w01 * v01.w + w10 * v10.w + w11 * v11.w;
  return r;
}

// Lines are stored [R][FEAT/4] float4 with the quad index XOR-swizzled by the knot index, so that
// 32 lanes reading the same channel quad at different knots spread over the 8 bank groups.
template <int FEAT>
__device__ __forceinline__ int swz(int i, int c4) {
  return c4 ^ (i & (FEAT / 4 - 1));
}

// linear interpolation of a line [R][FEAT] (smem) at u in [0,1], channel quad c4
template <int FEAT>
__device__ __forceinline__ float4 lerp_line(const float* line, int R, float u, int c4) {
  const float g = u * (float)(R - 1);
  const int i0 = min((int)floorf(g), R - 2);
  const float fa = g - (float)i0;
  const float4 a = reinterpret_cast<const float4*>(line + i0 * FEAT)[swz<FEAT>(i0, c4)];
  const float4 b = reinterpret_cast<const float4*>(line + (i0 + 1) * FEAT)[swz<FEAT>(i0 + 1, c4)];
  const float wa = 1.f - fa;
  return make_float4(wa * a.x + fa * b.x, wa * a.y + fa * b.y, wa * a.z + fa * b.z, wa * a.w + fa * b.w);
}

template <int WIDTH>
struct Tc2Smem {
  static constexpr int B_BYTES = 64 * WIDTH * 4;
  static constexpr int OFF_BHI = 0;
  static constexpr int OFF_BLO = OFF_BHI + B_BYTES;
  static constexpr int OFF_LINE = OFF_BLO + B_BYTES;
  static constexpr int OFF_U = OFF_LINE + kMaxLineFloats * 4;   // [kMaxG][128][4]
  static constexpr int OFF_WH = OFF_U + kMaxG * kM * 16;
  static constexpr int OFF_BD = OFF_WH + 10 * WIDTH * 4;
  static constexpr int OFF_BH = OFF_BD + WIDTH * 4;
  static constexpr int OFF_PART = OFF_BH + 16 * 4;
  static constexpr int OFF_BAR = OFF_PART + 3 * kM * 10 * 4;
  static constexpr int TOTAL = OFF_BAR + 16;
};

// registers <-> TMEM for N (multiple of 4) consecutive columns of this thread's lane
template <int N>
__device__ __forceinline__ void tmem_st_n(uint32_t taddr, const float* v) {
#pragma unroll
  for (int i = 0; i < N; i += 16) {
    if constexpr (N % 16 == 0) tc::tmem_st16(taddr + i, v + i);
  }
  if constexpr (N % 16 != 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4) tc::tmem_st4(taddr + i, v + i);
  }
}
template <int N>
__device__ __forceinline__ void tmem_ld_n(uint32_t taddr, float* v) {
  if constexpr (N % 16 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 16) tc::tmem_ld16(taddr + i, v + i);
  } else {
#pragma unroll
    for (int i = 0; i < N; i += 4) tc::tmem_ld4(taddr + i, v + i);
  }
}

template <int FEAT>
struct Parts {
  static constexpr int NP = FEAT >= 16 ? 4 : 2;       // warps per TMEM lane quarter
  static constexpr int THREADS = 128 * NP;
  static constexpr int FT = FEAT / NP;                // features per (thread, scale)
  static constexpr int QT = FT / 4;                   // channel quads per (thread, scale)
};

template <int FEAT, int WIDTH>
__global__ void __launch_bounds__(Parts<FEAT>::THREADS, 1)
deform_tc2_kernel(const __grid_constant__ DeformBatch p) {
  using SM = Tc2Smem<WIDTH>;
  constexpr int NP = Parts<FEAT>::NP, NT = Parts<FEAT>::THREADS, FT = Parts<FEAT>::FT, QT = Parts<FEAT>::QT;
  constexpr int MAXS = 64 / FEAT;              // max scales (IN <= 64)
  constexpr int DW = WIDTH < 32 ? 32 : WIDTH;  // D columns
  constexpr int WT = WIDTH / NP;               // hidden columns per thread in the epilogue
  constexpr uint32_t IDESC = tc::idesc_tf32(kM, WIDTH);
  const int NS = p.n_scales;
  const int IN = p.in_dim;
  const int KP = (IN + 7) & ~7;
  const uint32_t colA_hi = DW, colA_lo = DW + KP, colS = DW + 2 * KP;
  const int G = min(kMaxG, (kTmemCols - (int)colS) / IN);

  extern __shared__ __align__(128) unsigned char smem[];
  float* line = reinterpret_cast<float*>(smem + SM::OFF_LINE);
  float* U = reinterpret_cast<float*>(smem + SM::OFF_U);
  float* Wh = reinterpret_cast<float*>(smem + SM::OFF_WH);
  float* bd = reinterpret_cast<float*>(smem + SM::OFF_BD);
  float* bh = reinterpret_cast<float*>(smem + SM::OFF_BH);
  float* part_buf = reinterpret_cast<float*>(smem + SM::OFF_PART);   // [NP-1][128][10]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::OFF_BAR + 8);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, part = warp >> 2;
  const int row = quarter * 32 + lane;

  // ---- setup ----
  for (int i = tid; i < WIDTH * KP; i += NT) {
    const int n = i / KP, k = i - n * KP;
    const float w = k < IN ? p.w_d[n * IN + k] : 0.f;
    float hi, lo;
    tc::tf32_split(w, hi, lo);
    const uint32_t o = core_off(n, k, WIDTH);
    *reinterpret_cast<float*>(smem + SM::OFF_BHI + o) = hi;
    *reinterpret_cast<float*>(smem + SM::OFF_BLO + o) = lo;
  }
  for (int i = tid; i < 3 * WIDTH; i += NT) Wh[i] = p.w_x[i];
  for (int i = tid; i < 4 * WIDTH; i += NT) Wh[3 * WIDTH + i] = p.w_r[i];
  for (int i = tid; i < 3 * WIDTH; i += NT) Wh[7 * WIDTH + i] = p.w_s[i];
  for (int i = tid; i < WIDTH; i += NT) bd[i] = p.b_d[i];
  if (tid < 3) bh[tid] = p.b_x[tid];
  if (tid < 4) bh[3 + tid] = p.b_r[tid];
  if (tid < 3) bh[7 + tid] = p.b_s[tid];
  int line_off[MAXS];
  {
    int o = 0;
#pragma unroll
    for (int l = 0; l < MAXS; ++l) {
      line_off[l] = o;
      if (l < NS) o += 3 * p.res[l] * FEAT;
    }
  }
  if (tid == 0) {
    tc::mbar_init(bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, kTmemCols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
  if (part == 0) {   // zero the K padding columns of A once (never written afterwards)
    for (int k = IN; k < KP; k += 4) {
      const float z[4] = {0.f, 0.f, 0.f, 0.f};
      tc::tmem_st4(lane_base + colA_hi + k, z);
      tc::tmem_st4(lane_base + colA_lo + k, z);
    }
    tc::tmem_st_wait();
  }
  uint32_t phase = 0;
  const uint32_t b_hi = tc::smem_u32(smem + SM::OFF_BHI), b_lo = tc::smem_u32(smem + SM::OFF_BLO);

  const int64_t count = p.end - p.begin;
  const int64_t tiles = (count + kM - 1) / kM;
  const int64_t t_beg = tiles * blockIdx.x / gridDim.x, t_end = tiles * (blockIdx.x + 1) / gridDim.x;
  for (int64_t gstart = t_beg; gstart < t_end; gstart += G) {
    const int ng = (int)min((int64_t)G, t_end - gstart);
    // ---- group prologue: grid coordinates (smem) and spatial products S (TMEM) ----
    for (int gt = 0; gt < ng; ++gt) {
      const int64_t g = p.begin + (gstart + gt) * kM + row;
      const bool valid = g < p.end;
      float u[3] = {0.f, 0.f, 0.f};
      if (valid) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const float m = __ldg(p.means + g * 3 + a);
          u[a] = fminf(fmaxf((m - p.bmin[a]) / p.ext[a], 0.f), 1.f);
        }
      }
      if (part == 0) {
        float* Ur = U + (gt * kM + row) * 4;
        Ur[0] = u[0]; Ur[1] = u[1]; Ur[2] = u[2];
      }
#pragma unroll
      for (int l = 0; l < MAXS; ++l) {
        if (l >= NS) break;
        const int R = p.res[l];
        float sv[FT];
#pragma unroll
        for (int qq = 0; qq < QT; ++qq) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (valid) {
            const int c4 = part * QT + qq;
            v = bilerp4<FEAT>(p.planes[l][0], R, R, u[0], u[1], c4);
            const float4 b = bilerp4<FEAT>(p.planes[l][1], R, R, u[0], u[2], c4);
            const float4 c = bilerp4<FEAT>(p.planes[l][2], R, R, u[1], u[2], c4);
            v = make_float4(v.x * b.x * c.x, v.y * b.y * c.y, v.z * b.z * c.z, v.w * b.w * c.w);
          }
          sv[4 * qq + 0] = v.x; sv[4 * qq + 1] = v.y; sv[4 * qq + 2] = v.z; sv[4 * qq + 3] = v.w;
        }
        tmem_st_n<FT>(lane_base + colS + gt * IN + l * FEAT + part * FT, sv);
      }
    }
    tc::tmem_st_wait();
    for (int f = 0; f < p.n_t; ++f) {
      const float t = p.t[f];
      // ---- stage the temporal lines at t for all scales (time lerp of 2 knot rows) ----
      __syncthreads();
      {
        const int Tn = p.t_res;
        const float gt_ = t * (float)(Tn - 1);
        const int j0 = min((int)floorf(gt_), Tn - 2);
        const float ft = gt_ - (float)j0, wt = 1.f - ft;
#pragma unroll
        for (int l = 0; l < MAXS; ++l) {
          if (l >= NS) break;
          const int R = p.res[l];
          const int per_plane = R * (FEAT / 4);
          float4* dst = reinterpret_cast<float4*>(line + line_off[l]);
#pragma unroll
          for (int pl = 0; pl < 3; ++pl) {
            const float4* P0 = reinterpret_cast<const float4*>(p.planes[l][3 + pl]) + (size_t)j0 * per_plane;
            const float4* P1 = P0 + per_plane;
            for (int rem = tid; rem < per_plane; rem += NT) {
              const float4 a = __ldg(P0 + rem);
              const float4 b = __ldg(P1 + rem);
              const int i = rem / (FEAT / 4), c4 = rem - i * (FEAT / 4);
              dst[pl * per_plane + i * (FEAT / 4) + swz<FEAT>(i, c4)] =
                  make_float4(wt * a.x + ft * b.x, wt * a.y + ft * b.y, wt * a.z + ft * b.z, wt * a.w + ft * b.w);
            }
          }
        }
      }
      __syncthreads();
      for (int gt = 0; gt < ng; ++gt) {
        const int64_t g = p.begin + (gstart + gt) * kM + row;
        const bool valid = g < p.end;
        // prefetch the canonical attributes the update adds to (part 0 only)
        float cx[10];
        if (part == 0 && valid) {
#pragma unroll
          for (int c = 0; c < 3; ++c) cx[c] = __ldg(p.means + g * 3 + c);
#pragma unroll
          for (int c = 0; c < 4; ++c) cx[3 + c] = __ldg(p.quats + g * 4 + c);
#pragma unroll
          for (int c = 0; c < 3; ++c) cx[7 + c] = __ldg(p.log_scales + g * 3 + c);
        }
        const float* Ur = U + (gt * kM + row) * 4;
        const float ux = Ur[0], uy = Ur[1], uz = Ur[2];
        // ---- f_h = S . T_t -> hi/lo -> TMEM A ----
#pragma unroll
        for (int l = 0; l < MAXS; ++l) {
          if (l >= NS) break;
          const int R = p.res[l];
          float sv[FT], hi[FT], lo[FT];
          tmem_ld_n<FT>(lane_base + colS + gt * IN + l * FEAT + part * FT, sv);
          const float* lx = line + line_off[l];
          const float* ly = lx + R * FEAT;
          const float* lz = ly + R * FEAT;
#pragma unroll
          for (int qq = 0; qq < QT; ++qq) {
            const int c4 = part * QT + qq;
            const float4 a = lerp_line<FEAT>(lx, R, ux, c4);
            const float4 b = lerp_line<FEAT>(ly, R, uy, c4);
            const float4 c = lerp_line<FEAT>(lz, R, uz, c4);
            const float fh[4] = {sv[4 * qq + 0] * (a.x * b.x * c.x), sv[4 * qq + 1] * (a.y * b.y * c.y),
                                 sv[4 * qq + 2] * (a.z * b.z * c.z), sv[4 * qq + 3] * (a.w * b.w * c.w)};
#pragma unroll
            for (int e = 0; e < 4; ++e) tc::tf32_split(fh[e], hi[4 * qq + e], lo[4 * qq + e]);
          }
          tmem_st_n<FT>(lane_base + colA_hi + l * FEAT + part * FT, hi);
          tmem_st_n<FT>(lane_base + colA_lo + l * FEAT + part * FT, lo);
        }
        tc::tmem_st_wait();
        tc::fence_before_sync();
        __syncthreads();
        // ---- phi_d on the tensor core, A from TMEM, B = W_d hi/lo from smem ----
        if (tid == 0) {
          tc::fence_after_sync();
          for (int s = 0; s < KP / 8; ++s) {
            const uint32_t bo = (uint32_t)s * (2 * (WIDTH / 8) * 128);
            const uint64_t dbh = tc::smem_desc(b_hi + bo, (WIDTH / 8) * 128, 128);
            const uint64_t dbl = tc::smem_desc(b_lo + bo, (WIDTH / 8) * 128, 128);
            tc::mma_tf32_ts(tmem, tmem + colA_lo + 8 * s, dbh, IDESC, s > 0 ? 1u : 0u);
            tc::mma_tf32_ts(tmem, tmem + colA_hi + 8 * s, dbl, IDESC, 1u);
            tc::mma_tf32_ts(tmem, tmem + colA_hi + 8 * s, dbh, IDESC, 1u);
          }
          tc::mma_commit(bar);
        }
        tc::mbar_wait(bar, phase);
        phase ^= 1u;
        tc::fence_after_sync();
        // ---- epilogue: bias + ReLU + heads over this thread's WT hidden columns ----
        float ho[10];
#pragma unroll
        for (int o = 0; o < 10; ++o) ho[o] = 0.f;
        {
          const int col = part * WT;
          float v[WT];
          tmem_ld_n<WT>(lane_base + (uint32_t)col, v);
#pragma unroll
          for (int i = 0; i < WT; ++i) {
            const float fd = fmaxf(v[i] + bd[col + i], 0.f);
#pragma unroll
            for (int o = 0; o < 10; ++o) ho[o] = fmaf(fd, Wh[o * WIDTH + col + i], ho[o]);
          }
        }
        if (part > 0) {
#pragma unroll
          for (int o = 0; o < 10; ++o) part_buf[((part - 1) * kM + row) * 10 + o] = ho[o];
        }
        tc::fence_before_sync();
        __syncthreads();
        if (part == 0 && valid) {
#pragma unroll
          for (int o = 0; o < 10; ++o) {
            float acc = ho[o];
#pragma unroll
            for (int q = 0; q < NP - 1; ++q) acc += part_buf[(q * kM + row) * 10 + o];
            ho[o] = cx[o] + (acc + bh[o]);
          }
#pragma unroll
          for (int c = 0; c < 3; ++c) p.out_means[f][g * 3 + c] = ho[c];
#pragma unroll
          for (int c = 0; c < 4; ++c) p.out_quats[f][g * 4 + c] = ho[3 + c];
#pragma unroll
          for (int c = 0; c < 3; ++c) p.out_log_scales[f][g * 3 + c] = ho[7 + c];
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, kTmemCols);
  }
}

template <int FEAT, int WIDTH>
cudaError_t launch_tc2_t(const DeformBatch& p, cudaStream_t s) {
  using SM = Tc2Smem<WIDTH>;
  auto kern = deform_tc2_kernel<FEAT, WIDTH>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::TOTAL);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (p.end - p.begin + kM - 1) / kM;
  int64_t grid = std::min<int64_t>(sms, tiles);   // 1 CTA/SM: it owns all 512 TMEM columns
  if (grid < 1) return cudaSuccess;
  prof_mark(FGS_STAGE_DEFORM, true, s);
  kern<<<(unsigned)grid, Parts<FEAT>::THREADS, SM::TOTAL, s>>>(p);
  note_launches(1);
  prof_mark(FGS_STAGE_DEFORM, false, s);
  return cudaGetLastError();
}

}  // namespace

// True if the v2 schedule supports this field (lines of all scales fit the smem line buffer).
bool deform_tc2_supported(const DeformBatch& p) {
  if (!(p.feat == 8 || p.feat == 16 || p.feat == 32)) return false;
  if (p.in_dim > 64) return false;
  long lines = 0;
  for (int l = 0; l < p.n_scales; ++l) lines += 3L * p.res[l] * p.feat;
  return lines <= kMaxLineFloats;
}

cudaError_t launch_deform_tc2(const DeformBatch& p, cudaStream_t s) {
  if (p.end <= p.begin || p.n_t <= 0) return cudaSuccess;
#define FGS_DISPATCH_W(FEAT)                          \
  switch (p.width) {                                  \
    case 32: return launch_tc2_t<FEAT, 32>(p, s);     \
    case 64: return launch_tc2_t<FEAT, 64>(p, s);     \
    case 128: return launch_tc2_t<FEAT, 128>(p, s);   \
    default: return cudaErrorInvalidValue;            \
  }
  switch (p.feat) {
    case 8: FGS_DISPATCH_W(8)
    case 16: FGS_DISPATCH_W(16)
    case 32: FGS_DISPATCH_W(32)
    default: return cudaErrorInvalidValue;
  }
#undef FGS_DISPATCH_W
}

}  // namespace fgs
