// Gaussian deformation field, v3: warp-specialised tcgen05 pipeline (sm_100a).
// PAPER.md §4.2: Eq. 7 HexPlane query, phi_d, heads and additive update
// (P:797-802).  Same arithmetic as deform_tc2.cu; what changes is the schedule.
//
// One persistent CTA per SM over a contiguous range of 128-Gaussian tiles, processed in groups of G
// tiles; per group, for every time t of the batch, every tile of the group is one "tile-frame" i.
// Roles (FEAT >= 16: 768 threads = 6 warpgroups; FEAT = 8: 512 threads, 8 producer warps):
//   producers (warps 0-15) group prologue: the spatial-plane product S = xy . xz . yz of every
//                          (Gaussian, feature) of the group, parked in TENSOR MEMORY, and the knot
//                          window each axis of the group touches; per time t: the three temporal planes
//                          collapsed to 1-D lines at t over those windows only (smem); per tile-frame:
//                          f_h = S . line_x(u_x) . line_y(u_y) . line_z(u_z), split hi/lo (3xTF32) and
//                          stored to TMEM as the A operand.
//   epilogue (warps 16-19) one thread per Gaussian row: D -> bias + ReLU -> the 10 head dot products ->
//                          additive update -> global stores; releases D[i % 2].
//   MMA issuer (warp 20)   one thread: 3 x K/8 tcgen05.mma.kind::tf32 (A from TMEM, W_d hi/lo from
//                          smem) into accumulator D[i % 2]; commits to "A free" and "D[i % 2] full".
//                          Warps 21-23 are idle: they make the MMA role a whole warpgroup, so that
//                          setmaxnreg can move registers from the epilogue and MMA warpgroups (72, 24)
//                          to the producers (96) out of the launch's 80 per thread.
// Producer work on tile-frame i+1 and the epilogue of i-1 overlap the MMAs of i (mbarrier pipeline).
// TMEM columns: D0 | D1 | A_hi | A_lo | S[0..G).  Thread (warp w, lane) touches TMEM lane quarter w % 4.
// Experiment switches (never set in normal builds; FGS_NVCC_EXTRA="-DFGS_EXP_..." with tools/gpu_exp.sh):
// FGS_EXP_NOSTAGE (no time-line staging), FGS_EXP_NOLINE (no line reads), FGS_EXP_NOMMA (no MMAs),
// FGS_EXP_NOEPI (epilogue releases D without the heads) — each removes one part of the schedule so its
// share of the kernel time can be measured; results are wrong under any of them.
// FGS_EXP_TRACE records a per-warp clock64 timeline of CTA 0 (results unchanged; tools/deform_trace.py).
#include <cuda_runtime.h>
#include <limits.h>

#include <algorithm>

#include "fgs_internal.cuh"
#include "tc.cuh"

namespace fgs {

namespace {

constexpr int kM = 128;

// FGS_EXP_TRACE (experiment builds only): lane 0 of every warp of CTA 0 records (tag, clock64) events
// into g_trace[warp]; fgs_exp_trace copies them out (tools/deform_trace.py prints the role timeline)
#ifdef FGS_EXP_TRACE
constexpr int kTraceN = 2048;
__device__ unsigned long long g_trace[24][kTraceN];
#define FGS_TR(tag)                                                                                       \
  do {                                                                                                   \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && tr_n < kTraceN)                                     \
      g_trace[threadIdx.x >> 5][tr_n++] = ((unsigned long long)(tag) << 56) | (clock64() & 0xFFFFFFFFFFFFFFull); \
  } while (0)
#else
#define FGS_TR(tag) do {} while (0)
#endif
constexpr int kTmemCols = 512;
constexpr int kMaxG = 16;
// Shared buffer of the per-frame time lines: only the knot window each axis of a group touches is
// staged, compactly (Morton-ordered models: ~1/6 of the axis per group at D); a group whose windows do
// not fit reads the temporal planes from L2 instead (same arithmetic, bit-identical results).
constexpr int kLineBufFloats = 16384;          // 64 KB
constexpr int kEpiWarps = 4;
// Gaussians per pass of the spatial-plane sampling in the group prologue
constexpr int kProB = 4;
// Producer warps per TMEM lane quarter (each takes FEAT / NP features of every scale).
template <int FEAT>
struct Roles {
  static constexpr int NP = FEAT >= 16 ? 4 : 2;
  static constexpr int PROD_WARPS = 4 * NP;
  static constexpr int PROD_THREADS = 32 * PROD_WARPS;
  static constexpr int EPI0 = PROD_WARPS;                 // first epilogue warp
  static constexpr int MMA_WARP = PROD_WARPS + kEpiWarps;
  // the MMA warp's warpgroup is padded with 3 idle warps so that every role is whole warpgroups and the
  // register file can be re-split with setmaxnreg (producers up, epilogue and MMA down)
  static constexpr int THREADS = 32 * (MMA_WARP + 4);     // 768 (FEAT >= 16) or 512
  static constexpr bool REALLOC = PROD_WARPS == 16;
  // the CTA's pool is what the launch allocated (768 x 80 = 61440): 512 x 96 + 128 x 72 + 128 x 24 fills
  // it exactly (an increase the pool cannot serve blocks forever)
  static constexpr int REG_PROD = 96, REG_EPI = 72, REG_MMA = 24;
  static_assert(!REALLOC || (THREADS == 768 && 16 * REG_PROD + 4 * REG_EPI + 4 * REG_MMA == 24 * 80),
                "setmaxnreg budget must equal the launch allocation (768 threads x 80 registers)");
};

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
  // ((w00 v00 + w01 v01) + w10 v10) + w11 v11, two channels per instruction
  const float2 a00 = make_float2(w00, w00), a01 = make_float2(w01, w01);
  const float2 a10 = make_float2(w10, w10), a11 = make_float2(w11, w11);
  float2 lo = fmul2(a00, make_float2(v00.x, v00.y)), hi = fmul2(a00, make_float2(v00.z, v00.w));
  lo = ffma2(a01, make_float2(v01.x, v01.y), lo);
  hi = ffma2(a01, make_float2(v01.z, v01.w), hi);
  lo = ffma2(a10, make_float2(v10.x, v10.y), lo);
  hi = ffma2(a10, make_float2(v10.z, v10.w), hi);
  lo = ffma2(a11, make_float2(v11.x, v11.y), lo);
  hi = ffma2(a11, make_float2(v11.z, v11.w), hi);
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

// Lines are stored [R][FEAT/4] float4 with the quad index XOR-swizzled by the knot index.
template <int FEAT>
__device__ __forceinline__ int swz(int i, int c4) {
  return c4 ^ (i & (FEAT / 4 - 1));
}

template <int FEAT>
__device__ __forceinline__ int knot0(float u, int R) {
  return min((int)floorf(u * (float)(R - 1)), R - 2);
}

// (1 - w) a + w b in a fixed evaluation order (the staged and the L2 paths must agree bit for bit)
__device__ __forceinline__ float4 lerp4(float4 a, float4 b, float w) {
  // packed fp32x2 (FMUL2 / FFMA2): per lane exactly fmaf(w, b, wa * a)
  const float wa = 1.f - w;
  const float2 wa2 = make_float2(wa, wa), w2 = make_float2(w, w);
  const float2 lo = ffma2(w2, make_float2(b.x, b.y), fmul2(wa2, make_float2(a.x, a.y)));
  const float2 hi = ffma2(w2, make_float2(b.z, b.w), fmul2(wa2, make_float2(a.z, a.w)));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

// linear interpolation at u in [0,1], channel quad c4, of a line whose knot i sits at float offset
// off + i FEAT of `line` (smem; only the group's window of knots is present)
template <int FEAT>
__device__ __forceinline__ float4 lerp_line(const float* line, int off, int R, float u, int c4) {
  const float g = u * (float)(R - 1);
  const int i0 = min((int)floorf(g), R - 2);
  const float fa = g - (float)i0;
  FGS_DCHECK(i0 >= 0 && off + i0 * FEAT >= 0 && off + (i0 + 2) * FEAT <= kLineBufFloats);
  const float4 a = reinterpret_cast<const float4*>(line + off + i0 * FEAT)[swz<FEAT>(i0, c4)];
  const float4 b = reinterpret_cast<const float4*>(line + off + (i0 + 1) * FEAT)[swz<FEAT>(i0 + 1, c4)];
  return lerp4(a, b, fa);
}

// the same value straight from the temporal plane [t_res][R][FEAT] in global memory (L2): time lerp of
// the two rows at knots i0, i0+1, then the lerp in u — the staged path's operations in its order
template <int FEAT>
__device__ __noinline__ float4 lerp_plane(const float* __restrict__ P, int R, int j0, float ft, float u, int c4) {
  const float g = u * (float)(R - 1);
  const int i0 = min((int)floorf(g), R - 2);
  const float fa = g - (float)i0;
  const float4* r0 = reinterpret_cast<const float4*>(P + ((size_t)j0 * R + i0) * FEAT) + c4;
  const float4* r1 = reinterpret_cast<const float4*>(P + ((size_t)(j0 + 1) * R + i0) * FEAT) + c4;
  const float4 a = lerp4(__ldg(r0), __ldg(r1), ft);
  const float4 b = lerp4(__ldg(r0 + FEAT / 4), __ldg(r1 + FEAT / 4), ft);
  return lerp4(a, b, fa);
}

// Head outputs (transposed weights [W][NOUTP]; with the decoders 12 per pass of the epilogue): 10 geometry outputs
// (dX 3, dr 4, ds 3), then with the P:1232 decoders 3K colour outputs and 1 opacity output.
constexpr int kNoutColor = 60;   // 10 + 48 + 1 = 59 at SH degree 3, padded to a multiple of 12

template <int WIDTH, bool COLOR = false>
struct Tc3Smem {
  static constexpr int NOUTP = COLOR ? kNoutColor : 10;   // [W][10] without the decoders: column pairs 80 B
  static constexpr int B_BYTES = 64 * WIDTH * 4;
  static constexpr int OFF_BHI = 0;
  static constexpr int OFF_BLO = OFF_BHI + B_BYTES;
  // tiles per group the TMEM plan allows for phi_d width WIDTH at in_dim 64 (more for smaller in_dim)
  static constexpr int GMAX = WIDTH >= 128 ? 2 : (WIDTH >= 64 ? 4 : kMaxG);
  static constexpr int OFF_LINE = OFF_BLO + B_BYTES;
  static constexpr int OFF_U = OFF_LINE + kLineBufFloats * 4;   // [GMAX][128][4]
  static constexpr int OFF_WH = OFF_U + GMAX * kM * 16;
  static constexpr int OFF_BD = OFF_WH + NOUTP * WIDTH * 4;   // head weights transposed [W][NOUTP]
  static constexpr int OFF_BH = OFF_BD + WIDTH * 4;
  static constexpr int OFF_WIN = OFF_BH + NOUTP * 4;            // int [FGS_MAX_SCALES][3][2]
  static constexpr int OFF_SEG = OFF_WIN + FGS_MAX_SCALES * 6 * 4;   // int [13]: window offsets + fits
  static constexpr int OFF_BAR = OFF_SEG + 16 * 4;
  // barriers: 0 a_full, 1 a_free, 2-3 d_full, 4-5 d_free; then the TMEM base address
  static constexpr int TOTAL = OFF_BAR + 6 * 8 + 16;
  static_assert(OFF_BAR % 8 == 0 && OFF_WH % 16 == 0 && OFF_BD % 16 == 0, "smem carve-up alignment");
};

// With the colour decoders the epilogue (59 head outputs) is the bottleneck: it gets the registers
// (512 x 88 + 128 x 104 + 128 x 24 = 61440, the same pool)
constexpr int kRegProdColor = 88, kRegEpiColor = 104;
static_assert(16 * kRegProdColor + 4 * kRegEpiColor + 4 * 24 == 24 * 80, "setmaxnreg budget (colour)");

template <int N>
__device__ __forceinline__ void tmem_st_n(uint32_t taddr, const float* v) {
  if constexpr (N % 16 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 16) tc::tmem_st16(taddr + i, v + i);
  } else {
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

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}
template <int NTHREADS>
__device__ __forceinline__ void prod_sync() {   // named barrier over the producer warps only
  asm volatile("bar.sync 1, %0;" ::"n"(NTHREADS) : "memory");
}

template <int FEAT, int WIDTH, bool COLOR, bool SPLIT>
__global__ void __launch_bounds__(Roles<FEAT>::THREADS, 1) deform_tc3_kernel(const __grid_constant__ DeformBatch p) {
  using SM = Tc3Smem<WIDTH, COLOR>;
  constexpr int NOUTP = SM::NOUTP;
  using RL = Roles<FEAT>;
  constexpr int kThreads = RL::THREADS, kProdWarps = RL::PROD_WARPS, kProdThreads = RL::PROD_THREADS;
  constexpr int kMmaWarp = RL::MMA_WARP;
  constexpr int FT = FEAT / RL::NP;            // features per (producer thread, scale)
  constexpr int QT = FT / 4;
  constexpr int MAXS = 64 / FEAT;              // max scales (IN <= 64)
  static_assert(32 * FEAT * RL::PROD_WARPS <= kLineBufFloats, "prologue transpose tiles exceed the line buffer");
  constexpr int DW = WIDTH < 32 ? 32 : WIDTH;  // columns of one accumulator
  constexpr uint32_t IDESC = tc::idesc_tf32(kM, WIDTH);
  const int NS = p.n_scales;
  const int IN = p.in_dim;
  const int KP = (IN + 7) & ~7;
  const uint32_t colA_hi = 2 * DW, colA_lo = 2 * DW + KP, colS = 2 * DW + 2 * KP;
  const int G = min(SM::GMAX, (kTmemCols - (int)colS) / IN);
  FGS_DCHECK(G >= 1 && (int)colS + G * IN <= kTmemCols && NS <= MAXS && IN == NS * FEAT);

  extern __shared__ __align__(128) unsigned char smem[];
  float* line = reinterpret_cast<float*>(smem + SM::OFF_LINE);
  float* U = reinterpret_cast<float*>(smem + SM::OFF_U);
  float* Wh = reinterpret_cast<float*>(smem + SM::OFF_WH);
  float* bd = reinterpret_cast<float*>(smem + SM::OFF_BD);
  float* bh = reinterpret_cast<float*>(smem + SM::OFF_BH);
  int* win = reinterpret_cast<int*>(smem + SM::OFF_WIN);
  int* segoff = reinterpret_cast<int*>(smem + SM::OFF_SEG);   // [3 NS] float offset of knot 0; [15] fits
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM::OFF_BAR);
  uint64_t* a_full = bar + 0;
  uint64_t* a_free = bar + 1;
  uint64_t* d_full = bar + 2;
  uint64_t* d_free = bar + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 6);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef FGS_EXP_TRACE
  int tr_n = 0;
  if (blockIdx.x == 0 && lane == 0)
    for (int k = 0; k < kTraceN; ++k) g_trace[warp][k] = 0;
#endif

  // ---- setup (all threads) ----
  for (int i = tid; i < WIDTH * KP; i += kThreads) {
    const int n = i / KP, k = i - n * KP;
    const float w = k < IN ? p.w_d[n * IN + k] : 0.f;
    float hi, lo;
    tc::tf32_split(w, hi, lo);
    const uint32_t o = core_off(n, k, WIDTH);
    *reinterpret_cast<float*>(smem + SM::OFF_BHI + o) = hi;
    *reinterpret_cast<float*>(smem + SM::OFF_BLO + o) = lo;
  }
  const int n_c = COLOR ? p.n_c : 0;                 // colour outputs (0 without phi_C)
  const int n_out = 10 + n_c + ((COLOR && p.w_a) ? 1 : 0);
  for (int i = tid; i < NOUTP * WIDTH; i += kThreads) {
    const int c = i / NOUTP, o = i - NOUTP * c;    // WhT[c][o] = head output o, hidden column c
    float w = 0.f;
    if (o < 3) w = p.w_x[o * WIDTH + c];
    else if (o < 7) w = p.w_r[(o - 3) * WIDTH + c];
    else if (o < 10) w = p.w_s[(o - 7) * WIDTH + c];
    else if (o < 10 + n_c) w = p.w_c[(o - 10) * WIDTH + c];
    else if (o < n_out) w = p.w_a[c];
    Wh[i] = w;
  }
  for (int o = tid; o < NOUTP; o += kThreads) {
    float bb = 0.f;
    if (o < 3) bb = p.b_x[o];
    else if (o < 7) bb = p.b_r[o - 3];
    else if (o < 10) bb = p.b_s[o - 7];
    else if (o < 10 + n_c) bb = p.b_c[o - 10];
    else if (o < n_out) bb = p.b_a[0];
    bh[o] = bb;
  }
  for (int i = tid; i < WIDTH; i += kThreads) bd[i] = p.b_d[i];
  if (tid == 0) {
    tc::mbar_init(a_full, kProdWarps);
    tc::mbar_init(a_free, 1);
    tc::mbar_init(d_full + 0, 1);
    tc::mbar_init(d_full + 1, 1);
    tc::mbar_init(d_free + 0, kEpiWarps);
    tc::mbar_init(d_free + 1, kEpiWarps);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, kTmemCols);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  const int64_t count = p.end - p.begin;
  const int64_t tiles = (count + kM - 1) / kM;
  // tile indices fit 32 bits (the host rejects ranges of >= 2^31 tiles); 32-bit loop state keeps the
  // producers' register budget for the hot loop
  // Work split: whole tiles per CTA when there are at least as many tiles as CTAs; otherwise (small
  // models) CTAs take contiguous ranges of TILE-FRAMES (w = tile * n_t + f), so every SM works — at
  // most a CTA's first and last tile are shared with its neighbours (their spatial products are then
  // computed twice).  CTA c owns w in [w_beg, w_end).
  const int64_t NT = p.n_t;
  constexpr bool split = SPLIT;                    // chosen at launch: tiles < CTAs
  int64_t w_beg, w_end;
  if (!split) {
    w_beg = tiles * blockIdx.x / gridDim.x * NT;
    w_end = tiles * (blockIdx.x + 1) / gridDim.x * NT;
  } else {
    w_beg = tiles * NT * blockIdx.x / gridDim.x;
    w_end = tiles * NT * (blockIdx.x + 1) / gridDim.x;
  }
  const int t_beg = (int)(w_beg / NT), t_end = w_end > w_beg ? (int)((w_end - 1) / NT) + 1 : t_beg;
  auto in_range = [&](int t, int f) {
    if (!split) return true;
    const int64_t w = (int64_t)t * NT + f;
    return w >= w_beg && w < w_end;
  };
  auto group_needs = [&](int gstart, int ng, int f) {   // some tile of the group has frame f here
    if (!split) return true;
    bool any = false;
    for (int gt = 0; gt < ng; ++gt) any = any || in_range(gstart + gt, f);
    return any;
  };

  if (warp < kProdWarps) {
    // =============================================================== producers
    if constexpr (RL::REALLOC) tc::setmaxnreg_inc<COLOR ? kRegProdColor : RL::REG_PROD>();
    const int quarter = warp & 3, part = warp >> 2;   // part: which FT-feature slice of each scale
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    if (part == 0) {   // zero the K padding columns of A once (never written afterwards)
      for (int k = IN; k < KP; k += 4) {
        const float z[4] = {0.f, 0.f, 0.f, 0.f};
        tc::tmem_st4(lane_base + colA_hi + k, z);
        tc::tmem_st4(lane_base + colA_lo + k, z);
      }
      tc::tmem_st_wait();
    }
    uint32_t it = 0;   // tile-frame counter
    for (int gstart = t_beg; gstart < t_end; gstart += G) {
      const int ng = min(G, t_end - gstart);
      FGS_TR(1);   // group start
      // ---- group prologue: grid coordinates (smem), knot windows, spatial products S (TMEM) ----
      prod_sync<kProdThreads>();     // previous group's line / U readers are done
      if (tid < FGS_MAX_SCALES * 3) { win[2 * tid] = INT_MAX; win[2 * tid + 1] = INT_MIN; }
      prod_sync<kProdThreads>();
      // (1) grid coordinates u (smem U) and knot windows: thread (quarter, part) takes the tiles
      //     gt = part mod NP of the group
      for (int gt = part; gt < ng; gt += RL::NP) {
        // rows past the end of the range (ragged last tile) take the coordinates of the tile's row 0,
        // which always exists: their line reads then stay inside the group's knot windows (a padding
        // row at u = 0 could fall outside them and read below the staged segment — found by the checked
        // build).  Their S is 0 and their outputs are never stored.
        int64_t g = p.begin + (int64_t)(gstart + gt) * kM + row;
        if (g >= p.end) g = p.begin + (int64_t)(gstart + gt) * kM;
        float u[3] = {0.f, 0.f, 0.f};
        {
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const float m = __ldg(p.means + g * 3 + a);
            u[a] = fminf(fmaxf((m - p.bmin[a]) / p.ext[a], 0.f), 1.f);
          }
#pragma unroll
          for (int l = 0; l < MAXS; ++l) {
            if (l >= NS) break;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              const int i0 = knot0<FEAT>(u[a], p.res[l]);
              atomicMin(win + (l * 3 + a) * 2, i0);
              atomicMax(win + (l * 3 + a) * 2 + 1, i0 + 1);
            }
          }
        }
        FGS_DCHECK(gt < SM::GMAX);
        float* Ur = U + (gt * kM + row) * 4;
        Ur[0] = u[0]; Ur[1] = u[1]; Ur[2] = u[2];
      }
      prod_sync<kProdThreads>();     // U complete
      // (2) S = xy . xz . yz (bilinear, Eq. 7's spatial planes) of every (Gaussian, feature): one warp
      //     per (tile, scale) of its lane quarter, LANES OVER FEATURES so that every corner read is one
      //     coalesced 128-B plane row; the 32 x FEAT result is transposed through the (idle) line
      //     buffer so thread = Gaussian row for the TMEM store.
      {
        float* T = line + warp * (32 * FEAT);
        const bool fl = lane < FEAT;
        for (int unit = part; unit < ng * NS; unit += RL::NP) {
          const int gt = unit / NS, l = unit - gt * NS;
          const int R = p.res[l];
          const float Rm = (float)(R - 1);
          const float* Ur = U + (gt * kM + row) * 4;
          const float vm = p.begin + (int64_t)(gstart + gt) * kM + row < p.end ? 1.f : 0.f;
          int off[3];
          float fa[3], fb[3];
#pragma unroll
          for (int pl = 0; pl < 3; ++pl) {
            const float ga = Ur[pl < 2 ? 0 : 1] * Rm, gb = Ur[pl == 0 ? 1 : 2] * Rm;
            const int i0 = min((int)floorf(ga), R - 2), j0 = min((int)floorf(gb), R - 2);
            fa[pl] = ga - (float)i0;
            fb[pl] = gb - (float)j0;
            off[pl] = (j0 * R + i0) * FEAT;
          }
          const float* P0 = p.planes[l][0] + lane;
          const float* P1 = p.planes[l][1] + lane;
          const float* P2 = p.planes[l][2] + lane;
          const int rs = R * FEAT;
          // kProB Gaussians per pass: their 12 kProB corner reads are issued before any is used (the
          // prologue is bound by L2 latency, not bandwidth)
          for (int i0 = 0; i0 < 32; i0 += kProB) {
            float v[kProB][3][4];
#pragma unroll
            for (int b = 0; b < kProB; ++b) {
#pragma unroll
              for (int pl = 0; pl < 3; ++pl) {
                const int o = __shfl_sync(0xffffffffu, off[pl], i0 + b);
                const float* P = (pl == 0 ? P0 : pl == 1 ? P1 : P2) + o;
                v[b][pl][0] = v[b][pl][1] = v[b][pl][2] = v[b][pl][3] = 0.f;
                if (fl) {
                  v[b][pl][0] = __ldg(P); v[b][pl][1] = __ldg(P + FEAT);
                  v[b][pl][2] = __ldg(P + rs); v[b][pl][3] = __ldg(P + rs + FEAT);
                }
              }
            }
#pragma unroll
            for (int b = 0; b < kProB; ++b) {
              const int i = i0 + b;
              float s = __shfl_sync(0xffffffffu, vm, i);
#pragma unroll
              for (int pl = 0; pl < 3; ++pl) {
                const float a = __shfl_sync(0xffffffffu, fa[pl], i);
                const float bb = __shfl_sync(0xffffffffu, fb[pl], i);
                const float top = fmaf(a, v[b][pl][1], (1.f - a) * v[b][pl][0]);
                const float bot = fmaf(a, v[b][pl][3], (1.f - a) * v[b][pl][2]);
                s *= fmaf(bb, bot, (1.f - bb) * top);
              }
              if (fl) T[i * FEAT + (lane ^ (i & (FEAT - 1)))] = s;
            }
          }
          __syncwarp();
          FGS_DCHECK((int)colS + gt * IN + (l + 1) * FEAT <= kTmemCols);
          float sv[FEAT];
#pragma unroll
          for (int c = 0; c < FEAT; ++c) sv[c] = T[lane * FEAT + (c ^ (lane & (FEAT - 1)))];
          tmem_st_n<FEAT>(lane_base + colS + gt * IN + l * FEAT, sv);
          __syncwarp();
        }
      }
      tc::tmem_st_wait();
      FGS_TR(2);   // spatial products stored
      // ---- compact layout of the group's knot windows in the line buffer (or the L2 path) ----
      prod_sync<kProdThreads>();     // windows complete
      if (tid == 0) {
        int o = 0;
        for (int sg = 0; sg < 3 * NS; ++sg) {
          const int lo = win[2 * sg], hi = win[2 * sg + 1];
          segoff[sg] = o - lo * FEAT;                    // knot i of segment sg at o + (i - lo) FEAT
          if (lo <= hi) o += (hi - lo + 1) * FEAT;
        }
        segoff[15] = o <= kLineBufFloats ? 1 : 0;
      }
      prod_sync<kProdThreads>();
      const bool staged = segoff[15] != 0;
      for (int f = 0; f < p.n_t; ++f) {
        if (!group_needs(gstart, ng, f)) continue;    // CTA-uniform
        const float t = p.t[f];
        const int Tn = p.t_res;
        const float gt_ = t * (float)(Tn - 1);
        const int j0 = min((int)floorf(gt_), Tn - 2);
        const float ft = gt_ - (float)j0;
        // ---- stage the temporal lines at t over the group's knot windows (time lerp of 2 rows) ----
        prod_sync<kProdThreads>();   // U/win visible; previous frame's line readers done
        FGS_TR(3);   // staging start
#ifdef FGS_EXP_NOSTAGE
        if (false) {
#else
        if (staged) {
#endif
#pragma unroll
          for (int l = 0; l < MAXS; ++l) {
            if (l >= NS) break;
            const int R = p.res[l];
            const int per_plane = R * (FEAT / 4);
#pragma unroll
            for (int pl = 0; pl < 3; ++pl) {
              const int sg = l * 3 + pl;
              const int lo = win[2 * sg], hi = win[2 * sg + 1];
              if (lo > hi) continue;
              float4* dst = reinterpret_cast<float4*>(line + segoff[sg]);
              const float4* P0 = reinterpret_cast<const float4*>(p.planes[l][3 + pl]) + (size_t)j0 * per_plane;
              const float4* P1 = P0 + per_plane;
              const int n_items = (hi - lo + 1) * (FEAT / 4);
              for (int q = tid; q < n_items; q += kProdThreads) {
                const int rem = lo * (FEAT / 4) + q;
                const int i = rem / (FEAT / 4), c4 = rem - i * (FEAT / 4);
                FGS_DCHECK(segoff[sg] + i * FEAT >= 0 && segoff[sg] + (i + 1) * FEAT <= kLineBufFloats && i < R);
                dst[i * (FEAT / 4) + swz<FEAT>(i, c4)] = lerp4(__ldg(P0 + rem), __ldg(P1 + rem), ft);
              }
            }
          }
        }
        FGS_TR(4);   // staging issued
        prod_sync<kProdThreads>();
        FGS_TR(5);   // staging complete (all producers)
        for (int gt = 0; gt < ng; ++gt) {
          if (!in_range(gstart + gt, f)) continue;
          const uint32_t itc = it++;
          const float4 u4 = *reinterpret_cast<const float4*>(U + (gt * kM + row) * 4);   // one LDS.128
          const float ux = u4.x, uy = u4.y, uz = u4.z;
          float hi[MAXS][FT], lo[MAXS][FT];
#pragma unroll
          for (int l = 0; l < MAXS; ++l) {
            if (l >= NS) break;
            const int R = p.res[l];
            float sv[FT];
            tmem_ld_n<FT>(lane_base + colS + gt * IN + l * FEAT + part * FT, sv);
            float4 tl[QT][3];
#ifdef FGS_EXP_NOLINE
            if (true) {
#pragma unroll
              for (int qq = 0; qq < QT; ++qq) tl[qq][0] = tl[qq][1] = tl[qq][2] = make_float4(ux, uy, uz, 1.f);
            } else
#endif
            if (staged) {
              const int o0 = segoff[3 * l + 0], o1 = segoff[3 * l + 1], o2 = segoff[3 * l + 2];
#pragma unroll
              for (int qq = 0; qq < QT; ++qq) {
                const int c4 = part * QT + qq;
                tl[qq][0] = lerp_line<FEAT>(line, o0, R, ux, c4);
                tl[qq][1] = lerp_line<FEAT>(line, o1, R, uy, c4);
                tl[qq][2] = lerp_line<FEAT>(line, o2, R, uz, c4);
              }
            } else {
#pragma unroll
              for (int qq = 0; qq < QT; ++qq) {
                const int c4 = part * QT + qq;
                tl[qq][0] = lerp_plane<FEAT>(p.planes[l][3], R, j0, ft, ux, c4);
                tl[qq][1] = lerp_plane<FEAT>(p.planes[l][4], R, j0, ft, uy, c4);
                tl[qq][2] = lerp_plane<FEAT>(p.planes[l][5], R, j0, ft, uz, c4);
              }
            }
#pragma unroll
            for (int qq = 0; qq < QT; ++qq) {
              const float4 a = tl[qq][0], b = tl[qq][1], c = tl[qq][2];
              // S . (a . b . c), packed two channels per instruction
              const float2 p0 = fmul2(make_float2(sv[4 * qq + 0], sv[4 * qq + 1]),
                                      fmul2(fmul2(make_float2(a.x, a.y), make_float2(b.x, b.y)), make_float2(c.x, c.y)));
              const float2 p1 = fmul2(make_float2(sv[4 * qq + 2], sv[4 * qq + 3]),
                                      fmul2(fmul2(make_float2(a.z, a.w), make_float2(b.z, b.w)), make_float2(c.z, c.w)));
              const float fh[4] = {p0.x, p0.y, p1.x, p1.y};
#pragma unroll
              for (int e = 0; e < 4; ++e) tc::tf32_split(fh[e], hi[l][4 * qq + e], lo[l][4 * qq + e]);
            }
          }
          FGS_TR(6);   // A values computed
          // A is single-buffered: wait until the MMAs of tile-frame it-1 have read it
          if (itc > 0) tc::mbar_wait(a_free, (itc - 1) & 1u);
          tc::fence_after_sync();
          FGS_TR(7);   // A free
#pragma unroll
          for (int l = 0; l < MAXS; ++l) {
            if (l >= NS) break;
            tmem_st_n<FT>(lane_base + colA_hi + l * FEAT + part * FT, hi[l]);
            tmem_st_n<FT>(lane_base + colA_lo + l * FEAT + part * FT, lo[l]);
          }
          tc::tmem_st_wait();
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(a_full);
          FGS_TR(8);   // A stored + arrived
        }
      }
    }
  } else if (warp >= kMmaWarp) {
    // =============================================================== MMA issuer (+3 idle warps)
    if constexpr (RL::REALLOC) tc::setmaxnreg_dec<RL::REG_MMA>();
    if (warp == kMmaWarp && lane == 0) {
      const uint32_t b_hi = tc::smem_u32(smem + SM::OFF_BHI), b_lo = tc::smem_u32(smem + SM::OFF_BLO);
      uint32_t it = 0;
      for (int gstart = t_beg; gstart < t_end; gstart += G) {
        const int ng = min(G, t_end - gstart);
        for (int f = 0; f < p.n_t; ++f) {
          for (int gt = 0; gt < ng; ++gt) {
            if (!in_range(gstart + gt, f)) continue;
            const uint32_t itc = it++;
            const uint32_t buf = itc & 1u;
            FGS_TR(10);
            tc::mbar_wait(a_full, itc & 1u);
            FGS_TR(11);   // A full
            if (itc >= 2) tc::mbar_wait(d_free + buf, ((itc >> 1) - 1) & 1u);
            tc::fence_after_sync();
            FGS_TR(12);   // D free
            const uint32_t d = tmem + buf * DW;
#ifndef FGS_EXP_NOMMA
            for (int s = 0; s < KP / 8; ++s) {
              const uint32_t bo = (uint32_t)s * (2 * (WIDTH / 8) * 128);
              const uint64_t dbh = tc::smem_desc(b_hi + bo, (WIDTH / 8) * 128, 128);
              const uint64_t dbl = tc::smem_desc(b_lo + bo, (WIDTH / 8) * 128, 128);
              tc::mma_tf32_ts(d, tmem + colA_lo + 8 * s, dbh, IDESC, s > 0 ? 1u : 0u);
              tc::mma_tf32_ts(d, tmem + colA_hi + 8 * s, dbl, IDESC, 1u);
              tc::mma_tf32_ts(d, tmem + colA_hi + 8 * s, dbh, IDESC, 1u);
            }
#endif
            tc::mma_commit(a_free);
            tc::mma_commit(d_full + buf);
            FGS_TR(13);   // MMAs issued
          }
        }
      }
    }
  } else {
    // =============================================================== epilogue
    if constexpr (RL::REALLOC) {
      if constexpr (COLOR) tc::setmaxnreg_inc<kRegEpiColor>();
      else tc::setmaxnreg_dec<RL::REG_EPI>();
    }
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    uint32_t it = 0;
    for (int gstart = t_beg; gstart < t_end; gstart += G) {
      const int ng = min(G, t_end - gstart);
      for (int f = 0; f < p.n_t; ++f) {
        for (int gt = 0; gt < ng; ++gt) {
          if (!in_range(gstart + gt, f)) continue;
          const uint32_t itc = it++;
          const int64_t g = p.begin + (int64_t)(gstart + gt) * kM + row;
          const bool valid = g < p.end;
          float cx[10];
          if (valid) {
#pragma unroll
            for (int c = 0; c < 3; ++c) cx[c] = __ldg(p.means + g * 3 + c);
#pragma unroll
            for (int c = 0; c < 4; ++c) cx[3 + c] = __ldg(p.quats + g * 4 + c);
#pragma unroll
            for (int c = 0; c < 3; ++c) cx[7 + c] = __ldg(p.log_scales + g * 3 + c);
          }
          const uint32_t buf = itc & 1u;
          FGS_TR(20);
          tc::mbar_wait(d_full + buf, (itc >> 1) & 1u);
          tc::fence_after_sync();
          FGS_TR(21);   // D full
#ifdef FGS_EXP_NOEPI
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(d_free + buf);
          continue;
#endif
          // head outputs in passes of 12 over the hidden columns (one pass without the P:1232
          // decoders); the geometry outputs (pass 0) are kept, the colour / opacity ones stored
          float ho[12];
          const int npass = COLOR ? (n_out + 11) / 12 : 1;
          for (int pass = 0; pass < npass; ++pass) {
            float2 acc[6];
#pragma unroll
            for (int o = 0; o < 6; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
            for (int c0 = 0; c0 < WIDTH; c0 += 16) {
              float v[16];
              tc::tmem_ld16(lane_base + buf * DW + (uint32_t)c0, v);
              if (pass == npass - 1 && c0 + 16 >= WIDTH) {   // all of D read: hand the buffer back
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) mbar_arrive(d_free + buf);
              }
#pragma unroll
              for (int i = 0; i < 16; i += 2) {
                // bias added to the column pair (c, c + 1) by one FADD2 (each half rounded as the
                // scalar add); every output sums its columns in ascending order, as before
                const int c = c0 + i;
                const float2 z = fadd2(make_float2(v[i], v[i + 1]), make_float2(bd[c], bd[c + 1]));
                const float2 fa = make_float2(fmaxf(z.x, 0.f), fmaxf(z.x, 0.f));
                const float2 fb = make_float2(fmaxf(z.y, 0.f), fmaxf(z.y, 0.f));
                if constexpr (!COLOR) {
                  // the pair's 20 weights are 80 contiguous bytes ([W][10]): five 16-B loads
                  FGS_DCHECK((c + 2) * NOUTP <= NOUTP * WIDTH);
                  const float4* w4 = reinterpret_cast<const float4*>(Wh + c * NOUTP);
                  const float4 w0 = w4[0], w1 = w4[1], w2 = w4[2], w3 = w4[3], w5 = w4[4];
                  acc[0] = ffma2(fa, make_float2(w0.x, w0.y), acc[0]);
                  acc[1] = ffma2(fa, make_float2(w0.z, w0.w), acc[1]);
                  acc[2] = ffma2(fa, make_float2(w1.x, w1.y), acc[2]);
                  acc[3] = ffma2(fa, make_float2(w1.z, w1.w), acc[3]);
                  acc[4] = ffma2(fa, make_float2(w2.x, w2.y), acc[4]);
                  acc[0] = ffma2(fb, make_float2(w2.z, w2.w), acc[0]);
                  acc[1] = ffma2(fb, make_float2(w3.x, w3.y), acc[1]);
                  acc[2] = ffma2(fb, make_float2(w3.z, w3.w), acc[2]);
                  acc[3] = ffma2(fb, make_float2(w5.x, w5.y), acc[3]);
                  acc[4] = ffma2(fb, make_float2(w5.z, w5.w), acc[4]);
                } else {
#pragma unroll
                  for (int h = 0; h < 2; ++h) {
                    const float2 fd2 = h ? fb : fa;
                    FGS_DCHECK((c + h) * NOUTP + 12 * pass + 12 <= NOUTP * WIDTH);
                    const float4* w4 = reinterpret_cast<const float4*>(Wh + (c + h) * NOUTP + 12 * pass);
                    const float4 wa = w4[0], wb = w4[1], wc = w4[2];
                    acc[0] = ffma2(fd2, make_float2(wa.x, wa.y), acc[0]);
                    acc[1] = ffma2(fd2, make_float2(wa.z, wa.w), acc[1]);
                    acc[2] = ffma2(fd2, make_float2(wb.x, wb.y), acc[2]);
                    acc[3] = ffma2(fd2, make_float2(wb.z, wb.w), acc[3]);
                    acc[4] = ffma2(fd2, make_float2(wc.x, wc.y), acc[4]);
                    acc[5] = ffma2(fd2, make_float2(wc.z, wc.w), acc[5]);
                  }
                }
              }
            }
            if (pass == 0) {
#pragma unroll
              for (int o = 0; o < 6; ++o) { ho[2 * o] = acc[o].x; ho[2 * o + 1] = acc[o].y; }
            }
            if (COLOR && valid) {
#pragma unroll
              for (int j = 0; j < 12; ++j) {
                const int o = 12 * pass + j;
                const float a = (j & 1) ? acc[j >> 1].y : acc[j >> 1].x;
                if (o >= 10 && o < 10 + n_c)
                  p.out_sh[f][g * n_c + (o - 10)] = p.sh_in[g * n_c + (o - 10)] + (a + bh[o]);
                else if (o == 10 + n_c && o < n_out)
                  p.out_opacity[f][g] = p.opac_in[g] + (a + bh[o]);
              }
            }
          }
          if (valid) {
#pragma unroll
            for (int o = 0; o < 10; ++o) ho[o] = cx[o] + (ho[o] + bh[o]);
            // every replica (one by default; with fgs_deform_range_peers each rank's gather buffer,
            // remote ones written over NVLink right here, tile by tile)
            for (int q = 0; q < p.n_peer; ++q) {
              const int64_t off = p.peer_off[q];
              float* om = reinterpret_cast<float*>(reinterpret_cast<char*>(p.out_means[f] + g * 3) + off);
              float* oq = reinterpret_cast<float*>(reinterpret_cast<char*>(p.out_quats[f] + g * 4) + off);
              float* os = reinterpret_cast<float*>(reinterpret_cast<char*>(p.out_log_scales[f] + g * 3) + off);
#pragma unroll
              for (int c = 0; c < 3; ++c) om[c] = ho[c];
#pragma unroll
              for (int c = 0; c < 4; ++c) oq[c] = ho[3 + c];
#pragma unroll
              for (int c = 0; c < 3; ++c) os[c] = ho[7 + c];
            }
          }
          FGS_TR(22);   // rows stored
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

template <int FEAT, int WIDTH, bool COLOR>
cudaError_t launch_tc3_t(const DeformBatch& p, cudaStream_t s) {
  using SM = Tc3Smem<WIDTH, COLOR>;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (p.end - p.begin + kM - 1) / kM;
  // 1 CTA/SM (it owns all 512 TMEM columns); fewer tiles than SMs: split tiles by frame (the colour
  // decoders keep whole tiles)
  const bool split = !COLOR && tiles < sms;
  auto kern = split ? deform_tc3_kernel<FEAT, WIDTH, COLOR, !COLOR> : deform_tc3_kernel<FEAT, WIDTH, COLOR, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::TOTAL);
  if (e != cudaSuccess) return e;
  int64_t grid = split ? std::min<int64_t>(sms, tiles * (int64_t)p.n_t) : std::min<int64_t>(sms, tiles);
  if (grid < 1) return cudaSuccess;
  prof_mark(FGS_STAGE_DEFORM, true, s);
  kern<<<(unsigned)grid, Roles<FEAT>::THREADS, SM::TOTAL, s>>>(p);
  note_launches(1);
  prof_mark(FGS_STAGE_DEFORM, false, s);
  return cudaGetLastError();
}

}  // namespace

// True if the v3 schedule supports this field (lines of all scales fit the smem line buffer, the
// accumulators and A leave room for at least one tile of S in TMEM).
bool deform_tc3_supported(const DeformBatch& p) {
  if (!(p.feat == 8 || p.feat == 16 || p.feat == 32)) return false;
  if (p.in_dim > 64) return false;
  const int DW = p.width < 32 ? 32 : p.width, KP = (p.in_dim + 7) & ~7;
  return kTmemCols - (2 * DW + 2 * KP) >= p.in_dim;
}

cudaError_t launch_deform_tc3(const DeformBatch& p, cudaStream_t s) {
  if (p.end <= p.begin || p.n_t <= 0) return cudaSuccess;
  if ((p.end - p.begin + kM - 1) / kM >= (int64_t)INT_MAX) return cudaErrorInvalidValue;
  const bool color = p.w_c || p.w_a;
  if (p.n_c + 11 > kNoutColor) return cudaErrorInvalidValue;
#define FGS_DISPATCH_W(FEAT)                                                                        \
  switch (p.width) {                                                                                \
    case 32: return color ? launch_tc3_t<FEAT, 32, true>(p, s) : launch_tc3_t<FEAT, 32, false>(p, s);    \
    case 64: return color ? launch_tc3_t<FEAT, 64, true>(p, s) : launch_tc3_t<FEAT, 64, false>(p, s);    \
    case 128: return color ? launch_tc3_t<FEAT, 128, true>(p, s) : launch_tc3_t<FEAT, 128, false>(p, s); \
    default: return cudaErrorInvalidValue;                                                          \
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

#ifdef FGS_EXP_TRACE
extern "C" int fgs_exp_trace(void* dst) {   // 24 x kTraceN x 8 bytes of CTA 0's events
  return (int)cudaMemcpyFromSymbol(dst, fgs::g_trace, sizeof(fgs::g_trace));
}
#endif
