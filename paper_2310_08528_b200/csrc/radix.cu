// Radix binning path of the splatting (the north_star's "key duplication plus a
// hand-written radix sort on (tile, depth, index) keys"), for frames whose tile lists are long.
//
// The per-tile comparison sorts of render.cu cost O(L log L) per list; when the lists run to thousands
// of instances (large N at moderate resolution: the N-sweep of P:1013-1022 beyond ~300k Gaussians) a
// sort whose passes are linear in the data pays.  Per frame:
//   1. depth sort: the n Gaussians as 64-bit items (depth_key << 32 | gid), culled ones keyed
//      0xFFFFFFFF (last), stable LSD radix sort on the key in 4 passes of 8 bits.  Stable on a gid-ordered
//      input, so equal depth keys stay in gid order: the result is the (depth, index) order R14 needs.
//   2. emit: the instances of the Gaussians in that order, each Gaussian's tiles in row-major order, as
//      items (tile << 32 | gid) at offsets from an exclusive scan of tiles_touched in depth order.
//   3. tile partition: stable LSD radix passes on the tile field (8 bits each, 2 passes for up to 65536
//      tiles): the instances grouped by tile, each tile's run still in (depth, gid) order; the last pass
//      writes the (depth_key << 32 | gid) instances the blend reads, into the tile ranges tile_scan set.
// Every pass is the same three kernels: rx_hist (per-block digit histogram), rx_scan (per digit, the
// exclusive scan over blocks) and rx_scatter (per block: digit bases, a stable rank of each item among
// the block's items of its digit — warp match + per-warp prefix per 256-item round — into a digit-sorted
// shared-memory stage, then a coalesced write-out).  The emission is instance-parallel (each thread finds
// its Gaussian by binary search over the block's offsets).  All deterministic: the output is the unique
// sorted order.
//
// Selection (tile_scan_kernel sets cnt[8] per frame): FGS_TUNE_RADIX = 0 (default) never, 2 always, 1 when
// the frame's mean list length reaches FGS_TUNE_RADIX_MIN_LIST; launch_render launches the path only if
// some frame may take it (mode 2, or mode 1 with at least 64 Gaussians per tile).  Frames on this path
// skip duplicate_kernel and the per-tile sorts; the result is bit-identical to theirs.
// Measured: slower than the per-tile sorts at every N of the sweep (N = 1M, 4 frames of
// 800x800: 539 vs 349 us per frame for the whole render; 3M: 1360 vs 1140) — each instance crosses L2 /
// HBM about seven times here, while a tile's list stays in registers / shared memory through its sort —
// so the default is the per-tile sorts and this path is the north_star's radix formulation, kept exact
// and tested, selectable with FGS_TUNE_RADIX.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fgs_internal.cuh"

namespace fgs {

namespace {

constexpr int kRxThreads = 256;
constexpr int kRxRounds = kRxItems / kRxThreads;     // 16 rounds of 256 items per block
constexpr int kRxBins = 256;

__device__ __forceinline__ uint32_t* rcnt(const RenderBatch& b, int f) {
  return ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.cnt);
}
__device__ __forceinline__ bool radix_frame(const RenderBatch& b, int f) { return rcnt(b, f)[8] != 0u; }

// source / destination buffers of a pass: 0 = inst, 1 = inst2
__device__ __forceinline__ unsigned long long* rbuf(const RenderBatch& b, int f, int which) {
  return ws_ptr<unsigned long long>(b.ws, b.ws_stride, f, which ? b.L.inst2 : b.L.inst);
}

// items of the pass: kind 0 = the n Gaussians (depth sort), 1 = the frame's M instances (tile passes)
__device__ __forceinline__ int64_t rx_count(const RenderBatch& b, int f, int kind) {
  return kind == 0 ? b.n : (int64_t)rcnt(b, f)[1];
}

// (1) items of the depth sort, in gid order, into buffer `dst`
__global__ void __launch_bounds__(256) rx_init_kernel(const __grid_constant__ RenderBatch b, int dst) {
  const int f = blockIdx.y;
  if (!radix_frame(b, f)) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.n) return;
  const uint32_t tt = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.tt)[i];
  const uint32_t key = tt ? ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.keys)[i] : 0xFFFFFFFFu;
  rbuf(b, f, dst)[i] = ((unsigned long long)key << 32) | (uint32_t)i;
}

// per-block digit histogram -> hist[d * nblk + blk]
__global__ void __launch_bounds__(kRxThreads) rx_hist_kernel(const __grid_constant__ RenderBatch b, int src, int kind,
                                                            int shift) {
  const int f = blockIdx.y;
  if (!radix_frame(b, f)) return;
  const int64_t count = rx_count(b, f, kind);
  const int64_t beg = (int64_t)blockIdx.x * kRxItems;
  if (beg >= count) return;
  __shared__ uint32_t h[kRxThreads / 32][kRxBins];      // one histogram per warp
#pragma unroll
  for (int w = 0; w < kRxThreads / 32; ++w) h[w][threadIdx.x] = 0u;
  __syncthreads();
  const unsigned long long* s = rbuf(b, f, src);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = 0; r < kRxRounds; ++r) {
    const int64_t idx = beg + r * kRxThreads + threadIdx.x;
    const bool valid = idx < count;
    const uint32_t d = valid ? (uint32_t)(s[idx] >> shift) & 0xFFu : 0x100u;
    if (kind == 0) {
      // depth digits cluster (a few exponent / high-mantissa values): aggregate a warp's equal digits
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      if (valid && lane == __ffs(peers) - 1) atomicAdd(&h[warp][d], (uint32_t)__popc(peers));
    } else if (valid) {
      atomicAdd(&h[warp][d], 1u);          // tile digits spread: plain warp-private atomics
    }
  }
  __syncthreads();
  uint32_t t = 0;
#pragma unroll
  for (int w = 0; w < kRxThreads / 32; ++w) t += h[w][threadIdx.x];
  const int nblk = b.L.rx_blocks;
  ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.rx_hist)[threadIdx.x * nblk + blockIdx.x] = t;
}

// per digit d (blockIdx.x): exclusive scan of hist[d][0..nblk_eff) in place, total -> dtot[d]
__global__ void __launch_bounds__(kRxThreads) rx_scan_kernel(const __grid_constant__ RenderBatch b, int kind) {
  const int f = blockIdx.y;
  if (!radix_frame(b, f)) return;
  const int64_t count = rx_count(b, f, kind);
  const int nb = (int)((count + kRxItems - 1) / kRxItems);
  uint32_t* h = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.rx_hist) + (size_t)blockIdx.x * b.L.rx_blocks;
  const int per = (nb + kRxThreads - 1) / kRxThreads;
  const int c0 = min(nb, (int)threadIdx.x * per), c1 = min(nb, c0 + per);
  uint32_t s = 0;
  for (int i = c0; i < c1; ++i) s += h[i];
  __shared__ uint32_t sm[kRxThreads];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < kRxThreads; o <<= 1) {          // Hillis-Steele inclusive scan of the chunk sums
    const uint32_t v = threadIdx.x >= (unsigned)o ? sm[threadIdx.x - o] : 0u;
    __syncthreads();
    sm[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = sm[threadIdx.x] - s;
  for (int i = c0; i < c1; ++i) {
    const uint32_t v = h[i];
    h[i] = run;
    run += v;
  }
  if (threadIdx.x == kRxThreads - 1) ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.rx_dtot)[blockIdx.x] = sm[kRxThreads - 1];
}

// stable scatter of the block's items to dst; `final` writes the blend's (depth_key << 32 | gid).
// Each item's rank among the block's items of its digit (stable: warp match + per-warp prefix per 256-item
// round) places it in the block's digit-sorted order in shared memory; the write-out then walks that
// order, so consecutive threads store consecutive addresses of one digit's run (coalesced).
__global__ void __launch_bounds__(kRxThreads) rx_scatter_kernel(const __grid_constant__ RenderBatch b, int src, int dst,
                                                               int kind, int shift, int final_pass) {
  const int f = blockIdx.y;
  if (!radix_frame(b, f)) return;
  const int64_t count = rx_count(b, f, kind);
  const int64_t beg = (int64_t)blockIdx.x * kRxItems;
  if (beg >= count) return;
  const int nitems = (int)(count - beg < (int64_t)kRxItems ? count - beg : (int64_t)kRxItems);
  __shared__ uint32_t s_gbase[kRxBins], s_lbase[kRxBins], s_run[kRxBins], s_cnt[kRxThreads / 32][kRxBins];
  __shared__ unsigned long long stage[kRxItems];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d0 = threadIdx.x;                          // this thread's digit in the per-digit steps
  {
    const uint32_t* hs = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.rx_hist) + (size_t)d0 * b.L.rx_blocks;
    const uint32_t tot = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.rx_dtot)[d0];
    const int nb = (int)((count + kRxItems - 1) / kRxItems);
    const uint32_t my_off = hs[blockIdx.x];                       // exclusive over earlier blocks
    const uint32_t my_cnt = ((int)blockIdx.x + 1 < nb ? hs[blockIdx.x + 1] : tot) - my_off;
    // global digit bases: exclusive scan of the 256 digit totals; local: of this block's digit counts
    s_gbase[d0] = tot;
    s_lbase[d0] = my_cnt;
    __syncthreads();
    for (int o = 1; o < kRxBins; o <<= 1) {
      const uint32_t a = d0 >= o ? s_gbase[d0 - o] : 0u, c = d0 >= o ? s_lbase[d0 - o] : 0u;
      __syncthreads();
      s_gbase[d0] += a;
      s_lbase[d0] += c;
      __syncthreads();
    }
    const uint32_t gb = s_gbase[d0] - tot + my_off, lb = s_lbase[d0] - my_cnt;
    __syncthreads();
    s_gbase[d0] = gb;          // first global slot of this block's digit-d0 run
    s_lbase[d0] = lb;          // its first slot in the block's digit-sorted order
    s_run[d0] = 0u;
  }
  const unsigned long long* s = rbuf(b, f, src);
  const uint32_t lt = (1u << lane) - 1u;
  for (int r = 0; r < kRxRounds; ++r) {
#pragma unroll
    for (int w = 0; w < kRxThreads / 32; ++w) s_cnt[w][threadIdx.x] = 0u;
    __syncthreads();
    const int li = r * kRxThreads + threadIdx.x;
    const bool valid = li < nitems;
    const unsigned long long item = valid ? s[beg + li] : 0ull;
    const uint32_t d = valid ? (uint32_t)(item >> shift) & 0xFFu : 0x100u;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t lrank = __popc(peers & lt);
    if (valid && lrank == 0) s_cnt[warp][d] = __popc(peers);
    __syncthreads();
    {   // per digit (thread = digit): exclusive prefix over the warps, then the running block count
      uint32_t run = s_run[d0];
#pragma unroll
      for (int w = 0; w < kRxThreads / 32; ++w) {
        const uint32_t c = s_cnt[w][d0];
        s_cnt[w][d0] = run;
        run += c;
      }
      s_run[d0] = run;
    }
    __syncthreads();
    if (valid) {
      FGS_DCHECK(s_lbase[d] + s_cnt[warp][d] + lrank < (uint32_t)nitems);
      stage[s_lbase[d] + s_cnt[warp][d] + lrank] = item;
    }
    __syncthreads();           // s_cnt is read above before the next round zeroes it
  }
  unsigned long long* o = rbuf(b, f, dst);
  const uint32_t* keys = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.keys);
  const uint64_t cap = (uint64_t)b.L.cap;
  for (int lp = threadIdx.x; lp < nitems; lp += kRxThreads) {
    const unsigned long long it = stage[lp];
    const uint32_t d = (uint32_t)(it >> shift) & 0xFFu;
    const uint64_t pos = (uint64_t)s_gbase[d] + (uint32_t)(lp - (int)s_lbase[d]);
    FGS_DCHECK(pos < (uint64_t)count);
    if (pos < cap) {
      const uint32_t gid = (uint32_t)it;
      o[pos] = final_pass ? (((unsigned long long)keys[gid] << 32) | gid) : it;
    }
  }
}

// (2) emit, part 1: per block of 4096 depth-ordered Gaussians, the sum of their tiles_touched
__global__ void __launch_bounds__(kRxThreads) rx_emit_sum_kernel(const __grid_constant__ RenderBatch b, int src) {
  const int f = blockIdx.y;
  if (!radix_frame(b, f)) return;
  const int64_t beg = (int64_t)blockIdx.x * kRxItems;
  if (beg >= b.n) return;
  const unsigned long long* s = rbuf(b, f, src);
  const uint32_t* tt = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.tt);
  uint32_t acc = 0;
  for (int r = 0; r < kRxRounds; ++r) {
    const int64_t idx = beg + r * kRxThreads + threadIdx.x;
    if (idx < b.n) acc += tt[(uint32_t)s[idx]];
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ uint32_t sw[kRxThreads / 32];
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kRxThreads / 32; ++w) t += sw[w];
    ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.rx_bsum)[blockIdx.x] = t;
  }
}

// (2) emit, part 2: the block's offsets (base = the earlier blocks' sums; the in-block exclusive scan of
// tiles_touched in depth order, in shared memory), then the block's instances written INSTANCE-parallel:
// thread k of the block's run finds its Gaussian by binary search over the offsets and writes
// (tile << 32 | gid), tiles of a Gaussian in row-major order — consecutive threads, consecutive addresses
__global__ void __launch_bounds__(kRxThreads) rx_emit_kernel(const __grid_constant__ RenderBatch b, int src, int dst) {
  const int f = blockIdx.y;
  if (!radix_frame(b, f)) return;
  const int64_t beg = (int64_t)blockIdx.x * kRxItems;
  if (beg >= b.n) return;
  const int ng = (int)(b.n - beg < (int64_t)kRxItems ? b.n - beg : (int64_t)kRxItems);
  __shared__ uint32_t s_off[kRxItems + 1];
  __shared__ uint32_t s_gid[kRxItems];
  __shared__ uint32_t sm[kRxThreads];
  __shared__ uint64_t s_base;
  {
    const uint32_t* bs = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.rx_bsum);
    uint64_t part = 0;
    for (int i = threadIdx.x; i < (int)blockIdx.x; i += kRxThreads) part += bs[i];
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    __shared__ uint64_t sw[kRxThreads / 32];
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t t = 0;
      for (int w = 0; w < kRxThreads / 32; ++w) t += sw[w];
      s_base = t;
    }
  }
  const unsigned long long* s = rbuf(b, f, src);
  unsigned long long* o = rbuf(b, f, dst);
  const uint32_t* tt = ws_ptr<uint32_t>(b.ws, b.ws_stride, f, b.L.tt);
  const uint2* rect = ws_ptr<uint2>(b.ws, b.ws_stride, f, b.L.rect);
  const uint64_t cap = (uint64_t)b.L.cap;
  // thread t scans ranks [16 t, 16 t + 16) (blocked), the block prefix over threads is one scan
  const int j0 = threadIdx.x * kRxRounds;
  uint32_t loc[kRxRounds];
  uint32_t mine = 0;
#pragma unroll
  for (int j = 0; j < kRxRounds; ++j) {
    const int r = j0 + j;
    uint32_t n_t = 0;
    if (r < ng) {
      const uint32_t g = (uint32_t)s[beg + r];
      s_gid[r] = g;
      n_t = tt[g];
    }
    loc[j] = mine;
    mine += n_t;
  }
  sm[threadIdx.x] = mine;
  __syncthreads();
  for (int off = 1; off < kRxThreads; off <<= 1) {
    const uint32_t v = threadIdx.x >= (unsigned)off ? sm[threadIdx.x - off] : 0u;
    __syncthreads();
    sm[threadIdx.x] += v;
    __syncthreads();
  }
  const uint32_t tbase = sm[threadIdx.x] - mine;
#pragma unroll
  for (int j = 0; j < kRxRounds; ++j)
    if (j0 + j < ng) s_off[j0 + j] = tbase + loc[j];
  const uint32_t total = sm[kRxThreads - 1];
  if (threadIdx.x == 0) s_off[ng] = total;
  __syncthreads();
  const uint64_t base = s_base;
  for (uint32_t k = threadIdx.x; k < total; k += kRxThreads) {
    // the Gaussian of instance k: the last rank j with s_off[j] <= k (culled ranks, tiles_touched 0, sort
    // last and never match)
    int lo = 0, hi = ng - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= k) lo = mid; else hi = mid - 1;
    }
    const uint32_t g = s_gid[lo];
    FGS_DCHECK(lo >= 0 && lo < ng && (int64_t)g < b.n && k - s_off[lo] < tt[g]);
    const uint2 rc = rect[g];
    const int x0 = rc.x & 0xFFFF, y0 = rc.x >> 16, x1 = rc.y & 0xFFFF;
    const int w = x1 - x0;
    const int q = (int)(k - s_off[lo]);
    const int ty = y0 + q / w, tx = x0 + q % w;
    const uint64_t pos = base + k;
    if (pos < cap) o[pos] = ((unsigned long long)(ty * b.gx + tx) << 32) | g;
  }
}

}  // namespace

// Radix path of the frames that take it (all kernels return at once for the others).  Buffer plan: the
// depth sort runs inst2 -> inst -> inst2 -> inst -> inst2 (4 passes), emit inst2 -> inst, the two tile
// passes inst -> inst2 -> inst: the result lands in inst, where the blend reads the lists.
cudaError_t launch_radix_bin(const RenderBatch& b, cudaStream_t s) {
  const unsigned F = (unsigned)b.n_frames;
  const unsigned nb_n = (unsigned)((b.n + kRxItems - 1) / kRxItems);
  const unsigned nb_max = (unsigned)b.L.rx_blocks;
  rx_init_kernel<<<dim3((unsigned)((b.n + 255) / 256), F), 256, 0, s>>>(b, 1);
  int src = 1, launches = 1;
  for (int p = 0; p < 4; ++p) {           // depth key = bits 32..63 of the item
    const int shift = 32 + 8 * p;
    rx_hist_kernel<<<dim3(nb_n, F), kRxThreads, 0, s>>>(b, src, 0, shift);
    rx_scan_kernel<<<dim3(kRxBins, F), kRxThreads, 0, s>>>(b, 0);
    rx_scatter_kernel<<<dim3(nb_n, F), kRxThreads, 0, s>>>(b, src, 1 - src, 0, shift, 0);
    src = 1 - src;
    launches += 3;
  }
  rx_emit_sum_kernel<<<dim3(nb_n, F), kRxThreads, 0, s>>>(b, src);
  rx_emit_kernel<<<dim3(nb_n, F), kRxThreads, 0, s>>>(b, src, 1 - src);
  src = 1 - src;
  launches += 2;
  for (int p = 0; p < 2; ++p) {           // tile id = bits 32..47 of the item (<= 65536 tiles)
    const int shift = 32 + 8 * p;
    rx_hist_kernel<<<dim3(nb_max, F), kRxThreads, 0, s>>>(b, src, 1, shift);
    rx_scan_kernel<<<dim3(kRxBins, F), kRxThreads, 0, s>>>(b, 1);
    rx_scatter_kernel<<<dim3(nb_max, F), kRxThreads, 0, s>>>(b, src, 1 - src, 1, shift, p == 1);
    src = 1 - src;
    launches += 3;
  }
  note_launches(launches);
  return cudaGetLastError();
}

}  // namespace fgs
