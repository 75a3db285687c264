// emit.cu -- SURVEY §8(a) row a5 (tile-key duplication).
//
// Duplication happens between the depth digits and the tile digits of the
// (tile, depth) LSD radix sort (sort.cu): the splats arrive stably sorted by
// depth, and every splat's kept tiles (keys written by project.cu into the
// kept-tile list, row-major) are expanded into (tile key, splat) pairs in that
// order ("key-value pairs").
//
//   pairoff: exclusive scan of the kept-tile counts in depth order
//            (CTA tiles of 4096, reduce-then-scan) -> pair_off[p], P
//   expand : load-balanced expansion -- each warp owns 256 consecutive OUTPUT
//            positions q, brackets their splats [pa, pb] by a 32-ary cooperative
//            search of pair_off (so the heavy-tailed splat sizes -- near splats
//            are both the biggest and the first in depth order -- cost nothing
//            extra), loads the bracket 32 splats at a time into registers and
//            maps each position to its splat by a shuffle search; reads of the
//            list are contiguous runs, writes coalesced.
//            Fused: the 2 x 256-bin digit histogram of the tile keys.
//   (ranges: derived by the last tile-digit pass of the sort, sort.cu)
#include "gsc_internal.cuh"

namespace gsc {

constexpr int kXThreads = 256;
constexpr int kOffItems = 16;
constexpr int kOffTile = kXThreads * kOffItems;   // 4096 sorted positions per CTA tile
constexpr int kExpItems = 8;
constexpr int kExpChunk = 32 * kExpItems;  // output positions per warp chunk

// Exclusive scan of the kept counts in depth order as reduce-then-scan (no look-back: a single-pass
// scan spends most of its time waiting for predecessor tiles at this size).
//   pairoff_reduce: agg[tile] = sum of the tile's 4096 counts (tiles independent)
//   pairoff_scan:   prefix(tile) = sum of agg[< tile] (CTA-parallel, L2-resident), then the tile's
//                   local scan -> pair_off; the last tile also sets n_pairs / overflow.
__device__ __forceinline__ void pairoff_counts(const EmitIn &in, uint32_t C, uint32_t tile, uint32_t (&cnt)[kOffItems]) {
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const uint32_t p0 = tile * kOffTile + warp * (32 * kOffItems) + lane;   // warp w: positions [w*512, +512)
#pragma unroll
  for (int i = 0; i < kOffItems; ++i) {
    const uint32_t p = p0 + 32 * i;
    cnt[i] = p < C ? in.count[in.sorted[p]] : 0u;
  }
}

__global__ void __launch_bounds__(kXThreads)
pairoff_reduce_kernel(EmitIn in, uint32_t *__restrict__ agg, const FrameCounters *__restrict__ ctr) {
  __shared__ uint32_t s_w[kXThreads / 32];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  // when project's kept-tile list overflowed (list_overflow) the lists are incomplete: the frame then
  // has no pairs (n_pairs stays 0, an empty image; nothing reads the list out of bounds) and reports
  // GSC_ECAPACITY
  const uint32_t C = ctr->list_overflow ? 0u : ctr->n_splat;
  const uint32_t ntiles = (C + kOffTile - 1) / kOffTile;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    uint32_t cnt[kOffItems], sum = 0;
    pairoff_counts(in, C, tile, cnt);
    // the gathered counts, in depth order, parked in pair_off (the scan reads them coalesced and
    // overwrites them with the offsets)
    const uint32_t p0 = tile * kOffTile + warp * (32 * kOffItems) + lane;
#pragma unroll
    for (int i = 0; i < kOffItems; ++i) {
      sum += cnt[i];
      if (p0 + 32 * i < C) in.pair_off[p0 + 32 * i] = cnt[i];
    }
    sum = __reduce_add_sync(0xFFFFFFFFu, sum);
    if (lane == 0) s_w[warp] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
#pragma unroll
      for (int w = 0; w < kXThreads / 32; ++w) t += s_w[w];
      agg[tile] = t;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kXThreads)
pairoff_scan_kernel(EmitIn in, uint32_t cap, const uint32_t *__restrict__ agg, FrameCounters *__restrict__ ctr) {
  __shared__ uint32_t s_cnt[kXThreads / 32], s_pre[kXThreads / 32];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  // when project's kept-tile list overflowed (list_overflow) the lists are incomplete: the frame then
  // has no pairs (n_pairs stays 0, an empty image; nothing reads the list out of bounds) and reports
  // GSC_ECAPACITY
  const uint32_t C = ctr->list_overflow ? 0u : ctr->n_splat;
  const uint32_t ntiles = (C + kOffTile - 1) / kOffTile;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    uint32_t cnt[kOffItems], excl[kOffItems], run = 0;
    {   // the counts pairoff_reduce parked in pair_off (coalesced: no second gather)
      const uint32_t p0 = tile * kOffTile + warp * (32 * kOffItems) + lane;
#pragma unroll
      for (int i = 0; i < kOffItems; ++i) cnt[i] = p0 + 32 * i < C ? in.pair_off[p0 + 32 * i] : 0u;
    }
    // prefix of the earlier tiles
    uint32_t pre = 0;
    for (uint32_t j = threadIdx.x; j < tile; j += kXThreads) pre += agg[j];
    pre = __reduce_add_sync(0xFFFFFFFFu, pre);
#pragma unroll
    for (int i = 0; i < kOffItems; ++i) {
      uint32_t inc = cnt[i];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= (uint32_t)o) inc += t;
      }
      excl[i] = run + inc - cnt[i];
      run += __shfl_sync(0xFFFFFFFFu, inc, 31);
    }
    if (lane == 0) { s_cnt[warp] = run; s_pre[warp] = pre; }
    __syncthreads();
    uint32_t wex = 0, tot = 0;
    pre = 0;
#pragma unroll
    for (int w = 0; w < kXThreads / 32; ++w) {
      const uint32_t c = s_cnt[w];
      wex += (uint32_t)w < warp ? c : 0u;
      tot += c;
      pre += s_pre[w];
    }
    const uint32_t p0 = tile * kOffTile + warp * (32 * kOffItems) + lane;
#pragma unroll
    for (int i = 0; i < kOffItems; ++i) {
      const uint32_t p = p0 + 32 * i;
      if (p < C) in.pair_off[p] = pre + wex + excl[i];
    }
    if (threadIdx.x == 0 && tile == ntiles - 1) {
      const uint32_t all = pre + tot;
      ctr->n_pairs = all < cap ? all : cap;
      if (all > cap) ctr->overflow = 1u;
    }
    __syncthreads();   // s_cnt / s_pre reuse
  }
}

// largest p in [0, C) with pair_off[p] <= q (pair_off[0] = 0 <= q), whole warp
__device__ __forceinline__ uint32_t warp_find(const uint32_t *__restrict__ pair_off, uint32_t C, uint32_t q) {
  const uint32_t lane = lane_id();
  uint32_t lo = 0, hi = C - 1;
  while (hi - lo >= 32) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t idx = min(lo + lane * step, hi);
    const uint32_t mask = __ballot_sync(0xFFFFFFFFu, pair_off[idx] <= q);
    const uint32_t l = 31 - __clz(mask);
    const uint32_t nlo = min(lo + l * step, hi);
    if (l < 31) hi = min(hi, lo + (l + 1) * step - 1);
    lo = nlo;
  }
  const uint32_t idx = lo + lane;
  const bool ok = idx <= hi && pair_off[idx] <= q;
  const uint32_t mask = __ballot_sync(0xFFFFFFFFu, ok);
  return lo + (31 - __clz(mask));
}

__global__ void __launch_bounds__(kXThreads)
expand_kernel(EmitIn in, uint32_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out,
              FrameCounters *__restrict__ ctr, uint32_t tbits) {
  const uint32_t tmask = (1u << tbits) - 1u;
  __shared__ uint32_t s_hist[2][256];
  for (int k = threadIdx.x; k < 512; k += kXThreads) (&s_hist[0][0])[k] = 0;
  __syncthreads();
  const uint32_t lane = lane_id();
  // (P, C and the warp index broadcast from lane 0: warp-uniform by construction, and visibly so to
  // the compiler, which then drops the convergence checks around the searches' ballots)
  const uint32_t P = __shfl_sync(0xFFFFFFFFu, ctr->n_pairs, 0), C = __shfl_sync(0xFFFFFFFFu, ctr->n_splat, 0);
  const uint32_t nchunks = (P + kExpChunk - 1) / kExpChunk;
  const uint32_t gw = __shfl_sync(0xFFFFFFFFu, (blockIdx.x * kXThreads + threadIdx.x) >> 5, 0);
  const uint32_t nw = (gridDim.x * kXThreads) >> 5;
  for (uint32_t ch = gw; ch < nchunks; ch += nw) {
    const uint32_t q0 = ch * kExpChunk, q1 = min(q0 + kExpChunk, P) - 1;
    const uint32_t pa = warp_find(in.pair_off, C, q0), pb = warp_find(in.pair_off, C, q1);
    // the chunk's splats [pa, pb] in groups of 32 (one per lane: offset, splat id and list offset in
    // registers, coalesced loads); each position of the group's span finds its splat by a 5-step
    // shuffle search: one dependent global load per position (the list key)
    for (uint32_t g0 = pa; g0 <= pb; g0 += 32) {
      const uint32_t p = g0 + lane;
      const bool v = p <= pb;
      const uint32_t off = v ? in.pair_off[p] : 0xFFFFFFFFu;
      const uint32_t c = v ? in.sorted[p] : 0u;
      const uint32_t lo = v ? in.list_off[c] : 0u;
      const uint32_t gs = max(q0, __shfl_sync(0xFFFFFFFFu, off, 0));
      const uint32_t ge = g0 + 32 <= pb ? min(in.pair_off[g0 + 32], q1 + 1) : q1 + 1;   // exclusive
      for (uint32_t qb = gs; qb < ge; qb += 32) {
        const uint32_t q = qb + lane;
        uint32_t l = 0;
#pragma unroll
        for (uint32_t st = 16; st; st >>= 1)
          if (__shfl_sync(0xFFFFFFFFu, off, l + st) <= q) l += st;
        const uint32_t oc = __shfl_sync(0xFFFFFFFFu, c, l), ol = __shfl_sync(0xFFFFFFFFu, lo, l),
                       oo = __shfl_sync(0xFFFFFFFFu, off, l);
        if (q < ge) {
          GSC_CHECK(q < P && q >= oo && oc < C);
          const uint32_t key = in.list[ol + (q - oo)];
          keys_out[q] = key;
          vals_out[q] = oc;
          atomicAdd(&s_hist[0][key & tmask], 1u);          // the tile sort's two tbits-bit digits
          atomicAdd(&s_hist[1][(key >> tbits) & tmask], 1u);
        }
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 512; k += kXThreads) {
    const uint32_t v = (&s_hist[0][0])[k];
    if (v) atomicAdd(&ctr->hist_tile[0][0] + k, v);
  }
}

struct EmitGrids { int red, scan, exp; };
static PerDevice<EmitGrids> g_emit;

void launch_emit(const EmitIn &in, uint32_t cap, uint32_t *keys_out, uint32_t *vals_out, uint32_t *status,
                 FrameCounters *ctr, int tbits, int num_sms, cudaStream_t st) {
  const EmitGrids &g = g_emit.get([&](EmitGrids &g) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pairoff_reduce_kernel, kXThreads, 0);
    g.red = num_sms * (per_sm > 0 ? per_sm : 1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pairoff_scan_kernel, kXThreads, 0);
    g.scan = num_sms * (per_sm > 0 ? per_sm : 1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, expand_kernel, kXThreads, 0);
    g.exp = num_sms * (per_sm > 0 ? per_sm : 1);
  });
  pairoff_reduce_kernel<<<g.red, kXThreads, 0, st>>>(in, status, ctr);
  pairoff_scan_kernel<<<g.scan, kXThreads, 0, st>>>(in, cap, status, ctr);
  expand_kernel<<<g.exp, kXThreads, 0, st>>>(in, keys_out, vals_out, ctr, (uint32_t)tbits);
}

int emit_tile_size() { return kOffTile; }

}  // namespace gsc
