// sort.cu -- SURVEY §8(a) rows a5 (key duplication), a6 (radix sort by
// (tile, depth)) and a7 (tile ranges).
//
// The (tile, depth) order is produced as an LSD radix sort whose depth digits
// run BEFORE duplication: the splats are first stably sorted by their 32-bit
// depth key (4 onesweep passes over one key per splat), then duplicated into
// (tile, splat) pairs in depth order ("key-value pairs"), then stably
// sorted by the 14-bit tile id (2 onesweep passes).  Stability of every pass
// makes the result identical to one sort of 46-bit (tile << 32 | depth) keys
// with ties broken by the Gaussian slot g (the oracle's order), while moving
// ~2.5x fewer bytes than duplicating first.
//
// Onesweep pass (Adinets & Merrill 2022 style): one kernel per 8-bit digit;
// tiles of 4096 keys acquired in launch order through an atomic counter;
// stable block-local ranking (per-warp digit peer masks by shared atomicOr); per-digit decoupled look-back
// across tiles; scatter through shared memory for coalesced writes.  The
// global digit histograms come fused from the producing kernel (project for
// depth keys, emit for tile keys).  Look-back status words live in two
// buffers that alternate between passes; each pass clears the other buffer's
// entries for the tiles it owns, so no per-sort memset is needed (an even
// number of passes leaves buffer A clean).
#include "gsc_internal.cuh"

namespace gsc {

constexpr int kSThreads = 256;
constexpr int kSWarps = kSThreads / 32;
constexpr int kSItems = 16;
constexpr int kSTile = kSThreads * kSItems;   // 4096 keys
constexpr int kBins = 256;

struct SortSmem {
  uint2 kv[kSTile];                      // (key, value) interleaved: one 64-bit SMEM access per element
  uint32_t whist[kSWarps][kBins + 4];   // per-warp counts -> exclusive prefixes (bin 256 = invalid)
  uint32_t match[kSWarps][kBins + 4];   // per-warp lane masks of the current item's digit (kept zero)
  uint32_t blk_off[kBins];
  uint32_t gbase[kBins];
  uint32_t tile;
};

// kRanges (the last tile-digit pass): also derive the per-(eye, tile) ranges of the sorted pairs.
// In SMEM a digit's elements sit in input order, i.e. sorted by the full tile key (low digit sorted by
// the previous pass), so every run of one key inside the tile's digit segment is visible here; its
// first and last output positions go to ranges[key] by atomicMax of (~start, end) -- a key split
// across tiles keeps the smallest start and the largest end.  ranges is zeroed per frame
// (x = 0 decodes to an empty range).
template <bool kIota, bool kRanges>
__global__ void __launch_bounds__(kSThreads, 4)
onesweep_pass_kernel(const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
                     uint32_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out, uint2 *__restrict__ ranges,
                     const uint32_t *__restrict__ d_count, uint32_t shift, uint32_t dmask,
                     const uint32_t *__restrict__ hist,
                     uint32_t *__restrict__ status, uint32_t *__restrict__ status_clear,
                     uint32_t *__restrict__ tile_ctr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem &S = *reinterpret_cast<SortSmem *>(smem_raw);
  const uint32_t t = threadIdx.x, warp = t >> 5, lane = lane_id(), lt = lanemask_lt();
  const uint32_t n = *d_count;
  const uint32_t ntiles = (n + kSTile - 1) / kSTile;

  // exclusive scan of this pass's global digit histogram (every block, once)
  __shared__ uint32_t s_hex[kBins];
  {
    uint32_t h = hist[t];
    uint32_t inc = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= (uint32_t)o) inc += v;
    }
    __shared__ uint32_t s_w[kSWarps];
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint32_t wp = 0;
    for (uint32_t w = 0; w < warp; ++w) wp += s_w[w];
    s_hex[t] = wp + inc - h;
  }

  for (int k = t; k < kSWarps * (kBins + 4); k += kSThreads) (&S.match[0][0])[k] = 0;
  for (;;) {
    __syncthreads();
    if (t == 0) S.tile = atomicAdd(tile_ctr, 1u);
    for (int k = t; k < kSWarps * (kBins + 4); k += kSThreads) (&S.whist[0][0])[k] = 0;
    __syncthreads();
    const uint32_t tile = S.tile;
    if (tile >= ntiles) break;
    const uint32_t wbase = tile * kSTile + warp * (32 * kSItems);

    uint32_t key[kSItems], rank[kSItems];
#pragma unroll
    for (int i = 0; i < kSItems; ++i) {
      uint32_t idx = wbase + i * 32 + lane;
      key[i] = idx < n ? keys_in[idx] : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int i = 0; i < kSItems; ++i) {
      uint32_t idx = wbase + i * 32 + lane;
      uint32_t d = idx < n ? (key[i] >> shift) & dmask : (uint32_t)kBins;
      // peers = lanes holding the same digit: OR the lane bits into a per-digit shared word
      // (faster than match.any.sync here), then the lowest peer updates the count and clears it
      atomicOr(&S.match[warp][d], 1u << lane);
      __syncwarp();
      const uint32_t peers = S.match[warp][d];
      const uint32_t before = S.whist[warp][d];
      rank[i] = before + __popc(peers & lt);
      __syncwarp();
      if ((peers & lt) == 0) {
        S.whist[warp][d] = before + __popc(peers);
        S.match[warp][d] = 0;
      }
      __syncwarp();
    }
    __syncthreads();

    // per digit: exclusive prefix over warps, tile count, publish + look back
    {
      const uint32_t d = t;
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < kSWarps; ++w) {
        uint32_t c = S.whist[w][d];
        S.whist[w][d] = run;
        run += c;
      }
      uint32_t *st = status + (size_t)tile * kBins + d;
      uint32_t pre = 0;
      if (tile == 0) {
        st_volatile_u32(st, (2u << 30) | run);
      } else {
        st_volatile_u32(st, (1u << 30) | run);
        // look back 8 predecessor tiles per step with the 8 loads in flight together
        // (the inclusive frontier lags the aggregates in the first wave of tiles)
        int64_t p = (int64_t)tile - 1;
        bool found = false;
        while (!found) {
          uint32_t s[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            s[j] = (p - j >= 0) ? ld_volatile_u32(status + (size_t)(p - j) * kBins + d) : (2u << 30);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (found) break;
            while ((s[j] >> 30) == 0) s[j] = ld_volatile_u32(status + (size_t)(p - j) * kBins + d);
            pre += s[j] & 0x3FFFFFFFu;
            found = (s[j] >> 30) == 2u;
          }
          p -= 8;
        }
        st_volatile_u32(st, (2u << 30) | (pre + run));
      }
      status_clear[(size_t)tile * kBins + d] = 0u;
      S.gbase[d] = s_hex[d] + pre;
      // block-local exclusive scan of tile counts over digits
      uint32_t inc = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= (uint32_t)o) inc += v;
      }
      __shared__ uint32_t s_w2[kSWarps];
      if (lane == 31) s_w2[warp] = inc;
      __syncthreads();
      uint32_t wp = 0;
      for (uint32_t w = 0; w < warp; ++w) wp += s_w2[w];
      const uint32_t boff = wp + inc - run;
      S.blk_off[d] = boff;
      // fold the digit's block offset into the per-warp prefixes and its global base, so the scatter
      // and the write-out each read one digit-indexed word per element instead of two (the digit-
      // indexed SMEM reads are the bank-conflicted ones; the kernel is bound by the L1/SMEM pipe)
#pragma unroll 1
      for (int w = 0; w < kSWarps; ++w) S.whist[w][d] += boff;
      S.gbase[d] -= boff;
    }
    __syncthreads();

    // scatter into shared memory in (digit, original order)
#pragma unroll
    for (int i = 0; i < kSItems; ++i) {
      uint32_t idx = wbase + i * 32 + lane;
      if (idx < n) {
        uint32_t d = (key[i] >> shift) & dmask;
        uint32_t pos = S.whist[warp][d] + rank[i];
        GSC_CHECK(pos < (uint32_t)kSTile);
        S.kv[pos] = make_uint2(key[i], kIota ? idx : vals_in[idx]);
      }
    }
    __syncthreads();
    const uint32_t nvalid = min((uint32_t)kSTile, n - tile * kSTile);
    for (uint32_t i = t; i < nvalid; i += kSThreads) {
      const uint2 e = S.kv[i];
      const uint32_t k = e.x;
      uint32_t d = (k >> shift) & dmask;
      uint32_t o = S.gbase[d] + i;
      GSC_CHECK(o < n);
      keys_out[o] = k;
      vals_out[o] = e.y;
      if (kRanges) {
        constexpr uint32_t kM = 0x00FFFFFFu;   // tile key (bits 24..31: blend block mask)
        const uint32_t tk = k & kM;
        const bool first = i == 0 || (S.kv[i - 1].x & kM) != tk;
        const bool last = i + 1 == nvalid || (S.kv[i + 1].x & kM) != tk;
        if (first) atomicMax(&ranges[tk].x, ~o);
        if (last) atomicMax(&ranges[tk].y, o + 1);
      }
    }
  }
}

// ------------------------------------------------------------------ launchers
static PerDevice<int> g_sort_grid;

static int sort_setup(int num_sms) {
  return g_sort_grid.get([&](int &grid) {
    const int smem = (int)sizeof(SortSmem);
    cudaFuncSetAttribute(onesweep_pass_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(onesweep_pass_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(onesweep_pass_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, onesweep_pass_kernel<false, false>, kSThreads, smem);
    grid = num_sms * (per_sm > 0 ? per_sm : 1);
  });
}

// Sort `passes` (even) digits of `bits` bits each (shift 0, bits, 2 bits, ...; bits <= 8) of
// keys_a[0..*d_count) with payloads vals_a (iota payloads when `iota`).  Ping-pongs a -> b -> a;
// with an even pass count the result lands back in keys_a / vals_a.  `ranges` (optional): the last
// pass also derives the per-tile ranges of the sorted (tile) keys.
void launch_onesweep(uint32_t *keys_a, uint32_t *vals_a, uint32_t *keys_b, uint32_t *vals_b, bool iota,
                     const uint32_t *d_count, int passes, int bits, const uint32_t *hist /* [passes][256] */,
                     uint32_t *status_a, uint32_t *status_b, uint32_t *tile_ctrs, uint2 *ranges, int num_sms,
                     cudaStream_t st) {
  const int grid = sort_setup(num_sms);
  const int smem = (int)sizeof(SortSmem);
  const uint32_t dmask = (1u << bits) - 1u;
  for (int p = 0; p < passes; ++p) {
    const bool odd = p & 1;
    uint32_t *ki = odd ? keys_b : keys_a, *vi = odd ? vals_b : vals_a;
    uint32_t *ko = odd ? keys_a : keys_b, *vo = odd ? vals_a : vals_b;
    uint32_t *stc = odd ? status_b : status_a, *stx = odd ? status_a : status_b;
    const uint32_t shift = (uint32_t)(bits * p);
    if (p == 0 && iota)
      onesweep_pass_kernel<true, false><<<grid, kSThreads, smem, st>>>(
          ki, nullptr, ko, vo, nullptr, d_count, shift, dmask, hist + 256 * p, stc, stx, tile_ctrs + p);
    else if (p == passes - 1 && ranges)
      onesweep_pass_kernel<false, true><<<grid, kSThreads, smem, st>>>(
          ki, vi, ko, vo, ranges, d_count, shift, dmask, hist + 256 * p, stc, stx, tile_ctrs + p);
    else
      onesweep_pass_kernel<false, false><<<grid, kSThreads, smem, st>>>(
          ki, vi, ko, vo, nullptr, d_count, shift, dmask, hist + 256 * p, stc, stx, tile_ctrs + p);
  }
}

int sort_tile_size() { return kSTile; }

}  // namespace gsc
