// cull.cu -- SURVEY §8(a) rows a1 (frustum + LoD culling and cache classify)
// and a2 (depth policy + watermark).
//
// a1 (Alg. 1; readings R8/R9): for each anchor i,
//   visible_i = frustum(unified camera, margin m_i) and level_i <= l(d_i),
//   hit_i     = visible_i and birth_i > W_f          (watermark form of the
//               explicit eviction "invalidate lines at max reuse depth")
// with an ordered (ascending-id) compaction of X_f and of the miss list as
// reduce-then-scan over CTA tiles of 4096 anchors: cull_classify writes the
// frame's visibility bitset (also for |X_f \ X_f-1|), the miss bitset,
// birth_i = f for every miss (back-dated under GSC_F_STAGGER, R26) and
// per-tile counts; cull_compact expands the
// bitsets into the id lists at each tile's prefix.  (A single pass with a
// decoupled look-back spent ~30% of its stall samples waiting on it.)
//
// Layout: pos_m float4[N] = (x, y, z, m_i) -- one 16-byte coalesced load per
// anchor; level u8[N]; birth i32[N]; bitsets u32[ceil(N/32)] (visibility: ping-pong; misses).
// HBM bytes per anchor: 16 + 1 + 1/8 (+4 birth read per visible anchor -- the cache line is looked up
// only for visible anchors --, +4 per miss birth write, +4 per visible id, +4 per miss id).
#include "gsc_internal.cuh"

namespace gsc {

constexpr int kCullThreads = 512;
constexpr int kCullItems = 8;                                  // per thread
constexpr int kCullTile = kCullThreads * kCullItems;           // 4096 anchors

// (x, y) = (dot3(v, right), dot3(v, up)): the products as packed pairs (v_k broadcast, rp_k = (right_k,
// up_k)), the sums as scalar IEEE adds in dot3's order ((v0 b0 + v1 b1) + v2 b2).  Not add.rn.f32x2:
// ptxas fuses mul.rn.f32x2 -> add.rn.f32x2 into FFMA2 even under --fmad=false (checked in SASS), which
// would change the rounding; a scalar add.rn after a packed multiply is left alone.
__device__ __forceinline__ bool cull_visible(const UniC &u, f2p rp0, f2p rp1, f2p rp2, float4 pm, int level, int L,
                                             float d0) {
  float v0, v1;
  up2(add2(pk2(pm.x, pm.y), pk2(-u.p[0], -u.p[1])), v0, v1);   // fl(pm - p): adding -p is subtracting
  const float v2 = __fsub_rn(pm.z, u.p[2]);
  float p0x, p0y, p1x, p1y, p2x, p2y;
  up2(mul2(bc2(v0), rp0), p0x, p0y);
  up2(mul2(bc2(v1), rp1), p1x, p1y);
  up2(mul2(bc2(v2), rp2), p2x, p2y);
  const float x = __fadd_rn(__fadd_rn(p0x, p1x), p2x), y = __fadd_rn(__fadd_rn(p0y, p1y), p2y);
  const float z = dot3(v0, v1, v2, u.fwd);
  float m = pm.w;
  bool fr = (z >= __fsub_rn(u.near_plane, m)) && (z <= __fadd_rn(u.far_plane, m)) &&
            (__fsub_rn(fabsf(x), __fmul_rn(u.tx, z)) <= __fmul_rn(m, u.kx)) &&
            (__fsub_rn(fabsf(y), __fmul_rn(u.ty, z)) <= __fmul_rn(m, u.ky));
  if (!fr) return false;
  float s0, s1;
  up2(mul2(pk2(v0, v1), pk2(v0, v1)), s0, s1);
  float d2 = __fadd_rn(__fadd_rn(s0, s1), __fmul_rn(v2, v2));
  int lc;
  if (d2 == 0.0f) {
    lc = L - 1;
  } else {
    // e = ilogb(fl(d0 / fl(sqrt(d2)))) (R9, same op sequence as the oracle).  N9 fast path:
    // y = d0 * rsqrt.approx(d2) is within a few ulps of that quotient, so when y's mantissa is more
    // than 2^8 ulps away from both binade edges the exponent field of y is the exact e; only the
    // rest (and d2 outside the normal range of the approximation) takes the IEEE divide + sqrt.
    int e;
    const uint32_t yb = __float_as_uint(__fmul_rn(d0, rsqrtf(d2)));
    const uint32_t ym = yb & 0x7FFFFFu, yx = yb >> 23;
    if (d2 >= 1e-30f && d2 <= 1e30f && ym - 257u < 0x7FFFFFu - 513u && yx - 1u < 253u)
      e = (int)yx - 127;
    else
      e = ilogb_bits(__fdiv_rn(d0, __fsqrt_rn(d2)));
    // e in [-149, 127] or INT_MAX (inf / nan): clamp before the add (int arithmetic, no overflow)
    const int l = min(max(e, -1000), 1000) + (L - 1);
    lc = l < 0 ? 0 : (l > L - 1 ? L - 1 : l);
  }
  return level <= lc;
}

// Pass 1 (independent tiles): predicates, cache classify, birth update, the frame's visibility and
// miss bitsets, per-tile (visible, miss) counts -> agg[tile].  N < 2^31: 32-bit indices.
__global__ void __launch_bounds__(kCullThreads)
cull_classify_kernel(UniC u, int L, float d0, int N, const float4 *__restrict__ pos_m,
                     const uint8_t *__restrict__ level, int32_t *__restrict__ birth,
                     const uint32_t *__restrict__ prev_vis, uint32_t *__restrict__ cur_vis,
                     uint32_t *__restrict__ miss_bits, unsigned long long *__restrict__ agg,
                     FrameCounters *__restrict__ ctr, const PolicyState *__restrict__ pol) {
  __shared__ uint32_t s_wv[kCullThreads / 32], s_wm[kCullThreads / 32];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const uint32_t tile = blockIdx.x;
  const int32_t f = pol->frame, W = pol->W;
  const uint32_t n = (uint32_t)N;
  const uint32_t wbase = tile * kCullTile + warp * (32 * kCullItems);

  // all of the thread's anchor loads in flight before the first predicate (and the previous frame's
  // visibility words of the warp's 8 groups: lane k holds group k's)
  float4 pm[kCullItems];
  int lv[kCullItems];
#pragma unroll
  for (int it = 0; it < kCullItems; ++it) {
    const uint32_t i = wbase + it * 32 + lane;
    pm[it] = i < n ? pos_m[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    lv[it] = i < n ? level[i] : 0;
  }
  const uint32_t pw_lane =
      (lane < (uint32_t)kCullItems && wbase + lane * 32 < n) ? prev_vis[(wbase >> 5) + lane] : 0u;
  const f2p rp0 = pk2(u.right[0], u.up[0]), rp1 = pk2(u.right[1], u.up[1]), rp2 = pk2(u.right[2], u.up[2]);
  // predicates first; the cache lines (birth) are read for the visible anchors only, all in flight
  bool vis[kCullItems];
  int32_t bi[kCullItems];
#pragma unroll
  for (int it = 0; it < kCullItems; ++it) {
    const uint32_t i = wbase + it * 32 + lane;
    vis[it] = i < n && cull_visible(u, rp0, rp1, rp2, pm[it], lv[it], L, d0);
    bi[it] = vis[it] ? birth[i] : 0;
  }
  uint32_t cnt_v = 0, cnt_m = 0, cnt_new = 0;
#pragma unroll
  for (int it = 0; it < kCullItems; ++it) {
    const uint32_t i = wbase + it * 32 + lane;
    bool miss = false;
    if (vis[it]) {
      {
        miss = !(bi[it] > W);
        // derived this frame (Alg. 1 "update computation cache"); GSC_F_STAGGER (R26): a line filled
        // for the first time since the reset (birth INT32_MIN) is back-dated by min(i mod D, f-1-W)
        if (miss) {
          int32_t b = f;
          if (pol->stagger && bi[it] == INT32_MIN) {
            const int32_t s = (int32_t)((uint32_t)i % (uint32_t)pol->d_max), cap = f - 1 - W;
            b = f - (s < cap ? s : cap);
          }
          birth[i] = b;
        }
      }
    }
    const uint32_t mv = __ballot_sync(0xFFFFFFFFu, vis[it]);
    const uint32_t mm = __ballot_sync(0xFFFFFFFFu, miss);
    const uint32_t word = (wbase + it * 32) >> 5;
    const uint32_t pw = __shfl_sync(0xFFFFFFFFu, pw_lane, it);
    if (wbase + it * 32 < n) {
      if (lane == 0) { cur_vis[word] = mv; miss_bits[word] = mm; }
      cnt_new += __popc(mv & ~pw);
    }
    cnt_v += __popc(mv);
    cnt_m += __popc(mm);
  }
  if (lane == 0) { s_wv[warp] = cnt_v; s_wm[warp] = cnt_m; }
  if (lane == 0 && cnt_new) atomicAdd(&ctr->n_new, cnt_new);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tv = 0, tm = 0;
#pragma unroll
    for (int w = 0; w < kCullThreads / 32; ++w) { tv += s_wv[w]; tm += s_wm[w]; }
    agg[tile] = ((unsigned long long)tm << 31) | tv;
  }
}

__device__ __forceinline__ void policy_step(PolicyState *pol, const FrameCounters *ctr, FrameRecordDev *rec);

// Pass 2: ordered (ascending-id) compaction of X_f and of the miss list from the bitsets.  The
// tile's prefix is the sum of agg[< tile] (L2-resident, read by the whole CTA); warp w expands words
// [32 w, 32 w + 32) of the tile's 128 bitset words.
constexpr int kCompThreads = 128;
__global__ void __launch_bounds__(kCompThreads)
cull_compact_kernel(int N, const uint32_t *__restrict__ cur_vis, const uint32_t *__restrict__ miss_bits,
                    const unsigned long long *__restrict__ agg, uint32_t *__restrict__ visible,
                    uint32_t *__restrict__ misses, FrameCounters *__restrict__ ctr, PolicyState *__restrict__ pol,
                    FrameRecordDev *__restrict__ rec) {
  __shared__ unsigned long long s_red[kCompThreads / 32];
  __shared__ uint32_t s_wv[kCompThreads / 32], s_wm[kCompThreads / 32];
  const uint32_t t = threadIdx.x, warp = t >> 5, lane = lane_id(), lt = lanemask_lt();
  const uint32_t tile = blockIdx.x;
  const uint32_t nwords = (uint32_t)((N + 31) / 32);
  unsigned long long pre = 0;
  for (uint32_t j = t; j < tile; j += kCompThreads) pre += agg[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xFFFFFFFFu, pre, o);
  const uint32_t word = tile * (kCullTile / 32) + t;
  const uint32_t mv = word < nwords ? cur_vis[word] : 0u, mm = word < nwords ? miss_bits[word] : 0u;
  // warp-inclusive scans of the word counts
  uint32_t iv = __popc(mv), im = __popc(mm);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t a = __shfl_up_sync(0xFFFFFFFFu, iv, o), b = __shfl_up_sync(0xFFFFFFFFu, im, o);
    if (lane >= (uint32_t)o) { iv += a; im += b; }
  }
  if (lane == 31) { s_wv[warp] = iv; s_wm[warp] = im; }
  if (lane == 0) s_red[warp] = pre;
  __syncthreads();
  unsigned long long tpre = 0;
  uint32_t ov = 0, om = 0, tv = 0, tm = 0;
#pragma unroll
  for (int w = 0; w < kCompThreads / 32; ++w) {
    tpre += s_red[w];
    ov += (uint32_t)w < warp ? s_wv[w] : 0u;
    om += (uint32_t)w < warp ? s_wm[w] : 0u;
    tv += s_wv[w];
    tm += s_wm[w];
  }
  ov += (uint32_t)(tpre & 0x7FFFFFFFull);
  om += (uint32_t)((tpre >> 31) & 0x7FFFFFFFull);
  const uint32_t ntiles = (uint32_t)((N + kCullTile - 1) / kCullTile);
  if (t == 0 && tile == ntiles - 1) {   // totals, then a2 (n_new is final: pass 1 has completed)
    ctr->n_visible = (uint32_t)(tpre & 0x7FFFFFFFull) + tv;
    ctr->n_miss = (uint32_t)((tpre >> 31) & 0x7FFFFFFFull) + tm;
    policy_step(pol, ctr, rec);
  }
  // exclusive offsets of this lane's word; then the warp expands its 32 words one by one
  uint32_t ev = ov + iv - __popc(mv), em = om + im - __popc(mm);
  const uint32_t wbase = tile * kCullTile + warp * 1024;
  for (int j = 0; j < 32; ++j) {
    const uint32_t v = __shfl_sync(0xFFFFFFFFu, mv, j), m = __shfl_sync(0xFFFFFFFFu, mm, j);
    const uint32_t bv = __shfl_sync(0xFFFFFFFFu, ev, j), bm = __shfl_sync(0xFFFFFFFFu, em, j);
    const uint32_t i = wbase + 32 * j + lane;
    if (v >> lane & 1u) visible[bv + __popc(v & lt)] = i;
    if (m >> lane & 1u) misses[bm + __popc(m & lt)] = i;
  }
}

// a2: depth_{f+1} = H(rate), W_{f+1} = max(W_f, f+1 - depth_{f+1}) (Eq. 4; R10).
// H(num/den) = 1 + floor((2 (D-1)(den - num) + den) / (2 den)); frame 0 keeps D_max.
__device__ __forceinline__ void policy_step(PolicyState *pol, const FrameCounters *ctr, FrameRecordDev *rec) {
  const int32_t f = pol->frame, D = pol->d_max;
  const int32_t depth_used = pol->depth;
  const long long den = ctr->n_visible;
  const long long num = pol->literal ? (long long)ctr->n_miss : (long long)ctr->n_new;
  int32_t depth_next = depth_used;
  if (f > 0) {
    if (den <= 0) {
      depth_next = D;
    } else if (pol->guide == 1) {           // exponential: halve the depth per quarter of the rate (R23)
      const int32_t d = D >> (int32_t)((4LL * num) / den);
      depth_next = d < 1 ? 1 : d;
    } else if (pol->guide == 2) {           // staged: thresholds 1/10, 1/4, 1/2 (R23)
      depth_next = 10LL * num < den ? D : 4LL * num < den ? (D + 1) / 2 : 2LL * num < den ? (D + 3) / 4 : 1;
    } else {                                // linear: clamp(1 + round_half_away((D-1)(1-rate)), 1, D)
      depth_next = 1 + (int32_t)((2LL * (D - 1) * (den - num) + den) / (2LL * den));
    }
  }
  pol->depth = depth_next;
  const int32_t wn = (f + 1) - depth_next;
  pol->W = pol->W > wn ? pol->W : wn;
  pol->frame = f + 1;
  rec->frame = f;
  rec->depth_used = depth_used;
  rec->depth_next = depth_next;
  rec->n_visible = ctr->n_visible;
  rec->n_miss = ctr->n_miss;
  rec->n_new = ctr->n_new;
}
// (N = 0 only: otherwise the last cull_compact CTA runs the policy step)
__global__ void policy_kernel(PolicyState *pol, const FrameCounters *ctr, FrameRecordDev *rec) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  policy_step(pol, ctr, rec);
}

// final per-frame counts for the host record
__global__ void record_kernel(const FrameCounters *ctr, FrameRecordDev *rec) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  rec->n_splat = ctr->n_splat;
  rec->n_pairs_raw = ctr->n_pairs_raw;
  rec->overflow = ctr->overflow | ctr->list_overflow;
  rec->n_nonfinite = ctr->n_nonfinite;
  rec->n_fixup = ctr->n_fixup;
  rec->n_evals = ctr->n_evals;
  rec->n_exp = ctr->n_exp;
  rec->n_evals_list = ctr->n_evals_list;
}

// load-time: m_i = max_j |O_ij (.) s_i|_2 + 3.33 max_k s_ik  (R8), packed with pos
__global__ void margin_kernel(int N, const float *__restrict__ pos, const float *__restrict__ offs,
                              const float *__restrict__ scale, float4 *__restrict__ pos_m) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  float s0 = scale[3 * i], s1 = scale[3 * i + 1], s2 = scale[3 * i + 2];
  float mo = 0.0f;
  for (int j = 0; j < kK; ++j) {
    const float *o = offs + (size_t)i * kK * 3 + 3 * j;
    float a = __fmul_rn(o[0], s0), b = __fmul_rn(o[1], s1), c = __fmul_rn(o[2], s2);
    float nj = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(a, a), __fmul_rn(b, b)), __fmul_rn(c, c)));
    if (nj > mo) mo = nj;
  }
  float smax = s0;
  if (s1 > smax) smax = s1;
  if (s2 > smax) smax = s2;
  pos_m[i] = make_float4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], __fadd_rn(mo, __fmul_rn(3.33f, smax)));
}

// ---------------------------------------------------------------- launchers
// a1 + a2
void launch_cull(const FrameC &fc, int N, const float4 *pos_m, const uint8_t *level, int32_t *birth,
                 const uint32_t *prev_vis, uint32_t *cur_vis, uint32_t *miss_bits, uint32_t *visible,
                 uint32_t *misses, unsigned long long *agg, FrameCounters *ctr, PolicyState *pol,
                 FrameRecordDev *rec, cudaStream_t st) {
  int tiles = (N + kCullTile - 1) / kCullTile;
  if (tiles == 0) {
    policy_kernel<<<1, 32, 0, st>>>(pol, ctr, rec);
    return;
  }
  cull_classify_kernel<<<tiles, kCullThreads, 0, st>>>(fc.u, fc.L, fc.d0, N, pos_m, level, birth, prev_vis,
                                                        cur_vis, miss_bits, agg, ctr, pol);
  cull_compact_kernel<<<tiles, kCompThreads, 0, st>>>(N, cur_vis, miss_bits, agg, visible, misses, ctr, pol, rec);
}
void launch_record(const FrameCounters *ctr, FrameRecordDev *rec, cudaStream_t st) {
  record_kernel<<<1, 32, 0, st>>>(ctr, rec);
}
void launch_margin(int N, const float *pos, const float *offs, const float *scale, float4 *pos_m, cudaStream_t st) {
  if (N > 0) margin_kernel<<<(N + 255) / 256, 256, 0, st>>>(N, pos, offs, scale, pos_m);
}
int cull_tiles(int N) { return (N + kCullTile - 1) / kCullTile; }

}  // namespace gsc
