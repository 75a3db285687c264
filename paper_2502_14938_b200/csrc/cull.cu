// cull.cu -- SURVEY §8(a) rows a1 (frustum + LoD culling and cache classify)
// and a2 (depth policy + watermark).
//
// a1 (Alg. 1; readings R8/R9): for each anchor i,
//   visible_i = frustum(unified camera, margin m_i) and level_i <= l(d_i),
//   hit_i     = visible_i and birth_i > W_f          (watermark form of the
//               explicit eviction "invalidate lines at max reuse depth")
// with an ordered (ascending-id) compaction of X_f and of the miss list by a
// single-pass decoupled look-back scan, the visibility bitset of the frame
// (for |X_f \ X_f-1|) and birth_i = f written for every miss.
//
// Layout: pos_m float4[N] = (x, y, z, m_i) -- one 16-byte coalesced load per
// anchor; level u8[N]; birth i32[N]; bitset u32[ceil(N/32)] (ping-pong).
// HBM bytes per anchor: 16 + 1 + 4 + 1/8 (+4 per miss birth write, +4 per
// visible id, +4 per miss id).
#include "gsc_internal.cuh"

namespace gsc {

constexpr int kCullThreads = 256;
constexpr int kCullItems = 4;                                  // per thread
constexpr int kCullTile = kCullThreads * kCullItems;           // 1024 anchors

__device__ __forceinline__ bool cull_visible(const UniC &u, float4 pm, int level, int L, float d0) {
  float v0 = __fsub_rn(pm.x, u.p[0]), v1 = __fsub_rn(pm.y, u.p[1]), v2 = __fsub_rn(pm.z, u.p[2]);
  float x = dot3(v0, v1, v2, u.right), y = dot3(v0, v1, v2, u.up), z = dot3(v0, v1, v2, u.fwd);
  float m = pm.w;
  bool fr = (z >= __fsub_rn(u.near_plane, m)) && (z <= __fadd_rn(u.far_plane, m)) &&
            (__fsub_rn(fabsf(x), __fmul_rn(u.tx, z)) <= __fmul_rn(m, u.kx)) &&
            (__fsub_rn(fabsf(y), __fmul_rn(u.ty, z)) <= __fmul_rn(m, u.ky));
  if (!fr) return false;
  float d2 = __fadd_rn(__fadd_rn(__fmul_rn(v0, v0), __fmul_rn(v1, v1)), __fmul_rn(v2, v2));
  int lc;
  if (d2 == 0.0f) {
    lc = L - 1;
  } else {
    int e = ilogb_bits(__fdiv_rn(d0, __fsqrt_rn(d2)));
    long long l = (long long)e + (L - 1);
    lc = (int)(l < 0 ? 0 : (l > L - 1 ? L - 1 : l));
  }
  return level <= lc;
}

__global__ void __launch_bounds__(kCullThreads)
cull_classify_kernel(UniC u, int L, float d0, int N, const float4 *__restrict__ pos_m,
                     const uint8_t *__restrict__ level, int32_t *__restrict__ birth,
                     const uint32_t *__restrict__ prev_vis, uint32_t *__restrict__ cur_vis,
                     uint32_t *__restrict__ visible, uint32_t *__restrict__ misses,
                     unsigned long long *__restrict__ status, FrameCounters *__restrict__ ctr,
                     const PolicyState *__restrict__ pol) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_wv[kCullThreads / 32], s_wm[kCullThreads / 32];
  __shared__ unsigned long long s_prefix;
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->tile_cull, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int32_t f = pol->frame, W = pol->W;
  const int64_t wbase = (int64_t)tile * kCullTile + warp * (32 * kCullItems);

  uint32_t mv[kCullItems], mm[kCullItems];
  uint32_t cnt_v = 0, cnt_m = 0, cnt_new = 0;
#pragma unroll
  for (int it = 0; it < kCullItems; ++it) {
    int64_t i = wbase + it * 32 + lane;
    bool vis = false, miss = false;
    if (i < N) {
      float4 pm = pos_m[i];
      vis = cull_visible(u, pm, level[i], L, d0);
      if (vis) {
        int32_t b = birth[i];
        miss = !(b > W);
        if (miss) birth[i] = f;   // derived this frame (Alg. 1 "update computation cache")
      }
    }
    mv[it] = __ballot_sync(0xFFFFFFFFu, vis);
    mm[it] = __ballot_sync(0xFFFFFFFFu, miss);
    int64_t word = (wbase + it * 32) >> 5;
    if (wbase + it * 32 < N) {
      uint32_t pw = prev_vis[word];
      if (lane == 0) cur_vis[word] = mv[it];
      cnt_new += __popc(mv[it] & ~pw);
    }
    cnt_v += __popc(mv[it]);
    cnt_m += __popc(mm[it]);
  }
  if (lane == 0) { s_wv[warp] = cnt_v; s_wm[warp] = cnt_m; }
  if (lane == 0 && cnt_new) atomicAdd(&ctr->n_new, cnt_new);
  __syncthreads();

  // block aggregate and exclusive warp prefixes (warp 0)
  if (warp == 0) {
    uint32_t v = lane < kCullThreads / 32 ? s_wv[lane] : 0, m = lane < kCullThreads / 32 ? s_wm[lane] : 0;
    uint32_t iv = v, im = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t tv = __shfl_up_sync(0xFFFFFFFFu, iv, o), tm = __shfl_up_sync(0xFFFFFFFFu, im, o);
      if (lane >= (uint32_t)o) { iv += tv; im += tm; }
    }
    uint32_t tot_v = __shfl_sync(0xFFFFFFFFu, iv, 31), tot_m = __shfl_sync(0xFFFFFFFFu, im, 31);
    if (lane < kCullThreads / 32) { s_wv[lane] = iv - v; s_wm[lane] = im - m; }
    unsigned long long agg = ((unsigned long long)tot_m << 31) | tot_v;
    if (tile == 0) {
      if (lane == 0) st_volatile_u64(status, (2ull << 62) | agg);
      if (lane == 0) s_prefix = 0;
    } else {
      if (lane == 0) st_volatile_u64(status + tile, (1ull << 62) | agg);
      unsigned long long pre = lookback_u64(status, tile);
      if (lane == 0) {
        st_volatile_u64(status + tile, (2ull << 62) | (pre + agg));
        s_prefix = pre;
      }
    }
    uint32_t ntiles = (uint32_t)((N + kCullTile - 1) / kCullTile);
    if (lane == 0 && tile == ntiles - 1) {
      unsigned long long pre = (tile == 0) ? 0ull : s_prefix;
      unsigned long long tot = pre + agg;
      ctr->n_visible = (uint32_t)(tot & 0x7FFFFFFFull);
      ctr->n_miss = (uint32_t)((tot >> 31) & 0x7FFFFFFFull);
    }
  }
  __syncthreads();
  const unsigned long long pre = s_prefix;
  uint32_t ov = (uint32_t)(pre & 0x7FFFFFFFull) + s_wv[warp];
  uint32_t om = (uint32_t)((pre >> 31) & 0x7FFFFFFFull) + s_wm[warp];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int it = 0; it < kCullItems; ++it) {
    uint32_t i = (uint32_t)(wbase + it * 32 + lane);
    if (mv[it] >> lane & 1u) visible[ov + __popc(mv[it] & lt)] = i;
    if (mm[it] >> lane & 1u) misses[om + __popc(mm[it] & lt)] = i;
    ov += __popc(mv[it]);
    om += __popc(mm[it]);
  }
}

// a2: depth_{f+1} = H(rate), W_{f+1} = max(W_f, f+1 - depth_{f+1}) (Eq. 4; R10).
// H(num/den) = 1 + floor((2 (D-1)(den - num) + den) / (2 den)); frame 0 keeps D_max.
__global__ void policy_kernel(PolicyState *pol, const FrameCounters *ctr, FrameRecordDev *rec) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
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

// final per-frame counts for the host record
__global__ void record_kernel(const FrameCounters *ctr, FrameRecordDev *rec) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  rec->n_splat = ctr->n_splat;
  rec->n_pairs_raw = ctr->n_pairs_raw;
  rec->overflow = ctr->overflow;
  rec->n_evals = ctr->n_evals;
  rec->n_exp = ctr->n_exp;
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
void launch_cull(const FrameC &fc, int N, const float4 *pos_m, const uint8_t *level, int32_t *birth,
                 const uint32_t *prev_vis, uint32_t *cur_vis, uint32_t *visible, uint32_t *misses,
                 unsigned long long *status, FrameCounters *ctr, const PolicyState *pol, cudaStream_t st) {
  int tiles = (N + kCullTile - 1) / kCullTile;
  if (tiles == 0) return;
  cull_classify_kernel<<<tiles, kCullThreads, 0, st>>>(fc.u, fc.L, fc.d0, N, pos_m, level, birth, prev_vis,
                                                        cur_vis, visible, misses, status, ctr, pol);
}
void launch_policy(PolicyState *pol, const FrameCounters *ctr, FrameRecordDev *rec, cudaStream_t st) {
  policy_kernel<<<1, 32, 0, st>>>(pol, ctr, rec);
}
void launch_record(const FrameCounters *ctr, FrameRecordDev *rec, cudaStream_t st) {
  record_kernel<<<1, 32, 0, st>>>(ctr, rec);
}
void launch_margin(int N, const float *pos, const float *offs, const float *scale, float4 *pos_m, cudaStream_t st) {
  if (N > 0) margin_kernel<<<(N + 255) / 256, 256, 0, st>>>(N, pos, offs, scale, pos_m);
}
int cull_tiles(int N) { return (N + kCullTile - 1) / kCullTile; }

}  // namespace gsc
