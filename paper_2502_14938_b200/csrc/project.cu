// project.cu -- SURVEY §8(a) row a4: EWA projection,
// opacity-aware extent r^2 = 2 ln(255 alpha) ("considering the opacity
// can scale down the size of the ellipse") and the exact
// tile-coverage count (FlashGS citation), both eyes batched
// ("independently or in batching"; R19).
//
// Three kernels.  live_mark_kernel + live_kernel compact the LIVE visible
// slots s = v*K + j (255 alpha > 1; Gaussian g = X_f[v]*K + j) into live_g,
// in s order (hence ascending g), as reduce-then-scan over 4096-slot tiles
// (a live bitset and per-tile counts, then the expansion at each tile's prefix).
// project_kernel then projects live item i for eye e in lane (i, e) -- every
// lane busy -- walks the kept tiles of the warp's 32 splats (exact row-form
// tile test, N7) into the kept-tile list with each pair's blend-block mask,
// and writes splat c = e * n_live + i: per eye, c ascends with g -- the order
// that makes the later stable sorts break depth ties by g like the oracle.
// Live splats that project nowhere keep an entry with an empty box (0 tiles).
// Fused: the 4 x 256-bin digit histogram of the depth keys (first pass of the
// onesweep depth sort).
#include "gsc_internal.cuh"

namespace gsc {

constexpr int kPThreads = 256;
constexpr int kLThreads = 256;
constexpr int kLRounds = 16;                      // 32-slot rounds per warp
constexpr int kLTile = kLThreads * kLRounds;      // 4096 slots per CTA tile

struct SplatOut {
  float u, v, A, B, C, thr;
  float r2s;               // 2 ln(255 alpha): the significance radius^2, whatever extent the tiles use
  float sxx, syy;          // 2D covariance diagonal (after the 0.3 floor)
  uint32_t box_x, box_y;   // tx0 | tx1 << 16 ; ty0 | ty1 << 16 | eye << 31
  uint32_t n;
  float depth;
};

// returns 1: projected (o filled); 0: culled; -1: skipped for non-finite parameters ("non-finite
// splat parameters -> skip splat, count in FrameRecord diagnostics"): a non-finite mean or covariance
// entry, or a non-finite 2D covariance / determinant / conic / centre of a Gaussian in the depth range.
template <int kAbl>
__device__ __forceinline__ int project_one(const EyeC &ec, int width, int height, int TW, int TH, float r2s,
                                           const float4 &p0, const float4 &p1, const float4 &p2, SplatOut &o) {
  // (the live test 255 alpha > 1 was made by live_kernel; r2s = 2 ln(255 alpha) is eye-independent)
  if (!isfinite(p0.x) || !isfinite(p0.y) || !isfinite(p0.z) || !isfinite(p0.w) || !isfinite(p1.x) ||
      !isfinite(p1.y) || !isfinite(p1.z) || !isfinite(p1.w) || !isfinite(p2.x))
    return -1;
  float t0 = __fsub_rn(p0.x, ec.p[0]), t1 = __fsub_rn(p0.y, ec.p[1]), t2 = __fsub_rn(p0.z, ec.p[2]);
  float x = dot3(t0, t1, t2, ec.r0), y = dot3(t0, t1, t2, ec.r1), z = dot3(t0, t1, t2, ec.r2);
  if (!(z > ec.near_plane) || z > ec.far_plane) return 0;
  // N8: one reciprocal of z (and of det below), rounded once, multiplied in
  const float iz = __fdiv_rn(1.0f, z), iz2 = __fmul_rn(iz, iz);
  float xz = __fmul_rn(x, iz), yz = __fmul_rn(y, iz);
  float xc = __fmul_rn(fminf(fmaxf(xz, -ec.limx), ec.limx), z);
  float yc = __fmul_rn(fminf(fmaxf(yz, -ec.limy), ec.limy), z);
  float J00 = __fmul_rn(ec.fx, iz), J02 = __fmul_rn(-__fmul_rn(ec.fx, xc), iz2);
  float J11 = __fmul_rn(ec.fy, iz), J12 = __fmul_rn(-__fmul_rn(ec.fy, yc), iz2);
  float T[2][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T[0][k] = __fadd_rn(__fmul_rn(J00, ec.r0[k]), __fmul_rn(J02, ec.r2[k]));
    T[1][k] = __fadd_rn(__fmul_rn(J11, ec.r1[k]), __fmul_rn(J12, ec.r2[k]));
  }
  // Sigma (00 01 02 11 12 22) = (p0.w, p1.x, p1.y, p1.z, p1.w, p2.x)
  const float S[3][3] = {{p0.w, p1.x, p1.y}, {p1.x, p1.z, p1.w}, {p1.y, p1.w, p2.x}};
  float U[2][3];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      U[r][k] = __fadd_rn(__fadd_rn(__fmul_rn(T[r][0], S[0][k]), __fmul_rn(T[r][1], S[1][k])),
                          __fmul_rn(T[r][2], S[2][k]));
  float a = dot3(U[0][0], U[0][1], U[0][2], T[0]);
  float b = dot3(U[0][0], U[0][1], U[0][2], T[1]);
  float c = dot3(U[1][0], U[1][1], U[1][2], T[1]);
  a = __fadd_rn(a, 0.3f);
  c = __fadd_rn(c, 0.3f);
  float det = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, b));
  if (!isfinite(det)) return -1;
  if (!(det > 0.0f)) return 0;
  o.sxx = a;
  o.syy = c;
  const float idet = __fdiv_rn(1.0f, det);
  o.A = __fmul_rn(c, idet);
  o.B = __fmul_rn(-b, idet);
  o.C = __fmul_rn(a, idet);
  o.u = __fadd_rn(__fmul_rn(ec.fx, xz), ec.cx);
  o.v = __fadd_rn(__fmul_rn(ec.fy, yz), ec.cy);
  float r2 = r2s;
  o.r2s = r2s;
  if (kAbl & kAblFixedExtent) r2 = 9.0f;   // ablation (GSC_F_ABL_FIXED_EXTENT): fixed 3 sigma
  o.thr = __fadd_rn(__fmul_rn(r2, kKappa), kSlack);
  o.depth = z;
  if (!isfinite(o.A) || !isfinite(o.B) || !isfinite(o.C) || !isfinite(o.u) || !isfinite(o.v) || !isfinite(o.thr))
    return -1;
  float ex = __fadd_rn(__fsqrt_rn(__fmul_rn(o.thr, a)), 1.0f), ey = __fadd_rn(__fsqrt_rn(__fmul_rn(o.thr, c)), 1.0f);
  float fx0 = fmaxf(floorf(__fmul_rn(__fsub_rn(o.u, ex), 0.0625f)), 0.0f);
  float fx1 = fminf(floorf(__fmul_rn(__fadd_rn(o.u, ex), 0.0625f)), (float)(TW - 1));
  float fy0 = fmaxf(floorf(__fmul_rn(__fsub_rn(o.v, ey), 0.0625f)), 0.0f);
  float fy1 = fminf(floorf(__fmul_rn(__fadd_rn(o.v, ey), 0.0625f)), (float)(TH - 1));
  if (fx0 > fx1 || fy0 > fy1) return 0;
  int tx0 = (int)fx0, tx1 = (int)fx1, ty0 = (int)fy0, ty1 = (int)fy1;
  o.n = 0;   // kept tiles: counted by the warp-flattened walk
  o.box_x = (uint32_t)tx0 | ((uint32_t)tx1 << 16);
  o.box_y = (uint32_t)ty0 | ((uint32_t)ty1 << 16);
  return 1;
}

// Pass 1 (independent tiles of 4096 slots): live bitset of the visible slots + per-tile live counts.
__global__ void __launch_bounds__(kLThreads)
live_mark_kernel(const uint32_t *__restrict__ visible, const float *__restrict__ alpha,
                 uint32_t *__restrict__ live_bits, uint32_t *__restrict__ agg, const FrameCounters *__restrict__ ctr) {
  __shared__ uint32_t s_cnt[kLThreads / 32];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const uint32_t S = ctr->n_visible * (uint32_t)kK;
  const uint32_t ntiles = (S + kLTile - 1) / kLTile;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t s0 = tile * kLTile + warp * (32 * kLRounds) + lane;
    float al[kLRounds];
#pragma unroll
    for (int r = 0; r < kLRounds; ++r) {   // all of the thread's loads in flight before the ballots
      const uint32_t s = s0 + 32 * r;
      al[r] = 0.0f;
      if (s < S) {
        const uint32_t v = s / kK, j = s - v * kK;
        al[r] = alpha[visible[v] * kK + j];
      }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int r = 0; r < kLRounds; ++r) {
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, __fmul_rn(255.0f, al[r]) > 1.0f);
      const uint32_t w = (s0 - lane) / 32 + r;
      if (lane == 0 && 32 * w < S) live_bits[w] = m;
      cnt += __popc(m);
    }
    if (lane == 0) s_cnt[warp] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
#pragma unroll
      for (int w = 0; w < kLThreads / 32; ++w) t += s_cnt[w];
      agg[tile] = t;
    }
    __syncthreads();
  }
}

// Pass 2: ordered compaction of the live slots s (hence ascending g) from the bitset at each tile's
// prefix (sum of the earlier tiles' counts, L2-resident); the last tile sets n_splat = 2 x live.
// (A single pass with a CTA-wide decoupled look-back spent most of its stall samples in the look-back.)
__global__ void __launch_bounds__(kLThreads)
live_kernel(const uint32_t *__restrict__ visible, const uint32_t *__restrict__ live_bits,
            const uint32_t *__restrict__ agg, uint32_t *__restrict__ live_g, FrameCounters *__restrict__ ctr) {
  __shared__ uint32_t s_pre[kLThreads / 32], s_cnt[kLThreads / 32];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id(), lt = lanemask_lt();
  const uint32_t S = ctr->n_visible * (uint32_t)kK;
  const uint32_t ntiles = (S + kLTile - 1) / kLTile;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    uint32_t pre = 0;
    for (uint32_t j = threadIdx.x; j < tile; j += kLThreads) pre += agg[j];
    pre = __reduce_add_sync(0xFFFFFFFFu, pre);
    // warp w: words [16 w, 16 w + 16) of the tile (lane r < 16 holds word r)
    const uint32_t w0 = tile * (kLTile / 32) + warp * kLRounds;
    const uint32_t m = (lane < (uint32_t)kLRounds && 32 * (w0 + lane) < S) ? live_bits[w0 + lane] : 0u;
    const uint32_t c = __popc(m);
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= (uint32_t)o) inc += t;
    }
    if (lane == 31) s_cnt[warp] = inc;
    if (lane == 0) s_pre[warp] = pre;
    __syncthreads();
    uint32_t tpre = 0, wex = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kLThreads / 32; ++w) {
      tpre += s_pre[w];
      wex += (uint32_t)w < warp ? s_cnt[w] : 0u;
      tot += s_cnt[w];
    }
    if (threadIdx.x == 0 && tile == ntiles - 1) ctr->n_splat = 2 * (tpre + tot);
    const uint32_t ex = tpre + wex + inc - c;   // this lane's word's first output position
#pragma unroll
    for (int r = 0; r < kLRounds; ++r) {
      const uint32_t mr = __shfl_sync(0xFFFFFFFFu, m, r), br = __shfl_sync(0xFFFFFFFFu, ex, r);
      if ((mr >> lane) & 1u) {
        const uint32_t s = 32 * (w0 + r) + lane, v = s / kK, j = s - v * kK;
        live_g[br + __popc(mr & lt)] = visible[v] * kK + j;
      }
    }
    __syncthreads();   // s_pre / s_cnt reuse
  }
}

// ---- row form of the exact tile test (R14 / N7)
// Per-splat constants of the row walk.
struct RowSplat {
  float u, v, B, det, ey, bs, at, invA, xr_ext, xl_ext;
  int gx0, gx1, gy0, gy1;   // blend blocks (8x4 px, image-global) the splat's skip box meets
  int tx0, tx1, ty0;
  uint32_t kb;              // key base of the eye (eye * T_e)
};

__device__ __forceinline__ RowSplat row_splat(const SplatOut &o, float rx, float ry, uint32_t kb) {
  RowSplat r;
  const float det = __fsub_rn(__fmul_rn(o.A, o.C), __fmul_rn(o.B, o.B));
  const float bs = __fmul_rn(o.B, __fsqrt_rn(__fdiv_rn(o.thr, __fmul_rn(det, o.C))));
  const float at = __fmul_rn(o.A, o.thr), invA = __fdiv_rn(1.0f, o.A);
  r.u = o.u; r.v = o.v; r.B = o.B; r.det = det; r.at = at; r.invA = invA; r.bs = bs;
  r.ey = __fsqrt_rn(__fmul_rn(o.thr, __fdiv_rn(o.A, det)));
  // the rows' x-extremes when no clamp is active (dyr = -bs, dyl = bs), same expression as row_interval
  const float D = fmaxf(__fsub_rn(at, __fmul_rn(det, __fmul_rn(bs, bs))), 0.0f);
  const float sD = __fsqrt_rn(D), Bb = __fmul_rn(o.B, bs);
  r.xr_ext = __fadd_rn(o.u, __fmul_rn(__fsub_rn(sD, __fmul_rn(o.B, -bs)), invA));
  r.xl_ext = __fsub_rn(o.u, __fmul_rn(__fadd_rn(sD, Bb), invA));
  // blend.cu's block test for the 8x4 block (bx, by): u + rx >= 8 bx + 0.5, u - rx <= 8 bx + 7.5,
  // v + ry >= 4 by + 0.5, v - ry <= 4 by + 3.5 (pixel centres).  Its solutions are the ranges
  // [gx0, gx1] x [gy0, gy1] below, exactly: as in row_cols, each subtraction is exact wherever the
  // rounding could matter (Sterbenz / ulp <= 0.5) and the scalings are by powers of two.
  const float ux0 = __fsub_rn(o.u, rx), ux1 = __fadd_rn(o.u, rx);
  const float vy0 = __fsub_rn(o.v, ry), vy1 = __fadd_rn(o.v, ry);
  r.gx1 = (int)fminf(floorf(__fmul_rn(__fsub_rn(ux1, 0.5f), 0.125f)), 65536.0f);
  r.gx0 = (int)fmaxf(ceilf(__fmul_rn(__fsub_rn(ux0, 7.5f), 0.125f)), -1.0f);
  r.gy1 = (int)fminf(floorf(__fmul_rn(__fsub_rn(vy1, 0.5f), 0.25f)), 65536.0f);
  r.gy0 = (int)fmaxf(ceilf(__fmul_rn(__fsub_rn(vy0, 3.5f), 0.25f)), -1.0f);
  r.tx0 = (int)(o.box_x & 0xFFFFu); r.tx1 = (int)(o.box_x >> 16);
  r.ty0 = (int)(o.box_y & 0xFFFFu);
  r.kb = kb;
  return r;
}

// the cooperative walk's shared copy of the 32 lanes' RowSplats (SoA)
struct WarpRows {
  float u[32], v[32], B[32], det[32], ey[32], bs[32], at[32], invA[32], xr_ext[32], xl_ext[32];
  int gx0[32], gx1[32], gy0[32], gy1[32], tx0[32], tx1[32], ty0[32];
  uint32_t kb[32], excl[32], cnt[32];
  __device__ __forceinline__ void put(int l, const RowSplat &r) {
    u[l] = r.u; v[l] = r.v; B[l] = r.B; det[l] = r.det; ey[l] = r.ey; bs[l] = r.bs; at[l] = r.at;
    invA[l] = r.invA; xr_ext[l] = r.xr_ext; xl_ext[l] = r.xl_ext; gx0[l] = r.gx0; gx1[l] = r.gx1;
    gy0[l] = r.gy0; gy1[l] = r.gy1; tx0[l] = r.tx0; tx1[l] = r.tx1; ty0[l] = r.ty0; kb[l] = r.kb;
  }
  __device__ __forceinline__ RowSplat get(int l) const {
    RowSplat r;
    r.u = u[l]; r.v = v[l]; r.B = B[l]; r.det = det[l]; r.ey = ey[l]; r.bs = bs[l]; r.at = at[l];
    r.invA = invA[l]; r.xr_ext = xr_ext[l]; r.xl_ext = xl_ext[l]; r.gx0 = gx0[l]; r.gx1 = gx1[l];
    r.gy0 = gy0[l]; r.gy1 = gy1[l]; r.tx0 = tx0[l]; r.tx1 = tx1[l]; r.ty0 = ty0[l]; r.kb = kb[l];
    return r;
  }
};

// x-interval [xl, xr] of the ellipse {q <= thr} over the pixel-centre rows of tile row ty.  When the
// band contains the extreme rows dy = -/+ B s (the usual case) the clamps are inactive and the per-row
// expression equals the per-splat xr_ext / xl_ext bit for bit.
__device__ __forceinline__ bool row_interval(const RowSplat &r, int ty, int height, float &xl, float &xr) {
  const int py1 = min(16 * ty + 15, height - 1);
  const float Y0 = __fadd_rn((float)(16 * ty), 0.5f), Y1 = __fadd_rn((float)py1, 0.5f);
  const float lo = fmaxf(__fsub_rn(Y0, r.v), -r.ey), hi = fminf(__fsub_rn(Y1, r.v), r.ey);
  if (!(lo <= hi)) return false;
  const float dyr = fminf(fmaxf(-r.bs, lo), hi), dyl = fminf(fmaxf(r.bs, lo), hi);
  xr = r.xr_ext;
  xl = r.xl_ext;
  if (dyr != -r.bs || dyl != r.bs) {
    const float Dr = fmaxf(__fsub_rn(r.at, __fmul_rn(r.det, __fmul_rn(dyr, dyr))), 0.0f);
    xr = __fadd_rn(r.u, __fmul_rn(__fsub_rn(__fsqrt_rn(Dr), __fmul_rn(r.B, dyr)), r.invA));
    const float Dl = fmaxf(__fsub_rn(r.at, __fmul_rn(r.det, __fmul_rn(dyl, dyl))), 0.0f);
    xl = __fsub_rn(r.u, __fmul_rn(__fadd_rn(__fsqrt_rn(Dl), __fmul_rn(r.B, dyl)), r.invA));
  }
  return true;
}

// kept columns [a, b] of row ty inside the candidate box [tx0, tx1]: X0(tx) <= xr and X1(tx) >= xl with
// X0 = 16 tx + 0.5, X1 = min(16 tx + 15, W - 1) + 0.5.  b = floor((xr - 0.5)/16) and
// a = ceil((xl - 15.5)/16) are exact: for xr >= 0.5 (xl >= 7.75) the subtraction is exact (Sterbenz /
// ulp <= 0.5) and the scaling by 2^-4 too; below that the predicate holds for no (every) column >= 0
// whatever the rounding.  Only the image's last column has a smaller X1: checked explicitly.
__device__ __forceinline__ void row_cols(float xl, float xr, int tx0, int tx1, int width, int &a, int &b) {
  const float fb = floorf(__fmul_rn(__fsub_rn(xr, 0.5f), 0.0625f));
  const float fa = ceilf(__fmul_rn(__fsub_rn(xl, 15.5f), 0.0625f));
  b = (int)fminf(fmaxf(fb, (float)tx0 - 1.0f), (float)tx1);
  a = (int)fminf(fmaxf(fa, (float)tx0), (float)tx1 + 1.0f);
  if (a <= b && __fadd_rn((float)min(16 * a + 15, width - 1), 0.5f) < xl) ++a;
}

// kept columns [a, b] of row ty as keys (bits 0..23: eye * T_e + ty TW + tx) with the blend block mask
// (bits 24..31): bit 2k + j <=> the splat's skip box (u -/+ rx, v -/+ ry) meets the pixel centres of
// the tile's 8x4 block at columns 8j.., rows 4k.. -- the fp32 test blend.cu would run (N5).
__device__ __forceinline__ void emit_row(const RowSplat &r, int ty, int a, int b, int TW, uint32_t *list,
                                         uint32_t list_cap, uint32_t pos) {
  const uint32_t key0 = r.kb + (uint32_t)(ty * TW);
  // block rows k = 0..3 of tile row ty that the box meets -> bit pairs 2k, 2k+1
  const int klo = max(r.gy0 - 4 * ty, 0), khi = min(r.gy1 - 4 * ty, 3);
  const uint32_t ym = khi >= klo ? (4u << (2 * khi)) - (1u << (2 * klo)) : 0u;
  // block columns j = 0, 1 of tile column tx: both for the interior columns of [a, b] (the box spans
  // them), so only the row's first and last column need the test
  auto colmask = [&](int tx) -> uint32_t {
    const uint32_t xm = (r.gx0 <= 2 * tx && 2 * tx <= r.gx1 ? 1u : 0u) |
                        (r.gx0 <= 2 * tx + 1 && 2 * tx + 1 <= r.gx1 ? 2u : 0u);
    return (ym & (xm * 0x55u)) << 24;
  };
  const uint32_t ma = colmask(a), mb = colmask(b), mi = ym << 24;
  const uint32_t n = (uint32_t)(b - a + 1), key = key0 + (uint32_t)a;
  if (pos + n <= list_cap && pos + n >= pos) {   // (else the overflow flag is already set)
    uint32_t *dst = list + pos;
    dst[0] = key | ma;
    if (n > 1) dst[n - 1] = (key + n - 1) | mb;
    // interior keys (key + t) | mi, t = 1 .. n - 2: 16-byte stores where aligned (a per-lane loop over a
    // row's keys diverges across the warp's rows, 1 .. 120 keys: 4 keys per iteration cuts it 4x)
    uint32_t t = 1;
    const uint32_t vi = (key + 1) | mi;          // (key + t) | mi = vi + t - 1: no carry into bit 24
#pragma unroll 1
    for (; t + 1 < n && ((pos + t) & 3u); ++t) dst[t] = vi + t - 1;
#pragma unroll 1
    for (; t + 4 < n; t += 4)
      *reinterpret_cast<uint4 *>(dst + t) = make_uint4(vi + t - 1, vi + t, vi + t + 1, vi + t + 2);
#pragma unroll 1
    for (; t + 1 < n; ++t) dst[t] = vi + t - 1;
  }
}

constexpr uint32_t kSmallRows = 3;   // boxes of <= 3 tile rows: walked by their own lane

// Kept tiles of the 32 lanes' splats.  The warp bump-allocates the sum of the candidate box areas (an
// upper bound) from the kept-tile list.  A splat whose box has <= kSmallRows rows is walked by its own
// lane (row by row) into its own area; the rest -- the heavy tail of near, large splats -- are walked
// cooperatively: their rows laid end to end, 32 rows per step (one per lane), kept keys packed.
template <bool aabb>
__device__ __forceinline__ uint32_t warp_rows_list(WarpRows &ws, bool has, const SplatOut &o, float rx, float ry,
                                                   uint32_t kb, int width, int height, int TW, uint32_t *list,
                                                   uint32_t list_cap, uint32_t *list_top, uint32_t *overflow,
                                                   uint32_t &list_off) {
  const uint32_t lane = lane_id();
  RowSplat r{};
  uint32_t nrows = 0, area = 0;
  if (has) {
    r = row_splat(o, rx, ry, kb);
    nrows = (uint32_t)((int)((o.box_y >> 16) & 0x7FFFu) - r.ty0 + 1);
    area = nrows * (uint32_t)(r.tx1 - r.tx0 + 1);
  }
  const bool small = has && nrows <= kSmallRows, big = has && !small;
  // exclusive scans: small areas (own regions), big rows (cooperative items); totals
  uint32_t s_inc = small ? area : 0u, b_rows = big ? nrows : 0u, b_area = big ? area : 0u;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t t1 = __shfl_up_sync(0xFFFFFFFFu, s_inc, off), t2 = __shfl_up_sync(0xFFFFFFFFu, b_rows, off);
    if (lane >= (uint32_t)off) { s_inc += t1; b_rows += t2; }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) b_area += __shfl_xor_sync(0xFFFFFFFFu, b_area, off);
  const uint32_t s_tot = __shfl_sync(0xFFFFFFFFu, s_inc, 31), b_tot_rows = __shfl_sync(0xFFFFFFFFu, b_rows, 31);
  uint32_t base = 0;
  if (lane == 0) {
    const uint32_t need = s_tot + b_area;
    base = atomicAdd(list_top, need);
    if (base + need > list_cap || base + need < base) atomicExch(overflow, 1u);
  }
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  uint32_t n = 0;
  if (small) {
    const uint32_t pos0 = base + s_inc - area;
    list_off = pos0;
    for (uint32_t k = 0; k < nrows; ++k) {
      const int ty = r.ty0 + (int)k;
      float xl, xr;
      int a = 0, b = -1;
      if (aabb) { a = r.tx0; b = r.tx1; }
      else if (row_interval(r, ty, height, xl, xr)) row_cols(xl, xr, r.tx0, r.tx1, width, a, b);
      if (b >= a) {
        emit_row(r, ty, a, b, TW, list, list_cap, pos0 + n);
        n += (uint32_t)(b - a + 1);
      }
    }
  }
  if (b_tot_rows) {   // warp-uniform
    const uint32_t nb = big ? nrows : 0u;
    ws.excl[lane] = b_rows - nb;
    ws.cnt[lane] = 0;
    if (big) ws.put(lane, r);
    __syncwarp();
    uint32_t run = base + s_tot;
    for (uint32_t w0 = 0; w0 < b_tot_rows; w0 += 32) {
      const uint32_t w = w0 + lane;
      int owner = 0, a = 0, b = -1, ty = 0;
      RowSplat q{};
      if (w < b_tot_rows) {
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
          if (ws.excl[lo + step] <= w) lo += step;
        owner = lo;
        q = ws.get(lo);
        ty = q.ty0 + (int)(w - ws.excl[lo]);
        float xl, xr;
        if (aabb) { a = q.tx0; b = q.tx1; }
        else if (row_interval(q, ty, height, xl, xr)) row_cols(xl, xr, q.tx0, q.tx1, width, a, b);
      }
      const uint32_t m = b >= a ? (uint32_t)(b - a + 1) : 0u;
      uint32_t ex = m;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, ex, off);
        if (lane >= (uint32_t)off) ex += t;
      }
      const uint32_t step_tot = __shfl_sync(0xFFFFFFFFu, ex, 31);
      if (m) {
        atomicAdd(&ws.cnt[owner], m);
        emit_row(q, ty, a, b, TW, list, list_cap, run + ex - m);
      }
      run += step_tot;
    }
    __syncwarp();
    const uint32_t nbig = big ? ws.cnt[lane] : 0u;
    uint32_t e2 = nbig;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, e2, off);
      if (lane >= (uint32_t)off) e2 += t;
    }
    if (big) {
      n = nbig;
      list_off = base + s_tot + e2 - nbig;
    }
    __syncwarp();
  }
  if (!has) list_off = base;
  return n;
}

// Live item i (32 consecutive per warp) -> both eyes' splat records, then the
// exact kept-tile walk of the warp's 32 splats per eye (rows of the candidate
// boxes walked as one list) -> kept count and the kept-tile list (row-major
// keys eye*T_e + ty*TW + tx).  No ordering constraint between warps: each warp
// bump-allocates its list space.
template <int kAbl>   // kAbl*: F1 ablations (compile-time, so the method's kernel carries no extra state)
__global__ void __launch_bounds__(kPThreads, 4)   // 64 registers: 4 CTAs / SM (measured better than 80 / 3)
project_kernel(FrameC fc, const uint32_t *__restrict__ live_g, const float *__restrict__ alpha,
               const float4 *__restrict__ pool, SplatBufs sb, FrameCounters *__restrict__ ctr) {
  __shared__ uint32_t s_hist[4][256];
  __shared__ WarpRows s_wr[kPThreads / 32];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  WarpRows &ws = s_wr[warp];
  for (int k = threadIdx.x; k < 4 * 256; k += kPThreads) (&s_hist[0][0])[k] = 0;
  __syncthreads();
  // (n_live and the warp's first item broadcast from lane 0: warp-uniform by construction, and visibly
  // so to the compiler, which then drops the convergence checks around the walk's warp collectives)
  const uint32_t n_live = __shfl_sync(0xFFFFFFFFu, ctr->n_splat / 2, 0);
  const uint32_t nw = (gridDim.x * kPThreads) >> 5;
  const uint32_t base0 = __shfl_sync(0xFFFFFFFFu, ((blockIdx.x * kPThreads) >> 5) * 16 + warp * 16, 0);
  uint32_t pairs_local = 0;
  // lane = (item, eye): 16 live Gaussians per warp step, lanes 2k / 2k+1 take Gaussian k's left / right
  // eye (half the per-thread state of a lane doing both eyes: more warps in flight)
  const uint32_t e = lane & 1u;
  const EyeC &ec = e ? fc.eye[1] : fc.eye[0];
  for (uint32_t base = base0; base < n_live; base += nw * 16) {
    const uint32_t i = base + (lane >> 1);
    const bool valid = i < n_live;
    SplatOut o;
    bool ok = false;
    int pr = 0;
    uint32_t g = 0;
    float al = 0.0f;
    float4 q2 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
      g = live_g[i];
      al = alpha[g];
      const float4 q0 = pool[3 * (size_t)g];
      const float4 q1 = pool[3 * (size_t)g + 1];
      q2 = pool[3 * (size_t)g + 2];
      const float r2s = __fmul_rn(2.0f, log_s(__fmul_rn(255.0f, al)));   // r^2 = 2 ln(alpha/eps)
      pr = (e == 1 && (kAbl & kAblMono)) ? 0   // GSC_F_MONO: the right eye is not rendered
           : project_one<kAbl>(ec, fc.width, fc.height, fc.TW, fc.TH, r2s, q0, q1, q2, o);
      ok = pr > 0;
    }
    {
      const uint32_t nf = __ballot_sync(0xFFFFFFFFu, pr < 0);
      if (nf && lane == 0) atomicAdd(&ctr->n_nonfinite, (uint32_t)__popc(nf));
    }
    // skip bound = -ln(255 alpha) - 2^-7: below it alpha exp(power) < 1/255 for sure; (rx, ry) =
    // conservative half-extents of {q <= -2 pmin} (AABB of that ellipse, padded): a pixel outside them
    // has power < pmin, so the blend may skip it without changing a decision
    float pmin = 0.0f, rx = 0.0f, ry = 0.0f;
    if (ok) {
      pmin = __fsub_rn(__fmul_rn(-0.5f, o.r2s), 0.0078125f);
      const float qmax = __fmul_rn(-2.0f, pmin);
      rx = __fadd_rn(__fmul_rn(__fsqrt_rn(__fmul_rn(qmax, o.sxx)), 1.001f), 0.01f);
      ry = __fadd_rn(__fmul_rn(__fsqrt_rn(__fmul_rn(qmax, o.syy)), 1.001f), 0.01f);
    }
    uint32_t loff = 0;
    const uint32_t n = warp_rows_list<(kAbl & kAblAabbTiles) != 0>(ws, ok, o, rx, ry, e ? (uint32_t)fc.Te : 0u,
                                                                  fc.width, fc.height, fc.TW, sb.list, sb.list_cap,
                                                                  &ctr->list_top, &ctr->list_overflow, loff);
    if (!valid) continue;
    const uint32_t c = e * n_live + i;
    uint32_t dk = 0xFFFFFFFFu;      // a dead entry sorts last and owns no tile
    if (ok) {
      // blend-ready record (N6): (u, v, -A/2, -B), (-C/2, skip bound, alpha, r), (g, b); 40 bytes
      dk = __float_as_uint(o.depth);
      sb.spA[c] = make_float4(o.u, o.v, __fmul_rn(-0.5f, o.A), -o.B);
      sb.spB[c] = make_float4(__fmul_rn(-0.5f, o.C), pmin, al, q2.y);
      sb.spC[c] = make_float2(q2.z, q2.w);
    }
    sb.depth[c] = dk;
    sb.count[c] = n;
    sb.list_off[c] = loff;
    pairs_local += n;
#pragma unroll
    for (int d = 0; d < 4; ++d) atomicAdd(&s_hist[d][(dk >> (8 * d)) & 0xFFu], 1u);
  }
  for (int o = 16; o > 0; o >>= 1) pairs_local += __shfl_xor_sync(0xFFFFFFFFu, pairs_local, o);
  if (lane == 0 && pairs_local) atomicAdd(&ctr->n_pairs_raw, pairs_local);
  // flush the fused histogram
  __syncthreads();
  for (int k = threadIdx.x; k < 4 * 256; k += kPThreads) {
    uint32_t v = (&s_hist[0][0])[k];
    if (v) atomicAdd(&ctr->hist_depth[0][0] + k, v);
  }
}

struct ProjectGrids { int live, project; };
static PerDevice<ProjectGrids> g_proj;

void launch_project(const FrameC &fc, const uint32_t *visible, const float *alpha, const float4 *pool,
                    uint32_t *live_g, uint32_t *live_bits, const SplatBufs &sb, uint32_t *status,
                    FrameCounters *ctr, int num_sms, cudaStream_t st) {
  const ProjectGrids &g = g_proj.get([&](ProjectGrids &g) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, live_kernel, kLThreads, 0);
    g.live = num_sms * (per_sm > 0 ? per_sm : 1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, project_kernel<0>, kPThreads, 0);
    g.project = num_sms * (per_sm > 0 ? per_sm : 1);
  });
  live_mark_kernel<<<g.live, kLThreads, 0, st>>>(visible, alpha, live_bits, status, ctr);
  live_kernel<<<g.live, kLThreads, 0, st>>>(visible, live_bits, status, live_g, ctr);
  switch (fc.ablate) {
#define GSC_PROJ_CASE(k) \
  case k: project_kernel<k><<<g.project, kPThreads, 0, st>>>(fc, live_g, alpha, pool, sb, ctr); break;
    GSC_PROJ_CASE(0) GSC_PROJ_CASE(1) GSC_PROJ_CASE(2) GSC_PROJ_CASE(3)
    GSC_PROJ_CASE(4) GSC_PROJ_CASE(5) GSC_PROJ_CASE(6) GSC_PROJ_CASE(7)
#undef GSC_PROJ_CASE
    default: break;
  }
}
int project_tile_size() { return kLTile; }

}  // namespace gsc
