// blend.cu -- SURVEY §8(a) row a8: per-tile front-to-back alpha compositing
// for both eyes (Eq. 1; Alg. 1; reading R17).
//
// One 256-thread CTA per (eye, 16x16 tile); warp w owns the 8x4 pixel block
// at columns 8 (w & 1) .., rows 4 (w >> 1) .., one pixel per lane, and runs
// independently of the other warps (no block barrier): it walks the tile's
// depth-sorted pair list in chunks of 32 (pair keys prefetched two chunks
// ahead, the block's splat ids one), keeps the splats whose padded bounding
// box of {power >= skip bound} touches the block (one bit per block in the
// pair key, computed by project.cu's tile walk), stages those records in the
// warp's SMEM planes as pair groups (the 8 warps of a CTA fetch overlapping
// records, so most fetches are L1 hits), evaluates them two splats at a time
// with packed fp32x2 instructions in depth order, and leaves as soon as all 32
// of its pixels have terminated.  Skipping a (pixel, splat) by the box never
// changes a decision: outside it power < -ln(255 alpha) - 2^-7, so alpha' <
// 1/255 (N5).  The evaluation loop is warp-uniform: a lane that
// skips a splat, or has terminated, composites it with alpha' = 0, which
// leaves T and C bit-identical (fma(-0, T, T) = T, fma(c, 0, C) = C); the stop
// bookkeeping runs on a warp-uniform slow path taken only when some lane's T'
// nears the stop threshold.
// Per evaluated (pixel, splat), the op order of DESIGN.md N6 (the oracle's), except the exponential:
//   power  = fma(dx, fma(a', dx, b' dy), (c' dy) dy)      (skip if > 0)
//   alpha' = min(0.99, alpha exp(power))                  (skip if < 1/255)
//   T' = fma(-alpha', T, T); stop before T' < 1e-4; C = fma(c, alpha' T, C)
// exp runs on the SFU (ex2.approx); a pixel where the fast exponential could have
// flipped a skip or stop decision (alpha' within 2^-19 relative of 1/255, power > 0, T' within the
// band around 1e-4) is replayed exactly by blend_fixup_kernel, so every decision is the oracle's;
// pixels match it within ~1e-6 (<= 1e-4 where an unreplayed, immaterial stop flip remains), inside
// the north_star tolerance (2e-3 per channel, PSNR >= 55 dB).
#include "gsc_internal.cuh"

namespace gsc {

constexpr int kBThreads = 256;
constexpr float kLog2e = 1.44269502162933349609375f;
// The fast alpha' = min(0.99, alpha ex2.approx(fl(power log2e))) differs from the oracle's
// min(0.99, alpha exp_s(power)) by < 2^-20 relative for power in [skip bound, 0] (argument rounding
// <= 3.3e-7, ex2.approx <= 1.7e-7, exp_s <= 1 ulp, fl(log2e) and the two products' roundings; measured
// on every float of the range by tests/test_gpu_parity.py::test_fast_exp_error_bound), so the skip
// decision alpha' >= 1/255 can differ only inside 2^-19 relative of 1/255:
constexpr float kAlphaGuard = 7.5e-9f;    // >= 2^-19 x 1/255 (7.48e-9)
// |T_fast / T_exact - 1| <= 5e-4 at any point of a pixel's composite: the alpha' error of ex2.approx
// (<= 7e-7 relative) enters T' = T (1 - alpha') amplified by alpha'/(1 - alpha'), summed over the
// accepted splats with prod (1 - alpha') >= 1e-4 (<= 198 x 7e-7), plus <= 1 ulp of fma rounding per
// step over at most 2345 steps (alpha' >= 1/255): 1.4e-4 + 2.8e-4.  A stop decision T' < 1e-4 can
// differ from the oracle's only inside this band around 1e-4.
constexpr float kTBand = 5.0e-8f;          // 1e-4 x 5e-4
// A flipped stop decision moves the pixel by the contribution of the splat at the flip, w = alpha' T
// (the whole splat is in or out; after it the pixel stops at the next live splat).  Flips with
// w <= kJump are left alone (|pixel error| <= kJump + ~1e-6 < tests' BLEND_FAST_TOL = 2e-4); larger
// ones are replayed exactly.
constexpr float kJump = 1.0e-4f;

__device__ __forceinline__ void write_pixel(const FrameC &fc, int e, int px, int py, float T, float C0, float C1,
                                            float C2, void *out_l, void *out_r, int fmt) {
  const float o0 = __fmaf_rn(T, fc.bg[0], C0);
  const float o1 = __fmaf_rn(T, fc.bg[1], C1);
  const float o2 = __fmaf_rn(T, fc.bg[2], C2);
  void *out = e ? out_r : out_l;
  const size_t HW = (size_t)fc.width * fc.height, pix = (size_t)py * fc.width + px;
  if (fmt == 0) {
    float *o = reinterpret_cast<float *>(out);
    o[pix] = o0;
    o[HW + pix] = o1;
    o[2 * HW + pix] = o2;
  } else {
    auto q8 = [](float x) -> uint32_t {
      float y = fminf(fmaxf(__fmul_rn(x, 255.0f), 0.0f), 255.0f);
      return (uint32_t)__float2int_rn(y);
    };
    reinterpret_cast<uint32_t *>(out)[pix] = q8(o0) | (q8(o1) << 8) | (q8(o2) << 16) | (q8(1.0f - T) << 24);
  }
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr int kBWarps = kBThreads / 32;


__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d; asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d;
}
__device__ __forceinline__ float fminabs3(float a, float b, float c) {   // min(a, |b|, |c|)
  float d; asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(fabsf(b)), "f"(fabsf(c))); return d;
}
__device__ __forceinline__ float set_ge(float a, float b) {   // 1.0f if a >= b else 0.0f
  float d; asm("set.ge.f32.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f(uint32_t a, float x) { asm volatile("st.shared.f32 [%0], %1;" :: "r"(a), "f"(x)); }
__device__ __forceinline__ void sts_f2(uint32_t a, float x, float y) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" :: "r"(a), "f"(x), "f"(y));
}

// Per-warp staging planes: the block's splats in pair groups (slots 2k, 2k+1), so that one 16-byte load
// gives a field of both splats of a group, ready for the packed instructions:
//   P0 (u0 u1 v0 v1)  P1 (a'0 a'1 b'0 b'1)  P2 (c'0 c'1 alpha0 alpha1)  P3 (g0 b0 g1 b1)  P4 (r0 r1)
constexpr uint32_t kPl = 16 * 16;              // bytes per float4 plane (16 pair groups)
constexpr uint32_t kWarpStage = 4 * kPl + 16 * 8;   // + P4 (float2 per group) = 1152 bytes

template <bool kCount>   // kCount: accumulate n_evals / n_exp (GSC_F_COUNT_EVALS)
__global__ void __launch_bounds__(kBThreads)
blend_kernel(FrameC fc, const uint2 *__restrict__ ranges, const uint32_t *__restrict__ pair_keys,
             const uint32_t *__restrict__ pair_vals,
             const float4 *__restrict__ spA, const float4 *__restrict__ spB, const float2 *__restrict__ spC,
             void *__restrict__ out_l, void *__restrict__ out_r, int fmt, FrameCounters *__restrict__ ctr,
             uint32_t *__restrict__ fixup) {
  __shared__ __align__(16) unsigned char stage[kBWarps * kWarpStage];
  __shared__ uint32_t s_idx[kCount ? kBWarps * 32 : 1];   // (kCount) list index of each staged splat
  const int t = threadIdx.x;
  const uint32_t warp = (uint32_t)t >> 5, lane = lane_id();
  const int tile = blockIdx.x;
  const int e = tile >= fc.Te;
  const int tl = tile - e * fc.Te;
  const int tx = tl % fc.TW, ty = tl / fc.TW;
  // warp w owns the 8x4 block of columns 8 (w & 1) .. +7, rows 4 (w >> 1) .. +3 (squarer than 16x2:
  // fewer blocks per small splat)
  const int bx0 = tx * kTile + 8 * (int)(warp & 1), by0 = ty * kTile + 4 * (int)(warp >> 1);
  const int px = bx0 + (int)(lane & 7), py = by0 + (int)(lane >> 3);
  const bool inside = px < fc.width && py < fc.height;
  const float pxc = __fadd_rn((float)px, 0.5f), pyc = __fadd_rn((float)py, 0.5f);
  // ranges hold (~start, end) (sort.cu, last tile pass); an untouched tile (0, 0) is empty
  uint2 rg = make_uint2(~ranges[tile].x, ranges[tile].y);
  rg.x = __shfl_sync(0xFFFFFFFFu, rg.x, 0);   // (uniform by construction; tells the compiler)
  rg.y = __shfl_sync(0xFFFFFFFFu, rg.y, 0);
  float T = 1.0f, C0 = 0.0f;
  f2p C12 = pk2(0.0f, 0.0f);
  // bias of the exponent: 0 while the lane composites, -1000 once it has terminated (or lies outside
  // the image): ex2 then returns 0, so nothing is accepted any more (no predicate on the hot path)
  float bias = inside ? 0.0f : -1000.0f;
  // Fast-path threshold: a splat pair whose T' stays >= thr can flip no stop decision (T' >= 1e-4 +
  // kTBand) and needs none of the stop bookkeeping; below it (or once T sits inside the band: thr = T,
  // so only an accepted splat reaches it) the pair is replayed by the warp's exact step-by-step path.
  float thr = inside ? 0.0001f + kTBand : -1.0f;
  float trej = 1.0f;        // T' of the splat the lane stopped before (1: not stopped)
  float wl = 0.0f;          // contribution alpha' T of the last accepted splat of a slow-path pair
  float amarg = 1.0f;       // min over the lane's evaluations of |alpha' - 1/255|
  float xmax = -1.0f;       // max of the exponent argument: > 0 iff some evaluation had power > 0
  uint32_t nev = 0, nexp = 0, lstop = 0;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(stage + warp * kWarpStage);
  const uint32_t lt = lanemask_lt();

  // the pair keys run two chunks ahead and the block's splat ids one chunk ahead (registers), so a
  // chunk's staging waits only on its records, not on the key -> id -> record chain
  const uint32_t wbit = 24 + warp;
  uint32_t key0 = rg.x + lane < rg.y ? pair_keys[rg.x + lane] : 0u;
  uint32_t key1 = rg.x + 32 + lane < rg.y ? pair_keys[rg.x + 32 + lane] : 0u;
  uint32_t val0 = ((key0 >> wbit) & 1u) ? pair_vals[rg.x + lane] : 0u;
  for (uint32_t b = rg.x; b < rg.y; b += 32) {
    if (__all_sync(0xFFFFFFFFu, bias < 0.0f)) break;
    const uint32_t idx = b + lane;
    // the pair key's block mask (bit = warp) says whether the splat's box of {power >= skip bound}
    // meets this warp's 8x4 block (computed by project.cu with the fp32 test of DESIGN.md N5)
    const bool in = (key0 >> wbit) & 1u;   // (key0 = 0 past the end)
    const uint32_t c = val0;
    val0 = ((key1 >> wbit) & 1u) ? pair_vals[idx + 32] : 0u;
    key0 = key1;
    key1 = idx + 64 < rg.y ? pair_keys[idx + 64] : 0u;
    // compact the block's splats into the warp's pair-group planes, depth order preserved
    const uint32_t bits = __ballot_sync(0xFFFFFFFFu, in);
    const uint32_t n = __popc(bits);
    if (in) {
      const uint32_t slot = __popc(bits & lt);
      GSC_CHECK(slot < 32u && idx < ctr->n_pairs && c < ctr->n_splat);
      if (kCount) s_idx[warp * 32 + slot] = idx;
      const float4 A = spA[c], B = spB[c];
      const float2 Cc = spC[c];
      const uint32_t s = base + (slot >> 1) * 16 + (slot & 1) * 4;
      sts_f(s, A.x);
      sts_f(s + 8, A.y);
      sts_f(s + kPl, A.z);
      sts_f(s + kPl + 8, A.w);
      sts_f(s + 2 * kPl, B.x);
      sts_f(s + 2 * kPl + 8, B.z);
      sts_f2(base + 3 * kPl + (slot >> 1) * 16 + (slot & 1) * 8, Cc.x, Cc.y);
      sts_f(base + 4 * kPl + (slot >> 1) * 8 + (slot & 1) * 4, B.w);
    }
    if ((n & 1u) && lane == 0) {   // odd count: a zero splat (alpha 0: never accepted, guards quiet) in slot n
      const uint32_t s = base + (n >> 1) * 16 + 4;
      sts_f(s, 0.0f); sts_f(s + 8, 0.0f);
      sts_f(s + kPl, 0.0f); sts_f(s + kPl + 8, 0.0f);
      sts_f(s + 2 * kPl, 0.0f); sts_f(s + 2 * kPl + 8, 0.0f);
      sts_f2(base + 3 * kPl + (n >> 1) * 16 + 8, 0.0f, 0.0f);
      sts_f(base + 4 * kPl + (n >> 1) * 8 + 4, 0.0f);
    }
    __syncwarp();
    const uint32_t ng = (n + 1) >> 1;
    const bool done0 = bias < 0.0f;
    uint32_t jstop = n;     // (kCount) index of the splat the lane stopped before
#pragma unroll 2
    for (uint32_t g = 0; g < ng; ++g) {   // warp-uniform trip count, no divergent branch on the fast path
      const uint32_t p = base + 16 * g;
      const float4 P0 = lds_f4(p);                 // u0 u1 v0 v1
      const float4 P1 = lds_f4(p + kPl);           // a'0 a'1 b'0 b'1
      const float4 P2 = lds_f4(p + 2 * kPl);       // c'0 c'1 alpha0 alpha1
      const f2p dx = add2(pk2(P0.x, P0.y), bc2(-pxc));          // fl(u - pxc): adding -pxc is subtracting
      const f2p dy = add2(pk2(P0.z, P0.w), bc2(-pyc));
      const f2p qq = fma2(pk2(P1.x, P1.y), dx, mul2(pk2(P1.z, P1.w), dy));
      const f2p pw = fma2(dx, qq, mul2(mul2(pk2(P2.x, P2.y), dy), dy));   // N6, the oracle's bits
      float x0, x1;
      up2(fma2(pw, bc2(kLog2e), bc2(bias)), x0, x1);   // > 0 iff power > 0 while the lane composites
      xmax = fmax3(xmax, x0, x1);                       // (3DGS skips power > 0: left to the exact replay)
      f2p al = mul2(pk2(P2.z, P2.w), pk2(ex2_approx(x0), ex2_approx(x1)));
      float a0, a1;
      up2(al, a0, a1);
      a0 = fminf(0.99f, a0);
      a1 = fminf(0.99f, a1);
      float d0, d1;
      up2(add2(pk2(a0, a1), bc2(-kAlphaMin)), d0, d1);
      amarg = fminabs3(amarg, d0, d1);
      up2(mul2(pk2(a0, a1), pk2(set_ge(a0, kAlphaMin), set_ge(a1, kAlphaMin))), a0, a1);   // skip: alpha' = 0
      const float Tn0 = __fmaf_rn(-a0, T, T);
      const float Tn1 = __fmaf_rn(-a1, Tn0, Tn0);
      float w0, w1;
      if (__any_sync(0xFFFFFFFFu, Tn1 < thr)) {
        // slow path (rare: a stop, or T' near the stop threshold): the step-by-step decisions with the
        // bookkeeping the exactness guards need
        float wk[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float ak = k ? a1 : a0;
          const float Tn = __fmaf_rn(-ak, T, T);
          const bool term = Tn < 0.0001f && bias == 0.0f;   // stop before this splat
          if (kCount) {
            nexp += ak > 0.0f && !term && bias == 0.0f;
            if (term) {
              jstop = 2 * g + k;
              lstop = s_idx[warp * 32 + 2 * g + k];
            }
          }
          trej = term ? Tn : trej;
          const float w = (term || bias != 0.0f) ? 0.0f : __fmul_rn(ak, T);
          bias = term ? -1000.0f : bias;
          wl = w > 0.0f ? w : wl;
          T = w > 0.0f ? Tn : T;
          wk[k] = w;
        }
        w0 = wk[0];
        w1 = wk[1];
        thr = fminf(thr, T);
      } else {
        if (kCount) nexp += (a0 > 0.0f) + (a1 > 0.0f);
        w0 = __fmul_rn(a0, T);
        w1 = __fmul_rn(a1, Tn0);
        T = Tn1;
      }
      const float4 P3 = lds_f4(p + 3 * kPl);               // g0 b0 g1 b1
      const float2 P4 = lds_f2(base + 4 * kPl + 8 * g);    // r0 r1
      C0 = __fmaf_rn(P4.x, w0, C0);
      C0 = __fmaf_rn(P4.y, w1, C0);
      C12 = fma2(pk2(P3.x, P3.y), bc2(w0), C12);
      C12 = fma2(pk2(P3.z, P3.w), bc2(w1), C12);
    }
    if (kCount && !done0) nev += jstop + (jstop != n ? 1 : 0);
    __syncwarp();
  }
  // R5 exactness check: the fast exponential can flip a decision only (i) where alpha' came within
  // 2^-19 relative of 1/255 (skip), (ii) where power > 0 (skip), (iii) where T' came within kTBand of
  // 1e-4 (stop) -- for the splat the lane stopped before (trej) or its last accepted one (T; a splat
  // accepted by the fast path leaves T' >= 1e-4 + kTBand, so only a slow-path one can end in the band)
  // -- and a stop flip matters only if that splat's contribution exceeds kJump.  Such pixels (rare) go
  // to the exact replay (blend_fixup_kernel: the oracle's op sequence with exp_s); everywhere else
  // every decision is the oracle's.
  const bool redo = inside && (xmax > 0.0f || amarg <= kAlphaGuard ||
                               (fabsf(__fsub_rn(T, 0.0001f)) <= kTBand && wl > kJump) ||
                               (fabsf(__fsub_rn(trej, 0.0001f)) <= kTBand && __fsub_rn(T, trej) > kJump));
  const uint32_t rb = __ballot_sync(0xFFFFFFFFu, redo);
  if (rb) {
    uint32_t at = 0;
    if (lane == 0) at = atomicAdd(&ctr->n_fixup, (uint32_t)__popc(rb));
    at = __shfl_sync(0xFFFFFFFFu, at, 0);
    GSC_CHECK(!redo || at + __popc(rb & lt) < 2u * (uint32_t)(fc.width * fc.height));
    if (redo) fixup[at + __popc(rb & lt)] = ((uint32_t)e << 31) | (uint32_t)(py * fc.width + px);
  }
  if (kCount) {
    // the method's count (SURVEY d-3, the oracle's orc_blend_pixel): the tile-list entries up to and
    // including the one the pixel stopped before, the whole list if it never stopped
    uint32_t nlist = !inside ? 0u : bias < 0.0f ? lstop - rg.x + 1 : rg.y > rg.x ? rg.y - rg.x : 0u;   // (empty tile: (~0, 0))
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      nev += __shfl_xor_sync(0xFFFFFFFFu, nev, o);
      nexp += __shfl_xor_sync(0xFFFFFFFFu, nexp, o);
      nlist += __shfl_xor_sync(0xFFFFFFFFu, nlist, o);
    }
    if (lane == 0 && nlist) {
      atomicAdd(&ctr->n_evals, (unsigned long long)nev);
      atomicAdd(&ctr->n_exp, (unsigned long long)nexp);
      atomicAdd(&ctr->n_evals_list, (unsigned long long)nlist);
    }
  }
  if (!inside || redo) return;
  float C1, C2;
  up2(C12, C1, C2);
  write_pixel(fc, e, px, py, T, C0, C1, C2, out_l, out_r, fmt);
}

// GSC_F_BLEND_EXACT: the exact-exponential blend (round 1): exp_s (as exp_blend) on every evaluation that
// any lane of the warp needs, so every pixel is bit-identical to the oracle's (no replay needed).
template <bool kCount>
__global__ void __launch_bounds__(kBThreads)
blend_exact_kernel(FrameC fc, const uint2 *__restrict__ ranges, const uint32_t *__restrict__ pair_keys,
             const uint32_t *__restrict__ pair_vals,
             const float4 *__restrict__ spA, const float4 *__restrict__ spB, const float2 *__restrict__ spC,
             void *__restrict__ out_l, void *__restrict__ out_r, int fmt, FrameCounters *__restrict__ ctr) {
  // per-warp slots: [0, 32) = spA, [32, 64) = spB, [64, 96) = (g, b, -, -); one address register
  // walks all three (offsets 0, 512, 1024 bytes)
  __shared__ float4 slots[kBWarps][96];
  __shared__ uint32_t s_idx[kCount ? kBWarps * 32 : 1];   // (kCount) list index of each staged splat
  const int t = threadIdx.x;
  const uint32_t warp = (uint32_t)t >> 5, lane = lane_id();
  const int tile = blockIdx.x;
  const int e = tile >= fc.Te;
  const int tl = tile - e * fc.Te;
  const int tx = tl % fc.TW, ty = tl / fc.TW;
  // warp w owns the 8x4 block of columns 8 (w & 1) .. +7, rows 4 (w >> 1) .. +3 (squarer than 16x2:
  // fewer blocks per small splat)
  const int bx0 = tx * kTile + 8 * (int)(warp & 1), by0 = ty * kTile + 4 * (int)(warp >> 1);
  const int px = bx0 + (int)(lane & 7), py = by0 + (int)(lane >> 3);
  const bool inside = px < fc.width && py < fc.height;
  const float pxc = __fadd_rn((float)px, 0.5f), pyc = __fadd_rn((float)py, 0.5f);
  // ranges hold (~start, end) (sort.cu, last tile pass); an untouched tile (0, 0) is empty
  uint2 rg = make_uint2(~ranges[tile].x, ranges[tile].y);
  rg.x = __shfl_sync(0xFFFFFFFFu, rg.x, 0);   // (uniform by construction; tells the compiler)
  rg.y = __shfl_sync(0xFFFFFFFFu, rg.y, 0);
  float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
  // a lane's liveness floor on power: -inf while it composites, +inf once it has terminated (or lies
  // outside the image), so nothing is live for it any more (one FMNMX instead of a predicate chain)
  const float kInf = __int_as_float(0x7F800000);
  float pfloor = inside ? -kInf : kInf;
  uint32_t nev = 0, nexp = 0, lstop = 0;
  uint32_t base = (uint32_t)__cvta_generic_to_shared(&slots[warp][0]);
  asm volatile("" : "+r"(base));   // keep the slot address in a register
  const uint32_t lt = lanemask_lt();

  for (uint32_t b = rg.x; b < rg.y; b += 32) {
    if (__all_sync(0xFFFFFFFFu, pfloor > 0.0f)) break;
    const uint32_t idx = b + lane;
    // the pair key's block mask (bit = warp) says whether the splat's box of {power >= skip bound}
    // meets this warp's 8x4 block (computed by project.cu with the fp32 test of DESIGN.md N5)
    const bool in = idx < rg.y && ((pair_keys[idx] >> (24 + warp)) & 1u);
    // compact the block's splats into the warp's slots, depth order preserved
    const uint32_t bits = __ballot_sync(0xFFFFFFFFu, in);
    if (in) {
      const uint32_t c = pair_vals[idx];
      const uint32_t slot = __popc(bits & lt);
      if (kCount) s_idx[warp * 32 + slot] = idx;
      slots[warp][slot] = spA[c];
      slots[warp][32 + slot] = spB[c];
      *reinterpret_cast<float2 *>(&slots[warp][64 + slot]) = spC[c];
    }
    const uint32_t n = __popc(bits);
    __syncwarp();
    const uint32_t end = base + 16 * n;
    const bool done0 = pfloor > 0.0f;
    uint32_t pstop = end;
#pragma unroll 2
    for (uint32_t j = 0; j < n; ++j) {   // warp-uniform trip count
      const uint32_t p = base + 16 * j;
      const float4 a = lds_f4(p);          // (u, v, a' = -A/2, b' = -B)
      const float4 q = lds_f4(p + 512);    // (c' = -C/2, skip bound, alpha, r)
      const float dx = __fsub_rn(a.x, pxc), dy = __fsub_rn(a.y, pyc);
      const float qq = __fmaf_rn(a.z, dx, __fmul_rn(a.w, dy));
      const float power = __fmaf_rn(dx, qq, __fmul_rn(__fmul_rn(q.x, dy), dy));
      const bool live = power >= fmaxf(q.y, pfloor) && power <= 0.0f;
      if (!__any_sync(0xFFFFFFFFu, live)) continue;
      if (kCount) nexp += live;
      float al = fminf(0.99f, __fmul_rn(q.z, exp_blend(power)));   // garbage (discarded) if !live
      al = (live && al >= kAlphaMin) ? al : 0.0f;
      const float Tn = __fmaf_rn(-al, T, T);
      const bool term = Tn < 0.0001f;   // terminate before this splat; the rest is not evaluated
      if (kCount && term) {
        pstop = p;
        lstop = s_idx[warp * 32 + j];
      }
      if (!term) {
        const float w = __fmul_rn(al, T);
        const float2 gb = lds_f2(p + 1024);
        C0 = __fmaf_rn(q.w, w, C0);
        C1 = __fmaf_rn(gb.x, w, C1);
        C2 = __fmaf_rn(gb.y, w, C2);
        T = Tn;
      }
      // pfloor = term ? inf : pfloor as one predicated move (the C form compiles to three)
      asm("{\n .reg .pred p;\n setp.lt.f32 p, %1, 0f38D1B717;\n @p mov.b32 %0, 0x7F800000;\n}" : "+f"(pfloor) : "f"(Tn));
    }
    if (kCount && !done0) nev += (pstop - base) / 16 + (pfloor > 0.0f ? 1 : 0);
    __syncwarp();
  }
  if (kCount) {
    uint32_t nlist = !inside ? 0u : pfloor > 0.0f ? lstop - rg.x + 1 : rg.y > rg.x ? rg.y - rg.x : 0u;   // (as blend_kernel)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      nev += __shfl_xor_sync(0xFFFFFFFFu, nev, o);
      nexp += __shfl_xor_sync(0xFFFFFFFFu, nexp, o);
      nlist += __shfl_xor_sync(0xFFFFFFFFu, nlist, o);
    }
    if (lane == 0 && nlist) {
      atomicAdd(&ctr->n_evals, (unsigned long long)nev);
      atomicAdd(&ctr->n_exp, (unsigned long long)nexp);
      atomicAdd(&ctr->n_evals_list, (unsigned long long)nlist);
    }
  }
  if (!inside) return;
  write_pixel(fc, e, px, py, T, C0, C1, C2, out_l, out_r, fmt);
}

// Exact replay of the flagged pixels: the oracle's per-pixel loop (O-8, N6) with exp_s over
// the tile's sorted list (the pair key's block bit skips splats whose skip box misses the pixel's 8x4
// block: decision-preserving, N5).  One CTA of 8 warps per pixel: a window of 256 consecutive pairs is
// evaluated in parallel (warp w takes the window's chunk w: power / alpha' / the skip decisions exactly,
// the accepted ones compacted in order into the warp's SMEM row), then warp 0 composites the window's
// accepted splats in list order (the T chain is sequential).  Keys run three windows ahead, splat ids
// two, records one (registers), so a window waits on none of its own loads.
constexpr int kFixThreads = 256;
__global__ void __launch_bounds__(kFixThreads)
blend_fixup_kernel(FrameC fc, const uint2 *__restrict__ ranges, const uint32_t *__restrict__ pair_keys,
                   const uint32_t *__restrict__ pair_vals, const float4 *__restrict__ spA,
                   const float4 *__restrict__ spB, const float2 *__restrict__ spC, void *__restrict__ out_l,
                   void *__restrict__ out_r, int fmt, const FrameCounters *__restrict__ ctr,
                   const uint32_t *__restrict__ fixup) {
  constexpr int kW = kFixThreads / 32;
  __shared__ float4 s_acc[kW][32];   // accepted (alpha', r, g, b) of each chunk of the window, list order
  __shared__ uint32_t s_n[kW];
  __shared__ int s_stop;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, lt = lanemask_lt();
  const uint32_t nfix = ctr->n_fixup;
  for (uint32_t k = blockIdx.x; k < nfix; k += gridDim.x) {
    const uint32_t code = fixup[k];
    const int e = (int)(code >> 31);
    const int pix = (int)(code & 0x7FFFFFFFu);
    const int px = pix % fc.width, py = pix / fc.width;
    const int tile = e * fc.Te + (py / kTile) * fc.TW + px / kTile;
    const uint32_t wbit = 1u << (24 + ((px % kTile) >> 3) + 2 * ((py % kTile) >> 2));
    const float pxc = __fadd_rn((float)px, 0.5f), pyc = __fadd_rn((float)py, 0.5f);
    const uint32_t r0 = ~ranges[tile].x, r1 = ranges[tile].y;
    float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;   // (warp 0)
    auto key_at = [&](uint32_t i) -> uint32_t { return i < r1 ? pair_keys[i] : 0u; };
    const uint32_t t = threadIdx.x;
    uint32_t k0 = key_at(r0 + t), k1 = key_at(r0 + kFixThreads + t), k2 = key_at(r0 + 2 * kFixThreads + t);
    uint32_t v1 = (k1 & wbit) ? pair_vals[r0 + kFixThreads + t] : 0u;
    float4 nA = make_float4(0.f, 0.f, 0.f, 0.f), nB = nA;
    float2 nC = make_float2(0.f, 0.f);
    if (k0 & wbit) {
      const uint32_t c = pair_vals[r0 + t];
      GSC_CHECK(r0 + t < ctr->n_pairs && c < ctr->n_splat);
      nA = spA[c]; nB = spB[c]; nC = spC[c];
    }
    for (uint32_t wb = r0; wb < r1; wb += kFixThreads) {   // CTA-uniform
      const bool has = k0 & wbit;   // (k0 = 0 past the end)
      const float4 a = nA, q = nB;
      const float2 cc = nC;
      if (k1 & wbit) {
        GSC_CHECK(wb + kFixThreads + t < ctr->n_pairs && v1 < ctr->n_splat);
        nA = spA[v1]; nB = spB[v1]; nC = spC[v1];
      }
      v1 = (k2 & wbit) ? pair_vals[wb + 2 * kFixThreads + t] : 0u;
      k0 = k1;
      k1 = k2;
      k2 = key_at(wb + 3 * kFixThreads + t);
      bool ok = false;
      float al = 0.0f;
      if (has) {
        const float dx = __fsub_rn(a.x, pxc), dy = __fsub_rn(a.y, pyc);
        const float qq = __fmaf_rn(a.z, dx, __fmul_rn(a.w, dy));
        const float power = __fmaf_rn(dx, qq, __fmul_rn(__fmul_rn(q.x, dy), dy));
        if (!(power > 0.0f)) {
          al = fminf(0.99f, __fmul_rn(q.z, exp_s(power)));
          ok = al >= kAlphaMin;
        }
      }
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, ok);
      if (ok) s_acc[warp][__popc(m & lt)] = make_float4(al, q.w, cc.x, cc.y);
      if (lane == 0) s_n[warp] = __popc(m);
      __syncthreads();
      if (warp == 0) {
        bool stop = false;
        for (uint32_t w = 0; w < (uint32_t)kW && !stop; ++w) {
          const uint32_t n = s_n[w];
          for (uint32_t j = 0; j < n; ++j) {   // warp-uniform (broadcast reads)
            const float4 r = s_acc[w][j];
            const float Tn = __fmaf_rn(-r.x, T, T);
            if (Tn < 0.0001f) { stop = true; break; }
            const float wgt = __fmul_rn(r.x, T);
            C0 = __fmaf_rn(r.y, wgt, C0);
            C1 = __fmaf_rn(r.z, wgt, C1);
            C2 = __fmaf_rn(r.w, wgt, C2);
            T = Tn;
          }
        }
        if (lane == 0) s_stop = stop;
      }
      __syncthreads();
      if (s_stop) break;
    }
    if (t == 0) write_pixel(fc, e, px, py, T, C0, C1, C2, out_l, out_r, fmt);
    __syncthreads();   // (s_acc / s_n / s_stop reuse by the next pixel)
  }
}

void launch_blend(const FrameC &fc, const uint2 *ranges, const uint32_t *pair_keys, const uint32_t *pair_vals,
                  const float4 *spA, const float4 *spB, const float2 *spC, void *out_l, void *out_r, int fmt,
                  FrameCounters *ctr, uint32_t *fixup, bool count, bool exact, int num_sms, cudaStream_t st) {
  const int grid = (fc.ablate & kAblMono) ? fc.Te : 2 * fc.Te;   // GSC_F_MONO: left eye tiles only
  if (exact) {
    if (count)
      blend_exact_kernel<true><<<grid, kBThreads, 0, st>>>(fc, ranges, pair_keys, pair_vals, spA, spB, spC, out_l,
                                                           out_r, fmt, ctr);
    else
      blend_exact_kernel<false><<<grid, kBThreads, 0, st>>>(fc, ranges, pair_keys, pair_vals, spA, spB, spC, out_l,
                                                            out_r, fmt, ctr);
    return;
  }
  if (count)
    blend_kernel<true><<<grid, kBThreads, 0, st>>>(fc, ranges, pair_keys, pair_vals, spA, spB, spC, out_l, out_r, fmt,
                                                   ctr, fixup);
  else
    blend_kernel<false><<<grid, kBThreads, 0, st>>>(fc, ranges, pair_keys, pair_vals, spA, spB, spC, out_l, out_r, fmt,
                                                    ctr, fixup);
  blend_fixup_kernel<<<4 * num_sms, kFixThreads, 0, st>>>(fc, ranges, pair_keys, pair_vals, spA, spB, spC, out_l, out_r, fmt, ctr,
                                                  fixup);
}

// elementary-function self test (parity sweeps through the C ABI)
__global__ void elem_kernel(int fn, const float *__restrict__ in, float *__restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float x = in[i];
    out[i] = fn == 0 ? exp_s(x) : fn == 1 ? log_s(x) : fn == 2 ? tanh_s(x) : fn == 3 ? sigmoid_s(x)
             : fn == 4 ? exp_blend(x) : ex2_approx(__fmaf_rn(x, kLog2e, 0.0f));   // 5: the blend's fast exp
  }
}
void launch_elem(int fn, const float *in, float *out, size_t n, int num_sms, cudaStream_t st) {
  elem_kernel<<<num_sms * 8, 256, 0, st>>>(fn, in, out, n);
}

}  // namespace gsc
