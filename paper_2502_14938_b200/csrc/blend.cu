// blend.cu -- SURVEY §8(a) row a8: per-tile front-to-back alpha compositing
// for both eyes (Eq. 1; Alg. 1; reading R17).
//
// One 256-thread CTA per (eye, 16x16 tile); warp w owns the 8x4 pixel block
// at columns 8 (w & 1) .., rows 4 (w >> 1) .., one pixel per lane, and runs
// independently of the other warps (no block barrier): it walks the tile's
// depth-sorted pair list in chunks of 32, keeps the splats whose padded
// bounding box of {power >= skip bound} touches the block (one bit per block
// in the pair key, computed by project.cu's tile walk), stages those records
// in the warp's SMEM slots (the 8 warps of a CTA fetch overlapping records, so
// most fetches are L1 hits),
// evaluates them in depth order and leaves as soon as all 32 of its pixels
// have terminated.  Skipping a (pixel, splat) by the box never changes a
// decision: outside it power < -ln(255 alpha) - 2^-7, so alpha' < 1/255
// (N5).  The evaluation loop is warp-uniform (no divergent
// branches): a lane that skips a splat, or has terminated, composites it with
// alpha' = 0, which leaves T and C bit-identical (fma(-0, T, T) = T,
// fma(c, 0, C) = C); only when no lane of the warp needs the exp is the splat
// skipped outright.
// Per evaluated (pixel, splat), the exact op order of DESIGN.md N6
// (identical in the oracle):
//   power  = fma(dx, fma(a', dx, b' dy), (c' dy) dy)      (skip if > 0)
//   alpha' = min(0.99, alpha exp_s(power))                (skip if < 1/255)
//   T' = fma(-alpha', T, T); stop before T' < 1e-4; C = fma(c, alpha' T, C)
#include "gsc_internal.cuh"

namespace gsc {

constexpr int kBThreads = 256;
constexpr int kBWarps = kBThreads / 32;

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

template <bool kCount>   // kCount: accumulate n_evals / n_exp (GSC_F_COUNT_EVALS)
__global__ void __launch_bounds__(kBThreads)
blend_kernel(FrameC fc, const uint2 *__restrict__ ranges, const uint32_t *__restrict__ pair_keys,
             const uint32_t *__restrict__ pair_vals,
             const float4 *__restrict__ spA, const float4 *__restrict__ spB, const float4 *__restrict__ spC,
             void *__restrict__ out_l, void *__restrict__ out_r, int fmt, FrameCounters *__restrict__ ctr) {
  // per-warp slots: [0, 32) = spA, [32, 64) = spB, [64, 96) = (g, b, -, -); one address register
  // walks all three (offsets 0, 512, 1024 bytes)
  __shared__ float4 slots[kBWarps][96];
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
  uint32_t nev = 0, nexp = 0;
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
      slots[warp][slot] = spA[c];
      slots[warp][32 + slot] = spB[c];
      slots[warp][64 + slot] = spC[c];
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
      al = (al >= kAlphaMin) & live ? al : 0.0f;
      const float Tn = __fmaf_rn(-al, T, T);
      const bool term = Tn < 0.0001f;   // terminate before this splat; the rest is not evaluated
      if (kCount && term) pstop = p;
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
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      nev += __shfl_xor_sync(0xFFFFFFFFu, nev, o);
      nexp += __shfl_xor_sync(0xFFFFFFFFu, nexp, o);
    }
    if (lane == 0 && nev) {
      atomicAdd(&ctr->n_evals, (unsigned long long)nev);
      atomicAdd(&ctr->n_exp, (unsigned long long)nexp);
    }
  }
  if (!inside) return;
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

void launch_blend(const FrameC &fc, const uint2 *ranges, const uint32_t *pair_keys, const uint32_t *pair_vals,
                  const float4 *spA,
                  const float4 *spB, const float4 *spC, void *out_l, void *out_r, int fmt, FrameCounters *ctr,
                  bool count, cudaStream_t st) {
  const int grid = (fc.ablate & kAblMono) ? fc.Te : 2 * fc.Te;   // GSC_F_MONO: left eye tiles only
  if (count)
    blend_kernel<true><<<grid, kBThreads, 0, st>>>(fc, ranges, pair_keys, pair_vals, spA, spB, spC, out_l, out_r, fmt, ctr);
  else
    blend_kernel<false><<<grid, kBThreads, 0, st>>>(fc, ranges, pair_keys, pair_vals, spA, spB, spC, out_l, out_r, fmt, ctr);
}

// elementary-function self test (parity sweeps through the C ABI)
__global__ void elem_kernel(int fn, const float *__restrict__ in, float *__restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float x = in[i];
    out[i] = fn == 0 ? exp_s(x) : fn == 1 ? log_s(x) : fn == 2 ? tanh_s(x) : fn == 3 ? sigmoid_s(x) : exp_blend(x);
  }
}
void launch_elem(int fn, const float *in, float *out, size_t n, int num_sms, cudaStream_t st) {
  elem_kernel<<<num_sms * 8, 256, 0, st>>>(fn, in, out, n);
}

}  // namespace gsc
