// blend.cu -- SURVEY §8(a) row a8: per-tile front-to-back alpha compositing
// for both eyes (Eq. 1; Alg. 1; reading R17).
//
// One 256-thread CTA per (eye, 16x16 tile), one pixel per thread; warp w owns
// the 16x2 pixel strip of rows 2w, 2w+1.  The tile's depth-sorted splats are
// staged through shared memory in batches of 256 (40 bytes each); while
// staging, each thread also computes an 8-bit strip mask: bit w is set unless
// the padded bounding box of {power >= skip bound} misses strip w.  A warp
// then walks only the batch entries of its strip (ballot + ffs), stops as
// soon as all its 32 pixels have terminated, and the CTA leaves when all 256
// have (__syncthreads_count).  Skipping a (pixel, splat) this way never
// changes a decision: outside that box power < -ln(255 alpha) - 2^-7, so
// alpha' < 1/255 (N5).  Per evaluated (pixel, splat), the exact op
// order of DESIGN.md N6 (identical in the oracle):
//   power  = fma(dx, fma(a', dx, b' dy), (c' dy) dy)      (skip if > 0)
//   alpha' = min(0.99, alpha exp_s(power))                (skip if < 1/255)
//   T' = fma(-alpha', T, T); stop before T' < 1e-4; C = fma(c, alpha' T, C)
#include "gsc_internal.cuh"

namespace gsc {

constexpr int kBThreads = 256;

// explicit 32-bit shared-window loads (keeps the window base out of the hot loop)
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
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}

__global__ void __launch_bounds__(kBThreads)
blend_kernel(FrameC fc, const uint2 *__restrict__ ranges, const uint32_t *__restrict__ pair_vals,
             const float4 *__restrict__ spA, const float4 *__restrict__ spB, const float4 *__restrict__ spC,
             void *__restrict__ out_l, void *__restrict__ out_r, int fmt, FrameCounters *__restrict__ ctr) {
  __shared__ float4 sA[kBThreads];
  __shared__ float4 sB[kBThreads];
  __shared__ float2 sC[kBThreads];
  __shared__ uint32_t sM[kBThreads];
  __shared__ uint16_t sL[kBThreads / 32][kBThreads];
  const int t = threadIdx.x;
  const uint32_t warp = (uint32_t)t >> 5, lane = lane_id();
  const int tile = blockIdx.x;
  const int e = tile >= fc.Te;
  const int tl = tile - e * fc.Te;
  const int tx = tl % fc.TW, ty = tl / fc.TW;
  const int px = tx * kTile + (t & 15), py = ty * kTile + (t >> 4);
  const bool inside = px < fc.width && py < fc.height;
  const float pxc = __fadd_rn((float)px, 0.5f), pyc = __fadd_rn((float)py, 0.5f);
  const float X0 = __fadd_rn((float)(tx * kTile), 0.5f), X1 = __fadd_rn(X0, 15.0f);
  const float Yb = __fadd_rn((float)(ty * kTile), 0.5f);
  const uint2 rg = ranges[tile];
  float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
  int done = !inside;
  uint32_t nev = 0, nexp = 0;
  for (uint32_t b = rg.x; b < rg.y; b += kBThreads) {
    __syncthreads();
    const uint32_t idx = b + t;
    if (idx < rg.y) {
      const uint32_t c = pair_vals[idx];
      const float4 a = spA[c];
      const float4 cc = spC[c];
      sA[t] = a;
      sB[t] = spB[c];
      sC[t] = make_float2(cc.x, cc.y);
      uint32_t mask = 0;
      if (__fadd_rn(a.x, cc.z) >= X0 && __fsub_rn(a.x, cc.z) <= X1) {
        const float lo = __fsub_rn(a.y, cc.w), hi = __fadd_rn(a.y, cc.w);
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const float y0 = __fadd_rn(Yb, (float)(2 * w));
          if (hi >= y0 && lo <= __fadd_rn(y0, 1.0f)) mask |= 1u << w;
        }
      }
      sM[t] = mask;
    }
    __syncthreads();
    const int cnt = min((uint32_t)kBThreads, rg.y - b);
    if (!__all_sync(0xFFFFFFFFu, done)) {
      // this warp's strip list (batch indices in depth order)
      int n = 0;
      for (int c0 = 0; c0 < cnt; c0 += 32) {
        const bool in = c0 + (int)lane < cnt && ((sM[c0 + lane] >> warp) & 1u);
        const uint32_t bits = __ballot_sync(0xFFFFFFFFu, in);
        if (in) sL[warp][n + __popc(bits & lanemask_lt())] = (uint16_t)(c0 + lane);
        n += __popc(bits);
      }
      __syncwarp();
      uint32_t aA = (uint32_t)__cvta_generic_to_shared(sA), aB = (uint32_t)__cvta_generic_to_shared(sB);
      uint32_t aC = (uint32_t)__cvta_generic_to_shared(sC);
      uint32_t aL = (uint32_t)__cvta_generic_to_shared(&sL[warp][0]);
      // opaque to the compiler: keeps the addresses in registers instead of re-deriving the window base
      asm volatile("" : "+r"(aA), "+r"(aB), "+r"(aC), "+r"(aL));
      for (int i = 0; i < n; ++i) {
        if ((i & 7) == 0 && __all_sync(0xFFFFFFFFu, done)) break;
        if (done) continue;
        const uint32_t k = lds_u16(aL + 2 * i);
        ++nev;
        const float4 a = lds_f4(aA + 16 * k);     // (u, v, a' = -A/2, b' = -B)
        const float4 q = lds_f4(aB + 16 * k);     // (c' = -C/2, skip bound, alpha, r)
        const float dx = __fsub_rn(a.x, pxc), dy = __fsub_rn(a.y, pyc);
        const float qq = __fmaf_rn(a.z, dx, __fmul_rn(a.w, dy));
        const float power = __fmaf_rn(dx, qq, __fmul_rn(__fmul_rn(q.x, dy), dy));
        if (power < q.y || power > 0.0f) continue;
        ++nexp;
        const float al = fminf(0.99f, __fmul_rn(q.z, exp_core(power)));   // power in [-5.6, 0]
        if (al < kAlphaMin) continue;
        const float Tn = __fmaf_rn(-al, T, T);
        if (Tn < 0.0001f) { done = 1; continue; }
        const float w = __fmul_rn(al, T);
        const float2 gb = lds_f2(aC + 8 * k);
        C0 = __fmaf_rn(q.w, w, C0);
        C1 = __fmaf_rn(gb.x, w, C1);
        C2 = __fmaf_rn(gb.y, w, C2);
        T = Tn;
      }
    }
    if (__syncthreads_count(done) == kBThreads) break;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nev += __shfl_xor_sync(0xFFFFFFFFu, nev, o);
    nexp += __shfl_xor_sync(0xFFFFFFFFu, nexp, o);
  }
  if (lane == 0 && nev) {
    atomicAdd(&ctr->n_evals, (unsigned long long)nev);
    atomicAdd(&ctr->n_exp, (unsigned long long)nexp);
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

void launch_blend(const FrameC &fc, const uint2 *ranges, const uint32_t *pair_vals, const float4 *spA,
                  const float4 *spB, const float4 *spC, void *out_l, void *out_r, int fmt, FrameCounters *ctr,
                  cudaStream_t st) {
  blend_kernel<<<2 * fc.Te, kBThreads, 0, st>>>(fc, ranges, pair_vals, spA, spB, spC, out_l, out_r, fmt, ctr);
}

// elementary-function self test (parity sweeps through the C ABI)
__global__ void elem_kernel(int fn, const float *__restrict__ in, float *__restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float x = in[i];
    out[i] = fn == 0 ? exp_s(x) : fn == 1 ? log_s(x) : fn == 2 ? tanh_s(x) : sigmoid_s(x);
  }
}
void launch_elem(int fn, const float *in, float *out, size_t n, int num_sms, cudaStream_t st) {
  elem_kernel<<<num_sms * 8, 256, 0, st>>>(fn, in, out, n);
}

}  // namespace gsc
