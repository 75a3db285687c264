// gsc_internal.cuh -- product-side device types and helpers (B200 / sm_100a).
// Shares nothing with oracle/.  Arithmetic follows DESIGN.md "Numerics";
// every .cu is compiled with -fmad=false -prec-div=true -prec-sqrt=true
// -ftz=false so IEEE fp32 ops are emitted exactly as written (FMA only where
// __fmaf_rn is spelled out).
#pragma once
#include <cstdio>
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

namespace gsc {

constexpr int kF = 32;       // feature dim
constexpr int kK = 10;       // Gaussians per anchor
constexpr int kH = 32;       // hidden width per head
constexpr int kNOut = 11 * kK;
constexpr int kTile = 16;    // 16x16 pixel tiles

// ---- per-frame constants (host fp64 -> fp32, Eqs. 5-6) ----
struct EyeC {
  float p[3], r0[3], r1[3], r2[3];
  float fx, fy, cx, cy, near_plane, far_plane, limx, limy;
};
struct UniC {
  float p[3], right[3], up[3], fwd[3];
  float near_plane, far_plane, tx, ty, kx, ky;
};
struct FrameC {
  UniC u;
  EyeC eye[2];
  int width, height, TW, TH, Te;   // tiles per row / column / eye
  int L;
  float d0;
  float bg[3];
  int ablate;   // kAbl* bits (GSC_F_ABL_*): F1 ablations of the extent / tile test
};
constexpr int kAblFixedExtent = 1;
constexpr int kAblAabbTiles = 2;
constexpr int kAblMono = 4;       // GSC_F_MONO: left eye only (per-eye pipelines of the no-de-redundancy ablation)

// GSC_BOUNDS_CHECK (a debug build, tools/bounds_build.py): device-side checks of the data-dependent
// indices (staging slots, record / pair / list / output positions) that trap with a message when one is
// out of range -- the stand-in for compute-sanitizer memcheck where the pool does not offer it.  A
// no-op in the product build.
#ifdef GSC_BOUNDS_CHECK
#define GSC_CHECK(c)                                                                         \
  do {                                                                                       \
    if (!(c)) {                                                                              \
      printf("GSC_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c,    \
             (int)blockIdx.x, (int)threadIdx.x);                                             \
      __trap();                                                                              \
    }                                                                                        \
  } while (0)
#else
#define GSC_CHECK(c) do { } while (0)
#endif

// ---- device-resident counters, zeroed at every frame start ----
struct FrameCounters {
  uint32_t tile_cull, tile_derive, tile_project, tile_emit;
  uint32_t tile_sort[8];
  uint32_t n_visible, n_miss, n_new, n_splat;
  uint32_t n_pairs_raw;        // pairs the frame needed
  uint32_t n_pairs;            // min(raw, capacity)
  uint32_t overflow;
  uint32_t list_top;           // project: bump allocator of the kept-tile list
  unsigned long long n_evals;  // blend: (pixel, splat) evaluations executed
  unsigned long long n_exp;    // blend: evaluations that reached exp_s
  unsigned long long n_evals_list;   // blend: the method's evaluations (tile-list entries up to each pixel's stop)
  uint32_t tile_pairoff, tile_expand;
  uint32_t list_overflow;      // project: the kept-tile list ran out (the frame's pairs are dropped)
  uint32_t n_nonfinite;        // project: (Gaussian, eye) skipped for non-finite parameters
  uint32_t n_fixup;            // blend: pixels sent to the exact replay (R5 guard bands)
  uint32_t pad3[3];
  uint32_t hist_depth[4][256];
  uint32_t hist_tile[2][256];
};

// ---- persistent cache-policy state (not reset per frame) ----
struct PolicyState {
  int32_t frame;       // f of the next frame
  int32_t depth;       // depth_f in effect for the next frame
  int32_t W;           // watermark W_f = max_{f'<=f}(f' - depth_f')
  int32_t d_max;
  int32_t literal;     // GSC_F_DEPTH_LITERAL
  int32_t guide;       // guiding function: 0 linear, 1 exponential, 2 staged (GSC_F_GUIDE_*)
  int32_t stagger;     // GSC_F_STAGGER (R26)
  int32_t pad;
};

// compacted splat records (index c), written by project, read by emit/blend
struct SplatBufs {
  float4 *spA;       // (u, v, -A/2, -B)     A,B,C = conic (A dx^2 + 2B dx dy + C dy^2)
  float4 *spB;       // (-C/2, skip bound, alpha, r)
  float2 *spC;       // (g, b): the rest of the colour
  uint32_t *count;   // kept tiles
  uint32_t *depth;   // depth key = bits(z) (depth-sort input)
  uint32_t *list_off;  // start of the splat's kept-tile keys in `list`
  uint32_t *list;      // kept-tile keys (eye*T_e + ty*TW + tx), per splat contiguous, row-major
  uint32_t list_cap;
};

// R32 combine inputs of the real-weights derivation (F4-B)
struct CombineF32 {
  int dist, bank;                        // distance input, feature bank
  const float *Wb1, *bb1, *Wb2, *bb2;    // bank MLP [4][32], [32], [32][3], [3]
};

struct EmitIn {
  const uint32_t *sorted;    // splat indices in depth order
  const uint32_t *count;     // kept tiles per splat
  const uint32_t *list_off;
  const uint32_t *list;
  uint32_t *pair_off;        // exclusive scan of count in depth order
};

// snapshot copied to host every frame
struct FrameRecordDev {
  int32_t frame, depth_used, depth_next, pad0;
  uint32_t n_visible, n_miss, n_new, n_splat, n_pairs_raw, overflow, n_nonfinite, n_fixup;
  unsigned long long n_evals, n_exp, n_evals_list;
};

// Launch configuration kept per CUDA device (grid sizes from the device's occupancy, the
// MaxDynamicSharedMemorySize opt-ins, which are per-device attributes), initialised once per device,
// thread-safe: contexts on several devices of one process each get their own.
constexpr int kMaxDevices = 64;
template <typename T>
struct PerDevice {
  T v[kMaxDevices]{};
  std::once_flag once[kMaxDevices];
  template <typename Init>
  T &get(Init init) {
    int d = 0;
    cudaGetDevice(&d);
    if (d < 0 || d >= kMaxDevices) d = 0;
    std::call_once(once[d], [&] { init(v[d]); });
    return v[d];
  }
};

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ float f_of_u(uint32_t b) { return __uint_as_float(b); }
__device__ __forceinline__ uint32_t u_of_f(float f) { return __float_as_uint(f); }

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back over 32-bit status words: [31:30] flag (1 = aggregate,
// 2 = inclusive prefix), [29:0] value.  Called by one full warp; returns the
// exclusive prefix of `tile` (identical in all lanes).
__device__ __forceinline__ uint32_t lookback_u32(uint32_t *status, uint32_t tile) {
  constexpr uint32_t kMask = 0x3FFFFFFFu;
  uint32_t prefix = 0;
  int64_t base = (int64_t)tile - 1;
  const uint32_t lane = lane_id();
  while (base >= 0) {
    int64_t idx = base - (int64_t)lane;
    uint32_t s = 2u << 30;  // out of range counts as an inclusive zero
    if (idx >= 0) {
      do { s = ld_volatile_u32(status + idx); } while ((s >> 30) == 0);
    }
    uint32_t incl = __ballot_sync(0xFFFFFFFFu, (s >> 30) == 2u);
    uint32_t upto = incl ? (uint32_t)(__ffs(incl) - 1) : 31u;   // nearest inclusive lane
    uint32_t v = (lane <= upto) ? (s & kMask) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    prefix += v;
    if (incl) break;
    base -= 32;
  }
  return prefix;
}

// The same look-back run by a whole CTA of kThreads: every thread reads one
// predecessor status word, so one round trip covers kThreads tiles -- with a
// persistent grid of ~600 tiles in flight the inclusive frontier lags by
// about that many tiles, which a 32-wide warp window walks in ~20 serial
// round trips.  All threads must call it; returns the exclusive prefix in all
// of them.  `red` is kThreads/32 + 1 words of shared scratch.
template <int kThreads>
__device__ __forceinline__ uint32_t block_lookback_u32(uint32_t *status, uint32_t tile, uint32_t *red) {
  constexpr uint32_t kMask = 0x3FFFFFFFu;
  constexpr int kW = kThreads / 32;
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  uint32_t prefix = 0;
  int64_t base = (int64_t)tile - 1;
  while (base >= 0) {
    const int64_t idx = base - (int64_t)t;
    uint32_t s = 2u << 30;   // out of range counts as an inclusive zero
    if (idx >= 0) {
      do { s = ld_volatile_u32(status + idx); } while ((s >> 30) == 0);
    }
    // nearest inclusive predecessor = smallest thread index holding one
    const uint32_t incl = __ballot_sync(0xFFFFFFFFu, (s >> 30) == 2u);
    if (lane == 0) red[warp] = incl ? warp * 32 + (uint32_t)(__ffs(incl) - 1) : (uint32_t)kThreads;
    __syncthreads();
    uint32_t upto = kThreads;
#pragma unroll
    for (int w = 0; w < kW; ++w) upto = min(upto, red[w]);
    uint32_t v = t <= upto ? (s & kMask) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kW; ++w) prefix += red[w];
    __syncthreads();
    if (upto < (uint32_t)kThreads) break;
    base -= kThreads;
  }
  return prefix;
}

// block_lookback_u32 over 64-bit status words ([63:62] flag, [61:0] two packed counts, see below):
// one round trip covers kThreads predecessors.  All threads call it; `red` is kThreads/32 + 1 u64
// words of shared scratch.
template <int kThreads>
__device__ __forceinline__ unsigned long long block_lookback_u64(unsigned long long *status, uint32_t tile,
                                                                 unsigned long long *red) {
  constexpr unsigned long long kMask = (1ull << 62) - 1;
  constexpr int kW = kThreads / 32;
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  unsigned long long prefix = 0;
  int64_t base = (int64_t)tile - 1;
  while (base >= 0) {
    const int64_t idx = base - (int64_t)t;
    unsigned long long s = 2ull << 62;   // out of range counts as an inclusive zero
    if (idx >= 0) {
      do { s = ld_volatile_u64(status + idx); } while ((s >> 62) == 0);
    }
    const uint32_t incl = __ballot_sync(0xFFFFFFFFu, (s >> 62) == 2ull);
    if (lane == 0) red[warp] = incl ? warp * 32 + (uint32_t)(__ffs(incl) - 1) : (uint32_t)kThreads;
    __syncthreads();
    uint32_t upto = kThreads;
#pragma unroll
    for (int w = 0; w < kW; ++w) upto = min(upto, (uint32_t)red[w]);
    unsigned long long v = t <= upto ? (s & kMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kW; ++w) prefix += red[w];
    __syncthreads();
    if (upto < (uint32_t)kThreads) break;
    base -= kThreads;
  }
  return prefix;
}

// 64-bit status: [63:62] flag, [61:31] field b, [30:0] field a (two counts).
__device__ __forceinline__ unsigned long long lookback_u64(unsigned long long *status, uint32_t tile) {
  constexpr unsigned long long kMask = (1ull << 62) - 1;
  unsigned long long prefix = 0;
  int64_t base = (int64_t)tile - 1;
  const uint32_t lane = lane_id();
  while (base >= 0) {
    int64_t idx = base - (int64_t)lane;
    unsigned long long s = 2ull << 62;
    if (idx >= 0) {
      do { s = ld_volatile_u64(status + idx); } while ((s >> 62) == 0);
    }
    uint32_t incl = __ballot_sync(0xFFFFFFFFu, (s >> 62) == 2ull);
    uint32_t upto = incl ? (uint32_t)(__ffs(incl) - 1) : 31u;
    unsigned long long v = (lane <= upto) ? (s & kMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    prefix += v;
    if (incl) break;
    base -= 32;
  }
  return prefix;
}

// ---------------------------------------------------------------- elementary functions
// DESIGN.md Numerics N1-N4.  Independent implementation of the same op
// sequence the oracle uses; __fmaf_rn only where the definition says fma.
// exp_s on [-87, 0] where the result is normal (the blend's power range), in 13 instructions:
// s = t + 1.5 2^23 rounds t to the nearest integer n (ties to even, |t| < 2^22) and holds n in its low
// mantissa bits, so bits(s) << 23 = n << 23 (mod 2^32); multiplying the polynomial by 2^n is then an
// integer add into its exponent field, exact while the product is normal.  Same bits as exp_s there.
__device__ __forceinline__ float exp_blend(float x) {
  const float log2e = 1.44269502162933349609375f;
  const float ln2_hi = 0.693145751953125f;
  const float ln2_lo = 1.428606765330187045037746429443359375e-06f;
  const float magic = 12582912.0f;   // 1.5 * 2^23
  const float s = __fadd_rn(__fmul_rn(x, log2e), magic);
  const float n = __fsub_rn(s, magic);
  float r = __fmaf_rn(-n, ln2_hi, x);
  r = __fmaf_rn(-n, ln2_lo, r);
  float p = 1.98412698e-04f;
  p = __fmaf_rn(p, r, 1.38888889e-03f);
  p = __fmaf_rn(p, r, 8.33333377e-03f);
  p = __fmaf_rn(p, r, 4.16666679e-02f);
  p = __fmaf_rn(p, r, 1.66666672e-01f);
  p = __fmaf_rn(p, r, 0.5f);
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  return __uint_as_float(__float_as_uint(p) + (__float_as_uint(s) << 23));
}

__device__ __forceinline__ float exp_s(float x) {
  if (x != x) return x;
  if (x > 88.72283935546875f) return __int_as_float(0x7F800000);
  if (x < -87.33654022216797f) return 0.0f;
  const float log2e = 1.44269502162933349609375f;
  const float ln2_hi = 0.693145751953125f;
  const float ln2_lo = 1.428606765330187045037746429443359375e-06f;
  float n = rintf(__fmul_rn(x, log2e));
  float r = __fmaf_rn(-n, ln2_hi, x);
  r = __fmaf_rn(-n, ln2_lo, r);
  float p = 1.98412698e-04f;
  p = __fmaf_rn(p, r, 1.38888889e-03f);
  p = __fmaf_rn(p, r, 8.33333377e-03f);
  p = __fmaf_rn(p, r, 4.16666679e-02f);
  p = __fmaf_rn(p, r, 1.66666672e-01f);
  p = __fmaf_rn(p, r, 0.5f);
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  int ni = __float2int_rz(n);
  if (ni > 127) return __fmul_rn(__fmul_rn(p, __uint_as_float(0x7F000000u)), 2.0f);
  return __fmul_rn(p, __uint_as_float((uint32_t)(ni + 127) << 23));
}

__device__ __forceinline__ float log_s(float x) {
  if (x != x) return x;
  if (x < 0.0f) return __int_as_float(0x7FC00000);
  if (x == 0.0f) return __int_as_float(0xFF800000);
  if (x == __int_as_float(0x7F800000)) return x;
  uint32_t b = __float_as_uint(x);
  int k = 0;
  if (b < 0x00800000u) { x = __fmul_rn(x, 8388608.0f); b = __float_as_uint(x); k = -23; }
  k += (int)(b >> 23) - 127;
  float m = __uint_as_float((b & 0x007FFFFFu) | 0x3F800000u);
  if (m > 1.41421353816986083984375f) { m = __fmul_rn(m, 0.5f); k += 1; }
  float f = __fsub_rn(m, 1.0f);
  float s = __fdiv_rn(f, __fadd_rn(2.0f, f));
  float z = __fmul_rn(s, s);
  float R = __fmaf_rn(z, 0.222222222f, 0.285714298f);
  R = __fmaf_rn(z, R, 0.400000006f);
  R = __fmaf_rn(z, R, 0.666666687f);
  R = __fmul_rn(z, R);
  float hfsq = __fmul_rn(0.5f, __fmul_rn(f, f));
  float dk = __int2float_rn(k);
  const float ln2_hi = 0.693145751953125f;
  const float ln2_lo = 1.428606765330187045037746429443359375e-06f;
  float inner = __fadd_rn(__fmul_rn(s, __fadd_rn(hfsq, R)), __fmul_rn(dk, ln2_lo));
  float lg = __fsub_rn(f, __fsub_rn(hfsq, inner));
  return __fadd_rn(__fmul_rn(dk, ln2_hi), lg);
}

__device__ __forceinline__ float tanh_s(float x) {
  if (x != x) return x;
  float a = fabsf(x);
  float r;
  if (a < 0.5f) {
    float z = __fmul_rn(a, a);
    float p = 5.90027440e-04f;
    p = __fmaf_rn(p, z, -1.45583438e-03f);
    p = __fmaf_rn(p, z, 3.59212872e-03f);
    p = __fmaf_rn(p, z, -8.86323553e-03f);
    p = __fmaf_rn(p, z, 2.18694885e-02f);
    p = __fmaf_rn(p, z, -5.39682540e-02f);
    p = __fmaf_rn(p, z, 1.33333340e-01f);
    p = __fmaf_rn(p, z, -3.33333343e-01f);
    r = __fmaf_rn(__fmul_rn(a, z), p, a);
  } else {
    float e = exp_s(__fmul_rn(2.0f, a));
    r = __fsub_rn(1.0f, __fdiv_rn(2.0f, __fadd_rn(e, 1.0f)));
  }
  return copysignf(r, x);
}

__device__ __forceinline__ float sigmoid_s(float x) {
  return __fdiv_rn(1.0f, __fadd_rn(1.0f, exp_s(-x)));
}

// Packed fp32x2 helpers (sm_100a FADD2 / FMUL2 / FFMA2: two IEEE fp32 operations per instruction, each
// element rounded exactly as the scalar __fadd_rn / __fmul_rn / __fmaf_rn; a scalar operand is broadcast
// by the hardware, so a splat-pair or pixel constant costs no move).
struct f2p { unsigned long long r; };
__device__ __forceinline__ f2p pk2(float a, float b) {
  f2p o; asm("mov.b64 %0, {%1, %2};" : "=l"(o.r) : "f"(a), "f"(b)); return o;
}
__device__ __forceinline__ void up2(f2p x, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x.r));
}
__device__ __forceinline__ f2p add2(f2p a, f2p b) { f2p o; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r)); return o; }
__device__ __forceinline__ f2p mul2(f2p a, f2p b) { f2p o; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r)); return o; }
__device__ __forceinline__ f2p fma2(f2p a, f2p b, f2p c) {
  f2p o; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(o.r) : "l"(a.r), "l"(b.r), "l"(c.r)); return o;
}
__device__ __forceinline__ f2p bc2(float a) { return pk2(a, a); }
// exact dot product in the written order ((a0 b0 + a1 b1) + a2 b2)
__device__ __forceinline__ float dot3(float a0, float a1, float a2, const float *b) {
  return __fadd_rn(__fadd_rn(__fmul_rn(a0, b[0]), __fmul_rn(a1, b[1])), __fmul_rn(a2, b[2]));
}

// floor(log2(x)) of a positive finite or infinite float, from its bits
__device__ __forceinline__ int ilogb_bits(float x) {
  uint32_t b = __float_as_uint(x) & 0x7FFFFFFFu;
  if (b >= 0x7F800000u) return 0x7FFFFFFF;                // inf / nan
  if (b >= 0x00800000u) return (int)(b >> 23) - 127;      // normal
  return -127 - (__clz(b) - 9);                           // subnormal: 2^-126 * 0.m
}

// ---- constants of the extent / tile test / blend (R14, N5-N7) ----
constexpr float kKappa = 1.0009765625f;   // 1 + 2^-10
constexpr float kSlack = 0.015625f;       // 2^-6
constexpr float kAlphaMin = 0.0039215688593685626983642578125f;  // fp32(1/255)

}  // namespace gsc
