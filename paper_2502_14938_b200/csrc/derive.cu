// derive.cu -- SURVEY §8(a) row a3: derivation of the cache misses.
//
// Eq. 3: {mu_j, Sigma_j, c_j, alpha_j} = MLP_theta(f_i, d_view),
// three heads (opacity, colour, covariance; reading R3), each
// Linear(35->32) - ReLU - Linear(32->n), the three layer-1s fused into one
// 35x96 contraction ("fuses two layers into a single fused Matmul").
// Exact-integer grid formulation (R3/R6): int8 codes, layer-1 and layer-2
// accumulate exactly in int32, one RNE conversion o = fp32(z2) * 2^-21 -- so
// any summation order reproduces the oracle bit for bit.  Two kernels:
//
//  derive_mma_kernel (default): the contractions on the 5th-gen tensor cores.
//    128 anchors per CTA tile (M = 128), one CTA per SM owning all 512 TMEM
//    columns.  Layer 1: 2 x tcgen05.mma.kind::i8 (K = 64 bytes, N = 96,
//    s8 x s8 -> s32) into TMEM.  Epilogue 1 (tcgen05.ld): + bias, ReLU, split
//    into 3 unsigned byte limbs (hidden < 2^24, checked at load).  Layer 2:
//    per head h and limb l one tcgen05.mma (u8 x s8, K = 32, N = 16/32/80),
//    9 accumulators; z2 = sum_l 256^l D_{h,l} + 2^14 b2 in int32.  Operands
//    are staged in SMEM in the canonical no-swizzle K-major layout (8-row x
//    16-byte core matrices), MMAs issued by one thread, completion through
//    tcgen05.commit -> mbarrier.
//  derive_kernel (GSC_F_DERIVE_CUDA_CORES): the same integers by dp4a/IMAD.
//  derive_f32_kernel: the real-weights path (F4): fixed-order fp32 on the CUDA cores (below).
//
// Epilogue (Eq. 2), one thread per (anchor, Gaussian):
//   alpha = tanh_s (kept if > 0), rgb = sigmoid_s, S = s (.) sigmoid_s,
//   q normalised, Sigma = (R S)(R S)^T, mu = p + O (.) s.
// "precomputing mask indices": dead slots are written with alpha = 0
// and skipped by the projection's 4-byte alpha read.
//
// Output: the persistent Gaussian pool, direct-mapped slot g = i*K + j
// ("index mapping"): alpha f32[N*K] and pool float4[N*K][3] =
//   (mu.x mu.y mu.z S00) (S01 S02 S11 S12) (S22 r g b).
#include "gsc_internal.cuh"

namespace gsc {

// ------------------------------------------------------------------ shared pieces
// quantised view direction codes of anchor i (R3): q_k = clamp(rint(128 v_k/|v|), -127, 127)
__device__ __forceinline__ uint32_t view_codes(float4 pm, float pu0, float pu1, float pu2) {
  float v0 = __fsub_rn(pm.x, pu0), v1 = __fsub_rn(pm.y, pu1), v2 = __fsub_rn(pm.z, pu2);
  float n = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(v0, v0), __fmul_rn(v1, v1)), __fmul_rn(v2, v2)));
  float vv[3] = {v0, v1, v2};
  uint32_t w = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float dv = (n == 0.0f) ? 0.0f : __fdiv_rn(vv[k], n);
    int c = __float2int_rn(__fmul_rn(128.0f, dv));
    c = c < -127 ? -127 : (c > 127 ? 127 : c);
    w |= (uint32_t)(c & 0xFF) << (8 * k);
  }
  return w;
}

// Gaussian j of anchor i from its 110 layer-2 outputs oo (alpha K | colour 3K | cov 7K)
__device__ __forceinline__ void derive_gaussian(const float *oo, int j, uint32_t i, const float4 *__restrict__ pos_m,
                                                const float *__restrict__ offs, const float *__restrict__ scale,
                                                float *__restrict__ alpha, float4 *__restrict__ pool) {
  float al = tanh_s(oo[j]);
  float alive = al > 0.0f ? al : 0.0f;
  float rgb[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) rgb[k] = sigmoid_s(oo[kK + 3 * j + k]);
  const float *os = oo + 4 * kK + 7 * j;
  float s0 = scale[3 * i], s1 = scale[3 * i + 1], s2 = scale[3 * i + 2];
  float Sc[3] = {__fmul_rn(s0, sigmoid_s(os[0])), __fmul_rn(s1, sigmoid_s(os[1])), __fmul_rn(s2, sigmoid_s(os[2]))};
  float qw = os[3], qx = os[4], qy = os[5], qz = os[6];
  float qn2 = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(qw, qw), __fmul_rn(qx, qx)), __fmul_rn(qy, qy)),
                        __fmul_rn(qz, qz));
  if (qn2 == 0.0f) {
    qw = 1.0f; qx = qy = qz = 0.0f;
  } else {
    float qn = __fsqrt_rn(qn2);
    qw = __fdiv_rn(qw, qn); qx = __fdiv_rn(qx, qn); qy = __fdiv_rn(qy, qn); qz = __fdiv_rn(qz, qn);
  }
  float R[3][3];
  R[0][0] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fadd_rn(__fmul_rn(qy, qy), __fmul_rn(qz, qz))));
  R[0][1] = __fmul_rn(2.0f, __fsub_rn(__fmul_rn(qx, qy), __fmul_rn(qw, qz)));
  R[0][2] = __fmul_rn(2.0f, __fadd_rn(__fmul_rn(qx, qz), __fmul_rn(qw, qy)));
  R[1][0] = __fmul_rn(2.0f, __fadd_rn(__fmul_rn(qx, qy), __fmul_rn(qw, qz)));
  R[1][1] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fadd_rn(__fmul_rn(qx, qx), __fmul_rn(qz, qz))));
  R[1][2] = __fmul_rn(2.0f, __fsub_rn(__fmul_rn(qy, qz), __fmul_rn(qw, qx)));
  R[2][0] = __fmul_rn(2.0f, __fsub_rn(__fmul_rn(qx, qz), __fmul_rn(qw, qy)));
  R[2][1] = __fmul_rn(2.0f, __fadd_rn(__fmul_rn(qy, qz), __fmul_rn(qw, qx)));
  R[2][2] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fadd_rn(__fmul_rn(qx, qx), __fmul_rn(qy, qy))));
  float Mm[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) Mm[r][c] = __fmul_rn(R[r][c], Sc[c]);
  float cv[6];
  const int ia[6] = {0, 0, 0, 1, 1, 2}, ib[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
  for (int q = 0; q < 6; ++q) cv[q] = dot3(Mm[ia[q]][0], Mm[ia[q]][1], Mm[ia[q]][2], Mm[ib[q]]);
  float4 pm = pos_m[i];
  const float *oj = offs + (size_t)i * kK * 3 + 3 * j;
  float mu0 = __fadd_rn(pm.x, __fmul_rn(oj[0], s0));
  float mu1 = __fadd_rn(pm.y, __fmul_rn(oj[1], s1));
  float mu2 = __fadd_rn(pm.z, __fmul_rn(oj[2], s2));
  size_t g = (size_t)i * kK + j;
  alpha[g] = alive;
  pool[3 * g + 0] = make_float4(mu0, mu1, mu2, cv[0]);
  pool[3 * g + 1] = make_float4(cv[1], cv[2], cv[3], cv[4]);
  pool[3 * g + 2] = make_float4(cv[5], rgb[0], rgb[1], rgb[2]);
}

struct DeriveArgs {
  float pu0, pu1, pu2;
  const uint32_t *misses;
  const float4 *pos_m;
  const int8_t *feat;
  const float *offs, *scale;
  const int8_t *W1T;     // [96][36] (n-major, k contiguous, k = 35 zero)
  const int32_t *b1s;    // 128 * b1
  const int8_t *W2T;     // [110][32] (m-major, heads concatenated 10 | 30 | 70)
  const int32_t *b2s;    // 16384 * b2
  float *alpha;
  float4 *pool;
  FrameCounters *ctr;
};

// ------------------------------------------------------------------ CUDA-core kernel (dp4a)
constexpr int kDThreads = 256;
constexpr int kDA = 64;          // anchors per CTA iteration

struct DeriveSmem {
  int32_t W1w[96][9];            // [n][k/4] int8x4, k = 0..34 (+1 zero pad)
  int32_t b1s[96];
  int32_t W2w[kNOut][8];         // [m][u/4] int8x4
  int32_t b2s[kNOut];
  int32_t xw[kDA][9];            // input codes
  int32_t hid[kDA][96];          // ReLU(z1)
  float o[kDA][kNOut + 1];       // layer-2 outputs
  uint32_t anchor[kDA];
  uint32_t base;
};

__device__ __forceinline__ int sx8(int32_t w, int b) { return (int)(int8_t)((uint32_t)w >> (8 * b)); }

__global__ void __launch_bounds__(kDThreads) derive_kernel(DeriveArgs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DeriveSmem &S = *reinterpret_cast<DeriveSmem *>(smem_raw);
  const int t = threadIdx.x;
  for (int w = t; w < 96 * 9; w += kDThreads) S.W1w[w / 9][w % 9] = reinterpret_cast<const int32_t *>(p.W1T)[w];
  for (int w = t; w < 96; w += kDThreads) S.b1s[w] = p.b1s[w];
  for (int w = t; w < kNOut * 8; w += kDThreads) S.W2w[w / 8][w % 8] = reinterpret_cast<const int32_t *>(p.W2T)[w];
  for (int w = t; w < kNOut; w += kDThreads) S.b2s[w] = p.b2s[w];
  const uint32_t M = p.ctr->n_miss;

  for (;;) {
    __syncthreads();
    if (t == 0) S.base = atomicAdd(&p.ctr->tile_derive, 1u) * kDA;
    __syncthreads();
    const uint32_t base = S.base;
    if (base >= M) break;
    const int na = min((uint32_t)kDA, M - base);
    if (t < kDA) {
      uint32_t i = t < na ? p.misses[base + t] : 0u;
      S.anchor[t] = i;
      S.xw[t][8] = t < na ? view_codes(p.pos_m[i], p.pu0, p.pu1, p.pu2) : 0u;
    }
    for (int w = t; w < kDA * 8; w += kDThreads) {
      int a = w >> 3;
      S.xw[a][w & 7] = a < na ? reinterpret_cast<const int32_t *>(p.feat)[(size_t)p.misses[base + a] * 8 + (w & 7)] : 0;
    }
    __syncthreads();
    for (int o = t; o < kDA * 96; o += kDThreads) {
      int a = o / 96, n = o - a * 96;
      int acc = S.b1s[n];
#pragma unroll
      for (int w = 0; w < 9; ++w) acc = __dp4a(S.xw[a][w], S.W1w[n][w], acc);
      S.hid[a][n] = acc > 0 ? acc : 0;
    }
    __syncthreads();
    for (int o = t; o < kDA * kNOut; o += kDThreads) {
      int a = o / kNOut, m = o - a * kNOut;
      int h = m < kK ? 0 : (m < 4 * kK ? 1 : 2);
      const int32_t *hp = &S.hid[a][h * 32];
      int acc = S.b2s[m];
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        int32_t ww = S.W2w[m][w];
        acc += sx8(ww, 0) * hp[4 * w] + sx8(ww, 1) * hp[4 * w + 1] + sx8(ww, 2) * hp[4 * w + 2] +
               sx8(ww, 3) * hp[4 * w + 3];
      }
      S.o[a][m] = __fmul_rn(__int2float_rn(acc), 4.76837158203125e-07f);
    }
    __syncthreads();
    for (int e = t; e < na * kK; e += kDThreads) {
      int a = e / kK, j = e - a * kK;
      derive_gaussian(S.o[a], j, S.anchor[a], p.pos_m, p.offs, p.scale, p.alpha, p.pool);
    }
  }
}

// ------------------------------------------------------------------ real-weights kernel (F4, fp32)
// MLP_theta(f_i, d_view) (Eq. 3) with trained-style fp32 weights, the
// continuous view direction d_view = v / |v| (v = p_i - p_u, three IEEE divisions, 0 at the camera),
// and the fixed summation order of DESIGN.md F4 -- every output from its bias, inputs in ascending
// index order, one fma per term -- so the CUDA cores reproduce the oracle's orc_mlp_f32 bit for bit.
// (A tensor-core contraction would change the rounding: tf32 / bf16 operands are not fp32, and the
// MMA's accumulation order is not the written one.)  64 anchors per CTA iteration: layer 1 as
// 64 x 96 outputs (thread = (anchor, hidden unit), weights W1[k][n] read conflict-free across n,
// inputs broadcast), layer 2 as 64 x 110 outputs, then the shared epilogue (derive_gaussian).
// R32 combine inputs (kDist / kBank, F4-B; "first combine operator"): the distance
// |p_i - p_u| as the 36th input, and the feature bank -- one thread per anchor evaluates the bank MLP
// (4 -> 32 -> 3, softmax), then the blended features fh_k = fma(w2, f_k, fma(w1, f_{2 (k mod 16)},
// w0 f_{4 (k mod 8)})) are formed in SMEM by index arithmetic (no copies of the feature rows).
struct DeriveF32Args {
  float pu0, pu1, pu2;
  const uint32_t *misses;
  const float4 *pos_m;
  const float *feat;     // [N][32]
  const float *offs, *scale;
  const float *W1;       // [35][96]
  const float *b1;       // [96]
  const float *W2;       // [32][110] (heads side by side: alpha 0..9 | colour 10..39 | covariance 40..109)
  const float *b2;       // [110]
  CombineF32 cmb;
  float *alpha;
  float4 *pool;
  FrameCounters *ctr;
};

constexpr int kFA = 64;   // anchors per CTA iteration

struct DeriveF32Smem {
  float W1[kF + 4][96];      // (row kF + 3: the distance input, R32)
  float b1[96];
  float W2[kH][kNOut];
  float b2[kNOut];
  float Wb1[4][kF], bb1[kF], Wb2[kF][3], bb2[3];   // R32 feature bank
  float x[kFA][kF + 4];      // inputs (32 features, d_view, distance)
  float fr[kFA][kF + 1];     // raw features (feature bank)
  float wb[kFA][3];          // bank weights
  float hid[kFA][96 + 1];
  float o[kFA][kNOut + 1];
  uint32_t anchor[kFA];
  uint32_t base;
};

template <bool kDist, bool kBank>
__global__ void __launch_bounds__(kDThreads) derive_f32_kernel(DeriveF32Args p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DeriveF32Smem &S = *reinterpret_cast<DeriveF32Smem *>(smem_raw);
  const int t = threadIdx.x;
  constexpr int kNin = kF + 3 + (kDist ? 1 : 0);
  for (int w = t; w < kNin * 96; w += kDThreads) (&S.W1[0][0])[w] = p.W1[w];
  if (kBank) {
    for (int w = t; w < 4 * kF; w += kDThreads) (&S.Wb1[0][0])[w] = p.cmb.Wb1[w];
    for (int w = t; w < kF * 3; w += kDThreads) (&S.Wb2[0][0])[w] = p.cmb.Wb2[w];
    for (int w = t; w < kF; w += kDThreads) S.bb1[w] = p.cmb.bb1[w];
    for (int w = t; w < 3; w += kDThreads) S.bb2[w] = p.cmb.bb2[w];
  }
  for (int w = t; w < 96; w += kDThreads) S.b1[w] = p.b1[w];
  for (int w = t; w < kH * kNOut; w += kDThreads) (&S.W2[0][0])[w] = p.W2[w];
  for (int w = t; w < kNOut; w += kDThreads) S.b2[w] = p.b2[w];
  const uint32_t M = p.ctr->n_miss;
  for (;;) {
    __syncthreads();
    if (t == 0) S.base = atomicAdd(&p.ctr->tile_derive, 1u) * kFA;
    __syncthreads();
    const uint32_t base = S.base;
    if (base >= M) break;
    const int na = min((uint32_t)kFA, M - base);
    if (t < kFA) {
      const uint32_t i = t < na ? p.misses[base + t] : 0u;
      S.anchor[t] = i;
      const float4 pm = p.pos_m[i];
      const float v0 = __fsub_rn(pm.x, p.pu0), v1 = __fsub_rn(pm.y, p.pu1), v2 = __fsub_rn(pm.z, p.pu2);
      const float n = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(v0, v0), __fmul_rn(v1, v1)), __fmul_rn(v2, v2)));
      const float d0 = n == 0.0f ? 0.0f : __fdiv_rn(v0, n);
      const float d1 = n == 0.0f ? 0.0f : __fdiv_rn(v1, n);
      const float d2 = n == 0.0f ? 0.0f : __fdiv_rn(v2, n);
      S.x[t][kF + 0] = d0;
      S.x[t][kF + 1] = d1;
      S.x[t][kF + 2] = d2;
      S.x[t][kF + 3] = n;   // R32 distance input (read by layer 1 only with kDist)
      if (kBank) {
        // bank MLP (R32, the oracle's orc_bank_weights order): h = ReLU(bb1 + Wb1^T y), z = bb2 + Wb2^T h,
        // w = softmax(z) with the max subtracted
        const float y[4] = {d0, d1, d2, n};
        float z0 = S.bb2[0], z1 = S.bb2[1], z2 = S.bb2[2];
#pragma unroll 4
        for (int c = 0; c < kF; ++c) {
          float acc = S.bb1[c];
#pragma unroll
          for (int k = 0; k < 4; ++k) acc = __fmaf_rn(S.Wb1[k][c], y[k], acc);
          const float h = acc > 0.0f ? acc : 0.0f;
          z0 = __fmaf_rn(S.Wb2[c][0], h, z0);
          z1 = __fmaf_rn(S.Wb2[c][1], h, z1);
          z2 = __fmaf_rn(S.Wb2[c][2], h, z2);
        }
        const float zm = fmaxf(fmaxf(z0, z1), z2);
        const float e0 = exp_s(__fsub_rn(z0, zm)), e1 = exp_s(__fsub_rn(z1, zm)), e2 = exp_s(__fsub_rn(z2, zm));
        const float sum = __fadd_rn(__fadd_rn(e0, e1), e2);
        S.wb[t][0] = __fdiv_rn(e0, sum);
        S.wb[t][1] = __fdiv_rn(e1, sum);
        S.wb[t][2] = __fdiv_rn(e2, sum);
      }
    }
    for (int w = t; w < kFA * (kF / 4); w += kDThreads) {   // features: one float4 per thread
      const int a = w / (kF / 4), c4 = w % (kF / 4);
      const float4 f = a < na ? reinterpret_cast<const float4 *>(p.feat)[(size_t)p.misses[base + a] * (kF / 4) + c4]
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      float *dst = kBank ? &S.fr[a][4 * c4] : &S.x[a][4 * c4];
      dst[0] = f.x; dst[1] = f.y; dst[2] = f.z; dst[3] = f.w;
    }
    __syncthreads();
    if (kBank) {   // blended features (strides 4, 2, 1), fixed fma order
      for (int w = t; w < kFA * kF; w += kDThreads) {
        const int a = w / kF, k = w % kF;
        const float *fr = S.fr[a];
        S.x[a][k] = __fmaf_rn(S.wb[a][2], fr[k], __fmaf_rn(S.wb[a][1], fr[2 * (k % (kF / 2))],
                                                           __fmul_rn(S.wb[a][0], fr[4 * (k % (kF / 4))])));
      }
      __syncthreads();
    }
    for (int o = t; o < kFA * 96; o += kDThreads) {
      const int a = o / 96, n = o - a * 96;
      float acc = S.b1[n];
#pragma unroll
      for (int k = 0; k < kNin; ++k) acc = __fmaf_rn(S.W1[k][n], S.x[a][k], acc);
      S.hid[a][n] = acc > 0.0f ? acc : 0.0f;   // ReLU
    }
    __syncthreads();
    for (int o = t; o < kFA * kNOut; o += kDThreads) {
      const int a = o / kNOut, m = o - a * kNOut;
      const int h = m < kK ? 0 : (m < 4 * kK ? 1 : 2);
      const float *hp = &S.hid[a][h * kH];
      float acc = S.b2[m];
#pragma unroll
      for (int u = 0; u < kH; ++u) acc = __fmaf_rn(S.W2[u][m], hp[u], acc);
      S.o[a][m] = acc;
    }
    __syncthreads();
    for (int e = t; e < na * kK; e += kDThreads) {
      const int a = e / kK, j = e - a * kK;
      derive_gaussian(S.o[a], j, S.anchor[a], p.pos_m, p.offs, p.scale, p.alpha, p.pool);
    }
  }
}

// ------------------------------------------------------------------ tensor-core kernel (tcgen05, kind::i8)
constexpr int kMThreads = 512;
constexpr int kMA = 128;                 // anchors per tile = UMMA M
constexpr int kTmemCols = 512;
// TMEM column map (32-bit cells): layer-2 accumulators D2[h][l], then D1
__host__ __device__ constexpr int d2_npad(int h) { return h == 0 ? 16 : (h == 1 ? 32 : 80); }
__host__ __device__ constexpr int d2_col(int h, int l) { return h == 0 ? 16 * l : (h == 1 ? 48 + 32 * l : 144 + 80 * l); }
constexpr int kD1Col = 384;

struct MmaSmem {
  // canonical K-major no-swizzle tiles: 8-row x 16-byte core matrices, LBO = 128 B (K chunks),
  // SBO = (#K chunks) * 128 B (8-row groups)
  alignas(128) uint8_t X[kMA * 64];          // layer-1 A: 128 x 64 B (feature 32 | view 3 | 0)
  alignas(128) uint8_t W1[96 * 64];          // layer-1 B: 96 x 64 B
  alignas(128) uint8_t A2[3][kMA * 96];      // layer-2 A limbs: 128 x 96 B (hidden, 3 heads)
  alignas(128) uint8_t W2[128 * 32];         // layer-2 B: head rows 16 | 32 | 80, 32 B each
  float o[kMA][kNOut + 1];                   // layer-2 outputs (odd row stride: the per-row writes of epilogue 2 hit 32 banks)
  int32_t b1s[96];
  int32_t b2s[kNOut];
  uint32_t anchor[kMA];
  uint64_t mbar;
  uint32_t tmem_base;
  uint32_t base;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of (row, k-byte) in a canonical K-major no-swizzle tile with `kchunks` 16-byte chunks per row
__device__ __forceinline__ uint32_t kmaj_off(int row, int kbyte, int kchunks) {
  return (uint32_t)((row & 7) * 16 + (row >> 3) * (kchunks * 128) + (kbyte >> 4) * 128 + (kbyte & 15));
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);   // version 1, base offset 0, no swizzle
}

// instruction descriptor, kind::i8: D s32, A/B signedness, K-major both, N, M = 128
__device__ __forceinline__ uint32_t idesc_i8(int n, bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(kMA >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, int acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(mbar),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__global__ void __launch_bounds__(kMThreads, 1) derive_mma_kernel(DeriveArgs p) {
  extern __shared__ __align__(1024) unsigned char smem_mma[];
  MmaSmem &S = *reinterpret_cast<MmaSmem *>(smem_mma);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;

  // ---- one-time setup: weights into the canonical B layouts, biases, mbarrier, TMEM
  for (int idx = t; idx < 96 * 64; idx += kMThreads) {
    const int n = idx >> 6, kb = idx & 63;
    S.W1[kmaj_off(n, kb, 4)] = kb < 36 ? (uint8_t)p.W1T[n * 36 + kb] : 0;
  }
  for (int idx = t; idx < 128 * 32; idx += kMThreads) {
    const int r = idx >> 5, kb = idx & 31;       // padded output row r (head blocks 16 | 32 | 80), hidden kb
    int h, m;
    if (r < 16) { h = 0; m = r; } else if (r < 48) { h = 1; m = r - 16; } else { h = 2; m = r - 48; }
    const int nh = h == 0 ? kK : (h == 1 ? 3 * kK : 7 * kK);
    const int mo = (h == 0 ? 0 : (h == 1 ? kK : 4 * kK)) + m;
    const int hbase = h == 0 ? 0 : (h == 1 ? 16 : 48);
    S.W2[hbase * 32 + kmaj_off(m, kb, 2)] = m < nh ? (uint8_t)p.W2T[mo * 32 + kb] : 0;
  }
  for (int idx = t; idx < 96; idx += kMThreads) S.b1s[idx] = p.b1s[idx];
  for (int idx = t; idx < kNOut; idx += kMThreads) S.b2s[idx] = p.b2s[idx];
  const uint32_t mbar = smem_u32(&S.mbar);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  const uint32_t M = p.ctr->n_miss;
  uint32_t phase = 0;
  const uint32_t sX = smem_u32(S.X), sW1 = smem_u32(S.W1), sW2 = smem_u32(S.W2);

  for (;;) {
    if (t == 0) S.base = atomicAdd(&p.ctr->tile_derive, 1u) * kMA;
    __syncthreads();
    const uint32_t base = S.base;
    if (base >= M) break;
    const int na = min((uint32_t)kMA, M - base);

    // ---- A tile of layer 1: row a = [32 feature codes | 3 view codes | 0...] (64 B)
    if (t < kMA) {
      uint4 f0 = make_uint4(0, 0, 0, 0), f1 = f0, f2 = f0;
      uint32_t i = 0;
      if (t < na) {
        i = p.misses[base + t];
        const uint4 *fp = reinterpret_cast<const uint4 *>(p.feat + (size_t)i * kF);
        f0 = fp[0];
        f1 = fp[1];
        f2.x = view_codes(p.pos_m[i], p.pu0, p.pu1, p.pu2);
      }
      S.anchor[t] = i;
      *reinterpret_cast<uint4 *>(&S.X[kmaj_off(t, 0, 4)]) = f0;
      *reinterpret_cast<uint4 *>(&S.X[kmaj_off(t, 16, 4)]) = f1;
      *reinterpret_cast<uint4 *>(&S.X[kmaj_off(t, 32, 4)]) = f2;
      *reinterpret_cast<uint4 *>(&S.X[kmaj_off(t, 48, 4)]) = make_uint4(0, 0, 0, 0);
    }
    fence_async_smem();
    __syncthreads();

    // ---- layer 1 on the tensor core: D1[128 x 96] = X[128 x 64] W1^T  (2 K-steps of 32 bytes)
    if (t == 0) {
      tc_fence_after();
      const uint32_t id = idesc_i8(96, true, true);
#pragma unroll
      for (int s = 0; s < 2; ++s)
        mma_i8(tmem + kD1Col, umma_desc(sX + 256 * s, 128, 512), umma_desc(sW1 + 256 * s, 128, 512), id, s);
      mma_commit(mbar);
    }
    mbar_wait(mbar, phase);
    phase ^= 1;
    tc_fence_after();

    // ---- epilogue 1 (all 16 warps: warp w reads TMEM lane quarter w % 4 -- the quarter tcgen05.ld allows
    // it -- and the 16-column chunks c = w / 4, w / 4 + 4): bias, ReLU, byte limbs -> layer-2 A tiles
    {
      const int q = warp & 3, row = q * 32 + lane;
      const uint32_t lane_base = (uint32_t)(q * 32) << 16;
#pragma unroll 1
      for (int c = warp >> 2; c < 6; c += 4) {   // 16 hidden units per chunk
        uint32_t r[16];
        tmem_ld16(tmem + lane_base + kD1Col + 16 * c, r);
        tmem_wait_ld();
        uint32_t w0[4] = {0, 0, 0, 0}, w1[4] = {0, 0, 0, 0}, w2[4] = {0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          int z = (int)r[k] + S.b1s[16 * c + k];
          uint32_t h = z > 0 ? (uint32_t)z : 0u;
          w0[k >> 2] |= (h & 0xFFu) << (8 * (k & 3));
          w1[k >> 2] |= ((h >> 8) & 0xFFu) << (8 * (k & 3));
          w2[k >> 2] |= ((h >> 16) & 0xFFu) << (8 * (k & 3));
        }
        const uint32_t off = kmaj_off(row, 16 * c, 6);
        *reinterpret_cast<uint4 *>(&S.A2[0][off]) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
        *reinterpret_cast<uint4 *>(&S.A2[1][off]) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
        *reinterpret_cast<uint4 *>(&S.A2[2][off]) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
      }
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();

    // ---- layer 2: per head h (K = its 32 hidden units) and limb l: D2[h][l] = A2_l[:, 32h:32h+32] W2_h^T
    if (t == 0) {
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 3; ++h) {
        const uint32_t id = idesc_i8(d2_npad(h), false, true);
        const uint32_t bdesc_addr = sW2 + (h == 0 ? 0 : (h == 1 ? 16 : 48)) * 32;
#pragma unroll
        for (int l = 0; l < 3; ++l)
          mma_i8(tmem + d2_col(h, l), umma_desc(smem_u32(S.A2[l]) + 256 * h, 128, 768), umma_desc(bdesc_addr, 128, 256),
                 id, 0);
      }
      mma_commit(mbar);
    }
    mbar_wait(mbar, phase);
    phase ^= 1;
    tc_fence_after();

    // ---- epilogue 2 (all 16 warps, lane quarter w % 4, the 8 column chunks of the three heads -- 1 | 2 | 5
    // of 16 -- dealt round-robin to the quarter's 4 warps): z2 = sum_l 256^l D2[h][l] + 2^14 b2;
    // o = fp32(z2) 2^-21 -> SMEM
    {
      const int q = warp & 3, row = q * 32 + lane;
      const uint32_t lane_base = (uint32_t)(q * 32) << 16;
#pragma unroll 1
      for (int ck = warp >> 2; ck < 8; ck += 4) {
        const int h = ck == 0 ? 0 : (ck < 3 ? 1 : 2);
        const int c = 16 * (ck == 0 ? 0 : (ck < 3 ? ck - 1 : ck - 3));
        const int nh = h == 0 ? kK : (h == 1 ? 3 * kK : 7 * kK);
        const int mo = h == 0 ? 0 : (h == 1 ? kK : 4 * kK);
        {
          uint32_t r0[16], r1[16], r2[16];
          tmem_ld16(tmem + lane_base + d2_col(h, 0) + c, r0);
          tmem_ld16(tmem + lane_base + d2_col(h, 1) + c, r1);
          tmem_ld16(tmem + lane_base + d2_col(h, 2) + c, r2);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int m = c + k;
            if (m < nh) {
              // modular (two's complement) sum: exact because the true z2 fits int32 (load-time bound)
              const int z = (int)(r0[k] + (r1[k] << 8) + (r2[k] << 16) + (uint32_t)S.b2s[mo + m]);
              S.o[row][mo + m] = __fmul_rn(__int2float_rn(z), 4.76837158203125e-07f);
            }
          }
        }
      }
    }
    tc_fence_before();
    __syncthreads();

    // ---- Gaussian epilogue: 128 x 10 Gaussians over all 256 threads
    for (int e = t; e < na * kK; e += kMThreads) {
      const int a = e / kK, j = e - a * kK;
      derive_gaussian(S.o[a], j, S.anchor[a], p.pos_m, p.offs, p.scale, p.alpha, p.pool);
    }
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
  }
}

static PerDevice<int> g_mma_grid, g_derive_grid, g_f32_grid;

void launch_derive_f32(const float pu[3], const uint32_t *misses, const float4 *pos_m, const float *feat,
                       const float *offs, const float *scale, const float *W1, const float *b1, const float *W2,
                       const float *b2, const CombineF32 &cmb, float *alpha, float4 *pool, FrameCounters *ctr,
                       int num_sms, cudaStream_t st) {
  DeriveF32Args a{pu[0], pu[1], pu[2], misses, pos_m, feat, offs, scale, W1, b1, W2, b2, cmb, alpha, pool, ctr};
  const int smem = (int)sizeof(DeriveF32Smem);
  const int grid = g_f32_grid.get([&](int &grid) {
    cudaFuncSetAttribute(derive_f32_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(derive_f32_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(derive_f32_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(derive_f32_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, derive_f32_kernel<true, true>, kDThreads, smem);
    grid = num_sms * (per_sm > 0 ? per_sm : 1);
  });
  if (cmb.dist && cmb.bank) derive_f32_kernel<true, true><<<grid, kDThreads, smem, st>>>(a);
  else if (cmb.dist) derive_f32_kernel<true, false><<<grid, kDThreads, smem, st>>>(a);
  else if (cmb.bank) derive_f32_kernel<false, true><<<grid, kDThreads, smem, st>>>(a);
  else derive_f32_kernel<false, false><<<grid, kDThreads, smem, st>>>(a);
}

void launch_derive(const float pu[3], const uint32_t *misses, const float4 *pos_m, const int8_t *feat,
                   const float *offs, const float *scale, const int8_t *W1T, const int32_t *b1s, const int8_t *W2T,
                   const int32_t *b2s, float *alpha, float4 *pool, FrameCounters *ctr, int num_sms, bool use_mma,
                   cudaStream_t st) {
  DeriveArgs a{pu[0], pu[1], pu[2], misses, pos_m, feat, offs, scale, W1T, b1s, W2T, b2s, alpha, pool, ctr};
  if (use_mma) {
    const int smem = (int)sizeof(MmaSmem) + 1024;
    const int grid = g_mma_grid.get([&](int &grid) {
      cudaFuncSetAttribute(derive_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      grid = num_sms;   // one CTA per SM: each owns all 512 TMEM columns
    });
    derive_mma_kernel<<<grid, kMThreads, smem, st>>>(a);
    return;
  }
  const int smem = (int)sizeof(DeriveSmem);
  const int grid = g_derive_grid.get([&](int &grid) {
    cudaFuncSetAttribute(derive_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, derive_kernel, kDThreads, smem);
    grid = num_sms * (per_sm > 0 ? per_sm : 1);
  });
  derive_kernel<<<grid, kDThreads, smem, st>>>(a);
}

}  // namespace gsc
