// derive.cu -- SURVEY §8(a) row a3: derivation of the cache misses.
//
// Eq. 3: {mu_j, Sigma_j, c_j, alpha_j} = MLP_theta(f_i, d_view),
// three heads (opacity, colour, covariance; reading R3), each
// Linear(35->32) - ReLU - Linear(32->n), the three layer-1s fused into one
// 35x96 contraction ("fuses two layers into a single fused Matmul").
// Exact-integer grid formulation (R3/R6): int8 codes, layer-1 and layer-2
// accumulate exactly in int32, one RNE conversion o = fp32(z2) * 2^-21 -- so
// any summation order (CUDA cores here, tcgen05 kind::i8 in derive_mma.cu)
// reproduces the oracle bit for bit.  Epilogue (Eq. 2):
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

constexpr int kDThreads = 256;
constexpr int kDA = 64;          // anchors per CTA iteration

struct DeriveSmem {
  int32_t W1w[96][9];            // [n][k/4] int8x4, k = 0..34 (+1 zero pad)
  int32_t b1s[96];               // 128 * b1
  int32_t W2w[kNOut][8];         // [m][u/4] int8x4 (heads concatenated: 10 | 30 | 70)
  int32_t b2s[kNOut];            // 16384 * b2
  int32_t xw[kDA][9];            // input codes
  int32_t hid[kDA][96];          // ReLU(z1)
  float o[kDA][kNOut + 1];       // layer-2 outputs
  uint32_t anchor[kDA];
  uint32_t base;
};

__device__ __forceinline__ int sx8(int32_t w, int b) { return (int)(int8_t)((uint32_t)w >> (8 * b)); }

__global__ void __launch_bounds__(kDThreads)
derive_kernel(float pu0, float pu1, float pu2, const uint32_t *__restrict__ misses,
              const float4 *__restrict__ pos_m, const int8_t *__restrict__ feat,
              const float *__restrict__ offs, const float *__restrict__ scale,
              const int8_t *__restrict__ W1T /* [96][36] */, const int32_t *__restrict__ b1s,
              const int8_t *__restrict__ W2T /* [110][32] */, const int32_t *__restrict__ b2s,
              float *__restrict__ alpha, float4 *__restrict__ pool, FrameCounters *__restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DeriveSmem &S = *reinterpret_cast<DeriveSmem *>(smem_raw);
  const int t = threadIdx.x;
  for (int w = t; w < 96 * 9; w += kDThreads) S.W1w[w / 9][w % 9] = reinterpret_cast<const int32_t *>(W1T)[w];
  for (int w = t; w < 96; w += kDThreads) S.b1s[w] = b1s[w];
  for (int w = t; w < kNOut * 8; w += kDThreads) S.W2w[w / 8][w % 8] = reinterpret_cast<const int32_t *>(W2T)[w];
  for (int w = t; w < kNOut; w += kDThreads) S.b2s[w] = b2s[w];
  const uint32_t M = ctr->n_miss;

  for (;;) {
    __syncthreads();
    if (t == 0) S.base = atomicAdd(&ctr->tile_derive, 1u) * kDA;
    __syncthreads();
    const uint32_t base = S.base;
    if (base >= M) break;
    const int na = min((uint32_t)kDA, M - base);

    // ---- inputs: feature codes and the quantised view direction (R3)
    if (t < kDA) {
      uint32_t i = t < na ? misses[base + t] : 0u;
      S.anchor[t] = i;
      int q[3] = {0, 0, 0};
      if (t < na) {
        float4 pm = pos_m[i];
        float v0 = __fsub_rn(pm.x, pu0), v1 = __fsub_rn(pm.y, pu1), v2 = __fsub_rn(pm.z, pu2);
        float n = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(v0, v0), __fmul_rn(v1, v1)), __fmul_rn(v2, v2)));
        float vv[3] = {v0, v1, v2};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          float dv = (n == 0.0f) ? 0.0f : __fdiv_rn(vv[k], n);
          int c = __float2int_rn(__fmul_rn(128.0f, dv));
          q[k] = c < -127 ? -127 : (c > 127 ? 127 : c);
        }
      }
      S.xw[t][8] = (q[0] & 0xFF) | ((q[1] & 0xFF) << 8) | ((q[2] & 0xFF) << 16);
    }
    for (int w = t; w < kDA * 8; w += kDThreads) {
      int a = w >> 3;
      S.xw[a][w & 7] = a < na ? reinterpret_cast<const int32_t *>(feat)[(size_t)misses[base + a] * 8 + (w & 7)] : 0;
    }
    __syncthreads();

    // ---- layer 1: z1 = W1 x + 128 b1 (exact int32), ReLU
    for (int o = t; o < kDA * 96; o += kDThreads) {
      int a = o / 96, n = o - a * 96;
      int acc = S.b1s[n];
#pragma unroll
      for (int w = 0; w < 9; ++w) acc = __dp4a(S.xw[a][w], S.W1w[n][w], acc);
      S.hid[a][n] = acc > 0 ? acc : 0;
    }
    __syncthreads();

    // ---- layer 2 per head: z2 = W2 a + 2^14 b2 (exact int32); o = fp32(z2) * 2^-21
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

    // ---- epilogue: one thread per (anchor, Gaussian)
    for (int e = t; e < na * kK; e += kDThreads) {
      int a = e / kK, j = e - a * kK;
      uint32_t i = S.anchor[a];
      const float *oo = S.o[a];
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
      for (int q = 0; q < 6; ++q)
        cv[q] = dot3(Mm[ia[q]][0], Mm[ia[q]][1], Mm[ia[q]][2], Mm[ib[q]]);
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
  }
}

static int g_derive_grid = 0;

void launch_derive(const float pu[3], const uint32_t *misses, const float4 *pos_m, const int8_t *feat,
                   const float *offs, const float *scale, const int8_t *W1T, const int32_t *b1s, const int8_t *W2T,
                   const int32_t *b2s, float *alpha, float4 *pool, FrameCounters *ctr, int num_sms,
                   cudaStream_t st) {
  const int smem = (int)sizeof(DeriveSmem);
  if (g_derive_grid == 0) {
    cudaFuncSetAttribute(derive_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, derive_kernel, kDThreads, smem);
    g_derive_grid = num_sms * (per_sm > 0 ? per_sm : 1);
  }
  derive_kernel<<<g_derive_grid, kDThreads, smem, st>>>(pu[0], pu[1], pu[2], misses, pos_m, feat, offs, scale, W1T,
                                                         b1s, W2T, b2s, alpha, pool, ctr);
}

}  // namespace gsc
