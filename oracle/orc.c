/*
 * orc.c -- CPU ORACLE of the GS-Cache per-frame hot path (TEST INFRASTRUCTURE).
 * See orc.h.  Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md
 * line n; "N#" = DESIGN.md "Numerics" item; "R#" = SURVEY.md §8c-2 reading.
 *
 * Build: gcc -O2 -std=c11 -fopenmp -ffp-contract=off -fno-fast-math -fPIC -shared
 * Every parallel loop writes disjoint outputs, so results do not depend on the
 * thread count.
 */
#define _GNU_SOURCE
#include "orc.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define K ORC_K
#define F ORC_F
#define H ORC_H

static inline float f_of_u(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static inline uint32_t u_of_f(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

/* ======================================================================
 * N1-N4: elementary functions (own definitions, Cody-Waite + polynomial).
 * Implemented here and, independently, on the GPU; pinned against libm in
 * tests/test_oracle_elementary.py.
 * ====================================================================== */

/* N1 exp_s: x -> e^x.  NaN -> NaN; x > 88.72283935546875 -> +inf;
 * x < -87.33654 (below ln FLT_MIN) -> 0 (flushed, documented deviation). */
float orc_exp_s(float x) {
  if (x != x) return x;
  if (x > 88.72283935546875f) return INFINITY;
  if (x < -87.33654022216797f) return 0.0f;
  const float log2e = 1.44269502162933349609375f;   /* 0x3FB8AA3B */
  const float ln2_hi = 0.693145751953125f;           /* 0x3F317200, 15 significant bits */
  const float ln2_lo = 1.428606765330187045037746429443359375e-06f; /* 0x35BFBE8E */
  float t = x * log2e;
  float n = rintf(t);                                /* round half to even */
  float r = fmaf(-n, ln2_hi, x);                     /* exact (n ln2_hi has <= 24 bits) */
  r = fmaf(-n, ln2_lo, r);                           /* one rounding */
  /* Taylor degree 7 (|r| <= 0.3466: truncation < 6e-9 relative), Horner with fmaf */
  float p = 1.98412698e-04f;                         /* 1/5040 */
  p = fmaf(p, r, 1.38888889e-03f);                   /* 1/720 */
  p = fmaf(p, r, 8.33333377e-03f);                   /* 1/120 */
  p = fmaf(p, r, 4.16666679e-02f);                   /* 1/24  */
  p = fmaf(p, r, 1.66666672e-01f);                   /* 1/6   */
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  int ni = (int)n;
  if (ni > 127) return (p * f_of_u(0x7F000000u)) * 2.0f;   /* 2^127 * 2 */
  return p * f_of_u((uint32_t)(ni + 127) << 23);
}

/* N2 log_s: natural log for finite x > 0 (fdlibm-style reduction to
 * m in [sqrt(2)/2, sqrt(2)], f = m - 1, s = f/(2+f), atanh series). */
float orc_log_s(float x) {
  if (x != x) return x;
  if (x < 0.0f) return NAN;
  if (x == 0.0f) return -INFINITY;
  if (x == INFINITY) return x;
  uint32_t b = u_of_f(x);
  int k = 0;
  if (b < 0x00800000u) { x = x * 8388608.0f; b = u_of_f(x); k = -23; }
  k += (int)(b >> 23) - 127;
  float m = f_of_u((b & 0x007FFFFFu) | 0x3F800000u);  /* [1, 2) */
  if (m > 1.41421353816986083984375f) { m = m * 0.5f; k += 1; }
  float f = m - 1.0f;
  float s = f / (2.0f + f);
  float z = s * s;
  float R = fmaf(z, 0.222222222f, 0.285714298f);      /* 2/9, 2/7 */
  R = fmaf(z, R, 0.400000006f);                        /* 2/5 */
  R = fmaf(z, R, 0.666666687f);                        /* 2/3 */
  R = z * R;
  float hfsq = 0.5f * (f * f);
  float dk = (float)k;
  const float ln2_hi = 0.693145751953125f;
  const float ln2_lo = 1.428606765330187045037746429443359375e-06f;
  /* log(1+f) = f - (hfsq - s*(hfsq + R)) */
  float lg = f - (hfsq - (s * (hfsq + R) + dk * ln2_lo));
  return dk * ln2_hi + lg;
}

/* N3 tanh_s: odd Taylor polynomial for |x| < 0.5, else 1 - 2/(exp_s(2|x|)+1). */
float orc_tanh_s(float x) {
  if (x != x) return x;
  float a = fabsf(x);
  float r;
  if (a < 0.5f) {
    float z = a * a;
    float p = 5.90027440e-04f;                 /* 6404582/10854718875 */
    p = fmaf(p, z, -1.45583438e-03f);          /* -929569/638512875 */
    p = fmaf(p, z, 3.59212872e-03f);           /* 21844/6081075 */
    p = fmaf(p, z, -8.86323553e-03f);          /* -1382/155925 */
    p = fmaf(p, z, 2.18694885e-02f);           /* 62/2835 */
    p = fmaf(p, z, -5.39682540e-02f);          /* -17/315 */
    p = fmaf(p, z, 1.33333340e-01f);           /* 2/15 */
    p = fmaf(p, z, -3.33333343e-01f);          /* -1/3 */
    r = fmaf(a * z, p, a);
  } else {
    float e = orc_exp_s(2.0f * a);
    r = 1.0f - 2.0f / (e + 1.0f);
  }
  return copysignf(r, x);
}

/* N4 sigmoid_s(x) = 1 / (1 + exp_s(-x)). */
float orc_sigmoid_s(float x) { return 1.0f / (1.0f + orc_exp_s(-x)); }

void orc_elem_vec(int fn, const float *in, float *out, size_t n) {
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)n; ++i) {
    float x = in[i];
    out[i] = fn == 0 ? orc_exp_s(x) : fn == 1 ? orc_log_s(x) : fn == 2 ? orc_tanh_s(x) : orc_sigmoid_s(x);
  }
}

/* ======================================================================
 * O-1 cameras (fp64, rounded once to fp32).  SPEC S:40-49 conventions:
 * R(q) world-from-camera, right = R[:,0], up = R[:,1], forward = -R[:,2].
 * ====================================================================== */

static int quat_R(const double qin[4], double R[3][3]) {
  double n = sqrt(qin[0] * qin[0] + qin[1] * qin[1] + qin[2] * qin[2] + qin[3] * qin[3]);
  if (!(fabs(n - 1.0) <= 1e-6)) return -1;
  double w = qin[0] / n, x = qin[1] / n, y = qin[2] / n, z = qin[3] / n;
  R[0][0] = 1.0 - 2.0 * (y * y + z * z); R[0][1] = 2.0 * (x * y - w * z); R[0][2] = 2.0 * (x * z + w * y);
  R[1][0] = 2.0 * (x * y + w * z); R[1][1] = 1.0 - 2.0 * (x * x + z * z); R[1][2] = 2.0 * (y * z - w * x);
  R[2][0] = 2.0 * (x * z - w * y); R[2][1] = 2.0 * (y * z + w * x); R[2][2] = 1.0 - 2.0 * (x * x + y * y);
  return 0;
}

static int cfg_ok(const orc_config *c) {
  return c->width > 0 && c->height > 0 && c->near_plane > 0 && c->far_plane > c->near_plane &&
         c->fov_y > 0 && c->fov_y < M_PI && c->d_max >= 1;
}

int orc_eye_constants(const orc_config *cfg, const orc_eye *e, orc_eye_consts *o) {
  double R[3][3];
  if (!cfg_ok(cfg) || quat_R(e->q, R)) return -1;
  double ty = tan(cfg->fov_y / 2.0);
  double tx = ty * (double)cfg->width / (double)cfg->height;
  double fy = ((double)cfg->height / 2.0) / ty;
  for (int k = 0; k < 3; ++k) {
    o->p[k] = (float)e->p[k];
    o->r0[k] = (float)R[k][0];      /* right */
    o->r1[k] = (float)(-R[k][1]);   /* -up: image y points down */
    o->r2[k] = (float)(-R[k][2]);   /* forward */
  }
  o->fx = (float)fy; o->fy = (float)fy;
  o->cx = (float)((double)cfg->width / 2.0); o->cy = (float)((double)cfg->height / 2.0);
  o->near_plane = (float)cfg->near_plane; o->far_plane = (float)cfg->far_plane;
  o->limx = (float)(1.3 * tx); o->limy = (float)(1.3 * ty);
  return 0;
}

/* Eqs. 5-6: d_u = mu_D/|mu_D|, p_u = mu_P - d_u |p1-p2| / (2 tan(fov/2));
 * up per S:297; far extended by the pullback (R8). */
int orc_unify(const orc_config *cfg, const orc_eye *l, const orc_eye *r, orc_unified *o) {
  double RL[3][3], RR[3][3];
  if (!cfg_ok(cfg) || quat_R(l->q, RL) || quat_R(r->q, RR)) return -1;
  double ds[3], us[3], d[3], up[3], rt[3], pm[3], dp[3];
  for (int k = 0; k < 3; ++k) {
    ds[k] = (-RL[k][2]) + (-RR[k][2]);
    us[k] = RL[k][1] + RR[k][1];
    pm[k] = (l->p[k] + r->p[k]) / 2.0;
    dp[k] = l->p[k] - r->p[k];
  }
  double dn = sqrt(ds[0] * ds[0] + ds[1] * ds[1] + ds[2] * ds[2]);
  if (!(dn > 1e-6)) return -2; /* antiparallel eyes */
  for (int k = 0; k < 3; ++k) d[k] = ds[k] / dn;
  double b = sqrt(dp[0] * dp[0] + dp[1] * dp[1] + dp[2] * dp[2]);
  double ty = tan(cfg->fov_y / 2.0);
  double pb = b / (2.0 * ty);
  double ud = us[0] * d[0] + us[1] * d[1] + us[2] * d[2];
  for (int k = 0; k < 3; ++k) up[k] = us[k] - ud * d[k];
  double un = sqrt(up[0] * up[0] + up[1] * up[1] + up[2] * up[2]);
  if (!(un > 1e-9)) return -2;
  for (int k = 0; k < 3; ++k) up[k] = up[k] / un;
  rt[0] = d[1] * up[2] - d[2] * up[1];
  rt[1] = d[2] * up[0] - d[0] * up[2];
  rt[2] = d[0] * up[1] - d[1] * up[0];
  double tx = ty * (double)cfg->width / (double)cfg->height;
  for (int k = 0; k < 3; ++k) {
    double pu = pm[k] - d[k] * pb;
    o->p64[k] = pu; o->fwd64[k] = d[k]; o->up64[k] = up[k];
    o->p[k] = (float)pu; o->fwd[k] = (float)d[k]; o->up[k] = (float)up[k]; o->right[k] = (float)rt[k];
  }
  o->pullback64 = pb;
  o->near_plane = (float)cfg->near_plane;
  o->far_plane = (float)(cfg->far_plane + pb);
  o->tx = (float)tx; o->ty = (float)ty;
  o->kx = (float)sqrt(1.0 + tx * tx); o->ky = (float)sqrt(1.0 + ty * ty);
  return 0;
}

/* ======================================================================
 * O-2 anchor filtering: frustum (with margin, R8) + LoD (R9).
 * ====================================================================== */

static inline float dot3(const float *a, const float *b) {
  return ((a[0] * b[0]) + (a[1] * b[1])) + (a[2] * b[2]);
}

/* R8: m_i = max_j |O_ij (.) s_i|_2 + 3.33 max_k s_ik */
float orc_margin(const float *offs_i, const float *s) {
  float mo = 0.0f;
  for (int j = 0; j < K; ++j) {
    float a = offs_i[3 * j + 0] * s[0], b = offs_i[3 * j + 1] * s[1], c = offs_i[3 * j + 2] * s[2];
    float nj = sqrtf(((a * a) + (b * b)) + (c * c));
    if (nj > mo) mo = nj;
  }
  float smax = s[0];
  if (s[1] > smax) smax = s[1];
  if (s[2] > smax) smax = s[2];
  return mo + 3.33f * smax;
}

/* R9: l(d) = clamp(floor(log2(d0/d)) + L - 1, 0, L - 1); floor(log2) via ilogbf (exact). */
int orc_lod_cut(const orc_unified *u, int L, float d0, const float *p) {
  float v[3] = {p[0] - u->p[0], p[1] - u->p[1], p[2] - u->p[2]};
  float d2 = dot3(v, v);
  if (d2 == 0.0f) return L - 1;
  float t = d0 / sqrtf(d2);
  int e = ilogbf(t);
  long long l = (long long)e + (L - 1);
  if (l < 0) l = 0;
  if (l > L - 1) l = L - 1;
  return (int)l;
}

int orc_visible(const orc_unified *u, int L, float d0, const float *p, float m, int level) {
  float v[3] = {p[0] - u->p[0], p[1] - u->p[1], p[2] - u->p[2]};
  float x = dot3(v, u->right), y = dot3(v, u->up), z = dot3(v, u->fwd);
  int fr = (z >= u->near_plane - m) && (z <= u->far_plane + m) &&
           (fabsf(x) - u->tx * z <= m * u->kx) && (fabsf(y) - u->ty * z <= m * u->ky);
  if (!fr) return 0;
  return level <= orc_lod_cut(u, L, d0, p);
}

/* ======================================================================
 * O-3 cache: guiding function H (Eq. 4; "linear"; S:234 form).
 * H = 1 + floor((2(D-1)(den-num) + den) / (2 den)) = clamp(1 + round_half_away((D-1)(1 - num/den)), 1, D)
 * ====================================================================== */
int orc_depth_H(int d_max, int64_t num, int64_t den) {
  if (den <= 0) return d_max;
  return 1 + (int)((2 * (int64_t)(d_max - 1) * (den - num) + den) / (2 * den));
}

/* Guiding-function variants ("exponential response and staged response are needed" for
 * accelerating / staged motion; the paper gives no formulas -- readings R23):
 *   ORC_GUIDE_EXP:    depth = max(1, D >> floor(4 num/den))  (halve the depth per quarter of the rate)
 *   ORC_GUIDE_STAGED: depth = D if rate < 1/10, ceil(D/2) if rate < 1/4, ceil(D/4) if rate < 1/2, else 1
 * Both exact in integers; H(0) = D, H(1) = 1, monotone non-increasing like the linear one. */
int orc_depth_H_guide(int guide, int d_max, int64_t num, int64_t den) {
  if (guide == ORC_GUIDE_LINEAR) return orc_depth_H(d_max, num, den);
  if (den <= 0) return d_max;
  if (guide == ORC_GUIDE_EXP) {
    int64_t q = (4 * num) / den;                 /* 0..4 */
    int d = d_max >> (int)q;
    return d < 1 ? 1 : d;
  }
  /* staged */
  if (10 * num < den) return d_max;
  if (4 * num < den) return (d_max + 1) / 2;
  if (2 * num < den) return (d_max + 3) / 4;
  return 1;
}

/* Eq. 2: Sigma = R S S^T R^T; q = raw (w,x,y,z) normalised (zero -> identity),
 * R by the 3DGS rotation formula, M = R diag(S), Sigma = M M^T (6 entries 00 01 02 11 12 22). */
void orc_build_cov(const float qin[4], const float S[3], float cov[6]) {
  float qw = qin[0], qx = qin[1], qy = qin[2], qz = qin[3];
  float qn2 = (((qw * qw) + (qx * qx)) + (qy * qy)) + (qz * qz);
  if (qn2 == 0.0f) { qw = 1.0f; qx = qy = qz = 0.0f; }
  else { float qn = sqrtf(qn2); qw = qw / qn; qx = qx / qn; qy = qy / qn; qz = qz / qn; }
  float R[3][3];
  R[0][0] = 1.0f - 2.0f * ((qy * qy) + (qz * qz));
  R[0][1] = 2.0f * ((qx * qy) - (qw * qz));
  R[0][2] = 2.0f * ((qx * qz) + (qw * qy));
  R[1][0] = 2.0f * ((qx * qy) + (qw * qz));
  R[1][1] = 1.0f - 2.0f * ((qx * qx) + (qz * qz));
  R[1][2] = 2.0f * ((qy * qz) - (qw * qx));
  R[2][0] = 2.0f * ((qx * qz) - (qw * qy));
  R[2][1] = 2.0f * ((qy * qz) + (qw * qx));
  R[2][2] = 1.0f - 2.0f * ((qx * qx) + (qy * qy));
  float M[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) M[r][c] = R[r][c] * S[c];
  static const int ia[6] = {0, 0, 0, 1, 1, 2}, ib[6] = {0, 1, 2, 1, 2, 2};
  for (int e = 0; e < 6; ++e) {
    const float *ma = M[ia[e]], *mb = M[ib[e]];
    cov[e] = ((ma[0] * mb[0]) + (ma[1] * mb[1])) + (ma[2] * mb[2]);
  }
}

/* ======================================================================
 * O-4 derivation (Eq. 3) with the exact-grid MLP (R3/R6).
 * ====================================================================== */
/* F4 real-weights path: MLP_theta(f_i, d_view) of Eq. 3 with trained-style
 * fp32 weights -- the three heads of reading R3, each Linear(35->32)-ReLU-Linear(32->n), evaluated in
 * fp32 in a fixed order (F4): every output starts from its bias and accumulates its inputs
 * in ascending index order, one fused multiply-add (fmaf, one rounding) per term:
 *   h_c = max(0, fma(W1[34][c], x[34], ... fma(W1[0][c], x[0], b1[c])))
 *   o_m = fma(W2[31][m], h[31], ... fma(W2[0][m], h[0], b2[m]))   (h of the head of output m) */
void orc_mlp_f32(const orc_scene *sc, const float *x, float o[ORC_NOUT]) {
  float a[3 * H];
  const int nin = F + 3 + (sc->dist_input ? 1 : 0);
  for (int c = 0; c < 3 * H; ++c) {
    float acc = sc->b1f[c];
    for (int k = 0; k < nin; ++k) acc = fmaf(sc->W1f[k * 3 * H + c], x[k], acc);
    a[c] = acc > 0.0f ? acc : 0.0f;            /* ReLU */
  }
  const float *W2[3] = {sc->W2af, sc->W2cf, sc->W2sf};
  const float *b2[3] = {sc->b2af, sc->b2cf, sc->b2sf};
  const int nh[3] = {K, 3 * K, 7 * K};
  int base = 0;
  for (int h = 0; h < 3; ++h) {
    for (int m = 0; m < nh[h]; ++m) {
      float acc = b2[h][m];
      for (int u = 0; u < H; ++u) acc = fmaf(W2[h][u * nh[h] + m], a[h * H + u], acc);
      o[base + m] = acc;
    }
    base += nh[h];
  }
}

/* R32 feature bank (Scaffold-GS "first combine operator"; F4-B), written out in its
 * fixed op order: hidden h_c = ReLU(bb1_c + sum_k Wb1[k][c] y_k) (one fma per term, k ascending from the
 * bias); logits z_m = bb2_m + sum_c Wb2[c][m] h_c (same); softmax with the max subtracted:
 * e_m = exp_s(z_m - max z), s = (e_0 + e_1) + e_2, w_m = e_m / s. */
void orc_bank_weights(const orc_scene *sc, const float y[4], float w[3]) {
  float h[F];
  for (int c = 0; c < F; ++c) {
    float acc = sc->bb1[c];
    for (int k = 0; k < 4; ++k) acc = fmaf(sc->Wb1[k * F + c], y[k], acc);
    h[c] = acc > 0.0f ? acc : 0.0f;
  }
  float z[3];
  for (int m = 0; m < 3; ++m) {
    float acc = sc->bb2[m];
    for (int c = 0; c < F; ++c) acc = fmaf(sc->Wb2[c * 3 + m], h[c], acc);
    z[m] = acc;
  }
  const float zmax = fmaxf(fmaxf(z[0], z[1]), z[2]);
  float e[3];
  for (int m = 0; m < 3; ++m) e[m] = orc_exp_s(z[m] - zmax);
  const float s = (e[0] + e[1]) + e[2];
  for (int m = 0; m < 3; ++m) w[m] = e[m] / s;
}

/* The three resolutions of the anchor feature: stride 1 (f itself), stride 2 and stride 4 -- every
 * 2nd / 4th value, tiled back to F values -- blended as fma(w2, f_k, fma(w1, f2_k, w0 * f4_k)). */
void orc_bank_blend(const float f[F], const float w[3], float fh[F]) {
  for (int k = 0; k < F; ++k) {
    const float f4 = f[4 * (k % (F / 4))], f2 = f[2 * (k % (F / 2))];
    fh[k] = fmaf(w[2], f[k], fmaf(w[1], f2, w[0] * f4));
  }
}

void orc_derive_anchor(const orc_scene *sc, int i, const float pu[3], float *alpha, float *mu,
                       float *cov, float *rgb, float *o_raw) {
  const float *p = sc->pos + 3 * (size_t)i;
  const float *s = sc->scale + 3 * (size_t)i;
  float v[3] = {p[0] - pu[0], p[1] - pu[1], p[2] - pu[2]};
  float n = sqrtf(dot3(v, v));
  float o[ORC_NOUT];
  if (sc->real) {
    /* F4: continuous view direction d_view = v / |v| (three IEEE divisions; 0 at the camera) */
    float xf[F + 4];
    for (int k = 0; k < 3; ++k) xf[F + k] = (n == 0.0f) ? 0.0f : v[k] / n;
    xf[F + 3] = n;                               /* R32 distance input (read only when dist_input) */
    if (sc->bank) {                              /* R32 feature bank */
      const float y[4] = {xf[F], xf[F + 1], xf[F + 2], n};
      float w[3];
      orc_bank_weights(sc, y, w);
      orc_bank_blend(sc->featf + (size_t)i * F, w, xf);
    } else {
      for (int k = 0; k < F; ++k) xf[k] = sc->featf[(size_t)i * F + k];
    }
    orc_mlp_f32(sc, xf, o);
  } else {
    /* grid path (R3/R6): quantised view direction, exact-integer MLP */
    int x[F + 3];
    for (int k = 0; k < F; ++k) x[k] = sc->feat[(size_t)i * F + k];
    for (int k = 0; k < 3; ++k) {
      float dv = (n == 0.0f) ? 0.0f : v[k] / n;
      long q = lrintf(128.0f * dv);            /* round half to even */
      if (q < -127) q = -127;
      if (q > 127) q = 127;
      x[F + k] = (int)q;
    }
    /* layer 1 (three heads side by side): z1 = W1 x + 128 b1  (value z1 / 2^14) */
    int64_t a[3 * H];
    for (int c = 0; c < 3 * H; ++c) {
      int64_t acc = 128 * (int64_t)sc->b1[c];
      for (int k = 0; k < F + 3; ++k) acc += (int64_t)sc->W1[k * 3 * H + c] * x[k];
      a[c] = acc > 0 ? acc : 0;                  /* ReLU */
    }
    /* layer 2 per head: z2 = W2 a + 2^14 b2 (value z2 / 2^21); one RNE conversion */
    const int8_t *W2[3] = {sc->W2a, sc->W2c, sc->W2s};
    const int8_t *b2[3] = {sc->b2a, sc->b2c, sc->b2s};
    const int nh[3] = {K, 3 * K, 7 * K};
    int base = 0;
    for (int h = 0; h < 3; ++h) {
      for (int m = 0; m < nh[h]; ++m) {
        int64_t acc = 16384 * (int64_t)b2[h][m];
        for (int u = 0; u < H; ++u) acc += (int64_t)W2[h][u * nh[h] + m] * a[h * H + u];
        o[base + m] = (float)acc * 4.76837158203125e-07f; /* 2^-21, exact */
      }
      base += nh[h];
    }
  }
  if (o_raw) memcpy(o_raw, o, sizeof(o));
  const float *oa = o, *oc = o + K, *os = o + 4 * K;
  const float *offs = sc->offs + (size_t)i * K * 3;
  for (int j = 0; j < K; ++j) {
    float al = orc_tanh_s(oa[j]);                     /* tanh, keep alpha > 0 */
    alpha[j] = al > 0.0f ? al : 0.0f;
    for (int k = 0; k < 3; ++k) rgb[3 * j + k] = orc_sigmoid_s(oc[3 * j + k]);
    float S[3];
    for (int k = 0; k < 3; ++k) S[k] = s[k] * orc_sigmoid_s(os[7 * j + k]);
    float q4[4] = {os[7 * j + 3], os[7 * j + 4], os[7 * j + 5], os[7 * j + 6]};
    orc_build_cov(q4, S, cov + 6 * j);
    for (int k = 0; k < 3; ++k) mu[3 * j + k] = p[k] + offs[3 * j + k] * s[k];
  }
}

/* ======================================================================
 * O-5 projection (EWA), opacity-aware extent and exact tile test.
 * ====================================================================== */
#define ORC_KAPPA 1.0009765625f   /* 1 + 2^-10 */
#define ORC_SLACK 0.015625f       /* 2^-6 */

/* Returns 1 (projected), 0 (culled) or -1: skipped for non-finite splat parameters ("non-finite
 * splat parameters -> skip splat, count in FrameRecord diagnostics"): a non-finite mean or covariance
 * entry, or, for a Gaussian inside the depth range, a non-finite determinant, conic or centre. */
int orc_project(const orc_config *cfg, const orc_eye_consts *ec, float alpha, const float *mu,
                const float *cov, const float *rgb, orc_splat *o) {
  float rho = 255.0f * alpha;
  if (!(rho > 1.0f)) return 0;                              /* alpha <= eps => cull */
  for (int k = 0; k < 3; ++k)
    if (!isfinite(mu[k])) return -1;
  for (int k = 0; k < 6; ++k)
    if (!isfinite(cov[k])) return -1;
  float t[3] = {mu[0] - ec->p[0], mu[1] - ec->p[1], mu[2] - ec->p[2]};
  float x = dot3(t, ec->r0), y = dot3(t, ec->r1), z = dot3(t, ec->r2);
  if (!(z > ec->near_plane) || z > ec->far_plane) return 0;
  /* N8: one reciprocal of z (and of det below), rounded once, multiplied in */
  float iz = 1.0f / z, iz2 = iz * iz;
  float xz = x * iz, yz = y * iz;
  float xc = fminf(fmaxf(xz, -ec->limx), ec->limx) * z;
  float yc = fminf(fmaxf(yz, -ec->limy), ec->limy) * z;
  float J00 = ec->fx * iz, J02 = -(ec->fx * xc) * iz2;
  float J11 = ec->fy * iz, J12 = -(ec->fy * yc) * iz2;
  float T[2][3];
  for (int k = 0; k < 3; ++k) {
    T[0][k] = (J00 * ec->r0[k]) + (J02 * ec->r2[k]);
    T[1][k] = (J11 * ec->r1[k]) + (J12 * ec->r2[k]);
  }
  float S[3][3] = {{cov[0], cov[1], cov[2]}, {cov[1], cov[3], cov[4]}, {cov[2], cov[4], cov[5]}};
  float U[2][3];
  for (int r = 0; r < 2; ++r)
    for (int k = 0; k < 3; ++k) U[r][k] = ((T[r][0] * S[0][k]) + (T[r][1] * S[1][k])) + (T[r][2] * S[2][k]);
  float a = ((U[0][0] * T[0][0]) + (U[0][1] * T[0][1])) + (U[0][2] * T[0][2]);
  float b = ((U[0][0] * T[1][0]) + (U[0][1] * T[1][1])) + (U[0][2] * T[1][2]);
  float c = ((U[1][0] * T[1][0]) + (U[1][1] * T[1][1])) + (U[1][2] * T[1][2]);
  a = a + 0.3f;
  c = c + 0.3f;
  float det = (a * c) - (b * b);
  if (!isfinite(det)) return -1;
  if (!(det > 0.0f)) return 0;
  float idet = 1.0f / det;
  o->A = c * idet;
  o->B = (-b) * idet;
  o->C = a * idet;
  o->u = (ec->fx * xz) + ec->cx;
  o->v = (ec->fy * yz) + ec->cy;
  float r2 = 2.0f * orc_log_s(rho);                         /* r^2 = 2 ln(alpha/eps) */
  if (cfg->ablate & ORC_ABL_FIXED_EXTENT) r2 = 9.0f;        /* ablation: fixed 3 sigma */
  o->thr = (r2 * ORC_KAPPA) + ORC_SLACK;
  o->alpha = alpha;
  o->rgb[0] = rgb[0]; o->rgb[1] = rgb[1]; o->rgb[2] = rgb[2];
  o->depth = z;
  if (!isfinite(o->A) || !isfinite(o->B) || !isfinite(o->C) || !isfinite(o->u) || !isfinite(o->v) ||
      !isfinite(o->thr))
    return -1;
  /* candidate box: ellipse AABB sqrt(thr * Sigma'_xx) (+1 px pad), clamped to the screen tiles */
  int TW = (cfg->width + 15) / 16, TH = (cfg->height + 15) / 16;
  float ex = sqrtf(o->thr * a) + 1.0f, ey = sqrtf(o->thr * c) + 1.0f;
  float fx0 = fmaxf(floorf((o->u - ex) * 0.0625f), 0.0f);
  float fx1 = fminf(floorf((o->u + ex) * 0.0625f), (float)(TW - 1));
  float fy0 = fmaxf(floorf((o->v - ey) * 0.0625f), 0.0f);
  float fy1 = fminf(floorf((o->v + ey) * 0.0625f), (float)(TH - 1));
  if (fx0 > fx1 || fy0 > fy1 || !(ex == ex) || !(ey == ey)) {
    o->tx0 = 1; o->tx1 = 0; o->ty0 = 1; o->ty1 = 0; o->ntiles = 0;
    return 1;
  }
  o->tx0 = (int)fx0; o->tx1 = (int)fx1; o->ty0 = (int)fy0; o->ty1 = (int)fy1;
  int n = 0;
  for (int ty = o->ty0; ty <= o->ty1; ++ty)
    for (int tx = o->tx0; tx <= o->tx1; ++tx) n += orc_tile_kept(cfg, o, tx, ty);
  o->ntiles = n;
  return 1;
}

/* min over t in [lo,hi] of P d^2 + 2 Q d t + R t^2, clamped minimiser t* = -Q d / R */
/* R14: the clamped minimiser uses the reciprocal of R rounded once: t* = -(Q d) * fl(1/R) */
static inline float edge_q(float d, float lo, float hi, float P, float Q, float R) {
  float t = -(Q * d) * (1.0f / R);
  t = fminf(fmaxf(t, lo), hi);
  return ((P * (d * d)) + (2.0f * (Q * (d * t)))) + (R * (t * t));
}

/* q_min(tile): min of the conic form over the tile's pixel-centre rectangle (R14). */
float orc_tile_qmin(const orc_config *cfg, const orc_splat *s, int tx, int ty) {
  int px1 = 16 * tx + 15, py1 = 16 * ty + 15;
  if (px1 > cfg->width - 1) px1 = cfg->width - 1;
  if (py1 > cfg->height - 1) py1 = cfg->height - 1;
  float X0 = (float)(16 * tx) + 0.5f, X1 = (float)px1 + 0.5f;
  float Y0 = (float)(16 * ty) + 0.5f, Y1 = (float)py1 + 0.5f;
  if (s->u >= X0 && s->u <= X1 && s->v >= Y0 && s->v <= Y1) return 0.0f;
  float q = edge_q(X0 - s->u, Y0 - s->v, Y1 - s->v, s->A, s->B, s->C);
  float q2 = edge_q(X1 - s->u, Y0 - s->v, Y1 - s->v, s->A, s->B, s->C);
  if (q2 < q) q = q2;
  q2 = edge_q(Y0 - s->v, X0 - s->u, X1 - s->u, s->C, s->B, s->A);
  if (q2 < q) q = q2;
  q2 = edge_q(Y1 - s->v, X0 - s->u, X1 - s->u, s->C, s->B, s->A);
  if (q2 < q) q = q2;
  return q;
}

/* R14 (N7): row form of the exact tile test.  For tile row ty the ellipse
 * {q <= thr} meets the band of pixel-centre rows [Y0, Y1] in the x-interval
 * [xl, xr] (extremes of the ellipse's x-extent over the band; the extremes of
 * x over the ellipse lie at dy = -/+ B sqrt(thr / (det C)), clamped to the
 * band).  A tile is kept iff its pixel-centre column range [X0, X1] meets
 * [xl, xr] -- in exact arithmetic the same set as q_min(tile) <= thr. */
int orc_row_interval(const orc_config *cfg, const orc_splat *s, int ty, float *xl, float *xr) {
  float det = (s->A * s->C) - (s->B * s->B);
  float ey = sqrtf(s->thr * (s->A / det));
  float sd = sqrtf(s->thr / (det * s->C));
  int py1 = 16 * ty + 15;
  if (py1 > cfg->height - 1) py1 = cfg->height - 1;
  float Y0 = (float)(16 * ty) + 0.5f, Y1 = (float)py1 + 0.5f;
  float lo = fmaxf(Y0 - s->v, -ey), hi = fminf(Y1 - s->v, ey);
  if (!(lo <= hi)) return 0;
  float bs = s->B * sd;
  float at = s->A * s->thr;
  float invA = 1.0f / s->A;                          /* rounded once per splat (N7) */
  float dyr = fminf(fmaxf(-bs, lo), hi);
  float Dr = fmaxf(at - (det * (dyr * dyr)), 0.0f);
  *xr = s->u + ((sqrtf(Dr) - (s->B * dyr)) * invA);
  float dyl = fminf(fmaxf(bs, lo), hi);
  float Dl = fmaxf(at - (det * (dyl * dyl)), 0.0f);
  *xl = s->u - ((sqrtf(Dl) + (s->B * dyl)) * invA);
  return 1;
}

int orc_tile_kept(const orc_config *cfg, const orc_splat *s, int tx, int ty) {
  if (cfg->ablate & ORC_ABL_AABB_TILES) return 1;           /* ablation: candidate box only */
  float xl, xr;
  if (!orc_row_interval(cfg, s, ty, &xl, &xr)) return 0;
  int px1 = 16 * tx + 15;
  if (px1 > cfg->width - 1) px1 = cfg->width - 1;
  float X0 = (float)(16 * tx) + 0.5f, X1 = (float)px1 + 0.5f;
  return X0 <= xr && X1 >= xl;
}

/* ======================================================================
 * O-8 per-pixel front-to-back compositing (Eq. 1; 3DGS semantics, R17).
 * ====================================================================== */
#define ORC_ALPHA_MIN 0.0039215688593685626983642578125f  /* fp32(1/255) = 0x3B808081 */

/* N6: power = -1/2 (A dx^2 + 2 B dx dy + C dy^2) evaluated as
 *   dx (a' dx + b' dy) + c' dy^2 with a' = -A/2, b' = -B, c' = -C/2, i.e.
 *   q = fma(a', dx, b' dy); power = fma(dx, q, (c' dy) dy);
 * T' = fma(-alpha', T, T) = T (1 - alpha'); C += c (alpha' T) by fma. */
void orc_blend_pixel(const orc_splat *const *list, int n, float pxc, float pyc, const float bg[3],
                     float out[3], float *T_out, int *n_eval) {
  float T = 1.0f, C[3] = {0.0f, 0.0f, 0.0f};
  int ev = 0;
  for (int i = 0; i < n; ++i) {
    const orc_splat *s = list[i];
    ++ev;
    float dx = s->u - pxc, dy = s->v - pyc;
    float a2 = -0.5f * s->A, b2 = -s->B, c2 = -0.5f * s->C;
    float q = fmaf(a2, dx, b2 * dy);
    float power = fmaf(dx, q, (c2 * dy) * dy);
    if (power > 0.0f) continue;
    float al = fminf(0.99f, s->alpha * orc_exp_s(power));
    if (al < ORC_ALPHA_MIN) continue;
    float Tn = fmaf(-al, T, T);
    if (Tn < 0.0001f) break;
    float w = al * T;
    for (int k = 0; k < 3; ++k) C[k] = fmaf(s->rgb[k], w, C[k]);
    T = Tn;
  }
  for (int k = 0; k < 3; ++k) out[k] = fmaf(T, bg[k], C[k]);
  if (T_out) *T_out = T;
  if (n_eval) *n_eval = ev;
}

/* ======================================================================
 * Whole-frame state machine (Alg. 1).
 * ====================================================================== */
#define ORC_EMPTY INT32_MIN   /* birth of an empty cache line */
struct orc_state {
  orc_scene sc;
  orc_config cfg;
  int64_t frame;
  int depth;
  int32_t *birth;       /* ORC_EMPTY = empty (explicit eviction) */
  uint8_t *ever;        /* anchor derived at least once since the last reset (staggered expiry) */
  int64_t W;            /* W_f = max_{f' <= f} (f' - depth_f'), W_0 = -D_max (staggered expiry cap) */
  uint8_t *prev_vis, *cur_vis;
  float *margin;
  float *alpha, *mu, *cov, *rgb;    /* pool, slot g = i*K + j */
  uint32_t *visible, *misses;
  int n_visible, n_misses;
  /* raster intermediates */
  orc_splat *spl[2];
  uint32_t *spl_g[2];
  int64_t n_spl[2], cap_spl;
  uint64_t *pkeys; uint32_t *pg;     /* sorted pairs */
  int64_t n_pairs, cap_pairs;
};

orc_state *orc_create(const orc_scene *sc, const orc_config *cfg) {
  if (!cfg_ok(cfg)) return NULL;
  orc_state *st = (orc_state *)calloc(1, sizeof(orc_state));
  st->sc = *sc;
  st->cfg = *cfg;
  size_t N = (size_t)sc->N;
  st->birth = (int32_t *)malloc(N * sizeof(int32_t));
  st->ever = (uint8_t *)calloc(N, 1);
  st->prev_vis = (uint8_t *)calloc(N, 1);
  st->cur_vis = (uint8_t *)calloc(N, 1);
  st->margin = (float *)malloc(N * sizeof(float));
  st->alpha = (float *)calloc(N * K, sizeof(float));
  st->mu = (float *)calloc(N * K * 3, sizeof(float));
  st->cov = (float *)calloc(N * K * 6, sizeof(float));
  st->rgb = (float *)calloc(N * K * 3, sizeof(float));
  st->visible = (uint32_t *)malloc(N * sizeof(uint32_t));
  st->misses = (uint32_t *)malloc(N * sizeof(uint32_t));
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)N; ++i)
    st->margin[i] = orc_margin(sc->offs + (size_t)i * K * 3, sc->scale + (size_t)i * 3);
  orc_reset(st);
  return st;
}

void orc_reset(orc_state *st) {
  size_t N = (size_t)st->sc.N;
  st->frame = 0;
  st->depth = st->cfg.d_max;            /* Alg. 1 */
  st->W = -(int64_t)st->cfg.d_max;
  for (size_t i = 0; i < N; ++i) st->birth[i] = ORC_EMPTY;
  memset(st->ever, 0, N);
  memset(st->prev_vis, 0, N);
  st->n_visible = st->n_misses = 0;
}

void orc_destroy(orc_state *st) {
  if (!st) return;
  free(st->birth); free(st->ever); free(st->prev_vis); free(st->cur_vis); free(st->margin);
  free(st->alpha); free(st->mu); free(st->cov); free(st->rgb);
  free(st->visible); free(st->misses);
  for (int e = 0; e < 2; ++e) { free(st->spl[e]); free(st->spl_g[e]); }
  free(st->pkeys); free(st->pg);
  free(st);
}

typedef struct { uint64_t key; uint32_t g; } pair_t;
static int pair_cmp(const void *a, const void *b) {
  const pair_t *x = (const pair_t *)a, *y = (const pair_t *)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->g < y->g ? -1 : (x->g > y->g);
}
typedef struct { uint32_t depth_bits; uint32_t g; int idx; } zrec_t;
static int z_cmp(const void *a, const void *b) {
  const zrec_t *x = (const zrec_t *)a, *y = (const zrec_t *)b;
  if (x->depth_bits != y->depth_bits) return x->depth_bits < y->depth_bits ? -1 : 1;
  return x->g < y->g ? -1 : (x->g > y->g);
}

static void render_eye_tiled(orc_state *st, int e, float *img, orc_frame_stats *stats, int64_t pair_lo,
                             int64_t pair_hi);
static void render_eye_brute(orc_state *st, int e, float *img, orc_frame_stats *stats);

int orc_frame(orc_state *st, const orc_eye *l, const orc_eye *r, unsigned flags, orc_frame_stats *stats,
              float *img_l, float *img_r) {
  const orc_scene *sc = &st->sc;
  const orc_config *cfg = &st->cfg;
  int N = sc->N;
  orc_unified u;
  orc_eye_consts ec[2];
  int rc = orc_unify(cfg, l, r, &u);
  if (rc) return rc;
  if (orc_eye_constants(cfg, l, &ec[0]) || orc_eye_constants(cfg, r, &ec[1])) return -1;
  int64_t f = st->frame;
  int depth = st->depth;

  /* Alg. 1 l.185-187: invalidate lines at max reuse depth (explicit eviction) */
  for (int i = 0; i < N; ++i)
    if (st->birth[i] != ORC_EMPTY && f - st->birth[i] >= depth) st->birth[i] = ORC_EMPTY;

  /* Alg. 1 l.184 anchors indexing and filtering, through the unified camera */
#pragma omp parallel for schedule(static)
  for (int i = 0; i < N; ++i)
    st->cur_vis[i] = (uint8_t)orc_visible(&u, sc->L, sc->d0, sc->pos + 3 * (size_t)i, st->margin[i], sc->level[i]);
  int nv = 0, nm = 0, nnew = 0;
  for (int i = 0; i < N; ++i) {
    if (!st->cur_vis[i]) continue;
    st->visible[nv++] = (uint32_t)i;
    if (!st->prev_vis[i]) ++nnew;
    if (st->birth[i] == ORC_EMPTY) st->misses[nm++] = (uint32_t)i;   /* hit <=> live cache line */
  }
  st->n_visible = nv;
  st->n_misses = nm;

  /* Alg. 1 l.188-196: decode misses (through the unified viewpoint, R7), update cache */
#pragma omp parallel for schedule(dynamic, 64)
  for (int m = 0; m < nm; ++m) {
    int i = (int)st->misses[m];
    size_t g0 = (size_t)i * K;
    orc_derive_anchor(sc, i, u.p, st->alpha + g0, st->mu + 3 * g0, st->cov + 6 * g0, st->rgb + 3 * g0, NULL);
  }
  /* update computation cache: the line of a derived anchor is born now.  Staggered expiry (F3, R26):
   * a never-derived anchor's line is back-dated by s_i = min(i mod D_max, f - 1 - W_f) frames, so the
   * lines filled together on a cold frame expire spread over D_max frames instead of all at once;
   * the cap keeps birth > W_f (the line is live until its own age reaches the depth). */
  for (int m = 0; m < nm; ++m) {
    const uint32_t i = st->misses[m];
    int64_t b = f;
    if (cfg->stagger && !st->ever[i]) {
      int64_t s = (int64_t)(i % (uint32_t)cfg->d_max), cap = f - 1 - st->W;
      b = f - (s < cap ? s : cap);
    }
    st->birth[i] = (int32_t)b;
    st->ever[i] = 1;
  }

  /* Alg. 1 l.198: depth <- H(rate); R10: rate = novelty |X_f \ X_f-1| / |X_f|
   * (SPEC-literal alternative: miss rate). Frame 0 keeps D_max. */
  int depth_next = depth;
  if (f > 0) depth_next = orc_depth_H_guide(cfg->guide, cfg->d_max, cfg->depth_literal ? nm : nnew, nv);
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->frame = f;
    stats->n_visible = nv; stats->n_misses = nm; stats->n_hits = nv - nm; stats->n_new = nnew;
    stats->depth_used = depth; stats->depth_next = depth_next;
  }
  st->depth = depth_next;
  if ((f + 1) - depth_next > st->W) st->W = (f + 1) - depth_next;   /* W_{f+1} */
  uint8_t *tmp = st->prev_vis; st->prev_vis = st->cur_vis; st->cur_vis = tmp;
  st->frame = f + 1;

  if (!(flags & ORC_RASTER)) return 0;

  /* O-5 projection of every visible slot for both eyes (Alg. 1 l.200-202) */
  int64_t S = (int64_t)nv * K;
  if (st->cap_spl < S) {
    for (int e = 0; e < 2; ++e) {
      free(st->spl[e]); free(st->spl_g[e]);
      st->spl[e] = (orc_splat *)malloc((size_t)S * sizeof(orc_splat));
      st->spl_g[e] = (uint32_t *)malloc((size_t)S * sizeof(uint32_t));
    }
    st->cap_spl = S;
  }
  int TW = (cfg->width + 15) / 16, TH = (cfg->height + 15) / 16;
  int64_t Te = (int64_t)TW * TH;
  unsigned char *ok = (unsigned char *)malloc((size_t)(S > 0 ? S : 1));
  orc_splat *tmp_spl = (orc_splat *)malloc((size_t)(S > 0 ? S : 1) * sizeof(orc_splat));
  int64_t total_pairs = 0;
  int64_t eye_pairs[2] = {0, 0};
  for (int e = 0; e < 2; ++e) {
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t s = 0; s < S; ++s) {
      int64_t g = (int64_t)st->visible[s / K] * K + (s % K);
      int r = orc_project(cfg, &ec[e], st->alpha[g], st->mu + 3 * g, st->cov + 6 * g, st->rgb + 3 * g, &tmp_spl[s]);
      ok[s] = (unsigned char)(r > 0 ? 1 : r < 0 ? 2 : 0);
    }
    int64_t n = 0, np = 0, nlive = 0, nnf = 0;
    for (int64_t s = 0; s < S; ++s) {
      int64_t g = (int64_t)st->visible[s / K] * K + (s % K);
      if (e == 0 && st->alpha[g] > 0.0f) ++nlive;
      if (ok[s] == 2) ++nnf;                                /* non-finite: skipped and counted */
      if (ok[s] != 1) continue;
      st->spl[e][n] = tmp_spl[s];
      st->spl_g[e][n] = (uint32_t)g;
      np += tmp_spl[s].ntiles;
      ++n;
    }
    st->n_spl[e] = n;
    eye_pairs[e] = np;
    total_pairs += np;
    if (stats) {
      stats->n_splats[e] = n; stats->n_pairs[e] = np;
      stats->n_nonfinite += nnf;
      if (e == 0) stats->n_live = (int)nlive;
    }
  }
  free(ok); free(tmp_spl);

  /* O-6 key duplication: key = (eye*Te + tile) << 32 | bits(depth); value g; sort by (key, g) */
  if (st->cap_pairs < total_pairs) {
    free(st->pkeys); free(st->pg);
    st->pkeys = (uint64_t *)malloc((size_t)total_pairs * sizeof(uint64_t));
    st->pg = (uint32_t *)malloc((size_t)total_pairs * sizeof(uint32_t));
    st->cap_pairs = total_pairs;
  }
  pair_t *pairs = (pair_t *)malloc((size_t)(total_pairs > 0 ? total_pairs : 1) * sizeof(pair_t));
  int64_t w = 0;
  for (int e = 0; e < 2; ++e)
    for (int64_t n = 0; n < st->n_spl[e]; ++n) {
      const orc_splat *sp = &st->spl[e][n];
      if (sp->ntiles == 0) continue;
      for (int ty = sp->ty0; ty <= sp->ty1; ++ty)
        for (int tx = sp->tx0; tx <= sp->tx1; ++tx)
          if (orc_tile_kept(cfg, sp, tx, ty)) {
            uint64_t tile = (uint64_t)(e * Te + (int64_t)ty * TW + tx);
            pairs[w].key = (tile << 32) | u_of_f(sp->depth);
            pairs[w].g = st->spl_g[e][n];
            ++w;
          }
    }
  qsort(pairs, (size_t)w, sizeof(pair_t), pair_cmp);
  for (int64_t p = 0; p < w; ++p) { st->pkeys[p] = pairs[p].key; st->pg[p] = pairs[p].g; }
  free(pairs);
  st->n_pairs = w;

  /* O-7/O-8: per (eye, tile) ranges and blend */
  float *img[2] = {img_l, img_r};
  for (int e = 0; e < 2; ++e) {
    if (!img[e]) continue;
    if (flags & ORC_BRUTE) render_eye_brute(st, e, img[e], stats);
    else render_eye_tiled(st, e, img[e], stats, e == 0 ? 0 : eye_pairs[0], e == 0 ? eye_pairs[0] : w);
  }
  return 0;
}

/* find a splat record by (eye, g): splats are stored in ascending g per eye */
static const orc_splat *find_splat(const orc_state *st, int e, uint32_t g) {
  int64_t lo = 0, hi = st->n_spl[e] - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    uint32_t gm = st->spl_g[e][mid];
    if (gm == g) return &st->spl[e][mid];
    if (gm < g) lo = mid + 1; else hi = mid - 1;
  }
  return NULL;
}

static void render_eye_tiled(orc_state *st, int e, float *img, orc_frame_stats *stats, int64_t lo, int64_t hi) {
  const orc_config *cfg = &st->cfg;
  int W = cfg->width, Hh = cfg->height, TW = (W + 15) / 16, TH = (Hh + 15) / 16;
  int64_t Te = (int64_t)TW * TH;
  int64_t *start = (int64_t *)malloc((size_t)(Te + 1) * sizeof(int64_t));
  /* ranges [start[t], start[t+1]) over the sorted pairs of this eye */
  int64_t p = lo;
  for (int64_t t = 0; t <= Te; ++t) {
    while (p < hi && (int64_t)(st->pkeys[p] >> 32) - e * Te < t) ++p;
    start[t] = p;
  }
  int64_t evals = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : evals)
  for (int64_t t = 0; t < Te; ++t) {
    int64_t n = start[t + 1] - start[t];
    const orc_splat **list = (const orc_splat **)malloc((size_t)(n > 0 ? n : 1) * sizeof(void *));
    for (int64_t k = 0; k < n; ++k) list[k] = find_splat(st, e, st->pg[start[t] + k]);
    int tx = (int)(t % TW), ty = (int)(t / TW);
    for (int yy = 0; yy < 16; ++yy)
      for (int xx = 0; xx < 16; ++xx) {
        int px = 16 * tx + xx, py = 16 * ty + yy;
        if (px >= W || py >= Hh) continue;
        float out[3];
        int ev;
        orc_blend_pixel(list, (int)n, (float)px + 0.5f, (float)py + 0.5f, cfg->bg, out, NULL, &ev);
        evals += ev;
        for (int k = 0; k < 3; ++k) img[((size_t)k * Hh + py) * W + px] = out[k];
      }
    free(list);
  }
  free(start);
  if (stats) stats->n_evals += evals;
}

/* O1: every projected splat of the eye at every pixel, in (depth, g) order -- no tiles. */
static void render_eye_brute(orc_state *st, int e, float *img, orc_frame_stats *stats) {
  const orc_config *cfg = &st->cfg;
  int W = cfg->width, Hh = cfg->height;
  int64_t n = st->n_spl[e];
  zrec_t *z = (zrec_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(zrec_t));
  for (int64_t k = 0; k < n; ++k) { z[k].depth_bits = u_of_f(st->spl[e][k].depth); z[k].g = st->spl_g[e][k]; z[k].idx = (int)k; }
  qsort(z, (size_t)n, sizeof(zrec_t), z_cmp);
  const orc_splat **list = (const orc_splat **)malloc((size_t)(n > 0 ? n : 1) * sizeof(void *));
  for (int64_t k = 0; k < n; ++k) list[k] = &st->spl[e][z[k].idx];
  int64_t evals = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : evals)
  for (int py = 0; py < Hh; ++py)
    for (int px = 0; px < W; ++px) {
      float out[3];
      int ev;
      orc_blend_pixel(list, (int)n, (float)px + 0.5f, (float)py + 0.5f, cfg->bg, out, NULL, &ev);
      evals += ev;
      for (int k = 0; k < 3; ++k) img[((size_t)k * Hh + py) * W + px] = out[k];
    }
  free(list); free(z);
  if (stats) stats->n_evals += evals;
}

/* ---------------- accessors ---------------- */
int orc_get_visible(const orc_state *st, uint32_t *dst, int cap) {
  int n = st->n_visible < cap ? st->n_visible : cap;
  if (dst) memcpy(dst, st->visible, (size_t)n * 4);
  return st->n_visible;
}
int orc_get_misses(const orc_state *st, uint32_t *dst, int cap) {
  int n = st->n_misses < cap ? st->n_misses : cap;
  if (dst) memcpy(dst, st->misses, (size_t)n * 4);
  return st->n_misses;
}
int32_t orc_get_birth(const orc_state *st, int i) { return st->birth[i]; }
void orc_get_pool(const orc_state *st, int64_t s0, int64_t cnt, float *alpha, float *mu, float *cov, float *rgb) {
  if (alpha) memcpy(alpha, st->alpha + s0, (size_t)cnt * 4);
  if (mu) memcpy(mu, st->mu + 3 * s0, (size_t)cnt * 12);
  if (cov) memcpy(cov, st->cov + 6 * s0, (size_t)cnt * 24);
  if (rgb) memcpy(rgb, st->rgb + 3 * s0, (size_t)cnt * 12);
}
int64_t orc_get_pairs(const orc_state *st, uint64_t *keys, uint32_t *gs, int64_t cap) {
  int64_t n = st->n_pairs < cap ? st->n_pairs : cap;
  if (keys) memcpy(keys, st->pkeys, (size_t)n * 8);
  if (gs) memcpy(gs, st->pg, (size_t)n * 4);
  return st->n_pairs;
}
/* rec layout [12]: u v A B C alpha r g b depth thr ntiles */
int64_t orc_get_splats(const orc_state *st, int e, uint32_t *gs, float *rec, int64_t cap) {
  int64_t n = st->n_spl[e] < cap ? st->n_spl[e] : cap;
  for (int64_t k = 0; k < n; ++k) {
    const orc_splat *s = &st->spl[e][k];
    if (gs) gs[k] = st->spl_g[e][k];
    if (rec) {
      float *r = rec + 12 * k;
      r[0] = s->u; r[1] = s->v; r[2] = s->A; r[3] = s->B; r[4] = s->C; r[5] = s->alpha;
      r[6] = s->rgb[0]; r[7] = s->rgb[1]; r[8] = s->rgb[2]; r[9] = s->depth; r[10] = s->thr;
      r[11] = (float)s->ntiles;
    }
  }
  return st->n_spl[e];
}
int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
