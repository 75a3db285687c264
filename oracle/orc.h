/*
 * orc.h -- CPU ORACLE for the GS-Cache per-frame hot path (TEST INFRASTRUCTURE).
 *
 * This is test infrastructure, not product code.  Only tests/, the smoke()
 * entry of __graft_entry__.py and bench.py's cpu_baseline / --impl reference
 * legs may load it.  It shares no code with paper_2502_14938_b200/ (no common
 * headers, helpers, tables or constants); both sides read the same GSC2 scene
 * and trajectory produced by scenegen/.
 *
 * It is a plain, slow, step-by-step implementation of SURVEY.md §8(c)
 * (O-0 .. O-8), in the paper's order:
 *   binocular unify (Eqs. 5-6) -> anchor filtering + LoD
 *   (Alg. 1) -> cache state machine with explicit eviction
 *   (Alg. 1, Eq. 4) -> derivation of misses through the
 *   opacity / colour / covariance MLPs (Eq. 3, Eq. 2)
 *   -> EWA projection with opacity-aware extent and exact tile coverage
 *    -> (tile, depth) key duplication + sort -> per-tile
 *   front-to-back blending (Eq. 1, Alg. 1), both eyes.
 *
 * Every fp32 expression follows DESIGN.md "Numerics" op by op (no FMA except
 * the fmaf() Horner steps of the elementary functions); build with
 * -ffp-contract=off -fno-fast-math.
 */
#ifndef GSC_ORACLE_H
#define GSC_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_F 32
#define ORC_K 10
#define ORC_H 32
#define ORC_NOUT (ORC_K * 11)

typedef struct {
  int N, L;
  float d0;
  const float *pos;      /* [N*3] */
  const int8_t *feat;    /* [N*F] */
  const float *offs;     /* [N*K*3] */
  const float *scale;    /* [N*3] */
  const uint8_t *level;  /* [N] */
  const int8_t *W1, *b1, *W2a, *b2a, *W2c, *b2c, *W2s, *b2s;
  /* real-weights path: real != 0 selects fp32 features and decoder
   * weights (same shapes as the codes above, any values) and the unquantised view direction */
  int real;
  const float *featf;    /* [N*F] */
  const float *W1f, *b1f, *W2af, *b2af, *W2cf, *b2cf, *W2sf, *b2sf;   /* W1f: [F+3+dist_input][3H] */
  /* R32 (F4, Scaffold-GS combine inputs; real-weights scenes only): dist_input appends the
   * anchor-camera distance |p_i - p_u| to the MLP input; bank blends the features across strides
   * 4, 2, 1 with w = softmax(Wb2^T ReLU(Wb1^T (d_view, dist) + bb1) + bb2) */
  int dist_input, bank;
  const float *Wb1, *bb1, *Wb2, *bb2;   /* [4][F], [F], [F][3], [3] */
} orc_scene;

typedef struct {
  int width, height;
  double fov_y, near_plane, far_plane;
  float bg[3];
  int d_max;
  int depth_literal; /* 1: SPEC-literal H(miss rate); 0: H(novelty) */
  int guide;         /* guiding function H: ORC_GUIDE_LINEAR (default), _EXP, _STAGED (R23) */
  int ablate;        /* ORC_ABL_* bits (SURVEY §8(f) F1 ablations of P:256; 0 = the method) */
  int stagger;       /* 1: staggered expiry (R26): a never-derived anchor
                        missed at frame f gets birth f - min(i mod D_max, f - 1 - W_f), so the lines
                        filled together (first frame) expire spread over D_max frames */
} orc_config;

#define ORC_ABL_FIXED_EXTENT 1  /* extent r^2 = 9 (fixed 3 sigma) instead of 2 ln(255 alpha) */
#define ORC_ABL_AABB_TILES 2    /* every tile of the candidate box kept (no exact tile test) */

#define ORC_GUIDE_LINEAR 0
#define ORC_GUIDE_EXP 1
#define ORC_GUIDE_STAGED 2

typedef struct { double p[3]; double q[4]; } orc_eye;

typedef struct {
  float p[3], r0[3], r1[3], r2[3];
  float fx, fy, cx, cy, near_plane, far_plane, limx, limy;
} orc_eye_consts;

typedef struct {
  float p[3], right[3], up[3], fwd[3];
  float near_plane, far_plane, tx, ty, kx, ky;
  double p64[3], fwd64[3], up64[3], pullback64;
} orc_unified;

typedef struct {
  float u, v, A, B, C, alpha, rgb[3];
  float depth, thr;
  int tx0, tx1, ty0, ty1; /* candidate tile box, inclusive; tx0 > tx1 => empty */
  int ntiles;             /* kept tiles */
} orc_splat;

typedef struct {
  /* counts */
  int64_t frame;
  int n_visible, n_hits, n_misses, n_new, n_live, depth_used, depth_next;
  int64_t n_splats[2], n_pairs[2];
  int64_t n_evals; /* per-pixel splat evaluations in the blend */
  int64_t n_nonfinite; /* (Gaussian, eye) pairs skipped for non-finite splat parameters */
} orc_frame_stats;

/* ---- elementary functions (DESIGN.md Numerics E1-E4) ---- */
float orc_exp_s(float x);
float orc_log_s(float x);
float orc_tanh_s(float x);
float orc_sigmoid_s(float x);
void orc_elem_vec(int fn, const float *in, float *out, size_t n); /* fn: 0 exp 1 log 2 tanh 3 sigmoid */

/* ---- cameras (Eqs. 5-6) ---- */
int orc_eye_constants(const orc_config *cfg, const orc_eye *e, orc_eye_consts *out);
int orc_unify(const orc_config *cfg, const orc_eye *l, const orc_eye *r, orc_unified *out);

/* ---- per-element steps ---- */
float orc_margin(const float *offs_i, const float *s_i);
int orc_lod_cut(const orc_unified *u, int L, float d0, const float *p);
int orc_visible(const orc_unified *u, int L, float d0, const float *p, float margin, int level);
void orc_build_cov(const float q[4], const float S[3], float cov[6]);
/* F4: the fixed-order fp32 MLP of the real-weights path: x[35 + dist_input] (32 features, d_view,
 * [distance]) -> o[110] */
void orc_mlp_f32(const orc_scene *sc, const float *x, float o[ORC_NOUT]);
/* R32: the feature bank's softmax weights w[3] (strides 4, 2, 1) for y = (d_view, distance) */
void orc_bank_weights(const orc_scene *sc, const float y[4], float w[3]);
/* R32: the blended features fh[k] = w2 f_k + w1 f_{2 (k mod F/2)} + w0 f_{4 (k mod F/4)} (fixed fma order) */
void orc_bank_blend(const float f[ORC_F], const float w[3], float fh[ORC_F]);
void orc_derive_anchor(const orc_scene *sc, int i, const float pu[3], float *alpha, float *mu,
                       float *cov, float *rgb, float *o_raw /* [110] or NULL */);
/* 1 projected, 0 culled, -1 skipped for non-finite parameters (counted) */
int orc_project(const orc_config *cfg, const orc_eye_consts *ec, float alpha, const float *mu,
                const float *cov, const float *rgb, orc_splat *out);
int orc_tile_kept(const orc_config *cfg, const orc_splat *s, int tx, int ty);
float orc_tile_qmin(const orc_config *cfg, const orc_splat *s, int tx, int ty);
void orc_blend_pixel(const orc_splat *const *list, int n, float px_center_x, float px_center_y,
                     const float bg[3], float out[3], float *T_out, int *n_eval);
int orc_depth_H(int d_max, int64_t num, int64_t den);
int orc_depth_H_guide(int guide, int d_max, int64_t num, int64_t den);

/* ---- whole frames ---- */
typedef struct orc_state orc_state;
orc_state *orc_create(const orc_scene *sc, const orc_config *cfg);
void orc_destroy(orc_state *st);
void orc_reset(orc_state *st);

#define ORC_RASTER 1u   /* project + sort + blend (else cache state machine only) */
#define ORC_BRUTE  2u   /* O1 per-pixel brute force instead of the tiled O2 renderer */

/* outputs are optional (NULL to skip); img_* are planar [3][H][W] */
int orc_frame(orc_state *st, const orc_eye *l, const orc_eye *r, unsigned flags,
              orc_frame_stats *stats, float *img_l, float *img_r);

/* state / intermediate access after orc_frame (valid until the next call) */
int orc_get_visible(const orc_state *st, uint32_t *dst, int cap);
int orc_get_misses(const orc_state *st, uint32_t *dst, int cap);
int32_t orc_get_birth(const orc_state *st, int i);
void orc_get_pool(const orc_state *st, int64_t slot0, int64_t count, float *alpha, float *mu,
                  float *cov, float *rgb);
int64_t orc_get_pairs(const orc_state *st, uint64_t *keys, uint32_t *gs, int64_t cap);
int64_t orc_get_splats(const orc_state *st, int eye, uint32_t *gs, float *rec /* [n][12] */, int64_t cap);
int orc_num_threads(void);
void orc_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
