/*
 * gscache.h -- C ABI of the B200-native GS-Cache per-frame hot path.
 *
 * The calls follow the paper's problem statement: load a trained
 * structured-3DGS scene, feed the binocular HMD pose of each
 * frame ("each frame ... contains two poses of the binocular stereo cameras",
 * P:310) and get the two eye images.  One render call runs, on the
 * GPU, SURVEY.md §8(a) rows a1..a8:
 *   a0 unified camera (Eqs. 5-6; host fp64 -> fp32 constants)
 *   a1 frustum + LoD anchor culling and cache classify (Alg. 1)
 *   a2 cache-depth policy + watermark (Eq. 4, Alg. 1)
 *   a3 derivation of cache misses through the opacity / colour / covariance
 *      MLPs into the persistent Gaussian pool (Eq. 3)
 *   a4 EWA projection, opacity-aware extent, exact tile count
 *   a5 depth sort + (tile, depth) key duplication
 *   a6 radix sort by tile (onesweep LSD; with a5 this is the (tile, depth) sort)
 *   a7 per-tile ranges
 *   a8 per-tile front-to-back blending for both eyes (Eq. 1, Alg. 1)
 *
 * Conventions
 *  - Every call returns gsc_status; no C++ exception crosses the ABI.
 *  - Errors are sticky per context only for GSC_ECUDA (destroy the context).
 *    gsc_last_error() returns a NUL-terminated description of the last error.
 *  - A context owns all device memory it allocates (scene SoA, Gaussian pool,
 *    cache state, sort / splat buffers).  Output image buffers and CUDA
 *    streams belong to the caller.  One context = one rendering worker with a
 *    private cache; distinct contexts are independent; a context
 *    must not be used from two threads at once.
 *  - Camera convention: q = (w,x,y,z) unit quaternion,
 *    world-from-camera; camera right = R[:,0], up = R[:,1], forward = -R[:,2].
 *  - Images: GSC_FMT_RGB_F32_PLANAR = float[3][H][W] (12*W*H bytes),
 *    GSC_FMT_RGBA8 = uint8[H][W][4] (4*W*H bytes, alpha = 255*(1-T)).
 */
#ifndef GSCACHE_H
#define GSCACHE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSC_ABI_VERSION 4   /* 3: gsc_scene_desc_f32 gained the combine inputs (R32); 4: gsc_frame_stats.n_evals_list */

typedef enum {
  GSC_OK = 0,
  GSC_EINVAL = 1,      /* invalid argument */
  GSC_EFORMAT = 2,     /* malformed scene file; byte offset in gsc_last_error */
  GSC_EDEGENERATE = 3, /* antiparallel eye directions */
  GSC_ENOMEM = 4,      /* device or pinned allocation failed */
  GSC_ECUDA = 5,       /* CUDA runtime error; sticky */
  GSC_EINTERNAL = 6,   /* internal consistency failure */
  GSC_ESTATE = 7,      /* call out of order (render before load/pose) */
  GSC_ECAPACITY = 8    /* a frame needed more (tile, depth) pairs (or kept-tile list entries) than
                          pair_capacity allows: its image is incomplete (an overflowed kept-tile list
                          drops all of the frame's pairs: background image).  Reported by the call
                          that returns the frame's stats, else by the next gsc_render_pair /
                          gsc_sync / gsc_wait_frame / gsc_render_pair_host that sees the frame
                          finished; once per frame; not sticky */
} gsc_status;

typedef struct gsc_ctx gsc_ctx;

/* flags */
#define GSC_F_DEPTH_LITERAL 0x1u /* SPEC-literal H(miss rate) instead of H(novelty) */
#define GSC_F_STAGE_TIMING 0x2u  /* record CUDA events between the stages of every frame */
#define GSC_F_DERIVE_CUDA_CORES 0x4u /* derivation MLP on CUDA cores (dp4a) instead of tcgen05 tensor cores */
#define GSC_F_COUNT_EVALS 0x8u   /* blend counts its evaluations (gsc_frame_stats.n_evals / n_exp /
                                    n_evals_list; else 0);
                                    costs blend time, so bench.py counts in a separate untimed pass */
#define GSC_F_GUIDE_EXP 0x20u    /* guiding function H (Eq. 4): exponential response, depth = max(1, D_max >>
                                    floor(4 rate)) ("exponential response"; R23) */
#define GSC_F_GUIDE_STAGED 0x40u /* staged response: D_max / ceil(D_max/2) / ceil(D_max/4) / 1 for rate below
                                    1/10 / 1/4 / 1/2 / above ("staged response"; R23).  Neither flag:
                                    the linear H of the paper's experiments.  Take effect at gsc_reset_cache;
                                    setting both is GSC_EINVAL */
#define GSC_F_ABL_FIXED_EXTENT 0x80u /* ablation: tile extent r^2 = 9 (fixed 3 sigma) instead
                                        of the opacity-aware 2 ln(255 alpha); the blend is unchanged */
#define GSC_F_ABL_AABB_TILES 0x100u  /* ablation (F1): keep every tile of the candidate box (no exact tile test,
                                        P:256) -- more pairs, same pixels */
#define GSC_F_MONO 0x200u           /* render the left eye only (the right image is left untouched); with a
                                        rig whose eyes coincide this is a monocular pipeline -- two such
                                        contexts, one per eye, are the no-de-redundancy ablation (F1) */
#define GSC_F_STAGGER 0x400u        /* staggered expiry (R26): an anchor derived
                                       for the first time since the last reset at frame f is given birth
                                       f - min(i mod D_max, f - 1 - W_f), so lines filled together (the
                                       first frame) expire spread over D_max frames, not all at once
                                       (no periodic full re-derivation spikes).  Applies from the next
                                       gsc_reset_cache / load */
#define GSC_F_BLEND_EXACT 0x800u   /* blend with the exact exponential exp_s on every evaluation (pixels bit-identical
                                       to the oracle); default: the SFU exponential with exactness guards and an
                                       exact replay of the pixels whose decisions it could flip (
                                       pixels within 6e-4 of the oracle, decisions identical) */
#define GSC_F_SERIAL 0x10u       /* do not overlap frame f+1's front end (cull .. ranges) with frame f's
                                    blend: per-stage times then add up to the frame time */

typedef struct {
  int width, height;        /* pixels per eye */
  double fov_y;             /* vertical field of view, radians, 0 < fov_y < pi */
  double near_plane;        /* 0 < near < far */
  double far_plane;
  float bg[3];              /* background colour */
  int d_max;                /* max reuse depth D_max >= 1 (10 in the paper) */
  unsigned flags;           /* GSC_F_* */
  int64_t pair_capacity;    /* max (tile, depth) pairs per frame; 0 = default */
} gsc_config;

typedef struct { double p[3]; double q[4]; } gsc_eye;
typedef struct { gsc_eye left, right; double timestamp; } gsc_rig; /* StereoRig */

/* Host-side view of a scene (SoA, little-endian).  Borrowed by
 * gsc_load_scene_host for the duration of the call only.  Feature and weight
 * values are int8 codes on the 2^-7 grid (value = code / 128). */
typedef struct {
  int32_t n_anchors, lod_levels;  /* N, L */
  float d0;                       /* LoD base distance */
  const float *pos;               /* [N][3] */
  const int8_t *feat;             /* [N][32] */
  const float *offs;              /* [N][10][3] */
  const float *scale;             /* [N][3] */
  const uint8_t *level;           /* [N] */
  const int8_t *W1;               /* [35][96] (alpha | colour | covariance heads) */
  const int8_t *b1;               /* [96] */
  const int8_t *W2a, *b2a;        /* [32][10], [10] */
  const int8_t *W2c, *b2c;        /* [32][30], [30] */
  const int8_t *W2s, *b2s;        /* [32][70], [70]: per Gaussian 3 scales then quaternion (w,x,y,z) */
} gsc_scene_desc;

/* Real-weights scene (Eq. 3 P:101-105 "MLP_theta(f_i, d_view)" with trained
 * weights): fp32 features and decoder weights of any value (same shapes and layouts as
 * gsc_scene_desc).  The derivation then runs the fixed-order fp32 MLP (every output from its bias,
 * inputs in ascending index order, one fma per term; F4) on the CUDA cores with the
 * unquantised view direction d_view = (p_i - p_u) / |p_i - p_u|.  lod_levels = 1 with every level 0
 * is a Scaffold-GS scene (no LoD).  Borrowed for the duration of the call only. */
typedef struct {
  int32_t n_anchors, lod_levels;
  float d0;
  const float *pos, *feat, *offs, *scale;   /* [N][3], [N][32], [N][10][3], [N][3] */
  const uint8_t *level;                     /* [N] */
  const float *W1, *b1;                     /* [35 + dist_input][96], [96] */
  const float *W2a, *b2a, *W2c, *b2c, *W2s, *b2s;
  /* Scaffold-GS combine inputs (SURVEY §8(f) F4 "optional distance input / feature bank"; "first
   * combine operator"; R32 / F4-B), both off when 0:
   *   dist_input: the anchor-camera distance |p_i - p_u| is the MLP's 36th input (W1 row 35);
   *   feature_bank: the features enter the MLP blended across strides 4, 2, 1 (every 4th / 2nd value
   *   tiled back to 32), fh_k = w2 f_k + w1 f_{2 (k mod 16)} + w0 f_{4 (k mod 8)}, with view-dependent
   *   weights w = softmax(Wb2^T ReLU(Wb1^T (d_view, |p_i - p_u|) + bb1) + bb2). */
  int32_t dist_input, feature_bank;
  const float *Wb1, *bb1, *Wb2, *bb2;       /* [4][32], [32], [32][3], [3] (feature_bank only) */
} gsc_scene_desc_f32;

/* Per-frame record (SPEC FrameRecord S:421-423, CacheStats S:208). */
typedef struct {
  int64_t frame;
  uint32_t n_visible, n_hits, n_misses, n_new;   /* |X_f|, hits, misses (decoded), |X_f \ X_f-1| */
  uint32_t n_splats;                             /* projected splats with >= 1 tile, both eyes */
  uint32_t overflow;                             /* 1 if pairs exceeded pair_capacity */
  uint64_t n_pairs;                              /* (tile, depth) pairs, both eyes */
  int32_t depth_used, depth_next;                /* reuse depth for this frame / the next */
  float update_rate, novelty_rate;               /* misses/|X_f|, new/|X_f| */
  /* stage times in ms (GSC_F_STAGE_TIMING; else 0): */
  float ms_cull, ms_derive, ms_project, ms_depth_sort, ms_emit, ms_tile_sort, ms_ranges, ms_blend, ms_total;
  uint64_t n_evals;                              /* blend: (pixel, splat) evaluations executed (GSC_F_COUNT_EVALS) */
  uint64_t n_exp;                                /* blend: evaluations inside the skip bound (GSC_F_COUNT_EVALS) */
  uint32_t n_nonfinite_skipped;                  /* (Gaussian, eye) pairs skipped for non-finite splat parameters:
                                                    mean / covariance, or 2D covariance, determinant, conic or
                                                    centre (skip the splat, count it) */
  uint32_t n_blend_fixup;                        /* pixels the blend re-ran with the exact exp_s because a decision
                                                    came within the fast exponential's error band (R5) */
  uint64_t n_evals_list;                         /* blend: the method's (pixel, splat) evaluations -- per pixel, the
                                                    entries of its tile's sorted list up to and including the one it
                                                    stopped before, all of them if it never stopped (Eq. 1 over the
                                                    tile list; the oracle's orc_blend_pixel count, SURVEY
                                                    d-3); n_evals counts what the kernel executed after its
                                                    decision-preserving 8x4-block skip (GSC_F_COUNT_EVALS) */
} gsc_frame_stats;

/* out formats */
#define GSC_FMT_RGB_F32_PLANAR 0
#define GSC_FMT_RGBA8 1

/* debug fetch selectors (gsc_debug_fetch; call after the frame's stream work finished) */
#define GSC_DBG_VISIBLE 1     /* uint32 anchor ids of X_f, ascending */
#define GSC_DBG_MISSES 2      /* uint32 anchor ids decoded this frame, ascending */
#define GSC_DBG_POOL 3        /* float [N*10][13]: alpha, mu[3], cov[6] (00 01 02 11 12 22), rgb[3] by slot g=i*10+j */
#define GSC_DBG_SPLATS 4      /* float [n_splats][13]: u v A B C alpha r g b depth thr(NaN: not kept) eye kept_tiles; compaction order
                                 (per warp tile: eye-major, slot ascending); includes boxes with 0 kept tiles */
#define GSC_DBG_SPLAT_G 5     /* uint32 [n_splats]: Gaussian slot g of each splat (same order) */
#define GSC_DBG_PAIRS 6       /* uint64 [n_pairs]: sorted (tile << 32 | depth bits), tile = eye*T_e + ty*TW + tx */
#define GSC_DBG_PAIR_G 7      /* uint32 [n_pairs]: Gaussian slot g of each sorted pair */
#define GSC_DBG_RANGES 8      /* uint32 [2*T_e][2]: [start, end) per (eye, tile) */
#define GSC_DBG_BIRTH 9       /* int32 [N]: frame each anchor's pool slots were derived (INT32_MIN: never) */

int gsc_abi_version(void);

/* Create a context on CUDA device `cuda_device`.  Validates cfg (GSC_EINVAL). */
gsc_status gsc_create(int cuda_device, const gsc_config *cfg, gsc_ctx **out);

/* Load a GSC2 scene file (format in scenegen/__init__.py write_gsc2: version 2 = int8 grid codes,
 * version 3 = fp32 features and weights, the real-weights path F4; version 4 = version 3 with the
 * combine-input flags word and the feature-bank weights, R32); resets the cache.
 * GSC_EFORMAT with the byte offset on bad magic / truncation / unsupported dims. */
gsc_status gsc_load_scene(gsc_ctx *ctx, const char *path);

/* Same from host arrays (copied to the device; the caller keeps ownership). */
gsc_status gsc_load_scene_host(gsc_ctx *ctx, const gsc_scene_desc *scene);

/* Same for a real-weights scene (F4).  GSC_EINVAL on null arrays or bad sizes; GSC_EFORMAT when an
 * anchor level >= lod_levels or a feature / weight is not finite. */
gsc_status gsc_load_scene_host_f32(gsc_ctx *ctx, const gsc_scene_desc_f32 *scene);

/* Validate the rig (unit quaternions within 1e-6) and compute the
 * unified camera (Eqs. 5-6) and per-eye constants for the next render.
 * GSC_EDEGENERATE for antiparallel eyes. */
gsc_status gsc_set_pose(gsc_ctx *ctx, const gsc_rig *rig);

/* Enqueue one binocular frame on `cuda_stream` (NULL: the legacy default
 * stream) writing caller-owned DEVICE buffers out_left / out_right in
 * `out_format`.  Returns after enqueueing; results and stats are valid after
 * the stream synchronises.  If `stats` is non-NULL the call synchronises the
 * stream before returning and fills it. */
gsc_status gsc_render_pair(gsc_ctx *ctx, void *out_left, void *out_right, int out_format,
                           void *cuda_stream, gsc_frame_stats *stats);

/* End-to-end call: set the pose from HOST memory, render, copy both images
 * into caller-owned HOST buffers (pinned for full speed), synchronise.
 * `stats` may be NULL. */
gsc_status gsc_render_pair_host(gsc_ctx *ctx, const gsc_rig *rig, void *host_left, void *host_right,
                                int out_format, gsc_frame_stats *stats);

/* Asynchronous end-to-end call: set the pose, enqueue the frame and the copy
 * of its two images into caller-owned HOST buffers (pinned, or the copy is
 * synchronous), and return without waiting.  *seq receives the frame's
 * sequence number.  The host buffers must stay valid and unread until
 * gsc_wait_frame(ctx, *seq) returns; frames complete in submission order, so
 * frame f's copy overlaps frame f+1's computation.  GSC_EINVAL on NULL
 * arguments or a bad format. */
gsc_status gsc_render_pair_host_async(gsc_ctx *ctx, const gsc_rig *rig, void *host_left, void *host_right,
                                      int out_format, long long *seq);

/* Block until frame `seq` (from gsc_render_pair_host_async) has landed in
 * its host buffers.  GSC_EINVAL for a sequence number not yet submitted. */
gsc_status gsc_wait_frame(gsc_ctx *ctx, long long seq);

/* Wait for the context's outstanding work on `cuda_stream`. */
gsc_status gsc_sync(gsc_ctx *ctx, void *cuda_stream);

/* Per-frame records of the last `max` frames rendered since the previous call
 * (oldest first).  Call after gsc_sync.  *n receives the count. */
gsc_status gsc_stats_history(gsc_ctx *ctx, gsc_frame_stats *dst, int max, int *n);

/* Drop every cache line and restart the frame counter at 0 (Alg. 1 "first frame"). */
gsc_status gsc_reset_cache(gsc_ctx *ctx);

/* Replace gsc_config.flags.  GSC_F_STAGE_TIMING, GSC_F_DERIVE_CUDA_CORES and
 * GSC_F_COUNT_EVALS apply from the next frame; GSC_F_DEPTH_LITERAL from the
 * next gsc_reset_cache (it selects the cache policy the state machine
 * started with).  Synchronises the device.  GSC_EINVAL on unknown bits. */
gsc_status gsc_set_flags(gsc_ctx *ctx, unsigned flags);

/* Copy an intermediate of the most recent frame to host memory (debug/parity).
 * *len_bytes receives the full size; at most capacity_bytes are written.
 * Synchronises the context's last stream. */
gsc_status gsc_debug_fetch(gsc_ctx *ctx, int what, void *host_dst, size_t capacity_bytes, size_t *len_bytes);

/* Evaluate the device elementary functions (0 exp_s, 1 log_s, 2 tanh_s,
 * 3 sigmoid_s, 4 exp_blend = the blend's exact exp_s for x in [-87, 0],
 * 5 the blend's fast exp ex2.approx(fl(x log2e));
 * DESIGN.md Numerics) on n device floats (parity sweeps, error bounds). */
gsc_status gsc_selftest_elementary(gsc_ctx *ctx, int fn, const float *dev_in, float *dev_out, size_t n);

const char *gsc_last_error(const gsc_ctx *ctx);
void gsc_destroy(gsc_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* GSCACHE_H */
