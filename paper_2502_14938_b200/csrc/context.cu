// context.cu -- host runtime and the C ABI of include/gscache.h.
//
// Owns the device-resident scene (SoA), the persistent Gaussian pool (the
// cache), the cache-policy state, all per-frame buffers, and drives
// the per-frame kernel sequence of SURVEY §3 (3) on the caller's stream.
// No host synchronisation inside a frame: every data-dependent size (V, M,
// splats, pairs) stays on the device and the kernels read it there.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "../../include/gscache.h"
#include "gsc_internal.cuh"

namespace gsc {
// launchers (kernels in the other translation units)
void launch_cull(const FrameC &, int, const float4 *, const uint8_t *, int32_t *, const uint32_t *, uint32_t *,
                 uint32_t *, uint32_t *, uint32_t *, unsigned long long *, FrameCounters *, PolicyState *,
                 FrameRecordDev *, cudaStream_t);
void launch_record(const FrameCounters *, FrameRecordDev *, cudaStream_t);
void launch_margin(int, const float *, const float *, const float *, float4 *, cudaStream_t);
int cull_tiles(int N);
void launch_derive(const float pu[3], const uint32_t *, const float4 *, const int8_t *, const float *, const float *,
                   const int8_t *, const int32_t *, const int8_t *, const int32_t *, float *, float4 *,
                   FrameCounters *, int, bool, cudaStream_t);
void launch_project(const FrameC &, const uint32_t *, const float *, const float4 *, uint32_t *, uint32_t *,
                    const SplatBufs &,
                    uint32_t *, FrameCounters *, int, cudaStream_t);
int project_tile_size();
void launch_onesweep(uint32_t *, uint32_t *, uint32_t *, uint32_t *, bool, const uint32_t *, int, int, const uint32_t *,
                     uint32_t *, uint32_t *, uint32_t *, uint2 *, int, cudaStream_t);
void launch_emit(const EmitIn &, uint32_t, uint32_t *, uint32_t *, uint32_t *, FrameCounters *, int, int,
                 cudaStream_t);
void launch_blend(const FrameC &, const uint2 *, const uint32_t *, const uint32_t *, const float4 *, const float4 *,
                  const float2 *, void *, void *, int, FrameCounters *, uint32_t *, bool, bool, int, cudaStream_t);
void launch_elem(int, const float *, float *, size_t, int, cudaStream_t);
void launch_derive_f32(const float pu[3], const uint32_t *, const float4 *, const float *, const float *, const float *,
                       const float *, const float *, const float *, const float *, const CombineF32 &, float *, float4 *,
                       FrameCounters *, int, cudaStream_t);
int sort_tile_size();
int emit_tile_size();
}  // namespace gsc

using namespace gsc;

namespace {

constexpr int kRing = 2048;     // per-frame record / event ring
constexpr int kEvents = 10;     // stage boundaries per frame

template <typename T>
struct DevBuf {
  T *p = nullptr;
  size_t n = 0;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t count) {
    if (p) { cudaFree(p); p = nullptr; }
    n = count;
    return count ? cudaMalloc(&p, count * sizeof(T)) : cudaSuccess;
  }
};

struct FrameSlot {
  cudaEvent_t ev[kEvents];
  bool timed = false;
  bool used = false;
};

}  // namespace

struct gsc_ctx {
  int device = 0;
  gsc_config cfg{};
  int num_sms = 148;
  std::string err;
  bool sticky = false;
  // scene
  int N = 0, L = 0;
  float d0 = 0.0f;
  bool have_scene = false, have_pose = false;
  DevBuf<float4> pos_m;
  DevBuf<uint8_t> level;
  DevBuf<int8_t> feat;
  DevBuf<float> offs, scale;
  DevBuf<int8_t> W1T, W2T;
  DevBuf<int32_t> b1s, b2s;
  bool real = false;                 // real-weights scene (F4): fp32 features / weights below
  DevBuf<float> featf, W1f, b1f, W2f, b2f;   // [N][32], [35 + dist][96], [96], [32][110] (heads concatenated), [110]
  bool dist_input = false, bank = false;      // R32 combine inputs (real-weights scenes)
  DevBuf<float> Wb1f, bb1f, Wb2f, bb2f;       // feature bank MLP: [4][32], [32], [32][3], [3]
  // cache
  DevBuf<int32_t> birth;
  DevBuf<uint32_t> vis[2];
  DevBuf<uint32_t> miss_bits;   // the frame's miss bitset (cull pass 1 -> pass 2)
  int vis_cur = 0;
  DevBuf<float> alpha;
  DevBuf<float4> pool;
  DevBuf<PolicyState> policy;
  // per frame
  DevBuf<uint32_t> visible, misses;
  size_t cap_splat = 0, cap_pairs = 0;
  // What the blend of frame f reads lives in fs[f & 1]: the next frame's front end (cull .. ranges,
  // stream sA) runs while this frame's blend (stream sB) still reads its set (inter-frame pipeline).
  struct FrameSet {
    DevBuf<float4> spA, spB;
    DevBuf<float2> spC;
    DevBuf<uint32_t> pkey, pval;           // tile-sorted pairs
    DevBuf<uint2> ranges;
    DevBuf<unsigned char> zero_region;     // FrameCounters | cull status | project status | emit status
    FrameCounters *ctr() { return reinterpret_cast<FrameCounters *>(zero_region.p); }
  } fs[2];
  cudaStream_t sA = nullptr, sB = nullptr;
  cudaEvent_t ev_user[2] = {nullptr, nullptr}, ev_a[2] = {nullptr, nullptr}, ev_b[2] = {nullptr, nullptr};
  bool b_pending[2] = {false, false};
  DevBuf<uint32_t> count, dkey_a, dval_a, dkey_b, dval_b, list_off, pair_off, list, live_g;
  DevBuf<uint32_t> live_bits;   // live bitset of the visible slots (live_mark -> live)
  DevBuf<uint32_t> pkey_b, pval_b;         // tile-sort scratch (front end only)
  DevBuf<uint32_t> fixup;                  // blend: pixels for the exact replay (blends run in frame order)
  DevBuf<uint32_t> sort_status_a, sort_status_b;
  size_t zero_bytes = 0, off_cull = 0, off_proj = 0, off_emit = 0;
  DevBuf<FrameRecordDev> rec_dev;
  FrameRecordDev *rec_host = nullptr;    // pinned ring
  FrameSlot slots[kRing];
  int64_t frames_rendered = 0, frames_reported = 0;
  int64_t frames_checked = 0;            // frames whose capacity overflow flag has been reported
  FrameC fc{};
  float pu[3] = {0, 0, 0};
  cudaStream_t last_stream = nullptr;
  cudaStream_t own_stream = nullptr;
  // e2e staging: device images per frame parity (the copy of frame f overlaps the blend of frame f+1)
  DevBuf<unsigned char> img_dev[2][2];
  static constexpr int kHostRing = 8;
  cudaEvent_t host_done[kHostRing] = {};
  int64_t host_frame[kHostRing] = {};    // frame sequence number of each in-flight host submission
  int64_t host_submitted = 0;

  FrameSet &last_set() { return fs[(frames_rendered + 1) & 1]; }   // the set of the last rendered frame
};

static gsc_status fail(gsc_ctx *c, gsc_status s, const std::string &msg) {
  if (c) {
    c->err = msg;
    if (s == GSC_ECUDA) c->sticky = true;
  }
  return s;
}
#define CU(call)                                                                                   \
  do {                                                                                             \
    cudaError_t _e = (call);                                                                       \
    if (_e != cudaSuccess) return fail(ctx, GSC_ECUDA, std::string(#call ": ") + cudaGetErrorString(_e)); \
  } while (0)

static bool cfg_valid(const gsc_config *c) {
  return c && c->width > 0 && c->height > 0 && c->width <= 16 * 65535 && c->fov_y > 0 && c->fov_y < M_PI &&
         c->near_plane > 0 && c->far_plane > c->near_plane && c->d_max >= 1 &&
         2LL * ((c->width + 15) / 16) * ((c->height + 15) / 16) <= 65536 &&
         !((c->flags & GSC_F_GUIDE_EXP) && (c->flags & GSC_F_GUIDE_STAGED));
}

// ----------------------------------------------------------------------------------- camera (a0)
// Eqs. 5-6 in fp64, rounded once to fp32.  R(q) world-from-camera
// (S:41), right = R[:,0], up = R[:,1], forward = -R[:,2].
static bool quat_R(const double qi[4], double R[3][3]) {
  double n = std::sqrt(qi[0] * qi[0] + qi[1] * qi[1] + qi[2] * qi[2] + qi[3] * qi[3]);
  if (!(std::fabs(n - 1.0) <= 1e-6)) return false;
  double w = qi[0] / n, x = qi[1] / n, y = qi[2] / n, z = qi[3] / n;
  R[0][0] = 1.0 - 2.0 * (y * y + z * z); R[0][1] = 2.0 * (x * y - w * z); R[0][2] = 2.0 * (x * z + w * y);
  R[1][0] = 2.0 * (x * y + w * z); R[1][1] = 1.0 - 2.0 * (x * x + z * z); R[1][2] = 2.0 * (y * z - w * x);
  R[2][0] = 2.0 * (x * z - w * y); R[2][1] = 2.0 * (y * z + w * x); R[2][2] = 1.0 - 2.0 * (x * x + y * y);
  return true;
}

static gsc_status compute_frame_consts(gsc_ctx *ctx, const gsc_rig *rig) {
  const gsc_config &c = ctx->cfg;
  double RL[3][3], RR[3][3];
  if (!quat_R(rig->left.q, RL) || !quat_R(rig->right.q, RR))
    return fail(ctx, GSC_EINVAL, "rig quaternion not unit within 1e-6 (S:43)");
  for (int k = 0; k < 3; ++k)
    if (!std::isfinite(rig->left.p[k]) || !std::isfinite(rig->right.p[k])) return fail(ctx, GSC_EINVAL, "non-finite eye position");
  const double ty = std::tan(c.fov_y / 2.0);
  const double tx = ty * (double)c.width / (double)c.height;
  const double fy = ((double)c.height / 2.0) / ty;
  FrameC &fc = ctx->fc;
  const double (*Rs[2])[3] = {RL, RR};
  const gsc_eye *eyes[2] = {&rig->left, &rig->right};
  for (int e = 0; e < 2; ++e) {
    EyeC &ec = fc.eye[e];
    for (int k = 0; k < 3; ++k) {
      ec.p[k] = (float)eyes[e]->p[k];
      ec.r0[k] = (float)Rs[e][k][0];
      ec.r1[k] = (float)(-Rs[e][k][1]);
      ec.r2[k] = (float)(-Rs[e][k][2]);
    }
    ec.fx = (float)fy; ec.fy = (float)fy;
    ec.cx = (float)((double)c.width / 2.0); ec.cy = (float)((double)c.height / 2.0);
    ec.near_plane = (float)c.near_plane; ec.far_plane = (float)c.far_plane;
    ec.limx = (float)(1.3 * tx); ec.limy = (float)(1.3 * ty);
  }
  double ds[3], us[3], d[3], up[3], rt[3], pm[3], dp[3];
  for (int k = 0; k < 3; ++k) {
    ds[k] = (-RL[k][2]) + (-RR[k][2]);
    us[k] = RL[k][1] + RR[k][1];
    pm[k] = (rig->left.p[k] + rig->right.p[k]) / 2.0;
    dp[k] = rig->left.p[k] - rig->right.p[k];
  }
  double dn = std::sqrt(ds[0] * ds[0] + ds[1] * ds[1] + ds[2] * ds[2]);
  if (!(dn > 1e-6)) return fail(ctx, GSC_EDEGENERATE, "antiparallel eye directions (S:296)");
  for (int k = 0; k < 3; ++k) d[k] = ds[k] / dn;
  double b = std::sqrt(dp[0] * dp[0] + dp[1] * dp[1] + dp[2] * dp[2]);
  double pb = b / (2.0 * ty);
  double ud = us[0] * d[0] + us[1] * d[1] + us[2] * d[2];
  for (int k = 0; k < 3; ++k) up[k] = us[k] - ud * d[k];
  double un = std::sqrt(up[0] * up[0] + up[1] * up[1] + up[2] * up[2]);
  if (!(un > 1e-9)) return fail(ctx, GSC_EDEGENERATE, "eye up vectors degenerate (S:297)");
  for (int k = 0; k < 3; ++k) up[k] = up[k] / un;
  rt[0] = d[1] * up[2] - d[2] * up[1];
  rt[1] = d[2] * up[0] - d[0] * up[2];
  rt[2] = d[0] * up[1] - d[1] * up[0];
  UniC &u = fc.u;
  for (int k = 0; k < 3; ++k) {
    u.p[k] = (float)(pm[k] - d[k] * pb);
    u.fwd[k] = (float)d[k];
    u.up[k] = (float)up[k];
    u.right[k] = (float)rt[k];
    ctx->pu[k] = u.p[k];
  }
  u.near_plane = (float)c.near_plane;
  u.far_plane = (float)(c.far_plane + pb);
  u.tx = (float)tx; u.ty = (float)ty;
  u.kx = (float)std::sqrt(1.0 + tx * tx); u.ky = (float)std::sqrt(1.0 + ty * ty);
  fc.width = c.width; fc.height = c.height;
  fc.TW = (c.width + kTile - 1) / kTile;
  fc.TH = (c.height + kTile - 1) / kTile;
  fc.Te = fc.TW * fc.TH;
  fc.L = ctx->L; fc.d0 = ctx->d0;
  for (int k = 0; k < 3; ++k) fc.bg[k] = c.bg[k];
  return GSC_OK;
}

// ----------------------------------------------------------------------------------- scene load
static gsc_status reset_cache(gsc_ctx *ctx, cudaStream_t st);

static __global__ void fill_i32(int32_t *p, size_t n, int32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

// Exactly one of g (grid codes, R3/R6) and f (real fp32 weights, F4) is non-null.
static gsc_status upload_scene(gsc_ctx *ctx, const gsc_scene_desc *g, const gsc_scene_desc_f32 *f) {
  struct { int32_t n_anchors, lod_levels; float d0; const float *pos, *offs, *scale; const uint8_t *level; } c{};
  if (g) c = {g->n_anchors, g->lod_levels, g->d0, g->pos, g->offs, g->scale, g->level};
  else c = {f->n_anchors, f->lod_levels, f->d0, f->pos, f->offs, f->scale, f->level};
  const auto *s = &c;
  const int N = s->n_anchors;
  const bool wok = g ? (g->feat && g->W1 && g->b1 && g->W2a && g->b2a && g->W2c && g->b2c && g->W2s && g->b2s)
                     : (f->feat && f->W1 && f->b1 && f->W2a && f->b2a && f->W2c && f->b2c && f->W2s && f->b2s);
  if (N <= 0 || s->lod_levels < 1 || s->lod_levels > 64 || !(s->d0 > 0.0f) || !s->pos || !s->offs || !s->scale ||
      !s->level || !wok)
    return fail(ctx, GSC_EINVAL, "invalid scene description");
  if ((int64_t)N * kK >= (1LL << 29)) return fail(ctx, GSC_EINVAL, "scene too large (N*K must be < 2^29)");
  for (int i = 0; i < N; ++i)
    if (s->level[i] >= s->lod_levels) return fail(ctx, GSC_EFORMAT, "anchor level >= L at anchor " + std::to_string(i));
  std::vector<int8_t> W1T, W2T;
  std::vector<int32_t> b1s, b2s;
  std::vector<float> W2f, b2f;
  if (g) {
    // exact int32 range of the grid MLP (R3): |z1| <= hmax, |z2| < 2^31
    int64_t hmax = 0;
    for (int n = 0; n < 96; ++n) {
      int64_t acc = 128 * (int64_t)std::abs((int)g->b1[n]);
      for (int k = 0; k < kF + 3; ++k) acc += 127 * (int64_t)std::abs((int)g->W1[k * 96 + n]);
      hmax = std::max(hmax, acc);
    }
    if (hmax >= (1LL << 24)) return fail(ctx, GSC_EFORMAT, "hidden activations may exceed 24 bits (3 tensor-core limbs)");
    W1T.assign(96 * 36, 0); W2T.assign(kNOut * 32, 0); b1s.resize(96); b2s.resize(kNOut);
    for (int n = 0; n < 96; ++n) {
      for (int k = 0; k < kF + 3; ++k) W1T[n * 36 + k] = g->W1[k * 96 + n];
      b1s[n] = 128 * (int32_t)g->b1[n];
    }
    for (int m = 0; m < kNOut; ++m) {
      const int8_t *W2; int nh, mm; int8_t b;
      if (m < kK) { W2 = g->W2a; nh = kK; mm = m; b = g->b2a[mm]; }
      else if (m < 4 * kK) { W2 = g->W2c; nh = 3 * kK; mm = m - kK; b = g->b2c[mm]; }
      else { W2 = g->W2s; nh = 7 * kK; mm = m - 4 * kK; b = g->b2s[mm]; }
      int64_t bound = 16384 * (int64_t)std::abs((int)b);
      for (int u = 0; u < 32; ++u) {
        W2T[m * 32 + u] = W2[u * nh + mm];
        bound += hmax * std::abs((int)W2[u * nh + mm]);
      }
      if (bound >= (1LL << 31)) return fail(ctx, GSC_EFORMAT, "decoder weights exceed the exact int32 range");
      b2s[m] = 16384 * (int32_t)b;
    }
  } else {
    auto finite = [](const float *p, size_t n) {
      for (size_t k = 0; k < n; ++k)
        if (!std::isfinite(p[k])) return false;
      return true;
    };
    if ((f->dist_input != 0 && f->dist_input != 1) || (f->feature_bank != 0 && f->feature_bank != 1) ||
        (f->feature_bank && (!f->Wb1 || !f->bb1 || !f->Wb2 || !f->bb2)))
      return fail(ctx, GSC_EINVAL, "invalid combine-input flags or missing feature-bank weights");
    if (f->feature_bank && (!finite(f->Wb1, 4 * kF) || !finite(f->bb1, kF) || !finite(f->Wb2, kF * 3) ||
                            !finite(f->bb2, 3)))
      return fail(ctx, GSC_EFORMAT, "non-finite feature-bank weight");
    if (!finite(f->feat, (size_t)N * kF) || !finite(f->W1, (size_t)(35 + f->dist_input) * 96) || !finite(f->b1, 96) ||
        !finite(f->W2a, 32 * kK) || !finite(f->b2a, kK) || !finite(f->W2c, 32 * 3 * kK) || !finite(f->b2c, 3 * kK) ||
        !finite(f->W2s, 32 * 7 * kK) || !finite(f->b2s, 7 * kK))
      return fail(ctx, GSC_EFORMAT, "non-finite feature or decoder weight");
    // layer-2 weights of the three heads side by side: W2f[u][m], m = alpha 0..9 | colour 10..39 | cov 40..109
    W2f.assign(32 * kNOut, 0.0f); b2f.resize(kNOut);
    for (int m = 0; m < kNOut; ++m) {
      const float *W2; int nh, mm;
      if (m < kK) { W2 = f->W2a; nh = kK; mm = m; b2f[m] = f->b2a[mm]; }
      else if (m < 4 * kK) { W2 = f->W2c; nh = 3 * kK; mm = m - kK; b2f[m] = f->b2c[mm]; }
      else { W2 = f->W2s; nh = 7 * kK; mm = m - 4 * kK; b2f[m] = f->b2s[mm]; }
      for (int u = 0; u < 32; ++u) W2f[u * kNOut + m] = W2[u * nh + mm];
    }
  }
  ctx->have_scene = false;
  ctx->N = N; ctx->L = s->lod_levels; ctx->d0 = s->d0;
  const size_t NK = (size_t)N * kK;
  CU(ctx->pos_m.alloc(N));
  CU(ctx->level.alloc(N));
  CU(ctx->offs.alloc(NK * 3));
  CU(ctx->scale.alloc((size_t)N * 3));
  ctx->real = f != nullptr;
  CU(ctx->W1T.alloc(g ? 96 * 36 : 0));
  CU(ctx->W2T.alloc(g ? kNOut * 32 : 0));
  CU(ctx->b1s.alloc(g ? 96 : 0));
  CU(ctx->b2s.alloc(g ? kNOut : 0));
  CU(ctx->featf.alloc(f ? (size_t)N * kF : 0));
  const int w1rows = f ? 35 + f->dist_input : 0;
  ctx->dist_input = f && f->dist_input;
  ctx->bank = f && f->feature_bank;
  CU(ctx->W1f.alloc((size_t)w1rows * 96));
  CU(ctx->Wb1f.alloc(ctx->bank ? 4 * kF : 0));
  CU(ctx->bb1f.alloc(ctx->bank ? kF : 0));
  CU(ctx->Wb2f.alloc(ctx->bank ? kF * 3 : 0));
  CU(ctx->bb2f.alloc(ctx->bank ? 3 : 0));
  CU(ctx->b1f.alloc(f ? 96 : 0));
  CU(ctx->W2f.alloc(f ? 32 * kNOut : 0));
  CU(ctx->b2f.alloc(f ? kNOut : 0));
  DevBuf<float> pos;
  CU(pos.alloc((size_t)N * 3));
  CU(cudaMemcpy(pos.p, s->pos, (size_t)N * 12, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(ctx->level.p, s->level, N, cudaMemcpyHostToDevice));
  CU(ctx->feat.alloc(g ? (size_t)N * kF : 0));
  if (g) CU(cudaMemcpy(ctx->feat.p, g->feat, (size_t)N * kF, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(ctx->offs.p, s->offs, NK * 12, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(ctx->scale.p, s->scale, (size_t)N * 12, cudaMemcpyHostToDevice));
  if (g) {
    CU(cudaMemcpy(ctx->W1T.p, W1T.data(), W1T.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->W2T.p, W2T.data(), W2T.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->b1s.p, b1s.data(), 96 * 4, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->b2s.p, b2s.data(), kNOut * 4, cudaMemcpyHostToDevice));
  } else {
    CU(cudaMemcpy(ctx->featf.p, f->feat, (size_t)N * kF * 4, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->W1f.p, f->W1, (size_t)w1rows * 96 * 4, cudaMemcpyHostToDevice));
    if (ctx->bank) {
      CU(cudaMemcpy(ctx->Wb1f.p, f->Wb1, 4 * kF * 4, cudaMemcpyHostToDevice));
      CU(cudaMemcpy(ctx->bb1f.p, f->bb1, kF * 4, cudaMemcpyHostToDevice));
      CU(cudaMemcpy(ctx->Wb2f.p, f->Wb2, kF * 3 * 4, cudaMemcpyHostToDevice));
      CU(cudaMemcpy(ctx->bb2f.p, f->bb2, 3 * 4, cudaMemcpyHostToDevice));
    }
    CU(cudaMemcpy(ctx->b1f.p, f->b1, 96 * 4, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->W2f.p, W2f.data(), W2f.size() * 4, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->b2f.p, b2f.data(), kNOut * 4, cudaMemcpyHostToDevice));
  }
  launch_margin(N, pos.p, ctx->offs.p, ctx->scale.p, ctx->pos_m.p, nullptr);
  CU(cudaGetLastError());
  // cache + per-frame buffers
  CU(ctx->birth.alloc(N));
  const size_t words = ((size_t)N + 31) / 32 + 1;
  CU(ctx->vis[0].alloc(words));
  CU(ctx->vis[1].alloc(words));
  CU(ctx->miss_bits.alloc(words));
  CU(ctx->alpha.alloc(NK));
  CU(ctx->pool.alloc(NK * 3));
  CU(cudaMemset(ctx->alpha.p, 0, NK * 4));
  CU(cudaMemset(ctx->pool.p, 0, NK * 48));
  CU(ctx->visible.alloc(N));
  CU(ctx->misses.alloc(N));
  ctx->cap_splat = 2 * NK;
  for (auto &S : ctx->fs) {
    CU(S.spA.alloc(ctx->cap_splat));
    CU(S.spB.alloc(ctx->cap_splat));
    CU(S.spC.alloc(ctx->cap_splat));
  }
  CU(ctx->count.alloc(ctx->cap_splat));
  CU(ctx->live_g.alloc(ctx->cap_splat / 2));
  CU(ctx->live_bits.alloc(ctx->cap_splat / 64 + 1));
  CU(ctx->dkey_a.alloc(ctx->cap_splat));
  CU(ctx->dval_a.alloc(ctx->cap_splat));
  CU(ctx->dkey_b.alloc(ctx->cap_splat));
  CU(ctx->dval_b.alloc(ctx->cap_splat));
  int64_t pc = ctx->cfg.pair_capacity > 0 ? ctx->cfg.pair_capacity : std::max<int64_t>(1 << 24, 4 * (int64_t)NK);
  pc = std::min<int64_t>(pc, (1LL << 30) - 1);
  ctx->cap_pairs = (size_t)pc;
  CU(ctx->list_off.alloc(ctx->cap_splat));
  CU(ctx->pair_off.alloc(ctx->cap_splat));
  CU(ctx->list.alloc(std::min<size_t>(2 * ctx->cap_pairs, (1u << 31) - 1)));
  CU(ctx->pkey_b.alloc(ctx->cap_pairs));
  CU(ctx->fixup.alloc(2 * (size_t)ctx->cfg.width * ctx->cfg.height));
  CU(ctx->pval_b.alloc(ctx->cap_pairs));
  const int TW = (ctx->cfg.width + 15) / 16, TH = (ctx->cfg.height + 15) / 16;
  for (auto &S : ctx->fs) {
    CU(S.pkey.alloc(ctx->cap_pairs));
    CU(S.pval.alloc(ctx->cap_pairs));
    CU(S.ranges.alloc(2 * (size_t)TW * TH));
  }
  const size_t stiles = (std::max(ctx->cap_splat, ctx->cap_pairs) + sort_tile_size() - 1) / sort_tile_size();
  CU(ctx->sort_status_a.alloc(stiles * 256));
  CU(ctx->sort_status_b.alloc(stiles * 256));
  CU(cudaMemset(ctx->sort_status_a.p, 0, stiles * 1024));
  CU(cudaMemset(ctx->sort_status_b.p, 0, stiles * 1024));
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  ctx->off_cull = al(sizeof(FrameCounters));
  ctx->off_proj = ctx->off_cull + al((size_t)cull_tiles(N) * 8);
  ctx->off_emit = ctx->off_proj + al((ctx->cap_splat / 2 + project_tile_size() - 1) / project_tile_size() * 4);
  ctx->zero_bytes = ctx->off_emit + al((ctx->cap_splat + emit_tile_size() - 1) / emit_tile_size() * 4);
  for (auto &S : ctx->fs) {
    CU(S.zero_region.alloc(ctx->zero_bytes));
    CU(cudaMemset(S.zero_region.p, 0, ctx->zero_bytes));
  }
  // device staging images of the host-buffer calls (either format; per frame parity and eye)
  for (auto &par : ctx->img_dev)
    for (auto &im : par)
      if (im.n < (size_t)ctx->cfg.width * ctx->cfg.height * 12) CU(im.alloc((size_t)ctx->cfg.width * ctx->cfg.height * 12));
  CU(cudaDeviceSynchronize());
  ctx->have_scene = true;
  return reset_cache(ctx, nullptr);
}

static gsc_status reset_cache(gsc_ctx *ctx, cudaStream_t st) {
  if (!ctx->have_scene) return fail(ctx, GSC_ESTATE, "no scene loaded");
  fill_i32<<<ctx->num_sms * 4, 256, 0, st>>>(ctx->birth.p, ctx->N, INT32_MIN);
  CU(cudaGetLastError());
  CU(cudaMemsetAsync(ctx->vis[0].p, 0, ctx->vis[0].n * 4, st));
  CU(cudaMemsetAsync(ctx->vis[1].p, 0, ctx->vis[1].n * 4, st));
  PolicyState ps{};
  ps.frame = 0;
  ps.depth = ctx->cfg.d_max;              // Alg. 1 l.182 / frame 0 keeps D_max
  ps.W = -ctx->cfg.d_max;                 // W_0 = 0 - depth_0
  ps.d_max = ctx->cfg.d_max;
  ps.literal = (ctx->cfg.flags & GSC_F_DEPTH_LITERAL) ? 1 : 0;
  ps.guide = (ctx->cfg.flags & GSC_F_GUIDE_EXP) ? 1 : (ctx->cfg.flags & GSC_F_GUIDE_STAGED) ? 2 : 0;
  ps.stagger = (ctx->cfg.flags & GSC_F_STAGGER) ? 1 : 0;
  CU(cudaMemcpyAsync(ctx->policy.p, &ps, sizeof(ps), cudaMemcpyHostToDevice, st));
  CU(cudaStreamSynchronize(st));
  return GSC_OK;
}

// ----------------------------------------------------------------------------------- GSC2 file
static gsc_status load_file(gsc_ctx *ctx, const char *path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return fail(ctx, GSC_EINVAL, std::string("cannot open ") + path);
  std::vector<char> buf((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  const size_t hdr = 4 + 6 * 4 + 4 + 24;
  if (buf.size() < hdr) return fail(ctx, GSC_EFORMAT, "truncated header at offset " + std::to_string(buf.size()));
  if (std::memcmp(buf.data(), "GSC2", 4) != 0) return fail(ctx, GSC_EFORMAT, "bad magic at offset 0");
  uint32_t u[6];
  std::memcpy(u, buf.data() + 4, 24);
  if (u[0] < 2 || u[0] > 4) return fail(ctx, GSC_EFORMAT, "unsupported version at offset 4");
  const bool real = u[0] >= 3;   // versions 3, 4: fp32 features and decoder weights (F4)
  const size_t q = real ? 4 : 1;
  const uint32_t N = u[1], F = u[2], K = u[3], L = u[4], H = u[5];
  if (F != (uint32_t)kF || K != (uint32_t)kK || H != (uint32_t)kH)
    return fail(ctx, GSC_EFORMAT, "unsupported F/K/H at offset 12 (need 32/10/32)");
  float d0;
  std::memcpy(&d0, buf.data() + 28, 4);
  size_t off = hdr;
  uint32_t flags = 0;   // version 4: bit 0 distance input, bit 1 feature bank (R32)
  if (u[0] == 4) {
    if (off + 4 > buf.size()) return fail(ctx, GSC_EFORMAT, "truncated at offset " + std::to_string(off));
    std::memcpy(&flags, buf.data() + off, 4);
    off += 4;
    if (flags > 3) return fail(ctx, GSC_EFORMAT, "unknown flags at offset " + std::to_string(off - 4));
  }
  const uint32_t dist = flags & 1u, bank = (flags >> 1) & 1u;
  auto take = [&](size_t bytes, const char *what, const void **ptr) -> bool {
    if (off + bytes > buf.size()) return false;
    *ptr = buf.data() + off;
    off += bytes;
    return true;
  };
  const void *p[17];
  const size_t bytes[17] = {N * 12ull, N * 32ull * q, N * 120ull, N * 12ull, N * 1ull, (35 + dist) * 96ull * q,
                            96ull * q, 32 * 10ull * q, 10ull * q, 32 * 30ull * q, 30ull * q, 32 * 70ull * q, 70ull * q,
                            4 * 32ull * 4, 32ull * 4, 32 * 3ull * 4, 3ull * 4};
  const int narr = bank ? 17 : 13;
  for (int k = 0; k < narr; ++k)
    if (!take(bytes[k], "", &p[k])) return fail(ctx, GSC_EFORMAT, "truncated at offset " + std::to_string(off));
  // (the file buffer is char-aligned: copy the f32 / int8 arrays through vectors of their type)
  auto fv = [&](int k) { std::vector<float> v(bytes[k] / 4); std::memcpy(v.data(), p[k], bytes[k]); return v; };
  std::vector<float> pos = fv(0), offs = fv(2), scale = fv(3);
  if (real) {
    std::vector<float> w[17];
    for (int k : {1, 5, 6, 7, 8, 9, 10, 11, 12}) w[k] = fv(k);
    if (bank)
      for (int k : {13, 14, 15, 16}) w[k] = fv(k);
    gsc_scene_desc_f32 d{(int32_t)N, (int32_t)L, d0, pos.data(), w[1].data(), offs.data(), scale.data(),
                         (const uint8_t *)p[4], w[5].data(), w[6].data(), w[7].data(), w[8].data(), w[9].data(),
                         w[10].data(), w[11].data(), w[12].data(), (int32_t)dist, (int32_t)bank,
                         bank ? w[13].data() : nullptr, bank ? w[14].data() : nullptr,
                         bank ? w[15].data() : nullptr, bank ? w[16].data() : nullptr};
    return upload_scene(ctx, nullptr, &d);
  }
  gsc_scene_desc d{};
  d.n_anchors = (int32_t)N; d.lod_levels = (int32_t)L; d.d0 = d0;
  d.pos = pos.data(); d.feat = (const int8_t *)p[1]; d.offs = offs.data(); d.scale = scale.data();
  d.level = (const uint8_t *)p[4]; d.W1 = (const int8_t *)p[5]; d.b1 = (const int8_t *)p[6];
  d.W2a = (const int8_t *)p[7]; d.b2a = (const int8_t *)p[8]; d.W2c = (const int8_t *)p[9];
  d.b2c = (const int8_t *)p[10]; d.W2s = (const int8_t *)p[11]; d.b2s = (const int8_t *)p[12];
  return upload_scene(ctx, &d, nullptr);
}

// ----------------------------------------------------------------------------------- frame
// Streams and events, created once at gsc_create (nothing is created or allocated inside a frame).
static gsc_status ensure_streams(gsc_ctx *ctx) {
  if (ctx->sA) return GSC_OK;
  // (stream priorities were measured to make no difference: the two stages share every SM)
  CU(cudaStreamCreateWithFlags(&ctx->sA, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&ctx->sB, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
  for (int k = 0; k < 2; ++k) {
    CU(cudaEventCreateWithFlags(&ctx->ev_user[k], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ctx->ev_a[k], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ctx->ev_b[k], cudaEventDisableTiming));
  }
  for (auto &e : ctx->host_done) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return GSC_OK;
}

// Capacity overflows of frames rendered without a stats request are reported (GSC_ECAPACITY, naming the
// frame) by the next call that knows the frame finished: gsc_render_pair (non-blocking, from the
// blend-done events), gsc_sync, gsc_wait_frame, gsc_render_pair_host.  Each overflowed frame is
// reported once.
static gsc_status check_done(gsc_ctx *ctx, int64_t upto) {
  if (upto - ctx->frames_checked > kRing) ctx->frames_checked = upto - kRing;   // (ring overwritten)
  while (ctx->frames_checked < upto) {
    const int64_t f = ctx->frames_checked++;
    const FrameRecordDev &r = ctx->rec_host[f % kRing];
    if (r.overflow)
      return fail(ctx, GSC_ECAPACITY, "frame " + std::to_string(f) + " exceeded the pair capacity (needed " +
                                          std::to_string(r.n_pairs_raw) + " pairs); its image is incomplete");
  }
  return GSC_OK;
}

static gsc_status check_finished_nonblocking(gsc_ctx *ctx) {
  for (int64_t back = 1; back <= 2 && back <= ctx->frames_rendered; ++back) {
    const int64_t f = ctx->frames_rendered - back;
    if (f < ctx->frames_checked) break;
    const cudaError_t q = cudaEventQuery(ctx->ev_b[f & 1]);   // last recorded by frame f
    if (q == cudaSuccess) return check_done(ctx, f + 1);
    if (q != cudaErrorNotReady) return fail(ctx, GSC_ECUDA, std::string("cudaEventQuery: ") + cudaGetErrorString(q));
    if (cudaPeekAtLastError() == cudaErrorNotReady) (void)cudaGetLastError();
  }
  return GSC_OK;
}

// One frame = front end a1..a7 on stream sA, then blend a8 on stream sB, into frame set f & 1.  The
// caller's stream `st` orders only the output images: the blend waits for the caller's earlier work
// on `st`, and `st` waits for the blend.  Frame f+1's front end thus overlaps frame f's blend; it
// waits for the blend of frame f-1, the last reader of the set it overwrites.
static gsc_status render(gsc_ctx *ctx, void *out_l, void *out_r, int fmt, cudaStream_t st) {
  if (ctx->sticky) return fail(ctx, GSC_ECUDA, "context has a sticky CUDA error: " + ctx->err);
  if (!ctx->have_scene || !ctx->have_pose) return fail(ctx, GSC_ESTATE, "render before load_scene/set_pose");
  if (!out_l || !out_r || (fmt != GSC_FMT_RGB_F32_PLANAR && fmt != GSC_FMT_RGBA8))
    return fail(ctx, GSC_EINVAL, "bad output buffers or format");
  {
    const gsc_status cs = check_finished_nonblocking(ctx);
    if (cs != GSC_OK) return cs;
  }
  ctx->last_stream = st;
  const int slot_i = (int)(ctx->frames_rendered % kRing);
  const int k = (int)(ctx->frames_rendered & 1);
  auto &S = ctx->fs[k];
  // GSC_F_SERIAL: one internal stream, so consecutive frames do not overlap (stage times add up)
  cudaStream_t sA = ctx->sA, sB = (ctx->cfg.flags & GSC_F_SERIAL) ? ctx->sA : ctx->sB;
  FrameSlot &slot = ctx->slots[slot_i];
  const bool timed = (ctx->cfg.flags & GSC_F_STAGE_TIMING) != 0;
  if (timed && !slot.timed) {
    for (int e = 0; e < kEvents; ++e) CU(cudaEventCreate(&slot.ev[e]));
    slot.timed = true;
  }
  int evk = 0;
  auto mark = [&](cudaStream_t s) { if (timed) cudaEventRecord(slot.ev[evk++], s); };
  CU(cudaEventRecord(ctx->ev_user[k], st));
  if (ctx->b_pending[k]) CU(cudaStreamWaitEvent(sA, ctx->ev_b[k], 0));   // blend f-2 done with set k
  FrameCounters *ctr = S.ctr();
  ctx->fc.ablate = ((ctx->cfg.flags & GSC_F_ABL_FIXED_EXTENT) ? kAblFixedExtent : 0) |
                   ((ctx->cfg.flags & GSC_F_ABL_AABB_TILES) ? kAblAabbTiles : 0) |
                   ((ctx->cfg.flags & GSC_F_MONO) ? kAblMono : 0);
  const FrameC &fc = ctx->fc;
  mark(sA);
  CU(cudaMemsetAsync(S.zero_region.p, 0, ctx->zero_bytes, sA));
  CU(cudaMemsetAsync(S.ranges.p, 0, S.ranges.n * sizeof(uint2), sA));
  const int cur = ctx->vis_cur;
  // a1 + a2
  launch_cull(fc, ctx->N, ctx->pos_m.p, ctx->level.p, ctx->birth.p, ctx->vis[cur ^ 1].p, ctx->vis[cur].p,
              ctx->miss_bits.p, ctx->visible.p, ctx->misses.p, reinterpret_cast<unsigned long long *>(S.zero_region.p + ctx->off_cull),
              ctr, ctx->policy.p, ctx->rec_dev.p + slot_i, sA);
  mark(sA);
  // a3
  if (ctx->real)   // F4: fixed-order fp32 MLP on the CUDA cores
    launch_derive_f32(ctx->pu, ctx->misses.p, ctx->pos_m.p, ctx->featf.p, ctx->offs.p, ctx->scale.p, ctx->W1f.p,
                      ctx->b1f.p, ctx->W2f.p, ctx->b2f.p,
                      CombineF32{ctx->dist_input ? 1 : 0, ctx->bank ? 1 : 0, ctx->Wb1f.p, ctx->bb1f.p, ctx->Wb2f.p,
                                 ctx->bb2f.p},
                      ctx->alpha.p, ctx->pool.p, ctr, ctx->num_sms, sA);
  else
    launch_derive(ctx->pu, ctx->misses.p, ctx->pos_m.p, ctx->feat.p, ctx->offs.p, ctx->scale.p, ctx->W1T.p,
                  ctx->b1s.p, ctx->W2T.p, ctx->b2s.p, ctx->alpha.p, ctx->pool.p, ctr, ctx->num_sms,
                  (ctx->cfg.flags & GSC_F_DERIVE_CUDA_CORES) == 0, sA);
  mark(sA);
  // a4
  SplatBufs sb{S.spA.p, S.spB.p, S.spC.p, ctx->count.p, ctx->dkey_a.p, ctx->list_off.p, ctx->list.p,
               (uint32_t)ctx->list.n};
  launch_project(fc, ctx->visible.p, ctx->alpha.p, ctx->pool.p, ctx->live_g.p, ctx->live_bits.p, sb,
                 reinterpret_cast<uint32_t *>(S.zero_region.p + ctx->off_proj), ctr, ctx->num_sms, sA);
  mark(sA);
  // a5 (depth digits of the (tile, depth) sort)
  launch_onesweep(ctx->dkey_a.p, ctx->dval_a.p, ctx->dkey_b.p, ctx->dval_b.p, true, &ctr->n_splat, 4, 8,
                  &ctr->hist_depth[0][0], ctx->sort_status_a.p, ctx->sort_status_b.p, &ctr->tile_sort[0],
                  nullptr, ctx->num_sms, sA);
  mark(sA);
  // the tile keys (eye * T_e + tile) take 2 passes of 7-bit digits when they fit in 14 bits (1080p:
  // 2 T_e = 16320), else of 8-bit digits: 128 bins scatter in longer runs than 256
  const int tbits = 2 * fc.Te <= (1 << 14) ? 7 : 8;
  EmitIn ei{ctx->dval_a.p, ctx->count.p, ctx->list_off.p, ctx->list.p, ctx->pair_off.p};
  launch_emit(ei, (uint32_t)ctx->cap_pairs, S.pkey.p, S.pval.p,
              reinterpret_cast<uint32_t *>(S.zero_region.p + ctx->off_emit), ctr, tbits, ctx->num_sms, sA);
  mark(sA);
  // a6 (tile digits) + a7 (tile ranges, derived by the last pass)
  launch_onesweep(S.pkey.p, S.pval.p, ctx->pkey_b.p, ctx->pval_b.p, false, &ctr->n_pairs, 2, tbits,
                  &ctr->hist_tile[0][0], ctx->sort_status_a.p, ctx->sort_status_b.p, &ctr->tile_sort[4],
                  S.ranges.p, ctx->num_sms, sA);
  mark(sA);
  mark(sA);   // (a7 has no kernel of its own any more; the stage boundary is kept for the stats layout)
  CU(cudaEventRecord(ctx->ev_a[k], sA));
  // a8 on sB, after the front end and after the caller's earlier work on its stream
  CU(cudaStreamWaitEvent(sB, ctx->ev_a[k], 0));
  CU(cudaStreamWaitEvent(sB, ctx->ev_user[k], 0));
  mark(sB);
  launch_blend(fc, S.ranges.p, S.pkey.p, S.pval.p, S.spA.p, S.spB.p, S.spC.p, out_l, out_r, fmt, ctr, ctx->fixup.p,
               (ctx->cfg.flags & GSC_F_COUNT_EVALS) != 0, (ctx->cfg.flags & GSC_F_BLEND_EXACT) != 0, ctx->num_sms, sB);
  launch_record(ctr, ctx->rec_dev.p + slot_i, sB);
  CU(cudaMemcpyAsync(ctx->rec_host + slot_i, ctx->rec_dev.p + slot_i, sizeof(FrameRecordDev), cudaMemcpyDeviceToHost,
                     sB));
  mark(sB);
  CU(cudaEventRecord(ctx->ev_b[k], sB));
  ctx->b_pending[k] = true;
  CU(cudaStreamWaitEvent(st, ctx->ev_b[k], 0));
  CU(cudaGetLastError());
  slot.used = true;
  ctx->vis_cur ^= 1;
  ++ctx->frames_rendered;
  return GSC_OK;
}

static void fill_stats(gsc_ctx *ctx, int64_t frame_seq, gsc_frame_stats *s) {
  const int slot_i = (int)(frame_seq % kRing);
  const FrameRecordDev &r = ctx->rec_host[slot_i];
  std::memset(s, 0, sizeof(*s));
  s->frame = r.frame;
  s->n_visible = r.n_visible;
  s->n_misses = r.n_miss;
  s->n_hits = r.n_visible - r.n_miss;
  s->n_new = r.n_new;
  s->n_splats = r.n_splat;
  s->n_pairs = r.n_pairs_raw;
  s->overflow = r.overflow;
  s->n_evals = r.n_evals;
  s->n_exp = r.n_exp;
  s->n_evals_list = r.n_evals_list;
  s->n_nonfinite_skipped = r.n_nonfinite;
  s->n_blend_fixup = r.n_fixup;
  s->depth_used = r.depth_used;
  s->depth_next = r.depth_next;
  s->update_rate = r.n_visible ? (float)r.n_miss / (float)r.n_visible : 0.0f;
  s->novelty_rate = r.n_visible ? (float)r.n_new / (float)r.n_visible : 0.0f;
  FrameSlot &slot = ctx->slots[slot_i];
  if (slot.timed && (ctx->cfg.flags & GSC_F_STAGE_TIMING)) {
    // ev 0..7 on the front-end stream, ev 8..9 around the blend on the blend stream (the blend of
    // frame f overlaps the front end of frame f+1, so the stage times may sum to more than the
    // frame period)
    float ms[8] = {0};
    for (int k = 0; k < 7; ++k) cudaEventElapsedTime(&ms[k], slot.ev[k], slot.ev[k + 1]);
    cudaEventElapsedTime(&ms[7], slot.ev[8], slot.ev[9]);
    s->ms_cull = ms[0]; s->ms_derive = ms[1]; s->ms_project = ms[2]; s->ms_depth_sort = ms[3];
    s->ms_emit = ms[4]; s->ms_tile_sort = ms[5]; s->ms_ranges = ms[6]; s->ms_blend = ms[7];
    cudaEventElapsedTime(&s->ms_total, slot.ev[0], slot.ev[9]);
    (void)cudaGetLastError();   // an event query must not leave a sticky error behind
  }
}

// ----------------------------------------------------------------------------------- C ABI
extern "C" {

int gsc_abi_version(void) { return GSC_ABI_VERSION; }

gsc_status gsc_create(int cuda_device, const gsc_config *cfg, gsc_ctx **out) {
  if (!out) return GSC_EINVAL;
  *out = nullptr;
  if (!cfg_valid(cfg)) return GSC_EINVAL;
  std::unique_ptr<gsc_ctx> c(new gsc_ctx());
  gsc_ctx *ctx = c.get();
  ctx->device = cuda_device;
  ctx->cfg = *cfg;
  CU(cudaSetDevice(cuda_device));
  CU(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cuda_device));
  CU(ctx->policy.alloc(1));
  CU(ctx->rec_dev.alloc(kRing));
  CU(cudaMallocHost(&ctx->rec_host, kRing * sizeof(FrameRecordDev)));
  std::memset(ctx->rec_host, 0, kRing * sizeof(FrameRecordDev));
  if (ensure_streams(ctx) != GSC_OK) return GSC_ECUDA;
  *out = c.release();
  return GSC_OK;
}

gsc_status gsc_load_scene(gsc_ctx *ctx, const char *path) {
  if (!ctx || !path) return GSC_EINVAL;
  CU(cudaSetDevice(ctx->device));
  return load_file(ctx, path);
}

gsc_status gsc_load_scene_host(gsc_ctx *ctx, const gsc_scene_desc *scene) {
  if (!ctx || !scene) return GSC_EINVAL;
  CU(cudaSetDevice(ctx->device));
  return upload_scene(ctx, scene, nullptr);
}

gsc_status gsc_load_scene_host_f32(gsc_ctx *ctx, const gsc_scene_desc_f32 *scene) {
  if (!ctx || !scene) return GSC_EINVAL;
  CU(cudaSetDevice(ctx->device));
  return upload_scene(ctx, nullptr, scene);
}

gsc_status gsc_set_pose(gsc_ctx *ctx, const gsc_rig *rig) {
  if (!ctx || !rig) return GSC_EINVAL;
  gsc_status s = compute_frame_consts(ctx, rig);
  if (s == GSC_OK) ctx->have_pose = true;
  return s;
}

gsc_status gsc_render_pair(gsc_ctx *ctx, void *out_left, void *out_right, int out_format, void *cuda_stream,
                           gsc_frame_stats *stats) {
  if (!ctx) return GSC_EINVAL;
  CU(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  gsc_status s = render(ctx, out_left, out_right, out_format, st);
  if (s != GSC_OK) return s;
  if (stats) {
    CU(cudaStreamSynchronize(st));
    fill_stats(ctx, ctx->frames_rendered - 1, stats);
    ctx->frames_reported = ctx->frames_rendered;
    return check_done(ctx, ctx->frames_rendered);
  }
  return GSC_OK;
}

// enqueue: pose, frame into the device staging images of its parity, D2H copies; all on own_stream
static gsc_status render_host_enqueue(gsc_ctx *ctx, const gsc_rig *rig, void *host_left, void *host_right,
                                      int out_format) {
  if (out_format != GSC_FMT_RGB_F32_PLANAR && out_format != GSC_FMT_RGBA8) return GSC_EINVAL;
  gsc_status s = gsc_set_pose(ctx, rig);
  if (s != GSC_OK) return s;
  const size_t bytes = (size_t)ctx->cfg.width * ctx->cfg.height * (out_format == GSC_FMT_RGBA8 ? 4 : 12);
  auto &img = ctx->img_dev[ctx->frames_rendered & 1];   // allocated at scene load for either format
  s = render(ctx, img[0].p, img[1].p, out_format, ctx->own_stream);
  if (s != GSC_OK) return s;
  CU(cudaMemcpyAsync(host_left, img[0].p, bytes, cudaMemcpyDeviceToHost, ctx->own_stream));
  CU(cudaMemcpyAsync(host_right, img[1].p, bytes, cudaMemcpyDeviceToHost, ctx->own_stream));
  return GSC_OK;
}

gsc_status gsc_render_pair_host(gsc_ctx *ctx, const gsc_rig *rig, void *host_left, void *host_right, int out_format,
                                gsc_frame_stats *stats) {
  if (!ctx || !rig || !host_left || !host_right) return GSC_EINVAL;
  CU(cudaSetDevice(ctx->device));
  gsc_status s = render_host_enqueue(ctx, rig, host_left, host_right, out_format);
  if (s != GSC_OK) return s;
  CU(cudaStreamSynchronize(ctx->own_stream));
  if (stats) fill_stats(ctx, ctx->frames_rendered - 1, stats);
  return check_done(ctx, ctx->frames_rendered);
}

gsc_status gsc_render_pair_host_async(gsc_ctx *ctx, const gsc_rig *rig, void *host_left, void *host_right,
                                      int out_format, long long *seq) {
  if (!ctx || !rig || !host_left || !host_right || !seq) return GSC_EINVAL;
  CU(cudaSetDevice(ctx->device));
  const int64_t q = ctx->host_submitted;
  auto &ev = ctx->host_done[q % gsc_ctx::kHostRing];
  if (q >= gsc_ctx::kHostRing) CU(cudaEventSynchronize(ev));   // the slot's previous frame (kHostRing in flight)
  gsc_status s = render_host_enqueue(ctx, rig, host_left, host_right, out_format);
  if (s != GSC_OK) return s;
  CU(cudaEventRecord(ev, ctx->own_stream));
  ctx->host_frame[q % gsc_ctx::kHostRing] = ctx->frames_rendered - 1;
  *seq = q;
  ++ctx->host_submitted;
  return GSC_OK;
}

gsc_status gsc_wait_frame(gsc_ctx *ctx, long long seq) {
  if (!ctx || seq < 0 || seq >= ctx->host_submitted) return GSC_EINVAL;
  CU(cudaSetDevice(ctx->device));
  if (seq + gsc_ctx::kHostRing <= ctx->host_submitted) return GSC_OK;   // its slot was already waited for
  CU(cudaEventSynchronize(ctx->host_done[seq % gsc_ctx::kHostRing]));
  return check_done(ctx, ctx->host_frame[seq % gsc_ctx::kHostRing] + 1);
}

gsc_status gsc_sync(gsc_ctx *ctx, void *cuda_stream) {
  if (!ctx) return GSC_EINVAL;
  CU(cudaSetDevice(ctx->device));
  CU(cudaStreamSynchronize((cudaStream_t)cuda_stream));
  if (ctx->own_stream) CU(cudaStreamSynchronize(ctx->own_stream));
  if (ctx->sA) CU(cudaStreamSynchronize(ctx->sA));
  if (ctx->sB) CU(cudaStreamSynchronize(ctx->sB));
  return check_done(ctx, ctx->frames_rendered);
}

gsc_status gsc_stats_history(gsc_ctx *ctx, gsc_frame_stats *dst, int max, int *n) {
  if (!ctx || !n || (max > 0 && !dst)) return GSC_EINVAL;
  int64_t first = std::max(ctx->frames_reported, ctx->frames_rendered - (int64_t)kRing);
  int64_t cnt = ctx->frames_rendered - first;
  if (cnt > max) { first = ctx->frames_rendered - max; cnt = max; }
  for (int64_t k = 0; k < cnt; ++k) fill_stats(ctx, first + k, dst + k);
  *n = (int)cnt;
  ctx->frames_reported = ctx->frames_rendered;
  return GSC_OK;
}

gsc_status gsc_reset_cache(gsc_ctx *ctx) {
  if (!ctx) return GSC_EINVAL;
  CU(cudaSetDevice(ctx->device));
  CU(cudaDeviceSynchronize());
  return reset_cache(ctx, nullptr);
}

gsc_status gsc_set_flags(gsc_ctx *ctx, unsigned flags) {
  if (!ctx) return GSC_EINVAL;
  const unsigned known =
      GSC_F_DEPTH_LITERAL | GSC_F_STAGE_TIMING | GSC_F_DERIVE_CUDA_CORES | GSC_F_COUNT_EVALS | GSC_F_SERIAL |
      GSC_F_GUIDE_EXP | GSC_F_GUIDE_STAGED | GSC_F_ABL_FIXED_EXTENT | GSC_F_ABL_AABB_TILES | GSC_F_MONO | GSC_F_STAGGER |
      GSC_F_BLEND_EXACT;
  if (flags & ~known) return fail(ctx, GSC_EINVAL, "unknown flag bits");
  if ((flags & GSC_F_GUIDE_EXP) && (flags & GSC_F_GUIDE_STAGED)) return fail(ctx, GSC_EINVAL, "two guiding functions");
  CU(cudaSetDevice(ctx->device));
  CU(cudaDeviceSynchronize());
  ctx->cfg.flags = flags;
  return GSC_OK;
}

gsc_status gsc_debug_fetch(gsc_ctx *ctx, int what, void *host_dst, size_t cap, size_t *len) {
  if (!ctx || !len) return GSC_EINVAL;
  CU(cudaSetDevice(ctx->device));
  CU(cudaDeviceSynchronize());
  if (!ctx->have_scene || ctx->frames_rendered == 0) return fail(ctx, GSC_ESTATE, "no frame rendered");
  auto &S = ctx->last_set();
  FrameCounters c;
  CU(cudaMemcpy(&c, S.zero_region.p, sizeof(c), cudaMemcpyDeviceToHost));
  const size_t NK = (size_t)ctx->N * kK;
  const size_t ns = c.n_splat, np = c.n_pairs, nlive = ns / 2;
  auto copy_dev = [&](const void *src, size_t bytes) -> gsc_status {
    *len = bytes;
    if (host_dst && cap) CU(cudaMemcpy(host_dst, src, std::min(cap, bytes), cudaMemcpyDeviceToHost));
    return GSC_OK;
  };
  // splat c = eye * n_live + i is live Gaussian live_g[i] (project.cu); its depth key sits in the
  // depth-sorted (key, splat) arrays of the frame's depth sort
  std::vector<uint32_t> gof, dof;
  auto load_g = [&]() -> gsc_status {
    std::vector<uint32_t> lg(nlive);
    if (nlive) CU(cudaMemcpy(lg.data(), ctx->live_g.p, nlive * 4, cudaMemcpyDeviceToHost));
    gof.resize(ns);
    for (size_t k = 0; k < ns; ++k) gof[k] = lg[k % nlive];
    return GSC_OK;
  };
  auto load_depth = [&]() -> gsc_status {
    std::vector<uint32_t> dk(ns), dv(ns);
    if (ns) {
      CU(cudaMemcpy(dk.data(), ctx->dkey_a.p, ns * 4, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(dv.data(), ctx->dval_a.p, ns * 4, cudaMemcpyDeviceToHost));
    }
    dof.assign(ns, 0xFFFFFFFFu);
    for (size_t k = 0; k < ns; ++k)
      if (dv[k] < ns) dof[dv[k]] = dk[k];
    return GSC_OK;
  };
  switch (what) {
    case GSC_DBG_VISIBLE: return copy_dev(ctx->visible.p, (size_t)c.n_visible * 4);
    case GSC_DBG_MISSES: return copy_dev(ctx->misses.p, (size_t)c.n_miss * 4);
    case GSC_DBG_BIRTH: return copy_dev(ctx->birth.p, (size_t)ctx->N * 4);
    case GSC_DBG_SPLAT_G: {
      *len = ns * 4;
      if (!host_dst || !cap) return GSC_OK;
      if (load_g() != GSC_OK) return GSC_ECUDA;
      std::memcpy(host_dst, gof.data(), std::min(cap, ns * 4));
      return GSC_OK;
    }
    case GSC_DBG_PAIR_G: {
      *len = np * 4;
      if (!host_dst || !cap) return GSC_OK;
      std::vector<uint32_t> pv(np);
      CU(cudaMemcpy(pv.data(), S.pval.p, np * 4, cudaMemcpyDeviceToHost));
      if (load_g() != GSC_OK) return GSC_ECUDA;
      std::vector<uint32_t> out(np);
      for (size_t k = 0; k < np; ++k) out[k] = gof[pv[k]];
      std::memcpy(host_dst, out.data(), std::min(cap, np * 4));
      return GSC_OK;
    }
    case GSC_DBG_PAIRS: {
      *len = np * 8;
      if (!host_dst || !cap) return GSC_OK;
      std::vector<uint32_t> pk(np), pv(np);
      CU(cudaMemcpy(pk.data(), S.pkey.p, np * 4, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(pv.data(), S.pval.p, np * 4, cudaMemcpyDeviceToHost));
      if (load_depth() != GSC_OK) return GSC_ECUDA;
      std::vector<uint64_t> out(np);
      for (size_t k = 0; k < np; ++k)
        out[k] = ((uint64_t)(pk[k] & 0x00FFFFFFu) << 32) | dof[pv[k]];   // bits 24..31: blend block mask
      std::memcpy(host_dst, out.data(), std::min(cap, np * 8));
      return GSC_OK;
    }
    case GSC_DBG_RANGES: {   // stored as (~start, end); untouched (empty) tiles as (0, 0)
      *len = S.ranges.n * 8;
      if (!host_dst || !cap) return GSC_OK;
      std::vector<uint2> rg(S.ranges.n);
      CU(cudaMemcpy(rg.data(), S.ranges.p, S.ranges.n * 8, cudaMemcpyDeviceToHost));
      for (auto &r : rg) r = r.x ? make_uint2(~r.x, r.y) : make_uint2(0u, 0u);
      std::memcpy(host_dst, rg.data(), std::min(cap, rg.size() * 8));
      return GSC_OK;
    }
    case GSC_DBG_POOL: {
      *len = NK * 13 * 4;
      if (!host_dst || !cap) return GSC_OK;
      std::vector<float> a(NK);
      std::vector<float4> p(NK * 3);
      CU(cudaMemcpy(a.data(), ctx->alpha.p, NK * 4, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(p.data(), ctx->pool.p, NK * 48, cudaMemcpyDeviceToHost));
      std::vector<float> out(NK * 13);
      for (size_t g = 0; g < NK; ++g) {
        const float4 &q0 = p[3 * g], &q1 = p[3 * g + 1], &q2 = p[3 * g + 2];
        float r[13] = {a[g], q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z, q2.w};
        std::memcpy(&out[13 * g], r, sizeof(r));
      }
      std::memcpy(host_dst, out.data(), std::min(cap, out.size() * 4));
      return GSC_OK;
    }
    case GSC_DBG_SPLATS: {
      *len = ns * 13 * 4;
      if (!host_dst || !cap) return GSC_OK;
      std::vector<float4> A(ns), B(ns);
      std::vector<float2> Cc(ns);
      std::vector<uint32_t> cn(ns);
      CU(cudaMemcpy(A.data(), S.spA.p, ns * 16, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(B.data(), S.spB.p, ns * 16, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(Cc.data(), S.spC.p, ns * 8, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(cn.data(), ctx->count.p, ns * 4, cudaMemcpyDeviceToHost));
      if (load_depth() != GSC_OK) return GSC_ECUDA;
      std::vector<float> out(ns * 13);
      const float nan = std::nanf("");
      for (size_t k = 0; k < ns; ++k) {
        // records hold (u, v, -A/2, -B), (-C/2, bound, alpha, r), (g, b); -2 x (-A/2) is exact.  thr is not
        // kept per splat (NaN here); the kept-tile count and the sorted keys it decides are.
        float depth;
        std::memcpy(&depth, &dof[k], 4);
        float r[13] = {A[k].x, A[k].y, -2.0f * A[k].z, -A[k].w, -2.0f * B[k].x, B[k].z, B[k].w, Cc[k].x, Cc[k].y,
                       depth, nan, (float)(k >= nlive), (float)cn[k]};
        std::memcpy(&out[13 * k], r, sizeof(r));
      }
      std::memcpy(host_dst, out.data(), std::min(cap, out.size() * 4));
      return GSC_OK;
    }
    default: return fail(ctx, GSC_EINVAL, "unknown debug selector");
  }
}

gsc_status gsc_selftest_elementary(gsc_ctx *ctx, int fn, const float *dev_in, float *dev_out, size_t n) {
  if (!ctx || fn < 0 || fn > 5 || (n && (!dev_in || !dev_out))) return GSC_EINVAL;
  CU(cudaSetDevice(ctx->device));
  launch_elem(fn, dev_in, dev_out, n, ctx->num_sms, nullptr);
  CU(cudaGetLastError());
  CU(cudaDeviceSynchronize());
  return GSC_OK;
}

const char *gsc_last_error(const gsc_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void gsc_destroy(gsc_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (auto &s : ctx->slots)
    if (s.timed)
      for (int k = 0; k < kEvents; ++k) cudaEventDestroy(s.ev[k]);
  if (ctx->rec_host) cudaFreeHost(ctx->rec_host);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  for (int k = 0; k < 2; ++k) {
    if (ctx->ev_user[k]) cudaEventDestroy(ctx->ev_user[k]);
    if (ctx->ev_a[k]) cudaEventDestroy(ctx->ev_a[k]);
    if (ctx->ev_b[k]) cudaEventDestroy(ctx->ev_b[k]);
  }
  for (auto &e : ctx->host_done)
    if (e) cudaEventDestroy(e);
  if (ctx->sA) cudaStreamDestroy(ctx->sA);
  if (ctx->sB) cudaStreamDestroy(ctx->sB);
  delete ctx;
}

}  // extern "C"
