/*
 * ddvr.h -- C ABI of the B200-native differentiable emission-absorption
 * raymarcher (DiffDVR, arXiv 2107.12672).
 *
 * Drop-in boundary for the reference package ``voldiff`` (pure NumPy; it has
 * no FFI of its own).  Each entry point replaces one reference function on
 * the hot path -- the Python host side (paper_2107_12672_b200/_native.py) binds
 * them with ctypes exactly as a maintainer would from the reference:
 *
 *   ddvr_forward      <- voldiff.renderer.render              renderer.py:393-401
 *                        (_render_scene :376-390, _march_fused :306-357)
 *   ddvr_adjoint      <- voldiff.renderer.render_adjoint      renderer.py:688-700
 *                        (_adjoint_scene :655-685, _adjoint_tile :491-652)
 *   ddvr_ray_setup    <- voldiff.renderer._ray_setup/_step_counts  renderer.py:182-214, 360-368
 *   ddvr_l1_loss      <- voldiff.objectives.l1_loss            objectives.py:38-54
 *   ddvr_field_sample <- voldiff.field.trilinear_sample / trilinear_gradients
 *                                                              field.py:279-349, 379-517
 *   ddvr_tf_lookup    <- voldiff.field.tf_sample / tf_gradients field.py:525-579
 *   ddvr_opacity      <- voldiff.field.opacity_from_density   field.py:587-600
 *   ddvr_camera_rays  <- voldiff.field.camera_from_sphere / camera_gradients
 *                                                              field.py:186-271
 *   ddvr_last_error   <- the message of the raised voldiff error (errors.py:4-33)
 *
 * Conventions
 *   - every pointer marked (device) is CUDA device memory owned by the caller;
 *     nothing is allocated inside the library;
 *   - all calls are asynchronous and stream-ordered on ``stream`` (a
 *     cudaStream_t; NULL = legacy default stream);
 *   - gradient outputs ACCUMULATE (+=) into caller-zeroed buffers, so views can
 *     be summed across calls and reduced in place by NCCL;
 *   - volume layout (X,Y,Z) float32, z fastest (== ``values.ravel()``,
 *     field.py:311-324); images (V, rows, W, 4) float32 premultiplied rgb +
 *     alpha, row 0 = top (renderer.py:56-81, field.py:222);
 *   - return value is a ddvr_status; on error ddvr_last_error() (thread-local)
 *     holds the message.  Status codes map to the reference exceptions:
 *     INVALID_PARAMETER -> InvalidParameterError, INVALID_INPUT ->
 *     InvalidInputError, UNSUPPORTED -> UnsupportedConfigurationError.
 */
#ifndef DDVR_H
#define DDVR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DDVR_ABI_VERSION 4

typedef enum {
  DDVR_OK = 0,
  DDVR_INVALID_PARAMETER = 1,
  DDVR_INVALID_INPUT = 2,
  DDVR_UNSUPPORTED = 3,
  DDVR_CUDA_ERROR = 4
} ddvr_status;

/* differentiation targets (renderer.py:47); any non-empty combination */
typedef enum {
  DDVR_TARGET_CAMERA = 1,
  DDVR_TARGET_STEPSIZE = 2,
  DDVR_TARGET_TF = 4,
  DDVR_TARGET_VOLUME = 8
} ddvr_target;

/* transfer-function representations */
typedef enum {
  DDVR_TF_TEXTURE = 0,   /* R texels (r,g,b,tau), centres (r+.5)/R, clamp-to-edge (field.py:540-549) */
  DDVR_TF_PIECEWISE = 1, /* K knots (pos, r,g,b,tau), strictly increasing pos in [0,1] */
  DDVR_TF_GAUSSIAN = 2   /* G components (mu, sigma, r,g,b,tau): sum of bumps (tasks.py:751-766) */
} ddvr_tf_kind;

/* density grid on a world box (DensityVolume, field.py:35-77) */
typedef struct {
  const float* data;     /* (device) X*Y*Z floats, z fastest */
  int32_t dims[3];       /* X, Y, Z >= 1 */
  double box_min[3];
  double box_max[3];     /* box_max > box_min on every axis */
  const float* cells;    /* (device, nullable, 32-byte aligned) padded cell-record copy of
                            data built by ddvr_pack_cells: the 8 corner values of every
                            cell in one 32-byte record, so a sample is one 256-bit load.
                            NULL = gather the 8 corners from data. */
} ddvr_volume;

/* transfer function (TransferFunction, field.py:108-127) */
typedef struct {
  int32_t kind;          /* ddvr_tf_kind */
  int32_t count;         /* texture: R >= 1; piecewise: K >= 1; gaussian: G >= 1 */
  const float* params;   /* (device) texture (R,4); piecewise (K,5); gaussian (G,6) */
} ddvr_tf;

/* one spherical camera (SphericalCamera, field.py:130-156); arrays of these
 * live in DEVICE memory, one per view, so camera gradients can flow per view */
typedef struct {
  double lon_deg;
  double lat_deg;        /* |lat| < 90 - 1e-3 (validated by the host side) */
  double radius;         /* > 0 */
  double center[3];
  double fov_y_deg;      /* (0, 180) */
  double reserved;
} ddvr_camera;

#define DDVR_FLAG_WS_CONTINUE 1
#define DDVR_FLAG_WS_DEFER 2
#define DDVR_FLAG_DETERMINISTIC 4
#define DDVR_FLAG_BAND_TAPE 8
#define DDVR_FLAG_NO_EMPTY_SKIP 16
#define DDVR_FLAG_SPLIT_WALK 32
/* segment-split rays of a fused step (ddvr_forward_adjoint_l1, masks TF, TF|VOLUME and
   camera / stepsize alone): by default chosen from the ray count (ddvr_ray_split); these
   force it (at most one) */
#define DDVR_FLAG_RAY_SPLIT_OFF 64
#define DDVR_FLAG_RAY_SPLIT_2 128
#define DDVR_FLAG_RAY_SPLIT_4 256
#define DDVR_FLAG_RAY_SPLIT_8 512

/* march parameters (RenderConfig, renderer.py:84-106) */
typedef struct {
  double dt;             /* stepsize > 0 */
  int32_t width;         /* image size shared by all views, >= 1 */
  int32_t height;
  int32_t row0;          /* rows [row0, row1) are processed (row bands, renderer.py:491) */
  int32_t row1;          /* row1 <= 0 means height */
  int32_t early_stop;    /* 1: stop rays at alpha > 1-1e-4 (target "none", renderer.py:331-335) */
  int32_t flags;         /* 0, or for ddvr_adjoint / ddvr_forward_adjoint_l1 split over
                            several calls of one step (e.g. view chunks):
                            DDVR_FLAG_WS_CONTINUE  the workspace already holds this
                                                   step's partial gradients: not zeroed;
                            DDVR_FLAG_WS_DEFER     more calls follow: partial gradients
                                                   stay in the workspace (no fold into
                                                   d_volume, no reduction into d_tf)
                            DDVR_FLAG_DETERMINISTIC  (combinable) camera / stepsize
                                                   sums per CTA into the workspace,
                                                   reduced in a fixed order: d_camera
                                                   and d_dt bitwise reproducible
                                                   (ddvr_deterministic_bytes)
                            DDVR_FLAG_BAND_TAPE    (ddvr_forward_adjoint_l1, volume
                                                   target) the march records 1 bit
                                                   per sample -- whether the
                                                   absorption walk's d_hat is nonzero
                                                   -- and the walk reads it instead of
                                                   re-gathering the cell records
                                                   (ddvr_band_tape_bytes); identical
                                                   gradients, O(samples / 32) words.
                                                   With the empty-brick map in the
                                                   workspace the march also skips
                                                   32-sample blocks that lie in
                                                   all-zero 8^3-cell bricks (bitwise
                                                   the same outputs)
                            DDVR_FLAG_NO_EMPTY_SKIP  with DDVR_FLAG_BAND_TAPE: march
                                                   every block (no brick map)
                            DDVR_FLAG_SPLIT_WALK   with DDVR_FLAG_BAND_TAPE: march and
                                                   walk as two kernels (the march
                                                   hands each ray's walk weight to the
                                                   walk through the workspace,
                                                   ddvr_band_tape_bytes); by default
                                                   one kernel runs both per ray
                            DDVR_FLAG_RAY_SPLIT_OFF / _2 / _4 / _8  (fused step, TF
                                                   target without camera / stepsize)
                                                   threads per ray: 1, 2, 4 or 8
                                                   consecutive lanes march and walk
                                                   one sample segment each (default:
                                                   from the ray count) */
  float* tape;           /* (device, nullable) "stored" memory mode (renderer.py:507-513, 576-577):
                            forward writes the transmittance before every sample,
                            tape[ray * tape_stride + i]; the adjoint then reads it
                            instead of inverting.  NULL = inversion mode (default). */
  int64_t tape_stride;   /* >= max step count of any ray of the call */
  uint64_t* stats;       /* (device, nullable) 4 counters ADDED to by ddvr_forward_adjoint_l1
                            (measurement only): [0] samples of the call (sum of the
                            rays' step counts), [1] samples the march stepped over in
                            empty bricks, [2] samples the band-tape walk stepped over
                            (all-zero tape words), [3] rays.  Samples marched =
                            [0] - [1]; samples walked = [0] - [2]. */
} ddvr_params;

/* Front-to-back march of every view.  image_out (device) (V, rows, W, 4);
 * depth_out (device, nullable) (V, rows, W) receives each ray's optical depth
 * S = sum_i -ln(1 - a_i) = sum_i min(dt*tau_i, -ln EPS_ALPHA), summed in fp64
 * (transmittance T = exp(-S)).  The adjoint's inversion starts from it; it
 * never underflows, unlike T, and 1 - alpha loses T as alpha -> 1. */
int ddvr_forward(const ddvr_volume* vol, const ddvr_tf* tf, const ddvr_camera* cams,
                 int32_t n_views, const ddvr_params* p, float* image_out, float* depth_out,
                 void* stream);

/* Back-to-front adjoint with the inversion trick: per-ray state is O(1); no
 * per-sample tape.  image (device) (V, rows, W, 4) is the forward output for
 * the same inputs; depth (device, nullable) its optical-depth side output (if
 * NULL, S = -ln(1 - alpha)).  The walk inverts each compositing step exactly
 * in optical-depth form, S_prev = S + ln(1 - a), in fp64.
 * seed (device) (V, rows, W, 4) = dLoss/dImage.
 * Outputs (device, accumulate, NULL when the target bit is clear):
 *   d_volume float (X*Y*Z); d_tf double (same shape as tf->params);
 *   d_camera double (V, 2) per degree [lon, lat]; d_dt double (1).
 * workspace (device, 32-byte aligned): ddvr_adjoint_workspace_bytes() bytes
 * (cell-gradient records when vol->cells is set and the volume target is on,
 * TF-gradient slots when the tf target is on; zeroed, then folded into
 * d_volume / reduced into d_tf inside the call). */
int ddvr_adjoint(const ddvr_volume* vol, const ddvr_tf* tf, const ddvr_camera* cams,
                 int32_t n_views, const ddvr_params* p, const float* image, const float* depth,
                 const float* seed, uint32_t target_mask, float* d_volume, double* d_tf,
                 double* d_camera, double* d_dt, void* workspace, int64_t workspace_bytes,
                 void* stream);

/* One fused tomography step over n_views views (the render -> l1_loss ->
 * render_adjoint body of the reconstruction loop, tasks.py:397-481;
 * renderer.py:393-401, objectives.py:38-54, renderer.py:688-700): per ray, the
 * forward march, the L1 seed sign(image - ref) / count and the adjoint walk
 * run back to back in one kernel (the walk uses the exact fp64 optical depth).
 * refs (device) (V, rows, W, 4); count = the loss's global element count;
 * loss_out (device, double) += sum |image - ref| / count.  image_out and
 * depth_out (device, nullable) receive the rendered images.  Outputs and
 * workspace as ddvr_adjoint.  Needs vol->cells; no stored (tape) mode. */
int ddvr_forward_adjoint_l1(const ddvr_volume* vol, const ddvr_tf* tf, const ddvr_camera* cams,
                            int32_t n_views, const ddvr_params* p, const float* refs,
                            double count, uint32_t target_mask, float* image_out,
                            float* depth_out, double* loss_out, float* d_volume, double* d_tf,
                            double* d_camera, double* d_dt, void* workspace,
                            int64_t workspace_bytes, void* stream);

/* Forward-mode Jacobian of the image (render_forward_grad, renderer.py:410-464):
 * wrt = DDVR_TARGET_CAMERA (p = 2: d/dlon, d/dlat, per degree) or
 * DDVR_TARGET_STEPSIZE (p = 1); anything else is UNSUPPORTED.  image_out
 * (device) (V, rows, W, 4); jac_out (device) (V, rows, W, 4, p). */
int ddvr_forward_grad(const ddvr_volume* vol, const ddvr_tf* tf, const ddvr_camera* cams,
                      int32_t n_views, const ddvr_params* p, uint32_t wrt, float* image_out,
                      float* jac_out, void* stream);

/* Pre-shaded colour volumes (render_colorvol / render_colorvol_adjoint,
 * renderer.py:404-407, 703-709): cv->data is (X,Y,Z,4) float (r, g, b
 * emission, tau per voxel, 16-byte aligned), trilinear per channel without
 * the [0,1] clamp; cv->cells must be NULL.  Outputs as ddvr_forward /
 * ddvr_adjoint; d_color (device) (X,Y,Z,4) float accumulates (+=). */
int ddvr_forward_color(const ddvr_volume* cv, const ddvr_camera* cams, int32_t n_views,
                       const ddvr_params* p, float* image_out, float* depth_out, void* stream);
int ddvr_adjoint_color(const ddvr_volume* cv, const ddvr_camera* cams, int32_t n_views,
                       const ddvr_params* p, const float* image, const float* depth,
                       const float* seed, float* d_color, void* stream);

/* Workspace ddvr_adjoint needs for this volume, TF and target mask (0 if
 * none): the cell-gradient records (volume target with vol->cells) and the
 * per-CTA TF-gradient slots (tf target). */
int64_t ddvr_adjoint_workspace_bytes(const ddvr_volume* vol, const ddvr_tf* tf,
                                     uint32_t target_mask);

/* Extra workspace of a DDVR_FLAG_DETERMINISTIC ddvr_adjoint /
 * ddvr_forward_adjoint_l1 call over n_views views with params p: the caller
 * passes ddvr_adjoint_workspace_bytes rounded up to 256, plus this.  It holds
 *   - with the camera or stepsize target: per-CTA partials, reduced in a fixed order
 *     (d_camera and d_dt bitwise reproducible);
 *   - with the volume target and cell records: the cell-gradient moments as int64
 *     fixed point (round(fp32 moment * scale), scale = 2^50 / a bound of any one flush
 *     derived from the TF table and max|seed|): integer adds commute, so d_volume is
 *     bitwise reproducible for any order of the atomics.  Texel TFs and the volume
 *     target alone (mask DDVR_TARGET_VOLUME; other masks are UNSUPPORTED); for
 *     ddvr_adjoint one call per step (no WS_CONTINUE / WS_DEFER: the scale comes
 *     from that call's seed); the fused step's seed is +-1/count in every call.
 * (The in-CTA TF sums stay fp32 atomics: d_tf is reproducible to rounding.) */
int64_t ddvr_deterministic_bytes(const ddvr_volume* vol, int32_t n_views, const ddvr_params* p,
                                 uint32_t mask);

/* Extra workspace of a DDVR_FLAG_BAND_TAPE ddvr_forward_adjoint_l1 call: one
 * bit per sample for every ray, 32-bit words per ray bounded by the box
 * diagonal / dt.  Placed after the workspace (and the deterministic partials),
 * each part rounded up to 256 bytes: the tape, then the brick occupancy maps (2
 * bytes per brick of 8^3 cell records, rebuilt from vol->cells by every call; a
 * workspace that ends before the map runs without the empty-space skip), then a
 * float per ray (DDVR_FLAG_SPLIT_WALK: the march hands each ray's walk weight to a
 * separate walk kernel; a workspace that ends before it runs them fused).  Used
 * by the affine absorption walk (emission-free TF with a non-negative affine tau
 * column, volume target); other steps ignore it. */
int64_t ddvr_band_tape_bytes(const ddvr_volume* vol, int32_t n_views, const ddvr_params* p);

/* Threads per ray ddvr_forward_adjoint_l1 uses for this target mask, ray count
 * (views x band rows x width) and params.flags (DDVR_FLAG_RAY_SPLIT_*): for TF or
 * TF|VOLUME, 1 unless the rays alone would not fill the GPU, then the smallest of 2, 4, 8
 * giving ~113 K threads; for camera and / or stepsize alone, 2 below ~606 K rays (fewer
 * than 4 waves of one thread per ray), else 1, never with DDVR_FLAG_DETERMINISTIC (forced:
 * 2 or 4); other masks 1.  Host-side, no GPU work. */
int32_t ddvr_ray_split(uint32_t mask, int64_t rays, int32_t flags);

/* Size of the cell-record copy of a dims[0] x dims[1] x dims[2] volume:
 * (X+1) * (Y+1) * (Z+1) records of 8 floats -- cells -1 .. dim-1 on every
 * axis with edge-replicated corners, so clamp-to-edge (field.py:299-307)
 * needs no per-sample clamping. */
int64_t ddvr_cells_bytes(const int32_t dims[3]);

/* Build the cell records of vol->data into cells_out (device, 32-byte aligned,
 * ddvr_cells_bytes bytes).  Call again whenever the density changes. */
int ddvr_pack_cells(const ddvr_volume* vol, float* cells_out, void* stream);

/* Gather-roofline microbenchmark: the march's rays, stepping and
 * 256-bit cell-record gathers (hold != 0: reloaded only on a cell change, as
 * the march does; 0: one per sample) with one FADD per sample instead of the
 * shading.  out (device) (V, rows, W) float per-ray checksums.  Needs
 * vol->cells; vol->data may be NULL. */
int ddvr_gather_probe(const ddvr_volume* vol, const ddvr_camera* cams, int32_t n_views,
                      const ddvr_params* p, int32_t hold, float* out, void* stream);

/* opacity_entropy (objectives.py:95-126) of n_images (device) (n_pixels, 4)
 * float images: out (device, double, n_images x 4) receives [H, S, S+, T] per
 * image (normalised Shannon entropy of the alpha channel, alpha sum, positive
 * alpha sum, sum a log2 a); seed_out (device, nullable, same shape as the
 * images) the seed dH/dalpha in the alpha channel (rgb 0), non-finite values
 * mapped to +-1e6 and clipped like the reference.  Degenerate (S <= 0 or
 * n_pixels < 2): H = 0, zero seed. */
int ddvr_opacity_entropy(const float* images, int64_t n_pixels, int32_t n_images, double* out,
                         float* seed_out, void* stream);

/* Fused L1 loss + seed (objectives.py:38-54) over n floats: seed_out[i] =
 * sign(x-y)/count (sign(0)=0) and loss_out[0] += sum|x-y|/count (double).
 * count is the normaliser (total element count over all views/ranks). */
int ddvr_l1_loss(const float* x, const float* y, int64_t n, double count, float* seed_out,
                 double* loss_out, void* stream);

/* Ray setup only (parity tests): tn_tf (device, nullable) (V, rows, W, 2)
 * double; n_steps (device) (V, rows, W) int32; flags (device, nullable)
 * (V, rows, W) int32 = entry_axis | clamped << 2 | miss << 3. */
int ddvr_ray_setup(const ddvr_volume* vol, const ddvr_camera* cams, int32_t n_views,
                   const ddvr_params* p, double* tn_tf, int32_t* n_steps, int32_t* flags,
                   void* stream);

/* ---- the steps either side of the path ---- */

/* smoothness_prior_volume (objectives.py:72-92) times weight:
 * value_out[0] += weight * mean squared forward difference; grad_out +=
 * weight * gradient (float (X,Y,Z)).  Either output may be NULL. */
int ddvr_prior_volume(const float* values, const int32_t dims[3], double weight, float* grad_out,
                      double* value_out, void* stream);

/* smoothness_prior_tf (objectives.py:57-69) times weight, texels (R,4) float,
 * grad_out (R,4) double (+=), value_out double (+=). */
int ddvr_prior_tf(const float* texels, int32_t resolution, double weight, double* grad_out,
                  double* value_out, void* stream);

/* Adam with bias correction (optim.py:45-67) fused with the projection of
 * optim.py:70-89: after the update, element i is clamped to [lo, hi] when
 * stride <= 1 or i % stride == stride-1, else to [lo_other, hi_other]
 * (volume: stride 1, [0,1]; TF: stride 4, rgb [0, inf), tau [0, tau_max]). */
typedef struct {
  double lr, beta1, beta2, eps;
  int32_t step;          /* 1-based update count t */
  int32_t stride;
  float lo, hi, lo_other, hi_other;
} ddvr_adam;

/* params, m, v updated in place from grads (all float, n elements).  If
 * nonfinite (device int, caller-zeroed) is given, a non-finite gradient sets
 * it and the whole update is skipped (NumericalAbortError, optim.py:28-30). */
int ddvr_adam_step(float* params, const float* grads, float* m, float* v, int64_t n,
                   const ddvr_adam* cfg, int32_t* nonfinite, void* stream);

/* The same update with the step counter on the device, for CUDA-graph replay:
 * state (device, 4 int32, zeroed before the first step) holds t; each call
 * advances it (unless the update is skipped for a non-finite gradient) and
 * derives the bias corrections on the device.  cfg->step is ignored. */
int ddvr_adam_step_device(float* params, const float* grads, float* m, float* v, int64_t n,
                          const ddvr_adam* cfg, int32_t* state, int32_t* nonfinite,
                          void* stream);

/* upsample_volume (optim.py:92-129): dst (2X,2Y,2Z) from src (X,Y,Z). */
int ddvr_upsample_volume(const float* src, const int32_t dims[3], float* dst, void* stream);

/* project_params (optim.py:70-89) alone: element i clamped to [lo, hi] when
 * stride <= 1 or i % stride == stride-1, else to [lo_other, hi_other]; only
 * cfg->stride / lo / hi / lo_other / hi_other are read. */
int ddvr_project(float* params, int64_t n, const ddvr_adam* cfg, void* stream);

/* gd_step (optim.py:33-42): params -= lr * grads; a non-finite gradient sets
 * *nonfinite (device, caller-zeroed, nullable) and skips the update. */
int ddvr_gd_step(float* params, const float* grads, int64_t n, double lr, int32_t* nonfinite,
                 void* stream);

/* ---- point-wise field functions, fp64 ---
 * The march evaluates these inline; these entry points expose them over
 * caller-given points with the reference's operation order and separately
 * rounded arithmetic: trilinear_* and tf_* agree with the reference bit for
 * bit, the transcendental ones (camera, opacity) to libm's last ulp.  All
 * arrays are (device) doubles; every output is nullable. */

/* trilinear_sample / trilinear_gradients (field.py:279-349, 379-517) of the
 * (X,Y,Z) z-fastest double grid `values` on [box_min, box_max] at n points
 * (n, 3): value_out (n) = density clamped to [0, 1], 0 outside the box;
 * spatial_out (n, 3) world-space gradient, weights_out (n, 8) corner
 * sensitivities (both zeroed outside the box and where the clamp is active),
 * corners_out (n, 8) int64 flat corner indices (C order, field.py:311-324). */
int ddvr_field_sample(const double* values, const int32_t dims[3], const double box_min[3],
                      const double box_max[3], const double* points, int64_t n,
                      double* value_out, double* spatial_out, double* weights_out,
                      int64_t* corners_out, void* stream);

/* tf_sample / tf_gradients (field.py:525-579) of the texel TF (R, 4) at n
 * densities: out4 (n, 4) (rgb, tau); slope4 (n, 4) zero in the clamp-to-edge
 * regions; weights2 (n, 2) texel weights; idx2 (n, 2) int64 texel indices. */
int ddvr_tf_lookup(const double* texels, int32_t resolution, const double* density, int64_t n,
                   double* out4, double* slope4, double* weights2, int64_t* idx2, void* stream);

/* opacity_from_density (field.py:587-600): alpha = 1 - exp(-dt tau) clamped to
 * 1 - 1e-6, dalpha = dt exp(-dt tau) (0 where clamped), n segments. */
int ddvr_opacity(const double* tau, int64_t n, double dt, double* alpha, double* dalpha,
                 void* stream);

/* camera_from_sphere / camera_gradients (field.py:186-271) of one camera (host
 * struct) for an image width x height at n pixel coordinates u (column), v
 * (row), in [0, width) x [0, height): origin (n, 3), dir (n, 3) unit;
 * j_origin, j_dir (n, 3, 2) Jacobians w.r.t. (lon, lat) per degree, evaluated
 * with the reference's dual-number formulas (autodiff.py:39-141). */
int ddvr_camera_rays(const ddvr_camera* cam, int32_t width, int32_t height, const double* u,
                     const double* v, int64_t n, double* origin, double* dir, double* j_origin,
                     double* j_dir, void* stream);

/* ---- wire / disk formats (fileio.py:27-127) ------------------------------ */

/* Raw volume file -> device volume.  `raw` holds the file's little-endian f32
 * values in x-fastest order (fileio.py:32, 65: order="F"), already copied to
 * the device; `dst` receives the (X,Y,Z) z-fastest layout every other entry
 * point takes.  value_range = NULL or {lo, hi}: fused (v - lo) / (hi - lo)
 * normalisation (fileio.py:66-70), hi > lo.  Replaces the numpy reshape in
 * voldiff.fileio.load_volume (fileio.py:45-71). */
int ddvr_volume_from_raw(const float* raw, const int32_t dims[3], const double* value_range,
                         float* dst, void* stream);

/* Device (X,Y,Z) volume -> x-fastest raw file body (save_volume, fileio.py:27-40). */
int ddvr_volume_to_raw(const float* src, const int32_t dims[3], float* raw, void* stream);

/* n_pixels premultiplied rgba float4 -> 3*n_pixels bytes of binary-PPM body
 * composited over white (save_image, fileio.py:104-110). */
int ddvr_image_to_ppm(const float* images, int64_t n_pixels, uint8_t* out, void* stream);

/* Thread-local message of the last failing call ("" if none). */
const char* ddvr_last_error(void);

/* DDVR_ABI_VERSION of the loaded library. */
int32_t ddvr_abi_version(void);

/* Number of kernel launches this library issued since load (process-wide). */
int64_t ddvr_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* DDVR_H */
