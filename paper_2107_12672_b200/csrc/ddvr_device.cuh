#pragma once
// ddvr_device.cuh -- device code shared by the libddvr translation units.
//
// (ddvr_abi.cu: C ABI + small kernels; ddvr_fwd.cu: forward instantiations;
//  ddvr_adj_*.cu: adjoint instantiations.  Split only to compile in parallel.)
//
//
// Differentiable emission-absorption raymarcher (DiffDVR, arXiv 2107.12672),
// written for Blackwell from scratch.  The reference (voldiff, pure NumPy) is
// cited by file:line for each piece of semantics reproduced here.
//
// Kernels
//   dvr_forward_kernel  one thread per ray, 16x16-pixel CTAs (8x4-pixel warps),
//                       fp64 ray setup, exact fixed-point sample positions,
//                       one 256-bit gather per sample from the cell-record
//                       volume (8 corners per cell, 32 B), TF in shared
//                       memory, float4 image stores.
//   dvr_adjoint_kernel  same mapping; walks each ray back to front and recovers
//                       the transmittance before every sample by inverting the
//                       compositing step (T_prev = T / (1 - a)): O(1) state per
//                       ray, no tape.  Gradient scatter:
//                         volume  : per-ray cell-run accumulation of the 8
//                                   corner weights, flushed as two 128-bit
//                                   vector reds into a cell-gradient
//                                   workspace when the ray leaves a cell;
//                                   fold_cells_kernel sums them into voxels;
//                         tf      : per-ray texel-run accumulation, flushed to
//                                   per-CTA shared memory, then fp64 atomics;
//                         camera/stepsize: per-ray sums in registers, fp64
//                                   Jacobian chain per ray, warp-shuffle + CTA
//                                   reduction, one fp64 atomic per CTA.
//   pack_cells_kernel   builds the cell-record copy of a volume.
//   ray_setup_kernel    parity-test helper (tn, tf, n_steps, flags).
//   l1_loss_kernel      fused L1 loss value + seed (objectives.py:38-54).
//
// Tensor cores are deliberately unused: this is a gather-bound ray integral.

#include <cuda_runtime.h>

#include <atomic>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <type_traits>

#include "ddvr.h"

// Bounds-checked build (-DDDVR_CHECKED, tests/test_gpu_checked.py): every cell-record
// gather and cell-gradient flush, every empty-brick lookup, checks its index against
// the padded record grid and traps with the source line on a violation -- the
// memory-safety evidence of this path (compute-sanitizer is not available on the pool).
#ifdef DDVR_CHECKED
#define DDVR_REQUIRE(cond)                                                                 \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("ddvr check failed: %s (%s:%d) block (%d,%d,%d) thread %d\n", #cond, __FILE__, \
             __LINE__, blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x);                   \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define DDVR_REQUIRE(cond) ((void)0)
#endif


namespace ddvr_impl {


constexpr float kEpsAlpha = 1e-6f;          // field.py:25 (EPS_ALPHA)
constexpr float kAlphaStop = 1.f - 1e-4f;   // ALPHA_STOP (renderer.py:45)
constexpr double kStepEps = 1e-9;           // renderer.py:212
constexpr double kDeg = 3.14159265358979323846 / 180.0;   // field.py:27
constexpr int kTile = 16;                   // CTA = 16x16 pixels
constexpr int kThreads = kTile * kTile;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxTfBytes = 200 * 1024;     // TF tables + TF gradient in shared memory (B200: 227 KB/CTA)

// Sample positions are kept in 32.32 fixed-point GRID coordinates
// (g = (x - bmin)*scale - 0.5): g_i = g_0 + i*step with integer adds.  The
// only error is the 2^-33 rounding of g_0 and step: < 5e-7 voxel after 4k
// steps, a relative stepsize error of ~1e-9 (fp32 grid coordinates would
// quantise positions to ~1.5e-5 voxel at 256^3, which alone moves the
// cancellation-heavy camera gradient by ~3e-4), and it makes the adjoint's
// backward positions bitwise identical to the forward's (g -= step).
constexpr double kFix = 4294967296.0;                  // 2^32
constexpr float kInvFix = 2.3283064365386963e-10f;     // 2^-32

// ---------------------------------------------------------------------------
// kernel-side argument blocks (passed by value)
// ---------------------------------------------------------------------------

struct VolArgs {
  const float* __restrict__ data;    // (X,Y,Z) z fastest
  const float* __restrict__ cells;   // padded cell records (nullable): 8 corner values per cell
  const float* __restrict__ cell0;   // address of the record of cell (0,0,0) inside cells
  int X, Y, Z, YZ;
  int CY, CZ;              // padded cells along y and z: dim + 1 (cells -1 .. dim-1)
  int Xm2, Ym2, Zm2;       // max(dim-2, 0): highest cell index (field.py:302-304)
  int X1, Y1, Z1;          // dim-1: clamp bound (field.py:299-301)
  float tX, tY, tZ;        // cell fraction at the top clamp: 1 if dim > 1 else 0
  long long lo[3], hi[3];  // inside test, fixed-point grid units: [-0.5 - tol, dim - 0.5 + tol]
  long long top[3];        // (dim-1) in fixed point: spatial-gradient liveness (field.py:461-463)
  double bmin[3], bmax[3], scale[3];   // scale = dim / extent
  // fused band-tape march (DDVR_FLAG_BAND_TAPE, nullable): byte per brick of 8^3 padded
  // cell records (storage index >> 3 per axis), 1 = some record of the 2x2x2 bricks
  // b .. b+1 (those that exist) is nonzero
  const unsigned char* __restrict__ occ;
  int NBy, NBz;            // bricks along y and z: ceil((dim + 1) / 8)
  // DDVR_FLAG_DETERMINISTIC with the volume target (nullable): the cell-gradient
  // moments accumulate as int64 fixed point (round(moment * *det_scale)) at this
  // address (relative to cell (0,0,0), like cell0) -- integer adds commute, so the
  // sums and d_volume are the same bits for any order of the atomics
  unsigned long long* cells64;
  const double* det_scale;
};

// brick coordinate of the padded cell record at a fixed-point grid coordinate
__device__ __forceinline__ int brick_of(long long g, int top) {
  return (min(max((int)(g >> 32), -1), top) + 1) >> 3;
}

// The 32-sample block from grid position g reads only all-zero records: with fewer
// than 8 cells per axis between its first and last sample, its cells lie in the start
// brick and the next one in the direction of travel (back: bit k set = axis k goes
// down; clamping is monotone), which is the 2x2x2 window at this low corner.
__device__ __forceinline__ bool block_empty(const VolArgs& V, long long gx, long long gy,
                                            long long gz, int back) {
  const int x = max(brick_of(gx, V.X1) - (back & 1), 0);
  const int y = max(brick_of(gy, V.Y1) - ((back >> 1) & 1), 0);
  const int z = max(brick_of(gz, V.Z1) - (back >> 2), 0);
  DDVR_REQUIRE(x >= 0 && y >= 0 && z >= 0 && x <= (V.X1 + 1) >> 3 && y < V.NBy && z < V.NBz);
  return __ldg(V.occ + (x * V.NBy + y) * V.NBz + z) == 0;
}

struct TfArgs {
  const float* __restrict__ params;
  int kind, count;
  float fR, fR1;     // R, R-1
  int Rm2;           // max(R-2, 0)
  int stride;        // floats per parameter row: 4 texture, 5 piecewise, 6 gaussian
  // adjoint TF-gradient slots in the workspace (tf target): CTA b accumulates
  // into slot b % nslot, slot_floats floats each: an rgba block (count x 4,
  // 16-byte rows for vector reds), then count knot positions (piecewise) or
  // count (mu, sigma) pairs (gaussian)
  float* __restrict__ slots;
  int nslot, slot_floats;
};

// slot size in floats (a multiple of 8: 32-byte aligned slots)
inline int tf_slot_floats(int kind, int count) {
  const int extra = kind == DDVR_TF_PIECEWISE ? count : kind == DDVR_TF_GAUSSIAN ? 2 * count : 0;
  return (4 * count + extra + 7) & ~7;
}

struct Geometry {
  const ddvr_camera* __restrict__ cams;
  int W, H, row0, row1;
  double dt;
  float dt32;             // (float)dt: the stepsize of the fp32 march
  float* tape;            // stored memory mode (nullable)
  long long tape_stride;
  double* partials;       // DDVR_FLAG_DETERMINISTIC: per-CTA camera / stepsize sums
                          // (3 doubles per CTA) instead of fp64 atomics (nullable)
  unsigned* bits;         // DDVR_FLAG_BAND_TAPE: the fused absorption step's band bits,
                          // bits_words 32-bit words per ray, warp-interleaved (nullable)
  int bits_words;
  unsigned long long* stats;   // ddvr_params.stats (nullable): [samples, march skipped,
                               // walk skipped, rays], one atomic per warp
  float* ray_k;           // band-tape step split into march + walk kernels (nullable): the
                          // march's per-ray walk weight abs_k, (V, rows, W)
  int vgroup;             // CTAs cycle over groups of this many views per tile (1: view-major)
};

// Launchers with external linkage: each is defined (with its kernel
// instantiations) in one translation unit.
void launch_forward(bool early, bool cells, bool tape, dim3 grid, size_t smem, cudaStream_t st,
                    const VolArgs& V, const TfArgs& T, const Geometry& G, float* image,
                    float* depth);
void launch_gather_probe(bool hold, dim3 grid, cudaStream_t st, const VolArgs& V,
                         const Geometry& G, float* out);
void launch_forward_grad(int n_params, bool cells, dim3 grid, size_t smem, cudaStream_t st,
                         const VolArgs& V, const TfArgs& T, const Geometry& G, float* image,
                         float* jac);
void launch_forward_color(bool early, bool tape, dim3 grid, cudaStream_t st, const VolArgs& V,
                          const Geometry& G, float* image, float* depth);
void launch_adjoint_color(dim3 grid, cudaStream_t st, const VolArgs& V, const Geometry& G,
                          const float* image, const float* depth, const float* seed,
                          float* d_color);
// point-wise field functions in fp64 (ddvr_fields.cu)
void launch_field_sample(const double* values, const int dims[3], const double bmin[3],
                         const double bmax[3], const double* pts, long long n, double* value,
                         double* spatial, double* weights, long long* corners, cudaStream_t st);
void launch_tf_lookup(const double* texels, int R, const double* d, long long n, double* out4,
                      double* slope4, double* weights2, long long* idx2, cudaStream_t st);
void launch_opacity(const double* tau, long long n, double dt, double* alpha, double* dalpha,
                    cudaStream_t st);
void launch_camera_rays(const ddvr_camera& cam, int W, int H, const double* u, const double* v,
                        long long n, double* origin, double* dir, double* j_origin,
                        double* j_dir, cudaStream_t st);
// Fused step (ddvr_forward_adjoint_l1): each thread marches its ray forward,
// forms the L1 seed sign(image - ref) / count (objectives.py:38-54) and its
// loss term in registers, then walks back with the exact fp64 optical depth.
struct FusedArgs {
  const float* __restrict__ refs;   // (V, rows, W, 4) reference images
  float inv_count;                  // 1 / global element count (fp32 seed)
  double inv_count_d;
  double* loss;                     // += sum |image - ref| / count
  float* image_out;                 // optional (V, rows, W, 4)
  float* depth_out;                 // optional (V, rows, W)
};

#define DDVR_ADJ_LAUNCHER(NAME)                                                              \
  int NAME(unsigned mask, bool cells, dim3 grid, size_t smem, cudaStream_t st,             \
            const VolArgs& V, const TfArgs& T, const Geometry& G, const float* image,       \
            const float* depth, const float* seed, float* dv, float* dcells, double* dcam,  \
            double* ddt, const FusedArgs* fu)
DDVR_ADJ_LAUNCHER(launch_adjoint_g0);   // masks 1-3   (camera / stepsize)
DDVR_ADJ_LAUNCHER(launch_adjoint_g1);   // masks 4-7   (tf [+ camera / stepsize])
DDVR_ADJ_LAUNCHER(launch_adjoint_g2);   // masks 8-11  (volume [+ camera / stepsize])
DDVR_ADJ_LAUNCHER(launch_adjoint_g3);   // masks 12-15 (volume + tf [+ ...])
// fused TF-target steps (masks 4, 12) with segment-split rays (SPLIT = 2, 4, 8); returns
// the kernels launched (0: not instantiated)
int launch_adjoint_split(unsigned mask, int split, int n_views, size_t smem, cudaStream_t st,
                         const VolArgs& V, const TfArgs& T, const Geometry& G, float* dv,
                         float* dcells, double* dcam, double* ddt, const FusedArgs& fu);

#ifndef DDVR_CARVEOUT
#define DDVR_CARVEOUT -1
#endif
template <typename K>
inline void set_smem(K kernel, size_t smem) {
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (DDVR_CARVEOUT >= 0)
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, DDVR_CARVEOUT);
}

}  // namespace ddvr_impl

namespace {
using namespace ddvr_impl;

// per-view camera frame, computed once per CTA in fp64 (field.py:194-222)
struct Frame {
  double eye[3], f[3], r[3], up[3];
  double th, aspect;
  double jo[3][2];          // d eye / d(lon, lat), per degree
  double df[3][2], dr[3][2], du[3][2];
};

// fp64 helpers with pinned rounding (never contracted into FMA), so the ray
// setup reproduces NumPy's separately-rounded operations.
__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dd(double a, double b) { return __ddiv_rn(a, b); }

__device__ void make_frame(const ddvr_camera& c, int W, int H, Frame& F) {
  double lon_deg = fmod(c.lon_deg, 360.0);          // field.py:143 (lon % 360)
  if (lon_deg < 0.0) lon_deg = da(lon_deg, 360.0);
  const double lon = dm(lon_deg, kDeg);
  const double lat = dm(c.lat_deg, kDeg);
  double sl, cl, sp, cp;
  sincos(lat, &sl, &cl);
  sincos(lon, &sp, &cp);
  const double rho = c.radius;
  F.eye[0] = da(c.center[0], dm(rho, dm(cl, cp)));
  F.eye[1] = da(c.center[1], dm(rho, sl));
  F.eye[2] = da(c.center[2], dm(rho, dm(cl, sp)));
  double fx = -dm(cl, cp), fy = -sl, fz = -dm(cl, sp);
  const double fn = __dsqrt_rn(da(da(dm(fx, fx), dm(fy, fy)), dm(fz, fz)));
  fx = dd(fx, fn); fy = dd(fy, fn); fz = dd(fz, fn);
  double rx = -fz, rz = fx;
  const double rn = __dsqrt_rn(da(dm(rx, rx), dm(rz, rz)));
  rx = dd(rx, rn); rz = dd(rz, rn);
  F.f[0] = fx; F.f[1] = fy; F.f[2] = fz;
  F.r[0] = rx; F.r[1] = 0.0; F.r[2] = rz;
  F.up[0] = -dm(rz, fy);
  F.up[1] = ds(dm(rz, fx), dm(rx, fz));
  F.up[2] = dm(rx, fy);
  F.th = tan(dm(dm(0.5, c.fov_y_deg), kDeg));
  F.aspect = dd((double)W, (double)H);
  // analytic Jacobians (the reference evaluates them over duals, field.py:253-271)
  const double k = kDeg;
  F.jo[0][0] = -rho * cl * sp * k;  F.jo[0][1] = -rho * sl * cp * k;
  F.jo[1][0] = 0.0;                 F.jo[1][1] = rho * cl * k;
  F.jo[2][0] = rho * cl * cp * k;   F.jo[2][1] = -rho * sl * sp * k;
  F.df[0][0] = cl * sp * k;  F.df[0][1] = sl * cp * k;
  F.df[1][0] = 0.0;          F.df[1][1] = -cl * k;
  F.df[2][0] = -cl * cp * k; F.df[2][1] = sl * sp * k;
  F.dr[0][0] = cp * k;  F.dr[0][1] = 0.0;
  F.dr[1][0] = 0.0;     F.dr[1][1] = 0.0;
  F.dr[2][0] = sp * k;  F.dr[2][1] = 0.0;
  F.du[0][0] = sp * sl * k;  F.du[0][1] = -cp * cl * k;
  F.du[1][0] = 0.0;          F.du[1][1] = -sl * k;
  F.du[2][0] = -cp * sl * k; F.du[2][1] = -sp * cl * k;
}

// one ray: fp64 geometry and the fixed-point march parameters
struct Ray {
  long long g0[3]; // fixed-point grid coordinate of the entry point
  long long gs[3]; // fixed-point grid step per sample (dt * w * scale)
  float gw[3];     // grid-space direction per unit t (fp32, for dt gradients)
  int n;           // step count (renderer.py:209-214)
  int axis;        // face axis that decided the entry (renderer.py:198)
  bool clamped, miss;
  bool all_inside; // first and last samples inside => every sample inside (convex box)
  double o[3], w[3], tn, tf, su, sv, dn;
};

__device__ __forceinline__ bool inside_fx(const VolArgs& V, long long x, long long y, long long z) {
  return x >= V.lo[0] && x <= V.hi[0] && y >= V.lo[1] && y <= V.hi[1] && z >= V.lo[2] &&
         z <= V.hi[2];
}

// camera ray through pixel (u, v) + slab clipping + step count, fp64
// (field.py:218-228, renderer.py:182-214, 315)
__device__ void setup_ray(const Frame& F, const VolArgs& V, double dt, int W, int H, int u,
                          int v, Ray& r) {
  const double su = dm(dm(ds(dm(da((double)u, 0.5), dd(2.0, (double)W)), 1.0), F.th),
                       F.aspect);
  const double sv = dm(ds(1.0, dm(da((double)v, 0.5), dd(2.0, (double)H))), F.th);
  const double dx = da(da(F.f[0], dm(F.r[0], su)), dm(F.up[0], sv));
  const double dy = da(F.f[1], dm(F.up[1], sv));
  const double dz = da(da(F.f[2], dm(F.r[2], su)), dm(F.up[2], sv));
  const double dn = __dsqrt_rn(da(da(dm(dx, dx), dm(dy, dy)), dm(dz, dz)));
  r.su = su; r.sv = sv; r.dn = dn;
  r.w[0] = dd(dx, dn); r.w[1] = dd(dy, dn); r.w[2] = dd(dz, dn);
  r.o[0] = F.eye[0]; r.o[1] = F.eye[1]; r.o[2] = F.eye[2];
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    if (r.w[k] == 0.0) {   // parallel to the slab (renderer.py:194-197)
      const bool in_slab = r.o[k] >= V.bmin[k] && r.o[k] <= V.bmax[k];
      lo[k] = in_slab ? -INFINITY : INFINITY;
      hi[k] = in_slab ? INFINITY : -INFINITY;
    } else {
      const double t1 = dd(ds(V.bmin[k], r.o[k]), r.w[k]);
      const double t2 = dd(ds(V.bmax[k], r.o[k]), r.w[k]);
      lo[k] = fmin(t1, t2);
      hi[k] = fmax(t1, t2);
    }
  }
  // entry axis = first argmax of the near distances (renderer.py:198-200)
  int axis = 0;
  double tn = lo[0];
  if (lo[1] > tn) { tn = lo[1]; axis = 1; }
  if (lo[2] > tn) { tn = lo[2]; axis = 2; }
  double tf = fmin(fmin(hi[0], hi[1]), hi[2]);
  r.clamped = tn <= 0.0;
  tn = fmax(tn, 0.0);
  r.miss = !(tf > tn) || !isfinite(tn) || !isfinite(tf);
  if (r.miss) { tn = 0.0; tf = 0.0; }
  r.tn = tn; r.tf = tf; r.axis = axis;
  long long n = 0;
  if (!r.miss) {
    const double q = ceil(ds(dd(ds(tf, tn), dt), kStepEps));
    n = q > 0.0 ? (long long)q : 0;
    if (n > 0x7fffffff) n = 0x7fffffff;
  }
  r.n = (int)n;
  // entry point and grid-space march parameters (renderer.py:315 xo = o + tn*w)
  for (int k = 0; k < 3; ++k) {
    const double xo = da(r.o[k], dm(tn, r.w[k]));
    const double gw = dm(r.w[k], V.scale[k]);
    r.g0[k] = __double2ll_rn((dm(ds(xo, V.bmin[k]), V.scale[k]) - 0.5) * kFix);
    r.gs[k] = __double2ll_rn(dm(dt, gw) * kFix);
    r.gw[k] = (float)gw;
  }
  // Every sample lies on the segment [first, last]; the box is convex, so the
  // per-sample inside test of field.py:293-298 reduces to the two endpoints.
  const long long m = r.n > 0 ? (long long)(r.n - 1) : 0;
  r.all_inside = inside_fx(V, r.g0[0], r.g0[1], r.g0[2]) &&
                 inside_fx(V, r.g0[0] + m * r.gs[0], r.g0[1] + m * r.gs[1],
                           r.g0[2] + m * r.gs[2]);
}

// ---------------------------------------------------------------------------
// trilinear density (field.py:279-349, 379-500) in grid coordinates, fp32
// ---------------------------------------------------------------------------

// packed fp32 pair arithmetic (FFMA2 / FMUL2 on sm_100a; DDVR_F32X2=0 gives the
// same per-lane IEEE operations as scalar instructions, for A/B measurements)
#ifndef DDVR_F32X2
#define DDVR_F32X2 1
#endif
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
#if DDVR_F32X2
  return __ffma2_rn(a, b, c);
#else
  return make_float2(__fmaf_rn(a.x, b.x, c.x), __fmaf_rn(a.y, b.y, c.y));
#endif
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
#if DDVR_F32X2
  return __fmul2_rn(a, b);
#else
  return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
#endif
}
__device__ __forceinline__ float2 bcast(float a) { return make_float2(a, a); }

struct Cell {
  int cell;            // padded cell-record index relative to cell0 (may be negative)
  int base;            // flat voxel index of corner (ix, iy, iz)
  int ox, oy, oz;      // flat voxel offsets to the +x/+y/+z corners (0 on a clamped axis)
  float fx, fy, fz;    // cell fractions in [0, 1] (colour volumes)
  float ux, uy, uz;    // centred fractions f - 1/2 (the polynomial records)
  bool inside;
};

// one axis of _grid_setup (field.py:290-307) on a fixed-point coordinate,
// branch-free: gc = clip(g, 0, dim-1); i = clip(floor(gc), 0, dim-2); f = gc - i
__device__ __forceinline__ void axis_cell(long long g, int d1, int dm2, float ftop, int& i,
                                          float& f) {
  const int hi = (int)(g >> 32);
  const float fr = __fmul_rn(__uint2float_rn((unsigned)g), kInvFix);
  i = min(max(hi, 0), dm2);
  f = hi < 0 ? 0.f : (hi >= d1 ? ftop : fr);
}

// Voxel layout: the clamps of field.py:299-307 per sample.
__device__ __forceinline__ void locate_voxels(const VolArgs& V, long long gx, long long gy,
                                              long long gz, bool all_inside, Cell& c) {
  c.inside = all_inside || inside_fx(V, gx, gy, gz);
  int ix, iy, iz;
  axis_cell(gx, V.X1, V.Xm2, V.tX, ix, c.fx);
  axis_cell(gy, V.Y1, V.Ym2, V.tY, iy, c.fy);
  axis_cell(gz, V.Z1, V.Zm2, V.tZ, iz, c.fz);
  c.ux = __fsub_rn(c.fx, 0.5f);
  c.uy = __fsub_rn(c.fy, 0.5f);
  c.uz = __fsub_rn(c.fz, 0.5f);
  c.base = (ix * V.Y + iy) * V.Z + iz;
  c.cell = c.base;   // identifies the cell (its 8 corners) for the cell-run logic
  c.ox = ix + 1 < V.X ? V.YZ : 0;
  c.oy = iy + 1 < V.Y ? V.Z : 0;
  c.oz = iz + 1 < V.Z ? 1 : 0;
}

// Padded cell layout: records exist for cells -1 .. dim-1 on every axis with
// edge-replicated corners, so clamp-to-edge (field.py:299-307) is baked into
// the data: a sample in [-0.5, 0) reads cell -1 whose corners are both v[0],
// one in [dim-1, dim-0.5] reads cell dim-1 whose corners are both v[dim-1].
// Values, spatial derivatives (0 in the pad, field.py:459-484) and scatter
// weights (folded back onto the clamped voxel) equal the clamped ones; the
// only difference is the measure-zero point g == dim-1 exactly.  Cell
// location is then just the high word and the fraction of each coordinate.
__device__ __forceinline__ void locate_cells(const VolArgs& V, long long gx, long long gy,
                                             long long gz, bool all_inside, Cell& c) {
  int hx = (int)(gx >> 32), hy = (int)(gy >> 32), hz = (int)(gz >> 32);
  c.inside = true;
  if (!all_inside) {   // never taken for march samples (see Ray::all_inside); kept safe
    c.inside = inside_fx(V, gx, gy, gz);
    hx = min(max(hx, -1), V.X1);
    hy = min(max(hy, -1), V.Y1);
    hz = min(max(hz, -1), V.Z1);
  }
  // u = lo * 2^-32 - 1/2 in one FFMA (the fraction itself is not needed)
  const float2 uxy = fma2(make_float2(__uint2float_rn((unsigned)gx), __uint2float_rn((unsigned)gy)),
                          bcast(kInvFix), bcast(-0.5f));
  c.ux = uxy.x;
  c.uy = uxy.y;
  c.uz = __fmaf_rn(__uint2float_rn((unsigned)gz), kInvFix, -0.5f);
  c.fx = c.ux + 0.5f; c.fy = c.uy + 0.5f; c.fz = c.uz + 0.5f;   // unused on this path
  c.cell = (hx * V.CY + hy) * V.CZ + hz;
}

template <bool CELLS>
__device__ __forceinline__ void locate(const VolArgs& V, long long gx, long long gy, long long gz,
                                       bool all_inside, Cell& c) {
  if (CELLS) locate_cells(V, gx, gy, gz, all_inside, c);
  else locate_voxels(V, gx, gy, gz, all_inside, c);
}

__device__ __forceinline__ void ld256(const float* p, float v[8]) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                 "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}

// Predicated 256-bit gather: lanes with pred == false issue nothing and keep
// the registers they hold.  A ray stays in one cell for ~3 samples at
// dt = 0.2 voxel, so reloading only on a cell change cuts the L1 data-pipe
// wavefronts of the gather (the binding unit) without a divergent branch.
#ifndef DDVR_L2PF
#define DDVR_L2PF ".L2::256B"   // measured +1.4% fwd, +0.8% adj at C4 (tools/locality_probe.py)
#endif
__device__ __forceinline__ void ld256_if(bool pred, const float* p, float v[8]) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %8, 0;\n\t"
      "@q ld.global.nc" DDVR_L2PF ".v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%9];\n\t}"
      : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]),
        "+f"(v[7])
      : "r"((int)pred), "l"(p));
}

#ifndef DDVR_HOLD_CELL
#define DDVR_HOLD_CELL 1
#endif

#ifndef DDVR_EARLY_WALK
#define DDVR_EARLY_WALK 1
#endif
#ifndef DDVR_AFF_WALK
#define DDVR_AFF_WALK 1
#endif
#ifndef DDVR_ABS_MINB
#define DDVR_ABS_MINB 5
#endif
#ifndef DDVR_BITS_MARCH_UNROLL
#define DDVR_BITS_MARCH_UNROLL 4
#endif
#ifndef DDVR_EMIT_MARCH_UNROLL
#define DDVR_EMIT_MARCH_UNROLL 2   // the fused kernels' emitting marches (C5 +1.3%; the
                                   // 48-register forward kernel spills unrolled: C3 -6%)
#endif
#ifndef DDVR_BITS_WALK_UNROLL
#define DDVR_BITS_WALK_UNROLL 4
#endif
#ifndef DDVR_ABS_FUSED_MINB
#define DDVR_ABS_FUSED_MINB 4
#endif
#ifndef DDVR_ABS_WALK
#define DDVR_ABS_WALK 1
#endif

// predicated 128-bit vector red: no branch around it (the cell-run flush of
// the adjoint would otherwise be a divergent branch taken on most iterations)
__device__ __forceinline__ void red128_if(bool pred, float* p, float a, float b, float c,
                                          float d) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t"
      "@q red.global.add.v4.f32 [%1], {%2,%3,%4,%5};\n\t}" ::"r"((int)pred),
      "l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
      : "memory");
}

// both halves of a 32-byte moment record under ONE predicate: ptxas turns a
// predicated red into a branch around it, so one branch instead of two
__device__ __forceinline__ void red256_if(bool pred, float* p, const float a[8]) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t"
      "@q red.global.add.v4.f32 [%1], {%2,%3,%4,%5};\n\t"
      "@q red.global.add.v4.f32 [%1+16], {%6,%7,%8,%9};\n\t}" ::"r"((int)pred),
      "l"(p), "f"(a[0]), "f"(a[1]), "f"(a[2]), "f"(a[3]), "f"(a[4]), "f"(a[5]), "f"(a[6]),
      "f"(a[7])
      : "memory");
}

__device__ __forceinline__ void red64(float* p, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}

__device__ __forceinline__ void red128(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

// a padded cell-record index (relative to cell (0,0,0)) inside the record grid
__device__ __forceinline__ bool cell_ok(const VolArgs& V, long long cell) {
  const long long lo = -((long long)V.CY * V.CZ + V.CZ + 1);
  const long long hi = ((long long)V.X1 * V.CY + V.Y1) * V.CZ + V.Z1;
  return cell >= lo && cell <= hi;
}

// the cell-record gathers of the marches and walks (predicated / unconditional)
__device__ __forceinline__ void gather_if(const VolArgs& V, bool pred, int cell, float v[8]) {
  DDVR_REQUIRE(!pred || cell_ok(V, cell));
  ld256_if(pred, V.cell0 + 8 * (long long)cell, v);
}
__device__ __forceinline__ void gather(const VolArgs& V, int cell, float v[8]) {
  DDVR_REQUIRE(cell_ok(V, cell));
  ld256(V.cell0 + 8 * (long long)cell, v);
}

// One cell run's 8 moments into the cell-gradient workspace: two 128-bit vector reds
// (fp32), or in the deterministic mode eight int64 fixed-point adds.
template <bool DET>
__device__ __forceinline__ void flush_record(const VolArgs& V, float* __restrict__ d_cells,
                                             int cell, const float a[8]) {
  if (DET) {   // (fp32 product: each contribution keeps fp32's relative precision)
    const float sc = (float)__ldg(V.det_scale);
    unsigned long long* q = V.cells64 + 8 * (long long)cell;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      atomicAdd(q + k, (unsigned long long)__float2ll_rn(a[k] * sc));
  } else {
    float* q = d_cells + 8 * (long long)cell;
    red128(q, a[0], a[1], a[2], a[3]);
    red128(q + 4, a[4], a[5], a[6], a[7]);
  }
}

// The trilinear interpolant of a cell (field.py:318-349) as a polynomial in
// the centred fractions u = f - 1/2 in [-1/2, 1/2]:
//   rho(u) = sum_b c_b prod_{axes of b} u,   b = bx | by << 1 | bz << 2
// i.e. c = {c0, cx, cy, cxy, cz, cxz, cyz, cxyz} -- the corner-bit order of
// field.py:318-322 applied to the monomials -- with c = L v for the 8 corner
// values v (s = +1 on the + corner, -1 on the - corner):
//   c0 = sum v / 8, cx = sum s_x v / 4, cxy = sum s_x s_y v / 2, cxyz = sum s_x s_y s_z v.
// In this order the x-free and x-carrying coefficients of each (y, z) monomial
// sit in adjacent registers of the 256-bit gather, so the interpolant is two
// packed FFMA2 (sm_100a: two fp32 FMAs per lane and instruction), an FMUL, two
// FFMA and the FADD of c0 instead of 7 dependent FFMAs, and its partial products give the
// spatial derivative.  Built in fp64 (each coefficient rounded once) from pairwise
// x-sums / x-differences, so a replicated (edge-clamped) axis gives exactly
// zero coefficients: the clamp-to-edge semantics of the corner form are kept
// exactly.
__device__ __forceinline__ void corners_to_poly(const float w[8], float c[8]) {
  double v[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) v[b] = (double)w[b];
  const double d00 = v[1] - v[0], d10 = v[3] - v[2], d01 = v[5] - v[4], d11 = v[7] - v[6];
  const double s00 = v[1] + v[0], s10 = v[3] + v[2], s01 = v[5] + v[4], s11 = v[7] + v[6];
  c[0] = (float)(((s00 + s10) + (s01 + s11)) * 0.125);
  c[1] = (float)(((d00 + d10) + (d01 + d11)) * 0.25);
  c[2] = (float)(((s10 - s00) + (s11 - s01)) * 0.25);
  c[3] = (float)(((d10 - d00) + (d11 - d01)) * 0.5);
  c[4] = (float)(((s01 - s00) + (s11 - s10)) * 0.25);
  c[5] = (float)(((d01 - d00) + (d11 - d10)) * 0.5);
  c[6] = (float)(((s11 - s01) - (s10 - s00)) * 0.5);
  c[7] = (float)((d11 - d01) - (d10 - d00));
}

// The 8 monomials of a sample, phi = {1, ux, uy, ux uy, uz, ux uz, uy uz, ux uy uz}
// (the record order), scaled by w: the sample's contribution to a record's moment
// gradient.  One FMUL and three FMUL2.
__device__ __forceinline__ void monomials(float w, float ux, float uy, float uz, float2 m[4]) {
  m[0] = make_float2(w, __fmul_rn(w, ux));
  m[1] = mul2(bcast(uy), m[0]);
  m[2] = mul2(bcast(uz), m[0]);
  m[3] = mul2(bcast(uz), m[1]);
}

// acc = acc * keep + m over the 8 moments (four FFMA2)
__device__ __forceinline__ void moments_fma(float acc[8], float keep, const float2 m[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 a = fma2(make_float2(acc[2 * j], acc[2 * j + 1]), bcast(keep), m[j]);
    acc[2 * j] = a.x;
    acc[2 * j + 1] = a.y;
  }
}
// polynomial coefficients of the cell (one 256-bit record, or the 8 corner
// voxels converted in registers for the plain voxel layout)
template <bool CELLS>
__device__ __forceinline__ void fetch8(const VolArgs& V, const Cell& c, float v[8]) {
  if (CELLS) {
    gather(V, c.cell, v);
  } else {
    const float* p = V.data + c.base;
    float k[8];
    k[0] = __ldg(p);
    k[1] = __ldg(p + c.ox);
    k[2] = __ldg(p + c.oy);
    k[3] = __ldg(p + c.ox + c.oy);
    k[4] = __ldg(p + c.oz);
    k[5] = __ldg(p + c.ox + c.oz);
    k[6] = __ldg(p + c.oy + c.oz);
    k[7] = __ldg(p + c.ox + c.oy + c.oz);
    corners_to_poly(k, v);
  }
}

// Partial products of the interpolant, kept for the spatial derivative.
struct Interp {
  float rho;   // unclamped density
  float gx;    // d rho / d ux
  float2 q1;   // (cz + uy cyz, cxz + uy cxyz): d rho / d uz = q1.x + ux q1.y
};

__device__ __forceinline__ Interp interp(const Cell& c, const float k[8]) {
  Interp r;
  // lane pairs (x-free, x-carrying): q0 = (uy cy, cx + uy cxy) (the x-free lane
  // adds uy cy to 0: k[0] = c0 is added last), q1 = (cz + uy cyz, cxz + uy cxyz),
  // q = q0 + uz q1 = (rho - c0 at ux = 0, d rho / d ux)
  const float2 q0 = make_float2(__fmul_rn(c.uy, k[2]), __fmaf_rn(c.uy, k[3], k[1]));
  r.q1 = fma2(bcast(c.uy), make_float2(k[6], k[7]), make_float2(k[4], k[5]));
  const float2 q = fma2(bcast(c.uz), r.q1, q0);
  r.gx = q.y;
  // the variation first, the mean c0 last: one rounding at |rho| (the fp32
  // interpolant is then as accurate as the lerp form: rms 2.1e-8 against fp64
  // on uniform [0,1) corners)
  r.rho = __fadd_rn(k[0], __fmaf_rn(c.ux, q.y, q.x));
  return r;
}

// d rho / d uy and d rho / d uz (grid units)
__device__ __forceinline__ float interp_gy(const Cell& c, const float k[8]) {
  return __fmaf_rn(c.uz, __fmaf_rn(c.ux, k[7], k[6]), __fmaf_rn(c.ux, k[3], k[2]));
}
__device__ __forceinline__ float interp_gz(const Cell& c, const Interp& r) {
  return __fmaf_rn(c.ux, r.q1.y, r.q1.x);
}

// density actually used by the march: 0 outside the box, clamped to [0,1]
__device__ __forceinline__ float clamp_density(bool inside, float raw) {
  return inside ? fminf(fmaxf(raw, 0.f), 1.f) : 0.f;
}

// ---------------------------------------------------------------------------
// transfer functions (field.py:525-579; renderer.py:472-488)
// ---------------------------------------------------------------------------

// Dynamic shared memory of every kernel (R = TF texels; float offsets):
//   [0, 8(R+1))          the TF as two planes of R+1 float4 entries with guard
//                        entries at both ends (see texel_coord): texels [0, R+1),
//                        then the deltas next texel - texel [R+1, 2R+2) (float4
//                        index).  One 16-byte load per plane and sample: lanes of a
//                        warp reading up to 8 consecutive entries hit distinct banks
//                        (interleaved 32-byte pairs conflicted from 4 on)
//   [8(R+1), 12R+8)      the per-CTA TF gradient (adjoint, tf target)
//   [12R+8, 14R+10)      (tau, next tau - tau) float2 pairs: the table of an
//                        emission-free TF (rgb texels all zero, e.g. the
//                        absorption ramp of tasks.py:348-356), one 64-bit load
// (piecewise / Gaussian TFs use their own layouts, see pl_eval / gauss_eval)
// A file-scope symbol keeps loads in the shared window (no generic->shared
// conversion per access).
extern __shared__ float4 g_smem[];

// Texel tables carry guard entries: entry e = i + 1 for texel coordinate
// i in [-1, R-1], where entries 0 and R are clones of texels 0 and R-1 with a
// zero delta.  Clamp-to-edge (field.py:543-548) and the zero slope of the
// clamp bands (field.py:575-576) are then baked into the table: i = floor(t),
// w = t - i, no clamps and no live test.  (Only the measure-zero point
// t = R-1 exactly differs: the reference takes the left interval's slope.)
// Float offsets: texel and delta planes [0, 8(R+1)), TF gradient [8(R+1), 12R+8),
// tau pairs [12R+8, 14R+10).
__device__ __forceinline__ const float2* tau_table(const TfArgs& T) {
  return reinterpret_cast<const float2*>(g_smem) + (6 * T.count + 4);
}

// texel coordinate i = floor(d R - 1/2) in [-1, R-1] (d in [0, 1]) and weight w
__device__ __forceinline__ int texel_coord(const TfArgs& T, float d, float& w) {
  const float t = __fmaf_rn(d, T.fR, -0.5f);
  const float fl = floorf(t);
  w = __fsub_rn(t, fl);
  return (int)fl;
}

// tau-only lookup of an emission-free TF (same arithmetic as tf_eval's w channel)
__device__ __forceinline__ float tf_eval_tau(const TfArgs& T, float d, int& i0, float& w,
                                             float& slope_tau, bool want_slope) {
  i0 = texel_coord(T, d, w);
  const float2 q = tau_table(T)[i0 + 1];
  if (want_slope) slope_tau = q.y * T.fR;
  return __fmaf_rn(w, q.y, q.x);
}

// a + w dlt on the four channels (two FFMA2)
__device__ __forceinline__ float4 lerp_texel(float w, const float4& a, const float4& dlt) {
  const float2 xy = fma2(bcast(w), make_float2(dlt.x, dlt.y), make_float2(a.x, a.y));
  const float2 zw = fma2(bcast(w), make_float2(dlt.z, dlt.w), make_float2(a.z, a.w));
  return make_float4(xy.x, xy.y, zw.x, zw.y);
}

// texel table: R texels, centre of texel r at (r + 0.5)/R, clamp-to-edge
// (field.py:540-549); fR, fR1, Rm2 are precomputed on the host (TfArgs)
__device__ __forceinline__ float4 tf_eval(const TfArgs& T, float d, int& i0, float& w,
                                          float4& slope, bool want_slope) {
  i0 = texel_coord(T, d, w);
  const float4 a = g_smem[i0 + 1];
  const float4 dlt = g_smem[T.count + 2 + i0];
  if (want_slope) {   // guard entries have dlt = 0: the clamp bands' zero slope
    const float2 sxy = mul2(make_float2(dlt.x, dlt.y), bcast(T.fR));
    const float2 szw = mul2(make_float2(dlt.z, dlt.w), bcast(T.fR));
    slope = make_float4(sxy.x, sxy.y, szw.x, szw.y);
  }
  return lerp_texel(w, a, dlt);
}

// Piecewise-linear TF on non-uniform knots, params (K,5) = [pos, r, g, b, tau].
// No reference implementation: linear between knots, clamp-to-
// edge outside [pos_0, pos_K-1] with zero slope there, as the texel table
// (field.py:540-549, 575-576); equals it for knots at (r+0.5)/R.  Shared layout:
// float4 val[K], float4 slope[K] ((v_k+1 - v_k)/span_k), float pos[K].
// Returns the knot interval k (texel-like handle) and its weight w.
__device__ __forceinline__ float4 pl_eval(const TfArgs& T, float d, int& k, float& w,
                                          float4& slope, bool want_slope) {
  const int K = T.count;
  const float4* val = g_smem;
  const float4* slp = g_smem + K;
  const float* pos = reinterpret_cast<const float*>(g_smem + 2 * K);
  float4 sl = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 out;
  if (K == 1 || d <= pos[0]) {
    k = 0; w = 0.f; out = val[0];
  } else if (d >= pos[K - 1]) {
    k = K - 2; w = 1.f; out = val[K - 1];
  } else {   // pos[lo] <= d < pos[hi]
    int lo = 0, hi = K - 1;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pos[mid] <= d) lo = mid; else hi = mid;
    }
    k = lo;
    sl = slp[k];
    const float u = __fsub_rn(d, pos[k]);
    const float4 a = val[k];
    w = __fdiv_rn(u, __fsub_rn(pos[k + 1], pos[k]));
    out = make_float4(__fmaf_rn(u, sl.x, a.x), __fmaf_rn(u, sl.y, a.y), __fmaf_rn(u, sl.z, a.z),
                      __fmaf_rn(u, sl.w, a.w));
  }
  if (want_slope) slope = sl;
  return out;
}

// Analytic sum-of-Gaussians TF, params (G,6) = [mu, sigma, r, g, b, tau]:
// out(d) = sum_j exp(-(d-mu_j)^2 / 2 sigma_j^2) rgba_j.  No reference
// implementation: the optical model of the reference's 1-D demo
// (tasks.py:751-766).  Shared layout: float4 rgba[G], float4 (mu, log2e/2s^2,
// 1/s^2, s)[G].
__device__ __forceinline__ float4 gauss_eval(const TfArgs& T, float d, float4& slope,
                                             bool want_slope) {
  const float4* rgba = g_smem;
  const float4* prm = g_smem + T.count;
  float4 out = make_float4(0.f, 0.f, 0.f, 0.f), sl = out;
  for (int j = 0; j < T.count; ++j) {
    const float4 q = prm[j];
    const float4 c = rgba[j];
    const float z = __fsub_rn(d, q.x);
    float g;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(g) : "f"(-(z * z) * q.y));
    out.x += g * c.x; out.y += g * c.y; out.z += g * c.z; out.w += g * c.w;
    if (want_slope) {
      const float gd = -g * z * q.z;
      sl.x += gd * c.x; sl.y += gd * c.y; sl.z += gd * c.z; sl.w += gd * c.w;
    }
  }
  if (want_slope) slope = sl;
  return out;
}

constexpr int kTfTexture = DDVR_TF_TEXTURE, kTfPiecewise = DDVR_TF_PIECEWISE,
              kTfGaussian = DDVR_TF_GAUSSIAN;


// (rgb, tau) of density d and its slope, for TF kind KIND; i0/w identify the
// texel or knot interval (texture, piecewise).  EMIT=false: emission-free
// texel table (rgb identically 0).
template <int KIND, bool EMIT>
__device__ __forceinline__ float4 tf_sample(const TfArgs& T, float d, int& i0, float& w,
                                            float4& slope, bool want_slope) {
  if (KIND == kTfPiecewise) return pl_eval(T, d, i0, w, slope, want_slope);
  if (KIND == kTfGaussian) { i0 = 0; w = 0.f; return gauss_eval(T, d, slope, want_slope); }
  if (EMIT) return tf_eval(T, d, i0, w, slope, want_slope);
  float slope_tau = 0.f;
  const float tau = tf_eval_tau(T, d, i0, w, slope_tau, want_slope);
  if (want_slope) slope = make_float4(0.f, 0.f, 0.f, slope_tau);
  return make_float4(0.f, 0.f, 0.f, tau);
}

// Beer-Lambert segment opacity with the invertibility clamp (field.py:587-600)
struct Segment {
  float tau, e, ome, a;   // ome = 1 - a = max(e, EPS)
  float od;               // segment optical depth -ln(1 - a) = min(dt*tau, -ln EPS), exact
  bool a_clamped;
};

constexpr float kNegLnEps = 13.815510557964274f;   // -ln(EPS_ALPHA)

// How a = 1 - exp(-x), x = dt*tau, is evaluated.  Each CTA picks the cheapest
// mode that is exact to fp32 for x <= x_max = dt * max(tau texel):
//   kSegP3  x_max < 0.00896: a = x - x^2/2 + x^3/6 (truncation < 3e-8 relative)
//   kSegP7  x_max < ln2/2:   degree-7 Taylor polynomial of -expm1(-x) (< 5e-9)
//   kSegGen otherwise:       polynomial below ln2/2, 1 - exp(-x) above, EPS clamp
// In the polynomial modes e = 1 - a >= 0.7 is exact to half an ulp and the
// clamp cannot trigger.  (fp32 1 - __expf(-x) alone loses ~1e-5 relative on a
// at dt*tau ~ 5e-3.)
constexpr int kSegP3 = 0, kSegP7 = 1, kSegGen = 2;

template <int SEG>
__device__ __forceinline__ Segment segment(float tau_raw, float dt32) {
  Segment s;
  s.tau = fmaxf(tau_raw, 0.f);
  const float x = __fmul_rn(dt32, s.tau);
  if (SEG == kSegP3) {
    float p = __fmaf_rn(-x, 1.f / 6.f, 0.5f);
    p = __fmaf_rn(-x, p, 1.f);
    s.a = __fmul_rn(x, p);
    s.e = __fsub_rn(1.f, s.a);
    s.ome = s.e;
    s.a_clamped = false;
    s.od = x;
    return s;
  }
  float p = __fmaf_rn(-x, 1.f / 5040.f, 1.f / 720.f);
  p = __fmaf_rn(-x, p, 1.f / 120.f);
  p = __fmaf_rn(-x, p, 1.f / 24.f);
  p = __fmaf_rn(-x, p, 1.f / 6.f);
  p = __fmaf_rn(-x, p, 0.5f);
  p = __fmaf_rn(-x, p, 1.f);
  const float a_small = __fmul_rn(x, p);
  if (SEG == kSegP7) {
    s.a = a_small;
    s.e = __fsub_rn(1.f, a_small);
    s.ome = s.e;
    s.a_clamped = false;
    s.od = x;
    return s;
  }
  float e_big;   // exp(-x) = 2^(-x log2 e); ftz is harmless: e < 1e-6 is clamped below
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e_big) : "f"(__fmul_rn(x, -1.4426950408889634f)));
  const bool small = x < 0.34657359f;
  const float a_raw = small ? a_small : __fsub_rn(1.f, e_big);
  s.e = small ? __fsub_rn(1.f, a_small) : e_big;
  s.a_clamped = s.e < kEpsAlpha;                 // a_raw > 1 - EPS_ALPHA
  s.ome = s.a_clamped ? kEpsAlpha : s.e;
  s.a = s.a_clamped ? __fsub_rn(1.f, kEpsAlpha) : a_raw;
  s.od = s.a_clamped ? kNegLnEps : x;
  return s;
}

// ---------------------------------------------------------------------------
// shared prologue: TF table + view frame into shared memory
// ---------------------------------------------------------------------------

// shared TF table as (texel k, texel k+1 - texel k) planes: the lerp is then 4
// FFMA and the slope (field.py:576) needs no subtraction.  Returns (to every
// thread, after the barrier the caller issues) the segment mode of the CTA.
// s_info[0]: largest tau texel (bits), s_info[1]: 1 if any rgb texel is non-zero,
// s_info[2]: 1 if the tau column is NOT affine in the texel index, s_info[3..4]:
// the affine tau = a + b k (float bits; texel tables only, see tau_affine)
__device__ __forceinline__ void load_tf(const TfArgs& tf, unsigned* s_info) {
  if (tf.kind == kTfPiecewise) {
    const int K = tf.count;
    float* pos = reinterpret_cast<float*>(g_smem + 2 * K);
    for (int i = threadIdx.x; i < K; i += blockDim.x) {
      const float* a = tf.params + 5 * i;
      const float* b = tf.params + 5 * min(i + 1, K - 1);
      const float span = __fsub_rn(b[0], a[0]);
      const float inv = span > 0.f ? __frcp_rn(span) : 0.f;
      g_smem[i] = make_float4(a[1], a[2], a[3], a[4]);
      g_smem[K + i] = make_float4(__fsub_rn(b[1], a[1]) * inv, __fsub_rn(b[2], a[2]) * inv,
                                  __fsub_rn(b[3], a[3]) * inv, __fsub_rn(b[4], a[4]) * inv);
      pos[i] = a[0];
    }
    if (threadIdx.x == 0) { s_info[0] = 0x7f800000u; s_info[1] = 1u; s_info[2] = 1u; }
    return;   // (general segment mode, no texel-table specialisations)
  }
  if (tf.kind == kTfGaussian) {
    const int G = tf.count;
    for (int j = threadIdx.x; j < G; j += blockDim.x) {
      const float* a = tf.params + 6 * j;
      const float s2 = a[1] * a[1];
      g_smem[j] = make_float4(a[2], a[3], a[4], a[5]);
      g_smem[G + j] = make_float4(a[0], 1.4426950408889634f / (2.f * s2), 1.f / s2, a[1]);
    }
    if (threadIdx.x == 0) { s_info[0] = 0x7f800000u; s_info[1] = 1u; s_info[2] = 1u; }
    return;
  }
  const float4* src = reinterpret_cast<const float4*>(tf.params);
  float2* tau = reinterpret_cast<float2*>(g_smem) + (6 * tf.count + 4);
  float mx = 0.f;
  bool rgb = false, bent = false;
  // affine tau column (e.g. the absorption ramp of tasks.py:348-356): tau_k =
  // a + b k to within a few fp32 ulps of the end texels' magnitude
  const float aff_a = src[0].w;
  const float aff_b = tf.count > 1 ? __fdiv_rn(__fsub_rn(src[tf.count - 1].w, aff_a), tf.fR1) : 0.f;
  const double aff_tol = 5e-7 * fmax(fmax(fabs((double)aff_a), fabs((double)src[tf.count - 1].w)),
                                     1e-30);
  for (int e = threadIdx.x; e <= tf.count; e += blockDim.x) {   // guard entries 0 and R
    const float4 a = src[min(max(e - 1, 0), tf.count - 1)];
    const float4 b = src[min(e, tf.count - 1)];
    g_smem[e] = a;
    g_smem[tf.count + 1 + e] = make_float4(__fsub_rn(b.x, a.x), __fsub_rn(b.y, a.y),
                                    __fsub_rn(b.z, a.z), __fsub_rn(b.w, a.w));
    tau[e] = make_float2(a.w, __fsub_rn(b.w, a.w));
    mx = fmaxf(mx, a.w);   // interpolated tau never exceeds the largest texel
    rgb |= a.x != 0.f || a.y != 0.f || a.z != 0.f;
    const int k = min(max(e - 1, 0), tf.count - 1);
    bent |= fabs((double)a.w - ((double)aff_a + (double)aff_b * k)) > aff_tol;
  }
  // non-negative floats order like their bit patterns
  if (mx > 0.f) atomicMax(&s_info[0], __float_as_uint(mx));
  if (rgb) atomicOr(&s_info[1], 1u);
  if (bent) atomicOr(&s_info[2], 1u);
  if (threadIdx.x == 0) {
    s_info[3] = __float_as_uint(aff_a);
    s_info[4] = __float_as_uint(aff_b);
  }
}

// tau of an affine texel column at density d: the table lerp of field.py:540-549
// with clamp-to-edge is a + b clamp(t, 0, R-1), t = d R - 1/2; its slope is b
// for t in [0, R-1) and 0 in the clamp bands (the guard texels' zero deltas)
__device__ __forceinline__ float tau_affine(const TfArgs& T, float d, float a, float b) {
  const float t = __fmaf_rn(d, T.fR, -0.5f);
  return __fmaf_rn(b, fminf(fmaxf(t, 0.f), T.fR1), a);
}

__device__ __forceinline__ int seg_mode(float dt32, unsigned maxtau_bits) {
  const float xmax = dt32 * __uint_as_float(maxtau_bits);
  return xmax < 0.00896f ? kSegP3 : (xmax < 0.34657359f ? kSegP7 : kSegGen);
}

__device__ __forceinline__ void pixel_of_tile(const Geometry& G, int tx, int ty, int& px, int& py) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  px = tx * kTile + (warp & 1) * 8 + (lane & 7);
  py = G.row0 + ty * kTile + (warp >> 1) * 4 + (lane >> 3);
}
__device__ __forceinline__ void pixel_of(const Geometry& G, int& px, int& py) {
  pixel_of_tile(G, blockIdx.x, blockIdx.y, px, py);
}

// CTA -> (view, tile) with view groups (G.vgroup > 1): consecutive CTAs cycle over vgroup
// consecutive views on the same tile instead of running view after view.  Measured: C4's
// fused step 68.2 -> 64.8 ms with groups of 4, whether or not the views are ordered by
// direction (so not by L2 sharing of similar ray tubes; DRAM traffic 103 -> 94 GB per
// launch).  Bijective; the last group may hold fewer views.
__device__ __forceinline__ void cta_view_tile(int vg, int& view, int& tx, int& ty) {
  const unsigned tiles = gridDim.x * gridDim.y;
  const unsigned b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const unsigned g0 = b / ((unsigned)vg * tiles) * (unsigned)vg;
  const unsigned gs = min((unsigned)vg, gridDim.z - g0);
  const unsigned r = b - g0 * tiles;
  const unsigned tile = r / gs;
  view = (int)(g0 + (r - tile * gs));
  tx = (int)(tile % gridDim.x);
  ty = (int)(tile / gridDim.x);
}

// ---------------------------------------------------------------------------
// forward kernel (renderer.py:306-357)
// ---------------------------------------------------------------------------

// The march of one ray.  INSIDE: every lane of the warp has all_inside (the
// per-sample inside test and clamps are compiled out); SEG: segment mode.
template <bool EARLY, bool CELLS, bool TAPE, int SEG, bool INSIDE, bool EMIT, int KIND,
          bool AFF = false, bool BITS = false, int EU = 1>
__device__ __forceinline__ void march_ray(const VolArgs& V, const TfArgs& TF, float dt32,
                                          const Ray& r, float* __restrict__ tape, float4& rgba,
                                          double& depth, float aff_a = 0.f, float aff_b = 0.f,
                                          unsigned* __restrict__ bits = nullptr,
                                          unsigned bits_off = 0u, int* nskip = nullptr) {
  // T (transmittance, accurate as T -> 0) and A (alpha, accurate as A -> 0)
  // are both carried; A += T*a is the reference's A += (1-A)*a (renderer.py:350-355).
  // S, the ray's optical depth (T = exp(-S)), is summed in fp64 for the adjoint.
  float T = 1.f, A = 0.f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
  double S = 0.0;
  long long gx = r.g0[0], gy = r.g0[1], gz = r.g0[2];
  constexpr bool kHoldCell = CELLS && DDVR_HOLD_CELL;
  // Emission-free TF (rgb = 0) without tape or early stop: the compositing
  // A += (1 - A) a_i (renderer.py:350-355) is exactly A = 1 - prod(1 - a_i)
  // = -expm1(-S), S = sum of the segment optical depths min(dt tau, -ln EPS)
  // the march sums anyway (fp64) -- so only S is carried per sample.
  constexpr bool kAbs = !EMIT && !TAPE && !EARLY && KIND == kTfTexture && DDVR_ABS_WALK;
  // BITS (band tape): one bit per sample = the clamped density d is in the band
  // t = d R - 1/2 in [0, R-1).  That equals the affine absorption walk's d_hat
  // test (adjoint_ray: inside the box and t on the raw density in the band --
  // outside, or raw outside [0,1], d clamps to 0 or 1 and t leaves the band), so
  // the walk takes it from the tape instead of re-gathering the record.  Word k
  // of the ray (samples 32k..32k+31, sample 32k+31 at bit 0; a last partial word
  // holds its samples in the low bits, the last one at bit 0) sits at bits[32 k]:
  // lane-interleaved, one 128-byte store per warp and word.
  unsigned word = 0u;
  // BITS: the optical depth of the current 32-sample word in fp32, added to the fp64 S
  // once per word (32 terms of at most dt*tau_max: ~1e-7 of a word's depth)
  float Sb = 0.f;
  const float dt_a = dt32 * aff_a, dt_b = dt32 * aff_b;   // (band march)
  // one compositing step on a located sample and its record
  auto density = [&](const Cell& c, const float* k) {
    return clamp_density(INSIDE || c.inside, interp(c, k).rho);
  };
  // kStore: the word is stored at its last sample here (else by the caller's block loop)
  auto shade = [&](float d, int i, auto kStore) {
    if (TAPE) tape[i] = T;                     // stored mode (renderer.py:348-349)
    if (kAbs && AFF && BITS) {
      // band march (non-negative affine tau column): band bit = t in [0, R-1) -- the
      // texel table's slope band (its guard texel at R-1 has a zero delta; the
      // reference's closed live range differs only at t == R-1 exactly) -- pushed in at
      // the LSB (the walk pops it from there); dt*tau = dt*a + dt*b*clamp(t) in one
      // FFMA (tau >= 0 here)
      const float t = __fmaf_rn(d, TF.fR, -0.5f);
      const float tc = fminf(fmaxf(t, 0.f), TF.fR1);
      word = (word << 1) | (t >= 0.f && t < TF.fR1 ? 1u : 0u);
      if (decltype(kStore)::value && (i & 31) == 31) {
        bits[bits_off + ((i >> 5) << 5)] = word;
        word = 0u;
      }
      const float x = __fmaf_rn(dt_b, tc, dt_a);
      Sb = __fadd_rn(Sb, SEG == kSegGen ? fminf(x, kNegLnEps) : x);   // per word
      return;
    }
    if (kAbs && AFF) {   // affine tau column: no table lookup
      const float t = __fmaf_rn(d, TF.fR, -0.5f);
      const float tau = __fmaf_rn(aff_b, fminf(fmaxf(t, 0.f), TF.fR1), aff_a);   // tau_affine
      const float x = __fmul_rn(dt32, fmaxf(tau, 0.f));
      S += (double)(SEG == kSegGen ? fminf(x, kNegLnEps) : x);
      return;
    }
    int i0; float w;
    float4 slope;
    const float4 s = tf_sample<KIND, EMIT>(TF, d, i0, w, slope, false);
    if (kAbs) {   // segment optical depth only (the EPS clamp of field.py:587-600)
      const float x = __fmul_rn(dt32, fmaxf(s.w, 0.f));
      S += (double)(SEG == kSegGen ? fminf(x, kNegLnEps) : x);
      return;
    }
    const Segment g = segment<SEG>(s.w, dt32);
    const float Ta = __fmul_rn(T, g.a);
    if (EMIT) {
      const float2 c01 = fma2(bcast(Ta), make_float2(s.x, s.y), make_float2(c0, c1));
      c0 = c01.x;
      c1 = c01.y;
      c2 = __fmaf_rn(Ta, s.z, c2);
    }
    A = __fadd_rn(A, Ta);
    T = __fmul_rn(T, g.ome);
    S += (double)g.od;
  };
  float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  int held = INT_MIN;
  if (kHoldCell) {
    // The record of sample i+1 is requested as soon as sample i's interpolant
    // has consumed the registers (a later load may overwrite registers an
    // earlier instruction has read), so the gather overlaps sample i's TF,
    // opacity and compositing -- no extra registers.
    const bool ins = INSIDE || r.all_inside;
    Cell c;
    locate<CELLS>(V, gx, gy, gz, ins, c);
    gather_if(V, r.n > 0, c.cell, v);
    held = c.cell;
    // (the emitting variants spill at 48 registers when unrolled)
    constexpr int kMarchUnroll = kAbs ? (BITS ? DDVR_BITS_MARCH_UNROLL : 4) : EU;
    // kMore: the next sample exists (known inside whole words but the last)
    auto step_m = [&](int i, auto kStore, auto kMore) {
      // (band march of inside rays: the raw interpolant -- the band test and the clamp
      // of t to [0, R-1] give the same bit and tau as on the [0,1]-clamped density)
      const float d = (kAbs && AFF && BITS && INSIDE) ? interp(c, v).rho : density(c, v);
      gx += r.gs[0]; gy += r.gs[1]; gz += r.gs[2];
      locate<CELLS>(V, gx, gy, gz, ins, c);
      const bool more = decltype(kMore)::value || i + 1 < r.n;
      gather_if(V, more && c.cell != held, c.cell, v);
      held = c.cell;
      shade(d, i, kStore);
    };
    auto step = [&](int i, auto kStore) { step_m(i, kStore, std::false_type{}); };
    // Empty-space skip (band tape): when every sample of a block of 32 (one tape word)
    // lies in unoccupied bricks, each reads an all-zero record: d = 0, band bit 0 and --
    // when tau(0) = aff_a <= 0 -- an optical depth of exactly 0.  The block's word is
    // stored as 0 and the march moves on 32 steps: the same S, image and tape as
    // marching it.
    constexpr long long kSkipStep = (8LL << 32) / 31;   // 31 steps < 8 cells per axis
    const bool skip = BITS && V.occ != nullptr && aff_a <= 0.f &&
                      llabs(r.gs[0]) < kSkipStep && llabs(r.gs[1]) < kSkipStep &&
                      llabs(r.gs[2]) < kSkipStep;
    const int back = (r.gs[0] < 0 ? 1 : 0) | (r.gs[1] < 0 ? 2 : 0) | (r.gs[2] < 0 ? 4 : 0);
    if (BITS) {   // by tape words (the same arithmetic with and without the skip)
      for (int i0 = 0; i0 < r.n; i0 += 32) {
        if (skip && block_empty(V, gx, gy, gz, back)) {
          if (nskip) *nskip += min(32, r.n - i0);
          if (i0 + 32 <= r.n) bits[bits_off + i0] = 0u;   // word i0/32 (a last partial
          gx += 32 * r.gs[0]; gy += 32 * r.gs[1]; gz += 32 * r.gs[2];   // word: after the loop)
          if (i0 + 32 < r.n) {
            locate<CELLS>(V, gx, gy, gz, ins, c);
            gather(V, c.cell, v);
            held = c.cell;
          }
          continue;
        }
        if (i0 + 32 <= r.n) {   // a whole word: fixed trip count, one store after it
#pragma unroll kMarchUnroll
          for (int j = 0; j < 31; ++j) step_m(i0 + j, std::false_type{}, std::true_type{});
          step(i0 + 31, std::false_type{});
          bits[bits_off + i0] = word;
          word = 0u;
        } else {                // the last partial word (stored after the march)
          for (int i = i0; i < r.n; ++i) step(i, std::false_type{});
        }
        S += (double)Sb;
        Sb = 0.f;
      }
    } else {
#pragma unroll kMarchUnroll
      for (int i = 0; i < r.n; ++i) {
        if (EARLY && A > kAlphaStop) break;      // renderer.py:331-335
        step(i, std::true_type{});
      }
    }
  } else {
    for (int i = 0; i < r.n; ++i) {
      if (EARLY && A > kAlphaStop) break;      // renderer.py:331-335
      Cell c;
      locate<CELLS>(V, gx, gy, gz, INSIDE || r.all_inside, c);
      gx += r.gs[0]; gy += r.gs[1]; gz += r.gs[2];
      fetch8<CELLS>(V, c, v);
      shade(density(c, v), i, std::true_type{});
    }
  }
  if (BITS && (r.n & 31)) bits[bits_off + ((r.n >> 5) << 5)] = word;   // partial last word
  if (kAbs) A = (float)(-expm1(-S));
  rgba = make_float4(c0, c1, c2, A);
  depth = S;
}

// The march of one ray with the variant the CTA's TF selects (kind, emission,
// segment mode) and the warp's inside flag.  ABS_ONLY: only the emission-free
// texel variants are compiled (the absorption-only kernels).
template <bool EARLY, bool CELLS, bool TAPE, bool ABS_ONLY, int EU = 1>
__device__ __forceinline__ void march_dispatch(const VolArgs& V, const TfArgs& TFA, float dt32,
                                               const Ray& r, float* __restrict__ tape,
                                               bool warp_inside, bool emit, int mode,
                                               float4& rgba, double& S, const unsigned* info,
                                               unsigned* __restrict__ bits = nullptr,
                                               unsigned bits_off = 0u, int* nskip = nullptr) {
  // the affine-tau variant serves emission-free texel TFs without tape / early stop
  const bool aff = !EARLY && !TAPE && !emit && info[2] == 0u;
  const float aa = __uint_as_float(info[3]), ab = __uint_as_float(info[4]);
#define DDVR_MARCH(SEG, INS, EM) \
  march_ray<EARLY, CELLS, TAPE, SEG, INS, EM, kTfTexture, false, false, EU>(V, TFA, dt32, r, tape, \
                                                                          rgba, S)
#define DDVR_MARCH_SEG(INS, EM)                  \
  if (mode == kSegP3) DDVR_MARCH(kSegP3, INS, EM); \
  else if (mode == kSegP7) DDVR_MARCH(kSegP7, INS, EM); \
  else DDVR_MARCH(kSegGen, INS, EM);
#define DDVR_MARCH_AFF(SEG, INS) \
  march_ray<EARLY, CELLS, TAPE, SEG, INS, false, kTfTexture, true>(V, TFA, dt32, r, tape, rgba, \
                                                                    S, aa, ab)
#define DDVR_MARCH_SEG_AFF(INS)                  \
  if (mode == kSegP3) DDVR_MARCH_AFF(kSegP3, INS); \
  else if (mode == kSegP7) DDVR_MARCH_AFF(kSegP7, INS); \
  else DDVR_MARCH_AFF(kSegGen, INS);
#define DDVR_MARCH_BITS(SEG, INS)                                                          \
  march_ray<EARLY, CELLS, TAPE, SEG, INS, false, kTfTexture, true, true>(V, TFA, dt32, r, tape, \
                                                                          rgba, S, aa, ab, bits, \
                                                                          bits_off, nskip)
  if (ABS_ONLY && CELLS && !EARLY && !TAPE && bits) {   // (the caller checked the band walk)
    if (warp_inside) {
      if (mode == kSegP3) DDVR_MARCH_BITS(kSegP3, true); else DDVR_MARCH_BITS(kSegP7, true);
    } else {
      if (mode == kSegP3) DDVR_MARCH_BITS(kSegP3, false); else DDVR_MARCH_BITS(kSegP7, false);
    }
  } else if ((ABS_ONLY || (TFA.kind == kTfTexture && !emit)) && aff && !EARLY && !TAPE) {
    if (warp_inside) { DDVR_MARCH_SEG_AFF(true) } else { DDVR_MARCH_SEG_AFF(false) }
  } else if (ABS_ONLY) {
    if (warp_inside) { DDVR_MARCH_SEG(true, false) } else { DDVR_MARCH_SEG(false, false) }
  } else if (TFA.kind == kTfPiecewise) {
    march_ray<EARLY, CELLS, TAPE, kSegGen, false, true, kTfPiecewise>(V, TFA, dt32, r, tape,
                                                                       rgba, S);
  } else if (TFA.kind == kTfGaussian) {
    march_ray<EARLY, CELLS, TAPE, kSegGen, false, true, kTfGaussian>(V, TFA, dt32, r, tape,
                                                                      rgba, S);
  } else if (warp_inside) {
    if (emit) { DDVR_MARCH_SEG(true, true) } else { DDVR_MARCH_SEG(true, false) }
  } else {
    if (emit) { DDVR_MARCH_SEG(false, true) } else { DDVR_MARCH_SEG(false, false) }
  }
#undef DDVR_MARCH_BITS
#undef DDVR_MARCH_SEG_AFF
#undef DDVR_MARCH_AFF
#undef DDVR_MARCH_SEG
#undef DDVR_MARCH
}

#ifndef DDVR_FWD_MINB
#define DDVR_FWD_MINB 5
#endif
// CTAs per SM the adjoint is compiled for, per target mask (ptxas' own
// choice swings between 64 and 95 registers for the volume-only walk with
// unrelated code changes): volume-only fits 64 registers without spills
// (4 CTAs/SM); the camera/stepsize walks carry fp64 sums (ptxas' choice).
// The absorption-only kernel (ROLE 1) carries none of the emitting walk's
// state and is compiled for 5 CTAs/SM.
#ifndef DDVR_POS_MINB
#define DDVR_POS_MINB 4   // camera / stepsize walks (fp64 per-ray sums): 4 CTAs/SM at 64 registers
                          // (some spills to L1, which runs at 34% here) beat 3 at 80: C3 +2.4%,
                          // and 3 beat 2 by 13% (profiles/r02_minb3)
#endif
#ifndef DDVR_VOL_MINB
#define DDVR_VOL_MINB 4   // volume-target walks (ROLE 0: the emitting inversion walk)
#endif
#ifndef DDVR_TF_MINB
#define DDVR_TF_MINB 3    // TF-target walks
#endif
constexpr int adj_min_blocks(unsigned mask, int role, bool cells, bool fused) {
  return !cells ? 2   // voxel layout: 8 scalar gathers per sample, more live state
         // the fused absorption step carries the band-tape word and pointer
         // through the march: 64 registers (4 CTAs/SM) beat 48 with spills
         : (role == 1 && mask == DDVR_TARGET_VOLUME && fused) ? DDVR_ABS_FUSED_MINB
         : (role == 1 && mask == DDVR_TARGET_VOLUME) ? DDVR_ABS_MINB
         : mask == DDVR_TARGET_VOLUME ? DDVR_VOL_MINB
         // camera / stepsize with the TF target too: fp64 sums + texel runs (128 registers)
         : (mask & (DDVR_TARGET_CAMERA | DDVR_TARGET_STEPSIZE)) && (mask & DDVR_TARGET_TF) ? 2
         : (mask & (DDVR_TARGET_CAMERA | DDVR_TARGET_STEPSIZE)) ? DDVR_POS_MINB : DDVR_TF_MINB;
}
#ifdef DDVR_ADJ_MINB
#define DDVR_ADJ_BOUNDS __launch_bounds__(kThreads, DDVR_ADJ_MINB)
#else
// (segment-split TF steps are small: 2 CTAs/SM, the registers of the unsplit TF walk's
// spills; split camera / stepsize walks keep their 4 CTAs/SM)
#ifndef DDVR_SPLIT_MINB
#define DDVR_SPLIT_MINB 2
#endif
#define DDVR_ADJ_BOUNDS                                                                   \
  __launch_bounds__(kThreads, SPLIT > 1 && !(MASK & (DDVR_TARGET_CAMERA | DDVR_TARGET_STEPSIZE)) \
                                  ? DDVR_SPLIT_MINB                                         \
                                  : adj_min_blocks(MASK, ROLE, CELLS, FUSED))
#endif
template <bool EARLY, bool CELLS, bool TAPE>
__global__ void __launch_bounds__(kThreads, TAPE ? 4 : DDVR_FWD_MINB) dvr_forward_kernel(VolArgs V, TfArgs TFA, Geometry G,
                                                             float* __restrict__ image,
                                                             float* __restrict__ depth) {
  __shared__ Frame F;
  __shared__ unsigned s_info[5];
  const int view = blockIdx.z;
  if (threadIdx.x < 5) s_info[threadIdx.x] = 0u;
  __syncthreads();
  load_tf(TFA, s_info);
  if (threadIdx.x == 0) make_frame(G.cams[view], G.W, G.H, F);
  __syncthreads();
  const int mode = seg_mode(G.dt32, s_info[0]);
  const bool emit = s_info[1] != 0u;

  int px, py;
  pixel_of(G, px, py);
  const bool valid = px < G.W && py < G.row1;
  Ray r;
  r.n = 0;
  r.all_inside = true;
  if (valid) setup_ray(F, V, G.dt, G.W, G.H, px, py, r);
  const bool warp_inside = CELLS && __all_sync(0xffffffffu, r.all_inside);
  if (!valid) return;

  const size_t pix = ((size_t)view * (G.row1 - G.row0) + (py - G.row0)) * G.W + px;
  float* tape = TAPE ? G.tape + pix * G.tape_stride : nullptr;
  float4 rgba;
  double S;
  march_dispatch<EARLY, CELLS, TAPE, false>(V, TFA, G.dt32, r, tape, warp_inside, emit, mode,
                                             rgba, S, s_info);
  reinterpret_cast<float4*>(image)[pix] = rgba;
  if (depth) depth[pix] = (float)S;
}

// ---------------------------------------------------------------------------
// adjoint kernel (renderer.py:491-685)
// ---------------------------------------------------------------------------

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// flush of one cell run: into the cell-gradient workspace (two 128-bit vector
// reds) or, without cell records, straight into the voxel gradient
template <bool CELLS>
__device__ __forceinline__ void flush_cell(float* __restrict__ d_volume,
                                           float* __restrict__ d_cells, int cell, int base,
                                           int ox, int oy, int oz, const float acc[8]) {
  if (CELLS) {
    float* q = d_cells + 8 * (long long)cell;
    red128(q, acc[0], acc[1], acc[2], acc[3]);
    red128(q + 4, acc[4], acc[5], acc[6], acc[7]);
  } else {
    float* q = d_volume + base;
    atomicAdd(q, acc[0]);
    if (ox) atomicAdd(q + ox, acc[1]);
    if (oy) atomicAdd(q + oy, acc[2]);
    if (ox && oy) atomicAdd(q + ox + oy, acc[3]);
    if (oz) {
      atomicAdd(q + oz, acc[4]);
      if (ox) atomicAdd(q + ox + oz, acc[5]);
      if (oy) atomicAdd(q + oy + oz, acc[6]);
      if (ox && oy) atomicAdd(q + ox + oy + oz, acc[7]);
    }
  }
}

// flush of a texel / knot run (texel coordinate `run` and run + 1, weights
// accumulated in a0 / a1) into this CTA's TF-gradient slot: two 128-bit
// vector reds for the rgba rows (+ the knot-position gradient of a piecewise
// TF).  Global fp32 reds are native; shared-memory fp32 atomics are CAS loops
// on sm_100a and serialised on the few hot texels (the earlier design).
// (texel runs start at the guard coordinate -1, which maps onto texel 0)
__device__ __forceinline__ void tf_flush_run(float* slot, int count, int kind, int run,
                                             const float4& a0, const float4& a1, float p0,
                                             float p1) {
  const int j0 = max(run, 0);
  const int j1 = min(run + 1, count - 1);
  red128(slot + 4 * j0, a0.x, a0.y, a0.z, a0.w);
  red128(slot + 4 * j1, a1.x, a1.y, a1.z, a1.w);
  if (kind == kTfPiecewise) {
    atomicAdd(slot + 4 * count + j0, p0);
    atomicAdd(slot + 4 * count + j1, p1);
  }
}

#ifndef DDVR_TF_SLIDE
#define DDVR_TF_SLIDE 1   // 0: flush both rows of a texel run at every texel change (A/B)
#endif
// one row of a texel / knot run (coordinate k, clamped onto the table) into the slot
__device__ __forceinline__ void tf_flush_row(float* slot, int count, int kind, int k,
                                             const float4& a, float p) {
  const int j = min(max(k, 0), count - 1);
  red128(slot + 4 * j, a.x, a.y, a.z, a.w);
  if (kind == kTfPiecewise) atomicAdd(slot + 4 * count + j, p);
}

constexpr int kNoRun = INT_MIN;   // padded cell indices can be negative

// Per-ray adjoint accumulators that outlive the walk
struct AdjState {
  int run_cell, run_base, run_ox, run_oy, run_oz;   // volume cell run
  float acc8[8];
  int tf_run;                                       // TF texel/knot run (i0, i0+1)
  float4 tfa0, tfa1;
  float tfp0, tfp1;                                 // knot-position gradient (piecewise)
  // camera / stepsize per-ray sums (grid units) in fp64: thousands of terms
  // with cancellation (the per-sample terms stay fp32)
  double s1x, s1y, s1z, s2x, s2y, s2z, dt_bl, dt_pos;
  int i_off;   // sample index of the walk's first sample on the whole ray (segment-split rays)
};

// The backward walk of one ray (renderer.py:547-626).
template <unsigned MASK, bool CELLS, int SEG, bool INSIDE, bool EMIT, int KIND, bool TAPE,
          bool AFF = false, bool DET = false>
__device__ __forceinline__ void adjoint_ray(const VolArgs& V, const TfArgs& TF, float dt32,
                                            const Ray& r, double S, float4 sd,
                                            const float* __restrict__ tape, float* tf_slot,
                                            float* __restrict__ d_volume,
                                            float* __restrict__ d_cells, AdjState& st,
                                            float aff_a = 0.f, float aff_b = 0.f) {
  constexpr bool kCam = MASK & DDVR_TARGET_CAMERA;
  constexpr bool kStep = MASK & DDVR_TARGET_STEPSIZE;
  constexpr bool kTf = MASK & DDVR_TARGET_TF;
  constexpr bool kVol = MASK & DDVR_TARGET_VOLUME;
  constexpr bool kPos = kCam || kStep;
  constexpr bool kDhat = kPos || kVol;
  // Absorption-only walk: with an emission-free TF (rgb texels all zero) and
  // no TF target, the adjoint chain has a closed form.  The blend adjoint
  // gives a_hat_i = seed_a * prod_{j>i} (1 - a_j) and T_{i-1} = prod_{j<i}
  // (1 - a_j), so the Beer-Lambert term e_i * T_{i-1} * a_hat_i equals
  // seed_a * T_n for every unclamped segment (e_i = 1 - a_i there) and 0 for
  // a clamped one (renderer.py:583-596): tau_hat is a per-ray constant
  // dt * seed_a * T_n, T_n = exp(-S) from the forward's optical depth.  No
  // inversion, exp or fp64 per sample; identical in exact arithmetic to the
  // inversion walk (and closer to it in fp32 than the walked chain).
  constexpr bool kAbs = !EMIT && !kTf && !TAPE && KIND == kTfTexture && DDVR_ABS_WALK;
  const float abs_c = kAbs ? sd.w * (float)exp(-S) : 0.f;   // seed_a * T_n
  // d_hat per unit texel delta (AFF: the affine column's slope b folded in)
  const float abs_k = abs_c * dt32 * TF.fR * (AFF ? aff_b : 1.f);
  // emitting texel TF without the TF target: the slope is only needed dotted
  // with the output adjoint, so the raw delta is kept and R applied once
  constexpr bool kEmitTex = EMIT && !kTf && KIND == kTfTexture;
  // (kEmitTex: R folded into the rgb seed and into dt for the tau term of d_hat)
  const float sRx = sd.x * TF.fR, sRy = sd.y * TF.fR, sRz = sd.z * TF.fR;
  const float dtR = dt32 * TF.fR;

  // adjoint state: rgb seed is constant along the walk (renderer.py:540)
  float a_hat = sd.w;
  // last sample position; walk back with exact integer steps
  long long gx = r.g0[0] + (long long)(r.n - 1) * r.gs[0];
  long long gy = r.g0[1] + (long long)(r.n - 1) * r.gs[1];
  long long gz = r.g0[2] + (long long)(r.n - 1) * r.gs[2];

  constexpr bool kHoldCell = CELLS && DDVR_HOLD_CELL;
  // early issue (as in the march): the next sample's record is requested as
  // soon as this sample's interpolant has read the registers.  Not for the
  // camera / stepsize walks, whose spatial derivative reads the record later.
  constexpr bool kEarly = kHoldCell && !kPos && DDVR_EARLY_WALK;
  float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  int held = INT_MIN;
  Cell cnext;
  if (kEarly) {
    locate<CELLS>(V, gx, gy, gz, INSIDE || r.all_inside, cnext);
    gather_if(V, r.n > 0, cnext.cell, v);
    held = cnext.cell;
  }
#pragma unroll 1   // (unrolled, the walks spill at their register budgets)
  for (int i = r.n - 1; i >= 0; --i) {
    Cell c;
    if (kEarly) {
      c = cnext;
    } else {
      locate<CELLS>(V, gx, gy, gz, INSIDE || r.all_inside, c);
      if (kHoldCell) {
        gather_if(V, c.cell != held, c.cell, v);
        held = c.cell;
      } else {
        fetch8<CELLS>(V, c, v);
      }
    }
    const Interp ip = interp(c, v);
    if (kEarly) {   // v consumed: the record of sample i-1 is now in flight
      locate<CELLS>(V, gx - r.gs[0], gy - r.gs[1], gz - r.gs[2], INSIDE || r.all_inside, cnext);
      gather_if(V, i > 0 && cnext.cell != held, cnext.cell, v);
      held = cnext.cell;
    }
    const float raw = ip.rho;
    const bool inside = INSIDE || c.inside;
    const float d = clamp_density(inside, raw);
    int i0; float w;
    float4 slope, s;
    float dq = 0.f;   // kAbs: the raw texel delta (the slope is dq * R)
    float4 dl4 = make_float4(0.f, 0.f, 0.f, 0.f);   // kEmitTex: the raw texel delta
    // (emission-free tables never serve the tf target: rgb and its slope are 0)
    const bool want = kDhat || (kTf && KIND != kTfTexture);
    if (kEmitTex) {   // tf_eval with the raw delta kept (d_hat below folds R once)
      i0 = texel_coord(TF, d, w);
      const float4 a = g_smem[i0 + 1];
      dl4 = g_smem[TF.count + 2 + i0];
      s = lerp_texel(w, a, dl4);
      slope = make_float4(0.f, 0.f, 0.f, 0.f);
    } else if (kAbs && AFF) {
      // non-negative affine tau column in a polynomial segment mode, no
      // stepsize target (dispatch guarantees it): tau >= 0, no EPS clamp, and
      // the slope is b for t in [0, R-1), 0 in the clamp bands -- only the band test
      // is left per sample (b is folded into abs_k).  It is taken on the raw density:
      // t in [0, R-1) already implies raw in (0, 1), where
      // d == raw, so it also carries the [0,1] live test of field.py:486-489.
      i0 = 0; w = 0.f;
      const float t = __fmaf_rn(raw, TF.fR, -0.5f);
      dq = (t >= 0.f && t < TF.fR1) ? 1.f : 0.f;
      s = make_float4(0.f, 0.f, 0.f, 0.f);
      slope = make_float4(0.f, 0.f, 0.f, 0.f);
    } else if (kAbs) {
      i0 = texel_coord(TF, d, w);
      const float2 q = tau_table(TF)[i0 + 1];
      s = make_float4(0.f, 0.f, 0.f, __fmaf_rn(w, q.y, q.x));
      dq = q.y;
      slope = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      s = tf_sample<KIND, EMIT>(TF, d, i0, w, slope, want);
    }
    const Segment g = segment<SEG>(s.w, dt32);

    // Invert the compositing step (renderer.py:579, a_prev = (a - A)/(a - 1)).
    // In optical-depth form the inverse is exact: -ln(1 - a) = g.od, so the
    // depth before this sample is S - od (fp64, no drift over thousands of
    // steps) and T_prev = exp(-S_prev) is computed fresh each step.  The fp32
    // chain T_prev = T/(1 - a) drifts to ~1e-4 on camera gradients by 2.6k steps.
    // ("stored" mode reads T_prev from the tape instead, renderer.py:576-577)
    float Tp = 0.f;
    if (TAPE) {
      Tp = tape[i];
    } else if (!kAbs) {
      S -= (double)g.od;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(Tp) : "f"((float)S * -1.4426950408889634f));
    }

    // blend adjoint (renderer.py:583-589); emission-free: the rgb terms are 0
    // (written out per case: x + 0 and a * 0 do not fold under IEEE rules)
    const float cdot = EMIT ? s.x * sd.x + s.y * sd.y + s.z * sd.z : 0.f;
    const float seg_a_hat = EMIT ? Tp * (a_hat + cdot) : Tp * a_hat;
    const float aT = g.a * Tp;
    const float h0 = EMIT ? aT * sd.x : 0.f;   // d L / d rgb
    const float h1 = EMIT ? aT * sd.y : 0.f;
    const float h2 = EMIT ? aT * sd.z : 0.f;
    if (!kAbs) a_hat = EMIT ? g.ome * a_hat - g.a * cdot : g.ome * a_hat;
    // Beer-Lambert adjoint (renderer.py:592-596)
    const float a_raw_hat = g.a_clamped ? 0.f : seg_a_hat;
    const float ea = kAbs ? (g.a_clamped ? 0.f : abs_c) : g.e * a_raw_hat;
    const float tau_hat = s.w < 0.f ? 0.f : dt32 * ea;
    if (kStep) st.dt_bl += (double)(g.tau * ea);

    if (kTf && KIND == kTfGaussian) {   // every component: d out/d(mu, sigma, rgba)
      const float4* rgba = g_smem;
      const float4* prm = g_smem + TF.count;
      for (int j = 0; j < TF.count; ++j) {
        const float4 q = prm[j];
        const float4 cj = rgba[j];
        const float z = __fsub_rn(d, q.x);
        float gj;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(gj) : "f"(-(z * z) * q.y));
        const float proj = h0 * cj.x + h1 * cj.y + h2 * cj.z + tau_hat * cj.w;
        red128(tf_slot + 4 * j, gj * h0, gj * h1, gj * h2, gj * tau_hat);
        red64(tf_slot + 4 * TF.count + 2 * j, gj * z * q.z * proj,
              gj * z * z * q.z / q.w * proj);
      }
    } else if (kTf) {   // renderer.py:602-604: texels/knots i0, i0+1 with weights (1-w), w
      if (i0 != st.tf_run) {
        // The run's two rows (tf_run, tf_run + 1) slide with the texel: a step of one
        // texel keeps the shared row open (flushed later, once), only the row leaving
        // the window is flushed -- the walk's TF reds (the binding L1 traffic of the TF
        // walks) drop by the +-1 steps (C2 20%, C1 34% of the samples)
        const bool open = st.tf_run != kNoRun;
        const bool up = DDVR_TF_SLIDE && open && i0 == st.tf_run + 1;
        const bool down = DDVR_TF_SLIDE && open && i0 == st.tf_run - 1;
        if (open && !down) tf_flush_row(tf_slot, TF.count, KIND, st.tf_run, st.tfa0, st.tfp0);
        if (open && !up) tf_flush_row(tf_slot, TF.count, KIND, st.tf_run + 1, st.tfa1, st.tfp1);
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 a0 = up ? st.tfa1 : z4, a1 = down ? st.tfa0 : z4;
        const float p0 = up ? st.tfp1 : 0.f, p1 = down ? st.tfp0 : 0.f;
        st.tfa0 = a0; st.tfa1 = a1; st.tfp0 = p0; st.tfp1 = p1;
        st.tf_run = i0;
      }
      const float w0 = 1.f - w;
      st.tfa0.x += w0 * h0; st.tfa0.y += w0 * h1; st.tfa0.z += w0 * h2; st.tfa0.w += w0 * tau_hat;
      st.tfa1.x += w * h0;  st.tfa1.y += w * h1;  st.tfa1.z += w * h2;  st.tfa1.w += w * tau_hat;
      if (KIND == kTfPiecewise) {   // d out/d pos_k = slope (w - 1), d out/d pos_k+1 = -slope w
        const float dh = slope.x * h0 + slope.y * h1 + slope.z * h2 + slope.w * tau_hat;
        st.tfp0 += dh * (w - 1.f);
        st.tfp1 -= dh * w;
      }
    }
    if (kDhat) {
      // renderer.py:606 d_hat = slope . out4_hat
      // (kEmitTex: slope . (aT sd_rgb, tau_hat) = aT (delta_rgb . R sd_rgb) + delta_tau R tau_hat)
      const float d_hat =
          kAbs ? ((s.w < 0.f || g.a_clamped) ? 0.f : dq * abs_k)
          : kEmitTex ? __fmaf_rn(aT, dl4.x * sRx + dl4.y * sRy + dl4.z * sRz,
                                 dl4.w * (s.w < 0.f ? 0.f : dtR * ea))
          : EMIT ? slope.x * h0 + slope.y * h1 + slope.z * h2 + slope.w * tau_hat
                 : slope.w * tau_hat;
      const bool live = (kAbs && AFF) ? inside   // (the band test above covers [0,1])
                                      : inside && raw >= 0.f && raw <= 1.f;   // field.py:486-489
      if (kVol && CELLS) {   // renderer.py:607-608, accumulated per cell run
        // The run accumulates the 8 moments sum dh * phi(u) (monomials: the
        // record order) of the polynomial record: the record's gradient is
        // exactly these moments (rho is linear in the coefficients), and
        // fold_cells_kernel maps them back to corner voxels through L^T.
        // One FMUL, three FMUL2 and four FFMA2 per sample instead of the 8
        // corner weights (25 instructions).  Branch-free: the finished run is
        // flushed with predicated vector reds and the accumulators restart by
        // scaling them with 0.
        // (texel tables: outside the box, or raw outside [0, 1], the clamped density sits
        // in a clamp band whose guard texel has a zero delta -- d_hat is 0 already)
        const float dh = (live || kEmitTex) ? d_hat : 0.f;
        const bool fresh = c.cell != st.run_cell;
        // (affine absorption walk: every d_hat of a ray is 0 or abs_k, so a run
        // whose weight sum acc8[0] is 0 has all moments 0 -- no red)
        const bool flush = fresh && st.run_cell != kNoRun &&
                           (!(kAbs && AFF) || st.acc8[0] != 0.f);
        // (ptxas branches around a predicated red anyway: one branch for both
        // halves, and the record address is formed only inside it)
        DDVR_REQUIRE(!flush || cell_ok(V, st.run_cell));
#ifdef DDVR_WALK_NORED   // measurement variant: the reds replaced by a register sink
        if (flush) st.tfp0 += st.acc8[0] + st.acc8[3] + st.acc8[7];
#else
        if (flush) flush_record<DET>(V, d_cells, st.run_cell, st.acc8);
#endif
        float2 m[4];
        monomials(dh, c.ux, c.uy, c.uz, m);
        moments_fma(st.acc8, fresh ? 0.f : 1.f, m);
        st.run_cell = c.cell;
      } else if (kVol) {
        if (c.cell != st.run_cell) {
          DDVR_REQUIRE(st.run_cell == kNoRun || !CELLS || cell_ok(V, st.run_cell));
          if (st.run_cell != kNoRun)
            flush_cell<CELLS>(d_volume, d_cells, st.run_cell, st.run_base, st.run_ox, st.run_oy,
                              st.run_oz, st.acc8);
          st.run_cell = c.cell;
          if (!CELLS) { st.run_base = c.base; st.run_ox = c.ox; st.run_oy = c.oy; st.run_oz = c.oz; }
#pragma unroll
          for (int k = 0; k < 8; ++k) st.acc8[k] = 0.f;
        }
        // voxel layout: corner weights prod(1/2 -+ u) straight into d_volume
        const float dh = live ? d_hat : 0.f;
        const float z0 = dh * (0.5f - c.uz), z1 = dh * (0.5f + c.uz);
        const float fy = 0.5f + c.uy, fx = 0.5f + c.ux, ey = 0.5f - c.uy;
        const float y00 = z0 * ey, y10 = z0 * fy;
        const float y01 = z1 * ey, y11 = z1 * fy;
        const float ex = 0.5f - c.ux;
        st.acc8[0] += y00 * ex; st.acc8[1] += y00 * fx;
        st.acc8[2] += y10 * ex; st.acc8[3] += y10 * fx;
        st.acc8[4] += y01 * ex; st.acc8[5] += y01 * fx;
        st.acc8[6] += y11 * ex; st.acc8[7] += y11 * fx;
      }
      if (kPos && live) {   // renderer.py:609-623 (spatial gradient, field.py:446-484)
        const float t = __fmul_rn((float)(i + st.i_off), dt32);
        const float ddx = ip.gx;                     // field.py:446-484 from the partials
        const float ddy = interp_gy(c, v);
        const float ddz = interp_gz(c, ip);
        const float bx = (gx >= 0 && gx <= V.top[0]) ? ddx * d_hat : 0.f;
        const float by = (gy >= 0 && gy <= V.top[1]) ? ddy * d_hat : 0.f;
        const float bz = (gz >= 0 && gz <= V.top[2]) ? ddz * d_hat : 0.f;
        if (kCam) {
          st.s1x += bx; st.s1y += by; st.s1z += bz;
          st.s2x += (double)(t * bx); st.s2y += (double)(t * by); st.s2z += (double)(t * bz);
        }
        if (kStep)
          st.dt_pos += (double)((float)(i + st.i_off) * (r.gw[0] * bx + r.gw[1] * by + r.gw[2] * bz));
      }
    }
    gx -= r.gs[0]; gy -= r.gs[1]; gz -= r.gs[2];
  }
}

// The affine absorption walk (volume target) from the forward's band tape
// (DDVR_FLAG_BAND_TAPE, march_ray<..., BITS>): the d_hat of sample i is abs_k
// when bit i is set, else 0 -- the test adjoint_ray<..., AFF> evaluates on the
// re-gathered record -- so the walk needs no record gathers at all: positions,
// cell fractions, the cell-run moments and their flushes only.  Same moments,
// same runs, same flush order as the gathering walk.
template <bool INSIDE, bool DET = false>
__device__ __forceinline__ void abs_bits_walk(const VolArgs& V, const Ray& r, float abs_k,
                                              const unsigned* __restrict__ bits,
                                              unsigned bits_off, float* __restrict__ d_cells,
                                              AdjState& st, int* nskip = nullptr) {
  // Blocks of 32 samples (one tape word), back to front.  A block whose word is 0
  // adds nothing and is skipped whole: the open cell run is kept, and the first
  // sample of a later block in another cell flushes it -- the flush the
  // per-sample walk does at the first cell change inside the skipped block.
  // (a 32-bit word index from the uniform tape base: one register, not a pointer pair)
  constexpr int kUnroll = DDVR_BITS_WALK_UNROLL;   // (pragma arguments are not macro-expanded)
  // the tape streams from DRAM: the word of the next block is requested one block ahead
  int blk = (r.n - 1) >> 5;
  unsigned next = blk >= 0 ? bits[bits_off + ((unsigned)blk << 5)] : 0u;
  for (; blk >= 0; --blk) {
    unsigned word = next;
    if (blk > 0) next = bits[bits_off + ((unsigned)(blk - 1) << 5)];
    if (word == 0u) {
      if (nskip) *nskip += min(32, r.n - (blk << 5));
      continue;
    }
    const int i1 = min(r.n - 1, (blk << 5) + 31);   // the block's last sample
    long long gx = r.g0[0] + (long long)i1 * r.gs[0];
    long long gy = r.g0[1] + (long long)i1 * r.gs[1];
    long long gz = r.g0[2] + (long long)i1 * r.gs[2];
#pragma unroll kUnroll
    for (int i = i1; i >= (blk << 5); --i) {
      Cell c;
      locate<true>(V, gx, gy, gz, INSIDE || r.all_inside, c);
      const float dh = (word & 1u) ? abs_k : 0.f;   // sample i's bit is the lowest left
      word >>= 1;
      const bool fresh = c.cell != st.run_cell;
      // all d_hat of the ray share abs_k's sign: a zero weight sum = an empty run
      const bool flush = fresh && st.run_cell != kNoRun && st.acc8[0] != 0.f;
#ifdef DDVR_WALK_NORED   // measurement variant: the reds replaced by a register sink
      if (flush) st.tfp0 += st.acc8[0] + st.acc8[3] + st.acc8[7];
#else
      DDVR_REQUIRE(!flush || cell_ok(V, st.run_cell));
      if (flush) flush_record<DET>(V, d_cells, st.run_cell, st.acc8);
#endif
      float2 m[4];
      monomials(dh, c.ux, c.uy, c.uz, m);
      moments_fma(st.acc8, fresh ? 0.f : 1.f, m);
      st.run_cell = c.cell;
      gx -= r.gs[0]; gy -= r.gs[1]; gz -= r.gs[2];
    }
  }
}

#ifndef DDVR_RUN_WALK
#define DDVR_RUN_WALK 1
#endif

// The affine absorption walk by cell runs (rays inside the box).  Within one cell a
// ray's centred fractions are affine in the sample index, u_k = u_0 + k d (d = the
// grid step per sample), so the run's moments sum_k b_k dh phi(u_k) (phi = 1, ux, uy,
// ux uy, uz, ux uz, uy uz, ux uy uz; b_k the band bits, dh = abs_k) follow in closed
// form from the power sums P_j = sum_k b_k k^j, j <= 3 -- for a run with every bit
// set, P_j are those of 0 .. L-1.  Per run: its start position (fixed point, exact),
// its length (samples until the first cell boundary on any axis: one fp32 quotient
// per axis; an estimate off by one only moves a sample that sits within ~1e-7 voxel
// of the boundary onto the neighbouring cell's polynomial, which agrees there), the
// moments and one flush -- instead of per-sample positions, cell tests and moment
// updates.  The samples and runs are those of abs_bits_walk (same cells, same
// gradient up to fp32 rounding); all-zero remainders of tape words are skipped.
template <bool DET = false>
__device__ __forceinline__ void abs_runs_walk(const VolArgs& V, const Ray& r, float abs_k,
                                              const unsigned* __restrict__ bits,
                                              unsigned bits_off, float* __restrict__ d_cells,
                                              int* nskip) {
  const int n = r.n;
  if (n <= 0) return;
  // per-ray constants: the u step per sample and its products, scaled by the walk
  // weight abs_k (so a run's moments need the power sums unscaled), the run-length
  // divisors
  const float dx = (float)r.gs[0] * kInvFix, dy = (float)r.gs[1] * kInvFix,
              dz = (float)r.gs[2] * kInvFix;
  const float kx = abs_k * dx, ky = abs_k * dy, kz = abs_k * dz;
  const float kxy = kx * dy, kxz = kx * dz, kyz = ky * dz, kxyz = kxy * dz;
  // samples left in the cell along an axis: floor(num / |gs|) + 1 with num = 2^32-1-lo
  // (moving up) or lo (moving down); 1/|gs| = inf on an axis the ray never leaves
  const float ix = r.gs[0] != 0 ? __frcp_rn((float)llabs(r.gs[0])) : INFINITY;
  const float iy = r.gs[1] != 0 ? __frcp_rn((float)llabs(r.gs[1])) : INFINITY;
  const float iz = r.gs[2] != 0 ? __frcp_rn((float)llabs(r.gs[2])) : INFINITY;
  const unsigned sx = r.gs[0] > 0 ? 0xffffffffu : 0u, sy = r.gs[1] > 0 ? 0xffffffffu : 0u,
                 sz = r.gs[2] > 0 ? 0xffffffffu : 0u;
  const int last_word = (n - 1) >> 5;
  // the tape as a bit stream in sample order: bit j of rw(w) = sample 32 w + j
  auto rw = [&](int w) -> unsigned {
    if (w > last_word) return 0u;
    const unsigned word = bits[bits_off + ((unsigned)w << 5)];
    return __brev(word) >> (32 - min(32, n - 32 * w));
  };
  int wcur = 0;
  unsigned long long win = (unsigned long long)rw(0) | ((unsigned long long)rw(1) << 32);
  int i = 0;
  while (i < n) {
    const int w = i >> 5;
    if (w != wcur) {   // next word (one load), or a jump (two)
      win = w == wcur + 1 ? (win >> 32) | ((unsigned long long)rw(w + 1) << 32)
                          : (unsigned long long)rw(w) | ((unsigned long long)rw(w + 1) << 32);
      wcur = w;
    }
    if (((unsigned)win >> (i & 31)) == 0u) {   // the rest of this word adds nothing
      const int to = min(32 * (w + 1), n);
      if (nskip) *nskip += to - i;
      i = to;
      continue;
    }
    const long long gx = r.g0[0] + (long long)i * r.gs[0];
    const long long gy = r.g0[1] + (long long)i * r.gs[1];
    const long long gz = r.g0[2] + (long long)i * r.gs[2];
    const unsigned lx = (unsigned)gx, ly = (unsigned)gy, lz = (unsigned)gz;
    const float Lf = fminf(fminf(__uint2float_rn(lx ^ sx) * ix, __uint2float_rn(ly ^ sy) * iy),
                           __uint2float_rn(lz ^ sz) * iz);
    const int L = min((int)fminf(Lf, 31.f) + 1, n - i);   // 1 .. 32
    const unsigned full = L == 32 ? 0xffffffffu : (1u << L) - 1u;
    const unsigned m = (unsigned)(win >> (i & 31)) & full;
    i += L;
    if (m == 0u) continue;
    float P0, P1, P2, P3;
    if (m == full) {   // every sample of the run in the band: sums over 0 .. L-1
      P0 = (float)L;
      P1 = 0.5f * P0 * (P0 - 1.f);
      P2 = P1 * (2.f * P0 - 1.f) * (1.f / 3.f);
      P3 = P1 * P1;
    } else {
      P0 = P1 = P2 = P3 = 0.f;
      for (unsigned mm = m; mm; mm &= mm - 1u) {
        const float k = (float)(__ffs(mm) - 1);
        P0 += 1.f; P1 += k; P2 += k * k; P3 += k * k * k;
      }
    }
    // sum_k dh phi(u0 + k d) expanded in the power sums (dh = abs_k folded into q0 and
    // the k* constants), in the record order {1, ux, uy, ux uy, uz, ux uz, uy uz, ux uy uz}
    const float q0 = abs_k * P0;
    const float ux = __fmaf_rn(__uint2float_rn(lx), kInvFix, -0.5f);
    const float uy = __fmaf_rn(__uint2float_rn(ly), kInvFix, -0.5f);
    const float uz = __fmaf_rn(__uint2float_rn(lz), kInvFix, -0.5f);
    const float uxy = ux * uy, uxz = ux * uz, uyz = uy * uz;
    float a[8];
    a[0] = q0;
    a[1] = __fmaf_rn(ux, q0, kx * P1);
    a[2] = __fmaf_rn(uy, q0, ky * P1);
    a[4] = __fmaf_rn(uz, q0, kz * P1);
    a[3] = __fmaf_rn(uxy, q0, __fmaf_rn(__fmaf_rn(ux, ky, uy * kx), P1, kxy * P2));
    a[5] = __fmaf_rn(uxz, q0, __fmaf_rn(__fmaf_rn(ux, kz, uz * kx), P1, kxz * P2));
    a[6] = __fmaf_rn(uyz, q0, __fmaf_rn(__fmaf_rn(uy, kz, uz * ky), P1, kyz * P2));
    const float t1 = __fmaf_rn(uxy, kz, __fmaf_rn(uxz, ky, uyz * kx));
    const float t2 = __fmaf_rn(ux, kyz, __fmaf_rn(uy, kxz, uz * kxy));
    a[7] = __fmaf_rn(uxy * uz, q0, __fmaf_rn(t1, P1, __fmaf_rn(t2, P2, kxyz * P3)));
    const int cell = (((int)(gx >> 32)) * V.CY + (int)(gy >> 32)) * V.CZ + (int)(gz >> 32);
#ifdef DDVR_WALK_NORED   // measurement variant: no reds (the atomic-free floor)
    if (a[0] == 12345.f) d_cells[0] = a[7] + (float)cell;
#else
    DDVR_REQUIRE(cell_ok(V, cell));
    flush_record<DET>(V, d_cells, cell, a);
#endif
  }
}

// The band-tape class of a fused volume-only step (CTA-uniform: it depends on the TF
// table and dt only): an emission-free texel TF whose tau column is affine and
// non-negative, a polynomial segment mode, no tape.  Its walk is abs_bits_walk.
__device__ __forceinline__ bool band_class(const TfArgs& TFA, const Geometry& G,
                                           const unsigned* s_info, int mode) {
  return G.bits != nullptr && DDVR_ABS_WALK && DDVR_AFF_WALK && TFA.kind == kTfTexture &&
         G.tape == nullptr && s_info[1] == 0u && s_info[2] == 0u && mode != kSegGen &&
         __uint_as_float(s_info[3]) >= 0.f &&
         __fmaf_rn(__uint_as_float(s_info[4]), TFA.fR1, __uint_as_float(s_info[3])) >= 0.f;
}

// ROLE 0: every walk; ROLE 1: the absorption-only walk (emission-free texel
// TF, no TF target, no tape, cell records), launched next to ROLE 0 by the
// host for masks without the TF target.  The TF class is known only on the
// device (CTA prologue), so each role's CTAs return at once when the class
// belongs to the other role -- no host synchronisation.
// FUSED: the forward march and the L1 seed run in the same thread first
// (FusedArgs); image / depth / seed are then unused.
// SPLIT > 1 (fused TF-target steps without camera / stepsize, few rays): SPLIT
// consecutive lanes share one ray, lane k marching and walking the k-th of SPLIT equal
// sample segments (8-pixel-wide CTA tiles of kThreads/SPLIT rays).  Front-to-back
// compositing is associative, so the segments' (premultiplied rgb, alpha, depth)
// compose the ray's image exactly as the serial march (up to fp32 reassociation); the
// walk of segment k starts from the depth after its last sample (prefix of the
// segments' depths) and from the blend adjoint a_hat the later segments leave behind,
// a_hat = T_after sd_a - sd_rgb . C_after (C_after, T_after: the composite of segments
// k+1.. with T = 1 at their start) -- the value the serial walk reaches there
// (renderer.py:583-589 unrolled over those samples).  A ray's serial chain is then
// SPLIT times shorter, for steps too small to fill the GPU with one thread per ray.
template <unsigned MASK, bool CELLS, int ROLE, bool FUSED, bool DET = false, int SPLIT = 1>
__global__ void DDVR_ADJ_BOUNDS dvr_adjoint_kernel(
    VolArgs V, TfArgs TFA, Geometry G, const float* __restrict__ image,
    const float* __restrict__ depth, const float* __restrict__ seed, float* __restrict__ d_volume,
    float* __restrict__ d_cells, double* __restrict__ d_camera, double* __restrict__ d_dt,
    FusedArgs Fu) {
  constexpr bool kCam = MASK & DDVR_TARGET_CAMERA;
  constexpr bool kStep = MASK & DDVR_TARGET_STEPSIZE;
  constexpr bool kTf = MASK & DDVR_TARGET_TF;
  constexpr bool kVol = MASK & DDVR_TARGET_VOLUME;
  constexpr bool kPos = kCam || kStep;

  __shared__ Frame F;
  __shared__ double s_red[kWarps][3];
  __shared__ unsigned s_info[5];
  // this CTA's TF-gradient slot in the workspace
  float* tf_slot = kTf ? TFA.slots + (size_t)TFA.slot_floats *
                                         ((blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y *
                                           (size_t)blockIdx.z)) % TFA.nslot)
                       : nullptr;
  int view = blockIdx.z, tile_x = blockIdx.x, tile_y = blockIdx.y;
  if (SPLIT == 1 && G.vgroup > 1) cta_view_tile(G.vgroup, view, tile_x, tile_y);
  if (threadIdx.x < 5) s_info[threadIdx.x] = 0u;
  __syncthreads();
  load_tf(TFA, s_info);
  __syncthreads();
  {
    const bool abs_class = !kTf && CELLS && DDVR_ABS_WALK && TFA.kind == kTfTexture &&
                           G.tape == nullptr && s_info[1] == 0u;
    if (ROLE == 0 ? abs_class : !abs_class) return;   // CTA-uniform
  }
  // the band-tape step split into dvr_band_march_kernel + dvr_band_walk_kernel
  if (ROLE == 1 && FUSED && MASK == DDVR_TARGET_VOLUME && G.ray_k != nullptr &&
      band_class(TFA, G, s_info, seg_mode(G.dt32, s_info[0])))
    return;
  if (threadIdx.x == 0) make_frame(G.cams[view], G.W, G.H, F);
  __syncthreads();
  const int mode = seg_mode(G.dt32, s_info[0]);
  // the tf target needs the rgb channels even when they are zero
  const bool emit = kTf || s_info[1] != 0u;

  static_assert(SPLIT == 1 || (FUSED && kThreads % (8 * SPLIT) == 0 && 32 % SPLIT == 0),
                "segment-split rays: fused steps");
  int px, py, seg = 0;
  if (SPLIT > 1) {   // ray (threadIdx / SPLIT) of an 8 x (kThreads / SPLIT / 8) tile
    const int rid = threadIdx.x / SPLIT;
    seg = threadIdx.x % SPLIT;
    px = blockIdx.x * 8 + (rid & 7);
    py = G.row0 + blockIdx.y * (kThreads / SPLIT / 8) + (rid >> 3);
  } else {
    pixel_of_tile(G, tile_x, tile_y, px, py);
  }
  const bool valid = px < G.W && py < G.row1;

  Ray r;
  r.n = 0;
  r.all_inside = true;
  double S = 0.0;   // optical depth after the current sample (T = exp(-S))
  float4 sd = make_float4(0, 0, 0, 0);
  const float* tape = nullptr;
  size_t pix = 0;
  if (valid) {
    setup_ray(F, V, G.dt, G.W, G.H, px, py, r);
    pix = ((size_t)view * (G.row1 - G.row0) + (py - G.row0)) * G.W + px;
    if (!FUSED) {
      if (G.tape) tape = G.tape + pix * G.tape_stride;
      sd = reinterpret_cast<const float4*>(seed)[pix];
      // the forward's exact optical depth; without it, S = -ln(1 - alpha)
      S = depth ? (double)depth[pix]
                : -log1p(-(double)reinterpret_cast<const float4*>(image)[pix].w);
    }
  }
  const bool warp_inside = CELLS && __all_sync(0xffffffffu, r.all_inside);
  int seg_i0 = 0;   // the segment's first sample on the whole ray
  if (SPLIT > 1 && valid) {   // this lane's segment [i0, i1) of the ray's samples
    const int i0 = (int)((long long)r.n * seg / SPLIT);
    const int i1 = (int)((long long)r.n * (seg + 1) / SPLIT);
#pragma unroll
    for (int k = 0; k < 3; ++k) r.g0[k] += (long long)i0 * r.gs[k];
    r.n = i1 - i0;
    seg_i0 = i0;
  }
  // affine, non-negative tau column (the ramp), polynomial segment modes, no
  // stepsize target: the table-free walk
  const bool aff_walk = DDVR_AFF_WALK && !(MASK & DDVR_TARGET_STEPSIZE) && s_info[2] == 0u &&
                        mode != kSegGen && __uint_as_float(s_info[3]) >= 0.f &&
                        __fmaf_rn(__uint_as_float(s_info[4]), TFA.fR1,
                                  __uint_as_float(s_info[3])) >= 0.f;
  // band tape (fused volume-only absorption step): this lane's word 0
  constexpr bool kBitsKernel = FUSED && ROLE == 1 && CELLS && MASK == DDVR_TARGET_VOLUME;
  // (the host keeps the tape under 2^32 words: 32-bit word indices)
  unsigned* bits = kBitsKernel && G.bits && aff_walk ? G.bits : nullptr;
  // (by the logical CTA index tile + tiles * view: the same layout whatever order the CTAs
  // ran in, and the same as the split march / walk kernels')
  const unsigned bits_off =
      ((tile_x + gridDim.x * (tile_y + gridDim.y * view)) * kWarps + (threadIdx.x >> 5)) *
          32u * (unsigned)G.bits_words + (threadIdx.x & 31);
  int march_skip = 0, walk_skip = 0;   // measurement counters (G.stats)
  if (FUSED) {   // forward march (renderer.py:306-357) + L1 seed (objectives.py:38-54)
    double loss_part = 0.0;
    float4 rgba = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
      march_dispatch<false, CELLS, false, ROLE == 1, DDVR_EMIT_MARCH_UNROLL>(
          V, TFA, G.dt32, r, nullptr, warp_inside, s_info[1] != 0u, mode, rgba, S, s_info,
          kBitsKernel ? bits : nullptr, bits_off, kBitsKernel ? &march_skip : nullptr);
    }
    double S_tot = S;
    float4 after = make_float4(0.f, 0.f, 0.f, 0.f);   // SPLIT: composite of the later segments
    float T_after = 1.f;
    if (SPLIT > 1) {   // every lane of the warp: the segment groups exchange by shuffles
      if (!valid) { rgba = make_float4(0.f, 0.f, 0.f, 0.f); S = 0.0; }
      const int base = (threadIdx.x & 31) & ~(SPLIT - 1);
      float4 tot = make_float4(0.f, 0.f, 0.f, 0.f);
      float T_front = 1.f;
      double S_end = 0.0;
      S_tot = 0.0;
#pragma unroll
      for (int j = 0; j < SPLIT; ++j) {
        const float4 c = make_float4(__shfl_sync(0xffffffffu, rgba.x, base + j),
                                     __shfl_sync(0xffffffffu, rgba.y, base + j),
                                     __shfl_sync(0xffffffffu, rgba.z, base + j),
                                     __shfl_sync(0xffffffffu, rgba.w, base + j));
        const double Sj = __shfl_sync(0xffffffffu, S, base + j);
        const float Tj = (float)exp(-Sj);   // the segment's transmittance
        tot.x = __fmaf_rn(T_front, c.x, tot.x);   // front-to-back over (renderer.py:350-355)
        tot.y = __fmaf_rn(T_front, c.y, tot.y);
        tot.z = __fmaf_rn(T_front, c.z, tot.z);
        tot.w = __fmaf_rn(T_front, c.w, tot.w);
        T_front *= Tj;
        S_tot += Sj;
        if (j <= seg) S_end += Sj;
        if (j > seg) {
          after.x = __fmaf_rn(T_after, c.x, after.x);
          after.y = __fmaf_rn(T_after, c.y, after.y);
          after.z = __fmaf_rn(T_after, c.z, after.z);
          T_after *= Tj;
        }
      }
      rgba = tot;
      S = S_end;   // the walk of this segment starts after its last sample
    }
    if (valid) {
      const float4 ref = reinterpret_cast<const float4*>(Fu.refs)[pix];
      const float dx = rgba.x - ref.x, dy = rgba.y - ref.y, dz = rgba.z - ref.z,
                  dw = rgba.w - ref.w;
      auto sgn = [&](float v) { return v > 0.f ? Fu.inv_count : (v < 0.f ? -Fu.inv_count : 0.f); };
      sd = make_float4(sgn(dx), sgn(dy), sgn(dz), sgn(dw));
      if (seg == 0) {
        loss_part = fabs((double)dx) + fabs((double)dy) + fabs((double)dz) + fabs((double)dw);
        if (Fu.image_out) reinterpret_cast<float4*>(Fu.image_out)[pix] = rgba;
        if (Fu.depth_out) Fu.depth_out[pix] = (float)S_tot;
      }
      // SPLIT: the blend adjoint's a_hat after this segment (see the kernel comment);
      // sd.w only seeds a_hat in the emitting / TF walks
      if (SPLIT > 1)
        sd.w = __fmaf_rn(T_after, sd.w, -(sd.x * after.x + sd.y * after.y + sd.z * after.z));
    }
    loss_part = warp_sum(loss_part);
    if ((threadIdx.x & 31) == 0 && loss_part != 0.0) atomicAdd(Fu.loss, loss_part * Fu.inv_count_d);
  }

  AdjState st;
  st.run_cell = kNoRun; st.run_base = 0; st.run_ox = 0; st.run_oy = 0; st.run_oz = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) st.acc8[k] = 0.f;
  st.tf_run = kNoRun;
  st.tfa0 = make_float4(0, 0, 0, 0);
  st.tfa1 = make_float4(0, 0, 0, 0);
  st.tfp0 = st.tfp1 = 0.f;
  st.s1x = st.s1y = st.s1z = st.s2x = st.s2y = st.s2z = st.dt_bl = st.dt_pos = 0.0;
  st.i_off = seg_i0;

#define DDVR_WALK(SEG, INS, EM)                                                          \
  adjoint_ray<MASK, CELLS, SEG, INS, EM, kTfTexture, false, false, DET>(                   \
      V, TFA, G.dt32, r, S, sd, tape, tf_slot, d_volume, d_cells, st)
#define DDVR_WALK_SEG(INS, EM)                  \
  if (mode == kSegP3) DDVR_WALK(kSegP3, INS, EM); \
  else if (mode == kSegP7) DDVR_WALK(kSegP7, INS, EM); \
  else DDVR_WALK(kSegGen, INS, EM);
  // stored mode (tape) and the analytic TFs take the general variant
#define DDVR_WALK_GEN(KIND, TP)                                                           \
  adjoint_ray<MASK, CELLS, kSegGen, false, true, KIND, TP, false, DET>(                    \
      V, TFA, G.dt32, r, S, sd, tape, tf_slot, d_volume, d_cells, st)
#define DDVR_WALK_AFF(SEG, INS)                                                            \
  adjoint_ray<MASK, CELLS, SEG, INS, false, kTfTexture, false, true, DET>(                  \
      V, TFA, G.dt32, r, S, sd, tape, tf_slot, d_volume, d_cells, st,                       \
      __uint_as_float(s_info[3]), __uint_as_float(s_info[4]))
#define DDVR_WALK_SEG_AFF(INS)                  \
  if (mode == kSegP3) DDVR_WALK_AFF(kSegP3, INS); \
  else DDVR_WALK_AFF(kSegP7, INS);
  if (kBitsKernel && bits) {
    const float abs_k = sd.w * (float)exp(-S) * G.dt32 * TFA.fR * __uint_as_float(s_info[4]);
    if (warp_inside && DDVR_RUN_WALK)
      abs_runs_walk<DET>(V, r, abs_k, bits, bits_off, d_cells, &walk_skip);
    else if (warp_inside)
      abs_bits_walk<true, DET>(V, r, abs_k, bits, bits_off, d_cells, st, &walk_skip);
    else abs_bits_walk<false, DET>(V, r, abs_k, bits, bits_off, d_cells, st, &walk_skip);
  } else if (ROLE == 1 && aff_walk) {
    if (warp_inside) { DDVR_WALK_SEG_AFF(true) } else { DDVR_WALK_SEG_AFF(false) }
  } else if (ROLE == 1) {
    if (warp_inside) { DDVR_WALK_SEG(true, false) } else { DDVR_WALK_SEG(false, false) }
  } else if (G.tape) {
    if (TFA.kind == kTfPiecewise) DDVR_WALK_GEN(kTfPiecewise, true);
    else if (TFA.kind == kTfGaussian) DDVR_WALK_GEN(kTfGaussian, true);
    else DDVR_WALK_GEN(kTfTexture, true);
  } else if (TFA.kind == kTfPiecewise) {
    DDVR_WALK_GEN(kTfPiecewise, false);
  } else if (TFA.kind == kTfGaussian) {
    DDVR_WALK_GEN(kTfGaussian, false);
  } else if (warp_inside) {
    if (emit) { DDVR_WALK_SEG(true, true) }
    else if (!kTf) { DDVR_WALK_SEG(true, kTf) }   // kTf: never taken (EMIT=true re-use)
  } else {
    if (emit) { DDVR_WALK_SEG(false, true) }
    else if (!kTf) { DDVR_WALK_SEG(false, kTf) }
  }
#undef DDVR_WALK_SEG_AFF
#undef DDVR_WALK_AFF
#undef DDVR_WALK_SEG
#undef DDVR_WALK_GEN
#undef DDVR_WALK

  if (FUSED && G.stats) {   // measurement only: one atomic per warp and counter
    const unsigned long long c[4] = {
        warp_sum((unsigned long long)(valid ? r.n : 0)), warp_sum((unsigned long long)march_skip),
        warp_sum((unsigned long long)walk_skip),
        warp_sum((unsigned long long)(valid && seg == 0 ? 1 : 0))};
    if ((threadIdx.x & 31) == 0)
      for (int k = 0; k < 4; ++k)
        if (c[k]) atomicAdd(G.stats + k, c[k]);
  }
#ifdef DDVR_WALK_NORED
  if (!kTf && st.tfp0 == 12345.f && d_cells) d_cells[0] = st.tfp0;
#endif
  // ---- flush per-ray accumulators ----
  DDVR_REQUIRE(!(kVol && CELLS && st.run_cell != kNoRun) || cell_ok(V, st.run_cell));
  if (kVol && CELLS && st.run_cell != kNoRun)
    flush_record<DET>(V, d_cells, st.run_cell, st.acc8);
  else if (kVol && st.run_cell != kNoRun)
    flush_cell<CELLS>(d_volume, d_cells, st.run_cell, st.run_base, st.run_ox, st.run_oy,
                      st.run_oz, st.acc8);
  if (kTf && TFA.kind != kTfGaussian && st.tf_run != kNoRun)
    tf_flush_run(tf_slot, TFA.count, TFA.kind, st.tf_run, st.tfa0, st.tfa1, st.tfp0, st.tfp1);
  if (kPos) {
    double cam0 = 0.0, cam1 = 0.0, stp = 0.0;
    if (valid && r.n > 0) {
      if (kStep) stp = st.dt_bl + st.dt_pos;
      if (kCam) {
        // world-space sums: x_hat = scale * grid-space gradient (chain of g = (x-bmin)*scale)
        const double xo_h[3] = {st.s1x * V.scale[0], st.s1y * V.scale[1], st.s1z * V.scale[2]};
        const double w_h[3] = {st.s2x * V.scale[0], st.s2y * V.scale[1], st.s2z * V.scale[2]};
        // entry point xo = o + tn*w moves with the camera (renderer.py:629-639)
        const double sdot = r.w[0] * xo_h[0] + r.w[1] * xo_h[1] + r.w[2] * xo_h[2];
        const bool need = !r.clamped && !r.miss;
        double o_h[3], w_tot[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const bool sel = need && r.axis == k;
          o_h[k] = xo_h[k] - (sel ? sdot / r.w[k] : 0.0);
          w_tot[k] = w_h[k] + r.tn * xo_h[k] - (sel ? sdot * r.tn / r.w[k] : 0.0);
        }
        // d(direction)/d(lon,lat) at this pixel (field.py:253-271), per degree
        double dj[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          double draw[3];
#pragma unroll
          for (int k = 0; k < 3; ++k)
            draw[k] = F.df[k][j] + F.dr[k][j] * r.su + F.du[k][j] * r.sv;
          const double proj = r.w[0] * draw[0] + r.w[1] * draw[1] + r.w[2] * draw[2];
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < 3; ++k)
            acc += w_tot[k] * (draw[k] - r.w[k] * proj) / r.dn + o_h[k] * F.jo[k][j];
          dj[j] = acc;
        }
        cam0 = dj[0];
        cam1 = dj[1];
      }
    }
    cam0 = warp_sum(cam0);
    cam1 = warp_sum(cam1);
    stp = warp_sum(stp);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { s_red[warp][0] = cam0; s_red[warp][1] = cam1; s_red[warp][2] = stp; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double t0 = 0, t1 = 0, t2 = 0;
      for (int k = 0; k < kWarps; ++k) { t0 += s_red[k][0]; t1 += s_red[k][1]; t2 += s_red[k][2]; }
      if (G.partials) {   // deterministic mode: reduced in CTA order afterwards
        // (the logical CTA index tile + tiles * view, whatever order the CTAs ran in)
        double* q = G.partials + 3 * (tile_x + gridDim.x * (tile_y + gridDim.y * (size_t)view));
        q[0] = t0; q[1] = t1; q[2] = t2;
      } else {
        if (kCam) { atomicAdd(d_camera + 2 * view, t0); atomicAdd(d_camera + 2 * view + 1, t1); }
        if (kStep) atomicAdd(d_dt, t2);
      }
    }
  }
}


// ---------------------------------------------------------------------------
// The band-tape step as two kernels (G.ray_k set): the march is gather-latency
// bound and the walk is issue bound, and their union in one thread held the
// fused kernel to 64 registers (4 CTAs/SM).  Apart they run at their own
// occupancy; the march hands each ray's walk weight abs_k = seed_a T_n dt R b
// to the walk through (V, rows, W) floats (4 B per ray).
// ---------------------------------------------------------------------------

#ifndef DDVR_BAND_MARCH_MINB
#define DDVR_BAND_MARCH_MINB 4
#endif
#ifndef DDVR_BAND_WALK_MINB
#define DDVR_BAND_WALK_MINB 4
#endif

// shared prologue of the two kernels: TF table, class test, frame, this lane's ray
struct BandRay {
  Ray r;
  bool valid, warp_inside;
  size_t pix;
  unsigned bits_off;
  int mode;
};

__device__ __forceinline__ bool band_prologue(const VolArgs& V, const TfArgs& TFA,
                                              const Geometry& G, Frame& F, unsigned* s_info,
                                              BandRay& b) {
  if (threadIdx.x < 5) s_info[threadIdx.x] = 0u;
  __syncthreads();
  load_tf(TFA, s_info);
  __syncthreads();
  b.mode = seg_mode(G.dt32, s_info[0]);
  if (!band_class(TFA, G, s_info, b.mode)) return false;   // CTA-uniform
  if (threadIdx.x == 0) make_frame(G.cams[blockIdx.z], G.W, G.H, F);
  __syncthreads();
  int px, py;
  pixel_of(G, px, py);
  b.valid = px < G.W && py < G.row1;
  b.r.n = 0;
  b.r.all_inside = true;
  b.pix = 0;
  if (b.valid) {
    setup_ray(F, V, G.dt, G.W, G.H, px, py, b.r);
    b.pix = ((size_t)blockIdx.z * (G.row1 - G.row0) + (py - G.row0)) * G.W + px;
  }
  b.warp_inside = __all_sync(0xffffffffu, b.r.all_inside);
  b.bits_off = ((blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) * kWarps +
                (threadIdx.x >> 5)) * 32u * (unsigned)G.bits_words + (threadIdx.x & 31);
  return true;
}

// forward march (renderer.py:306-357) with the band tape + L1 seed (objectives.py:38-54)
// and the walk weight of the closed-form absorption adjoint (see adjoint_ray)
template <int kUnused = 0>   // (a template: instantiated only where launched)
__global__ void __launch_bounds__(kThreads, DDVR_BAND_MARCH_MINB)
    dvr_band_march_kernel(VolArgs V, TfArgs TFA, Geometry G, FusedArgs Fu) {
  __shared__ Frame F;
  __shared__ unsigned s_info[5];
  BandRay b;
  if (!band_prologue(V, TFA, G, F, s_info, b)) return;
  int march_skip = 0;
  double loss_part = 0.0;
  double S = 0.0;
  if (b.valid) {
    float4 rgba;
    const float aa = __uint_as_float(s_info[3]), ab = __uint_as_float(s_info[4]);
#define DDVR_BAND_MARCH(SEG, INS)                                                            \
  march_ray<false, true, false, SEG, INS, false, kTfTexture, true, true>(                     \
      V, TFA, G.dt32, b.r, nullptr, rgba, S, aa, ab, G.bits, b.bits_off, &march_skip)
    if (b.warp_inside) {
      if (b.mode == kSegP3) DDVR_BAND_MARCH(kSegP3, true); else DDVR_BAND_MARCH(kSegP7, true);
    } else {
      if (b.mode == kSegP3) DDVR_BAND_MARCH(kSegP3, false); else DDVR_BAND_MARCH(kSegP7, false);
    }
#undef DDVR_BAND_MARCH
    const float4 ref = reinterpret_cast<const float4*>(Fu.refs)[b.pix];
    const float dx = rgba.x - ref.x, dy = rgba.y - ref.y, dz = rgba.z - ref.z,
                dw = rgba.w - ref.w;
    const float sw = dw > 0.f ? Fu.inv_count : (dw < 0.f ? -Fu.inv_count : 0.f);
    loss_part = fabs((double)dx) + fabs((double)dy) + fabs((double)dz) + fabs((double)dw);
    if (Fu.image_out) reinterpret_cast<float4*>(Fu.image_out)[b.pix] = rgba;
    if (Fu.depth_out) Fu.depth_out[b.pix] = (float)S;
    // d_hat per set band bit: seed_a T_n dt R b (the walk of adjoint_ray<..., AFF>)
    G.ray_k[b.pix] = sw * (float)exp(-S) * G.dt32 * TFA.fR * __uint_as_float(s_info[4]);
  }
  loss_part = warp_sum(loss_part);
  if ((threadIdx.x & 31) == 0 && loss_part != 0.0) atomicAdd(Fu.loss, loss_part * Fu.inv_count_d);
  if (G.stats) {
    const unsigned long long c[3] = {warp_sum((unsigned long long)(b.valid ? b.r.n : 0)),
                                     warp_sum((unsigned long long)march_skip),
                                     warp_sum((unsigned long long)(b.valid ? 1 : 0))};
    if ((threadIdx.x & 31) == 0) {
      if (c[0]) atomicAdd(G.stats + 0, c[0]);
      if (c[1]) atomicAdd(G.stats + 1, c[1]);
      if (c[2]) atomicAdd(G.stats + 3, c[2]);
    }
  }
}

// the affine absorption walk from the band tape (abs_bits_walk) + the cell-run flushes
template <bool DET = false>
__global__ void __launch_bounds__(kThreads, DDVR_BAND_WALK_MINB)
    dvr_band_walk_kernel(VolArgs V, TfArgs TFA, Geometry G, float* __restrict__ d_cells) {
  __shared__ Frame F;
  __shared__ unsigned s_info[5];
  BandRay b;
  if (!band_prologue(V, TFA, G, F, s_info, b)) return;
  AdjState st;
  st.run_cell = kNoRun;
  st.tfp0 = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) st.acc8[k] = 0.f;
  int walk_skip = 0;
  if (b.valid) {
    const float abs_k = G.ray_k[b.pix];
    if (b.warp_inside && DDVR_RUN_WALK)
      abs_runs_walk<DET>(V, b.r, abs_k, G.bits, b.bits_off, d_cells, &walk_skip);
    else if (b.warp_inside)
      abs_bits_walk<true, DET>(V, b.r, abs_k, G.bits, b.bits_off, d_cells, st, &walk_skip);
    else abs_bits_walk<false, DET>(V, b.r, abs_k, G.bits, b.bits_off, d_cells, st, &walk_skip);
    DDVR_REQUIRE(st.run_cell == kNoRun || cell_ok(V, st.run_cell));
    if (st.run_cell != kNoRun && st.acc8[0] != 0.f)
      flush_record<DET>(V, d_cells, st.run_cell, st.acc8);
#ifdef DDVR_WALK_NORED
    if (st.tfp0 == 12345.f) G.ray_k[b.pix] = st.tfp0;
#endif
  }
  if (G.stats) {
    const unsigned long long c = warp_sum((unsigned long long)walk_skip);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(G.stats + 2, c);
  }
}

}  // namespace
