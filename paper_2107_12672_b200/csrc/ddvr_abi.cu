// ddvr_abi.cu -- the C ABI of include/ddvr.h: validation, launches, small kernels.
// (Device code: ddvr_device.cuh; kernel instantiations: ddvr_fwd.cu, ddvr_adj_g*.cu.)
#include <algorithm>
#include <cstdlib>

#include "ddvr_device.cuh"

namespace {
using namespace ddvr_impl;

thread_local char g_err[1024] = "";
std::atomic<int64_t> g_launches{0};

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(DDVR_CUDA_ERROR, "%s: %s", what, cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return DDVR_OK;
}

// ---------------------------------------------------------------------------
// cell-record layout: pack (volume -> cells) and fold (cell gradients -> voxels)
// ---------------------------------------------------------------------------

// (x, y, z) of flat voxel index id (z fastest) with 32-bit division below 2^31 voxels
__device__ __forceinline__ void vox_coords(long long id, long long n, int Y, int Z, int& x, int& y,
                                           int& z) {
  if (n < (1ll << 31)) {
    const unsigned u = (unsigned)id, yz = (unsigned)Y * (unsigned)Z;
    x = (int)(u / yz);
    const unsigned r = u - (unsigned)x * yz;
    y = (int)(r / (unsigned)Z);
    z = (int)(r - (unsigned)y * (unsigned)Z);
  } else {
    z = (int)(id % Z);
    const long long xy = id / Z;
    y = (int)(xy % Y);
    x = (int)(xy / Y);
  }
}

// Padded record of cell (i,j,k), i in [-1, X-1] (storage index i+1): the
// polynomial coefficients (corners_to_poly) of its 8 edge-clamped corners
//   v[b] = vol[clamp(i+bx, 0, X-1)][clamp(j+by, 0, Y-1)][clamp(k+bz, 0, Z-1)],
//   b = bx | by << 1 | bz << 2 (the corner order of field.py:318-322).
__global__ void __launch_bounds__(256) pack_cells_kernel(VolArgs V, float* __restrict__ cells,
                                                       long long ncells) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= ncells) return;
  int i, j, k;
  vox_coords(id, ncells, V.CY, V.CZ, i, j, k);
  --i; --j; --k;
  const int i0 = max(i, 0), j0 = max(j, 0), k0 = max(k, 0);
  const int i1 = min(i + 1, V.X - 1), j1 = min(j + 1, V.Y - 1), k1 = min(k + 1, V.Z - 1);
  const float* p = V.data;
  auto at = [&](int a, int b, int c) { return __ldg(p + ((size_t)a * V.Y + b) * V.Z + c); };
  const float v[8] = {at(i0, j0, k0), at(i1, j0, k0), at(i0, j1, k0), at(i1, j1, k0),
                      at(i0, j0, k1), at(i1, j0, k1), at(i0, j1, k1), at(i1, j1, k1)};
  float k8[8];
  corners_to_poly(v, k8);
  float4* q = reinterpret_cast<float4*>(cells + 8 * id);
  q[0] = make_float4(k8[0], k8[1], k8[2], k8[3]);
  q[1] = make_float4(k8[4], k8[5], k8[6], k8[7]);
}

// gradient of corner b of a record from the record's moment gradient m
// (d rho / d v_b = sum_k L[k][b] phi_k, so g_b = sum_k L[k][b] m_k)
__device__ __forceinline__ float corner_from_moments(const float4& a, const float4& h, int b) {
  const float sx = (b & 1) ? 1.f : -1.f, sy = (b & 2) ? 1.f : -1.f, sz = (b & 4) ? 1.f : -1.f;
  // (moment order {1, ux, uy, ux uy, uz, ux uz, uy uz, ux uy uz}, corners_to_poly)
  float g = a.x * 0.125f;
  g = fmaf(0.25f * sx, a.y, g);
  g = fmaf(0.25f * sy, a.z, g);
  g = fmaf(0.5f * sx * sy, a.w, g);
  g = fmaf(0.25f * sz, h.x, g);
  g = fmaf(0.5f * sx * sz, h.y, g);
  g = fmaf(0.5f * sy * sz, h.z, g);
  return fmaf(sx * sy * sz, h.w, g);
}

// one voxel of the fold (any position, either moment format)
__device__ void fold_voxel(const VolArgs& V, const unsigned long long* c64, double inv,
                           const float* __restrict__ d_cells, float* __restrict__ d_volume,
                           long long id, int x, int y, int z) {
  // per axis, the (storage cell index, corner bit) pairs whose clamped corner is this voxel
  int ci[3][4], cb[3][4], cn[3];
  const int dims[3] = {V.X, V.Y, V.Z};
  const int pos[3] = {x, y, z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int n = 0;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int d = -2; d <= 1; ++d) {
        const int i = pos[a] + d;                    // padded cell index in [-1, dim-1]
        if (i < -1 || i > dims[a] - 1) continue;
        const int corner = min(max(i + b, 0), dims[a] - 1);
        if (corner == pos[a] && n < 4) { ci[a][n] = i + 1; cb[a][n] = b; ++n; }
      }
    cn[a] = n;
  }
  float s = 0.f;
  for (int a = 0; a < cn[0]; ++a)
    for (int b = 0; b < cn[1]; ++b)
      for (int c = 0; c < cn[2]; ++c) {
        const size_t cell = ((size_t)ci[0][a] * V.CY + ci[1][b]) * V.CZ + ci[2][c];
        const int corner = cb[0][a] | cb[1][b] << 1 | cb[2][c] << 2;
        if (c64) {
          const long long* q = reinterpret_cast<const long long*>(c64 + 8 * cell);
          const float4 m0 = make_float4((float)(q[0] * inv), (float)(q[1] * inv),
                                        (float)(q[2] * inv), (float)(q[3] * inv));
          const float4 m1 = make_float4((float)(q[4] * inv), (float)(q[5] * inv),
                                        (float)(q[6] * inv), (float)(q[7] * inv));
          s += corner_from_moments(m0, m1, corner);
        } else {
          const float4* m = reinterpret_cast<const float4*>(d_cells + 8 * cell);
          s += corner_from_moments(m[0], m[1], corner);
        }
      }
  d_volume[id] += s;
}

// The fold split by position: interior voxels (1 <= coordinate <= dim-2 on every axis)
// read exactly the 8 records of the 2x2x2 block ending at their own record, corner b from
// storage (x+1, y+1, z+1) - b, no clamping; the boundary shell takes fold_voxel's
// clamped pair lists.  Separate index spaces, so no warp mixes the two paths (with one
// thread per voxel every warp of a 64-voxel row held an edge voxel and ran both).
__global__ void __launch_bounds__(256) fold_interior_kernel(VolArgs V,
                                                          const float* __restrict__ d_cells,
                                                          float* __restrict__ d_volume,
                                                          long long n) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= n) return;
  int x, y, z;
  vox_coords(id, n, V.Y - 2, V.Z - 2, x, y, z);
  ++x; ++y; ++z;
  const float* base = d_cells + 8 * (((long long)(x + 1) * V.CY + (y + 1)) * V.CZ + (z + 1));
  const long long sx = 8ll * V.CY * V.CZ, sy = 8ll * V.CZ;
  float s = 0.f;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const float4* m = reinterpret_cast<const float4*>(
        base - ((b & 1) ? sx : 0) - ((b & 2) ? sy : 0) - ((b & 4) ? 8 : 0));
    s += corner_from_moments(__ldg(m), __ldg(m + 1), b);
  }
  d_volume[((long long)x * V.Y + y) * V.Z + z] += s;
}

// shell voxel k of an X x Y x Z grid (faces x = 0, X-1; then y = 0, Y-1 without them;
// then z = 0, Z-1 without either): its coordinates
__device__ __forceinline__ void shell_coords(long long k, int X, int Y, int Z, int& x, int& y,
                                             int& z) {
  const long long fx = (long long)Y * Z;                        // one x face
  const long long fy = (long long)max(X - 2, 0) * Z;            // one y face, x interior
  const long long fz = (long long)max(X - 2, 0) * max(Y - 2, 0);   // one z face
  const int nx = X > 1 ? 2 : 1, ny = Y > 1 ? 2 : 1;
  if (k < nx * fx) {
    const int f = (int)(k / fx);
    const long long r = k - f * fx;
    x = f ? X - 1 : 0; y = (int)(r / Z); z = (int)(r - (long long)y * Z);
    return;
  }
  k -= nx * fx;
  if (k < ny * fy) {
    const int f = (int)(k / fy);
    const long long r = k - f * fy;
    y = f ? Y - 1 : 0; x = 1 + (int)(r / Z); z = (int)(r - (long long)(x - 1) * Z);
    return;
  }
  k -= ny * fy;
  const int f = (int)(k / fz);
  const long long r = k - f * fz;
  z = f ? Z - 1 : 0; x = 1 + (int)(r / max(Y - 2, 1)); y = 1 + (int)(r - (long long)(x - 1) * max(Y - 2, 1));
}

// A boundary voxel (dims >= 2 on every axis): per axis the pairs (storage pos, corner 1)
// and (pos + 1, corner 0) of an interior voxel, plus (pos, 0) on the low face and
// (pos + 1, 1) on the high face -- the clamped corners of the padded cells (the pair
// lists fold_voxel builds) as 3 x 3 x 3 predicated terms in registers
__global__ void __launch_bounds__(256) fold_shell_kernel(VolArgs V,
                                                       const float* __restrict__ d_cells,
                                                       float* __restrict__ d_volume,
                                                       long long n) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int p[3];
  shell_coords(k, V.X, V.Y, V.Z, p[0], p[1], p[2]);
  const int dims[3] = {V.X, V.Y, V.Z};
  int sa[3][3], ba[3][3];
  bool va[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const bool lo = p[a] == 0, hi = p[a] == dims[a] - 1;
    sa[a][0] = p[a];     ba[a][0] = 1; va[a][0] = true;
    sa[a][1] = p[a] + 1; ba[a][1] = 0; va[a][1] = true;
    sa[a][2] = lo ? p[a] : p[a] + 1; ba[a][2] = lo ? 0 : 1; va[a][2] = lo || hi;
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        if (!(va[0][i] && va[1][j] && va[2][l])) continue;
        const long long cell = ((long long)sa[0][i] * V.CY + sa[1][j]) * V.CZ + sa[2][l];
        const float4* m = reinterpret_cast<const float4*>(d_cells + 8 * cell);
        s += corner_from_moments(__ldg(m), __ldg(m + 1), ba[0][i] | ba[1][j] << 1 | ba[2][l] << 2);
      }
  d_volume[((long long)p[0] * V.Y + p[1]) * V.Z + p[2]] += s;
}

// d_volume[x,y,z] += the gradient of every record corner that pack_cells_kernel
// filled from voxel (x,y,z) (its exact transpose, padding included); the
// adjoint leaves each record's moment gradient, mapped back per corner here
// (one 32-byte sector per contributing record, as the corner form read)
__global__ void __launch_bounds__(256) fold_cells_kernel(VolArgs V,
                                                       const float* __restrict__ d_cells,
                                                       float* __restrict__ d_volume,
                                                       long long nvox) {
  // the deterministic mode's int64 fixed-point moments (V.cells64 relative to cell 0)
  const unsigned long long* c64 =
      V.cells64 ? V.cells64 - (V.cell0 - V.cells) : nullptr;
  const double inv = c64 ? 1.0 / __ldg(V.det_scale) : 0.0;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nvox) return;
  int x, y, z;
  vox_coords(id, nvox, V.Y, V.Z, x, y, z);
  fold_voxel(V, c64, inv, d_cells, d_volume, id, x, y, z);
}

// ---------------------------------------------------------------------------
// ray setup (parity helper) and fused L1 loss
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kThreads) ray_setup_kernel(VolArgs V, Geometry G,
                                                           double* __restrict__ tn_tf,
                                                           int32_t* __restrict__ n_steps,
                                                           int32_t* __restrict__ flags) {
  __shared__ Frame F;
  const int view = blockIdx.z;
  if (threadIdx.x == 0) make_frame(G.cams[view], G.W, G.H, F);
  __syncthreads();
  int px, py;
  pixel_of(G, px, py);
  if (px >= G.W || py >= G.row1) return;
  Ray r;
  setup_ray(F, V, G.dt, G.W, G.H, px, py, r);
  const size_t pix = ((size_t)view * (G.row1 - G.row0) + (py - G.row0)) * G.W + px;
  n_steps[pix] = r.n;
  if (tn_tf) { tn_tf[2 * pix] = r.tn; tn_tf[2 * pix + 1] = r.tf; }
  if (flags) flags[pix] = r.axis | (r.clamped ? 4 : 0) | (r.miss ? 8 : 0);
}

__global__ void __launch_bounds__(256) l1_loss_kernel(const float* __restrict__ x,
                                                    const float* __restrict__ y, int64_t n,
                                                    float inv_count, double inv_count_d,
                                                    float* __restrict__ seed,
                                                    double* __restrict__ loss) {
  __shared__ double s_part[8];
  double part = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float dlt = x[i] - y[i];
    part += fabs((double)dlt);
    if (seed) seed[i] = dlt > 0.f ? inv_count : (dlt < 0.f ? -inv_count : 0.f);
  }
  part = warp_sum(part);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0 && loss) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += s_part[k];
    atomicAdd(loss, t * inv_count_d);
  }
}

// opacity_entropy (objectives.py:95-126), per image v of n pixels:
// S = sum a, S+ = sum_{a>0} a, T = sum_{a>0} a log2 a (fp64, alpha channel);
// with p = a / S, F = sum_{p>0} p log2 p = T / S - log2(S) S+ / S, H = -F / log2 n.
__global__ void __launch_bounds__(256) entropy_sums_kernel(const float4* __restrict__ img,
                                                          int64_t n, double* __restrict__ out) {
  __shared__ double part[8][3];
  const float4* im = img + (size_t)blockIdx.y * n;
  double s = 0.0, sp = 0.0, t = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double a = (double)im[i].w;
    s += a;
    if (a > 0.0) { sp += a; t += a * log2(a); }
  }
  s = warp_sum(s); sp = warp_sum(sp); t = warp_sum(t);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { part[w][0] = s; part[w][1] = sp; part[w][2] = t; }
  __syncthreads();
  if (threadIdx.x < 3) {
    double acc = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) acc += part[k][threadIdx.x];
    atomicAdd(out + 4 * blockIdx.y + 1 + threadIdx.x, acc);
  }
}

// H per image and the alpha-channel seed dH/da_k = -(log2 p_k - F) / (S log2 n),
// non-finite -> +-1e6 and clipped to [-1e6, 1e6] (objectives.py:118-125); rgb seed 0.
// The degenerate case (S <= 0 or n < 2) gives H = 0 and a zero seed.
__global__ void __launch_bounds__(256) entropy_seed_kernel(const float4* __restrict__ img,
                                                          int64_t n, double* __restrict__ out,
                                                          float4* __restrict__ seed) {
  const int v = blockIdx.y;
  const double S = out[4 * v + 1], Sp = out[4 * v + 2], T = out[4 * v + 3];
  const bool degenerate = !(S > 0.0) || n < 2;
  const double log_n = log2((double)n);
  const double F = degenerate ? 0.0 : T / S - log2(S) * Sp / S;
  if (blockIdx.x == 0 && threadIdx.x == 0) out[4 * v] = degenerate ? 0.0 : -F / log_n;
  if (!seed) return;
  const float4* im = img + (size_t)v * n;
  float4* sd = seed + (size_t)v * n;
  constexpr double kBound = 1e6;   // _ENTROPY_GRAD_BOUND, objectives.py:20
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double g = 0.0;
    if (!degenerate) {
      const double p = (double)im[i].w / S;
      // log2 of p <= 0 is -inf or nan: both map to +1e6 in the reference
      g = p > 0.0 ? fmin(fmax(-(log2(p) - F) / (S * log_n), -kBound), kBound) : kBound;
    }
    sd[i] = make_float4(0.f, 0.f, 0.f, (float)g);
  }
}

// ---------------------------------------------------------------------------
// host-side validation and launch
// ---------------------------------------------------------------------------

// padded cell grid: cells -1 .. dim-1 on every axis
long long cell_count(const int32_t dims[3]) {
  return (long long)(dims[0] + 1) * (dims[1] + 1) * (dims[2] + 1);
}

int make_vol(const ddvr_volume* vol, VolArgs& V, bool need_data = true) {
  if (!vol) return set_error(DDVR_INVALID_PARAMETER, "volume descriptor is NULL");
  for (int k = 0; k < 3; ++k) {
    if (vol->dims[k] < 1)
      return set_error(DDVR_INVALID_PARAMETER, "volume values must be a non-empty 3D array");
    if (!(vol->box_max[k] > vol->box_min[k]) || !std::isfinite(vol->box_min[k]) ||
        !std::isfinite(vol->box_max[k]))
      return set_error(DDVR_INVALID_PARAMETER,
                       "world box must have positive extent on each axis");
  }
  const long long nvox = (long long)vol->dims[0] * vol->dims[1] * vol->dims[2];
  if (nvox > 0x7fffffffLL)
    return set_error(DDVR_UNSUPPORTED, "volume has more than 2^31 voxels");
  // cell indices are int32 (relative to cell (0,0,0)): the padded grid must fit
  if (vol->cells && (long long)(vol->dims[0] + 1) * (vol->dims[1] + 1) * (vol->dims[2] + 1) >
                        0x7fffffffLL)
    return set_error(DDVR_UNSUPPORTED, "cell-record grid has more than 2^31 cells");
  if (need_data && !vol->data) return set_error(DDVR_INVALID_INPUT, "volume data pointer is NULL");
  if (vol->cells && ((uintptr_t)vol->cells & 31) != 0)
    return set_error(DDVR_INVALID_INPUT, "cell records must be 32-byte aligned");
  V.data = vol->data;
  V.cells = vol->cells;
  V.occ = nullptr;   // set by run_adjoint for the fused band-tape step
  V.cells64 = nullptr;   // set by run_adjoint in the deterministic volume mode
  V.det_scale = nullptr;
  V.NBy = (vol->dims[1] + 8) >> 3; V.NBz = (vol->dims[2] + 8) >> 3;
  V.X = vol->dims[0]; V.Y = vol->dims[1]; V.Z = vol->dims[2];
  V.YZ = V.Y * V.Z;
  V.CY = V.Y + 1; V.CZ = V.Z + 1;
  V.cell0 = V.cells ? V.cells + 8 * (((long long)V.CY + 1) * V.CZ + 1) : nullptr;
  V.Xm2 = V.X >= 2 ? V.X - 2 : 0; V.Ym2 = V.Y >= 2 ? V.Y - 2 : 0; V.Zm2 = V.Z >= 2 ? V.Z - 2 : 0;
  V.X1 = V.X - 1; V.Y1 = V.Y - 1; V.Z1 = V.Z - 1;
  V.tX = V.X > 1 ? 1.f : 0.f; V.tY = V.Y > 1 ? 1.f : 0.f; V.tZ = V.Z > 1 ? 1.f : 0.f;
  // inside test in grid units.  Every sample of a march lies in [tn, tf) of the
  // exact slab, so the reference's 1e-9*extent tolerance (field.py:293) only has
  // to absorb rounding of the fixed-point entry point: 1e-6 voxel of slack.
  const double tol = 1e-6;
  for (int k = 0; k < 3; ++k) {
    V.lo[k] = (long long)llrint((-0.5 - tol) * kFix);
    V.hi[k] = (long long)llrint(((double)vol->dims[k] - 0.5 + tol) * kFix);
    V.top[k] = (long long)(vol->dims[k] - 1) << 32;
    V.bmin[k] = vol->box_min[k];
    V.bmax[k] = vol->box_max[k];
    V.scale[k] = (double)vol->dims[k] / (vol->box_max[k] - vol->box_min[k]);
  }
  return DDVR_OK;
}

int make_tf(const ddvr_tf* tf, TfArgs& A, size_t& smem_per_table) {
  if (!tf) return set_error(DDVR_INVALID_PARAMETER, "transfer function descriptor is NULL");
  if (tf->kind != DDVR_TF_TEXTURE && tf->kind != DDVR_TF_PIECEWISE &&
      tf->kind != DDVR_TF_GAUSSIAN)
    return set_error(DDVR_UNSUPPORTED, "transfer-function kind %d is not built", tf->kind);
  const int stride = tf->kind == DDVR_TF_TEXTURE ? 4 : tf->kind == DDVR_TF_PIECEWISE ? 5 : 6;
  if (tf->count < 1)
    return set_error(DDVR_INVALID_PARAMETER,
                     "transfer function must have shape (R, %d), R >= 1", stride);
  if (!tf->params) return set_error(DDVR_INVALID_INPUT, "transfer function pointer is NULL");
  if (((uintptr_t)tf->params & (tf->kind == DDVR_TF_TEXTURE ? 15 : 3)) != 0)
    return set_error(DDVR_INVALID_INPUT, "transfer function parameters are misaligned");
  const size_t n = (size_t)tf->count;
  // shared layouts (see g_smem / pl_eval / gauss_eval), gradient rows included:
  //   texture   2(n+1) pair float4 + 4n gradient floats + (n+1) tau-pair float2
  //   piecewise 2n float4 + n pos floats (pad to 9n floats) + 5n gradient floats
  //   gaussian  2n float4 + 6n gradient floats
  smem_per_table = tf->kind == DDVR_TF_TEXTURE ? (14 * n + 10) * sizeof(float)
                   : tf->kind == DDVR_TF_PIECEWISE ? (9 * n + 5 * n) * sizeof(float)
                                                   : (8 * n + 6 * n) * sizeof(float);
  A.stride = stride;
  if (smem_per_table > (size_t)kMaxTfBytes)
    return set_error(DDVR_UNSUPPORTED, "transfer function resolution %d exceeds %d texels",
                     tf->count, kMaxTfBytes / 56);
  A.params = tf->params;
  A.slots = nullptr;
  A.nslot = 0;
  A.slot_floats = tf_slot_floats(tf->kind, tf->count);
  A.kind = tf->kind;
  A.count = tf->count;
  A.fR = (float)tf->count;
  A.fR1 = (float)(tf->count - 1);
  A.Rm2 = tf->count >= 2 ? tf->count - 2 : 0;
  return DDVR_OK;
}

int make_geo(const ddvr_camera* cams, int n_views, const ddvr_params* p, Geometry& G) {
  if (!p) return set_error(DDVR_INVALID_PARAMETER, "params is NULL");
  if (!(p->dt > 0.0) || !std::isfinite(p->dt))
    return set_error(DDVR_INVALID_PARAMETER, "stepsize must be positive");
  if (p->width < 1 || p->height < 1)
    return set_error(DDVR_INVALID_PARAMETER, "image size must be at least 1x1");
  if (n_views < 0 || n_views > 65535)
    return set_error(DDVR_INVALID_PARAMETER, "view count %d out of range", n_views);
  if (n_views > 0 && !cams) return set_error(DDVR_INVALID_INPUT, "camera array is NULL");
  G.cams = cams;
  G.W = p->width;
  G.H = p->height;
  G.row0 = p->row0;
  G.row1 = p->row1 <= 0 ? p->height : p->row1;
  if (G.row0 < 0 || G.row0 > G.row1 || G.row1 > G.H)
    return set_error(DDVR_INVALID_PARAMETER, "row band [%d, %d) outside image height %d", G.row0,
                     G.row1, G.H);
  G.dt = p->dt;
  G.dt32 = (float)p->dt;
  G.tape = p->tape;
  G.tape_stride = p->tape_stride;
  G.partials = nullptr;
  G.bits = nullptr;
  G.bits_words = 0;
  G.stats = reinterpret_cast<unsigned long long*>(p->stats);
  G.ray_k = nullptr;
  G.vgroup = 1;
  if (G.tape && G.tape_stride < 0)
    return set_error(DDVR_INVALID_PARAMETER, "negative tape stride");
  return DDVR_OK;
}

dim3 grid_of(const Geometry& G, int n_views) {
  return dim3((G.W + kTile - 1) / kTile, (G.row1 - G.row0 + kTile - 1) / kTile, n_views);
}

// ---------------------------------------------------------------------------
// steps either side of the path: priors, Adam, upsample
// ---------------------------------------------------------------------------

__device__ __forceinline__ void block_add_double(double part, double* out) {
  __shared__ double s_part[32];
  part = warp_sum(part);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0 && out) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += s_part[k];
    atomicAdd(out, t);
  }
}

// smoothness_prior_volume (objectives.py:72-92): P = sum of squared forward
// differences along each axis / their count; grad[x] is gathered from the
// (up to) six differences touching voxel x -- no atomics.
__global__ void __launch_bounds__(256) prior_volume_kernel(const float* __restrict__ v, int X,
                                                         int Y, int Z, double scale,
                                                         float* __restrict__ grad,
                                                         double* __restrict__ value) {
  const long long n = (long long)X * Y * Z;
  const long long stride = (long long)gridDim.x * blockDim.x;
  double part = 0.0;
  const long long sx = (long long)Y * Z, sy = Z;
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < n; id += stride) {
    int x, y, z;
    vox_coords(id, n, Y, Z, x, y, z);
    const float c = v[id];
    float g = 0.f;
    if (x + 1 < X) { const float d = v[id + sx] - c; g -= 2.f * d; part += (double)d * d; }
    if (x > 0) g += 2.f * (c - v[id - sx]);
    if (y + 1 < Y) { const float d = v[id + sy] - c; g -= 2.f * d; part += (double)d * d; }
    if (y > 0) g += 2.f * (c - v[id - sy]);
    if (z + 1 < Z) { const float d = v[id + 1] - c; g -= 2.f * d; part += (double)d * d; }
    if (z > 0) g += 2.f * (c - v[id - 1]);
    if (grad) grad[id] += (float)(scale * g);
  }
  block_add_double(part * scale, value);
}

// smoothness_prior_tf (objectives.py:57-69): mean squared adjacent-texel difference
__global__ void prior_tf_kernel(const float* __restrict__ t, int R, double scale,
                                double* __restrict__ grad, double* __restrict__ value) {
  double part = 0.0;
  for (int i = threadIdx.x; i < 4 * R; i += blockDim.x) {
    const int k = i >> 2;
    const double c = t[i];
    double g = 0.0;
    if (k + 1 < R) { const double d = (double)t[i + 4] - c; g -= 2.0 * d; part += d * d; }
    if (k > 0) g += 2.0 * (c - (double)t[i - 4]);
    if (grad) grad[i] += scale * g;
  }
  block_add_double(part * scale, value);
}

__global__ void __launch_bounds__(256) finite_check_kernel(const float* __restrict__ g,
                                                         long long n, int* __restrict__ flag) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  bool bad = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    bad |= !isfinite(g[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// adam_step (optim.py:45-67) + project_params (optim.py:70-89), skipped entirely
// when finite_check_kernel flagged a non-finite gradient (optim.py:28-30)
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ p,
                                                 const float* __restrict__ g,
                                                 float* __restrict__ m, float* __restrict__ v,
                                                 long long n, ddvr_adam a, float bc1, float bc2,
                                                 const int* __restrict__ flag,
                                                 const int32_t* __restrict__ state) {
  if (flag && *flag) return;
  if (state) {   // device step counter: bias corrections from adam_prep_kernel
    bc1 = __int_as_float(state[1]);
    bc2 = __int_as_float(state[2]);
  }
  const long long stride = (long long)gridDim.x * blockDim.x;
  const float b1 = (float)a.beta1, b2 = (float)a.beta2, lr = (float)a.lr, eps = (float)a.eps;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    float pi = p[i] - lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
    const bool last = a.stride <= 1 || (int)(i % a.stride) == a.stride - 1;
    pi = last ? fminf(fmaxf(pi, a.lo), a.hi) : fminf(fmaxf(pi, a.lo_other), a.hi_other);
    p[i] = pi;
  }
}

// project_params (optim.py:70-89) and gd_step (optim.py:33-42)
__global__ void __launch_bounds__(256) project_kernel(float* __restrict__ p, long long n,
                                                    ddvr_adam a) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool last = a.stride <= 1 || (int)(i % a.stride) == a.stride - 1;
    const float pi = p[i];
    p[i] = last ? fminf(fmaxf(pi, a.lo), a.hi) : fminf(fmaxf(pi, a.lo_other), a.hi_other);
  }
}

__global__ void __launch_bounds__(256) gd_kernel(float* __restrict__ p,
                                               const float* __restrict__ g, long long n,
                                               float lr, const int* __restrict__ flag) {
  if (flag && *flag) return;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    p[i] -= lr * g[i];
}

// Device-side Adam step counter (ddvr_adam_step_device): t = state[0] + 1 and the
// bias corrections 1 - beta^t (fp64, rounded once), unless the update is skipped
// for a non-finite gradient -- so a captured CUDA graph replays correct steps.
__global__ void adam_prep_kernel(int32_t* __restrict__ state, double beta1, double beta2,
                                 const int* __restrict__ flag) {
  if (threadIdx.x != 0 || (flag && *flag)) return;
  const int t = state[0] + 1;
  state[0] = t;
  state[1] = __float_as_int((float)(1.0 - pow(beta1, (double)t)));
  state[2] = __float_as_int((float)(1.0 - pow(beta2, (double)t)));
}

// upsample_volume (optim.py:92-129): fine node j at coarse coordinate (j - 0.5)/2,
// i0 = clip(floor, 0, n-2), edge half-cells extrapolate; separable, so the
// three axis passes collapse into one trilinear gather per fine voxel
__device__ __forceinline__ void up_axis(int j, int n, int& i0, int& i1, float& f) {
  if (n == 1) { i0 = i1 = 0; f = 0.f; return; }
  const float g = ((float)j - 0.5f) * 0.5f;
  i0 = min(max((int)floorf(g), 0), n - 2);
  i1 = i0 + 1;
  f = g - (float)i0;
}

__global__ void __launch_bounds__(256) upsample_kernel(const float* __restrict__ src, int X,
                                                     int Y, int Z, float* __restrict__ dst) {
  const long long n = 8LL * X * Y * Z;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < n; id += stride) {
    const int z = (int)(id % (2 * Z));
    const int y = (int)((id / (2 * Z)) % (2 * Y));
    const int x = (int)(id / (4LL * Y * Z));
    int x0, x1, y0, y1, z0, z1;
    float fx, fy, fz;
    up_axis(x, X, x0, x1, fx);
    up_axis(y, Y, y0, y1, fy);
    up_axis(z, Z, z0, z1, fz);
    auto at = [&](int a, int b, int c) { return src[((long long)a * Y + b) * Z + c]; };
    const float c00 = (1.f - fz) * at(x0, y0, z0) + fz * at(x0, y0, z1);
    const float c01 = (1.f - fz) * at(x0, y1, z0) + fz * at(x0, y1, z1);
    const float c10 = (1.f - fz) * at(x1, y0, z0) + fz * at(x1, y0, z1);
    const float c11 = (1.f - fz) * at(x1, y1, z0) + fz * at(x1, y1, z1);
    const float c0 = (1.f - fy) * c00 + fy * c01;
    const float c1 = (1.f - fy) * c10 + fy * c11;
    dst[id] = (1.f - fx) * c0 + fx * c1;
  }
}

// Swap the outer and inner axes of a C-order (A,B,C) float array into (C,B,A):
// the raw file is x-fastest (fileio.py:32, 65), the device volume z-fastest.
// 32x32 tiles through padded shared memory so both the read (along C) and the
// write (along A) are 128-byte coalesced; blockIdx.z walks B.  With a value
// range the load-side normalisation (fileio.py:66-70) is fused, computed in
// fp64 and rounded once, which is what the reference's float64 result becomes
// when it is rounded to the device's fp32.
constexpr int kSwapTile = 32;
template <bool NORM>
__global__ void __launch_bounds__(256) swap_xz_kernel(const float* __restrict__ src, int A, int B,
                                                      int C, double lo, double span,
                                                      float* __restrict__ dst) {
  __shared__ float tile[kSwapTile][kSwapTile + 1];
  const int c0 = blockIdx.x * kSwapTile, a0 = blockIdx.y * kSwapTile;
  for (int b = blockIdx.z; b < B; b += gridDim.z) {
    for (int i = threadIdx.y; i < kSwapTile; i += 8) {
      const int a = a0 + i, c = c0 + threadIdx.x;
      if (a < A && c < C) {
        float v = __ldg(src + ((long long)a * B + b) * C + c);
        if (NORM) v = (float)__ddiv_rn(__dsub_rn((double)v, lo), span);
        tile[i][threadIdx.x] = v;
      }
    }
    __syncthreads();
    for (int i = threadIdx.y; i < kSwapTile; i += 8) {
      const int c = c0 + i, a = a0 + threadIdx.x;
      if (a < A && c < C) dst[((long long)c * B + b) * A + a] = tile[threadIdx.x][i];
    }
    __syncthreads();
  }
}

// Binary PPM body over white (fileio.py:104-110): rgb + (1 - alpha), clamped to
// [0,1], x255, rounded half-to-even like np.round; fp64 from the fp32 image.
__global__ void __launch_bounds__(256) ppm_kernel(const float4* __restrict__ img, long long n,
                                                  uint8_t* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float4 p = img[i];
    const double w = 1.0 - (double)p.w;
    const float ch[3] = {p.x, p.y, p.z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double v = fmin(fmax((double)ch[k] + w, 0.0), 1.0);
      out[3 * i + k] = (uint8_t)__double2int_rn(255.0 * v);
    }
  }
}

// d_tf (fp64, the parameter layout count x stride) += sum over the CTA slots
// (tf_slot layout: rgba rows, then knot positions / (mu, sigma) pairs).
// 32 outputs x 8 slot lanes per block, reduced through shared memory.
// One output (texel channel, knot position, ...) per lane, 32 lanes of slots per output:
// slot lane ty sums slots ty, ty + 32, ... with four independent accumulators (slot
// index mod 4) so the L2 loads overlap, then fixed-order combines -- the same sum for
// every run (the TF gradient is reproducible bit for bit).
__global__ void __launch_bounds__(1024) tf_slots_reduce_kernel(const float* __restrict__ slots,
                                                               int nslot, int slot_floats,
                                                               int kind, int count,
                                                               double* __restrict__ d_tf) {
  __shared__ double part[32][33];
  const int stride = kind == DDVR_TF_TEXTURE ? 4 : kind == DDVR_TF_PIECEWISE ? 5 : 6;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int k = blockIdx.x * 32 + tx;
  const int nout = count * stride;
  int pos = 0;
  if (k < nout) {
    const int j = k / stride, c = k % stride;
    if (kind == DDVR_TF_TEXTURE) pos = 4 * j + c;
    else if (kind == DDVR_TF_PIECEWISE) pos = c == 0 ? 4 * count + j : 4 * j + c - 1;
    else pos = c < 2 ? 4 * count + 2 * j + c : 4 * j + c - 2;
  }
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (k < nout) {
    const float* q = slots + pos;
    int sl = ty;
    for (; sl + 96 < nslot; sl += 128) {
      a0 += (double)q[(size_t)sl * slot_floats];
      a1 += (double)q[(size_t)(sl + 32) * slot_floats];
      a2 += (double)q[(size_t)(sl + 64) * slot_floats];
      a3 += (double)q[(size_t)(sl + 96) * slot_floats];
    }
    for (; sl < nslot; sl += 32) a0 += (double)q[(size_t)sl * slot_floats];
  }
  part[ty][tx] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (ty == 0 && k < nout) {
    double t = 0.0;
#pragma unroll
    for (int r = 0; r < 32; ++r) t += part[r][tx];
    d_tf[k] += t;
  }
}

// DDVR_FLAG_DETERMINISTIC: the per-CTA camera / stepsize sums (3 doubles per
// CTA, CTA index = tile + tiles * view) reduced in a fixed order -- each
// thread strides over the CTAs in index order, then a fixed shared-memory tree
// -- so d_camera and d_dt are bitwise reproducible.  Blocks [0, cam_blocks)
// reduce view b's camera pair, the block after them the stepsize total.
__global__ void __launch_bounds__(256) partials_reduce_kernel(const double* __restrict__ part,
                                                            int tiles, int n_views,
                                                            int cam_blocks,
                                                            double* __restrict__ d_camera,
                                                            double* __restrict__ d_dt) {
  __shared__ double s0[256], s1[256];
  const int b = blockIdx.x, t = threadIdx.x;
  double a0 = 0.0, a1 = 0.0;
  if (b < cam_blocks) {
    const double* q = part + 3 * (size_t)b * tiles;
    for (int k = t; k < tiles; k += 256) { a0 += q[3 * k]; a1 += q[3 * k + 1]; }
  } else {
    const long long n = (long long)tiles * n_views;
    for (long long k = t; k < n; k += 256) a0 += part[3 * k + 2];
  }
  s0[t] = a0; s1[t] = a1;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (t < w) { s0[t] += s0[t + w]; s1[t] += s1[t + w]; }
    __syncthreads();
  }
  if (t == 0) {
    if (b < cam_blocks) { d_camera[2 * b] += s0[0]; d_camera[2 * b + 1] += s1[0]; }
    else *d_dt += s0[0];
  }
}

int grid_blocks(long long n) {
  long long b = (n + 255) / 256;
  return (int)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

extern "C" {

const char* ddvr_last_error(void) { return g_err; }

int32_t ddvr_abi_version(void) { return DDVR_ABI_VERSION; }

int64_t ddvr_launch_count(void) { return g_launches.load(); }

int64_t ddvr_cells_bytes(const int32_t dims[3]) {
  if (!dims || dims[0] < 1 || dims[1] < 1 || dims[2] < 1) return 0;
  return cell_count(dims) * 8 * (int64_t)sizeof(float);
}

int ddvr_pack_cells(const ddvr_volume* vol, float* cells_out, void* stream) {
  g_err[0] = 0;
  VolArgs V;
  int rc;
  if ((rc = make_vol(vol, V))) return rc;
  if (!cells_out) return set_error(DDVR_INVALID_INPUT, "cell output pointer is NULL");
  if (((uintptr_t)cells_out & 31) != 0)
    return set_error(DDVR_INVALID_INPUT, "cell records must be 32-byte aligned");
  const long long n = cell_count(vol->dims);
  pack_cells_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(V, cells_out,
                                                                                  n);
  return check_launch("pack_cells_kernel");
}

// Workspace layout: [cell-gradient records (volume target, cell layout)]
// [TF-gradient slots (tf target)], each part 256-byte aligned.
static int64_t ws_cells_bytes(const ddvr_volume* vol, uint32_t mask) {
  if (!vol || !vol->cells || !(mask & DDVR_TARGET_VOLUME)) return 0;
  return (ddvr_cells_bytes(vol->dims) + 255) & ~(int64_t)255;
}

static int tf_nslot(int slot_floats) {
  const int64_t budget = 32ll << 20;   // <= 32 MiB of slots
  const int64_t n = budget / ((int64_t)slot_floats * 4);
  return (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, n));
}

static int64_t ws_tf_bytes(const ddvr_tf* tf, uint32_t mask) {
  if (!tf || !(mask & DDVR_TARGET_TF) || tf->count < 1) return 0;
  const int sf = tf_slot_floats(tf->kind, tf->count);
  return (int64_t)tf_nslot(sf) * sf * 4;
}

int64_t ddvr_adjoint_workspace_bytes(const ddvr_volume* vol, const ddvr_tf* tf, uint32_t mask) {
  return ws_cells_bytes(vol, mask) + ws_tf_bytes(tf, mask);
}

// DDVR_FLAG_DETERMINISTIC partials: after the 256-aligned end of the workspace
static int64_t det_bytes(int64_t ctas, uint32_t mask) {
  if (!(mask & (DDVR_TARGET_CAMERA | DDVR_TARGET_STEPSIZE))) return 0;
  return (ctas * 3 * 8 + 255) & ~(int64_t)255;
}

// DDVR_FLAG_DETERMINISTIC with the volume target and cell records: a 256-byte header
// (the fixed-point scale, the seed bound) and the int64 cell-gradient moments (8 per
// padded cell record), after the partials
static int64_t det_vol_bytes(const ddvr_volume* vol, uint32_t mask) {
  if (!vol || !vol->cells || !(mask & DDVR_TARGET_VOLUME)) return 0;
  return 256 + 2 * ((ddvr_cells_bytes(vol->dims) + 255) & ~(int64_t)255);
}

// max |seed| over n floats as ordered float bits (non-negative floats order like ints)
__global__ void __launch_bounds__(256) seed_absmax_kernel(const float* __restrict__ seed,
                                                        long long n,
                                                        unsigned* __restrict__ out) {
  float m = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    m = fmaxf(m, fabsf(seed[i]));
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
}

// The fixed-point scale of the deterministic cell gradients: 2^50 / C, C a bound of any
// one flush's moment (a run of at most lmax samples, |phi| <= 1, |d_hat| <= dmax).  From
// the blend / Beer-Lambert adjoint (renderer.py:583-608) with |seed| <= smax, rgb <= c:
//   |d_hat| <= R smax (3 max|delta rgb| + dt max|delta tau| (2 + 6 c))
// (the affine absorption walk's d_hat = seed_a T_n dt R b is the delta-tau term).  Each
// flush is then < 2^50 and a cell's int64 sum has room for 8192 such flushes; fp32
// moments keep ~2^-50 of C in the quantisation.
__global__ void __launch_bounds__(256) det_scale_kernel(const float* __restrict__ texels,
                                                      int R, double dt, double lmax,
                                                      double smax_host,
                                                      double* __restrict__ header) {
  __shared__ float s_max[3][256];
  float drgb = 0.f, dtau = 0.f, rgb = 0.f;
  for (int k = threadIdx.x; k < R; k += blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(texels)[k];
    const float4 b = reinterpret_cast<const float4*>(texels)[min(k + 1, R - 1)];
    drgb = fmaxf(drgb, fmaxf(fabsf(b.x - a.x), fmaxf(fabsf(b.y - a.y), fabsf(b.z - a.z))));
    dtau = fmaxf(dtau, fabsf(b.w - a.w));
    rgb = fmaxf(rgb, fmaxf(fabsf(a.x), fmaxf(fabsf(a.y), fabsf(a.z))));
  }
  s_max[0][threadIdx.x] = drgb; s_max[1][threadIdx.x] = dtau; s_max[2][threadIdx.x] = rgb;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < blockDim.x; ++t) {
      drgb = fmaxf(drgb, s_max[0][t]); dtau = fmaxf(dtau, s_max[1][t]); rgb = fmaxf(rgb, s_max[2][t]);
    }
    const double smax = smax_host >= 0.0 ? smax_host
                        : (double)__uint_as_float(reinterpret_cast<unsigned*>(header + 1)[0]);
    const double dmax = (double)R * smax * (3.0 * drgb + dt * dtau * (2.0 + 6.0 * rgb));
    const double c = lmax * dmax;
    header[0] = c > 0.0 ? 1125899906842624.0 / c : 1.0;   // 2^50 / C
  }
}

// Brick occupancy maps of the fused band-tape step: bricks of 8^3 padded cell records
// (storage indices [8b, 8b+8) per axis), a byte per brick for the occupancy and for
// the 2x2x2 window OR the march reads (VolArgs::occ).
static int64_t brick_map_bytes(const int32_t dims[3]) {
  const int64_t nb = (int64_t)((dims[0] + 8) >> 3) * ((dims[1] + 8) >> 3) * ((dims[2] + 8) >> 3);
  return (2 * nb + 255) & ~(int64_t)255;
}

// occ[b] = some record of brick b has a nonzero coefficient (one CTA per brick; the
// records of a z-run of the brick are contiguous 256-byte lines)
__global__ void __launch_bounds__(256) brick_occupancy_kernel(const float* __restrict__ cells,
                                                            int CX, int CY, int CZ, int NBy,
                                                            int NBz,
                                                            unsigned char* __restrict__ occ) {
  const int b = blockIdx.x;
  const int bz = b % NBz, by = (b / NBz) % NBy, bx = b / (NBz * NBy);
  bool nz = false;
  for (int r = threadIdx.x; r < 512; r += 256) {
    const int sx = 8 * bx + (r >> 6), sy = 8 * by + ((r >> 3) & 7), sz = 8 * bz + (r & 7);
    if (sx < CX && sy < CY && sz < CZ) {
      const uint4* q = reinterpret_cast<const uint4*>(
          cells + 8 * (((long long)sx * CY + sy) * CZ + sz));
      const uint4 a = __ldg(q), c = __ldg(q + 1);
      nz |= ((a.x | a.y | a.z | a.w | c.x | c.y | c.z | c.w) & 0x7fffffffu) != 0u;
    }
  }
  nz = __syncthreads_or(nz);
  if (threadIdx.x == 0) occ[b] = nz ? 1 : 0;
}

// win[b] = some brick of the window b .. b+1 (per axis, those that exist) is occupied
__global__ void __launch_bounds__(256) brick_window_kernel(const unsigned char* __restrict__ occ,
                                                         int NBx, int NBy, int NBz,
                                                         unsigned char* __restrict__ win) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= NBx * NBy * NBz) return;
  const int bz = b % NBz, by = (b / NBz) % NBy, bx = b / (NBz * NBy);
  unsigned char any = 0;
  for (int x = bx; x <= min(bx + 1, NBx - 1); ++x)
    for (int y = by; y <= min(by + 1, NBy - 1); ++y)
      for (int z = bz; z <= min(bz + 1, NBz - 1); ++z) any |= occ[(x * NBy + y) * NBz + z];
  win[b] = any;
}

// DDVR_FLAG_BAND_TAPE: 32-bit words per ray, from an upper bound of any ray's
// step count: n = ceil(chord / dt - 1e-9) <= diag / dt + 1 (renderer.py:209-214)
static int band_words(const double bmin[3], const double bmax[3], double dt) {
  double d2 = 0.0;
  for (int a = 0; a < 3; ++a) d2 += (bmax[a] - bmin[a]) * (bmax[a] - bmin[a]);
  const double nmax = std::floor(std::sqrt(d2) / dt) + 3.0;
  return (int)std::min<double>((nmax + 31.0) / 32.0, 1 << 26);
}

// per-ray walk weights of the split band-tape step (one float per thread of the grid)
static int64_t ray_k_bytes(int64_t ctas) { return (ctas * kThreads * 4 + 255) & ~(int64_t)255; }

static int64_t grid_ctas(int32_t n_views, const ddvr_params* p) {
  const int row1 = p->row1 <= 0 ? p->height : p->row1;
  const int rows = std::max(0, row1 - p->row0);
  return (int64_t)((p->width + kTile - 1) / kTile) * ((rows + kTile - 1) / kTile) * n_views;
}

// Segment-split rays for a fused step with the TF target (masks 4 and 12: no camera /
// stepsize) whose rays alone would not fill the GPU: the smallest SPLIT in {2, 4, 8} that
// gives ~113 K threads (148 SMs x 3 CTAs x 256), else 1.  DDVR_SPLIT=1|2|4|8 in the
// environment overrides it (A/B measurements; 16 only there).
static int split_of(uint32_t mask, long long rays, int32_t flags) {
  // camera / stepsize alone (no TF, no volume): 2 or 4 lanes per ray, not with the
  // deterministic mode (its partials are per CTA of the one-thread-per-ray grid); by default
  // 2 while one thread per ray would run under 4 waves of 4 CTAs/SM -- halving the CTAs'
  // length halves the last wave's tail (C3: 1.7 waves, 82.4 -> 88.3 G samples/s)
  const bool pos = mask && !(mask & ~(uint32_t)(DDVR_TARGET_CAMERA | DDVR_TARGET_STEPSIZE));
  if (pos) {
    if (flags & (DDVR_FLAG_DETERMINISTIC | DDVR_FLAG_RAY_SPLIT_OFF | DDVR_FLAG_RAY_SPLIT_8))
      return 1;
    if (flags & DDVR_FLAG_RAY_SPLIT_2) return 2;
    if (flags & DDVR_FLAG_RAY_SPLIT_4) return 4;
    return rays < 4ll * 148 * 4 * kThreads ? 2 : 1;
  }
  if (mask != DDVR_TARGET_TF && mask != (DDVR_TARGET_TF | DDVR_TARGET_VOLUME)) return 1;
  if (flags & DDVR_FLAG_RAY_SPLIT_OFF) return 1;
  if (flags & DDVR_FLAG_RAY_SPLIT_2) return 2;
  if (flags & DDVR_FLAG_RAY_SPLIT_4) return 4;
  if (flags & DDVR_FLAG_RAY_SPLIT_8) return 8;
  static const int forced = [] {
    const char* e = std::getenv("DDVR_SPLIT");
    const int v = e ? std::atoi(e) : 0;
    return v == 1 || v == 2 || v == 4 || v == 8 || v == 16 ? v : 0;
  }();
  if (forced) return forced;
  constexpr long long kFill = 148ll * 3 * kThreads;
  int k = 1;
  while (k < 8 && rays * k < kFill) k *= 2;
  return k;
}

int32_t ddvr_ray_split(uint32_t mask, int64_t rays, int32_t flags) {
  return split_of(mask, rays, flags);
}

int64_t ddvr_band_tape_bytes(const ddvr_volume* vol, int32_t n_views, const ddvr_params* p) {
  if (!vol || !p || n_views < 0 || p->width < 1 || p->height < 1 || !(p->dt > 0.0)) return 0;
  if (vol->dims[0] < 1 || vol->dims[1] < 1 || vol->dims[2] < 1) return 0;
  const int64_t b = grid_ctas(n_views, p) * kThreads * band_words(vol->box_min, vol->box_max,
                                                                  p->dt) * 4;
  // the tape, then the empty-brick map (optional: a workspace without it marches every
  // block), then the per-ray walk weights of the split march / walk kernels (optional:
  // without them the step runs as one fused kernel)
  return ((b + 255) & ~(int64_t)255) + brick_map_bytes(vol->dims) +
         ray_k_bytes(grid_ctas(n_views, p));
}

int64_t ddvr_deterministic_bytes(const ddvr_volume* vol, int32_t n_views, const ddvr_params* p,
                                 uint32_t mask) {
  if (!p || n_views < 0 || p->width < 1 || p->height < 1) return 0;
  const int row1 = p->row1 <= 0 ? p->height : p->row1;
  const int rows = std::max(0, row1 - p->row0);
  const int64_t ctas = (int64_t)((p->width + kTile - 1) / kTile) * ((rows + kTile - 1) / kTile) *
                       n_views;
  return det_bytes(ctas, mask) + det_vol_bytes(vol, mask);
}

int ddvr_forward(const ddvr_volume* vol, const ddvr_tf* tf, const ddvr_camera* cams,
                 int32_t n_views, const ddvr_params* p, float* image_out, float* depth_out,
                 void* stream) {
  g_err[0] = 0;
  VolArgs V;
  TfArgs T;
  Geometry G;
  size_t tbl;
  int rc;
  if ((rc = make_vol(vol, V)) || (rc = make_tf(tf, T, tbl)) || (rc = make_geo(cams, n_views, p, G)))
    return rc;
  if (!image_out) return set_error(DDVR_INVALID_INPUT, "image output pointer is NULL");
  if (n_views == 0 || G.row1 == G.row0) return DDVR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid = grid_of(G, n_views);
  const bool early = p->early_stop != 0, cells = V.cells != nullptr, tape = G.tape != nullptr;
launch_forward(early, cells, tape, grid, tbl, st, V, T, G, image_out, depth_out);
  return check_launch("dvr_forward_kernel");
}

// Shared body of ddvr_adjoint and ddvr_forward_adjoint_l1 (fu != NULL):
// target/output/workspace validation, workspace zeroing, the adjoint (or fused)
// launch, TF-slot reduction and the cell-gradient fold.
static int run_adjoint(const ddvr_volume* vol, const ddvr_tf* tf, VolArgs& V, TfArgs& T,
                       Geometry& G, size_t tbl, int32_t n_views, const float* image,
                       const float* depth, const float* seed, uint32_t mask, float* d_volume,
                       double* d_tf, double* d_camera, double* d_dt, void* workspace,
                       int64_t workspace_bytes, void* stream, const FusedArgs* fu,
                       int32_t flags) {
  int rc;
  if (flags & ~(DDVR_FLAG_WS_CONTINUE | DDVR_FLAG_WS_DEFER | DDVR_FLAG_DETERMINISTIC |
                DDVR_FLAG_BAND_TAPE | DDVR_FLAG_NO_EMPTY_SKIP | DDVR_FLAG_SPLIT_WALK |
                DDVR_FLAG_RAY_SPLIT_OFF | DDVR_FLAG_RAY_SPLIT_2 | DDVR_FLAG_RAY_SPLIT_4 |
                DDVR_FLAG_RAY_SPLIT_8))
    return set_error(DDVR_INVALID_PARAMETER, "unknown params.flags bits 0x%x", flags);
  {
    const int32_t sf = flags & (DDVR_FLAG_RAY_SPLIT_OFF | DDVR_FLAG_RAY_SPLIT_2 |
                                DDVR_FLAG_RAY_SPLIT_4 | DDVR_FLAG_RAY_SPLIT_8);
    if (sf & (sf - 1))
      return set_error(DDVR_INVALID_PARAMETER, "at most one DDVR_FLAG_RAY_SPLIT_* flag (0x%x)", sf);
  }
  if (mask == 0 || (mask & ~15u))
    return set_error(DDVR_UNSUPPORTED, "adjoint requires a differentiation target (mask %u)", mask);
  if ((mask & DDVR_TARGET_VOLUME) && !d_volume)
    return set_error(DDVR_INVALID_INPUT, "d_volume is NULL but the volume target is set");
  if ((mask & DDVR_TARGET_TF) && !d_tf)
    return set_error(DDVR_INVALID_INPUT, "d_tf is NULL but the tf target is set");
  if ((mask & DDVR_TARGET_CAMERA) && !d_camera)
    return set_error(DDVR_INVALID_INPUT, "d_camera is NULL but the camera target is set");
  if ((mask & DDVR_TARGET_STEPSIZE) && !d_dt)
    return set_error(DDVR_INVALID_INPUT, "d_dt is NULL but the stepsize target is set");
  const int64_t ws_cells = ws_cells_bytes(vol, mask), ws_tf = ws_tf_bytes(tf, mask);
  const int64_t ws_need = ws_cells + ws_tf;
  const dim3 grid = grid_of(G, n_views);
  const int64_t ws_part = (flags & DDVR_FLAG_DETERMINISTIC)
                              ? det_bytes((int64_t)grid.x * grid.y * grid.z, mask) : 0;
  const int64_t ws_dvol = (flags & DDVR_FLAG_DETERMINISTIC) ? det_vol_bytes(vol, mask) : 0;
  const int64_t ws_det = ws_part + ws_dvol;
  const int64_t det_off = (ws_need + 255) & ~(int64_t)255;
  if (ws_dvol > 0 && T.kind != DDVR_TF_TEXTURE)
    return set_error(DDVR_UNSUPPORTED, "the deterministic density gradient needs a texel TF");
  if (ws_dvol > 0 && mask != DDVR_TARGET_VOLUME)
    return set_error(DDVR_UNSUPPORTED, "the deterministic density gradient is computed for the "
                     "volume target alone (mask %u)", mask);
  if (ws_dvol > 0 && !fu && (flags & (DDVR_FLAG_WS_CONTINUE | DDVR_FLAG_WS_DEFER)))
    return set_error(DDVR_UNSUPPORTED, "the deterministic density gradient of ddvr_adjoint "
                     "takes its fixed-point scale from the call's seed: one call per step");
  if (ws_need > 0 && (!workspace || workspace_bytes < ws_need))
    return set_error(DDVR_INVALID_INPUT,
                     "this target mask needs a %lld-byte workspace "
                     "(ddvr_adjoint_workspace_bytes)", (long long)ws_need);
  if (ws_det > 0 && (!workspace || workspace_bytes < det_off + ws_det))
    return set_error(DDVR_INVALID_INPUT,
                     "the deterministic mode needs a %lld-byte workspace "
                     "(ddvr_adjoint_workspace_bytes rounded up to 256 + ddvr_deterministic_bytes)",
                     (long long)(det_off + ws_det));
  // band tape: fused volume-only steps only (else the flag is ignored)
  const bool band = (flags & DDVR_FLAG_BAND_TAPE) && fu && mask == DDVR_TARGET_VOLUME && V.cells;
  const int64_t tape_off = det_off + ((ws_det + 255) & ~(int64_t)255);
  const int64_t ws_band = band ? (int64_t)grid.x * grid.y * grid.z * kThreads *
                                     band_words(V.bmin, V.bmax, G.dt) * 4 : 0;
  if (ws_band > (16ll << 30))
    return set_error(DDVR_UNSUPPORTED, "band tape of %lld bytes exceeds 16 GiB (2^32 words): "
                     "split the views into chunks", (long long)ws_band);
  if (ws_band > 0 && (!workspace || workspace_bytes < tape_off + ws_band))
    return set_error(DDVR_INVALID_INPUT,
                     "the band tape needs a %lld-byte workspace (ddvr_adjoint_workspace_bytes "
                     "rounded up to 256 [+ ddvr_deterministic_bytes rounded up to 256] + "
                     "ddvr_band_tape_bytes)", (long long)(tape_off + ws_band));
  if (ws_band > 0) {
    G.bits = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + tape_off);
    G.bits_words = band_words(V.bmin, V.bmax, G.dt);
  }
  // View groups (cta_view_tile): the adjoint / fused CTAs cycle over 4 views per tile
  // instead of running view after view (C4 263 -> 278 G samples/s, with or without views
  // ordered by direction).  DDVR_VGROUP=<n> in the environment overrides it (A/B).
  {
    static const int vg = [] {
      const char* e = std::getenv("DDVR_VGROUP");
      const int v = e ? std::atoi(e) : 4;
      return v >= 1 && v <= 4096 ? v : 4;
    }();
    G.vgroup = n_views > 1 ? vg : 1;
  }
  const int64_t map_off = tape_off + ((ws_band + 255) & ~(int64_t)255);
  const bool brick_map = ws_band > 0 && !(flags & DDVR_FLAG_NO_EMPTY_SKIP) &&
                         workspace_bytes >= map_off + brick_map_bytes(vol->dims);
  // DDVR_FLAG_SPLIT_WALK: the band-tape step as two kernels (march, walk)
  const int64_t rayk_off = map_off + brick_map_bytes(vol->dims);
  if (ws_band > 0 && (flags & DDVR_FLAG_SPLIT_WALK) &&
      workspace_bytes >= rayk_off + ray_k_bytes((int64_t)grid.x * grid.y * grid.z))
    G.ray_k = reinterpret_cast<float*>(static_cast<char*>(workspace) + rayk_off);
  if (workspace && ((uintptr_t)workspace & 31) != 0)
    return set_error(DDVR_INVALID_INPUT, "workspace must be 32-byte aligned");
  if (n_views == 0 || G.row1 == G.row0) return DDVR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = tbl;
  const bool cells = V.cells != nullptr;
  if (ws_dvol > 0) {   // int64 fixed-point cell gradients (order-independent sums)
    double* header = reinterpret_cast<double*>(static_cast<char*>(workspace) + det_off + ws_part);
    unsigned long long* c64 = reinterpret_cast<unsigned long long*>(
        reinterpret_cast<char*>(header) + 256);
    V.cells64 = c64 + (V.cell0 - V.cells);   // relative to cell (0,0,0), like cell0
    V.det_scale = header;
    if (!(flags & DDVR_FLAG_WS_CONTINUE)) {   // the first call of the step fixes the scale
      cudaError_t e = cudaMemsetAsync(header, 0, (size_t)ws_dvol, st);
      if (e != cudaSuccess)
        return set_error(DDVR_CUDA_ERROR, "workspace memset: %s", cudaGetErrorString(e));
      double smax_host = -1.0;
      if (fu) {
        smax_host = (double)fu->inv_count;   // the L1 seed is +-1/count
      } else {
        const long long n = 4ll * n_views * (G.row1 - G.row0) * G.W;
        seed_absmax_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 8), 256, 0,
                             st>>>(seed, n, reinterpret_cast<unsigned*>(header + 1));
        if ((rc = check_launch("seed_absmax_kernel"))) return rc;
      }
      // the longest run of samples in one cell: the cell diagonal over the smallest step
      const double smin = std::min(V.scale[0], std::min(V.scale[1], V.scale[2]));
      const double lmax = std::ceil(std::sqrt(3.0) / (G.dt * smin)) + 2.0;
      det_scale_kernel<<<1, 256, 0, st>>>(T.params, T.count, G.dt, lmax, smax_host, header);
      if ((rc = check_launch("det_scale_kernel"))) return rc;
    }
  }
  if (ws_part > 0) {   // every call reduces its own partials (also under WS_DEFER)
    G.partials = reinterpret_cast<double*>(static_cast<char*>(workspace) + det_off);
    cudaError_t e = cudaMemsetAsync(G.partials, 0, (size_t)ws_part, st);
    if (e != cudaSuccess)
      return set_error(DDVR_CUDA_ERROR, "partials memset: %s", cudaGetErrorString(e));
  }
  float* d_cells_all = ws_cells > 0 ? static_cast<float*>(workspace) : nullptr;
  // the kernel indexes cell gradients relative to cell (0,0,0), like V.cell0
  float* d_cells = d_cells_all ? d_cells_all + (V.cell0 - V.cells) : nullptr;
  if (ws_tf > 0) {
    T.slots = reinterpret_cast<float*>(static_cast<char*>(workspace) + ws_cells);
    T.nslot = tf_nslot(T.slot_floats);
  }
  if (ws_need > 0 && !(flags & DDVR_FLAG_WS_CONTINUE)) {
    cudaError_t e = cudaMemsetAsync(workspace, 0, (size_t)ws_need, st);
    if (e != cudaSuccess)
      return set_error(DDVR_CUDA_ERROR, "workspace memset: %s", cudaGetErrorString(e));
  }
  if (brick_map) {   // the march skips 32-sample blocks that lie in empty bricks
    const int NBx = (V.X + 8) >> 3, nb = NBx * V.NBy * V.NBz;
    unsigned char* occ = static_cast<unsigned char*>(workspace) + map_off;
    brick_occupancy_kernel<<<nb, 256, 0, st>>>(V.cells, V.X + 1, V.CY, V.CZ, V.NBy, V.NBz, occ);
    if ((rc = check_launch("brick_occupancy_kernel"))) return rc;
    brick_window_kernel<<<(nb + 255) / 256, 256, 0, st>>>(occ, NBx, V.NBy, V.NBz, occ + nb);
    if ((rc = check_launch("brick_window_kernel"))) return rc;
    V.occ = occ + nb;
  }
  auto launch = mask <= 3 ? launch_adjoint_g0 : mask <= 7 ? launch_adjoint_g1
              : mask <= 11 ? launch_adjoint_g2 : launch_adjoint_g3;
  const int split = fu && cells ? split_of(mask, (long long)n_views * (G.row1 - G.row0) * G.W, flags)
                                  : 1;
  if (ws_tf > 0 && !(flags & (DDVR_FLAG_WS_CONTINUE | DDVR_FLAG_WS_DEFER))) {
    // a one-call step uses (and reduces) only as many TF slots as it has CTAs
    const long long ctas =
        split > 1 ? (long long)((G.W + 7) / 8) *
                        ((G.row1 - G.row0 + kThreads / split / 8 - 1) / (kThreads / split / 8)) *
                        n_views
                  : (long long)grid.x * grid.y * grid.z;
    T.nslot = (int)std::min<long long>(T.nslot, ctas);
  }
  const int n_kernels =
      split > 1 ? launch_adjoint_split(mask, split, n_views, smem, st, V, T, G, d_volume, d_cells,
                                       d_camera, d_dt, *fu)
                : launch(mask, cells, grid, smem, st, V, T, G, image, depth, seed, d_volume,
                         d_cells, d_camera, d_dt, fu);
  if ((rc = check_launch(fu ? "dvr_adjoint_kernel (fused)" : "dvr_adjoint_kernel"))) return rc;
  g_launches.fetch_add(n_kernels - 1, std::memory_order_relaxed);
  if (ws_part > 0) {
    const int tiles = (int)(grid.x * grid.y);
    const int cam_blocks = (mask & DDVR_TARGET_CAMERA) ? n_views : 0;
    const int blocks = cam_blocks + ((mask & DDVR_TARGET_STEPSIZE) ? 1 : 0);
    partials_reduce_kernel<<<blocks, 256, 0, st>>>(G.partials, tiles, n_views, cam_blocks,
                                                   d_camera, d_dt);
    if ((rc = check_launch("partials_reduce_kernel"))) return rc;
  }
  if (flags & DDVR_FLAG_WS_DEFER) return DDVR_OK;   // a later call of this step folds
  if (ws_tf > 0) {
    const int nout = T.count * T.stride;
    tf_slots_reduce_kernel<<<(nout + 31) / 32, 1024, 0, st>>>(T.slots, T.nslot, T.slot_floats,
                                                             T.kind, T.count, d_tf);
    if ((rc = check_launch("tf_slots_reduce_kernel"))) return rc;
  }
  if (d_cells) {
    const long long nvox = (long long)V.X * V.Y * V.Z;
    if (!V.cells64 && V.X >= 3 && V.Y >= 3 && V.Z >= 3) {   // interior + boundary shell
      const long long nin = (long long)(V.X - 2) * (V.Y - 2) * (V.Z - 2), nsh = nvox - nin;
      fold_interior_kernel<<<(unsigned)((nin + 255) / 256), 256, 0, st>>>(V, d_cells_all,
                                                                         d_volume, nin);
      if ((rc = check_launch("fold_interior_kernel"))) return rc;
      fold_shell_kernel<<<(unsigned)((nsh + 255) / 256), 256, 0, st>>>(V, d_cells_all, d_volume,
                                                                      nsh);
      return check_launch("fold_shell_kernel");
    }
    fold_cells_kernel<<<(unsigned)((nvox + 255) / 256), 256, 0, st>>>(V, d_cells_all, d_volume,
                                                                     nvox);
    return check_launch("fold_cells_kernel");
  }
  return DDVR_OK;
}

int ddvr_adjoint(const ddvr_volume* vol, const ddvr_tf* tf, const ddvr_camera* cams,
                 int32_t n_views, const ddvr_params* p, const float* image, const float* depth,
                 const float* seed, uint32_t mask, float* d_volume, double* d_tf,
                 double* d_camera, double* d_dt, void* workspace, int64_t workspace_bytes,
                 void* stream) {
  g_err[0] = 0;
  VolArgs V;
  TfArgs T;
  Geometry G;
  size_t tbl;
  int rc;
  if ((rc = make_vol(vol, V)) || (rc = make_tf(tf, T, tbl)) || (rc = make_geo(cams, n_views, p, G)))
    return rc;
  if (mask == 0 || (mask & ~15u))
    return set_error(DDVR_UNSUPPORTED, "adjoint requires a differentiation target (mask %u)", mask);
  if (!seed) return set_error(DDVR_INVALID_INPUT, "seed pointer is NULL");
  if (!image && !depth) return set_error(DDVR_INVALID_INPUT, "image and optical depth are NULL");
  return run_adjoint(vol, tf, V, T, G, tbl, n_views, image, depth, seed, mask, d_volume, d_tf,
                     d_camera, d_dt, workspace, workspace_bytes, stream, nullptr, p->flags);
}

int ddvr_forward_adjoint_l1(const ddvr_volume* vol, const ddvr_tf* tf, const ddvr_camera* cams,
                            int32_t n_views, const ddvr_params* p, const float* refs,
                            double count, uint32_t mask, float* image_out, float* depth_out,
                            double* loss_out, float* d_volume, double* d_tf, double* d_camera,
                            double* d_dt, void* workspace, int64_t workspace_bytes,
                            void* stream) {
  g_err[0] = 0;
  VolArgs V;
  TfArgs T;
  Geometry G;
  size_t tbl;
  int rc;
  if ((rc = make_vol(vol, V)) || (rc = make_tf(tf, T, tbl)) || (rc = make_geo(cams, n_views, p, G)))
    return rc;
  if (!V.cells)
    return set_error(DDVR_UNSUPPORTED, "the fused step needs cell records (ddvr_pack_cells)");
  if (G.tape) return set_error(DDVR_UNSUPPORTED, "the fused step has no stored (tape) mode");
  if (!refs) return set_error(DDVR_INVALID_INPUT, "reference image pointer is NULL");
  if (!loss_out) return set_error(DDVR_INVALID_INPUT, "loss pointer is NULL");
  if (!(count > 0.0)) return set_error(DDVR_INVALID_PARAMETER, "element count must be positive");
  FusedArgs fu{refs, (float)(1.0 / count), 1.0 / count, loss_out, image_out, depth_out};
  return run_adjoint(vol, tf, V, T, G, tbl, n_views, nullptr, nullptr, nullptr, mask, d_volume,
                     d_tf, d_camera, d_dt, workspace, workspace_bytes, stream, &fu, p->flags);
}

int ddvr_forward_grad(const ddvr_volume* vol, const ddvr_tf* tf, const ddvr_camera* cams,
                      int32_t n_views, const ddvr_params* p, uint32_t wrt, float* image_out,
                      float* jac_out, void* stream) {
  g_err[0] = 0;
  VolArgs V;
  TfArgs T;
  Geometry G;
  size_t tbl;
  int rc;
  if ((rc = make_vol(vol, V)) || (rc = make_tf(tf, T, tbl)) || (rc = make_geo(cams, n_views, p, G)))
    return rc;
  if (wrt != DDVR_TARGET_CAMERA && wrt != DDVR_TARGET_STEPSIZE)   // renderer.py:428-431
    return set_error(DDVR_UNSUPPORTED, "forward mode supports camera and stepsize, not mask %u",
                     wrt);
  if (!image_out || !jac_out) return set_error(DDVR_INVALID_INPUT, "output pointer is NULL");
  if (n_views == 0 || G.row1 == G.row0) return DDVR_OK;
  launch_forward_grad(wrt == DDVR_TARGET_CAMERA ? 2 : 1, V.cells != nullptr, grid_of(G, n_views),
                      tbl, (cudaStream_t)stream, V, T, G, image_out, jac_out);
  return check_launch("dvr_forward_grad_kernel");
}

int ddvr_forward_color(const ddvr_volume* cv, const ddvr_camera* cams, int32_t n_views,
                       const ddvr_params* p, float* image_out, float* depth_out, void* stream) {
  g_err[0] = 0;
  VolArgs V;
  Geometry G;
  int rc;
  if ((rc = make_vol(cv, V)) || (rc = make_geo(cams, n_views, p, G))) return rc;
  if (cv->cells) return set_error(DDVR_UNSUPPORTED, "colour volumes use the voxel layout");
  if (((uintptr_t)cv->data & 15) != 0)
    return set_error(DDVR_INVALID_INPUT, "colour volume must be 16-byte aligned");
  if (!image_out) return set_error(DDVR_INVALID_INPUT, "image output pointer is NULL");
  if (n_views == 0 || G.row1 == G.row0) return DDVR_OK;
  launch_forward_color(p->early_stop != 0, G.tape != nullptr, grid_of(G, n_views),
                       (cudaStream_t)stream, V, G, image_out, depth_out);
  return check_launch("dvr_forward_color_kernel");
}

int ddvr_adjoint_color(const ddvr_volume* cv, const ddvr_camera* cams, int32_t n_views,
                       const ddvr_params* p, const float* image, const float* depth,
                       const float* seed, float* d_color, void* stream) {
  g_err[0] = 0;
  VolArgs V;
  Geometry G;
  int rc;
  if ((rc = make_vol(cv, V)) || (rc = make_geo(cams, n_views, p, G))) return rc;
  if (cv->cells) return set_error(DDVR_UNSUPPORTED, "colour volumes use the voxel layout");
  if (((uintptr_t)cv->data & 15) != 0 || (d_color && ((uintptr_t)d_color & 15) != 0))
    return set_error(DDVR_INVALID_INPUT, "colour volume and gradient must be 16-byte aligned");
  if (!seed || !d_color) return set_error(DDVR_INVALID_INPUT, "seed or d_color pointer is NULL");
  if (!image && !depth) return set_error(DDVR_INVALID_INPUT, "image and optical depth are NULL");
  if (n_views == 0 || G.row1 == G.row0) return DDVR_OK;
  launch_adjoint_color(grid_of(G, n_views), (cudaStream_t)stream, V, G, image, depth, seed,
                       d_color);
  return check_launch("dvr_adjoint_color_kernel");
}

int ddvr_l1_loss(const float* x, const float* y, int64_t n, double count, float* seed_out,
                 double* loss_out, void* stream) {
  g_err[0] = 0;
  if (n < 0) return set_error(DDVR_INVALID_PARAMETER, "negative element count");
  if (!(count > 0.0)) return set_error(DDVR_INVALID_PARAMETER, "normaliser must be positive");
  if (n == 0) return DDVR_OK;
  if (!x || !y) return set_error(DDVR_INVALID_INPUT, "image or reference pointer is NULL");
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  l1_loss_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(x, y, n, (float)(1.0 / count),
                                                           1.0 / count, seed_out, loss_out);
  return check_launch("l1_loss_kernel");
}

int ddvr_gather_probe(const ddvr_volume* vol, const ddvr_camera* cams, int32_t n_views,
                      const ddvr_params* p, int32_t hold, float* out, void* stream) {
  g_err[0] = 0;
  VolArgs V;
  Geometry G;
  int rc;
  if ((rc = make_vol(vol, V, false)) || (rc = make_geo(cams, n_views, p, G))) return rc;
  if (!V.cells) return set_error(DDVR_INVALID_INPUT, "the gather probe needs cell records");
  if (!out) return set_error(DDVR_INVALID_INPUT, "output pointer is NULL");
  if (n_views == 0 || G.row1 == G.row0) return DDVR_OK;
  launch_gather_probe(hold != 0, grid_of(G, n_views), (cudaStream_t)stream, V, G, out);
  return check_launch("gather_probe_kernel");
}

int ddvr_opacity_entropy(const float* images, int64_t n_pixels, int32_t n_images, double* out,
                         float* seed_out, void* stream) {
  g_err[0] = 0;
  if (n_pixels < 0 || n_images < 0)
    return set_error(DDVR_INVALID_PARAMETER, "negative image count or size");
  if (n_images == 0) return DDVR_OK;
  if (!images || !out) return set_error(DDVR_INVALID_INPUT, "image or output pointer is NULL");
  if (n_images > 65535) return set_error(DDVR_UNSUPPORTED, "more than 65535 images per call");
  if ((reinterpret_cast<uintptr_t>(images) | reinterpret_cast<uintptr_t>(seed_out)) & 15)
    return set_error(DDVR_INVALID_INPUT, "images and seed must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * 4 * (size_t)n_images, st);
  if (e != cudaSuccess) return set_error(DDVR_CUDA_ERROR, "entropy memset: %s", cudaGetErrorString(e));
  const unsigned bx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n_pixels + 255) / 256, 148));
  const auto* im = reinterpret_cast<const float4*>(images);
  int rc;
  if (n_pixels > 0) {
    entropy_sums_kernel<<<dim3(bx, n_images), 256, 0, st>>>(im, n_pixels, out);
    if ((rc = check_launch("entropy_sums_kernel"))) return rc;
  }
  entropy_seed_kernel<<<dim3(bx, n_images), 256, 0, st>>>(im, n_pixels, out,
                                                          reinterpret_cast<float4*>(seed_out));
  return check_launch("entropy_seed_kernel");
}

int ddvr_ray_setup(const ddvr_volume* vol, const ddvr_camera* cams, int32_t n_views,
                   const ddvr_params* p, double* tn_tf, int32_t* n_steps, int32_t* flags,
                   void* stream) {
  g_err[0] = 0;
  VolArgs V;
  Geometry G;
  int rc;
  if ((rc = make_vol(vol, V, false)) || (rc = make_geo(cams, n_views, p, G))) return rc;
  if (!n_steps) return set_error(DDVR_INVALID_INPUT, "n_steps pointer is NULL");
  if (n_views == 0 || G.row1 == G.row0) return DDVR_OK;
  ray_setup_kernel<<<grid_of(G, n_views), kThreads, 0, (cudaStream_t)stream>>>(V, G, tn_tf,
                                                                              n_steps, flags);
  return check_launch("ray_setup_kernel");
}

int ddvr_prior_volume(const float* values, const int32_t dims[3], double weight, float* grad_out,
                      double* value_out, void* stream) {
  g_err[0] = 0;
  if (!dims || dims[0] < 1 || dims[1] < 1 || dims[2] < 1)
    return set_error(DDVR_INVALID_PARAMETER, "volume values must be a non-empty 3D array");
  if (!values) return set_error(DDVR_INVALID_INPUT, "volume pointer is NULL");
  const long long X = dims[0], Y = dims[1], Z = dims[2];
  const long long count = (X > 1 ? (X - 1) * Y * Z : 0) + (Y > 1 ? X * (Y - 1) * Z : 0) +
                          (Z > 1 ? X * Y * (Z - 1) : 0);
  if (count == 0) return DDVR_OK;    // objectives.py:90-91: prior 0, gradient 0
  prior_volume_kernel<<<grid_blocks(X * Y * Z), 256, 0, (cudaStream_t)stream>>>(
      values, dims[0], dims[1], dims[2], weight / (double)count, grad_out, value_out);
  return check_launch("prior_volume_kernel");
}

int ddvr_prior_tf(const float* texels, int32_t resolution, double weight, double* grad_out,
                  double* value_out, void* stream) {
  g_err[0] = 0;
  if (resolution < 1)
    return set_error(DDVR_INVALID_PARAMETER, "transfer function must have shape (R, 4), R >= 1");
  if (!texels) return set_error(DDVR_INVALID_INPUT, "texel pointer is NULL");
  if (resolution < 2) return DDVR_OK;   // objectives.py:61-62
  prior_tf_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(texels, resolution,
                                                        weight / (4.0 * (resolution - 1)),
                                                        grad_out, value_out);
  return check_launch("prior_tf_kernel");
}

int ddvr_adam_step(float* params, const float* grads, float* m, float* v, int64_t n,
                   const ddvr_adam* cfg, int32_t* nonfinite, void* stream) {
  g_err[0] = 0;
  if (!cfg) return set_error(DDVR_INVALID_PARAMETER, "adam config is NULL");
  if (!(cfg->lr > 0.0)) return set_error(DDVR_INVALID_PARAMETER, "learning rate must be positive");
  if (cfg->step < 1) return set_error(DDVR_INVALID_PARAMETER, "adam step must be >= 1");
  if (n < 0) return set_error(DDVR_INVALID_PARAMETER, "negative parameter count");
  if (n == 0) return DDVR_OK;
  if (!params || !grads || !m || !v)
    return set_error(DDVR_INVALID_INPUT, "parameter, gradient or moment pointer is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  if (nonfinite) {
    finite_check_kernel<<<grid_blocks(n), 256, 0, st>>>(grads, n, nonfinite);
    int rc = check_launch("finite_check_kernel");
    if (rc) return rc;
  }
  const float bc1 = (float)(1.0 - pow(cfg->beta1, (double)cfg->step));
  const float bc2 = (float)(1.0 - pow(cfg->beta2, (double)cfg->step));
  adam_kernel<<<grid_blocks(n), 256, 0, st>>>(params, grads, m, v, n, *cfg, bc1, bc2, nonfinite,
                                               nullptr);
  return check_launch("adam_kernel");
}

int ddvr_adam_step_device(float* params, const float* grads, float* m, float* v, int64_t n,
                          const ddvr_adam* cfg, int32_t* state, int32_t* nonfinite,
                          void* stream) {
  g_err[0] = 0;
  if (!cfg) return set_error(DDVR_INVALID_PARAMETER, "adam config is NULL");
  if (!(cfg->lr > 0.0)) return set_error(DDVR_INVALID_PARAMETER, "learning rate must be positive");
  if (n < 0) return set_error(DDVR_INVALID_PARAMETER, "negative parameter count");
  if (!state) return set_error(DDVR_INVALID_INPUT, "adam state pointer is NULL");
  if (n == 0) return DDVR_OK;
  if (!params || !grads || !m || !v)
    return set_error(DDVR_INVALID_INPUT, "parameter, gradient or moment pointer is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (nonfinite) {
    finite_check_kernel<<<grid_blocks(n), 256, 0, st>>>(grads, n, nonfinite);
    if ((rc = check_launch("finite_check_kernel"))) return rc;
  }
  adam_prep_kernel<<<1, 32, 0, st>>>(state, cfg->beta1, cfg->beta2, nonfinite);
  if ((rc = check_launch("adam_prep_kernel"))) return rc;
  adam_kernel<<<grid_blocks(n), 256, 0, st>>>(params, grads, m, v, n, *cfg, 1.f, 1.f, nonfinite,
                                               state);
  return check_launch("adam_kernel");
}

int ddvr_project(float* params, int64_t n, const ddvr_adam* cfg, void* stream) {
  g_err[0] = 0;
  if (!cfg) return set_error(DDVR_INVALID_PARAMETER, "projection config is NULL");
  if (n < 0) return set_error(DDVR_INVALID_PARAMETER, "negative parameter count");
  if (n == 0) return DDVR_OK;
  if (!params) return set_error(DDVR_INVALID_INPUT, "parameter pointer is NULL");
  project_kernel<<<grid_blocks(n), 256, 0, (cudaStream_t)stream>>>(params, n, *cfg);
  return check_launch("project_kernel");
}

int ddvr_gd_step(float* params, const float* grads, int64_t n, double lr, int32_t* nonfinite,
                 void* stream) {
  g_err[0] = 0;
  if (!(lr > 0.0)) return set_error(DDVR_INVALID_PARAMETER, "learning rate must be positive");
  if (n < 0) return set_error(DDVR_INVALID_PARAMETER, "negative parameter count");
  if (n == 0) return DDVR_OK;
  if (!params || !grads) return set_error(DDVR_INVALID_INPUT, "parameter or gradient pointer is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (nonfinite) {
    finite_check_kernel<<<grid_blocks(n), 256, 0, st>>>(grads, n, nonfinite);
    if ((rc = check_launch("finite_check_kernel"))) return rc;
  }
  gd_kernel<<<grid_blocks(n), 256, 0, st>>>(params, grads, n, (float)lr, nonfinite);
  return check_launch("gd_kernel");
}

int ddvr_field_sample(const double* values, const int32_t dims[3], const double box_min[3],
                      const double box_max[3], const double* points, int64_t n,
                      double* value_out, double* spatial_out, double* weights_out,
                      int64_t* corners_out, void* stream) {
  g_err[0] = 0;
  if (!dims || dims[0] < 1 || dims[1] < 1 || dims[2] < 1)
    return set_error(DDVR_INVALID_PARAMETER, "volume values must be a non-empty 3D array");
  if (!box_min || !box_max) return set_error(DDVR_INVALID_PARAMETER, "box is NULL");
  for (int a = 0; a < 3; ++a)
    if (!(box_max[a] > box_min[a]))
      return set_error(DDVR_INVALID_PARAMETER, "box_max must exceed box_min on every axis");
  if (n < 0) return set_error(DDVR_INVALID_PARAMETER, "negative point count");
  if (n == 0) return DDVR_OK;
  if (!values || !points) return set_error(DDVR_INVALID_INPUT, "values or points pointer is NULL");
  const int d[3] = {dims[0], dims[1], dims[2]};
  launch_field_sample(values, d, box_min, box_max, points, n, value_out, spatial_out,
                      weights_out, reinterpret_cast<long long*>(corners_out),
                      (cudaStream_t)stream);
  return check_launch("field_sample_kernel");
}

int ddvr_tf_lookup(const double* texels, int32_t resolution, const double* density, int64_t n,
                   double* out4, double* slope4, double* weights2, int64_t* idx2, void* stream) {
  g_err[0] = 0;
  if (resolution < 1) return set_error(DDVR_INVALID_PARAMETER, "transfer function needs >= 1 texel");
  if (n < 0) return set_error(DDVR_INVALID_PARAMETER, "negative sample count");
  if (n == 0) return DDVR_OK;
  if (!texels || !density) return set_error(DDVR_INVALID_INPUT, "texels or density pointer is NULL");
  launch_tf_lookup(texels, resolution, density, n, out4, slope4, weights2,
                   reinterpret_cast<long long*>(idx2), (cudaStream_t)stream);
  return check_launch("tf_lookup_kernel");
}

int ddvr_opacity(const double* tau, int64_t n, double dt, double* alpha, double* dalpha,
                 void* stream) {
  g_err[0] = 0;
  if (n < 0) return set_error(DDVR_INVALID_PARAMETER, "negative sample count");
  if (n == 0) return DDVR_OK;
  if (!tau) return set_error(DDVR_INVALID_INPUT, "tau pointer is NULL");
  launch_opacity(tau, n, dt, alpha, dalpha, (cudaStream_t)stream);
  return check_launch("opacity_kernel");
}

int ddvr_camera_rays(const ddvr_camera* cam, int32_t width, int32_t height, const double* u,
                     const double* v, int64_t n, double* origin, double* dir, double* j_origin,
                     double* j_dir, void* stream) {
  g_err[0] = 0;
  if (!cam) return set_error(DDVR_INVALID_PARAMETER, "camera is NULL");
  if (width < 1 || height < 1) return set_error(DDVR_INVALID_PARAMETER, "image size must be >= 1");
  if (!(cam->radius > 0.0)) return set_error(DDVR_INVALID_PARAMETER, "camera radius must be positive");
  if (!(cam->fov_y_deg > 0.0 && cam->fov_y_deg < 180.0))
    return set_error(DDVR_INVALID_PARAMETER, "fov_y_deg must lie in (0, 180)");
  if (!(fabs(cam->lat_deg) < 90.0 - 1e-3))
    return set_error(DDVR_INVALID_PARAMETER, "latitude too close to a pole");
  if (n < 0) return set_error(DDVR_INVALID_PARAMETER, "negative pixel count");
  if (n == 0) return DDVR_OK;
  if (!u || !v) return set_error(DDVR_INVALID_INPUT, "pixel coordinate pointer is NULL");
  launch_camera_rays(*cam, width, height, u, v, n, origin, dir, j_origin, j_dir,
                     (cudaStream_t)stream);
  return check_launch("camera_rays_kernel");
}

int ddvr_upsample_volume(const float* src, const int32_t dims[3], float* dst, void* stream) {
  g_err[0] = 0;
  if (!dims || dims[0] < 1 || dims[1] < 1 || dims[2] < 1)
    return set_error(DDVR_INVALID_PARAMETER, "volume values must be a non-empty 3D array");
  if (!src || !dst) return set_error(DDVR_INVALID_INPUT, "volume pointer is NULL");
  upsample_kernel<<<grid_blocks(8LL * dims[0] * dims[1] * dims[2]), 256, 0,
                    (cudaStream_t)stream>>>(src, dims[0], dims[1], dims[2], dst);
  return check_launch("upsample_kernel");
}

static int swap_xz(const float* src, int A, int B, int C, const double* range, float* dst,
                   void* stream) {
  const dim3 grid((C + kSwapTile - 1) / kSwapTile, (A + kSwapTile - 1) / kSwapTile,
                  std::max(1, std::min(65535, (B + 3) / 4)));   // 4 slices per CTA
  if ((long long)grid.y > 65535) return set_error(DDVR_UNSUPPORTED, "volume axis too large");
  if (range) {
    swap_xz_kernel<true><<<grid, dim3(kSwapTile, 8), 0, (cudaStream_t)stream>>>(
        src, A, B, C, range[0], range[1] - range[0], dst);
  } else {
    swap_xz_kernel<false><<<grid, dim3(kSwapTile, 8), 0, (cudaStream_t)stream>>>(
        src, A, B, C, 0.0, 1.0, dst);
  }
  return check_launch("swap_xz_kernel");
}

int ddvr_volume_from_raw(const float* raw, const int32_t dims[3], const double* value_range,
                         float* dst, void* stream) {
  g_err[0] = 0;
  if (!dims || dims[0] < 1 || dims[1] < 1 || dims[2] < 1)
    return set_error(DDVR_INVALID_PARAMETER, "volume values must be a non-empty 3D array");
  if (value_range && !(value_range[1] > value_range[0]))
    return set_error(DDVR_INVALID_PARAMETER, "value_range must be increasing");
  if (!raw || !dst) return set_error(DDVR_INVALID_INPUT, "volume pointer is NULL");
  if (raw == dst) return set_error(DDVR_INVALID_INPUT, "in-place layout swap is not supported");
  return swap_xz(raw, dims[2], dims[1], dims[0], value_range, dst, stream);
}

int ddvr_volume_to_raw(const float* src, const int32_t dims[3], float* raw, void* stream) {
  g_err[0] = 0;
  if (!dims || dims[0] < 1 || dims[1] < 1 || dims[2] < 1)
    return set_error(DDVR_INVALID_PARAMETER, "volume values must be a non-empty 3D array");
  if (!raw || !src) return set_error(DDVR_INVALID_INPUT, "volume pointer is NULL");
  if (raw == src) return set_error(DDVR_INVALID_INPUT, "in-place layout swap is not supported");
  return swap_xz(src, dims[0], dims[1], dims[2], nullptr, raw, stream);
}

int ddvr_image_to_ppm(const float* images, int64_t n_pixels, uint8_t* out, void* stream) {
  g_err[0] = 0;
  if (n_pixels < 0) return set_error(DDVR_INVALID_PARAMETER, "negative pixel count");
  if (n_pixels == 0) return DDVR_OK;
  if (!images || !out) return set_error(DDVR_INVALID_INPUT, "image pointer is NULL");
  if (reinterpret_cast<uintptr_t>(images) & 15)
    return set_error(DDVR_INVALID_INPUT, "images must be 16-byte aligned");
  ppm_kernel<<<grid_blocks(n_pixels), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(images), n_pixels, out);
  return check_launch("ppm_kernel");
}

}  // extern "C"
