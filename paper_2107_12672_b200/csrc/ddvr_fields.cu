// ddvr_fields.cu -- the point-wise field functions of the hot path as public
// device calls: camera rays and their
// (lon, lat) Jacobians, trilinear sampling and its gradients, the texel TF
// lookup and its gradients, and the Beer-Lambert segment opacity.
//
// The march kernels evaluate these inline in fp32 on cell records; here they
// run in fp64 over caller-given points with the reference's operation order and
// separately rounded +,-,*,/,sqrt (dm/da/ds/dd: never contracted into FMA), so
// the results are the reference's bit for bit wherever no transcendental is
// involved (trilinear_*, tf_*), and within an ulp of libm elsewhere.
#include "ddvr_device.cuh"

namespace {
using namespace ddvr_impl;

// ---------------------------------------------------------------------------
// trilinear_sample / trilinear_gradients (field.py:279-349, 379-517)
// ---------------------------------------------------------------------------
struct FieldArgs {
  const double* __restrict__ values;    // (X,Y,Z) z fastest
  int X, Y, Z;
  double bmin[3], bmax[3];
};

__global__ void __launch_bounds__(256) field_sample_kernel(
    FieldArgs F, const double* __restrict__ pts, long long n, double* __restrict__ value_out,
    double* __restrict__ spatial_out, double* __restrict__ weights_out,
    long long* __restrict__ corners_out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int dims[3] = {F.X, F.Y, F.Z};
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    // _grid_setup (field.py:279-308)
    double g[3], f[3], s[3];
    long long ix[3];
    bool inside = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double x = pts[3 * p + a];
      const double ext = ds(F.bmax[a], F.bmin[a]);
      s[a] = dd((double)dims[a], ext);
      g[a] = ds(dm(ds(x, F.bmin[a]), s[a]), 0.5);
      const double tol = dm(1e-9, ext);
      inside = inside && x >= ds(F.bmin[a], tol) && x <= da(F.bmax[a], tol);
      const double gc = fmin(fmax(g[a], 0.0), (double)(dims[a] - 1));   // np.clip
      long long i = (long long)floor(gc);
      i = i < 0 ? 0 : i;
      const long long top = dims[a] - 2 > 0 ? dims[a] - 2 : 0;
      ix[a] = i > top ? top : i;
      f[a] = ds(gc, (double)ix[a]);
    }
    // _corner_indices (field.py:311-324), C order, corner b = bx | by << 1 | bz << 2
    long long j[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) j[a] = ix[a] + 1 < dims[a] - 1 ? ix[a] + 1 : dims[a] - 1;
    long long cidx[8];
    double v[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const long long cx = (b & 1) ? j[0] : ix[0], cy = (b & 2) ? j[1] : ix[1],
                      cz = (b & 4) ? j[2] : ix[2];
      cidx[b] = (cx * F.Y + cy) * F.Z + cz;
      v[b] = F.values[cidx[b]];
    }
    // _corner_weights (field.py:327-333) and the sequential corner sum (:343-345)
    const double ex = ds(1.0, f[0]), ey = ds(1.0, f[1]), ez = ds(1.0, f[2]);
    double w[8];
#pragma unroll
    for (int b = 0; b < 8; ++b)
      w[b] = dm(dm((b & 1) ? f[0] : ex, (b & 2) ? f[1] : ey), (b & 4) ? f[2] : ez);
    double out = dm(w[0], v[0]);
#pragma unroll
    for (int b = 1; b < 8; ++b) out = da(out, dm(w[b], v[b]));
    // live mask: inside and the [0,1] clamp inactive (field.py:486-499)
    const double mask = (inside && out >= 0.0 && out <= 1.0) ? 1.0 : 0.0;
    if (spatial_out) {
      // partials w.r.t. the fractions (field.py:444-457), left-to-right sums
      const double fx = f[0], fy = f[1], fz = f[2];
      const double dfx = da(da(da(dm(dm(ey, ez), ds(v[1], v[0])), dm(dm(fy, ez), ds(v[3], v[2]))),
                               dm(dm(ey, fz), ds(v[5], v[4]))),
                            dm(dm(fy, fz), ds(v[7], v[6])));
      const double dfy = da(da(da(dm(dm(ex, ez), ds(v[2], v[0])), dm(dm(fx, ez), ds(v[3], v[1]))),
                               dm(dm(ex, fz), ds(v[6], v[4]))),
                            dm(dm(fx, fz), ds(v[7], v[5])));
      const double dfz = da(da(da(dm(dm(ex, ey), ds(v[4], v[0])), dm(dm(fx, ey), ds(v[5], v[1]))),
                               dm(dm(ex, fy), ds(v[6], v[2]))),
                            dm(dm(fx, fy), ds(v[7], v[3])));
      const double dfa[3] = {dfx, dfy, dfz};
#pragma unroll
      for (int a = 0; a < 3; ++a) {   // world units, 0 where the edge clamp froze g (:459-484)
        const bool live = g[a] >= 0.0 && g[a] <= (double)dims[a] - 1.0;
        spatial_out[3 * p + a] = dm(dm(dfa[a], live ? s[a] : 0.0), mask);
      }
    }
    if (weights_out) {
#pragma unroll
      for (int b = 0; b < 8; ++b) weights_out[8 * p + b] = dm(w[b], mask);
    }
    if (corners_out) {
#pragma unroll
      for (int b = 0; b < 8; ++b) corners_out[8 * p + b] = cidx[b];
    }
    if (value_out) {
      out = inside ? out : 0.0;
      value_out[p] = fmin(fmax(out, 0.0), 1.0);
    }
  }
}

// ---------------------------------------------------------------------------
// tf_sample / tf_gradients (field.py:525-579)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) tf_lookup_kernel(
    const double* __restrict__ T, int R, const double* __restrict__ d, long long n,
    double* __restrict__ out4, double* __restrict__ slope4, double* __restrict__ weights2,
    long long* __restrict__ idx2) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    const double dv = d[p];
    const double dc = fmin(fmax(dv, 0.0), 1.0);
    const double t = ds(dm(dc, (double)R), 0.5);
    const double f = fmin(fmax(t, 0.0), (double)(R - 1));
    long long i0 = (long long)floor(f);
    const long long top = R - 2 > 0 ? R - 2 : 0;
    i0 = i0 < 0 ? 0 : (i0 > top ? top : i0);
    const long long i1 = i0 + 1 < R - 1 ? i0 + 1 : R - 1;
    const double w = ds(f, (double)i0), ew = ds(1.0, w);
    if (out4) {
#pragma unroll
      for (int c = 0; c < 4; ++c) out4[4 * p + c] = da(dm(ew, T[4 * i0 + c]), dm(w, T[4 * i1 + c]));
    }
    if (slope4) {
      const double live =
          (t >= 0.0 && t <= (double)R - 1.0 && dv >= 0.0 && dv <= 1.0) ? 1.0 : 0.0;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        slope4[4 * p + c] = dm(dm(ds(T[4 * i1 + c], T[4 * i0 + c]), (double)R), live);
    }
    if (weights2) { weights2[2 * p] = ew; weights2[2 * p + 1] = w; }
    if (idx2) { idx2[2 * p] = i0; idx2[2 * p + 1] = i1; }
  }
}

// ---------------------------------------------------------------------------
// opacity_from_density (field.py:587-600), EPS_ALPHA field.py:25
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) opacity_kernel(const double* __restrict__ tau, long long n,
                                                      double dt, double* __restrict__ alpha,
                                                      double* __restrict__ dalpha) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const double top = ds(1.0, 1e-6);
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    const double e = exp(dm(-dt, tau[p]));
    const double a = ds(1.0, e);
    const bool clamped = a > top;
    if (alpha) alpha[p] = clamped ? top : a;
    if (dalpha) dalpha[p] = clamped ? 0.0 : dm(dt, e);
  }
}

// ---------------------------------------------------------------------------
// camera_from_sphere / camera_gradients (field.py:186-271): the reference's dual
// numbers with p = 2 (autodiff.py:39-141), the same formulas term by term
// ---------------------------------------------------------------------------
struct D2 {
  double v, d0, d1;
};
__device__ __forceinline__ D2 cst(double x) { return {x, 0.0, 0.0}; }
__device__ __forceinline__ D2 add(D2 a, D2 b) { return {da(a.v, b.v), da(a.d0, b.d0), da(a.d1, b.d1)}; }
__device__ __forceinline__ D2 sub(D2 a, D2 b) { return {ds(a.v, b.v), ds(a.d0, b.d0), ds(a.d1, b.d1)}; }
__device__ __forceinline__ D2 neg(D2 a) { return {-a.v, -a.d0, -a.d1}; }
__device__ __forceinline__ D2 mul(D2 a, D2 b) {   // a.val * b.der + b.val * a.der
  return {dm(a.v, b.v), da(dm(a.v, b.d0), dm(b.v, a.d0)), da(dm(a.v, b.d1), dm(b.v, a.d1))};
}
__device__ __forceinline__ D2 div(D2 a, D2 b) {   // (a.der - val * b.der) * (1 / b.val)
  const double val = dd(a.v, b.v), inv = dd(1.0, b.v);
  return {val, dm(ds(a.d0, dm(val, b.d0)), inv), dm(ds(a.d1, dm(val, b.d1)), inv)};
}
__device__ __forceinline__ D2 dsqrt(D2 a) {
  const double s = __dsqrt_rn(a.v), two_s = dm(2.0, s);
  return {s, dd(a.d0, two_s), dd(a.d1, two_s)};
}
__device__ __forceinline__ D2 dsin(D2 a) {
  const double c = cos(a.v);
  return {sin(a.v), dm(c, a.d0), dm(c, a.d1)};
}
__device__ __forceinline__ D2 dcos(D2 a) {
  const double ms = -sin(a.v);
  return {cos(a.v), dm(ms, a.d0), dm(ms, a.d1)};
}

__global__ void __launch_bounds__(128) camera_rays_kernel(
    ddvr_camera cam, int W, int H, const double* __restrict__ u, const double* __restrict__ v,
    long long n, double* __restrict__ origin, double* __restrict__ dir,
    double* __restrict__ j_origin, double* __restrict__ j_dir) {
  double lon_deg = fmod(cam.lon_deg, 360.0);   // SphericalCamera stores lon % 360 (field.py:143)
  if (lon_deg < 0.0) lon_deg = da(lon_deg, 360.0);
  const D2 lon = mul(D2{lon_deg, 1.0, 0.0}, cst(kDeg));
  const D2 lat = mul(D2{cam.lat_deg, 0.0, 1.0}, cst(kDeg));
  const D2 cl = dcos(lat), sl = dsin(lat), cp = dcos(lon), sp = dsin(lon);
  const D2 rho = cst(cam.radius);
  const D2 o[3] = {add(mul(rho, mul(cl, cp)), cst(cam.center[0])),
                   add(mul(rho, sl), cst(cam.center[1])),
                   add(mul(rho, mul(cl, sp)), cst(cam.center[2]))};
  D2 fx = neg(mul(cl, cp)), fy = neg(sl), fz = neg(mul(cl, sp));
  const D2 fn = dsqrt(add(add(mul(fx, fx), mul(fy, fy)), mul(fz, fz)));
  fx = div(fx, fn); fy = div(fy, fn); fz = div(fz, fn);
  D2 rx = neg(fz), rz = fx;
  const D2 rn = dsqrt(add(mul(rx, rx), mul(rz, rz)));
  rx = div(rx, rn); rz = div(rz, rn);
  const D2 ux = neg(mul(rz, fy));
  const D2 uy = sub(mul(rz, fx), mul(rx, fz));
  const D2 uz = mul(rx, fy);
  const double th = tan(dm(dm(0.5, cam.fov_y_deg), kDeg));
  const double aspect = dd((double)W, (double)H);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    const D2 su = cst(dm(dm(ds(dm(da(u[p], 0.5), dd(2.0, (double)W)), 1.0), th), aspect));
    const D2 sv = cst(dm(ds(1.0, dm(da(v[p], 0.5), dd(2.0, (double)H))), th));
    const D2 dx = add(add(fx, mul(rx, su)), mul(ux, sv));
    const D2 dy = add(fy, mul(uy, sv));
    const D2 dz = add(add(fz, mul(rz, su)), mul(uz, sv));
    const D2 dn = dsqrt(add(add(mul(dx, dx), mul(dy, dy)), mul(dz, dz)));
    const D2 d[3] = {div(dx, dn), div(dy, dn), div(dz, dn)};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (origin) origin[3 * p + a] = o[a].v;
      if (dir) dir[3 * p + a] = d[a].v;
      if (j_origin) { j_origin[6 * p + 2 * a] = o[a].d0; j_origin[6 * p + 2 * a + 1] = o[a].d1; }
      if (j_dir) { j_dir[6 * p + 2 * a] = d[a].d0; j_dir[6 * p + 2 * a + 1] = d[a].d1; }
    }
  }
}

int blocks_for(long long n, int threads) {
  const long long b = (n + threads - 1) / threads;
  return (int)(b < 148 * 8 ? (b > 0 ? b : 1) : 148 * 8);
}

}  // namespace

namespace ddvr_impl {

void launch_field_sample(const double* values, const int dims[3], const double bmin[3],
                         const double bmax[3], const double* pts, long long n, double* value,
                         double* spatial, double* weights, long long* corners, cudaStream_t st) {
  FieldArgs F{values, dims[0], dims[1], dims[2], {bmin[0], bmin[1], bmin[2]},
              {bmax[0], bmax[1], bmax[2]}};
  field_sample_kernel<<<blocks_for(n, 256), 256, 0, st>>>(F, pts, n, value, spatial, weights,
                                                          corners);
}

void launch_tf_lookup(const double* texels, int R, const double* d, long long n, double* out4,
                      double* slope4, double* weights2, long long* idx2, cudaStream_t st) {
  tf_lookup_kernel<<<blocks_for(n, 256), 256, 0, st>>>(texels, R, d, n, out4, slope4, weights2,
                                                       idx2);
}

void launch_opacity(const double* tau, long long n, double dt, double* alpha, double* dalpha,
                    cudaStream_t st) {
  opacity_kernel<<<blocks_for(n, 256), 256, 0, st>>>(tau, n, dt, alpha, dalpha);
}

void launch_camera_rays(const ddvr_camera& cam, int W, int H, const double* u, const double* v,
                        long long n, double* origin, double* dir, double* j_origin,
                        double* j_dir, cudaStream_t st) {
  camera_rays_kernel<<<blocks_for(n, 128), 128, 0, st>>>(cam, W, H, u, v, n, origin, dir,
                                                         j_origin, j_dir);
}

}  // namespace ddvr_impl
