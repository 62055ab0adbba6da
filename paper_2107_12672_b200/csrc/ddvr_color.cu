// ddvr_color.cu -- pre-shaded colour volumes: render_colorvol and
// render_colorvol_adjoint (renderer.py:404-407, 703-709).
//
// The volume is (X,Y,Z,4) float, one float4 (r, g, b emission, tau) per voxel;
// a sample is the per-channel trilinear interpolant (field.py:361-376: no
// [0,1] clamp, 0 outside the box), then the same Beer-Lambert compositing as
// the density path.  The adjoint walks back with the same exact optical-depth
// inversion and scatters w8 (inside-masked) x the out4 adjoint into the 8
// corner voxels (renderer.py:611-613), accumulated per cell run and flushed
// with 128-bit vector reds.
#include "ddvr_device.cuh"

namespace {
using namespace ddvr_impl;

__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

__device__ __forceinline__ float4 lerp4(float f, const float4& a, const float4& b) {
  return make_float4(__fmaf_rn(f, __fsub_rn(b.x, a.x), a.x), __fmaf_rn(f, __fsub_rn(b.y, a.y), a.y),
                     __fmaf_rn(f, __fsub_rn(b.z, a.z), a.z), __fmaf_rn(f, __fsub_rn(b.w, a.w), a.w));
}

// per-channel trilinear interpolant of the 8 corner float4s (0 outside)
__device__ __forceinline__ float4 sample_color(const VolArgs& V, const Cell& c) {
  const float* p = V.data + 4 * (size_t)c.base;
  const int ox = 4 * c.ox, oy = 4 * c.oy, oz = 4 * c.oz;
  const float4 a00 = lerp4(c.fx, ldg4(p), ldg4(p + ox));
  const float4 a10 = lerp4(c.fx, ldg4(p + oy), ldg4(p + ox + oy));
  const float4 a01 = lerp4(c.fx, ldg4(p + oz), ldg4(p + ox + oz));
  const float4 a11 = lerp4(c.fx, ldg4(p + oy + oz), ldg4(p + ox + oy + oz));
  const float4 s = lerp4(c.fz, lerp4(c.fy, a00, a10), lerp4(c.fy, a01, a11));
  return c.inside ? s : make_float4(0.f, 0.f, 0.f, 0.f);
}

template <bool EARLY, bool TAPE>
__global__ void __launch_bounds__(kThreads) dvr_forward_color_kernel(VolArgs V, Geometry G,
                                                                   float* __restrict__ image,
                                                                   float* __restrict__ depth) {
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
  float* tape = TAPE ? G.tape + pix * G.tape_stride : nullptr;
  float T = 1.f, A = 0.f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
  double S = 0.0;
  long long gx = r.g0[0], gy = r.g0[1], gz = r.g0[2];
  for (int i = 0; i < r.n; ++i) {
    if (EARLY && A > kAlphaStop) break;        // renderer.py:331-335
    if (TAPE) tape[i] = T;
    Cell c;
    locate_voxels(V, gx, gy, gz, r.all_inside, c);
    gx += r.gs[0]; gy += r.gs[1]; gz += r.gs[2];
    const float4 s = sample_color(V, c);
    const Segment g = segment<kSegGen>(s.w, G.dt32);
    const float Ta = __fmul_rn(T, g.a);
    c0 = __fmaf_rn(Ta, s.x, c0);
    c1 = __fmaf_rn(Ta, s.y, c1);
    c2 = __fmaf_rn(Ta, s.z, c2);
    A = __fadd_rn(A, Ta);
    T = __fmul_rn(T, g.ome);
    S += (double)g.od;
  }
  reinterpret_cast<float4*>(image)[pix] = make_float4(c0, c1, c2, A);
  if (depth) depth[pix] = (float)S;
}

__global__ void __launch_bounds__(kThreads) dvr_adjoint_color_kernel(
    VolArgs V, Geometry G, const float* __restrict__ image, const float* __restrict__ depth,
    const float* __restrict__ seed, float* __restrict__ d_color) {
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
  const float* tape = G.tape ? G.tape + pix * G.tape_stride : nullptr;
  const float4 sd = reinterpret_cast<const float4*>(seed)[pix];
  double S = depth ? (double)depth[pix]
                   : -log1p(-(double)reinterpret_cast<const float4*>(image)[pix].w);
  const float dt32 = G.dt32;
  float a_hat = sd.w;
  // per cell run: the 8 corner float4 gradients accumulate in registers and are
  // flushed with 8 vector reds when the ray leaves the cell (~1 sample in 3 at
  // dt = 0.2 voxel) instead of on every sample
  float4 acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  int run_base = INT_MIN, run_ox = 0, run_oy = 0, run_oz = 0;
  auto flush = [&]() {
    float* base = d_color + 4 * (size_t)run_base;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float* q = base + ((k & 1) ? 4 * run_ox : 0) + ((k & 2) ? 4 * run_oy : 0) +
                 ((k & 4) ? 4 * run_oz : 0);
      red128(q, acc[k].x, acc[k].y, acc[k].z, acc[k].w);
    }
  };
  long long gx = r.g0[0] + (long long)(r.n - 1) * r.gs[0];
  long long gy = r.g0[1] + (long long)(r.n - 1) * r.gs[1];
  long long gz = r.g0[2] + (long long)(r.n - 1) * r.gs[2];
  for (int i = r.n - 1; i >= 0; --i) {
    Cell c;
    locate_voxels(V, gx, gy, gz, r.all_inside, c);
    const float4 s = sample_color(V, c);
    const Segment g = segment<kSegGen>(s.w, dt32);
    float Tp;
    if (tape) {
      Tp = tape[i];
    } else {   // exact inversion in optical-depth form (see the density adjoint)
      S -= (double)g.od;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(Tp) : "f"((float)S * -1.4426950408889634f));
    }
    // blend + Beer-Lambert adjoint (renderer.py:583-596)
    const float cdot = s.x * sd.x + s.y * sd.y + s.z * sd.z;
    const float seg_a_hat = Tp * (a_hat + cdot);
    const float aT = g.a * Tp;
    a_hat = g.ome * a_hat - g.a * cdot;
    const float a_raw_hat = g.a_clamped ? 0.f : seg_a_hat;
    const float tau_hat = s.w < 0.f ? 0.f : dt32 * g.e * a_raw_hat;
    const float4 o4 = make_float4(aT * sd.x, aT * sd.y, aT * sd.z, tau_hat);
    if (c.inside) {   // renderer.py:611-613: w8 (inside-masked) x out4_hat per corner
      if (c.base != run_base) {
        if (run_base != INT_MIN) flush();
        run_base = c.base; run_ox = c.ox; run_oy = c.oy; run_oz = c.oz;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      const float ex = 1.f - c.fx, ey = 1.f - c.fy, ez = 1.f - c.fz;
      const float wz[2] = {ez, c.fz}, wy[2] = {ey, c.fy}, wx[2] = {ex, c.fx};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float wk = wx[k & 1] * wy[(k >> 1) & 1] * wz[(k >> 2) & 1];
        acc[k].x = __fmaf_rn(wk, o4.x, acc[k].x);
        acc[k].y = __fmaf_rn(wk, o4.y, acc[k].y);
        acc[k].z = __fmaf_rn(wk, o4.z, acc[k].z);
        acc[k].w = __fmaf_rn(wk, o4.w, acc[k].w);
      }
    }
    gx -= r.gs[0]; gy -= r.gs[1]; gz -= r.gs[2];
  }
  if (run_base != INT_MIN) flush();
}

}  // namespace

namespace ddvr_impl {

void launch_forward_color(bool early, bool tape, dim3 grid, cudaStream_t st, const VolArgs& V,
                          const Geometry& G, float* image, float* depth) {
  if (early && tape) dvr_forward_color_kernel<true, true><<<grid, kThreads, 0, st>>>(V, G, image, depth);
  else if (early) dvr_forward_color_kernel<true, false><<<grid, kThreads, 0, st>>>(V, G, image, depth);
  else if (tape) dvr_forward_color_kernel<false, true><<<grid, kThreads, 0, st>>>(V, G, image, depth);
  else dvr_forward_color_kernel<false, false><<<grid, kThreads, 0, st>>>(V, G, image, depth);
}

void launch_adjoint_color(dim3 grid, cudaStream_t st, const VolArgs& V, const Geometry& G,
                          const float* image, const float* depth, const float* seed,
                          float* d_color) {
  dvr_adjoint_color_kernel<<<grid, kThreads, 0, st>>>(V, G, image, depth, seed, d_color);
}

}  // namespace ddvr_impl
