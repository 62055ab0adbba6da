// ddvr_fwdgrad.cu -- forward-mode Jacobian of the image w.r.t. the camera pose
// (p = 2: lon, lat per degree) or the stepsize (p = 1): the reference's
// render_forward_grad (renderer.py:410-464), which re-runs _march over dual
// numbers (renderer.py:269-303) with the entry point differentiated through
// the deciding face (_entry_param_dual, renderer.py:217-231).
//
// Same ray setup, fixed-point positions, cell records and TF tables as the
// forward kernel; each sample carries d(position)/d(theta) -> d(density) (the
// spatial gradient, field.py:446-484) -> d(rgb, tau) (TF slope) -> d(alpha)
// -> the compositing recurrence T' = T(1-a), C += T a c, A += T a.
#include "ddvr_device.cuh"

namespace {
using namespace ddvr_impl;

template <int P, bool CELLS, int KIND>
__global__ void __launch_bounds__(kThreads) dvr_forward_grad_kernel(VolArgs V, TfArgs TFA,
                                                                  Geometry G,
                                                                  float* __restrict__ image,
                                                                  float* __restrict__ jac) {
  __shared__ Frame F;
  __shared__ unsigned s_info[5];
  const int view = blockIdx.z;
  if (threadIdx.x < 5) s_info[threadIdx.x] = 0u;
  __syncthreads();
  load_tf(TFA, s_info);
  if (threadIdx.x == 0) make_frame(G.cams[view], G.W, G.H, F);
  __syncthreads();

  int px, py;
  pixel_of(G, px, py);
  if (px >= G.W || py >= G.row1) return;
  Ray r;
  setup_ray(F, V, G.dt, G.W, G.H, px, py, r);
  const float dt32 = G.dt32;

  // d(grid position)/d(theta) = dg0 + t * dgw (camera); = i * gw (stepsize)
  float dg0[3][P], dgw[3][P];
  if (P == 2) {
    const bool need = !r.clamped && !r.miss;
#pragma unroll
    for (int j = 0; j < P; ++j) {
      double draw[3], dw[3], dxo[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) draw[k] = F.df[k][j] + F.dr[k][j] * r.su + F.du[k][j] * r.sv;
      const double proj = r.w[0] * draw[0] + r.w[1] * draw[1] + r.w[2] * draw[2];
#pragma unroll
      for (int k = 0; k < 3; ++k) dw[k] = (draw[k] - r.w[k] * proj) / r.dn;
      // tn = (face - o_k) / w_k for the deciding axis k (renderer.py:217-231)
      double dtn = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (need && r.axis == k) dtn = -(F.jo[k][j] + r.tn * dw[k]) / r.w[k];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        dxo[k] = F.jo[k][j] + dtn * r.w[k] + r.tn * dw[k];
        dg0[k][j] = (float)(dxo[k] * V.scale[k]);
        dgw[k][j] = (float)(dw[k] * V.scale[k]);
      }
    }
  }

  float T = 1.f, A = 0.f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
  float dT[P], dA[P], dC[3][P];
#pragma unroll
  for (int j = 0; j < P; ++j) { dT[j] = 0.f; dA[j] = 0.f; dC[0][j] = dC[1][j] = dC[2][j] = 0.f; }
  long long gx = r.g0[0], gy = r.g0[1], gz = r.g0[2];
  for (int i = 0; i < r.n; ++i) {
    Cell c;
    locate<CELLS>(V, gx, gy, gz, r.all_inside, c);
    float v[8];
    fetch8<CELLS>(V, c, v);
    const Interp ip = interp(c, v);
    const float raw = ip.rho;
    const float d = clamp_density(c.inside, raw);
    const bool live = c.inside && raw >= 0.f && raw <= 1.f;   // field.py:486-489
    // spatial gradient in grid units, zero where the edge clamp froze the axis
    float ddx = ip.gx;
    float ddy = interp_gy(c, v);
    float ddz = interp_gz(c, ip);
    ddx = (live && gx >= 0 && gx <= V.top[0]) ? ddx : 0.f;
    ddy = (live && gy >= 0 && gy <= V.top[1]) ? ddy : 0.f;
    ddz = (live && gz >= 0 && gz <= V.top[2]) ? ddz : 0.f;
    const float t = __fmul_rn((float)i, dt32);
    int i0; float w; float4 slope;
    const float4 s = tf_sample<KIND, true>(TFA, d, i0, w, slope, true);
    const Segment g = segment<kSegGen>(s.w, dt32);
    const float Ta = __fmul_rn(T, g.a);
#pragma unroll
    for (int j = 0; j < P; ++j) {
      float dd;
      if (P == 2) {
        dd = ddx * (dg0[0][j] + t * dgw[0][j]) + ddy * (dg0[1][j] + t * dgw[1][j]) +
             ddz * (dg0[2][j] + t * dgw[2][j]);
      } else {   // x_i = xo + (i dt) w: d x_i / d dt = i w (grid units: i gw)
        dd = (float)i * (ddx * r.gw[0] + ddy * r.gw[1] + ddz * r.gw[2]);
      }
      const float dc0 = slope.x * dd, dc1 = slope.y * dd, dc2 = slope.z * dd;
      const float dtau = s.w < 0.f ? 0.f : slope.w * dd;
      // a = 1 - exp(-dt tau): da = e * d(dt tau); zero where the EPS clamp is active
      const float dx = P == 1 ? dt32 * dtau + g.tau : dt32 * dtau;
      const float da = g.a_clamped ? 0.f : g.e * dx;
      const float dTa = dT[j] * g.a + T * da;
      dC[0][j] += dTa * s.x + Ta * dc0;
      dC[1][j] += dTa * s.y + Ta * dc1;
      dC[2][j] += dTa * s.z + Ta * dc2;
      dA[j] += dTa;
      dT[j] = dT[j] * g.ome - T * da;
    }
    c0 = __fmaf_rn(Ta, s.x, c0);
    c1 = __fmaf_rn(Ta, s.y, c1);
    c2 = __fmaf_rn(Ta, s.z, c2);
    A = __fadd_rn(A, Ta);
    T = __fmul_rn(T, g.ome);
    gx += r.gs[0]; gy += r.gs[1]; gz += r.gs[2];
  }
  const size_t pix = ((size_t)view * (G.row1 - G.row0) + (py - G.row0)) * G.W + px;
  reinterpret_cast<float4*>(image)[pix] = make_float4(c0, c1, c2, A);
  float* jp = jac + pix * 4 * P;   // (..., 4, P): channel-major like renderer.py:454-457
#pragma unroll
  for (int j = 0; j < P; ++j) {
    jp[0 * P + j] = dC[0][j];
    jp[1 * P + j] = dC[1][j];
    jp[2 * P + j] = dC[2][j];
    jp[3 * P + j] = dA[j];
  }
}

template <int P, bool CELLS>
void fwdgrad(int kind, dim3 grid, size_t smem, cudaStream_t st, const VolArgs& V,
             const TfArgs& T, const Geometry& G, float* image, float* jac) {
  if (kind == kTfPiecewise) {
    auto k = dvr_forward_grad_kernel<P, CELLS, kTfPiecewise>;
    set_smem(k, smem);
    k<<<grid, kThreads, smem, st>>>(V, T, G, image, jac);
  } else if (kind == kTfGaussian) {
    auto k = dvr_forward_grad_kernel<P, CELLS, kTfGaussian>;
    set_smem(k, smem);
    k<<<grid, kThreads, smem, st>>>(V, T, G, image, jac);
  } else {
    auto k = dvr_forward_grad_kernel<P, CELLS, kTfTexture>;
    set_smem(k, smem);
    k<<<grid, kThreads, smem, st>>>(V, T, G, image, jac);
  }
}

}  // namespace

namespace ddvr_impl {

void launch_forward_grad(int n_params, bool cells, dim3 grid, size_t smem, cudaStream_t st,
                         const VolArgs& V, const TfArgs& T, const Geometry& G, float* image,
                         float* jac) {
  if (n_params == 2) {
    if (cells) fwdgrad<2, true>(T.kind, grid, smem, st, V, T, G, image, jac);
    else fwdgrad<2, false>(T.kind, grid, smem, st, V, T, G, image, jac);
  } else {
    if (cells) fwdgrad<1, true>(T.kind, grid, smem, st, V, T, G, image, jac);
    else fwdgrad<1, false>(T.kind, grid, smem, st, V, T, G, image, jac);
  }
}

}  // namespace ddvr_impl
