// ddvr_probe.cu -- the gather-roofline microbenchmark ("a measured
// 8-corner gather microbenchmark peak").
//
// Walks exactly the rays of the march (same ray setup, 32.32 fixed-point
// stepping, padded cell records) and issues the same 256-bit record gathers --
// held (reloaded only on a cell change, as the march does) or one per sample --
// but does a single FADD per sample instead of the interpolation, TF and
// compositing.  Its sample rate is the ceiling any kernel with this gather
// pattern can reach on this volume and these views; bench.py reports the
// march's and the fused step's fraction of it.
#include "ddvr_device.cuh"

namespace {
using namespace ddvr_impl;

template <bool HOLD>
__global__ void __launch_bounds__(kThreads, 6) gather_probe_kernel(VolArgs V, Geometry G,
                                                                   float* __restrict__ out) {
  __shared__ Frame F;
  const int view = blockIdx.z;
  if (threadIdx.x == 0) make_frame(G.cams[view], G.W, G.H, F);
  __syncthreads();
  int px, py;
  pixel_of(G, px, py);
  if (px >= G.W || py >= G.row1) return;
  Ray r;
  setup_ray(F, V, G.dt, G.W, G.H, px, py, r);
  long long gx = r.g0[0], gy = r.g0[1], gz = r.g0[2];
  float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  int held = INT_MIN;
  float acc = 0.f;
  for (int i = 0; i < r.n; ++i) {
    Cell c;
    locate_cells(V, gx, gy, gz, r.all_inside, c);
    gx += r.gs[0]; gy += r.gs[1]; gz += r.gs[2];
    gather_if(V, !HOLD || c.cell != held, c.cell, v);
    held = c.cell;
    acc += v[0];
  }
  out[((size_t)view * (G.row1 - G.row0) + (py - G.row0)) * G.W + px] = acc;
}

}  // namespace

namespace ddvr_impl {

void launch_gather_probe(bool hold, dim3 grid, cudaStream_t st, const VolArgs& V,
                         const Geometry& G, float* out) {
  if (hold) gather_probe_kernel<true><<<grid, kThreads, 0, st>>>(V, G, out);
  else gather_probe_kernel<false><<<grid, kThreads, 0, st>>>(V, G, out);
}

}  // namespace ddvr_impl
