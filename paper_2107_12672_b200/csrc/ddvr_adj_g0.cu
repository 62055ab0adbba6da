// ddvr_adj_g0.cu -- adjoint kernel instantiations for target masks 1-3.
#include "ddvr_device.cuh"

namespace ddvr_impl {

template <unsigned M, bool CELLS>
static void adj(dim3 grid, size_t smem, cudaStream_t st, const VolArgs& V, const TfArgs& T,
                const Geometry& G, const float* image, const float* depth, const float* seed,
                float* dv, float* dcells, double* dtf, double* dcam, double* ddt) {
  auto k = dvr_adjoint_kernel<M, CELLS>;
  set_smem(k, smem);
  k<<<grid, kThreads, smem, st>>>(V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
}

DDVR_ADJ_LAUNCHER(launch_adjoint_g0) {
  switch (mask) {
    case 1:
      if (cells) adj<1, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<1, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    case 2:
      if (cells) adj<2, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<2, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    case 3:
      if (cells) adj<3, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<3, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    default:
      break;
  }
}

}  // namespace ddvr_impl
