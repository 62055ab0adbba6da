// ddvr_adj_g1.cu -- adjoint kernel instantiations for target masks 4-7.
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

DDVR_ADJ_LAUNCHER(launch_adjoint_g1) {
  switch (mask) {
    case 4:
      if (cells) adj<4, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<4, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    case 5:
      if (cells) adj<5, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<5, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    case 6:
      if (cells) adj<6, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<6, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    case 7:
      if (cells) adj<7, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<7, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    default:
      break;
  }
}

}  // namespace ddvr_impl
