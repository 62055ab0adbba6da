// ddvr_adj_g2.cu -- adjoint kernel instantiations for target masks 8-11.
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

DDVR_ADJ_LAUNCHER(launch_adjoint_g2) {
  switch (mask) {
    case 8:
      if (cells) adj<8, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<8, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    case 9:
      if (cells) adj<9, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<9, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    case 10:
      if (cells) adj<10, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<10, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    case 11:
      if (cells) adj<11, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<11, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    default:
      break;
  }
}

}  // namespace ddvr_impl
