// ddvr_adj_g3.cu -- adjoint kernel instantiations for target masks 12-15.
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

DDVR_ADJ_LAUNCHER(launch_adjoint_g3) {
  switch (mask) {
    case 12:
      if (cells) adj<12, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<12, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    case 13:
      if (cells) adj<13, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<13, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    case 14:
      if (cells) adj<14, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<14, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    case 15:
      if (cells) adj<15, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      else adj<15, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dtf, dcam, ddt);
      break;
    default:
      break;
  }
}

}  // namespace ddvr_impl
