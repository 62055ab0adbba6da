// ddvr_adj_g3.cu -- adjoint kernel instantiations for target masks 12-15.
#include "ddvr_device.cuh"

namespace ddvr_impl {

template <unsigned M, bool CELLS, bool FUSED>
static int adj2(dim3 grid, size_t smem, cudaStream_t st, const VolArgs& V, const TfArgs& T,
                const Geometry& G, const float* image, const float* depth, const float* seed,
                float* dv, float* dcells, double* dcam, double* ddt,
                const FusedArgs& fu) {
  auto k = dvr_adjoint_kernel<M, CELLS, 0, FUSED>;
  set_smem(k, smem);
  k<<<grid, kThreads, smem, st>>>(V, T, G, image, depth, seed, dv, dcells, dcam, ddt, fu);
  if constexpr (CELLS && !(M & DDVR_TARGET_TF)) {   // the absorption-only walk
    auto k1 = dvr_adjoint_kernel<M, CELLS, 1, FUSED>;
    set_smem(k1, smem);
    k1<<<grid, kThreads, smem, st>>>(V, T, G, image, depth, seed, dv, dcells, dcam, ddt, fu);
    return 2;
  }
  return 1;
}

// fused (forward + L1 seed + adjoint) kernels exist for the cell layout only
template <unsigned M, bool CELLS>
static int adj(dim3 grid, size_t smem, cudaStream_t st, const VolArgs& V, const TfArgs& T,
               const Geometry& G, const float* image, const float* depth, const float* seed,
               float* dv, float* dcells, double* dcam, double* ddt,
               const FusedArgs* fu) {
  if (fu) {
    if constexpr (CELLS)
      return adj2<M, true, true>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dcam,
                                 ddt, *fu);
    return 0;
  }
  return adj2<M, CELLS, false>(grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dcam,
                               ddt, FusedArgs{});
}

#define DDVR_ADJ_ARGS grid, smem, st, V, T, G, image, depth, seed, dv, dcells, dcam, ddt, fu
DDVR_ADJ_LAUNCHER(launch_adjoint_g3) {
  switch (mask) {
    case 12:
      return cells ? adj<12, true>(DDVR_ADJ_ARGS) : adj<12, false>(DDVR_ADJ_ARGS);
    case 13:
      return cells ? adj<13, true>(DDVR_ADJ_ARGS) : adj<13, false>(DDVR_ADJ_ARGS);
    case 14:
      return cells ? adj<14, true>(DDVR_ADJ_ARGS) : adj<14, false>(DDVR_ADJ_ARGS);
    case 15:
      return cells ? adj<15, true>(DDVR_ADJ_ARGS) : adj<15, false>(DDVR_ADJ_ARGS);
    default:
      return 0;
  }
}

#undef DDVR_ADJ_ARGS

}  // namespace ddvr_impl
