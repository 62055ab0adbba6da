// ddvr_adj_g2.cu -- adjoint kernel instantiations for target masks 8-11.
#include "ddvr_device.cuh"

namespace ddvr_impl {

template <unsigned M, bool CELLS, bool FUSED, bool DET = false>
static int adj2(dim3 grid, size_t smem, cudaStream_t st, const VolArgs& V, const TfArgs& T,
                const Geometry& G, const float* image, const float* depth, const float* seed,
                float* dv, float* dcells, double* dcam, double* ddt,
                const FusedArgs& fu) {
  // the deterministic density gradient (int64 cell moments) has its own instantiations
  // for the volume target alone (the flush's conversions would cost registers elsewhere)
  if constexpr (M == DDVR_TARGET_VOLUME && CELLS && !DET) {
    if (V.cells64)
      return adj2<M, CELLS, FUSED, true>(grid, smem, st, V, T, G, image, depth, seed, dv,
                                         dcells, dcam, ddt, fu);
  }
  auto k = dvr_adjoint_kernel<M, CELLS, 0, FUSED, DET>;
  set_smem(k, smem);
  k<<<grid, kThreads, smem, st>>>(V, T, G, image, depth, seed, dv, dcells, dcam, ddt, fu);
  if constexpr (CELLS && !(M & DDVR_TARGET_TF)) {   // the absorption-only walk
    auto k1 = dvr_adjoint_kernel<M, CELLS, 1, FUSED, DET>;
    set_smem(k1, smem);
    k1<<<grid, kThreads, smem, st>>>(V, T, G, image, depth, seed, dv, dcells, dcam, ddt, fu);
    if constexpr (M == DDVR_TARGET_VOLUME && FUSED) {
      if (G.ray_k) {   // the band-tape step as march + walk kernels (ROLE 1 returns for it)
        set_smem(dvr_band_march_kernel<0>, smem);
        dvr_band_march_kernel<0><<<grid, kThreads, smem, st>>>(V, T, G, fu);
        set_smem(dvr_band_walk_kernel<DET>, smem);
        dvr_band_walk_kernel<DET><<<grid, kThreads, smem, st>>>(V, T, G, dcells);
        return 4;
      }
    }
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
DDVR_ADJ_LAUNCHER(launch_adjoint_g2) {
  switch (mask) {
    case 8:
      return cells ? adj<8, true>(DDVR_ADJ_ARGS) : adj<8, false>(DDVR_ADJ_ARGS);
    case 9:
      return cells ? adj<9, true>(DDVR_ADJ_ARGS) : adj<9, false>(DDVR_ADJ_ARGS);
    case 10:
      return cells ? adj<10, true>(DDVR_ADJ_ARGS) : adj<10, false>(DDVR_ADJ_ARGS);
    case 11:
      return cells ? adj<11, true>(DDVR_ADJ_ARGS) : adj<11, false>(DDVR_ADJ_ARGS);
    default:
      return 0;
  }
}

#undef DDVR_ADJ_ARGS

}  // namespace ddvr_impl
