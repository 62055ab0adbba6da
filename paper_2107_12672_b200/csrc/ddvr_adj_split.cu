// ddvr_adj_split.cu -- segment-split instantiations of the fused step (dvr_adjoint_kernel
// with SPLIT > 1): TF-target masks without camera / stepsize, for steps with too few rays
// to fill the GPU one thread per ray (C1: 16 K rays).  See the kernel comment.
#include "ddvr_device.cuh"

namespace ddvr_impl {

template <unsigned M, int K>
static int adj_split(const Geometry& G, int n_views, size_t smem, cudaStream_t st,
                     const VolArgs& V, const TfArgs& T, float* dv, float* dcells,
                     const FusedArgs& fu) {
  auto k = dvr_adjoint_kernel<M, true, 0, true, false, K>;
  set_smem(k, smem);
  const dim3 grid((G.W + 7) / 8, (G.row1 - G.row0 + kThreads / K / 8 - 1) / (kThreads / K / 8),
                  n_views);
  k<<<grid, kThreads, smem, st>>>(V, T, G, nullptr, nullptr, nullptr, dv, dcells, nullptr,
                                  nullptr, fu);
  return 1;
}

template <unsigned M>
static int adj_split_k(int split, const Geometry& G, int n_views, size_t smem, cudaStream_t st,
                       const VolArgs& V, const TfArgs& T, float* dv, float* dcells,
                       const FusedArgs& fu) {
  switch (split) {
    case 2: return adj_split<M, 2>(G, n_views, smem, st, V, T, dv, dcells, fu);
    case 4: return adj_split<M, 4>(G, n_views, smem, st, V, T, dv, dcells, fu);
    case 8: return adj_split<M, 8>(G, n_views, smem, st, V, T, dv, dcells, fu);
    case 16: return adj_split<M, 16>(G, n_views, smem, st, V, T, dv, dcells, fu);
    default: return 0;
  }
}

int launch_adjoint_split(unsigned mask, int split, int n_views, size_t smem, cudaStream_t st,
                         const VolArgs& V, const TfArgs& T, const Geometry& G, float* dv,
                         float* dcells, const FusedArgs& fu) {
  if (mask == DDVR_TARGET_TF)
    return adj_split_k<DDVR_TARGET_TF>(split, G, n_views, smem, st, V, T, dv, dcells, fu);
  if (mask == (DDVR_TARGET_TF | DDVR_TARGET_VOLUME))
    return adj_split_k<DDVR_TARGET_TF | DDVR_TARGET_VOLUME>(split, G, n_views, smem, st, V, T,
                                                            dv, dcells, fu);
  return 0;
}

}  // namespace ddvr_impl
