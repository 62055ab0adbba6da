// ddvr_adj_split.cu -- segment-split instantiations of the fused step (dvr_adjoint_kernel
// with SPLIT > 1): TF-target masks without camera / stepsize, for steps with too few rays
// to fill the GPU one thread per ray (C1: 16 K rays), and the camera / stepsize masks
// (forced by DDVR_FLAG_RAY_SPLIT_2 / _4).  See the kernel comment.
#include "ddvr_device.cuh"

namespace ddvr_impl {

template <unsigned M, int K>
static int adj_split(const Geometry& G, int n_views, size_t smem, cudaStream_t st,
                     const VolArgs& V, const TfArgs& T, float* dv, float* dcells,
                     double* dcam, double* ddt, const FusedArgs& fu) {
  auto k = dvr_adjoint_kernel<M, true, 0, true, false, K>;
  set_smem(k, smem);
  const dim3 grid((G.W + 7) / 8, (G.row1 - G.row0 + kThreads / K / 8 - 1) / (kThreads / K / 8),
                  n_views);
  k<<<grid, kThreads, smem, st>>>(V, T, G, nullptr, nullptr, nullptr, dv, dcells, dcam, ddt,
                                  fu);
  return 1;
}

#define DDVR_SPLIT_ARGS G, n_views, smem, st, V, T, dv, dcells, dcam, ddt, fu
template <unsigned M>
static int adj_split_k(int split, const Geometry& G, int n_views, size_t smem, cudaStream_t st,
                       const VolArgs& V, const TfArgs& T, float* dv, float* dcells,
                       double* dcam, double* ddt, const FusedArgs& fu) {
  constexpr bool kPos = M & (DDVR_TARGET_CAMERA | DDVR_TARGET_STEPSIZE);
  switch (split) {   // (camera / stepsize walks: 2 and 4 lanes per ray)
    case 2: return adj_split<M, 2>(DDVR_SPLIT_ARGS);
    case 4: return adj_split<M, 4>(DDVR_SPLIT_ARGS);
    case 8: if constexpr (!kPos) return adj_split<M, 8>(DDVR_SPLIT_ARGS); return 0;
    case 16: if constexpr (!kPos) return adj_split<M, 16>(DDVR_SPLIT_ARGS); return 0;
    default: return 0;
  }
}

int launch_adjoint_split(unsigned mask, int split, int n_views, size_t smem, cudaStream_t st,
                         const VolArgs& V, const TfArgs& T, const Geometry& G, float* dv,
                         float* dcells, double* dcam, double* ddt, const FusedArgs& fu) {
  constexpr unsigned kC = DDVR_TARGET_CAMERA, kS = DDVR_TARGET_STEPSIZE;
  switch (mask) {
    case DDVR_TARGET_TF:
      return adj_split_k<DDVR_TARGET_TF>(split, DDVR_SPLIT_ARGS);
    case DDVR_TARGET_TF | DDVR_TARGET_VOLUME:
      return adj_split_k<DDVR_TARGET_TF | DDVR_TARGET_VOLUME>(split, DDVR_SPLIT_ARGS);
    case kC: return adj_split_k<kC>(split, DDVR_SPLIT_ARGS);
    case kS: return adj_split_k<kS>(split, DDVR_SPLIT_ARGS);
    case kC | kS: return adj_split_k<kC | kS>(split, DDVR_SPLIT_ARGS);
    default: return 0;
  }
}
#undef DDVR_SPLIT_ARGS

}  // namespace ddvr_impl
