// ddvr_fwd.cu -- instantiations of the forward march kernel (see ddvr_device.cuh).
#include "ddvr_device.cuh"

namespace ddvr_impl {

template <bool EARLY, bool CELLS, bool TAPE>
static void fwd(dim3 grid, size_t smem, cudaStream_t st, const VolArgs& V, const TfArgs& T,
                const Geometry& G, float* image, float* depth) {
  auto k = dvr_forward_kernel<EARLY, CELLS, TAPE>;
  set_smem(k, smem);
  k<<<grid, kThreads, smem, st>>>(V, T, G, image, depth);
}

void launch_forward(bool early, bool cells, bool tape, dim3 grid, size_t smem, cudaStream_t st,
                    const VolArgs& V, const TfArgs& T, const Geometry& G, float* image,
                    float* depth) {
#define DDVR_FWD(E, C, P) \
  if (early == E && cells == C && tape == P) fwd<E, C, P>(grid, smem, st, V, T, G, image, depth);
  DDVR_FWD(false, false, false) DDVR_FWD(false, false, true) DDVR_FWD(false, true, false)
  DDVR_FWD(false, true, true) DDVR_FWD(true, false, false) DDVR_FWD(true, false, true)
  DDVR_FWD(true, true, false) DDVR_FWD(true, true, true)
#undef DDVR_FWD
}

}  // namespace ddvr_impl
