// k_simt.cu — instantiations of the CUDA-core attention kernel (attention.cuh
// attn_simt_kernel): fp32 caches (the reference-precision path) and head_dim 32.
#include "launch.cuh"

namespace hylra {
namespace host {

template <typename T, int D, int GM, bool GATHER>
static cudaError_t launch_simt(dim3 grid, cudaStream_t st, const AttnParams& p) {
  attn_simt_kernel<T, D, GM, GATHER><<<grid, 128, 0, st>>>(p);
  return cudaGetLastError();
}

template <typename T, bool GATHER>
static cudaError_t dispatch_simt(int D, int G, dim3 grid, cudaStream_t st, const AttnParams& p) {
#define HY_SIMT_D(DD)                                                  \
  if (D == DD) {                                                       \
    if (G <= 1) return launch_simt<T, DD, 1, GATHER>(grid, st, p);     \
    if (G <= 4) return launch_simt<T, DD, 4, GATHER>(grid, st, p);     \
    if (G <= 8) return launch_simt<T, DD, 8, GATHER>(grid, st, p);     \
    return launch_simt<T, DD, 16, GATHER>(grid, st, p);                \
  }
  HY_SIMT_D(32)
  HY_SIMT_D(64)
  HY_SIMT_D(128)
#undef HY_SIMT_D
  return cudaErrorInvalidValue;
}

cudaError_t run_attn_simt(bool f32, bool gather, int D, int G, dim3 grid, cudaStream_t st,
                          const AttnParams& p) {
  if (f32)
    return gather ? dispatch_simt<float, true>(D, G, grid, st, p)
                  : dispatch_simt<float, false>(D, G, grid, st, p);
  return gather ? dispatch_simt<__nv_bfloat16, true>(D, G, grid, st, p)
                : dispatch_simt<__nv_bfloat16, false>(D, G, grid, st, p);
}

}  // namespace host
}  // namespace hylra
