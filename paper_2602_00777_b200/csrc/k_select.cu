// k_select.cu — instantiations of the standalone top-k SELECT kernels: select.cuh
// topk_select_kernel<NT> (one CTA per row) and rowsel.cuh rowsel_kernel<C> (one C-CTA
// cluster per row, the row resident in shared memory).
#include <algorithm>

#include "launch.cuh"

namespace hylra {
namespace host {

template <int NT>
static cudaError_t launch_select_nt(dim3 grid, size_t smem, cudaStream_t st,
                                    const SelectParams& p) {
  const size_t most = std::max(sel_smem_bytes(kSelMaxTokens, NT),
                               sel_hist_smem_bytes(kSelMaxTokens, NT));
  if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(topk_select_kernel<NT>),
                                      most))
    return e;
  return launch_pdl(topk_select_kernel<NT>, grid, dim3(NT), smem, st, p);
}

cudaError_t run_select(int nt, dim3 grid, size_t smem, cudaStream_t st, const SelectParams& p) {
  switch (nt) {
    case 1024: return launch_select_nt<1024>(grid, smem, st, p);
    case 512: return launch_select_nt<512>(grid, smem, st, p);
    case 256: return launch_select_nt<256>(grid, smem, st, p);
    case 128: return launch_select_nt<128>(grid, smem, st, p);
    default: return cudaErrorInvalidValue;
  }
}

// rowsel_kernel<C>: one C-CTA cluster per row (C = 1 is an ordinary launch), with
// programmatic dependent launch like every other kernel of the step.
template <int C>
static cudaError_t launch_rowsel_c(int slice, dim3 grid, size_t smem, cudaStream_t st,
                                   const SelectParams& p) {
  if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(rowsel_kernel<C>),
                                      rowsel_smem_bytes(kRowselMaxSlice)))
    return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kRowselThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (C > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = C;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, rowsel_kernel<C>, p, slice);
}

cudaError_t run_rowsel(int cluster, int slice, dim3 grid, size_t smem, cudaStream_t st,
                       const SelectParams& p) {
  switch (cluster) {
    case 1: return launch_rowsel_c<1>(slice, grid, smem, st, p);
    case 2: return launch_rowsel_c<2>(slice, grid, smem, st, p);
    case 4: return launch_rowsel_c<4>(slice, grid, smem, st, p);
    case 8: return launch_rowsel_c<8>(slice, grid, smem, st, p);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace host
}  // namespace hylra
