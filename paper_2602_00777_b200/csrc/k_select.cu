// k_select.cu — instantiations of the standalone top-k SELECT kernel (select.cuh
// topk_select_kernel<NT>, one CTA per row).
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

}  // namespace host
}  // namespace hylra
