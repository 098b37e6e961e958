// k_reuse.cu — instantiations of the REUSE tensor-core kernel (attention.cuh attn_mma_kernel
// with GATHER = true: cp.async row gather of the selected rows, subset softmax) and the
// dispatcher of both tensor-core families.
#include "launch.cuh"

namespace hylra {
namespace host {

cudaError_t run_full_mma(int D, bool big, dim3 grid, cudaStream_t st, const CUtensorMap& tk,
                         const CUtensorMap& tv, const AttnParams& p, const SelectParams& sp);

template <int D, bool GBIG>
static cudaError_t launch_reuse(dim3 grid, cudaStream_t st, const CUtensorMap& tk,
                                const CUtensorMap& tv, const AttnParams& p,
                                const SelectParams& sp) {
  constexpr int S = mma_stages<D, true, GBIG>();
  auto kern = attn_mma_kernel<D, true, GBIG, S>;
  constexpr size_t smem = mma_smem_bytes<D, true, GBIG>();
  if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem)) return e;
  if (p.cluster_merge > 8)
    if (cudaError_t e = ensure_nonportable_cluster(reinterpret_cast<const void*>(kern))) return e;
  return launch_pdl_cluster(kern, grid, dim3(attn_threads<true>()), smem, st, p.cluster_merge,
                            tk, tv, p, sp);
}

cudaError_t run_attn_mma(int D, bool gather, bool big, dim3 grid, cudaStream_t st,
                         const CUtensorMap& tk, const CUtensorMap& tv, const AttnParams& p,
                         const SelectParams& sp) {
  if (!gather) return run_full_mma(D, big, grid, st, tk, tv, p, sp);
  if (D == 128) return big ? launch_reuse<128, true>(grid, st, tk, tv, p, sp)
                           : launch_reuse<128, false>(grid, st, tk, tv, p, sp);
  if (D == 64) return big ? launch_reuse<64, true>(grid, st, tk, tv, p, sp)
                          : launch_reuse<64, false>(grid, st, tk, tv, p, sp);
  return cudaErrorInvalidValue;
}

}  // namespace host
}  // namespace hylra

#ifdef HYLRA_TRACE
extern "C" int hylra_trace_set_reuse(void* buf) {
  return cudaMemcpyToSymbol(hylra::g_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : 5;
}
#endif
