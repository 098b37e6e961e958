// k_full.cu — instantiations of the FULL tensor-core kernel (attention.cuh attn_mma_kernel
// with GATHER = false: TMA-streamed split-K flash-decode with fused score emission and the
// optional fused select), one translation unit so the library builds in parallel.
#include "launch.cuh"

namespace hylra {
namespace host {

template <int D, bool GBIG>
static cudaError_t launch_full(dim3 grid, cudaStream_t st, const CUtensorMap& tk,
                               const CUtensorMap& tv, const AttnParams& p, const SelectParams& sp) {
  constexpr int S = mma_stages<D, false, GBIG>();
  auto kern = attn_mma_kernel<D, false, GBIG, S>;
  constexpr size_t smem = mma_smem_bytes<D, false, GBIG>();
  if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem)) return e;
  return launch_pdl(kern, grid, dim3(attn_threads<false>()), smem, st, tk, tv, p, sp);
}

cudaError_t run_full_mma(int D, bool big, dim3 grid, cudaStream_t st, const CUtensorMap& tk,
                         const CUtensorMap& tv, const AttnParams& p, const SelectParams& sp) {
  if (D == 128) return big ? launch_full<128, true>(grid, st, tk, tv, p, sp)
                           : launch_full<128, false>(grid, st, tk, tv, p, sp);
  if (D == 64) return big ? launch_full<64, true>(grid, st, tk, tv, p, sp)
                          : launch_full<64, false>(grid, st, tk, tv, p, sp);
  return cudaErrorInvalidValue;
}

}  // namespace host
}  // namespace hylra

#ifdef HYLRA_TRACE
// diagnostics build only: per-CTA trace rows of the standalone FULL / REUSE launches (this
// translation unit's copy of the trace symbol; scripts/trace_layer.py)
extern "C" int hylra_trace_set_full(void* buf) {
  return cudaMemcpyToSymbol(hylra::g_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : 5;
}
#endif
