// k_step.cu — instantiations of the single-launch step kernel (attention.cuh
// step_mma_kernel: every FULL item with its select fused, then every REUSE item).
#include "launch.cuh"

namespace hylra {
namespace host {

// Its parameters stay within the classic 4 KB kernel-parameter space.
static_assert(2 * sizeof(CUtensorMap) + 2 * sizeof(AttnParams) + sizeof(SelectParams) +
                      sizeof(StepSync) <= 4096,
              "step_mma_kernel parameters exceed 4 KB");

template <int D, bool GBIG>
static cudaError_t launch_step(int n_items, cudaStream_t st, const CUtensorMap& tk,
                               const CUtensorMap& tv, const AttnParams& pf, const AttnParams& pr,
                               const SelectParams& sp, const StepSync& ss) {
  constexpr int S = mma_stages<D, true, GBIG>();
  auto kern = step_mma_kernel<D, GBIG, S>;
  constexpr size_t smem = mma_smem_bytes<D, true, GBIG>();
  if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem)) return e;
  return launch_pdl(kern, dim3(n_items), dim3(attn_threads<true>()), smem, st, tk, tv, pf, pr, sp,
                    ss);
}

cudaError_t run_step_mma(int D, bool big, int n_items, cudaStream_t st, const CUtensorMap& tk,
                         const CUtensorMap& tv, const AttnParams& pf, const AttnParams& pr,
                         const SelectParams& sp, const StepSync& ss) {
  if (D == 128) return big ? launch_step<128, true>(n_items, st, tk, tv, pf, pr, sp, ss)
                           : launch_step<128, false>(n_items, st, tk, tv, pf, pr, sp, ss);
  if (D == 64) return big ? launch_step<64, true>(n_items, st, tk, tv, pf, pr, sp, ss)
                          : launch_step<64, false>(n_items, st, tk, tv, pf, pr, sp, ss);
  return cudaErrorInvalidValue;
}

}  // namespace host
}  // namespace hylra

#ifdef HYLRA_TRACE
// diagnostics build only: the per-CTA trace buffer of the single-launch kernel (8 x int64
// per ticket) and the fused selects' phase records, or NULL (the device symbols live in this
// translation unit, with the kernel that writes them)
extern "C" int hylra_trace_set(void* buf) {
  return cudaMemcpyToSymbol(hylra::g_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : 5;
}
extern "C" int hylra_trace_set_select_info(void* buf) {
  return cudaMemcpyToSymbol(hylra::g_sel_info, &buf, sizeof(buf)) == cudaSuccess ? 0 : 5;
}
#endif
