// launch.cuh — host-side launch plumbing shared by the translation units of libhylra.so:
// per-device attributes and SM count, programmatic dependent launch, and the entry points
// of the kernel translation units (k_full.cu, k_reuse.cu, k_simt.cu, k_step.cu, k_select.cu).
// Each kernel template is instantiated in exactly one of those units so the library builds
// in parallel; hylra_abi.cu holds the host logic and the extern "C" surface.
#pragma once

#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "attention.cuh"
#include "select.cuh"
#include "rowsel.cuh"

namespace hylra {
namespace host {

// Per-device facts and function attributes. The library may drive several devices from one
// process (one host thread per GPU, or one thread switching devices), so nothing
// device-specific is cached per process: the SM count is read from the current device and
// the dynamic shared-memory opt-in (cudaFuncSetAttribute applies per device context) is
// made once per (kernel, device).
inline int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    dev = 0;
  }
  return dev;
}

inline int num_sms() {
  static std::mutex mu;
  static std::map<int, int> sms;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  auto it = sms.find(dev);
  if (it != sms.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 148;  // B200; only reached without a usable device (the launch then fails loudly)
  }
  sms[dev] = n;
  return n;
}

inline cudaError_t ensure_smem_attr(const void* func, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  const auto key = std::make_pair(func, current_device());
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= smem) return cudaSuccess;
  const cudaError_t e =
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) done[key] = smem;
  return e;
}
// Clusters of more than 8 CTAs (the portable limit) need the kernel's opt-in, per device.
inline cudaError_t ensure_nonportable_cluster(const void* func) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, bool> done;
  const auto key = std::make_pair(func, current_device());
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(key)) return cudaSuccess;
  const cudaError_t e =
      cudaFuncSetAttribute(func, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) done[key] = true;
  return e;
}
// ------------------------------------------------------------------ launches
// Programmatic dependent launch for the step's kernels (FULL, SELECT, REUSE): each may be
// scheduled while its predecessor drains (the kernels wait on griddepcontrol before
// touching memory). HYLRA_PDL=0 turns it off.
inline bool pdl_enabled() {
  static int v = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = std::getenv("HYLRA_PDL");
    v = (e && *e) ? (atoi(e) != 0) : 1;
  });
  return v == 1;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// The same, launched as clusters of cluster_x CTAs along x (1: no cluster attribute).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                               cudaStream_t st, int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// REUSE split-K merge through a CTA cluster's shared memory (default on; env
// HYLRA_CLUSTER_MERGE, tuning knob "cluster_merge")
inline bool cluster_merge_enabled();

// ------------------------------------------------------------------ kernel tables
template <int D, bool GATHER, bool GBIG>
constexpr int mma_stages() {
  return D == 128 ? 3 : 5;
}
template <int D, bool GATHER, bool GBIG>
constexpr size_t mma_smem_bytes() {
  // + the REUSE index staging area, which FULL CTAs use for the score-row histogram, and
  // the FULL CTAs' per-stage score buffers (attention.cuh attn_mma_item)
  return (size_t)mma_stages<D, GATHER, GBIG>() * MmaSmem<D>::kStageBytes + 1024 + 256 +
         kIdxStage * sizeof(int32_t) + 2 * mma_stages<D, GATHER, GBIG>() * kTileRows * 4;
}

// Kernel-unit entry points (each defined in its own translation unit).
cudaError_t run_attn_mma(int D, bool gather, bool big, dim3 grid, cudaStream_t st,
                         const CUtensorMap& tk, const CUtensorMap& tv, const AttnParams& p,
                         const SelectParams& sp);
cudaError_t run_attn_simt(bool f32, bool gather, int D, int G, dim3 grid, cudaStream_t st,
                          const AttnParams& p);
cudaError_t run_step_mma(int D, bool big, int n_items, cudaStream_t st, const CUtensorMap& tk,
                         const CUtensorMap& tv, const AttnParams& pf, const AttnParams& pr,
                         const SelectParams& sp, const StepSync& ss);
cudaError_t run_select(int nt, dim3 grid, size_t smem, cudaStream_t st, const SelectParams& p);
cudaError_t run_rowsel(int cluster, int slice, dim3 grid, size_t smem, cudaStream_t st,
                       const SelectParams& p);

// Process-wide tuning overrides set through hylra_set_tuning (-1: the environment /
// automatic rule applies).
struct Tuning {
  std::atomic<int> rowsel{-1};
  std::atomic<int> select_threads{-1};
  std::atomic<int> rowsel_cluster{-1};
  std::atomic<int> gather_tma{-1};
  std::atomic<int> bulk_merge{-1};
  std::atomic<int> cluster_merge{-1};
  std::atomic<int> reuse_prefetch{-1};
  std::atomic<int> fused_fine_splits{-1};
};
inline Tuning& tuning() {
  static Tuning t;
  return t;
}

// The shared-memory-resident select (rowsel.cuh) for the rows it covers; HYLRA_ROWSEL=0
// (or hylra_set_tuning("rowsel", 0)) keeps every row on select_row (A/B runs).
// REUSE launches gather rows by TMA (tile::gather4) instead of cp.async where the cache is
// contiguous; HYLRA_GATHER_TMA / hylra_set_tuning("gather_tma", v) (default: off).
// split-K final merge stages the partials by cp.async.bulk (default on; env HYLRA_BULK_MERGE)
inline bool bulk_merge_enabled() {
  const int o = tuning().bulk_merge.load(std::memory_order_relaxed);
  if (o >= 0) return o != 0;
  static int v = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = std::getenv("HYLRA_BULK_MERGE");
    v = (e && *e) ? (atoi(e) != 0) : 1;
  });
  return v != 0;
}
inline bool cluster_merge_enabled() {
  const int o = tuning().cluster_merge.load(std::memory_order_relaxed);
  if (o >= 0) return o != 0;
  static int v = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = std::getenv("HYLRA_CLUSTER_MERGE");
    v = (e && *e) ? (atoi(e) != 0) : 1;
  });
  return v != 0;
}
inline bool gather_tma_enabled() {
  const int o = tuning().gather_tma.load(std::memory_order_relaxed);
  if (o >= 0) return o != 0;
  static int v = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = std::getenv("HYLRA_GATHER_TMA");
    v = (e && *e) ? (atoi(e) != 0) : 0;
  });
  return v == 1;
}

inline bool rowsel_enabled() {
  const int o = tuning().rowsel.load(std::memory_order_relaxed);
  if (o >= 0) return o != 0;
  static int v = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = std::getenv("HYLRA_ROWSEL");
    v = (e && *e) ? (atoi(e) != 0) : 1;
  });
  return v == 1;
}

}  // namespace host
}  // namespace hylra
