// hylra_abi.cu — extern "C" entry points of libhylra.so (declared in include/hylra.h).
//
// Host side of the drop-in boundary: validates shapes (ConfigurationError /
// InvalidInputError, reference errors.py:4-21), picks the kernel family, sizes the
// split-K grid for the device's SM count, encodes the TMA tensor maps and enqueues on the caller's
// stream. No allocation, no synchronisation, no retained state besides cached
// function attributes.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/hylra.h"
#include "append.cuh"
#include "blocks.cuh"
#include "launch.cuh"
#include "overlap.cuh"

using namespace hylra;
using namespace hylra::host;

namespace {

constexpr size_t kHeader = 256;
// REUSE L2 prefetch distance in 64-row tiles. Swept on B200 at cfg2 B=8 once the CTA's
// indices are staged in shared memory: 0/1/2/3/4/6/8/12/16 tiles -> 305.6/307.0/311.1/
// 314.8/318.5/329.8/338.5/346.9/347.9 us (before staging, 2 tiles won: 306 vs 345 us).
constexpr int kReusePrefetchTiles = 0;

thread_local char g_err[512] = "";
std::atomic<uint64_t> g_launches{0};

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(HYLRA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return HYLRA_OK;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int scores_row_stride(const hylra_geometry* g) { return (g->capacity + 7) & ~7; }

int check_geometry(const hylra_geometry* g) {
  if (g == nullptr) return fail(HYLRA_ERR_CONFIGURATION, "geometry is NULL");
  if (g->batch < 1 || g->q_heads < 1 || g->kv_heads < 1 || g->capacity < 1 || g->num_layers < 1)
    return fail(HYLRA_ERR_CONFIGURATION, "non-positive dimension in geometry");
  if (g->q_heads % g->kv_heads != 0)
    return fail(HYLRA_ERR_CONFIGURATION, "q_heads %d is not a multiple of kv_heads %d", g->q_heads,
                g->kv_heads);
  const int G = g->q_heads / g->kv_heads;
  if (G > kMaxG) return fail(HYLRA_ERR_CONFIGURATION, "group size %d exceeds %d", G, kMaxG);
  if (g->head_dim != 32 && g->head_dim != 64 && g->head_dim != 128)
    return fail(HYLRA_ERR_CONFIGURATION, "head_dim %d not in {32, 64, 128}", g->head_dim);
  if (g->dtype != HYLRA_BF16 && g->dtype != HYLRA_F32)
    return fail(HYLRA_ERR_CONFIGURATION, "unknown dtype %d", g->dtype);
  return HYLRA_OK;
}

// Split-K sizing: how many CTAs (splits) share one (layer, b, kv-head) pair's rows.
// Rules from B200 sweeps of cfg2 shapes at B = 1/4/8 (scripts/split_sweep.py; 2 CTAs of
// the attention kernel are resident per SM, S = 296 slots):
//  * a CTA pays a fixed cost (pipeline fill, q load, split merge), and with ~25 GB/s per
//    CTA (3-stage ring) a partial last wave runs almost as long as a full one;
//  * REUSE, at most one wave of pairs: split only up to one wave of >= 8-tile splits
//    (B=1 24 layers: 65.7 us at 8 splits/pair -> 45.3 at 1; B=1 5 layers: 16.6 at 4);
//  * REUSE, 1-4 waves of pairs: unsplit unless that leaves a nearly empty last wave
//    (B=4 24 layers: 145 us unsplit vs 155 at 4; B=8 5 layers, 1.08 waves: 83 us
//    unsplit -> 76 at 4 splits);
//  * REUSE, >= 4 waves of pairs: unsplit 32-tile units (B=8 24 layers: 259 vs 265-270 us
//    at 2 splits); "pairs" above count 32-tile units of a pair (longer selections start
//    out split);
//  * FULL: ~4 waves of >= 32-tile splits, or up to one wave of shorter splits when
//    rows are few (B=1: 186.5 -> 168.8 us).
// HYLRA_{FULL,REUSE}_{WAVES,MIN_TILES} replace a rule by "waves x S CTAs, >= min tiles
// per split" for tuning experiments.
int splits_by_waves(int pairs, int tiles, int waves, int min_tiles) {
  const int kSlots = 2 * num_sms();
  int s = (kSlots * waves + pairs - 1) / pairs;
  return std::min(s, std::max(1, tiles / min_tiles));
}

// REUSE launches under one wave of 32-tile units: the smallest split (tiles per CTA; 4:
// one-layer REUSE at cfg2 B=1 in the layer-sequential step, 4 vs 8 tiles: 576 vs 619 us/step);
// HYLRA_REUSE_SMALL_TILES overrides (A/B runs).
int small_reuse_tiles() {
  static int v = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = std::getenv("HYLRA_REUSE_SMALL_TILES");
    v = (e && *e) ? std::max(1, atoi(e)) : 4;
  });
  return v;
}

// Tuning knob "fused_fine_splits" (default off): FULL launches with fused selects (the
// fusedsel schedule) over few pairs take finer splits, so the pairs' final CTAs, which run
// the selects, finish staggered under the streaming of the other splits instead of together
// at the end. Measured: cfg2 B=1 fusedsel 220.7 -> 213.9 us, B=2 393 us (single 406), cfg4
// B=4 627 us (single 647). Off by default because the outputs then differ from the other
// schedules' at bf16 level (a different split partition rounds P = exp(s - m) to bf16
// against a different running max), and every batched schedule returns bit-identical
// outputs by design (tests/test_gpu_kernels.py, test_gpu_select.py).
constexpr int kFineMaxPairs = 64;

int choose_splits(int pairs, int tiles, bool gather, bool fine = false) {
  static int env[2][2];
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* n) {
      const char* v = std::getenv(n);
      return (v && *v) ? std::max(1, atoi(v)) : 0;
    };
    env[0][0] = get("HYLRA_FULL_WAVES");
    env[0][1] = get("HYLRA_FULL_MIN_TILES");
    env[1][0] = get("HYLRA_REUSE_WAVES");
    env[1][1] = get("HYLRA_REUSE_MIN_TILES");
  });
  const int* e = env[gather ? 1 : 0];
  const int kSlots = 2 * num_sms();  // 2 attention CTAs resident per SM
  int s;
  if (e[0] || e[1]) {
    s = splits_by_waves(pairs, tiles, e[0] ? e[0] : 8, e[1] ? e[1] : 4);
  } else if (!gather && fine && pairs <= kFineMaxPairs) {
    s = splits_by_waves(pairs, tiles, 8, 8);
  } else if (!gather) {
    s = splits_by_waves(pairs, tiles, 4, 32);
    // up to one full wave when the rows allow (never just over one: N=8K B=1 at 5 splits
    // = 320 CTAs took 60.7 us, at 4 = 256 CTAs 47.9 us)
    const int fill = std::max(1, kSlots / pairs);
    s = std::max(s, std::min(fill, std::max(1, tiles / 4)));
  } else {
    // REUSE: CTAs of at most 32 tiles (1 MiB of K/V at d=128) — the 128K config's 4096-row
    // selections at 64-tile CTAs left a long tail (300 -> 368 us)
    const int s0 = std::max(1, (tiles + 31) / 32);
    const long units = (long)pairs * s0;
    if (units >= 4l * kSlots) {
      // many waves of 32-tile units: unsplit. cfg2 B=8 (5.2 waves): REUSE 259 vs 265-270 us
      // at 2 splits, single-launch step 1453 vs 1474 us (once the producer warps staged the
      // indices together, the per-CTA start cost no longer favoured shorter units)
      s = s0;
    } else if (units <= kSlots) {
      // under one wave (few pairs: one layer, small batch): split down to kSmallReuseTiles-
      // tile CTAs, up to one wave (the final merge stages the split scales in shared memory,
      // so many splits cost little)
      s = std::max(s0, std::min(kSlots / pairs, tiles / small_reuse_tiles()));
    } else {
      const long full_waves = units / kSlots, rest = units % kSlots;
      s = (full_waves >= 2 || 2 * rest >= kSlots) ? s0
                                                  : std::max(s0, splits_by_waves(pairs, tiles, 4, 8));
    }
  }
  s = std::max(1, std::min(s, tiles));
  const int tps = (tiles + s - 1) / s;
  return (tiles + tps - 1) / tps;
}

bool use_mma_path(const hylra_geometry* g) {
  return g->dtype == HYLRA_BF16 && (g->head_dim == 64 || g->head_dim == 128);
}

struct AttnLayout {
  int pairs, splits, tiles, tps;
  size_t off_counters, off_ml, off_o, total;
};

// Split-K counters of one launch: one int per (layer slot, b, kv-head) pair, always sized for
// kMaxSlots slots so their place and extent depend on the geometry's B and Hkv only — never
// on n_valid, the row count or the layer count of a call. Counters are left zeroed by the
// merging CTA, but the float partials that follow them are not: were the counter region
// to move or grow between calls on one workspace, a counter could start on a stale partial
// and the merge would never fire.
size_t counter_region_bytes(const hylra_geometry* g) {
  return align_up(sizeof(int) * (size_t)kMaxSlots * g->batch * g->kv_heads, 256);
}

// ext_ctr: the counters live elsewhere (the decode step's fixed counter regions) and the
// layout holds only the partials
AttnLayout attn_layout(const hylra_geometry* g, int n_layers, int rows, bool gather,
                       bool ext_ctr = false, bool fine = false) {
  AttnLayout a{};
  const int G = g->q_heads / g->kv_heads;
  a.pairs = n_layers * g->batch * g->kv_heads;
  a.tiles = std::max(1, (rows + kTileRows - 1) / kTileRows);
  a.splits = choose_splits(a.pairs, a.tiles, gather, fine);
  a.tps = (a.tiles + a.splits - 1) / a.splits;
  const size_t parts = a.splits;  // partial slots per pair
  a.off_counters = ext_ctr ? 0 : kHeader;
  const size_t ctr_end = ext_ctr ? 0 : kHeader + counter_region_bytes(g);
  a.off_ml = align_up(ctr_end, 256);
  a.off_o = align_up(a.off_ml + sizeof(float) * 2 * (size_t)a.pairs * parts * G, 256);
  a.total = align_up(a.off_o + sizeof(float) * (size_t)a.pairs * parts * G * g->head_dim, 256);
  if (parts == 1) a.total = std::max<size_t>(ctr_end, 256);
  return a;
}

// ------------------------------------------------------------------ tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

int encode_kv_map(CUtensorMap* map, const hylra_geometry* g, const void* base, int kv_layers) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return fail(HYLRA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int D = g->head_dim;
  const cuuint64_t es = 2;  // bf16
  cuuint64_t dims[5] = {(cuuint64_t)D, (cuuint64_t)g->capacity, (cuuint64_t)g->kv_heads,
                        (cuuint64_t)g->batch, (cuuint64_t)kv_layers};
  // strides of dims 1..4 in bytes; size-1 dims get a harmless dense stride
  cuuint64_t st[4];
  st[0] = (cuuint64_t)D * es;
  st[1] = g->kv_heads > 1 ? (cuuint64_t)g->kv_stride_head * es : st[0] * g->capacity;
  st[2] = g->batch > 1 ? (cuuint64_t)g->kv_stride_batch * es : st[1] * g->kv_heads;
  st[3] = kv_layers > 1 ? (cuuint64_t)g->kv_stride_layer * es : st[2] * g->batch;
  for (int i = 0; i < 4; ++i)
    if (st[i] % 16 != 0 || st[i] >= (1ull << 40))
      return fail(HYLRA_ERR_CONFIGURATION, "KV stride %d (%llu B) not TMA-compatible", i,
                  (unsigned long long)st[i]);
  cuuint32_t box[5] = {64, (cuuint32_t)kTileRows, 1, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, st, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HYLRA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return HYLRA_OK;
}

// Validated AttnParams of one FULL or REUSE launch (or of one half of a single-launch step).
// 2-D row view [rows][D] of a contiguous [L][B][Hkv][cap][D] bf16 cache for the REUSE
// TMA gather (box: 64 columns x 1 row, 128-byte swizzle: the 4-row gathers land in the
// same swizzled tile layout as the FULL kernel's boxes).
int encode_row_view(CUtensorMap* map, const hylra_geometry* g, const void* base, int rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return fail(HYLRA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)g->head_dim, (cuuint64_t)rows};
  cuuint64_t st[1] = {(cuuint64_t)g->head_dim * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, st, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HYLRA_ERR_CUDA, "cuTensorMapEncodeTiled (rows) failed (%d)", (int)r);
  return HYLRA_OK;
}

int make_attn_params(AttnParams* pp, AttnLayout* lay_out, const hylra_geometry* g, bool gather,
                     const void* q, const void* k, const void* v, int n_valid, int n_rows,
                     int n_layers, const int32_t* layer_ids, const int32_t* src_slots,
                     const int32_t* idx, const int32_t* counts, int k_stride, int sel_group,
                     float* out, float* scores, void* ws, size_t ws_bytes, int* flags,
                     const int32_t* kv_layer_ids, int kv_layer_count, int* counters = nullptr,
                     bool fine = false) {
  if (int e = check_geometry(g)) return e;
  if (n_layers < 1 || n_layers > kMaxSlots)
    return fail(HYLRA_ERR_CONFIGURATION, "n_layers %d not in [1, %d]", n_layers, kMaxSlots);
  if (n_valid < 1 || n_valid > g->capacity)
    return fail(HYLRA_ERR_INVALID_INPUT, "n_valid %d not in [1, capacity=%d]", n_valid,
                g->capacity);
  if (n_rows < 1) return fail(HYLRA_ERR_INVALID_INPUT, "no rows to attend over");
  if (!q || !k || !v || !out || !ws || !layer_ids)
    return fail(HYLRA_ERR_CONFIGURATION, "NULL pointer argument");
  const AttnLayout lay = attn_layout(g, n_layers, n_rows, gather, counters != nullptr, fine);
  if (ws_bytes < lay.total)
    return fail(HYLRA_ERR_CONFIGURATION, "workspace %zu B < required %zu B", ws_bytes, lay.total);
  const int G = g->q_heads / g->kv_heads;
  AttnParams p{};
  p.q = q; p.k = k; p.v = v; p.out = out; p.scores = scores; p.idx = idx; p.counts = counts;
  uint8_t* w = static_cast<uint8_t*>(ws);
  p.counters = counters ? counters : reinterpret_cast<int*>(w + lay.off_counters);
  p.ws_ml = reinterpret_cast<float*>(w + lay.off_ml);
  p.ws_o = reinterpret_cast<float*>(w + lay.off_o);
  p.flags = flags;
  p.q_sl = g->q_stride_layer; p.q_sb = g->q_stride_batch;
  p.kv_sl = g->kv_stride_layer; p.kv_sb = g->kv_stride_batch; p.kv_sh = g->kv_stride_head;
  p.o_sl = g->out_stride_layer; p.o_sb = g->out_stride_batch;
  p.B = g->batch; p.Hkv = g->kv_heads; p.G = G;
  p.cap = scores_row_stride(g);
  p.n_valid = n_valid; p.n_rows = n_rows; p.n_slots = n_layers;
  p.splits = lay.splits; p.tiles_per_split = lay.tps;
  p.k_stride = k_stride; p.sel_group = sel_group > 0 ? sel_group : 1;
  p.n_groups = g->kv_heads / p.sel_group;
  p.inv_sqrt_d = (float)(1.0 / std::sqrt((double)g->head_dim));
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)g->head_dim));
  {
    const int o = tuning().reuse_prefetch.load(std::memory_order_relaxed);
    p.prefetch = o >= 0 ? o : kReusePrefetchTiles;
  }
  p.bulk_merge = bulk_merge_enabled() ? 1 : 0;
  const int n_kv = kv_layer_ids ? kv_layer_count : g->num_layers;
  for (int i = 0; i < n_layers; ++i) {
    if (layer_ids[i] < 0 || layer_ids[i] >= g->num_layers)
      return fail(HYLRA_ERR_CONFIGURATION, "layer id %d out of range", layer_ids[i]);
    p.layers[i] = layer_ids[i];
    p.kv_layers[i] = kv_layer_ids ? kv_layer_ids[i] : layer_ids[i];
    if (p.kv_layers[i] < 0 || p.kv_layers[i] >= n_kv)
      return fail(HYLRA_ERR_CONFIGURATION, "KV layer %d out of range", p.kv_layers[i]);
    p.src_slot[i] = src_slots ? src_slots[i] : 0;
  }
  *pp = p;
  *lay_out = lay;
  return HYLRA_OK;
}

int launch_attention(const hylra_geometry* g, bool gather, const void* q, const void* k,
                     const void* v, int n_valid, int n_rows, int n_layers,
                     const int32_t* layer_ids, const int32_t* src_slots, const int32_t* idx,
                     const int32_t* counts, int k_stride, int sel_group, float* out,
                     float* scores, void* ws, size_t ws_bytes, int* flags, cudaStream_t st,
                     const int32_t* kv_layer_ids = nullptr, int kv_layer_count = 0,
                     const SelectParams* fused = nullptr, int fuse_nslots = 0,
                     const int32_t* blk = nullptr, int blk_stride = 0, int blk_size = 0,
                     int* counters = nullptr, unsigned* hist = nullptr, int early = 0) {
  AttnParams p{};
  AttnLayout lay{};
  const bool fine = fused != nullptr && fuse_nslots > 0 && !gather && blk == nullptr &&
                    use_mma_path(g) &&
                    tuning().fused_fine_splits.load(std::memory_order_relaxed) > 0;
  if (int e = make_attn_params(&p, &lay, g, gather, q, k, v, n_valid, n_rows, n_layers, layer_ids,
                               src_slots, idx, counts, k_stride, sel_group, out, scores, ws,
                               ws_bytes, flags, kv_layer_ids, kv_layer_count, counters, fine))
    return e;
  p.early = early;
  // block-mode REUSE by TMA tiles of the selected blocks: REUSE split rules, the streaming
  // (TMA) kernel
  if (blk != nullptr) {
    if (!gather || !use_mma_path(g) || blk_size % kTileRows != 0 || scores != nullptr)
      return fail(HYLRA_ERR_CONFIGURATION, "block tiles need a tensor-core REUSE launch");
    p.blk = blk;
    p.blk_stride = blk_stride;
    p.blk_size = blk_size;
    gather = false;
  }
  const int G = g->q_heads / g->kv_heads;
  const int n_kv = kv_layer_ids ? kv_layer_count : g->num_layers;
  dim3 grid(lay.splits, g->kv_heads, g->batch * n_layers);
  cudaError_t ce;
  static const SelectParams no_select{};
  const SelectParams& sp = fused ? *fused : no_select;
  p.fuse_select = (fused && !gather && use_mma_path(g)) ? fuse_nslots : 0;
  // (a split's 16-bit histogram counters hold < 65536 tokens)
  p.hist = (!gather && scores != nullptr && p.tiles_per_split * kTileRows < 65536) ? hist
                                                                                : nullptr;
  if (use_mma_path(g)) {
    CUtensorMap tk{}, tv{};
    if (!gather) {
      if (int e = encode_kv_map(&tk, g, k, n_kv)) return e;
      if (int e = encode_kv_map(&tv, g, v, n_kv)) return e;
    } else if (gather_tma_enabled() && counts == nullptr &&
               lay.tps * kTileRows <= kIdxStage) {
      // the TMA row gather needs the cache contiguous across (layer, b, kv-head) blocks
      const int64_t blk = (int64_t)g->capacity * g->head_dim;
      const int64_t rows = (int64_t)n_kv * g->batch * g->kv_heads * g->capacity;
      const bool contiguous = (g->kv_heads == 1 || g->kv_stride_head == blk) &&
                              (g->batch == 1 || g->kv_stride_batch == blk * g->kv_heads) &&
                              (n_kv == 1 || g->kv_stride_layer == blk * g->kv_heads * g->batch);
      if (contiguous && rows < (1ll << 31) - 1) {
        if (int e = encode_row_view(&tk, g, k, (int)rows)) return e;
        if (int e = encode_row_view(&tv, g, v, (int)rows)) return e;
        p.gather_tma = 1;
        p.gather_rows = (int)rows;
        p.cap_rows = g->capacity;
      }
    }
    // a small REUSE launch split 2-16 ways (at most one CTA per SM): the splits of a pair as
    // one CTA cluster, merged through distributed shared memory (grid.x == splits). Larger
    // launches keep the global merge: clusters of 2-CTA SMs pack GPCs unevenly (cfg2 B=4,
    // 256 CTAs: 11.4 vs 10.1 us per layer-sequential REUSE layer)
    if (gather && !p.gather_tma && lay.splits >= 2 && lay.splits <= 16 &&
        (long)grid.x * grid.y * grid.z <= num_sms() && cluster_merge_enabled())
      p.cluster_merge = lay.splits;
    ce = run_attn_mma(g->head_dim, gather, G > 8, grid, st, tk, tv, p, sp);
  } else {
    ce = run_attn_simt(g->dtype == HYLRA_F32, gather, g->head_dim, G, grid, st, p);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_check(ce, gather ? "reuse_decode launch" : "full_decode launch");
}

// SELECT CTA width: one CTA per row; few rows (small batch) get wide CTAs so each row's
// passes finish sooner, many rows keep 256-thread CTAs (4 per SM, all rows resident).
// HYLRA_SELECT_THREADS overrides (256 / 512 / 1024) for tuning.
int select_threads(int rows) {
  static int forced = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* v = std::getenv("HYLRA_SELECT_THREADS");
    const int t = (v && *v) ? atoi(v) : 0;
    // 128 = the fused select's width (diagnostics: scripts/select_diag.py)
    forced = (t == 128 || t == 256 || t == 512 || t == 1024) ? t : 0;
  });
  const int o = tuning().select_threads.load(std::memory_order_relaxed);
  if (o == 128 || o == 256 || o == 512 || o == 1024) return o;
  if (forced) return forced;
  if (rows <= num_sms()) return 1024;
  if (rows <= 2 * num_sms()) return 512;
  return 256;
}

struct BlockRows {  // block mode: rows are pooled block scores
  int block_size = 1, n_tokens = 0, row_stride = 0;
  const float* tok_scores = nullptr;  // the token scores they were pooled from
};

// Validated SelectParams for n_slots score slots (shared by the SELECT kernel and the
// selection fused into the FULL kernel).
int build_select_params(SelectParams* out, const hylra_geometry* g, const float* scores,
                        int n_slots, int n_valid, int budget, int sel_group, const void* q,
                        const void* k, const int32_t* layer_ids, int32_t* idx, int k_stride,
                        int32_t* info, int* flags, const BlockRows& br,
                        const int32_t* kv_layer_ids, const int32_t* out_slots) {
  if (int e = check_geometry(g)) return e;
  if (budget < 1) return fail(HYLRA_ERR_INVALID_INPUT, "budget must be >= 1, got %d", budget);
  if (n_slots < 1 || n_slots > kMaxSlots)
    return fail(HYLRA_ERR_CONFIGURATION, "n_slots %d not in [1, %d]", n_slots, kMaxSlots);
  if (n_valid < 1 || n_valid > g->capacity)
    return fail(HYLRA_ERR_INVALID_INPUT, "n_valid %d not in [1, capacity=%d]", n_valid,
                g->capacity);
  if (sel_group < 1 || g->kv_heads % sel_group != 0)
    return fail(HYLRA_ERR_CONFIGURATION, "sel_group %d does not divide kv_heads %d", sel_group,
                g->kv_heads);
  const int k_eff = std::min(budget, n_valid);
  const bool blocks = br.block_size > 1;
  if (k_stride < k_eff)
    return fail(HYLRA_ERR_CONFIGURATION, "k_stride %d < selection size %d", k_stride, k_eff);
  if (n_valid > kSelMaxTokens)
    return fail(HYLRA_ERR_CONFIGURATION, "selection rows longer than %d tokens", kSelMaxTokens);
  if (!scores || !idx) return fail(HYLRA_ERR_CONFIGURATION, "NULL pointer argument");
  SelectParams p{};
  p.scores = scores; p.idx = idx; p.info = info; p.flags = flags;
  p.q = (q && k && layer_ids) ? q : nullptr;
  p.k = k;
  p.dtype = g->dtype;
  p.q_sl = g->q_stride_layer; p.q_sb = g->q_stride_batch;
  p.kv_sl = g->kv_stride_layer; p.kv_sb = g->kv_stride_batch; p.kv_sh = g->kv_stride_head;
  p.B = g->batch; p.Hkv = g->kv_heads; p.G = g->q_heads / g->kv_heads; p.D = g->head_dim;
  p.sel_group = sel_group; p.n_groups = g->kv_heads / sel_group;
  p.n_valid = n_valid; p.k_eff = k_eff; p.k_stride = k_stride;
  p.row_stride = blocks ? br.row_stride : scores_row_stride(g);
  p.pre_grouped = blocks ? 1 : 0;
  p.block_size = blocks ? br.block_size : 1;
  p.n_tokens = blocks ? br.n_tokens : n_valid;
  p.tok_scores = blocks ? br.tok_scores : nullptr;
  p.tok_row_stride = scores_row_stride(g);
  p.tau_rel = 1.0f / 4096.0f;
  for (int i = 0; i < n_slots; ++i) {
    const int l = layer_ids ? layer_ids[i] : 0;
    if (l < 0 || l >= g->num_layers)
      return fail(HYLRA_ERR_CONFIGURATION, "layer id %d out of range", l);
    p.layers[i] = l;
    p.kv_layers[i] = kv_layer_ids ? kv_layer_ids[i] : l;
    p.out_slot[i] = out_slots ? out_slots[i] : i;
  }
  *out = p;
  return HYLRA_OK;
}

int launch_select(const hylra_geometry* g, const float* scores, int n_slots, int n_valid,
                  int budget, int sel_group, const void* q, const void* k,
                  const int32_t* layer_ids, int32_t* idx, int k_stride, int32_t* info,
                  int* flags, cudaStream_t st, const BlockRows& br = BlockRows(),
                  const int32_t* kv_layer_ids = nullptr, const int32_t* out_slots = nullptr,
                  int force_nt = 0, int32_t* idx_mirror = nullptr, unsigned* hist = nullptr,
                  bool compact = false) {
  SelectParams p{};
  if (int e = build_select_params(&p, g, scores, n_slots, n_valid, budget, sel_group, q, k,
                                  layer_ids, idx, k_stride, info, flags, br, kv_layer_ids,
                                  out_slots))
    return e;
  p.idx_mirror = idx_mirror;
  p.hist = hist;
  cudaError_t ce;
  // token rows that fit a CTA cluster's shared memory take the shared-memory-resident
  // select (rowsel.cuh; same index sets) when the launch fits one wave of SMs (one CTA per
  // SM: with more rows the streaming select's 4 CTAs per SM win), unless a CTA width is
  // forced or the FULL kernel's row histograms must be consumed (HYLRA_ROWSEL=0: off;
  // hylra_set_tuning("rowsel", 1): whatever the row count)
  const int n_eff = br.block_size > 1 ? p.n_valid : n_valid;
  const int rows = p.n_groups * g->batch * n_slots;
  int csz = rowsel_cluster(n_eff);
  const int forced_rs = tuning().rowsel.load(std::memory_order_relaxed);
  if (csz > 0) {
    // few rows: spread each over more CTAs (the select is instruction-bound per SM), as
    // long as the whole launch stays within one wave of SMs
    const int forced = tuning().rowsel_cluster.load(std::memory_order_relaxed);
    if (forced == 1 || forced == 2 || forced == 4 || forced == 8) csz = std::max(csz, forced);
    else if (!compact)
      // (compact: a select on a side stream beside streaming launches keeps to the fewest
      // SMs, leaving the rest to them; cfg2 B=1 dual step 217 vs 242 us)
      while (csz < kRowselMaxCluster && rows * csz * 2 <= num_sms() &&
             n_eff / (2 * csz) >= kRowselMinSlice)
        csz *= 2;
  }
  const bool one_wave = csz > 0 && rows * csz <= num_sms();
  if (rowsel_enabled() && (one_wave || forced_rs == 1) && !force_nt && !hist &&
      br.block_size <= 1 && csz > 0 &&
      p.k_eff < n_eff && n_eff > kSmallN && (reinterpret_cast<uintptr_t>(scores) & 15) == 0) {
    const int S = rowsel_slice(n_eff, csz);
    dim3 grid(p.n_groups * csz, g->batch, n_slots);
    ce = run_rowsel(csz, S, grid, rowsel_smem_bytes(S), st, p);
    if (ce != cudaSuccess) return cuda_check(ce, "rowsel launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_check(cudaGetLastError(), "rowsel launch");
  }
  dim3 grid(p.n_groups, g->batch, n_slots);
  const int nt = force_nt ? force_nt : select_threads(p.n_groups * g->batch * n_slots);
  size_t smem = sel_smem_bytes(n_valid, nt);
  if (hist) smem = std::max(smem, sel_hist_smem_bytes(n_valid, nt));
  p.smem_bytes = (uint32_t)smem;
  ce = run_select(nt, grid, smem, st, p);
  if (ce != cudaSuccess) return cuda_check(ce, "topk_select launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_check(cudaGetLastError(), "topk_select launch");
}

int nb_stride_of(int n_blocks) { return (n_blocks + 7) & ~7; }

// pool -> select -> expand for n_slots layers (see blocks.cuh)
int launch_block_select(const hylra_geometry* g, const float* scores, int n_slots, int n_valid,
                        int block_budget, int block_size, int sel_group, const void* q,
                        const void* k, const int32_t* layer_ids, float* bscores,
                        int32_t* blocks_out, int bk_stride, int32_t* tokens_out,
                        int tok_stride, int32_t* counts_out, int32_t* info, int* flags,
                        cudaStream_t st, int32_t* idx_mirror = nullptr) {
  if (block_size < 1) return fail(HYLRA_ERR_INVALID_INPUT, "block_size must be >= 1");
  if (block_budget < 1)
    return fail(HYLRA_ERR_INVALID_INPUT, "block_budget must be >= 1, got %d", block_budget);
  if (sel_group < 1 || g->kv_heads % sel_group != 0)
    return fail(HYLRA_ERR_CONFIGURATION, "sel_group %d does not divide kv_heads", sel_group);
  const int nb = (n_valid + block_size - 1) / block_size;
  const int bb = std::min(block_budget, nb);
  const int groups = g->kv_heads / sel_group;
  if (bk_stride < bb || (tokens_out && tok_stride < bb * block_size))
    return fail(HYLRA_ERR_CONFIGURATION, "block/token output strides too small");
  const int rows = n_slots * g->batch * groups;
  const int rs = scores_row_stride(g), nbs = nb_stride_of(nb);
  const int w = block_size / 4;
  if (block_size % 4 == 0 && w <= 32 && (w & (w - 1)) == 0) {
    dim3 grid(rows, (n_valid + 4 * kPoolVec * kPoolThreads - 1) / (4 * kPoolVec * kPoolThreads));
    auto kern = w == 1    ? block_pool_vec_kernel<1>
                : w == 2  ? block_pool_vec_kernel<2>
                : w == 4  ? block_pool_vec_kernel<4>
                : w == 8  ? block_pool_vec_kernel<8>
                : w == 16 ? block_pool_vec_kernel<16>
                          : block_pool_vec_kernel<32>;
    kern<<<grid, kPoolThreads, 0, st>>>(scores, g->kv_heads, sel_group, rs, n_valid, bscores,
                                        nbs);
  } else {
    dim3 grid(rows, (nb + kPoolThreads / 32 - 1) / (kPoolThreads / 32));
    block_pool_kernel<<<grid, kPoolThreads, 0, st>>>(scores, g->batch, g->kv_heads, sel_group,
                                                     rs, n_valid, block_size, bscores, nbs);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (int e = cuda_check(cudaGetLastError(), "block_pool launch")) return e;
  BlockRows br;
  br.block_size = block_size;
  br.n_tokens = n_valid;
  br.row_stride = nb_stride_of(nb);
  br.tok_scores = scores;
  if (int e = launch_select(g, bscores, n_slots, nb, block_budget, sel_group, q, k, layer_ids,
                            blocks_out, bk_stride, info, flags, st, br, nullptr, nullptr, 0,
                            idx_mirror))
    return e;
  if (tokens_out) {
    block_expand_kernel<<<n_slots * g->batch * groups, kPoolThreads, 0, st>>>(
        blocks_out, bk_stride, bb, block_size, n_valid, tokens_out, tok_stride, counts_out);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (int e = cuda_check(cudaGetLastError(), "block_expand launch")) return e;
  }
  return HYLRA_OK;
}

struct StepLayout {
  std::vector<int32_t> full_ids, reuse_ids, reuse_src;
  int k_eff, n_groups;
  int bb = 0, tok_stride = 0;                   // block mode
  size_t off_bscores = 0, off_tokens = 0, off_counts = 0;
  int aug_stride = 0;                           // sink / recent augmentation
  size_t off_aug = 0, off_aug_counts = 0;
  size_t off_scores, off_attn, attn_bytes, off_attn_r, attn_bytes_r, total;
  size_t off_sync = 0;  // single-launch step: ticket / done counters + selection ready flags
  size_t off_ctr_f = 0, off_ctr_r = 0;  // split-K counters of the FULL / REUSE launches
  size_t off_hist = 0;                  // score-row histograms (0: none)
  // cooperative select of the single-launch step (select.cuh coop_*; with the histograms):
  // per score row a 64-byte record (zero at rest), a candidate list and a bitmap
  size_t off_coop = 0, off_coop_cv = 0, off_coop_ci = 0, off_coop_bits = 0;
  int coop_words = 0;
  int n_ready = 0;
  int* ctr_f(uint8_t* w) const { return reinterpret_cast<int*>(w + off_ctr_f); }
  int* ctr_r(uint8_t* w) const { return reinterpret_cast<int*>(w + off_ctr_r); }
  unsigned* hist(uint8_t* w) const {
    return off_hist ? reinterpret_cast<unsigned*>(w + off_hist) : nullptr;
  }
};

// Score-row histograms (select.cuh kHistBins): the cooperative selects of the single-launch
// step (fuse_select = 3) need them; the other schedules' selects use them only with
// HYLRA_HIST=1. Measured on B200 (scripts/schedules.py, profiles/r02_hist_ab.txt): counting
// them costs the FULL kernel ~2-5% (cfg2 B=8 single 1.472 vs 1.450 ms, B=1 FULL launch 181 vs
// 173 us) and saves less than that in the selects, so the sampled selects stay the default.
bool hist_enabled() {
  static int v = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = std::getenv("HYLRA_HIST");
    v = (e && *e) ? (atoi(e) != 0) : 0;
  });
  return v == 1;
}

int step_layout(const hylra_geometry* g, const uint8_t* actions, int n_valid, int budget,
                int sel_group, StepLayout* s, int block_size = 1, int sinks = 0,
                int recent = 0) {
  if (int e = check_geometry(g)) return e;
  if (!actions) return fail(HYLRA_ERR_CONFIGURATION, "actions is NULL");
  if (actions[0] != 1)
    return fail(HYLRA_ERR_INVALID_INPUT, "the first layer of a policy must run full attention");
  if (budget < 1) return fail(HYLRA_ERR_INVALID_INPUT, "budget must be >= 1, got %d", budget);
  if (n_valid < 1 || n_valid > g->capacity)
    return fail(HYLRA_ERR_INVALID_INPUT, "n_valid %d not in [1, capacity]", n_valid);
  if (sel_group < 1 || g->kv_heads % sel_group != 0)
    return fail(HYLRA_ERR_CONFIGURATION, "sel_group %d does not divide kv_heads", sel_group);
  s->full_ids.clear(); s->reuse_ids.clear(); s->reuse_src.clear();
  int cur = -1;
  for (int l = 0; l < g->num_layers; ++l) {
    if (actions[l]) {
      cur = (int)s->full_ids.size();
      s->full_ids.push_back(l);
    } else {
      s->reuse_ids.push_back(l);
      s->reuse_src.push_back(cur);
    }
  }
  if ((int)s->full_ids.size() > kMaxSlots || (int)s->reuse_ids.size() > kMaxSlots)
    return fail(HYLRA_ERR_CONFIGURATION, "more than %d layers of one kind", kMaxSlots);
  s->n_groups = g->kv_heads / sel_group;
  const size_t nf = s->full_ids.size();
  // Layout: every word a kernel expects to find zeroed (the single-launch sync words, the
  // split-K counters) comes first, at offsets that depend only on the geometry and the
  // policy; everything sized by n_valid (block / augmentation rows, split-K partials)
  // follows. A decoder stepping over a growing cache reuses its workspace across many
  // n_valid values, and a counter that landed on an earlier step's partials would never
  // fire its merge.
  s->n_ready = (int)(nf * g->batch * s->n_groups);
  s->off_sync = kHeader;  // ticket / done, then ready flags and group counters [n_ready] each
  s->off_ctr_f = align_up(s->off_sync + 256 + 2 * sizeof(int) * (size_t)s->n_ready, 256);
  s->off_ctr_r = s->off_ctr_f + counter_region_bytes(g);
  // the FULL kernel's per-score-row histograms (select.cuh kHistBins), read and re-zeroed by
  // the selects: token mode, per-KV-head rows, tensor-core FULL path
  size_t off = s->off_ctr_r + counter_region_bytes(g);
  if (block_size == 1 && sel_group == 1 && use_mma_path(g)) {
    const size_t rows = nf * g->batch * g->kv_heads;
    s->off_hist = off;
    off = align_up(off + sizeof(unsigned) * kHistBins * rows, 256);
    s->off_coop = off;
    off = align_up(off + sizeof(CoopRow) * rows, 256);
    s->off_coop_cv = off;
    off = align_up(off + sizeof(float) * kHistCandCap * rows, 256);
    s->off_coop_ci = off;
    off = align_up(off + sizeof(int) * kHistCandCap * rows, 256);
    s->coop_words = (g->capacity + 31) / 32;
    s->off_coop_bits = off;
    off = align_up(off + sizeof(uint32_t) * s->coop_words * rows, 256);
  }
  s->off_scores = off;
  const size_t scores_b = sizeof(float) * nf * g->batch * g->kv_heads * scores_row_stride(g);
  off = align_up(s->off_scores + scores_b, 256);
  if (block_size > 1) {
    // budget counts blocks; REUSE layers read the coverage (<= bb * block_size tokens)
    const int nb = (n_valid + block_size - 1) / block_size;
    s->bb = std::min(budget, nb);
    s->k_eff = s->bb * block_size;  // coverage upper bound; per-row counts trim it
    s->tok_stride = s->bb * block_size;
    const size_t rows = nf * g->batch * s->n_groups;
    s->off_bscores = off;
    off = align_up(off + sizeof(float) * rows * nb_stride_of(nb), 256);
    s->off_tokens = off;
    off = align_up(off + sizeof(int32_t) * rows * s->tok_stride, 256);
    s->off_counts = off;
    off = align_up(off + sizeof(int32_t) * rows, 256);
  } else {
    s->k_eff = std::min(budget, n_valid);
    if (sinks < 0 || recent < 0)
      return fail(HYLRA_ERR_INVALID_INPUT, "include_sinks and include_recent must be >= 0");
    if ((sinks > 0 || recent > 0) && !s->reuse_ids.empty()) {
      const size_t rows = nf * g->batch * s->n_groups;
      s->aug_stride = std::min(n_valid, s->k_eff + sinks + recent);
      s->off_aug = off;
      off = align_up(off + sizeof(int32_t) * rows * s->aug_stride, 256);
      s->off_aug_counts = off;
      off = align_up(off + sizeof(int32_t) * rows, 256);
    }
  }
  // split-K partials of the FULL and REUSE launches (their counters are the fixed regions
  // above). FULL layers may be launched in two groups (hylra_decode_step_ex with a side
  // stream), REUSE layers in chunks (layer events): size for the largest any group needs
  // (fewer pairs can mean more splits). Partials are always written before they are read.
  s->off_attn = off;
  s->attn_bytes = 0;
  for (int n = 1; n <= (int)nf; ++n)
    s->attn_bytes = std::max({s->attn_bytes, attn_layout(g, n, n_valid, false, true).total,
                              attn_layout(g, n, n_valid, false, true, true).total});
  s->off_attn_r = align_up(s->off_attn + s->attn_bytes, 256);
  s->attn_bytes_r = 0;
  for (int n = 1; n <= (int)s->reuse_ids.size(); ++n)
    s->attn_bytes_r = std::max(
        s->attn_bytes_r,
        attn_layout(g, n, s->aug_stride ? s->aug_stride : s->k_eff, true, true).total);
  s->total = align_up(s->off_attn_r + s->attn_bytes_r, 256);
  return HYLRA_OK;
}

// Device address of caller memory that kernels may read: device memory as is, page-locked
// host memory through its mapping (UVA). Pageable host memory is rejected.
int device_view(const void* ptr, const void** dev, const char* what) {
  if (!ptr) return fail(HYLRA_ERR_CONFIGURATION, "%s is NULL", what);
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return fail(HYLRA_ERR_CONFIGURATION, "%s: not a CUDA-visible pointer", what);
  }
  if (a.type == cudaMemoryTypeUnregistered)
    return fail(HYLRA_ERR_CONFIGURATION,
                "%s must be device memory or page-locked (pinned) host memory", what);
  *dev = a.devicePointer ? a.devicePointer : ptr;
  return HYLRA_OK;
}

// hylra_step_options idx_mirror (device or pinned host memory) as a device address.
int mirror_view(const hylra_step_options* opt, int32_t** out) {
  *out = nullptr;
  if (!opt || !opt->idx_mirror) return HYLRA_OK;
  const void* dev = nullptr;
  if (int e = device_view(opt->idx_mirror, &dev, "idx_mirror")) return e;
  *out = static_cast<int32_t*>(const_cast<void*>(dev));
  return HYLRA_OK;
}

// One decode step: FULL layers (+ scores) -> SELECT -> [augment] -> REUSE layers. With
// `split`, FULL layers read a compact device cache and REUSE layers a compact cache that
// may live in page-locked host memory (index-guided offload: only selected rows cross the
// link); otherwise both read the one [L][B][Hkv][cap][d] cache.
struct SplitKv {
  const void *kf, *vf, *kr, *vr;
};

// The single-launch kernel for this geometry (tensor-core path).
int dispatch_step(const hylra_geometry* g, cudaStream_t st, const CUtensorMap& tk,
                  const CUtensorMap& tv, const AttnParams& pf, const AttnParams& pr,
                  const SelectParams& sp, const StepSync& ss) {
  const int G = g->q_heads / g->kv_heads;
  cudaError_t ce;
  ce = run_step_mma(g->head_dim, G > 8, ss.n_items, st, tk, tv, pf, pr, sp, ss);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_check(ce, "single-launch step");
}

// The fused select of the FULL kernel uses the drained pipeline buffers as its shared
// memory (128 threads).
bool fused_select_fits(const hylra_geometry* g, int n_valid) {
  const size_t ring = g->head_dim == 128
                          ? (size_t)mma_stages<128, false, false>() * MmaSmem<128>::kStageBytes
                          : (size_t)mma_stages<64, false, false>() * MmaSmem<64>::kStageBytes;
  return n_valid <= kSelMaxTokens && sel_smem_bytes(n_valid, kConsumerWarps * 32, true) <= ring;
}

// Options of hylra_decode_step_ex (all optional; see include/hylra.h).
struct StepOpts {
  bool fuse = false;  // selects of the FULL layers feeding REUSE fused into the FULL kernel
  bool unified = false;  // single-launch step (fuse_select == 2 or 3)
  bool coop = false;     // ... with the cooperative selects (fuse_select == 3)
  const void* app_k = nullptr;  // the step's new K/V rows [L][B][Hkv][d] (append_* options)
  const void* app_v = nullptr;
  int app_pos = -1;
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, select = nullptr, full = nullptr, join = nullptr;
  cudaEvent_t reuse_wait = nullptr;
  void* const* layer_events = nullptr;
  int32_t* idx_mirror = nullptr;  // device address of the selections' second copy
};

int record(void* const* evs, int l, cudaStream_t st) {
  if (!evs || !evs[l]) return HYLRA_OK;
  return cuda_check(cudaEventRecord(static_cast<cudaEvent_t>(evs[l]), st), "event record");
}

// The step's append option (hylra_step_options append_*): validated here; in_kernel fills
// *ap for the single-launch kernel (its FULL items write the rows), else hylra_append_kv
// runs ahead of the step on the same stream.
int append_impl(const hylra_geometry* g, void* k, void* v, const void* k_rows,
                const void* v_rows, int pos, int n_layers, const int32_t* layer_ids, int* flags,
                cudaStream_t st);

int step_append(const hylra_geometry* g, const void* k, const void* v, const void* rows_k,
                const void* rows_v, int pos, int n_valid, bool in_kernel, StepAppend* ap,
                int* flags, cudaStream_t st) {
  if (!rows_k || !rows_v)
    return fail(HYLRA_ERR_CONFIGURATION, "append needs both append_k_rows and append_v_rows");
  if (pos < 0 || pos >= n_valid)
    return fail(HYLRA_ERR_INVALID_INPUT, "append_pos %d not in [0, n_valid=%d)", pos, n_valid);
  if (!in_kernel)
    return append_impl(g, const_cast<void*>(k), const_cast<void*>(v), rows_k, rows_v, pos, 0,
                       nullptr, flags, st);
  ap->flags = flags;
  if (int e = device_view(rows_k, reinterpret_cast<const void**>(&ap->k_rows), "append_k_rows"))
    return e;
  if (int e = device_view(rows_v, reinterpret_cast<const void**>(&ap->v_rows), "append_v_rows"))
    return e;
  const int64_t es = 2, row_bytes = (int64_t)g->head_dim * es;  // tensor-core path: bf16
  if ((g->kv_stride_layer * es) % 16 || (g->kv_stride_batch * es) % 16 ||
      (g->kv_stride_head * es) % 16 || reinterpret_cast<uintptr_t>(k) % 16 ||
      reinterpret_cast<uintptr_t>(v) % 16 || reinterpret_cast<uintptr_t>(ap->k_rows) % 16 ||
      reinterpret_cast<uintptr_t>(ap->v_rows) % 16)
    return fail(HYLRA_ERR_CONFIGURATION, "append needs 16-byte aligned rows and strides");
  ap->k = static_cast<uint8_t*>(const_cast<void*>(k));
  ap->v = static_cast<uint8_t*>(const_cast<void*>(v));
  ap->kv_sl = g->kv_stride_layer * es;
  ap->kv_sb = g->kv_stride_batch * es;
  ap->kv_sh = g->kv_stride_head * es;
  ap->pos = pos;
  ap->pos_bytes = (int64_t)pos * row_bytes;
  ap->chunks = (int)(row_bytes / 16);
  return HYLRA_OK;
}

int decode_step_impl(const hylra_geometry* g, const void* q, const void* k, const void* v,
                     int n_valid, const uint8_t* actions, int budget, int sel_group, int refine,
                     int sinks, int recent, float* out, int32_t* idx, int k_stride, void* ws,
                     size_t ws_bytes, void* stream, const SplitKv* split,
                     const StepOpts& o = StepOpts()) {
  StepLayout s;
  if (int e = step_layout(g, actions, n_valid, budget, sel_group, &s, 1, sinks, recent)) return e;
  if (!ws || ws_bytes < s.total)
    return fail(HYLRA_ERR_CONFIGURATION, "workspace %zu B < required %zu B", ws_bytes, s.total);
  if (k_stride < s.k_eff)
    return fail(HYLRA_ERR_CONFIGURATION, "k_stride %d < selection size %d", k_stride, s.k_eff);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  int* flags = reinterpret_cast<int*>(w);
  float* scores = reinterpret_cast<float*>(w + s.off_scores);
  void* aws = w + s.off_attn;
  const int nf = (int)s.full_ids.size();
  const int nr = (int)s.reuse_ids.size();
  const void* kf = split ? split->kf : k;
  const void* vf = split ? split->vf : v;
  const size_t score_slot = (size_t)g->batch * g->kv_heads * scores_row_stride(g);
  // per score row; slot stride below. Off (null) unless the cooperative single-launch step or
  // HYLRA_HIST=1 asks for them
  unsigned* hist = (o.coop || hist_enabled()) ? s.hist(w) : nullptr;
  const size_t hist_slot = (size_t)g->batch * g->kv_heads * kHistBins;

  // FULL layer groups: A = the FULL layers some REUSE layer inherits from (the selection the
  // REUSE launch waits for), B = the others. With a side stream the selects leave the
  // critical path:  stream: FULL(A) -> FULL(B) -> REUSE;  side: SELECT(A) under FULL(B),
  // SELECT(B) under REUSE. The selects are latency-bound (one CTA per row, ~30 us at any
  // row count), the FULL and REUSE launches HBM-bound; the side stream has the higher
  // priority so select CTAs are dispatched ahead of queued streaming CTAs.
  std::vector<int32_t> a_ids, a_slot, a_kv, b_ids, b_slot, b_kv;
  for (int i = 0; i < nf; ++i) {
    const int l = s.full_ids[i];
    const bool feeds = l + 1 < g->num_layers && actions[l + 1] == 0;
    (feeds ? a_ids : b_ids).push_back(l);
    (feeds ? a_slot : b_slot).push_back(i);
    (feeds ? a_kv : b_kv).push_back(i);  // compact KV index (split caches) = FULL slot
  }
  const bool dual = o.side && !a_ids.empty() && !b_ids.empty() && !s.aug_stride;
  // fused selects (StepOpts::fuse): tensor-core FULL path, per-KV-head rows, A non-empty;
  // the select's shared memory must fit in the FULL kernel's pipeline buffers
  const bool fused_sel = o.fuse && o.side && !a_ids.empty() && !s.aug_stride && sel_group == 1 &&
                         use_mma_path(g) && fused_select_fits(g, n_valid);
  // single-launch step: every select fused into the FULL items, REUSE items in the same grid
  const bool unified = o.unified && use_mma_path(g) && fused_select_fits(g, n_valid) &&
                       !o.layer_events;
  // the step's new K/V rows: written inside the single-launch kernel, else by the append
  // kernel ahead of the step
  const bool appending = o.app_k != nullptr || o.app_v != nullptr;
  if (appending && split)
    return fail(HYLRA_ERR_CONFIGURATION, "append is not supported with split caches");
  StepAppend app{};
  if (appending)
    if (int e = step_append(g, k, v, o.app_k, o.app_v, o.app_pos, n_valid, unified, &app, flags,
                            st))
      return e;
  if (unified) {
    std::vector<int32_t> ab_ids(a_ids), ab_slot(a_slot), ab_kv(a_kv);
    ab_ids.insert(ab_ids.end(), b_ids.begin(), b_ids.end());
    ab_slot.insert(ab_slot.end(), b_slot.begin(), b_slot.end());
    ab_kv.insert(ab_kv.end(), b_kv.begin(), b_kv.end());
    SelectParams sp{};
    if (int e = build_select_params(&sp, g, scores, nf, n_valid, budget, sel_group,
                                    refine ? q : nullptr, refine ? kf : nullptr, ab_ids.data(),
                                    idx, k_stride, nullptr, flags, BlockRows(),
                                    split ? ab_kv.data() : nullptr, ab_slot.data()))
      return e;
    sp.idx_mirror = o.idx_mirror;
    // sinks / recent: the final CTA of each pair also writes the augmented row
    const int32_t* ridx = idx;
    const int32_t* rcnt = nullptr;
    int rstride = k_stride, rk = s.k_eff;
    if (s.aug_stride) {
      sp.cov_tokens = reinterpret_cast<int32_t*>(w + s.off_aug);
      sp.cov_counts = reinterpret_cast<int32_t*>(w + s.off_aug_counts);
      sp.cov_stride = s.aug_stride;
      sp.sinks = sinks;
      sp.recent = recent;
      ridx = sp.cov_tokens;
      rcnt = sp.cov_counts;
      rstride = rk = s.aug_stride;
    }
    AttnParams pf{}, pr{};
    AttnLayout lf{}, lr{};
    // sel_group: the fused select of a pair's final CTA covers its selection group
    if (int e = make_attn_params(&pf, &lf, g, false, q, kf, vf, n_valid, n_valid, nf,
                                 ab_ids.data(), nullptr, nullptr, nullptr, 0, sel_group, out,
                                 scores, aws, s.attn_bytes, flags,
                                 split ? ab_kv.data() : nullptr, nf, s.ctr_f(w)))
      return e;
    pf.fuse_select = nf;
    if (lf.tps * kTileRows >= 65536) hist = nullptr;  // 16-bit per-split histogram counters
    pf.hist = hist;
    sp.hist = hist;
    if (hist && o.coop) {
      sp.coop = reinterpret_cast<CoopRow*>(w + s.off_coop);
      sp.coop_cv = reinterpret_cast<float*>(w + s.off_coop_cv);
      sp.coop_ci = reinterpret_cast<int*>(w + s.off_coop_ci);
      sp.coop_bits = reinterpret_cast<uint32_t*>(w + s.off_coop_bits);
      sp.coop_words = s.coop_words;
    }
    const long items_f = (long)lf.splits * g->kv_heads * g->batch * nf;
    long items_r = 0;
    std::vector<int32_t> rkv(nr);
    for (int i = 0; i < nr; ++i) rkv[i] = i;
    if (nr > 0) {
      if (int e = make_attn_params(&pr, &lr, g, true, q, split ? split->kr : k,
                                   split ? split->vr : v, n_valid, rk, nr,
                                   s.reuse_ids.data(), s.reuse_src.data(), ridx, rcnt, rstride,
                                   sel_group, out, nullptr, w + s.off_attn_r, s.attn_bytes_r,
                                   flags, split ? rkv.data() : nullptr, nr, s.ctr_r(w)))
        return e;
      items_r = (long)lr.splits * g->kv_heads * g->batch * nr;
    }
    if (items_f + items_r > INT32_MAX) return fail(HYLRA_ERR_CONFIGURATION, "grid too large");
    CUtensorMap tk{}, tv{};
    if (int e = encode_kv_map(&tk, g, kf, split ? nf : g->num_layers)) return e;
    if (int e = encode_kv_map(&tv, g, vf, split ? nf : g->num_layers)) return e;
    StepSync ss{};
    ss.ctr = reinterpret_cast<int*>(w + s.off_sync);
    ss.ready = ss.ctr + 64;
    ss.group = ss.ready + s.n_ready;
    ss.n_ready = s.n_ready;
    ss.n_full_items = (int)items_f;
    ss.n_items = (int)(items_f + items_r);
    ss.app = app;
    if (o.reuse_wait)
      if (int e = cuda_check(cudaStreamWaitEvent(st, o.reuse_wait, 0), "stream wait event"))
        return e;
    return dispatch_step(g, st, tk, tv, pf, pr, sp, ss);
  }
  if (o.side && !(o.fork && o.join && (o.fuse || (o.select && o.full))))
    return fail(HYLRA_ERR_CONFIGURATION, "a side stream needs its four events");
  // groups of FULL layers: one launch (all FULL layers) or two (A then B)
  struct Group {
    const std::vector<int32_t>* ids;
    const std::vector<int32_t>* slots;
    const std::vector<int32_t>* kv;
    int score_base;
  };
  std::vector<int32_t> all_slot(nf), all_kv(nf);
  for (int i = 0; i < nf; ++i) all_slot[i] = all_kv[i] = i;
  const Group g_all{&s.full_ids, &all_slot, &all_kv, 0};
  const Group g_a{&a_ids, &a_slot, &a_kv, 0};
  const Group g_b{&b_ids, &b_slot, &b_kv, (int)a_ids.size()};
  auto full = [&](const Group& gr, cudaStream_t sx, const SelectParams* fused = nullptr,
                  int n_fused = 0) -> int {
    const int n = (int)gr.ids->size();
    if (int e = launch_attention(g, false, q, kf, vf, n_valid, n_valid, n, gr.ids->data(),
                                 nullptr, nullptr, nullptr, 0, 1, out,
                                 scores + gr.score_base * score_slot, aws, s.attn_bytes, flags, sx,
                                 split ? gr.kv->data() : nullptr, nf, fused, n_fused, nullptr, 0,
                                 0, s.ctr_f(w), hist ? hist + gr.score_base * hist_slot : nullptr))
      return e;
    for (int l : *gr.ids)
      if (int e = record(o.layer_events, l, sx)) return e;
    return HYLRA_OK;
  };
  auto select = [&](const Group& gr, cudaStream_t sx, int force_nt = 0) -> int {
    return launch_select(g, scores + gr.score_base * score_slot, (int)gr.ids->size(), n_valid,
                         budget, sel_group, refine ? q : nullptr, refine ? kf : nullptr,
                         gr.ids->data(), idx, k_stride, nullptr, flags, sx, BlockRows(),
                         split ? gr.kv->data() : nullptr, gr.slots->data(), force_nt,
                         o.idx_mirror, hist ? hist + gr.score_base * hist_slot : nullptr,
                         sx != st);
  };
  auto reuse = [&](cudaStream_t sx) -> int {
    if (s.reuse_ids.empty()) return HYLRA_OK;
    const int32_t* ridx = idx;
    const int32_t* rcnt = nullptr;
    int rstride = k_stride, rk = s.k_eff;
    if (s.aug_stride) {
      int32_t* aug = reinterpret_cast<int32_t*>(w + s.off_aug);
      int32_t* acnt = reinterpret_cast<int32_t*>(w + s.off_aug_counts);
      const int rows = nf * g->batch * s.n_groups;
      augment_kernel<<<rows, kPoolThreads, 0, sx>>>(idx, k_stride, s.k_eff, n_valid, sinks,
                                                    recent, aug, s.aug_stride, acnt);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      if (int e = cuda_check(cudaGetLastError(), "augment launch")) return e;
      ridx = aug;
      rcnt = acnt;
      rstride = rk = s.aug_stride;
    }
    if (o.reuse_wait)
      if (int e = cuda_check(cudaStreamWaitEvent(sx, o.reuse_wait, 0), "stream wait event"))
        return e;
    std::vector<int32_t> rkv(nr);  // compact KV layer index of each REUSE slot
    for (int i = 0; i < nr; ++i) rkv[i] = i;
    // one launch, or one per chunk of REUSE layers ending at a layer that carries an event
    int c0 = 0;
    for (int i = 0; i < nr; ++i) {
      const int l = s.reuse_ids[i];
      const bool mark = o.layer_events && o.layer_events[l];
      if (!(mark || i == nr - 1)) continue;
      const int n = i + 1 - c0;
      if (int e = launch_attention(g, true, q, split ? split->kr : k, split ? split->vr : v,
                                   n_valid, rk, n, s.reuse_ids.data() + c0,
                                   s.reuse_src.data() + c0, ridx, rcnt, rstride, sel_group, out,
                                   nullptr, w + s.off_attn_r, s.attn_bytes_r, flags, sx,
                                   split ? rkv.data() + c0 : nullptr, nr, nullptr, 0, nullptr,
                                   0, 0, s.ctr_r(w)))
        return e;
      if (int e = record(o.layer_events, l, sx)) return e;
      c0 = i + 1;
    }
    return HYLRA_OK;
  };

  if (!dual && !fused_sel) {
    if (int e = full(g_all, st)) return e;
    if (int e = select(g_all, st)) return e;
    return reuse(st);
  }
  auto rec = [](cudaEvent_t ev, cudaStream_t sx) {
    return cuda_check(cudaEventRecord(ev, sx), "event record");
  };
  auto wait = [](cudaStream_t sx, cudaEvent_t ev) {
    return cuda_check(cudaStreamWaitEvent(sx, ev, 0), "stream wait event");
  };
  if (fused_sel) {
    // one FULL launch over A then B; A's selections are taken inside it by the last CTA of
    // each pair (A's pairs come first in the grid, so those selects run under B's
    // streaming); SELECT(B) runs on the side stream under the REUSE launch
    std::vector<int32_t> ab_ids(a_ids), ab_slot(a_slot), ab_kv(a_kv);
    ab_ids.insert(ab_ids.end(), b_ids.begin(), b_ids.end());
    ab_slot.insert(ab_slot.end(), b_slot.begin(), b_slot.end());
    ab_kv.insert(ab_kv.end(), b_kv.begin(), b_kv.end());
    const Group g_ab{&ab_ids, &ab_slot, &ab_kv, 0};
    SelectParams sp{};
    if (int e = build_select_params(&sp, g, scores, (int)ab_ids.size(), n_valid, budget,
                                    sel_group, refine ? q : nullptr, refine ? kf : nullptr,
                                    ab_ids.data(), idx, k_stride, nullptr, flags, BlockRows(),
                                    split ? ab_kv.data() : nullptr, ab_slot.data()))
      return e;
    sp.idx_mirror = o.idx_mirror;
    sp.hist = hist;
    if (int e = full(g_ab, st, &sp, (int)a_ids.size())) return e;
    if (!b_ids.empty()) {
      if (int e = rec(o.fork, st)) return e;
      if (int e = wait(o.side, o.fork)) return e;
      if (int e = select(g_b, o.side)) return e;
      if (int e = rec(o.join, o.side)) return e;
    }
    if (int e = reuse(st)) return e;
    return b_ids.empty() ? HYLRA_OK : wait(st, o.join);
  }
  // side: SELECT(A) once FULL(A) is done, SELECT(B) once FULL(B) is done
  if (int e = full(g_a, st)) return e;
  if (int e = rec(o.fork, st)) return e;
  if (int e = wait(o.side, o.fork)) return e;
  if (int e = select(g_a, o.side)) return e;
  if (int e = rec(o.select, o.side)) return e;
  if (int e = full(g_b, st)) return e;
  if (int e = rec(o.full, st)) return e;
  if (int e = wait(o.side, o.full)) return e;
  if (int e = select(g_b, o.side)) return e;
  if (int e = rec(o.join, o.side)) return e;
  // stream: REUSE once SELECT(A) is done (long before FULL(B) ends), then join
  if (int e = wait(st, o.select)) return e;
  if (int e = reuse(st)) return e;
  return wait(st, o.join);
}

// HYLRA_BLOCK_TILES=1: block-mode REUSE streams the selected blocks as TMA tiles instead of
// gathering the coverage row by row. Bit-identical; measured at cfg2 B=8 (block_size 128,
// 16 blocks): REUSE alone 248 vs 254 us, but the graph-replayed step 1.56 vs 1.52-1.55 ms,
// so the gather stays the default (scripts/block_ab.py).
bool block_tiles_off() {
  const char* e = std::getenv("HYLRA_BLOCK_TILES");
  return !(e && *e && atoi(e) == 1);
}

}  // namespace

// ======================================================================== extern "C"
extern "C" {


int hylra_abi_version(void) { return HYLRA_ABI_VERSION; }

const char* hylra_status_string(int status) {
  switch (status) {
    case HYLRA_OK: return "ok";
    case HYLRA_ERR_CONFIGURATION: return "ConfigurationError";
    case HYLRA_ERR_INVALID_INPUT: return "InvalidInputError";
    case HYLRA_ERR_INVALID_SELECTION: return "InvalidSelectionError";
    case HYLRA_ERR_NUMERIC_INPUT: return "NumericInputError";
    case HYLRA_ERR_CUDA: return "CudaError";
    default: return "unknown status";
  }
}

const char* hylra_last_error(void) { return g_err; }

uint64_t hylra_launch_count(void) { return g_launches.load(); }

int hylra_set_tuning(const char* name, int value) {
  if (!name) return fail(HYLRA_ERR_CONFIGURATION, "NULL tuning name");
  std::atomic<int>* knob = nullptr;
  if (!strcmp(name, "rowsel")) knob = &tuning().rowsel;
  else if (!strcmp(name, "select_threads")) knob = &tuning().select_threads;
  else if (!strcmp(name, "rowsel_cluster")) knob = &tuning().rowsel_cluster;
  else if (!strcmp(name, "gather_tma")) knob = &tuning().gather_tma;
  else if (!strcmp(name, "bulk_merge")) knob = &tuning().bulk_merge;
  else if (!strcmp(name, "cluster_merge")) knob = &tuning().cluster_merge;
  else if (!strcmp(name, "reuse_prefetch")) knob = &tuning().reuse_prefetch;
  else if (!strcmp(name, "fused_fine_splits")) knob = &tuning().fused_fine_splits;
  if (!knob) return fail(HYLRA_ERR_CONFIGURATION, "unknown tuning knob '%s'", name);
  knob->store(value < 0 ? -1 : value, std::memory_order_relaxed);
  return HYLRA_OK;
}

size_t hylra_attention_workspace_bytes(const hylra_geometry* g, int n_layers, int rows) {
  if (check_geometry(g) || n_layers < 1) return 0;
  // either op (FULL or REUSE) may use the workspace
  return std::max({attn_layout(g, n_layers, std::max(rows, 1), false).total,
                   attn_layout(g, n_layers, std::max(rows, 1), false, false, true).total,
                   attn_layout(g, n_layers, std::max(rows, 1), true).total});
}

size_t hylra_select_workspace_bytes(const hylra_geometry* g, int n_slots, int sel_group) {
  (void)g; (void)n_slots; (void)sel_group;
  return kHeader;  // flag word only
}

int hylra_full_decode(const hylra_geometry* g, const void* q, const void* k, const void* v,
                      int n_valid, int n_layers, const int32_t* layer_ids, float* out,
                      float* scores, void* ws, size_t ws_bytes, void* stream) {
  return launch_attention(g, false, q, k, v, n_valid, n_valid, n_layers, layer_ids, nullptr,
                          nullptr, nullptr, 0, 1, out, scores, ws, ws_bytes, static_cast<int*>(ws),
                          static_cast<cudaStream_t>(stream));
}

int hylra_topk_select(const hylra_geometry* g, const float* scores, int n_slots, int n_valid,
                      int budget, int sel_group, const void* q, const void* k,
                      const int32_t* layer_ids, int32_t* idx, int k_stride, int32_t* info,
                      void* ws, size_t ws_bytes, void* stream) {
  return hylra_topk_select_ex(g, scores, n_slots, n_valid, budget, sel_group, q, k, layer_ids,
                              idx, k_stride, info, ws, ws_bytes, stream, 0);
}

int hylra_topk_select_ex(const hylra_geometry* g, const float* scores, int n_slots,
                         int n_valid, int budget, int sel_group, const void* q, const void* k,
                         const int32_t* layer_ids, int32_t* idx, int k_stride, int32_t* info,
                         void* ws, size_t ws_bytes, void* stream, int options) {
  if (!ws || ws_bytes < kHeader) return fail(HYLRA_ERR_CONFIGURATION, "select workspace too small");
  return launch_select(g, scores, n_slots, n_valid, budget, sel_group, q, k, layer_ids, idx,
                       k_stride, info, static_cast<int*>(ws), static_cast<cudaStream_t>(stream),
                       BlockRows(), nullptr, nullptr, 0, nullptr, nullptr,
                       (options & HYLRA_SELECT_COMPACT) != 0);
}

int hylra_decode_layer(const hylra_geometry* g, const void* q, const void* k, const void* v,
                       int n_valid, int layer, int full, int slot, int budget, int sel_group,
                       int refine, int prefetch, float* out, float* scores, int32_t* idx,
                       int k_stride, void* ws, size_t ws_bytes, void* stream) {
  if (!g) return fail(HYLRA_ERR_CONFIGURATION, "NULL geometry");
  if (int e = check_geometry(g)) return e;
  if (budget < 1) return fail(HYLRA_ERR_INVALID_INPUT, "budget must be >= 1, got %d", budget);
  if (sel_group < 1 || g->kv_heads % sel_group != 0)
    return fail(HYLRA_ERR_CONFIGURATION, "sel_group %d does not divide kv_heads %d", sel_group,
                g->kv_heads);
  if (slot < 0 || slot >= kMaxSlots)
    return fail(HYLRA_ERR_CONFIGURATION, "slot %d not in [0, %d)", slot, kMaxSlots);
  if (!ws || ws_bytes < kHeader)
    return fail(HYLRA_ERR_CONFIGURATION, "layer workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int* flags = static_cast<int*>(ws);
  const int32_t ids[1] = {layer};
  const int32_t src[1] = {slot};
  const int k_eff = std::min(budget, n_valid);
  // the early loads need the TMA / cp.async producer warps of the tensor-core kernels
  const int early = (prefetch && use_mma_path(g)) ? 1 : 0;
  if (full) {
    if (idx && !scores)
      return fail(HYLRA_ERR_CONFIGURATION, "a FULL layer's selection needs its score rows");
    if (int e = launch_attention(g, false, q, k, v, n_valid, n_valid, 1, ids, nullptr, nullptr,
                                 nullptr, 0, 1, out, scores, ws, ws_bytes, flags, st, nullptr, 0,
                                 nullptr, 0, nullptr, 0, 0, nullptr, nullptr, early))
      return e;
    if (!idx) return HYLRA_OK;
    return launch_select(g, scores, 1, n_valid, budget, sel_group, refine ? q : nullptr,
                         refine ? k : nullptr, ids, idx, k_stride, nullptr, flags, st,
                         BlockRows(), nullptr, src);
  }
  if (!idx) return fail(HYLRA_ERR_CONFIGURATION, "a REUSE layer needs the selections");
  if (k_stride < k_eff)
    return fail(HYLRA_ERR_CONFIGURATION, "k_stride %d < selection size %d", k_stride, k_eff);
  return launch_attention(g, true, q, k, v, n_valid, k_eff, 1, ids, src, idx, nullptr, k_stride,
                          sel_group, out, nullptr, ws, ws_bytes, flags, st, nullptr, 0, nullptr,
                          0, nullptr, 0, 0, nullptr, nullptr, early);
}

int hylra_reuse_decode(const hylra_geometry* g, const void* q, const void* k, const void* v,
                       int n_valid, int n_layers, const int32_t* layer_ids,
                       const int32_t* src_slots, const int32_t* idx, const int32_t* counts,
                       int k_stride, int k_eff, int sel_group, float* out, void* ws,
                       size_t ws_bytes, void* stream) {
  if (!idx || !src_slots) return fail(HYLRA_ERR_CONFIGURATION, "NULL selection argument");
  if (k_eff < 1 || k_eff > k_stride)
    return fail(HYLRA_ERR_INVALID_SELECTION, "selection size %d not in [1, k_stride=%d]", k_eff,
                k_stride);
  if (sel_group < 1 || (g && g->kv_heads % sel_group != 0))
    return fail(HYLRA_ERR_CONFIGURATION, "sel_group %d does not divide kv_heads", sel_group);
  return launch_attention(g, true, q, k, v, n_valid, k_eff, n_layers, layer_ids, src_slots, idx,
                          counts, k_stride, sel_group, out, nullptr, ws, ws_bytes,
                          static_cast<int*>(ws), static_cast<cudaStream_t>(stream));
}

size_t hylra_decode_step_workspace_bytes(const hylra_geometry* g, const uint8_t* actions,
                                         int n_valid, int budget, int sel_group, int sinks,
                                         int recent) {
  StepLayout s;
  if (step_layout(g, actions, n_valid, budget, sel_group, &s, 1, sinks, recent)) return 0;
  return s.total;
}

int hylra_decode_step(const hylra_geometry* g, const void* q, const void* k, const void* v,
                      int n_valid, const uint8_t* actions, int budget, int sel_group,
                      int refine, int sinks, int recent, float* out, int32_t* idx,
                      int k_stride, void* ws, size_t ws_bytes, void* stream) {
  return decode_step_impl(g, q, k, v, n_valid, actions, budget, sel_group, refine, sinks, recent,
                          out, idx, k_stride, ws, ws_bytes, stream, nullptr);
}

int hylra_decode_step_ex(const hylra_geometry* g, const void* q, const void* k, const void* v,
                         int n_valid, const uint8_t* actions, int budget, int sel_group,
                         int refine, int sinks, int recent, float* out, int32_t* idx,
                         int k_stride, void* ws, size_t ws_bytes, void* stream,
                         const hylra_step_options* opt) {
  StepOpts o;
  if (opt) {
    o.fuse = opt->fuse_select != 0;
    o.unified = opt->fuse_select == 2 || opt->fuse_select == 3;
    o.coop = opt->fuse_select == 3;
    o.app_k = opt->append_k_rows;
    o.app_v = opt->append_v_rows;
    o.app_pos = opt->append_pos;
    o.side = static_cast<cudaStream_t>(opt->side_stream);
    o.fork = static_cast<cudaEvent_t>(opt->fork_event);
    o.select = static_cast<cudaEvent_t>(opt->select_event);
    o.full = static_cast<cudaEvent_t>(opt->full_event);
    o.join = static_cast<cudaEvent_t>(opt->join_event);
    o.reuse_wait = static_cast<cudaEvent_t>(opt->reuse_wait_event);
    o.layer_events = opt->layer_events;
    if (int e = mirror_view(opt, &o.idx_mirror)) return e;
  }
  return decode_step_impl(g, q, k, v, n_valid, actions, budget, sel_group, refine, sinks, recent,
                          out, idx, k_stride, ws, ws_bytes, stream, nullptr, o);
}

int hylra_decode_step_offload(const hylra_geometry* g, const void* q, const void* k_full,
                              const void* v_full, const void* k_reuse, const void* v_reuse,
                              int n_valid, const uint8_t* actions, int budget, int sel_group,
                              int refine, int sinks, int recent, float* out, int32_t* idx,
                              int k_stride, void* ws, size_t ws_bytes, void* stream) {
  if (int e = check_geometry(g)) return e;
  if (!actions) return fail(HYLRA_ERR_CONFIGURATION, "actions is NULL");
  bool any_reuse = false;
  for (int l = 0; l < g->num_layers; ++l) any_reuse |= actions[l] == 0;
  SplitKv sp{};
  if (int e = device_view(k_full, &sp.kf, "k_full")) return e;
  if (int e = device_view(v_full, &sp.vf, "v_full")) return e;
  if (any_reuse) {
    if (int e = device_view(k_reuse, &sp.kr, "k_reuse")) return e;
    if (int e = device_view(v_reuse, &sp.vr, "v_reuse")) return e;
  }
  return decode_step_impl(g, q, nullptr, nullptr, n_valid, actions, budget, sel_group, refine,
                          sinks, recent, out, idx, k_stride, ws, ws_bytes, stream, &sp);
}

int hylra_append_kv(const hylra_geometry* g, void* k, void* v, const void* k_rows,
                    const void* v_rows, int pos, int n_layers, const int32_t* layer_ids,
                    void* stream) {
  return append_impl(g, k, v, k_rows, v_rows, pos, n_layers, layer_ids, nullptr,
                     static_cast<cudaStream_t>(stream));
}

int hylra_append_kv_checked(const hylra_geometry* g, void* k, void* v, const void* k_rows,
                            const void* v_rows, int pos, int n_layers, const int32_t* layer_ids,
                            void* ws, void* stream) {
  if (!ws) return fail(HYLRA_ERR_CONFIGURATION, "NULL workspace");
  return append_impl(g, k, v, k_rows, v_rows, pos, n_layers, layer_ids, static_cast<int*>(ws),
                     static_cast<cudaStream_t>(stream));
}

int hylra_check_cache(const hylra_geometry* g, const void* k, const void* v, int n_valid,
                      int n_layers, const int32_t* layer_ids, void* ws, void* stream) {
  if (int e = check_geometry(g)) return e;
  if (!k || !v || !ws) return fail(HYLRA_ERR_CONFIGURATION, "NULL pointer argument");
  if (n_valid < 1 || n_valid > g->capacity)
    return fail(HYLRA_ERR_INVALID_INPUT, "n_valid %d not in [1, capacity=%d]", n_valid,
                g->capacity);
  const int L = layer_ids ? n_layers : g->num_layers;
  if (L < 1 || L > kMaxSlots)
    return fail(HYLRA_ERR_CONFIGURATION, "n_layers %d not in [1, %d]", L, kMaxSlots);
  CheckParams p{};
  const int es = g->dtype == HYLRA_BF16 ? 2 : 4;
  const int64_t bytes = (int64_t)n_valid * g->head_dim * es;
  if (bytes % 16 || (g->kv_stride_layer * es) % 16 || (g->kv_stride_batch * es) % 16 ||
      (g->kv_stride_head * es) % 16 || reinterpret_cast<uintptr_t>(k) % 16 ||
      reinterpret_cast<uintptr_t>(v) % 16)
    return fail(HYLRA_ERR_CONFIGURATION, "cache check needs 16-byte aligned rows and strides");
  p.k = static_cast<const uint8_t*>(k);
  p.v = static_cast<const uint8_t*>(v);
  p.flags = static_cast<int*>(ws);
  p.kv_sl = g->kv_stride_layer * es;
  p.kv_sb = g->kv_stride_batch * es;
  p.kv_sh = g->kv_stride_head * es;
  p.block_chunks = bytes / 16;
  p.B = g->batch;
  p.Hkv = g->kv_heads;
  p.bf16 = g->dtype == HYLRA_BF16;
  p.n_layers = L;
  for (int i = 0; i < L; ++i) {
    const int l = layer_ids ? layer_ids[i] : i;
    if (l < 0 || l >= g->num_layers)
      return fail(HYLRA_ERR_CONFIGURATION, "layer id %d out of range", l);
    p.layers[i] = l;
  }
  // a few waves of CTAs over all blocks
  const int64_t blocks = 2ll * L * g->batch * g->kv_heads;
  if (blocks > 65535) return fail(HYLRA_ERR_CONFIGURATION, "too many cache blocks to check");
  const int64_t per_cta = (int64_t)kCheckThreads * kCheckUnroll;
  const int64_t want = std::max<int64_t>(1, 8ll * num_sms() * 8 / blocks);
  const int gx = (int)std::min<int64_t>(want, (p.block_chunks + per_cta - 1) / per_cta);
  check_finite_kernel<<<dim3(gx, (unsigned)blocks), kCheckThreads, 0,
                        static_cast<cudaStream_t>(stream)>>>(p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_check(cudaGetLastError(), "cache check launch");
}

}  // extern "C"

namespace {
int append_impl(const hylra_geometry* g, void* k, void* v, const void* k_rows,
                const void* v_rows, int pos, int n_layers, const int32_t* layer_ids, int* flags,
                cudaStream_t st) {
  if (int e = check_geometry(g)) return e;
  if (!k || !v) return fail(HYLRA_ERR_CONFIGURATION, "NULL cache pointer");
  if (pos < 0 || pos >= g->capacity)
    return fail(HYLRA_ERR_INVALID_INPUT, "pos %d not in [0, capacity=%d)", pos, g->capacity);
  const int L = layer_ids ? n_layers : g->num_layers;
  if (L < 1 || L > kMaxSlots)
    return fail(HYLRA_ERR_CONFIGURATION, "n_layers %d not in [1, %d]", L, kMaxSlots);
  AppendParams p{};
  if (int e = device_view(k_rows, reinterpret_cast<const void**>(&p.k_rows), "k_rows")) return e;
  if (int e = device_view(v_rows, reinterpret_cast<const void**>(&p.v_rows), "v_rows")) return e;
  const int es = g->dtype == HYLRA_BF16 ? 2 : 4;
  const int64_t row_bytes = (int64_t)g->head_dim * es;
  if (row_bytes % 16 != 0 || (g->kv_stride_layer * es) % 16 != 0 ||
      (g->kv_stride_batch * es) % 16 != 0 || (g->kv_stride_head * es) % 16 != 0 ||
      reinterpret_cast<uintptr_t>(k) % 16 != 0 || reinterpret_cast<uintptr_t>(v) % 16 != 0 ||
      reinterpret_cast<uintptr_t>(p.k_rows) % 16 != 0 ||
      reinterpret_cast<uintptr_t>(p.v_rows) % 16 != 0)
    return fail(HYLRA_ERR_CONFIGURATION, "append needs 16-byte aligned rows and strides");
  p.k = static_cast<uint8_t*>(k);
  p.v = static_cast<uint8_t*>(v);
  p.kv_sl = g->kv_stride_layer * es;
  p.kv_sb = g->kv_stride_batch * es;
  p.kv_sh = g->kv_stride_head * es;
  p.pos_bytes = (int64_t)pos * row_bytes;
  p.B = g->batch;
  p.Hkv = g->kv_heads;
  p.chunks = (int)(row_bytes / 16);
  p.n_layers = L;
  for (int i = 0; i < L; ++i) {
    const int l = layer_ids ? layer_ids[i] : i;
    if (l < 0 || l >= g->num_layers)
      return fail(HYLRA_ERR_CONFIGURATION, "layer id %d out of range", l);
    p.layers[i] = l;
  }
  const int64_t total = 2ll * L * g->batch * g->kv_heads * p.chunks;
  const unsigned blocks = (unsigned)((total + kAppendThreads - 1) / kAppendThreads);
  p.flags = flags;
  p.bf16 = g->dtype == HYLRA_BF16;
  append_kv_kernel<<<blocks, kAppendThreads, 0, st>>>(p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_check(cudaGetLastError(), "append launch");
}
}  // namespace

extern "C" {

int hylra_augment_selection(const int32_t* idx, int rows, int k_eff, int k_stride, int n_valid,
                            int sinks, int recent, int32_t* out, int out_stride,
                            int32_t* counts, void* stream) {
  if (!idx || !out || !counts) return fail(HYLRA_ERR_CONFIGURATION, "NULL pointer argument");
  if (sinks < 0 || recent < 0)
    return fail(HYLRA_ERR_INVALID_INPUT, "include_sinks and include_recent must be >= 0");
  if (rows < 1 || k_eff < 1 || k_eff > k_stride || n_valid < 1)
    return fail(HYLRA_ERR_INVALID_INPUT, "invalid augmentation dimensions");
  if (out_stride < std::min(n_valid, k_eff + sinks + recent))
    return fail(HYLRA_ERR_CONFIGURATION, "out_stride %d too small", out_stride);
  augment_kernel<<<rows, kPoolThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      idx, k_stride, k_eff, n_valid, sinks, recent, out, out_stride, counts);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_check(cudaGetLastError(), "augment launch");
}

int hylra_block_select(const hylra_geometry* g, const float* scores, int n_slots, int n_valid,
                       int block_budget, int block_size, int sel_group, const void* q,
                       const void* k, const int32_t* layer_ids, int32_t* blocks, int bk_stride,
                       int32_t* tokens, int tok_stride, int32_t* counts, int32_t* info, void* ws,
                       size_t ws_bytes, void* stream) {
  if (int e = check_geometry(g)) return e;
  if (!scores || !blocks || !ws) return fail(HYLRA_ERR_CONFIGURATION, "NULL pointer argument");
  if (n_valid < 1 || n_valid > g->capacity)
    return fail(HYLRA_ERR_INVALID_INPUT, "n_valid %d not in [1, capacity]", n_valid);
  if (block_size < 1) return fail(HYLRA_ERR_INVALID_INPUT, "block_size must be >= 1");
  if (sel_group < 1 || g->kv_heads % sel_group != 0)
    return fail(HYLRA_ERR_CONFIGURATION, "sel_group %d does not divide kv_heads", sel_group);
  if (n_slots < 1 || n_slots > kMaxSlots)
    return fail(HYLRA_ERR_CONFIGURATION, "n_slots %d not in [1, %d]", n_slots, kMaxSlots);
  const int nb = (n_valid + block_size - 1) / block_size;
  const size_t need = kHeader + sizeof(float) * (size_t)n_slots * g->batch *
                                    (g->kv_heads / sel_group) * nb_stride_of(nb);
  if (ws_bytes < need)
    return fail(HYLRA_ERR_CONFIGURATION, "workspace %zu B < required %zu B", ws_bytes, need);
  return launch_block_select(g, scores, n_slots, n_valid, block_budget, block_size, sel_group, q,
                             k, layer_ids, reinterpret_cast<float*>(static_cast<uint8_t*>(ws) +
                                                                    kHeader),
                             blocks, bk_stride, tokens, tok_stride, counts, info,
                             static_cast<int*>(ws), static_cast<cudaStream_t>(stream));
}

size_t hylra_decode_step_blocks_workspace_bytes(const hylra_geometry* g, const uint8_t* actions,
                                                int n_valid, int block_budget, int block_size,
                                                int sel_group) {
  StepLayout s;
  if (block_size < 1 || step_layout(g, actions, n_valid, block_budget, sel_group, &s, block_size))
    return 0;
  return s.total;
}

int hylra_decode_step_blocks_ex(const hylra_geometry* g, const void* q, const void* k,
                                const void* v, int n_valid, const uint8_t* actions,
                                int block_budget, int block_size, int sel_group, int refine,
                                float* out, int32_t* blocks, int bk_stride, void* ws,
                                size_t ws_bytes, void* stream, const hylra_step_options* opt) {
  if (block_size < 1) return fail(HYLRA_ERR_INVALID_INPUT, "block_size must be >= 1");
  StepLayout s;
  if (int e = step_layout(g, actions, n_valid, block_budget, sel_group, &s, block_size)) return e;
  if (!ws || ws_bytes < s.total)
    return fail(HYLRA_ERR_CONFIGURATION, "workspace %zu B < required %zu B", ws_bytes, s.total);
  if (!blocks || bk_stride < s.bb)
    return fail(HYLRA_ERR_CONFIGURATION, "block output stride %d < %d", bk_stride, s.bb);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  int* flags = reinterpret_cast<int*>(w);
  float* scores = reinterpret_cast<float*>(w + s.off_scores);
  int32_t* toks = reinterpret_cast<int32_t*>(w + s.off_tokens);
  int32_t* cnts = reinterpret_cast<int32_t*>(w + s.off_counts);
  const int nf = (int)s.full_ids.size();
  const int nr = (int)s.reuse_ids.size();
  const int nb = (n_valid + block_size - 1) / block_size;
  const bool single = opt && opt->fuse_select == 2 && sel_group == 1 && use_mma_path(g) &&
                      fused_select_fits(g, nb);
  int32_t* mirror = nullptr;
  if (int e = mirror_view(opt, &mirror)) return e;
  // the step's new K/V rows: written by the single-launch kernel, else appended ahead
  StepAppend app{};
  if (opt && (opt->append_k_rows || opt->append_v_rows))
    if (int e = step_append(g, k, v, opt->append_k_rows, opt->append_v_rows, opt->append_pos,
                            n_valid, single, &app, flags, st))
      return e;
  // single-launch block step (fuse_select = 2): the final CTA of every FULL pair pools its
  // row into blocks, selects them and writes the token coverage the REUSE items gather
  if (single) {
    std::vector<int32_t> ab_ids, ab_slot, b_ids, b_slot;
    for (int i = 0; i < nf; ++i) {
      const int l = s.full_ids[i];
      const bool feeds = l + 1 < g->num_layers && actions[l + 1] == 0;
      (feeds ? ab_ids : b_ids).push_back(l);
      (feeds ? ab_slot : b_slot).push_back(i);
    }
    ab_ids.insert(ab_ids.end(), b_ids.begin(), b_ids.end());
    ab_slot.insert(ab_slot.end(), b_slot.begin(), b_slot.end());
    BlockRows br;
    br.block_size = block_size;
    br.n_tokens = n_valid;
    br.row_stride = nb_stride_of(nb);
    br.tok_scores = scores;
    SelectParams sp{};
    if (int e = build_select_params(&sp, g, reinterpret_cast<float*>(w + s.off_bscores), nf, nb,
                                    block_budget, 1, refine ? q : nullptr, refine ? k : nullptr,
                                    ab_ids.data(), blocks, bk_stride, nullptr, flags, br, nullptr,
                                    ab_slot.data()))
      return e;
    sp.idx_mirror = mirror;
    sp.cov_tokens = toks;
    sp.cov_counts = cnts;
    sp.cov_stride = s.tok_stride;
    AttnParams pf{}, pr{};
    AttnLayout lf{}, lr{};
    if (int e = make_attn_params(&pf, &lf, g, false, q, k, v, n_valid, n_valid, nf, ab_ids.data(),
                                 nullptr, nullptr, nullptr, 0, 1, out, scores, w + s.off_attn,
                                 s.attn_bytes, flags, nullptr, 0, s.ctr_f(w)))
      return e;
    pf.fuse_select = nf;
    const long items_f = (long)lf.splits * g->kv_heads * g->batch * nf;
    long items_r = 0;
    if (nr > 0) {
      if (int e = make_attn_params(&pr, &lr, g, true, q, k, v, n_valid, s.k_eff, nr,
                                   s.reuse_ids.data(), s.reuse_src.data(), toks, cnts,
                                   s.tok_stride, 1, out, nullptr, w + s.off_attn_r,
                                   s.attn_bytes_r, flags, nullptr, 0, s.ctr_r(w)))
        return e;
      items_r = (long)lr.splits * g->kv_heads * g->batch * nr;
    }
    if (items_f + items_r > INT32_MAX) return fail(HYLRA_ERR_CONFIGURATION, "grid too large");
    CUtensorMap tk{}, tv{};
    if (int e = encode_kv_map(&tk, g, k, g->num_layers)) return e;
    if (int e = encode_kv_map(&tv, g, v, g->num_layers)) return e;
    StepSync ss{};
    ss.ctr = reinterpret_cast<int*>(w + s.off_sync);
    ss.ready = ss.ctr + 64;
    ss.group = ss.ready + s.n_ready;
    ss.n_ready = s.n_ready;
    ss.n_full_items = (int)items_f;
    ss.n_items = (int)(items_f + items_r);
    ss.app = app;
    return dispatch_step(g, st, tk, tv, pf, pr, sp, ss);
  }
  if (int e = launch_attention(g, false, q, k, v, n_valid, n_valid, nf, s.full_ids.data(), nullptr,
                               nullptr, nullptr, 0, 1, out, scores, w + s.off_attn, s.attn_bytes,
                               flags, st, nullptr, 0, nullptr, 0, nullptr, 0, 0, s.ctr_f(w)))
    return e;
  if (int e = launch_block_select(g, scores, nf, n_valid, block_budget, block_size, sel_group,
                                  refine ? q : nullptr, refine ? k : nullptr, s.full_ids.data(),
                                  reinterpret_cast<float*>(w + s.off_bscores), blocks, bk_stride,
                                  s.reuse_ids.empty() ? nullptr : toks, s.tok_stride, cnts,
                                  nullptr, flags, st, mirror))
    return e;
  if (!s.reuse_ids.empty()) {
    // whole blocks of 64-row multiples can stream as TMA tiles (the coverage rows are
    // contiguous within a block; HYLRA_BLOCK_TILES=1), else the coverage is gathered
    const bool tiles = use_mma_path(g) && block_size % kTileRows == 0 && !block_tiles_off();
    if (int e = launch_attention(g, true, q, k, v, n_valid, s.k_eff, (int)s.reuse_ids.size(),
                                 s.reuse_ids.data(), s.reuse_src.data(), toks, cnts, s.tok_stride,
                                 sel_group, out, nullptr, w + s.off_attn_r, s.attn_bytes_r, flags,
                                 st, nullptr, 0, nullptr, 0, tiles ? blocks : nullptr, bk_stride,
                                 block_size, s.ctr_r(w)))
      return e;
  }
  return HYLRA_OK;
}

int hylra_decode_step_blocks(const hylra_geometry* g, const void* q, const void* k,
                             const void* v, int n_valid, const uint8_t* actions,
                             int block_budget, int block_size, int sel_group, int refine,
                             float* out, int32_t* blocks, int bk_stride, void* ws,
                             size_t ws_bytes, void* stream) {
  return hylra_decode_step_blocks_ex(g, q, k, v, n_valid, actions, block_budget, block_size,
                                     sel_group, refine, out, blocks, bk_stride, ws, ws_bytes,
                                     stream, nullptr);
}

int hylra_overlap_counts(const int32_t* idx, int steps, int layers, int rows, int k,
                         int k_stride, int n_tokens, int32_t* counts, void* stream) {
  if (!idx || !counts) return fail(HYLRA_ERR_CONFIGURATION, "NULL pointer argument");
  if (steps < 1 || layers < 1 || rows < 1 || k < 1 || k_stride < k || n_tokens < 1)
    return fail(HYLRA_ERR_INVALID_INPUT, "invalid overlap dimensions");
  // chunks: as large as 200 KB of bitmaps allows, then split until the grid covers about
  // two CTAs per SM
  const size_t budget = 200 * 1024;
  int chunk = (int)std::min<size_t>(budget / (layers * 4) * 32, (size_t)((n_tokens + 31) & ~31));
  chunk = std::max(32, chunk & ~31);
  while (chunk > 1024 && (int64_t)rows * steps * ((n_tokens + chunk - 1) / chunk) < 2 * num_sms())
    chunk = std::max(1024, ((chunk / 2) + 31) & ~31);
  const size_t smem = (size_t)layers * (chunk / 32) * 4;
  if (smem > 220 * 1024) return fail(HYLRA_ERR_CONFIGURATION, "too many layers (%d)", layers);
  if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(overlap_counts_kernel),
                                      220 * 1024))
    return cuda_check(e, "overlap attribute");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the chunks add their counts: start from zero
  if (int e = cuda_check(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)steps * rows *
                                                        layers * layers, st),
                         "overlap counts zero"))
    return e;
  dim3 grid(rows, steps, (n_tokens + chunk - 1) / chunk);
  overlap_counts_kernel<<<grid, kOvThreads, smem, st>>>(idx, layers, rows, k, k_stride, n_tokens,
                                                        chunk, counts);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_check(cudaGetLastError(), "overlap launch");
}

int hylra_read_flags(const void* ws, int32_t* flags_host, void* stream) {
  if (!ws || !flags_host) return fail(HYLRA_ERR_CONFIGURATION, "NULL pointer argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int e = cuda_check(cudaMemcpyAsync(flags_host, ws, sizeof(int32_t), cudaMemcpyDeviceToHost, st),
                         "read flags"))
    return e;
  return cuda_check(cudaStreamSynchronize(st), "read flags sync");
}

int hylra_clear_flags(void* ws, void* stream) {
  if (!ws) return fail(HYLRA_ERR_CONFIGURATION, "NULL pointer argument");
  return cuda_check(
      cudaMemsetAsync(ws, 0, 2 * sizeof(int32_t), static_cast<cudaStream_t>(stream)),
      "clear flags");
}

}  // extern "C"
