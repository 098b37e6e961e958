// attention.cuh — FULL (split-K flash-decode + fused selection-score emission) and
// REUSE (sparse-gather subset attention) kernels.
//
// Reference semantics (pkg/src/layerreuse/):
//   FULL  : attention.py:210-226 full_attention — logits = K q / sqrt(d), max-subtracted
//           softmax, out = w^T V — for every query head, plus engine.py:177-181, the
//           selection score agg[n] = sum_h logits_h[n].
//   REUSE : attention.py:229-241 _subset_attention — gather K[idx], V[idx], softmax
//           renormalised over the subset only.
//
// One CTA serves one (layer slot, b, kv-head) pair and a contiguous range of rows
// (split-K). All G = Hq/Hkv query heads of the group are processed together so each
// K/V row is read from HBM exactly once per layer. Splits are merged with the
// log-sum-exp rule by the last CTA of the pair to finish (no second launch).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "select.cuh"

namespace hylra {

constexpr int kTileRows = 64;   // rows per pipeline stage
constexpr int kConsumerWarps = 4;
// REUSE producer warps: the gather's cp.async rows of a stage are split between them
// (HYLRA_GATHER_PRODUCERS in {1, 2, 4} at build time; FULL always has one TMA warp).
#ifndef HYLRA_GATHER_PRODUCERS
#define HYLRA_GATHER_PRODUCERS 2
#endif
constexpr int kGatherProducers = HYLRA_GATHER_PRODUCERS;
template <bool GATHER>
constexpr int attn_threads() { return 32 * (kConsumerWarps + (GATHER ? kGatherProducers : 1)); }
constexpr int kMaxG = 16;
constexpr int kIdxStage = 2048;  // REUSE: indices staged in shared memory per CTA
// FULL CTAs use the same 8 KB for their share of the score-row histogram: kHistBins 16-bit
// counters packed two per word (a split holds < 65536 tokens: hylra_abi.cu checks)
static_assert(kIdxStage * 4 == kHistBins * 2, "the staging area holds the 16-bit histogram");

struct AttnParams {
  const void* q;
  const void* k;
  const void* v;
  float* out;
  float* scores;        // FULL: [slot][b][kh][cap] or null
  unsigned* hist;       // FULL: [slot][b][kh][kHistBins] first-level histogram of the score
                        // row (select.cuh), accumulated by every split, or null
  const int32_t* idx;   // REUSE: [src_slot][b][group][k_stride]
  const int32_t* counts;  // REUSE: optional rows per selection row (block coverage)
  // block-mode REUSE by TMA tiles (blk != null; tensor-core path, blk_size % 64 == 0): the
  // selection row's ascending block ids [src_slot][b][grp][blk_stride]; tile t of the pair
  // covers cache rows blk[t / (blk_size/64)] * blk_size + (t % (blk_size/64)) * 64 + [0, 64)
  const int32_t* blk;
  int blk_stride, blk_size;
  float* ws_o;          // [pair][split][G][D]
  float* ws_ml;         // [pair][split][G][2]
  int* counters;        // [pair]
  int* flags;
  int64_t q_sl, q_sb;
  int64_t kv_sl, kv_sb, kv_sh;
  int64_t o_sl, o_sb;
  int B, Hkv, G, cap;
  int n_valid;          // valid cache rows
  int n_rows;           // rows this op attends over: n_valid (FULL) or k_eff (REUSE)
  int n_slots;          // layer slots of the launch
  int splits;
  int tiles_per_split;
  int k_stride, sel_group, n_groups;
  float scale_log2;     // log2(e) / sqrt(d)
  int prefetch;         // REUSE: L2 prefetch distance in tiles
  float inv_sqrt_d;
  int layers[kMaxSlots];     // q / out layer of each slot
  int kv_layers[kMaxSlots];  // K / V layer of each slot (differs for split caches)
  int src_slot[kMaxSlots];
  // FULL: launch-local slots [0, fuse_select) select their rows inside the kernel (the last
  // CTA of a pair, once the pair's score row is complete); SelectParams come alongside
  int fuse_select;
  // layer-sequential launches (hylra_decode_layer prefetch): the producer warps load K/V (and,
  // REUSE, the indices) before griddepcontrol.wait — the caller guarantees the previous launch
  // on the stream wrote none of them — so the pipeline fills while that launch drains; the
  // consumer warps still wait before reading q
  int early;
  // REUSE gather by TMA (tile::gather4 through 2-D row views of K and V passed in the tmk /
  // tmv slots; contiguous caches, uniform rows, indices staged): rows of (kv layer, b, kh)
  // start at row ((kvl B + b) Hkv + kh) cap of the view; 0: the cp.async gather
  int gather_tma;
  int gather_rows;  // rows of the 2-D views (an index past them is zero-filled)
  int cap_rows;     // cache rows per (kv layer, b, kh) block (capacity)
  int bulk_merge;   // split-K final merge: partials staged by cp.async.bulk (merge_and_store)
  // REUSE launched as clusters of its `splits` CTAs (grid.x == splits <= 16): the splits of a
  // pair merge through distributed shared memory (cluster_merge_store), no global round trips
  int cluster_merge;
};

// Stage n selection indices from global into shared memory, validated (out-of-range ->
// row 0 + HYLRA_FLAG_INDEX_OUT_OF_RANGE). The `parts` producer warps share the work (warp
// `part` takes every parts-th 32-group slice) with 16-byte loads when the source is 16-byte
// aligned: a 2048-row range is one round trip (8 x 16 B in flight per lane), not the 8
// dependent rounds of one warp's 4-byte loads (~1 us each before the first gather). The
// caller synchronises the producer warps afterwards.
__device__ __forceinline__ void stage_indices(const int32_t* __restrict__ src, int n, int n_valid,
                                              int32_t* dst, int* flags, int lane, int part,
                                              int parts) {
  constexpr int U = 8;
  bool bad = false;
  auto fix = [&](int v) {
    const bool ok = v >= 0 && v < n_valid;
    bad |= !ok;
    return ok ? v : 0;
  };
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int n4 = n >> 2;
    const int4* s4 = reinterpret_cast<const int4*>(src);
    int4* d4 = reinterpret_cast<int4*>(dst);
    for (int g0 = 0; g0 < n4; g0 += 32 * parts * U) {
      int4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int g = g0 + (u * parts + part) * 32 + lane;
        // coherent loads: the indices may have been written earlier in a single-launch step
        r[u] = g < n4 ? __ldcg(s4 + g) : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int g = g0 + (u * parts + part) * 32 + lane;
        if (g < n4) d4[g] = make_int4(fix(r[u].x), fix(r[u].y), fix(r[u].z), fix(r[u].w));
      }
    }
    if (part == 0 && lane < (n & 3)) {
      const int j = (n4 << 2) + lane;
      dst[j] = fix(__ldcg(src + j));
    }
  } else {
    for (int j0 = 0; j0 < n; j0 += 32 * parts * U) {
      int r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + (u * parts + part) * 32 + lane;
        r[u] = (j < n) ? __ldcg(src + j) : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + (u * parts + part) * 32 + lane;
        if (j < n) dst[j] = fix(r[u]);
      }
    }
  }
  if (bad) atomicOr(flags, 1);
}

// ---------------------------------------------------------------------------------
// Cross-warp merge + split-K combine (shared by both kernel families).
// sm_m/sm_l: [4][16], sm_o: [4][16][D] partial states of the 4 consumer warps, with
// m in raw dot units (scaled by scale_log2 inside exp2).
// scratch (optional, scratch_floats floats of shared memory the caller no longer uses): the
// final CTA stages every split's (m, l) there and merges the output partials with 8 float4
// L2 loads in flight per thread — a one-layer launch at B = 1 has ~40 splits per pair, whose
// merge as dependent per-split loads took ~20 us. Same arithmetic, same order, either way.
// bulk (optional, bulk_cap bytes of drained pipeline buffers, 16-byte aligned): when the
// pair's partials fit, the final CTA pulls all of them (and the (m, l) pairs) into shared
// memory with cp.async.bulk — ONE round trip instead of one per 8 splits: the 37-split merge
// of a one-layer FULL launch at B = 1 was the launch's ~7 us tail (scripts/trace_layer.py).
template <int D>
__device__ __forceinline__ bool merge_and_store(const AttnParams& p, int slot, int b, int kh,
                                                int split, const float* sm_m,
                                                const float* sm_l, const float* sm_o,
                                                int tid, int nthreads, int bar_id,
                                                float* scratch = nullptr,
                                                int scratch_floats = 0,
                                                uint8_t* bulk = nullptr,
                                                uint32_t bulk_cap = 0) {
  const int G = p.G;
  const int layer = p.layers[slot];
  const int pair = (slot * p.B + b) * p.Hkv + kh;
  float* out_base = p.out + layer * p.o_sl + b * p.o_sb + (int64_t)(kh * G) * D;
  const float c = p.scale_log2;
  if (p.splits == 1) {
    for (int e = tid; e < G * D; e += nthreads) {
      const int g = e / D, d = e % D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, sm_m[w * 16 + g]);
      float acc = 0.f, L = 0.f;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) {
        const float mw = sm_m[w * 16 + g];
        const float s = (mw == -INFINITY) ? 0.f : exp2f((mw - M) * c);
        acc += sm_o[(w * 16 + g) * D + d] * s;
        L += sm_l[w * 16 + g] * s;
      }
      const float val = acc / L;
      if (!isfinite(val)) atomicOr(p.flags, 2);  // NaN/inf in q, K or V
      out_base[g * D + d] = val;
    }
    return true;
  }
  const int part = pair * p.splits + split;
  float* wo = p.ws_o + (int64_t)part * G * D;
  float* wml = p.ws_ml + (int64_t)part * G * 2;
  for (int e = tid; e < G * D; e += nthreads) {
    const int g = e / D, d = e % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, sm_m[w * 16 + g]);
    float acc = 0.f, L = 0.f;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) {
      const float mw = sm_m[w * 16 + g];
      const float s = (mw == -INFINITY) ? 0.f : exp2f((mw - M) * c);
      acc += sm_o[(w * 16 + g) * D + d] * s;
      L += sm_l[w * 16 + g] * s;
    }
    wo[g * D + d] = acc;
    if (d == 0) {
      wml[g * 2 + 0] = M;
      wml[g * 2 + 1] = L;
    }
  }
  __threadfence();
  __shared__ int s_last;
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads) : "memory");
  if (tid == 0) {
    const int prev = atomicAdd(p.counters + pair, 1);
    s_last = (prev == p.splits - 1);
  }
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads) : "memory");
  if (!s_last) return false;
  __threadfence();
  const float* po = p.ws_o + (int64_t)pair * p.splits * G * D;
  const float* pml = p.ws_ml + (int64_t)pair * p.splits * G * 2;
  const int SG = p.splits * G;
  if (scratch != nullptr && 3 * SG + 2 * kMaxG <= scratch_floats) {
    float* s_ml = scratch;          // [split][g][m, l]
    float* s_sc = scratch + 2 * SG;  // [split][g] rescale factor
    float* s_M = s_sc + SG;          // [g]
    float* s_L = s_M + kMaxG;        // [g]
    const uint32_t po_bytes = (uint32_t)SG * D * 4;
    const uint32_t ml_bytes = (uint32_t)SG * 8;
    const bool use_bulk = bulk != nullptr && po_bytes <= bulk_cap &&
                          (reinterpret_cast<uintptr_t>(po) & 15) == 0;
    const bool ml_bulk = use_bulk && ((reinterpret_cast<uintptr_t>(pml) | ml_bytes) & 15) == 0 &&
                         (smem_u32(s_ml) & 15) == 0;
    __shared__ __align__(8) uint64_t s_bulk_bar;
    if (use_bulk) {
      // every thread's generic accesses of the buffers (ring reads, sm_o) before the async
      // proxy's writes; the partials (other CTAs' stores, acquired above) before its reads
      fence_proxy_async_smem();
      asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads) : "memory");
      if (tid == 0) {
        mbar_init(&s_bulk_bar, 1);
        mbar_fence_init();
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mbar_arrive_expect_tx(&s_bulk_bar, po_bytes + (ml_bulk ? ml_bytes : 0u));
        for (uint32_t off = 0; off < po_bytes; off += 32768u)
          bulk_load(bulk + off, reinterpret_cast<const uint8_t*>(po) + off,
                    min(32768u, po_bytes - off), &s_bulk_bar);
        if (ml_bulk) bulk_load(s_ml, pml, ml_bytes, &s_bulk_bar);
      }
    }
    if (!ml_bulk) {
      const float2* pml2 = reinterpret_cast<const float2*>(pml);
      for (int i = tid; i < SG; i += nthreads) {
        const float2 x = __ldcg(pml2 + i);
        s_ml[2 * i] = x.x;
        s_ml[2 * i + 1] = x.y;
      }
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads) : "memory");
    if (use_bulk) mbar_wait(&s_bulk_bar, 0);
    for (int g = tid; g < G; g += nthreads) {
      float M = -INFINITY;
      for (int s = 0; s < p.splits; ++s) M = fmaxf(M, s_ml[2 * (s * G + g)]);
      s_M[g] = M;
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads) : "memory");
    for (int i = tid; i < SG; i += nthreads) {
      const float ms = s_ml[2 * i];
      s_sc[i] = (ms == -INFINITY) ? 0.f : exp2f((ms - s_M[i % G]) * c);
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads) : "memory");
    for (int g = tid; g < G; g += nthreads) {
      float L = 0.f;
      for (int s = 0; s < p.splits; ++s) L = fmaf(s_ml[2 * (s * G + g) + 1], s_sc[s * G + g], L);
      s_L[g] = L;
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads) : "memory");
    constexpr int D4 = D / 4;
    const float4* po4 = reinterpret_cast<const float4*>(po);
    for (int e4 = tid; e4 < G * D4; e4 += nthreads) {
      const int g = e4 / D4, d = (e4 % D4) * 4;
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
      int s = 0;
      auto add = [&](const float4& x, float sc) {
        a0 = fmaf(x.x, sc, a0);
        a1 = fmaf(x.y, sc, a1);
        a2 = fmaf(x.z, sc, a2);
        a3 = fmaf(x.w, sc, a3);
      };
      if (use_bulk) {
        const float4* bo4 = reinterpret_cast<const float4*>(bulk);
        for (; s < p.splits; ++s) add(bo4[s * G * D4 + e4], s_sc[s * G + g]);
      }
      for (; s + 8 <= p.splits; s += 8) {
        float4 x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = __ldcg(po4 + (int64_t)(s + u) * G * D4 + e4);
#pragma unroll
        for (int u = 0; u < 8; ++u) add(x[u], s_sc[(s + u) * G + g]);
      }
      for (; s < p.splits; ++s) add(__ldcg(po4 + (int64_t)s * G * D4 + e4), s_sc[s * G + g]);
      const float L = s_L[g];
      const float v0 = a0 / L, v1 = a1 / L, v2 = a2 / L, v3 = a3 / L;
      if (!(isfinite(v0) && isfinite(v1) && isfinite(v2) && isfinite(v3)))
        atomicOr(p.flags, 2);  // NaN/inf in q, K or V
      float* o = out_base + g * D + d;
      o[0] = v0;
      o[1] = v1;
      o[2] = v2;
      o[3] = v3;
    }
    if (use_bulk && tid == 0) mbar_inval(&s_bulk_bar);
  } else {
    for (int e = tid; e < G * D; e += nthreads) {
      const int g = e / D, d = e % D;
      float M = -INFINITY;
      for (int s = 0; s < p.splits; ++s) M = fmaxf(M, __ldcg(pml + (s * G + g) * 2));
      float acc = 0.f, L = 0.f;
      for (int s = 0; s < p.splits; ++s) {
        const float ms = __ldcg(pml + (s * G + g) * 2);
        const float sc = (ms == -INFINITY) ? 0.f : exp2f((ms - M) * c);
        acc = fmaf(__ldcg(po + (int64_t)(s * G + g) * D + d), sc, acc);
        L = fmaf(__ldcg(pml + (s * G + g) * 2 + 1), sc, L);
      }
      const float val = acc / L;
      if (!isfinite(val)) atomicOr(p.flags, 2);  // NaN/inf in q, K or V
      out_base[g * D + d] = val;
    }
  }
  if (tid == 0) p.counters[pair] = 0;  // leave the workspace zeroed for the next call
  return true;
}

// Cluster barrier over every thread of the CTA cluster (release / acquire: shared-memory
// writes before it are visible to the peers' DSMEM reads after it).
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}

// Split-K merge of a REUSE launch whose splits of one pair form a thread-block cluster
// (p.cluster_merge = C = splits; rank = split). Each CTA combines its 4 warps into its split
// partial IN ITS OWN SHARED MEMORY (`part`: [G][D] o, then [G][2] (m, l)); after a cluster
// barrier every rank merges a 1/C slice of the pair's G x D outputs, reading all C partials
// through DSMEM, and stores it. Arithmetic and order are merge_and_store's (the CTA
// partial, then the staged merge's max / scale / fmaf chain over splits in ascending
// order), so the outputs are bit-identical to the global-memory merge — without the
// partial stores, fence, counter atomic and L2 re-reads (~3-5 us of a one-layer REUSE
// launch at B = 1, scripts/trace_layer.py). The consumer threads call it; the producer
// warps meet both cluster barriers in attn_mma_kernel.
template <int D>
__device__ __forceinline__ void cluster_merge_store(const AttnParams& p, int slot, int b, int kh,
                                                    int split, const float* sm_m,
                                                    const float* sm_l, const float* sm_o,
                                                    float* part, float* scratch) {
  const int G = p.G, C = p.cluster_merge, tid = threadIdx.x;
  constexpr int NT = kConsumerWarps * 32;
  const int layer = p.layers[slot];
  float* out_base = p.out + layer * p.o_sl + b * p.o_sb + (int64_t)(kh * G) * D;
  const float c = p.scale_log2;
  float* pml = part + G * D;
  for (int e = tid; e < G * D; e += NT) {
    const int g = e / D, d = e % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, sm_m[w * 16 + g]);
    float acc = 0.f, L = 0.f;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) {
      const float mw = sm_m[w * 16 + g];
      const float sc = (mw == -INFINITY) ? 0.f : exp2f((mw - M) * c);
      acc += sm_o[(w * 16 + g) * D + d] * sc;
      L += sm_l[w * 16 + g] * sc;
    }
    part[e] = acc;
    if (d == 0) {
      pml[g * 2 + 0] = M;
      pml[g * 2 + 1] = L;
    }
  }
  cluster_sync_all();  // (1) every split's partial is in its CTA's shared memory
  auto cl = cooperative_groups::this_cluster();
  const int SG = C * G;
  float* s_ml = scratch;           // [split][g][m, l]
  float* s_sc = scratch + 2 * SG;  // [split][g]
  float* s_M = s_sc + SG;          // [g]
  float* s_L = s_M + kMaxG;        // [g]
  for (int i = tid; i < SG; i += NT) {
    const float* r = cl.map_shared_rank(pml, i / G);
    s_ml[2 * i] = r[2 * (i % G)];
    s_ml[2 * i + 1] = r[2 * (i % G) + 1];
  }
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  for (int g = tid; g < G; g += NT) {
    float M = -INFINITY;
    for (int s2 = 0; s2 < C; ++s2) M = fmaxf(M, s_ml[2 * (s2 * G + g)]);
    s_M[g] = M;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  for (int i = tid; i < SG; i += NT) {
    const float ms = s_ml[2 * i];
    s_sc[i] = (ms == -INFINITY) ? 0.f : exp2f((ms - s_M[i % G]) * c);
  }
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  for (int g = tid; g < G; g += NT) {
    float L = 0.f;
    for (int s2 = 0; s2 < C; ++s2) L = fmaf(s_ml[2 * (s2 * G + g) + 1], s_sc[s2 * G + g], L);
    s_L[g] = L;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  constexpr int D4 = D / 4;
  const int n4 = G * D4, per = (n4 + C - 1) / C;
  const int e_end = min(n4, (split + 1) * per);
  for (int e4 = split * per + tid; e4 < e_end; e4 += NT) {
    const int g = e4 / D4, d = (e4 % D4) * 4;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    for (int s2 = 0; s2 < C; ++s2) {
      const float4 x = reinterpret_cast<const float4*>(cl.map_shared_rank(part, s2))[e4];
      const float sc = s_sc[s2 * G + g];
      a0 = fmaf(x.x, sc, a0);
      a1 = fmaf(x.y, sc, a1);
      a2 = fmaf(x.z, sc, a2);
      a3 = fmaf(x.w, sc, a3);
    }
    const float L = s_L[g];
    const float v0 = a0 / L, v1 = a1 / L, v2 = a2 / L, v3 = a3 / L;
    if (!(isfinite(v0) && isfinite(v1) && isfinite(v2) && isfinite(v3)))
      atomicOr(p.flags, 2);  // NaN/inf in q, K or V
    float* o = out_base + g * D + d;
    o[0] = v0;
    o[1] = v1;
    o[2] = v2;
    o[3] = v3;
  }
  cluster_sync_all();  // (2) no CTA leaves while a peer may still read its partial
}

// ---------------------------------------------------------------------------------
// Tensor-core path (bf16 K/V/q). 4 consumer warps + 1 producer warp.
// Stage = 64 K rows + 64 V rows in 128B-swizzled boxes of 64 columns (the TMA
// SWIZZLE_128B layout): element (r, col) of a box lives at
//   r*128 + (((col/8) ^ (r%8)) * 16) + (col%8)*2.
// Warp w owns rows 16w..16w+15 of every stage: S = Q K^T via mma.m16n8k16 with the G
// group heads packed into the M=16 rows (rows >= G are zero), online softmax in
// registers, P re-used as the A operand of O += P V (FA2 register layout).
template <int D>
struct MmaSmem {
  static constexpr int kBoxes = D / 64;
  static constexpr int kTileBytes = kTileRows * D * 2;          // one of K or V
  static constexpr int kStageBytes = 2 * kTileBytes;
};

__device__ __forceinline__ uint32_t swz_addr(uint32_t tile_base, int r, int chunk) {
  // chunk = 16-byte column chunk index over the full row (0 .. D/8-1)
  return tile_base + (chunk >> 3) * (kTileRows * 128) + r * 128 + (((chunk & 7) ^ (r & 7)) << 4);
}

// One 64-row stage for one consumer warp (its 16 rows): S = Q K^T on tensor cores, the
// tail mask, the selection-score emission (FULL), the online softmax and O += P V.
// Returns a word that depends on every V fragment loaded from the stage: the caller stores
// it to shared memory before releasing the stage, so the release cannot overtake the last
// ldmatrix reads (see the empty-barrier arrive below).
template <int D, bool GATHER, bool GBIG>
__device__ __forceinline__ uint32_t mma_consume_tile(const AttnParams& p, uint32_t kt, uint32_t vt,
                                                 const uint32_t (&qa)[D / 16][4],
                                                 float (&o)[D / 8][4], float& m0, float& m1,
                                                 float& l0, float& l1, int row0, int n_rows,
                                                 float* score_row, float* score_buf,
                                                 int lane) {
  const int g = lane >> 2;
  const int t = lane & 3;
  const float c = p.scale_log2;
  const int rbase = ((threadIdx.x >> 5) & 3) * 16;
  const int lk_row = rbase + (lane & 7) + ((lane >> 4) << 3);   // K: matrices (n0,k0)(n0,k1)(n1,k0)(n1,k1)
  const int lk_chk = (lane >> 3) & 1;
  const int lv_row = rbase + (lane & 7) + (((lane >> 3) & 1) << 3);  // V: (k0,n)(k1,n)(k0,n+1)(k1,n+1)
  const int lv_chk = lane >> 4;
  // ---- S = Q K^T (16 x 16 per warp)
  float sacc[2][4];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    uint32_t b0, b1, b2, b3;
    ldsm_x4(swz_addr(kt, lk_row, 2 * ks + lk_chk), b0, b1, b2, b3);
    mma_bf16_16816(sacc[0], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
    mma_bf16_16816(sacc[1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b2, b3);
  }

  // ---- mask rows past the end of the range
  const bool tail = row0 + 16 > n_rows;
  if (tail) {
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (row0 + nt * 8 + 2 * t + e >= n_rows) {
          sacc[nt][e] = -INFINITY;
          sacc[nt][2 + e] = -INFINITY;
        }
      }
  }

  // ---- selection score: sum over the group's heads (rows) of q.k, times 1/sqrt(d)
  if (!GATHER && score_row != nullptr) {
    float v00 = sacc[0][0], v01 = sacc[0][1], v10 = sacc[1][0], v11 = sacc[1][1];
    if (GBIG) {
      v00 += sacc[0][2];
      v01 += sacc[0][3];
      v10 += sacc[1][2];
      v11 += sacc[1][3];
    }
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      v00 += __shfl_xor_sync(0xffffffffu, v00, off);
      v01 += __shfl_xor_sync(0xffffffffu, v01, off);
      v10 += __shfl_xor_sync(0xffffffffu, v10, off);
      v11 += __shfl_xor_sync(0xffffffffu, v11, off);
    }
    if (g == 0) {
      const int n0 = row0 + 2 * t;
      const int n1 = row0 + 8 + 2 * t;
      const float s00 = v00 * p.inv_sqrt_d, s01 = v01 * p.inv_sqrt_d;
      const float s10 = v10 * p.inv_sqrt_d, s11 = v11 * p.inv_sqrt_d;
      if (!tail) {
        *reinterpret_cast<float2*>(score_row + n0) = make_float2(s00, s01);
        *reinterpret_cast<float2*>(score_row + n1) = make_float2(s10, s11);
      } else {
        if (n0 < n_rows) score_row[n0] = s00;
        if (n0 + 1 < n_rows) score_row[n0 + 1] = s01;
        if (n1 < n_rows) score_row[n1] = s10;
        if (n1 + 1 < n_rows) score_row[n1 + 1] = s11;
      }
      // the tile's scores for the producer warp's histogram count (released with the stage)
      if (score_buf != nullptr) {
        const int r0 = (row0 & (kTileRows - 1)) + 2 * t;
        *reinterpret_cast<float2*>(score_buf + r0) = make_float2(s00, s01);
        *reinterpret_cast<float2*>(score_buf + r0 + 8) = make_float2(s10, s11);
      }
    }
  }

  // ---- online softmax (row g, and row g+8 when G > 8)
  uint32_t pa0, pa1, pa2, pa3;
  {
    float mx = fmaxf(fmaxf(sacc[0][0], sacc[0][1]), fmaxf(sacc[1][0], sacc[1][1]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float mn = fmaxf(m0, mx);
    const float mu = (mn == -INFINITY) ? 0.f : mn;
    const float alpha = fast_exp2((m0 - mu) * c);
    const float mc = mu * c;
    const float p00 = fast_exp2(fmaf(sacc[0][0], c, -mc));
    const float p01 = fast_exp2(fmaf(sacc[0][1], c, -mc));
    const float p10 = fast_exp2(fmaf(sacc[1][0], c, -mc));
    const float p11 = fast_exp2(fmaf(sacc[1][1], c, -mc));
    l0 = fmaf(l0, alpha, (p00 + p01) + (p10 + p11));
    m0 = mn;
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {
      o[j][0] *= alpha;
      o[j][1] *= alpha;
    }
    pa0 = pack_bf16(p00, p01);
    pa2 = pack_bf16(p10, p11);
  }
  if (GBIG) {
    float mx = fmaxf(fmaxf(sacc[0][2], sacc[0][3]), fmaxf(sacc[1][2], sacc[1][3]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float mn = fmaxf(m1, mx);
    const float mu = (mn == -INFINITY) ? 0.f : mn;
    const float alpha = fast_exp2((m1 - mu) * c);
    const float mc = mu * c;
    const float p00 = fast_exp2(fmaf(sacc[0][2], c, -mc));
    const float p01 = fast_exp2(fmaf(sacc[0][3], c, -mc));
    const float p10 = fast_exp2(fmaf(sacc[1][2], c, -mc));
    const float p11 = fast_exp2(fmaf(sacc[1][3], c, -mc));
    l1 = fmaf(l1, alpha, (p00 + p01) + (p10 + p11));
    m1 = mn;
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {
      o[j][2] *= alpha;
      o[j][3] *= alpha;
    }
    pa1 = pack_bf16(p00, p01);
    pa3 = pack_bf16(p10, p11);
  } else {
    pa1 = 0u;
    pa3 = 0u;
  }

  // ---- O += P V
  uint32_t dep = 0u;
#pragma unroll
  for (int j = 0; j < D / 8; j += 2) {
    uint32_t b0, b1, b2, b3;
    ldsm_x4_t(swz_addr(vt, lv_row, j + lv_chk), b0, b1, b2, b3);
    mma_bf16_16816(o[j], pa0, pa1, pa2, pa3, b0, b1);
    mma_bf16_16816(o[j + 1], pa0, pa1, pa2, pa3, b2, b3);
    dep ^= b0 ^ b1 ^ b2 ^ b3;
  }
  return dep;
}

// Consumer release of a pipeline stage. mbarrier.arrive does not wait for the warp's
// outstanding ldmatrix reads: ptxas scheduled the arrive right after the last two V
// ldmatrix of the stage (their HMMAs after it), so the producer could refill the stage
// (TMA / cp.async) before those reads happened — V columns 96..127 of a tile then came
// from the next tile, rarely, when a co-resident CTA loaded the shared-memory pipe
// (scripts/determinism.py). The shared store of a word computed from every fragment
// cannot issue before the ldmatrix results are back, and the arrive (release) is ordered
// after the store.
__device__ __forceinline__ void release_stage(uint64_t* empty, uint32_t* scratch, uint32_t dep,
                                              int lane) {
  __syncwarp();
  if (lane == 0) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(scratch)), "r"(dep) : "memory");
    mbar_arrive(empty);
  }
}

// The 1024-B aligned start of the dynamic shared memory, as POINTER ARITHMETIC on the
// __shared__ array: the compiler keeps the shared state space and emits LDS/STS/ATOMS for
// every access through it (incl. the fused select's). Aligning through an integer cast loses
// it: the select's histogram / bitmap atomics then compiled to generic ATOM.E.*.STRONG.GPU,
// and with those, FULL pairs streaming on the same SM came out non-deterministic (a few
// per launch, ~1e-3 off; scripts/determinism.py).
__device__ __forceinline__ uint8_t* align_smem_1024(uint8_t* raw) {
  return raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
}

#ifdef HYLRA_TRACE
// Diagnostics build only (-DHYLRA_TRACE, scripts/trace_single.py): per single-launch CTA,
// globaltimer marks [0 ticket, 1 select start, 2 REUSE ready, 3 select end, 4 done, 5 smid]
static __device__ long long* g_trace;
__shared__ int g_trace_row;
__device__ __forceinline__ long long* hylra_trace_rec() { return g_trace + g_trace_row * 8; }
__device__ __forceinline__ void hylra_trace_mark(int k) {
  if (g_trace == nullptr) return;
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  hylra_trace_rec()[k] = t;
}
#endif


// Block mode, fused (single-launch step, sel_group 1): the final CTA of a FULL pair pools its
// token score row into the block row the select reads (block max, as block_pool_kernel;
// one thread per block, 16-byte loads) ...
__device__ __forceinline__ void fused_block_pool(const SelectParams& sp, int Hkv, int kh, int b,
                                                 int slot) {
  const int tid = threadIdx.x, bs = sp.block_size, n = sp.n_tokens, nb = sp.n_valid;
  const float* trow = sp.tok_scores + ((int64_t)(slot * sp.B + b) * Hkv + kh) * sp.tok_row_stride;
  float* brow = const_cast<float*>(sp.scores) +
                ((int64_t)(slot * sp.B + b) * sp.n_groups + kh) * sp.row_stride;
  for (int blk = tid; blk < nb; blk += kConsumerWarps * 32) {
    const int t0 = blk * bs, t1 = min(n, t0 + bs);
    float m = -INFINITY;
    if (bs % 4 == 0 && t1 - t0 == bs) {
      const float4* r4 = reinterpret_cast<const float4*>(trow + t0);
#pragma unroll 8
      for (int j = 0; j < bs / 4; ++j) {
        const float4 x = __ldcg(r4 + j);
        m = fmaxf(m, fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w)));
      }
    } else {
      for (int t = t0; t < t1; ++t) m = fmaxf(m, __ldcg(trow + t));
    }
    brow[blk] = m;
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");  // the block row is written
}

// ... and after the select writes the selected blocks' token coverage for the REUSE items
// (block_expand_kernel's layout: ascending tokens, -1 past the cache, count per row).
__device__ __forceinline__ void fused_block_expand(const SelectParams& sp, int kh, int b,
                                                   int slot) {
  asm volatile("bar.sync 1, 128;" ::: "memory");  // the selected blocks are written
  const int tid = threadIdx.x, bs = sp.block_size, n = sp.n_tokens, bb = sp.k_eff;
  const int64_t row = (int64_t)(sp.out_slot[slot] * sp.B + b) * sp.n_groups + kh;
  const int32_t* br = sp.idx + row * sp.k_stride;
  int32_t* tr = sp.cov_tokens + row * sp.cov_stride;
  for (int e = tid; e < bb * bs; e += kConsumerWarps * 32) {
    const int tok = br[e / bs] * bs + e % bs;
    tr[e] = tok < n ? tok : -1;
  }
  if (tid == 0) sp.cov_counts[row] = (bb - 1) * bs + min(bs, n - br[bb - 1] * bs);
}

// Token mode with sinks / recent, fused: after the select the final CTA writes the
// augmented row sorted(sel | [0, sinks) | [n - recent, n)) and its length (augment_kernel,
// engine.py:122-126 _augment_selection) for the REUSE items.
__device__ __forceinline__ void fused_augment(const SelectParams& sp, int kh, int b, int slot) {
  asm volatile("bar.sync 1, 128;" ::: "memory");  // the selection is written
  constexpr int NT = kConsumerWarps * 32;
  const int tid = threadIdx.x, n = sp.n_valid, k = sp.k_eff;
  const int64_t row = (int64_t)(sp.out_slot[slot] * sp.B + b) * sp.n_groups + kh;
  const int32_t* src = sp.idx + row * sp.k_stride;
  int32_t* dst = sp.cov_tokens + row * sp.cov_stride;
  const int s = min(sp.sinks, n), u0 = max(n - sp.recent, 0);
  if (u0 <= s) {  // the two ranges already cover every token
    for (int i = tid; i < n; i += NT) dst[i] = i;
    if (tid == 0) sp.cov_counts[row] = n;
    return;
  }
  // selected tokens strictly between the ranges: [lower_bound(s), lower_bound(u0))
  __shared__ int s_lb[2];
  if (tid < 2) {
    const int key = tid == 0 ? s : u0;
    int a = 0, z = k;
    while (a < z) {
      const int m = (a + z) >> 1;
      if (src[m] < key) a = m + 1;
      else z = m;
    }
    s_lb[tid] = a;
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  const int mid0 = s_lb[0], mid = s_lb[1] - s_lb[0];
  for (int i = tid; i < s; i += NT) dst[i] = i;
  for (int i = tid; i < mid; i += NT) dst[s + i] = src[mid0 + i];
  for (int i = tid; i < n - u0; i += NT) dst[s + mid + i] = u0 + i;
  if (tid == 0) sp.cov_counts[row] = s + mid + (n - u0);
}

// One work item of the tensor-core kernels: the rows [split range] of one (layer slot, b,
// kv-head) pair. `smem` is the 1024-B aligned dynamic shared memory. REUSE items with
// `ready_wait` first wait for their selection row's ready flag (single-launch step); FULL
// items with `ready_set` publish each fused selection's ready flag.
template <int D, bool GATHER, bool GBIG, int STAGES>
__device__ __forceinline__ void attn_mma_item(const CUtensorMap& tmk, const CUtensorMap& tmv,
                                              const AttnParams& p, const SelectParams& sp,
                                              uint8_t* smem, int split, int kh, int slot, int b,
                                              const int* ready_wait, int* ready_set,
                                              int* group_ctr = nullptr) {
  using SM = MmaSmem<D>;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * SM::kStageBytes);
  uint64_t* empty_bar = full_bar + STAGES;

  const int layer = p.layers[slot];
  const int kvl = p.kv_layers[slot];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  const int n_tiles = (p.n_rows + kTileRows - 1) / kTileRows;
  const int t_begin = split * p.tiles_per_split;
  const int t_end = min(n_tiles, t_begin + p.tiles_per_split);
  const int n_my = t_end - t_begin;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar + s, (GATHER && !p.gather_tma) ? 32 * kGatherProducers : 1);
      mbar_init(empty_bar + s, kConsumerWarps);
    }
    mbar_fence_init();
  }
  // before any global read: the previous launch may still be writing (early: only the reads
  // of q wait, in the consumer warps below)
  if (!p.early) pdl_wait();
  if (ready_wait != nullptr && threadIdx.x == 0) {
    // single-launch step: this item's selection row (and its coverage count) is written by
    // a FULL item of the same grid. Bounded: a flag that never comes (it cannot, short of a
    // corrupted workspace) turns into HYLRA_FLAG_INTERNAL after ~2 s instead of a hung GPU.
    for (long long spins = 0; ld_acquire_gpu(ready_wait) == 0; ++spins) {
      if (spins > (1ll << 25)) {
        atomicOr(p.flags, 8);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (ready_wait != nullptr) (void)ld_acquire_gpu(ready_wait);  // every thread: acquire
#ifdef HYLRA_TRACE
  if (ready_wait != nullptr && threadIdx.x == 0) hylra_trace_mark(2);
#endif
  // rows of this pair: uniform, or the selection row's own length (block coverage); read
  // coherently (written earlier in the step)
  const int n_rows = ((GATHER || p.blk != nullptr) && p.counts != nullptr)
                         ? min(p.n_rows, __ldcg(p.counts + (int64_t)(p.src_slot[slot] * p.B + b) *
                                                               p.n_groups + kh / p.sel_group))
                         : p.n_rows;

  // FULL pairs whose row is selected count the row's first-level histogram (select.cuh
  // hist_bin) in shared memory: the consumer warps leave each tile's 64 scores in a per-stage
  // buffer, the producer warp (otherwise waiting on the ring) counts them once the stage is
  // released, and adds its counts to the row's global histogram at the end, so the select
  // needs no sampling pass nor a pass to bracket the k-th value.
  uint32_t* hist_smem = nullptr;  // kHistBins 16-bit counters, two per word (the staging area)
  float* score_buf = nullptr;     // [2 STAGES][64] scores of tile t in buffer t % (2 STAGES)
  if (!GATHER && p.scores != nullptr && p.hist != nullptr) {
    hist_smem = reinterpret_cast<uint32_t*>(smem + STAGES * SM::kStageBytes + 256);
    score_buf = reinterpret_cast<float*>(smem + STAGES * SM::kStageBytes + 256 + kIdxStage * 4);
  }

  if (warp >= kConsumerWarps) {
    // ------------------------------------------------------------- producer warp
    if constexpr (!GATHER) {
      if (warp == kConsumerWarps) {
        // the scores of tile t (score buffer t % (2 STAGES)) into the shared-memory histogram
        auto count_tile = [&](int t) {
          const float* sb = score_buf + (t % (2 * STAGES)) * kTileRows;
#pragma unroll
          for (int j = lane; j < kTileRows; j += 32) {
            if ((t_begin + t) * kTileRows + j < n_rows) {
              const int bin = hist_bin(sb[j]);
              atomicAdd(hist_smem + (bin >> 1), 1u << ((bin & 1) << 4));
            }
          }
        };
        if (hist_smem != nullptr)
          for (int j = lane; j < kHistBins / 2; j += 32) hist_smem[j] = 0u;
        if (lane == 0) {
          tma_prefetch_desc(&tmk);
          tma_prefetch_desc(&tmv);
        }
        const uint64_t pol = l2_policy_evict_first();
        // block-mode REUSE: tile t covers rows blk[t / tpb] * blk_size + (t % tpb) * 64; the
        // block ids are loaded kAhead tiles ahead so no TMA issue waits on a global load
        constexpr int kAhead = 4;
        const int tpb = p.blk != nullptr ? p.blk_size / kTileRows : 1;
        const int32_t* bl =
            p.blk == nullptr ? nullptr
                             : p.blk + ((int64_t)(p.src_slot[slot] * p.B + b) * p.n_groups +
                                        kh / p.sel_group) * p.blk_stride;
        int ahead[kAhead];
#pragma unroll
        for (int j = 0; j < kAhead; ++j)
          ahead[j] = (bl != nullptr && j < n_my) ? __ldcg(bl + (t_begin + j) / tpb) : 0;
        for (int i = 0; i < n_my; ++i) {
          const int s = i % STAGES;
          int row = (t_begin + i) * kTileRows;
          if (bl != nullptr) {
            row = ahead[0] * p.blk_size + ((t_begin + i) % tpb) * kTileRows;
#pragma unroll
            for (int j = 0; j + 1 < kAhead; ++j) ahead[j] = ahead[j + 1];
            ahead[kAhead - 1] = (i + kAhead < n_my) ? __ldcg(bl + (t_begin + i + kAhead) / tpb) : 0;
          }
          mbar_wait(empty_bar + s, ((i / STAGES) & 1) ^ 1);
          if (lane == 0) {
            uint8_t* kt = smem + s * SM::kStageBytes;
            uint8_t* vt = kt + SM::kTileBytes;
            mbar_arrive_expect_tx(full_bar + s, SM::kStageBytes);
#pragma unroll
            for (int bx = 0; bx < SM::kBoxes; ++bx) {
              tma_load_5d(kt + bx * kTileRows * 128, &tmk, full_bar + s, bx * 64, row, kh, b,
                          kvl, pol);
              tma_load_5d(vt + bx * kTileRows * 128, &tmv, full_bar + s, bx * 64, row, kh, b,
                          kvl, pol);
            }
          }
          // the stage's previous tile is consumed: count its scores behind the refill (its score
          // buffer is rewritten only by tile i + STAGES, whose load is issued after this count)
          if (hist_smem != nullptr && i >= STAGES) count_tile(i - STAGES);
          __syncwarp();
        }
        if (hist_smem != nullptr) {
          // the last STAGES tiles; the consumer warps then add the counts to the row's
          // histogram (behind the same fence as their split-K partials)
          for (int t = max(0, n_my - STAGES); t < n_my; ++t) {
            mbar_wait(empty_bar + t % STAGES, (t / STAGES) & 1);
            count_tile(t);
          }
          asm volatile("bar.arrive 4, %0;" ::"n"(32 * (kConsumerWarps + 1)) : "memory");
        }
      }
    } else {
      // gather: every lane copies 2 rows (K and V) per stage with 16-byte cp.async
      const __nv_bfloat16* kbase = reinterpret_cast<const __nv_bfloat16*>(p.k) +
                                   kvl * p.kv_sl + b * p.kv_sb + kh * p.kv_sh;
      const __nv_bfloat16* vbase = reinterpret_cast<const __nv_bfloat16*>(p.v) +
                                   kvl * p.kv_sl + b * p.kv_sb + kh * p.kv_sh;
      const int32_t* ib = p.idx + ((int64_t)(p.src_slot[slot] * p.B + b) * p.n_groups +
                                   kh / p.sel_group) * p.k_stride;
      // Lane roles: a row of D bf16 is D/8 16-byte chunks; CH = D/8 consecutive lanes copy
      // one row, so each cp.async instruction touches 32/CH whole rows (few L1 wavefronts).
      constexpr int CH = D / 8;
      constexpr int RPI = 32 / CH;  // rows per instruction
      const int my_ch = lane % CH;
      const int my_sub = lane / CH;
      // The CTA's whole index range is staged (validated) in shared memory once, so neither
      // the copies nor the L2 prefetches wait on a dependent global index load.
      int32_t* sidx = reinterpret_cast<int32_t*>(smem + STAGES * SM::kStageBytes + 256);
      const int pos_begin = t_begin * kTileRows;
      const int n_pos = min(n_rows, t_end * kTileRows) - pos_begin;
      const bool staged = n_pos <= kIdxStage;
      if (staged) {
        stage_indices(ib + pos_begin, n_pos, p.n_valid, sidx, p.flags, lane,
                      warp - kConsumerWarps, kGatherProducers);
        if (kGatherProducers > 1)
          asm volatile("bar.sync 3, %0;" ::"n"(32 * kGatherProducers) : "memory");
        else
          __syncwarp();
      }
      if (p.gather_tma && staged) {
        // TMA gather: one lane issues 4-row gathers per stage (K and V, each 128-byte
        // column box); the staged indices become rows of the 2-D views
        // the producer warps' lane 0s share each stage's rows (the first one also arms
        // the stage's transaction count: a gather completing before it is armed only
        // drives the count negative within the phase, which cannot complete before the
        // arrival)
        const int part = warp - kConsumerWarps;
        constexpr int kRowsPer = kTileRows / kGatherProducers;
        if (lane == 0) {
          const uint64_t pol = l2_policy_evict_first();
          const int base_row = ((kvl * p.B + b) * p.Hkv + kh) * p.cap_rows;
          for (int i = 0; i < n_my; ++i) {
            const int s = i % STAGES;
            mbar_wait(empty_bar + s, ((i / STAGES) & 1) ^ 1);
            uint8_t* kt = smem + s * SM::kStageBytes;
            uint8_t* vt = kt + SM::kTileBytes;
            if (part == 0) mbar_arrive_expect_tx(full_bar + s, SM::kStageBytes);
            const int pos0 = (t_begin + i) * kTileRows;
#pragma unroll 4
            for (int r = part * kRowsPer; r < (part + 1) * kRowsPer; r += 4) {
              int rw[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int pos = pos0 + r + u;
                rw[u] = pos < n_rows ? base_row + sidx[pos - pos_begin] : p.gather_rows;
              }
#pragma unroll
              for (int bx = 0; bx < SM::kBoxes; ++bx) {
                tma_gather4(kt + bx * kTileRows * 128 + r * 128, &tmk, full_bar + s, bx * 64,
                            rw[0], rw[1], rw[2], rw[3], pol);
                tma_gather4(vt + bx * kTileRows * 128 + r * 128, &tmv, full_bar + s, bx * 64,
                            rw[0], rw[1], rw[2], rw[3], pol);
              }
            }
          }
        }
        return;
      }
      auto row_at = [&](int pos) -> int {  // pos < n_rows
        if (staged) return sidx[pos - pos_begin];
        int row = __ldcg(ib + pos);
        if (row < 0 || row >= p.n_valid) {
          atomicOr(p.flags, 1);
          row = 0;
        }
        return row;
      };
      auto load_idx = [&](int tile, int rr) -> int {
        const int pos = tile * kTileRows + lane + 32 * rr;
        return (pos < n_rows) ? row_at(pos) : 0;
      };
      // L2 prefetch of the rows kPrefetch tiles ahead of the shared-memory pipeline: the
      // scattered 2*D-byte rows have a long loaded latency and shared memory bounds the
      // bytes in flight, so line prefetches (LSU path; one per 128-byte line) keep HBM
      // busy beyond the smem ring
      const int kPrefetch = p.prefetch;
      auto prefetch_tile = [&](int tile) {
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int pos = tile * kTileRows + lane + 32 * rr;
          if (pos < n_rows) {
            const int row = row_at(pos);
#pragma unroll
            for (int off = 0; off < D * 2; off += 128) {
              asm volatile("prefetch.global.L2 [%0];" ::"l"(
                  reinterpret_cast<const char*>(kbase + (int64_t)row * D) + off));
              asm volatile("prefetch.global.L2 [%0];" ::"l"(
                  reinterpret_cast<const char*>(vbase + (int64_t)row * D) + off));
            }
          }
        }
      };
      for (int t = 0; t < min(kPrefetch, n_my); ++t) prefetch_tile(t_begin + t);
      int nx0 = 0, nx1 = 0;
      if (n_my > 0) {
        nx0 = load_idx(t_begin, 0);
        nx1 = load_idx(t_begin, 1);
      }
      for (int i = 0; i < n_my; ++i) {
        const int s = i % STAGES;
        const int cur0 = nx0, cur1 = nx1;
        if (kPrefetch > 0 && i + kPrefetch < n_my) prefetch_tile(t_begin + i + kPrefetch);
        if (i + 1 < n_my) {
          nx0 = load_idx(t_begin + i + 1, 0);
          nx1 = load_idx(t_begin + i + 1, 1);
        }
        mbar_wait(empty_bar + s, ((i / STAGES) & 1) ^ 1);
        const uint32_t kt = smem_u32(smem + s * SM::kStageBytes);
        const uint32_t vt = kt + SM::kTileBytes;
        const int pos0 = (t_begin + i) * kTileRows;
        // producer warp pw copies rows [pw, pw + 1) * kTileRows / kGatherProducers
        constexpr int ITP = kTileRows / RPI / kGatherProducers;
        const int it0 = (warp - kConsumerWarps) * ITP;
#pragma unroll
        for (int iu = 0; iu < ITP; ++iu) {
          const int it = it0 + iu;
          const int r = it * RPI + my_sub;  // row of the tile this lane copies now
          // it*RPI < 32 is warp-uniform (RPI divides 32), so every lane offers the same half
          const int src = __shfl_sync(0xffffffffu, (it * RPI < 32) ? cur0 : cur1, r & 31);
          const bool valid = pos0 + r < n_rows;
          const uint32_t off = swz_addr(0, r, my_ch);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(kt + off),
                       "l"(kbase + (int64_t)src * D + my_ch * 8), "r"(valid ? 16 : 0)
                       : "memory");
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(vt + off),
                       "l"(vbase + (int64_t)src * D + my_ch * 8), "r"(valid ? 16 : 0)
                       : "memory");
        }
        cp_async_mbar_arrive_noinc(full_bar + s);
      }
    }
    return;
  }

  // --------------------------------------------------------------- consumer warps
  if (p.early) pdl_wait();  // q may be the previous launch's output
  const int g = lane >> 2;  // row of the m16n8 fragments (query head within the group)
  const int t = lane & 3;
  const int G = p.G;

  // Q A-fragments for all D/16 k-steps.
  uint32_t qa[D / 16][4];
  {
    const __nv_bfloat16* qb = reinterpret_cast<const __nv_bfloat16*>(p.q) + layer * p.q_sl +
                              b * p.q_sb + (int64_t)(kh * G) * D;
    const bool r0ok = g < G;
    const bool r1ok = GBIG && (g + 8) < G;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
      const int c0 = ks * 16 + 2 * t;
      qa[ks][0] = r0ok ? *reinterpret_cast<const uint32_t*>(qb + g * D + c0) : 0u;
      qa[ks][2] = r0ok ? *reinterpret_cast<const uint32_t*>(qb + g * D + c0 + 8) : 0u;
      qa[ks][1] = r1ok ? *reinterpret_cast<const uint32_t*>(qb + (g + 8) * D + c0) : 0u;
      qa[ks][3] = r1ok ? *reinterpret_cast<const uint32_t*>(qb + (g + 8) * D + c0 + 8) : 0u;
    }
  }

  float o[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  float* score_row = nullptr;
  if (!GATHER && p.scores != nullptr)
    score_row = p.scores + ((int64_t)(slot * p.B + b) * p.Hkv + kh) * p.cap;

  const int rbase = warp * 16;
  // one word per consumer warp between the barriers and the REUSE index staging area
  uint32_t* release_word = reinterpret_cast<uint32_t*>(smem + STAGES * SM::kStageBytes + 128);

  for (int i = 0; i < n_my; ++i) {
    const int s = i % STAGES;
    mbar_wait(full_bar + s, (i / STAGES) & 1);
    const uint32_t kt = smem_u32(smem + s * SM::kStageBytes);
    const uint32_t vt = kt + SM::kTileBytes;
    const int row0 = (t_begin + i) * kTileRows + rbase;  // first row of this warp's slice

    const uint32_t dep = mma_consume_tile<D, GATHER, GBIG>(
        p, kt, vt, qa, o, m0, m1, l0, l1, row0, n_rows, score_row,
        score_buf != nullptr ? score_buf + (i % (2 * STAGES)) * kTileRows : nullptr, lane);
    release_stage(empty_bar + s, release_word + warp, dep, lane);
#ifdef HYLRA_TRACE
    if (i == 0 && threadIdx.x == 0) hylra_trace_mark(6);
#endif
  }
#ifdef HYLRA_TRACE
  if (threadIdx.x == 0) hylra_trace_mark(7);
#endif
  pdl_launch_dependents();
  if (hist_smem != nullptr) {
    // the producer warp has counted every tile: this split's counts join the row's
    // histogram (L2 reductions, nonzero bins only), made visible by the fence of the
    // cooperative arrival or of the split-K merge below (or the kernel's end)
    asm volatile("bar.sync 4, %0;" ::"n"(32 * (kConsumerWarps + 1)) : "memory");
    unsigned* hist_row = p.hist + ((int64_t)(slot * p.B + b) * p.Hkv + kh) * kHistBins;
    for (int j = threadIdx.x; j < kHistBins / 2; j += 128) {
      const uint32_t w = hist_smem[j];
      if (w & 0xffffu) atomicAdd(hist_row + 2 * j, w & 0xffffu);
      if (w >> 16) atomicAdd(hist_row + 2 * j + 1, w >> 16);
    }
  }

  // ---- cooperative select (single-launch step, select.cuh coop_*): arrive as soon as this
  //      split's scores and histogram reductions are out; the last split to arrive publishes
  //      the row's candidate range; the split's slice of scores is prefetched into the drained
  //      pipeline buffers (past the merge's region) while the merge below runs
  __shared__ Red sel_red;
  __shared__ int s_coop;
  const bool coop = !GATHER && sp.coop != nullptr && slot < p.fuse_select;
  const int srow = (slot * p.B + b) * p.Hkv + kh;  // score / histogram / coop row
  CoopRow* rec = coop ? sp.coop + srow : nullptr;
  constexpr int kSliceOff = ((2 * kConsumerWarps * 16 + kConsumerWarps * 16 * D) * 4 + 1023) & ~1023;
  constexpr int kSliceCap = STAGES * SM::kStageBytes - kSliceOff;
  const int s0 = t_begin * kTileRows, s1 = min(n_rows, t_end * kTileRows);
  const bool slice_smem = coop && (s1 - s0) * 4 <= kSliceCap;
  if (coop) {
    __threadfence();  // this split's scores and histogram reductions, before its arrival
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 0) s_coop = atomicAdd(&rec->arrive1, 1) == p.splits - 1;
    if (slice_smem) {
      const int n16 = ((s1 - s0) + 3) >> 2;  // 16-byte chunks (rows are padded to 8 scores)
      for (int i = threadIdx.x; i < n16; i += 128)
        cp_async_16(smem + kSliceOff + 16 * i, score_row + s0 + 4 * i, true);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (s_coop) {
      __threadfence();
      coop_publish<kConsumerWarps * 32>(sp, srow, rec, n_rows, sel_red);
    }
  }

  // ---- merge the 4 warps through shared memory (pipeline buffers are drained)
  asm volatile("bar.sync 1, 128;" ::: "memory");
  float* sm_m = reinterpret_cast<float*>(smem);
  float* sm_l = sm_m + kConsumerWarps * 16;
  float* sm_o = sm_l + kConsumerWarps * 16;
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  if (GBIG) {
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  }
  if (t == 0) {
    sm_m[warp * 16 + g] = m0;
    sm_l[warp * 16 + g] = l0;
    sm_m[warp * 16 + g + 8] = GBIG ? m1 : -INFINITY;
    sm_l[warp * 16 + g + 8] = GBIG ? l1 : 0.f;
  }
#pragma unroll
  for (int j = 0; j < D / 8; ++j) {
    *reinterpret_cast<float2*>(sm_o + (warp * 16 + g) * D + 8 * j + 2 * t) =
        make_float2(o[j][0], o[j][1]);
    if (GBIG)
      *reinterpret_cast<float2*>(sm_o + (warp * 16 + g + 8) * D + 8 * j + 2 * t) =
          make_float2(o[j][2], o[j][3]);
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  // the merge's scratch: the REUSE index staging area / FULL histogram + score buffers, idle
  // once the main loop is done; its bulk staging area: the drained pipeline buffers (not
  // while the cooperative select's slice prefetch is landing in them)
  if (GATHER && p.cluster_merge > 1) {
    constexpr int kPartOff = ((2 * kConsumerWarps * 16 + kConsumerWarps * 16 * D) * 4 + 127) & ~127;
    cluster_merge_store<D>(p, slot, b, kh, split, sm_m, sm_l, sm_o,
                           reinterpret_cast<float*>(smem + kPartOff),
                           reinterpret_cast<float*>(smem + STAGES * SM::kStageBytes + 256));
    return;
  }
  const bool final_cta = merge_and_store<D>(
      p, slot, b, kh, split, sm_m, sm_l, sm_o, threadIdx.x, 128, 1,
      reinterpret_cast<float*>(smem + STAGES * SM::kStageBytes + 256),
      kIdxStage + 2 * STAGES * kTileRows, p.bulk_merge ? smem : nullptr,
      slice_smem ? 0u : (uint32_t)(STAGES * SM::kStageBytes));
  if constexpr (!GATHER) {
    if (coop) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");  // the slice is in, the merge is done
      const bool last = coop_classify<kConsumerWarps * 32>(
          sp, srow, rec, score_row,
          slice_smem ? reinterpret_cast<const float*>(smem + kSliceOff) : nullptr, s0, s1,
          n_rows, p.splits, sel_red);
      if (last) {
#ifdef HYLRA_TRACE
        if (threadIdx.x == 0) hylra_trace_mark(1);
#endif
        asm volatile("bar.sync 1, 128;" ::: "memory");
        coop_final<kConsumerWarps * 32>(sp, kh, b, slot, srow, rec, smem, (size_t)STAGES * SM::kStageBytes,
                                        sel_red);
        if (sp.cov_tokens != nullptr) fused_augment(sp, kh, b, slot);
#ifdef HYLRA_TRACE
        if (threadIdx.x == 0) hylra_trace_mark(3);
#endif
        if (ready_set != nullptr) {
          asm volatile("bar.sync 1, 128;" ::: "memory");  // the row's indices are written
          if (threadIdx.x == 0) {
            __threadfence();
            st_release_gpu(ready_set + (sp.out_slot[slot] * p.B + b) * p.n_groups + kh, 1);
          }
        }
      }
      return;
    }
    // fused selection: the pair's score row is complete (every split wrote its part before
    // the counter), so its top-k is taken right here while other CTAs keep streaming;
    // the drained pipeline buffers hold the select's shared memory
    if (final_cta && slot < p.fuse_select) {
      __shared__ int s_group_last;
      asm volatile("bar.sync 1, 128;" ::: "memory");  // merge reads of smem are done
      __threadfence();
      const int grp = kh / p.sel_group;
      bool run = true;
      if (p.sel_group > 1) {
        // the selection row sums the scores of sel_group KV heads (single-launch step): the
        // last of those pairs to finish selects; its counter resets itself
        if (threadIdx.x == 0) {
          const int row = (sp.out_slot[slot] * p.B + b) * p.n_groups + grp;
          s_group_last = atomicAdd(group_ctr + row, 1) == p.sel_group - 1;
          if (s_group_last) group_ctr[row] = 0;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        run = s_group_last != 0;
        if (run) __threadfence();
      }
      if (run) {
#ifdef HYLRA_TRACE
        if (threadIdx.x == 0) hylra_trace_mark(1);
#endif
        if (sp.block_size > 1) fused_block_pool(sp, p.Hkv, kh, b, slot);
        select_row<kConsumerWarps * 32, true>(sp, grp, b, slot, smem, sel_red, false,
                                              (size_t)STAGES * SM::kStageBytes);
        if (sp.block_size > 1) fused_block_expand(sp, kh, b, slot);
        else if (sp.cov_tokens != nullptr) fused_augment(sp, grp, b, slot);
#ifdef HYLRA_TRACE
        if (threadIdx.x == 0) hylra_trace_mark(3);
#endif
        if (ready_set != nullptr) {
          asm volatile("bar.sync 1, 128;" ::: "memory");  // the row's indices are written
          if (threadIdx.x == 0) {
            __threadfence();
            st_release_gpu(ready_set + (sp.out_slot[slot] * p.B + b) * p.n_groups + grp, 1);
          }
        }
      }
    }
  }
}

template <int D, bool GATHER, bool GBIG, int STAGES>
__global__ void __launch_bounds__(attn_threads<GATHER>(), 2)
    attn_mma_kernel(const __grid_constant__ CUtensorMap tmk,
                    const __grid_constant__ CUtensorMap tmv, const AttnParams p,
                    const __grid_constant__ SelectParams sp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
#ifdef HYLRA_TRACE
  // one trace row per CTA: [0 start, 4 done, 5 smid, 6 first stage consumed, 7 main loop end]
  if (threadIdx.x == 0) {
    g_trace_row = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    hylra_trace_mark(0);
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (g_trace != nullptr) hylra_trace_rec()[5] = smid;
  }
#endif
  attn_mma_item<D, GATHER, GBIG, STAGES>(tmk, tmv, p, sp, smem, blockIdx.x, blockIdx.y,
                                         blockIdx.z / p.B, blockIdx.z % p.B, nullptr, nullptr);
  if (GATHER && p.cluster_merge > 1 && (threadIdx.x >> 5) >= kConsumerWarps) {
    cluster_sync_all();  // the consumer warps' cluster_merge_store barriers (1) and (2)
    cluster_sync_all();
  }
#ifdef HYLRA_TRACE
  if (threadIdx.x == 0) hylra_trace_mark(4);
#endif
}

// ---------------------------------------------------------------------------------
// Single-launch step: every FULL item (pairs of the layers some REUSE layer inherits from
// first, selections fused), then every REUSE item, in ONE grid. Items are claimed in
// ticket order (atomic counter) rather than by blockIdx, so a REUSE item waiting on its
// selection's ready flag only ever waits on FULL items already claimed by resident CTAs:
// no deadlock whatever the CTA dispatch order. The FULL tail (last splits, fused selects)
// overlaps the REUSE gathers instead of ending a launch. The last CTA to finish resets the
// ticket, the done counter and the ready flags (the workspace stays zeroed between steps).
// The step's new K/V rows (hylra_step_options append_*), written by the FULL items
// themselves: the split whose tile range holds row `pos` writes its own pair's FULL-layer
// row before its TMA loads (generic writes, then a proxy fence, then the TMA), and the
// splits of every FULL pair share out the rows of the REUSE layers that inherit its
// selection (visible to those REUSE items through the same ready flag they wait on).
struct StepAppend {
  const uint4* k_rows;  // [L][B][Hkv][d] in 16-byte chunks (device or pinned host), or null
  const uint4* v_rows;
  uint8_t* k;           // cache bases (bytes)
  uint8_t* v;
  int* flags;           // a non-finite new row sets HYLRA_FLAG_NON_FINITE_CACHE
  int64_t kv_sl, kv_sb, kv_sh, pos_bytes;  // bytes
  int pos, chunks;                          // chunks = 16-byte chunks per row
};

struct StepSync {
  int* ctr;     // [0] ticket, [1] done
  int* ready;   // [n_full][B][n_groups]
  int* group;   // [n_full][B][n_groups] pairs of a selection group done (sel_group > 1)
  int n_ready;
  int n_full_items, n_items;
  StepAppend app;
};

// One (layer, b, kv-head) row pair of the step's new K/V rows into the cache: threads
// [0, 2 chunks) copy one 16-byte chunk each (K then V).
__device__ __forceinline__ void append_row(const StepAppend& a, int B, int Hkv, int row_layer,
                                           int cache_layer, int b, int kh) {
  const int t = threadIdx.x;
  if (t >= 2 * a.chunks) return;
  const bool is_v = t >= a.chunks;
  const int c = is_v ? t - a.chunks : t;
  const int64_t src = (((int64_t)row_layer * B + b) * Hkv + kh) * a.chunks + c;
  const uint4 val = is_v ? a.v_rows[src] : a.k_rows[src];
  uint8_t* dst = (is_v ? a.v : a.k) + cache_layer * a.kv_sl + b * a.kv_sb + kh * a.kv_sh +
                 a.pos_bytes;
  reinterpret_cast<uint4*>(dst)[c] = val;
  // bf16 (the tensor-core path): any all-ones exponent among the 8 values
  const uint32_t w[4] = {val.x, val.y, val.z, val.w};
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    bad |= ((w[i] & 0x7f80u) == 0x7f80u) || ((w[i] & 0x7f800000u) == 0x7f800000u);
  if (bad) atomicOr(a.flags, 16);
}

template <int D, bool GBIG, int STAGES>
__global__ void __launch_bounds__(attn_threads<true>(), 2)
    step_mma_kernel(const __grid_constant__ CUtensorMap tmk,
                    const __grid_constant__ CUtensorMap tmv, const AttnParams pf,
                    const AttnParams pr, const __grid_constant__ SelectParams sp,
                    const StepSync ss) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ int s_ticket;
  pdl_wait();
  if (threadIdx.x == 0) s_ticket = atomicAdd(ss.ctr, 1);
  __syncthreads();
  // modulo: even a counter left non-zero (a workspace that was not zeroed) hands out every
  // item exactly once, so no REUSE item can wait on a FULL item that never runs
  int t = s_ticket % ss.n_items;
#ifdef HYLRA_TRACE
  if (threadIdx.x == 0) {
    g_trace_row = t;
    hylra_trace_mark(0);
    unsigned sm;
    asm("mov.u32 %0, %%smid;" : "=r"(sm));
    if (g_trace != nullptr) hylra_trace_rec()[5] = sm;
  }
#endif
  if (t < ss.n_full_items) {
    const int split = t % pf.splits;
    t /= pf.splits;
    const int kh = t % pf.Hkv;
    t /= pf.Hkv;
    const int slot = t / pf.B, b = t % pf.B;
    if (ss.app.k_rows != nullptr) {
      if (split == (ss.app.pos / kTileRows) / pf.tiles_per_split)
        append_row(ss.app, pf.B, pf.Hkv, pf.layers[slot], pf.kv_layers[slot], b, kh);
      int j = 0;
      for (int r = 0; r < pr.n_slots; ++r) {
        if (pr.src_slot[r] != sp.out_slot[slot]) continue;
        if (j % pf.splits == split)
          append_row(ss.app, pf.B, pf.Hkv, pr.layers[r], pr.kv_layers[r], b, kh);
        ++j;
      }
      // the writes are read by this CTA's TMA (async proxy) and by other CTAs' cp.async
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    attn_mma_item<D, false, GBIG, STAGES>(tmk, tmv, pf, sp, smem, split, kh, slot, b, nullptr,
                                          ss.ready, ss.group);
  } else {
    t -= ss.n_full_items;
    const int split = t % pr.splits;
    t /= pr.splits;
    const int kh = t % pr.Hkv;
    t /= pr.Hkv;
    const int slot = t / pr.B, b = t % pr.B;
    const int* rw = ss.ready + (pr.src_slot[slot] * pr.B + b) * pr.n_groups + kh / pr.sel_group;
    attn_mma_item<D, true, GBIG, STAGES>(tmk, tmv, pr, sp, smem, split, kh, slot, b, rw, nullptr);
  }
  // every warp is done with the item (barrier 2: barrier 0 belongs to the fused select's 128
  // threads while the producer warps wait here)
  asm volatile("bar.sync 2, %0;" ::"n"(32 * (kConsumerWarps + kGatherProducers)) : "memory");
#ifdef HYLRA_TRACE
  if (threadIdx.x == 0) hylra_trace_mark(4);
#endif
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ss.ctr + 1, 1) == ss.n_items - 1) {
      for (int i = 0; i < ss.n_ready; ++i) ss.ready[i] = 0;
      ss.ctr[0] = 0;
      ss.ctr[1] = 0;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------------
// CUDA-core path: fp32 caches (the reference-precision path, tolerance 1e-3) and any
// shape the tensor-core path does not cover (d = 32, bf16 with G > 16 is rejected).
// Each warp walks rows r = split_begin + warp, +4, ...; lane holds d-slice
// lane + 32 j, dot products are warp-reduced, softmax state is per head.
template <typename T, int D, int GMAX, bool GATHER>
__global__ void __launch_bounds__(128)
    attn_simt_kernel(const AttnParams p) {
  constexpr int J = D / 32;
  __shared__ float sm_m[kConsumerWarps * 16];
  __shared__ float sm_l[kConsumerWarps * 16];
  __shared__ float sm_o[kConsumerWarps * 16 * D];

  const int split = blockIdx.x;
  const int kh = blockIdx.y;
  const int slot = blockIdx.z / p.B;
  const int b = blockIdx.z % p.B;
  const int layer = p.layers[slot];
  const int kvl = p.kv_layers[slot];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int G = p.G;
  const float c = p.scale_log2;

  const int n_rows = (GATHER && p.counts != nullptr)
                         ? min(p.n_rows, __ldg(p.counts + (int64_t)(p.src_slot[slot] * p.B + b) *
                                                              p.n_groups + kh / p.sel_group))
                         : p.n_rows;
  const int r_begin = split * p.tiles_per_split * kTileRows;
  const int r_end = min(n_rows, r_begin + p.tiles_per_split * kTileRows);

  const T* qb = reinterpret_cast<const T*>(p.q) + layer * p.q_sl + b * p.q_sb +
                (int64_t)(kh * G) * D;
  const T* kb = reinterpret_cast<const T*>(p.k) + kvl * p.kv_sl + b * p.kv_sb + kh * p.kv_sh;
  const T* vb = reinterpret_cast<const T*>(p.v) + kvl * p.kv_sl + b * p.kv_sb + kh * p.kv_sh;
  const int32_t* ib = nullptr;
  if (GATHER)
    ib = p.idx + ((int64_t)(p.src_slot[slot] * p.B + b) * p.n_groups + kh / p.sel_group) *
                     p.k_stride;
  float* score_row = nullptr;
  if (!GATHER && p.scores != nullptr)
    score_row = p.scores + ((int64_t)(slot * p.B + b) * p.Hkv + kh) * p.cap;

  float qv[GMAX][J];
#pragma unroll
  for (int g = 0; g < GMAX; ++g)
#pragma unroll
    for (int j = 0; j < J; ++j) qv[g][j] = (g < G) ? to_f32(qb[g * D + lane + 32 * j]) : 0.f;

  float m[GMAX], l[GMAX], acc[GMAX][J];
#pragma unroll
  for (int g = 0; g < GMAX; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int j = 0; j < J; ++j) acc[g][j] = 0.f;
  }

  for (int r = r_begin + warp; r < r_end; r += kConsumerWarps) {
    int row = r;
    if (GATHER) {
      row = __ldg(ib + r);
      if (row < 0 || row >= p.n_valid) {
        if (lane == 0) atomicOr(p.flags, 1);
        continue;
      }
    }
    float kv[J], vv[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      kv[j] = to_f32(kb[(int64_t)row * D + lane + 32 * j]);
      vv[j] = to_f32(vb[(int64_t)row * D + lane + 32 * j]);
    }
    float dot[GMAX];
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < J; ++j) s = fmaf(qv[g][j], kv[j], s);
      dot[g] = (g < G) ? warp_sum(s) : 0.f;
    }
    if (score_row != nullptr && lane == 0) {
      float agg = 0.f;
#pragma unroll
      for (int g = 0; g < GMAX; ++g) agg += dot[g] * p.inv_sqrt_d;
      score_row[r] = agg;
    }
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      if (g < G) {
        const float mn = fmaxf(m[g], dot[g]);
        const float alpha = exp2f((m[g] - mn) * c);
        const float pr = exp2f((dot[g] - mn) * c);
        l[g] = fmaf(l[g], alpha, pr);
        m[g] = mn;
#pragma unroll
        for (int j = 0; j < J; ++j) acc[g][j] = fmaf(acc[g][j], alpha, pr * vv[j]);
      }
    }
  }

#pragma unroll
  for (int g = 0; g < GMAX; ++g) {
    if (g < G) {
      if (lane == 0) {
        sm_m[warp * 16 + g] = m[g];
        sm_l[warp * 16 + g] = l[g];
      }
#pragma unroll
      for (int j = 0; j < J; ++j) sm_o[(warp * 16 + g) * D + lane + 32 * j] = acc[g][j];
    }
  }
  __syncthreads();
  merge_and_store<D>(p, slot, b, kh, split, sm_m, sm_l, sm_o, threadIdx.x, 128, 1);
}

}  // namespace hylra
