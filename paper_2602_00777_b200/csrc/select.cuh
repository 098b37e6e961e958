// select.cuh — exact top-k selection over per-(slot, b, group) score rows.
//
// Reference: pkg/src/layerreuse/attention.py:264-275 topk_of_logits — the min(budget, N)
// highest logits, ties won by the LOWER index (stable argsort of -logits), returned
// ascending; engine.py:169 clamps the budget per step; engine.py:177-183 scores are the
// head-order sum of per-head scaled logits.
//
// One CTA per row (256 threads and ~29 KB of shared memory when rows are many: 4 CTAs per
// SM, all rows of a step resident at once; 512 / 1024 threads when rows are few); no
// global atomics. Fast path:
//   A. bracket the k-th rank with [lo, hi] from the quantiles of 1024 strided samples;
//   B. one vectorised pass: "definitely selected" bits (s > hi) go straight into a shared
//      bitmap, scores inside [lo, hi] into a 2048-bin linear histogram; max|s| and the
//      non-finite check ride along;
//   C. the bin holding rank k (from the top) is found with one block scan;
//   D. a second (L2-resident) pass sets the bits of the higher bins and collects the few
//      scores of the bins around it; the exact k-th value T comes from those. The boundary
//      window — the ties at T, or with refinement every score within tau of T, re-scored in
//      float64 from the original q / K rows with heads summed in reference order — is
//      ranked by (score desc, index asc) and its top members join the bitmap;
//   E. index-ordered compaction of the bitmap (one block scan per 8K-token chunk) writes
//      the indices ascending: the reference's canonical TopKSet order.
// Degenerate rows (massive ties, failed brackets, oversized windows) take a generic path:
// full-row MSB radix select, then the same window logic, or an index-ordered tie pass.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace hylra {

// Threads per CTA (one CTA per row) is a template parameter NT in {256, 512, 1024}: rows
// are few at small batch (64 at cfg2 B=1), so a wider CTA shortens each row's passes;
// with many rows 256-thread CTAs keep every row resident at once (4 per SM).
constexpr int kSelMaxThreads = 1024;
constexpr int kSelMaxWarps = kSelMaxThreads / 32;
constexpr int kBins = 2048;
constexpr int kCandCap = 1024;            // scores collected around the k-th bin
constexpr int kSmallN = 2048;             // rows sorted outright (small-row path)
constexpr int kSelMaxTokens = 262144;     // longest row (bitmap = 32 KB)

// First-level histogram of a score row, built by the FULL kernel as it emits the scores
// (every split adds its tokens with L2 reductions): bin = the top 12 bits of the
// order-preserving key, so a bin spans 1/8 of a binary octave. The select reads it (and
// zeroes it for the next step) to find the bin holding the k-th value without touching the
// row, then makes ONE pass over the row. kHistCandCap bounds the tokens of that bin (plus
// the refinement margin) the pass may collect; past it the row takes the sampled path.
constexpr int kHistShift = 20;
constexpr int kHistBins = 1 << (32 - kHistShift);  // 4096
constexpr int kHistCandCap = 4096;
__device__ __forceinline__ int hist_bin(float v) { return (int)(float_key(v) >> kHistShift); }
template <int NT>
__host__ __device__ constexpr int sel_chunk() { return NT * 32; }  // tokens per bitmap chunk (one word per thread)

// Per-row state of the cooperative select (below): zero at rest, re-zeroed by the row's final
// CTA.
struct CoopRow {
  int arrive1, arrive2, flag, b1;
  float c_lo, c_hi;
  int n_cand, c_above;
  unsigned vmax_key, vmin_nkey;  // atomicMax of float_key(max) and of ~float_key(min)
  int bad, pad[5];
};
static_assert(sizeof(CoopRow) == 64, "CoopRow is 64 bytes");

struct SelectParams {
  const float* scores;  // [slot][b][kh][row_stride]
  int32_t* idx;         // [slot][b][grp][k_stride]
  int32_t* idx_mirror;  // optional second copy of idx (same layout), e.g. pinned host memory
                        // the caller reads after the step: stored alongside idx, no copy
  unsigned* hist;       // optional [slot][b][kh][kHistBins] row histograms written by the FULL
                        // kernel (token rows, sel_group 1): read and re-zeroed by the select
  uint32_t smem_bytes;  // dynamic shared memory of the standalone select kernel
  // cooperative select (single-launch step, token rows, sel_group 1; null: off): per score
  // row its record, candidate list [kHistCandCap] and bitmap [coop_words]
  CoopRow* coop;
  float* coop_cv;
  int* coop_ci;
  uint32_t* coop_bits;
  int coop_words;
  int32_t* info;        // [row][8] or null
  int* flags;
  const void* q;        // refinement inputs (null: refinement off)
  const void* k;
  int dtype;
  int64_t q_sl, q_sb, kv_sl, kv_sb, kv_sh;
  int B, Hkv, G, D, sel_group, n_groups;
  int n_valid, k_eff, k_stride, row_stride;
  float tau_rel;
  int pre_grouped;  // score rows already summed per group ([slot][b][grp][row_stride])
  int block_size;   // 1: token selection; >1: rows are block scores over n_tokens tokens
  int n_tokens;
  const float* tok_scores;  // block mode: token scores [slot][b][kh][tok_row_stride] or null
  int tok_row_stride;
  int layers[kMaxSlots];     // q layer of each slot
  int kv_layers[kMaxSlots];  // K layer of each slot (refinement)
  int out_slot[kMaxSlots];   // idx / info slot each score slot's selection is written to
  // block mode fused into the FULL kernel (single-launch step): the final CTA of a pair pools
  // its token scores into the block row (`scores`), selects, then writes the token coverage
  // [row][cov_stride] and its length cov_counts[row] for the REUSE items
  // Token mode with sinks / recent (cov_tokens set, block_size 1): the augmented selection
  // sorted(sel | [0, sinks) | [n - recent, n)) and its length, as augment_kernel
  int32_t* cov_tokens;
  int32_t* cov_counts;
  int cov_stride;
  int sinks, recent;
};

// Dynamic shared memory: the bitmap sized for the row, then fixed arrays.
__host__ __device__ constexpr size_t sel_bitmap_bytes(int n, int nt) {
  return (size_t)((n + nt * 32 - 1) / (nt * 32)) * (nt * 32) / 8;
}
// Band list: indices of the scores inside the bracket [lo, hi], collected by pass B so the
// second pass reads only them (4096 entries per 256 threads; it shares the small-row keys
// region, which the large-row path does not otherwise use before the window step).
// `big`: the fused select of the FULL kernel, whose shared memory (the drained pipeline
// ring) has room for 8192 band entries.
__host__ __device__ constexpr int sel_band_cap(int nt, bool big = false) {
  return big ? 8192 : (16 * nt > 4096 ? 16 * nt : 4096);
}
__host__ __device__ constexpr size_t sel_keys_bytes(int nt, bool big = false) {
  return (size_t)(kSmallN * 8 > sel_band_cap(nt, big) * 4 ? kSmallN * 8
                                                           : sel_band_cap(nt, big) * 4);
}
__host__ __device__ constexpr size_t sel_fixed_bytes(int nt, bool big = false) {
  return kBins * 4 + kCandCap * (8 + 4) + nt * 4 + sel_keys_bytes(nt, big);
}
__host__ __device__ constexpr size_t sel_smem_bytes(int n, int nt, bool big = false) {
  return sel_bitmap_bytes(n, nt) + sel_fixed_bytes(nt, big);
}
// The histogram path: bitmap, candidates (value + index), then a scratch area for the exact
// T's digit histogram and the float64 window arrays.
__host__ __device__ constexpr size_t sel_hist_smem_bytes(int n, int nt) {
  return sel_bitmap_bytes(n, nt) + (size_t)kHistCandCap * 8 + (size_t)kHistBins * 4;
}

#ifdef HYLRA_TRACE
// diagnostics build only: per-row phase cycles of selections that have no info buffer
// (the fused ones), [row][8] as SelectParams::info
static __device__ int32_t* g_sel_info;
#endif

struct SelSmem {
  uint32_t* bitmap;  // [chunks * NT]
  unsigned* hist;    // [kBins]
  double* cv;        // [kCandCap] window scores (fp32 value, then float64 re-score)
  int* ci;           // [kCandCap] window token indices
  float* xchg;       // [NT]
  uint64_t* keys;    // [kSmallN] small-row sort keys
  int* band;         // [sel_band_cap(NT, big)] pass-B band list (aliases keys)
};

template <int NT>
__device__ __forceinline__ SelSmem carve(uint8_t* base, int n) {
  SelSmem m;
  const size_t bb = sel_bitmap_bytes(n, NT);
  m.bitmap = reinterpret_cast<uint32_t*>(base);
  m.hist = reinterpret_cast<unsigned*>(base + bb);
  m.cv = reinterpret_cast<double*>(base + bb + kBins * 4);
  m.ci = reinterpret_cast<int*>(base + bb + kBins * 4 + kCandCap * 8);
  m.xchg = reinterpret_cast<float*>(m.ci + kCandCap);
  m.keys = reinterpret_cast<uint64_t*>(m.xchg + NT);
  m.band = reinterpret_cast<int*>(m.keys);
  return m;
}

// ----------------------------------------------------------------------------- helpers
// A row whose float64 refinement window held more than kCandCap scores: its boundary
// follows fp32 order (ties to the lower index) instead of the reference's float64 order.
// Flag bit 4 plus a count of such rows in the word after the flag word (hylra.h).
__device__ __forceinline__ void refine_skipped(int* flags) {
  atomicOr(flags, 4);
  atomicAdd(flags + 1, 1);
}

struct Red {
  int i[kSelMaxWarps];
  float f[kSelMaxWarps];
  int wt[kSelMaxWarps];
  float pf[kSelMaxWarps];
  int pi[kSelMaxWarps];
  int misc[16];
  unsigned hist256[256];
};

// The CTA-wide barrier of the select code: barrier 0 over the NT threads running it — the
// whole CTA of topk_select_kernel, or the 4 consumer warps of the FULL kernel when the
// selection is fused into it (its producer warp has exited by then).
template <int NT>
__device__ __forceinline__ void sel_sync() {
  asm volatile("bar.sync 0, %0;" ::"n"(NT) : "memory");
}

// Block reductions: warps reduce with shuffles, the NT/32 warp partials go through shared
// memory and every warp reduces them again with shuffles (one shared load per lane instead
// of NT/32 per thread — the 1024-thread CTAs spent ~20% of their instructions there).
__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NT>
__device__ __forceinline__ int block_sum_int(int v, Red& r) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum_int(v);
  sel_sync<NT>();
  if (lane == 0) r.i[warp] = v;
  sel_sync<NT>();
  return warp_sum_int(lane < NT / 32 ? r.i[lane] : 0);
}
template <int NT>
__device__ __forceinline__ float block_max_float(float v, Red& r) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_max(v);
  sel_sync<NT>();
  if (lane == 0) r.f[warp] = v;
  sel_sync<NT>();
  return warp_max(lane < NT / 32 ? r.f[lane] : -INFINITY);
}

// Pass B's five reductions in one round: max, max, sum, sum, sum.
template <int NT>
__device__ __forceinline__ void block_reduce_pass_b(float& a, float& b, int& c, int& d, int& e,
                                                    Red& r) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_max(a);
  b = warp_max(b);
  c = warp_sum_int(c);
  d = warp_sum_int(d);
  e = warp_sum_int(e);
  sel_sync<NT>();
  if (lane == 0) {
    r.f[warp] = a;
    r.pf[warp] = b;
    r.i[warp] = c;
    r.wt[warp] = d;
    r.pi[warp] = e;
  }
  sel_sync<NT>();
  const bool in = lane < NT / 32;
  a = warp_max(in ? r.f[lane] : -INFINITY);
  b = warp_max(in ? r.pf[lane] : -INFINITY);
  c = warp_sum_int(in ? r.i[lane] : 0);
  d = warp_sum_int(in ? r.wt[lane] : 0);
  e = warp_sum_int(in ? r.pi[lane] : 0);
}

// Block exclusive scan of one int; returns the exclusive prefix, *total = block sum.
template <int NT>
__device__ __forceinline__ int block_scan(int v, int* total, Red& r) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  sel_sync<NT>();
  if (lane == 31) r.wt[warp] = x;
  sel_sync<NT>();
  // lane l scans the warp totals 0..l
  int t = lane < NT / 32 ? r.wt[lane] : 0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, t, o);
    if (lane >= o) t += y;
  }
  *total = __shfl_sync(0xffffffffu, t, 31);
  const int pre = __shfl_sync(0xffffffffu, t, (warp + 31) & 31);  // inclusive of warp-1
  return (warp > 0 ? pre : 0) + x - v;
}

// Block exclusive scan of 4 words at once (for packed 16-bit counts: every partial sum of
// a half stays below 2^16, so halves never carry into each other); tot = block sums.
template <int NT>
__device__ __forceinline__ void block_scan4(const uint32_t (&v)[4], uint32_t (&ex)[4],
                                            uint32_t (&tot)[4], Red& r) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) x[q] = v[q];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x[q], o);
      if (lane >= o) x[q] += y;
    }
  }
  uint32_t* arr[4] = {reinterpret_cast<uint32_t*>(r.i), reinterpret_cast<uint32_t*>(r.wt),
                      reinterpret_cast<uint32_t*>(r.pi), reinterpret_cast<uint32_t*>(r.f)};
  sel_sync<NT>();
  if (lane == 31) {
#pragma unroll
    for (int q = 0; q < 4; ++q) arr[q][warp] = x[q];
  }
  sel_sync<NT>();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t t = lane < NT / 32 ? arr[q][lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    const uint32_t pre = __shfl_sync(0xffffffffu, t, (warp + 31) & 31);  // through warp-1
    tot[q] = __shfl_sync(0xffffffffu, t, 31);
    ex[q] = (warp > 0 ? pre : 0u) + x[q] - v[q];
  }
}

// The finished selection row, copied to its mirror (hylra_step_options idx_mirror; often
// pinned host memory) with coalesced 16-byte stores once the row is complete: the
// compaction's own stores are scattered 4-byte writes, which across the link would cost
// far more than the row's 8 KB. The barrier makes every thread's idx stores visible.
template <int NT>
__device__ __forceinline__ void copy_to_mirror(const int32_t* out, int32_t* mir, int k) {
  if (mir == nullptr) return;
  sel_sync<NT>();
  const int tid = threadIdx.x;
  int done = 0;
  if (((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(mir)) & 15) == 0) {
    const int k4 = k >> 2;
    for (int i = tid; i < k4; i += NT)
      reinterpret_cast<int4*>(mir)[i] = __ldcg(reinterpret_cast<const int4*>(out) + i);
    done = k4 << 2;
  }
  for (int i = done + tid; i < k; i += NT) mir[i] = __ldcg(out + i);
}

// Warp-aggregated append: each thread adds `cnt` items; returns its first slot.
__device__ __forceinline__ int warp_append(int cnt, int* counter) {
  const int lane = threadIdx.x & 31;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int base = 0;
  if (lane == 31 && incl > 0) base = atomicAdd(counter, incl);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + incl - cnt;
}

struct RowReader {
  const float* base;  // score row of the group's first kv head
  int64_t hstride;    // elements between the group's kv-head rows
  int sg;
  __device__ __forceinline__ float at(int i) const {
    float s = __ldcg(base + i);
    for (int h = 1; h < sg; ++h) s += __ldcg(base + h * hstride + i);
    return s;
  }
  __device__ __forceinline__ float4 at4(int i4) const {
    float4 s = __ldcg(reinterpret_cast<const float4*>(base) + i4);
    for (int h = 1; h < sg; ++h) {
      const float4 t = __ldcg(reinterpret_cast<const float4*>(base + h * hstride) + i4);
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    return s;
  }
};

__device__ __forceinline__ float lane4(const float4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

template <typename T>
__device__ __forceinline__ double elem_f64(const void* p, int64_t i) {
  return (double)to_f32(reinterpret_cast<const T*>(p)[i]);
}

// float64 selection score of a token: agg = sum over (kv head of the group, query head g)
// of (q . k) / sqrt(d) in the reference's head order (engine.py:177-181). kLpt lanes share a
// token (lane sub handles dims sub, sub + kLpt, ...), so a warp scores kTpw tokens at once;
// every lane of the warp must call it (sub-group shuffles).
constexpr int kLpt = 8, kTpw = 32 / kLpt;
static __device__ double token_score_f64(const SelectParams& p, int layer, int kvl, int b, int grp,
                                  int tok) {
  const int sub = threadIdx.x & (kLpt - 1);
  const double sqd = sqrt((double)p.D);
  double agg = 0.0;
  for (int hh = 0; hh < p.sel_group; ++hh) {
    const int kh = grp * p.sel_group + hh;
    const int64_t koff = kvl * p.kv_sl + b * p.kv_sb + kh * p.kv_sh + (int64_t)tok * p.D;
    for (int g = 0; g < p.G; ++g) {
      const int64_t qoff = layer * p.q_sl + b * p.q_sb + (int64_t)(kh * p.G + g) * p.D;
      double part0 = 0.0, part1 = 0.0;
      if (p.dtype == 0) {
#pragma unroll 4
        for (int i = sub; i < p.D; i += 2 * kLpt) {
          part0 += elem_f64<__nv_bfloat16>(p.q, qoff + i) * elem_f64<__nv_bfloat16>(p.k, koff + i);
          part1 += elem_f64<__nv_bfloat16>(p.q, qoff + i + kLpt) *
                   elem_f64<__nv_bfloat16>(p.k, koff + i + kLpt);
        }
      } else {
#pragma unroll 4
        for (int i = sub; i < p.D; i += 2 * kLpt) {
          part0 += elem_f64<float>(p.q, qoff + i) * elem_f64<float>(p.k, koff + i);
          part1 += elem_f64<float>(p.q, qoff + i + kLpt) * elem_f64<float>(p.k, koff + i + kLpt);
        }
      }
      double part = part0 + part1;
#pragma unroll
      for (int o = kLpt / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      agg += part / sqd;
    }
  }
  return agg;
}

// float64 scores of candidate tokens toks[0..n); kTpw tokens per warp.
template <int NT>
__device__ void rescore_f64(const SelectParams& p, int slot, int b, int grp, const int* toks,
                            double* vals, int n) {
  const int warp = threadIdx.x >> 5, sub = threadIdx.x & (kLpt - 1);
  const int slot_in_warp = (threadIdx.x & 31) / kLpt;
  for (int c0 = warp * kTpw; c0 < n; c0 += (NT / 32) * kTpw) {  // warp-uniform trip count
    const int c = c0 + slot_in_warp;
    const double agg = token_score_f64(p, p.layers[slot], p.kv_layers[slot], b, grp,
                                       toks[min(c, n - 1)]);
    if (sub == 0 && c < n) vals[c] = agg;
  }
}

__device__ __forceinline__ unsigned long long f64_key(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_f64(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// float64 scores of candidate BLOCKS blocks[0..n): the max over the block's tokens of the
// token score (engine.py:256-262 + attention.py:287-295); the per-block max goes through
// ordered 64-bit keys in place of vals. vals[c] holds the block's fp32 score on entry.
// Only tokens whose fp32 score is >= that score - tau are re-scored: with fp32 scores within
// tau/2 of float64 (the premise of the refinement window), the float64 maximiser t* obeys
// s32(t*) >= s64(t*) - tau/2 >= s64(t_max32) - tau/2 >= s32(t_max32) - tau. If more than
// kSmallN tokens qualify (or token scores are absent) every token is re-scored.
template <int NT>
__device__ void rescore_f64_blocks(const SelectParams& p, int slot, int b, int grp,
                                   const int* blocks, double* vals, int n, float tau,
                                   uint64_t* list) {
  __shared__ int s_cnt;
  const int warp = threadIdx.x >> 5, sub = threadIdx.x & (kLpt - 1);
  const int slot_in_warp = (threadIdx.x & 31) / kLpt;
  const int bs = p.block_size;
  const int total = n * bs;
  if (threadIdx.x == 0) s_cnt = p.tok_scores ? 0 : kSmallN + 1;
  sel_sync<NT>();
  if (p.tok_scores) {
    const float* trow = p.tok_scores +
                        ((int64_t)(slot * p.B + b) * p.Hkv + grp * p.sel_group) * p.tok_row_stride;
    for (int e = threadIdx.x; e < total; e += NT) {
      const int c = e / bs;
      const int tok = blocks[c] * bs + (e - c * bs);
      if (tok >= p.n_tokens) continue;
      float s = trow[tok];  // the pooling kernel's fp32 head-order sum
      for (int h = 1; h < p.sel_group; ++h) s += trow[(int64_t)h * p.tok_row_stride + tok];
      if (s >= (float)vals[c] - tau) {
        const int pos = atomicAdd(&s_cnt, 1);
        if (pos < kSmallN) list[pos] = ((uint64_t)c << 32) | (uint32_t)tok;
      }
    }
  }
  sel_sync<NT>();
  const bool listed = s_cnt <= kSmallN;
  const int items = listed ? s_cnt : total;
  unsigned long long* vk = reinterpret_cast<unsigned long long*>(vals);
  for (int c = threadIdx.x; c < n; c += NT) vk[c] = 0ull;
  sel_sync<NT>();
  for (int e0 = warp * kTpw; e0 < items; e0 += (NT / 32) * kTpw) {  // warp-uniform trips
    const int e = min(e0 + slot_in_warp, items - 1);
    int c, tok;
    if (listed) {
      c = (int)(list[e] >> 32);
      tok = (int)(uint32_t)list[e];
    } else {
      c = e / bs;
      tok = blocks[c] * bs + (e - c * bs);
    }
    const bool ok = e0 + slot_in_warp < items && tok < p.n_tokens;
    const double agg = token_score_f64(p, p.layers[slot], p.kv_layers[slot], b, grp,
                                       ok ? tok : blocks[c] * bs);
    if (ok && sub == 0) atomicMax(vk + c, f64_key(agg));
  }
  sel_sync<NT>();
  for (int c = threadIdx.x; c < n; c += NT) vals[c] = key_f64(vk[c]);
}

// MSB-first 4 x 8-bit radix select of the rank-`rank` (1-based, descending) score of the
// row: T, #(s > T). Degenerate-row fallback only.
template <int NT>
__device__ void radix_select_row(const RowReader& rd, int n, int rank, Red& r, float* T_out,
                                 int* gt_out) {
  const int tid = threadIdx.x, lane = tid & 31;
  uint32_t prefix = 0, mask = 0;
  int krem = rank;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int j = tid; j < 256; j += NT) r.hist256[j] = 0;
    sel_sync<NT>();
    for (int base = 0; base < n; base += NT) {
      const int j = base + tid;
      bool act = false;
      unsigned dig = 0;
      if (j < n) {
        const uint32_t key = float_key(rd.at(j));
        act = (key & mask) == prefix;
        dig = (key >> shift) & 255u;
      }
      const unsigned am = __ballot_sync(0xffffffffu, act);
      if (act) {
        const unsigned peers = __match_any_sync(am, dig);
        if (lane == __ffs(peers) - 1) atomicAdd(r.hist256 + dig, (unsigned)__popc(peers));
      }
    }
    sel_sync<NT>();
    if (tid == 0) {
      int acc = 0, d = 255;
      for (; d > 0; --d) {
        if (acc + (int)r.hist256[d] >= krem) break;
        acc += r.hist256[d];
      }
      r.misc[8] = d;
      r.misc[9] = acc;
    }
    sel_sync<NT>();
    krem -= r.misc[9];
    prefix |= (uint32_t)r.misc[8] << shift;
    mask |= 255u << shift;
    sel_sync<NT>();
  }
  *T_out = key_float(prefix);
  *gt_out = rank - krem;
}

// Descending bitonic sort of np (power of two) 64-bit keys in shared memory.
template <int NT>
__device__ void bitonic_sort_desc(uint64_t* a, int np) {
  for (int size = 2; size <= np; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (np >> 1); t += NT) {
        const int i = 2 * t - (t & (stride - 1));
        const int j = i + stride;
        const uint64_t x = a[i], y = a[j];
        if ((x < y) == ((i & size) == 0)) {
          a[i] = y;
          a[j] = x;
        }
      }
      sel_sync<NT>();
    }
  }
}

// Rows of at most kSmallN scores (block rows, short caches): one exact sort of
// (score desc, index asc) keys replaces phases A-D. Tokens ranked above the window are set
// in the bitmap; the window [T - tau, T + tau] (refine) goes to cv/ci for the shared
// re-score + rank step. Without refinement (or with non-finite scores, or a window larger
// than kCandCap, flagged 4) the first k sorted entries are the answer.
template <int NT>
__device__ void small_row_select(const SelectParams& p, const RowReader& rd, int n, int k,
                                 bool refine, const SelSmem& sm, Red& red, int* above_w,
                                 int* nw_out, float* tau_out) {
  const int tid = threadIdx.x;
  uint64_t* keys = sm.keys;
  int np = 64;
  while (np < n) np <<= 1;
  float nanacc = 0.f, mx = 0.f;
  for (int i = tid; i < np; i += NT) {
    uint64_t key = 0ull;  // padding sorts after every real entry
    if (i < n) {
      const float v = rd.at(i);
      nanacc = fmaf(v, 0.f, nanacc);
      mx = fmaxf(mx, fabsf(v));
      key = ((uint64_t)float_key(v) << 32) | (uint32_t)(~(uint32_t)i);
    }
    keys[i] = key;
  }
  const int bad = block_sum_int<NT>(nanacc != nanacc ? 1 : 0, red);
  mx = block_max_float<NT>(mx, red);
  if (bad && tid == 0) atomicOr(p.flags, 2);
  sel_sync<NT>();
  bitonic_sort_desc<NT>(keys, np);
  auto val = [&](int pos) { return key_float((uint32_t)(keys[pos] >> 32)); };
  auto tok = [&](int pos) { return (int)(~(uint32_t)keys[pos]); };
  int a = k, z = k;
  if (refine && !bad) {
    const float T = val(k - 1);
    const float tau = *tau_out = fmaxf(p.tau_rel * mx, 1e-30f);
    const float lo_w = T - tau, hi_w = T + tau;
    int ca = 0, cz = 0;
    for (int pos = tid; pos < n; pos += NT) {
      const float v = val(pos);
      ca += v > hi_w;
      cz += v >= lo_w;
    }
    a = block_sum_int<NT>(ca, red);
    z = block_sum_int<NT>(cz, red);
    if (z - a > kCandCap) {
      if (tid == 0) refine_skipped(p.flags);
      a = z = k;
    }
  }
  for (int pos = tid; pos < z; pos += NT) {
    const int i = tok(pos);
    if (pos < a) {
      atomicOr(sm.bitmap + (i >> 5), 1u << (i & 31));
    } else {
      sm.cv[pos - a] = (double)val(pos);
      sm.ci[pos - a] = i;
    }
  }
  *above_w = a;
  *nw_out = z - a;
}

// ----------------------------------------------------------------------------- hist path
// The rank-`rank` (1-based, descending) value among nc floats in shared memory: MSB-first
// 4 x 8-bit radix select on the order-preserving keys; warp 0 scans each digit histogram.
template <int NT>
__device__ float smem_kth_largest(const float* v, int nc, int rank, Red& r) {
  const int tid = threadIdx.x, lane = tid & 31;
  uint32_t prefix = 0, mask = 0;
  int krem = rank;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int j = tid; j < 256; j += NT) r.hist256[j] = 0;
    sel_sync<NT>();
    for (int j = tid; j < nc; j += NT) {
      const uint32_t key = float_key(v[j]);
      if ((key & mask) == prefix) atomicAdd(r.hist256 + ((key >> shift) & 255u), 1u);
    }
    sel_sync<NT>();
    if (tid < 32) {
      // lane l owns digits 255 - 8l .. 248 - 8l (descending)
      int h[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        h[j] = (int)r.hist256[255 - 8 * lane - j];
        sum += h[j];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int acc = incl - sum;  // digits above this lane's
      if (acc < krem && krem <= incl) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (acc < krem && krem <= acc + h[j]) {
            r.misc[8] = 255 - 8 * lane - j;
            r.misc[9] = acc;
          }
          acc += h[j];
        }
      }
    }
    sel_sync<NT>();
    krem -= r.misc[9];
    prefix |= (uint32_t)r.misc[8] << shift;
    mask |= 255u << shift;
    sel_sync<NT>();
  }
  return key_float(prefix);
}

// The rank-r (1-based, descending) value among the nc candidates, most of which share the
// top kHistShift-complement bits b1: candidates above bin b1 rank first; inside b1 two digit
// rounds (bits 19..8 through a 4096-bin histogram in `scratch`, then bits 7..0) find the
// exact key. Falls back to the 4-round radix select when T lies outside b1.
template <int NT>
__device__ float cand_kth_largest(const float* v, int nc, int r, int b1, unsigned* scratch,
                                  Red& red) {
  const int tid = threadIdx.x;
  int hi = 0, in = 0;
  for (int j = tid; j < nc; j += NT) {
    const int bj = hist_bin(v[j]);
    hi += bj > b1;
    in += bj == b1;
  }
  for (int j = tid; j < kHistBins; j += NT) scratch[j] = 0u;
  hi = block_sum_int<NT>(hi, red);
  in = block_sum_int<NT>(in, red);
  if (r <= hi || r > hi + in) return smem_kth_largest<NT>(v, nc, r, red);
  int rr = r - hi;
  // digit 1: bits 19..8
  for (int j = tid; j < nc; j += NT) {
    const uint32_t key = float_key(v[j]);
    if ((int)(key >> kHistShift) == b1) atomicAdd(scratch + ((key >> 8) & 0xFFFu), 1u);
  }
  sel_sync<NT>();
  constexpr int PER = kHistBins / NT;
  int h[PER], sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    h[j] = (int)scratch[tid * PER + j];
    sum += h[j];
  }
  int tot;
  const int ex = block_scan<NT>(sum, &tot, red);
  int acc = tot - ex - sum;  // members in higher threads' digits
  if (acc < rr && rr <= acc + sum) {
#pragma unroll
    for (int j = PER - 1; j >= 0; --j) {
      if (acc < rr && rr <= acc + h[j]) {
        red.misc[8] = tid * PER + j;
        red.misc[9] = acc;
      }
      acc += h[j];
    }
  }
  for (int j = tid; j < 256; j += NT) red.hist256[j] = 0u;
  sel_sync<NT>();
  const uint32_t d1 = (uint32_t)red.misc[8];
  rr -= red.misc[9];
  const uint32_t pre = ((uint32_t)b1 << kHistShift) | (d1 << 8);
  // digit 2: bits 7..0
  for (int j = tid; j < nc; j += NT) {
    const uint32_t key = float_key(v[j]);
    if ((key >> 8) == (pre >> 8)) atomicAdd(red.hist256 + (key & 255u), 1u);
  }
  sel_sync<NT>();
  if (tid < 32) {
    int hh[8], ss = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      hh[j] = (int)red.hist256[255 - 8 * tid - j];
      ss += hh[j];
    }
    int incl = ss;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (tid >= o) incl += y;
    }
    int a = incl - ss;
    if (a < rr && rr <= incl) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (a < rr && rr <= a + hh[j]) red.misc[10] = 255 - 8 * tid - j;
        a += hh[j];
      }
    }
  }
  sel_sync<NT>();
  return key_float(pre | (uint32_t)red.misc[10]);
}

// Step 1 of the histogram path: from this thread's PER = kHistBins / NT bins of a row
// histogram (ascending from bin tid * PER), the bin b1 holding rank k from the top and the
// candidate value range [c_lo, c_hi] = b1 widened by the refinement half-width bound
// tau_rel * max|s| (max|s| bounded by the occupied range of bins). False when the
// histogram does not describe the row (count != n) or holds +-inf / NaN bins.
template <int NT>
__device__ bool hist_b1(const uint32_t (&hb)[kHistBins / NT], int n, int k, bool refine,
                        float tau_rel, Red& red, int* b1_out, float* c_lo, float* c_hi) {
  constexpr int PER = kHistBins / NT;
  const int tid = threadIdx.x;
  int sum = 0, nz_hi = -1, nz_lo = kHistBins;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    sum += (int)hb[j];
    if (hb[j]) {
      nz_hi = tid * PER + j;
      nz_lo = min(nz_lo, tid * PER + j);
    }
  }
  int tot;
  const int ex = block_scan<NT>(sum, &tot, red);
  const int above_blk = tot - ex - sum;  // tokens in higher threads' bins
  if (tid == 0) red.misc[0] = -1;
  sel_sync<NT>();
  if (above_blk < k && k <= above_blk + sum) {
    int acc = above_blk;
#pragma unroll
    for (int j = PER - 1; j >= 0; --j) {
      if (acc < k && k <= acc + (int)hb[j]) red.misc[0] = tid * PER + j;
      acc += (int)hb[j];
    }
  }
  {
    float fhi = (float)nz_hi, flo = (float)(-nz_lo);
    int z0 = 0, z1 = 0, z2 = 0;
    block_reduce_pass_b<NT>(fhi, flo, z0, z1, z2, red);
    nz_hi = (int)fhi;
    nz_lo = -(int)flo;
  }
  const int b1 = red.misc[0];
  constexpr int kInfHi = (int)(0xFF800000u >> kHistShift);
  constexpr int kInfLo = (int)(0x007FFFFFu >> kHistShift);
  if (tot != n || b1 < 0 || nz_hi >= kInfHi || nz_lo <= kInfLo) return false;
  const float vmax_b = key_float(((uint32_t)nz_hi << kHistShift) | ((1u << kHistShift) - 1));
  const float vmin_b = key_float((uint32_t)nz_lo << kHistShift);
  const float tau_b = refine ? fmaxf(tau_rel * fmaxf(fabsf(vmax_b), fabsf(vmin_b)), 1e-30f) : 0.f;
  *b1_out = b1;
  *c_lo = key_float((uint32_t)b1 << kHistShift) - tau_b;
  *c_hi = key_float(((uint32_t)b1 << kHistShift) | ((1u << kHistShift) - 1)) + tau_b;
  return true;
}

// Step 3 of the histogram path, shared with the cooperative select: the exact k-th value T
// (rank r among the nc candidates), then candidates above the window [T - tau, T + tau]
// (T exactly without refinement) join `bitmap`, the window goes to wv / wi in `scratch`
// (>= kHistBins * 4 bytes). *above_add = candidates above the window. False when the window
// exceeds kCandCap.
template <int NT>
__device__ bool cands_window(const float* cand_v, const int* cand_i, int nc, int r, int b1,
                            float tau, bool refine, uint8_t* scratch, uint32_t* bitmap,
                            Red& red, double** wv_out, int** wi_out, int* above_add,
                            int* nw_out) {
  const int tid = threadIdx.x;
  const float T = cand_kth_largest<NT>(cand_v, nc, r, b1, reinterpret_cast<unsigned*>(scratch),
                                       red);
  const float lo_w = refine ? T - tau : T, hi_w = refine ? T + tau : T;
  double* wv = reinterpret_cast<double*>(scratch);
  int* wi = reinterpret_cast<int*>(scratch + (size_t)kCandCap * 8);
  if (tid == 0) red.misc[5] = 0;
  sel_sync<NT>();
  int abv = 0;
  for (int base = 0; base < nc; base += NT) {  // warp-uniform trip count (warp_append)
    const int j = base + tid;
    bool in = false;
    float v = 0.f;
    int ii = 0;
    if (j < nc) {
      v = cand_v[j];
      ii = cand_i[j];
      if (v > hi_w) {
        atomicOr(bitmap + (ii >> 5), 1u << (ii & 31));
        ++abv;
      } else {
        in = v >= lo_w;
      }
    }
    const int pos = warp_append(in ? 1 : 0, &red.misc[5]);
    if (in && pos < kCandCap) {
      wv[pos] = (double)v;
      wi[pos] = ii;
    }
  }
  *above_add = block_sum_int<NT>(abv, red);  // (its barriers publish misc[5])
  const int nw = red.misc[5];
  sel_sync<NT>();
  if (nw > kCandCap) return false;
  *wv_out = wv;
  *wi_out = wi;
  *nw_out = nw;
  return true;
}

// Histogram-driven prefix of a token row's selection (sel_group 1, n > kSmallN), replacing
// the sampled passes A-D: hb = this thread's kHistBins / NT bins of the row's histogram
// (ascending from bin tid * (kHistBins / NT)), read and re-zeroed by the caller.
//  1. the bin b1 holding rank k from the top, the count above it and the occupied range of
//     bins (which bounds max|s|, hence the refinement half-width tau) — no row access;
//  2. ONE pass over the row (two chunks of loads in flight): tokens above b1 widened by tau go
//     straight into the bitmap, tokens of b1 (+- tau) into a candidate list, with max/min and
//     the non-finite check riding along;
//  3. the exact k-th value T among the candidates; candidates above the window
//     [T - tau, T + tau] (T exactly without refinement) join the bitmap, the window goes to
//     wv / wi for the float64 re-score and rank step of the caller.
// Same T, tau and window as the sampled path, hence the same selection. Returns false (the
// caller then runs the sampled path) when the histogram does not describe the row, a bin
// holds too many candidates, the row holds NaN / inf, or the window exceeds kCandCap.
template <int NT>
__device__ __forceinline__ bool hist_select(const SelectParams& p, const RowReader& rd,
                                            const uint32_t (&hb)[kHistBins / NT], int n, int k,
                                            bool refine,
                                            uint8_t* sraw, Red& red, double** wv_out,
                                            int** wi_out, int* above_out, int* nw_out,
                                            float* tau_out, int* cin_out, long long* marks) {
  constexpr int kChunk = sel_chunk<NT>();
  const int tid = threadIdx.x;
  // ---- 1. the bin of rank k
  int b1;
  float c_lo, c_hi;
  if (!hist_b1<NT>(hb, n, k, refine, p.tau_rel, red, &b1, &c_lo, &c_hi)) return false;
  marks[0] = clock64();

  // ---- 2. one pass over the row
  const size_t bb = sel_bitmap_bytes(n, NT);
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(sraw);
  float* cand_v = reinterpret_cast<float*>(sraw + bb);
  int* cand_i = reinterpret_cast<int*>(sraw + bb + 4 * (size_t)kHistCandCap);
  uint8_t* scratch = sraw + bb + 8 * (size_t)kHistCandCap;
  const int nwords = (int)(bb / 4);
  for (int w = tid; w < nwords; w += NT) bitmap[w] = 0u;
  if (tid == 0) red.misc[3] = 0;
  sel_sync<NT>();
  const int nch = (n + kChunk - 1) / kChunk;
  const int n4 = (n + 3) >> 2;
  float nanacc = 0.f, vmax = -INFINITY, vmin = INFINITY;
  int c_above = 0;
  // the next chunk's loads are in flight while the current one is classified
  auto load = [&](int c, float4 (&vv)[8]) {
    const int w4 = (c * kChunk + tid * 32) >> 2;
#pragma unroll
    for (int u = 0; u < 8; ++u) vv[u] = (w4 + u < n4) ? rd.at4(w4 + u) : make_float4(0, 0, 0, 0);
  };
  auto classify = [&](int c, const float4 (&vv)[8]) {
    const int w4 = (c * kChunk + tid * 32) >> 2;
    uint32_t word = 0u, cand = 0u;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const float v = lane4(vv[u], cc);
        if (4 * (w4 + u) + cc < n) {
          nanacc = fmaf(v, 0.f, nanacc);
          vmax = fmaxf(vmax, v);
          vmin = fminf(vmin, v);
          word |= (v > c_hi) ? (1u << (u * 4 + cc)) : 0u;
          cand |= (v >= c_lo && v <= c_hi) ? (1u << (u * 4 + cc)) : 0u;
        }
      }
    }
    bitmap[c * NT + tid] = word;
    c_above += __popc(word);
    int pos = warp_append(__popc(cand), &red.misc[3]);
    while (cand) {
      const int bit = __ffs(cand) - 1;
      cand &= cand - 1;
      if (pos < kHistCandCap) {
        float e = vv[0].x;
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            if (u * 4 + cc == bit) e = lane4(vv[u], cc);
        cand_v[pos] = e;
        cand_i[pos] = 4 * w4 + bit;
      }
      ++pos;
    }
  };
  {
    float4 va[8], vb[8];
    if (nch > 0) load(0, va);
    for (int c = 0; c < nch; c += 2) {
      if (c + 1 < nch) load(c + 1, vb);
      classify(c, va);
      if (c + 1 < nch) {
        if (c + 2 < nch) load(c + 2, va);
        classify(c + 1, vb);
      }
    }
  }
  int bad, dummy = 0;
  {
    float nmin = -vmin;
    bad = nanacc != nanacc ? 1 : 0;
    block_reduce_pass_b<NT>(vmax, nmin, bad, c_above, dummy, red);
    vmin = -nmin;
  }
  const int nc = red.misc[3];
  const int r = k - c_above;
  *cin_out = nc;
  marks[1] = clock64();
  if (bad || nc > kHistCandCap || r < 1 || r > nc) {
    sel_sync<NT>();
    return false;
  }
  // ---- 3. exact T, the window and the candidates above it
  const float tau = refine ? fmaxf(p.tau_rel * fmaxf(fabsf(vmax), fabsf(vmin)), 1e-30f) : 0.f;
  int above_add = 0;
  if (!cands_window<NT>(cand_v, cand_i, nc, r, b1, tau, refine, scratch, bitmap, red, wv_out,
                        wi_out, &above_add, nw_out))
    return false;
  marks[2] = clock64();
  *above_out = c_above + above_add;
  *tau_out = tau;
  return true;
}

// Phase-record of one selection row (info[] / diagnostics).
struct SelStats {
  int mode, cin;
  long long t0, t1, t2, t3;
};

// The common tail of every selection path: the boundary window wv / wi (nw scores, fp32
// values) is re-scored in float64 (refine) and its top k - above_w by (score desc, index
// asc) join `bitmap`, whose tokens above the window are already set; then the index-ordered
// compaction of the bitmap (word w = tokens [32 w, 32 w + 32)) writes the k indices
// ascending (the reference's canonical TopKSet order), copied to the mirror if any.
template <int NT>
__device__ void select_finish(const SelectParams& p, int grp, int b, int slot, uint32_t* bitmap,
                              double* wv, int* wi, int nw, int above_w, float tau_w, bool refine,
                              int n, int k, int32_t* out, int32_t* mir, int32_t* info, Red& red,
                              bool release, uint64_t* keys, const SelStats& st) {
  constexpr int kChunk = sel_chunk<NT>();
  const int tid = threadIdx.x;
  const int nch = (n + kChunk - 1) / kChunk;
  // ---- window: re-score (refine) and keep the top k - above_w by (score desc, index asc)
  if (nw > 0) {
    sel_sync<NT>();
    if (refine) {
      if (p.block_size > 1)
        rescore_f64_blocks<NT>(p, slot, b, grp, wi, wv, nw, tau_w, keys);
      else rescore_f64<NT>(p, slot, b, grp, wi, wv, nw);
      sel_sync<NT>();
    }
    const int take = k - above_w;
    for (int j = tid; j < nw; j += NT) {
      const double vj = wv[j];
      const int ij = wi[j];
      int rank = 0;
      for (int i = 0; i < nw; ++i) {
        const double vi = wv[i];
        rank += (vi > vj) || (vi == vj && wi[i] < ij);
      }
      if (rank < take) atomicOr(bitmap + (ij >> 5), 1u << (ij & 31));
    }
  }
  sel_sync<NT>();

  const long long t4 = clock64();  // window done: compaction next
  if (release) pdl_launch_dependents();
  // ---- E. index-ordered compaction of the bitmap: 8 chunks per block scan (their
  //         per-thread counts packed 2 x 16 bits per word), 2 barriers per 8 chunks
  int run = 0;
  if (nch == 1) {  // one chunk (wide CTAs, short rows): a single-word scan
    const uint32_t w = bitmap[tid];
    int tot;
    int pos = block_scan<NT>(__popc(w), &tot, red);
    uint32_t m = w;
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      if (pos < k) out[pos] = tid * 32 + bit;
      ++pos;
    }
    run = tot;
  }
  for (int c0 = 0; nch > 1 && c0 < nch; c0 += 8) {
    uint32_t w[8], pk[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      w[j] = (c0 + j < nch) ? bitmap[(c0 + j) * NT + tid] : 0u;
      pk[j >> 1] |= (uint32_t)__popc(w[j]) << (16 * (j & 1));
    }
    uint32_t ex[4], tot[4];
    block_scan4<NT>(pk, ex, tot, red);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (c0 + j >= nch) break;
      int pos = run + (int)((ex[j >> 1] >> (16 * (j & 1))) & 0xffffu);
      uint32_t m = w[j];
      while (m) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        if (pos < k) out[pos] = (c0 + j) * kChunk + tid * 32 + bit;
        ++pos;
      }
      run += (int)((tot[j >> 1] >> (16 * (j & 1))) & 0xffffu);
    }
  }
  // invariant: exactly k indices were emitted
  if (tid == 0 && run != k) atomicOr(p.flags, 8);
  copy_to_mirror<NT>(out, mir, k);
  if (info && tid == 0) {
    info[0] = k;
    info[1] = nw;
    info[2] = st.mode;
    info[3] = st.cin;
    info[4] = (int32_t)(st.t1 - st.t0);
    info[5] = (int32_t)(st.t2 - st.t1);
    info[6] = (int32_t)(st.t3 - st.t2);
    info[7] = (int32_t)(t4 - st.t3);
#ifdef HYLRA_TRACE
    info[1] = (int32_t)(clock64() - t4);  // diagnostics build: compaction cycles in place of nw
#endif
  }
}

// ----------------------------------------------------------------------------- kernel
// One selection row (slot, b, grp) by the NT threads 0..NT-1 of the calling CTA, with
// sel_smem_bytes(n_valid, NT) bytes of shared memory at sraw. Called by
// topk_select_kernel (one CTA per row) and, fused, by the FULL kernel's last CTA of a
// pair (NT = 128 consumer threads). release: let dependent launches start before the
// compaction (standalone kernel only).
// PIPE: pass B keeps the next chunk's loads in flight while it processes the current one
// (twice the registers: the fused select of the FULL kernel, which has them to spare).
template <int NT, bool PIPE = false>
__device__ void select_row(const SelectParams& p, int grp, int b, int slot, uint8_t* sraw,
                           Red& red, bool release, size_t smem_avail) {
  constexpr int kChunk = sel_chunk<NT>();
  const int tid = threadIdx.x;
  const int n = p.n_valid;
  const int k = p.k_eff;
  const int n4 = (n + 3) >> 2;
  const int row_id = (p.out_slot[slot] * p.B + b) * p.n_groups + grp;
  int32_t* out = p.idx + (int64_t)row_id * p.k_stride;
  int32_t* mir = p.idx_mirror ? p.idx_mirror + (int64_t)row_id * p.k_stride : nullptr;
  int32_t* info = p.info ? p.info + row_id * 8 : nullptr;
#ifdef HYLRA_TRACE
  if (info == nullptr && g_sel_info != nullptr) info = g_sel_info + row_id * 8;
#endif
  const SelSmem sm = carve<NT>(sraw, n);
  constexpr int kBandCap = sel_band_cap(NT, PIPE);
  const long long t0 = clock64();

  RowReader rd;
  if (p.pre_grouped) {
    rd.base = p.scores + ((int64_t)(slot * p.B + b) * p.n_groups + grp) * p.row_stride;
    rd.sg = 1;
  } else {
    rd.base = p.scores + ((int64_t)(slot * p.B + b) * p.Hkv + grp * p.sel_group) * p.row_stride;
    rd.sg = p.sel_group;
  }
  rd.hstride = p.row_stride;

  // the row's histogram (token rows, sel_group 1; FULL kernel): read into registers and
  // re-zeroed for the next step, whatever path the row then takes
  constexpr int HPER = kHistBins / NT;
  uint32_t hb[HPER];
  const bool use_hist = p.hist != nullptr && p.sel_group == 1 && !p.pre_grouped;
  const bool try_hist = use_hist && k < n && n > kSmallN &&
                        sel_hist_smem_bytes(n, NT) <= smem_avail;
  if (use_hist) {
    uint4* h4 = reinterpret_cast<uint4*>(
        p.hist + ((int64_t)(slot * p.B + b) * p.Hkv + grp) * kHistBins + tid * HPER);
#pragma unroll
    for (int q = 0; q < HPER / 4; ++q) {
      const uint4 x = __ldcg(h4 + q);
      hb[4 * q] = x.x;
      hb[4 * q + 1] = x.y;
      hb[4 * q + 2] = x.z;
      hb[4 * q + 3] = x.w;
      h4[q] = make_uint4(0, 0, 0, 0);
    }
  }

  if (k >= n) {
    // the budget covers the cache: every index (after the non-finite check)
    float nanacc = 0.f;
    for (int i = tid; i < n; i += NT) {
      nanacc = fmaf(rd.at(i), 0.f, nanacc);
      out[i] = i;
    }
    if (block_sum_int<NT>(nanacc != nanacc ? 1 : 0, red) && tid == 0) atomicOr(p.flags, 2);
    if (info && tid == 0) {
      for (int j = 0; j < 8; ++j) info[j] = 0;
      info[0] = k;
    }
    copy_to_mirror<NT>(out, mir, k);
    return;
  }

  const int nwords = (int)(sel_bitmap_bytes(n, NT) / 4);
  const bool refine = p.q != nullptr;
  const int nch = (n + kChunk - 1) / kChunk;
  int above_w = 0, nw = 0, mode = 0, cin = 0;
  float tau_w = 0.f;  // refinement half-width
  double* wv = sm.cv;  // the boundary window (value, index) for the re-score / rank step
  int* wi = sm.ci;
  long long t1, t2, t3;
  long long hm[3] = {0, 0, 0};
  const bool hist_done = try_hist &&
                         hist_select<NT>(p, rd, hb, n, k, refine, sraw, red, &wv, &wi,
                                         &above_w, &nw, &tau_w, &cin, hm);
  if (!hist_done) {
    for (int w = tid; w < nwords; w += NT) sm.bitmap[w] = 0u;
    for (int j = tid; j < kBins; j += NT) sm.hist[j] = 0u;
    if (tid == 0) red.misc[3] = red.misc[5] = 0;
  }
  if (hist_done) {
    // phases: histogram + bin of rank k | row pass | exact T | window (+ the rest below)
    mode = 6;
    t1 = hm[0];
    t2 = hm[1];
    t3 = clock64();
  } else if (n <= kSmallN) {
    small_row_select<NT>(p, rd, n, k, refine, sm, red, &above_w, &nw, &tau_w);
    mode = 3;
    t1 = t2 = t3 = clock64();
  } else {
    // ---- A. brackets [lo, hi] around the k-th rank from strided samples: their quantiles
    //         are read off a 1024-bin histogram over [sample min, sample max] (no sort);
    //         edges are widened outward so the bracket stays conservative. 4 NT samples;
    //         the fused select takes 2048 on rows over 64K tokens (a narrower band for
    //         passes H and D). Elsewhere the extra scattered reads measured slower, as the
    //         rows of a standalone launch at large batch no longer sit in L2 (cfg2 B=16,
    //         128K B=32).
    float hi, lo;
    // band expected to overflow the band list: build the histogram inside pass B instead
    bool inline_hist;
    auto pass_a = [&](auto spt_c) {
      constexpr int SPT = decltype(spt_c)::value, kS = SPT * NT, BPT = 1024 / NT;
      float smp[SPT];
      float smin = INFINITY, smax = -INFINITY;
#pragma unroll
      for (int j = 0; j < SPT; ++j) {
        smp[j] = rd.at((int)(((int64_t)(tid + j * NT) * n) / kS));
        smin = fminf(smin, smp[j]);
        smax = fmaxf(smax, smp[j]);
      }
      smax = block_max_float<NT>(smax, red);
      smin = -block_max_float<NT>(-smin, red);
      const float pr = (float)k / (float)n;
      const float delta = 3.0f * sqrtf(kS * pr * (1.0f - pr)) + 2.0f;
      const int hi_i = max(0, (int)floorf(pr * kS - delta));        // ranks from the top
      const int lo_i = min(kS - 1, (int)ceilf(pr * kS + delta));
      // (wide CTAs keep it inline: enough warps per scheduler to hide the atomics)
      inline_hist = NT >= 512 ||
                    (int64_t)(lo_i - hi_i + 3) * n > (int64_t)kBandCap * kS * 3 / 4;
      const float sscale = (smax > smin) ? 1024.f / (smax - smin) : 0.f;
      auto sbin = [&](float v) { return min(1023, max(0, (int)((v - smin) * sscale))); };
#pragma unroll
      for (int j = 0; j < SPT; ++j)
        if (isfinite(smp[j])) atomicAdd(sm.hist + sbin(smp[j]), 1u);
      sel_sync<NT>();
      // thread t scans sample bins 1023 - BPT t .. 1024 - BPT (t + 1) (descending)
      int hb[BPT], s4 = 0;
#pragma unroll
      for (int j = 0; j < BPT; ++j) {
        hb[j] = (int)sm.hist[1023 - (tid * BPT + j)];
        s4 += hb[j];
      }
      int tot;
      const int ex = block_scan<NT>(s4, &tot, red);
      int acc = ex;
#pragma unroll
      for (int j = 0; j < BPT; ++j) {
        const int bin = 1023 - (tid * BPT + j);
        // samples ranked [acc, acc + hb[j]) from the top live in this bin
        if (acc <= hi_i && hi_i < acc + hb[j]) red.misc[12] = bin;
        if (acc <= lo_i && lo_i < acc + hb[j]) red.misc[13] = bin;
        acc += hb[j];
      }
      if (tid == 0) red.misc[3] = red.misc[5] = 0;
      sel_sync<NT>();
      const int bh = red.misc[12], bl = red.misc[13];
      // hi: upper edge of the hi_i-th sample's bin (the top sample's bin: the sample max);
      // lo: lower edge of the lo_i-th sample's bin
      hi = (bh >= 1023) ? smax : smin + (float)(bh + 1) / sscale;
      lo = smin + (float)bl / sscale;
      for (int j = tid; j < kBins; j += NT) sm.hist[j] = 0u;
      sel_sync<NT>();
    };
    constexpr int kSptLong = NT >= 512 ? 4 : 2048 / NT;
    if (PIPE && n > 65536) pass_a(std::integral_constant<int, kSptLong>{});
    else pass_a(std::integral_constant<int, 4>{});
    t1 = clock64();

    // ---- B. above-bits -> bitmap, [lo, hi] -> histogram, max|s|, non-finite check.
    // Thread t owns 32 consecutive tokens of each 8K chunk: 8 float4, one bitmap word.
    // One retry with a bracket reaching the row's max (or min) if the sample bracket missed.
    const int nfull = n / kChunk;
    float mabs = 0.f, vmax = -INFINITY, vmin = INFINITY;
    int cgt = 0, bad = 0;
    bool brackets = false;
    float scale = 0.f;
    for (int attempt = 0; attempt < 2; ++attempt) {
      brackets = isfinite(lo) && isfinite(hi) && lo < hi;
      if (!brackets) {
        lo = -INFINITY;
        hi = INFINITY;
      }
      scale = brackets ? (float)kBins / (hi - lo) : 0.f;
      const float blo = lo, bhi = hi, bsc = scale;
      float nanacc = 0.f;
      int cg = 0, ci = 0;
      if (tid == 0) red.misc[10] = 0;  // band list length
      sel_sync<NT>();
      // per chunk: above-bits -> bitmap, band bits -> band list, max / min / NaN
      auto pass_b = [&](auto full_c, auto inl_c, int c, const float4 (&vv)[8]) {
        constexpr bool full = decltype(full_c)::value;
        constexpr bool inl = decltype(inl_c)::value;
        const int w4 = (c * kChunk + tid * 32) >> 2;
        uint32_t word = 0u, band = 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const float v = lane4(vv[u], cc);
            if (full || 4 * (w4 + u) + cc < n) {
              nanacc = fmaf(v, 0.f, nanacc);  // NaN iff some score is NaN or inf
              vmax = fmaxf(vmax, v);
              vmin = fminf(vmin, v);
              word |= (v > bhi) ? (1u << (u * 4 + cc)) : 0u;
              if (inl) {
                if (brackets && v >= blo && v <= bhi) {
                  atomicAdd(sm.hist + min(kBins - 1, (int)((v - blo) * bsc)), 1u);
                  band |= 1u << (u * 4 + cc);
                }
              } else {
                band |= (brackets && v >= blo && v <= bhi) ? (1u << (u * 4 + cc)) : 0u;
              }
            }
          }
        }
        sm.bitmap[c * NT + tid] = word;
        cg += __popc(word);
        ci += __popc(band);
        // band members' indices -> the band list (dropped past its capacity: pass H and
        // pass D then fall back to re-reading the row)
        int pos = warp_append(__popc(band), &red.misc[10]);
        while (band) {
          const int bit = __ffs(band) - 1;
          band &= band - 1;
          if (pos < kBandCap) sm.band[pos] = 4 * w4 + bit;
          ++pos;
        }
      };
      auto load_chunk = [&](int c, float4 (&vv)[8]) {
        const int w4 = (c * kChunk + tid * 32) >> 2;
        if (c < nfull) {
#pragma unroll
          for (int u = 0; u < 8; ++u) vv[u] = rd.at4(w4 + u);
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            vv[u] = (w4 + u < n4) ? rd.at4(w4 + u) : make_float4(0, 0, 0, 0);
        }
      };
      auto run_b = [&](int c, const float4 (&vv)[8]) {
        if (NT >= 512 || inline_hist) {
          if (c < nfull) pass_b(std::true_type{}, std::true_type{}, c, vv);
          else pass_b(std::false_type{}, std::true_type{}, c, vv);
        } else {
          if (c < nfull) pass_b(std::true_type{}, std::false_type{}, c, vv);
          else pass_b(std::false_type{}, std::false_type{}, c, vv);
        }
      };
      if constexpr (PIPE) {
        float4 va[8], vb[8];
        if (nch > 0) load_chunk(0, va);
        for (int c = 0; c < nch; c += 2) {
          if (c + 1 < nch) load_chunk(c + 1, vb);
          run_b(c, va);
          if (c + 1 < nch) {
            if (c + 2 < nch) load_chunk(c + 2, va);
            run_b(c + 1, vb);
          }
        }
      } else {
        for (int c = 0; c < nch; ++c) {
          float4 vv[8];
          load_chunk(c, vv);
          run_b(c, vv);
        }
      }
      {
        float nmin = -vmin;
        int nb = nanacc != nanacc ? 1 : 0;
        block_reduce_pass_b<NT>(vmax, nmin, nb, cg, ci, red);
        vmin = -nmin;
        bad = nb;
        cgt = cg;
        cin = ci;
      }
      mabs = fmaxf(fabsf(vmax), fabsf(vmin));
      if (bad || !brackets || (cgt < k && k <= cgt + cin) || attempt == 1) break;
      // retry once: the k-th value lies above hi (too many above) or below lo; the new
      // band's size is unknown, its histogram is built in the pass
      inline_hist = true;
      if (cgt >= k) {
        lo = hi;
        hi = vmax;
      } else {
        hi = lo;
        lo = vmin;
      }
      for (int j = tid; j < kBins; j += NT) sm.hist[j] = 0u;
      sel_sync<NT>();
    }
    if (bad && tid == 0) atomicOr(p.flags, 2);
    auto bin_of = [&](float v) { return min(kBins - 1, (int)((v - lo) * scale)); };
    // ---- H. histogram of the band [lo, hi] around rank k, built from the band list: only
    //         those scores are re-read (L2), 4 loads in flight per thread. Only the final
    //         bracket's histogram is needed, and only on the fast path.
    if (!inline_hist && brackets && cgt < k && k <= cgt + cin) {
      const int nband = red.misc[10];
      if (nband <= kBandCap) {
        constexpr int U = 4;
        for (int base = 0; base < nband; base += NT * U) {
          float v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = base + u * NT + tid;
            v[u] = j < nband ? rd.at(sm.band[j]) : 0.f;
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (base + u * NT + tid < nband) atomicAdd(sm.hist + bin_of(v[u]), 1u);
        }
      } else {
        for (int i4 = tid; i4 < n4; i4 += NT) {
          const float4 v4 = rd.at4(i4);
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const float v = lane4(v4, cc);
            if (4 * i4 + cc < n && v >= lo && v <= hi) atomicAdd(sm.hist + bin_of(v), 1u);
          }
        }
      }
      sel_sync<NT>();
    }
    t2 = clock64();

    const float tau = tau_w = fmaxf(p.tau_rel * mabs, 1e-30f);
    float T = 0.f, lo_w = 0.f, hi_w = 0.f;
    int why = 0;
    bool fast = brackets && cgt < k && k <= cgt + cin;
    if (!fast) why = !brackets ? 16 : (cgt >= k ? 32 : 48);
    if (fast) {
      // ---- C. bin b* holding rank r = k - cgt counted from the top
      const int r = k - cgt;
      constexpr int PER = kBins / NT;  // bins per thread, descending order
      int hb[PER], s = 0;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        hb[j] = (int)sm.hist[kBins - 1 - (tid * PER + j)];
        s += hb[j];
      }
      int tot;
      const int ex = block_scan<NT>(s, &tot, red);
      if (ex < r && r <= ex + s) {
        int acc = ex;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          if (acc < r && r <= acc + hb[j]) {
            red.misc[1] = kBins - 1 - (tid * PER + j);
            red.misc[2] = acc;
          }
          acc += hb[j];
        }
      }
      sel_sync<NT>();
      const int bstar = red.misc[1], cum_above = red.misc[2];
      // candidate bins [b_lo, b_hi]: b* widened by the refinement tolerance
      const int wb = refine ? (int)ceilf(tau * scale) + 1 : 0;
      const int b_lo = max(0, bstar - wb), b_hi = min(kBins - 1, bstar + wb);
      int above_bins = 0;
#pragma unroll
      for (int j = 0; j < PER; ++j) above_bins += (kBins - 1 - (tid * PER + j) > b_hi) ? hb[j] : 0;
      above_bins = block_sum_int<NT>(above_bins, red);

      // ---- D. second pass (L2): higher bins join the bitmap, candidate bins are collected.
      // bin_of is monotone, so "bin > b_hi" and "bin >= b_lo" are exact value thresholds,
      // found once by bisection over the ordered float keys.
      if (tid < 2) {
        const int target = (tid == 0) ? b_hi + 1 : b_lo;  // smallest v with bin_of(v) >= target
        uint32_t a = float_key(lo), z = float_key(hi);     // bin_of(lo)=0, bin_of(hi)=kBins-1
        if (target <= 0) {
          red.misc[6 + tid] = __float_as_int(lo);
        } else if (target > kBins - 1 || bin_of(hi) < target) {
          red.misc[6 + tid] = __float_as_int(INFINITY);
        } else {
          while (a < z) {  // invariant: bin_of(key_float(z)) >= target
            const uint32_t mid = a + (z - a) / 2;
            if (bin_of(key_float(mid)) >= target) z = mid;
            else a = mid + 1;
          }
          red.misc[6 + tid] = __float_as_int(key_float(z));
        }
      }
      sel_sync<NT>();
      const float v_hi = __int_as_float(red.misc[6]);  // v >= v_hi  <=>  bin > b_hi
      const float v_lo = __int_as_float(red.misc[7]);  // v >= v_lo  <=>  bin >= b_lo
      auto pass_d = [&](int c, bool full) {
        const int w4 = (c * kChunk + tid * 32) >> 2;
        float4 vv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          vv[u] = (full || w4 + u < n4) ? rd.at4(w4 + u) : make_float4(0, 0, 0, 0);
        uint32_t word = 0u, cand = 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const float v = lane4(vv[u], cc);
            const bool ok = full || 4 * (w4 + u) + cc < n;
            // above hi: already set in pass B; [v_hi, hi]: set now
            word |= (ok && v >= v_hi && v <= hi) ? (1u << (u * 4 + cc)) : 0u;
            // inside the band only: scores above hi were counted (and set) by pass B
            cand |= (ok && v >= v_lo && v < v_hi && v <= hi) ? (1u << (u * 4 + cc)) : 0u;
          }
        }
        if (word) sm.bitmap[c * NT + tid] |= word;
        int pos = warp_append(__popc(cand), &red.misc[3]);
        while (cand) {
          const int bit = __ffs(cand) - 1;
          cand &= cand - 1;
          if (pos < kCandCap) {
            float e = vv[0].x;
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
              for (int cc = 0; cc < 4; ++cc)
                if (u * 4 + cc == bit) e = lane4(vv[u], cc);
            sm.cv[pos] = (double)e;
            sm.ci[pos] = 4 * w4 + bit;
          }
          ++pos;
        }
      };
      const int nband = red.misc[10];
      if (nband <= kBandCap) {
        // the band list holds every score in [lo, hi]: only those are re-read
        constexpr int U = NT >= 512 ? 1 : 4;  // loads in flight per thread
        for (int base = 0; base < nband; base += NT * U) {
          int iu[U];
          float vu[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = base + u * NT + tid;
            iu[u] = j < nband ? sm.band[j] : 0;
            vu[u] = j < nband ? rd.at(iu[u]) : -INFINITY;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = iu[u];
            const float v = vu[u];
            const bool in = base + u * NT + tid < nband;
            if (in && v >= v_hi) atomicOr(sm.bitmap + (i >> 5), 1u << (i & 31));
            const bool cand = in && v >= v_lo && v < v_hi;
            int pos = warp_append(cand ? 1 : 0, &red.misc[3]);
            if (cand && pos < kCandCap) {
              sm.cv[pos] = (double)v;
              sm.ci[pos] = i;
            }
          }
        }
      } else {
        for (int c = 0; c < nfull; ++c) pass_d(c, true);
        if (nfull < nch) pass_d(nfull, false);
      }
      sel_sync<NT>();
      const int nc = red.misc[3];
      fast = nc >= 1 && nc <= kCandCap;
      if (!fast) why = 64;
      if (fast) {
        // exact T: rank r2 among the members of bin b*
        const int r2 = r - cum_above;
        for (int j = tid; j < nc; j += NT) {
          const float vj = (float)sm.cv[j];
          if (bin_of(vj) != bstar) continue;
          int gt = 0, ge = 0;
          for (int i = 0; i < nc; ++i) {
            const float vi = (float)sm.cv[i];
            if (bin_of(vi) != bstar) continue;
            gt += vi > vj;
            ge += vi >= vj;
          }
          if (gt < r2 && r2 <= ge) red.misc[4] = __float_as_int(vj);
        }
        sel_sync<NT>();
        T = __int_as_float(red.misc[4]);
        lo_w = refine ? T - tau : T;
        hi_w = refine ? T + tau : T;
        const int blw = lo_w >= lo ? bin_of(lo_w) : -1;
        const int bhw = hi_w <= hi ? bin_of(hi_w) : kBins;
        fast = blw >= b_lo && bhw <= b_hi;  // the window lies inside the candidate bins
        if (!fast) why = 80;
      }
      if (fast) {
        // keep the window in place; candidates above it are selected outright
        int abv = 0;
        for (int base = 0; base < nc; base += NT) {
          const int j = base + tid;
          double v = 0.0;
          int ii = 0;
          bool in = false;
          if (j < nc) {
            v = sm.cv[j];
            ii = sm.ci[j];
            in = (float)v >= lo_w && (float)v <= hi_w;
            if ((float)v > hi_w) {
              atomicOr(sm.bitmap + (ii >> 5), 1u << (ii & 31));
              ++abv;
            }
          }
          sel_sync<NT>();
          const int pos = warp_append(in ? 1 : 0, &red.misc[5]);
          if (in) {
            sm.cv[pos] = v;
            sm.ci[pos] = ii;
          }
        }
        above_w = cgt + above_bins + block_sum_int<NT>(abv, red);
        nw = red.misc[5];
        mode = refine ? 2 : 0;
      }
    }
    if (!fast) {
      // ---------------------------------------------------------------- generic path
      mode = 1 + why;
      int c_gt = 0;
      // why 80: the fast path found the exact k-th value T, only its refinement window
      // reaches past the band's bins: T stands, one pass over the row collects the window
      const bool t_known = why == 80;
      if (!t_known) radix_select_row<NT>(rd, n, k, red, &T, &c_gt);
      lo_w = refine ? T - tau : T;
      hi_w = refine ? T + tau : T;
      for (int w = tid; w < nwords; w += NT) sm.bitmap[w] = 0u;
      if (tid == 0) red.misc[5] = 0;
      sel_sync<NT>();
      int abv = 0, gt = 0;
      for (int b4 = 0; b4 < n4; b4 += 2 * NT) {  // 2 x 16-byte loads in flight per thread
        float4 va[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int i4 = b4 + u * NT + tid;
          va[u] = i4 < n4 ? rd.at4(i4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        uint32_t win = 0u;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int i = 4 * (b4 + u * NT + tid) + cc;
            const float v = lane4(va[u], cc);
            const bool ok = i < n;
            if (ok && v > hi_w) {
              atomicOr(sm.bitmap + (i >> 5), 1u << (i & 31));
              ++abv;
            }
            gt += (ok && v > T) ? 1 : 0;
            win |= (ok && v >= lo_w && v <= hi_w) ? (1u << (u * 4 + cc)) : 0u;
          }
        }
        int pos = warp_append(__popc(win), &red.misc[5]);
        while (win) {
          const int bit = __ffs(win) - 1;
          win &= win - 1;
          const int i = 4 * (b4 + (bit >> 2) * NT + tid) + (bit & 3);
          if (pos < kCandCap) {
            sm.cv[pos] = (double)lane4((bit >> 2) ? va[1] : va[0], bit & 3);
            sm.ci[pos] = i;
          }
          ++pos;
        }
      }
      if (t_known) c_gt = block_sum_int<NT>(gt, red);
      above_w = block_sum_int<NT>(abv, red);
      nw = red.misc[5];
      if (nw > kCandCap) {
        // the window cannot be held: resolve the exact fp32 ties at T by index order
        if (refine && tid == 0) refine_skipped(p.flags);
        if (refine) {
          for (int w = tid; w < nwords; w += NT) sm.bitmap[w] = 0u;
          sel_sync<NT>();
          for (int base = 0; base < n; base += NT) {
            const int i = base + tid;
            if (i < n && rd.at(i) > T) atomicOr(sm.bitmap + (i >> 5), 1u << (i & 31));
          }
        }
        int taken = refine ? c_gt : above_w;
        for (int base = 0; base < n; base += NT) {
          const int i = base + tid;
          const bool tie = i < n && rd.at(i) == T;
          int tot;
          const int pre = block_scan<NT>(tie ? 1 : 0, &tot, red);
          if (tie && taken + pre < k) atomicOr(sm.bitmap + (i >> 5), 1u << (i & 31));
          taken += tot;
        }
        nw = 0;
        mode = 5;
      }
    }
    t3 = clock64();
  }

  SelStats st{mode, cin, t0, t1, t2, t3};
  select_finish<NT>(p, grp, b, slot, sm.bitmap, wv, wi, nw, above_w, tau_w, refine, n, k, out,
                    mir, info, red, release, sm.keys, st);
}

// ----------------------------------------------------------------------------- cooperative
// Cooperative selection of a FULL pair's row inside the single-launch step (token rows,
// sel_group 1). Selected by the pair's final CTA alone, a row is read in full (the score row
// and its histogram) through ONE SM while every other SM streams K/V at the HBM roofline;
// that SM's share of the saturated memory system (~10 GB/s) made the select ~40 us, the
// critical path of small-batch steps (scripts/trace_single.py). Here the splits of the pair
// share the work, each on its own slice of the row, in parallel across SMs:
//  1. each split, done streaming, arrives on `arrive1`; the last one reads the row histogram
//     (re-zeroing it), finds the bin of rank k and publishes the candidate range
//     (coop_publish, release flag);
//  2. each split classifies its slice, prefetched into shared memory while its split-K merge
//     runs: bitmap words (tokens above the range) to the row's global bitmap, candidates to
//     the row's global list, max / min / non-finite / counts by atomics; then it arrives on
//     `arrive2` (coop_classify);
//  3. the last one resolves the row — exact T among the candidates, the float64 window, the
//     compaction — and re-zeroes the record (coop_final).
// Same T, tau and window as the single-CTA paths, hence the same selection. A row the
// histogram cannot serve, or with NaN / inf or too many candidates, is selected by step 3's
// CTA through the sampled path over the global row.

// Step 1: all NT threads of the last split to arrive.
template <int NT>
__device__ void coop_publish(const SelectParams& p, int row, CoopRow* rec, int n, Red& red) {
  constexpr int HPER = kHistBins / NT;
  const int tid = threadIdx.x;
  uint32_t hb[HPER];
  uint4* h4 = reinterpret_cast<uint4*>(p.hist + (int64_t)row * kHistBins + tid * HPER);
#pragma unroll
  for (int q = 0; q < HPER / 4; ++q) {
    const uint4 x = __ldcg(h4 + q);
    hb[4 * q] = x.x;
    hb[4 * q + 1] = x.y;
    hb[4 * q + 2] = x.z;
    hb[4 * q + 3] = x.w;
    h4[q] = make_uint4(0, 0, 0, 0);
  }
  int b1 = -1;
  float c_lo = 0.f, c_hi = 0.f;
  const bool refine = p.q != nullptr;
  const bool ok = p.k_eff < n && n > kSmallN &&
                  hist_b1<NT>(hb, n, p.k_eff, refine, p.tau_rel, red, &b1, &c_lo, &c_hi);
  if (tid == 0) {
    rec->b1 = ok ? b1 : -1;
    rec->c_lo = c_lo;
    rec->c_hi = c_hi;
    __threadfence();
    st_release_gpu(&rec->flag, 1);
  }
}

// Step 2: all NT threads of every split. slice = the split's scores [s0, s1) in shared
// memory (or null: read from the global row). Returns true in the last split to arrive.
template <int NT>
__device__ bool coop_classify(const SelectParams& p, int row, CoopRow* rec,
                              const float* score_row, const float* slice, int s0, int s1,
                              int n, int splits, Red& red) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    // bounded: a flag that never comes (a corrupted workspace) becomes HYLRA_FLAG_INTERNAL
    for (long long spins = 0; ld_acquire_gpu(&rec->flag) == 0; ++spins) {
      if (spins > (1ll << 25)) {
        atomicOr(p.flags, 8);
        break;
      }
      __nanosleep(32);
    }
  }
  sel_sync<NT>();
  (void)ld_acquire_gpu(&rec->flag);
  const int b1 = __ldcg(&rec->b1);
  if (b1 >= 0) {
    const float c_lo = __ldcg(&rec->c_lo), c_hi = __ldcg(&rec->c_hi);
    uint32_t* bits = p.coop_bits + (int64_t)row * p.coop_words;
    float* cv = p.coop_cv + (int64_t)row * kHistCandCap;
    int* ci = p.coop_ci + (int64_t)row * kHistCandCap;
    float nanacc = 0.f, vmax = -INFINITY, vmin = INFINITY;
    int c_above = 0;
    const int w0 = s0 >> 5, w1 = (s1 + 31) >> 5;
    for (int base = w0; base < w1; base += NT) {  // warp-uniform trips (warp_append)
      const int w = base + tid;
      uint32_t word = 0u, cand = 0u;
      float4 vv[8];
      if (w < w1) {
        const float4* src = slice ? reinterpret_cast<const float4*>(slice + (32 * w - s0))
                                  : reinterpret_cast<const float4*>(score_row + 32 * w);
#pragma unroll
        for (int u = 0; u < 8; ++u) vv[u] = slice ? src[u] : __ldcg(src + u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const float v = lane4(vv[u], cc);
            if (32 * w + 4 * u + cc < s1) {
              nanacc = fmaf(v, 0.f, nanacc);
              vmax = fmaxf(vmax, v);
              vmin = fminf(vmin, v);
              word |= (v > c_hi) ? (1u << (u * 4 + cc)) : 0u;
              cand |= (v >= c_lo && v <= c_hi) ? (1u << (u * 4 + cc)) : 0u;
            }
          }
        }
        bits[w] = word;
        c_above += __popc(word);
      }
      int pos = warp_append(__popc(cand), &rec->n_cand);
      while (cand) {
        const int bit = __ffs(cand) - 1;
        cand &= cand - 1;
        if (pos < kHistCandCap) {
          float e = vv[0].x;
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int cc = 0; cc < 4; ++cc)
              if (u * 4 + cc == bit) e = lane4(vv[u], cc);
          cv[pos] = e;
          ci[pos] = 32 * w + bit;
        }
        ++pos;
      }
    }
    float nmin = -vmin;
    int bad = nanacc != nanacc ? 1 : 0, dummy = 0;
    block_reduce_pass_b<NT>(vmax, nmin, bad, c_above, dummy, red);
    if (tid == 0) {
      atomicAdd(&rec->c_above, c_above);
      atomicMax(&rec->vmax_key, float_key(vmax));
      atomicMax(&rec->vmin_nkey, ~float_key(-nmin));
      if (bad) atomicOr(&rec->bad, 1);
    }
  }
  __threadfence();
  sel_sync<NT>();
  if (tid == 0) red.misc[15] = atomicAdd(&rec->arrive2, 1) == splits - 1;
  sel_sync<NT>();
  const bool last = red.misc[15] != 0;
  if (last) __threadfence();
  return last;
}

// Step 3: all NT threads of the last split; sraw = `avail` bytes of free shared memory.
template <int NT>
__device__ void coop_final(const SelectParams& p, int grp, int b, int slot, int row,
                           CoopRow* rec, uint8_t* sraw, size_t avail, Red& red) {
  const int tid = threadIdx.x;
  const int n = p.n_valid, k = p.k_eff;
  const long long t0 = clock64();
  const int b1 = __ldcg(&rec->b1);
  const int nc = __ldcg(&rec->n_cand);
  const int c_above = __ldcg(&rec->c_above);
  const int bad = __ldcg(&rec->bad);
  const float vmax = key_float(__ldcg(&rec->vmax_key));
  const float vmin = key_float(~__ldcg(&rec->vmin_nkey));
  const int r = k - c_above;
  const size_t bb = sel_bitmap_bytes(n, NT);
  const bool refine = p.q != nullptr;
  bool ok = b1 >= 0 && !bad && nc <= kHistCandCap && r >= 1 && r <= nc &&
            bb + (size_t)kHistCandCap * 8 + (size_t)kHistBins * 4 <= avail;
  const int row_id = (p.out_slot[slot] * p.B + b) * p.n_groups + grp;
  int32_t* out = p.idx + (int64_t)row_id * p.k_stride;
  int32_t* mir = p.idx_mirror ? p.idx_mirror + (int64_t)row_id * p.k_stride : nullptr;
  int32_t* info = p.info ? p.info + row_id * 8 : nullptr;
#ifdef HYLRA_TRACE
  if (info == nullptr && g_sel_info != nullptr) info = g_sel_info + row_id * 8;
#endif
  if (ok) {
    uint32_t* bitmap = reinterpret_cast<uint32_t*>(sraw);
    float* cand_v = reinterpret_cast<float*>(sraw + bb);
    int* cand_i = reinterpret_cast<int*>(sraw + bb + 4 * (size_t)kHistCandCap);
    uint8_t* scratch = sraw + bb + 8 * (size_t)kHistCandCap;
    const uint32_t* bits = p.coop_bits + (int64_t)row * p.coop_words;
    const float* cv = p.coop_cv + (int64_t)row * kHistCandCap;
    const int* ci = p.coop_ci + (int64_t)row * kHistCandCap;
    const int words = (n + 31) >> 5, nwords = (int)(bb / 4);
    for (int w = tid; w < nwords; w += NT) bitmap[w] = w < words ? __ldcg(bits + w) : 0u;
    for (int j = tid; j < nc; j += NT) {
      cand_v[j] = __ldcg(cv + j);
      cand_i[j] = __ldcg(ci + j);
    }
    sel_sync<NT>();
    const long long t1 = clock64();
    const float tau = refine ? fmaxf(p.tau_rel * fmaxf(fabsf(vmax), fabsf(vmin)), 1e-30f) : 0.f;
    double* wv = nullptr;
    int* wi = nullptr;
    int above_add = 0, nw = 0;
    ok = cands_window<NT>(cand_v, cand_i, nc, r, b1, tau, refine, scratch, bitmap, red, &wv, &wi,
                          &above_add, &nw);
    if (ok) {
      SelStats st{7, nc, t0, t1, t1, clock64()};
      select_finish<NT>(p, grp, b, slot, bitmap, wv, wi, nw, c_above + above_add, tau, refine, n,
                        k, out, mir, info, red, false, nullptr, st);
    }
  }
  if (!ok) {  // the sampled path over the global row (the histogram is already re-zeroed)
    SelectParams q = p;
    q.hist = nullptr;
    q.coop = nullptr;
    sel_sync<NT>();
    select_row<NT, true>(q, grp, b, slot, sraw, red, false, avail);
  }
  if (tid == 0) {  // every other split is past its last access to the record
    rec->arrive1 = 0;
    rec->arrive2 = 0;
    rec->flag = 0;
    rec->n_cand = 0;
    rec->c_above = 0;
    rec->vmax_key = 0u;
    rec->vmin_nkey = 0u;
    rec->bad = 0;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) topk_select_kernel(const SelectParams p) {
  extern __shared__ __align__(16) uint8_t sraw[];
  __shared__ Red red;
  pdl_wait();
  select_row<NT>(p, blockIdx.x, blockIdx.y, blockIdx.z, sraw, red, true, p.smem_bytes);
}

}  // namespace hylra
