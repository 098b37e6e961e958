// rowsel.cuh — shared-memory-resident exact top-k of one score row per CTA cluster.
//
// Same rule as select.cuh (attention.py:264-275 topk_of_logits: the k highest, ties to the
// LOWER index, ascending output; the float64 boundary refinement of hylra_topk_select), so
// its index sets are bit-identical to select_row's. What differs is where the row lives:
// select_row streams the row from L2 two or three times with a few loads in flight per
// thread (latency-bound: ~30 us for one 32K row on an idle GPU), while here the row is
// pulled into shared memory ONCE by the bulk-copy engine (cp.async.bulk, the whole slice in
// flight at once) and every pass runs out of shared memory.
//
// Long rows are split over a thread-block CLUSTER of C CTAs (C in {1, 2, 4, 8}: up to 40960
// tokens per CTA, 160 KB of row + 28 KB of tables), one contiguous slice each: block-local
// histograms and candidates, merged through distributed shared memory (DSMEM) — the
// "block-local candidates, then a global merge" of the north star. Per row:
//   0. bulk-load the slice (sel_group > 1: the group's other kv-head rows added in head
//      order, as RowReader::at);
//   1. min / max / non-finite of the row (cluster reduction);
//   2. a 2048-bin linear histogram over [min, max] (monotone bin_of, as select_row's),
//      summed over the cluster: the bin b* holding rank k and the bins within the
//      refinement half-width tau of it;
//   3. bits of tokens in bins above that band -> the slice's bitmap; the band's tokens
//      (value, index) -> CTA 0's candidate list (DSMEM, warp-aggregated);
//   4. CTA 0: the exact k-th value T among b*'s members, the window [T - tau, T + tau]
//      (refine) or {T} (no refine); candidates above the window are selected, the window is
//      re-scored in float64 (rescore_f64, heads summed in reference order) and its top
//      k - above members by (score desc, index asc) join the owning CTA's bitmap;
//   5. index-ordered compaction: each CTA writes its slice's indices at the offset of the
//      slices before it.
// Degenerate rows (non-finite scores, a band over kCandCap candidates, a window reaching
// past the band) take the generic path: an exact 3-round MSB radix select of T over the
// shared-memory keys, one pass collecting the window, and — if the window exceeds kCandCap —
// the exact fp32 ties at T in index order (HYLRA_FLAG_REFINE_SKIPPED when refining), exactly
// as select_row.
#pragma once

#include <cooperative_groups.h>

#include "select.cuh"

namespace hylra {

constexpr int kRowselThreads = 1024;
constexpr int kRowselMaxSlice = 40960;  // tokens of a row per CTA
constexpr int kRowselMaxCluster = 8;
// no finer split when spreading few rows over SMs: a 32K row on 8 CTAs (4096 tokens each)
// spends ~14K cycles summing the cluster histograms through DSMEM against ~10K on 4 CTAs
// (scripts/rowsel_prof.py); layer-sequential cfg2 B=1 497 vs 514 us
constexpr int kRowselMinSlice = 8192;

// Tokens per CTA for an n-token row on a C-CTA cluster (a whole number of bitmap words).
__host__ __device__ constexpr int rowsel_slice(int n, int c) { return ((n + c - 1) / c + 31) & ~31; }
// Dynamic shared memory: row slice, window values / indices, two histograms, bitmap.
constexpr int kRsQMax = 2048;  // staged query floats: sel_group x G x D (refinement)
__host__ __device__ constexpr size_t rowsel_smem_bytes(int slice) {
  return (size_t)slice * 4 + (size_t)kCandCap * 12 + 2 * kBins * 4 + (size_t)slice / 8 +
         (size_t)kRsQMax * 4 + 128;
}
// Smallest cluster (power of two, <= kRowselMaxCluster) whose slices fit; 0 = none.
__host__ __device__ constexpr int rowsel_cluster(int n) {
  return n <= kRowselMaxSlice ? 1
         : n <= 2 * kRowselMaxSlice ? 2
         : n <= 4 * kRowselMaxSlice ? 4
         : n <= 8 * kRowselMaxSlice ? 8 : 0;
}

struct RsStat {  // one CTA's partial statistics, read by its cluster peers
  float vmax, vmin;
  int bad, above, gt, ties, sel, pad;
};
struct RsShared {  // CTA 0's decisions and the cluster-wide candidate list length
  int n_cand, mode, generic, nw, above_w, taken_gt, pad[2];
  float T, lo_w, hi_w, tau;
};

template <int C>
__device__ __forceinline__ void rs_sync() {
  if constexpr (C > 1) cooperative_groups::this_cluster().sync();
  else __syncthreads();
}
template <int C, typename T>
__device__ __forceinline__ T* rs_peer(T* p, int r) {
  if constexpr (C > 1) return cooperative_groups::this_cluster().map_shared_rank(p, r);
  else return p;
}

// float64 selection score of window token `tok` (token_score_f64's arithmetic, operation for
// operation, so the two selects rank a window identically) with the group's query heads
// staged in shared memory as floats (qs[(hh G + g) D + i], exact bf16 / fp32 values) and the
// token's K values fetched once into registers: one memory round trip per token instead of
// one per query head. kLpt lanes per token; every lane of the warp must call it.
__device__ __forceinline__ double rs_token_score(const SelectParams& p, const float* qs, int kvl,
                                                 int b, int grp, int tok) {
  const int sub = threadIdx.x & (kLpt - 1);
  const double sqd = sqrt((double)p.D);
  constexpr int kMaxPer = 128 / kLpt;  // K values per lane (head_dim <= 128)
  double agg = 0.0;
  for (int hh = 0; hh < p.sel_group; ++hh) {
    const int kh = grp * p.sel_group + hh;
    const int64_t koff = kvl * p.kv_sl + b * p.kv_sb + kh * p.kv_sh + (int64_t)tok * p.D;
    // all of the token's loads issued back to back (branch-free: the dtype test is hoisted
    // and indices past head_dim are clamped, their values unused): one memory latency
    float kv[kMaxPer];
    if (p.dtype == 0) {
      const __nv_bfloat16* kp = reinterpret_cast<const __nv_bfloat16*>(p.k) + koff;
#pragma unroll
      for (int j = 0; j < kMaxPer; ++j) kv[j] = __bfloat162float(kp[min(sub + j * kLpt, p.D - 1)]);
    } else {
      const float* kp = reinterpret_cast<const float*>(p.k) + koff;
#pragma unroll
      for (int j = 0; j < kMaxPer; ++j) kv[j] = kp[min(sub + j * kLpt, p.D - 1)];
    }
    for (int g = 0; g < p.G; ++g) {
      const float* qr = qs + (hh * p.G + g) * p.D;
      double part0 = 0.0, part1 = 0.0;
#pragma unroll
      for (int j = 0; j + 1 < kMaxPer; j += 2) {
        const int i = sub + j * kLpt;
        if (i < p.D) {
          part0 += (double)qr[i] * (double)kv[j];
          part1 += (double)qr[i + kLpt] * (double)kv[j + 1];
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

// One token per warp, its query heads in parallel: lanes g' * kLpt + sub (g' < 32 / kLpt)
// evaluate head 4c + g' of each chunk c of 4 heads with token_score_f64's per-head arithmetic
// (the same sub lanes, the same xor tree inside the 8-lane group), and every lane then adds
// the heads' part / sqrt(d) in head order — the reference order, bit for bit the per-token
// evaluation of rs_token_score, with the heads' dependent chains overlapped.
__device__ __forceinline__ double rs_token_score_wide(const SelectParams& p, const float* qs,
                                                      int kvl, int b, int grp, int tok) {
  constexpr int kHpw = 32 / kLpt;  // heads per warp pass
  const int lane = threadIdx.x & 31, sub = lane & (kLpt - 1), gl = lane / kLpt;
  const double sqd = sqrt((double)p.D);
  constexpr int kMaxPer = 128 / kLpt;
  double agg = 0.0;
  for (int hh = 0; hh < p.sel_group; ++hh) {
    const int kh = grp * p.sel_group + hh;
    const int64_t koff = kvl * p.kv_sl + b * p.kv_sb + kh * p.kv_sh + (int64_t)tok * p.D;
    float kv[kMaxPer];
    if (p.dtype == 0) {
      const __nv_bfloat16* kp = reinterpret_cast<const __nv_bfloat16*>(p.k) + koff;
#pragma unroll
      for (int j = 0; j < kMaxPer; ++j) kv[j] = __bfloat162float(kp[min(sub + j * kLpt, p.D - 1)]);
    } else {
      const float* kp = reinterpret_cast<const float*>(p.k) + koff;
#pragma unroll
      for (int j = 0; j < kMaxPer; ++j) kv[j] = kp[min(sub + j * kLpt, p.D - 1)];
    }
    for (int g0 = 0; g0 < p.G; g0 += kHpw) {
      const int g = min(g0 + gl, p.G - 1);
      const float* qr = qs + (hh * p.G + g) * p.D;
      double part0 = 0.0, part1 = 0.0;
#pragma unroll
      for (int j = 0; j + 1 < kMaxPer; j += 2) {
        const int i = sub + j * kLpt;
        if (i < p.D) {
          part0 += (double)qr[i] * (double)kv[j];
          part1 += (double)qr[i + kLpt] * (double)kv[j + 1];
        }
      }
      double part = part0 + part1;
#pragma unroll
      for (int o = kLpt / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      const double term = part / sqd;
#pragma unroll
      for (int u = 0; u < kHpw; ++u) {
        const double t = __shfl_sync(0xffffffffu, term, u * kLpt);
        if (g0 + u < p.G) agg += t;
      }
    }
  }
  return agg;
}

template <int NT>
__device__ void rs_rescore(const SelectParams& p, const float* qs, int slot, int b, int grp,
                           const int* toks, double* vals, int n) {
  if (qs == nullptr) {
    rescore_f64<NT>(p, slot, b, grp, toks, vals, n);
    return;
  }
  if (n <= NT / 32) {  // few tokens: one per warp, heads in parallel
    const int warp = threadIdx.x >> 5;
    if (warp < n) {
      const double agg = rs_token_score_wide(p, qs, p.kv_layers[slot], b, grp, toks[warp]);
      if ((threadIdx.x & 31) == 0) vals[warp] = agg;
    }
    return;
  }
  const int warp = threadIdx.x >> 5, sub = threadIdx.x & (kLpt - 1);
  const int slot_in_warp = (threadIdx.x & 31) / kLpt;
  for (int c0 = warp * kTpw; c0 < n; c0 += (NT / 32) * kTpw) {  // warp-uniform trip count
    const int c = c0 + slot_in_warp;
    const double agg = rs_token_score(p, qs, p.kv_layers[slot], b, grp, toks[min(c, n - 1)]);
    if (sub == 0 && c < n) vals[c] = agg;
  }
}

template <int C>
__global__ void __launch_bounds__(kRowselThreads, 1) rowsel_kernel(const SelectParams p, int S) {
  constexpr int NT = kRowselThreads, NW = NT / 32;
  extern __shared__ __align__(128) uint8_t rs_smem[];
  __shared__ uint64_t bar;
  __shared__ RsStat st;
  __shared__ RsShared sh;
  __shared__ RsStat all;  // the cluster totals (warp 0 folds the peers' RsStat)
  __shared__ Red red;
  const int cr = C > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  const int grp = blockIdx.x / C, b = blockIdx.y, slot = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = p.n_valid, k = p.k_eff;
  const int lo = cr * S;
  const int m = max(0, min(n - lo, S));  // tokens of this slice
  const int words = (m + 31) >> 5;
  float* row = reinterpret_cast<float*>(rs_smem);
  double* wv = reinterpret_cast<double*>(rs_smem + (size_t)S * 4);  // CTA 0: candidates / window
  int* wi = reinterpret_cast<int*>(wv + kCandCap);
  unsigned* hist = reinterpret_cast<unsigned*>(wi + kCandCap);  // [2][kBins]
  uint32_t* bitmap = hist + 2 * kBins;                          // [S / 32]
  float* qs = reinterpret_cast<float*>(bitmap + S / 32);        // [kRsQMax] staged queries
  const int row_id = (p.out_slot[slot] * p.B + b) * p.n_groups + grp;
  int32_t* out = p.idx + (int64_t)row_id * p.k_stride;
  int32_t* mir = p.idx_mirror ? p.idx_mirror + (int64_t)row_id * p.k_stride : nullptr;
  const bool refine = p.q != nullptr;
  const long long t0 = clock64();
#ifdef HYLRA_ROWSEL_PROF
  // diagnostics build: per-phase clock marks of CTA 0 in info[0..7]
  long long pm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define RS_MARK(i) pm[i] = clock64()
#else
#define RS_MARK(i)
#endif

  for (int j = tid; j < 2 * kBins; j += NT) hist[j] = 0u;
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    st = RsStat{-INFINITY, INFINITY, 0, 0, 0, 0, 0, 0};
    sh = RsShared{};
  }
  __syncthreads();
  pdl_wait();

  // ---- 0. the slice into shared memory (rows are padded to 8 scores: the 16-byte
  //         round-up stays inside the row)
  const float* rbase = p.pre_grouped
      ? p.scores + ((int64_t)(slot * p.B + b) * p.n_groups + grp) * p.row_stride
      : p.scores + ((int64_t)(slot * p.B + b) * p.Hkv + grp * p.sel_group) * p.row_stride;
  const int sg = p.pre_grouped ? 1 : p.sel_group;
  const uint32_t bytes = (uint32_t)((m * 4 + 15) & ~15);
  if (bytes > 0 && tid == 0) {
    mbar_arrive_expect_tx(&bar, bytes);
    for (uint32_t off = 0; off < bytes; off += 32768u)
      bulk_load(rs_smem + off, reinterpret_cast<const uint8_t*>(rbase + lo) + off,
                min(32768u, bytes - off), &bar);
  }
  // CTA 0 stages the group's query heads for the float64 re-score while the slice lands
  const int nq = p.sel_group * p.G * p.D;
  const bool stage_q = refine && cr == 0 && nq <= kRsQMax && p.D <= 128 && p.D % 16 == 0;
  if (stage_q) {
    for (int e = tid; e < nq; e += NT) {
      const int head = e / p.D, i = e % p.D;  // head = hh G + g
      const int hh = head / p.G, g = head % p.G;
      const int kh = grp * p.sel_group + hh;
      const int64_t qo = p.layers[slot] * p.q_sl + b * p.q_sb + (int64_t)(kh * p.G + g) * p.D + i;
      qs[e] = p.dtype == 0 ? (float)elem_f64<__nv_bfloat16>(p.q, qo) : (float)elem_f64<float>(p.q, qo);
    }
  }
  const float* qsp = stage_q ? qs : nullptr;
  if (bytes > 0) mbar_wait(&bar, 0);
  const long long t1 = clock64();  // the slice is in
  RS_MARK(0);
  for (int h = 1; h < sg; ++h) {  // the group's other kv-head rows, head order
    const float* rh = rbase + (int64_t)h * p.row_stride + lo;
    for (int i = tid; i < m; i += NT) row[i] += __ldcg(rh + i);
    __syncthreads();
  }

  // ---- 1. min / max / non-finite
  {
    float vmax = -INFINITY, vmin = INFINITY, nanacc = 0.f;
    const int m4 = m >> 2;
    for (int i4 = tid; i4 < m4; i4 += NT) {
      const float4 v = reinterpret_cast<const float4*>(row)[i4];
      nanacc = fmaf(v.x, 0.f, fmaf(v.y, 0.f, fmaf(v.z, 0.f, fmaf(v.w, 0.f, nanacc))));
      vmax = fmaxf(vmax, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
      vmin = fminf(vmin, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
    }
    for (int i = 4 * m4 + tid; i < m; i += NT) {
      const float v = row[i];
      nanacc = fmaf(v, 0.f, nanacc);
      vmax = fmaxf(vmax, v);
      vmin = fminf(vmin, v);
    }
    float nmin = -vmin;
    int bad = nanacc != nanacc ? 1 : 0, z0 = 0, z1 = 0;
    block_reduce_pass_b<NT>(vmax, nmin, bad, z0, z1, red);
    if (tid == 0) {
      st.vmax = vmax;
      st.vmin = -nmin;
      st.bad = bad;
    }
  }
  RS_MARK(1);
  rs_sync<C>();
  if (warp == 0) {
    RsStat q = lane < C ? *rs_peer<C>(&st, lane) : RsStat{-INFINITY, INFINITY, 0, 0, 0, 0, 0, 0};
    const float vmax = warp_max(q.vmax), vmin = -warp_max(-q.vmin);
    const int bad = warp_sum_int(q.bad);
    if (lane == 0) {
      all.vmax = vmax;
      all.vmin = vmin;
      all.bad = bad;
    }
  }
  __syncthreads();
  const float gmax = all.vmax, gmin = all.vmin;
  const bool bad = all.bad != 0;
  if (bad && cr == 0 && tid == 0) atomicOr(p.flags, 2);
  const float mabs = fmaxf(fabsf(gmax), fabsf(gmin));
  const float tau = fmaxf(p.tau_rel * mabs, 1e-30f);

  // ---- 2. linear histogram over [min, max]
  const float scale = gmax > gmin ? (float)kBins / (gmax - gmin) : 0.f;
  auto bin_of = [&](float v) { return min(kBins - 1, (int)((v - gmin) * scale)); };
  bool generic = bad || !(isfinite(gmin) && isfinite(gmax));
  int b_lo = 0, b_hi = kBins - 1, bstar = 0, cum_above = 0, above_bins = 0;
  if (!generic) {
    for (int i = tid; i < m; i += NT) atomicAdd(hist + bin_of(row[i]), 1u);
    rs_sync<C>();
    // thread t: bins kBins-1-2t, kBins-2-2t (descending), summed over the cluster
    int hb[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int bin = kBins - 1 - (2 * tid + j);
      unsigned s = 0;
#pragma unroll
      for (int r = 0; r < C; ++r) s += *rs_peer<C>(hist + bin, r);
      hb[j] = (int)s;
    }
    int tot;
    const int ex = block_scan<NT>(hb[0] + hb[1], &tot, red);
    if (ex < k && k <= ex + hb[0] + hb[1]) {
      const bool first = k <= ex + hb[0];
      red.misc[1] = kBins - 1 - (2 * tid + (first ? 0 : 1));
      red.misc[2] = first ? ex : ex + hb[0];
    }
    sel_sync<NT>();
    bstar = red.misc[1];
    cum_above = red.misc[2];
    const int wb = refine ? (int)ceilf(tau * scale) + 1 : 0;
    b_lo = max(0, bstar - wb);
    b_hi = min(kBins - 1, bstar + wb);
    int ab = 0, nc = 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int bin = kBins - 1 - (2 * tid + j);
      ab += bin > b_hi ? hb[j] : 0;
      nc += (bin >= b_lo && bin <= b_hi) ? hb[j] : 0;
    }
    int z0 = 0;
    float f0 = 0.f, f1 = 0.f;
    block_reduce_pass_b<NT>(f0, f1, ab, nc, z0, red);
    above_bins = ab;
    generic = nc > kCandCap;
  }

  const long long t2 = clock64();  // histogram done
  RS_MARK(2);
  if (!generic) {
    // ---- 3. bits above the band -> bitmap; the band -> CTA 0's candidate list
    int* ncand0 = rs_peer<C>(&sh.n_cand, 0);
    double* wv0 = rs_peer<C>(wv, 0);
    int* wi0 = rs_peer<C>(wi, 0);
    for (int w = warp; w < words; w += NW) {
      const int i = 32 * w + lane;
      const float v = i < m ? row[i] : -INFINITY;
      const int bn = bin_of(v);
      const bool in = i < m;
      const uint32_t up = __ballot_sync(0xffffffffu, in && bn > b_hi);
      const uint32_t cand = __ballot_sync(0xffffffffu, in && bn >= b_lo && bn <= b_hi);
      if (lane == 0) bitmap[w] = up;
      if (cand) {
        int base = 0;
        if (lane == 0) base = atomicAdd(ncand0, __popc(cand));
        base = __shfl_sync(0xffffffffu, base, 0);
        if ((cand >> lane) & 1u) {
          const int pos = base + __popc(cand & ((1u << lane) - 1u));
          wv0[pos] = (double)v;
          wi0[pos] = lo + i;
        }
      }
    }
    rs_sync<C>();
    RS_MARK(3);
    // ---- 4. CTA 0: exact T, the window, float64 re-score, winners -> owners' bitmaps
    if (cr == 0) {
      const int nc = sh.n_cand;
      const int r2 = k - cum_above;  // rank of T among b*'s members
      // b*'s members (<= nc <= kCandCap) into the idle second histogram, then ranked there
      float* mem = reinterpret_cast<float*>(hist + kBins);
      if (tid == 0) red.misc[3] = 0;
      sel_sync<NT>();
      for (int base = 0; base < nc; base += NT) {
        const int j = base + tid;
        const float vj = j < nc ? (float)wv[j] : 0.f;
        const bool in = j < nc && bin_of(vj) == bstar;
        const int pos = warp_append(in ? 1 : 0, &red.misc[3]);
        if (in) mem[pos] = vj;
      }
      sel_sync<NT>();
      const int nm = red.misc[3];
      for (int j = tid; j < nm; j += NT) {
        const float vj = mem[j];
        int gt = 0, ge = 0;
        for (int i = 0; i < nm; ++i) {
          const float vi = mem[i];
          gt += vi > vj;
          ge += vi >= vj;
        }
        if (gt < r2 && r2 <= ge) red.misc[4] = __float_as_int(vj);
      }
      sel_sync<NT>();
      const float T = __int_as_float(red.misc[4]);
      RS_MARK(4);
      const float lo_w = refine ? T - tau : T, hi_w = refine ? T + tau : T;
      const int blw = lo_w >= gmin ? bin_of(lo_w) : -1;
      const int bhw = hi_w <= gmax ? bin_of(hi_w) : kBins;
      if (blw >= b_lo && bhw <= b_hi) {
        // candidates above the window are selected; the window is compacted in place
        if (tid == 0) red.misc[5] = 0;
        int abv = 0;
        for (int base = 0; base < nc; base += NT) {
          const int j = base + tid;
          double v = 0.0;
          int ii = 0;
          bool in = false;
          if (j < nc) {
            v = wv[j];
            ii = wi[j];
            in = (float)v >= lo_w && (float)v <= hi_w;
            if ((float)v > hi_w) {
              atomicOr(rs_peer<C>(bitmap, ii / S) + ((ii % S) >> 5), 1u << (ii & 31));
              ++abv;
            }
          }
          sel_sync<NT>();
          const int pos = warp_append(in ? 1 : 0, &red.misc[5]);
          if (in) {
            wv[pos] = v;
            wi[pos] = ii;
          }
        }
        const int above_w = above_bins + block_sum_int<NT>(abv, red);
        const int nw = red.misc[5];
        if (tid == 0) {
          sh.mode = refine ? 7 : 8;
          sh.nw = nw;
          sh.above_w = above_w;
        }
        RS_MARK(5);
        if (nw > 0) {
          sel_sync<NT>();
          if (refine) {
            rs_rescore<NT>(p, qsp, slot, b, grp, wi, wv, nw);
            sel_sync<NT>();
          }
          RS_MARK(6);
          const int take = k - above_w;
          for (int j = tid; j < nw; j += NT) {
            const double vj = wv[j];
            const int ij = wi[j];
            int rank = 0;
            for (int i = 0; i < nw; ++i) {
              const double vi = wv[i];
              rank += (vi > vj) || (vi == vj && wi[i] < ij);
            }
            if (rank < take)
              atomicOr(rs_peer<C>(bitmap, ij / S) + ((ij % S) >> 5), 1u << (ij & 31));
          }
        }
      } else if (tid == 0) {
        sh.generic = 1;  // the window reaches past the band: T stands, the generic pass
        sh.T = T;        // collects the window
      }
    }
    rs_sync<C>();
    generic = rs_peer<C>(&sh, 0)->generic != 0;
  }

  if (generic) {
    // ---------------------------------------------------------------- generic path
    RsShared* s0 = rs_peer<C>(&sh, 0);
    float T;
    if (s0->generic) {
      T = s0->T;  // known from the band; only its window was too wide for it
    } else {
      // exact T: MSB-first radix select over the order-preserving keys, 11 + 11 + 10 bits,
      // histograms summed over the cluster (alternating buffers: a peer may still be
      // reading the previous round's)
      uint32_t prefix = 0u;
      int rank = k;
      rs_sync<C>();  // the peers are done reading step 2's histogram before it is re-zeroed
      for (int round = 0; round < 3; ++round) {
        const int shift = round == 0 ? 21 : (round == 1 ? 10 : 0);
        const int nb = round == 2 ? 1024 : 2048;
        const uint32_t pmask = round == 0 ? 0u : (round == 1 ? 0xffe00000u : 0xfffffc00u);
        unsigned* h = hist + (round & 1) * kBins;
        for (int j = tid; j < kBins; j += NT) h[j] = 0u;
        __syncthreads();
        for (int i = tid; i < m; i += NT) {
          const uint32_t key = float_key(row[i]);
          if ((key & pmask) == prefix) atomicAdd(h + ((key >> shift) & (nb - 1)), 1u);
        }
        rs_sync<C>();
        int hb[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int d = nb - 1 - (2 * tid + j);
          unsigned s = 0;
          if (d >= 0) {
#pragma unroll
            for (int r = 0; r < C; ++r) s += *rs_peer<C>(h + d, r);
          }
          hb[j] = (int)s;
        }
        int tot;
        const int ex = block_scan<NT>(hb[0] + hb[1], &tot, red);
        if (ex < rank && rank <= ex + hb[0] + hb[1]) {
          const bool first = rank <= ex + hb[0];
          red.misc[1] = nb - 1 - (2 * tid + (first ? 0 : 1));
          red.misc[2] = first ? ex : ex + hb[0];
        }
        sel_sync<NT>();
        prefix |= (uint32_t)red.misc[1] << shift;
        rank -= red.misc[2];
        sel_sync<NT>();
      }
      T = key_float(prefix);
    }
    const float lo_w = refine ? T - tau : T, hi_w = refine ? T + tau : T;
    // one pass: bits above the window, the window -> CTA 0, counts above T / ties at T
    if (cr == 0 && tid == 0) sh.n_cand = 0;
    rs_sync<C>();
    int* ncand0 = rs_peer<C>(&sh.n_cand, 0);
    double* wv0 = rs_peer<C>(wv, 0);
    int* wi0 = rs_peer<C>(wi, 0);
    int abv = 0, gt = 0;
    for (int w = warp; w < words; w += NW) {
      const int i = 32 * w + lane;
      const bool in = i < m;
      const float v = in ? row[i] : 0.f;
      const uint32_t up = __ballot_sync(0xffffffffu, in && v > hi_w);
      const uint32_t win = __ballot_sync(0xffffffffu, in && v >= lo_w && v <= hi_w);
      gt += (in && v > T) ? 1 : 0;
      if (lane == 0) {
        bitmap[w] = up;
        abv += __popc(up);
      }
      if (win) {
        int base = 0;
        if (lane == 0) base = atomicAdd(ncand0, __popc(win));
        base = __shfl_sync(0xffffffffu, base, 0);
        const int pos = base + __popc(win & ((1u << lane) - 1u));
        if (((win >> lane) & 1u) && pos < kCandCap) {
          wv0[pos] = (double)v;
          wi0[pos] = lo + i;
        }
      }
    }
    {
      int z = 0;
      float f0 = 0.f, f1 = 0.f;
      block_reduce_pass_b<NT>(f0, f1, abv, gt, z, red);
      if (tid == 0) {
        st.above = abv;
        st.gt = gt;
      }
    }
    rs_sync<C>();
    int above_w = 0, c_gt = 0;
    if (warp == 0) {
      const RsStat q = lane < C ? *rs_peer<C>(&st, lane) : RsStat{};
      above_w = warp_sum_int(lane < C ? q.above : 0);
      c_gt = warp_sum_int(lane < C ? q.gt : 0);
      if (lane == 0) {
        red.misc[8] = above_w;
        red.misc[9] = c_gt;
      }
    }
    __syncthreads();
    above_w = red.misc[8];
    c_gt = red.misc[9];
    const int nw = s0->n_cand;
    if (nw <= kCandCap) {
      if (cr == 0) {
        if (tid == 0) {
          sh.mode = 1 + (refine ? 2 : 0) + 64;
          sh.nw = nw;
          sh.above_w = above_w;
        }
        if (nw > 0) {
          if (refine) {
            rs_rescore<NT>(p, qsp, slot, b, grp, wi, wv, nw);
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
            if (rank < take)
              atomicOr(rs_peer<C>(bitmap, ij / S) + ((ij % S) >> 5), 1u << (ij & 31));
          }
        }
      }
    } else {
      // the window cannot be held: {s > T} plus the exact fp32 ties at T in index order
      if (refine && cr == 0 && tid == 0) refine_skipped(p.flags);
      if (cr == 0 && tid == 0) {
        sh.mode = 5;
        sh.nw = 0;
      }
      // warp w owns the contiguous words [w * wpw, (w + 1) * wpw): ties in index order
      const int wpw = (words + NW - 1) / NW;
      const int w0 = min(words, warp * wpw), w1 = min(words, w0 + wpw);
      int ties = 0;
      for (int w = w0; w < w1; ++w) {
        const int i = 32 * w + lane;
        const bool in = i < m;
        const float v = in ? row[i] : 0.f;
        const uint32_t up = __ballot_sync(0xffffffffu, in && v > T);
        const uint32_t tie = __ballot_sync(0xffffffffu, in && v == T);
        if (lane == 0) bitmap[w] = up;
        ties += __popc(tie);
      }
      int tot;
      const int wex = block_scan<NT>(lane == 0 ? ties : 0, &tot, red);  // ties before this warp
      if (tid == 0) st.ties = tot;
      rs_sync<C>();
      int off = 0;  // ties of the slices before this one
      for (int r = 0; r < cr; ++r) off += rs_peer<C>(&st, r)->ties;
      const int need = k - c_gt;
      int run = off + __shfl_sync(0xffffffffu, wex, 0);
      for (int w = w0; w < w1; ++w) {
        const int i = 32 * w + lane;
        const bool in = i < m;
        const bool t_ = in && row[i] == T;
        const uint32_t tie = __ballot_sync(0xffffffffu, t_);
        const int my = run + __popc(tie & ((1u << lane) - 1u));
        const uint32_t take = __ballot_sync(0xffffffffu, t_ && my < need);
        if (lane == 0) bitmap[w] |= take;
        run += __popc(tie);
      }
    }
    rs_sync<C>();
  }
  const long long t3 = clock64();
  RS_MARK(7);
  pdl_launch_dependents();

  // ---- 5. index-ordered compaction: thread t owns the contiguous words [t wpt, (t+1) wpt);
  //         one block scan of their counts, slice offsets from the peers' counts
  const int wpt = (words + NT - 1) / NT;
  const int w0 = min(words, tid * wpt), w1 = min(words, w0 + wpt);
  int cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(bitmap[w]);
  int tot;
  const int tex = block_scan<NT>(cnt, &tot, red);
  if (tid == 0) st.sel = tot;
  rs_sync<C>();
  int off = 0, total = 0;
#pragma unroll
  for (int r = 0; r < C; ++r) {
    const int s = rs_peer<C>(&st, r)->sel;
    off += r < cr ? s : 0;
    total += s;
  }
  int pos = off + tex;
  for (int w = w0; w < w1; ++w) {
    uint32_t word = bitmap[w];
    while (word) {
      const int bit = __ffs(word) - 1;
      word &= word - 1;
      if (pos < k) out[pos] = lo + 32 * w + bit;
      ++pos;
    }
  }
  if (cr == 0 && tid == 0 && total != k) atomicOr(p.flags, 8);  // invariant: k indices
  if (mir != nullptr) {
    __syncthreads();
    const int e = min(k, off + tot);
    for (int i = off + tid; i < e; i += NT) mir[i] = __ldcg(out + i);
  }
  if (cr == 0 && tid == 0 && p.info != nullptr) {
    int32_t* info = p.info + row_id * 8;
    info[0] = k;
    info[1] = sh.nw;
    info[2] = sh.mode;
    info[3] = C;
    info[4] = (int32_t)(t1 - t0);
    info[5] = (int32_t)(t2 - t1);
    info[6] = (int32_t)(t3 - t2);
    info[7] = (int32_t)(clock64() - t3);
#ifdef HYLRA_ROWSEL_PROF
    for (int j = 7; j > 0; --j) info[j] = (int32_t)(pm[j] - pm[j - 1]);
    info[0] = (int32_t)(pm[0] - t0);
#endif
  }
  rs_sync<C>();  // no CTA leaves while a peer may still read its shared memory
#undef RS_MARK
}

}  // namespace hylra
