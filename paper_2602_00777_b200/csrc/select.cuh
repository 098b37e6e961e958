// select.cuh — exact top-k selection over per-(slot, b, group) score rows.
//
// Reference: pkg/src/layerreuse/attention.py:264-275 topk_of_logits — the min(budget, N)
// highest logits, ties won by the LOWER index (stable argsort of -logits), returned
// ascending; engine.py:169 clamps the budget per step; engine.py:177-183 scores are the
// head-order sum of per-head scaled logits.
//
// Algorithm (one 1024-thread CTA per row, no global atomics):
//   1. stage the row (sum of `sel_group` score rows, head order) in shared memory when it
//      fits, and reduce max|s| / non-finite flag;
//   2. find the exact k-th largest value T:
//        fast path  — sort a strided sample, bracket the k-th rank with [lo, hi], count the
//                     elements above/at the brackets, collect the strictly-inside band and
//                     bitonic-sort it (rows with n <= band cap are sorted whole);
//        fallback   — MSB-first 4x8-bit radix select with warp-aggregated histograms
//                     (degenerate samples, e.g. massive ties);
//   3. optional float64 boundary refinement: every element within tau of T is re-scored
//      in float64 from the original q / K rows (summing heads in reference order) and the
//      boundary is re-resolved on those exact scores with the lower-index tie rule;
//   4. index-ordered stream compaction (ballot-free block scan) writes the selected
//      indices ascending, which is the reference's canonical TopKSet order for free.
#pragma once

#include "common.cuh"

namespace hylra {

constexpr int kSelThreads = 1024;
constexpr int kBandCap = 8192;     // strictly-inside band capacity (floats)
constexpr int kRefineCap = 1024;   // float64 refinement candidates
constexpr int kCacheMax = 32768;   // rows up to this length are staged in shared memory

struct SelectParams {
  const float* scores;  // [slot][b][kh][row_stride]
  int32_t* idx;         // [slot][b][grp][k_stride]
  int32_t* info;        // [row][4] or null
  int* flags;
  const void* q;        // refinement inputs (null: refinement off)
  const void* k;
  int dtype;
  int64_t q_sl, q_sb, kv_sl, kv_sb, kv_sh;
  int B, Hkv, G, D, sel_group, n_groups;
  int n_valid, k_eff, k_stride, row_stride;
  int cache_row;
  float tau_rel;
  int layers[kMaxSlots];
};

// ----------------------------------------------------------------------------- helpers
__device__ __forceinline__ int block_sum_int(int v, int* red) {
  // red: >= 33 ints of shared scratch
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int x = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[32] = x;
  }
  __syncthreads();
  return red[32];
}
__device__ __forceinline__ float block_max_float(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    float x = (lane < (int)(blockDim.x >> 5)) ? red[lane] : -INFINITY;
    x = warp_max(x);
    if (lane == 0) red[32] = x;
  }
  __syncthreads();
  return red[32];
}

// Bitonic sort (descending) of P floats in shared memory, P a power of two.
__device__ void bitonic_desc_f32(float* a, int P) {
  for (int kk = 2; kk <= P; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const float x = a[i], y = a[ixj];
          const bool desc = (i & kk) == 0;
          if (desc ? (x < y) : (x > y)) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}
// Bitonic sort of (value desc, index asc) pairs; P a power of two.
__device__ void bitonic_desc_f64_idx(double* v, int* id, int P) {
  for (int kk = 2; kk <= P; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const double x = v[i], y = v[ixj];
          const int xi = id[i], yi = id[ixj];
          // "x before y" in the target order: larger value first, then smaller index
          const bool x_first = (x > y) || (x == y && xi < yi);
          const bool want_x_first = (i & kk) == 0;
          if (x_first != want_x_first) {
            v[i] = y;
            v[ixj] = x;
            id[i] = yi;
            id[ixj] = xi;
          }
        }
      }
      __syncthreads();
    }
  }
}
// Ascending bitonic sort of ints.
__device__ void bitonic_asc_i32(int* a, int P) {
  for (int kk = 2; kk <= P; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int x = a[i], y = a[ixj];
          const bool asc = (i & kk) == 0;
          if (asc ? (x > y) : (x < y)) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

struct RowReader {
  const float* base;  // score row of the group's first kv head
  int64_t hstride;
  int sg;
  const float* cache;
  __device__ __forceinline__ float load_raw(int n) const {
    float s = 0.f;
    for (int h = 0; h < sg; ++h) s += __ldg(base + h * hstride + n);
    return s;
  }
  __device__ __forceinline__ float operator()(int n) const {
    return cache ? cache[n] : load_raw(n);
  }
};

template <typename T>
__device__ __forceinline__ double elem_f64(const void* p, int64_t i) {
  return (double)to_f32(reinterpret_cast<const T*>(p)[i]);
}

// ----------------------------------------------------------------------------- kernel
__global__ void __launch_bounds__(kSelThreads, 1) topk_select_kernel(const SelectParams p) {
  extern __shared__ __align__(16) uint8_t sraw[];
  __shared__ int red[40];
  __shared__ float fred[40];
  __shared__ int s_misc[16];
  __shared__ unsigned s_hist[256];

  const int grp = blockIdx.x, b = blockIdx.y, slot = blockIdx.z;
  const int tid = threadIdx.x;
  const int n = p.n_valid;
  const int k = p.k_eff;
  const int row_id = (slot * p.B + b) * p.n_groups + grp;
  int32_t* out = p.idx + (int64_t)row_id * p.k_stride;

  // shared memory carve-up
  float* cache = nullptr;
  uint8_t* cur = sraw;
  if (p.cache_row) {
    cache = reinterpret_cast<float*>(cur);
    cur += ((n + 3) & ~3) * sizeof(float);
  }
  float* sample = reinterpret_cast<float*>(cur);  // 2048 floats
  cur += 2048 * sizeof(float);
  float* band = reinterpret_cast<float*>(cur);    // kBandCap floats; reused by refinement
  double* rv = reinterpret_cast<double*>(cur);    // kRefineCap doubles
  int* rid = reinterpret_cast<int*>(cur + kRefineCap * sizeof(double));
  int* chosen = rid + kRefineCap;

  RowReader rd;
  rd.base = p.scores + ((int64_t)(slot * p.B + b) * p.Hkv + grp * p.sel_group) * p.row_stride;
  rd.hstride = p.row_stride;
  rd.sg = p.sel_group;
  rd.cache = nullptr;

  // ---- 1. stage + stats
  float mabs = 0.f;
  int bad = 0;
  for (int i = tid; i < n; i += kSelThreads) {
    const float v = rd.load_raw(i);
    if (cache) cache[i] = v;
    if (!isfinite(v)) bad = 1;
    else mabs = fmaxf(mabs, fabsf(v));
  }
  mabs = block_max_float(mabs, fred);
  bad = block_sum_int(bad, red);
  if (bad && tid == 0) atomicOr(p.flags, 2);
  rd.cache = cache;

  if (k >= n) {
    for (int i = tid; i < n; i += kSelThreads) out[i] = i;
    if (p.info && tid == 0) {
      int32_t* inf = p.info + row_id * 4;
      inf[0] = k; inf[1] = 0; inf[2] = 0; inf[3] = 0;
    }
    return;
  }

  // ---- 2. exact k-th largest value T, with c_gt = #(v > T), c_eq = #(v == T)
  float T = 0.f;
  int c_gt = 0, c_eq = 0, mode = 0, band_n = 0;
  bool found = false;
  {
    float lo = -INFINITY, hi = INFINITY;
    if (n > kBandCap) {
      const int S = (n >= 65536) ? 2048 : 1024;
      for (int j = tid; j < S; j += kSelThreads) sample[j] = rd((int)(((int64_t)j * n) / S));
      __syncthreads();
      bitonic_desc_f32(sample, S);
      const double pr = (double)k / n;
      const double delta = 3.0 * sqrt(S * pr * (1.0 - pr)) + 2.0;
      const int hi_i = (int)floor(pr * S - delta);
      const int lo_i = (int)ceil(pr * S + delta);
      hi = (hi_i >= 0) ? sample[hi_i] : INFINITY;
      lo = (lo_i < S) ? sample[lo_i] : -INFINITY;
      __syncthreads();
    }
    if (tid == 0) s_misc[0] = 0;
    __syncthreads();
    int cgt = 0, ceqh = 0, ceql = 0;
    const int lane = tid & 31;
    for (int base = 0; base < n; base += kSelThreads) {
      const int i = base + tid;
      float v = 0.f;
      bool inb = false;
      if (i < n) {
        v = rd(i);
        cgt += (v > hi);
        ceqh += (v == hi);
        ceql += (v == lo) && (lo != hi);
        inb = (v > lo) && (v < hi);
      }
      const unsigned m = __ballot_sync(0xffffffffu, inb);
      if (m) {
        int wbase = 0;
        if (lane == 0) wbase = atomicAdd(&s_misc[0], __popc(m));
        wbase = __shfl_sync(0xffffffffu, wbase, 0);
        const int pos = wbase + __popc(m & ((1u << lane) - 1u));
        if (inb && pos < kBandCap) band[pos] = v;
      }
    }
    cgt = block_sum_int(cgt, red);
    ceqh = block_sum_int(ceqh, red);
    ceql = block_sum_int(ceql, red);
    const int nin = s_misc[0];
    band_n = nin;
    __syncthreads();
    if (nin <= kBandCap) {
      if (k <= cgt) {
        found = false;
      } else if (k <= cgt + ceqh) {
        T = hi; c_gt = cgt; c_eq = ceqh; found = true;
      } else if (k <= cgt + ceqh + nin) {
        const int r = k - cgt - ceqh;  // 1-based rank inside the band
        const int P = next_pow2(nin);
        for (int j = nin + tid; j < P; j += kSelThreads) band[j] = -INFINITY;
        __syncthreads();
        bitonic_desc_f32(band, P);
        T = band[r - 1];
        int above = 0, eq = 0;
        for (int j = tid; j < nin; j += kSelThreads) {
          above += band[j] > T;
          eq += band[j] == T;
        }
        above = block_sum_int(above, red);
        eq = block_sum_int(eq, red);
        c_gt = cgt + ceqh + above;
        c_eq = eq;
        found = true;
      } else if (lo != hi && k <= cgt + ceqh + nin + ceql) {
        T = lo; c_gt = cgt + ceqh + nin; c_eq = ceql; found = true;
      }
    }
  }
  if (!found) {
    // MSB-first radix select on order-preserving keys, descending rank k.
    mode = 1;
    uint32_t prefix = 0, mask = 0;
    int krem = k;
    int last_cnt = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int j = tid; j < 256; j += kSelThreads) s_hist[j] = 0;
      __syncthreads();
      for (int base = 0; base < n; base += kSelThreads) {
        const int i = base + tid;
        bool act = false;
        unsigned dig = 0;
        if (i < n) {
          const uint32_t key = float_key(rd(i));
          act = (key & mask) == prefix;
          dig = (key >> shift) & 255u;
        }
        const unsigned am = __ballot_sync(0xffffffffu, act);
        if (act) {
          const unsigned peers = __match_any_sync(am, dig);
          if ((threadIdx.x & 31) == (__ffs(peers) - 1)) atomicAdd(&s_hist[dig], __popc(peers));
        }
      }
      __syncthreads();
      if (tid == 0) {
        int acc = 0, d = 255;
        for (; d > 0; --d) {
          if (acc + (int)s_hist[d] >= krem) break;
          acc += s_hist[d];
        }
        s_misc[1] = d;
        s_misc[2] = acc;
        s_misc[3] = s_hist[d];
      }
      __syncthreads();
      const int d = s_misc[1];
      krem -= s_misc[2];
      last_cnt = s_misc[3];
      prefix |= (uint32_t)d << shift;
      mask |= 255u << shift;
      __syncthreads();
    }
    T = key_float(prefix);
    c_gt = k - krem;
    c_eq = last_cnt;
    found = true;
  }

  // ---- 3. optional float64 boundary refinement
  float gt_thr = T;       // "definitely selected" strictly above this
  int need = k - c_gt;    // lowest-index elements equal to T (mode B)
  bool refined = false;
  int n_cand = 0;
  if (p.q != nullptr) {
    const float tau = fmaxf(p.tau_rel * mabs, 1e-30f);
    const float lo_r = T - tau, hi_r = T + tau;
    if (tid == 0) s_misc[0] = 0;
    __syncthreads();
    int above = 0;
    const int lane = tid & 31;
    for (int base = 0; base < n; base += kSelThreads) {
      const int i = base + tid;
      bool inb = false;
      if (i < n) {
        const float v = rd(i);
        above += v > hi_r;
        inb = (v >= lo_r) && (v <= hi_r);
      }
      const unsigned m = __ballot_sync(0xffffffffu, inb);
      if (m) {
        int wbase = 0;
        if (lane == 0) wbase = atomicAdd(&s_misc[0], __popc(m));
        wbase = __shfl_sync(0xffffffffu, wbase, 0);
        const int pos = wbase + __popc(m & ((1u << lane) - 1u));
        if (inb && pos < kRefineCap) rid[pos] = i;
      }
    }
    above = block_sum_int(above, red);
    n_cand = s_misc[0];
    __syncthreads();
    if (n_cand <= kRefineCap) {
      // float64 re-score: agg = sum over (kv head in group, query head g) of (q . k) / sqrt(d)
      const int warp = tid >> 5;
      const int layer = p.layers[slot];
      const double sqd = sqrt((double)p.D);
      for (int c = warp; c < n_cand; c += kSelThreads / 32) {
        const int tok = rid[c];
        double agg = 0.0;
        for (int hh = 0; hh < p.sel_group; ++hh) {
          const int kh = grp * p.sel_group + hh;
          const int64_t koff = layer * p.kv_sl + b * p.kv_sb + kh * p.kv_sh + (int64_t)tok * p.D;
          for (int g = 0; g < p.G; ++g) {
            const int64_t qoff = layer * p.q_sl + b * p.q_sb + (int64_t)(kh * p.G + g) * p.D;
            double part = 0.0;
            for (int i = lane; i < p.D; i += 32) {
              if (p.dtype == 0)
                part += elem_f64<__nv_bfloat16>(p.q, qoff + i) * elem_f64<__nv_bfloat16>(p.k, koff + i);
              else
                part += elem_f64<float>(p.q, qoff + i) * elem_f64<float>(p.k, koff + i);
            }
            const double dot = warp_sum_f64(part);
            agg += dot / sqd;
          }
        }
        if (lane == 0) rv[c] = agg;
      }
      __syncthreads();
      const int P = next_pow2(max(n_cand, 1));
      for (int j = n_cand + tid; j < P; j += kSelThreads) {
        rv[j] = -INFINITY;
        rid[j] = 0x7fffffff;
      }
      __syncthreads();
      bitonic_desc_f64_idx(rv, rid, P);
      const int r = k - above;  // picks from the band
      for (int j = tid; j < P; j += kSelThreads) chosen[j] = (j < r) ? rid[j] : 0x7fffffff;
      __syncthreads();
      bitonic_asc_i32(chosen, P);
      gt_thr = hi_r;
      need = r;
      refined = true;
      n_cand = r;  // number of chosen band members (searched below)
    } else if (tid == 0) {
      atomicOr(p.flags, 4);
    }
    __syncthreads();
  }

  // ---- 4. index-ordered compaction. sel(i) = v > gt_thr || (eqflag(i) && eq_rank(i) < need)
  //      eqflag = (v == T) normally; after refinement = chosen band member.
  {
    const int lane = tid & 31, warp = tid >> 5;
    int run_gt = 0, run_eq = 0;
    const float lo_band = refined ? (T - fmaxf(p.tau_rel * mabs, 1e-30f)) : T;
    for (int base = 0; base < n; base += kSelThreads * 4) {
      int fl_gt[4], fl_eq[4];
      int cnt = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = base + tid * 4 + e;
        fl_gt[e] = 0;
        fl_eq[e] = 0;
        if (i < n) {
          const float v = rd(i);
          if (v > gt_thr) {
            fl_gt[e] = 1;
          } else if (!refined) {
            fl_eq[e] = (v == T);
          } else if (v >= lo_band) {
            // binary search in the ascending chosen list
            int lo = 0, hi = n_cand;
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (chosen[mid] < i) lo = mid + 1;
              else hi = mid;
            }
            fl_eq[e] = (lo < n_cand && chosen[lo] == i);
          }
        }
        cnt += fl_gt[e] | (fl_eq[e] << 16);
      }
      // block exclusive scan of packed (gt | eq<<16) counts
      int x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      __syncthreads();
      if (lane == 31) red[warp] = x;
      __syncthreads();
      if (warp == 0) {
        int w = red[lane];
        int ws = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, ws, o);
          if (lane >= o) ws += y;
        }
        red[lane] = ws - w;  // exclusive warp offsets
        if (lane == 31) red[32] = ws;
      }
      __syncthreads();
      int pre = red[warp] + x - cnt;  // exclusive prefix for this thread
      int gt_before = run_gt + (pre & 0xffff);
      int eq_before = run_eq + (pre >> 16);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = base + tid * 4 + e;
        const bool sel = fl_gt[e] || (fl_eq[e] && eq_before < need);
        if (sel) {
          const int pos = gt_before + min(eq_before, need);
          if (pos < k) out[pos] = i;
        }
        gt_before += fl_gt[e];
        eq_before += fl_eq[e];
      }
      const int tot = red[32];
      run_gt += tot & 0xffff;
      run_eq += tot >> 16;
    }
  }
  if (p.info && tid == 0) {
    int32_t* inf = p.info + row_id * 4;
    inf[0] = k;
    inf[1] = refined ? n_cand : -1;
    inf[2] = mode + (refined ? 2 : 0);
    inf[3] = band_n;
  }
}

}  // namespace hylra
