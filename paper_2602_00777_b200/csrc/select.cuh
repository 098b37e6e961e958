// select.cuh — exact top-k selection over per-(slot, b, group) score rows.
//
// Reference: pkg/src/layerreuse/attention.py:264-275 topk_of_logits — the min(budget, N)
// highest logits, ties won by the LOWER index (stable argsort of -logits), returned
// ascending; engine.py:169 clamps the budget per step; engine.py:177-183 scores are the
// head-order sum of per-head scaled logits.
//
// One 1024-thread CTA per row, no global atomics:
//   A. sample 1024 scores (strided) and bitonic-sort them in registers/shuffles (shared
//      memory only for the 15 exchange stages with stride >= 32) -> brackets [lo, hi]
//      around the k-th rank;
//   B. ONE vectorised pass over the row: stage it in shared memory (rows <= 32K),
//      reduce max|s| and the non-finite flag, count the elements above / at the brackets
//      and collect the strictly-inside band (warp-aggregated appends);
//   C. exact k-th largest value T = radix select (4 x 8 bit, warp-aggregated shared
//      histograms) inside the band; fallback = the same radix select over the whole row
//      (degenerate samples, e.g. massive ties);
//   D. optional float64 boundary refinement: every element within tau of T is re-scored
//      in float64 from the original q / K rows (heads summed in reference order) and the
//      boundary is re-resolved on those scores with the lower-index tie rule;
//   E. index-ordered stream compaction (block scan of packed counts) writes the selected
//      indices ascending — the reference's canonical TopKSet order.
#pragma once

#include "common.cuh"

namespace hylra {

constexpr int kSelThreads = 1024;
constexpr int kSample = 1024;
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

// Warp-aggregated append: every thread contributes `cnt` items; returns the thread's
// first slot. One shared atomic per warp.
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

// Descending bitonic sort of one float per thread (blockDim = 1024); shuffles for
// strides < 32, shared memory for the rest.
__device__ float bitonic1024_desc(float x, float* xchg) {
  const int tid = threadIdx.x;
  for (int kk = 2; kk <= kSelThreads; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      float y;
      if (j >= 32) {
        xchg[tid] = x;
        __syncthreads();
        y = xchg[tid ^ j];
        __syncthreads();
      } else {
        y = __shfl_xor_sync(0xffffffffu, x, j);
      }
      const bool desc = (tid & kk) == 0;
      const bool lower = (tid & j) == 0;
      x = (lower == desc) ? fmaxf(x, y) : fminf(x, y);
    }
  }
  return x;
}

// Bitonic sort of (value desc, index asc) pairs in shared memory; P a power of two.
__device__ void bitonic_desc_f64_idx(double* v, int* id, int P) {
  for (int kk = 2; kk <= P; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const double x = v[i], y = v[ixj];
          const int xi = id[i], yi = id[ixj];
          const bool x_first = (x > y) || (x == y && xi < yi);
          const bool want_x_first = (i & kk) == 0;
          if (x_first != want_x_first) {
            v[i] = y; v[ixj] = x; id[i] = yi; id[ixj] = xi;
          }
        }
      }
      __syncthreads();
    }
  }
}
// Ascending bitonic sort of ints in shared memory; P a power of two.
__device__ void bitonic_asc_i32(int* a, int P) {
  for (int kk = 2; kk <= P; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int x = a[i], y = a[ixj];
          const bool asc = (i & kk) == 0;
          if (asc ? (x > y) : (x < y)) { a[i] = y; a[ixj] = x; }
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
  int64_t hstride;    // elements between the group's kv-head rows
  int sg;
  int n;
  const float* cache;
  __device__ __forceinline__ float load_raw(int i) const {
    float s = __ldg(base + i);
    for (int h = 1; h < sg; ++h) s += __ldg(base + h * hstride + i);
    return s;
  }
  __device__ __forceinline__ float4 load4_raw(int i4) const {
    float4 s = __ldg(reinterpret_cast<const float4*>(base) + i4);
    for (int h = 1; h < sg; ++h) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(base + h * hstride) + i4);
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    return s;
  }
  __device__ __forceinline__ float operator()(int i) const { return cache ? cache[i] : load_raw(i); }
  __device__ __forceinline__ float4 get4(int i4) const {
    return cache ? reinterpret_cast<const float4*>(cache)[i4] : load4_raw(i4);
  }
};

__device__ __forceinline__ float f4at(const float4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

template <typename T>
__device__ __forceinline__ double elem_f64(const void* p, int64_t i) {
  return (double)to_f32(reinterpret_cast<const T*>(p)[i]);
}

// Exact rank-`rank` (1-based, descending) element of a set by MSB-first 4 x 8-bit radix
// select on order-preserving keys. `get(j)` for j < count; returns T, #greater, #equal.
template <typename Get>
__device__ void radix_select_desc(const Get& get, int count, int rank, unsigned* hist,
                                  int* misc, float* T_out, int* gt_out, int* eq_out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t prefix = 0, mask = 0;
  int krem = rank, last = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    if (tid < 256) hist[tid] = 0;
    __syncthreads();
    for (int base = 0; base < count; base += kSelThreads) {
      const int j = base + tid;
      bool act = false;
      unsigned dig = 0;
      if (j < count) {
        const uint32_t key = float_key(get(j));
        act = (key & mask) == prefix;
        dig = (key >> shift) & 255u;
      }
      const unsigned am = __ballot_sync(0xffffffffu, act);
      if (act) {
        const unsigned peers = __match_any_sync(am, dig);
        if (lane == __ffs(peers) - 1) atomicAdd(hist + dig, (unsigned)__popc(peers));
      }
    }
    __syncthreads();
    if (warp == 0) {
      int c[8], s = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        c[u] = (int)hist[255 - 8 * lane - u];
        s += c[u];
      }
      int incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int excl = incl - s;
      const unsigned m = __ballot_sync(0xffffffffu, excl < krem && krem <= incl);
      if (lane == (m ? __ffs(m) - 1 : 31)) {
        int acc = excl, d = 255 - 8 * lane - 7, cnt = c[7];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (acc + c[u] >= krem) { d = 255 - 8 * lane - u; cnt = c[u]; break; }
          acc += c[u];
        }
        misc[8] = d;
        misc[9] = acc;
        misc[10] = cnt;
      }
    }
    __syncthreads();
    const int d = misc[8];
    krem -= misc[9];
    last = misc[10];
    prefix |= (uint32_t)d << shift;
    mask |= 255u << shift;
    __syncthreads();
  }
  *T_out = key_float(prefix);
  *gt_out = rank - krem;
  *eq_out = last;
}

// ----------------------------------------------------------------------------- kernel
__global__ void __launch_bounds__(kSelThreads, 1) topk_select_kernel(const SelectParams p) {
  extern __shared__ __align__(16) uint8_t sraw[];
  __shared__ int red[40];
  __shared__ float fred[40];
  __shared__ int s_misc[16];
  __shared__ unsigned s_hist[256];
  __shared__ float s_xchg[kSelThreads];

  const int grp = blockIdx.x, b = blockIdx.y, slot = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31;
  const int n = p.n_valid;
  const int k = p.k_eff;
  const int n4 = (n + 3) >> 2;
  const int row_id = (slot * p.B + b) * p.n_groups + grp;
  int32_t* out = p.idx + (int64_t)row_id * p.k_stride;

  float* cache = nullptr;
  uint8_t* cur = sraw;
  if (p.cache_row) {
    cache = reinterpret_cast<float*>(cur);
    cur += (size_t)n4 * 16;
  }
  float* band = reinterpret_cast<float*>(cur);    // kBandCap floats; reused by refinement
  double* rv = reinterpret_cast<double*>(cur);    // kRefineCap doubles
  int* rid = reinterpret_cast<int*>(cur + kRefineCap * sizeof(double));
  int* chosen = rid + kRefineCap;

  RowReader rd;
  rd.base = p.scores + ((int64_t)(slot * p.B + b) * p.Hkv + grp * p.sel_group) * p.row_stride;
  rd.hstride = p.row_stride;
  rd.sg = p.sel_group;
  rd.n = n;
  rd.cache = nullptr;

  // ---- A. brackets from a sorted sample
  float lo = -INFINITY, hi = INFINITY;
  if (n > kBandCap && k < n) {
    float x = rd.load_raw((int)(((int64_t)tid * n) / kSample));
    x = bitonic1024_desc(x, s_xchg);
    s_xchg[tid] = x;
    __syncthreads();
    const double pr = (double)k / n;
    const double delta = 3.0 * sqrt(kSample * pr * (1.0 - pr)) + 2.0;
    const int hi_i = (int)floor(pr * kSample - delta);
    const int lo_i = (int)ceil(pr * kSample + delta);
    hi = (hi_i >= 0) ? s_xchg[hi_i] : INFINITY;
    lo = (lo_i < kSample) ? s_xchg[lo_i] : -INFINITY;
    __syncthreads();
  }

  // ---- B. one pass: stage, stats, bracket counts, band collection
  if (tid == 0) s_misc[0] = 0;
  __syncthreads();
  float mabs = 0.f;
  int bad = 0, cgt = 0, ceqh = 0, ceql = 0;
  constexpr int U = 4;
  for (int base4 = 0; base4 < n4; base4 += kSelThreads * U) {
    float4 vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i4 = base4 + u * kSelThreads + tid;
      vv[u] = (i4 < n4) ? rd.load4_raw(i4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    int nb = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i4 = base4 + u * kSelThreads + tid;
      if (i4 < n4 && cache) reinterpret_cast<float4*>(cache)[i4] = vv[u];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = 4 * i4 + c;
        if (i4 < n4 && i < n) {
          const float v = f4at(vv[u], c);
          if (!isfinite(v)) bad = 1;
          else mabs = fmaxf(mabs, fabsf(v));
          cgt += v > hi;
          ceqh += v == hi;
          ceql += (v == lo) && (lo != hi);
          nb += (v > lo) && (v < hi);
        }
      }
    }
    int pos = warp_append(nb, &s_misc[0]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i4 = base4 + u * kSelThreads + tid;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = 4 * i4 + c;
        if (i4 < n4 && i < n) {
          const float v = f4at(vv[u], c);
          if ((v > lo) && (v < hi)) {
            if (pos < kBandCap) band[pos] = v;
            ++pos;
          }
        }
      }
    }
  }
  mabs = block_max_float(mabs, fred);
  bad = block_sum_int(bad, red);
  cgt = block_sum_int(cgt, red);
  ceqh = block_sum_int(ceqh, red);
  ceql = block_sum_int(ceql, red);
  if (bad && tid == 0) atomicOr(p.flags, 2);
  rd.cache = cache;
  const int nin = s_misc[0];
  __syncthreads();

  if (k >= n) {
    for (int i = tid; i < n; i += kSelThreads) out[i] = i;
    if (p.info && tid == 0) {
      int32_t* inf = p.info + row_id * 4;
      inf[0] = k; inf[1] = 0; inf[2] = 0; inf[3] = 0;
    }
    return;
  }

  // ---- C. exact k-th largest value T with c_gt = #(v > T)
  float T = 0.f;
  int c_gt = 0, c_eq = 0, mode = 0;
  bool found = false;
  if (nin <= kBandCap) {
    if (k <= cgt) {
      found = false;
    } else if (k <= cgt + ceqh) {
      T = hi; c_gt = cgt; c_eq = ceqh; found = true;
    } else if (k <= cgt + ceqh + nin) {
      int above = 0;
      auto getb = [&](int j) { return band[j]; };
      radix_select_desc(getb, nin, k - cgt - ceqh, s_hist, s_misc, &T, &above, &c_eq);
      c_gt = cgt + ceqh + above;
      found = true;
    } else if (lo != hi && k <= cgt + ceqh + nin + ceql) {
      T = lo; c_gt = cgt + ceqh + nin; c_eq = ceql; found = true;
    }
  }
  if (!found) {
    mode = 1;
    radix_select_desc(rd, n, k, s_hist, s_misc, &T, &c_gt, &c_eq);
  }

  // ---- D. optional float64 boundary refinement
  float gt_thr = T;     // "definitely selected" strictly above this
  int need = k - c_gt;  // lowest-index elements equal to T (unrefined)
  bool refined = false;
  int n_cand = 0;
  const float tau = fmaxf(p.tau_rel * mabs, 1e-30f);
  const float lo_r = T - tau, hi_r = T + tau;
  if (p.q != nullptr) {
    if (tid == 0) s_misc[0] = 0;
    __syncthreads();
    int above = 0;
    for (int base4 = 0; base4 < n4; base4 += kSelThreads) {
      const int i4 = base4 + tid;
      float4 vv = make_float4(0.f, 0.f, 0.f, 0.f);
      int nb = 0;
      if (i4 < n4) {
        vv = rd.get4(i4);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (4 * i4 + c < n) {
            const float v = f4at(vv, c);
            above += v > hi_r;
            nb += (v >= lo_r) && (v <= hi_r);
          }
        }
      }
      int pos = warp_append(nb, &s_misc[0]);
      if (nb) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int i = 4 * i4 + c;
          const float v = f4at(vv, c);
          if (i < n && (v >= lo_r) && (v <= hi_r)) {
            if (pos < kRefineCap) rid[pos] = i;
            ++pos;
          }
        }
      }
    }
    above = block_sum_int(above, red);
    n_cand = s_misc[0];
    __syncthreads();
    if (n_cand <= kRefineCap) {
      // float64 re-score: agg = sum over (kv head of the group, query head g) of q.k/sqrt(d)
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
            agg += warp_sum_f64(part) / sqd;
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
      n_cand = r;
    } else if (tid == 0) {
      atomicOr(p.flags, 4);
    }
    __syncthreads();
  }

  // ---- E. index-ordered compaction: sel(i) = v > gt_thr || (eq(i) && eq_rank(i) < need)
  {
    const int warp = tid >> 5;
    int run_gt = 0, run_eq = 0;
    for (int base4 = 0; base4 < n4; base4 += kSelThreads) {
      const int i4 = base4 + tid;
      int fl_gt[4], fl_eq[4];
      int cnt = 0;
      float4 vv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i4 < n4) vv = rd.get4(i4);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = 4 * i4 + c;
        fl_gt[c] = 0;
        fl_eq[c] = 0;
        if (i4 < n4 && i < n) {
          const float v = f4at(vv, c);
          if (v > gt_thr) {
            fl_gt[c] = 1;
          } else if (!refined) {
            fl_eq[c] = (v == T);
          } else if (v >= lo_r) {
            int a = 0, z = n_cand;
            while (a < z) {
              const int mid = (a + z) >> 1;
              if (chosen[mid] < i) a = mid + 1;
              else z = mid;
            }
            fl_eq[c] = (a < n_cand && chosen[a] == i);
          }
        }
        cnt += fl_gt[c] | (fl_eq[c] << 16);
      }
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
        const int w = red[lane];
        int ws = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, ws, o);
          if (lane >= o) ws += y;
        }
        red[lane] = ws - w;
        if (lane == 31) red[32] = ws;
      }
      __syncthreads();
      const int pre = red[warp] + x - cnt;
      int gt_before = run_gt + (pre & 0xffff);
      int eq_before = run_eq + (pre >> 16);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const bool sel = fl_gt[c] || (fl_eq[c] && eq_before < need);
        if (sel) {
          const int pos = gt_before + min(eq_before, need);
          if (pos < k) out[pos] = 4 * i4 + c;
        }
        gt_before += fl_gt[c];
        eq_before += fl_eq[c];
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
    inf[3] = nin;
  }
}

}  // namespace hylra
