// blocks.cuh — block-level selection support (paper §3.5 "adaptation to block-level
// sparsity"; reference engine.py:212-286 hybrid_decode_blocks).
//
//   block_pool_kernel   : block score = max over the block's tokens of the head-summed
//                         selection score (attention.py:287-295 block_max_of_logits); the
//                         final block may be narrower than block_size.
//   block_expand_kernel : selected blocks (ascending) -> ascending token coverage and its
//                         length (attention.py:166-182 BlockSet.token_coverage), which the
//                         REUSE kernel consumes with per-row counts.
// Block selection itself is the token SELECT kernel run over the pooled rows (same
// lower-index tie rule: ties go to the lower block), with a block-aware float64 refinement.
#pragma once

#include "common.cuh"

namespace hylra {

constexpr int kPoolThreads = 256;

// grid (groups * B * slots, ceil(n_blocks / 8)); one warp per block, coalesced loads:
// scores [slot][b][kh][row_stride] -> bscores [slot][b][grp][nb_stride]
__global__ void __launch_bounds__(kPoolThreads)
    block_pool_kernel(const float* __restrict__ scores, int B, int Hkv, int sel_group,
                      int row_stride, int n_tokens, int block_size, float* __restrict__ bscores,
                      int nb_stride) {
  const int n_groups = Hkv / sel_group;
  const int row = blockIdx.x;  // (slot * B + b) * n_groups + grp
  const int grp = row % n_groups, sb = row / n_groups;
  const float* base = scores + ((int64_t)sb * Hkv + grp * sel_group) * row_stride;
  float* outr = bscores + (int64_t)row * nb_stride;
  const int nb = (n_tokens + block_size - 1) / block_size;
  const int lane = threadIdx.x & 31;
  const int blk = blockIdx.y * (kPoolThreads / 32) + (threadIdx.x >> 5);
  if (blk >= nb) return;
  const int t0 = blk * block_size, t1 = min(n_tokens, t0 + block_size);
  float m = -INFINITY;
  for (int t = t0 + lane; t < t1; t += 32) {
    float s = __ldg(base + t);
    for (int h = 1; h < sel_group; ++h) s += __ldg(base + (int64_t)h * row_stride + t);
    m = fmaxf(m, s);
  }
  m = warp_max(m);
  if (lane == 0) outr[blk] = m;
}

// Vectorised pooling for block_size = 4 * W, W a power of two <= 32: each lane owns a
// float4 of tokens, W lanes cover one block (a warp is block-aligned because W | 32), four
// float4 loads in flight per thread. grid (groups * B * slots, ceil(n / (4 * 4 * 256))).
constexpr int kPoolVec = 4;
template <int W>
__global__ void __launch_bounds__(kPoolThreads)
    block_pool_vec_kernel(const float* __restrict__ scores, int Hkv, int sel_group,
                          int row_stride, int n_tokens, float* __restrict__ bscores,
                          int nb_stride) {
  const int n_groups = Hkv / sel_group;
  const int row = blockIdx.x;
  const int grp = row % n_groups, sb = row / n_groups;
  const float* base = scores + ((int64_t)sb * Hkv + grp * sel_group) * row_stride;
  float* outr = bscores + (int64_t)row * nb_stride;
  const int j0 = blockIdx.y * (kPoolThreads * kPoolVec) + threadIdx.x;  // float4 index
  float4 v[kPoolVec];
#pragma unroll
  for (int u = 0; u < kPoolVec; ++u) {
    const int j = j0 + u * kPoolThreads;
    v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (4 * j < n_tokens) {
      for (int h = 0; h < sel_group; ++h) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(base + (int64_t)h * row_stride) + j);
        v[u].x += x.x;
        v[u].y += x.y;
        v[u].z += x.z;
        v[u].w += x.w;
      }
    }
  }
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < kPoolVec; ++u) {
    const int j = j0 + u * kPoolThreads;
    const int t = 4 * j;
    float m = -INFINITY;
    if (t < n_tokens) m = v[u].x;
    if (t + 1 < n_tokens) m = fmaxf(m, v[u].y);
    if (t + 2 < n_tokens) m = fmaxf(m, v[u].z);
    if (t + 3 < n_tokens) m = fmaxf(m, v[u].w);
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((lane & (W - 1)) == 0 && t < n_tokens) outr[t / (4 * W)] = m;
  }
}

// grid (rows): blocks [row][bk_stride] (ascending, bb valid) -> tokens [row][tok_stride],
// counts[row] = number of covered tokens (< n_tokens).
__global__ void __launch_bounds__(kPoolThreads)
    block_expand_kernel(const int32_t* __restrict__ blocks, int bk_stride, int bb,
                        int block_size, int n_tokens, int32_t* __restrict__ tokens,
                        int tok_stride, int32_t* __restrict__ counts) {
  const int row = blockIdx.x;
  const int32_t* br = blocks + (int64_t)row * bk_stride;
  int32_t* tr = tokens + (int64_t)row * tok_stride;
  // every block but possibly the last selected one is full width (ascending order)
  for (int e = threadIdx.x; e < bb * block_size; e += kPoolThreads) {
    const int j = e / block_size, o = e % block_size;
    const int tok = br[j] * block_size + o;
    tr[e] = (tok < n_tokens) ? tok : -1;
  }
  if (threadIdx.x == 0) {
    const int last = br[bb - 1];
    counts[row] = (bb - 1) * block_size + min(block_size, n_tokens - last * block_size);
  }
}

}  // namespace hylra

namespace hylra {

// Sink / recent augmentation of REUSE selections (engine.py:122-126 _augment_selection):
// out = sorted(sel | [0, sinks) | [n - recent, n)). grid (rows); idx rows are ascending.
__global__ void __launch_bounds__(kPoolThreads)
    augment_kernel(const int32_t* __restrict__ idx, int k_stride, int k_eff, int n, int sinks,
                   int recent, int32_t* __restrict__ out, int out_stride,
                   int32_t* __restrict__ counts) {
  const int row = blockIdx.x;
  const int32_t* src = idx + (int64_t)row * k_stride;
  int32_t* dst = out + (int64_t)row * out_stride;
  const int s = min(sinks, n);
  const int u0 = max(n - recent, 0);
  if (u0 <= s) {  // the two ranges already cover every token
    for (int i = threadIdx.x; i < n; i += kPoolThreads) dst[i] = i;
    if (threadIdx.x == 0) counts[row] = n;
    return;
  }
  // selected tokens strictly between the ranges: [lower_bound(s), lower_bound(u0))
  __shared__ int s_lb[2];
  if (threadIdx.x < 2) {
    const int key = threadIdx.x == 0 ? s : u0;
    int a = 0, z = k_eff;
    while (a < z) {
      const int m = (a + z) >> 1;
      if (src[m] < key) a = m + 1;
      else z = m;
    }
    s_lb[threadIdx.x] = a;
  }
  __syncthreads();
  const int mid0 = s_lb[0], mid = s_lb[1] - s_lb[0];
  for (int i = threadIdx.x; i < s; i += kPoolThreads) dst[i] = i;
  for (int i = threadIdx.x; i < mid; i += kPoolThreads) dst[s + i] = src[mid0 + i];
  for (int i = threadIdx.x; i < n - u0; i += kPoolThreads) dst[s + mid + i] = u0 + i;
  if (threadIdx.x == 0) counts[row] = s + mid + (n - u0);
}

}  // namespace hylra
