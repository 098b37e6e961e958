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

// grid (groups, B, slots); scores [slot][b][kh][row_stride] -> bscores [slot][b][grp][nb_stride]
__global__ void __launch_bounds__(kPoolThreads)
    block_pool_kernel(const float* __restrict__ scores, int B, int Hkv, int sel_group,
                      int row_stride, int n_tokens, int block_size, float* __restrict__ bscores,
                      int nb_stride) {
  const int grp = blockIdx.x, b = blockIdx.y, slot = blockIdx.z;
  const int n_groups = Hkv / sel_group;
  const float* base = scores + ((int64_t)(slot * B + b) * Hkv + grp * sel_group) * row_stride;
  float* outr = bscores + ((int64_t)(slot * B + b) * n_groups + grp) * nb_stride;
  const int nb = (n_tokens + block_size - 1) / block_size;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // one warp per block: lanes stride over the block's tokens (coalesced), then max-reduce
  for (int blk = warp; blk < nb; blk += kPoolThreads / 32) {
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
