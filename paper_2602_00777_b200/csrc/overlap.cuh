// overlap.cuh — pairwise top-k selection overlap counts for the layer-similarity profile.
//
// Reference: pkg/src/layerreuse/profiling.py:38-47 overlap_ratio (|a & b| / k) and
// profiling.py:126-145 build_similarity_matrix (every pair i < j of every step). The GPU
// produces the exact integer numerators |S_i & S_j|; the host applies the reference's
// float64 fold (count / k, mean over steps, triu = 0, diag = 1) so the matrix, its sha256
// and the DP policy are bit-identical.
//
// One CTA per (row, step). The token axis is processed in chunks; each layer's index
// set is scattered into a shared-memory bitmap of the chunk and every pair (i <= j) is
// reduced with popc(a & b) over the chunk's words.
#pragma once

#include "common.cuh"

namespace hylra {

constexpr int kOvThreads = 512;

__global__ void __launch_bounds__(kOvThreads)
    overlap_counts_kernel(const int32_t* __restrict__ idx, int layers, int rows, int k,
                          int k_stride, int n_tokens, int chunk_bits, int32_t* counts) {
  extern __shared__ __align__(16) uint32_t bm[];  // [layers][chunk_bits/32] then [pairs]
  const int r = blockIdx.x, t = blockIdx.y;
  const int W = chunk_bits >> 5;
  const int n_pairs = layers * (layers + 1) / 2;
  int* pc = reinterpret_cast<int*>(bm + layers * W);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < n_pairs; i += kOvThreads) pc[i] = 0;

  for (int c0 = 0; c0 < n_tokens; c0 += chunk_bits) {
    for (int i = tid; i < layers * W; i += kOvThreads) bm[i] = 0u;
    __syncthreads();
    for (int l = 0; l < layers; ++l) {
      const int32_t* s = idx + ((int64_t)(t * layers + l) * rows + r) * k_stride;
      for (int e = tid; e < k; e += kOvThreads) {
        const int tok = __ldg(s + e) - c0;
        if (tok >= 0 && tok < chunk_bits) atomicOr(bm + l * W + (tok >> 5), 1u << (tok & 31));
      }
    }
    __syncthreads();
    for (int pr = warp; pr < n_pairs; pr += kOvThreads / 32) {
      // pair index -> (j, i) with i <= j, row-major lower triangle
      int j = (int)((sqrtf(8.f * pr + 1.f) - 1.f) * 0.5f);
      while ((j + 1) * (j + 2) / 2 <= pr) ++j;
      while (j * (j + 1) / 2 > pr) --j;
      const int i = pr - j * (j + 1) / 2;
      const uint32_t* a = bm + i * W;
      const uint32_t* bb = bm + j * W;
      int acc = 0;
      for (int w = lane; w < W; w += 32) acc += __popc(a[w] & bb[w]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) pc[pr] += acc;
    }
    __syncthreads();
  }
  int32_t* outc = counts + (int64_t)(t * rows + r) * layers * layers;
  for (int pr = tid; pr < n_pairs; pr += kOvThreads) {
    int j = (int)((sqrtf(8.f * pr + 1.f) - 1.f) * 0.5f);
    while ((j + 1) * (j + 2) / 2 <= pr) ++j;
    while (j * (j + 1) / 2 > pr) --j;
    const int i = pr - j * (j + 1) / 2;
    outc[j * layers + i] = pc[pr];
    outc[i * layers + j] = pc[pr];
  }
}

}  // namespace hylra
