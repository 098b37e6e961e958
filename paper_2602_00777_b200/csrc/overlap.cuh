// overlap.cuh — pairwise top-k selection overlap counts for the layer-similarity profile.
//
// Reference: pkg/src/layerreuse/profiling.py:38-47 overlap_ratio (|a & b| / k) and
// profiling.py:126-145 build_similarity_matrix (every pair i < j of every step). The GPU
// produces the exact integer numerators |S_i & S_j|; the host applies the reference's
// float64 fold (count / k, mean over steps, triu = 0, diag = 1) so the matrix, its sha256
// and the DP policy are bit-identical.
//
// One CTA per (row, step, token chunk): each layer's sorted set contributes only its tokens
// inside the chunk (found by binary search, one warp per layer), scattered into a
// shared-memory bitmap of the chunk; every pair (i <= j) is reduced with popc(a & b) over the
// chunk's words and added to the (zeroed) counts with integer atomics — exact, so the sum over
// chunks is the same integer whatever the order. Chunks are sized so the grid fills the GPU
// (round 1 ran one CTA per (row, step) over every chunk: 32 CTAs, 135 us for config 5's
// profiling pass).
#pragma once

#include "common.cuh"

namespace hylra {

constexpr int kOvThreads = 512;

__device__ __forceinline__ int ov_lower_bound(const int32_t* s, int n, int key) {
  int a = 0, z = n;
  while (a < z) {
    const int m = (a + z) >> 1;
    if (__ldg(s + m) < key) a = m + 1;
    else z = m;
  }
  return a;
}

__global__ void __launch_bounds__(kOvThreads)
    overlap_counts_kernel(const int32_t* __restrict__ idx, int layers, int rows, int k,
                          int k_stride, int n_tokens, int chunk_bits, int32_t* counts) {
  extern __shared__ __align__(16) uint32_t bm[];  // [layers][chunk_bits/32]
  const int r = blockIdx.x, t = blockIdx.y;
  const int c0 = blockIdx.z * chunk_bits;
  const int W = chunk_bits >> 5;
  const int n_pairs = layers * (layers + 1) / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < layers * W; i += kOvThreads) bm[i] = 0u;
  __syncthreads();
  for (int l = warp; l < layers; l += kOvThreads / 32) {
    const int32_t* s = idx + ((int64_t)(t * layers + l) * rows + r) * k_stride;
    int lo = 0, hi = 0;
    if (lane == 0) {
      lo = ov_lower_bound(s, k, c0);
      hi = lo + ov_lower_bound(s + lo, k - lo, c0 + chunk_bits);
    }
    lo = __shfl_sync(0xffffffffu, lo, 0);
    hi = __shfl_sync(0xffffffffu, hi, 0);
    for (int e = lo + lane; e < hi; e += 32) {
      const int tok = __ldg(s + e) - c0;
      atomicOr(bm + l * W + (tok >> 5), 1u << (tok & 31));
    }
  }
  __syncthreads();
  int32_t* outc = counts + (int64_t)(t * rows + r) * layers * layers;
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
    if (lane == 0 && acc) {
      atomicAdd(outc + j * layers + i, acc);
      if (i != j) atomicAdd(outc + i * layers + j, acc);
    }
  }
}

}  // namespace hylra
