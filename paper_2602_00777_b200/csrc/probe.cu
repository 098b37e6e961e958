// probe.cu — measurement-only microbenchmark (libhylra_probe.so, not part of the product
// ABI): the HBM ceiling of the REUSE access pattern.
//
// gather_probe_kernel reads exactly the K and V rows a REUSE launch reads — for every
// (layer, b, kv-head) pair the rows idx[src][b][kh][0..k) of that pair's cache block — with
// nothing else to do: indices staged in shared memory, 16 lanes per 256-byte row (16-byte
// loads), 8 loads of K and of V in flight per lane, an XOR fold to keep the loads live. Its bytes / time is the gather roofline the
// REUSE kernel's achieved GB/s is judged against (bench.py "reuse_gather_peak_gbs").
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

namespace {

struct ProbeParams {
  const uint8_t* k;
  const uint8_t* v;
  const int32_t* idx;
  int64_t kv_sl, kv_sb, kv_sh;  // bytes
  int row_bytes;                // d * element size (multiple of 16, <= 512)
  int B, Hkv, k_rows, k_stride;
  int n_layers;
  int layers[64];
  int src_slot[64];
  uint32_t* sink;
};

constexpr int kThreads = 256;
constexpr int kUnroll = 8;
constexpr int kMaxStage = 4096;  // indices of one CTA's row range staged in shared memory

// grid (splits, pairs): the CTA stages its index range in shared memory (one coalesced
// pass), then its warps stream the rows: per iteration a warp has kUnroll loads of K and V
// in flight per lane (kUnroll * 32 / chunks rows).
__global__ void __launch_bounds__(kThreads) gather_probe_kernel(const ProbeParams p) {
  __shared__ int32_t sidx[kMaxStage];
  const int chunks = p.row_bytes / 16;       // 16-B chunks per row
  const int rpo = 32 / chunks;               // rows one warp instruction covers
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / chunks, ch = lane % chunks;
  const int pair = blockIdx.y;
  const int kh = pair % p.Hkv, b = (pair / p.Hkv) % p.B, slot = pair / (p.Hkv * p.B);
  const int per = (p.k_rows + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(p.k_rows, r0 + per);
  const int n = max(0, min(r1 - r0, kMaxStage));
  const int32_t* ib = p.idx + ((int64_t)(p.src_slot[slot] * p.B + b) * p.Hkv + kh) * p.k_stride + r0;
  for (int j = threadIdx.x; j < n; j += kThreads) sidx[j] = __ldg(ib + j);
  __syncthreads();
  const int l = p.layers[slot];
  const uint8_t* kb = p.k + l * p.kv_sl + b * p.kv_sb + kh * p.kv_sh;
  const uint8_t* vb = p.v + l * p.kv_sl + b * p.kv_sb + kh * p.kv_sh;
  uint32_t acc = 0;
  const int step = rpo * kUnroll;
  for (int base = warp * step; base < n; base += (kThreads / 32) * step) {
    uint4 kv[kUnroll], vv[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int r = base + u * rpo + sub;
      kv[u] = vv[u] = make_uint4(0, 0, 0, 0);
      if (r < n) {
        const int64_t off = (int64_t)sidx[r] * p.row_bytes;
        kv[u] = __ldcs(reinterpret_cast<const uint4*>(kb + off) + ch);
        vv[u] = __ldcs(reinterpret_cast<const uint4*>(vb + off) + ch);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      acc ^= kv[u].x ^ kv[u].y ^ kv[u].z ^ kv[u].w ^ vv[u].x ^ vv[u].y ^ vv[u].z ^ vv[u].w;
  }
  if (acc == 0x9e3779b9u) p.sink[0] = acc;  // practically never: keeps the loads live
}

}  // namespace

extern "C" int hylra_probe_gather(const void* k, const void* v, const int32_t* idx,
                                  int64_t kv_sl, int64_t kv_sb, int64_t kv_sh, int row_bytes,
                                  int B, int Hkv, int k_rows, int k_stride, int n_layers,
                                  const int32_t* layers, const int32_t* src_slots, void* sink,
                                  int blocks_per_sm, void* stream) {
  if (row_bytes % 16 != 0 || row_bytes > 512 || n_layers < 1 || n_layers > 64) return 1;
  ProbeParams p{};
  p.k = static_cast<const uint8_t*>(k);
  p.v = static_cast<const uint8_t*>(v);
  p.idx = idx;
  p.kv_sl = kv_sl; p.kv_sb = kv_sb; p.kv_sh = kv_sh;
  p.row_bytes = row_bytes;
  p.B = B; p.Hkv = Hkv; p.k_rows = k_rows; p.k_stride = k_stride;
  p.n_layers = n_layers;
  for (int i = 0; i < n_layers; ++i) {
    p.layers[i] = layers[i];
    p.src_slot[i] = src_slots[i];
  }
  p.sink = static_cast<uint32_t*>(sink);
  // blocks_per_sm here: splits per pair (the grid is splits x pairs)
  const int pairs = n_layers * B * Hkv;
  dim3 grid(blocks_per_sm, pairs);
  if ((k_rows + blocks_per_sm - 1) / blocks_per_sm > kMaxStage) return 1;
  // HYLRA_PROBE_SMEM (bytes of unused dynamic shared memory per CTA) caps CTAs per SM, i.e.
  // the bytes in flight: the experiment that tells whether in-flight bytes bound a gather
  const char* e = getenv("HYLRA_PROBE_SMEM");
  const int smem = (e && *e) ? atoi(e) : 0;
  if (smem + (int)sizeof(int32_t) * kMaxStage > 48 * 1024)
    cudaFuncSetAttribute(gather_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  gather_probe_kernel<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
