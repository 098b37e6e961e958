// append.cuh — write one decode step's new key/value rows into the KV cache.
//
// The reference grows its cache by one row per step (synthetic.py:154-187 `grown_arrays`,
// engine.py:167-169 n_t = N + t); here the caller hands the new rows of every layer,
// [L][B][Hkv][d], and they land at cache row `pos` of each selected layer. The rows may
// sit in page-locked host memory: each thread then reads its 16-byte chunk across the link
// itself (zero-copy), so a host-resident step input needs no separate H2D copy.
#pragma once

#include "attention.cuh"

namespace hylra {

constexpr int kAppendThreads = 256;

// Any NaN / inf among the 8 bf16 or 4 fp32 values of a 16-byte chunk (all-ones exponent).
__device__ __forceinline__ bool chunk_non_finite(const uint4& c, bool bf16) {
  const uint32_t w[4] = {c.x, c.y, c.z, c.w};
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (bf16) bad |= ((w[i] & 0x7f80u) == 0x7f80u) || ((w[i] & 0x7f800000u) == 0x7f800000u);
    else bad |= (w[i] & 0x7f800000u) == 0x7f800000u;
  }
  return bad;
}

struct AppendParams {
  const uint4* k_rows;  // [L][B][Hkv][d] elements, 16-byte chunks
  const uint4* v_rows;
  uint8_t* k;           // cache base (bytes)
  uint8_t* v;
  int* flags;           // workspace flag word or null: a non-finite new row sets
                        // HYLRA_FLAG_NON_FINITE_CACHE (attention.py:43-44)
  int bf16;
  int64_t kv_sl, kv_sb, kv_sh;  // cache strides in bytes
  int64_t pos_bytes;            // pos * d * element size
  int B, Hkv, chunks;           // chunks = d * element size / 16 per row
  int n_layers;
  int layers[kMaxSlots];        // cache layer of each slot (rows indexed by the same id)
};

// One thread per 16-byte chunk of the selected layers' K and V rows.
__global__ void __launch_bounds__(kAppendThreads) append_kv_kernel(const AppendParams p) {
  const int64_t per_tensor = (int64_t)p.n_layers * p.B * p.Hkv * p.chunks;
  const int64_t i = (int64_t)blockIdx.x * kAppendThreads + threadIdx.x;
  if (i >= 2 * per_tensor) return;
  const bool is_v = i >= per_tensor;
  int64_t r = is_v ? i - per_tensor : i;
  const int c = (int)(r % p.chunks);
  r /= p.chunks;
  const int h = (int)(r % p.Hkv);
  r /= p.Hkv;
  const int b = (int)(r % p.B);
  const int l = p.layers[r / p.B];
  const int64_t src = (((int64_t)l * p.B + b) * p.Hkv + h) * p.chunks + c;
  const uint4 val = is_v ? p.v_rows[src] : p.k_rows[src];
  uint8_t* dst = (is_v ? p.v : p.k) + l * p.kv_sl + b * p.kv_sb + h * p.kv_sh + p.pos_bytes;
  reinterpret_cast<uint4*>(dst)[c] = val;
  if (p.flags != nullptr && chunk_non_finite(val, p.bf16 != 0)) atomicOr(p.flags, 16);
}

// Whole-cache validation (attention.py:38-46,61-71: the reference copies every layer's K/V
// into read-only float64 arrays and rejects any non-finite entry at construction). One
// streaming pass over rows [0, n_valid) of the listed layers: 16-byte loads, 4 in flight per
// thread, evict-first; any NaN / inf sets HYLRA_FLAG_NON_FINITE_CACHE. grid = (chunks of a
// (layer, b, kv-head) block, blocks); a block = rows [0, n_valid) of one (layer, b, kv-head).
constexpr int kCheckThreads = 256, kCheckUnroll = 4;

struct CheckParams {
  const uint8_t* k;
  const uint8_t* v;
  int* flags;
  int64_t kv_sl, kv_sb, kv_sh;  // bytes
  int64_t block_chunks;         // 16-byte chunks of one (layer, b, kv-head) block
  int B, Hkv, bf16, n_layers;
  int layers[kMaxSlots];
};

__global__ void __launch_bounds__(kCheckThreads) check_finite_kernel(const CheckParams p) {
  int r = blockIdx.y;
  const int h = r % p.Hkv;
  r /= p.Hkv;
  const int b = r % p.B;
  r /= p.B;
  const bool is_v = r >= p.n_layers;
  const int l = p.layers[is_v ? r - p.n_layers : r];
  const uint4* base = reinterpret_cast<const uint4*>((is_v ? p.v : p.k) + l * p.kv_sl +
                                                     b * p.kv_sb + h * p.kv_sh);
  bool bad = false;
  const int64_t step = (int64_t)gridDim.x * kCheckThreads * kCheckUnroll;
  for (int64_t i0 = (int64_t)blockIdx.x * kCheckThreads * kCheckUnroll + threadIdx.x;
       i0 < p.block_chunks; i0 += step) {
    uint4 v[kCheckUnroll];
#pragma unroll
    for (int u = 0; u < kCheckUnroll; ++u) {
      const int64_t i = i0 + (int64_t)u * kCheckThreads;
      v[u] = i < p.block_chunks ? __ldcs(base + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kCheckUnroll; ++u) bad |= chunk_non_finite(v[u], p.bf16 != 0);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(p.flags, 16);
}

}  // namespace hylra
