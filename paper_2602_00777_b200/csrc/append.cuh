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

struct AppendParams {
  const uint4* k_rows;  // [L][B][Hkv][d] elements, 16-byte chunks
  const uint4* v_rows;
  uint8_t* k;           // cache base (bytes)
  uint8_t* v;
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
}

}  // namespace hylra
