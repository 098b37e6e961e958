/*
 * decode_step.c — a C host driving the drop-in boundary (include/hylra.h) directly: no
 * Python, no torch. It is what a non-Python caller of the reference's layer-policy
 * interface (a cgo / JNI / N-API binding, or a C++ serving loop) does per decode step.
 *
 *   gcc -O2 -std=c11 examples/decode_step.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2602_00777_b200 -lhylra -L/usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$PWD/paper_2602_00777_b200 -o decode_step && ./decode_step
 *
 * Policy [FULL, REUSE, FULL, REUSE], B = 2, Hq = 8, Hkv = 2 (GQA 4), d = 128, bf16 cache of
 * N = 4096 rows, budget 256. Checks, against a float64 evaluation on the host: the FULL
 * layers' top-k sets (exact), every layer's output (relative L2 < 2e-2 per head), and that
 * REUSE layers read their source FULL layer's set. Exit status 0 = all checks passed.
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hylra.h"

enum { L = 4, B = 2, HQ = 8, HKV = 2, D = 128, N = 4096, BUDGET = 256, G = HQ / HKV };

static uint16_t f2bf(float f) {  /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static double bf2d(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint64_t rng = 88172645463325252ull;
static float gauss(void) {  /* xorshift + Box-Muller */
  double u1, u2;
  rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17;
  u1 = ((rng >> 11) + 1.0) / 9007199254740993.0;
  rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17;
  u2 = (rng >> 11) / 9007199254740992.0;
  return (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
}

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
  return 2; } } while (0)
#define HY(x) do { int s_ = (x); if (s_ != HYLRA_OK) { \
  fprintf(stderr, "%s: %s\n", hylra_status_string(s_), hylra_last_error()); return 3; } } while (0)

int main(void) {
  const size_t nq = (size_t)L * B * HQ * D, nkv = (size_t)L * B * HKV * N * D;
  uint16_t* hq = malloc(nq * 2);
  uint16_t* hk = malloc(nkv * 2);
  uint16_t* hv = malloc(nkv * 2);
  for (size_t i = 0; i < nq; ++i) hq[i] = f2bf(gauss());
  for (size_t i = 0; i < nkv; ++i) hk[i] = f2bf(gauss());
  for (size_t i = 0; i < nkv; ++i) hv[i] = f2bf(gauss());

  hylra_geometry g = {0};
  g.batch = B; g.q_heads = HQ; g.kv_heads = HKV; g.head_dim = D; g.capacity = N;
  g.dtype = HYLRA_BF16; g.num_layers = L;
  g.q_stride_layer = (int64_t)B * HQ * D; g.q_stride_batch = HQ * D;
  g.kv_stride_head = (int64_t)N * D; g.kv_stride_batch = (int64_t)HKV * N * D;
  g.kv_stride_layer = (int64_t)B * HKV * N * D;
  g.out_stride_layer = (int64_t)B * HQ * D; g.out_stride_batch = HQ * D;
  const uint8_t actions[L] = {1, 0, 1, 0};
  const int n_full = 2, k_eff = BUDGET;

  void *dq, *dk, *dv, *dws;
  float* dout;
  int32_t* didx;
  CK(cudaMalloc(&dq, nq * 2));
  CK(cudaMalloc(&dk, nkv * 2));
  CK(cudaMalloc(&dv, nkv * 2));
  CK(cudaMalloc((void**)&dout, nq * 4));
  CK(cudaMalloc((void**)&didx, sizeof(int32_t) * n_full * B * HKV * k_eff));
  const size_t ws_bytes = hylra_decode_step_workspace_bytes(&g, actions, N, BUDGET, 1, 0, 0);
  if (ws_bytes == 0) { fprintf(stderr, "workspace query: %s\n", hylra_last_error()); return 3; }
  CK(cudaMalloc(&dws, ws_bytes));
  CK(cudaMemset(dws, 0, ws_bytes));  /* zeroed once; the kernels leave it zeroed */
  CK(cudaMemcpy(dq, hq, nq * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dk, hk, nkv * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, hv, nkv * 2, cudaMemcpyHostToDevice));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));

  for (int rep = 0; rep < 2; ++rep)  /* the same workspace serves every step */
    HY(hylra_decode_step(&g, dq, dk, dv, N, actions, BUDGET, 1, 1, 0, 0, dout, didx, k_eff,
                         dws, ws_bytes, st));
  CK(cudaStreamSynchronize(st));
  int32_t flags = 0;
  HY(hylra_read_flags(dws, &flags, st));
  if (flags) { fprintf(stderr, "device flags %d\n", flags); return 4; }

  float* hout = malloc(nq * 4);
  int32_t* hidx = malloc(sizeof(int32_t) * n_full * B * HKV * k_eff);
  CK(cudaMemcpy(hout, dout, nq * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hidx, didx, sizeof(int32_t) * n_full * B * HKV * k_eff, cudaMemcpyDeviceToHost));

  /* float64 host check: the reference's algorithm (engine.py:167-197) per KV-head group */
  double* agg = malloc(sizeof(double) * N);
  double* lg = malloc(sizeof(double) * N);
  int* sel = malloc(sizeof(int) * N);
  int* cur = malloc(sizeof(int) * k_eff);
  double worst = 0.0;
  int slot = -1, bad_sets = 0;
  for (int l = 0; l < L; ++l) {
    if (actions[l]) ++slot;
    for (int b = 0; b < B; ++b)
      for (int kh = 0; kh < HKV; ++kh) {
        const uint16_t* K = hk + (((size_t)l * B + b) * HKV + kh) * N * D;
        const uint16_t* V = hv + (((size_t)l * B + b) * HKV + kh) * N * D;
        const int32_t* got = hidx + (((size_t)slot * B + b) * HKV + kh) * k_eff;
        if (actions[l]) {  /* summed logits of the group, top-k, lower index on ties */
          for (int n = 0; n < N; ++n) agg[n] = 0.0;
          for (int gq = 0; gq < G; ++gq) {
            const uint16_t* q = hq + (((size_t)l * B + b) * HQ + kh * G + gq) * D;
            for (int n = 0; n < N; ++n) {
              double s = 0.0;
              for (int i = 0; i < D; ++i) s += bf2d(q[i]) * bf2d(K[(size_t)n * D + i]);
              agg[n] += s / sqrt((double)D);
            }
          }
          for (int n = 0; n < N; ++n) sel[n] = 0;
          for (int r = 0; r < k_eff; ++r) {  /* k passes of argmax (lowest index wins) */
            int best = -1;
            for (int n = 0; n < N; ++n)
              if (!sel[n] && (best < 0 || agg[n] > agg[best])) best = n;
            sel[best] = 1;
          }
          int pos = 0;
          for (int n = 0; n < N; ++n)
            if (sel[n]) cur[pos++] = n;
          for (int r = 0; r < k_eff; ++r) bad_sets += got[r] != cur[r];
        } else {  /* REUSE: the source FULL layer's set */
          for (int r = 0; r < k_eff; ++r) cur[r] = got[r];
        }
        for (int gq = 0; gq < G; ++gq) {  /* attention over all rows (FULL) or the set */
          const int hqi = kh * G + gq;
          const uint16_t* q = hq + (((size_t)l * B + b) * HQ + hqi) * D;
          const int m = actions[l] ? N : k_eff;
          double mx = -INFINITY, num = 0.0, den = 0.0, o[D];
          for (int j = 0; j < m; ++j) {
            const int n = actions[l] ? j : cur[j];
            double s = 0.0;
            for (int i = 0; i < D; ++i) s += bf2d(q[i]) * bf2d(K[(size_t)n * D + i]);
            lg[j] = s / sqrt((double)D);
            if (lg[j] > mx) mx = lg[j];
          }
          for (int i = 0; i < D; ++i) o[i] = 0.0;
          for (int j = 0; j < m; ++j) {
            const int n = actions[l] ? j : cur[j];
            const double w = exp(lg[j] - mx);
            den += w;
            for (int i = 0; i < D; ++i) o[i] += w * bf2d(V[(size_t)n * D + i]);
          }
          const float* got_o = hout + (((size_t)l * B + b) * HQ + hqi) * D;
          for (int i = 0; i < D; ++i) {
            o[i] /= den;
            num += (got_o[i] - o[i]) * (got_o[i] - o[i]);
          }
          double ref2 = 0.0;
          for (int i = 0; i < D; ++i) ref2 += o[i] * o[i];
          const double rel = sqrt(num / ref2);
          if (rel > worst) worst = rel;
        }
      }
  }
  /* the same step as ONE kernel (hylra_decode_step_ex, fuse_select = 2): same split-K
     partitions, so outputs and selections must match the 3-launch step bit for bit */
  hylra_step_options opt;
  memset(&opt, 0, sizeof(opt));
  opt.fuse_select = 2;
  const unsigned long long before = hylra_launch_count();
  CK(cudaMemset(dout, 0, nq * 4));
  CK(cudaMemset(didx, 0, sizeof(int32_t) * n_full * B * HKV * k_eff));
  HY(hylra_decode_step_ex(&g, dq, dk, dv, N, actions, BUDGET, 1, 1, 0, 0, dout, didx, k_eff, dws,
                          ws_bytes, st, &opt));
  CK(cudaStreamSynchronize(st));
  const unsigned long long single_launches = hylra_launch_count() - before;
  float* hout1 = malloc(nq * 4);
  int32_t* hidx1 = malloc(sizeof(int32_t) * n_full * B * HKV * k_eff);
  CK(cudaMemcpy(hout1, dout, nq * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hidx1, didx, sizeof(int32_t) * n_full * B * HKV * k_eff, cudaMemcpyDeviceToHost));
  const int single_same = memcmp(hout1, hout, nq * 4) == 0 &&
                          memcmp(hidx1, hidx, sizeof(int32_t) * n_full * B * HKV * k_eff) == 0;
  printf("decode_step.c: launches %llu, worst relative L2 %.2e, set mismatches %d, "
         "single-launch step: %llu launch, bit-identical %d\n",
         (unsigned long long)hylra_launch_count(), worst, bad_sets, single_launches, single_same);
  free(hout1);
  free(hidx1);
  if (!single_same || single_launches != 1) return 5;
  cudaFree(dq); cudaFree(dk); cudaFree(dv); cudaFree(dout); cudaFree(didx); cudaFree(dws);
  cudaStreamDestroy(st);
  return (worst < 2e-2 && bad_sets == 0) ? 0 : 1;
}
