// point_mlp.cuh — the shared point MLP of S4-S5 on CUDA cores (fp32), for one 64-row tile:
//   h1 = ReLU(W1 p + b1), h2 = ReLU(W2 h1 + b2), acc = W3 h2
// Used by the fp32 crop encoder (kernels_encoder_f32.cu) and the encode-once grid encoder
// (kernels_cells.cu); 256 threads, H <= 256 in steps of 32.
//
// Layers 2 and 3 are register-tiled FFMA GEMMs: thread (ty, tx) = (warp, lane) accumulates rows
// 8 ty .. 8 ty + 7 x features 4 tx .. 4 tx + 3 and 128 + 4 tx .. 128 + 4 tx + 3 (64 accumulators;
// per k, 2 broadcast float4 loads of h and 2 float4 loads of W feed 32 FFMA2s with h as the broadcast
// operand), with W streamed through shared memory in 16-row chunks (cp.async, double-buffered) instead
// of one global load per k.  Every
// output is the same k-ascending fmaf chain as a plain dot product, so the results are bitwise those of
// a thread-per-feature loop.  On return hT[f][r] holds feature f's layer-3 accumulators of the 64 rows
// (the callers' cell walks run per feature, reading them from shared memory).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace locc {
namespace {

constexpr int kMlpTR = 64;            // rows per tile
constexpr int kMlpLDH = kMlpTR + 4;   // padded row stride of the transposed activation tile
constexpr int kMlpKC = 16;            // weight rows per shared-memory chunk
// shared memory of one tile: staged rows, the transposed activations [256][kMlpLDH], two weight chunks
constexpr size_t kMlpSmemBytes = sizeof(float4) * kMlpTR + sizeof(float) * 256 * kMlpLDH +
                                 sizeof(float) * 2 * kMlpKC * 256;

__device__ __forceinline__ void mlp_cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

// Rows k0 .. k0 + kMlpKC - 1 of WT ([H in][H out]) into dst (row stride 256), as one cp.async group.
__device__ __forceinline__ void mlp_load_chunk(const float* WT, int H, int k0, float* dst) {
  const int q = H >> 2;  // float4 per row
  for (int i = threadIdx.x; i < kMlpKC * q; i += 256) {
    const int kk = i / q, c4 = i - kk * q;
    mlp_cp_async16(dst + kk * 256 + 4 * c4, WT + (int64_t)(k0 + kk) * H + 4 * c4);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// rows_s: [64] staged rows (x, y, z, *); hT: [256][kMlpLDH] shared scratch followed by the weight
// chunks (2 x kMlpKC x 256 floats).  Leaves the layer-3 pre-bias accumulators in hT[f * kMlpLDH + r].
// Contains __syncthreads (call block-wide); the caller syncs before the next tile's call.
__device__ __forceinline__ void point_mlp_tile(const DevParams& P, const float4* rows_s, float* hT, float4 w1, int f,
                                               bool act) {
  constexpr int TR = kMlpTR, LDH = kMlpLDH, KC = kMlpKC;
  const int H = P.H;
  float* wbuf = hT + 256 * LDH;
  const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
  // layer 1 (fp32 FFMA), thread f = feature f
  if (act) {
#pragma unroll
    for (int r = 0; r < TR; r += 4) {
      float v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 p = rows_s[r + j];
        const float h = fmaf(w1.x, p.x, fmaf(w1.y, p.y, fmaf(w1.z, p.z, w1.w)));
        v[j] = fmaxf(h, 0.f);
      }
      *reinterpret_cast<float4*>(&hT[f * LDH + r]) = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
  // this thread's features of the GEMM tile: 4 tx + j (j < 4) and 128 + 4 tx + j - 4 (j >= 4)
  const bool g0 = 4 * tx < H, g1 = 128 + 4 * tx < H;
  for (int layer = 0; layer < 2; ++layer) {
    const float* WT = layer == 0 ? P.w2T : P.w3T;
    float2 c[8][4];  // c[i][m] = features (2 m, 2 m + 1) of the thread's 8 (FFMA2 pairs)
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int m = 0; m < 4; ++m) c[i][m] = make_float2(0.f, 0.f);
    mlp_load_chunk(WT, H, 0, wbuf);
    const int nch = H / KC;
    for (int ch = 0; ch < nch; ++ch) {
      float* wc = wbuf + (ch & 1) * KC * 256;
      if (ch + 1 < nch) {
        mlp_load_chunk(WT, H, (ch + 1) * KC, wbuf + ((ch + 1) & 1) * KC * 256);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();  // chunk ch (and, at ch = 0, this layer's h) visible to every thread
#pragma unroll 4
      for (int kk = 0; kk < KC; ++kk) {
        const int k = ch * KC + kk;
        const float4 ha = *reinterpret_cast<const float4*>(&hT[k * LDH + 8 * ty]);
        const float4 hb = *reinterpret_cast<const float4*>(&hT[k * LDH + 8 * ty + 4]);
        const float4 wa = g0 ? *reinterpret_cast<const float4*>(&wc[kk * 256 + 4 * tx]) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 wb = g1 ? *reinterpret_cast<const float4*>(&wc[kk * 256 + 128 + 4 * tx])
                             : make_float4(0.f, 0.f, 0.f, 0.f);
        const float h[8] = {ha.x, ha.y, ha.z, ha.w, hb.x, hb.y, hb.z, hb.w};
        const float2 w2[4] = {make_float2(wa.x, wa.y), make_float2(wa.z, wa.w), make_float2(wb.x, wb.y),
                              make_float2(wb.z, wb.w)};
        // FFMA2 with h as the broadcast operand: per element the same fmaf(w, h, c) as a scalar loop
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int m = 0; m < 4; ++m) c[i][m] = __ffma2_rn(w2[m], make_float2(h[i], h[i]), c[i][m]);
      }
      __syncthreads();  // every read of chunk ch (and, at the last chunk, of h) done
    }
    // back to the transposed layout: layer 2's h2 = ReLU(acc + b2) feeds layer 3; layer 3's raw
    // accumulators go to the per-feature threads
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int fj = (j < 4 ? 4 * tx : 124 + 4 * tx) + j;
      if (fj < H) {
        const float bj = layer == 0 ? P.b2[fj] : 0.f;
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float cv = (j & 1) ? c[i][j >> 1].y : c[i][j >> 1].x;
          v[i] = layer == 0 ? fmaxf(cv + bj, 0.f) : cv;
        }
        *reinterpret_cast<float4*>(&hT[fj * LDH + 8 * ty]) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(&hT[fj * LDH + 8 * ty + 4]) = make_float4(v[4], v[5], v[6], v[7]);
      }
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace locc
