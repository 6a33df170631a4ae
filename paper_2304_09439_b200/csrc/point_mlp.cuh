// point_mlp.cuh — the shared point MLP of S4-S5 on CUDA cores (fp32), for one 64-row tile:
//   h1 = ReLU(W1 p + b1), h2 = ReLU(W2 h1 + b2), acc = W3 h2
// Thread f owns feature f (H <= 256).  Used by the fp32 crop encoder (kernels_encoder_f32.cu) and
// the encode-once grid encoder (kernels_cells.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace locc {
namespace {

constexpr int kMlpTR = 64;            // rows per tile
constexpr int kMlpLDH = kMlpTR + 4;   // padded row stride of the transposed activation tile

// rows_s: [64] staged rows (x, y, z, *); hT: [H][kMlpLDH] shared scratch.  Returns the layer-3
// pre-bias accumulators of feature f for the 64 rows.  Contains __syncthreads (call block-wide).
__device__ __forceinline__ void point_mlp_tile(const DevParams& P, const float4* rows_s, float* hT,
                                               float (&acc)[kMlpTR], float4 w1, float b2, int f, bool act) {
  constexpr int TR = kMlpTR, LDH = kMlpLDH;
  const int H = P.H;
  // layer 1 (fp32 FFMA)
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
  __syncthreads();
  for (int layer = 0; layer < 2; ++layer) {
    const float* WT = layer == 0 ? P.w2T : P.w3T;
#pragma unroll
    for (int r = 0; r < TR; ++r) acc[r] = 0.f;
    if (act) {
#pragma unroll 2
      for (int k = 0; k < H; ++k) {
        const float w = __ldg(WT + (int64_t)k * H + f);
        const float4* hk = reinterpret_cast<const float4*>(&hT[k * LDH]);
#pragma unroll
        for (int r = 0; r < TR / 4; ++r) {
          const float4 h = hk[r];
          acc[4 * r + 0] = fmaf(w, h.x, acc[4 * r + 0]);
          acc[4 * r + 1] = fmaf(w, h.y, acc[4 * r + 1]);
          acc[4 * r + 2] = fmaf(w, h.z, acc[4 * r + 2]);
          acc[4 * r + 3] = fmaf(w, h.w, acc[4 * r + 3]);
        }
      }
    }
    __syncthreads();
    if (layer == 0) {
      if (act) {
#pragma unroll
        for (int r = 0; r < TR; r += 4)
          *reinterpret_cast<float4*>(&hT[f * LDH + r]) =
              make_float4(fmaxf(acc[r] + b2, 0.f), fmaxf(acc[r + 1] + b2, 0.f), fmaxf(acc[r + 2] + b2, 0.f),
                          fmaxf(acc[r + 3] + b2, 0.f));
      }
      __syncthreads();
    }
  }
}

}  // namespace
}  // namespace locc
