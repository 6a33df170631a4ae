// kernels_encoder_f32.cu — S4-S7 on CUDA cores in fp32 (LOCC_PREC_FP32; the parity path and the
// FFMA baseline the tensor-core encoder is measured against).
//
// Work unit: a chunk of kSegPerChunk whole (pair, side) segments = a contiguous row range of the
// compacted row buffer.  Thread f owns feature f (H <= 256) and, for each 64-row tile:
//   h1 = ReLU(W1 p + b1)               (input = local xyz, reading Q6)
//   h2 = ReLU(W2 h1 + b2), acc3 = W3 h2 ("3 layers of MLP with 256 neurons")
// then walks the tile's rows in order with its 64 accumulators of layer 3: the rows are sorted by
// (segment, cell), so the cell-wise max pool is a running max that closes at each
// cell end, g = ReLU(max + b3) (bias+ReLU is monotone, so this equals the max of ReLU(acc + b3)),
// and the occupied-cell mean ("average pooling") a running sum in ascending
// cell order, divided by C at the segment end.  Projection to F happens in the predictor kernel.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"
#include "point_mlp.cuh"

namespace locc {
namespace {

constexpr int TR = kMlpTR;
constexpr int LDH = kMlpLDH;

__global__ void __launch_bounds__(256, 2) encoder_f32_kernel(DevParams P, Batch b) {
  extern __shared__ float4 smem4[];
  float4* rows_s = smem4;                        // [TR]
  float* hT = reinterpret_cast<float*>(smem4 + TR);  // [H][LDH]
  const int H = P.H;
  const int f = threadIdx.x;
  const bool act = f < H;
  const int64_t s0 = (int64_t)blockIdx.x * kSegPerChunk;
  const int64_t s1 = min(s0 + kSegPerChunk, b.G);
  const int64_t r0 = b.offsets[s0], r1 = b.offsets[s1];
  if (r0 == r1) return;

  float4 w1 = make_float4(0.f, 0.f, 0.f, 0.f);
  float b3 = 0.f;
  if (act) {
    w1 = P.w1b[f];
    b3 = P.b3[f];
  }
  float run_max = -INFINITY, run_sum = 0.f;
  int run_cells = 0;

  for (int64_t t0 = r0; t0 < r1; t0 += TR) {
    const int nr = (int)min((int64_t)TR, r1 - t0);
    if (f < TR) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (f < nr) {  // the row's coordinates from the shape table (own shape of the row's segment)
        LOCC_CHECK(t0 + f < b.rows_cap);
        const uint2 rw = b.rows[t0 + f];
        LOCC_CHECK((rw.x >> kRowSegShift) < b.G && rw.y < (uint32_t)b.K);
        const int own = __float_as_int(b.xf[4 * (int64_t)(rw.x >> kRowSegShift) + 3].x);
        LOCC_CHECK((unsigned)own < (unsigned)b.S);
        const float4 p = b.pts[(int64_t)own * b.K + rw.y];
        v = make_float4(p.x, p.y, p.z, __uint_as_float(rw.x));
      }
      rows_s[f] = v;
    }
    __syncthreads();
    point_mlp_tile(P, rows_s, hT, w1, f, act);
    const float* acc = hT + f * LDH;  // feature f's layer-3 accumulators of the tile's rows
    // S6-S7: segmented cell max + occupied-cell sum over the tile's rows (row flags are uniform)
    if (act) {
#pragma unroll 4
      for (int r = 0; r < TR; ++r) {
        const uint32_t fl = __float_as_uint(rows_s[r].w);
        if (r < nr && !(fl & kRowFlagPad)) {
          run_max = fmaxf(run_max, acc[r]);
          if (fl & kRowFlagCellEnd) {
            run_sum += fmaxf(run_max + b3, 0.f);
            ++run_cells;
            run_max = -INFINITY;
          }
          if (fl & kRowFlagSegEnd) {
            const int64_t seg = fl >> kRowSegShift;
            LOCC_CHECK(seg < b.G && run_cells > 0);
            b.pooled[seg * H + f] = __fdiv_rn(run_sum, (float)run_cells);
            run_sum = 0.f;
            run_cells = 0;
          }
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_encoder_f32(const DevParams& P, const Batch& b, cudaStream_t st) {
  const int64_t chunks = (b.G + kSegPerChunk - 1) / kSegPerChunk;
  if (chunks == 0) return cudaSuccess;
  const size_t sm = kMlpSmemBytes;
  const cudaError_t attr = smem_optin(encoder_f32_kernel, sm);
  if (attr != cudaSuccess) return attr;
  encoder_f32_kernel<<<(unsigned)chunks, 256, sm, st>>>(P, b);
  return cudaGetLastError();
}

}  // namespace locc
