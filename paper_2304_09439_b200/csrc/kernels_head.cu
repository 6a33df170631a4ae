// kernels_head.cu — S7 projection + S8-S9 collision predictor, fp32 on CUDA cores.
//
// Per pair: e_s = W_F m_s + b_F (one linear layer to F; e_s = 0
// for an empty crop); z_s = [e_s ; canonical unit quaternion ; translation]
// (reading Q12); u_s = ReLU^3 of the shared 3x128 object MLP; v = max(u_A, u_B) ("max-pooling
// across object pairs"); 3x128 ReLU; linear; sigmoid; label = p > 0.5.  Both crops empty ->
// short-circuit: p = 0, label 0, logit -inf.
//
// A block of 128 threads evaluates PB pairs (2*PB sides): thread o computes output unit o of a
// layer for all rows it serves, weights read as coalesced rows of W^T, activations broadcast
// from shared memory.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"
#include "quat.cuh"

namespace locc {
namespace {

constexpr int PB = 16;          // pairs per block
constexpr int NS = 2 * PB;      // sides per block
constexpr int ZW = 320;         // row stride of the activation buffers (>= H, F+7, 128)

template <int R>
__device__ __forceinline__ void dense_rows(const float* __restrict__ WT, const float* __restrict__ bias, int n_in,
                                           int n_out, const float* in, float* out, bool relu) {
  for (int o = threadIdx.x; o < n_out; o += blockDim.x) {
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    for (int i = 0; i < n_in; ++i) {
      const float w = __ldg(WT + (int64_t)i * n_out + o);
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = fmaf(w, in[r * ZW + i], acc[r]);
    }
    const float bo = bias[o];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float v = acc[r] + bo;
      out[r * ZW + o] = relu ? fmaxf(v, 0.f) : v;
    }
  }
}

__global__ void __launch_bounds__(128) head_kernel(DevParams P, Batch b, float* __restrict__ probs,
                                                   uint8_t* __restrict__ labels, float* __restrict__ logits,
                                                   float* __restrict__ emb) {
  extern __shared__ float sm[];
  float* X = sm;             // [NS][ZW]  pooled features, later object MLP activations
  float* Z = X + NS * ZW;    // [NS][ZW]
  __shared__ int nside[NS];
  const int H = P.H, F = P.F;
  const int64_t i0 = (int64_t)blockIdx.x * PB;
  const int npairs = (int)min((int64_t)PB, b.B - i0);
  for (int s = threadIdx.x; s < NS; s += blockDim.x) nside[s] = s < 2 * npairs ? b.counts[2 * i0 + s] : 0;
  __syncthreads();
  // pooled features (empty or padding sides -> 0)
  for (int idx = threadIdx.x; idx < NS * H; idx += blockDim.x) {
    const int s = idx / H, j = idx - s * H;
    X[s * ZW + j] = nside[s] > 0 ? b.pooled[(2 * i0 + s) * (int64_t)H + j] : 0.f;
  }
  __syncthreads();
  // S7 projection e = W_F m + b_F -> Z[:, 0:F]
  dense_rows<NS>(P.wfT, P.bf, H, F, X, Z, false);
  __syncthreads();
  // z = [e (0 if empty); canonical q; t]
  for (int s = threadIdx.x; s < NS; s += blockDim.x) {
    if (nside[s] == 0)
      for (int j = 0; j < F; ++j) Z[s * ZW + j] = 0.f;
    float* z = Z + s * ZW + F;
    if (s < 2 * npairs) {
      const float* pose = b.poses + (2 * i0 + s) * 7;
      double q[4] = {1.0, 0.0, 0.0, 0.0};
      quat_unit(pose, q);
      double sg = 1.0;
      for (int c = 0; c < 4; ++c)
        if (q[c] != 0.0) {
          sg = q[c] > 0.0 ? 1.0 : -1.0;
          break;
        }
      for (int c = 0; c < 4; ++c) z[c] = __double2float_rn(sg * q[c]);
      for (int c = 0; c < 3; ++c) z[4 + c] = pose[4 + c];
    } else {
      for (int c = 0; c < 7; ++c) z[c] = 0.f;
    }
    if (emb && s < 2 * npairs)
      for (int j = 0; j < F; ++j) emb[(2 * i0 + s) * (int64_t)F + j] = Z[s * ZW + j];
  }
  __syncthreads();
  // S8 object MLP (shared by both sides)
  dense_rows<NS>(P.o1T, P.ob1, F + 7, kPredW, Z, X, true);
  __syncthreads();
  dense_rows<NS>(P.o2T, P.ob2, kPredW, kPredW, X, Z, true);
  __syncthreads();
  dense_rows<NS>(P.o3T, P.ob3, kPredW, kPredW, Z, X, true);
  __syncthreads();
  // S9 max across the pair -> Z rows 0..PB-1
  for (int idx = threadIdx.x; idx < PB * kPredW; idx += blockDim.x) {
    const int p = idx / kPredW, j = idx - p * kPredW;
    Z[p * ZW + j] = fmaxf(X[(2 * p) * ZW + j], X[(2 * p + 1) * ZW + j]);
  }
  __syncthreads();
  dense_rows<PB>(P.p1T, P.pb1, kPredW, kPredW, Z, X, true);
  __syncthreads();
  dense_rows<PB>(P.p2T, P.pb2, kPredW, kPredW, X, Z, true);
  __syncthreads();
  dense_rows<PB>(P.p3T, P.pb3, kPredW, kPredW, Z, X, true);
  __syncthreads();
  // output unit + sigmoid: warp w handles pairs w, w+4, ...
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int p = w; p < npairs; p += blockDim.x >> 5) {
    float acc = 0.f;
    for (int j = lane; j < kPredW; j += 32) acc = fmaf(P.wout[j], X[p * ZW + j], acc);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const int64_t i = i0 + p;
      float lg, pr;
      if (nside[2 * p] + nside[2 * p + 1] == 0) {
        lg = -INFINITY;
        pr = 0.f;
      } else {
        lg = acc + P.bout[0];
        pr = 1.f / (1.f + expf(-lg));
        atomicAdd(&b.stats->evaluated_pairs, 1ull);
      }
      probs[i] = pr;
      if (labels) labels[i] = pr > 0.5f ? 1 : 0;
      if (logits) logits[i] = lg;
    }
  }
}

}  // namespace

cudaError_t launch_head(const DevParams& P, const Batch& b, float* probs, uint8_t* labels, float* logits, float* emb,
                        cudaStream_t st) {
  if (b.B == 0) return cudaSuccess;
  const size_t sm = sizeof(float) * 2 * NS * ZW;
  static const cudaError_t attr =
      cudaFuncSetAttribute(head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (attr != cudaSuccess) return attr;
  head_kernel<<<(unsigned)((b.B + PB - 1) / PB), 128, sm, st>>>(P, b, probs, labels, logits, emb);
  return cudaGetLastError();
}

}  // namespace locc
