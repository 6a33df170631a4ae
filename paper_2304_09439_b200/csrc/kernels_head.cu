// kernels_head.cu — S7 projection + S8-S9 collision predictor, fp32 on CUDA cores.
//
// Per pair: e_s = W_F m_s + b_F (one linear layer to F; e_s = 0
// for an empty crop); z_s = [e_s ; canonical unit quaternion ; translation]
// (reading Q12); u_s = ReLU^3 of the shared 3x128 object MLP; v = max(u_A, u_B) ("max-pooling
// across object pairs"); 3x128 ReLU; linear; sigmoid; label = p > 0.5.  Both crops empty ->
// short-circuit: p = 0, label 0, logit -inf.
//
// A block of 128 threads evaluates PB = 16 pairs (32 sides).  Activations live in shared memory
// transposed, [feature][row] with rows contiguous, so a thread computing output unit o for all rows
// reads 4 rows per LDS.128 and updates 2 rows per packed FFMA2; weights are coalesced rows of W^T.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"
#include "quat.cuh"
#include "tc_ptx.cuh"

namespace locc {
namespace {

using tc::f2;
using tc::f2_hi;
using tc::f2_lo;
using tc::ffma2;

constexpr int PB = 16;      // pairs per block
constexpr int NS = 2 * PB;  // sides per block
constexpr int LD = 36;      // row stride (floats) of the transposed activation buffers

// out[o][r] = act(sum_i WT[i][o] in[i][r] + b[o]) for o in [o0, o0 + n_out step ostep), r < R.
template <int R>
__device__ __forceinline__ void dense_t(const float* __restrict__ WT, const float* __restrict__ bias, int n_in,
                                        int n_out, const float* in, int r0, float* out, bool relu, int o, int ostep) {
  for (; o < n_out; o += ostep) {
    unsigned long long acc[R / 2];
#pragma unroll
    for (int r = 0; r < R / 2; ++r) acc[r] = 0ull;
#pragma unroll 4
    for (int i = 0; i < n_in; ++i) {
      const float w = __ldg(WT + (int64_t)i * n_out + o);
      const unsigned long long w2 = f2(w, w);
      const float4* x = reinterpret_cast<const float4*>(in + i * LD + r0);
#pragma unroll
      for (int r = 0; r < R / 4; ++r) {
        const float4 v = x[r];
        acc[2 * r] = ffma2(w2, f2(v.x, v.y), acc[2 * r]);
        acc[2 * r + 1] = ffma2(w2, f2(v.z, v.w), acc[2 * r + 1]);
      }
    }
    const float bo = bias[o];
    float4* y = reinterpret_cast<float4*>(out + o * LD + r0);
#pragma unroll
    for (int r = 0; r < R / 4; ++r) {
      float a0 = f2_lo(acc[2 * r]) + bo, a1 = f2_hi(acc[2 * r]) + bo;
      float a2 = f2_lo(acc[2 * r + 1]) + bo, a3 = f2_hi(acc[2 * r + 1]) + bo;
      if (relu) {
        a0 = fmaxf(a0, 0.f);
        a1 = fmaxf(a1, 0.f);
        a2 = fmaxf(a2, 0.f);
        a3 = fmaxf(a3, 0.f);
      }
      y[r] = make_float4(a0, a1, a2, a3);
    }
  }
}

__global__ void __launch_bounds__(128) head_kernel(DevParams P, Batch b, float* __restrict__ probs,
                                                   uint8_t* __restrict__ labels, float* __restrict__ logits,
                                                   float* __restrict__ emb) {
  extern __shared__ float4 sm4[];
  float* X = reinterpret_cast<float*>(sm4);  // [256][LD]
  float* Y = X + 256 * LD;                   // [128][LD]
  float* Z = Y + 128 * LD;                   // [F + 7][LD]
  __shared__ int nside[NS];
  const int H = P.H, F = P.F, tid = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.x * PB;
  const int npairs = (int)min((int64_t)PB, b.B - i0);
  if (tid < NS) nside[tid] = tid < 2 * npairs ? b.counts[2 * i0 + tid] : 0;
  __syncthreads();
  // pooled features, transposed (empty or padding sides -> 0)
  for (int idx = tid; idx < NS * H; idx += blockDim.x) {
    const int s = idx / H, j = idx - s * H;
    X[j * LD + s] = nside[s] > 0 ? b.pooled[(2 * i0 + s) * (int64_t)H + j] : 0.f;
  }
  __syncthreads();
  // S7 projection e = W_F m + b_F -> Z[0:F]: thread (o, row half)
  dense_t<NS / 2>(P.wfT, P.bf, H, F, X, (tid >> 6) * (NS / 2), Z, false, tid & 63, 64);
  __syncthreads();
  // z = [e (0 if empty); canonical q; t]
  if (tid < NS) {
    const int s = tid;
    if (nside[s] == 0)
      for (int j = 0; j < F; ++j) Z[j * LD + s] = 0.f;
    float zq[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
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
      for (int c = 0; c < 4; ++c) zq[c] = __double2float_rn(sg * q[c]);
      for (int c = 0; c < 3; ++c) zq[4 + c] = pose[4 + c];
    }
    for (int c = 0; c < 7; ++c) Z[(F + c) * LD + s] = zq[c];
  }
  __syncthreads();
  if (emb)
    for (int idx = tid; idx < 2 * npairs * F; idx += blockDim.x) {
      const int s = idx / F, j = idx - s * F;
      emb[(2 * i0 + s) * (int64_t)F + j] = Z[j * LD + s];
    }
  // S8 object MLP (shared by both sides)
  dense_t<NS>(P.o1T, P.ob1, F + 7, kPredW, Z, 0, Y, true, tid, 128);
  __syncthreads();
  dense_t<NS>(P.o2T, P.ob2, kPredW, kPredW, Y, 0, X, true, tid, 128);
  __syncthreads();
  dense_t<NS>(P.o3T, P.ob3, kPredW, kPredW, X, 0, Y, true, tid, 128);
  __syncthreads();
  // S9 max across the pair -> X[o][p]
  for (int idx = tid; idx < PB * kPredW; idx += blockDim.x) {
    const int o = idx / PB, p = idx - o * PB;
    X[o * LD + p] = fmaxf(Y[o * LD + 2 * p], Y[o * LD + 2 * p + 1]);
  }
  __syncthreads();
  dense_t<PB>(P.p1T, P.pb1, kPredW, kPredW, X, 0, Y, true, tid, 128);
  __syncthreads();
  dense_t<PB>(P.p2T, P.pb2, kPredW, kPredW, Y, 0, X, true, tid, 128);
  __syncthreads();
  dense_t<PB>(P.p3T, P.pb3, kPredW, kPredW, X, 0, Y, true, tid, 128);
  __syncthreads();
  // output unit + sigmoid
  if (tid < npairs) {
    const int p = tid;
    float acc = 0.f;
    for (int j = 0; j < kPredW; ++j) acc = fmaf(P.wout[j], Y[j * LD + p], acc);
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

}  // namespace

cudaError_t launch_head(const DevParams& P, const Batch& b, float* probs, uint8_t* labels, float* logits, float* emb,
                        cudaStream_t st) {
  if (b.B == 0) return cudaSuccess;
  const size_t sm = sizeof(float) * (size_t)(256 + 128 + P.F + 7) * LD;
  static const cudaError_t attr = cudaFuncSetAttribute(head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       (int)(sizeof(float) * (256 + 128 + 256 + 7) * LD));
  if (attr != cudaSuccess) return attr;
  head_kernel<<<(unsigned)((b.B + PB - 1) / PB), 128, sm, st>>>(P, b, probs, labels, logits, emb);
  return cudaGetLastError();
}

}  // namespace locc
