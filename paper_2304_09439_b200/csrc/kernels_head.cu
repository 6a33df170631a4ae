// kernels_head.cu — S7 projection + S8-S9 collision predictor, fp32 on CUDA cores.
//
// Per pair: e_s = W_F m_s + b_F (one linear layer to F; e_s = 0
// for an empty crop); z_s = [e_s ; canonical unit quaternion ; translation]
// (reading Q12); u_s = ReLU^3 of the shared 3x128 object MLP; v = max(u_A, u_B) ("max-pooling
// across object pairs"); 3x128 ReLU; linear; sigmoid; label = p > 0.5.  Both crops empty ->
// short-circuit: p = 0, label 0, logit -inf.
//
// head_tile_kernel: one 256-thread block per 64 pairs (128 sides), all layers fused.  Activations
// stay in shared memory, transposed ([feature][row]); every layer is a small fp32 GEMM with a
// register tile of RT rows x 8 outputs per thread (64 or 32 independent FFMAs per k) and the
// layer's weights streamed through shared memory in 32-row chunks (register double buffer), so a
// weight is fetched once per 128 (or 64) rows.  head_kernel is the generic fallback (any H, F).
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

// ------------------------------------------------------------------ fused tile kernel (H = 256, F = 64)
constexpr int kTP = 64;           // pairs per block
constexpr int kTS = 2 * kTP;      // sides per block
constexpr int kLD = kTS + 4;      // row stride (floats) of the transposed activation buffers
constexpr int kKC = 32;           // weight rows per staged chunk
constexpr int kHeadThreads = 256;

struct HeadSmem {
  float u[128][kLD];   // activations, ping (u and v together: the projection's 256-feature input)
  float v[128][kLD];   // activations, pong
  float z[72][kLD];    // z = [e ; q ; t] per side
  float w[2][kKC][128];  // weight chunks
  int nside[kTS];
};

// out[n][r] = act(sum_k W[k][n] in[k][r] + b[n]), r < ROWS, n < N; W = transposed weights [K][N]
// (global, row-major).  in / out: [feature][kLD] shared buffers.  RT rows x 8 outputs per thread.
// kMode 0: forward (+ bias, optional ReLU).  Reverse mode (NEXT-2): 1 = no bias; 2 = no bias and the
// result multiplied by the ReLU mask bit of the layer below (mask [N][ROWS / 32] words, bit r of row r).
template <int ROWS, int N, bool kRelu, int kMode = 0>
__device__ __forceinline__ void dense(const float* __restrict__ W, const float* __restrict__ bias, int K,
                                      const float (*in)[kLD], float (*out)[kLD], float (*ws)[kKC][128],
                                      const uint32_t* __restrict__ mask = nullptr) {
  constexpr int CG = N / 8;                  // column groups
  constexpr int RG = kHeadThreads / CG;      // row groups
  constexpr int RT = ROWS / RG;              // rows per thread
  static_assert(RT % 4 == 0 && RT * RG == ROWS, "tile");
  const int tid = threadIdx.x;
  const int c0 = (tid % CG) * 8, r0 = (tid / CG) * RT;
  unsigned long long acc[RT][4];  // (column 2j, column 2j+1) per row, packed for FFMA2
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0ull;
  // weight chunk kc: rows [32kc, 32kc+32) x N floats, N / 4 float4 per row
  constexpr int F4 = kKC * N / 4;            // float4 per chunk
  constexpr int PER = (F4 + kHeadThreads - 1) / kHeadThreads;
  const int nchunks = (K + kKC - 1) / kKC;
  float4 pre[PER];
  auto fetch = [&](int kc) {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = tid + i * kHeadThreads;
      const int row = e / (N / 4), col4 = e % (N / 4);
      const int k = kc * kKC + row;
      pre[i] = (e < F4 && k < K) ? __ldg(reinterpret_cast<const float4*>(W + (int64_t)k * N) + col4)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = tid + i * kHeadThreads;
      if (e < F4) *reinterpret_cast<float4*>(&ws[buf][e / (N / 4)][4 * (e % (N / 4))]) = pre[i];
    }
  };
  fetch(0);
  stash(0);
  __syncthreads();
  for (int kc = 0; kc < nchunks; ++kc) {
    const int buf = kc & 1;
    if (kc + 1 < nchunks) fetch(kc + 1);  // in flight while this chunk is consumed
    const int kn = min(kKC, K - kc * kKC);
    // operands of step kk + 1 are loaded while step kk is multiplied (shared-memory latency hidden)
    float4 xa[RT / 4], wa, wb;
    auto load = [&](int kk) {
      const int k = kc * kKC + kk;
#pragma unroll
      for (int r = 0; r < RT; r += 4) xa[r / 4] = *reinterpret_cast<const float4*>(&in[k][r0 + r]);
      wa = *reinterpret_cast<const float4*>(&ws[buf][kk][c0]);
      wb = *reinterpret_cast<const float4*>(&ws[buf][kk][c0 + 4]);
    };
    load(0);
#pragma unroll 2
    for (int kk = 0; kk < kn; ++kk) {
      float a[RT];
#pragma unroll
      for (int r = 0; r < RT; r += 4) {
        a[r] = xa[r / 4].x;
        a[r + 1] = xa[r / 4].y;
        a[r + 2] = xa[r / 4].z;
        a[r + 3] = xa[r / 4].w;
      }
      const unsigned long long w2[4] = {f2(wa.x, wa.y), f2(wa.z, wa.w), f2(wb.x, wb.y), f2(wb.z, wb.w)};
      if (kk + 1 < kn) load(kk + 1);
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        const unsigned long long a2 = f2(a[r], a[r]);
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = ffma2(a2, w2[c], acc[r][c]);
      }
    }
    if (kc + 1 < nchunks) stash(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float b = kMode == 0 ? bias[c0 + c] : 0.f;
#pragma unroll
    for (int r = 0; r < RT; r += 4) {
      float v4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v4[q] = ((c & 1) ? f2_hi(acc[r + q][c >> 1]) : f2_lo(acc[r + q][c >> 1])) + b;
      if (kMode == 2) {
        const uint32_t mw = mask[(c0 + c) * (ROWS / 32) + ((r0 + r) >> 5)] >> ((r0 + r) & 31);
#pragma unroll
        for (int q = 0; q < 4; ++q) v4[q] = (mw >> q) & 1u ? v4[q] : 0.f;
      }
      float4 y = make_float4(v4[0], v4[1], v4[2], v4[3]);
      if (kRelu) y = make_float4(fmaxf(y.x, 0.f), fmaxf(y.y, 0.f), fmaxf(y.z, 0.f), fmaxf(y.w, 0.f));
      *reinterpret_cast<float4*>(&out[c0 + c][r0 + r]) = y;
    }
  }
  __syncthreads();
}

// NEXT-2 reverse mode: ReLU masks of the forward (bit r of word [feature][r / 32] = row r's activation
// > 0) and the side the max across the pair selected (bit p = u_A > u_B, ties -> B as the forward).
struct GradMasks {
  uint32_t obj[3][128][kTS / 32];   // a1, a2, u per side
  uint32_t pair[3][128][kTP / 32];  // c1, c2, c3 per pair
  uint32_t selA[128][kTP / 32];
};
struct HeadGradSmem {
  HeadSmem h;
  GradMasks m;
};

// mask[f][w] bit l = buf[f][32w + l] > 0, f < 128, rows < ROWS (one ballot per word).
template <int ROWS>
__device__ __forceinline__ void record_mask(const float (*buf)[kLD], uint32_t (*mask)[ROWS / 32]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = warp; i < 128 * (ROWS / 32); i += kHeadThreads / 32) {
    const int f = i / (ROWS / 32), w = i % (ROWS / 32);
    const uint32_t bits = __ballot_sync(0xffffffffu, buf[f][32 * w + lane] > 0.f);
    if (lane == 0) mask[f][w] = bits;
  }
}

// NEXT-2: d logit / d [q_A, t_A, q_B, t_B] by reverse mode through the predictor (oracle:
// head_grad).  On entry S.u holds c3 (pair layer 3 output) and the forward masks are recorded.
// Each backward layer is dense<> over the original [out][in] weights (= the transpose of the
// forward's), masked by the ReLU of the layer below; the object MLP's first layer only needs its
// 7 pose columns (o1p [7][128]).  Quaternion: dq = s (dq^ - q^ (q^ . dq^)) / |q| (fp64 q^, |q|).
__device__ __forceinline__ void head_tile_backward(const DevParams& P, const Batch& b, HeadSmem& S,
                                                   const GradMasks& GM, int64_t i0, int npairs,
                                                   float* __restrict__ grad) {
  const int tid = threadIdx.x;
  __syncthreads();  // the output stage read S.u
  for (int e = tid; e < 128 * kTP; e += kHeadThreads) {  // d/d pre3 (pair) = w_out [c3 > 0]
    const int n = e / kTP, p = e % kTP;
    S.v[n][p] = (GM.pair[2][n][p >> 5] >> (p & 31)) & 1u ? __ldg(P.wout + n) : 0.f;
  }
  __syncthreads();
  dense<kTP, 128, false, 2>(P.p3, nullptr, 128, S.v, S.u, S.w, &GM.pair[1][0][0]);  // d/d pre2 (pair)
  dense<kTP, 128, false, 2>(P.p2, nullptr, 128, S.u, S.v, S.w, &GM.pair[0][0][0]);  // d/d pre1 (pair)
  dense<kTP, 128, false, 1>(P.p1, nullptr, 128, S.v, S.u, S.w);                     // d/d v
  for (int e = tid; e < 128 * kTS; e += kHeadThreads) {  // d/d pre3 (object) per side
    const int n = e / kTS, s = e % kTS, p = s >> 1;
    const bool selA = (GM.selA[n][p >> 5] >> (p & 31)) & 1u;
    const bool pos = (GM.obj[2][n][s >> 5] >> (s & 31)) & 1u;
    S.v[n][s] = (pos && (selA == ((s & 1) == 0))) ? S.u[n][p] : 0.f;
  }
  __syncthreads();
  dense<kTS, 128, false, 2>(P.o3, nullptr, 128, S.v, S.u, S.w, &GM.obj[1][0][0]);  // d/d pre2 (object)
  dense<kTS, 128, false, 2>(P.o2, nullptr, 128, S.u, S.v, S.w, &GM.obj[0][0][0]);  // d/d pre1 (object)
  // d/d z[F + c] = sum_o O1[o][F + c] g[o]: side s = tid & 127, components c = tid >> 7, +2, ...
  {
    const int s = tid & (kTS - 1);
    for (int c = tid >> 7; c < 7; c += kHeadThreads / kTS) {
      const float* w = P.o1p + c * 128;
      float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
      for (int o = 0; o < 128; o += 2) {
        a0 = fmaf(__ldg(w + o), S.v[o][s], a0);
        a1 = fmaf(__ldg(w + o + 1), S.v[o + 1][s], a1);
      }
      S.z[c][s] = a0 + a1;
    }
  }
  __syncthreads();
  if (tid < 2 * npairs) {
    const int s = tid;
    const int64_t side = 2 * i0 + s;
    float* g = grad + side * 7;
    if (S.nside[s & ~1] + S.nside[s | 1] == 0) {
      for (int c = 0; c < 7; ++c) g[c] = 0.f;  // short-circuit: constant logit
    } else {
      const float* pose = b.poses + side * 7;
      const double q[4] = {pose[0], pose[1], pose[2], pose[3]};
      const double n = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
      double sg = 1.0;
      for (int c = 0; c < 4; ++c)
        if (q[c] != 0.0) {
          sg = q[c] > 0.0 ? 1.0 : -1.0;
          break;
        }
      double qh[4], dot = 0.0;
      for (int c = 0; c < 4; ++c) {
        qh[c] = sg * q[c] / n;
        dot += qh[c] * (double)S.z[c][s];
      }
      for (int c = 0; c < 4; ++c) g[c] = (float)(sg * ((double)S.z[c][s] - qh[c] * dot) / n);
      for (int c = 4; c < 7; ++c) g[c] = S.z[c][s];
    }
  }
}

template <bool kGrad, bool kEmbIn>
__global__ void __launch_bounds__(kHeadThreads, 1) head_tile_kernel(DevParams P, Batch b, float* __restrict__ probs,
                                                                    uint8_t* __restrict__ labels,
                                                                    float* __restrict__ logits, float* __restrict__ emb,
                                                                    float* __restrict__ grad) {
  extern __shared__ float4 smem4[];
  HeadSmem& S = *reinterpret_cast<HeadSmem*>(smem4);
  GradMasks& GM = reinterpret_cast<HeadGradSmem*>(smem4)->m;  // only touched when kGrad
  const int tid = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.x * kTP;
  const int npairs = (int)min((int64_t)kTP, b.B - i0);
  if (tid < kTS) S.nside[tid] = tid < 2 * npairs ? b.counts[2 * i0 + tid] : 0;
  // z rows F..F+6: canonical unit quaternion and translation per side (fp64 normalisation, Q12)
  if (tid < kTS) {
    const int s = tid;
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
    for (int c = 0; c < 7; ++c) S.z[64 + c][s] = zq[c];
    S.z[71][s] = 0.f;
  }
  if constexpr (kEmbIn) {
    // encode-once mode (NEXT-1): e is the selection's pooled cell embedding, [G][64]
    __syncthreads();  // nside
    for (int e = tid; e < kTS * 16; e += kHeadThreads) {
      const int s = e >> 4, j4 = e & 15;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (S.nside[s] > 0) x = __ldg(reinterpret_cast<const float4*>(b.emb_in + (2 * i0 + s) * (int64_t)64) + j4);
      S.z[4 * j4][s] = x.x;
      S.z[4 * j4 + 1][s] = x.y;
      S.z[4 * j4 + 2][s] = x.z;
      S.z[4 * j4 + 3][s] = x.w;
    }
  } else {
  // S7 projection e = W_F m + b_F: the pooled rows (256 features) are staged transposed into u..v
  // (contiguous: one [256][kLD] buffer); empty and padding sides read as 0
    float (*m)[kLD] = reinterpret_cast<float (*)[kLD]>(&S.u[0][0]);  // u and v are contiguous
    __syncthreads();  // nside
#pragma unroll 1
    for (int e0 = 0; e0 < kTS * 64; e0 += 8 * kHeadThreads) {  // 8 loads in flight per thread
      float4 x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = e0 + i * kHeadThreads + tid, s = e / 64, j4 = e % 64;
        x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (S.nside[s] > 0) {
          x[i] = __ldg(reinterpret_cast<const float4*>(b.pooled + (2 * i0 + s) * (int64_t)256) + j4);
          if (b.cells_c) {  // the tensor-core encoder leaves cell sums: m = S / C
            const float c = (float)b.cells_c[2 * i0 + s], rc = __frcp_rn(c);
            x[i] = make_float4(div_count(x[i].x, c, rc), div_count(x[i].y, c, rc), div_count(x[i].z, c, rc),
                               div_count(x[i].w, c, rc));
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = e0 + i * kHeadThreads + tid, s = e / 64, j4 = e % 64;
        m[4 * j4][s] = x[i].x;
        m[4 * j4 + 1][s] = x[i].y;
        m[4 * j4 + 2][s] = x[i].z;
        m[4 * j4 + 3][s] = x[i].w;
      }
    }
    __syncthreads();
    dense<kTS, 64, false>(P.wfT, P.bf, 256, m, S.z, S.w);
  }
  // e = 0 for empty sides; debug copy
  for (int e = tid; e < 64 * kTS; e += kHeadThreads) {
    const int j = e / kTS, s = e % kTS;
    if (S.nside[s] == 0) S.z[j][s] = 0.f;
  }
  __syncthreads();
  if (emb)
    for (int e = tid; e < 2 * npairs * 64; e += kHeadThreads) {
      const int s = e / 64, j = e % 64;
      emb[(2 * i0 + s) * (int64_t)64 + j] = S.z[j][s];
    }
  // S8 object MLP (shared by both sides)
  dense<kTS, 128, true>(P.o1T, P.ob1, 71, S.z, S.u, S.w);
  if (kGrad) record_mask<kTS>(S.u, GM.obj[0]);
  dense<kTS, 128, true>(P.o2T, P.ob2, 128, S.u, S.v, S.w);
  if (kGrad) record_mask<kTS>(S.v, GM.obj[1]);
  dense<kTS, 128, true>(P.o3T, P.ob3, 128, S.v, S.u, S.w);
  if (kGrad) {
    record_mask<kTS>(S.u, GM.obj[2]);
    const int warp = tid >> 5, lane = tid & 31;
    for (int i = warp; i < 128 * (kTP / 32); i += kHeadThreads / 32) {
      const int o = i / (kTP / 32), w = i % (kTP / 32), p = 32 * w + lane;
      const uint32_t bits = __ballot_sync(0xffffffffu, S.u[o][2 * p] > S.u[o][2 * p + 1]);
      if (lane == 0) GM.selA[o][w] = bits;
    }
  }
  // S9 max across the pair -> v[o][p]
  for (int e = tid; e < 128 * kTP; e += kHeadThreads) {
    const int o = e / kTP, p = e % kTP;
    S.v[o][p] = fmaxf(S.u[o][2 * p], S.u[o][2 * p + 1]);
  }
  __syncthreads();
  dense<kTP, 128, true>(P.p1T, P.pb1, 128, S.v, S.u, S.w);
  if (kGrad) record_mask<kTP>(S.u, GM.pair[0]);
  dense<kTP, 128, true>(P.p2T, P.pb2, 128, S.u, S.v, S.w);
  if (kGrad) record_mask<kTP>(S.v, GM.pair[1]);
  dense<kTP, 128, true>(P.p3T, P.pb3, 128, S.v, S.u, S.w);
  if (kGrad) record_mask<kTP>(S.u, GM.pair[2]);
  // output unit: 4 threads per pair, 32 features each, then combined
  {
    const int p = tid >> 2, part = tid & 3;
    float acc = 0.f;
    for (int j = 32 * part; j < 32 * part + 32; ++j) acc = fmaf(P.wout[j], S.u[j][p], acc);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (part == 0 && p < npairs) {
      const int64_t i = i0 + p;
      float lg, pr;
      if (S.nside[2 * p] + S.nside[2 * p + 1] == 0) {
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
  if constexpr (kGrad) head_tile_backward(P, b, S, GM, i0, npairs, grad);
}

// ------------------------------------------------------------------ generic fallback (any H, F)
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
  if (b.emb_in) {  // encode-once mode: e is the selection's pooled cell embedding [G][F]
    for (int idx = tid; idx < NS * F; idx += blockDim.x) {
      const int s = idx / F, j = idx - s * F;
      Z[j * LD + s] = nside[s] > 0 ? b.emb_in[(2 * i0 + s) * (int64_t)F + j] : 0.f;
    }
  } else {
    for (int idx = tid; idx < NS * H; idx += blockDim.x) {
      const int s = idx / H, j = idx - s * H;
      X[j * LD + s] = nside[s] > 0 ? (b.cells_c ? __fdiv_rn(b.pooled[(2 * i0 + s) * (int64_t)H + j],
                                                             (float)b.cells_c[2 * i0 + s])
                                                  : b.pooled[(2 * i0 + s) * (int64_t)H + j])
                                   : 0.f;  // (head_kernel: configurations other than H = 256, F = 64)
    }
    __syncthreads();
    dense_t<NS / 2>(P.wfT, P.bf, H, F, X, (tid >> 6) * (NS / 2), Z, false, tid & 63, 64);
  }
  __syncthreads();
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
  dense_t<NS>(P.o1T, P.ob1, F + 7, kPredW, Z, 0, Y, true, tid, 128);
  __syncthreads();
  dense_t<NS>(P.o2T, P.ob2, kPredW, kPredW, Y, 0, X, true, tid, 128);
  __syncthreads();
  dense_t<NS>(P.o3T, P.ob3, kPredW, kPredW, X, 0, Y, true, tid, 128);
  __syncthreads();
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
                        float* grad, cudaStream_t st) {
  if (b.B == 0) return cudaSuccess;
  if (P.H == 256 && P.F == 64) {
    const unsigned grid = (unsigned)((b.B + kTP - 1) / kTP);
    const cudaError_t attr = [] {  // once per (device, kernel), see smem_optin
      const size_t g = sizeof(HeadGradSmem), f = sizeof(HeadSmem);
      cudaError_t e = smem_optin(head_tile_kernel<true, true>, g);
      if (e == cudaSuccess) e = smem_optin(head_tile_kernel<true, false>, g);
      if (e == cudaSuccess) e = smem_optin(head_tile_kernel<false, true>, f);
      if (e == cudaSuccess) e = smem_optin(head_tile_kernel<false, false>, f);
      return e;
    }();
    if (attr != cudaSuccess) return attr;
    auto run = [&](auto kern, size_t sm, float* g) {
      kern<<<grid, kHeadThreads, sm, st>>>(P, b, probs, labels, logits, emb, g);
      return cudaGetLastError();
    };
    if (grad)
      return b.emb_in ? run(head_tile_kernel<true, true>, sizeof(HeadGradSmem), grad)
                      : run(head_tile_kernel<true, false>, sizeof(HeadGradSmem), grad);
    if (b.emb_in) return run(head_tile_kernel<false, true>, sizeof(HeadSmem), nullptr);
    return run(head_tile_kernel<false, false>, sizeof(HeadSmem), nullptr);
  }
  if (grad) return cudaErrorNotSupported;  // the pose gradient is built for H = 256, F = 64
  const size_t sm = sizeof(float) * (size_t)(256 + 128 + P.F + 7) * LD;
  const cudaError_t attr2 = smem_optin(head_kernel, sizeof(float) * (256 + 128 + 256 + 7) * LD);
  if (attr2 != cudaSuccess) return attr2;
  head_kernel<<<(unsigned)((b.B + PB - 1) / PB), 128, sm, st>>>(P, b, probs, labels, logits, emb);
  return cudaGetLastError();
}

}  // namespace locc
