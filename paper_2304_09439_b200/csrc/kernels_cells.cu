// kernels_cells.cu — NEXT-1: the paper's own encode-once inference (DESIGN.md
// readings Q27-Q30).  Each shape is encoded ONCE into an M x M x M x F embedding grid (PAPER.md:331-333,
// :421-422); a query then only selects the cells near the other object and average-pools their
// embeddings, so its cost does not depend on K.
//
//   grid_encode_kernel   point MLP over all K points of a shape, cell-wise max -> G [S][M^3][H] (fp32
//                        contexts; bf16 contexts: 2 x 2 tensor-core GEMMs, layer 1 fused -> cell_max)
//   conv3d_kernel        one 3x3x3 layer of the U-Net as an implicit GEMM (fp32 FFMA2): rows = output
//                        positions of one shape, columns = 128 output channels, K = 27 taps x C_in
//                        (two inputs = the concatenation skip); deconv layers run as the equivalent
//                        conv (flipped taps, padding 2 - p) — the same sums, in another order
//   unet_tail_kernel     global average of the last conv, [d1 ; g] -> linear F, and the
//                        cell centres used by the selection
//   cells_select_kernel  per (pair, side): the O4 distance test on the M^3 cell centres with the own
//                        cell's half diagonal as margin, selection bits, mean of the selected rows of E
// The predictor is head_tile_kernel reading e from the selection (Batch::emb_in).
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <stdint.h>

#include "geom.cuh"
#include "internal.h"
#include "point_mlp.cuh"
#include "tc_ptx.cuh"

namespace locc {
namespace {

using tc::f2;
using tc::f2_hi;
using tc::f2_lo;
using tc::ffma2;

// ---------------------------------------------------------------- Q27: cell-max grid of every shape
// One block per shape, thread f = feature f.  The shape's points are cell-sorted (S0), so the cell-wise
// max is a running max closed at each cell change; ReLU(max + b3) = max of ReLU(acc + b3).  Empty cells
// stay 0 (the buffer is cleared first).
__global__ void __launch_bounds__(256, 2) grid_encode_kernel(DevParams P, ShapeTable T, int M, float* __restrict__ G) {
  extern __shared__ float4 smem4[];
  float4* rows_s = smem4;                                // [64]
  float* hT = reinterpret_cast<float*>(smem4 + kMlpTR);  // [H][kMlpLDH]
  __shared__ int next_cell;
  const int H = P.H, f = threadIdx.x, s = blockIdx.x;
  const bool act = f < H;
  float4 w1 = make_float4(0.f, 0.f, 0.f, 0.f);
  float b3 = 0.f;
  if (act) {
    w1 = P.w1b[f];
    b3 = P.b3[f];
  }
  const float4* pts = T.pts + (int64_t)s * T.K;
  float* Gs = G + (int64_t)s * M * M * M * H;
  float run_max = -INFINITY;
  for (int t0 = 0; t0 < T.K; t0 += kMlpTR) {
    const int nr = min(kMlpTR, T.K - t0);
    if (f < kMlpTR) rows_s[f] = f < nr ? pts[t0 + f] : make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
    if (f == 0) next_cell = t0 + kMlpTR < T.K ? __float_as_int(pts[t0 + kMlpTR].w) : -1;
    __syncthreads();
    point_mlp_tile(P, rows_s, hT, w1, f, act);
    const float* acc = hT + f * kMlpLDH;  // feature f's layer-3 accumulators of the tile's rows
    if (act) {
#pragma unroll 4
      for (int r = 0; r < kMlpTR; ++r) {
        if (r < nr) {
          run_max = fmaxf(run_max, acc[r]);
          const int cell = __float_as_int(rows_s[r].w);
          const int nxt = r + 1 < nr ? __float_as_int(rows_s[r + 1].w) : next_cell;
          if (nxt != cell) {
            Gs[(int64_t)cell * H + f] = fmaxf(run_max + b3, 0.f);
            run_max = -INFINITY;
          }
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- Q27 on the tensor cores (bf16 contexts)
// The same grid as grid_encode_kernel, layer by layer over a chunk of shapes (all their points as flat
// rows): layers 2 and 3 as 3xTF32 GEMMs on tcgen05 (launch_gemm_tc, kernels_conv_tc.cu; layer 2's A
// rows are h1 = ReLU(W1 p + b1), K = 3, computed in its producers), then cell_max_kernel: per shape and feature, the running
// max over the cell-sorted points, closed at each cell change.  h3 = ReLU(acc + b3) >= 0, so the max of
// h3 equals ReLU(max acc + b3) and empty cells keep the cleared 0.
__global__ void __launch_bounds__(256) cell_max_kernel(const float* __restrict__ h3, const float4* __restrict__ pts,
                                                       int K, int nc, float* __restrict__ G) {
  const int f = threadIdx.x;
  const float* hs = h3 + (int64_t)blockIdx.x * K * 256 + f;
  const float4* ps = pts + (int64_t)blockIdx.x * K;
  float* Gs = G + (int64_t)blockIdx.x * nc * 256 + f;
  if (K == 0) return;
  int cell = __float_as_int(__ldg(&ps[0].w));
  float run = 0.f;
  for (int r0 = 0; r0 < K; r0 += 8) {
    float v[8];
    int cl[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = r0 + u;
      v[u] = r < K ? __ldg(hs + (int64_t)r * 256) : 0.f;
      cl[u] = r < K ? __float_as_int(__ldg(&ps[r].w)) : -1;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (cl[u] < 0) break;  // past the shape's last point
      if (cl[u] != cell) {
        Gs[(int64_t)cell * 256] = run;
        run = 0.f;
        cell = cl[u];
      }
      run = fmaxf(run, v[u]);
    }
  }
  Gs[(int64_t)cell * 256] = run;
}

// ---------------------------------------------------------------- Q28: U-Net layers (implicit GEMM)
constexpr int kCvBM = 64;   // output positions per block
constexpr int kCvBK = 32;   // input channels per staged chunk
constexpr int kCvLDA = kCvBM + 4;
constexpr size_t kCvSmem = sizeof(float) * 2 * kCvBK * (kCvLDA + 128);

struct ConvArgs {
  const float* x1;  // [S][Di^3][C1]
  const float* x2;  // [S][Di^3][C2] or null (channels C1.. of the concatenation)
  int C1, C2;
  int Di, Do, pad;  // y[q] = sum_k x[q + k - pad] (taps k = kx + 3 (ky + 3 kz))
  const float* Wt;  // [27][C1 + C2][128]
  const float* bias;
  float* y;         // [S][Do^3][128], ReLU applied
};

__global__ void __launch_bounds__(256) conv3d_kernel(ConvArgs a) {
  extern __shared__ float4 cv_smem[];
  float (*As)[kCvBK][kCvLDA] = reinterpret_cast<float (*)[kCvBK][kCvLDA]>(cv_smem);  // [2][ci][position]
  float (*Bs)[kCvBK][128] = reinterpret_cast<float (*)[kCvBK][128]>(
      reinterpret_cast<float*>(cv_smem) + 2 * kCvBK * kCvLDA);                       // [2][ci][out channel]
  const int tid = threadIdx.x, s = blockIdx.y, q0 = blockIdx.x * kCvBM;
  const int Cin = a.C1 + a.C2, Di3 = a.Di * a.Di * a.Di, nq = a.Do * a.Do * a.Do;
  const int c0 = (tid & 15) * 8, r0 = (tid >> 4) * 4;  // 4 positions x 8 channels per thread
  unsigned long long acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0ull;
  // the two positions this thread gathers (one float4 of 4 channels each) per chunk
  int gq[2], gc4[2], gz[2], gy[2], gx[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int e = tid + 256 * i;
    gq[i] = e >> 3;
    gc4[i] = e & 7;
    const int q = q0 + gq[i];
    gx[i] = q % a.Do;
    gy[i] = (q / a.Do) % a.Do;
    gz[i] = q < nq ? q / (a.Do * a.Do) : -1000;
  }
  const int nci = Cin / kCvBK, nchunks = 27 * nci;
  float4 pa[2], pb[4];
  auto fetch = [&](int ch) {
    const int k = ch / nci, ci0 = (ch - k * nci) * kCvBK;
    const int kx = k % 3 - a.pad, ky = (k / 3) % 3 - a.pad, kz = k / 9 - a.pad;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int ix = gx[i] + kx, iy = gy[i] + ky, iz = gz[i] + kz;
      pa[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ix >= 0 && iy >= 0 && iz >= 0 && ix < a.Di && iy < a.Di && iz < a.Di) {
        const int64_t pos = (int64_t)s * Di3 + (iz * a.Di + iy) * a.Di + ix;
        const int ci = ci0 + 4 * gc4[i];
        pa[i] = ci < a.C1 ? __ldg(reinterpret_cast<const float4*>(a.x1 + pos * a.C1 + ci))
                          : __ldg(reinterpret_cast<const float4*>(a.x2 + pos * a.C2 + (ci - a.C1)));
      }
    }
    const float* w = a.Wt + ((int64_t)k * Cin + ci0) * 128;
#pragma unroll
    for (int i = 0; i < 4; ++i) pb[i] = __ldg(reinterpret_cast<const float4*>(w) + tid + 256 * i);
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int c = 4 * gc4[i];
      As[buf][c][gq[i]] = pa[i].x;
      As[buf][c + 1][gq[i]] = pa[i].y;
      As[buf][c + 2][gq[i]] = pa[i].z;
      As[buf][c + 3][gq[i]] = pa[i].w;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + 256 * i;
      *reinterpret_cast<float4*>(&Bs[buf][e >> 5][4 * (e & 31)]) = pb[i];
    }
  };
  fetch(0);
  stash(0);
  __syncthreads();
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nchunks) fetch(ch + 1);
#pragma unroll 4
    for (int kk = 0; kk < kCvBK; ++kk) {
      const float4 xa = *reinterpret_cast<const float4*>(&As[buf][kk][r0]);
      const float4 wa = *reinterpret_cast<const float4*>(&Bs[buf][kk][c0]);
      const float4 wb = *reinterpret_cast<const float4*>(&Bs[buf][kk][c0 + 4]);
      const unsigned long long w2[4] = {f2(wa.x, wa.y), f2(wa.z, wa.w), f2(wb.x, wb.y), f2(wb.z, wb.w)};
      const float xr[4] = {xa.x, xa.y, xa.z, xa.w};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const unsigned long long x2 = f2(xr[r], xr[r]);
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = ffma2(x2, w2[c], acc[r][c]);
      }
    }
    if (ch + 1 < nchunks) stash(buf ^ 1);
    __syncthreads();
  }
  float bias[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) bias[c] = __ldg(a.bias + c0 + c);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int q = q0 + r0 + r;
    if (q >= nq) continue;
    float v[8];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      v[2 * c] = fmaxf(f2_lo(acc[r][c]) + bias[2 * c], 0.f);
      v[2 * c + 1] = fmaxf(f2_hi(acc[r][c]) + bias[2 * c + 1], 0.f);
    }
    float4* yo = reinterpret_cast<float4*>(a.y + ((int64_t)s * nq + q) * 128 + c0);
    yo[0] = make_float4(v[0], v[1], v[2], v[3]);
    yo[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}

// ---------------------------------------------------------------- Q28 tail + Q29 cell centres
// g = mean over the (M-2)^3 positions of c4 ("average pooling ... global feature");
// E[c] = W_P [d1[c] ; g] + b_P; cell centres lo + (i + 1/2) ext / M in fp64, rounded once.
__global__ void __launch_bounds__(256) unet_tail_kernel(UNetParams U, ShapeTable T, int M, int F, int global_max,
                                                        const float* __restrict__ c4, const float* __restrict__ d1,
                                                        float* __restrict__ E, float* __restrict__ ctr) {
  extern __shared__ float sm[];
  float* pW = sm;                  // [F][257] (padded: thread f reads row f)
  float* g = pW + (size_t)F * 257;  // [128]
  float* gb = g + 128;             // [F]
  const int s = blockIdx.x, tid = threadIdx.x, nc = M * M * M, D = M - 2, n4 = D * D * D;
  for (int e = tid; e < F * 256; e += 256) pW[(e >> 8) * 257 + (e & 255)] = U.pW[e];
  if (tid < 128) {  // global feature: average (default) or max of the last conv layer
    float acc = 0.f;
    const float* x = c4 + (int64_t)s * n4 * 128 + tid;
    if (global_max) {
      for (int q = 0; q < n4; ++q) acc = fmaxf(acc, x[(int64_t)q * 128]);  // c4 >= 0 (ReLU)
      g[tid] = acc;
    } else {
      for (int q = 0; q < n4; ++q) acc += x[(int64_t)q * 128];
      g[tid] = __fdiv_rn(acc, (float)n4);
    }
  }
  __syncthreads();
  if (tid < F) {
    float acc = U.pb[tid];
    for (int j = 0; j < 128; ++j) acc = fmaf(pW[tid * 257 + 128 + j], g[j], acc);
    gb[tid] = acc;
  }
  __syncthreads();
  // thread (f, group): 4 cells at a time, so each weight read from shared memory feeds 4 FMAs; the d1
  // rows are read by all threads of a feature group alike (L1 broadcast)
  const int ngrp = 256 / F;
  for (int e = tid; e < ngrp * F; e += 256) {
    const int grp = e / F, f = e - grp * F;
    const float* w = pW + f * 257;
    for (int c0 = 4 * grp; c0 < nc; c0 += 4 * ngrp) {
      const float4* x[4];
      float a0[4], a1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[u] = reinterpret_cast<const float4*>(d1 + ((int64_t)s * nc + min(c0 + u, nc - 1)) * 128);
        a0[u] = a1[u] = 0.f;
      }
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        const float w0 = w[4 * j], w1 = w[4 * j + 1], w2 = w[4 * j + 2], w3 = w[4 * j + 3];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 v = __ldg(x[u] + j);
          a0[u] = fmaf(w0, v.x, a0[u]);
          a1[u] = fmaf(w1, v.y, a1[u]);
          a0[u] = fmaf(w2, v.z, a0[u]);
          a1[u] = fmaf(w3, v.w, a1[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c0 + u < nc) E[((int64_t)s * nc + c0 + u) * F + f] = (a0[u] + a1[u]) + gb[f];
    }
  }
  // the centres are separable: per axis d the M values lo_d + (i + 1/2) ext_d / M -> ctr[s][8 d + i]
  const float4 lo = T.lo[s], hi = T.hi[s];
  if (tid < 24) {
    const int d = tid >> 3, i = tid & 7;
    const float l = d == 0 ? lo.x : d == 1 ? lo.y : lo.z, h = d == 0 ? hi.x : d == 1 ? hi.y : hi.z;
    const double ext = __dsub_rn((double)h, (double)l);
    ctr[(int64_t)s * 24 + tid] =
        i < M ? __double2float_rn(__dadd_rn((double)l, __ddiv_rn(__dmul_rn(__dadd_rn((double)i, 0.5), ext), (double)M)))
              : 0.f;
  }
}

// ---------------------------------------------------------------- Q29: selection + pooled embedding
// One warp per (pair, side) segment.  Cell c of the own shape is selected iff its centre, moved into the
// other object's frame with the crop's fp32 transform, is within the OWN cell half-diagonal of the other
// AABB (keep_point with eps^2 = own lo.w).  e = mean over the selected cells of E (fp32 sums).
// kM > 0: the grid edge as a compile-time constant (the index arithmetic of the M^3 centre tests
// becomes multiply-shifts); 0 = any M.
template <int kM>
__global__ void __launch_bounds__(256) cells_select_kernel(ShapeTable T, CellsTable C, Batch b, int F,
                                                           uint32_t* __restrict__ cells, float* __restrict__ emb) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= b.G) return;
  const int M = kM > 0 ? kM : C.M;
  const int nc = M * M * M, nw = (nc + 31) >> 5;
  int own = 0, other = 0;
  Xf X;
  float* e = emb + g * F;
  if (!segment_load(b, g, own, other, X)) {
    if (lane == 0) b.counts[g] = 0;
    for (int f = lane; f < F; f += 32) e[f] = 0.f;
    return;
  }
  LOCC_CHECK(nc <= 512 && (unsigned)own < (unsigned)T.S && (unsigned)other < (unsigned)T.S);
  float4 lo = T.lo[other];
  lo.w = T.lo[own].w;  // the own cell's half-diagonal squared as the margin
  const float4 hi = T.hi[other];
  const float axv = lane < 24 ? __ldg(C.ctr + (int64_t)own * 24 + lane) : 0.f;  // centre value per axis, index
  uint32_t words[16];
  int n = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    words[j] = 0u;
    if (j < nw) {
      const int c = 32 * j + lane;
      const int ix = c % M, iy = (c / M) % M, iz = c / (M * M);
      const float px = __shfl_sync(0xffffffffu, axv, ix & 7), py = __shfl_sync(0xffffffffu, axv, 8 + (iy & 7));
      const float pz = __shfl_sync(0xffffffffu, axv, 16 + (iz & 7));
      const bool keep = c < nc && keep_point(X, px, py, pz, lo, hi);
      words[j] = __ballot_sync(0xffffffffu, keep);
      n += __popc(words[j]);
    }
  }
  // mean of the selected rows (F = 64): the selected cell ids are listed in shared memory, then each
  // half-warp reads one row as 16 float4 (lane l: features 4 (l & 15) ..), 8 rows in flight per warp
  __shared__ uint16_t sel_list[8][512];
  uint16_t* list = sel_list[threadIdx.x >> 5];
  int at = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j < nw) {
      if ((words[j] >> lane) & 1u) list[at + __popc(words[j] & ((1u << lane) - 1u))] = (uint16_t)(32 * j + lane);
      at += __popc(words[j]);
    }
  }
  __syncwarp();
  if (F != 64) {  // any F <= 256: lane owns features lane, lane + 32, ...; rows in ascending order
    const float* Es = C.E + (int64_t)own * nc * F;
    for (int f0 = 0; f0 < F; f0 += 32) {
      const int f = f0 + lane;
      float a = 0.f;
      for (int i = 0; i < n; ++i) a = __fadd_rn(a, f < F ? __ldg(Es + (int64_t)list[i] * F + f) : 0.f);
      if (f < F) e[f] = n ? __fdiv_rn(a, (float)n) : 0.f;
    }
  } else {
  const float4* Es4 = reinterpret_cast<const float4*>(C.E + (int64_t)own * nc * 64);
  const int half = lane >> 4, f4 = lane & 15;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i0 = 0; i0 < n; i0 += 8) {
    float4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + 2 * j + half;
      v[j] = i < n ? __ldg(Es4 + (int)list[i] * 16 + f4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc.x = __fadd_rn(acc.x, v[j].x);
      acc.y = __fadd_rn(acc.y, v[j].y);
      acc.z = __fadd_rn(acc.z, v[j].z);
      acc.w = __fadd_rn(acc.w, v[j].w);
    }
  }
  acc.x = __fadd_rn(acc.x, __shfl_xor_sync(0xffffffffu, acc.x, 16));
  acc.y = __fadd_rn(acc.y, __shfl_xor_sync(0xffffffffu, acc.y, 16));
  acc.z = __fadd_rn(acc.z, __shfl_xor_sync(0xffffffffu, acc.z, 16));
  acc.w = __fadd_rn(acc.w, __shfl_xor_sync(0xffffffffu, acc.w, 16));
  if (half == 0) {
    const float fn = (float)n;
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (n) r = make_float4(__fdiv_rn(acc.x, fn), __fdiv_rn(acc.y, fn), __fdiv_rn(acc.z, fn), __fdiv_rn(acc.w, fn));
    reinterpret_cast<float4*>(e)[f4] = r;
  }
  }
  if (cells) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < nw && lane == j) cells[g * nw + j] = words[j];
  }
  if (lane == 0) {
    b.counts[g] = n;
    if (n) atomicAdd(&b.stats->nonempty_sides, 1ull);
  }
}

}  // namespace

cudaError_t launch_grid_encode(const DevParams& P, const ShapeTable& T, int M, float* G, cudaStream_t st) {
  const size_t sm = kMlpSmemBytes;
  const cudaError_t attr = smem_optin(grid_encode_kernel, sm);
  if (attr != cudaSuccess) return attr;
  cudaError_t e = cudaMemsetAsync(G, 0, sizeof(float) * (size_t)T.S * M * M * M * P.H, st);
  if (e != cudaSuccess) return e;
  grid_encode_kernel<<<T.S, 256, sm, st>>>(P, T, M, G);
  return cudaGetLastError();
}

// Rows per chunk of the tensor-core grid encode: whole shapes, about 2^20 rows (1 GiB per activation;
// LOCC_GRID_CHUNK=<rows> overrides, for the tests of the chunk boundaries).
int64_t grid_tc_chunk_rows(const ShapeTable& T) {
  const int64_t K = T.K > 0 ? T.K : 1;
  const char* env = getenv("LOCC_GRID_CHUNK");
  const int64_t target = env ? std::max<int64_t>(1, atoll(env)) : (int64_t(1) << 20);
  const int64_t spc = std::max<int64_t>(1, std::min<int64_t>(T.S, target / K));
  return spc * K;
}

cudaError_t launch_grid_encode_tc(const DevParams& P, const ShapeTable& T, int M, float* G, float* bufA, float* bufB,
                                  int num_sms, cudaStream_t st) {
  const int nc = M * M * M;
  cudaError_t e = cudaMemsetAsync(G, 0, sizeof(float) * (size_t)T.S * nc * 256, st);
  if (e != cudaSuccess || T.K == 0) return e;
  const int64_t spc = grid_tc_chunk_rows(T) / T.K;
  const uint8_t* w2 = P.grid_tc_img;
  const uint8_t* w3 = P.grid_tc_img + 16 * 32768;
  for (int64_t s0 = 0; s0 < T.S; s0 += spc) {
    const int64_t ns = std::min<int64_t>(spc, T.S - s0), rows = ns * T.K;
    const float4* pts = T.pts + s0 * T.K;
    for (int half = 0; half < 2; ++half)
      if ((e = launch_gemm_tc(nullptr, 256, rows, w2 + (size_t)half * 8 * 32768, P.b2 + 128 * half, bufB, 256,
                              128 * half, num_sms, st, pts, P.w1b)) != cudaSuccess)
        return e;
    for (int half = 0; half < 2; ++half)
      if ((e = launch_gemm_tc(bufB, 256, rows, w3 + (size_t)half * 8 * 32768, P.b3 + 128 * half, bufA, 256, 128 * half,
                              num_sms, st)) != cudaSuccess)
        return e;
    cell_max_kernel<<<(unsigned)ns, 256, 0, st>>>(bufA, pts, T.K, nc, G + (size_t)s0 * nc * 256);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Activation scratch of the U-Net: c1..c4, d4, d3, d2 [S][(M-2)^3][128] and d1 [S][M^3][128].
size_t unet_act_floats(int S, int M) {
  const size_t n4 = (size_t)(M - 2) * (M - 2) * (M - 2), n6 = (size_t)M * M * M;
  return (size_t)S * 128 * (7 * n4 + n6);
}

cudaError_t launch_unet(const UNetParams& U, const ShapeTable& T, int M, int H, int F, int global_max, const float* G,
                        float* act, float* E, float* ctr, bool tc, int num_sms, cudaStream_t st) {
  const int D = M - 2, S = T.S;
  const size_t n4 = (size_t)S * D * D * D * 128;
  float* c[4];
  for (int i = 0; i < 4; ++i) c[i] = act + i * n4;
  float* d4 = act + 4 * n4;
  float* d3 = act + 5 * n4;
  float* d2 = act + 6 * n4;
  float* d1 = act + 7 * n4;
  auto conv = [&](const float* x1, int C1, const float* x2, int C2, int Di, int Do, int pad, int l, float* y) {
    if (tc) return launch_conv_tc(x1, C1, x2, C2, Di, Do, pad, S, U.img[l], U.b[l], y, num_sms, st);
    ConvArgs a{x1, x2, C1, C2, Di, Do, pad, U.Wt[l], U.b[l], y};
    dim3 grid((unsigned)((Do * Do * Do + kCvBM - 1) / kCvBM), (unsigned)S);
    conv3d_kernel<<<grid, 256, kCvSmem, st>>>(a);
    return cudaGetLastError();
  };
  const cudaError_t attr0 = smem_optin(conv3d_kernel, kCvSmem);
  if (attr0 != cudaSuccess) return attr0;
  cudaError_t e;
  if ((e = conv(G, H, nullptr, 0, M, D, 0, 0, c[0])) != cudaSuccess) return e;        // valid
  for (int i = 1; i < 4; ++i)
    if ((e = conv(c[i - 1], 128, nullptr, 0, D, D, 1, i, c[i])) != cudaSuccess) return e;  // same
  // deconv (transposed, stride 1) with padding p == conv with flipped taps and padding 2 - p
  if ((e = conv(c[3], 128, nullptr, 0, D, D, 1, 4, d4)) != cudaSuccess) return e;
  if ((e = conv(d4, 128, c[2], 128, D, D, 1, 5, d3)) != cudaSuccess) return e;
  if ((e = conv(d3, 128, c[1], 128, D, D, 1, 6, d2)) != cudaSuccess) return e;
  if ((e = conv(d2, 128, c[0], 128, D, M, 2, 7, d1)) != cudaSuccess) return e;      // transposed valid
  const size_t sm = sizeof(float) * ((size_t)F * 257 + 128 + F);
  const cudaError_t attr = smem_optin(unet_tail_kernel, sizeof(float) * (64 * 257 + 128 + 64));
  if (attr != cudaSuccess) return attr;
  unet_tail_kernel<<<S, 256, sm, st>>>(U, T, M, F, global_max, c[3], d1, E, ctr);
  return cudaGetLastError();
}

cudaError_t launch_cells_select(const ShapeTable& T, const CellsTable& C, const Batch& b, int F, uint32_t* cells,
                                float* emb_out, cudaStream_t st) {
  if (b.G == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((b.G * 32 + 255) / 256);
  if (C.M == 6)
    cells_select_kernel<6><<<grid, 256, 0, st>>>(T, C, b, F, cells, emb_out);
  else
    cells_select_kernel<0><<<grid, 256, 0, st>>>(T, C, b, F, cells, emb_out);
  return cudaGetLastError();
}

}  // namespace locc
