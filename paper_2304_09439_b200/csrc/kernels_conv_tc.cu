// kernels_conv_tc.cu — the encode-once U-Net's 3x3x3 layers on the 5th-generation tensor cores
// (NEXT-1, readings Q28, Q32; the CUDA-core conv3d_kernel in kernels_cells.cu is the fp32
// contexts' path).  Each layer is an implicit GEMM: rows = output positions over all shapes (flattened
// (shape, position)), N = 128 output channels, K = 27 taps x C_in, in 32-channel chunks of one tap.
// tcgen05.mma kind::tf32 with the 3xTF32 split (hi = tf32(x), lo = tf32(x - hi); hi hi + hi lo + lo hi),
// fp32 accumulators in TMEM; deconvolutions run as convolutions with flipped taps (weights pre-flipped).
//
// Persistent CTAs, a PAIR of 128-row tiles per pass (each weight chunk read from L2 once per 256 output
// rows: at 128 rows the weight stream was the L2-bound half of the runtime), 6 warps:
//   warp 0     weight producer: the layer's pre-split, pre-swizzled chunks [128 out x 32 K] (32 KB,
//              hi then lo, SW128 K-major) through a 5-stage ring (cp.async.bulk)
//   warp 1     MMA issuer: 2 x 12 TS MMAs per chunk (A from TMEM), one accumulator per tile
//   warps 2-5  im2col producers (thread = row r of both tiles = TMEM lane): gather the 32 input channels
//              of the row's tap position (zero outside the grid; issued one chunk ahead, so the loads
//              overlap the split and store of the previous chunk), split, tcgen05.st into a 2-stage A
//              ring in TMEM; after the pair's last chunk, the epilogue: bias + ReLU, rows to global
// TMEM: D_u = columns 128 u (u = 0, 1), A stage s = 256 + 128 s (tile 0 hi, lo; tile 1 hi, lo: 32 each).
// With ntaps = 1 the same kernel is a plain GEMM y = ReLU(x W^T + b) over flat rows: the tensor-core grid
// encode's layers 2 and 3 (kernels_cells.cu, one launch per 128-column half of the 256 outputs); for
// layer 2 the A rows are layer 1 of the rows' points, computed in the producers (pts mode).
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"
#include "tc_ptx.cuh"

namespace locc {
namespace {

using namespace tc;

constexpr int kCtStages = 5, kCtA = 2;
constexpr int kCtChunk = 32768, kCtHalf = 16384;

struct __align__(1024) ConvTcSmem {
  uint8_t w[kCtStages][kCtChunk];
  float bias[128];
  float4 w1b[256];  // layer-1 weights (w0, w1, w2, b) of the fused grid-encode layer 2 (pts mode)
  uint64_t w_full[kCtStages], w_empty[kCtStages], a_full[kCtA], a_empty[kCtA], d_full, d_empty;
  uint32_t tmem_base;
};

struct ConvTcArgs {
  const float* x1;  // [S][Di^3][C1]
  const float* x2;  // [S][Di^3][C2] or null (channels C1.. of the concatenation)
  int C1, C2, Di, Do, pad, S;
  const uint8_t* img;  // chunks (tap k, 32-channel block c) in order k-major
  const float* bias;
  float* y;            // [S][Do^3][128], ReLU applied (row stride ldy, columns ycol..ycol+127)
  int ntaps;           // 27: the 3x3x3 conv; 1: a plain GEMM, row r reads x1[r] (rows = flat_rows)
  int64_t flat_rows;
  int ldy, ycol;
  const float4* pts;  // pts mode (ntaps = 1, C1 = 256): x1 is not read; the A row is computed on the fly
  const float4* w1b;  // as h1 = ReLU(W1 p + b1) of the row's point (the grid encode's layer 1, fused)
};

// fp32 -> nearest tf32 (ties away from zero) in an fp32 container: bit-identical to cvt.rna.tf32.f32,
// but two integer ops on the ALU pipe instead of a conversion (a quarter-rate pipe, the producers' limit)
__device__ __forceinline__ float tf32r(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

__global__ void __launch_bounds__(192, 1) conv_tc_kernel(ConvTcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  ConvTcSmem& S = *reinterpret_cast<ConvTcSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Cin = a.C1 + a.C2, nci = Cin / 32, nch = a.ntaps * nci;
  const int nq = a.Do * a.Do * a.Do;
  const int64_t rows = a.ntaps == 1 ? a.flat_rows : (int64_t)a.S * nq, ntiles = (rows + 255) / 256;  // tile pairs
  for (int i = threadIdx.x; i < 128; i += blockDim.x) S.bias[i] = a.bias[i];
  if (a.pts)
    for (int i = threadIdx.x; i < 256; i += blockDim.x) S.w1b[i] = a.w1b[i];
  if (threadIdx.x == 0) {
    for (int i = 0; i < kCtStages; ++i) {
      mbar_init(&S.w_full[i], 1);
      mbar_init(&S.w_empty[i], 1);
    }
    for (int i = 0; i < kCtA; ++i) {
      mbar_init(&S.a_full[i], 128);
      mbar_init(&S.a_empty[i], 1);
    }
    mbar_init(&S.d_full, 1);
    mbar_init(&S.d_empty, 128);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_1cta(&S.tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    uint32_t n = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int j = 0; j < nch; ++j, ++n) {
        const uint32_t st = n % kCtStages;
        if (lane == 0) {
          if (n >= kCtStages) mbar_wait_spin(&S.w_empty[st], ((n / kCtStages) - 1) & 1);
          mbar_arrive_expect_tx(&S.w_full[st], kCtChunk);
          bulk_g2s(S.w[st], a.img + (size_t)j * kCtChunk, kCtChunk, &S.w_full[st]);
        }
        __syncwarp();
      }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_tf32_f32(128, 128);
    uint32_t n = 0, m = 0, it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      if (it > 0) {
        mbar_wait_spin(&S.d_empty, (it - 1) & 1);  // the previous pair's accumulators have been read
        tc_fence_after();
      }
      for (int j = 0; j < nch; ++j, ++n, ++m) {
        const uint32_t sw = n % kCtStages, sa = m % kCtA;
        mbar_wait_spin(&S.a_full[sa], (m / kCtA) & 1);
        mbar_wait_spin(&S.w_full[sw], (n / kCtStages) & 1);
        tc_fence_after();
        const uint32_t bhi = smem_u32(S.w[sw]), blo = bhi + kCtHalf;
        if (elect_one()) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {  // the weight chunk feeds both tiles of the pair
            const uint32_t d = tmem + 128 * u, ahi = tmem + 256 + 128 * sa + 64 * u, alo = ahi + 32;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              mma_tf32_ts(d, ahi + 8 * k, smem_desc_sw128(bhi + 32 * k, 1024), idesc, (j | k) != 0);
              mma_tf32_ts(d, ahi + 8 * k, smem_desc_sw128(blo + 32 * k, 1024), idesc, 1);
              mma_tf32_ts(d, alo + 8 * k, smem_desc_sw128(bhi + 32 * k, 1024), idesc, 1);
            }
          }
          mma_commit_1cta(&S.w_empty[sw]);
          mma_commit_1cta(&S.a_empty[sa]);
          if (j == nch - 1) mma_commit_1cta(&S.d_full);
        }
        __syncwarp();
      }
    }
  } else {
    const int q = warp & 3, r = 32 * q + lane;
    const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16);
    const int Di3 = a.Di * a.Di * a.Di;
    // the row's output position in tile u of pair t (computed once per pair)
    struct Pos {
      int64_t row;
      bool valid;
      int s, qx, qy, qz;
    };
    auto pos_of = [&](int64_t t, int u) {
      Pos P;
      P.row = t * 256 + 128 * u + r;
      P.valid = P.row < rows;
      P.s = P.qx = P.qy = P.qz = 0;
      if (a.ntaps != 1 && P.valid) {
        P.s = (int)(P.row / nq);
        const int qp = (int)(P.row % nq);
        P.qx = qp % a.Do, P.qy = (qp / a.Do) % a.Do, P.qz = qp / (a.Do * a.Do);
      }
      return P;
    };
    // gather of chunk j (tap k, channels 32c..32c+31) of the row at P; zero outside the grid
    auto gather = [&](const Pos& P, int j, float (&x)[32]) {
      const int k = j / nci, c = j - k * nci;
      bool in = P.valid;
      int64_t pos = P.row;
      if (a.ntaps != 1) {
        const int ix = P.qx + k % 3 - a.pad, iy = P.qy + (k / 3) % 3 - a.pad, iz = P.qz + k / 9 - a.pad;
        in = P.valid && ix >= 0 && iy >= 0 && iz >= 0 && ix < a.Di && iy < a.Di && iz < a.Di;
        pos = (int64_t)P.s * Di3 + (iz * a.Di + iy) * a.Di + ix;
      }
      if (in && a.pts) {
        const float4 p = __ldg(a.pts + pos);
#pragma unroll
        for (int v = 0; v < 32; ++v) {
          const float4 w = S.w1b[32 * c + v];
          x[v] = fmaxf(fmaf(w.x, p.x, fmaf(w.y, p.y, fmaf(w.z, p.z, w.w))), 0.f);
        }
      } else if (in) {
        const int ci = 32 * c;
        const float4* src = ci < a.C1 ? reinterpret_cast<const float4*>(a.x1 + pos * a.C1 + ci)
                                      : reinterpret_cast<const float4*>(a.x2 + pos * a.C2 + (ci - a.C1));
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const float4 f = __ldg(src + v);
          x[4 * v] = f.x, x[4 * v + 1] = f.y, x[4 * v + 2] = f.z, x[4 * v + 3] = f.w;
        }
      } else {
#pragma unroll
        for (int v = 0; v < 32; ++v) x[v] = 0.f;
      }
    };
    auto split = [](const float (&x)[32], uint32_t (&h)[32], uint32_t (&l)[32]) {
#pragma unroll
      for (int v = 0; v < 32; ++v) {
        const float hv = tf32r(x[v]);
        h[v] = __float_as_uint(hv);
        l[v] = __float_as_uint(tf32r(x[v] - hv));
      }
    };
    uint32_t m = 0, it = 0;
    float xa[32], xb[32];  // the next chunk's gathers (tiles 0 and 1 of the pair), issued one chunk ahead
    Pos ca = pos_of(blockIdx.x, 0), cb = pos_of(blockIdx.x, 1);
    if ((int64_t)blockIdx.x < ntiles) {
      gather(ca, 0, xa);
      gather(cb, 0, xb);
    }
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const Pos na = pos_of(t + gridDim.x, 0), nb = pos_of(t + gridDim.x, 1);
      const bool more = t + gridDim.x < ntiles;
      for (int j = 0; j < nch; ++j, ++m) {
        const uint32_t sa = m % kCtA;
        const uint32_t col = trow + 256 + 128 * sa;
        uint32_t h[32], l[32];
        split(xa, h, l);
        if (j + 1 < nch)
          gather(ca, j + 1, xa);
        else if (more)
          gather(na, 0, xa);
        if (m >= kCtA) mbar_wait(&S.a_empty[sa], ((m / kCtA) - 1) & 1);  // the MMAs have read stage sa
        tc_fence_after();
        tmem_st32(col, h);
        tmem_st32(col + 32, l);
        tmem_st_wait();
        split(xb, h, l);
        if (j + 1 < nch)
          gather(cb, j + 1, xb);
        else if (more)
          gather(nb, 0, xb);
        tmem_st32(col + 64, h);
        tmem_st32(col + 96, l);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&S.a_full[sa]);
      }
      // epilogue: ReLU(D_u + b) -> y[row of tile u]
      mbar_wait(&S.d_full, it & 1);
      tc_fence_after();
#pragma unroll 1
      for (int u = 0; u < 2; ++u) {
        const Pos& P = u == 0 ? ca : cb;
#pragma unroll 1
        for (int c0 = 0; c0 < 128; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(trow + 128 * u + c0, v);
          tmem_ld_wait();
          if (P.valid) {
            float4* yo = reinterpret_cast<float4*>(a.y + P.row * a.ldy + a.ycol + c0);
#pragma unroll
            for (int w = 0; w < 8; ++w)
              yo[w] = make_float4(fmaxf(__uint_as_float(v[4 * w]) + S.bias[c0 + 4 * w], 0.f),
                                  fmaxf(__uint_as_float(v[4 * w + 1]) + S.bias[c0 + 4 * w + 1], 0.f),
                                  fmaxf(__uint_as_float(v[4 * w + 2]) + S.bias[c0 + 4 * w + 2], 0.f),
                                  fmaxf(__uint_as_float(v[4 * w + 3]) + S.bias[c0 + 4 * w + 3], 0.f));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&S.d_empty);
      ca = na;
      cb = nb;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc_1cta(tmem, 512);
}

}  // namespace

cudaError_t launch_conv_tc(const float* x1, int C1, const float* x2, int C2, int Di, int Do, int pad, int S,
                           const uint8_t* img, const float* bias, float* y, int num_sms, cudaStream_t st) {
  const size_t sm = sizeof(ConvTcSmem) + 1024;
  const cudaError_t attr = smem_optin(conv_tc_kernel, sizeof(ConvTcSmem) + 1024);
  if (attr != cudaSuccess) return attr;
  const int64_t rows = (int64_t)S * Do * Do * Do, ntiles = (rows + 255) / 256;
  const unsigned grid = (unsigned)(ntiles < num_sms ? ntiles : num_sms);
  ConvTcArgs a{x1, x2, C1, C2, Di, Do, pad, S, img, bias, y, 27, 0, 128, 0, nullptr, nullptr};
  conv_tc_kernel<<<grid, 192, sm, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_gemm_tc(const float* x, int C, int64_t rows, const uint8_t* img, const float* bias, float* y,
                           int ldy, int ycol, int num_sms, cudaStream_t st, const float4* pts, const float4* w1b) {
  if (rows == 0) return cudaSuccess;
  const size_t sm = sizeof(ConvTcSmem) + 1024;
  const cudaError_t attr = smem_optin(conv_tc_kernel, sizeof(ConvTcSmem) + 1024);
  if (attr != cudaSuccess) return attr;
  const int64_t ntiles = (rows + 255) / 256;
  const unsigned grid = (unsigned)(ntiles < num_sms ? ntiles : num_sms);
  ConvTcArgs a{x, nullptr, C, 0, 1, 1, 0, 1, img, bias, y, 1, rows, ldy, ycol, pts, w1b};
  conv_tc_kernel<<<grid, 192, sm, st>>>(a);
  return cudaGetLastError();
}

}  // namespace locc
