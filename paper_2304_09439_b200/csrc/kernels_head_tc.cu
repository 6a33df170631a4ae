// kernels_head_tc.cu — S8-S9 collision predictor on the 5th-generation tensor cores, fp32-accurate.
//
// Same function as head_tile_kernel ([e ; q ; t] -> 3 x 128 ReLU shared by both
// objects -> max across the pair -> 3 x 128 ReLU -> linear -> sigmoid), for the encode-once mode where
// e arrives pooled (Batch::emb_in).  Each layer is a [rows x K] x [K x 128] GEMM on tcgen05.mma
// kind::tf32 with the "3xTF32" split: every fp32 operand x = hi + lo, hi = tf32(x) and lo = tf32(x - hi),
// both rounded to nearest (so the tensor core reads them exactly), and A B ~= A_hi B_hi + A_hi B_lo +
// A_lo B_hi — relative error ~2^-22 per product (the dropped lo lo term), the order of fp32 FFMA
// summation, so the 1e-5 probability bar of the fp32 path holds (tested against the fp64 oracle).  Accumulators in TMEM (128 columns), operands K-major SW128 in shared memory.
//
// Persistent CTAs (one per SM), 64 pairs (128 sides) per tile, 6 warps:
//   warp 0     weight producer: streams the 23 pre-split, pre-swizzled 32-K chunks of the six layers'
//              weights (32 KB each: hi then lo) through a 2-stage ring with cp.async.bulk
//   warp 1     MMA issuer (one elected lane): 12 MMAs (4 K-steps x 3 products) per chunk
//   warps 2-5  epilogue (TMEM lane quadrant = warp % 4, thread = row): stage z for layer 1, then per
//              layer tcgen05.ld the accumulator row, bias + ReLU, split, write the next layer's A
//              operand (the max across the pair = a lane shuffle: sides 2p, 2p+1 are adjacent lanes)
// Pair layers run M = 128 with rows 64..127 zero (64 pairs per tile).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"
#include "quat.cuh"
#include "tc_ptx.cuh"

namespace locc {
namespace {

using namespace tc;

constexpr int kHP = 64;             // pairs per tile
constexpr int kChunkBytes = 32768;  // one 32-K chunk of one layer: hi [128 x 32] then lo, SW128
constexpr int kHalfChunk = 16384;
constexpr int kLayers = 6;
constexpr int kChunks = 23;         // obj1 3 (K = 71 padded to 96), obj2, obj3, pair1..3 4 each
constexpr int kThreadsTC = 192;
constexpr int kBwd = 5;             // reverse-mode GEMMs: pair3^T, pair2^T, pair1^T, obj3^T, obj2^T (4 chunks each)
__constant__ int kLayerChunks[kLayers + kBwd] = {3, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4};

struct __align__(1024) HeadTcSmem {
  uint8_t a_hi[4 * kHalfChunk];     // A operand, 4 K-blocks of [128 rows x 32 fp32] SW128
  uint8_t a_lo[4 * kHalfChunk];
  uint8_t w[2][kChunkBytes];        // weight ring
  float bias[kLayers][128];
  float wout[128];
  float bout;
  float bf[64];
  int nside[128];
  // reverse mode (kGrad): ReLU masks of the forward (bit c of word [l][row][c / 32] = activation > 0;
  // l = obj1, obj2, obj3 (side rows), pair1, pair2, pair3 (pair rows)), the max's routing (bit = u_A > u_B)
  // and obj.l1's 7 pose columns
  uint32_t mask[kLayers][128][4];
  uint32_t selA[64][4];
  float o1p[7][128];
  uint64_t w_full[2], w_empty[2], a_full, d_full;
  uint32_t tmem_base;
};

// Round to the nearest tf32 (ties away): a value the tensor core reads exactly.
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Write 4 consecutive K values (k0 .. k0+3, k0 % 4 == 0) of row r into the split A operand:
// hi = tf32(x), lo = tf32(x - hi) (x - hi is exact in fp32; |lo| <= 2^-11 |x|, error <= 2^-23 |x|).
__device__ __forceinline__ void put4(HeadTcSmem& S, int r, int k0, float x0, float x1, float x2, float x3) {
  const float h0 = tf32_rna(x0), h1 = tf32_rna(x1), h2 = tf32_rna(x2), h3 = tf32_rna(x3);
  const uint32_t off = (uint32_t)(k0 >> 5) * kHalfChunk + sw128_off((uint32_t)r, (uint32_t)((k0 & 31) >> 2));
  st_shared_v4(smem_u32(S.a_hi) + off, __float_as_uint(h0), __float_as_uint(h1), __float_as_uint(h2),
               __float_as_uint(h3));
  st_shared_v4(smem_u32(S.a_lo) + off, __float_as_uint(tf32_rna(x0 - h0)), __float_as_uint(tf32_rna(x1 - h1)),
               __float_as_uint(tf32_rna(x2 - h2)), __float_as_uint(tf32_rna(x3 - h3)));
}

// kProj (crop path): e = W_F m + b_F is computed first on the tensor cores too — two passes of 4 K-chunks
// (m = the pooled 256-vector, staged 128 K at a time into the A buffer), N = 64, then z as above.
// kGrad: after the forward, the reverse pass d logit / d pose (NEXT-2; oracle head_grad) runs as five
// more GEMMs on the transposed weights (pre-split images), masked by the recorded ReLU decisions.
template <bool kProj, bool kGrad>
__global__ void __launch_bounds__(kThreadsTC, 1) head_tc_kernel(DevParams P, Batch b, float* __restrict__ probs,
                                                                uint8_t* __restrict__ labels,
                                                                float* __restrict__ logits, float* __restrict__ emb,
                                                                float* __restrict__ grad) {
  extern __shared__ uint8_t smem_raw[];
  HeadTcSmem& S = *reinterpret_cast<HeadTcSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (b.B + kHP - 1) / kHP;
  const float* bias_src = P.head_tc_bias;  // [6][128] biases, wout [128], bout, b_F [64]
  for (int i = threadIdx.x; i < kLayers * 128; i += kThreadsTC) S.bias[i / 128][i % 128] = bias_src[i];
  for (int i = threadIdx.x; i < 128; i += kThreadsTC) S.wout[i] = bias_src[kLayers * 128 + i];
  for (int i = threadIdx.x; i < 64; i += kThreadsTC) S.bf[i] = bias_src[kLayers * 128 + 129 + i];
  if constexpr (kGrad)
    for (int i = threadIdx.x; i < 7 * 128; i += kThreadsTC) S.o1p[i / 128][i % 128] = P.o1p[i];
  if (threadIdx.x == 0) {
    S.bout = bias_src[kLayers * 128 + 128];
    mbar_init(&S.w_full[0], 1);
    mbar_init(&S.w_full[1], 1);
    mbar_init(&S.w_empty[0], 1);
    mbar_init(&S.w_empty[1], 1);
    mbar_init(&S.a_full, 128);
    mbar_init(&S.d_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_1cta(&S.tmem_base, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    // ---------------------------------------------------------------- weight producer
    const uint8_t* img = static_cast<const uint8_t*>(P.head_tc_img);
    const uint8_t* pimg = static_cast<const uint8_t*>(P.head_tc_proj);
    const uint8_t* bimg = static_cast<const uint8_t*>(P.head_tc_bwd);
    constexpr int kPre = kProj ? 8 : 0, kPost = kGrad ? 4 * kBwd : 0;
    uint32_t n = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int c = 0; c < kPre + kChunks + kPost; ++c, ++n) {
        const int st = n & 1;
        if (lane == 0) {
          if (n >= 2) mbar_wait_spin(&S.w_empty[st], ((n >> 1) - 1) & 1);
          mbar_arrive_expect_tx(&S.w_full[st], kChunkBytes);
          const uint8_t* src = c < kPre ? pimg + (size_t)c * kChunkBytes
                               : c < kPre + kChunks ? img + (size_t)(c - kPre) * kChunkBytes
                                                    : bimg + (size_t)(c - kPre - kChunks) * kChunkBytes;
          bulk_g2s(S.w[st], src, kChunkBytes, &S.w_full[st]);
        }
        __syncwarp();
      }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t ahi = smem_u32(S.a_hi), alo = smem_u32(S.a_lo);
    constexpr int kL0 = kProj ? -2 : 0;
    uint32_t n = 0, aph = 0;
    constexpr int kLEnd = kGrad ? kLayers + kBwd : kLayers;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int l = kL0; l < kLEnd; ++l) {
        // l = -2, -1: the projection's two K halves (N = 64; the second accumulates onto the first)
        const uint32_t idesc = l < 0 ? idesc_tf32_f32(128, 64) : idesc_tf32_f32(128, 128);
        const int nch = l < 0 ? 4 : kLayerChunks[l];
        mbar_wait_spin(&S.a_full, aph);
        aph ^= 1;
        tc_fence_after();
        for (int j = 0; j < nch; ++j, ++n) {
          const int st = n & 1;
          mbar_wait_spin(&S.w_full[st], (n >> 1) & 1);
          tc_fence_after();
          const uint32_t bhi = smem_u32(S.w[st]), blo = bhi + kHalfChunk;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t ao = (uint32_t)j * kHalfChunk + 32u * k, bo = 32u * k;
              mma_tf32_ss(tmem, smem_desc_sw128(ahi + ao, 1024), smem_desc_sw128(bhi + bo, 1024), idesc,
                          (l == -1) || (j | k) != 0);
              mma_tf32_ss(tmem, smem_desc_sw128(ahi + ao, 1024), smem_desc_sw128(blo + bo, 1024), idesc, 1);
              mma_tf32_ss(tmem, smem_desc_sw128(alo + ao, 1024), smem_desc_sw128(bhi + bo, 1024), idesc, 1);
            }
            mma_commit_1cta(&S.w_empty[st]);
            if (j == nch - 1) mma_commit_1cta(&S.d_full);
          }
          __syncwarp();
        }
      }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5)
    const int q = warp & 3, r = 32 * q + lane;  // TMEM lane quadrant, row
    const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16);
    uint32_t dph = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t i0 = t * kHP;
      const int npairs = (int)min((int64_t)kHP, b.B - i0);
      // z = [e ; canonical q ; t ; 0...] (K = 96) for side r (e = 0 for an empty side)
      {
        float z[8];
        const bool live = r < 2 * npairs;
        const int64_t g = 2 * i0 + r;
        const int ns = live ? b.counts[g] : 0;
        S.nside[r] = ns;
        if constexpr (kProj) {
          // m (the pooled 256-vector) in two K halves through the A buffer; e = D + b_F afterwards
          const float4* m4 = reinterpret_cast<const float4*>(b.pooled + g * 256);
          for (int h = 0; h < 2; ++h) {
            if (h == 1) {
              mbar_wait(&S.d_full, dph);  // the first half has been consumed
              dph ^= 1;
            }
            for (int k0 = 0; k0 < 128; k0 += 4) {
              float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
              if (ns > 0) v = __ldg(m4 + ((128 * h + k0) >> 2));
              put4(S, r, k0, v.x, v.y, v.z, v.w);
            }
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(&S.a_full);
          }
          mbar_wait(&S.d_full, dph);
          dph ^= 1;
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < 64; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(trow + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; k += 4) {
              float x[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) x[u] = ns > 0 ? __uint_as_float(v[k + u]) + S.bf[c0 + k + u] : 0.f;
              put4(S, r, c0 + k, x[0], x[1], x[2], x[3]);
              if (emb && live) *reinterpret_cast<float4*>(emb + g * 64 + c0 + k) = make_float4(x[0], x[1], x[2], x[3]);
            }
          }
        } else {
          const float4* e4 = reinterpret_cast<const float4*>(b.emb_in + g * 64);
          for (int k0 = 0; k0 < 64; k0 += 4) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ns > 0) v = __ldg(e4 + (k0 >> 2));
            put4(S, r, k0, v.x, v.y, v.z, v.w);
          }
        }
        for (int c = 0; c < 8; ++c) z[c] = 0.f;
        if (live) {
          const float* pose = b.poses + g * 7;
          double qd[4] = {1.0, 0.0, 0.0, 0.0};
          quat_unit(pose, qd);
          double sg = 1.0;
          for (int c = 0; c < 4; ++c)
            if (qd[c] != 0.0) {
              sg = qd[c] > 0.0 ? 1.0 : -1.0;
              break;
            }
          for (int c = 0; c < 4; ++c) z[c] = __double2float_rn(sg * qd[c]);
          for (int c = 0; c < 3; ++c) z[4 + c] = pose[4 + c];
        }
        put4(S, r, 64, z[0], z[1], z[2], z[3]);
        put4(S, r, 68, z[4], z[5], z[6], 0.f);
        for (int k0 = 72; k0 < 96; k0 += 4) put4(S, r, k0, 0.f, 0.f, 0.f, 0.f);
      }
      fence_proxy_async_smem();
      asm volatile("bar.sync 1, 128;" ::: "memory");  // nside of every side visible to the output rows
      tc_fence_before();
      mbar_arrive(&S.a_full);
      for (int l = 0; l < kLayers; ++l) {
        mbar_wait(&S.d_full, dph);
        dph ^= 1;
        tc_fence_after();
        const float* bl = S.bias[l];
        if (l < 2 || (l >= 3 && l < 5)) {
          // hidden layer: ReLU(D + b) -> next A (pair layers: rows >= 64 are padding -> 0)
          const bool pad = l >= 3 && r >= 64;
#pragma unroll 1
          for (int c0 = 0; c0 < 128; c0 += 32) {
            uint32_t bits = 0;
            uint32_t v[32];
            tmem_ld32(trow + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; k += 4) {
              float x[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) x[u] = pad ? 0.f : fmaxf(__uint_as_float(v[k + u]) + bl[c0 + k + u], 0.f);
              put4(S, r, c0 + k, x[0], x[1], x[2], x[3]);
              if (kGrad)
                bits |= (uint32_t)(x[0] > 0.f) << k | (uint32_t)(x[1] > 0.f) << (k + 1) |
                        (uint32_t)(x[2] > 0.f) << (k + 2) | (uint32_t)(x[3] > 0.f) << (k + 3);
            }
            if (kGrad) S.mask[l][r][c0 >> 5] = bits;
          }
        } else if (l == 2) {
          // object layer 3, then the max across the pair: pair p = r / 2 (even lanes) -> row p,
          // odd lanes write the padding rows 64 + (r - 1) / 2 as 0
          const int prow = (r & 1) ? 64 + (r >> 1) : (r >> 1);
#pragma unroll 1
          for (int c0 = 0; c0 < 128; c0 += 32) {
            uint32_t v[32], mb = 0, sb = 0;
            tmem_ld32(trow + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; k += 4) {
              float x[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float mine = fmaxf(__uint_as_float(v[k + u]) + bl[c0 + k + u], 0.f);
                const float other = __shfl_xor_sync(0xffffffffu, mine, 1);
                x[u] = (r & 1) ? 0.f : fmaxf(mine, other);
                if (kGrad) {
                  mb |= (uint32_t)(mine > 0.f) << (k + u);
                  sb |= (uint32_t)(mine > other) << (k + u);  // even lane: u_A > u_B (ties -> B)
                }
              }
              put4(S, prow, c0 + k, x[0], x[1], x[2], x[3]);
            }
            if (kGrad) {
              S.mask[2][r][c0 >> 5] = mb;
              if (!(r & 1)) S.selA[r >> 1][c0 >> 5] = sb;
            }
          }
        } else {
          // pair layer 3 + output unit: row p < 64 = pair p
          float acc = 0.f;
#pragma unroll 1
          for (int c0 = 0; c0 < 128; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(trow + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; ++k)
              acc = fmaf(S.wout[c0 + k], fmaxf(__uint_as_float(v[k]) + bl[c0 + k], 0.f), acc);
            if (kGrad) {  // reverse mode starts here: d logit / d pre3 = w_out [c3 > 0] (pair rows)
#pragma unroll
              for (int k = 0; k < 32; k += 4) {
                float x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  x[u] = (r < 64 && __uint_as_float(v[k + u]) + bl[c0 + k + u] > 0.f) ? S.wout[c0 + k + u] : 0.f;
                put4(S, r, c0 + k, x[0], x[1], x[2], x[3]);
              }
            }
          }
          if (r < npairs) {
            const int64_t i = i0 + r;
            float lg, pr;
            if (S.nside[2 * r] + S.nside[2 * r + 1] == 0) {
              lg = -INFINITY;
              pr = 0.f;
            } else {
              lg = acc + S.bout;
              pr = 1.f / (1.f + expf(-lg));
              atomicAdd(&b.stats->evaluated_pairs, 1ull);
            }
            probs[i] = pr;
            if (labels) labels[i] = pr > 0.5f ? 1 : 0;
            if (logits) logits[i] = lg;
          }
        }
        if (kGrad || l < kLayers - 1) {
          if (kGrad && l == 2) asm volatile("bar.sync 1, 128;" ::: "memory");  // masks/selA visible to pair rows
          fence_proxy_async_smem();
          tc_fence_before();
          mbar_arrive(&S.a_full);
        }
      }
      if constexpr (kGrad) {
        // reverse GEMMs: B1 (pair3^T) -> d/d c2, B2 -> d/d c1, B3 (pair1^T) -> d/d v, B4 (obj3^T) -> d/d a2,
        // B5 (obj2^T) -> d/d a1
        for (int l = 0; l < kBwd; ++l) {
          mbar_wait(&S.d_full, dph);
          dph ^= 1;
          tc_fence_after();
          if (l == 0 || l == 1) {
            // mask by c2 / c1 (pair rows), next A; rows >= 64 stay 0
            const int ml = 4 - l;
#pragma unroll 1
            for (int c0 = 0; c0 < 128; c0 += 32) {
              uint32_t v[32];
              tmem_ld32(trow + c0, v);
              tmem_ld_wait();
              const uint32_t m = r < 64 ? S.mask[ml][r][c0 >> 5] : 0u;
#pragma unroll
              for (int k = 0; k < 32; k += 4) {
                float x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) x[u] = (m >> (k + u)) & 1u ? __uint_as_float(v[k + u]) : 0.f;
                put4(S, r, c0 + k, x[0], x[1], x[2], x[3]);
              }
            }
          } else if (l == 2) {
            // d/d v (pair row p) routed to the side the max selected, masked by u > 0: rows 2p, 2p+1
            if (r < 64) {  // pair row p = r writes side rows 2p, 2p+1 (the MMA has consumed A)
#pragma unroll 1
              for (int c0 = 0; c0 < 128; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(trow + c0, v);
                tmem_ld_wait();
                const uint32_t sa = S.selA[r][c0 >> 5], ma = S.mask[2][2 * r][c0 >> 5] & sa,
                               mbb = S.mask[2][2 * r + 1][c0 >> 5] & ~sa;
#pragma unroll
                for (int k = 0; k < 32; k += 4) {
                  float xa[4], xb[4];
#pragma unroll
                  for (int u = 0; u < 4; ++u) {
                    const float gv = __uint_as_float(v[k + u]);
                    xa[u] = (ma >> (k + u)) & 1u ? gv : 0.f;
                    xb[u] = (mbb >> (k + u)) & 1u ? gv : 0.f;
                  }
                  put4(S, 2 * r, c0 + k, xa[0], xa[1], xa[2], xa[3]);
                  put4(S, 2 * r + 1, c0 + k, xb[0], xb[1], xb[2], xb[3]);
                }
              }
            } else {
              // quadrants 2, 3 read their (padding) accumulator rows too: tcgen05.ld is warp-collective
#pragma unroll 1
              for (int c0 = 0; c0 < 128; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(trow + c0, v);
                tmem_ld_wait();
              }
            }
          } else if (l == 3) {
            // d/d a2 (side rows) masked by a2 > 0
#pragma unroll 1
            for (int c0 = 0; c0 < 128; c0 += 32) {
              uint32_t v[32];
              tmem_ld32(trow + c0, v);
              tmem_ld_wait();
              const uint32_t m = S.mask[1][r][c0 >> 5];
#pragma unroll
              for (int k = 0; k < 32; k += 4) {
                float x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) x[u] = (m >> (k + u)) & 1u ? __uint_as_float(v[k + u]) : 0.f;
                put4(S, r, c0 + k, x[0], x[1], x[2], x[3]);
              }
            }
          } else {
            // d/d a1 masked by a1 > 0 = d/d pre1; d/d z[F + c] = sum_o O1[o][F + c] d/d pre1[o]
            float gz[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
            for (int c0 = 0; c0 < 128; c0 += 32) {
              uint32_t v[32];
              tmem_ld32(trow + c0, v);
              tmem_ld_wait();
              const uint32_t m = S.mask[0][r][c0 >> 5];
#pragma unroll
              for (int k = 0; k < 32; ++k) {
                const float x = (m >> k) & 1u ? __uint_as_float(v[k]) : 0.f;
#pragma unroll
                for (int c = 0; c < 7; ++c) gz[c] = fmaf(S.o1p[c][c0 + k], x, gz[c]);
              }
            }
            const int64_t side = 2 * i0 + r;
            if (r < 2 * npairs) {
              float* gout = grad + side * 7;
              if (S.nside[r & ~1] + S.nside[r | 1] == 0) {
                for (int c = 0; c < 7; ++c) gout[c] = 0.f;
              } else {
                const float* pose = b.poses + side * 7;
                const double qv[4] = {pose[0], pose[1], pose[2], pose[3]};
                const double nq = sqrt(((qv[0] * qv[0] + qv[1] * qv[1]) + qv[2] * qv[2]) + qv[3] * qv[3]);
                double sg = 1.0;
                for (int c = 0; c < 4; ++c)
                  if (qv[c] != 0.0) {
                    sg = qv[c] > 0.0 ? 1.0 : -1.0;
                    break;
                  }
                double qh[4], dot = 0.0;
                for (int c = 0; c < 4; ++c) {
                  qh[c] = sg * qv[c] / nq;
                  dot += qh[c] * (double)gz[c];
                }
                for (int c = 0; c < 4; ++c) gout[c] = (float)(sg * ((double)gz[c] - qh[c] * dot) / nq);
                for (int c = 4; c < 7; ++c) gout[c] = gz[c];
              }
            }
          }
          if (l < kBwd - 1) {
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(&S.a_full);
          }
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // this tile's nside reads precede the next tile's writes
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc_1cta(tmem, 128);
}

}  // namespace

size_t head_tc_smem_bytes() { return sizeof(HeadTcSmem) + 1024; }

cudaError_t launch_head_tc(const DevParams& P, const Batch& b, float* probs, uint8_t* labels, float* logits,
                           float* emb, float* grad, int num_sms, cudaStream_t st) {
  if (b.B == 0) return cudaSuccess;
  const bool proj = b.emb_in == nullptr;  // crop path: project the pooled vectors first
  if (grad && !P.head_tc_bwd) return cudaErrorNotSupported;
  const int64_t ntiles = (b.B + kHP - 1) / kHP;
  const unsigned grid = (unsigned)(ntiles < num_sms ? ntiles : num_sms);
  auto run = [&](auto kern) {
    const cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)head_tc_smem_bytes());
    if (attr != cudaSuccess) return attr;
    kern<<<grid, kThreadsTC, head_tc_smem_bytes(), st>>>(P, b, probs, labels, logits, emb, grad);
    return cudaGetLastError();
  };
  if (proj) return grad ? run(head_tc_kernel<true, true>) : run(head_tc_kernel<true, false>);
  return grad ? run(head_tc_kernel<false, true>) : run(head_tc_kernel<false, false>);
}

}  // namespace locc
