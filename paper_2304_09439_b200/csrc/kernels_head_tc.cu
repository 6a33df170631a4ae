// kernels_head_tc.cu — S8-S9 collision predictor on the 5th-generation tensor cores, fp32-accurate.
//
// Same function as head_tile_kernel ([e ; q ; t] -> 3 x 128 ReLU shared by both
// objects -> max across the pair -> 3 x 128 ReLU -> linear -> sigmoid).  Each layer is a [rows x K] x
// [K x 128] GEMM on tcgen05.mma kind::tf32 with the "3xTF32" split: every fp32 operand x = hi + lo,
// hi = tf32(x) and lo = tf32(x - hi), both rounded to nearest (so the tensor core reads them exactly),
// and A B ~= A_hi B_hi + A_hi B_lo + A_lo B_hi — relative error ~2^-22 per product (the dropped lo lo
// term); reading Q32 gives the measured bar.
//
// Persistent CTAs (one per SM), 64 pairs (128 sides) per tile:
//   warp 0     weight producer: streams pre-split, pre-swizzled 32-K weight chunks (32 KB: [128 x 32]
//              hi then lo, K-major SW128, built at weight load) through a 5-stage ring (cp.async.bulk)
//   warp 1     MMA issuer (one elected lane): 12 MMAs (4 K-steps x 3 products) per chunk, A from TMEM
//   warps 2+   epilogue (TMEM lane quadrant = warp % 4, thread = row r): per layer tcgen05.ld the
//              accumulator row, bias + ReLU, split, and tcgen05.st the next layer's A row (hi, lo);
//              8 warps (two column halves per row) in the forward variants, 4 with the gradient
// TMEM (512 columns): two accumulators D0 = 0..127 and D1 = 384..511 used by alternate layers,
// A_hi = 128..255, A_lo = 256..383 (A: row = lane, K = column), so the operands never touch shared
// memory and 160 KB of it holds the weight ring.  The epilogue hands the next layer's A over per
// 32-column K chunk (one mbarrier per chunk) and the MMA warp issues that chunk's products at once, into
// the other accumulator: layer l + 1's MMAs overlap layer l's epilogue.
// Rows: side s of the tile in row s (pair p = sides 2p, 2p+1); the pair layers keep pair p in row 2p
// and zeros in the odd rows, so the max across the pair and the gradient's routing back to the two
// sides are shuffles between adjacent lanes.
//
// kProj (crop path): e = W_F m + b_F first, also on the tensor cores (m = the pooled 256-vector in two
// K halves, N = 64).  kGrad: after the forward, the reverse pass d logit / d pose (NEXT-2; oracle
// head_grad) as five more GEMMs on the transposed weights, masked by the recorded ReLU decisions.
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
constexpr int kStages = 5;          // weight ring
constexpr int kLayers = 6;
constexpr int kChunks = 23;         // obj1 3 (K = 71 padded to 96), obj2, obj3, pair1..3 4 each
constexpr int kBwd = 5;             // reverse GEMMs: pair3^T, pair2^T, pair1^T, obj3^T, obj2^T (4 chunks each)
constexpr uint32_t kColD0 = 0, kColD1 = 384, kColAH = 128, kColAL = 256;
// Accumulator of the stage with D counter sd (both projection halves share one stage's accumulator).
__device__ __forceinline__ uint32_t dcol(uint32_t sd) { return (sd & 1) ? kColD1 : kColD0; }
__constant__ int kLayerChunks[kLayers + kBwd] = {3, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4};

struct __align__(1024) HeadTcSmem {
  uint8_t w[kStages][kChunkBytes];  // weight ring
  float bias[kLayers][128];
  float wout[128];
  float bout;
  float bf[64];
  int nside[128];
  float part[2][128];  // the output unit's partial sums of the two column groups
  // reverse mode (kGrad): ReLU masks of the forward (bit c of word [l][row][c / 32] = activation > 0;
  // l = obj1, obj2, obj3 (side rows), pair1, pair2 (pair rows 2p)), the max's routing per pair (bit =
  // u_A > u_B, ties -> B) and obj.l1's 7 pose columns
  uint32_t mask[kLayers][128][4];
  uint32_t selA[64][4];
  float o1p[7][128];
  uint64_t w_full[kStages], w_empty[kStages], a_full[4], d_full;  // a_full[j]: A's K chunk j written
  uint32_t tmem_base;
};

// Round to the nearest tf32 (ties away): a value the tensor core reads exactly.  Bit-identical to
// cvt.rna.tf32.f32, as two integer ops on the ALU pipe instead of a conversion.
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// Split 32 values (this thread's row, K columns c0..c0+31) and store them as A_hi / A_lo.
__device__ __forceinline__ void put32(uint32_t arow, int c0, const float (&x)[32]) {
  uint32_t h[32], l[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const float hv = tf32_rna(x[k]);
    h[k] = __float_as_uint(hv);
    l[k] = __float_as_uint(tf32_rna(x[k] - hv));
  }
  tmem_st32(arow + kColAH + c0, h);
  tmem_st32(arow + kColAL + c0, l);
}

// This warp's rows of A's K chunk (columns c0 .. c0 + 31) are written: one arrival per warp (a chunk is
// written by the 4 warps of one column group, one per TMEM lane quadrant).
__device__ __forceinline__ void chunk_ready(HeadTcSmem& S, int c0) {
  tmem_st_wait();
  tc_fence_before();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(&S.a_full[c0 >> 5]);
}

// kGrad variants keep 4 epilogue warps (their register footprint); the forward variants run 8, two per
// TMEM lane quadrant, each taking half of the columns.
template <bool kProj, bool kGrad>
__global__ void __launch_bounds__(kGrad ? 192 : 320, 1) head_tc_kernel(DevParams P, Batch b, float* __restrict__ probs,
                                                                uint8_t* __restrict__ labels,
                                                                float* __restrict__ logits, float* __restrict__ emb,
                                                                float* __restrict__ grad) {
  constexpr int kEW = kGrad ? 4 : 8;         // epilogue warps
  constexpr int kNT = 64 + 32 * kEW;         // threads
  constexpr int kHalves = kEW / 4;           // column groups per row
  constexpr int kCols = 128 / kHalves;       // accumulator columns per epilogue thread
  extern __shared__ uint8_t smem_raw[];
  HeadTcSmem& S = *reinterpret_cast<HeadTcSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (b.B + kHP - 1) / kHP;
  const float* bias_src = P.head_tc_bias;  // [6][128] biases, wout [128], bout, b_F [64]
  for (int i = threadIdx.x; i < kLayers * 128; i += kNT) S.bias[i / 128][i % 128] = bias_src[i];
  for (int i = threadIdx.x; i < 128; i += kNT) S.wout[i] = bias_src[kLayers * 128 + i];
  for (int i = threadIdx.x; i < 64; i += kNT) S.bf[i] = bias_src[kLayers * 128 + 129 + i];
  if constexpr (kGrad)
    for (int i = threadIdx.x; i < 7 * 128; i += kNT) S.o1p[i / 128][i % 128] = P.o1p[i];
  if (threadIdx.x == 0) {
    S.bout = bias_src[kLayers * 128 + 128];
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&S.w_full[i], 1);
      mbar_init(&S.w_empty[i], 1);
    }
    for (int j = 0; j < 4; ++j) mbar_init(&S.a_full[j], 4);
    mbar_init(&S.d_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_1cta(&S.tmem_base, 512);
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
        const uint32_t st = n % kStages;
        if (lane == 0) {
          if (n >= kStages) mbar_wait_spin(&S.w_empty[st], ((n / kStages) - 1) & 1);
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
    constexpr int kL0 = kProj ? -2 : 0;
    constexpr int kLEnd = kGrad ? kLayers + kBwd : kLayers;
    uint32_t n = 0, aph = 0, sd = 0;  // aph bit j: phase of a_full[j]; sd: accumulator counter
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int l = kL0; l < kLEnd; ++l) {
        // l = -2, -1: the projection's two K halves (N = 64; the second accumulates onto the first)
        const uint32_t idesc = l < 0 ? idesc_tf32_f32(128, 64) : idesc_tf32_f32(128, 128);
        const int nch = l < 0 ? 4 : kLayerChunks[l];
        const uint32_t d = tmem + dcol(sd);
        for (int j = 0; j < nch; ++j, ++n) {
          mbar_wait_spin(&S.a_full[j], (aph >> j) & 1);  // A's chunk j of this stage
          aph ^= 1u << j;
          const uint32_t st = n % kStages;
          mbar_wait_spin(&S.w_full[st], (n / kStages) & 1);
          tc_fence_after();
          const uint32_t bhi = smem_u32(S.w[st]), blo = bhi + kHalfChunk;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t kc = (uint32_t)(32 * j + 8 * k), bo = 32u * k;
              mma_tf32_ts(d, tmem + kColAH + kc, smem_desc_sw128(bhi + bo, 1024), idesc, (l == -1) || (j | k) != 0);
              mma_tf32_ts(d, tmem + kColAH + kc, smem_desc_sw128(blo + bo, 1024), idesc, 1);
              mma_tf32_ts(d, tmem + kColAL + kc, smem_desc_sw128(bhi + bo, 1024), idesc, 1);
            }
            mma_commit_1cta(&S.w_empty[st]);
            if (j == nch - 1) mma_commit_1cta(&S.d_full);
          }
          __syncwarp();
        }
        if (l != -2) ++sd;
      }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5)
    const int q = warp & 3, r = 32 * q + lane;  // TMEM lane quadrant, row
    const int half = (warp - 2) >> 2;          // column group (0 when kHalves == 1)
    const int cb = half * kCols, eb = half * (kCols / 2);  // first column of 128-wide / 64-wide rows
    const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16);
    const bool odd = r & 1;
    uint32_t dph = 0, sd = 0;  // d_full phase; accumulator counter (as the MMA warp's)
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t i0 = t * kHP;
      const int npairs = (int)min((int64_t)kHP, b.B - i0);
      const bool live = r < 2 * npairs;
      const int64_t g = 2 * i0 + r;
      LOCC_CHECK(!live || g < b.G);
      const int ns = live ? b.counts[g] : 0;
      S.nside[r] = ns;
      // ---- z = [e ; canonical q ; t ; 0...] (K = 96) for side r (e = 0 for an empty side)
      if constexpr (kProj) {
        // m (the pooled 256-vector) in two K halves through A; e = D + b_F afterwards
        const float4* m4 = reinterpret_cast<const float4*>(b.pooled + g * 256);
        // the tensor-core encoder leaves cell sums: m = S / C (IEEE division)
        const float cnt = (b.cells_c && ns > 0) ? (float)b.cells_c[g] : 1.f, rcnt = __frcp_rn(cnt);
        LOCC_CHECK_V(ns == 0 || (cnt >= 1.f && cnt <= (float)ns), g, (int64_t)ns * 100000 + (int64_t)cnt);  // 1 <= cells <= kept
        for (int h = 0; h < 2; ++h) {
          if (h == 1) {  // the first half has been consumed
            mbar_wait(&S.d_full, dph);
            dph ^= 1;
            tc_fence_after();
          }
#pragma unroll 1
          for (int c0 = cb; c0 < cb + kCols; c0 += 32) {
            float x[32];
#pragma unroll
            for (int k = 0; k < 32; k += 4) {
              float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
              if (ns > 0) {
                v = __ldg(m4 + ((128 * h + c0 + k) >> 2));
                if (b.cells_c)
                  v = make_float4(div_count(v.x, cnt, rcnt), div_count(v.y, cnt, rcnt), div_count(v.z, cnt, rcnt),
                                  div_count(v.w, cnt, rcnt));
              }
              x[k] = v.x, x[k + 1] = v.y, x[k + 2] = v.z, x[k + 3] = v.w;
            }
            put32(trow, c0, x);
            chunk_ready(S, c0);
          }
        }
        mbar_wait(&S.d_full, dph);
        dph ^= 1;
        tc_fence_after();
#pragma unroll 1
        for (int c0 = eb; c0 < eb + kCols / 2; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(trow + dcol(sd) + c0, v);
          tmem_ld_wait();
          float x[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) x[k] = ns > 0 ? __uint_as_float(v[k]) + S.bf[c0 + k] : 0.f;
          put32(trow, c0, x);
          chunk_ready(S, c0);
          if (emb && live)
#pragma unroll
            for (int k = 0; k < 32; k += 4)
              *reinterpret_cast<float4*>(emb + g * 64 + c0 + k) = make_float4(x[k], x[k + 1], x[k + 2], x[k + 3]);
        }
        ++sd;
      } else {
        const float4* e4 = reinterpret_cast<const float4*>(b.emb_in + g * 64);
#pragma unroll 1
        for (int c0 = eb; c0 < eb + kCols / 2; c0 += 32) {
          float x[32];
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ns > 0) v = __ldg(e4 + ((c0 + k) >> 2));
            x[k] = v.x, x[k + 1] = v.y, x[k + 2] = v.z, x[k + 3] = v.w;
          }
          put32(trow, c0, x);
          chunk_ready(S, c0);
        }
      }
      {
        float x[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) x[k] = 0.f;
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
#pragma unroll
          for (int c = 0; c < 4; ++c) x[c] = __double2float_rn(sg * qd[c]);
#pragma unroll
          for (int c = 0; c < 3; ++c) x[4 + c] = pose[4 + c];
        }
        if (half == kHalves - 1) {
          put32(trow, 64, x);
          chunk_ready(S, 64);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEW) : "memory");  // nside of every side visible to the pair rows
      // ---- forward layers
      for (int l = 0; l < kLayers; ++l) {
        mbar_wait(&S.d_full, dph);
        dph ^= 1;
        tc_fence_after();
        const float* bl = S.bias[l];
        if (l < 2) {
          // object layers 1, 2 (side rows): ReLU(D + b) -> next A
#pragma unroll 1
          for (int c0 = cb; c0 < cb + kCols; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(trow + dcol(sd) + c0, v);
            tmem_ld_wait();
            float x[32];
            uint32_t bits = 0;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              x[k] = fmaxf(__uint_as_float(v[k]) + bl[c0 + k], 0.f);
              bits |= (uint32_t)(x[k] > 0.f) << k;
            }
            put32(trow, c0, x);
            chunk_ready(S, c0);
            if (kGrad) S.mask[l][r][c0 >> 5] = bits;
          }
        } else if (l == 2) {
          // object layer 3, then the max across the pair into row 2p (odd rows -> 0)
#pragma unroll 1
          for (int c0 = cb; c0 < cb + kCols; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(trow + dcol(sd) + c0, v);
            tmem_ld_wait();
            float x[32];
            uint32_t mb = 0, sb = 0;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const float mine = fmaxf(__uint_as_float(v[k]) + bl[c0 + k], 0.f);
              const float other = __shfl_xor_sync(0xffffffffu, mine, 1);
              x[k] = odd ? 0.f : fmaxf(mine, other);
              mb |= (uint32_t)(mine > 0.f) << k;
              sb |= (uint32_t)(mine > other) << k;  // even lane: u_A > u_B (ties -> B)
            }
            put32(trow, c0, x);
            chunk_ready(S, c0);
            if (kGrad) {
              S.mask[2][r][c0 >> 5] = mb;
              if (!odd) S.selA[r >> 1][c0 >> 5] = sb;
            }
          }
          if (kGrad) asm volatile("bar.sync 1, %0;" ::"n"(32 * kEW) : "memory");  // selA visible to the odd rows
        } else if (l < 5) {
          // pair layers 1, 2 (pair p in row 2p): ReLU(D + b) -> next A, odd rows 0
#pragma unroll 1
          for (int c0 = cb; c0 < cb + kCols; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(trow + dcol(sd) + c0, v);
            tmem_ld_wait();
            float x[32];
            uint32_t bits = 0;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              x[k] = odd ? 0.f : fmaxf(__uint_as_float(v[k]) + bl[c0 + k], 0.f);
              bits |= (uint32_t)(x[k] > 0.f) << k;
            }
            put32(trow, c0, x);
            chunk_ready(S, c0);
            if (kGrad) S.mask[l][r][c0 >> 5] = bits;
          }
        } else {
          // pair layer 3 + output unit (even row 2p = pair p); kGrad: d logit / d pre3 = w_out [c3 > 0]
          float acc = 0.f;
#pragma unroll 1
          for (int c0 = cb; c0 < cb + kCols; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(trow + dcol(sd) + c0, v);
            tmem_ld_wait();
            float x[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const float pre = __uint_as_float(v[k]) + bl[c0 + k];
              acc = fmaf(S.wout[c0 + k], fmaxf(pre, 0.f), acc);
              x[k] = (!odd && pre > 0.f) ? S.wout[c0 + k] : 0.f;
            }
            if (kGrad) {
              put32(trow, c0, x);
              chunk_ready(S, c0);
            }
          }
          if constexpr (kHalves == 2) {
            S.part[half][r] = acc;
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kEW) : "memory");
            acc = S.part[0][r] + S.part[1][r];
          }
          const int p = r >> 1;
          if (half == 0 && !odd && p < npairs) {
            const int64_t i = i0 + p;
            float lg, pr;
            if (S.nside[r] + S.nside[r + 1] == 0) {
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
        ++sd;
      }
      if constexpr (kGrad) {
        // ---- reverse GEMMs: B1 (pair3^T) -> d/d c2, B2 -> d/d c1, B3 (pair1^T) -> d/d v,
        //      B4 (obj3^T) -> d/d a2, B5 (obj2^T) -> d/d a1
        for (int l = 0; l < kBwd; ++l) {
          mbar_wait(&S.d_full, dph);
          dph ^= 1;
          tc_fence_after();
          if (l < 2 || l == 3) {
            // mask by c2 / c1 (pair rows; odd rows stay 0) or by a2 (side rows)
            const int ml = l == 3 ? 1 : 4 - l;
#pragma unroll 1
            for (int c0 = cb; c0 < cb + kCols; c0 += 32) {
              uint32_t v[32];
              tmem_ld32(trow + dcol(sd) + c0, v);
              tmem_ld_wait();
              const uint32_t m = S.mask[ml][r][c0 >> 5];
              float x[32];
#pragma unroll
              for (int k = 0; k < 32; ++k) x[k] = (m >> k) & 1u ? __uint_as_float(v[k]) : 0.f;
              put32(trow, c0, x);
              chunk_ready(S, c0);
            }
          } else if (l == 2) {
            // d/d v of pair p (row 2p) routed to the side the max selected, masked by u > 0
#pragma unroll 1
            for (int c0 = cb; c0 < cb + kCols; c0 += 32) {
              uint32_t v[32];
              tmem_ld32(trow + dcol(sd) + c0, v);
              tmem_ld_wait();
              const uint32_t sa = S.selA[r >> 1][c0 >> 5];
              const uint32_t m = S.mask[2][r][c0 >> 5] & (odd ? ~sa : sa);
              float x[32];
#pragma unroll
              for (int k = 0; k < 32; ++k) {
                const float gv = __shfl_sync(0xffffffffu, __uint_as_float(v[k]), lane & ~1);
                x[k] = (m >> k) & 1u ? gv : 0.f;
              }
              put32(trow, c0, x);
              chunk_ready(S, c0);
            }
          } else {
            // d/d a1 masked by a1 > 0 = d/d pre1; d/d z[F + c] = sum_o O1[o][F + c] d/d pre1[o]
            float gz[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
            for (int c0 = cb; c0 < cb + kCols; c0 += 32) {
              uint32_t v[32];
              tmem_ld32(trow + dcol(sd) + c0, v);
              tmem_ld_wait();
              const uint32_t m = S.mask[0][r][c0 >> 5];
#pragma unroll
              for (int k = 0; k < 32; ++k) {
                const float x = (m >> k) & 1u ? __uint_as_float(v[k]) : 0.f;
#pragma unroll
                for (int c = 0; c < 7; ++c) gz[c] = fmaf(S.o1p[c][c0 + k], x, gz[c]);
              }
            }
            if (live) {
              float* gout = grad + g * 7;
              if (S.nside[r & ~1] + S.nside[r | 1] == 0) {
                for (int c = 0; c < 7; ++c) gout[c] = 0.f;
              } else {
                const float* pose = b.poses + g * 7;
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
          ++sd;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEW) : "memory");  // this tile's nside reads precede the next tile's writes
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc_1cta(tmem, 512);
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
  const int threads = grad ? 192 : 320;
  const cudaError_t attr = [] {  // once per (device, kernel), see smem_optin
    const size_t sm = head_tc_smem_bytes();
    cudaError_t e = smem_optin(head_tc_kernel<true, true>, sm);
    if (e == cudaSuccess) e = smem_optin(head_tc_kernel<true, false>, sm);
    if (e == cudaSuccess) e = smem_optin(head_tc_kernel<false, true>, sm);
    if (e == cudaSuccess) e = smem_optin(head_tc_kernel<false, false>, sm);
    return e;
  }();
  if (attr != cudaSuccess) return attr;
  auto run = [&](auto kern) {
    kern<<<grid, threads, head_tc_smem_bytes(), st>>>(P, b, probs, labels, logits, emb, grad);
    return cudaGetLastError();
  };
  if (proj) return grad ? run(head_tc_kernel<true, true>) : run(head_tc_kernel<true, false>);
  return grad ? run(head_tc_kernel<false, true>) : run(head_tc_kernel<false, false>);
}

}  // namespace locc
