// kernels_encoder_tc.cu — S4-S7 on the 5th-generation tensor cores (LOCC_PREC_BF16).
//
// One persistent launch; CTA pairs (clusters of 2 on a TPC) run cta_group::2 tcgen05.mma with
// fp32 accumulators in TMEM.  Work unit: a chunk of whole (pair, side) segments of the compacted
// row buffer (rows sorted by segment, then cell), cut into 256-row tiles; CTA r of the pair owns
// the tile rows {64r..64r+63} and {128+64r..128+64r+63}.  Per tile:
//
//   L1 (CUDA cores, fp32 FFMA)  h1 = ReLU(W1 p + b1) -> bf16, written as the A operand of L2
//                               (K-major, 128-byte swizzle) — PAPER.md:331, :421, :425
//   L2 (tcgen05, SS)            D2[256 rows x 256 features] = h1 * W2^T; A = h1 (each CTA its 128
//                               rows), B = W2 (each CTA 128 of the 256 output features, resident
//                               in shared memory for the whole launch)
//   epi L2 (TMEM -> regs)       h2 = ReLU(D2 + b2) -> bf16, written row-major (K-major) as the B
//                               operand of L3 — each CTA keeps its own rows: no exchange
//   L3 (tcgen05, TS)            D3[256 features x 128 rows] = W3 * h2^T, twice per tile (rows
//                               0-127, 128-255); A = W3 resident in TMEM (each CTA 128 features),
//                               B = h2 (each CTA 64 of the 128 rows)
//   epi L3 (TMEM -> regs)       thread = output feature, walking the rows in order: cell-wise max
//                               (PAPER.md:331), g = ReLU(max + b3), running sum over occupied cells
//                               in ascending order, mean at the segment end
//
// Layer 2 is computed "rows x features" and layer 3 "features x rows" so that layer 2's epilogue
// produces layer 3's operand in place and layer 3's epilogue sees each feature's rows in one
// thread — the segmented cell max needs no cross-lane reduction.
//
// Roles (512 threads): warp 0 = TMEM allocation + MMA issue (leader CTA), warps 4-7 = epi L3,
// warps 8-11 = epi L2, warps 12-15 = L1.  mbarriers link the roles across both CTAs.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"
#include "tc_ptx.cuh"

namespace locc {

namespace {

using namespace tc;

constexpr int kThreads = 512;
constexpr int kTileRows = 256;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColW3 = 0;    // W3 (this CTA's 128 output features), 128 columns of bf16x2
constexpr uint32_t kColD2 = 128;  // D2: 256 columns
constexpr uint32_t kColD3 = 384;  // D3: 128 columns
constexpr uint32_t kIdescL2 = idesc_bf16_f32(256, 256);
constexpr uint32_t kIdescL3 = idesc_bf16_f32(256, 128);

struct alignas(1024) Smem {
  uint8_t w2[65536];  // B of L2: this CTA's 128 W2 rows, 4 K blocks x [128 rows x 128 B], SW128
  uint8_t h1[65536];  // A of L2: this CTA's 128 rows of h1, same layout
  uint8_t h2[65536];  // B of L3: this CTA's 128 rows of h2, same layout
  uint32_t flags[kTileRows];
  uint64_t bar[8];
  uint32_t tmem_base;
};

enum { B_H1_FULL = 0, B_H1_EMPTY, B_D2_FULL, B_E2_DONE, B_H2_EMPTY, B_D3_FULL, B_D3_EMPTY, B_WLOAD };

struct TcArgs {
  TcL1 l1;
  const float* b3;
  const uint8_t* w2img;   // [2 ranks][65536 B] pre-swizzled
  const uint32_t* w3img;  // [256 rows][128] bf16x2
  const float4* rows;
  const int64_t* offsets;
  float* pooled;
  int64_t G;
  int64_t n_chunks;
  int seg_per_chunk;
};

// Iterates the (chunk, tile) sequence of this cluster; every role walks the same sequence.
struct TileIter {
  const int64_t* off;
  int64_t G, n_chunks, chunk, step;
  int spc;
  int64_t r1 = 0, t0 = 0;
  __device__ TileIter(const TcArgs& a, int64_t first, int64_t stride)
      : off(a.offsets), G(a.G), n_chunks(a.n_chunks), chunk(first - stride), step(stride), spc(a.seg_per_chunk) {}
  __device__ bool next(int64_t& row0, int& nrows) {
    while (t0 >= r1) {
      chunk += step;
      if (chunk >= n_chunks) return false;
      const int64_t s0 = chunk * spc;
      const int64_t s1 = min(s0 + spc, G);
      t0 = off[s0];
      r1 = off[s1];
    }
    row0 = t0;
    nrows = (int)min((int64_t)kTileRows, r1 - t0);
    t0 += kTileRows;
    return true;
  }
};

__device__ __forceinline__ uint32_t tile_row_of_local(uint32_t rank, uint32_t i) {
  return i < 64 ? 64 * rank + i : 128 + 64 * rank + (i - 64);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1) encoder_tc_kernel(const __grid_constant__ TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int64_t cid = cluster_id_x(), ncl = nclusters_x();

  // ---------------------------------------------------------------- setup
  if (threadIdx.x == 0) {
    mbar_init(&S.bar[B_H1_FULL], 8);    // 4 L1 warps x 2 CTAs (leader's copy is used)
    mbar_init(&S.bar[B_H1_EMPTY], 1);   // MMA commit
    mbar_init(&S.bar[B_D2_FULL], 1);
    mbar_init(&S.bar[B_E2_DONE], 8);    // 4 epi-L2 warps x 2 CTAs
    mbar_init(&S.bar[B_H2_EMPTY], 1);
    mbar_init(&S.bar[B_D3_FULL], 1);
    mbar_init(&S.bar[B_D3_EMPTY], 8);   // 4 epi-L3 warps x 2 CTAs
    mbar_init(&S.bar[B_WLOAD], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&S.bar[B_WLOAD], 65536);
    for (int kb = 0; kb < 4; ++kb)
      bulk_g2s(S.w2 + kb * 16384, a.w2img + (size_t)rank * 65536 + kb * 16384, 16384, &S.bar[B_WLOAD]);
  }
  if (warp == 0) tmem_alloc_2cta(&S.tmem_base, kTmemCols);
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  if (warp >= 4 && warp < 8) {  // W3 rows of this CTA's features -> TMEM (A operand of L3)
    const uint32_t q = warp - 4;
    const uint32_t f = 128 * rank + 32 * q + lane;
    const uint32_t* src = a.w3img + (size_t)f * 128;
    for (int j = 0; j < 16; ++j) {
      uint32_t v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = src[8 * j + e];
      tmem_st8(tmem + ((32 * q) << 16) + kColW3 + 8 * j, v);
    }
    tmem_st_wait();
  }
  if (threadIdx.x == 0) mbar_wait(&S.bar[B_WLOAD], 0);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();

  // ---------------------------------------------------------------- roles
  if (warp == 0) {
    // ============ MMA issuer (leader CTA, one thread) ============
    if (rank == 0 && lane == 0) {
      TileIter it_(a, cid, ncl);
      int64_t row0;
      int nrows;
      uint32_t it = 0, u3 = 0;
      const uint32_t a_h1 = smem_u32(S.h1), b_w2 = smem_u32(S.w2), b_h2 = smem_u32(S.h2);
      while (it_.next(row0, nrows)) {
        mbar_wait(&S.bar[B_H1_FULL], it & 1);
        mbar_wait(&S.bar[B_E2_DONE], (it & 1) ^ 1);  // D2 drained by the previous tile's epilogue
        tc_fence_after();
#pragma unroll 1
        for (int k = 0; k < 16; ++k) {
          const uint32_t koff = (k >> 2) * 16384 + (k & 3) * 32;
          mma_ss_2cta(tmem + kColD2, smem_desc_sw128(a_h1 + koff, 1024), smem_desc_sw128(b_w2 + koff, 1024), kIdescL2,
                      k > 0);
        }
        mma_commit_2cta(&S.bar[B_H1_EMPTY], 3);
        mma_commit_2cta(&S.bar[B_D2_FULL], 3);
        mbar_wait(&S.bar[B_E2_DONE], it & 1);  // h2 of this tile written in both CTAs
        tc_fence_after();
        const int np = nrows > 128 ? 2 : 1;
        for (int p = 0; p < np; ++p) {
          mbar_wait(&S.bar[B_D3_EMPTY], (u3 & 1) ^ 1);
          tc_fence_after();
#pragma unroll 1
          for (int k = 0; k < 16; ++k) {
            const uint32_t koff = (k >> 2) * 16384 + (k & 3) * 32 + p * 8192;
            mma_ts_2cta(tmem + kColD3, tmem + kColW3 + 8 * k, smem_desc_sw128(b_h2 + koff, 1024), kIdescL3, k > 0);
          }
          mma_commit_2cta(&S.bar[B_D3_FULL], 3);
          ++u3;
        }
        mma_commit_2cta(&S.bar[B_H2_EMPTY], 3);
        ++it;
      }
    }
  } else if (warp >= 12) {
    // ============ L1: thread = row, all H features, fp32 FFMA -> bf16 A operand ============
    const uint32_t i = 32 * (warp - 12) + lane;  // local row 0..127
    const uint32_t trow = tile_row_of_local(rank, i);
    TileIter it_(a, cid, ncl);
    int64_t row0;
    int nrows;
    uint32_t it = 0;
    const uint32_t h1 = smem_u32(S.h1);
    while (it_.next(row0, nrows)) {
      float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
      if ((int)trow < nrows) p = a.rows[row0 + trow];
      mbar_wait(&S.bar[B_H1_EMPTY], (it & 1) ^ 1);
#pragma unroll
      for (int c = 0; c < 32; ++c) {  // 32 chunks of 8 features
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float4 wa = a.l1.w1b[8 * c + 2 * e], wb = a.l1.w1b[8 * c + 2 * e + 1];
          const float ha = fmaf(wa.x, p.x, fmaf(wa.y, p.y, fmaf(wa.z, p.z, wa.w)));
          const float hb = fmaf(wb.x, p.x, fmaf(wb.y, p.y, fmaf(wb.z, p.z, wb.w)));
          w[e] = pack_relu_bf16x2(ha, hb);
        }
        st_shared_v4(h1 + (c >> 3) * 16384 + sw128_off(i, c & 7), w[0], w[1], w[2], w[3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&S.bar[B_H1_FULL], 0);
      ++it;
    }
  } else if (warp >= 8) {
    // ============ epi L2: thread = row, D2 -> ReLU(+b2) -> bf16 B operand of L3 ============
    const uint32_t q = warp - 8;
    const uint32_t i = 32 * q + lane;
    const uint32_t tbase = tmem + ((32 * q) << 16) + kColD2;
    TileIter it_(a, cid, ncl);
    int64_t row0;
    int nrows;
    uint32_t it = 0;
    const uint32_t h2 = smem_u32(S.h2);
    while (it_.next(row0, nrows)) {
      mbar_wait(&S.bar[B_D2_FULL], it & 1);
      mbar_wait(&S.bar[B_H2_EMPTY], (it & 1) ^ 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 8; ++c) {  // 8 chunks of 32 features
        uint32_t v[32];
        tmem_ld32(tbase + 32 * c, v);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int f = 32 * c + 8 * g + 2 * e;
            w[e] = pack_relu_bf16x2(__uint_as_float(v[8 * g + 2 * e]) + a.l1.b2[f],
                                    __uint_as_float(v[8 * g + 2 * e + 1]) + a.l1.b2[f + 1]);
          }
          st_shared_v4(h2 + (c >> 1) * 16384 + sw128_off(i, (c & 1) * 4 + g), w[0], w[1], w[2], w[3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&S.bar[B_E2_DONE], 0);
      ++it;
    }
  } else if (warp >= 4) {
    // ============ epi L3: thread = output feature, walk rows: cell max, occupied-cell mean ============
    const uint32_t q = warp - 4;
    const uint32_t f = 128 * rank + 32 * q + lane;
    const uint32_t tbase = tmem + ((32 * q) << 16) + kColD3;
    const float b3 = a.b3[f];
    float run_max = -INFINITY, run_sum = 0.f;
    int run_cells = 0;
    TileIter it_(a, cid, ncl);
    int64_t row0;
    int nrows;
    uint32_t u3 = 0;
    const uint32_t t128 = threadIdx.x - 128;  // 0..127 within the epi-L3 group
    while (it_.next(row0, nrows)) {
      asm volatile("bar.sync 1, 128;" ::: "memory");  // previous tile's flags no longer read
      for (int r = t128; r < kTileRows; r += 128)
        S.flags[r] = r < nrows ? __float_as_uint(a.rows[row0 + r].w) : 0u;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int np = nrows > 128 ? 2 : 1;
      for (int p = 0; p < np; ++p) {
        mbar_wait(&S.bar[B_D3_FULL], u3 & 1);
        tc_fence_after();
        const int ncols = min(128, nrows - 128 * p);
        for (int c = 0; c < 4; ++c) {
          if (32 * c >= ncols) break;
          uint32_t v[32];
          tmem_ld32(tbase + 32 * c, v);
          tmem_ld_wait();
          const int n = min(32, ncols - 32 * c);
          const uint32_t* fl = S.flags + 128 * p + 32 * c;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (j < n) {
              const uint32_t w = fl[j];
              run_max = fmaxf(run_max, __uint_as_float(v[j]));
              if (w & kRowFlagCellEnd) {
                run_sum += fmaxf(run_max + b3, 0.f);
                ++run_cells;
                run_max = -INFINITY;
                if (w & kRowFlagSegEnd) {
                  a.pooled[(int64_t)(w >> kRowSegShift) * 256 + f] = __fdiv_rn(run_sum, (float)run_cells);
                  run_sum = 0.f;
                  run_cells = 0;
                }
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&S.bar[B_D3_EMPTY], 0);
        ++u3;
      }
    }
  }

  // ---------------------------------------------------------------- teardown
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 0) tmem_dealloc_2cta(tmem, kTmemCols);
}

}  // namespace

size_t encoder_tc_smem_bytes() { return sizeof(Smem) + 1024; }

cudaError_t launch_encoder_tc(const DevParams& P, const TcL1& l1, const Batch& b, int num_sms, cudaStream_t st) {
  const int spc = 16;
  const int64_t chunks = (b.G + spc - 1) / spc;
  if (chunks == 0) return cudaSuccess;
  if (!P.tc_w2 || !P.tc_w3) return cudaErrorInvalidValue;
  TcArgs args;
  args.l1 = l1;
  args.b3 = P.b3;
  args.w2img = static_cast<const uint8_t*>(P.tc_w2);
  args.w3img = static_cast<const uint32_t*>(P.tc_w3);
  args.rows = b.rows;
  args.offsets = b.offsets;
  args.pooled = b.pooled;
  args.G = b.G;
  args.n_chunks = chunks;
  args.seg_per_chunk = spc;
  const size_t smem = encoder_tc_smem_bytes();
  static const cudaError_t attr =
      cudaFuncSetAttribute(encoder_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (attr != cudaSuccess) return attr;
  int grid = (num_sms / 2) * 2;
  const int64_t max_useful = 2 * chunks;
  if (grid > max_useful) grid = (int)max_useful;
  encoder_tc_kernel<<<grid, kThreads, smem, st>>>(args);
  return cudaGetLastError();
}

}  // namespace locc
