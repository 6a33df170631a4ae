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
// Roles (13 warps): warps 0-7 = epi L2 of tile t then layer 1 of tile t+1, warps 8-11 = epi L3,
// warp 12 = TMEM allocation + MMA issue (leader CTA).  mbarriers link the roles across both
// CTAs; layer 3 starts per 32-feature K chunk as soon as epi L2 has written it; TMEM regions rotate
// between tiles so the MMAs of one tile overlap the layer-3 epilogue of the previous one.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"
#include "tc_ptx.cuh"

namespace locc {

namespace {

using namespace tc;

// Warp roles (13 warps).  TMEM lane access is restricted to lane quarter (warp % 4), so each
// TMEM-reading group covers the four quarters.
constexpr int kWarps = 13;
constexpr int kThreads = 32 * kWarps;
// The warp scheduler favours higher warp ids, so the sequential layer-3 walk and the MMA issuer get
// the high ids.
constexpr int kWarpW = 0;    // warps 0..7: epilogue of L2 (thread = row, half the features each),
                             // then layer 1 of the next tile (thread = 4 features x 32 rows)
constexpr int kWarpE3 = 8;   // warps 8..11: epilogue of L3 (thread = output feature)
constexpr int kWarpMMA = 12; // warp 12: TMEM allocation + MMA issue (leader CTA)
constexpr int kTileRows = 256;
constexpr uint32_t kTmemCols = 512;
// TMEM columns: W3 (A of L3: this CTA's 128 features as bf16x2) and three 128-column regions that
// rotate between the accumulators: even tiles D2 = [RA|RB], D3p0 = RC, D3p1 = RA; odd tiles
// D2 = [RB|RC], D3p0 = RA, D3p1 = RC.  A region is rewritten only one full layer after its
// previous consumer started, so the MMAs never wait for a layer-3 epilogue in steady state.
constexpr uint32_t kColW3 = 0, kColRA = 128, kColRB = 256, kColRC = 384;
constexpr uint32_t kIdescL2 = idesc_bf16_f32(256, 256);
constexpr uint32_t kIdescL3 = idesc_bf16_f32(256, 128);

__device__ __forceinline__ uint32_t d2_col(uint32_t par) { return par ? kColRB : kColRA; }
__device__ __forceinline__ uint32_t d3_col(uint32_t par, int p) {
  return p == 0 ? (par ? kColRA : kColRC) : (par ? kColRC : kColRA);
}

struct alignas(1024) Smem {
  uint8_t w2[65536];  // B of L2: this CTA's 128 W2 rows, 4 K blocks x [128 rows x 128 B], SW128
  uint8_t h1[65536];  // A of L2: this CTA's 128 rows of h1, same layout
  uint8_t h2[65536];  // B of L3: this CTA's 128 rows of h2, same layout
  float px[128], py[128], pz[128];  // this CTA's rows of the tile (layer-1 input), SoA
  float b2[256];
  uint32_t flags[kTileRows];  // row flags of the whole tile (epi L3)
  uint32_t masks[16];         // cell-end bits [0..7], segment-end bits [8..15] per 32-row chunk
  uint64_t bar[13];
  uint32_t tmem_base;
};

enum {
  B_H1_FULL = 0, B_H1_EMPTY, B_D2_FULL, B_E2K0, B_E2K1, B_E2K2, B_E2K3, B_H2_EMPTY, B_D3F0, B_D3F1, B_D3E0,
  B_D3E1, B_WLOAD
};

struct TcArgs {
  const float4* w1b;      // [256] (w0, w1, w2, b1)
  const float* b2;
  const float* b3;
  const uint8_t* w2img;   // [2 ranks][65536 B] pre-swizzled
  const uint32_t* w3img;  // [256 rows][128] bf16x2
  const float4* rows;
  const int64_t* offsets;
  float* pooled;
  int64_t G;
  int64_t n_chunks;
  int seg_per_chunk;
  long long* trace;  // debug timeline (LOCC_TC_TRACE): [2 ranks][64 tiles][16 events] of cluster 0
};

constexpr int kTraceTiles = 64;
__device__ __forceinline__ void trace_ev(const TcArgs& a, uint32_t rank, int64_t cid, uint32_t tile, int ev) {
  if (a.trace && cid == 0 && tile < kTraceTiles) a.trace[(rank * kTraceTiles + tile) * 16 + ev] = clock64();
}

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

// One 32-column chunk of the layer-3 walk for this thread's feature.  Columns are tile rows in
// order; `ce`/`se` flag the last row of a cell / of a segment (uniform across the warp).  The common
// chunk (32 valid rows, no segment end) runs branch-free: per row one max, and at a cell end the
// cell's pooled value g = ReLU(max + b3) is added (fma with 0/1) and the running max reset.
__device__ __forceinline__ void walk_chunk(const uint32_t (&v)[32], int n, uint32_t ce, uint32_t se,
                                           const uint32_t* flags, float b3, float& run_max, float& run_sum,
                                           int& run_cells, float* pooled, uint32_t f) {
  if (n == 32 && se == 0) {
    run_cells += __popc(ce);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const bool e = (ce >> j) & 1u;
      run_max = fmaxf(run_max, __uint_as_float(v[j]));
      run_sum = fmaf(e ? 1.f : 0.f, fmaxf(run_max + b3, 0.f), run_sum);
      run_max = e ? -INFINITY : run_max;
    }
    return;
  }
#pragma unroll 1
  for (int j = 0; j < n; ++j) {
    float x = 0.f;
#pragma unroll
    for (int t = 0; t < 32; ++t) x = t == j ? __uint_as_float(v[t]) : x;
    run_max = fmaxf(run_max, x);
    if ((ce >> j) & 1u) {
      run_sum += fmaxf(run_max + b3, 0.f);
      ++run_cells;
      run_max = -INFINITY;
      if ((se >> j) & 1u) {
        pooled[(int64_t)(flags[j] >> kRowSegShift) * 256 + f] = __fdiv_rn(run_sum, (float)run_cells);
        run_sum = 0.f;
        run_cells = 0;
      }
    }
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1) encoder_tc_kernel(const __grid_constant__ TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023));
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int64_t cid = cluster_id_x(), ncl = nclusters_x();

  // ---------------------------------------------------------------- setup
  if (threadIdx.x == 0) {
    mbar_init(&S.bar[B_H1_FULL], 16);  // 8 worker warps x 2 CTAs (the leader's copy is used)
    mbar_init(&S.bar[B_H1_EMPTY], 1);  // MMA commits
    mbar_init(&S.bar[B_D2_FULL], 1);
    for (int j = 0; j < 4; ++j) mbar_init(&S.bar[B_E2K0 + j], 16);  // 8 worker warps x 2 CTAs
    mbar_init(&S.bar[B_H2_EMPTY], 1);
    mbar_init(&S.bar[B_D3F0], 1);
    mbar_init(&S.bar[B_D3F1], 1);
    mbar_init(&S.bar[B_D3E0], 8);  // 4 epi-L3 warps x 2 CTAs
    mbar_init(&S.bar[B_D3E1], 8);
    mbar_init(&S.bar[B_WLOAD], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&S.bar[B_WLOAD], 65536);
    for (int kb = 0; kb < 4; ++kb)
      bulk_g2s(S.w2 + kb * 16384, a.w2img + (size_t)rank * 65536 + kb * 16384, 16384, &S.bar[B_WLOAD]);
  }
  for (int i = threadIdx.x; i < 256; i += kThreads) S.b2[i] = a.b2[i];
  if (warp == kWarpMMA) tmem_alloc_2cta(&S.tmem_base, kTmemCols);
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  if (warp >= kWarpE3 && warp < kWarpE3 + 4) {  // W3 rows of this CTA's features -> TMEM (A of L3)
    const uint32_t q = warp & 3;
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
  if (warp == kWarpMMA) {
    // ============ MMA issuer (leader CTA, one thread) ============
    if (rank == 0 && lane == 0) {
      TileIter iter(a, cid, ncl);
      int64_t row0;
      int nrows;
      uint32_t it = 0, n0 = 0, n1 = 0;
      bool prev_p1 = false;
      const uint32_t a_h1 = smem_u32(S.h1), b_w2 = smem_u32(S.w2), b_h2 = smem_u32(S.h2);
      while (iter.next(row0, nrows)) {
        const uint32_t par = it & 1;
        mbar_wait(&S.bar[B_H1_FULL], par);
        trace_ev(a, rank, cid, it, 0);
        // D2 = [RA|RB] (even) or [RB|RC] (odd): RA resp. RC last held L3p0 of the previous tile;
        // RB held the previous D2, drained before that tile's L3 could start.
        if (it > 0) mbar_wait(&S.bar[B_D3E0], (n0 - 1) & 1);
        trace_ev(a, rank, cid, it, 1);
        tc_fence_after();
        const uint32_t dcol = tmem + d2_col(par);
#pragma unroll 1
        for (int k = 0; k < 16; ++k) {
          const uint32_t koff = (k >> 2) * 16384 + (k & 3) * 32;
          mma_ss_2cta(dcol, smem_desc_sw128(a_h1 + koff, 1024), smem_desc_sw128(b_w2 + koff, 1024), kIdescL2, k > 0);
        }
        mma_commit_2cta(&S.bar[B_H1_EMPTY], 3);
        mma_commit_2cta(&S.bar[B_D2_FULL], 3);
        trace_ev(a, rank, cid, it, 2);
        // L3p0 -> RC (even) / RA (odd): last held L3p1 of the previous tile, if it had one
        if (prev_p1) mbar_wait(&S.bar[B_D3E1], (n1 - 1) & 1);
        trace_ev(a, rank, cid, it, 3);
        const int np = nrows > 128 ? 2 : 1;
        {
          const uint32_t d3 = tmem + d3_col(par, 0);
#pragma unroll 1
          for (int j = 0; j < 4; ++j) {  // K chunk j = features {32j..32j+31} and {128+32j..}
            mbar_wait(&S.bar[B_E2K0 + j], par);
            tc_fence_after();
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int s = 0; s < 2; ++s) {
                const int k = 8 * h + 2 * j + s;
                const uint32_t koff = (k >> 2) * 16384 + (k & 3) * 32;
                mma_ts_2cta(d3, tmem + kColW3 + 8 * k, smem_desc_sw128(b_h2 + koff, 1024), kIdescL3, (j | h | s) != 0);
              }
          }
          mma_commit_2cta(&S.bar[B_D3F0], 3);
          trace_ev(a, rank, cid, it, 4);
        }
        if (np == 2) {
          const uint32_t d3 = tmem + d3_col(par, 1);
#pragma unroll 1
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int s = 0; s < 2; ++s) {
                const int k = 8 * h + 2 * j + s;
                const uint32_t koff = (k >> 2) * 16384 + (k & 3) * 32 + 8192;
                mma_ts_2cta(d3, tmem + kColW3 + 8 * k, smem_desc_sw128(b_h2 + koff, 1024), kIdescL3, (j | h | s) != 0);
              }
          mma_commit_2cta(&S.bar[B_D3F1], 3);
          trace_ev(a, rank, cid, it, 5);
        }
        mma_commit_2cta(&S.bar[B_H2_EMPTY], 3);
        ++n0;
        if (np == 2) ++n1;
        prev_p1 = np == 2;
        ++it;
      }
    }
  } else if (warp < kWarpE3) {
    // ============ workers: epi L2 of tile t, then layer 1 of tile t+1 ============
    const uint32_t q = warp & 3;                 // TMEM lane quarter (epi L2 rows 32q..32q+31)
    const uint32_t half = (warp - kWarpW) >> 2;  // epi L2 features [128 half, +128)
    const uint32_t row = 32 * q + lane;
    const uint32_t lt = threadIdx.x - 32 * kWarpW;  // 0..255
    const uint32_t fq = lt & 63, rq = lt >> 6;      // layer 1: features 4fq..4fq+3, rows 32rq..32rq+31
    unsigned long long wx[4], wy[4], wz[4], wb[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 w = a.w1b[4 * fq + k];
      wx[k] = f2(w.x, w.x);
      wy[k] = f2(w.y, w.y);
      wz[k] = f2(w.z, w.z);
      wb[k] = f2(w.w, w.w);
    }
    const uint32_t l1_base = smem_u32(S.h1) + ((4 * fq) >> 6) * 16384 + (((4 * fq) & 7) << 1);
    const uint32_t l1_chunk = ((4 * fq) & 63) >> 3;
    const uint32_t h2 = smem_u32(S.h2);

    auto layer1 = [&](uint32_t t, int64_t r0, int nr) {
      asm volatile("bar.sync 2, 256;" ::: "memory");  // previous tile's rows no longer read
      if (lt < 128) {
        const uint32_t trow = tile_row_of_local(rank, lt);
        float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
        if ((int)trow < nr) p = a.rows[r0 + trow];
        S.px[lt] = p.x;
        S.py[lt] = p.y;
        S.pz[lt] = p.z;
      }
      asm volatile("bar.sync 2, 256;" ::: "memory");
      mbar_wait(&S.bar[B_H1_EMPTY], (t & 1) ^ 1);
      if (lt == 0) trace_ev(a, rank, cid, t, 6);
#pragma unroll 1
      for (uint32_t r8 = 32 * rq; r8 < 32 * rq + 32; r8 += 8) {
#pragma unroll
        for (uint32_t v = 0; v < 8; v += 2) {
          const uint32_t r = r8 + v;
          const unsigned long long x2 = *reinterpret_cast<const unsigned long long*>(&S.px[r]);
          const unsigned long long y2 = *reinterpret_cast<const unsigned long long*>(&S.py[r]);
          const unsigned long long z2 = *reinterpret_cast<const unsigned long long*>(&S.pz[r]);
          unsigned long long h[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) h[k] = ffma2(wx[k], x2, ffma2(wy[k], y2, ffma2(wz[k], z2, wb[k])));
          const uint32_t base = l1_base + (r8 >> 3) * 1024;
          st_shared_v2(base + v * 128 + ((l1_chunk ^ v) << 4), pack_relu_bf16x2(f2_lo(h[0]), f2_lo(h[1])),
                       pack_relu_bf16x2(f2_lo(h[2]), f2_lo(h[3])));
          st_shared_v2(base + (v + 1) * 128 + ((l1_chunk ^ (v + 1)) << 4), pack_relu_bf16x2(f2_hi(h[0]), f2_hi(h[1])),
                       pack_relu_bf16x2(f2_hi(h[2]), f2_hi(h[3])));
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&S.bar[B_H1_FULL], 0);
      if (lt == 0) trace_ev(a, rank, cid, t, 7);
    };

    TileIter iter_l1(a, cid, ncl), iter(a, cid, ncl);
    int64_t row0, l1_row0;
    int nrows, l1_nrows;
    uint32_t it = 0;
    if (iter_l1.next(l1_row0, l1_nrows)) layer1(0, l1_row0, l1_nrows);
    while (iter.next(row0, nrows)) {
      mbar_wait(&S.bar[B_D2_FULL], it & 1);
      if (lt == 0) trace_ev(a, rank, cid, it, 8);
      mbar_wait(&S.bar[B_H2_EMPTY], (it & 1) ^ 1);
      if (lt == 0) trace_ev(a, rank, cid, it, 9);
      tc_fence_after();
      const uint32_t tbase = tmem + ((32 * q) << 16) + d2_col(it & 1) + 128 * half;
      uint32_t va[32], vb[32];
      tmem_ld32(tbase, va);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t(&v)[32] = (c & 1) ? vb : va;
        uint32_t(&nx)[32] = (c & 1) ? va : vb;
        tmem_ld_wait();
        if (c < 3) tmem_ld32(tbase + 32 * (c + 1), nx);
        const int cc = 4 * half + c;  // feature chunk (32 features)
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const float* bp = &S.b2[32 * cc + 8 * g];
          const unsigned long long* b2p = reinterpret_cast<const unsigned long long*>(bp);
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const unsigned long long s = fadd2(f2(__uint_as_float(v[8 * g + 2 * e]), __uint_as_float(v[8 * g + 2 * e + 1])), b2p[e]);
            w[e] = pack_relu_bf16x2(f2_lo(s), f2_hi(s));
          }
          st_shared_v4(h2 + (cc >> 1) * 16384 + sw128_off(row, (cc & 1) * 4 + g), w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&S.bar[B_E2K0 + c], 0);
      }
      if (lt == 0) trace_ev(a, rank, cid, it, 10);
      ++it;
      if (iter_l1.next(l1_row0, l1_nrows)) layer1(it, l1_row0, l1_nrows);
    }
  } else {
    // ============ epi L3: thread = output feature; walk rows: cell max, occupied-cell mean ============
    const uint32_t q = warp & 3;
    const uint32_t eg = warp - kWarpE3;  // 0..3: which 32-row chunks this warp flags
    const uint32_t f = 128 * rank + 32 * q + lane;
    const float b3 = a.b3[f];
    float run_max = -INFINITY, run_sum = 0.f;
    int run_cells = 0;
    TileIter iter(a, cid, ncl);
    int64_t row0;
    int nrows;
    uint32_t it = 0, c0 = 0, c1 = 0;
    while (iter.next(row0, nrows)) {
      asm volatile("bar.sync 1, 128;" ::: "memory");  // previous tile's flags no longer read
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 128 * h + 32 * eg + lane;
        const uint32_t fl = r < nrows ? __float_as_uint(a.rows[row0 + r].w) : 0u;
        S.flags[r] = fl;
        const uint32_t ce = __ballot_sync(0xffffffffu, fl & kRowFlagCellEnd);
        const uint32_t se = __ballot_sync(0xffffffffu, fl & kRowFlagSegEnd);
        if (lane == 0) {
          S.masks[4 * h + eg] = ce;
          S.masks[8 + 4 * h + eg] = se;
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (lane == 0 && eg == 0) trace_ev(a, rank, cid, it, 11);
      const int np = nrows > 128 ? 2 : 1;
      for (int p = 0; p < np; ++p) {
        mbar_wait(&S.bar[p ? B_D3F1 : B_D3F0], (p ? c1 : c0) & 1);
        if (lane == 0 && eg == 0) trace_ev(a, rank, cid, it, 12 + 2 * p);
        tc_fence_after();
        const uint32_t tbase = tmem + ((32 * q) << 16) + d3_col(it & 1, p);
        const int ncols = min(128, nrows - 128 * p);
        uint32_t va[32], vb[32];
        tmem_ld32(tbase, va);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (32 * c < ncols) {
            uint32_t(&v)[32] = (c & 1) ? vb : va;
            uint32_t(&nx)[32] = (c & 1) ? va : vb;
            tmem_ld_wait();
            if (c < 3 && 32 * (c + 1) < ncols) tmem_ld32(tbase + 32 * (c + 1), nx);
            walk_chunk(v, min(32, ncols - 32 * c), S.masks[4 * p + c], S.masks[8 + 4 * p + c],
                       S.flags + 128 * p + 32 * c, b3, run_max, run_sum, run_cells, a.pooled, f);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&S.bar[p ? B_D3E1 : B_D3E0], 0);
        if (lane == 0 && eg == 0) trace_ev(a, rank, cid, it, 13 + 2 * p);
        if (p) ++c1; else ++c0;
      }
      ++it;
    }
  }

  // ---------------------------------------------------------------- teardown
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == kWarpMMA) tmem_dealloc_2cta(tmem, kTmemCols);
}

}  // namespace

size_t encoder_tc_smem_bytes() { return sizeof(Smem) + 1024; }

cudaError_t launch_encoder_tc(const DevParams& P, const TcL1& l1, const Batch& b, int num_sms, cudaStream_t st,
                              long long* trace) {
  const int spc = 16;
  const int64_t chunks = (b.G + spc - 1) / spc;
  if (chunks == 0) return cudaSuccess;
  if (!P.tc_w2 || !P.tc_w3) return cudaErrorInvalidValue;
  (void)l1;
  TcArgs args;
  args.w1b = P.w1b;
  args.b2 = P.b2;
  args.b3 = P.b3;
  args.w2img = static_cast<const uint8_t*>(P.tc_w2);
  args.w3img = static_cast<const uint32_t*>(P.tc_w3);
  args.rows = b.rows;
  args.offsets = b.offsets;
  args.pooled = b.pooled;
  args.G = b.G;
  args.n_chunks = chunks;
  args.seg_per_chunk = spc;
  args.trace = trace;
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
