// kernels_encoder_tc.cu — S4-S7 on the 5th-generation tensor cores (LOCC_PREC_BF16).
//
// One persistent launch; CTA pairs (clusters of 2 on a TPC) run cta_group::2 tcgen05.mma with
// fp32 accumulators in TMEM.  Work unit: a chunk of whole (pair, side) segments of the compacted
// row buffer (rows sorted by segment, then cell), cut into 256-row tiles; CTA r of the pair owns
// the tile rows {64r..64r+63} and {128+64r..128+64r+63}.  Per tile:
//
//   L1 (CUDA cores, fp32 FFMA2)  h1 = ReLU(W1 p + b1) -> bf16, written as the A operand of L2
//                                (K-major, 128-byte swizzle) — PAPER.md:331, :421, :425
//   L2 (tcgen05, SS)             D2 = 1 * b2 + h1 * W2^T [256 rows x 256 features] as two N = 128
//                                halves (L2a, L2b); A = h1 (each CTA its 128 rows), B = W2 (each CTA
//                                64 rows of each half, resident in shared memory with a bias block:
//                                the first MMA of a half multiplies a column of ones with b2)
//   epi L2 (TMEM -> regs)        h2 = ReLU(D2) -> bf16, written row-major (K-major) as the B operand
//                                of L3 — each CTA keeps its own rows: no exchange
//   L3 (tcgen05, TS)             D3[256 features x 128 rows] = b3 * 1 + W3 * h2^T, twice per tile
//                                (rows 0-127, 128-255); A = W3 resident in TMEM (each CTA 128
//                                features), B = h2 (each CTA 64 of the 128 rows); the first MMA of a
//                                part multiplies b3 (three bf16 terms, in the bias block) with ones
//   epi L3 (TMEM -> regs)        thread = output feature, walking the rows in order: cell-wise max
//                                of ReLU(D3), sum over occupied cells in blocks of 16
//                                rows, mean at the segment end — e3_walk.cuh
//
// Layer 2 is computed "rows x features" and layer 3 "features x rows" so that layer 2's epilogue
// produces layer 3's operand in place and layer 3's epilogue sees each feature's rows in one
// thread — the segmented cell max needs no cross-lane reduction.
//
// Roles (17 warps): warps 0-7 = layer 1 (a warp pair per 64-feature K block of h1, the weights of its
// features in registers), warps 8-11 = epi L2, warps 12-15 = epi L3, warp 16 = TMEM allocation + MMA
// issue (leader CTA).  mbarriers link the roles across both CTAs.  h1 is handed over per K block in
// both directions (layer 1 of tile t+1 overwrites K block kb as soon as L2 of tile t has consumed it); layer 3 accumulates per 32-feature K chunk as
// epi L2 writes them; accumulators rotate over three TMEM regions (struct Regions) so that the
// tensor core runs the next tile's first layer-2 half while the epilogues still drain this one.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "internal.h"
#include "tc_ptx.cuh"
#include "e3_walk.cuh"


namespace locc {

namespace {

using namespace tc;
using namespace e3;

// Warp roles.  TMEM lane access is restricted to lane quarter (warp % 4), so each TMEM-reading
// group starts at a multiple of 4.  The warp scheduler favours higher warp ids, so the sequential
// layer-3 walk and the MMA issuer get the high ids and layer 1 (which has the most slack) the low.
// 17 warps = at most 5 per scheduler, which leaves 96 registers per thread.
constexpr int kL1Warps = 8;  // layer 1: warps 0-7, a warp pair per K block
constexpr int kL1Threads = 32 * kL1Warps;
constexpr int kE2Warps = 4;  // epi L2: warps 8-11, both halves in turn
constexpr int kWarpL1 = 0, kWarpE2 = 8, kWarpE3 = 12;
constexpr int kWarpMMA = 16;  // warp 16: TMEM allocation + MMA issue (leader CTA)
constexpr int kWarps = 17;
constexpr int kThreads = 32 * kWarps;
constexpr int kTileRows = 256;
constexpr uint32_t kTmemCols = 512;
// TMEM columns: W3 (A of L3: this CTA's 128 features as bf16x2) and three 128-column regions
// R(i) = 128 + 128 i, assigned per tile as described at struct Regions.
constexpr uint32_t kColW3 = 0, kColR0 = 128;
// The per-tile event trace (LOCC_TC_TRACE=1 at run time) is compiled in only with -DLOCC_TRACE_BUILD=1
// (tools/trace_run.py builds it; its checks cost several % of the step in the hot loops).  Events go
// to shared memory (cheap stores) and are copied out at the end of the launch.
#ifndef LOCC_TRACE_BUILD
#define LOCC_TRACE_BUILD 0
#endif
constexpr uint32_t kIdescN128 = idesc_bf16_f32(256, 128);

__device__ __forceinline__ uint32_t region_col(uint32_t i) { return kColR0 + 128 * i; }

// Layer 2 runs as two N = 128 halves (L2a: features 0-127, L2b: 128-255), layer 3 as two 128-row
// parts.  Regions: a tile's pair (P, Q) takes L2a -> P and L2b -> Q; L3p0 then reuses P once epi L2
// has drained it, and L3p1 always goes to the third region R(2), so it can start on the first K half
// (written by epi L2 from L2a) while L2b is still being drained.  The next tile swaps P and Q: its
// L2a reuses this tile's L2b region (drained before this tile's L3 finished) and its L2b the region
// of this tile's L3p0 (freed by the layer-3 epilogue).
constexpr uint32_t kRegionP1 = 2;
struct Regions {
  uint32_t P = 0, Q = 1;
  __device__ void next() {
    const uint32_t t = P;
    P = Q;
    Q = t;
  }
};

enum {
  B_H1F0 = 0, B_H1E0 = 4, B_D2AF = 8, B_D2BF, B_E2K0, B_H2_EMPTY = B_E2K0 + 8, B_D3F0, B_D3F1, B_D3E0, B_D3E1, B_WLOAD, B_PROBE, B_PROBE_END = B_PROBE + 5,
  kNumBars = B_PROBE_END
};

struct alignas(1024) Smem {
  uint8_t w2[5 * 16384];  // B of L2: this CTA's 128 W2 rows, 4 K blocks x [128 rows x 128 B], SW128,
                          // + a bias block: K = 0..2 of row i = b2 of L2 image row i, K = 16..18 of
                          // row m = b3 of this CTA's feature m, each split into three bf16 terms
  uint8_t ones[1024];     // the other operand of the bias MMAs: one 8-row SW128 atom with K = 0..2 and
                          // K = 16..18 = 1 (all rows alike: SBO = 0)
  uint8_t h1[65536];  // A of L2: this CTA's 128 rows of h1, same layout
  uint8_t h2[65536];  // B of L3: this CTA's 128 rows of h2, same layout
  float px[2][128], py[2][128], pz[2][128];  // this CTA's rows of a tile (layer-1 input), double buffered
  uint32_t flags[kTileRows];  // row flags of the whole tile (epi L3)
  alignas(16) uint32_t masks[16];  // per part p: [8p + C] cell ends, [8p + 4 + C] segment ends of step C (interleaved)
  uint64_t bar[kNumBars];
  int64_t range[2];  // this cluster's rows [range[0], range[1]) (whole segments)
  uint32_t tmem_base;
#if LOCC_TRACE_BUILD
  long long tr[32][32];  // LOCC_TC_TRACE: event clocks of the first 32 tiles, copied out at the end
#endif
};


struct TcArgs {
  const float4* w1b;      // [256] (w0, w1, w2, b1)
  const float* b3;
  const uint8_t* w2img;   // [2 ranks][5 x 16384 B] pre-swizzled (W2 + bias block)
  const uint32_t* w3img;  // [256 rows][128] bf16x2
  const uint2* rows;      // (flags, point index) per row; coordinates in pts[own K + k]
  const float4* pts;
  const float4* xf;       // per-segment transforms (own shape id in [4 seg + 3].x)
  int K;
  const int64_t* offsets;
  float* pooled;     // [G][256] cell sums (the predictor divides by cells_c)
  int32_t* cells_c;  // [G] occupied cells per segment
  int64_t G;
  int S;             // shapes (checked builds)
  int64_t rows_cap;  // rows capacity (checked builds)
  long long* trace;  // debug timeline (LOCC_TC_TRACE): [2 ranks][64 tiles][16 events] of cluster 0
};

constexpr int kTraceTiles = 64;  // tiles per rank in the trace buffer (the kernel records the first 32)
constexpr int kTraceEv = 32;     // events per tile (see tools/trace_events.py)
#if LOCC_TRACE_BUILD
#define TRACE_EV(it, ev)                                                     \
  do {                                                                       \
    if (a.trace && cid == 0 && (it) < 32) S.tr[(it)][(ev)] = clock64();     \
  } while (0)
#else
#define TRACE_EV(it, ev) \
  do {                   \
  } while (0)
#endif

// First row of the first segment whose rows start at or after `target` (offsets[G] = all rows).
__device__ int64_t seg_boundary_at(const TcArgs& a, int64_t target) {
  int64_t lo = 0, hi = a.G;  // offsets[hi] >= target always
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a.offsets[mid] >= target) hi = mid; else lo = mid + 1;
  }
  return a.offsets[lo];
}

// Iterates the tiles of this cluster's rows; every role walks the same sequence.  Each cluster owns
// one contiguous range of whole segments holding ~1/nclusters of the batch's rows (computed once per
// CTA in the setup), so only its last tile is partial.
struct TileIter {
  int64_t t0, r1;
  bool started = false;
  __device__ TileIter(int64_t begin, int64_t end) : t0(begin), r1(end) {}
  // first = true for the cluster's first tile (a range starts on a segment boundary)
  __device__ bool next(int64_t& row0, int& nrows, bool& first) {
    if (t0 >= r1) return false;
    first = !started;
    started = true;
    row0 = t0;
    nrows = (int)min((int64_t)kTileRows, r1 - t0);
    t0 += kTileRows;
    return true;
  }
  __device__ bool next(int64_t& row0, int& nrows) {
    bool f;
    return next(row0, nrows, f);
  }
};

// One warp of a role group polls the mbarrier; the others wait on a named barrier (no issue slots).
// (Spinning instead of the sleeping try_wait made no difference.)
template <int ID, int NTHREADS>
__device__ __forceinline__ void group_wait(uint64_t* bar, uint32_t parity, bool poller) {
  if (poller) mbar_wait(bar, parity);
  __syncwarp();
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(NTHREADS) : "memory");
}

__device__ __forceinline__ uint32_t tile_row_of_local(uint32_t rank, uint32_t i) {
  return i < 64 ? 64 * rank + i : 128 + 64 * rank + (i - 64);
}

// Layer-3 MMAs of K chunk j (features 32j..32j+31, written by epi L2 as one chunk): K steps 2j, 2j+1.
// A = W3 columns in TMEM (8 columns of bf16x2 per K step), B = h2 (+rowoff: descriptor offset of the
// part's 64 rows); they accumulate onto the part's bias MMA (D3 = b3 * 1).
__device__ __forceinline__ void l3_chunk(uint32_t d3, uint32_t w3, uint64_t dH2, int j, uint32_t rowoff) {
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int k = 2 * j + s;
    const uint32_t koff = (k >> 2) * 1024 + (k & 3) * 2 + rowoff;
    mma_ts_2cta(d3, w3 + 8 * k, dH2 + koff, kIdescN128, 1);
  }
}

template <bool kDet>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1) encoder_tc_kernel(const __grid_constant__ TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023));
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int64_t cid = cluster_id_x(), ncl = nclusters_x();

  // ---------------------------------------------------------------- setup
  if (threadIdx.x == 0) {
    for (int kb = 0; kb < 4; ++kb) {
      mbar_init(&S.bar[B_H1F0 + kb], 4);  // the 2 layer-1 warps of K block kb x 2 CTAs (the leader's copy is used)
      mbar_init(&S.bar[B_H1E0 + kb], 1);   // MMA commits
    }
    mbar_init(&S.bar[B_D2AF], 1);
    mbar_init(&S.bar[B_D2BF], 1);
    for (int j = 0; j < 8; ++j) mbar_init(&S.bar[B_E2K0 + j], 8);  // the 4 epi-L2 warps of a half x 2 CTAs
    mbar_init(&S.bar[B_H2_EMPTY], 1);
    mbar_init(&S.bar[B_D3F0], 1);
    mbar_init(&S.bar[B_D3F1], 1);
    mbar_init(&S.bar[B_D3E0], 8);  // 4 epi-L3 warps x 2 CTAs
    mbar_init(&S.bar[B_D3E1], 8);
    mbar_init(&S.bar[B_WLOAD], 1);
    for (int g = 0; g < 5; ++g) mbar_init(&S.bar[B_PROBE + g], 1);  // LOCC_TC_TRACE: completion probes
#if LOCC_TRACE_BUILD
    for (int i = 0; i < 32 * 32; ++i) S.tr[i / 32][i % 32] = 0;
#endif
    const int64_t R = a.offsets[a.G];
    S.range[0] = cid == 0 ? 0 : seg_boundary_at(a, R * cid / ncl);
    S.range[1] = cid + 1 == ncl ? R : seg_boundary_at(a, R * (cid + 1) / ncl);
    fence_mbar_init();
    mbar_arrive_expect_tx(&S.bar[B_WLOAD], 5 * 16384);
    for (int kb = 0; kb < 5; ++kb)
      bulk_g2s(S.w2 + kb * 16384, a.w2img + (size_t)rank * 5 * 16384 + kb * 16384, 16384, &S.bar[B_WLOAD]);
  }
  for (int i = threadIdx.x; i < 256; i += kThreads) {  // ones atom: row i>>5, 4-byte word i&31
    const uint32_t row = i >> 5, word = i & 31;
    const uint32_t chunk = (word >> 2) ^ row;  // logical 16-byte chunk of this physical word
    uint32_t v = 0;
    if ((chunk == 0 || chunk == 2) && (word & 3) == 0) v = 0x3F803F80u;  // K = 0, 1 (16, 17)
    if ((chunk == 0 || chunk == 2) && (word & 3) == 1) v = 0x00003F80u;  // K = 2 (18)
    reinterpret_cast<uint32_t*>(S.ones)[i] = v;
  }
  fence_proxy_async_smem();
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
  if (warp == kWarpMMA && rank == 1) {
    if (LOCC_TRACE_BUILD && a.trace && cid == 0 && lane == 0) {
      // debug: one thread timestamps tensor-core completions (probe barriers) in this SM's clock
      TileIter pit(S.range[0], S.range[1]);
      int64_t r0;
      int pn = 0;
      bool pmore = pit.next(r0, pn);
      uint32_t ptile = 0, pg = 0, np1 = 0;
      while (pmore) {
        const uint32_t ng = pn > 128 ? 5 : 4;  // L2a, L2b, L3p0 first K half, L3p0, L3p1
        if (mbar_try_wait(&S.bar[B_PROBE + pg], (pg == 4 ? np1 : ptile) & 1)) {
          if (ptile < 32) a.trace[(2 * kTraceTiles + ptile) * kTraceEv + pg] = clock64();
          if (++pg == ng) {
            if (ng == 5) ++np1;
            pg = 0;
            ++ptile;
            pmore = pit.next(r0, pn);
          }
        }
      }
    }
  } else if (warp == kWarpMMA) {
    // ============ MMA issuer (leader CTA, whole warp; one elected lane issues) ============
    if (rank == 0) {
      TileIter iter(S.range[0], S.range[1]);
      int64_t row0;
      int nrows;
      uint32_t it = 0, n0 = 0, n1 = 0;
      int last_p1 = -1;  // index (among all part-1s) of the last L3p1 issued: R(2)'s previous user
      Regions R;
      // descriptors are fixed for the launch: K step k of a K-major SW128 operand is +32 B (+2 in
      // the descriptor's address field) within a K block and +16384 B (+1024) per K block; the
      // second 64-row half of an operand image is +8192 B (+512)
      const uint64_t dA1 = smem_desc_sw128(smem_u32(S.h1), 1024), dW2 = smem_desc_sw128(smem_u32(S.w2), 1024);
      const uint64_t dH2 = smem_desc_sw128(smem_u32(S.h2), 1024), dOne = smem_desc_sw128(smem_u32(S.ones), 0);
      const uint64_t dB2 = dW2 + 4 * 1024;
      const uint32_t r3 = tmem + region_col(kRegionP1);
      while (iter.next(row0, nrows)) {
        const uint32_t par = it & 1;
        const bool p1 = nrows > 128;
        const uint32_t rp = tmem + region_col(R.P), rq = tmem + region_col(R.Q);
        // L2a -> P: the previous tile's L2b region, drained before that tile's L3 was issued
        if (lane == 0) { TRACE_EV(it, 1); }
        tc_fence_after();
        if (elect_one()) mma_ss_2cta(rp, dOne, dB2, kIdescN128, 0);  // D = 1 * b2 (hi + mid + lo)
        __syncwarp();
#pragma unroll 1
        for (int kb = 0; kb < 4; ++kb) {
          mbar_wait_spin(&S.bar[B_H1F0 + kb], par);
          if (kb == 0 && lane == 0) { TRACE_EV(it, 0); }
          tc_fence_after();
          if (elect_one()) {
            const uint32_t koff = kb * 1024;
#pragma unroll
            for (int s = 0; s < 4; ++s) mma_ss_2cta(rp, dA1 + koff + 2 * s, dW2 + koff + 2 * s, kIdescN128, 1);
          }
          __syncwarp();
        }
        if (elect_one()) {
          mma_commit_2cta(&S.bar[B_D2AF], 3);
          if (LOCC_TRACE_BUILD && a.trace) mma_commit_2cta(&S.bar[B_PROBE + 0], 3);
        }
        __syncwarp();
        if (lane == 0) TRACE_EV(it, 20);  // L2a issued
        // L2b -> Q: the previous tile's L3p0 region
        if (it > 0) mbar_wait_spin(&S.bar[B_D3E0], (n0 - 1) & 1);
        if (lane == 0) { TRACE_EV(it, 2); }
        tc_fence_after();
        if (elect_one()) {
          mma_ss_2cta(rq, dOne, dB2 + 512, kIdescN128, 0);
#pragma unroll
          for (int kb = 0; kb < 4; ++kb) {
            const uint32_t koff = kb * 1024;
#pragma unroll
            for (int s = 0; s < 4; ++s)
              mma_ss_2cta(rq, dA1 + koff + 2 * s, dW2 + koff + 512 + 2 * s, kIdescN128, 1);
            mma_commit_2cta(&S.bar[B_H1E0 + kb], 3);  // h1 K block kb read by both halves
          }
          mma_commit_2cta(&S.bar[B_D2BF], 3);
          if (LOCC_TRACE_BUILD && a.trace) mma_commit_2cta(&S.bar[B_PROBE + 1], 3);
        }
        __syncwarp();
        if (lane == 0) TRACE_EV(it, 21);  // L2b issued
        // Layer 3, first K half (features 0-127, from L2a): L3p0 -> P once epi L2 has drained all of
        // it, L3p1 -> R(2) once the layer-3 epilogue has walked its previous part there
#pragma unroll 1
        for (int j = 0; j < 4; ++j) mbar_wait_spin(&S.bar[B_E2K0 + j], par);
        if (lane == 0) { TRACE_EV(it, 3); }
        tc_fence_after();
        if (elect_one()) {
          // D3 = b3 (hi + mid + lo) for every row: K = 16..18 (+32 B) of the bias block and the ones atom
          mma_ss_2cta(rp, dB2 + 2, dOne + 2, kIdescN128, 0);
#pragma unroll
          for (int j = 0; j < 4; ++j) l3_chunk(rp, tmem + kColW3, dH2, j, 0);
          if (LOCC_TRACE_BUILD && a.trace) mma_commit_2cta(&S.bar[B_PROBE + 2], 3);
        }
        __syncwarp();
        if (lane == 0) TRACE_EV(it, 22);  // L3p0 first half issued
        if (p1) {
          if (last_p1 >= 0) mbar_wait_spin(&S.bar[B_D3E1], last_p1 & 1);
          tc_fence_after();
          if (elect_one()) {
            mma_ss_2cta(r3, dB2 + 2, dOne + 2, kIdescN128, 0);
#pragma unroll
            for (int j = 0; j < 4; ++j) l3_chunk(r3, tmem + kColW3, dH2, j, 512);
          }
          __syncwarp();
          if (lane == 0) TRACE_EV(it, 23);  // L3p1 first half issued
        }
        // second K half (features 128-255) chunk by chunk as epi L2 writes it
#pragma unroll 1
        for (int j = 4; j < 8; ++j) {
          mbar_wait_spin(&S.bar[B_E2K0 + j], par);
          if (lane == 0) TRACE_EV(it, 12 + j);  // 16..19: chunk j of h2 seen
          tc_fence_after();
          if (elect_one()) {
            l3_chunk(rp, tmem + kColW3, dH2, j, 0);
            if (j == 7) {
              mma_commit_2cta(&S.bar[B_D3F0], 3);
              if (LOCC_TRACE_BUILD && a.trace) mma_commit_2cta(&S.bar[B_PROBE + 3], 3);
            }
            if (p1) l3_chunk(r3, tmem + kColW3, dH2, j, 512);
          }
          __syncwarp();
        }
        if (lane == 0) { TRACE_EV(it, 4); }
        if (elect_one()) {
          if (p1) {
            mma_commit_2cta(&S.bar[B_D3F1], 3);
            if (LOCC_TRACE_BUILD && a.trace) mma_commit_2cta(&S.bar[B_PROBE + 4], 3);
          }
          mma_commit_2cta(&S.bar[B_H2_EMPTY], 3);
        }
        __syncwarp();
        if (p1) {
          if (lane == 0) { TRACE_EV(it, 5); }
          last_p1 = (int)n1;
          ++n1;
        }
        R.next();
        ++n0;
        ++it;
      }
    }
  } else if (warp >= kWarpL1 && warp < kWarpL1 + kL1Warps) {
    // ============ layer 1: a warp pair per K block kb; thread = features 64kb + 4fq .. +3 (their
    // weights in registers for the whole launch, as fp32 pairs of adjacent features) x local rows
    // 32rg .. 32rg + 31; FFMA2 with the row's coordinate as the broadcast operand ============
    const uint32_t lt = threadIdx.x - 32 * kWarpL1;  // 0..255
    const uint32_t wl = lt >> 5, kb = wl >> 1;
    const uint32_t fq = lane & 15, rg = 2 * (wl & 1) + (lane >> 4);
    unsigned long long wA[4], wB[4];  // (w0, w1, w2, b1) of features (4fq, 4fq+1) and (4fq+2, 4fq+3)
    {
      const float4* w = a.w1b + 64 * kb + 4 * fq;
      const float4 f0 = w[0], f1 = w[1], f2_ = w[2], f3 = w[3];
      wA[0] = f2(f0.x, f1.x); wA[1] = f2(f0.y, f1.y); wA[2] = f2(f0.z, f1.z); wA[3] = f2(f0.w, f1.w);
      wB[0] = f2(f2_.x, f3.x); wB[1] = f2(f2_.y, f3.y); wB[2] = f2(f2_.z, f3.z); wB[3] = f2(f2_.w, f3.w);
    }
    const uint32_t h1 = smem_u32(S.h1) + kb * 16384 + ((4 * fq) & 7) * 2;
    const uint32_t chunk = (4 * fq) >> 3;  // 16-byte chunk of the 128-byte row
    TileIter iter(S.range[0], S.range[1]), ahead(S.range[0], S.range[1]);
    int64_t row0, nrow0;
    int nrows, nnrows;
    auto stage = [&](float4 p, uint32_t buf) {
      if (lt < 128) {
        S.px[buf][lt] = p.x;
        S.py[buf][lt] = p.y;
        S.pz[buf][lt] = p.z;
      }
    };
    auto fetch = [&](bool ok, int64_t r0, int nr) {
      float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ok && lt < 128) {
        const uint32_t trow = tile_row_of_local(rank, lt);
        if ((int)trow < nr) {
          LOCC_CHECK(r0 + trow < a.offsets[a.G] && r0 + trow < a.rows_cap);
          const uint2 rw = a.rows[r0 + trow];
          LOCC_CHECK((rw.x >> kRowSegShift) < a.G && rw.y < (uint32_t)a.K);
          const int own = __float_as_int(a.xf[4 * (int64_t)(rw.x >> kRowSegShift) + 3].x);
          LOCC_CHECK((unsigned)own < (unsigned)a.S);
          p = a.pts[(int64_t)own * a.K + rw.y];
        }
      }
      return p;
    };
    bool have_next = ahead.next(nrow0, nnrows);
    stage(fetch(have_next, nrow0, nnrows), 0);
    uint32_t it = 0;
    while (iter.next(row0, nrows)) {
      const uint32_t buf = it & 1;
      asm volatile("bar.sync 2, %0;" ::"n"(kL1Threads) : "memory");  // rows of tile it staged; buffer buf^1 free
      have_next = ahead.next(nrow0, nnrows);
      const float4 pf = fetch(have_next, nrow0, nnrows);  // next tile's row, in flight during this tile
      // K block kb free (layer 2 of the previous tile has read it): one warp of the pair polls
      if ((wl & 1) == 0) mbar_wait(&S.bar[B_H1E0 + kb], (it & 1) ^ 1);
      __syncwarp();
      asm volatile("bar.sync %0, 64;" ::"r"(5 + kb) : "memory");
      if (lt == 0) TRACE_EV(it, 6);
#pragma unroll 1  // (unrolled x2 was 0.5 % slower: instruction-cache footprint)
      for (uint32_t g = 0; g < 8; ++g) {  // local rows lr .. lr + 3
        const uint32_t lr = 32 * rg + 4 * g;
        const float4 x = *reinterpret_cast<const float4*>(&S.px[buf][lr]);
        const float4 y = *reinterpret_cast<const float4*>(&S.py[buf][lr]);
        const float4 z = *reinterpret_cast<const float4*>(&S.pz[buf][lr]);
        const float xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w}, zs[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const unsigned long long X = f2(xs[v], xs[v]), Y = f2(ys[v], ys[v]), Z = f2(zs[v], zs[v]);
          const unsigned long long hA = ffma2(wA[0], X, ffma2(wA[1], Y, ffma2(wA[2], Z, wA[3])));
          const unsigned long long hB = ffma2(wB[0], X, ffma2(wB[1], Y, ffma2(wB[2], Z, wB[3])));
          st_shared_v2(h1 + sw128_off(lr + v, chunk),
                       pack_relu_bf16x2(f2_lo(hA), f2_hi(hA)), pack_relu_bf16x2(f2_lo(hB), f2_hi(hB)));
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&S.bar[B_H1F0 + kb], 0);
      if (lt == 0) TRACE_EV(it, 7);
      stage(pf, buf ^ 1);
      ++it;
    }
  } else if (warp >= kWarpE2 && warp < kWarpE2 + kE2Warps) {
    // ============ epi L2: thread = row; the two halves in turn ============
    const uint32_t q = warp & 3;  // TMEM lane quarter (rows 32q..32q+31)
    const uint32_t row = 32 * q + lane;
    const uint32_t lt = threadIdx.x - 32 * kWarpE2;
    const uint32_t h2 = smem_u32(S.h2);
    TileIter iter(S.range[0], S.range[1]);
    int64_t row0;
    int nrows;
    uint32_t it = 0;
    Regions R;
    while (iter.next(row0, nrows)) {
#pragma unroll 1
      for (uint32_t half = 0; half < 2; ++half) {
        if ((warp & 3) == 0) {  // one warp per group polls; the group waits on a named barrier
          mbar_wait(&S.bar[half ? B_D2BF : B_D2AF], it & 1);
          if (lt == 0) TRACE_EV(it, half ? 11 : 8);  // D2AF / D2BF seen
          if (half == 0) mbar_wait(&S.bar[B_H2_EMPTY], (it & 1) ^ 1);
          if (lt == 0 && half == 0) TRACE_EV(it, 9);
        }
        __syncwarp();
        asm volatile("bar.sync 3, 128;" ::: "memory");
        tc_fence_after();
        const uint32_t tbase = tmem + ((32 * q) << 16) + region_col(half ? R.Q : R.P);
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
          for (int g = 0; g < 4; ++g) {  // D2 already holds the bias (see the MMA issuer)
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              w[e] = pack_relu_bf16x2(__uint_as_float(v[8 * g + 2 * e]), __uint_as_float(v[8 * g + 2 * e + 1]));
            st_shared_v4(h2 + (cc >> 1) * 16384 + sw128_off(row, (cc & 1) * 4 + g), w[0], w[1], w[2], w[3]);
          }
          fence_proxy_async_smem();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(&S.bar[B_E2K0 + 4 * half + c], 0);
        }
      }
      if (lt == 0) TRACE_EV(it, 10);
      ++it;
      R.next();
    }
  } else {
    // ============ epi L3: thread = output feature; walk rows: cell max, occupied-cell mean ============
    const uint32_t q = warp & 3;
    const uint32_t eg = warp - kWarpE3;  // 0..3: flags of rows 32eg.. and the masks of step eg
    const uint32_t f = 128 * rank + 32 * q + lane;
    Walk w{0.f, 0.f, 0};
    TileIter iter(S.range[0], S.range[1]);
    int64_t row0;
    int nrows;
    bool first;
    uint32_t it = 0, c0 = 0, c1 = 0;
    Regions R;
    while (iter.next(row0, nrows, first)) {
      if (first) w.m = 0.f;
      asm volatile("bar.sync 1, 128;" ::: "memory");  // previous tile's flags no longer read
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 128 * h + 32 * eg + lane;
        S.flags[r] = r < nrows ? a.rows[row0 + r].x : 0u;
        LOCC_CHECK(r >= nrows || (row0 + r < a.offsets[a.G] && (S.flags[r] >> kRowSegShift) < a.G));
        const int r2 = interleaved_row(h, eg, lane);  // interleaved masks of step eg of part h
        const uint32_t fl = r2 < nrows ? a.rows[row0 + r2].x : 0u;
        const uint32_t ce = __ballot_sync(0xffffffffu, fl & kRowFlagCellEnd);
        const uint32_t se = __ballot_sync(0xffffffffu, fl & kRowFlagSegEnd);
        if (lane == 0) {
          S.masks[8 * h + eg] = ce;
          S.masks[8 * h + 4 + eg] = se;
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int np = nrows > 128 ? 2 : 1;
#pragma unroll 1
      for (int p = 0; p < np; ++p) {
        group_wait<1, 128>(&S.bar[p ? B_D3F1 : B_D3F0], (p ? c1 : c0) & 1, warp == kWarpE3);
        if (lane == 0 && eg == 0) TRACE_EV(it, 12 + 2 * p);
        tc_fence_after();
        const uint32_t tb = tmem + ((32 * q) << 16) + region_col(p ? kRegionP1 : R.P);
        if (kDet)
          e3_part2_det(tb, S.masks + 8 * p, S.flags + 128 * p, w, a.pooled, a.cells_c, f);
        else
          e3_part2(tb, S.masks + 8 * p, S.flags + 128 * p, w, a.pooled, a.cells_c, f);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&S.bar[p ? B_D3E1 : B_D3E0], 0);
        if (lane == 0) TRACE_EV(it, 24 + 4 * p + eg);  // 24..31: each E3 warp's part p done
        if (lane == 0 && eg == 0) TRACE_EV(it, 13 + 2 * p);
        if (p) ++c1; else ++c0;
      }
      ++it;
      R.next();
    }
  }

  // ---------------------------------------------------------------- teardown
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == kWarpMMA) tmem_dealloc_2cta(tmem, kTmemCols);
#if LOCC_TRACE_BUILD
  if (a.trace && cid == 0)
    for (int i = threadIdx.x; i < 32 * 32; i += kThreads) a.trace[(rank * kTraceTiles + i / 32) * kTraceEv + i % 32] = S.tr[i / 32][i % 32];
#endif
}

}  // namespace

size_t encoder_tc_smem_bytes() { return sizeof(Smem) + 1024; }

cudaError_t launch_encoder_tc(const DevParams& P, const TcL1& l1, const Batch& b, int num_sms, cudaStream_t st,
                              long long* trace, bool deterministic) {
  // Work unit: each cluster takes one contiguous range of whole segments with ~1/clusters of the rows
  // (the kernel splits the batch by its row offsets); a batch of G segments needs at most G clusters.
  if (b.G == 0) return cudaSuccess;
  const int64_t clusters = std::min<int64_t>(num_sms / 2, b.G);
  if (!P.tc_w2 || !P.tc_w3) return cudaErrorInvalidValue;
  (void)l1;
  TcArgs args;
  args.w1b = P.w1b;
  args.b3 = P.b3;
  args.w2img = static_cast<const uint8_t*>(P.tc_w2);
  args.w3img = static_cast<const uint32_t*>(P.tc_w3);
  args.rows = b.rows;
  args.pts = b.pts;
  args.xf = b.xf;
  args.K = b.K;
  args.offsets = b.offsets;
  args.pooled = b.pooled;
  args.cells_c = b.cells_c;
  if (!b.cells_c) return cudaErrorInvalidValue;
  args.G = b.G;
  args.S = b.S;
  args.rows_cap = b.rows_cap;
  args.trace = trace;
  const size_t smem = encoder_tc_smem_bytes();
  const cudaError_t attr = deterministic ? smem_optin(encoder_tc_kernel<true>, smem)
                                         : smem_optin(encoder_tc_kernel<false>, smem);
  if (attr != cudaSuccess) return attr;
  const int grid = (int)(2 * clusters);
  if (deterministic)
    encoder_tc_kernel<true><<<grid, kThreads, smem, st>>>(args);
  else
    encoder_tc_kernel<false><<<grid, kThreads, smem, st>>>(args);
  return cudaGetLastError();
}

}  // namespace locc
