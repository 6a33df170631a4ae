// kernels_geom.cu — S0 shape prep, S1 relative transforms, S2-S3 transform + crop + compaction.
//
// Geometry is prescribed arithmetic so that crop masks, kept counts and
// occupied-cell counts are bit-exact across implementations: every fp64/fp32 operation below is
// an explicit round-to-nearest intrinsic, so nvcc cannot contract or reorder it.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"
#include "geom.cuh"
#include "quat.cuh"

namespace locc {
namespace {

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- S0 shape prep
// AABB ("compute the AABB of each object's mesh"), eps = half the cell diagonal of
// this shape used when it is the counter object (a3^3 read as a3^2), cell ids
// floor((p - lo) * M / ext) clamped to M-1.
__global__ void shape_bounds_kernel(const float* __restrict__ in, int K, int M, float4* __restrict__ lo_out,
                                    float4* __restrict__ hi_out, uint16_t* __restrict__ cell_tmp,
                                    int* __restrict__ bad) {
  const int s = blockIdx.x;
  const float* p = in + (int64_t)s * K * 3;
  float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  int nonfinite = 0;
  for (int k = threadIdx.x; k < K; k += blockDim.x)
    for (int d = 0; d < 3; ++d) {
      float v = p[3 * k + d];
      nonfinite |= !isfinite(v);
      mn[d] = fminf(mn[d], v);
      mx[d] = fmaxf(mx[d], v);
    }
  __shared__ float red[2][3][32];
  __shared__ int nf_any;
  if (threadIdx.x == 0) nf_any = 0;
  __syncthreads();
  for (int d = 0; d < 3; ++d)
    for (int o = 16; o; o >>= 1) {
      mn[d] = fminf(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
      mx[d] = fmaxf(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
    }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (nonfinite) atomicOr(&nf_any, 1);
  if (l == 0)
    for (int d = 0; d < 3; ++d) {
      red[0][d][w] = mn[d];
      red[1][d][w] = mx[d];
    }
  __syncthreads();
  __shared__ float lo_s[3], hi_s[3];
  __shared__ double ext_s[3];
  if (threadIdx.x == 0) {
    double a[3];
    for (int d = 0; d < 3; ++d) {
      float a0 = red[0][d][0], b0 = red[1][d][0];
      for (int i = 1; i < nw; ++i) {
        a0 = fminf(a0, red[0][d][i]);
        b0 = fmaxf(b0, red[1][d][i]);
      }
      lo_s[d] = a0;
      hi_s[d] = b0;
      ext_s[d] = __dsub_rn((double)b0, (double)a0);
      a[d] = __ddiv_rn(ext_s[d], (double)M);
    }
    const double e2 = __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dmul_rn(a[0], a[0]), __dmul_rn(a[1], a[1])),
                                                __dmul_rn(a[2], a[2])));
    lo_out[s] = make_float4(lo_s[0], lo_s[1], lo_s[2], __double2float_rn(e2));
    hi_out[s] = make_float4(hi_s[0], hi_s[1], hi_s[2], 0.f);
    if (nf_any) atomicOr(bad, 1);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    int c[3];
    for (int d = 0; d < 3; ++d) {
      const double ext = ext_s[d];
      if (ext == 0.0) {
        c[d] = 0;
        continue;
      }
      const double u = __ddiv_rn(__dmul_rn(__dsub_rn((double)p[3 * k + d], (double)lo_s[d]), (double)M), ext);
      const double f = floor(u);
      c[d] = f >= (double)(M - 1) ? M - 1 : (int)f;
    }
    cell_tmp[(int64_t)s * K + k] = (uint16_t)(c[0] + M * (c[1] + M * c[2]));
  }
}

// Stable counting sort of each shape's points by cell id: points of one cell become contiguous
// and keep their caller order, so a compacted crop is already grouped by cell (the encoder's
// cell-wise max pool then walks runs).  perm maps the sorted slot back to the caller's index.
__global__ void shape_sort_kernel(const float* __restrict__ in, int K, int M, const uint16_t* __restrict__ cell_tmp,
                                  float4* __restrict__ pts, uint16_t* __restrict__ perm) {
  extern __shared__ int cnt[];  // [M^3]
  const int s = blockIdx.x, nc = M * M * M;
  const uint16_t* cell = cell_tmp + (int64_t)s * K;
  for (int c = threadIdx.x; c < nc; c += blockDim.x) cnt[c] = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) atomicAdd(&cnt[cell[k]], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int c = 0; c < nc; ++c) {
      int v = cnt[c];
      cnt[c] = run;
      run += v;
    }
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const float* p = in + (int64_t)s * K * 3;
  for (int base = 0; base < K; base += 32) {
    const int k = base + lane;
    const bool valid = k < K;
    const int c = valid ? (int)cell[k] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, c);
    const int rank = __popc(peers & lanemask_lt());
    int pos = 0;
    if (valid) pos = cnt[c] + rank;
    __syncwarp();
    if (valid && rank == 0) cnt[c] += __popc(peers);
    __syncwarp();
    if (valid) {
      pts[(int64_t)s * K + pos] = make_float4(p[3 * k], p[3 * k + 1], p[3 * k + 2], __int_as_float(c));
      perm[(int64_t)s * K + pos] = (uint16_t)k;
    }
  }
}

// ---------------------------------------------------------------- S1 per segment
// One thread per (pair, side) segment: validate the inputs and write the transform (segment_setup's
// prescribed fp64 arithmetic, rounded once to fp32) for the crop and cell-selection kernels.
__global__ void __launch_bounds__(128) segment_xf_kernel(ShapeTable T, Batch b) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= b.G) return;
  int own = -1, other = -1;
  Xf X{};
  if (!segment_setup(T, b, g, own, other, X)) {
    own = other = -1;
    atomicAdd(&b.stats->bad_input, 1ull);
  }
  float4* x = b.xf + 4 * g;
  x[0] = make_float4(X.R[0], X.R[1], X.R[2], X.t[0]);
  x[1] = make_float4(X.R[3], X.R[4], X.R[5], X.t[1]);
  x[2] = make_float4(X.R[6], X.R[7], X.R[8], X.t[2]);
  x[3] = make_float4(__int_as_float(own), __int_as_float(other), 0.f, 0.f);
}

// ---------------------------------------------------------------- S2-S3 pass 1: counts
// One warp per segment: float4 point loads (coalesced, 512 B per warp step), fp32 transform +
// eps test, warp ballot.  Writes n_s and C_s (occupied cells among the kept points: cell runs,
// the points being cell-sorted) and, in debug mode, the caller-order keep mask.
// kOcc: also count the occupied cells C_s (only when the caller asked for them: a debug output).
template <bool kOcc>
__global__ void __launch_bounds__(256) crop_count_kernel(ShapeTable T, Batch b, int words) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= b.G) return;
  int own = 0, other = 0;
  Xf X;
  if (!segment_load(b, g, own, other, X)) {
    if (lane == 0) {
      b.counts[g] = 0;
      b.occ[g] = 0;
    }
    return;
  }
  LOCC_CHECK((unsigned)own < (unsigned)T.S && (unsigned)other < (unsigned)T.S);
  const float4 lo = T.lo[other], hi = T.hi[other];
  const float4* pts = T.pts + (int64_t)own * T.K;
  const uint16_t* perm = T.perm + (int64_t)own * T.K;
  uint32_t* mask = b.masks ? b.masks + g * words : nullptr;
  uint32_t* kb = b.kbits + g * ((T.K + 31) >> 5);
  int n = 0, C = 0, carry = -1;
  // four 32-point steps per round: their loads are in flight together (the table lives in L2)
  for (int base0 = 0; base0 < T.K; base0 += 128) {
    float4 pp[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = base0 + 32 * j + lane;
      pp[j] = k < T.K ? pts[k] : make_float4(0.f, 0.f, 0.f, __int_as_float(-2));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
    const int base = base0 + 32 * j;
    if (base >= T.K) break;
    const int k = base + lane;
    const float4 p = pp[j];
    const bool keep = k < T.K && keep_point(X, p.x, p.y, p.z, lo, hi);
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) kb[base >> 5] = m;  // the emit pass replays these decisions
    if (m == 0) continue;
    if (kOcc) {
      const int cell = __float_as_int(p.w);
      const unsigned before = m & lanemask_lt();
      const int src = before ? 31 - __clz(before) : lane;
      int prev = __shfl_sync(0xffffffffu, cell, src);
      if (!before) prev = carry;
      C += __popc(__ballot_sync(0xffffffffu, keep && prev != cell));
      carry = __shfl_sync(0xffffffffu, cell, 31 - __clz(m));
    }
    n += __popc(m);
    if (mask && keep) {
      const int ck = perm[k];
      atomicOr(mask + (ck >> 5), 1u << (ck & 31));
    }
    }
  }
  if (lane == 0) {
    b.counts[g] = n;
    if (kOcc) b.occ[g] = C;
    if (n) {
      atomicAdd(&b.stats->kept_rows, (unsigned long long)n);
      atomicAdd(&b.stats->nonempty_sides, 1ull);
    }
  }
}

// ---------------------------------------------------------------- S2-S3 pass 2: compaction
// Same keep decisions (same function), rows written densely at offsets[g] in cell-sorted order:
// (x, y, z) in the object's LOCAL frame (the encoder input, reading Q6) and a flags word
// (segment << 2 | last-of-segment << 1 | last-of-cell).  "Last of cell" needs the next kept
// point, so the last kept point of each 32-point step is held back until the next step.
__global__ void __launch_bounds__(256) crop_emit_kernel(ShapeTable T, Batch b) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= b.G) return;
  const int n = b.counts[g];
  if (n == 0) return;
  int own = 0, other = 0;
  Xf X;
  if (!segment_load(b, g, own, other, X)) return;
  const float4* pts = T.pts + (int64_t)own * T.K;
  const int nsteps = (T.K + 31) >> 5;
  const uint32_t* kb = b.kbits + g * nsteps;
  LOCC_CHECK((unsigned)own < (unsigned)T.S);
  LOCC_CHECK(b.offsets[g] >= 0 && b.offsets[g] + seg_rows(n) <= b.rows_cap &&
             b.offsets[g + 1] - b.offsets[g] == seg_rows(n));
  uint2* out = b.rows + b.offsets[g];
  const uint32_t segbits = (uint32_t)g << kRowSegShift;
  int written = 0;        // kept rows before this step
  bool pending = false;   // a held-back row (warp-uniform)
  int pk = 0;             // held-back row's point index (valid in every lane)
  int pcell = 0, pidx = 0;
  for (int base0 = 0; base0 < T.K; base0 += 128) {
    // four steps in flight together: the count pass's ballots, then only the kept points' loads
    float4 pp[4];
    unsigned mm[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int step = (base0 >> 5) + j;
      mm[j] = step < nsteps ? kb[step] : 0u;
      const int k = base0 + 32 * j + lane;
      pp[j] = (mm[j] >> lane) & 1u ? pts[k] : make_float4(0.f, 0.f, 0.f, __int_as_float(-2));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
    const int base = base0 + 32 * j;
    if (base >= T.K) break;
    const float4 p = pp[j];
    const unsigned m = mm[j];
    const bool keep = (m >> lane) & 1u;
    if (m == 0) continue;
    const int cell = __float_as_int(p.w);
    const int first = __ffs(m) - 1, last = 31 - __clz(m);
    const unsigned after = m & ~(0xffffffffu >> (31 - lane));  // kept lanes above this one
    const int nxt = after ? __ffs(after) - 1 : lane;
    const int next_cell = __shfl_sync(0xffffffffu, cell, nxt);
    const int first_cell = __shfl_sync(0xffffffffu, cell, first);
    if (pending && lane == 0) {
      LOCC_CHECK(pidx >= 0 && pidx < n);
      const uint32_t f = segbits | (pcell != first_cell ? kRowFlagCellEnd : 0);
      out[pidx] = make_uint2(f, (uint32_t)pk);
    }
    const int idx = written + __popc(m & lanemask_lt());
    const int k = base + lane;
    if (keep && lane != last) {
      LOCC_CHECK(idx < n);
      const uint32_t f = segbits | (cell != next_cell ? kRowFlagCellEnd : 0);
      out[idx] = make_uint2(f, (uint32_t)k);
    }
    pk = __shfl_sync(0xffffffffu, k, last);
    pcell = __shfl_sync(0xffffffffu, cell, last);
    pidx = written + __popc(m) - 1;
    pending = true;
    written += __popc(m);
    }
  }
  if (pending && lane == 0) {
    const uint32_t f = segbits | kRowFlagCellEnd | kRowFlagSegEnd;
    out[pidx] = make_uint2(f, (uint32_t)pk);
  }
  // padding up to the next multiple of kSegAlign rows
  const int pad_end = (int)seg_rows(n);
  for (int i = n + lane; i < pad_end; i += 32) out[i] = make_uint2(segbits | kRowFlagPad, 0u);
}

// ---------------------------------------------------------------- S2-S3 fused: transform + crop + compaction
// One kernel for the whole crop (K <= kFusedMaxK).  A block of kCropWarps warps takes kCropWarps
// consecutive segments (one per warp); blocks claim their segment ranges in order from a counter, so
// every predecessor of a claimed range is already running.
//   1. Per warp: float4 point loads (four 32-point steps in flight), the transform + eps test, a warp
//      ballot; each kept point's sorted index k and its "last of cell" bit (the next kept point's cell
//      differs) go to the warp's shared-memory list at its rank (ballot prefix count): the count pass
//      and the row staging are one pass over the points.
//   2. The block's footprints seg_rows(n) are scanned in shared memory; warp 0 runs a decoupled
//      look-back over the blocks: it publishes the block's aggregate, sums its predecessors' (32 per
//      round, lane-parallel) back to the first one that has published an inclusive prefix, and
//      publishes its own.  lb[t] = flag << 62 | value, flag 1 = aggregate, 2 = inclusive prefix, 0 =
//      not yet (lb zeroed before the launch; lb[nblocks] is the claim counter).
//   3. Each warp's staged rows leave as the encoder's 8-byte rows at its offset (coalesced), then the
//      padding.
// Same keep decisions, counts, occupied cells, debug masks and row words as crop_count + scan +
// crop_emit, which remain for K > kFusedMaxK (tests/test_parity_gpu.py checks the two bitwise equal).
constexpr int kCropWarps = 8;
constexpr unsigned long long kLbAgg = 1ull << 62, kLbPre = 2ull << 62, kLbVal = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// keep_point with the x and y rows of the transform and of the box test as pairs (FFMA2/FADD2 with the
// point's coordinates as broadcast operands): each element's arithmetic and rounding are keep_point's,
// so the decisions are bitwise the same.  Rxy[j] = (R[j], R[3 + j]), txy = (t0, t1), loxy/hixy likewise.
struct Xf2 {
  float2 Rxy[3], txy, loxy, nhixy;  // nhixy = -(hi.x, hi.y)
  float Rz[3], tz, loz, nhiz, eps2;
};

__device__ __forceinline__ bool keep_point_xy(const Xf2& Q, const float4& p) {
  const float2 x = make_float2(p.x, p.x), y = make_float2(p.y, p.y), z = make_float2(p.z, p.z);
  const float2 pxy = __ffma2_rn(Q.Rxy[0], x, __ffma2_rn(Q.Rxy[1], y, __ffma2_rn(Q.Rxy[2], z, Q.txy)));
  const float pz = __fmaf_rn(Q.Rz[0], p.x, __fmaf_rn(Q.Rz[1], p.y, __fmaf_rn(Q.Rz[2], p.z, Q.tz)));
  const float2 l = __fadd2_rn(Q.loxy, make_float2(-pxy.x, -pxy.y)), h = __fadd2_rn(pxy, Q.nhixy);
  const float dx = fmaxf(fmaxf(l.x, h.x), 0.f), dy = fmaxf(fmaxf(l.y, h.y), 0.f);
  const float dz = fmaxf(fmaxf(__fsub_rn(Q.loz, pz), __fadd_rn(pz, Q.nhiz)), 0.f);
  return __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, __fmul_rn(dz, dz))) <= Q.eps2;
}

template <bool kOcc>
__global__ void __launch_bounds__(32 * kCropWarps) crop_compact_kernel(ShapeTable T, Batch b, int words,
                                                                      unsigned long long* __restrict__ lb,
                                                                      int64_t nblocks) {
  extern __shared__ uint32_t crop_list[];
  __shared__ int64_t s_tile;
  __shared__ uint32_t s_foot[kCropWarps];
  __shared__ unsigned long long s_off[kCropWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cap = (T.K + 31) & ~31;
  uint32_t* list = crop_list + w * cap;  // each kept point in order: sorted index k | cell id << 16
  const uint32_t list_sa = (uint32_t)__cvta_generic_to_shared(list);
  if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(lb + nblocks, 1ull);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t g = tile * kCropWarps + w;
  int own = 0, other = 0;
  Xf X;
  int n = 0, C = 0;
  if (g < b.G && segment_load(b, g, own, other, X)) {
    LOCC_CHECK((unsigned)own < (unsigned)T.S && (unsigned)other < (unsigned)T.S);
    const float4 lo = T.lo[other], hi = T.hi[other];
    Xf2 Q;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      Q.Rxy[j] = make_float2(X.R[j], X.R[3 + j]);
      Q.Rz[j] = X.R[6 + j];
    }
    Q.txy = make_float2(X.t[0], X.t[1]);
    Q.tz = X.t[2];
    Q.loxy = make_float2(lo.x, lo.y);
    Q.nhixy = make_float2(-hi.x, -hi.y);
    Q.loz = lo.z;
    Q.nhiz = -hi.z;
    Q.eps2 = lo.w;
    const float4* pts = T.pts + (int64_t)own * T.K;
    const uint16_t* perm = T.perm + (int64_t)own * T.K;
    uint32_t* mask = b.masks ? b.masks + g * words : nullptr;
    int carry = -1;
    for (int base0 = 0; base0 < T.K; base0 += 128) {
      float4 pp[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = base0 + 32 * j + lane;
        pp[j] = k < T.K ? pts[k] : make_float4(0.f, 0.f, 0.f, __int_as_float(-2));
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = base0 + 32 * j + lane;
        const bool keep = k < T.K && keep_point_xy(Q, pp[j]);
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (m == 0) continue;
        if (keep) {
          const int idx = n + __popc(m & lanemask_lt());
          LOCC_CHECK(idx < cap);
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(list_sa + 4u * idx),
                       "r"((uint32_t)k | (uint32_t)__float_as_int(pp[j].w) << 16) : "memory");
          if (mask) {
            const int ck = perm[k];
            atomicOr(mask + (ck >> 5), 1u << (ck & 31));
          }
        }
        if (kOcc) {  // occupied cells: kept points whose cell differs from the previous kept point's
          const int cell = __float_as_int(pp[j].w);
          const unsigned before = m & lanemask_lt();
          int prev = __shfl_sync(0xffffffffu, cell, before ? 31 - __clz(before) : lane);
          if (!before) prev = carry;
          C += __popc(__ballot_sync(0xffffffffu, keep && prev != cell));
          carry = __shfl_sync(0xffffffffu, cell, 31 - __clz(m));
        }
        n += __popc(m);
      }
    }
  }
  if (lane == 0) s_foot[w] = (uint32_t)seg_rows(n);
  __syncthreads();
  // ---- 2. block scan + decoupled look-back over the blocks (warp 0)
  if (w == 0) {
    uint32_t f = lane < kCropWarps ? s_foot[lane] : 0u, x = f;
#pragma unroll
    for (int o = 1; o < kCropWarps; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const unsigned long long agg = __shfl_sync(0xffffffffu, x, kCropWarps - 1);
    if (lane == 0) st_relaxed_u64(lb + tile, (tile == 0 ? kLbPre : kLbAgg) | agg);
    unsigned long long excl = 0;
    if (tile > 0) {
      for (int64_t hi = tile - 1;; hi -= 32) {
        const int64_t i = hi - lane;
        unsigned long long v = kLbPre;  // before block 0: prefix 0
        if (i >= 0) {
          v = ld_relaxed_u64(lb + i);
          for (unsigned ns = 32; (v >> 62) == 0; ns = ns < 256 ? 2 * ns : ns) {
            __nanosleep(ns);
            v = ld_relaxed_u64(lb + i);
          }
        }
        const unsigned pm = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        const int lim = pm ? __ffs(pm) - 1 : 31;  // lanes 0..lim: aggregates, then lim's inclusive prefix
        unsigned long long y = lane <= lim ? (v & kLbVal) : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
        excl += y;
        if (pm) break;
      }
      if (lane == 0) st_relaxed_u64(lb + tile, kLbPre | (excl + agg));
    }
    if (lane < kCropWarps) s_off[lane] = excl + x - f;
    if (lane == 0 && (tile + 1) * kCropWarps >= b.G) b.offsets[b.G] = (int64_t)(excl + agg);
  }
  __syncthreads();
  if (g >= b.G) return;
  // ---- 3. rows out
  const unsigned long long off = s_off[w], foot = s_foot[w];
  if (lane == 0) {
    b.offsets[g] = (int64_t)off;
    b.counts[g] = n;
    if (kOcc) b.occ[g] = C;
    if (n) {
      atomicAdd(&b.stats->kept_rows, (unsigned long long)n);
      atomicAdd(&b.stats->nonempty_sides, 1ull);
    }
  }
  LOCC_CHECK((int64_t)(off + foot) <= b.rows_cap);
  __syncwarp();  // the list was written by every lane
  uint2* out = b.rows + off;
  const uint32_t segbits = (uint32_t)g << kRowSegShift;
  // a row ends its cell iff the next kept row's cell differs (the last row ends cell and segment)
  for (int i = lane; i < (int)foot; i += 32) {
    uint2 r = make_uint2(segbits | kRowFlagPad, 0u);
    if (i < n) {
      const uint32_t e = list[i], nx = i + 1 < n ? list[i + 1] : 0xffff0000u;
      r = make_uint2(segbits | ((e ^ nx) >> 16 ? kRowFlagCellEnd : 0) | (i == n - 1 ? kRowFlagSegEnd : 0), e & 0xffffu);
    }
    out[i] = r;
  }
}

// ---------------------------------------------------------------- exclusive scan of segment footprints
// Block size of the scan kernels: 256 threads, so that a scan block fits next to a persistent encoder
// CTA (the overlapped crop pipeline).
constexpr int kScanBS = 256;

__global__ void __launch_bounds__(kScanBS) scan_blocks_kernel(const int32_t* __restrict__ in, int64_t G,
                                                              int64_t* __restrict__ out, int64_t* __restrict__ sums) {
  __shared__ int64_t ws[kScanBS / 32];
  const int64_t i = (int64_t)blockIdx.x * kScanBS + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t v = i < G ? seg_rows(in[i]) : 0, x = v;  // segment footprint: kept rows + padding
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t s = lane < kScanBS / 32 ? ws[lane] : 0, t = s;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kScanBS / 32) ws[lane] = t - s;
    if (lane == kScanBS / 32 - 1) sums[blockIdx.x] = t;
  }
  __syncthreads();
  if (i < G) out[i] = x - v + ws[w];
}

__global__ void __launch_bounds__(kScanBS) scan_top_kernel(int64_t* __restrict__ sums, int64_t nb,
                                                           int64_t* __restrict__ total) {
  __shared__ int64_t ws[kScanBS / 32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = 0; base < nb; base += kScanBS) {
    const int64_t i = base + threadIdx.x;
    int64_t v = i < nb ? sums[i] : 0, x = v;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
      int64_t s = lane < kScanBS / 32 ? ws[lane] : 0, t = s;
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      if (lane < kScanBS / 32) ws[lane] = t - s;
    }
    __syncthreads();
    const int64_t c = carry;
    if (i < nb) sums[i] = c + x - v + ws[w];
    __syncthreads();
    if (threadIdx.x == kScanBS - 1) carry = c + x + ws[w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kScanBS) scan_add_kernel(int64_t* __restrict__ out, int64_t G,
                                                           const int64_t* __restrict__ sums) {
  const int64_t i = (int64_t)blockIdx.x * kScanBS + threadIdx.x;
  if (i < G) out[i] += sums[blockIdx.x];
}

}  // namespace

cudaError_t launch_shape_prep(const float* pts_in, int S, int K, int M, float4* pts, uint16_t* perm, float4* lo,
                              float4* hi, uint16_t* cell_tmp, int* bad, cudaStream_t st) {
  shape_bounds_kernel<<<S, 256, 0, st>>>(pts_in, K, M, lo, hi, cell_tmp, bad);
  const size_t sm = sizeof(int) * (size_t)M * M * M;
  shape_sort_kernel<<<S, 256, sm, st>>>(pts_in, K, M, cell_tmp, pts, perm);
  return cudaGetLastError();
}

cudaError_t launch_segment_xf(const ShapeTable& T, const Batch& b, cudaStream_t st) {
  if (b.G == 0) return cudaSuccess;
  segment_xf_kernel<<<(unsigned)((b.G + 127) / 128), 128, 0, st>>>(T, b);
  return cudaGetLastError();
}

cudaError_t launch_crop_count(const ShapeTable& T, const Batch& b, int words, cudaStream_t st) {
  if (b.G == 0) return cudaSuccess;
  // 128-thread blocks: small enough to be co-resident with a persistent encoder CTA (overlapped crop)
  const int64_t blocks = (b.G * 32 + 127) / 128;
  if (b.want_occ)
    crop_count_kernel<true><<<(unsigned)blocks, 128, 0, st>>>(T, b, words);
  else
    crop_count_kernel<false><<<(unsigned)blocks, 128, 0, st>>>(T, b, words);
  return cudaGetLastError();
}

size_t scan_tmp_elems(int64_t G) { return (size_t)((G + kScanBS - 1) / kScanBS) + 1; }

cudaError_t launch_scan(const int32_t* counts, int64_t G, int64_t* offsets, int64_t* block_tmp, cudaStream_t st) {
  const int64_t nb = (G + kScanBS - 1) / kScanBS;
  if (nb == 0) return cudaMemsetAsync(offsets, 0, sizeof(int64_t), st);
  scan_blocks_kernel<<<(unsigned)nb, kScanBS, 0, st>>>(counts, G, offsets, block_tmp);
  scan_top_kernel<<<1, kScanBS, 0, st>>>(block_tmp, nb, offsets + G);
  scan_add_kernel<<<(unsigned)nb, kScanBS, 0, st>>>(offsets, G, block_tmp);
  return cudaGetLastError();
}

cudaError_t launch_crop_emit(const ShapeTable& T, const Batch& b, cudaStream_t st) {
  if (b.G == 0) return cudaSuccess;
  const int64_t blocks = (b.G * 32 + 127) / 128;
  crop_emit_kernel<<<(unsigned)blocks, 128, 0, st>>>(T, b);
  return cudaGetLastError();
}

size_t crop_compact_smem(int K) { return (size_t)kCropWarps * ((K + 31) & ~31) * sizeof(uint32_t); }

size_t crop_compact_lb_words(int64_t G) { return (size_t)((G + kCropWarps - 1) / kCropWarps) + 1; }

cudaError_t launch_crop_compact(const ShapeTable& T, const Batch& b, int words, unsigned long long* lb,
                                cudaStream_t st) {
  if (b.G == 0) return cudaMemsetAsync(b.offsets, 0, sizeof(int64_t), st);
  if (T.K > kFusedMaxK) return cudaErrorInvalidValue;
  const int64_t blocks = (b.G + kCropWarps - 1) / kCropWarps;
  cudaError_t e = cudaMemsetAsync(lb, 0, sizeof(unsigned long long) * (size_t)(blocks + 1), st);
  if (e != cudaSuccess) return e;
  const size_t sm = crop_compact_smem(T.K);
  e = b.want_occ ? smem_optin(crop_compact_kernel<true>, sm) : smem_optin(crop_compact_kernel<false>, sm);
  if (e != cudaSuccess) return e;
  if (b.want_occ)
    crop_compact_kernel<true><<<(unsigned)blocks, 32 * kCropWarps, sm, st>>>(T, b, words, lb, blocks);
  else
    crop_compact_kernel<false><<<(unsigned)blocks, 32 * kCropWarps, sm, st>>>(T, b, words, lb, blocks);
  return cudaGetLastError();
}

}  // namespace locc
