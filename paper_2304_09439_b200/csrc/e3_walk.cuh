// e3_walk.cuh — the layer-3 epilogue walk of the tensor-core encoder (kernels_encoder_tc.cu): per
// output feature, the rows of a tile in order -> cell-wise max, g = ReLU(max + b3),
// sum over occupied cells, mean at the segment end.  Shared with
// tools/e3_microbench.cu, which times these routines in isolation.
#pragma once
#include <stdint.h>

#include "internal.h"
#include "tc_ptx.cuh"

namespace locc {
namespace e3 {

using namespace tc;

// Layer-3 walk state of one output feature.  m runs from -b3 so that ReLU(max + b3) = m + b3 at a
// cell end (max(x, -b3) + b3 rounds to exactly the same value as ReLU(x + b3)); s sums m over the
// occupied cells of the open segment and the mean is (s + c b3) / c.
struct Walk {
  float m, s;
  int c;
};
// A walker that starts in the middle of the row sequence (the second half of a layer-3 part) runs
// from an empty state without waiting for its predecessor, exactly like the carried walker: its
// first cell (the "head") is in truth the continuation of the cell its predecessor left open, and
// its first segment end closes the predecessor's segment.  It therefore keeps the head cell out of
// its sums (hm = its max) and defers the mean of its first segment (s1, c1, seg1); merge2() adds
// max(predecessor's open max, hm) as one cell and completes that segment.
struct Tail {
  Walk w;
  float hm, s1;
  int c1;
  uint32_t seg1;
  bool ce, se;  // seen a cell end / a segment end (warp-uniform)
};

// Out of line: called once per segment end, kept out of the walk's instruction stream.
__device__ __noinline__ void store_mean(float* pooled, uint32_t seg, uint32_t f, float s, int c, float b3) {
  pooled[(int64_t)seg * 256 + f] = __fdividef(fmaf((float)c, b3, s), (float)c);
}

// ---------------------------------------------------------------------------------------------
// Two walkers with interleaved masks (the encoder's layer-3 epilogue).  For step C (0..3) of a
// 128-row part, the carried walker X takes rows 16C..16C+15 and the tail walker Y rows 64+16C..;
// their cell-end bits come in one word with bit 2j = X row j and bit 2j+1 = Y row j (built directly
// by the ballot in the flags phase), so both walkers' per-row predicates are extracted 7 at a time.
// Segments are padded to 16 rows (kSegAlign), so a segment end is the last real row of its step:
// the step is walked like any other and the segment closed after it.
// Tail semantics: Y's (s, c) exclude its head cell (kept as hm), see merge2().

constexpr uint32_t kEven = 0x55555555u, kOdd = 0xAAAAAAAAu;

// One step.  kFirst: Y's first cell end is in this step at bit `firstbit` (its head cell ends there:
// not added, its max kept as hm).
template <bool kFirst>
__device__ __forceinline__ void step2(const uint32_t (&vx)[16], const uint32_t (&vy)[16], uint32_t ce2,
                                      uint32_t firstbit, Walk& x, Tail& t, float nb3) {
  Walk& y = t.w;
  const uint32_t add = kFirst ? ce2 & ~firstbit : ce2;
  float hm = nb3;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    x.m = fmaxf(x.m, __uint_as_float(vx[j]));
    if ((add >> (2 * j)) & 1u) x.s += x.m;
    if ((ce2 >> (2 * j)) & 1u) x.m = nb3;
    y.m = fmaxf(y.m, __uint_as_float(vy[j]));
    if (kFirst && ((firstbit >> (2 * j + 1)) & 1u)) hm = y.m;
    if ((add >> (2 * j + 1)) & 1u) y.s += y.m;
    if ((ce2 >> (2 * j + 1)) & 1u) y.m = nb3;
  }
  x.c += __popc(add & kEven);
  y.c += __popc(add & kOdd);
  if (kFirst) {
    t.hm = hm;
    t.ce = true;
  }
}

// After a step with segment ends: close them (X: store the mean; Y: store, or keep aside if it is
// Y's first segment end) and restart the walkers (the rest of the step is padding).
__device__ __forceinline__ void seg_close(uint32_t se2, const uint32_t* flx, const uint32_t* fly, Walk& x, Tail& t,
                                          float nb3, float b3, float* pooled, uint32_t f) {
  if (se2 & kEven) {
    const int jx = (__ffs(se2 & kEven) - 1) >> 1;
    store_mean(pooled, flx[jx] >> kRowSegShift, f, x.s, x.c, b3);
    x = Walk{nb3, 0.f, 0};
  }
  if (se2 & kOdd) {
    Walk& y = t.w;
    const int jy = (__ffs(se2 & kOdd) - 2) >> 1;
    const uint32_t seg = fly[jy] >> kRowSegShift;
    if (t.se) {
      store_mean(pooled, seg, f, y.s, y.c, b3);
    } else {
      t.s1 = y.s;
      t.c1 = y.c;
      t.seg1 = seg;
      t.se = true;
    }
    y = Walk{nb3, 0.f, 0};
  }
}

// x <- x followed by the tail walker's rows (Y's sums exclude its head cell).
__device__ __forceinline__ void merge2(Walk& x, const Tail& t, float b3, float* pooled, uint32_t f) {
  if (!t.ce) {
    x.m = fmaxf(x.m, t.w.m);
    return;
  }
  const float hv = fmaxf(x.m, t.hm);  // the cell open across the boundary
  if (t.se) {
    store_mean(pooled, t.seg1, f, x.s + hv + t.s1, x.c + 1 + t.c1, b3);
    x = t.w;
  } else {
    x.s = x.s + hv + t.w.s;
    x.c = x.c + 1 + t.w.c;
    x.m = t.w.m;
  }
}

__device__ __forceinline__ uint32_t sel4(const uint4& v, int c) {
  return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}

// A 128-row part: four straight-line steps with a register double buffer of TMEM columns.
// mk[0..3] = interleaved cell ends of steps 0..3, mk[4..7] = interleaved segment ends.
__device__ __forceinline__ void e3_part2(uint32_t tbase, const uint32_t* mk, const uint32_t* fl, Walk& w, float nb3,
                                         float b3, float* pooled, uint32_t f) {
  Tail t;
  t.w = Walk{nb3, 0.f, 0};
  t.hm = nb3;
  t.s1 = 0.f;
  t.c1 = 0;
  t.seg1 = 0;
  t.ce = false;
  t.se = false;
  const uint4 ce = *reinterpret_cast<const uint4*>(mk);
  const uint4 se = *reinterpret_cast<const uint4*>(mk + 4);
  uint32_t xa[16], ya[16], xb[16], yb[16];
  tmem_ld16(tbase, xa);
  tmem_ld16(tbase + 64, ya);
  if (ce.x & kOdd) {  // Y's head ends in step 0 (~97%): straight-line steps
    const uint32_t yc = ce.x & kOdd;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t(&vx)[16] = (c & 1) ? xb : xa;
      uint32_t(&vy)[16] = (c & 1) ? yb : ya;
      uint32_t(&nx)[16] = (c & 1) ? xa : xb;
      uint32_t(&ny)[16] = (c & 1) ? ya : yb;
      tmem_ld_wait();
      if (c < 3) {
        tmem_ld16(tbase + 16 * (c + 1), nx);
        tmem_ld16(tbase + 64 + 16 * (c + 1), ny);
      }
      if (c == 0)
        step2<true>(vx, vy, sel4(ce, c), yc & (0u - yc), w, t, nb3);
      else
        step2<false>(vx, vy, sel4(ce, c), 0u, w, t, nb3);
      if (sel4(se, c)) seg_close(sel4(se, c), fl + 16 * c, fl + 64 + 16 * c, w, t, nb3, b3, pooled, f);
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      if (c > 0) {
        tmem_ld16(tbase + 16 * c, xa);
        tmem_ld16(tbase + 64 + 16 * c, ya);
      }
      tmem_ld_wait();
      const uint32_t cec = sel4(ce, c), sec = sel4(se, c);
      const uint32_t yc = cec & kOdd;
      if (!t.ce && yc != 0)
        step2<true>(xa, ya, cec, yc & (0u - yc), w, t, nb3);
      else
        step2<false>(xa, ya, cec, 0u, w, t, nb3);
      if (sec) seg_close(sec, fl + 16 * c, fl + 64 + 16 * c, w, t, nb3, b3, pooled, f);
    }
  }
  merge2(w, t, b3, pooled, f);
}

// Flags phase: the ballot of warp eg over part p gives the interleaved masks of step eg when lane L
// reads row 64 (L & 1) + 16 eg + (L >> 1) of the part; returns that row's index within the tile.
__device__ __forceinline__ int interleaved_row(int p, int eg, int lane) {
  return 128 * p + 64 * (lane & 1) + 16 * eg + (lane >> 1);
}

}  // namespace e3
}  // namespace locc
