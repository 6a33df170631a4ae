// e3_walk.cuh — the layer-3 epilogue walk of the tensor-core encoder (kernels_encoder_tc.cu): per
// output feature, the rows of a tile in order -> cell-wise max of h3 = ReLU(D3), the
// layer-3 accumulator D3 = b3 + W3 h2 (b3 enters through a bias MMA, like b2), sum over the occupied
// cells in ascending cell order, mean at the segment end.  Shared with
// tools/e3_microbench.cu, which times these routines in isolation.
//
// Summation order (reading Q24).  The fast walk (e3_part2, opt-in: locc_set_deterministic(ctx,
// 0)) splits each 128-row part between two walkers (rows 0-63 carried, rows 64-127 started fresh and
// merged), so the fp32 order in which a segment's cell values are summed depends on where the segment
// falls relative to row 64 of its part: batch composition can move the pooled mean by a few ulps.  The
// deterministic walk (the default; e3_part2_det) uses an order fixed by the segment itself: its rows are
// padded to a multiple of 16 (kSegAlign) and start on a 16-row boundary, so they fall into 16-row
// blocks fixed relative to the segment, and the pooled sum is the fold of per-block sums,
//     S = ((P_0 + P_1) + P_2) + ...,   P_b = ((g_1 + g_2) + g_3) + ...,
// g_1, g_2, ... the values of the cells that END in block b, in row (= ascending cell) order; a
// block in which no cell ends adds +0.  Then every output is bitwise independent of batch
// composition, pair order, sub-batching and GPU count.
#pragma once
#include <stdint.h>

#include "internal.h"
#include "tc_ptx.cuh"

namespace locc {
namespace e3 {

using namespace tc;

// Walk state of one output feature: m = running max of the open cell (from 0: ReLU(max D3) =
// max ReLU(D3)), s = fold of the block sums of the open segment, c = its closed cells.
struct Walk {
  float m, s;
  int c;
};

// A segment's pooled features leave the walk as the cell SUM with the cell count (written once, by
// feature 0); the predictor divides (IEEE, off the walk: a division here sits on the encoder's
// critical loop).  Inlined: an out-of-line call made the compiler spill the walk's live registers
// around it (deterministic walk 3.93 -> 4.29 M checks/s at C3 inlined, default walk +1 %).
__device__ __forceinline__ void store_sum(float* pooled, int32_t* cells_c, uint32_t seg, uint32_t f, float s, int c) {
  pooled[(int64_t)seg * 256 + f] = s;
  if (f == 0) cells_c[seg] = c;
}

constexpr uint32_t kEven = 0x55555555u, kOdd = 0xAAAAAAAAu;

__device__ __forceinline__ uint32_t sel4(const uint4& v, int c) {
  return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}

// ---------------------------------------------------------------------------------------------
// The walk (default).  Two walkers with interleaved masks: for step C (0..3) of a 128-row part, the
// carried walker X takes rows 16C..16C+15 and the tail walker Y rows 64+16C..; their cell-end bits
// come in one word with bit 2j = X row j and bit 2j+1 = Y row j (built directly by the ballot in the
// flags phase), so both walkers' per-row predicates are extracted 7 at a time.  Segments are padded
// to 16 rows (kSegAlign), so a segment end is the last real row of its step: the step is walked like
// any other and the segment closed after it.  Summation order: X's cells sequentially; Y's tail sum
// s1 (from 0) joins X's at the merge as (S + v) + s1 — so the fp32 order of a segment's cell sum
// depends on where the segment falls relative to the part's row 64 (reading Q24: a few ulps).
// The deterministic walk below (locc_set_deterministic) removes that dependence.
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


// ---------------------------------------------------------------------------------------------
// Two walkers with interleaved masks (the encoder's layer-3 epilogue).  For step C (0..3) of a
// 128-row part, the carried walker X takes rows 16C..16C+15 and the tail walker Y rows 64+16C..;
// their cell-end bits come in one word with bit 2j = X row j and bit 2j+1 = Y row j (built directly
// by the ballot in the flags phase), so both walkers' per-row predicates are extracted 7 at a time.
// Segments are padded to 16 rows (kSegAlign), so a segment end is the last real row of its step:
// the step is walked like any other and the segment closed after it.
// Tail semantics: Y's (s, c) exclude its head cell (kept as hm), see merge2().


// One step.  kFirst: Y's first cell end is in this step at bit `firstbit` (its head cell ends there:
// not added, its max kept as hm).
template <bool kFirst>
__device__ __forceinline__ void step2(const uint32_t (&vx)[16], const uint32_t (&vy)[16], uint32_t ce2,
                                      uint32_t firstbit, Walk& x, Tail& t) {
  constexpr float nb3 = 0.f;
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
                                          float* pooled, int32_t* cellc, uint32_t f) {
  constexpr float nb3 = 0.f;
  if (se2 & kEven) {
    const int jx = (__ffs(se2 & kEven) - 1) >> 1;
    store_sum(pooled, cellc, flx[jx] >> kRowSegShift, f, x.s, x.c);
    x = Walk{nb3, 0.f, 0};
  }
  if (se2 & kOdd) {
    Walk& y = t.w;
    const int jy = (__ffs(se2 & kOdd) - 2) >> 1;
    const uint32_t seg = fly[jy] >> kRowSegShift;
    if (t.se) {
      store_sum(pooled, cellc, seg, f, y.s, y.c);
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
__device__ __forceinline__ void merge2(Walk& x, const Tail& t, float* pooled, int32_t* cellc, uint32_t f) {
  if (!t.ce) {
    x.m = fmaxf(x.m, t.w.m);
    return;
  }
  const float hv = fmaxf(x.m, t.hm);  // the cell open across the boundary
  if (t.se) {
    store_sum(pooled, cellc, t.seg1, f, x.s + hv + t.s1, x.c + 1 + t.c1);
    x = t.w;
  } else {
    x.s = x.s + hv + t.w.s;
    x.c = x.c + 1 + t.w.c;
    x.m = t.w.m;
  }
}


// A 128-row part: four straight-line steps with a register double buffer of TMEM columns.
// mk[0..3] = interleaved cell ends of steps 0..3, mk[4..7] = interleaved segment ends.
__device__ __forceinline__ void e3_part2(uint32_t tbase, const uint32_t* mk, const uint32_t* fl, Walk& w,
                                         float* pooled, int32_t* cellc, uint32_t f) {
  constexpr float nb3 = 0.f;
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
        step2<true>(vx, vy, sel4(ce, c), yc & (0u - yc), w, t);
      else
        step2<false>(vx, vy, sel4(ce, c), 0u, w, t);
      if (sel4(se, c)) seg_close(sel4(se, c), fl + 16 * c, fl + 64 + 16 * c, w, t, pooled, cellc, f);
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
        step2<true>(xa, ya, cec, yc & (0u - yc), w, t);
      else
        step2<false>(xa, ya, cec, 0u, w, t);
      if (sec) seg_close(sec, fl + 16 * c, fl + 64 + 16 * c, w, t, pooled, cellc, f);
    }
  }
  merge2(w, t, pooled, cellc, f);
}

// ---------------------------------------------------------------------------------------------
// The deterministic walk (locc_set_deterministic): the same two walkers, the fixed blocked order of
// the header comment.  Two walkers with interleaved masks (the encoder's layer-3 epilogue).  For block C (0..3) of a
// 128-row part, walker X takes rows 16C..16C+15 and walker Y rows 64+16C..; their cell-end bits come
// in one word with bit 2j = X row j and bit 2j+1 = Y row j (built directly by the ballot in the flags
// phase), so both walkers' per-row predicates are extracted 7 at a time.  A segment end is the last
// real row of its block (the rest is padding): the block is walked like any other and the segment
// closed after it.
//
// X continues the carried segment.  Y starts at row 64 without waiting for X: until its first
// segment end ("head mode", blocks 0..ys) its cells belong to the segment X has open.  The first
// cell that ends in Y's rows (in block b0) is the one open across row 64: its value is
// v = max(X's open max, Y's), known only to the merge, and it is the first term of P_b0.  So in block
// b0 Y keeps its last two cell values (prev, last) instead of summing: with one or two cell ends in
// the block that is all P_b0 = v or v + last needs; with more (rare) the merge re-walks block b0 from
// TMEM with the true running max.  Y keeps the block sums of its later head blocks apart (hp1..hp3),
// and the merge folds P_b0 and them onto X's sum in block order.  After its first segment end Y walks
// whole segments and sums them itself.


// One block of both walkers: X folds its cell values into px; Y folds them into py, or, with kYHead,
// shifts them through (prev, last).
template <bool kYHead>
__device__ __forceinline__ void step2(const uint32_t (&vx)[16], const uint32_t (&vy)[16], uint32_t ce2, Walk& x,
                                      Walk& y, float& px, float& py, float& prev, float& last) {
  px = py = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    x.m = fmaxf(x.m, __uint_as_float(vx[j]));
    if ((ce2 >> (2 * j)) & 1u) px += x.m;
    if ((ce2 >> (2 * j)) & 1u) x.m = 0.f;
    y.m = fmaxf(y.m, __uint_as_float(vy[j]));
    if ((ce2 >> (2 * j + 1)) & 1u) {
      if (kYHead) {
        prev = last;
        last = y.m;
      } else {
        py += y.m;
      }
    }
    if ((ce2 >> (2 * j + 1)) & 1u) y.m = 0.f;
  }
  x.c += __popc(ce2 & kEven);
  y.c += __popc(ce2 & kOdd);
}


// Y's head bookkeeping of one walk (one part).
struct Head {
  float prev = 0.f, last = 0.f, hm0 = 0.f;  // block b0's last two cell values; Y's max entering b0
  float hp1 = 0.f, hp2 = 0.f, hp3 = 0.f;    // block sums of Y's head blocks 1..3 after b0
  int hc = 0;                               // Y's head cells
};

// One block of the part (walkers X and Y) with Y's head bookkeeping.
template <bool kYHead>
__device__ __forceinline__ void block(int c, const uint32_t (&vx)[16], const uint32_t (&vy)[16], uint32_t cec,
                                      uint32_t sec, int ys, int b0, Walk& w, Walk& y, Head& h, const uint32_t* fl,
                                      float* pooled, int32_t* cellc, uint32_t f) {
  float px, py;
  if (kYHead) h.hm0 = y.m;
  step2<kYHead>(vx, vy, cec, w, y, px, py, h.prev, h.last);
  w.s += px;  // a block without cell ends adds +0 (exact)
  if (c > ys)
    y.s += py;
  else if (!kYHead && c > b0)  // (named scalars: c is a runtime value on the slow path)
    (c == 1 ? h.hp1 : c == 2 ? h.hp2 : h.hp3) = py;
  if (sec) {
    if (sec & kEven) {  // X closes its segment (the rest of its block is padding)
      const int jx = (__ffs(sec & kEven) - 1) >> 1;
      store_sum(pooled, cellc, fl[16 * c + jx] >> kRowSegShift, f, w.s, w.c);
      w = Walk{0.f, 0.f, 0};
    }
    if (sec & kOdd) {
      if (c > ys) {  // a whole segment of Y's own
        const int jy = (__ffs(sec & kOdd) - 2) >> 1;
        store_sum(pooled, cellc, fl[64 + 16 * c + jy] >> kRowSegShift, f, y.s, y.c);
      } else {
        h.hc = y.c;  // Y's head cells (its head segment is closed in the merge)
      }
      y = Walk{0.f, 0.f, 0};
    }
  }
}

// A 128-row part: four straight-line blocks with a register double buffer of TMEM columns, then the
// merge.  mk[0..3] = interleaved cell ends of blocks 0..3, mk[4..7] = interleaved segment ends.  `w`
// is X's carried state in and the part's final state out.
__device__ __forceinline__ void e3_part2_det(uint32_t tbase, const uint32_t* mk, const uint32_t* fl, Walk& w,
                                         float* pooled, int32_t* cellc, uint32_t f) {
  const uint4 ce = *reinterpret_cast<const uint4*>(mk);
  const uint4 se = *reinterpret_cast<const uint4*>(mk + 4);
  // Y's first segment end is in block ys (4 = none in this part); its first cell end in block b0
  const int ys = (se.x & kOdd) ? 0 : (se.y & kOdd) ? 1 : (se.z & kOdd) ? 2 : (se.w & kOdd) ? 3 : 4;
  const int b0 = (ce.x & kOdd) ? 0 : (ce.y & kOdd) ? 1 : (ce.z & kOdd) ? 2 : (ce.w & kOdd) ? 3 : 4;
  const uint32_t yb0 = b0 < 4 ? sel4(ce, b0) & kOdd : 0u;  // Y's cell ends in block b0
  const bool rewalk = __popc(yb0) > 2;                      // rare: the merge re-walks block b0
  Walk y{0.f, 0.f, 0};
  Head h;
  uint32_t xa[16], ya[16], xb[16], yb[16];
  tmem_ld16(tbase, xa);
  tmem_ld16(tbase + 64, ya);
  if (b0 == 0) {  // Y's first cell end in block 0 (the common case): the head bookkeeping in block 0 only
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
      } else if (rewalk) {
        tmem_ld16(tbase + 64, nx);  // block 0's Y columns again, for the merge's re-walk (xa is free)
      }
      if (c == 0)
        block<true>(c, vx, vy, sel4(ce, c), sel4(se, c), ys, 0, w, y, h, fl, pooled, cellc, f);
      else
        block<false>(c, vx, vy, sel4(ce, c), sel4(se, c), ys, 0, w, y, h, fl, pooled, cellc, f);
    }
  } else {
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
      } else if (rewalk) {
        tmem_ld16(tbase + 64 + 16 * b0, nx);  // block b0's Y columns again, for the merge's re-walk (xa is free)
      }
      if (c == b0)
        block<true>(c, vx, vy, sel4(ce, c), sel4(se, c), ys, b0, w, y, h, fl, pooled, cellc, f);
      else
        block<false>(c, vx, vy, sel4(ce, c), sel4(se, c), ys, b0, w, y, h, fl, pooled, cellc, f);
    }
  }
  if (ys == 4) h.hc = y.c;
  // merge: X's sum continues with Y's head blocks b0..ys in block order
  if (b0 < 4) {
    float pb0;
    if (!rewalk) {
      const bool one = (yb0 & (yb0 - 1)) == 0;
      const float v = fmaxf(w.m, one ? h.last : h.prev);  // the cell open across row 64
      pb0 = one ? v : v + h.last;
    } else {  // re-walk block b0 (in xa) from the head cell's true running max
      tmem_ld_wait();
      float m = fmaxf(w.m, h.hm0);
      pb0 = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        m = fmaxf(m, __uint_as_float(xa[j]));
        if ((yb0 >> (2 * j + 1)) & 1u) pb0 += m;
        if ((yb0 >> (2 * j + 1)) & 1u) m = 0.f;
      }
    }
    float s = w.s + pb0;
    if (b0 < 1 && 1 <= ys) s += h.hp1;
    if (b0 < 2 && 2 <= ys) s += h.hp2;
    if (b0 < 3 && 3 <= ys) s += h.hp3;
    const int cnt = w.c + h.hc;
    if (ys < 4) {  // Y's first segment end closed X's segment
      const int jy = (__ffs(sel4(se, ys) & kOdd) - 2) >> 1;
      store_sum(pooled, cellc, fl[64 + 16 * ys + jy] >> kRowSegShift, f, s, cnt);
      w = y;
    } else {
      w.s = s;
      w.c = cnt;
      w.m = y.m;  // the cell open after Y's last cell end
    }
  } else {
    w.m = fmaxf(w.m, y.m);  // no cell ends in Y's rows: one cell continues through the part
  }
}

// Flags phase: the ballot of warp eg over part p gives the interleaved masks of step eg when lane L
// reads row 64 (L & 1) + 16 eg + (L >> 1) of the part; returns that row's index within the tile.
__device__ __forceinline__ int interleaved_row(int p, int eg, int lane) {
  return 128 * p + 64 * (lane & 1) + 16 * eg + (lane >> 1);
}

}  // namespace e3
}  // namespace locc
