// geom.cuh — S1 relative transforms and the O4 distance test, shared by the crop kernels
// (kernels_geom.cu) and the encode-once cell selection (kernels_cells.cu) of liblocc.so.
// Prescribed arithmetic: explicit round-to-nearest intrinsics only.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"
#include "quat.cuh"

namespace locc {
namespace {

// ---------------------------------------------------------------- S1 relative transforms
// normalise in fp64; q_BA = conj(q_B) (x) q_A with the grouping that
// makes conj(q) (x) q cancel exactly; R(q) in fp64; t_BA = R_B^T (t_A - t_B); each entry
// rounded once to fp32.
struct Xf {
  float R[9];
  float t[3];
};

__device__ __forceinline__ void qmul(const double a[4], const double b[4], double r[4]) {
  r[0] = __dsub_rn(__dmul_rn(a[0], b[0]), __dadd_rn(__dadd_rn(__dmul_rn(a[1], b[1]), __dmul_rn(a[2], b[2])), __dmul_rn(a[3], b[3])));
  r[1] = __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[1]), __dmul_rn(b[0], a[1])), __dsub_rn(__dmul_rn(a[2], b[3]), __dmul_rn(a[3], b[2])));
  r[2] = __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[2]), __dmul_rn(b[0], a[2])), __dsub_rn(__dmul_rn(a[3], b[1]), __dmul_rn(a[1], b[3])));
  r[3] = __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[3]), __dmul_rn(b[0], a[3])), __dsub_rn(__dmul_rn(a[1], b[2]), __dmul_rn(a[2], b[1])));
}

__device__ __forceinline__ void qmat(const double q[4], double R[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(y, y), __dmul_rn(z, z))));
  R[1] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(x, y), __dmul_rn(w, z)));
  R[2] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, z), __dmul_rn(w, y)));
  R[3] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, y), __dmul_rn(w, z)));
  R[4] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, x), __dmul_rn(z, z))));
  R[5] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(y, z), __dmul_rn(w, x)));
  R[6] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(x, z), __dmul_rn(w, y)));
  R[7] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(y, z), __dmul_rn(w, x)));
  R[8] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y))));
}

// Transform taking points of the object posed (qs, ts) into the frame of the object posed (qo, to).
__device__ __forceinline__ void relative_xf(const double qs[4], const float* ts, const double qo[4],
                                            const float* to, Xf& X) {
  const double cj[4] = {qo[0], -qo[1], -qo[2], -qo[3]};
  double qr[4], R[9], Ro[9];
  qmul(cj, qs, qr);
  qmat(qr, R);
  qmat(qo, Ro);
  const double d0 = __dsub_rn((double)ts[0], (double)to[0]);
  const double d1 = __dsub_rn((double)ts[1], (double)to[1]);
  const double d2 = __dsub_rn((double)ts[2], (double)to[2]);
#pragma unroll
  for (int i = 0; i < 9; ++i) X.R[i] = __double2float_rn(R[i]);
#pragma unroll
  for (int i = 0; i < 3; ++i)
    X.t[i] = __double2float_rn(__dadd_rn(__dadd_rn(__dmul_rn(Ro[i], d0), __dmul_rn(Ro[3 + i], d1)), __dmul_rn(Ro[6 + i], d2)));
}

// O4: keep iff squared distance from the transformed point to the counter AABB <= eps^2.
__device__ __forceinline__ bool keep_point(const Xf& X, float x, float y, float z, const float4& lo,
                                           const float4& hi) {
  const float px = __fmaf_rn(X.R[0], x, __fmaf_rn(X.R[1], y, __fmaf_rn(X.R[2], z, X.t[0])));
  const float py = __fmaf_rn(X.R[3], x, __fmaf_rn(X.R[4], y, __fmaf_rn(X.R[5], z, X.t[1])));
  const float pz = __fmaf_rn(X.R[6], x, __fmaf_rn(X.R[7], y, __fmaf_rn(X.R[8], z, X.t[2])));
  const float dx = fmaxf(fmaxf(__fsub_rn(lo.x, px), __fsub_rn(px, hi.x)), 0.f);
  const float dy = fmaxf(fmaxf(__fsub_rn(lo.y, py), __fsub_rn(py, hi.y)), 0.f);
  const float dz = fmaxf(fmaxf(__fsub_rn(lo.z, pz), __fsub_rn(pz, hi.z)), 0.f);
  const float d2 = __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, __fmul_rn(dz, dz)));
  return d2 <= lo.w;
}

// Resolve segment g = 2*pair + side: own shape, counter shape, transform.  False = invalid input.
__device__ __forceinline__ bool segment_setup(const ShapeTable& T, const Batch& b, int64_t g, int& own,
                                              int& other, Xf& X) {
  const int64_t i = g >> 1;
  const int side = (int)(g & 1);
  const int a = b.pairs[2 * i], c = b.pairs[2 * i + 1];
  if (a < 0 || a >= T.S || c < 0 || c >= T.S) return false;
  const float* pA = b.poses + 14 * i;
  const float* pB = pA + 7;
  for (int j = 0; j < 14; ++j)
    if (!isfinite(pA[j])) return false;
  double qA[4], qB[4];
  if (!quat_unit(pA, qA) || !quat_unit(pB, qB)) return false;
  if (side == 0) {
    own = a;
    other = c;
    relative_xf(qA, pA + 4, qB, pB + 4, X);
  } else {
    own = c;
    other = a;
    relative_xf(qB, pB + 4, qA, pA + 4, X);
  }
  return true;
}

// The segment's transform as written by segment_xf_kernel (one thread per segment, so the fp64
// quaternion work is not repeated by every lane of every kernel that needs it).  False = invalid.
__device__ __forceinline__ bool segment_load(const Batch& b, int64_t g, int& own, int& other, Xf& X) {
  const float4* x = b.xf + 4 * g;
  const float4 r0 = x[0], r1 = x[1], r2 = x[2], id = x[3];
  own = __float_as_int(id.x);
  other = __float_as_int(id.y);
  X.R[0] = r0.x, X.R[1] = r0.y, X.R[2] = r0.z, X.t[0] = r0.w;
  X.R[3] = r1.x, X.R[4] = r1.y, X.R[5] = r1.z, X.t[1] = r1.w;
  X.R[6] = r2.x, X.R[7] = r2.y, X.R[8] = r2.z, X.t[2] = r2.w;
  return own >= 0;
}

}  // namespace
}  // namespace locc
