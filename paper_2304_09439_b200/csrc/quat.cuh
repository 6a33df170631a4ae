// quat.cuh — O1 quaternion normalisation (fp64, explicit round-to-nearest), shared by the crop
// and the predictor kernels of liblocc.so.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

namespace locc {

// n^2 = ((w*w + x*x) + y*y) + z*z from the fp32 inputs in fp64; reject n^2 < 1e-12.
__device__ __forceinline__ bool quat_unit(const float* q7, double q[4]) {
  const double w = q7[0], x = q7[1], y = q7[2], z = q7[3];
  const double n2 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(w, w), __dmul_rn(x, x)), __dmul_rn(y, y)), __dmul_rn(z, z));
  if (!(n2 >= 1e-12) || !isfinite(n2)) return false;
  const double s = __dsqrt_rn(n2);
  q[0] = __ddiv_rn(w, s);
  q[1] = __ddiv_rn(x, s);
  q[2] = __ddiv_rn(y, s);
  q[3] = __ddiv_rn(z, s);
  return true;
}


}  // namespace locc
