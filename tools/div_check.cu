// div_check.cu — exhaustive check that the predictor's division of a pooled cell sum by the cell
// count C (1..216) — q = x * rc, rc = RN(1 / C), corrected once with the exact FMA residual — equals the
// IEEE quotient __fdiv_rn(x, C) for every fp32 x in [1, 2) (all 2^23 mantissas; the relation is
// invariant under scaling x by powers of two away from overflow / underflow) and for x = 0.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/div_check tools/div_check.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float div_count(float x, float c, float rc) {
  const float q0 = x * rc;
  const float r = fmaf(-q0, c, x);
  return fmaf(r, rc, q0);
}

__global__ void check(unsigned long long* bad, int* first) {
  const unsigned m = blockIdx.x * blockDim.x + threadIdx.x;  // mantissa 0 .. 2^23 - 1
  if (m >= (1u << 23)) return;
  const float x = __uint_as_float(0x3F800000u | m);
  for (int c = 1; c <= 216; ++c) {
    const float fc = (float)c, rc = __frcp_rn(fc);
    const float a = div_count(x, fc, rc), b = __fdiv_rn(x, fc);
    if (__float_as_uint(a) != __float_as_uint(b)) {
      atomicAdd(bad, 1ull);
      atomicCAS(first, 0, (int)(m * 256 + c));
    }
    // also half the range below 1 (exponent -1) and the sums of small dyadic values
    const float x2 = x * 0.5f;
    if (__float_as_uint(div_count(x2, fc, rc)) != __float_as_uint(__fdiv_rn(x2, fc))) atomicAdd(bad, 1ull);
  }
}

int main() {
  unsigned long long* bad;
  int* first;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&first, 4);
  *bad = 0;
  *first = 0;
  check<<<(1u << 23) / 256, 256>>>(bad, first);
  cudaDeviceSynchronize();
  printf("div_count vs __fdiv_rn: %llu mismatches over 2 x 2^23 mantissas x C = 1..216 (first m*256+c = %d)\n", *bad,
         *first);
  return *bad != 0;
}
