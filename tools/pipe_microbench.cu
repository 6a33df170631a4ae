// pipe_microbench.cu — issue cost per warp instruction (cycles per SMSP) of the CUDA-core ops the
// encoder's epilogues and layer 1 use: FFMA, FFMA2 (fma.rn.f32x2), FADD2, FMNMX, FSEL, F2FP (packed
// ReLU bf16x2 convert).  8 independent chains per thread, W warps per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/pipemb tools/pipe_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2304_09439_b200/csrc/tc_ptx.cuh"

using namespace locc::tc;

template <int OP>
__global__ void k(int iters, float seed, long long* out, float* sink) {
  float a[8];
  unsigned long long p[8];
  uint32_t u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = seed + i + threadIdx.x;
    p[i] = f2(a[i], a[i] + 1.f);
    u[i] = __float_as_uint(a[i]);
  }
  const unsigned long long c2 = f2(seed, seed * 0.5f);
  const float c = seed * 0.25f;
  bool pr[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) pr[i] = (u[i] >> 3) & 1;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (OP == 0) a[i] = fmaf(a[i], c, 0.5f * c);
        if (OP == 1) p[i] = ffma2(p[i], c2, c2);
        if (OP == 2) p[i] = fadd2(p[i], c2);
        if (OP == 3) a[i] = fmaxf(a[i], c + (float)i);
        if (OP == 4) a[i] = pr[(i + r) & 7] ? c : a[i] * 1.0f;
        if (OP == 5) u[i] = pack_relu_bf16x2(__uint_as_float(u[i]), c);
      }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + f2_lo(p[i]) + __uint_as_float(u[i]);
  if (s == 1234.5f) sink[0] = s;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps) {
  long long* d;
  float* sink;
  cudaMalloc(&d, sizeof(long long));
  cudaMalloc(&sink, 4);
  const int iters = 1000;
  for (int r = 0; r < 2; ++r) k<OP><<<1, 32 * warps>>>(iters, 1.0001f, d, sink);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double per_smsp = (double)warps / 4.0 * iters * 64;
  printf("%-8s warps=%2d  %6.2f cycles per warp-instruction per SMSP\n", name, warps, h / per_smsp);
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("FFMA", w);
    run<1>("FFMA2", w);
    run<2>("FADD2", w);
    run<3>("FMNMX", w);
    run<4>("FSEL", w);
    run<5>("F2FP", w);
  }
  return 0;
}
