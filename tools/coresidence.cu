// coresidence.cu — can small blocks run beside a persistent 1-CTA-per-SM kernel shaped like the
// tensor-core encoder (544 threads, 96 registers, ~220 KB dynamic shared memory, clusters of 2)?
// A "hog" kernel spins for ~20 ms; a small kernel (128 threads) launched on a low-priority stream
// right after records how many of its blocks finished before the hog ended.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/coresidence tools/coresidence.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <bool kCluster, int kT = 544>
__global__ void __launch_bounds__(kT, 1) hog(unsigned long long ns, unsigned long long* end) {
  extern __shared__ char sm[];
  const unsigned long long t0 = gtime();
  float r[84];
#pragma unroll
  for (int i = 0; i < 84; ++i) r[i] = threadIdx.x * (i + 1);
  while (gtime() - t0 < ns) {
#pragma unroll
    for (int i = 0; i < 84; ++i) r[i] = r[i] * 0.999f + r[(i + 1) % 84];
    __nanosleep(200);
  }
  float x = 0.f;
#pragma unroll
  for (int i = 0; i < 84; ++i) x += r[i];
  sm[threadIdx.x] = (char)x;
  if (threadIdx.x == 0) atomicMax(end, gtime());
}

template <int kThreadsPerBlock, int kMinBlocks>
__global__ void __launch_bounds__(kThreadsPerBlock, kMinBlocks) small(unsigned long long* done_before,
                                                                     const unsigned long long* hog_end,
                                                                     unsigned long long* first_start) {
  const unsigned long long t = gtime();
  if (threadIdx.x == 0) atomicMin(first_start, t);
  constexpr int kR = 65536 / (kThreadsPerBlock * kMinBlocks) >= 48 ? 38 : 22;
  float r[kR];
#pragma unroll
  for (int i = 0; i < kR; ++i) r[i] = threadIdx.x * (i + 1);
  for (int k = 0; k < 50; ++k) {
#pragma unroll
    for (int i = 0; i < kR; ++i) r[i] = r[i] * 0.999f + r[(i + 3) % kR];
  }
  float x = 0.f;
#pragma unroll
  for (int i = 0; i < kR; ++i) x += r[i];
  if (threadIdx.x == 0 && x != 0.f) atomicAdd(done_before, 1ull);
}

template <int T, int MB, int HT = 544>
void run(const char* name, cudaStream_t s0, cudaStream_t s1, unsigned long long* d, int nsm) {
  cudaFuncSetAttribute(hog<true, HT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220160);
  unsigned long long init[3] = {0, 0, ~0ull};
  cudaMemcpy(d, init, 24, cudaMemcpyHostToDevice);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nsm);
  cfg.blockDim = dim3(HT);
  cfg.dynamicSmemBytes = 220160;
  cfg.stream = s0;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, hog<true, HT>, 20000000ull, d);
  small<T, MB><<<nsm * 20 * 128 / T, T, 0, s1>>>(d + 1, d, d + 2);
  cudaDeviceSynchronize();
  unsigned long long r[3];
  cudaMemcpy(r, d, 24, cudaMemcpyDeviceToHost);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, small<T, MB>);
  printf("hog %d threads; %s (%d threads/block, %d regs): first block %+.2f ms relative to the hog's end (%s)\n", HT, name, T, fa.numRegs,
         ((double)r[2] - (double)r[0]) / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int lo, hi;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStream_t s0, s1;
  cudaStreamCreateWithPriority(&s0, cudaStreamNonBlocking, hi);
  cudaStreamCreateWithPriority(&s1, cudaStreamNonBlocking, lo);
  unsigned long long* d;
  cudaMalloc(&d, 64);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  run<128, 10>("128-thread blocks <= 48 regs", s0, s1, d, nsm);
  run<128, 16>("128-thread blocks <= 32 regs", s0, s1, d, nsm);
  run<64, 20>("64-thread blocks <= 48 regs", s0, s1, d, nsm);
  run<32, 40>("32-thread blocks <= 48 regs", s0, s1, d, nsm);
  run<128, 10, 512>("128-thread blocks <= 48 regs", s0, s1, d, nsm);
  run<128, 16, 512>("128-thread blocks <= 32 regs", s0, s1, d, nsm);
  run<128, 10, 416>("128-thread blocks <= 48 regs", s0, s1, d, nsm);
  return 0;
}
