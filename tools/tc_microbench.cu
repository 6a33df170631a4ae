// tc_microbench.cu — throughput of the tcgen05 MMA shapes the encoder uses, in isolation.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tcmb tools/tc_microbench.cu
// Each cluster of 2 CTAs issues `reps` x 16 MMAs (one 256-deep K loop) back to back from the
// leader, commits, waits; cycles per MMA are reported next to the ideal of the pacing law.
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2304_09439_b200/csrc/tc_ptx.cuh"

using namespace locc::tc;

struct alignas(1024) Sm {
  uint8_t a[65536];
  uint8_t b[65536];
  uint64_t bar[2];
  uint32_t tmem;
};

template <int MODE>  // 0: SS M256 N256 (L2); 1: TS M256 N128 (L3); 2: SS M256 N128; 3: TS M256 N256
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mb_kernel(int reps, long long* out) {
  extern __shared__ uint8_t raw[];
  Sm& S = *reinterpret_cast<Sm*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const uint32_t rank = cluster_ctarank();
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
    reinterpret_cast<uint32_t*>(S.a)[i] = 0x3f803f80u;
    reinterpret_cast<uint32_t*>(S.b)[i] = 0x3f803f80u;
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&S.bar[0], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_2cta(&S.tmem, 512);
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = S.tmem;
  long long t0 = 0, t1 = 0;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t sa = smem_u32(S.a), sb = smem_u32(S.b);
    const uint32_t id = MODE == 0 || MODE == 3 ? idesc_bf16_f32(256, 256) : idesc_bf16_f32(256, 128);
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int k = 0; k < 16; ++k) {
        const uint32_t koff = (k >> 2) * 16384 + (k & 3) * 32;
        if (MODE == 0 || MODE == 2)
          mma_ss_2cta(tm + 128, smem_desc_sw128(sa + koff, 1024), smem_desc_sw128(sb + koff, 1024), id, k > 0);
        else
          mma_ts_2cta(tm + 256, tm + 8 * k, smem_desc_sw128(sb + koff, 1024), id, k > 0);
      }
    }
    mma_commit_2cta(&S.bar[0], 3);
    mbar_wait(&S.bar[0], 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  if (rank == 1 && threadIdx.x == 0) mbar_wait(&S.bar[0], 0);
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc_2cta(tm, 512);
}

template <int MODE>
void run(const char* name, int grid, double ideal) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * grid);
  cudaMemset(d, 0, sizeof(long long) * grid);
  const int smem = sizeof(Sm) + 1024;
  cudaFuncSetAttribute(mb_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 200;
  mb_kernel<MODE><<<grid, 128, smem>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < grid; i += 2) mx = h[i] > mx ? h[i] : mx;
  printf("%-28s grid %3d: %s  cycles/MMA %.1f (ideal %.1f)\n", name, grid, cudaGetErrorString(e),
         (double)mx / (reps * 16), ideal);
  cudaFree(d);
}

int main() {
  for (int grid : {2, 148}) {
    run<0>("SS 2cta M256 N256", grid, 128);
    run<2>("SS 2cta M256 N128", grid, 64);
    run<1>("TS 2cta M256 N128", grid, 64);
    run<3>("TS 2cta M256 N256", grid, 128);
  }
  return 0;
}
