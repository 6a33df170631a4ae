// tile_mma_bench.cu — the encoder's per-tile tensor-core instruction stream without any waits:
// L2a, L2b (bias MMA + 16 K steps each, N = 128, SS), L3 two parts (16 K steps each, TS), with the
// encoder's commits, repeated for many tiles.  Cycles per tile vs the 66 x 64 = 4224 ideal.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tile_mma_bench tools/tile_mma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2304_09439_b200/csrc/tc_ptx.cuh"

using namespace locc::tc;

struct alignas(1024) Sm {
  uint8_t w2[5 * 16384];
  uint8_t h1[65536];
  uint8_t h2[65536];
  uint8_t ones[1024];
  uint64_t bar[16];
  uint32_t tmem;
};

template <int MODE>  // 0: full tile stream, 1: no commits, 2: L2 only, 3: L3 only, 4: no bias MMAs
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1) k(int tiles, long long* out) {
  extern __shared__ uint8_t raw[];
  Sm& S = *reinterpret_cast<Sm*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const uint32_t rank = cluster_ctarank();
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (int)(sizeof(Sm) - 1024) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(&S)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&S.bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_2cta(&S.tmem, 512);
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = S.tmem;
  if (rank == 0 && threadIdx.x == 0) {
    const uint64_t dA1 = smem_desc_sw128(smem_u32(S.h1), 1024), dW2 = smem_desc_sw128(smem_u32(S.w2), 1024);
    const uint64_t dH2 = smem_desc_sw128(smem_u32(S.h2), 1024), dOne = smem_desc_sw128(smem_u32(S.ones), 0);
    const uint64_t dB2 = dW2 + 4 * 1024;
    const uint32_t id = idesc_bf16_f32(256, 128);
    long long t0 = 0;
    for (int t = 0; t < tiles + 4; ++t) {
      if (t == 4) t0 = clock64();
      const uint32_t rp = tm + 128 + 128 * (t & 1), rq = tm + 128 + 128 * ((t + 1) & 1), r3 = tm + 384;
      if (MODE != 3) {
        if (MODE != 4) mma_ss_2cta(rp, dOne, dB2, id, 0);
#pragma unroll
        for (int kb = 0; kb < 4; ++kb)
#pragma unroll
          for (int s = 0; s < 4; ++s) mma_ss_2cta(rp, dA1 + kb * 1024 + 2 * s, dW2 + kb * 1024 + 2 * s, id, MODE == 4 ? (kb | s) != 0 : 1);
        if (MODE != 1) mma_commit_2cta(&S.bar[0], 3);
        if (MODE != 4) mma_ss_2cta(rq, dOne, dB2 + 512, id, 0);
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
#pragma unroll
          for (int s = 0; s < 4; ++s)
            mma_ss_2cta(rq, dA1 + kb * 1024 + 2 * s, dW2 + kb * 1024 + 512 + 2 * s, id, MODE == 4 ? (kb | s) != 0 : 1);
          if (MODE != 1) mma_commit_2cta(&S.bar[1 + kb], 3);
        }
        if (MODE != 1) mma_commit_2cta(&S.bar[5], 3);
      }
      if (MODE != 2) {
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
          mma_ts_2cta(rp, tm + 8 * kk, dH2 + (kk >> 2) * 1024 + (kk & 3) * 2, id, kk != 0);
        if (MODE != 1) mma_commit_2cta(&S.bar[6], 3);
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
          mma_ts_2cta(r3, tm + 8 * kk, dH2 + (kk >> 2) * 1024 + (kk & 3) * 2 + 512, id, kk != 0);
        if (MODE != 1) {
          mma_commit_2cta(&S.bar[7], 3);
          mma_commit_2cta(&S.bar[8], 3);
        }
      }
    }
    mma_commit_2cta(&S.bar[9], 3);
    mbar_wait(&S.bar[9], 0);
    out[0] = clock64() - t0;
  }
  if (rank == 1 && threadIdx.x == 0) mbar_wait(&S.bar[9], 0);
  tc_fence_before();
  cluster_sync();
  if (warp == 1) tmem_dealloc_2cta(tm, 512);
}

template <int MODE>
void run(const char* name, double ideal) {
  long long* d;
  cudaMalloc(&d, 8);
  const int smem = sizeof(Sm) + 1024;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = 400;
  k<MODE><<<2, 64, smem>>>(tiles, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-34s %s  %7.0f cycles/tile (ideal %.0f)\n", name, cudaGetErrorString(e), (double)h / tiles, ideal);
  cudaFree(d);
}

int main() {
  run<0>("full tile stream", 66 * 64);
  run<1>("no commits", 66 * 64);
  run<2>("L2 halves only", 34 * 64);
  run<3>("L3 parts only", 32 * 64);
  run<4>("no bias MMAs", 64 * 64);
  return 0;
}
