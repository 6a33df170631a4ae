// tmem_microbench.cu — tcgen05.ld (TMEM -> registers) bandwidth per SM, alone and while the tensor
// core runs the encoder's MMA shapes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tmmb tools/tmem_microbench.cu
// Each CTA of a 2-CTA cluster runs NW loader warps (warp w reads lane quarter w % 4); each loader
// reads `reps` x 128 columns (4 x tcgen05.ld.32x32b.x32) and folds them into a checksum.  With
// MMA != 0 the leader also issues back-to-back L2 (SS N256) or L3 (TS N128) MMAs into columns the
// loaders do not read, to expose contention between epilogue reads and the MMA datapath.
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

template <int NW, int MMA, int WAITALL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * (NW + 1), 1)
    mb_kernel(int reps, int mma_reps, long long* out, unsigned* sink) {
  extern __shared__ uint8_t raw[];
  Sm& S = *reinterpret_cast<Sm*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const uint32_t rank = cluster_ctarank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
    reinterpret_cast<uint32_t*>(S.a)[i] = 0x3f803f80u;
    reinterpret_cast<uint32_t*>(S.b)[i] = 0x3f803f80u;
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&S.bar[0], 1);
    fence_mbar_init();
  }
  if (warp == NW) tmem_alloc_2cta(&S.tmem, 512);
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = S.tmem;
  if (warp < NW) {
    const uint32_t q = warp & 3;
    const uint32_t base = tm + ((32 * q) << 16) + 128 * ((warp >> 2) & 1);  // columns 0..255
    unsigned acc = 0;
    __syncwarp();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      uint32_t v[4][32];
      if (WAITALL) {
#pragma unroll
        for (int c = 0; c < 2; ++c) tmem_ld32(base + 32 * c, v[c]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int j = 0; j < 32; ++j) acc ^= v[c][j];
#pragma unroll
        for (int c = 2; c < 4; ++c) tmem_ld32(base + 32 * c, v[c]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 2; c < 4; ++c)
#pragma unroll
          for (int j = 0; j < 32; ++j) acc ^= v[c][j];
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          tmem_ld32(base + 32 * c, v[0]);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) acc ^= v[0][j];
        }
      }
    }
    const long long t1 = clock64();
    if (lane == 0) out[(blockIdx.x * (NW + 1) + warp)] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc;
  } else if (MMA && rank == 0 && lane == 0) {
    const uint32_t sa = smem_u32(S.a), sb = smem_u32(S.b);
    const long long t0 = clock64();
    for (int r = 0; r < mma_reps; ++r) {
      for (int k = 0; k < 16; ++k) {
        const uint32_t koff = (k >> 2) * 16384 + (k & 3) * 32;
        if (MMA == 1)
          mma_ss_2cta(tm + 256, smem_desc_sw128(sa + koff, 1024), smem_desc_sw128(sb + koff, 1024),
                      idesc_bf16_f32(256, 256), k > 0);
        else
          mma_ts_2cta(tm + 384, tm + 256 + 8 * k, smem_desc_sw128(sb + koff, 1024), idesc_bf16_f32(256, 128), k > 0);
      }
    }
    mma_commit_2cta(&S.bar[0], 3);
    mbar_wait(&S.bar[0], 0);
    out[(blockIdx.x * (NW + 1) + NW)] = clock64() - t0;
  }
  if (MMA && rank == 1 && threadIdx.x == 32 * NW) mbar_wait(&S.bar[0], 0);
  tc_fence_before();
  cluster_sync();
  if (warp == NW) tmem_dealloc_2cta(tm, 512);
}

template <int NW, int MMA, int WAITALL>
void run(const char* name, int reps, int mma_reps) {
  const int grid = 2;
  long long* d;
  unsigned* sink;
  cudaMalloc(&d, sizeof(long long) * grid * (NW + 1));
  cudaMalloc(&sink, 4);
  cudaMemset(d, 0, sizeof(long long) * grid * (NW + 1));
  const size_t smem = sizeof(Sm) + 1024;
  cudaFuncSetAttribute(mb_kernel<NW, MMA, WAITALL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int it = 0; it < 2; ++it) mb_kernel<NW, MMA, WAITALL><<<grid, 32 * (NW + 1), smem>>>(reps, mma_reps, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[64];
  cudaMemcpy(h, d, sizeof(long long) * grid * (NW + 1), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int w = 0; w < NW; ++w) mx = h[w] > mx ? h[w] : mx;
  const double bytes = (double)NW * reps * 32 * 128 * 4;
  printf("%-34s err=%d  load: %8lld cyc  %6.1f B/cyc/SM  %6.1f cyc per warp-x32", name, (int)e, mx, bytes / mx,
         (double)mx / (reps * 4) );
  if (MMA) printf("   mma: %lld cyc for %d MMAs = %.1f cyc/MMA", h[NW], mma_reps * 16, (double)h[NW] / (mma_reps * 16));
  printf("\n");
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  run<1, 0, 0>("1 warp, wait each", 256, 0);
  run<1, 0, 1>("1 warp, 2 in flight", 256, 0);
  run<4, 0, 0>("4 warps, wait each", 256, 0);
  run<4, 0, 1>("4 warps, 2 in flight", 256, 0);
  run<8, 0, 0>("8 warps, wait each", 256, 0);
  run<8, 0, 1>("8 warps, 2 in flight", 256, 0);
  run<12, 0, 1>("12 warps, 2 in flight", 256, 0);
  run<16, 0, 1>("16 warps, 2 in flight", 256, 0);
  run<8, 1, 1>("8 warps + L2 SS N256 MMAs", 256, 64);
  run<8, 2, 1>("8 warps + L3 TS N128 MMAs", 256, 128);
  run<4, 2, 1>("4 warps + L3 TS N128 MMAs", 256, 128);
  run<0 + 1, 1, 1>("1 warp + L2 SS N256 MMAs", 64, 64);
  return 0;
}
