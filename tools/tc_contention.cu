// tc_contention.cu — does shared-memory traffic from CUDA-core warps slow tcgen05.mma?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tcc tools/tc_contention.cu
// The leader of each 2-CTA cluster issues back-to-back MMAs of one shape (operands in shared
// memory, as in the encoder's layer 2 / layer 3) while NW warps per CTA stream st.shared.v4 or
// ld.shared.v4 over a separate 64 KB buffer.  Prints cycles per MMA and the noise bandwidth.
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2304_09439_b200/csrc/tc_ptx.cuh"

using namespace locc::tc;

struct alignas(1024) Sm {
  uint8_t a[65536];
  uint8_t b[65536];
  uint8_t noise[65536];
  uint64_t bar[2];
  uint32_t tmem;
  volatile int stop;
};

// SHAPE 0: SS N256, 1: SS N128, 2: TS N128.  NOISE 0: none, 1: st.shared.v4, 2: ld.shared.v4
template <int SHAPE, int NOISE, int NW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * (NW + 1), 1) k(int reps, long long* out) {
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
    mbar_init(&S.bar[1], 1);
    S.stop = 0;
    fence_mbar_init();
  }
  if (warp == NW) tmem_alloc_2cta(&S.tmem, 512);
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = S.tmem;
  if (warp < NW) {
    const uint32_t base = smem_u32(S.noise) + warp * 4096 + lane * 16;
    uint32_t acc = 0;
    long long n = 0;
    const long long t0 = clock64();
    while (!S.stop) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t ad = base + (i & 7) * 512;
        if (NOISE == 1) st_shared_v4(ad, acc, i, n, 7);
        if (NOISE == 2) {
          uint32_t x, y, z, w;
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(ad));
          acc ^= x ^ y ^ z ^ w;
        }
      }
      n += 8;
      if (NOISE == 0) break;
    }
    const long long t1 = clock64();
    if (lane == 0 && rank == 0) out[64 + warp] = (long long)((double)n * 512 / (double)(t1 - t0 + 1) * 1000);
    if (acc == 0x1234567u) out[127] = acc;
  } else if (rank == 0 && lane == 0) {
    const uint32_t sa = smem_u32(S.a), sb = smem_u32(S.b);
    const uint32_t id = SHAPE == 0 ? idesc_bf16_f32(256, 256) : idesc_bf16_f32(256, 128);  // SHAPE 1, 3-5: N128
    // warm up, then time
    long long t0 = 0;
    for (int r = 0; r < reps + 4; ++r) {
      if (r == 4) t0 = clock64();
      for (int kk = 0; kk < 16; ++kk) {
        const uint32_t koff = (kk >> 2) * 16384 + (kk & 3) * 32;
        if (SHAPE == 4) {  // SS N128 with a commit (to a spare barrier) after every 4 MMAs
          mma_ss_2cta(tm + 128, smem_desc_sw128(sa + koff, 1024), smem_desc_sw128(sb + koff, 1024), id, kk > 0);
          if ((kk & 3) == 3) mma_commit_2cta(&S.bar[1], 3);
        } else if (SHAPE == 5) {  // SS N128 with a commit after every MMA
          mma_ss_2cta(tm + 128, smem_desc_sw128(sa + koff, 1024), smem_desc_sw128(sb + koff, 1024), id, kk > 0);
          mma_commit_2cta(&S.bar[1], 3);
        } else if (SHAPE == 3)
          mma_ss_2cta(tm + 128, smem_desc_sw128(sa, 0), smem_desc_sw128(sb + koff, 1024), id, kk > 0);
        else if (SHAPE < 2)
          mma_ss_2cta(tm + 128, smem_desc_sw128(sa + koff, 1024), smem_desc_sw128(sb + koff, 1024), id, kk > 0);
        else
          mma_ts_2cta(tm + 256, tm + 8 * kk, smem_desc_sw128(sb + koff, 1024), id, kk > 0);
      }
    }
    mma_commit_2cta(&S.bar[0], 3);
    mbar_wait(&S.bar[0], 0);
    out[0] = clock64() - t0;
  }
  if (rank == 1 && threadIdx.x == 32 * NW) mbar_wait(&S.bar[0], 0);
  // stop the noise warps of both CTAs
  if (threadIdx.x == 32 * NW) {
    S.stop = 1;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == NW) tmem_dealloc_2cta(tm, 512);
}

template <int SHAPE, int NOISE, int NW>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 128);
  cudaMemset(d, 0, sizeof(long long) * 128);
  const int smem = sizeof(Sm) + 1024;
  cudaFuncSetAttribute(k<SHAPE, NOISE, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 200;
  k<SHAPE, NOISE, NW><<<2, 32 * (NW + 1), smem>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[128];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double bw = 0;
  for (int w = 0; w < NW; ++w) bw += h[64 + w] / 1000.0;
  const double ideal = SHAPE == 0 ? 128 : 64;
  printf("%-40s %s  cycles/MMA %6.1f (ideal %.0f)  noise %.1f B/cycle/CTA\n", name, cudaGetErrorString(e),
         (double)h[0] / (reps * 16), ideal, bw);
  cudaFree(d);
}

int main() {
  run<3, 0, 1>("SS N128 A-desc SBO=0 (bias MMA), quiet");
  run<4, 0, 1>("SS N128 + commit every 4 MMAs");
  run<5, 0, 1>("SS N128 + commit every MMA");
  run<0, 0, 1>("SS N256, quiet");
  run<1, 0, 1>("SS N128, quiet");
  run<2, 0, 1>("TS N128, quiet");
  run<0, 1, 4>("SS N256 + 4 warps st.shared");
  run<1, 1, 4>("SS N128 + 4 warps st.shared");
  run<2, 1, 4>("TS N128 + 4 warps st.shared");
  run<0, 1, 8>("SS N256 + 8 warps st.shared");
  run<1, 1, 8>("SS N128 + 8 warps st.shared");
  run<2, 1, 8>("TS N128 + 8 warps st.shared");
  run<0, 2, 8>("SS N256 + 8 warps ld.shared");
  run<1, 2, 8>("SS N128 + 8 warps ld.shared");
  run<2, 2, 8>("TS N128 + 8 warps ld.shared");
  return 0;
}
