// internal.h — device-side data layout shared by the liblocc.so translation units.
// Product code only (never included by oracle/).  See DESIGN.md "Data layout in HBM".
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

namespace locc {

constexpr int kPredW = 128;        // predictor width, "3 layers of 128 neurons"
constexpr int kSegPerChunk = 8;    // encoder work unit: 8 whole (pair, side) segments = 4 pairs
constexpr int kRowFlagCellEnd = 1; // row flag: last kept row of its cell within the segment
constexpr int kRowFlagSegEnd = 2;  // row flag: last kept row of the segment
constexpr int kRowFlagPad = 4;     // row flag: padding row after the segment's last kept row
constexpr int kRowSegShift = 3;    // flags word = (segment << 3) | pad << 2 | seg_end << 1 | cell_end
// Each segment's rows are padded to a multiple of kSegAlign, so a segment starts on a 16-row step
// of the encoder's layer-3 walk and a segment end is followed only by padding within its step.
constexpr int kSegAlign = 16;
__host__ __device__ constexpr int64_t seg_rows(int64_t kept) { return (kept + kSegAlign - 1) / kSegAlign * kSegAlign; }

// Checked build (-DLOCC_CHECKED=1, `tools/checked_run.py`): device-side bounds checks on the hot
// kernels' global-memory indices — this pool's substitute for compute-sanitizer memcheck, which is
// closed here.  A failed check prints the condition and traps (the call returns LOCC_E_CUDA).
#ifndef LOCC_CHECKED
#define LOCC_CHECKED 0
#endif
#if LOCC_CHECKED
#define LOCC_CHECK(cond)                                                               \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("LOCC_CHECK failed: %s (%s:%d, block %d thread %d)\n", #cond, __FILE__, \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                             \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
// ... and with two values of the failing case
#define LOCC_CHECK_V(cond, u, v)                                                                        \
  do {                                                                                                  \
    if (!(cond)) {                                                                                      \
      printf("LOCC_CHECK failed: %s [%s = %lld, %s = %lld] (%s:%d, block %d thread %d)\n", #cond, #u, \
             (long long)(u), #v, (long long)(v), __FILE__, __LINE__, (int)blockIdx.x, (int)threadIdx.x);  \
      __trap();                                                                                         \
    }                                                                                                   \
  } while (0)
#else
#define LOCC_CHECK_V(cond, u, v) \
  do {                           \
  } while (0)
#define LOCC_CHECK(cond) \
  do {                   \
  } while (0)
#endif

// S0 output (one copy per context, resident for the context's lifetime).
struct ShapeTable {
  const float4* pts;    // [S][K] cell-sorted points: (x, y, z, __int_as_float(cell id))
  const uint16_t* perm; // [S][K] sorted position -> caller's point index
  const float4* lo;     // [S] (lo.x, lo.y, lo.z, eps^2)
  const float4* hi;     // [S] (hi.x, hi.y, hi.z, 0)
  int S, K;
};

// Parameters on the device (fp32 unless noted).  "T" = transposed to [in][out] so that a
// thread per output unit reads coalesced rows.
struct DevParams {
  int H, F;
  const float* w1;   // [H][3] + b1 [H] packed as float4 (w0, w1, w2, b) per unit: w1b [H]
  const float4* w1b;
  const float* w2T;  // [H in][H out]
  const float* b2;
  const float* w3T;
  const float* b3;
  const float* wfT;  // [H][F]
  const float* bf;
  const float* o1T;  // [F+7][128]
  const float* ob1;
  const float* o2T;  // [128][128]
  const float* ob2;
  const float* o3T;
  const float* ob3;
  const float* p1T;
  const float* pb1;
  const float* p2T;
  const float* pb2;
  const float* p3T;
  const float* pb3;
  const float* wout; // [128]
  const float* bout; // [1]
  // original [out][in] layouts for the reverse mode (NEXT-2): d/d in = W^T d/d out
  const float* o1p;  // the 7 pose columns of obj.l1, [7][128]
  const float* o2;
  const float* o3;
  const float* p1;
  const float* p2;
  const float* p3;
  const void* head_tc_img;    // tensor-core predictor: 23 pre-split (tf32 hi/lo), SW128 weight chunks
  const void* head_tc_proj;   // the projection W_F as 8 such chunks (rows 0..63)
  const void* head_tc_bwd;    // reverse mode: pair3^T, pair2^T, pair1^T, obj3^T, obj2^T as 20 such chunks
  const float* head_tc_bias;  // [6][128] layer biases, wout [128], bout, b_F [64]
  const void* tc_w2; // bf16 W2/W3 pre-arranged as the encoder_tc shared-memory image
  const void* tc_w3;
  const uint8_t* grid_tc_img;  // tensor-core grid encode (H = 256): W2 then W3, each as 2 output halves
                               // x 8 pre-split SW128 chunks [128 out x 32 in] (kernels_conv_tc.cu format)
};

// NEXT-1 (encode-once) U-Net parameters, rearranged for the implicit-GEMM conv kernel:
// Wt[l] = [27][Cin][128] (tap-major; deconv layers stored as the equivalent conv: taps flipped).
struct UNetParams {
  const float* Wt[8];  // 0..3 = c1..c4, 4..7 = d4, d3, d2, d1
  const float* b[8];
  const uint8_t* img[8];  // tensor-core (bf16 contexts) images: per layer 27 x C_in/32 chunks of
                          // [128 out x 32 in] tf32 hi then lo, SW128 K-major (kernels_conv_tc.cu)
  const float* pW;     // [F][256] projection of [d1 ; g]
  const float* pb;     // [F]
};

// Per-shape cached embedding grids of the encode-once mode.
struct CellsTable {
  const float* E;      // [S][M^3][F] cell embeddings
  const float* ctr;    // [S][3][8] cell-centre coordinates per axis in the shape's frame (i < M)
  int M;
};

// NEXT-3 closed-loop step constants (see include/locc.h locc_sim_config).
struct SimParams {
  double hd;  // substep length (s), for the substep times
  float h;
  float g[3];
  float ks, kd;
  float amp[3];
  float freq;
  float slack;
};

// Device counters of one query (int64 atomics), zeroed per query.
struct DevStats {
  unsigned long long kept_rows;
  unsigned long long nonempty_sides;
  unsigned long long evaluated_pairs;
  unsigned long long bad_input;  // nonzero: an id was out of range or a pose invalid
};

// One sub-batch of pairs as seen by the kernels.
struct Batch {
  const int32_t* pairs;  // [B][2]
  const float* poses;    // [B][2][7]
  int64_t B;             // pairs in this sub-batch
  int64_t G;             // segments = 2B
  int32_t* counts;       // [G] n_s
  int32_t* occ;          // [G] C_s (from the crop; written only when want_occ)
  int want_occ;          // the caller asked for C_s (locc_query_debug)
  int64_t* offsets;      // [G+1] exclusive scan of counts
  uint2* rows;           // [sum pad16(n)] kept rows: (flags, point index k in the own shape's sorted table)
  int64_t rows_cap;      // capacity of `rows` in rows (checked builds)
  const float4* pts;     // the shape table's sorted points [S][K] (the rows' coordinates: pts[own K + k])
  int K;
  int S;                 // shapes in the table (checked builds)
  float* pooled;         // [G][H] mean over occupied cells of the cell-max features, or their SUM when
                         // cells_c is set (the tensor-core encoder; the predictor divides)
  int32_t* cells_c;      // [G] occupied cells C of each non-empty segment when pooled holds sums, else null
  const float* emb_in;   // encode-once mode: [G][F] pooled cell embeddings (the predictor's e); else null
  float4* xf;            // [G][4] per-segment transform into the other object's frame (segment_xf_kernel):
                         // rows (R00 R01 R02 t0), (R10 R11 R12 t1), (R20 R21 R22 t2), (own, other, -, -) as ints;
                         // own = -1 for an invalid segment (id out of range, non-finite pose, |q|^2 < 1e-12)
  uint32_t* masks;       // nullable [B][2][ceil(K/32)] caller-order keep bits (debug)
  uint32_t* kbits;       // [G][ceil(K/32)] keep ballots in sorted order (crop_count -> crop_emit)
  DevStats* stats;
};

// Layer-1 weights and layer-2 bias of the tensor-core encoder, passed by value as kernel
// parameters (constant bank) so every FFMA/FADD reads them as a uniform operand.
struct TcL1 {
  float4 w1b[256];  // (w0, w1, w2, b1) per feature of encoder layer 1
  float b2[256];
};

// Launchers (kernels_*.cu).  All asynchronous on `st`.
cudaError_t launch_shape_prep(const float* pts_in, int S, int K, int M, float4* pts, uint16_t* perm,
                              float4* lo, float4* hi, uint16_t* cell_tmp, int* bad, cudaStream_t st);
cudaError_t launch_segment_xf(const ShapeTable& T, const Batch& b, cudaStream_t st);
cudaError_t launch_crop_count(const ShapeTable& T, const Batch& b, int words, cudaStream_t st);
cudaError_t launch_scan(const int32_t* counts, int64_t G, int64_t* offsets, int64_t* block_tmp,
                        cudaStream_t st);
cudaError_t launch_crop_emit(const ShapeTable& T, const Batch& b, cudaStream_t st);
// S2-S3 fused (transform + crop + compaction with a decoupled look-back, one launch; K <= kFusedMaxK):
// lb = crop_compact_lb_words(G) look-back words (zeroed by the launcher on `st`).
constexpr int kFusedMaxK = 2048;  // eight warps' shared-memory row lists: 64 KB per block
size_t crop_compact_lb_words(int64_t G);
cudaError_t launch_crop_compact(const ShapeTable& T, const Batch& b, int words, unsigned long long* lb,
                                cudaStream_t st);
cudaError_t launch_encoder_f32(const DevParams& P, const Batch& b, cudaStream_t st);
cudaError_t launch_encoder_tc(const DevParams& P, const TcL1& l1, const Batch& b, int num_sms, cudaStream_t st,
                              long long* trace = nullptr, bool deterministic = false);
cudaError_t launch_head(const DevParams& P, const Batch& b, float* probs, uint8_t* labels,
                        float* logits, float* emb, float* grad, cudaStream_t st);
// NEXT-1 encode-once mode (kernels_cells.cu)
cudaError_t launch_grid_encode(const DevParams& P, const ShapeTable& T, int M, float* G, cudaStream_t st);
cudaError_t launch_unet(const UNetParams& U, const ShapeTable& T, int M, int H, int F, int global_max, const float* G,
                        float* act, float* E, float* ctr, bool tc, int num_sms, cudaStream_t st);
cudaError_t launch_conv_tc(const float* x1, int C1, const float* x2, int C2, int Di, int Do, int pad, int S,
                           const uint8_t* img, const float* bias, float* y, int num_sms, cudaStream_t st);
size_t unet_act_floats(int S, int M);
cudaError_t launch_gemm_tc(const float* x, int C, int64_t rows, const uint8_t* img, const float* bias, float* y,
                           int ldy, int ycol, int num_sms, cudaStream_t st, const float4* pts = nullptr,
                           const float4* w1b = nullptr);
int64_t grid_tc_chunk_rows(const ShapeTable& T);
cudaError_t launch_grid_encode_tc(const DevParams& P, const ShapeTable& T, int M, float* G, float* bufA, float* bufB,
                                  int num_sms, cudaStream_t st);
cudaError_t launch_cells_select(const ShapeTable& T, const CellsTable& C, const Batch& b, int F, uint32_t* cells,
                                float* emb_out, cudaStream_t st);
// NEXT-3 closed loop (kernels_sim.cu)
cudaError_t launch_sim_set_t0(double* t0_dev, double t0, cudaStream_t st);
cudaError_t launch_sim_prepare(const ShapeTable& T, const SimParams& sp, int E, const int32_t* ids, float* state,
                               const double* t0_dev, int n, int32_t* pairs, float* poses, uint8_t* culled,
                               unsigned long long* bad, cudaStream_t st);
cudaError_t launch_sim_integrate(const SimParams& sp, int E, const float* body, float* state, const float* logits,
                                 const float* grad, const uint8_t* culled, int32_t* contacts, const double* t0_dev,
                                 int n, cudaStream_t st);
cudaError_t launch_head_tc(const DevParams& P, const Batch& b, float* probs, uint8_t* labels, float* logits,
                           float* emb, float* grad, int num_sms, cudaStream_t st);
size_t scan_tmp_elems(int64_t G);
size_t encoder_tc_smem_bytes();

// x / c for a pooled cell sum x and a cell count c (1 <= c <= 216): x * RN(1/c) corrected once with the
// exact FMA residual (Markstein) — bitwise the IEEE quotient __fdiv_rn(x, c) (tools/div_check.cu checks
// every fp32 mantissa in two binades against it for c = 1..216; normal range) at a multiply and two FMAs.
__device__ __forceinline__ float div_count(float x, float c, float rc) {
  const float q0 = x * rc;
  return fmaf(fmaf(-q0, c, x), rc, q0);
}

// Opts kernel `fn` into `bytes` of dynamic shared memory on the CURRENT device.  Function attributes
// are per device, so this is done once per (device, kernel) and remembered (locc_runtime.cu); every
// launcher with more than 48 KB calls it before its launch.
cudaError_t smem_optin(const void* fn, size_t bytes);
template <class K>
cudaError_t smem_optin(K* fn, size_t bytes) {
  return smem_optin(reinterpret_cast<const void*>(fn), bytes);
}

}  // namespace locc
