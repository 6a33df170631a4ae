/* locc_oracle.h — plain, slow, CPU reference of the LOCC batched collision query.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2304_09439_b200/, include/locc.h) never links, imports or calls it, and
 * this file shares no code, header, constant or helper with the CUDA path.
 *
 * What it computes is SURVEY.md §8(c) O0-O9 (the reading of PAPER.md §"Local
 * object crop collision network" lines 325-345 and Appendix "Architecture
 * Details" lines 420-425 adopted for this build; DESIGN.md lists every reading).
 * Geometry (O0-O4) is prescribed fp32/fp64 arithmetic so crop masks can be
 * compared bit-exactly; the network (O6-O9) is fp64.  `bf16_emul` = 1 rounds
 * h1, W2, h2, W3 to bf16 (round-to-nearest-even) before their products — the
 * arithmetic the bf16 tensor-core path is defined to perform.
 *
 * Beyond the headline path: the pose gradient (NEXT-2, oracle_head_grad /
 * oracle_query_grad, fp64 reverse mode), the encode-once mode with the 3D U-Net (NEXT-1,
 * oracle_conv3d / oracle_encode_grid / oracle_query_cells) and the closed-loop substep (NEXT-3,
 * oracle_sim_run); readings Q26-Q31.
 *
 * Parity pins: tests/test_oracle_*.py (network, geometry, grad: finite differences, a closed-form
 * head, symmetries; cells: scipy correlate/convolve, the adjoint identity, a delta-kernel U-Net probe,
 * a box-intersection superset property, a worked example; sim: discrete closed forms, score descent,
 * body-swap symmetry; pins: closed-form probes of the encoder and predictor ReLUs and hidden biases and of
 * the U-Net skip concatenation, each with a mutation check, tests/test_oracle_pins.py and
 * tools/oracle_mutations.py).  "parity unpinned": absolute probabilities of any trained LOCC (no trained
 * weights exist).
 *
 * Return codes: 0 ok; -1 invalid argument; -2 bad shape table; -3 bad weights.
 */
#ifndef LOCC_ORACLE_H
#define LOCC_ORACLE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t M, H, F;    /* voxel grid edge, point-feature width, cell-feature width */
  int32_t bf16_emul;  /* 0: fp64 network; 1: bf16-operand emulation of layers 2-3 */
  int32_t n_threads;  /* 0 = hardware_concurrency */
  int32_t global_max; /* encode-once U-Net global feature: 0 = average (default), 1 = max */
} oracle_cfg;

/* O0 for one shape: lo/hi (float3), eps2, per-point cell ids [K]. */
int oracle_shape_prep(const float* pts /*[K][3]*/, int32_t K, int32_t M, float lo[3], float hi[3],
                      float* eps2, int32_t* cell /*[K]*/);

/* O1-O3 for one pair: R_BA (row-major 3x3), t_BA, R_AB, t_AB, each rounded once to fp32. */
int oracle_rel_transform(const float poseA[7], const float poseB[7], float R_BA[9], float t_BA[3],
                         float R_AB[9], float t_AB[3]);

/* Whole query O0-O9.  Any output pointer may be NULL.  masks: [N][2][ceil(K/32)] bit k of
 * word k/32 = caller's point k kept.  emb: [N][2][F].  Short-circuit: prob 0, label 0,
 * logit -inf.  Returns nonzero on invalid input (ids out of range, |q|^2 < 1e-12, K < 1,
 * non-finite values) without guaranteeing outputs. */
int oracle_query(const oracle_cfg* cfg, const float* weights, size_t n_weights, const float* points,
                 int32_t S, int32_t K, const int32_t* pairs, const float* poses, int64_t N,
                 double* probs, uint8_t* labels, double* logits, int32_t* kept, int32_t* occ,
                 uint32_t* masks, double* emb);

/* NEXT-2: predictor forward + reverse-mode gradient of the logit w.r.t. the raw pose inputs
 * [q_A(4), t_A(3), q_B(4), t_B(3)] at given embeddings e_A, e_B (fp64, poses as doubles so finite
 * differences can probe it).  Crops and embeddings are constant in the pose (see the .cpp). */
int oracle_head_grad(const oracle_cfg* cfg, const float* weights, size_t n_weights, const double* eA,
                     const double* eB, const double poseA[7], const double poseB[7], double* logit,
                     double grad[14]);

/* Whole query plus the pose gradient of each logit: grad [N][14] (zero for short-circuited pairs,
 * whose logit is the constant -inf).  logits, margin may be NULL.  margin [N]: the smallest
 * |pre-activation| over the predictor's ReLUs and |u_A - u_B| over the max's routed features (inf
 * for a short-circuit) — how close the pair's gradient is to a discontinuity. */
int oracle_query_grad(const oracle_cfg* cfg, const float* weights, size_t n_weights, const float* points,
                      int32_t S, int32_t K, const int32_t* pairs, const float* poses, int64_t N, double* logits,
                      double* grad, double* margin);

/* ---- NEXT-1: encode-once LOCC (the paper's own inference design, Q27-Q30) ----
 * U-Net parameters (canonical order): c1 [128][H][27], c2..c4 [128][128][27], d4 [128][128][27],
 * d3, d2, d1 [128][256][27] (each W then b [128]); proj W [F][256], b [F].  Kernel index
 * k = kx + 3 (ky + 3 kz); grids channel-last, position x + D (y + D z). */
int64_t oracle_unet_n_params(int32_t H, int32_t F);

/* One 3x3x3 stride-1 layer in fp64 (b nullable): transposed = 0: cross-correlation with zero padding
 * pad, y [(D+2pad-2)^3][Cout]; transposed = 1: the transposed convolution (scatter definition),
 * y [(D+2-2pad)^3][Cout].  W [Cout][Cin][27]. */
int oracle_conv3d(const double* x, int32_t D, int32_t Cin, const double* W, const double* b, int32_t Cout,
                  int32_t pad, int32_t transposed, double* y);

/* Encode one shape: G [M^3][H] cell-wise max of the point MLP over all K points (nullable), E [M^3][F]
 * the embedding grid (nullable).  M >= 3. */
int oracle_encode_grid(const oracle_cfg* cfg, const float* weights, size_t n_weights, const float* unet_w,
                       size_t n_unet, const float* pts, int32_t K, double* G, double* E);

/* Query through the cached grids: nsel [N][2] selected cells, cells [N][2][ceil(M^3/32)] selection
 * bits, emb [N][2][F] pooled embeddings, grids [S][M^3][F] (only referenced shapes written); all
 * nullable.  Short-circuit when neither side selects a cell. */
int oracle_query_cells(const oracle_cfg* cfg, const float* weights, size_t n_weights, const float* unet_w,
                       size_t n_unet, const float* points, int32_t S, int32_t K, const int32_t* pairs,
                       const float* poses, int64_t N, double* probs, uint8_t* labels, double* logits,
                       int32_t* nsel, uint32_t* cells, double* emb, double* grids);

/* ---- NEXT-3: closed-loop rigid-body substeps with LOCC as the contact detector (Q31) ----
 * sim (13 doubles): h, substeps, detector (0 crop / 1 encode-once cells), gravity[3], ks, kd,
 * amp[3], freq, slack.  ids int32 [E][3] (body 0 = kinematic bowl); body [E][3][4] = m, Ixx, Iyy, Izz
 * (body frame); state [E][3][13] = q, t, v, w (world) in/out; contacts int32 [E][3] = contact substeps
 * per pair (nullable); margins [E][4] = min |logit|, min ReLU margin, min broad-phase gap, min
 * |ks s + kd ds/dt| (nullable).  unet_w needed for detector 1. */
int oracle_sim_run(const oracle_cfg* cfg, const float* weights, size_t n_weights, const float* unet_w,
                   size_t n_unet, const float* points, int32_t S, int32_t K, const double* sim, int32_t E,
                   const int32_t* ids, const double* body, double* state, double t0, int32_t* contacts,
                   double* margins);

/* Parse a weight manifest + .bin (format in include/locc.h) into `out` (canonical order).
 * Returns the float count, or a negative code; writes M, H, F. */
int64_t oracle_load_weights(const char* manifest, float* out, size_t cap, int32_t* M, int32_t* H,
                            int32_t* F);

/* Canonical parameter count for (H, F). */
int64_t oracle_n_params(int32_t H, int32_t F);

#ifdef __cplusplus
}
#endif
#endif
