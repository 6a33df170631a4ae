/* locc.h — C ABI of the B200-native LOCC batched collision query (liblocc.so).
 *
 * LOCC (arXiv 2304.09439, "Local object crop collision network"): for each pair of objects
 * (shape ids + SE(3) poses) return the collision probability and label.  Per pair the library
 * runs, entirely in its own CUDA kernels for sm_100a:
 *   S0 shape prep (once per shape table)   AABB, cell ids, eps
 *   S1 relative transforms                 T_BA, T_AB from the poses
 *   S2-S3 transform + crop + compaction    keep p iff dist(T p, AABB_other) <= eps_other
 *                                                                          PAPER.md:335-337, :424
 *   S4-S5 per-point encoder                3 -> H -> H -> H, ReLU
 *   S6 cell-wise max pool                  over the kept points of a cell PAPER.md:331, :421
 *   S7 mean over occupied cells, linear F  "average pooling" + linear
 *   S8-S9 collision predictor              [e;pose] -> 3x128 -> max over pair -> 3x128 -> 1 -> sigmoid
 *                                                                          PAPER.md:424-425
 * The exact arithmetic of every step (and every reading of an ambiguous passage) is
 * SURVEY.md §8(c) O0-O9, restated in DESIGN.md.  Threshold: label = p > 0.5 (ties negative).
 *
 * Conventions
 *   - Points: float32 [S][K][3], metres, each shape in its own local frame.
 *   - Pose: float32 [7] = (qw, qx, qy, qz, tx, ty, tz); the quaternion need not be unit
 *     (it is normalised in fp64), |q|^2 must be >= 1e-12.
 *   - Pair i: side 0 = object A = pairs[2i] with poses[14i .. 14i+6]; side 1 = B = pairs[2i+1]
 *     with poses[14i+7 .. 14i+13].
 *   - Buffers are caller-owned.  Every pointer passed to one call must have the same residency
 *     (all host, or all device memory of the context's device); the library detects which.
 *   - A context is not reentrant; separate contexts are independent.  Multi-GPU (
 *     pairs are independent), two forms, both sharding the batch into contiguous
 *     shards of ceil(N/G) pairs:
 *       * one process, G devices: locc_config.n_devices > 1 — the context drives one sub-context
 *         per device (its own stream, scratch, weights and shape table) and splits every query;
 *         device-resident caller buffers live on the home device (device_ids[0]) and the other
 *         devices read their shard's inputs and write their outputs there directly over NVLink
 *         (peer access), or through peer copies when peer access is unavailable;
 *       * one process per GPU: locc_comm_init + locc_query_allgather — each rank computes its
 *         shard and the library gathers every rank's results on every rank with NCCL (the only
 *         collective of the path: 9 B per pair).
 *   - Errors: every function returns a locc_status; on error no output is guaranteed written
 *     and locc_last_error() holds a thread-local detail string.  No exception crosses the ABI.
 */
#ifndef LOCC_H
#define LOCC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LOCC_OK = 0,
  LOCC_E_INVALID_ARG = -1, /* bad pointer/size/id/pose/config value */
  LOCC_E_SHAPE = -2,       /* bad shape table: S < 1, K < 1, K > 65535, non-finite point */
  LOCC_E_WEIGHTS = -3,     /* manifest/tensor name/shape mismatch, wrong count, non-finite */
  LOCC_E_CUDA = -4,        /* a CUDA runtime call or kernel failed */
  LOCC_E_OOM = -5,         /* device allocation failed */
  LOCC_E_NCCL = -6,        /* NCCL missing (dlopen of libnccl.so.2) or an NCCL call failed */
  LOCC_E_STATE = -7        /* query before weights and shapes were set */
} locc_status;

typedef enum {
  LOCC_PREC_FP32 = 0, /* encoder layers 2-3 as fp32 FFMA on CUDA cores */
  LOCC_PREC_BF16 = 1  /* encoder layers 2-3 on tcgen05 tensor cores: bf16 h1, W2, h2, W3,
                         fp32 accumulate; layer 1 and pooling stay fp32; the predictor (projection,
                         object and pair MLPs, and its pose gradient) runs on the tensor cores with
                         fp32-accurate 3xTF32 products (reading Q32) */
} locc_precision;

typedef struct {
  int32_t M;         /* voxel grid edge (M = 6); 1 <= M <= 15 */
  int32_t H;         /* point-feature width; 256 for BF16, 32..256 step 32 for FP32 */
  int32_t F;         /* cell-feature width; 1..256 */
  int32_t precision; /* locc_precision */
  int32_t device;    /* CUDA device ordinal; -1 = the calling thread's current device (ignored when
                        n_devices > 1) */
  int32_t n_devices; /* 0 or 1: one device.  > 1: the context drives n_devices devices of this process
                        (one sub-context each, queries sharded into contiguous ceil(N/G) blocks) */
  int64_t max_batch; /* pairs per internal sub-batch per device (bounds scratch memory); 0 = 262144 */
  const int32_t* device_ids; /* n_devices CUDA ordinals (NULL = 0 .. n_devices-1); the first is the
                                home device of device-resident caller buffers.  An ordinal may repeat
                                (sub-contexts sharing a GPU, e.g. to test the sharding on one device).
                                Copied at locc_create. */
} locc_config;

typedef struct locc_ctx locc_ctx;

/* Per-query statistics of the last locc_query / locc_query_debug on this context. */
typedef struct {
  int64_t pairs;            /* N */
  int64_t evaluated_pairs;  /* pairs with n_A + n_B > 0 (the rest are short-circuited) */
  int64_t kept_rows;        /* sum over pairs of n_A + n_B: rows through the encoder */
  int64_t nonempty_sides;   /* sides with n_s > 0 */
  int64_t sub_batches;      /* internal sub-batches */
  int64_t kernel_launches;  /* kernels the library launched for the query */
  double  encoder_ms;       /* device time of the encoder launches (CUDA events; 0 if timing off) */
  double  total_ms;         /* device time of the whole query on its stream (0 if timing off) */
  double  head_ms;          /* device time of the predictor launches (0 if timing off); in the
                               encode-once mode encoder_ms is the cell selection's time */
  double  crop_ms;          /* device time of the transform + crop + compaction launches (0 if timing off) */
  int64_t graph_replay;     /* 1 if the query was replayed from the context's CUDA graph (asynchronous
                               device-buffer queries of one sub-batch; see locc_query) */
} locc_stats;

/* Create a context on cfg->device, or on the cfg->n_devices devices of cfg->device_ids (peer access
 * is enabled between the home device and every other device where the hardware allows it).
 * Every other call fans out to the sub-contexts; locc_get_stats sums the counts and takes the
 * maximum of the per-device times.  Out: *out (free with locc_destroy).
 * Errors: INVALID_ARG (null, M/H/F/precision out of range, bad device ordinal), CUDA, OOM. */
locc_status locc_create(const locc_config* cfg, locc_ctx** out);

/* Load parameters from the checkpoint format: text manifest
 * `manifest_path` with header "locc-weights 1 M H F" then one line per tensor
 * "name out in offset_bytes" in canonical order
 *   enc.l1 [H][3], enc.l2 [H][H], enc.l3 [H][H], enc.proj [F][H], obj.l1 [128][F+7],
 *   obj.l2, obj.l3, pair.l1, pair.l2, pair.l3 [128][128], out [1][128]
 * each as "<layer>.W out in off" (row-major [out][in]) followed by "<layer>.b out 1 off",
 * and the little-endian fp32 payload in the file with the manifest's stem and extension .bin.
 * M, H, F must equal the context's.  Copies to the device; the caller keeps the files.
 * Errors: WEIGHTS (parse error, name/shape/M/H/F mismatch, short file, non-finite value). */
locc_status locc_load_weights(locc_ctx* ctx, const char* manifest_path);

/* Same, from a host array of n_floats fp32 values in the canonical order above. */
locc_status locc_load_weights_mem(locc_ctx* ctx, const float* flat, size_t n_floats);

/* Set the shape table: points [S][K][3] (host or device pointer, caller keeps ownership).
 * The library copies it and computes S0 on the device: AABB lo/hi (min/max of the points),
 * eps^2 = (float)(0.25*((a.x^2 + a.y^2) + a.z^2)), a = ext/M in fp64, cell ids
 * floor((p-lo)*M/ext) clamped to M-1 (0 on a zero-extent axis), and a stable cell-sorted
 * copy of the points.  Errors: SHAPE (S < 1, K < 1, K > 65535, non-finite), INVALID_ARG, CUDA, OOM. */
locc_status locc_set_shapes(locc_ctx* ctx, const float* points, int32_t S, int32_t K);

/* Batched query.  pairs int32 [N][2] in [0, S); poses float32 [N][2][7]; out probs float32 [N];
 * labels uint8 [N] (nullable; p > 0.5); logits float32 [N] (nullable).  Short-circuited pairs
 * (both crops empty): prob 0, label 0, logit -inf.
 * stream: cudaStream_t, or NULL for the library's own stream.  Host-resident buffers: the call
 * copies them in and out and returns when the outputs are written.  Device-resident buffers:
 * with stream == NULL the call returns after completion; with a caller stream it is
 * asynchronous on that stream (and validation of ids/poses happens on the device: an invalid
 * id or pose makes the call return INVALID_ARG only in the synchronous form).
 * CUDA graph: an asynchronous device-buffer call whose N fits one internal sub-batch is captured
 * on the second call with the same arguments (pointers, N, stream) and context state (weights,
 * shapes, grids, precision, determinism, no scratch reallocated since), then replayed as one graph
 * launch; the buffers' CONTENTS may change between calls.  Same for locc_query_grad and
 * locc_query_cells (without its debug outputs).  LOCC_NO_GRAPH=1 disables it.
 * Errors: INVALID_ARG (N < 0, null buffers, id out of range, non-finite pose, |q|^2 < 1e-12),
 * STATE (no weights or no shapes), CUDA, OOM. */
locc_status locc_query(locc_ctx* ctx, const int32_t* pairs, const float* poses, int64_t N,
                       float* probs, uint8_t* labels, float* logits, void* stream);

/* locc_query plus every intermediate needed for bit-exact parity (all nullable):
 * kept int32 [N][2] (n_A, n_B), occ int32 [N][2] (occupied cells C_A, C_B),
 * masks uint32 [N][2][ceil(K/32)] (bit k of word k/32 = the CALLER's point k was kept),
 * emb float32 [N][2][F] (e_A, e_B; 0 for an empty side).  Same residency rule. */
locc_status locc_query_debug(locc_ctx* ctx, const int32_t* pairs, const float* poses, int64_t N,
                             float* probs, uint8_t* labels, float* logits, int32_t* kept,
                             int32_t* occ, uint32_t* masks, float* emb, void* stream);

/* locc_query plus the pose gradient of each logit (the paper's use of the
 * network inside gradient-based planning, PAPER.md §"Introduction"/§"Experiments"):
 * grad float32 [N][14] = d logit_i / d (q_A[4], t_A[3], q_B[4], t_B[3]) of pair i, in the order of
 * poses[14i .. 14i+13].  The crops are held fixed (the crop mask is piecewise constant in the pose,
 * so no gradient flows through it), ReLU'(x) = [x > 0], the max across the pair routes the gradient
 * to the side it selected (u_A > u_B -> A, ties -> B), and the raw quaternion's gradient includes
 * the normalisation and canonical sign: dq = s (dq^ - q^ (q^ . dq^)) / |q|.  Short-circuited pairs
 * (constant logit -inf): grad 0.  Computed in the same fused predictor kernel as the forward: fp32 on
 * CUDA cores in fp32 contexts, 3xTF32 on the tensor cores in bf16 contexts (Q32).
 * Requires H = 256, F = 64.  Same residency, stream and error rules as locc_query.
 * Errors: INVALID_ARG (as locc_query, null grad, H/F not 256/64), STATE, CUDA, OOM. */
locc_status locc_query_grad(locc_ctx* ctx, const int32_t* pairs, const float* poses, int64_t N,
                            float* probs, uint8_t* labels, float* logits, float* grad, void* stream);

/* ---- Encode-once mode: the paper's own inference design ----
 * every shape is encoded ONCE into an M x M x M x F embedding grid
 * (point MLP over all K points -> cell-wise max -> 3D U-Net -> linear), cached on the device; a query
 * transforms the M^3 cell centres of each object into the other's frame, selects the cells within
 * the own cell's half diagonal (the "margin ... distance from the center point to a vertex of a
 * cell") of the other AABB, average-pools the selected embeddings and runs the same
 * predictor.  Query cost is independent of K.  fp32 (bf16 contexts: the tensor-core 3xTF32
 * predictor for F = 64); readings Q27-Q30 in DESIGN.md.  Requires 3 <= M <= 8, H a multiple of 32,
 * F <= 64 (the appendix's F = 16 included).
 *
 * U-Net parameters, canonical order (each W then b [128]; kernels [out][in][27], tap k = kx + 3 (ky
 * + 3 kz)): c1 [128][H][27], c2, c3, c4 [128][128][27], d4 [128][128][27], d3, d2, d1 [128][256][27];
 * then proj W [F][256], b [F].  Count: locc_unet_n_params(H, F). */
int64_t locc_unet_n_params(int32_t H, int32_t F);

/* Load the U-Net parameters (host array of n_floats fp32, canonical order above).
 * Errors: INVALID_ARG (null), WEIGHTS (count, non-finite), CUDA, OOM. */
locc_status locc_load_unet_weights_mem(locc_ctx* ctx, const float* flat, size_t n_floats);

/* The U-Net's global feature ("average pooling ... just before the deconvolution" vs
 * :421 "max pooling to get global features"): 0 = average (default, reading Q28), 1 = max.  Takes
 * effect at the next locc_encode_shapes (the cached grids are invalidated).  Errors: INVALID_ARG. */
locc_status locc_set_unet_global_pool(locc_ctx* ctx, int32_t mode);

/* Encode every shape of the current table and cache the grids on the device (synchronous).  Must be
 * re-run after locc_set_shapes / locc_load_weights / locc_load_unet_weights_mem.  fp32 contexts: CUDA
 * cores (fp32); bf16 contexts: the point MLP's layers 2-3 (H = 256) and the U-Net on the tensor cores
 * in 3xTF32 (Q30, Q32), with about 1 GiB of transient scratch per 2^20 points encoded.
 * Errors: STATE (weights, U-Net weights or shapes missing), INVALID_ARG (M, H, F), CUDA, OOM. */
locc_status locc_encode_shapes(locc_ctx* ctx);

/* Copy the cached grids to out float32 [S][M^3][F] (host or device; nullable) and report the device
 * time of the last locc_encode_shapes in *encode_ms (nullable).  Errors: STATE (nothing encoded). */
locc_status locc_get_cell_embeddings(locc_ctx* ctx, float* out, double* encode_ms);

/* Batched query through the cached grids.  Same inputs, outputs, residency, stream and error rules as
 * locc_query, plus nullable debug outputs: nsel int32 [N][2] selected cells per side, cells uint32
 * [N][2][ceil(M^3/32)] (bit c of word c/32 = cell c = x + M (y + M z) selected), emb float32 [N][2][F]
 * pooled embeddings (0 for a side with no cell).  Short-circuit (prob 0, label 0, logit -inf) when
 * neither side selects a cell.  Errors: as locc_query; STATE if the shapes are not encoded. */
locc_status locc_query_cells(locc_ctx* ctx, const int32_t* pairs, const float* poses, int64_t N,
                             float* probs, uint8_t* labels, float* logits, int32_t* nsel, uint32_t* cells,
                             float* emb, void* stream);

/* ---- Closed-loop simulation step (reading Q31) ----
 * PAPER.md:18-24, :91, :187-192 (BRAX-LOCC: objects dropped into a shaken bowl; the OCN's pose gradient
 * gives the contact direction), SPEC.md S:638-665 (penalty resolution).  E independent environments, 3
 * bodies each: body 0 the kinematic bowl, shaken as t = amp sin(2 pi freq tau), bodies 1, 2 dynamic;
 * pairs (0,1), (0,2), (1,2).  One substep of length h at time tau: bowl pose; world-AABB broad phase with
 * `slack`; the LOCC query with the pose gradient (detector 0: the crop path in the context's precision;
 * 1: the encode-once path); contact iff unculled and logit > 0; per contact, with g_t the translational
 * and G_w[k] = g_q . (1/2 (0, e_k) (x) q) the rotational gradient of the logit s of each body,
 * n = |(g_t, G_w) of both bodies|, ds/dt = sum g_t . v + G_w . w, lambda = max(0, ks s + kd ds/dt):
 * force -lambda g_t / n, torque -lambda G_w / n on the dynamic bodies; semi-implicit Euler
 * (v += h (F/m + gravity), w += h R diag(1/I) R^T tau, t += h v, q = normalise(q + h/2 (0,w) (x) q)). */
typedef struct {
  double h;           /* substep length, s (dt = 0.01/4 s split into 4 substeps) */
  int32_t substeps;   /* substeps per call */
  int32_t detector;   /* 0 = crop path, 1 = encode-once path (needs locc_encode_shapes) */
  float gravity[3];   /* m/s^2 */
  float ks, kd;       /* penalty stiffness (N per logit unit) and damping (N s per logit unit) */
  float amp[3];       /* bowl shake amplitude, m */
  float freq;         /* bowl shake frequency, Hz */
  float slack;        /* broad-phase AABB slack, m */
} locc_sim_config;

/* Advance E environments by cfg->substeps substeps starting at time t0.  DEVICE buffers: ids int32
 * [E][3] shape ids; body float32 [E][3][4] = mass, body-frame principal inertia (Ixx, Iyy, Izz); state
 * float32 [E][3][13] = q (4), t (3), v (3), w (3), world frame, updated in place; contacts int32 [E][3]
 * (nullable) = substeps in contact per pair.  stream NULL: synchronous; else asynchronous on it.
 * An environment with a body id outside [0, S) has its pairs culled for that substep (no contact
 * forces; nothing out of range is read); the synchronous form then returns INVALID_ARG.  The
 * substeps are captured into a CUDA graph on the second call with identical arguments and replayed
 * while no context state or scratch buffer has changed.
 * Errors: INVALID_ARG (sizes, host buffers, H/F not 256/64, bad ids), STATE (weights/shapes/encoding),
 * CUDA, OOM. */
locc_status locc_sim_run(locc_ctx* ctx, const locc_sim_config* cfg, int32_t E, const int32_t* ids,
                         const float* body, float* state, double t0, int32_t* contacts, void* stream);

/* ---- Multi-process sharding with a library-owned NCCL gather ----
 * One process (one single-device context) per GPU.  NCCL is loaded at run time (dlopen of
 * libnccl.so.2: the copy already in the process, e.g. PyTorch's, else the system's); the handshake
 * is the caller's: rank 0 calls locc_comm_unique_id and sends the 128 bytes to the other ranks
 * (e.g. with torch.distributed), then every rank calls locc_comm_init.  */

/* Write a new NCCL unique id (128 bytes) to out.  Errors: INVALID_ARG (null), NCCL. */
locc_status locc_comm_unique_id(uint8_t out[128]);

/* Join the world of `world` ranks as `rank` on the context's device (ncclCommInitRank).  A context
 * holds one communicator; calling again replaces it.  Errors: INVALID_ARG (null, world < 1, rank out
 * of [0, world), multi-device context), NCCL, CUDA. */
locc_status locc_comm_init(locc_ctx* ctx, int32_t world, int32_t rank, const uint8_t id[128]);

/* Sharded query of a GLOBAL batch of N pairs over the communicator's ranks: this rank reads only its
 * contiguous shard [lo, hi) = [r ceil(N/W), min(N, (r+1) ceil(N/W))) of pairs/poses, computes it
 * with locc_query's arithmetic, writes it at [lo, hi) of probs/labels/logits, and the library then
 * gathers every rank's shard into the same global output arrays on every rank (one NCCL group of
 * in-place broadcasts, one per rank's shard; labels and logits nullable, the same on every rank).
 * Pairs outside the shard are never read, so a rank need only fill its own slice of pairs/poses.
 * Every rank must call it with the same N.  Host or device buffers (same rules as locc_query; host
 * outputs are staged through device memory for NCCL); stream NULL = synchronous.
 * Errors: as locc_query; STATE (no communicator); NCCL. */
locc_status locc_query_allgather(locc_ctx* ctx, const int32_t* pairs, const float* poses, int64_t N,
                                 float* probs, uint8_t* labels, float* logits, void* stream);

/* Switch the encoder precision of an existing context (LOCC_PREC_FP32 / LOCC_PREC_BF16). */
locc_status locc_set_precision(locc_ctx* ctx, int32_t precision);

/* Bitwise reproducibility of LOCC_PREC_BF16 contexts (reading Q24).  1 (default): the
 * tensor-core encoder's layer-3 epilogue sums a segment's cell values in an order fixed by the
 * segment's own rows (16-row blocks), so every output is bitwise independent of batch composition
 * (N, pair order, sub-batching, GPU count).  0: a faster walk (~5 % at C3) whose order
 * depends on where the segment falls in its 128-row part, so batch composition can move a probability
 * by a few fp32 ulps (<= 1e-5).  FP32 contexts are always bitwise reproducible.
 * Errors: INVALID_ARG (null). */
locc_status locc_set_deterministic(locc_ctx* ctx, int32_t enabled);

/* Enable (1) / disable (0) CUDA-event timing of the encoder and of the whole query. */
locc_status locc_set_timing(locc_ctx* ctx, int32_t enabled);

/* Statistics of the last query (requires a completed query; reads device counters). */
locc_status locc_get_stats(locc_ctx* ctx, locc_stats* out);

/* Free the context and all its device memory.  NULL-safe. */
void locc_destroy(locc_ctx* ctx);

const char* locc_status_string(locc_status s);
const char* locc_last_error(void);

/* Library version, e.g. "locc-b200 0.1 sm_100a". */
const char* locc_version(void);

#ifdef __cplusplus
}
#endif
#endif
