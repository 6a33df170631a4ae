// locc_runtime.cu — host runtime behind the C ABI of include/locc.h.
//
// Owns the per-context device state (parameters, shape table, scratch), validates inputs, splits a
// query into sub-batches that bound the scratch memory, and launches the kernels of one pass of
// the hot path on one stream:
//   segment_xf -> crop_compact (fused transform + crop + compaction; crop_count -> scan -> crop_emit
//   for K > kFusedMaxK) -> encoder (fp32 or tcgen05) -> head
// No exception crosses the ABI; every CUDA call is checked and mapped to a locc_status.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types and enums only: NCCL is loaded at run time (dlopen), never linked

#include "../../include/locc.h"
#include "internal.h"
#include "tc_ptx.cuh"

using namespace locc;

cudaError_t locc::smem_optin(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;  // (device, kernel) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{dev, fn}];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

struct locc_ctx;
locc_status locc_upload_tc_weights(locc_ctx* c, const float* flat);

namespace {

thread_local std::string g_err;

locc_status fail(locc_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CK(call)                                                                                     \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) {                                                                         \
      return fail(e_ == cudaErrorMemoryAllocation ? LOCC_E_OOM : LOCC_E_CUDA, "%s: %s (%s:%d)", #call, \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                                       \
    }                                                                                                \
  } while (0)

// Bumped whenever any device buffer is (re)allocated: a captured CUDA graph holds raw pointers into
// the scratch buffers, so it is valid only while this epoch is unchanged (locc_sim_run's key).
std::atomic<uint64_t> g_alloc_epoch{0};

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n && p) return cudaSuccess;
    ++g_alloc_epoch;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 256));
    if (e == cudaSuccess) n = std::max<size_t>(bytes, 256);
    return e;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

int64_t n_params(int H, int F) {
  auto L = [](int64_t o, int64_t i) { return o * i + o; };
  return L(H, 3) + 2 * L(H, H) + L(F, H) + L(kPredW, F + 7) + 5 * L(kPredW, kPredW) + L(1, kPredW);
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

struct locc_ctx {
  locc_config cfg{};
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // host-buffer queries: input uploads overlap the previous sub-batch
  cudaStream_t crop_stream = nullptr;  // crop of sub-batch s + 1 overlaps the encoder of sub-batch s
  cudaEvent_t ev_q0 = nullptr, ev_crop[2] = {}, ev_done[2] = {}, ev_cs[64] = {}, ev_ce[64] = {};
  cudaEvent_t ev[2] = {};          // whole-query timing
  cudaEvent_t ev_in[2] = {}, ev_free[2] = {};  // input buffer k & 1: uploaded / released by the kernels
  std::vector<cudaEvent_t> enc_ev;  // per sub-batch encoder start/stop pairs
  std::vector<cudaEvent_t> head_ev;  // per sub-batch predictor stop (its start = the encoder stop)
  std::vector<cudaEvent_t> crop_ev;  // per sub-batch crop start (its stop = the encoder start)
  bool timing = false;
  bool deterministic = true;  // bf16 encoder: the deterministic layer-3 walk (default; locc_set_deterministic)
  bool has_weights = false, has_shapes = false;
  // parameters
  DevBuf params, tc_img, head_tc_img, grid_tc_img;
  DevParams P{};
  TcL1 tc_l1{};
  // shapes
  DevBuf sh_pts, sh_perm, sh_lo, sh_hi;
  ShapeTable T{};
  // scratch for one sub-batch
  int64_t cap_B = 0;
  bool force_2pass = false;  // LOCC_CROP_2PASS at creation: the two-pass crop at any K
  DevBuf trace;
  DevBuf in_pairs, in_poses, in_pairs2, in_poses2, counts, occ, offsets, scan_tmp, rows, pooled, stats, xf, kbits,
      cellc, lb;
  // second buffer set of the overlapped crop pipeline (sub-batches alternate between the two)
  DevBuf counts2, offsets2, scan_tmp2, rows2, pooled2, xf2, kbits2, cellc2, lb2;
  int64_t cap_B2 = 0;
  DevBuf out_probs, out_labels, out_logits, out_kept, out_occ, out_masks, out_emb, out_grad;
  locc_stats last{};
  int64_t timed_subs = 0;  // sub-batches whose encoder events await reading
  bool timed_overlap = false;  // the last timed query ran the overlapped crop pipeline
  // NEXT-1 encode-once mode
  bool has_unet = false, has_cells = false;
  int unet_global_max = 0;  // U-Net global feature: 0 average, 1 max
  DevBuf unet_params, unet_img, cells_E, cells_ctr, cells_emb;
  UNetParams U{};
  CellsTable cells{};
  double encode_ms = 0.0;  // device time of the last locc_encode_shapes
  // NEXT-3 closed-loop scratch
  int64_t sim_cap = 0;
  DevBuf sim_pairs, sim_poses, sim_probs, sim_logits, sim_grad, sim_culled, sim_t0, sim_bad;
  // CUDA graph of one locc_sim_run's substeps, replayed while its inputs are unchanged
  uint64_t generation = 1;  // bumped by every call that changes weights, shapes, grids or precision
  struct SimKey {
    locc_sim_config cfg;
    int32_t E;
    const void *ids, *body, *state, *contacts, *stream;
    uint64_t gen;
    uint64_t alloc_epoch;  // g_alloc_epoch: no scratch buffer the graph points into was reallocated
  } sim_key{};
  int sim_seen = 0;  // calls with sim_key so far (capture on the second)
  int64_t sim_launches = 0;  // kernels inside the captured graph
  cudaGraphExec_t sim_exec = nullptr;
  // CUDA graph of one asynchronous device-buffer query of a single sub-batch (locc_query,
  // locc_query_grad, locc_query_cells), replayed while the call's arguments and the context's state
  // are unchanged: the ~8 launches of a small query become one
  struct QueryKey {
    int32_t kind;  // 0 query, 1 grad, 2 cells
    int32_t precision, det;
    int64_t N;
    const void *pairs, *poses, *probs, *labels, *logits, *extra, *stream;
    uint64_t gen, alloc_epoch;
  } q_key{};
  int q_seen = 0;
  locc_stats q_last{};  // the stats the captured call left
  cudaGraphExec_t q_exec = nullptr;
  // multi-device group (locc_config.n_devices > 1): one single-device sub-context per device; this
  // context's own device is the home device (device_ids[0]) and its state is only the fan-out
  std::vector<locc_ctx*> kids;
  std::vector<char> kid_direct;  // kid i's kernels may address the home device's memory (peer access)
  static constexpr int kGrpBufs = 12;
  DevBuf grp_buf[kGrpBufs];      // this kid's staged shard buffers (no peer access)
  cudaEvent_t grp_ev = nullptr;  // this kid's "shard done" event (recorded on its stream)
  // multi-process communicator (locc_comm_init): ncclComm_t, world size, rank
  void* nccl_comm = nullptr;
  int world = 1, rank = 0;
  DevBuf ag_out[3];  // device staging of host outputs of locc_query_allgather
};

namespace {

// fp32 -> nearest tf32 (ties away from zero), kept in an fp32 container: what cvt.rna.tf32.f32 does.
float tf32_rna_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) != 0x7F800000u) u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// Derived device layouts of the canonical flat parameter vector (see internal.h DevParams).
locc_status upload_params(locc_ctx* c, const float* flat) {
  const int H = c->cfg.H, F = c->cfg.F, P = kPredW;
  struct L {
    const float *W, *b;
    int o, i;
  };
  const float* q = flat;
  auto take = [&q](int o, int i) {
    L l{q, q + (int64_t)o * i, o, i};
    q += (int64_t)o * i + o;
    return l;
  };
  L e1 = take(H, 3), e2 = take(H, H), e3 = take(H, H), pj = take(F, H), o1 = take(P, F + 7), o2 = take(P, P),
    o3 = take(P, P), p1 = take(P, P), p2 = take(P, P), p3 = take(P, P), out = take(1, P);
  std::vector<float> img;
  std::vector<size_t> off;
  auto push = [&](const float* src, size_t n) {
    while (img.size() % 64) img.push_back(0.f);  // 256-byte alignment
    off.push_back(img.size());
    img.insert(img.end(), src, src + n);
  };
  auto pushT = [&](const L& l) {
    std::vector<float> t((size_t)l.o * l.i);
    for (int o = 0; o < l.o; ++o)
      for (int i = 0; i < l.i; ++i) t[(size_t)i * l.o + o] = l.W[(size_t)o * l.i + i];
    push(t.data(), t.size());
  };
  std::vector<float> w1b((size_t)H * 4);
  for (int f = 0; f < H; ++f) {
    for (int j = 0; j < 3; ++j) w1b[4 * f + j] = e1.W[3 * f + j];
    w1b[4 * f + 3] = e1.b[f];
  }
  push(w1b.data(), w1b.size());  // 0
  pushT(e2);                     // 1
  push(e2.b, H);                 // 2
  pushT(e3);                     // 3
  push(e3.b, H);                 // 4
  pushT(pj);                     // 5
  push(pj.b, F);                 // 6
  pushT(o1);                     // 7
  push(o1.b, P);                 // 8
  pushT(o2);                     // 9
  push(o2.b, P);                 // 10
  pushT(o3);                     // 11
  push(o3.b, P);                 // 12
  pushT(p1);                     // 13
  push(p1.b, P);                 // 14
  pushT(p2);                     // 15
  push(p2.b, P);                 // 16
  pushT(p3);                     // 17
  push(p3.b, P);                 // 18
  push(out.W, P);                // 19
  push(out.b, 1);                // 20
  {                              // 21: obj.l1's pose columns [7][128] (reverse mode)
    std::vector<float> t((size_t)7 * P);
    for (int c = 0; c < 7; ++c)
      for (int o = 0; o < P; ++o) t[(size_t)c * P + o] = o1.W[(size_t)o * o1.i + F + c];
    push(t.data(), t.size());
  }
  push(o2.W, (size_t)P * P);     // 22..26: original [out][in] layouts (reverse mode)
  push(o3.W, (size_t)P * P);
  push(p1.W, (size_t)P * P);
  push(p2.W, (size_t)P * P);
  push(p3.W, (size_t)P * P);
  // 27: tensor-core predictor bias block [6][128] + wout [128] + bout
  std::vector<float> hb;
  for (const L* l : {&o1, &o2, &o3, &p1, &p2, &p3}) hb.insert(hb.end(), l->b, l->b + P);
  hb.insert(hb.end(), out.W, out.W + P);
  hb.push_back(out.b[0]);
  hb.insert(hb.end(), pj.b, pj.b + F);
  push(hb.data(), hb.size());
  const size_t bytes = img.size() * sizeof(float);
  CK(c->params.ensure(bytes));
  CK(cudaMemcpy(c->params.p, img.data(), bytes, cudaMemcpyHostToDevice));
  const float* d = c->params.as<float>();
  DevParams& D = c->P;
  D.H = H;
  D.F = F;
  D.w1 = nullptr;
  D.w1b = reinterpret_cast<const float4*>(d + off[0]);
  D.w2T = d + off[1];
  D.b2 = d + off[2];
  D.w3T = d + off[3];
  D.b3 = d + off[4];
  D.wfT = d + off[5];
  D.bf = d + off[6];
  D.o1T = d + off[7];
  D.ob1 = d + off[8];
  D.o2T = d + off[9];
  D.ob2 = d + off[10];
  D.o3T = d + off[11];
  D.ob3 = d + off[12];
  D.p1T = d + off[13];
  D.pb1 = d + off[14];
  D.p2T = d + off[15];
  D.pb2 = d + off[16];
  D.p3T = d + off[17];
  D.pb3 = d + off[18];
  D.wout = d + off[19];
  D.bout = d + off[20];
  D.o1p = d + off[21];
  D.o2 = d + off[22];
  D.o3 = d + off[23];
  D.p1 = d + off[24];
  D.p2 = d + off[25];
  D.p3 = d + off[26];
  D.head_tc_bias = d + off[27];
  // tensor-core predictor weights: per layer, 32-K chunks of [128 out x 32 in] K-major SW128 images,
  // hi = tf32(w) then lo = tf32(w - hi) (see kernels_head_tc.cu)
  D.head_tc_img = nullptr;
  D.head_tc_proj = nullptr;
  D.head_tc_bwd = nullptr;
  if (F + 7 <= 96) {
    std::vector<uint8_t> himg;
    for (const L* l : {&o1, &o2, &o3, &p1, &p2, &p3}) {
      const int nch = (l->i + 31) / 32;
      for (int j = 0; j < nch; ++j) {
        const size_t base = himg.size();
        himg.resize(base + 32768, 0);
        for (int n = 0; n < P; ++n)
          for (int k = 0; k < 32; ++k) {
            const int kk = 32 * j + k;
            const float w = kk < l->i ? l->W[(size_t)n * l->i + kk] : 0.f;
            const float hi = tf32_rna_host(w);
            const float lo = tf32_rna_host(w - hi);
            const size_t off = tc::sw128_off((uint32_t)n, (uint32_t)(k >> 2)) + (size_t)(k & 3) * 4;
            std::memcpy(&himg[base + off], &hi, 4);
            std::memcpy(&himg[base + 16384 + off], &lo, 4);
          }
      }
    }
    // the projection W_F [F][H] as 8 chunks of [64 rows x 32 K] (rows 64..127 of each chunk unused)
    const size_t proj_at = himg.size();
    if (H == 256 && F == 64)
      for (int j = 0; j < 8; ++j) {
        const size_t base = himg.size();
        himg.resize(base + 32768, 0);
        for (int n = 0; n < F; ++n)
          for (int k = 0; k < 32; ++k) {
            const float w = pj.W[(size_t)n * H + 32 * j + k];
            const float hi = tf32_rna_host(w);
            const float lo = tf32_rna_host(w - hi);
            const size_t off = tc::sw128_off((uint32_t)n, (uint32_t)(k >> 2)) + (size_t)(k & 3) * 4;
            std::memcpy(&himg[base + off], &hi, 4);
            std::memcpy(&himg[base + 16384 + off], &lo, 4);
          }
      }
    // reverse mode: the transposed weights B[n = in][k = out] = W[out][in] of pair3, pair2, pair1, obj3, obj2
    const size_t bwd_at = himg.size();
    for (const L* l : {&p3, &p2, &p1, &o3, &o2})
      for (int j = 0; j < 4; ++j) {
        const size_t base = himg.size();
        himg.resize(base + 32768, 0);
        for (int n = 0; n < P; ++n)
          for (int k = 0; k < 32; ++k) {
            const float w = l->W[(size_t)(32 * j + k) * l->i + n];
            const float hi = tf32_rna_host(w);
            const float lo = tf32_rna_host(w - hi);
            const size_t off = tc::sw128_off((uint32_t)n, (uint32_t)(k >> 2)) + (size_t)(k & 3) * 4;
            std::memcpy(&himg[base + off], &hi, 4);
            std::memcpy(&himg[base + 16384 + off], &lo, 4);
          }
      }
    CK(c->head_tc_img.ensure(himg.size()));
    CK(cudaMemcpy(c->head_tc_img.p, himg.data(), himg.size(), cudaMemcpyHostToDevice));
    D.head_tc_img = c->head_tc_img.p;
    D.head_tc_proj = (H == 256 && F == 64) ? static_cast<const uint8_t*>(c->head_tc_img.p) + proj_at : nullptr;
    D.head_tc_bwd = static_cast<const uint8_t*>(c->head_tc_img.p) + bwd_at;
  }
  D.tc_w2 = nullptr;
  D.tc_w3 = nullptr;
  // tensor-core grid encode (encode-once, bf16 contexts): e2, e3 as [half][chunk] images, same format
  D.grid_tc_img = nullptr;
  if (H == 256) {
    std::vector<uint8_t> gimg;
    for (const L* l : {&e2, &e3})
      for (int half = 0; half < 2; ++half)
        for (int j = 0; j < 8; ++j) {
          const size_t base = gimg.size();
          gimg.resize(base + 32768, 0);
          for (int n = 0; n < 128; ++n)
            for (int k = 0; k < 32; ++k) {
              const float w = l->W[(size_t)(128 * half + n) * H + 32 * j + k];
              const float hi = tf32_rna_host(w);
              const float lo = tf32_rna_host(w - hi);
              const size_t off = tc::sw128_off((uint32_t)n, (uint32_t)(k >> 2)) + (size_t)(k & 3) * 4;
              std::memcpy(&gimg[base + off], &hi, 4);
              std::memcpy(&gimg[base + 16384 + off], &lo, 4);
            }
        }
    CK(c->grid_tc_img.ensure(gimg.size()));
    CK(cudaMemcpy(c->grid_tc_img.p, gimg.data(), gimg.size(), cudaMemcpyHostToDevice));
    D.grid_tc_img = c->grid_tc_img.as<uint8_t>();
  }
  c->has_weights = true;
  return LOCC_OK;
}

// The two-pass crop (crop_count -> scan -> crop_emit) for K > kFusedMaxK, or on request (LOCC_CROP_2PASS:
// A/B timing and bitwise comparison of the fused kernel; read when the context is created).
bool crop_2pass(const locc_ctx* c) { return c->T.K > kFusedMaxK || c->force_2pass; }

// The second buffer set of the overlapped crop pipeline.
locc_status ensure_scratch2(locc_ctx* c, int64_t B) {
  const int K = c->T.K;
  const int64_t G = 2 * B;
  if (B > c->cap_B2) {
    CK(c->counts2.ensure(sizeof(int32_t) * G));
    CK(c->offsets2.ensure(sizeof(int64_t) * (G + 1)));
    CK(c->lb2.ensure(sizeof(unsigned long long) * crop_compact_lb_words(G)));
    if (crop_2pass(c)) CK(c->scan_tmp2.ensure(sizeof(int64_t) * scan_tmp_elems(G)));
    CK(c->rows2.ensure(sizeof(uint2) * (size_t)G * seg_rows(K)));
    CK(c->pooled2.ensure(sizeof(float) * (size_t)G * c->cfg.H));
    CK(c->cellc2.ensure(sizeof(int32_t) * G));
    CK(c->xf2.ensure(sizeof(float4) * 4 * G));
    if (crop_2pass(c)) CK(c->kbits2.ensure(sizeof(uint32_t) * G * ((K + 31) / 32)));
    c->cap_B2 = B;
  }
  return LOCC_OK;
}

locc_status ensure_scratch(locc_ctx* c, int64_t B, bool need_masks, bool need_grad) {
  const int K = c->T.K;
  const int64_t G = 2 * B;
  if (B > c->cap_B) {
    CK(c->in_pairs.ensure(sizeof(int32_t) * 2 * B));
    CK(c->in_poses.ensure(sizeof(float) * 14 * B));
    CK(c->in_pairs2.ensure(sizeof(int32_t) * 2 * B));
    CK(c->in_poses2.ensure(sizeof(float) * 14 * B));
    CK(c->counts.ensure(sizeof(int32_t) * G));
    CK(c->xf.ensure(sizeof(float4) * 4 * G));
    if (crop_2pass(c)) CK(c->kbits.ensure(sizeof(uint32_t) * G * ((K + 31) / 32)));
    CK(c->lb.ensure(sizeof(unsigned long long) * crop_compact_lb_words(G)));
    CK(c->occ.ensure(sizeof(int32_t) * G));
    CK(c->offsets.ensure(sizeof(int64_t) * (G + 1)));
    if (crop_2pass(c)) CK(c->scan_tmp.ensure(sizeof(int64_t) * scan_tmp_elems(G)));
    CK(c->rows.ensure(sizeof(uint2) * (size_t)G * seg_rows(K)));
    CK(c->pooled.ensure(sizeof(float) * (size_t)G * c->cfg.H));
    CK(c->cellc.ensure(sizeof(int32_t) * G));
    CK(c->out_probs.ensure(sizeof(float) * B));
    CK(c->out_labels.ensure(B));
    CK(c->out_logits.ensure(sizeof(float) * B));
    CK(c->out_kept.ensure(sizeof(int32_t) * G));
    CK(c->out_occ.ensure(sizeof(int32_t) * G));
    CK(c->out_emb.ensure(sizeof(float) * (size_t)G * c->cfg.F));
    c->cap_B = B;
  }
  CK(c->stats.ensure(sizeof(DevStats)));
  if (need_masks) CK(c->out_masks.ensure(sizeof(uint32_t) * (size_t)G * ((K + 31) / 32)));
  if (need_grad) CK(c->out_grad.ensure(sizeof(float) * (size_t)14 * c->cap_B));
  return LOCC_OK;
}

// S1-S3 of one sub-batch on `st`: per-segment transforms, then the fused crop (crop_compact) or, for
// K > kFusedMaxK (its shared-memory row list would not fit), crop_count -> scan -> crop_emit.
cudaError_t launch_crop(locc_ctx* c, const Batch& b, int words, bool set2, cudaStream_t st) {
  cudaError_t e = launch_segment_xf(c->T, b, st);
  if (e != cudaSuccess) return e;
  if (!crop_2pass(c))
    return launch_crop_compact(c->T, b, words, (set2 ? c->lb2 : c->lb).as<unsigned long long>(), st);
  if ((e = launch_crop_count(c->T, b, words, st)) != cudaSuccess) return e;
  if ((e = launch_scan(b.counts, b.G, b.offsets, (set2 ? c->scan_tmp2 : c->scan_tmp).as<int64_t>(), st)) != cudaSuccess)
    return e;
  return launch_crop_emit(c->T, b, st);
}

// The predictor runs on the tensor cores (3xTF32, kernels_head_tc.cu) in LOCC_PREC_BF16 contexts; the
// LOCC_PREC_FP32 parity path keeps the CUDA-core fp32 predictor (reading Q32).
bool use_head_tc(const locc_ctx* c) {
  return c->cfg.precision == LOCC_PREC_BF16 && c->P.head_tc_img && !getenv("LOCC_HEAD_FFMA");
}

int64_t batch_cap(const locc_ctx* c) {
  int64_t B = c->cfg.max_batch > 0 ? c->cfg.max_batch : 262144;
  // bound the compacted-row buffer (worst case every point kept) to ~12 GiB
  const int64_t rows_budget = (int64_t)12 << 30;
  const int64_t per_pair = 2LL * seg_rows(c->T.K) * (int64_t)sizeof(uint2);
  B = std::min<int64_t>(B, std::max<int64_t>(1, rows_budget / per_pair));
  return std::min<int64_t>(B, (int64_t)1 << 29);
}

// Elapsed times of the last timed query (its events must have completed).
locc_status read_timing(locc_ctx* c) {
  if (!c->timed_subs) return LOCC_OK;
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
  c->last.total_ms = ms;
  double enc = 0.0, head = 0.0, crop = 0.0;
  for (int64_t s = 0; s < c->timed_subs; ++s) {
    CK(cudaEventElapsedTime(&ms, c->enc_ev[2 * s], c->enc_ev[2 * s + 1]));
    enc += ms;
    CK(cudaEventElapsedTime(&ms, c->enc_ev[2 * s + 1], c->head_ev[s]));
    head += ms;
    if (c->timed_overlap) {
      if (s < 64) {
        CK(cudaEventElapsedTime(&ms, c->ev_cs[s], c->ev_ce[s]));
        crop += ms;
      }
    } else {
      CK(cudaEventElapsedTime(&ms, c->crop_ev[s], c->enc_ev[2 * s]));
      crop += ms;
    }
  }
  c->last.encoder_ms = enc;
  c->last.head_ms = head;
  c->last.crop_ms = crop;
  if (getenv("LOCC_TIMELINE")) {  // diagnostic: each sub-batch's stages relative to the query start (ms)
    auto at = [&](cudaEvent_t e) {
      float t = 0.f;
      return cudaEventElapsedTime(&t, c->ev[0], e) == cudaSuccess ? t : -1.f;
    };
    for (int64_t s = 0; s < c->timed_subs; ++s)
      fprintf(stderr, "timeline sub %lld: crop %.2f-%.2f encoder %.2f-%.2f head end %.2f\n", (long long)s,
              c->timed_overlap && s < 64 ? at(c->ev_cs[s]) : at(c->crop_ev[s]),
              c->timed_overlap && s < 64 ? at(c->ev_ce[s]) : at(c->enc_ev[2 * s]), at(c->enc_ev[2 * s]),
              at(c->enc_ev[2 * s + 1]), at(c->head_ev[s]));
  }
  c->timed_subs = 0;
  return LOCC_OK;
}

locc_status run_query(locc_ctx* c, const int32_t* pairs, const float* poses, int64_t N, float* probs,
                      uint8_t* labels, float* logits, int32_t* kept, int32_t* occ, uint32_t* masks, float* emb,
                      float* grad, void* stream, bool cells = false) {
  if (!c) return fail(LOCC_E_INVALID_ARG, "null context");
  if (N < 0) return fail(LOCC_E_INVALID_ARG, "N < 0");
  if (!c->has_weights || !c->has_shapes) return fail(LOCC_E_STATE, "weights and shapes must be set before a query");
  if (cells && !c->has_cells)
    return fail(LOCC_E_STATE, "locc_encode_shapes must run (after weights, U-Net weights and shapes) first");
  if (N == 0) {
    c->last = locc_stats{};
    return LOCC_OK;
  }
  if (!pairs || !poses || !probs) return fail(LOCC_E_INVALID_ARG, "pairs, poses and probs must be non-null");
  CK(cudaSetDevice(c->device));
  const bool dev = is_device_ptr(pairs);
  if (grad && (c->cfg.H != 256 || c->cfg.F != 64))
    return fail(LOCC_E_INVALID_ARG, "the pose gradient is built for H = 256, F = 64");
  const void* all[] = {poses, probs, labels, logits, kept, occ, masks, emb, grad};
  for (const void* p : all)
    if (p && is_device_ptr(p) != dev)
      return fail(LOCC_E_INVALID_ARG, "all buffers of one call must be host or all device memory");
  // Inputs are validated on the device (segment_xf_kernel: ids in range, finite
  // poses, |q|^2 >= 1e-12); an invalid segment is counted and the call returns LOCC_E_INVALID_ARG.
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  const bool sync = !dev || !stream;
  const int64_t Bcap = std::min<int64_t>(N, batch_cap(c));
  const int K = c->T.K, ncell = c->cfg.M * c->cfg.M * c->cfg.M;
  const int words = cells ? (ncell + 31) / 32 : (K + 31) / 32;
  locc_status s = ensure_scratch(c, Bcap, masks != nullptr && !cells, grad != nullptr);
  if (s != LOCC_OK) return s;
  if (cells) {
    CK(c->cells_emb.ensure(sizeof(float) * (size_t)2 * Bcap * c->cfg.F));
    if (masks) CK(c->out_masks.ensure(sizeof(uint32_t) * (size_t)2 * Bcap * words));
  }
  DevStats* dstats = c->stats.as<DevStats>();
  CK(cudaMemsetAsync(dstats, 0, sizeof(DevStats), st));
  // Overlapped crop pipeline (crop path, no debug outputs, >= 2 sub-batches): the crop of
  // sub-batch s + 1 runs on a low-priority stream into the other buffer set while the encoder runs
  // sub-batch s — the crop warps fill issue slots the latency-bound encoder leaves idle.
  const int64_t n_sub_all = (N + Bcap - 1) / Bcap;
  const bool overlap = !cells && !kept && !occ && !masks && !emb && n_sub_all >= 2 &&
                       c->cfg.precision == LOCC_PREC_BF16 && !getenv("LOCC_NO_OVERLAP");
  if (overlap) {
    s = ensure_scratch2(c, Bcap);
    if (s != LOCC_OK) return s;
    CK(cudaEventRecord(c->ev_q0, st));
    CK(cudaStreamWaitEvent(c->crop_stream, c->ev_q0, 0));
  }
  c->timed_overlap = overlap;
  const int64_t n_sub = (N + Bcap - 1) / Bcap;
  if (c->timing) {
    while ((int64_t)c->enc_ev.size() < 2 * n_sub) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->enc_ev.push_back(e);
    }
    while ((int64_t)c->head_ev.size() < n_sub) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->head_ev.push_back(e);
    }
    while ((int64_t)c->crop_ev.size() < n_sub) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->crop_ev.push_back(e);
    }
    CK(cudaEventRecord(c->ev[0], st));
  }
  int64_t launches = 0, subs = 0;
  for (int64_t i0 = 0; i0 < N;) {
    const int64_t B = std::min(Bcap, N - i0);
    Batch b{};
    b.B = B;
    b.G = 2 * B;
    if (dev) {
      b.pairs = pairs + 2 * i0;
      b.poses = poses + 14 * i0;
    } else {
      // upload on the copy stream into buffer subs & 1 (released by sub-batch subs - 2), so it overlaps
      // the kernels of the previous sub-batch
      const int buf = (int)(subs & 1);
      DevBuf& dp = buf ? c->in_pairs2 : c->in_pairs;
      DevBuf& dq = buf ? c->in_poses2 : c->in_poses;
      if (subs >= 2) CK(cudaStreamWaitEvent(c->copy_stream, c->ev_free[buf], 0));
      CK(cudaMemcpyAsync(dp.p, pairs + 2 * i0, sizeof(int32_t) * 2 * B, cudaMemcpyHostToDevice, c->copy_stream));
      CK(cudaMemcpyAsync(dq.p, poses + 14 * i0, sizeof(float) * 14 * B, cudaMemcpyHostToDevice, c->copy_stream));
      CK(cudaEventRecord(c->ev_in[buf], c->copy_stream));
      CK(cudaStreamWaitEvent(st, c->ev_in[buf], 0));
      if (overlap) CK(cudaStreamWaitEvent(c->crop_stream, c->ev_in[buf], 0));
      b.pairs = dp.as<int32_t>();
      b.poses = dq.as<float>();
    }
    const bool set2 = overlap && (subs & 1);
    b.counts = (dev && kept) ? kept + 2 * i0 : (set2 ? c->counts2 : c->counts).as<int32_t>();
    b.occ = (dev && occ) ? occ + 2 * i0 : c->occ.as<int32_t>();
    b.want_occ = occ != nullptr;
    b.offsets = (set2 ? c->offsets2 : c->offsets).as<int64_t>();
    b.rows = (set2 ? c->rows2 : c->rows).as<uint2>();
    b.rows_cap = 2 * (set2 ? c->cap_B2 : c->cap_B) * seg_rows(c->T.K);
#if LOCC_CHECKED
    if (getenv("LOCC_CHECK_SELFTEST")) b.rows_cap = 1;  // tools/checked_run.py: a check must fire
#endif
    b.pts = c->T.pts;
    b.K = c->T.K;
    b.S = c->T.S;
    b.pooled = (set2 ? c->pooled2 : c->pooled).as<float>();
    // the tensor-core encoder leaves cell sums and counts (the predictor divides); fp32: means
    b.cells_c = (!cells && c->cfg.precision == LOCC_PREC_BF16) ? (set2 ? c->cellc2 : c->cellc).as<int32_t>() : nullptr;
    b.stats = dstats;
    b.xf = (set2 ? c->xf2 : c->xf).as<float4>();
    b.kbits = (set2 ? c->kbits2 : c->kbits).as<uint32_t>();
    b.masks = nullptr;
    if (masks) {
      b.masks = dev ? masks + (size_t)2 * i0 * words : c->out_masks.as<uint32_t>();
      CK(cudaMemsetAsync(b.masks, 0, sizeof(uint32_t) * (size_t)2 * B * words, st));
    }
    float* d_probs = dev ? probs + i0 : c->out_probs.as<float>();
    uint8_t* d_labels = labels ? (dev ? labels + i0 : c->out_labels.as<uint8_t>()) : nullptr;
    float* d_logits = logits ? (dev ? logits + i0 : c->out_logits.as<float>()) : nullptr;
    float* d_emb = emb ? (dev ? emb + (size_t)2 * i0 * c->cfg.F : c->out_emb.as<float>()) : nullptr;
    float* d_grad = grad ? (dev ? grad + 14 * i0 : c->out_grad.as<float>()) : nullptr;

    if (cells) {
      // encode-once mode: select cells, pool the cached embeddings, then the predictor
      if (c->timing) CK(cudaEventRecord(c->crop_ev[subs], st));
      if (c->timing) CK(cudaEventRecord(c->enc_ev[2 * subs], st));
      float* e_in = (emb && dev) ? emb + (size_t)2 * i0 * c->cfg.F : c->cells_emb.as<float>();
      CK(launch_segment_xf(c->T, b, st));
      CK(launch_cells_select(c->T, c->cells, b, c->cfg.F, b.masks, e_in, st));
      if (c->timing) CK(cudaEventRecord(c->enc_ev[2 * subs + 1], st));
      b.emb_in = e_in;
      if (occ) CK(cudaMemsetAsync(b.occ, 0, sizeof(int32_t) * 2 * B, st));
      if (use_head_tc(c) && c->cfg.F == 64)
        CK(launch_head_tc(c->P, b, d_probs, d_labels, d_logits, nullptr, d_grad, c->num_sms, st));
      else
        CK(launch_head(c->P, b, d_probs, d_labels, d_logits, nullptr, d_grad, st));
      if (c->timing) CK(cudaEventRecord(c->head_ev[subs], st));
      if (emb) d_emb = e_in;  // the selection wrote e (0 for an empty side) in place
      launches += 3;
    } else {
    if (overlap) {
      const int j = (int)(subs & 1);
      cudaStream_t cs = c->crop_stream;
      if (subs >= 2) CK(cudaStreamWaitEvent(cs, c->ev_done[j], 0));  // sub-batch s - 2 done with set j
      if (c->timing && subs < 64) CK(cudaEventRecord(c->ev_cs[subs], cs));
      CK(launch_crop(c, b, words, set2, cs));
      if (c->timing && subs < 64) CK(cudaEventRecord(c->ev_ce[subs], cs));
      CK(cudaEventRecord(c->ev_crop[j], cs));
      CK(cudaStreamWaitEvent(st, c->ev_crop[j], 0));
    } else {
      if (c->timing) CK(cudaEventRecord(c->crop_ev[subs], st));
      CK(launch_crop(c, b, words, false, st));
    }
    if (c->timing) CK(cudaEventRecord(c->enc_ev[2 * subs], st));
    if (c->cfg.precision == LOCC_PREC_BF16) {
      long long* trace = nullptr;
      if (getenv("LOCC_TC_TRACE") && subs == 0) {
        CK(c->trace.ensure(sizeof(long long) * 3 * 64 * 32));
        CK(cudaMemsetAsync(c->trace.p, 0, sizeof(long long) * 3 * 64 * 32, st));
        trace = c->trace.as<long long>();
      }
      CK(launch_encoder_tc(c->P, c->tc_l1, b, c->num_sms, st, trace, c->deterministic));
      if (trace) {
        std::vector<long long> h(3 * 64 * 32);
        CK(cudaMemcpyAsync(h.data(), trace, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int rk = 0; rk < 3; ++rk) {  // rank 0, rank 1, tensor-core probes (rank 1 clock)
          const long long t0 = 0;  // raw clock64 (ranks 1 and 2 share the clock of CTA 1's SM)
          for (int t = 0; t < 64; ++t) {
            fprintf(stderr, "trace r%d t%02d", rk, t);
            for (int e = 0; e < 32; ++e) {
              long long v = h[(rk * 64 + t) * 32 + e];
              fprintf(stderr, " %7lld", v ? v - t0 : -1);
            }
            fprintf(stderr, "\n");
          }
        }
      }
    } else {
      CK(launch_encoder_f32(c->P, b, st));
    }
    if (c->timing) CK(cudaEventRecord(c->enc_ev[2 * subs + 1], st));
    if (use_head_tc(c) && c->P.head_tc_proj)
      CK(launch_head_tc(c->P, b, d_probs, d_labels, d_logits, d_emb, d_grad, c->num_sms, st));
    else
      CK(launch_head(c->P, b, d_probs, d_labels, d_logits, d_emb, d_grad, st));
    if (c->timing) CK(cudaEventRecord(c->head_ev[subs], st));
    if (overlap) CK(cudaEventRecord(c->ev_done[subs & 1], st));
    launches += crop_2pass(c) ? 8 : 4;
    }
    if (!dev) CK(cudaEventRecord(c->ev_free[subs & 1], st));  // the kernels are done with the inputs
    ++subs;
    if (!dev) {
      CK(cudaMemcpyAsync(probs + i0, d_probs, sizeof(float) * B, cudaMemcpyDeviceToHost, st));
      if (labels) CK(cudaMemcpyAsync(labels + i0, d_labels, B, cudaMemcpyDeviceToHost, st));
      if (logits) CK(cudaMemcpyAsync(logits + i0, d_logits, sizeof(float) * B, cudaMemcpyDeviceToHost, st));
      if (kept) CK(cudaMemcpyAsync(kept + 2 * i0, b.counts, sizeof(int32_t) * 2 * B, cudaMemcpyDeviceToHost, st));
      if (occ) CK(cudaMemcpyAsync(occ + 2 * i0, b.occ, sizeof(int32_t) * 2 * B, cudaMemcpyDeviceToHost, st));
      if (masks)
        CK(cudaMemcpyAsync(masks + (size_t)2 * i0 * words, b.masks, sizeof(uint32_t) * (size_t)2 * B * words,
                           cudaMemcpyDeviceToHost, st));
      if (emb)
        CK(cudaMemcpyAsync(emb + (size_t)2 * i0 * c->cfg.F, d_emb, sizeof(float) * (size_t)2 * B * c->cfg.F,
                           cudaMemcpyDeviceToHost, st));
      if (grad) CK(cudaMemcpyAsync(grad + 14 * i0, d_grad, sizeof(float) * 14 * B, cudaMemcpyDeviceToHost, st));
    } else {
      if (kept && b.counts != kept + 2 * i0)
        CK(cudaMemcpyAsync(kept + 2 * i0, b.counts, sizeof(int32_t) * 2 * B, cudaMemcpyDeviceToDevice, st));
    }
    i0 += B;
  }
  if (c->timing) CK(cudaEventRecord(c->ev[1], st));
  c->last = locc_stats{};
  c->last.pairs = N;
  c->last.sub_batches = subs;
  c->last.kernel_launches = launches;
  c->timed_subs = c->timing ? subs : 0;
  if (sync) {
    CK(cudaStreamSynchronize(st));
    DevStats hs;
    CK(cudaMemcpy(&hs, dstats, sizeof hs, cudaMemcpyDeviceToHost));
    c->last.kept_rows = (int64_t)hs.kept_rows;
    c->last.nonempty_sides = (int64_t)hs.nonempty_sides;
    c->last.evaluated_pairs = (int64_t)hs.evaluated_pairs;
    locc_status ts = read_timing(c);
    if (ts != LOCC_OK) return ts;
    if (hs.bad_input) return fail(LOCC_E_INVALID_ARG, "%llu segments had an out-of-range id or invalid pose",
                                  (unsigned long long)hs.bad_input);
  }
  return LOCC_OK;
}


// ---------------------------------------------------------------- multi-device groups (n_devices > 1)
// A shard's view of one caller buffer: base pointer, bytes per pair (or environment), and whether the
// shard reads it (in) and/or writes it (out).
struct Slice {
  const void* base;
  size_t unit;
  bool in, out;
};

bool is_group(const locc_ctx* c) { return c && !c->kids.empty(); }

int pointer_device(const void* p) {
  cudaPointerAttributes a;
  if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) ? a.device : -1;
}

// Runs fn(kid, ptrs, n, stream) on every device's contiguous shard of N units: [g ceil(N/G), ...).
// Host buffers: one host thread per device, each a synchronous shard call (stream = NULL).  Device
// buffers (home device): every kid stream waits for the caller's stream, reads its inputs and writes
// its outputs in place (peer access, `direct`) or through peer copies of its slices, and the caller's
// stream waits for every kid; stream == NULL makes the whole call synchronous, after which `check`
// validates every kid (device-side input errors).
template <class Fn, class Check>
locc_status group_run(locc_ctx* c, int64_t N, const Slice* sl, int nsl, bool dev, void* stream, bool allow_direct,
                      Fn fn, Check check) {
  const int G = (int)c->kids.size();
  const int64_t per = (N + G - 1) / G;
  int cur = 0;
  cudaGetDevice(&cur);
  locc_status res = LOCC_OK;
  if (!dev) {
    std::vector<std::thread> th;
    std::vector<locc_status> st(G, LOCC_OK);
    std::vector<std::string> msg(G);
    for (int g = 0; g < G; ++g) {
      const int64_t lo = std::min<int64_t>(N, g * per), hi = std::min<int64_t>(N, lo + per);
      if (hi <= lo) continue;
      th.emplace_back([&, g, lo, hi] {
        void* p[locc_ctx::kGrpBufs] = {};
        for (int i = 0; i < nsl; ++i)
          p[i] = sl[i].base ? (void*)(static_cast<const char*>(sl[i].base) + lo * sl[i].unit) : nullptr;
        st[g] = fn(c->kids[g], p, hi - lo, nullptr);
        if (st[g] != LOCC_OK) msg[g] = g_err;
      });
    }
    for (auto& t : th) t.join();
    for (int g = 0; g < G && res == LOCC_OK; ++g)
      if (st[g] != LOCC_OK) {
        res = st[g];
        g_err = "device " + std::to_string(c->kids[g]->device) + ": " + msg[g];
      }
    cudaSetDevice(cur);
    return res;
  }
  CK(cudaSetDevice(c->device));
  cudaStream_t hs = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  CK(cudaEventRecord(c->ev_q0, hs));
  for (int g = 0; g < G && res == LOCC_OK; ++g) {
    locc_ctx* k = c->kids[g];
    const int64_t lo = std::min<int64_t>(N, g * per), hi = std::min<int64_t>(N, lo + per), n = hi - lo;
    if (n <= 0) continue;
    const bool direct = k->device == c->device || (allow_direct && c->kid_direct[g]);
    CK(cudaSetDevice(k->device));
    CK(cudaStreamWaitEvent(k->stream, c->ev_q0, 0));
    void* p[locc_ctx::kGrpBufs] = {};
    for (int i = 0; i < nsl; ++i) {
      if (!sl[i].base) continue;
      char* at = const_cast<char*>(static_cast<const char*>(sl[i].base)) + lo * sl[i].unit;
      if (direct) {
        p[i] = at;
        continue;
      }
      CK(k->grp_buf[i].ensure(n * sl[i].unit));
      p[i] = k->grp_buf[i].p;
      if (sl[i].in) CK(cudaMemcpyPeerAsync(p[i], k->device, at, c->device, n * sl[i].unit, k->stream));
    }
    res = fn(k, p, n, k->stream);
    if (res != LOCC_OK) break;
    if (!direct)
      for (int i = 0; i < nsl; ++i)
        if (sl[i].base && sl[i].out)
          CK(cudaMemcpyPeerAsync(const_cast<char*>(static_cast<const char*>(sl[i].base)) + lo * sl[i].unit,
                                 c->device, p[i], k->device, n * sl[i].unit, k->stream));
    CK(cudaEventRecord(k->grp_ev, k->stream));
    CK(cudaSetDevice(c->device));
    CK(cudaStreamWaitEvent(hs, k->grp_ev, 0));
  }
  if (res == LOCC_OK && !stream) {
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(hs));
    for (int g = 0; g < G && res == LOCC_OK; ++g) {
      const int64_t lo = std::min<int64_t>(N, g * per), hi = std::min<int64_t>(N, lo + per);
      if (hi > lo) res = check(c->kids[g]);
    }
  }
  cudaSetDevice(cur);
  return res;
}

// After a synchronous group call: the kid's device counters (and input validation) of its shard.
locc_status kid_query_check(locc_ctx* k) {
  CK(cudaSetDevice(k->device));
  DevStats hs;
  CK(cudaMemcpy(&hs, k->stats.p, sizeof hs, cudaMemcpyDeviceToHost));
  k->last.kept_rows = (int64_t)hs.kept_rows;
  k->last.nonempty_sides = (int64_t)hs.nonempty_sides;
  k->last.evaluated_pairs = (int64_t)hs.evaluated_pairs;
  locc_status ts = read_timing(k);
  if (ts != LOCC_OK) return ts;
  if (hs.bad_input)
    return fail(LOCC_E_INVALID_ARG, "device %d: %llu segments had an out-of-range id or invalid pose", k->device,
                (unsigned long long)hs.bad_input);
  return LOCC_OK;
}

locc_status kid_sim_check(locc_ctx* k) {
  CK(cudaSetDevice(k->device));
  unsigned long long bad = 0;
  CK(cudaMemcpy(&bad, k->sim_bad.p, sizeof bad, cudaMemcpyDeviceToHost));
  if (bad) return fail(LOCC_E_INVALID_ARG, "device %d: %llu environment substeps had a body id outside [0, S)",
                       k->device, bad);
  return LOCC_OK;
}

// A query of any kind over the group's devices (run_query's arguments, sharded by pair).
locc_status group_query(locc_ctx* c, const int32_t* pairs, const float* poses, int64_t N, float* probs,
                        uint8_t* labels, float* logits, int32_t* kept, int32_t* occ, uint32_t* masks, float* emb,
                        float* grad, void* stream, bool cells) {
  if (N < 0) return fail(LOCC_E_INVALID_ARG, "N < 0");
  if (N == 0) return LOCC_OK;
  if (!pairs || !poses || !probs) return fail(LOCC_E_INVALID_ARG, "pairs, poses and probs must be non-null");
  const int home_dev = pointer_device(pairs);
  const bool dev = home_dev >= 0;
  const void* all[] = {poses, probs, labels, logits, kept, occ, masks, emb, grad};
  for (const void* p : all)
    if (p && pointer_device(p) != home_dev)
      return fail(LOCC_E_INVALID_ARG, "all buffers of one call must be host memory or all on the home device");
  if (dev && home_dev != c->device)
    return fail(LOCC_E_INVALID_ARG, "device buffers must be on the home device %d (got %d)", c->device, home_dev);
  const locc_ctx* k0 = c->kids[0];
  const int ncell = c->cfg.M * c->cfg.M * c->cfg.M;
  const size_t words = cells ? (ncell + 31) / 32 : (k0->T.K + 31) / 32;
  const Slice sl[] = {{pairs, 8, true, false},           {poses, 56, true, false},
                      {probs, 4, false, true},           {labels, 1, false, true},
                      {logits, 4, false, true},          {kept, 8, false, true},
                      {occ, 8, false, true},             {masks, 8 * words, false, true},
                      {emb, 8 * (size_t)c->cfg.F, false, true}, {grad, 56, false, true}};
  // debug outputs are zeroed with memsets on the kid's stream: those go through the kid's own buffers
  const bool allow_direct = !kept && !occ && !masks && !emb;
  return group_run(
      c, N, sl, 10, dev, stream, allow_direct,
      [&](locc_ctx* k, void** p, int64_t n, void* st) {
        return run_query(k, (const int32_t*)p[0], (const float*)p[1], n, (float*)p[2], (uint8_t*)p[3],
                         (float*)p[4], (int32_t*)p[5], (int32_t*)p[6], (uint32_t*)p[7], (float*)p[8], (float*)p[9],
                         st, cells);
      },
      kid_query_check);
}

// Fan-out of a per-context call to every kid (first error wins).
template <class Fn>
locc_status fan_out(locc_ctx* c, Fn fn) {
  int cur = 0;
  cudaGetDevice(&cur);
  locc_status s = LOCC_OK;
  for (locc_ctx* k : c->kids)
    if ((s = fn(k)) != LOCC_OK) break;
  cudaSetDevice(cur);
  return s;
}

// ---------------------------------------------------------------- NCCL (loaded at run time)
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // prefer a copy already in the process (PyTorch's), else the loader's search path
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.why = std::string("dlopen libnccl.so.2: ") + (e ? e : "not found");
      return a;
    }
    bool all = true;
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      all &= f != nullptr;
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.Broadcast, "ncclBroadcast");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    a.ok = all;
    if (!all) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

#define NK(call)                                                                                    \
  do {                                                                                              \
    ncclResult_t r_ = (call);                                                                       \
    if (r_ != ncclSuccess)                                                                          \
      return fail(LOCC_E_NCCL, "%s: %s (%s:%d)", #call, nccl().GetErrorString(r_), __FILE__, __LINE__); \
  } while (0)

// Every rank's shard [lo_q, hi_q) of the global arrays, broadcast in place from rank q to all ranks.
locc_status allgather_slices(locc_ctx* c, int64_t N, float* probs, uint8_t* labels, float* logits, cudaStream_t st) {
  const NcclApi& A = nccl();
  ncclComm_t comm = static_cast<ncclComm_t>(c->nccl_comm);
  const int64_t per = (N + c->world - 1) / c->world;
  NK(A.GroupStart());
  for (int q = 0; q < c->world; ++q) {
    const int64_t lo = std::min<int64_t>(N, q * per), n = std::min<int64_t>(N, lo + per) - lo;
    if (n <= 0) continue;
    NK(A.Broadcast(probs + lo, probs + lo, (size_t)n, ncclFloat32, q, comm, st));
    if (labels) NK(A.Broadcast(labels + lo, labels + lo, (size_t)n, ncclUint8, q, comm, st));
    if (logits) NK(A.Broadcast(logits + lo, logits + lo, (size_t)n, ncclFloat32, q, comm, st));
  }
  NK(A.GroupEnd());
  return LOCC_OK;
}

bool read_file(const std::string& path, std::vector<char>& out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  out.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
  return true;
}

}  // namespace

extern "C" {

const char* locc_version(void) { return "locc-b200 0.1 sm_100a"; }

const char* locc_last_error(void) { return g_err.c_str(); }

const char* locc_status_string(locc_status s) {
  switch (s) {
    case LOCC_OK: return "LOCC_OK";
    case LOCC_E_INVALID_ARG: return "LOCC_E_INVALID_ARG";
    case LOCC_E_SHAPE: return "LOCC_E_SHAPE";
    case LOCC_E_WEIGHTS: return "LOCC_E_WEIGHTS";
    case LOCC_E_CUDA: return "LOCC_E_CUDA";
    case LOCC_E_OOM: return "LOCC_E_OOM";
    case LOCC_E_NCCL: return "LOCC_E_NCCL";
    case LOCC_E_STATE: return "LOCC_E_STATE";
  }
  return "LOCC_E_UNKNOWN";
}

locc_status locc_create(const locc_config* cfg, locc_ctx** out) {
  if (!cfg || !out) return fail(LOCC_E_INVALID_ARG, "null argument");
  *out = nullptr;
  if (cfg->M < 1 || cfg->M > 15) return fail(LOCC_E_INVALID_ARG, "M must be in [1, 15]");
  if (cfg->F < 1 || cfg->F > 256) return fail(LOCC_E_INVALID_ARG, "F must be in [1, 256]");
  if (cfg->precision != LOCC_PREC_FP32 && cfg->precision != LOCC_PREC_BF16)
    return fail(LOCC_E_INVALID_ARG, "unknown precision %d", cfg->precision);
  if (cfg->H < 32 || cfg->H > 256 || cfg->H % 32) return fail(LOCC_E_INVALID_ARG, "H must be 32..256, step 32");
  if (cfg->precision == LOCC_PREC_BF16 && cfg->H != 256)
    return fail(LOCC_E_INVALID_ARG, "the tensor-core encoder is built for H = 256");
  if (cfg->max_batch < 0) return fail(LOCC_E_INVALID_ARG, "max_batch < 0");
  if (cfg->n_devices < 0 || cfg->n_devices > 64) return fail(LOCC_E_INVALID_ARG, "n_devices must be in [0, 64]");
  if (cfg->n_devices > 1) {
    // a group: the home context (streams and events on device_ids[0]) plus one sub-context per device
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    std::vector<int> ids(cfg->n_devices);
    for (int i = 0; i < cfg->n_devices; ++i) {
      ids[i] = cfg->device_ids ? cfg->device_ids[i] : i;
      if (ids[i] < 0 || ids[i] >= ndev) return fail(LOCC_E_INVALID_ARG, "device_ids[%d] = %d of %d devices", i, ids[i], ndev);
    }
    locc_config one = *cfg;
    one.n_devices = 0;
    one.device_ids = nullptr;
    one.device = ids[0];
    locc_ctx* g = nullptr;
    locc_status s = locc_create(&one, &g);
    if (s != LOCC_OK) return s;
    for (int i = 0; i < cfg->n_devices; ++i) {
      one.device = ids[i];
      locc_ctx* k = nullptr;
      s = locc_create(&one, &k);
      if (s == LOCC_OK && cudaEventCreateWithFlags(&k->grp_ev, cudaEventDisableTiming) != cudaSuccess)
        s = fail(LOCC_E_CUDA, "event creation on device %d", ids[i]);
      if (k) {
        g->kids.push_back(k);
        int can = 0;
        if (ids[i] != ids[0] && cudaDeviceCanAccessPeer(&can, ids[i], ids[0]) == cudaSuccess && can) {
          cudaSetDevice(ids[i]);
          const cudaError_t e = cudaDeviceEnablePeerAccess(ids[0], 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) can = 0;
          cudaGetLastError();
        }
        g->kid_direct.push_back((char)(ids[i] == ids[0] || can));
      }
      if (s != LOCC_OK) {
        locc_destroy(g);
        return s;
      }
    }
    g->cfg.n_devices = cfg->n_devices;
    cudaSetDevice(ids[0]);
    *out = g;
    return LOCC_OK;
  }
  int dev = cfg->device;
  if (dev < 0) CK(cudaGetDevice(&dev));
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (dev >= ndev) return fail(LOCC_E_INVALID_ARG, "device %d of %d", dev, ndev);
  CK(cudaSetDevice(dev));
  locc_ctx* c = new (std::nothrow) locc_ctx();
  if (!c) return fail(LOCC_E_OOM, "host allocation");
  c->cfg = *cfg;
  c->cfg.device_ids = nullptr;  // not owned (the group keeps its sub-contexts instead)
  c->device = dev;
  c->force_2pass = getenv("LOCC_CROP_2PASS") != nullptr;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) == cudaSuccess) c->num_sms = prop.multiProcessorCount;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);  // lo = least urgent: the encoder's CTAs go first
    e = cudaStreamCreateWithPriority(&c->crop_stream, cudaStreamNonBlocking, lo);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_q0, cudaEventDisableTiming);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&c->ev_crop[i], cudaEventDisableTiming);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming);
  for (int i = 0; i < 64 && e == cudaSuccess; ++i) e = cudaEventCreate(&c->ev_cs[i]);
  for (int i = 0; i < 64 && e == cudaSuccess; ++i) e = cudaEventCreate(&c->ev_ce[i]);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaEventCreate(&c->ev[i]);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&c->ev_free[i], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    locc_destroy(c);
    return fail(LOCC_E_CUDA, "stream/event creation: %s", cudaGetErrorString(e));
  }
  *out = c;
  return LOCC_OK;
}

void locc_destroy(locc_ctx* c) {
  if (!c) return;
  for (locc_ctx* k : c->kids) locc_destroy(k);
  c->kids.clear();
  if (c->nccl_comm && nccl().ok) nccl().CommDestroy(static_cast<ncclComm_t>(c->nccl_comm));
  cudaSetDevice(c->device);
  if (c->grp_ev) cudaEventDestroy(c->grp_ev);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (c->ev_in[i]) cudaEventDestroy(c->ev_in[i]);
    if (c->ev_free[i]) cudaEventDestroy(c->ev_free[i]);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->crop_stream) {
    cudaStreamSynchronize(c->crop_stream);
    cudaStreamDestroy(c->crop_stream);
  }
  if (c->ev_q0) cudaEventDestroy(c->ev_q0);
  for (int i = 0; i < 2; ++i) {
    if (c->ev_crop[i]) cudaEventDestroy(c->ev_crop[i]);
    if (c->ev_done[i]) cudaEventDestroy(c->ev_done[i]);
  }
  for (int i = 0; i < 64; ++i) {
    if (c->ev_cs[i]) cudaEventDestroy(c->ev_cs[i]);
    if (c->ev_ce[i]) cudaEventDestroy(c->ev_ce[i]);
  }
  if (c->sim_exec) cudaGraphExecDestroy(c->sim_exec);
  if (c->q_exec) cudaGraphExecDestroy(c->q_exec);
  for (auto& e : c->enc_ev) cudaEventDestroy(e);
  for (auto& e : c->head_ev) cudaEventDestroy(e);
  for (auto& e : c->crop_ev) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

locc_status locc_set_precision(locc_ctx* c, int32_t precision) {
  if (!c) return fail(LOCC_E_INVALID_ARG, "null context");
  if (precision != LOCC_PREC_FP32 && precision != LOCC_PREC_BF16)
    return fail(LOCC_E_INVALID_ARG, "unknown precision %d", precision);
  if (precision == LOCC_PREC_BF16 && c->cfg.H != 256)
    return fail(LOCC_E_INVALID_ARG, "the tensor-core encoder is built for H = 256");
  if (is_group(c)) {
    locc_status s = fan_out(c, [&](locc_ctx* k) { return locc_set_precision(k, precision); });
    if (s != LOCC_OK) return s;
  }
  c->cfg.precision = precision;
  ++c->generation;
  return LOCC_OK;
}

locc_status locc_set_deterministic(locc_ctx* c, int32_t enabled) {
  if (!c) return fail(LOCC_E_INVALID_ARG, "null context");
  if (c->deterministic != (enabled != 0)) ++c->generation;  // a captured sim graph holds the kernel choice
  c->deterministic = enabled != 0;
  if (is_group(c)) return fan_out(c, [&](locc_ctx* k) { return locc_set_deterministic(k, enabled); });
  return LOCC_OK;
}

locc_status locc_set_timing(locc_ctx* c, int32_t enabled) {
  if (!c) return fail(LOCC_E_INVALID_ARG, "null context");
  c->timing = enabled != 0;
  if (is_group(c)) return fan_out(c, [&](locc_ctx* k) { return locc_set_timing(k, enabled); });
  return LOCC_OK;
}

locc_status locc_get_stats(locc_ctx* c, locc_stats* out) {
  if (!c || !out) return fail(LOCC_E_INVALID_ARG, "null argument");
  if (is_group(c)) {  // counts summed over the devices' shards, times the slowest device's
    locc_stats a{};
    locc_status s = fan_out(c, [&](locc_ctx* k) {
      locc_stats ks{};
      locc_status r = locc_get_stats(k, &ks);
      a.pairs += ks.pairs;
      a.evaluated_pairs += ks.evaluated_pairs;
      a.kept_rows += ks.kept_rows;
      a.nonempty_sides += ks.nonempty_sides;
      a.sub_batches += ks.sub_batches;
      a.kernel_launches += ks.kernel_launches;
      a.encoder_ms = std::max(a.encoder_ms, ks.encoder_ms);
      a.total_ms = std::max(a.total_ms, ks.total_ms);
      a.head_ms = std::max(a.head_ms, ks.head_ms);
      a.crop_ms = std::max(a.crop_ms, ks.crop_ms);
      a.graph_replay += ks.graph_replay;
      return r;
    });
    *out = a;
    return s;
  }
  if (c->last.pairs > 0 && c->last.kept_rows == 0 && c->last.evaluated_pairs == 0) {
    // asynchronous query: read the device counters now
    CK(cudaSetDevice(c->device));
    CK(cudaDeviceSynchronize());
    DevStats hs;
    CK(cudaMemcpy(&hs, c->stats.p, sizeof hs, cudaMemcpyDeviceToHost));
    c->last.kept_rows = (int64_t)hs.kept_rows;
    c->last.nonempty_sides = (int64_t)hs.nonempty_sides;
    c->last.evaluated_pairs = (int64_t)hs.evaluated_pairs;
    locc_status ts = read_timing(c);
    if (ts != LOCC_OK) return ts;
  }
  *out = c->last;
  return LOCC_OK;
}

locc_status locc_load_weights_mem(locc_ctx* c, const float* flat, size_t n) {
  if (!c || !flat) return fail(LOCC_E_INVALID_ARG, "null argument");
  const int64_t want = n_params(c->cfg.H, c->cfg.F);
  if ((int64_t)n != want)
    return fail(LOCC_E_WEIGHTS, "expected %lld floats for H=%d F=%d, got %zu", (long long)want, c->cfg.H, c->cfg.F, n);
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(flat[i])) return fail(LOCC_E_WEIGHTS, "non-finite parameter at %zu", i);
  if (is_group(c)) {
    locc_status s = fan_out(c, [&](locc_ctx* k) { return locc_load_weights_mem(k, flat, n); });
    c->has_weights = s == LOCC_OK;
    c->has_cells = false;
    return s;
  }
  CK(cudaSetDevice(c->device));
  c->has_cells = false;  // the cached grids depend on the encoder weights
  ++c->generation;
  locc_status s = upload_params(c, flat);
  if (s != LOCC_OK) return s;
  if (c->cfg.H == 256) s = locc_upload_tc_weights(c, flat);
  return s;
}

locc_status locc_load_weights(locc_ctx* c, const char* manifest) {
  if (!c || !manifest) return fail(LOCC_E_INVALID_ARG, "null argument");
  std::ifstream f(manifest);
  if (!f) return fail(LOCC_E_WEIGHTS, "cannot open %s", manifest);
  std::string magic;
  int ver = 0, M = 0, H = 0, F = 0;
  f >> magic >> ver >> M >> H >> F;
  if (!f || magic != "locc-weights" || ver != 1) return fail(LOCC_E_WEIGHTS, "%s: bad header", manifest);
  if (M != c->cfg.M || H != c->cfg.H || F != c->cfg.F)
    return fail(LOCC_E_WEIGHTS, "manifest M/H/F = %d/%d/%d, context %d/%d/%d", M, H, F, c->cfg.M, c->cfg.H, c->cfg.F);
  std::string path(manifest), bin = path;
  const size_t dot = path.find_last_of('.'), slash = path.find_last_of('/');
  if (dot != std::string::npos && (slash == std::string::npos || dot > slash)) bin = path.substr(0, dot);
  bin += ".bin";
  std::vector<char> raw;
  if (!read_file(bin, raw)) return fail(LOCC_E_WEIGHTS, "cannot read %s", bin.c_str());
  const char* names[] = {"enc.l1", "enc.l2", "enc.l3", "enc.proj", "obj.l1", "obj.l2",
                         "obj.l3", "pair.l1", "pair.l2", "pair.l3", "out"};
  const int shp[11][2] = {{H, 3}, {H, H}, {H, H}, {F, H}, {kPredW, F + 7}, {kPredW, kPredW},
                          {kPredW, kPredW}, {kPredW, kPredW}, {kPredW, kPredW}, {kPredW, kPredW}, {1, kPredW}};
  std::vector<float> flat;
  flat.reserve(n_params(H, F));
  for (int l = 0; l < 11; ++l)
    for (int wb = 0; wb < 2; ++wb) {
      std::string name;
      long long o = -1, in = -1, off = -1;
      f >> name >> o >> in >> off;
      const std::string want = std::string(names[l]) + (wb ? ".b" : ".W");
      const long long eo = shp[l][0], ei = wb ? 1 : shp[l][1];
      if (!f || name != want || o != eo || in != ei)
        return fail(LOCC_E_WEIGHTS, "%s: expected tensor %s [%lld][%lld], got '%s' [%lld][%lld]", manifest,
                    want.c_str(), eo, ei, name.c_str(), o, in);
      const size_t bytes = (size_t)(o * in) * sizeof(float);
      if (off < 0 || (size_t)off + bytes > raw.size())
        return fail(LOCC_E_WEIGHTS, "%s: tensor %s beyond the end of %s", manifest, want.c_str(), bin.c_str());
      const size_t at = flat.size();
      flat.resize(at + (size_t)(o * in));
      std::memcpy(flat.data() + at, raw.data() + off, bytes);
    }
  return locc_load_weights_mem(c, flat.data(), flat.size());
}

locc_status locc_set_shapes(locc_ctx* c, const float* points, int32_t S, int32_t K) {
  if (!c) return fail(LOCC_E_INVALID_ARG, "null context");
  if (!points) return fail(LOCC_E_INVALID_ARG, "null points");
  if (S < 1 || K < 1 || K > 65535) return fail(LOCC_E_SHAPE, "need S >= 1 and 1 <= K <= 65535 (S=%d K=%d)", S, K);
  const size_t n = (size_t)S * K * 3;
  if (is_group(c)) {  // every device gets its own copy of the table (a device pointer is read back once)
    std::vector<float> host;
    const float* src = points;
    if (is_device_ptr(points)) {
      host.resize(n);
      CK(cudaMemcpy(host.data(), points, n * sizeof(float), cudaMemcpyDeviceToHost));
      src = host.data();
    }
    locc_status s = fan_out(c, [&](locc_ctx* k) { return locc_set_shapes(k, src, S, K); });
    c->has_shapes = s == LOCC_OK;
    c->has_cells = false;
    c->T.S = S;
    c->T.K = K;
    return s;
  }
  CK(cudaSetDevice(c->device));
  DevBuf tmp, cell, bad;
  const float* src = points;
  if (!is_device_ptr(points)) {
    CK(tmp.ensure(n * sizeof(float)));
    CK(cudaMemcpyAsync(tmp.p, points, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    src = tmp.as<float>();
  }
  CK(c->sh_pts.ensure(sizeof(float4) * (size_t)S * K));
  CK(c->sh_perm.ensure(sizeof(uint16_t) * (size_t)S * K));
  CK(c->sh_lo.ensure(sizeof(float4) * S));
  CK(c->sh_hi.ensure(sizeof(float4) * S));
  CK(cell.ensure(sizeof(uint16_t) * (size_t)S * K));
  CK(bad.ensure(sizeof(int)));
  CK(cudaMemsetAsync(bad.p, 0, sizeof(int), c->stream));
  CK(launch_shape_prep(src, S, K, c->cfg.M, c->sh_pts.as<float4>(), c->sh_perm.as<uint16_t>(), c->sh_lo.as<float4>(),
                       c->sh_hi.as<float4>(), cell.as<uint16_t>(), bad.as<int>(), c->stream));
  int hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (hbad) {
    c->has_shapes = false;
    return fail(LOCC_E_SHAPE, "non-finite point coordinate");
  }
  c->T.pts = c->sh_pts.as<float4>();
  c->T.perm = c->sh_perm.as<uint16_t>();
  c->T.lo = c->sh_lo.as<float4>();
  c->T.hi = c->sh_hi.as<float4>();
  c->T.S = S;
  c->has_cells = false;  // the cached grids belong to the previous shape table
  ++c->generation;
  if (c->T.K != K) c->cap_B = c->cap_B2 = 0;  // row buffers depend on K
  c->T.K = K;
  c->has_shapes = true;
  return LOCC_OK;
}

// An asynchronous query of device buffers that fits one sub-batch runs from a CUDA graph: the first
// call with a given key runs directly (allocating any scratch), the second is captured, later ones
// replay it.  The key holds every argument and the context's generation (weights, shapes, grids,
// precision, determinism) and allocation epoch (no scratch buffer the graph points into was
// reallocated); anything else — host buffers, the synchronous form, timing, LOCC_NO_GRAPH=1 — runs
// directly.
extern "C++" {
template <class Run>
locc_status graphed_query(locc_ctx* c, int32_t kind, const int32_t* pairs, const float* poses, int64_t N,
                          const float* probs, const void* labels, const float* logits, const void* extra,
                          void* stream, Run&& run) {
  const bool eligible = c && stream && N > 0 && pairs && poses && probs && c->has_weights && c->has_shapes &&
                        !c->timing && N <= batch_cap(c) && is_device_ptr(pairs) && !getenv("LOCC_NO_GRAPH") &&
                        !getenv("LOCC_TC_TRACE");
  if (!eligible) return run();
  locc_ctx::QueryKey key;
  std::memset(&key, 0, sizeof key);
  key.kind = kind;
  key.precision = c->cfg.precision;
  key.det = c->deterministic;
  key.N = N;
  key.pairs = pairs;
  key.poses = poses;
  key.probs = probs;
  key.labels = labels;
  key.logits = logits;
  key.extra = extra;
  key.stream = stream;
  key.gen = c->generation;
  key.alloc_epoch = g_alloc_epoch.load();
  if (std::memcmp(&key, &c->q_key, sizeof key) != 0) {
    if (c->q_exec) cudaGraphExecDestroy(c->q_exec);
    c->q_exec = nullptr;
    c->q_key = key;
    c->q_seen = 0;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (c->q_exec) {
    CK(cudaSetDevice(c->device));
    CK(cudaGraphLaunch(c->q_exec, st));
    c->last = c->q_last;
    c->last.graph_replay = 1;
    return LOCC_OK;
  }
  if (c->q_seen < 1) {
    locc_status s = run();
    if (s == LOCC_OK) ++c->q_seen;
    c->q_key.alloc_epoch = g_alloc_epoch.load();  // what this direct call allocated is what a capture uses
    return s;
  }
  CK(cudaSetDevice(c->device));
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  const locc_status s = run();
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(st, &graph);
  if (s == LOCC_OK && ec == cudaSuccess && graph && cudaGraphInstantiate(&c->q_exec, graph, 0) != cudaSuccess)
    c->q_exec = nullptr;
  if (graph) cudaGraphDestroy(graph);
  cudaGetLastError();
  if (!c->q_exec || s != LOCC_OK) {  // not capturable: this key stays on the direct path
    c->q_seen = -(1 << 30);
    return run();
  }
  c->q_last = c->last;
  CK(cudaGraphLaunch(c->q_exec, st));
  c->last.graph_replay = 1;
  return LOCC_OK;
}
}  // extern "C++"

locc_status locc_query(locc_ctx* c, const int32_t* pairs, const float* poses, int64_t N, float* probs,
                       uint8_t* labels, float* logits, void* stream) {
  if (is_group(c))
    return group_query(c, pairs, poses, N, probs, labels, logits, nullptr, nullptr, nullptr, nullptr, nullptr, stream,
                       false);
  return graphed_query(c, 0, pairs, poses, N, probs, labels, logits, nullptr, stream, [&] {
    return run_query(c, pairs, poses, N, probs, labels, logits, nullptr, nullptr, nullptr, nullptr, nullptr, stream);
  });
}

locc_status locc_query_debug(locc_ctx* c, const int32_t* pairs, const float* poses, int64_t N, float* probs,
                             uint8_t* labels, float* logits, int32_t* kept, int32_t* occ, uint32_t* masks,
                             float* emb, void* stream) {
  if (is_group(c))
    return group_query(c, pairs, poses, N, probs, labels, logits, kept, occ, masks, emb, nullptr, stream, false);
  return run_query(c, pairs, poses, N, probs, labels, logits, kept, occ, masks, emb, nullptr, stream);
}

locc_status locc_query_grad(locc_ctx* c, const int32_t* pairs, const float* poses, int64_t N, float* probs,
                            uint8_t* labels, float* logits, float* grad, void* stream) {
  if (N > 0 && !grad) return fail(LOCC_E_INVALID_ARG, "grad must be non-null");
  if (is_group(c))
    return group_query(c, pairs, poses, N, probs, labels, logits, nullptr, nullptr, nullptr, nullptr, grad, stream, false);
  return graphed_query(c, 1, pairs, poses, N, probs, labels, logits, grad, stream, [&] {
    return run_query(c, pairs, poses, N, probs, labels, logits, nullptr, nullptr, nullptr, nullptr, grad, stream);
  });
}

// ---------------------------------------------------------------- NEXT-1: encode-once mode
int64_t locc_unet_n_params(int32_t H, int32_t F) {
  const int64_t C = 128;
  return C * 27 * (H + 3 * C + C + 3 * 2 * C) + 8 * C + (int64_t)F * 2 * C + F;
}

locc_status locc_load_unet_weights_mem(locc_ctx* c, const float* flat, size_t n) {
  if (!c || !flat) return fail(LOCC_E_INVALID_ARG, "null argument");
  const int H = c->cfg.H, F = c->cfg.F, C = 128;
  const int64_t want = locc_unet_n_params(H, F);
  if ((int64_t)n != want)
    return fail(LOCC_E_WEIGHTS, "expected %lld U-Net floats for H=%d F=%d, got %zu", (long long)want, H, F, n);
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(flat[i])) return fail(LOCC_E_WEIGHTS, "non-finite U-Net parameter at %zu", i);
  if (is_group(c)) {
    locc_status s = fan_out(c, [&](locc_ctx* k) { return locc_load_unet_weights_mem(k, flat, n); });
    c->has_unet = s == LOCC_OK;
    c->has_cells = false;
    return s;
  }
  CK(cudaSetDevice(c->device));
  // Wt[l][k][i][o] = W[o][i][k] for the convs; the deconvs as the equivalent conv: taps flipped (26 - k)
  const int cin[8] = {H, C, C, C, C, 2 * C, 2 * C, 2 * C};
  std::vector<float> img;
  size_t offW[8], offb[8];
  const float* q = flat;
  for (int l = 0; l < 8; ++l) {
    offW[l] = img.size();
    img.resize(img.size() + (size_t)27 * cin[l] * C);
    float* wt = img.data() + offW[l];
    for (int o = 0; o < C; ++o)
      for (int i = 0; i < cin[l]; ++i)
        for (int k = 0; k < 27; ++k) {
          const int kk = l < 4 ? k : 26 - k;
          wt[((size_t)kk * cin[l] + i) * C + o] = q[((size_t)o * cin[l] + i) * 27 + k];
        }
    q += (size_t)C * cin[l] * 27;
    offb[l] = img.size();
    img.insert(img.end(), q, q + C);
    q += C;
  }
  // tensor-core images of the 8 layers: chunk (tap k, channel block cb) = [128 out x 32 in], tf32 hi then
  // lo, SW128 K-major — from the conv-form Wt[k][i][o] above (deconv taps already flipped)
  std::vector<uint8_t> timg;
  size_t offT[8];
  for (int l = 0; l < 8; ++l) {
    offT[l] = timg.size();
    const float* wt = img.data() + offW[l];
    for (int k = 0; k < 27; ++k)
      for (int cb = 0; cb < cin[l] / 32; ++cb) {
        const size_t base = timg.size();
        timg.resize(base + 32768, 0);
        for (int o = 0; o < C; ++o)
          for (int kk = 0; kk < 32; ++kk) {
            const float w = wt[((size_t)k * cin[l] + 32 * cb + kk) * C + o];
            const float hi = tf32_rna_host(w), lo = tf32_rna_host(w - hi);
            const size_t off = tc::sw128_off((uint32_t)o, (uint32_t)(kk >> 2)) + (size_t)(kk & 3) * 4;
            std::memcpy(&timg[base + off], &hi, 4);
            std::memcpy(&timg[base + 16384 + off], &lo, 4);
          }
      }
  }
  const size_t offP = img.size();
  img.insert(img.end(), q, q + (size_t)F * 2 * C);
  q += (size_t)F * 2 * C;
  const size_t offPb = img.size();
  img.insert(img.end(), q, q + F);
  CK(c->unet_params.ensure(sizeof(float) * img.size()));
  CK(cudaMemcpy(c->unet_params.p, img.data(), sizeof(float) * img.size(), cudaMemcpyHostToDevice));
  const float* d = c->unet_params.as<float>();
  for (int l = 0; l < 8; ++l) {
    c->U.Wt[l] = d + offW[l];
    c->U.b[l] = d + offb[l];
  }
  CK(c->unet_img.ensure(timg.size()));
  CK(cudaMemcpy(c->unet_img.p, timg.data(), timg.size(), cudaMemcpyHostToDevice));
  for (int l = 0; l < 8; ++l) c->U.img[l] = c->unet_img.as<uint8_t>() + offT[l];
  c->U.pW = d + offP;
  c->U.pb = d + offPb;
  c->has_unet = true;
  c->has_cells = false;
  ++c->generation;
  return LOCC_OK;
}

locc_status locc_set_unet_global_pool(locc_ctx* c, int32_t mode) {
  if (!c) return fail(LOCC_E_INVALID_ARG, "null context");
  if (mode != 0 && mode != 1) return fail(LOCC_E_INVALID_ARG, "global pool mode must be 0 (average) or 1 (max)");
  if (is_group(c)) {
    locc_status s = fan_out(c, [&](locc_ctx* k) { return locc_set_unet_global_pool(k, mode); });
    if (s == LOCC_OK && c->unet_global_max != mode) c->has_cells = false;
    c->unet_global_max = mode;
    return s;
  }
  if (c->unet_global_max != mode) {
    c->unet_global_max = mode;
    c->has_cells = false;  // the grids must be re-encoded
    ++c->generation;
  }
  return LOCC_OK;
}

locc_status locc_encode_shapes(locc_ctx* c) {
  if (!c) return fail(LOCC_E_INVALID_ARG, "null context");
  if (is_group(c)) {  // every device encodes its own copy of the table, concurrently
    std::vector<std::thread> th;
    std::vector<locc_status> st(c->kids.size(), LOCC_OK);
    std::vector<std::string> msg(c->kids.size());
    for (size_t i = 0; i < c->kids.size(); ++i)
      th.emplace_back([&, i] {
        st[i] = locc_encode_shapes(c->kids[i]);
        if (st[i] != LOCC_OK) msg[i] = g_err;
      });
    for (auto& t : th) t.join();
    double ms = 0.0;
    for (size_t i = 0; i < c->kids.size(); ++i) {
      if (st[i] != LOCC_OK) {
        g_err = msg[i];
        return st[i];
      }
      ms = std::max(ms, c->kids[i]->encode_ms);
    }
    c->encode_ms = ms;
    c->has_cells = true;
    return LOCC_OK;
  }
  if (!c->has_weights || !c->has_shapes || !c->has_unet)
    return fail(LOCC_E_STATE, "weights, U-Net weights and shapes must be set before locc_encode_shapes");
  const int M = c->cfg.M, H = c->cfg.H, F = c->cfg.F, S = c->T.S;
  if (M < 3 || M > 8 || H % 32 || F > 64)
    return fail(LOCC_E_INVALID_ARG, "encode-once mode is built for 3 <= M <= 8, H a multiple of 32, F <= 64");
  CK(cudaSetDevice(c->device));
  const int nc = M * M * M;
  DevBuf G, act;
  CK(G.ensure(sizeof(float) * (size_t)S * nc * H));
  CK(act.ensure(sizeof(float) * unet_act_floats(S, M)));
  CK(c->cells_E.ensure(sizeof(float) * (size_t)S * nc * F));
  CK(c->cells_ctr.ensure(sizeof(float) * (size_t)S * 24));
  // the grid encode's layers 2-3 and the U-Net on the tensor cores (3xTF32) in bf16 contexts, on CUDA
  // cores (fp32) in fp32 ones
  const bool bf16 = c->cfg.precision == LOCC_PREC_BF16;
  const bool grid_tc = bf16 && c->P.grid_tc_img && !getenv("LOCC_GRID_FFMA");
  DevBuf bufA, bufB;  // the tensor-core grid encode's activations (allocated outside the timed region)
  if (grid_tc) {
    const size_t nb = sizeof(float) * 256 * (size_t)grid_tc_chunk_rows(c->T);
    CK(bufA.ensure(nb));
    CK(bufB.ensure(nb));
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, c->stream));
  if (grid_tc) {
    CK(launch_grid_encode_tc(c->P, c->T, M, G.as<float>(), bufA.as<float>(), bufB.as<float>(), c->num_sms,
                             c->stream));
  } else {
    CK(launch_grid_encode(c->P, c->T, M, G.as<float>(), c->stream));
  }
  const bool tc = bf16 && !getenv("LOCC_CONV_FFMA");
  CK(launch_unet(c->U, c->T, M, H, F, c->unet_global_max, G.as<float>(), act.as<float>(), c->cells_E.as<float>(),
                 c->cells_ctr.as<float>(), tc, c->num_sms, c->stream));
  CK(cudaEventRecord(e1, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  c->encode_ms = ms;
  ++c->generation;
  c->cells.E = c->cells_E.as<float>();
  c->cells.ctr = c->cells_ctr.as<float>();
  c->cells.M = M;
  c->has_cells = true;
  return LOCC_OK;
}

locc_status locc_get_cell_embeddings(locc_ctx* c, float* out, double* encode_ms) {
  if (!c) return fail(LOCC_E_INVALID_ARG, "null context");
  if (is_group(c)) {  // every device holds the same grids: read the first one's
    locc_status s = locc_get_cell_embeddings(c->kids[0], out, nullptr);
    if (s == LOCC_OK && encode_ms) *encode_ms = c->encode_ms;
    return s;
  }
  if (!c->has_cells) return fail(LOCC_E_STATE, "no encoded shapes");
  CK(cudaSetDevice(c->device));
  if (out) {
    const size_t bytes = sizeof(float) * (size_t)c->T.S * c->cfg.M * c->cfg.M * c->cfg.M * c->cfg.F;
    CK(cudaMemcpy(out, c->cells_E.p, bytes, is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
  }
  if (encode_ms) *encode_ms = c->encode_ms;
  return LOCC_OK;
}

locc_status locc_query_cells(locc_ctx* c, const int32_t* pairs, const float* poses, int64_t N, float* probs,
                             uint8_t* labels, float* logits, int32_t* nsel, uint32_t* cells, float* emb,
                             void* stream) {
  if (is_group(c))
    return group_query(c, pairs, poses, N, probs, labels, logits, nsel, nullptr, cells, emb, nullptr, stream, true);
  if (nsel || cells || emb)  // debug outputs: direct
    return run_query(c, pairs, poses, N, probs, labels, logits, nsel, nullptr, cells, emb, nullptr, stream, true);
  return graphed_query(c, 2, pairs, poses, N, probs, labels, logits, nullptr, stream, [&] {
    return run_query(c, pairs, poses, N, probs, labels, logits, nullptr, nullptr, nullptr, nullptr, nullptr, stream,
                     true);
  });
}

// ---------------------------------------------------------------- NEXT-3: closed-loop substeps
locc_status locc_sim_run(locc_ctx* c, const locc_sim_config* cfg, int32_t E, const int32_t* ids, const float* body,
                         float* state, double t0, int32_t* contacts, void* stream) {
  if (!c || !cfg) return fail(LOCC_E_INVALID_ARG, "null argument");
  if (E < 0 || cfg->substeps < 1 || !(cfg->h > 0.0)) return fail(LOCC_E_INVALID_ARG, "need E >= 0, substeps >= 1, h > 0");
  if (cfg->detector != 0 && cfg->detector != 1) return fail(LOCC_E_INVALID_ARG, "detector must be 0 or 1");
  if (!c->has_weights || !c->has_shapes) return fail(LOCC_E_STATE, "weights and shapes must be set");
  if (cfg->detector == 1 && !c->has_cells) return fail(LOCC_E_STATE, "detector 1 needs locc_encode_shapes");
  if (c->cfg.H != 256 || c->cfg.F != 64) return fail(LOCC_E_INVALID_ARG, "the pose gradient is built for H = 256, F = 64");
  if (E == 0) return LOCC_OK;
  if (!ids || !body || !state) return fail(LOCC_E_INVALID_ARG, "ids, body and state must be non-null");
  if (is_group(c)) {  // environments sharded over the devices (each env's bodies stay together)
    const int hd = pointer_device(state);
    if (hd != c->device || pointer_device(ids) != hd || pointer_device(body) != hd ||
        (contacts && pointer_device(contacts) != hd))
      return fail(LOCC_E_INVALID_ARG, "locc_sim_run takes device buffers on the home device %d", c->device);
    const Slice sl[] = {{ids, 12, true, false}, {body, 48, true, false}, {state, 156, true, true},
                        {contacts, 12, false, true}};
    // contacts are zeroed with a memset on the kid's stream: then the kid works on its own copies
    return group_run(
        c, E, sl, 4, true, stream, contacts == nullptr,
        [&](locc_ctx* k, void** p, int64_t n, void* st) {
          return locc_sim_run(k, cfg, (int32_t)n, (const int32_t*)p[0], (const float*)p[1], (float*)p[2], t0,
                              (int32_t*)p[3], st);
        },
        kid_sim_check);
  }
  if (!is_device_ptr(ids) || !is_device_ptr(body) || !is_device_ptr(state) || (contacts && !is_device_ptr(contacts)))
    return fail(LOCC_E_INVALID_ARG, "locc_sim_run takes device buffers");
  CK(cudaSetDevice(c->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  const int64_t NP = 3 * (int64_t)E;
  if (NP > c->sim_cap) {
    CK(c->sim_pairs.ensure(sizeof(int32_t) * 2 * NP));
    CK(c->sim_poses.ensure(sizeof(float) * 14 * NP));
    CK(c->sim_probs.ensure(sizeof(float) * NP));
    CK(c->sim_logits.ensure(sizeof(float) * NP));
    CK(c->sim_grad.ensure(sizeof(float) * 14 * NP));
    CK(c->sim_culled.ensure(NP));
    c->sim_cap = NP;
  }
  SimParams sp{};
  sp.h = (float)cfg->h;
  for (int i = 0; i < 3; ++i) {
    sp.g[i] = cfg->gravity[i];
    sp.amp[i] = cfg->amp[i];
  }
  sp.ks = cfg->ks;
  sp.kd = cfg->kd;
  sp.freq = cfg->freq;
  sp.slack = cfg->slack;
  sp.hd = cfg->h;
  CK(c->sim_t0.ensure(sizeof(double)));
  CK(c->sim_bad.ensure(sizeof(unsigned long long)));
  double* t0_dev = c->sim_t0.as<double>();
  unsigned long long* bad = c->sim_bad.as<unsigned long long>();
  CK(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st));
  CK(launch_sim_set_t0(t0_dev, t0, st));
  // the substeps: enqueued directly, or captured once into a CUDA graph and replayed while the call's
  // inputs (sizes, constants, buffers, stream) and the context's state are unchanged — one launch
  // instead of ~10 per substep (LOCC_NO_GRAPH=1 disables it)
  auto enqueue = [&](int64_t& launches) -> locc_status {
    if (contacts) CK(cudaMemsetAsync(contacts, 0, sizeof(int32_t) * NP, st));
    for (int n = 0; n < cfg->substeps; ++n) {
      CK(launch_sim_prepare(c->T, sp, E, ids, state, t0_dev, n, c->sim_pairs.as<int32_t>(), c->sim_poses.as<float>(),
                            c->sim_culled.as<uint8_t>(), bad, st));
      locc_status s = run_query(c, c->sim_pairs.as<int32_t>(), c->sim_poses.as<float>(), NP,
                                c->sim_probs.as<float>(), nullptr, c->sim_logits.as<float>(), nullptr, nullptr,
                                nullptr, nullptr, c->sim_grad.as<float>(), st, cfg->detector == 1);
      if (s != LOCC_OK) return s;
      launches += c->last.kernel_launches + 2;
      CK(launch_sim_integrate(sp, E, body, state, c->sim_logits.as<float>(), c->sim_grad.as<float>(),
                              c->sim_culled.as<uint8_t>(), contacts, t0_dev, n, st));
    }
    return LOCC_OK;
  };
  locc_ctx::SimKey key{};
  key.cfg = *cfg;
  key.E = E;
  key.ids = ids;
  key.body = body;
  key.state = state;
  key.contacts = contacts;
  key.stream = st;
  key.gen = c->generation;
  key.alloc_epoch = g_alloc_epoch.load();
  const bool same = std::memcmp(&key, &c->sim_key, sizeof key) == 0;
  if (!same) {
    if (c->sim_exec) cudaGraphExecDestroy(c->sim_exec);
    c->sim_exec = nullptr;
    c->sim_key = key;
    c->sim_seen = 0;
  }
  int64_t launches = 0;
  const bool graphs = !getenv("LOCC_NO_GRAPH") && !c->timing;
  if (graphs && !c->sim_exec && c->sim_seen >= 1) {
    // capture (the first call with this key has already run directly: all scratch is allocated)
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    locc_status s = enqueue(launches);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(st, &graph);
    if (s == LOCC_OK && ec == cudaSuccess && graph) {
      if (cudaGraphInstantiate(&c->sim_exec, graph, 0) != cudaSuccess) c->sim_exec = nullptr;
    }
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    if (!c->sim_exec) {  // capture not possible: stay on the direct path for this key
      c->sim_seen = -1 << 30;
      launches = 0;
      locc_status s2 = enqueue(launches);
      if (s2 != LOCC_OK) return s2;
    } else {
      CK(cudaGraphLaunch(c->sim_exec, st));
      c->sim_launches = launches;
    }
  } else if (graphs && c->sim_exec) {
    CK(cudaGraphLaunch(c->sim_exec, st));
    launches = c->sim_launches;
  } else {
    locc_status s = enqueue(launches);
    if (s != LOCC_OK) return s;
  }
  ++c->sim_seen;
  c->sim_key.alloc_epoch = g_alloc_epoch.load();  // the scratch this call allocated is what a capture uses
  c->last.kernel_launches = launches;
  if (!stream) {
    // synchronous form: report environments whose body ids were out of range (their pairs were culled)
    unsigned long long hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hbad) return fail(LOCC_E_INVALID_ARG, "%llu environment substeps had a body id outside [0, S)", hbad);
  }
  return LOCC_OK;
}

// ---------------------------------------------------------------- multi-process NCCL gather
locc_status locc_comm_unique_id(uint8_t out[128]) {
  if (!out) return fail(LOCC_E_INVALID_ARG, "null argument");
  const NcclApi& A = nccl();
  if (!A.ok) return fail(LOCC_E_NCCL, "%s", A.why.c_str());
  ncclUniqueId id;
  NK(A.GetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, 128);
  return LOCC_OK;
}

locc_status locc_comm_init(locc_ctx* c, int32_t world, int32_t rank, const uint8_t id[128]) {
  if (!c || !id) return fail(LOCC_E_INVALID_ARG, "null argument");
  if (is_group(c)) return fail(LOCC_E_INVALID_ARG, "locc_comm_init takes a single-device context (one per rank)");
  if (world < 1 || rank < 0 || rank >= world) return fail(LOCC_E_INVALID_ARG, "rank %d of world %d", rank, world);
  const NcclApi& A = nccl();
  if (!A.ok) return fail(LOCC_E_NCCL, "%s", A.why.c_str());
  CK(cudaSetDevice(c->device));
  if (c->nccl_comm) {
    A.CommDestroy(static_cast<ncclComm_t>(c->nccl_comm));
    c->nccl_comm = nullptr;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  ncclComm_t comm = nullptr;
  NK(A.CommInitRank(&comm, world, uid, rank));
  c->nccl_comm = comm;
  c->world = world;
  c->rank = rank;
  return LOCC_OK;
}

locc_status locc_query_allgather(locc_ctx* c, const int32_t* pairs, const float* poses, int64_t N, float* probs,
                                 uint8_t* labels, float* logits, void* stream) {
  if (!c) return fail(LOCC_E_INVALID_ARG, "null context");
  if (!c->nccl_comm) return fail(LOCC_E_STATE, "locc_comm_init first");
  if (N < 0) return fail(LOCC_E_INVALID_ARG, "N < 0");
  if (N == 0) return LOCC_OK;
  if (!pairs || !poses || !probs) return fail(LOCC_E_INVALID_ARG, "pairs, poses and probs must be non-null");
  const int64_t per = (N + c->world - 1) / c->world;
  const int64_t lo = std::min<int64_t>(N, c->rank * per), n = std::min<int64_t>(N, lo + per) - lo;
  const bool dev = is_device_ptr(probs);
  CK(cudaSetDevice(c->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  if (dev) {
    if (n > 0) {  // this rank's shard, asynchronously on st (input errors are reported below if synchronous)
      locc_status s = run_query(c, pairs + 2 * lo, poses + 14 * lo, n, probs + lo, labels ? labels + lo : nullptr,
                                logits ? logits + lo : nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, st);
      if (s != LOCC_OK) return s;
    }
    locc_status s = allgather_slices(c, N, probs, labels, logits, st);
    if (s != LOCC_OK) return s;
    if (!stream) {
      CK(cudaStreamSynchronize(st));
      if (n > 0) return kid_query_check(c);
    }
    return LOCC_OK;
  }
  // host buffers: the shard runs synchronously from host memory, then the slices meet in device
  // staging buffers for the collective and the whole result is copied back
  CK(c->ag_out[0].ensure(sizeof(float) * N));
  if (labels) CK(c->ag_out[1].ensure(N));
  if (logits) CK(c->ag_out[2].ensure(sizeof(float) * N));
  float* dp = c->ag_out[0].as<float>();
  uint8_t* dl = labels ? c->ag_out[1].as<uint8_t>() : nullptr;
  float* dg = logits ? c->ag_out[2].as<float>() : nullptr;
  if (n > 0) {
    locc_status s = run_query(c, pairs + 2 * lo, poses + 14 * lo, n, probs + lo, labels ? labels + lo : nullptr,
                              logits ? logits + lo : nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    if (s != LOCC_OK) return s;
    CK(cudaMemcpyAsync(dp + lo, probs + lo, sizeof(float) * n, cudaMemcpyHostToDevice, st));
    if (dl) CK(cudaMemcpyAsync(dl + lo, labels + lo, n, cudaMemcpyHostToDevice, st));
    if (dg) CK(cudaMemcpyAsync(dg + lo, logits + lo, sizeof(float) * n, cudaMemcpyHostToDevice, st));
  }
  locc_status s = allgather_slices(c, N, dp, dl, dg, st);
  if (s != LOCC_OK) return s;
  CK(cudaMemcpyAsync(probs, dp, sizeof(float) * N, cudaMemcpyDeviceToHost, st));
  if (dl) CK(cudaMemcpyAsync(labels, dl, N, cudaMemcpyDeviceToHost, st));
  if (dg) CK(cudaMemcpyAsync(logits, dg, sizeof(float) * N, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return LOCC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- tensor-core weight image
namespace {
uint16_t bf16_rne(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
float bf16_to_float(uint16_t h) {
  const uint32_t u = (uint32_t)h << 16;
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}
// b = hi + mid + lo exactly (three bf16 terms of 8 significant bits each cover fp32's 24), stored at
// dst[0..5] (K = k0, k0 + 1, k0 + 2 of an SW128 row chunk).
void put_bias3(uint8_t* dst, float b) {
  const uint16_t hi = bf16_rne(b);
  const float r1 = b - bf16_to_float(hi);
  const uint16_t mid = bf16_rne(r1);
  const uint16_t lo = bf16_rne(r1 - bf16_to_float(mid));
  std::memcpy(dst + 0, &hi, 2);
  std::memcpy(dst + 2, &mid, 2);
  std::memcpy(dst + 4, &lo, 2);
}
}  // namespace

// W2 as the B operand of layer 2, computed as two N = 128 halves: per CTA rank r the 64 output
// features [64r, 64r+64) of half 0 (image rows 0-63) and [128+64r, +64) of half 1 (rows 64-127),
// K-major, 4 K blocks of [128 rows x 128 B] with the 128-byte swizzle (16-byte chunk j of row i stored at
// chunk j ^ (i & 7)) — the exact shared-memory image, so one bulk copy places it.  A fifth block
// holds b2 as the K = 0..2 entries (b2 = hi + mid + lo, each bf16, exact), which the kernel
// multiplies with a column of ones so that the first layer-2 MMA initialises D2 with the bias.
// W3 as the TMEM A operand of layer 3: row f = 128 columns of bf16x2 (K = 2c low, 2c+1 high).
// Also keeps layer 1 (w, b) and b2 for the kernel-parameter block.
constexpr size_t kTcW2Bytes = 5 * 16384;  // per CTA rank
locc_status locc_upload_tc_weights(locc_ctx* c, const float* flat) {
  const int H = 256;
  const float* w1 = flat;
  const float* b1 = w1 + 3 * H;
  const float* w2 = b1 + H;
  const float* b2 = w2 + H * H;
  const float* w3 = b2 + H;
  const float* b3 = w3 + H * H;
  for (int f = 0; f < H; ++f) {
    c->tc_l1.w1b[f] = make_float4(w1[3 * f], w1[3 * f + 1], w1[3 * f + 2], b1[f]);
    c->tc_l1.b2[f] = b2[f];
  }
  std::vector<uint8_t> img(2 * kTcW2Bytes + (size_t)H * 128 * 4, 0);
  for (int r = 0; r < 2; ++r)
    for (int i = 0; i < 128; ++i) {
      // image row i: layer-2 half i / 64 (features 0-127 or 128-255), of which CTA r supplies 64 rows
      const int n = 128 * (i >> 6) + 64 * r + (i & 63);
      for (int kb = 0; kb < 4; ++kb)
        for (int j = 0; j < 8; ++j) {
          uint8_t* dst = img.data() + r * kTcW2Bytes + kb * 16384 + locc::tc::sw128_off(i, j);
          for (int e = 0; e < 8; ++e) {
            const uint16_t v = bf16_rne(w2[(size_t)n * H + 64 * kb + 8 * j + e]);
            std::memcpy(dst + 2 * e, &v, 2);
          }
        }
      // bias block: K = 0..2 of row i = b2 of image row i's feature n (B of layer 2's bias MMA),
      // K = 16..18 of row i = b3 of this CTA's feature 128 r + i (A of layer 3's bias MMA)
      put_bias3(img.data() + r * kTcW2Bytes + 4 * 16384 + locc::tc::sw128_off(i, 0), b2[n]);
      put_bias3(img.data() + r * kTcW2Bytes + 4 * 16384 + locc::tc::sw128_off(i, 2), b3[128 * r + i]);
    }
  uint32_t* w3img = reinterpret_cast<uint32_t*>(img.data() + 2 * kTcW2Bytes);
  for (int f = 0; f < H; ++f)
    for (int cc = 0; cc < 128; ++cc)
      w3img[(size_t)f * 128 + cc] =
          (uint32_t)bf16_rne(w3[(size_t)f * H + 2 * cc]) | ((uint32_t)bf16_rne(w3[(size_t)f * H + 2 * cc + 1]) << 16);
  CK(c->tc_img.ensure(img.size()));
  CK(cudaMemcpy(c->tc_img.p, img.data(), img.size(), cudaMemcpyHostToDevice));
  c->P.tc_w2 = c->tc_img.p;
  c->P.tc_w3 = static_cast<uint8_t*>(c->tc_img.p) + 2 * kTcW2Bytes;
  return LOCC_OK;
}
