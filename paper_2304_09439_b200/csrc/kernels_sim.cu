// kernels_sim.cu — NEXT-3: a Brax-style closed-loop substep with LOCC as the contact detector
// (reading Q31).  Per environment: body 0 =
// the kinematic (shaken) bowl, bodies 1, 2 dynamic; pairs (0,1), (0,2), (1,2).  State per body (13 floats):
// q, t, v, w (world frame).  One substep = sim_prepare_kernel (bowl pose, broad phase, the detector's
// pair/pose lists) -> the LOCC query with the pose gradient (crop or encode-once) -> sim_integrate_kernel
// (penalty along the descent of the logit, semi-implicit Euler).  One thread per environment: the
// per-environment work is a few hundred flops next to the query's ~0.5 MFLOP per pair.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"

namespace locc {
namespace {

__device__ __forceinline__ void rot_of(const float* q, float R[9]) {
  const float n = sqrtf(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
  const float w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
  R[0] = 1.f - 2.f * (y * y + z * z);
  R[1] = 2.f * (x * y - w * z);
  R[2] = 2.f * (x * z + w * y);
  R[3] = 2.f * (x * y + w * z);
  R[4] = 1.f - 2.f * (x * x + z * z);
  R[5] = 2.f * (y * z - w * x);
  R[6] = 2.f * (x * z - w * y);
  R[7] = 2.f * (y * z + w * x);
  R[8] = 1.f - 2.f * (x * x + y * y);
}

// (a) (x) (b), Hamilton product
__device__ __forceinline__ void qmulf(const float a[4], const float b[4], float r[4]) {
  r[0] = a[0] * b[0] - ((a[1] * b[1] + a[2] * b[2]) + a[3] * b[3]);
  r[1] = (a[0] * b[1] + b[0] * a[1]) + (a[2] * b[3] - a[3] * b[2]);
  r[2] = (a[0] * b[2] + b[0] * a[2]) + (a[3] * b[1] - a[1] * b[3]);
  r[3] = (a[0] * b[3] + b[0] * a[3]) + (a[1] * b[2] - a[2] * b[1]);
}

__device__ __forceinline__ void set_bowl(const SimParams& sp, float* b, double tau) {
  const double w2 = 2.0 * 3.14159265358979323846 * (double)sp.freq;
  const double sn = sin(w2 * tau), cs = cos(w2 * tau);
  for (int i = 0; i < 3; ++i) {
    b[4 + i] = (float)((double)sp.amp[i] * sn);
    b[7 + i] = (float)((double)sp.amp[i] * w2 * cs);
    b[10 + i] = 0.f;
  }
}

__constant__ int kPairA[3] = {0, 0, 1};
__constant__ int kPairB[3] = {1, 2, 2};

// The substep's time is read from the device (t0 + n h), so a captured CUDA graph of the substeps can
// be replayed for any start time t0 (set by sim_set_t0_kernel before the replay).
__global__ void sim_set_t0_kernel(double* t0_dev, double t0) { *t0_dev = t0; }

__global__ void __launch_bounds__(128) sim_prepare_kernel(ShapeTable T, SimParams sp, int E,
                                                          const int32_t* __restrict__ ids, float* __restrict__ state,
                                                          const double* __restrict__ t0_dev, int n,
                                                          int32_t* __restrict__ pairs,
                                                          float* __restrict__ poses, uint8_t* __restrict__ culled,
                                                          unsigned long long* __restrict__ bad) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const double tau = *t0_dev + n * sp.hd;
  float* st = state + (int64_t)e * 39;
  set_bowl(sp, st, tau);
  // a body id outside the shape table: count it and cull the environment's pairs (the query then only
  // sees in-range ids; locc_sim_run reports the count in its synchronous form)
  bool ok = true;
  for (int b = 0; b < 3; ++b) ok &= (unsigned)ids[3 * e + b] < (unsigned)T.S;
  if (!ok) {
    atomicAdd(bad, 1ull);
    for (int p = 0; p < 3; ++p) {
      const int64_t i = 3 * (int64_t)e + p;
      pairs[2 * i] = pairs[2 * i + 1] = 0;
      for (int j = 0; j < 14; ++j) poses[14 * i + j] = (j % 7) == 0 ? 1.f : 0.f;
      culled[i] = 1;
    }
    return;
  }
  float cw[3][3], hw[3][3];
  for (int b = 0; b < 3; ++b) {  // world AABB of every body: centre R c + t, half-extent |R| e
    const int sid = ids[3 * e + b];
    const float4 lo = T.lo[sid], hi = T.hi[sid];
    const float cl[3] = {0.5f * (lo.x + hi.x), 0.5f * (lo.y + hi.y), 0.5f * (lo.z + hi.z)};
    const float hl[3] = {0.5f * (hi.x - lo.x), 0.5f * (hi.y - lo.y), 0.5f * (hi.z - lo.z)};
    float R[9];
    rot_of(st + 13 * b, R);
    for (int r = 0; r < 3; ++r) {
      cw[b][r] = st[13 * b + 4 + r] + (R[3 * r] * cl[0] + R[3 * r + 1] * cl[1] + R[3 * r + 2] * cl[2]);
      hw[b][r] = fabsf(R[3 * r]) * hl[0] + fabsf(R[3 * r + 1]) * hl[1] + fabsf(R[3 * r + 2]) * hl[2];
    }
  }
  for (int p = 0; p < 3; ++p) {
    const int64_t i = 3 * (int64_t)e + p;
    const int a = kPairA[p], c = kPairB[p];
    pairs[2 * i] = ids[3 * e + a];
    pairs[2 * i + 1] = ids[3 * e + c];
    for (int j = 0; j < 7; ++j) {
      poses[14 * i + j] = st[13 * a + j];
      poses[14 * i + 7 + j] = st[13 * c + j];
    }
    float gmax = -INFINITY;
    for (int r = 0; r < 3; ++r) gmax = fmaxf(gmax, fabsf(cw[a][r] - cw[c][r]) - (hw[a][r] + hw[c][r] + sp.slack));
    culled[i] = gmax > 0.f;
  }
}

__global__ void __launch_bounds__(128) sim_integrate_kernel(SimParams sp, int E, const float* __restrict__ body,
                                                            float* __restrict__ state, const float* __restrict__ logits,
                                                            const float* __restrict__ grad,
                                                            const uint8_t* __restrict__ culled,
                                                            int32_t* __restrict__ contacts,
                                                            const double* __restrict__ t0_dev, int n) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  float* st = state + (int64_t)e * 39;
  float Fo[3][3] = {}, To[3][3] = {};
  for (int p = 0; p < 3; ++p) {
    const int64_t i = 3 * (int64_t)e + p;
    const float s = logits[i];
    if (culled[i] || !(s > 0.f)) continue;  // contact iff unculled and p > 1/2
    if (contacts) ++contacts[i];
    const int bx[2] = {kPairA[p], kPairB[p]};
    float gt[2][3], gw[2][3], nrm2 = 0.f, sdot = 0.f;
    for (int side = 0; side < 2; ++side) {
      const float* g = grad + 14 * i + 7 * side;
      const float* X = st + 13 * bx[side];
      for (int k = 0; k < 3; ++k) {
        const float ek[4] = {0.f, k == 0 ? 1.f : 0.f, k == 1 ? 1.f : 0.f, k == 2 ? 1.f : 0.f};
        float d[4];
        qmulf(ek, X, d);
        gw[side][k] = 0.5f * (((g[0] * d[0] + g[1] * d[1]) + g[2] * d[2]) + g[3] * d[3]);
        gt[side][k] = g[4 + k];
        nrm2 += gt[side][k] * gt[side][k] + gw[side][k] * gw[side][k];
        sdot += gt[side][k] * X[7 + k] + gw[side][k] * X[10 + k];
      }
    }
    const float nrm = sqrtf(nrm2);
    if (!(nrm > 1e-12f)) continue;
    const float raw = sp.ks * s + sp.kd * sdot;
    const float lam = raw > 0.f ? raw : 0.f;
    for (int side = 0; side < 2; ++side)
      for (int k = 0; k < 3; ++k) {
        Fo[bx[side]][k] -= lam * gt[side][k] / nrm;
        To[bx[side]][k] -= lam * gw[side][k] / nrm;
      }
  }
  for (int bi = 1; bi < 3; ++bi) {  // semi-implicit Euler of the dynamic bodies
    float* X = st + 13 * bi;
    const float* bd = body + ((int64_t)e * 3 + bi) * 4;
    float R[9];
    rot_of(X, R);
    float tb[3], dw[3];
    for (int k = 0; k < 3; ++k) tb[k] = ((R[k] * To[bi][0] + R[3 + k] * To[bi][1]) + R[6 + k] * To[bi][2]) / bd[1 + k];
    for (int r = 0; r < 3; ++r) dw[r] = (R[3 * r] * tb[0] + R[3 * r + 1] * tb[1]) + R[3 * r + 2] * tb[2];
    for (int k = 0; k < 3; ++k) {
      X[7 + k] += sp.h * (Fo[bi][k] / bd[0] + sp.g[k]);
      X[10 + k] += sp.h * dw[k];
    }
    for (int k = 0; k < 3; ++k) X[4 + k] += sp.h * X[7 + k];
    const float w4[4] = {0.f, X[10], X[11], X[12]};
    float wq[4];
    qmulf(w4, X, wq);
    float qn[4];
    for (int k = 0; k < 4; ++k) qn[k] = X[k] + 0.5f * sp.h * wq[k];
    const float nn = sqrtf(((qn[0] * qn[0] + qn[1] * qn[1]) + qn[2] * qn[2]) + qn[3] * qn[3]);
    for (int k = 0; k < 4; ++k) X[k] = qn[k] / nn;
  }
  set_bowl(sp, st, *t0_dev + (n + 1) * sp.hd);
}

}  // namespace

cudaError_t launch_sim_set_t0(double* t0_dev, double t0, cudaStream_t st) {
  sim_set_t0_kernel<<<1, 1, 0, st>>>(t0_dev, t0);
  return cudaGetLastError();
}

cudaError_t launch_sim_prepare(const ShapeTable& T, const SimParams& sp, int E, const int32_t* ids, float* state,
                               const double* t0_dev, int n, int32_t* pairs, float* poses, uint8_t* culled,
                               unsigned long long* bad, cudaStream_t st) {
  if (E == 0) return cudaSuccess;
  sim_prepare_kernel<<<(E + 127) / 128, 128, 0, st>>>(T, sp, E, ids, state, t0_dev, n, pairs, poses, culled, bad);
  return cudaGetLastError();
}

cudaError_t launch_sim_integrate(const SimParams& sp, int E, const float* body, float* state, const float* logits,
                                 const float* grad, const uint8_t* culled, int32_t* contacts, const double* t0_dev,
                                 int n, cudaStream_t st) {
  if (E == 0) return cudaSuccess;
  sim_integrate_kernel<<<(E + 127) / 128, 128, 0, st>>>(sp, E, body, state, logits, grad, culled, contacts, t0_dev,
                                                          n);
  return cudaGetLastError();
}

}  // namespace locc
