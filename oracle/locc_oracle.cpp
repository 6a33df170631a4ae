// locc_oracle.cpp — plain CPU reference of the LOCC batched collision query.
//
// TEST INFRASTRUCTURE ONLY (see locc_oracle.h).  Shares nothing with the CUDA path.
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fPIC -shared -pthread (never -ffast-math:
// the crop masks must come out of exactly the fp32 operations written below).
//
// Each step cites the passage it follows.  P:n = PAPER.md line n, S:n = SPEC.md line n,
// and "O<k>" = the step of SURVEY.md §8(c) that fixes the reading used by this build.
#include "locc_oracle.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr int kP = 128;  // predictor MLP width: "3 layers of 128 neurons"

// ------------------------------------------------------------------ parameters
// Canonical order (SURVEY.md §8(c) "Parameter layout"), row-major [out][in], W then b.
struct Layer {
  const float* W;
  const float* b;
  int out, in;
};
struct Params {
  Layer enc1, enc2, enc3, proj, obj1, obj2, obj3, pair1, pair2, pair3, out;
};

int64_t n_params(int H, int F) {
  auto L = [](int64_t o, int64_t i) { return o * i + o; };
  return L(H, 3) + L(H, H) + L(H, H) + L(F, H) + L(kP, F + 7) + 5 * L(kP, kP) + L(1, kP);
}

Params bind_params(const float* w, int H, int F) {
  Params p;
  const float* c = w;
  auto take = [&c](int o, int i) {
    Layer l{c, c + (int64_t)o * i, o, i};
    c += (int64_t)o * i + o;
    return l;
  };
  p.enc1 = take(H, 3);
  p.enc2 = take(H, H);
  p.enc3 = take(H, H);
  p.proj = take(F, H);
  p.obj1 = take(kP, F + 7);
  p.obj2 = take(kP, kP);
  p.obj3 = take(kP, kP);
  p.pair1 = take(kP, kP);
  p.pair2 = take(kP, kP);
  p.pair3 = take(kP, kP);
  p.out = take(1, kP);
  return p;
}

// bf16 round-to-nearest-even of a double (8 significant bits), used only in bf16_emul mode.
double bf16_rne(double x) {
  if (x == 0.0 || !std::isfinite(x)) return x;
  int e;
  double m = std::frexp(x, &e);                // x = m * 2^e, 0.5 <= |m| < 1
  double r = std::nearbyint(std::ldexp(m, 8));  // default rounding mode: ties to even
  return std::ldexp(r, e - 8);
}

// y = act(W x + b) in fp64, plain dot products in index order.  `Wd` = the weights as
// doubles (already bf16-rounded in bf16_emul mode); `round_in` rounds x to bf16 first.
void dense(const Layer& L, const double* Wd, const double* x, double* y, bool relu, bool round_in) {
  std::vector<double> xr(x, x + L.in);
  if (round_in)
    for (double& v : xr) v = bf16_rne(v);
  for (int o = 0; o < L.out; ++o) {
    double acc = 0.0;
    for (int i = 0; i < L.in; ++i) acc += Wd[(int64_t)o * L.in + i] * xr[i];
    acc += (double)L.b[o];
    y[o] = relu ? (acc > 0.0 ? acc : 0.0) : acc;
  }
}
void dense(const Layer& L, const double* x, double* y, bool relu) {
  std::vector<double> Wd(L.W, L.W + (int64_t)L.out * L.in);
  dense(L, Wd.data(), x, y, relu, false);
}

// Weights of one layer widened to fp64, optionally rounded to bf16 (bf16_emul mode).
std::vector<double> widen(const Layer& L, bool round) {
  std::vector<double> w(L.W, L.W + (int64_t)L.out * L.in);
  if (round)
    for (double& v : w) v = bf16_rne(v);
  return w;
}

// ------------------------------------------------------------------ O0: shape precompute
// AABB of the cloud ("compute the AABB of each object's mesh"; Q7: from the points),
// M x M x M grid over it, eps = half the cell diagonal of this shape, used
// when this shape is the *counter* object (P:424 eps = sqrt(a1^2+a2^2+a3^2)/2, a3^3 read
// as the typo a3^2), cell binning floor((p-lo)*M/ext) clamped to M-1.
struct ShapeInfo {
  float lo[3], hi[3];
  float eps2;
  std::vector<int32_t> cell;  // per point, caller's order
};

bool shape_prep(const float* pts, int K, int M, ShapeInfo& s) {
  if (K < 1 || M < 1) return false;
  for (int d = 0; d < 3; ++d) {
    s.lo[d] = pts[d];
    s.hi[d] = pts[d];
  }
  for (int k = 0; k < K; ++k)
    for (int d = 0; d < 3; ++d) {
      float v = pts[3 * k + d];
      if (!std::isfinite(v)) return false;
      if (v < s.lo[d]) s.lo[d] = v;
      if (v > s.hi[d]) s.hi[d] = v;
    }
  double ext[3], a[3];
  for (int d = 0; d < 3; ++d) {
    ext[d] = (double)s.hi[d] - (double)s.lo[d];
    a[d] = ext[d] / (double)M;
  }
  s.eps2 = (float)(0.25 * ((a[0] * a[0] + a[1] * a[1]) + a[2] * a[2]));
  s.cell.assign(K, 0);
  for (int k = 0; k < K; ++k) {
    int c[3];
    for (int d = 0; d < 3; ++d) {
      if (ext[d] == 0.0) {
        c[d] = 0;
        continue;
      }
      double u = (((double)pts[3 * k + d] - (double)s.lo[d]) * (double)M) / ext[d];
      double f = std::floor(u);
      c[d] = f >= (double)(M - 1) ? M - 1 : (int)f;
    }
    s.cell[k] = c[0] + M * (c[1] + M * c[2]);
  }
  return true;
}

// ------------------------------------------------------------------ O1-O3: relative pose
struct Quat {
  double w, x, y, z;
};

// O1: normalise in fp64 from the fp32 inputs.
bool normalise(const float* q7, Quat& q) {
  double w = q7[0], x = q7[1], y = q7[2], z = q7[3];
  double n2 = ((w * w + x * x) + y * y) + z * z;
  if (!(n2 >= 1e-12) || !std::isfinite(n2)) return false;
  double s = std::sqrt(n2);
  q = {w / s, x / s, y / s, z / s};
  return true;
}

// O2: Hamilton product q1 (x) q2 = (w1w2 - v1.v2, w1 v2 + w2 v1 + v1 x v2), grouped so that
// conj(q) (x) q has an exactly zero vector part.
Quat hamilton(const Quat& a, const Quat& b) {
  Quat r;
  r.w = a.w * b.w - ((a.x * b.x + a.y * b.y) + a.z * b.z);
  r.x = (a.w * b.x + b.w * a.x) + (a.y * b.z - a.z * b.y);
  r.y = (a.w * b.y + b.w * a.y) + (a.z * b.x - a.x * b.z);
  r.z = (a.w * b.z + b.w * a.z) + (a.x * b.y - a.y * b.x);
  return r;
}
Quat conj(const Quat& q) { return {q.w, -q.x, -q.y, -q.z}; }

// O3: rotation matrix of a quaternion (fp64).
void rotmat(const Quat& q, double R[3][3]) {
  const double w = q.w, x = q.x, y = q.y, z = q.z;
  R[0][0] = 1.0 - 2.0 * (y * y + z * z);
  R[0][1] = 2.0 * (x * y - w * z);
  R[0][2] = 2.0 * (x * z + w * y);
  R[1][0] = 2.0 * (x * y + w * z);
  R[1][1] = 1.0 - 2.0 * (x * x + z * z);
  R[1][2] = 2.0 * (y * z - w * x);
  R[2][0] = 2.0 * (x * z - w * y);
  R[2][1] = 2.0 * (y * z + w * x);
  R[2][2] = 1.0 - 2.0 * (x * x + y * y);
}

// Frame of B seen from A: p_B = R_B^T (R_A p + t_A - t_B) = R(conj(qB) (x) qA) p + R_B^T (t_A - t_B)
// ("create the OBB of shape embeddings of two objects by using their poses").
void relative(const Quat& qA, const float* tA, const Quat& qB, const float* tB, float Rout[9],
              float tout[3]) {
  double R[3][3], RB[3][3];
  rotmat(hamilton(conj(qB), qA), R);
  rotmat(qB, RB);
  double d[3] = {(double)tA[0] - (double)tB[0], (double)tA[1] - (double)tB[1],
                 (double)tA[2] - (double)tB[2]};
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) Rout[3 * i + j] = (float)R[i][j];
    tout[i] = (float)((RB[0][i] * d[0] + RB[1][i] * d[1]) + RB[2][i] * d[2]);
  }
}

// ------------------------------------------------------------------ O4: crop
// Keep point p of one object iff the Euclidean distance from its position in the other
// object's frame to the other object's AABB is <= eps_other (S:359 applied
// to points; reading Q8).  fp32, exactly these operations.
int crop(const float* pts, int K, const float R[9], const float t[3], const ShapeInfo& other,
         std::vector<uint8_t>& keep) {
  keep.assign(K, 0);
  int n = 0;
  for (int k = 0; k < K; ++k) {
    const float x = pts[3 * k], y = pts[3 * k + 1], z = pts[3 * k + 2];
    float p[3];
    for (int i = 0; i < 3; ++i)
      p[i] = std::fmaf(R[3 * i], x, std::fmaf(R[3 * i + 1], y, std::fmaf(R[3 * i + 2], z, t[i])));
    float dd[3];
    for (int i = 0; i < 3; ++i) {
      float a = other.lo[i] - p[i];
      float b = p[i] - other.hi[i];
      float m = std::fmaxf(a, b);
      dd[i] = std::fmaxf(m, 0.0f);
    }
    float zz = dd[2] * dd[2];
    float d2 = std::fmaf(dd[0], dd[0], std::fmaf(dd[1], dd[1], zz));
    if (d2 <= other.eps2) {
      keep[k] = 1;
      ++n;
    }
  }
  return n;
}

// ------------------------------------------------------------------ O6-O7: encoder + pooling
// Per kept point: 3 ReLU layers of width H ("3 layers of MLP with 256 neurons",
// P:425 ReLU), input = the point's local-frame coordinates (reading Q6).  Cell-wise max over
// the kept points of each cell, average over the occupied cells (P:335, P:424
// "average pooling", reading Q11), then one linear layer to F (reading Q5).
// Returns C (occupied cells); e = 0 when no point is kept.
struct EncW {
  std::vector<double> w1, w2, w3, wf;  // fp64 copies; w2, w3 bf16-rounded in bf16_emul mode
};

int encode(const Params& P, const EncW& W, const float* pts, int K, const ShapeInfo& s,
           const std::vector<uint8_t>& keep, int M, int H, int F, bool emul, double* e) {
  const int ncell = M * M * M;
  std::vector<double> g((size_t)ncell * H, 0.0);
  std::vector<uint8_t> occ(ncell, 0);
  std::vector<double> x(3), h1(H), h2(H), h3(H);
  int n = 0;
  for (int k = 0; k < K; ++k) {
    if (!keep[k]) continue;
    ++n;
    for (int d = 0; d < 3; ++d) x[d] = pts[3 * k + d];
    if (emul) {
      // bf16 mode: layer 1 is fp32 arithmetic by definition of the bf16 path, and
      // its bf16 rounding is a quantisation decision taken in the kernel's precision, so h1 is
      // formed exactly as fp32 fma(w0, x, fma(w1, y, fma(w2, z, b))) before rounding.
      for (int o = 0; o < H; ++o) {
        const float* w = P.enc1.W + 3 * o;
        float h = std::fmaf(w[0], pts[3 * k], std::fmaf(w[1], pts[3 * k + 1], std::fmaf(w[2], pts[3 * k + 2], P.enc1.b[o])));
        h1[o] = h > 0.0f ? (double)h : 0.0;
      }
    } else {
      dense(P.enc1, W.w1.data(), x.data(), h1.data(), true, false);
    }
    dense(P.enc2, W.w2.data(), h1.data(), h2.data(), true, emul);
    dense(P.enc3, W.w3.data(), h2.data(), h3.data(), true, emul);
    const int c = s.cell[k];
    double* gc = &g[(size_t)c * H];
    if (!occ[c]) {
      occ[c] = 1;
      for (int j = 0; j < H; ++j) gc[j] = h3[j];
    } else {
      for (int j = 0; j < H; ++j) gc[j] = h3[j] > gc[j] ? h3[j] : gc[j];
    }
  }
  if (n == 0) {
    for (int j = 0; j < F; ++j) e[j] = 0.0;
    return 0;
  }
  std::vector<double> m(H, 0.0);
  int C = 0;
  for (int c = 0; c < ncell; ++c) {  // ascending cell order
    if (!occ[c]) continue;
    ++C;
    for (int j = 0; j < H; ++j) m[j] += g[(size_t)c * H + j];
  }
  for (int j = 0; j < H; ++j) m[j] /= (double)C;
  dense(P.proj, W.wf.data(), m.data(), e, false, false);
  return C;
}

// ------------------------------------------------------------------ O8-O9: predictor
// [e ; pose] -> 3x128 ReLU (shared by both objects) -> elementwise max across the pair ->
// 3x128 ReLU -> linear -> sigmoid.  Pose = own world pose, unit quaternion with
// the first non-zero component made positive, then translation (reading Q12).
void object_mlp(const Params& P, const double* e, int F, const Quat& q, const float* t, double* u) {
  std::vector<double> z(F + 7), a(kP), b(kP);
  for (int j = 0; j < F; ++j) z[j] = e[j];
  double qc[4] = {q.w, q.x, q.y, q.z};
  double sgn = 1.0;
  for (int i = 0; i < 4; ++i)
    if (qc[i] != 0.0) {
      sgn = qc[i] > 0.0 ? 1.0 : -1.0;
      break;
    }
  for (int i = 0; i < 4; ++i) z[F + i] = sgn * qc[i];
  for (int i = 0; i < 3; ++i) z[F + 4 + i] = t[i];
  dense(P.obj1, z.data(), a.data(), true);
  dense(P.obj2, a.data(), b.data(), true);
  dense(P.obj3, b.data(), u, true);
}

double pair_head(const Params& P, const double* uA, const double* uB) {
  std::vector<double> v(kP), a(kP), b(kP), c(kP);
  for (int j = 0; j < kP; ++j) v[j] = uA[j] > uB[j] ? uA[j] : uB[j];
  dense(P.pair1, v.data(), a.data(), true);
  dense(P.pair2, a.data(), b.data(), true);
  dense(P.pair3, b.data(), c.data(), true);
  double logit;
  dense(P.out, c.data(), &logit, false);
  return logit;
}

// ------------------------------------------------------------------ NEXT-2: pose gradient
// d logit / d (q_A, t_A, q_B, t_B) of the predictor at fixed crops (the crop mask is
// piecewise constant in the pose, so nothing flows through it; the encoder sees local-frame points,
// so e does not depend on the pose).  Plain reverse-mode chain rule in fp64 over the same layers as
// object_mlp / pair_head; ReLU'(x) = [x > 0]; the max across the pair passes the gradient to the
// side it selected (uA > uB -> A, else B, as pair_head).  Raw quaternion q -> q^ = sgn q / |q| with
// |q| from O1's grouping and sgn the canonical sign (Q12): dq = sgn (dq^ - q^ (q^ . dq^)) / |q|.
// grad = [d/dq_A (4), d/dt_A (3), d/dq_B (4), d/dt_B (3)].
struct ObjAct {
  std::vector<double> z, a1, a2, u;
};

// dense + ReLU that also lowers mg to the smallest |pre-activation| seen: how far a ReLU decision is
// from its threshold (reported so tests can set aside pairs whose fp32 decisions may legitimately flip).
void dense_relu_mg(const Layer& L, const double* x, double* y, double& mg) {
  dense(L, x, y, false);
  for (int o = 0; o < L.out; ++o) {
    mg = std::min(mg, std::fabs(y[o]));
    y[o] = y[o] > 0.0 ? y[o] : 0.0;
  }
}

void object_fwd(const Params& P, const double* e, int F, const double qh[4], const double t[3], ObjAct& A,
                double& mg) {
  A.z.assign(F + 7, 0.0);
  A.a1.assign(kP, 0.0);
  A.a2.assign(kP, 0.0);
  A.u.assign(kP, 0.0);
  for (int j = 0; j < F; ++j) A.z[j] = e[j];
  for (int i = 0; i < 4; ++i) A.z[F + i] = qh[i];
  for (int i = 0; i < 3; ++i) A.z[F + 4 + i] = t[i];
  dense_relu_mg(P.obj1, A.z.data(), A.a1.data(), mg);
  dense_relu_mg(P.obj2, A.a1.data(), A.a2.data(), mg);
  dense_relu_mg(P.obj3, A.a2.data(), A.u.data(), mg);
}

// y = W^T g (W row-major [out][in]): the transpose product of reverse mode.
void dense_T(const Layer& L, const double* g, double* y) {
  for (int i = 0; i < L.in; ++i) y[i] = 0.0;
  for (int o = 0; o < L.out; ++o)
    for (int i = 0; i < L.in; ++i) y[i] += (double)L.W[(int64_t)o * L.in + i] * g[o];
}

// O1 + Q12 on a raw quaternion held in doubles: q^ (canonical sign), |q| and the sign.
bool canonical(const double q[4], double qh[4], double& norm, double& sgn) {
  const double n2 = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
  if (!(n2 >= 1e-12)) return false;
  norm = std::sqrt(n2);
  double n[4];
  for (int i = 0; i < 4; ++i) n[i] = q[i] / norm;
  sgn = 1.0;
  for (int i = 0; i < 4; ++i)
    if (n[i] != 0.0) {
      sgn = n[i] > 0.0 ? 1.0 : -1.0;
      break;
    }
  for (int i = 0; i < 4; ++i) qh[i] = sgn * n[i];
  return true;
}

double head_grad(const Params& P, const double* eA, const double* eB, int F, const double qA[4], const double tA[3],
                 const double qB[4], const double tB[3], double grad[14], double* margin = nullptr) {
  double qhA[4], qhB[4], nA, nB, sA, sB;
  canonical(qA, qhA, nA, sA);
  canonical(qB, qhB, nB, sB);
  ObjAct A, B;
  double mg = INFINITY;
  object_fwd(P, eA, F, qhA, tA, A, mg);
  object_fwd(P, eB, F, qhB, tB, B, mg);
  std::vector<double> v(kP), c1(kP), c2(kP), c3(kP);
  for (int j = 0; j < kP; ++j) {
    v[j] = A.u[j] > B.u[j] ? A.u[j] : B.u[j];
    if (v[j] > 0.0) mg = std::min(mg, std::fabs(A.u[j] - B.u[j]));  // the max's routing decision
  }
  dense_relu_mg(P.pair1, v.data(), c1.data(), mg);
  dense_relu_mg(P.pair2, c1.data(), c2.data(), mg);
  dense_relu_mg(P.pair3, c2.data(), c3.data(), mg);
  if (margin) *margin = mg;
  double logit;
  dense(P.out, c3.data(), &logit, false);
  // reverse mode
  std::vector<double> g(kP), h(kP);
  for (int j = 0; j < kP; ++j) g[j] = c3[j] > 0.0 ? (double)P.out.W[j] : 0.0;  // d/d pre3 of pair
  dense_T(P.pair3, g.data(), h.data());                                         // d/d c2
  for (int j = 0; j < kP; ++j) g[j] = c2[j] > 0.0 ? h[j] : 0.0;
  dense_T(P.pair2, g.data(), h.data());  // d/d c1
  for (int j = 0; j < kP; ++j) g[j] = c1[j] > 0.0 ? h[j] : 0.0;
  std::vector<double> gv(kP);
  dense_T(P.pair1, g.data(), gv.data());  // d/d v
  auto side = [&](const ObjAct& S, bool is_a, const double qh[4], double norm, double sgn, double* out7) {
    std::vector<double> gu(kP), x(kP), y(kP), gz(F + 7);
    for (int j = 0; j < kP; ++j) {
      const bool sel = is_a ? (A.u[j] > B.u[j]) : !(A.u[j] > B.u[j]);
      gu[j] = sel ? gv[j] : 0.0;
    }
    for (int j = 0; j < kP; ++j) x[j] = S.u[j] > 0.0 ? gu[j] : 0.0;
    dense_T(P.obj3, x.data(), y.data());  // d/d a2
    for (int j = 0; j < kP; ++j) x[j] = S.a2[j] > 0.0 ? y[j] : 0.0;
    dense_T(P.obj2, x.data(), y.data());  // d/d a1
    for (int j = 0; j < kP; ++j) x[j] = S.a1[j] > 0.0 ? y[j] : 0.0;
    dense_T(P.obj1, x.data(), gz.data());  // d/d z
    const double* gq = gz.data() + F;
    const double dot = ((qh[0] * gq[0] + qh[1] * gq[1]) + qh[2] * gq[2]) + qh[3] * gq[3];
    for (int i = 0; i < 4; ++i) out7[i] = sgn * (gq[i] - qh[i] * dot) / norm;
    for (int i = 0; i < 3; ++i) out7[4 + i] = gz[F + 4 + i];
  };
  side(A, true, qhA, nA, sA, grad);
  side(B, false, qhB, nB, sB, grad + 7);
  return logit;
}

// ------------------------------------------------------------------ NEXT-1: encode-once LOCC
// The paper's own inference design (readings Q27-Q30): each shape
// is encoded ONCE into an M x M x M x F embedding grid; a query only selects cells and pools them.
//
// Grids are channel-last, position index x + D (y + D z) (the cell-id order of O0).  3D kernels
// W[o][i][k], k = kx + 3 (ky + 3 kz) (the same order), 3 x 3 x 3, stride 1.

// conv3d ("3D convolution layers ... filter of size (3,3,3)"): cross-correlation with zero
// padding p: y[q][o] = b[o] + sum_k sum_i W[o][i][k] x[q + k - p][i], q in [0, D + 2p - 2)^3.
void conv3d(const double* x, int D, int Cin, const double* W, const double* b, int Cout, int p, double* y) {
  const int Do = D + 2 * p - 2;
  for (int qz = 0; qz < Do; ++qz)
    for (int qy = 0; qy < Do; ++qy)
      for (int qx = 0; qx < Do; ++qx) {
        double* yq = y + ((int64_t)(qz * Do + qy) * Do + qx) * Cout;
        for (int o = 0; o < Cout; ++o) {
          double acc = b ? b[o] : 0.0;
          for (int k = 0; k < 27; ++k) {
            const int iz = qz + k / 9 - p, iy = qy + (k / 3) % 3 - p, ix = qx + k % 3 - p;
            if (iz < 0 || iy < 0 || ix < 0 || iz >= D || iy >= D || ix >= D) continue;
            const double* xi = x + ((int64_t)(iz * D + iy) * D + ix) * Cin;
            for (int i = 0; i < Cin; ++i) acc += W[((int64_t)o * Cin + i) * 27 + k] * xi[i];
          }
          yq[o] = acc;
        }
      }
}

// deconv3d ("deconvolution layers with the same parameters in reverse order"): the transposed
// convolution, by its definition — every input position q scatters W[o][i][k] x[q][i] to output
// position q + k - p; output size D + 2 - 2p (p = 1: same size; p = 0: undoes a valid conv).
void deconv3d(const double* x, int D, int Cin, const double* W, const double* b, int Cout, int p, double* y) {
  const int Do = D + 2 - 2 * p;
  for (int64_t q = 0; q < (int64_t)Do * Do * Do; ++q)
    for (int o = 0; o < Cout; ++o) y[q * Cout + o] = b ? b[o] : 0.0;
  for (int iz = 0; iz < D; ++iz)
    for (int iy = 0; iy < D; ++iy)
      for (int ix = 0; ix < D; ++ix) {
        const double* xi = x + ((int64_t)(iz * D + iy) * D + ix) * Cin;
        for (int k = 0; k < 27; ++k) {
          const int qz = iz + k / 9 - p, qy = iy + (k / 3) % 3 - p, qx = ix + k % 3 - p;
          if (qz < 0 || qy < 0 || qx < 0 || qz >= Do || qy >= Do || qx >= Do) continue;
          double* yq = y + ((int64_t)(qz * Do + qy) * Do + qx) * Cout;
          for (int o = 0; o < Cout; ++o) {
            double acc = 0.0;
            for (int i = 0; i < Cin; ++i) acc += W[((int64_t)o * Cin + i) * 27 + k] * xi[i];
            yq[o] += acc;
          }
        }
      }
}

void relu_inplace(std::vector<double>& v) {
  for (double& a : v) a = a > 0.0 ? a : 0.0;
}

// [a ; b] per position ("skip connection with concatenation").
std::vector<double> concat(const std::vector<double>& a, int Ca, const std::vector<double>& b, int Cb, int64_t npos) {
  std::vector<double> r((size_t)npos * (Ca + Cb));
  for (int64_t q = 0; q < npos; ++q) {
    for (int c = 0; c < Ca; ++c) r[q * (Ca + Cb) + c] = a[q * Ca + c];
    for (int c = 0; c < Cb; ++c) r[q * (Ca + Cb) + Ca + c] = b[q * Cb + c];
  }
  return r;
}

constexpr int kU = 128;  // U-Net channels ("# channels of 3D CNN ... 128")

// Canonical U-Net parameter order (Q30): c1 [128][H][27], c2..c4 [128][128][27], d4 [128][128][27],
// d3, d2, d1 [128][256][27], each W then b [128]; proj W [F][256], b [F].
int64_t unet_n_params(int H, int F) {
  return (int64_t)kU * 27 * (H + 3 * kU + kU + 3 * 2 * kU) + 8 * kU + (int64_t)F * 2 * kU + F;
}

struct UNetW {
  std::vector<double> W[8], b[8], pW, pb;  // 0..3 = c1..c4, 4..7 = d4, d3, d2, d1
};

UNetW bind_unet(const float* u, int H, int F) {
  UNetW U;
  const int cin[8] = {H, kU, kU, kU, kU, 2 * kU, 2 * kU, 2 * kU};
  for (int l = 0; l < 8; ++l) {
    const int64_t n = (int64_t)kU * cin[l] * 27;
    U.W[l].assign(u, u + n);
    u += n;
    U.b[l].assign(u, u + kU);
    u += kU;
  }
  U.pW.assign(u, u + (int64_t)F * 2 * kU);
  u += (int64_t)F * 2 * kU;
  U.pb.assign(u, u + F);
  return U;
}

// Q27: every point of the shape through the point MLP (the same 3 layers as O6), cell-
// wise max ("cell-wise max-pooling"); an empty cell is 0.  G: [M^3][H].
void grid_maxpool(const Params& P, const EncW& EW, const float* pts, int K, const ShapeInfo& s, int M, int H,
                  std::vector<double>& G) {
  const int ncell = M * M * M;
  G.assign((size_t)ncell * H, 0.0);
  std::vector<uint8_t> occ(ncell, 0);
  std::vector<double> x(3), h1(H), h2(H), h3(H);
  for (int k = 0; k < K; ++k) {
    for (int d = 0; d < 3; ++d) x[d] = pts[3 * k + d];
    dense(P.enc1, EW.w1.data(), x.data(), h1.data(), true, false);
    dense(P.enc2, EW.w2.data(), h1.data(), h2.data(), true, false);
    dense(P.enc3, EW.w3.data(), h2.data(), h3.data(), true, false);
    double* gc = &G[(size_t)s.cell[k] * H];
    if (!occ[s.cell[k]]) {
      occ[s.cell[k]] = 1;
      for (int j = 0; j < H; ++j) gc[j] = h3[j];
    } else {
      for (int j = 0; j < H; ++j) gc[j] = h3[j] > gc[j] ? h3[j] : gc[j];
    }
  }
}

// Q28: the 3D U-Net: 4 conv (128 ch, 3^3, ReLU; the first valid M^3 -> (M-2)^3,
// the rest same), global average of the last conv's features, 4 deconv in reverse order with
// concatenation skips (d4 <- c4; d3 <- [d4; c3]; d2 <- [d3; c2]; d1 <- [d2; c1], the last one the
// transposed valid conv back to M^3), the global feature tiled and concatenated, one linear layer to F
// (P:422).  E: [M^3][F].
void unet(const UNetW& U, const std::vector<double>& G, int M, int H, int F, std::vector<double>& E,
          bool global_max = false) {
  const int D = M - 2;
  const int64_t n4 = (int64_t)D * D * D, n6 = (int64_t)M * M * M;
  std::vector<double> c1(n4 * kU), c2(n4 * kU), c3(n4 * kU), c4(n4 * kU), d4(n4 * kU), d3(n4 * kU), d2(n4 * kU),
      d1(n6 * kU);
  conv3d(G.data(), M, H, U.W[0].data(), U.b[0].data(), kU, 0, c1.data());
  relu_inplace(c1);
  conv3d(c1.data(), D, kU, U.W[1].data(), U.b[1].data(), kU, 1, c2.data());
  relu_inplace(c2);
  conv3d(c2.data(), D, kU, U.W[2].data(), U.b[2].data(), kU, 1, c3.data());
  relu_inplace(c3);
  conv3d(c3.data(), D, kU, U.W[3].data(), U.b[3].data(), kU, 1, c4.data());
  relu_inplace(c4);
  std::vector<double> g(kU, 0.0);
  if (global_max) {  // the appendix's reading ("we apply max pooling to get global features")
    for (int64_t q = 0; q < n4; ++q)
      for (int c = 0; c < kU; ++c) g[c] = std::max(g[c], c4[q * kU + c]);  // c4 >= 0 (ReLU)
  } else {
    for (int64_t q = 0; q < n4; ++q)
      for (int c = 0; c < kU; ++c) g[c] += c4[q * kU + c];
    for (int c = 0; c < kU; ++c) g[c] /= (double)n4;
  }
  deconv3d(c4.data(), D, kU, U.W[4].data(), U.b[4].data(), kU, 1, d4.data());
  relu_inplace(d4);
  std::vector<double> x = concat(d4, kU, c3, kU, n4);
  deconv3d(x.data(), D, 2 * kU, U.W[5].data(), U.b[5].data(), kU, 1, d3.data());
  relu_inplace(d3);
  x = concat(d3, kU, c2, kU, n4);
  deconv3d(x.data(), D, 2 * kU, U.W[6].data(), U.b[6].data(), kU, 1, d2.data());
  relu_inplace(d2);
  x = concat(d2, kU, c1, kU, n4);
  deconv3d(x.data(), D, 2 * kU, U.W[7].data(), U.b[7].data(), kU, 0, d1.data());
  relu_inplace(d1);
  E.assign((size_t)n6 * F, 0.0);
  for (int64_t c = 0; c < n6; ++c)
    for (int f = 0; f < F; ++f) {
      double acc = 0.0;
      for (int j = 0; j < kU; ++j) acc += U.pW[(int64_t)f * 2 * kU + j] * d1[c * kU + j];
      for (int j = 0; j < kU; ++j) acc += U.pW[(int64_t)f * 2 * kU + kU + j] * g[j];
      E[c * F + f] = acc + U.pb[f];
    }
}

// Q29: cell centre of cell (ix, iy, iz) in the shape's own frame, fp64 rounded once to fp32.
void cell_centre(const ShapeInfo& s, int M, int c, float out[3]) {
  const int i[3] = {c % M, (c / M) % M, c / (M * M)};
  for (int d = 0; d < 3; ++d) {
    const double ext = (double)s.hi[d] - (double)s.lo[d];
    out[d] = (float)((double)s.lo[d] + (((double)i[d] + 0.5) * ext) / (double)M);
  }
}

// Q29: cell c of this object is selected iff its centre, moved into the other object's
// frame by (R, t), lies within this object's own cell half-diagonal (the "margin ... distance from the
// center point to a vertex of a cell") of the other's AABB — O4's fp32 test on the cell centre.
int select_cells(const ShapeInfo& self, int M, const float R[9], const float t[3], const ShapeInfo& other,
                 std::vector<uint8_t>& sel) {
  const int ncell = M * M * M;
  std::vector<float> ctr((size_t)3 * ncell);
  for (int c = 0; c < ncell; ++c) cell_centre(self, M, c, &ctr[3 * c]);
  ShapeInfo o = other;  // other's AABB with this object's margin
  o.eps2 = self.eps2;
  return crop(ctr.data(), ncell, R, t, o, sel);
}

// ------------------------------------------------------------------ NEXT-3: closed-loop step
// A Brax-style rigid-body substep with LOCC as the contact detector (SPEC.md
// S:638-665; reading Q31).  Per environment: body 0 = the kinematic bowl (shaken), bodies 1, 2
// dynamic; pairs (0,1), (0,2), (1,2).  State per body: q (4), t (3), v (3), w (3), world frame.
// Per substep of length h at time tau:
//   1. bowl: q kept, t = A sin(2 pi f tau), v = 2 pi f A cos(2 pi f tau), w = 0
//   2. broad phase per pair: world AABBs (centre R c + t, half-extent |R| e) overlap within `slack`
//   3. detector: logit s and d s / d(q_A, t_A, q_B, t_B) (the query + NEXT-2 gradient, crop or cells)
//   4. contact iff not culled and s > 0 (p > 1/2)
//   5. penalty along the descent of s: per side X the translational gradient g_t and the
//      rotational one G_w[k] = g_q . (1/2 (0, e_k) (x) q); n = |(all g_t, G_w)|; ds/dt = sum g_t.v + G_w.w;
//      lambda = max(0, ks s + kd ds/dt); F_X = -lambda g_t / n, tau_X = -lambda G_w / n (dynamic bodies)
//   6. semi-implicit Euler: v += h (F / m + gravity); w += h R diag(1/I) R^T tau; t += h v;
//      q = normalise(q + h/2 (0, w) (x) q)
// Margins reported per environment (min over the call): |s| and the predictor's ReLU margin over the
// unculled pairs, the broad-phase decision distance, |ks s + kd ds/dt| over contacts.
struct SimCfg {
  double h;
  int32_t substeps, detector;
  double gravity[3], ks, kd, amp[3], freq, slack;
};

void quat_left_e(const double q[4], int k, double out[4]) {  // (0, e_k) (x) q
  const Quat e{0.0, k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0};
  const Quat r = hamilton(e, Quat{q[0], q[1], q[2], q[3]});
  out[0] = r.w;
  out[1] = r.x;
  out[2] = r.y;
  out[3] = r.z;
}

bool finite_n(const float* p, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

}  // namespace

extern "C" {

int64_t oracle_n_params(int32_t H, int32_t F) { return n_params(H, F); }

int oracle_shape_prep(const float* pts, int32_t K, int32_t M, float lo[3], float hi[3], float* eps2,
                      int32_t* cell) {
  ShapeInfo s;
  if (!pts || !shape_prep(pts, K, M, s)) return -2;
  for (int d = 0; d < 3; ++d) {
    lo[d] = s.lo[d];
    hi[d] = s.hi[d];
  }
  *eps2 = s.eps2;
  if (cell) std::memcpy(cell, s.cell.data(), sizeof(int32_t) * K);
  return 0;
}

int oracle_rel_transform(const float poseA[7], const float poseB[7], float R_BA[9], float t_BA[3],
                         float R_AB[9], float t_AB[3]) {
  Quat qA, qB;
  if (!normalise(poseA, qA) || !normalise(poseB, qB)) return -1;
  relative(qA, poseA + 4, qB, poseB + 4, R_BA, t_BA);
  relative(qB, poseB + 4, qA, poseA + 4, R_AB, t_AB);
  return 0;
}

int oracle_query(const oracle_cfg* cfg, const float* weights, size_t n_weights, const float* points,
                 int32_t S, int32_t K, const int32_t* pairs, const float* poses, int64_t N,
                 double* probs, uint8_t* labels, double* logits, int32_t* kept, int32_t* occ,
                 uint32_t* masks, double* emb) {
  if (!cfg || cfg->M < 1 || cfg->H < 1 || cfg->F < 1 || N < 0) return -1;
  const int M = cfg->M, H = cfg->H, F = cfg->F;
  const bool emul = cfg->bf16_emul != 0;
  if (!weights || (int64_t)n_weights != n_params(H, F) || !finite_n(weights, (int64_t)n_weights)) return -3;
  if (!points || S < 1 || K < 1) return -2;
  if (N > 0 && (!pairs || !poses)) return -1;
  for (int64_t i = 0; i < 2 * N; ++i)
    if (pairs[i] < 0 || pairs[i] >= S) return -1;
  if (!finite_n(poses, 14 * N)) return -1;
  Params P = bind_params(weights, H, F);
  EncW EW{widen(P.enc1, false), widen(P.enc2, emul), widen(P.enc3, emul), widen(P.proj, false)};

  std::vector<ShapeInfo> shapes(S);
  for (int s = 0; s < S; ++s)
    if (!shape_prep(points + (int64_t)s * K * 3, K, M, shapes[s])) return -2;
  for (int64_t i = 0; i < 2 * N; ++i) {
    Quat q;
    if (!normalise(poses + 7 * i, q)) return -1;
  }

  const int words = (K + 31) / 32;
  std::atomic<int64_t> next(0);
  auto worker = [&]() {
    std::vector<uint8_t> keepA, keepB;
    std::vector<double> eA(F), eB(F), uA(kP), uB(kP);
    for (;;) {
      const int64_t i = next.fetch_add(1);
      if (i >= N) break;
      const int a = pairs[2 * i], b = pairs[2 * i + 1];
      const float* pA = poses + 14 * i;
      const float* pB = pA + 7;
      Quat qA, qB;
      normalise(pA, qA);
      normalise(pB, qB);
      float R_BA[9], t_BA[3], R_AB[9], t_AB[3];
      relative(qA, pA + 4, qB, pB + 4, R_BA, t_BA);
      relative(qB, pB + 4, qA, pA + 4, R_AB, t_AB);
      const float* ptsA = points + (int64_t)a * K * 3;
      const float* ptsB = points + (int64_t)b * K * 3;
      const int nA = crop(ptsA, K, R_BA, t_BA, shapes[b], keepA);
      const int nB = crop(ptsB, K, R_AB, t_AB, shapes[a], keepB);
      if (kept) {
        kept[2 * i] = nA;
        kept[2 * i + 1] = nB;
      }
      if (masks) {
        uint32_t* mA = masks + (2 * i) * words;
        uint32_t* mB = mA + words;
        std::memset(mA, 0, sizeof(uint32_t) * 2 * words);
        for (int k = 0; k < K; ++k) {
          if (keepA[k]) mA[k / 32] |= 1u << (k % 32);
          if (keepB[k]) mB[k / 32] |= 1u << (k % 32);
        }
      }
      // O5: both crops empty -> disjoint, short-circuit.
      int CA = 0, CB = 0;
      double logit, prob;
      if (nA + nB == 0) {
        for (int j = 0; j < F; ++j) eA[j] = eB[j] = 0.0;
        logit = -INFINITY;
        prob = 0.0;
      } else {
        CA = encode(P, EW, ptsA, K, shapes[a], keepA, M, H, F, emul, eA.data());
        CB = encode(P, EW, ptsB, K, shapes[b], keepB, M, H, F, emul, eB.data());
        object_mlp(P, eA.data(), F, qA, pA + 4, uA.data());
        object_mlp(P, eB.data(), F, qB, pB + 4, uB.data());
        logit = pair_head(P, uA.data(), uB.data());
        prob = 1.0 / (1.0 + std::exp(-logit));
      }
      if (occ) {
        occ[2 * i] = CA;
        occ[2 * i + 1] = CB;
      }
      if (emb)
        for (int j = 0; j < F; ++j) {
          emb[(2 * i) * F + j] = eA[j];
          emb[(2 * i + 1) * F + j] = eB[j];
        }
      if (probs) probs[i] = prob;
      if (logits) logits[i] = logit;
      if (labels) labels[i] = prob > 0.5 ? 1 : 0;  // ties negative
    }
  };
  int nt = cfg->n_threads > 0 ? cfg->n_threads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (nt > N) nt = (int)(N > 0 ? N : 1);
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  return 0;
}

int oracle_head_grad(const oracle_cfg* cfg, const float* weights, size_t n_weights, const double* eA,
                     const double* eB, const double poseA[7], const double poseB[7], double* logit, double grad[14]) {
  if (!cfg || !weights || (int64_t)n_weights != n_params(cfg->H, cfg->F)) return -3;
  const Params P = bind_params(weights, cfg->H, cfg->F);
  double qh[4], nrm, sg;
  if (!canonical(poseA, qh, nrm, sg) || !canonical(poseB, qh, nrm, sg)) return -1;
  const double l = head_grad(P, eA, eB, cfg->F, poseA, poseA + 4, poseB, poseB + 4, grad);
  if (logit) *logit = l;
  return 0;
}

int oracle_query_grad(const oracle_cfg* cfg, const float* weights, size_t n_weights, const float* points,
                      int32_t S, int32_t K, const int32_t* pairs, const float* poses, int64_t N, double* logits,
                      double* grad, double* margin) {
  if (!cfg || N < 0) return -1;
  const int F = cfg->F;
  std::vector<double> emb((size_t)(2 * N > 0 ? 2 * N : 1) * F), lg((size_t)(N > 0 ? N : 1));
  std::vector<int32_t> kept((size_t)(2 * N > 0 ? 2 * N : 1));
  const int rc = oracle_query(cfg, weights, n_weights, points, S, K, pairs, poses, N, nullptr, nullptr, lg.data(),
                              kept.data(), nullptr, nullptr, emb.data());
  if (rc) return rc;
  const Params P = bind_params(weights, cfg->H, F);
  for (int64_t i = 0; i < N; ++i) {
    double* g = grad + 14 * i;
    if (logits) logits[i] = lg[i];
    if (kept[2 * i] + kept[2 * i + 1] == 0) {  // short-circuit: constant -inf, zero gradient
      for (int j = 0; j < 14; ++j) g[j] = 0.0;
      if (margin) margin[i] = INFINITY;
      continue;
    }
    double pa[7], pb[7];
    for (int j = 0; j < 7; ++j) {
      pa[j] = poses[14 * i + j];
      pb[j] = poses[14 * i + 7 + j];
    }
    head_grad(P, emb.data() + (2 * i) * F, emb.data() + (2 * i + 1) * F, F, pa, pa + 4, pb, pb + 4, g,
              margin ? margin + i : nullptr);
  }
  return 0;
}

int64_t oracle_unet_n_params(int32_t H, int32_t F) { return unet_n_params(H, F); }

int oracle_conv3d(const double* x, int32_t D, int32_t Cin, const double* W, const double* b, int32_t Cout,
                  int32_t pad, int32_t transposed, double* y) {
  if (!x || !W || !y || D < 1 || Cin < 1 || Cout < 1 || pad < 0 || pad > 2) return -1;
  if (transposed)
    deconv3d(x, D, Cin, W, b, Cout, pad, y);
  else
    conv3d(x, D, Cin, W, b, Cout, pad, y);
  return 0;
}

int oracle_encode_grid(const oracle_cfg* cfg, const float* weights, size_t n_weights, const float* unet_w,
                       size_t n_unet, const float* pts, int32_t K, double* G, double* E) {
  if (!cfg || cfg->M < 3 || cfg->H < 1 || cfg->F < 1) return -1;
  const int M = cfg->M, H = cfg->H, F = cfg->F;
  if (!weights || (int64_t)n_weights != n_params(H, F)) return -3;
  if (!unet_w || (int64_t)n_unet != unet_n_params(H, F)) return -3;
  ShapeInfo s;
  if (!pts || !shape_prep(pts, K, M, s)) return -2;
  const Params P = bind_params(weights, H, F);
  const EncW EW{widen(P.enc1, false), widen(P.enc2, false), widen(P.enc3, false), widen(P.proj, false)};
  std::vector<double> g, e;
  grid_maxpool(P, EW, pts, K, s, M, H, g);
  if (G) std::memcpy(G, g.data(), sizeof(double) * g.size());
  unet(bind_unet(unet_w, H, F), g, M, H, F, e, cfg->global_max != 0);
  if (E) std::memcpy(E, e.data(), sizeof(double) * e.size());
  return 0;
}

int oracle_query_cells(const oracle_cfg* cfg, const float* weights, size_t n_weights, const float* unet_w,
                       size_t n_unet, const float* points, int32_t S, int32_t K, const int32_t* pairs,
                       const float* poses, int64_t N, double* probs, uint8_t* labels, double* logits,
                       int32_t* nsel, uint32_t* cells, double* emb, double* grids) {
  if (!cfg || cfg->M < 3 || cfg->H < 1 || cfg->F < 1 || N < 0) return -1;
  const int M = cfg->M, H = cfg->H, F = cfg->F, ncell = M * M * M, words = (ncell + 31) / 32;
  if (!weights || (int64_t)n_weights != n_params(H, F) || !finite_n(weights, (int64_t)n_weights)) return -3;
  if (!unet_w || (int64_t)n_unet != unet_n_params(H, F) || !finite_n(unet_w, (int64_t)n_unet)) return -3;
  if (!points || S < 1 || K < 1) return -2;
  if (N > 0 && (!pairs || !poses)) return -1;
  for (int64_t i = 0; i < 2 * N; ++i)
    if (pairs[i] < 0 || pairs[i] >= S) return -1;
  if (!finite_n(poses, 14 * N)) return -1;
  for (int64_t i = 0; i < 2 * N; ++i) {
    Quat q;
    if (!normalise(poses + 7 * i, q)) return -1;
  }
  const Params P = bind_params(weights, H, F);
  const EncW EW{widen(P.enc1, false), widen(P.enc2, false), widen(P.enc3, false), widen(P.proj, false)};
  const UNetW U = bind_unet(unet_w, H, F);
  std::vector<ShapeInfo> shapes(S);
  for (int s = 0; s < S; ++s)
    if (!shape_prep(points + (int64_t)s * K * 3, K, M, shapes[s])) return -2;
  // encode once per referenced shape (the cached embedding of P:331)
  std::vector<uint8_t> used(S, 0);
  for (int64_t i = 0; i < 2 * N; ++i) used[pairs[i]] = 1;
  std::vector<std::vector<double>> E(S);
  int nt = cfg->n_threads > 0 ? cfg->n_threads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  {
    std::atomic<int> next(0);
    auto enc = [&]() {
      std::vector<double> g;
      for (;;) {
        const int s = next.fetch_add(1);
        if (s >= S) break;
        if (!used[s]) continue;
        grid_maxpool(P, EW, points + (int64_t)s * K * 3, K, shapes[s], M, H, g);
        unet(U, g, M, H, F, E[s], cfg->global_max != 0);
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < std::min(nt, S); ++t) pool.emplace_back(enc);
    enc();
    for (auto& th : pool) th.join();
  }
  if (grids)
    for (int s = 0; s < S; ++s)
      if (used[s]) std::memcpy(grids + (int64_t)s * ncell * F, E[s].data(), sizeof(double) * ncell * F);
  std::atomic<int64_t> next(0);
  auto worker = [&]() {
    std::vector<uint8_t> selA, selB;
    std::vector<double> eA(F), eB(F), uA(kP), uB(kP);
    for (;;) {
      const int64_t i = next.fetch_add(1);
      if (i >= N) break;
      const int a = pairs[2 * i], b = pairs[2 * i + 1];
      const float* pA = poses + 14 * i;
      const float* pB = pA + 7;
      Quat qA, qB;
      normalise(pA, qA);
      normalise(pB, qB);
      float R_BA[9], t_BA[3], R_AB[9], t_AB[3];
      relative(qA, pA + 4, qB, pB + 4, R_BA, t_BA);
      relative(qB, pB + 4, qA, pA + 4, R_AB, t_AB);
      const int nA = select_cells(shapes[a], M, R_BA, t_BA, shapes[b], selA);
      const int nB = select_cells(shapes[b], M, R_AB, t_AB, shapes[a], selB);
      if (nsel) {
        nsel[2 * i] = nA;
        nsel[2 * i + 1] = nB;
      }
      if (cells) {
        uint32_t* mA = cells + (2 * i) * words;
        uint32_t* mB = mA + words;
        std::memset(mA, 0, sizeof(uint32_t) * 2 * words);
        for (int c = 0; c < ncell; ++c) {
          if (selA[c]) mA[c / 32] |= 1u << (c % 32);
          if (selB[c]) mB[c / 32] |= 1u << (c % 32);
        }
      }
      // P:337 "average pooling" of the selected cells' features (ascending cell order); 0 if none
      auto pool_sel = [&](const std::vector<double>& Es, const std::vector<uint8_t>& sel, int n, double* e) {
        for (int f = 0; f < F; ++f) e[f] = 0.0;
        if (n == 0) return;
        for (int c = 0; c < ncell; ++c)
          if (sel[c])
            for (int f = 0; f < F; ++f) e[f] += Es[(int64_t)c * F + f];
        for (int f = 0; f < F; ++f) e[f] /= (double)n;
      };
      double logit, prob;
      if (nA + nB == 0) {  // disjoint: short-circuit
        for (int f = 0; f < F; ++f) eA[f] = eB[f] = 0.0;
        logit = -INFINITY;
        prob = 0.0;
      } else {
        pool_sel(E[a], selA, nA, eA.data());
        pool_sel(E[b], selB, nB, eB.data());
        object_mlp(P, eA.data(), F, qA, pA + 4, uA.data());
        object_mlp(P, eB.data(), F, qB, pB + 4, uB.data());
        logit = pair_head(P, uA.data(), uB.data());
        prob = 1.0 / (1.0 + std::exp(-logit));
      }
      if (emb)
        for (int f = 0; f < F; ++f) {
          emb[(2 * i) * F + f] = eA[f];
          emb[(2 * i + 1) * F + f] = eB[f];
        }
      if (probs) probs[i] = prob;
      if (logits) logits[i] = logit;
      if (labels) labels[i] = prob > 0.5 ? 1 : 0;
    }
  };
  int nq = nt;
  if (nq > N) nq = (int)(N > 0 ? N : 1);
  std::vector<std::thread> pool;
  for (int t = 1; t < nq; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  return 0;
}

int oracle_sim_run(const oracle_cfg* cfg, const float* weights, size_t n_weights, const float* unet_w,
                   size_t n_unet, const float* points, int32_t S, int32_t K, const double* sim, int32_t E,
                   const int32_t* ids, const double* body, double* state, double t0, int32_t* contacts,
                   double* margins) {
  if (!cfg || !sim || E < 0 || !ids || !body || !state) return -1;
  SimCfg c;
  c.h = sim[0];
  c.substeps = (int32_t)sim[1];
  c.detector = (int32_t)sim[2];
  for (int i = 0; i < 3; ++i) c.gravity[i] = sim[3 + i];
  c.ks = sim[6];
  c.kd = sim[7];
  for (int i = 0; i < 3; ++i) c.amp[i] = sim[8 + i];
  c.freq = sim[11];
  c.slack = sim[12];
  if (!(c.h > 0.0) || c.substeps < 1) return -1;
  if (c.detector == 1 && (!unet_w || (int64_t)n_unet != unet_n_params(cfg->H, cfg->F))) return -3;
  const int M = cfg->M, H = cfg->H, F = cfg->F, ncell = M * M * M;
  if (!weights || (int64_t)n_weights != n_params(H, F)) return -3;
  std::vector<ShapeInfo> shapes(S);
  for (int s = 0; s < S; ++s)
    if (!shape_prep(points + (int64_t)s * K * 3, K, M, shapes[s])) return -2;
  const Params P = bind_params(weights, H, F);
  // encode-once detector: the referenced grids, once per call
  std::vector<std::vector<double>> grids(S);
  if (c.detector == 1) {
    const EncW EW{widen(P.enc1, false), widen(P.enc2, false), widen(P.enc3, false), widen(P.proj, false)};
    const UNetW U = bind_unet(unet_w, H, F);
    std::vector<uint8_t> used(S, 0);
    for (int64_t i = 0; i < 3 * (int64_t)E; ++i) used[ids[i]] = 1;
    std::vector<double> g;
    for (int s = 0; s < S; ++s)
      if (used[s]) {
        grid_maxpool(P, EW, points + (int64_t)s * K * 3, K, shapes[s], M, H, g);
        unet(U, g, M, H, F, grids[s], cfg->global_max != 0);
      }
  }
  const int pa_[3] = {0, 0, 1}, pb_[3] = {1, 2, 2};
  const int64_t NP = 3 * (int64_t)E;
  std::vector<int32_t> pairs(2 * NP);
  std::vector<float> poses(14 * NP);
  std::vector<double> lg(NP), gr(14 * NP), mg(NP);
  std::vector<uint8_t> culled(NP);
  if (contacts)
    for (int64_t i = 0; i < NP; ++i) contacts[i] = 0;
  if (margins)
    for (int64_t i = 0; i < 4 * (int64_t)E; ++i) margins[i] = INFINITY;
  for (int n = 0; n < c.substeps; ++n) {
    const double tau = t0 + n * c.h, w2 = 2.0 * M_PI * c.freq;
    for (int e = 0; e < E; ++e) {  // 1. the kinematic bowl
      double* b = state + (int64_t)e * 39;
      for (int i = 0; i < 3; ++i) {
        b[4 + i] = c.amp[i] * std::sin(w2 * tau);
        b[7 + i] = c.amp[i] * w2 * std::cos(w2 * tau);
        b[10 + i] = 0.0;
      }
    }
    for (int e = 0; e < E; ++e)  // 2. broad phase + the detector's inputs
      for (int p = 0; p < 3; ++p) {
        const int64_t i = 3 * (int64_t)e + p;
        const double* X[2] = {state + (int64_t)e * 39 + 13 * pa_[p], state + (int64_t)e * 39 + 13 * pb_[p]};
        double cw[2][3], hw[2][3];
        for (int side = 0; side < 2; ++side) {
          const int sid = ids[3 * e + (side ? pb_[p] : pa_[p])];
          pairs[2 * i + side] = sid;
          for (int j = 0; j < 7; ++j) poses[14 * i + 7 * side + j] = (float)X[side][j];
          const ShapeInfo& sh = shapes[sid];
          double q[4] = {X[side][0], X[side][1], X[side][2], X[side][3]}, R[3][3];
          const double nq = std::sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
          rotmat(Quat{q[0] / nq, q[1] / nq, q[2] / nq, q[3] / nq}, R);
          for (int r = 0; r < 3; ++r) {
            cw[side][r] = X[side][4 + r];
            hw[side][r] = 0.0;
            for (int k = 0; k < 3; ++k) {
              const double cl = 0.5 * ((double)sh.lo[k] + (double)sh.hi[k]), hl = 0.5 * ((double)sh.hi[k] - (double)sh.lo[k]);
              cw[side][r] += R[r][k] * cl;
              hw[side][r] += std::fabs(R[r][k]) * hl;
            }
          }
        }
        double gmax = -INFINITY;  // culled iff some axis separates: max gap > 0
        for (int r = 0; r < 3; ++r)
          gmax = std::max(gmax, std::fabs(cw[0][r] - cw[1][r]) - (hw[0][r] + hw[1][r] + c.slack));
        culled[i] = gmax > 0.0;
        if (margins) margins[4 * e + 2] = std::min(margins[4 * e + 2], std::fabs(gmax));
      }
    // 3. detector
    if (c.detector == 0) {
      const int rc = oracle_query_grad(cfg, weights, n_weights, points, S, K, pairs.data(), poses.data(), NP,
                                       lg.data(), gr.data(), mg.data());
      if (rc) return rc;
    } else {
      for (int64_t i = 0; i < NP; ++i) {
        const int a = pairs[2 * i], b = pairs[2 * i + 1];
        const float* pA = &poses[14 * i];
        const float* pB = pA + 7;
        Quat qA, qB;
        if (!normalise(pA, qA) || !normalise(pB, qB)) return -1;
        float R_BA[9], t_BA[3], R_AB[9], t_AB[3];
        relative(qA, pA + 4, qB, pB + 4, R_BA, t_BA);
        relative(qB, pB + 4, qA, pA + 4, R_AB, t_AB);
        std::vector<uint8_t> sA, sB;
        const int nA = select_cells(shapes[a], M, R_BA, t_BA, shapes[b], sA);
        const int nB = select_cells(shapes[b], M, R_AB, t_AB, shapes[a], sB);
        double* g = &gr[14 * i];
        if (nA + nB == 0) {
          lg[i] = -INFINITY;
          for (int j = 0; j < 14; ++j) g[j] = 0.0;
          mg[i] = INFINITY;
          continue;
        }
        std::vector<double> eA(F, 0.0), eB(F, 0.0);
        for (int cc = 0; cc < ncell; ++cc) {
          if (sA[cc])
            for (int f = 0; f < F; ++f) eA[f] += grids[a][(int64_t)cc * F + f];
          if (sB[cc])
            for (int f = 0; f < F; ++f) eB[f] += grids[b][(int64_t)cc * F + f];
        }
        for (int f = 0; f < F; ++f) {
          if (nA) eA[f] /= (double)nA;
          if (nB) eB[f] /= (double)nB;
        }
        double da[7], db[7];
        for (int j = 0; j < 7; ++j) {
          da[j] = pA[j];
          db[j] = pB[j];
        }
        lg[i] = head_grad(P, eA.data(), eB.data(), F, da, da + 4, db, db + 4, g, &mg[i]);
      }
    }
    // 4.-6. contacts, penalty, integration
    for (int e = 0; e < E; ++e) {
      double Fo[3][3] = {}, To[3][3] = {};
      double* st = state + (int64_t)e * 39;
      for (int p = 0; p < 3; ++p) {
        const int64_t i = 3 * (int64_t)e + p;
        if (culled[i]) continue;
        if (margins) {
          margins[4 * e] = std::min(margins[4 * e], std::fabs(lg[i]));
          margins[4 * e + 1] = std::min(margins[4 * e + 1], mg[i]);
        }
        if (!(lg[i] > 0.0)) continue;
        if (contacts) ++contacts[i];
        const int bx[2] = {pa_[p], pb_[p]};
        double gt[2][3], gw[2][3], nrm2 = 0.0, sdot = 0.0;
        for (int side = 0; side < 2; ++side) {
          const double* g = &gr[14 * i + 7 * side];
          const double* X = st + 13 * bx[side];
          for (int k = 0; k < 3; ++k) {
            double d[4];
            quat_left_e(X, k, d);
            gw[side][k] = 0.5 * (((g[0] * d[0] + g[1] * d[1]) + g[2] * d[2]) + g[3] * d[3]);
            gt[side][k] = g[4 + k];
            nrm2 += gt[side][k] * gt[side][k] + gw[side][k] * gw[side][k];
            sdot += gt[side][k] * X[7 + k] + gw[side][k] * X[10 + k];
          }
        }
        const double nrm = std::sqrt(nrm2);
        if (!(nrm > 1e-12)) continue;
        const double raw = c.ks * lg[i] + c.kd * sdot;
        if (margins) margins[4 * e + 3] = std::min(margins[4 * e + 3], std::fabs(raw));
        const double lam = raw > 0.0 ? raw : 0.0;
        for (int side = 0; side < 2; ++side)
          for (int k = 0; k < 3; ++k) {
            Fo[bx[side]][k] -= lam * gt[side][k] / nrm;
            To[bx[side]][k] -= lam * gw[side][k] / nrm;
          }
      }
      for (int bi = 1; bi < 3; ++bi) {
        double* X = st + 13 * bi;
        const double* bd = body + ((int64_t)e * 3 + bi) * 4;  // m, Ixx, Iyy, Izz
        double q[4] = {X[0], X[1], X[2], X[3]}, R[3][3];
        const double nq = std::sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
        rotmat(Quat{q[0] / nq, q[1] / nq, q[2] / nq, q[3] / nq}, R);
        double tb[3], dw[3];
        for (int k = 0; k < 3; ++k) tb[k] = (R[0][k] * To[bi][0] + R[1][k] * To[bi][1]) + R[2][k] * To[bi][2];
        for (int k = 0; k < 3; ++k) tb[k] /= bd[1 + k];
        for (int r = 0; r < 3; ++r) dw[r] = (R[r][0] * tb[0] + R[r][1] * tb[1]) + R[r][2] * tb[2];
        for (int k = 0; k < 3; ++k) {
          X[7 + k] += c.h * (Fo[bi][k] / bd[0] + c.gravity[k]);
          X[10 + k] += c.h * dw[k];
        }
        for (int k = 0; k < 3; ++k) X[4 + k] += c.h * X[7 + k];
        const Quat wq = hamilton(Quat{0.0, X[10], X[11], X[12]}, Quat{q[0], q[1], q[2], q[3]});
        double qn[4] = {q[0] + 0.5 * c.h * wq.w, q[1] + 0.5 * c.h * wq.x, q[2] + 0.5 * c.h * wq.y,
                        q[3] + 0.5 * c.h * wq.z};
        const double nn = std::sqrt(((qn[0] * qn[0] + qn[1] * qn[1]) + qn[2] * qn[2]) + qn[3] * qn[3]);
        for (int k = 0; k < 4; ++k) X[k] = qn[k] / nn;
      }
    }
  }
  const double tau = t0 + c.substeps * c.h, w2 = 2.0 * M_PI * c.freq;  // the bowl at the end time
  for (int e = 0; e < E; ++e) {
    double* b = state + (int64_t)e * 39;
    for (int i = 0; i < 3; ++i) {
      b[4 + i] = c.amp[i] * std::sin(w2 * tau);
      b[7 + i] = c.amp[i] * w2 * std::cos(w2 * tau);
      b[10 + i] = 0.0;
    }
  }
  return 0;
}

int64_t oracle_load_weights(const char* manifest, float* out, size_t cap, int32_t* M, int32_t* H,
                            int32_t* F) {
  FILE* f = std::fopen(manifest, "r");
  if (!f) return -3;
  char magic[64];
  int ver = 0;
  if (std::fscanf(f, "%63s %d %d %d %d", magic, &ver, M, H, F) != 5 || std::string(magic) != "locc-weights" ||
      ver != 1) {
    std::fclose(f);
    return -3;
  }
  const char* names[] = {"enc.l1", "enc.l2", "enc.l3", "enc.proj", "obj.l1", "obj.l2",
                         "obj.l3", "pair.l1", "pair.l2", "pair.l3", "out"};
  const int h = *H, fo = *F;
  const int shp[11][2] = {{h, 3}, {h, h}, {h, h}, {fo, h}, {kP, fo + 7}, {kP, kP},
                          {kP, kP}, {kP, kP}, {kP, kP}, {kP, kP}, {1, kP}};
  std::string bin(manifest);
  size_t dot = bin.find_last_of('.');
  size_t slash = bin.find_last_of('/');
  if (dot != std::string::npos && (slash == std::string::npos || dot > slash)) bin = bin.substr(0, dot);
  bin += ".bin";
  FILE* fb = std::fopen(bin.c_str(), "rb");
  if (!fb) {
    std::fclose(f);
    return -3;
  }
  int64_t total = n_params(h, fo);
  if ((int64_t)cap < total) {
    std::fclose(f);
    std::fclose(fb);
    return -3;
  }
  int64_t pos = 0;
  for (int l = 0; l < 11; ++l)
    for (int wb = 0; wb < 2; ++wb) {
      char name[128];
      long long o, in, off;
      if (std::fscanf(f, "%127s %lld %lld %lld", name, &o, &in, &off) != 4) goto bad;
      std::string want = std::string(names[l]) + (wb == 0 ? ".W" : ".b");
      long long eo = shp[l][0], ei = wb == 0 ? shp[l][1] : 1;
      if (want != name || o != eo || in != ei) goto bad;
      if (std::fseek(fb, (long)off, SEEK_SET) != 0) goto bad;
      if ((long long)std::fread(out + pos, sizeof(float), (size_t)(o * in), fb) != o * in) goto bad;
      pos += o * in;
    }
  std::fclose(f);
  std::fclose(fb);
  return pos;
bad:
  std::fclose(f);
  std::fclose(fb);
  return -3;
}

}  // extern "C"
