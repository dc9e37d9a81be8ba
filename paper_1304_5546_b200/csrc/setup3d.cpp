// Host fp64 setup of the 3D tetrahedral Maxwell operator.
//
// Reference tetrahedron (the 2D construction of setup.cpp one dimension up):
//   * warp-and-blend nodes (warburton_explicit_2006, cited at PAPER.md:278-279): equispaced
//     barycentric points of the equilateral tetrahedron, each face's 2D warp (setup.cpp warpfactor)
//     blended into the interior with the 3D alpha table, mapped to (r, s, t); t slowest, r fastest;
//   * orthonormal modes phi_ijk in collapsed coordinates, V, Vr, Vs, Vt; D = V_d V^-1;
//   * M = (V V^T)^-1; face mass (V2D V2D^T)^-1 with the triangle basis on each face's own two
//     coordinates; LIFT = V (V^T E).
// Mesh: faces f0 (v0,v1,v2), f1 (v0,v1,v3), f2 (v1,v2,v3), f3 (v0,v2,v3) matched by sorted vertex
// triple; rx..tz = the inverse Jacobian; outward normals -grad t, -grad s, grad(r+s+t), -grad r;
// sJ = J |n| (= face area / 2), Fsc = sJ / J; vmapP by the face nodes' barycentric weights on the
// shared global vertices (exact), verified against coordinates.
#include "setup3d.h"

#include <algorithm>
#include <array>
#include <cmath>

#include "../../include/dg.h"

namespace dg {

namespace {

[[noreturn]] void fail3(int st, const std::string& m) { throw SetupError{st, m}; }

const double kAlpha3[15] = {0.0, 0.0, 0.0, 0.1002, 1.1332, 1.5608, 1.3413, 1.2577,
                            1.1603, 1.10153, 0.6080, 0.4523, 0.8856, 0.8717, 0.9655};
const int kFaceVerts[4][3] = {{0, 1, 2}, {0, 1, 3}, {1, 2, 3}, {0, 2, 3}};

// the 2D warp-and-blend shift of points with face barycentrics (L1, L2, L3)
void face_shift(int n, double alpha, const std::vector<double>& L1, const std::vector<double>& L2,
                const std::vector<double>& L3, std::vector<double>& dx, std::vector<double>& dy) {
  const size_t m = L1.size();
  std::vector<double> a1(m), a2(m), a3(m);
  for (size_t i = 0; i < m; ++i) {
    a1[i] = L3[i] - L2[i];
    a2[i] = L1[i] - L3[i];
    a3[i] = L2[i] - L1[i];
  }
  const auto w1 = warpfactor(n, a1), w2 = warpfactor(n, a2), w3 = warpfactor(n, a3);
  dx.resize(m);
  dy.resize(m);
  for (size_t i = 0; i < m; ++i) {
    const double f1 = 4.0 * L2[i] * L3[i] * w1[i] * (1.0 + alpha * alpha * L1[i] * L1[i]);
    const double f2 = 4.0 * L1[i] * L3[i] * w2[i] * (1.0 + alpha * alpha * L2[i] * L2[i]);
    const double f3 = 4.0 * L1[i] * L2[i] * w3[i] * (1.0 + alpha * alpha * L3[i] * L3[i]);
    dx[i] = f1 + std::cos(2.0 * M_PI / 3.0) * f2 + std::cos(4.0 * M_PI / 3.0) * f3;
    dy[i] = std::sin(2.0 * M_PI / 3.0) * f2 + std::sin(4.0 * M_PI / 3.0) * f3;
  }
}

void nodes3D(int n, std::vector<double>& r, std::vector<double>& s, std::vector<double>& t) {
  const double alpha = n <= 15 ? kAlpha3[n - 1] : 1.0;
  const double tol = 1e-10;
  std::vector<double> L[4];  // L[0] = (1+t)/2, L[1] = (1+s)/2, L[2] = -(1+r+s+t)/2, L[3] = (1+r)/2
  for (int k = 0; k <= n; ++k)
    for (int j = 0; j <= n - k; ++j)
      for (int i = 0; i <= n - k - j; ++i) {
        const double rr = -1.0 + 2.0 * i / n, ss = -1.0 + 2.0 * j / n, tt = -1.0 + 2.0 * k / n;
        L[0].push_back((1.0 + tt) / 2.0);
        L[1].push_back((1.0 + ss) / 2.0);
        L[2].push_back(-(1.0 + rr + ss + tt) / 2.0);
        L[3].push_back((1.0 + rr) / 2.0);
      }
  const size_t Np = L[0].size();
  const double q3 = std::sqrt(3.0), q6 = std::sqrt(6.0);
  const std::array<double, 3> v[4] = {{-1.0, -1.0 / q3, -1.0 / q6}, {1.0, -1.0 / q3, -1.0 / q6},
                                      {0.0, 2.0 / q3, -1.0 / q6}, {0.0, 0.0, 3.0 / q6}};
  auto sub = [](std::array<double, 3> a, std::array<double, 3> b) {
    return std::array<double, 3>{a[0] - b[0], a[1] - b[1], a[2] - b[2]};
  };
  auto mid = [](std::array<double, 3> a, std::array<double, 3> b) {
    return std::array<double, 3>{0.5 * (a[0] + b[0]), 0.5 * (a[1] + b[1]), 0.5 * (a[2] + b[2])};
  };
  auto unit = [](std::array<double, 3> a) {
    const double l = std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    return std::array<double, 3>{a[0] / l, a[1] / l, a[2] / l};
  };
  const std::array<double, 3> t1[4] = {unit(sub(v[1], v[0])), unit(sub(v[1], v[0])), unit(sub(v[2], v[1])),
                                       unit(sub(v[2], v[0]))};
  const std::array<double, 3> t2[4] = {unit(sub(v[2], mid(v[0], v[1]))), unit(sub(v[3], mid(v[0], v[1]))),
                                       unit(sub(v[3], mid(v[1], v[2]))), unit(sub(v[3], mid(v[0], v[2])))};
  std::vector<std::array<double, 3>> X(Np), shift(Np, {0.0, 0.0, 0.0});
  for (size_t i = 0; i < Np; ++i)
    for (int d = 0; d < 3; ++d)
      X[i][d] = L[2][i] * v[0][d] + L[3][i] * v[1][d] + L[1][i] * v[2][d] + L[0][i] * v[3][d];
  // faces: (La, Lb, Lc, Ld) = (L1,L2,L3,L4), (L2,L1,L3,L4), (L3,L1,L4,L2), (L4,L1,L3,L2) in 1-based L
  const int order[4][4] = {{0, 1, 2, 3}, {1, 0, 2, 3}, {2, 0, 3, 1}, {3, 0, 2, 1}};
  for (int f = 0; f < 4; ++f) {
    const auto &La = L[order[f][0]], &Lb = L[order[f][1]], &Lc = L[order[f][2]], &Ld = L[order[f][3]];
    std::vector<double> w1, w2;
    face_shift(n, alpha, Lb, Lc, Ld, w1, w2);
    for (size_t i = 0; i < Np; ++i) {
      double blend = Lb[i] * Lc[i] * Ld[i];
      const double denom = (Lb[i] + 0.5 * La[i]) * (Lc[i] + 0.5 * La[i]) * (Ld[i] + 0.5 * La[i]);
      if (denom > tol) blend = (1.0 + (alpha * La[i]) * (alpha * La[i])) * blend / denom;
      const int inside = (Lb[i] > tol) + (Lc[i] > tol) + (Ld[i] > tol);
      if (La[i] < tol && inside < 3) {
        for (int d = 0; d < 3; ++d) shift[i][d] = w1[i] * t1[f][d] + w2[i] * t2[f][d];
      } else {
        for (int d = 0; d < 3; ++d) shift[i][d] += blend * w1[i] * t1[f][d] + blend * w2[i] * t2[f][d];
      }
    }
  }
  // equilateral -> reference: X - (v1+v2+v3-v0)/2 = [ (v1-v0)/2 (v2-v0)/2 (v3-v0)/2 ] (r,s,t)
  std::vector<double> A(9);
  for (int d = 0; d < 3; ++d)
    for (int c = 0; c < 3; ++c) A[d * 3 + c] = 0.5 * (v[c + 1][d] - v[0][d]);
  std::vector<double> B(3 * Np);
  for (size_t i = 0; i < Np; ++i)
    for (int d = 0; d < 3; ++d)
      B[d * Np + i] = X[i][d] + shift[i][d] - 0.5 * (v[1][d] + v[2][d] + v[3][d] - v[0][d]);
  lu_solve(3, A, (int)Np, B);
  r.assign(B.begin(), B.begin() + Np);
  s.assign(B.begin() + Np, B.begin() + 2 * Np);
  t.assign(B.begin() + 2 * Np, B.end());
}

// orthonormal tetrahedron mode phi_ijk and its gradient (collapsed coordinates, chain rule)
void tet_mode(const std::vector<double>& r, const std::vector<double>& s, const std::vector<double>& t, int i, int j,
              int k, double* phi, double* dr, double* ds, double* dt) {
  const int n = (int)r.size();
  std::vector<double> a(n), b(n), c(n), fa(n), dfa(n), gb(n), dgb(n), hc(n), dhc(n);
  for (int q = 0; q < n; ++q) {
    a[q] = (s[q] + t[q] != 0.0) ? 2.0 * (1.0 + r[q]) / (-s[q] - t[q]) - 1.0 : -1.0;
    b[q] = (t[q] != 1.0) ? 2.0 * (1.0 + s[q]) / (1.0 - t[q]) - 1.0 : -1.0;
    c[q] = t[q];
  }
  jacobiP(a.data(), n, 0, 0, i, fa.data());
  gradJacobiP(a.data(), n, 0, 0, i, dfa.data());
  jacobiP(b.data(), n, 2.0 * i + 1, 0, j, gb.data());
  gradJacobiP(b.data(), n, 2.0 * i + 1, 0, j, dgb.data());
  jacobiP(c.data(), n, 2.0 * (i + j) + 2, 0, k, hc.data());
  gradJacobiP(c.data(), n, 2.0 * (i + j) + 2, 0, k, dhc.data());
  const double scale = std::pow(2.0, 2 * i + j + 1.5);
  for (int q = 0; q < n; ++q) {
    const double hb = 0.5 * (1.0 - b[q]), hcq = 0.5 * (1.0 - c[q]);
    if (phi) phi[q] = 2.0 * std::sqrt(2.0) * fa[q] * gb[q] * std::pow(1.0 - b[q], i) * hc[q] * std::pow(1.0 - c[q], i + j);
    double vr = dfa[q] * gb[q] * hc[q];
    if (i > 0) vr *= std::pow(hb, i - 1);
    if (i + j > 0) vr *= std::pow(hcq, i + j - 1);
    double tmp = dgb[q] * std::pow(hb, i);
    if (i > 0) tmp -= 0.5 * i * gb[q] * std::pow(hb, i - 1);
    if (i + j > 0) tmp *= std::pow(hcq, i + j - 1);
    tmp = fa[q] * tmp * hc[q];
    const double vs = 0.5 * (1.0 + a[q]) * vr + tmp;
    double vt = 0.5 * (1.0 + a[q]) * vr + 0.5 * (1.0 + b[q]) * tmp;
    double tc = dhc[q] * std::pow(hcq, i + j);
    if (i + j > 0) tc -= 0.5 * (i + j) * hc[q] * std::pow(hcq, i + j - 1);
    vt += fa[q] * gb[q] * tc * std::pow(hb, i);
    if (dr) dr[q] = scale * vr;
    if (ds) ds[q] = scale * vs;
    if (dt) dt[q] = scale * vt;
  }
}

std::vector<double> transpose(const std::vector<double>& A, int n) {
  std::vector<double> T(A.size());
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) T[i * n + j] = A[j * n + i];
  return T;
}

}  // namespace

RefTet build_reftet(int N) {
  if (N < 1 || N > 15) fail3(DG_E_DEGREE, "degree N must be in [1, 15]");
  RefTet R;
  R.N = N;
  R.Np = (N + 1) * (N + 2) * (N + 3) / 6;
  R.Nfp = (N + 1) * (N + 2) / 2;
  const int Np = R.Np, Nfp = R.Nfp;
  nodes3D(N, R.r, R.s, R.t);
  if ((int)R.r.size() != Np) fail3(DG_E_STATE, "3D node count");
  R.V.assign(Np * Np, 0.0);
  std::vector<double> Vd[3] = {std::vector<double>(Np * Np), std::vector<double>(Np * Np),
                               std::vector<double>(Np * Np)};
  std::vector<double> phi(Np), d0(Np), d1(Np), d2(Np);
  int col = 0;
  for (int i = 0; i <= N; ++i)
    for (int j = 0; j <= N - i; ++j)
      for (int k = 0; k <= N - i - j; ++k, ++col) {
        tet_mode(R.r, R.s, R.t, i, j, k, phi.data(), d0.data(), d1.data(), d2.data());
        for (int q = 0; q < Np; ++q) {
          R.V[q * Np + col] = phi[q];
          Vd[0][q * Np + col] = d0[q];
          Vd[1][q * Np + col] = d1[q];
          Vd[2][q * Np + col] = d2[q];
        }
      }
  const std::vector<double> VT = transpose(R.V, Np);
  std::vector<double>* D[3] = {&R.Dr, &R.Ds, &R.Dt};
  for (int d = 0; d < 3; ++d) {  // V^T D^T = Vd^T
    std::vector<double> X = transpose(Vd[d], Np);
    lu_solve(Np, VT, Np, X);
    *D[d] = transpose(X, Np);
  }
  std::vector<double> VVt(Np * Np, 0.0);
  for (int i = 0; i < Np; ++i)
    for (int j = 0; j < Np; ++j) {
      double acc = 0.0;
      for (int k = 0; k < Np; ++k) acc += R.V[i * Np + k] * R.V[j * Np + k];
      VVt[i * Np + j] = acc;
    }
  R.M.assign(Np * Np, 0.0);
  for (int i = 0; i < Np; ++i) R.M[i * Np + i] = 1.0;
  lu_solve(Np, VVt, Np, R.M);
  R.Fmask.assign(4 * Nfp, -1);
  int cnt[4] = {0, 0, 0, 0};
  for (int q = 0; q < Np; ++q) {
    const bool on[4] = {std::fabs(1.0 + R.t[q]) < 1e-10, std::fabs(1.0 + R.s[q]) < 1e-10,
                        std::fabs(1.0 + R.r[q] + R.s[q] + R.t[q]) < 1e-10, std::fabs(1.0 + R.r[q]) < 1e-10};
    for (int f = 0; f < 4; ++f)
      if (on[f]) {
        if (cnt[f] >= Nfp) fail3(DG_E_DEGREE, "3D face mask overflow");
        R.Fmask[f * Nfp + cnt[f]++] = q;
      }
  }
  for (int f = 0; f < 4; ++f)
    if (cnt[f] != Nfp) fail3(DG_E_DEGREE, "3D face mask incomplete");
  // E [Np][4 Nfp]: face mass (V2D V2D^T)^-1 on each face's own two coordinates
  std::vector<double> E(Np * 4 * Nfp, 0.0);
  for (int f = 0; f < 4; ++f) {
    std::vector<double> fu(Nfp), fv(Nfp);
    for (int i = 0; i < Nfp; ++i) {
      const int q = R.Fmask[f * Nfp + i];
      fu[i] = (f == 0 || f == 1) ? R.r[q] : R.s[q];
      fv[i] = f == 0 ? R.s[q] : R.t[q];
    }
    std::vector<double> V2(Nfp * Nfp), m(Nfp);
    int c2 = 0;
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j, ++c2) {
        simplex_mode(fu, fv, i, j, m.data(), nullptr, nullptr);
        for (int q = 0; q < Nfp; ++q) V2[q * Nfp + c2] = m[q];
      }
    std::vector<double> VV(Nfp * Nfp, 0.0), Mf(Nfp * Nfp, 0.0);
    for (int i = 0; i < Nfp; ++i)
      for (int j = 0; j < Nfp; ++j) {
        double acc = 0.0;
        for (int k = 0; k < Nfp; ++k) acc += V2[i * Nfp + k] * V2[j * Nfp + k];
        VV[i * Nfp + j] = acc;
      }
    for (int i = 0; i < Nfp; ++i) Mf[i * Nfp + i] = 1.0;
    lu_solve(Nfp, VV, Nfp, Mf);
    for (int i = 0; i < Nfp; ++i)
      for (int j = 0; j < Nfp; ++j) E[R.Fmask[f * Nfp + i] * (4 * Nfp) + f * Nfp + j] = Mf[i * Nfp + j];
  }
  const int NF = 4 * Nfp;
  std::vector<double> VtE(Np * NF, 0.0);
  for (int i = 0; i < Np; ++i)
    for (int k = 0; k < Np; ++k) {
      const double vv = R.V[k * Np + i];
      for (int j = 0; j < NF; ++j) VtE[i * NF + j] += vv * E[k * NF + j];
    }
  R.LIFT.assign(Np * NF, 0.0);
  for (int i = 0; i < Np; ++i)
    for (int k = 0; k < Np; ++k) {
      const double vv = R.V[i * Np + k];
      for (int j = 0; j < NF; ++j) R.LIFT[i * NF + j] += vv * VtE[k * NF + j];
    }
  return R;
}

void element_nodes3d(const RefTet& ref, const Mesh3D& m, int64_t k, double* x, double* y, double* z) {
  const int64_t* v = &m.EToV[4 * k];
  for (int i = 0; i < ref.Np; ++i) {
    const double w0 = -(1.0 + ref.r[i] + ref.s[i] + ref.t[i]) / 2, w1 = (1.0 + ref.r[i]) / 2,
                 w2 = (1.0 + ref.s[i]) / 2, w3 = (1.0 + ref.t[i]) / 2;
    x[i] = w0 * m.VX[v[0]] + w1 * m.VX[v[1]] + w2 * m.VX[v[2]] + w3 * m.VX[v[3]];
    y[i] = w0 * m.VY[v[0]] + w1 * m.VY[v[1]] + w2 * m.VY[v[2]] + w3 * m.VY[v[3]];
    z[i] = w0 * m.VZ[v[0]] + w1 * m.VZ[v[1]] + w2 * m.VZ[v[2]] + w3 * m.VZ[v[3]];
  }
}

void build_mesh3d(const RefTet& ref, int64_t Nv, const double* VX, const double* VY, const double* VZ, int64_t K,
                  const int64_t* EToV, Mesh3D& m) {
  if (K < 1 || Nv < 4) fail3(DG_E_ARG, "empty mesh");
  m.K = K;
  m.Nv = Nv;
  m.VX.assign(VX, VX + Nv);
  m.VY.assign(VY, VY + Nv);
  m.VZ.assign(VZ, VZ + Nv);
  m.EToV.assign(EToV, EToV + 4 * K);
  for (int64_t i = 0; i < 4 * K; ++i)
    if (m.EToV[i] < 0 || m.EToV[i] >= Nv) fail3(DG_E_ARG, "EToV vertex id out of range");
  // geometry (re-orienting negative elements by swapping local vertices 1 <-> 2)
  const int Np = ref.Np, Nfp = ref.Nfp;
  for (auto* vec : {&m.rx, &m.ry, &m.rz, &m.sx, &m.sy, &m.sz, &m.tx, &m.ty, &m.tz, &m.J}) vec->assign(K, 0.0);
  for (auto* vec : {&m.nx, &m.ny, &m.nz, &m.sJ, &m.Fsc}) vec->assign(4 * K, 0.0);
  for (int64_t k = 0; k < K; ++k) {
    int64_t* v = &m.EToV[4 * k];
    auto jac = [&](double A[3][3]) {
      const double* C[3] = {VX, VY, VZ};
      for (int d = 0; d < 3; ++d)
        for (int c = 0; c < 3; ++c) A[d][c] = 0.5 * (C[d][v[c + 1]] - C[d][v[0]]);
      return A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
             A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
    };
    double A[3][3];
    double J = jac(A);
    if (J < 0) {
      std::swap(v[1], v[2]);
      ++m.n_swapped;
      J = jac(A);
    }
    double hmax = 0.0;
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b)
        hmax = std::max(hmax, std::hypot(std::hypot(VX[v[a]] - VX[v[b]], VY[v[a]] - VY[v[b]]), VZ[v[a]] - VZ[v[b]]));
    if (!(J > 1e-14 * hmax * hmax * hmax)) fail3(DG_E_MESH_DEGENERATE, "degenerate tetrahedron");
    // inverse Jacobian: rows grad r, grad s, grad t (cofactors / J)
    const double inv[3][3] = {{(A[1][1] * A[2][2] - A[1][2] * A[2][1]) / J, (A[0][2] * A[2][1] - A[0][1] * A[2][2]) / J,
                               (A[0][1] * A[1][2] - A[0][2] * A[1][1]) / J},
                              {(A[1][2] * A[2][0] - A[1][0] * A[2][2]) / J, (A[0][0] * A[2][2] - A[0][2] * A[2][0]) / J,
                               (A[0][2] * A[1][0] - A[0][0] * A[1][2]) / J},
                              {(A[1][0] * A[2][1] - A[1][1] * A[2][0]) / J, (A[0][1] * A[2][0] - A[0][0] * A[2][1]) / J,
                               (A[0][0] * A[1][1] - A[0][1] * A[1][0]) / J}};
    m.rx[k] = inv[0][0]; m.ry[k] = inv[0][1]; m.rz[k] = inv[0][2];
    m.sx[k] = inv[1][0]; m.sy[k] = inv[1][1]; m.sz[k] = inv[1][2];
    m.tx[k] = inv[2][0]; m.ty[k] = inv[2][1]; m.tz[k] = inv[2][2];
    m.J[k] = J;
    const double nraw[4][3] = {{-inv[2][0], -inv[2][1], -inv[2][2]},
                               {-inv[1][0], -inv[1][1], -inv[1][2]},
                               {inv[0][0] + inv[1][0] + inv[2][0], inv[0][1] + inv[1][1] + inv[2][1],
                                inv[0][2] + inv[1][2] + inv[2][2]},
                               {-inv[0][0], -inv[0][1], -inv[0][2]}};
    for (int f = 0; f < 4; ++f) {
      const double l = std::sqrt(nraw[f][0] * nraw[f][0] + nraw[f][1] * nraw[f][1] + nraw[f][2] * nraw[f][2]);
      m.nx[4 * k + f] = nraw[f][0] / l;
      m.ny[4 * k + f] = nraw[f][1] / l;
      m.nz[4 * k + f] = nraw[f][2] / l;
      m.sJ[4 * k + f] = l * J;
      m.Fsc[4 * k + f] = l;
    }
  }
  // connectivity: sort (sorted vertex triple, element, face) records
  struct Rec { std::array<int64_t, 3> key; int64_t k; int f; };
  std::vector<Rec> recs;
  recs.reserve(4 * K);
  for (int64_t k = 0; k < K; ++k)
    for (int f = 0; f < 4; ++f) {
      std::array<int64_t, 3> key = {m.EToV[4 * k + kFaceVerts[f][0]], m.EToV[4 * k + kFaceVerts[f][1]],
                                    m.EToV[4 * k + kFaceVerts[f][2]]};
      std::sort(key.begin(), key.end());
      recs.push_back({key, k, f});
    }
  std::sort(recs.begin(), recs.end(), [](const Rec& a, const Rec& b) {
    return a.key != b.key ? a.key < b.key : (a.k != b.k ? a.k < b.k : a.f < b.f);
  });
  m.EToE.resize(4 * K);
  m.EToF.resize(4 * K);
  for (int64_t k = 0; k < K; ++k)
    for (int f = 0; f < 4; ++f) {
      m.EToE[4 * k + f] = k;
      m.EToF[4 * k + f] = (int8_t)f;
    }
  for (size_t i = 0; i < recs.size();) {
    size_t j = i;
    while (j < recs.size() && recs[j].key == recs[i].key) ++j;
    if (j - i > 2) fail3(DG_E_MESH_NONMANIFOLD, "a face shared by more than two tetrahedra");
    if (j - i == 2) {
      const Rec &a = recs[i], &b = recs[i + 1];
      m.EToE[4 * a.k + a.f] = b.k;
      m.EToF[4 * a.k + a.f] = (int8_t)b.f;
      m.EToE[4 * b.k + b.f] = a.k;
      m.EToF[4 * b.k + b.f] = (int8_t)a.f;
    }
    i = j;
  }
  // face maps: node i of face f has barycentric weights w_v on the face's 3 global vertices; the
  // neighbour node is the one of face f' with the same weights on the same global vertices
  std::vector<double> bary(4 * Np);
  for (int i = 0; i < Np; ++i) {
    bary[4 * i + 0] = -(1.0 + ref.r[i] + ref.s[i] + ref.t[i]) / 2;
    bary[4 * i + 1] = (1.0 + ref.r[i]) / 2;
    bary[4 * i + 2] = (1.0 + ref.s[i]) / 2;
    bary[4 * i + 3] = (1.0 + ref.t[i]) / 2;
  }
  m.vmapP.assign(K * 4 * Nfp, 0);
  std::vector<double> x1(Np), y1(Np), z1(Np), x2(Np), y2(Np), z2(Np);
  for (int64_t k = 0; k < K; ++k) {
    for (int f = 0; f < 4; ++f) {
      const int64_t k2 = m.EToE[4 * k + f];
      const int f2 = m.EToF[4 * k + f];
      int64_t* out = &m.vmapP[(k * 4 + f) * Nfp];
      if (k2 == k && f2 == f) {
        for (int i = 0; i < Nfp; ++i) out[i] = k * Np + ref.Fmask[f * Nfp + i];
        continue;
      }
      element_nodes3d(ref, m, k, x1.data(), y1.data(), z1.data());
      element_nodes3d(ref, m, k2, x2.data(), y2.data(), z2.data());
      double h = 0.0;
      for (int a = 0; a < 3; ++a) {
        const int64_t va = m.EToV[4 * k + kFaceVerts[f][a]], vb = m.EToV[4 * k + kFaceVerts[f][(a + 1) % 3]];
        h = std::max(h, std::hypot(std::hypot(VX[va] - VX[vb], VY[va] - VY[vb]), VZ[va] - VZ[vb]));
      }
      for (int i = 0; i < Nfp; ++i) {
        const int n1 = ref.Fmask[f * Nfp + i];
        // weights of node n1 keyed by global vertex id
        int64_t wid[3];
        double wv[3];
        for (int a = 0; a < 3; ++a) {
          wid[a] = m.EToV[4 * k + kFaceVerts[f][a]];
          wv[a] = bary[4 * n1 + kFaceVerts[f][a]];
        }
        int best = -1;
        double bd = 1e300;
        for (int j = 0; j < Nfp; ++j) {
          const int n2 = ref.Fmask[f2 * Nfp + j];
          double d = 0.0;
          for (int a = 0; a < 3; ++a) {
            const int lv = kFaceVerts[f2][a];
            const int64_t gv = m.EToV[4 * k2 + lv];
            const int b = gv == wid[0] ? 0 : (gv == wid[1] ? 1 : (gv == wid[2] ? 2 : -1));
            if (b < 0) fail3(DG_E_MESH_NONCONFORMING, "neighbouring faces do not share their vertices");
            d = std::max(d, std::fabs(wv[b] - bary[4 * n2 + lv]));
          }
          if (d < bd) {
            bd = d;
            best = n2;
          }
        }
        const double dist = std::hypot(std::hypot(x1[n1] - x2[best], y1[n1] - y2[best]), z1[n1] - z2[best]);
        if (bd > 1e-12 || dist > 1e-8 * h) fail3(DG_E_MESH_NONCONFORMING, "face nodes of neighbours do not match");
        out[i] = k2 * Np + best;
      }
    }
  }
}

}  // namespace dg
