// Host fp64 setup of the nodal-DG TM Maxwell operator.
//
// Reference element:
//   * warp-and-blend nodes (PAPER.md:275-279 cites warburton_explicit_2006;
//     alpha table SURVEY.md Appendix A; reading A6), r fastest, rows bottom->top;
//   * orthonormal Koornwinder-Dubiner basis, V, Vr, Vs;
//   * Dr = Vr V^-1, Ds = Vs V^-1 (the D^{d nu} of PAPER.md:296-299);
//   * M = (V V^T)^-1 (the reference mass matrix of PAPER.md:291-295);
//   * LIFT = V (V^T E) with E holding the 1D face mass blocks (V1D V1D^T)^-1
//     (eq. 8; reading A8: 1D parameter interval
//     [-1,1] on every face, the face Jacobian sJ = L/2 is applied separately).
// Mesh:
//   * faces f0=(v0,v1), f1=(v1,v2), f2=(v2,v0), matched by sorted vertex pair
//     (SPEC.md:159-167); boundary EToE=k, EToF=f;
//   * affine geometry rx, sx, ry, sy, J, nx, ny, sJ, Fsc = sJ/J
//     (PAPER.md:286-307, 628-630);
//   * vmapP by the CLOSED-FORM reversal rule of SURVEY.md §8(c) O7 (traversal
//     d = (+1,+1,-1)), verified against physical node coordinates;
//   * contiguous block partition and halo face-point lists.
#include "setup.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <tuple>

#include "../../include/dg.h"

namespace dg {

namespace {
[[noreturn]] void fail(int st, const std::string& m) { throw SetupError{st, m}; }
}  // namespace

// ---------------------------------------------------------------- 1D polynomials
// Orthonormal Jacobi polynomial P_n^{(a,b)} at x[0..nx) (three-term recurrence).
void jacobiP(const double* x, int nx, double a, double b, int n, double* out) {
  const double g0 = std::pow(2.0, a + b + 1) / (a + b + 1) * std::tgamma(a + 1) * std::tgamma(b + 1) /
                    std::tgamma(a + b + 1);
  std::vector<double> pm(nx, 1.0 / std::sqrt(g0)), p(nx), pn(nx);
  if (n == 0) { std::copy(pm.begin(), pm.end(), out); return; }
  const double g1 = (a + 1) * (b + 1) / (a + b + 3) * g0;
  for (int i = 0; i < nx; ++i) p[i] = ((a + b + 2) * x[i] / 2 + (a - b) / 2) / std::sqrt(g1);
  double aold = 2.0 / (2 + a + b) * std::sqrt((a + 1) * (b + 1) / (a + b + 3));
  for (int i = 1; i < n; ++i) {
    const double h1 = 2 * i + a + b;
    const double anew = 2.0 / (h1 + 2) *
                        std::sqrt((i + 1) * (i + 1 + a + b) * (i + 1 + a) * (i + 1 + b) / (h1 + 1) / (h1 + 3));
    const double bnew = -(a * a - b * b) / h1 / (h1 + 2);
    for (int q = 0; q < nx; ++q) pn[q] = (-aold * pm[q] + (x[q] - bnew) * p[q]) / anew;
    pm.swap(p);
    p.swap(pn);
    aold = anew;
  }
  std::copy(p.begin(), p.end(), out);
}

void gradJacobiP(const double* x, int nx, double a, double b, int n, double* out) {
  if (n == 0) { std::fill(out, out + nx, 0.0); return; }
  jacobiP(x, nx, a + 1, b + 1, n - 1, out);
  const double f = std::sqrt(n * (n + a + b + 1.0));
  for (int i = 0; i < nx; ++i) out[i] *= f;
}

// Eigenvalues of a symmetric tridiagonal matrix (diag d[n], off-diag e[n-1]) by
// Sturm-sequence bisection; ascending.
std::vector<double> sym_tridiag_eigenvalues(const std::vector<double>& d, const std::vector<double>& e) {
  const int n = (int)d.size();
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < n; ++i) {
    double rad = (i > 0 ? std::fabs(e[i - 1]) : 0.0) + (i < n - 1 ? std::fabs(e[i]) : 0.0);
    lo = std::min(lo, d[i] - rad);
    hi = std::max(hi, d[i] + rad);
  }
  auto count_below = [&](double x) {
    int c = 0;
    double q = 1.0;
    for (int i = 0; i < n; ++i) {
      q = (d[i] - x) - (i > 0 ? e[i - 1] * e[i - 1] / q : 0.0);
      if (q == 0.0) q = -1e-300;
      if (q < 0) ++c;
    }
    return c;
  };
  std::vector<double> ev(n);
  for (int k = 0; k < n; ++k) {
    double a = lo, b = hi;
    for (int it = 0; it < 200; ++it) {
      const double m = 0.5 * (a + b);
      if (m <= a || m >= b) break;
      if (count_below(m) > k) b = m; else a = m;
    }
    ev[k] = 0.5 * (a + b);
  }
  return ev;
}

// LU with partial pivoting; solves A X = B in place of B ([n][nrhs], row-major).
void lu_solve(int n, std::vector<double> A, int nrhs, std::vector<double>& B) {
  for (int c = 0; c < n; ++c) {
    int p = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(A[r * n + c]) > std::fabs(A[p * n + c])) p = r;
    if (A[p * n + c] == 0.0) fail(DG_E_ARG, "singular matrix in setup");
    if (p != c) {
      for (int j = 0; j < n; ++j) std::swap(A[c * n + j], A[p * n + j]);
      for (int j = 0; j < nrhs; ++j) std::swap(B[c * nrhs + j], B[p * nrhs + j]);
    }
    for (int r = c + 1; r < n; ++r) {
      const double f = A[r * n + c] / A[c * n + c];
      if (f == 0.0) continue;
      for (int j = c; j < n; ++j) A[r * n + j] -= f * A[c * n + j];
      for (int j = 0; j < nrhs; ++j) B[r * nrhs + j] -= f * B[c * nrhs + j];
    }
  }
  for (int c = n - 1; c >= 0; --c) {
    for (int j = 0; j < nrhs; ++j) {
      double s = B[c * nrhs + j];
      for (int k = c + 1; k < n; ++k) s -= A[c * n + k] * B[k * nrhs + j];
      B[c * nrhs + j] = s / A[c * n + c];
    }
  }
}

// Gauss nodes of P^{(a,b)}_{n+1} (Golub-Welsch; J_00 := 0 when a+b = 0).
std::vector<double> jacobiGQ(double a, double b, int n) {
  if (n == 0) return {-(a - b) / (a + b + 2)};
  std::vector<double> d(n + 1), e(n);
  for (int i = 0; i <= n; ++i) {
    const double h1 = 2.0 * i + a + b;
    d[i] = (h1 == 0.0) ? 0.0 : -0.5 * (a * a - b * b) / (h1 + 2) / h1;
  }
  if (a + b < 1e-15) d[0] = 0.0;
  for (int i = 1; i <= n; ++i) {
    const double h1 = 2.0 * (i - 1) + a + b;
    e[i - 1] = 2.0 / (h1 + 2) * std::sqrt(i * (i + a + b) * (i + a) * (i + b) / (h1 + 1) / (h1 + 3));
  }
  return sym_tridiag_eigenvalues(d, e);
}

std::vector<double> jacobiGL(double a, double b, int n) {
  if (n == 1) return {-1.0, 1.0};
  std::vector<double> x{-1.0};
  auto xi = jacobiGQ(a + 1, b + 1, n - 2);
  x.insert(x.end(), xi.begin(), xi.end());
  x.push_back(1.0);
  return x;
}

// V1D[i][j] = P_j(r_i), row-major [nr][n+1]
std::vector<double> vandermonde1D(int n, const std::vector<double>& r) {
  const int nr = (int)r.size();
  std::vector<double> V(nr * (n + 1)), col(nr);
  for (int j = 0; j <= n; ++j) {
    jacobiP(r.data(), nr, 0, 0, j, col.data());
    for (int i = 0; i < nr; ++i) V[i * (n + 1) + j] = col[i];
  }
  return V;
}

namespace {
const double kAlphaOpt[15] = {0.0000, 0.0000, 1.4152, 0.1001, 0.2751, 0.9800, 1.0999, 1.2832,
                              1.3648, 1.4773, 1.4959, 1.5743, 1.5770, 1.6223, 1.6258};

}  // namespace

// Edge warp of the warp-and-blend construction.
std::vector<double> warpfactor(int n, const std::vector<double>& rout) {
  const int nr = (int)rout.size();
  auto lgl = jacobiGL(0, 0, n);
  std::vector<double> req(n + 1);
  for (int i = 0; i <= n; ++i) req[i] = -1.0 + 2.0 * i / n;
  auto Veq = vandermonde1D(n, req);  // [n+1][n+1]
  // Lmat = Veq^T \ Pmat, Pmat[i][q] = P_i(rout_q)
  std::vector<double> VeqT((n + 1) * (n + 1));
  for (int i = 0; i <= n; ++i)
    for (int j = 0; j <= n; ++j) VeqT[i * (n + 1) + j] = Veq[j * (n + 1) + i];
  std::vector<double> P((n + 1) * nr), col(nr);
  for (int i = 0; i <= n; ++i) {
    jacobiP(rout.data(), nr, 0, 0, i, col.data());
    for (int q = 0; q < nr; ++q) P[i * nr + q] = col[q];
  }
  lu_solve(n + 1, VeqT, nr, P);
  std::vector<double> warp(nr, 0.0);
  for (int q = 0; q < nr; ++q) {
    double w = 0.0;
    for (int i = 0; i <= n; ++i) w += P[i * nr + q] * (lgl[i] - req[i]);
    const bool inside = std::fabs(rout[q]) < 1.0 - 1.0e-10;
    warp[q] = inside ? w / (1.0 - rout[q] * rout[q]) : 0.0;
  }
  return warp;
}

namespace {
void nodes2D(int n, std::vector<double>& r, std::vector<double>& s) {
  const double alpha = n < 16 ? kAlphaOpt[n - 1] : 5.0 / 3.0;
  const int Np = (n + 1) * (n + 2) / 2;
  std::vector<double> L1(Np), L2(Np), L3(Np), X(Np), Y(Np);
  int sk = 0;
  for (int row = 0; row <= n; ++row)
    for (int m = 0; m <= n - row; ++m) {
      L1[sk] = (double)row / n;
      L3[sk] = (double)m / n;
      ++sk;
    }
  std::vector<double> d1(Np), d2(Np), d3(Np);
  for (int i = 0; i < Np; ++i) {
    L2[i] = 1.0 - L1[i] - L3[i];
    X[i] = -L2[i] + L3[i];
    Y[i] = (-L2[i] - L3[i] + 2.0 * L1[i]) / std::sqrt(3.0);
    d1[i] = L3[i] - L2[i];
    d2[i] = L1[i] - L3[i];
    d3[i] = L2[i] - L1[i];
  }
  auto w1 = warpfactor(n, d1), w2 = warpfactor(n, d2), w3 = warpfactor(n, d3);
  const double c2 = std::cos(2.0 * M_PI / 3.0), c4 = std::cos(4.0 * M_PI / 3.0);
  const double s2 = std::sin(2.0 * M_PI / 3.0), s4 = std::sin(4.0 * M_PI / 3.0);
  r.resize(Np);
  s.resize(Np);
  for (int i = 0; i < Np; ++i) {
    const double warp1 = 4.0 * L2[i] * L3[i] * w1[i] * (1.0 + (alpha * L1[i]) * (alpha * L1[i]));
    const double warp2 = 4.0 * L1[i] * L3[i] * w2[i] * (1.0 + (alpha * L2[i]) * (alpha * L2[i]));
    const double warp3 = 4.0 * L1[i] * L2[i] * w3[i] * (1.0 + (alpha * L3[i]) * (alpha * L3[i]));
    const double x = X[i] + 1.0 * warp1 + c2 * warp2 + c4 * warp3;
    const double y = Y[i] + 0.0 * warp1 + s2 * warp2 + s4 * warp3;
    // equilateral -> reference (barycentric)
    const double l1 = (std::sqrt(3.0) * y + 1.0) / 3.0;
    const double l2 = (-3.0 * x - std::sqrt(3.0) * y + 2.0) / 6.0;
    const double l3 = (3.0 * x - std::sqrt(3.0) * y + 2.0) / 6.0;
    r[i] = -l2 + l3 - l1;
    s[i] = -l2 - l3 + l1;
  }
}

}  // namespace

// Orthonormal simplex mode phi_ij and its gradient at (r, s) via collapsed (a, b).
void simplex_mode(const std::vector<double>& r, const std::vector<double>& s, int i, int j, double* phi,
                  double* dr, double* ds) {
  const int n = (int)r.size();
  std::vector<double> a(n), b(n), fa(n), dfa(n), gb(n), dgb(n);
  for (int q = 0; q < n; ++q) {
    a[q] = (s[q] != 1.0) ? 2.0 * (1.0 + r[q]) / (1.0 - s[q]) - 1.0 : -1.0;
    b[q] = s[q];
  }
  jacobiP(a.data(), n, 0, 0, i, fa.data());
  gradJacobiP(a.data(), n, 0, 0, i, dfa.data());
  jacobiP(b.data(), n, 2.0 * i + 1, 0, j, gb.data());
  gradJacobiP(b.data(), n, 2.0 * i + 1, 0, j, dgb.data());
  for (int q = 0; q < n; ++q) {
    const double omb = 1.0 - b[q];
    if (phi) phi[q] = std::sqrt(2.0) * fa[q] * gb[q] * std::pow(omb, i);
    if (dr || ds) {
      double vr = dfa[q] * gb[q];
      double vs = dfa[q] * (gb[q] * (0.5 * (1.0 + a[q])));
      if (i > 0) {
        const double h = std::pow(0.5 * omb, i - 1);
        vr *= h;
        vs *= h;
      }
      double tmp = dgb[q] * std::pow(0.5 * omb, i);
      if (i > 0) tmp -= 0.5 * i * gb[q] * std::pow(0.5 * omb, i - 1);
      vs += fa[q] * tmp;
      const double sc = std::pow(2.0, i + 0.5);
      if (dr) dr[q] = sc * vr;
      if (ds) ds[q] = sc * vs;
    }
  }
}

RefElem build_refelem(int N) {
  if (N < 1 || N > 15) fail(DG_E_DEGREE, "degree N must be in [1, 15]");
  RefElem R;
  R.N = N;
  R.Np = (N + 1) * (N + 2) / 2;
  R.Nfp = N + 1;
  const int Np = R.Np, Nfp = R.Nfp;
  nodes2D(N, R.r, R.s);
  R.V.assign(Np * Np, 0.0);
  std::vector<double> Vr(Np * Np), Vs(Np * Np), phi(Np), dr(Np), ds(Np);
  int col = 0;
  for (int i = 0; i <= N; ++i)
    for (int j = 0; j <= N - i; ++j, ++col) {
      simplex_mode(R.r, R.s, i, j, phi.data(), dr.data(), ds.data());
      for (int q = 0; q < Np; ++q) {
        R.V[q * Np + col] = phi[q];
        Vr[q * Np + col] = dr[q];
        Vs[q * Np + col] = ds[q];
      }
    }
  // D = Vr V^-1  <=>  V^T D^T = Vr^T
  std::vector<double> VT(Np * Np);
  for (int i = 0; i < Np; ++i)
    for (int j = 0; j < Np; ++j) VT[i * Np + j] = R.V[j * Np + i];
  auto transpose = [&](const std::vector<double>& A) {
    std::vector<double> T(Np * Np);
    for (int i = 0; i < Np; ++i)
      for (int j = 0; j < Np; ++j) T[i * Np + j] = A[j * Np + i];
    return T;
  };
  std::vector<double> X = transpose(Vr);
  lu_solve(Np, VT, Np, X);
  R.Dr = transpose(X);
  X = transpose(Vs);
  lu_solve(Np, VT, Np, X);
  R.Ds = transpose(X);
  // M = (V V^T)^-1
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
  // Fmask: s = -1, r + s = 0, r = -1 (tol 1e-12), increasing node index
  R.Fmask.assign(3 * Nfp, -1);
  int cnt[3] = {0, 0, 0};
  for (int q = 0; q < Np; ++q) {
    const bool on[3] = {std::fabs(R.s[q] + 1.0) < 1e-12, std::fabs(R.r[q] + R.s[q]) < 1e-12,
                        std::fabs(R.r[q] + 1.0) < 1e-12};
    for (int f = 0; f < 3; ++f)
      if (on[f]) {
        if (cnt[f] >= Nfp) fail(DG_E_DEGREE, "face mask overflow");
        R.Fmask[f * Nfp + cnt[f]++] = q;
      }
  }
  for (int f = 0; f < 3; ++f)
    if (cnt[f] != Nfp) fail(DG_E_DEGREE, "face mask incomplete");
  // Emat [Np][3Nfp]: 1D face mass (V1D V1D^T)^-1 at the face rows
  std::vector<double> E(Np * 3 * Nfp, 0.0);
  for (int f = 0; f < 3; ++f) {
    std::vector<double> fr(Nfp);
    for (int i = 0; i < Nfp; ++i) {
      const int q = R.Fmask[f * Nfp + i];
      fr[i] = (f == 2) ? R.s[q] : R.r[q];
    }
    auto V1 = vandermonde1D(N, fr);  // [Nfp][Nfp]
    std::vector<double> VV(Nfp * Nfp, 0.0), Mf(Nfp * Nfp, 0.0);
    for (int i = 0; i < Nfp; ++i)
      for (int j = 0; j < Nfp; ++j) {
        double acc = 0.0;
        for (int k = 0; k < Nfp; ++k) acc += V1[i * Nfp + k] * V1[j * Nfp + k];
        VV[i * Nfp + j] = acc;
      }
    for (int i = 0; i < Nfp; ++i) Mf[i * Nfp + i] = 1.0;
    lu_solve(Nfp, VV, Nfp, Mf);
    for (int i = 0; i < Nfp; ++i)
      for (int j = 0; j < Nfp; ++j) E[R.Fmask[f * Nfp + i] * (3 * Nfp) + f * Nfp + j] = Mf[i * Nfp + j];
  }
  // LIFT = V (V^T E)
  std::vector<double> VtE(Np * 3 * Nfp, 0.0);
  for (int i = 0; i < Np; ++i)
    for (int k = 0; k < Np; ++k) {
      const double v = R.V[k * Np + i];
      if (v == 0.0) continue;
      for (int j = 0; j < 3 * Nfp; ++j) VtE[i * 3 * Nfp + j] += v * E[k * 3 * Nfp + j];
    }
  R.LIFT.assign(Np * 3 * Nfp, 0.0);
  for (int i = 0; i < Np; ++i)
    for (int k = 0; k < Np; ++k) {
      const double v = R.V[i * Np + k];
      for (int j = 0; j < 3 * Nfp; ++j) R.LIFT[i * 3 * Nfp + j] += v * VtE[k * 3 * Nfp + j];
    }
  return R;
}

// ---------------------------------------------------------------- mesh
void element_nodes(const RefElem& ref, const Mesh& m, int64_t k, double* x, double* y) {
  const int64_t* v = &m.EToV[3 * k];
  const double x0 = m.VX[v[0]], x1 = m.VX[v[1]], x2 = m.VX[v[2]];
  const double y0 = m.VY[v[0]], y1 = m.VY[v[1]], y2 = m.VY[v[2]];
  for (int q = 0; q < ref.Np; ++q) {
    const double r = ref.r[q], s = ref.s[q];
    x[q] = -(r + s) / 2 * x0 + (1 + r) / 2 * x1 + (1 + s) / 2 * x2;
    y[q] = -(r + s) / 2 * y0 + (1 + r) / 2 * y1 + (1 + s) / 2 * y2;
  }
}

namespace {
// closed-form neighbour point: traversal d = (+1, +1, -1)
inline int partner_index(int f, int f2, int i, int Nfp) {
  const int d[3] = {1, 1, -1};
  return (d[f] == d[f2]) ? Nfp - 1 - i : i;
}
}  // namespace

void face_maps(const RefElem& ref, const Mesh& m, int64_t kl, int64_t* vmapM, int64_t* vmapP) {
  const int Np = ref.Np, Nfp = ref.Nfp;
  const int64_t k = m.local[kl];
  for (int f = 0; f < 3; ++f) {
    const int64_t k2 = m.EToE[3 * k + f];
    const int f2 = m.EToF[3 * k + f];
    for (int i = 0; i < Nfp; ++i) {
      const int64_t own = k * Np + ref.Fmask[f * Nfp + i];
      if (vmapM) vmapM[f * Nfp + i] = own;
      if (vmapP)
        vmapP[f * Nfp + i] = (k2 == k && f2 == f) ? own
                             : k2 * Np + ref.Fmask[f2 * Nfp + partner_index(f, f2, i, Nfp)];
    }
  }
}

void build_mesh(const RefElem& ref, int64_t Nv, const double* VX, const double* VY, int64_t K,
                const int64_t* EToV, const int8_t* bctag, int rank, int nranks, const int32_t* part,
                Mesh& m) {
  const int Np = ref.Np, Nfp = ref.Nfp;
  if (K < 1 || Nv < 3) fail(DG_E_ARG, "mesh needs K >= 1 elements and Nv >= 3 vertices");
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(DG_E_ARG, "bad rank / nranks");
  m.K = K;
  m.Nv = Nv;
  m.VX.assign(VX, VX + Nv);
  m.VY.assign(VY, VY + Nv);
  m.EToV.assign(EToV, EToV + 3 * K);
  m.n_swapped = 0;
  // orientation
  for (int64_t k = 0; k < K; ++k) {
    int64_t* v = &m.EToV[3 * k];
    for (int i = 0; i < 3; ++i)
      if (v[i] < 0 || v[i] >= Nv) fail(DG_E_ARG, "EToV entry out of range at element " + std::to_string(k));
    if (v[0] == v[1] || v[1] == v[2] || v[0] == v[2])
      fail(DG_E_MESH_DEGENERATE, "repeated vertex in element " + std::to_string(k));
    const double det = (m.VX[v[1]] - m.VX[v[0]]) * (m.VY[v[2]] - m.VY[v[0]]) -
                       (m.VX[v[2]] - m.VX[v[0]]) * (m.VY[v[1]] - m.VY[v[0]]);
    if (det < 0) {
      std::swap(v[1], v[2]);
      ++m.n_swapped;
    }
  }
  // connectivity by sorted vertex pairs
  m.EToE.resize(3 * K);
  m.EToF.resize(3 * K);
  struct FaceRec { int64_t a, b, k; int8_t f; };
  std::vector<FaceRec> faces(3 * K);
  for (int64_t k = 0; k < K; ++k)
    for (int f = 0; f < 3; ++f) {
      int64_t a = m.EToV[3 * k + f], b = m.EToV[3 * k + (f + 1) % 3];
      if (a > b) std::swap(a, b);
      faces[3 * k + f] = {a, b, k, (int8_t)f};
      m.EToE[3 * k + f] = k;
      m.EToF[3 * k + f] = (int8_t)f;
    }
  std::sort(faces.begin(), faces.end(), [](const FaceRec& x, const FaceRec& y) {
    return std::tie(x.a, x.b, x.k, x.f) < std::tie(y.a, y.b, y.k, y.f);
  });
  for (size_t i = 0; i < faces.size();) {
    size_t j = i + 1;
    while (j < faces.size() && faces[j].a == faces[i].a && faces[j].b == faces[i].b) ++j;
    if (j - i > 2)
      fail(DG_E_MESH_NONMANIFOLD, "edge (" + std::to_string(faces[i].a) + "," + std::to_string(faces[i].b) +
                                      ") shared by " + std::to_string(j - i) + " elements");
    if (j - i == 2) {
      const FaceRec &p = faces[i], &q = faces[i + 1];
      m.EToE[3 * p.k + p.f] = q.k;
      m.EToF[3 * p.k + p.f] = q.f;
      m.EToE[3 * q.k + q.f] = p.k;
      m.EToF[3 * q.k + q.f] = p.f;
    }
    i = j;
  }
  // boundary tags: every boundary face is PEC
  m.pec.assign(3 * K, 0);
  for (int64_t k = 0; k < K; ++k)
    for (int f = 0; f < 3; ++f) {
      const bool bnd = m.EToE[3 * k + f] == k && m.EToF[3 * k + f] == f;
      const int tag = bctag ? bctag[3 * k + f] : 0;
      if (tag != 0 && tag != 1) fail(DG_E_UNSUPPORTED_BC, "unsupported boundary tag " + std::to_string(tag));
      if (tag == 1 && !bnd) fail(DG_E_UNSUPPORTED_BC, "PEC tag on an interior face of element " + std::to_string(k));
      m.pec[3 * k + f] = bnd ? 1 : 0;
    }
  // partition
  m.rank = rank;
  m.nranks = nranks;
  m.part.resize(K);
  if (part) {
    for (int64_t k = 0; k < K; ++k) {
      if (part[k] < 0 || part[k] >= nranks) fail(DG_E_ARG, "part[] entry out of range");
      m.part[k] = part[k];
    }
  } else {
    for (int r = 0; r < nranks; ++r)
      for (int64_t k = (int64_t)r * K / nranks; k < (int64_t)(r + 1) * K / nranks; ++k) m.part[k] = r;
  }
  m.local.clear();
  m.g2l.assign(K, -1);
  for (int64_t k = 0; k < K; ++k)
    if (m.part[k] == rank) {
      m.g2l[k] = (int64_t)m.local.size();
      m.local.push_back(k);
    }
  const int64_t Kl = (int64_t)m.local.size();
  // geometry of local elements
  m.rx.resize(Kl); m.sx.resize(Kl); m.ry.resize(Kl); m.sy.resize(Kl); m.J.resize(Kl);
  m.nx.resize(3 * Kl); m.ny.resize(3 * Kl); m.sJ.resize(3 * Kl); m.Fsc.resize(3 * Kl);
  for (int64_t kl = 0; kl < Kl; ++kl) {
    const int64_t k = m.local[kl];
    const int64_t* v = &m.EToV[3 * k];
    const double x0 = m.VX[v[0]], x1 = m.VX[v[1]], x2 = m.VX[v[2]];
    const double y0 = m.VY[v[0]], y1 = m.VY[v[1]], y2 = m.VY[v[2]];
    const double xr = (x1 - x0) / 2, xs = (x2 - x0) / 2, yr = (y1 - y0) / 2, ys = (y2 - y0) / 2;
    const double J = xr * ys - xs * yr;
    const double e0 = std::hypot(x1 - x0, y1 - y0), e1 = std::hypot(x2 - x1, y2 - y1), e2 = std::hypot(x0 - x2, y0 - y2);
    const double emax = std::max(e0, std::max(e1, e2));
    if (!(std::fabs(J) >= 1e-14 * emax * emax)) fail(DG_E_MESH_DEGENERATE, "degenerate element " + std::to_string(k));
    m.J[kl] = J;
    m.rx[kl] = ys / J; m.sx[kl] = -yr / J; m.ry[kl] = -xs / J; m.sy[kl] = xr / J;
    const double nxu[3] = {yr, ys - yr, -ys}, nyu[3] = {-xr, xr - xs, xs};
    for (int f = 0; f < 3; ++f) {
      const double sJ = std::hypot(nxu[f], nyu[f]);
      m.nx[3 * kl + f] = nxu[f] / sJ;
      m.ny[3 * kl + f] = nyu[f] / sJ;
      m.sJ[3 * kl + f] = sJ;
      m.Fsc[3 * kl + f] = sJ / J;
    }
  }
  // verify the closed-form partner rule against physical coordinates
  {
    std::vector<double> xa(Np), ya(Np), xb(Np), yb(Np);
    for (int64_t kl = 0; kl < Kl; ++kl) {
      const int64_t k = m.local[kl];
      element_nodes(ref, m, k, xa.data(), ya.data());
      for (int f = 0; f < 3; ++f) {
        const int64_t k2 = m.EToE[3 * k + f];
        const int f2 = m.EToF[3 * k + f];
        if (k2 == k && f2 == f) continue;
        element_nodes(ref, m, k2, xb.data(), yb.data());
        const int64_t a = m.EToV[3 * k + f], b = m.EToV[3 * k + (f + 1) % 3];
        const double L = std::hypot(m.VX[a] - m.VX[b], m.VY[a] - m.VY[b]);
        for (int i = 0; i < Nfp; ++i) {
          const int q = ref.Fmask[f * Nfp + i];
          const int q2 = ref.Fmask[f2 * Nfp + partner_index(f, f2, i, Nfp)];
          if (!(std::hypot(xa[q] - xb[q2], ya[q] - yb[q2]) <= 1e-8 * L))
            fail(DG_E_MESH_NONCONFORMING, "face nodes of element " + std::to_string(k) + " face " +
                                              std::to_string(f) + " do not match the neighbour's");
        }
      }
    }
  }
  // halo lists and per-point neighbour locations
  m.nbr_local.assign(Kl * 3 * Nfp, 0);
  struct RecvRec { int src; int64_t kl; int f, i; int64_t gdof; };
  struct SendRec { int dst; int64_t k2; int f2, i2; int64_t gdof; };
  std::vector<RecvRec> rr;
  std::vector<SendRec> sr;
  for (int64_t kl = 0; kl < Kl; ++kl) {
    const int64_t k = m.local[kl];
    for (int f = 0; f < 3; ++f) {
      const int64_t k2 = m.EToE[3 * k + f];
      const int f2 = m.EToF[3 * k + f];
      for (int i = 0; i < Nfp; ++i) {
        const int64_t pt = (kl * 3 + f) * Nfp + i;
        if (k2 == k && f2 == f) {
          m.nbr_local[pt] = kl * Np + ref.Fmask[f * Nfp + i];
        } else if (m.part[k2] == rank) {
          m.nbr_local[pt] = m.g2l[k2] * Np + ref.Fmask[f2 * Nfp + partner_index(f, f2, i, Nfp)];
        } else {
          rr.push_back({m.part[k2], kl, f, i, k2 * Np + ref.Fmask[f2 * Nfp + partner_index(f, f2, i, Nfp)]});
        }
      }
      // what rank part[k2] needs from me across this face: its points (k2, f2, i2), in its order
      if (k2 != k && m.part[k2] != rank)
        for (int i2 = 0; i2 < Nfp; ++i2)
          sr.push_back({m.part[k2], k2, f2, i2, k * Np + ref.Fmask[f * Nfp + partner_index(f2, f, i2, Nfp)]});
    }
  }
  std::stable_sort(rr.begin(), rr.end(), [](const RecvRec& x, const RecvRec& y) { return x.src < y.src; });
  std::sort(sr.begin(), sr.end(), [](const SendRec& x, const SendRec& y) {
    return std::tie(x.dst, x.k2, x.f2, x.i2) < std::tie(y.dst, y.k2, y.f2, y.i2);
  });
  std::vector<int> nb;
  for (auto& x : rr) nb.push_back(x.src);
  for (auto& x : sr) nb.push_back(x.dst);
  std::sort(nb.begin(), nb.end());
  nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
  m.nbr = nb;
  const size_t nn = nb.size();
  m.recv_off.assign(nn + 1, 0);
  m.send_off.assign(nn + 1, 0);
  m.recv_gdof.clear(); m.recv_point.clear(); m.send_gdof.clear();
  size_t a = 0, b = 0;
  for (size_t t = 0; t < nn; ++t) {
    while (a < rr.size() && rr[a].src == nb[t]) {
      const int64_t slot = (int64_t)m.recv_gdof.size();
      m.recv_gdof.push_back(rr[a].gdof);
      const int64_t pt = (rr[a].kl * 3 + rr[a].f) * Nfp + rr[a].i;
      m.recv_point.push_back(pt);
      m.nbr_local[pt] = -(1 + slot);
      ++a;
    }
    m.recv_off[t + 1] = (int64_t)m.recv_gdof.size();
    while (b < sr.size() && sr[b].dst == nb[t]) m.send_gdof.push_back(sr[b++].gdof);
    m.send_off[t + 1] = (int64_t)m.send_gdof.size();
  }
}

std::vector<int64_t> locality_order(const Mesh& m) {
  const int64_t Kl = (int64_t)m.local.size();
  std::vector<double> cx(Kl), cy(Kl);
  double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
  for (int64_t kl = 0; kl < Kl; ++kl) {
    const int64_t* v = &m.EToV[3 * m.local[kl]];
    cx[kl] = (m.VX[v[0]] + m.VX[v[1]] + m.VX[v[2]]) / 3.0;
    cy[kl] = (m.VY[v[0]] + m.VY[v[1]] + m.VY[v[2]]) / 3.0;
    x0 = std::min(x0, cx[kl]); x1 = std::max(x1, cx[kl]);
    y0 = std::min(y0, cy[kl]); y1 = std::max(y1, cy[kl]);
  }
  const double span = std::max(std::max(x1 - x0, y1 - y0), 1e-300);
  auto spread = [](uint64_t v) {  // interleave the low 21 bits with zeros
    v &= 0x1fffff;
    v = (v | (v << 32)) & 0x1f00000000ffffULL;
    v = (v | (v << 16)) & 0x1f0000ff0000ffULL;
    v = (v | (v << 8)) & 0x100f00f00f00f00fULL;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ULL;
    v = (v | (v << 2)) & 0x1249249249249249ULL;
    return v;
  };
  std::vector<std::pair<uint64_t, int64_t>> key(Kl);
  for (int64_t kl = 0; kl < Kl; ++kl) {
    const uint64_t ix = (uint64_t)std::min(2097151.0, std::floor((cx[kl] - x0) / span * 2097151.0));
    const uint64_t iy = (uint64_t)std::min(2097151.0, std::floor((cy[kl] - y0) / span * 2097151.0));
    key[kl] = {spread(ix) | (spread(iy) << 1), kl};
  }
  std::sort(key.begin(), key.end());
  std::vector<int64_t> perm(Kl);
  for (int64_t i = 0; i < Kl; ++i) perm[i] = key[i].second;
  return perm;
}

}  // namespace dg
