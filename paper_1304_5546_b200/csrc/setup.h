// Host-side (fp64) setup of the nodal-DG TM Maxwell operator: reference
// element, connectivity, affine geometry, face maps, partition and halo lists.
// Independent C++ implementation (shares nothing with oracle/).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace dg {

struct SetupError {
  int status;           // dg_status value
  std::string msg;
};

// Reference element of degree N.
struct RefElem {
  int N = 0, Np = 0, Nfp = 0;
  std::vector<double> r, s;        // [Np]
  std::vector<double> V;           // [Np][Np] row-major, V[i][j] = phi_j(r_i, s_i)
  std::vector<double> Dr, Ds;      // [Np][Np]
  std::vector<double> M;           // [Np][Np] reference mass matrix (V V^T)^{-1}
  std::vector<double> LIFT;        // [Np][3 Nfp]
  std::vector<int> Fmask;          // [3][Nfp]
};

RefElem build_refelem(int N);      // throws SetupError

// Global mesh + this rank's partition.
struct Mesh {
  int64_t K = 0, Nv = 0;
  std::vector<double> VX, VY;
  std::vector<int64_t> EToV;       // [K][3] after orientation
  std::vector<int64_t> EToE;       // [K][3]
  std::vector<int8_t> EToF;        // [K][3]
  std::vector<int8_t> pec;         // [K][3] 1 = PEC boundary face
  int64_t n_swapped = 0;
  // partition
  int rank = 0, nranks = 1;
  std::vector<int32_t> part;       // [K] element -> rank
  std::vector<int64_t> local;      // local -> global element id, ascending
  std::vector<int64_t> g2l;        // [K] global -> local id or -1
  // per local element geometry
  std::vector<double> rx, sx, ry, sy, J;      // [Kl]
  std::vector<double> nx, ny, sJ, Fsc;        // [Kl][3]
  // halo: neighbour ranks ascending
  std::vector<int> nbr;
  std::vector<int64_t> send_off, recv_off;    // [n_nbr + 1]
  std::vector<int64_t> send_gdof;             // canonical global DOFs I send
  std::vector<int64_t> recv_gdof;             // canonical global DOFs I receive
  std::vector<int64_t> recv_point;            // local face point fed by each received value
  // per local face point: neighbour location; >= 0: local canonical DOF (kl*Np+n),
  // < 0: -(1 + halo slot).  Boundary points refer to their own node.
  std::vector<int64_t> nbr_local;             // [Kl][3][Nfp]
};

// Orient, connect, geometry, maps, partition and halo lists.  Throws SetupError.
void build_mesh(const RefElem& ref, int64_t Nv, const double* VX, const double* VY, int64_t K,
                const int64_t* EToV, const int8_t* bctag, int rank, int nranks, const int32_t* part,
                Mesh& m);

// Device storage order of the local elements: a permutation slot -> local id
// sorted by the Morton (Z-order) code of the element centroids, so that a
// 32-element tile is a compact patch and most face neighbours share its tile
// (the "blocking strategy" against fetching faces twice).
std::vector<int64_t> locality_order(const Mesh& m);

// Canonical global maps for a local element (vmapM / vmapP of SURVEY.md §8(c) O7).
void face_maps(const RefElem& ref, const Mesh& m, int64_t kl, int64_t* vmapM, int64_t* vmapP);

// Physical node coordinates of a global element.
void element_nodes(const RefElem& ref, const Mesh& m, int64_t k, double* x, double* y);

// Polynomial building blocks (setup.cpp), shared by the 2D and 3D (setup3d.cpp) reference elements.
void jacobiP(const double* x, int nx, double a, double b, int n, double* out);      // orthonormal P_n^(a,b)
void gradJacobiP(const double* x, int nx, double a, double b, int n, double* out);
std::vector<double> jacobiGQ(double a, double b, int n);    // Gauss nodes (Sturm bisection)
std::vector<double> jacobiGL(double a, double b, int n);    // Gauss-Lobatto nodes
std::vector<double> vandermonde1D(int n, const std::vector<double>& r);
std::vector<double> warpfactor(int n, const std::vector<double>& rout);  // edge warp / (1 - r^2), 0 at the ends
// orthonormal triangle mode phi_ij (and d/dr, d/ds) at points (r, s); any output may be NULL
void simplex_mode(const std::vector<double>& r, const std::vector<double>& s, int i, int j, double* phi,
                  double* dr, double* ds);

// Small dense linear algebra (row-major), exposed for the unit tests of the library.
void lu_solve(int n, std::vector<double> A, int nrhs, std::vector<double>& B);  // A X = B, B [n][nrhs]
std::vector<double> sym_tridiag_eigenvalues(const std::vector<double>& d, const std::vector<double>& e);

}  // namespace dg
