// Host-side (fp64) setup of the 3D tetrahedral Maxwell operator (the paper's
// hedge workload): reference tetrahedron, connectivity, affine geometry, face maps.
// Independent C++ implementation (shares nothing with oracle/).
#pragma once
#include <cstdint>
#include <vector>

#include "setup.h"

namespace dg {

// Reference tetrahedron {r,s,t >= -1, r+s+t <= -1} of degree N.
struct RefTet {
  int N = 0, Np = 0, Nfp = 0;
  std::vector<double> r, s, t;     // [Np]
  std::vector<double> V;           // [Np][Np]
  std::vector<double> Dr, Ds, Dt;  // [Np][Np]
  std::vector<double> M;           // [Np][Np] = (V V^T)^-1
  std::vector<double> LIFT;        // [Np][4 Nfp]
  std::vector<int> Fmask;          // [4][Nfp]: t = -1, s = -1, r+s+t = -1, r = -1
};
RefTet build_reftet(int N);        // throws SetupError

struct Mesh3D {
  int64_t K = 0, Nv = 0;
  std::vector<double> VX, VY, VZ;
  std::vector<int64_t> EToV;       // [K][4] after orientation
  std::vector<int64_t> EToE;       // [K][4]
  std::vector<int8_t> EToF;        // [K][4]
  int64_t n_swapped = 0;
  std::vector<double> rx, ry, rz, sx, sy, sz, tx, ty, tz, J;   // [K]
  std::vector<double> nx, ny, nz, sJ, Fsc;                     // [K][4]
  std::vector<int64_t> vmapP;      // [K][4][Nfp] canonical k Np + n (boundary: own node)
};
// Orientation, connectivity by sorted vertex triple, geometry, face maps (matched by the face nodes'
// barycentric weights on the shared global vertices, verified against coordinates).
void build_mesh3d(const RefTet& ref, int64_t Nv, const double* VX, const double* VY, const double* VZ,
                  int64_t K, const int64_t* EToV, Mesh3D& m);
void element_nodes3d(const RefTet& ref, const Mesh3D& m, int64_t k, double* x, double* y, double* z);

}  // namespace dg
