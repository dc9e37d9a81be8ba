"""3D tetrahedral meshes: orientation, connectivity, affine geometry, face maps (TEST INFRASTRUCTURE;
SURVEY.md §8(f) row 4; the 2D O5-O7 one dimension up).

* Faces f0 = (v0,v1,v2), f1 = (v0,v1,v3), f2 = (v1,v2,v3), f3 = (v0,v2,v3) (the reference faces
  t = -1, s = -1, r+s+t = -1, r = -1), matched by sorted vertex triple; a boundary face has
  EToE = k, EToF = f; > 2 elements on one face is a non-manifold error.
* Negatively oriented elements get local vertices 1 <-> 2 swapped (the 2D auto-fix).
* x = -(1+r+s+t)/2 x0 + (1+r)/2 x1 + (1+s)/2 x2 + (1+t)/2 x3; the inverse Jacobian gives rx ... tz;
  outward face normals grad-based: f0 -grad t, f1 -grad s, f2 grad(r+s+t), f3 -grad r; sJ = J |n|
  (= face area / 2), Fsc = sJ / J.
* vmapM = k Np + Fmask[f, i]; vmapP by matching physical coordinates of the neighbour's face nodes.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import MeshError
from .refelem3d import FACE_VERTS


def signed_volume6(VX, VY, VZ, EToV):
    P = np.stack([VX[EToV], VY[EToV], VZ[EToV]], axis=-1)
    return np.einsum("ki,ki->k", P[:, 1] - P[:, 0], np.cross(P[:, 2] - P[:, 0], P[:, 3] - P[:, 0]))


def orient(VX, VY, VZ, EToV):
    EToV = np.array(EToV, dtype=np.int64, copy=True)
    neg = signed_volume6(VX, VY, VZ, EToV) < 0
    EToV[neg, 1], EToV[neg, 2] = EToV[neg, 2].copy(), EToV[neg, 1].copy()
    return EToV, int(neg.sum())


def connect(EToV):
    K = EToV.shape[0]
    EToE = np.tile(np.arange(K)[:, None], (1, 4))
    EToF = np.tile(np.arange(4)[None, :], (K, 1))
    faces = {}
    for k in range(K):
        for f, vs in enumerate(FACE_VERTS):
            key = tuple(sorted(int(EToV[k, v]) for v in vs))
            faces.setdefault(key, []).append((k, f))
    for key, lst in faces.items():
        if len(lst) > 2:
            raise MeshError(f"non-manifold face {key} shared by {len(lst)} elements")
        if len(lst) == 2:
            (k1, f1), (k2, f2) = lst
            EToE[k1, f1], EToF[k1, f1] = k2, f2
            EToE[k2, f2], EToF[k2, f2] = k1, f1
    return EToE, EToF


@dataclass
class Geometry3D:
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray          # [K][Np]
    rx: np.ndarray
    ry: np.ndarray
    rz: np.ndarray
    sx: np.ndarray
    sy: np.ndarray
    sz: np.ndarray
    tx: np.ndarray
    ty: np.ndarray
    tz: np.ndarray         # [K]
    J: np.ndarray          # [K]
    nx: np.ndarray
    ny: np.ndarray
    nz: np.ndarray         # [K][4]
    sJ: np.ndarray
    Fsc: np.ndarray        # [K][4]


def geometry(VX, VY, VZ, EToV, ref) -> Geometry3D:
    v = [EToV[:, i] for i in range(4)]
    r, s, t = ref.r, ref.s, ref.t

    def phys(C):
        c0, c1, c2, c3 = (C[vi][:, None] for vi in v)
        return -(1 + r + s + t) / 2 * c0 + (1 + r) / 2 * c1 + (1 + s) / 2 * c2 + (1 + t) / 2 * c3

    x, y, z = phys(VX), phys(VY), phys(VZ)
    # constant Jacobian matrix d(x,y,z)/d(r,s,t)
    A = np.empty((EToV.shape[0], 3, 3))
    for row, C in enumerate((VX, VY, VZ)):
        A[:, row, 0] = (C[v[1]] - C[v[0]]) / 2
        A[:, row, 1] = (C[v[2]] - C[v[0]]) / 2
        A[:, row, 2] = (C[v[3]] - C[v[0]]) / 2
    J = np.linalg.det(A)
    if np.any(J <= 0):
        raise MeshError("degenerate or inverted tetrahedron")
    Ai = np.linalg.inv(A)  # rows: grad r, grad s, grad t
    rx, ry, rz = Ai[:, 0, 0], Ai[:, 0, 1], Ai[:, 0, 2]
    sx, sy, sz = Ai[:, 1, 0], Ai[:, 1, 1], Ai[:, 1, 2]
    tx, ty, tz = Ai[:, 2, 0], Ai[:, 2, 1], Ai[:, 2, 2]
    nraw = np.stack([-Ai[:, 2], -Ai[:, 1], Ai[:, 0] + Ai[:, 1] + Ai[:, 2], -Ai[:, 0]], axis=1)  # [K][4][3]
    norm = np.linalg.norm(nraw, axis=2)
    n = nraw / norm[:, :, None]
    sJ = norm * J[:, None]
    return Geometry3D(x, y, z, rx, ry, rz, sx, sy, sz, tx, ty, tz, J, n[:, :, 0], n[:, :, 1], n[:, :, 2],
                      sJ, sJ / J[:, None])


def maps(ref, geo, EToE, EToF, tol_rel=1e-10):
    """vmapM, vmapP [K][4][Nfp] (global DOF k Np + n) by coordinate matching."""
    K, Np, Nfp = geo.x.shape[0], ref.Np, ref.Nfp
    vmapM = np.zeros((K, 4, Nfp), dtype=np.int64)
    vmapP = np.zeros((K, 4, Nfp), dtype=np.int64)
    h = np.cbrt(6.0 * geo.J.min())  # a length scale
    for k in range(K):
        for f in range(4):
            idM = ref.Fmask[f]
            vmapM[k, f] = k * Np + idM
            k2, f2 = EToE[k, f], EToF[k, f]
            if k2 == k and f2 == f:
                vmapP[k, f] = vmapM[k, f]
                continue
            idP = ref.Fmask[f2]
            PM = np.stack([geo.x[k, idM], geo.y[k, idM], geo.z[k, idM]], axis=1)
            PP = np.stack([geo.x[k2, idP], geo.y[k2, idP], geo.z[k2, idP]], axis=1)
            D = np.linalg.norm(PM[:, None, :] - PP[None, :, :], axis=2)
            j = np.argmin(D, axis=1)
            if D[np.arange(Nfp), j].max() > 1e-8 * h:
                raise MeshError(f"face nodes of elements {k} and {k2} do not match")
            vmapP[k, f] = k2 * Np + idP[j]
    return vmapM, vmapP
