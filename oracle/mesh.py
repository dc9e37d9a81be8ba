"""O5-O7: connectivity, affine geometry, face maps, partition (TEST INFRASTRUCTURE).

* Faces f0 = (v0,v1), f1 = (v1,v2), f2 = (v2,v0); matched by sorted vertex
  pair; boundary faces get EToE = k, EToF = f; > 2 elements on one edge is a
  non-manifold error.
* Clockwise elements are re-oriented by swapping local vertices 1 <-> 2
  (SURVEY §8(b)).
* Affine map Psi(r,s) = A_k (r,s)^T + b_k:
  x = -(r+s)/2 x0 + (1+r)/2 x1 + (1+s)/2 x2; the entries of A_k^{-1} are
  rx, sx, ry, sy (eq. 6); J = |A_k|;
  outward normals / face Jacobians sJ = L_f / 2 (reading A8); Fsc = sJ / J
  ("the surface Jacobian divided by the element's volume Jacobian",
  PAPER.md:628-630).  SURVEY O6.
* vmapM = k Np + Fmask[f, i]; vmapP by MATCHING PHYSICAL COORDINATES of the
  neighbour's face nodes (distance < 1e-10 * edge length), the plain
  definition of "the index of its facial neighbor" (
  SPEC.md:182).  Boundary: vmapP = vmapM.
* Partition (CPU fake partition, SURVEY.md §4 "Pin 2" and §8(e)): contiguous
  element blocks [r K / P, (r+1) K / P); halo lists of face points.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class MeshError(ValueError):
    pass


def orient(VX, VY, EToV):
    """Return (EToV', n_swapped): clockwise elements get vertices 1 <-> 2 swapped."""
    EToV = np.array(EToV, dtype=np.int64, copy=True)
    x = VX[EToV]
    y = VY[EToV]
    det = (x[:, 1] - x[:, 0]) * (y[:, 2] - y[:, 0]) - (x[:, 2] - x[:, 0]) * (y[:, 1] - y[:, 0])
    cw = det < 0
    EToV[cw, 1], EToV[cw, 2] = EToV[cw, 2].copy(), EToV[cw, 1].copy()
    return EToV, int(cw.sum())


def connect(EToV):
    """(EToE int64 [K][3], EToF int64 [K][3]) by sorted vertex pairs."""
    K = EToV.shape[0]
    EToE = np.tile(np.arange(K)[:, None], (1, 3))
    EToF = np.tile(np.arange(3)[None, :], (K, 1))
    faces = {}
    for k in range(K):
        for f in range(3):
            a, b = int(EToV[k, f]), int(EToV[k, (f + 1) % 3])
            key = (a, b) if a < b else (b, a)
            faces.setdefault(key, []).append((k, f))
    for key, lst in faces.items():
        if len(lst) > 2:
            raise MeshError(f"non-manifold edge {key} shared by {len(lst)} elements")
        if len(lst) == 2:
            (k1, f1), (k2, f2) = lst
            EToE[k1, f1], EToF[k1, f1] = k2, f2
            EToE[k2, f2], EToF[k2, f2] = k1, f1
    return EToE, EToF


@dataclass
class Geometry:
    rx: np.ndarray   # [K]
    sx: np.ndarray
    ry: np.ndarray
    sy: np.ndarray
    J: np.ndarray    # [K]  = |A_k|
    nx: np.ndarray   # [K][3]
    ny: np.ndarray
    sJ: np.ndarray   # [K][3] = L_f / 2
    Fsc: np.ndarray  # [K][3] = sJ / J
    x: np.ndarray    # [K][Np] physical node coordinates
    y: np.ndarray


def geometry(VX, VY, EToV, ref) -> Geometry:
    """Affine geometric factors and node coordinates."""
    x0, x1, x2 = (VX[EToV[:, i]] for i in range(3))
    y0, y1, y2 = (VY[EToV[:, i]] for i in range(3))
    r, s = ref.r, ref.s
    x = (-(r + s) / 2)[None, :] * x0[:, None] + ((1 + r) / 2)[None, :] * x1[:, None] \
        + ((1 + s) / 2)[None, :] * x2[:, None]
    y = (-(r + s) / 2)[None, :] * y0[:, None] + ((1 + r) / 2)[None, :] * y1[:, None] \
        + ((1 + s) / 2)[None, :] * y2[:, None]
    xr, xs = (x1 - x0) / 2, (x2 - x0) / 2
    yr, ys = (y1 - y0) / 2, (y2 - y0) / 2
    J = xr * ys - xs * yr
    emax = np.maximum.reduce([np.hypot(x1 - x0, y1 - y0), np.hypot(x2 - x1, y2 - y1),
                              np.hypot(x0 - x2, y0 - y2)])
    bad = np.abs(J) < 1e-14 * emax ** 2
    if bad.any():
        raise MeshError(f"degenerate element {int(np.nonzero(bad)[0][0])}")
    if (J < 0).any():
        raise MeshError("clockwise element after orientation")
    rx, sx, ry, sy = ys / J, -yr / J, -xs / J, xr / J
    nx = np.stack([yr, ys - yr, -ys], axis=1)
    ny = np.stack([-xr, xr - xs, xs], axis=1)
    sJ = np.hypot(nx, ny)
    nx = nx / sJ
    ny = ny / sJ
    Fsc = sJ / J[:, None]
    return Geometry(rx, sx, ry, sy, J, nx, ny, sJ, Fsc, x, y)


def maps(ref, geo: Geometry, EToE, EToF, EToV, VX, VY):
    """(vmapM, vmapP) int64 [K][3][Nfp] in canonical global index k*Np + n."""
    K = EToE.shape[0]
    Np, Nfp = ref.Np, ref.Nfp
    vmapM = np.empty((K, 3, Nfp), dtype=np.int64)
    for f in range(3):
        vmapM[:, f, :] = np.arange(K)[:, None] * Np + ref.Fmask[f][None, :]
    vmapP = vmapM.copy()
    xf = geo.x.ravel()
    yf = geo.y.ravel()
    for k in range(K):
        for f in range(3):
            k2, f2 = int(EToE[k, f]), int(EToF[k, f])
            if k2 == k and f2 == f:
                continue
            a, b = EToV[k, f], EToV[k, (f + 1) % 3]
            L = np.hypot(VX[a] - VX[b], VY[a] - VY[b])
            idM = vmapM[k, f]
            idN = vmapM[k2, f2]
            d = np.hypot(xf[idM][:, None] - xf[idN][None, :], yf[idM][:, None] - yf[idN][None, :])
            j = np.argmin(d, axis=1)
            if not np.all(d[np.arange(Nfp), j] < 1e-10 * L):
                raise MeshError(f"trace match failure on element {k} face {f}")
            vmapP[k, f] = idN[j]
    return vmapM, vmapP


# ----------------------------------------------------------------------------
# Partition and halo lists
# ----------------------------------------------------------------------------
def block_partition(K: int, P: int):
    """part[k] = rank for contiguous blocks [r K / P, (r+1) K / P)."""
    part = np.empty(K, dtype=np.int64)
    for r in range(P):
        part[(r * K) // P:((r + 1) * K) // P] = r
    return part


def halo_lists(part, rank: int, EToE, EToF, vmapP, Np: int):
    """Halo lists of ``rank`` under element->rank map ``part``.

    recv[src] = list of (k, f, i) face points of OWN elements whose trace
                partner lives on rank src, in increasing (k, f, i);
    need[src] = the partner's canonical global DOF (k' Np + n') for each entry.
    send[dst] = canonical global DOF indices of own nodes that rank dst needs,
                in dst's (k', f', i) order -- i.e. need[rank] as computed by dst.
    """
    K = EToE.shape[0]
    recv, need = {}, {}
    own = np.nonzero(part == rank)[0]
    for k in own:
        for f in range(3):
            k2 = int(EToE[k, f])
            if k2 == k or part[k2] == rank:
                continue
            src = int(part[k2])
            for i in range(vmapP.shape[2]):
                recv.setdefault(src, []).append((int(k), f, i))
                need.setdefault(src, []).append(int(vmapP[k, f, i]))
    send = {}
    for dst in sorted(set(int(p) for p in np.unique(part)) - {rank}):
        lst = []
        for k in np.nonzero(part == dst)[0]:
            for f in range(3):
                k2 = int(EToE[k, f])
                if k2 != k and part[k2] == rank:
                    lst.extend(int(v) for v in vmapP[k, f])
        if lst:
            send[dst] = lst
    return recv, need, send
