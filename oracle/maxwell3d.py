"""3D Maxwell semi-discrete operator, energy and driver (TEST INFRASTRUCTURE).

Fields (Hx, Hy, Hz, Ex, Ey, Ez), eps = mu = 1, PEC walls:
    dH/dt = -curl E + LIFT(Fsc fH),   dE/dt = curl H + LIFT(Fsc fE)
(the TM system of PAPER.md:167-181 is its z-independent reduction).  With [q] = q- - q+ (local minus
neighbour) the lifted upwind flux is ONE HALF of the jump form, as in 2D (reading A3):
    fH = 1/2 ( n x [E] + alpha (n (n . [H]) - [H]) )
    fE = 1/2 (-n x [H] + alpha (n (n . [E]) - [E]) )
which reduces exactly to the 2D TM flux (Hz = Ex = Ey = 0, nz = 0); PEC: E+ = -E-, H+ = H-.
Curl by the chain rule, d/dx = rx Dr + sx Ds + tx Dt (eq. 6 in 3D).  LSERK4 as in 2D (oracle.lserk4).
"""
from __future__ import annotations

import numpy as np

from . import lserk4, mesh3d, refelem3d


def grad(ref, geo, u):
    ur = u @ ref.Dr.T
    us = u @ ref.Ds.T
    ut = u @ ref.Dt.T
    gx = geo.rx[:, None] * ur + geo.sx[:, None] * us + geo.tx[:, None] * ut
    gy = geo.ry[:, None] * ur + geo.sy[:, None] * us + geo.ty[:, None] * ut
    gz = geo.rz[:, None] * ur + geo.sz[:, None] * us + geo.tz[:, None] * ut
    return gx, gy, gz


def curl(ref, geo, Fx, Fy, Fz):
    _, yx, zx = grad(ref, geo, Fx)
    xy, _, zy = grad(ref, geo, Fy)
    xz, yz, _ = grad(ref, geo, Fz)
    return yz - zy, zx - xz, xy - yx


class Oracle3D:
    def __init__(self, N, VX, VY, VZ, EToV, alpha=1.0):
        self.N = N
        self.alpha = float(alpha)
        self.ref = refelem3d.build(N)
        self.VX, self.VY, self.VZ = (np.asarray(a, dtype=np.float64) for a in (VX, VY, VZ))
        self.EToV, self.n_swapped = mesh3d.orient(self.VX, self.VY, self.VZ, np.asarray(EToV))
        self.K = self.EToV.shape[0]
        self.EToE, self.EToF = mesh3d.connect(self.EToV)
        self.geo = mesh3d.geometry(self.VX, self.VY, self.VZ, self.EToV, self.ref)
        self.vmapM, self.vmapP = mesh3d.maps(self.ref, self.geo, self.EToE, self.EToF)
        K = self.K
        self.bnd = (self.EToE == np.arange(K)[:, None]) & (self.EToF == np.arange(4)[None, :])

    @property
    def Np(self):
        return self.ref.Np

    def flux(self, q):
        """(fHx, fHy, fHz, fEx, fEy, fEz), Fsc-scaled, [K][4][Nfp]."""
        Nfp = self.ref.Nfp
        flat = [a.ravel() for a in q]
        dq = [a[self.vmapM] - a[self.vmapP] for a in flat]
        bnd = self.bnd[:, :, None] & np.ones((1, 1, Nfp), dtype=bool)
        for c in range(3):          # PEC: H+ = H- ([H] = 0), E+ = -E- ([E] = 2 E-)
            dq[c] = np.where(bnd, 0.0, dq[c])
            dq[3 + c] = np.where(bnd, 2.0 * flat[3 + c][self.vmapM], dq[3 + c])
        nx, ny, nz = (a[:, :, None] for a in (self.geo.nx, self.geo.ny, self.geo.nz))
        Fsc = self.geo.Fsc[:, :, None]
        dHx, dHy, dHz, dEx, dEy, dEz = dq
        ndH = nx * dHx + ny * dHy + nz * dHz
        ndE = nx * dEx + ny * dEy + nz * dEz
        a = self.alpha
        fHx = (ny * dEz - nz * dEy) + a * (nx * ndH - dHx)
        fHy = (nz * dEx - nx * dEz) + a * (ny * ndH - dHy)
        fHz = (nx * dEy - ny * dEx) + a * (nz * ndH - dHz)
        fEx = -(ny * dHz - nz * dHy) + a * (nx * ndE - dEx)
        fEy = -(nz * dHx - nx * dHz) + a * (ny * ndE - dEy)
        fEz = -(nx * dHy - ny * dHx) + a * (nz * ndE - dEz)
        return tuple(0.5 * Fsc * f for f in (fHx, fHy, fHz, fEx, fEy, fEz))

    def rhs(self, q, which="full"):
        Hx, Hy, Hz, Ex, Ey, Ez = q
        K, Np = self.K, self.Np
        zero = np.zeros((K, Np))
        if which != "surface":
            cE = curl(self.ref, self.geo, Ex, Ey, Ez)
            cH = curl(self.ref, self.geo, Hx, Hy, Hz)
            vol = (-cE[0], -cE[1], -cE[2], cH[0], cH[1], cH[2])
        else:
            vol = (zero,) * 6
        if which == "volume":
            return vol
        f = self.flux(q)
        return tuple(v + fl.reshape(K, -1) @ self.ref.LIFT.T for v, fl in zip(vol, f))

    def run(self, q0, dt, nsteps):
        q = tuple(np.array(a, dtype=np.float64) for a in q0)
        res = tuple(np.zeros_like(a) for a in q)
        for _ in range(nsteps):
            q, res = lserk4.step(q, res, dt, self.rhs)
        return q

    def energy(self, q):
        """1/2 sum_k J_k sum_fields u^T M u."""
        return 0.5 * sum(float(np.einsum("k,ki,ij,kj->", self.geo.J, a, self.ref.M, a)) for a in q)
