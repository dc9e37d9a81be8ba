"""O8: the semi-discrete DG right-hand side (TEST INFRASTRUCTURE).

Per element k (eq. 9 with reading A2; eq. 2a-c with A1):

    d/dt Hx = -D^{k,y} Ez                 + LIFT (Fsc . fHx)
    d/dt Hy = +D^{k,x} Ez                 + LIFT (Fsc . fHy)
    d/dt Ez = D^{k,x} Hy - D^{k,y} Hx     + LIFT (Fsc . fEz)

with D^{k,x} = rx Dr + sx Ds, D^{k,y} = ry Dr + sy Ds (eq. 6)
and LIFT = M^{-1} M^{dI} (eq. 8).

Flux gather: per face point record (idM, idP, nx, ny, Fsc,
Bsc); jumps [q] = q^- - q^+ (PAPER.md:271), the exterior Ez is Bsc * Ez[idP]
(reading A7: PEC boundary idP = idM, Bsc = -1).

Constant material (eps = mu = 1): the lifted flux is
ONE HALF of eq. 5 (reading A3):
    fHx = 1/2 (ny [Ez] + a (nx (nx[Hx] + ny[Hy]) - [Hx]))
    fHy = 1/2 (-nx [Ez] + a (ny (nx[Hx] + ny[Hy]) - [Hy]))
    fEz = 1/2 (ny [Hx] - nx [Hy] - a [Ez])

Piecewise-constant material (extension, reading A12; Z = sqrt(mu/eps),
Y = 1/Z, local side "-", neighbour "+", boundary Z+ = Z-):
    [Ht] = nx [Hy] - ny [Hx]
    gH   = (Y+ [Ez] + a [Ht]) / (Y+ + Y-)
    fHx  = ny gH ;  fHy = -nx gH ;  fEz = -(Z+ [Ht] + a [Ez]) / (Z+ + Z-)
and the three rows are then multiplied by 1/mu, 1/mu, 1/eps.
"""
from __future__ import annotations

import numpy as np


def volume(ref, geo, Hx, Hy, Ez):
    """Volume term of eq. 9: (-Dy Ez, Dx Ez, Dx Hy - Dy Hx), per element.

    Fields are [K][Np]; D applied per element as a plain matrix-vector product
    (batched einsum is the library primitive)."""
    def Dx(u):
        return geo.rx[:, None] * np.einsum("ij,kj->ki", ref.Dr, u) + \
               geo.sx[:, None] * np.einsum("ij,kj->ki", ref.Ds, u)

    def Dy(u):
        return geo.ry[:, None] * np.einsum("ij,kj->ki", ref.Dr, u) + \
               geo.sy[:, None] * np.einsum("ij,kj->ki", ref.Ds, u)

    return -Dy(Ez), Dx(Ez), Dx(Hy) - Dy(Hx)


def surfinfo(ref, geo, vmapM, vmapP, EToE, EToF):
    """Flat per-face-point records (idM, idP, nx, ny, Fsc, Bsc) [K][3][Nfp]
    (SPEC.md:130-136)."""
    K = vmapM.shape[0]
    Nfp = ref.Nfp
    bnd = (EToE == np.arange(K)[:, None]) & (EToF == np.arange(3)[None, :])
    Bsc = np.where(bnd, -1.0, 1.0)[:, :, None] * np.ones((1, 1, Nfp))
    nx = geo.nx[:, :, None] * np.ones((1, 1, Nfp))
    ny = geo.ny[:, :, None] * np.ones((1, 1, Nfp))
    Fsc = geo.Fsc[:, :, None] * np.ones((1, 1, Nfp))
    return dict(idM=vmapM, idP=vmapP, nx=nx, ny=ny, Fsc=Fsc, Bsc=Bsc, bnd=bnd)


def flux(si, Hx, Hy, Ez, alpha=1.0, Zm=None, Zp=None):
    """Fsc-scaled lifted flux values [3][K][3][Nfp] (the vector f^k of eq. 8)."""
    hx, hy, ez = Hx.ravel(), Hy.ravel(), Ez.ravel()
    idM, idP = si["idM"], si["idP"]
    dHx = hx[idM] - hx[idP]
    dHy = hy[idM] - hy[idP]
    dEz = ez[idM] - si["Bsc"] * ez[idP]
    nx, ny, Fsc = si["nx"], si["ny"], si["Fsc"]
    if Zm is None:
        ndotdH = nx * dHx + ny * dHy
        fHx = ny * dEz + alpha * (nx * ndotdH - dHx)
        fHy = -nx * dEz + alpha * (ny * ndotdH - dHy)
        fEz = ny * dHx - nx * dHy - alpha * dEz
        return 0.5 * Fsc * fHx, 0.5 * Fsc * fHy, 0.5 * Fsc * fEz
    Ym, Yp = 1.0 / Zm, 1.0 / Zp
    dHt = nx * dHy - ny * dHx
    gH = (Yp * dEz + alpha * dHt) / (Yp + Ym)
    fHx = ny * gH
    fHy = -nx * gH
    fEz = -(Zp * dHt + alpha * dEz) / (Zp + Zm)
    return Fsc * fHx, Fsc * fHy, Fsc * fEz


def lift(ref, f):
    """LIFT applied per element to the 3 Nfp face vector: [K][3][Nfp] -> [K][Np]."""
    K = f.shape[0]
    return np.einsum("ij,kj->ki", ref.LIFT, f.reshape(K, 3 * ref.Nfp))


def material_impedance(EToE, eps, mu, Nfp):
    """(Zm, Zp) per face point [K][3][Nfp]; boundary faces use Zp = Zm."""
    Z = np.sqrt(np.asarray(mu, dtype=np.float64) / np.asarray(eps, dtype=np.float64))
    Zm = np.repeat(Z[:, None], 3, axis=1)
    Zp = Z[EToE]
    return (Zm[:, :, None] * np.ones((1, 1, Nfp)), Zp[:, :, None] * np.ones((1, 1, Nfp)))


def rhs(ref, geo, si, Hx, Hy, Ez, alpha=1.0, eps=None, mu=None, EToE=None, which="full"):
    """d/dt (Hx, Hy, Ez) of the semi-discrete scheme; which in {full, volume, surface}."""
    K = Hx.shape[0]
    zero = np.zeros((K, ref.Np))
    vHx, vHy, vEz = volume(ref, geo, Hx, Hy, Ez) if which != "surface" else (zero, zero, zero)
    if which == "volume":
        sHx = sHy = sEz = zero
    else:
        if eps is None and mu is None:
            fHx, fHy, fEz = flux(si, Hx, Hy, Ez, alpha)
        else:
            eps_ = np.ones(K) if eps is None else np.asarray(eps, dtype=np.float64)
            mu_ = np.ones(K) if mu is None else np.asarray(mu, dtype=np.float64)
            Zm, Zp = material_impedance(EToE, eps_, mu_, ref.Nfp)
            fHx, fHy, fEz = flux(si, Hx, Hy, Ez, alpha, Zm, Zp)
        sHx, sHy, sEz = lift(ref, fHx), lift(ref, fHy), lift(ref, fEz)
    rHx, rHy, rEz = vHx + sHx, vHy + sHy, vEz + sEz
    if eps is not None or mu is not None:
        eps_ = np.ones(K) if eps is None else np.asarray(eps, dtype=np.float64)
        mu_ = np.ones(K) if mu is None else np.asarray(mu, dtype=np.float64)
        rHx = rHx / mu_[:, None]
        rHy = rHy / mu_[:, None]
        rEz = rEz / eps_[:, None]
    return rHx, rHy, rEz
