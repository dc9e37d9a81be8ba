"""O10: discrete Maxwell energy and the semi-discrete energy rate (TEST INFRASTRUCTURE).

E = 1/2 sum_k J_k ( mu_k (Hx^T M Hx + Hy^T M Hy) + eps_k Ez^T M Ez ),
with the element mass matrix M^k = |A_k| M (
SURVEY O10).

``energy_rate_expected`` is the face-integral form of dE/dt for the flux of
operator.py (pin P11; material form from reading A12):
  constant material: -(a/2) sum_interior int([Ez]^2 + [Ht]^2) - a sum_PEC int Ez^2
  material:          -a sum_interior int([Ez]^2 + Z+ Z- [Ht]^2)/(Z+ + Z-)
                     - a sum_PEC int Ez^2 / Z
Each face integral is sJ_f * g^T M^Gamma g with the 1D face mass matrix
(reading A8); every interior face is counted once.
"""
from __future__ import annotations

import numpy as np


def inner(ref, geo, u, v, w=None):
    """sum_k J_k w_k u_k^T M v_k."""
    val = geo.J[:, None] * np.einsum("ki,ij,kj->k", u, ref.M, v)[:, None]
    if w is not None:
        val = val * np.asarray(w)[:, None]
    return float(val.sum())


def energy(ref, geo, Hx, Hy, Ez, eps=None, mu=None):
    mu_ = None if mu is None else np.asarray(mu)
    eps_ = None if eps is None else np.asarray(eps)
    return 0.5 * (inner(ref, geo, Hx, Hx, mu_) + inner(ref, geo, Hy, Hy, mu_)
                  + inner(ref, geo, Ez, Ez, eps_))


def energy_rate(ref, geo, q, dq, eps=None, mu=None):
    """dE/dt = <q, R(q)> in the material-weighted mass inner product."""
    Hx, Hy, Ez = q
    rHx, rHy, rEz = dq
    mu_ = None if mu is None else np.asarray(mu)
    eps_ = None if eps is None else np.asarray(eps)
    return inner(ref, geo, Hx, rHx, mu_) + inner(ref, geo, Hy, rHy, mu_) + inner(ref, geo, Ez, rEz, eps_)


def energy_rate_expected(ref, geo, si, EToE, EToF, Hx, Hy, Ez, alpha, eps=None, mu=None):
    K = Hx.shape[0]
    hx, hy, ez = Hx.ravel(), Hy.ravel(), Ez.ravel()
    material = eps is not None or mu is not None
    if material:
        eps_ = np.ones(K) if eps is None else np.asarray(eps, dtype=np.float64)
        mu_ = np.ones(K) if mu is None else np.asarray(mu, dtype=np.float64)
        Z = np.sqrt(mu_ / eps_)
    total = 0.0
    for k in range(K):
        for f in range(3):
            k2, f2 = int(EToE[k, f]), int(EToF[k, f])
            idM = si["idM"][k, f]
            idP = si["idP"][k, f]
            Mf = ref.Mface[f]
            sJ = geo.sJ[k, f]
            if k2 == k and f2 == f:           # PEC wall: [Ez] = 2 Ez-, [H] = 0
                e = ez[idM]
                val = sJ * e @ Mf @ e
                total += -alpha * (val / Z[k] if material else val)
                continue
            if k2 < k or (k2 == k and f2 < f):  # count each interior face once
                continue
            nx, ny = geo.nx[k, f], geo.ny[k, f]
            dE = ez[idM] - ez[idP]
            dHt = nx * (hy[idM] - hy[idP]) - ny * (hx[idM] - hx[idP])
            if material:
                Zm, Zp = Z[k], Z[k2]
                total += -alpha * sJ * (dE @ Mf @ dE + Zm * Zp * (dHt @ Mf @ dHt)) / (Zm + Zp)
            else:
                total += -0.5 * alpha * sJ * (dE @ Mf @ dE + dHt @ Mf @ dHt)
    return total
