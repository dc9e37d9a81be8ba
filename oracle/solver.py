"""Convenience driver over the oracle pieces (TEST INFRASTRUCTURE).

setup:  refelem.build -> mesh.orient -> mesh.connect -> mesh.geometry ->
        mesh.maps -> operator.surfinfo          (SURVEY.md §3 call stack 3)
run:    for step: lserk4.step(rhs)
"""
from __future__ import annotations

import numpy as np

from . import energy as _energy
from . import lserk4, mesh, operator, refelem


class Oracle:
    def __init__(self, N, VX, VY, EToV, eps=None, mu=None, alpha=1.0):
        self.N = N
        self.alpha = float(alpha)
        self.ref = refelem.build(N)
        self.VX = np.asarray(VX, dtype=np.float64)
        self.VY = np.asarray(VY, dtype=np.float64)
        self.EToV, self.n_swapped = mesh.orient(self.VX, self.VY, np.asarray(EToV))
        self.K = self.EToV.shape[0]
        self.EToE, self.EToF = mesh.connect(self.EToV)
        self.geo = mesh.geometry(self.VX, self.VY, self.EToV, self.ref)
        self.vmapM, self.vmapP = mesh.maps(self.ref, self.geo, self.EToE, self.EToF,
                                           self.EToV, self.VX, self.VY)
        self.si = operator.surfinfo(self.ref, self.geo, self.vmapM, self.vmapP, self.EToE, self.EToF)
        self.eps = None if eps is None else np.asarray(eps, dtype=np.float64)
        self.mu = None if mu is None else np.asarray(mu, dtype=np.float64)

    @property
    def Np(self):
        return self.ref.Np

    def rhs(self, q, which="full"):
        Hx, Hy, Ez = q
        return operator.rhs(self.ref, self.geo, self.si, Hx, Hy, Ez, self.alpha,
                            self.eps, self.mu, self.EToE, which)

    def run(self, q0, dt, nsteps, res0=None, callback=None):
        q = tuple(np.array(a, dtype=np.float64) for a in q0)
        res = tuple(np.zeros_like(a) for a in q) if res0 is None else res0
        for n in range(nsteps):
            q, res = lserk4.step(q, res, dt, self.rhs)
            if callback is not None:
                callback(n + 1, q)
        return q

    def energy(self, q):
        return _energy.energy(self.ref, self.geo, *q, eps=self.eps, mu=self.mu)
