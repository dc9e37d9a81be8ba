"""O2-O4: the reference triangle (TEST INFRASTRUCTURE).

Reference triangle I = {(r,s): r,s >= -1, r+s <= 0}, vertices (-1,-1), (1,-1),
(-1,1).  Follows:
* nodes: warp-and-blend (PAPER.md:275-279 cites warburton_explicit_2006;
  construction and alpha table per SURVEY.md §8(c) O2 and Appendix A; reading
  A6).  Node order: r fastest, rows bottom -> top.
* basis: orthonormal Koornwinder-Dubiner polynomials (
  SURVEY O3; collapsed coordinates with a := -1 on s = 1).
* Dr = Vr V^-1, Ds = Vs V^-1: the matrices D^{d nu} of PAPER.md:296-299.
* mass matrix M_ij = int_I l_i l_j dV and face mass
  matrices M^Gamma_ij = int_Gamma l_i l_j dS are computed
  BY THEIR DEFINITION with a tensor Gauss quadrature (exact for these
  polynomial degrees), each face parametrised by t in [-1, 1] (reading A8:
  the face Jacobian J_n = sJ = L/2 is applied separately, on every face).
* M^{dI} concatenates the three face blocks (eq. 8);
  LIFT = M^{-1} M^{dI}.
* Fmask_f = node indices on face f (s=-1 / r+s=0 / r=-1, tol 1e-12) in
  increasing node index (reading A9).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .jacobi import grad_jacobi_p, jacobi_gl, jacobi_p, vandermonde_1d

# Warp-and-blend optimised alpha, N = 1..15; 5/3 beyond.
ALPHA_OPT = [0.0000, 0.0000, 1.4152, 0.1001, 0.2751, 0.9800, 1.0999, 1.2832,
             1.3648, 1.4773, 1.4959, 1.5743, 1.5770, 1.6223, 1.6258]

N_MIN, N_MAX = 1, 15


def warpfactor(n: int, rout):
    """1D edge warp: interpolate (GLL - equispaced) at rout, divided by 1 - r^2
    in the interior and set to 0 at the ends."""
    rout = np.asarray(rout, dtype=np.float64)
    lglr = jacobi_gl(0, 0, n)
    req = np.linspace(-1.0, 1.0, n + 1)
    veq = vandermonde_1d(n, req)
    pmat = np.stack([jacobi_p(rout, 0, 0, i) for i in range(n + 1)], axis=0)
    lmat = np.linalg.solve(veq.T, pmat)
    warp = lmat.T @ (lglr - req)
    zerof = np.abs(rout) < 1.0 - 1.0e-10
    sf = 1.0 - (zerof * rout) ** 2
    return warp / sf + warp * (zerof - 1.0)


def nodes_equilateral(n: int):
    """Warp-and-blend nodes on the equilateral triangle."""
    alpha = ALPHA_OPT[n - 1] if n < 16 else 5.0 / 3.0
    L1, L3 = [], []
    for row in range(n + 1):          # L1 = row / N (bottom row first)
        for m in range(n + 1 - row):  # L3 = m / N (r fastest)
            L1.append(row / n)
            L3.append(m / n)
    L1 = np.array(L1)
    L3 = np.array(L3)
    L2 = 1.0 - L1 - L3
    x = -L2 + L3
    y = (-L2 - L3 + 2.0 * L1) / math.sqrt(3.0)
    blend1 = 4.0 * L2 * L3
    blend2 = 4.0 * L1 * L3
    blend3 = 4.0 * L1 * L2
    warpf1 = warpfactor(n, L3 - L2)
    warpf2 = warpfactor(n, L1 - L3)
    warpf3 = warpfactor(n, L2 - L1)
    warp1 = blend1 * warpf1 * (1.0 + (alpha * L1) ** 2)
    warp2 = blend2 * warpf2 * (1.0 + (alpha * L2) ** 2)
    warp3 = blend3 * warpf3 * (1.0 + (alpha * L3) ** 2)
    x = x + 1.0 * warp1 + math.cos(2.0 * math.pi / 3.0) * warp2 + math.cos(4.0 * math.pi / 3.0) * warp3
    y = y + 0.0 * warp1 + math.sin(2.0 * math.pi / 3.0) * warp2 + math.sin(4.0 * math.pi / 3.0) * warp3
    return x, y


def xy_to_rs(x, y):
    """Equilateral (x, y) -> reference (r, s)."""
    L1 = (math.sqrt(3.0) * y + 1.0) / 3.0
    L2 = (-3.0 * x - math.sqrt(3.0) * y + 2.0) / 6.0
    L3 = (3.0 * x - math.sqrt(3.0) * y + 2.0) / 6.0
    r = -L2 + L3 - L1
    s = -L2 - L3 + L1
    return r, s


def nodes(n: int):
    """Warp-and-blend nodes (r, s) of degree n, Np = (n+1)(n+2)/2."""
    x, y = nodes_equilateral(n)
    return xy_to_rs(x, y)


def rs_to_ab(r, s):
    """Collapsed coordinates a = 2(1+r)/(1-s) - 1 (a := -1 at s = 1), b = s."""
    r = np.asarray(r, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    a = np.empty_like(r)
    top = s == 1.0
    a[~top] = 2.0 * (1.0 + r[~top]) / (1.0 - s[~top]) - 1.0
    a[top] = -1.0
    return a, s.copy()


def simplex_2dp(a, b, i: int, j: int):
    """Orthonormal mode phi_ij = sqrt(2) P_i(a) P_j^{(2i+1,0)}(b) (1-b)^i."""
    h1 = jacobi_p(a, 0, 0, i)
    h2 = jacobi_p(b, 2 * i + 1, 0, j)
    return math.sqrt(2.0) * h1 * h2 * (1.0 - b) ** i


def grad_simplex_2dp(a, b, i: int, j: int):
    """(d/dr, d/ds) of phi_ij by the chain rule through (a, b)."""
    fa = jacobi_p(a, 0, 0, i)
    dfa = grad_jacobi_p(a, 0, 0, i)
    gb = jacobi_p(b, 2 * i + 1, 0, j)
    dgb = grad_jacobi_p(b, 2 * i + 1, 0, j)
    dr = dfa * gb
    if i > 0:
        dr = dr * (0.5 * (1.0 - b)) ** (i - 1)
    ds = dfa * (gb * (0.5 * (1.0 + a)))
    if i > 0:
        ds = ds * (0.5 * (1.0 - b)) ** (i - 1)
    tmp = dgb * (0.5 * (1.0 - b)) ** i
    if i > 0:
        tmp = tmp - 0.5 * i * gb * (0.5 * (1.0 - b)) ** (i - 1)
    ds = ds + fa * tmp
    dr = 2.0 ** (i + 0.5) * dr
    ds = 2.0 ** (i + 0.5) * ds
    return dr, ds


def modes(n: int):
    """Mode order: i outer, j inner, i + j <= n."""
    return [(i, j) for i in range(n + 1) for j in range(n + 1 - i)]


def vandermonde_2d(n: int, r, s):
    a, b = rs_to_ab(r, s)
    return np.stack([simplex_2dp(a, b, i, j) for (i, j) in modes(n)], axis=1)


def grad_vandermonde_2d(n: int, r, s):
    a, b = rs_to_ab(r, s)
    cols = [grad_simplex_2dp(a, b, i, j) for (i, j) in modes(n)]
    return np.stack([c[0] for c in cols], axis=1), np.stack([c[1] for c in cols], axis=1)


def triangle_quadrature(q: int):
    """Collapsed tensor Gauss rule on I with q x q points (exact for total
    degree <= 2q-2 in (r, s)); numpy's Gauss-Legendre is the library primitive."""
    g, w = np.polynomial.legendre.leggauss(q)
    A, B = np.meshgrid(g, g, indexing="ij")
    WA, WB = np.meshgrid(w, w, indexing="ij")
    r = 0.5 * (1.0 + A) * (1.0 - B) - 1.0
    s = B
    wt = WA * WB * 0.5 * (1.0 - B)
    return r.ravel(), s.ravel(), wt.ravel()


def face_points(f: int, t):
    """Face parametrisation t in [-1, 1] in increasing-node-index direction:
    f0: (t, -1) from v0 to v1; f1: (-t, t) from v1 to v2; f2: (-1, t) from v0 to v2."""
    t = np.asarray(t, dtype=np.float64)
    if f == 0:
        return t, -np.ones_like(t)
    if f == 1:
        return -t, t
    return -np.ones_like(t), t


@dataclass
class RefElement:
    N: int
    Np: int
    Nfp: int
    r: np.ndarray
    s: np.ndarray
    V: np.ndarray
    Vr: np.ndarray
    Vs: np.ndarray
    Dr: np.ndarray
    Ds: np.ndarray
    M: np.ndarray          # reference mass matrix, by quadrature
    Mface: list            # three Nfp x Nfp face mass matrices (t in [-1,1])
    Fmask: np.ndarray      # [3][Nfp]
    LIFT: np.ndarray       # Np x 3Nfp

    def lagrange_at(self, r, s):
        """Values l_j(r, s) of the nodal basis at points: Phi(r,s) V^{-1}."""
        return np.linalg.solve(self.V.T, vandermonde_2d(self.N, r, s).T).T


def build(n: int) -> RefElement:
    """Reference element of degree n (SPEC.md:70-78 interface)."""
    if not (N_MIN <= n <= N_MAX):
        raise ValueError(f"degree {n} outside [{N_MIN}, {N_MAX}]")
    Np = (n + 1) * (n + 2) // 2
    Nfp = n + 1
    r, s = nodes(n)
    V = vandermonde_2d(n, r, s)
    Vr, Vs = grad_vandermonde_2d(n, r, s)
    # D = Vr V^{-1}  <=>  D V = Vr  <=>  V^T D^T = Vr^T
    Dr = np.linalg.solve(V.T, Vr.T).T
    Ds = np.linalg.solve(V.T, Vs.T).T
    ref = RefElement(n, Np, Nfp, r, s, V, Vr, Vs, Dr, Ds, None, None, None, None)
    # mass matrix by its definition, int_I l_i l_j
    qr, qs, qw = triangle_quadrature(n + 2)
    L = ref.lagrange_at(qr, qs)
    ref.M = (L * qw[:, None]).T @ L
    # face masks
    tol = 1e-12
    f0 = np.nonzero(np.abs(s + 1.0) < tol)[0]
    f1 = np.nonzero(np.abs(r + s) < tol)[0]
    f2 = np.nonzero(np.abs(r + 1.0) < tol)[0]
    ref.Fmask = np.stack([f0, f1, f2]).astype(np.int64)
    assert ref.Fmask.shape == (3, Nfp)
    # face mass matrices by their definition, int_{-1}^{1} l_i l_j dt
    g, w = np.polynomial.legendre.leggauss(n + 2)
    ref.Mface = []
    Mdi = np.zeros((Np, 3 * Nfp))
    for f in range(3):
        fr, fs = face_points(f, g)
        Lf = ref.lagrange_at(fr, fs)                 # [q][Np]
        Mf_full = (Lf * w[:, None]).T @ Lf          # [Np][Np], zero off the face rows
        ref.Mface.append(Mf_full[np.ix_(ref.Fmask[f], ref.Fmask[f])])
        Mdi[:, f * Nfp:(f + 1) * Nfp] = Mf_full[:, ref.Fmask[f]]
    ref.LIFT = np.linalg.solve(ref.M, Mdi)
    return ref
