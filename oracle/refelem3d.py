"""3D reference tetrahedron (TEST INFRASTRUCTURE, the paper's hedge workload,
PAPER.md:920-928 "Three Dimensions").

Reference tetrahedron {r, s, t >= -1, r + s + t <= -1}, vertices v0 (-1,-1,-1), v1 (1,-1,-1),
v2 (-1,1,-1), v3 (-1,-1,1).  The method is the 2D one one dimension up (PAPER.md:275-374 written
for d dimensions):
* nodes: warp-and-blend on the tetrahedron (the construction of warburton_explicit_2006, cited at
  PAPER.md:278-279): equispaced barycentric points on the equilateral tetrahedron, each face's 2D
  warp (the 2D construction, with the 3D alpha table) blended into the interior, mapped to (r,s,t);
  node order t slowest, then s, r fastest (reading A6-3D);
* basis: orthonormal Koornwinder-Dubiner modes in collapsed coordinates (a, b, c)
  (PAPER.md:320-324), mode order i, j, k with k fastest;
* Dr, Ds, Dt = V_{r,s,t} V^-1;
* M and the face mass matrices BY THEIR DEFINITION with collapsed Gauss quadrature (exact);
* Fmask: face 0 t = -1, face 1 s = -1, face 2 r + s + t = -1, face 3 r = -1 (vertex triples
  (0,1,2), (0,1,3), (1,2,3), (0,2,3)), nodes in increasing index;
* LIFT = M^-1 M^{dI} (eq. 8).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .jacobi import grad_jacobi_p, jacobi_gl, jacobi_p
from .refelem import vandermonde_2d

# Warp-and-blend alpha for the tetrahedron, N = 1..15 (the cited construction's optimised table);
# 1 beyond.  A convention like the 2D table (reading A6): pinned by the node set's symmetry, GLL
# edges and 2D-construction faces, not by the paper.
ALPHA_OPT_3D = [0.0, 0.0, 0.0, 0.1002, 1.1332, 1.5608, 1.3413, 1.2577, 1.1603, 1.10153,
                0.6080, 0.4523, 0.8856, 0.8717, 0.9655]
N_MIN, N_MAX = 1, 15
FACE_VERTS = ((0, 1, 2), (0, 1, 3), (1, 2, 3), (0, 2, 3))

# equilateral tetrahedron used by the construction
_V = np.array([[-1.0, -1.0 / math.sqrt(3.0), -1.0 / math.sqrt(6.0)],
               [1.0, -1.0 / math.sqrt(3.0), -1.0 / math.sqrt(6.0)],
               [0.0, 2.0 / math.sqrt(3.0), -1.0 / math.sqrt(6.0)],
               [0.0, 0.0, 3.0 / math.sqrt(6.0)]])


def equinodes(n: int):
    """Equispaced (r, s, t): t slowest, then s, r fastest."""
    r, s, t = [], [], []
    for kk in range(n + 1):
        for jj in range(n + 1 - kk):
            for ii in range(n + 1 - kk - jj):
                r.append(-1.0 + 2.0 * ii / n)
                s.append(-1.0 + 2.0 * jj / n)
                t.append(-1.0 + 2.0 * kk / n)
    return np.array(r), np.array(s), np.array(t)


def edge_warp(n: int, x):
    """(GLL - equispaced) interpolated at x and divided by 1 - x^2: the 1D warp of the 2D
    construction (refelem.warpfactor) written as the Lagrange sum with the (1 - x^2) factor
    cancelled analytically, so it is finite at x = +-1."""
    x = np.asarray(x, dtype=np.float64)
    xeq = np.linspace(-1.0, 1.0, n + 1)
    xgl = jacobi_gl(0, 0, n)
    out = np.zeros_like(x)
    for i in range(1, n):  # the end points' shifts are zero
        d = np.full_like(x, xgl[i] - xeq[i])
        for j in range(1, n):
            if j != i:
                d = d * (x - xeq[j]) / (xeq[i] - xeq[j])
        # l_i(x) = prod_{j != i} (x - x_j)/(x_i - x_j); the j = 0, n factors (x + 1)(x - 1) /
        # ((x_i + 1)(x_i - 1)) are divided by (1 - x^2) = -(x + 1)(x - 1)
        d = d / (-(xeq[i] + 1.0) * (xeq[i] - 1.0))
        out = out + d
    return out


def face_shift(n: int, alpha: float, L1, L2, L3):
    """The 2D warp-and-blend shift (dx, dy) of a face with barycentrics L1, L2, L3."""
    w1 = 4.0 * L2 * L3 * edge_warp(n, L3 - L2) * (1.0 + (alpha * L1) ** 2)
    w2 = 4.0 * L1 * L3 * edge_warp(n, L1 - L3) * (1.0 + (alpha * L2) ** 2)
    w3 = 4.0 * L1 * L2 * edge_warp(n, L2 - L1) * (1.0 + (alpha * L3) ** 2)
    dx = w1 + math.cos(2.0 * math.pi / 3.0) * w2 + math.cos(4.0 * math.pi / 3.0) * w3
    dy = math.sin(2.0 * math.pi / 3.0) * w2 + math.sin(4.0 * math.pi / 3.0) * w3
    return dx, dy


def nodes(n: int):
    """Warp-and-blend nodes (r, s, t) of degree n, Np = (n+1)(n+2)(n+3)/6."""
    alpha = ALPHA_OPT_3D[n - 1] if n <= 15 else 1.0
    tol = 1e-10
    r, s, t = equinodes(n)
    L1 = (1.0 + t) / 2.0
    L2 = (1.0 + s) / 2.0
    L3 = -(1.0 + r + s + t) / 2.0
    L4 = (1.0 + r) / 2.0
    v1, v2, v3, v4 = _V
    t1 = [v2 - v1, v2 - v1, v3 - v2, v3 - v1]
    t2 = [v3 - 0.5 * (v1 + v2), v4 - 0.5 * (v1 + v2), v4 - 0.5 * (v2 + v3), v4 - 0.5 * (v1 + v3)]
    t1 = [a / np.linalg.norm(a) for a in t1]
    t2 = [a / np.linalg.norm(a) for a in t2]
    X = np.outer(L3, v1) + np.outer(L4, v2) + np.outer(L2, v3) + np.outer(L1, v4)
    shift = np.zeros_like(X)
    for face in range(4):
        La, Lb, Lc, Ld = [(L1, L2, L3, L4), (L2, L1, L3, L4), (L3, L1, L4, L2), (L4, L1, L3, L2)][face]
        warp1, warp2 = face_shift(n, alpha, Lb, Lc, Ld)
        blend = Lb * Lc * Ld
        denom = (Lb + 0.5 * La) * (Lc + 0.5 * La) * (Ld + 0.5 * La)
        ok = denom > tol
        blend = np.where(ok, (1.0 + (alpha * La) ** 2) * blend / np.where(ok, denom, 1.0), blend)
        shift = shift + np.outer(blend * warp1, t1[face]) + np.outer(blend * warp2, t2[face])
        onface = (La < tol) & (((Lb > tol).astype(int) + (Lc > tol) + (Ld > tol)) < 3)
        shift[onface] = np.outer(warp1[onface], t1[face]) + np.outer(warp2[onface], t2[face])
    X = X + shift
    return xyz_to_rst(X[:, 0], X[:, 1], X[:, 2])


def xyz_to_rst(X, Y, Z):
    """Equilateral-tetrahedron coordinates -> (r, s, t): X = (v1+v2+v3+v0... ) affine inverse."""
    v1, v2, v3, v4 = _V
    rhs = np.stack([X, Y, Z]) - 0.5 * (v2 + v3 + v4 - v1)[:, None]
    A = np.stack([0.5 * (v2 - v1), 0.5 * (v3 - v1), 0.5 * (v4 - v1)], axis=1)
    rst = np.linalg.solve(A, rhs)
    return rst[0], rst[1], rst[2]


def rst_to_abc(r, s, t):
    """Collapsed coordinates a = 2(1+r)/(-s-t) - 1 (-1 where s + t = 0), b = 2(1+s)/(1-t) - 1
    (-1 where t = 1), c = t."""
    r, s, t = (np.asarray(v, dtype=np.float64) for v in (r, s, t))
    a = np.full_like(r, -1.0)
    m = (s + t) != 0.0
    a[m] = 2.0 * (1.0 + r[m]) / (-s[m] - t[m]) - 1.0
    b = np.full_like(r, -1.0)
    m = t != 1.0
    b[m] = 2.0 * (1.0 + s[m]) / (1.0 - t[m]) - 1.0
    return a, b, t.copy()


def modes(n: int):
    return [(i, j, k) for i in range(n + 1) for j in range(n + 1 - i) for k in range(n + 1 - i - j)]


def simplex_3dp(a, b, c, i, j, k):
    """phi_ijk = 2 sqrt(2) P_i(a) P_j^{(2i+1,0)}(b) (1-b)^i P_k^{(2i+2j+2,0)}(c) (1-c)^(i+j)."""
    h1 = jacobi_p(a, 0, 0, i)
    h2 = jacobi_p(b, 2 * i + 1, 0, j)
    h3 = jacobi_p(c, 2 * (i + j) + 2, 0, k)
    return 2.0 * math.sqrt(2.0) * h1 * h2 * (1.0 - b) ** i * h3 * (1.0 - c) ** (i + j)


def grad_simplex_3dp(a, b, c, i, j, k):
    """(d/dr, d/ds, d/dt) of phi_ijk by the chain rule through (a, b, c)."""
    fa, dfa = jacobi_p(a, 0, 0, i), grad_jacobi_p(a, 0, 0, i)
    gb, dgb = jacobi_p(b, 2 * i + 1, 0, j), grad_jacobi_p(b, 2 * i + 1, 0, j)
    hc, dhc = jacobi_p(c, 2 * (i + j) + 2, 0, k), grad_jacobi_p(c, 2 * (i + j) + 2, 0, k)
    dr = dfa * (gb * hc)
    if i > 0:
        dr = dr * (0.5 * (1.0 - b)) ** (i - 1)
    if i + j > 0:
        dr = dr * (0.5 * (1.0 - c)) ** (i + j - 1)
    ds = 0.5 * (1.0 + a) * dr
    tmp = dgb * (0.5 * (1.0 - b)) ** i
    if i > 0:
        tmp = tmp + (-0.5 * i) * (gb * (0.5 * (1.0 - b)) ** (i - 1))
    if i + j > 0:
        tmp = tmp * (0.5 * (1.0 - c)) ** (i + j - 1)
    tmp = fa * (tmp * hc)
    ds = ds + tmp
    dt = 0.5 * (1.0 + a) * dr + 0.5 * (1.0 + b) * tmp
    tmp = dhc * (0.5 * (1.0 - c)) ** (i + j)
    if i + j > 0:
        tmp = tmp - 0.5 * (i + j) * (hc * (0.5 * (1.0 - c)) ** (i + j - 1))
    tmp = fa * (gb * tmp)
    tmp = tmp * (0.5 * (1.0 - b)) ** i
    dt = dt + tmp
    scale = 2.0 ** (2 * i + j + 1.5)
    return dr * scale, ds * scale, dt * scale


def vandermonde_3d(n, r, s, t):
    a, b, c = rst_to_abc(r, s, t)
    return np.stack([simplex_3dp(a, b, c, *m) for m in modes(n)], axis=1)


def grad_vandermonde_3d(n, r, s, t):
    a, b, c = rst_to_abc(r, s, t)
    cols = [grad_simplex_3dp(a, b, c, *m) for m in modes(n)]
    return tuple(np.stack([col[d] for col in cols], axis=1) for d in range(3))


def tet_quadrature(q: int):
    """Collapsed tensor Gauss-Jacobi-free rule (Gauss-Legendre in each collapsed direction with the
    Duffy Jacobian), exact for total degree <= 2q - 3 in (r, s, t)."""
    g, w = np.polynomial.legendre.leggauss(q)
    A, B, C = np.meshgrid(g, g, g, indexing="ij")
    WA, WB, WC = np.meshgrid(w, w, w, indexing="ij")
    # (a, b, c) in [-1,1]^3 -> (r, s, t): t = c, s = (1+b)(1-c)/2 - 1, r = (1+a)(-s-t)/2 - 1
    t = C
    s = 0.5 * (1.0 + B) * (1.0 - C) - 1.0
    r = 0.5 * (1.0 + A) * (-s - t) - 1.0
    jac = 0.5 * (-s - t) * 0.5 * (1.0 - C)  # dr/da * ds/db (dt/dc = 1)
    return r.ravel(), s.ravel(), t.ravel(), (WA * WB * WC * jac).ravel()


def face_coords(f: int, u, v):
    """Face f's points from its 2D reference coordinates (u, v) on the reference triangle:
    f0 (u, v, -1), f1 (u, -1, v), f2 (-1-u-v, u, v), f3 (-1, u, v).  The face's own 2D coordinates
    are the two of (r, s, t) kept, as in the 2D lift construction (reading A8 one dimension up)."""
    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    m1 = -np.ones_like(u)
    return [(u, v, m1), (u, m1, v), (-1.0 - u - v, u, v), (m1, u, v)][f]


@dataclass
class RefTet:
    N: int
    Np: int
    Nfp: int
    r: np.ndarray
    s: np.ndarray
    t: np.ndarray
    V: np.ndarray
    Dr: np.ndarray
    Ds: np.ndarray
    Dt: np.ndarray
    M: np.ndarray
    Fmask: np.ndarray   # [4][Nfp]
    Mface: list         # 4 x [Nfp][Nfp], face reference coordinates (area 2)
    LIFT: np.ndarray    # [Np][4 Nfp]

    def lagrange_at(self, r, s, t):
        return np.linalg.solve(self.V.T, vandermonde_3d(self.N, r, s, t).T).T


def build(n: int) -> RefTet:
    if not (N_MIN <= n <= N_MAX):
        raise ValueError(f"degree {n} outside [{N_MIN}, {N_MAX}]")
    Np = (n + 1) * (n + 2) * (n + 3) // 6
    Nfp = (n + 1) * (n + 2) // 2
    r, s, t = nodes(n)
    V = vandermonde_3d(n, r, s, t)
    Vr, Vs, Vt = grad_vandermonde_3d(n, r, s, t)
    Dr = np.linalg.solve(V.T, Vr.T).T
    Ds = np.linalg.solve(V.T, Vs.T).T
    Dt = np.linalg.solve(V.T, Vt.T).T
    ref = RefTet(n, Np, Nfp, r, s, t, V, Dr, Ds, Dt, None, None, None, None)
    qr, qs, qt, qw = tet_quadrature(n + 3)
    L = ref.lagrange_at(qr, qs, qt)
    ref.M = (L * qw[:, None]).T @ L
    tol = 1e-10
    masks = [np.abs(1.0 + t) < tol, np.abs(1.0 + s) < tol, np.abs(1.0 + r + s + t) < tol, np.abs(1.0 + r) < tol]
    ref.Fmask = np.stack([np.nonzero(m)[0] for m in masks]).astype(np.int64)
    assert ref.Fmask.shape == (4, Nfp)
    # face mass matrices int_face l_i l_j dA over the face's 2D reference triangle (area 2)
    from .refelem import triangle_quadrature
    fu, fv, fw = triangle_quadrature(n + 2)
    Mdi = np.zeros((Np, 4 * Nfp))
    ref.Mface = []
    for f in range(4):
        Lf = ref.lagrange_at(*face_coords(f, fu, fv))
        Mf = (Lf * fw[:, None]).T @ Lf
        ref.Mface.append(Mf[np.ix_(ref.Fmask[f], ref.Fmask[f])])
        Mdi[:, f * Nfp:(f + 1) * Nfp] = Mf[:, ref.Fmask[f]]
    ref.LIFT = np.linalg.solve(ref.M, Mdi)
    return ref


def face_vandermonde(ref: RefTet, f: int):
    """2D Vandermonde of face f's nodes in its own (u, v) coordinates (for tests)."""
    cols = [(ref.r, ref.s), (ref.r, ref.t), (ref.s, ref.t), (ref.s, ref.t)][f]
    ids = ref.Fmask[f]
    return vandermonde_2d(ref.N, cols[0][ids], cols[1][ids])
