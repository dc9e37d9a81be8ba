"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NONE of the DG method's arithmetic (no basis, operators,
geometry, flux or time stepping).  It only produces what a user would hand to
``dg_setup`` / ``dg_set_fields`` / ``dg_run``:

* the structured unit-square triangulation of SURVEY.md §8(c) A16
  (vertex id = j*(nx+1)+i; cell (i,j) -> elements 2(j*nx+i) = (v00,v10,v11)
  and 2(j*nx+i)+1 = (v00,v11,v01), both counter-clockwise);
* the exact PEC-cavity mode of the (corrected) TM system
  (eq. 2a-c with the A1 reading), formula as SPEC.md:431;
* the exact two-layer cavity mode for the
  piecewise-constant material extension (A12);
* seeded perturbations (np.random.default_rng(20261017));
* a CFL time-step estimate (dt is a caller input, A13).
"""
from __future__ import annotations

import math

import numpy as np

SEED = 20261017
# Config C4 parity start time: the (1,1) cavity mode at phase w t0 = pi/4 (w = pi sqrt 2), where
# |Ez| = cos(pi/4) and |H| = (pi/w) sin(pi/4) = 1/2 -- every field is O(1), so the per-field A14
# quotient is well conditioned (A14)
C4_T0 = 0.25 / math.sqrt(2.0)


def balanced_start(T, m=1, n=1):
    """Start time t0 of the exact cavity mode (m, n) such that the state at the END of a run of length
    T has phase w (t0 + T) = pi/4: every field is O(1) where a parity test measures it, so the per-field
    A14 quotient is well conditioned (DESIGN.md §2 A14).  t0 may be negative (the exact mode is valid
    for every t)."""
    w = math.pi * math.sqrt(m * m + n * n)
    return math.pi / (4.0 * w) - T


# ----------------------------------------------------------------------------
# Mesh
# ----------------------------------------------------------------------------
def rect_mesh(nx: int, ny: int | None = None, x0=0.0, x1=1.0, y0=0.0, y1=1.0):
    """Structured triangulation of [x0,x1]x[y0,y1] into 2*nx*ny CCW triangles.

    Returns (VX, VY, EToV) with EToV int64 [K][3], 0-based.
    """
    if ny is None:
        ny = nx
    if nx < 1 or ny < 1 or not (x1 > x0 and y1 > y0):
        raise ValueError("degenerate rectangle mesh request")
    xs = np.linspace(x0, x1, nx + 1)
    ys = np.linspace(y0, y1, ny + 1)
    VX = np.tile(xs, ny + 1)
    VY = np.repeat(ys, nx + 1)
    i = np.tile(np.arange(nx), ny)
    j = np.repeat(np.arange(ny), nx)
    v00 = j * (nx + 1) + i
    v10 = v00 + 1
    v01 = v00 + (nx + 1)
    v11 = v01 + 1
    EToV = np.empty((2 * nx * ny, 3), dtype=np.int64)
    EToV[0::2] = np.stack([v00, v10, v11], axis=1)
    EToV[1::2] = np.stack([v00, v11, v01], axis=1)
    return VX, VY, EToV


def jittered_mesh(n: int, amp=0.25, seed=7):
    """The A16 n x n mesh with every interior vertex moved by a seeded uniform offset of up to
    amp/n in x and y (general affine elements: no two share a Jacobian)."""
    VX, VY, E = rect_mesh(n)
    rng = np.random.default_rng(seed)
    inner = (VX > 0) & (VX < 1) & (VY > 0) & (VY < 1)
    VX = VX + amp / n * rng.uniform(-1, 1, VX.shape) * inner
    VY = VY + amp / n * rng.uniform(-1, 1, VY.shape) * inner
    return VX, VY, E


def two_layer_material(VX, VY, EToV, eps_right=2.25, x_interface=0.5):
    """Piecewise-constant eps (1 | eps_right at x = x_interface), mu = 1 (config C5)."""
    xc = VX[EToV].mean(axis=1)
    eps = np.where(xc > x_interface, eps_right, 1.0)
    mu = np.ones_like(eps)
    return eps, mu


# ----------------------------------------------------------------------------
# Exact solutions
# ----------------------------------------------------------------------------
def cavity_mode(x, y, t, m=1, n=1):
    """Exact PEC unit-square cavity mode.

    Ez = sin(m pi x) sin(n pi y) cos(w t)
    Hx = -(n pi / w) sin(m pi x) cos(n pi y) sin(w t)
    Hy =  (m pi / w) cos(m pi x) sin(n pi y) sin(w t),   w = pi sqrt(m^2+n^2)
    """
    w = math.pi * math.sqrt(m * m + n * n)
    sx, cx = np.sin(m * math.pi * x), np.cos(m * math.pi * x)
    sy, cy = np.sin(n * math.pi * y), np.cos(n * math.pi * y)
    Ez = sx * sy * math.cos(w * t)
    Hx = -(n * math.pi / w) * sx * cy * math.sin(w * t)
    Hy = (m * math.pi / w) * cx * sy * math.sin(w * t)
    return Hx, Hy, Ez


def two_layer_omega(eps1=1.0, eps2=2.25, mu1=1.0, mu2=1.0):
    """First root w (both k_i real) of (k1/mu1) cot(k1/2) = -(k2/mu2) cot(k2/2),
    k_i^2 = w^2 eps_i mu_i - pi^2 (y-mode 1).
    Written as k1/mu1 cos(k1/2) sin(k2/2) + k2/mu2 cos(k2/2) sin(k1/2) = 0."""
    def f(w):
        k1 = math.sqrt(w * w * eps1 * mu1 - math.pi ** 2)
        k2 = math.sqrt(w * w * eps2 * mu2 - math.pi ** 2)
        return (k1 / mu1) * math.cos(k1 / 2) * math.sin(k2 / 2) + \
               (k2 / mu2) * math.cos(k2 / 2) * math.sin(k1 / 2)
    # scan upward from where both wavenumbers are real for the first sign change, then bisect
    w0 = math.pi / math.sqrt(min(eps1 * mu1, eps2 * mu2)) * (1 + 1e-9)
    step = 1e-3
    a = w0
    fa = f(a)
    while True:
        b = a + step
        fb = f(b)
        if fa == 0.0:
            return a
        if fa * fb < 0:
            break
        a, fa = b, fb
        if a > 100:
            raise RuntimeError("no root found")
    for _ in range(200):
        mid = 0.5 * (a + b)
        fm = f(mid)
        if fa * fm <= 0:
            b = mid
        else:
            a, fa = mid, fm
    return 0.5 * (a + b)


def two_layer_mode(x, y, t, side, eps1=1.0, eps2=2.25, mu1=1.0, mu2=1.0, omega=None):
    """Exact two-layer cavity mode.

    ``side`` is 0 (x < 1/2, eps1) or 1 (x > 1/2, eps2) per point; each element
    takes X from its own side so the interface sits on element faces.
    """
    w = omega if omega is not None else two_layer_omega(eps1, eps2, mu1, mu2)
    k1 = math.sqrt(w * w * eps1 * mu1 - math.pi ** 2)
    k2 = math.sqrt(w * w * eps2 * mu2 - math.pi ** 2)
    C = math.sin(k1 / 2) / math.sin(k2 / 2)
    side = np.asarray(side)
    X = np.where(side == 0, np.sin(k1 * x), C * np.sin(k2 * (1 - x)))
    dX = np.where(side == 0, k1 * np.cos(k1 * x), -C * k2 * np.cos(k2 * (1 - x)))
    mu = np.where(side == 0, mu1, mu2)
    Ez = X * np.sin(math.pi * y) * math.cos(w * t)
    Hx = -(math.pi / (mu * w)) * X * np.cos(math.pi * y) * math.sin(w * t)
    Hy = (1.0 / (mu * w)) * dX * np.sin(math.pi * y) * math.sin(w * t)
    return Hx, Hy, Ez


def perturbation(shape, amplitude=1e-3, seed=SEED):
    """Seeded normal perturbation [3][...] (Hx, Hy, Ez), SURVEY.md §8(d)."""
    rng = np.random.default_rng(seed)
    return amplitude * rng.standard_normal((3,) + tuple(shape))


# ----------------------------------------------------------------------------
# Time step (a caller input, A13)
# ----------------------------------------------------------------------------
def cfl_dt(VX, VY, EToV, N, cfl=1.0, eps=None, mu=None):
    """dt = cfl * (2/3) * min_k(r_in,k * sqrt(eps_k mu_k)) * (x1 - x0) where
    r_in is the inscribed radius and x0 < x1 the first two Gauss-Legendre nodes
    of order N+1 (numpy.polynomial.legendre.leggauss)."""
    P = np.stack([VX[EToV], VY[EToV]], axis=-1)
    l0 = np.linalg.norm(P[:, 1] - P[:, 0], axis=1)
    l1 = np.linalg.norm(P[:, 2] - P[:, 1], axis=1)
    l2 = np.linalg.norm(P[:, 0] - P[:, 2], axis=1)
    sper = 0.5 * (l0 + l1 + l2)
    area = np.sqrt(sper * (sper - l0) * (sper - l1) * (sper - l2))
    rin = area / sper
    if eps is not None:
        rin = rin * np.sqrt(np.asarray(eps) * (np.asarray(mu) if mu is not None else 1.0))
    g = np.sort(np.polynomial.legendre.leggauss(N + 1)[0])
    rmin = abs(g[1] - g[0]) if N >= 1 else 2.0
    return cfl * (2.0 / 3.0) * float(rin.min()) * rmin


# ----------------------------------------------------------------------------
# 3D (tetrahedral Maxwell, the paper's hedge workload)
# ----------------------------------------------------------------------------
def cube_tet_mesh(n: int):
    """Structured tetrahedral mesh of [0,1]^3: n^3 cells, each split into the 6 Kuhn tetrahedra
    (v000, v000 + e_a, v000 + e_a + e_b, v111) for the 6 axis orders (a, b, c) -- conforming across
    cells.  Vertex id = i + (n+1)(j + (n+1)k).  Returns (VX, VY, VZ, EToV int64 [6 n^3][4]); the
    elements come in either orientation (the setup re-orients them)."""
    import itertools

    if n < 1:
        raise ValueError("n >= 1")
    g = np.linspace(0.0, 1.0, n + 1)
    K3 = np.arange(n + 1)
    I, J, Kk = np.meshgrid(K3, K3, K3, indexing="ij")
    vid = lambda i, j, k: i + (n + 1) * (j + (n + 1) * k)  # noqa: E731
    VX = np.empty((n + 1) ** 3)
    VY = np.empty_like(VX)
    VZ = np.empty_like(VX)
    VX[vid(I, J, Kk)] = g[I]
    VY[vid(I, J, Kk)] = g[J]
    VZ[vid(I, J, Kk)] = g[Kk]
    ci, cj, ck = (a.ravel() for a in np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij"))
    order = np.argsort(ck * n * n + cj * n + ci, kind="stable")  # cells x fastest
    ci, cj, ck = ci[order], cj[order], ck[order]
    tets = []
    for perm in itertools.permutations(range(3)):
        p = [np.zeros(3, dtype=np.int64)]
        for ax in perm:
            nxt = p[-1].copy()
            nxt[ax] += 1
            p.append(nxt)
        tets.append(np.stack([vid(ci + q[0], cj + q[1], ck + q[2]) for q in p], axis=1))
    EToV = np.stack(tets, axis=1).reshape(-1, 4)
    return VX, VY, VZ, EToV


# the (1,1,1) PEC cube-cavity mode, E = (a1 cos sin sin, a2 sin cos sin, a3 sin sin cos) cos(wt),
# a1 + a2 + a3 = 0 (div E = 0), w = pi sqrt(3); H from dH/dt = -curl E has amplitudes
# (a3 - a2, a1 - a3, a2 - a1) = (-5, 4, 1): all six components non-zero (a per-field check of a field
# that is identically zero would only measure the perturbation)
CUBE_MODE_A = (1.0, 2.0, -3.0)


def cube_cavity_mode(x, y, z, t, a=CUBE_MODE_A):
    """Exact PEC unit-cube cavity mode (1,1,1) of mu dH/dt = -curl E, eps dE/dt = curl H (eps=mu=1).
    Returns (Hx, Hy, Hz, Ex, Ey, Ez)."""
    a1, a2, a3 = a
    w = math.pi * math.sqrt(3.0)
    sx, cx = np.sin(math.pi * x), np.cos(math.pi * x)
    sy, cy = np.sin(math.pi * y), np.cos(math.pi * y)
    sz, cz = np.sin(math.pi * z), np.cos(math.pi * z)
    ct, st = math.cos(w * t), math.sin(w * t)
    Ex = a1 * cx * sy * sz * ct
    Ey = a2 * sx * cy * sz * ct
    Ez = a3 * sx * sy * cz * ct
    k = -(math.pi / w) * st  # H = -(curl E)(x) sin(wt) / w
    Hx = k * (a3 - a2) * sx * cy * cz
    Hy = k * (a1 - a3) * cx * sy * cz
    Hz = k * (a2 - a1) * cx * cy * sz
    return Hx, Hy, Hz, Ex, Ey, Ez


def cube_balanced_start(T):
    """Start time whose run of length T ends at phase w t = pi/4 (every field O(1))."""
    w = math.pi * math.sqrt(3.0)
    return math.pi / (4.0 * w) - T


def cfl_dt_3d(VX, VY, VZ, EToV, N, cfl=1.0):
    """dt = cfl * (2/3) * min_k r_in,k * (x1 - x0): inscribed radius of each tetrahedron (3 V / total
    face area) times the first Gauss-Legendre node gap of order N+1 (the 2D estimate's rule)."""
    P = np.stack([VX[EToV], VY[EToV], VZ[EToV]], axis=-1)
    vol = np.abs(np.einsum("ki,ki->k", P[:, 1] - P[:, 0],
                           np.cross(P[:, 2] - P[:, 0], P[:, 3] - P[:, 0]))) / 6.0
    area = 0.0
    for a, b, c in ((0, 1, 2), (0, 1, 3), (1, 2, 3), (0, 2, 3)):
        area = area + 0.5 * np.linalg.norm(np.cross(P[:, b] - P[:, a], P[:, c] - P[:, a]), axis=1)
    rin = 3.0 * vol / area
    g, _ = np.polynomial.legendre.leggauss(N + 1)
    return cfl * (2.0 / 3.0) * float(rin.min()) * float(g[1] - g[0])
