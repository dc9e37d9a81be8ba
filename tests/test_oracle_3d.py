"""Pins of the 3D oracle (oracle/refelem3d.py, mesh3d.py, maxwell3d.py) against
what mathematics fixes: exact differentiation, orthonormality, the reference volume, lift consistency,
the node set's symmetry / GLL edges / 2D-construction faces, closed element surfaces, the face-map
involution, exact curls, the energy-rate identity (signs, the 1/2, the PEC mirror) and convergence
to the exact PEC cube-cavity mode."""
import itertools
import math

import numpy as np
import pytest

import dginputs
from oracle import jacobi, refelem
from oracle import refelem3d as R3
from oracle.maxwell3d import Oracle3D


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6])
def test_reference_tet_operators(N):
    ref = R3.build(N)
    assert ref.Np == (N + 1) * (N + 2) * (N + 3) // 6 and ref.Nfp == (N + 1) * (N + 2) // 2
    err = 0.0
    for a in range(N + 1):
        for b in range(N + 1 - a):
            for c in range(N + 1 - a - b):
                u = ref.r ** a * ref.s ** b * ref.t ** c
                du = (a * ref.r ** max(a - 1, 0) * ref.s ** b * ref.t ** c,
                      b * ref.r ** a * ref.s ** max(b - 1, 0) * ref.t ** c,
                      c * ref.r ** a * ref.s ** b * ref.t ** max(c - 1, 0))
                for D, d in zip((ref.Dr, ref.Ds, ref.Dt), du):
                    err = max(err, np.abs(D @ u - d).max())
    assert err < 1e-12
    one = np.ones(ref.Np)
    assert abs(one @ ref.M @ one - 4.0 / 3.0) < 1e-13          # |reference tetrahedron| = 4/3
    assert np.abs(ref.V.T @ ref.M @ ref.V - np.eye(ref.Np)).max() < 1e-12   # orthonormal modes
    for f in range(4):                                          # lift consistency: face area 2
        blk = ref.LIFT[:, f * ref.Nfp:(f + 1) * ref.Nfp]
        assert abs(one @ ref.M @ blk @ np.ones(ref.Nfp) - 2.0) < 1e-12


@pytest.mark.parametrize("N", [2, 3, 4, 5])
def test_node_set_symmetry_edges_and_faces(N):
    r, s, t = R3.nodes(N)
    L = np.stack([-(1 + r + s + t) / 2, (1 + r) / 2, (1 + s) / 2, (1 + t) / 2], axis=1)
    key = lambda A: np.array(sorted(map(tuple, np.round(A, 10))))  # noqa: E731
    base = key(L)
    for p in itertools.permutations(range(4)):                 # invariant under the tet's symmetries
        assert np.abs(key(L[:, list(p)]) - base).max() < 1e-12
    e = (np.abs(s + 1) < 1e-10) & (np.abs(t + 1) < 1e-10)        # edge nodes = Gauss-Lobatto points
    assert np.abs(np.sort(r[e]) - jacobi.jacobi_gl(0, 0, N)).max() < 1e-14
    # face t = -1 = the 2D warp-and-blend set (the independent 2D implementation, refelem) built with
    # the 3D alpha
    saved = refelem.ALPHA_OPT[N - 1]
    try:
        refelem.ALPHA_OPT[N - 1] = R3.ALPHA_OPT_3D[N - 1]
        r2, s2 = refelem.nodes(N)
    finally:
        refelem.ALPHA_OPT[N - 1] = saved
    f0 = np.abs(t + 1) < 1e-10
    a = np.array(sorted(zip(np.round(r[f0], 11), np.round(s[f0], 11))))
    b = np.array(sorted(zip(np.round(r2, 11), np.round(s2, 11))))
    assert np.abs(a - b).max() < 1e-10


def _jittered_cube(n, amp=0.05, seed=3):
    VX, VY, VZ, E = dginputs.cube_tet_mesh(n)
    rng = np.random.default_rng(seed)
    inner = (VX > 0) & (VX < 1) & (VY > 0) & (VY < 1) & (VZ > 0) & (VZ < 1)
    return (VX + amp * rng.uniform(-1, 1, VX.shape) * inner, VY + amp * rng.uniform(-1, 1, VX.shape) * inner,
            VZ + amp * rng.uniform(-1, 1, VX.shape) * inner, E)


def test_mesh_geometry_and_maps():
    VX, VY, VZ, E = _jittered_cube(2)
    o = Oracle3D(3, VX, VY, VZ, E)
    assert o.K == 48 and o.n_swapped == 24
    one = np.ones(o.Np)
    assert abs(float(o.geo.J.sum() * (one @ o.ref.M @ one)) - 1.0) < 1e-12   # volume of the cube
    # closed surfaces: sum_f area_f n_f = 0 (area = 2 sJ)
    Sn = np.stack([(2 * o.geo.sJ * c).sum(axis=1) for c in (o.geo.nx, o.geo.ny, o.geo.nz)], axis=1)
    assert np.abs(Sn).max() < 1e-13
    # boundary faces lie on the cube's surface with the outward normal
    K = o.K
    for k in range(K):
        for f in range(4):
            if o.bnd[k, f]:
                ids = o.ref.Fmask[f]
                P = np.stack([o.geo.x[k, ids], o.geo.y[k, ids], o.geo.z[k, ids]], axis=1)
                n = np.array([o.geo.nx[k, f], o.geo.ny[k, f], o.geo.nz[k, f]])
                ax = int(np.argmax(np.abs(n)))
                assert abs(abs(n[ax]) - 1) < 1e-12 and np.ptp(P[:, ax]) < 1e-12
                assert (P[0, ax] > 0.5) == (n[ax] > 0)
    # vmapP is an involution face by face (a node can sit on several faces) and points at
    # coincident nodes
    for k in range(K):
        for f in range(4):
            k2, f2 = o.EToE[k, f], o.EToF[k, f]
            pair = dict(zip(o.vmapM[k2, f2], o.vmapP[k2, f2]))
            for m, p_ in zip(o.vmapM[k, f], o.vmapP[k, f]):
                assert pair[p_] == m
    vP = o.vmapP.ravel()
    vM = o.vmapM.ravel()
    X = np.stack([o.geo.x.ravel(), o.geo.y.ravel(), o.geo.z.ravel()], axis=1)
    assert np.abs(X[vM] - X[vP]).max() < 1e-12


def test_volume_curl_of_linear_fields_exact():
    VX, VY, VZ, E = _jittered_cube(2)
    o = Oracle3D(2, VX, VY, VZ, E)
    x, y, z = o.geo.x, o.geo.y, o.geo.z
    zero = np.zeros_like(x)
    # E = (y, z, x): curl E = (-1, -1, -1) -> dH/dt = (1, 1, 1); H = (z, x, y): curl H = (1, 1, 1)
    vol = o.rhs((z, x, y, y, z, x), which="volume")
    for c in range(3):
        assert np.abs(vol[c] - 1.0).max() < 1e-12
        assert np.abs(vol[3 + c] - 1.0).max() < 1e-12
    # the full operator of a smooth continuous field equals its volume term (no jumps) away from walls
    q = (zero, zero, zero, y * (1 - y), zero, zero)
    full, volq = o.rhs(q), o.rhs(q, which="volume")
    inner = ~o.bnd.any(axis=1)
    for a, b in zip(full, volq):
        assert np.abs(a[inner] - b[inner]).max() < 1e-11


@pytest.mark.parametrize("alpha", [1.0, 0.0])
def test_energy_rate_identity(alpha):
    """<q, R(q)>_M = -(alpha/2) sum_interior int (|n x [E]|^2 + |n x [H]|^2) - alpha sum_PEC int |n x E|^2
    for any q (interior faces counted once): pins the flux signs, the 1/2 and the PEC mirror."""
    VX, VY, VZ, E = _jittered_cube(2)
    o = Oracle3D(3, VX, VY, VZ, E, alpha=alpha)
    rng = np.random.default_rng(5)
    q = tuple(rng.standard_normal((o.K, o.Np)) for _ in range(6))
    lhs = sum(float(np.einsum("k,ki,ij,kj->", o.geo.J, a, o.ref.M, b)) for a, b in zip(q, o.rhs(q)))
    flat = [a.ravel() for a in q]
    rhs = 0.0
    for k in range(o.K):
        for f in range(4):
            iM, iP = o.vmapM[k, f], o.vmapP[k, f]
            n = np.array([o.geo.nx[k, f], o.geo.ny[k, f], o.geo.nz[k, f]])
            Mf = o.ref.Mface[f] * o.geo.sJ[k, f]
            if o.bnd[k, f]:
                nE = np.cross(n, np.stack([flat[3 + c][iM] for c in range(3)], axis=1))
                rhs -= alpha * sum(nE[:, c] @ Mf @ nE[:, c] for c in range(3))
            else:
                nE = np.cross(n, np.stack([flat[3 + c][iM] - flat[3 + c][iP] for c in range(3)], axis=1))
                nH = np.cross(n, np.stack([flat[c][iM] - flat[c][iP] for c in range(3)], axis=1))
                rhs -= 0.25 * alpha * sum(nE[:, c] @ Mf @ nE[:, c] + nH[:, c] @ Mf @ nH[:, c] for c in range(3))
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_cube_cavity_convergence():
    """The exact (1,1,1) PEC cube mode: N = 3, n = 1, 2, 4 cells per side, T = 0.1 -- observed rate
    approaching N + 1 (measured 2.8, 3.9)."""
    N, T = 3, 0.1
    errs = []
    for n in (1, 2, 4):
        VX, VY, VZ, E = dginputs.cube_tet_mesh(n)
        o = Oracle3D(N, VX, VY, VZ, E)
        steps = int(math.ceil(T / dginputs.cfl_dt_3d(VX, VY, VZ, E, N)))
        x, y, z = o.geo.x, o.geo.y, o.geo.z
        qT = o.run(dginputs.cube_cavity_mode(x, y, z, 0.0), T / steps, steps)
        d = [a - b for a, b in zip(qT, dginputs.cube_cavity_mode(x, y, z, T))]
        errs.append(math.sqrt(2.0 * o.energy(d)))
    rates = [math.log2(a / b) for a, b in zip(errs, errs[1:])]
    assert rates[0] > 2.5 and rates[1] > 3.5, (errs, rates)


def test_energy_non_increasing_and_conserved():
    VX, VY, VZ, E = dginputs.cube_tet_mesh(2)
    for alpha in (1.0, 0.0):
        o = Oracle3D(2, VX, VY, VZ, E, alpha=alpha)
        q = dginputs.cube_cavity_mode(o.geo.x, o.geo.y, o.geo.z, 0.05)
        q = tuple(a + b for a, b in zip(q, dginputs.perturbation(o.geo.x.shape, 1e-2)[[0, 1, 2, 0, 1, 2]]))
        # central flux (alpha = 0) conserves the semi-discrete energy; LSERK4 damps it only at
        # O(dt^4): the small step keeps that below 1e-6 over the run
        dt = dginputs.cfl_dt_3d(VX, VY, VZ, E, 2) * (1.0 if alpha == 1.0 else 0.1)
        Es = [o.energy(q)]
        for _ in range(5):
            q = o.run(q, dt, 4)
            Es.append(o.energy(q))
        if alpha == 1.0:
            assert all(b <= a * (1 + 1e-14) for a, b in zip(Es, Es[1:]))
        else:
            assert abs(Es[-1] / Es[0] - 1) < 1e-6
