"""Pins of oracle O5-O8 (connectivity, geometry, maps, flux, RHS) and O10 (energy).

Pins: SPEC.md:145-146, 165-166, 175-176, 190-191, 301, 311-312, 321, 346;
the closed-form neighbour rule of SURVEY.md §8(c) O7 (written here, not in the
oracle); exact polynomial derivatives; the energy-rate identity P11 (checks the
1/2 of reading A3, the signs of A1/A2, the PEC mirror A7 and alpha); its
material form (A12).
"""
import math

import numpy as np
import pytest

import dginputs
from conftest import floats, read_golden
from oracle import energy, mesh, operator, refelem
from oracle.solver import Oracle


# ---------------------------------------------------------------- mesh
def test_rect_mesh_counts():
    VX, VY, E = dginputs.rect_mesh(1)
    assert len(VX) == 4 and E.shape == (2, 3)
    VX, VY, E = dginputs.rect_mesh(2)
    assert len(VX) == 9 and E.shape == (8, 3)
    # CCW
    x, y = VX[E], VY[E]
    det = (x[:, 1] - x[:, 0]) * (y[:, 2] - y[:, 0]) - (x[:, 2] - x[:, 0]) * (y[:, 1] - y[:, 0])
    assert (det > 0).all()


def test_connect_conventions_and_involution():
    VX, VY, E = dginputs.rect_mesh(5, 3)
    EToE, EToF = mesh.connect(E)
    K = E.shape[0]
    nb = 0
    for k in range(K):
        for f in range(3):
            k2, f2 = EToE[k, f], EToF[k, f]
            if k2 == k:
                assert f2 == f
                nb += 1
            else:
                assert EToE[k2, f2] == k and EToF[k2, f2] == f
    assert nb == 2 * (5 + 3)  # boundary edges of a 5x3 grid
    # two-triangle square: exactly one shared face pair
    _, _, E2 = dginputs.rect_mesh(1)
    EE, EF = mesh.connect(E2)
    assert (EE != np.arange(2)[:, None]).sum() == 2
    # single triangle: EToE = [k,k,k]
    EE1, EF1 = mesh.connect(np.array([[0, 1, 2]]))
    assert EE1.tolist() == [[0, 0, 0]] and EF1.tolist() == [[0, 1, 2]]


def test_non_manifold_rejected():
    E = np.array([[0, 1, 2], [1, 0, 3], [0, 1, 4]])
    with pytest.raises(mesh.MeshError):
        mesh.connect(E)


def test_orientation_swap():
    VX = np.array([0.0, 1.0, 0.0])
    VY = np.array([0.0, 0.0, 1.0])
    E, n = mesh.orient(VX, VY, np.array([[0, 2, 1]]))
    assert n == 1 and E.tolist() == [[0, 1, 2]]


def test_geometry_spec_examples():
    g = read_golden("spec_geometry_examples.txt")
    ref = refelem.build(2)
    v = floats(g["ref_vertices"])
    geo = mesh.geometry(np.array(v[0::2]), np.array(v[1::2]), np.array([[0, 1, 2]]), ref)
    assert np.allclose([geo.rx[0], geo.sx[0], geo.ry[0], geo.sy[0], geo.J[0]], floats(g["ref_rx_sx_ry_sy_J"]))
    assert np.allclose([geo.nx[0, 0], geo.ny[0, 0]], floats(g["ref_face0_normal"]))
    v = floats(g["unit_vertices"])
    geo = mesh.geometry(np.array(v[0::2]), np.array(v[1::2]), np.array([[0, 1, 2]]), ref)
    assert abs(geo.J[0] - float(g["unit_J"])) < 1e-15
    assert np.allclose([geo.rx[0], geo.sx[0], geo.ry[0], geo.sy[0]], floats(g["unit_rx_sx_ry_sy"]))
    assert np.allclose([geo.nx[0, 1], geo.ny[0, 1]], floats(g["unit_face1_normal"]), atol=1e-15)
    # node coordinates of an affine copy reproduce the map of the vertices
    assert np.allclose(geo.x[0][[0, ref.Nfp - 1, ref.Np - 1]], [0, 1, 0])


def test_geometry_invariants_random_mesh():
    rng = np.random.default_rng(1)
    VX, VY, E = dginputs.rect_mesh(6, 5, 0, 3, 0, 2)
    VX = VX + 0.1 * rng.uniform(-1, 1, VX.shape) * ((VX > 0) & (VX < 3))
    VY = VY + 0.1 * rng.uniform(-1, 1, VY.shape) * ((VY > 0) & (VY < 2))
    ref = refelem.build(3)
    geo = mesh.geometry(VX, VY, E, ref)
    assert abs((2 * geo.J).sum() - 6.0) < 1e-12
    assert np.abs((geo.sJ * geo.nx).sum(1)).max() < 1e-14
    assert np.abs((geo.sJ * geo.ny).sum(1)).max() < 1e-14
    assert np.allclose(geo.nx ** 2 + geo.ny ** 2, 1.0)
    # A^-1 A = I: (rx, sx; ry, sy) times (xr, xs; yr, ys)
    x0, x1, x2 = (VX[E[:, i]] for i in range(3))
    y0, y1, y2 = (VY[E[:, i]] for i in range(3))
    xr, xs, yr, ys = (x1 - x0) / 2, (x2 - x0) / 2, (y1 - y0) / 2, (y2 - y0) / 2
    assert np.allclose(geo.rx * xr + geo.ry * yr, 1) and np.allclose(geo.rx * xs + geo.ry * ys, 0)
    assert np.allclose(geo.sx * xr + geo.sy * yr, 0) and np.allclose(geo.sx * xs + geo.sy * ys, 1)
    # sJ = L/2, Fsc = sJ/J
    L0 = np.hypot(x1 - x0, y1 - y0)
    assert np.allclose(geo.sJ[:, 0], L0 / 2) and np.allclose(geo.Fsc, geo.sJ / geo.J[:, None])


def _closed_form_vmapP(ref, EToE, EToF):
    """SURVEY.md §8(c) O7 closed-form rule, written independently of the oracle:
    traversal d = (+1, +1, -1) for faces (0, 1, 2); i' = Nfp-1-i if d_f == d_f' else i."""
    K = EToE.shape[0]
    d = [1, 1, -1]
    out = np.empty((K, 3, ref.Nfp), dtype=np.int64)
    for k in range(K):
        for f in range(3):
            k2, f2 = EToE[k, f], EToF[k, f]
            for i in range(ref.Nfp):
                if k2 == k and f2 == f:
                    out[k, f, i] = k * ref.Np + ref.Fmask[f][i]
                else:
                    i2 = ref.Nfp - 1 - i if d[f] == d[f2] else i
                    out[k, f, i] = k2 * ref.Np + ref.Fmask[f2][i2]
    return out


@pytest.mark.parametrize("N", [1, 2, 4, 7])
def test_maps_coordinates_and_closed_form(N):
    rng = np.random.default_rng(N)
    VX, VY, E = dginputs.rect_mesh(4, 3)
    VX = VX + 0.05 * rng.uniform(-1, 1, VX.shape) * ((VX > 0) & (VX < 1))
    o = Oracle(N, VX, VY, E)
    x, y = o.geo.x.ravel(), o.geo.y.ravel()
    assert np.abs(x[o.vmapM] - x[o.vmapP]).max() < 1e-9
    assert np.abs(y[o.vmapM] - y[o.vmapP]).max() < 1e-9
    assert np.array_equal(o.vmapP, _closed_form_vmapP(o.ref, o.EToE, o.EToF))
    # involution of the pairing
    flatM, flatP = o.vmapM.ravel(), o.vmapP.ravel()
    pos = {}
    for idx, (m, p) in enumerate(zip(flatM, flatP)):
        pos.setdefault(int(m), []).append(idx)
    for m, p in zip(flatM, flatP):
        assert any(flatP[j] == m for j in pos[int(p)])


# ---------------------------------------------------------------- flux / rhs
def test_spec_flux_example():
    g = read_golden("spec_flux_example.txt")
    si = dict(idM=np.array([0]), idP=np.array([0]), nx=np.array([float(g["nx"])]),
              ny=np.array([float(g["ny"])]), Fsc=np.array([float(g["Fsc"])]), Bsc=np.array([float(g["Bsc"])]))
    q = [np.array([float(g[k])]) for k in ("Hx", "Hy", "Ez")]
    for alpha, key in ((1.0, "alpha1_out"), (0.0, "alpha0_out")):
        out = operator.flux(si, *q, alpha=alpha)
        # the oracle lifts 1/2 of eq. 5 (reading A3): SPEC's pre-1/2 value times 1/2
        assert np.allclose([o[0] for o in out], 0.5 * np.array(floats(g[key])))


def _mesh(N, n=4, jitter=0.0, seed=3):
    VX, VY, E = dginputs.rect_mesh(n)
    if jitter:
        rng = np.random.default_rng(seed)
        inner = (VX > 0) & (VX < 1) & (VY > 0) & (VY < 1)
        VX = VX + jitter / n * rng.uniform(-1, 1, VX.shape) * inner
        VY = VY + jitter / n * rng.uniform(-1, 1, VY.shape) * inner
    return VX, VY, E


@pytest.mark.parametrize("N", [1, 3, 5])
def test_volume_linear_Ez(N):
    # Ez = y, H = 0 -> rhsHx = -1, rhsHy = 0, rhsEz = 0 (volume term)
    o = Oracle(N, *_mesh(N, 3, 0.3))
    Z = np.zeros_like(o.geo.x)
    r = o.rhs((Z, Z, o.geo.y.copy()), which="volume")
    assert np.allclose(r[0], -1, atol=1e-12) and np.allclose(r[1], 0, atol=1e-12)
    assert np.allclose(r[2], 0, atol=1e-12)


@pytest.mark.parametrize("N", [4, 6])
def test_full_rhs_exact_for_polynomial_fields_vanishing_on_wall(N):
    # Ez = x(1-x)y(1-y) vanishes on the PEC wall and is continuous; H polynomial
    # and continuous -> all jumps vanish, the RHS is the exact derivative of eq. 2
    o = Oracle(N, *_mesh(N, 3, 0.3))
    x, y = o.geo.x, o.geo.y
    Ez = x * (1 - x) * y * (1 - y)
    Hx = x ** 2 * y - 3 * y ** 3
    Hy = x * y * y + 2 * x
    r = o.rhs((Hx, Hy, Ez))
    Ez_x = (1 - 2 * x) * y * (1 - y)
    Ez_y = x * (1 - x) * (1 - 2 * y)
    Hy_x = y * y + 2
    Hx_y = x ** 2 - 9 * y ** 2
    assert np.allclose(r[0], -Ez_y, atol=1e-11)
    assert np.allclose(r[1], Ez_x, atol=1e-11)
    assert np.allclose(r[2], Hy_x - Hx_y, atol=1e-10)


def test_surface_lift_single_element_identity():
    # flux 1 on face 0 of Ez only -> 1^T M dEz = 1/2 * 2 = 1 (reference element)
    ref = refelem.build(3)
    f = np.zeros((1, 3, ref.Nfp))
    f[0, 0, :] = 0.5 * 1.0
    d = operator.lift(ref, f)
    assert abs(np.ones(ref.Np) @ ref.M @ d[0] - 1.0) < 1e-12


def test_rhs_linearity_and_determinism():
    o = Oracle(3, *_mesh(3, 3, 0.2))
    rng = np.random.default_rng(5)
    q1 = tuple(rng.standard_normal(o.geo.x.shape) for _ in range(3))
    q2 = tuple(rng.standard_normal(o.geo.x.shape) for _ in range(3))
    a, b = 0.7, -1.3
    lhs = o.rhs(tuple(a * u + b * v for u, v in zip(q1, q2)))
    r1, r2 = o.rhs(q1), o.rhs(q2)
    for L, u, v in zip(lhs, r1, r2):
        assert np.allclose(L, a * u + b * v, atol=1e-11 * max(1, np.abs(L).max()))
    again = o.rhs(q1)
    assert all(np.array_equal(u, v) for u, v in zip(r1, again))


@pytest.mark.parametrize("N,alpha", [(1, 1.0), (3, 0.0), (3, 1.0), (5, 1.0), (5, 0.0)])
def test_energy_rate_identity_constant_material(N, alpha):
    # <q, R(q)>_M equals the face-integral form; alpha = 0 conserves
    o = Oracle(N, *_mesh(N, 3, 0.3), alpha=alpha)
    rng = np.random.default_rng(N)
    q = tuple(rng.standard_normal(o.geo.x.shape) for _ in range(3))
    lhs = energy.energy_rate(o.ref, o.geo, q, o.rhs(q))
    rhs = energy.energy_rate_expected(o.ref, o.geo, o.si, o.EToE, o.EToF, *q, alpha)
    scale = energy.energy(o.ref, o.geo, *q) * o.geo.Fsc.max()
    assert abs(lhs - rhs) < 1e-12 * scale
    if alpha == 0.0:
        assert abs(lhs) < 1e-12 * scale
    else:
        assert lhs < 0


@pytest.mark.parametrize("alpha", [0.0, 1.0])
def test_energy_rate_identity_material(alpha):
    # reading A12: weighted identity with random piecewise-constant eps, mu
    N = 3
    VX, VY, E = _mesh(N, 3, 0.3)
    rng = np.random.default_rng(11)
    K = E.shape[0]
    eps = rng.uniform(1, 3, K)
    mu = rng.uniform(0.5, 2, K)
    o = Oracle(N, VX, VY, E, eps=eps, mu=mu, alpha=alpha)
    q = tuple(rng.standard_normal(o.geo.x.shape) for _ in range(3))
    lhs = energy.energy_rate(o.ref, o.geo, q, o.rhs(q), eps=eps, mu=mu)
    rhs = energy.energy_rate_expected(o.ref, o.geo, o.si, o.EToE, o.EToF, *q, alpha, eps=eps, mu=mu)
    scale = energy.energy(o.ref, o.geo, *q, eps=eps, mu=mu) * o.geo.Fsc.max()
    assert abs(lhs - rhs) < 1e-12 * scale


def test_material_reduces_to_constant_flux():
    # A12 with eps = mu = 1 equals 1/2 eq. 5 (to rounding)
    VX, VY, E = _mesh(3, 3, 0.3)
    o1 = Oracle(3, VX, VY, E)
    o2 = Oracle(3, VX, VY, E, eps=np.ones(E.shape[0]), mu=np.ones(E.shape[0]))
    rng = np.random.default_rng(2)
    q = tuple(rng.standard_normal(o1.geo.x.shape) for _ in range(3))
    for a, b in zip(o1.rhs(q), o2.rhs(q)):
        assert np.allclose(a, b, atol=1e-12)


def test_fake_partition_halo_rhs_matches_global():
    # SURVEY §4 Pin 2: per-rank RHS from own data + received halo traces equals the global RHS
    N = 3
    o = Oracle(N, *_mesh(N, 4, 0.2))
    rng = np.random.default_rng(9)
    q = tuple(rng.standard_normal(o.geo.x.shape) for _ in range(3))
    full = o.rhs(q)
    P = 3
    part = mesh.block_partition(o.K, P)
    flat = [u.ravel() for u in q]
    for rank in range(P):
        recv, need, send = mesh.halo_lists(part, rank, o.EToE, o.EToF, o.vmapP, o.Np)
        # what each source sends to me, in my order, must equal what I need
        for src in recv:
            _, _, send_src = mesh.halo_lists(part, src, o.EToE, o.EToF, o.vmapP, o.Np)
            assert send_src[rank] == need[src]
        # rebuild a rank-local field array whose non-owned entries are ONLY the halo values
        own = np.nonzero(part == rank)[0]
        local = [np.full_like(u, np.nan) for u in flat]
        for c in range(3):
            idx = (own[:, None] * o.Np + np.arange(o.Np)[None, :]).ravel()
            local[c][idx] = flat[c][idx]
            for src in need:
                ids = np.array(need[src])
                local[c][ids] = flat[c][ids]       # values arriving over the exchange
        sub = tuple(u.reshape(o.K, o.Np) for u in local)
        # the flux of own elements only touches own + halo values
        si = {k: (v[own] if isinstance(v, np.ndarray) and v.shape[0] == o.K else v) for k, v in o.si.items()}
        geo_sub = mesh.Geometry(*(getattr(o.geo, a)[own] for a in
                                  ("rx", "sx", "ry", "sy", "J", "nx", "ny", "sJ", "Fsc", "x", "y")))
        fl = operator.flux(si, *sub, alpha=o.alpha)
        vol = operator.volume(o.ref, geo_sub, *(u[own] for u in sub))
        for c in range(3):
            part_rhs = vol[c] + operator.lift(o.ref, fl[c])
            assert np.array_equal(part_rhs, full[c][own])
