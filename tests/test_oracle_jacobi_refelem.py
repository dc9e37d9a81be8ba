"""Pins of oracle O1-O4 (Jacobi polynomials, nodes, Dr/Ds, M, LIFT) against what
the paper and mathematics fix -- never against the oracle itself.

Pins: SPEC.md:44-45, 56-58, 66-68, 78, 81-83, 498-499 (invariants / examples),
closed-form Gauss-Lobatto nodes, the library Legendre routines (special case
a = b = 0), exact monomial differentiation, the Dirichlet simplex integral,
and SURVEY.md Appendix A (independent transcription of the node set, A6).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from conftest import floats, read_golden
from oracle import jacobi, refelem


# ---------------------------------------------------------------- O1 Jacobi
@pytest.mark.parametrize("n", range(0, 9))
def test_jacobi_00_is_normalised_legendre(n):
    # special case reducing to a library routine: P_n^(0,0) = sqrt((2n+1)/2) L_n
    x = np.linspace(-1, 1, 37)
    leg = np.polynomial.legendre.Legendre.basis(n)
    assert np.allclose(jacobi.jacobi_p(x, 0, 0, n), math.sqrt((2 * n + 1) / 2) * leg(x), atol=1e-13)
    assert np.allclose(jacobi.grad_jacobi_p(x, 0, 0, n), math.sqrt((2 * n + 1) / 2) * leg.deriv()(x),
                       atol=1e-11)


@pytest.mark.parametrize("a,b", [(0, 0), (1, 0), (3, 0), (1, 1), (5, 0), (2, 3)])
def test_jacobi_orthonormal_under_weight(a, b):
    # int (1-x)^a (1+x)^b P_m P_n = delta_mn, using a high-order Gauss-Legendre
    # rule from numpy (weight polynomial integrated exactly)
    g, w = np.polynomial.legendre.leggauss(40)
    wt = w * (1 - g) ** a * (1 + g) ** b
    P = np.stack([jacobi.jacobi_p(g, a, b, n) for n in range(8)])
    G = (P * wt) @ P.T
    assert np.allclose(G, np.eye(8), atol=1e-12)


@pytest.mark.parametrize("n", range(0, 10))
def test_gauss_00_matches_numpy_leggauss(n):
    x, w = jacobi.jacobi_gq(0, 0, n)
    xr, wr = np.polynomial.legendre.leggauss(n + 1)
    assert np.allclose(np.sort(x), np.sort(xr), atol=1e-14)
    assert np.allclose(w[np.argsort(x)], wr[np.argsort(xr)], atol=1e-13)


def test_gauss_lobatto_closed_forms():
    assert np.allclose(jacobi.jacobi_gl(0, 0, 1), [-1, 1])
    assert np.allclose(jacobi.jacobi_gl(0, 0, 2), [-1, 0, 1], atol=1e-15)
    s5 = 1 / math.sqrt(5)
    assert np.allclose(jacobi.jacobi_gl(0, 0, 3), [-1, -s5, s5, 1], atol=1e-15)
    s37 = math.sqrt(3 / 7)
    assert np.allclose(jacobi.jacobi_gl(0, 0, 4), [-1, -s37, 0, s37, 1], atol=1e-15)
    # general N: interior GLL nodes are the roots of L_N'
    for n in range(5, 12):
        roots = np.sort(np.polynomial.legendre.Legendre.basis(n).deriv().roots())
        assert np.allclose(jacobi.jacobi_gl(0, 0, n)[1:-1], roots, atol=1e-13)


# ---------------------------------------------------------------- quadrature used by the oracle
@pytest.mark.parametrize("a,b", [(0, 0), (1, 0), (0, 3), (2, 2), (5, 4), (9, 1)])
def test_triangle_quadrature_dirichlet_integral(a, b):
    # int_I (1+r)^a (1+s)^b = 4 * 2^(a+b) a! b! / (a+b+2)!
    r, s, w = refelem.triangle_quadrature(8)
    exact = 4 * 2 ** (a + b) * math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)
    assert abs(np.sum(w * (1 + r) ** a * (1 + s) ** b) - exact) < 1e-12 * max(1, exact)


# ---------------------------------------------------------------- O2 nodes
def _tri_symmetries(r, s):
    # barycentric (l0, l1, l2) of vertices (-1,-1), (1,-1), (-1,1)
    l1 = (1 + r) / 2
    l2 = (1 + s) / 2
    l0 = 1 - l1 - l2
    out = []
    for perm in [(0, 1, 2), (1, 2, 0), (2, 0, 1), (0, 2, 1), (2, 1, 0), (1, 0, 2)]:
        L = [l0, l1, l2]
        m1, m2 = L[perm[1]], L[perm[2]]
        out.append((2 * m1 - 1, 2 * m2 - 1))
    return out


@pytest.mark.parametrize("n", range(1, 16))
def test_nodes_symmetric_and_edge_gll(n):
    r, s = refelem.nodes(n)
    Np = (n + 1) * (n + 2) // 2
    assert r.shape == (Np,)
    pts = np.stack([r, s], 1)
    for (r2, s2) in _tri_symmetries(r, s):
        q = np.stack([r2, s2], 1)
        d = np.abs(pts[:, None, :] - q[None, :, :]).max(axis=2).min(axis=1)
        assert d.max() < 1e-10
    gll = jacobi.jacobi_gl(0, 0, n)
    bottom = np.sort(r[np.abs(s + 1) < 1e-12])
    assert np.allclose(bottom, gll, atol=1e-13)
    # nodes lie in the closed triangle
    assert (r >= -1 - 1e-13).all() and (s >= -1 - 1e-13).all() and (r + s <= 1e-13).all()


def test_nodes_low_order_closed_form():
    r, s = refelem.nodes(1)
    assert np.allclose(np.stack([r, s], 1), [[-1, -1], [1, -1], [-1, 1]], atol=1e-15)
    r, s = refelem.nodes(2)
    assert np.allclose(np.stack([r, s], 1),
                       [[-1, -1], [0, -1], [1, -1], [-1, 0], [0, 0], [-1, 1]], atol=1e-15)


def test_appendixA_anchors():
    g = read_golden("appendixA_anchors.txt")
    ref4 = refelem.build(4)
    assert ref4.Fmask.ravel().tolist() == [int(v) for v in floats(g["N4_Fmask"])]
    assert np.allclose([ref4.r[6], ref4.s[6]], floats(g["N4_node6"]), atol=1e-14)
    assert abs(ref4.Dr[1, 0] - float(g["N4_Dr_1_0"])) < 1e-13
    assert abs(ref4.LIFT[0, 0] - float(g["N4_LIFT_0_0"])) < 1e-12
    assert abs(np.abs(ref4.Dr).sum() - float(g["N4_sum_abs_Dr"])) < 1e-11
    ref5 = refelem.build(5)
    assert np.allclose([ref5.r[7], ref5.s[7]], floats(g["N5_node7"]), atol=1e-14)
    assert abs(ref5.Dr[1, 0] - float(g["N5_Dr_1_0"])) < 1e-13
    assert abs(ref5.LIFT[0, 0] - float(g["N5_LIFT_0_0"])) < 1e-12
    assert abs(np.abs(ref5.Dr).sum() - float(g["N5_sum_abs_Dr"])) < 1e-10
    ref8 = refelem.build(8)
    assert np.allclose([ref8.r[10], ref8.s[10]], floats(g["N8_node10"]), atol=1e-14)
    assert abs(np.abs(ref8.Dr).sum() - float(g["N8_sum_abs_Dr"])) < 1e-9


# ---------------------------------------------------------------- O3 basis / D
@pytest.mark.parametrize("n", range(1, 6))
def test_basis_gram_identity(n):
    # orthonormality under quadrature; phi_00 = 1/sqrt(2)
    r, s, w = refelem.triangle_quadrature(n + 3)
    V = refelem.vandermonde_2d(n, r, s)
    assert np.allclose((V * w[:, None]).T @ V, np.eye(V.shape[1]), atol=1e-12)
    assert np.allclose(V[:, 0], 1 / math.sqrt(2), atol=1e-15)


@pytest.mark.parametrize("n", range(1, 10))
def test_D_exact_on_monomials(n):
    # Dr, Ds differentiate r^i s^j (i+j <= N) exactly
    ref = refelem.build(n)
    r, s = ref.r, ref.s
    err = 0.0
    for i in range(n + 1):
        for j in range(n + 1 - i):
            u = r ** i * s ** j
            ur = i * r ** max(i - 1, 0) * s ** j if i > 0 else 0 * r
            us = j * r ** i * s ** max(j - 1, 0) if j > 0 else 0 * r
            err = max(err, np.abs(ref.Dr @ u - ur).max(), np.abs(ref.Ds @ u - us).max())
    assert err < 1e-12 * max(1, n * n)
    assert np.abs(ref.Dr @ np.ones(ref.Np)).max() < 1e-12
    assert np.abs(ref.Ds @ np.ones(ref.Np)).max() < 1e-12
    # derivative of the endpoint GLL Lagrange polynomial: Dr[0,0] = -N(N+1)/4
    assert abs(ref.Dr[0, 0] + n * (n + 1) / 4) < 1e-11


def test_spec_example_N4_r2s():
    ref = refelem.build(4)
    assert np.abs(ref.Dr @ (ref.r ** 2 * ref.s) - 2 * ref.r * ref.s).max() < 1e-10
    ref3 = refelem.build(3)
    assert np.allclose(ref3.Dr @ ref3.r, 1.0, atol=1e-13)


# ---------------------------------------------------------------- O4 M, Fmask, LIFT
@pytest.mark.parametrize("n", range(1, 10))
def test_mass_and_lift(n):
    ref = refelem.build(n)
    one = np.ones(ref.Np)
    # 1^T M 1 = area of I = 2; M equals the textbook (V V^T)^-1
    assert abs(one @ ref.M @ one - 2.0) < 1e-12
    assert np.allclose(ref.M, np.linalg.inv(ref.V @ ref.V.T), atol=1e-12)
    assert np.allclose(ref.M, ref.M.T, atol=1e-15)
    for f in range(3):
        Mf = ref.Mface[f]
        assert np.allclose(Mf, Mf.T, atol=1e-15)
        assert np.linalg.eigvalsh(Mf).min() > 0  # SPD
        # face mass of the 1D GLL Lagrange basis: 1^T Mf 1 = 2 (parameter length)
        assert abs(np.ones(ref.Nfp) @ Mf @ np.ones(ref.Nfp) - 2.0) < 1e-12
        # lift consistency: 1^T M LIFT e_f = 2
        e = np.zeros(3 * ref.Nfp)
        e[f * ref.Nfp:(f + 1) * ref.Nfp] = 1.0
        assert abs(one @ ref.M @ ref.LIFT @ e - 2.0) < 1e-11
    # Fmask closed form: row j of the node triangle starts at sum_{t<j}(N+1-t)
    start = np.concatenate([[0], np.cumsum([n + 1 - t for t in range(n)])])
    assert ref.Fmask[0].tolist() == list(range(n + 1))
    assert ref.Fmask[1].tolist() == [int(start[j] + n - j) for j in range(n + 1)]
    assert ref.Fmask[2].tolist() == [int(start[j]) for j in range(n + 1)]


def test_lift_of_face_polynomial_matches_surface_integral():
    # int_I l_i (LIFT g) = sum_f int_{f} l_i g dt for any face data g: check with a polynomial
    ref = refelem.build(5)
    g = np.random.default_rng(0).standard_normal(3 * ref.Nfp)
    lhs = ref.M @ ref.LIFT @ g
    rhs = np.zeros(ref.Np)
    gq, wq = np.polynomial.legendre.leggauss(12)
    for f in range(3):
        fr, fs = refelem.face_points(f, gq)
        Lf = ref.lagrange_at(fr, fs)
        # g interpolated on the face by the face-node Lagrange values
        gf = Lf[:, ref.Fmask[f]] @ g[f * ref.Nfp:(f + 1) * ref.Nfp]
        rhs += (Lf * (wq * gf)[:, None]).sum(axis=0)
    assert np.allclose(lhs, rhs, atol=1e-12)


def test_degree_range():
    with pytest.raises(ValueError):
        refelem.build(0)
    with pytest.raises(ValueError):
        refelem.build(16)
