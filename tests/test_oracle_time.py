"""Pins of oracle O9 (LSERK4) and the whole discrete solver (P13-P16).

Pins: the exact rational coefficients, the stability
polynomial's Taylor coefficients 1, 1, 1/2, 1/6, 1/24 (fourth order, a closed
form), stage times = c, y' = -y; the exact PEC cavity mode
 with the observed h-order ~ N+1 (BASELINE.json north_star;
SPEC.md:501); energy monotonicity / conservation; the
exact two-layer cavity; the C1 anchor of SURVEY Appendix B.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import dginputs
from conftest import read_golden
from oracle import energy, lserk4
from oracle.solver import Oracle


def test_coefficients_match_golden():
    g = read_golden("lserk4_coefficients.txt")
    for key, fr in (("a", lserk4.A_FRAC), ("b", lserk4.B_FRAC), ("c", lserk4.C_FRAC)):
        assert [Fraction(t) for t in g[key].split()] == fr


def _poly_mul(p, q):
    out = [Fraction(0)] * (len(p) + len(q) - 1)
    for i, a in enumerate(p):
        for j, b in enumerate(q):
            out[i + j] += a * b
    return out


def _poly_add(p, q):
    n = max(len(p), len(q))
    return [(p[i] if i < len(p) else 0) + (q[i] if i < len(q) else 0) for i in range(n)]


def test_stability_polynomial_fourth_order():
    # y' = lambda y, z = lambda dt: run the scheme in exact rational polynomial arithmetic
    y = [Fraction(1)]
    res = [Fraction(0)]
    z = [Fraction(0), Fraction(1)]
    for a, b in zip(lserk4.A_FRAC, lserk4.B_FRAC):
        res = _poly_add([a * c for c in res], _poly_mul(z, y))
        y = _poly_add(y, [b * c for c in res])
    for k, want in enumerate([1, 1, Fraction(1, 2), Fraction(1, 6), Fraction(1, 24)]):
        assert abs(float(y[k] - want)) < 1e-14, (k, float(y[k]))
    assert abs(float(y[5]) - 1 / 200) < 1e-4  # 0.005


def test_stage_times_equal_c():
    # y' = 1: after stage i the state equals c_{i+1} dt (and dt after the last)
    y, res = Fraction(0), Fraction(0)
    for i, (a, b) in enumerate(zip(lserk4.A_FRAC, lserk4.B_FRAC)):
        res = a * res + 1
        y = y + b * res
        want = lserk4.C_FRAC[i + 1] if i < 4 else Fraction(1)
        assert abs(float(y - want)) < 1e-12


def test_scalar_decay():
    y, res = (np.array([1.0]),), (np.array([0.0]),)
    y, res = lserk4.step(y, res, 0.1, lambda q: (-q[0],))
    assert abs(y[0][0] - math.exp(-0.1)) < 1e-7


def test_c1_anchor():
    # SURVEY P14 anchor (independent transcription): C1 after 100 steps
    g = read_golden("survey_c1_anchor.txt")
    VX, VY, E = dginputs.rect_mesh(16)
    o = Oracle(4, VX, VY, E)
    q0 = dginputs.cavity_mode(o.geo.x, o.geo.y, 0.0)
    assert abs(o.energy(q0) - float(g["E0"])) < 1e-15
    dt = dginputs.cfl_dt(VX, VY, o.EToV, 4)
    assert abs(dt - float(g["dt"])) < 1e-15
    q = o.run(q0, dt, 100)
    ex = dginputs.cavity_mode(o.geo.x, o.geo.y, 100 * dt)
    err = np.abs(q[2] - ex[2]).max()
    assert abs(err / float(g["max_abs_Ez_error_after_100_steps"]) - 1) < 5e-3
    # exact energy of the cavity mode is 1/8; discrete energy non-increasing
    assert o.energy(q) <= o.energy(q0)


def _l2_err(o, q, ex):
    return math.sqrt(sum(energy.inner(o.ref, o.geo, a - b, a - b) for a, b in zip(q, ex)))


@pytest.mark.parametrize("N", [1, 2, 3])
def test_h_convergence_cavity(N):
    # cavity (1,1), meshes 4/8/16, t = 0.5 at cfl 0.5; order >= N + 0.5
    errs = []
    for n in (4, 8, 16):
        VX, VY, E = dginputs.rect_mesh(n)
        o = Oracle(N, VX, VY, E)
        dt0 = dginputs.cfl_dt(VX, VY, o.EToV, N, cfl=0.5)
        T = 0.5
        nsteps = int(math.ceil(T / dt0))
        dt = T / nsteps
        q = o.run(dginputs.cavity_mode(o.geo.x, o.geo.y, 0.0), dt, nsteps)
        errs.append(_l2_err(o, q, dginputs.cavity_mode(o.geo.x, o.geo.y, T)))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert min(rates) >= N + 0.5, (errs, rates)


def test_n_convergence_cavity():
    """N-refinement (p-convergence, north_star; PAPER.md:66-68 high order): at fixed h (2x2 cells,
    K = 8) the error of the exact PEC cavity mode (1,1) after T = 0.2 (dt = CFL/4 so
    the LSERK4 error stays below the spatial one) falls geometrically with N = 1..9, faster than
    any fixed algebraic rate: every step in N divides the mass-matrix L2 error by > 3 and the ratio
    grows (measured 4.3 -> 12.4); N = 9 reaches < 1e-8."""
    VX, VY, E = dginputs.rect_mesh(2)
    T = 0.2
    errs = []
    for N in range(1, 10):
        o = Oracle(N, VX, VY, E)
        steps = int(math.ceil(T / (0.25 * dginputs.cfl_dt(VX, VY, E, N))))
        qT = o.run(dginputs.cavity_mode(o.geo.x, o.geo.y, 0.0), T / steps, steps)
        d = [a - b for a, b in zip(qT, dginputs.cavity_mode(o.geo.x, o.geo.y, T))]
        errs.append(math.sqrt(2.0 * o.energy(d)))
    ratios = [a / b for a, b in zip(errs, errs[1:])]
    assert min(ratios) > 3.0, (errs, ratios)
    assert ratios[-1] > 2 * ratios[0], ratios  # geometric-or-better: the per-N gain does not fade
    assert errs[-1] < 1e-8, errs


def test_energy_behaviour():
    # alpha = 1: non-increasing per step; alpha = 0: conserved up to
    # the RK error, which must shrink at >= 4th order in dt
    VX, VY, E = dginputs.rect_mesh(4)
    o = Oracle(3, VX, VY, E, alpha=1.0)
    q0 = dginputs.cavity_mode(o.geo.x, o.geo.y, 0.0)
    pert = dginputs.perturbation(o.geo.x.shape, 1e-2)  # rough data
    qp = tuple(a + b for a, b in zip(q0, pert))
    dt = dginputs.cfl_dt(VX, VY, o.EToV, 3)
    Es = [o.energy(qp)]
    o.run(qp, dt, 300, callback=lambda n, q: Es.append(o.energy(q)))
    Es = np.array(Es)
    assert (np.diff(Es) <= 1e-12 * Es[0]).all() and Es[-1] < Es[0]
    o0 = Oracle(3, VX, VY, E, alpha=0.0)
    drift = []
    for cfl in (0.5, 0.25):
        dt = dginputs.cfl_dt(VX, VY, o0.EToV, 3, cfl=cfl)
        Es = [o0.energy(q0)]
        o0.run(q0, dt, int(round(300 * 0.5 / cfl)), callback=lambda n, q: Es.append(o0.energy(q)))
        drift.append(np.abs(np.array(Es) - Es[0]).max() / Es[0])
    assert drift[0] < 1e-6 and drift[0] / drift[1] > 16


@pytest.mark.slow
def test_two_layer_cavity_convergence():
    # eps 1 | 2.25 at x = 1/2, mu = 1; exact omega and h-rate ~ N+1
    g = read_golden("survey_c1_anchor.txt")
    w = dginputs.two_layer_omega()
    assert abs(w - float(g["two_layer_omega"])) < 1e-11
    N = 3
    errs = []
    for n in (4, 8):
        VX, VY, E = dginputs.rect_mesh(n)
        eps, mu = dginputs.two_layer_material(VX, VY, E)
        o = Oracle(N, VX, VY, E, eps=eps, mu=mu)
        side = np.repeat((eps > 1.0).astype(int)[:, None], o.Np, axis=1)
        q0 = dginputs.two_layer_mode(o.geo.x, o.geo.y, 0.0, side, omega=w)
        T = 0.3
        dt0 = dginputs.cfl_dt(VX, VY, o.EToV, N, eps=eps, mu=mu)
        nsteps = int(math.ceil(T / dt0))
        q = o.run(q0, T / nsteps, nsteps)
        ex = dginputs.two_layer_mode(o.geo.x, o.geo.y, T, side, omega=w)
        errs.append(_l2_err(o, q, ex))
    assert errs[1] < 1e-4
    assert math.log2(errs[0] / errs[1]) >= N + 0.5
