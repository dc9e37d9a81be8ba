"""O9: low-storage explicit Runge-Kutta (TEST INFRASTRUCTURE).

The paper only says "simple, explicit Runge-Kutta methods" (PAPER.md:423-426,
659-663); reading A10 adopts the Carpenter-Kennedy 5-stage 4th-order
low-storage scheme of the cited textbook, coefficients
from SURVEY.md Appendix A:

    for i = 0..4:  res <- a_i res + dt R(q);   q <- q + b_i res      (res = 0 at start)
"""
from __future__ import annotations

from fractions import Fraction

A_FRAC = [Fraction(0),
          Fraction(-567301805773, 1357537059087),
          Fraction(-2404267990393, 2016746695238),
          Fraction(-3550918686646, 2091501179385),
          Fraction(-1275806237668, 842570457699)]
B_FRAC = [Fraction(1432997174477, 9575080441755),
          Fraction(5161836677717, 13612068292357),
          Fraction(1720146321549, 2090206949498),
          Fraction(3134564353537, 4481467310338),
          Fraction(2277821191437, 14882151754819)]
C_FRAC = [Fraction(0),
          Fraction(1432997174477, 9575080441755),
          Fraction(2526269341429, 6820363962896),
          Fraction(2006345519317, 3224310063776),
          Fraction(2802321613138, 2924317926251)]

A = [float(x) for x in A_FRAC]
B = [float(x) for x in B_FRAC]
C = [float(x) for x in C_FRAC]
STAGES = 5


def step(q, res, dt, R):
    """One LSERK4 step on a tuple of arrays.  R(q) -> tuple of d/dt arrays.
    Returns (q', res').  Arrays are not modified in place."""
    q = list(q)
    res = list(res)
    for i in range(STAGES):
        k = R(tuple(q))
        res = [A[i] * r + dt * kk for r, kk in zip(res, k)]
        q = [qq + B[i] * r for qq, r in zip(q, res)]
    return tuple(q), tuple(res)
