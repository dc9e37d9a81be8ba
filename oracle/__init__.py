"""Plain, slow, fp64 CPU oracle for the nodal-DG 2D TM Maxwell hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  The
product (``paper_1304_5546_b200``: C++ setup + CUDA kernels behind the C ABI
in ``include/dg.h``) never imports, links or executes anything in here, and
this package imports nothing from the product.  The two share only the seeded
input generators in ``dginputs`` (which hold none of the method's arithmetic).

Each function cites the passage it follows: PAPER.md (the method) by line and
equation label, the textbook it defers to through
SURVEY.md §8(c) O1-O11 and Appendix A, and SPEC.md for conventions.  Readings
of garbled or silent passages are listed in DESIGN.md.

Modules
-------
jacobi    O1   orthonormal Jacobi polynomials, Gauss / Gauss-Lobatto nodes
refelem   O2-O4 warp-and-blend nodes, Koornwinder-Dubiner basis, Dr/Ds,
               mass / face-mass matrices by quadrature, Fmask, LIFT
mesh      O5-O7 connectivity, affine geometry, vmapM/vmapP by coordinates,
               element partition + halo lists (CPU fake partition)
operator  O8   the semi-discrete DG right-hand side (eq. 9 + 1/2 eq. 5, A12)
lserk4    O9   low-storage RK (Carpenter-Kennedy 5-stage, 4th order)
energy    O10  discrete Maxwell energy and the energy-rate identity
solver         convenience driver: setup + run(dt, nsteps)

Parity pinning status: every function is pinned by tests/test_oracle_*.py
except where a docstring says "parity unpinned" (none at present; the node
set's alpha table A6 is pinned only by an independent transcription, see
DESIGN.md).
"""
