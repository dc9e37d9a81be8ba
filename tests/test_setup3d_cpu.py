"""CPU tests of the 3D host setup (C++, csrc/setup3d.cpp) against the independent 3D oracle
(oracle/refelem3d.py, mesh3d.py): operators <= 1e-12 relative, connectivity and face maps bit-exact,
geometry <= 1e-13.  Host-only contexts (device = -1) touch no GPU."""
import numpy as np
import pytest

import dginputs
from oracle.maxwell3d import Oracle3D

dg3 = pytest.importorskip("paper_1304_5546_b200.dg3", reason="libdg.so not built")


def _jittered_cube(n, amp=0.05, seed=3):
    VX, VY, VZ, E = dginputs.cube_tet_mesh(n)
    rng = np.random.default_rng(seed)
    inner = (VX > 0) & (VX < 1) & (VY > 0) & (VY < 1) & (VZ > 0) & (VZ < 1)
    return (VX + amp * rng.uniform(-1, 1, VX.shape) * inner, VY + amp * rng.uniform(-1, 1, VX.shape) * inner,
            VZ + amp * rng.uniform(-1, 1, VX.shape) * inner, E)


def test_library_exports_every_dg3_symbol():
    import re
    import os
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "dg3.h")).read()
    declared = set(re.findall(r"\b(dg3_\w+)\s*\(", hdr))
    assert declared == set(dg3.EXPORTS3)
    for name in declared:
        assert hasattr(dg3._lib, name)


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6])
def test_host_setup_matches_oracle(N):
    VX, VY, VZ, E = _jittered_cube(2)
    c = dg3.dg3_setup(N, VX, VY, VZ, E, device=-1)
    o = Oracle3D(N, VX, VY, VZ, E)
    assert (c.Np, c.Nfp, c.K, c.n_swapped) == (o.Np, o.ref.Nfp, o.K, o.n_swapped)
    op = c.operators()
    for k in ("r", "s", "t"):
        assert np.abs(op[k] - getattr(o.ref, k)).max() < 1e-14
    for k in ("Dr", "Ds", "Dt", "LIFT"):
        ref = getattr(o.ref, k)
        assert np.abs(op[k] - ref).max() <= 1e-13 * np.abs(ref).max()
    assert np.array_equal(op["Fmask"], o.ref.Fmask)
    mp = c.maps()
    assert np.array_equal(mp["EToE"], o.EToE) and np.array_equal(mp["EToF"], o.EToF)
    assert np.array_equal(mp["vmapP"], o.vmapP)
    g = c.geometry()
    want = np.stack([o.geo.rx, o.geo.ry, o.geo.rz, o.geo.sx, o.geo.sy, o.geo.sz, o.geo.tx, o.geo.ty, o.geo.tz], 1)
    assert np.abs(g["gfac"] - want).max() < 1e-12
    for k in ("J", "nx", "ny", "nz", "sJ", "Fsc"):
        assert np.abs(g[k] - getattr(o.geo, k)).max() < 1e-12
    x, y, z = c.nodes()
    assert max(np.abs(x - o.geo.x).max(), np.abs(y - o.geo.y).max(), np.abs(z - o.geo.z).max()) < 1e-14
    c.destroy()


def test_setup_errors():
    VX, VY, VZ, E = dginputs.cube_tet_mesh(1)
    with pytest.raises(dg3._dg.DGError) as e:
        dg3.dg3_setup(0, VX, VY, VZ, E, device=-1)
    assert e.value.name == "DG_E_DEGREE"
    bad = E.copy()
    bad[0, 3] = bad[0, 2]  # a degenerate (flat) tetrahedron
    with pytest.raises(dg3._dg.DGError) as e:
        dg3.dg3_setup(2, VX, VY, VZ, bad, device=-1)
    assert e.value.name in ("DG_E_MESH_DEGENERATE", "DG_E_MESH_NONMANIFOLD")
    three = np.concatenate([E, E[:1]])  # a face shared by three tetrahedra
    with pytest.raises(dg3._dg.DGError) as e:
        dg3.dg3_setup(2, VX, VY, VZ, three, device=-1)
    assert e.value.name == "DG_E_MESH_NONMANIFOLD"
    c = dg3.dg3_setup(2, VX, VY, VZ, E, device=-1)
    with pytest.raises(dg3._dg.DGError) as e:  # host-only: no compute
        c.run(1e-3, 1)
    assert e.value.name == "DG_E_STATE"
    c.destroy()
