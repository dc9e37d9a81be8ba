"""GPU parity of the persistent, software-pipelined stage kernels as the full-size runs drive them.

At full size every CTA of the persistent grid walks many tiles: slot reuse, mbarrier phase
flips, next-tile TMA / gather issue, neighbour-code rotation, L2 prefetch and (S = 3) the split
buffers all run.  On an oracle-sized mesh the grid would give each CTA one tile, so these tests
cap the grid (dg_options.max_ctas) to make every CTA walk 5-6 tiles -- through both parities of
every mbarrier -- and compare element by element with the fp64 oracle after 100 LSERK4 steps:
every compiled (N, precision) kernel, fused and split, constant and piecewise-constant material.

Bar (BASELINE.json north_star, per field): for each F in (Hx, Hy, Ez),
max|F_gpu - F_orc| / max|F_orc| <= 1e-12 (fp64) / 2e-5 (fp32).  The input is the (1,1) cavity
mode started so that it ends the run at phase pi/4 (dginputs.balanced_start: every field O(1) where
the error is measured) plus a seeded 1e-2 perturbation.
"""
import numpy as np
import pytest

import dginputs
from oracle.solver import Oracle

pytestmark = pytest.mark.gpu

dg = pytest.importorskip("paper_1304_5546_b200.dg", reason="libdg.so not built")

TOL = {8: 1e-12, 4: 2e-5}
N_CELLS = 16          # K = 512: 16 tiles of 32 elements
MAX_CTAS = 3          # -> 5-6 tiles per persistent CTA
STEPS = 100


def _jittered(n, amp=0.25, seed=7):
    return dginputs.jittered_mesh(n, amp, seed)


def per_field(got, want):
    """SURVEY A14 per field: [max|a - b| / max|b| for each field]."""
    return [float(np.abs(a - b).max() / np.abs(b).max()) for a, b in zip(got, want)]


_CACHE = {}


def _case(N, material):
    """(mesh, eps, mu, q0, dt, oracle fields after STEPS steps), computed once per (N, material)."""
    key = (N, material)
    if key not in _CACHE:
        VX, VY, E = _jittered(N_CELLS, seed=100 + N)
        eps = mu = None
        if material:
            rng = np.random.default_rng(N)
            eps = rng.uniform(1.0, 3.0, E.shape[0])
            mu = rng.uniform(0.5, 2.0, E.shape[0])
        o = Oracle(N, VX, VY, E, eps=eps, mu=mu)
        dt = dginputs.cfl_dt(VX, VY, E, N, eps=eps, mu=mu)
        q0 = dginputs.cavity_mode(o.geo.x, o.geo.y, dginputs.balanced_start(STEPS * dt))
        q0 = tuple(a + b for a, b in zip(q0, dginputs.perturbation(o.geo.x.shape, 1e-2, seed=N)))
        _CACHE[key] = (VX, VY, E, eps, mu, q0, dt, o.run(q0, dt, STEPS))
    return _CACHE[key]


def _run(N, prec, fused, material=False, **opts):
    """100 steps of the cached case through the library; opts are dg_options fields."""
    VX, VY, E, eps, mu, q0, dt, want = _case(N, material)
    c = dg.dg_setup(N, VX, VY, E, eps=eps, mu=mu, precision=prec, fused=fused, **opts)
    c.set_fields(*q0)
    c.run(dt, STEPS)
    c.sync()
    got = c.get_fields()
    cfg = c.kernel_config()
    c.destroy()
    return got, want, cfg


@pytest.mark.parametrize("fused", [True, False], ids=["fused", "split"])
@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("N", list(range(1, 10)))
def test_multi_tile_pipeline_100_steps(N, prec, fused):
    got, want, cfg = _run(N, prec, fused, max_ctas=MAX_CTAS)
    errs = per_field(got, want)
    print(f"N={N} prec={prec} {'fused' if fused else 'split'} {cfg['contraction']} S={cfg['slots']}: "
          f"per-field {['%.2e' % e for e in errs]}")
    assert max(errs) <= TOL[prec], errs


@pytest.mark.parametrize("fused", [True, False], ids=["fused", "split"])
@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("N", [2, 5, 8, 9])
def test_multi_tile_pipeline_material_100_steps(N, prec, fused):
    got, want, cfg = _run(N, prec, fused, material=True, max_ctas=MAX_CTAS)
    errs = per_field(got, want)
    print(f"material N={N} prec={prec} {'fused' if fused else 'split'}: per-field {['%.2e' % e for e in errs]}")
    assert max(errs) <= TOL[prec], errs


@pytest.mark.parametrize("prec", [4, 8])
@pytest.mark.parametrize("N", [3, 5, 8, 9])
def test_grid_and_tile_order_never_change_the_result(N, prec):
    """The tiles a CTA walks, and the order it walks them in, are scheduling only: every grid cap
    (1 CTA walking all 16 tiles ... every resident CTA) and both tile orders give bitwise the
    same fields (the kernels are deterministic: no atomics, fixed per-element arithmetic)."""
    VX, VY, E, eps, mu, q0, dt, _ = _case(N, False)
    ref = None
    for max_ctas, order in ((0, 0), (1, 0), (2, 1), (5, 0), (0, 1)):
        c = dg.dg_setup(N, VX, VY, E, precision=prec, max_ctas=max_ctas, tile_order=order)
        c.set_fields(*q0)
        c.run(dt, 7)
        got = c.get_fields()
        c.destroy()
        if ref is None:
            ref = got
        else:
            for a, b in zip(got, ref):
                assert np.array_equal(a, b), (max_ctas, order)


@pytest.mark.parametrize("N", [4, 5, 6, 7, 8])
def test_fp64_dmma_teams_partitions_bitwise(N):
    """The fp64 DMMA unit teams (N >= 4) and the warp-specialised kernel (DMMA warps + flux warps,
    N = 5-8): 3 in-process partitions -- the NCCL path's interior-then-boundary tile lists, halo by
    device copies -- give bitwise the fields of one partition (P17), as do grid caps and tile order."""
    VX, VY, E, eps, mu, q0, dt, _ = _case(N, False)
    c = dg.dg_setup(N, VX, VY, E, precision=8)
    cfg = c.kernel_config()
    c.set_fields(*q0)
    c.run(dt, 7)
    ref = c.get_fields()
    c.destroy()
    assert cfg["dmma_units"], cfg
    cs = [dg.dg_setup(N, VX, VY, E, precision=8, rank=r, nranks=3, transport=1, max_ctas=2, tile_order=1)
          for r in range(3)]
    for c in cs:
        c.set_fields(*(a[c.local_elements()] for a in q0))
    dg.dg_run_group(cs, dt, 7)
    for c in cs:
        gid = c.local_elements()
        for a, b in zip(c.get_fields(), ref):
            assert np.array_equal(a, b[gid])
        c.destroy()


def test_check_every_reports_first_bad_step():
    VX, VY, E = dginputs.rect_mesh(4)
    for every, want in ((1, 1), (3, 3)):
        c = dg.dg_setup(3, VX, VY, E, precision=8, check_every=every)
        z = np.zeros((c.K_local, c.Np))
        bad = z.copy()
        bad[3, 2] = np.nan
        c.set_fields(z, z, bad)
        c.run(1e-3, 7)
        with pytest.raises(dg.DGError) as e:
            c.sync()
        assert e.value.name == "DG_E_DIVERGED"
        assert f"first found at step {want} " in str(e.value), str(e.value)
        c.set_fields(z, z, z)  # a fresh state clears the record
        c.run(1e-3, 4)
        c.sync()
        c.destroy()


def test_fields_through_device_pointers():
    """dg_set_fields / dg_get_fields take this device's memory as well as host memory."""
    torch = pytest.importorskip("torch")
    VX, VY, E = dginputs.rect_mesh(6)
    c = dg.dg_setup(4, VX, VY, E, precision=8)
    x, y = c.nodes()
    q0 = dginputs.cavity_mode(x, y, dginputs.C4_T0)
    c.set_fields(*[torch.from_numpy(a.copy()).cuda() for a in q0])
    back = c.get_fields()
    for a, b in zip(back, q0):
        assert np.array_equal(a, b)
    c.run(1e-3, 3)
    host = c.get_fields()
    dev = tuple(torch.empty(c.K_local, c.Np, dtype=torch.float64, device="cuda") for _ in range(3))
    c.get_fields(dev)
    for a, b in zip(dev, host):
        assert np.array_equal(a.cpu().numpy(), b)
    with pytest.raises(ValueError):
        c.set_fields(*[torch.from_numpy(a.copy()).float().cuda() for a in q0])
    c.destroy()


GATE = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "pipeline_gate_n12.npz")


@pytest.mark.parametrize("prec", [8, 4])
def test_tuner_oracle_gate_on_the_shipped_build(prec):
    """tools/tune.py's oracle gate, run on the shipped kernels: the stored fp64 oracle fields
    (tests/golden/pipeline_gate_n12.npz, tools/make_pipeline_gate_golden.py) after 100 steps on the
    jittered 12x12 mesh, grid capped at 2 CTAs; per-field A14 for every N."""
    G = np.load(GATE)
    for N in range(1, 10):
        c = dg.dg_setup(N, G["VX"], G["VY"], G["EToV"], precision=prec, max_ctas=2)
        x, y = c.nodes()
        q0 = dginputs.cavity_mode(x, y, float(G[f"t0_{N}"]))
        q0 = tuple(a + b for a, b in zip(q0, dginputs.perturbation(x.shape, float(G["amplitude"]), seed=N)))
        c.set_fields(*q0)
        c.run(float(G[f"dt{N}"]), int(G["steps"]))
        got = c.get_fields()
        c.destroy()
        errs = per_field(got, [G[f"{nm}{N}"] for nm in ("Hx", "Hy", "Ez")])
        assert max(errs) <= TOL[prec], (N, errs)


# ---------------------------------------------------------------- the tcgen05 kernel variant (fp32)
@pytest.mark.parametrize("fused", [True, False], ids=["fused", "split"])
@pytest.mark.parametrize("N", list(range(1, 10)))
def test_tcgen05_variant_multi_tile_100_steps(N, fused):
    """dg_options.kernel_variant = 1: the fp32 contractions on the 5th-generation tensor cores
    (tcgen05.mma kind::tf32, A operands and accumulators in TMEM, 128-element groups), the grid capped
    so every CTA walks several groups (K = 512: 4 groups, max_ctas = 2)."""
    got, want, cfg = _run(N, 4, fused, max_ctas=2, kernel_variant=1)
    assert cfg["contraction"] == "tcgen05_3xtf32"
    errs = per_field(got, want)
    print(f"tcgen05 N={N} {'fused' if fused else 'split'}: per-field {['%.2e' % e for e in errs]}")
    assert max(errs) <= TOL[4], errs


@pytest.mark.parametrize("N", [2, 5, 8])
def test_tcgen05_variant_material_100_steps(N):
    got, want, _ = _run(N, 4, True, material=True, max_ctas=2, kernel_variant=1)
    errs = per_field(got, want)
    assert max(errs) <= TOL[4], errs


@pytest.mark.parametrize("N", [1, 5, 9])
def test_tcgen05_variant_eval_rhs(N):
    """Single operator evaluations (full, volume only, surface only) of the tcgen05 kernels."""
    VX, VY, E = _jittered(7, seed=N)
    o = Oracle(N, VX, VY, E)
    q = dginputs.perturbation(o.geo.x.shape, 1.0, seed=N)
    c = dg.dg_setup(N, VX, VY, E, precision=4, kernel_variant=1)
    c.set_fields(*q)
    for which in ("full", "volume", "surface"):
        got, want = c.eval_rhs(which), o.rhs(q, which=which)
        err = max(float(np.abs(a - b).max() / np.abs(b).max()) for a, b in zip(got, want))
        assert err < 1e-5 * N, (which, err)
    c.destroy()


@pytest.mark.parametrize("N", [3, 5])
def test_tcgen05_variant_grid_order_and_partitions_bitwise(N):
    """Scheduling never changes the tcgen05 result: grid caps, tile order, and 3 in-process partitions
    (interior then boundary GROUP lists, halo by device copies) are bitwise equal to one run."""
    VX, VY, E, eps, mu, q0, dt, _ = _case(N, False)
    ref = None
    for max_ctas, order in ((0, 0), (1, 0), (3, 1)):
        c = dg.dg_setup(N, VX, VY, E, precision=4, max_ctas=max_ctas, tile_order=order, kernel_variant=1)
        c.set_fields(*q0)
        c.run(dt, 7)
        got = c.get_fields()
        c.destroy()
        if ref is None:
            ref = got
        else:
            for a, b in zip(got, ref):
                assert np.array_equal(a, b), (max_ctas, order)
    cs = [dg.dg_setup(N, VX, VY, E, precision=4, rank=r, nranks=3, transport=1, kernel_variant=1) for r in range(3)]
    for c in cs:
        c.set_fields(*(a[c.local_elements()] for a in q0))
    dg.dg_run_group(cs, dt, 7)
    for c in cs:
        gid = c.local_elements()
        for a, b in zip(c.get_fields(), ref):
            assert np.array_equal(a, b[gid])
        c.destroy()
