"""CUDA-graph replay of dg_run (dg_set_graphs): the same kernels with the same arguments, so
the fields must be bitwise equal to eager launches -- across both ping-pong parities, a dt
change (recapture), the split variant and a re-enable after dg_set_graphs(0)."""
import numpy as np
import pytest

import dginputs

pytestmark = pytest.mark.gpu

dg = pytest.importorskip("paper_1304_5546_b200.dg", reason="libdg.so not built")


def _run(N, prec, fused, graphs, schedule):
    VX, VY, E = dginputs.rect_mesh(12)
    c = dg.dg_setup(N, VX, VY, E, precision=prec, fused=fused)
    c.set_graphs(graphs)
    x, y = c.nodes()
    q0 = dginputs.cavity_mode(x, y, 0.0)
    c.set_fields(*(a + b for a, b in zip(q0, dginputs.perturbation(x.shape, 1e-2))))
    for dt, n in schedule:
        c.run(dt, n)
    c.sync()
    out = c.get_fields()
    st = c.kernel_stats()
    c.destroy()
    return out, st


@pytest.mark.parametrize("N,prec,fused", [(5, 4, True), (5, 8, True), (4, 8, False), (8, 8, True)])
def test_graph_replay_bitwise_equals_eager(N, prec, fused):
    dt = 1e-3
    sched = [(dt, 1), (dt, 3), (dt, 4), (0.5 * dt, 3), (dt, 2)]  # odd counts: both parities; dt change
    eager, st_e = _run(N, prec, fused, False, sched)
    graph, st_g = _run(N, prec, fused, True, sched)
    for a, b in zip(eager, graph):
        assert np.array_equal(a, b)
    # every replayed step is counted as its 5 (fused) or 10 (split) launches
    assert st_e["fused"]["launches"] == st_g["fused"]["launches"]
    assert st_e["volume"]["launches"] == st_g["volume"]["launches"]
    assert st_e["surface"]["launches"] == st_g["surface"]["launches"]


def test_graphs_toggle_midrun():
    VX, VY, E = dginputs.rect_mesh(8)
    x = None
    res = []
    for toggles in ((True, True, True), (True, False, True), (False, False, False)):
        c = dg.dg_setup(5, VX, VY, E, precision=8)
        x, y = c.nodes()
        c.set_fields(*dginputs.cavity_mode(x, y, 0.0))
        for g in toggles:
            c.set_graphs(g)
            c.run(2e-3, 5)
        res.append(c.get_fields())
        c.destroy()
    for other in res[1:]:
        for a, b in zip(res[0], other):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("fused", [True, False])
def test_profiled_graph_replay(fused):
    """dg_profile with graphs on: the replayed graph carries event-record nodes around every
    launch; same fields bitwise as the unprofiled replay, every launch timed, times > 0."""
    VX, VY, E = dginputs.rect_mesh(12)
    outs = []
    for prof in (False, True):
        c = dg.dg_setup(5, VX, VY, E, precision=4, fused=fused)
        x, y = c.nodes()
        c.set_fields(*dginputs.cavity_mode(x, y, 0.0))
        c.run(1e-3, 2)
        c.profile(prof)
        c.run(1e-3, 5)  # both parities
        st = c.kernel_stats()
        outs.append(c.get_fields())
        c.destroy()
        if prof:
            kinds = ("fused",) if fused else ("volume", "surface")
            for k in kinds:
                assert st[k]["launches"] == 25 and st[k]["timed"] == 25, st
                assert st[k]["ms"] > 0
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
