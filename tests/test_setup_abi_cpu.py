"""CPU tests of the C ABI library (no GPU): it loads, exports every symbol
include/dg.h declares, and its HOST setup (C++ fp64: operators, geometry,
connectivity, face maps, partition/halo lists) agrees with the independent
oracle -- bit-exact for integer/index data, <= 1e-13 for operators.
Host-only contexts (device = -1) never touch CUDA; compute calls fail loudly.
"""
import os
import re

import numpy as np
import pytest

import dginputs
from oracle import mesh as omesh
from oracle.solver import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
dg = pytest.importorskip("paper_1304_5546_b200.dg", reason="libdg.so not built")


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "dg.h")).read()
    declared = set(re.findall(r"^\s*(?:dg_status|void|const char\*)\s+(dg_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(dg._lib, name), name
    assert declared == set(dg.EXPORTS)
    # the binding's constants mirror the header
    assert f"#define DG_ABI_VERSION {dg.ABI_VERSION}" in hdr
    assert f"#define DG_MAX_KERNEL_N {dg.MAX_KERNEL_N}" in hdr


@pytest.mark.parametrize("prec", [4, 8])
def test_kernel_config_matches_tune_table(prec):
    """dg_get_kernel_config reports the knob set csrc/tune.json picked for each (N, precision)
    (the library was built from that table), and shared memory fits one B200 SM."""
    import json
    tune = json.load(open(os.path.join(ROOT, "paper_1304_5546_b200", "csrc", "tune.json")))
    VX, VY, E = dginputs.rect_mesh(1)
    for N in range(1, dg.MAX_KERNEL_N + 1):
        c = dg.dg_setup(N, VX, VY, E, device=-1, precision=prec)
        k = c.kernel_config()
        c.destroy()
        t = tune[f"N{N}_{'f32' if prec == 4 else 'f64'}"]
        want = ("tcgen05_3xtf32" if t["M"] == 3 else "3xtf32" if prec == 4 else "dmma_fp64") if t["M"] else "fma"
        assert k["contraction"] == want, (N, k)
        assert k["slots"] == t["S"] and k["teams_cap"] == t["C"]
        # residual staged by TMA: the 3xTF32 path (fp32) and the DMMA unit teams (fp64, M=4), knob Q
        assert k["residual_tma"] == bool(t["M"] in ((1, 2) if prec == 4 else (4,)) and t.get("Q", 1))
        assert k["dmma_units"] == (prec == 8 and t["M"] == 4)
        assert k["warp_specialised"] == (prec == 8 and t["M"] == 4 and bool(t.get("K", 0)))
        if k["dmma_units"]:  # U DMMA warps (a multiple of 4), plus H flux warps when warp-specialised
            assert t["U"] % 4 == 0
            assert k["threads"] == 32 * (t["U"] + (t.get("H", 4) if t.get("K", 0) else 0))
        assert k["flux_first"] == bool(t.get("F", 0))
        assert k["ops_global"] == bool(t.get("G", 0))
        assert k["flux_in_fragments"] == bool(t["M"] == 1 and prec == 4 and t.get("X", 0))
        assert k["pass_interleave"] == bool(t["M"] and prec == 4 and t.get("I", 0))
        assert k["compressed_connectivity"] == (t.get("Z", 0) == 1)
        assert k["compressed_geometry"] == (t.get("Z", 0) in (1, 2))
        assert 0 < k["smem_bytes"] <= 227 * 1024 and k["threads"] % 32 == 0
        if prec == 4:  # the tcgen05 variant module of every fp32 N
            c = dg.dg_setup(N, VX, VY, E, device=-1, precision=4, kernel_variant=1)
            kt = c.kernel_config()
            c.destroy()
            assert kt["contraction"] == "tcgen05_3xtf32" and kt["threads"] == 256, (N, kt)
            assert 0 < kt["smem_bytes"] <= 227 * 1024


def _jittered(n, amp=0.25, seed=7, nx=None):
    VX, VY, E = dginputs.rect_mesh(n, nx)
    rng = np.random.default_rng(seed)
    inner = (VX > 0) & (VX < 1) & (VY > 0) & (VY < 1)
    VX = VX + amp / n * rng.uniform(-1, 1, VX.shape) * inner
    VY = VY + amp / n * rng.uniform(-1, 1, VY.shape) * inner
    return VX, VY, E


@pytest.mark.parametrize("N", list(range(1, 13)))
def test_operators_match_oracle(N):
    VX, VY, E = dginputs.rect_mesh(1)
    c = dg.dg_setup(N, VX, VY, E, device=-1)
    ops = c.operators()
    o = Oracle(N, VX, VY, E)
    ref = o.ref
    tol = 1e-13 * max(1.0, np.abs(ref.Dr).max())
    assert np.abs(ops["r"] - ref.r).max() < 1e-14 and np.abs(ops["s"] - ref.s).max() < 1e-14
    assert np.abs(ops["Dr"] - ref.Dr).max() < tol
    assert np.abs(ops["Ds"] - ref.Ds).max() < tol
    assert np.abs(ops["LIFT"] - ref.LIFT).max() < 1e-13 * max(1.0, np.abs(ref.LIFT).max())
    assert np.array_equal(ops["Fmask"], ref.Fmask)
    c.destroy()


@pytest.mark.parametrize("N,n,P", [(1, 3, 1), (4, 5, 1), (5, 4, 3), (8, 3, 2)])
def test_geometry_maps_nodes_match_oracle(N, n, P):
    VX, VY, E = _jittered(n)
    o = Oracle(N, VX, VY, E)
    part = omesh.block_partition(o.K, P)
    for rank in range(P):
        c = dg.dg_setup(N, VX, VY, E, device=-1, rank=rank, nranks=P)
        gid = c.local_elements()
        assert np.array_equal(gid, np.nonzero(part == rank)[0])
        g = c.geometry()
        for key in ("rx", "sx", "ry", "sy", "J"):
            ref = getattr(o.geo, key)[gid]
            assert np.abs(g[key] - ref).max() <= 1e-13 * np.abs(ref).max(), key
        for key in ("nx", "ny", "sJ", "Fsc"):
            ref = getattr(o.geo, key)[gid]
            assert np.abs(g[key] - ref).max() <= 1e-13 * np.abs(ref).max(), key
        m = c.maps()
        assert np.array_equal(m["EToE"], o.EToE[gid])
        assert np.array_equal(m["EToF"], o.EToF[gid])
        assert np.array_equal(m["vmapM"], o.vmapM[gid])
        assert np.array_equal(m["vmapP"], o.vmapP[gid])
        x, y = c.nodes()
        assert np.abs(x - o.geo.x[gid]).max() < 1e-14 and np.abs(y - o.geo.y[gid]).max() < 1e-14
        # halo lists == the oracle's fake partition (SURVEY §4 Pin 2), bit-exact
        recv, need, send = omesh.halo_lists(part, rank, o.EToE, o.EToF, o.vmapP, o.Np)
        h = c.halo()
        assert h["nbr"].tolist() == sorted(set(recv) | set(send))
        for t, peer in enumerate(h["nbr"]):
            sg = h["send_gdof"][h["send_off"][t]:h["send_off"][t + 1]]
            rg = h["recv_gdof"][h["recv_off"][t]:h["recv_off"][t + 1]]
            rp = h["recv_point"][h["recv_off"][t]:h["recv_off"][t + 1]]
            assert sg.tolist() == send.get(int(peer), [])
            assert rg.tolist() == need.get(int(peer), [])
            lid = {int(k): i for i, k in enumerate(gid)}
            want = [(lid[k] * 3 + f) * o.ref.Nfp + i for (k, f, i) in recv.get(int(peer), [])]
            assert rp.tolist() == want
        c.destroy()


def test_orientation_and_errors():
    VX = np.array([0.0, 1.0, 0.0, 1.0])
    VY = np.array([0.0, 0.0, 1.0, 1.0])
    c = dg.dg_setup(2, VX, VY, np.array([[0, 2, 1], [1, 3, 2]]), device=-1)
    assert c.n_swapped == 1
    c.destroy()
    with pytest.raises(dg.DGError) as e:
        dg.dg_setup(0, VX, VY, np.array([[0, 1, 2]]), device=-1)
    assert e.value.name == "DG_E_DEGREE"
    with pytest.raises(dg.DGError) as e:
        dg.dg_setup(16, VX, VY, np.array([[0, 1, 2]]), device=-1)
    assert e.value.name == "DG_E_DEGREE"
    with pytest.raises(dg.DGError) as e:   # three triangles on edge (0,1)
        dg.dg_setup(2, np.array([0, 1, 0.5, 0.5, 0.2]), np.array([0, 0, 1, -1, 0.7]),
                    np.array([[0, 1, 2], [1, 0, 3], [0, 1, 4]]), device=-1)
    assert e.value.name == "DG_E_MESH_NONMANIFOLD"
    with pytest.raises(dg.DGError) as e:
        dg.dg_setup(2, np.array([0, 1, 2.0]), np.array([0, 0, 0.0]), np.array([[0, 1, 2]]), device=-1)
    assert e.value.name == "DG_E_MESH_DEGENERATE"
    with pytest.raises(dg.DGError) as e:
        dg.dg_setup(2, VX, VY, np.array([[0, 1, 2]]), bctag=np.array([[2, 0, 0]]), device=-1)
    assert e.value.name == "DG_E_UNSUPPORTED_BC"
    _, _, E2 = dginputs.rect_mesh(1)
    with pytest.raises(dg.DGError) as e:   # PEC tag on the shared diagonal
        dg.dg_setup(2, VX, VY, E2, bctag=np.array([[0, 0, 1], [1, 0, 0]]), device=-1)
    assert e.value.name == "DG_E_UNSUPPORTED_BC"
    with pytest.raises(dg.DGError) as e:
        dg.dg_setup(2, VX, VY, E2, eps=np.ones(2), device=-1)
    assert e.value.name == "DG_E_ARG"


def test_host_only_context_refuses_compute():
    VX, VY, E = dginputs.rect_mesh(2)
    c = dg.dg_setup(3, VX, VY, E, device=-1)
    z = np.zeros((c.K_local, c.Np))
    for call in (lambda: c.set_fields(z, z, z), lambda: c.run(0.1, 1), lambda: c.sync(),
                 lambda: c.eval_rhs(0), lambda: c.get_fields()):
        with pytest.raises(dg.DGError) as e:
            call()
        assert e.value.name == "DG_E_STATE"
    c.destroy()


def test_large_mesh_setup_is_fast_and_consistent():
    # C3-sized host setup (K = 2*128^2) in C++: maps are an involution, halo lists symmetric
    import time
    VX, VY, E = dginputs.rect_mesh(128)
    t = time.time()
    cs = [dg.dg_setup(5, VX, VY, E, device=-1, rank=r, nranks=4) for r in range(4)]
    assert time.time() - t < 20
    halos = [c.halo() for c in cs]
    for r, h in enumerate(halos):
        for t_, peer in enumerate(h["nbr"]):
            hp = halos[peer]
            u = hp["nbr"].tolist().index(r)
            mine = h["recv_gdof"][h["recv_off"][t_]:h["recv_off"][t_ + 1]]
            theirs = hp["send_gdof"][hp["send_off"][u]:hp["send_off"][u + 1]]
            assert np.array_equal(mine, theirs)


def test_field_buffers_are_validated_before_the_call():
    """dg.py checks dtype / contiguity / size of field buffers (numpy and torch) before handing raw
    pointers to dg_set_fields / dg_get_fields (host-only context: the C call is never reached)."""
    import torch

    VX, VY, E = dginputs.rect_mesh(2)
    c = dg.dg_setup(3, VX, VY, E, device=-1)
    n = c.K_local * c.Np
    with pytest.raises(ValueError):
        c.set_fields(*(torch.zeros(n, dtype=torch.float32) for _ in range(3)))
    with pytest.raises(ValueError):
        c.set_fields(*(torch.zeros(2 * n, dtype=torch.float64)[::2] for _ in range(3)))
    with pytest.raises(ValueError):
        c.get_fields(tuple(np.empty(n, dtype=np.float32) for _ in range(3)))
    with pytest.raises(ValueError):
        c.get_fields(tuple(np.empty(n + 1) for _ in range(3)))
    with pytest.raises(dg.DGError) as e:  # well-formed buffers reach the library: host-only context
        c.set_fields(*(np.zeros(n) for _ in range(3)))
    assert e.value.name == "DG_E_STATE"
    c.destroy()


def test_abi2_options_are_validated():
    VX, VY, E = dginputs.rect_mesh(2)
    for kw in (dict(max_ctas=-1), dict(check_every=-2), dict(tile_order=2)):
        with pytest.raises(dg.DGError) as e:
            dg.dg_setup(3, VX, VY, E, device=-1, **kw)
        assert e.value.name == "DG_E_ARG"
    dg.dg_setup(3, VX, VY, E, device=-1, max_ctas=3, tile_order=1, check_every=5).destroy()
