"""World-size-2 CPU tests of the multi-rank (N > 1) host path with torch.distributed/gloo.

Each rank builds a HOST-ONLY context (device = -1) for its partition of the
same global mesh, exactly as bench.py does under torchrun, and:
  * the halo lists agree across ranks (what rank r sends is what its neighbour
    expects, checked by exchanging the lists over gloo);
  * the halo protocol delivers the right data: each rank sends its own field
    values at its send list over gloo send/recv, and the received ghosts,
    plugged into the oracle's flux on the rank's own elements, reproduce the
    global oracle RHS bitwise (SURVEY.md §4 "Pin 2", §8(e));
  * the ncclUniqueId handshake of bench.py works (rank 0 makes it, the other
    receives the same 128 bytes by broadcast_object_list).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    import sys

    sys.path.insert(0, ROOT)
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import dginputs
        from oracle import mesh as omesh
        from oracle import operator as oop
        from oracle.solver import Oracle
        from paper_1304_5546_b200 import dg

        N = 3
        VX, VY, E = dginputs.rect_mesh(6)
        rng = np.random.default_rng(0)
        inner = (VX > 0) & (VX < 1) & (VY > 0) & (VY < 1)
        VX = VX + 0.03 * rng.uniform(-1, 1, VX.shape) * inner
        ctx = dg.dg_setup(N, VX, VY, E, device=-1, rank=rank, nranks=world)
        h = ctx.halo()
        gid = ctx.local_elements()
        # 1. list agreement
        lists = [None] * world
        dist.all_gather_object(lists, {"nbr": h["nbr"].tolist(),
                                       "send": [h["send_gdof"][h["send_off"][t]:h["send_off"][t + 1]].tolist()
                                                for t in range(len(h["nbr"]))],
                                       "recv": [h["recv_gdof"][h["recv_off"][t]:h["recv_off"][t + 1]].tolist()
                                                for t in range(len(h["nbr"]))]})
        for t, peer in enumerate(h["nbr"]):
            other = lists[peer]
            u = other["nbr"].index(rank)
            assert other["send"][u] == lists[rank]["recv"][t]
        # 2. data exchange over gloo reproduces the global RHS on own elements
        o = Oracle(N, VX, VY, E)
        q = tuple(dginputs.perturbation(o.geo.x.shape, 1.0, seed=3))   # the same global field on all ranks
        full = o.rhs(q)
        flat = [a.ravel() for a in q]
        local = [np.full_like(a, np.nan) for a in flat]
        own = (gid[:, None] * o.Np + np.arange(o.Np)[None, :]).ravel()
        for c in range(3):
            local[c][own] = flat[c][own]
        reqs = []
        recv_bufs = []
        for t, peer in enumerate(h["nbr"]):
            sg = h["send_gdof"][h["send_off"][t]:h["send_off"][t + 1]]
            sendbuf = torch.from_numpy(np.stack([local[c][sg] for c in range(3)]))  # only own values
            rg = h["recv_gdof"][h["recv_off"][t]:h["recv_off"][t + 1]]
            rbuf = torch.empty((3, len(rg)), dtype=torch.float64)
            reqs.append(dist.isend(sendbuf, int(peer)))
            reqs.append(dist.irecv(rbuf, int(peer)))
            recv_bufs.append((rg, rbuf))
        for r in reqs:
            r.wait()
        for rg, rbuf in recv_bufs:
            for c in range(3):
                local[c][rg] = rbuf[c].numpy()
        sub = tuple(a.reshape(o.K, o.Np) for a in local)
        si = {k: (v[gid] if isinstance(v, np.ndarray) and v.shape[0] == o.K else v) for k, v in o.si.items()}
        geo = omesh.Geometry(*(getattr(o.geo, a)[gid] for a in
                               ("rx", "sx", "ry", "sy", "J", "nx", "ny", "sJ", "Fsc", "x", "y")))
        fl = oop.flux(si, *sub, alpha=1.0)
        vol = oop.volume(o.ref, geo, *(a[gid] for a in sub))
        for c in range(3):
            assert np.array_equal(vol[c] + oop.lift(o.ref, fl[c]), full[c][gid])
        # 3. ncclUniqueId handshake (bench.py)
        try:
            ids = [dg.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(ids, src=0)
            got = ids[0]
            assert isinstance(got, bytes) and len(got) == 128
            both = [None] * world
            dist.all_gather_object(both, got)
            assert both[0] == both[1]
        except dg.DGError:
            pass  # no libnccl on this host: the GPU box has it
        ctx.destroy()
        dist.destroy_process_group()
        out_q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback

        out_q.put((rank, traceback.format_exc()))


def test_two_rank_gloo_halo_protocol():
    pytest.importorskip("paper_1304_5546_b200.dg", reason="libdg.so not built")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert results[r] == "ok", results[r]
