"""Exercise the NCCL transport (transport = 0) with 2 ranks: torchrun --nproc-per-node 2.

    python -m torch.distributed.run --standalone --nproc-per-node 2 tools/nccl_same_gpu.py [fused]

Every rank uses cuda:0 when only one GPU is visible (NCCL may refuse duplicate GPUs; that is
reported, not hidden).  The id is broadcast over gloo.  Rank 0 compares the gathered
2-partition fields with a 1-partition run: they must be bitwise equal.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dginputs  # noqa: E402
from paper_1304_5546_b200 import dg  # noqa: E402


def main():
    fused = (sys.argv[1] != "split") if len(sys.argv) > 1 else True
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count()
    ids = [dg.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    N, n, steps, dt = 5, 40, 7, 1e-3
    VX, VY, E = dginputs.rect_mesh(n)
    eps, mu = dginputs.two_layer_material(VX, VY, E)
    try:
        c = dg.dg_setup(N, VX, VY, E, eps=eps, mu=mu, precision=8, device=dev, rank=rank, nranks=world,
                        fused=fused, transport=0, nccl_id=ids[0])
    except dg.DGError as e:
        print(f"rank {rank}: dg_setup failed: {e}", flush=True)
        dist.barrier()
        return 3
    gid = c.local_elements()
    x, y = c.nodes()
    q0 = dginputs.cavity_mode(x, y, 0.0)
    c.set_fields(*(a + b for a, b in zip(q0, dginputs.perturbation(x.shape, 1e-2, seed=rank))))
    # the perturbation must be a function of the global element: rebuild from the global arrays
    c1 = dg.dg_setup(N, VX, VY, E, eps=eps, mu=mu, precision=8, device=dev) if rank == 0 else None
    xg, yg = dg.dg_setup(N, VX, VY, E, device=-1).nodes()
    qg = tuple(a + b for a, b in zip(dginputs.cavity_mode(xg, yg, 0.0), dginputs.perturbation(xg.shape, 1e-2)))
    c.set_fields(*(a[gid] for a in qg))
    c.run(dt, steps)
    c.sync()
    got = c.get_fields()
    parts = [None] * world
    dist.all_gather_object(parts, (gid, got))
    st = c.kernel_stats()
    c.destroy()
    if rank == 0:
        c1.set_fields(*qg)
        c1.run(dt, steps)
        ref = c1.get_fields()
        c1.destroy()
        ok = True
        for g, f in parts:
            for a, b in zip(f, ref):
                ok &= np.array_equal(a, b[g])
        print(f"NCCL {world} ranks ({'fused' if fused else 'split'}): bitwise equal to 1 rank: {ok}; "
              f"halo pack launches {st['helper']['launches']}", flush=True)
        dist.barrier()
        return 0 if ok else 1
    dist.barrier()
    return 0


if __name__ == "__main__":
    sys.exit(main())
