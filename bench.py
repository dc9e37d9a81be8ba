"""Benchmark: DG DOF-updates/s of the LSERK4 TM-Maxwell step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--order N] [--n CELLS] [--prec 4|8] [--split]

Default workload = config C4 (BASELINE.json configs[3], the north-star target):
unit-square PEC cavity, A16 mesh of 724 x 724 cells (K = 1,048,352 triangles),
N = 5, fp32, cavity mode (1,1) initial data, dt from the CFL estimate.  One
"step" = one LSERK4 step = 5 stage launches of the fused volume+flux+LIFT+RK
kernel over every element.  metric value = Np * K * 3 fields * 5 stages * steps
/ (max over ranks of the CUDA-event time of the K timed steps); inputs are
resident in HBM when the timed region starts; the working set (~0.8 GB at
C4) is larger than the 126 MB L2, so no explicit flush is needed.

Under torchrun (N > 1) every rank owns a contiguous block of elements
(SURVEY.md §8(e)); face traces cross ranks by NCCL send/recv inside the stage
loop (strong scaling: K fixed).

--impl reference times the fp64 NumPy oracle (oracle/, the only "reference"
this paper-only task has) on host cores, on a bounded sample of the same
workload per step; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import dginputs  # noqa: E402

METRIC = "DG DOF-updates/s (fp32/fp64) and % of kernel roofline at 1/2/4/8 B200"
L2_BYTES = 126 * 1024 * 1024
FLUSH_BYTES = 512 * 1024 * 1024
UNIT = "DOF-updates/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def compute_peak(prec, contraction):
    """Measured arithmetic peak (TFLOP/s) of the pipe the contraction runs on, and its label:
    FFMA / DFMA from profiles/r01_peaks_fma_hbm.json (tools/peaks.cu), mma.sync TF32 / DMMA
    from profiles/r01_peaks_mma.json (tools/mma_peaks.cu).  3xTF32 issues 3 tensor products
    per fp32 product, so its fp32-equivalent peak is the TF32 rate / 3."""
    def load(name):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as fh:
                return json.load(fh)
        except Exception:
            return {}
    fma, mma = load("r01_peaks_fma_hbm.json"), load("r01_peaks_mma.json")
    if contraction == "dmma_fp64":
        return "tensor", float(mma.get("dmma_tflops", 36.0)), "measured DMMA m8n8k4 (tools/mma_peaks.cu)"
    if contraction == "3xtf32":
        return ("tensor", float(mma.get("tf32_tflops", 275.0)) / 3,
                "measured TF32 mma.sync m16n8k8 / 3 (tools/mma_peaks.cu)")
    if contraction == "tcgen05_3xtf32":
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
                bf16 = float(json.load(fh)["bf16_tflops"])
            src = "MEASURED_PEAKS.json bf16 x 1/2 (tf32 rate) / 3 (3xTF32)"
        except Exception:
            bf16, src = 2250.0, "nominal bf16 2.25 PF x 1/2 / 3"
        return "tensor", bf16 / 2 / 3, src
    if prec == 8:
        return "alu", float(fma.get("dfma_reg_tflops", 35.45)), "measured DFMA (tools/peaks.cu)"
    return "alu", float(fma.get("ffma_reg_tflops", 70.23)), "measured FFMA (tools/peaks.cu)"


def algorithmic_bytes_per_element_stage(Np, s, kind="fused"):
    """Bytes the method must move per element per LSERK4 stage, averaged over the 5 stages
    (DESIGN.md §Roofline).  fused: q_in read + q_out write (6 Np) + residual read on stages 1-4
    and write on stages 0-3 (2 * 0.8 * 3 Np) in the arithmetic type (s bytes), + 13 geometry words
    (rx, sx, ry, sy; nx, ny, Fsc per face) in the arithmetic type + 4 words of connectivity
    (3 neighbour ids + packed face ids).  Neighbour traces are L2 hits (not DRAM).
    Split variant: volume = q read + rhsV write (6 Np) + rx, sx, ry, sy; surface = q read,
    rhsV read, q_out write (9 Np) + the residual (4.8 Np) + 9 face words + connectivity."""
    if kind == "volume":
        return 6.0 * Np * s + 4 * s
    if kind == "surface":
        return (9.0 + 4.8) * Np * s + 9 * s + 16
    return (6.0 + 4.8) * Np * s + 13 * s + 16


def flops_per_element_stage(N, kind="fused"):
    Np, Nfp = (N + 1) * (N + 2) // 2, N + 1
    vol = 8 * Np * Np + 8 * Np            # 4 mat-vecs (FMA = 2) + chain rule / curl
    lift = 2 * 3 * Np * 3 * Nfp           # LIFT on 3 fields
    flux = 3 * Nfp * 3 * 12               # jumps + upwind flux per face point
    rk = 3 * Np * 4                       # res = a res + dt rhs; q += b res
    if kind == "volume":
        return vol
    if kind == "surface":
        return lift + flux + rk + 3 * Np  # + rhsV added
    return vol + lift + flux + rk


def physical_gpu(local_rank):
    """The nvidia-smi / NVML id of this rank's GPU: CUDA_VISIBLE_DEVICES maps the visible ordinal
    local_rank to a physical index or a GPU UUID (nvidia-smi -i accepts both)."""
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        if local_rank < len(ids):
            return ids[local_rank]
    return str(local_rank)


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons of one GPU, sampled every 10 ms by NVML in a
    thread (nvidia-smi every ~100 ms as a fallback); summary() keeps the samples taken inside the
    timed window [t0, t1] (time.perf_counter)."""

    NAMES = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
             ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id):
        self.gpu_id = gpu_id
        self.samples = []  # (t, sm_mhz, max_mhz, [reasons])
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self.source = None

    def _nvml(self):
        import pynvml

        pynvml.nvmlInit()
        gid = self.gpu_id
        if gid.startswith("GPU-") or gid.startswith("MIG-"):
            h = pynvml.nvmlDeviceGetHandleByUUID(gid)
        else:
            h = pynvml.nvmlDeviceGetHandleByIndex(int(gid))
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        self.source = "nvml"
        while not self._stop.is_set():
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((time.perf_counter(), float(sm), float(mx),
                                 [n for n, b in self.NAMES if bits & b]))
            self._stop.wait(0.01)

    def _smi(self):
        self.source = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                v = [x.strip() for x in out.split(",")]
                if len(v) >= 6:
                    names = [n for n, _ in self.NAMES[:4]]
                    self.samples.append((time.perf_counter(), float(v[0]), float(v[1]),
                                         [n for n, x in zip(names, v[2:6]) if x == "Active"]))
            except Exception:
                pass
            self._stop.wait(0.05)

    def _run(self):
        try:
            self._nvml()
        except Exception:
            if not self._stop.is_set():
                self._smi()

    def __enter__(self):
        self._t.start()
        t_end = time.perf_counter() + 5.0  # NVML init can take a while: sample before the timed region starts
        while not self.samples and self._t.is_alive() and time.perf_counter() < t_end:
            time.sleep(0.005)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self, t0=None, t1=None):
        inside = [x for x in self.samples if (t0 is None or x[0] >= t0) and (t1 is None or x[0] <= t1)]
        use = inside or self.samples
        if not use:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "gpu": self.gpu_id}
        return {"sm_mhz": statistics.median(x[1] for x in use), "sm_max_mhz": max(x[2] for x in use),
                "reasons": sorted({r for x in use for r in x[3]}), "samples": len(use),
                "samples_in_timed_region": len(inside), "source": self.source, "gpu": self.gpu_id}


CONFIGS = {  # BASELINE.json configs shaped for one bench line (rank-level workloads)
    "c4": dict(order=5, n=724, prec=4, material=False),   # configs[3]: the north-star target
    "c5": dict(order=8, n=1448, prec=8, material=True),   # configs[4]: N=8, K=4.19M, fp64, eps 1 | 2.25
    "c5w": dict(order=8, n=512, prec=8, material=True),   # configs[4] weak scaling: ~524k elements per GPU
}


def initial_fields(x, y, eps=None):
    """Cavity mode (1,1); with the two-layer material, its exact mode."""
    if eps is None:
        return dginputs.cavity_mode(x, y, 0.0)
    side = np.repeat((np.asarray(eps) > 1.0).astype(int)[:, None], x.shape[1], axis=1)
    return dginputs.two_layer_mode(x, y, 0.0, side)


def workload(args):
    N, n, prec = args.order, args.n, args.prec
    VX, VY, E = dginputs.rect_mesh(n)
    K = E.shape[0]
    Np = (N + 1) * (N + 2) // 2
    eps = mu = None
    if args.material:
        eps, mu = dginputs.two_layer_material(VX, VY, E)
    dt = dginputs.cfl_dt(VX, VY, E, N, eps=eps, mu=mu)
    tag = {"c4": "C4", "c5": "C5 (strong, 1 rank)", "c5w": "C5 (weak, per-GPU size)"}.get(args.config, "custom")
    name = (f"{tag}: 2D TM Maxwell PEC unit-square cavity, N={N}, K={K:,} triangles "
            f"({n}x{n} A16 mesh), {'fp32' if prec == 4 else 'fp64'}, LSERK4, "
            + ("two-layer eps 1|2.25 material" if args.material else "cavity mode (1,1)"))
    return VX, VY, E, K, Np, dt, name, eps, mu


def oracle_sample(N, n_sample, steps, material=False):
    """Time the fp64 NumPy oracle (as it stands) on an n_sample x n_sample mesh, one thread
    (BLAS pools limited to 1; the oracle's einsum contractions are single-threaded C loops)."""
    from threadpoolctl import threadpool_limits

    from oracle.solver import Oracle

    with threadpool_limits(limits=1):
        VX, VY, E = dginputs.rect_mesh(n_sample)
        eps = mu = None
        if material:
            eps, mu = dginputs.two_layer_material(VX, VY, E)
        o = Oracle(N, VX, VY, E, eps=eps, mu=mu)
        q = initial_fields(o.geo.x, o.geo.y, eps)
        dt = dginputs.cfl_dt(VX, VY, E, N, eps=eps, mu=mu)
        t0 = time.perf_counter()
        o.run(q, dt, steps)
        sec = time.perf_counter() - t0
    dof = o.Np * o.K * 3 * 5 * steps
    return dof / sec, sec, o.K


def _oracle_worker(a):
    return oracle_sample(*a)


def oracle_all_cores(N, n_sample, steps, material=False, cores=None):
    """The same bounded sample on every host core at once: `cores` independent oracle processes
    (one per core, each single-threaded), throughput = their summed DOF-updates / wall time.
    Returns (value, wall seconds, K, cores)."""
    import multiprocessing as mp

    cores = cores or os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        pool.map(_oracle_worker, [(1, 2, 1, False)] * cores)  # start-up + imports outside the clock
        t0 = time.perf_counter()
        res = pool.map(_oracle_worker, [(N, n_sample, steps, material)] * cores)
        wall = time.perf_counter() - t0
    Np = (N + 1) * (N + 2) // 2
    dof = sum(Np * r[2] * 3 * 5 * steps for r in res)
    return dof / wall, wall, res[0][2], cores


def cpu_baseline(N, n_sample, steps, material=False):
    """cpu_baseline of the bench line: the oracle on all host cores (headline) and on one."""
    v1, sec1, Ks = oracle_sample(N, n_sample, steps, material)
    va, wall, _, cores = oracle_all_cores(N, n_sample, steps, material)
    return {"value": va, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"fp64 NumPy oracle, N={N}, K={Ks} ({n_sample}x{n_sample} A16 mesh)"
                      f"{', two-layer material' if material else ''}, {steps} LSERK4 steps: "
                      f"{cores} independent single-threaded processes at once ({wall:.1f} s wall)",
            "single_thread": {"value": v1, "unit": UNIT, "cores": 1, "seconds": sec1}}


_REF = {}


def _ref_init(N, n_sample, material):
    """Reference-arm worker: build the oracle on the sample mesh once per process."""
    from threadpoolctl import threadpool_limits

    from oracle.solver import Oracle

    _REF["limits"] = threadpool_limits(limits=1)
    VX, VY, E = dginputs.rect_mesh(n_sample)
    eps = mu = None
    if material:
        eps, mu = dginputs.two_layer_material(VX, VY, E)
    o = Oracle(N, VX, VY, E, eps=eps, mu=mu)
    _REF.update(o=o, q=initial_fields(o.geo.x, o.geo.y, eps), dt=dginputs.cfl_dt(VX, VY, E, N, eps=eps, mu=mu))


def _ref_step(_):
    o = _REF["o"]
    _REF["q"] = o.run(_REF["q"], _REF["dt"], 1)
    return o.Np * o.K * 3 * 5


def run_reference(args, rank, world):
    """The reference arm: the fp64 NumPy oracle as it stands on every host core -- one
    single-threaded process per core, each advancing its own copy of the bounded sample (an
    n_sample x n_sample A16 mesh); one bench step = one LSERK4 step of every copy."""
    if rank != 0:
        return
    import multiprocessing as mp

    N = args.order
    _, _, _, K, Np, _, name, _, _ = workload(args)
    n_sample = args.ref_n
    cores = os.cpu_count() or 1
    with mp.get_context("spawn").Pool(cores, initializer=_ref_init, initargs=(N, n_sample, args.material)) as pool:
        for _ in range(args.warmup):
            pool.map(_ref_step, range(cores), chunksize=1)
        t0 = time.perf_counter()
        dof = 0
        for _ in range(args.steps):
            dof += sum(pool.map(_ref_step, range(cores), chunksize=1))
        sec = time.perf_counter() - t0
    value = dof / sec
    Ks = 2 * n_sample * n_sample
    sample = (f"fp64 NumPy oracle, N={N}, {n_sample}x{n_sample} A16 mesh (K={Ks}) per process"
              f"{', two-layer material' if args.material else ''}, {cores} single-threaded processes (one per "
              f"host core), {args.steps} steps after {args.warmup} warm-up")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": name, "reference_sample_K": Ks, "processes": cores},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_1304_5546_b200 import dg

    torch.cuda.set_device(local_rank)
    dist = None
    nccl_id = None
    if world > 1:
        import torch.distributed as dist_

        dist = dist_
        ids = [dg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        nccl_id = ids[0]
    VX, VY, E, K, Np, dt, name, eps, mu = workload(args)
    ctx = dg.dg_setup(args.order, VX, VY, E, eps=eps, mu=mu, precision=args.prec, device=local_rank, rank=rank,
                      nranks=world, fused=not args.split, transport=0, nccl_id=nccl_id,
                      kernel_variant=args.variant)
    x, y = ctx.nodes()
    eps_l = None if eps is None else eps[ctx.local_elements()]
    q0 = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in initial_fields(x, y, eps_l)]
    ctx.set_fields(*q0)
    stream = torch.cuda.ExternalStream(ctx.stream())

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # per-GPU working set (q ping-pong + residual + geometry + neighbour codes): when it is not
    # well above the 126 MB L2, the timed steps are separated by an L2 flush (a 512 MB write
    # outside the event brackets) so every step starts from HBM
    s = args.prec
    K_local = ctx.K_local
    ngeo = 32 if args.material else 16
    ws_bytes = 9 * K_local * Np * s + ngeo * K_local * s + 3 * (args.order + 1) * 4 * K_local
    flush = ws_bytes < 2 * L2_BYTES
    fbuf = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device="cuda") if flush else None
    # warm-up
    ctx.run(dt, args.warmup)
    ctx.sync()
    # timed region: exactly K steps as dg_run runs them (CUDA-graph replay), events on the
    # library's stream; the statistics reset first so gpu_launches counts this region only
    ctx.profile(True)
    ctx.profile(False)
    with ClockSampler(physical_gpu(local_rank)) as clk:
        time.sleep(0.05)
        barrier()
        t_wall = time.perf_counter()
        if not flush:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.run(dt, args.steps)
            e1.record(stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
        else:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            with torch.cuda.stream(stream):
                for a, b in evs:
                    fbuf.fill_(1.0)  # L2 flush, outside the bracket
                    a.record(stream)
                    ctx.run(dt, 1)
                    b.record(stream)
            evs[-1][1].synchronize()
            ms = sum(a.elapsed_time(b) for a, b in evs)
        t_wall_end = time.perf_counter()
        t_wall = t_wall_end - t_wall
        barrier()
    clocks = clk.summary(t_wall_end - t_wall, t_wall_end)
    launches = sum(v["launches"] for v in ctx.kernel_stats().values())
    kcfg = ctx.kernel_config()
    ctx.sync()
    # per-launch kernel durations (roofline): a separate profiled pass -- the same graph replay with
    # event-record nodes around every launch (dg_profile), read back between steps
    prof_steps = min(args.steps, 20)
    ctx.profile(True)
    if flush:
        with torch.cuda.stream(stream):
            for _ in range(prof_steps):
                fbuf.fill_(1.0)
                ctx.run(dt, 1)
    else:
        ctx.run(dt, prof_steps)
    stats = ctx.kernel_stats()
    ctx.profile(False)
    ctx.sync()
    if dist is not None:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = Np * K * 3 * 5 * args.steps / (ms * 1e-3)
    hbm, peak_src = peaks()
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            traffic_tab = json.load(fh)
    except Exception:
        traffic_tab = {}

    def roofline(kind):
        """Roofline of one stage kernel: algorithmic bytes and flops per launch over its average
        event-timed launch.  The binding roof is HBM unless the arithmetic intensity exceeds the
        ridge of the pipe the contraction runs on (C5: N=8 fp64, 6.3 flop/B > 36 TF / 6.54 TB/s)."""
        # kernel time per stage.  Single rank, fused: the timed region holds nothing but the stage
        # kernel (the profiles/ launch list), so its own CUDA-event time per stage is the launch time
        # (the profiled replay's event-record nodes add ~2%: reported alongside).  Otherwise (split, or a
        # multi-rank stage = pack + two launches) the profiled replay's per-launch event brackets.
        k_ms_events = stats[kind]["ms"] / (5 * prof_steps)
        k_ms = (ms / args.steps / 5) if (kind == "fused" and world == 1) else k_ms_events
        abytes = algorithmic_bytes_per_element_stage(Np, s, kind) * K_local
        flops = flops_per_element_stage(args.order, kind) * K_local
        achieved = abytes / (k_ms * 1e-3) / 1e9
        tflops = flops / (k_ms * 1e-3) / 1e12
        cbound, cpeak, csrc = compute_peak(s, kcfg["contraction"])
        hbm_roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "peak_source": peak_src}
        cmp_roof = {"bound": cbound, "achieved": tflops, "peak": cpeak, "unit": "TFLOP/s",
                    "frac": tflops / cpeak, "peak_source": csrc}
        intensity = flops / abytes
        main, alt = (cmp_roof, hbm_roof) if intensity > cpeak * 1e3 / hbm else (hbm_roof, cmp_roof)
        return dict(main, traffic=traffic_tab.get(f"N{args.order}_p{s}_n{args.n}_P{world}_{kind}"),
                    kernel=f"stage_kernel<{kind}>", algorithmic_bytes_per_launch=abytes, avg_launch_ms=k_ms,
                    timing=("timed region per stage (CUDA events on the library stream)" if k_ms is not k_ms_events
                            else "profiled graph replay, event-record nodes around each launch"),
                    event_bracket_ms=k_ms_events,
                    launches_per_stage=stats[kind]["timed"] / (5 * prof_steps),
                    # the timed region itself holds only this kernel (fused variant, profiles/ launch list):
                    # its CUDA-event time per stage, graph replay without the per-launch event nodes
                    region_ms_per_stage=(ms / args.steps / 5) if kind == "fused" else None,
                    region_frac=(abytes / (ms / args.steps / 5 * 1e-3) / 1e9 / hbm) if kind == "fused" else None,
                    flops_per_launch=flops, achieved_tflops=tflops, intensity_flop_per_byte=intensity,
                    ridge_flop_per_byte=cpeak * 1e3 / hbm,
                    other_roof={k: alt[k] for k in ("bound", "achieved", "peak", "unit", "frac", "peak_source")})

    if args.split:  # the dominant (longer) kernel; the other one alongside
        kinds = sorted(("volume", "surface"), key=lambda k: -stats[k]["ms"])
        roof = roofline(kinds[0])
        roof["second_kernel"] = roofline(kinds[1])
    else:
        roof = roofline("fused")
    # e2e through the public API with host buffers (job level: set fields, K steps, get fields)
    barrier()
    outs = [torch.empty_like(a).pin_memory() for a in q0]
    t0 = time.perf_counter()
    ctx.set_fields(*q0)
    ctx.run(dt, args.steps)
    ctx.get_fields(outs)
    e2e_sec = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_sec], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_sec = float(t.item())
    fbytes = 3 * K * Np * 8
    e2e = {"value": Np * K * 3 * 5 * args.steps / e2e_sec, "unit": UNIT,
           "h2d_bytes_per_step": fbytes / args.steps, "d2h_bytes_per_step": fbytes / args.steps,
           "scope": "dg_set_fields(pinned host fp64) + dg_run(K steps) + dg_get_fields(pinned host fp64)"}
    ctx.destroy()
    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.order, args.ref_n, args.ref_steps, args.material)
    ws_mb = ws_bytes / 1e6
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.config == "c5w" else "strong", "vs_baseline": None,
            "dtype": "f32" if s == 4 else "f64", "data": "synthetic",
            "config": {"workload": name, "N": args.order, "K": K, "Np": Np, "dt": dt,
                       "variant": "split" if args.split else "fused", "parallelism": f"element-partition x{world}",
                       "l2": (f"L2 flushed between timed steps (512 MB write outside the event brackets): "
                              f"per-GPU working set {ws_mb:.0f} MB is not > 2x the 126 MB L2") if flush else
                             f"no flush: per-GPU working set {ws_mb:.0f} MB > 2x the 126 MB L2",
                       "contraction": {"fma": "CUDA-core FMA", "dmma_fp64": "fp64 tensor cores (DMMA)",
                                       "3xtf32": "fp32 via 3xTF32 tensor-core split (hi*hi+lo*hi+hi*lo, "
                                                 "fp32 accumulate; mma.sync)",
                                       "tcgen05_3xtf32": "fp32 via 3xTF32 on tcgen05.mma kind::tf32 (TMEM "
                                                         "accumulators, 128-element groups)"}[kcfg["contraction"]],
                       "kernel_config": kcfg},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "wall_s_timed": t_wall}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- 3D (hedge)
def bytes_3d(Np, Nfp, s, kind):
    """Algorithmic bytes per element per stage of the 3D kernels: volume = read the
    6 fields + 9 geometry words, write rhsV; surface = read rhsV, q (RK) and the residual on stages
    1-4, write q_out and the residual on stages 0-3, + 20 face words + 4 Nfp neighbour codes (the
    traces are re-reads of q: L2 hits, not counted)."""
    if kind == "volume":
        return (12 * Np + 9) * s
    if kind == "fused":  # q in / out, the residual (read on stages 1-4, written on 0-3), 9 + 20 geometry words
        return (12 * Np + 2 * 0.8 * 6 * Np + 29) * s + 4 * Nfp * 4
    return (12 * Np + 2 * 0.8 * 6 * Np + 20) * s + 4 * Nfp * 4


def flops_3d(N, kind):
    Np, Nfp = (N + 1) * (N + 2) * (N + 3) // 6, (N + 1) * (N + 2) // 2
    if kind == "volume":
        return 2 * 18 * Np * Np + 36 * 2 * Np   # 18 mat-vecs + the chain-rule combinations
    if kind == "fused":
        return flops_3d(N, "volume") + flops_3d(N, "surface")
    NF = 4 * Nfp
    return 2 * 6 * Np * NF + NF * 6 * 12 + 6 * Np * 5  # LIFT of 6 fields + flux + rhsV add and LSERK4


def run_3d(args):
    """The 3D tetrahedral Maxwell step (config 'hedge3d'): PEC unit cube, n^3 cells x 6 Kuhn tetrahedra,
    the (1,1,1) cavity mode, LSERK4; one step = 5 stages x (the fused stage kernel, or with --split /
    where the fused tile does not fit: volume kernel + surface/LIFT/RK kernel)."""
    import torch

    from paper_1304_5546_b200 import dg3

    torch.cuda.set_device(0)
    N, n, prec = args.order, args.n, args.prec
    VX, VY, VZ, E = dginputs.cube_tet_mesh(n)
    K = E.shape[0]
    c = dg3.dg3_setup(N, VX, VY, VZ, E, precision=prec, fused=not args.split)
    Np, Nfp = c.Np, c.Nfp
    x, y, z = c.nodes()
    c.set_fields(*dginputs.cube_cavity_mode(x, y, z, 0.0))
    dt = dginputs.cfl_dt_3d(VX, VY, VZ, E, N)
    stream = torch.cuda.ExternalStream(c.stream())
    c.run(dt, args.warmup)
    c.sync()
    c.profile(True)
    c.profile(False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(physical_gpu(0)) as clk:
        t0 = time.perf_counter()
        e0.record(stream)
        c.run(dt, args.steps)
        e1.record(stream)
        e1.synchronize()
        t1 = time.perf_counter()
    ms = e0.elapsed_time(e1)
    launches = sum(v["launches"] for v in c.kernel_stats().values())
    prof = min(args.steps, 10)
    c.profile(True)
    c.run(dt, prof)
    st = c.kernel_stats()
    c.profile(False)
    c.sync()
    hbm, peak_src = peaks()
    s = prec
    roofs = {}
    kinds = [k for k in ("fused", "volume", "surface") if st[k]["timed"] > 0]
    for kind in kinds:
        k_ms = st[kind]["ms"] / (5 * prof)
        ab = bytes_3d(Np, Nfp, s, kind) * K
        fl = flops_3d(N, kind) * K
        cb, cp, csrc = compute_peak(s, "fma")
        gbs, tfl = ab / (k_ms * 1e-3) / 1e9, fl / (k_ms * 1e-3) / 1e12
        hroof = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm, "peak_source": peak_src}
        croof = {"bound": cb, "achieved": tfl, "peak": cp, "unit": "TFLOP/s", "frac": tfl / cp, "peak_source": csrc}
        main, alt = (croof, hroof) if fl / ab > cp * 1e3 / hbm else (hroof, croof)
        roofs[kind] = dict(main, kernel=f"{kind}3d", avg_launch_ms=k_ms, algorithmic_bytes_per_launch=ab,
                           flops_per_launch=fl, achieved_gflops=tfl * 1e3,
                           other_roof={k: alt[k] for k in ("bound", "achieved", "peak", "unit", "frac")})
    dom = max(roofs, key=lambda k: roofs[k]["avg_launch_ms"])
    roof = dict(roofs[dom])
    if len(roofs) > 1:
        roof["second_kernel"] = roofs["volume" if dom == "surface" else "surface"]
    # e2e through the public API: set fields (host fp64), K steps, get fields
    host = [np.ascontiguousarray(a) for a in dginputs.cube_cavity_mode(x, y, z, 0.0)]
    t0e = time.perf_counter()
    c.set_fields(*host)
    c.run(dt, args.steps)
    c.get_fields()
    e2e_s = time.perf_counter() - t0e
    c.destroy()
    value = Np * K * 6 * 5 * args.steps / (ms * 1e-3)
    fbytes = 6 * K * Np * 8
    flops_step = 5 * K * (flops_3d(N, "volume") + flops_3d(N, "surface"))
    line = {"metric": METRIC + " [3D tetrahedral path]", "value": value, "unit": UNIT + " (6 fields)", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "none", "vs_baseline": None, "dtype": "f32" if prec == 4 else "f64", "data": "synthetic",
            "config": {"workload": f"hedge3d: 3D TM/TE Maxwell PEC unit cube, N={N}, K={K:,} tetrahedra "
                                   f"({n}^3 cells x 6), {'fp32' if prec == 4 else 'fp64'}, LSERK4, cavity mode (1,1,1)",
                       "N": N, "K": K, "Np": Np,
                       "kernels": ("fused stage: volume (18 mat-vecs) + flux + LIFT + LSERK4 (FMA)" if kinds == ["fused"]
                                   else "volume (18 mat-vecs) + surface/LIFT/LSERK4 (FMA)"),
                       "l2": f"no flush: working set {(9 * K * Np * s) / 1e6:.0f} MB"},
            "gflops": flops_step / (ms / args.steps * 1e-3) / 1e9,
            "roofline": roof, "cpu_baseline": None,
            "e2e": {"value": Np * K * 6 * 5 * args.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": fbytes / args.steps,
                    "d2h_bytes_per_step": fbytes / args.steps},
            "gpu_launches": launches, "clocks": clk.summary(t0, t1)}
    print(json.dumps(line), flush=True)


def visible_gpus():
    """Number of CUDA devices this process can see (0 without a driver)."""
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


def spawn_ranks(n):
    """bench.py --gpus N without a launcher: re-run this command under torchrun, one rank per GPU
    (the driver's own launch line: --nnodes=1 --master-addr 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def run_partitions_dry(args):
    """P in-process partitions of the workload on one GPU, advanced by dg_run_group: the multi-GPU
    data path (element partition, halo pack, interior-then-boundary tile-list launches) with the
    NCCL transport replaced by device copies.  Not a scaling number: all P partitions share one GPU."""
    import torch

    from paper_1304_5546_b200 import dg

    P = args.partitions
    torch.cuda.set_device(0)
    VX, VY, E, K, Np, dt, name, eps, mu = workload(args)
    cs = [dg.dg_setup(args.order, VX, VY, E, eps=eps, mu=mu, precision=args.prec, device=0, rank=r, nranks=P,
                      fused=not args.split, transport=1) for r in range(P)]
    for c in cs:
        x, y = c.nodes()
        eps_l = None if eps is None else eps[c.local_elements()]
        c.set_fields(*initial_fields(x, y, eps_l))
    stream = torch.cuda.ExternalStream(cs[0].stream())
    dg.dg_run_group(cs, dt, args.warmup)
    torch.cuda.synchronize()
    for c in cs:
        c.profile(True)
        c.profile(False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(physical_gpu(0)) as clk:
        t0 = time.perf_counter()
        e0.record(stream)
        dg.dg_run_group(cs, dt, args.steps)
        e1.record(stream)
        e1.synchronize()
        t1 = time.perf_counter()
    ms = e0.elapsed_time(e1)
    launches = sum(v["launches"] for c in cs for v in c.kernel_stats().values())
    halo = sum(c.n_halo_points for c in cs)
    for c in cs:
        c.destroy()
    line = {"metric": METRIC, "value": Np * K * 3 * 5 * args.steps / (ms * 1e-3), "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "none (dry run)", "dry_run": True, "vs_baseline": None,
            "dtype": "f32" if args.prec == 4 else "f64",
            "data": "synthetic",
            "config": {"workload": name, "N": args.order, "K": K, "variant": "split" if args.split else "fused",
                       "parallelism": f"{P} in-process partitions on 1 GPU (transport 1: halo pack, device-copy "
                                      f"exchange, interior then boundary tile-list launches)",
                       "halo_points": halo},
            "roofline": None, "cpu_baseline": None, "e2e": None, "gpu_launches": launches,
            "clocks": clk.summary(t0, t1)}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS) + ["custom"],
                    help="workload preset (BASELINE.json configs); --order/--n/--prec/--material override")
    ap.add_argument("--order", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--prec", type=int, default=None, choices=[4, 8])
    ap.add_argument("--material", action="store_true", default=None)
    ap.add_argument("--split", action="store_true", help="volume + surface/RK kernels instead of fused")
    ap.add_argument("--variant", default="tuned", choices=["tuned", "tcgen05"],
                    help="stage kernels: the tuned set (csrc/tune.json) or the fp32 tcgen05 variant")
    ap.add_argument("--ref-n", type=int, default=48, help="oracle sample mesh cells per side")
    ap.add_argument("--ref-steps", type=int, default=200)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dim", type=int, default=2, choices=[2, 3],
                    help="3: the 3D tetrahedral path (config hedge3d: --order N, --n cells per cube side)")
    ap.add_argument("--partitions", type=int, default=0,
                    help="dry run of the multi-GPU data path on ONE GPU: P in-process partitions "
                         "(transport 1, dg_run_group)")
    args = ap.parse_args()
    if args.dim == 3:
        args.config = "hedge3d"
        args.order = args.order or 4
        args.n = args.n or 40
        args.prec = args.prec or 4
    preset = CONFIGS.get(args.config, CONFIGS["c4"])
    for key, val in preset.items():
        if getattr(args, key) is None:
            setattr(args, key, val)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.partitions == 0 and args.impl == "ours":
        visible = visible_gpus()
        if visible >= args.gpus:
            spawn_ranks(args.gpus)  # does not return
        # fewer GPUs than ranks (e.g. a 1-GPU development box): the labelled dry run of the same data
        # path -- args.gpus in-process partitions on one GPU -- instead of ranks that cannot start
        print(f"warning: --gpus {args.gpus} but {visible} GPU(s) visible: dry run with {args.gpus} in-process "
              f"partitions on one GPU", file=sys.stderr)
        args.partitions = args.gpus
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.config == "c5w" and args.n == CONFIGS["c5w"]["n"]:  # weak scaling: ~524k elements per GPU
        args.n = {1: 512, 2: 724, 4: 1024, 8: 1448}.get(world_env, int(round(512 * world_env ** 0.5)))
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.partitions > 0:
        run_partitions_dry(args)
        return
    if args.dim == 3:
        run_3d(args)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
