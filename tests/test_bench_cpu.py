"""bench.py host logic on CPU: the reference arm's JSON line (the oracle timed on host cores, the
one place besides cpu_baseline where bench.py runs oracle/) and the roofline bookkeeping
(algorithmic bytes and flops per element-stage) against hand counts."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_reference_arm_json_line():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "3", "--ref-n", "6"], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["higher_is_better"] is True
    assert line["value"] > 0 and line["steps"] == 2 and line["warmup"] == 3
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == line["value"] and "6x6" in cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("C4")


def test_reference_arm_other_ranks_print_nothing():
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "3", "--ref-n", "4"], capture_output=True, text=True,
                       timeout=300, env=env)
    assert p.returncode == 0 and p.stdout.strip() == ""


def test_algorithmic_bytes_and_flops_hand_counts():
    # N=5: Np = 21, Nfp = 6.  Fused: (6 + 4.8) Np words + 13 geometry words + 16 B connectivity
    assert bench.algorithmic_bytes_per_element_stage(21, 4) == 10.8 * 21 * 4 + 13 * 4 + 16 == 975.2
    assert bench.algorithmic_bytes_per_element_stage(21, 8) == 10.8 * 21 * 8 + 13 * 8 + 16
    # N=8 fp64 (C5): Np = 45 -> 4.01 KB per element-stage
    assert abs(bench.algorithmic_bytes_per_element_stage(45, 8) - 4008.0) < 1e-9
    # split: volume q + rhsV + 4 words; surface q, rhsV, q_out + residual + 9 face words + codes
    assert bench.algorithmic_bytes_per_element_stage(21, 4, "volume") == 6 * 21 * 4 + 4 * 4
    assert bench.algorithmic_bytes_per_element_stage(21, 4, "surface") == 13.8 * 21 * 4 + 9 * 4 + 16
    # flops: 8 Np^2 + 8 Np (volume) + 18 Np Nfp (LIFT) + 108 Nfp (flux) + 12 Np (RK)
    assert bench.flops_per_element_stage(5) == 8 * 441 + 8 * 21 + 18 * 21 * 6 + 108 * 6 + 12 * 21 == 6864
    assert bench.flops_per_element_stage(5, "volume") + bench.flops_per_element_stage(5, "surface") \
        == 6864 + 3 * 21


def test_spawn_ranks_builds_torchrun_command(monkeypatch):
    seen = {}

    def fake_execv(exe, cmd):
        seen["cmd"] = cmd
        raise SystemExit(0)

    monkeypatch.setattr(os, "execv", fake_execv)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    try:
        bench.spawn_ranks(4)
    except SystemExit:
        pass
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--nnodes=1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]


def test_physical_gpu_follows_cuda_visible_devices(monkeypatch):
    monkeypatch.setenv("CUDA_VISIBLE_DEVICES", "3,5")
    assert bench.physical_gpu(1) == "5"
    monkeypatch.setenv("CUDA_VISIBLE_DEVICES", "GPU-abc,GPU-def")
    assert bench.physical_gpu(0) == "GPU-abc"
    monkeypatch.delenv("CUDA_VISIBLE_DEVICES")
    assert bench.physical_gpu(2) == "2"


def test_clock_summary_keeps_the_timed_window():
    c = bench.ClockSampler("0")
    c.samples = [(0.0, 900.0, 1965.0, []), (1.0, 1965.0, 1965.0, ["sw_power_cap"]),
                 (2.0, 1965.0, 1965.0, []), (3.0, 120.0, 1965.0, ["hw_slowdown"])]
    s = c.summary(0.5, 2.5)
    assert s["sm_mhz"] == 1965.0 and s["reasons"] == ["sw_power_cap"] and s["samples_in_timed_region"] == 2


def test_cpu_baseline_all_cores_and_single_thread():
    cb = bench.cpu_baseline(2, 3, 2)
    assert cb["kind"] == "oracle" and cb["cores"] == (os.cpu_count() or 1) and cb["value"] > 0
    assert cb["single_thread"]["cores"] == 1 and cb["single_thread"]["value"] > 0
    assert "3x3" in cb["sample"]


def test_gpus_without_enough_devices_falls_back_to_the_labelled_dry_run(monkeypatch):
    """--gpus N with fewer visible GPUs runs the in-process partition dry run (not torchrun ranks)."""
    called = {}
    monkeypatch.setattr(bench, "visible_gpus", lambda: 1)
    monkeypatch.setattr(bench, "spawn_ranks", lambda n: called.setdefault("spawn", n))
    monkeypatch.setattr(bench, "run_partitions_dry", lambda a: called.setdefault("dry", a.partitions))
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--steps", "3"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    bench.main()
    assert called == {"dry": 2}
