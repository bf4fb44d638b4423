"""bench.py keeps its contract: one JSON line with the keys the driver reads
(metric, value, e2e, roofline, cpu_baseline, clocks, gpu_launches, ...), for
the B200 arm (GPU) and the reference arm (CPU, the unmodified reference)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "locmax")):
        pytest.skip("reference not installed (tools/install_reference.sh)")
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-sample-scale", "11"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "edges/s"
    assert d["metric"] == "input edges/s to full local max maximal matching"
    assert d["higher_is_better"] is True and d["n_gpus"] == 1
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] == 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_b200_arm_line():
    d = _run(["--workload", "rmat20", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"])
    assert d["metric"] == "input edges/s to full local max maximal matching" and d["unit"] == "edges/s"
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["steps"] == 3 and d["warmup"] == 3
    assert d["n_gpus"] == 1 and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["dtype"] and d["data"] == "synthetic" and d["config"]["workload"] == "rmat20"
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == "edges/s"
    m = d["config"]["m"]
    assert e["h2d_bytes_per_step"] == 16 * m and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    assert d["step_roofline"]["frac"] > 0
    assert d["cpu_baseline"] is None                       # --no-cpu-baseline
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and isinstance(c["reasons"], list)
    assert d["gpu_launches"] > 0
    assert d["device_memory"]["load_peak_GB"] >= d["device_memory"]["after_load_GB"] > 0


@pytest.mark.gpu
def test_two_rank_line_over_gloo():
    """The N-GPU line (torchrun, one rank per GPU) end to end: distributed
    RMAT build, the round protocol, the per-rank e2e leg (local edges from
    page-locked host memory), rank 0's CPU baseline -- two ranks on the test
    box's one GPU with gloo's host-staged collectives (--backend is test only;
    the driver's runs use NCCL)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29537", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--backend", "gloo", "--workload", "rmat16", "--steps", "3", "--warmup", "3",
           "--cpu-baseline-scale", "12"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                         env=dict(os.environ, OMP_NUM_THREADS="1"))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["build"].startswith("distributed")
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["value"] > 0 and d["gpu_launches"] > 0
