"""bench.py keeps the driver's JSON-line contract (both arms), on tiny sizes."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--workload", "mu1m", "--warm", "3000",
              "--wave", "256", "--capacity", "300000"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_device_arm_line():
    d = _run(["--steps", "4", "--warmup", "3", "--workload", "mu1m", "--warm", "20000", "--wave", "1024",
              "--capacity", "2000000", "--parity-waves", "1", "--profile-steps", "2"])
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["unit"] == "decisions/s" and d["scaling"] == "weak"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["peak"] > 0 and 0 <= r["frac"] < 1 and r["achieved"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["config"]["commit"]["parallel_waves"] > 0
    assert 0 < d["hit_rate"] < 1
    assert d["parity"]["identical"] and d["parity"]["waves_checked"] == 1, d["parity"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


@pytest.mark.gpu
def test_device_arm_two_replicas_one_gpu():
    """bench.py --gpus 2 relaunches itself under torch.distributed.run; both
    replicas (here on cuda:0, gloo for the demand all-reduce) take their
    segment-hash shard of one stream, and each shard matches the oracle."""
    d = _run(["--gpus", "2", "--same-device", "--backend", "gloo", "--workload", "c3", "--warm", "1024",
              "--wave", "256", "--capacity", "700000", "--steps", "3", "--warmup", "3", "--parity-waves", "1",
              "--profile-steps", "1", "--e2e-steps", "2"], timeout=900)
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["parity"]["identical"] and d["parity"]["identical_all_shards"], d["parity"]
    assert d["config"]["admitted_per_rank"] > 0
    assert d["cpu_baseline"] is None  # the CPU baseline is an N=1 leg


def test_reference_arm_n2():
    d = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--workload", "mu1m",
              "--warm", "2000", "--wave", "256", "--capacity", "200000", "--ref-seconds", "0.5"])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
