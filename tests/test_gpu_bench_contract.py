"""The bench.py JSON line keeps the driver's contract (keys, types, units)."""

import json
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_bench_line_has_every_contract_key(cuda):
    # the default run: configs[4] (64 waveforms of 2^23 samples), complex128
    d = _run("--steps", "3", "--warmup", "3", "--no-cpu-baseline", timeout=1200)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["dtype"].startswith("c128")
    assert d["config"]["baseline_config_index"] == 4 and "workload" in d["config"]
    assert d["config"]["waveforms_per_gpu"] == 64
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0 < r["frac"] < 1
    e = d["e2e"]
    assert e["value"] > 0
    assert e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 64 * 2 * (1 << 23) * 16
    assert d["gpu_launches"] == 3
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    x = d["extras"]
    for k in ("c64_same_workload", "configs1_c128", "configs1_c64", "run_dbp_wall"):
        assert k in x, k
    assert x["c64_same_workload"]["value"] > d["value"]
    assert d["kernel"]["name"].startswith("cbessfm_")


def test_bench_gpus_flag_launches_ranks(cuda):
    # --gpus N without a launcher re-executes under torch.distributed.run;
    # gloo keeps every rank on cuda:0 (control flow only, not a measurement)
    import os
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2",
                          "--workload", "cfg2", "--steps", "2", "--warmup", "3",
                          "--no-extras"], cwd=ROOT, capture_output=True, text=True,
                         timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 2
    assert d["gather"] is not None and d["gather"]["bytes_per_rank"] > 0
    assert d["config"]["waveforms_total"] == 2


def test_bench_rejects_world_mismatch():
    import os
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2"],
                         cwd=ROOT, capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_reference_arm_line(cuda):
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["baseline_config_index"] == 4
