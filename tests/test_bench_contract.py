"""bench.py's driver contract on CPU: the reference arm (the oracle, which needs no GPU) prints one JSON
line with the contract's keys at the same workload description as the GPU arm, and `--gpus 2` without a
launcher re-executes itself under torch.distributed.run (two ranks; rank 0 alone prints)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "higher_is_better", "n_gpus", "steps", "warmup", "ms_per_step", "scaling",
        "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"}


def _run(args, timeout=600):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return lines


def test_reference_arm_json_line():
    lines = _run(["--impl", "reference", "--config", "c1", "--steps", "4", "--warmup", "2"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["higher_is_better"] is False and d["unit"] == "ms/IPM-iter"
    assert d["steps"] == 3 and d["steps_requested"] == 4 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["N"] == 50 and d["config"]["n"] == 67 * 51 and d["value"] > 0


def test_gpus_flag_spawns_ranks():
    """--gpus 2 re-executes under torch.distributed.run: two processes, one JSON line (rank 0)."""
    lines = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1", "--gpus", "2"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"].startswith("replicas x2")


import pytest  # noqa: E402


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """The GPU arm on the small config: one JSON line with the contract's keys, the roofline / CPU
    baseline / e2e / clocks objects and a positive count of the library's own kernel launches."""
    lines = _run(["--config", "c1", "--steps", "3", "--warmup", "3"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert (KEYS - {"impl"}) <= set(d), KEYS - set(d)
    assert d["dtype"] == "f64" and d["higher_is_better"] is False and d["value"] > 0 and d["n_gpus"] == 1
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1 and r["achieved"] > 0
    assert r["traffic"] is None  # the committed ncu capture is of C3, not of this config
    assert abs(r["frac"] - r["achieved"] / r["peak"]) <= 1e-9 * r["frac"]
    e = d["e2e"]
    assert e["value"] >= d["value"] * 0.5 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
