"""bench.py keeps the driver's JSON contract: one line, the required keys, the reference arm (the CPU oracle)
runnable without a GPU, the GPU arm with roofline / cpu_baseline / e2e / clocks / spmv objects."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e"]


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_is_the_oracle():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "0"], timeout=600)
    for k in KEYS:
        assert k in d, k
    assert d["impl"] == "reference" and d["config"]["workload"] == "cfg0"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and d["value"] > 0 and cb["value"] == d["value"]
    assert cb["cores"] >= 1 and "host cores" in cb["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_default_workload_is_cfg4():
    """The driver's bench line is the largest single-GPU configuration (cfg4: HBM regime)."""
    sys.path.insert(0, ROOT)
    import bench
    old = sys.argv
    try:
        sys.argv = ["bench.py"]
        assert bench.parse().config == 4
    finally:
        sys.argv = old
    cfg, what = bench.oracle_sample_cfg(4)
    assert cfg["h"] == 1 / 16 and cfg["grid"] == [4, 4, 4] and "upper bound" in what


@pytest.mark.gpu
def test_gpu_arm_contract():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--steps", "3", "--warmup", "3", "--no-cpu-baseline"], timeout=900)
    for k in KEYS + ["roofline", "clocks", "gpu_launches", "spmv"]:
        assert k in d, k
    assert d["config"]["workload"] == "cfg4" and d["dtype"] == "f64" and d["higher_is_better"] is True
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["gpu_launches"] > 0 and d["value"] > 0
    assert d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
