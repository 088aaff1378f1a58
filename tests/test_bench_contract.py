"""bench.py's JSON-line contract (the driver parses it): the reference arm on the host cores (CPU), and a short run of
our arm at reduced sequence length on the GPU (incl. the one-rank NCCL exchange path).  Full-size numbers come from the
driver's own bench runs; these tests only pin the fields and their consistency."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    """--impl reference: the fp64 oracle on the host (this tier's reference arm), same metric / unit / config as ours."""
    r = _bench("--impl", "reference", "--steps", "1", "--warmup", "0", timeout=600)
    assert r["impl"] == "reference"
    assert r["unit"] == "tokens/s" and r["higher_is_better"] is True and r["value"] > 0
    assert r["steps"] == 1 and r["n_gpus"] == 1 and r["ms_per_step"] > 0
    assert r["cpu_baseline"]["kind"] == "oracle" and r["cpu_baseline"]["cores"] >= 1
    assert r["cpu_baseline"]["value"] == r["value"]
    assert r["e2e"] == {"value": r["value"], "unit": r["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert r["config"]["S"] == 524288 and r["config"]["head_dim"] == 80


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [(), ("--exchange-path",)])
def test_our_arm_line_small(extra):
    r = _bench("--seq", "131072", "--steps", "1", "--warmup", "3", "--no-cpu-baseline", *extra)
    assert r["unit"] == "tokens/s" and r["value"] > 0 and r["n_gpus"] == 1 and r["steps"] == 1 and r["warmup"] == 3
    assert abs(r["value"] - r["config"]["S"] / (r["ms_per_step"] / 1e3)) <= 1e-6 * r["value"]
    rf = r["roofline"]
    assert rf["bound"] == "tensor" and rf["unit"] == "TFLOP/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert r["gpu_launches"] > 0
    assert set(r["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    e = r["e2e"]
    assert e["unit"] == "tokens/s" and e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["outputs_equal_device_path"] is True
    if extra:
        assert r["exchange"] is not None and r["exchange"]["count_per_step"] > 0
        assert r["config"]["parallelism"].endswith("nccl1")
    else:
        assert r["exchange"] is None
