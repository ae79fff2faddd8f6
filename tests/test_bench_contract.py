"""bench.py contract on CPU: the reference arm (the compiled reference in
oracle/_ref, timed on this host) prints one JSON line with the keys the driver
reads, for the CPU-runnable BASELINE config."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    from oracle import REF_DIR
    if not any(REF_DIR.glob("libfsk_ref_fast_v*.so")):
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--config", "cfg1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["unit"] == "iterations/s"
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in line["config"]


def test_uniform_weights_pass_reference_validation():
    """Weights for the BASELINE sizes pass core.cpp:27-33's naive-sum check
    (plain 1/n fails at n = 1e5, SURVEY §0 finding 4)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", ROOT / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for n in (4096, 10000, 65536, 100000, 1 << 20):
        w = bench.uniform_weights(n)
        s = 0.0
        for v in w:
            s += v
        assert abs(s - 1.0) <= 1e-12
