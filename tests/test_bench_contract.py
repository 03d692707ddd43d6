"""The bench's reference arm runs on CPU: check its JSON-line contract (-m "not gpu")."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C1", "--steps", "2",
                          "--warmup", "1", "--cpu-seconds", "0.5"], cwd=ROOT, capture_output=True, text=True,
                         timeout=300, check=True).stdout.strip().splitlines()
    assert len(out) == 1
    d = json.loads(out[0])
    for k in ["impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"]:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["config"]["workload"] == "C1"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
