"""The bench.py reference arm runs on CPU and prints the JSON line the driver parses
(contract keys, impl, cpu_baseline and e2e blocks)."""

import json
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    t0 = time.perf_counter()
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "impl",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] and d["metric"] == "train tokens/s (Ulysses SP)"
    # a MEASURED sample (not an extrapolation): the claimed per-step time fits the run
    wall = time.perf_counter() - t0
    assert (d["steps"] + d["warmup"]) * d["ms_per_step"] / 1e3 <= wall
    assert abs(d["value"] * d["ms_per_step"] / 1e3 - d["config"]["tokens_per_step"]) < 1e-6
    s3 = d["cpu_baseline"]["baseline_md_s3"]
    assert s3["c1_end_to_end"]["tokens_per_s"]["fp64"] > 0 and len(s3["a2a_gbs"]) == 2
