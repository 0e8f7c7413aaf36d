"""bench.py's reference arm (CPU only) prints one JSON line with the contract's
keys for the configuration it actually ran, and exits 0 on non-zero ranks."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env_extra=None):
    env = dict(os.environ, **(env_extra or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=env, timeout=600, cwd=ROOT)


def test_reference_arm_json_line():
    p = run(["--impl", "reference", "--steps", "5", "--warmup", "3", "--log2n", "18"])
    assert p.returncode == 0, p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    # the full configuration is run (no extrapolation from a sample); the step
    # counts are the ones actually timed
    assert d["config"]["n"] == 1 << 18
    assert d["steps"] == 3 and d["warmup"] in (0, 1)
    cb = d["cpu_baseline"]
    assert len(cb["seconds"]) == d["steps"]
    assert abs(d["ms_per_step"] - sorted(cb["seconds"])[1] * 1e3) < 0.1
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]


def test_reference_arm_non_zero_rank_is_silent():
    p = run(["--impl", "reference", "--steps", "1", "--warmup", "3", "--log2n", "16"],
            {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert p.returncode == 0 and p.stdout.strip() == ""
