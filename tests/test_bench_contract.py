"""bench.py's reference arm runs on CPU (it times the oracle):
check its JSON line carries the keys the driver reads, and that a non-zero
rank under torchrun exits without output."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None):
    e = dict(os.environ, **(env or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, timeout=600, cwd=ROOT, env=e)


def test_reference_arm_json():
    res = run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "cfg2"])
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_silent():
    res = run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "cfg1"],
              env={"RANK": "1", "WORLD_SIZE": "2"})
    assert res.returncode == 0 and not [l for l in res.stdout.splitlines() if l.startswith("{")]


@pytest.mark.gpu
def test_bench_json_on_gpu():
    """Our arm at the smallest config: every key the driver reads, sane values."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    res = run(["--config", "cfg1", "--steps", "3", "--warmup", "3"])
    assert res.returncode == 0, res.stderr[-3000:]
    d = json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    # the timed solve checks itself against the exact modal recurrence
    assert d["parity"]["ok"], d["parity"]
    assert d["parity"]["max_abs_dk_vs_modal"] <= 1e-10 and d["parity"]["u_T_rel_err_vs_modal"] <= 1e-12
    assert d["roofline"]["within_peak"]
    # the reference arm reports the same workload config
    ref = run(["--impl", "reference", "--config", "cfg1", "--steps", "1", "--warmup", "0"])
    r = json.loads([l for l in ref.stdout.splitlines() if l.startswith("{")][-1])
    assert r["config"] == d["config"]

