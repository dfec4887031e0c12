"""bench.py's driver contract, checked on the CPU: the reference arm (the fp64 oracle timed on the
host cores, a bounded sample of the bench workload) prints ONE JSON line with the contract's keys,
and the product arm has no CPU fallback -- without a GPU it exits non-zero instead of timing
anything."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)


def _one_line(p):
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_json_line():
    """The default workload (config 3): SURVEY.md 8(d)'s oracle sample -- layer 0 over the longest and the
    shortest sequence at full length, extrapolated by the FLOP ratio, CPU model recorded."""
    d = _one_line(_run("--impl", "reference", "--steps", "1", "--warmup", "0"))
    assert d["steps"] == 1 and d["warmup"] == 0
    assert d["config"]["workload"].startswith("gpt3_13b: 40 layers")
    assert "longest (502)" in d["cpu_baseline"]["sample"] and "shortest (47)" in d["cpu_baseline"]["sample"]
    assert "extrapolated" in d["cpu_baseline"]["sample"] and d["cpu_baseline"]["cpu_model"]


def test_reference_arm_contract_keys():
    d = _one_line(_run("--impl", "reference", "--config", "gpt2s", "--steps", "1", "--warmup", "3"))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["steps"] == 1 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["unit"] == "tokens/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"].startswith("gpt2s: 12 layers")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_product_arm_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    p = _run("--steps", "1", "--warmup", "3", timeout=300)
    assert p.returncode != 0
    assert not [l for l in p.stdout.splitlines() if l.strip().startswith("{")]


def test_self_launch_multi_rank():
    """`bench.py --gpus 2` outside torchrun relaunches itself under torch.distributed.run (two ranks,
    rendezvous on 127.0.0.1); only rank 0 prints, exactly one JSON line."""
    d = _one_line(_run("--gpus", "2", "--impl", "reference", "--config", "gpt2s", "--steps", "1", "--warmup", "3"))
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["tp"] == 2


def test_self_launch_refuses_missing_gpus():
    """The product arm with --gpus 2 and no GPUs: one JSON error line, non-zero exit, nothing timed."""
    p = _run("--gpus", "2", "--steps", "1", "--warmup", "3", timeout=300)
    assert p.returncode != 0
    lines = [l for l in p.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1 and "error" in json.loads(lines[0])
