"""The bench.py contract on a B200: one JSON line with the keys the driver reads, consistent
units, the device-timed and end-to-end legs, the roofline of the attention kernel and the
launch count claim. Short run (2 timed chunks, no long video, no CPU baseline)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra):
    r = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3",
                        "--skip-long-video", *extra],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "roofline", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["unit"] == "latent frames/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and abs(d["value"] - 3 * 1e3 / d["ms_per_step"]) < 1e-6 * d["value"]
    e2e = d["e2e"]
    # the streaming e2e overlaps its copies with compute: bounded by the faster device rate
    assert e2e["unit"] == d["unit"]
    assert 0 < e2e["value"] <= max(d["value"], d["graph_replay"]["value"]) * 1.02
    assert e2e["h2d_bytes_per_step"] == 4 * 4680 * 1536 * 2   # 4 denoise steps of bf16 noise
    assert e2e["d2h_bytes_per_step"] == 4680 * 1536 * 2       # one bf16 latent
    rf = d["roofline"]
    assert rf["bound"] == "tensor" and rf["unit"] == "TFLOP/s"
    assert 0 < rf["frac"] <= 1.0 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    # every timed chunk runs 120 layer calls of three kernels (QKV+RoPE, attention, O-proj)
    assert d["gpu_launches"] == 2 * 120 * 3
    assert "workload" in d["config"] and d["config"]["seq_len"] == 4680
    assert d["clocks"]["samples"] > 0


def test_bench_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference"
    if "unavailable" in d:
        pytest.skip(d["unavailable"])
    assert d["unit"] == "latent frames/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("reference", "port")


def test_bench_two_ranks_spawns_itself():
    """--gpus 2 without torchrun: bench.py launches its two ranks itself (PEER transport; both
    on cuda:0 here, a path check) and rank 0 prints the whole-job line with the exchange."""
    d = _run("--gpus", "2", "--same-device", "--no-cpu-baseline")
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "sp2"
    assert d["config"]["same_device"] is True
    ex = d["exchange"]
    # Ulysses at P = 2: q, k, v, o -- each rank sends half of each (L/2, C) slab to its peer
    assert ex["bytes_per_call_per_rank"] == 4 * (4680 // 2) * 1536 * 2 // 2
    assert d["value"] > 0 and d["e2e"]["value"] > 0
