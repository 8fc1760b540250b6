"""The GPU fp64 oracle (oracle/gpu_oracle.py) pinned to the CPU oracle (oracle/spattn_oracle.cpp,
itself pinned bit-exactly to the reference's checksums in tests/test_oracle.py). Runs on the
CPU (torch float64, device="cpu"): the same code the Wan-shape GPU parity tests run on cuda.
Only the summation order of the matmuls differs, so the bar is 1e-12 relative."""
import numpy as np
import pytest

from oracle import gpu_oracle, oracle

TINY = dict(frames=3, grid_h=8, grid_w=8, num_blocks=3, layers=2, heads=4, head_dim=64)
DESK = dict(frames=3, grid_h=4, grid_w=4, num_blocks=5, layers=4, heads=8, head_dim=16)


def _rel_max(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


@pytest.mark.parametrize("kw,steps,window", [(TINY, 2, None), (TINY, 4, None), (TINY, 2, 3),
                                             (DESK, 2, None), (DESK, 2, 3)])
def test_gpu_oracle_equals_cpu_oracle(kw, steps, window):
    ref = oracle.generate(**kw, steps=steps, window=window)
    m = gpu_oracle.ReferenceModel(**kw, steps=steps, window=window, round_inputs=False, device="cpu")
    got = m.generate().reshape(ref.shape)
    assert _rel_max(got, ref) < 1e-12


def test_gpu_oracle_equals_cpu_oracle_wan_mode():
    """QK-RMSNorm + adaLN modulation + gated residual (the extensions), bf16-rounded inputs."""
    kw = dict(TINY)
    dim = kw["heads"] * kw["head_dim"]
    rng = np.random.default_rng(3)
    w = oracle.round_bf16(rng.standard_normal((kw["layers"], 4, dim, dim)) / np.sqrt(dim))
    mod = rng.standard_normal((kw["layers"], 3, dim)) * 0.3
    nw = 1 + 0.1 * rng.standard_normal((kw["layers"], 2, dim))
    ref = oracle.generate(**kw, steps=2, weights=w, round_inputs=True, qk_norm=True, norm_weights=nw,
                          modulation=mod)
    m = gpu_oracle.ReferenceModel(**kw, steps=2, weights=w, qk_norm=True, norm_weights=nw,
                                  modulation=mod, device="cpu")
    got = m.generate().reshape(ref.shape)
    assert _rel_max(got, ref) < 1e-12


def test_gpu_oracle_fault_injection_matches():
    """force_start_frame_zero (generator.hpp:30-32): block 0 unchanged, later blocks differ,
    exactly as the CPU oracle."""
    kw = dict(TINY, layers=1)
    ref = oracle.generate(**kw, steps=1, force_start_frame_zero=True)
    m = gpu_oracle.ReferenceModel(**kw, steps=1, round_inputs=False, force_start_frame_zero=True,
                                  device="cpu")
    got = m.generate().reshape(ref.shape)
    assert _rel_max(got, ref) < 1e-12
