"""CPU tests of the C-ABI boundary and the host-side logic (no kernel launches).

* libspx.so loads on a machine without a GPU and exports every function include/spx.h
  declares (and the ctypes table binds exactly those);
* host functions of the library (reference RNG, seeded weights, bf16 rounding, RoPE table,
  time index, config validation) agree bit-exactly with the oracle / reference goldens.
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spx.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spx_[a-z0-9_]+)\s*\(", text)))


def lib():
    from paper_2603_06664_b200._lib import lib as _l

    return _l()


def test_library_loads_without_gpu():
    assert lib().spx_abi_version() == 1


def test_every_declared_symbol_is_exported():
    funcs = header_functions()
    assert len(funcs) > 50
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2603_06664_b200", "libspx.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (spx_\w+)", out))
    missing = [f for f in funcs if f not in exported]
    assert not missing, missing


def test_ctypes_table_matches_header():
    from paper_2603_06664_b200._lib import EXPORTED

    assert sorted(EXPORTED) == header_functions()


def test_status_names_cover_reference_errors():
    names = [lib().spx_status_name(i).decode() for i in range(11)]
    assert names[1:8] == ["ShapeError", "PartitionError", "ConfigError", "RangeError", "AlignmentError",
                          "EmptyCacheError", "CollectiveError"]


def test_derive_seed_and_noise_match_oracle():
    l = lib()
    for args in [(0, 0x10, 0, 0), (0, 0x20, 0, 0), (7, 3, 2, 1)]:
        assert l.spx_derive_seed(*args) == oracle.derive_seed(*args)
    n = 4 * 8 * 8 * 4 * 64
    got = np.empty(n)
    assert l.spx_block_noise(0, 1, 3, n, 64, got.ctypes.data_as(ctypes.POINTER(ctypes.c_double))) == 0
    ref = oracle.block_noise(0, 1, 3, (n // 64, 64))
    assert np.array_equal(got, ref.reshape(-1))


def test_seeded_weights_match_oracle():
    dim = 64
    w = [np.empty((dim, dim)) for _ in range(4)]
    ptrs = [a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for a in w]
    assert lib().spx_layer_weights(0, 3, dim, *ptrs) == 0
    ref = oracle.layer_weights(0, 3, dim)
    for m in range(4):
        assert np.array_equal(w[m], ref[m])


def test_bf16_rounding_matches_oracle():
    from paper_2603_06664_b200.spattn import bf16_bits_to_float, float_to_bf16_bits

    x = np.concatenate([np.random.default_rng(0).standard_normal(5000) * s for s in (1e-3, 0.1, 10.0)])
    x = np.concatenate([x, [0.0, -0.0, 1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8)]])
    got = bf16_bits_to_float(float_to_bf16_bits(x))
    assert np.array_equal(got, oracle.round_bf16(x))


def test_rope_table_host_values_bit_exact():
    from paper_2603_06664_b200 import spattn

    t = spattn.precompute_frequencies(21, 30, 52, 128)
    assert t.split() == spattn.BandSplit(22, 21, 21)
    assert t.cos_at(0, 1, 1) == 0.79125771813778545 and t.sin_at(0, 1, 1) == 0.61148280718870973
    assert t.cos_at(1, 29, 20) == 0.99998989077996614
    for band, pos, pair in [(0, 20, 21), (1, 3, 0), (2, 51, 20), (2, 0, 5)]:
        c, s = oracle.table_at(128, band, pos, pair)
        assert (t.cos_at(band, pos, pair), t.sin_at(band, pos, pair)) == (c, s)


def test_rope_table_errors():
    from paper_2603_06664_b200 import spattn

    with pytest.raises(spattn.ConfigError):
        spattn.precompute_frequencies(3, 4, 4, 15)  # odd head_dim
    with pytest.raises(spattn.ConfigError):
        spattn.precompute_frequencies(0, 4, 4, 16)
    with pytest.raises(spattn.ConfigError):
        spattn.precompute_frequencies(3, 4, 4, 16, base=-1.0)
    with pytest.raises(spattn.RangeError):
        spattn.precompute_frequencies(3, 4, 4, 16).cos_at(0, 3, 0)


def test_global_time_index_matches_oracle():
    from paper_2603_06664_b200 import spattn

    rng = np.random.default_rng(0)
    for _ in range(200):
        P = int(rng.choice([1, 2, 4, 8]))
        hw = int(rng.integers(1, 2000))
        F = int(rng.integers(1, 4))
        Lp = (F * hw * P) // P
        i = int(rng.integers(0, Lp))
        r = int(rng.integers(0, P))
        s = int(rng.integers(0, 300))
        assert spattn.global_time_index(i, r, Lp, hw, s) == oracle.global_time_index(i, r, Lp, hw, s)


def test_config_validation_mirrors_reference():
    from paper_2603_06664_b200 import spattn

    wan = dict(grid_per_block=spattn.GridSpec(3, 30, 52), heads=12, head_dim=128, layers=30)
    for P in (1, 2, 4, 8):  # P = 8 with H = 12 runs 4 head groups x 2 query splits
        spattn.GenerationConfig(world_size=P, **wan).validate()
    with pytest.raises(spattn.PartitionError):
        spattn.GenerationConfig(world_size=7, **wan).validate()  # 4680 % 7 != 0
    with pytest.raises(spattn.ConfigError):
        spattn.GenerationConfig(layers=0, **{k: v for k, v in wan.items() if k != "layers"}).validate()
    with pytest.raises(spattn.ConfigError):
        spattn.GenerationConfig(window_frames=2, **wan).validate()  # window < tau
    with pytest.raises(spattn.ShapeError):
        spattn.GenerationConfig(grid_per_block=spattn.GridSpec(0, 4, 4), heads=4, head_dim=64).validate()
    spattn.GenerationConfig().validate()  # reference default D = 16: SIMT attention path
    with pytest.raises(spattn.UnsupportedError):
        spattn.GenerationConfig(head_dim=24, heads=8).validate()  # D must divide 256
    with pytest.raises(spattn.UnsupportedError):
        spattn.GenerationConfig(wan_block=True).validate()  # the full block needs D >= 64


def test_checksum_matches_reference_report_format():
    """spx_checksum_f64 == tensor_checksum (report.cpp:264-279): the C1 tiny P=1 output of the
    pinned oracle hashes to the reference's published block-0 checksum."""
    import numpy as np

    from oracle import oracle
    from paper_2603_06664_b200 import spattn

    x = np.random.default_rng(0).standard_normal((5, 7))
    assert spattn.tensor_checksum(x) == oracle.checksum(x)
    out = oracle.generate(frames=3, grid_h=8, grid_w=8, num_blocks=1, layers=2, steps=2, heads=4,
                          head_dim=64)
    assert spattn.tensor_checksum(out[0]) == "ca4d9813b02c388e"
