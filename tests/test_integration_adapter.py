"""The reference-side adapter of INTEGRATION.md (integration/spx_adapter.hpp) compiled against
the reference's own headers and sources (integration/Makefile: /root/reference/proj/src
compiled in place, linked with libspx.so) and run: libspx's RoPE tables equal the reference's
precompute_frequencies bit for bit, global_time_index agrees, status codes arrive as the
reference's exception classes; on a GPU the reference's default configuration goes through
spx_adapter::generate and is compared with the reference's own generate()."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


def _binary():
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "integration")], check=True)
    if not os.path.exists(BIN):
        pytest.skip("adapter_check not built (no reference tree here and no prebuilt binary)")
    return BIN


def test_adapter_compiles_against_reference_and_runs_host_calls():
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "adapter ok" in r.stdout
    assert r.stdout.count("ok   rope table") == 3


@pytest.mark.gpu
def test_adapter_generate_matches_reference_generate(cuda):
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("ok   desk generate() P=") == 4, r.stdout
