"""PEER transport (one process per rank, CUDA IPC buffers, device-side flag barriers) on one
B200: every rank is a separate process on cuda:0, the host exchange of buffer handles goes
through torch.distributed (gloo). The reference's invariant -- SP output == P=1 output
(proj/tests/test_sp_attention.cpp:116-130) -- holds bit-exactly, as for the LOCAL transport,
and the ledger equals the LOCAL run's."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _run_ranks(world, tmp_path, window=None, wan=False, mode=None, env=None):
    port = _free_port()
    args = [str(window if window is not None else -1)] + (["wan"] if wan else []) + \
        ([mode] if mode else [])
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "peer_worker.py"), str(r),
                               str(world), str(port), str(tmp_path)] + args,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                              env=dict(os.environ, **(env or {})))
             for r in range(world)]
    logs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(out.decode(errors="replace")[-3000:])
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{logs[r]}"
    if mode == "stall":
        return (tmp_path / "stall.txt").read_text()
    return [np.load(tmp_path / f"rank{r}.npy") for r in range(world)], \
        [np.load(tmp_path / f"stats{r}.npy") for r in range(world)]


@pytest.mark.parametrize("world,window", [(2, None), (4, None), (2, 3), (8, None)])
def test_peer_transport_bit_identical_to_p1(cuda, tmp_path, world, window):
    """P = 8 on H = 4 runs the 4 head groups x 2 query splits partition."""
    import peer_worker
    from paper_2603_06664_b200 import spattn as s

    slices, stats = _run_ranks(world, tmp_path, window)
    got = np.concatenate(slices, axis=1)  # rank-ordered rows of every block
    base = peer_worker.make_engine(s, 1, s.CommWorld(1), window).generate()
    assert got.shape == base.shape
    assert np.array_equal(got, base)
    local = peer_worker.make_engine(s, world, s.CommWorld(world, [0] * world), window)
    local.generate()
    want = local.stats()
    for st in stats:
        assert list(st) == [want[k] for k in sorted(want)]


def test_peer_transport_wan_mode_bit_identical_to_p1(cuda, tmp_path):
    """QK-RMSNorm + adaLN modulation (seeded per layer) over the PEER transport, P = 4."""
    import peer_worker
    from paper_2603_06664_b200 import spattn as s

    slices, _ = _run_ranks(4, tmp_path, wan=True)
    got = np.concatenate(slices, axis=1)
    base = peer_worker.make_engine(s, 1, s.CommWorld(1), None, wan=True).generate()
    assert np.array_equal(got, base)


def test_peer_barrier_times_out_with_collective_error(cuda, tmp_path):
    """A rank that never enters the layer calls: the other rank's device barrier gives up after
    SPX_PEER_TIMEOUT_MS and the engine raises CollectiveError (the reference's behaviour for a
    rank that leaves the collective order, collectives.cpp:42-52, 88-102) instead of hanging."""
    outcome = _run_ranks(2, tmp_path, mode="stall", env={"SPX_PEER_TIMEOUT_MS": "1500"})
    assert outcome.startswith("CollectiveError"), outcome
    assert "rank 1" in outcome
