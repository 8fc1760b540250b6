"""Multi-process CPU test of the N > 1 (NCCL) exchange schedule, with gloo standing in for NCCL.

Each process is one rank. It packs its q/k/v slabs exactly as the fused K3 kernel does on the
NCCL transport (per head-group slabs of its L/P rows), stores its self-destined part in place,
then executes the transfer list the library's engine executes (spx_exchange_plan, the same
list run_plan() posts inside one ncclGroupStart/End) with gloo isend/irecv, and checks the
result against the reference permutation semantics (proj/src/collectives.cpp:203-276):
q/KV-ring rows (i * L/P + s) of rank (p, g) hold source i's rows s for the heads of group g,
and the output exchange returns each source's rows. Covers Ulysses (P | H) and the
head-group x query-split partition (P = 8, H = 12).
"""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _plan(which, rank, P, H, L, D, base):
    from paper_2603_06664_b200._lib import check, lib

    out = (ctypes.c_int64 * (6 * 256))()
    n = ctypes.c_int64()
    check(lib().spx_exchange_plan(which, rank, P, H, L, D, base, out, 256, ctypes.byref(n)))
    return [tuple(out[6 * i:6 * i + 5]) for i in range(n.value)]


def _partition(P, H, L, D):
    from paper_2603_06664_b200._lib import check, lib

    out = (ctypes.c_int64 * 5)()
    check(lib().spx_partition(P, H, L, D, out))
    return tuple(out)


def _source_tensor(i, which, Lp, H, D):
    # unique, exactly representable values: (source, tensor, row, head, dim)
    s = np.arange(Lp)[:, None, None]
    h = np.arange(H)[None, :, None]
    d = np.arange(D)[None, None, :]
    return (i * 1e6 + which * 1e5 + s * 1e3 + h * 10 + d * 0.5).astype(np.float64)


def _worker(rank, P, H, L, D, port, ring_frames_rows, base_row, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        G, S, Lp, Lq, Hl = _partition(P, H, L, D)
        g, p = rank % G, rank // G
        slab = Lp * Hl * D
        src = {w: _source_tensor(rank, w, Lp, H, D) for w in range(3)}
        bufs = {b: None for b in range(8)}
        # K3 pack (NCCL transport): slab per head group, row-major (L/P, H/G, D)
        for w, b in ((0, 0), (1, 1), (2, 2)):
            bufs[b] = np.concatenate([src[w][:, gg * Hl:(gg + 1) * Hl].reshape(-1) for gg in range(G)])
        bufs[4] = np.full(Lq * Hl * D, np.nan)
        ring_rows = ring_frames_rows
        bufs[5] = np.full(ring_rows * Hl * D, np.nan)
        bufs[6] = np.full(ring_rows * Hl * D, np.nan)
        # self part stored in place by K3
        bufs[4][(rank % G) * slab:(rank % G + 1) * slab] = bufs[0][g * slab:(g + 1) * slab]
        r0 = (base_row + rank * Lp) * Hl * D
        bufs[5][r0:r0 + slab] = bufs[1][g * slab:(g + 1) * slab]
        bufs[6][r0:r0 + slab] = bufs[2][g * slab:(g + 1) * slab]

        def run(plan):
            tens = {b: torch.from_numpy(bufs[b]) for b in bufs if bufs[b] is not None}
            reqs = []
            for peer, is_send, b, off, n in plan:
                view = tens[b][off:off + n]
                reqs.append(dist.isend(view.contiguous(), peer) if is_send else ("recv", b, off, n, peer))
            # post receives into temporaries in list order, then copy back
            pend = []
            for item in reqs:
                if isinstance(item, tuple):
                    _, b, off, n, peer = item
                    t = torch.empty(n, dtype=torch.float64)
                    pend.append((dist.irecv(t, peer), b, off, n, t))
            for item in reqs:
                if not isinstance(item, tuple):
                    item.wait()
            for req, b, off, n, t in pend:
                req.wait()
                bufs[b][off:off + n] = t.numpy()

        run(_plan(0, rank, P, H, L, D, base_row))

        # check q / ring against the permutation formula
        q = bufs[4].reshape(Lq, Hl, D)
        for c in range(G):
            i = p * G + c
            expect = _source_tensor(i, 0, Lp, H, D)[:, g * Hl:(g + 1) * Hl]
            assert np.array_equal(q[c * Lp:(c + 1) * Lp], expect), (rank, i)
        ring_k = bufs[5].reshape(ring_rows, Hl, D)
        ring_v = bufs[6].reshape(ring_rows, Hl, D)
        for i in range(P):
            rows = slice(base_row + i * Lp, base_row + (i + 1) * Lp)
            assert np.array_equal(ring_k[rows], _source_tensor(i, 1, Lp, H, D)[:, g * Hl:(g + 1) * Hl])
            assert np.array_equal(ring_v[rows], _source_tensor(i, 2, Lp, H, D)[:, g * Hl:(g + 1) * Hl])

        # output exchange: this rank's attention rows (split p, group g) back to their sources
        o = q * 2.0 + 1.0  # stand-in attention output (Lq, Hl, D), same row ownership as q
        bufs[3] = np.concatenate([o[c * Lp:(c + 1) * Lp].reshape(-1) for c in range(G)])
        bufs[7] = np.full(G * slab, np.nan)
        bufs[7][g * slab:(g + 1) * slab] = bufs[3][(rank % G) * slab:(rank % G + 1) * slab]
        run(_plan(1, rank, P, H, L, D, base_row))
        orecv = bufs[7].reshape(G, Lp, Hl, D)
        mine = _source_tensor(rank, 0, Lp, H, D) * 2.0 + 1.0
        for gg in range(G):
            assert np.array_equal(orecv[gg], mine[:, gg * Hl:(gg + 1) * Hl]), (rank, gg)
        q_out.put((rank, "ok"))
    except Exception as e:  # surfaced to the parent
        q_out.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P,H,L,D", [(2, 4, 48, 8), (4, 8, 48, 4), (8, 12, 96, 4), (4, 12, 48, 4)])
def test_exchange_plan_realizes_reference_permutation(P, H, L, D):
    base_row = 2 * L  # the block sits in the third block slot of the ring
    ring_rows = 4 * L
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, H, L, D, port, ring_rows, base_row, q)) for r in range(P)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=120) for _ in range(P))
    for pr in procs:
        pr.join(timeout=60)
    assert all(v == "ok" for v in results.values()), results


def test_partition_rules():
    assert _partition(1, 12, 4680, 128) == (1, 1, 4680, 4680, 12)
    assert _partition(2, 12, 4680, 128) == (2, 1, 2340, 4680, 6)
    assert _partition(4, 12, 4680, 128) == (4, 1, 1170, 4680, 3)
    assert _partition(8, 12, 4680, 128) == (4, 2, 585, 2340, 3)  # SURVEY 8e scheme R


def test_plan_ledger_counts_match_reference_formula():
    # Ulysses: per call 3 (P-1) E/P (fused) + (P-1) E/P (output), E = L*H*D per rank-block
    for P in (2, 4):
        L, H, D = 48, 8, 4
        _, _, Lp, _, Hl = _partition(P, H, L, D)
        sent = sum(n for r in range(P) for (_, s, _, _, n) in _plan(0, r, P, H, L, D, 0) if s)
        assert sent == 3 * (P - 1) * L * H * D // P
        sent_o = sum(n for r in range(P) for (_, s, _, _, n) in _plan(1, r, P, H, L, D, 0) if s)
        assert sent_o == (P - 1) * L * H * D // P
