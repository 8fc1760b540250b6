"""One rank of a PEER-transport run (spawned by tests/test_gpu_peer.py; also usable by hand):
the engine's exchange buffers are mapped between processes through CUDA IPC and the
Causal-RoPE SP schedule runs with device-side flag barriers. Several ranks may share one
GPU (the driver time-slices their contexts), which is how the multi-process path is tested
on a single B200.

usage: python tests/peer_worker.py RANK WORLD PORT OUT_DIR [window_frames|-1] [wan|stall]
  stall: ranks > 0 map the buffers and then never enter the layer calls; rank 0 must get a
         CollectiveError from the bounded PEER barrier (SPX_PEER_TIMEOUT_MS) instead of hanging
"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TINY = dict(frames=3, grid_h=8, grid_w=8, num_blocks=3, layers=2, heads=4, head_dim=64)


def scaled_weights(dim, layers, scale_qk, seed):
    from oracle import oracle

    rng = np.random.default_rng(seed)
    w = rng.standard_normal((layers, 4, dim, dim)) / math.sqrt(dim)
    w[:, 0:2] *= scale_qk
    return oracle.round_bf16(w)


def make_engine(s, world_size, world, window=None, wan=False):
    from oracle import oracle

    kw = TINY
    cfg = s.GenerationConfig(grid_per_block=s.GridSpec(kw["frames"], kw["grid_h"], kw["grid_w"]),
                             num_blocks=kw["num_blocks"], layers=kw["layers"], denoise_steps=2,
                             heads=kw["heads"], head_dim=kw["head_dim"], world_size=world_size,
                             window_frames=window, qk_norm=wan, adaln=wan)
    w = scaled_weights(kw["heads"] * kw["head_dim"], kw["layers"], 1.0 if wan else 4.0, seed=7)
    eng = s.Engine(cfg, world=world, seed_weights=False)
    for l in range(cfg.layers):
        eng.set_layer_weights_bits(l, *[oracle.to_bf16_bits(w[l, m]) for m in range(4)])
        if wan:  # non-trivial adaLN modulation (zero would make every layer the identity)
            m = (np.random.default_rng(100 + l).standard_normal((3, kw["heads"] * kw["head_dim"])) * 0.3)
            eng.set_modulation(l, *m.astype(np.float32))
    return eng


def main():
    rank, world_size, port, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    window = int(sys.argv[5]) if len(sys.argv) > 5 and int(sys.argv[5]) > 0 else None
    wan = len(sys.argv) > 6 and sys.argv[6] == "wan"
    stall = len(sys.argv) > 6 and sys.argv[6] == "stall"
    import torch
    import torch.distributed as dist

    from paper_2603_06664_b200 import spattn as s

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world_size)
    world = s.CommWorld.peer(rank, world_size, 0)
    eng = make_engine(s, world_size, world, window, wan)
    eng.connect_peers(dist.all_gather_object)
    if stall:
        if rank == 0:
            try:
                eng.generate()
                outcome = "no error"
            except s.CollectiveError as e:
                outcome = "CollectiveError: " + str(e)
            with open(os.path.join(out, "stall.txt"), "w") as f:
                f.write(outcome)
        dist.barrier()
        del eng
        dist.destroy_process_group()
        return
    got = eng.generate()  # (blocks, L/P rows of this rank, H, D) bf16 bits
    np.save(os.path.join(out, f"rank{rank}.npy"), got)
    stats = eng.stats()
    np.save(os.path.join(out, f"stats{rank}.npy"),
            np.array([stats[k] for k in sorted(stats)], dtype=np.int64))
    dist.barrier()  # every peer is done reading this rank's buffers before they are freed
    del eng
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
