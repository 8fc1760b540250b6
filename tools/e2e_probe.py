"""End-to-end gap probe: where the e2e chunk time goes beyond the device-timed chunk.

Times, for the Wan chunk at P = 1 (wall clock, synchronised per chunk):
  device   -- spx_engine_generate_block_device, back to back (no sync between chunks)
  dev_sync -- the same with a synchronise after every chunk (launch ramp + sync cost)
  e2e      -- spx_engine_generate_block from pinned host noise to pinned host latents
  h2d/d2h  -- plain pinned copies of one step's noise / one latent

usage: python tools/e2e_probe.py [--chunks K]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06664_b200 import spattn  # noqa: E402
from paper_2603_06664_b200._lib import check, lib, ptr_array  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", type=int, default=10)
    args = ap.parse_args()
    F, Hg, Wg, H, D, layers, steps = 3, 30, 52, 12, 128, 30, 4
    L, C = F * Hg * Wg, H * D
    world = spattn.CommWorld(1, [0])
    cfg = spattn.GenerationConfig(grid_per_block=spattn.GridSpec(F, Hg, Wg), num_blocks=1,
                                  layers=layers, denoise_steps=steps, heads=H, head_dim=D,
                                  world_size=1, seed=0, profile=False)
    eng = spattn.Engine(cfg, world=world)
    noise = torch.randn(steps, L, C, device="cuda").mul_(D ** -0.5).to(torch.bfloat16)
    out = torch.empty(L, C, device="cuda", dtype=torch.bfloat16)
    noise_h = noise.cpu().pin_memory()
    out_h = torch.empty(L, C, dtype=torch.bfloat16).pin_memory()
    nptr, optr = ptr_array([noise.data_ptr()]), ptr_array([out.data_ptr()])

    def sync():
        check(lib().spx_engine_synchronize(eng._h))
        torch.cuda.synchronize()

    def dev():
        check(lib().spx_engine_generate_block_device(eng._h, 0, nptr, optr))

    def e2e():
        check(lib().spx_engine_generate_block(eng._h, 0, noise_h.data_ptr(), out_h.data_ptr()))

    for _ in range(3):
        dev()
        e2e()
    sync()
    res = {}
    t0 = time.perf_counter()
    for _ in range(args.chunks):
        dev()
    sync()
    res["device_ms"] = (time.perf_counter() - t0) / args.chunks * 1e3
    t0 = time.perf_counter()
    for _ in range(args.chunks):
        dev()
        sync()
    res["dev_sync_ms"] = (time.perf_counter() - t0) / args.chunks * 1e3
    t0 = time.perf_counter()
    for _ in range(args.chunks):
        e2e()
    sync()
    res["e2e_ms"] = (time.perf_counter() - t0) / args.chunks * 1e3
    step_h = noise_h[0]
    dst = torch.empty(L, C, device="cuda", dtype=torch.bfloat16)
    for name, fn in (("h2d_step_ms", lambda: dst.copy_(step_h, non_blocking=True)),
                     ("d2h_latent_ms", lambda: out_h.copy_(dst, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        res[name] = (time.perf_counter() - t0) / 20 * 1e3
    res["h2d_GBs"] = step_h.numel() * 2 / res["h2d_step_ms"] / 1e6
    res["d2h_GBs"] = out_h.numel() * 2 / res["d2h_latent_ms"] / 1e6
    print({k: round(v, 3) for k, v in res.items()})




def enqueue_cost():
    """host cost of enqueueing one chunk (GPU idle at the start, no sync inside)"""
    F, Hg, Wg, H, D, layers, steps = 3, 30, 52, 12, 128, 30, 4
    L, C = F * Hg * Wg, H * D
    cfg = spattn.GenerationConfig(grid_per_block=spattn.GridSpec(F, Hg, Wg), num_blocks=1,
                                  layers=layers, denoise_steps=steps, heads=H, head_dim=D,
                                  world_size=1, seed=0, profile=False)
    eng = spattn.Engine(cfg, world=spattn.CommWorld(1, [0]))
    noise = torch.randn(steps, L, C, device="cuda").to(torch.bfloat16)
    out = torch.empty(L, C, device="cuda", dtype=torch.bfloat16)
    nptr, optr = ptr_array([noise.data_ptr()]), ptr_array([out.data_ptr()])
    for _ in range(3):
        check(lib().spx_engine_generate_block_device(eng._h, 0, nptr, optr))
    check(lib().spx_engine_synchronize(eng._h))
    res = []
    for _ in range(5):
        t0 = time.perf_counter()
        check(lib().spx_engine_generate_block_device(eng._h, 0, nptr, optr))
        t1 = time.perf_counter()
        check(lib().spx_engine_synchronize(eng._h))
        t2 = time.perf_counter()
        res.append((round((t1 - t0) * 1e3, 3), round((t2 - t0) * 1e3, 3)))
    print({"enqueue_ms, enqueue+sync_ms": res})


if __name__ == "__main__":
    if "--enqueue" in sys.argv:
        enqueue_cost()
    else:
        main()
