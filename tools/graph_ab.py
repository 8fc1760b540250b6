"""A/B: per-step CUDA graphs vs launch-by-launch enqueue for the C2 chunk (device time, CUDA
events on the engine stream, alternating 3 x 2 runs of 10 chunks on one engine)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06664_b200 import spattn  # noqa: E402
from paper_2603_06664_b200._lib import check, lib, ptr_array  # noqa: E402

cfg = spattn.GenerationConfig(grid_per_block=spattn.GridSpec(3, 30, 52), num_blocks=1, layers=30,
                              denoise_steps=4, heads=12, head_dim=128)
eng = spattn.Engine(cfg)
noise = (torch.randn(4, 4680, 1536, device="cuda") * 0.088).to(torch.bfloat16)
out = torch.empty(4680, 1536, device="cuda", dtype=torch.bfloat16)
sp = ctypes.c_void_p()
check(lib().spx_world_stream(eng.world._h, 0, ctypes.byref(sp)))
stream = torch.cuda.ExternalStream(sp.value)


def chunk():
    check(lib().spx_engine_generate_block_device(eng._h, 0, ptr_array([noise.data_ptr()]),
                                                 ptr_array([out.data_ptr()])))


for g in (0, 1):
    eng.set_graphs(bool(g))
    for _ in range(3):
        chunk()
check(lib().spx_engine_synchronize(eng._h))
for rep in range(3):
    for g in (0, 1):
        eng.set_graphs(bool(g))
        chunk()
        check(lib().spx_engine_synchronize(eng._h))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(10):
            chunk()
        e1.record(stream)
        check(lib().spx_engine_synchronize(eng._h))
        print(f"rep {rep} graphs {g}: {e0.elapsed_time(e1) / 10:.3f} ms/chunk", flush=True)
