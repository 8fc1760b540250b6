"""One C2 chunk through the engine in a chosen mode, for profilers (ncu -k ... python
tools/wan_chunk.py MODE): MODE = ref (reference semantics), wan (QK-RMSNorm + adaLN), full (the
full Wan2.1 block). Device-resident noise, one warm chunk then one profiled chunk."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06664_b200 import spattn  # noqa: E402
from paper_2603_06664_b200._lib import check, lib, ptr_array  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "ref"
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = spattn.GenerationConfig(grid_per_block=spattn.GridSpec(3, 30, 52), num_blocks=1, layers=layers,
                              denoise_steps=4, heads=12, head_dim=128, qk_norm=mode == "wan",
                              adaln=mode == "wan", wan_block=mode == "full")
eng = spattn.Engine(cfg)
noise = (torch.randn(4, 4680, 1536, device="cuda") * 0.088).to(torch.bfloat16)
out = torch.empty(4680, 1536, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    check(lib().spx_engine_generate_block_device(eng._h, 0, ptr_array([noise.data_ptr()]),
                                                 ptr_array([out.data_ptr()])))
check(lib().spx_engine_synchronize(eng._h))
print("chunk ok", mode, layers)
