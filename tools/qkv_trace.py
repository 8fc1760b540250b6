"""Per-tile timeline of the QKV projection with the fused RoPE + pack epilogue inside the
engine (SPX_GEMM_EXPERIMENT=5 traces the rope-epilogue launches only). Reports, per tile, the
MMA main loop (leader CTAs), the epilogue, and whether the MMA of tile i+2 waited on the TMEM
buffer the epilogue of tile i frees. usage: SPX_GEMM_EXPERIMENT=5 SPX_GRAPHS=0 python tools/qkv_trace.py [ref|plain]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_06664_b200 import spattn  # noqa: E402
from paper_2603_06664_b200._lib import check, lib, ptr_array  # noqa: E402

cfg = spattn.GenerationConfig(grid_per_block=spattn.GridSpec(3, 30, 52), num_blocks=1, layers=1,
                              denoise_steps=1, heads=12, head_dim=128)
eng = spattn.Engine(cfg)
noise = (torch.randn(1, 4680, 1536, device="cuda") * 0.088).to(torch.bfloat16)
out = torch.empty(4680, 1536, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    check(lib().spx_engine_generate_block_device(eng._h, 0, ptr_array([noise.data_ptr()]),
                                                 ptr_array([out.data_ptr()])))
check(lib().spx_engine_synchronize(eng._h))
tr = np.zeros(1024 * 64, dtype=np.int64)
check(lib().spx_debug_gemm_trace(tr.ctypes.data, tr.size))
tr = tr.reshape(1024, 16, 4)
live = tr[:, 14, 0] != 0
t = tr[live].astype(np.float64)
n = len(t)
clk = 1.0 / 1900.0
mma, epi, wait = [], [], []
for c in range(n):
    for it in range(14):
        a = t[c, it]
        if a[2] and a[3]:
            epi.append((a[3] - a[2]) * clk)
        if a[0] and a[1]:
            mma.append((a[1] - a[0]) * clk)
        if it + 2 < 14 and t[c, it + 2, 0] and a[3]:
            wait.append((t[c, it + 2, 0] - a[3]) * clk)  # < 0: the MMA started before this epilogue ended?
gs, ge = t[:, 14, 0], t[:, 14, 1]
print(json.dumps({"ctas": n, "span_us": round(float((ge.max() - gs.min()) / 1e3), 2),
                  "mma_per_tile_us(mean,max)": [round(float(np.mean(mma)), 2), round(float(np.max(mma)), 2)] if mma else None,
                  "epilogue_per_tile_us(mean,max)": [round(float(np.mean(epi)), 2), round(float(np.max(epi)), 2)],
                  "mma(i+2)_start_minus_epi(i)_end_us(mean,min)": [round(float(np.mean(wait)), 2), round(float(np.min(wait)), 2)] if wait else None,
                  "tiles_per_cta(max)": int(max(int(((t[c, :14, 3]) != 0).sum()) for c in range(n)))}))
