"""Phase timeline of the fused O-projection + LayerNorm/modulation kernel (gemm_ln.cu) inside a
Wan-mode layer call (SPX_GEMM_EXPERIMENT=8). usage: SPX_GEMM_EXPERIMENT=8 SPX_GRAPHS=0 python tools/ln_trace.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_06664_b200 import spattn  # noqa: E402
from paper_2603_06664_b200._lib import check, lib, ptr_array  # noqa: E402

cfg = spattn.GenerationConfig(grid_per_block=spattn.GridSpec(3, 30, 52), num_blocks=1, layers=2,
                              denoise_steps=1, heads=12, head_dim=128, qk_norm=True, adaln=True)
eng = spattn.Engine(cfg)
noise = (torch.randn(1, 4680, 1536, device="cuda") * 0.088).to(torch.bfloat16)
out = torch.empty(4680, 1536, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    check(lib().spx_engine_generate_block_device(eng._h, 0, ptr_array([noise.data_ptr()]),
                                                 ptr_array([out.data_ptr()])))
check(lib().spx_engine_synchronize(eng._h))
tr = np.zeros(1024 * 64, dtype=np.int64)
check(lib().spx_debug_gemm_trace(tr.ctypes.data, tr.size))
t = tr.reshape(1024, 64)[:, :10].astype(np.float64)
t = t[(t[:, 0] != 0) & (t[:, 9] != 0)]
clk = 1.0 / 1900.0
names = ["prologue+pdl", "mainloop", "residual_tma", "pass1", "cluster_sync1", "pass2+sync2", "store_x_new",
         "pass4+store_x_mod", "sync3"]
d = np.diff(t, axis=1) * clk
print(json.dumps({"ctas": len(t), **{n: round(float(d[:, i].mean()), 2) for i, n in enumerate(names)},
                  "total_us(mean,max)": [round(float(((t[:, 9] - t[:, 0]) * clk).mean()), 2),
                                         round(float(((t[:, 9] - t[:, 0]) * clk).max()), 2)]}))
