"""Per-tile timeline of the last GEMM of a Wan-mode layer call (the O-projection with the
gated residual epilogue) inside the engine (SPX_GEMM_EXPERIMENT=7 traces every GEMM launch; the
buffer keeps the last one). usage: SPX_GEMM_EXPERIMENT=7 SPX_GRAPHS=0 python tools/oproj_trace.py [wan|ref]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_06664_b200 import spattn  # noqa: E402
from paper_2603_06664_b200._lib import check, lib, ptr_array  # noqa: E402

wan = (sys.argv[1] if len(sys.argv) > 1 else "wan") == "wan"
cfg = spattn.GenerationConfig(grid_per_block=spattn.GridSpec(3, 30, 52), num_blocks=1, layers=2,
                              denoise_steps=1, heads=12, head_dim=128, qk_norm=wan, adaln=wan)
eng = spattn.Engine(cfg)
noise = (torch.randn(1, 4680, 1536, device="cuda") * 0.088).to(torch.bfloat16)
out = torch.empty(4680, 1536, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    check(lib().spx_engine_generate_block_device(eng._h, 0, ptr_array([noise.data_ptr()]),
                                                 ptr_array([out.data_ptr()])))
check(lib().spx_engine_synchronize(eng._h))
tr = np.zeros(1024 * 64, dtype=np.int64)
check(lib().spx_debug_gemm_trace(tr.ctypes.data, tr.size))
t = tr.reshape(1024, 16, 4)
t = t[t[:, 14, 0] != 0].astype(np.float64)
clk = 1.0 / 1900.0
c0 = t[:, 15, 0]
gs, ge = (t[:, 14, 0] - t[:, 14, 0].min()) / 1e3, (t[:, 14, 1] - t[:, 14, 0].min()) / 1e3
seq = [[round(float((t[0, i, k] - c0[0]) * clk), 2) for k in range(4)] for i in range(3) if t[0, i, 3]]
mma = [(t[c, i, 1] - t[c, i, 0]) * clk for c in range(len(t)) for i in range(3) if t[c, i, 1]]
epi = [(t[c, i, 3] - t[c, i, 2]) * clk for c in range(len(t)) for i in range(3) if t[c, i, 3]]
print(json.dumps({"mode": "wan" if wan else "ref", "ctas": len(t), "span_us": round(float(ge.max()), 2),
                  "start_skew_us": round(float(gs.max()), 2),
                  "prologue_us(mean)": round(float(((t[:, 15, 1] - c0) * clk).mean()), 2),
                  "mma_per_tile_us(mean,max)": [round(float(np.mean(mma)), 2), round(float(np.max(mma)), 2)],
                  "epilogue_per_tile_us(mean,max)": [round(float(np.mean(epi)), 2), round(float(np.max(epi)), 2)],
                  "cta0_tiles_us": seq, "cta_us(mean,max)": [round(float((ge - gs).mean()), 2), round(float((ge - gs).max()), 2)]}))
