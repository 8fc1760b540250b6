"""Kernel spans of one Wan-shape chunk (SPX_SPAN_TRACE=1): per-kernel device duration (first
CTA start -> last CTA end, globaltimer) and the gap to the previous kernel, averaged per layer
call. usage: SPX_SPAN_TRACE=1 python tools/span_probe.py [--wan]"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_06664_b200 import spattn  # noqa: E402
from paper_2603_06664_b200._lib import check, lib, ptr_array  # noqa: E402

wan = "--wan" in sys.argv
F, Hg, Wg, H, D, layers, steps = 3, 30, 52, 12, 128, 30, 4
L, C = F * Hg * Wg, H * D
cfg = spattn.GenerationConfig(grid_per_block=spattn.GridSpec(F, Hg, Wg), num_blocks=1, layers=layers,
                              denoise_steps=steps, heads=H, head_dim=D, world_size=1, seed=0,
                              qk_norm=wan, adaln=wan)
eng = spattn.Engine(cfg)
noise = torch.randn(steps, L, C, device="cuda").mul_(D ** -0.5).to(torch.bfloat16)
out = torch.empty(L, C, device="cuda", dtype=torch.bfloat16)


def chunk():
    check(lib().spx_engine_generate_block_device(eng._h, 0, ptr_array([noise.data_ptr()]),
                                                 ptr_array([out.data_ptr()])))


for _ in range(2):
    chunk()
check(lib().spx_engine_synchronize(eng._h))
n0 = ctypes.c_int64()
check(lib().spx_debug_spans(None, 0, ctypes.byref(n0)))
chunk()
check(lib().spx_engine_synchronize(eng._h))
n1 = ctypes.c_int64()
check(lib().spx_debug_spans(None, 0, ctypes.byref(n1)))
buf = np.zeros(2 * n1.value, dtype=np.uint64)
check(lib().spx_debug_spans(buf.ctypes.data, buf.size, ctypes.byref(n1)))
sp = buf.reshape(-1, 2)[n0.value:n1.value].astype(np.float64) / 1e3  # us
names = {3: ["qkv_gemm", "attention", "o_gemm"],
         4: ["qkv_gemm", "k3_norm_rope", "attention", "o_gemm"]}
per = len(sp) // (layers * steps)
dur = sp[:, 1] - sp[:, 0]
gap = np.concatenate([[0.0], sp[1:, 0] - sp[:-1, 1]])
inc = np.concatenate([[0.0], sp[1:, 1] - sp[:-1, 1]])  # last-CTA end to last-CTA end: the kernel's share of the chunk
res = {"kernels_per_call": per, "chunk_span_ms": float((sp[-1, 1] - sp[0, 0]) / 1e3)}
for k in range(per):
    res[names[per][k] if per in names else f"k{k}"] = {"dur_us": round(float(dur[k::per].mean()), 2),
                                              "gap_before_us": round(float(gap[k::per][1:].mean()), 2),
                                              "end_to_end_us": round(float(inc[k::per][1:].mean()), 2)}
print(json.dumps(res))
