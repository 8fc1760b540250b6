"""Per-CTA clock64 timeline of one attention launch (SPX_ATTN_EXPERIMENT=5): marks after the
prologue, end of the softmax loop, partial written (split-KV), CTA end. usage:
SPX_ATTN_EXPERIMENT=5 [SPX_ATTN_SPLITS=s] python tools/attn_trace.py SQxSKVxH"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_06664_b200._lib import check, lib  # noqa: E402

sq, skv, H = (int(v) for v in sys.argv[1].split("x"))
D = 128
q = (torch.randn(1, sq, H, D, device="cuda") * 0.5).to(torch.bfloat16)
k = (torch.randn(1, skv, H, D, device="cuda") * 0.5).to(torch.bfloat16)
v = torch.randn(1, skv, H, D, device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    check(lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 1, sq, skv, H, D, st))
torch.cuda.synchronize()
tr = np.zeros(1024 * 64, dtype=np.int64)
check(lib().spx_debug_gemm_trace(tr.ctypes.data, tr.size))
tr = tr.reshape(1024, 64)[:, :7]
n = int((tr[:, 0] != 0).sum())
t = tr[:n].astype(np.float64) / 1965.0  # us at 1965 MHz (SM clock cycles)
rel = t - t[:, :1]
print(json.dumps({"entry_to_prologue_end_us(mean,max)": [round(float((t[:, 0] - t[:, 4]).mean()), 2),
                                                         round(float((t[:, 0] - t[:, 4]).max()), 2)]}))
print(json.dumps({"shape": sys.argv[1], "ctas": n,
                  "mean_us[loop_end, partial_done, cta_end, entry, counted, merge_loaded]": [round(float(x), 2) for x in
                                                              np.where(tr[:n, 1:] != 0, rel[:, 1:], np.nan).mean(0)],
                  "max_us": [round(float(x), 2) for x in np.nanmax(np.where(tr[:n, 1:] != 0, rel[:, 1:], np.nan), 0)]}))
