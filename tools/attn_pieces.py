"""Per-piece timeline of the v3 attention (SPX_ATTN_EXPERIMENT=5): for each CTA, clock64 marks
after the PDL wait, then per piece its softmax-loop end and epilogue end, and the CTA end;
printed as means over CTAs in us relative to the PDL wait. usage:
SPX_ATTN_EXPERIMENT=5 [SPX_ATTN_TRIPLE=0] python tools/attn_pieces.py SQxSKVxH"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_06664_b200._lib import check, lib  # noqa: E402

for shape in sys.argv[1:]:
    sq, skv, H = (int(v) for v in shape.split("x"))
    D = 128
    q = (torch.randn(1, sq, H, D, device="cuda") * 0.5).to(torch.bfloat16)
    k = (torch.randn(1, skv, H, D, device="cuda") * 0.5).to(torch.bfloat16)
    v = torch.randn(1, skv, H, D, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    st = torch.cuda.current_stream().cuda_stream
    torch.cuda.synchronize()
    tr = np.zeros(1024 * 64, dtype=np.int64)
    check(lib().spx_debug_gemm_trace(tr.ctypes.data, tr.size))  # clear
    for _ in range(2):
        check(lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 1, sq, skv, H, D, st))
        torch.cuda.synchronize()
    check(lib().spx_debug_gemm_trace(tr.ctypes.data, tr.size))
    t = tr.reshape(1024, 64).astype(np.float64)
    t = t[t[:, 0] != 0]
    clk = 1.0 / 1900.0
    out = {"shape": shape, "ctas": len(t)}
    for name, idx in [("piece0_loop_end", 10), ("piece0_epi_end", 20), ("piece1_loop_end", 11),
                      ("piece1_epi_end", 21), ("piece2_loop_end", 12), ("piece2_epi_end", 22), ("cta_end", 3)]:
        m = t[:, idx] != 0
        if m.any():
            out[name] = [round(float(((t[m, idx] - t[m, 0]) * clk).mean()), 2),
                         round(float(((t[m, idx] - t[m, 0]) * clk).max()), 2)]
    print(json.dumps(out), flush=True)
