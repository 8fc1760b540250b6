"""One spx_attention call on random inputs vs an fp32 torch reference (debug helper).
usage: python tools/attn_case.py SQxSKVxHxD"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06664_b200._lib import check, lib  # noqa: E402

sq, skv, H, D = (int(v) for v in sys.argv[1].split("x"))
q = torch.randn(1, sq, H, D, device="cuda").to(torch.bfloat16)
k = torch.randn(1, skv, H, D, device="cuda").to(torch.bfloat16)
v = torch.randn(1, skv, H, D, device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
check(lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 1, sq, skv, H, D,
                          torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
qf, kf, vf = (t.float().transpose(1, 2) for t in (q, k, v))
ref = (torch.softmax(qf @ kf.transpose(-1, -2) / math.sqrt(D), dim=-1) @ vf).transpose(1, 2)
err = float((o.float() - ref).norm() / ref.norm())
print(sys.argv[1], "rel_l2", err, flush=True)
