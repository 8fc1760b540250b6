"""One attention case against fp32 (debug): usage: python tools/attn_case2.py SQxSKVxH [v3flag]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06664_b200._lib import check, lib  # noqa: E402

sq, skv, H = (int(v) for v in sys.argv[1].split("x"))
if len(sys.argv) > 2:
    check(lib().spx_debug_set_attn_v3(int(sys.argv[2])))
D = 128
g = torch.Generator(device="cuda").manual_seed(sq + skv + H)
q = torch.randn(1, sq, H, D, device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn(1, skv, H, D, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(1, skv, H, D, device="cuda", generator=g).to(torch.bfloat16)
o = torch.empty_like(q)
check(lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 1, sq, skv, H, D,
                          torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
qf, kf, vf = (t.float().transpose(1, 2) for t in (q, k, v))
ref = (torch.softmax(qf @ kf.transpose(-1, -2) / math.sqrt(D), dim=-1) @ vf).transpose(1, 2)
of = o.float()
bad = ~torch.isfinite(of)
print(sys.argv[1:], "rel_l2", float((of - ref).norm() / ref.norm()), "nonfinite", int(bad.sum()),
      "bad rows (first)", torch.nonzero(bad.any(-1).any(-1)[0])[:5].flatten().tolist(),
      "bad heads", torch.nonzero(bad.any(-1).any(1)[0]).flatten().tolist())
