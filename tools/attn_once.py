"""One spx_attention call at 4680 x 32760 x 12 (D = 128), 4 times: a target for ncu captures."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2603_06664_b200._lib import check, lib
sq, skv, H, D = 4680, 32760, 12, 128
q = (torch.randn(1, sq, H, D, device="cuda") * 0.5).to(torch.bfloat16)
k = (torch.randn(1, skv, H, D, device="cuda") * 0.5).to(torch.bfloat16)
v = torch.randn(1, skv, H, D, device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
for _ in range(4):
    check(lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 1, sq, skv, H, D, torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
