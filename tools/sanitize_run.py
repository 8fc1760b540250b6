"""A small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every
kernel family once at small shapes -- GEMM variants and epilogues, attention v2 / v3 (persistent
over several tiles per CTA, the 2-CTA pair split) / split-KV / small-D, K3 / K1, the engine (P = 1
and 2, Wan mode incl. the fused O-projection + LayerNorm at C = 1536, the Wan block), the
PEER-free paths."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06664_b200 import spattn  # noqa: E402
from paper_2603_06664_b200._lib import check, lib  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
torch.manual_seed(0)
# GEMM: every tile variant, bias / GELU / residual epilogues
for v in range(6):  # 5 = split-K (2-CTA clusters)
    check(lib().spx_debug_set_gemm_variant(v))
    M, K, N = 300, 128, 512
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, device="cuda")
    check(lib().spx_project_tokens_ex(x.data_ptr(), w.data_ptr(), y.data_ptr(), M, K, N, b.data_ptr(), 3,
                                      None, None, st))
    check(lib().spx_project_tokens_ex(x.data_ptr(), w.data_ptr(), y.data_ptr(), M, K, N, None, 1,
                                      y.data_ptr(), b.data_ptr(), st))
check(lib().spx_debug_set_gemm_variant(-1))
torch.cuda.synchronize()
# attention: v2, v3, split-KV (workspace and DSMEM pair), small D
for v3 in (0, 2):
    check(lib().spx_debug_set_attn_v3(v3))
    for sq, skv, H, D in [(256, 640, 2, 128), (130, 300, 1, 64)]:
        q = torch.randn(1, sq, H, D, device="cuda").to(torch.bfloat16)
        k = torch.randn(1, skv, H, D, device="cuda").to(torch.bfloat16)
        o = torch.empty_like(q)
        check(lib().spx_attention(q.data_ptr(), k.data_ptr(), k.data_ptr(), o.data_ptr(), 1, sq, skv, H, D, st))
check(lib().spx_debug_set_attn_v3(1))
for splits in (2, 3):
    check(lib().spx_debug_set_attn_splits(splits))
    q = torch.randn(1, 256, 2, 128, device="cuda").to(torch.bfloat16)
    k = torch.randn(1, 1200, 2, 128, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    check(lib().spx_attention(q.data_ptr(), k.data_ptr(), k.data_ptr(), o.data_ptr(), 1, 256, 1200, 2, 128, st))
check(lib().spx_debug_set_attn_splits(0))
# the persistent v3 with several tiles per CTA (more tiles than SMs)
q = torch.randn(1, 128 * 10, 16, 128, device="cuda").to(torch.bfloat16)
k = torch.randn(1, 256, 16, 128, device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
check(lib().spx_attention(q.data_ptr(), k.data_ptr(), k.data_ptr(), o.data_ptr(), 1, 1280, 256, 16, 128, st))
for D in (16, 32):
    q = torch.randn(1, 48, 8, D, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    check(lib().spx_attention(q.data_ptr(), q.data_ptr(), q.data_ptr(), o.data_ptr(), 1, 48, 48, 8, D, st))
torch.cuda.synchronize()
# engine: reference semantics P = 1, 2 (LOCAL), desk D = 16, Wan mode, the full Wan block
for kw in [dict(heads=4, head_dim=64, world_size=1), dict(heads=4, head_dim=64, world_size=2),
           dict(heads=8, head_dim=16, world_size=2),
           dict(heads=4, head_dim=64, world_size=1, qk_norm=True, adaln=True),
           dict(heads=4, head_dim=64, world_size=1, wan_block=True, text_len=64, text_dim=128)]:
    cfg = spattn.GenerationConfig(grid_per_block=spattn.GridSpec(3, 4, 8), num_blocks=2, layers=2,
                                  denoise_steps=2, **kw)
    spattn.Engine(cfg).generate()
torch.cuda.synchronize()
# Wan mode at C = 1536 with >= 25 row tiles: the O-projection fused with the next layer's
# LayerNorm + modulation (gemm_ln.cu)
cfg = spattn.GenerationConfig(grid_per_block=spattn.GridSpec(3, 32, 32), num_blocks=1, layers=2,
                              denoise_steps=1, heads=12, head_dim=128, qk_norm=True, adaln=True)
spattn.Engine(cfg).generate()
torch.cuda.synchronize()
print("sanitize workload done")
