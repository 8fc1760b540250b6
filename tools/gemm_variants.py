"""Time spx_project_tokens for every GEMM tile variant (planner override) on given shapes.
usage: python tools/gemm_variants.py [MxKxN,...]   (default: the Wan O-projection 4680x1536x1536)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06664_b200._lib import check, lib  # noqa: E402
from tools.kbench import stream_handle, timeit  # noqa: E402

NAMES = {-1: "planner", 0: "pair256", 1: "pair128", 2: "single256", 3: "single128", 4: "single192"}
shapes = [tuple(int(v) for v in s.split("x")) for s in
          (sys.argv[1] if len(sys.argv) > 1 else "4680x1536x1536").split(",")]
torch.cuda.set_stream(torch.cuda.Stream())  # graph capture needs a non-default stream
for M, K, N in shapes:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for v in NAMES:
        check(lib().spx_debug_set_gemm_variant(v))
        ms = timeit(lambda: check(lib().spx_project_tokens(x.data_ptr(), w.data_ptr(), y.data_ptr(),
                                                           M, K, N, stream_handle())), 20)
        print(json.dumps({"M": M, "K": K, "N": N, "variant": NAMES[v], "ms": round(ms, 4),
                          "tflops": round(2.0 * M * N * K / ms / 1e9, 1)}), flush=True)
    check(lib().spx_debug_set_gemm_variant(-1))
