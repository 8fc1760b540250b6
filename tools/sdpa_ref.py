"""Library attention on the same shapes (context for the attention roofline): torch SDPA with
the cuDNN and flash backends, bf16, B=1. Device time from CUDA-graph-captured launches."""
import json
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel


def timeit(fn, iters=20):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(iters):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for sq, skv, H in [(4680, 4680, 12), (4680, 32760, 12)]:
    q = torch.randn(1, H, sq, 128, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(1, H, skv, 128, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(1, H, skv, 128, device="cuda", dtype=torch.bfloat16)
    for name, be in [("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                     ("efficient", SDPBackend.EFFICIENT_ATTENTION)]:
        try:
            with sdpa_kernel([be]):
                ms = timeit(lambda: F.scaled_dot_product_attention(q, k, v))
            tf = 4.0 * sq * skv * H * 128 / (ms * 1e-3) / 1e12
            print(json.dumps({"backend": name, "sq": sq, "skv": skv, "heads": H, "ms": round(ms, 4),
                              "tflops": round(tf, 1)}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"backend": name, "error": str(e)[:200]}), flush=True)
