"""Hang/race stress for the attention and GEMM kernels: many launches over many shapes,
each synchronised under a watchdog (prints the last shape before a hang)."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_06664_b200._lib import check, lib  # noqa: E402

last = {"shape": None, "t": time.time()}


def watchdog():
    while True:
        time.sleep(5)
        if time.time() - last["t"] > 30:
            print("HANG at", last["shape"], flush=True)
            os._exit(3)


threading.Thread(target=watchdog, daemon=True).start()
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
shapes = [(192, 192, 4, 64), (4680, 4680, 12, 128), (2340, 4680, 3, 128), (128, 128, 2, 128),
          (100, 60, 1, 128), (300, 1000, 2, 64), (1170, 9360, 3, 128), (585, 4680, 6, 128)]
s = torch.cuda.current_stream().cuda_stream
for it in range(iters):
    sq, skv, H, D = shapes[it % len(shapes)]
    q = torch.randn(1, sq, H, D, device="cuda").to(torch.bfloat16)
    k = torch.randn(1, skv, H, D, device="cuda").to(torch.bfloat16)
    v = torch.randn(1, skv, H, D, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    last["shape"] = ("attn", sq, skv, H, D, it)
    for _ in range(5):
        check(lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 1, sq, skv, H, D, s))
    torch.cuda.synchronize()
    last["t"] = time.time()
    assert torch.isfinite(o.float()).all(), ("nonfinite", last["shape"])
print("stress ok", iters, flush=True)
