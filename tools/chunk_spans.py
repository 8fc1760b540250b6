"""Per-chunk device spans over a run of back-to-back C2 chunks (SPX_SPAN_TRACE=1, eager): first
kernel start to last kernel end of each chunk, and the gap between chunks -- does the chunk time
drift under sustained load (power), and how much lies outside the kernels?
usage: SPX_SPAN_TRACE=1 python tools/chunk_spans.py [chunks]"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_06664_b200 import spattn  # noqa: E402
from paper_2603_06664_b200._lib import check, lib, ptr_array  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = spattn.GenerationConfig(grid_per_block=spattn.GridSpec(3, 30, 52), num_blocks=1, layers=30,
                              denoise_steps=4, heads=12, head_dim=128)
eng = spattn.Engine(cfg)
noise = (torch.randn(4, 4680, 1536, device="cuda") * 0.088).to(torch.bfloat16)
out = torch.empty(4680, 1536, device="cuda", dtype=torch.bfloat16)
sp = ctypes.c_void_p()
check(lib().spx_world_stream(eng.world._h, 0, ctypes.byref(sp)))
stream = torch.cuda.ExternalStream(sp.value)


def chunk():
    check(lib().spx_engine_generate_block_device(eng._h, 0, ptr_array([noise.data_ptr()]),
                                                 ptr_array([out.data_ptr()])))


for _ in range(3):
    chunk()
check(lib().spx_engine_synchronize(eng._h))
c0 = ctypes.c_int64()
check(lib().spx_debug_spans(None, 0, ctypes.byref(c0)))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(n):
    chunk()
e1.record(stream)
check(lib().spx_engine_synchronize(eng._h))
c1 = ctypes.c_int64()
check(lib().spx_debug_spans(None, 0, ctypes.byref(c1)))
buf = np.zeros(2 * c1.value, dtype=np.uint64)
check(lib().spx_debug_spans(buf.ctypes.data, buf.size, ctypes.byref(c1)))
s = buf.reshape(-1, 2)[c0.value:c1.value].astype(np.float64) / 1e6  # ms
per = len(s) // n
spans = [float(s[(k + 1) * per - 1, 1] - s[k * per, 0]) for k in range(n)]
gaps = [float(s[(k + 1) * per, 0] - s[(k + 1) * per - 1, 1]) for k in range(n - 1)]
busy = float(np.sum(s[:, 1] - s[:, 0]))
print(json.dumps({"chunks": n, "kernels_per_chunk": per, "event_ms_per_chunk": e0.elapsed_time(e1) / n,
                  "span_ms": [round(x, 3) for x in spans], "gap_between_chunks_ms": [round(x, 3) for x in gaps]}))
