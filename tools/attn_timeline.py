"""Per-CTA / per-SM timeline of one attention launch (SPX_ATTN_EXPERIMENT=5 marks; globaltimer
for the cross-SM view, clock64 for the in-CTA phases). usage:
SPX_ATTN_EXPERIMENT=5 [SPX_ATTN_SPLITS=s] python tools/attn_timeline.py SQxSKVxH [...]"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_06664_b200._lib import check, lib  # noqa: E402

assert os.environ.get("SPX_ATTN_EXPERIMENT") == "5", "set SPX_ATTN_EXPERIMENT=5"
for shape in sys.argv[1:]:
    sq, skv, H = (int(v) for v in shape.split("x"))
    D = 128
    q = (torch.randn(1, sq, H, D, device="cuda") * 0.5).to(torch.bfloat16)
    k = (torch.randn(1, skv, H, D, device="cuda") * 0.5).to(torch.bfloat16)
    v = torch.randn(1, skv, H, D, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(4):
        check(lib().spx_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 1, sq, skv, H, D, st))
    torch.cuda.synchronize()
    tr = np.zeros(1024 * 64, dtype=np.int64)
    check(lib().spx_debug_gemm_trace(tr.ctypes.data, tr.size))
    tr = tr.reshape(1024, 64)
    live = tr[:, 7] != 0
    t = tr[live]
    n = len(t)
    g0 = t[:, 7].min()
    ent, end = (t[:, 7] - g0) / 1e3, (t[:, 8] - g0) / 1e3  # us
    clk = 1.0 / 1900.0  # us per cycle (approximate SM clock under load)
    pro = (t[:, 0] - t[:, 4]) * clk
    loop = np.where(t[:, 1] != 0, (t[:, 1] - t[:, 0]) * clk, np.nan)
    epi = np.where(t[:, 1] != 0, (t[:, 3] - t[:, 1]) * clk, np.nan)
    by_sm = collections.defaultdict(list)
    for i in range(n):
        by_sm[int(t[i, 9])].append((ent[i], end[i]))
    gaps = []
    for sm, lst in by_sm.items():
        lst.sort()
        for a, b in zip(lst, lst[1:]):
            gaps.append(b[0] - a[1])
    busy = sum(e - s for lst in by_sm.values() for s, e in lst)
    span = float(end.max())
    print(json.dumps({
        "shape": shape, "ctas": n, "sms_used": len(by_sm), "span_us": round(span, 2),
        "cta_us(mean,min,max)": [round(float((end - ent).mean()), 2), round(float((end - ent).min()), 2),
                                  round(float((end - ent).max()), 2)],
        "prologue_us(mean)": round(float(pro.mean()), 2),
        "loop_us(mean)": round(float(np.nanmean(loop)), 2) if np.isfinite(loop).any() else None,
        "epilogue_us(mean)": round(float(np.nanmean(epi)), 2) if np.isfinite(epi).any() else None,
        "gap_between_ctas_us(mean,max)": [round(float(np.mean(gaps)), 2), round(float(np.max(gaps)), 2)] if gaps else None,
        "sm_busy_frac": round(busy / (148 * span), 3),
        "last_start_us": round(float(ent.max()), 2),
    }), flush=True)
