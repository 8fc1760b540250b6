"""Per-CTA timeline of one GEMM launch (SPX_GEMM_EXPERIMENT=7: per-tile clock64 marks [mma
start, mma issued, epilogue start, epilogue end], CTA start / prologue end / end, globaltimer
start / end). usage: SPX_GEMM_EXPERIMENT=7 [SPX_GEMM_VARIANT=v] python tools/gemm_timeline.py MxKxN [...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_06664_b200._lib import check, lib  # noqa: E402

assert os.environ.get("SPX_GEMM_EXPERIMENT") == "7", "set SPX_GEMM_EXPERIMENT=7"
for shape in sys.argv[1:]:
    M, K, N = (int(v) for v in shape.split("x"))
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(4):
        check(lib().spx_project_tokens(x.data_ptr(), w.data_ptr(), y.data_ptr(), M, K, N, st))
    torch.cuda.synchronize()
    tr = np.zeros(1024 * 64, dtype=np.int64)
    check(lib().spx_debug_gemm_trace(tr.ctypes.data, tr.size))
    tr = tr.reshape(1024, 16, 4)
    live = tr[:, 14, 0] != 0
    t = tr[live]
    n = len(t)
    clk = 1.0 / 1900.0
    g0 = t[:, 14, 0].min()
    gs, ge = (t[:, 14, 0] - g0) / 1e3, (t[:, 14, 1] - g0) / 1e3
    c0, cpro, cend = t[:, 15, 0], t[:, 15, 1], t[:, 15, 2]
    tiles = [(t[:, i, :] != 0).all(1) for i in range(14)]
    ntile = np.sum(tiles, axis=0)
    first_mma = (t[:, 0, 0] - cpro) * clk
    main0 = (t[:, 0, 1] - t[:, 0, 0]) * clk
    epi0 = (t[:, 0, 3] - t[:, 0, 2]) * clk
    wait_epi0 = (t[:, 0, 2] - t[:, 0, 1]) * clk
    last = ntile - 1
    tail = np.array([(cend[i] - t[i, last[i], 3]) * clk for i in range(n)])
    # the first CTA's marks relative to its start (us): per tile [mma start, mma issued, epi start, epi end]
    seq = [[round(float((t[0, i, k] - c0[0]) * clk), 2) if t[0, i, k] else None for k in range(4)]
           for i in range(int(ntile[0]))]
    print(json.dumps({"cta0_tiles_us": seq, "cta0_prologue_end_us": round(float((cpro[0] - c0[0]) * clk), 2),
                      "cta0_end_us": round(float((cend[0] - c0[0]) * clk), 2)}))
    print(json.dumps({
        "shape": shape, "ctas": n, "span_us": round(float(ge.max()), 2),
        "tiles_per_cta(max)": int(ntile.max()),
        "start_skew_us(max)": round(float(gs.max()), 2),
        "prologue_us": round(float(((cpro - c0) * clk).mean()), 2),
        "prologue_to_first_mma_us": round(float(first_mma.mean()), 2),
        "tile0_mainloop_us": round(float(main0.mean()), 2),
        "tile0_commit_to_epi_us": round(float(wait_epi0.mean()), 2),
        "tile0_epilogue_us": round(float(epi0.mean()), 2),
        "after_last_epi_us": round(float(tail.mean()), 2),
        "cta_us(mean,max)": [round(float((ge - gs).mean()), 2), round(float((ge - gs).max()), 2)],
    }), flush=True)
